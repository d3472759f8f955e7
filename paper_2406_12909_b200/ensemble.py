"""GPU ensemble inference over GFMP checkpoints (ensemble.py:121-186).

``ensemble_predict`` builds ONE device batch (CSR/CSC on the device), runs
each member's forward pass through the sm_100a kernels into a stacked
(K, B) / (K, N, 3) device buffer, and reduces the member spread on the
device -- population sigma (divide by K, exactly 0 where all members agree
bitwise) and the per-structure force-sigma reduction (max | mean | l2).
Only the (B,) results come back to the host, as numpy like the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import ConfigError, ValidationError
from .model import ModelParams, forward_batch, make_batch

FORCE_REDUCTIONS = ("max", "mean", "l2")  # ensemble.py:27


@dataclass
class EnsemblePrediction:
    """ensemble.py:151-156."""
    energy_mean: np.ndarray   # (G,)
    energy_sigma: np.ndarray  # (G,)
    force_sigma: np.ndarray   # (G,) reduced per structure
    member_count: int


def population_sigma(stack: torch.Tensor, dim: int = 0) -> torch.Tensor:
    """ensemble.py:121-130: sqrt(mean((x - mean)^2)) over ``dim``; entries
    whose members agree bitwise are exactly 0."""
    sigma = stack.std(dim=dim, correction=0)
    spread = stack.amax(dim=dim) - stack.amin(dim=dim)
    return torch.where(spread == 0, torch.zeros_like(sigma), sigma)


def reduce_force_sigma(sigma_comp: torch.Tensor, graph_of_node: torch.Tensor,
                       n_graphs: int, how: str = "max") -> torch.Tensor:
    """ensemble.py:133-148 as a segmented reduction over each structure's
    3·n components (structures are contiguous node ranges)."""
    if how not in FORCE_REDUCTIONS:
        raise ConfigError(f"force reduction must be one of {FORCE_REDUCTIONS}")
    idx = graph_of_node.long()
    out = torch.zeros(n_graphs, dtype=sigma_comp.dtype, device=sigma_comp.device)
    if how == "max":
        return out.scatter_reduce_(0, idx, sigma_comp.amax(dim=1), "amax", include_self=False)
    count = torch.zeros_like(out).index_add_(0, idx, torch.full_like(sigma_comp[:, 0], 3.0))
    if how == "mean":
        return out.index_add_(0, idx, sigma_comp.sum(dim=1)) / count
    return torch.sqrt(out.index_add_(0, idx, (sigma_comp * sigma_comp).sum(dim=1)) / count)


def ensemble_predict(members, records, force_reduction: str = "max", device=None,
                     dtype=torch.float64) -> EnsemblePrediction:
    """ensemble.py:159-186.  ``members``: checkpoints (``model_config`` +
    reference-order ``flat``), e.g. from ``train.load_checkpoint``.  Float64
    by default (the reference's arithmetic); float32 for throughput."""
    members = list(members)
    if not members:
        raise ValidationError("ensemble needs at least one member")
    if force_reduction not in FORCE_REDUCTIONS:
        raise ConfigError(f"force reduction must be one of {FORCE_REDUCTIONS}")
    batch = make_batch(list(records), device=device, dtype=dtype)
    B, N = batch.n_graphs, batch.n_nodes
    e_stack = torch.empty(len(members), B, dtype=dtype, device=batch.device)
    f_stack = torch.empty(len(members), N, 3, dtype=dtype, device=batch.device)
    for i, member in enumerate(members):
        params = ModelParams.from_flat(member.model_config, member.flat, device=batch.device,
                                       dtype=dtype)
        e_stack[i], f_stack[i] = forward_batch(params, batch)
    f_sigma = reduce_force_sigma(population_sigma(f_stack), batch.graph_of_node, B,
                                 force_reduction)
    return EnsemblePrediction(
        energy_mean=e_stack.mean(dim=0).cpu().numpy().astype(np.float64),
        energy_sigma=population_sigma(e_stack).cpu().numpy().astype(np.float64),
        force_sigma=f_sigma.cpu().numpy().astype(np.float64),
        member_count=len(members))
