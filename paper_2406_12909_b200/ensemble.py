"""GPU ensemble inference over GFMP checkpoints (ensemble.py:121-186).

``ensemble_predict`` builds ONE device batch (CSR/CSC on the device), runs
each member's forward pass through the sm_100a kernels into a stacked
(K, B) / (K, N, 3) device buffer, and reduces the member spread on the
device in numpy's float64 operation order -- mean and population sigma
(divide by K, exactly 0 where all members agree bitwise; gfm_member_stats)
and the per-structure force-sigma reduction (max | mean | l2 with numpy's
pairwise sums; gfm_force_sigma_reduce) -- so they are bit-identical to the
reference's for identical member predictions.
Only the (B,) results come back to the host, as numpy like the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_handle
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


def population_sigma(stack: torch.Tensor) -> torch.Tensor:
    """ensemble.py:121-130 over the member axis 0 of a device stack: numpy's
    std (ddof 0) in its float64 operation order (gfm_member_stats); entries
    whose members agree bitwise are exactly 0."""
    _, sigma = member_stats(stack, want_mean=False)
    return sigma


def member_stats(stack: torch.Tensor, want_mean: bool = True):
    """(mean, population sigma) over axis 0 of a (K, ...) device stack, one
    kernel, numpy's order (sum over members in member order, / K)."""
    if not stack.is_cuda:
        raise ValidationError("member_stats needs a device tensor")
    stack = stack.contiguous()
    K = int(stack.shape[0])
    n = stack[0].numel()
    mean = torch.empty(stack.shape[1:], dtype=stack.dtype, device=stack.device) \
        if want_mean else None
    sigma = torch.empty(stack.shape[1:], dtype=stack.dtype, device=stack.device)
    call("gfm_member_stats", ptr(stack), K, n, ptr(mean), ptr(sigma),
         _lib.dtype_code(stack.dtype), stream_handle())
    return mean, sigma


def reduce_force_sigma(sigma_comp: torch.Tensor, node_offsets: torch.Tensor,
                       how: str = "max") -> torch.Tensor:
    """ensemble.py:133-148: each structure's (n, 3) block of component
    spreads -> max | mean | rms (numpy's pairwise sums), one thread per
    structure (gfm_force_sigma_reduce).  ``node_offsets``: device int32
    (B + 1,), structures contiguous."""
    if how not in FORCE_REDUCTIONS:
        raise ConfigError(f"force reduction must be one of {FORCE_REDUCTIONS}")
    B = int(node_offsets.shape[0]) - 1
    out = torch.empty(max(B, 0), dtype=sigma_comp.dtype, device=sigma_comp.device)
    call("gfm_force_sigma_reduce", ptr(sigma_comp.contiguous()), ptr(node_offsets), B,
         FORCE_REDUCTIONS.index(how), ptr(out), _lib.dtype_code(sigma_comp.dtype),
         stream_handle())
    return out


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
    f_sigma = reduce_force_sigma(population_sigma(f_stack), batch.node_offsets, force_reduction)
    e_mean, e_sigma = member_stats(e_stack)
    return EnsemblePrediction(
        energy_mean=e_mean.cpu().numpy().astype(np.float64),
        energy_sigma=e_sigma.cpu().numpy().astype(np.float64),
        force_sigma=f_sigma.cpu().numpy().astype(np.float64),
        member_count=len(members))
