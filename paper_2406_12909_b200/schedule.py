"""Per-rank batch schedule and a minimal in-memory record store.

Reference: epoch_permutation / epoch_schedule (ddstore.py:500-543), which
define each rank's batch composition, and the ``fetch_batch`` /
``ownership[group].n_samples`` surface of DDStore (ddstore.py:316-490) that
``train()`` uses.  The distributed store itself is out of scope; any object
with that surface (including gfmkit's DDStore) can be passed to ``train``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError


class EpochSchedule:
    def __init__(self, epoch, base_seed, batch_size, n_ranks, per_rank):
        self.epoch = epoch
        self.base_seed = base_seed
        self.batch_size = batch_size
        self.n_ranks = n_ranks
        self.per_rank = per_rank

    def for_rank(self, rank: int):
        return self.per_rank[rank]

    def max_batches(self) -> int:
        return max((len(b) for b in self.per_rank), default=0)


def epoch_permutation(n_samples: int, base_seed: int, epoch: int) -> np.ndarray:
    """The global shuffle every rank derives identically (ddstore.py:515-517)."""
    return np.random.default_rng([int(base_seed), int(epoch)]).permutation(n_samples)


def epoch_schedule(n_samples, n_ranks, batch_size, base_seed, epoch) -> EpochSchedule:
    """Permutation index k goes to rank k mod P; each rank's stream is cut into
    batch_size chunks, short last batch kept (ddstore.py:520-543)."""
    if batch_size < 1:
        raise ValidationError(f"batch_size must be >= 1, got {batch_size}")
    perm = epoch_permutation(n_samples, base_seed, epoch)
    per_rank = []
    for rank in range(n_ranks):
        stream = perm[rank::n_ranks]
        per_rank.append([stream[i:i + batch_size] for i in range(0, stream.shape[0], batch_size)])
    return EpochSchedule(epoch, base_seed, batch_size, n_ranks, per_rank)


@dataclass
class _Ownership:
    n_samples: int


class RecordStore:
    """Local, in-memory stand-in for DDStore: ``{group: [records]}``."""

    def __init__(self, groups: dict):
        self._groups = {k: list(v) for k, v in groups.items()}
        self.ownership = {k: _Ownership(len(v)) for k, v in self._groups.items()}

    def fetch_batch(self, group, indices):
        recs = self._groups[group]
        return [recs[int(i)] for i in indices]

    def close(self):
        pass
