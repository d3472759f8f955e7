"""Phase accounting inside the step (PhaseClock, telemetry.py:41-86).

Host wall-clock per phase, as the reference reports it; for device time the
trainer also records CUDA events per phase (``DeviceClock``).
"""

from __future__ import annotations

import threading
import time
from contextlib import contextmanager

from .errors import ValidationError

PHASES = ("dataload", "forward", "backward", "sync")


class PhaseClock:
    def __init__(self):
        self._lock = threading.Lock()
        self._t = {p: 0.0 for p in PHASES}

    @contextmanager
    def phase(self, name):
        t0 = time.perf_counter()
        try:
            yield
        finally:
            dt = time.perf_counter() - t0
            with self._lock:
                self._t[name] = self._t.get(name, 0.0) + dt

    def totals(self) -> dict:
        with self._lock:
            return dict(self._t)

    def reset(self):
        with self._lock:
            for k in self._t:
                self._t[k] = 0.0


def compute_lif(per_rank_times) -> float:
    """Load-imbalance factor: max over ranks / mean over ranks (>= 1)
    (scaling.py:54-61, same errors)."""
    times = [float(t) for t in per_rank_times]
    if not times:
        raise ValidationError("LIF needs at least one rank time")
    if any(t <= 0 for t in times):
        raise ValidationError("LIF requires strictly positive rank times")
    return max(times) / (sum(times) / len(times))


def wait_fraction(per_rank_times) -> float:
    """Mean over ranks of (slowest - own) / slowest; 0 when balanced
    (scaling.py:64-72)."""
    times = [float(t) for t in per_rank_times]
    if not times:
        return 0.0
    peak = max(times)
    if peak <= 0:
        return 0.0
    return sum((peak - t) / peak for t in times) / len(times)
