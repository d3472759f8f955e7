"""Phase accounting inside the step (PhaseClock, telemetry.py:41-86).

``PhaseClock``: host wall-clock per phase, as the reference reports it --
around asynchronous launches that is enqueue time.  ``DeviceClock``: the
same phases timed on the device with CUDA events on the launching stream
(``train(device_clock=...)``), read once per epoch.  ``compute_lif`` /
``wait_fraction``: the scaling report's load-balance measures
(scaling.py:54-72).
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


class DeviceClock:
    """Device time per phase: a CUDA event pair per phase occurrence on the
    current stream; ``totals()`` synchronises once and sums the elapsed
    times (seconds), cumulative like PhaseClock.totals()."""

    def __init__(self):
        self._pending = []  # (name, start event, end event)
        self._t = {}

    @contextmanager
    def phase(self, name):
        import torch

        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        try:
            yield
        finally:
            b.record()
            self._pending.append((name, a, b))

    def totals(self) -> dict:
        for name, a, b in self._pending:
            b.synchronize()
            self._t[name] = self._t.get(name, 0.0) + a.elapsed_time(b) / 1e3
        self._pending.clear()
        return dict(self._t)


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
