"""Phase accounting inside the step (PhaseClock, telemetry.py:41-86).

Host wall-clock per phase, as the reference reports it; for device time the
trainer also records CUDA events per phase (``DeviceClock``).
"""

from __future__ import annotations

import threading
import time
from contextlib import contextmanager

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


def compute_lif(times):
    """Load-imbalance factor max/mean over ranks (scaling.py:54-61)."""
    times = [float(t) for t in times]
    mean = sum(times) / len(times) if times else 0.0
    return max(times) / mean if mean > 0 else 1.0


def wait_fraction(step_time, busy_time):
    """Share of a step spent waiting at the collective (scaling.py:64-72)."""
    return max(0.0, (step_time - busy_time) / step_time) if step_time > 0 else 0.0
