"""Thread ranks in one process (create_thread_comms, comm.py:219-230): the
host collectives on CPU -- float64 sums in ascending rank order, bitwise
(comm.py:143-147), mean, gather / broadcast / barrier, count checks."""

import threading

import numpy as np
import pytest

from paper_2406_12909_b200.comm import LocalComm, create_thread_comms
from paper_2406_12909_b200.errors import ValidationError


def _run(size, fn):
    comms = create_thread_comms(size, timeout=20)
    out = [None] * size
    err = []

    def work(r):
        try:
            out[r] = fn(comms[r])
        except Exception as e:  # noqa: BLE001
            err.append(e)
            comms[r]._hub.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(30)
    if err:
        raise err[0]
    return out


def test_single_rank_is_local():
    assert isinstance(create_thread_comms(1)[0], LocalComm)


@pytest.mark.parametrize("size", [2, 3, 5])
def test_host_collectives(size):
    rng = np.random.default_rng(size)
    vecs = [rng.standard_normal(1001) * 10.0 ** rng.integers(-8, 8, 1001) for _ in range(size)]
    want = vecs[0].copy()
    for v in vecs[1:]:
        want += v

    def fn(c):
        s = c.allreduce_sum(vecs[c.rank])
        m = c.allreduce_mean(vecs[c.rank])
        c.barrier()
        g = c.gather_obj(("rank", c.rank))
        b = c.broadcast_obj({"x": 7} if c.rank == 0 else None)
        return s, m, g, b

    out = _run(size, fn)
    for r, (s, m, g, b) in enumerate(out):
        np.testing.assert_array_equal(s, want)
        np.testing.assert_array_equal(m, want / size)
        assert g == ([("rank", k) for k in range(size)] if r == 0 else None)
        assert b == {"x": 7}


def test_count_mismatch_raises():
    with pytest.raises(ValidationError):
        _run(2, lambda c: c.allreduce_sum(np.zeros(3 + c.rank)))
