"""Collectives: the reference's ``Comm`` plug-in contract over NCCL.

Reference: ``Comm`` / ``LocalComm`` / ``StarComm`` (comm.py:55-216).  The
star hub over TCP / in-process channels is replaced by ``torch.distributed``
(one process per GPU, NCCL over NVLink 5 / NVSwitch; gloo on CPU for tests).

Two reduction modes:

* ``deterministic=False`` (default for training): NCCL ``all_reduce(SUM)`` in
  place on the float32 ``[grad | loss | 1]`` vector.  Every rank receives
  identical bytes (so parameters stay bitwise equal across ranks, the
  reference's invariant, train.py:1-10), but the summation order is NCCL's.
* ``deterministic=True``: ``all_gather`` then a local sum in ascending rank
  order -- the reference's exact contract (comm.py:143-147): the result equals
  ``((g0 + g1) + g2) + ...`` bit for bit.
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import ValidationError


class Comm:
    """Collective interface shared by all transports (comm.py:55-77)."""

    rank: int
    size: int

    def allreduce_mean(self, vec):
        raise NotImplementedError

    def allreduce_sum(self, vec):
        raise NotImplementedError

    def allreduce_sum_(self, tensor: torch.Tensor) -> torch.Tensor:
        """In-place device allreduce (the training hot path)."""
        out = self.allreduce_sum(tensor.detach().cpu().numpy())
        tensor.copy_(torch.as_tensor(out, dtype=tensor.dtype))
        return tensor

    def barrier(self) -> None:
        raise NotImplementedError

    def gather_obj(self, obj, root: int = 0):
        raise NotImplementedError

    def broadcast_obj(self, obj, root: int = 0):
        raise NotImplementedError

    def close(self) -> None:
        pass


class LocalComm(Comm):
    """The one-rank degenerate case (comm.py:80-100)."""

    def __init__(self):
        self.rank = 0
        self.size = 1

    def allreduce_mean(self, vec):
        return _copy(vec)

    def allreduce_sum(self, vec):
        return _copy(vec)

    def allreduce_sum_(self, tensor):
        return tensor

    def barrier(self):
        return None

    def gather_obj(self, obj, root: int = 0):
        return [obj]

    def broadcast_obj(self, obj, root: int = 0):
        return obj


def _copy(vec):
    if isinstance(vec, torch.Tensor):
        return vec.clone()
    return np.array(vec, dtype=np.float64, copy=True)


class TorchComm(Comm):
    """``torch.distributed`` process group as a ``Comm`` (NCCL or gloo).

    ``allreduce_sum`` keeps the reference semantics for host numpy vectors
    (float64, ascending-rank order when deterministic) and also accepts
    device tensors; ``allreduce_sum_`` is the in-place device path used by
    the trainer."""

    def __init__(self, group=None, deterministic: bool = False, device=None):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise ValidationError("torch.distributed is not initialised")
        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self.deterministic = deterministic
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) \
                if self.backend == "nccl" else torch.device("cpu")
        self.device = torch.device(device)

    # -- vector collectives -------------------------------------------------
    def _reduce_tensor(self, t: torch.Tensor) -> torch.Tensor:
        dist = self._dist
        if self.size == 1:
            return t
        if self.deterministic:
            parts = [torch.empty_like(t) for _ in range(self.size)]
            dist.all_gather(parts, t, group=self.group)
            # ascending rank order, always, accumulated in float64 like the
            # reference's float64 vectors (comm.py:143-147)
            out = parts[0].to(torch.float64)
            for p in parts[1:]:
                out += p.to(torch.float64)
            t.copy_(out.to(t.dtype))
            return t
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def _check_count(self, n: int):
        counts = torch.tensor([n], dtype=torch.int64, device=self.device)
        mx = counts.clone()
        self._dist.all_reduce(mx, op=self._dist.ReduceOp.MAX, group=self.group)
        mn = counts.clone()
        self._dist.all_reduce(mn, op=self._dist.ReduceOp.MIN, group=self.group)
        if int(mx.item()) != int(mn.item()):
            raise ValidationError(
                f"allreduce count mismatch: rank {self.rank} has {n}, others differ")

    def allreduce_sum(self, vec, check_count: bool = True):
        if isinstance(vec, torch.Tensor):
            t = vec.detach().to(self.device).clone()
            if check_count:
                self._check_count(t.numel())
            return self._reduce_tensor(t)
        arr = np.ascontiguousarray(vec, dtype=np.float64)
        if check_count:
            self._check_count(arr.size)
        t = torch.from_numpy(arr.copy()).to(self.device)
        return self._reduce_tensor(t).cpu().numpy()

    def allreduce_mean(self, vec):
        out = self.allreduce_sum(vec)
        return out / self.size

    def allreduce_sum_(self, tensor):
        return self._reduce_tensor(tensor)

    # -- control collectives ---------------------------------------------------
    def barrier(self):
        if self.backend == "nccl":
            self._dist.barrier(group=self.group, device_ids=[self.device.index])
        else:
            self._dist.barrier(group=self.group)

    def gather_obj(self, obj, root: int = 0):
        if root != 0:
            raise ValidationError("gathers go to rank 0 only (comm.py:182-184)")
        out = [None] * self.size if self.rank == 0 else None
        self._dist.gather_object(obj, out, dst=0, group=self.group)
        return out

    def broadcast_obj(self, obj, root: int = 0):
        if root != 0:
            raise ValidationError("broadcasts come from rank 0 only (comm.py:199-201)")
        box = [obj if self.rank == 0 else None]
        self._dist.broadcast_object_list(box, src=0, group=self.group)
        return box[0]


class _PeerHub:
    """Shared state of the thread ranks of one process."""

    def __init__(self, size: int, timeout: float):
        import threading
        self.size = size
        self.timeout = timeout
        self.barrier = threading.Barrier(size)
        self.slots = [None] * size


class ThreadPeerComm(Comm):
    """Thread ranks in ONE process (the reference's thread mode,
    create_thread_comms, comm.py:219-230; cli.py:297-311): one thread per
    rank, each driving its own GPU.  Host collectives exchange objects
    through shared slots and sum float64 vectors in ascending rank order
    (comm.py:143-147).  The device allreduce copies every peer's tensor over
    NVLink (peer copies ordered by CUDA events, no host round trip of the
    data) and sums them in ascending rank order in float64 on every rank, so
    all ranks hold identical bytes.  The rendezvous is a host barrier, so a
    step using this comm cannot be captured in a CUDA graph
    (``capturable = False``: runners step eagerly)."""

    capturable = False

    def __init__(self, rank: int, hub: _PeerHub):
        self.rank = rank
        self.size = hub.size
        self._hub = hub

    def _exchange(self, obj):
        h = self._hub
        h.slots[self.rank] = obj
        h.barrier.wait(h.timeout)
        out = list(h.slots)
        h.barrier.wait(h.timeout)  # nobody reposts before everyone has read
        return out

    def _host_sum(self, vec):
        vec = np.ascontiguousarray(vec, dtype=np.float64)
        parts = self._exchange(vec)
        for r, p in enumerate(parts):
            if p.shape != vec.shape:
                raise ValidationError(f"allreduce count mismatch: rank {r} sent {p.shape[0]}, "
                                      f"rank {self.rank} has {vec.shape[0]}")
        total = parts[0].astype(np.float64, copy=True)
        for p in parts[1:]:  # ascending rank order, always
            total += p
        return total

    def allreduce_sum(self, vec):
        return self._host_sum(vec)

    def allreduce_mean(self, vec):
        return self._host_sum(vec) / self.size

    def allreduce_sum_(self, tensor):
        if self.size == 1:
            return tensor
        dev = tensor.device
        s = torch.cuda.current_stream(dev)
        posted = torch.cuda.Event()
        posted.record(s)
        parts = self._exchange((tensor, posted))
        if any(p[0].shape != tensor.shape or p[0].dtype != tensor.dtype for p in parts):
            raise ValidationError("allreduce_sum_: ranks passed different shapes / dtypes")
        with torch.cuda.device(dev):
            for _, ev in parts:
                s.wait_event(ev)
            out = parts[0][0].to(dev, torch.float64)
            for t, _ in parts[1:]:
                out += t.to(dev, torch.float64)
            read = torch.cuda.Event()
            read.record(s)
        # every rank has read every tensor before any rank overwrites its own
        done = self._exchange(read)
        with torch.cuda.device(dev):
            for ev in done:
                s.wait_event(ev)
            tensor.copy_(out.to(tensor.dtype))
        return tensor

    def barrier(self):
        self._exchange(None)

    def gather_obj(self, obj, root: int = 0):
        if root != 0:
            raise ValidationError("gathers go to rank 0 only (comm.py:182-184)")
        out = self._exchange(obj)
        return out if self.rank == 0 else None

    def broadcast_obj(self, obj, root: int = 0):
        if root != 0:
            raise ValidationError("broadcasts come from rank 0 only (comm.py:199-201)")
        return self._exchange(obj if self.rank == 0 else None)[0]


def create_thread_comms(size: int, timeout: float = 60.0) -> list:
    """``size`` thread-rank comms of this process (comm.py:219-230); rank r's
    thread calls ``torch.cuda.set_device`` for its GPU and trains with
    ``comms[r]``."""
    if size == 1:
        return [LocalComm()]
    hub = _PeerHub(size, timeout)
    return [ThreadPeerComm(r, hub) for r in range(size)]


def allreduce_gradients(comm: Comm, grad):
    """Average gradients across ranks (comm.py:271-276)."""
    return comm.allreduce_mean(grad)
