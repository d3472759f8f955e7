"""ctypes binding of the in-tree C-ABI library ``_lib/libgfm_b200.so``.

The library is the product: there is no CPU or PyTorch fallback.  If the
shared object is missing (not built) or no CUDA device is present, every
compute entry point raises :class:`ExtensionMissingError` loudly.
Declarations mirror ``include/gfm_b200.h``.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import GFMError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
# GFM_LIB_PATH: an alternative in-tree build of the same library (A/B runs)
LIB_PATH = os.environ.get("GFM_LIB_PATH") or os.path.join(_HERE, "_lib", "libgfm_b200.so")

F32, F64 = 0, 1
PART_SUM, PART_MEAN, PART_MAX, PART_STD = 1, 2, 4, 8
FLAG_SCALAR = 1
FLAG_ARGMAX_U8 = 2
FLAG_AGG_PREPPED = 4
FLAG_W_CSC = 8
FLAG_GATHER_LOCAL = 16
ABI_VERSION = 3

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_L = ctypes.c_longlong
_S = ctypes.c_size_t

class ReduceJob(ctypes.Structure):
    """gfm_reduce_job (include/gfm_b200.h): one deferred split-K reduction"""
    _fields_ = [("ws", ctypes.c_void_p), ("splits", ctypes.c_int), ("N", ctypes.c_int),
                ("K1", ctypes.c_int), ("K2", ctypes.c_int), ("with_bias", ctypes.c_int),
                ("trans", ctypes.c_int), ("g1", ctypes.c_void_p), ("g2", ctypes.c_void_p),
                ("gb", ctypes.c_void_p)]


_JOBP = ctypes.POINTER(ReduceJob)

# name -> (restype, argtypes); the single source of truth for the Python side
SIGNATURES = {
    "gfm_abi_version": (_I, []),
    "gfm_last_error": (ctypes.c_char_p, []),
    "gfm_device_sm_count": (_I, []),
    "gfm_stream_sync": (_I, [_P]),
    "gfm_set_gemm_mode": (_I, [_I]),
    "gfm_get_gemm_mode": (_I, []),
    "gfm_set_tc_pairs": (_I, [_I]),
    "gfm_tc_pair_launches": (_L, []),
    "gfm_graph_of_node": (_I, [_P, _I, _P, _P]),
    "gfm_gather_structures": (_I, [_P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P]),
    "gfm_gather_batch": (_I, [_P, _P, _I, _I] + [_P] * 25 + [_I, _P]),
    "gfm_gather_blocks": (_I, [_P, _I, _P, _P, _I, _P, _P, _P, _P]),
    "gfm_permute": (_I, [_P, _I, _P, _P, _P, _I, _P]),
    "gfm_eval_errors": (_I, [_P, _P, _P, _I, _P, _P, _I, _P, _I, _P]),
    "gfm_member_stats": (_I, [_P, _I, _L, _P, _P, _I, _P]),
    "gfm_force_sigma_reduce": (_I, [_P, _P, _I, _I, _P, _I, _P]),
    "gfm_record_scan": (_I, [_P, _P, _P, _I, _P, _P, _P, _P]),
    "gfm_record_decode": (_I, [_P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "gfm_scan_workspace_bytes": (_S, [_I]),
    "gfm_exclusive_scan": (_I, [_P, _I, _P, _P, _P]),
    "gfm_radius_count": (_I, [_P, _P, _P, _I, _P, _D, _I, _P, _P]),
    "gfm_radius_fill": (_I, [_P, _P, _P, _I, _P, _D, _I, _P, _P, _P, _P, _P, _I, _P]),
    "gfm_csr_workspace_bytes": (_S, [_I, _I, _I]),
    "gfm_csr_build": (_I, [_P, _P, _P, _I, _P, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P,
                           _P, _I, _P, _P]),
    "gfm_csc_from_csr": (_I, [_P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P]),
    "gfm_radius_batch_workspace_bytes": (_S, [_I]),
    "gfm_radius_batch_overflow_index": (_I, [_I]),
    "gfm_radius_batch": (_I, [_P, _P, _I, _I, _I, _P, _D, _I, _P, _P, _P, _P, _P, _P, _P, _P,
                              _P, _I, _P, _I, _P]),
    "gfm_embed": (_I, [_P, _I, _P, _I, _P, _I, _P]),
    "gfm_agg_parts_count": (_I, [_I]),
    "gfm_agg_fwd": (_I, [_P, _I, _I, _P, _P, _P, _I, _P, _P, _P, _I, _I, _P]),
    "gfm_agg_bwd_workspace_bytes": (_S, [_I, _I, _I, _I]),
    "gfm_agg_bwd": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P,
                         _I, _I, _P]),
    "gfm_linear_fwd": (_I, [_P, _I, _I, _P, _I, _I, _P, _I, _P, _I, _P, _I, _P, _I, _I, _P, _I,
                            _I, _P]),
    "gfm_linear_bwd_data": (_I, [_P, _I, _I, _P, _I, _P, _I, _I, _P, _I, _I, _P, _I, _P, _I,
                                 _P, _I, _I, _P]),
    "gfm_linear_bwd_weight_workspace_bytes": (_S, [_I, _I, _I, _I, _I, _I]),
    "gfm_linear_bwd_weight": (_I, [_P, _I, _I, _P, _I, _P, _I, _I, _P, _I, _I, _I, _P, _P, _P,
                                   _P, _I, _P]),
    "gfm_linear_bwd_weight_partials": (_I, [_P, _I, _I, _P, _I, _P, _I, _I, _P, _I, _I, _I, _P,
                                            _P, _P, _P, _JOBP, _I, _P]),
    "gfm_splitk_reduce_batch": (_I, [_JOBP, _I, _I, _P]),
    "gfm_force_fwd": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P]),
    "gfm_force_bwd_workspace_bytes": (_S, [_I, _I, _I]),
    "gfm_force_bwd": (_I, [_P, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                           _P, _P, _P, _I, _I, _P]),
    "gfm_layer_bwd_data_agg_workspace_bytes": (_S, [_I]),
    "gfm_layer_bwd_data_agg": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "gfm_force_bwd_edges": (_I, [_P, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                 _P, _P, _P, _I, _I, _P]),
    "gfm_force_bwd_grads": (_I, [_P, _I, _I, _P, _P, _P, _P, _I, _P]),
    "gfm_force_bwd_finish": (_I, [_P, _I, _I, _P, _P, _P, _P, _I, _P]),
    "gfm_energy_readout": (_I, [_P, _I, _I, _P, _P, _P, _I, _P, _P, _I, _P]),
    "gfm_loss_workspace_bytes": (_S, []),
    "gfm_loss_seeds": (_I, [_P, _P, _P, _I, _P, _P, _I, _P, _D, _D, _P, _P, _P, _P, _P, _I, _P]),
    "gfm_energy_seed": (_I, [_P, _P, _I, _I, _P, _P, _P, _I, _P, _I, _P]),
    "gfm_embedding_grad_workspace_bytes": (_S, [_I, _I, _I]),
    "gfm_embedding_grad": (_I, [_P, _I, _P, _I, _P, _P, _I, _P]),
    "gfm_nonfinite_flag": (_I, [_P, _L, _I, _P, _P]),
    "gfm_adam_step": (_I, [_P, _I, _L, _D, _P, _P, _P, _P, _D, _D, _D, _D, _P, _P, _P]),
    "gfm_adam_advance": (_I, [_P, _D, _D, _P, _P, _L, _P, _P]),
    "gfm_nonfinite_advance": (_I, [_P, _L, _I, _P, _P, _D, _D, _P, _P, _L, _P]),
    "gfm_sgd_step": (_I, [_P, _I, _L, _D, _P, _D, _P, _P, _P]),
    "gfm_cast_f64_to_f32": (_I, [_P, _L, _P, _P]),
    "gfm_egnn_edge_fwd": (_I, [_P, _I, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P, _I, _P, _I, _P, _P,
                               _P, _I, _P]),
    "gfm_egnn_edge_bwd": (_I, [_P, _I, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _I, _P, _I,
                               _P, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P]),
    "gfm_egnn_tanh_fwd": (_I, [_P, _P, _I, _P, _I, _I, _P, _P, _I, _I, _P]),
    "gfm_egnn_tanh_bwd": (_I, [_P, _I, _P, _I, _P, _P, _I, _I, _I, _P, _P, _I, _I, _P]),
    "gfm_egnn_energy": (_I, [_P, _P, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P, _I, _P]),
    "gfm_egnn_head_seed": (_I, [_P, _P, _I, _I, _D, _P, _I, _P, _P, _I, _I, _P]),
    "gfm_colsum_workspace_bytes": (_S, [_I, _I]),
    "gfm_colsum": (_I, [_P, _I, _I, _I, _P, _I, _P, _I, _P]),
    "gfm_scale": (_I, [_P, _L, _D, _P, _I, _P]),
}


class ExtensionMissingError(GFMError, ImportError):
    """The sm_100a library is not built or cannot run here (no silent fallback)."""


class KernelError(GFMError, RuntimeError):
    """A C-ABI entry point returned a nonzero status."""


_lock = threading.Lock()
_lib = None


def load(require_device: bool = False):
    """Load and type the shared library (no device needed unless asked)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ExtensionMissingError(
                    f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                    "(make -C paper_2406_12909_b200/csrc); there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.gfm_abi_version() != ABI_VERSION:
                raise ExtensionMissingError("libgfm_b200.so ABI version mismatch; rebuild")
            _lib = lib
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise ExtensionMissingError("no CUDA device: the gfm_b200 kernels need a B200")
    return _lib


def call(name: str, *args) -> None:
    """Invoke an int-returning entry point; raise on a nonzero status."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.gfm_last_error().decode(errors="replace")
        if rc == -1:
            raise ValidationError(f"{name}: {msg}")
        raise KernelError(f"{name} failed ({rc}): {msg}")


def query(name: str, *args) -> int:
    return int(getattr(load(), name)(*args))


def ptr(t) -> int | None:
    """Device pointer of a tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dtype_code(dtype) -> int:
    import torch

    if dtype == torch.float32:
        return F32
    if dtype == torch.float64:
        return F64
    raise ValidationError(f"unsupported compute dtype {dtype} (float32 or float64)")
