"""ctypes binding of libduoserve_sm100.so (include/duoserve_b200.h).

This is the only place the package touches the C-ABI.  There is no CPU
fallback: if the library is missing, or a compute entry point fails (for
instance because no sm_100 device is present), a ``DeviceError`` is raised.
Device tensors are passed as raw pointers (``tensor.data_ptr()``), streams
as ``torch.cuda.current_stream().cuda_stream``.  ctypes releases the GIL for
the duration of each call.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libduoserve_sm100.so"
HEADER_PATH = Path(__file__).resolve().parent.parent / "include" / "duoserve_b200.h"

DS_MAX_HIDDEN = 8
DS_MAX_EXPERTS = 64


class DeviceError(RuntimeError):
    """A C-ABI call failed (CUDA error, bad argument, or missing library)."""

    def __init__(self, fn: str, status: int, message: str):
        self.fn, self.status = fn, status
        super().__init__(f"{fn} failed with status {status}: {message}")


class MlpDesc(C.Structure):
    _fields_ = [("input_dim", C.c_int), ("output_dim", C.c_int), ("n_hidden", C.c_int),
                ("hidden", C.c_int * DS_MAX_HIDDEN)]

    @classmethod
    def make(cls, input_dim: int, output_dim: int, hidden) -> "MlpDesc":
        hidden = list(hidden)
        if len(hidden) > DS_MAX_HIDDEN:
            raise ValueError(f"at most {DS_MAX_HIDDEN} hidden layers supported")
        d = cls()
        d.input_dim, d.output_dim, d.n_hidden = int(input_dim), int(output_dim), len(hidden)
        for i, h in enumerate(hidden):
            d.hidden[i] = int(h)
        return d


class W4Linear(C.Structure):
    _fields_ = [("codes", C.c_void_p), ("scales", C.c_void_p), ("zeros", C.c_void_p)]


class W4Expert(C.Structure):
    _fields_ = [("w1", W4Linear), ("w3", W4Linear), ("w2", W4Linear)]


_P = C.c_void_p
_I = C.c_int
_SZ = C.c_size_t

# name -> (restype, argtypes)
_SIGS = {
    "ds_abi_version": (_I, []),
    "ds_last_error": (C.c_char_p, []),
    "ds_device_info": (_I, [C.POINTER(_I), C.POINTER(_I)]),
    "ds_mlp_container_doubles": (_SZ, [C.POINTER(MlpDesc)]),
    "ds_mlp_packed_doubles": (_SZ, [C.POINTER(MlpDesc)]),
    "ds_mlp_pack": (_I, [C.POINTER(MlpDesc), _P, _P, _P]),
    "ds_mlp_workspace_bytes": (_SZ, [C.POINTER(MlpDesc), _I]),
    "ds_predictor_forward": (_I, [C.POINTER(MlpDesc), _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I,
                                  _P, _P, _P, _SZ, _P]),
    "ds_mlp_forward_features": (_I, [C.POINTER(MlpDesc), _P, _P, _I, _I, _P, _P, _P, _SZ, _P]),
    "ds_gate_topk": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _I, _I, _P]),
    "ds_permute": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "ds_unpermute_combine": (_I, [_P, _P, _P, _P, _I, _I, _I, _P, _P]),
    "ds_cache_check": (_I, [_P, _P, _I, _I, _P, _P]),
    "ds_unpermute_partial": (_I, [_P, _P, _P, _P, C.c_uint64, _I, _I, _I, _P, _P]),
    "ds_route_histogram": (_I, [_P, _I, _I, _I, _I, _P, _P, _P]),
    "ds_w4_expert_layout": (_SZ, [_I, _I, _I, C.POINTER(_SZ * 9)]),
    "ds_w4_generate": (_I, [C.c_uint64, _I, _I, _I, _I, _I, _P, _P]),
    "ds_w4_dequant": (_I, [C.POINTER(W4Linear), _I, _I, _I, _P, _P]),
    "ds_w4_swiglu_gemv": (_I, [_P, _I, C.POINTER(W4Expert), _I, _I, _I, _P, _P]),
    "ds_w4_down_gemv": (_I, [_P, _I, C.POINTER(W4Expert), _I, _I, _I, _P, _I, _P, _P]),
    "ds_w4_expert_gemv": (_I, [_P, _I, C.POINTER(W4Expert), _I, _I, _I, _P, _P, _I, _P, _P, _P, _P]),
    "ds_w4_expert_gemv_graph": (_I, [_P, _I, C.POINTER(W4Expert), _I, _I, _I, _P, _P, _I, _P, _P, _P, _P, _P]),
    "ds_w4_graph_cache_clear": (_I, []),
    "ds_rmsnorm": (_I, [_P, _I, _I, _P, C.c_float, _P, _P]),
    "ds_residual_rmsnorm": (_I, [_P, _P, _I, _I, _P, C.c_float, _P, _P, _P]),
    "ds_rope_kv_decode": (_I, [_P, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P]),
    "ds_k4_device_span": (_I, [C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
    "ds_k3_device_span": (_I, [C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
    "ds_combine_finalize": (_I, [_P, _P, _I, _I, _P, _P]),
    "ds_w4_grouped_ffn_workspace": (_SZ, [_I, _I, _I]),
    "ds_w4_linear_layout": (_SZ, [_I, _I, _I, C.POINTER(_SZ * 3)]),
    "ds_w4_generate_linear": (_I, [C.c_uint64, _I, _I, _I, _I, _I, _I, _P, _P]),
    "ds_w4_linear_gemv": (_I, [_P, _I, C.POINTER(W4Linear), _I, _I, _I, _P, _P]),
    "ds_w4_linear_workspace": (_SZ, [_I, _I, _I]),
    "ds_w4_linear_gemm": (_I, [_P, _I, C.POINTER(W4Linear), _I, _I, _I, _P, _P, _SZ, _P]),
    "ds_link_create": (_I, [_P, _SZ, _I, C.POINTER(_P)]),
    "ds_link_destroy": (_I, [_P]),
    "ds_link_submit": (_I, [_P, _P, _P, _SZ, _P, _P, C.POINTER(C.c_uint64)]),
    "ds_link_cancel": (_I, [_P, C.c_uint64, C.POINTER(_SZ)]),
    "ds_link_submit_chunked": (_I, [_P, _P, _P, _SZ, _SZ, _P, _P, C.POINTER(C.c_uint64)]),
    "ds_link_promote": (_I, [_P, C.c_uint64]),
    "ds_link_wait_issued": (_I, [_P, C.c_uint64]),
    "ds_link_idle": (_I, [_P]),
    "ds_link_stats": (_I, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "ds_link_reset_stats": (_I, [_P]),
    "ds_link_trace": (_I, [_P, _I]),
    "ds_link_trace_read": (_I, [_P, _P, C.POINTER(C.c_float), C.POINTER(C.c_float), _SZ, C.POINTER(_SZ)]),
    "ds_h2d_sm_copy": (_I, [_P, _P, _SZ, _I, _P]),
    "ds_debug_k4v6_timeline": (_I, [_P, _I]),
    "ds_debug_k3_timeline": (_I, [_P, _I, _I]),
    "ds_l2_persist_window": (_I, [_P, _P, _SZ, C.c_float]),
    "ds_h2d_tma_copy": (_I, [_P, _P, _SZ, _I, _P]),
    "ds_w4_grouped_ffn": (_I, [_P, C.POINTER(_I), _I, C.POINTER(W4Expert), _I, _I, _I, _P, _P, _P, _SZ, _P]),
    "ds_w4_grouped_ffn_seg_workspace": (_SZ, [C.POINTER(_I), C.POINTER(_I), _I, _I, _I, _I]),
    "ds_w4_grouped_ffn_seg_ev": (_I, [_P, C.POINTER(_I), C.POINTER(_I), _I, C.POINTER(W4Expert), _I, _I, _I, _P, _P,
                                      _P, _SZ, _P, _P, _P]),
    "ds_w4_grouped_ffn_ev": (_I, [_P, C.POINTER(_I), _I, C.POINTER(W4Expert), _I, _I, _I, _P, _P, _P, _SZ, _P, _P,
                                  _P]),
}

_lib = None


def load() -> C.CDLL:
    """Load (once) and type the library; raises DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise DeviceError("load", -1, f"{LIB_PATH} not built; run `python -m paper_2509_07379_b200.build`")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name, None)
        if fn is None:
            raise DeviceError("load", -1, f"{LIB_PATH.name} does not export {name}")
        fn.restype = res
        fn.argtypes = args
    if lib.ds_abi_version() != 1:
        raise DeviceError("load", -1, "ABI version mismatch")
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point; raise DeviceError on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.ds_last_error().decode(errors="replace")
        raise DeviceError(name, rc, msg)


def query(name: str, *args):
    return getattr(load(), name)(*args)


def ptr(t) -> C.c_void_p | None:
    """Device (or host) pointer of a torch tensor, None for None."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def stream_ptr(stream=None) -> C.c_void_p:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)
