"""torch-facing wrappers of the C-ABI hot-path kernels (device tensors in,
device tensors out, launched on the current stream).  No CPU fallback."""

from __future__ import annotations

import ctypes as C
from functools import lru_cache

import torch

from . import _lib
from ._lib import ptr, stream_ptr

# kernels launched by this process through the wrappers below (bench.py's
# "gpu_launches" evidence); keyed by C-ABI entry point
LAUNCHES: dict = {}


def _count(name: str, n: int = 1) -> None:
    LAUNCHES[name] = LAUNCHES.get(name, 0) + n


def launch_total() -> int:
    return sum(LAUNCHES.values())


@lru_cache(maxsize=None)
def expert_layout(d: int, ff: int, G: int):
    """(section offsets [9], total bytes) of one W4 expert blob."""
    offs = (C.c_size_t * 9)()
    total = _lib.query("ds_w4_expert_layout", d, ff, G, C.byref(offs))
    if total == 0:
        raise ValueError(f"unsupported expert shape d={d} ff={ff} G={G}")
    return tuple(offs), int(total)


def expert_struct(base_ptr: int, d: int, ff: int, G: int) -> _lib.W4Expert:
    offs, _ = expert_layout(d, ff, G)
    e = _lib.W4Expert()
    for m, lin in enumerate((e.w1, e.w3, e.w2)):
        lin.codes, lin.scales, lin.zeros = base_ptr + offs[m], base_ptr + offs[3 + m], base_ptr + offs[6 + m]
    return e


def w4_generate(seed: int, layer: int, expert: int, d: int, ff: int, G: int, blob: torch.Tensor) -> None:
    _lib.call("ds_w4_generate", seed, layer, expert, d, ff, G, ptr(blob), stream_ptr())
    _count("ds_w4_generate", 9)


def gate_topk(x: torch.Tensor, wg: torch.Tensor, k: int, idx: torch.Tensor, w: torch.Tensor,
              counts: torch.Tensor | None = None, hist: torch.Tensor | None = None, layer: int = 0,
              logits: torch.Tensor | None = None) -> None:
    T, d = x.shape
    M = wg.shape[0]
    if idx.shape[0] < T or w.shape[0] < T or idx.shape[-1] < k or w.shape[-1] < k:
        raise ValueError(f"gate_topk: idx {tuple(idx.shape)} / w {tuple(w.shape)} too small for {T} tokens x top-{k}")
    if hist is not None and hist.shape[0] < T:
        raise ValueError(f"gate_topk: hist has {hist.shape[0]} rows for {T} tokens")
    stride = hist.shape[-1] if hist is not None else 0
    _lib.call("ds_gate_topk", ptr(x), ptr(wg), T, d, M, k, ptr(idx), ptr(w), ptr(logits), ptr(counts),
              ptr(hist), stride, layer, stream_ptr())
    _count("ds_gate_topk")


def permute(idx: torch.Tensor, x: torch.Tensor, M: int, offsets, pos, src, xperm) -> None:
    T, k = idx.shape
    if x.shape[0] < T or pos.numel() < T * k or src.numel() < T * k or (xperm is not None and xperm.shape[0] < T * k):
        raise ValueError(f"permute: buffers too small for {T} tokens x top-{k}")
    _lib.call("ds_permute", ptr(idx), ptr(x), T, x.shape[1], M, k, ptr(offsets), ptr(pos), ptr(src),
              ptr(xperm), stream_ptr())
    _count("ds_permute", 2 if xperm is not None else 1)


def unpermute_combine(y: torch.Tensor, pos, w, resid, out) -> None:
    T, k = w.shape
    _lib.call("ds_unpermute_combine", ptr(y), ptr(pos), ptr(w), ptr(resid), T, resid.shape[1], k, ptr(out),
              stream_ptr())
    _count("ds_unpermute_combine")


def unpermute_partial(y: torch.Tensor, pos, w, idx, owned_mask: int, out: torch.Tensor) -> None:
    T, k = w.shape
    _lib.call("ds_unpermute_partial", ptr(y), ptr(pos), ptr(w), ptr(idx), owned_mask, T, out.shape[1], k, ptr(out),
              stream_ptr())
    _count("ds_unpermute_partial")


def _gemv_passes(R: int, G: int) -> int:
    """kernel launches of one K4 call: the mma.sync GEMV (G = 128, R >= 2) takes
    8 rows per pass, the FHFMA GEMV 4/2/1 (csrc/w4.cu k4_use_mma)."""
    if G == 128 and R >= 2:
        return (R + 7) // 8
    return R // 4 + (R % 4) // 2 + (R % 2)


def swiglu_gemv(x: torch.Tensor, e: _lib.W4Expert, d: int, ff: int, G: int, h: torch.Tensor) -> None:
    _lib.call("ds_w4_swiglu_gemv", ptr(x), x.shape[0], C.byref(e), d, ff, G, ptr(h), stream_ptr())
    _count("ds_w4_swiglu_gemv", _gemv_passes(x.shape[0], G))


def down_gemv(h: torch.Tensor, e: _lib.W4Expert, d: int, ff: int, G: int, route_w: torch.Tensor,
              route_stride: int, acc: torch.Tensor) -> None:
    _lib.call("ds_w4_down_gemv", ptr(h), h.shape[0], C.byref(e), d, ff, G, ptr(route_w), route_stride, ptr(acc),
              stream_ptr())
    _count("ds_w4_down_gemv", _gemv_passes(h.shape[0], G))


def _native_events(*evs):
    """cudaEvent_t handles of torch events for the C side to (re-)record.
    torch creates the CUDA event lazily on its first record, so record each
    once here (a placeholder the native record overwrites; it also marks the
    torch wrapper as recorded for elapsed_time)."""
    out = []
    for ev in evs:
        if ev is None:
            out.append(None)
            continue
        ev.record()
        out.append(C.c_void_p(ev.cuda_event))
    return out


def expert_gemv(x: torch.Tensor, e: _lib.W4Expert, d: int, ff: int, G: int, h: torch.Tensor, route_w: torch.Tensor,
                route_stride: int, acc: torch.Tensor, ev_start=None, ev_end=None) -> None:
    """K4 for one expert in one C call (SwiGLU GEMV + PDL down GEMV); the
    optional torch.cuda.Events are recorded natively around the launches."""
    evs = _native_events(ev_start, ev_end)
    _lib.call("ds_w4_expert_gemv", ptr(x), x.shape[0], C.byref(e), d, ff, G, ptr(h), ptr(route_w), route_stride,
              ptr(acc), evs[0], evs[1], stream_ptr())
    n = _gemv_passes(x.shape[0], G)
    _count("ds_w4_swiglu_gemv", n)
    _count("ds_w4_down_gemv", n)


def expert_gemv_graph(x: torch.Tensor, e: _lib.W4Expert, d: int, ff: int, G: int, h: torch.Tensor,
                      route_w: torch.Tensor, route_stride: int, acc: torch.Tensor, wait_event=None, ev_start=None,
                      ev_end=None) -> None:
    """K4 for one expert as ONE launch of a cached device-resident CUDA graph:
    [wait for wait_event] -> ev_start -> K4 -> ev_end (csrc/w4.cu,
    ds_w4_expert_gemv_graph): no host-submitted command sits between the
    slot's data landing and the kernel starting."""
    evs = _native_events(ev_start, ev_end)
    w = None
    if wait_event is not None:
        if not wait_event.cuda_event:
            raise _lib.DeviceError("expert_gemv_graph: wait event was never recorded")
        w = C.c_void_p(wait_event.cuda_event)
    _lib.call("ds_w4_expert_gemv_graph", ptr(x), x.shape[0], C.byref(e), d, ff, G, ptr(h), ptr(route_w),
              route_stride, ptr(acc), w, evs[0], evs[1], stream_ptr())
    n = _gemv_passes(x.shape[0], G)
    _count("ds_w4_swiglu_gemv", n)
    _count("ds_w4_down_gemv", n)


def rmsnorm(x: torch.Tensor, gamma: torch.Tensor, eps: float, out: torch.Tensor) -> torch.Tensor:
    R, d = x.shape
    _lib.call("ds_rmsnorm", ptr(x), R, d, ptr(gamma), eps, ptr(out), stream_ptr())
    _count("ds_rmsnorm")
    return out


def residual_rmsnorm(h: torch.Tensor, y: torch.Tensor, gamma: torch.Tensor, eps: float, h1: torch.Tensor,
                     a: torch.Tensor) -> None:
    R, d = h.shape
    _lib.call("ds_residual_rmsnorm", ptr(h), ptr(y), R, d, ptr(gamma), eps, ptr(h1), ptr(a), stream_ptr())
    _count("ds_residual_rmsnorm")


def rope_kv_decode(y: torch.Tensor, nh: int, nkv: int, hd: int, cos: torch.Tensor, sin: torch.Tensor,
                   pos: torch.Tensor, q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor) -> None:
    """k_cache / v_cache: one layer's [nkv, max_seq, hd] bf16 cache; pos int64 [1] on the device."""
    if pos.dtype != torch.int64 or not (k_cache.is_contiguous() and v_cache.is_contiguous()):
        raise ValueError("rope_kv_decode: pos must be int64 and the caches contiguous")
    _lib.call("ds_rope_kv_decode", ptr(y), nh, nkv, hd, ptr(cos), ptr(sin), ptr(pos), k_cache.shape[1], ptr(q),
              ptr(k_cache), ptr(v_cache), stream_ptr())
    _count("ds_rope_kv_decode")


def k4_device_span() -> tuple:
    """(ns, launches): device-clock totals of every fused K4 launch so far."""
    ns, n = C.c_ulonglong(0), C.c_ulonglong(0)
    _lib.call("ds_k4_device_span", C.byref(ns), C.byref(n))
    return ns.value, n.value


def k3_device_span() -> tuple:
    """(ns, calls): device-clock totals of every timed grouped-FFN (K3) call so far."""
    ns, n = C.c_ulonglong(0), C.c_ulonglong(0)
    _lib.call("ds_k3_device_span", C.byref(ns), C.byref(n))
    return ns.value, n.value


def w4_graph_cache_clear() -> None:
    _lib.call("ds_w4_graph_cache_clear")


def combine_finalize(acc: torch.Tensor, resid: torch.Tensor, out: torch.Tensor) -> None:
    _lib.call("ds_combine_finalize", ptr(acc), ptr(resid), resid.shape[0], resid.shape[1], ptr(out), stream_ptr())
    _count("ds_combine_finalize")


def grouped_ffn_segments(x: torch.Tensor, segments: list, experts: list, d: int, ff: int, G: int,
                         h: torch.Tensor, y: torch.Tensor, ws: torch.Tensor, ev_start=None, ev_end=None) -> None:
    """K3 over arbitrary row segments [(row_start, rows)] of x / h / y, one
    expert per segment, in ONE grouped launch (e.g. a layer's pinned experts)."""
    E = len(experts)
    rs = (C.c_int * E)(*[int(a) for a, _ in segments])
    nr = (C.c_int * E)(*[int(b) for _, b in segments])
    arr = (_lib.W4Expert * E)(*experts)
    evs = _native_events(ev_start, ev_end) if (ev_start is not None or ev_end is not None) else (None, None)
    _lib.call("ds_w4_grouped_ffn_seg_ev", ptr(x), rs, nr, E, arr, d, ff, G, ptr(h), ptr(y), ptr(ws), ws.numel(),
              evs[0], evs[1], stream_ptr())
    _count("ds_w4_grouped_ffn", 3)


def grouped_ffn_segments_workspace(segments: list, d: int, ff: int, G: int) -> int:
    E = len(segments)
    rs = (C.c_int * E)(*[int(a) for a, _ in segments])
    nr = (C.c_int * E)(*[int(b) for _, b in segments])
    return int(_lib.query("ds_w4_grouped_ffn_seg_workspace", rs, nr, E, d, ff, G))


def grouped_ffn_workspace(rows: int, d: int, ff: int) -> int:
    return int(_lib.query("ds_w4_grouped_ffn_workspace", rows, d, ff))


def grouped_ffn(xperm: torch.Tensor, offsets: list, experts: list, d: int, ff: int, G: int, h: torch.Tensor,
                y: torch.Tensor, ws: torch.Tensor, ev_start=None, ev_end=None) -> None:
    """K3.  ev_start / ev_end (torch.cuda.Event, optional) are recorded natively
    around the launches (host-side preparation excluded)."""
    E = len(experts)
    off = (C.c_int * (E + 1))(*[int(o) for o in offsets])
    arr = (_lib.W4Expert * E)(*experts)
    if ev_start is None and ev_end is None:
        _lib.call("ds_w4_grouped_ffn", ptr(xperm), off, E, arr, d, ff, G, ptr(h), ptr(y), ptr(ws), ws.numel(),
                  stream_ptr())
    else:
        evs = _native_events(ev_start, ev_end)
        _lib.call("ds_w4_grouped_ffn_ev", ptr(xperm), off, E, arr, d, ff, G, ptr(h), ptr(y), ptr(ws), ws.numel(),
                  evs[0], evs[1], stream_ptr())
    _count("ds_w4_grouped_ffn", 3)


def route_histogram(paths: torch.Tensor, M: int, pop_counts: torch.Tensor, aff_counts: torch.Tensor) -> None:
    N, L, k = paths.shape
    _lib.call("ds_route_histogram", ptr(paths), N, L, M, k, ptr(pop_counts), ptr(aff_counts), stream_ptr())
    _count("ds_route_histogram")


# ------------------------------------------------------------- W4 linears
# the non-MoE projections (attention q|k|v, o) in the experts' W4 format

@lru_cache(maxsize=None)
def linear_layout(K: int, N: int, G: int):
    """(section offsets [codes, scales, zeros], total bytes) of one W4 linear blob."""
    offs = (C.c_size_t * 3)()
    total = _lib.query("ds_w4_linear_layout", K, N, G, C.byref(offs))
    if total == 0:
        raise ValueError(f"unsupported W4 linear shape K={K} N={N} G={G}")
    return tuple(offs), int(total)


class W4Lin:
    """One resident W4 linear y = x W^T (W [N, K]): its device blob + the C struct."""

    def __init__(self, blob: torch.Tensor, K: int, N: int, G: int):
        offs, total = linear_layout(K, N, G)
        if blob.numel() < total or blob.dtype != torch.uint8:
            raise ValueError("W4Lin: blob too small")
        self.blob, self.K, self.N, self.G = blob, K, N, G
        self.st = _lib.W4Linear()
        base = blob.data_ptr()
        self.st.codes, self.st.scales, self.st.zeros = base + offs[0], base + offs[1], base + offs[2]

    @classmethod
    def generate(cls, seed: int, layer: int, tag: int, matrix: int, K: int, N: int, G: int, device) -> "W4Lin":
        _, total = linear_layout(K, N, G)
        blob = torch.empty(total, dtype=torch.uint8, device=device)
        _lib.call("ds_w4_generate_linear", seed, layer, tag, matrix, K, N, G, ptr(blob), stream_ptr())
        _count("ds_w4_generate_linear", 3)
        return cls(blob, K, N, G)

    @property
    def nbytes(self) -> int:
        return self.blob.numel()


def linear_workspace(rows: int, K: int, N: int) -> int:
    return int(_lib.query("ds_w4_linear_workspace", rows, K, N))


GEMV_MAX_ROWS = 16      # rows at or below which the GEMV (K4) path is used


def w4_linear(x: torch.Tensor, lin: W4Lin, y: torch.Tensor, ws: torch.Tensor | None = None) -> torch.Tensor:
    """y[R, N] (f32) = x[R, K] (bf16) W^T: the K4 GEMV for R <= GEMV_MAX_ROWS
    (exact (q - z) s products), the tcgen05 GEMM above (bf16-rounded weights)."""
    R = x.shape[0]
    if x.shape[1] != lin.K or y.shape[0] < R or y.shape[1] != lin.N:
        raise ValueError(f"w4_linear: x {tuple(x.shape)} / y {tuple(y.shape)} vs W [{lin.N}, {lin.K}]")
    if R <= GEMV_MAX_ROWS:
        _lib.call("ds_w4_linear_gemv", ptr(x), R, C.byref(lin.st), lin.K, lin.N, lin.G, ptr(y), stream_ptr())
        _count("ds_w4_linear_gemv", _gemv_passes(R, lin.G))
    else:
        nb = ws.numel() if ws is not None else 0
        _lib.call("ds_w4_linear_gemm", ptr(x), R, C.byref(lin.st), lin.K, lin.N, lin.G, ptr(y), ptr(ws), nb,
                  stream_ptr())
        _count("ds_w4_linear_gemm", 2)
    return y
