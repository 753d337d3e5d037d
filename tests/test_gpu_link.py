"""K6 link trace: one copy-busy span per transfer (closed when it completes or
is cancelled), bytes land intact, and the cancelled transfer's span ends
before the next transfer's begins."""
import ctypes as C

import pytest

from paper_2509_07379_b200 import _lib

pytestmark = pytest.mark.gpu


def test_link_trace_one_span_per_transfer(cuda):
    import torch
    n = 64 << 20
    src = torch.randint(0, 255, (3, n), dtype=torch.uint8).pin_memory()
    dst = torch.zeros((3, n), dtype=torch.uint8, device=cuda)
    cs = torch.cuda.Stream()
    h = C.c_void_p()
    _lib.call("ds_link_create", C.c_void_p(cs.cuda_stream), 16 << 20, 2, C.byref(h))
    try:
        ref = torch.cuda.Event(enable_timing=True)
        ref.record(cs)
        cs.synchronize()
        _lib.call("ds_link_trace", h, 1)
        t = [C.c_uint64() for _ in range(3)]
        # a whole transfer, a speculative one (1 MB chunks) cancelled mid-way, a whole one
        _lib.call("ds_link_submit", h, _lib.ptr(dst[0]), _lib.ptr(src[0]), n, None, None, C.byref(t[0]))
        _lib.call("ds_link_submit_chunked", h, _lib.ptr(dst[1]), _lib.ptr(src[1]), n, 1 << 20, None, None,
                  C.byref(t[1]))
        _lib.call("ds_link_wait_issued", h, t[0].value)
        issued = C.c_size_t()
        _lib.call("ds_link_cancel", h, t[1].value, C.byref(issued))
        _lib.call("ds_link_submit", h, _lib.ptr(dst[2]), _lib.ptr(src[2]), n, None, None, C.byref(t[2]))
        _lib.call("ds_link_wait_issued", h, t[2].value)
        cs.synchronize()
        a, b = (C.c_float * 16)(), (C.c_float * 16)()
        cnt = C.c_size_t()
        _lib.call("ds_link_trace_read", h, C.c_void_p(ref.cuda_event), a, b, 16, C.byref(cnt))
    finally:
        _lib.call("ds_link_destroy", h)
    assert torch.equal(dst[0].cpu(), src[0]) and torch.equal(dst[2].cpu(), src[2])
    spans = [(a[i], b[i]) for i in range(cnt.value)]
    # the cancelled transfer has a span only if any of its chunks was issued
    assert len(spans) == (3 if issued.value > 0 else 2), (spans, issued.value)
    for s, e in spans:
        assert e > s
    for (s0, e0), (s1, e1) in zip(spans, spans[1:]):
        assert s1 >= e0 - 1e-3
