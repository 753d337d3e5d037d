"""K1/K2 routing and K4 W4 GEMV on the B200 vs the CPU oracle."""

import ctypes as Cc

import numpy as np
import pytest
import torch

from oracle import routing_ref as RR
from oracle import w4_ref as WR
from paper_2509_07379_b200 import _lib

pytestmark = pytest.mark.gpu


def _bf16_bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _rand_bf16(shape, std, gen):
    return (torch.randn(shape, generator=gen) * std).to(torch.bfloat16)


@pytest.mark.parametrize("T,d,M,k", [(1, 4096, 8, 2), (64, 256, 8, 2), (512, 4096, 8, 2), (37, 6144, 8, 2),
                                     (5, 512, 16, 4)])
def test_gate_topk_bit_exact(T, d, M, k, cuda):
    g = torch.Generator().manual_seed(T * 7 + d)
    x = _rand_bf16((T, d), 1.0, g)
    wg = _rand_bf16((M, d), 0.02, g)
    if T == 5:  # force exact ties: duplicate expert rows
        wg[3] = wg[1]
    xd, wd = x.to(cuda), wg.to(cuda)
    idx = torch.empty((T, k), dtype=torch.int32, device=cuda)
    w = torch.empty((T, k), dtype=torch.float32, device=cuda)
    lg = torch.empty((T, M), dtype=torch.float64, device=cuda)
    cnt = torch.zeros(M, dtype=torch.int32, device=cuda)
    hist = torch.zeros((T, 3 * k), dtype=torch.int32, device=cuda)
    _lib.call("ds_gate_topk", _lib.ptr(xd), _lib.ptr(wd), T, d, M, k, _lib.ptr(idx), _lib.ptr(w),
              _lib.ptr(lg), _lib.ptr(cnt), _lib.ptr(hist), 3 * k, 1, _lib.stream_ptr())
    torch.cuda.synchronize()
    ref_lg = RR.gate_logits(_bf16_bits(x), _bf16_bits(wg))
    assert np.array_equal(lg.cpu().numpy(), ref_lg)           # bitwise f64 logits
    ref_idx, ref_w = RR.topk_route(ref_lg, k)
    assert np.array_equal(idx.cpu().numpy(), ref_idx)
    assert np.allclose(w.cpu().numpy(), ref_w, rtol=1e-6, atol=0)
    assert np.array_equal(cnt.cpu().numpy(), np.bincount(ref_idx.reshape(-1), minlength=M))
    h = hist.cpu().numpy()
    assert np.array_equal(h[:, k:2 * k], ref_idx + 1) and not h[:, :k].any()


@pytest.mark.parametrize("T,M,k", [(1, 8, 2), (512, 8, 2), (3000, 8, 2), (100, 16, 4)])
def test_permute_and_combine(T, M, k, cuda):
    rng = np.random.default_rng(T)
    idx = np.sort(np.stack([rng.choice(M, k, replace=False) for _ in range(T)]), axis=1).astype(np.int32)
    d = 256
    x = _rand_bf16((T, d), 1.0, torch.Generator().manual_seed(1))
    offs = torch.empty(M + 1, dtype=torch.int32, device=cuda)
    pos = torch.empty(T * k, dtype=torch.int32, device=cuda)
    src = torch.empty(T * k, dtype=torch.int32, device=cuda)
    xp = torch.empty((T * k, d), dtype=torch.bfloat16, device=cuda)
    idx_d = torch.from_numpy(idx).to(cuda)
    xd = x.to(cuda)
    _lib.call("ds_permute", _lib.ptr(idx_d), _lib.ptr(xd), T, d, M, k, _lib.ptr(offs), _lib.ptr(pos),
              _lib.ptr(src), _lib.ptr(xp), _lib.stream_ptr())
    torch.cuda.synchronize()
    r_off, r_pos, r_src = RR.permute(idx, M)
    assert np.array_equal(offs.cpu().numpy(), r_off)
    assert np.array_equal(pos.cpu().numpy(), r_pos)
    assert np.array_equal(src.cpu().numpy(), r_src)
    assert torch.equal(xp.cpu(), x[torch.from_numpy(r_src).long()])
    # combine
    y = torch.randn((T * k, d), generator=torch.Generator().manual_seed(2))
    wts = torch.rand((T, k), generator=torch.Generator().manual_seed(3))
    out = torch.empty((T, d), dtype=torch.bfloat16, device=cuda)
    yd, wd = y.to(cuda), wts.to(cuda)
    _lib.call("ds_unpermute_combine", _lib.ptr(yd), _lib.ptr(pos), _lib.ptr(wd), _lib.ptr(xd), T, d, k,
              _lib.ptr(out), _lib.stream_ptr())
    torch.cuda.synchronize()
    ref = RR.combine(y.numpy(), r_pos, wts.numpy(), x.float().numpy())
    assert np.array_equal(out.float().cpu().numpy(), ref)


def _layout(d, ff, G):
    offs = (Cc.c_size_t * 9)()
    total = _lib.query("ds_w4_expert_layout", d, ff, G, Cc.byref(offs))
    return list(offs), total


def _expert_struct(blob, offs):
    base = blob.data_ptr()
    e = _lib.W4Expert()
    for m, lin in enumerate((e.w1, e.w3, e.w2)):
        lin.codes, lin.scales, lin.zeros = base + offs[m], base + offs[3 + m], base + offs[6 + m]
    return e


@pytest.mark.parametrize("d,ff", [(256, 896), (4096, 14336)])
def test_w4_generate_matches_oracle(d, ff, cuda):
    G = 128
    offs, total = _layout(d, ff, G)
    blob = torch.empty(total, dtype=torch.uint8, device=cuda)
    blob.zero_()
    _lib.call("ds_w4_generate", 1234, 3, 5, d, ff, G, _lib.ptr(blob), _lib.stream_ptr())
    torch.cuda.synchronize()
    ref = WR.gen_expert_blob(1234, 3, 5, d, ff, G)
    assert np.array_equal(blob.cpu().numpy(), ref)


def test_w4_dequant_bit_exact(cuda):
    d, ff, G = 256, 896, 128
    offs, total = _layout(d, ff, G)
    blob = torch.zeros(total, dtype=torch.uint8, device=cuda)
    _lib.call("ds_w4_generate", 9, 0, 1, d, ff, G, _lib.ptr(blob), _lib.stream_ptr())
    e = _expert_struct(blob, offs)
    for m, (K, N, lin) in enumerate([(d, ff, e.w1), (d, ff, e.w3), (ff, d, e.w2)]):
        out = torch.empty((N, K), dtype=torch.bfloat16, device=cuda)
        _lib.call("ds_w4_dequant", Cc.byref(lin), K, N, G, _lib.ptr(out), _lib.stream_ptr())
        torch.cuda.synchronize()
        c, s, z = WR.gen_linear(9, 0, 1, m, K, N, G)
        assert np.array_equal(_bf16_bits(out), WR.dequant(c, s, z, K, N, G))


@pytest.mark.parametrize("d,ff,R,G", [(256, 896, 1, 128), (4096, 14336, 1, 128), (4096, 14336, 3, 128),
                                      (4096, 14336, 1, 64), (6144, 16384, 1, 64),
                                      (6144, 16384, 1, 128), (256, 896, 6, 128), (4096, 14336, 8, 128),
                                      (256, 896, 11, 128), (512, 1024, 3, 64), (256, 896, 5, 64)])
def test_w4_gemv_vs_f64_reference(d, ff, R, G, cuda):
    """K4 decode GEMV (G = 128: v3, mma.sync; G = 64: v2, FHFMA).  Both factorise
    the group scale out of the dot product, so the reference weights are the
    EXACT (q - z) * s (oracle.w4_ref.dequant_exact); against those the only
    error is f32 accumulation.  R = 11 crosses the 8-row pass boundary."""
    offs, total = _layout(d, ff, G)
    blob = torch.zeros(total, dtype=torch.uint8, device=cuda)
    _lib.call("ds_w4_generate", 77, 2, 3, d, ff, G, _lib.ptr(blob), _lib.stream_ptr())
    e = _expert_struct(blob, offs)
    x = _rand_bf16((R, d), 1.0, torch.Generator().manual_seed(5))
    xd = x.to(cuda)
    h = torch.empty((R, ff), dtype=torch.bfloat16, device=cuda)
    _lib.call("ds_w4_swiglu_gemv", _lib.ptr(xd), R, Cc.byref(e), d, ff, G, _lib.ptr(h), _lib.stream_ptr())
    rw = torch.rand(R, generator=torch.Generator().manual_seed(6)).to(cuda)
    acc = torch.zeros((R, d), dtype=torch.float32, device=cuda)
    _lib.call("ds_w4_down_gemv", _lib.ptr(h), R, Cc.byref(e), d, ff, G, _lib.ptr(rw), 1, _lib.ptr(acc),
              _lib.stream_ptr())
    torch.cuda.synchronize()
    W = [torch.from_numpy(WR.dequant_exact(*WR.gen_linear(77, 2, 3, m, K, N, G), K, N, G)).to(cuda)
         for m, (K, N) in enumerate([(d, ff), (d, ff), (ff, d)])]
    xf = xd.double()
    a, b = xf @ W[0].T, xf @ W[1].T
    h_ref = torch.nn.functional.silu(a) * b
    hb = h.double()
    rel = ((hb - h_ref).norm() / h_ref.norm()).item()
    assert rel < 3e-3, rel                       # h is rounded to bf16 once (<= 2^-9 relative)
    y_ref = (hb @ W[2].T) * rw.double()[:, None]
    rel2 = ((acc.double() - y_ref).norm() / y_ref.norm()).item()
    assert rel2 < 2e-5, rel2                     # f32 accumulation only

def _dense(e, d, ff, G, cuda):
    W = []
    for K, N, lin in [(d, ff, e.w1), (d, ff, e.w3), (ff, d, e.w2)]:
        out = torch.empty((N, K), dtype=torch.bfloat16, device=cuda)
        _lib.call("ds_w4_dequant", Cc.byref(lin), K, N, G, _lib.ptr(out), _lib.stream_ptr())
        W.append(out.double())
    return W


@pytest.mark.parametrize("d,ff,rows", [(256, 896, [7, 64, 0, 130]), (4096, 14336, [128, 100, 3]),
                                       (6144, 16384, [200]), (256, 896, [1]), (4096, 14336, [300, 17])])
def test_w4_grouped_ffn_tcgen05(d, ff, rows, cuda):
    """K3 (tcgen05/TMEM/TMA) vs an f64 reference on the bit-exact dequantised weights.
    Row counts cover the 128-row token tile, the 256-row tile (> 128 rows) and
    two 256-row m-blocks (300)."""
    G = 128
    offs, total = _layout(d, ff, G)
    E = len(rows)
    blobs = [torch.zeros(total, dtype=torch.uint8, device=cuda) for _ in range(E)]
    for i, b in enumerate(blobs):
        _lib.call("ds_w4_generate", 5, 1, i, d, ff, G, _lib.ptr(b), _lib.stream_ptr())
    experts = (_lib.W4Expert * E)(*[_expert_struct(b, offs) for b in blobs])
    offsets = np.concatenate([[0], np.cumsum(rows)]).astype(np.int32)
    R = int(offsets[-1])
    x = _rand_bf16((max(R, 1), d), 1.0, torch.Generator().manual_seed(11)).to(cuda)
    h = torch.empty((max(R, 1), ff), dtype=torch.bfloat16, device=cuda)
    y = torch.empty((max(R, 1), d), dtype=torch.float32, device=cuda)
    ws_bytes = _lib.query("ds_w4_grouped_ffn_workspace", R, d, ff)
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=cuda)
    off_c = (Cc.c_int * (E + 1))(*offsets.tolist())
    _lib.call("ds_w4_grouped_ffn", _lib.ptr(x), off_c, E, experts, d, ff, G, _lib.ptr(h), _lib.ptr(y),
              _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    torch.cuda.synchronize()
    for i in range(E):
        lo, hi = int(offsets[i]), int(offsets[i + 1])
        if lo == hi:
            continue
        W1, W3, W2 = _dense(experts[i], d, ff, G, cuda)
        xf = x[lo:hi].double()
        h_ref = torch.nn.functional.silu(xf @ W1.T) * (xf @ W3.T)
        hb = h[lo:hi].double()
        rel = ((hb - h_ref).norm() / h_ref.norm()).item()
        assert rel < 4e-3, (i, rel)
        y_ref = hb @ W2.T
        rel2 = ((y[lo:hi].double() - y_ref).norm() / y_ref.norm()).item()
        assert rel2 < 5e-5, (i, rel2)           # f32 accumulation over K up to 16384


@pytest.mark.parametrize("d,ff", [(4096, 14336), (6144, 16384)])
def test_expert_gemv_and_timed_grouped_ffn_match_split_calls(cuda, d, ff):
    """ds_w4_expert_gemv (one call: the fused v6 launch at 8x7B shapes, else
    SwiGLU + PDL down; native timing events) gives the separate calls' h bit
    for bit and their output to f32 summation order (v6 splits the down
    projection's K in halves); ds_w4_grouped_ffn_ev equals ds_w4_grouped_ffn
    and records a positive span."""
    import torch
    from paper_2509_07379_b200 import ops
    G = 128
    offs, total = _layout(d, ff, G)
    blob = torch.zeros(total, dtype=torch.uint8, device=cuda)
    _lib.call("ds_w4_generate", 11, 0, 2, d, ff, G, _lib.ptr(blob), _lib.stream_ptr())
    e = _expert_struct(blob, offs)
    x = _rand_bf16((1, d), 1.0, torch.Generator().manual_seed(3)).to(cuda)
    rw = torch.tensor([0.75], device=cuda)
    h1 = torch.empty((1, ff), dtype=torch.bfloat16, device=cuda)
    a1 = torch.zeros((1, d), device=cuda)
    ops.swiglu_gemv(x, e, d, ff, G, h1)
    ops.down_gemv(h1, e, d, ff, G, rw, 1, a1)
    h2 = torch.empty_like(h1)
    a2 = torch.zeros_like(a1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ops.expert_gemv(x, e, d, ff, G, h2, rw, 1, a2, ev0, ev1)
    torch.cuda.synchronize()
    assert torch.equal(h1, h2)
    assert ((a1 - a2).norm() / a1.norm()).item() < 1e-6
    assert ev0.elapsed_time(ev1) > 0
    R = 128
    xp = _rand_bf16((R, d), 1.0, torch.Generator().manual_seed(4)).to(cuda)
    ws = torch.empty(max(ops.grouped_ffn_workspace(R, d, ff), 16), dtype=torch.uint8, device=cuda)
    hh1, y1 = torch.empty((R, ff), dtype=torch.bfloat16, device=cuda), torch.empty((R, d), device=cuda)
    hh2, y2 = torch.empty_like(hh1), torch.empty_like(y1)
    ops.grouped_ffn(xp, [0, R], [e], d, ff, G, hh1, y1, ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ops.grouped_ffn(xp, [0, R], [e], d, ff, G, hh2, y2, ws, e0, e1)
    torch.cuda.synchronize()
    assert torch.equal(hh1, hh2) and torch.equal(y1, y2)
    assert e0.elapsed_time(e1) > 0


def test_staged_gemv_concurrent_streams_and_repeat(cuda):
    """K4 v5 hands row blocks out through a per-launch ticket counter reset by
    its last CTA: four expert GEMVs issued on two streams at once (they share
    the SMs, each takes a ticket slot of its own) and 70 back-to-back launches
    (the 64-slot counter ring wraps) give bit-identical results to one
    expert at a time."""
    from paper_2509_07379_b200 import ops
    d, ff, G = 4096, 14336, 128
    offs, total = _layout(d, ff, G)
    E = 4
    blobs = torch.zeros((E, total), dtype=torch.uint8, device=cuda)
    for i in range(E):
        _lib.call("ds_w4_generate", 21, 1, i, d, ff, G, _lib.ptr(blobs[i]), _lib.stream_ptr())
    es = [_expert_struct(blobs[i], offs) for i in range(E)]
    x = _rand_bf16((1, d), 1.0, torch.Generator().manual_seed(8)).to(cuda)
    rw = torch.tensor([0.5], device=cuda)
    ref_h, ref_a = [], []
    for i in range(E):
        h = torch.empty((1, ff), dtype=torch.bfloat16, device=cuda)
        a = torch.zeros((1, d), device=cuda)
        ops.expert_gemv(x, es[i], d, ff, G, h, rw, 1, a)
        torch.cuda.synchronize()
        ref_h.append(h)
        ref_a.append(a)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    hs = [torch.empty((1, ff), dtype=torch.bfloat16, device=cuda) for _ in range(E)]
    acs = [torch.zeros((1, d), device=cuda) for _ in range(E)]
    torch.cuda.synchronize()
    for i in range(E):
        with torch.cuda.stream(streams[i % 2]):
            ops.expert_gemv(x, es[i], d, ff, G, hs[i], rw, 1, acs[i])
    torch.cuda.synchronize()
    for i in range(E):
        assert torch.equal(hs[i], ref_h[i]) and torch.equal(acs[i], ref_a[i]), i
    h = torch.empty((1, ff), dtype=torch.bfloat16, device=cuda)
    for r in range(70):
        a = torch.zeros((1, d), device=cuda)
        ops.expert_gemv(x, es[r % E], d, ff, G, h, rw, 1, a)
        if r % 10 == 9 or r == 69:
            torch.cuda.synchronize()
            assert torch.equal(h, ref_h[r % E]) and torch.equal(a, ref_a[r % E]), r


def test_cache_check_matches_sim_ref_refetch_rule(cuda):
    """K7 ds_cache_check (sync point 1 on the device: bit j of miss[t] set when
    the gate's j-th expert is not in the resident prediction) gives exactly
    sim_ref's refetch sets for random gate / prediction pairs."""
    import numpy as np
    import torch
    from oracle import sim_ref
    rng = np.random.default_rng(5)
    T, k, M, L = 257, 2, 8, 2
    idx = np.stack([np.sort(rng.choice(M, k, replace=False)) for _ in range(T)]).astype(np.int32)
    pred = np.stack([np.sort(rng.choice(M, k, replace=False)) for _ in range(T)]).astype(np.int32)
    di, dp = torch.from_numpy(idx).to(cuda), torch.from_numpy(pred).to(cuda)
    miss = torch.empty(T, dtype=torch.int32, device=cuda)
    _lib.call("ds_cache_check", _lib.ptr(di), _lib.ptr(dp), T, k, _lib.ptr(miss), _lib.stream_ptr())
    torch.cuda.synchronize()
    got = miss.cpu().numpy()
    paths = [((0, 1), tuple(int(e) for e in idx[t])) for t in range(T)]
    preds = [[None, tuple(int(e) for e in pred[t])] for t in range(T)]
    log, _ = sim_ref.cache_log_decode(paths, preds, L)
    for t in range(T):
        ref = log[2 * t + 1]["refetch"]
        assert [int(idx[t, j]) for j in range(k) if got[t] >> j & 1] == ref, t


def test_grouped_ffn_segments_one_launch(cuda):
    """ds_w4_grouped_ffn_seg_ev: three experts over NON-contiguous row
    segments in one grouped launch (the engine's pinned experts of a layer)
    match per-expert launches (h bit-exact where the token tile agrees, y to
    f32 split order), and rows outside every segment are never written."""
    import torch
    from paper_2509_07379_b200 import ops
    d, ff, G = 4096, 14336, 128
    offs, total = _layout(d, ff, G)
    E = 3
    blobs = torch.zeros((E, total), dtype=torch.uint8, device=cuda)
    for i in range(E):
        _lib.call("ds_w4_generate", 31, 2, i, d, ff, G, _lib.ptr(blobs[i]), _lib.stream_ptr())
    es = [_expert_struct(blobs[i], offs) for i in range(E)]
    R = 400
    segs = [(10, 37), (120, 150), (300, 90)]            # gaps between the segments
    x = _rand_bf16((R, d), 1.0, torch.Generator().manual_seed(6)).to(cuda)
    h = torch.full((R, ff), 7.0, dtype=torch.bfloat16, device=cuda)
    y = torch.full((R, d), -3.0, device=cuda)
    ws = torch.empty(max(ops.grouped_ffn_segments_workspace(segs, d, ff, G), 16), dtype=torch.uint8, device=cuda)
    ops.grouped_ffn_segments(x, segs, es, d, ff, G, h, y, ws)
    torch.cuda.synchronize()
    inside = torch.zeros(R, dtype=torch.bool)
    for i, (a, n) in enumerate(segs):
        inside[a:a + n] = True
        h1 = torch.empty((n, ff), dtype=torch.bfloat16, device=cuda)
        y1 = torch.empty((n, d), device=cuda)
        w1 = torch.empty(max(ops.grouped_ffn_workspace(n, d, ff), 16), dtype=torch.uint8, device=cuda)
        ops.grouped_ffn(x[a:a + n], [0, n], [es[i]], d, ff, G, h1, y1, w1)
        torch.cuda.synchronize()
        hd = (h[a:a + n].float() - h1.float()).norm() / h1.float().norm()
        assert hd.item() < 1e-3, (i, hd.item())          # bf16 h; a tile change moves the f32 sum order only
        rel = ((y[a:a + n] - y1).norm() / y1.norm()).item()
        assert rel < 1e-4, (i, rel)
    out = ~inside.to(cuda)
    assert bool((y[out] == -3.0).all()) and bool((h[out] == 7.0).all())


@pytest.mark.gpu
@pytest.mark.parametrize("d,ff", [(4096, 14336), (6144, 16384), (256, 896)])
def test_expert_gemv_graph_matches_eager(cuda, d, ff):
    """ds_w4_expert_gemv_graph (one launch of a cached device-resident graph:
    wait on the slot's ready event -> span events -> K4) gives the eager
    call's h and output bit for bit, on the first (capture) and on repeated
    (cached, events swapped) launches, after the waited-on copy landed; the
    device-clock K4 counter advances for the fused 8x7B launch."""
    import torch
    from paper_2509_07379_b200 import ops
    G = 128
    offs, total = _layout(d, ff, G)
    src = torch.zeros(total, dtype=torch.uint8, device=cuda)
    _lib.call("ds_w4_generate", 13, 1, 3, d, ff, G, _lib.ptr(src), _lib.stream_ptr())
    host = src.cpu().pin_memory()
    slot = torch.zeros_like(src)
    e = _expert_struct(slot, offs)
    x = _rand_bf16((1, d), 1.0, torch.Generator().manual_seed(5)).to(cuda)
    rw = torch.tensor([0.5], device=cuda)
    h_ref = torch.empty((1, ff), dtype=torch.bfloat16, device=cuda)
    a_ref = torch.zeros((1, d), device=cuda)
    slot.copy_(src)
    ops.expert_gemv(x, e, d, ff, G, h_ref, rw, 1, a_ref)
    torch.cuda.synchronize()
    cs = torch.cuda.Stream()
    h = torch.empty_like(h_ref)
    a = torch.zeros_like(a_ref)
    n0 = ops.k4_device_span()[1]
    for it in range(3):
        slot.zero_()
        a.zero_()
        torch.cuda.synchronize()
        ready = torch.cuda.Event()
        with torch.cuda.stream(cs):
            slot.copy_(host, non_blocking=True)        # the expert lands only on the copy stream
            ready.record(cs)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ops.expert_gemv_graph(x, e, d, ff, G, h, rw, 1, a, ready, ev0, ev1)
        torch.cuda.synchronize()
        assert torch.equal(h, h_ref), it
        assert torch.equal(a, a_ref), it
        assert ev0.elapsed_time(ev1) > 0
    # no wait event, no span events (a pinned expert outside the profiler's sample)
    a.zero_()
    ops.expert_gemv_graph(x, e, d, ff, G, h, rw, 1, a)
    torch.cuda.synchronize()
    assert torch.equal(a, a_ref)
    if (d, ff) == (4096, 14336):
        assert ops.k4_device_span()[1] >= n0 + 4
    ops.w4_graph_cache_clear()
