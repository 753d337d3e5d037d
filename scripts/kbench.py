"""Standalone kernel timing (CUDA events, L2 flushed between iterations) for
the hot-path kernels at Mixtral-8x7B / 8x22B shapes; also the ncu target.

    python scripts/kbench.py [--shape mixtral-8x7b] [--iters 20] [--only k4,k3,k5,k1]
"""
import argparse, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2509_07379_b200 import _lib, ops, config as C, predictor as P
from paper_2509_07379_b200.engine import Engine  # noqa: F401

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="mixtral-8x7b")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--only", default="k4,k3,k5,k1")
ap.add_argument("--rows", type=int, default=128)
a = ap.parse_args()
dev = torch.device("cuda")
sh = C.load_shape(a.shape)
d, ff, G = sh.hidden, sh.ffn, sh.group_size
peaks = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()) \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650, "bf16_tflops": 1590}
offs, total = ops.expert_layout(d, ff, G)
NB = 4
blobs = torch.empty((NB, total), dtype=torch.uint8, device=dev)
for i in range(NB):
    ops.w4_generate(1, 0, i, d, ff, G, blobs[i])
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}


def timeit(fn, iters, flush_l2=True):
    ts = []
    for i in range(iters + 3):
        if flush_l2:
            flush.zero_()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); fn(i); e1.record(s); e1.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) / 1e3)
    return float(np.median(ts))


only = a.only.split(",")
if "k4" in only:
    x = (torch.randn(1, d, device=dev) * 1).to(torch.bfloat16)
    h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
    acc = torch.zeros(1, d, device=dev)
    rw = torch.ones(1, device=dev)
    es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
    t1 = timeit(lambda i: ops.swiglu_gemv(x, es[i % NB], d, ff, G, h), a.iters)
    t2 = timeit(lambda i: ops.down_gemv(h, es[i % NB], d, ff, G, rw, 1, acc), a.iters)
    b1 = offs[1] - offs[0]
    bytes13 = 2 * (ff * d // 2 + ff * (d // G) * 2 + ff * (d // G) // 2)
    bytes2 = d * ff // 2 + d * (ff // G) * 2 + d * (ff // G) // 2
    res["k4_swiglu"] = {"us": t1 * 1e6, "GBs": bytes13 / t1 / 1e9, "frac": bytes13 / t1 / 1e9 / peaks["hbm_gbs"]}
    res["k4_down"] = {"us": t2 * 1e6, "GBs": bytes2 / t2 / 1e9, "frac": bytes2 / t2 / 1e9 / peaks["hbm_gbs"]}
    # the roofline unit of bench.py: one expert = SwiGLU GEMV + down GEMV back to back
    t12 = timeit(lambda i: (ops.swiglu_gemv(x, es[i % NB], d, ff, G, h),
                            ops.down_gemv(h, es[i % NB], d, ff, G, rw, 1, acc)), a.iters)
    res["k4_expert"] = {"us": t12 * 1e6, "GBs": total / t12 / 1e9, "frac": total / t12 / 1e9 / peaks["hbm_gbs"]}
    # back to back without the flush kernel in between (4 experts x 91.5 MB cycle through a 126 MB L2,
    # so the weights are still cold); the flush kernel's different shared-memory carveout is not in front
    t12n = timeit(lambda i: (ops.swiglu_gemv(x, es[i % NB], d, ff, G, h),
                             ops.down_gemv(h, es[i % NB], d, ff, G, rw, 1, acc)), a.iters, flush_l2=False)
    res["k4_expert_noflush"] = {"us": t12n * 1e6, "GBs": total / t12n / 1e9,
                                "frac": total / t12n / 1e9 / peaks["hbm_gbs"]}
    # the engine's call: ds_w4_expert_gemv (one cooperative launch for R = 1)
    tf = timeit(lambda i: ops.expert_gemv(x, es[i % NB], d, ff, G, h, rw, 1, acc), a.iters)
    res["k4_expert_call"] = {"us": tf * 1e6, "GBs": total / tf / 1e9, "frac": total / tf / 1e9 / peaks["hbm_gbs"]}
    # the serving loop runs K4 after the GPU idled ~1-2 ms waiting on the host link:
    # same unit timed after an idle gap (no L2 flush kernel right before it)
    tis = []
    for i in range(a.iters + 3):
        torch.cuda.synchronize()
        time.sleep(0.002)                       # GPU idle, as while the link streams an expert
        s_ = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_)
        ops.swiglu_gemv(x, es[i % NB], d, ff, G, h)
        ops.down_gemv(h, es[i % NB], d, ff, G, rw, 1, acc)
        e1.record(s_)
        e1.synchronize()
        if i >= 3:
            tis.append(e0.elapsed_time(e1) / 1e3)
    ti = float(np.median(tis))
    # same, with one CTA spinning on a side stream during the gap (GPU kept busy)
    side = torch.cuda.Stream(priority=0)
    tws = []
    for i in range(a.iters + 3):
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            torch.cuda._sleep(int(2.2e6))           # ~1.1 ms at 1.9 GHz, overlapping the gap
        time.sleep(0.001)
        s_ = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_)
        ops.swiglu_gemv(x, es[i % NB], d, ff, G, h)
        ops.down_gemv(h, es[i % NB], d, ff, G, rw, 1, acc)
        e1.record(s_)
        e1.synchronize()
        if i >= 3:
            tws.append(e0.elapsed_time(e1) / 1e3)
    tw = float(np.median(tws))
    res["k4_expert_after_busy_gap"] = {"us": tw * 1e6, "GBs": total / tw / 1e9, "frac": total / tw / 1e9 / peaks["hbm_gbs"]}
    res["k4_expert_after_idle"] = {"us": ti * 1e6, "GBs": total / ti / 1e9, "frac": total / ti / 1e9 / peaks["hbm_gbs"]}
if "k3" in only:
    R = a.rows
    xp = (torch.randn(R, d, device=dev)).to(torch.bfloat16)
    hh = torch.empty(R, ff, dtype=torch.bfloat16, device=dev)
    y = torch.empty(R, d, device=dev)
    ws = torch.empty(max(ops.grouped_ffn_workspace(R, d, ff), 16), dtype=torch.uint8, device=dev)
    es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
    t = timeit(lambda i: ops.grouped_ffn(xp, [0, R], [es[i % NB]], d, ff, G, hh, y, ws), a.iters)
    fl = 6.0 * R * d * ff
    res["k3_grouped_ffn"] = {"rows": R, "us": t * 1e6, "TFLOPs": fl / t / 1e12, "frac": fl / t / 1e12 / peaks["bf16_tflops"]}
if "k5" in only:
    L, M, k = sh.num_layers, sh.num_experts, sh.top_k
    net = P.ExpertMLP(P.feature_length(L, M, k), M, seed=0)
    dm = net.device(dev)
    pop = torch.full((L, M), 1.0 / M, dtype=torch.float64, device=dev)
    aff = torch.full((L - 1, M, M), 1.0 / M, dtype=torch.float64, device=dev)
    hist = torch.randint(1, M + 1, (1, L * k), dtype=torch.int32, device=dev)
    tg = torch.full((1,), L // 2, dtype=torch.int32, device=dev)
    out = torch.empty(1, k, dtype=torch.int32, device=dev)
    t = timeit(lambda i: dm.predict_state(hist, tg, pop, aff, L, M, k, 0, k, out=out), a.iters, flush_l2=False)
    tc = timeit(lambda i: dm.predict_state(hist, tg, pop, aff, L, M, k, 0, k, out=out), a.iters, flush_l2=True)
    res["k5_predictor_B1"] = {"us_l2_warm": t * 1e6, "us_cold": tc * 1e6, "weight_bytes": dm.nbytes,
                              "GBs_cold": dm.nbytes / tc / 1e9}
if "k1" in only:
    for T in (1, 512):
        xx = torch.randn(T, d, device=dev).to(torch.bfloat16)
        wg = (torch.randn(sh.num_experts, d, device=dev) * 0.02).to(torch.bfloat16)
        idx = torch.empty(T, 2, dtype=torch.int32, device=dev)
        w = torch.empty(T, 2, device=dev)
        t = timeit(lambda i: ops.gate_topk(xx, wg, 2, idx, w), a.iters)
        res[f"k1_gate_T{T}"] = {"us": t * 1e6}
print(json.dumps(res, indent=1))
