"""BASELINE config 4: Mixtral-8x7B-shaped W4 sweep, batch 1-32 x prompt
128-2048 — the dense-prefill (K3, tcgen05 grouped GEMM) vs sparse-decode
(K4, GEMV) crossover, measured per expert on the B200, and the per-layer
MoE compute vs host-link time at each (batch, prompt) point.

    python scripts/sweep.py [--shape mixtral-8x7b] [--out gpurun_out/sweep.json]

Per rows-per-expert R: K4 time (swiglu_gemv + down_gemv, R rows) and K3 time
(one-expert grouped FFN) with L2 flushed between iterations, CUDA events.
Per (batch B, prompt P): T = B*P prefill tokens -> expected activated experts
per layer |A| = M(1 - (1 - k/M)^T) and rows/expert T*k/|A|; prefill MoE
compute/layer = |A| * min(K3, K4)(rows) vs link time |A| * expert_bytes / H2D;
decode at batch B: |A_B| experts/layer with B*k/|A_B| rows each.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2509_07379_b200 import _lib, config as C, ops

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="mixtral-8x7b")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--out", default="gpurun_out/sweep.json")
a = ap.parse_args()
_lib.load()
dev = torch.device("cuda")
sh = C.load_shape(a.shape)
d, ff, G, M, k = sh.hidden, sh.ffn, sh.group_size, sh.num_experts, sh.top_k
offs, total = ops.expert_layout(d, ff, G)
NB = 3
blobs = torch.empty((NB, total), dtype=torch.uint8, device=dev)
for i in range(NB):
    ops.w4_generate(1, 0, i, d, ff, G, blobs[i])
es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timeit(fn):
    ts = []
    for i in range(a.iters + 2):
        flush.zero_()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn(i)
        e1.record(s)
        e1.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) / 1e3)
    return float(np.median(ts))


# host-link peak (pinned H2D of one expert blob)
host = torch.empty(total, dtype=torch.uint8, pin_memory=True)
cs = torch.cuda.Stream()
with torch.cuda.stream(cs):
    for _ in range(2):
        blobs[0].copy_(host, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    for _ in range(8):
        blobs[0].copy_(host, non_blocking=True)
    e1.record(cs)
e1.synchronize()
h2d = 8 * total / (e0.elapsed_time(e1) / 1e3) / 1e9
ops.w4_generate(1, 0, 0, d, ff, G, blobs[0])

rows_list = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]
per_rows = {}
maxR = max(rows_list)
x = torch.randn(maxR, d, device=dev).to(torch.bfloat16)
hbuf = torch.empty(maxR, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(maxR, d, device=dev)
rw = torch.ones(maxR, device=dev)
y = torch.empty(maxR, d, device=dev)
ws = torch.empty(max(ops.grouped_ffn_workspace(maxR, d, ff), 256), dtype=torch.uint8, device=dev)
for R in rows_list:
    # K4 takes <= 64 activation rows per call (decode batches); beyond that only K3
    t4 = timeit(lambda i: (ops.swiglu_gemv(x[:R], es[i % NB], d, ff, G, hbuf[:R]),
                           ops.down_gemv(hbuf[:R], es[i % NB], d, ff, G, rw, 1, acc[:R]))) if R <= 64 else float("inf")
    t3 = timeit(lambda i: ops.grouped_ffn(x[:R], [0, R], [es[i % NB]], d, ff, G, hbuf[:R], y[:R], ws))
    fl = 6.0 * R * d * ff
    per_rows[R] = {"k4_us": round(t4 * 1e6, 2) if t4 < float("inf") else None, "k3_us": round(t3 * 1e6, 2),
                   "k4_GBs": round(total / t4 / 1e9, 1), "k3_TFLOPs": round(fl / t3 / 1e12, 1),
                   "best": "K4 gemv" if t4 < t3 else "K3 tcgen05"}
    print(R, per_rows[R], flush=True)


def interp(R: float, key: str) -> float:
    rs = sorted(r for r in per_rows if per_rows[r][key] is not None)
    if R <= rs[0]:
        return per_rows[rs[0]][key] * 1e-6
    for lo, hi in zip(rs, rs[1:]):
        if R <= hi:
            f = (R - lo) / (hi - lo)
            return ((1 - f) * per_rows[lo][key] + f * per_rows[hi][key]) * 1e-6
    return per_rows[rs[-1]][key] * 1e-6 * R / rs[-1]


points = []
link_t = total / (h2d * 1e9)
for B in (1, 2, 4, 8, 16, 32):
    for P in (128, 256, 512, 1024, 2048):
        T = B * P
        A = M * (1 - (1 - k / M) ** T)
        rows = T * k / A
        comp = A * min(interp(rows, "k3_us"), interp(rows, "k4_us"))
        Ad = M * (1 - (1 - k / M) ** B)
        rows_d = B * k / Ad
        comp_d = Ad * min(interp(rows_d, "k3_us"), interp(rows_d, "k4_us"))
        points.append({"batch": B, "prompt": P, "prefill_tokens": T, "active_experts": round(A, 3),
                       "prefill_rows_per_expert": round(rows, 1),
                       "prefill_kernel": "K3" if interp(rows, "k3_us") < interp(rows, "k4_us") else "K4",
                       "prefill_moe_compute_ms_per_layer": round(1e3 * comp, 3),
                       "prefill_link_ms_per_layer": round(1e3 * A * link_t, 3),
                       "decode_active_experts": round(Ad, 3), "decode_rows_per_expert": round(rows_d, 2),
                       "decode_kernel": "K3" if interp(rows_d, "k3_us") < interp(rows_d, "k4_us") else "K4",
                       "decode_moe_compute_ms_per_layer": round(1e3 * comp_d, 3),
                       "decode_link_ms_per_layer": round(1e3 * Ad * link_t, 3)})
crossover = next((R for R in rows_list if per_rows[R]["k4_us"] is None or per_rows[R]["k3_us"] < per_rows[R]["k4_us"]),
                 None)
out = {"shape": sh.name, "expert_bytes": total, "h2d_GBs": round(h2d, 2), "per_rows": per_rows,
       "k3_beats_k4_from_rows": crossover, "points": points}
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(out, indent=1))
print(json.dumps({"h2d_GBs": out["h2d_GBs"], "crossover_rows": crossover}))
