"""Calibrate the reference CostModel (config.py:62-85) from B200 measurements
and check the simulator against the measured runtime.

    python scripts/calibrate_cost.py [--shape mixtral-8x7b] [--prefill 512] [--decode 16]
                                     [--out gpurun_out/calib.json]

1. Components, CUDA events, median of N:
   * link: pinned H2D of one expert blob (bandwidth) and of 4 KiB (latency);
   * non-MoE per layer: attention block (RMSNorm, QKV, RoPE, SDPA, O-proj,
     residual) for 1 decode token and for the T-token prefill pass;
   * gate (K1) at T = 1;
   * expert FFN: K4 (1 row) and K3 (grouped, 32..256 rows) -> an affine
     base + rows * per_token fit (the CostModel's expert compute model);
   * predictor (K5, B = 1).
2. The preset ``presets/<shape>-b200.json`` (reference schema: model + cost)
   written to --out (commit it by hand).
3. One request through ``Engine`` (prefill + decode, policy duoserve):
   its recorded routing and predictions are replayed through
   ``simulator.simulate_request`` with the calibrated cost, and the simulated
   TTFT / decode ms per token are reported next to the measured ones; the
   baselines (ondemand, prefetchall, oracle) are simulated on the same routing.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2509_07379_b200 import _lib, ops, config as C, simulator as S, trace as T
from paper_2509_07379_b200.model import KVCache, attention_block, init_dense_weights, rope_tables
from paper_2509_07379_b200.predictor import ExpertMLP, PrecomputedPredictor, feature_length

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="mixtral-8x7b")
ap.add_argument("--prefill", type=int, default=512)
ap.add_argument("--decode", type=int, default=16)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--out", default="gpurun_out/calib.json")
a = ap.parse_args()
_lib.load()
dev = torch.device("cuda")
sh = C.load_shape(a.shape)
d, ff, G, L, M, k = sh.hidden, sh.ffn, sh.group_size, sh.num_layers, sh.num_experts, sh.top_k
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timeit(fn, iters=a.iters, flush_l2=True, stream=None):
    ts = []
    s = stream or torch.cuda.current_stream()
    for i in range(iters + 2):
        if flush_l2:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn(i)
        e1.record(s)
        e1.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) / 1e3)
    return float(statistics.median(ts))


res = {}
# ---- link
offs, blob = ops.expert_layout(d, ff, G)
host = torch.empty(blob, dtype=torch.uint8).pin_memory()
dst = torch.empty(blob, dtype=torch.uint8, device=dev)
cs = torch.cuda.Stream()
def copies(n, src, dst_):
    def f(i):
        for _ in range(n):
            dst_.copy_(src, non_blocking=True)
    return f


with torch.cuda.stream(cs):
    t_blob = timeit(copies(8, host, dst), iters=5, flush_l2=False, stream=cs) / 8   # back to back, like the link
    small_h = torch.empty(4096, dtype=torch.uint8).pin_memory()
    small_d = torch.empty(4096, dtype=torch.uint8, device=dev)
    t_small = timeit(copies(1, small_h, small_d), iters=50, flush_l2=False, stream=cs)
bw = blob / t_blob
res["link"] = {"blob_bytes": blob, "blob_us": t_blob * 1e6, "small_us": t_small * 1e6, "GBs": bw / 1e9}
del host

# ---- non-MoE (attention block) and gate
W = init_dense_weights(sh, 1, device=dev)
P = a.prefill
kv = KVCache(sh, P + a.decode + 8, dev)
cos, sin = rope_tables(sh, P + a.decode + 8, dev)
hp = (torch.randn(P, d, device=dev) * 0.5).to(torch.bfloat16)
# eager prefill attention, back to back (the engine issues it eagerly too)
t_attn_p = timeit(lambda i: [attention_block(sh, W.layers[0], hp, kv, 0, 0, cos, sin) for _ in range(4)]) / 4
h1 = hp[:1].clone()
t_attn_d = timeit(lambda i: attention_block(sh, W.layers[0], h1, kv, 0, P, cos, sin))
idx = torch.empty(P, k, dtype=torch.int32, device=dev)
wt = torch.empty(P, k, device=dev)
t_gate = timeit(lambda i: ops.gate_topk(h1, W.layers[0]["wg"], k, idx[:1], wt[:1]))
t_gate_p = timeit(lambda i: ops.gate_topk(hp, W.layers[0]["wg"], k, idx, wt))
res["non_moe"] = {"attn_decode_us": t_attn_d * 1e6, "attn_prefill_us": t_attn_p * 1e6,
                  "gate_decode_us": t_gate * 1e6, "gate_prefill_us": t_gate_p * 1e6}

# ---- expert FFN: K4 at 1 row, K3 at 32..256 rows
NB = 3
blobs = torch.empty((NB, blob), dtype=torch.uint8, device=dev)
for i in range(NB):
    ops.w4_generate(1, 0, i, d, ff, G, blobs[i])
es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
x1 = (torch.randn(1, d, device=dev)).to(torch.bfloat16)
hb = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)
t_k4 = timeit(lambda i: (ops.swiglu_gemv(x1, es[i % NB], d, ff, G, hb),
                         ops.down_gemv(hb, es[i % NB], d, ff, G, rw, 1, acc)))
pts = [(1, t_k4)]
for R in (32, 64, 128, 256):
    xp = (torch.randn(R, d, device=dev)).to(torch.bfloat16)
    hh = torch.empty(R, ff, dtype=torch.bfloat16, device=dev)
    y = torch.empty(R, d, device=dev)
    ws = torch.empty(max(ops.grouped_ffn_workspace(R, d, ff), 16), dtype=torch.uint8, device=dev)
    pts.append((R, timeit(lambda i: ops.grouped_ffn(xp, [0, R], [es[i % NB]], d, ff, G, hh, y, ws))))
rows = np.array([p[0] for p in pts], dtype=np.float64)
ts = np.array([p[1] for p in pts])
per_tok, base = np.polyfit(rows, ts, 1)
res["expert"] = {"points_us": {int(r): t * 1e6 for r, t in pts}, "base_us": base * 1e6,
                 "per_token_us": per_tok * 1e6}

# ---- predictor K5 (B = 1)
net = ExpertMLP(feature_length(L, M, k), M, seed=0)
dm = net.device(dev)
pop = torch.full((L, M), 1.0 / M, dtype=torch.float64, device=dev)
aff = torch.full((L - 1, M, M), 1.0 / M, dtype=torch.float64, device=dev)
hist = torch.randint(1, M + 1, (1, L * k), dtype=torch.int32, device=dev)
tg = torch.full((1,), L // 2, dtype=torch.int32, device=dev)
out = torch.empty(1, k, dtype=torch.int32, device=dev)
t_pred = timeit(lambda i: dm.predict_state(hist, tg, pop, aff, L, M, k, 0, k, out=out), flush_l2=False)
res["predictor_us"] = t_pred * 1e6
del blobs, W, kv
torch.cuda.empty_cache()

# ---- preset (reference schema)
cfg = C.model_config_for_shape(sh, predictor_mem_bytes=dm.nbytes,
                               kv_reserve_bytes=2 * L * sh.n_kv_heads * (P + a.decode + 8) * sh.head_dim * 2)
cost = C.CostModel(link_bandwidth_bytes_per_s=bw, link_latency_s=max(t_small, 1e-7),
                   expert_compute_base_s=max(base, 1e-7), expert_compute_per_token_s=max(per_tok, 1e-9),
                   non_moe_compute_per_layer_s=t_attn_d, gate_compute_s=t_gate, predictor_latency_s=t_pred)
preset = json.loads(C.config_to_json(cfg, cost))
preset["model"]["name"] = f"{sh.name}-b200"
res["preset"] = preset
res["prefill_non_moe_s"] = t_attn_p + t_gate_p - t_gate

# ---- measured request vs simulated replay of its decisions
from bench import predictor_inputs  # noqa: E402
from paper_2509_07379_b200.engine import Engine  # noqa: E402
net, popm, affm = predictor_inputs(sh)
eng = Engine(sh, "duoserve", seed=0, device=dev, predictor=net, pop=popm, aff=affm,
             max_seq=P + a.decode + 8, max_prefill=P)
ids = torch.randint(0, sh.vocab, (P,), generator=torch.Generator().manual_seed(1))
meas = []
for rep in range(2):
    eng.reset()
    s = torch.cuda.current_stream()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(s)
    eng.prefill(ids.to(dev))
    e1.record(s)
    for _ in range(a.decode):
        eng.decode_step()
    e2.record(s)
    torch.cuda.synchronize()
    meas.append({"ttft_ms": e0.elapsed_time(e1), "decode_ms_per_token": e1.elapsed_time(e2) / a.decode})
m = meas[-1]
# decode non-MoE + gate as the engine runs it: the per-layer CUDA graph replay
if getattr(eng, "g_graphs", None):
    gr = eng.g_graphs[1]
    t_graph = timeit(lambda i: [gr.replay() for _ in range(8)], flush_l2=False) / 8
    res["non_moe"]["decode_graph_us"] = t_graph * 1e6
    cost = C.CostModel(link_bandwidth_bytes_per_s=cost.link_bandwidth_bytes_per_s,
                       link_latency_s=cost.link_latency_s, expert_compute_base_s=cost.expert_compute_base_s,
                       expert_compute_per_token_s=cost.expert_compute_per_token_s,
                       non_moe_compute_per_layer_s=max(t_graph - t_gate, 1e-7), gate_compute_s=t_gate,
                       predictor_latency_s=cost.predictor_latency_s)
    preset = json.loads(C.config_to_json(cfg, cost))
    preset["model"]["name"] = f"{sh.name}-b200"
    res["preset"] = preset
traces = [T.ActivationTrace(0, "prefill", t, tuple(tuple(int(e) for e in eng.paths_prefill[t, l]) for l in range(L)))
          for t in range(P)]
traces += [T.ActivationTrace(0, "decode", P + t, tuple(tuple(sorted(p)) for p in path))
           for t, path in enumerate(eng.paths_decode[:a.decode])]
table = {}
for r in eng.log:
    if r["phase"] == "decode" and "pred" in r:
        table[(0, P + r["token"], r["layer"])] = tuple(r["pred"])
pp = PrecomputedPredictor(table)
sim = {}
# the runtime's cancellation: depth x speculative chunk still in flight after the gate
cancel = eng.link.depth * eng.link.spec_chunk
for pol in ("duoserve", "duoserve+cancel", "oracle", "ondemand", "prefetchall"):
    mm, _, log = S.simulate_request(pol.split("+")[0], traces, cfg, cost, net=pp,
                                    prefill_non_moe_s=res["prefill_non_moe_s"],
                                    cancel_chunk_bytes=cancel if pol.endswith("+cancel") else None,
                                    return_log=True)
    sim[pol] = {"ttft_ms": mm.ttft_s * 1e3, "decode_ms_per_token": (mm.e2e_s - mm.ttft_s) * 1e3 / a.decode,
                "refetch_count": mm.refetch_count, "link_bytes": mm.link_bytes}
    if pol.startswith("duoserve"):
        rt = [dict(r, token=P + r["token"]) if "token" in r else r for r in eng.log]
        sim[pol]["log_equals_runtime"] = log == rt
res["request"] = {"measured": m, "simulated": sim, "prefill": P, "decode": a.decode}
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(res, indent=1) + "\n")
print(json.dumps(res, indent=1))
