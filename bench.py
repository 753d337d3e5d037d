#!/usr/bin/env python
"""Benchmark: Mixtral-8x7B-shaped W4 e2e latency (TTFT, decode tok/s) at
<= 15 % expert residency (BASELINE.json metric, configs[1]: batch 1, prefill
512 + decode 128, 1 x B200, random-init weights, synthetic prompt ids).

One "step" = one request through the public serving API: Engine.prefill
(512 prompt tokens) + 128 Engine.decode_step() calls, with the DuoServe
schedule (2k = 4 expert slots in HBM, all 256 experts streamed from pinned
host memory; predictor-driven decode prefetch).

    python bench.py [--steps K] [--warmup W] [--gpus N] [--config mixtral-8x7b]
    python bench.py --impl reference      # CPU oracle port of the reference path

Under torchrun (N > 1) every rank serves an independent replica (the path is
single-GPU by design; expert-parallel 8x22B is a separate
extension): scaling "weak", the time is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Mixtral-8x7B W4 e2e latency (TTFT, decode tok/s) at 15% expert residency"
UNIT = "ms/request (prefill 512 + decode 128, batch 1)"


def unit_for(args) -> str:
    return f"ms/request (prefill {args.prefill} + decode {args.decode}, batch 1)"


def workload_config(shape, args, n_requests: int = 1) -> dict:
    """The workload both arms measure (identical dicts, so the reference arm's
    line describes the same config); implementation details go to "setup"."""
    return {"workload": f"{shape.name}-shaped W4 random-init, batch 1, prefill {args.prefill} + decode "
                        f"{args.decode}",
            "model": shape.name, "global_batch": n_requests, "seq_len": args.prefill + args.decode,
            "prefill": args.prefill, "decode": args.decode,
            "l2": "inputs > L2: every expert byte is streamed from pinned host memory per request"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral-8x7b")
    ap.add_argument("--policy", default="duoserve", choices=["duoserve", "oracle", "ondemand", "prefetchall"])
    ap.add_argument("--prefill", type=int, default=512)
    ap.add_argument("--decode", type=int, default=128)
    ap.add_argument("--warmup-decode", type=int, default=None,
                    help="decode tokens per warm-up step (default: same as --decode)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the oracle check of the served request (routing, predicted sets, cache log)")
    ap.add_argument("--no-cancel", action="store_true",
                    help="paper-faithful decode: whole-expert prefetch, no cancellation of wrong prefetches")
    ap.add_argument("--chunk-mb", type=float, default=256.0,
                    help="chunk size of confirmed transfers (re-fetches, promoted prefetches); >= the expert = whole-expert copies")
    ap.add_argument("--link-depth", type=int, default=2)
    ap.add_argument("--pin-mb", type=float, default=-1.0,
                    help="residency-budget policy: HBM (MiB) for the most popular experts, pinned for the request; "
                         "-1 (default) = whatever keeps the measured peak under the residency cap, 0 = off")
    ap.add_argument("--residency-cap", type=float, default=0.15,
                    help="peak device bytes / W4 model bytes the auto pin budget stays under (PAPER: ~15 %%)")
    ap.add_argument("--predictor", default="trained", choices=["trained", "random"],
                    help="trained: the paper's preprocess on this model (serve calibration prompts on-demand, "
                         "count pop/aff on the GPU, train the ExpertMLP on the GPU); random: ExpertMLP(seed=0) "
                         "with pop/aff from synthetic traces (SURVEY.md §8d)")
    ap.add_argument("--calib-requests", type=int, default=4)
    ap.add_argument("--calib-decode", type=int, default=32)
    ap.add_argument("--train-epochs", type=int, default=15)
    ap.add_argument("--spec-chunk-mb", type=float, default=0.5,
                    help="chunk size of speculative (predicted) prefetches until the gate confirms them")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--ep", action="store_true",
                    help="under torchrun: expert parallelism (rank r owns experts e %% N == r, per-rank pinned "
                         "shard + cache, NCCL all-reduce combine) on ONE request instead of N replicas")
    ap.add_argument("--ep-combine", default="allreduce", choices=["allreduce", "alltoall"],
                    help="--ep combine collective: one all-reduce, or all_to_all_single + all-gather")
    ap.add_argument("--also-22b", type=int, default=1,
                    help="default 8x7B run on one GPU: also serve one Mixtral-8x22B request (BASELINE configs[2]) "
                         "in a subprocess after the timed region and attach its line as 'config_8x22b'")
    ap.add_argument("--sweep", action="store_true",
                    help="BASELINE config 4: batch x prompt grid through BatchEngine (one JSON document)")
    ap.add_argument("--sweep-batches", default="1,2,4,8,16,32")
    ap.add_argument("--sweep-prompts", default="128,256,512,1024,2048")
    ap.add_argument("--sweep-decode", type=int, default=16)
    ap.add_argument("--out", default=None, help="also write the JSON line to this file")
    return ap.parse_args()


# ----------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self) -> dict:
        self.f.flush()
        rows = []
        for line in Path(self.f.name).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return 0, 1, 0
    import torch
    import torch.distributed as dist
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    return dist.get_rank(), ws, lr


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


def ncu_traffic() -> dict:
    """DRAM bytes (read + write) per roofline unit from the committed ncu
    --set full captures (profiles/ncu_traffic.json, written by
    scripts/ncu_traffic.py), keyed like KernelProfiler's kernel names."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    return json.loads(p.read_text()) if p.exists() else {}


def predictor_inputs(shape, seed: int = 0):
    """ExpertMLP(d_in, 8, seed=0) + pop/aff from generate_traces(default_generator_params(L, 8, 0.8, seed=7))
    (SURVEY.md §8d)."""
    from paper_2509_07379_b200 import config as C, predictor as P, stats as S, trace as T
    cfg = C.model_config_for_shape(shape)
    ds = T.generate_traces(T.default_generator_params(shape.num_layers, shape.num_experts, 0.8, seed=7), cfg,
                           n_requests=4, decode_len=16, prefill_len=16)
    pop, aff = S.build_popularity(ds), S.build_affinity(ds)
    net = P.ExpertMLP(P.feature_length(shape.num_layers, shape.num_experts, shape.top_k), shape.num_experts,
                      seed=seed, meta={"L": shape.num_layers, "M": shape.num_experts, "k": shape.top_k,
                                       "affinity_mode": "pool"})
    return net, pop, aff


# ------------------------------------------------------------- CPU baseline
_CPU_W = {}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _cpu_weights(shape):
    """Dequantised fp32 weights of layer 0 (8 experts + the W4 attention
    projections), generated and dequantised by the oracle once per process
    (not timed: it stands in for loading the model)."""
    if shape.name in _CPU_W:
        return _CPU_W[shape.name]
    import torch
    from oracle import w4_ref
    d, ff, G, M = shape.hidden, shape.ffn, shape.group_size, shape.num_experts
    f32 = lambda c, s_, z, K, N: torch.from_numpy(w4_ref.bf16_bits_to_f32(w4_ref.dequant(c, s_, z, K, N, G)))
    experts = [[f32(*w4_ref.gen_linear(0, 0, e, m, K, N, G), K, N) for m, (K, N) in
                enumerate([(d, ff), (d, ff), (ff, d)])] for e in range(M)]
    hd = shape.head_dim
    nq = (shape.n_heads + 2 * shape.n_kv_heads) * hd
    wqkv = f32(*w4_ref.gen_linear(0, 0, 63, 0, d, nq, G), d, nq)
    wo = f32(*w4_ref.gen_linear(0, 0, 63, 1, shape.n_heads * hd, d, G), shape.n_heads * hd, d)
    _CPU_W[shape.name] = (experts, wqkv, wo)
    return _CPU_W[shape.name]


def cpu_reference_sample(shape, prefill: int, decode_sample: int = 2, threads: int | None = None,
                         do_prefill: bool = True) -> dict:
    """The reference path on the host cores (oracle port, torch fp32 on
    dequantised W4 weights): the prefill of `prefill` tokens through ALL L
    layers (RMSNorm, W4 q|k|v / o projections + causal attention, the gate of
    oracle/routing_ref — HF MixtralTopKRouter semantics — and the grouped
    SwiGLU experts), then `decode_sample` decode tokens through all L layers
    (attention over the cache, gate, 2 experts, the reference predictor step
    construct_input + ExpertMLP eval + topk, predictor.py:80-106/197-232/
    419-421) and lm_head.  Every layer reuses layer 0's dequantised weights
    (identical arithmetic cost; dequantising 256 experts in numpy is model
    loading, not serving).  Decode is scaled from the sample to 128 tokens."""
    import numpy as np
    import torch
    import torch.nn.functional as F
    from oracle import predictor_ref, routing_ref, w4_ref
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    d, M, k, L = shape.hidden, shape.num_experts, shape.top_k, shape.num_layers
    nh, nkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim
    experts, wqkv, wo = _cpu_weights(shape)
    rng = np.random.default_rng(0)
    wg_bits = [w4_ref.bf16_round_bits((rng.standard_normal((M, d)) * 0.02).astype(np.float32)) for _ in range(L)]
    lm_head = torch.randn(d, shape.vocab) * 0.02
    net = predictor_ref.RefNet(predictor_ref_dim(shape), M, (2048, 1024, 512, 256, 128, 64), 0)
    pop = np.full((L, M), 1.0 / M)
    aff = np.full((L - 1, M, M), 1.0 / M)
    bf = lambda t: t.to(torch.bfloat16).float()

    def norm(x):
        return bf(x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + 1e-5))

    def attention(x, K_cache, V_cache, pos0):
        T = x.shape[0]
        y = bf(norm(x) @ wqkv.T)
        q = y[:, :nh * hd].view(T, nh, hd).transpose(0, 1)
        kk = y[:, nh * hd:(nh + nkv) * hd].view(T, nkv, hd).transpose(0, 1)
        vv = y[:, (nh + nkv) * hd:].view(T, nkv, hd).transpose(0, 1)
        K_cache = kk if K_cache is None else torch.cat([K_cache, kk], 1)
        V_cache = vv if V_cache is None else torch.cat([V_cache, vv], 1)
        o = F.scaled_dot_product_attention(q.unsqueeze(0), K_cache.unsqueeze(0), V_cache.unsqueeze(0),
                                           is_causal=pos0 == 0 and T > 1, enable_gqa=True)[0]
        return bf(x + o.transpose(0, 1).reshape(T, nh * hd) @ wo.T), K_cache, V_cache

    def moe(x, l):
        a = norm(x)
        bits = a.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        idx, w = routing_ref.topk_route(routing_ref.gate_logits(bits, wg_bits[l]), k)
        out = torch.zeros_like(a)
        wt = torch.from_numpy(w)
        for e in range(M):
            for j in range(k):
                rows = np.nonzero(idx[:, j] == e)[0]
                if rows.size:
                    W1, W3, W2 = experts[e]
                    xr = a[rows]
                    h = bf(F.silu(xr @ W1.T) * (xr @ W3.T))
                    out[rows] += wt[rows, j:j + 1] * (h @ W2.T)
        return bf(x + out), idx

    x0 = bf(torch.randn(prefill, d))
    caches = [[None, None] for _ in range(L)]
    t_prefill = None
    x = x0
    if do_prefill:
        t0 = time.perf_counter()
        for l in range(L):
            x, caches[l][0], caches[l][1] = attention(x, None, None, 0)
            x, _ = moe(x, l)
        (norm(x[-1:]) @ lm_head).argmax()
        t_prefill = time.perf_counter() - t0
    else:                                          # a short context for the decode sample
        for l in range(L):
            _, caches[l][0], caches[l][1] = attention(x0[:16], None, None, 0)
    t0 = time.perf_counter()
    xt = x[-1:]
    for step in range(decode_sample):
        path = []
        for l in range(L):
            xt, caches[l][0], caches[l][1] = attention(xt, caches[l][0], caches[l][1], 1)
            xt, idx = moe(xt, l)
            path.append(tuple(int(e) for e in idx[0]))
            if l + 1 < L:                          # the predictor step for the next layer
                feats = predictor_ref.features(tuple(path) + ((0, 1),) * (L - l - 1), l + 1, pop, aff)
                predictor_ref.topk_indices(net.forward(feats), k)
        (norm(xt) @ lm_head).argmax()
    t_dec = (time.perf_counter() - t0) / decode_sample
    return {"ttft_ms": 1e3 * t_prefill if t_prefill is not None else None, "decode_ms_per_token": 1e3 * t_dec,
            "cores": threads, "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "timed_s": round((t_prefill or 0.0) + t_dec * decode_sample, 2),
            "sample": (f"{shape.name} shape, torch fp32 on dequantised W4 weights: prefill of {prefill} tokens "
                       f"through all {L} layers (attention + gate + grouped SwiGLU experts) timed in full"
                       if do_prefill else f"{shape.name} shape, torch fp32 on dequantised W4 weights") +
                      f"; {decode_sample} decode tokens through all {L} layers (attention, gate, 2 experts, "
                      f"reference predictor step) timed and scaled to the request's decode length; every "
                      f"layer reuses layer 0's weights (same arithmetic)"}


def cpu_baseline_entry(shape, prefill: int, decode: int, unit: str = UNIT) -> dict:
    """cpu_baseline object: all host threads (the headline) plus a 1-thread
    decode arm."""
    cb = cpu_reference_sample(shape, prefill)
    one = cpu_reference_sample(shape, prefill, decode_sample=1, threads=1, do_prefill=False)
    v = cb["ttft_ms"] + decode * cb["decode_ms_per_token"]
    return {"value": round(v, 1), "unit": unit, "cores": cb["cores"], "kind": "port", "sample": cb["sample"],
            "cpu_model": cb["cpu_model"], "nproc": cb["nproc"], "ttft_ms": round(cb["ttft_ms"], 1),
            "decode_ms_per_token": round(cb["decode_ms_per_token"], 1), "timed_s": cb["timed_s"],
            "single_thread": {"cores": 1, "decode_ms_per_token": round(one["decode_ms_per_token"], 1),
                              "timed_s": one["timed_s"]}}


def parity_leg(eng, args, shape, net, pop, aff, timed: dict, one_step) -> dict:
    """Checker leg (after the timed region; the oracle is test infrastructure):
    the timed request's predicted sets and cache log vs oracle/predictor_ref +
    oracle/sim_ref, then one more (untimed) serve of the same request with the
    gate inputs captured: routing teacher-forced vs oracle/routing_ref, and
    its cache log equal to the timed one (determinism)."""
    from oracle import check_request, predictor_ref
    L, k = shape.num_layers, shape.top_k
    t0 = time.time()
    ref_net = None
    if args.policy == "duoserve":
        # the served net through the reference's container format (predictor.py:577-646)
        from paper_2509_07379_b200 import predictor as P
        with tempfile.TemporaryDirectory() as td:
            P.save_model(net, Path(td) / "net.bin")
            ref_net = predictor_ref.load_container(Path(td) / "net.bin")
    pol = "duoserve" if args.policy == "duoserve" else args.policy
    out = {}
    if args.policy in ("duoserve", "ondemand", "prefetchall") and not eng.ep:
        out.update(check_request.check_request(timed["log"], timed["paths_prefill"], timed["paths_decode"], L, k,
                                               ref_net, pop.values if pop is not None else None,
                                               aff.values if aff is not None else None, policy=pol,
                                               pinned=sorted(eng.pinned) or None))
    eng.capture = []
    rerun = one_step(len(timed["paths_decode"]))
    cap, eng.capture = eng.capture, None
    out["routing"] = check_request.check_routing(cap, [eng.W.layers[l]["wg"] for l in range(L)], k)
    out["rerun_log_equal"] = rerun["log"] == timed["log"]
    out["rerun_tokens_equal"] = rerun["tokens"] == timed["tokens"]
    out["check_s"] = round(time.time() - t0, 1)
    return out


def calibrate(shape, args, serve_kw, store, rank, ws, ep):
    """The paper's preprocess on the served model:
    serve --calib-requests prompts (seeds disjoint from the timed request's)
    with on-demand scheduling while the gate's device counters record
    popularity / affinity, train the ExpertMLP on the GPU, evaluate it on the
    held-out requests.  Returns (PreprocessResult, dense weights, store) so
    the serving engine reuses the weights and the pinned expert store."""
    import torch
    from paper_2509_07379_b200.engine import Engine
    from paper_2509_07379_b200.preprocess import preprocess
    col = Engine(shape, "ondemand", store=store, collect_stats=True, **serve_kw)
    g = torch.Generator().manual_seed(10_000 + args.seed + (0 if ep else 1000 * rank))
    prompts = [torch.randint(0, shape.vocab, (args.prefill,), generator=g) for _ in range(args.calib_requests)]
    pre = preprocess(col, prompts, args.calib_decode, epochs=args.train_epochs, seed=args.seed)
    if ep is not None and ws > 1:
        # every rank saw the same routing; serve rank 0's net everywhere (bitwise identical predictions)
        import torch.distributed as dist
        obj = [pre if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        pre = obj[0]
    dense, store = col.W, col.store
    col.close()
    del col
    torch.cuda.empty_cache()
    return pre, dense, store


def preprocess_summary(pre, shape) -> dict:
    r = pre.train_report
    return {"table": pre.table(shape.name), "timings_s": pre.timings_s, "n_traces": pre.n_traces,
            "train": {"epochs": r.epochs, "n_samples": r.n_samples, "batch_size": r.batch_size,
                      "first_loss": round(r.epoch_losses[0], 5) if r.epoch_losses else None,
                      "last_loss": round(r.epoch_losses[-1], 5) if r.epoch_losses else None}}


def predictor_ref_dim(shape):
    return shape.num_layers * shape.top_k + 2 * shape.num_experts + 1


# ------------------------------------------------------------------ arms
def run_reference(args):
    """The reference path on the host cores (see cpu_reference_sample).  Each
    step is one bounded sample (the full prefill through all L layers plus a
    few decode tokens); `value` is the ms/request it implies, `ms_per_step` the
    wall time a step actually took, so steps x ms_per_step is this run's own
    timed region."""
    rank, ws, _ = dist_init()
    if rank != 0:
        return
    from paper_2509_07379_b200.config import load_shape
    shape = load_shape(args.config)
    vals, walls = [], []
    samp = None
    for i in range(args.warmup + args.steps):
        w0 = time.perf_counter()
        r = cpu_reference_sample(shape, args.prefill)
        w = time.perf_counter() - w0
        if i >= args.warmup:
            vals.append(r["ttft_ms"] + args.decode * r["decode_ms_per_token"])
            walls.append(1e3 * w)
            samp = r
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 1), "unit": unit_for(args), "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(statistics.median(walls), 1),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": workload_config(shape, args),
            "ttft_ms": round(samp["ttft_ms"], 1),
            "decode_tok_s": round(1e3 / samp["decode_ms_per_token"], 3),
            "value_from_sample": "ttft (measured, all layers) + decode tokens x measured ms/token of the sample",
            "cpu_baseline": {"value": round(v, 1), "unit": unit_for(args), "cores": samp["cores"], "kind": "port",
                             "sample": samp["sample"], "cpu_model": samp["cpu_model"], "nproc": samp["nproc"]},
            "e2e": {"value": round(v, 1), "unit": unit_for(args), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    rank, ws, lr = dist_init()
    dev = torch.device("cuda", lr)
    torch.cuda.set_device(dev)
    from paper_2509_07379_b200 import numa
    numa_info = numa.bind_to_gpu_node(lr)    # pinned store + link threads on the GPU's own socket
    from paper_2509_07379_b200 import _lib, ops
    _lib.load()                          # fail loudly if the CUDA library is missing
    from paper_2509_07379_b200.config import load_shape
    from paper_2509_07379_b200.engine import Engine
    shape = load_shape(args.config)
    t_setup = time.time()
    if args.pin_mb > 0 and args.policy == "prefetchall":
        raise SystemExit("--pin-mb does not apply to --policy prefetchall (every expert is streamed by design)")
    wd = args.warmup_decode if args.warmup_decode is not None else args.decode
    # replicas: an independent request per rank; EP: every rank serves the same request
    gen = torch.Generator().manual_seed(args.seed + (0 if args.ep else 1000 * rank))
    ids_host = torch.randint(0, shape.vocab, (args.prefill,), generator=gen).pin_memory()
    ep = None
    if args.ep and ws > 1:
        from paper_2509_07379_b200.ep import EPConfig
        ep = EPConfig(rank, ws, combine=args.ep_combine)
    store = None
    if ws > 1 and ep is None:
        # replicas of one model: one shared pinned copy of the expert store per
        # (host, PID namespace, NUMA node) — i.e. one per socket
        from paper_2509_07379_b200.engine import HostExpertStore
        grp, members = numa.store_sharing_group(numa_info["node"])
        if len(members) > 1:
            store = HostExpertStore(shape, args.seed, dev, shared_group=grp)
    n_record = max(args.decode, wd)
    serve_kw = dict(seed=args.seed, device=dev, ep=ep, max_seq=args.prefill + max(n_record, args.calib_decode) + 8,
                    max_prefill=args.prefill, cancel_mispredicted=not args.no_cancel, chunk_mb=args.chunk_mb,
                    link_depth=args.link_depth, spec_chunk_mb=args.spec_chunk_mb)
    needs_stats = args.policy in ("duoserve", "oracle") or (args.pin_mb != 0 and args.policy != "prefetchall")
    pre = None
    dense = None
    if needs_stats and args.predictor == "trained" and args.policy != "prefetchall":
        # the paper's preprocess on this model, on this GPU
        pre, dense, store = calibrate(shape, args, serve_kw, store, rank, ws, ep)
        net, pop, aff = pre.net, pre.pop, pre.aff
    elif needs_stats:
        net, pop, aff = predictor_inputs(shape)
    else:
        net, pop, aff = None, None, None
    if args.policy == "oracle":
        # record the routing once with the predictor-driven engine, then replay
        # it as the perfect predictor (SPEC DuoServeOracle) on the same weights
        rec = Engine(shape, "duoserve", dense=dense, store=store, predictor=net, pop=pop, aff=aff, **serve_kw)
        rec.reset()
        rec.generate(ids_host, n_record + 1)
        eng = Engine(shape, "oracle", dense=rec.W, store=rec.store, oracle_paths=rec.paths_decode, pop=pop,
                     **serve_kw)
        del rec
    else:
        eng = Engine(shape, args.policy, dense=dense, store=store, predictor=net, pop=pop, aff=aff, **serve_kw)
    setup_s = time.time() - t_setup
    prof = eng.enable_profile()
    eng.link_peak_gbs()

    def one_step(n_decode: int):
        eng.reset()
        c0 = eng.h2d_bytes()
        s = torch.cuda.current_stream()
        e0, e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), \
            torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record(s)
        ids = ids_host.to(dev, non_blocking=True)       # H2D of the prompt inside the step
        tok0 = eng.prefill(ids)                          # returns a host int (D2H)
        e1.record(s)
        w1 = time.perf_counter()
        toks = [tok0]
        for _ in range(n_decode):
            toks.append(eng.decode_step())
        e2.record(s)
        torch.cuda.synchronize()
        w2 = time.perf_counter()
        return {"ttft_ms": e0.elapsed_time(e1), "decode_ms": e1.elapsed_time(e2),
                "floors": eng.streamed_bytes_floor(),
                "host_wait_ms": {k_: round(1e3 * v_, 1) for k_, v_ in eng.host_wait.items()},
                "e2e_wall_ms": 1e3 * (w2 - w0), "ttft_wall_ms": 1e3 * (w1 - w0),
                "h2d_experts": eng.h2d_bytes() - c0, "tokens": toks,
                "d2h": eng.d2h_bytes, "log": eng.log, "paths_prefill": eng.paths_prefill,
                "paths_decode": eng.paths_decode}

    # first warm-up step without pinned experts: its peak sizes the residency budget
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    one_step(wd)
    base_peak = torch.cuda.max_memory_allocated(dev)
    pin_info = {"budget_bytes": 0, "experts": 0}
    if args.pin_mb != 0 and args.policy != "prefetchall":
        cap_bytes = int(args.residency_cap * shape.total_bytes)
        budget = int(args.pin_mb * 2**20) if args.pin_mb > 0 else cap_bytes - base_peak - (64 << 20)
        n_pin = eng.pin_experts(pop, budget) if budget > 0 else 0
        pin_info = {"budget_bytes": max(budget, 0), "experts": n_pin, "peak_before_pinning": int(base_peak),
                    "cap_bytes": cap_bytes, "chosen_by": "popularity measured on this model's calibration requests"
                    if pre is not None else "popularity of the synthetic traces"}
    for _ in range(max(args.warmup - 1, 0)):
        one_step(wd)
    prof.reset()
    k4dev0 = ops.k4_device_span()                # device-clock K4 / K3 totals before the timed steps
    k3dev0 = ops.k3_device_span()
    torch.cuda.reset_peak_memory_stats(dev)     # residency = peak of the serving loop, not of setup
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    res = []
    with ClockSampler(lr) as clk:
        torch.cuda.nvtx.range_push("timed")          # ncu --nvtx --nvtx-include "timed/"
        for _ in range(args.steps):
            res.append(one_step(args.decode))
        torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    # one extra, untimed step with the device timeline on (per-chunk timing
    # events): link busy fraction and copy/compute overlap fraction
    n_spans = {n: len(v) for n, v in prof.spans.items()}     # the roofline uses the timed steps only
    k4dev1 = ops.k4_device_span()
    k3dev1 = ops.k3_device_span()
    tl = eng.enable_timeline()
    eng.reset()
    tl.begin()
    timeline_bytes = one_step(args.decode)["h2d_experts"]
    timeline = tl.end()
    ms_step = statistics.median(r["ttft_ms"] + r["decode_ms"] for r in res)
    e2e_ms = statistics.median(r["e2e_wall_ms"] for r in res)
    if ws > 1:
        t = torch.tensor([ms_step, e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step, e2e_ms = t.tolist()
    if rank != 0:
        return
    r0 = res[len(res) // 2]
    ttft = statistics.median(r["ttft_ms"] for r in res)
    dec_ms = statistics.median(r["decode_ms"] for r in res)
    peaks = measured_peaks()
    link_gbs = eng.link_peak_gbs()
    h2d_step = r0["h2d_experts"] + args.prefill * 8
    prof.spans = {n: v[:n_spans[n]] for n, v in prof.spans.items() if n in n_spans}
    kern = prof.summary(peaks)
    traffic = ncu_traffic()
    for kk in kern["all"] + ([kern["dominant"]] if kern["dominant"] else []):
        kk["peak_of"] = "fallback (B200_PROFILING.md)" if peaks.get("_fallback") else "measured (MEASURED_PEAKS.json)"
        if kk["kernel"].startswith("K4") and k4dev1[1] > k4dev0[1]:
            # every fused K4 launch of the timed steps on the device clock
            # (first CTA entry -> last CTA exit): the kernel's own duration; the
            # event spans above also hold ~20 us of event-timestamp cost per
            # span while the copy engine streams (scripts/launchprobe.cu)
            n_dev = k4dev1[1] - k4dev0[1]
            us = (k4dev1[0] - k4dev0[0]) / 1e3 / n_dev
            ach = kk["bytes_per_launch"] / us / 1e3
            kk["device_clock"] = {"launches": n_dev, "avg_us": round(us, 2), "achieved": round(ach, 1),
                                  "frac": round(ach / kk["peak"], 4),
                                  "how": "%globaltimer, first CTA entry -> last CTA exit, every launch"}
        if kk["kernel"].startswith("K3") and k3dev1[1] > k3dev0[1]:
            # every timed grouped-FFN call on the device clock (GEMM1's first
            # CTA entry -> a one-thread kernel right after the call's last one)
            n_dev = k3dev1[1] - k3dev0[1]
            us = (k3dev1[0] - k3dev0[0]) / 1e3 / n_dev
            ach = kk["flops_per_launch"] / us / 1e6
            kk["device_clock"] = {"launches": n_dev, "avg_us": round(us, 2), "achieved": round(ach, 1),
                                  "frac": round(ach / kk["peak"], 4),
                                  "how": "%globaltimer, GEMM1 first CTA entry -> span-close kernel, every call"}
        t = traffic.get(kk["kernel"])
        if t is not None:
            kk["traffic"] = t["bytes_per_unit"]
            kk["traffic_source"] = t["source"]
    res_b = eng.resident_bytes()
    peak_dev = torch.cuda.max_memory_allocated(dev)
    line = {
        "metric": METRIC, "value": round(ms_step, 1), "unit": unit_for(args), "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 1), "higher_is_better": False,
        "scaling": "strong" if ep else "weak",
        "vs_baseline": None, "dtype": "bf16 activations, W4 (int4 g128) experts, f32 accumulate",
        "data": "synthetic (random-init W4 experts from a counter-based generator, random prompt ids)",
        "config": workload_config(shape, args, 1 if ep else ws),
        "setup": {"serving": f"1 request per GPU, policy {args.policy}"
                             f"{'' if args.no_cancel else ' + chunked cancellable prefetch'}",
                  "parallelism": (f"ep{ws}-{ep.combine}" if ep else f"replicas{ws}") if ws > 1 else "single-gpu",
                  "expert_slots": eng.n_slots, "numa": numa_info},
        "ttft_ms": round(ttft, 2), "decode_tok_s": round(args.decode / (dec_ms / 1e3), 3),
        "decode_ms_per_token": round(dec_ms / args.decode, 3),
        "residency": {"peak_device_bytes": int(peak_dev), "model_bytes": int(shape.total_bytes),
                      "fraction": round(peak_dev / shape.total_bytes, 4), **{k: int(v) for k, v in res_b.items()}},
        "link": {"h2d_bytes_per_request": int(r0["h2d_experts"]),
                 "achieved_gbs": round(r0["h2d_experts"] / ((ttft + dec_ms) / 1e3) / 1e9, 2),
                 "peak_gbs_measured": round(link_gbs, 2),
                 "frac": round(r0["h2d_experts"] / ((ttft + dec_ms) / 1e3) / 1e9 / link_gbs, 3),
                 "ttft_floor_ms": round(eng.prefill_bytes_floor() / link_gbs / 1e6, 1),
                 "decode_floor_ms_per_token": round(eng.decode_bytes_floor() / link_gbs / 1e6, 2),
                 "pinned_aware_floor": {
                     "ttft_ms": round(r0["floors"]["prefill_bytes"] / link_gbs / 1e6, 1),
                     "decode_ms_per_token": round(r0["floors"]["decode_bytes_per_token"] / link_gbs / 1e6, 2),
                     "request_ms": round((r0["floors"]["prefill_bytes"] + args.decode *
                                          r0["floors"]["decode_bytes_per_token"]) / link_gbs / 1e6, 1),
                     "frac_of_measured": round((r0["floors"]["prefill_bytes"] + args.decode *
                                                r0["floors"]["decode_bytes_per_token"]) / link_gbs / 1e6 /
                                               (r0["ttft_ms"] + r0["decode_ms"]), 3)},
                 "timeline": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in timeline.items()},
                 "busy_gbs": round(timeline_bytes / (timeline["copy_busy_ms"] / 1e3) / 1e9, 2)
                 if timeline["copy_busy_ms"] else None},
        "roofline": kern["dominant"],
        "kernels": kern["all"],
        "gpu_launches": kern["launches"],
        "e2e": {"value": round(e2e_ms, 1), "unit": unit_for(args), "h2d_bytes_per_step": int(h2d_step),
                "d2h_bytes_per_step": int(r0["d2h"])},
        "clocks": clk.summary(),
        "setup_s": round(setup_s, 1),
        "predictor": {**eng.hit_summary(), "source": args.predictor,
                      "host_wait_ms_per_request": r0.get("host_wait_ms"),
                      **({"preprocess": preprocess_summary(pre, shape)} if pre is not None else {})},
        "pinning": pin_info,
    }
    if not args.no_parity and rank == 0:
        line["parity"] = parity_leg(eng, args, shape, net, pop, aff, r0, one_step)
    if not args.no_cpu_baseline and ws == 1:
        line["cpu_baseline"] = cpu_baseline_entry(shape, args.prefill, args.decode, unit_for(args))
    if args.also_22b and ws == 1 and shape.name == "mixtral-8x7b" and args.policy == "duoserve":
        # free this engine's device and pinned host memory, then BASELINE configs[2] in its own process
        st_ = eng.store
        eng.close()
        del eng, prof, tl, one_step, dense, res, r0
        st_.close()
        del st_
        store = None
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        if hasattr(torch._C, "_host_emptyCache"):
            torch._C._host_emptyCache()              # return the cached pinned store to the OS
        line["config_8x22b"] = run_22b_subprocess(args)
    out = json.dumps(line)
    print(out)
    if args.out:
        Path(args.out).write_text(out + "\n")


def run_22b_subprocess(args, timeout_s: int = 900) -> dict:
    """BASELINE configs[2] (Mixtral-8x22B-shaped W4, batch 1, prefill 512) on
    this GPU through the same public API, in a child process (its 70 GB
    pinned expert store and any failure stay out of the headline run): one
    warm-up and one timed request, decode 32 tokens, auto pinning under the
    15 % cap, ExpertMLP(seed=0) predictor (no calibration pass)."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--config", "mixtral-8x22b", "--steps", "1", "--warmup", "1",
           "--decode", "32", "--predictor", "random", "--no-cpu-baseline", "--also-22b", "0",
           "--prefill", str(args.prefill)]
    t0 = time.time()
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s)
    except subprocess.TimeoutExpired:
        return {"error": f"timed out after {timeout_s} s"}
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if r.returncode != 0 or not lines:
        return {"error": f"rc={r.returncode}", "stderr_tail": r.stderr[-600:]}
    d = json.loads(lines[-1])
    keep = ("value", "unit", "ttft_ms", "decode_tok_s", "decode_ms_per_token", "residency", "link", "roofline",
            "predictor", "pinning", "parity", "clocks", "config", "setup", "e2e")
    out = {k: d[k] for k in keep if k in d}
    out["command"] = " ".join(cmd[1:])
    out["wall_s"] = round(time.time() - t0, 1)
    return out


def run_sweep(args):
    """BASELINE config 4 (Mixtral-8x7B W4, batch 1-32 x prompt 128-2048): per
    grid point one warm-up and one timed request of B sequences through
    BatchEngine (prefill B x P, then --sweep-decode decode steps), measured
    with CUDA events: TTFT, decode ms/step, tokens/s, activated experts per
    layer (prefill and decode), rows per expert (the K4 GEMV vs tcgen05 GEMM
    crossover), predictor hit rates, host-link bytes and peak device bytes."""
    import torch
    from paper_2509_07379_b200 import _lib
    from paper_2509_07379_b200.config import load_shape
    from paper_2509_07379_b200.engine import BatchEngine, Engine
    _lib.load()
    dev = torch.device("cuda", 0)
    shape = load_shape(args.config)
    batches = [int(x) for x in args.sweep_batches.split(",")]
    prompts = [int(x) for x in args.sweep_prompts.split(",")]
    D = args.sweep_decode
    t0 = time.time()
    serve_kw = dict(seed=args.seed, device=dev, max_seq=args.prefill + max(args.calib_decode, D) + 8,
                    max_prefill=args.prefill, cancel_mispredicted=not args.no_cancel, chunk_mb=args.chunk_mb,
                    link_depth=args.link_depth, spec_chunk_mb=args.spec_chunk_mb)
    if args.predictor == "trained":
        pre, dense, store = calibrate(shape, args, serve_kw, None, 0, 1, None)
        net, pop, aff = pre.net, pre.pop, pre.aff
    else:
        net, pop, aff = predictor_inputs(shape)
        tmp = Engine(shape, "ondemand", **serve_kw)
        dense, store = tmp.W, tmp.store
        tmp.close()
        del tmp
    points = []
    for P in prompts:
        for B in batches:
            eng = BatchEngine(shape, "duoserve", batch=B, max_prompt=P, max_seq=P + D + 8, dense=dense,
                              store=store, predictor=net, pop=pop, aff=aff, seed=args.seed, device=dev,
                              cancel_mispredicted=not args.no_cancel, chunk_mb=args.chunk_mb,
                              link_depth=args.link_depth, spec_chunk_mb=args.spec_chunk_mb)
            g = torch.Generator().manual_seed(args.seed + 7 * B + P)
            ids = torch.randint(0, shape.vocab, (B, P), generator=g).pin_memory()
            prof = eng.enable_profile()
            res = None
            torch.cuda.reset_peak_memory_stats(dev)
            for it in range(2):                       # warm-up, timed
                eng.reset()
                prof.reset()
                c0 = eng.h2d_bytes()
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                torch.cuda.synchronize()
                e0.record()
                eng.prefill(ids.to(dev, non_blocking=True))
                e1.record()
                for _ in range(D):
                    eng.decode_step()
                e2.record()
                torch.cuda.synchronize()
                res = (e0.elapsed_time(e1), e1.elapsed_time(e2), eng.h2d_bytes() - c0)
            ttft, dec_ms, h2d = res
            L = shape.num_layers
            pre_act = [len(r["activated"]) for r in eng.log if r["phase"] == "prefill"]
            dec_act = [len(r.get("gate", r.get("fetch", []))) for r in eng.log if r["phase"] == "decode"]
            rows = [r for _, _, gates in eng._batch_sets for r in gates]
            kern = prof.summary(measured_peaks())
            hs = eng.hit_summary()
            par = None
            if not args.no_parity:               # oracle checker leg (test infrastructure, untimed)
                from oracle import check_request, predictor_ref
                from paper_2509_07379_b200 import predictor as P_
                with tempfile.TemporaryDirectory() as td:
                    P_.save_model(net, Path(td) / "net.bin")
                    ref_net = predictor_ref.load_container(Path(td) / "net.bin")
                par = check_request.check_request_batch(eng.log, eng.paths_prefill, eng.paths_decode,
                                                        eng._batch_sets, shape.num_layers, shape.top_k, ref_net,
                                                        pop.values, aff.values)
            points.append({
                "batch": B, "prompt": P, "decode_steps": D, "ttft_ms": round(ttft, 2),
                "decode_ms_per_step": round(dec_ms / D, 3),
                "decode_tok_s": round(B * D / (dec_ms / 1e3), 2),
                "prefill_tok_s": round(B * P / (ttft / 1e3), 1),
                "activated_per_layer": {"prefill": round(sum(pre_act) / max(len(pre_act), 1), 3),
                                        "decode": round(sum(dec_act) / max(len(dec_act), 1), 3)},
                "decode_rows_per_expert": round(B * shape.top_k / max(sum(dec_act) / max(len(dec_act), 1), 1e-9), 3),
                "predictor": {k: hs[k] for k in ("topk_hit_rate", "at_least_one_rate", "prefetch_hits",
                                                 "prefetch_misses")},
                "parity": par,
                "h2d_gb_per_request": round(h2d / 1e9, 3),
                "peak_device_gb": round(torch.cuda.max_memory_allocated(dev) / 1e9, 3),
                "kernels": [{k: r[k] for k in ("kernel", "launches", "avg_us", "achieved", "unit", "frac")}
                            for r in kern["all"]],
            })
            print(json.dumps(points[-1]), flush=True)
            eng.close()
            del eng
            torch.cuda.empty_cache()
    doc = {"metric": "BASELINE config 4 sweep: TTFT / decode tok/s / activated experts / predictor hit rate",
           "config": {"model": shape.name, "batches": batches, "prompts": prompts, "decode_steps": D,
                      "policy": "duoserve", "predictor": args.predictor,
                      "slots": "2 * min(M, k * B) (B = 1: the SPEC's 2k)"},
           "points": points, "wall_s": round(time.time() - t0, 1),
           "note": "residency cap applies to the batch-1 metric config; activations and KV of large batches "
                   "exceed it by construction"}
    out = json.dumps(doc)
    print(out)
    if args.out:
        Path(args.out).write_text(out + "\n")


def main():
    args = parse()
    if args.sweep:
        run_sweep(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
