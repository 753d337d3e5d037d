"""Where does the in-loop K4 span go?  Runs the bench's engine (Mixtral-8x7B
W4, duoserve) for prefill P + decode D with the native spans on and splits
the K4 spans of the decode layers by (position in the layer's compute order,
prefetch hit / re-fetch), and times the same C call standalone with its
stream idle vs busy when the start event is recorded.

    python scripts/k4_inloop.py [--prefill 128] [--decode 16] [--out gpurun_out/k4_inloop.json]
"""
import argparse, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2509_07379_b200 import ops
from paper_2509_07379_b200.config import load_shape
from paper_2509_07379_b200.engine import Engine

ap = argparse.ArgumentParser()
ap.add_argument("--prefill", type=int, default=128)
ap.add_argument("--decode", type=int, default=16)
ap.add_argument("--out", default="gpurun_out/k4_inloop.json")
ap.add_argument("--policy", default="duoserve")
ap.add_argument("--k5-serial", action="store_true", help="run K5 on the compute stream (no overlap with K4)")
a = ap.parse_args()
dev = torch.device("cuda")
shape = load_shape("mixtral-8x7b")
net, pop, aff = bench.predictor_inputs(shape)
eng = Engine(shape, a.policy, seed=0, device=dev, predictor=net, pop=pop, aff=aff,
             max_seq=a.prefill + a.decode + 8, max_prefill=a.prefill)
prof = eng.enable_profile()
if a.k5_serial and eng.driver is not None:
    eng.driver.stream = torch.cuda.current_stream()
ids = torch.randint(0, shape.vocab, (a.prefill,), generator=torch.Generator().manual_seed(1)).to(dev)
res = {}
for it in range(2):
    eng.reset()
    prof.reset()
    eng.prefill(ids)
    for _ in range(a.decode):
        eng.decode_step()
    torch.cuda.synchronize()
spans = prof.spans["K4 w4_swiglu_gemv+down_gemv"]
us = [s[0].elapsed_time(s[1]) * 1e3 for s in spans]
labels = []
for r in eng.log:
    if r["phase"] != "decode":
        continue
    E = r.get("gate") or r.get("fetch")
    miss = set(r.get("refetch", []))
    order = [e for e in E if e not in miss] + sorted(miss)
    for j, e in enumerate(order):
        labels.append((j, e in miss, r["layer"]))
assert len(labels) == len(us), (len(labels), len(us))
groups = {}
for (j, m, l), t in zip(labels, us):
    for key in (f"pos{j}", f"pos{j}_{'miss' if m else 'hit'}", "layer0" if l == 0 else "layer>0", "all"):
        groups.setdefault(key, []).append(t)
res["inloop"] = {k: {"n": len(v), "mean_us": float(np.mean(v)), "median_us": float(np.median(v)),
                     "p10_us": float(np.percentile(v, 10)), "p90_us": float(np.percentile(v, 90))}
                 for k, v in sorted(groups.items())}

# the same C call standalone, natively recorded events, stream idle vs busy at the start event
d, ff, G = shape.hidden, shape.ffn, shape.group_size
offs, total = ops.expert_layout(d, ff, G)
NB = 4
blobs = torch.empty((NB, total), dtype=torch.uint8, device=dev)
for i in range(NB):
    ops.w4_generate(1, 0, i, d, ff, G, blobs[i])
es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)


host_src = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
dma_dst = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
copy_stream = torch.cuda.Stream()


def run(mode, iters=30):
    ts = []
    for i in range(iters + 3):
        torch.cuda.synchronize()
        time.sleep(0.002)
        if mode == "dma":                        # a host->HBM copy in flight on the copy engine (~4.6 ms)
            with torch.cuda.stream(copy_stream):
                dma_dst.copy_(host_src, non_blocking=True)
            time.sleep(0.0005)
        if mode == "busy":
            torch.cuda._sleep(200000)            # ~100 us on the same stream: start event queued behind it
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ops.expert_gemv(x, es[i % NB], d, ff, G, h, rw, 1, acc, e0, e1)
        e1.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return {"median_us": float(np.median(ts)), "mean_us": float(np.mean(ts))}


res["standalone_idle_stream"] = run("idle")
res["standalone_busy_stream"] = run("busy")
res["standalone_during_h2d_copy"] = run("dma")
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(res, indent=1))
print(json.dumps(res, indent=1))
