"""Where the decode reaction window goes (Mixtral-8x7B, batch 1).

After layer l's last expert lands, the link has nothing certain to move until
layer l+1's gate result reaches the host and its misses are submitted; this
window is spent on speculative chunks that are mostly wrong with a
random-init model.  Measures its parts:
  * the per-layer decode front (attention + norm + K1 gate, one CUDA graph)
    and the combine, idle GPU, CUDA events;
  * K1 alone (T = 1);
  * host time from the gate result to the layer's transfers submitted
    (Engine.host_wait["decide"]) over a few served tokens.

    python scripts/decode_window.py [--out gpurun_out/decode_window.json]
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_07379_b200 import ops  # noqa: E402
from paper_2509_07379_b200.config import load_shape  # noqa: E402
from paper_2509_07379_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/decode_window.json")
ap.add_argument("--tokens", type=int, default=8)
a = ap.parse_args()
shape = load_shape("mixtral-8x7b")
net, pop, aff = bench.predictor_inputs(shape)
eng = Engine(shape, "duoserve", seed=0, predictor=net, pop=pop, aff=aff, max_seq=600, max_prefill=512)
ids = torch.randint(0, shape.vocab, (512,), generator=torch.Generator().manual_seed(1))
eng.prefill(ids)
for _ in range(2):
    eng.decode_step()
for k_ in eng.host_wait:
    eng.host_wait[k_] = 0.0
t0 = time.perf_counter()
for _ in range(a.tokens):
    eng.decode_step()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / a.tokens
L = shape.num_layers
res = {"tokens": a.tokens, "ms_per_token": round(1e3 * wall, 2),
       "host_per_layer_us": {k_: round(1e6 * v / (a.tokens * L), 1) for k_, v in eng.host_wait.items()}}


def timed(fn, n=20):
    out = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3)
    return round(statistics.median(out), 2)


torch.cuda.synchronize()
res["front_graph_us"] = timed(lambda: eng.g_graphs[5].replay())
res["gate_k1_us"] = timed(lambda: ops.gate_topk(eng.g_a2, eng.W.layers[5]["wg"], eng.k, eng.idx1, eng.w1))
res["combine_us"] = timed(lambda: ops.combine_finalize(eng.acc, eng.g_h1, eng.g_h))
res["empty_event_pair_us"] = timed(lambda: None)
print(json.dumps(res, indent=1))
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(res, indent=1) + "\n")
