"""K4 expert-GEMV spans (native CUDA events) queued back to back vs launched
on an idle stream: how much host submission latency an event span picks up
when the stream is idle, with and without the launch gate (DS_LAUNCH_GATE).

    python scripts/k4_idle.py            # gate on (default)
    DS_LAUNCH_GATE=0 python scripts/k4_idle.py
"""
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2509_07379_b200 import _lib, ops  # noqa: E402
from paper_2509_07379_b200.config import load_shape  # noqa: E402

_lib.load()
dev = torch.device("cuda")
sh = load_shape(sys.argv[1] if len(sys.argv) > 1 else "mixtral-8x7b")
d, ff, G = sh.hidden, sh.ffn, sh.group_size
_, blob = ops.expert_layout(d, ff, G)
NB = 4
blobs = torch.empty((NB, blob), dtype=torch.uint8, device=dev)
for i in range(NB):
    ops.w4_generate(1, 0, i, d, ff, G, blobs[i])
es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)


def ev():
    return torch.cuda.Event(enable_timing=True)


def call(i, evs):
    ops.expert_gemv(x, es[i % NB], d, ff, G, h, rw, 1, acc, *evs)


for i in range(10):
    call(i, (None, None))
torch.cuda.synchronize()
out = {"gate": os.environ.get("DS_LAUNCH_GATE", "1")}
spans = []
for i in range(40):
    e = (ev(), ev())
    call(i, e)
    spans.append(e)
torch.cuda.synchronize()
out["queued_us"] = round(statistics.median(a.elapsed_time(b) * 1e3 for a, b in spans[5:]), 2)
spans = []
for i in range(40):
    torch.cuda.synchronize()
    e = (ev(), ev())
    call(i, e)
    spans.append(e)
torch.cuda.synchronize()
out["idle_us"] = round(statistics.median(a.elapsed_time(b) * 1e3 for a, b in spans[5:]), 2)
# wall time of idle launches (host call -> sync), for reference
import time
ws = []
for i in range(40):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    call(i, (None, None))
    torch.cuda.synchronize()
    ws.append(time.perf_counter() - t0)
out["idle_wall_us"] = round(1e6 * statistics.median(ws[5:]), 2)
print(json.dumps(out))
