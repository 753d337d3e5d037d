"""Is the in-loop K4 slowdown inside the kernel or around it?

K4 v6 launches with per-CTA %globaltimer stamps (DS_K4_V6_TIMELINE=1), once
on an idle GPU and once while the copy engine streams a 4-expert H2D chain
(the decode link's traffic).  Per launch: the CUDA-event span on the launching
stream and the kernel-internal time (first CTA entry -> last CTA exit).  If the
kernel-internal time stays at its idle value while the event span grows, the
extra time is front-end/launch latency (command fetch over a saturated host
link), not HBM interference.

    python scripts/k4_ce_timeline.py [--out gpurun_out/k4_ce_timeline.json]
"""
import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

os.environ["DS_K4_V6_TIMELINE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_07379_b200 import _lib, ops  # noqa: E402
from paper_2509_07379_b200.config import load_shape  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/k4_ce_timeline.json")
a = ap.parse_args()
_lib.load()
dev = torch.device("cuda")
sh = load_shape("mixtral-8x7b")
d, ff, G = sh.hidden, sh.ffn, sh.group_size
_, blob = ops.expert_layout(d, ff, G)
slots = torch.empty((4, blob), dtype=torch.uint8, device=dev)
for i in range(4):
    ops.w4_generate(1, 0, i, d, ff, G, slots[i])
store = torch.empty((4, blob), dtype=torch.uint8).pin_memory()
for i in range(4):
    store[i].copy_(slots[i])
es = [ops.expert_struct(slots[i].data_ptr(), d, ff, G) for i in range(4)]
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)
cs = torch.cuda.Stream()
n = torch.cuda.get_device_properties(0).multi_processor_count
spin = torch.empty(1 << 26, dtype=torch.float32, device=dev)


def ev():
    return torch.cuda.Event(enable_timing=True)


def one(copy: bool):
    torch.cuda.synchronize()
    if copy:
        with torch.cuda.stream(cs):
            for j in range(3):
                slots[1 + j].copy_(store[1 + j], non_blocking=True)
        # let the copy reach steady state before K4 starts
        for _ in range(4):
            spin.mul_(1.0)
    e0, e1 = ev(), ev()
    e0.record()
    ops.expert_gemv(x, es[0], d, ff, G, h, rw, 1, acc)
    e1.record()
    e1.synchronize()
    buf = (C.c_ulonglong * (n * 8))()
    _lib.call("ds_debug_k4v6_timeline", buf, n)
    st = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8).astype(np.int64)
    t0 = st[:, 0].min()
    ent = (st[:, 0] - t0) / 1e3
    ex = (st[:, 4] - t0) / 1e3
    pa = (st[:, 1] - t0) / 1e3
    torch.cuda.synchronize()
    return {"event_us": round(e0.elapsed_time(e1) * 1e3, 2), "kernel_us": round(float(ex.max()), 2),
            "entry_spread_us": round(float(ent.max()), 2), "phaseA_median_us": round(float(np.median(pa)), 2),
            "exit_median_us": round(float(np.median(ex)), 2)}


def graph_idle():
    """The graph launch with no copy running (its span's own overhead)."""
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    ops.expert_gemv_graph(x, es[0], d, ff, G, h, rw, 1, acc, None, e0, e1)
    e1.synchronize()
    return {"event_us": round(e0.elapsed_time(e1) * 1e3, 2)}


def gated(graph: bool):
    """The decode pattern: K4 on slot 0 queued behind the copy of its expert
    (ready event), the copy engine busy with the next experts afterwards.
    Returns copy-done -> span start, the span, and the kernel-internal time."""
    torch.cuda.synchronize()
    ready, c0 = ev(), ev()
    with torch.cuda.stream(cs):
        c0.record(cs)
        slots[0].copy_(store[0], non_blocking=True)
        ready.record(cs)
        for j in range(2):
            slots[1 + j].copy_(store[1 + j], non_blocking=True)
    e0, e1 = ev(), ev()
    if graph:
        ops.expert_gemv_graph(x, es[0], d, ff, G, h, rw, 1, acc, ready, e0, e1)
    else:
        torch.cuda.current_stream().wait_event(ready)
        ops.expert_gemv(x, es[0], d, ff, G, h, rw, 1, acc, e0, e1)
    e1.synchronize()
    buf = (C.c_ulonglong * (n * 8))()
    _lib.call("ds_debug_k4v6_timeline", buf, n)
    st = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8).astype(np.int64)
    torch.cuda.synchronize()
    return {"ready_to_start_us": round(ready.elapsed_time(e0) * 1e3, 2),
            "event_us": round(e0.elapsed_time(e1) * 1e3, 2),
            "ready_to_end_us": round(ready.elapsed_time(e1) * 1e3, 2),
            "kernel_us": round(float((st[:, 4].max() - st[:, 0].min()) / 1e3), 2)}


for _ in range(5):
    one(False)
out = {"idle": [one(False) for _ in range(6)], "beside_copy": [one(True) for _ in range(6)]}
out["graph_idle"] = [graph_idle() for _ in range(6)]
for mode in ("eager", "graph"):
    for _ in range(2):
        gated(mode == "graph")
    out[f"gated_{mode}"] = [gated(mode == "graph") for _ in range(6)]
for k, v in out.items():
    print(k, json.dumps(v[-3:]), flush=True)
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(out, indent=1) + "\n")
