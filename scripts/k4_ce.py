"""Discriminate what makes K4 slow next to a copy-engine H2D copy (see
scripts/k4_gap.py): back-to-back vs single calls, a cross-stream event wait
vs none, copy destination adjacent to the K4 weights vs a separate buffer.

    python scripts/k4_ce.py [--out gpurun_out/k4_ce.json]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2509_07379_b200 import _lib, ops  # noqa: E402
from paper_2509_07379_b200.config import load_shape  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/k4_ce.json")
a = ap.parse_args()
_lib.load()
dev = torch.device("cuda")
sh = load_shape("mixtral-8x7b")
d, ff, G = sh.hidden, sh.ffn, sh.group_size
_, blob = ops.expert_layout(d, ff, G)
NB = 4
blobs = torch.empty((NB, blob), dtype=torch.uint8, device=dev)
for i in range(NB):
    ops.w4_generate(1, 0, i, d, ff, G, blobs[i])
es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
BIG = 256 << 20
src = torch.empty(BIG, dtype=torch.uint8).pin_memory()
src[::4096] = 1
sep = torch.empty(BIG, dtype=torch.uint8, device=dev)
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)
cs = torch.cuda.Stream()


def ev(t=True):
    return torch.cuda.Event(enable_timing=t)


def k4(i, e=(None, None)):
    ops.expert_gemv(x, es[i % NB], d, ff, G, h, rw, 1, acc, *e)


def copy(dst_kind, n=blob):
    with torch.cuda.stream(cs):
        if dst_kind == "sep":
            sep[:n].copy_(src[:n], non_blocking=True)
        else:
            blobs[1].copy_(src[:blob], non_blocking=True)


for i in range(20):
    k4(i)
torch.cuda.synchronize()
out = {}


def run(name, dst_kind, n_k4, wait_event, sleep_us=50, reps=15):
    ts = []
    for r in range(reps):
        torch.cuda.synchronize()
        pre = ev(False)
        pre.record(cs)
        copy(dst_kind, BIG if dst_kind == "sep" else blob)
        if wait_event:
            torch.cuda.current_stream().wait_event(pre)
        torch.cuda._sleep(int(sleep_us * 1965))
        spans = []
        for i in range(n_k4):
            e = (ev(), ev())
            k4(i if n_k4 > 1 else 2, e)
            spans.append(e)
        torch.cuda.synchronize()
        ts += [s.elapsed_time(t) * 1e3 for s, t in spans]
    out[name] = round(statistics.median(ts), 2)


run("alone_b2b", None, 30, False) if False else None
ts = []
for r in range(5):
    spans = []
    for i in range(30):
        e = (ev(), ev())
        k4(i, e)
        spans.append(e)
    torch.cuda.synchronize()
    ts += [s.elapsed_time(t) * 1e3 for s, t in spans]
out["alone_b2b"] = round(statistics.median(ts), 2)
run("sep_b2b_nowait", "sep", 30, False)
run("sep_single_nowait", "sep", 1, False)
run("sep_single_wait", "sep", 1, True)
run("sep_b2b_wait", "sep", 30, True)
run("adj_single_nowait", "adj", 1, False)
run("adj_b2b_nowait", "adj", 20, False)
print(json.dumps(out))
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(out, indent=1) + "\n")
