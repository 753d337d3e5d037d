"""Why is the first K4 of a decode layer slower in the serving loop than the
same call back to back?  Native (gated) CUDA-event spans of one 8x7B expert:

  gap_<g>ms      isolated call after the GPU sat idle for g ms
  fresh          on a slot the copy engine just filled (stream-ordered after it)
  fresh_overlap  same, while the copy engine streams the next expert
  other_overlap  on a slot not just written, while the copy engine streams

    python scripts/k4_gap.py [--out gpurun_out/k4_gap.json]
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2509_07379_b200 import _lib, ops  # noqa: E402
from paper_2509_07379_b200.config import load_shape  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/k4_gap.json")
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
host = torch.empty((2, blob), dtype=torch.uint8).pin_memory()
host.copy_(blobs[:2].cpu())
es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)
cs = torch.cuda.Stream()


def ev(t=True):
    return torch.cuda.Event(enable_timing=t)


def k4(i, e):
    ops.expert_gemv(x, es[i], d, ff, G, h, rw, 1, acc, *e)


for i in range(20):
    k4(i % NB, (None, None))
torch.cuda.synchronize()
out = {}
N = 25
for g in (0.0, 0.2, 1.0, 2.0, 5.0):
    ts = []
    for i in range(N):
        torch.cuda.synchronize()
        if g:
            time.sleep(g / 1e3)
        e = (ev(), ev())
        k4(i % NB, e)
        e[1].synchronize()
        ts.append(e[0].elapsed_time(e[1]) * 1e3)
    out[f"gap_{g}ms"] = round(statistics.median(ts), 2)


def copy_then(target_fresh: bool, overlap: bool, delay_us: float = 0.0, chunks: int = 1):
    ts = []
    for i in range(N):
        torch.cuda.synchronize()
        ready = ev(False)
        with torch.cuda.stream(cs):
            blobs[0].copy_(host[0], non_blocking=True)
            ready.record(cs)
            if overlap:
                step = blob // chunks
                for c in range(chunks):
                    hi = blob if c == chunks - 1 else (c + 1) * step
                    blobs[1][c * step:hi].copy_(host[1][c * step:hi], non_blocking=True)
        torch.cuda.current_stream().wait_event(ready)
        if delay_us:
            torch.cuda._sleep(int(delay_us * 1965))
        e = (ev(), ev())
        k4(0 if target_fresh else 2, e)
        torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]) * 1e3)
    return round(statistics.median(ts), 2)


out["fresh"] = copy_then(True, False)
out["fresh_overlap"] = copy_then(True, True)
out["other_overlap"] = copy_then(False, True)
out["other_after_copy"] = copy_then(False, False)
for dl in (5, 20, 50, 100, 300, 800):
    out[f"fresh_overlap_delay{dl}us"] = copy_then(True, True, delay_us=dl)
for ch in (4, 16, 64):
    out[f"fresh_overlap_{ch}chunks"] = copy_then(True, True, chunks=ch)
print(json.dumps(out))
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(out, indent=1) + "\n")
