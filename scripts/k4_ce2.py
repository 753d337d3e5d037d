"""K4 spans over time beside copy-engine H2D copies laid out like the
engine's (experts of a [L, M, blob] pinned store into a 4-slot HBM cache):
each K4 launch's start offset from the copy start and its duration, for a
1-expert copy and a 4-expert copy chain, to see whether the copy engine
slows K4 for the whole copy or only part of it.

    python scripts/k4_ce2.py [--out gpurun_out/k4_ce2.json]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2509_07379_b200 import _lib, ops  # noqa: E402
from paper_2509_07379_b200.config import load_shape  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/k4_ce2.json")
a = ap.parse_args()
_lib.load()
dev = torch.device("cuda")
sh = load_shape("mixtral-8x7b")
d, ff, G = sh.hidden, sh.ffn, sh.group_size
_, blob = ops.expert_layout(d, ff, G)
slots = torch.empty((4, blob), dtype=torch.uint8, device=dev)
for i in range(4):
    ops.w4_generate(1, 0, i, d, ff, G, slots[i])
store = torch.empty((8, blob), dtype=torch.uint8).pin_memory()
for i in range(8):
    store[i].copy_(slots[i % 4])
es = [ops.expert_struct(slots[i].data_ptr(), d, ff, G) for i in range(4)]
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)
cs = torch.cuda.Stream()


def ev():
    return torch.cuda.Event(enable_timing=True)


for i in range(10):
    ops.expert_gemv(x, es[0], d, ff, G, h, rw, 1, acc)
torch.cuda.synchronize()
out = {}
for n_exp, n_k4 in ((1, 40), (4, 120)):
    runs = []
    for trial in range(3):
        torch.cuda.synchronize()
        ref = ev()
        ref.record()
        c0, c1 = ev(), ev()
        with torch.cuda.stream(cs):
            c0.record(cs)
            for j in range(n_exp):
                slots[1 + (j % 3)].copy_(store[(trial + j) % 8], non_blocking=True)
            c1.record(cs)
        spans = []
        for i in range(n_k4):
            e = (ev(), ev())
            ops.expert_gemv(x, es[0], d, ff, G, h, rw, 1, acc, *e)
            spans.append(e)
        torch.cuda.synchronize()
        cst, cen = ref.elapsed_time(c0) * 1e3, ref.elapsed_time(c1) * 1e3
        rows = [(round(ref.elapsed_time(s) * 1e3 - cst, 1), round(s.elapsed_time(t) * 1e3, 1)) for s, t in spans]
        runs.append({"copy_us": round(cen - cst, 1), "k4": rows})
    out[f"copy_{n_exp}_experts"] = runs
    r = runs[-1]
    inside = [dur for st, dur in r["k4"] if 0 <= st < r["copy_us"]]
    after = [dur for st, dur in r["k4"] if st >= r["copy_us"]]
    print(n_exp, "copy us", r["copy_us"], "K4 inside: n", len(inside), "mean", round(sum(inside) / max(len(inside), 1), 1),
          "after: n", len(after), "mean", round(sum(after) / max(len(after), 1), 1), flush=True)
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(out) + "\n")
