"""Does an SM pass over the pinned source (ds_h2d_sm_copy into a scratch
buffer) before the copy-engine H2D change how much that copy slows K4?
Also: repeated CE copies of the same source (second pass warm).

    python scripts/k4_touch.py
"""
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2509_07379_b200 import _lib, ops  # noqa: E402
from paper_2509_07379_b200.config import load_shape  # noqa: E402

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
srcs = [torch.empty(BIG, dtype=torch.uint8).pin_memory() for _ in range(3)]
for s_ in srcs:
    s_[::4096] = 1
dst = torch.empty(BIG, dtype=torch.uint8, device=dev)
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)
cs = torch.cuda.Stream()


def ev(t=True):
    return torch.cuda.Event(enable_timing=t)


def k4(i, e=(None, None)):
    ops.expert_gemv(x, es[i % NB], d, ff, G, h, rw, 1, acc, *e)


def touch(src):
    _lib.call("ds_h2d_sm_copy", C.c_void_p(dst.data_ptr()), C.c_void_p(src.data_ptr()), BIG, 32,
              C.c_void_p(cs.cuda_stream))
    cs.synchronize()


def under_ce(src, n_k4=20, reps=5):
    ts = []
    for r in range(reps):
        torch.cuda.synchronize()
        with torch.cuda.stream(cs):
            dst.copy_(src, non_blocking=True)
        torch.cuda._sleep(int(100 * 1965))
        spans = []
        for i in range(n_k4):
            e = (ev(), ev())
            k4(i, e)
            spans.append(e)
        torch.cuda.synchronize()
        ts += [s.elapsed_time(t) * 1e3 for s, t in spans]
    return round(statistics.median(ts), 2)


for i in range(20):
    k4(i)
torch.cuda.synchronize()
out = {"cold_src0_first": under_ce(srcs[0], reps=1), "src0_repeat": under_ce(srcs[0])}
touch(srcs[1])
out["touched_src1"] = under_ce(srcs[1])
out["untouched_src2"] = under_ce(srcs[2])
touch(srcs[2])
out["src2_after_touch"] = under_ce(srcs[2])
print(json.dumps(out))
