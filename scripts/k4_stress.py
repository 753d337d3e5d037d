"""Stress the K4 expert GEMV (ds_w4_expert_gemv): N back-to-back calls on one
stream, then on two streams at once, with a sync every 1000 calls; prints the
count done.  Run under `timeout` (a hang shows as a missing 'done' line).

    python scripts/k4_stress.py [--shape mixtral-8x22b] [--n 200000]
"""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2509_07379_b200 import ops
from paper_2509_07379_b200.config import load_shape

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="mixtral-8x22b")
ap.add_argument("--n", type=int, default=200000)
a = ap.parse_args()
dev = torch.device("cuda")
sh = load_shape(a.shape)
d, ff, G = sh.hidden, sh.ffn, sh.group_size
offs, total = ops.expert_layout(d, ff, G)
NB = 2
blobs = torch.empty((NB, total), dtype=torch.uint8, device=dev)
for i in range(NB):
    ops.w4_generate(1, 0, i, d, ff, G, blobs[i])
es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
hs = [torch.empty(1, ff, dtype=torch.bfloat16, device=dev) for _ in range(2)]
accs = [torch.zeros(1, d, device=dev) for _ in range(2)]
rw = torch.ones(1, device=dev)
t0 = time.time()
for i in range(a.n):
    ops.expert_gemv(x, es[i % NB], d, ff, G, hs[0], rw, 1, accs[0])
    if i % 1000 == 999:
        torch.cuda.synchronize()
print(f"one stream: {a.n} calls in {time.time() - t0:.1f} s", flush=True)
ss = [torch.cuda.Stream(), torch.cuda.Stream()]
t0 = time.time()
for i in range(a.n // 2):
    for j in range(2):
        with torch.cuda.stream(ss[j]):
            ops.expert_gemv(x, es[(i + j) % NB], d, ff, G, hs[j], rw, 1, accs[j])
    if i % 500 == 499:
        torch.cuda.synchronize()
torch.cuda.synchronize()
print(f"two streams: {a.n} calls in {time.time() - t0:.1f} s", flush=True)
print("done", flush=True)
