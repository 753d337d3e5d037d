"""TMA-driven host->HBM copy (ds_h2d_tma_copy) vs the copy engine: link GB/s
and the K4 expert GEMV span while each runs.

    python scripts/tma_link.py [--out gpurun_out/tma_link.json]
"""
import argparse
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2509_07379_b200 import _lib, ops  # noqa: E402
from paper_2509_07379_b200.config import load_shape  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/tma_link.json")
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
src = torch.randint(0, 255, (BIG,), dtype=torch.uint8).pin_memory()
dst = torch.empty(BIG, dtype=torch.uint8, device=dev)
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)
cs = torch.cuda.Stream()
out = {}


def ev(t=True):
    return torch.cuda.Event(enable_timing=t)


def tma(n, ctas):
    _lib.call("ds_h2d_tma_copy", C.c_void_p(dst.data_ptr()), C.c_void_p(src.data_ptr()), n, ctas,
              C.c_void_p(cs.cuda_stream))


def ce(n, ctas=0):
    with torch.cuda.stream(cs):
        dst[:n].copy_(src[:n], non_blocking=True)


def k4(i, e=(None, None)):
    ops.expert_gemv(x, es[i % NB], d, ff, G, h, rw, 1, acc, *e)


dst.zero_()
tma(blob - blob % 16, 2)
cs.synchronize()
n = blob - blob % 16
out["tma_exact"] = bool(torch.equal(dst[:n].cpu(), src[:n]))


def gbs(fn, n, ctas, iters=5):
    ts = []
    for _ in range(iters + 1):
        e0, e1 = ev(), ev()
        e0.record(cs)
        fn(n, ctas)
        e1.record(cs)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(n / (statistics.median(ts[1:]) / 1e3) / 1e9, 2)


out["ce_gbs"] = gbs(ce, BIG, 0)
out["tma_gbs"] = {c: gbs(tma, BIG, c) for c in (1, 2, 4, 8, 16)}
print(json.dumps(out), flush=True)
for i in range(20):
    k4(i)
torch.cuda.synchronize()


def k4_under(fn, ctas, n_k4, reps=10):
    ts = []
    for r in range(reps):
        torch.cuda.synchronize()
        fn(BIG, ctas)
        torch.cuda._sleep(int(100 * 1965))
        spans = []
        for i in range(n_k4):
            e = (ev(), ev())
            k4(i, e)
            spans.append(e)
        torch.cuda.synchronize()
        ts += [s.elapsed_time(t) * 1e3 for s, t in spans]
    return round(statistics.median(ts), 2)


res = {"alone": k4_under(lambda n, c: None, 0, 30)}
res["ce_b2b"] = k4_under(ce, 0, 30)
res["ce_single"] = k4_under(ce, 0, 1)
for c in (1, 2, 4, 8):
    res[f"tma{c}_b2b"] = k4_under(tma, c, 30)
    res[f"tma{c}_single"] = k4_under(tma, c, 1)
out["k4_us"] = res


def link_under_k4(fn, ctas):
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record(cs)
    fn(BIG, ctas)
    e1.record(cs)
    n = 0
    while not e1.query() and n < 3000:
        k4(n)
        n += 1
        if n % 50 == 0:
            torch.cuda.current_stream().synchronize()
    torch.cuda.synchronize()
    return round(BIG / (e0.elapsed_time(e1) / 1e3) / 1e9, 2), n


out["link_under_k4"] = {"ce": link_under_k4(ce, 0), **{f"tma{c}": link_under_k4(tma, c) for c in (1, 2, 4, 8)}}
print(json.dumps(out))
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(out, indent=1) + "\n")
