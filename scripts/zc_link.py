"""SM-driven host->HBM copy (ds_h2d_sm_copy) vs the copy engine: link
bandwidth, and what each costs the K4 expert GEMV running beside it.

    python scripts/zc_link.py [--out gpurun_out/zc_link.json]
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
ap.add_argument("--out", default="gpurun_out/zc_link.json")
ap.add_argument("--shape", default="mixtral-8x7b")
a = ap.parse_args()
_lib.load()
dev = torch.device("cuda")
sh = load_shape(a.shape)
d, ff, G = sh.hidden, sh.ffn, sh.group_size
offs, blob = ops.expert_layout(d, ff, G)
NB = 4
blobs = torch.empty((NB, blob), dtype=torch.uint8, device=dev)
for i in range(NB):
    ops.w4_generate(1, 0, i, d, ff, G, blobs[i])
es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)
BIG = 256 << 20
src = torch.empty(BIG, dtype=torch.uint8).pin_memory()
src[::4096] = 1
dst = torch.empty(BIG, dtype=torch.uint8, device=dev)
cs = torch.cuda.Stream()
out = {"shape": a.shape, "expert_bytes": blob}


def ev():
    return torch.cuda.Event(enable_timing=True)


def sm_copy(nbytes, ctas, stream):
    _lib.call("ds_h2d_sm_copy", C.c_void_p(dst.data_ptr()), C.c_void_p(src.data_ptr()), nbytes, ctas,
              C.c_void_p(stream.cuda_stream))


def ce_copy(nbytes, stream):
    with torch.cuda.stream(stream):
        dst[:nbytes].copy_(src[:nbytes], non_blocking=True)


def link_gbs(fn, nbytes, iters=5):
    ts = []
    for _ in range(iters + 1):
        e0, e1 = ev(), ev()
        e0.record(cs)
        fn(nbytes)
        e1.record(cs)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(nbytes / (statistics.median(ts[1:]) / 1e3) / 1e9, 2)


out["ce_gbs_expert"] = link_gbs(lambda n: ce_copy(n, cs), blob)
out["ce_gbs_256mb"] = link_gbs(lambda n: ce_copy(n, cs), BIG)
# correctness of the SM copy
dst.zero_()
sm_copy(blob - blob % 16, 32, cs)
cs.synchronize()
out["sm_copy_exact"] = bool(torch.equal(dst[:blob - blob % 16].cpu(), src[:blob - blob % 16]))
out["sm_gbs_expert"] = {}
for ctas in (2, 4, 8, 16, 32, 64, 148):
    out["sm_gbs_expert"][ctas] = link_gbs(lambda n: sm_copy(n - n % 16, ctas, cs), blob)
print(json.dumps(out), flush=True)


def k4(i):
    ops.expert_gemv(x, es[i % NB], d, ff, G, h, rw, 1, acc)


def k4_times(bg=None, iters=30):
    """Median K4 expert time on the current stream, with `bg` (a copy) launched first on cs."""
    torch.cuda.synchronize()
    if bg is not None:
        bg()
        # give the copy a head start so every K4 overlaps it
        torch.cuda._sleep(20000)
    ts = []
    for i in range(iters):
        e0, e1 = ev(), ev()
        e0.record()
        k4(i)
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    return round(statistics.median(a.elapsed_time(b) * 1e3 for a, b in ts), 2)


for i in range(10):
    k4(i)
torch.cuda.synchronize()
res = {"alone": k4_times(None)}
res["ce_256mb"] = k4_times(lambda: ce_copy(BIG, cs))
for ctas in (4, 8, 16, 32):
    res[f"sm{ctas}_256mb"] = k4_times(lambda: sm_copy(BIG, ctas, cs))
out["k4_us"] = res


# link bandwidth while K4 runs back to back on the compute stream
def link_under_k4(fn, nbytes):
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record(cs)
    fn(nbytes)
    e1.record(cs)
    n = 0
    while not e1.query() and n < 2000:
        k4(n)
        n += 1
        if n % 50 == 0:
            torch.cuda.current_stream().synchronize()
    torch.cuda.synchronize()
    return round(nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9, 2), n


out["link_under_k4"] = {"ce": link_under_k4(lambda n: ce_copy(n, cs), BIG)}
for ctas in (8, 16, 32):
    out["link_under_k4"][f"sm{ctas}"] = link_under_k4(lambda n: sm_copy(n, ctas, cs), BIG)
print(json.dumps(out), flush=True)
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(out, indent=1) + "\n")
