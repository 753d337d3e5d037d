"""How much does a host->HBM copy on the copy engine slow an HBM-bound kernel?
Times (CUDA events, median of 30) the K4 expert GEMV and a plain elementwise
streaming kernel, each alone and while a pinned H2D copy is in flight, with
the copy's destination either one large buffer or a 1 MB ring.

    python scripts/dma_interference.py [--out gpurun_out/dma_interference.json]
"""
import argparse, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2509_07379_b200 import ops
from paper_2509_07379_b200.config import load_shape

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/dma_interference.json")
a = ap.parse_args()
dev = torch.device("cuda")
sh = load_shape("mixtral-8x7b")
d, ff, G = sh.hidden, sh.ffn, sh.group_size
offs, total = ops.expert_layout(d, ff, G)
NB = 4
blobs = torch.empty((NB, total), dtype=torch.uint8, device=dev)
for i in range(NB):
    ops.w4_generate(1, 0, i, d, ff, G, blobs[i])
es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)
src_big = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
dst_big = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
src_small = torch.empty(1 << 20, dtype=torch.uint8).pin_memory()
dst_small = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
ea = torch.empty(64 << 20, dtype=torch.float32, device=dev)     # 256 MB in, 256 MB out
eb = torch.empty_like(ea)
cs = torch.cuda.Stream()


def thp_pinned(nbytes):
    """Anonymous mapping advised for transparent huge pages, touched, then page-locked with cudaHostRegister."""
    import mmap
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    try:
        m.madvise(mmap.MADV_HUGEPAGE)
    except (AttributeError, OSError):
        pass
    arr = np.frombuffer(m, dtype=np.uint8)
    arr[::4096] = 1
    t = torch.from_numpy(arr)
    rc = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), nbytes, 0)
    assert int(rc) == 0, rc
    return t, m


src_thp, _keep = thp_pinned(256 << 20)
thp_info = Path("/sys/kernel/mm/transparent_hugepage/enabled").read_text().strip() \
    if Path("/sys/kernel/mm/transparent_hugepage/enabled").exists() else "n/a"


def dma(kind):
    with torch.cuda.stream(cs):
        if kind == "big":
            dst_big.copy_(src_big, non_blocking=True)          # ~4.6 ms
        elif kind == "ring":
            for _ in range(256):
                dst_small.copy_(src_small, non_blocking=True)
        elif kind == "src_big_dst_ring":
            for j in range(256):
                dst_small.copy_(src_big[j << 20:(j + 1) << 20], non_blocking=True)
        elif kind == "src_ring_dst_big":
            for j in range(256):
                dst_big[j << 20:(j + 1) << 20].copy_(src_small, non_blocking=True)
        elif kind == "thp_big":
            dst_big.copy_(src_thp, non_blocking=True)


def timed(fn, kind, iters=30, one_blob=False):
    ts = []
    for i in range(iters + 3):
        torch.cuda.synchronize()
        time.sleep(0.001)
        if kind:
            dma(kind)
            time.sleep(0.0005)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(0 if one_blob else i % NB)
        e1.record()
        e1.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return round(float(np.median(ts)), 2)


k4 = lambda i: ops.expert_gemv(x, es[i], d, ff, G, h, rw, 1, acc)
ew = lambda i: torch.add(ea, 1.0, out=eb)
res = {"thp": thp_info}
for kind in (None, "big", "ring", "src_big_dst_ring", "src_ring_dst_big", "thp_big"):
    tag = kind or "alone"
    res[f"k4_{tag}_us"] = timed(k4, kind)
    t = timed(ew, kind)
    res[f"elementwise_{tag}_us"] = t
    res[f"elementwise_{tag}_GBs"] = round(2 * ea.numel() * 4 / t / 1e3, 1)
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(res, indent=1))
print(json.dumps(res, indent=1))
