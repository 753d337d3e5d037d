"""Decode-link chunk-size sweep: tok/s and wasted bytes vs chunk size."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
from paper_2509_07379_b200.config import load_shape
from paper_2509_07379_b200.engine import Engine
shape = load_shape(sys.argv[1] if len(sys.argv) > 1 else "mixtral-8x7b")
net, pop, aff = bench.predictor_inputs(shape)
eng = Engine(shape, "duoserve", seed=0, predictor=net, pop=pop, aff=aff, max_seq=600, max_prefill=512)
ids = torch.randint(0, shape.vocab, (512,), generator=torch.Generator().manual_seed(1))
out = []
for depth, mb in [(2, 8), (2, 4), (2, 2), (3, 2), (2, 1), (4, 1)]:
    eng.link.depth = depth
    eng.link.set_chunk(int(mb * 2**20))
    eng.reset(); eng.prefill(ids)
    for _ in range(2): eng.decode_step()
    eng.link.reset_stats()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    n = 16
    for _ in range(n): eng.decode_step()
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    st = eng.link.stats()
    out.append({"depth": depth, "chunk_mb": mb, "tok_s": round(n / dt, 3), "ms_per_tok": round(1e3 * dt / n, 2),
                "wasted_MB_per_tok": round(st["wasted_prefetch_bytes"] / n / 2**20, 1),
                "issued_GB_per_tok": round(st["bytes_issued"] / n / 1e9, 3),
                "link_GBs": round(st["bytes_issued"] / dt / 1e9, 2)})
    print(out[-1], flush=True)
