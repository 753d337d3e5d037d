"""Per-CTA timeline of K3 (DS_K3_TIMELINE=1): GEMM1 and GEMM2 stamps (entry,
scales staged, first MMA issued, last MMA issued, accumulators ready, exit),
us from GEMM1's earliest entry; min / median / max over CTAs.

    python scripts/k3_timeline.py [rows]
"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

os.environ["DS_K3_TIMELINE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_07379_b200 import _lib, ops  # noqa: E402
from paper_2509_07379_b200.config import load_shape  # noqa: E402

_lib.load()
dev = torch.device("cuda")
sh = load_shape("mixtral-8x7b")
d, ff, G = sh.hidden, sh.ffn, sh.group_size
R = int(sys.argv[1]) if len(sys.argv) > 1 else 151
_, blob = ops.expert_layout(d, ff, G)
b = torch.empty(blob, dtype=torch.uint8, device=dev)
ops.w4_generate(1, 0, 0, d, ff, G, b)
e = ops.expert_struct(b.data_ptr(), d, ff, G)
x = torch.randn(R, d, device=dev).to(torch.bfloat16)
h = torch.empty(R, ff, dtype=torch.bfloat16, device=dev)
y = torch.empty(R, d, device=dev)
ws = torch.empty(max(ops.grouped_ffn_workspace(R, d, ff), 16), dtype=torch.uint8, device=dev)
names = ["entry", "scales_staged", "first_mma", "last_mma", "acc_ready", "exit"]
for it in range(4):
    ops.grouped_ffn(x, [0, R], [e], d, ff, G, h, y, ws)
    torch.cuda.synchronize()
out = {}
t0 = None
for nmat, n in ((2, 112), (1, 128)):
    buf = (C.c_ulonglong * (n * 8))()
    _lib.call("ds_debug_k3_timeline", buf, nmat, n)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8).astype(np.int64)
    valid = a[:, 0] > 0
    a = a[valid]
    if t0 is None:
        t0 = a[:, 0].min()
    row = {"ctas": int(valid.sum())}
    for i, nm in enumerate(names):
        v = (a[:, i] - t0) / 1e3
        v = v[a[:, i] > 0]
        if v.size:
            row[nm] = [round(float(v.min()), 2), round(float(np.median(v)), 2), round(float(v.max()), 2)]
    out["gemm1" if nmat == 2 else "gemm2"] = row
print(json.dumps(out, indent=1))
