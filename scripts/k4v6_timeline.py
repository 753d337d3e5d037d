"""Per-CTA timeline of the fused K4 v6 launch (DS_K4_V6_TIMELINE=1 must be
set): entry, phase A consumed, barrier passed, h staged, exit (us from the
earliest entry; min / median / max over CTAs)."""
import ctypes as C
import json
import os
import sys
from pathlib import Path

os.environ["DS_K4_V6_TIMELINE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_07379_b200 import _lib, ops  # noqa: E402
from paper_2509_07379_b200.config import load_shape  # noqa: E402

_lib.load()
dev = torch.device("cuda")
sh = load_shape(sys.argv[1] if len(sys.argv) > 1 else "mixtral-8x7b")
d, ff, G = sh.hidden, sh.ffn, sh.group_size
_, blob = ops.expert_layout(d, ff, G)
NB = 4
blobs = torch.empty((NB, blob), dtype=torch.uint8, device=dev)
for i in range(NB):
    ops.w4_generate(1, 0, i, d, ff, G, blobs[i])
es = [ops.expert_struct(blobs[i].data_ptr(), d, ff, G) for i in range(NB)]
x = torch.randn(1, d, device=dev).to(torch.bfloat16)
h = torch.empty(1, ff, dtype=torch.bfloat16, device=dev)
acc = torch.zeros(1, d, device=dev)
rw = torch.ones(1, device=dev)
n = torch.cuda.get_device_properties(0).multi_processor_count
names = ["entry", "phaseA_done", "barrier_passed", "h_staged", "exit"]
runs = []
for it in range(8):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    ops.expert_gemv(x, es[it % NB], d, ff, G, h, rw, 1, acc)
    ev1.record()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (n * 8))()
    _lib.call("ds_debug_k4v6_timeline", buf, n)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8).astype(np.int64)
    t0 = a[:, 0].min()
    row = {"event_us": round(ev0.elapsed_time(ev1) * 1e3, 2)}
    for i, nm in enumerate(names):
        v = (a[:, i] - t0) / 1e3
        v = v[a[:, i] > 0]
        if v.size:
            row[nm] = [round(float(v.min()), 2), round(float(np.median(v)), 2), round(float(v.max()), 2)]
    runs.append(row)
print(json.dumps(runs[3:], indent=1))
