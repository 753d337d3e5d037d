import ctypes as Cc, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2509_07379_b200 import _lib, ops
cuda = torch.device('cuda')
G = 128
for (d, ff) in [(256, 896), (1024, 1024), (4096, 14336)]:
    offs, total = ops.expert_layout(d, ff, G)
    blob = torch.zeros(total, dtype=torch.uint8, device=cuda)
    ops.w4_generate(77, 2, 3, d, ff, G, blob)
    e = ops.expert_struct(blob.data_ptr(), d, ff, G)
    W = []
    for K, N, lin in [(d, ff, e.w1), (d, ff, e.w3), (ff, d, e.w2)]:
        out = torch.empty((N, K), dtype=torch.bfloat16, device=cuda)
        _lib.call("ds_w4_dequant", Cc.byref(lin), K, N, G, _lib.ptr(out), _lib.stream_ptr())
        W.append(out.double())
    for trial in range(3):
        if trial == 0:
            h = (torch.randn((1, ff), generator=torch.Generator().manual_seed(5)) * 0.3).to(torch.bfloat16).to(cuda)
        elif trial == 1:
            h = torch.ones((1, ff), dtype=torch.bfloat16, device=cuda)
        else:
            h = torch.zeros((1, ff), dtype=torch.bfloat16, device=cuda); h[0, 0] = 1.0
        acc = torch.zeros((1, d), dtype=torch.float32, device=cuda)
        rw = torch.ones(1, device=cuda)
        ops.down_gemv(h, e, d, ff, G, rw, 1, acc)
        torch.cuda.synchronize()
        ref = h.double() @ W[2].T
        err = (acc.double() - ref)
        print(d, ff, trial, "rel", (err.norm() / ref.norm()).item(), "maxabs", err.abs().max().item(),
              "argmax", err.abs().argmax().item(), "ref@", ref.flatten()[err.abs().argmax()].item())
