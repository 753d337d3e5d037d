"""W4 linears (the resident attention projections): generator bytes equal
oracle/w4_ref, and y = x W^T through the C-ABI (K4 GEMV for <= 16 rows with
the exact (q - z) s products; the tcgen05 GEMM above with bf16-rounded
weights) within f32-accumulation tolerance of an f64 reference on the same
weights, at the tiny, 8x7B and 8x22B projection shapes."""

import numpy as np
import pytest
import torch

from oracle import w4_ref
from paper_2509_07379_b200 import ops
from tests import w4_torch

pytestmark = pytest.mark.gpu

REL_TOL = 2e-5


def _weights(lin, exact):
    offs, _ = ops.linear_layout(lin.K, lin.N, lin.G)
    K, N, G = lin.K, lin.N, lin.G
    b = lin.blob
    c = b[offs[0]:offs[0] + N * K // 2].view(torch.int32).view(N, K // 8)
    s = b[offs[1]:offs[1] + N * (K // G) * 2].view(torch.bfloat16).view(N, K // G)
    z = b[offs[2]:offs[2] + (N * (K // G) + 1) // 2]
    return w4_torch.linear_weights(K, N, c, s, z, G, exact)


@pytest.mark.parametrize("K,N", [(256, 512), (256, 256), (4096, 6144), (4096, 4096), (6144, 8192), (6144, 6144)])
def test_w4_linear_rows(K, N, cuda):
    lin = ops.W4Lin.generate(9, 2, 63, 0, K, N, 128, cuda)
    if K * N <= 256 * 512:
        c, s, z = w4_ref.gen_linear(9, 2, 63, 0, K, N, 128)
        offs, _ = ops.linear_layout(K, N, 128)
        b = lin.blob.cpu().numpy()
        assert np.array_equal(b[offs[0]:offs[0] + c.nbytes].view(np.uint32).reshape(c.shape), c)
        assert np.array_equal(b[offs[1]:offs[1] + s.nbytes].view(np.uint16).reshape(s.shape), s)
        assert np.array_equal(b[offs[2]:offs[2] + z.nbytes], z)
    Wx, Wr = _weights(lin, True), _weights(lin, False)
    g = torch.Generator(device=cuda).manual_seed(K + N)
    for R in (1, 3, 16, 17, 64, 512):
        x = torch.randn((R, K), generator=g, device=cuda).to(torch.bfloat16)
        y = torch.empty((R, N), dtype=torch.float32, device=cuda)
        nb = ops.linear_workspace(R, K, N)
        ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=cuda)
        ops.w4_linear(x, lin, y, ws)
        ref = x.double() @ (Wx if R <= ops.GEMV_MAX_ROWS else Wr).T
        rel = ((y.double() - ref).norm() / ref.norm()).item()
        assert rel <= REL_TOL, (K, N, R, rel)
