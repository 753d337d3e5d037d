"""The fused decode front (csrc/front.cu) against the torch ops it replaces
(model.attention_decode_static + rms_norm): same W4 projections, same
attention; only reduction orders differ, so h1 / a2 agree to a few bf16 ulps
and the KV-cache writes bit for bit (RoPE has no reduction)."""
import pytest

from paper_2509_07379_b200 import config as C
from paper_2509_07379_b200.model import (KVCache, attention_decode_static, decode_front_fused, init_dense_weights,
                                         rms_norm, rope_tables)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,pos", [("tiny-4x8", 0), ("tiny-4x8", 37), ("mixtral-8x7b", 511)])
def test_fused_front_matches_torch(cuda, name, pos):
    import torch
    sh = C.load_shape(name)
    W = init_dense_weights(sh, seed=2, device=cuda)
    L = W.layers[1]
    max_seq = 600
    cos, sin = rope_tables(sh, max_seq, cuda)
    g = torch.Generator().manual_seed(4)
    h = (torch.randn((1, sh.hidden), generator=g) * 0.5).to(torch.bfloat16).to(cuda)
    kv_a, kv_b = KVCache(sh, max_seq, cuda), KVCache(sh, max_seq, cuda)
    hist = (torch.randn(kv_a.k.shape, generator=g) * 0.3).to(torch.bfloat16).to(cuda)
    hv = (torch.randn(kv_a.v.shape, generator=g) * 0.3).to(torch.bfloat16).to(cuda)
    for kv in (kv_a, kv_b):
        kv.k.copy_(hist)
        kv.v.copy_(hv)
    p = torch.tensor([pos], dtype=torch.long, device=cuda)
    ar = torch.arange(max_seq, device=cuda)
    mask = torch.where(ar <= pos, 0.0, float("-inf")).to(torch.bfloat16).view(1, 1, 1, max_seq)
    h1_ref = attention_decode_static(sh, L, h, kv_a, 1, p, mask, cos, sin)
    a2_ref = rms_norm(h1_ref, L["ln2"], sh.rms_eps)
    h1, a2 = torch.empty_like(h), torch.empty_like(h)
    decode_front_fused(sh, L, h, kv_b, 1, p, mask, cos, sin, h1, a2)
    torch.cuda.synchronize()
    assert torch.equal(kv_a.k, kv_b.k) and torch.equal(kv_a.v, kv_b.v)
    for got, ref in ((h1, h1_ref), (a2, a2_ref)):
        rel = ((got.float() - ref.float()).norm() / ref.float().norm()).item()
        assert rel < 4e-3, rel
        # a handful of one-ulp differences from the f32 reduction order at most
        assert (got != ref).float().mean().item() < 0.05
