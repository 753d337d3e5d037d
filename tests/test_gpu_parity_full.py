"""End-to-end parity at the metric configs (BASELINE configs[1] and [2]):
Mixtral-8x7B- and 8x22B-shaped W4 random-init models served by the B200
Engine (policy duoserve, 4 expert slots), prefill 512 + 8 decode tokens,
checked against the CPU oracle:

  * routing: every routed token of every layer, teacher forced (the GPU's gate
    input through oracle/routing_ref) — bit-exact indices;
  * predicted sets: every decode prediction vs oracle/predictor_ref (the
    reference's ExpertMLP + State Constructor, PrecomputedPredictor.from_net,
    /root/reference/pkg/src/duoserve/predictor.py:480-510) — bit-exact;
  * cache log vs oracle/sim_ref — equal;
  * MoE block output of layers {0, L/2, L-1} (prefill and two decode tokens)
    given the GPU's block input: f64 reference on the same W4 weights
    (prefill: the bf16-rounded dequantised weights K3 consumes; decode: the
    exact (q - z) s products K4 factorises) with the intermediate h rounded
    to bf16 as both kernels do; out_ref = bf16(h_in + reference).  The GPU
    accumulates in f32, so an output can land a bf16 rounding step away:
    >= MOE_EXACT_FRAC of the elements bit-identical, rel-L2(out - out_ref)
    <= MOE_REL_TOL of ||out_ref|| and max|out - out_ref| <= MOE_MAX_RMS of
    rms(out_ref) (near-zero outputs after cancellation carry the f32-vs-f64
    sum difference, so no per-element ulp bound).
Full-model CPU logits do not fit in host RAM at these shapes, so the
floating-point check goes layer by layer.
"""

import gc

import numpy as np
import pytest
import torch

from oracle import check_request, predictor_ref, w4_ref
from paper_2509_07379_b200 import _lib, ops
from paper_2509_07379_b200 import config as C
from paper_2509_07379_b200 import predictor as P
from paper_2509_07379_b200 import stats as S
from paper_2509_07379_b200 import trace as T
from paper_2509_07379_b200.engine import Engine
from tests import w4_torch

pytestmark = pytest.mark.gpu

PREFILL, DECODE = 512, 8
MOE_EXACT_FRAC = 0.85     # measured 0.891 (layer 0, W4 attention; 8x7B and 8x22B) .. 0.997 (layer 31)
MOE_REL_TOL = 2e-3        # measured <= 9.1e-4 (layer 0) and <= 2.5e-4 (layers 16, 31)
MOE_MAX_RMS = 0.1


def _predictor_inputs(shape):
    """As bench.py: ExpertMLP(d_in, 8, seed=0) + pop/aff from synthetic traces."""
    cfg = C.model_config_for_shape(shape)
    ds = T.generate_traces(T.default_generator_params(shape.num_layers, shape.num_experts, 0.8, seed=7), cfg,
                           n_requests=4, decode_len=16, prefill_len=16)
    pop, aff = S.build_popularity(ds), S.build_affinity(ds)
    net = P.ExpertMLP(P.feature_length(shape.num_layers, shape.num_experts, shape.top_k), shape.num_experts,
                      seed=0, meta={"L": shape.num_layers, "M": shape.num_experts, "k": shape.top_k,
                                    "affinity_mode": "pool"})
    return net, pop, aff


@pytest.fixture(scope="module", params=["mixtral-8x7b", "mixtral-8x22b"])
def served(request, cuda):
    shape = C.load_shape(request.param)
    net, pop, aff = _predictor_inputs(shape)
    eng = Engine(shape, "duoserve", seed=0, device=cuda, predictor=net, pop=pop, aff=aff,
                 max_seq=PREFILL + DECODE + 8, max_prefill=PREFILL)
    L = shape.num_layers
    eng.capture = []
    eng.capture_moe = {0, L // 2, L - 1}
    ids = torch.randint(0, shape.vocab, (PREFILL,), generator=torch.Generator().manual_seed(1))
    toks = eng.generate(ids, DECODE + 1)
    torch.cuda.synchronize()
    yield dict(shape=shape, eng=eng, net=net, pop=pop, aff=aff, toks=toks)
    eng.store.close()
    del eng
    gc.collect()
    torch.cuda.empty_cache()


def test_routing_bit_exact_teacher_forced(served):
    eng, shape = served["eng"], served["shape"]
    L = shape.num_layers
    r = check_request.check_routing(eng.capture, [eng.W.layers[l]["wg"] for l in range(L)], shape.top_k)
    print(shape.name, r)
    assert r["routed_tokens"] == PREFILL * L + DECODE * L
    assert r["mismatches"] == 0, r


def test_predicted_sets_and_cache_log_equal_oracle(served):
    eng, shape = served["eng"], served["shape"]
    L, k = shape.num_layers, shape.top_k
    net = served["net"]
    ref_net = predictor_ref.RefNet(net.input_dim, shape.num_experts, net.hidden, 0)
    assert len(eng.paths_decode) == DECODE
    r = check_request.check_request(eng.log, eng.paths_prefill, eng.paths_decode, L, k, ref_net,
                                    served["pop"].values, served["aff"].values)
    print(shape.name, r)
    assert r["predicted_sets"] == DECODE * (L - 1)
    assert r["set_mismatches"] == 0 and r["log_equal"], r


def test_moe_block_outputs_within_tolerance(served, cuda):
    eng, shape = served["eng"], served["shape"]
    d, ff, G, k = shape.hidden, shape.ffn, shape.group_size, shape.top_k
    recs = [r for r in eng.moe_records if r["phase"] == "prefill" or r["token"] in (0, DECODE - 1)]
    assert len(recs) == 3 * 3
    for rec in recs:
        l = rec["layer"]
        a = rec["a"].to(cuda)
        idx = rec["idx"].numpy()
        w = rec["w"][: idx.shape[0]].to(cuda, torch.float64)
        acc = torch.zeros((a.shape[0], d), dtype=torch.float64, device=cuda)
        for e in np.unique(idx):
            W = w4_torch.expert_weights(eng.store.blob(l, int(e)).to(cuda), d, ff, G,
                                        exact=rec["phase"] == "decode")
            for j in range(k):
                rows = torch.from_numpy(np.nonzero(idx[:, j] == e)[0]).to(cuda)
                if rows.numel():
                    acc[rows] += w[rows, j:j + 1] * w4_torch.expert_ffn(a[rows], W)
            del W
        h_in = rec["h_in"].to(cuda).double()
        out = rec["out"].to(cuda)
        ref_out = (h_in + acc).to(torch.bfloat16)
        exact = (ref_out.view(torch.int16) == out.view(torch.int16)).float().mean().item()
        o, r = out.double(), ref_out.double()
        rel = ((o - r).norm() / r.norm()).item()
        mx = ((o - r).abs().max() / r.pow(2).mean().sqrt()).item()
        contrib = ((o - h_in - acc).norm() / acc.norm()).item()
        print(f"{shape.name} {rec['phase']} layer {l} token {rec['token']}: bit-identical {exact:.4f}, "
              f"rel-L2 {rel:.2e} (of the block's contribution {contrib:.2e}), max/rms {mx:.3f}")
        assert exact >= MOE_EXACT_FRAC, (rec["phase"], l, exact)
        assert rel <= MOE_REL_TOL, (rec["phase"], l, rel)
        assert mx <= MOE_MAX_RMS, (rec["phase"], l, mx)


@pytest.mark.parametrize("name,m", [("mixtral-8x7b", 0), ("mixtral-8x22b", 2)])
def test_w4_dequant_full_shape_bit_exact(name, m, cuda):
    """ds_w4_generate + ds_w4_dequant at full expert shapes (4096 x 14336 W1;
    16384 x 6144 W2) equal oracle/w4_ref bit for bit, and so does the torch
    unpack the block check above uses."""
    shape = C.load_shape(name)
    d, ff, G = shape.hidden, shape.ffn, shape.group_size
    K, N = [(d, ff), (d, ff), (ff, d)][m]
    _, total = ops.expert_layout(d, ff, G)
    blob = torch.empty(total, dtype=torch.uint8, device=cuda)
    ops.w4_generate(0, 3, 5, d, ff, G, blob)
    st = ops.expert_struct(blob.data_ptr(), d, ff, G)
    lin = [st.w1, st.w3, st.w2][m]
    out = torch.empty((N, K), dtype=torch.bfloat16, device=cuda)
    _lib.call("ds_w4_dequant", Cc_byref(lin), K, N, G, _lib.ptr(out), _lib.stream_ptr())
    torch.cuda.synchronize()
    c, s, z = w4_ref.gen_linear(0, 3, 5, m, K, N, G)
    ref = w4_ref.dequant(c, s, z, K, N, G)
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(got, ref)
    tw = w4_torch.expert_weights(blob, d, ff, G, exact=False, dtype=torch.float32)[m]
    assert torch.equal(tw.to(torch.bfloat16).view(torch.int16), out.view(torch.int16))


def Cc_byref(x):
    import ctypes
    return ctypes.byref(x)
