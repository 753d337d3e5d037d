"""The paper's preprocess loop on the device at
tiny-4x8: serve calibration prompts on-demand, count pop/aff with the gate's
device counters, train the ExpertMLP on the GPU, then serve with it.

  * the device counters equal the reference statistics (stats.py:52-71) of
    the collected traces bit for bit;
  * the trained net's predicted sets on the served request equal the
    reference predictor's (oracle/predictor_ref, PrecomputedPredictor.from_net
    semantics) and the cache log equals sim_ref driven by them;
  * pinning by the measured popularity keeps tokens and logs consistent."""

import numpy as np
import pytest
import torch

from oracle import check_request, predictor_ref
from paper_2509_07379_b200 import config as C
from paper_2509_07379_b200 import predictor as P
from paper_2509_07379_b200 import stats as S
from paper_2509_07379_b200.engine import Engine
from paper_2509_07379_b200.model import init_dense_weights
from paper_2509_07379_b200.preprocess import preprocess, rank_popular

pytestmark = pytest.mark.gpu

PREFILL, DECODE = 48, 12


@pytest.fixture(scope="module")
def pre(cuda):
    shape = C.load_shape("tiny-4x8")
    dense = init_dense_weights(shape, seed=1, device="cpu").to(cuda)
    col = Engine(shape, "ondemand", seed=3, dense=dense, collect_stats=True, max_seq=PREFILL + DECODE + 8,
                 max_prefill=PREFILL)
    g = torch.Generator().manual_seed(5)
    prompts = [torch.randint(0, shape.vocab, (PREFILL,), generator=g) for _ in range(4)]
    res = preprocess(col, prompts, DECODE, epochs=3, seed=0)
    return dict(shape=shape, dense=dense, col=col, res=res, prompts=prompts)


def test_device_counters_equal_reference_stats(pre):
    from paper_2509_07379_b200.preprocess import collect_routing
    col, res = pre["col"], pre["res"]
    col.route_stats.reset()
    ds = collect_routing(col, pre["prompts"], DECODE)
    assert len(ds.traces) == 4 * (PREFILL + DECODE) == res.n_traces
    pop, aff = col.route_stats.matrices()
    ref_pop, ref_aff = S.build_popularity(ds), S.build_affinity(ds)
    assert np.array_equal(pop.values, ref_pop.values)
    assert np.array_equal(aff.values, ref_aff.values)
    assert np.array_equal(res.pop.values, ref_pop.values)


def test_trained_net_learns_and_reports(pre):
    res = pre["res"]
    losses = res.train_report.epoch_losses
    assert len(losses) == 3 and all(np.isfinite(losses)) and losses[-1] < losses[0]
    row = res.table("tiny-4x8")
    assert 0.0 <= row["all_tokens"]["top2"] <= row["all_tokens"]["at_least_one"] <= 1.0
    assert row["decode_tokens"]["n"] > 0


def test_serving_with_trained_net_matches_oracle(pre, cuda, tmp_path):
    shape, res = pre["shape"], pre["res"]
    L = shape.num_layers
    eng = Engine(shape, "duoserve", seed=3, dense=pre["dense"], store=pre["col"].store, predictor=res.net,
                 pop=res.pop, aff=res.aff, max_seq=PREFILL + DECODE + 8, max_prefill=PREFILL)
    ids = torch.randint(0, shape.vocab, (PREFILL,), generator=torch.Generator().manual_seed(77))
    toks = eng.generate(ids, DECODE)
    P.save_model(res.net, tmp_path / "net.bin")
    ref_net = predictor_ref.load_container(tmp_path / "net.bin")
    c = check_request.check_request(eng.log, eng.paths_prefill, eng.paths_decode, L, 2, ref_net, res.pop.values,
                                    res.aff.values)
    assert c["set_mismatches"] == 0 and c["log_equal"], c
    # residency budget spent on the measured most-popular experts: same tokens, log = sim_ref's pinned extension
    n = eng.pin_experts(res.pop, 3 * eng.store.blob_bytes)
    assert n == 3 and sorted(eng.pinned) == sorted(rank_popular(res.pop)[:3])
    eng.reset()
    assert eng.generate(ids, DECODE) == toks
    c = check_request.check_request(eng.log, eng.paths_prefill, eng.paths_decode, L, 2, ref_net, res.pop.values,
                                    res.aff.values, pinned=sorted(eng.pinned))
    assert c["set_mismatches"] == 0 and c["log_equal"], c
