"""ExpertMLP training (paper_2509_07379_b200/training.py)
against the reference: the golden nets in tests/golden/model_trained_*.bin
were produced by the reference's own train() (oracle/gen_golden.py:
epochs=25, batch_size=64, learning_rate=3e-3, seed=5, hidden=TEST_HIDDEN);
the same call here follows the same random stream, so the epoch losses agree
to rounding and the weights to ~1e-6 relative (f64 summation order only)."""

import json

import numpy as np
import pytest

from paper_2509_07379_b200 import config as C, predictor as P, stats as S, trace as T

CASES = (("alpha08", "traces_tiny.jsonl"), ("chain", "traces_chain.jsonl"))


def _cfg(L=4):
    return C.ModelConfig(name="golden", num_layers=L, num_experts=8, top_k=2, total_param_bytes=10**9,
                         non_moe_bytes=10**8, predictor_mem_bytes=0, kv_reserve_bytes=0)


def _data(golden, traces):
    ds = T.load_traces(golden / traces, _cfg())
    return ds, S.build_popularity(ds), S.build_affinity(ds)


def _check_against_golden(golden, tag, traces, device):
    ds, pop, aff = _data(golden, traces)
    net, rep = P.train(ds, pop, aff, epochs=25, batch_size=64, learning_rate=3e-3, seed=5,
                       hidden=P.TEST_HIDDEN, device=device)
    ref = P.load_model(golden / f"model_trained_{tag}.bin")
    man = json.loads((golden / "MANIFEST.json").read_text())
    ref_losses = man["fixtures"][f"model_trained_{tag}.bin"]["losses"]
    assert np.allclose(rep.epoch_losses[-3:], ref_losses, rtol=1e-10, atol=0)
    for a, b in zip(net.parameters(), ref.parameters()):
        assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-3)) < 1e-4
    for a, b in zip(net.run_mean + net.run_var, ref.run_mean + ref.run_var):
        assert np.max(np.abs(a - b)) < 1e-6
    assert rep.n_samples == len(ds.traces) * (ds.L - 1) and len(rep.epoch_losses) == 25
    return net, ds, pop, aff


@pytest.mark.parametrize("tag,traces", CASES)
def test_train_matches_reference_golden_cpu(golden, tag, traces):
    _check_against_golden(golden, tag, traces, "cpu")


def test_training_set_and_loss_mirror_reference(golden):
    ds, pop, aff = _data(golden, "traces_tiny.jsonl")
    X, Y = P.build_training_set(ds, pop, aff)
    assert X.shape == (len(ds.traces) * 3, P.feature_length(4, 8, 2)) and Y.sum() == X.shape[0] * 2
    t = ds.traces[5]
    assert np.array_equal(X[5 * 3 + 1], P.construct_input(t, 2, pop, aff).as_features(8))
    # bce_loss clips like the reference (predictor.py:277-286)
    assert abs(P.bce_loss(np.array([[1.0, 0.0]]), np.array([[1.0, 0.0]])) - 2 * -np.log(1 - 1e-7)) < 1e-15
    with pytest.raises(P.PredictorError):
        P.bce_loss(np.zeros((2, 3)), np.zeros((3, 2)))
    with pytest.raises(P.PredictorError):
        P.build_training_set(T.TraceDataset("x", 4, 8, 2, []), pop, aff)


def test_gradient_check_and_edge_cases(golden):
    ds, pop, aff = _data(golden, "traces_chain.jsonl")
    X, Y = P.build_training_set(ds, pop, aff)
    net = P.ExpertMLP(X.shape[1], 8, hidden=(4, 4), seed=3)
    assert P.gradient_check(net, X[:16], Y[:16], device="cpu") < 1e-6
    net0, rep0 = P.train(ds, pop, aff, epochs=0, hidden=P.TEST_HIDDEN, seed=1, device="cpu")
    fresh = P.ExpertMLP(X.shape[1], 8, hidden=P.TEST_HIDDEN, seed=1)
    assert all(np.array_equal(a, b) for a, b in zip(net0.parameters(), fresh.parameters()))
    assert rep0.epoch_losses == [] and rep0.to_dict()["schema_version"] == 1
    with pytest.raises(P.TrainingDivergedError):
        P.train(ds, pop, aff, epochs=3, batch_size=16, learning_rate=float("inf"), hidden=(4, 4), seed=0, device="cpu")


@pytest.mark.gpu
@pytest.mark.parametrize("tag,traces", CASES)
def test_train_on_gpu_matches_reference_and_predicts_like_it(golden, cuda, tag, traces):
    """On the B200 (float64 cuBLAS) the trained net matches the reference's,
    and the K5 kernel's predicted sets from it equal the sets the reference
    computed from ITS trained net (tests/golden/pred_trained_*.npz)."""
    net, ds, pop, aff = _check_against_golden(golden, tag, traces, cuda)
    g = np.load(golden / f"pred_trained_{tag}.npz")
    keys = [tuple(int(v) for v in k) for k in g["keys"]]
    by_key = {(t.request_id, t.token_index): t for t in ds.traces}
    sets = P.MLPPredictor(net, pop, aff).predict_batch([by_key[k[:2]] for k in keys], [k[2] for k in keys])
    got = np.array([list(s) for s in sets])
    probs = g["probs"]
    top = np.sort(probs, axis=1)
    margin = top[:, -2] - top[:, -3]                  # k-th vs (k+1)-th probability (k = 2)
    mism = np.any(got != g["sets"], axis=1)
    assert not np.any(mism & (margin > 1e-4)), np.nonzero(mism)
