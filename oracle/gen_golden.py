"""Generate tests/golden/ from the REFERENCE itself (run in the build
container, where /root/reference exists; the GPU box only reads the
committed fixtures).

    python oracle/gen_golden.py

Every fixture records the reference call that produced it.  Reference
modules used: duoserve.config / trace / stats / predictor
(/root/reference/pkg/src/duoserve).
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> None:
    sys.path.insert(0, str(REF))
    from duoserve import config as rc, predictor as rp, stats as rs, trace as rt

    OUT.mkdir(parents=True, exist_ok=True)
    manifest = {"generator": "oracle/gen_golden.py", "reference": str(REF), "fixtures": {}}

    def cfg_for(name, L, M=8, k=2):
        return rc.ModelConfig(name=name, num_layers=L, num_experts=M, top_k=k,
                              total_param_bytes=10**9, non_moe_bytes=10**8,
                              predictor_mem_bytes=0, kv_reserve_bytes=0)

    # ---- traces (byte-exact JSONL) + stats ------------------------------
    shapes = {"tiny": (4, 3, 16, 64), "mixtral-8x7b": (32, 1, 8, 8), "mixtral-8x22b": (56, 1, 4, 4)}
    datasets = {}
    for name, (L, nreq, dec, pre) in shapes.items():
        cfg = cfg_for(name, L)
        ds = rt.generate_traces(rt.default_generator_params(L, 8, 0.8, seed=7), cfg, nreq, dec, pre)
        rt.save_traces(ds, OUT / f"traces_{name}.jsonl")
        pop, aff = rs.build_popularity(ds), rs.build_affinity(ds)
        rs.save_matrices(pop, aff, OUT / f"matrices_{name}.json")
        datasets[name] = (cfg, ds, pop, aff)
        manifest["fixtures"][f"traces_{name}.jsonl"] = (
            f"generate_traces(default_generator_params({L},8,0.8,seed=7), L={L}, n_requests={nreq}, "
            f"decode_len={dec}, prefill_len={pre}); save_traces")
        manifest["fixtures"][f"matrices_{name}.json"] = "build_popularity/build_affinity; save_matrices"
    # chain + toy-4x2 datasets
    cfg = cfg_for("chain", 4)
    ds_chain = rt.generate_traces(rt.chain_generator_params(4, 8, seed=3), cfg, 2, 8, 8)
    rt.save_traces(ds_chain, OUT / "traces_chain.jsonl")
    toy_cfg, _ = rc.load_preset("toy-4x2")
    ds_toy = rt.generate_traces(rt.default_generator_params(4, 4, 0.5, seed=1), toy_cfg, 2, 4, 4)
    rt.save_traces(ds_toy, OUT / "traces_toy-4x2.jsonl")
    manifest["fixtures"]["traces_chain.jsonl"] = "generate_traces(chain_generator_params(4,8,seed=3), 2, 8, 8)"
    manifest["fixtures"]["traces_toy-4x2.jsonl"] = "generate_traces(default_generator_params(4,4,0.5,seed=1), toy-4x2, 2, 4, 4)"

    # ---- predictor vectors ------------------------------------------------
    def dump_predictions(tag, net, ds, pop, aff, mode="pool"):
        lookup = rp.PrecomputedPredictor.from_net(net, ds, pop, aff)
        keys, rows, sets = [], [], []
        for t in ds.traces:
            for l in range(1, ds.L):
                keys.append((t.request_id, t.token_index, l))
                rows.append(rp.construct_input(t, l, pop, aff, mode).as_features(ds.M))
                sets.append(lookup.predict(t, l))
        X = np.stack(rows)
        P = net.forward(X, train=False)
        # single-call path (MLPPredictor.predict) on the first few keys
        single = rp.MLPPredictor(net, pop, aff)
        n_single = min(16, len(keys))
        by_key = {(t.request_id, t.token_index): t for t in ds.traces}
        single_sets = [single.predict(by_key[k[:2]], k[2]) for k in keys[:n_single]]
        np.savez_compressed(OUT / f"pred_{tag}.npz", keys=np.array(keys, dtype=np.int64),
                            features=X, probs=P, sets=np.array(sets, dtype=np.int32),
                            single_sets=np.array(single_sets, dtype=np.int32))
        digest = hashlib.sha256(b"".join(
            np.ascontiguousarray(a, dtype="<f8").tobytes() for _, a in rp._array_specs(net))).hexdigest()
        manifest["fixtures"][f"pred_{tag}.npz"] = {
            "call": "PrecomputedPredictor.from_net + MLPPredictor.predict + ExpertMLP.forward(train=False)",
            "net": {"input_dim": net.input_dim, "hidden": list(net.hidden), "seed": net.seed,
                    "meta": net.meta}, "weights_sha256": digest}

    for name in shapes:
        cfg, ds, pop, aff = datasets[name]
        d_in = rp.feature_length(cfg.num_layers, 8, 2)
        for seed in (0, 1):
            net = rp.ExpertMLP(d_in, 8, seed=seed, meta={"L": cfg.num_layers, "M": 8, "k": 2,
                                                         "affinity_mode": "pool"})
            dump_predictions(f"{name}_full_s{seed}", net, ds, pop, aff)
    cfg, ds, pop, aff = datasets["tiny"]
    # concat affinity mode, full width
    net = rp.ExpertMLP(rp.feature_length(4, 8, 2, "concat"), 8, seed=2,
                       meta={"L": 4, "M": 8, "k": 2, "affinity_mode": "concat"})
    dump_predictions("tiny_concat_s2", net, ds, pop, aff, mode="concat")
    # trained nets (test width) — containers committed
    for tag, dsx in (("alpha08", ds), ("chain", ds_chain)):
        popx, affx = rs.build_popularity(dsx), rs.build_affinity(dsx)
        net, rep = rp.train(dsx, popx, affx, epochs=25, batch_size=64, learning_rate=3e-3, seed=5,
                            hidden=rp.TEST_HIDDEN)
        rp.save_model(net, OUT / f"model_trained_{tag}.bin")
        rs.save_matrices(popx, affx, OUT / f"matrices_trained_{tag}.json")
        dump_predictions(f"trained_{tag}", net, dsx, popx, affx)
        manifest["fixtures"][f"model_trained_{tag}.bin"] = {
            "call": "train(epochs=25,batch_size=64,learning_rate=3e-3,seed=5,hidden=TEST_HIDDEN); save_model",
            "losses": rep.epoch_losses[-3:]}
        rep_eval = rp.evaluate(net, dsx, popx, affx)
        (OUT / f"eval_trained_{tag}.json").write_text(json.dumps(rep_eval.to_dict(), sort_keys=True))
    # zero-weight net: probabilities exactly 0.5
    zero = rp.ExpertMLP(rp.feature_length(4, 8, 2), 8, hidden=rp.TEST_HIDDEN, seed=0)
    for W in zero.W:
        W[...] = 0.0
    rp.save_model(zero, OUT / "model_zero.bin")

    # ---- SPEC known answers ----------------------------
    A = rt.ActivationTrace(0, "decode", 0, ((0, 1), (2, 3), (0, 2), (1, 3)))
    B = rt.ActivationTrace(1, "decode", 0, ((0, 2), (2, 3), (0, 1), (1, 3)))
    dsAB = rt.TraceDataset("toy-4x2", 4, 4, 2, [A, B])
    popAB, affAB = rs.build_popularity(dsAB), rs.build_affinity(dsAB)
    sv = rp.construct_input(A, 1, popAB, affAB)
    known = {
        "pop_layer0": popAB.values[0].tolist(),
        "aff_l0_row0": affAB.values[0][0].tolist(),
        "construct_A_l1_history": sv.history.tolist(),
        "construct_A_l1_layer_pos": sv.layer_pos,
        "topk_ex1": list(rp.topk_indices(np.array([.9, .1, .8, .2]), 2)),
        "topk_equal": list(rp.topk_indices(np.array([.5, .5, .5, .5]), 2)),
        "bce_half_M8": rp.bce_loss(np.full((1, 8), 0.5), np.zeros((1, 8))),
        "slot_counts_8x7b": {p.value: rc.slot_count(p, rc.load_preset("mixtral-8x7b")[0])
                             for p in rc.SchedulerPolicy},
        "expert_bytes": {n: rc.load_preset(n)[0].expert_bytes for n in rc.preset_names()},
    }
    (OUT / "known_answers.json").write_text(json.dumps(known, indent=1, sort_keys=True))
    manifest["fixtures"]["known_answers.json"] = "SPEC.md:185,194,256,265,274,301-302 via the reference"
    (OUT / "MANIFEST.json").write_text(json.dumps(manifest, indent=1, sort_keys=True))
    print("wrote", len(list(OUT.iterdir())), "files to", OUT)


if __name__ == "__main__":
    main()
