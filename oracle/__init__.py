"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain numpy restatements of the reference's algorithms for the hot path
(/root/reference/pkg/src/duoserve and SPEC.md), each function citing the
reference file:line it follows.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this package,
and only as the checker or the timed CPU baseline — never as the product
path.  The product (paper_2509_07379_b200) never imports it.

Pinning status:
  predictor_ref  — PINNED: checked against golden vectors produced by the
                   reference itself (oracle/gen_golden.py -> tests/golden/).
  stats_ref      — PINNED: same, plus the reference's stats_oracle.
  sim_ref        — PINNED to the SPEC's hand-traced timeline fixtures
                    and memory example; the
                   reference ships no simulator code (SPEC-only module).
  routing_ref / w4_ref / model_ref — gate, W4 FFN and logits have no
                   reference code (third-party vLLM/AWQ);
                   pinned against the installed third-party HF transformers
                   5.5.0 Mixtral block (tests/golden/hf_mixtral_*.npz made by
                   oracle/gen_golden.py) for routing/FFN semantics.
"""
