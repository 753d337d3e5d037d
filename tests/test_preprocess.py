"""Host logic of the preprocess loop (no GPU): engine paths -> traces, pin order."""

import numpy as np

from paper_2509_07379_b200.preprocess import engine_traces, rank_popular
from paper_2509_07379_b200.stats import PopularityMatrix
from paper_2509_07379_b200.trace import TraceDataset


class _Eng:
    def __init__(self):
        self.paths_prefill = np.array([[[0, 3], [1, 2]], [[2, 5], [0, 7]]], dtype=np.int32)   # [T=2, L=2, k=2]
        self.paths_decode = [((1, 4), (3, 6))]


def test_engine_traces_positions_and_phases():
    tr = engine_traces(_Eng(), 7)
    assert [(t.request_id, t.phase, t.token_index) for t in tr] == [(7, "prefill", 0), (7, "prefill", 1),
                                                                   (7, "decode", 2)]
    assert tr[1].path == ((2, 5), (0, 7)) and tr[2].path == ((1, 4), (3, 6))
    TraceDataset("x", 2, 8, 2, tr)          # validates shape, sortedness and phase order


def test_rank_popular_order_and_ties():
    vals = np.array([[0.1, 0.3, 0.3, 0.0], [0.3, 0.05, 0.2, 0.0]])
    pop = PopularityMatrix(vals, np.zeros(vals.shape, dtype=np.int64), 1)
    assert rank_popular(pop)[:4] == [(0, 1), (0, 2), (1, 0), (1, 2)]
    assert rank_popular(pop, experts=[0, 2])[:2] == [(0, 2), (1, 0)]


def test_streamed_bytes_floor_excludes_pinned():
    """Engine.streamed_bytes_floor: prefill counts activated minus pinned,
    decode counts gate minus pinned (l >= 1) and the on-demand fetch (l = 0)."""
    from paper_2509_07379_b200.engine import Engine

    class _S:
        blob_bytes = 10

    e = Engine.__new__(Engine)
    e.store, e.owned_set = _S(), set(range(8))
    e.log = [{"phase": "prefill", "layer": 0, "fetch": [0, 2], "activated": [0, 2, 5], "pinned": [5]},
             {"phase": "prefill", "layer": 1, "fetch": [1], "activated": [1]},
             {"phase": "decode", "token": 0, "layer": 0, "fetch": [3], "kind": "ondemand", "pinned": [4]},
             {"phase": "decode", "token": 0, "layer": 1, "pred": [1, 2], "gate": [2, 6], "refetch": [6],
              "pinned": [6]}]
    f = e.streamed_bytes_floor()
    assert f == {"prefill_bytes": 30, "decode_bytes_per_token": 20.0}
