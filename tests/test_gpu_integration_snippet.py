"""INTEGRATION.md's ctypes binding (the `duoserve/_b200.py` a reference
maintainer would add) executed verbatim against the in-tree library: its
B200MLPPredictor must predict exactly the reference predictor's sets
(oracle/predictor_ref, PrecomputedPredictor.from_net semantics,
/root/reference/pkg/src/duoserve/predictor.py:480-510).  `duoserve.predictor`
is shimmed to this repo's mirror (same `_array_specs`, predictor.py:577-600);
`cuda.bindings.runtime` (cuda-python) provides the device memory."""

import re
import sys
import types
from pathlib import Path

import numpy as np
import pytest

from oracle import predictor_ref
from paper_2509_07379_b200 import _lib
from paper_2509_07379_b200 import config as C
from paper_2509_07379_b200 import predictor as P
from paper_2509_07379_b200 import stats as S
from paper_2509_07379_b200 import trace as T

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _snippet() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    m = re.search(r"```python\n(# duoserve/_b200.py.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its duoserve/_b200.py snippet"
    return m.group(1)


def test_integration_snippet_predicts_reference_sets(cuda, tmp_path):
    pytest.importorskip("cuda.bindings.runtime")
    pkg = types.ModuleType("duoserve")
    pred = types.ModuleType("duoserve.predictor")
    pred._array_specs = P._array_specs
    pkg.predictor = pred
    saved = {k: sys.modules.get(k) for k in ("duoserve", "duoserve.predictor")}
    sys.modules["duoserve"], sys.modules["duoserve.predictor"] = pkg, pred
    try:
        _run_snippet(tmp_path)
    finally:
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v


def _run_snippet(tmp_path):
    src = _snippet().replace('C.CDLL("libduoserve_sm100.so")', f'C.CDLL("{_lib.LIB_PATH}")')
    ns = {}
    exec(compile(src, "INTEGRATION.md:_b200.py", "exec"), ns)
    cfg, _ = C.load_preset("tiny-4x8")
    ds = T.generate_traces(T.default_generator_params(4, 8, 0.8, seed=7), cfg, 6, 8, 8)
    pop, aff = S.build_popularity(ds), S.build_affinity(ds)
    net = P.ExpertMLP(P.feature_length(4, 8, 2), 8, seed=3, meta={"L": 4, "M": 8, "k": 2, "affinity_mode": "pool"})
    b2 = ns["B200MLPPredictor"](net, pop, aff, max_batch=256)
    traces = [t for t in ds.traces][:40]
    rows = [(t, l) for t in traces for l in range(1, 4)]
    got = b2.predict_batch([t for t, _ in rows], [l for _, l in rows])
    P.save_model(net, tmp_path / "net.bin")
    ref = predictor_ref.load_container(tmp_path / "net.bin")
    want, _ = predictor_ref.predict_sets(ref, [t.path for t, _ in rows], [l for _, l in rows], pop.values,
                                         aff.values, 2)
    assert [tuple(sorted(int(e) for e in r)) for r in got] == [tuple(int(e) for e in w) for w in want]
    assert b2.predict(traces[0], 2) == tuple(int(e) for e in want[1])
