"""Next-layer expert predictor — drop-in mirror of ``duoserve.predictor``
(``/root/reference/pkg/src/duoserve/predictor.py``) whose inference runs on
the B200 through the fused K5 kernel (``ds_predictor_forward``).

Mirrored surface:
  FULL_HIDDEN / TEST_HIDDEN, PredictorError ....... predictor.py:24-33
  StateVector, feature_length, construct_input .... predictor.py:53-106
  ExpertMLP (init, parameters, eval forward) ....... predictor.py:141-232
  predict_topk, topk_indices ........................ predictor.py:411-421
  MLPPredictor / OraclePredictor / ComplementPredictor /
  PopularityPredictor / PrecomputedPredictor ........ predictor.py:424-510
  HitRateReport, evaluate ........................... predictor.py:513-570
  save_model / load_model (container format) ....... predictor.py:577-646

What runs where:
  * ``ExpertMLP.forward(X, train=False)`` and every predictor built on an
    ExpertMLP execute on the GPU (``DeviceMLP``): the State Constructor is
    fused into the kernel, which reads the selection history, the
    popularity row and the affinity matrix from HBM.  There is no CPU
    forward in this package; without the CUDA library these raise
    ``DeviceError``.
  * ``construct_input`` is kept on the host for API parity (it is what the
    kernel computes; tests compare both).
  * Training (predictor.py:109-130, 234-404: ``build_training_set``,
    ``bce_loss``, ``train``, ``gradient_check``, ``TrainReport``) is the
    offline preprocess; it runs on the GPU in torch float64 (training.py) and
    is re-exported here under the reference's names.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .stats import AffinityMatrix, PopularityMatrix
from .trace import ActivationTrace, TraceDataset

FULL_HIDDEN = (2048, 1024, 512, 256, 128, 64)
TEST_HIDDEN = (8, 8, 8, 8, 8, 8)
_INIT_TAG = 0x4D4C50  # SeedSequence((seed, 0x4D4C50)) — predictor.py:158


class PredictorError(ValueError):
    """Invalid predictor input, shape mismatch or malformed model file."""


class TrainingDivergedError(RuntimeError):
    def __init__(self, learning_rate: float, epoch: int, batch_index: int):
        self.learning_rate, self.epoch, self.batch_index = learning_rate, epoch, batch_index
        super().__init__(f"non-finite loss at epoch {epoch}, batch {batch_index} "
                         f"(learning_rate={learning_rate})")


# --------------------------------------------------------------------------
# State Constructor (host restatement, kept for API parity)

@dataclass(frozen=True, eq=False)
class StateVector:
    history: np.ndarray     # (L*k,) int64 — expert+1, 0 = pad
    popularity: np.ndarray  # (M,)
    affinity: np.ndarray    # (M,) pooled or (k*M,) concatenated
    layer_pos: float

    def as_features(self, M: int) -> np.ndarray:
        return np.concatenate([self.history.astype(np.float64) / M, self.popularity,
                               self.affinity, np.array([self.layer_pos])])


def feature_length(L: int, M: int, k: int, affinity_mode: str = "pool") -> int:
    return L * k + M + (M if affinity_mode == "pool" else k * M) + 1


def _mode_code(mode: str) -> int:
    if mode not in ("pool", "concat"):
        raise PredictorError(f"affinity_mode must be 'pool' or 'concat', got {mode!r}")
    return 0 if mode == "pool" else 1


def construct_input(trace: ActivationTrace, l: int, pop: PopularityMatrix, aff: AffinityMatrix,
                    affinity_mode: str = "pool") -> StateVector:
    L, k = len(trace.path), len(trace.path[0])
    _mode_code(affinity_mode)
    if not 1 <= l < L:
        raise PredictorError(f"target layer must be in [1, {L}); layer 0 is fetched after the gate")
    hist = np.zeros(L * k, dtype=np.int64)
    done = np.asarray(trace.path[:l], dtype=np.int64).reshape(-1) + 1
    hist[:done.size] = done
    rows = aff.values[l - 1][list(trace.path[l - 1])]
    pooled = rows.mean(axis=0) if affinity_mode == "pool" else rows.reshape(-1)
    return StateVector(history=hist, popularity=pop.values[l].copy(), affinity=pooled.copy(),
                       layer_pos=l / (L - 1))


# --------------------------------------------------------------------------
# the network (weights on the host as the master copy; inference on device)

class ExpertMLP:
    """Seven-layer multi-label classifier (predictor.py:141-232).

    Parameters live in float64 numpy arrays exactly as in the reference (so
    the container round-trips bitwise); ``forward`` in eval mode runs the
    fused sm_100a kernel.  The device copy is (re)packed lazily and cached
    until ``invalidate_device()`` is called after an in-place edit.
    """

    def __init__(self, input_dim: int, output_dim: int, hidden=FULL_HIDDEN, dropout: float = 0.1,
                 seed: int = 0, meta: dict | None = None):
        self.input_dim, self.output_dim = int(input_dim), int(output_dim)
        self.hidden = tuple(int(h) for h in hidden)
        self.dropout, self.seed = float(dropout), int(seed)
        self.meta = dict(meta or {})
        dims = (self.input_dim, *self.hidden, self.output_dim)
        rng = np.random.default_rng(np.random.SeedSequence((seed, _INIT_TAG)))
        # He-normal init, drawn layer by layer in order (predictor.py:159-161)
        self.W = []
        for fan_in, fan_out in zip(dims[:-1], dims[1:]):
            self.W.append(rng.normal(0.0, np.sqrt(2.0 / fan_in), size=(fan_in, fan_out)))
        self.b = [np.zeros(n) for n in dims[1:]]
        self.gamma = [np.ones(h) for h in self.hidden]
        self.beta = [np.zeros(h) for h in self.hidden]
        self.run_mean = [np.zeros(h) for h in self.hidden]
        self.run_var = [np.ones(h) for h in self.hidden]
        self._device = None

    def parameters(self) -> list:
        out = []
        for i, (w, b) in enumerate(zip(self.W, self.b)):
            out += [w, b]
            if i < len(self.hidden):
                out += [self.gamma[i], self.beta[i]]
        return out

    def invalidate_device(self) -> None:
        self._device = None

    def device(self, device=None) -> "DeviceMLP":
        if self._device is None:
            self._device = DeviceMLP(self, device)
        return self._device

    def forward(self, X, train: bool = False, dropout_rng=None, update_running: bool = False):
        if train or update_running:
            raise PredictorError("training-mode forward is an offline preprocess and is not "
                                 "implemented on the serving path")
        X = np.asarray(X, dtype=np.float64)
        single = X.ndim == 1
        X2 = X[None, :] if single else X
        if X2.ndim != 2 or X2.shape[1] != self.input_dim:
            raise PredictorError(f"input has shape {X.shape}, expected (*, {self.input_dim})")
        probs = self.device().forward_features(X2)
        return probs[0] if single else probs


def topk_indices(scores, k: int) -> tuple:
    """Stable argsort of -scores, first k, returned sorted (predictor.py:419-421)."""
    order = np.argsort(-np.asarray(scores), kind="stable")[:k]
    return tuple(sorted(int(i) for i in order))


def predict_topk(net: ExpertMLP, state, k: int) -> tuple:
    if isinstance(state, StateVector):
        state = state.as_features(net.output_dim)
    return topk_indices(net.forward(state), k)


# --------------------------------------------------------------------------
# device side

def _container_blob(net: ExpertMLP) -> np.ndarray:
    return np.concatenate([np.ascontiguousarray(a, dtype="<f8").reshape(-1) for _, a in _array_specs(net)])


class DeviceMLP:
    """Packed fp64 weights of one ExpertMLP in HBM + the K5 launchers."""

    def __init__(self, net: ExpertMLP, device=None):
        import torch
        from . import _lib
        self.torch = torch
        self.lib = _lib
        self.device = torch.device(device or "cuda")
        self.desc = _lib.MlpDesc.make(net.input_dim, net.output_dim, net.hidden)
        n_cont = _lib.query("ds_mlp_container_doubles", self.desc)
        n_pack = _lib.query("ds_mlp_packed_doubles", self.desc)
        blob = _container_blob(net)
        if blob.size != n_cont:
            raise PredictorError(f"container has {blob.size} doubles, kernel expects {n_cont}")
        cont = torch.from_numpy(blob).to(self.device)
        self.packed = torch.empty(n_pack, dtype=torch.float64, device=self.device)
        _lib.call("ds_mlp_pack", self.desc, _lib.ptr(cont), _lib.ptr(self.packed), _lib.stream_ptr())
        torch.cuda.current_stream().synchronize()
        self.M = net.output_dim
        self.input_dim = net.input_dim
        self.nbytes = self.packed.numel() * 8
        self._ws = {}

    def workspace(self, B: int):
        t = self.torch
        need = self.lib.query("ds_mlp_workspace_bytes", self.desc, max(B, 1))
        ws = self._ws.get("buf")
        if ws is None or ws.numel() < need:
            ws = t.empty(need, dtype=t.uint8, device=self.device)
            self._ws["buf"] = ws
        return ws

    def forward_features(self, X: np.ndarray, topk: int = 0):
        t = self.torch
        B = X.shape[0]
        Xd = t.from_numpy(np.ascontiguousarray(X, dtype=np.float64)).to(self.device)
        probs = t.empty((B, self.M), dtype=t.float64, device=self.device)
        out = t.empty((B, max(topk, 1)), dtype=t.int32, device=self.device)
        ws = self.workspace(B)
        self.lib.call("ds_mlp_forward_features", self.desc, self.lib.ptr(self.packed), self.lib.ptr(Xd),
                      B, topk, self.lib.ptr(out), self.lib.ptr(probs), self.lib.ptr(ws), ws.numel(),
                      self.lib.stream_ptr())
        p = probs.cpu().numpy()
        return (p, out.cpu().numpy()) if topk else p

    def predict_state(self, hist, target, pop_d, aff_d, L: int, M: int, k: int, mode: int, topk: int,
                      out=None, probs=None, stream=None):
        """Device-resident launch: hist [B, L*k] int32, target [B] int32 (all device)."""
        t = self.torch
        B = hist.shape[0]
        if out is None:
            out = t.empty((B, topk), dtype=t.int32, device=self.device)
        ws = self.workspace(B)
        from .ops import _count
        _count("ds_predictor_forward", 1 if B <= 8 else 9)
        self.lib.call("ds_predictor_forward", self.desc, self.lib.ptr(self.packed), self.lib.ptr(hist),
                      self.lib.ptr(target), self.lib.ptr(pop_d), self.lib.ptr(aff_d), L, M, k, mode, B,
                      topk, self.lib.ptr(out), self.lib.ptr(probs), self.lib.ptr(ws), ws.numel(),
                      self.lib.stream_ptr(stream))
        return out


class StatsOnDevice:
    """pop (L, M) and aff (L-1, M, M) float64 tables resident in HBM."""

    def __init__(self, pop: PopularityMatrix, aff: AffinityMatrix, device=None):
        import torch
        self.pop = torch.from_numpy(np.ascontiguousarray(pop.values, dtype=np.float64)).to(device or "cuda")
        self.aff = torch.from_numpy(np.ascontiguousarray(aff.values, dtype=np.float64)).to(device or "cuda")
        self.L, self.M = pop.values.shape


def _history_rows(traces, layers, L: int, k: int) -> np.ndarray:
    """(B, L*k) int32 histories: full paths +1 (the kernel masks layers >= l)."""
    paths = np.asarray([t.path for t in traces], dtype=np.int32).reshape(len(traces), L * k)
    return paths + 1


# --------------------------------------------------------------------------
# predictor protocol (name + predict(trace, l) -> sorted tuple)

class MLPPredictor:
    """ExpertMLP bound to its statistics; every call runs the fused kernel."""

    name = "expert-mlp"

    def __init__(self, net: ExpertMLP, pop: PopularityMatrix, aff: AffinityMatrix):
        self.net, self.pop, self.aff = net, pop, aff
        self.affinity_mode = net.meta.get("affinity_mode", "pool")
        self._mode = _mode_code(self.affinity_mode)
        self._stats = None

    def _dev(self):
        if self._stats is None:
            self._stats = StatsOnDevice(self.pop, self.aff)
        return self.net.device(), self._stats

    def predict_batch(self, traces, layers, with_probs: bool = False):
        """Batched predictions for (traces[i], layers[i]) pairs -> (B, k) int32."""
        import torch
        traces = list(traces)
        layers = np.asarray(layers, dtype=np.int32)
        if not traces:
            return np.zeros((0, 0), dtype=np.int32)
        L, k = len(traces[0].path), len(traces[0].path[0])
        if layers.min() < 1 or layers.max() >= L:
            raise PredictorError(f"target layer must be in [1, {L}); layer 0 is fetched after the gate")
        k_out = int(self.net.meta.get("k", k))
        dev, st = self._dev()
        M = st.M
        if self.net.input_dim != feature_length(L, M, k, self.affinity_mode):
            raise PredictorError("network input_dim does not match the trace shape")
        hist = torch.from_numpy(_history_rows(traces, layers, L, k)).to(dev.device)
        tgt = torch.from_numpy(layers).to(dev.device)
        probs = torch.empty((len(traces), M), dtype=torch.float64, device=dev.device) if with_probs else None
        out = dev.predict_state(hist, tgt, st.pop, st.aff, L, M, k, self._mode, k_out, probs=probs)
        res = out.cpu().numpy()
        return (res, probs.cpu().numpy()) if with_probs else res

    def predict(self, trace: ActivationTrace, l: int) -> tuple:
        return tuple(int(e) for e in self.predict_batch([trace], [l])[0])


class OraclePredictor:
    name = "oracle"

    def predict(self, trace: ActivationTrace, l: int) -> tuple:
        return tuple(trace.path[l])


class ComplementPredictor:
    """Adversarial stub: the first k experts outside the true selection."""

    name = "complement"

    def __init__(self, M: int):
        self.M = M

    def predict(self, trace: ActivationTrace, l: int) -> tuple:
        true = set(trace.path[l])
        k = len(trace.path[l])
        wrong = [e for e in range(self.M) if e not in true]
        if len(wrong) < k:
            raise PredictorError(f"complement stub needs M >= 2k, have M={self.M}, k={k}")
        return tuple(wrong[:k])


class PopularityPredictor:
    name = "popularity-topk"

    def __init__(self, pop: PopularityMatrix, k: int):
        self.pop, self.k = pop, k

    def predict(self, trace: ActivationTrace, l: int) -> tuple:
        return topk_indices(self.pop.values[l], self.k)


class PrecomputedPredictor:
    """Lookup table filled by one batched device pass (predictor.py:480-510)."""

    name = "expert-mlp"

    def __init__(self, table: dict):
        self.table = table

    @classmethod
    def from_net(cls, net: ExpertMLP, ds: TraceDataset, pop: PopularityMatrix,
                 aff: AffinityMatrix) -> "PrecomputedPredictor":
        if not ds.traces or ds.L < 2:
            return cls({})
        pred = MLPPredictor(net, pop, aff)
        traces = [t for t in ds.traces for _ in range(1, ds.L)]
        layers = [l for _ in ds.traces for l in range(1, ds.L)]
        sets = pred.predict_batch(traces, layers)
        table = {(t.request_id, t.token_index, l): tuple(int(e) for e in s)
                 for t, l, s in zip(traces, layers, sets)}
        return cls(table)

    def predict(self, trace: ActivationTrace, l: int) -> tuple:
        return self.table[(trace.request_id, trace.token_index, l)]


@dataclass
class HitRateReport:
    topk_hit_rate: float
    at_least_one_rate: float
    per_layer: list
    n_evaluated: int
    predictor: str = "expert-mlp"

    def to_dict(self) -> dict:
        return {"schema_version": 1, "predictor": self.predictor, "topk_hit_rate": self.topk_hit_rate,
                "at_least_one_rate": self.at_least_one_rate, "per_layer": self.per_layer,
                "n_evaluated": self.n_evaluated}


def evaluate(predictor, ds_test: TraceDataset, pop: PopularityMatrix | None = None,
             aff: AffinityMatrix | None = None) -> HitRateReport:
    """Top-k-exact and at-least-one hit rates over (trace, l >= 1) (predictor.py:532-570)."""
    if not ds_test.traces:
        raise PredictorError("cannot evaluate on an empty test set")
    if isinstance(predictor, ExpertMLP):
        if pop is None or aff is None:
            raise PredictorError("evaluating a raw network needs popularity and affinity")
        predictor = MLPPredictor(predictor, pop, aff)
    if isinstance(predictor, MLPPredictor):
        name = predictor.name
        predictor = PrecomputedPredictor.from_net(predictor.net, ds_test, predictor.pop, predictor.aff)
    else:
        name = getattr(predictor, "name", type(predictor).__name__)
    L = ds_test.L
    exact = np.zeros(L, dtype=np.int64)
    any_hit = np.zeros(L, dtype=np.int64)
    n = np.zeros(L, dtype=np.int64)
    for t in ds_test.traces:
        for l in range(1, L):
            p, q = set(predictor.predict(t, l)), set(t.path[l])
            exact[l] += p == q
            any_hit[l] += bool(p & q)
            n[l] += 1
    per_layer = [{"layer": l, "topk_hit_rate": exact[l] / n[l], "at_least_one_rate": any_hit[l] / n[l],
                  "n": int(n[l])} for l in range(1, L)]
    for row in per_layer:
        row["topk_hit_rate"] = float(row["topk_hit_rate"])
        row["at_least_one_rate"] = float(row["at_least_one_rate"])
    total = int(n.sum())
    return HitRateReport(topk_hit_rate=float(exact.sum() / total),
                         at_least_one_rate=float(any_hit.sum() / total),
                         per_layer=per_layer, n_evaluated=total, predictor=name)


# --------------------------------------------------------------------------
# model container (predictor.py:577-646)

def _array_specs(net: ExpertMLP) -> list:
    specs = []
    for i, (w, b) in enumerate(zip(net.W, net.b)):
        specs += [(f"W{i}", w), (f"b{i}", b)]
    for i in range(len(net.hidden)):
        specs += [(f"gamma{i}", net.gamma[i]), (f"beta{i}", net.beta[i]),
                  (f"run_mean{i}", net.run_mean[i]), (f"run_var{i}", net.run_var[i])]
    return specs


def save_model(net: ExpertMLP, path) -> None:
    specs = _array_specs(net)
    header = {"format": "duoserve-expertmlp", "version": 1, "input_dim": net.input_dim,
              "output_dim": net.output_dim, "hidden": list(net.hidden), "dropout": net.dropout,
              "seed": net.seed, "meta": net.meta,
              "arrays": [{"name": n, "shape": list(a.shape)} for n, a in specs]}
    with Path(path).open("wb") as f:
        f.write(json.dumps(header, sort_keys=True).encode("utf-8") + b"\n")
        for _, a in specs:
            f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def load_model(path) -> ExpertMLP:
    path = Path(path)
    raw = path.read_bytes()
    nl = raw.find(b"\n")
    if nl < 0:
        raise PredictorError(f"{path}: not a model container (missing header)")
    try:
        head = json.loads(raw[:nl].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as e:
        raise PredictorError(f"{path}: bad model header: {e}") from e
    if head.get("format") != "duoserve-expertmlp" or head.get("version") != 1:
        raise PredictorError(f"{path}: unsupported model format/version")
    net = ExpertMLP(head["input_dim"], head["output_dim"], hidden=head["hidden"],
                    dropout=head["dropout"], seed=head.get("seed", 0), meta=head.get("meta", {}))
    arrays, off = {}, nl + 1
    for spec in head["arrays"]:
        shape = tuple(spec["shape"])
        cnt = int(np.prod(shape)) if shape else 1
        end = off + 8 * cnt
        if end > len(raw):
            raise PredictorError(f"{path}: truncated model data at array {spec['name']}")
        arrays[spec["name"]] = np.frombuffer(raw[off:end], dtype="<f8").reshape(shape).copy()
        off = end
    try:
        for i in range(len(net.W)):
            net.W[i], net.b[i] = arrays[f"W{i}"], arrays[f"b{i}"]
        for i in range(len(net.hidden)):
            net.gamma[i], net.beta[i] = arrays[f"gamma{i}"], arrays[f"beta{i}"]
            net.run_mean[i], net.run_var[i] = arrays[f"run_mean{i}"], arrays[f"run_var{i}"]
    except KeyError as e:
        raise PredictorError(f"{path}: model container missing array {e}") from e
    return net


# training (offline preprocess, predictor.py:109-130, 234-404) runs on the GPU
# in torch float64: training.py
from .training import TrainReport, bce_loss, build_training_set, gradient_check, train  # noqa: E402,F401
