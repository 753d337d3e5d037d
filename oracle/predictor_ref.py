"""numpy restatement of the reference predictor's inference path (oracle).

Follows /root/reference/pkg/src/duoserve/predictor.py exactly, op for op:
  features      predictor.py:66-72 (as_features), :80-106 (construct_input)
  eval forward  predictor.py:197-232 (train=False branch)
  sigmoid       predictor.py:132-138
  topk          predictor.py:419-421
He init         predictor.py:150-166
Container I/O   predictor.py:577-646
"""

from __future__ import annotations

import json

import numpy as np

BN_EPS = 1e-5  # predictor.py:27


def features(path, l: int, pop_values: np.ndarray, aff_values: np.ndarray, mode: str = "pool") -> np.ndarray:
    """predictor.py:80-106 + :66-72 for one (path, target layer l)."""
    L, k = len(path), len(path[0])
    M = pop_values.shape[1]
    assert 1 <= l < L
    history = np.zeros(L * k, dtype=np.int64)
    flat = [e + 1 for sel in path[:l] for e in sel]
    history[: len(flat)] = flat
    rows = aff_values[l - 1][list(path[l - 1])]
    affv = rows.mean(axis=0) if mode == "pool" else rows.reshape(-1)
    return np.concatenate([history.astype(np.float64) / M, pop_values[l].copy(), affv.copy(),
                           np.array([l / (L - 1)])])


def sigmoid(z: np.ndarray) -> np.ndarray:
    """predictor.py:132-138."""
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


class RefNet:
    """Weights in the reference's layout (W[i] is (in, out))."""

    def __init__(self, input_dim, output_dim, hidden, seed=0, dropout=0.1, meta=None):
        self.input_dim, self.output_dim, self.hidden = input_dim, output_dim, tuple(hidden)
        self.seed, self.dropout, self.meta = seed, dropout, dict(meta or {})
        rng = np.random.default_rng(np.random.SeedSequence((seed, 0x4D4C50)))
        dims = [input_dim, *self.hidden, output_dim]
        self.W = [rng.normal(0.0, np.sqrt(2.0 / dims[i]), size=(dims[i], dims[i + 1]))
                  for i in range(len(dims) - 1)]
        self.b = [np.zeros(dims[i + 1]) for i in range(len(dims) - 1)]
        self.gamma = [np.ones(h) for h in self.hidden]
        self.beta = [np.zeros(h) for h in self.hidden]
        self.run_mean = [np.zeros(h) for h in self.hidden]
        self.run_var = [np.ones(h) for h in self.hidden]

    def forward(self, X: np.ndarray) -> np.ndarray:
        """Eval-mode forward, predictor.py:197-232."""
        A = np.asarray(X, dtype=np.float64)
        single = A.ndim == 1
        if single:
            A = A[None, :]
        for i in range(len(self.hidden)):
            Z = A @ self.W[i] + self.b[i]
            inv_std = 1.0 / np.sqrt(self.run_var[i] + BN_EPS)
            zhat = (Z - self.run_mean[i]) * inv_std
            H = self.gamma[i] * zhat + self.beta[i]
            A = np.maximum(H, 0.0)
        P = sigmoid(A @ self.W[-1] + self.b[-1])
        return P[0] if single else P


def topk_indices(scores, k: int) -> tuple:
    """predictor.py:419-421."""
    order = np.argsort(-np.asarray(scores), kind="stable")
    return tuple(sorted(int(i) for i in order[:k]))


def topk_margin(scores, k: int) -> float:
    """p_(k) - p_(k+1) of one row (how close the set decision was)."""
    s = np.sort(np.asarray(scores))[::-1]
    return float(s[k - 1] - s[k]) if len(s) > k else float("inf")


def load_container(path) -> RefNet:
    """predictor.py:610-646."""
    raw = open(path, "rb").read()
    nl = raw.find(b"\n")
    head = json.loads(raw[:nl].decode())
    net = RefNet(head["input_dim"], head["output_dim"], head["hidden"], head.get("seed", 0),
                 head["dropout"], head.get("meta", {}))
    off = nl + 1
    arrs = {}
    for spec in head["arrays"]:
        shape = tuple(spec["shape"])
        n = int(np.prod(shape)) if shape else 1
        arrs[spec["name"]] = np.frombuffer(raw[off:off + 8 * n], dtype="<f8").reshape(shape).copy()
        off += 8 * n
    for i in range(len(net.W)):
        net.W[i], net.b[i] = arrs[f"W{i}"], arrs[f"b{i}"]
    for i in range(len(net.hidden)):
        net.gamma[i], net.beta[i] = arrs[f"gamma{i}"], arrs[f"beta{i}"]
        net.run_mean[i], net.run_var[i] = arrs[f"run_mean{i}"], arrs[f"run_var{i}"]
    return net


def container_bytes(net: RefNet) -> bytes:
    """predictor.py:590-607 byte stream (for digest comparison)."""
    specs = []
    for i in range(len(net.W)):
        specs += [(f"W{i}", net.W[i]), (f"b{i}", net.b[i])]
    for i in range(len(net.hidden)):
        specs += [(f"gamma{i}", net.gamma[i]), (f"beta{i}", net.beta[i]),
                  (f"run_mean{i}", net.run_mean[i]), (f"run_var{i}", net.run_var[i])]
    head = {"format": "duoserve-expertmlp", "version": 1, "input_dim": net.input_dim,
            "output_dim": net.output_dim, "hidden": list(net.hidden), "dropout": net.dropout,
            "seed": net.seed, "meta": net.meta,
            "arrays": [{"name": n, "shape": list(a.shape)} for n, a in specs]}
    out = json.dumps(head, sort_keys=True).encode() + b"\n"
    return out + b"".join(np.ascontiguousarray(a, dtype="<f8").tobytes() for _, a in specs)


def predict_sets(net: RefNet, paths, layers, pop_values, aff_values, k: int, mode: str = "pool",
                 batched: bool = True):
    """Predicted sorted sets + probabilities for (paths[i], layers[i])."""
    X = np.stack([features(p, l, pop_values, aff_values, mode) for p, l in zip(paths, layers)])
    P = net.forward(X) if batched else np.stack([net.forward(x) for x in X])
    return [topk_indices(p, k) for p in P], P
