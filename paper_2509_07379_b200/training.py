"""ExpertMLP training on the GPU — the reference's offline preprocess
(``/root/reference/pkg/src/duoserve/predictor.py:109-130, 234-404``; SURVEY.md
§8f row 3) in torch float64 on the B200.

Same public API as the reference (``build_training_set``, ``bce_loss``,
``TrainReport``, ``train``, ``gradient_check``; re-exported by
``paper_2509_07379_b200.predictor``) and the same algorithm, step for step:

* data — one sample per (trace, target layer l ≥ 1): the State Constructor
  features and the multi-hot gate selection (predictor.py:109-129);
* init — ``ExpertMLP(d_in, M, hidden, dropout, seed)`` (He-normal from
  ``SeedSequence((seed, 0x4D4C50))``, bit-identical to the reference);
* schedule — per epoch a permutation, per batch one dropout mask per hidden
  layer, both drawn from ``default_rng(SeedSequence((seed, 0x5452)))`` in the
  reference's order (masks are drawn on the host and uploaded, so the
  trajectory follows the reference's random stream exactly);
* forward — Linear → batch-norm on batch statistics (population variance,
  running stats updated with momentum 0.1 and the n/(n−1) correction) →
  ReLU → dropout, then Linear → sigmoid (predictor.py:197-232);
* objective / gradient — mean over the batch of BCE summed over experts; the
  gradient is the reference's analytic (P − Y)/B at the output
  (predictor.py:234-274), obtained by autograd on the logit form;
* optimiser — Adam (β1 0.9, β2 0.999, ε 1e-8) with the reference's update
  expression and operation order (predictor.py:313-336).

What differs is the floating-point summation order of the f64 matrix
products (cuBLAS vs BLAS), so losses and weights agree with the reference to
rounding, not bit for bit (tests/test_training.py pins the tolerance against
golden runs of the reference).  The trained network is an ordinary
``ExpertMLP``: save_model / load_model / the K5 inference kernel use it as is.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .stats import AffinityMatrix, PopularityMatrix
from .trace import TraceDataset

_BN_EPS = 1e-5
_BN_MOMENTUM = 0.1
_CLAMP_EPS = 1e-7
_TRAIN_TAG = 0x5452      # SeedSequence((seed, 0x5452)) — predictor.py:356


def build_training_set(ds: TraceDataset, pop: PopularityMatrix, aff: AffinityMatrix,
                       affinity_mode: str = "pool") -> tuple[np.ndarray, np.ndarray]:
    """One sample per (trace, target layer l in [1, L)): features and multi-hot labels."""
    from .predictor import PredictorError, construct_input, feature_length
    if len(ds.traces) == 0:
        raise PredictorError("cannot build a training set from an empty dataset")
    d = feature_length(ds.L, ds.M, ds.k, affinity_mode)
    n = len(ds.traces) * (ds.L - 1)
    X = np.empty((n, d))
    Y = np.zeros((n, ds.M))
    row = 0
    for trace in ds.traces:
        for l in range(1, ds.L):
            X[row] = construct_input(trace, l, pop, aff, affinity_mode).as_features(ds.M)
            Y[row, list(trace.path[l])] = 1.0
            row += 1
    return X, Y


def bce_loss(probs, labels) -> float:
    """Binary cross-entropy summed over experts, averaged over the batch."""
    from .predictor import PredictorError
    probs = np.asarray(probs, dtype=np.float64)
    labels = np.asarray(labels, dtype=np.float64)
    if probs.shape != labels.shape:
        raise PredictorError(f"shape mismatch: probs {probs.shape} vs labels {labels.shape}")
    p = np.clip(probs, _CLAMP_EPS, 1.0 - _CLAMP_EPS)
    per_sample = -(labels * np.log(p) + (1.0 - labels) * np.log(1.0 - p)).sum(axis=-1)
    return float(np.mean(per_sample))


@dataclass
class TrainReport:
    epochs: int
    seed: int
    batch_size: int
    learning_rate: float
    n_samples: int
    epoch_losses: list = field(default_factory=list)

    def to_dict(self) -> dict:
        return {"schema_version": 1, "epochs": self.epochs, "seed": self.seed, "batch_size": self.batch_size,
                "learning_rate": self.learning_rate, "n_samples": self.n_samples,
                "epoch_losses": self.epoch_losses}


class _DeviceNet:
    """The network's parameters and running statistics as float64 tensors."""

    def __init__(self, net, device):
        import torch
        self.torch = torch
        self.net = net
        t = lambda a: torch.tensor(a, dtype=torch.float64, device=device)
        self.W = [t(w).requires_grad_() for w in net.W]
        self.b = [t(b).requires_grad_() for b in net.b]
        self.gamma = [t(g).requires_grad_() for g in net.gamma]
        self.beta = [t(b).requires_grad_() for b in net.beta]
        self.run_mean = [t(m) for m in net.run_mean]
        self.run_var = [t(v) for v in net.run_var]

    def parameters(self) -> list:
        out = []
        for i in range(len(self.W)):
            out += [self.W[i], self.b[i]]
            if i < len(self.gamma):
                out += [self.gamma[i], self.beta[i]]
        return out

    def logits(self, X, masks=None, update_running: bool = False):
        """Training-mode forward (batch statistics) -> output logits."""
        torch = self.torch
        A = X
        for i in range(len(self.gamma)):
            Z = A @ self.W[i] + self.b[i]
            mu = Z.mean(dim=0)
            var = Z.var(dim=0, unbiased=False)
            if update_running:
                with torch.no_grad():
                    n = Z.shape[0]
                    unbiased = var * n / (n - 1) if n > 1 else var
                    self.run_mean[i] = (1 - _BN_MOMENTUM) * self.run_mean[i] + _BN_MOMENTUM * mu
                    self.run_var[i] = (1 - _BN_MOMENTUM) * self.run_var[i] + _BN_MOMENTUM * unbiased
            inv_std = 1.0 / torch.sqrt(var + _BN_EPS)
            H = self.gamma[i] * ((Z - mu) * inv_std) + self.beta[i]
            A = torch.relu(H)
            if masks is not None and masks[i] is not None:
                A = A * masks[i]
        return A @ self.W[-1] + self.b[-1]

    def loss_and_grads(self, X, Y, masks=None, update_running: bool = False):
        """(mean BCE of the clipped sigmoid, reported like bce_loss; grads of
        sum-over-experts BCE averaged over the batch = (P - Y)/B at the logits)."""
        torch = self.torch
        z = self.logits(X, masks, update_running)
        obj = torch.nn.functional.binary_cross_entropy_with_logits(z, Y, reduction="sum") / X.shape[0]
        params = self.parameters()
        grads = torch.autograd.grad(obj, params)
        with torch.no_grad():
            p = torch.sigmoid(z).clamp(_CLAMP_EPS, 1.0 - _CLAMP_EPS)
            loss = float((-(Y * torch.log(p) + (1.0 - Y) * torch.log(1.0 - p)).sum(dim=-1)).mean())
        return loss, grads

    def write_back(self) -> None:
        """Copy the trained values into the host ExpertMLP (in place, like the reference's Adam)."""
        net = self.net
        for dst, src in ((net.W, self.W), (net.b, self.b), (net.gamma, self.gamma), (net.beta, self.beta)):
            for i, t in enumerate(src):
                dst[i][...] = t.detach().cpu().numpy()
        net.run_mean = [m.cpu().numpy().copy() for m in self.run_mean]
        net.run_var = [v.cpu().numpy().copy() for v in self.run_var]
        net.invalidate_device()


def _device(device):
    import torch
    if device is not None:
        return torch.device(device)
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


def train(ds_train: TraceDataset, pop: PopularityMatrix, aff: AffinityMatrix, epochs: int = 20,
          batch_size: int = 256, learning_rate: float = 1e-3, seed: int = 0, hidden=None, dropout: float = 0.1,
          affinity_mode: str = "pool", device=None):
    """Mini-batch Adam on the BCE objective; deterministic given the seed
    (predictor.py:339-370).  Runs on the GPU (float64) when one is present."""
    import torch
    from .predictor import FULL_HIDDEN, ExpertMLP, TrainingDivergedError
    hidden = FULL_HIDDEN if hidden is None else hidden
    X, Y = build_training_set(ds_train, pop, aff, affinity_mode)
    meta = {"L": ds_train.L, "M": ds_train.M, "k": ds_train.k, "affinity_mode": affinity_mode}
    net = ExpertMLP(X.shape[1], ds_train.M, hidden=hidden, dropout=dropout, seed=seed, meta=meta)
    report = TrainReport(epochs=epochs, seed=seed, batch_size=batch_size, learning_rate=learning_rate,
                         n_samples=X.shape[0])
    if epochs == 0:
        return net, report
    dev = _device(device)
    dn = _DeviceNet(net, dev)
    Xd = torch.tensor(X, dtype=torch.float64, device=dev)
    Yd = torch.tensor(Y, dtype=torch.float64, device=dev)
    rng = np.random.default_rng(np.random.SeedSequence((seed, _TRAIN_TAG)))
    params = dn.parameters()
    m = [torch.zeros_like(p) for p in params]
    v = [torch.zeros_like(p) for p in params]
    b1, b2, eps = 0.9, 0.999, 1e-8
    t = 0
    n = X.shape[0]
    for epoch in range(epochs):
        perm = rng.permutation(n)
        total = 0.0
        for bi, start in enumerate(range(0, n, batch_size)):
            sel = perm[start:start + batch_size]
            masks = None
            if dropout > 0.0:
                # one mask per hidden layer, drawn in forward order (predictor.py:222-224)
                masks = [torch.tensor((rng.random((len(sel), h)) >= dropout) / (1.0 - dropout),
                                      dtype=torch.float64, device=dev) for h in hidden]
            idx = torch.as_tensor(sel, device=dev)
            loss, grads = dn.loss_and_grads(Xd[idx], Yd[idx], masks, update_running=True)
            if not np.isfinite(loss):
                raise TrainingDivergedError(learning_rate, epoch, bi)
            t += 1
            b1t, b2t = 1.0 - b1 ** t, 1.0 - b2 ** t
            with torch.no_grad():
                for p, g, mm, vv in zip(params, grads, m, v):
                    mm.mul_(b1)
                    mm.add_((1.0 - b1) * g)
                    vv.mul_(b2)
                    vv.add_((1.0 - b2) * g * g)
                    p.sub_(learning_rate * (mm / b1t) / (torch.sqrt(vv / b2t) + eps))
            total += loss * len(sel)
        report.epoch_losses.append(total / n)
    dn.write_back()
    return net, report


def gradient_check(net, X, Y, step: float = 1e-4, device=None) -> float:
    """Max relative error between the analytic gradient and central
    differences (predictor.py:373-408): dropout off, batch norm on the batch
    statistics of the fixed batch."""
    import torch
    dev = _device(device)
    dn = _DeviceNet(net, dev)
    Xd = torch.tensor(np.asarray(X, dtype=np.float64), device=dev)
    Yd = torch.tensor(np.asarray(Y, dtype=np.float64), device=dev)
    _, analytic = dn.loss_and_grads(Xd, Yd)

    def loss_at() -> float:
        with torch.no_grad():
            z = dn.logits(Xd)
            p = torch.sigmoid(z).clamp(_CLAMP_EPS, 1.0 - _CLAMP_EPS)
            return float((-(Yd * torch.log(p) + (1.0 - Yd) * torch.log(1.0 - p)).sum(dim=-1)).mean())

    worst = 0.0
    for p, g in zip(dn.parameters(), analytic):
        flat = p.detach().view(-1)
        gflat = g.reshape(-1)
        for j in range(flat.numel()):
            orig = float(flat[j])
            flat[j] = orig + step
            up = loss_at()
            flat[j] = orig - step
            down = loss_at()
            flat[j] = orig
            numeric = (up - down) / (2.0 * step)
            a = float(gflat[j])
            worst = max(worst, abs(a - numeric) / max(abs(a), abs(numeric), 1.0))
    return worst
