"""Popularity / affinity statistics — drop-in mirror of ``duoserve.stats``
(``/root/reference/pkg/src/duoserve/stats.py``).

These tables are the State Constructor's inputs: ``pop[l]`` (L, M) and
``aff[l]`` (L-1, M, M).  They are built offline from traces (stats.py:52-71:
integer counts, one normalisation; unobserved affinity rows stay all-zero)
and uploaded once to HBM for the device predictor.

``build_popularity`` / ``build_affinity`` here count with integer
bincount/outer-product arithmetic (exact, order independent), so their
values equal the reference's bit for bit; ``count_on_device`` offloads the
same integer histogram to the GPU kernel ``ds_route_histogram`` (online trace
collection from the device gate).
"""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .trace import TraceDataset


class StatsError(ValueError):
    """Statistics requested over an unusable dataset or malformed file."""


@dataclass(frozen=True, eq=False)
class PopularityMatrix:
    values: np.ndarray   # (L, M) float64; row l = counts[l] / (N k)
    counts: np.ndarray   # (L, M) int64
    n_episodes: int


@dataclass(frozen=True, eq=False)
class AffinityMatrix:
    values: np.ndarray   # (L-1, M, M) float64; observed rows sum to 1
    counts: np.ndarray   # (L-1, M, M) int64


def _onehot(ds: TraceDataset) -> np.ndarray:
    """(N, L, M) int64 selection indicator."""
    paths = ds.paths_array()                       # (N, L, k)
    N = paths.shape[0]
    X = np.zeros((N, ds.L, ds.M), dtype=np.int64)
    n_idx = np.arange(N)[:, None, None]
    l_idx = np.arange(ds.L)[None, :, None]
    X[n_idx, l_idx, paths] = 1
    return X


def normalize_popularity(counts: np.ndarray, n_episodes: int) -> PopularityMatrix:
    counts = np.asarray(counts, dtype=np.int64)
    return PopularityMatrix(values=counts / counts.sum(axis=1, keepdims=True), counts=counts,
                            n_episodes=int(n_episodes))


def normalize_affinity(counts: np.ndarray) -> AffinityMatrix:
    counts = np.asarray(counts, dtype=np.int64)
    tot = counts.sum(axis=2, keepdims=True)
    vals = np.zeros(counts.shape, dtype=np.float64)
    np.divide(counts, tot, out=vals, where=tot > 0)
    return AffinityMatrix(values=vals, counts=counts)


def build_popularity(ds: TraceDataset) -> PopularityMatrix:
    if not ds.traces:
        raise StatsError("cannot build popularity from an empty dataset")
    return normalize_popularity(_onehot(ds).sum(axis=0), len(ds.traces))


def build_affinity(ds: TraceDataset) -> AffinityMatrix:
    if not ds.traces:
        raise StatsError("cannot build affinity from an empty dataset")
    if ds.L < 2:
        raise StatsError(f"affinity needs at least 2 layers, model has {ds.L}")
    X = _onehot(ds)
    # integer co-occurrence counts c[l, i, j] = #traces with i at l and j at l+1
    counts = np.einsum("nli,nlj->lij", X[:, :-1, :], X[:, 1:, :])
    return normalize_affinity(counts)


def matrices_to_json(pop: PopularityMatrix, aff: AffinityMatrix) -> str:
    doc = {"schema_version": 1,
           "popularity": pop.values.tolist(),
           "affinity": aff.values.tolist(),
           "counts": {"popularity": pop.counts.tolist(), "affinity": aff.counts.tolist()},
           "n": pop.n_episodes}
    return json.dumps(doc, sort_keys=True) + "\n"


def save_matrices(pop: PopularityMatrix, aff: AffinityMatrix, path) -> None:
    Path(path).write_text(matrices_to_json(pop, aff), encoding="utf-8")


def load_matrices(path) -> tuple[PopularityMatrix, AffinityMatrix]:
    path = Path(path)
    try:
        doc = json.loads(path.read_text(encoding="utf-8"))
    except (OSError, json.JSONDecodeError) as e:
        raise StatsError(f"cannot load matrices from {path}: {e}") from e
    try:
        pop = PopularityMatrix(np.array(doc["popularity"], dtype=np.float64),
                               np.array(doc["counts"]["popularity"], dtype=np.int64), int(doc["n"]))
        aff = AffinityMatrix(np.array(doc["affinity"], dtype=np.float64),
                             np.array(doc["counts"]["affinity"], dtype=np.int64))
    except (KeyError, TypeError, ValueError) as e:
        raise StatsError(f"{path}: bad matrices document: {e}") from e
    return pop, aff


def export_csv(pop: PopularityMatrix, aff: AffinityMatrix, out_dir) -> list[Path]:
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    L, M = pop.values.shape
    files = []

    def write(path, header, rows):
        with path.open("w", newline="", encoding="utf-8") as f:
            w = csv.writer(f)
            w.writerow(header)
            w.writerows(rows)
        files.append(path)

    write(out_dir / "popularity.csv", ["layer"] + [f"expert_{i}" for i in range(M)],
          [[l] + [repr(float(v)) for v in pop.values[l]] for l in range(L)])
    for l in range(L - 1):
        write(out_dir / f"affinity_l{l}_l{l + 1}.csv", ["expert"] + [f"next_{j}" for j in range(M)],
              [[i] + [repr(float(v)) for v in aff.values[l, i]] for i in range(M)])
    return files


# --------------------------------------------------------------------------
# Online collection on the device ("data
# collection and inference serving ... simultaneously")

class OnlineRoutingStats:
    """int64 popularity / affinity counters in HBM, fed with gate selections
    [N, L, k] by the ``ds_route_histogram`` kernel while serving.  Integer
    counting is order independent, so ``matrices()`` equals
    ``build_popularity`` / ``build_affinity`` over the same selections bit for
    bit (stats.py:52-71)."""

    def __init__(self, L: int, M: int, k: int, device):
        import torch
        if L < 2:
            raise StatsError(f"affinity needs at least 2 layers, model has {L}")
        self.L, self.M, self.k = L, M, k
        self.pop_counts = torch.zeros((L, M), dtype=torch.int64, device=device)
        self.aff_counts = torch.zeros((L - 1, M, M), dtype=torch.int64, device=device)
        self.n_episodes = 0

    def add(self, paths) -> None:
        """paths: device int32 [N, L, k] of expert indices."""
        from . import ops
        if paths.dim() != 3 or tuple(paths.shape[1:]) != (self.L, self.k):
            raise StatsError(f"paths must be [N, {self.L}, {self.k}], got {tuple(paths.shape)}")
        if paths.shape[0] == 0:
            return
        ops.route_histogram(paths.contiguous(), self.M, self.pop_counts, self.aff_counts)
        self.n_episodes += int(paths.shape[0])

    def reset(self) -> None:
        self.pop_counts.zero_()
        self.aff_counts.zero_()
        self.n_episodes = 0

    def matrices(self) -> tuple[PopularityMatrix, AffinityMatrix]:
        if self.n_episodes == 0:
            raise StatsError("no routing collected yet")
        return (normalize_popularity(self.pop_counts.cpu().numpy(), self.n_episodes),
                normalize_affinity(self.aff_counts.cpu().numpy()))


def count_on_device(ds: TraceDataset, device="cuda") -> tuple[PopularityMatrix, AffinityMatrix]:
    """build_popularity + build_affinity with the counting on the GPU."""
    import torch
    if not ds.traces:
        raise StatsError("cannot build popularity from an empty dataset")
    st = OnlineRoutingStats(ds.L, ds.M, ds.k, device)
    st.add(torch.as_tensor(ds.paths_array().astype(np.int32), device=device))
    return st.matrices()
