"""Brute-force popularity/affinity recount (oracle).

Restates stats.py:74-108 (stats_oracle): naive loops over traces, integer
counts, one normalisation; unobserved affinity rows stay zero (stats.py:69-70).
"""

from __future__ import annotations

import numpy as np


def recount(paths, L: int, M: int):
    """paths: iterable of L-tuples of selections.  Returns (pop_values,
    pop_counts, aff_values, aff_counts) as numpy arrays."""
    pc = [[0] * M for _ in range(L)]
    ac = [[[0] * M for _ in range(M)] for _ in range(L - 1)]
    n = 0
    for path in paths:
        n += 1
        for l in range(L):
            for i in range(M):
                if i in path[l]:
                    pc[l][i] += 1
        for l in range(L - 1):
            for i in range(M):
                for j in range(M):
                    if i in path[l] and j in path[l + 1]:
                        ac[l][i][j] += 1
    pv = [[pc[l][i] / sum(pc[l]) for i in range(M)] for l in range(L)]
    av = [[[0.0] * M for _ in range(M)] for _ in range(L - 1)]
    for l in range(L - 1):
        for i in range(M):
            tot = sum(ac[l][i])
            if tot > 0:
                for j in range(M):
                    av[l][i][j] = ac[l][i][j] / tot
    return np.array(pv), np.array(pc, dtype=np.int64), np.array(av), np.array(ac, dtype=np.int64)
