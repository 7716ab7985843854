"""Seeded synthetic workloads of the reference benchmark (product side).

Thin wrappers over the C-ABI's pd_workload_* (csrc/workload.cpp), which
restate bench.cpp:42-70,350-383 and model.cpp:157-185 bit for bit.
"""
from __future__ import annotations

import numpy as np

from . import _capi


def workload_seed(seed: int, n_links: int, n_groups: int) -> int:
    return int(_capi.load().pd_workload_seed(seed, n_links, n_groups))


def workload_chains(cell_seed: int, n_links: int, count: int, g0: int = 0) -> np.ndarray:
    """Chains [g0, g0 + count) of the cell as (count, n_links, 31) LinkSpec records."""
    out = np.empty((count, n_links, _capi.LINK_FIELDS))
    _capi.load().pd_workload_chains(cell_seed, n_links, g0, count, _capi.dptr(out))
    return out


def workload_inputs(cell_seed: int, n_links: int, n_groups: int, repeat: int):
    """(q, qdot, drive), each (n_groups, n_links), uniform in [-1, 1]."""
    q = np.empty((n_groups, n_links))
    qd = np.empty_like(q)
    dr = np.empty_like(q)
    _capi.load().pd_workload_inputs(cell_seed, n_links, n_groups, repeat, _capi.dptr(q), _capi.dptr(qd),
                                    _capi.dptr(dr))
    return q, qd, dr


def random_chain(n_links: int, seed: int) -> np.ndarray:
    out = np.empty((n_links, _capi.LINK_FIELDS))
    _capi.load().pd_random_chain(n_links, seed, _capi.dptr(out))
    return out
