"""Diagnostic: same-algorithm and cross-algorithm gaps for long chains, to tell
conditioning from kernel error (GPU vs CPU oracle, CFA vs ABIA vs JSIIA)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_06779_b200 as pd  # noqa: E402
from oracle import pyoracle as po  # noqa: E402


def gap(a, b):
    return np.linalg.norm(a - b) / max(1.0, np.linalg.norm(b))


ctx = pd.Context(0)
for n, B, lo in ((700, 2, 1.0), (700, 2, 3.0), (1050, 1, 1.0), (300, 3, 1.0)):
    links = np.stack([po.random_chain(n, 5100 + 7 * n + c)[0] for c in range(B)])
    rng = np.random.default_rng(n + B)
    q, qd, tau = (rng.uniform(-lo, lo, (B, n)) for _ in range(3))
    ctx.set_models(links, None)
    g = {a: ctx.solve(getattr(pd.FdAlgo, a), q, qd, tau)[0] for a in ("abia", "jsiia", "cfa")}
    o = {a: po.batch_forward_dynamics(a, links, [0, 0, -9.81], q, qd, tau)[0] for a in ("abia", "jsiia", "cfa")}
    for b in range(B):
        print(f"n={n} |q|<={lo} b={b}: gpu-oracle abia {gap(g['abia'][b], o['abia'][b]):.1e} "
              f"jsiia {gap(g['jsiia'][b], o['jsiia'][b]):.1e} cfa {gap(g['cfa'][b], o['cfa'][b]):.1e} | "
              f"oracle cfa-abia {gap(o['cfa'][b], o['abia'][b]):.1e} jsiia-abia {gap(o['jsiia'][b], o['abia'][b]):.1e} | "
              f"gpu cfa-abia {gap(g['cfa'][b], o['abia'][b]):.1e} gpu jsiia-abia {gap(g['jsiia'][b], o['abia'][b]):.1e}")
