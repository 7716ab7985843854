"""Where does the CFA c3 (4,096 x 256) gap to the oracle come from?
Solves the c3 workload with: the default CFA route (CTA-scan tau_delta),
the tau_delta lane pre-pass (selection batch forced large), GPU ABIA and
GPU JSIIA; compares each against oracle CFA / ABIA on the worst slots."""
import sys, os, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_06779_b200 as pd
from oracle import pyoracle as po

def gaps(a, b):
    return np.linalg.norm(a - b, axis=1) / np.maximum(1.0, np.linalg.norm(b, axis=1))

n, B = 256, 4096
cell = po.workload_seed(42, n, B)
links = po.workload_chains(cell, n, B)
q, qd, tau = po.workload_inputs(cell, n, B, 0)
ctx = pd.Context(0)
ctx.set_models(links, None)
res = {}
for name, algo, sel in [("cfa_cta", pd.FdAlgo.cfa, 0), ("cfa_prepass", pd.FdAlgo.cfa, 1 << 20),
                        ("abia", pd.FdAlgo.abia, 0), ("jsiia", pd.FdAlgo.jsiia, 0)]:
    ctx.set_selection_batch(sel)
    qdd, st, _, _ = ctx.solve(algo, q, qd, tau)
    res[name] = qdd
    print(name, ctx.last_variant(), (st == 0).all(), flush=True)
ctx.set_selection_batch(0)
g = gaps(res["cfa_cta"], res["abia"])
worst = np.argsort(g)[-24:]
sub = lambda a: a[worst]
ocfa, _ = po.batch_forward_dynamics("cfa", links[worst], [0, 0, -9.81], q[worst], qd[worst], tau[worst])
oabia, _ = po.batch_forward_dynamics("abia", links[worst], [0, 0, -9.81], q[worst], qd[worst], tau[worst])
ojs, _ = po.batch_forward_dynamics("jsiia", links[worst], [0, 0, -9.81], q[worst], qd[worst], tau[worst])
rows = {}
for k in ["cfa_cta", "cfa_prepass", "abia", "jsiia"]:
    rows[k + "_vs_oabia"] = gaps(sub(res[k]), oabia)
    rows[k + "_vs_ocfa"] = gaps(sub(res[k]), ocfa)
rows["ocfa_vs_oabia"] = gaps(ocfa, oabia)
rows["ojsiia_vs_oabia"] = gaps(ojs, oabia)
for k, v in rows.items():
    print(f"{k:24s} median {np.median(v):.2e} max {v.max():.2e}")
print("all-slot gpu abia vs gpu cfa_cta: max", g.max(), "gpu prepass vs cta:", gaps(res["cfa_prepass"], res["cfa_cta"]).max())
