"""Dev tool: elementwise / normwise gradient error of the GMM kernels on the
test cases (run once per env setting, e.g. DEXLET_GMM_BWD_PAIR=1)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05372_b200 as dx
from oracle import gmm as G

def rel(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / (1.0 + np.maximum(np.abs(a), np.abs(b)))))

def normrel(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))

ctx = dx.Context(0)
for n, k in [(1000, 3), (4999, 10), (8192, 17), (20000, 24), (100000, 64)]:
    a, mu, icf, x = G.gmm_inputs(n, 64, k, seed=100 + k)
    g = dx.GMM(ctx, 64, k, n)
    r = g(a, mu, icf, x)
    w = G.gmm_objective_grad(a, mu, icf, x)
    print(("pair" if os.environ.get("DEXLET_GMM_BWD_PAIR") else "quad"), n, k, "obj %.1e" % rel(r[0], w[0]),
          " ".join("%s %.2e/%.2e" % (nm, rel(u, v), normrel(u, v)) for nm, u, v in zip(("da", "dm", "di"), r[1:], w[1:])),
          "max|di| %.1f" % np.max(np.abs(w[3])), flush=True)
