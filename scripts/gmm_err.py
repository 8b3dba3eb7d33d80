"""Dev tool: GMM gradient error at the BASELINE size (n = 1M, K = 200) against
the committed fp64 golden (tests/golden/gmm_1m_k200.npz): elementwise
(rtMaxRelDiff) and normwise per block, and where the worst entries are."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2104_05372_b200 as dx
from paper_2104_05372_b200 import programs as P

z = np.load(os.path.join(ROOT, "tests", "golden", "gmm_1m_k200.npz"))
n, d, k = int(z["n"]), int(z["d"]), int(z["k"])
a, mu, icf, x = P.gmm_inputs(n, d, k, seed=int(z["seed"]))
assert float(x.astype(np.float64).sum()) == float(z["x_checksum"])
g = dx.GMM(dx.Context(0), d, k, n)
err, da, dm, di = g(a, mu, icf, x)
print("objective rel %.2e (got %.10g want %.10g)" % (abs(err - z["err"]) / (1 + abs(z["err"])), err, z["err"]))
for nm, got, want in (("d_alphas", da, z["d_alphas"]), ("d_means", dm, z["d_means"]), ("d_icf", di, z["d_icf"])):
    got = np.asarray(got, np.float64).ravel()
    want = np.asarray(want, np.float64).ravel()
    r = np.abs(got - want) / (1 + np.maximum(np.abs(got), np.abs(want)))
    j = int(np.argmax(r))
    cols = want.size // k
    print(f"{nm}: rel {r.max():.2e} norm {np.abs(got - want).max() / max(1, np.abs(want).max()):.2e}; worst at "
          f"component {j // cols} entry {j % cols}: got {got[j]:.6g} want {want[j]:.6g}; "
          f"abs err max {np.abs(got - want).max():.3g}, median |want| {np.median(np.abs(want)):.3g}, "
          f"entries > 1e-4: {(r > 1e-4).sum()} of {r.size}", flush=True)
