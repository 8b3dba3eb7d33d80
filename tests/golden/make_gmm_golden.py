"""Generates tests/golden/gmm_1m_k200.npz: the fp64 ADBench restatement
(oracle/gmm.py) evaluated at the BASELINE GMM size (configs[2]: n = 1M, d = 64,
K = 200, inputs P.gmm_inputs(seed=20211)).  The oracle takes minutes at this
size, so the GPU test compares against these committed values instead of
re-running it.  Gradients are stored as float32 (6e-8 relative rounding, far
below the tolerances they are checked at); the objective as float64.

    python tests/golden/make_gmm_golden.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import numpy as np

from oracle import gmm as G
from paper_2104_05372_b200 import programs as P

N, D, K, SEED = 1_000_000, 64, 200, 20211

if __name__ == "__main__":
    a, mu, icf, x = P.gmm_inputs(N, D, K, seed=SEED)
    err, da, dm, di = G.gmm_objective_grad(a, mu, icf, x)
    np.savez_compressed(os.path.join(HERE, "gmm_1m_k200.npz"), n=N, d=D, k=K, seed=SEED, err=np.float64(err),
                        d_alphas=da.astype(np.float32), d_means=dm.astype(np.float32), d_icf=di.astype(np.float32),
                        x_checksum=np.float64(x.astype(np.float64).sum()))
    print("err", err)
