import sys
import numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2104_05372_b200 as dx
from oracle import gmm as G
ctx = dx.Context(0)
for (n, k) in [(4999, 10), (4999, 2), (256, 2), (128, 1)]:
    a, mu, icf, x = G.gmm_inputs(n, 64, k, seed=100 + k)
    g = dx.GMM(ctx, 64, k, n)
    err, da, dm, di = g(a, mu, icf, x)
    w = G.gmm_objective_grad(a, mu, icf, x)
    wdi = w[3]
    diag = np.abs(di[:, :64] - wdi[:, :64]); off = np.abs(di[:, 64:] - wdi[:, 64:])
    print(n, k, "diag maxabs", diag.max(), "mag", np.abs(wdi[:, :64]).max(), "off maxabs", off.max(), "mag", np.abs(wdi[:, 64:]).max())
    print("   rel diag", (diag / (1 + np.abs(wdi[:, :64]))).max(), "rel off", (off / (1 + np.abs(wdi[:, 64:]))).max())
    print("   da", np.abs(da - w[1]).max(), np.abs(w[1]).max(), "dm", np.abs(dm - w[2]).max(), np.abs(w[2]).max())
    i = np.unravel_index(np.argmax(off), off.shape); print("   worst off", i, di[:, 64:][i], wdi[:, 64:][i])
