"""Dev tool: GMM parity at a small size + timing at BASELINE size on cuda:0."""
import sys, time
import numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2104_05372_b200 as dx
from oracle import gmm as G

def rel(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / (1.0 + np.maximum(np.abs(a), np.abs(b)))))

ctx = dx.Context(0)
for n, k in [(1000, 3), (4999, 10)]:
    a, mu, icf, x = G.gmm_inputs(n, 64, k, seed=100 + k)
    g = dx.GMM(ctx, 64, k, n)
    t = time.time()
    err, da, dm, di = g(a, mu, icf, x)
    w = G.gmm_objective_grad(a, mu, icf, x)
    print(n, k, "err", err, w[0], "rel", rel(err, w[0]), "da", rel(da, w[1]), "dm", rel(dm, w[2]), "di", rel(di, w[3]), flush=True)
if len(sys.argv) > 1:
    n, k = 1_000_000, 200
    a, mu, icf, x = G.gmm_inputs(n, 64, k)
    g = dx.GMM(ctx, 64, k, n)
    g.set_params(a, mu, icf); g.set_points(x)
    g.enable_timing(True)
    for it in range(4):
        g.run(); r = g.get()
    print("full err", r[0])
    print(g.kernel_times())
    e0 = ctx.event()
    for it in range(5): g.run()
    e1 = ctx.event()
    print("ms/eval", ctx.elapsed_ms(e0, e1) / 5)
