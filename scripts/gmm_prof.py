"""Dev tool: one GMM fwd+grad at a given size (for ncu)."""
import sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2104_05372_b200 as dx
from oracle import gmm as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 200
ctx = dx.Context(0)
a, mu, icf, x = G.gmm_inputs(n, 64, k)
g = dx.GMM(ctx, 64, k, n)
g.set_params(a, mu, icf); g.set_points(x)
for _ in range(2):
    g.run(); g.get()
print("ok")
