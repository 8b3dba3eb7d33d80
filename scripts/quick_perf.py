"""Dev tool: time one program on the device (CUDA events) at a given size."""
import sys, time
import numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2104_05372_b200 as dx
from paper_2104_05372_b200 import programs as P

def timeit(prog, iters=20, warm=3):
    for _ in range(warm): prog.run()
    ctx = prog.ctx; ctx.sync()
    e0 = ctx.event()
    for _ in range(iters): prog.run()
    e1 = ctx.event()
    return ctx.elapsed_ms(e0, e1) / iters

ctx = dx.Context(0)
which = sys.argv[1] if len(sys.argv) > 1 else "kmeans"
if which == "kmeans":
    n, d, k = (int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000), 16, 64
    pts, asg, cs = P.kmeans_inputs(n, d, k)
    t = time.time(); prog = dx.Program(P.kmeans_cost_grad(n, d, k), ctx=ctx); print("compile", time.time()-t)
    print(prog.plan.split("--- optimized")[0])
    out = prog(pts, asg, cs)
    ms = timeit(prog)
    byts = n*d*4 + n*4 + 2*k*d*4
    print(f"kmeans cost+grad: {ms*1e3:.1f} us/eval  {byts/ms/1e6:.1f} GB/s  cost={out[0][0]:.6g}")
    e = pts.astype(np.float64) - cs.astype(np.float64)[asg]
    cost = (e*e).sum(); g = np.zeros((k, d)); np.add.at(g, asg, -2*e)
    print("cost rel", abs(out[0][0]-cost)/(1+abs(cost)), "grad rel", np.max(np.abs(out[1]-g.ravel())/(1+np.abs(g.ravel()))))
elif which in ("hist", "histz"):
    n, k = 1 << 28, 4096
    keys = P.histogram_inputs(n, k, zipf=1.1 if which == "histz" else 0.0)
    prog = dx.Program(P.histogram(n, k), ctx=ctx)
    out = prog(keys)
    ms = timeit(prog, 10)
    print(f"hist: {ms*1e3:.1f} us  {(n*4+k*4)/ms/1e6:.1f} GB/s  exact={np.array_equal(out[0], np.bincount(keys, minlength=k))}")
