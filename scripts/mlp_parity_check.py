"""Dev tool: MLP parity (rtMaxRelDiff) against the fp64 restatement at bench and test shapes."""
import sys, os, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import oracle
import paper_2104_05372_b200 as dx
from paper_2104_05372_b200 import programs as P
from oracle import restate
ctx = dx.Context(0)
for (b, i, h, o) in [(8192, 1024, 1024, 1024), (3200, 64, 1024, 64), (2048, 256, 256, 256)]:
    x, w1, w2 = P.mlp_inputs(b, i, h, o)
    prog = dx.Program(P.mlp_grad(b, i, h, o), ctx=ctx)
    loss, d1, d2 = prog(x, [w1, w2])
    t = time.time(); rl, r1, r2 = restate.mlp_grad(x, w1, w2)
    print((b, i, h, o), "n256" if "n256" in prog.plan else "n128", "loss %.2e d1 %.2e d2 %.2e" % (
        oracle.rel_diff(loss, np.array([rl])), oracle.rel_diff(d1, r1.ravel()), oracle.rel_diff(d2, r2.ravel())), flush=True)
