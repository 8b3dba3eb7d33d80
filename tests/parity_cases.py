"""Shared parity cases: program source + seeded inputs at oracle-friendly sizes."""
import numpy as np

from paper_2104_05372_b200 import programs as P


def _rng(seed=20211):
    return np.random.default_rng(seed)


def cases():
    r = _rng()
    out = []
    x4, y4 = P.matmul_inputs(4)
    out.append(("matmul_fwd_4", P.matmul_fwd(4), [x4, y4]))
    x16, y16 = P.matmul_inputs(16)
    out.append(("matmul_fwd_16", P.matmul_fwd(16), [x16, y16]))
    out.append(("matmul_grad_8", P.matmul_grad(8), list(P.matmul_inputs(8))))
    out.append(("matmul_grad_24", P.matmul_grad(24), list(P.matmul_inputs(24, seed=3))))
    pts, asg, cs = P.kmeans_inputs(200, 16, 8)
    out.append(("kmeans_cost_grad_200", P.kmeans_cost_grad(200, 16, 8), [pts, asg, cs]))
    out.append(("kmeans_grad_200", P.kmeans_grad(200, 16, 8), [pts, asg, cs]))
    pts, asg, cs = P.kmeans_inputs(1000, 4, 5, seed=7)
    out.append(("kmeans_cost_grad_d4", P.kmeans_cost_grad(1000, 4, 5), [pts, asg, cs]))
    pts, asg, cs = P.kmeans_inputs(300, 40, 6, seed=9)
    out.append(("kmeans_cost_grad_d40", P.kmeans_cost_grad(300, 40, 6), [pts, asg, cs]))
    pts, asg, cs = P.kmeans_inputs(64, 3, 4, seed=11)
    out.append(("kmeans_assign_64", P.kmeans_assign(64, 3, 4), [pts, cs]))
    out.append(("histogram_1000_7", P.histogram(1000, 7), [P.histogram_inputs(1000, 7)]))
    out.append(("histogram_5000_4096", P.histogram(5000, 4096), [P.histogram_inputs(5000, 4096)]))
    out.append(("histogram_zipf", P.histogram(4000, 64), [P.histogram_inputs(4000, 64, zipf=1.1)]))
    x, w1, w2 = P.mlp_inputs(8, 6, 5, 4)
    out.append(("mlp_grad_small", P.mlp_grad(8, 6, 5, 4), [x, [w1, w2]]))
    out.append(("sumsq_37", P.sumsq(37), [r.standard_normal(37)]))
    out.append(("dot_grad_9", P.dot_grad(9), [r.standard_normal(9), r.standard_normal(9)]))
    out.append(("revdot_grad_10", P.revdot_grad(10), [r.standard_normal(10)]))
    out.append(("scatter_slice_grad", P.scatter_slice_grad(50, 6),
                [r.standard_normal(50), r.integers(0, 6, 50)]))
    out.append(("cumulative_12", P.cumulative(12), [r.standard_normal(12)]))
    out.append(("pair_index_3x5", P.pair_index_sum(3, 5), [r.standard_normal((3, 5))]))
    out.append(("either_case_33", P.either_case(33), [r.standard_normal(33), r.standard_normal(33)]))
    out.append(("mandelbrot_8x6", P.mandelbrot(8, 6, 20),
                [np.linspace(-2.0, 0.5, 8), np.linspace(-1.0, 1.0, 6)]))
    # frontend_ext (exp/log): the evaluator extended the same way is the checker
    out.append(("softplus_grad_40", P.softplus_grad(40), [r.standard_normal(40)]))
    out.append(("leaky_relu_grad_30", P.leaky_relu_grad(30), [r.standard_normal(30), np.array([1.0, 0.1])]))
    v = r.standard_normal((6, 9))
    out.append(("logsumexp_grad_6x9", P.logsumexp_grad(6, 9), [v, v.max(1)]))
    for (n, d, K, seed) in ((50, 3, 2, 1), (300, 8, 5, 2), (120, 5, 3, 3)):  # d=5: f64 staged tables > 128 B
        from oracle import gmm as G
        a, mu, icf, x = G.gmm_inputs(n, d, K, seed=seed)
        dgi, tri, lm, lw = P.gmm_tables(d)
        mx, ma = P.gmm_stabilizers(a, mu, icf, x)
        out.append((f"gmm_program_{n}_{d}_{K}", P.gmm_program(n, d, K),
                    [x, mx, ma, dgi, tri, lm, lw, [a, mu, icf]]))
    # empty index sets (Fin 0): no iteration, zero cells (eval.cpp:295-308, 452-464)
    e0 = np.zeros(0, np.float32)
    out.append(("empty_sum", "main = \\x:((Fin 0)=>Float). sum x\n", [e0]))
    out.append(("empty_hist", "main = \\p:((Fin 0)=>(Fin 4)). yieldAccum \\h. for i. h!(p.i) += 1.0\n",
                [np.zeros(0, np.int32)]))
    out.append(("empty_map", "main = \\x:((Fin 0)=>Float). for i. (x.i) * 2.0\n", [e0]))
    out.append(("empty_rows", "main = \\x:((Fin 3)=>((Fin 0)=>Float)). for i. sum (x.i)\n", [e0]))
    out.append(("empty_grad", "main = \\x:((Fin 0)=>Float).\n  f = \\v:((Fin 0)=>Float). sum (for i. (v.i) * (v.i))\n"
                "  grad f x\n", [e0]))
    return out


def case(name):
    for c in cases():
        if c[0] == name:
            return c
    raise KeyError(name)
