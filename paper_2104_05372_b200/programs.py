"""Benchmark and parity programs, written in the reference's surface language.

Each builder returns source text defining ``main = \\x1:T1. ... body`` (inputs
are bound as runtime values, never literals -- SURVEY.md §8c harness caveat).
They are the programs of SURVEY.md appendix A, parameterized by size, plus the
reference's own data-corpus fixtures re-expressed with inputs.

Input generators are seeded numpy (``np.random.default_rng``); leaves follow the
C-ABI flattening (include/dexlet_cuda.h): tables row-major by ordinal, index
members as ordinals.
"""
from __future__ import annotations

import numpy as np


def _mat(n, m):
    return f"((Fin {n})=>((Fin {m})=>Float))"


def matmul_fwd(n: int) -> str:
    """config 1 forward: `for i k. sum for j. x.i.j * y.j.k`."""
    return (f"main = \\x:{_mat(n, n)}. \\y:{_mat(n, n)}. "
            f"for i k. sum (for j. (x.i.j) * (y.j.k))\n")


def contraction(m: int, n: int, k: int, x_kmajor: bool = True, y_kmajor: bool = False) -> str:
    """Rectangular `for i l. sum for j. x.(i,j) * y.(j,l)` with either storage
    order of each operand (x_kmajor: x is (Fin m)=>(Fin k); y_kmajor: y is
    (Fin n)=>(Fin k)).  The tcgen05 GEMM path's parity cases."""
    xt = _mat(m, k) if x_kmajor else _mat(k, m)
    yt = _mat(n, k) if y_kmajor else _mat(k, n)
    xr = "x.i.j" if x_kmajor else "x.j.i"
    yr = "y.l.j" if y_kmajor else "y.j.l"
    return (f"main = \\x:{xt}. \\y:{yt}. "
            f"for i l. sum (for j. ({xr}) * ({yr}))\n")


def contraction_inputs(m: int, n: int, k: int, x_kmajor: bool = True, y_kmajor: bool = False, seed: int = 20211):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (m, k) if x_kmajor else (k, m)).astype(np.float32)
    y = rng.uniform(-1, 1, (n, k) if y_kmajor else (k, n)).astype(np.float32)
    return x, y


def matmul_grad(n: int) -> str:
    """config 1: value and gradient of sum(x . y) w.r.t. x (linearize + transpose)."""
    return (f"main = \\x:{_mat(n, n)}. \\y:{_mat(n, n)}.\n"
            f"  f = \\a:{_mat(n, n)}. sum (for i. sum (for k. sum (for j. (a.i.j) * (y.j.k))))\n"
            f"  pr = linearize f x\n"
            f"  (fst pr, transpose (snd pr) 1.0)\n")


def kmeans_cost_grad(n: int, d: int, k: int) -> str:
    """config 2: k-means cost and its gradient w.r.t. the centroids at fixed
    assignments (SURVEY.md appendix A program 2; value_and_grad form)."""
    return (f"main = \\pts:{_mat(n, d)}. \\asg:((Fin {n})=>(Fin {k})). \\cs:{_mat(k, d)}.\n"
            f"  f = \\c:{_mat(k, d)}. sum (for i. sum (for j.\n"
            f"    e = (pts.i.j) - (c.(asg.i).j)\n"
            f"    e * e))\n"
            f"  pr = linearize f cs\n"
            f"  (fst pr, transpose (snd pr) 1.0)\n")


def kmeans_grad(n: int, d: int, k: int) -> str:
    return (f"main = \\pts:{_mat(n, d)}. \\asg:((Fin {n})=>(Fin {k})). \\cs:{_mat(k, d)}.\n"
            f"  f = \\c:{_mat(k, d)}. sum (for i. sum (for j.\n"
            f"    e = (pts.i.j) - (c.(asg.i).j)\n"
            f"    e * e))\n"
            f"  grad f cs\n")


def kmeans_assign(n: int, d: int, k: int) -> str:
    """k-means assignment pass (primal only; `<` has no tangent): strict `<`,
    first minimum wins (SURVEY.md appendix A program 2')."""
    return (f"main = \\pts:{_mat(n, d)}. \\cs:{_mat(k, d)}.\n"
            f"  for i.\n"
            f"    ds = for c. sum (for j.\n"
            f"      e = (pts.i.j) - (cs.c.j)\n"
            f"      e * e)\n"
            f"    best = yieldState (1.0e30, (@0 : Fin {k})) \\b.\n"
            f"      for c.\n"
            f"        cur = get b\n"
            f"        b := (if (ds.c) < (fst cur) then (ds.c, c) else cur)\n"
            f"      ()\n"
            f"    snd best\n")


def histogram(n: int, k: int) -> str:
    """config 4: `h!(p.i) += 1.0` into k bins (Float counts, exact)."""
    return (f"main = \\p:((Fin {n})=>(Fin {k})). yieldAccum \\h.\n"
            f"  for i. h!(p.i) += 1.0\n")


def mlp_grad(b: int, i: int, h: int, o: int) -> str:
    """config 5: 2-layer MLP, square activation, loss and grads over (W1 & W2)."""
    w = f"({_mat(i, h)} & {_mat(h, o)})"
    return (f"main = \\x:{_mat(b, i)}. \\w:{w}.\n"
            f"  loss = \\p:{w}.\n"
            f"    w1 = fst p\n"
            f"    w2 = snd p\n"
            f"    hh = for bb h2.\n"
            f"      z = sum (for ii. (x.bb.ii) * (w1.ii.h2))\n"
            f"      z * z\n"
            f"    y = for bb oo. sum (for h2. (hh.bb.h2) * (w2.h2.oo))\n"
            f"    sum (for bb. sum (for oo. (y.bb.oo) * (y.bb.oo)))\n"
            f"  pr = linearize loss w\n"
            f"  (fst pr, transpose (snd pr) 1.0)\n")


def sumsq(n: int) -> str:
    return f"main = \\xs:((Fin {n})=>Float). sum (for i. (xs.i) * (xs.i))\n"


def dot_grad(n: int) -> str:
    return (f"main = \\xs:((Fin {n})=>Float). \\c:((Fin {n})=>Float).\n"
            f"  f = \\v:((Fin {n})=>Float). sum (for i. ((v.i) * (c.i)) + (v.i))\n"
            f"  grad f xs\n")


def revdot_grad(n: int) -> str:
    return (f"main = \\xs:((Fin {n})=>Float).\n"
            f"  f = \\v:((Fin {n})=>Float). sum (for i. (v.i) * (v.(reverse i)))\n"
            f"  grad f xs\n")


def scatter_slice_grad(n: int, k: int) -> str:
    """acceptance.cpp:289-321 'scatter-slice' case, sized."""
    return (f"main = \\xs:((Fin {n})=>Float). \\idx:((Fin {n})=>(Fin {k})).\n"
            f"  f = \\v:((Fin {n})=>Float). sum (yieldAccum \\h.\n"
            f"    for i. h!(idx.i) += (v.i) * (v.i))\n"
            f"  grad f xs\n")


def cumulative(n: int) -> str:
    """State: sequential recurrence (blocked from chunking, eval.cpp:298)."""
    return (f"main = \\xs:((Fin {n})=>Float). yieldState 0.0 \\s.\n"
            f"  for i. s := ((get s) * 0.5) + (xs.i)\n"
            f"  ()\n")


def pair_index_sum(n: int, m: int) -> str:
    return (f"main = \\x:({_mat(n, m)}). for p:((Fin {n}) & (Fin {m})).\n"
            f"  i = fst p\n"
            f"  j = snd p\n"
            f"  (x.i.j) * (itof (ord p))\n")


def either_case(n: int) -> str:
    return (f"main = \\xs:((Fin {n})=>Float). \\ys:((Fin {n})=>Float). for i.\n"
            f"  if (xs.i) < (ys.i) then (ys.i) - (xs.i) else (xs.i) * 2.0\n")


def mandelbrot(w: int, h: int, iters: int) -> str:
    """Escape-time per pixel with State (tests/fixtures/mandelbrot.dexlet shape)."""
    return (f"main = \\cr:((Fin {w})=>Float). \\ci:((Fin {h})=>Float).\n"
            f"  for y x.\n"
            f"    res = yieldState ((0.0, 0.0), 0.0) \\s.\n"
            f"      for k:(Fin {iters}).\n"
            f"        cur = get s\n"
            f"        z = fst cur\n"
            f"        zr = fst z\n"
            f"        zi = snd z\n"
            f"        mag = (zr * zr) + (zi * zi)\n"
            f"        s := (if mag < 4.0 then ((((zr * zr) - (zi * zi)) + (cr.x), ((2.0 * zr) * zi) + (ci.y)), (snd cur) + 1.0) else cur)\n"
            f"      ()\n"
            f"    snd res\n")


# ---- seeded inputs ------------------------------------------------------------

def kmeans_inputs(n: int, d: int, k: int, seed: int = 20211):
    rng = np.random.default_rng(seed)
    pts = rng.standard_normal((n, d)).astype(np.float32)
    cs = pts[rng.choice(n, size=k, replace=False)].copy() if n >= k else rng.standard_normal((k, d)).astype(np.float32)
    # assignments: argmin with strict `<`, first minimum (computed in f64)
    asg = np.empty(n, dtype=np.int32)
    bs = 1 << 16
    c64 = cs.astype(np.float64)
    for s in range(0, n, bs):
        p = pts[s:s + bs].astype(np.float64)
        dd = ((p[:, None, :] - c64[None, :, :]) ** 2).sum(-1)
        asg[s:s + bs] = np.argmin(dd, axis=1)
    return pts, asg, cs


def histogram_inputs(n: int, k: int, seed: int = 20211, zipf: float = 0.0):
    rng = np.random.default_rng(seed)
    if zipf > 0:
        keys = (rng.zipf(zipf, size=n) - 1) % k
        return keys.astype(np.int32)
    return rng.integers(0, k, size=n, dtype=np.int32)


def matmul_inputs(n: int, seed: int = 20211):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, (n, n)).astype(np.float32),
            rng.uniform(-1, 1, (n, n)).astype(np.float32))


def mlp_inputs(b: int, i: int, h: int, o: int, seed: int = 20211):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((b, i)).astype(np.float32)
    w1 = (rng.standard_normal((i, h)) / np.sqrt(i)).astype(np.float32)
    w2 = (rng.standard_normal((h, o)) / np.sqrt(h)).astype(np.float32)
    return x, w1, w2


def gmm_inputs(n: int, d: int, K: int, seed: int = 20211):
    """Synthetic inputs of SURVEY.md §8(d) config 3 (ADBench form): x, means ~
    N(0,1), icf ~ U(-0.1, 0.1), alphas ~ N(0,1), fp32."""
    rng = np.random.default_rng(seed)
    alphas = rng.standard_normal(K).astype(np.float32)
    means = rng.standard_normal((K, d)).astype(np.float32)
    icf = rng.uniform(-0.1, 0.1, (K, d * (d + 1) // 2)).astype(np.float32)
    x = rng.standard_normal((n, d)).astype(np.float32)
    return alphas, means, icf, x
