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


def gmm_program(n: int, d: int, K: int, gamma: float = 1.0, m: int = 0) -> str:
    """config 3 as a dexlet program (needs the frontend_ext `exp`/`log`): the
    ADBench GMM objective and its gradient w.r.t. (alphas, (means, icf)).

    ADBench's `gmm_objective` (oracle/gmm.py) in the language's own terms:
    Q_k x = exp(icf_k[:d]) * x + L_k x (the log-diagonal slots selected by the
    index table `dgi`, r -> r) with the strictly lower triangle packed
    column by column, selected by the index table `tri` (row r, column c ->
    packed slot) under the 0/1 mask `lm` (r > c); `lw` masks the packed
    lower part of icf in the Wishart prior.  The log-sum-exps are stabilised
    by their maxima as ADBench does, passed as inputs `mx` (per point, over
    the components) and `ma` (over the alphas): in the language a `case` on
    `<` cannot be differentiated (the simplifier turns it into a data sum),
    and d/dtheta [m + log sum exp(beta - m)] does not depend on m, so the
    maxima are constants of the gradient -- a stop-gradient, as ADBench's own
    logsumexp.  `gmm_stabilizers` computes them (a forward-only program, or
    numpy).  Constant terms (the 2 pi term and the Wishart normaliser) are
    source literals."""
    import math
    T = d * (d + 1) // 2
    nn = d + m + 1
    lgd = 0.25 * d * (d - 1) * math.log(math.pi) + sum(math.lgamma(0.5 * nn + 0.5 * (1 - j)) for j in range(1, d + 1))
    C = nn * d * (math.log(gamma) - 0.5 * math.log(2)) - lgd
    c0 = -n * d * 0.5 * math.log(2 * math.pi) - K * C

    def lit(v):
        return repr(float(v))
    P = f"(((Fin {K})=>Float) & ({_mat(K, d)} & {_mat(K, T)}))"
    return (f"main = \\x:{_mat(n, d)}. \\mx:((Fin {n})=>Float). \\ma:((Fin 1)=>Float). "
            f"\\dgi:((Fin {d})=>(Fin {T})). \\tri:((Fin {d})=>((Fin {d})=>(Fin {T}))). \\lm:{_mat(d, d)}. \\lw:((Fin {T})=>Float). "
            f"\\th:{P}.\n"
            f"  f = \\p:{P}.\n"
            f"    al = fst p\n"
            f"    mi = snd p\n"
            f"    mu = fst mi\n"
            f"    ic = snd mi\n"
            f"    sqs = for k. sum (for r. ic.k.(dgi.r))\n"
            f"    lse = for i.\n"
            f"      s = sum (for k.\n"
            f"        sq = sum (for r.\n"
            f"          qr = (exp (ic.k.(dgi.r))) * ((x.i.r) - (mu.k.r)) + sum (for c. ((lm.r.c) * (ic.k.(tri.r.c))) * ((x.i.c) - (mu.k.c)))\n"
            f"          qr * qr)\n"
            f"        exp ((((al.k) + (sqs.k)) - 0.5 * sq) - (mx.i)))\n"
            f"      (mx.i) + log s\n"
            f"    sa = sum (for k. exp ((al.k) - (ma.(@0 : Fin 1))))\n"
            f"    wi = sum (for k.\n"
            f"      dg = sum (for r. (exp (ic.k.(dgi.r))) * (exp (ic.k.(dgi.r))))\n"
            f"      lo = sum (for t. ((lw.t) * (ic.k.t)) * (ic.k.t))\n"
            f"      {lit(0.5 * gamma * gamma)} * (dg + lo) - {lit(m)} * (sqs.k))\n"
            f"    (({lit(c0)} + sum lse) - {lit(n)} * ((ma.(@0 : Fin 1)) + log sa)) + wi\n"
            f"  pr = linearize f th\n"
            f"  (fst pr, transpose (snd pr) 1.0)\n")


def gmm_tables(d: int):
    """Index/mask inputs of gmm_program: dgi [d] (r -> slot r), tri [d][d] (packed slot of L[r][c]
    for r > c, ADBench column-major order; 0 elsewhere), lm [d][d] (1.0 for
    r > c) and lw [T] (1.0 on the packed lower part, slots >= d)."""
    T = d * (d + 1) // 2
    tri = np.zeros((d, d), dtype=np.int32)
    lm = np.zeros((d, d), dtype=np.float32)
    li = 0
    for c in range(d):
        for r in range(c + 1, d):
            tri[r, c] = d + li
            lm[r, c] = 1.0
            li += 1
    lw = np.zeros(T, dtype=np.float32)
    lw[d:] = 1.0
    dgi = np.arange(d, dtype=np.int32)
    return dgi, tri, lm, lw


def gmm_stabilizers(alphas, means, icf, x):
    """The log-sum-exp maxima of gmm_program (fp64 numpy, forward only):
    mx[i] = max_k beta[i][k], ma = max_k alphas[k]."""
    x = np.asarray(x, dtype=np.float64)
    alphas = np.asarray(alphas, dtype=np.float64)
    means = np.asarray(means, dtype=np.float64)
    icf = np.asarray(icf, dtype=np.float64)
    n, d = x.shape
    K = len(alphas)
    _, tri, lm, _ = gmm_tables(d)
    Q = np.zeros((K, d, d))
    r, c = np.nonzero(lm)
    Q[:, r, c] = icf[:, tri[r, c]]
    Q[:, np.arange(d), np.arange(d)] = np.exp(icf[:, :d])
    sum_qs = icf[:, :d].sum(1)
    beta = np.empty((n, K))
    for k in range(K):
        y = (x - means[k]) @ Q[k].T
        beta[:, k] = alphas[k] + sum_qs[k] - 0.5 * (y * y).sum(1)
    return beta.max(1), np.array([alphas.max()])


def softplus_grad(n: int) -> str:
    """frontend_ext: gradient of sum log(1 + exp v) (= the logistic sigmoid)."""
    return (f"main = \\xs:((Fin {n})=>Float).\n"
            f"  f = \\v:((Fin {n})=>Float). sum (for i. log (1.0 + exp (v.i)))\n"
            f"  grad f xs\n")


def logsumexp_grad(b: int, k: int) -> str:
    """frontend_ext: value and gradient of sum_i (m_i + log sum_j exp(v_ij - m_i))
    with the row maxima m as an input (a stop-gradient)."""
    return (f"main = \\v:{_mat(b, k)}. \\m:((Fin {b})=>Float).\n"
            f"  f = \\a:{_mat(b, k)}. sum (for i. (m.i) + log (sum (for j. exp ((a.i.j) - (m.i)))))\n"
            f"  pr = linearize f v\n"
            f"  (fst pr, transpose (snd pr) 1.0)\n")


def leaky_relu_grad(n: int) -> str:
    """frontend_ext `<` tangent: value and gradient of sum (c.(v < 0) * v)^2,
    c = (slope for v >= 0, slope for v < 0) indexed by the Bool itself."""
    return (f"main = \\xs:((Fin {n})=>Float). \\c:((Either Unit Unit)=>Float).\n"
            f"  f = \\v:((Fin {n})=>Float). sum (for i.\n"
            f"    y = (c.((v.i) < 0.0)) * (v.i)\n"
            f"    y * y)\n"
            f"  pr = linearize f xs\n"
            f"  (fst pr, transpose (snd pr) 1.0)\n")
