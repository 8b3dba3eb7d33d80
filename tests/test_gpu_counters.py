"""GPU: the reference acceptance gate's work criteria on the device path.

EvalCounters (eval.hpp:60-65) come from count mode (DXL_F_COUNT,
dxl_program_counters; evalExprDevice fills the same struct): kernels count the
+ - * / they execute and every `+=`.  The programs and thresholds are those of
/root/reference/proj/tests/acceptance.cpp:459-569 (criteria 6 and 7), run as
whole-file programs as the gate's runSimpl does."""
import numpy as np
import pytest

import paper_2104_05372_b200 as dx

pytestmark = pytest.mark.gpu
K_WORK = 4  # acceptance.cpp kWorkFactor


def _vec(n, mod):
    return [float((i % mod) + 1) for i in range(n)]


def _lit(v):
    return "[" + ", ".join(repr(x) for x in v) + "]"


def _count(ctx, src):
    p = dx.Program(src, entry=None, ctx=ctx, flags=dx.DXL_F_COUNT)
    out = p()
    return p.counters(), out


def test_criterion7_histogram_does_exactly_n_updates(ctx):
    """acceptance.cpp:540-569: exactly n accumulator updates, exact counts."""
    for n, k in ((5, 3), (64, 7), (100, 10)):
        pts = ", ".join(f"@{i % k}" for i in range(n))
        src = f"points : (Fin {n}) => (Fin {k}) = [{pts}]\nhist = yieldAccum \\h.\n  for i. h!(points.i) += 1.0\nhist\n"
        c, out = _count(ctx, src)
        assert c["accumUpdates"] == n, (n, k, c)
        want = [n // k + (1 if b < n % k else 0) for b in range(k)]
        np.testing.assert_array_equal(out[0], want)


def test_criterion6_tangent_within_4x(ctx):
    """acceptance.cpp:466-480: the tangent of sumsq costs <= 4x the primal."""
    n = 64
    fn = "f = \\xs:((Fin 64)=>Float). sum (for i. (xs.i) * (xs.i))\n"
    primal, _ = _count(ctx, fn + "y = f " + _lit(_vec(n, 7)) + "\ny\n")
    tangent, _ = _count(ctx, fn + "p = linearize f " + _lit(_vec(n, 7)) + "\ndf = snd p\ndy = df " +
                        _lit(_vec(n, 3)) + "\ndy\n")
    assert primal["arithmeticOps"] > 0 and primal["accumUpdates"] > 0, primal
    assert tangent["arithmeticOps"] <= K_WORK * primal["arithmeticOps"], (tangent, primal)
    assert tangent["accumUpdates"] <= K_WORK * primal["accumUpdates"], (tangent, primal)


def test_criterion6_transpose_within_4x(ctx):
    """acceptance.cpp:481-494: transposing a linear scale costs <= 4x."""
    n = 64
    fn = "c = " + _lit(_vec(n, 5)) + "\nf = \\xs:((Fin 64)=>Float). for i : Fin 64. (xs.i) * (c.i)\n"
    primal, _ = _count(ctx, fn + "y = f " + _lit(_vec(n, 7)) + "\ny\n")
    trans, _ = _count(ctx, fn + "t = transpose f " + _lit(_vec(n, 3)) + "\nt\n")
    budget = K_WORK * (primal["arithmeticOps"] + primal["accumUpdates"])
    assert trans["arithmeticOps"] <= budget and trans["accumUpdates"] <= budget, (trans, primal)


def test_criterion6_scatter_transpose_linear_in_n(ctx):
    """acceptance.cpp:495-525: the transposed indexed scatter does n updates
    plus a constant (<= 4) independent of the target size k."""
    overhead = None
    for n in (16, 64):
        for k in (4, 8):
            idx = ", ".join(f"@{(i * 3) % k}" for i in range(n))
            fn = (f"idx : (Fin {n}) => (Fin {k}) = [{idx}]\nf = \\x:((Fin {n})=>Float). yieldAccum \\h.\n"
                  f"  for i. h!(idx.i) += x.i\n")
            c, _ = _count(ctx, fn + "t = transpose f " + _lit(_vec(k, 3)) + "\nt\n")
            extra = c["accumUpdates"] - n
            if overhead is None:
                overhead = extra
            assert extra == overhead and 0 <= extra <= 4, (n, k, c)


def test_counters_match_reference_on_kmeans(ctx):
    """Same units as the reference: the k-means cost program's counts equal
    the reference evaluator's up to the work the lowering removes (never more)."""
    import oracle
    from paper_2104_05372_b200 import programs as P
    n, d, k = 300, 4, 5
    pts, asg, cs = P.kmeans_inputs(n, d, k)
    src = P.kmeans_cost_grad(n, d, k)
    p = dx.Program(src, ctx=ctx, flags=dx.DXL_F_COUNT)
    got = p(pts, asg, cs)
    c = p.counters()
    want = oracle.RefProgram(src)(pts, asg, cs)
    for g, w in zip(got, want):
        assert oracle.rel_diff(g, w) <= 1e-4
    assert c["arithmeticOps"] >= 3 * n * d  # e, e*e, and the transposed 2e per element
    assert c["accumUpdates"] >= n * d      # one dC update per element
