"""CPU: pin the oracle before trusting it.

* the reference evaluator harness (oracle/_ref) reproduces the known answers
  of the reference's own test suites (tests/kat_cases.py);
* it reproduces the committed golden vectors (tests/golden/parity_golden.json);
* the fp64 numpy restatements used for full-size checks agree with it;
* the reference's own acceptance gate passes (10/10) when /root/reference is
  present (built from its sources by oracle/Makefile).
"""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle
from oracle import restate
from paper_2104_05372_b200 import programs as P
from tests.kat_cases import KATS

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = "/root/reference/proj"

pytestmark = pytest.mark.skipif(not oracle.available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("name,src,entry,expected,cite", KATS, ids=[k[0] for k in KATS])
def test_reference_kats(name, src, entry, expected, cite):
    got = oracle.RefProgram(src, entry)()
    assert len(got) == len(expected), cite
    for g, e in zip(got, expected):
        np.testing.assert_allclose(g, e, rtol=0, atol=1e-12, err_msg=cite)


def test_histogram_kat_counts_work():
    """accumUpdates == n exactly (reference test_eval.cpp:82-92)."""
    prog = oracle.RefProgram(KATS[1][1], "hist")
    prog()
    assert prog.counters["accumUpdates"] == 5


def _golden():
    with open(os.path.join(HERE, "golden", "parity_golden.json")) as f:
        return json.load(f)


def _inputs(case):
    out = []
    for leaves, dts in zip(case["inputs"], case["input_dtypes"]):
        out.append([np.asarray(l, dtype=dt) for l, dt in zip(leaves, dts)])
    return out


@pytest.mark.parametrize("name", sorted(_golden().keys()))
def test_golden_reproduced(name):
    case = _golden()[name]
    got = oracle.RefProgram(case["source"])(*_inputs(case))
    assert len(got) == len(case["outputs"])
    for g, w in zip(got, case["outputs"]):
        np.testing.assert_array_equal(np.asarray(g, dtype=np.float64), np.asarray(w, dtype=np.float64))


def test_restate_kmeans_matches_reference():
    pts, asg, cs = P.kmeans_inputs(500, 16, 8, seed=3)
    cost, dC = oracle.RefProgram(P.kmeans_cost_grad(500, 16, 8))(pts, asg, cs)
    rc, rg = restate.kmeans_cost_grad(pts, asg, cs)
    assert oracle.rel_diff(np.array([rc]), cost) <= 1e-12
    assert oracle.rel_diff(rg.ravel(), dC) <= 1e-12


def test_restate_histogram_matches_reference():
    keys = P.histogram_inputs(3000, 97, seed=4)
    (h,) = oracle.RefProgram(P.histogram(3000, 97))(keys)
    np.testing.assert_array_equal(h, restate.histogram(keys, 97))


def test_restate_matmul_matches_reference():
    x, y = P.matmul_inputs(12, seed=5)
    loss, dx = oracle.RefProgram(P.matmul_grad(12))(x, y)
    rl, rdx = restate.matmul_grad(x, y)
    assert oracle.rel_diff(np.array([rl]), loss) <= 1e-12
    assert oracle.rel_diff(rdx.ravel(), dx) <= 1e-12
    (z,) = oracle.RefProgram(P.matmul_fwd(12))(x, y)
    assert oracle.rel_diff(restate.matmul_fwd(x, y).ravel(), z) <= 1e-12


def test_restate_mlp_matches_reference():
    x, w1, w2 = P.mlp_inputs(6, 5, 4, 3, seed=6)
    loss, dw1, dw2 = oracle.RefProgram(P.mlp_grad(6, 5, 4, 3))(x, [w1, w2])
    rl, r1, r2 = restate.mlp_grad(x, w1, w2)
    assert oracle.rel_diff(np.array([rl]), loss) <= 1e-12
    assert oracle.rel_diff(r1.ravel(), dw1) <= 1e-12
    assert oracle.rel_diff(r2.ravel(), dw2) <= 1e-12


def test_parallel_chunks_agree():
    """Reference chunked evaluation agrees with sequential (test_eval.cpp:157-177)."""
    pts, asg, cs = P.kmeans_inputs(300, 4, 5, seed=8)
    prog = oracle.RefProgram(P.kmeans_cost_grad(300, 4, 5))
    base = prog(pts, asg, cs, chunks=1)
    for c in (2, 3, 7):
        other = prog(pts, asg, cs, chunks=c)
        for a, b in zip(base, other):
            assert oracle.rel_diff(a, b) <= 1e-12


@pytest.mark.skipif(not os.path.isdir(REF), reason="needs /root/reference")
def test_reference_acceptance_gate():
    subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "_ref/acceptance", f"REF={REF}"],
                          stdout=subprocess.DEVNULL)
    out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "acceptance")], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS criterion") == 10, out.stdout


# ---- frontend_ext (exp/log, the `<` tangent) -------------------

@pytest.mark.parametrize("n,d,K,gamma,m", [(7, 3, 2, 1.0, 0), (20, 5, 4, 1.0, 0), (33, 4, 3, 0.7, 2),
                                           (64, 8, 6, 1.0, 0)])
def test_gmm_program_pins_adbench_restatement(n, d, K, gamma, m):
    """The ADBench GMM written in the language (programs.gmm_program, exp/log
    from frontend_ext) and differentiated by the reference's own
    linearize/transpose, evaluated by the reference evaluator (extended the
    same way), equals the fp64 ADBench restatement oracle/gmm.py: objective
    and every gradient entry to 1e-12 -- the GMM oracle is pinned by the
    reference's evaluator."""
    from oracle import gmm as G
    a, mu, icf, x = G.gmm_inputs(n, d, K, seed=n + d)
    dgi, tri, lm, lw = P.gmm_tables(d)
    mx, ma = P.gmm_stabilizers(a, mu, icf, x)
    got = oracle.RefProgram(P.gmm_program(n, d, K, gamma, m))(x, mx, ma, dgi, tri, lm, lw, [a, mu, icf])
    werr, wda, wdm, wdi = G.gmm_objective_grad(a, mu, icf, x, gamma, m)
    for g, w in zip(got, (np.array([werr]), wda, wdm.ravel(), wdi.ravel())):
        assert oracle.rel_diff(g, w) <= 1e-12


def test_gmm_program_gradient_is_stabilizer_free():
    """mx/ma are constants of the gradient (d/dt [m + log sum exp(b - m)]
    does not depend on m): shifting them changes nothing but rounding."""
    from oracle import gmm as G
    n, d, K = 15, 3, 3
    a, mu, icf, x = G.gmm_inputs(n, d, K, seed=4)
    tabs = P.gmm_tables(d)
    mx, ma = P.gmm_stabilizers(a, mu, icf, x)
    prog = oracle.RefProgram(P.gmm_program(n, d, K))
    base = prog(x, mx, ma, *tabs, [a, mu, icf])
    other = prog(x, mx + 3.0, ma - 2.0, *tabs, [a, mu, icf])
    for u, v in zip(base, other):
        assert oracle.rel_diff(u, v) <= 1e-12


def test_exp_log_finite_differences():
    """Central finite differences of an exp/log program against its
    linearize/transpose gradient, in the style of the reference's FD gate
    (tests/acceptance.cpp:262-284, tolerance 1e-4)."""
    n = 12
    r = np.random.default_rng(3)
    xs = r.standard_normal(n)
    f_src = (f"main = \\xs:((Fin {n})=>Float). sum (for i. log (1.0 + exp (xs.i)) + "
             f"exp ((xs.i) * 0.5) * log (2.0 + (xs.i) * (xs.i)))\n")
    f = oracle.RefProgram(f_src)
    g_src = (f"main = \\xs:((Fin {n})=>Float).\n  f = \\v:((Fin {n})=>Float). sum (for i. log (1.0 + exp (v.i)) + "
             f"exp ((v.i) * 0.5) * log (2.0 + (v.i) * (v.i)))\n  grad f xs\n")
    g = oracle.RefProgram(g_src)(xs)[0]
    h = 1e-6
    for i in range(n):
        e = np.zeros(n)
        e[i] = h
        fd = (f(xs + e)[0][0] - f(xs - e)[0][0]) / (2 * h)
        assert abs(fd - g[i]) <= 1e-4 * max(1.0, abs(g[i]))


def test_less_has_a_trivial_tangent():
    """`<` in a differentiated function linearizes (unit tangent) instead of
    raising E-tangent.  Its Bool result indexes a table over Either Unit Unit
    -- a piecewise function such as a (leaky) ReLU, c.(z < 0) * z.  (A case
    on it whose branches return floats is still rejected: the simplifier
    turns such a case into a data sum, which has no tangent.)"""
    src = ("main = \\xs:((Fin 3)=>Float). \\c:((Either Unit Unit)=>Float).\n"
           "  f = \\v:((Fin 3)=>Float). sum (for i. (c.((v.i) < 0.0)) * ((v.i) * (v.i)))\n"
           "  grad f xs\n")
    g = oracle.RefProgram(src)(np.array([1.0, -2.0, 0.5]), np.array([1.0, 0.25]))[0]
    np.testing.assert_allclose(g, [2.0, -1.0, 1.0], rtol=0, atol=1e-12)
