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
