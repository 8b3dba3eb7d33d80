"""GPU: known answers of the reference test suites, golden vectors, and
full-size (BASELINE.json) parity through size-independent properties and the
fp64 restatements (oracle/restate.py, pinned in tests/test_oracle.py).

Tolerances: float outputs rtMaxRelDiff (eval.cpp:758-763) <= 1e-4 in f32,
<= 1e-9 in f64 mode; integer/index outputs and histograms bit-exact."""
import json
import os

import numpy as np
import pytest

import oracle
import paper_2104_05372_b200 as dx
from oracle import restate
from paper_2104_05372_b200 import programs as P
from tests.kat_cases import KATS

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("name,src,entry,expected,cite", KATS, ids=[k[0] for k in KATS])
@pytest.mark.parametrize("f64", [False, True], ids=["f32", "f64"])
def test_reference_kats_on_device(ctx, name, src, entry, expected, cite, f64):
    got = dx.Program(src, entry, ctx=ctx, float64=f64)()
    assert len(got) == len(expected), cite
    for g, e in zip(got, expected):
        np.testing.assert_allclose(g, e, rtol=0, atol=1e-12 if f64 else 1e-5, err_msg=cite)


def _golden():
    with open(os.path.join(HERE, "golden", "parity_golden.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", sorted(_golden().keys()))
def test_golden_vectors(ctx, name):
    case = _golden()[name]
    inputs = [[np.asarray(l, dtype=dt) for l, dt in zip(leaves, dts)]
              for leaves, dts in zip(case["inputs"], case["input_dtypes"])]
    for f64, tol in ((False, 1e-4), (True, 1e-9)):
        got = dx.Program(case["source"], ctx=ctx, float64=f64)(*inputs)
        for g, w, kind in zip(got, case["outputs"], case["output_kinds"]):
            w = np.asarray(w, dtype=np.float64)
            if kind == "float":
                assert oracle.rel_diff(g, w) <= tol, (name, f64)
            else:
                np.testing.assert_array_equal(g.astype(np.int64), w.astype(np.int64))


def test_kmeans_full_size(ctx):
    """BASELINE configs[1]: n=1M, d=16, K=64, f32 vs the fp64 restatement."""
    n, d, k = 1_000_000, 16, 64
    pts, asg, cs = P.kmeans_inputs(n, d, k)
    cost, dC = dx.Program(P.kmeans_cost_grad(n, d, k), ctx=ctx)(pts, asg, cs)
    rc, rg = restate.kmeans_cost_grad(pts, asg, cs)
    assert oracle.rel_diff(cost, np.array([rc])) <= 1e-4
    assert oracle.rel_diff(dC, rg.ravel()) <= 1e-4


def test_kmeans_full_size_f64_tight(ctx):
    n, d, k = 1_000_000, 16, 64
    pts, asg, cs = P.kmeans_inputs(n, d, k)
    cost, dC = dx.Program(P.kmeans_cost_grad(n, d, k), ctx=ctx, float64=True)(pts, asg, cs)
    rc, rg = restate.kmeans_cost_grad(pts, asg, cs)
    assert oracle.rel_diff(cost, np.array([rc])) <= 1e-9
    assert oracle.rel_diff(dC, rg.ravel()) <= 1e-9


def test_histogram_full_size_bit_exact(ctx):
    """BASELINE configs[3]: 2^28 int32 keys into 4096 bins, uniform and Zipf."""
    n, k = 1 << 28, 4096
    prog = dx.Program(P.histogram(n, k), ctx=ctx)
    for zipf in (0.0, 1.1):
        keys = P.histogram_inputs(n, k, seed=11, zipf=zipf)
        (h,) = prog(keys)
        np.testing.assert_array_equal(h, np.bincount(keys, minlength=k).astype(np.float64))
        assert h.sum() == n  # checksum of counts


def test_matmul_256_fwd_grad(ctx):
    """BASELINE configs[0]: n=256 forward + gradient."""
    x, y = P.matmul_inputs(256)
    (z,) = dx.Program(P.matmul_fwd(256), ctx=ctx)(x, y)
    assert oracle.rel_diff(z, restate.matmul_fwd(x, y).ravel()) <= 1e-4
    loss, gx = dx.Program(P.matmul_grad(256), ctx=ctx)(x, y)
    rl, rg = restate.matmul_grad(x, y)
    assert oracle.rel_diff(loss, np.array([rl])) <= 1e-4
    assert oracle.rel_diff(gx, rg.ravel()) <= 1e-4


# Elementwise bar for the f32 MLP gradients at the BASELINE size.  Measured
# control (scripts/fp32_control.py, profiles/r02_fp32_control.txt): numpy
# float32 with BLAS sgemm reaches rtMaxRelDiff 2.55e-3 (dW1) / 8.8e-4 (dW2)
# against the fp64 restatement; even fp32 storage of z, h, y, dz with exactly
# accumulated GEMMs gives 3.7e-4 (dW1).  The gradients' smallest entries
# (~0.1) are differences of 8192 terms whose sum magnitude is ~1e3-1e4, so
# the reference's 1e-4 elementwise bar is out of reach of any fp32 pipeline
# at this size; the f32 path is held to 2x the sgemm control elementwise and
# to 1e-5 normwise, and the f64 parity mode (below) meets 1e-4 (in fact 1e-9).
MLP_F32_ELEMWISE = 5e-3
MLP_F32_NORMWISE = 1e-5


def _normrel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


def test_mlp_full_size_f32(ctx):
    """BASELINE configs[4]: batch 8192, 1024^3, square activation (tcgen05 3xTF32 GEMMs)."""
    b, i, h, o = 8192, 1024, 1024, 1024
    x, w1, w2 = P.mlp_inputs(b, i, h, o)
    prog = dx.Program(P.mlp_grad(b, i, h, o), ctx=ctx)
    assert "tcgen05 gemm" in prog.plan
    loss, d1, d2 = prog(x, [w1, w2])
    rl, r1, r2 = restate.mlp_grad(x, w1, w2)
    assert oracle.rel_diff(loss, np.array([rl])) <= 1e-4
    for got, want in ((d1, r1), (d2, r2)):
        assert _normrel(got, want) <= MLP_F32_NORMWISE
        assert oracle.rel_diff(got, want.ravel()) <= MLP_F32_ELEMWISE


def test_mlp_full_size_f64_mode(ctx):
    """The same program in the f64 parity mode (float64=True: f64 GEMMs and
    f64 intermediates, as the reference evaluates) meets the reference's
    elementwise 1e-4 at the full BASELINE size -- held here to 1e-9."""
    b, i, h, o = 8192, 1024, 1024, 1024
    x, w1, w2 = P.mlp_inputs(b, i, h, o)
    prog = dx.Program(P.mlp_grad(b, i, h, o), ctx=ctx, float64=True)
    assert "f64 gemm" in prog.plan
    loss, d1, d2 = prog(x, [w1, w2])
    rl, r1, r2 = restate.mlp_grad(x, w1, w2)
    assert oracle.rel_diff(loss, np.array([rl])) <= 1e-9
    assert oracle.rel_diff(d1, r1.ravel()) <= 1e-9
    assert oracle.rel_diff(d2, r2.ravel()) <= 1e-9


def test_matmul_256_f64_mode(ctx):
    x, y = P.matmul_inputs(256)
    loss, gx = dx.Program(P.matmul_grad(256), ctx=ctx, float64=True)(x, y)
    rl, rg = restate.matmul_grad(x, y)
    assert oracle.rel_diff(loss, np.array([rl])) <= 1e-9
    assert oracle.rel_diff(gx, rg.ravel()) <= 1e-9


def test_mlp_small_width(ctx):
    x, w1, w2 = P.mlp_inputs(256, 64, 64, 32)
    loss, d1, d2 = dx.Program(P.mlp_grad(256, 64, 64, 32), ctx=ctx)(x, [w1, w2])
    rl, r1, r2 = restate.mlp_grad(x, w1, w2)
    assert oracle.rel_diff(loss, np.array([rl])) <= 1e-4
    assert oracle.rel_diff(d1, r1.ravel()) <= 1e-4
    assert oracle.rel_diff(d2, r2.ravel()) <= 1e-4


def test_sharded_plan_single_rank_matches(ctx):
    """(rank 0 of world 1) == unsharded; world>1 uses NCCL (not in this box)."""
    n, d, k = 50_000, 16, 64
    pts, asg, cs = P.kmeans_inputs(n, d, k)
    a = dx.Program(P.kmeans_cost_grad(n, d, k), ctx=ctx)(pts, asg, cs)
    b = dx.Program(P.kmeans_cost_grad(n, d, k), ctx=ctx, rank=0, world=1)(pts, asg, cs)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_device_resident_inputs_zero_copy(ctx):
    """Inputs bound as device pointers (no H2D) give the same answer."""
    import torch
    n, d, k = 10_000, 16, 8
    pts, asg, cs = P.kmeans_inputs(n, d, k)
    prog = dx.Program(P.kmeans_cost_grad(n, d, k), ctx=ctx)
    want = prog(pts, asg, cs)
    tp = torch.from_numpy(pts).cuda()
    ta = torch.from_numpy(asg).cuda()
    tc = torch.from_numpy(cs).cuda()
    torch.cuda.synchronize()
    prog.bind_input_device(0, 0, tp.data_ptr())
    prog.bind_input_device(1, 0, ta.data_ptr())
    prog.bind_input_device(2, 0, tc.data_ptr())
    prog.run()
    got = [prog.get_output(0), prog.get_output(1)]
    for x, y in zip(got, want):
        assert oracle.rel_diff(x, y) <= 1e-6


def test_cpp_evalExprDevice_selftest():
    """C++ drop-in API (include/dexlet_device.hpp): reference-parsed programs,
    env-bound RtVal inputs, evalExprDevice instead of evalExpr."""
    import subprocess
    exe = os.path.join(os.path.dirname(HERE), "paper_2104_05372_b200", "bin", "dexlet_device_selftest")
    if not os.path.exists(exe):
        pytest.fail("selftest binary missing: run __graft_entry__.build()")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") == 10, out.stdout


@pytest.mark.parametrize("n,d,k", [(1_000_003, 8, 33), (777, 32, 5), (65, 16, 1), (31, 4, 3), (100_001, 16, 64)])
def test_group_mode_kmeans_shapes(ctx, n, d, k):
    """Group mode (G = d lanes per point, lane-owned table words, chunked
    register prefetch): ragged chunk counts, G in {4, 8, 16, 32}, a single
    centroid -- against the fp64 restatement, and bit-identical repeats."""
    pts, asg, cs = P.kmeans_inputs(n, d, k, seed=n % 97)
    prog = dx.Program(P.kmeans_cost_grad(n, d, k), ctx=ctx)
    if d < 32:  # d = 32 rows: the reverse nest is flattened (lane per element) instead
        assert f"dx_gl = dx_lane % {d}" in prog.source
    cost, dC = prog(pts, asg, cs)
    rc, rg = restate.kmeans_cost_grad(pts, asg, cs)
    assert oracle.rel_diff(cost, np.array([rc])) <= 1e-4
    assert oracle.rel_diff(dC, rg.ravel()) <= 1e-4
    if d < 32:  # group mode folds in a fixed order (the d = 32 path adds through shared atomics)
        again = prog(pts, asg, cs)
        assert np.array_equal(again[0], cost) and np.array_equal(again[1], dC)


def test_group_mode_pipelined_runs_match(ctx):
    """DXL_F_PIPELINE (inputs streamed before the PDL wait) gives the same
    bits as the default launch over many back-to-back runs."""
    n, d, k = 200_000, 16, 64
    pts, asg, cs = P.kmeans_inputs(n, d, k)
    a = dx.Program(P.kmeans_cost_grad(n, d, k), ctx=ctx)
    b = dx.Program(P.kmeans_cost_grad(n, d, k), ctx=ctx, flags=dx.DXL_F_PIPELINE)
    want = a(pts, asg, cs)
    for i, arr in enumerate((pts, asg, cs)):
        b.set_input(i, 0, arr)
    for _ in range(10):
        b.run()
    got = [b.get_output(0), b.get_output(1)]
    for x, y in zip(want, got):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("n", [10, 1 << 20])
def test_revdot_grad_two_index_forms(ctx, n):
    """grad of sum v.i * v.(reverse i) writes the cotangent at i and at n-1-i
    from the same ordinal: two threads touch each element, so the cell must
    not be owner-computed (was a cross-warp read-modify-write race at large
    n).  Exact answer 2 v[n-1-i]."""
    rng = np.random.default_rng(n)
    v = rng.standard_normal(n).astype(np.float32)
    g = dx.Program(P.revdot_grad(n), ctx=ctx)(v)
    g = g[0] if isinstance(g, (tuple, list)) else g
    want = 2.0 * v[::-1].astype(np.float64)
    assert oracle.rel_diff(np.asarray(g, dtype=np.float64).ravel(), want) <= 1e-6


def test_owner_cells_overwrite_after_zero(ctx):
    """Owner-computed cells written right after their zero-fill are stored
    (no zero pass, no read-modify-write); GEMM cell outputs likewise.  The
    MLP plan carries no zero-fill besides the scalar loss, and the gradients
    still match the fp64 restatement (small widths, 1e-4)."""
    x, w1, w2 = P.mlp_inputs(512, 64, 64, 32)
    prog = dx.Program(P.mlp_grad(512, 64, 64, 32), ctx=ctx)
    loss, d1, d2 = prog(x, [w1, w2])
    rl, r1, r2 = restate.mlp_grad(x, w1, w2)
    assert oracle.rel_diff(loss, np.array([rl])) <= 1e-4
    assert oracle.rel_diff(d1, r1.ravel()) <= 1e-4
    assert oracle.rel_diff(d2, r2.ravel()) <= 1e-4
    # repeated runs: the stored cells do not accumulate across runs
    loss2, e1, e2 = prog(x, [w1, w2])
    assert np.array_equal(d1, e1) and np.array_equal(d2, e2)
