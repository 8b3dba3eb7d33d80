"""GPU: dense contraction nests on the tcgen05 GEMM (dx_gemm.cuh) vs the fp64
restatement (oracle/restate.py, pinned against the reference in
tests/test_oracle.py) and, at small sizes, the reference evaluator itself.

Tolerance: rtMaxRelDiff (eval.cpp:758-763) <= 1e-4 (f32 mode: fp16x3 --
every operand row scaled by a power of two and split into two fp16 values,
the hi*hi + hi*lo + lo*hi products accumulated in fp32 in TMEM, K-ordered
within a tile)."""
import numpy as np
import pytest

import oracle
import paper_2104_05372_b200 as dx
from oracle import restate
from paper_2104_05372_b200 import programs as P

pytestmark = pytest.mark.gpu

SHAPES = [
    (64, 64, 64, True, False),
    (256, 256, 256, True, False),
    (200, 136, 68, True, False),     # ragged M, N; K not a multiple of 32
    (130, 260, 32, False, True),     # both operands transposed relative to the natural order
    (128, 128, 4, True, True),       # K below one k-block
    (1000, 520, 1024, False, False),
    (384, 128, 4096, True, True),    # long K: many pipeline wraps; split-K 4
    (256, 256, 8192, True, False),   # split-K 8 (4 tiles would leave 144 SMs idle)
    (1, 1, 8, True, False),          # single element
    (12800, 256, 96, True, False),   # 200 tiles
    (12800, 512, 40, False, True),   # (same, transposed operands)
]


@pytest.mark.parametrize("m,n,k,xk,yk", SHAPES)
def test_contraction_on_tensor_cores(ctx, m, n, k, xk, yk):
    src = P.contraction(m, n, k, xk, yk)
    x, y = P.contraction_inputs(m, n, k, xk, yk)
    prog = dx.Program(src, ctx=ctx)
    assert "tcgen05 gemm" in prog.plan
    (c,) = prog(x, y)
    want = restate.contraction(x, y, xk, yk)
    assert oracle.rel_diff(c, want.ravel()) <= 1e-4
    if m * n * k <= 1 << 21:
        (r,) = oracle.RefProgram(src)(x, y)
        assert oracle.rel_diff(c, r) <= 1e-4


def test_gemm_repeat_deterministic(ctx):
    m, n, k = 512, 384, 512
    src = P.contraction(m, n, k)
    x, y = P.contraction_inputs(m, n, k)
    prog = dx.Program(src, ctx=ctx)
    a = prog(x, y)[0]
    b = prog(x, y)[0]
    np.testing.assert_array_equal(a, b)


def test_gemm_precision_at_fp32_level(ctx):
    """fp16x3: error ~fp32 rounding, far below a single fp16 or tf32 pass (~1e-3)."""
    m = n = k = 512
    x, y = P.contraction_inputs(m, n, k, seed=7)
    (c,) = dx.Program(P.contraction(m, n, k), ctx=ctx)(x, y)
    want = restate.contraction(x, y)
    err = np.abs(c.reshape(m, n) - want).max() / np.abs(want).max()
    assert err < 2e-6, err


def test_matmul_fwd_uses_gemm(ctx):
    x, y = P.matmul_inputs(256)
    prog = dx.Program(P.matmul_fwd(256), ctx=ctx)
    assert "tcgen05 gemm fp16x3 256x256x256" in prog.plan
    (z,) = prog(x, y)
    assert oracle.rel_diff(z, restate.matmul_fwd(x, y).ravel()) <= 1e-4


def test_split_k_plan_and_determinism(ctx):
    """Under-filled long-K GEMMs split K across CTAs; the parts of a tile are
    added in part order (ticket), so repeated runs are bit-identical."""
    m, n, k = 256, 256, 8192
    src = P.contraction(m, n, k)
    x, y = P.contraction_inputs(m, n, k, seed=3)
    prog = dx.Program(src, ctx=ctx)
    assert "split-K" in prog.plan
    a = prog(x, y)[0]
    b = prog(x, y)[0]
    np.testing.assert_array_equal(a, b)
    assert oracle.rel_diff(a, restate.contraction(x, y).ravel()) <= 1e-4


@pytest.mark.parametrize("xk,yk", [(True, False), (False, True)])
def test_fp16x3_row_scales_cover_fp32_range(ctx, xk, yk):
    """Per-row power-of-two scales: rows of both operands spanning 1e-30 ..
    1e30 (far outside fp16's range), zero rows, and K not a multiple of 8
    still give fp32-level results (each output is one row pair's dot product,
    so the scales factor out exactly)."""
    m, n, k = 160, 136, 100
    x, y = P.contraction_inputs(m, n, k, xk, yk, seed=11)
    x = np.array(x, dtype=np.float32)
    y = np.array(y, dtype=np.float32)
    xr = np.logspace(-15, 15, m).astype(np.float32)
    yr = np.logspace(15, -15, n).astype(np.float32)
    if xk:  # x is [m][k]
        x *= xr[:, None]
        x[7] = 0.0
    else:   # x is [k][m]
        x *= xr[None, :]
        x[:, 7] = 0.0
    if yk:  # y is [n][k]
        y *= yr[:, None]
    else:   # y is [k][n]
        y *= yr[None, :]
    (c,) = dx.Program(P.contraction(m, n, k, xk, yk), ctx=ctx)(x, y)
    want = restate.contraction(x, y, xk, yk)
    mag = restate.contraction(np.abs(x), np.abs(y), xk, yk)  # sum |x||y| per output
    c = np.asarray(c, dtype=np.float64).reshape(m, n)
    ok = mag > 0
    assert np.max(np.abs(c - want)[ok] / mag[ok]) <= 1e-6
    assert np.all(c[7] == 0.0)
