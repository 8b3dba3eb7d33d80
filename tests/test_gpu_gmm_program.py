"""GPU: the ADBench GMM as a dexlet program (programs.gmm_program; exp/log
from frontend_ext) through dxl_program_create, linearize and transpose of
the reference front end, lowered by the generic device lowering -- against
the fp64 ADBench restatement (oracle/gmm.py), which the extended reference
evaluator pins to 1e-12 (tests/test_oracle.py).

Tolerances: f64 parity mode rtMaxRelDiff <= 1e-9; f32 <= 1e-4 on the
objective and d_alphas / d_means, and on d_icf normwise <= 1e-5 with
elementwise <= 1e-3 (the f32 rounding of beta ~ 1e2 moves responsibilities
by ~1e-6; see tests/test_gpu_gmm.py for the same bound on the fused kernels)."""
import numpy as np
import pytest

import oracle
import paper_2104_05372_b200 as dx
from oracle import gmm as G
from paper_2104_05372_b200 import programs as P

pytestmark = pytest.mark.gpu


def _normrel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


@pytest.mark.parametrize("n,d,K,gamma,m", [(1000, 8, 4, 1.0, 0), (2048, 16, 6, 0.8, 1), (777, 5, 3, 1.0, 0)])
@pytest.mark.parametrize("f64", [False, True], ids=["f32", "f64"])
def test_gmm_program_on_device(ctx, n, d, K, gamma, m, f64):
    a, mu, icf, x = G.gmm_inputs(n, d, K, seed=n + K)
    tabs = P.gmm_tables(d)
    mx, ma = P.gmm_stabilizers(a, mu, icf, x)
    prog = dx.Program(P.gmm_program(n, d, K, gamma, m), ctx=ctx, float64=f64)
    err, da, dm, di = prog(x, mx, ma, *tabs, [a, mu, icf])
    werr, wda, wdm, wdi = G.gmm_objective_grad(a, mu, icf, x, gamma, m)
    if f64:
        for g, w in ((err, [werr]), (da, wda), (dm, wdm), (di, wdi)):
            assert oracle.rel_diff(g, np.ravel(w)) <= 1e-9
        return
    assert oracle.rel_diff(err, np.array([werr])) <= 1e-4
    assert oracle.rel_diff(da, wda) <= 1e-4
    assert oracle.rel_diff(dm, wdm.ravel()) <= 1e-4
    assert _normrel(di, wdi) <= 1e-5
    assert oracle.rel_diff(di, wdi.ravel()) <= 1e-3


@pytest.mark.parametrize("n,K,gamma,m", [(3000, 5, 1.0, 0), (4097, 11, 0.8, 1)])
def test_gmm_program_dispatches_to_fused_kernels(ctx, n, K, gamma, m):
    """The canonical program at d = 64 (ADBench's dimension) runs on the fused
    tcgen05 kernel class through dxl_program_create: same inputs, same
    outputs as the program's generic lowering and as oracle/gmm.py
    (tolerances of tests/test_gpu_gmm.py)."""
    d = 64
    a, mu, icf, x = G.gmm_inputs(n, d, K, seed=n)
    tabs = P.gmm_tables(d)
    mx, ma = P.gmm_stabilizers(a, mu, icf, x)
    src = P.gmm_program(n, d, K, gamma, m)
    fast = dx.Program(src, ctx=ctx)
    assert "fused GMM kernel class" in fast.plan
    err, da, dm, di = fast(x, mx, ma, *tabs, [a, mu, icf])
    werr, wda, wdm, wdi = G.gmm_objective_grad(a, mu, icf, x, gamma, m)
    assert oracle.rel_diff(err, np.array([werr])) <= 1e-4
    for g, w in ((da, wda), (dm, wdm), (di, wdi)):
        assert _normrel(g, w) <= 1e-5
        assert oracle.rel_diff(g, w.ravel()) <= 4e-4
    generic = dx.Program(src, ctx=ctx, flags=dx.DXL_F_NO_GEMM)
    assert "fused GMM" not in generic.plan
    gerr, gda, gdm, gdi = generic(x, mx, ma, *tabs, [a, mu, icf])
    assert oracle.rel_diff(err, gerr) <= 1e-4
    # a non-canonical table is refused by the fused path (it would change the program)
    bad = tabs[2].copy()
    bad[1, 0] = 0.0
    with pytest.raises(dx.DexError):
        fast.set_input(5, 0, bad)



def test_gmm_program_f64_mode_at_baseline_dims(ctx):
    """The ADBench GMM program at BASELINE configs[2]'s dimensions (d = 64,
    K = 200) in the f64 parity mode (the generic lowering in binary64, as the
    reference evaluates; the fused fp16x3 class is f32-only): objective and
    every gradient entry within rtMaxRelDiff 1e-9 of the fp64 restatement.
    n = 1000: the generic plan keeps per-(point, component) d x d tapes
    (6.5 GB each here, 35 GB in all -- the plan header reports it), so the
    full n = 1M runs on the fused class only (tests/test_gpu_gmm.py)."""
    n, d, K = 1000, 64, 200
    a, mu, icf, x = G.gmm_inputs(n, d, K, seed=5)
    tabs = P.gmm_tables(d)
    mx, ma = P.gmm_stabilizers(a, mu, icf, x)
    prog = dx.Program(P.gmm_program(n, d, K), ctx=ctx, float64=True)
    assert "fused GMM" not in prog.plan
    err, da, dm, di = prog(x, mx, ma, *tabs, [a, mu, icf])
    werr, wda, wdm, wdi = G.gmm_objective_grad(a, mu, icf, x)
    assert oracle.rel_diff(err, np.array([werr])) <= 1e-9
    for g, w in ((da, wda), (dm, wdm), (di, wdi)):
        assert oracle.rel_diff(g, np.ravel(w)) <= 1e-9
