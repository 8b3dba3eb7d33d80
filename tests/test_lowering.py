"""CPU: structure of the lowering plans (which kernel class / Accum strategy
each benchmark program gets) and evidence in the compiled sm_100a code."""
import ctypes
import os
import shutil
import subprocess
import tempfile

import pytest

import paper_2104_05372_b200 as dx
from paper_2104_05372_b200 import programs as P


def _kernels(plan):
    return [l for l in plan.splitlines() if " kernel " in l]


def _cubin(source):
    lib = dx.lib()
    lib.dxc_module_cubin.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.POINTER(ctypes.c_size_t)]
    n = ctypes.c_size_t()
    assert lib.dxc_module_cubin(source.encode(), None, 0, ctypes.byref(n)) == 0
    buf = ctypes.create_string_buffer(n.value)
    assert lib.dxc_module_cubin(source.encode(), buf, n.value, ctypes.byref(n)) == 0
    return buf.raw


def _sass(source):
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump unavailable")
    with tempfile.NamedTemporaryFile(suffix=".cubin", delete=False) as f:
        f.write(_cubin(source))
        path = f.name
    try:
        return subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    finally:
        os.unlink(path)


def test_kmeans_value_and_grad_is_one_fused_kernel():
    """Forward tape inlined into both consumers (no HBM tape), the cotangent
    broadcast folded (accum-to-map), cost and gradient loops fused
    horizontally: one kernel in group mode (16 lanes per point, one lane per
    column) that also folds the partials after a ticket grid barrier and owns
    the zero-fills (the plan is that single launch)."""
    prog = dx.Program(P.kmeans_cost_grad(100_000, 16, 64), ctx=None)
    ks = _kernels(prog.plan)
    assert len(ks) == 1, prog.plan
    assert "zero b" not in prog.plan.split("---")[0], prog.plan
    src = prog.source
    assert "const int dx_gl = dx_lane % 16" in src   # 16 lanes per point
    assert "dx_grp_sum" not in src                  # per-point costs: lane partials straight into the cost register
    assert "*(float*)((char*)dx_wtl1 + " in src      # lane-owned words of the warp's dC table
    assert "wtg3" in src                             # centroids: one interleaved copy per group (no bank conflicts)
    assert src.count("dx_l2_prefetch(") >= 3         # TMA bulk L2 prefetch of the chunk after next
    assert "dx_warp_tab_flush<16, 64, 20>" in src
    # one point stream: 16 loads at constant offsets from one base, for a/b x first/refill x full/ragged
    assert src.count("__ldcs(dx_b0 + ") == 128
    assert src.count("__shfl_sync(DX_FULL, gp") == 32  # assignments: one load per chunk, shuffled to the groups
    assert ", false, true, 1LL);" in src            # fold overwrites the (never zeroed) cell
    assert "dx_spread_barrier(" in src and "dx_coop_fold_b<double, dx_f>" in src
    assert "dx_warp_sum(rp0)" in src                # register partial for the cost: warp sums share the table flush's barrier
    sass = _sass(src)
    assert "STL" not in sass and "LDL" not in sass  # prefetch buffers stay in registers


def test_histogram_uses_exact_shared_counters():
    prog = dx.Program(P.histogram(1 << 20, 4096), ctx=None)
    assert len(_kernels(prog.plan)) == 1
    assert "dx_count_smem" in prog.source
    # u32 counters (4096-word partial rows) folded in fixed block order (u64
    # group sums) and scaled by the constant by the last blocks of the launch
    assert "dx_lbd_group<unsigned, long long>" in prog.source
    assert "dx_lbd_final<long long, double>" in prog.source
    sass = _sass(prog.source)
    assert "ATOMS" in sass and "LDG.E.128" in sass


def test_matmul_forward_flattens_perfect_nest():
    """The generic path flattens `for i k.` into one 4096-ordinal kernel
    (with the GEMM class disabled; by default this nest is a GEMM)."""
    prog = dx.Program(P.matmul_fwd(64), ctx=None, float64=True, flags=dx.F_NO_GEMM)
    ks = _kernels(prog.plan)
    assert len(ks) == 1 and "n=4096" in ks[0], prog.plan


def test_state_loop_runs_on_one_device_thread():
    """`get`/`:=` on an outer cell blocks chunking (ParScan, eval.cpp:548-600):
    the loop becomes a serial kernel, never a CPU loop."""
    prog = dx.Program(P.cumulative(50), ctx=None)
    ks = _kernels(prog.plan)
    assert len(ks) == 1 and "serial" in ks[0]


def test_dead_cells_are_not_allocated():
    prog = dx.Program(P.kmeans_grad(10_000, 16, 8), ctx=None)
    # the n-element cotangent broadcast cell of the transposed sum is never
    # materialized: no zero-fill of 10000 elements remains
    assert "(10000)" not in prog.plan


def test_sharded_plan_merges_cells_in_one_collective():
    """Both Accum cells of the fused k-means kernel (cost, dC) are merged by
    one grouped all-gather + rank-ordered fold (eval.cpp:357-366 order)."""
    prog = dx.Program(P.kmeans_cost_grad(1000, 16, 8), ctx=None, rank=1, world=2)
    plan = prog.plan.split("---")[0]
    assert plan.count("merge 2 Accum deltas") == 1 and "allreduce" not in plan


def test_contraction_recognized_as_gemm():
    """`for i l. sum for j. x*y` lowers to operand prologues + the tcgen05 GEMM
    in f32 mode whatever the operands' storage order; f64 parity mode keeps
    the generic loop kernel."""
    for xk, yk in ((True, False), (False, True), (False, False), (True, True)):
        p = dx.Program(P.contraction(200, 136, 68, xk, yk), ctx=None).plan
        assert "tcgen05 gemm fp16x3 200x136x68" in p and p.count("gemm operand ") - p.count("gemm operand row max") == 2, p
    p = dx.Program(P.contraction(64, 64, 6), ctx=None).plan      # K padded to 8 in the operands
    assert "tcgen05 gemm fp16x3 64x64x6" in p
    assert "tcgen05" not in dx.Program(P.contraction(64, 64, 64), ctx=None, float64=True).plan
    src = dx.Program(P.contraction(64, 64, 64), ctx=None).source
    sass = _sass(src)
    assert "UTCHMMA" in sass and "UTMALDG.2D" in sass and "LDTM" in sass  # tcgen05.mma, TMA, tcgen05.ld


def test_mlp_and_matmul_grad_on_tensor_cores():
    """The AD programs: every contraction of the forward tape and of the
    transposed loops is a GEMM (MLP: Z = XW1, Y = HW2, dH, dW2, dW1); the AoS
    tapes are split, never materialized whole."""
    p = dx.Program(P.mlp_grad(8192, 1024, 1024, 1024), ctx=None).plan
    assert p.count("tcgen05 gemm") == 5, p
    assert p.count("(+=)") == 0  # cells right after their zero-fill are stored, not accumulated
    zeros = [l for l in p.split("---")[0].splitlines() if " zero b" in l]
    assert all(l.endswith("(1)") or l.endswith("(1024)") for l in zeros), zeros  # the loss cell and row-max words only
    assert p.count("copy b") == 2  # the cotangent deltas move into the zero-pending weight cells
    assert "8589934592" not in p  # no B*H*I tape
    p = dx.Program(P.matmul_grad(256), ctx=None).plan
    assert p.count("tcgen05 gemm") == 2, p


def test_row_sum_runs_one_warp_per_row():
    """A short outer loop over a long reduction (the matmul's row sums) runs
    one warp per ordinal: the lanes split the inner loop and warp-sum."""
    prog = dx.Program(P.matmul_grad(256), ctx=None)
    assert "(warp per ordinal)" in prog.plan
    src = prog.source
    assert "+= 32)" in src and "dx_warp_sum(" in src


def test_effect_nest_flattened_and_broadcast_kept_lazy():
    """MLP dY: the per-row cotangent broadcast stays a lazy map inside the
    kernel (no local array) and the (batch, out) nest runs flattened."""
    prog = dx.Program(P.mlp_grad(8192, 64, 64, 1024), ctx=None)
    assert "(flattened)" in prog.plan
    src = prog.source
    i = src.index("(flattened)")
    body = src[i:src.index('extern "C"', i)]
    assert "[1024] = {}" not in body


def test_long_k_gemm_is_split():
    prog = dx.Program(P.contraction(256, 256, 8192), ctx=None)
    assert "split-K 8" in prog.plan
    prog = dx.Program(P.contraction(1000, 520, 1024), ctx=None)
    assert "split-K" not in prog.plan  # enough output tiles, short K


def test_tiny_map_bodies_keep_three_vector_loads_in_flight():
    prog = dx.Program(P.histogram(1 << 20, 4096), ctx=None)
    assert prog.source.count("const int4 w = *(const int4*)") == 3


def test_transposed_gemm_operands_use_a_tiled_prologue():
    # an operand read along its row variable (stride 1 over rows) goes through
    # 32 x 64 tiles transposed in shared memory, after a column-max pass with a
    # thread per row; a K-contiguous operand is split warp per row (16-byte
    # loads when aligned); both with per-row fp16 scales, fp32 arithmetic
    prog = dx.Program(P.contraction(130, 260, 36, True, False), ctx=None)
    ops = [l for l in prog.plan.split("\n") if "gemm operand" in l and "row max" not in l]
    assert len(ops) == 2
    assert "tiled transpose" not in ops[0] and "tiled transpose" in ops[1]
    assert "gemm operand row max" in prog.plan      # per-row max pass of the transposed operand
    assert "unsigned short th[64 * 33 + 1]" in prog.source
    assert "atomicMax(mx + r, __float_as_uint(mm))" in prog.source
    assert "dx_f16_split_sc(" in prog.source
    assert "for (long long r = blockIdx.x * 8LL + (threadIdx.x >> 5)" in prog.source
    assert prog.source.count("dx_f16_scale(") >= 2


EMPTY_PROGRAMS = [
    "main = \\x:((Fin 0)=>Float). sum x\n",
    "main = \\p:((Fin 0)=>(Fin 4)). yieldAccum \\h. for i. h!(p.i) += 1.0\n",
    "main = \\x:((Fin 0)=>Float). for i. (x.i) * 2.0\n",
    "main = \\x:((Fin 3)=>((Fin 0)=>Float)). for i. sum (x.i)\n",
    "main = \\x:((Fin 0)=>Float).\n  f = \\v:((Fin 0)=>Float). sum (for i. (v.i) * (v.i))\n  grad f x\n",
]


@pytest.mark.parametrize("src", EMPTY_PROGRAMS)
def test_empty_index_sets_lower_without_kernels(src):
    """Fin 0 loops enumerate nothing (eval.cpp:295-308): no kernel is launched
    for them and cells keep their zero (eval.cpp:452-464); lowering must not
    divide by the empty size (it used to abort the host with SIGFPE)."""
    prog = dx.Program(src, ctx=None)
    assert "kernel dxk" not in prog.plan or "(Fin 3)" in src


def test_no_experiment_switches_in_library():
    """Only the cache/dump/diagnostic environment variables remain in the
    product library (no DEXLET_* switch changes a result)."""
    import re
    here = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2104_05372_b200", "csrc")
    found = set()
    for f in os.listdir(here):
        if f.endswith((".cpp", ".inc", ".cuh", ".hpp")):
            found |= set(re.findall(r'getenv\("([A-Z_]+)"\)', open(os.path.join(here, f)).read()))
    assert found <= {"DEXLET_CACHE_DIR", "HOME", "DEXLET_NO_DISK_CACHE", "DEXLET_DUMP_DIR", "DEXLET_DEBUG_CONTRACT"}, found


def test_mlp_world2_plan_is_data_parallel():
    """configs[4] sharded on the batch: every contraction stays
    on the tensor cores (forward GEMMs split by rows, weight-gradient GEMMs
    split over K = batch), the activations and their cotangents never leave
    the rank (no all-reduce of maps), and the Accum deltas -- dW1, dW2 and
    the loss -- go out in one fused merge (the reference's chunk-order
    overlay merge, eval.cpp:357-366)."""
    b, i, h, o = 2048, 256, 256, 128
    for rank in (0, 1):
        plan = dx.Program(P.mlp_grad(b, i, h, o), ctx=None, rank=rank, world=2).plan.split("---")[0]
        assert plan.count("tcgen05 gemm") == 5, plan
        assert "gemm fp16x3 1024x" in plan  # M-split: the rank's 1024 batch rows
        assert "allreduce" not in plan, plan
        merges = [l for l in plan.splitlines() if "merge" in l]
        assert len(merges) == 1, plan
        assert f"merge 3 Accum deltas ({i * h + h * o + 1} values)" in merges[0], merges


def test_gmm_program_recognizer():
    """dxl_gmm_program_match: the canonical ADBench program (any sizes, any
    Wishart gamma / m) is recognized and its parameters read back; a change
    to the objective is not."""
    assert dx.gmm_program_match(P.gmm_program(3000, 64, 5)) == (3000, 64, 5, 1.0, 0)
    n, d, k, g, m = dx.gmm_program_match(P.gmm_program(4097, 64, 11, 0.8, 1))
    assert (n, d, k, m) == (4097, 64, 11, 1) and abs(g - 0.8) < 1e-12
    src = P.gmm_program(100, 5, 3)
    assert dx.gmm_program_match(src) == (100, 5, 3, 1.0, 0)
    assert dx.gmm_program_match(src.replace("0.5 * sq", "0.25 * sq")) is None
    assert dx.gmm_program_match(src.replace("log s", "s")) is None
    assert dx.gmm_program_match(P.kmeans_cost_grad(10, 2, 2)) is None


def test_fp32_split_matches_fp64_split():
    """The fp32 operand prologue path (dx_f16_split_sc, dx_gemm.cuh) claims
    bit-identical fp16 hi/lo images to the fp64 form dx_f16_split((double)x * sc):
    x * sc with sc a power of two is the exact product rounded once to fp32 in
    both, and x - hi is exact in fp32.  Checked here with numpy's round-to-nearest
    conversions on values spanning the fp32 range and every scale a row can get
    (max |v| of the row into [2^13, 2^14))."""
    import numpy as np
    rng = np.random.default_rng(7)
    x = (rng.standard_normal(200_000) * np.exp2(rng.integers(-60, 60, 200_000))).astype(np.float32)
    x[:1000] = 0.0
    x[1000:1010] = np.float32(-0.0)
    for e in range(-60, 61, 7):
        row = x[np.abs(x) < np.float32(2.0 ** e)]
        if row.size == 0:
            continue
        sc = 2.0 ** (14 - e)                      # dx_f16_scale for a row max in [2^(e-1), 2^e)
        # fp32 path
        xs = row * np.float32(sc)
        hi = xs.astype(np.float16)
        lo = (xs - hi.astype(np.float32)).astype(np.float16)
        # fp64 path
        xd = row.astype(np.float64) * sc
        hi_d = xd.astype(np.float32).astype(np.float16)
        lo_d = (xd - hi_d.astype(np.float64)).astype(np.float32).astype(np.float16)
        assert np.array_equal(hi.view(np.uint16), hi_d.view(np.uint16)), e
        assert np.array_equal(lo.view(np.uint16), lo_d.view(np.uint16)), e
