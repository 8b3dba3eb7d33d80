"""CPU: the C-ABI library loads, exports every symbol include/dexlet_cuda.h
declares, and its host-side logic (lowering, error codes, index-set math,
chunking) works without a GPU.  No device compute here."""
import ctypes
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

import paper_2104_05372_b200 as dx
from paper_2104_05372_b200 import programs as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    with open(os.path.join(ROOT, "include", "dexlet_cuda.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(dx[cl]_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    syms = _header_symbols()
    assert len(syms) >= 40
    lib = ctypes.CDLL(dx.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(dx.ABI_SYMBOLS) | set(syms)
    assert sorted(dx.ABI_SYMBOLS) == syms


def test_reference_evaluator_not_linked():
    """The product library contains the reference front end but never its
    evaluator: no CPU fallback path exists (eval.cpp is not linked)."""
    nm = shutil.which("nm")
    if not nm:
        pytest.skip("nm unavailable")
    out = subprocess.run([nm, "-C", "-D", "--defined-only", dx.LIB_PATH], capture_output=True, text=True).stdout
    assert re.search(r"dexlet::evalExpr\(", out) is None
    assert re.search(r"dexlet::evalParallelFor\(", out) is None
    assert re.search(r"dexlet::evalExprDevice\(", out)  # the device twin is there
    assert "dexlet::parseProgram" in out  # front end is there
    assert "dxl_program_run" in out


def test_chunk_rule_matches_reference():
    """eval.cpp:323-330: base = total/chunks, the first rem chunks get +1."""
    for total, parts in [(10, 3), (7, 7), (5, 8), (1_000_000, 8), (13, 1)]:
        covered = []
        eff = min(parts, total)
        base, rem = total // eff, total % eff
        start = 0
        for c in range(parts):
            lo, hi = dx.chunk_range(total, parts, c)
            if c < eff:
                ln = base + (1 if c < rem else 0)
                assert (lo, hi) == (start, start + ln)
                start += ln
            else:
                assert lo == hi
            covered.extend(range(lo, hi))
        assert covered == list(range(total))


def test_desc_helpers():
    lib = dx.lib()
    v = ctypes.c_int64()
    assert lib.dxc_desc_size(b"PF3EF2U", ctypes.byref(v)) == 0 and v.value == 9
    assert lib.dxc_desc_reverse(b"F10", 3, ctypes.byref(v)) == 0 and v.value == 6
    assert lib.dxc_desc_reverse(b"F10", 10, ctypes.byref(v)) == dx.DXC_E_BOUNDS


@pytest.mark.parametrize("src", [
    P.kmeans_cost_grad(1000, 16, 64), P.kmeans_grad(100, 8, 4), P.histogram(1 << 20, 4096),
    P.matmul_fwd(64), P.matmul_grad(32), P.mlp_grad(16, 8, 8, 4), P.kmeans_assign(100, 3, 5),
    P.cumulative(9), P.either_case(7), P.mandelbrot(4, 3, 5), P.pair_index_sum(3, 4),
])
@pytest.mark.parametrize("f64", [False, True])
def test_lower_and_compile_without_gpu(src, f64):
    """Lowering + NVRTC sm_100a compilation need no device (ctx=None)."""
    prog = dx.Program(src, ctx=None, float64=f64)
    assert "extern \"C\" __global__" in prog.source or "0 kernels" in prog.plan
    assert prog.output_leaves()


def test_leaf_layout():
    prog = dx.Program(P.mlp_grad(8, 6, 5, 4), ctx=None)
    assert prog.input_leaves() == [[(dx.LEAF_FLOAT, 48)], [(dx.LEAF_FLOAT, 30), (dx.LEAF_FLOAT, 20)]]
    assert prog.output_leaves() == [(dx.LEAF_FLOAT, 1), (dx.LEAF_FLOAT, 30), (dx.LEAF_FLOAT, 20)]
    prog = dx.Program(P.histogram(100, 7), ctx=None)
    assert prog.input_leaves() == [[(dx.LEAF_INDEX, 100)]]


@pytest.mark.parametrize("src,code", [
    ("main = \\x:((Fin 3)=>Float). for i. (x.i) +\n", dx.DXC_E_PARSE),
    ("main = \\x:((Fin 3)=>Float). for i. (x.i) + (ord i)\n", dx.DXC_E_TYPE),
    ("main = \\x:((Fin 3)=>Float). x.(@5 : Fin 3)\n", dx.DXC_E_BOUNDS),
    ("main = \\x:((Fin 3)=>Float). y\n", dx.DXC_E_TYPE),
])
def test_error_codes(src, code):
    with pytest.raises(dx.DexError) as e:
        dx.Program(src, ctx=None)
    assert e.value.code == code, e.value.message


def test_no_device_calls_fail_loudly():
    """Without a GPU, device entry points report an error instead of
    computing anything on the CPU."""
    if dx.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(dx.DexError):
        dx.Context(0)
    prog = dx.Program(P.histogram(10, 3), ctx=None)
    with pytest.raises(dx.DexError):
        prog.run()


def test_gmm_header_symbols_exported():
    """include/dexlet_gmm.h: every declared entry point is exported."""
    with open(os.path.join(ROOT, "include", "dexlet_gmm.h")) as f:
        syms = sorted(set(re.findall(r"\b(dxg_[a-z0-9_]+)\s*\(", f.read())))
    assert len(syms) >= 10
    lib = ctypes.CDLL(dx.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(dx.GMM_ABI_SYMBOLS) == syms


def test_gmm_module_compiles_for_sm100a():
    """The fused GMM kernels NVRTC-compile for sm_100a (no GPU needed) and the
    contractions are tcgen05 MMAs (UTCHMMA in the SASS)."""
    from paper_2104_05372_b200.csrc_sources import gmm_module_source  # noqa: F401
    src = gmm_module_source()
    lib = dx.lib()
    lib.dxc_module_cubin.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    n = ctypes.c_size_t()
    assert lib.dxc_module_cubin(src.encode(), None, 0, ctypes.byref(n)) == 0, lib.dxc_last_error()
    buf = ctypes.create_string_buffer(n.value)
    assert lib.dxc_module_cubin(src.encode(), buf, n.value, ctypes.byref(n)) == 0
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump unavailable")
    import tempfile
    with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
        f.write(buf.raw)
        f.flush()
        sass = subprocess.run([cuobjdump, "-sass", f.name], capture_output=True, text=True).stdout
    for k in dx.GMM_KERNELS:
        assert f"Function : {k}" in sass, k
    assert "UTCHMMA" in sass
    assert "UBLKCP" in sass


def test_gmm_abi_rejects_bad_arguments():
    """Argument checks run before any device work (no GPU needed)."""
    lib = dx.lib()
    g = ctypes.c_void_p()
    assert lib.dxg_gmm_create(None, 64, 4, 100, 100, ctypes.byref(g)) == dx.DXC_E_ARG
    assert lib.dxg_gmm_set_params(None, None, None, None) == dx.DXC_E_ARG
    assert lib.dxg_gmm_set_points(None, None) == dx.DXC_E_ARG
    assert lib.dxg_gmm_run(None, 1.0, 0, 1) == dx.DXC_E_ARG
