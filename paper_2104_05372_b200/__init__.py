"""B200 execution backend for the data-parallel core of dexlet (arXiv 2104.05372).

Thin ctypes binding over the C-ABI of ``libdexlet_cuda.so`` (include/dexlet_cuda.h).
The product path is C++/CUDA: the reference front end (parse, typecheck,
simplify, linearize/transpose, optimize) compiled unmodified, then device
lowering of every ``for``/``runAccum`` nest into NVRTC-compiled sm_100a kernels
built on the hand-written device runtime ``csrc/dx_device.cuh``.

There is no CPU fallback: if the shared library is missing this module raises
at import, and on a machine without a GPU only compile-only programs
(``Program(..., ctx=None)``) can be created.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdexlet_cuda.so")



class _LazyLib:
    """libdexlet_cuda.so, mapped on first use: importing the package (e.g. for
    the input generators in ``programs``) does not load the CUDA library.  A
    missing library raises on that first use -- there is no CPU fallback."""

    def __init__(self):
        self._cdll = None

    def load(self) -> ctypes.CDLL:
        if self._cdll is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `make -C paper_2104_05372_b200/csrc` "
                    "(or __graft_entry__.build()); the backend has no CPU fallback")
            cdll = ctypes.CDLL(LIB_PATH)
            for name, res, args in _SIGS:
                f = getattr(cdll, name)
                f.restype = res
                f.argtypes = list(args)
            self._cdll = cdll
        return self._cdll

    def __getattr__(self, name):
        return getattr(self.load(), name)


_lib = _LazyLib()
_SIGS = []

# status codes (include/dexlet_cuda.h)
DXC_OK = 0
DXC_E_PARSE = 1
DXC_E_TYPE = 4
DXC_E_SIZE = 11
DXC_E_BOUNDS = 12
DXC_E_REF = 13
DXC_E_PARALLEL = 14
DXC_E_INTERNAL = 15
DXC_E_CUDA = 100
DXC_E_ARG = 101

# dxl_options.flags (include/dexlet_cuda.h)
DXL_F_NO_FUSION = 1
DXL_F_NO_ROWSCATTER = 2
DXL_F_DUMP = 4
DXL_F_TEST_COMM_MISMATCH = 8
DXL_F_NO_GEMM = 16
DXL_F_PIPELINE = 32
DXL_F_COUNT = 64

LEAF_FLOAT, LEAF_INT, LEAF_INDEX = 0, 1, 2
DXC_F32, DXC_F64, DXC_I32, DXC_I64, DXC_U32 = 0, 1, 2, 3, 4

F_NO_FUSION = 1
F_NO_ROWSCATTER = 2
F_DUMP = 4
F_TEST_COMM_MISMATCH = 8  # test only: one device emulating the ranks of a sharded plan
F_NO_GEMM = 16  # contractions through the generic SIMT lowering

_ERRNAMES = {
    DXC_E_PARSE: "E-parse", DXC_E_TYPE: "E-type", DXC_E_SIZE: "E-size",
    DXC_E_BOUNDS: "E-bounds", DXC_E_REF: "E-ref", DXC_E_PARALLEL: "E-parallel",
    DXC_E_INTERNAL: "E-internal", DXC_E_CUDA: "E-cuda", DXC_E_ARG: "E-arg",
}


class DexError(RuntimeError):
    """Mirror of dexlet::DexError (reference include/dexlet/errors.hpp:62-99)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[{_ERRNAMES.get(code, code)}] {message}")
        self.code = code
        self.message = message


class DxlOptions(ctypes.Structure):
    _fields_ = [("float64", ctypes.c_int), ("rank", ctypes.c_int), ("world", ctypes.c_int),
                ("threads", ctypes.c_int), ("flags", ctypes.c_int)]


def _sig(name, res, *args):
    _SIGS.append((name, res, args))


_vp = ctypes.c_void_p
_ip = ctypes.POINTER(ctypes.c_int)
_i64p = ctypes.POINTER(ctypes.c_int64)
_sig("dxc_last_error", ctypes.c_char_p)
_sig("dxc_init", ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp))
_sig("dxc_destroy", ctypes.c_int, _vp)
_sig("dxc_device_count", ctypes.c_int, _ip)
_sig("dxc_sm_count", ctypes.c_int, _vp, _ip)
_sig("dxc_stream", _vp, _vp)
_sig("dxc_sync", ctypes.c_int, _vp)
_sig("dxc_host_alloc", ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(_vp))
_sig("dxc_host_free", ctypes.c_int, _vp)
_sig("dxc_event_record", ctypes.c_int, _vp, ctypes.POINTER(_vp))
_sig("dxc_capture_begin", ctypes.c_int, _vp)
_sig("dxl_gmm_program_match", ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int),
     ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int))
_sig("dxl_program_counters", ctypes.c_int, _vp, ctypes.POINTER(ctypes.c_longlong))
_sig("dxc_capture_end", ctypes.c_int, _vp, ctypes.POINTER(_vp))
_sig("dxc_graph_launch", ctypes.c_int, _vp, _vp)
_sig("dxc_graph_destroy", ctypes.c_int, _vp)
_sig("dxc_event_elapsed_ms", ctypes.c_int, _vp, _vp, ctypes.POINTER(ctypes.c_float))
_sig("dxc_event_destroy", ctypes.c_int, _vp)
_sig("dxc_nccl_unique_id", ctypes.c_int, _vp)
_sig("dxc_comm_init", ctypes.c_int, _vp, _vp, ctypes.c_int, ctypes.c_int)
_sig("dxc_allreduce_sum", ctypes.c_int, _vp, _vp, ctypes.c_size_t, ctypes.c_int)
_sig("dxc_desc_size", ctypes.c_int, ctypes.c_char_p, _i64p)
_sig("dxc_desc_reverse", ctypes.c_int, ctypes.c_char_p, ctypes.c_int64, _i64p)
_sig("dxc_chunk_range", ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _i64p, _i64p)
_sig("dxl_program_create", ctypes.c_int, _vp, ctypes.c_char_p, ctypes.c_char_p,
     ctypes.POINTER(DxlOptions), ctypes.POINTER(_vp))
_sig("dxl_program_destroy", ctypes.c_int, _vp)
_sig("dxl_program_num_inputs", ctypes.c_int, _vp, _ip)
_sig("dxl_program_input_num_leaves", ctypes.c_int, _vp, ctypes.c_int, _ip)
_sig("dxl_program_input_leaf", ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, _ip, _i64p)
_sig("dxl_program_output_num_leaves", ctypes.c_int, _vp, _ip)
_sig("dxl_program_output_leaf", ctypes.c_int, _vp, ctypes.c_int, _ip, _i64p)
_sig("dxl_program_set_input", ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int)
_sig("dxl_program_set_input_n", ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int64)
_sig("dxl_program_check", ctypes.c_int, _vp)
_sig("dxl_program_set_input_rows", ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int64,
     ctypes.c_int64)
_sig("dxl_program_bind_input_device", ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, _vp)
_sig("dxl_program_input_device_ptr", ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp))
_sig("dxl_program_run", ctypes.c_int, _vp)
_sig("dxl_program_get_output", ctypes.c_int, _vp, ctypes.c_int, _vp, ctypes.c_int)
_sig("dxl_program_output_device_ptr", ctypes.c_int, _vp, ctypes.c_int, ctypes.POINTER(_vp))
_sig("dxl_program_source", ctypes.c_char_p, _vp)
_sig("dxl_program_plan", ctypes.c_char_p, _vp)
_sig("dxl_program_num_launches", ctypes.c_int, _vp, _ip)
_sig("dxl_program_enable_kernel_timing", ctypes.c_int, _vp, ctypes.c_int)
_sig("dxl_program_kernel_times", ctypes.c_int, _vp, ctypes.POINTER(ctypes.c_float), ctypes.c_int, _ip)
_sig("dxl_program_kernel_names", ctypes.c_char_p, _vp)
_sig("dxc_l2_flush", ctypes.c_int, _vp, ctypes.c_size_t)
_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)
_sig("dxg_gmm_create", ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
     ctypes.POINTER(_vp))
_sig("dxg_gmm_destroy", ctypes.c_int, _vp)
_sig("dxg_gmm_set_params", ctypes.c_int, _vp, _vp, _vp, _vp)
_sig("dxg_gmm_set_points", ctypes.c_int, _vp, _vp)
_sig("dxg_gmm_input_device_ptrs", ctypes.c_int, _vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
     ctypes.POINTER(_vp), ctypes.POINTER(_vp))
_sig("dxg_gmm_run", ctypes.c_int, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_int)
_sig("dxg_gmm_get", ctypes.c_int, _vp, _vp, _vp, _vp, _vp)
_sig("dxg_gmm_objective", ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _vp, _vp, _vp, _vp,
     ctypes.c_double, ctypes.c_int, _vp)
_sig("dxg_gmm_objective_grad", ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _vp, _vp, _vp,
     _vp, ctypes.c_double, ctypes.c_int, _vp, _vp)
_sig("dxg_gmm_enable_timing", ctypes.c_int, _vp, ctypes.c_int)
_sig("dxg_gmm_kernel_times", ctypes.c_int, _vp, _f32p, ctypes.c_int, _ip)

#: every symbol declared in include/dexlet_cuda.h
ABI_SYMBOLS = [
    "dxc_last_error", "dxc_init", "dxc_destroy", "dxc_device_count", "dxc_sm_count", "dxc_stream",
    "dxc_sync", "dxc_buf_alloc", "dxc_buf_free", "dxc_buf_ptr", "dxc_buf_upload", "dxc_buf_download",
    "dxc_buf_zero", "dxc_host_alloc", "dxc_host_free", "dxc_module_compile", "dxc_module_cubin",
    "dxc_launch", "dxc_event_record", "dxc_event_elapsed_ms", "dxc_event_destroy",
    "dxc_capture_begin", "dxc_capture_end", "dxc_graph_launch", "dxc_graph_destroy", "dxl_program_counters",
    "dxl_program_set_input_rows", "dxl_gmm_program_match",
    "dxc_nccl_unique_id", "dxc_comm_init", "dxc_allreduce_sum", "dxl_program_create",
    "dxl_program_destroy", "dxl_program_num_inputs", "dxl_program_input_num_leaves",
    "dxl_program_input_leaf", "dxl_program_output_num_leaves", "dxl_program_output_leaf",
    "dxl_program_set_input", "dxl_program_bind_input_device", "dxl_program_input_device_ptr",
    "dxl_program_run", "dxl_program_get_output", "dxl_program_output_device_ptr",
    "dxl_program_source", "dxl_program_plan", "dxl_program_num_launches", "dxc_desc_size",
    "dxc_desc_reverse", "dxc_chunk_range", "dxc_l2_flush", "dxl_program_enable_kernel_timing",
    "dxl_program_kernel_times", "dxl_program_kernel_names", "dxl_program_set_input_n", "dxl_program_check",
]
#: every symbol declared in include/dexlet_gmm.h
GMM_ABI_SYMBOLS = [
    "dxg_gmm_create", "dxg_gmm_destroy", "dxg_gmm_set_params", "dxg_gmm_set_points",
    "dxg_gmm_input_device_ptrs", "dxg_gmm_grad_device_ptrs", "dxg_gmm_run", "dxg_gmm_get", "dxg_gmm_objective",
    "dxg_gmm_objective_grad", "dxg_gmm_enable_timing", "dxg_gmm_kernel_times",
]
GMM_KERNELS = ["dx_gmm_absmax", "dx_gmm_prep_q", "dx_gmm_prep_x", "dx_gmm_fwd", "dx_gmm_lse", "dx_gmm_sum", "dx_gmm_bwd",
               "dx_gmm_moments", "dx_gmm_finish"]


def _check(rc: int):
    if rc != DXC_OK:
        raise DexError(rc, _lib.dxc_last_error().decode(errors="replace"))


def lib() -> ctypes.CDLL:
    return _lib.load()


def loaded() -> bool:
    """Whether libdexlet_cuda.so has been mapped into this process."""
    return _lib._cdll is not None


def gmm_program_match(source: str):
    """(n, d, K, gamma, m) when `source` is the canonical ADBench GMM program
    (programs.gmm_program), else None."""
    n, d, k, m = ctypes.c_int64(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    g = ctypes.c_double()
    if not _lib.dxl_gmm_program_match(source.encode(), ctypes.byref(n), ctypes.byref(d), ctypes.byref(k),
                                      ctypes.byref(g), ctypes.byref(m)):
        return None
    return n.value, d.value, k.value, g.value, m.value


def chunk_range(total: int, parts: int, c: int) -> Tuple[int, int]:
    """Contiguous chunk `c` of `parts` (reference eval.cpp:323-330)."""
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.dxc_chunk_range(total, parts, c, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def device_count() -> int:
    n = ctypes.c_int()
    rc = _lib.dxc_device_count(ctypes.byref(n))
    return n.value if rc == DXC_OK else 0


class Context:
    """One GPU: primary CUDA context + a stream (replaces the chunk threads)."""

    def __init__(self, device: int = 0):
        h = _vp()
        _check(_lib.dxc_init(device, ctypes.byref(h)))
        self.handle = h
        self.device = device

    @property
    def stream(self) -> int:
        return _lib.dxc_stream(self.handle)

    def sm_count(self) -> int:
        n = ctypes.c_int()
        _check(_lib.dxc_sm_count(self.handle, ctypes.byref(n)))
        return n.value

    def sync(self):
        _check(_lib.dxc_sync(self.handle))

    def event(self):
        e = _vp()
        _check(_lib.dxc_event_record(self.handle, ctypes.byref(e)))
        return e

    @staticmethod
    def elapsed_ms(e0, e1) -> float:
        ms = ctypes.c_float()
        _check(_lib.dxc_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
        return ms.value

    @staticmethod
    def destroy_event(e):
        _lib.dxc_event_destroy(e)

    def capture(self, fn):
        """Run fn() with the context stream captured; returns a graph handle
        replayed by graph_launch (every launch fn issued, in order)."""
        _check(_lib.dxc_capture_begin(self.handle))
        try:
            fn()
        finally:
            g = _vp()
            rc = _lib.dxc_capture_end(self.handle, ctypes.byref(g))
        _check(rc)
        return g

    def graph_launch(self, g):
        _check(_lib.dxc_graph_launch(self.handle, g))

    @staticmethod
    def graph_destroy(g):
        _check(_lib.dxc_graph_destroy(g))

    def l2_flush(self, nbytes: int = 256 << 20):
        """Overwrite a scratch buffer larger than the 126 MB L2 (on our stream)."""
        _check(_lib.dxc_l2_flush(self.handle, nbytes))

    def init_comm(self, unique_id: bytes, nranks: int, rank: int):
        buf = ctypes.create_string_buffer(unique_id, 128)
        _check(_lib.dxc_comm_init(self.handle, buf, nranks, rank))

    def close(self):
        if self.handle:
            _lib.dxc_destroy(self.handle)
            self.handle = None


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.dxc_nccl_unique_id(buf))
    return buf.raw


_NP_DT = {DXC_F32: np.float32, DXC_F64: np.float64, DXC_I32: np.int32, DXC_I64: np.int64,
          DXC_U32: np.uint32}
_DT_OF = {np.dtype(np.float32): DXC_F32, np.dtype(np.float64): DXC_F64, np.dtype(np.int32): DXC_I32,
          np.dtype(np.int64): DXC_I64, np.dtype(np.uint32): DXC_U32}


class Program:
    """A dexlet program lowered for the device.

    ``source`` defines ``entry = \\x1:T1. ... \\xk:Tk. body``; inputs are the
    lambda parameters, flattened to SoA leaves (a table of pairs is a pair of
    tables), row-major by index-set ordinal.  Index leaves are ordinals.
    """

    def __init__(self, source: str, entry: str = "main", ctx: Optional[Context] = None,
                 float64: bool = False, rank: int = 0, world: int = 1, threads: int = 0,
                 flags: int = 0):
        opts = DxlOptions(1 if float64 else 0, rank, world, threads, flags)
        h = _vp()
        entry = entry or ""  # "" / None: the whole file (its final expression, no inputs)
        _check(_lib.dxl_program_create(ctx.handle if ctx else None, source.encode(), entry.encode(),
                                       ctypes.byref(opts), ctypes.byref(h)))
        self.handle = h
        self.ctx = ctx
        self.float64 = float64

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _lib.dxl_program_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    @property
    def source(self) -> str:
        return _lib.dxl_program_source(self.handle).decode()

    @property
    def plan(self) -> str:
        return _lib.dxl_program_plan(self.handle).decode()

    def num_launches(self) -> int:
        n = ctypes.c_int()
        _check(_lib.dxl_program_num_launches(self.handle, ctypes.byref(n)))
        return n.value

    def enable_kernel_timing(self, on: bool = True):
        _check(_lib.dxl_program_enable_kernel_timing(self.handle, 1 if on else 0))

    def kernel_times(self):
        """[(kernel name, ms)] of the last run (CUDA events inside the graph)."""
        cap = 256
        arr = (ctypes.c_float * cap)()
        n = ctypes.c_int()
        _check(_lib.dxl_program_kernel_times(self.handle, arr, cap, ctypes.byref(n)))
        names = _lib.dxl_program_kernel_names(self.handle).decode().split("\n")
        return [(names[i], arr[i]) for i in range(min(n.value, cap))]

    def input_leaves(self) -> List[List[Tuple[int, int]]]:
        n = ctypes.c_int()
        _check(_lib.dxl_program_num_inputs(self.handle, ctypes.byref(n)))
        out = []
        for i in range(n.value):
            m = ctypes.c_int()
            _check(_lib.dxl_program_input_num_leaves(self.handle, i, ctypes.byref(m)))
            leaves = []
            for l in range(m.value):
                k, c = ctypes.c_int(), ctypes.c_int64()
                _check(_lib.dxl_program_input_leaf(self.handle, i, l, ctypes.byref(k), ctypes.byref(c)))
                leaves.append((k.value, c.value))
            out.append(leaves)
        return out

    def output_leaves(self) -> List[Tuple[int, int]]:
        n = ctypes.c_int()
        _check(_lib.dxl_program_output_num_leaves(self.handle, ctypes.byref(n)))
        out = []
        for l in range(n.value):
            k, c = ctypes.c_int(), ctypes.c_int64()
            _check(_lib.dxl_program_output_leaf(self.handle, l, ctypes.byref(k), ctypes.byref(c)))
            out.append((k.value, c.value))
        return out

    def set_input(self, i: int, leaf: int, arr: np.ndarray):
        arr = np.ascontiguousarray(arr)
        dt = _DT_OF.get(arr.dtype)
        if dt is None:
            raise DexError(DXC_E_ARG, f"input {i} leaf {leaf}: unsupported dtype {arr.dtype}")
        _check(_lib.dxl_program_set_input_n(self.handle, i, leaf, arr.ctypes.data_as(_vp), dt, arr.size))

    def set_input_rows(self, i: int, leaf: int, rows: np.ndarray, row_lo: int):
        """Upload a rank-local shard: `rows` are rows [row_lo, row_lo + len)
        of the leaf's leading dimension, in the leaf's storage dtype
        (float32 / float64 in f64 mode, int32 for index leaves)."""
        rows = np.ascontiguousarray(rows)
        dt = _DT_OF.get(rows.dtype)
        if dt is None:
            raise DexError(DXC_E_ARG, f"input {i} leaf {leaf}: unsupported dtype {rows.dtype}")
        n = rows.shape[0] if rows.ndim else 0
        _check(_lib.dxl_program_set_input_rows(self.handle, i, leaf, rows.ctypes.data_as(_vp), dt, row_lo,
                                               row_lo + n))

    def set_input_rows_ptr(self, i: int, leaf: int, host_ptr: int, dtype: int, row_lo: int, row_hi: int):
        _check(_lib.dxl_program_set_input_rows(self.handle, i, leaf, _vp(host_ptr), dtype, row_lo, row_hi))

    def counters(self) -> dict:
        """EvalCounters of the last run (programs created with DXL_F_COUNT)."""
        out = (ctypes.c_longlong * 4)()
        _check(_lib.dxl_program_counters(self.handle, out))
        return {"arithmeticOps": out[0], "accumUpdates": out[1], "cellsAllocated": out[2],
                "nodesEvaluated": out[3]}

    def check(self):
        """Raise DexError(E-bounds) if an index check failed (synchronizes)."""
        _check(_lib.dxl_program_check(self.handle))

    def set_input_ptr(self, i: int, leaf: int, host_ptr: int, dtype: int):
        _check(_lib.dxl_program_set_input(self.handle, i, leaf, _vp(host_ptr), dtype))

    def bind_input_device(self, i: int, leaf: int, devptr: int):
        _check(_lib.dxl_program_bind_input_device(self.handle, i, leaf, _vp(devptr)))

    def input_device_ptr(self, i: int, leaf: int) -> int:
        p = _vp()
        _check(_lib.dxl_program_input_device_ptr(self.handle, i, leaf, ctypes.byref(p)))
        return p.value or 0

    def output_device_ptr(self, leaf: int) -> int:
        p = _vp()
        _check(_lib.dxl_program_output_device_ptr(self.handle, leaf, ctypes.byref(p)))
        return p.value or 0

    def run(self):
        _check(_lib.dxl_program_run(self.handle))

    def get_output(self, leaf: int, dtype: int = DXC_F64) -> np.ndarray:
        kinds = self.output_leaves()
        k, c = kinds[leaf]
        out = np.empty(c, dtype=_NP_DT[dtype])
        _check(_lib.dxl_program_get_output(self.handle, leaf, out.ctypes.data_as(_vp), dtype))
        return out

    def get_output_ptr(self, leaf: int, host_ptr: int, dtype: int):
        _check(_lib.dxl_program_get_output(self.handle, leaf, _vp(host_ptr), dtype))

    def __call__(self, *inputs: Sequence[np.ndarray]) -> List[np.ndarray]:
        """Run with one list of leaf arrays per input; returns output leaves
        (floats as f64, ints/indices as i64)."""
        for i, leaves in enumerate(inputs):
            if isinstance(leaves, np.ndarray):
                leaves = [leaves]
            for l, a in enumerate(leaves):
                self.set_input(i, l, a)
        self.run()
        res = []
        for l, (k, c) in enumerate(self.output_leaves()):
            res.append(self.get_output(l, DXC_F64 if k == LEAF_FLOAT else DXC_I64))
        return res


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


class GMM:
    """Fused GMM objective + gradient on the device (include/dexlet_gmm.h):
    ADBench's ``gmm_objective(d, k, n, alphas, means, icf, x, wishart, err)``
    and its gradient, 1 <= d <= 64 (d < 64 exactly zero-padded to the 64-wide
    kernels), fp32 inputs, fp64 results.  ``n_global`` is the
    total point count when this rank holds a contiguous shard of the points."""

    def __init__(self, ctx: Context, d: int, k: int, n: int, n_global: Optional[int] = None):
        h = _vp()
        _check(_lib.dxg_gmm_create(ctx.handle, d, k, n, n if n_global is None else n_global, ctypes.byref(h)))
        self.handle, self.ctx, self.d, self.k, self.n = h, ctx, d, k, n

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _lib.dxg_gmm_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def set_params(self, alphas, means, icf):
        self._keep = [np.ascontiguousarray(a, dtype=np.float32) for a in (alphas, means, icf)]
        _check(_lib.dxg_gmm_set_params(self.handle, *(_ptr(a) for a in self._keep)))

    def set_points(self, x):
        self._x = np.ascontiguousarray(x, dtype=np.float32)
        _check(_lib.dxg_gmm_set_points(self.handle, _ptr(self._x)))

    def set_params_ptr(self, alphas: int, means: int, icf: int):
        _check(_lib.dxg_gmm_set_params(self.handle, _vp(alphas), _vp(means), _vp(icf)))

    def set_points_ptr(self, x: int):
        _check(_lib.dxg_gmm_set_points(self.handle, _vp(x)))

    def run(self, gamma: float = 1.0, m: int = 0, grad: bool = True):
        _check(_lib.dxg_gmm_run(self.handle, gamma, m, 1 if grad else 0))

    def enable_timing(self, on: bool = True):
        _check(_lib.dxg_gmm_enable_timing(self.handle, 1 if on else 0))

    def kernel_times(self):
        arr = (ctypes.c_float * 16)()
        n = ctypes.c_int()
        _check(_lib.dxg_gmm_kernel_times(self.handle, arr, 16, ctypes.byref(n)))
        return [(GMM_KERNELS[i], arr[i]) for i in range(n.value)]

    def get(self, grad: bool = True):
        err = np.zeros(1)
        if not grad:
            _check(_lib.dxg_gmm_get(self.handle, _ptr(err), None, None, None))
            return float(err[0])
        icf_sz = self.d * (self.d + 1) // 2
        da = np.empty(self.k)
        dm = np.empty((self.k, self.d))
        di = np.empty((self.k, icf_sz))
        _check(_lib.dxg_gmm_get(self.handle, _ptr(err), _ptr(da), _ptr(dm), _ptr(di)))
        return float(err[0]), da, dm, di

    def __call__(self, alphas, means, icf, x, gamma: float = 1.0, m: int = 0, grad: bool = True):
        self.set_params(alphas, means, icf)
        self.set_points(x)
        self.run(gamma, m, grad)
        return self.get(grad)
