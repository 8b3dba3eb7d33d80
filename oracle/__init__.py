"""ORACLE / TEST INFRASTRUCTURE ONLY.

Checkers for the device backend.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` legs may import this
package, and only as the thing checked against or timed beside -- never as the
product path.

* :class:`RefProgram` -- the unmodified reference evaluator (``evalExpr``,
  /root/reference/proj/src/eval.cpp:621-633) compiled from the reference's own
  sources by ``oracle/Makefile`` into ``oracle/_ref/libdexlet_ref.so``, driven
  through a C-ABI harness (``oracle/ref_harness.cpp``) with inputs bound as
  runtime env values exactly like the reference's tests.
* :mod:`oracle.restate` -- fp64 numpy restatements of the benchmark programs
  for full-size parity where the reference is too slow (validated against
  :class:`RefProgram` at reduced sizes in tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libdexlet_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def _load():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{REF_LIB} missing: run `make -C oracle` where /root/reference exists")
        lib = ctypes.CDLL(REF_LIB)
        vp, ip, i64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64)
        lib.dxo_last_error.restype = ctypes.c_char_p
        lib.dxo_program_create.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(vp)]
        lib.dxo_program_destroy.argtypes = [vp]
        lib.dxo_program_num_inputs.argtypes = [vp]
        lib.dxo_program_input_num_leaves.argtypes = [vp, ctypes.c_int]
        lib.dxo_program_input_leaf.argtypes = [vp, ctypes.c_int, ctypes.c_int, ip, i64p]
        lib.dxo_program_set_input_f64.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp]
        lib.dxo_program_set_input_i64.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp]
        lib.dxo_program_run.argtypes = [vp, ctypes.c_int, vp, ctypes.POINTER(ctypes.c_double)]
        lib.dxo_program_num_outputs.argtypes = [vp]
        lib.dxo_program_output_leaf.argtypes = [vp, ctypes.c_int, ip, i64p]
        lib.dxo_program_get_output_f64.argtypes = [vp, ctypes.c_int, vp]
        lib.dxo_program_ir.argtypes = [vp]
        lib.dxo_program_ir.restype = ctypes.c_char_p
        lib.dxo_run_source.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t]
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"oracle status {code}: {message}")
        self.code = code
        self.message = message


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, _load().dxo_last_error().decode(errors="replace"))


class RefProgram:
    """The reference evaluator on a program ``entry = \\x1:T1. ... body``."""

    def __init__(self, source: str, entry: str = "main"):
        lib = _load()
        h = ctypes.c_void_p()
        _check(lib.dxo_program_create(source.encode(), entry.encode(), ctypes.byref(h)))
        self.h = h
        self.counters = None
        self.ms = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _load().dxo_program_destroy(self.h)
        except Exception:
            pass

    @property
    def ir(self) -> str:
        return _load().dxo_program_ir(self.h).decode()

    def input_leaves(self):
        lib = _load()
        out = []
        for i in range(lib.dxo_program_num_inputs(self.h)):
            leaves = []
            for l in range(lib.dxo_program_input_num_leaves(self.h, i)):
                k, c = ctypes.c_int(), ctypes.c_int64()
                lib.dxo_program_input_leaf(self.h, i, l, ctypes.byref(k), ctypes.byref(c))
                leaves.append((k.value, c.value))
            out.append(leaves)
        return out

    def __call__(self, *inputs, chunks: int = 1) -> List[np.ndarray]:
        lib = _load()
        kinds = self.input_leaves()
        for i, leaves in enumerate(inputs):
            if isinstance(leaves, np.ndarray):
                leaves = [leaves]
            for l, a in enumerate(leaves):
                k, c = kinds[i][l]
                if k == 0:
                    arr = np.ascontiguousarray(a, dtype=np.float64).ravel()
                    assert arr.size == c, (i, l, arr.size, c)
                    _check(lib.dxo_program_set_input_f64(self.h, i, l, arr.ctypes.data_as(ctypes.c_void_p)))
                else:
                    arr = np.ascontiguousarray(a, dtype=np.int64).ravel()
                    assert arr.size == c, (i, l, arr.size, c)
                    _check(lib.dxo_program_set_input_i64(self.h, i, l, arr.ctypes.data_as(ctypes.c_void_p)))
        cnt = (ctypes.c_int64 * 4)()
        ms = ctypes.c_double()
        _check(lib.dxo_program_run(self.h, chunks, cnt, ctypes.byref(ms)))
        self.counters = dict(arithmeticOps=cnt[0], accumUpdates=cnt[1], cellsAllocated=cnt[2],
                             nodesEvaluated=cnt[3])
        self.ms = ms.value
        res = []
        for l in range(lib.dxo_program_num_outputs(self.h)):
            k, c = ctypes.c_int(), ctypes.c_int64()
            lib.dxo_program_output_leaf(self.h, l, ctypes.byref(k), ctypes.byref(c))
            out = np.empty(c.value, dtype=np.float64)
            lib.dxo_program_get_output_f64(self.h, l, out.ctypes.data_as(ctypes.c_void_p))
            res.append(out if k.value == 0 else out.astype(np.int64))
        return res


def run_source(source: str, chunks: int = 1) -> str:
    """Whole-file run like the reference tests' runSimpl; printResult text."""
    lib = _load()
    buf = ctypes.create_string_buffer(1 << 20)
    _check(lib.dxo_run_source(source.encode(), chunks, buf, len(buf)))
    return buf.value.decode()


def rel_diff(a: np.ndarray, b: np.ndarray) -> float:
    """max |a-b| / (1 + max(|a|,|b|)) -- rtMaxRelDiff (eval.cpp:758-763)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return float("inf")
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / (1.0 + np.maximum(np.abs(a), np.abs(b)))))
