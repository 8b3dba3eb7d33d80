// dexlet_device.hpp — C++ host API of the B200 backend, the device twin of the
// reference evaluator's entry point
//
//   RtPtr evalExpr(const EnvPtr&, const ExprPtr&, const EvalOptions& = {},
//                  EvalCounters* = nullptr);              // reference eval.hpp:74-75
//
// evalExprDevice takes the same post-optimize, first-order expression
// (isFirstOrder, reference simplify.hpp:32) and the same runtime environment
// of boxed RtVal values (reference eval.hpp:17-51), lowers every for /
// runAccum nest to sm_100a kernels and returns the result as the same boxed
// RtVal tree.  Errors are DexError with the reference's ErrCodes
// (reference errors.hpp:10-108); there is no CPU fallback.
#pragma once

#include "dexlet/eval.hpp"
#include "dexlet/ir.hpp"

namespace dexlet {

struct DeviceOptions {
  int device = 0;        // CUDA device ordinal
  bool float64 = false;  // Float arithmetic in f64 (parity mode) instead of f32
  int rank = 0;          // multi-GPU: this process's shard (see dxl_options)
  int world = 1;         // number of GPUs sharing every outer loop
};

// The device counterpart of evalExpr.  With `counters`, the program is
// lowered in count mode (DXL_F_COUNT) and arithmeticOps / accumUpdates /
// cellsAllocated receive the work the lowered program executes (the
// reference's units: one per evaluated + - * /, one per `+=`, one per
// runAccum / runState cell); nodesEvaluated stays untouched (no IR walk).
// The reference acceptance gate's work criteria (acceptance.cpp:459-569)
// run on these counts (tests/test_gpu_full.py::test_work_criteria_*).
RtPtr evalExprDevice(const EnvPtr& env, const ExprPtr& e, const DeviceOptions& opts = {},
                     EvalCounters* counters = nullptr);

}  // namespace dexlet
