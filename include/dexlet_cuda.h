/*
 * dexlet_cuda.h — C-ABI drop-in boundary of the B200 execution backend for the
 * data-parallel core (`for` / `runAccum` / `+=`) of the dexlet evaluator.
 *
 * The reference has no plugin hook: `Interp` lives in an anonymous namespace
 * (reference proj/src/eval.cpp:16,93) and the only entry points are the C++
 * functions of proj/include/dexlet/eval.hpp.  Each function below names the
 * reference interface it stands in for.  There are no C++ or torch types in
 * these signatures: plain pointers, sizes and integer status codes, so that
 * ctypes / cgo / JNI bindings can call them.
 *
 * Two levels:
 *   dxc_*  device runtime: context, buffers, modules, launches, collectives.
 *   dxl_*  program level: a dexlet program + input leaves in, output leaves
 *          out; the C-ABI form of `evalExpr(env, optimize(simplify(e)))`
 *          (reference eval.hpp:74-75, tests/acceptance.cpp:68-71).
 *
 * Status codes mirror dexlet::ErrCode (reference include/dexlet/errors.hpp:10-26):
 * no exceptions cross the ABI; the C++ host wrapper rethrows DexError.
 */
#ifndef DEXLET_CUDA_H
#define DEXLET_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (ErrCode mirror, errors.hpp:10-26) ---------------------- */
enum {
  DXC_OK = 0,
  DXC_E_PARSE = 1,        /* E-parse                                        */
  DXC_E_TYPE = 4,         /* E-type (and the other front-end codes 2..10)   */
  DXC_E_SIZE = 11,        /* E-size: index-set size not resolvable          */
  DXC_E_BOUNDS = 12,      /* E-bounds: ordinal outside its index set        */
  DXC_E_REF = 13,         /* E-ref                                          */
  DXC_E_PARALLEL = 14,    /* E-parallel: loop body blocks parallelism       */
  DXC_E_INTERNAL = 15,    /* E-internal: broken invariant / not lowerable   */
  DXC_E_CUDA = 100,       /* CUDA driver / NVRTC / NCCL failure             */
  DXC_E_ARG = 101         /* bad argument to an ABI call                    */
};

/* scalar kinds of flattened leaves (SoA, row-major by index-set ordinal,
 * reference index_set.cpp:74-97 / eval.cpp:683-697) */
enum {
  DXC_LEAF_FLOAT = 0,     /* Float  (reference: double)                      */
  DXC_LEAF_INT = 1,       /* Int    (reference: long long)                   */
  DXC_LEAF_INDEX = 2      /* index-set member, stored as its ordinal         */
};

/* host element types accepted / produced at the boundary */
enum { DXC_F32 = 0, DXC_F64 = 1, DXC_I32 = 2, DXC_I64 = 3, DXC_U32 = 4 };

typedef struct dxc_ctx dxc_ctx;
typedef struct dxc_buf dxc_buf;
typedef struct dxc_module dxc_module;
typedef struct dxl_program dxl_program;

/* Last error message of the calling thread ("" when none). */
const char* dxc_last_error(void);

/* ---- device runtime ------------------------------------------------------- */
/* Replaces: the std::thread fork-join executor of Interp::parallelFor
 * (eval.cpp:310-369).  One context per GPU, one stream per context. */
int dxc_init(int device, dxc_ctx** out);
int dxc_destroy(dxc_ctx* ctx);
int dxc_device_count(int* out);
int dxc_sm_count(dxc_ctx* ctx, int* out);
/* The stream all work of this context is issued on (a CUstream). */
void* dxc_stream(dxc_ctx* ctx);
int dxc_sync(dxc_ctx* ctx);

/* Device buffers.  Replaces the boxed RTable/RScalar heap (eval.hpp:36-51)
 * with flat SoA storage; the library owns the memory. */
int dxc_buf_alloc(dxc_ctx* ctx, size_t bytes, dxc_buf** out);
int dxc_buf_free(dxc_buf* buf);
void* dxc_buf_ptr(dxc_buf* buf);
int dxc_buf_upload(dxc_buf* buf, size_t offset, const void* host, size_t bytes);
int dxc_buf_download(dxc_buf* buf, size_t offset, void* host, size_t bytes);
int dxc_buf_zero(dxc_buf* buf);
/* Page-locked host memory for end-to-end (host buffer) runs. */
int dxc_host_alloc(size_t bytes, void** out);
int dxc_host_free(void* p);

/* Modules: CUDA C++ source compiled for sm_100a by NVRTC (cached by hash).
 * The generated per-nest kernels are built on the hand-written device
 * runtime (dx_device.cuh) that the library prepends. */
int dxc_module_compile(dxc_ctx* ctx, const char* source, dxc_module** out);
int dxc_module_cubin(const char* source, void* out, size_t cap, size_t* size);
int dxc_launch(dxc_ctx* ctx, dxc_module* mod, const char* kernel, unsigned grid,
               unsigned block, unsigned smem, void** args);

/* Writes `bytes` of a context-owned scratch buffer on the context stream:
 * evicts the 126 MB L2 between timed iterations of a benchmark. */
int dxc_l2_flush(dxc_ctx* ctx, size_t bytes);

/* Events on the context stream (device-side timing). */
int dxc_event_record(dxc_ctx* ctx, void** ev);
/* Capture everything issued on the context stream between begin and end
 * (e.g. K dxl_program_run calls) into one instantiated CUDA graph. */
int dxc_capture_begin(dxc_ctx* ctx);
int dxc_capture_end(dxc_ctx* ctx, void** graph_exec);
int dxc_graph_launch(dxc_ctx* ctx, void* graph_exec);
int dxc_graph_destroy(void* graph_exec);
int dxc_event_elapsed_ms(void* ev0, void* ev1, float* ms);
int dxc_event_destroy(void* ev);

/* Collectives: replaces the left-to-right addRt merge of chunk overlays
 * (eval.cpp:357-366) across GPUs.  NCCL is loaded at run time (the copy
 * torch already mapped when present).  unique_id is 128 bytes. */
int dxc_nccl_unique_id(void* out128);
int dxc_comm_init(dxc_ctx* ctx, const void* unique_id128, int nranks, int rank);
int dxc_allreduce_sum(dxc_ctx* ctx, void* devptr, size_t count, int dtype);

/* ---- program level -------------------------------------------------------- */
/* Options for dxl_program_create.  Mirrors EvalOptions (eval.hpp:67-69): the
 * reference's `chunks` becomes (rank, world) sharding of every outermost
 * parallel loop, contiguous ranges by the chunk rule of eval.cpp:323-330. */
typedef struct dxl_options {
  int float64;      /* 1: Float computes in f64 (parity mode); 0: f32      */
  int rank;         /* this process's shard (0 when world == 1)            */
  int world;        /* number of GPUs sharing every outer loop             */
  int threads;      /* threads per block for parallel nests (0 = 256)      */
  int flags;        /* DXL_F_* below                                       */
} dxl_options;

enum {
  DXL_F_NO_FUSION = 1,     /* materialize every pure loop (debug)           */
  DXL_F_NO_ROWSCATTER = 2, /* use smem atomics instead of warp row flushes  */
  DXL_F_DUMP = 4,          /* write generated CUDA to $DEXLET_DUMP_DIR      */
  DXL_F_TEST_COMM_MISMATCH = 8, /* TEST ONLY: run a (world, rank) plan over a
                                 * communicator of another size (one device
                                 * emulating the ranks); never in production */
  DXL_F_NO_GEMM = 16,      /* contractions (and the canonical GMM program)
                            * through the generic SIMT lowering              */
  DXL_F_COUNT = 64,        /* count work like EvalCounters (eval.hpp:60-65):
                            * executed + - * /, accum updates, cells; read
                            * with dxl_program_counters.  Diagnostics mode:
                            * contractions use the generic (counted) kernels */
  DXL_F_PIPELINE = 32      /* back-to-back runs may overlap: a kernel that
                            * reads only program inputs streams them before
                            * waiting (griddepcontrol.wait) for the previous
                            * launch on the context stream.  The caller
                            * promises that no kernel on that stream writes
                            * the inputs while runs are in flight (host
                            * uploads through set_input are stream-ordered
                            * and always safe).                              */
};

/* Parse, typecheck, simplify, optimize and lower `entry` of `source`, where
 * entry = \x1:T1. ... \xk:Tk. body with literal Fin sizes in the Ti.
 * Reference path: parseProgram (parser.cpp:1651), checkExpr (typecheck.cpp:578),
 * simplify + optimize (simplify.cpp:1081,1107), then — instead of
 * evalExpr (eval.cpp:621) — device lowering of every for/runAccum nest.
 * entry NULL or "": the whole file (declarations around its final
 * expression, no inputs), as the reference harness's runSimpl evaluates it
 * (tests/acceptance.cpp:68-71).
 * ctx may be NULL: lower and compile only (no device needed). */
int dxl_program_create(dxc_ctx* ctx, const char* source, const char* entry,
                       const dxl_options* opts, dxl_program** out);
int dxl_program_destroy(dxl_program* p);

int dxl_program_num_inputs(dxl_program* p, int* out);
int dxl_program_input_num_leaves(dxl_program* p, int input, int* out);
int dxl_program_input_leaf(dxl_program* p, int input, int leaf, int* kind,
                           int64_t* count);
int dxl_program_output_num_leaves(dxl_program* p, int* out);
int dxl_program_output_leaf(dxl_program* p, int leaf, int* kind, int64_t* count);

/* Input leaves: copied from host memory (dtype DXC_*), or bound zero-copy to
 * device memory already holding the leaf in the program's storage type
 * (f32 or f64 for Float per options.float64, i32 for Index, i64 for Int).
 * `host` must hold the leaf's element count (dxl_program_input_leaf);
 * dxl_program_set_input_n takes that count and returns E-size on mismatch.
 * Index leaves uploaded from host memory are range-checked on the device
 * right after the upload (the check fromOrdinal performs in the reference,
 * index_set.cpp:99-106); device-bound index leaves are checked (and clamped)
 * by the kernels that read them.  Either violation is reported as E-bounds
 * by dxl_program_get_output and by dxl_program_check. */
int dxl_program_set_input(dxl_program* p, int input, int leaf, const void* host,
                          int dtype);
/* Rank-local input shards: host holds only rows [row_lo, row_hi) of the
 * leaf's leading table dimension (row-major, the leaf's storage type); they
 * are uploaded into those rows of the device leaf.  A sharded plan reads an
 * input only at its own rows when its kernels do (the plan dump marks such
 * reads), so each rank uploads its chunk (dxc_chunk_range) instead of the
 * whole input. */
int dxl_program_set_input_rows(dxl_program* p, int input, int leaf, const void* host, int dtype, int64_t row_lo,
                               int64_t row_hi);
int dxl_program_set_input_n(dxl_program* p, int input, int leaf, const void* host,
                            int dtype, int64_t count);
int dxl_program_bind_input_device(dxl_program* p, int input, int leaf,
                                  void* devptr);
int dxl_program_input_device_ptr(dxl_program* p, int input, int leaf, void** out);

/* Executes the lowered plan asynchronously on the context stream. */
int dxl_program_run(dxl_program* p);
/* Synchronizes the stream and returns E-bounds if any index check (upload
 * or in-kernel) failed since the leaves were set; DXC_OK otherwise. */
/* 1 when `source` is the canonical ADBench GMM program (programs.gmm_program:
 * that text, whitespace aside, for some sizes and Wishart (gamma, m)); then
 * dxl_program_create runs it on the fused GMM kernel class (dexlet_gmm.h)
 * when d = 64, f32, one rank.  Fills the recognized parameters. */
int dxl_gmm_program_match(const char* source, int64_t* n, int* d, int* k, double* gamma, int* m);
/* Work counters of the last run (DXL_F_COUNT programs): out[0] arithmetic
 * ops, out[1] accumulator updates, out[2] cells allocated, out[3]
 * nodesEvaluated (0: there is no IR walk on the device).  Semantics of
 * EvalCounters (eval.hpp:60-65) as the lowered program executes them: host-
 * folded arithmetic and the broadcast updates an accum-to-map replaces are
 * added statically; a lazy element inlined once is counted once. */
int dxl_program_counters(dxl_program* p, long long* out4);
int dxl_program_check(dxl_program* p);
/* Copies an output leaf to host memory (synchronizes the stream). */
int dxl_program_get_output(dxl_program* p, int leaf, void* host, int dtype);
int dxl_program_output_device_ptr(dxl_program* p, int leaf, void** out);

/* Introspection: generated CUDA source, kernel count, per-run launch count,
 * text summary of the lowering plan. */
const char* dxl_program_source(dxl_program* p);
const char* dxl_program_plan(dxl_program* p);
int dxl_program_num_launches(dxl_program* p, int* out);
/* Per-kernel device time of the last run, from CUDA events recorded around
 * every kernel inside the (graph-captured) plan when timing was enabled
 * before the first run.  names: '\n'-separated kernel names. */
int dxl_program_enable_kernel_timing(dxl_program* p, int on);
int dxl_program_kernel_times(dxl_program* p, float* ms, int cap, int* n);
const char* dxl_program_kernel_names(dxl_program* p);

/* Index-set ordinal math (reference index_set.cpp:74-125), exported so host
 * bindings can lay out inputs exactly like the device does.  A descriptor is
 * a prefix string: "U" unit, "F<n>" Fin n, "P<a><b>" pair, "E<a><b>" either. */
int dxc_desc_size(const char* desc, int64_t* out);
int dxc_desc_reverse(const char* desc, int64_t ordinal, int64_t* out);
/* Chunk rule of eval.cpp:323-330: range [lo,hi) of part `c` of `parts`. */
int dxc_chunk_range(int64_t total, int parts, int c, int64_t* lo, int64_t* hi);

#ifdef __cplusplus
}
#endif

#endif /* DEXLET_CUDA_H */
