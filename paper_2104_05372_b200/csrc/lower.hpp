// Device lowering of first-order dexlet IR (the output of the reference's
// optimize(), proj/src/simplify.cpp:1107-1111) into a plan of sm_100a kernels.
//
// This is the B200 replacement of Interp (proj/src/eval.cpp:93-546): instead
// of walking the boxed RtVal tree per iteration, every host-level `for` /
// `runAccum` nest becomes one generated CUDA kernel (built on the hand-written
// primitives of dx_device.cuh) over flat SoA buffers.
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "dexlet/index_set.hpp"
#include "dexlet/ir.hpp"

namespace dexlet {
namespace dev {

// Storage kinds of plan buffers.
// Float (f32|f64 per mode), Int (i64), Index (i32), counters, and D: Float
// Accum/State cells, always f64 in HBM (the reference accumulates in double).
enum class SK { F, I, X, U32, D };

// Resolved device type of a value (index-set sizes concrete).
struct DType;
using DTy = std::shared_ptr<const DType>;
struct DType {
  enum K { Float, Int, Unit, Idx, Pair, Table, Ref, Sum } k;  // Sum: data Either (a | b)
  DescPtr desc;  // Idx: its index set; Table: its domain
  DTy a, b;      // Pair/Sum: components; Table: a = element; Ref: a = payload
};

struct LeafInfo {
  SK kind;
  long long count;  // scalars of this leaf per value
  DescPtr desc;     // Idx leaves: the index set of the member
};
void leavesOf(const DTy& t, std::vector<LeafInfo>& out, long long mult = 1);
std::string showType(const DTy& t);

struct BufDecl {
  enum Role { Input, Cell, Output, Partial, Const, Temp, Flag, Sync } role;  // Sync: zeroed once, persistent
  SK kind;
  long long elems;
  int input = -1, leaf = -1;
  std::vector<double> initF;     // Const / host-known cell values (Float)
  std::vector<long long> initI;  // Const (Int / Index)
  long long partialWidth = 0;    // Partial: elements per block (sized at prepare)
  int partialKernel = -1;        // Partial: the step index of its kernel
};

struct KArg {
  enum K { Buf, I64, TMap } k;
  int buf = -1;
  long long off = 0;   // Buf: element offset
  long long i = 0;     // I64 value
  int special = 0;     // 1: range lo, 2: range hi
  // TMap: 2-D tensor map over buffer `buf` viewed as rows of `rowLen`
  // elements starting at element `off`; box = boxRows x rowLen; swizzle bytes
  long long rowLen = 0, rows = 0;
  int boxRows = 0, swizzle = 0;
  int boxCols = 0;     // box width in elements (0: the whole row)
  int f16 = 0;         // TMap over fp16 elements (2 bytes; the buffer is declared as U32 pairs)
};

struct Step {
  enum K { Zero, Upload, Kernel, Finalize, Allreduce, AddBuf, CopyBuf, Convert, Merge } k;
  int buf = -1, buf2 = -1;
  long long off = 0, off2 = 0, elems = 0;
  // Kernel
  std::string name;
  std::vector<KArg> args;
  long long total = 0;  // iterations of the outer loop (1 for serial)
  bool serial = false;
  bool sharded = false;
  int threads = 256;
  int smem = 0;           // dynamic shared memory bytes
  int minGrid = 0;        // ordinals per thread (U)
  bool warpRow = false;   // one warp per ordinal (32 threads per iteration)
  int grp = 0;            // group mode: G lanes per ordinal, minGrid ordinals per group and chunk
  bool coop = false;      // cooperative launch (in-kernel grid barrier + finalize)
  bool dead = false;      // Zero step taken over by the first kernel writing the buffer
  long long fixedGrid = 0;  // >0: launch exactly this many blocks (tile kernels: GEMM, transpose)
  // Finalize: partial buf -> cell (buf, off, elems = width)
  enum FinK { Seq, Tree, Count } fin = Seq;
  int kernelStep = -1;
  double scale = 1.0;
  // Merge: rank-ordered merge of per-rank Accum deltas into their cells (one
  // grouped NCCL all-gather into buf, then cell = ((cell + d_0) + d_1) + ...)
  struct MergeItem {
    int delta, cell;
    long long elems;
    long long rowN = 0, rowW = 0;  // Owner-only updates: rows of a rowN-ordinal range, rowW words each
  };
  std::vector<MergeItem> merge;
  std::string note;
  // Sharding dataflow (see dropLocalCollectives): the buffers a kernel step
  // reads; those it reads only at its own ordinal's row (buf -> row length,
  // base offset 0) over its shard of `total`; and, on an Allreduce of a
  // sharded kernel's map output, the row sharding of that buffer.
  bool rwKnown = false;
  std::set<int> readBufs;
  std::map<int, long long> rowReads;
  long long rowsOf = 0;        // rowReads are the rank's rows of this many ordinals
  std::set<int> rowBad;        // (lowering scratch) bufs read outside the own rows
  bool rowsShifted = false;    // fixed-grid kernel of a sharded contraction (rowReads valid)
  long long rowShardN = 0, rowShardW = 0;
  // Sharded kernels over several flattened dims: the shard is the chunk of
  // the first dim's ordinals times rowBlock (the product of the others), so
  // a rank's elements are whole rows of the first dim.
  long long rowBlock = 1;
};

struct OutLeaf {
  SK kind;
  long long count;
  DescPtr desc;           // index leaves
  bool host = false;      // value known on the host
  std::vector<double> hostF;
  std::vector<long long> hostI;
  int buf = -1;
  long long off = 0;
};

struct InLeaf {
  SK kind;
  long long count;
  DescPtr desc;
  int buf;
};

struct Plan {
  bool f64 = false;
  int rank = 0, world = 1;
  std::vector<BufDecl> bufs;
  std::vector<Step> steps;
  std::string source;           // generated kernels (device runtime prepended at compile)
  std::vector<std::vector<InLeaf>> inputs;
  std::vector<DTy> inputTypes;
  std::vector<Name> inputNames;
  std::vector<OutLeaf> outputs;
  DTy outputType;
  int errFlagBuf = -1;          // E-bounds flag raised by fused index checks
  int numKernels = 0;
  bool gemm = false;            // uses the tcgen05 contraction kernels (dx_gemm.cuh)
  // Work counters (EvalCounters, eval.hpp:60-65) in count mode: kernels add
  // the + - * / they execute and the += they perform into countBuf (2 x u64,
  // zeroed by the plan's first step); work the lowering did at build time or
  // replaced wholesale (host-folded arithmetic, accum-to-map broadcasts,
  // contraction GEMMs) is added as static per-run counts.
  int countBuf = -1;
  long long staticOps = 0, staticAccums = 0, cellsAllocated = 0;
  std::string summary() const;
};

struct LowerOptions {
  bool f64 = false;
  int rank = 0, world = 1;
  int threads = 256;
  bool noFusion = false;
  bool noRowScatter = false;
  bool noGemm = false;
  bool pipeline = false;  // DXL_F_PIPELINE: stream inputs before the PDL wait
  bool count = false;     // DXL_F_COUNT: count executed ops / accum updates
};

// Lowers `e` (first-order, post-optimize) whose free variables are the
// given inputs.  Throws DexError(Internal, ...) when a construct is not
// lowerable: there is no CPU fallback.
Plan lowerProgram(const ExprPtr& e, const std::vector<std::pair<Name, ValuePtr>>& inputs,
                  const LowerOptions& opts);

}  // namespace dev
}  // namespace dexlet
