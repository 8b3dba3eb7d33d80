// Device lowering: first-order dexlet IR -> plan of generated sm_100a kernels.
//
// Semantics follow the reference evaluator node by node (proj/src/eval.cpp):
//   EFor       eval.cpp:295-308   -> a kernel over the index set (outermost
//                                    loop), or an in-thread loop (nested)
//   parallelFor eval.cpp:310-369  -> grid-stride sharding; (rank, world)
//                                    contiguous ranges by the chunk rule :323-330
//   ParScan    eval.cpp:548-600   -> blocksParallel(): State on outer cells
//                                    forces a single-thread (serial) kernel
//   runAccum   eval.cpp:437-464   -> zeroed cell (registers / smem / HBM)
//   EAccum     eval.cpp:482-492   -> strategy per cell: owner RMW, register
//                                    partials, smem privatized, warp row
//                                    flush, u32 counters, global red.add
//   ESlice     eval.cpp:390-396   -> offset arithmetic on the ref path
//   EIndex     eval.cpp:286-293   -> SoA load at the ordinal (or inlined view)
//   EBinOp/EUnOp eval.cpp:500-533 -> scalar C expressions
//   ordinal/fromOrdinal eval.cpp:683-723, index_set.cpp:74-125
//                                 -> row-major pair / left-first either math
// Pure loops are not materialized eagerly: like the reference's views they
// stay lazy and are inlined at unique (bijective) or cheap use sites, which
// fuses the forward "tape" loops that linearize emits (autodiff.cpp:230-255)
// into their transposed consumers (autodiff.cpp:705-717).

#include "lower.hpp"

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <functional>
#include <map>
#include <set>
#include <sstream>

#include "dexlet/errors.hpp"
#include "dexlet/printer.hpp"
#include "runtime.hpp"

namespace dexlet {
namespace dev {

[[noreturn]] static void notLowerable(const std::string& what, Span sp = {}) {
  fail(ErrCode::Internal, "not lowerable to the device: " + what, sp);
}

// ---------------------------------------------------------------------------
// Types.

static DescPtr boolDesc() {
  static DescPtr d = descEither(descUnit(), descUnit());
  return d;
}
static DTy mkT(DType::K k, DescPtr d = nullptr, DTy a = nullptr, DTy b = nullptr) {
  return std::make_shared<DType>(DType{k, std::move(d), std::move(a), std::move(b)});
}
static DTy tFloat() { static DTy t = mkT(DType::Float); return t; }
static DTy tInt() { static DTy t = mkT(DType::Int); return t; }
static DTy tUnit() { static DTy t = mkT(DType::Unit); return t; }
static DTy tIdx(DescPtr d) { return mkT(DType::Idx, std::move(d)); }
static DTy tPair(DTy a, DTy b) { return mkT(DType::Pair, nullptr, std::move(a), std::move(b)); }
static DTy tTable(DescPtr d, DTy e) { return mkT(DType::Table, std::move(d), std::move(e)); }
// Type of the table-of-pairs held as a Zip of `depth` table levels.
static DTy zipTy(const DTy& ta, const DTy& tb, int depth) {
  if (depth == 0) return tPair(ta, tb);
  return tTable(ta->desc, zipTy(ta->a, tb->a, depth - 1));
}
static DTy tRef(DTy p) { return mkT(DType::Ref, nullptr, std::move(p)); }
static DTy tSum(DTy a, DTy b) { return mkT(DType::Sum, nullptr, std::move(a), std::move(b)); }
// Is this core type an index set (Unit, Fin, pairs/sums of index sets)?
static bool isIndexSetType(const ValuePtr& t) {
  if (isBase(t, BaseKind::Unit)) return true;
  if (as<VFinType>(t)) return true;
  if (const auto* p = as<VPairType>(t)) return isIndexSetType(p->l) && isIndexSetType(p->r);
  if (const auto* e = as<VEitherType>(t)) return isIndexSetType(e->l) && isIndexSetType(e->r);
  return false;
}

static std::string showDesc(const DescPtr& d) {
  switch (d->kind) {
    case IndexSetDesc::Kind::Unit: return "Unit";
    case IndexSetDesc::Kind::Fin: return "Fin " + std::to_string(d->finSize);
    case IndexSetDesc::Kind::Pair: return "(" + showDesc(d->left) + " & " + showDesc(d->right) + ")";
    case IndexSetDesc::Kind::Either: return "Either (" + showDesc(d->left) + ") (" + showDesc(d->right) + ")";
  }
  return "?";
}

std::string showType(const DTy& t) {
  switch (t->k) {
    case DType::Float: return "Float";
    case DType::Int: return "Int";
    case DType::Unit: return "Unit";
    case DType::Idx: return showDesc(t->desc);
    case DType::Pair: return "(" + showType(t->a) + " & " + showType(t->b) + ")";
    case DType::Table: return "(" + showDesc(t->desc) + ") => " + showType(t->a);
    case DType::Ref: return "Ref " + showType(t->a);
    case DType::Sum: return "Either (" + showType(t->a) + ") (" + showType(t->b) + ")";
  }
  return "?";
}

// An index-set member is flattened like the reference's RtVal: a Fin member
// is its ordinal, a pair of members is a pair, an Either member is stored as
// its ordinal in the Either set (fromOrdinalRt rebuilds it, eval.cpp:699-723).
void leavesOf(const DTy& t, std::vector<LeafInfo>& out, long long mult) {
  if (!t) notLowerable("value of unknown element type (lazy table without annotation)");
  switch (t->k) {
    case DType::Float: out.push_back({SK::F, mult, nullptr}); return;
    case DType::Int: out.push_back({SK::I, mult, nullptr}); return;
    case DType::Unit: return;
    case DType::Idx:
      if (t->desc->kind == IndexSetDesc::Kind::Unit) return;
      out.push_back({SK::X, mult, t->desc});
      return;
    case DType::Pair: leavesOf(t->a, out, mult); leavesOf(t->b, out, mult); return;
    case DType::Table: leavesOf(t->a, out, mult * size(t->desc)); return;
    case DType::Ref: return;
    case DType::Sum:  // tag (0 = Left) then both payloads
      out.push_back({SK::X, mult, boolDesc()});
      leavesOf(t->a, out, mult);
      leavesOf(t->b, out, mult);
      return;
  }
}
static std::vector<LeafInfo> leaves(const DTy& t) {
  std::vector<LeafInfo> v;
  leavesOf(t, v);
  return v;
}
static size_t numLeaves(const DTy& t) { return leaves(t).size(); }

// Index-set member types: Fin/Either -> Idx; Pair -> Pair of members; Unit.
static DTy memberType(const DescPtr& d) {
  switch (d->kind) {
    case IndexSetDesc::Kind::Unit: return tUnit();
    case IndexSetDesc::Kind::Fin: return tIdx(d);
    case IndexSetDesc::Kind::Pair: return tPair(memberType(d->left), memberType(d->right));
    case IndexSetDesc::Kind::Either: return tIdx(d);
  }
  return tUnit();
}

static size_t storageBytesOf(SK k, bool f64 = false) {
  switch (k) {
    case SK::F: return f64 ? 8 : 4;
    case SK::I: return 8;
    case SK::D: return 8;
    default: return 4;
  }
}

// ---------------------------------------------------------------------------
// Small C-expression helpers (keep generated offsets folded).

static bool isIntLit(const std::string& s, long long* v = nullptr) {
  if (s.empty()) return false;
  size_t i = (s[0] == '-') ? 1 : 0;
  if (i >= s.size()) return false;
  for (size_t k = i; k < s.size(); ++k)
    if (s[k] < '0' || s[k] > '9') return false;
  if (v) *v = std::stoll(s);
  return true;
}
static std::string lit(long long v) { return std::to_string(v); }
static std::string eAdd(const std::string& a, const std::string& b) {
  long long x, y;
  bool ax = isIntLit(a, &x), by = isIntLit(b, &y);
  if (ax && by) return lit(x + y);
  if (ax && x == 0) return b;
  if (by && y == 0) return a;
  return "(" + a + " + " + b + ")";
}
static std::string eMul(const std::string& a, long long k) {
  long long x;
  if (k == 0) return "0";
  if (isIntLit(a, &x)) return lit(x * k);
  if (k == 1) return a;
  return "(" + a + " * " + lit(k) + "LL)";
}
static std::string eSub(long long k, const std::string& a) {
  long long x;
  if (isIntLit(a, &x)) return lit(k - x);
  return "(" + lit(k) + "LL - " + a + ")";
}
static std::string litF(double d, bool f64) {
  if (std::isinf(d)) return d > 0 ? (f64 ? "(1.0/0.0)" : "(1.0f/0.0f)") : (f64 ? "(-1.0/0.0)" : "(-1.0f/0.0f)");
  if (std::isnan(d)) return f64 ? "(0.0/0.0)" : "(0.0f/0.0f)";
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", d);
  std::string s = buf;
  if (s.find_first_of(".en") == std::string::npos) s += ".0";
  if (!f64) s = "((float)" + s + ")";
  return s;
}

// ---------------------------------------------------------------------------
// Host-level values: constants folded on the host, device buffers, refs into
// cells, and lazy (unmaterialized) pure loops.

struct HVal;
using HV = std::shared_ptr<const HVal>;
struct HEnvNode;
using HEnvP = std::shared_ptr<const HEnvNode>;
struct HEnvNode {
  Name n;
  HV v;
  HEnvP next;
};
static HEnvP hbind(HEnvP e, const Name& n, HV v) {
  return std::make_shared<HEnvNode>(HEnvNode{n, std::move(v), std::move(e)});
}
static HV hlookup(const HEnvP& e, const Name& n) {
  for (const HEnvNode* p = e.get(); p; p = p->next.get())
    if (p->n == n) return p->v;
  return nullptr;
}

struct LazyState {
  HV materialized;
  HV split;  // Zip: cheap components lazy, the rest materialized (splitMaterialize)
};

struct HVal {
  enum K { Const, Unit, Pair, Buf, Ref, Lazy, Zip } k;
  DTy ty;
  int zipDepth = 0;   // Zip: table levels above the pair (a, b: tables of its two halves)
  double f = 0;       // Const Float
  long long i = 0;    // Const Int / Idx ordinal
  HV a, b;            // Pair
  std::vector<int> bufs;           // Buf: per leaf
  std::vector<long long> offs;     // Buf / Ref: per-leaf element offsets
  int cell = -1;                   // Ref
  // Lazy pure loop `for binder:desc. body` closed over env
  Name binder;
  DescPtr desc;
  ExprPtr body;
  HEnvP env;
  bool cheap = false;
  std::shared_ptr<LazyState> st;
};

static HV hConstF(double v) {
  auto h = std::make_shared<HVal>(); h->k = HVal::Const; h->ty = tFloat(); h->f = v; return h;
}
static HV hConstI(long long v) {
  auto h = std::make_shared<HVal>(); h->k = HVal::Const; h->ty = tInt(); h->i = v; return h;
}
static HV hConstIdx(long long ord, DescPtr d) {
  if (d->kind == IndexSetDesc::Kind::Unit) {
    auto h = std::make_shared<HVal>(); h->k = HVal::Unit; h->ty = tUnit(); return h;
  }
  auto h = std::make_shared<HVal>(); h->k = HVal::Const; h->ty = tIdx(d); h->i = ord; return h;
}
static HV hUnit() {
  static HV u = [] { auto h = std::make_shared<HVal>(); h->k = HVal::Unit; h->ty = tUnit(); return HV(h); }();
  return u;
}
static HV hPair(HV a, HV b) {
  auto h = std::make_shared<HVal>(); h->k = HVal::Pair; h->ty = tPair(a->ty, b->ty);
  h->a = std::move(a); h->b = std::move(b); return h;
}

// Member value (host) for ordinal `o` of desc `d`, like fromOrdinalRt.
static HV hFromOrdinal(long long o, const DescPtr& d) {
  switch (d->kind) {
    case IndexSetDesc::Kind::Unit: return hUnit();
    case IndexSetDesc::Kind::Fin: return hConstIdx(o, d);
    case IndexSetDesc::Kind::Pair: {
      long long rs = size(d->right);
      return hPair(hFromOrdinal(o / rs, d->left), hFromOrdinal(o % rs, d->right));
    }
    case IndexSetDesc::Kind::Either: return hConstIdx(o, d);
  }
  return hUnit();
}
static bool hOrdinal(const HV& v, const DescPtr& d, long long* out) {
  switch (d->kind) {
    case IndexSetDesc::Kind::Unit: *out = 0; return true;
    case IndexSetDesc::Kind::Fin:
    case IndexSetDesc::Kind::Either:
      if (v->k != HVal::Const) return false;
      *out = v->i;
      return true;
    case IndexSetDesc::Kind::Pair: {
      if (v->k != HVal::Pair) return false;
      long long l, r;
      if (!hOrdinal(v->a, d->left, &l) || !hOrdinal(v->b, d->right, &r)) return false;
      *out = l * size(d->right) + r;
      return true;
    }
  }
  return false;
}

// ---------------------------------------------------------------------------
// Kernel-level values (codegen).

struct KVal;
using KV = std::shared_ptr<const KVal>;

struct Slot {
  std::string base;  // C pointer / array name
  std::string off;   // element offset expression
  int level = -1;    // deepest loop depth the offset depends on
  bool global = false;
  bool ro = false;
  bool input = false;  // Input buffer (index leaves get range-checked)
  int buf = -1;        // plan buffer (global) or -1
  SK kind = SK::F;
  long long align = 1; // offset is a multiple of this many elements
  int cellLeaf = -1;   // Ref slots into a global cell: which leaf of the cell
  // Streaming row: offset == (kernel ordinal) * streamL + streamBase + rowOff,
  // so the tile kernel can fetch the block's rows by TMA into shared memory.
  bool stream = false;
  long long streamL = 0, streamBase = 0;
  int streamU = 0;     // which of the thread's U ordinals (dx_o<u>)
  long long rowW = 0;  // indexed first by the kernel's dim-0 ordinal: within that row of rowW elements
  std::string rowOff;
};

static long long alignOf(long long c) {
  if (c == 0) return 1 << 20;
  long long a = 1;
  while ((c % (a * 2)) == 0 && a < (1 << 20)) a *= 2;
  return a;
}
static long long gcdll(long long a, long long b) {
  while (b) { long long t = a % b; a = b; b = t; }
  return a;
}

struct LazyK;
struct KEnvNode;
using KEnvP = std::shared_ptr<const KEnvNode>;
struct KEnvNode {
  Name n;
  KV v;
  KEnvP next;
};

struct KScope {
  KEnvP local;
  HEnvP host;
  std::set<int> covered;  // loops considered bound for lazies created here
  bool inBranch = false;
};

struct LazyK {
  Name binder;
  DescPtr desc;
  ExprPtr body;
  KScope scope;
  std::set<int> covered;
  bool cheap = false;
  uint64_t key = 0;
  HV hostOrigin;  // set when this is an imported host lazy
};

struct KVal {
  enum K { Scalar, Unit, Pair, Table, Ref, Lazy, Sum, Zip } k;
  DTy ty;
  int zipDepth = 0;   // Zip: table levels above the pair (a, b: the two halves)
  std::string e;      // Scalar expression; Sum: tag expression (0 = Left)
  int level = -1;
  bool isConst = false;
  double cf = 0;
  long long ci = 0;
  int loopId = -1;    // Idx: exactly loop var (or its reverse) of this loop
  std::string rev;    // Idx: cheaper expression of the reverse, if known
  std::string grpPart;  // group mode: e sums this local cell's per-lane partials (see closeLoop)
  KV a, b;
  std::vector<Slot> slots;  // Table / Ref, per leaf
  int cell = -1;            // Ref: plan cell (global) or -1 (local)
  std::vector<KV> path;     // Ref: indices sliced so far (inside the kernel)
  std::string prefixOff;    // Ref: offset before the last slice (leaf 0)
  int prefixLevel = -1;
  long long lastDim = 0;    // Ref: size of the last sliced domain
  std::shared_ptr<LazyK> lz;
};

static KV kUnit() {
  static KV u = [] { auto k = std::make_shared<KVal>(); k->k = KVal::Unit; k->ty = tUnit(); return KV(k); }();
  return u;
}
static KV kPair(KV a, KV b) {
  auto k = std::make_shared<KVal>(); k->k = KVal::Pair; k->ty = tPair(a->ty, b->ty);
  k->level = std::max(a->level, b->level);
  k->a = std::move(a); k->b = std::move(b); return k;
}
static KV kScalar(DTy ty, std::string e, int level) {
  auto k = std::make_shared<KVal>(); k->k = KVal::Scalar; k->ty = std::move(ty);
  k->e = std::move(e); k->level = level; return k;
}

// ---------------------------------------------------------------------------
// Cells (runAccum / runState handlers at host level).

struct Cell {
  DTy payload;
  std::vector<LeafInfo> lv;
  std::vector<int> bufs;
  bool accum = true;
  bool dirty = false;                     // device holds the value
  std::vector<std::vector<double>> host;  // host-known value per leaf (when !dirty)
  HV lazy;                                // value is this lazy table (accum-to-map)
};

// Per-kernel view of one cell leaf.
struct CellUse {
  int cell = -1, leaf = -1;
  enum Strat { Owner, Reg, Smem, Count, Row, TileRow, Global, Direct } strat = Global;
  // pass-0 analysis
  bool any = false, allOwner = true, allConst = true, allRow = true;
  double constVal = 0;
  bool haveConst = false;
  long long rowD = 0;
  int rowSitesN = 0;     // row-eligible accumulation sites (pass 0)
  bool vec4 = false;     // TileRow with float4 column blocks (f32, D % 4 == 0)
  bool warpTab = false;  // TileRow realised as warp-private tables (dx_warp_tab)
  bool ownRows = true;   // Owner accesses all at row dx_o0 (the rank's own rows when sharded)
  bool ownTop = true;    // Owner sites all unconditional at kernel level, at the ordinal's own element
  bool overwrite = false, firstDone = false;  // first site stores (the cell's zero-fill was dropped)
  std::string ownKey;    // the owner sites' element index (all sites must agree: ordinal o and n-1-o
                         // from two sites would be two threads' read-modify-writes of one element)
  int aliasStage = -1;   // TMA-staged stream buffer whose stage doubles as the row tile
  long long width = 0;
  int partialBuf = -1;
  int targetBuf = -1;   // cell leaf buffer or its delta (sharded)
  std::string pname;    // param name for target
  int smemOff = 0;
};

struct RowSite {
  int cu;        // CellUse index
  long long D;
  int id;
};

// ---------------------------------------------------------------------------

class Lowering;

struct KGen {
  Lowering& L;
  bool serial = false;
  bool sharded = false;
  long long total = 1;
  int pass = 0;           // 0: analysis (may repeat), 1: emission
  bool redo = false;
  std::set<uint64_t> matLocal;  // in-thread lazies to materialize
  std::string* out = nullptr;
  int ind = 1;
  int tmp = 0;
  int loopCounter = 0;
  std::vector<int> loopStack;     // active loop ids (kernel dims first)
  std::map<int, int> loopDepth;   // id -> depth (kernel dims depth 0)
  std::map<int, long long> loopTrip;
  std::vector<std::pair<int, KV>> kernelVars;  // kernel dims (loop id, binder value)
  std::map<int, std::string> params;  // buf -> param name
  std::set<int> writtenBufs;
  std::vector<CellUse> cells;
  std::map<std::pair<int, int>, int> cellIndex;
  std::vector<RowSite> rowSites;
  int rowSiteCounter = 0;
  int accumSiteCounter = 0;
  int U = 1;                      // ordinals per thread
  std::map<std::string, int> freshCell;  // local scalar Accum cells still zero -> loop depth
  int threads = 256;              // block size chosen for this kernel
  std::set<int> streamBufs;       // ro buffers read at exactly the ordinal
  std::set<int> stateCells;       // host-level State cells read/written (serial kernels)
  // TMA staging analysis (pass 0) and decisions (pass 1)
  std::map<int, std::pair<long long, long long>> streamUse;  // buf -> (row length, base offset)
  std::set<int> nonStream, needAlign;
  std::set<int> staged, wholeStaged;
  // group mode: whole-staged gather tables stored as 32/G interleaved copies
  // of each G-element row (group gi reads copy gi: no bank conflicts)
  std::set<int> grpInter;
  std::map<int, int> tensorStaged;  // buf -> swizzle mask (TMA 2-D with SWIZZLE_{32,64,128}B)
  bool tile = false;
  bool usesErr = false;
  bool usesScratch = false;
  int curBranch = 0;
  // Warp-per-ordinal mode for kernels whose outer loop is short and whose
  // body is a long reduction loop into local scalar cells (row sums): the
  // lanes split that loop and warp-sum the cells after it.
  bool warpRowOK = true;          // pass 0: nothing disqualifies the mode
  int laneLoopId = -1;            // pass 0: the reduction loop (depth 1, trip >= 64, effect-only)
  bool inCand = false;            // pass 0: inside the candidate loop's body
  bool warpRow = false;           // pass 1: emit in warp-per-ordinal mode
  bool inLaneLoop = false;        // pass 1: inside the lane loop's body
  std::set<std::string> innerCells, laneCells;  // local cells created in / reduced after the lane loop
  // Group mode (sub-warp per ordinal) for kernels whose in-thread loops all
  // run over one short index set of G = D members (k-means rows, D | 32):
  // G lanes share an ordinal, every depth-1 loop becomes "lane gl of the
  // group runs iteration gl", row scatters r!key!j become conflict-free
  // warp-private table updates, and the rows read at the ordinal stream in
  // coalesced (128 bytes per warp instruction) through a double-buffered
  // register prefetch.  Pass 0 decides eligibility; pass 1 emits.
  bool grpOK = true;              // pass 0: nothing disqualifies the mode
  long long grpTrip = 0;          // pass 0: trip of the depth-1 loops
  int grp = 0;                    // pass 1: G (0 = thread per ordinal)
  int grpU = 1;                   // pass 1: ordinals per group per chunk
  std::map<std::string, int> localDepth;      // local array -> loop depth at creation
  std::vector<std::set<std::string>> grpFresh; // per open lane loop: fresh scalar cells at entry
  std::vector<std::set<std::string>> grpSum;   // per open lane loop: outer cells to group-sum after it
  // stream rows read at (ordinal, lane column): the skeleton prefetches them
  // into registers gp<id>_<u> (pass 1), double-buffered across chunks
  struct GrpStream {
    int buf;
    long long L, base;
    std::string col;  // column expression in dx_gl
    SK kind;
    long long chk;    // index leaf of an input: range-checked (E-bounds) when prefetched
  };
  std::vector<GrpStream> grpStreams;
  std::set<int> grpStreamBad;
  int grpRowCell = -1;            // pass 1: the row cell's CellUse index
  std::map<std::string, KV> instMemo;  // kernel-level lazy instantiations of this iteration
  std::string dim0Ord;            // ordinal expression of the first kernel dim (this iteration)
  std::map<int, std::set<long long>> rowUse;  // pass 0: buf -> row widths of its dim-0-row reads
  std::set<int> rowBad;                       // pass 0: bufs also read elsewhere
  bool hasBranch = false;         // pass 0: the body branches (keeps group sums eager)
  std::map<std::string, int> grpPending;  // local cells holding per-lane partials (sum deferred)
  std::string curLaneVar;         // variable of the open depth-1 loop
  bool curLaneRev = false;        // ... which runs lane gl on iteration n-1-gl
  std::map<std::string, int> grpStreamId;  // "buf|column" -> prefetch stream id (pass 0 order)

  explicit KGen(Lowering& l) : L(l) {}

  int lines = 0;
  void line(const std::string& s) {
    ++lines;
    if (!out) return;
    out->append(ind * 2, ' ');
    out->append(s);
    out->push_back('\n');
  }
  std::string fresh(const char* p) { return std::string(p) + std::to_string(tmp++); }
  int depth() const { return loopStack.empty() ? 0 : loopDepth.at(loopStack.back()); }
};

class Lowering {
 public:
  LowerOptions opt;
  Plan plan;
  std::vector<Cell> cells;
  int kernelCounter = 0;

  explicit Lowering(const LowerOptions& o) : opt(o) {
    plan.f64 = o.f64;
    plan.rank = o.rank;
    plan.world = o.world;
  }

  std::string fty() const { return opt.f64 ? "double" : "float"; }
  std::string ctype(SK k) const {
    switch (k) {
      case SK::F: return "dx_f";
      case SK::D: return "double";
      case SK::I: return "long long";
      case SK::X: return "int";
      case SK::U32: return "unsigned";
    }
    return "dx_f";
  }

  int newBuf(BufDecl::Role role, SK kind, long long elems) {
    BufDecl b;
    b.role = role;
    b.kind = kind;
    b.elems = elems;
    plan.bufs.push_back(b);
    return (int)plan.bufs.size() - 1;
  }

  // ------------------------------------------------------------------
  // Type resolution (Fin sizes from literals or Int constants in scope).

  using SizeLookup = std::function<bool(const Name&, long long*)>;

  long long sizeOf(const ValuePtr& v, const SizeLookup& look) {
    if (const auto* i = as<VLitInt>(v)) return i->v;
    if (const auto* var = as<VVar>(v)) {
      long long x;
      if (look(var->name, &x)) return x;
    }
    fail(ErrCode::UnresolvedSize, "Fin size did not resolve to a constant integer",
         v ? v->span : Span{});
  }

  DescPtr resolveDesc(const ValuePtr& t, const SizeLookup& look) {
    if (isBase(t, BaseKind::Unit)) return descUnit();
    if (const auto* f = as<VFinType>(t)) {
      long long n = sizeOf(f->size, look);
      if (n < 0) fail(ErrCode::UnresolvedSize, "negative Fin size", t->span);
      return descFin(n);
    }
    if (const auto* p = as<VPairType>(t)) return descPair(resolveDesc(p->l, look), resolveDesc(p->r, look));
    if (const auto* e = as<VEitherType>(t)) return descEither(resolveDesc(e->l, look), resolveDesc(e->r, look));
    fail(ErrCode::UnresolvedSize, "type " + printValue(t) + " is not a resolvable index set",
         t ? t->span : Span{});
  }

  DTy resolveType(const ValuePtr& t, const SizeLookup& look) {
    if (isBase(t, BaseKind::Float)) return tFloat();
    if (isBase(t, BaseKind::Int)) return tInt();
    if (isBase(t, BaseKind::Unit)) return tUnit();
    if (as<VFinType>(t)) return tIdx(resolveDesc(t, look));
    if (const auto* e = as<VEitherType>(t)) {
      // Either of index sets is itself an index set (stored as its ordinal);
      // other sums are data: a tag plus both payloads.
      if (isIndexSetType(e->l) && isIndexSetType(e->r))
        return tIdx(descEither(resolveDesc(e->l, look), resolveDesc(e->r, look)));
      return tSum(resolveType(e->l, look), resolveType(e->r, look));
    }
    if (const auto* p = as<VPairType>(t)) return tPair(resolveType(p->l, look), resolveType(p->r, look));
    if (const auto* a = as<VArrayType>(t)) return tTable(resolveDesc(a->dom, look), resolveType(a->cod, look));
    if (const auto* r = as<VRefType>(t)) return tRef(resolveType(r->payload, look));
    notLowerable("type " + printValue(t), t ? t->span : Span{});
  }

  // Static element type of a view/loop body: the type of its returned value,
  // from let annotations or the types of the names it mentions.
  DTy staticBodyType(const ExprPtr& body, const SizeLookup& look,
                     const std::function<DTy(const Name&)>& outer) {
    std::map<uint64_t, ValuePtr> annots;
    ExprPtr cur = body;
    while (const auto* l = as<ELet>(cur)) {
      if (l->annot) annots[l->binder.uid] = l->annot;
      cur = l->body;
    }
    const auto* r = as<ERet>(cur);
    if (!r) return nullptr;
    std::function<DTy(const ValuePtr&)> vt = [&](const ValuePtr& v) -> DTy {
      try {
        if (as<VLitFloat>(v)) return tFloat();
        if (as<VLitInt>(v)) return tInt();
        if (as<VLitUnit>(v)) return tUnit();
        if (const auto* x = as<VVar>(v)) {
          auto it = annots.find(x->name.uid);
          if (it != annots.end()) return resolveType(it->second, look);
          return outer(x->name);
        }
        if (const auto* p = as<VPair>(v)) {
          DTy a = vt(p->l), b = vt(p->r);
          return (a && b) ? tPair(a, b) : nullptr;
        }
        if (const auto* w = as<VView>(v)) {
          DTy e = staticBodyType(w->body, look, outer);
          return e ? tTable(resolveDesc(w->annot, look), e) : nullptr;
        }
        if (const auto* f = as<VFinLit>(v)) return tIdx(descFin(sizeOf(f->size, look)));
      } catch (const DexError&) {
      }
      return nullptr;
    };
    return vt(r->value);
  }

  // Table type of a lazy loop from its let annotation (element type may be
  // unknown when the binding has none).
  DTy annotTableType(const ValuePtr& annot, const DescPtr& d, const SizeLookup& look) {
    if (annot) {
      try {
        DTy t = resolveType(annot, look);
        if (t->k == DType::Table) return t;
      } catch (const DexError&) {
      }
    }
    return tTable(d, nullptr);
  }

  SizeLookup hostLook(const HEnvP& env) {
    return [env](const Name& n, long long* out) {
      HV v = hlookup(env, n);
      if (v && v->k == HVal::Const && v->ty->k == DType::Int) {
        *out = v->i;
        return true;
      }
      return false;
    };
  }

  // ------------------------------------------------------------------
  // Cells.

  int newCell(const DTy& payload, bool accum) {
    plan.cellsAllocated++;
    Cell c;
    c.payload = payload;
    c.lv = leaves(payload);
    c.accum = accum;
    for (auto& l : c.lv) {
      SK k = (l.kind == SK::F && !opt.f64) ? SK::D : l.kind;  // cells accumulate in f64
      int b = newBuf(BufDecl::Cell, k, l.count);
      c.bufs.push_back(b);
      c.host.emplace_back(l.count, 0.0);
      Step z;
      z.k = Step::Zero;
      z.buf = b;
      z.elems = l.count;
      plan.steps.push_back(z);
    }
    cells.push_back(std::move(c));
    return (int)cells.size() - 1;
  }

  // Makes the device copy of a cell authoritative before a kernel touches it.
  void cellToDevice(int ci) {
    Cell& c = cells[ci];
    if (c.lazy) {
      HV lz = c.lazy;
      c.lazy = nullptr;
      c.dirty = true;
      std::vector<long long> offs(c.bufs.size(), 0);
      materializeInto(lz, c.bufs, offs);
      return;
    }
    if (c.dirty) return;
    c.dirty = true;
    for (size_t l = 0; l < c.bufs.size(); ++l) {
      bool nz = false;
      for (double v : c.host[l]) nz |= (v != 0.0);
      if (!nz) continue;
      Step u;
      u.k = Step::Upload;
      u.buf = c.bufs[l];
      u.elems = (long long)c.host[l].size();
      SK ck = plan.bufs[c.bufs[l]].kind;
      int cb = newBuf(BufDecl::Const, ck, u.elems);
      if (ck == SK::F || ck == SK::D) plan.bufs[cb].initF = c.host[l];
      else for (double v : c.host[l]) plan.bufs[cb].initI.push_back((long long)v);
      u.buf2 = cb;
      addStep(u);
    }
  }

  // Current value of a cell as a host value.
  HV cellValue(int ci) {
    Cell& c = cells[ci];
    if (c.lazy) return c.lazy;
    if (!c.dirty && c.payload->k != DType::Table) return hostConstOf(c.payload, c, 0);
    cellToDevice(ci);
    std::vector<long long> offs(c.bufs.size(), 0);
    return hvFromBufs(c.payload, c.bufs, offs);
  }

  HV hostConstOf(const DTy& t, Cell& c, size_t leafBase) {
    switch (t->k) {
      case DType::Float: return hConstF(c.host[leafBase][0]);
      case DType::Int: return hConstI((long long)c.host[leafBase][0]);
      case DType::Idx: return hConstIdx((long long)c.host[leafBase][0], t->desc);
      case DType::Unit: return hUnit();
      case DType::Pair: {
        HV a = hostConstOf(t->a, c, leafBase);
        HV b = hostConstOf(t->b, c, leafBase + numLeaves(t->a));
        return hPair(a, b);
      }
      default: notLowerable("host constant of " + showType(t));
    }
  }

  HV hvFromBufs(const DTy& t, const std::vector<int>& bufs, const std::vector<long long>& offs,
                size_t base = 0) {
    switch (t->k) {
      case DType::Unit: return hUnit();
      case DType::Pair: {
        size_t na = numLeaves(t->a);
        HV a = hvFromBufs(t->a, bufs, offs, base);
        HV b = hvFromBufs(t->b, bufs, offs, base + na);
        return hPair(a, b);
      }
      case DType::Idx:
        if (t->desc->kind == IndexSetDesc::Kind::Unit) return hUnit();
        [[fallthrough]];
      default: {
        auto h = std::make_shared<HVal>();
        h->k = HVal::Buf;
        h->ty = t;
        size_t n = numLeaves(t);
        for (size_t l = 0; l < n; ++l) {
          h->bufs.push_back(bufs[base + l]);
          h->offs.push_back(offs[base + l]);
        }
        return h;
      }
    }
  }

  // ------------------------------------------------------------------
  // Static scans.

  // True when `body` performs Get/Put on a ref it does not handle itself
  // (the reference's ParScan, eval.cpp:548-600), or contains App.
  bool blocksParallel(const ExprPtr& body) {
    std::set<Name> local;
    bool blocked = false;
    std::function<void(const ExprPtr&)> scan = [&](const ExprPtr& e) {
      if (blocked) return;
      std::visit(
          [&](const auto& n) {
            using T = std::decay_t<decltype(n)>;
            if constexpr (std::is_same_v<T, ELet>) {
              scan(n.bound);
              if (const auto* s = as<ESlice>(n.bound)) {
                const auto* v = as<VVar>(s->ref);
                if (v && local.count(v->name)) local.insert(n.binder);
              }
              scan(n.body);
            } else if constexpr (std::is_same_v<T, EApp> || std::is_same_v<T, ELinearize> ||
                                 std::is_same_v<T, ETranspose>) {
              blocked = true;
            } else if constexpr (std::is_same_v<T, EFor>) {
              scan(n.body);
            } else if constexpr (std::is_same_v<T, ECase>) {
              scan(n.leftBody);
              scan(n.rightBody);
            } else if constexpr (std::is_same_v<T, ERunState> || std::is_same_v<T, ERunAccum>) {
              local.insert(n.action.ref);
              scan(n.action.body);
            } else if constexpr (std::is_same_v<T, EGet> || std::is_same_v<T, EPut>) {
              const auto* v = as<VVar>(n.ref);
              if (!(v && local.count(v->name))) blocked = true;
            }
          },
          e->node);
    };
    scan(body);
    return blocked;
  }

  // True when the loop body has no effect on refs it does not create.
  bool pureBody(const ExprPtr& body) {
    std::set<Name> local;
    bool impure = false;
    std::function<void(const ExprPtr&)> scan = [&](const ExprPtr& e) {
      if (impure) return;
      std::visit(
          [&](const auto& n) {
            using T = std::decay_t<decltype(n)>;
            if constexpr (std::is_same_v<T, ELet>) {
              scan(n.bound);
              if (const auto* s = as<ESlice>(n.bound)) {
                const auto* v = as<VVar>(s->ref);
                if (v && local.count(v->name)) local.insert(n.binder);
              }
              scan(n.body);
            } else if constexpr (std::is_same_v<T, EApp> || std::is_same_v<T, ELinearize> ||
                                 std::is_same_v<T, ETranspose>) {
              impure = true;
            } else if constexpr (std::is_same_v<T, EFor>) {
              scan(n.body);
            } else if constexpr (std::is_same_v<T, ECase>) {
              scan(n.leftBody);
              scan(n.rightBody);
            } else if constexpr (std::is_same_v<T, ERunState> || std::is_same_v<T, ERunAccum>) {
              local.insert(n.action.ref);
              scan(n.action.body);
            } else if constexpr (std::is_same_v<T, EGet> || std::is_same_v<T, EPut> ||
                                 std::is_same_v<T, EAccum>) {
              const auto* v = as<VVar>(n.ref);
              if (!(v && local.count(v->name))) impure = true;
            }
          },
          e->node);
    };
    scan(body);
    return !impure;
  }

  // Cheap loop bodies are recomputed at every use instead of materialized.
  bool cheapBody(const ExprPtr& body) {
    // a perfect-nest wrapper `let t = for k. B; t` is as cheap as B per element
    if (const auto* l = as<ELet>(body)) {
      const auto* f = as<EFor>(l->bound);
      const auto* r = as<ERet>(l->body);
      const auto* rv = r ? as<VVar>(r->value) : nullptr;
      if (f && rv && rv->name == l->binder && pureBody(f->body)) return cheapBody(f->body);
    }
    int stmts = 0;
    bool heavy = false;
    std::function<void(const ExprPtr&)> scan = [&](const ExprPtr& e) {
      std::visit(
          [&](const auto& n) {
            using T = std::decay_t<decltype(n)>;
            ++stmts;
            if constexpr (std::is_same_v<T, ELet>) {
              scan(n.bound);
              scan(n.body);
            } else if constexpr (std::is_same_v<T, EFor> || std::is_same_v<T, ERunAccum> ||
                                 std::is_same_v<T, ERunState> || std::is_same_v<T, ECase>) {
              heavy = true;
            }
          },
          e->node);
    };
    scan(body);
    return !heavy && stmts <= 24;
  }

  // Binder used only as `reverse binder` (the transposed loops of
  // autodiff.cpp:705-717): iterate the reversed order directly.
  bool onlyReversed(const Name& b, const ExprPtr& body) {
    bool other = false, any = false;
    std::function<void(const ValuePtr&)> sv = [&](const ValuePtr& v) {
      if (!v) return;
      if (const auto* x = as<VVar>(v)) {
        if (x->name == b) other = true;
        return;
      }
      for (const Name& n : freeVars(v))
        if (n == b) other = true;
    };
    std::function<void(const ExprPtr&)> scan = [&](const ExprPtr& e) {
      if (other) return;
      if (const auto* u = as<EUnOp>(e)) {
        if (u->op == UnOp::ReverseIndex) {
          const auto* x = as<VVar>(u->v);
          if (x && x->name == b) { any = true; return; }
        }
      }
      if (const auto* l = as<ELet>(e)) {
        scan(l->bound);
        if (l->annot) sv(l->annot);
        scan(l->body);
        return;
      }
      if (const auto* c = as<ECase>(e)) {
        sv(c->scrutinee);
        scan(c->leftBody);
        scan(c->rightBody);
        return;
      }
      if (const auto* f = as<EFor>(e)) {
        sv(f->annot);
        scan(f->body);
        return;
      }
      if (const auto* r = as<ERunAccum>(e)) {
        sv(r->action.refAnnot);
        scan(r->action.body);
        return;
      }
      if (const auto* r = as<ERunState>(e)) {
        sv(r->init);
        sv(r->action.refAnnot);
        scan(r->action.body);
        return;
      }
      for (const Name& n : freeVars(e))
        if (n == b) other = true;
    };
    scan(body);
    return any && !other;
  }

  // ------------------------------------------------------------------
  // Host level.

  HV hvalue(const HEnvP& env, const ValuePtr& v) {
    if (const auto* x = as<VVar>(v)) {
      HV r = hlookup(env, x->name);
      if (!r) fail(ErrCode::Internal, "variable '" + printName(x->name) + "' has no binding", v->span);
      return r;
    }
    if (const auto* f = as<VLitFloat>(v)) return hConstF(f->v);
    if (const auto* i = as<VLitInt>(v)) return hConstI(i->v);
    if (as<VLitUnit>(v)) return hUnit();
    if (const auto* fl = as<VFinLit>(v)) {
      long long n = sizeOf(fl->size, hostLook(env));
      if (fl->ordinal < 0 || fl->ordinal >= n)
        fail(ErrCode::OutOfBounds, "index literal @" + std::to_string(fl->ordinal) +
                                       " is outside Fin " + std::to_string(n), v->span);
      return hConstIdx(fl->ordinal, descFin(n));
    }
    if (const auto* p = as<VPair>(v)) return hPair(hvalue(env, p->l), hvalue(env, p->r));
    if (as<VInjLeft>(v) || as<VInjRight>(v)) {
      bool left = as<VInjLeft>(v) != nullptr;
      ValuePtr payloadV = left ? as<VInjLeft>(v)->payload : as<VInjRight>(v)->payload;
      ValuePtr otherT = left ? as<VInjLeft>(v)->otherType : as<VInjRight>(v)->otherType;
      HV p = hvalue(env, payloadV);
      DescPtr od = resolveDesc(otherT, hostLook(env));
      DescPtr md = memberDesc(p->ty);
      long long o;
      if (!md || !hOrdinal(p, md, &o)) notLowerable("host sum value over non-index payload", v->span);
      DescPtr d = left ? descEither(md, od) : descEither(od, md);
      return hConstIdx(left ? o : size(od) + o, d);
    }
    if (const auto* vw = as<VView>(v)) {
      auto h = std::make_shared<HVal>();
      h->k = HVal::Lazy;
      h->binder = vw->binder;
      h->desc = resolveDesc(vw->annot, hostLook(env));
      h->body = vw->body;
      h->env = env;
      h->cheap = cheapBody(vw->body);
      h->st = std::make_shared<LazyState>();
      h->ty = tTable(h->desc, staticBodyType(vw->body, hostLook(env), [&](const Name& n) -> DTy {
        HV x = hlookup(env, n);
        return x ? x->ty : nullptr;
      }));
      return h;
    }
    if (const auto* t = as<VTableLit>(v)) {
      DescPtr d = resolveDesc(t->dom, hostLook(env));
      std::vector<HV> elems;
      for (auto& e : t->elems) elems.push_back(hvalue(env, e));
      return constTable(d, elems, v->span);
    }
    if (const auto* vc = as<VValueCase>(v)) {
      // lazy case over function branches (reference eval.cpp:180-185): a
      // host-known scrutinee picks its branch here, anything else runs on
      // one device thread
      HV sc = hvalue(env, vc->scrutinee);
      const auto* lf = as<VLam>(vc->leftFn);
      const auto* rf = as<VLam>(vc->rightFn);
      if (lf && rf && sc->k == HVal::Const && sc->ty->k == DType::Idx &&
          sc->ty->desc->kind == IndexSetDesc::Kind::Either) {
        DescPtr d = sc->ty->desc;
        long long ls = size(d->left);
        if (sc->i < ls) return hexpr(hbind(env, lf->binder, hFromOrdinal(sc->i, d->left)), lf->body);
        return hexpr(hbind(env, rf->binder, hFromOrdinal(sc->i - ls, d->right)), rf->body);
      }
      return serialKernel(env, eRet(v), nullptr);
    }
    notLowerable("value " + printValue(v), v->span);
  }

  static DescPtr memberDesc(const DTy& t) {
    switch (t->k) {
      case DType::Idx: return t->desc;
      case DType::Unit: return descUnit();
      case DType::Pair: {
        DescPtr a = memberDesc(t->a), b = memberDesc(t->b);
        return (a && b) ? descPair(a, b) : nullptr;
      }
      default: return nullptr;
    }
  }

  // Literal table of host constants -> Const buffers (SoA).
  HV constTable(const DescPtr& d, const std::vector<HV>& elems, Span sp) {
    if (elems.empty()) notLowerable("empty table literal", sp);
    DTy et = elems[0]->ty;
    DTy t = tTable(d, et);
    std::vector<LeafInfo> lv = leaves(t);
    std::vector<int> bufs;
    std::vector<long long> offs;
    for (auto& l : lv) {
      bufs.push_back(newBuf(BufDecl::Const, l.kind, l.count));
      offs.push_back(0);
    }
    size_t ne = numLeaves(et);
    std::vector<LeafInfo> elv = leaves(et);
    for (size_t k = 0; k < elems.size(); ++k) {
      std::vector<double> fl;
      flattenConst(elems[k], fl, sp);
      size_t pos = 0;
      for (size_t l = 0; l < ne; ++l) {
        BufDecl& b = plan.bufs[bufs[l]];
        for (long long q = 0; q < elv[l].count; ++q, ++pos) {
          if (b.kind == SK::F) b.initF.push_back(fl[pos]);
          else b.initI.push_back((long long)fl[pos]);
        }
      }
    }
    for (size_t l = 0; l < bufs.size(); ++l) {
      Step u;
      u.k = Step::Upload;
      u.buf = bufs[l];
      u.buf2 = bufs[l];
      u.elems = lv[l].count;
      addStep(u);
    }
    return hvFromBufs(t, bufs, offs);
  }

  void flattenConst(const HV& v, std::vector<double>& out, Span sp) {
    // leaf-major order within one element (matches leavesOf)
    std::vector<std::vector<double>> perLeaf;
    std::function<void(const HV&)> go = [&](const HV& x) {
      switch (x->k) {
        case HVal::Const:
          perLeaf.push_back({x->ty->k == DType::Float ? x->f : (double)x->i});
          return;
        case HVal::Unit: return;
        case HVal::Pair: go(x->a); go(x->b); return;
        case HVal::Buf: {
          // a nested table literal: its Const buffers hold the values
          std::vector<LeafInfo> lv = leaves(x->ty);
          for (size_t l = 0; l < lv.size(); ++l) {
            const BufDecl& b = plan.bufs[x->bufs[l]];
            if (b.role != BufDecl::Const) notLowerable("non-constant element in a table literal", sp);
            std::vector<double> vals;
            for (long long q = 0; q < lv[l].count; ++q) {
              const long long at = x->offs[l] + q;
              vals.push_back(b.kind == SK::F ? b.initF.at(at) : (double)b.initI.at(at));
            }
            perLeaf.push_back(std::move(vals));
          }
          return;
        }
        default: notLowerable("non-constant element in a table literal", sp);
      }
    };
    go(v);
    for (auto& l : perLeaf) out.insert(out.end(), l.begin(), l.end());
  }

  HV hexpr(const HEnvP& env, const ExprPtr& e) {
    if (const auto* l = as<ELet>(e)) {
      HV b = hbound(env, l->bound, l->annot);
      return hexpr(hbind(env, l->binder, b), l->body);
    }
    return hbound(env, e, nullptr);
  }

  HV hbound(const HEnvP& env, const ExprPtr& e, const ValuePtr& annot) {
    if (const auto* r = as<ERet>(e)) return hvalue(env, r->value);
    if (as<ELet>(e)) return hexpr(env, e);
    if (const auto* f = as<EFor>(e)) return hostFor(env, *f, e, annot);
    if (const auto* r = as<ERunAccum>(e)) return hostRunAccum(env, *r, e);
    if (const auto* r = as<ERunState>(e)) return hostRunState(env, *r, e);
    if (const auto* s = as<ESlice>(e)) {
      HV ref = hvalue(env, s->ref);
      HV idx = hvalue(env, s->idx);
      if (ref->k != HVal::Ref) notLowerable("slice of a non-reference", e->span);
      const DTy& pt = ref->ty->a;
      if (pt->k != DType::Table) notLowerable("slice of a non-table reference", e->span);
      long long o;
      if (hOrdinal(idx, pt->desc, &o)) {
        auto h = std::make_shared<HVal>(*ref);
        h->ty = tRef(pt->a);
        std::vector<LeafInfo> el = leaves(pt->a);
        for (size_t l = 0; l < h->offs.size(); ++l) h->offs[l] += o * el[l].count;
        return h;
      }
      return serialKernel(env, e, annot);
    }
    if (const auto* x = as<EFst>(e)) {
      HV v = hvalue(env, x->v);
      if (v->k == HVal::Pair) return v->a;
      notLowerable("fst of a non-pair", e->span);
    }
    if (const auto* x = as<ESnd>(e)) {
      HV v = hvalue(env, x->v);
      if (v->k == HVal::Pair) return v->b;
      notLowerable("snd of a non-pair", e->span);
    }
    if (const auto* x = as<EIndex>(e)) {
      HV arr = hvalue(env, x->arr);
      HV idx = hvalue(env, x->idx);
      if (arr->k == HVal::Buf && arr->ty->k == DType::Table) {
        long long o;
        if (hOrdinal(idx, arr->ty->desc, &o)) {
          DTy et = arr->ty->a;
          std::vector<LeafInfo> el = leaves(et);
          std::vector<long long> offs = arr->offs;
          for (size_t l = 0; l < offs.size(); ++l) offs[l] += o * el[l].count;
          return hvFromBufs(et, arr->bufs, offs);
        }
      }
      return serialKernel(env, e, annot);
    }
    if (const auto* b = as<EBinOp>(e)) {
      HV l = hvalue(env, b->l), r = hvalue(env, b->r);
      if (l->k == HVal::Const && r->k == HVal::Const) {
        if (b->op != BinOp::Less) plan.staticOps++;  // evaluated once, at lowering time
        switch (b->op) {
          case BinOp::Add: return hConstF(l->f + r->f);
          case BinOp::Sub: return hConstF(l->f - r->f);
          case BinOp::Mul: return hConstF(l->f * r->f);
          case BinOp::Div: return hConstF(l->f / r->f);
          case BinOp::Less: return hConstIdx((l->f < r->f) ? 1 : 0, boolDesc());  // Left = false
        }
      }
      return serialKernel(env, e, annot);
    }
    if (const auto* u = as<EUnOp>(e)) {
      HV v = hvalue(env, u->v);
      switch (u->op) {
        case UnOp::Ordinal: {
          DescPtr d = memberDesc(v->ty);
          long long o;
          if (d && hOrdinal(v, d, &o)) return hConstI(o);
          break;
        }
        case UnOp::IntToFloat:
          if (v->k == HVal::Const) return hConstF((double)v->i);
          break;
        case UnOp::ReverseIndex: {
          DescPtr d = memberDesc(v->ty);
          long long o;
          if (d && hOrdinal(v, d, &o)) return hFromOrdinal(size(d) - 1 - o, d);
          break;
        }
        case UnOp::Exp:  // frontend_ext (exp/log), folded in double like the evaluator
          if (v->k == HVal::Const) return hConstF(std::exp(v->f));
          break;
        case UnOp::Log:
          if (v->k == HVal::Const) return hConstF(std::log(v->f));
          break;
      }
      return serialKernel(env, e, annot);
    }
    if (const auto* c = as<ECase>(e)) {
      HV s = hvalue(env, c->scrutinee);
      if (s->k == HVal::Const && s->ty->k == DType::Idx && s->ty->desc->kind == IndexSetDesc::Kind::Either) {
        DescPtr d = s->ty->desc;
        long long ls = size(d->left);
        if (s->i < ls) return hexpr(hbind(env, c->leftBinder, hFromOrdinal(s->i, d->left)), c->leftBody);
        return hexpr(hbind(env, c->rightBinder, hFromOrdinal(s->i - ls, d->right)), c->rightBody);
      }
      return serialKernel(env, e, annot);
    }
    if (const auto* a = as<EAccum>(e)) return hostAccum(env, *a, e, annot);
    if (const auto* g = as<EGet>(e)) {
      HV ref = hvalue(env, g->ref);
      if (ref->k == HVal::Ref) {
        Cell& c = cells[ref->cell];
        if (!c.dirty && !c.lazy && ref->ty->a->k != DType::Table) {
          // scalar / pair path into a host-known cell
          Cell tmp;
          std::vector<LeafInfo> pl = leaves(ref->ty->a);
          for (size_t l = 0; l < pl.size(); ++l) tmp.host.push_back({c.host[l][ref->offs[l]]});
          return hostConstOf(ref->ty->a, tmp, 0);
        }
      }
      return serialKernel(env, e, annot);
    }
    if (const auto* p = as<EPut>(e)) {
      HV ref = hvalue(env, p->ref);
      HV v = hvalue(env, p->value);
      if (ref->k == HVal::Ref) {
        Cell& c = cells[ref->cell];
        std::vector<double> fl;
        bool isConst = true;
        std::function<void(const HV&)> go = [&](const HV& x) {
          if (x->k == HVal::Const) fl.push_back(x->ty->k == DType::Float ? x->f : (double)x->i);
          else if (x->k == HVal::Pair) { go(x->a); go(x->b); }
          else if (x->k != HVal::Unit) isConst = false;
        };
        go(v);
        if (!c.dirty && !c.lazy && isConst && ref->ty->a->k != DType::Table) {
          for (size_t l = 0; l < fl.size(); ++l) c.host[l][ref->offs[l]] = fl[l];
          return hUnit();
        }
      }
      return serialKernel(env, e, annot);
    }
    if (as<EApp>(e)) notLowerable("application (program is not first-order)", e->span);
    if (as<ELinearize>(e) || as<ETranspose>(e))
      notLowerable("linearize/transpose must be eliminated by simplification", e->span);
    notLowerable("expression", e->span);
  }

  HV hostAccum(const HEnvP& env, const EAccum& a, const ExprPtr& e, const ValuePtr& annot) {
    HV ref = hvalue(env, a.ref);
    HV v = hvalue(env, a.value);
    if (ref->k != HVal::Ref) notLowerable("accumulation into a non-reference", e->span);
    Cell& c = cells[ref->cell];
    if (!c.dirty && !c.lazy && v->k == HVal::Const && v->ty->k == DType::Float) {
      c.host[0][ref->offs[0]] += v->f;
      plan.staticAccums++;
      return hUnit();
    }
    if (!c.dirty && !c.lazy && v->k == HVal::Pair) {
      std::vector<double> fl;
      bool ok = true;
      std::function<void(const HV&)> go = [&](const HV& x) {
        if (x->k == HVal::Const && x->ty->k == DType::Float) fl.push_back(x->f);
        else if (x->k == HVal::Pair) { go(x->a); go(x->b); }
        else ok = false;
      };
      go(v);
      if (ok && fl.size() == ref->offs.size()) {
        for (size_t l = 0; l < fl.size(); ++l) c.host[l][ref->offs[l]] += fl[l];
        plan.staticAccums++;
        return hUnit();
      }
    }
    if (HV r = hostAccumTables(ref, v)) return r;
    return serialKernel(env, e, annot);
  }

  // Structurally zero lazy tables (`view i. 0.0`, the zero cotangents of
  // the pair-of-tables accumulations in transposed programs).
  static bool zeroBody(const ExprPtr& e) {
    const auto* r = as<ERet>(e);
    if (!r) return false;
    std::function<bool(const ValuePtr&)> zv = [&](const ValuePtr& v) -> bool {
      if (const auto* f = as<VLitFloat>(v)) return f->v == 0.0;
      if (const auto* w = as<VView>(v)) return zeroBody(w->body);
      if (const auto* p = as<VPair>(v)) return zv(p->l) && zv(p->r);
      return false;
    };
    return zv(r->value);
  }

  // `ref += v` at host level with v a (pair of) device tables: one parallel
  // add per leaf into the cell (zero views skipped), never a serial kernel.
  HV hostAccumTables(const HV& ref, const HV& v) {
    struct Add {
      size_t leaf;
      HV src;
    };
    std::vector<Add> adds;
    std::function<bool(const HV&, size_t)> walk = [&](const HV& x, size_t base) -> bool {
      switch (x->k) {
        case HVal::Pair: return walk(x->a, base) && walk(x->b, base + numLeaves(x->a->ty));
        case HVal::Unit: return true;
        case HVal::Const: return x->ty->k == DType::Float && x->f == 0.0;
        case HVal::Lazy:
          if (x->st->materialized) return walk(x->st->materialized, base);
          if (zeroBody(x->body)) return true;
          if (!x->ty || x->ty->k != DType::Table) return false;
          adds.push_back({base, x});
          return true;
        case HVal::Buf:
          if (x->ty->k != DType::Table) return false;
          adds.push_back({base, x});
          return true;
        default: return false;
      }
    };
    if (!walk(v, 0)) return nullptr;
    for (auto& a : adds) {
      std::vector<LeafInfo> lv = leaves(a.src->ty);
      for (size_t l = 0; l < lv.size(); ++l)
        if (lv[l].kind != SK::F) return nullptr;
    }
    cellToDevice(ref->cell);
    for (auto& a : adds) {
      HV src = a.src->k == HVal::Lazy ? materialize(a.src) : a.src;
      std::vector<LeafInfo> lv = leaves(src->ty);
      for (size_t l = 0; l < lv.size(); ++l) {
        Step st;
        st.k = Step::AddBuf;
        st.buf = cells[ref->cell].bufs[a.leaf + l];
        st.off = ref->offs[a.leaf + l];
        st.buf2 = src->bufs[l];
        st.off2 = src->offs[l];
        st.elems = lv[l].count;
        // into a whole cell right after its zero-fill: a copy (or an f32 ->
        // f64 conversion) replaces the zero pass and the read-modify-write
        if (st.off == 0 && st.elems == plan.bufs[st.buf].elems && takeZero(st.buf))
          st.k = plan.bufs[st.buf].kind == plan.bufs[st.buf2].kind ? Step::CopyBuf : Step::Convert;
        addStep(st);
      }
    }
    return hUnit();
  }

  HV hostRunAccum(const HEnvP& env, const ERunAccum& r, const ExprPtr& e) {
    const auto* ra = as<VRefType>(r.action.refAnnot);
    if (!ra) fail(ErrCode::Internal, "runAccum reached the lowering unannotated", e->span);
    DTy payload = resolveType(ra->payload, hostLook(env));
    int ci = newCell(payload, true);
    auto ref = std::make_shared<HVal>();
    ref->k = HVal::Ref;
    ref->ty = tRef(payload);
    ref->cell = ci;
    ref->offs.assign(cells[ci].bufs.size(), 0);
    HEnvP env2 = hbind(env, r.action.ref, ref);
    HV res = hexpr(env2, r.action.body);
    HV val = cellValue(ci);
    return hPair(res, val);
  }

  HV hostRunState(const HEnvP& env, const ERunState& r, const ExprPtr& e) {
    const auto* ra = as<VRefType>(r.action.refAnnot);
    HV init = hvalue(env, r.init);
    DTy payload = ra ? resolveType(ra->payload, hostLook(env)) : init->ty;
    int ci = newCell(payload, false);
    Cell& c = cells[ci];
    // initialize: host constants fold, device values copy
    std::vector<double> fl;
    bool isConst = true;
    std::function<void(const HV&)> go = [&](const HV& x) {
      if (x->k == HVal::Const) fl.push_back(x->ty->k == DType::Float ? x->f : (double)x->i);
      else if (x->k == HVal::Pair) { go(x->a); go(x->b); }
      else if (x->k != HVal::Unit) isConst = false;
    };
    go(init);
    if (isConst && payload->k != DType::Table) {
      for (size_t l = 0; l < fl.size() && l < c.host.size(); ++l) c.host[l][0] = fl[l];
    } else {
      c.dirty = true;
      std::vector<long long> offs(c.bufs.size(), 0);
      copyValueInto(init, c.bufs, offs, e->span);
    }
    auto ref = std::make_shared<HVal>();
    ref->k = HVal::Ref;
    ref->ty = tRef(payload);
    ref->cell = ci;
    ref->offs.assign(c.bufs.size(), 0);
    HV res = hexpr(hbind(env, r.action.ref, ref), r.action.body);
    HV val = cellValue(ci);
    return hPair(res, val);
  }

  // Writes a host value into buffers (device copies / kernels).
  void copyValueInto(const HV& v, const std::vector<int>& bufs, const std::vector<long long>& offs,
                     Span sp, size_t base = 0) {
    switch (v->k) {
      case HVal::Unit: return;
      case HVal::Pair: {
        size_t na = numLeaves(v->a->ty);
        copyValueInto(v->a, bufs, offs, sp, base);
        copyValueInto(v->b, bufs, offs, sp, base + na);
        return;
      }
      case HVal::Buf: {
        std::vector<LeafInfo> lv = leaves(v->ty);
        for (size_t l = 0; l < lv.size(); ++l) {
          Step s;
          s.k = plan.bufs[bufs[base + l]].kind == plan.bufs[v->bufs[l]].kind ? Step::CopyBuf : Step::Convert;
          s.buf = bufs[base + l];
          s.off = offs[base + l];
          s.buf2 = v->bufs[l];
          s.off2 = v->offs[l];
          s.elems = lv[l].count;
          addStep(s);
        }
        return;
      }
      case HVal::Lazy: {
        std::vector<int> b(bufs.begin() + base, bufs.end());
        std::vector<long long> o(offs.begin() + base, offs.end());
        materializeInto(v, b, o);
        return;
      }
      case HVal::Zip: {  // table of pairs: leaves of the first half, then the second
        copyValueInto(v->a, bufs, offs, sp, base);
        copyValueInto(v->b, bufs, offs, sp, base + numLeaves(v->a->ty));
        return;
      }
      case HVal::Const: {
        int cb = newBuf(BufDecl::Const, plan.bufs[bufs[base]].kind, 1);
        if (v->ty->k == DType::Float) plan.bufs[cb].initF = {v->f};
        else plan.bufs[cb].initI = {v->i};
        Step u; u.k = Step::Upload; u.buf = cb; u.buf2 = cb; u.elems = 1; addStep(u);
        Step s; s.k = Step::CopyBuf; s.buf = bufs[base]; s.off = offs[base]; s.buf2 = cb; s.off2 = 0; s.elems = 1;
        addStep(s);
        return;
      }
      default: notLowerable("copy of a reference value", sp);
    }
  }

  // ------------------------------------------------------------------
  // Accum-to-map: `runAccum r. for j. (b = reverse j;) r!b += v` with v not
  // touching r is the table `for b. v` (every element written exactly once
  // into a zero cell).  Detected on the loop; the cell keeps a lazy value
  // so the broadcast cotangents of transposed `sum`s (autodiff.cpp:760-772)
  // never hit HBM.
  bool tryAccumToMap(const HEnvP& env, const EFor& f, const DescPtr& d) {
    if (opt.noFusion) return false;
    // Collect the let chain.
    std::vector<const ELet*> lets;
    ExprPtr cur = f.body;
    while (const auto* l = as<ELet>(cur)) {
      lets.push_back(l);
      cur = l->body;
    }
    int accIdx = -1;
    for (size_t i = 0; i < lets.size(); ++i) {
      const ExprPtr& b = lets[i]->bound;
      if (as<EAccum>(b)) {
        if (accIdx >= 0) return false;
        accIdx = (int)i;
      }
      if (as<EFor>(b) || as<ERunAccum>(b) || as<ERunState>(b) || as<ECase>(b) || as<EPut>(b) || as<EGet>(b))
        return false;
    }
    if (accIdx < 0) return false;
    const auto* acc = as<EAccum>(lets[accIdx]->bound);
    const auto* refVar = as<VVar>(acc->ref);
    if (!refVar) return false;
    // ref must be `sl = R!x` with R a host Ref to a fresh, untouched cell
    const ESlice* sl = nullptr;
    for (size_t i = 0; i < (size_t)accIdx; ++i)
      if (lets[i]->binder == refVar->name) sl = as<ESlice>(lets[i]->bound);
    if (!sl) return false;
    const auto* rootVar = as<VVar>(sl->ref);
    if (!rootVar) return false;
    HV root = hlookup(env, rootVar->name);
    if (!root || root->k != HVal::Ref) return false;
    Cell& c = cells[root->cell];
    if (!c.accum || c.dirty || c.lazy) return false;
    for (auto& hv : c.host)
      for (double x : hv)
        if (x != 0.0) return false;
    for (long long o : root->offs)
      if (o != 0) return false;
    if (c.payload->k != DType::Table || !descEq(c.payload->desc, d)) return false;
    // index: loop binder, or a let-bound `reverse binder`
    const auto* ix = as<VVar>(sl->idx);
    if (!ix) return false;
    bool reversed = false;
    if (ix->name != f.binder) {
      const ELet* rl = nullptr;
      for (size_t i = 0; i < (size_t)accIdx; ++i)
        if (lets[i]->binder == ix->name) rl = lets[i];
      if (!rl) return false;
      const auto* u = as<EUnOp>(rl->bound);
      if (!u || u->op != UnOp::ReverseIndex) return false;
      const auto* uv = as<VVar>(u->v);
      if (!uv || uv->name != f.binder) return false;
      reversed = true;
    }
    // value must not mention the ref or slices of it
    for (const Name& n : freeVars(acc->value))
      if (n == rootVar->name || n == refVar->name) return false;
    // everything after the accumulation must be trivial (return of unit)
    for (size_t i = accIdx + 1; i < lets.size(); ++i) {
      if (!as<ERet>(lets[i]->bound)) return false;
    }
    // Build `for m. (let j = reverse m;) <lets except slice/accum>; ret v`
    ExprPtr body = eRet(acc->value);
    for (int i = accIdx - 1; i >= 0; --i) {
      if (lets[i]->binder == refVar->name) continue;  // the slice
      // drop lets mentioning the ref (only the slice may)
      bool mentions = false;
      for (const Name& n : freeVars(lets[i]->bound))
        if (n == rootVar->name || n == refVar->name) mentions = true;
      if (mentions) return false;
      body = eLet(lets[i]->binder, lets[i]->annot, lets[i]->bound, body);
    }
    Name m = f.binder;
    if (reversed) {
      m = NameSupply::fresh("m");
      body = eLet(f.binder, f.annot, eUn(UnOp::ReverseIndex, vVar(m)), body);
    }
    auto h = std::make_shared<HVal>();
    h->k = HVal::Lazy;
    h->binder = m;
    h->desc = d;
    h->body = body;
    h->env = env;
    h->cheap = cheapBody(body);
    h->st = std::make_shared<LazyState>();
    h->ty = c.payload;
    c.lazy = h;
    plan.staticAccums += size(d);  // the n broadcast updates the map replaces
    return true;
  }

  HV hostFor(const HEnvP& env, const EFor& f, const ExprPtr& e, const ValuePtr& annot) {
    DescPtr d = resolveDesc(f.annot, hostLook(env));
    if (pureBody(f.body)) {
      auto h = std::make_shared<HVal>();
      h->k = HVal::Lazy;
      h->binder = f.binder;
      h->desc = d;
      h->body = f.body;
      h->env = env;
      h->cheap = cheapBody(f.body);
      h->st = std::make_shared<LazyState>();
      h->ty = annotTableType(annot, d, hostLook(env));
      if (opt.noFusion) return materialize(h);
      return h;
    }
    if (tryAccumToMap(env, f, d)) {
      auto h = std::make_shared<HVal>();
      h->k = HVal::Buf;
      h->ty = tTable(d, tUnit());
      return h;
    }
    bool serial = blocksParallel(f.body);
    return loopKernel(env, f, d, serial, e->span);
  }

  HV materialize(const HV& lz) {
    if (lz->k != HVal::Lazy) return lz;
    if (lz->st->materialized) return lz->st->materialized;
    HV r = loopKernelLazy(lz, nullptr, nullptr);
    lz->st->materialized = r;
    return r;
  }

  void materializeInto(const HV& lz, const std::vector<int>& bufs, const std::vector<long long>& offs) {
    if (lz->st->materialized) {
      copyValueInto(lz->st->materialized, bufs, offs, Span{});
      return;
    }
    loopKernelLazy(lz, &bufs, &offs);
  }

  // Kernel drivers (defined after KGen helpers).
  HV loopKernel(const HEnvP& env, const EFor& f, const DescPtr& d, bool serial, Span sp);
  HV flattenEffectNest(const HEnvP& env, const EFor& f, const DescPtr& d);
  HV loopKernelLazy(const HV& lz, const std::vector<int>* intoBufs, const std::vector<long long>* intoOffs);
  HV splitMaterialize(const HV& lz);
  ValuePtr typeValue(const DTy& t);
  HV contractNest(const HEnvP& env, const EFor& f, const DescPtr& d);
  HV contractMaterialize(const HV& lz, const std::vector<DescPtr>& dims, const std::vector<Name>& binders,
                         const ExprPtr& body, const std::vector<int>* intoBufs,
                         const std::vector<long long>* intoOffs);
  HV serialKernel(const HEnvP& env, const ExprPtr& e, const ValuePtr& annot);

  // ------------------------------------------------------------------
  // Kernel codegen.

  SizeLookup kernelLook(KGen& g, const KScope& s) {
    return [this, &g, s](const Name& n, long long* out) {
      for (const KEnvNode* p = s.local.get(); p; p = p->next.get()) {
        if (p->n == n) {
          if (p->v->k == KVal::Scalar && p->v->isConst) {
            *out = p->v->ci;
            return true;
          }
          return false;
        }
      }
      return hostLook(s.host)(n, out);
    };
  }

  KV lookupK(KGen& g, const KScope& s, const Name& n, Span sp) {
    for (const KEnvNode* p = s.local.get(); p; p = p->next.get())
      if (p->n == n) return p->v;
    HV h = hlookup(s.host, n);
    if (!h) fail(ErrCode::Internal, "variable '" + printName(n) + "' has no binding", sp);
    return importHost(g, h);
  }

  static KScope kbind(const KScope& s, const Name& n, KV v) {
    KScope r = s;
    r.local = std::make_shared<KEnvNode>(KEnvNode{n, std::move(v), s.local});
    return r;
  }

  std::string param(KGen& g, int buf, bool write) {
    if (write) g.writtenBufs.insert(buf);
    auto it = g.params.find(buf);
    if (it != g.params.end()) return it->second;
    std::string p = "p" + std::to_string(buf);
    g.params[buf] = p;
    return p;
  }

  KV importHost(KGen& g, const HV& h) {
    switch (h->k) {
      case HVal::Const: {
        KV k;
        if (h->ty->k == DType::Float) {
          auto x = kScalar(h->ty, litF(h->f, opt.f64), -1);
          auto m = std::const_pointer_cast<KVal>(x);
          m->isConst = true; m->cf = h->f;
          return x;
        }
        auto x = kScalar(h->ty, lit(h->i), -1);
        auto m = std::const_pointer_cast<KVal>(x);
        m->isConst = true; m->ci = h->i;
        if (h->ty->k == DType::Idx) m->rev = lit(size(h->ty->desc) - 1 - h->i);
        return x;
      }
      case HVal::Unit: return kUnit();
      case HVal::Pair: return kPair(importHost(g, h->a), importHost(g, h->b));
      case HVal::Buf: {
        std::vector<LeafInfo> lv = leaves(h->ty);
        std::vector<Slot> slots;
        for (size_t l = 0; l < lv.size(); ++l) {
          Slot s;
          s.buf = h->bufs[l];
          s.base = param(g, h->bufs[l], false);
          s.off = lit(h->offs[l]);
          s.align = alignOf(h->offs[l]);
          s.global = true;
          s.ro = true;
          s.input = plan.bufs[h->bufs[l]].role == BufDecl::Input;
          s.kind = plan.bufs[h->bufs[l]].kind;
          slots.push_back(s);
        }
        return viewSlots(g, h->ty, slots);
      }
      case HVal::Ref: {
        auto k = std::make_shared<KVal>();
        k->k = KVal::Ref;
        k->ty = h->ty;
        k->cell = h->cell;
        Cell& c = cells[h->cell];
        for (size_t l = 0; l < c.bufs.size(); ++l) {
          Slot s;
          s.buf = c.bufs[l];
          s.base = "";  // resolved per strategy at the access
          s.off = lit(h->offs[l]);
          s.global = true;
          s.kind = plan.bufs[c.bufs[l]].kind;
          s.cellLeaf = (int)l;
          k->slots.push_back(s);
        }
        return k;
      }
      case HVal::Zip: {
        auto k = std::make_shared<KVal>();
        k->k = KVal::Zip;
        k->ty = h->ty;
        k->zipDepth = h->zipDepth;
        k->a = importHost(g, h->a);
        k->b = importHost(g, h->b);
        return k;
      }
      case HVal::Lazy: {
        if (h->st->materialized) return importHost(g, h->st->materialized);
        if (h->st->split) return importHost(g, h->st->split);
        auto k = std::make_shared<KVal>();
        k->k = KVal::Lazy;
        k->ty = h->ty;
        auto lz = std::make_shared<LazyK>();
        lz->binder = h->binder;
        lz->desc = h->desc;
        lz->body = h->body;
        lz->scope.host = h->env;
        lz->cheap = h->cheap;
        lz->key = h->binder.uid;
        lz->hostOrigin = h;
        k->lz = lz;
        return k;
      }
    }
    notLowerable("host value");
  }

  // Pass-0 bookkeeping of read-only HBM reads for TMA staging decisions.
  void noteRead(KGen& g, const Slot& s, bool vector) {
    if (g.pass != 0 || !s.global || !s.ro || s.buf < 0) return;
    if (s.rowW > 0) g.rowUse[s.buf].insert(s.rowW);
    else g.rowBad.insert(s.buf);
    if (s.stream) {
      auto it = g.streamUse.find(s.buf);
      if (it == g.streamUse.end()) g.streamUse[s.buf] = {s.streamL, s.streamBase};
      else if (it->second != std::make_pair(s.streamL, s.streamBase)) g.nonStream.insert(s.buf);
      if (vector) g.needAlign.insert(s.buf);
    } else {
      g.nonStream.insert(s.buf);
    }
  }

  // Build a value from leaf slots (loads scalars into fresh registers).
  KV viewSlots(KGen& g, const DTy& t, const std::vector<Slot>& slots, size_t base = 0) {
    switch (t->k) {
      case DType::Unit: return kUnit();
      case DType::Pair: {
        size_t na = numLeaves(t->a);
        KV a = viewSlots(g, t->a, slots, base);
        KV b = viewSlots(g, t->b, slots, base + na);
        return kPair(a, b);
      }
      case DType::Sum: {
        KV tag = viewSlots(g, tIdx(boolDesc()), slots, base);
        KV a = viewSlots(g, t->a, slots, base + 1);
        KV b = viewSlots(g, t->b, slots, base + 1 + numLeaves(t->a));
        auto k = std::make_shared<KVal>();
        k->k = KVal::Sum;
        k->e = tag->e;
        k->a = a;
        k->b = b;
        k->ty = t;
        k->level = tag->level;
        return k;
      }
      case DType::Table: {
        // Small contiguous rows of read-only HBM tables are fetched whole with
        // 16-byte loads into registers (nvcc does not vectorize the scalar
        // per-column loads itself); the row's columns are then register reads.
        if (g.grp == 0 && numLeaves(t) == 1 && slots[base].global && slots[base].ro && slots[base].kind != SK::X &&
            t->a->k != DType::Table && t->a->k != DType::Pair) {
          const Slot& s0 = slots[base];
          long long cnt = leaves(t)[0].count;
          int es = (int)storageBytesOf(s0.kind, opt.f64);
          const bool fl = s0.kind == SK::F || s0.kind == SK::D;
          int vw = 16 / es;  // elements per 16-byte load
          if (cnt <= 32 && cnt % vw == 0 && s0.align % vw == 0) noteRead(g, s0, true);
          if (cnt <= 32 && cnt % vw == 0 && s0.align % vw == 0 && g.out) {
            std::string r = g.fresh("row");
            std::string B = std::to_string(s0.buf);
            // address of the q-th 16-byte block of the row
            std::string addrq = "(const " + std::string(es == 8 ? (fl ? "double2" : "longlong2") : (fl ? "float4" : "int4")) + "*)(" + s0.base + " + " + s0.off + " + q * " + lit(vw) + ")";
            if (s0.stream && g.staged.count(s0.buf) && g.tensorStaged.count(s0.buf))
              addrq = "(const float4*)((const char*)(sb" + B + " + dx_sh" + B + ") + dx_swz((unsigned)(threadIdx.x * " +
                      lit(s0.streamL * es) + " + (" + s0.rowOff + ") * " + lit(es) + " + q * 16), " +
                      lit(g.tensorStaged[s0.buf]) + "))";
            else if (s0.stream && g.staged.count(s0.buf))
              addrq = "(const float4*)(sb" + B + " + dx_sh" + B + " + threadIdx.x * " + lit(s0.streamL) + " + " +
                      s0.rowOff + " + q * " + lit(vw) + ")";
            else if (g.grpInter.count(s0.buf))
              addrq = "(const float4*)((const char*)wt" + B + " + (((unsigned)(" + s0.off + " + q * " + lit(vw) + ") / " +
                      lit(g.grp) + "u) * 32u + dx_gi * " + lit(g.grp) + " + (unsigned)(" + s0.off + " + q * " + lit(vw) +
                      ") % " + lit(g.grp) + "u) * " + lit(es) + ")";
            else if (g.wholeStaged.count(s0.buf))
              addrq = "(const float4*)((const char*)wt" + B + " + dx_swz((unsigned)((" + s0.off + ") * " + lit(es) +
                      " + q * 16), 3))";
            std::string ct = fl ? "dx_f" : ctype(s0.kind);
            std::string vt = es == 8 ? (fl ? "double2" : "longlong2") : (fl ? "float4" : "int4");
            g.line(ct + " " + r + "[" + lit(std::max(1LL, (long long)cnt)) + "];");
            g.line("#pragma unroll");
            g.line("for (int q = 0; q < " + lit(cnt / vw) + "; ++q) { const " + vt + " w = *(const " + vt + "*)(" +
                   addrq + "); " +
                   (vw == 4 ? r + "[4*q] = w.x; " + r + "[4*q+1] = w.y; " + r + "[4*q+2] = w.z; " + r + "[4*q+3] = w.w; }"
                            : r + "[2*q] = w.x; " + r + "[2*q+1] = w.y; }"));
            auto k = std::make_shared<KVal>();
            k->k = KVal::Table;
            k->ty = t;
            Slot ls;
            ls.base = r;
            ls.off = "0";
            ls.kind = s0.kind;
            ls.level = s0.level;
            k->slots.push_back(ls);
            k->level = s0.level;
            return k;
          }
        }
        auto k = std::make_shared<KVal>();
        k->k = KVal::Table;
        k->ty = t;
        size_t n = numLeaves(t);
        int lev = -1;
        for (size_t l = 0; l < n; ++l) {
          k->slots.push_back(slots[base + l]);
          lev = std::max(lev, slots[base + l].level);
        }
        k->level = lev;
        return k;
      }
      case DType::Idx:
        if (t->desc->kind == IndexSetDesc::Kind::Unit) return kUnit();
        [[fallthrough]];
      case DType::Float:
      case DType::Int: {
        const Slot& s = slots[base];
        if (!s.global && s.off == "0" && g.grpPending.count(s.base)) {
          auto k = std::const_pointer_cast<KVal>(
              kScalar(t, "dx_grp_sum<" + lit(g.grpPending[s.base]) + ">(" + s.base + "[0])", s.level));
          k->grpPart = s.base;
          return k;
        }
        std::string v = g.fresh("v");
        std::string ld = (s.global && s.ro) ? "dx_ld(" + s.base + " + " + s.off + ")"
                                            : s.base + "[" + s.off + "]";
        noteRead(g, s, false);
        {
          std::string B = std::to_string(s.buf);
          int eb = (int)storageBytesOf(s.kind, opt.f64);
          std::string ct = ctype(s.kind);
          if (s.global && s.ro && s.stream && g.staged.count(s.buf) && g.tensorStaged.count(s.buf))
            ld = "*(const " + ct + "*)((const char*)(sb" + B + " + dx_sh" + B + ") + dx_swz((unsigned)(threadIdx.x * " +
                 lit(s.streamL * eb) + " + (" + s.rowOff + ") * " + lit(eb) + "), " + lit(g.tensorStaged[s.buf]) + "))";
          else if (s.global && s.ro && s.stream && g.staged.count(s.buf))
            ld = "sb" + B + "[dx_sh" + B + " + threadIdx.x * " + lit(s.streamL) + " + " + s.rowOff + "]";
          else if (s.global && s.ro && g.grpInter.count(s.buf))
            ld = "*(const " + ct + "*)((const char*)wtg" + B + " + ((unsigned)(" + s.off + ") / " + lit(g.grp) + "u) * " +
                 lit(32 * eb) + "u + ((int)((unsigned)(" + s.off + ") % " + lit(g.grp) + "u) - dx_gl) * " + lit(eb) + ")";
          else if (s.global && s.ro && g.wholeStaged.count(s.buf))
            ld = "*(const " + ct + "*)((const char*)wt" + B + " + dx_swz((unsigned)((" + s.off + ") * " + lit(eb) +
                 "), 3))";
        }
        if (s.global && s.ro && s.off.rfind("dx_o", 0) == 0 && isIntLit(s.off.substr(4)) &&
            (s.kind == SK::X || (s.kind == SK::F && !opt.f64))) {
          // streaming read at the thread's own ordinal: served by the
          // per-thread vector prefetch of the U ordinals (see emitKernel)
          g.streamBufs.insert(s.buf);
          if (g.pass == 1 && g.U > 1 && g.grp == 0) ld = "pf" + std::to_string(s.buf) + "_" + s.off.substr(4);
        }
        bool prechecked = false;
        if (!g.serial && s.global && s.ro && s.stream && !opt.f64) {
          // group mode: a row element read at (ordinal, column) where the
          // column is a literal or the lane loop's variable (or its reverse)
          // is served by the chunk prefetch registers gp<id>_<u>
          std::string col;
          long long cv;
          const std::string fwd = "dx_gl", bwd = "(" + lit(g.grpTrip - 1) + " - dx_gl)";
          if (isIntLit(s.rowOff, &cv)) col = lit(cv);
          else if (s.rowOff == "dx_gl") col = fwd;
          else if (!g.curLaneVar.empty() && s.rowOff == g.curLaneVar) col = g.curLaneRev ? bwd : fwd;
          else if (!g.curLaneVar.empty() && g.grpTrip > 0 && s.rowOff == "(" + lit(g.grpTrip - 1) + "LL - " + g.curLaneVar + ")")
            col = g.curLaneRev ? fwd : bwd;
          if (!col.empty()) {
            const std::string key = std::to_string(s.buf) + "|" + col;
            auto it = g.grpStreamId.find(key);
            if (g.pass == 0 && it == g.grpStreamId.end()) {
              g.grpStreamId[key] = (int)g.grpStreams.size();
              const long long chk = (t->k == DType::Idx && s.input) ? size(t->desc) : 0;
              g.grpStreams.push_back({s.buf, s.streamL, s.streamBase, col, s.kind, chk});
            } else if (g.pass == 1 && g.grp > 0 && it != g.grpStreamId.end()) {
              ld = "gp" + std::to_string(it->second) + "_" + std::to_string(s.streamU);
              if (g.grpStreams[it->second].chk > 0) prechecked = true;
            }
          }
        }
        g.line((t->k == DType::Float ? std::string("dx_f") : ctype(s.kind)) + " " + v + " = " + ld + ";");
        if (t->k == DType::Idx && s.input && !prechecked) {
          g.usesErr = true;
          g.line(v + " = dx_chk_idx(" + v + ", " + lit(size(t->desc)) + ", dx_bad);");
        }
        return kScalar(t, v, s.level);
      }
      default: notLowerable("view of " + showType(t));
    }
  }

  // Ordinal expression of an index member value.
  std::string ordinalOf(const KV& v, const DescPtr& d, int* level) {
    switch (d->kind) {
      case IndexSetDesc::Kind::Unit: return "0";
      case IndexSetDesc::Kind::Fin:
      case IndexSetDesc::Kind::Either:
        if (v->k != KVal::Scalar) notLowerable("index member shape");
        *level = std::max(*level, v->level);
        return v->e;
      case IndexSetDesc::Kind::Pair: {
        if (v->k != KVal::Pair) notLowerable("pair index member shape");
        std::string l = ordinalOf(v->a, d->left, level);
        std::string r = ordinalOf(v->b, d->right, level);
        return eAdd(eMul(l, size(d->right)), r);
      }
    }
    return "0";
  }

  // Member value for ordinal expression `o` (fromOrdinalRt, eval.cpp:699-723).
  KV fromOrdinalK(KGen& g, const std::string& o, const DescPtr& d, int level, int loopId,
                  const std::string& rev) {
    switch (d->kind) {
      case IndexSetDesc::Kind::Unit: return kUnit();
      case IndexSetDesc::Kind::Fin:
      case IndexSetDesc::Kind::Either: {
        auto k = std::const_pointer_cast<KVal>(kScalar(tIdx(d), o, level));
        k->loopId = loopId;
        k->rev = rev;
        long long c;
        if (isIntLit(o, &c)) { k->isConst = true; k->ci = c; }
        return k;
      }
      case IndexSetDesc::Kind::Pair: {
        long long rs = size(d->right);
        std::string hi = g.fresh("ih"), lo = g.fresh("il");
        g.line("const long long " + hi + " = (" + o + ") / " + lit(rs) + "LL;");
        g.line("const long long " + lo + " = (" + o + ") % " + lit(rs) + "LL;");
        return kPair(fromOrdinalK(g, hi, d->left, level, -1, ""), fromOrdinalK(g, lo, d->right, level, -1, ""));
      }
    }
    return kUnit();
  }

  KV constK(double f) {
    auto x = std::const_pointer_cast<KVal>(kScalar(tFloat(), litF(f, opt.f64), -1));
    x->isConst = true;
    x->cf = f;
    return x;
  }

  // ---- expressions ----------------------------------------------------

  KV kvalue(KGen& g, const KScope& s, const ValuePtr& v) {
    if (const auto* x = as<VVar>(v)) return lookupK(g, s, x->name, v->span);
    if (const auto* f = as<VLitFloat>(v)) return constK(f->v);
    if (const auto* i = as<VLitInt>(v)) {
      auto x = std::const_pointer_cast<KVal>(kScalar(tInt(), lit(i->v) + "LL", -1));
      x->isConst = true;
      x->ci = i->v;
      return x;
    }
    if (as<VLitUnit>(v)) return kUnit();
    if (const auto* fl = as<VFinLit>(v)) {
      long long n = sizeOf(fl->size, kernelLook(g, s));
      if (fl->ordinal < 0 || fl->ordinal >= n)
        fail(ErrCode::OutOfBounds, "index literal @" + std::to_string(fl->ordinal) +
                                       " is outside Fin " + std::to_string(n), v->span);
      return fromOrdinalK(g, lit(fl->ordinal), descFin(n), -1, -1, lit(n - 1 - fl->ordinal));
    }
    if (const auto* p = as<VPair>(v)) return kPair(kvalue(g, s, p->l), kvalue(g, s, p->r));
    if (as<VInjLeft>(v) || as<VInjRight>(v)) {
      bool left = as<VInjLeft>(v) != nullptr;
      ValuePtr payloadV = left ? as<VInjLeft>(v)->payload : as<VInjRight>(v)->payload;
      ValuePtr otherT = left ? as<VInjLeft>(v)->otherType : as<VInjRight>(v)->otherType;
      KV p = kvalue(g, s, payloadV);
      DescPtr md = memberDesc(p->ty);
      if (md && isIndexSetType(otherT)) {
        DescPtr od = resolveDesc(otherT, kernelLook(g, s));
        int lev = -1;
        std::string o = ordinalOf(p, md, &lev);
        DescPtr d = left ? descEither(md, od) : descEither(od, md);
        return fromOrdinalK(g, left ? o : eAdd(lit(size(od)), o), d, lev, -1, "");
      }
      // data sum: tag + both payloads (the absent one is zero)
      KV other = zeroK(g, resolveType(otherT, kernelLook(g, s)));
      auto k = std::make_shared<KVal>();
      k->k = KVal::Sum;
      k->e = left ? "0" : "1";
      k->isConst = true;
      k->ci = left ? 0 : 1;
      k->a = left ? p : other;
      k->b = left ? other : p;
      k->level = p->level;
      k->ty = tSum(k->a->ty, k->b->ty);
      return k;
    }
    if (const auto* vc = as<VValueCase>(v)) {
      // lazy case over function branches (reference eval.cpp:180-185)
      KV sc = kvalue(g, s, vc->scrutinee);
      const auto* lf = as<VLam>(vc->leftFn);
      const auto* rf = as<VLam>(vc->rightFn);
      if (!lf || !rf) notLowerable("vcase over non-lambda branches", v->span);
      return branchK(g, s, sc, lf->binder, lf->body, rf->binder, rf->body, v->span);
    }
    if (const auto* vw = as<VView>(v)) {
      auto k = std::make_shared<KVal>();
      k->k = KVal::Lazy;
      auto lz = std::make_shared<LazyK>();
      lz->binder = vw->binder;
      lz->desc = resolveDesc(vw->annot, kernelLook(g, s));
      lz->body = vw->body;
      lz->scope = s;
      lz->covered = s.covered;
      lz->cheap = cheapBody(vw->body);
      lz->key = vw->binder.uid;
      k->ty = tTable(lz->desc, staticBodyType(vw->body, kernelLook(g, s), [&](const Name& n) -> DTy {
        for (const KEnvNode* q = s.local.get(); q; q = q->next.get())
          if (q->n == n) return q->v->ty;
        HV h = hlookup(s.host, n);
        return h ? h->ty : nullptr;
      }));
      k->lz = lz;
      return k;
    }
    if (const auto* t = as<VTableLit>(v)) {
      DescPtr d = resolveDesc(t->dom, kernelLook(g, s));
      std::vector<KV> elems;
      for (auto& e : t->elems) elems.push_back(kvalue(g, s, e));
      if (elems.empty()) notLowerable("empty table literal", v->span);
      DTy tt = tTable(d, elems[0]->ty);
      std::vector<Slot> slots = localArrays(g, tt);
      std::vector<LeafInfo> el = leaves(elems[0]->ty);
      for (size_t i = 0; i < elems.size(); ++i) {
        std::vector<Slot> es = slots;
        for (size_t l = 0; l < es.size(); ++l) es[l].off = eAdd(es[l].off, lit((long long)i * el[l].count));
        storeK(g, elems[i], es);
      }
      return viewSlots(g, tt, slots);
    }
    notLowerable("value " + printValue(v), v->span);
  }

  std::vector<Slot> localArrays(KGen& g, const DTy& t, bool zero = false) {
    std::vector<Slot> slots;
    std::string nm = g.fresh("t");
    std::vector<LeafInfo> lv = leaves(t);
    for (size_t l = 0; l < lv.size(); ++l) {
      Slot s;
      s.base = nm + "_" + std::to_string(l);
      s.off = "0";
      s.kind = lv[l].kind;
      g.localDepth[s.base] = g.serial ? 0 : g.depth();
      // a scalar float accumulator starts at -0.0: -0.0 + x == x for every x
      // (+0.0 + x is not an identity for x = -0.0), so the compiler folds the
      // first add and contracts the next multiply-add into one FFMA
      const bool negZero = zero && lv[l].count == 1 && (s.kind == SK::F || s.kind == SK::D);
      g.line(ctype(s.kind) + " " + s.base + "[" + lit(std::max(1LL, (long long)lv[l].count)) + "]" +
             (negZero ? " = {(" + ctype(s.kind) + ")-0.0}" : zero ? " = {}" : "") + ";");
      slots.push_back(s);
    }
    return slots;
  }

  // Store a value into leaf slots (plain stores; used for outputs and locals).
  void storeK(KGen& g, const KV& v, const std::vector<Slot>& slots, size_t base = 0) {
    switch (v->k) {
      case KVal::Unit: return;
      case KVal::Scalar: {
        if (v->ty->k == DType::Idx && v->ty->desc->kind == IndexSetDesc::Kind::Unit) return;
        const Slot& s = slots[base];
        if (s.global) g.writtenBufs.insert(s.buf);
        g.line(s.base + "[" + s.off + "] = " + v->e + ";");
        return;
      }
      case KVal::Pair: {
        size_t na = numLeaves(v->a->ty);
        storeK(g, v->a, slots, base);
        storeK(g, v->b, slots, base + na);
        return;
      }
      case KVal::Sum: {
        const Slot& s0 = slots[base];
        if (s0.global) g.writtenBufs.insert(s0.buf);
        g.line(s0.base + "[" + s0.off + "] = " + v->e + ";");
        storeK(g, v->a, slots, base + 1);
        storeK(g, v->b, slots, base + 1 + numLeaves(v->a->ty));
        return;
      }
      case KVal::Table: {
        std::vector<LeafInfo> lv = leaves(v->ty);
        for (size_t l = 0; l < lv.size(); ++l) {
          const Slot& d = slots[base + l];
          const Slot& src = v->slots[l];
          if (d.global) g.writtenBufs.insert(d.buf);
          std::string q = g.fresh("q");
          if (src.global && src.ro && g.pass == 0) {
            g.nonStream.insert(src.buf);
            if (src.rowW > 0) g.rowUse[src.buf].insert(src.rowW);
            else g.rowBad.insert(src.buf);
          }
          std::string ld = (src.global && src.ro) ? "dx_ld(" + src.base + " + " + eAdd(src.off, q) + ")"
                                                  : src.base + "[" + eAdd(src.off, q) + "]";
          g.line("for (long long " + q + " = 0; " + q + " < " + lit(lv[l].count) + "; ++" + q + ") " +
                 d.base + "[" + eAdd(d.off, q) + "] = " + ld + ";");
        }
        return;
      }
      case KVal::Lazy: {
        // materialize the lazy table element by element
        const auto& lz = v->lz;
        long long n = size(lz->desc);
        std::string q = g.fresh("m");
        int id = openLoop(g, n);
        if (g.loopDepth[id] == 1) g.curLaneVar = q;
        // group mode: materializing into a local table from a lane loop
        // would leave each lane with one element of it
        if (g.pass == 0 && g.loopDepth[id] == 1)
          for (size_t l = base; l < slots.size(); ++l)
            if (!slots[l].global) g.grpOK = false;
        if (laneLoop(g, id)) g.line(loopHead(g, id, q, n));
        else
          g.line(std::string(n <= 32 ? "#pragma unroll\n" : "") + std::string(g.ind * 2, ' ') +
                 "for (int " + q + " = 0; " + q + " < " + lit(n) + "; ++" + q + ") {");
        g.ind++;
        KV idx = fromOrdinalK(g, q, lz->desc, g.loopDepth[id], id, eSub(n - 1, q));
        KV elem = instantiate(g, v, idx);
        std::vector<LeafInfo> el = leaves(elem->ty);
        std::vector<Slot> es(slots.begin() + base, slots.begin() + base + el.size());
        for (size_t l = 0; l < es.size(); ++l) es[l].off = eAdd(es[l].off, eMul(q, el[l].count));
        storeK(g, elem, es);
        g.ind--;
        g.line("}");
        closeLoop(g);
        return;
      }
      default: notLowerable("store of " + showType(v->ty));
    }
  }

  int openLoop(KGen& g, long long trip) {
    int id = ++g.loopCounter;
    g.loopDepth[id] = (int)g.loopStack.size() - (int)g.kernelVars.size() + 1;
    g.loopTrip[id] = trip;
    g.loopStack.push_back(id);
    if (g.loopDepth[id] == 1 && !g.serial) {
      if (g.pass == 0) {
        if (g.grpTrip == 0) g.grpTrip = trip;
        else if (g.grpTrip != trip) g.grpOK = false;
      }
      // every lane loop: the scalar cells that are still zero at its entry
      std::set<std::string> fresh;
      for (auto& [b, d] : g.freshCell) fresh.insert(b);
      g.grpFresh.push_back(fresh);
      g.grpSum.emplace_back();
    }
    return id;
  }
  // Group mode: the loop at depth 1 is a lane loop (one iteration per lane).
  bool laneLoop(KGen& g, int id) const { return g.grp > 0 && g.loopDepth.at(id) == 1; }
  // Header of a depth-1 loop: a C for loop, or in group mode the lane's own
  // iteration.
  std::string loopHead(KGen& g, int id, const std::string& q, long long n, const std::string& ty = "int",
                       bool rev = false) {
    // a loop indexed only through `reverse` runs lane gl on iteration n-1-gl,
    // so its reversed index (the one the body uses) is the lane itself
    if (laneLoop(g, id)) return "{ const " + ty + " " + q + " = " + (rev ? lit(n - 1) + " - dx_gl" : "dx_gl") + ";";
    return "for (" + ty + " " + q + " = 0; " + q + " < " + lit(n) + "; ++" + q + ") {";
  }
  void closeLoop(KGen& g) {
    const int id = g.loopStack.back();
    if (!g.serial && g.loopDepth[id] == 1 && !g.grpSum.empty()) {
      // group mode: outer scalar cells accumulated by the lanes are summed
      // over the group (fixed xor tree) once the lane loop is done
      // Without branches in the body every read of the cell is convergent:
      // the sum is deferred to the reads (a read that only feeds a scalar
      // Accum cell adds the lane partials instead, see accumScalar)
      if (g.grp > 0)
        for (const std::string& c : g.grpSum.back()) {
          if (g.hasBranch) g.line(c + "[0] = dx_grp_sum<" + lit(g.grp) + ">(" + c + "[0]);");
          else g.grpPending[c] = g.grp;
        }
      g.grpFresh.pop_back();
      g.grpSum.pop_back();
      g.curLaneVar.clear();
      g.curLaneRev = false;
    }
    g.loopStack.pop_back();
  }

  // Instantiate a lazy table at index `idx`.
  KV instantiate(KGen& g, const KV& lzv, const KV& idx) {
    const auto& lz = lzv->lz;
    KScope s = lz->scope;
    s.covered = lz->covered;
    if (idx->k == KVal::Scalar && idx->loopId >= 0) s.covered.insert(idx->loopId);
    if (idx->k == KVal::Pair) {
      // pair index from kernel dims: cover all component loops
      std::function<void(const KV&)> cov = [&](const KV& x) {
        if (x->k == KVal::Scalar && x->loopId >= 0) s.covered.insert(x->loopId);
        if (x->k == KVal::Pair) { cov(x->a); cov(x->b); }
      };
      cov(idx);
    }
    s = kbind(s, lz->binder, idx);
    return kexpr(g, s, lz->body, nullptr);
  }

  KV indexK(KGen& g, const KScope& s, const KV& arr, const KV& idx, Span sp) {
    if (arr->k == KVal::Table) {
      int lev = std::max(arr->level, -1);
      std::string o = ordinalOf(idx, arr->ty->desc, &lev);
      DTy et = arr->ty->a;
      std::vector<LeafInfo> el = leaves(et);
      std::vector<Slot> slots = arr->slots;
      for (size_t l = 0; l < slots.size(); ++l) {
        long long b0;
        if (slots[l].stream) {
          slots[l].rowOff = eAdd(slots[l].rowOff, eMul(o, el[l].count));
        } else if (slots[l].global && slots[l].ro && isIntLit(slots[l].off, &b0) &&
                   (o == "dx_o0" || (g.grp > 0 && o.rfind("dx_o", 0) == 0 && isIntLit(o.substr(4))))) {
          slots[l].stream = true;
          slots[l].streamU = std::stoi(o.substr(4));
          slots[l].streamL = el[l].count;
          slots[l].streamBase = b0;
          slots[l].rowOff = "0";
        }
        long long z;
        if (slots[l].global && o == g.dim0Ord && isIntLit(slots[l].off, &z) && z == 0) slots[l].rowW = el[l].count;
        slots[l].off = eAdd(slots[l].off, eMul(o, el[l].count));
        long long oc;
        slots[l].align = gcdll(slots[l].align, isIntLit(o, &oc) ? alignOf(oc * el[l].count) : el[l].count);
        slots[l].level = std::max(slots[l].level, lev);
      }
      return viewSlots(g, et, slots);
    }
    if (arr->k == KVal::Zip) {
      KV ai = indexK(g, s, arr->a, idx, sp), bi = indexK(g, s, arr->b, idx, sp);
      if (arr->zipDepth <= 1) return kPair(ai, bi);
      auto k = std::make_shared<KVal>();
      k->k = KVal::Zip;
      k->zipDepth = arr->zipDepth - 1;
      k->ty = arr->ty->a;
      k->level = std::max(ai->level, bi->level);
      k->a = ai;
      k->b = bi;
      return k;
    }
    if (arr->k == KVal::Lazy) {
      const auto& lz = arr->lz;
      // uniqueness: every active loop is covered by the lazy's creation
      // context or by this index, so each element is computed once.
      std::set<int> cov = lz->covered;
      std::function<void(const KV&)> addCov = [&](const KV& x) {
        if (x->k == KVal::Scalar && x->loopId >= 0) cov.insert(x->loopId);
        if (x->k == KVal::Pair) { addCov(x->a); addCov(x->b); }
      };
      addCov(idx);
      bool unique = true;
      for (int id : g.loopStack)
        if (!cov.count(id)) unique = false;
      if (!unique && !lz->cheap) {
        if (lz->hostOrigin) {
          HV m = splitMaterialize(lz->hostOrigin);
          if (!m) m = materialize(lz->hostOrigin);
          return indexK(g, s, importHost(g, m), idx, sp);
        }
        if (!g.matLocal.count(lz->key)) {
          g.matLocal.insert(lz->key);
          g.redo = true;
        }
      }
      // the same pure lazy element instantiated twice at kernel level in one
      // iteration (a forward tape read by the fused forward and transposed
      // loops) is computed once: its variables are in scope for the rest of
      // the iteration's block
      if (!g.serial && !s.inBranch && g.depth() == 0) {
        std::function<std::string(const KV&)> ik = [&](const KV& x) -> std::string {
          if (x->k == KVal::Scalar) return x->e;
          if (x->k == KVal::Pair) return "(" + ik(x->a) + "," + ik(x->b) + ")";
          if (x->k == KVal::Unit) return "()";
          return "";
        };
        const std::string ix = ik(idx);
        if (!ix.empty()) {
          const void* who = lz->hostOrigin ? (const void*)lz->hostOrigin.get() : (const void*)lz.get();
          const std::string key = std::to_string((unsigned long long)(uintptr_t)who) + "@" + ix;
          auto it = g.instMemo.find(key);
          if (it != g.instMemo.end()) return it->second;
          KV r = instantiate(g, arr, idx);
          g.instMemo[key] = r;
          return r;
        }
      }
      return instantiate(g, arr, idx);
    }
    notLowerable("indexing a value of type " + showType(arr->ty), sp);
  }

  KV kexpr(KGen& g, const KScope& s, const ExprPtr& e, const ValuePtr& annot) {
    if (const auto* l = as<ELet>(e)) {
      KV b = kexpr(g, s, l->bound, l->annot);
      return kexpr(g, kbind(s, l->binder, b), l->body, nullptr);
    }
    if (const auto* r = as<ERet>(e)) return kvalue(g, s, r->value);
    if (const auto* x = as<EIndex>(e)) return indexK(g, s, kvalue(g, s, x->arr), kvalue(g, s, x->idx), e->span);
    if (const auto* x = as<EFst>(e)) {
      KV v = kvalue(g, s, x->v);
      if (v->k != KVal::Pair) notLowerable("fst of a non-pair", e->span);
      return v->a;
    }
    if (const auto* x = as<ESnd>(e)) {
      KV v = kvalue(g, s, x->v);
      if (v->k != KVal::Pair) notLowerable("snd of a non-pair", e->span);
      return v->b;
    }
    if (const auto* b = as<EBinOp>(e)) return binop(g, b->op, kvalue(g, s, b->l), kvalue(g, s, b->r), e->span);
    if (const auto* u = as<EUnOp>(e)) return unop(g, u->op, kvalue(g, s, u->v), e->span);
    if (const auto* f = as<EFor>(e)) return forK(g, s, *f, e, annot);
    if (const auto* c = as<ECase>(e)) return caseK(g, s, *c, e);
    if (const auto* sl = as<ESlice>(e)) return sliceK(g, s, kvalue(g, s, sl->ref), kvalue(g, s, sl->idx), e->span);
    if (const auto* r = as<ERunAccum>(e)) return runAccumK(g, s, *r, e);
    if (const auto* r = as<ERunState>(e)) return runStateK(g, s, *r, e);
    if (const auto* a = as<EAccum>(e)) {
      KV ref = kvalue(g, s, a->ref);
      KV v = kvalue(g, s, a->value);
      if (opt.count) g.line("++dx_cacc;");  // one EAccum (eval.cpp:482-492), any payload
      accumK(g, s, ref, v, e->span);
      return kUnit();
    }
    if (const auto* gt = as<EGet>(e)) {
      KV ref = kvalue(g, s, gt->ref);
      return getK(g, ref, e->span);
    }
    if (const auto* p = as<EPut>(e)) {
      KV ref = kvalue(g, s, p->ref);
      KV v = kvalue(g, s, p->value);
      putK(g, ref, v, e->span);
      return kUnit();
    }
    if (as<EApp>(e)) notLowerable("application (program is not first-order)", e->span);
    notLowerable("expression", e->span);
  }

  KV binop(KGen& g, BinOp op, const KV& l, const KV& r, Span sp) {
    if (l->k != KVal::Scalar || r->k != KVal::Scalar) notLowerable("arithmetic on non-scalars", sp);
    if (opt.count && op != BinOp::Less) g.line("++dx_cops;");  // eval.cpp:500-514 counts each
    int lev = std::max(l->level, r->level);
    if (l->isConst && r->isConst && l->ty->k == DType::Float && r->ty->k == DType::Float) {
      switch (op) {
        case BinOp::Add: return constK(l->cf + r->cf);
        case BinOp::Sub: return constK(l->cf - r->cf);
        case BinOp::Mul: return constK(l->cf * r->cf);
        case BinOp::Div: return constK(l->cf / r->cf);
        case BinOp::Less: break;
      }
    }
    // Identities that only change the sign of a zero result (the reference's
    // `0.0 + x` / `0.0 - x` from zeroed Accum cells and transposed negations):
    // x+0 -> x, 0+x -> x, x-0 -> x, 0-x -> -x, x*1 -> x, 1*x -> x.
    if (l->ty->k == DType::Float && r->ty->k == DType::Float) {
      if (op == BinOp::Add && l->isConst && l->cf == 0.0) return r;
      if ((op == BinOp::Add || op == BinOp::Sub) && r->isConst && r->cf == 0.0) return l;
      if (op == BinOp::Mul && l->isConst && l->cf == 1.0) return r;
      if ((op == BinOp::Mul || op == BinOp::Div) && r->isConst && r->cf == 1.0) return l;
      if (op == BinOp::Sub && l->isConst && l->cf == 0.0) {
        std::string v = g.fresh("f");
        g.line("const dx_f " + v + " = -(" + r->e + ");");
        return kScalar(tFloat(), v, lev);
      }
    }
    std::string v = g.fresh("f");
    const char* o = "+";
    switch (op) {
      case BinOp::Add: o = "+"; break;
      case BinOp::Sub: o = "-"; break;
      case BinOp::Mul: o = "*"; break;
      case BinOp::Div: o = "/"; break;
      case BinOp::Less: {
        // RSumVal{isLeft = !(l < r)} (eval.cpp:509-512): Left is "false",
        // ordinal 0 in Either Unit Unit; Right (ordinal 1) when l < r
        g.line("const int " + v + " = (" + l->e + " < " + r->e + ") ? 1 : 0;");
        auto k = std::const_pointer_cast<KVal>(kScalar(tIdx(boolDesc()), v, lev));
        return k;
      }
    }
    // `__fmul_rn`-style intrinsics keep the compiler from contracting into
    // FMAs differently from the reference's separately rounded ops only in
    // f64 parity mode; f32 mode lets nvcc fuse.
    if (opt.f64) {
      const char* fn = op == BinOp::Add ? "__dadd_rn" : op == BinOp::Sub ? "__dsub_rn" : op == BinOp::Mul ? "__dmul_rn" : "__ddiv_rn";
      g.line("const dx_f " + v + " = " + fn + "(" + l->e + ", " + r->e + ");");
    } else {
      g.line("const dx_f " + v + " = " + l->e + " " + o + " " + r->e + ";");
    }
    return kScalar(tFloat(), v, lev);
  }

  KV unop(KGen& g, UnOp op, const KV& v, Span sp) {
    switch (op) {
      case UnOp::Ordinal: {
        DescPtr d = memberDesc(v->ty);
        if (!d) notLowerable("ord of a non-index", sp);
        int lev = v->level;
        std::string o = ordinalOf(v, d, &lev);
        auto k = std::const_pointer_cast<KVal>(kScalar(tInt(), "((long long)(" + o + "))", lev));
        long long c;
        if (isIntLit(o, &c)) { k->isConst = true; k->ci = c; }
        return k;
      }
      case UnOp::IntToFloat: {
        if (v->isConst) return constK((double)v->ci);
        std::string x = g.fresh("f");
        g.line("const dx_f " + x + " = (dx_f)(" + v->e + ");");
        return kScalar(tFloat(), x, v->level);
      }
      case UnOp::ReverseIndex: {
        DescPtr d = memberDesc(v->ty);
        if (!d) notLowerable("reverse of a non-index", sp);
        if (v->k == KVal::Scalar && !v->rev.empty()) {
          auto k = std::const_pointer_cast<KVal>(kScalar(v->ty, v->rev, v->level));
          k->rev = v->e;
          k->loopId = v->loopId;
          long long c;
          if (isIntLit(k->e, &c)) { k->isConst = true; k->ci = c; }
          return k;
        }
        int lev = v->level;
        std::string o = ordinalOf(v, d, &lev);
        std::string r = g.fresh("r");
        g.line("const long long " + r + " = " + eSub(size(d) - 1, o) + ";");
        int lid = (v->k == KVal::Scalar) ? v->loopId : -1;
        return fromOrdinalK(g, r, d, lev, lid, o);
      }
      case UnOp::Exp:  // frontend_ext: exp / log (libdevice, correctly rounded to <= 2 ulp in f32)
      case UnOp::Log: {
        const char* fn = op == UnOp::Exp ? (opt.f64 ? "exp" : "expf") : (opt.f64 ? "log" : "logf");
        if (v->isConst && v->ty->k == DType::Float) return constK(op == UnOp::Exp ? std::exp(v->cf) : std::log(v->cf));
        std::string x = g.fresh("f");
        g.line("const dx_f " + x + " = " + fn + "(" + v->e + ");");
        return kScalar(tFloat(), x, v->level);
      }
    }
    notLowerable("unary op", sp);
  }

  KV forK(KGen& g, const KScope& s, const EFor& f, const ExprPtr& e, const ValuePtr& annot) {
    DescPtr d = resolveDesc(f.annot, kernelLook(g, s));
    long long n = size(d);
    if (pureBody(f.body) && !g.matLocal.count(f.binder.uid) && !opt.noFusion) {
      auto k = std::make_shared<KVal>();
      k->k = KVal::Lazy;
      auto lz = std::make_shared<LazyK>();
      lz->binder = f.binder;
      lz->desc = d;
      lz->body = f.body;
      lz->scope = s;
      lz->covered = s.covered;
      lz->cheap = cheapBody(f.body);
      lz->key = f.binder.uid;
      k->ty = annotTableType(annot, d, kernelLook(g, s));
      k->lz = lz;
      return k;
    }
    // Emit the loop body into a side buffer first to learn the element type.
    std::string q = g.fresh("j");
    int id = openLoop(g, n);
    const bool laneRev = g.loopDepth[id] == 1 && onlyReversed(f.binder, f.body);
    if (g.loopDepth[id] == 1) { g.curLaneVar = q; g.curLaneRev = laneRev; }
    const bool cand = g.pass == 0 && g.loopDepth[id] == 1 && n >= 64 && g.laneLoopId < 0 && !g.inCand;
    const bool lane = g.pass == 1 && g.warpRow && id == g.laneLoopId;
    if (cand) { g.inCand = true; g.innerCells.clear(); }
    if (lane) { g.inLaneLoop = true; g.innerCells.clear(); g.laneCells.clear(); }
    std::string saved;
    std::string* outer = g.out;
    std::string bodyCode;
    g.out = outer ? &bodyCode : nullptr;
    int savedInd = g.ind;
    g.ind = savedInd + 1;
    KScope bs = s;
    bs.covered.insert(id);
    // a reversed lane loop's reversed index is the lane itself
    KV idx = fromOrdinalK(g, q, d, g.loopDepth[id], id, laneRev && laneLoop(g, id) ? std::string("dx_gl") : eSub(n - 1, q));
    KV elem = kexpr(g, kbind(bs, f.binder, idx), f.body, nullptr);
    // result storage
    DTy tt = tTable(d, elem->ty);
    std::vector<LeafInfo> el = leaves(elem->ty);
    if (cand) {
      g.inCand = false;
      if (el.empty()) g.laneLoopId = id;  // effect-only: a reduction into local cells
    }
    if (lane) g.inLaneLoop = false;
    g.out = outer;
    g.ind = savedInd;
    // group mode: a depth-1 loop producing a local table would leave each
    // lane with one element of it
    if (g.pass == 0 && g.loopDepth[id] == 1 && !el.empty()) g.grpOK = false;
    std::vector<Slot> slots;
    if (!el.empty()) slots = localArrays(g, tt);
    if (g.out) {
      // lane loops: 8 iterations unrolled so their independent loads are in
      // flight together (each lane still adds in ascending q order)
      if (laneLoop(g, id)) g.line(loopHead(g, id, q, n, "int", laneRev));
      else {
        g.line(std::string(lane ? "#pragma unroll 8" : n <= 32 ? "#pragma unroll" : "#pragma unroll 1"));
        if (lane) g.line("for (int " + q + " = dx_lane; " + q + " < " + lit(n) + "; " + q + " += 32) {");
        else g.line("for (int " + q + " = 0; " + q + " < " + lit(n) + "; ++" + q + ") {");
      }
      g.out->append(bodyCode);
    }
    g.ind = savedInd + 1;
    if (!el.empty()) {
      std::vector<Slot> es = slots;
      for (size_t l = 0; l < es.size(); ++l) es[l].off = eMul(q, el[l].count);
      storeK(g, elem, es);
    }
    g.ind = savedInd;
    g.line("}");
    if (lane)  // every lane holds a partial of each cell the loop accumulated
      for (const std::string& c : g.laneCells) g.line(c + "[0] = dx_warp_sum(" + c + "[0]);");
    closeLoop(g);
    if (el.empty()) {
      auto k = std::make_shared<KVal>();
      k->k = KVal::Table;
      k->ty = tt;
      return k;
    }
    return viewSlots(g, tt, slots);
  }

  KV caseK(KGen& g, const KScope& s, const ECase& c, const ExprPtr& e) {
    KV sc = kvalue(g, s, c.scrutinee);
    return branchK(g, s, sc, c.leftBinder, c.leftBody, c.rightBinder, c.rightBody, e->span);
  }

  // Zero of a data type (absent payload of a sum).
  KV zeroK(KGen& g, const DTy& t) {
    switch (t->k) {
      case DType::Float: return constK(0.0);
      case DType::Int: {
        auto x = std::const_pointer_cast<KVal>(kScalar(t, "0LL", -1));
        x->isConst = true;
        return x;
      }
      case DType::Idx: return fromOrdinalK(g, "0", t->desc, -1, -1, lit(size(t->desc) - 1));
      case DType::Unit: return kUnit();
      case DType::Pair: return kPair(zeroK(g, t->a), zeroK(g, t->b));
      case DType::Sum: {
        auto k = std::make_shared<KVal>();
        k->k = KVal::Sum;
        k->e = "0";
        k->isConst = true;
        k->a = zeroK(g, t->a);
        k->b = zeroK(g, t->b);
        k->ty = t;
        return k;
      }
      default: notLowerable("zero of " + showType(t));
    }
  }

  // Two-way branch on an Either index member or a data sum
  // (ECase eval.cpp:382-388, VValueCase eval.cpp:180-185).
  KV branchK(KGen& g, const KScope& s, const KV& sc, const Name& lb, const ExprPtr& lbody, const Name& rb,
             const ExprPtr& rbody, Span sp) {
    KV lpay, rpay;
    std::string cond;
    bool isSum = sc->k == KVal::Sum;
    if (isSum) {
      if (sc->isConst) {
        return sc->ci == 0 ? kexpr(g, kbind(s, lb, sc->a), lbody, nullptr) : kexpr(g, kbind(s, rb, sc->b), rbody, nullptr);
      }
      cond = "(" + sc->e + " == 0)";
    } else {
      if (sc->k != KVal::Scalar || sc->ty->k != DType::Idx || sc->ty->desc->kind != IndexSetDesc::Kind::Either)
        notLowerable("case on a non-sum", sp);
      DescPtr d = sc->ty->desc;
      long long ls = size(d->left);
      if (sc->isConst) {
        if (sc->ci < ls) return kexpr(g, kbind(s, lb, fromOrdinalK(g, lit(sc->ci), d->left, -1, -1, "")), lbody, nullptr);
        return kexpr(g, kbind(s, rb, fromOrdinalK(g, lit(sc->ci - ls), d->right, -1, -1, "")), rbody, nullptr);
      }
      cond = "(" + sc->e + " < " + lit(ls) + ")";
    }
    g.hasBranch = true;
    std::string* outer = g.out;
    int savedInd = g.ind;
    std::string lc, rc;
    KScope bs = s;
    bs.inBranch = true;
    g.out = outer ? &lc : nullptr;
    g.ind = savedInd + 1;
    if (isSum) lpay = sc->a;
    else lpay = fromOrdinalK(g, sc->e, sc->ty->desc->left, sc->level, -1, "");
    KV lv = kexpr(g, kbind(bs, lb, lpay), lbody, nullptr);
    g.out = outer ? &rc : nullptr;
    if (isSum) rpay = sc->b;
    else rpay = fromOrdinalK(g, "(" + sc->e + " - " + lit(size(sc->ty->desc->left)) + ")", sc->ty->desc->right, sc->level, -1, "");
    KV rv = kexpr(g, kbind(bs, rb, rpay), rbody, nullptr);
    g.out = outer;
    g.ind = savedInd;
    // merge results through declared variables
    std::vector<std::string> decls;
    std::vector<std::pair<std::string, std::string>> la, ra;
    std::function<KV(const KV&, const KV&)> merge = [&](const KV& a, const KV& b) -> KV {
      if (a->k == KVal::Unit) return kUnit();
      if (a->k == KVal::Pair && b->k == KVal::Pair) return kPair(merge(a->a, b->a), merge(a->b, b->b));
      if ((a->k == KVal::Scalar || a->k == KVal::Sum) && a->k == b->k) {
        std::string v = g.fresh("c");
        std::string ct = a->ty->k == DType::Float ? "dx_f" : "long long";
        decls.push_back(ct + " " + v + ";");
        la.push_back({v, a->e});
        ra.push_back({v, b->e});
        if (a->k == KVal::Sum) {
          auto k = std::make_shared<KVal>();
          k->k = KVal::Sum;
          k->e = v;
          k->a = merge(a->a, b->a);
          k->b = merge(a->b, b->b);
          k->ty = a->ty;
          k->level = std::max(std::max(a->level, b->level), sc->level);
          return k;
        }
        auto k = std::const_pointer_cast<KVal>(kScalar(a->ty, v, std::max(std::max(a->level, b->level), sc->level)));
        return k;
      }
      if (a->k == KVal::Table && a->slots.empty() && b->k == KVal::Table && b->slots.empty()) return a;
      notLowerable("case branches returning " + showType(a->ty), sp);
    };
    KV res = merge(lv, rv);
    for (auto& dcl : decls) g.line(dcl);
    g.line("if " + cond + " {");
    if (g.out) g.out->append(lc);
    g.ind++;
    for (auto& p : la) g.line(p.first + " = " + p.second + ";");
    g.ind--;
    g.line("} else {");
    if (g.out) g.out->append(rc);
    g.ind++;
    for (auto& p : ra) g.line(p.first + " = " + p.second + ";");
    g.ind--;
    g.line("}");
    return res;
  }

  KV sliceK(KGen& g, const KScope& s, const KV& ref, const KV& idx, Span sp) {
    if (ref->k != KVal::Ref) notLowerable("slice of a non-reference", sp);
    const DTy& pt = ref->ty->a;
    if (pt->k != DType::Table) notLowerable("slice of a non-table reference", sp);
    int lev = -1;
    std::string o = ordinalOf(idx, pt->desc, &lev);
    auto k = std::make_shared<KVal>(*ref);
    k->ty = tRef(pt->a);
    std::vector<LeafInfo> el = leaves(pt->a);
    k->prefixOff = ref->slots.empty() ? "0" : ref->slots[0].off;
    k->prefixLevel = ref->slots.empty() ? -1 : ref->slots[0].level;
    k->lastDim = size(pt->desc);
    for (size_t l = 0; l < k->slots.size(); ++l) {
      k->slots[l].off = eAdd(k->slots[l].off, eMul(o, el[l].count));
      k->slots[l].level = std::max(k->slots[l].level, lev);
    }
    k->path.push_back(idx);
    return k;
  }

  // In-kernel accum-to-map (the kernel twin of tryAccumToMap): the action
  //   <lets not touching r>; let t = for j. (<pure lets>; sl = r!j' ; sl += v); t
  // with j' = j or reverse j and v independent of r makes the final value the
  // table `for j'. v`, kept lazy (inlined at its uses) instead of a local
  // array filled by a loop.  This is the per-row cotangent broadcast of every
  // transposed `sum` inside a kernel (autodiff.cpp:760-772).
  KV accumToMapK(KGen& g, const KScope& s0, const ERunAccum& r, const DTy& payload) {
    if (opt.noFusion || payload->k != DType::Table || payload->a->k != DType::Float) return nullptr;
    const Name rref = r.action.ref;
    std::vector<const ELet*> pre;
    ExprPtr cur = r.action.body;
    const EFor* f = nullptr;
    while (const auto* l = as<ELet>(cur)) {
      if (const auto* ff = as<EFor>(l->bound)) {
        const auto* ret = as<ERet>(l->body);
        const auto* rv = ret ? as<VVar>(ret->value) : nullptr;
        if (!rv || rv->name != l->binder) return nullptr;
        f = ff;
        break;
      }
      for (const Name& n : freeVars(l->bound))
        if (n == rref) return nullptr;
      pre.push_back(l);
      cur = l->body;
    }
    if (!f) return nullptr;
    // the loop body: lets ending in `sl += v`, then a trivial return
    std::vector<const ELet*> lets;
    ExprPtr b = f->body;
    while (const auto* l = as<ELet>(b)) {
      lets.push_back(l);
      b = l->body;
    }
    int accIdx = -1;
    for (size_t i = 0; i < lets.size(); ++i)
      if (as<EAccum>(lets[i]->bound)) {
        if (accIdx >= 0) return nullptr;
        accIdx = (int)i;
      }
    if (accIdx < 0) return nullptr;
    const auto* acc = as<EAccum>(lets[accIdx]->bound);
    const auto* refVar = as<VVar>(acc->ref);
    if (!refVar) return nullptr;
    const ESlice* sl = nullptr;
    for (int i = 0; i < accIdx; ++i)
      if (lets[i]->binder == refVar->name) sl = as<ESlice>(lets[i]->bound);
    const auto* root = sl ? as<VVar>(sl->ref) : nullptr;
    if (!root || root->name != rref) return nullptr;
    const auto* ix = as<VVar>(sl->idx);
    if (!ix) return nullptr;
    bool reversed = false;
    if (ix->name != f->binder) {
      const ELet* rl = nullptr;
      for (int i = 0; i < accIdx; ++i)
        if (lets[i]->binder == ix->name) rl = lets[i];
      const auto* u = rl ? as<EUnOp>(rl->bound) : nullptr;
      const auto* uv = u && u->op == UnOp::ReverseIndex ? as<VVar>(u->v) : nullptr;
      if (!uv || uv->name != f->binder) return nullptr;
      reversed = true;
    }
    for (const Name& n : freeVars(acc->value))
      if (n == rref || n == refVar->name) return nullptr;
    for (size_t i = accIdx + 1; i < lets.size(); ++i)
      if (!as<ERet>(lets[i]->bound)) return nullptr;
    if (!as<ERet>(b)) return nullptr;
    ExprPtr body = eRet(acc->value);
    for (int i = accIdx - 1; i >= 0; --i) {
      if (lets[i]->binder == refVar->name) continue;
      for (const Name& n : freeVars(lets[i]->bound))
        if (n == rref || n == refVar->name) return nullptr;
      if (!pureBody(lets[i]->bound)) return nullptr;
      body = eLet(lets[i]->binder, lets[i]->annot, lets[i]->bound, body);
    }
    DescPtr d = resolveDesc(f->annot, kernelLook(g, s0));
    if (!descEq(d, payload->desc)) return nullptr;
    if (opt.count) g.line("dx_cacc += " + lit(size(d)) + ";");  // the broadcast updates the map replaces
    // evaluate the prefix lets, then the map
    KScope s = s0;
    for (const ELet* l : pre) s = kbind(s, l->binder, kexpr(g, s, l->bound, l->annot));
    Name m = f->binder;
    if (reversed) {
      m = NameSupply::fresh("m");
      body = eLet(f->binder, f->annot, eUn(UnOp::ReverseIndex, vVar(m)), body);
    }
    auto k = std::make_shared<KVal>();
    k->k = KVal::Lazy;
    auto lz = std::make_shared<LazyK>();
    lz->binder = m;
    lz->desc = d;
    lz->body = body;
    lz->scope = s;
    lz->covered = s.covered;
    lz->cheap = cheapBody(body);
    lz->key = m.uid;
    k->ty = payload;
    k->lz = lz;
    auto unitTab = std::make_shared<KVal>();
    unitTab->k = KVal::Table;
    unitTab->ty = tTable(d, tUnit());
    return kPair(unitTab, k);
  }

  KV runAccumK(KGen& g, const KScope& s, const ERunAccum& r, const ExprPtr& e) {
    const auto* ra = as<VRefType>(r.action.refAnnot);
    if (!ra) fail(ErrCode::Internal, "runAccum reached the lowering unannotated", e->span);
    DTy payload = resolveType(ra->payload, kernelLook(g, s));
    if (KV m = accumToMapK(g, s, r, payload)) return m;
    if (opt.count) g.line("++dx_ccell;");
    std::vector<Slot> slots = localArrays(g, payload, true);
    std::vector<LeafInfo> plv = leaves(payload);
    if (g.inCand || g.inLaneLoop)
      for (auto& sl : slots) g.innerCells.insert(sl.base);
    for (size_t l = 0; l < slots.size(); ++l)
      if (plv[l].count == 1) g.freshCell[slots[l].base] = (int)g.loopStack.size();
    auto ref = std::make_shared<KVal>();
    ref->k = KVal::Ref;
    ref->ty = tRef(payload);
    ref->slots = slots;
    KV res = kexpr(g, kbind(s, r.action.ref, ref), r.action.body, nullptr);
    for (auto& sl : slots) g.freshCell.erase(sl.base);
    return kPair(res, viewSlots(g, payload, slots));
  }

  KV runStateK(KGen& g, const KScope& s, const ERunState& r, const ExprPtr& e) {
    KV init = kvalue(g, s, r.init);
    const auto* ra = as<VRefType>(r.action.refAnnot);
    DTy payload = ra ? resolveType(ra->payload, kernelLook(g, s)) : init->ty;
    if (opt.count) g.line("++dx_ccell;");
    std::vector<Slot> slots = localArrays(g, payload);
    storeK(g, init, slots);
    auto ref = std::make_shared<KVal>();
    ref->k = KVal::Ref;
    ref->ty = tRef(payload);
    ref->slots = slots;
    KV res = kexpr(g, kbind(s, r.action.ref, ref), r.action.body, nullptr);
    return kPair(res, viewSlots(g, payload, slots));
  }

  // Global cell leaf as seen by this kernel.
  CellUse& cellUse(KGen& g, int cell, int leaf) {
    auto key = std::make_pair(cell, leaf);
    auto it = g.cellIndex.find(key);
    if (it != g.cellIndex.end()) return g.cells[it->second];
    CellUse cu;
    cu.cell = cell;
    cu.leaf = leaf;
    cu.width = cells[cell].lv[leaf].count;
    g.cells.push_back(cu);
    g.cellIndex[key] = (int)g.cells.size() - 1;
    return g.cells.back();
  }

  // Is `path` exactly the kernel's own iteration (owner computes)?
  bool ownerPath(KGen& g, const KV& ref, int cell) {
    if (g.serial || g.kernelVars.empty()) return false;
    if (ref->path.size() < g.kernelVars.size()) return false;
    DTy t = cells[cell].payload;
    for (size_t i = 0; i < g.kernelVars.size(); ++i) {
      const KV& p = ref->path[i];
      if (p->k != KVal::Scalar || p->loopId != g.kernelVars[i].first) return false;
      if (t->k != DType::Table) return false;
      const KV& kvv = g.kernelVars[i].second;
      if (!kvv || kvv->ty->k != DType::Idx || !descEq(t->desc, kvv->ty->desc)) return false;
      t = t->a;
    }
    return true;
  }

  void accumScalar(KGen& g, const KScope& s, const KV& ref, size_t leaf, const std::string& valE,
                   const KV& val, Span sp) {
    const Slot& sl = ref->slots[leaf];
    if (ref->cell < 0 && !g.serial && g.depth() >= 1) {
      // group mode: a kernel-level local cell accumulated by the lanes must be
      // a scalar that is still zero at the lane loop's entry; each lane then
      // holds a partial and the group sums them after the loop (closeLoop)
      auto ld = g.localDepth.find(sl.base);
      const bool outer = ld == g.localDepth.end() || ld->second == 0;
      if (outer && !g.grpSum.empty()) {
        if (g.pass == 0 && (sl.off != "0" || ref->slots.size() != 1 || !g.grpFresh.back().count(sl.base)))
          g.grpOK = false;
        g.grpSum.back().insert(sl.base);
      }
    }
    if (ref->cell < 0 && g.grpPending.count(sl.base)) {  // written again: sum the partials now
      g.line(sl.base + "[0] = dx_grp_sum<" + lit(g.grpPending[sl.base]) + ">(" + sl.base + "[0]);");
      g.grpPending.erase(sl.base);
    }
    if (ref->cell < 0) {  // thread-local cell
      if ((g.inCand || g.inLaneLoop) && !g.innerCells.count(sl.base)) {
        // an outer cell accumulated by the reduction loop: scalar cells only
        if (sl.off != "0" || ref->slots.size() != 1) g.warpRowOK = false;
        if (g.inLaneLoop) g.laneCells.insert(sl.base);
      }
      auto fr = g.freshCell.find(sl.base);
      if (fr != g.freshCell.end() && fr->second == (int)g.loopStack.size() && sl.off == "0") {
        // first write into a zeroed cell, executed at most once: a store
        g.line(sl.base + "[0] = " + valE + ";");
      } else {
        g.line(sl.base + "[" + sl.off + "] += " + valE + ";");
      }
      if (fr != g.freshCell.end()) g.freshCell.erase(fr);
      return;
    }
    g.warpRowOK = false;  // a plan cell: every lane would add its contribution
    int site = g.accumSiteCounter++;
    CellUse& cu = cellUse(g, ref->cell, sl.cellLeaf);
    // group mode: at kernel level every lane of the group computes the same
    // value; only scalar cells (one guarded register add) are allowed there
    const bool grpTop = !g.serial && g.depth() == 0;
    if (g.pass == 0 && grpTop && cu.width != 1) g.grpOK = false;
    if (g.pass == 0) {
      cu.any = true;
      std::string key;
      if (ownerPath(g, ref, ref->cell))
        for (size_t i = 0; i < g.kernelVars.size(); ++i) key += ref->path[i]->e + ";";
      if (!ownerPath(g, ref, ref->cell) || (!cu.ownKey.empty() && cu.ownKey != key)) cu.allOwner = false;
      else if ((cu.ownKey = key), ref->path.empty() || ref->path[0]->e != g.dim0Ord)
        cu.ownRows = false;  // the row must be the dim-0 ordinal itself (not n-1-o)
      if (!grpTop || s.inBranch || ref->path.size() != g.kernelVars.size()) cu.ownTop = false;
      if (val && val->isConst && val->ty->k == DType::Float && val->cf == std::floor(val->cf) &&
          std::fabs(val->cf) < 1e6) {
        if (!cu.haveConst) { cu.haveConst = true; cu.constVal = val->cf; }
        else if (cu.constVal != val->cf) cu.allConst = false;
      } else {
        cu.allConst = false;
      }
      // row: last path index is the innermost in-thread loop var at depth 1,
      // the prefix is invariant in that loop, not inside a branch.
      bool row = false;
      if (!ref->path.empty() && !s.inBranch && !g.serial) {
        const KV& last = ref->path.back();
        if (last->k == KVal::Scalar && last->loopId >= 0 && !g.loopStack.empty() &&
            last->loopId == g.loopStack.back() && g.loopDepth[last->loopId] == 1 &&
            ref->prefixLevel < 1 && ref->lastDim == g.loopTrip[last->loopId] && ref->lastDim <= 32 &&
            ref->slots.size() == 1 && ref->ty->a->k == DType::Float) {
          if (cu.rowD == 0 || cu.rowD == ref->lastDim) {
            cu.rowD = ref->lastDim;
            row = true;
            cu.rowSitesN++;
          }
        }
      }
      if (!row) cu.allRow = false;
    }
    if (g.pass == 0 || !g.out) return;
    std::string tgt = cu.pname;
    switch (cu.strat) {
      case CellUse::Owner:
      case CellUse::Direct:
        if (cu.overwrite && !cu.firstDone) {
          // every ordinal's first (unconditional) write to its own element
          g.line(tgt + "[" + sl.off + "] = " + valE + ";");
          cu.firstDone = true;
        } else {
          g.line(tgt + "[" + sl.off + "] += " + valE + ";");
        }
        break;
      case CellUse::Reg:
        if (g.grp > 0 && grpTop && val && !val->grpPart.empty() && valE == val->e)  // lane partials
          g.line("rp" + std::to_string(&cu - &g.cells[0]) + " += " + val->grpPart + "[0];");
        else if (g.grp > 0 && grpTop)
          g.line("if (dx_gl == 0) rp" + std::to_string(&cu - &g.cells[0]) + " += " + valE + ";");
        else
          g.line("rp" + std::to_string(&cu - &g.cells[0]) + " += " + valE + ";");
        break;
      case CellUse::Smem:
        g.line("dx_red_smem(&sm" + std::to_string(&cu - &g.cells[0]) + "[" + sl.off + "], " + valE + ");");
        break;
      case CellUse::Count:
        g.line("dx_count_smem(sm" + std::to_string(&cu - &g.cells[0]) + ", (int)(" + sl.off + "), __activemask());");
        break;
      case CellUse::Row:
      case CellUse::TileRow: {
        const KV& last = ref->path.back();
        if (g.grp > 0) {
          // lane (group gi, column c) adds into its own word of the warp's
          // table row: copy gi holds columns [gi*G, gi*G + G)
          // (byte offsets from the lane's own word: one multiply-add per
          // access; the column term folds away when it is the lane column)
          g.line("*(float*)((char*)dx_wtl" + std::to_string(&cu - &g.cells[0]) + " + ((unsigned)((" + ref->prefixOff +
                 ") / " + lit(cu.rowD) + "LL) << 7) + ((int)(" + last->e + ") - dx_gl) * 4) += " + valE + ";");
          break;
        }
        int rid = g.rowSiteCounter++;
        std::string rv = "rowv" + std::to_string(rid), rk = "rowk" + std::to_string(rid);
        // one row site per cell, directly in the loop over the row's columns:
        // every column is written exactly once per iteration
        g.line(rv + "[" + last->e + "] " + (cu.rowSitesN == 1 ? "=" : "+=") + " " + valE + ";");
        g.line(rk + " = (int)((" + ref->prefixOff + ") / " + lit(cu.rowD) + "LL);");
        if ((int)g.rowSites.size() <= rid)
          g.rowSites.push_back({(int)(&cu - &g.cells[0]), cu.rowD, rid});
        break;
      }
      case CellUse::Global:
        g.line("dx_red_global(&" + tgt + "[" + sl.off + "], " + valE + ");");
        break;
    }
    (void)site;
    (void)sp;
  }

  static KV subRef(const KV& ref, const DTy& payload, size_t from, size_t n) {
    auto r = std::make_shared<KVal>(*ref);
    r->ty = tRef(payload);
    r->slots.assign(ref->slots.begin() + from, ref->slots.begin() + from + n);
    if (!r->slots.empty()) {
      r->prefixOff = r->slots[0].off;
      r->prefixLevel = r->slots[0].level;
    }
    return r;
  }

  void accumK(KGen& g, const KScope& s, const KV& ref, const KV& v, Span sp) {
    if (ref->k != KVal::Ref) notLowerable("accumulation into a non-reference", sp);
    switch (v->k) {
      case KVal::Unit: return;
      case KVal::Scalar:
        if (v->ty->k != DType::Float) notLowerable("accumulating a non-float", sp);
        if (v->isConst && v->cf == 0.0) return;  // += 0 (zero views of transposed pairs)
        accumScalar(g, s, ref, 0, v->e, v, sp);
        return;
      case KVal::Pair: {
        // refs to pair payloads: each component owns its own leaves
        const DTy& pt = ref->ty->a;
        if (pt->k != DType::Pair) notLowerable("pair accumulated into a non-pair reference", sp);
        size_t na = numLeaves(pt->a);
        size_t nb = numLeaves(pt->b);
        accumK(g, s, subRef(ref, pt->a, 0, na), v->a, sp);
        accumK(g, s, subRef(ref, pt->b, na, nb), v->b, sp);
        return;
      }
      case KVal::Table:
      case KVal::Lazy: {
        // elementwise over the table: slice + accumulate
        DescPtr d = v->k == KVal::Lazy ? v->lz->desc : v->ty->desc;
        long long n = size(d);
        std::string q = g.fresh("a");
        int id = openLoop(g, n);
        if (g.loopDepth[id] == 1) g.curLaneVar = q;
        if (!laneLoop(g, id)) g.line(std::string(n <= 32 ? "#pragma unroll" : "#pragma unroll 1"));
        g.line(loopHead(g, id, q, n));
        g.ind++;
        KScope bs = s;
        bs.covered.insert(id);
        KV idx = fromOrdinalK(g, q, d, g.loopDepth[id], id, eSub(n - 1, q));
        KV sub = sliceK(g, bs, ref, idx, sp);
        KV elem = indexK(g, bs, v, idx, sp);
        accumK(g, bs, sub, elem, sp);
        g.ind--;
        g.line("}");
        closeLoop(g);
        return;
      }
      default: notLowerable("accumulating " + showType(v->ty), sp);
    }
  }

  KV getK(KGen& g, const KV& ref, Span sp) {
    if (ref->k != KVal::Ref) notLowerable("get of a non-reference", sp);
    if (g.inCand) g.warpRowOK = false;
    std::vector<Slot> slots = ref->slots;
    if (ref->cell >= 0) {
      if (!g.serial) fail(ErrCode::StateInParallel, "state cell read inside a parallel kernel", sp);
      g.stateCells.insert(ref->cell);
      for (size_t l = 0; l < slots.size(); ++l) {
        slots[l].base = param(g, cells[ref->cell].bufs[slots[l].cellLeaf], true);
        slots[l].ro = false;
      }
    }
    return viewSlots(g, ref->ty->a, slots);
  }

  void putK(KGen& g, const KV& ref, const KV& v, Span sp) {
    g.warpRowOK = false;
    if (g.pass == 0 && !g.serial && g.depth() >= 1)  // group mode: a lane writing replicated state
      for (const Slot& sl : ref->slots) {
        auto ld = g.localDepth.find(sl.base);
        if (ld == g.localDepth.end() || ld->second == 0) g.grpOK = false;
      }
    if (ref->k != KVal::Ref) notLowerable("put of a non-reference", sp);
    std::vector<Slot> slots = ref->slots;
    for (const Slot& sl : slots) g.grpPending.erase(sl.base);  // overwritten: partials dropped
    if (ref->cell >= 0) {
      if (!g.serial) fail(ErrCode::StateInParallel, "state cell written inside a parallel kernel", sp);
      g.stateCells.insert(ref->cell);
      for (size_t l = 0; l < slots.size(); ++l) {
        slots[l].base = param(g, cells[ref->cell].bufs[slots[l].cellLeaf], true);
        slots[l].buf = cells[ref->cell].bufs[slots[l].cellLeaf];
        slots[l].global = true;
      }
    }
    storeK(g, v, slots);
  }

  // ------------------------------------------------------------------
  // Kernel assembly.

  struct KernelBody {
    // emits the per-iteration body; returns the element value (for outputs)
    std::function<KV(KGen&, const KScope&)> body;
    DescPtr desc;         // iteration space (nullptr: serial single thread)
    std::vector<DescPtr> dims;
    std::vector<bool> dimReversed;
    std::vector<Name> dimBinders;
    HEnvP env;
    std::string note;
  };

  std::string kernelName() { return "dxk_" + std::to_string(kernelCounter++); }

  // Effect-only parallel loops waiting to be fused horizontally with the
  // next independent loop over the same index set (one pass over HBM).
  std::vector<KernelBody> pending;
  bool flushing = false;

  // The buffer's pending zero-fill, if the last step touching it is one: the
  // next kernel can overwrite the buffer instead (the step is dropped).
  bool takeZero(int b) {
    for (size_t i = plan.steps.size(); i-- > 0;) {
      Step& st = plan.steps[i];
      bool refs = st.buf == b || st.buf2 == b;
      for (auto& a : st.args) refs |= (a.k == KArg::Buf || a.k == KArg::TMap) && a.buf == b;
      if (!refs) continue;
      if (st.k == Step::Zero && st.buf == b && st.off == 0 && !st.dead &&
          (st.elems <= 0 || st.elems >= plan.bufs[b].elems)) {
        st.dead = true;
        return true;
      }
      return false;
    }
    return false;
  }

  void addStep(const Step& st) {
    if (st.k != Step::Zero && !pending.empty() && !flushing) flushPending();
    plan.steps.push_back(st);
  }
  void flushPending();

  // Generates, registers and schedules one kernel made of one or more parts
  // sharing an iteration space.  Outputs (the loop's element at its ordinal)
  // only for single-part kernels.
  HV emitKernel(const std::vector<KernelBody>& parts, bool serial, const std::vector<int>* intoBufs,
                const std::vector<long long>* intoOffs);
  HV requestKernel(const KernelBody& kb, bool serial, const std::vector<int>* intoBufs,
                   const std::vector<long long>* intoOffs);
  struct Analysis {
    DTy elemTy;
    std::set<int> reads, writes;
    std::set<int> cells;
  };
  Analysis analyze(const std::vector<KernelBody>& parts, bool serial);
  KV runParts(KGen& g, const std::vector<KernelBody>& parts, bool serial, int U,
              std::vector<int>& outBufs, std::vector<long long>& outOffs,
              const std::vector<int>* intoBufs, const std::vector<long long>* intoOffs);

  void decideStrategies(KGen& g);
};

// ---------------------------------------------------------------------------

static int tileThreads() {
  return 256;
}


void Lowering::decideStrategies(KGen& g) {
  int esize = opt.f64 ? 8 : 4;
  const int smemCap = 160 * 1024;
  g.threads = opt.threads;
  int warps = std::max(1, opt.threads / 32);
  int smemUsed = 0;
  bool privatized = false;
  bool tileRowTaken = false;
  for (size_t i = 0; i < g.cells.size(); ++i) {
    CellUse& cu = g.cells[i];
    SK kind = cells[cu.cell].lv[cu.leaf].kind;
    if (g.serial) { cu.strat = CellUse::Direct; continue; }
    if (kind != SK::F) { cu.strat = CellUse::Global; continue; }
    if (cu.allOwner) { cu.strat = CellUse::Owner; continue; }
    privatized = true;
    if (cu.width == 1) { cu.strat = CellUse::Reg; g.usesScratch = true; continue; }
    if (cu.allConst && cu.haveConst && cu.width <= 32768 && smemUsed + cu.width * 4 <= smemCap) {
      cu.strat = CellUse::Count;
      cu.smemOff = smemUsed;
      smemUsed += (int)cu.width * 4;
      continue;
    }
    if (cu.allRow && cu.rowD > 0 && cu.rowSitesN == 1 && !opt.noRowScatter && !tileRowTaken) {
      long long Kr = cu.width / cu.rowD;
      const int NT = tileThreads();
      long long need = (long long)NT * (cu.rowD + 1) * esize + (NT / 32) * Kr * 4 + (Kr + 1) * 4 + NT * 4 + 64;
      if (Kr >= 1 && Kr <= 256 && (NT % Kr == 0 || Kr <= 32) && cu.width <= 16 * NT &&
          smemUsed + need <= smemCap) {
        cu.strat = CellUse::TileRow;
        cu.smemOff = smemUsed;
        smemUsed += (int)need;
        tileRowTaken = true;
        continue;
      }
    }
    if (cu.allRow && cu.rowD > 0 && !opt.noRowScatter) {
      long long need = (long long)warps * cu.width * esize;
      if (smemUsed + need + warps * (32 * 33 + 32) * esize <= smemCap) {
        cu.strat = CellUse::Row;
        cu.smemOff = smemUsed;
        smemUsed += (int)need;
        continue;
      }
    }
    if (cu.width * esize <= 48 * 1024 && smemUsed + cu.width * esize <= smemCap) {
      cu.strat = CellUse::Smem;
      cu.smemOff = smemUsed;
      smemUsed += (int)(cu.width * esize);
      continue;
    }
    privatized = false;
    cu.strat = CellUse::Global;
  }
  if (g.serial || !privatized) return;
  if (tileRowTaken) {
    // tile-sorted rows: block-uniform tiles (see dx_tile_rows)
    const int NT = tileThreads();
    g.threads = NT;
    int off = 0;
    for (auto& cu : g.cells) {
      if (cu.strat == CellUse::Smem) { cu.smemOff = off; off += (int)(cu.width * esize); }
      if (cu.strat == CellUse::Count) { cu.smemOff = off; off += (int)(cu.width * 4); }
      if (cu.strat == CellUse::Row) cu.strat = CellUse::Smem, cu.smemOff = off, off += (int)(cu.width * esize);
    }
    for (auto& cu : g.cells) {
      if (cu.strat != CellUse::TileRow) continue;
      long long Kr = cu.width / cu.rowD;
      cu.smemOff = (off + 15) / 16 * 16;
      // WarpTab: warp-private interleaved tables, no sort and no block
      // barrier per tile (dx_warp_tab); needs (K+1) x 128 B per warp.
      long long wt = (long long)(NT / 32) * (Kr + 1) * 128;
      cu.warpTab = !opt.f64 && cu.rowD % 4 == 0 && 32 % cu.rowD == 0 &&
                   cu.smemOff + wt + (long long)NT * cu.rowD * 4 <= (NT > 256 ? 200 : 150) * 1024;
      cu.vec4 = cu.warpTab || (!opt.f64 && cu.rowD % 4 == 0 && Kr * (cu.rowD / 4) <= NT);
      if (cu.warpTab) {
        off = cu.smemOff + (int)(wt + (long long)NT * cu.rowD * 4);
        continue;
      }
      off = cu.smemOff + (int)(NT * (cu.rowD + 1) * esize + (NT / 32) * Kr * 4 + (Kr + 1) * 4 + NT * 4 + 64);
    }
    return;
  }
  // Privatized cells: fat persistent blocks (one or two per SM), so that the
  // per-block partials, and their finalize, stay small.  Row tables are
  // per warp: recompute their offsets for the chosen block size.
  for (int T : {1024, 512}) {
    int w = T / 32;
    int used = 0;
    long long maxD = 0;
    for (auto& cu : g.cells) {
      if (cu.strat == CellUse::Smem) used += (int)(cu.width * esize);
      if (cu.strat == CellUse::Count) used += (int)(cu.width * 4);
      if (cu.strat == CellUse::Row) { used += (int)(w * cu.width * esize); maxD = std::max(maxD, cu.rowD); }
    }
    if (maxD > 0) used += w * (32 * (int)(maxD + 1) + 32) * esize + 16;
    if (used > 200 * 1024) continue;
    g.threads = T;
    int off = 0;
    for (auto& cu : g.cells) {
      if (cu.strat == CellUse::Smem) { cu.smemOff = off; off += (int)(cu.width * esize); }
      if (cu.strat == CellUse::Count) { cu.smemOff = off; off += (int)(cu.width * 4); }
      if (cu.strat == CellUse::Row) { cu.smemOff = off; off += (int)(w * cu.width * esize); }
    }
    return;
  }
}

KV Lowering::runParts(KGen& g, const std::vector<KernelBody>& parts, bool serial, int U,
                      std::vector<int>& outBufs, std::vector<long long>& outOffs,
                      const std::vector<int>* intoBufs, const std::vector<long long>* intoOffs) {
  if (g.pass == 0) {
    g.warpRowOK = true;
    g.laneLoopId = -1;
    g.grpOK = true;
    g.grpTrip = 0;
    g.grpStreams.clear();
    g.grpStreamId.clear();
    g.grpStreamBad.clear();
  }
  g.inCand = g.inLaneLoop = false;
  g.localDepth.clear();
  g.instMemo.clear();
  g.grpPending.clear();
  if (g.pass == 0) g.hasBranch = false;
  g.grpFresh.clear();
  g.grpSum.clear();
  g.loopStack.clear();
  g.loopDepth.clear();
  g.loopTrip.clear();
  g.kernelVars.clear();
  g.loopCounter = 0;
  g.tmp = 0;
  g.rowSiteCounter = 0;
  g.accumSiteCounter = 0;
  g.lines = 0;
  const KernelBody& kb0 = parts[0];
  long long total = serial ? 1 : size(kb0.desc);
  // kernel dims: loop ids 1..k at depth 0, shared by all parts
  std::vector<int> dimIds;
  if (!serial) {
    for (size_t i = 0; i < kb0.dims.size(); ++i) {
      int id = ++g.loopCounter;
      g.loopDepth[id] = 0;
      g.loopTrip[id] = size(kb0.dims[i]);
      g.loopStack.push_back(id);
      dimIds.push_back(id);
    }
  }
  KV last;
  for (int u = 0; u < (serial ? 1 : U); ++u) {
    std::string o = serial ? "0" : "dx_o" + std::to_string(u);
    g.instMemo.clear();  // each ordinal's block has its own variables
    for (auto& cu : g.cells) cu.firstDone = false;  // each ordinal's first owner write stores
    if (!serial && U > 1) g.line(g.grp > 0 ? "if (dx_ok" + std::to_string(u) + ") {" : "if (" + o + " < dx_hi) {");
    if (!serial && U > 1) g.ind++;
    // dimension ordinals of this iteration
    std::vector<std::string> ords;
    if (!serial) {
      long long rest = total;
      for (size_t i = 0; i < kb0.dims.size(); ++i) {
        rest = size(kb0.dims[i]) ? rest / size(kb0.dims[i]) : 0;  // Fin 0: empty space
        if (kb0.dims.size() == 1) ords.push_back(o);
        else {
          std::string ord = g.fresh("kd");
          g.line("const long long " + ord + " = (" + o + " / " + lit(rest) + "LL) % " + lit(size(kb0.dims[i])) + "LL;");
          ords.push_back(ord);
        }
      }
    }
    if (!ords.empty()) g.dim0Ord = ords[0];
    for (const KernelBody& kb : parts) {
      KScope s;
      s.host = kb.env;
      g.kernelVars.clear();
      if (!serial) {
        for (size_t i = 0; i < kb.dims.size(); ++i) {
          int id = dimIds[i];
          s.covered.insert(id);
          long long n = size(kb.dims[i]);
          KV v;
          if (kb.dimReversed[i]) v = fromOrdinalK(g, eSub(n - 1, ords[i]), kb.dims[i], 0, id, ords[i]);
          else v = fromOrdinalK(g, ords[i], kb.dims[i], 0, id, eSub(n - 1, ords[i]));
          g.kernelVars.push_back({id, v});
          s = kbind(s, kb.dimBinders[i], v);
        }
      }
      KV elem = kb.body(g, s);
      last = elem;
      if (!elem) continue;
      std::vector<LeafInfo> el = leaves(elem->ty);
      if (el.empty() || g.pass != 1) continue;
      if (outBufs.empty()) {
        if (intoBufs) {
          outBufs = *intoBufs;
          outOffs = *intoOffs;
        } else {
          DTy tt = serial ? elem->ty : tTable(kb.desc, elem->ty);
          for (auto& l : leaves(tt)) {
            outBufs.push_back(newBuf(BufDecl::Output, l.kind, l.count));
            outOffs.push_back(0);
          }
        }
      }
      // output ordinal: the binders' own ordinal (reversed dims store reversed)
      std::string oo = "0";
      if (!serial) {
        std::string acc = "0";
        for (size_t i = 0; i < g.kernelVars.size(); ++i) {
          int lev = 0;
          std::string oi = ordinalOf(g.kernelVars[i].second, kb.dims[i], &lev);
          acc = eAdd(eMul(acc, size(kb.dims[i])), oi);
        }
        oo = acc;
      }
      std::vector<Slot> slots;
      for (size_t l = 0; l < el.size(); ++l) {
        Slot s2;
        s2.buf = outBufs[l];
        s2.base = param(g, outBufs[l], true);
        s2.off = eAdd(lit(outOffs[l]), eMul(oo, el[l].count));
        s2.global = true;
        s2.kind = plan.bufs[outBufs[l]].kind;
        slots.push_back(s2);
      }
      storeK(g, elem, slots);
    }
    if (!serial && U > 1) g.ind--;
    if (!serial && U > 1) g.line("}");
  }
  return last;
}

Lowering::Analysis Lowering::analyze(const std::vector<KernelBody>& parts, bool serial) {
  KGen g(*this);
  g.serial = serial;
  Analysis a;
  std::vector<int> ob;
  std::vector<long long> oo;
  for (int it = 0; it < 8; ++it) {
    g.pass = 0;
    g.redo = false;
    g.out = nullptr;
    g.cells.clear();
    g.cellIndex.clear();
    g.params.clear();
    g.writtenBufs.clear();
    KV e = runParts(g, parts, serial, 1, ob, oo, nullptr, nullptr);
    if (e) a.elemTy = e->ty;
    if (!g.redo) break;
  }
  for (auto& [b, n] : g.params) (g.writtenBufs.count(b) ? a.writes : a.reads).insert(b);
  for (auto& cu : g.cells) {
    a.cells.insert(cu.cell);
    for (int b : cells[cu.cell].bufs) a.writes.insert(b);
  }
  return a;
}

void Lowering::flushPending() {
  if (pending.empty() || flushing) return;
  flushing = true;
  std::vector<KernelBody> parts;
  parts.swap(pending);
  emitKernel(parts, false, nullptr, nullptr);
  flushing = false;
}

HV Lowering::requestKernel(const KernelBody& kb, bool serial, const std::vector<int>* intoBufs,
                           const std::vector<long long>* intoOffs) {
  bool effectOnly = false;
  if (!serial && !intoBufs && !opt.noFusion) {
    Analysis a = analyze({kb}, false);
    effectOnly = !a.elemTy || leaves(a.elemTy).empty();
    if (effectOnly) {
      for (auto ci : a.cells) cellToDevice(ci);
      bool fuse = !pending.empty();
      if (fuse) {
        const KernelBody& p0 = pending[0];
        if (p0.dims.size() != kb.dims.size()) fuse = false;
        for (size_t i = 0; fuse && i < kb.dims.size(); ++i)
          if (!descEq(p0.dims[i], kb.dims[i])) fuse = false;
        if (fuse) {
          Analysis pa = analyze(pending, false);
          for (int b : a.reads) if (pa.writes.count(b)) fuse = false;
          for (int b : pa.reads) if (a.writes.count(b)) fuse = false;
          for (int c : a.cells) if (pa.cells.count(c)) fuse = false;
        }
      }
      if (!fuse) flushPending();
      pending.push_back(kb);
      auto h = std::make_shared<HVal>();
      h->k = HVal::Buf;
      h->ty = tTable(kb.desc, a.elemTy ? a.elemTy : tUnit());
      return h;
    }
  }
  flushPending();
  return emitKernel({kb}, serial, intoBufs, intoOffs);
}

HV Lowering::emitKernel(const std::vector<KernelBody>& parts, bool serial, const std::vector<int>* intoBufs,
                        const std::vector<long long>* intoOffs) {
  const KernelBody& kb0 = parts[0];
  long long total = serial ? 1 : size(kb0.desc);
  // an empty index set (Fin 0): no iteration, no effect, empty outputs -- the
  // reference's enumerate is empty too (eval.cpp:295-308); cells keep their
  // zeroOfType value (eval.cpp:452-464).  Nothing is compiled or launched.
  const bool empty = !serial && total == 0;
  std::string kname = kernelName();
  std::vector<int> outBufs;
  std::vector<long long> outOffs;
  DTy elemTy;
  std::string note;
  for (auto& p : parts) note += (note.empty() ? "" : " + ") + p.note;

  KGen g(*this);
  g.serial = serial;
  g.total = total;
  g.sharded = !serial && plan.world > 1;
  // pass 0: analysis, repeated until the local materialization set is stable
  for (int it = 0; it < 8; ++it) {
    g.pass = 0;
    g.redo = false;
    g.out = nullptr;
    g.cells.clear();
    g.cellIndex.clear();
    g.rowSites.clear();
    g.params.clear();
    g.writtenBufs.clear();
    g.streamBufs.clear();
    g.stateCells.clear();
    g.streamUse.clear();
    g.nonStream.clear();
    g.rowUse.clear();
    g.rowBad.clear();
    g.needAlign.clear();
    g.usesErr = false;
    g.usesScratch = false;
    KV e = runParts(g, parts, serial, 1, outBufs, outOffs, intoBufs, intoOffs);
    if (e) elemTy = e->ty;
    if (!g.redo) break;
  }
  decideStrategies(g);
  bool hasRow = false;
  for (auto& cu : g.cells) hasRow |= cu.strat == CellUse::Row || cu.strat == CellUse::TileRow;
  // TMA staging for block-uniform tile kernels: rows read at the kernel
  // ordinal stream in by cp.async.bulk (double-buffered, one tile ahead);
  // small read-only gather tables are copied to shared memory once.
  g.tile = false;
  for (auto& cu : g.cells) g.tile |= cu.strat == CellUse::TileRow || cu.strat == CellUse::Row;
  g.staged.clear();
  g.wholeStaged.clear();
  g.tensorStaged.clear();
  if (g.tile) {
    int es = opt.f64 ? 8 : 4;
    long long budget = 96 * 1024;
    for (auto& [b, lb] : g.streamUse) {
      if (g.nonStream.count(b)) continue;
      int eb = (int)storageBytesOf(plan.bufs[b].kind, opt.f64);
      bool aligned = (lb.first * eb) % 16 == 0 && (lb.second * eb) % 16 == 0;
      if (g.needAlign.count(b) && !aligned) continue;
      long long stage = (long long)g.threads * lb.first * eb + 32;
      if (2 * stage > budget) continue;
      budget -= 2 * stage + 2048;
      g.staged.insert(b);
      long long rowB = lb.first * eb;
      if (g.needAlign.count(b) && !opt.f64 && plan.bufs[b].kind == SK::F && aligned &&
          (rowB == 32 || rowB == 64 || rowB == 128) && g.threads % 256 == 0)
        g.tensorStaged[b] = rowB == 32 ? 1 : rowB == 64 ? 3 : 7;
    }
    for (int b : g.nonStream) {
      if (g.streamUse.count(b)) continue;
      long long bytes = plan.bufs[b].elems * (long long)storageBytesOf(plan.bufs[b].kind, opt.f64);
      bytes = (bytes + 127) / 128 * 128;  // swizzled 128-byte rows
      if (bytes <= 0 || bytes > 16 * 1024 || bytes > budget) continue;
      budget -= bytes;
      g.wholeStaged.insert(b);
    }
    (void)es;
  }
  for (auto& cu : g.cells) {
    cu.aliasStage = -1;
    if (cu.strat != CellUse::TileRow || !cu.vec4) continue;
    for (auto& [b, mask] : g.tensorStaged)
      if (g.streamUse[b].first == cu.rowD && plan.bufs[b].kind == SK::F)
        cu.aliasStage = b;
  }
  // Group mode (see KGen::grpOK): the row scatter of a WarpTab cell with
  // G = D lanes per ordinal; every other cell must be a scalar register cell.
  // Measured on B200 (scripts/kmicro2.cu, k-means 1M x 16, K = 64, back to
  // back): 20.4 us per step against 30.6 us for the thread-per-ordinal TMA
  // tile kernel (its row transposes cost 113 shared wavefronts per 32 points;
  // the group layout needs 64 and no tile barrier).
  g.grp = 0;
  g.grpRowCell = -1;
  int grpWarps = 0;
  if (!serial && !opt.count && g.grpOK && kb0.dims.size() == 1 && !opt.f64 && g.grpTrip >= 4 && g.grpTrip <= 32 &&
      32 % g.grpTrip == 0 && total > 0) {
    bool ok = true;
    for (size_t i = 0; i < g.cells.size(); ++i) {
      const CellUse& cu = g.cells[i];
      if (cu.strat == CellUse::Reg) continue;
      // any row-scatter cell (TileRow, or Row / Smem when the tile sort's
      // limits ruled TileRow out) becomes the group's lane-owned table
      if (cu.allRow && cu.rowSitesN == 1 && cu.rowD == g.grpTrip && g.grpRowCell < 0 && cu.width % cu.rowD == 0 &&
          cells[cu.cell].lv[cu.leaf].kind == SK::F &&
          (cu.strat == CellUse::TileRow || cu.strat == CellUse::Row || cu.strat == CellUse::Smem)) {
        g.grpRowCell = (int)i;
        continue;
      }
      ok = false;
    }
    if (ok && g.grpRowCell >= 0) {
      const CellUse& rc = g.cells[g.grpRowCell];
      const long long tabB = (rc.width / rc.rowD + 1) * 128;
      grpWarps = (int)std::min<long long>(20, (200 * 1024) / tabB);
      if (grpWarps >= 4) g.grp = (int)g.grpTrip;
    }
  }
  if (g.grp > 0) {
    CellUse& rc = g.cells[g.grpRowCell];
    rc.strat = CellUse::TileRow;
    rc.warpTab = true;
    rc.vec4 = true;
    rc.aliasStage = -1;
    rc.smemOff = 0;
    g.threads = grpWarps * 32;
    g.tile = false;
    g.staged.clear();
    g.wholeStaged.clear();
    g.grpInter.clear();
    g.tensorStaged.clear();
    // small read-only gather tables (centroids) are copied into shared memory
    // once per block (LDS with 32-bit addresses instead of L1 gathers); a
    // table of whole G-element rows is stored as 32/G interleaved copies, so
    // the two (or more) groups of a warp reading different rows at their lane
    // columns hit disjoint banks
    long long room = 224 * 1024 - (long long)grpWarps * ((rc.width / rc.rowD) + 1) * 128;
    for (int b : g.nonStream) {
      if (g.streamUse.count(b)) continue;
      long long bytes = plan.bufs[b].elems * (long long)storageBytesOf(plan.bufs[b].kind, opt.f64);
      const bool inter = plan.bufs[b].elems % g.grpTrip == 0;
      if (inter) bytes *= 32 / g.grpTrip;
      bytes = (bytes + 127) / 128 * 128;  // swizzled 128-byte rows
      if (bytes <= 0 || bytes > (inter ? 32 : 16) * 1024 || bytes + 16 > room) continue;
      room -= bytes + 16;
      g.wholeStaged.insert(b);
      if (inter) g.grpInter.insert(b);
    }
  }
  // warp per ordinal for short outer loops over long reductions (row sums)
  g.warpRow = !serial && !opt.count && g.warpRowOK && g.laneLoopId >= 0 && g.cells.empty() && !hasRow && !g.tile &&
              kb0.dims.size() == 1 && total <= 148LL * 256;
  // tiny bodies: several consecutive ordinals per thread (vector loads, ILP)
  int U = g.warpRow ? 1 : (!serial && !hasRow && g.lines <= 16 && g.loopCounter <= (int)kb0.dims.size()) ? 4 : 1;
  // group mode: 16 ordinals per group and chunk, all their prefetch loads
  // in flight together (one 128-byte warp load per ordinal pair at G = 16)
  if (g.grp > 0) U = 16;
  g.grpU = U;
  // more 16-byte loads in flight per thread for the tiniest bodies (histograms):
  // one load per thread and grid-stride step leaves HBM latency exposed
  if (U == 4 && g.lines <= 8) {
    U = 12;  // measured on the 2^28-key histogram: 4 -> 240 us, 8 -> 215, 12 -> 209, 16 -> 242
  }
  // cells must be on the device before this kernel
  for (auto& cu : g.cells) cellToDevice(cu.cell);
  for (int ci : g.stateCells) cellToDevice(ci);
  for (auto& cu : g.cells) {
    Cell& c = cells[cu.cell];
    cu.targetBuf = c.bufs[cu.leaf];
    if (g.sharded) {
      cu.targetBuf = newBuf(BufDecl::Temp, plan.bufs[c.bufs[cu.leaf]].kind, cu.width);
      Step z; z.k = Step::Zero; z.buf = cu.targetBuf; z.elems = cu.width; addStep(z);
    }
    // an owner-computed cell whose every element is written by its own
    // ordinal, unconditionally, right after the cell's zero-fill: the first
    // write stores (no zero pass over HBM, no read-modify-write)
    cu.overwrite = cu.firstDone = false;
    if (cu.strat == CellUse::Owner && cu.any && cu.ownTop && !serial && !g.sharded && plan.world == 1 && !opt.count &&
        g.grp == 0 && parts.size() == 1 && total == cu.width && takeZero(cu.targetBuf))
      cu.overwrite = true;
  }
  // pass 1: emission
  std::string body;
  g.pass = 1;
  g.U = U;
  std::set<int> streams = g.streamBufs;
  g.out = &body;
  g.ind = serial ? 2 : 3;
  g.params.clear();
  g.writtenBufs.clear();
  g.rowSites.clear();
  for (auto& cu : g.cells) cu.pname = param(g, cu.targetBuf, true);
  runParts(g, parts, serial, U, outBufs, outOffs, intoBufs, intoOffs);
  if (opt.count) param(g, plan.countBuf, true);

  // Partial buffers for privatized strategies.
  for (size_t i = 0; i < g.cells.size(); ++i) {
    CellUse& cu = g.cells[i];
    if (cu.strat == CellUse::Reg || cu.strat == CellUse::Smem || cu.strat == CellUse::Row ||
        cu.strat == CellUse::Count || cu.strat == CellUse::TileRow) {
      SK pk = cu.strat == CellUse::Count ? SK::U32 : SK::F;
      cu.partialBuf = newBuf(BufDecl::Partial, pk, 0);
      plan.bufs[cu.partialBuf].partialWidth = cu.width;
    }
  }

  // In-kernel finalize: the blocks fold the partials themselves, last block
  // done per group of DX_LBD_GB, then the last group (dx_lbd_* in
  // dx_device.cuh): no grid barrier, no cooperative launch, no extra kernel.
  bool fold = false;
  for (auto& cu : g.cells) fold |= cu.partialBuf >= 0;
  if (serial || total == 0) fold = false;
  // Two forms (measured on B200, bench.py back to back): narrow partial rows
  // (k-means: 1025 words) fold fastest after a grid barrier, every block
  // folding 8 columns (31.0 vs 38.8 us per 1M-point step); wide rows
  // (histogram: 4096 counters x ~1200 blocks = 19 MB of partials) fold
  // fastest last-block-done, groups folding as their blocks finish (193 vs
  // 218 us per 2^28-key step).
  long long widest = 0;
  for (auto& cu : g.cells)
    if (cu.partialBuf >= 0) widest = std::max(widest, cu.width);
  const bool lbd = fold && widest >= 2048;
  const bool coop = fold && !lbd;
  int tickBuf = -1, syncBuf = -1;
  std::vector<int> gpartBuf(g.cells.size(), -1);
  if (coop) {
    syncBuf = newBuf(BufDecl::Sync, SK::U32, 2 * 16 * 8);  // DX_NCTR counters, one 128-byte line each
    param(g, syncBuf, true);
  }
  if (lbd) {
    tickBuf = newBuf(BufDecl::Sync, SK::U32, 1026);  // DX_LBD_WORDS
    param(g, tickBuf, true);
    for (size_t i = 0; i < g.cells.size(); ++i) {
      CellUse& cu = g.cells[i];
      if (cu.partialBuf < 0) continue;
      gpartBuf[i] = newBuf(BufDecl::Partial, cu.strat == CellUse::Count ? SK::I : SK::D, 0);
      plan.bufs[gpartBuf[i]].partialWidth = cu.width;  // grid x width (>= groups x width)
      param(g, gpartBuf[i], true);
    }
  }

  // Assemble source.
  std::ostringstream src;
  std::function<std::string(const std::string&, const std::string&)> grpLoad;
  std::function<std::string(const std::string&)> grpPrefetch;
  std::function<bool(const KGen::GrpStream&)> grpBcast;
  int warps = std::max(1, g.threads / 32);
  int esize = opt.f64 ? 8 : 4;
  int smem = 0;
  long long maxRowD = 0;
  for (auto& cu : g.cells) {
    if (cu.strat == CellUse::Smem) smem = std::max<int>(smem, cu.smemOff + (int)(cu.width * esize));
    if (cu.strat == CellUse::Count) smem = std::max<int>(smem, cu.smemOff + (int)(cu.width * 4));
    if (cu.strat == CellUse::Row) {
      smem = std::max<int>(smem, cu.smemOff + (int)(warps * cu.width * esize));
      maxRowD = std::max(maxRowD, cu.rowD);
    }
    if (cu.strat == CellUse::TileRow && cu.warpTab) {
      long long Kr = cu.width / cu.rowD;
      long long wt = (long long)(g.threads / 32) * (Kr + 1) * 128;
      long long etB = (cu.aliasStage >= 0 || g.grp > 0) ? 0 : (long long)g.threads * cu.rowD * 4;
      smem = std::max<int>(smem, cu.smemOff + (int)(wt + etB));
    } else if (cu.strat == CellUse::TileRow) {
      long long Kr = cu.width / cu.rowD;
      long long etB = cu.aliasStage >= 0 ? 0 : (long long)g.threads * (cu.rowD + 1) * esize;
      smem = std::max<int>(smem, cu.smemOff + (int)(etB + (g.threads / 32) * Kr * 4 + (Kr + 1) * 4 + g.threads * 4 + 64));
    }
  }
  int tileCell = -1;
  for (size_t i = 0; i < g.cells.size(); ++i)
    if (g.cells[i].strat == CellUse::TileRow) tileCell = (int)i;
  // WarpTab kernels fed by the TMA ring: warps share nothing but the stages
  int stageOff = (smem + 15) / 16 * 16;
  if (maxRowD > 0) smem = stageOff + warps * (32 * (int)(maxRowD + 1) + 32) * esize;
  // TMA staging areas
  std::map<int, int> stageAt, wholeAt;
  std::map<int, long long> stageElems;
  for (int b : g.staged) {
    int eb = (int)storageBytesOf(plan.bufs[b].kind, opt.f64);
    long long L = g.streamUse[b].first;
    if (g.tensorStaged.count(b)) {
      // swizzled TMA tiles: 1024-byte aligned stages of exactly one box
      long long elems = ((long long)g.threads * L * eb + 1023) / 1024 * 1024 / eb;
      smem = (smem + 1023) / 1024 * 1024;
      stageAt[b] = smem;
      stageElems[b] = elems;
      smem += (int)(2 * elems * eb);
      continue;
    }
    long long elems = ((long long)g.threads * L * eb + 32 + 15) / 16 * 16 / eb;  // + shift slack
    smem = (smem + 15) / 16 * 16;
    stageAt[b] = smem;
    stageElems[b] = elems;
    smem += (int)(2 * elems * eb);
  }
  if (!g.tensorStaged.empty()) smem += 1024;  // dynamic smem base is only 16-byte aligned
  for (int b : g.wholeStaged) {
    int eb = (int)storageBytesOf(plan.bufs[b].kind, opt.f64);
    smem = (smem + 15) / 16 * 16;
    wholeAt[b] = smem;
    // the copy is swizzled within 128-byte rows (dx_swz(.., 3)): a partial
    // last row still spans the whole row; group-interleaved copies take 32/G
    // times the table
    const long long copies = g.grpInter.count(b) ? 32 / g.grp : 1;
    smem += (int)((plan.bufs[b].elems * eb * copies + 127) / 128 * 128);
  }

  src << "// " << note << "\n";
  src << "extern \"C\" __global__ void __launch_bounds__(" << (serial ? 32 : g.threads) << ") " << kname << "(";
  std::vector<KArg> args;
  std::vector<std::string> aligns;
  bool first = true;
  auto comma = [&] { if (!first) src << ", "; first = false; };
  for (auto& [buf, pname] : g.params) {
    comma();
    bool w = g.writtenBufs.count(buf) > 0;
    std::string ct = ctype(plan.bufs[buf].kind);
    if (w) src << ct << "* " << pname;
    else src << "const " << ct << "* __restrict__ " << pname;
    // every plan buffer is a cuMemAlloc base (256-byte aligned); offsets live
    // in the index expressions, so the compiler may vectorize
    aligns.push_back("  " + pname + " = (" + (w ? "" : "const ") + ct + "*)__builtin_assume_aligned(" + pname + ", 16);\n");
    KArg a; a.k = KArg::Buf; a.buf = buf; args.push_back(a);
  }
  for (auto& [b, mask] : g.tensorStaged) {
    comma();
    src << "const __grid_constant__ dx_tmap tm" << b;
    KArg a;
    a.k = KArg::TMap;
    a.buf = b;
    a.rowLen = g.streamUse[b].first;
    a.off = g.streamUse[b].second;
    a.rows = (plan.bufs[b].elems - a.off) / a.rowLen;
    a.boxRows = std::min(g.threads, 256);  // TMA box dims are <= 256: larger tiles take several boxes
    a.swizzle = (mask + 1) * 16;
    args.push_back(a);
  }
  for (size_t i = 0; i < g.cells.size(); ++i) {
    CellUse& cu = g.cells[i];
    if (cu.partialBuf < 0) continue;
    comma();
    src << (cu.strat == CellUse::Count ? "unsigned" : "dx_f") << "* __restrict__ part" << i;
    KArg a; a.k = KArg::Buf; a.buf = cu.partialBuf; args.push_back(a);
  }
  comma();
  src << "long long dx_lo, long long dx_hi, int* dx_err) {\n";
  { KArg a; a.k = KArg::I64; a.special = 1; args.push_back(a); }
  { KArg a; a.k = KArg::I64; a.special = 2; args.push_back(a); }
  { KArg a; a.k = KArg::Buf; a.buf = plan.errFlagBuf; args.push_back(a); }
  for (auto& al : aligns) src << al;
  src << "  int dx_bad = 0;\n";
  if (opt.count) src << "  unsigned long long dx_cops = 0, dx_cacc = 0, dx_ccell = 0;\n";

  if (serial) {
    src << "  if (blockIdx.x != 0 || threadIdx.x != 0) return;\n  {\n" << body << "  }\n";
    if (opt.count)
      src << "  dx_count_add((unsigned long long*)" << g.params[plan.countBuf] << ", dx_cops, dx_cacc, dx_ccell);\n";
    src << "  if (dx_bad) atomicOr(dx_err, 1);\n}\n\n";
  } else {
    src << "  const int dx_lane = threadIdx.x & 31, dx_warp = threadIdx.x >> 5;\n";
    src << "  (void)dx_lane; (void)dx_warp;\n";
    // programmatic dependent launch: wait for the previous launch on the
    // stream before touching anything it may write -- at entry, or (opt-in
    // pipelining, DXL_F_PIPELINE) after the streaming loop when the kernel
    // reads program inputs only
    bool lateWait = opt.pipeline && g.grp > 0;
    for (auto& [b, pname] : g.params)
      if (!g.writtenBufs.count(b) && plan.bufs[b].role != BufDecl::Input && plan.bufs[b].role != BufDecl::Const)
        lateWait = false;
    if (!lateWait) src << "  dx_pdl_wait();\n";
    if (!lateWait && coop)
      src << "  __shared__ unsigned long long dx_ep;\n  if (threadIdx.x == 0) dx_ep = dx_bar_epoch((const unsigned long long*)"
          << g.params[syncBuf] << ");\n";
    if (g.grp > 0) {
      // group mode: chunk c of a warp = ordinals [c*CH, c*CH + CH), group gi
      // takes ordinals c*CH + u*GPW + gi (u < U); the rows it reads at its
      // ordinal are prefetched one chunk ahead into registers (double
      // buffer a/b), the first two chunks before the shared-memory set-up
      const int G = g.grp, GPW = 32 / G;
      const long long CH = (long long)GPW * U;
      src << "  const int dx_gl = dx_lane % " << G << ", dx_gi = dx_lane / " << G << ";\n";
      src << "  const long long dx_glo = dx_lo, dx_nch = (dx_hi - dx_lo + " << CH - 1 << ") / " << CH
          << ", dx_nfull = (dx_hi - dx_lo) / " << CH << ";\n";
      // chunk c goes to block c mod grid (every SM gets the same number of
      // chunks, +-1), then to the block's warps in turn: at any time the
      // grid streams one window of the input (measured: per-warp contiguous
      // ranges, which balance the warps exactly, were 1 us slower at 1M
      // points)
      src << "  const long long dx_w0 = (long long)blockIdx.x + (long long)gridDim.x * dx_warp, dx_tw = (long long)gridDim.x * "
          << g.threads / 32 << ";\n";
      // a per-ordinal scalar (a literal column: k-means assignments) is
      // loaded once per chunk, lane l taking ordinal l, and shuffled to the
      // groups (CH <= 32)
      auto bcast = [&, CH](const KGen::GrpStream& gs) {
        long long c;
        return CH <= 32 && isIntLit(gs.col, &c);
      };
      for (size_t id = 0; id < g.grpStreams.size(); ++id) {
        const auto& gs = g.grpStreams[id];
        std::string ct = gs.kind == SK::F ? "dx_f" : ctype(gs.kind);
        if (bcast(gs)) src << "  " << ct << " gpa" << id << "k = 0, gpb" << id << "k = 0;\n";
        else src << "  " << ct << " gpa" << id << "[" << U << "], gpb" << id << "[" << U << "];\n";
      }
      grpBcast = bcast;
      grpLoad = [&, CH, GPW, bcast](const std::string& ab, const std::string& chE) {
        // full chunks: unguarded loads at constant offsets from one base per
        // stream (the compiler folds u into the address immediate); the
        // ragged chunk guards each ordinal
        std::ostringstream o;
        o << "{ const long long dx_cn = " << chE << ", dx_c0 = dx_glo + dx_cn * " << CH << "LL + dx_gi;\n";
        for (int full = 1; full >= 0; --full) {
          o << (full ? "      if (dx_cn < dx_nfull) {\n" : "      } else {\n");
          for (size_t id = 0; id < g.grpStreams.size(); ++id) {
            const auto& gs = g.grpStreams[id];
            std::string ct = gs.kind == SK::F ? "dx_f" : ctype(gs.kind);
            if (bcast(gs)) {
              std::string ldx = "__ldcs(" + g.params[gs.buf] + " + (dx_c0 - dx_gi + dx_lane) * " + lit(gs.L) + "LL + " +
                                lit(gs.base) + "LL + " + gs.col + ")";
              if (gs.chk > 0) ldx = "dx_chk_idx(" + ldx + ", " + lit(gs.chk) + ", dx_bad)";
              o << "        gp" << ab << id << "k = dx_lane < " << CH << (full ? "" : " && dx_c0 - dx_gi + dx_lane < dx_hi")
                << " ? " << ldx << " : (" << ct << ")0;\n";
              continue;
            }
            o << "        const " << ct << "* dx_b" << id << " = " << g.params[gs.buf] << " + dx_c0 * " << gs.L << "LL + "
              << gs.base << "LL + " << gs.col << ";\n";
            for (int u = 0; u < U; ++u) {
              std::string ldx = "__ldcs(dx_b" + std::to_string(id) + " + " + lit((long long)u * GPW * gs.L) + ")";
              if (gs.chk > 0) ldx = "dx_chk_idx(" + ldx + ", " + lit(gs.chk) + ", dx_bad)";
              if (full) o << "        gp" << ab << id << "[" << u << "] = " << ldx << ";\n";
              else
                o << "        gp" << ab << id << "[" << u << "] = dx_c0 + " << u * GPW << " < dx_hi ? " << ldx << " : (" << ct
                  << ")0;\n";
            }
          }
        }
        o << "      }\n    }\n";
        return o.str();
      };
      // the register prefetch is one chunk deep; the TMA engine pulls the
      // chunk after it into L2 (lane 0, whole rows of every stream) so the
      // register loads are served by L2 (measured: 20.8 -> 20.2 us per 1M
      // points)
      grpPrefetch = [&, CH](const std::string& chE) {
        std::ostringstream o;
        o << "if (dx_lane == 0 && " << chE << " < dx_nfull) { const long long dx_pc = dx_glo + (" << chE << ") * " << CH << "LL;";
        std::set<int> done;
        for (size_t id = 0; id < g.grpStreams.size(); ++id) {
          const auto& gs = g.grpStreams[id];
          const long long bytes = CH * gs.L * (long long)storageBytesOf(gs.kind, opt.f64);
          if (bytes % 16 || bytes > (1 << 20) || !done.insert(gs.buf).second) continue;
          o << " dx_l2_prefetch(" << g.params[gs.buf] << " + dx_pc * " << gs.L << "LL, " << bytes << "u);";
        }
        o << " }\n";
        return o.str();
      };
      src << "  " << grpPrefetch("dx_w0 + 2 * dx_tw") << "  " << grpPrefetch("dx_w0 + 3 * dx_tw");
      src << "  if (dx_w0 < dx_nch) " << grpLoad("a", "dx_w0");
      src << "  if (dx_w0 + dx_tw < dx_nch) " << grpLoad("b", "dx_w0 + dx_tw");
    }
    if (smem > 0 && g.tensorStaged.empty()) src << "  extern __shared__ __align__(16) unsigned char dx_smem[];\n";
    if (smem > 0 && !g.tensorStaged.empty()) {
      // swizzled TMA destinations need 1024-byte alignment
      src << "  extern __shared__ __align__(1024) unsigned char dx_smem_raw[];\n";
      src << "  unsigned char* dx_smem = dx_smem_raw + ((1024u - (dx_smem_addr(dx_smem_raw) & 1023u)) & 1023u);\n";
    }
    bool needSync = false;
    if (!g.staged.empty()) {
      src << "  __shared__ __align__(8) unsigned long long dx_bar[2], dx_empty[2];\n";
      for (int b : g.staged) {
        std::string ct = ctype(plan.bufs[b].kind);
        src << "  " << ct << "* sb" << b << " = (" << ct << "*)(dx_smem + " << stageAt[b] << ");\n";
      }
      src << "  if (threadIdx.x == 0) { dx_mbar_init(&dx_bar[0], 1); dx_mbar_init(&dx_bar[1], 1); dx_mbar_init(&dx_empty[0], "
          << g.threads / 32 << "); dx_mbar_init(&dx_empty[1], " << g.threads / 32 << "); dx_fence_mbar_init(); }\n";
      // thread 0 streams the rows of tile `tb` into stage `stg` (16-byte
      // aligned superset of the byte range; readers add the shift)
      src << "  auto dx_issue = [&](int stg, long long tb) {\n";
      src << "    const long long r0 = dx_lo + tb, r1 = (r0 + " << g.threads << " < dx_hi) ? r0 + " << g.threads << " : dx_hi;\n";
      src << "    unsigned tot = 0;\n";
      for (int b : g.staged) {
        int eb = (int)storageBytesOf(plan.bufs[b].kind, opt.f64);
        auto lb = g.streamUse[b];
        std::string B = std::to_string(b);
        if (g.tensorStaged.count(b)) {
          src << "    tot += " << (long long)g.threads * lb.first * eb << "u;  // full box (OOB rows zero-filled)\n";
          continue;
        }
        src << "    const long long a" << B << " = ((r0 * " << lb.first << "LL + " << lb.second << "LL) * " << eb
            << "LL) & ~15LL;\n";
        src << "    const long long n" << B << " = ((((r1 * " << lb.first << "LL + " << lb.second << "LL) * " << eb
            << "LL) + 15LL) & ~15LL) - a" << B << ";\n";
        src << "    tot += (unsigned)n" << B << ";\n";
      }
      src << "    dx_mbar_expect_tx(&dx_bar[stg], tot);\n";
      for (int b : g.staged) {
        std::string B = std::to_string(b);
        if (g.tensorStaged.count(b)) {
          for (int bx = 0; bx < std::max(1, g.threads / 256); ++bx)
            src << "    dx_tma_2d(sb" << B << " + stg * " << stageElems[b] << "LL + " << (long long)bx * 256 * g.streamUse[b].first
                << "LL, &tm" << B << ", 0, (int)r0 + " << bx * 256 << ", &dx_bar[stg]);\n";
          continue;
        }
        src << "    dx_bulk_g2s(sb" << B << " + stg * " << stageElems[b] << "LL, (const char*)p" << B << " + a" << B
            << ", (unsigned)n" << B << ", &dx_bar[stg]);\n";
      }
      src << "  };\n";
      // first tile in flight before the shared-memory set-up below
      if (tileCell >= 0 || g.tile)
        src << "  if (threadIdx.x == 0 && (long long)blockIdx.x * blockDim.x < (dx_hi - dx_lo + " << (U - 1) << ") / " << U << ") dx_issue(0, (long long)blockIdx.x * blockDim.x);\n";
      needSync = true;
    }
    for (size_t i = 0; i < g.cells.size(); ++i) {
      CellUse& cu = g.cells[i];
      std::string I = std::to_string(i);
      switch (cu.strat) {
        case CellUse::Reg: src << "  dx_f rp" << I << " = 0;\n"; break;
        case CellUse::Smem:
          src << "  dx_f* sm" << I << " = (dx_f*)(dx_smem + " << cu.smemOff << ");\n";
          src << "  for (int t = threadIdx.x; t < " << cu.width << "; t += blockDim.x) sm" << I << "[t] = 0;\n";
          needSync = true;
          break;
        case CellUse::Count:
          src << "  unsigned* sm" << I << " = (unsigned*)(dx_smem + " << cu.smemOff << ");\n";
          src << "  for (int t = threadIdx.x; t < " << cu.width << "; t += blockDim.x) sm" << I << "[t] = 0u;\n";
          needSync = true;
          break;
        case CellUse::TileRow: {
          long long Kr = cu.width / cu.rowD;
          int nacc = (int)((cu.width + g.threads - 1) / g.threads);
          long long et = cu.aliasStage >= 0 ? 0 : (long long)g.threads * (cu.rowD + 1) * esize;
          if (cu.warpTab) {
            long long wt = (long long)(g.threads / 32) * (Kr + 1) * 32;
            src << "  float* wtab" << I << " = (float*)(dx_smem + " << cu.smemOff << ");\n";
            src << "  dx_f* et" << I << " = (dx_f*)(dx_smem + " << cu.smemOff + wt * 4 << ");\n";
            src << "  for (int t = threadIdx.x; t < " << wt / 4 << "; t += blockDim.x) reinterpret_cast<float4*>(wtab" << I
                << ")[t] = make_float4(0.f, 0.f, 0.f, 0.f);\n";
            if (g.grp > 0)
              src << "  float* dx_wt" << I << " = wtab" << I << " + dx_warp * " << (Kr + 1) * 32 << ";\n  float* dx_wtl" << I
                  << " = dx_wt" << I << " + dx_gi * " << g.grp << " + dx_gl;\n";
            needSync = true;
            break;
          }
          if (cu.vec4) src << "  float4 acc" << I << " = make_float4(0.f, 0.f, 0.f, 0.f);\n";
          else {
            src << "  dx_f acc" << I << "[" << nacc << "];\n";
            src << "#pragma unroll\n  for (int t = 0; t < " << nacc << "; ++t) acc" << I << "[t] = 0;\n";
          }
          src << "  dx_f* et" << I << " = (dx_f*)(dx_smem + " << cu.smemOff << ");\n";
          src << "  int* wc" << I << " = (int*)(dx_smem + " << cu.smemOff + et << ");\n";
          src << "  int* st" << I << " = wc" << I << " + " << (g.threads / 32) * Kr << ";\n";
          src << "  int* pm" << I << " = st" << I << " + " << Kr + 1 << ";\n";
          if (cu.vec4) {
            src << "  for (int t = threadIdx.x; t < " << (g.threads / 32) * Kr << "; t += blockDim.x) wc" << I << "[t] = 0;\n";
            needSync = true;
          }
          break;
        }
        case CellUse::Row:
          src << "  dx_f* rt" << I << " = (dx_f*)(dx_smem + " << cu.smemOff << ");\n";
          src << "  for (int t = threadIdx.x; t < " << warps * cu.width << "; t += blockDim.x) rt" << I << "[t] = 0;\n";
          needSync = true;
          break;
        default: break;
      }
    }
    if (maxRowD > 0)
      src << "  dx_f* dx_stage = (dx_f*)(dx_smem + " << stageOff << ") + dx_warp * " << 32 * (maxRowD + 1) + 32 << ";\n";
    for (int b : g.wholeStaged) {
      std::string ct = ctype(plan.bufs[b].kind);
      src << "  " << ct << "* wt" << b << " = (" << ct << "*)(dx_smem + " << wholeAt[b] << ");\n";
      if (g.grpInter.count(b)) {
        const int G = g.grp;
        src << "  for (int t = threadIdx.x; t < " << plan.bufs[b].elems << "; t += blockDim.x) { const " << ct << " v = p" << b
            << "[t];\n#pragma unroll\n    for (int c = 0; c < " << 32 / G << "; ++c) wt" << b << "[(t / " << G << ") * 32 + c * " << G
            << " + t % " << G << "] = v; }\n";
        src << "  const " << ct << "* wtg" << b << " = wt" << b << " + dx_gi * " << G << " + dx_gl;\n";
        needSync = true;
        continue;
      }
      src << "  for (int t = threadIdx.x; t < " << plan.bufs[b].elems << "; t += blockDim.x) *(" << ct
          << "*)((char*)wt" << b << " + dx_swz((unsigned)(t * " << storageBytesOf(plan.bufs[b].kind, opt.f64)
          << "), 3)) = p" << b << "[t];\n";
      needSync = true;
    }
    if (needSync) src << "  __syncthreads();\n";
    // warp-uniform grid-stride loop over groups of U consecutive ordinals
    src << "  const long long dx_n = (dx_hi - dx_lo + " << (U - 1) << ") / " << U << ";\n";
    src << "  const long long dx_stride = (long long)gridDim.x * blockDim.x;\n";
    if (g.grp == 0 && (tileCell >= 0 || g.tile) && !g.staged.empty()) {
      // TMA pipeline: tile t+1 is in flight while tile t is computed
      src << "  int dx_it = 0;\n";
      src << "  for (long long dx_base = (long long)blockIdx.x * blockDim.x; dx_base < dx_n; dx_base += dx_stride, ++dx_it) {\n";
      src << "    const int dx_stg = dx_it & 1;\n";
      src << "    if (threadIdx.x == 0 && dx_base + dx_stride < dx_n) { dx_fence_proxy_async(); dx_issue(dx_stg ^ 1, dx_base + dx_stride); }\n";
      for (int b : g.staged) {
        int eb = (int)storageBytesOf(plan.bufs[b].kind, opt.f64);
        auto lb = g.streamUse[b];
        if (g.tensorStaged.count(b)) {
          src << "    const int dx_sh" << b << " = dx_stg * " << stageElems[b] << ";\n";
          continue;
        }
        src << "    const int dx_sh" << b << " = dx_stg * " << stageElems[b] << " + (int)((((dx_lo + dx_base) * "
            << lb.first << "LL + " << lb.second << "LL) * " << eb << "LL) & 15LL) / " << eb << ";\n";
      }
      src << "    dx_mbar_wait(&dx_bar[dx_stg], (unsigned)((dx_it >> 1) & 1));\n";
      src << "    const long long dx_s = dx_base + threadIdx.x;\n";
    } else if (g.grp == 0 && tileCell >= 0) {
      // block-uniform tiles: every thread runs the same trip count
      src << "  for (long long dx_base = (long long)blockIdx.x * blockDim.x; dx_base < dx_n; dx_base += dx_stride) {\n";
      src << "    const long long dx_s = dx_base + threadIdx.x;\n";
    } else if (g.grp > 0) {
      const int GPW = 32 / g.grp;
      const long long CH = (long long)GPW * U;
      auto chunk = [&](const std::string& ab, const std::string& cb) {
        std::ostringstream o;
        o << "      const long long dx_cb = " << cb << ";\n";
        for (size_t id = 0; id < g.grpStreams.size(); ++id) {
          const auto& gs = g.grpStreams[id];
          std::string ct = gs.kind == SK::F ? "dx_f" : ctype(gs.kind);
          for (int u = 0; u < U; ++u) {
            if (grpBcast(gs))
              o << "      const " << ct << " gp" << id << "_" << u << " = __shfl_sync(DX_FULL, gp" << ab << id << "k, "
                << u * GPW << " + dx_gi);\n";
            else
              o << "      const " << ct << " gp" << id << "_" << u << " = gp" << ab << id << "[" << u << "];\n";
          }
        }
        for (int u = 0; u < U; ++u)
          o << "      const long long dx_o" << u << " = dx_glo + dx_cb * " << CH << "LL + " << u * GPW << " + dx_gi;\n";
        // full chunks (all but at most one per launch) run the bodies
        // unguarded, in convergent code; the ragged chunk guards each ordinal
        // and sums over its group's lanes only (the guard is group-uniform)
        std::string tail = body;
        for (size_t at = 0; (at = tail.find("dx_grp_sum<", at)) != std::string::npos; at += 13)
          tail.replace(at, 11, "dx_grp_sum_m<");
        o << "      if (dx_cb < dx_nfull) {\n";
        for (int u = 0; u < U; ++u) o << "        const bool dx_ok" << u << " = true;\n";
        o << body << "      } else {\n";
        for (int u = 0; u < U; ++u) o << "        const bool dx_ok" << u << " = dx_o" << u << " < dx_hi;\n";
        o << tail << "      }\n";
        o << "      " << grpPrefetch("dx_cb + 4 * dx_tw");
        o << "      if (dx_cb + 2 * dx_tw < dx_nch) " << grpLoad(ab, "dx_cb + 2 * dx_tw");
        return o.str();
      };
      src << "  for (long long dx_ch = dx_w0; dx_ch < dx_nch; dx_ch += 2 * dx_tw) {\n";
      src << "    {\n" << chunk("a", "dx_ch") << "    }\n";
      src << "    if (dx_ch + dx_tw < dx_nch) {\n" << chunk("b", "dx_ch + dx_tw") << "    }\n";
      src << "  }\n";
      src << "  dx_pdl_trigger();\n";
      if (lateWait) src << "  dx_pdl_wait();\n";
      if (lateWait && coop)
        src << "  __shared__ unsigned long long dx_ep;\n  if (threadIdx.x == 0) dx_ep = dx_bar_epoch((const unsigned long long*)"
            << g.params[syncBuf] << ");\n";
    } else if (g.warpRow) {
      // one warp per ordinal (warp-uniform), the lanes split the reduction loop
      src << "  for (long long dx_base = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; dx_base < dx_n; dx_base += dx_stride >> 5) {\n";
      src << "    const long long dx_s = dx_base;\n";
    } else {
      src << "  for (long long dx_base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); dx_base < dx_n; dx_base += dx_stride) {\n";
      src << "    const long long dx_s = dx_base + dx_lane;\n";
    }
    if (g.grp == 0) {
    for (int u = 0; u < U; ++u)
      src << "    const long long dx_o" << u << " = dx_lo + dx_s * " << U << " + " << u << ";\n";
    for (auto& rs : g.rowSites) {
      src << "    dx_f rowv" << rs.id << "[" << rs.D << "];\n";
      src << "#pragma unroll\n    for (int t = 0; t < " << rs.D << "; ++t) rowv" << rs.id << "[t] = 0;\n";
      src << "    int rowk" << rs.id << " = -1;\n";
    }
    if (U > 1) {
      // one 16-byte load per stream buffer for the thread's U ordinals
      for (int b : streams) {
        auto it = g.params.find(b);
        if (it == g.params.end()) continue;
        std::string ct = ctype(plan.bufs[b].kind);
        std::string vt = plan.bufs[b].kind == SK::F ? "float4" : "int4";
        std::string P = "pf" + std::to_string(b) + "_";
        for (int g4 = 0; g4 < U; g4 += 4) {
          const std::string a0 = std::to_string(g4), a1 = std::to_string(g4 + 1), a2 = std::to_string(g4 + 2),
                            a3 = std::to_string(g4 + 3);
          src << "    " << ct << " " << P << a0 << " = 0, " << P << a1 << " = 0, " << P << a2 << " = 0, " << P << a3
              << " = 0;\n";
          src << "    if ((dx_lo & 3) == 0 && dx_o" << a3 << " < dx_hi) { const " << vt << " w = *(const " << vt << "*)("
              << it->second << " + dx_o" << a0 << "); " << P << a0 << " = w.x; " << P << a1 << " = w.y; " << P << a2
              << " = w.z; " << P << a3 << " = w.w; }\n";
          src << "    else {";
          for (int u = g4; u < g4 + 4; ++u)
            src << " if (dx_o" << u << " < dx_hi) " << P << u << " = " << it->second << "[dx_o" << u << "];";
          src << " }\n";
        }
      }
    }
    src << "    if (dx_s < dx_n) {\n" << body << "    }\n";
    for (auto& rs : g.rowSites) {
      const CellUse& cu = g.cells[rs.cu];
      if (cu.strat == CellUse::TileRow) {
        std::string I = std::to_string(rs.cu);
        long long Kr = cu.width / cu.rowD;
        int nacc = (int)((cu.width + g.threads - 1) / g.threads);
        if (cu.vec4) {
          // The output rows may overwrite the TMA stage holding this tile's
          // input rows when the shapes and swizzles agree: thread t only ever
          // reads its own staged row before writing its own output row.
          std::string etp = "et" + I;
          if (cu.aliasStage >= 0)
            etp = "(sb" + std::to_string(cu.aliasStage) + " + dx_sh" + std::to_string(cu.aliasStage) + ")";
          src << "    dx_tile_store4<" << rs.D << ">(" << etp << ", threadIdx.x, rowv" << rs.id << ");\n";
          if (cu.warpTab) {
            src << "    dx_warp_tab<" << rs.D << ", " << Kr << ">(" << etp << ", rowk" << rs.id << ", wtab" << I
                << " + dx_warp * " << (Kr + 1) * 32 << ");\n";
            src << "    __syncthreads();  // every warp is done with this TMA stage\n";
            continue;
          }
          src << "    dx_tile_rows4<" << rs.D << ", " << Kr << ", " << g.threads << ">(" << etp << ", rowk" << rs.id
              << ", wc" << I << ", st" << I << ", pm" << I << ", acc" << I << ");\n";
          continue;
        }
        src << "#pragma unroll\n    for (int t = 0; t < " << rs.D << "; ++t) et" << I << "[threadIdx.x * " << rs.D + 1
            << " + t] = rowv" << rs.id << "[t];\n";
        src << "    dx_tile_rows<dx_f, " << rs.D << ", " << Kr << ", " << g.threads << ", " << nacc << ">(et" << I
            << ", rowk" << rs.id << ", wc" << I << ", st" << I << ", pm" << I << ", acc" << I << ");\n";
        continue;
      }
      src << "    dx_row_flush<dx_f, " << rs.D << ">(rt" << rs.cu << " + dx_warp * " << cu.width
          << ", dx_stage, rowk" << rs.id << ", rowv" << rs.id << ");\n";
    }
    if (tileCell < 0 && g.tile && !g.staged.empty())
      src << "    __syncthreads();  // every thread is done with this TMA stage\n";
    src << "  }\n";
    }  // g.grp == 0
    if (opt.count)
      src << "  dx_count_flush((unsigned long long*)" << g.params[plan.countBuf] << ", dx_cops, dx_cacc, dx_ccell);\n";
    // last-block-done kernels collect the E-bounds flags of the launch in a
    // ticket word; the final block forwards them (and initializes the error
    // flag when this kernel is its first writer)
    const bool lbdErr = lbd && takeZero(plan.errFlagBuf);
    const bool coopErr = coop && takeZero(plan.errFlagBuf);
    if (!lbd && !coopErr) src << "  if (dx_bad) atomicOr(dx_err, 1);\n";
    // epilogue: block partials.  Register cells: warp sums into scratch
    // first; the block barrier they need is the one the next flush (or an
    // explicit one) executes anyway; warp 0 then adds the warp sums (the
    // dx_block_sum tree, one barrier instead of two).
    bool regPending = false;
    for (size_t i = 0; i < g.cells.size(); ++i)
      if (g.cells[i].strat == CellUse::Reg) {
        const std::string I = std::to_string(i);
        src << "  __shared__ dx_f scr" << I << "[32];\n  { const dx_f s = dx_warp_sum(rp" << I
            << "); if (dx_lane == 0) scr" << I << "[dx_warp] = s; }\n";
        regPending = true;
      }
    auto regFinish = [&]() {
      if (!regPending) return;
      for (size_t i = 0; i < g.cells.size(); ++i)
        if (g.cells[i].strat == CellUse::Reg) {
          const std::string I = std::to_string(i);
          src << "  if (dx_warp == 0) { dx_f r = dx_lane < (int)((blockDim.x + 31) >> 5) ? scr" << I
              << "[dx_lane] : (dx_f)0; r = dx_warp_sum(r); if (dx_lane == 0) part" << I << "[blockIdx.x] = r; }\n";
        }
      regPending = false;
    };
    bool synced = false;  // a flush below began with a block barrier
    for (size_t i = 0; i < g.cells.size(); ++i) {
      CellUse& cu = g.cells[i];
      std::string I = std::to_string(i);
      if (cu.strat == CellUse::Smem || cu.strat == CellUse::Count || cu.strat == CellUse::Row ||
          (cu.strat == CellUse::TileRow && cu.warpTab))
        synced = true;
      switch (cu.strat) {
        case CellUse::Reg:
          break;
        case CellUse::Smem:
        case CellUse::Count:
          src << "  __syncthreads();\n  for (int t = threadIdx.x; t < " << cu.width << "; t += blockDim.x) part" << I
              << "[(long long)blockIdx.x * " << cu.width << " + t] = sm" << I << "[t];\n";
          break;
        case CellUse::TileRow: {
          int nacc = (int)((cu.width + g.threads - 1) / g.threads);
          if (cu.warpTab) {
            src << "  dx_warp_tab_flush<" << cu.rowD << ", " << cu.width / cu.rowD << ", " << g.threads / 32 << ">(wtab" << I
                << ", part" << I << " + (long long)blockIdx.x * " << cu.width << ");\n";
            break;
          }
          if (cu.vec4) {
            std::string scratch = cu.aliasStage >= 0 ? "sb" + std::to_string(cu.aliasStage) : "et" + I;
            src << "  dx_tile_rows4_flush<" << cu.rowD << ", " << cu.width / cu.rowD << ", " << g.threads << ">(" << scratch
                << ", acc" << I << ", part" << I << " + (long long)blockIdx.x * " << cu.width << ");\n";
            break;
          }
          src << "#pragma unroll\n  for (int t = 0; t < " << nacc << "; ++t) { const int e = threadIdx.x + t * "
              << g.threads << "; if (e < " << cu.width << ") part" << I << "[(long long)blockIdx.x * " << cu.width
              << " + e] = acc" << I << "[t]; }\n";
          break;
        }
        case CellUse::Row:
          src << "  __syncthreads();\n  for (int t = threadIdx.x; t < " << cu.width << "; t += blockDim.x) {\n"
              << "    dx_f s = 0;\n    for (int w = 0; w < " << warps << "; ++w) s += rt" << I << "[w * " << cu.width
              << " + t];\n    part" << I << "[(long long)blockIdx.x * " << cu.width << " + t] = s;\n  }\n";
          break;
        default: break;
      }
    }
    if (regPending && !synced) src << "  __syncthreads();\n";
    regFinish();
    if (coop) {
      if (coopErr) src << "  if (blockIdx.x == 0 && threadIdx.x == 0) *dx_err = 0;\n";
      src << "  dx_spread_barrier((unsigned long long*)" << g.params[syncBuf] << ", dx_ep);\n";
      if (coopErr) src << "  if (dx_bad) atomicOr(dx_err, 1);\n";
      long long foldBase = 0;
      for (size_t i = 0; i < g.cells.size(); ++i) {
        CellUse& cu = g.cells[i];
        if (cu.partialBuf < 0) continue;
        std::string ct = ctype(plan.bufs[cu.targetBuf].kind);
        bool counts = cu.strat == CellUse::Count;
        // a cell whose only pending step is its zero-fill is overwritten
        const bool store = takeZero(cu.targetBuf);
        // the cells' columns share one warp index space: every column is one
        // warp's fold, all in flight together
        src << "  dx_coop_fold_b<" << ct << ", " << (counts ? "unsigned" : "dx_f") << ">(part" << i << ", "
            << cu.width << "LL, (" << ct << ")" << litF(counts ? cu.constVal : 1.0, true) << ", " << cu.pname
            << ", " << (counts ? "true" : "false") << ", " << (store ? "true" : "false") << ", " << foldBase << "LL);\n";
        foldBase += (cu.width + 31) / 32;
      }
    }
    if (lbd) {
      const std::string T = g.params[tickBuf];
      src << "  {\n    const int dx_ng = (gridDim.x + DX_LBD_GB - 1) / DX_LBD_GB, dx_grp = blockIdx.x / DX_LBD_GB;\n"
          << "    const int dx_gsz = min(DX_LBD_GB, (int)gridDim.x - dx_grp * DX_LBD_GB);\n"
          << "    if (dx_bad) atomicOr(&" << T << "[DX_LBD_ERR], 1u);\n"
          << "    if (dx_lbd_arrive(" << T << ", dx_grp, (unsigned)dx_gsz)) {\n";
      for (size_t i = 0; i < g.cells.size(); ++i) {
        CellUse& cu = g.cells[i];
        if (cu.partialBuf < 0) continue;
        bool counts = cu.strat == CellUse::Count;
        src << "      dx_lbd_group<" << (counts ? "unsigned, long long" : "dx_f, double") << ">(part" << i << ", "
            << cu.width << "LL, " << g.params[gpartBuf[i]] << ", dx_grp, dx_grp * DX_LBD_GB, dx_gsz);\n";
      }
      src << "      if (threadIdx.x == 0) " << T << "[dx_grp] = 0u;\n"
          << "      if (dx_lbd_arrive(" << T << ", DX_LBD_TOP, (unsigned)dx_ng)) {\n";
      for (size_t i = 0; i < g.cells.size(); ++i) {
        CellUse& cu = g.cells[i];
        if (cu.partialBuf < 0) continue;
        std::string ct = ctype(plan.bufs[cu.targetBuf].kind);
        bool counts = cu.strat == CellUse::Count;
        // a cell whose only pending step is its zero-fill is overwritten
        const bool store = takeZero(cu.targetBuf);
        src << "        dx_lbd_final<" << (counts ? "long long" : "double") << ", " << ct << ">(" << g.params[gpartBuf[i]]
            << ", " << cu.width << "LL, dx_ng, (" << ct << ")" << litF(counts ? cu.constVal : 1.0, true) << ", "
            << cu.pname << ", " << (counts ? "true" : "false") << ", " << (store ? "true" : "false") << ");\n";
      }
      src << "        if (threadIdx.x == 0) {\n          " << T << "[DX_LBD_TOP] = 0u;\n"
          << "          const unsigned e = atomicExch(&" << T << "[DX_LBD_ERR], 0u);\n"
          << (lbdErr ? "          *dx_err = (int)e;\n" : "          if (e) atomicOr(dx_err, 1);\n")
          << "        }\n      }\n    }\n  }\n";
    }
    src << "}\n\n";
  }
  if (!empty) {
    plan.source += src.str();
    plan.numKernels++;
  }

  // Output buffers for sharded kernels are summed across ranks: zero first.
  if (g.sharded) {
    for (size_t l = 0; l < outBufs.size(); ++l) {
      Step z; z.k = Step::Zero; z.buf = outBufs[l]; z.off = outOffs[l];
      z.elems = elemTy ? leaves(serial ? elemTy : tTable(kb0.desc, elemTy))[l].count : 0;
      addStep(z);
    }
  }

  if (!empty) {
  Step ks;
  ks.k = Step::Kernel;
  ks.name = kname;
  ks.args = args;
  ks.total = total;
  ks.serial = serial;
  ks.sharded = g.sharded;
  ks.threads = serial ? 32 : g.threads;
  ks.smem = smem;
  ks.minGrid = U;
  ks.warpRow = g.warpRow;
  ks.grp = g.grp;
  ks.coop = coop;
  ks.note = note + (g.warpRow ? " (warp per ordinal)" : "");
  ks.rwKnown = true;
  for (auto& [b, pn] : g.params)
    if (!g.writtenBufs.count(b)) ks.readBufs.insert(b);
  for (auto& cu : g.cells) ks.readBufs.insert(cu.targetBuf);  // += reads the cell (or its delta)
  if (g.sharded && !kb0.dims.empty() && total > 0) {
    const long long n0 = size(kb0.dims[0]);
    ks.rowBlock = n0 > 0 ? total / n0 : 1;
    ks.rowsOf = n0;
    // every read of the buffer is inside the row of the kernel's own dim-0
    // ordinal (one row width): the rank reads only its own rows
    for (auto& [b, ws] : g.rowUse)
      if (!g.rowBad.count(b) && ws.size() == 1) ks.rowReads[b] = *ws.begin();
  }
  addStep(ks);
  int kstep = (int)plan.steps.size() - 1;
  for (auto& cu : g.cells)
    if (cu.partialBuf >= 0) plan.bufs[cu.partialBuf].partialKernel = kstep;
  for (int gb : gpartBuf)
    if (gb >= 0) plan.bufs[gb].partialKernel = kstep;

  // Finalize privatized partials into the cell (fixed block order).
  for (size_t i = 0; i < g.cells.size(); ++i) {
    CellUse& cu = g.cells[i];
    if (cu.partialBuf < 0 || fold) continue;
    Step f;
    f.k = Step::Finalize;
    f.buf = cu.targetBuf;
    f.buf2 = cu.partialBuf;
    f.elems = cu.width;
    f.kernelStep = kstep;
    f.fin = cu.strat == CellUse::Count ? Step::Count : Step::Seq;
    f.scale = cu.constVal;
    addStep(f);
  }
  if (g.sharded) {
    // every Accum delta of this kernel in one grouped all-gather, then the
    // rank-ordered fold into the cells
    if (!g.cells.empty()) {
      Step m;
      m.k = Step::Merge;
      long long mtotal = 0;
      for (auto& cu : g.cells) {
        Step::MergeItem mi{cu.targetBuf, cells[cu.cell].bufs[cu.leaf], cu.width};
        // Owner updates (the path starts with the kernel's own ordinal): each
        // rank's delta is zero outside its own rows
        const long long n0 = kb0.dims.empty() ? 0 : size(kb0.dims[0]);
        if (cu.strat == CellUse::Owner && cu.ownRows && n0 > 0 && cu.width % n0 == 0) {
          mi.rowN = n0;
          mi.rowW = cu.width / n0;
        }
        m.merge.push_back(mi);
        mtotal += cu.width;
      }
      m.buf = newBuf(BufDecl::Temp, SK::D, mtotal * plan.world);  // gathered deltas
      m.elems = mtotal;
      addStep(m);
    }
    for (size_t l = 0; l < outBufs.size(); ++l) {
      Step a; a.k = Step::Allreduce; a.buf = outBufs[l]; a.off = outOffs[l];
      a.elems = leaves(tTable(kb0.desc, elemTy))[l].count;
      // a map over the kernel's own ordinal: rank r holds rows of its shard
      bool fwd = true;  // reversed dims store row n-1-o
      for (auto& kb : parts) fwd = fwd && !kb.dimReversed.empty() && !kb.dimReversed[0];
      const long long n0 = kb0.dims.empty() ? 0 : size(kb0.dims[0]);
      if (fwd && outOffs[l] == 0 && n0 > 0 && a.elems % n0 == 0) {
        a.rowShardN = n0;
        a.rowShardW = a.elems / n0;
      }
      addStep(a);
    }
  }
  }  // !empty
  if (!elemTy) return hUnit();
  DTy rt = serial ? elemTy : tTable(kb0.desc, elemTy);
  if (outBufs.empty()) {
    if (serial) return hUnit();
    auto h = std::make_shared<HVal>();
    h->k = HVal::Buf;
    h->ty = rt;
    return h;
  }
  return hvFromBufs(rt, outBufs, outOffs);
}

HV Lowering::loopKernel(const HEnvP& env, const EFor& f, const DescPtr& d, bool serial, Span sp) {
  if (serial) {
    // whole loop inside one device thread (State forbids chunking, eval.cpp:298-299)
    ExprPtr loop = mkExpr(f, sp);
    KernelBody kb;
    kb.body = [this, loop](KGen& g, const KScope& s) { return kexpr(g, s, loop, nullptr); };
    kb.env = env;
    kb.note = "serial loop " + printName(f.binder);
    return requestKernel(kb, true, nullptr, nullptr);
  }
  if (HV gm = contractNest(env, f, d)) return gm;
  if (HV fl = flattenEffectNest(env, f, d)) return fl;
  KernelBody kb;
  kb.desc = d;
  kb.dims = {d};
  kb.dimBinders = {f.binder};
  kb.dimReversed = {onlyReversed(f.binder, f.body)};
  ExprPtr body = f.body;
  kb.body = [this, body](KGen& g, const KScope& s) { return kexpr(g, s, body, nullptr); };
  kb.env = env;
  kb.note = "parallel for " + printName(f.binder);
  return requestKernel(kb, false, nullptr, nullptr);
}

// Effectful nests `for i. <pure lets>; (let t = for j. B; t)` whose outer loop
// alone cannot fill the GPU (the MLP's dY rows: 8192 x 1024) run over the
// flattened (i, j) space, j fastest: the pure lets are recomputed per element
// (they are per-row scalars), and per-row writes r!i!j become coalesced
// owner writes instead of one 4 KB-strided row per thread.
static bool hasLoop(const ExprPtr& e) {
  bool found = false;
  std::function<void(const ExprPtr&)> scan = [&](const ExprPtr& x) {
    if (found) return;
    std::visit(
        [&](const auto& n) {
          using T = std::decay_t<decltype(n)>;
          if constexpr (std::is_same_v<T, EFor>) found = true;
          else if constexpr (std::is_same_v<T, ELet>) { scan(n.bound); scan(n.body); }
          else if constexpr (std::is_same_v<T, ECase>) { scan(n.leftBody); scan(n.rightBody); }
          else if constexpr (std::is_same_v<T, ERunState> || std::is_same_v<T, ERunAccum>) scan(n.action.body);
        },
        x->node);
  };
  scan(e);
  return found;
}

// A runAccum whose action is loop-free lets followed by the broadcast loop
// `for j. r!j' += v` (what accumToMapK turns into a lazy map): cheap to
// recompute per element once lowered.
static bool mapLikeRunAccum(const ERunAccum& r) {
  ExprPtr cur = r.action.body;
  while (const auto* l = as<ELet>(cur)) {
    if (const auto* f = as<EFor>(l->bound)) {
      const auto* ret = as<ERet>(l->body);
      const auto* rv = ret ? as<VVar>(ret->value) : nullptr;
      if (!rv || rv->name != l->binder || hasLoop(f->body)) return false;
      int accs = 0;
      for (ExprPtr b = f->body; const auto* bl = as<ELet>(b); b = bl->body) accs += as<EAccum>(bl->bound) != nullptr;
      return accs == 1;
    }
    if (hasLoop(l->bound)) return false;
    cur = l->body;
  }
  return false;
}

HV Lowering::flattenEffectNest(const HEnvP& env, const EFor& f, const DescPtr& d) {
  if (opt.noFusion) return nullptr;
  const long long n = size(d);
  if (n >= 148LL * 1024) return nullptr;  // the outer loop fills the GPU already
  std::vector<const ELet*> pre;
  ExprPtr cur = f.body;
  const EFor* inner = nullptr;
  const ELet* innerLet = nullptr;
  while (const auto* l = as<ELet>(cur)) {
    if (const auto* ff = as<EFor>(l->bound)) {
      const auto* ret = as<ERet>(l->body);
      const auto* rv = ret ? as<VVar>(ret->value) : nullptr;
      if (!rv || rv->name != l->binder) return nullptr;
      inner = ff;
      innerLet = l;
      break;
    }
    if (!pureBody(l->bound) || as<ERunState>(l->bound) || as<EFor>(l->bound)) return nullptr;
    // recomputed per element: only loop-free lets, or runAccums that are a
    // loop-free chain ending in the accum-to-map broadcast
    if (const auto* ra = as<ERunAccum>(l->bound)) {
      if (!mapLikeRunAccum(*ra)) return nullptr;
    } else if (hasLoop(l->bound)) {
      return nullptr;
    }
    pre.push_back(l);
    cur = l->body;
  }
  if (!inner || pureBody(inner->body)) return nullptr;
  DescPtr d2;
  try {
    d2 = resolveDesc(inner->annot, hostLook(env));
  } catch (const DexError&) {
    return nullptr;
  }
  if (size(d2) < 32) return nullptr;
  (void)innerLet;
  ExprPtr body = inner->body;
  for (size_t i = pre.size(); i-- > 0;) body = eLet(pre[i]->binder, pre[i]->annot, pre[i]->bound, body);
  KernelBody kb;
  kb.desc = descPair(d, d2);
  kb.dims = {d, d2};
  kb.dimBinders = {f.binder, inner->binder};
  // loops indexed only through `reverse` (transposed nests) run reversed, so
  // element (i, j) of the body is ordinal (i, j): forward rows, and under
  // sharding the rank's own rows
  kb.dimReversed = {onlyReversed(f.binder, body), onlyReversed(inner->binder, body)};
  kb.body = [this, body](KGen& g, const KScope& s) { return kexpr(g, s, body, nullptr); };
  kb.env = env;
  kb.note = "parallel for " + printName(f.binder) + " x " + printName(inner->binder) + " (flattened)";
  HV r = requestKernel(kb, false, nullptr, nullptr);
  // an effect-only nest: (Fin n) => (Fin m) => Unit
  auto h = std::make_shared<HVal>();
  h->k = HVal::Buf;
  h->ty = tTable(d, tTable(d2, tUnit()));
  (void)r;
  return h;
}

HV Lowering::loopKernelLazy(const HV& lz, const std::vector<int>* intoBufs,
                            const std::vector<long long>* intoOffs) {
  // Flatten perfect nests `for i. (let t = for k. B; t)` into one iteration
  // space (row-major ordinal == nested table layout).
  KernelBody kb;
  std::vector<DescPtr> dims = {lz->desc};
  std::vector<Name> binders = {lz->binder};
  ExprPtr body = lz->body;
  while (true) {
    const auto* l = as<ELet>(body);
    if (!l) break;
    const auto* inner = as<EFor>(l->bound);
    const auto* ret = as<ERet>(l->body);
    if (!inner || !ret) break;
    const auto* rv = as<VVar>(ret->value);
    if (!rv || rv->name != l->binder) break;
    if (!pureBody(inner->body)) break;
    DescPtr d2;
    try {
      d2 = resolveDesc(inner->annot, hostLook(lz->env));
    } catch (const DexError&) {
      break;
    }
    dims.push_back(d2);
    binders.push_back(inner->binder);
    body = inner->body;
  }
  if (HV gm = contractMaterialize(lz, dims, binders, body, intoBufs, intoOffs)) return gm;
  DescPtr all = dims[0];
  for (size_t i = 1; i < dims.size(); ++i) all = descPair(all, dims[i]);
  // a flattened kernel iterates the pair set; its output layout is the
  // nested table (same row-major ordinal)
  kb.desc = all;
  kb.dims = dims;
  kb.dimBinders = binders;
  for (size_t i = 0; i < dims.size(); ++i) kb.dimReversed.push_back(false);
  if (dims.size() == 1) kb.dimReversed[0] = onlyReversed(binders[0], body);
  kb.body = [this, body](KGen& g, const KScope& s) { return kexpr(g, s, body, nullptr); };
  kb.env = lz->env;
  kb.note = "materialize " + printName(lz->binder);
  HV r = requestKernel(kb, false, intoBufs, intoOffs);
  // re-type as the nested table
  if (dims.size() > 1 && r->k == HVal::Buf && r->ty->k == DType::Table) {
    DTy et = r->ty->a;
    for (size_t i = dims.size(); i-- > 0;) et = tTable(dims[i], et);
    auto h = std::make_shared<HVal>(*r);
    h->ty = et;
    return h;
  }
  return r;
}

// ---------------------------------------------------------------------------
// Split materialization of tuple-valued lazy tables.
//
// LinFor (autodiff.cpp:230-255) turns every forward loop into a tape whose
// elements pair the primal with its partials, e.g. per (bb, h2) of the MLP
// `(for ii. (x, (w1, x*w1)), (z, z*z))`.  Materializing such a table stores
// the cheap inner triples (B*H*I of them: 100 GB at the MLP config) only to
// read back values recomputable from the inputs.  Instead the element tuple
// is split: components cheap to recompute stay a lazy projection (inlined at
// each use), the others are materialized as their own table (where the
// contraction lowering can pick them up).  The result is a Zip: the table of
// pairs held as a pair of tables over the same index levels.
ValuePtr Lowering::typeValue(const DTy& t) {
  if (!t) return nullptr;
  switch (t->k) {
    case DType::Float: return vBase(BaseKind::Float);
    case DType::Int: return vBase(BaseKind::Int);
    case DType::Unit: return vBase(BaseKind::Unit);
    case DType::Pair: {
      ValuePtr a = typeValue(t->a), b = typeValue(t->b);
      return a && b ? vPairType(a, b) : nullptr;
    }
    case DType::Table: {
      ValuePtr e = typeValue(t->a);
      if (!e || t->desc->kind != IndexSetDesc::Kind::Fin) return nullptr;
      return vArray(vFin(vInt(size(t->desc))), e);
    }
    default: return nullptr;
  }
}

HV Lowering::splitMaterialize(const HV& lz) {
  if (lz->k != HVal::Lazy) return nullptr;
  if (lz->st->split) return lz->st->split;
  if (opt.noFusion) return nullptr;
  // the perfect nest (as loopKernelLazy flattens it)
  std::vector<const ELet*> wraps;
  std::vector<const EFor*> fors;
  std::vector<DescPtr> descs = {lz->desc};
  ExprPtr body = lz->body;
  while (true) {
    const auto* l = as<ELet>(body);
    if (!l) break;
    const auto* inner = as<EFor>(l->bound);
    const auto* ret = as<ERet>(l->body);
    if (!inner || !ret) break;
    const auto* rv = as<VVar>(ret->value);
    if (!rv || rv->name != l->binder || !pureBody(inner->body)) break;
    DescPtr d2;
    try {
      d2 = resolveDesc(inner->annot, hostLook(lz->env));
    } catch (const DexError&) {
      break;
    }
    wraps.push_back(l);
    fors.push_back(inner);
    descs.push_back(d2);
    body = inner->body;
  }
  std::vector<const ELet*> chain;
  ExprPtr cur = body;
  while (const auto* l = as<ELet>(cur)) {
    chain.push_back(l);
    cur = l->body;
  }
  const auto* rt = as<ERet>(cur);
  if (!rt || !as<VPair>(rt->value)) return nullptr;
  DTy et = lz->ty;
  for (size_t i = 0; i < descs.size(); ++i) {
    if (!et || et->k != DType::Table) return nullptr;
    et = et->a;
  }
  if (!et || et->k != DType::Pair) return nullptr;
  std::map<Name, const ELet*> defs;
  for (const ELet* l : chain) defs[l->binder] = l;
  std::map<Name, bool> memo;
  std::function<bool(const Name&)> cheapName = [&](const Name& n) -> bool {
    auto d = defs.find(n);
    if (d == defs.end()) return true;  // binder or outer value
    auto m = memo.find(n);
    if (m != memo.end()) return m->second;
    memo[n] = false;
    const ExprPtr& b = d->second->bound;
    bool ok;
    if (const auto* f = as<EFor>(b)) ok = pureBody(f->body) && cheapBody(f->body);
    else ok = !as<ERunAccum>(b) && !as<ERunState>(b) && !as<ECase>(b) && !as<EApp>(b);
    if (ok)
      for (const Name& fv : freeVars(b))
        if (!cheapName(fv)) ok = false;
    memo[n] = ok;
    return ok;
  };
  auto cheapVal = [&](const ValuePtr& v) {
    for (const Name& fv : freeVars(v))
      if (!cheapName(fv)) return false;
    return true;
  };
  std::function<bool(const ValuePtr&)> anyCheap = [&](const ValuePtr& v) -> bool {
    if (const auto* p = as<VPair>(v)) return anyCheap(p->l) || anyCheap(p->r);
    return cheapVal(v);
  };
  std::function<bool(const ValuePtr&)> allCheap = [&](const ValuePtr& v) -> bool {
    if (const auto* p = as<VPair>(v)) return allCheap(p->l) && allCheap(p->r);
    return cheapVal(v);
  };
  // Table-valued components whose own elements are mixed tuples (a tape of
  // tapes, e.g. matmul `for i. (for k. (for j. (x, (y, x*y)), sum_j), sum_k)`)
  // are split recursively first; the other projections then read the split
  // (bound to a fresh name) instead of recomputing it.
  std::map<Name, HV> shared;
  std::map<Name, Name> sharedName;
  const int depth = (int)descs.size();
  std::function<bool(const ValuePtr&)> tupleTable = [&](const ValuePtr& v) -> bool {
    const auto* x = as<VVar>(v);
    if (!x || !defs.count(x->name)) return false;
    const auto* f = as<EFor>(defs[x->name]->bound);
    if (!f || !pureBody(f->body) || cheapName(x->name)) return false;
    ExprPtr c = f->body;
    while (const auto* l = as<ELet>(c)) c = l->body;
    const auto* r = as<ERet>(c);
    return r && as<VPair>(r->value);
  };
  std::function<bool(const ValuePtr&)> hasTupleTable = [&](const ValuePtr& v) -> bool {
    if (const auto* p = as<VPair>(v)) return hasTupleTable(p->l) || hasTupleTable(p->r);
    return tupleTable(v);
  };
  if ((!anyCheap(rt->value) && !hasTupleTable(rt->value)) || allCheap(rt->value)) return nullptr;
  HEnvP penv = lz->env;
  auto projection = [&](const ValuePtr& v, const DTy& vty, bool mat) -> HV {
    ExprPtr inner = eRet(v);
    NameSet need = freeVars(v);
    for (auto it = chain.rbegin(); it != chain.rend(); ++it) {
      const ELet* l = *it;
      if (!need.count(l->binder)) continue;
      auto sh = sharedName.find(l->binder);
      if (sh != sharedName.end()) {
        // let t = Z.b0.b1...  (the recursive split of this component)
        std::vector<Name> bs = {lz->binder};
        for (auto* f : fors) bs.push_back(f->binder);
        std::vector<Name> tmp;
        for (size_t i = 0; i < bs.size(); ++i) tmp.push_back(NameSupply::fresh("zip"));
        inner = eLet(l->binder, l->annot, eRet(vVar(tmp.back())), inner);
        for (size_t i = bs.size(); i-- > 0;)
          inner = eLet(tmp[i], nullptr, eIndex(vVar(i == 0 ? sh->second : tmp[i - 1]), vVar(bs[i])), inner);
        continue;
      }
      inner = eLet(l->binder, l->annot, l->bound, inner);
      for (const Name& n : freeVars(l->bound)) need.insert(n);
    }
    DTy ty = vty;
    for (size_t i = fors.size(); i-- > 0;) {
      ty = tTable(descs[i + 1], ty);
      inner = eLet(wraps[i]->binder, typeValue(ty), eFor(fors[i]->binder, fors[i]->annot, inner),
                   eRet(vVar(wraps[i]->binder)));
    }
    auto h = std::make_shared<HVal>(*lz);
    h->body = inner;
    h->ty = tTable(lz->desc, ty);
    h->env = penv;
    h->cheap = cheapBody(inner);
    h->st = std::make_shared<LazyState>();
    return mat ? materialize(h) : HV(h);
  };
  // recursive splits of tuple-valued table components (before their readers)
  std::function<void(const ValuePtr&, const DTy&)> pre = [&](const ValuePtr& v, const DTy& vty) {
    if (const auto* p = as<VPair>(v)) {
      if (vty->k != DType::Pair) return;
      pre(p->l, vty->a);
      pre(p->r, vty->b);
      return;
    }
    if (!tupleTable(v)) return;
    const Name& t = as<VVar>(v)->name;
    if (shared.count(t)) return;
    HV P = projection(v, vty, false);
    HV S = splitMaterialize(P);
    if (!S) S = materialize(P);
    shared[t] = S;
    Name z = NameSupply::fresh("zip");
    sharedName[t] = z;
    penv = hbind(penv, z, S);
  };
  pre(rt->value, et);
  std::function<HV(const ValuePtr&, const DTy&)> split = [&](const ValuePtr& v, const DTy& vty) -> HV {
    if (const auto* x = as<VVar>(v))
      if (shared.count(x->name)) return shared[x->name];
    if (allCheap(v)) return projection(v, vty, false);
    const auto* p = as<VPair>(v);
    if (p && (anyCheap(v) || hasTupleTable(v)) && vty->k == DType::Pair) {
      HV a = split(p->l, vty->a), b = split(p->r, vty->b);
      auto z = std::make_shared<HVal>();
      z->k = HVal::Zip;
      z->zipDepth = depth;
      z->a = a;
      z->b = b;
      z->ty = zipTy(a->ty, b->ty, depth);
      return z;
    }
    return projection(v, vty, true);
  };
  HV r = split(rt->value, et);
  lz->st->split = r;
  return r;
}

#include "contract.inc"

HV Lowering::serialKernel(const HEnvP& env, const ExprPtr& e, const ValuePtr& annot) {
  KernelBody kb;
  kb.body = [this, e](KGen& g, const KScope& s) { return kexpr(g, s, e, nullptr); };
  kb.env = env;
  kb.note = "serial statement";
  (void)annot;
  return requestKernel(kb, true, nullptr, nullptr);
}

// ---------------------------------------------------------------------------

std::string Plan::summary() const {
  std::ostringstream o;
  long long bytes = 0, big = 0;  // device buffers (partials are sized by the grid at prepare: excluded)
  int bigB = -1;
  for (size_t i = 0; i < bufs.size(); ++i) {
    const BufDecl& b = bufs[i];
    if (b.role == BufDecl::Partial) continue;
    const long long by = std::max(1LL, b.elems) * (long long)storageBytesOf(b.kind, f64);
    bytes += by;
    if (by > big) big = by, bigB = (int)i;
  }
  char mb[32];
  snprintf(mb, sizeof mb, "%.1f", bytes / 1048576.0);
  o << "plan: " << steps.size() << " steps, " << numKernels << " kernels, " << bufs.size()
    << " buffers (" << mb << " MiB; largest b" << bigB << " " << big / 1048576 << " MiB), " << (f64 ? "f64" : "f32")
    << ", world " << world << "\n";
  for (size_t i = 0; i < steps.size(); ++i) {
    const Step& s = steps[i];
    o << "  [" << i << "] ";
    switch (s.k) {
      case Step::Zero: o << "zero b" << s.buf << " (" << s.elems << ")"; break;
      case Step::Upload: o << "upload b" << s.buf << " <- const b" << s.buf2 << " (" << s.elems << ")"; break;
      case Step::Kernel:
        o << "kernel " << s.name << (s.serial ? " serial" : "") << (s.coop ? " coop" : "") << " n=" << s.total
          << " smem=" << s.smem << "  // " << s.note;
        if (world > 1 && s.rwKnown) {  // sharded dataflow: what the kernel reads, own rows marked
          o << "  [reads";
          for (int b : s.readBufs) {
            o << " b" << b;
            auto it = s.rowReads.find(b);
            if (it != s.rowReads.end()) o << "(rows of " << s.rowsOf << " x" << it->second << ")";
          }
          o << "]";
        }
        break;
      case Step::Finalize:
        o << "finalize b" << s.buf << " <- partials b" << s.buf2 << " w=" << s.elems
          << (s.fin == Step::Count ? " count" : s.fin == Step::Tree ? " tree" : " seq");
        break;
      case Step::Allreduce: o << "allreduce b" << s.buf << " (" << s.elems << ")"; break;
      case Step::Merge:
        o << "merge " << s.merge.size() << " Accum deltas (" << s.elems
          << " values): one grouped all-gather, rank-ordered fold";
        break;
      case Step::AddBuf: o << "add b" << s.buf << " += b" << s.buf2; break;
      case Step::CopyBuf: o << "copy b" << s.buf << "+" << s.off << " <- b" << s.buf2 << "+" << s.off2 << " (" << s.elems << ")"; break;
      case Step::Convert: o << "convert b" << s.buf << "+" << s.off << " <- b" << s.buf2 << "+" << s.off2 << " (" << s.elems << ")"; break;
    }
    o << "\n";
  }
  return o.str();
}

// Data-parallel dataflow for sharded plans (world > 1).  A sharded kernel
// over N ordinals leaves rank r with the rows of its chunk of N: the rows of
// a map it produced (zero-filled elsewhere) and of an Accum cell it updated
// only at its own ordinal (Owner).  The plan summed such buffers across ranks
// right after the producer (an Allreduce, or the rank-ordered Merge of the
// cell deltas).  That collective is dropped when every later reader of the
// buffer (until it is overwritten) is a sharded kernel over the same N that
// reads it only at its own ordinal's row of the same width, and the buffer
// is not a program output: the rows the readers touch are exactly the local
// ones.  A dropped Merge item becomes a local add of the rank's own delta.
// This is what keeps batch-sharded networks (configs[4]) from exchanging
// their activations: only the parameter cotangents are merged.
static void dropLocalCollectives(Plan& plan) {
  if (plan.world <= 1) return;
  std::set<int> outputs;
  for (auto& o : plan.outputs)
    if (o.buf >= 0) outputs.insert(o.buf);
  auto reads = [&](const Step& st, int b) {
    switch (st.k) {
      case Step::Zero: return false;
      case Step::Kernel:
        if (st.rwKnown) return st.readBufs.count(b) > 0;
        for (auto& a : st.args)
          if ((a.k == KArg::Buf || a.k == KArg::TMap) && a.buf == b) return true;
        return false;
      case Step::Merge:
        for (auto& mi : st.merge)
          if (mi.delta == b || mi.cell == b) return true;
        return st.buf == b;
      default: return st.buf == b || st.buf2 == b;
    }
  };
  auto localOnly = [&](size_t from, int b, long long N, long long W) {
    if (outputs.count(b) || N <= 0 || W <= 0) return false;
    for (size_t j = from; j < plan.steps.size(); ++j) {
      const Step& st = plan.steps[j];
      if (st.dead) continue;
      if (st.k == Step::Zero && st.buf == b && st.off == 0) return true;  // overwritten: no later reader
      if (!reads(st, b)) continue;
      if (st.k != Step::Kernel || !st.rwKnown || !(st.sharded || st.rowsShifted) || st.rowsOf != N) return false;
      auto it = st.rowReads.find(b);
      if (it == st.rowReads.end() || it->second != W) return false;
    }
    return true;
  };
  std::vector<Step> out;
  for (size_t i = 0; i < plan.steps.size(); ++i) {
    Step st = plan.steps[i];
    if (st.k == Step::Allreduce && localOnly(i + 1, st.buf, st.rowShardN, st.rowShardW)) continue;
    if (st.k == Step::Merge) {
      std::vector<Step::MergeItem> keep;
      std::vector<Step> adds;
      for (auto& mi : st.merge) {
        if (localOnly(i + 1, mi.cell, mi.rowN, mi.rowW)) {
          Step a;
          a.k = Step::AddBuf;
          a.buf = mi.cell;
          a.buf2 = mi.delta;
          a.elems = mi.elems;
          adds.push_back(a);
        } else {
          keep.push_back(mi);
        }
      }
      if (!keep.empty()) {
        long long tot = 0;
        for (auto& mi : keep) tot += mi.elems;
        st.merge = keep;
        st.elems = tot;
        out.push_back(st);
      }
      for (auto& a : adds) out.push_back(a);
      continue;
    }
    out.push_back(st);
  }
  // kernel step indices referenced by partial buffers / finalize steps moved
  std::vector<int> remap(plan.steps.size(), -1);
  // recompute the kernel indices: kernels keep their relative order and are
  // never dropped, so the k-th kernel step maps to the k-th kernel step
  std::vector<int> oldK, newK;
  for (size_t i = 0; i < plan.steps.size(); ++i)
    if (plan.steps[i].k == Step::Kernel) oldK.push_back((int)i);
  for (size_t i = 0; i < out.size(); ++i)
    if (out[i].k == Step::Kernel) newK.push_back((int)i);
  for (size_t t = 0; t < oldK.size() && t < newK.size(); ++t) remap[oldK[t]] = newK[t];
  for (auto& st : out)
    if (st.kernelStep >= 0) st.kernelStep = remap[st.kernelStep];
  for (auto& b : plan.bufs)
    if (b.partialKernel >= 0) b.partialKernel = remap[b.partialKernel];
  plan.steps = out;
}

// Sharded plans: each Merge (grouped all-gather + rank-ordered fold of Accum
// deltas) moves down to just before the first later step that touches one of
// its cells or deltas; merges that meet are fused, so a plan whose cells are
// read only at the end (a network's parameter cotangents, the loss) does one
// collective.
static void fuseMerges(Plan& plan) {
  if (plan.world <= 1) return;
  auto touches = [&](const Step& st, const std::set<int>& bufs) {
    auto hit = [&](int b) { return b >= 0 && bufs.count(b) > 0; };
    if (hit(st.buf) || hit(st.buf2)) return true;
    for (auto& a : st.args)
      if ((a.k == KArg::Buf || a.k == KArg::TMap) && hit(a.buf)) return true;
    for (auto& mi : st.merge)
      if (hit(mi.delta) || hit(mi.cell)) return true;
    return false;
  };
  std::vector<Step> out;
  std::vector<Step> pending;
  std::set<int> pbufs;
  auto flush = [&]() {
    if (pending.empty()) return;
    Step m = pending[0];
    for (size_t i = 1; i < pending.size(); ++i)
      for (auto& mi : pending[i].merge) m.merge.push_back(mi);
    long long tot = 0;
    for (auto& mi : m.merge) tot += mi.elems;
    m.elems = tot;
    if (pending.size() > 1) {  // one gather buffer for all
      BufDecl d = plan.bufs[m.buf];
      d.elems = tot * plan.world;
      plan.bufs.push_back(d);
      m.buf = (int)plan.bufs.size() - 1;
    }
    out.push_back(m);
    pending.clear();
    pbufs.clear();
  };
  for (auto& st : plan.steps) {
    if (st.k == Step::Merge && !st.dead) {
      pending.push_back(st);
      for (auto& mi : st.merge) { pbufs.insert(mi.delta); pbufs.insert(mi.cell); }
      continue;
    }
    if (!pending.empty() && touches(st, pbufs)) flush();
    out.push_back(st);
  }
  flush();
  // kernel indices keep their relative order (kernels never move past each other)
  std::vector<int> oldK, newK;
  for (size_t i = 0; i < plan.steps.size(); ++i)
    if (plan.steps[i].k == Step::Kernel) oldK.push_back((int)i);
  for (size_t i = 0; i < out.size(); ++i)
    if (out[i].k == Step::Kernel) newK.push_back((int)i);
  std::vector<int> remap(plan.steps.size(), -1);
  for (size_t t = 0; t < oldK.size() && t < newK.size(); ++t) remap[oldK[t]] = newK[t];
  for (auto& st : out)
    if (st.kernelStep >= 0) st.kernelStep = remap[st.kernelStep];
  for (auto& b : plan.bufs)
    if (b.partialKernel >= 0) b.partialKernel = remap[b.partialKernel];
  plan.steps = out;
}

Plan lowerProgram(const ExprPtr& e, const std::vector<std::pair<Name, ValuePtr>>& inputs,
                  const LowerOptions& opts) {
  Lowering L(opts);
  L.plan.errFlagBuf = L.newBuf(BufDecl::Flag, SK::X, 1);
  {
    Step z; z.k = Step::Zero; z.buf = L.plan.errFlagBuf; z.elems = 1; L.plan.steps.push_back(z);
  }
  if (opts.count) {  // [ops, accum updates, cells] of one run
    L.plan.countBuf = L.newBuf(BufDecl::Flag, SK::I, 3);
    Step z; z.k = Step::Zero; z.buf = L.plan.countBuf; z.elems = 3; L.plan.steps.push_back(z);
  }
  HEnvP env;
  for (size_t i = 0; i < inputs.size(); ++i) {
    DTy t = L.resolveType(inputs[i].second, L.hostLook(env));
    std::vector<LeafInfo> lv = leaves(t);
    std::vector<int> bufs;
    std::vector<long long> offs;
    std::vector<InLeaf> in;
    for (size_t l = 0; l < lv.size(); ++l) {
      int b = L.newBuf(BufDecl::Input, lv[l].kind, lv[l].count);
      L.plan.bufs[b].input = (int)i;
      L.plan.bufs[b].leaf = (int)l;
      bufs.push_back(b);
      offs.push_back(0);
      in.push_back({lv[l].kind, lv[l].count, lv[l].desc, b});
    }
    L.plan.inputs.push_back(in);
    L.plan.inputTypes.push_back(t);
    L.plan.inputNames.push_back(inputs[i].first);
    env = hbind(env, inputs[i].first, L.hvFromBufs(t, bufs, offs));
  }
  HV res = L.hexpr(env, e);
  // Outputs: materialize lazies, flatten.
  std::function<void(const HV&)> out = [&](const HV& v) {
    switch (v->k) {
      case HVal::Unit: return;
      case HVal::Pair: out(v->a); out(v->b); return;
      case HVal::Const: {
        OutLeaf o;
        o.kind = v->ty->k == DType::Float ? SK::F : (v->ty->k == DType::Int ? SK::I : SK::X);
        o.count = 1;
        o.desc = v->ty->k == DType::Idx ? v->ty->desc : nullptr;
        o.host = true;
        if (o.kind == SK::F) o.hostF = {v->f};
        else o.hostI = {v->i};
        L.plan.outputs.push_back(o);
        return;
      }
      case HVal::Buf: {
        std::vector<LeafInfo> lv = leaves(v->ty);
        for (size_t l = 0; l < lv.size(); ++l) {
          OutLeaf o;
          o.kind = L.plan.bufs[v->bufs[l]].kind;
          o.count = lv[l].count;
          o.desc = lv[l].desc;
          o.buf = v->bufs[l];
          o.off = v->offs[l];
          L.plan.outputs.push_back(o);
        }
        return;
      }
      case HVal::Lazy: out(L.materialize(v)); return;
      case HVal::Zip: out(L.materialize(v->a)); out(L.materialize(v->b)); return;
      case HVal::Ref: notLowerable("reference escaping the program");
    }
  };
  std::function<HV(const HV&)> force = [&](const HV& v) -> HV {
    if (v->k == HVal::Lazy) return L.materialize(v);
    if (v->k == HVal::Pair) return hPair(force(v->a), force(v->b));
    return v;
  };
  res = force(res);
  L.flushPending();
  L.plan.outputType = res->ty;
  out(res);
  dropLocalCollectives(L.plan);
  fuseMerges(L.plan);
  // Dead buffers (e.g. cells whose value stayed lazy and was fused away):
  // drop their zero-fills and never allocate them.
  std::vector<bool> live(L.plan.bufs.size(), false);
  live[L.plan.errFlagBuf] = true;
  for (auto& in : L.plan.inputs)
    for (auto& l : in) live[l.buf] = true;
  for (auto& o : L.plan.outputs)
    if (o.buf >= 0) live[o.buf] = true;
  for (auto& st : L.plan.steps) {
    if (st.k == Step::Zero) continue;
    if (st.buf >= 0) live[st.buf] = true;
    if (st.buf2 >= 0) live[st.buf2] = true;
    for (auto& mi : st.merge) live[mi.delta] = live[mi.cell] = true;
    for (auto& a : st.args)
      if ((a.k == KArg::Buf || a.k == KArg::TMap) && a.buf >= 0) live[a.buf] = true;
  }
  std::vector<Step> kept;
  for (auto& st : L.plan.steps) {
    if ((st.k == Step::Zero && !live[st.buf]) || st.dead) continue;
    kept.push_back(st);
  }
  // kernel step indices referenced by partial buffers / finalize steps moved
  std::vector<int> remap(L.plan.steps.size(), -1);
  for (size_t i = 0, j = 0; i < L.plan.steps.size(); ++i) {
    const Step& st = L.plan.steps[i];
    if ((st.k == Step::Zero && !live[st.buf]) || st.dead) continue;
    remap[i] = (int)j++;
  }
  for (auto& st : kept)
    if (st.kernelStep >= 0) st.kernelStep = remap[st.kernelStep];
  for (auto& b : L.plan.bufs)
    if (b.partialKernel >= 0) b.partialKernel = remap[b.partialKernel];
  for (size_t b = 0; b < L.plan.bufs.size(); ++b)
    if (!live[b]) L.plan.bufs[b].elems = -1;  // not allocated
  L.plan.steps = std::move(kept);
  if (L.plan.gemm) L.plan.source = std::string(dxrt::gemmSource()) + "\n" + L.plan.source;
  return std::move(L.plan);
}

}  // namespace dev
}  // namespace dexlet
