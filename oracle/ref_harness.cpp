// ORACLE / TEST INFRASTRUCTURE ONLY — never part of the product path.
//
// C-ABI harness around the reference evaluator (dexlet `evalExpr`,
// /root/reference/proj/src/eval.cpp:621-633) so tests, smoke() and the bench's
// cpu_baseline leg can run the unmodified reference on exactly the inputs the
// device path sees.  The reference library is compiled from its own sources
// by oracle/Makefile into oracle/_ref/ (never copied into this repo).
//
// Harness shape follows the reference's own tests: parse -> checkExpr ->
// simplify -> optimize -> evalExpr with inputs bound as runtime env values
// (tests/acceptance.cpp:54-71), never as literals.
//
// Flattening convention (shared with include/dexlet_cuda.h): a value is a list
// of SoA leaves; tables are row-major by index-set ordinal (index_set.cpp:74-97),
// a table of pairs is a pair of tables, index members are ordinals.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "dexlet/errors.hpp"
#include "dexlet/eval.hpp"
#include "dexlet/index_set.hpp"
#include "dexlet/parser.hpp"
#include "dexlet/printer.hpp"
#include "dexlet/simplify.hpp"
#include "dexlet/typecheck.hpp"

using namespace dexlet;

namespace {

thread_local std::string g_err;

struct Leaf {
  int kind;  // 0 float, 1 int, 2 index
  std::vector<double> f;
  std::vector<long long> i;
  long long count() const { return kind == 0 ? (long long)f.size() : (long long)i.size(); }
};

// Static shape of an input type (literal sizes).
struct Shape {
  enum K { Float, Int, Unit, Idx, Pair, Table } k;
  DescPtr desc;
  std::shared_ptr<Shape> a, b;
};
using ShapeP = std::shared_ptr<Shape>;

ShapeP shapeOf(const ValuePtr& t) {
  auto s = std::make_shared<Shape>();
  if (isBase(t, BaseKind::Float)) { s->k = Shape::Float; return s; }
  if (isBase(t, BaseKind::Int)) { s->k = Shape::Int; return s; }
  if (isBase(t, BaseKind::Unit)) { s->k = Shape::Unit; return s; }
  if (as<VFinType>(t) || as<VEitherType>(t)) { s->k = Shape::Idx; s->desc = descFromType(t); return s; }
  if (const auto* p = as<VPairType>(t)) { s->k = Shape::Pair; s->a = shapeOf(p->l); s->b = shapeOf(p->r); return s; }
  if (const auto* a = as<VArrayType>(t)) { s->k = Shape::Table; s->desc = descFromType(a->dom); s->a = shapeOf(a->cod); return s; }
  fail(ErrCode::Internal, "oracle: unsupported input type " + printValue(t));
}

void leavesOf(const ShapeP& s, long long mult, std::vector<std::pair<int, long long>>& out) {
  switch (s->k) {
    case Shape::Float: out.push_back({0, mult}); return;
    case Shape::Int: out.push_back({1, mult}); return;
    case Shape::Unit: return;
    case Shape::Idx:
      if (s->desc->kind == IndexSetDesc::Kind::Unit) return;
      out.push_back({2, mult});
      return;
    case Shape::Pair: leavesOf(s->a, mult, out); leavesOf(s->b, mult, out); return;
    case Shape::Table: leavesOf(s->a, mult * size(s->desc), out); return;
  }
}

size_t numLeaves(const ShapeP& s) {
  std::vector<std::pair<int, long long>> v;
  leavesOf(s, 1, v);
  return v.size();
}

// Builds the boxed RtVal for element `e` of a value with leaves `L`.
RtPtr unflatten(const ShapeP& s, const std::vector<Leaf*>& L, size_t base, long long e, long long per) {
  switch (s->k) {
    case Shape::Float: return mkRt(RScalar{L[base]->f[e]});
    case Shape::Int: return mkRt(RIntVal{L[base]->i[e]});
    case Shape::Unit: return mkRt(RUnitVal{});
    case Shape::Idx:
      if (s->desc->kind == IndexSetDesc::Kind::Unit) return mkRt(RUnitVal{});
      return fromOrdinalRt(L[base]->i[e], s->desc);  // bounds-checked (E-bounds)
    case Shape::Pair: {
      RtPtr a = unflatten(s->a, L, base, e, per);
      RtPtr b = unflatten(s->b, L, base + numLeaves(s->a), e, per);
      return mkRt(RPairVal{a, b});
    }
    case Shape::Table: {
      long long n = size(s->desc);
      std::vector<RtPtr> elems;
      elems.reserve(n);
      for (long long k = 0; k < n; ++k) elems.push_back(unflatten(s->a, L, base, e * n + k, per));
      return mkRt(RTable{s->desc, std::move(elems)});
    }
  }
  return nullptr;
}

// Flattens a runtime value into SoA leaves (kinds inferred from the value).
void flatten(const RtPtr& v, std::vector<Leaf>& out) {
  if (const auto* x = asRt<RScalar>(v)) { Leaf l; l.kind = 0; l.f = {x->v}; out.push_back(l); return; }
  if (const auto* x = asRt<RIntVal>(v)) { Leaf l; l.kind = 1; l.i = {x->v}; out.push_back(l); return; }
  if (asRt<RUnitVal>(v)) return;
  if (asRt<RIndexVal>(v) || asRt<RSumVal>(v)) {
    DescPtr d = descOfRt(v);
    if (!d) fail(ErrCode::Internal, "oracle: sum value without index shape");
    if (d->kind == IndexSetDesc::Kind::Unit) return;
    Leaf l; l.kind = 2; l.i = {ordinalOfRt(v)}; out.push_back(l); return;
  }
  if (const auto* p = asRt<RPairVal>(v)) {
    // pairs of index members flatten componentwise, like the device
    flatten(p->l, out);
    flatten(p->r, out);
    return;
  }
  if (const auto* t = asRt<RTable>(v)) {
    std::vector<std::vector<Leaf>> per;
    for (const auto& e : t->elems) {
      std::vector<Leaf> le;
      flatten(e, le);
      per.push_back(std::move(le));
    }
    if (per.empty()) return;
    size_t nl = per[0].size();
    for (size_t l = 0; l < nl; ++l) {
      Leaf acc;
      acc.kind = per[0][l].kind;
      for (auto& pe : per) {
        acc.f.insert(acc.f.end(), pe[l].f.begin(), pe[l].f.end());
        acc.i.insert(acc.i.end(), pe[l].i.begin(), pe[l].i.end());
      }
      out.push_back(std::move(acc));
    }
    return;
  }
  if (const auto* c = asRt<RClosure>(v)) {
    // a lazy `view` result: force it element by element through the
    // reference's own indexing (EIndex applies the closure, eval.cpp:286-293)
    const auto* view = as<VView>(c->fn);
    if (!view) fail(ErrCode::Internal, "oracle: cannot flatten a function result");
    DescPtr d = descFromType(view->annot);
    std::vector<RtPtr> elems;
    Name arr = NameSupply::fresh("oracle_view"), idx = NameSupply::fresh("oracle_idx");
    for (long long k = 0; k < size(d); ++k) {
      EnvPtr env = envBind(envBind(nullptr, arr, v), idx, fromOrdinalRt(k, d));
      elems.push_back(evalExpr(env, eIndex(vVar(arr), vVar(idx))));
    }
    flatten(mkRt(RTable{d, std::move(elems)}), out);
    return;
  }
  fail(ErrCode::Internal, "oracle: cannot flatten a reference result");
}

}  // namespace

struct dxo_program {
  ExprPtr optimized;
  std::vector<Name> names;
  std::vector<ShapeP> shapes;
  std::vector<std::vector<Leaf>> inputs;
  std::vector<Leaf> outputs;
  EvalCounters counters;
  std::string ir;
};

#define GUARD_BEGIN try {
#define GUARD_END                                                        \
  }                                                                      \
  catch (const DexError& e) {                                            \
    g_err = std::string(errCodeName(e.code())) + ": " + e.message();     \
    return 1000 + (int)e.code();                                         \
  }                                                                      \
  catch (const std::exception& e) {                                      \
    g_err = e.what();                                                    \
    return 999;                                                          \
  }

extern "C" {

const char* dxo_last_error(void) { return g_err.c_str(); }

// Status: 0 ok; 1000 + ErrCode for DexError (errors.hpp:10-26); 999 other.
int dxo_program_create(const char* source, const char* entry, dxo_program** out) {
  GUARD_BEGIN
  NameSupply::reset(1000000);
  ElabProgram p = parseProgram(source, "program.dexlet");
  if (!entry || !*entry) {
    // whole file (the reference harness's runSimpl, tests/acceptance.cpp:68-71)
    auto* prog = new dxo_program();
    ExprPtr e = p.whole();
    TypeEnv env;
    checkExpr(Capability::pure(), env, e);
    SimplResult r = simplify(env, e);
    prog->optimized = optimize(contextFill(r.ctx, eRet(r.residual)));
    prog->ir = printExpr(prog->optimized);
    *out = prog;
    return 0;
  }
  const ElabDecl* m = p.find(entry);
  if (!m) fail(ErrCode::UnboundVariable, std::string("entry '") + entry + "' is not defined");
  auto* prog = new dxo_program();
  std::vector<std::pair<Name, ValuePtr>> params;
  ExprPtr b = m->bound;
  while (true) {
    const ERet* r = as<ERet>(b);
    if (!r) break;
    const VLam* l = as<VLam>(r->value);
    if (!l) break;
    params.push_back({NameSupply::fresh(l->binder.text), l->annot});
    b = l->body;
  }
  TypeEnv env;
  for (auto& [n, t] : params) {
    env.bind(n, t);
    prog->names.push_back(n);
    prog->shapes.push_back(shapeOf(t));
    std::vector<std::pair<int, long long>> lv;
    leavesOf(prog->shapes.back(), 1, lv);
    std::vector<Leaf> leaves;
    for (auto& [k, c] : lv) {
      Leaf l;
      l.kind = k;
      if (k == 0) l.f.assign(c, 0.0);
      else l.i.assign(c, 0);
      leaves.push_back(l);
    }
    prog->inputs.push_back(std::move(leaves));
  }
  Name last = m->binder;
  std::vector<std::pair<Name, ExprPtr>> apps;
  for (auto& [n, t] : params) {
    Name a = NameSupply::fresh("ap");
    apps.push_back({a, eApp(vVar(last), vVar(n))});
    last = a;
  }
  ExprPtr e = eRet(vVar(last));
  for (auto it = apps.rbegin(); it != apps.rend(); ++it) e = eLet(it->first, nullptr, it->second, e);
  for (auto it = p.decls.rbegin(); it != p.decls.rend(); ++it) e = eLet(it->binder, nullptr, it->bound, e);
  checkExpr(Capability::pure(), env, e);
  SimplResult r = simplify(env, e);
  prog->optimized = optimize(contextFill(r.ctx, eRet(r.residual)));
  prog->ir = printExpr(prog->optimized);
  *out = prog;
  return 0;
  GUARD_END
}

int dxo_program_destroy(dxo_program* p) {
  delete p;
  return 0;
}

int dxo_program_num_inputs(dxo_program* p) { return (int)p->inputs.size(); }
int dxo_program_input_num_leaves(dxo_program* p, int i) { return (int)p->inputs[i].size(); }
int dxo_program_input_leaf(dxo_program* p, int i, int l, int* kind, int64_t* count) {
  *kind = p->inputs[i][l].kind;
  *count = p->inputs[i][l].count();
  return 0;
}

int dxo_program_set_input_f64(dxo_program* p, int i, int l, const double* data) {
  Leaf& leaf = p->inputs[i][l];
  if (leaf.kind == 0) std::memcpy(leaf.f.data(), data, leaf.f.size() * sizeof(double));
  else for (size_t k = 0; k < leaf.i.size(); ++k) leaf.i[k] = (long long)data[k];
  return 0;
}

int dxo_program_set_input_i64(dxo_program* p, int i, int l, const int64_t* data) {
  Leaf& leaf = p->inputs[i][l];
  if (leaf.kind == 0) for (size_t k = 0; k < leaf.f.size(); ++k) leaf.f[k] = (double)data[k];
  else std::memcpy(leaf.i.data(), data, leaf.i.size() * sizeof(int64_t));
  return 0;
}

// Evaluates with EvalOptions{chunks} (eval.hpp:67-69); fills counters
// [arithmeticOps, accumUpdates, cellsAllocated, nodesEvaluated] and the
// wall time of evalExpr alone in *ms.
int dxo_program_run(dxo_program* p, int chunks, int64_t* counters4, double* ms) {
  GUARD_BEGIN
  EnvPtr env;
  for (size_t i = 0; i < p->inputs.size(); ++i) {
    std::vector<Leaf*> L;
    for (auto& l : p->inputs[i]) L.push_back(&l);
    env = envBind(env, p->names[i], unflatten(p->shapes[i], L, 0, 0, 1));
  }
  EvalOptions o;
  o.chunks = chunks < 1 ? 1 : chunks;
  EvalCounters c;
  auto t0 = std::chrono::steady_clock::now();
  RtPtr r = evalExpr(env, p->optimized, o, &c);
  auto t1 = std::chrono::steady_clock::now();
  if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  p->outputs.clear();
  flatten(r, p->outputs);
  p->counters = c;
  if (counters4) {
    counters4[0] = c.arithmeticOps;
    counters4[1] = c.accumUpdates;
    counters4[2] = c.cellsAllocated;
    counters4[3] = c.nodesEvaluated;
  }
  return 0;
  GUARD_END
}

int dxo_program_num_outputs(dxo_program* p) { return (int)p->outputs.size(); }
int dxo_program_output_leaf(dxo_program* p, int l, int* kind, int64_t* count) {
  *kind = p->outputs[l].kind;
  *count = p->outputs[l].count();
  return 0;
}
int dxo_program_get_output_f64(dxo_program* p, int l, double* out) {
  const Leaf& leaf = p->outputs[l];
  if (leaf.kind == 0) std::memcpy(out, leaf.f.data(), leaf.f.size() * sizeof(double));
  else for (size_t k = 0; k < leaf.i.size(); ++k) out[k] = (double)leaf.i[k];
  return 0;
}
const char* dxo_program_ir(dxo_program* p) { return p->ir.c_str(); }

// Runs a whole source file the way the reference's tests do
// (`runSimpl`, tests/acceptance.cpp:68-71): result printed by printResult.
int dxo_run_source(const char* source, int chunks, char* out, size_t cap) {
  GUARD_BEGIN
  NameSupply::reset();
  ElabProgram p = parseProgram(source, "t.dexlet");
  TypeEnv env;
  checkExpr(Capability::pure(), env, p.whole());
  ExprPtr e = optimize(simplifyExpr(p.whole()));
  EvalOptions o;
  o.chunks = chunks < 1 ? 1 : chunks;
  std::string s = printResult(evalExpr(nullptr, e, o));
  std::snprintf(out, cap, "%s", s.c_str());
  return 0;
  GUARD_END
}

}  // extern "C"
