// evalExprDevice: the C++ drop-in twin of the reference's evalExpr
// (reference proj/include/dexlet/eval.hpp:74-75, proj/src/eval.cpp:621-633).
//
// Free variables of `e` are read from the boxed runtime environment, packed
// into SoA leaves (the layout of include/dexlet_cuda.h), the expression is
// lowered and run on the GPU, and the output leaves are unpacked back into an
// RtVal tree.  The reference's RtVal helpers that live in eval.cpp (envLookup,
// fromOrdinalRt, ...) are not linked into this library -- the evaluator is
// not part of the product -- so the few needed here are restated locally.

#include "dexlet_device.hpp"

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "dexlet/errors.hpp"
#include "dexlet/index_set.hpp"
#include "dexlet/printer.hpp"
#include "lower.hpp"
#include "program_impl.hpp"
#include "runtime.hpp"

namespace dexlet {
namespace {

RtPtr lookup(const EnvPtr& env, const Name& n) {
  for (const EnvNode* p = env.get(); p; p = p->next.get())
    if (p->name == n) return p->v;
  return nullptr;
}

// Core type of a runtime value (sizes literal), for the lowering's inputs.
ValuePtr typeOfRt(const RtPtr& v) {
  if (asRt<RScalar>(v)) return vBase(BaseKind::Float);
  if (asRt<RIntVal>(v)) return vBase(BaseKind::Int);
  if (asRt<RUnitVal>(v)) return vBase(BaseKind::Unit);
  if (const auto* i = asRt<RIndexVal>(v)) return descType(i->desc);
  if (const auto* s = asRt<RSumVal>(v)) {
    if (s->eitherDesc) return descType(s->eitherDesc);
    fail(ErrCode::Internal, "device inputs: data sum values are not supported");
  }
  if (const auto* p = asRt<RPairVal>(v)) return vPairType(typeOfRt(p->l), typeOfRt(p->r));
  if (const auto* t = asRt<RTable>(v)) {
    if (t->elems.empty()) fail(ErrCode::Internal, "device inputs: empty table");
    return vArray(descType(t->dom), typeOfRt(t->elems[0]));
  }
  fail(ErrCode::Internal, "device inputs: closures and references cannot be uploaded");
}

long long ordinalOf(const RtPtr& v) {
  if (asRt<RUnitVal>(v)) return 0;
  if (const auto* i = asRt<RIndexVal>(v)) return i->ord;
  if (const auto* s = asRt<RSumVal>(v)) {
    if (!s->eitherDesc) fail(ErrCode::Internal, "sum member has no index shape");
    return s->isLeft ? ordinalOf(s->payload) : size(s->eitherDesc->left) + ordinalOf(s->payload);
  }
  fail(ErrCode::Internal, "value is not an index-set member");
}

// Flatten into per-leaf double vectors (SoA, row-major by ordinal).
void flatten(const RtPtr& v, std::vector<std::vector<double>>& leaves, size_t& leaf) {
  if (const auto* s = asRt<RScalar>(v)) { leaves[leaf++].push_back(s->v); return; }
  if (const auto* i = asRt<RIntVal>(v)) { leaves[leaf++].push_back((double)i->v); return; }
  if (asRt<RUnitVal>(v)) return;
  if (asRt<RIndexVal>(v) || asRt<RSumVal>(v)) {
    const auto* iv = asRt<RIndexVal>(v);
    if (iv && iv->desc->kind == IndexSetDesc::Kind::Unit) return;
    leaves[leaf++].push_back((double)ordinalOf(v));
    return;
  }
  if (const auto* p = asRt<RPairVal>(v)) {
    flatten(p->l, leaves, leaf);
    flatten(p->r, leaves, leaf);
    return;
  }
  if (const auto* t = asRt<RTable>(v)) {
    size_t start = leaf;
    size_t end = start;
    for (const auto& e : t->elems) {
      size_t l = start;
      flatten(e, leaves, l);
      end = l;
    }
    leaf = end;
    return;
  }
  fail(ErrCode::Internal, "device inputs: unsupported runtime value");
}

RtPtr memberOf(long long o, const DescPtr& d) {
  switch (d->kind) {
    case IndexSetDesc::Kind::Unit: return mkRt(RUnitVal{});
    case IndexSetDesc::Kind::Fin: return mkRt(RIndexVal{o, d});
    case IndexSetDesc::Kind::Pair: {
      long long rs = size(d->right);
      return mkRt(RPairVal{memberOf(o / rs, d->left), memberOf(o % rs, d->right)});
    }
    case IndexSetDesc::Kind::Either: {
      long long ls = size(d->left);
      if (o < ls) return mkRt(RSumVal{true, memberOf(o, d->left), d});
      return mkRt(RSumVal{false, memberOf(o - ls, d->right), d});
    }
  }
  return mkRt(RUnitVal{});
}

// Rebuild a boxed value of device type `t` from output leaves.
RtPtr unflatten(const dev::DTy& t, const std::vector<std::vector<double>>& L, size_t& leaf, long long e) {
  using dev::DType;
  switch (t->k) {
    case DType::Float: return mkRt(RScalar{L[leaf++][e]});
    case DType::Int: return mkRt(RIntVal{(long long)L[leaf++][e]});
    case DType::Unit: return mkRt(RUnitVal{});
    case DType::Idx:
      if (t->desc->kind == IndexSetDesc::Kind::Unit) return mkRt(RUnitVal{});
      return memberOf((long long)L[leaf++][e], t->desc);
    case DType::Pair: {
      RtPtr a = unflatten(t->a, L, leaf, e);
      RtPtr b = unflatten(t->b, L, leaf, e);
      return mkRt(RPairVal{a, b});
    }
    case DType::Table: {
      long long n = size(t->desc);
      size_t start = leaf, end = leaf;
      std::vector<RtPtr> elems;
      elems.reserve(n);
      for (long long k = 0; k < n; ++k) {
        size_t l = start;
        elems.push_back(unflatten(t->a, L, l, e * n + k));
        end = l;
      }
      leaf = end;
      return mkRt(RTable{t->desc, std::move(elems)});
    }
    default: fail(ErrCode::Internal, "device outputs: unsupported result type");
  }
}

dxrt::Ctx* contextFor(int device) {
  static std::mutex mu;
  static std::map<int, dxrt::Ctx*> ctxs;
  std::lock_guard<std::mutex> lk(mu);
  auto it = ctxs.find(device);
  if (it != ctxs.end()) return it->second;
  dxrt::Ctx* c = nullptr;
  if (dxrt::Ctx::create(device, &c)) fail(ErrCode::Internal, "CUDA: " + dxrt::lastError());
  ctxs[device] = c;
  return c;
}

void checkRc(int rc) {
  if (rc) fail(ErrCode::Internal, "device: " + dxrt::lastError());
}

}  // namespace

RtPtr evalExprDevice(const EnvPtr& env, const ExprPtr& e, const DeviceOptions& opts, EvalCounters* counters) {
  // inputs = free variables bound in the environment
  std::vector<std::pair<Name, ValuePtr>> inputs;
  std::vector<RtPtr> values;
  for (const Name& n : freeVars(e)) {
    RtPtr v = lookup(env, n);
    // freeVars also reports type-level names (effect regions in Ref
    // annotations); only runtime values become device inputs.  A value
    // that is genuinely missing makes the lowering fail loudly.
    if (!v) continue;
    inputs.push_back({n, typeOfRt(v)});
    values.push_back(v);
  }
  dev::LowerOptions lo;
  lo.f64 = opts.float64;
  lo.rank = opts.rank;
  lo.world = opts.world;
  // counters requested: count mode (kernels add the + - * / and += they
  // execute; see dxl_program_counters for what is added statically)
  lo.count = counters != nullptr;
  if (lo.count) lo.noGemm = true;
  dev::Program prog;
  prog.ctx = contextFor(opts.device);
  prog.plan = dev::lowerProgram(e, inputs, lo);
  prog.plan.source = std::string(lo.f64 ? "typedef double dx_f;\n" : "typedef float dx_f;\n") + prog.plan.source;
  checkRc(prog.prepare());
  prog.ctx->makeCurrent();
  // pack + upload inputs
  for (size_t i = 0; i < values.size(); ++i) {
    const auto& in = prog.plan.inputs[i];
    std::vector<std::vector<double>> leaves(in.size());
    size_t leaf = 0;
    flatten(values[i], leaves, leaf);
    for (size_t l = 0; l < in.size(); ++l) {
      if ((long long)leaves[l].size() != in[l].count) fail(ErrCode::Internal, "device inputs: leaf size mismatch");
      std::vector<char> buf(in[l].count * dev::storageBytes(in[l].kind, lo.f64));
      for (long long k = 0; k < in[l].count; ++k) {
        double x = leaves[l][k];
        char* p = buf.data() + k * dev::storageBytes(in[l].kind, lo.f64);
        switch (in[l].kind) {
          case dev::SK::F:
            if (lo.f64) std::memcpy(p, &x, 8);
            else { float f = (float)x; std::memcpy(p, &f, 4); }
            break;
          case dev::SK::I: { long long v = (long long)x; std::memcpy(p, &v, 8); break; }
          default: { int v = (int)x; std::memcpy(p, &v, 4); break; }
        }
      }
      checkRc(dxrt::check(cuMemcpyHtoD(prog.devptr[in[l].buf], buf.data(), buf.size()), "upload"));
    }
  }
  checkRc(prog.run());
  checkRc(dxrt::check(cuStreamSynchronize(prog.ctx->stream), "sync"));
  int flag = 0;
  checkRc(dxrt::check(cuMemcpyDtoH(&flag, prog.devptr[prog.plan.errFlagBuf], 4), "flag"));
  if (flag) fail(ErrCode::OutOfBounds, "an index value is outside its index set");
  if (counters) {  // EvalCounters semantics (eval.hpp:60-65), summed like the reference's
    long long c[3] = {0, 0, 0};
    checkRc(dxrt::check(cuMemcpyDtoH(c, prog.devptr[prog.plan.countBuf], sizeof c), "counters"));
    counters->arithmeticOps += c[0] + prog.plan.staticOps;
    counters->accumUpdates += c[1] + prog.plan.staticAccums;
    counters->cellsAllocated += c[2] + prog.plan.cellsAllocated;
  }
  // download + unpack outputs
  std::vector<std::vector<double>> outs;
  for (const auto& o : prog.plan.outputs) {
    std::vector<double> vals;
    if (o.host) {
      vals.push_back(o.kind == dev::SK::F || o.kind == dev::SK::D ? o.hostF[0] : (double)o.hostI[0]);
    } else {
      size_t es = dev::storageBytes(o.kind, lo.f64);
      std::vector<char> raw(o.count * es);
      checkRc(dxrt::check(cuMemcpyDtoH(raw.data(), prog.devptr[o.buf] + o.off * es, raw.size()), "download"));
      for (long long k = 0; k < o.count; ++k) {
        const char* p = raw.data() + k * es;
        double x = 0;
        if (o.kind == dev::SK::F || o.kind == dev::SK::D) {
          if (es == 8) std::memcpy(&x, p, 8);
          else { float f; std::memcpy(&f, p, 4); x = f; }
        } else if (o.kind == dev::SK::I) {
          long long v; std::memcpy(&v, p, 8); x = (double)v;
        } else {
          int v; std::memcpy(&v, p, 4); x = v;
        }
        vals.push_back(x);
      }
    }
    outs.push_back(std::move(vals));
  }
  size_t leaf = 0;
  return unflatten(prog.plan.outputType, outs, leaf, 0);
}

}  // namespace dexlet
