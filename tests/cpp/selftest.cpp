// C++ API self-test: the reference front end (linked in libdexlet_cuda.so)
// parses/typechecks/simplifies programs exactly like the reference tests'
// runSimpl (tests/acceptance.cpp:68-71) and evalExprDevice replaces evalExpr.
// Inputs are bound as runtime env values.  Expected values are the
// reference tests' known answers.  Exit 0 on success.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "dexlet/errors.hpp"
#include "dexlet/parser.hpp"
#include "dexlet/printer.hpp"
#include "dexlet/simplify.hpp"
#include "dexlet/typecheck.hpp"
#include "dexlet_device.hpp"

using namespace dexlet;

static int failures = 0;

static ExprPtr compile(const std::string& src) {
  NameSupply::reset();
  ElabProgram p = parseProgram(src, "t.dexlet");
  TypeEnv env;
  checkExpr(Capability::pure(), env, p.whole());
  return optimize(simplifyExpr(p.whole()));
}

static std::vector<double> floats(const RtPtr& v) {
  std::vector<double> out;
  if (const auto* s = asRt<RScalar>(v)) return {s->v};
  if (const auto* t = asRt<RTable>(v))
    for (const auto& e : t->elems) {
      auto sub = floats(e);
      out.insert(out.end(), sub.begin(), sub.end());
    }
  if (const auto* p = asRt<RPairVal>(v)) {
    auto a = floats(p->l), b = floats(p->r);
    out.insert(out.end(), a.begin(), a.end());
    out.insert(out.end(), b.begin(), b.end());
  }
  return out;
}

static void expect(const char* name, const std::string& src, const std::vector<double>& want, bool f64) {
  try {
    DeviceOptions o;
    o.float64 = f64;
    RtPtr r = evalExprDevice(nullptr, compile(src), o);
    std::vector<double> got = floats(r);
    bool ok = got.size() == want.size();
    for (size_t i = 0; ok && i < got.size(); ++i) ok = std::fabs(got[i] - want[i]) <= (f64 ? 1e-12 : 1e-5);
    std::printf("%s %s (%s)\n", ok ? "PASS" : "FAIL", name, f64 ? "f64" : "f32");
    if (!ok) ++failures;
  } catch (const DexError& e) {
    std::printf("FAIL %s: %s\n", name, e.what());
    ++failures;
  }
}

// env-bound inputs, as the reference harness does
static void expectEnv(bool f64) {
  NameSupply::reset(1000000);
  ElabProgram p = parseProgram(
      "main = \\x:((Fin 2)=>((Fin 2)=>Float)). \\y:((Fin 2)=>((Fin 2)=>Float)). "
      "for i k. sum (for j. (x.i.j) * (y.j.k))\n",
      "t.dexlet");
  const ElabDecl* m = p.find("main");
  Name xn = NameSupply::fresh("x"), yn = NameSupply::fresh("y");
  ValuePtr T = vArray(vFin(vInt(2)), vArray(vFin(vInt(2)), vBase(BaseKind::Float)));
  TypeEnv tenv;
  tenv.bind(xn, T);
  tenv.bind(yn, T);
  Name a1 = NameSupply::fresh("ap"), a2 = NameSupply::fresh("ap");
  ExprPtr e = eLet(m->binder, nullptr, m->bound,
                   eLet(a1, nullptr, eApp(vVar(m->binder), vVar(xn)),
                        eLet(a2, nullptr, eApp(vVar(a1), vVar(yn)), eRet(vVar(a2)))));
  checkExpr(Capability::pure(), tenv, e);
  SimplResult r = simplify(tenv, e);
  ExprPtr o = optimize(contextFill(r.ctx, eRet(r.residual)));
  auto mat = [](double a, double b, double c, double d) {
    DescPtr f2 = descFin(2);
    auto row = [&](double u, double v) { return mkRt(RTable{f2, {mkRt(RScalar{u}), mkRt(RScalar{v})}}); };
    return mkRt(RTable{f2, {row(a, b), row(c, d)}});
  };
  auto bind = [](EnvPtr env, const Name& n, RtPtr v) {
    return std::make_shared<EnvNode>(EnvNode{n, std::move(v), std::move(env)});
  };
  EnvPtr env = bind(bind(nullptr, xn, mat(1, 2, 3, 4)), yn, mat(5, 6, 7, 8));
  DeviceOptions opts;
  opts.float64 = f64;
  std::vector<double> got = floats(evalExprDevice(env, o, opts));
  std::vector<double> want = {19, 22, 43, 50};
  bool ok = got == want;
  std::printf("%s env-bound matmul (%s)\n", ok ? "PASS" : "FAIL", f64 ? "f64" : "f32");
  if (!ok) ++failures;
}

int main() {
  for (bool f64 : {false, true}) {
    expect("matmul_2x2 (test_eval.cpp:60-80)",
           "x = [[1.0, 2.0], [3.0, 4.0]]\ny = [[5.0, 6.0], [7.0, 8.0]]\n"
           "z = for i k.\n  prods = for j. (x.i.j) * (y.j.k)\n  sum prods\nz\n",
           {19, 22, 43, 50}, f64);
    expect("histogram (test_eval.cpp:82-92)",
           "points : (Fin 5) => (Fin 3) = [@0, @1, @0, @2, @0]\n"
           "hist = yieldAccum \\h.\n  for i. h!(points.i) += 1.0\nhist\n",
           {3, 1, 1}, f64);
    expect("grad trace product (test_autodiff.cpp:199-220)",
           "b = [[5.0, 6.0], [7.0, 8.0]]\n"
           "f = \\a:((Fin 2)=>((Fin 2)=>Float)).\n  m = for i k. sum (for j. (a.i.j) * (b.j.k))\n"
           "  sum (for i. m.i.i)\ng = grad f [[1.0, 2.0], [3.0, 4.0]]\ng\n",
           {5, 7, 6, 8}, f64);
    expect("stateful recurrence grad (test_autodiff.cpp:184-197)",
           "f = \\xs:((Fin 3)=>Float). yieldState 0.0 \\s.\n  for i. s := ((get s) * 2.0) + (xs.i)\n  ()\n"
           "g = grad f [1.0, 2.0, 3.0]\ng\n",
           {4, 2, 1}, f64);
    expectEnv(f64);
  }
  return failures ? 1 : 0;
}
