#!/usr/bin/env python3
"""Front-end extension: `exp` / `log` in the language, and a (trivial) tangent
for `<` -- SURVEY.md section 8(f) item 4.

The reference IR has no transcendental operators (ir.hpp:124 UnOp = Ordinal,
IntToFloat, ReverseIndex) and linearize rejects comparisons
(autodiff.cpp:194-195), so the ADBench GMM objective (configs[2]) and any
max-stabilised log-sum-exp cannot be written as a dexlet program.  This
script is the extension layer: it copies the reference front end from
$REF (read-only, never edited) into a build directory and applies a short
list of anchored insertions -- every inserted line is ours and listed below,
every anchor must match exactly once (the build fails loudly otherwise).
Nothing is committed but this file; the patched copies live under build/.

  usage: extend.py REF_PROJ_DIR OUT_DIR

Semantics added (each cites the reference site it extends):
  * UnOp::Exp, UnOp::Log            ir.hpp:124
  * surface syntax `exp x`, `log x` parser.cpp:602-615 (elaboration), 1388-1390 (core)
  * typing Float -> Float           typecheck.cpp:464-477
  * printing                        printer.cpp:356-358
  * linearize: d exp x = exp x * dx (primal bound once in the context),
               d log x = dx / x     autodiff.cpp:200-204
  * linearize: x < y has a unit tangent (case on it needs no tangent of the
               scrutinee, autodiff.cpp:266-275)           autodiff.cpp:194-195
  * evaluation (oracle only): std::exp / std::log in double  eval.cpp:516-533
Transposition needs no change: the tangents above use only Mul and Div with
one linear side, which transpose already handles (autodiff.cpp:620-640).
"""
import os
import shutil
import sys

EDITS = [
    ("include/dexlet/ir.hpp",
     "enum class UnOp { Ordinal, IntToFloat, ReverseIndex };",
     "enum class UnOp { Ordinal, IntToFloat, ReverseIndex, Exp, Log };  // Exp, Log: frontend_ext"),
    ("src/parser.cpp",
     '    if (s == "sum") {',
     '''    if (s == "exp" || s == "log") {  // frontend_ext: transcendental unary ops
      const bool isExp = s == "exp";
      return unary(
          [&](EV a, Span p) {
            ValuePtr ft = vBase(BaseKind::Float);
            return EV{emit(b, eUn(isExp ? UnOp::Exp : UnOp::Log, a.v, p), ft), ft};
          },
          isExp ? "exp" : "log");
    }
    if (s == "sum") {'''),
    ("src/parser.cpp",
     '    if (isIdent("reverse")) { ++pos; return eUn(UnOp::ReverseIndex, coreAtom(), sp); }',
     '''    if (isIdent("reverse")) { ++pos; return eUn(UnOp::ReverseIndex, coreAtom(), sp); }
    if (isIdent("exp")) { ++pos; return eUn(UnOp::Exp, coreAtom(), sp); }  // frontend_ext
    if (isIdent("log")) { ++pos; return eUn(UnOp::Log, coreAtom(), sp); }  // frontend_ext'''),
    ("src/typecheck.cpp",
     '''      case UnOp::ReverseIndex:
        requireConstraint(Constraint::IdxSet, t, sp);
        return t;''',
     '''      case UnOp::ReverseIndex:
        requireConstraint(Constraint::IdxSet, t, sp);
        return t;
      case UnOp::Exp:  // frontend_ext
      case UnOp::Log:
        expectType(t, tFloat(), sp, "exp/log operand");
        return tFloat();'''),
    ("src/printer.cpp",
     'case UnOp::ReverseIndex: out += "reverse "; break;',
     'case UnOp::ReverseIndex: out += "reverse "; break;\n'
     '                case UnOp::Exp: out += "exp "; break;  // frontend_ext\n'
     '                case UnOp::Log: out += "log "; break;'),
    ("src/autodiff.cpp",
     '''      case BinOp::Less:
        fail(ErrCode::UnsupportedTangent, "comparison has no tangent", sp);''',
     '''      case BinOp::Less:  // frontend_ext: a comparison's tangent is trivial
        return {{}, primal, eRet(vUnit())};'''),
    ("src/autodiff.cpp",
     '''  Res linNode(Delta&, const EUnOp& n, Span sp) {
    ExprPtr primal = eUn(n.op, n.v, sp);
    if (n.op == UnOp::IntToFloat) return {{}, primal, eRet(vFloat(0.0))};''',
     '''  Res linNode(Delta& d, const EUnOp& n, Span sp) {
    ExprPtr primal = eUn(n.op, n.v, sp);
    if (n.op == UnOp::IntToFloat) return {{}, primal, eRet(vFloat(0.0))};
    if (n.op == UnOp::Exp) {  // frontend_ext: d exp x = exp x * dx
      Name y = NameSupply::fresh("ex");
      env.bind(y, floatT());  // the tangent is typechecked in this env (linNode(ELet))
      SimplContext ctx;
      ctx.bindings.push_back(Binding{y, floatT(), primal});
      return {std::move(ctx), eRet(vVar(y)), eBin(BinOp::Mul, vVar(y), deltaOf(d, n.v), sp)};
    }
    if (n.op == UnOp::Log)  // frontend_ext: d log x = dx / x
      return {{}, primal, eBin(BinOp::Div, deltaOf(d, n.v), n.v, sp)};'''),
    ("src/eval.cpp",
     '''      case UnOp::ReverseIndex: {
        DescPtr d = descOfRt(v);''',
     '''      case UnOp::Exp:  // frontend_ext
      case UnOp::Log: {
        const auto* x = asRt<RScalar>(v);
        if (!x) fail(ErrCode::Internal, "exp/log operand is not a float", sp);
        return rtScalar(n.op == UnOp::Exp ? std::exp(x->v) : std::log(x->v));
      }
      case UnOp::ReverseIndex: {
        DescPtr d = descOfRt(v);'''),
]


def main():
    ref, out = sys.argv[1], sys.argv[2]
    tmp = out + ".tmp"
    shutil.rmtree(tmp, ignore_errors=True)
    for sub in ("include/dexlet", "src"):
        os.makedirs(os.path.join(tmp, sub))
        for f in sorted(os.listdir(os.path.join(ref, sub))):
            shutil.copyfile(os.path.join(ref, sub, f), os.path.join(tmp, sub, f))
    for rel, anchor, repl in EDITS:
        p = os.path.join(tmp, rel)
        with open(p) as f:
            text = f.read()
        n = text.count(anchor)
        if n != 1:
            sys.exit(f"frontend_ext: anchor matched {n} times in {rel}: {anchor[:60]!r}")
        with open(p, "w") as f:
            f.write(text.replace(anchor, repl))
    # replace atomically, keeping timestamps of unchanged files for make
    for sub in ("include/dexlet", "src"):
        os.makedirs(os.path.join(out, sub), exist_ok=True)
        for f in sorted(os.listdir(os.path.join(tmp, sub))):
            src, dst = os.path.join(tmp, sub, f), os.path.join(out, sub, f)
            if not os.path.exists(dst) or open(src).read() != open(dst).read():
                shutil.copyfile(src, dst)
    shutil.rmtree(tmp)


if __name__ == "__main__":
    main()
