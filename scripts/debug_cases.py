"""Dev tool: run named parity cases on the device and print got vs want."""
import sys, traceback
import numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import oracle
import paper_2104_05372_b200 as dx
from tests.parity_cases import cases
ctx = dx.Context(0)
names = sys.argv[1:]
for name, src, inputs in cases():
    if names and name not in names: continue
    print("=" * 20, name)
    try:
        want = oracle.RefProgram(src)(*inputs)
    except Exception as e:
        print("ORACLE ERROR", e); print(src); continue
    for f64 in (False, True):
        try:
            p = dx.Program(src, ctx=ctx, float64=f64)
            got = p(*inputs)
            for g, w in zip(got, want):
                d = oracle.rel_diff(g, w)
                print(f"f64={f64} reldiff={d:.3g}", "" if d < 1e-4 else f"\n got={g[:12]}\n want={w[:12]}")
            if f64 and any(oracle.rel_diff(g, w) > 1e-9 for g, w in zip(got, want)):
                print(p.plan)
                print(p.source[-6000:])
        except Exception as e:
            print("DEVICE ERROR", e)
