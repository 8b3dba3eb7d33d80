"""Generates tests/golden/fixtures_golden.json from the reference's own test
fixtures (/root/reference/proj/tests/fixtures/*.dexlet; their `-- expect:`
headers drive the reference acceptance gate's criterion 1,
tests/acceptance.cpp:112-152).  For every file the expected outcome is taken
from the unmodified reference itself (oracle/_ref): the output leaves of the
whole-file evaluation (runSimpl, acceptance.cpp:68-71) for `-- expect: ok`
files, the error code for `-- expect: error` files.  The fixture text is
embedded as test input (the GPU box has no /root/reference).

    python tests/golden/make_fixture_golden.py
"""
import glob
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle

FIXTURES = "/root/reference/proj/tests/fixtures"

if __name__ == "__main__":
    out = {}
    for path in sorted(glob.glob(os.path.join(FIXTURES, "*.dexlet"))):
        name = os.path.basename(path)[:-len(".dexlet")]
        src = open(path).read()
        head = src.splitlines()[0] if src else ""
        case = {"source": src, "expect": head[len("-- expect: "):] if head.startswith("-- expect:") else "ok"}
        try:
            res = oracle.RefProgram(src, "")()
            case["outputs"] = [r.tolist() for r in res]
            case["output_kinds"] = ["int" if r.dtype.kind == "i" else "float" for r in res]
        except oracle.OracleError as e:
            case["error"] = str(e)
        out[name] = case
    with open(os.path.join(HERE, "fixtures_golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(len(out), "fixtures")
