"""Generates tests/golden/*.json by running the unmodified reference evaluator
(oracle/_ref, built from /root/reference sources) on the seeded parity cases.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The JSON files are committed so the GPU box (no /root/reference) can check the
device path against the reference's own outputs.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from tests.parity_cases import cases  # noqa: E402


def _leaves(x):
    return [x] if isinstance(x, np.ndarray) else list(x)


def main():
    out = {}
    for name, src, inputs in cases():
        ref = oracle.RefProgram(src)
        res = ref(*inputs)
        out[name] = {
            "source": src,
            "inputs": [[np.asarray(l).ravel().tolist() for l in _leaves(x)] for x in inputs],
            "input_dtypes": [[str(np.asarray(l).dtype) for l in _leaves(x)] for x in inputs],
            "outputs": [r.tolist() for r in res],
            "output_kinds": ["float" if r.dtype == np.float64 else "int" for r in res],
            "counters": ref.counters,
        }
    path = os.path.join(HERE, "parity_golden.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(f"wrote {path}: {len(out)} cases")


if __name__ == "__main__":
    main()
