"""Generates tests/golden/*.npz: outputs of the UNMODIFIED reference
(oracle/_ref/libmmplan_ref.so, compiled from /root/reference by
oracle/Makefile) on seeded inputs of the hot path.  Run in the build
container (it needs /root/reference); the fixtures then pin the oracle port
and the CUDA path anywhere, including boxes without the reference.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import golden_inputs as GI  # noqa: E402


def main():
    import oracle
    if not oracle.ref_available():
        oracle.build(ref=True)
    ref = oracle.ref()
    for name, fn in GI.CASES.items():
        out = fn(ref)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, {k: np.asarray(v).shape for k, v in out.items()})


if __name__ == "__main__":
    main()
