"""Loader for tests/golden (fixtures generated from the unmodified reference by
tests/golden/make_golden.py)."""
import json
import os

import numpy as np

from oracle import CsrMatrix

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))


def case(name):
    meta = MANIFEST[name]
    arrays = dict(np.load(os.path.join(GOLDEN, name + ".npz"))) if meta.get("type") != "small_dense" else {}
    return meta, arrays


def matrix(arrays):
    return CsrMatrix(arrays["offs"], arrays["cols"], arrays["vals"])


def names(type_=None):
    return sorted(k for k, v in MANIFEST.items() if type_ is None or v.get("type") == type_)


def rel_diff(a, b):
    """tests/support/oracles.hpp:141-144"""
    s = max(abs(a), abs(b))
    return 0.0 if s == 0.0 else abs(a - b) / s
