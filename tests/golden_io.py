"""Loaders for the golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def kernel_cases(kind=None):
    cases = load_json("kernel_cases.json")
    return [c for c in cases if kind is None or c["kind"] == kind]


def vec_arrays(v):
    """(size, indices-or-None, values ndarray, zero) of a JSON vector."""
    if v is None:
        return None
    dt = np.dtype(v["dtype"])
    vals = np.asarray(v["values"], dtype=dt)
    idx = None if v["indices"] is None else np.asarray(v["indices"], dtype=np.int64)
    return v["size"], idx, vals, dt.type(v["zero"])


def mat_arrays(m):
    dt = np.dtype(m["dtype"])
    return (np.asarray(m["rows"], np.int64), np.asarray(m["cols"], np.int64),
            np.asarray(m["values"], dtype=dt), m["nrows"], m["ncols"], m["has_csc"])


def canonical(size, idx, vals, zero):
    """Canonical (indices, values) as Vector.extract_tuples gives them."""
    if idx is not None:
        return idx, vals
    i = np.flatnonzero(vals != zero).astype(np.int64)
    return i, vals[i]


def same_values(got, want, rtol=1e-10):
    got = np.asarray(got)
    want = np.asarray(want)
    if got.shape != want.shape:
        return False
    if got.dtype.kind == "f" or want.dtype.kind == "f":
        both_inf = np.isinf(got) & np.isinf(want) & (np.sign(got) == np.sign(want))
        ok = both_inf | np.isclose(got, want, rtol=rtol, atol=0.0)
        return bool(ok.all())
    return bool(np.array_equal(got, want))
