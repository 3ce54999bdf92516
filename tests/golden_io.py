"""Loaders for the golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name))


def unpack_bits(packed, ncols):
    return np.unpackbits(packed, axis=1)[:, :ncols].astype(bool)


def hsa_cases(kind):
    """Yield (meta, arrays) for 'aligned' or 'framewise' fixtures."""
    meta = load_json(f"hsa_{kind}.json")
    arr = load_npz(f"hsa_{kind}.npz")
    for m in meta:
        yield m, arr


def case_inputs(m):
    from oracle.lf_oracle import synthetic_qkv
    f, n, i, d = m["f"], m["n"], m["i"], m["d"]
    q, k, v = synthetic_qkv(m["seed"], f * n, i * f * n, d, bf16=not m.get("fp32_inputs", False))
    return q[0], k[0], v[0]
