"""Loaders for the golden vectors written by tests/golden/make_golden.py."""

import json
import os
from functools import lru_cache

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(None)
def npz(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


@lru_cache(None)
def meta():
    with open(os.path.join(GOLDEN, "meta.json")) as fh:
        return json.load(fh)


@lru_cache(None)
def pack_cases():
    with open(os.path.join(GOLDEN, "pack.json")) as fh:
        return json.load(fh)


def group(d, name):
    pre = name + "/"
    return {k[len(pre):]: v for k, v in d.items() if k.startswith(pre)}


def canon(d):
    d = np.array(d, dtype=np.float64, copy=True)
    d[d == 0] = 0.0
    return d


def same_bits(a, b):
    a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))
