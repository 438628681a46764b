"""Digest helpers shared by the tests (same convention as tests/golden/make_goldens.py)."""

import hashlib

import numpy as np


def digest(edges, weights) -> str:
    e = np.ascontiguousarray(edges, dtype="<i8")
    w = np.ascontiguousarray(weights, dtype="<f8")
    return hashlib.sha256(e.tobytes() + w.tobytes()).hexdigest()[:16]


def array_digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
