"""Helpers to read tests/golden/*.json (reference-generated fixtures)."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str) -> dict:
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<" + a.dtype.str[1:]).tobytes()).hexdigest()


def unhex(xs) -> np.ndarray:
    return np.array([float.fromhex(x) for x in xs], dtype=np.float64)


def small_edges(rec: dict):
    e = np.array(rec["edges"], dtype=np.uint64).reshape(-1, 2)
    return rec["n"], e[:, 0].copy(), e[:, 1].copy()
