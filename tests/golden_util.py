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


# ---------------------------------------------------------------- edge lists
_M64 = (1 << 64) - 1


class SplitMix64:
    """SplitMix64 (rng.hpp:11-29) for deterministic text generation."""

    def __init__(self, seed: int):
        self.s = seed & _M64

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & _M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)


def roundtrip_texts(trials: int = 25) -> list[bytes]:
    """Inputs shaped like io_ingest_test.cpp:75-93 (RenderRoundTrip): 1..40
    lines of "a<TAB>b" with ids < 50 from SplitMix64(3)."""
    rng = SplitMix64(3)
    out = []
    for _ in range(trials):
        lines = 1 + rng.next() % 40
        out.append(b"".join(b"%d\t%d\n" % (rng.next() % 50, rng.next() % 50) for _ in range(lines)))
    return out


def render_edge_list(edges: np.ndarray, header=()) -> bytes:
    """fpr::write_edge_list (edge_list.hpp:84-89): '# ' header lines, then "src dst"."""
    head = b"".join(b"# " + h.encode() + b"\n" for h in header)
    return head + b"".join(b"%d %d\n" % (int(s), int(d)) for s, d in edges)


_WS = [b" ", b"\t", b"\r", b"  ", b" \t "]


def fuzz_text(seed: int, lines: int, bad_rate: float = 0.0) -> bytes:
    """Deterministic SNAP-style text: sparse ids, mixed separators, comment /
    blank / whitespace-only lines, CRLF endings, optional malformed lines."""
    rng = np.random.default_rng(seed)
    parts = []
    for k in range(lines):
        r = rng.random()
        if r < 0.05:
            parts.append(b"# comment " + str(k).encode())
        elif r < 0.07:
            parts.append(b"%" + b" header")
        elif r < 0.09:
            parts.append(b"")
        elif r < 0.10:
            parts.append(_WS[rng.integers(len(_WS))])
        elif r < 0.10 + bad_rate:
            parts.append([b"1 x", b"7", b"1 2 3", b"-4 5", b"18446744073709551616 1", b"\x0b3 4",
                          b"2 3#", b"  # indented"][rng.integers(8)])
        else:
            a, b = (int(x) for x in rng.integers(0, 1 << int(rng.integers(4, 64)), size=2, dtype=np.uint64))
            if rng.random() < 0.05:
                a = b  # self-loop
            lead = _WS[rng.integers(len(_WS))] if rng.random() < 0.2 else b""
            tail = _WS[rng.integers(len(_WS))] if rng.random() < 0.2 else b""
            zeros = b"0" * int(rng.integers(0, 3)) if rng.random() < 0.1 else b""
            parts.append(lead + zeros + str(a).encode() + _WS[rng.integers(len(_WS))] + str(b).encode() + tail)
        if rng.random() < 0.1:
            parts[-1] += b"\r"
    text = b"\n".join(parts)
    return text if rng.random() < 0.5 else text + b"\n"


def sparse_text_from_edges(src: np.ndarray, dst: np.ndarray, mult: int = 2654435761, add: int = 12345,
                           comment_every: int = 1000) -> bytes:
    """A large deterministic text: ids remapped sparsely (raw = id*mult + add),
    with a comment line every `comment_every` edges."""
    rs = (src.astype(np.uint64) * np.uint64(mult) + np.uint64(add)).astype(np.uint64)
    rd = (dst.astype(np.uint64) * np.uint64(mult) + np.uint64(add)).astype(np.uint64)
    lines = np.char.add(np.char.add(rs.astype(str), " "), rd.astype(str))
    chunks = []
    for i in range(0, len(lines), comment_every):
        chunks.append("# block %d" % (i // comment_every))
        chunks.extend(lines[i:i + comment_every].tolist())
    return ("\n".join(chunks) + "\n").encode()
