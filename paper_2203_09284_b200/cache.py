"""FPRG binary graph cache, byte-compatible with the reference's
graph_cache.hpp (:21-97): magic "FPRG", u32 version 1, then n, m and the three
CSR arrays (in_start[n+1], in_src[m], out_degree[n]) as little-endian u64.
Hands device-built graphs (fpr_b200_graph_download_csr) to CPU tools and the
reference, and caches generated graphs between runs."""
from __future__ import annotations

import os

import numpy as np

from . import Graph

MAGIC = b"FPRG"
VERSION = 1


class CacheError(RuntimeError):
    """graph_cache.hpp:15-17 CacheError (a std::runtime_error)."""


def save_cache(g: Graph, path: str) -> None:
    """save_cache (graph_cache.hpp:65-76)."""
    try:
        f = open(path, "wb")
    except OSError:
        raise CacheError(f"graph cache: cannot open '{path}' for writing")
    with f:
        try:
            f.write(MAGIC)
            f.write(np.uint32(VERSION).astype("<u4").tobytes())
            f.write(np.array([g.n, g.m], dtype="<u8").tobytes())
            for a in (g.in_start, g.in_src, g.out_degree):
                np.ascontiguousarray(a, dtype="<u8").tofile(f)
        except OSError:
            raise CacheError(f"graph cache: write to '{path}' failed")


def load_cache(path: str) -> Graph:
    """load_cache (graph_cache.hpp:78-97)."""
    try:
        f = open(path, "rb")
    except OSError:
        raise CacheError(f"graph cache: cannot open '{path}'")
    with f:
        magic = f.read(4)
        if len(magic) < 4:
            raise CacheError("graph cache: truncated file")
        if magic != MAGIC:
            raise CacheError("graph cache: bad magic bytes")
        v = f.read(4)
        if len(v) < 4:
            raise CacheError("graph cache: truncated file")
        version = int(np.frombuffer(v, "<u4")[0])
        if version != VERSION:
            raise CacheError(f"graph cache: unsupported format version {version}")
        hdr = f.read(16)
        if len(hdr) < 16:
            raise CacheError("graph cache: truncated file")
        n, m = (int(x) for x in np.frombuffer(hdr, "<u8"))
        arrays = []
        for count in (n + 1, m, n):
            a = np.fromfile(f, dtype="<u8", count=count)
            if len(a) != count:
                raise CacheError("graph cache: truncated file")
            arrays.append(a.astype(np.uint64))
    return Graph(n, m, *arrays)
