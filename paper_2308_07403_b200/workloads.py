"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference measures on no public dataset; every config is a seeded
random graph. The Erdos-Renyi pattern is drawn exactly as
the reference's ``gen_random_dense`` does (pkg/src/rdist/graphs.py:185-195:
``default_rng(seed).random((n, n)) < p`` with the diagonal cleared), so the
same seed gives the same graph on either side. The directed lattice (config
2) and the uniform-[1,5] weighted graph (config 4) have no reference
generator; they are defined here.

Unweighted graphs can be produced directly as bit-packed adjacency (row i,
bit j%32 of word j/32 set <=> edge j -> i), the device input format of
``rdb_build_m_bits``; config 5 (N = 32768) is only built that way, in row
chunks, without ever materialising the 8.6 GB float64 matrix.
"""

from __future__ import annotations

import numpy as np

from .graphs import Graph, GraphKind

CFG1 = dict(n=512, p=0.05, gamma=1e-3)
CFG2 = dict(n=1024, batch=256, er_p=0.02, er_gamma=1e-2, lattice_side=32, lattice_keep=0.8, lattice_gamma=0.1)
CFG3 = dict(n=8192, p=0.5, gamma=1e-5)
CFG4 = dict(n=4096, p=0.1, w_lo=1.0, w_hi=5.0, gamma=1e-3)
CFG5 = dict(n=32768, p=0.01, gamma=1e-4)


def er_present(n: int, p: float, seed: int) -> np.ndarray:
    """Boolean edge pattern present[i][j] (edge j -> i), diagonal cleared."""
    if n < 2:
        raise ValueError(f"n must be >= 2, got {n}")
    if not 0 < p <= 1:
        raise ValueError(f"p must be in (0, 1], got {p}")
    present = np.random.default_rng(seed).random((n, n)) < p
    np.fill_diagonal(present, False)
    return present


def weights_from_present(present: np.ndarray) -> np.ndarray:
    return np.where(present, 1.0, np.inf)


def er_graph(n: int, p: float, seed: int) -> Graph:
    return Graph(n, weights_from_present(er_present(n, p, seed)), GraphKind.UNWEIGHTED)


def lattice_present(side: int, keep: float, seed: int) -> np.ndarray:
    """Directed side x side grid: each of a vertex's up-to-4 arcs to its grid
    neighbours is kept independently with probability ``keep``.
    Vertex v = y * side + x."""
    n = side * side
    rng = np.random.default_rng(seed)
    draws = rng.random((4, side, side)) < keep  # arcs v -> right, left, down, up
    present = np.zeros((n, n), dtype=bool)
    ys, xs = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    src = ys * side + xs
    for d, (dy, dx) in enumerate(((0, 1), (0, -1), (1, 0), (-1, 0))):
        ty, tx = ys + dy, xs + dx
        ok = (ty >= 0) & (ty < side) & (tx >= 0) & (tx < side) & draws[d]
        dst = ty * side + tx
        present[dst[ok], src[ok]] = True
    return present


def lattice_graph(side: int, keep: float, seed: int) -> Graph:
    return Graph(side * side, weights_from_present(lattice_present(side, keep, seed)), GraphKind.UNWEIGHTED)


def weighted_er_graph(n: int, p: float, w_lo: float, w_hi: float, seed: int) -> Graph:
    """Config 4: ER pattern as gen_random_dense, then W ~ U[w_lo, w_hi] on present edges."""
    rng = np.random.default_rng(seed)
    present = rng.random((n, n)) < p
    np.fill_diagonal(present, False)
    w = rng.uniform(w_lo, w_hi, size=(n, n))
    return Graph(n, np.where(present, w, np.inf), GraphKind.REAL_WEIGHTED)


def pack_bits(present: np.ndarray) -> np.ndarray:
    """(..., n, n) bool -> (..., n, ceil(n/32)) uint32, bit j%32 of word j/32."""
    n = present.shape[-1]
    wpr = (n + 31) // 32
    pad = wpr * 32 - n
    if pad:
        widths = [(0, 0)] * (present.ndim - 1) + [(0, pad)]
        present = np.pad(present, widths)
    packed = np.packbits(present, axis=-1, bitorder="little")
    return np.ascontiguousarray(packed).view(np.uint32).reshape(present.shape[:-1] + (wpr,))


def unpack_bits(bits: np.ndarray, n: int) -> np.ndarray:
    b = np.ascontiguousarray(bits).view(np.uint8)
    return np.unpackbits(b, axis=-1, bitorder="little")[..., :n].astype(bool)


def cfg2_seeds(batch: int = 256, rank: int = 0) -> list[tuple[str, int]]:
    """(kind, seed) per graph: first half ER, second half lattices; ``rank``
    offsets the seeds so data-parallel ranks get distinct graphs."""
    half = batch // 2
    off = 100_000 * rank
    return [("er", 2000 + off + s) for s in range(half)] + [
        ("lattice", 1000 + off + s) for s in range(batch - half)
    ]


def cfg2_present(kind: str, seed: int) -> np.ndarray:
    if kind == "er":
        return er_present(CFG2["n"], CFG2["er_p"], seed)
    return lattice_present(CFG2["lattice_side"], CFG2["lattice_keep"], seed)


def cfg2_gamma(kind: str) -> float:
    return CFG2["er_gamma"] if kind == "er" else CFG2["lattice_gamma"]


def cfg2_batch(batch: int = 256, rank: int = 0) -> tuple[np.ndarray, np.ndarray, list[tuple[str, int]]]:
    """(bits (batch, n, n/32) uint32, gammas (batch,) float64, seeds)."""
    seeds = cfg2_seeds(batch, rank)
    n = CFG2["n"]
    bits = np.empty((batch, n, (n + 31) // 32), dtype=np.uint32)
    gammas = np.empty(batch, dtype=np.float64)
    for b, (kind, seed) in enumerate(seeds):
        bits[b] = pack_bits(cfg2_present(kind, seed))
        gammas[b] = cfg2_gamma(kind)
    return bits, gammas, seeds


def er_bits_chunked(n: int, p: float, seed: int, chunk_rows: int = 1024) -> np.ndarray:
    """Bit-packed gen_random_dense(n, p, seed) pattern, drawn in row chunks
    from the same RNG stream (equal to one (n, n) draw)."""
    rng = np.random.default_rng(seed)
    wpr = (n + 31) // 32
    out = np.empty((n, wpr), dtype=np.uint32)
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        blk = rng.random((r1 - r0, n)) < p
        idx = np.arange(r0, r1)
        blk[idx - r0, idx] = False
        out[r0:r1] = pack_bits(blk)
    return out


def er_bits_rows(n: int, p: float, seed: int, rows) -> np.ndarray:
    """Bit-packed rows ``rows`` (ascending global indices) of the
    gen_random_dense(n, p, seed) pattern without drawing the others: the
    pattern is one row-major ``random((n, n))`` draw from PCG64(seed), one
    64-bit output per double, so row i starts after i * n outputs and
    ``PCG64.advance`` jumps there. A rank of the 2D block-cyclic grid builds
    only its own row blocks this way (config 5)."""
    rows = np.asarray(rows, dtype=np.int64)
    wpr = (n + 31) // 32
    out = np.empty((rows.size, wpr), dtype=np.uint32)
    k = 0
    while k < rows.size:  # runs of consecutive rows share one jump
        e = k + 1
        while e < rows.size and rows[e] == rows[e - 1] + 1 and e - k < 2048:
            e += 1
        bg = np.random.PCG64(seed)
        bg.advance(int(rows[k]) * n)
        blk = np.random.Generator(bg).random((e - k, n)) < p
        blk[np.arange(e - k), rows[k:e]] = False
        out[k:e] = pack_bits(blk)
        k = e
    return out


def _rows_job(args):
    n, p, seed, r0, r1 = args
    return r0, er_bits_rows(n, p, seed, np.arange(r0, r1))


def er_bits_parallel(n: int, p: float, seed: int, procs: int | None = None, chunk_rows: int = 1024) -> np.ndarray:
    """er_bits_chunked(n, p, seed) drawn by ``procs`` forked workers, each
    jumping the generator to its row chunk (identical bits; config 5's 1.07e9
    draws take ~30 s on one core)."""
    import multiprocessing as mp
    import os

    procs = procs or os.cpu_count() or 1
    wpr = (n + 31) // 32
    out = np.empty((n, wpr), dtype=np.uint32)
    jobs = [(n, p, seed, r0, min(n, r0 + chunk_rows)) for r0 in range(0, n, chunk_rows)]
    if procs <= 1 or len(jobs) == 1:
        for j in jobs:
            r0, blk = _rows_job(j)
            out[r0 : r0 + blk.shape[0]] = blk
        return out
    with mp.get_context("fork").Pool(min(procs, len(jobs))) as pool:
        for r0, blk in pool.imap_unordered(_rows_job, jobs):
            out[r0 : r0 + blk.shape[0]] = blk
    return out
