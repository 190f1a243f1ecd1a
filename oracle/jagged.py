"""Numpy restatement of the reference sequence chunking (TEST ORACLE).

Follows ``/root/reference/pkg/src/jaggedcp/jagged.py``:

* ``split_even``            -> jagged.py:143-146 (remainder to earliest parts)
* ``make_minichunks``       -> jagged.py:149-166 (2*cp chunks per sequence)
* ``make_contiguous_chunks``-> jagged.py:169-173 (naive cp chunks)
* ``chunk_assignment``      -> jagged.py:176-184 (rank i owns i, 2cp-1-i)
* ``chunk_owner_map``       -> jagged.py:187-198
* ``rank_major_row_order``  -> jagged.py:201-218 (rank -> seq -> chunk asc)
* ``rank_row_ranges``       -> jagged.py:221-229

Layouts are returned as plain ``(cp_size, chunks_per_seq, lengths[B][C],
ranges[B][C])`` tuples of python ints.
"""

from __future__ import annotations

import numpy as np


def split_even(length: int, parts: int) -> list[int]:
    base, rem = divmod(int(length), parts)
    return [base + 1 if p < rem else base for p in range(parts)]


def _layout(seq_lengths, cp_size: int, parts: int):
    lens, ranges = [], []
    for L in seq_lengths:
        if L < 0:
            raise ValueError("sequence lengths must be non-negative")
        sizes = split_even(int(L), parts)
        bounds = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        lens.append(tuple(sizes))
        ranges.append(tuple((int(bounds[c]), int(bounds[c + 1])) for c in range(parts)))
    return (cp_size, parts, tuple(lens), tuple(ranges))


def make_minichunks(seq_lengths, cp_size: int):
    if cp_size < 1:
        raise ValueError("cp_size must be >= 1")
    return _layout(seq_lengths, cp_size, 2 * cp_size)


def make_contiguous_chunks(seq_lengths, cp_size: int):
    if cp_size < 1:
        raise ValueError("cp_size must be >= 1")
    return _layout(seq_lengths, cp_size, cp_size)


def chunk_assignment(cp_size: int) -> dict[int, tuple[int, int]]:
    if cp_size < 1:
        raise ValueError("cp_size must be >= 1")
    return {r: (r, 2 * cp_size - 1 - r) for r in range(cp_size)}


def chunk_owner_map(layout) -> tuple[int, ...]:
    cp, n = layout[0], layout[1]
    if n == 2 * cp:
        owners = [0] * n
        for rank, (a, b) in chunk_assignment(cp).items():
            owners[a] = rank
            owners[b] = rank
        return tuple(owners)
    if n == cp:
        return tuple(range(n))
    raise ValueError(f"layout has {n} chunks per sequence for cp_size {cp}")


def rank_major_row_order(offsets, layout) -> tuple[np.ndarray, list[int]]:
    cp, n, _, ranges = layout
    owners = chunk_owner_map(layout)
    parts, slab = [], [0] * cp
    for rank in range(cp):
        for b in range(len(ranges)):
            base = int(offsets[b])
            for c in range(n):
                if owners[c] != rank:
                    continue
                s, e = ranges[b][c]
                parts.append(np.arange(base + s, base + e, dtype=np.int64))
                slab[rank] += e - s
    perm = np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)
    return perm, slab


def rank_row_ranges(layout) -> list[tuple[int, int]]:
    cp, n, lens, _ = layout
    owners = chunk_owner_map(layout)
    sizes = [0] * cp
    for b in range(len(lens)):
        for c in range(n):
            sizes[owners[c]] += lens[b][c]
    bounds = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return [(int(bounds[r]), int(bounds[r + 1])) for r in range(cp)]
