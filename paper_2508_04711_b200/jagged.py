"""Jagged containers and sequence chunking on the GPU.

Mirror of ``jaggedcp/jagged.py`` (/root/reference/pkg/src/jaggedcp/jagged.py)
with the same names, argument meaning and errors:

* values live on the GPU (bf16 by default); offsets are kept both as a device
  int64 tensor (for kernels) and as a host numpy copy (for plans / Python-side
  validation, the reference's own representation);
* the integer plan (split_even / make_minichunks / chunk_assignment /
  rank-major order) is computed by the C ABI (``jh_plan_build``,
  ``jh_rank_major_perm``), bit-exact with jagged.py:143-258;
* row permutations run as the vectorised gather/scatter kernel
  (``jh_gather_rows`` / ``jh_scatter_rows``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib, kernels
from ._lib import check

DEFAULT_DTYPE = torch.bfloat16


def _device(device=None) -> torch.device:
    d = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if d.type != "cuda":
        raise ValueError("jagged tensors live on a CUDA device (there is no CPU path)")
    return d


def _check_offsets(offsets: np.ndarray, total_rows: int) -> None:
    """jagged.py:27-37 (same messages)."""
    if offsets.ndim != 1 or offsets.size < 1:
        raise ValueError("offsets must be a 1-D array with at least one entry")
    if offsets[0] != 0:
        raise ValueError("offsets must start at 0")
    if np.any(np.diff(offsets) < 0):
        raise ValueError("offsets not monotone")
    if offsets[-1] != total_rows:
        raise ValueError(f"offsets end at {int(offsets[-1])} but values have {total_rows} rows")


def _host_offsets(offsets) -> np.ndarray:
    if isinstance(offsets, torch.Tensor):
        return offsets.detach().cpu().numpy().astype(np.int64)
    return np.array(offsets, dtype=np.int64)


@dataclass(frozen=True)
class JaggedTensor:
    """jagged.py:40-61: flat values (T, D) + offsets (B+1,)."""

    values: torch.Tensor
    offsets: torch.Tensor  # int64, device
    max_length: int
    host_offsets: np.ndarray  # int64, host copy

    @property
    def num_sequences(self) -> int:
        return len(self.host_offsets) - 1

    @property
    def total_tokens(self) -> int:
        return self.values.shape[0]

    @property
    def embed_dim(self) -> int:
        return self.values.shape[1]

    def sequence(self, b: int) -> torch.Tensor:
        return self.values[int(self.host_offsets[b]): int(self.host_offsets[b + 1])]


@dataclass(frozen=True)
class JaggedIntSeries:
    """jagged.py:64-80: one int64 per token (timestamps)."""

    values: torch.Tensor
    offsets: torch.Tensor
    host_offsets: np.ndarray

    @property
    def num_sequences(self) -> int:
        return len(self.host_offsets) - 1

    @property
    def total_tokens(self) -> int:
        return self.values.shape[0]

    def sequence(self, b: int) -> torch.Tensor:
        return self.values[int(self.host_offsets[b]): int(self.host_offsets[b + 1])]


def new_jagged(values, offsets, max_length: int, device=None, dtype=DEFAULT_DTYPE, copy: bool = True) -> JaggedTensor:
    """jagged.py:83-105: validate and build.  The container owns its storage:
    values are copied (to the device / dtype) unless ``copy=False`` and they
    already are a contiguous device tensor of ``dtype`` (then adopted)."""
    dev = _device(device if device is not None else (values.device if isinstance(values, torch.Tensor)
                                                      and values.is_cuda else None))
    if isinstance(values, torch.Tensor):
        vals = values
    else:
        arr = np.asarray(values)
        vals = torch.from_numpy(np.ascontiguousarray(arr.astype(np.float32) if arr.dtype != np.float32 else arr))
    if vals.dim() != 2:
        raise ValueError(f"values must be 2-D (total_tokens x embed_dim), got ndim={vals.dim()}")
    offs = _host_offsets(offsets)
    _check_offsets(offs, vals.shape[0])
    if max_length < 0:
        raise ValueError("max_length must be non-negative")
    seq_lengths = np.diff(offs)
    if seq_lengths.size and int(seq_lengths.max()) > max_length:
        raise ValueError(f"sequence length {int(seq_lengths.max())} exceeds max_length {max_length}")
    v = vals.to(device=dev, dtype=dtype, non_blocking=True).contiguous()
    if copy and v.data_ptr() == getattr(values, "data_ptr", lambda: None)():
        v = v.clone()  # the container owns its storage (jagged.py:95)
    o = _h2d(offs, dev)
    return JaggedTensor(v, o, int(max_length), offs)


def _h2d(a: np.ndarray, dev) -> torch.Tensor:
    """Host int64 array -> device without stalling the host (a pageable
    host->device copy first waits for the stream to drain)."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    if torch.device(dev).type == "cuda":
        t = t.pin_memory()
    return t.to(dev, non_blocking=True)


def new_int_series(values, offsets, device=None) -> JaggedIntSeries:
    """jagged.py:108-114."""
    dev = _device(device if device is not None else (values.device if isinstance(values, torch.Tensor)
                                                      and values.is_cuda else None))
    vals = values if isinstance(values, torch.Tensor) else torch.from_numpy(np.array(values, dtype=np.int64))
    if vals.dim() != 1:
        raise ValueError("int series values must be 1-D (one integer per token)")
    offs = _host_offsets(offsets)
    _check_offsets(offs, vals.shape[0])
    v = vals.to(device=dev, dtype=torch.int64, non_blocking=True).contiguous()
    return JaggedIntSeries(v, _h2d(offs, dev), offs)


def lengths(jt) -> np.ndarray:
    """jagged.py:117-119."""
    return np.diff(jt.host_offsets)


@dataclass(frozen=True)
class MiniChunkLayout:
    """jagged.py:122-140."""

    cp_size: int
    chunks_per_seq: int
    chunk_lengths: tuple
    chunk_ranges: tuple

    @property
    def num_sequences(self) -> int:
        return len(self.chunk_lengths)

    def seq_lengths(self) -> tuple:
        return tuple(sum(c) for c in self.chunk_lengths)


def _plan_arrays(seq_lengths: Sequence[int], cp_size: int, mode: int):
    """Exact integer plan through jh_plan_build (cp_engine.py:105-147)."""
    if cp_size < 1:
        raise ValueError("cp_size must be >= 1")
    lens = np.ascontiguousarray(np.asarray(list(seq_lengths), dtype=np.int64))
    if lens.size and lens.min() < 0:
        raise ValueError("sequence lengths must be non-negative")
    n = lens.size
    C = 2 * cp_size if mode == 0 else cp_size
    cl = np.zeros(max(n * C, 1), dtype=np.int64)
    cs = np.zeros(max(n * C, 1), dtype=np.int64)
    co = np.zeros(C, dtype=np.int32)
    P64 = ctypes.POINTER(ctypes.c_int64)
    check(_lib.lib().jh_plan_build(lens.ctypes.data_as(P64) if n else None, n, cp_size, mode,
                                   cl.ctypes.data_as(P64), cs.ctypes.data_as(P64),
                                   co.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))), "plan")
    return cl[: n * C].reshape(n, C), cs[: n * C].reshape(n, C), co


def _layout(seq_lengths, cp_size: int, mode: int) -> MiniChunkLayout:
    cl, cs, _ = _plan_arrays(seq_lengths, cp_size, mode)
    C = cl.shape[1] if cl.ndim == 2 and cl.size else (2 * cp_size if mode == 0 else cp_size)
    lens = tuple(tuple(int(x) for x in row) for row in cl)
    ranges = tuple(tuple((int(cs[b, c]), int(cs[b, c] + cl[b, c])) for c in range(C)) for b in range(len(lens)))
    return MiniChunkLayout(cp_size, C, lens, ranges)


def split_even(length: int, parts: int) -> list[int]:
    """jagged.py:143-146."""
    base, rem = divmod(int(length), parts)
    return [base + 1 if p < rem else base for p in range(parts)]


def make_minichunks(seq_lengths, cp_size: int) -> MiniChunkLayout:
    """jagged.py:162-166: 2*cp near-even chunks per sequence."""
    return _layout(seq_lengths, cp_size, 0)


def make_contiguous_chunks(seq_lengths, cp_size: int) -> MiniChunkLayout:
    """jagged.py:169-173: naive cp chunks per sequence."""
    return _layout(seq_lengths, cp_size, 1)


def chunk_assignment(cp_size: int) -> dict[int, tuple[int, int]]:
    """jagged.py:176-184: rank i owns mini-chunks i and 2cp-1-i."""
    if cp_size < 1:
        raise ValueError("cp_size must be >= 1")
    return {r: (r, 2 * cp_size - 1 - r) for r in range(cp_size)}


def chunk_owner_map(layout: MiniChunkLayout) -> tuple[int, ...]:
    """jagged.py:187-198."""
    n = layout.chunks_per_seq
    if n == 2 * layout.cp_size:
        return tuple(int(x) for x in _plan_arrays([], layout.cp_size, 0)[2])
    if n == layout.cp_size:
        return tuple(range(n))
    raise ValueError(f"layout has {n} chunks per sequence for cp_size {layout.cp_size}")


def _mode_of(layout: MiniChunkLayout) -> int:
    if layout.chunks_per_seq == 2 * layout.cp_size:
        return 0
    if layout.chunks_per_seq == layout.cp_size:
        return 1
    raise ValueError(f"layout has {layout.chunks_per_seq} chunks per sequence for cp_size {layout.cp_size}")


def rank_major_perm(host_offsets: np.ndarray, cp_size: int, mode: int) -> tuple[np.ndarray, np.ndarray]:
    """jagged.py:201-218 through jh_rank_major_perm: (perm[T], slab_rows[cp])."""
    offs = np.ascontiguousarray(np.asarray(host_offsets, dtype=np.int64))
    T = int(offs[-1]) if offs.size else 0
    perm = np.zeros(max(T, 1), dtype=np.int64)
    slab = np.zeros(cp_size, dtype=np.int64)
    P64 = ctypes.POINTER(ctypes.c_int64)
    check(_lib.lib().jh_rank_major_perm(offs.ctypes.data_as(P64), offs.size - 1, cp_size, mode,
                                        perm.ctypes.data_as(P64), slab.ctypes.data_as(P64)), "rank_major_perm")
    return perm[:T], slab


def rank_row_ranges(layout: MiniChunkLayout) -> list[tuple[int, int]]:
    """jagged.py:221-229."""
    owners = chunk_owner_map(layout)
    sizes = [0] * layout.cp_size
    for b in range(layout.num_sequences):
        for c in range(layout.chunks_per_seq):
            sizes[owners[c]] += layout.chunk_lengths[b][c]
    bounds = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return [(int(bounds[r]), int(bounds[r + 1])) for r in range(layout.cp_size)]


def reorder_balanced(jt: JaggedTensor, layout: MiniChunkLayout):
    """jagged.py:232-245: rows to rank-major order on the GPU.

    Returns (reordered JaggedTensor, perm) with ``reordered.values[i] ==
    jt.values[perm[i]]``; perm is a device int64 tensor."""
    if layout.num_sequences != jt.num_sequences:
        raise ValueError("layout does not match the tensor's sequence count")
    if tuple(int(x) for x in lengths(jt)) != layout.seq_lengths():
        raise ValueError("layout chunk lengths do not sum to the tensor's sequence lengths")
    perm_h, _ = rank_major_perm(jt.host_offsets, layout.cp_size, _mode_of(layout))
    perm = _h2d(perm_h, jt.values.device)
    vals = kernels.gather_rows(jt.values, perm)
    return JaggedTensor(vals, jt.offsets, jt.max_length, jt.host_offsets), perm


def inverse_reorder(jt: JaggedTensor, permutation) -> JaggedTensor:
    """jagged.py:248-258: undo a reorder_balanced permutation (GPU scatter)."""
    perm = permutation if isinstance(permutation, torch.Tensor) else torch.from_numpy(
        np.asarray(permutation, dtype=np.int64))
    perm = perm.to(device=jt.values.device, dtype=torch.int64)
    n = jt.total_tokens
    if tuple(perm.shape) != (n,):
        raise ValueError(f"permutation has {perm.numel()} entries for {n} rows")
    if n and (int(perm.min()) < 0 or int(perm.max()) >= n or int(torch.bincount(perm, minlength=n).max()) > 1):
        raise ValueError("permutation is not a bijection on row indices")
    vals = kernels.scatter_rows(jt.values, perm)
    return JaggedTensor(vals, jt.offsets, jt.max_length, jt.host_offsets)


def jagged_to_padded(jt: JaggedTensor, max_len: int | None = None) -> torch.Tensor:
    """(new) [B, max_len, D] zero-padded copy of a jagged tensor."""
    ml = jt.max_length if max_len is None else int(max_len)
    return kernels.jagged_to_padded(jt.values, jt.offsets, ml)


def padded_to_jagged(padded: torch.Tensor, offsets, max_length: int | None = None) -> JaggedTensor:
    """(new) inverse of jagged_to_padded."""
    offs = _host_offsets(offsets)
    dev = padded.device
    o = _h2d(offs, dev)
    vals = kernels.padded_to_jagged(padded, o, int(offs[-1]))
    return JaggedTensor(vals, o, int(padded.shape[1] if max_length is None else max_length), offs)
