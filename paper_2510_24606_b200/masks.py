"""Drop-in for ``dhsa.masks``: token-level sparsity masks from chunk scores,
for prefill and decode, computed by the selection kernels of libdhsa_b200.

Reference: masks.py (CostCounters :38-52, SparsityMask :55-84, upsample
:87-100, topk_row :103-122, mask_from_chunk_scores :125-140, prefill_mask
:143-150, decode rows :153-202, DecodeSession :205-237).  Selection runs as
the exact chunk walk (select.cu) and never materialises the L x L upsampled
matrix; selected indices are identical to the reference's (same tie-break,
same forced self, same budget).  Cost counters are updated with the
reference's counts.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .chunk_repr import centroids_dev, reps_dev, scores_dev
from .chunking import check_boundaries, extend_for_decode
from .core import TokenSequence

__all__ = ["CostCounters", "SparsityMask", "upsample", "topk_row", "mask_from_chunk_scores",
           "prefill_mask", "decode_mask_row", "DecodeSession"]

TILE = 64


@dataclass
class CostCounters:
    """Score evaluations and mask-admitted attention pairs (masks.py:38-52)."""

    score_ops: int = 0
    attended_pairs: int = 0

    def add_score_ops(self, n: int):
        self.score_ops += int(n)

    def add_attended(self, n: int):
        self.attended_pairs += int(n)

    def total(self) -> int:
        return self.score_ops + self.attended_pairs


@dataclass(frozen=True)
class SparsityMask:
    """Per-row allowed key positions; rows sorted, unique, causal, with self."""

    length: int
    rows: tuple

    def __post_init__(self):
        if self.length < 1 or len(self.rows) != self.length:
            raise ValueError("mask must have one row per token")
        checked = []
        for i, r in enumerate(self.rows):
            idx = np.asarray(r, dtype=np.intp)
            if idx.size == 0 or idx.min() < 0 or idx.max() > i:
                raise ValueError(f"mask row {i} is empty or not causal")
            if idx.size > 1 and np.any(idx[1:] <= idx[:-1]):
                raise ValueError(f"mask row {i} is not sorted and unique")
            if i not in idx:
                raise ValueError(f"mask row {i} does not include itself")
            checked.append(idx)
        object.__setattr__(self, "rows", tuple(checked))

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.length, self.length), dtype=bool)
        for i, idx in enumerate(self.rows):
            dense[i, idx] = True
        return dense

    def row_sizes(self) -> np.ndarray:
        return np.array([len(r) for r in self.rows], dtype=np.intp)


def upsample(chunk_scores, bounds) -> np.ndarray:
    """Token pair (i, j) gets the score of (chunk(i), chunk(j)) (masks.py:87-100)."""
    s = np.asarray(chunk_scores, dtype=np.float64)
    bs = check_boundaries(bounds)
    n = len(bs) - 1
    if s.shape != (n, n):
        raise ValueError(f"expected a {n}x{n} score matrix, got {s.shape}")
    L = bs[-1]
    out = _dev.empty((L, L))
    s_dev, b_dev = _dev.f64(s), _dev.i32(bs)  # keep alive until the launch is enqueued
    _lib.call("dhsa_upsample", _lib.ptr(s_dev), _lib.ptr(b_dev), n, L, _lib.ptr(out),
              _dev.stream())
    return _dev.host(out)


def _rows_select(scores_dev_t, sc_stride, bounds, rows, budget):
    """Run dhsa_rows_select for token rows ``rows``; returns index arrays."""
    import torch

    n = len(bounds) - 1
    L = bounds[-1]
    cap = _dev.tile_capacity(n, budget, L, TILE)
    tiles = _dev.empty((len(rows), cap, 2), dtype=torch.int32)
    ntiles = _dev.empty((len(rows),), dtype=torch.int32)
    # device temporaries must outlive the (asynchronous) launch: the caching
    # allocator would otherwise hand their memory to the next allocation
    b_dev, r_dev = _dev.i32(bounds), _dev.i32(rows)
    scratch = _dev.select_scratch(n, len(rows))
    _lib.call("dhsa_rows_select", _lib.ptr(scores_dev_t), int(sc_stride), _lib.ptr(b_dev), n,
              _lib.ptr(r_dev), len(rows), int(budget), TILE, _lib.ptr(tiles), cap,
              _lib.ptr(ntiles), _lib.ptr(scratch), _dev.stream())
    return _dev.tiles_to_rows(_dev.host(tiles), _dev.host(ntiles))


def topk_row(scores, row, budget) -> np.ndarray:
    """Causal top-k of one row with forced self and lower-index ties
    (masks.py:103-122)."""
    if budget < 1:
        raise ValueError("budget must be >= 1")
    s = np.asarray(scores, dtype=np.float64)
    if s.ndim != 1 or s.size < row + 1:
        raise ValueError("scores must cover positions 0..row")
    row = int(row)
    # every position is its own chunk; all rows share one score vector
    bounds = list(range(row + 2))
    return _rows_select(_dev.f64(s[: row + 1]), 0, bounds, [row], budget)[0]


def _mask_from_dev_scores(sc, bs, budget, counters):
    L = bs[-1]
    rows = _rows_select(sc, sc.shape[1], bs, list(range(L)), budget)
    mask = SparsityMask(length=L, rows=tuple(rows))
    if counters is not None:
        counters.add_attended(int(mask.row_sizes().sum()))
    return mask


def mask_from_chunk_scores(chunk_scores, bounds, budget,
                           counters: CostCounters | None = None) -> SparsityMask:
    """Full prefill mask from a chunk-level score matrix (masks.py:125-140)."""
    bs = check_boundaries(bounds)
    s = np.asarray(chunk_scores, dtype=np.float64)
    n = len(bs) - 1
    if s.shape != (n, n):
        raise ValueError(f"expected a {n}x{n} score matrix, got {s.shape}")
    if budget < 1:
        raise ValueError("budget must be >= 1")
    return _mask_from_dev_scores(_dev.f64(s), bs, budget, counters)


def prefill_mask(seq: TokenSequence, bounds, budget,
                 counters: CostCounters | None = None) -> SparsityMask:
    """Chunk, score and select the full mask (masks.py:143-150), device-resident."""
    qc, kc, bs = reps_dev(seq, bounds)
    sc = scores_dev(qc, kc)
    if counters is not None:
        counters.add_score_ops(sc.numel())
    if budget < 1:
        raise ValueError("budget must be >= 1")
    return _mask_from_dev_scores(sc, bs, budget, counters)


class _DecodeState:
    """One decode unit on the device: prompt centroid cache, fp64 running
    sum of generated keys and the generated-token count (masks.py:214-222)."""

    def __init__(self, cached_dev, prompt_bounds, gen_sum_dev, gen_count):
        import torch

        self.bounds = prompt_bounds
        self.n = len(prompt_bounds) - 1
        self.d = cached_dev.shape[1]
        self.cached = cached_dev
        self.gen_sum = gen_sum_dev
        self.gen_count = _dev.i32([gen_count])
        self.b = _dev.i32(prompt_bounds)
        self.plen = _dev.i32([prompt_bounds[-1]])
        self.nch = _dev.i32([self.n])
        self.scores = _dev.empty((1, self.n + 1))
        self.torch = torch

    def row(self, q, k_new, budget, update: bool, length: int):
        """Scores + selection for the newest token; optionally folds k_new
        into the running sum (masks.py:235) and advances the count."""
        torch = self.torch
        lay = _lib.layout(bounds=self.b, plen=self.plen, nchunks=self.nch, max_chunks=self.n)
        st = _dev.stream()
        _lib.call("dhsa_decode_score", _lib.F64, _lib.ptr(q), _lib.ptr(self.cached), self.n * self.d,
                  _lib.ptr(self.gen_sum), _lib.ptr(self.gen_count),
                  _lib.ptr(k_new) if update else 0, 0, 0, 0, 0, lay, 1, 1, self.d,
                  _lib.AGG["none"], _lib.ptr(self.scores), self.n + 1, st)
        cap = _dev.tile_capacity(self.n + 1, budget, length, TILE)
        tiles = _dev.empty((1, cap, 2), dtype=torch.int32)
        ntiles = _dev.empty((1,), dtype=torch.int32)
        scratch = _dev.select_scratch(self.n + 1, 1)
        _lib.call("dhsa_decode_select", _lib.ptr(self.scores), self.n + 1, lay,
                  _lib.ptr(self.gen_count), 1, 1, int(budget), TILE, _lib.ptr(tiles), cap,
                  _lib.ptr(ntiles), _lib.ptr(scratch), st)
        if update:
            _lib.call("dhsa_decode_advance", _lib.ptr(self.gen_count), 1, st)
        return _dev.tiles_to_rows(_dev.host(tiles), _dev.host(ntiles))[0]


def _count_decode(counters, n_prompt, gen_count, row):
    if counters is not None:
        counters.add_score_ops(n_prompt + (1 if gen_count >= 1 else 0) + 1)
        counters.add_attended(len(row))


def decode_mask_row(prompt_bounds, cached_chunk_keys, generated_keys, current_query,
                    total_length, budget, counters: CostCounters | None = None) -> np.ndarray:
    """Mask row of the newest token from cached prompt chunks (masks.py:176-202)."""
    bs = check_boundaries(prompt_bounds)
    gen = np.asarray(generated_keys, dtype=np.float64)
    if gen.ndim != 2 or gen.shape[0] < 1:
        raise ValueError("generated_keys must hold at least the current key")
    if bs[-1] + gen.shape[0] != total_length:
        raise ValueError(
            f"prompt length {bs[-1]} + {gen.shape[0]} generated keys "
            f"!= total_length {total_length}")
    extend_for_decode(bs, total_length)  # same validation as the reference
    g = gen.shape[0] - 1
    cached = _dev.f64(cached_chunk_keys)
    if cached.dim() != 2 or cached.shape[0] != len(bs) - 1:
        raise ValueError("cached_chunk_keys must be [num_chunks, dim]")
    gdev = _dev.f64(gen)
    if g >= 1:
        gen_sum = centroids_dev(gdev[:g].contiguous(), [0, g], normalize=False)[0, 0].contiguous()
    else:
        gen_sum = _dev.zeros((gen.shape[1],))
    if budget < 1:
        raise ValueError("budget must be >= 1")
    state = _DecodeState(cached, bs, gen_sum, g)
    q = _dev.f64(np.asarray(current_query, dtype=np.float64).reshape(1, -1))
    row = state.row(q, None, budget, update=False, length=total_length)
    _count_decode(counters, len(bs) - 1, g, row)
    return row


class DecodeSession:
    """Stateful decoding with a device-resident centroid cache and an O(1)
    running sum of generated keys (masks.py:205-237)."""

    def __init__(self, prompt_keys, prompt_bounds, budget,
                 counters: CostCounters | None = None):
        keys = np.asarray(prompt_keys, dtype=np.float64)
        self.prompt_bounds = check_boundaries(prompt_bounds, keys.shape[0])
        self.budget = int(budget)
        self.counters = counters
        cached = centroids_dev(_dev.f64(keys), self.prompt_bounds)[0]
        self._state = _DecodeState(cached, self.prompt_bounds, _dev.zeros((keys.shape[1],)), 0)
        self._gen_count = 0
        self._cached_host = None

    @property
    def cached_chunk_keys(self) -> np.ndarray:
        if self._cached_host is None:
            self._cached_host = _dev.host(self._state.cached)
        return self._cached_host

    @property
    def total_length(self) -> int:
        return self.prompt_bounds[-1] + self._gen_count

    def step(self, query, key) -> np.ndarray:
        """Admit one generated token; return its mask row (masks.py:228-237)."""
        if self.budget < 1:
            raise ValueError("budget must be >= 1")
        q = _dev.f64(np.asarray(query, dtype=np.float64).reshape(1, -1))
        k = _dev.f64(np.asarray(key, dtype=np.float64).reshape(1, -1))
        row = self._state.row(q, k, self.budget, update=True, length=self.total_length + 1)
        _count_decode(self.counters, len(self.prompt_bounds) - 1, self._gen_count, row)
        self._gen_count += 1
        return row
