"""Drop-in for ``dhsa.core`` on the hot path: ``TokenSequence`` and the exact
(masked) causal attention ``dense_attention``.

Reference: core.py:35-66 (TokenSequence), core.py:69-77 (softmax_row),
core.py:80-119 (_mask_rows, dense_attention), core.py:122-152
(causal_attention_probs, cosine_similarity).  The attention runs on the GPU through ``dhsa_attn`` in
fp64 (DFMA, online softmax), so outputs agree with the float64 reference to
~1e-15; masks are validated on the host with the reference's error messages.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib

__all__ = ["TokenSequence", "softmax_row", "dense_attention", "causal_attention_probs",
           "cosine_similarity"]


def _matrix(x, name):
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {a.shape}")
    if not np.isfinite(a).all():
        raise ValueError(f"{name} contains non-finite values")
    return a


@dataclass(frozen=True)
class TokenSequence:
    """Per-token queries, keys and values of one head, float64 [length, dim]."""

    queries: np.ndarray
    keys: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        q = _matrix(self.queries, "queries")
        k = _matrix(self.keys, "keys")
        v = _matrix(self.values, "values")
        if not (q.shape == k.shape == v.shape):
            raise ValueError(
                f"queries/keys/values shapes differ: {q.shape}, {k.shape}, {v.shape}")
        if q.shape[0] < 1:
            raise ValueError("sequence must contain at least one token")
        object.__setattr__(self, "queries", q)
        object.__setattr__(self, "keys", k)
        object.__setattr__(self, "values", v)

    @property
    def length(self) -> int:
        return self.queries.shape[0]

    @property
    def dim(self) -> int:
        return self.queries.shape[1]


def softmax_row(scores) -> np.ndarray:
    """Numerically stable softmax of a 1-D score vector (core.py:69-77),
    computed in fp64 on the device (dhsa_softmax_rows)."""
    s = np.asarray(scores, dtype=np.float64)
    if s.ndim != 1 or s.size == 0:
        raise ValueError("softmax_row expects a non-empty 1-D array")
    if not np.all(np.isfinite(s)):
        raise ValueError("softmax_row: non-finite scores")
    x = _dev.f64(s)
    out = _dev.empty((s.size,))
    _lib.call("dhsa_softmax_rows", _lib.ptr(x), 1, s.size, _lib.ptr(out), _dev.stream())
    return _dev.host(out)


def _validated_rows(mask, length):
    """Per-row sorted unique index arrays, validated like core.py:80-95."""
    rows = mask.rows if hasattr(mask, "rows") else mask
    if len(rows) != length:
        raise ValueError(f"mask has {len(rows)} rows, sequence has {length}")
    out = []
    for i, r in enumerate(rows):
        idx = np.asarray(r, dtype=np.intp)
        if idx.size == 0:
            raise ValueError(f"mask row {i} is empty")
        if idx.min() < 0 or idx.max() > i:
            raise ValueError(f"mask row {i} is not causal")
        if i not in idx:
            raise ValueError(f"mask row {i} does not include itself")
        out.append(np.unique(idx))
    return out


def rows_to_tiles(rows, tile=64):
    """Index rows -> (start, count) tiles of consecutive indices, <= tile each."""
    per_row = []
    for idx in rows:
        idx = np.asarray(idx, dtype=np.int64)
        brk = np.flatnonzero(np.diff(idx) != 1) + 1
        starts = idx[np.r_[0, brk]]
        ends = idx[np.r_[brk - 1, len(idx) - 1]] + 1
        t = []
        for s, e in zip(starts.tolist(), ends.tolist()):
            for a in range(s, e, tile):
                t.append((a, min(tile, e - a)))
        per_row.append(t)
    cap = max(len(t) for t in per_row)
    tiles = np.zeros((len(rows), cap, 2), dtype=np.int32)
    ntiles = np.zeros(len(rows), dtype=np.int32)
    for r, t in enumerate(per_row):
        tiles[r, : len(t)] = t
        ntiles[r] = len(t)
    return tiles, ntiles


def attend_tiles(q, k, v, tiles, ntiles, splits=1):
    """fp64 attention of each row of q over its tiles (device tensors)."""
    L, d = q.shape
    out = _dev.empty((L, d))
    cap = tiles.shape[1]
    ws = cnt = None
    if splits > 1:
        nbytes = _lib.load().dhsa_attn_workspace_size(_lib.F64, L, 1, d, splits)
        ws = _dev.empty((max(1, nbytes // 8),))
        import torch

        cnt = _dev.zeros((L,), dtype=torch.int32)
    _lib.call("dhsa_attn", _lib.F64, _lib.ptr(q), _lib.ptr(k), _lib.ptr(v), L * d, L, L, L, 1, d,
              _lib.ptr(tiles), cap, _lib.ptr(ntiles), splits, _lib.ptr(out), _lib.ptr(ws),
              _lib.ptr(cnt), 0, _dev.stream())
    return out


def dense_attention(seq: TokenSequence, mask=None) -> np.ndarray:
    """Causal softmax(q k / sqrt(d)) v, optionally restricted to ``mask`` rows
    (core.py:98-119).  ``mask`` is a SparsityMask or a sequence of index rows."""
    L = seq.length
    if mask is None:
        rows = [np.arange(i + 1) for i in range(L)]
    else:
        rows = _validated_rows(mask, L)
    return _dev.host(attention_dev(seq, rows))


def attention_dev(seq: TokenSequence, rows):
    """fp64 masked causal attention of validated index rows -> device [L, d]."""
    tiles, ntiles = rows_to_tiles(rows)
    q, k, v = _dev.f64(seq.queries), _dev.f64(seq.keys), _dev.f64(seq.values)
    return attend_tiles(q, k, v, _dev.i32(tiles), _dev.i32(ntiles))


def causal_probs_dev(seq: TokenSequence):
    """Device [L, L] fp64 causal softmax probabilities (dhsa_causal_probs)."""
    L, d = seq.queries.shape
    q, k = _dev.f64(seq.queries), _dev.f64(seq.keys)
    out = _dev.empty((L, L))
    _lib.call("dhsa_causal_probs", _lib.ptr(q), _lib.ptr(k), L, d, _lib.ptr(out), _dev.stream())
    return out


def causal_attention_probs(seq: TokenSequence) -> np.ndarray:
    """Full causal attention probability matrix, rows summing to 1 and zeros
    above the diagonal (core.py:122-136), computed in fp64 on the device."""
    return _dev.host(causal_probs_dev(seq))


def cosine_rows_dev(a, b):
    """Per-row cosine of two device [rows, d] fp64 tensors -> device [rows]."""
    rows, d = a.shape
    out = _dev.empty((rows,))
    _lib.call("dhsa_row_cosine", _lib.ptr(a), _lib.ptr(b), rows, d, _lib.ptr(out), _dev.stream())
    return out


def cosine_similarity(a, b) -> float:
    """Cosine of two vectors; 0.0 when either has zero norm, clamped to
    [-1, 1] (core.py:139-152); computed on the device (dhsa_row_cosine)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape or a.ndim != 1:
        raise ValueError("cosine_similarity expects two equal-length vectors")
    if a.size == 0:
        return 0.0
    return float(_dev.host(cosine_rows_dev(_dev.f64(a[None]), _dev.f64(b[None])))[0])
