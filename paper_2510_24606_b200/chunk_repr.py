"""Drop-in for ``dhsa.chunk_repr``: length-normalised chunk centroids and the
chunk-level score matrix, computed by the K1 centroid kernel and the fp64
chunk-score kernel of libdhsa_b200.

Reference: chunk_repr.py:38-54 (aggregate_chunk), :57-68 (aggregate_rows),
:71-94 (ChunkReps, build_chunk_reps), :97-103 (chunk_similarity).
Centroids are bit-identical to the reference (same fp64 addition order,
correctly rounded sqrt and division); scores are fp64 dot products.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .chunking import check_boundaries
from .core import TokenSequence

__all__ = ["ChunkReps", "aggregate_chunk", "aggregate_rows", "build_chunk_reps",
           "chunk_similarity"]


def centroids_dev(x, bounds, normalize=True, units=1):
    """x: device f64 [units, L, d] (or [L, d]); bounds: python list shared by
    all units.  Returns device f64 [units, n_chunks, d]."""
    if x.dim() == 2:
        x = x.unsqueeze(0)
    U, L, d = x.shape
    n = len(bounds) - 1
    b = _dev.i32(bounds)
    plen = _dev.i32([L] * U)
    nch = _dev.i32([n] * U)
    out = _dev.empty((U, n, d))
    lay = _lib.layout(bounds=b, plen=plen, nchunks=nch, max_chunks=n)
    _lib.call("dhsa_centroids", _lib.F64, _lib.ptr(x), L * d, d, U, lay, int(bool(normalize)),
              _lib.ptr(out), n * d, _dev.stream())
    return out


def scores_dev(qc, kc):
    """S_c = Q_c K_c^T (fp64, no scaling) for device [n, d] x [m, d]."""
    n, d = qc.shape
    m = kc.shape[0]
    out = _dev.empty((n, m))
    _lib.call("dhsa_chunk_scores", _lib.ptr(qc), _lib.ptr(kc), n, m, d, 1, n * d, m * d,
              _lib.ptr(out), n * m, _dev.stream())
    return out


def aggregate_chunk(tokens, valid_count=None) -> np.ndarray:
    """sum(tokens) / sqrt(n) with the sum accumulated row by row
    (chunk_repr.py:38-54); trailing zero padding rows beyond ``valid_count``
    are summed (exact no-ops) but not counted."""
    t = np.asarray(tokens, dtype=np.float64)
    if t.ndim != 2:
        raise ValueError("chunk must be a 2-D (tokens, dim) array")
    n = t.shape[0] if valid_count is None else int(valid_count)
    if n < 1:
        raise ValueError("chunk must contain at least one token")
    if n > t.shape[0]:
        raise ValueError(f"valid_count {n} exceeds {t.shape[0]} rows")
    s = centroids_dev(_dev.f64(t), [0, t.shape[0]], normalize=False)[0, 0]
    return _dev.host(s / math.sqrt(n))


def aggregate_rows(matrix, bounds) -> np.ndarray:
    """One centroid per chunk of ``matrix`` rows (chunk_repr.py:57-68)."""
    m = np.asarray(matrix, dtype=np.float64)
    bs = check_boundaries(bounds, m.shape[0])
    return _dev.host(centroids_dev(_dev.f64(m), bs)[0])


@dataclass(frozen=True)
class ChunkReps:
    """Aggregated chunk-level queries and keys for one sequence."""

    chunk_queries: np.ndarray
    chunk_keys: np.ndarray
    lengths: np.ndarray
    bounds: tuple

    @property
    def num_chunks(self) -> int:
        return len(self.lengths)


def reps_dev(seq: TokenSequence, bounds):
    """Device (Q_c, K_c) for a sequence: one K1 launch over [Q; K]."""
    import torch

    bs = check_boundaries(bounds, seq.length)
    qk = torch.stack([_dev.f64(seq.queries), _dev.f64(seq.keys)])
    c = centroids_dev(qk, bs, units=2)
    return c[0], c[1], bs


def build_chunk_reps(seq: TokenSequence, bounds) -> ChunkReps:
    """Aggregate a sequence's queries and keys chunk by chunk (chunk_repr.py:85-94)."""
    qc, kc, bs = reps_dev(seq, bounds)
    return ChunkReps(chunk_queries=_dev.host(qc), chunk_keys=_dev.host(kc),
                     lengths=np.diff(np.asarray(bs, dtype=np.intp)), bounds=tuple(bs))


def chunk_similarity(reps: ChunkReps) -> np.ndarray:
    """Q_c K_c^T, plain dot products (chunk_repr.py:97-103)."""
    return _dev.host(scores_dev(_dev.f64(reps.chunk_queries), _dev.f64(reps.chunk_keys)))
