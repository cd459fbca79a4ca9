"""paper_2510_24606_b200 — B200-native (sm_100a) DHSA sparse-attention hot path.

Drop-in for the hot-path surface of the reference package ``dhsa``
(/root/reference/pkg/src/dhsa/__init__.py:7-49): the same names and
signatures for chunk representations, sparsity masks (prefill and decode) and
masked attention, computed by hand-written CUDA kernels in libdhsa_b200.so,
plus the batched decode engine ``SparseDecoder`` that the benchmark drives.
There is no CPU fallback: GPU entry points raise if the library or the
device is missing.
"""

from .chunking import check_boundaries, extend_for_decode, nms_boundaries, static_boundaries
from .core import TokenSequence, causal_attention_probs, cosine_similarity, dense_attention, \
    softmax_row
from .chunk_repr import ChunkReps, aggregate_chunk, aggregate_rows, build_chunk_reps, \
    chunk_similarity
from . import harness, predictor, serialization
from .masks import CostCounters, DecodeSession, SparsityMask, decode_mask_row, \
    mask_from_chunk_scores, prefill_mask, topk_row, upsample

__version__ = "0.1.0"

__all__ = [
    "TokenSequence", "softmax_row", "dense_attention", "causal_attention_probs",
    "cosine_similarity",
    "check_boundaries", "static_boundaries", "nms_boundaries", "extend_for_decode",
    "ChunkReps", "aggregate_chunk", "aggregate_rows", "build_chunk_reps", "chunk_similarity",
    "CostCounters", "SparsityMask", "upsample", "topk_row", "mask_from_chunk_scores",
    "prefill_mask", "decode_mask_row", "DecodeSession",
    "SparseDecoder", "SparsePrefill", "SplitKVShard", "SplitKVGroup", "predictor",
    "harness",
]


def __getattr__(name):
    if name == "SparseDecoder":
        from .decode import SparseDecoder

        return SparseDecoder
    if name == "SparsePrefill":
        from .prefill import SparsePrefill

        return SparsePrefill
    if name in ("SplitKVShard", "SplitKVGroup"):
        from . import splitkv

        return getattr(splitkv, name)
    raise AttributeError(name)
