"""Drop-in for the mask-quality part of ``dhsa.harness`` (SURVEY.md section
8(f) row 3): attention-mass recall, output fidelity, head-aggregated chunk
scores, the per-method masks and the ``compare`` protocol, computed on the
device (fp64 kernels of libdhsa_b200: dhsa_causal_probs, dhsa_mask_recall,
dhsa_row_cosine, dhsa_mean, dhsa_stack_reduce, plus the drop-in centroid,
score, selection, attention and predictor kernels).

Reference: harness.py:265-285 (attention_mass_recall, output_fidelity),
:288-306 (aggregated_chunk_scores), :309-343 (method_mask), :346-401
(compare).  ``compare`` takes a corpus with the reference's structure
(``.sequences``, each with ``.heads`` of TokenSequence-like q/k/v and
``.bounds``; e.g. a reference ``PlantedCorpus``); corpus generation and
the training-side harness are out of scope.  Values
agree with the reference within fp64 rounding (the dot-product and
reduction orders differ; selections are exact).
"""

from __future__ import annotations

import time

import numpy as np

from . import _dev, _lib
from .chunk_repr import reps_dev, scores_dev
from .chunking import nms_boundaries, static_boundaries
from .core import TokenSequence, attention_dev, causal_probs_dev, cosine_rows_dev, \
    _validated_rows
from .masks import CostCounters, SparsityMask, _mask_from_dev_scores

__all__ = ["attention_mass_recall", "output_fidelity", "aggregated_chunk_scores", "method_mask",
           "compare", "COMPARE_METHODS"]

COMPARE_METHODS = ("dense", "static", "dhsa_oracle", "dhsa_predicted")


def _mean_dev(x) -> float:
    out = _dev.empty((1,))
    _lib.call("dhsa_mean", _lib.ptr(x), x.numel(), _lib.ptr(out), _dev.stream())
    return float(_dev.host(out)[0])


def _csr(rows):
    ptr = np.zeros(len(rows) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(r) for r in rows])
    idx = np.concatenate([np.asarray(r, dtype=np.int32) for r in rows])
    import torch

    return torch.from_numpy(ptr).to(_dev.device()), _dev.i32(idx)


def _recall_dev(P_dev, rows) -> float:
    L = len(rows)
    ptr, idx = _csr(rows)
    frac = _dev.empty((L,))
    _lib.call("dhsa_mask_recall", _lib.ptr(P_dev), P_dev.shape[1], L, _lib.ptr(ptr),
              _lib.ptr(idx), _lib.ptr(frac), _dev.stream())
    return _mean_dev(frac)


def attention_mass_recall(attention_probs, mask: SparsityMask) -> float:
    """Mean fraction of each row's causal attention mass that the mask
    captures (harness.py:265-276)."""
    P = np.asarray(attention_probs, dtype=np.float64)
    if P.shape != (mask.length, mask.length):
        raise ValueError("probability matrix and mask sizes differ")
    return _recall_dev(_dev.f64(P), mask.rows)


def _seq(head) -> TokenSequence:
    if isinstance(head, TokenSequence):
        return head
    return TokenSequence(head.queries, head.keys, head.values)


def output_fidelity(seq, mask: SparsityMask, dense_out=None) -> float:
    """Mean per-row cosine between masked and dense attention outputs
    (harness.py:279-285)."""
    seq = _seq(seq)
    rows = _validated_rows(mask, seq.length)
    if dense_out is None:
        d = attention_dev(seq, [np.arange(i + 1) for i in range(seq.length)])
    else:
        d = _dev.f64(dense_out)
    s = attention_dev(seq, rows)
    return _mean_dev(cosine_rows_dev(s, d))


def _aggregated_dev(seq, bounds, agg, counters):
    import torch

    if agg not in ("max", "mean"):
        raise ValueError(f"unknown aggregation {agg!r}")
    per_head = []
    for head in seq.heads:
        qc, kc, bs = reps_dev(_seq(head), bounds)
        per_head.append(scores_dev(qc, kc))
    if counters is not None:
        counters.add_score_ops(sum(s.numel() for s in per_head))
    stack = torch.stack(per_head)
    H, n, _ = stack.shape
    out = _dev.empty((n, n))
    _lib.call("dhsa_stack_reduce", _lib.ptr(stack), H, n * n, _lib.AGG[agg], _lib.ptr(out),
              _dev.stream())
    return out, bs


def aggregated_chunk_scores(seq, bounds, agg="max",
                            counters: CostCounters | None = None) -> np.ndarray:
    """Per-head chunk similarities reduced over the heads by "max" or "mean"
    (harness.py:288-306); one chunk-pair score per head is counted."""
    out, _ = _aggregated_dev(seq, bounds, agg, counters)
    return _dev.host(out)


def _length(seq) -> int:
    att = getattr(seq, "attention", None)
    return int(att.shape[0]) if att is not None else int(np.shape(seq.heads[0].queries)[0])


def method_mask(seq, method, budget, chunk_size=64, predictor=None, agg="max", min_conf=0.5,
                nms_window=8, max_chunks=16, counters: CostCounters | None = None):
    """One sequence's mask for a named method (harness.py:309-343): "dense"
    (full causal), "static" (fixed grid), "dhsa_oracle" (the planted
    boundaries ``seq.bounds``), "dhsa_predicted" (predictor scores of head
    0's keys -> nms_boundaries); all chunk methods share the head-aggregated
    scoring and the exact selection."""
    length = _length(seq)
    if method == "dense":
        rows = tuple(np.arange(i + 1) for i in range(length))
        mask = SparsityMask(length=length, rows=rows)
        if counters is not None:
            counters.add_score_ops(length * (length + 1) // 2)
            counters.add_attended(length * (length + 1) // 2)
        return mask
    if method == "static":
        bounds = static_boundaries(length, chunk_size)
    elif method == "dhsa_oracle":
        bounds = seq.bounds
    elif method == "dhsa_predicted":
        if predictor is None:
            raise ValueError("dhsa_predicted requires a predictor")
        from .predictor import boundary_scores, predictable_positions

        scores = boundary_scores(seq.heads[0].keys, predictor)
        if counters is not None:
            counters.add_score_ops(len(predictable_positions(length, predictor.window)))
        bounds = nms_boundaries(scores, min_conf=min_conf, window=nms_window,
                                max_chunks=max_chunks)
    else:
        raise ValueError(f"unknown method {method!r}")
    sc, bs = _aggregated_dev(seq, bounds, agg, counters)
    if budget < 1:
        raise ValueError("budget must be >= 1")
    return _mask_from_dev_scores(sc, bs, budget, counters)


def compare(corpus, budget, chunk_size=64, predictor=None, methods=COMPARE_METHODS, agg="max",
            min_conf=0.5, nms_window=8, max_chunks=16, fidelity=True):
    """Every method over a corpus (harness.py:346-401): per-sequence rows
    {sequence, method, recall, fidelity, score_ops, attended_pairs}, a
    per-method summary {mean_recall, mean_fidelity, score_ops,
    attended_pairs, total_ops} and per-method wall-clock seconds.  The
    causal probabilities and dense outputs of every head stay on the
    device across methods."""
    methods = [m for m in methods]
    for m in methods:
        if m not in COMPARE_METHODS:
            raise ValueError(f"unknown method {m!r}")
    heads = [[_seq(h) for h in seq.heads] for seq in corpus.sequences]
    probs = [[causal_probs_dev(h) for h in hs] for hs in heads]
    dense_outs = None
    if fidelity:
        dense_outs = [[attention_dev(h, [np.arange(i + 1) for i in range(h.length)]) for h in hs]
                      for hs in heads]
    rows, summary, timings = [], {}, {}
    for method in methods:
        t0 = time.monotonic()
        total = CostCounters()
        recalls, fids = [], []
        for i, seq in enumerate(corpus.sequences):
            c = CostCounters()
            mask = method_mask(seq, method, budget, chunk_size=chunk_size, predictor=predictor,
                               agg=agg, min_conf=min_conf, nms_window=nms_window,
                               max_chunks=max_chunks, counters=c)
            recall = float(np.mean([_recall_dev(P, mask.rows) for P in probs[i]]))
            if fidelity:
                fid = float(np.mean([_mean_dev(cosine_rows_dev(attention_dev(h, mask.rows), o))
                                     for h, o in zip(heads[i], dense_outs[i])]))
            else:
                fid = float("nan")
            rows.append({"sequence": i, "method": method, "recall": recall, "fidelity": fid,
                         "score_ops": c.score_ops, "attended_pairs": c.attended_pairs})
            recalls.append(recall)
            fids.append(fid)
            total.add_score_ops(c.score_ops)
            total.add_attended(c.attended_pairs)
        summary[method] = {
            "mean_recall": float(np.mean(recalls)),
            "mean_fidelity": float(np.mean(fids)) if fidelity else None,
            "score_ops": total.score_ops,
            "attended_pairs": total.attended_pairs,
            "total_ops": total.total(),
        }
        timings[method] = time.monotonic() - t0
    return rows, summary, timings
