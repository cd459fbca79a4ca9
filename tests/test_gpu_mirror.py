"""GPU parity of the drop-in API (reference names and signatures) against
the golden vectors produced by the reference itself and the CPU oracle.
Index rows must match exactly; fp64 values within the reference's own
tolerances (1e-12)."""

import numpy as np
import pytest

import golden_io as G
import paper_2510_24606_b200 as P
from oracle import dhsa_oracle as O

pytestmark = pytest.mark.gpu


def test_topk_row_golden():
    for scores, row, budget, want in G.topk_cases():
        got = P.topk_row(scores, row, budget)
        assert np.array_equal(got, want), (scores, row, budget)


def test_topk_row_reference_examples(rng):
    assert P.topk_row(np.zeros(8), 5, 3).tolist() == [0, 1, 5]
    assert P.topk_row(np.array([5.0, 4.0, 3.0, -10.0]), 3, 3).tolist() == [0, 1, 3]
    assert P.topk_row(rng.standard_normal(10), 6, 1).tolist() == [6]
    assert P.topk_row(rng.standard_normal(5), 0, 4).tolist() == [0]
    assert P.topk_row(rng.standard_normal(6), 4, 64).tolist() == [0, 1, 2, 3, 4]
    s = rng.standard_normal(16)
    prev = set()
    for budget in range(1, 18):
        cur = set(P.topk_row(s, 15, budget).tolist())
        assert prev <= cur and len(cur) == min(budget, 16)
        prev = cur


def test_centroids_golden_bitwise():
    for rec in G.records("centroids.npz"):
        got = P.aggregate_rows(rec["m"], rec["bounds"])
        assert np.array_equal(got, rec["c"])


def test_aggregate_chunk(rng):
    t = np.tile(np.array([[1.0, -2.0]]), (4, 1))
    assert P.aggregate_chunk(t).tolist() == [2.0, -4.0]
    tokens = rng.standard_normal((5, 3))
    padded = np.vstack([tokens, np.zeros((3, 3))])
    assert np.array_equal(P.aggregate_chunk(padded, valid_count=5), P.aggregate_chunk(tokens))
    one = rng.standard_normal((1, 5))
    assert np.array_equal(P.aggregate_chunk(one), one[0])
    assert np.array_equal(P.aggregate_chunk(tokens), O.centroid(tokens))


def test_chunk_similarity(rng):
    reps = P.ChunkReps(np.array([[2.0, 0.0]]), np.array([[3.0, 0.0]]), np.array([1]), (0, 1))
    assert P.chunk_similarity(reps)[0, 0] == 6.0
    seq = P.TokenSequence(*(rng.standard_normal((12, 4)) for _ in range(3)))
    reps = P.build_chunk_reps(seq, [0, 3, 7, 12])
    assert list(reps.lengths) == [3, 4, 5] and reps.bounds == (0, 3, 7, 12)
    assert np.array_equal(reps.chunk_queries, O.centroids(seq.queries, [0, 3, 7, 12]))
    assert np.array_equal(reps.chunk_keys, O.centroids(seq.keys, [0, 3, 7, 12]))
    np.testing.assert_allclose(P.chunk_similarity(reps),
                               O.chunk_scores(reps.chunk_queries, reps.chunk_keys), atol=1e-12)


def test_upsample(rng):
    bounds = [0, 2, 5, 9]
    s = rng.standard_normal((3, 3))
    up = P.upsample(s, bounds)
    lens = np.diff(bounds)
    assert np.array_equal(up, np.repeat(np.repeat(s, lens, 0), lens, 1))


def test_decode_sessions_golden():
    for rec in G.records("decode.npz"):
        Pn = rec["prompt"]
        sess = P.DecodeSession(rec["k"][:Pn], rec["bounds"], rec["budget"])
        assert np.array_equal(sess.cached_chunk_keys, rec["cached"])
        for s, want in enumerate(rec["rows"]):
            t = Pn + s
            got = sess.step(rec["q"][t], rec["k"][t])
            assert np.array_equal(got, want), (s, got, want)
            stateless = P.decode_mask_row(rec["bounds"], rec["cached"], rec["k"][Pn:t + 1],
                                          rec["q"][t], t + 1, rec["budget"])
            assert np.array_equal(stateless, want)
        assert sess.total_length == Pn + len(rec["rows"])


def test_decode_counters(rng):
    k = rng.standard_normal((14, 3))
    q = rng.standard_normal((14, 3))
    c = P.CostCounters()
    sess = P.DecodeSession(k[:10], [0, 6, 10], 4, counters=c)
    r1 = sess.step(q[10], k[10])
    r2 = sess.step(q[11], k[11])
    assert c.score_ops == 3 + 4  # 2 prompt chunks + singleton, then + gen chunk
    assert c.attended_pairs == len(r1) + len(r2)
    assert len(r2) == 4 and r2[-1] == 11


def test_prefill_masks_and_attention_golden():
    for rec in G.records("prefill.npz"):
        seq = P.TokenSequence(rec["q"], rec["k"], rec["v"])
        mask = P.prefill_mask(seq, rec["bounds"], rec["budget"])
        assert len(mask.rows) == len(rec["rows"])
        for a, b in zip(mask.rows, rec["rows"]):
            assert np.array_equal(a, b)
        out = P.dense_attention(seq, mask)
        np.testing.assert_allclose(out, rec["out"], rtol=0, atol=1e-12)


def test_full_budget_is_dense_bitwise(rng):
    for L in (4, 16, 33):
        seq = P.TokenSequence(*(rng.standard_normal((L, 5)) for _ in range(3)))
        mask = P.prefill_mask(seq, sorted({0, 1, L // 2, L}), budget=L)
        assert all(len(mask.rows[i]) == i + 1 for i in range(L))
        assert np.array_equal(P.dense_attention(seq, mask.rows), P.dense_attention(seq))
        want = O.attend_rows(seq.queries, seq.keys, seq.values,
                             [np.arange(i + 1) for i in range(L)])
        np.testing.assert_allclose(P.dense_attention(seq), want, atol=1e-12)


def test_prefill_counters(rng):
    seq = P.TokenSequence(*(rng.standard_normal((12, 3)) for _ in range(3)))
    c = P.CostCounters()
    mask = P.prefill_mask(seq, [0, 4, 8, 12], budget=4, counters=c)
    assert c.score_ops == 9
    assert c.attended_pairs == int(mask.row_sizes().sum())


def test_mask_from_chunk_scores_matches_oracle_walk(rng):
    for _ in range(40):
        L = int(rng.integers(1, 200))
        cuts = sorted(set(rng.integers(1, max(L, 2), size=int(rng.integers(0, 9))).tolist()))
        bounds = [0] + [c for c in cuts if c < L] + [L]
        n = len(bounds) - 1
        s = rng.standard_normal((n, n))
        if rng.random() < 0.5:
            s = np.round(s)
        budget = int(rng.integers(1, L + 3))
        mask = P.mask_from_chunk_scores(s, bounds, budget)
        for i in range(L):
            l = int(np.searchsorted(bounds, i, side="right") - 1)
            want = O.ranges_to_indices(O.walk_ranges(s[l], bounds, i, budget), i)
            assert np.array_equal(mask.rows[i], want)


def test_dense_attention_masked_vs_oracle(rng):
    for _ in range(20):
        L = int(rng.integers(1, 40))
        d = int(rng.choice([1, 3, 8, 64, 130]))
        seq = P.TokenSequence(*(rng.standard_normal((L, d)) for _ in range(3)))
        rows = [sorted(set(j for j in range(i) if rng.random() < 0.5) | {i}) for i in range(L)]
        want = O.attend_rows(seq.queries, seq.keys, seq.values, rows)
        np.testing.assert_allclose(P.dense_attention(seq, rows), want, atol=1e-12)


def test_topk_row_beyond_shared_memory(rng):
    """topk_row over ~40K positions (one chunk per token, more keys than the
    select's shared memory holds): the global-scratch select gives the
    reference's row (masks.py:103-122), ties included."""
    s = rng.standard_normal(40000)
    s[100:300] = s[5]  # a tie class
    for row, budget in ((39999, 4097), (30000, 20000), (39999, 1), (25000, 40000)):
        want = O.token_topk(s, row, budget)
        assert np.array_equal(P.topk_row(s, row, budget), want), (row, budget)



def test_softmax_row_reference_cases(rng):
    """core.py:69-77 and the reference's own softmax tests (test_core.py:32-56)."""
    for _ in range(20):
        s = rng.standard_normal(int(rng.integers(1, 300))) * 10.0
        e = np.exp(s - s.max())
        np.testing.assert_allclose(P.softmax_row(s), e / e.sum(), atol=1e-14)
        p = P.softmax_row(s)
        assert abs(p.sum() - 1.0) < 1e-12 and np.all(p > 0)
    s = rng.standard_normal(6)
    np.testing.assert_allclose(P.softmax_row(s), P.softmax_row(s + 123.0), atol=1e-12)
    np.testing.assert_allclose(P.softmax_row(np.zeros(5)), np.full(5, 0.2))
    p = P.softmax_row(np.array([1000.0, 999.0]))
    assert np.all(np.isfinite(p)) and abs(p.sum() - 1.0) < 1e-12
    for bad in (np.zeros(0), np.zeros((2, 2)), np.array([1.0, np.inf])):
        with pytest.raises(ValueError):
            P.softmax_row(bad)


@pytest.mark.parametrize("D", [128, 64, 6, 5])
def test_centroids_bf16_kernels_bitwise(D):
    """K1 over bf16 inputs (the decode / prefill cache dtype) through every
    load width — 16-byte rows (D % 8 == 0), bf16x2 (D even), scalar — with
    static and ragged explicit chunks, bitwise equal to the sequential fp64
    sums of chunk_repr.py:29-68 (oracle centroids pinned to the reference)."""
    import torch

    from paper_2510_24606_b200 import _lib

    rng = np.random.default_rng(D)
    U, L = 3, 700
    x = torch.from_numpy(rng.standard_normal((U, L, D), dtype=np.float32) * 7).bfloat16().cuda()
    xh = x.double().cpu().numpy()
    ragged = [0, 1, 9, 64, 65, 200, 333, 334, 600, 700]
    for bounds in (None, ragged):
        plen = torch.full((U,), L, dtype=torch.int32, device="cuda")
        if bounds is None:
            nc = (L + 63) // 64
            lay = _lib.layout(plen=plen, block=64, max_chunks=nc)
            bl = O.static_grid(L, 64)
        else:
            nc = len(bounds) - 1
            kb = torch.tensor([bounds] * U, dtype=torch.int32, device="cuda")
            ncs = torch.full((U,), nc, dtype=torch.int32, device="cuda")
            lay = _lib.layout(bounds=kb, bounds_stride=nc + 1, nchunks=ncs, plen=plen,
                              max_chunks=nc)
            bl = bounds
        out = torch.zeros(U, nc, D, dtype=torch.float64, device="cuda")
        _lib.call("dhsa_centroids", _lib.BF16, _lib.ptr(x), L * D, D, U, lay, 1, _lib.ptr(out),
                  nc * D, _lib.stream_handle())
        got = out.cpu().numpy()
        for u in range(U):
            assert np.array_equal(got[u], O.centroids(xh[u], bl)), (D, u, bounds)
