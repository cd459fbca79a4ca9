"""Property-based invariants of the GPU drop-in path (hypothesis), the
counterpart of the reference's property suite for the hot path
(tests/test_properties.py of the reference: top-K row contract and budget
nesting, upsample partition lookup, decode session == prefill on random
partitions, mask rows follow the chunk scores).  Every draw runs the CUDA
kernels and is checked against the CPU oracle or the contract itself; the
CPU-only properties (NMS, wire formats) run without a GPU."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import dhsa_oracle as O

finite = st.floats(min_value=-100.0, max_value=100.0, allow_nan=False, width=64)


@st.composite
def scored_row(draw):
    n = draw(st.integers(1, 24))
    scores = np.array(draw(st.lists(finite, min_size=n, max_size=n)))
    if draw(st.booleans()):  # heavy ties
        scores = np.round(scores / 50.0)
    row = draw(st.integers(0, n - 1))
    budget = draw(st.integers(1, n + 4))
    return scores, row, budget


@st.composite
def partition(draw, max_length=24):
    length = draw(st.integers(1, max_length))
    cuts = draw(st.sets(st.integers(1, max(1, length - 1)), max_size=6))
    return length, [0] + sorted(c for c in cuts if c < length) + [length]


# ----------------------------------------------------------------- GPU --

@pytest.mark.gpu
@given(scored_row())
@settings(max_examples=200, deadline=None)
def test_topk_row_contract(case):
    """Self included, causal, sorted unique, |row| = min(budget, row+1), and
    equal to the stable-argsort oracle (masks.py:103-122)."""
    import paper_2510_24606_b200 as P

    scores, row, budget = case
    got = P.topk_row(scores, row, budget)
    assert row in got
    assert np.all(np.diff(got) > 0) and got[0] >= 0 and got[-1] <= row
    assert len(got) == min(budget, row + 1)
    assert np.array_equal(got, O.token_topk(scores, row, budget))


@pytest.mark.gpu
@given(scored_row())
@settings(max_examples=100, deadline=None)
def test_topk_budget_nesting(case):
    import paper_2510_24606_b200 as P

    scores, row, budget = case
    small = set(P.topk_row(scores, row, budget).tolist())
    big = set(P.topk_row(scores, row, budget + 1).tolist())
    assert small <= big


@pytest.mark.gpu
@given(partition(), st.data())
@settings(max_examples=40, deadline=None)
def test_upsample_partition_lookup(part, data):
    """S_t[i][j] = S_c[chunk(i)][chunk(j)] (masks.py:87-100)."""
    import paper_2510_24606_b200 as P

    length, bounds = part
    n = len(bounds) - 1
    sc = np.array(data.draw(st.lists(finite, min_size=n * n, max_size=n * n))).reshape(n, n)
    up = P.upsample(sc, bounds)
    cid = np.searchsorted(bounds, np.arange(length), side="right") - 1
    assert np.array_equal(up, sc[cid][:, cid])


@pytest.mark.gpu
@given(partition(max_length=16), st.integers(1, 18), st.data())
@settings(max_examples=100, deadline=None)
def test_mask_rows_follow_chunk_scores(part, budget, data):
    """mask_from_chunk_scores rows = topk_row over the upsampled row, for
    any partition (masks.py:125-140)."""
    import paper_2510_24606_b200 as P

    length, bounds = part
    n = len(bounds) - 1
    sc = np.array(data.draw(st.lists(finite, min_size=n * n, max_size=n * n))).reshape(n, n)
    if data.draw(st.booleans()):
        sc = np.round(sc / 40.0)
    mask = P.mask_from_chunk_scores(sc, bounds, budget)
    cid = np.searchsorted(bounds, np.arange(length), side="right") - 1
    for i in range(length):
        want = O.token_topk(sc[cid[i]][cid], i, budget)
        assert np.array_equal(mask.rows[i], want), (i, bounds, budget)


@pytest.mark.gpu
@given(partition(max_length=12), st.integers(1, 4), st.integers(1, 16),
       st.integers(0, 2 ** 31 - 1))
@settings(max_examples=80, deadline=None)
def test_session_matches_prefill(part, extra, budget, seed):
    """The decode row of token t (DecodeSession, masks.py:205-237) equals
    row t of prefill_mask over the decode-extended boundaries
    (chunking.extend_for_decode), step after step."""
    import paper_2510_24606_b200 as P

    length, bounds = part
    rng = np.random.default_rng(seed)
    d = 4
    total = length + extra
    q = rng.integers(-3, 4, size=(total, d)).astype(np.float64)  # exact scores
    k = rng.integers(-3, 4, size=(total, d)).astype(np.float64)
    v = rng.standard_normal((total, d))
    sess = P.DecodeSession(k[:length], bounds, budget)
    for t in range(length, total):
        row = sess.step(q[t], k[t])
        eb = P.extend_for_decode(bounds, t + 1)
        seq = P.TokenSequence(q[:t + 1], k[:t + 1], v[:t + 1])
        want = P.prefill_mask(seq, eb, budget).rows[t]
        assert np.array_equal(row, want), (t, bounds, budget)


# ----------------------------------------------------------------- CPU --

@given(st.integers(2, 40), st.integers(0, 8), st.integers(1, 6), st.data())
@settings(max_examples=60, deadline=None)
def test_nms_partition_contract(length, window, max_chunks, data):
    """nms_boundaries returns a valid partition with at most max_chunks
    chunks, invariant under a positive rescaling of the scores."""
    from paper_2510_24606_b200.chunking import check_boundaries, nms_boundaries

    sc = np.array(data.draw(st.lists(st.floats(0.0, 1.0), min_size=length, max_size=length)))
    b = nms_boundaries(sc, 0.1, window, max_chunks)
    check_boundaries(b, length)
    assert len(b) - 1 <= max_chunks
    assert nms_boundaries(sc * 2.0, 0.2, window, max_chunks) == b  # exact scaling


@given(st.integers(1, 20), st.integers(0, 2 ** 31 - 1))
@settings(max_examples=40, deadline=None)
def test_mask_wire_round_trip(length, seed):
    """DHSAMSK1 bitsets and the JSON form round-trip any causal rows."""
    import os
    import tempfile

    from paper_2510_24606_b200 import serialization as S

    rng = np.random.default_rng(seed)
    rows = [np.unique(np.r_[rng.integers(0, i + 1, size=rng.integers(0, i + 1)), i])
            for i in range(length)]

    class M:
        pass

    m = M()
    m.length, m.rows = length, rows
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "m.msk")
        S.save_mask(p, m)
        L2, back = S.load_mask(p)
    assert L2 == length and all(np.array_equal(a, b) for a, b in zip(rows, back))
    L3, back = S.mask_from_json(S.mask_to_json(m))
    assert L3 == length and all(np.array_equal(a, b) for a, b in zip(rows, back))
