"""Pin the CPU oracle against the golden vectors the reference produced
(tests/golden/make_golden.py).  No GPU needed."""

import numpy as np
import pytest

import golden_io as G
from oracle import dhsa_oracle as O


@pytest.mark.parametrize("method", ["walk", "token"])
def test_topk_known_answers(method):
    for scores, row, budget, want in G.topk_cases():
        if method == "token":
            got = O.token_topk(scores, row, budget)
        else:
            got = O.ranges_to_indices(
                O.walk_ranges(scores, list(range(len(scores) + 1)), row, budget), row)
        assert np.array_equal(got, want), (scores, row, budget)


def test_topk_reference_examples():
    # tests/test_masks.py:92-99 of the reference
    assert O.token_topk(np.zeros(8), 5, 3).tolist() == [0, 1, 5]
    assert O.token_topk(np.array([5.0, 4.0, 3.0, -10.0]), 3, 3).tolist() == [0, 1, 3]
    with pytest.raises(ValueError):
        O.token_topk(np.zeros(4), 2, 0)


def test_centroids_bitwise():
    for rec in G.records("centroids.npz"):
        got = O.centroids(rec["m"], rec["bounds"])
        assert np.array_equal(got, rec["c"])


@pytest.mark.parametrize("method", ["walk", "token"])
def test_decode_sessions(method):
    for rec in G.records("decode.npz"):
        P = rec["prompt"]
        sess = O.DecodeOracle(rec["k"][:P], rec["bounds"], rec["budget"])
        assert np.array_equal(sess.cached, rec["cached"])
        for s, want in enumerate(rec["rows"]):
            t = P + s
            got = sess.step(rec["q"][t], rec["k"][t], method=method)
            assert np.array_equal(got, want)


def test_prefill_rows_and_attention():
    for rec in G.records("prefill.npz"):
        rows = O.prefill_rows(rec["q"], rec["k"], rec["bounds"], rec["budget"])
        assert len(rows) == len(rec["rows"])
        for a, b in zip(rows, rec["rows"]):
            assert np.array_equal(a, b)
        out = O.attend_rows(rec["q"], rec["k"], rec["v"], rows)
        np.testing.assert_allclose(out, rec["out"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("agg,slot", [("max", 0), ("mean", 1)])
@pytest.mark.parametrize("method", ["walk", "token"])
def test_group_rows(agg, slot, method):
    for rec in G.records("group.npz"):
        k, qh = rec["k"], rec["q"]
        pb = [int(x) for x in rec["prompt_bounds"]]
        P, g = pb[-1], rec["gen"]
        t = P + g
        cached = O.centroids(k[:P], pb)
        gsum = O.running_sum(k[P:t]) if g else np.zeros(k.shape[1])
        got = O.decode_row_group(pb, cached, gsum, g, k[t], qh[:, t], rec["budget"],
                                 agg=agg, method=method)
        assert np.array_equal(got, rec["rows"][slot])


def test_c1_decode_and_attention():
    gd = G.c1_golden()
    L, steps = gd["L"], gd["steps"]
    bounds = O.static_grid(L, 64)
    for h in range(gd["H"]):
        sess = O.DecodeOracle(gd["k"][h, :L], bounds, gd["budget"])
        for s in range(steps):
            t = L + s
            row = sess.step(gd["q"][h, t], gd["k"][h, t])
            assert np.array_equal(row, G.ranges_to_idx(gd["rows"][(h, s)], t))
            o = O.attend_row(gd["q"][h, t], gd["k"][h, : t + 1], gd["v"][h, : t + 1], row)
            np.testing.assert_allclose(o, gd["out"][h, s], rtol=0, atol=1e-12)


def test_walk_equals_token_topk_random(rng):
    """Appendix-A equivalence on fresh random + tie-heavy cases."""
    for _ in range(300):
        L = int(rng.integers(1, 60))
        cuts = sorted(set(rng.integers(1, max(L, 2), size=int(rng.integers(0, 6))).tolist()))
        bounds = [0] + [c for c in cuts if c < L] + [L]
        n = len(bounds) - 1
        s = rng.standard_normal(n)
        if rng.random() < 0.5:
            s = np.round(s)
        row = int(rng.integers(0, L))
        budget = int(rng.integers(1, L + 3))
        tok = np.repeat(s, np.diff(bounds))
        a = O.token_topk(tok, row, budget)
        b = O.ranges_to_indices(O.walk_ranges(s, bounds, row, budget), row)
        assert np.array_equal(a, b)


def test_mask_quality_oracle_pinned_to_reference_harness():
    """oracle.mask_quality (the checker of the GPU mask-quality metrics) vs
    the reference harness's own per-row attention_mass_recall fractions and
    output_fidelity cosines (harness.py:265-285, quality_bf16.npz from
    make_golden.gen_quality), with the oracle's own prefill rows."""
    import golden_io as G

    z = G.load("quality_bf16.npz")
    budget = int(z["budget"])
    for i in range(2):
        q, k, v = z[f"q_{i}"], z[f"k_{i}"], z[f"v_{i}"]
        L = q.shape[0]
        for m in ("static", "dhsa_oracle"):
            bounds = O.static_grid(L, 64) if m == "static" else [int(x) for x in z[f"bounds_{i}"]]
            rows = O.prefill_rows(q, k, bounds, budget)
            want = G.unpack_rows(z[f"rows_{m}_{i}"], z[f"rows_{m}_{i}_off"])
            for r, w in zip(z["sample"], want):
                assert np.array_equal(rows[r], w), (i, m, r)
            rec, cos = O.mask_quality(q, k, v, rows)
            np.testing.assert_allclose(rec, z[f"recall_{m}_{i}"], rtol=0, atol=1e-12)
            np.testing.assert_allclose(cos, z[f"cos_{m}_{i}"], rtol=0, atol=1e-12)
