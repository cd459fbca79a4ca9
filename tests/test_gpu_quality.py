"""Mask-quality metrics on the GPU against the reference harness's own
outputs (fixtures from tests/golden/make_golden.py
gen_quality, produced by running /root/reference's harness):

* the drop-in harness (``paper_2510_24606_b200.harness``: compare,
  method_mask, attention_mass_recall, output_fidelity, and core's
  causal_attention_probs / cosine_similarity) on a planted corpus at the
  reference's shapes — integer counts exact, masks exact, metric values
  within fp64 rounding (1e-12);
* the batched tcgen05 path (``prefill.mask_quality``: row statistics of the
  sparse and a dense run) at d = 128 with bf16-valued inputs — sampled mask
  rows exact, per-row recall / cosine within the bf16 tolerance."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

import golden_io as G

pytestmark = pytest.mark.gpu

METHODS = ("dense", "static", "dhsa_oracle", "dhsa_predicted")


def _corpus(z, n):
    import paper_2510_24606_b200 as P

    seqs = []
    for i in range(n):
        q, k, v = z[f"q_{i}"], z[f"k_{i}"], z[f"v_{i}"]
        heads = tuple(P.TokenSequence(q[h], k[h], v[h]) for h in range(q.shape[0]))
        seqs.append(SimpleNamespace(heads=heads, bounds=tuple(int(b) for b in z[f"bounds_{i}"])))
    return SimpleNamespace(sequences=tuple(seqs))


def _kw(z):
    from paper_2510_24606_b200.predictor import init_predictor

    pred = init_predictor(32, window=4, heads=8, hidden=int(z["pred_hidden"]),
                          seed=int(z["pred_seed"]))
    return dict(chunk_size=int(z["chunk_size"]), predictor=pred, min_conf=float(z["min_conf"]),
                nms_window=int(z["nms_window"]), max_chunks=int(z["max_chunks"]))


def test_compare_matches_reference_harness():
    from paper_2510_24606_b200 import harness as H

    z = G.load("quality.npz")
    corpus = _corpus(z, 3)
    rows, summary, timings = H.compare(corpus, int(z["budget"]), methods=METHODS, **_kw(z))
    table = np.array([[r["sequence"], METHODS.index(r["method"]), r["score_ops"],
                       r["attended_pairs"]] for r in rows])
    assert np.array_equal(table, z["table"])
    np.testing.assert_allclose([r["recall"] for r in rows], z["recall"], rtol=0, atol=1e-12)
    np.testing.assert_allclose([r["fidelity"] for r in rows], z["fidelity"], rtol=0, atol=1e-12)
    got = np.array([[summary[m]["mean_recall"], summary[m]["mean_fidelity"],
                     summary[m]["score_ops"], summary[m]["attended_pairs"],
                     summary[m]["total_ops"]] for m in METHODS])
    np.testing.assert_allclose(got, z["summary"], rtol=0, atol=1e-12)
    assert set(timings) == set(METHODS)


def test_method_masks_and_metrics_match_reference():
    import paper_2510_24606_b200 as P
    from paper_2510_24606_b200 import harness as H

    z = G.load("quality.npz")
    corpus = _corpus(z, 1)
    seq0 = corpus.sequences[0]
    kw = _kw(z)
    for m in METHODS:
        mask = H.method_mask(seq0, m, int(z["budget"]), **kw)
        want = G.unpack_rows(z[f"mask_{m}"], z[f"mask_{m}_off"])
        assert len(mask.rows) == len(want)
        for a, b in zip(mask.rows, want):
            assert np.array_equal(a, b), m
    mask = H.method_mask(seq0, "dhsa_oracle", int(z["budget"]), chunk_size=int(z["chunk_size"]))
    rec = [H.attention_mass_recall(P.causal_attention_probs(h), mask) for h in seq0.heads]
    fid = [H.output_fidelity(h, mask) for h in seq0.heads]
    np.testing.assert_allclose(rec, z["head_recall"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(fid, z["head_fidelity"], rtol=0, atol=1e-12)
    with pytest.raises(ValueError, match="sizes differ"):
        H.attention_mass_recall(np.eye(3), mask)
    with pytest.raises(ValueError, match="unknown method"):
        H.method_mask(seq0, "bogus", 10)
    with pytest.raises(ValueError, match="requires a predictor"):
        H.method_mask(seq0, "dhsa_predicted", 10)


def test_causal_probs_and_cosine_match_reference():
    import paper_2510_24606_b200 as P

    z = G.load("quality.npz")
    seq = P.TokenSequence(z["small_q"], z["small_k"], z["small_v"])
    np.testing.assert_allclose(P.causal_attention_probs(seq), z["small_probs"], rtol=0,
                               atol=1e-14)
    a, b = z["cos_ab"]
    got = [P.cosine_similarity(a, b), P.cosine_similarity(a, -a),
           P.cosine_similarity(np.zeros(9), b)]
    np.testing.assert_allclose(got, z["cos"], rtol=0, atol=1e-14)
    with pytest.raises(ValueError, match="equal-length"):
        P.cosine_similarity(a, b[:3])


def test_aggregated_chunk_scores_matches_oracle():
    from oracle import dhsa_oracle as O
    from paper_2510_24606_b200 import harness as H

    z = G.load("quality.npz")
    seq = _corpus(z, 1).sequences[0]
    b = list(seq.bounds)
    per = np.stack([O.chunk_scores(O.centroids(h.queries, b), O.centroids(h.keys, b))
                    for h in seq.heads])
    np.testing.assert_allclose(H.aggregated_chunk_scores(seq, b, "max"), per.max(axis=0),
                               rtol=0, atol=1e-12)
    np.testing.assert_allclose(H.aggregated_chunk_scores(seq, b, "mean"), per.mean(axis=0),
                               rtol=0, atol=1e-12)


@pytest.mark.parametrize("method", ["static", "dhsa_oracle"])
def test_batched_mask_quality_matches_reference(method):
    """SparsePrefill (tcgen05) + prefill.mask_quality on the planted d = 128
    corpus: both sequences as the batch, one head each (the harness's head
    aggregation is the identity); bf16-exact inputs."""
    from paper_2510_24606_b200.prefill import SparsePrefill, mask_quality

    z = G.load("quality_bf16.npz")
    budget = int(z["budget"])
    B, L, D = 2, z["q_0"].shape[0], z["q_0"].shape[1]

    def dev(name):
        return torch.from_numpy(np.stack([z[f"{name}_{i}"] for i in range(B)])[:, None]) \
            .to(torch.bfloat16).cuda().contiguous()

    q, k, v = dev("q"), dev("k"), dev("v")
    bounds = None if method == "static" else [[int(x) for x in z[f"bounds_{i}"]]
                                              for i in range(B)]
    pf = SparsePrefill(B, 1, 1, D, L, budget=budget, agg="max", bounds=bounds)
    rec, cos = mask_quality(q, k, v, pf)
    torch.cuda.synchronize()
    rec, cos = rec.double().cpu().numpy(), cos.double().cpu().numpy()
    hp = pf.host_plans()
    for i in range(B):
        want = G.unpack_rows(z[f"rows_{method}_{i}"], z[f"rows_{method}_{i}_off"])
        for r, w in zip(z["sample"], want):
            assert np.array_equal(pf.row_indices(i, int(r), hp), w), (i, r)
        # recall: fp32 row statistics of bf16-exact scores (ex2.approx)
        np.testing.assert_allclose(rec[i, 0], z[f"recall_{method}_{i}"], rtol=0, atol=2e-3)
        # cosine of bf16 outputs
        np.testing.assert_allclose(cos[i, 0], z[f"cos_{method}_{i}"], rtol=0, atol=2e-2)
        assert abs(rec[i, 0].mean() - z[f"recall_{method}_{i}"].mean()) < 5e-4
        assert abs(cos[i, 0].mean() - z[f"cos_{method}_{i}"].mean()) < 5e-3
