"""Analytic cost accounting of the batched engines:
``SparseDecoder.cost_counters`` / ``SparsePrefill.cost_counters`` must equal
the reference's CostCounters tallies (masks.py:38-52) — per q head the
decode row's score count (masks.py:166-167) and admitted pairs (:171-172),
or prefill_mask's N_c^2 scores and row sizes (masks.py:138-139, 147-148) —
here obtained by running the drop-in DecodeSession / prefill_mask (the
reference's counting code paths) on the same shapes.  Group aggregation
counts one score matrix per head (harness.py:300-301) and one mask per
kv group."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("agg", ["max", "none"])
@pytest.mark.parametrize("budget", [40, 303, 1000])
def test_decoder_counters_match_reference_counting(agg, budget):
    import paper_2510_24606_b200 as P
    from paper_2510_24606_b200.decode import SparseDecoder

    B, Hq, Hkv, D, Pn, steps = 2, 4, 2, 128, 300, 5
    rng = np.random.default_rng(3)
    k = torch.from_numpy(rng.standard_normal((B, Hkv, Pn + steps, D), dtype=np.float32)).bfloat16()
    v = torch.from_numpy(rng.standard_normal((B, Hkv, Pn + steps, D), dtype=np.float32)).bfloat16()
    q = torch.from_numpy(rng.standard_normal((B, Hq, steps, D), dtype=np.float32)).bfloat16()
    dec = SparseDecoder(B, Hq, Hkv, D, Pn + steps + 1, block=64, budget=budget,
                        dtype=torch.bfloat16, agg=agg)
    dec.prefill(k[:, :, :Pn].cuda(), v[:, :, :Pn].cuda())
    for s in range(steps):
        dec.step(q[:, :, s].contiguous().cuda(), k[:, :, Pn + s].contiguous().cuda(),
                 v[:, :, Pn + s].contiguous().cuda())
    got = dec.cost_counters()
    # the reference's counting: one DecodeSession per q head (3 heads' worth
    # is enough: every head of this layout counts the same)
    kh = k.double().numpy()
    qh = q.double().numpy()
    ref = P.CostCounters()
    sess = P.DecodeSession(kh[0, 0, :Pn], P.static_boundaries(Pn, 64), budget, counters=ref)
    for s in range(steps):
        sess.step(qh[0, 0, s], kh[0, 0, Pn + s])
    heads = B * Hq
    rows = heads if agg == "none" else B * Hkv
    assert got.score_ops == ref.score_ops * heads
    assert got.attended_pairs == ref.attended_pairs * rows


@pytest.mark.parametrize("agg", ["max", "none"])
def test_prefill_counters_match_reference_counting(agg):
    import paper_2510_24606_b200 as P
    from paper_2510_24606_b200.prefill import SparsePrefill

    B, Hq, Hkv, D, L, budget = 1, 4, 2, 128, 300, 130
    rng = np.random.default_rng(4)
    q, k, v = (torch.from_numpy(rng.standard_normal((B, h, L, D), dtype=np.float32)).bfloat16()
               .cuda() for h in (Hq, Hkv, Hkv))
    bounds = [0, 5, 64, 70, 200, 260, 300]
    for bnd in (None, bounds):
        pf = SparsePrefill(B, Hq, Hkv, D, L, budget=budget, agg=agg, bounds=bnd)
        pf(q, k, v)
        got = pf.cost_counters()
        ref = P.CostCounters()
        seq = P.TokenSequence(q[0, 0].double().cpu().numpy(), k[0, 0].double().cpu().numpy(),
                              v[0, 0].double().cpu().numpy())
        P.prefill_mask(seq, P.static_boundaries(L, 64) if bnd is None else bnd, budget,
                       counters=ref)
        rows = B * Hq if agg == "none" else B * Hkv
        assert got.score_ops == ref.score_ops * B * Hq
        assert got.attended_pairs == ref.attended_pairs * rows
