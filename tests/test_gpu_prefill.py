"""GPU parity of the tcgen05 sparse prefill (config C5's path) against the
CPU oracle: the per-row index sets the plans encode must equal the oracle's
prefill rows (masks.prefill_mask semantics: topk_row on the upsampled row,
head-aggregated S_c for GQA groups) index-for-index, and the attention output
must match the float64 row body (core.py:113-118) within 2e-2 of max|o_ref|
per (sequence, head) — the bf16 tolerance of the north star."""

import numpy as np
import pytest
import torch

from oracle import dhsa_oracle as O

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2


def _inputs(B, Hq, Hkv, L, D, seed, kind="normal"):
    rng = np.random.default_rng(seed)

    def draw(*shape):
        if kind == "int":
            return rng.integers(-3, 4, size=shape).astype(np.float32)
        return rng.standard_normal(shape, dtype=np.float32)

    q, k, v = draw(B, Hq, L, D), draw(B, Hkv, L, D), draw(B, Hkv, L, D)
    if kind == "wide":  # large logits: exercises the online-softmax rescaling
        q *= 8.0
    if kind == "ties":
        k[:, :, 128:192] = k[:, :, 0:64]
    t = {n: torch.from_numpy(np.ascontiguousarray(x)).bfloat16() for n, x in
         dict(q=q, k=k, v=v).items()}
    host = {n: x.double().numpy() for n, x in t.items()}
    return t, host


def _run(B, Hq, Hkv, L, top_k=None, budget=None, agg="max", seed=0, kind="normal",
         check_rows=None, check_out=True, bounds=None):
    """``bounds``: None (static grid), one list, or one list per kv unit."""
    from paper_2510_24606_b200.prefill import SparsePrefill

    D = 128
    G = Hq // Hkv
    t, host = _inputs(B, Hq, Hkv, L, D, seed, kind)
    pf = SparsePrefill(B, Hq, Hkv, D, L, top_k=top_k or 4, budget=budget, agg=agg,
                       bounds=bounds)
    out = pf(t["q"].cuda(), t["k"].cuda(), t["v"].cuda())
    torch.cuda.synchronize()
    pf.check_capacity()
    o = out.double().cpu().numpy()
    hp = pf.host_plans()
    worst = 0.0
    for b in range(B):
        for h in range(Hkv):
            u = b * Hkv + h
            if bounds is None:
                ub = O.static_grid(L, 64)
            elif np.isscalar(bounds[0]):
                ub = list(bounds)
            else:
                ub = list(bounds[u])
            qh = host["q"][b, h * G:(h + 1) * G]
            kh = np.repeat(host["k"][b, h][None], G, axis=0)
            if agg == "none":
                per = [O.prefill_rows(qh[j], kh[j], ub, pf.budget) for j in range(G)]
            else:
                rows = O.prefill_rows(qh, kh, ub, pf.budget, agg=agg)
                per = [rows] * G
            check = range(L) if check_rows is None else check_rows
            for j in range(G):
                s = u * G + j if agg == "none" else u
                for i in check:
                    got = pf.row_indices(s, i, hp)
                    assert np.array_equal(got, per[j][i]), (b, h, j, i, len(got), len(per[j][i]))
            if check_out:
                for j in range(G):
                    ref = O.attend_rows(qh[j], host["k"][b, h], host["v"][b, h], per[j])
                    err = np.abs(o[b, h * G + j] - ref).max() / np.abs(ref).max()
                    worst = max(worst, err)
    return worst


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_prefill_group_sizes(G):
    worst = _run(B=1, Hq=2 * G, Hkv=2, L=1024, top_k=4, agg="max", seed=G,
                 check_rows=range(0, 1024, 7))
    assert worst <= TOL_BF16, worst


@pytest.mark.parametrize("agg", ["mean", "none"])
def test_prefill_aggregations(agg):
    worst = _run(B=2, Hq=8, Hkv=2, L=768, top_k=3, agg=agg, seed=11,
                 check_rows=range(0, 768, 5))
    assert worst <= TOL_BF16, worst


@pytest.mark.parametrize("budget", [1, 2, 63, 64, 100, 257, 5000])
def test_prefill_budgets(budget):
    """Self only, cut chunks (K*64 and odd budgets), more than the context."""
    worst = _run(B=1, Hq=4, Hkv=1, L=640, budget=budget, agg="max", seed=budget,
                 check_rows=range(640))
    assert worst <= TOL_BF16, worst


def test_prefill_ragged_length():
    """L not a multiple of 64: the last chunk is short."""
    worst = _run(B=1, Hq=4, Hkv=1, L=1000, top_k=5, agg="max", seed=4, check_rows=range(1000))
    assert worst <= TOL_BF16, worst


@pytest.mark.parametrize("kind", ["ties", "int", "wide"])
def test_prefill_ties(kind):
    """Exact score ties (duplicated blocks / small integers): lower chunk
    index first, as the reference's stable argsort."""
    worst = _run(B=1, Hq=4, Hkv=1, L=512, top_k=3, agg="max", seed=9, kind=kind,
                 check_rows=range(512))
    assert worst <= TOL_BF16, worst


def test_prefill_4k_topk16():
    worst = _run(B=1, Hq=8, Hkv=2, L=4096, top_k=16, agg="max", seed=21,
                 check_rows=range(0, 4096, 31))
    assert worst <= TOL_BF16, worst


@pytest.mark.parametrize("L", [1, 40, 64, 65, 130])
def test_prefill_tiny_lengths(L):
    """A single (short) chunk, exactly one block, one block + 1 token."""
    worst = _run(B=1, Hq=4, Hkv=1, L=L, top_k=1, agg="max", seed=60 + L, check_rows=range(L))
    assert worst <= TOL_BF16, worst


@pytest.mark.parametrize("persistent", ["0", "1"])
def test_prefill_both_grids(persistent, monkeypatch):
    """The persistent plan-pulling grid and the one-CTA-per-plan grid give the
    same (exact) selections and in-tolerance outputs."""
    monkeypatch.setenv("DHSA_PREFILL_PERSISTENT", persistent)
    worst = _run(B=2, Hq=8, Hkv=2, L=1536, top_k=6, agg="max", seed=77,
                 check_rows=range(0, 1536, 11))
    assert worst <= TOL_BF16, worst


def test_prefill_mask_export_matches_reference_format(tmp_path):
    """GPU plan -> DHSAMSK1 bitsets: the file written from the device bitsets
    equals the file of the oracle's rows (the reference's format)."""
    from paper_2510_24606_b200 import serialization as S
    from paper_2510_24606_b200.prefill import SparsePrefill

    L, D = 700, 128
    t, host = _inputs(1, 4, 1, L, D, 81)
    pf = SparsePrefill(1, 4, 1, D, L, budget=150, agg="max")
    pf(t["q"].cuda(), t["k"].cuda(), t["v"].cuda())
    bits = pf.mask_bitsets()
    S.save_mask_bitsets(tmp_path / "gpu.msk", L, bits[0])
    rows = O.prefill_rows(host["q"][0], np.repeat(host["k"][0, 0][None], 4, axis=0),
                          O.static_grid(L, 64), pf.budget)

    class M:
        length = L

    m = M()
    m.rows = rows
    S.save_mask(tmp_path / "oracle.msk", m)
    assert (tmp_path / "gpu.msk").read_bytes() == (tmp_path / "oracle.msk").read_bytes()


@pytest.mark.parametrize("agg", ["max", "none"])
def test_mask_quality_matches_reference_metrics(agg):
    """GPU attention-mass recall and output cosine per row (dense run on the
    same tcgen05 kernel) vs the float64 restatement of the reference's
    harness metrics; the means are what attention_mass_recall /
    output_fidelity report."""
    from paper_2510_24606_b200.prefill import SparsePrefill, mask_quality

    B, Hq, Hkv, L, D = 1, 4, 1, 640, 128
    t, host = _inputs(B, Hq, Hkv, L, D, 91)
    pf = SparsePrefill(B, Hq, Hkv, D, L, top_k=2, agg=agg)
    rec, cos = mask_quality(t["q"].cuda(), t["k"].cuda(), t["v"].cuda(), pf)
    rec, cos = rec.cpu().numpy(), cos.cpu().numpy()
    bounds = O.static_grid(L, 64)
    kh = np.repeat(host["k"][0, 0][None], Hq, axis=0)
    shared = O.prefill_rows(host["q"][0], kh, bounds, pf.budget) if agg == "max" else None
    for h in range(Hq):
        rows = shared if shared is not None else O.prefill_rows(host["q"][0, h], kh[h], bounds,
                                                                pf.budget)
        r_ref, c_ref = O.mask_quality(host["q"][0, h], host["k"][0, 0], host["v"][0, 0], rows)
        assert np.abs(rec[0, h] - r_ref).max() <= 1e-2
        assert abs(rec[0, h].mean() - r_ref.mean()) <= 2e-3
        assert np.abs(cos[0, h] - c_ref).max() <= 1e-2
        assert abs(cos[0, h].mean() - c_ref.mean()) <= 2e-3


# ------------------------------------------- dynamic chunks (8f row 1) --

def _rand_bounds(rng, L, short=True, long=True):
    """Random boundary list mixing 1..63-token, 64-aligned and > 64-token
    chunks (up to 300 tokens)."""
    b, pos = [0], 0
    while pos < L:
        r = rng.random()
        if short and r < 0.35:
            n = int(rng.integers(1, 64))
        elif long and r < 0.7:
            n = int(rng.integers(65, 300))
        else:
            n = 64 * int(rng.integers(1, 3))
        pos = min(L, pos + n)
        b.append(pos)
    return b


@pytest.mark.parametrize("budget", [1, 50, 257, 700, 3000])
def test_prefill_dynamic_shared_bounds(budget):
    """One explicit boundary list (short, long and aligned chunks) for every
    unit: rows index-exact, outputs within tolerance."""
    rng = np.random.default_rng(budget)
    L = 1500
    worst = _run(B=1, Hq=4, Hkv=1, L=L, budget=budget, agg="max", seed=budget,
                 bounds=_rand_bounds(rng, L), check_rows=range(L))
    assert worst <= TOL_BF16, worst


@pytest.mark.parametrize("agg", ["max", "mean", "none"])
def test_prefill_dynamic_per_unit_bounds(agg):
    """A different boundary list per kv unit (B=2 x Hkv=2)."""
    rng = np.random.default_rng(5)
    L = 1200
    bounds = [_rand_bounds(rng, L) for _ in range(4)]
    worst = _run(B=2, Hq=8, Hkv=2, L=L, budget=400, agg=agg, seed=13, bounds=bounds,
                 check_rows=range(0, L, 3))
    assert worst <= TOL_BF16, worst


def test_prefill_dynamic_nms_bounds():
    """Boundaries from nms_boundaries over per-position scores (the paper's
    pipeline: predictor scores -> NMS -> chunks)."""
    from paper_2510_24606_b200.chunking import nms_boundaries

    rng = np.random.default_rng(8)
    L = 2048
    bounds = nms_boundaries(rng.random(L), min_conf=0.2, window=24, max_chunks=40)
    worst = _run(B=1, Hq=4, Hkv=1, L=L, budget=513, agg="max", seed=8, bounds=bounds,
                 check_rows=range(0, L, 2))
    assert worst <= TOL_BF16, worst


@pytest.mark.parametrize("case", ["one_chunk", "singletons", "ties"])
def test_prefill_dynamic_extremes(case):
    """One chunk of the whole sequence (diagonal blocks only, many query
    tiles), all-singleton chunks (one token each), and exact score ties over
    unequal chunks."""
    rng = np.random.default_rng(3)
    if case == "one_chunk":
        L, bounds, budget, kind = 1000, [0, 1000], 300, "normal"
    elif case == "singletons":
        L, bounds, budget, kind = 300, list(range(301)), 65, "normal"
    else:
        L, budget, kind = 768, 200, "ties"
        bounds = [0, 64, 128, 192, 250, 400, 401, 530, 768]
    worst = _run(B=1, Hq=4, Hkv=1, L=L, budget=budget, agg="max", seed=4, kind=kind,
                 bounds=bounds, check_rows=range(L))
    assert worst <= TOL_BF16, worst


@pytest.mark.parametrize("persistent", ["0", "1"])
def test_prefill_dynamic_both_grids(persistent, monkeypatch):
    monkeypatch.setenv("DHSA_PREFILL_PERSISTENT", persistent)
    rng = np.random.default_rng(21)
    L = 2000
    bounds = [_rand_bounds(rng, L) for _ in range(2)]
    worst = _run(B=1, Hq=8, Hkv=2, L=L, budget=600, agg="max", seed=21, bounds=bounds,
                 check_rows=range(0, L, 7))
    assert worst <= TOL_BF16, worst


def test_prefill_dynamic_mask_export():
    """Device bitsets of a dynamic-chunk plan equal the oracle rows."""
    from paper_2510_24606_b200 import serialization as S
    from paper_2510_24606_b200.prefill import SparsePrefill

    rng = np.random.default_rng(2)
    L = 700
    bounds = _rand_bounds(rng, L)
    t, host = _inputs(1, 4, 1, L, 128, 2)
    pf = SparsePrefill(1, 4, 1, 128, L, budget=150, agg="max", bounds=bounds)
    pf(t["q"].cuda(), t["k"].cuda(), t["v"].cuda())
    bits = pf.mask_bitsets().cpu().numpy()[0]
    rows = O.prefill_rows(host["q"][0], np.repeat(host["k"][0], 4, axis=0), bounds, 150)
    assert np.array_equal(bits, S.rows_to_bitsets(L, rows))


def test_mask_quality_dynamic_bounds():
    """Recall / cosine per row with an explicit boundary list."""
    from paper_2510_24606_b200.prefill import SparsePrefill, mask_quality

    rng = np.random.default_rng(17)
    B, Hq, Hkv, L, D = 1, 4, 1, 700, 128
    bounds = _rand_bounds(rng, L)
    t, host = _inputs(B, Hq, Hkv, L, D, 92)
    pf = SparsePrefill(B, Hq, Hkv, D, L, budget=150, agg="max", bounds=bounds)
    rec, cos = mask_quality(t["q"].cuda(), t["k"].cuda(), t["v"].cuda(), pf)
    rec, cos = rec.cpu().numpy(), cos.cpu().numpy()
    kh = np.repeat(host["k"][0, 0][None], Hq, axis=0)
    rows = O.prefill_rows(host["q"][0], kh, bounds, pf.budget)
    for h in range(Hq):
        r_ref, c_ref = O.mask_quality(host["q"][0, h], host["k"][0, 0], host["v"][0, 0], rows)
        assert np.abs(rec[0, h] - r_ref).max() <= 1e-2
        assert np.abs(cos[0, h] - c_ref).max() <= 1e-2


def test_predictor_nms_prefill_pipeline():
    """The paper's pipeline on the GPU: boundary predictor over each kv
    head's keys (fp64) -> nms_boundaries -> per-unit chunk lists -> sparse
    prefill; rows index-exact against the oracle on the same boundaries."""
    from paper_2510_24606_b200.chunking import nms_boundaries
    from paper_2510_24606_b200.predictor import boundary_scores, init_predictor

    L, Hkv = 1200, 2
    t, host = _inputs(1, 8, Hkv, L, 128, 23)
    params = init_predictor(128, window=4, heads=8, hidden=64, seed=3)
    bounds = [nms_boundaries(boundary_scores(host["k"][0, h], params), min_conf=0.05,
                             window=16, max_chunks=40) for h in range(Hkv)]
    assert all(len(b) > 3 for b in bounds)
    worst = _run(B=1, Hq=8, Hkv=Hkv, L=L, budget=300, agg="max", seed=23, bounds=bounds,
                 check_rows=range(0, L, 3))
    assert worst <= TOL_BF16, worst


def test_prefill_plan_capacity_refused():
    """Dynamic chunks so short that a walk of budget-1 tokens needs more plan
    entries than a CTA stages: refused with ValueError (no silently
    unwritten rows)."""
    from paper_2510_24606_b200.prefill import SparsePrefill

    L = 8192
    bounds = list(range(0, L, 2)) + [L]
    with pytest.raises(ValueError, match="plan"):
        SparsePrefill(1, 4, 1, 128, L, budget=4097, agg="max", bounds=bounds)
