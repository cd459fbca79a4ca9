"""GPU parity of the sequence-sharded split-KV decode (config C4's path) on
one device: W shards driven in one process (SplitKVGroup — the collectives
become concatenations, every kernel is the multi-GPU one).  Selections must
equal the unsharded oracle walk index-for-index (global chunk ids carry the
reference tie-break across shard borders); outputs within 2e-2 (bf16) of the
float64 row body core.py:113-118."""

import numpy as np
import pytest
import torch

from decode_harness import TOL, make_inputs, tiles_to_idx
from oracle import dhsa_oracle as O

pytestmark = pytest.mark.gpu


def _run(W, B, Hq, Hkv, D, P, steps, top_k, agg, kind="normal", seed=0, budget=None,
         bounds=None):
    from paper_2510_24606_b200.splitkv import SplitKVGroup

    t, host = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=seed, kind=kind)
    if kind == "ties":  # identical blocks in the first and the last shard
        t["k"][:, :, P - 64:P] = t["k"][:, :, 0:64]
        host["k"] = t["k"].to(torch.float64).numpy()
    grp = SplitKVGroup(B, Hq, Hkv, D, P, W, block=64, top_k=top_k, budget=budget, agg=agg,
                       max_new=steps + 1, bounds=bounds)
    grp.prefill(t["k"][:, :, :P].cuda(), t["v"][:, :, :P].cuda())
    G = Hq // Hkv
    budget = grp.shards[0].budget
    if bounds is None:
        bounds = O.static_grid(P, 64)
    oracles = {}
    for u in range(B * Hkv):
        b, h = divmod(u, Hkv)
        n = G if agg == "none" else 1
        oracles[u] = [O.DecodeOracle(host["k"][b, h, :P], bounds, budget) for _ in range(n)]
    worst = 0.0
    for s in range(steps):
        pos = P + s
        out = grp.step(t["q"][:, :, s].contiguous().cuda(), t["k"][:, :, pos].contiguous().cuda(),
                       t["v"][:, :, pos].contiguous().cuda())
        torch.cuda.synchronize()
        for sh in grp.shards:
            sh.check_capacity()
        sel = grp.selection()
        o = out.double().cpu().numpy()
        for u in range(B * Hkv):
            b, h = divmod(u, Hkv)
            qh = host["q"][b, h * G:(h + 1) * G, s]
            kk = host["k"][b, h, pos]
            if agg == "none":
                rows = [oracles[u][j].step(qh[j], kk) for j in range(G)]
                for j in range(G):
                    assert np.array_equal(tiles_to_idx(sel[u * G + j]), rows[j]), (s, u, j)
            else:
                row = oracles[u][0].step_group(qh, kk, agg=agg)
                rows = [row] * G
                got = tiles_to_idx(sel[u])
                assert np.array_equal(got, row), (s, u, len(got), len(row))
            for j in range(G):
                ref = O.attend_row(qh[j], host["k"][b, h, :pos + 1], host["v"][b, h, :pos + 1],
                                   rows[j])
                err = np.abs(o[b, h * G + j] - ref).max() / np.abs(ref).max()
                worst = max(worst, err)
    return worst


@pytest.mark.parametrize("W", [1, 2, 3, 4])
def test_splitkv_matches_unsharded_walk(W):
    worst = _run(W, B=2, Hq=8, Hkv=2, D=128, P=4096, steps=4, top_k=8, agg="max")
    assert worst <= TOL[torch.bfloat16], worst


@pytest.mark.parametrize("agg", ["mean", "none"])
def test_splitkv_aggregations(agg):
    worst = _run(3, B=1, Hq=8, Hkv=2, D=128, P=3000, steps=3, top_k=4, agg=agg, seed=3)
    assert worst <= TOL[torch.bfloat16], worst


@pytest.mark.parametrize("kind", ["ties", "int"])
def test_splitkv_ties_cross_shard(kind):
    """Duplicated blocks in different shards (exact score ties): the global
    chunk id decides, as the reference's stable argsort does."""
    worst = _run(4, B=1, Hq=4, Hkv=1, D=64, P=2048, steps=3, top_k=6, agg="max", kind=kind,
                 seed=5)
    assert worst <= TOL[torch.bfloat16], worst


@pytest.mark.parametrize("budget", [1, 64, 100, 5000])
def test_splitkv_budget_edges(budget):
    """Self only, a cut chunk, and a budget larger than the context."""
    worst = _run(2, B=1, Hq=4, Hkv=1, D=128, P=1500, steps=3, top_k=1, agg="max",
                 budget=budget, seed=7)
    assert worst <= TOL[torch.bfloat16], worst


def test_splitkv_ragged_prompt():
    """Prompt length not a multiple of the block: the last shard's last chunk
    is short; 3 shards."""
    worst = _run(3, B=1, Hq=4, Hkv=1, D=128, P=3001, steps=3, top_k=5, agg="max", seed=9)
    assert worst <= TOL[torch.bfloat16], worst


def _dyn_bounds(seed, P):
    rng = np.random.default_rng(seed)
    b, pos = [0], 0
    while pos < P:
        pos = min(P, pos + int(rng.choice([int(rng.integers(1, 64)), int(rng.integers(64, 400))])))
        b.append(pos)
    return b


@pytest.mark.parametrize("W", [1, 2, 3])
def test_splitkv_dynamic_chunks(W):
    """Explicit boundary list (1..400-token chunks) cut at chunk starts over
    W shards: the global walk over candidates of any length equals the
    unsharded walk."""
    P = 3000
    worst = _run(W, B=1, Hq=8, Hkv=2, D=128, P=P, steps=3, top_k=8, agg="max", seed=W,
                 bounds=_dyn_bounds(W, P))
    assert worst <= TOL[torch.bfloat16], worst


def test_splitkv_dynamic_small_budget_many_chunks():
    """Many short chunks: the candidate capacity bound from the local chunk
    lengths (shortest chunks first) holds."""
    P = 1200
    b = list(range(0, 600, 5)) + list(range(600, 1200, 97)) + [1200]
    worst = _run(2, B=1, Hq=4, Hkv=1, D=128, P=P, steps=3, top_k=1, agg="max", budget=130,
                 seed=4, bounds=b)
    assert worst <= TOL[torch.bfloat16], worst
