"""Shared driver for decode parity: runs SparseDecoder and the CPU oracle on
the same seeded inputs (rounded to the cache dtype, upcast for the oracle)
and compares selections (exact) and outputs (stated tolerance)."""

import numpy as np
import torch

from oracle import dhsa_oracle as O

TOL = {torch.bfloat16: 2e-2, torch.float32: 1e-5, torch.float64: 1e-12}


def tiles_to_idx(tiles):
    parts = [np.arange(s, s + c) for s, c in tiles]
    return np.sort(np.concatenate(parts)).astype(np.int64)


def make_inputs(B, Hq, Hkv, D, P, steps, dtype, seed=0, kind="normal"):
    rng = np.random.default_rng(seed)

    def draw(*shape):
        if kind == "int":
            return rng.integers(-3, 4, size=shape).astype(np.float32)
        if kind == "ties":
            return rng.integers(-1, 2, size=shape).astype(np.float32)
        return rng.standard_normal(shape, dtype=np.float32)

    k = draw(B, Hkv, P + steps, D)
    v = draw(B, Hkv, P + steps, D)
    q = draw(B, Hq, steps, D)  # queries of the decoded tokens only
    if kind == "ties":  # duplicated blocks: exact score ties between chunks
        k[:, :, 64:128] = k[:, :, 0:64]
    t = {n: torch.from_numpy(np.ascontiguousarray(a)).to(dtype) for n, a in
         dict(k=k, v=v, q=q).items()}
    host = {n: x.to(torch.float64).numpy() for n, x in t.items()}
    return t, host


def run_and_check(dec, t, host, P, steps, agg, check_units=None, check_out=True):
    """Prefill + `steps` decode steps; compare every step on `check_units`."""
    B, Hq, Hkv, D, G = dec.B, dec.Hq, dec.Hkv, dec.D, dec.G
    dev = dec.dev
    dec.prefill(t["k"][:, :, :P].to(dev), t["v"][:, :, :P].to(dev))
    units = range(B * Hkv) if check_units is None else check_units
    bounds = O.static_grid(P, dec.block)
    oracles = {}
    for u in units:
        b, h = divmod(u, Hkv)
        if agg == "none":
            oracles[u] = [O.DecodeOracle(host["k"][b, h, :P], bounds, dec.budget) for _ in range(G)]
        else:
            oracles[u] = O.DecodeOracle(host["k"][b, h, :P], bounds, dec.budget)
    worst = 0.0
    for s in range(steps):
        pos = P + s
        q = t["q"][:, :, s].contiguous().to(dev)
        kn = t["k"][:, :, pos].contiguous().to(dev)
        vn = t["v"][:, :, pos].contiguous().to(dev)
        out = dec.step(q, kn, vn)
        torch.cuda.synchronize()
        sel = dec.selection()
        o = out.to(torch.float64).cpu().numpy()
        for u in units:
            b, h = divmod(u, Hkv)
            qh = host["q"][b, h * G:(h + 1) * G, s]
            kk = host["k"][b, h, pos]
            if agg == "none":
                rows = [oracles[u][j].step(qh[j], kk) for j in range(G)]
                for j in range(G):
                    got = tiles_to_idx(sel[u * G + j])
                    assert np.array_equal(got, rows[j]), (s, u, j)
            else:
                row = oracles[u].step_group(qh, kk, agg=agg)
                rows = [row] * G
                got = tiles_to_idx(sel[u])
                assert np.array_equal(got, row), (s, u, len(got), len(row))
            if check_out:
                for j in range(G):
                    ref = O.attend_row(qh[j], host["k"][b, h, :pos + 1], host["v"][b, h, :pos + 1],
                                       rows[j])
                    err = np.abs(o[b, h * G + j] - ref).max() / np.abs(ref).max()
                    worst = max(worst, err)
    return worst
