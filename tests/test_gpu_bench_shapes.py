"""GPU parity at the benchmark's own shapes and on the kernel branches those
shapes execute (VERDICT r1 "parity at the bench's own shapes"):

* C5: 32K-token sparse prefill, 32 q / 8 kv heads, top-k 16..256 (budgets up
  to 16,385): sampled rows of sampled kv groups — diagonal-cut rows, chunk
  starts and ends, the first row that cannot keep every causal token —
  against the oracle chunk walk over the fp64 S_c (masks.py:125-150) and the
  float64 row body (core.py:113-118).
* C4: one shard holding 320K and 1M tokens (more than 4,915 chunks per unit:
  the 1024-thread certified select with global-memory scratch,
  decode_sketch.cu) and the 1M sequence over 8 shards (SplitKVGroup), against
  the unsharded DecodeOracle walk (masks.py:153-173, 205-237).
* The >1024-uncertain-chunk fallback of the certified select (a 64-bit radix
  select over the exact scores): zero queries and duplicated blocks at 128K.
* Adversarial near-ties at the certified sketch bound: a dense cluster of
  chunks whose exact fp64 scores straddle the cut within a few E.
* The C3 bench state: 1,500 decode steps (a ~1,500-token generated chunk)
  before the selection is checked.

Selections: bit-exact token indices.  Outputs: max|o - o_ref| <= 2e-2 *
max|o_ref| per (sequence, q head) (bf16).  Large inputs are generated on the
device; the oracle sees the same bf16 values upcast to float64, and the
attention reference gathers only the selected K/V rows."""

import os

import numpy as np
import pytest
import torch

from decode_harness import tiles_to_idx
from oracle import dhsa_oracle as O

pytestmark = pytest.mark.gpu

TOL = 2e-2


def _gen(seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return g


def _randn(shape, g, scale=1.0):
    return (torch.randn(*shape, device="cuda", generator=g) * scale).bfloat16()


def _host(t):
    return t.double().cpu().numpy()


def _attn_ref(q, K_dev, V_dev, idx):
    """core.py:113-118 on the selected rows only (gathered on the device)."""
    ii = torch.as_tensor(idx, device=K_dev.device)
    return O.attend_row(q, _host(K_dev[ii]), _host(V_dev[ii]), np.arange(len(idx)))


# ------------------------------------------------------------------ C5 ----

_C5 = {}


def _c5_setup():
    """One 32K sequence (Hq 32, Hkv 8, d 128) and the oracle S_c of the
    checked kv groups, shared by the top-k sweep."""
    if _C5:
        return _C5
    B, Hq, Hkv, D, L = 1, 32, 8, 128, 32768
    g = _gen(77)
    q, k, v = _randn((B, Hq, L, D), g), _randn((B, Hkv, L, D), g), _randn((B, Hkv, L, D), g)
    bounds = O.static_grid(L, 64)
    units = {}
    for h in (0, 5):
        kc = O.centroids(_host(k[0, h]), bounds)
        s = np.stack([O.chunk_scores(O.centroids(_host(q[0, h * 4 + j]), bounds), kc)
                      for j in range(4)])
        units[h] = s.max(axis=0)
    _C5.update(q=q, k=k, v=v, units=units, bounds=bounds, shape=(B, Hq, Hkv, D, L))
    return _C5


def _c5_rows(L, budget, rng):
    rows = {0, 1, 63, 64, 65, 127, 128, L - 1, L - 64, L - 65}
    for r in (budget - 2, budget - 1, budget, budget + 1, budget + 63, budget + 64):
        if 0 <= r < L:
            rows.add(r)
    for c in rng.integers(budget // 64, L // 64, size=24):
        rows.update({int(c) * 64, int(c) * 64 + 1, int(c) * 64 + 31, int(c) * 64 + 63})
    rows.update(int(x) for x in rng.integers(0, L, size=24))
    return sorted(r for r in rows if 0 <= r < L)


@pytest.mark.parametrize("top_k", [16, 32, 64, 128, 256])
def test_c5_32k_topk_sweep(top_k):
    from paper_2510_24606_b200.prefill import SparsePrefill

    st = _c5_setup()
    B, Hq, Hkv, D, L = st["shape"]
    pf = SparsePrefill(B, Hq, Hkv, D, L, top_k=top_k, agg="max")
    out = pf(st["q"], st["k"], st["v"])
    torch.cuda.synchronize()
    hp = pf.host_plans()
    rows = _c5_rows(L, pf.budget, np.random.default_rng(top_k))
    worst = 0.0
    for h, s in st["units"].items():
        for i in rows:
            l = i // 64
            want = O.ranges_to_indices(O.walk_ranges(s[l], st["bounds"], i, pf.budget), i)
            got = pf.row_indices(h, i, hp)
            assert np.array_equal(got, want), (top_k, h, i, len(got), len(want))
        for i in rows[::3]:
            want = pf.row_indices(h, i, hp)
            for j in range(4):
                qh = h * 4 + j
                ref = _attn_ref(_host(st["q"][0, qh, i]), st["k"][0, h], st["v"][0, h], want)
                o = _host(out[0, qh, i])
                worst = max(worst, np.abs(o - ref).max() / np.abs(ref).max())
    assert worst <= TOL, worst


# ---------------------------------------------------------- decode utils --

def _check_decode_step(sel, o, units, oracles, q_h, k_h, K, V, G, pos):
    """Compare one step on `units`: oracles[u] steps (state advanced)."""
    worst = 0.0
    for u in units:
        row = oracles[u].step_group(q_h[u], k_h[u], agg="max")
        got = tiles_to_idx(sel[u])
        assert np.array_equal(got, row), (u, pos, len(got), len(row))
        for j in range(G):
            ref = _attn_ref(q_h[u][j], K[u], V[u], row)
            worst = max(worst, np.abs(o[u * G + j] - ref).max() / np.abs(ref).max())
    return worst


# ------------------------------------------------------------------ C4 ----

@pytest.mark.parametrize("P,direct", [(327680, True), (1048576, True), (327680, False),
                                      (1048576, False)])
def test_c4_one_shard_wide_units(P, direct):
    """W=1 over 5,120 / 16,384 chunks per unit — the C4 bench's own path at
    1M: direct = the plain decode step (the 1024-thread compact select,
    17,408 chunks per CTA), else the split kernels (candidate-mode generic
    1024-thread select with global scratch, global walk, record merge)."""
    from paper_2510_24606_b200.splitkv import LocalComm, SplitKVShard

    B, Hq, Hkv, D, steps = 1, 32, 8, 128, 3
    G = Hq // Hkv
    sh = SplitKVShard(B, Hq, Hkv, D, P, rank=0, world=1, top_k=64, max_new=steps + 1,
                      direct=direct)
    assert sh.direct == direct
    g = _gen(P % 1000 + 1)
    d = sh.dec
    for t in (d.k_cache, d.v_cache):
        t[:, :, :P].normal_(generator=g)
    d.prefill(d.k_cache, d.v_cache, prompt_len=P)
    units = [0, 3, 7]
    bounds = O.static_grid(P, 64)
    oracles = {u: O.DecodeOracle(_host(d.k_cache[0, u, :P]), bounds, sh.budget) for u in units}
    comm = LocalComm()
    worst = 0.0
    for s in range(steps):
        q = _randn((B, Hq, D), g)
        kn, vn = _randn((B, Hkv, D), g), _randn((B, Hkv, D), g)
        out = sh.step(q, kn, vn, comm)
        torch.cuda.synchronize()
        sh.check_capacity()
        sel = sh.selection()
        qh = {u: _host(q[0, u * G:(u + 1) * G]) for u in units}
        kh = {u: _host(kn[0, u]) for u in units}
        worst = max(worst, _check_decode_step(
            sel, _host(out[0]), units, oracles, qh, kh,
            {u: d.k_cache[0, u] for u in units}, {u: d.v_cache[0, u] for u in units}, G, P + s))
    assert worst <= TOL, worst


def test_c4_1m_eight_shards():
    """The 1M-token sequence over 8 shards (SplitKVGroup: every kernel and
    the exchange layout of the 8-GPU run, collectives as concatenations)."""
    from paper_2510_24606_b200.splitkv import SplitKVGroup

    B, Hq, Hkv, D, P, W, steps = 1, 32, 8, 128, 1048576, 8, 2
    G = Hq // Hkv
    g = _gen(8)
    k, v = _randn((B, Hkv, P + steps, D), g), _randn((B, Hkv, P + steps, D), g)
    grp = SplitKVGroup(B, Hq, Hkv, D, P, W, top_k=64, max_new=steps + 1)
    grp.prefill(k[:, :, :P], v[:, :, :P])
    units = [1, 6]
    bounds = O.static_grid(P, 64)
    oracles = {u: O.DecodeOracle(_host(k[0, u, :P]), bounds, grp.shards[0].budget) for u in units}
    worst = 0.0
    for s in range(steps):
        q = _randn((B, Hq, D), g)
        kn, vn = k[:, :, P + s].contiguous(), v[:, :, P + s].contiguous()
        out = grp.step(q, kn, vn)
        torch.cuda.synchronize()
        for shd in grp.shards:
            shd.check_capacity()
        sel = [tiles for tiles in grp.selection()]
        qh = {u: _host(q[0, u * G:(u + 1) * G]) for u in units}
        kh = {u: _host(kn[0, u]) for u in units}
        worst = max(worst, _check_decode_step(
            sel, _host(out[0]), units, oracles, qh, kh,
            {u: k[0, u] for u in units}, {u: v[0, u] for u in units}, G, P + s))
    assert worst <= TOL, worst


# ------------------------------------------------- certified select edges --

def _uncertain_counts(dec, fn):
    """Run fn() with the select's debug record on; returns the uncertain
    (fp64 re-scored) chunk count per unit (decode_sketch.cu dbg[16u+15])."""
    dbg = torch.zeros(262144, dtype=torch.int64, device="cuda")
    os.environ["DHSA_DEBUG_TIMING"] = str(dbg.data_ptr())
    try:
        fn()
        torch.cuda.synchronize()
    finally:
        del os.environ["DHSA_DEBUG_TIMING"]
    return dbg[: dec.U * 16].view(dec.U, 16)[:, 15].cpu().numpy()


def _decode_case(k, v, qs, ks, vs, P, G, units=None, agg="max", top_k=64, count_unc=False):
    from paper_2510_24606_b200.decode import SparseDecoder

    B, Hkv = k.shape[0], k.shape[1]
    D = k.shape[3]
    steps = qs.shape[0]
    dec = SparseDecoder(B, Hkv * G, Hkv, D, P + steps, block=64, top_k=top_k,
                        dtype=torch.bfloat16, agg=agg)
    assert dec.scoring == "sketch"
    dec.prefill(k[:, :, :P], v[:, :, :P])
    units = list(range(B * Hkv)) if units is None else units
    bounds = O.static_grid(P, 64)
    oracles = {u: O.DecodeOracle(_host(k[u // Hkv, u % Hkv, :P]), bounds, dec.budget)
               for u in units}
    unc = []
    worst = 0.0
    for s in range(steps):
        out = torch.empty(B, Hkv * G, D, dtype=torch.bfloat16, device="cuda")
        run = lambda: dec.step(qs[s], ks[s], vs[s], out=out)  # noqa: E731
        if count_unc:
            unc.append(_uncertain_counts(dec, run))
        else:
            run()
        torch.cuda.synchronize()
        sel = dec.selection()
        o = _host(out).reshape(B * Hkv * G, D)
        qh = {u: _host(qs[s][u // Hkv, (u % Hkv) * G:(u % Hkv + 1) * G]) for u in units}
        kh = {u: _host(ks[s][u // Hkv, u % Hkv]) for u in units}
        Kd = {u: dec.k_cache[u // Hkv, u % Hkv] for u in units}
        Vd = {u: dec.v_cache[u // Hkv, u % Hkv] for u in units}
        worst = max(worst, _check_decode_step(sel, o, units, oracles, qh, kh, Kd, Vd, G, P + s))
    return worst, unc


@pytest.mark.parametrize("case", ["zero_query", "duplicated_blocks", "three_patterns"])
def test_radix_fallback_at_128k(case):
    """More than 1,024 chunks within the certified band: every score ties
    (zero query; every block identical), so the select's exact 64-bit radix
    fallback decides (ties to the lower chunk index, masks.py:119 stable
    argsort); three distinct blocks put one ~680-chunk tie class at the cut
    (the exact rank walk over a large uncertain set)."""
    B, Hkv, G, D, P, steps = 1, 2, 4, 128, 131072, 2
    g = _gen(11)
    k, v = _randn((B, Hkv, P + steps, D), g), _randn((B, Hkv, P + steps, D), g)
    if case == "duplicated_blocks":
        k[:, :, :P] = k[:, :, :64].repeat(1, 1, P // 64, 1)
    elif case == "three_patterns":
        pick = torch.randint(0, 3, (P // 64,), generator=torch.Generator().manual_seed(3))
        blocks = k[:, :, :192].view(B, Hkv, 3, 64, D)
        k[:, :, :P] = blocks[:, :, pick.cuda()].reshape(B, Hkv, P, D)
    qs = _randn((steps, B, Hkv * G, D), g)
    if case == "zero_query":
        qs.zero_()
    ks = k[:, :, P:P + steps].permute(2, 0, 1, 3).contiguous()
    vs = v[:, :, P:P + steps].permute(2, 0, 1, 3).contiguous()
    worst, unc = _decode_case(k, v, qs, ks, vs, P, G, count_unc=True)
    if case == "three_patterns":  # one ~680-chunk tie class at the cut: exact rank walk
        assert min(int(x.min()) for x in unc) > 300, unc
    else:  # every chunk in the band: the radix fallback ran
        assert min(int(x.min()) for x in unc) > 1024, unc
    assert worst <= TOL, worst


@pytest.mark.parametrize("agg", ["max", "none"])
def test_certified_bound_near_ties(agg):
    """A dense cluster of 120 chunks whose exact fp64 scores lie within +-4E
    of one value (E = the select's certified sketch error bound), with the
    selection cut in the middle of the cluster and per-chunk sketch rounding
    errors that differ: chunks 0.5E .. 4E from the cut and from each other
    must be re-scored and ordered exactly (group max, and per-head rows)."""
    from paper_2510_24606_b200.decode import SparseDecoder

    B, Hkv, G, D, P = 1, 1, 4, 128, 131072
    g = _gen(21)
    k = _randn((B, Hkv, P + 1, D), g)
    v = _randn((B, Hkv, P + 1, D), g)
    q = _randn((B, Hkv * G, D), g)
    q[:, 1:] = q[:, :1]  # equal heads: the cluster is a cluster for every head
    q[:, :, 0] = 1.0
    kc = k[0, 0, :P].view(P // 64, 64, D)
    # dim 0 of every token of a chunk is one bf16 value a: the chunk's exact
    # score is its dims-1.. score + 8 a q0 (centroid = sum / sqrt(64))
    kc[:, :, 0] = 0
    bounds = O.static_grid(P, 64)
    s = O.centroids(_host(k[0, 0, :P]), bounds) @ _host(q[0, 0])
    order = np.argsort(-s, kind="stable")
    # E in score units, as the select computes it (sinfo of a built sketch)
    probe = SparseDecoder(B, G, Hkv, D, P + 1, top_k=64, dtype=torch.bfloat16, agg="max")
    probe.prefill(k[:, :, :P], v[:, :, :P])
    kexp, cmax, dmax = probe.sinfo[0, :3].tolist()
    del probe
    qn = float(np.linalg.norm(_host(q[0, 0])))
    E = 1.01 * (qn * dmax + (2 ** -14 + 1e-6) * qn * cmax) / 2.0 ** (-kexp)
    # chunks ranked 4..123 retargeted into [T - 4E, T + 4E], T above every
    # other chunk but the top 4: the 64th largest score (the cut) falls in
    # the middle of the cluster
    cluster = order[4:124]
    T = s[order[130]] + 10 * E
    rng = np.random.default_rng(4)
    targets = T + E * rng.uniform(-4.0, 4.0, size=len(cluster))
    a = torch.from_numpy(((targets - s[cluster]) / 8.0).astype(np.float32)).cuda().bfloat16()
    kc[torch.as_tensor(cluster, device="cuda"), :, 0] = a[:, None]
    s2 = O.centroids(_host(k[0, 0, :P]), bounds) @ _host(q[0, 0])
    cut = np.sort(s2)[::-1][63]
    assert np.sort(np.abs(s2 - cut))[40] < 2 * E  # the cut sits inside the cluster
    qs = q[None]
    ks = k[:, :, P:P + 1].permute(2, 0, 1, 3).contiguous()
    vs = v[:, :, P:P + 1].permute(2, 0, 1, 3).contiguous()
    if agg == "max":
        worst, unc = _decode_case(k, v, qs, ks, vs, P, G, agg="max", count_unc=True)
        assert int(unc[0][0]) >= 20, unc  # many chunks re-scored in fp64
        assert worst <= TOL, worst
        return
    dec = SparseDecoder(B, G, Hkv, D, P + 1, top_k=64, dtype=torch.bfloat16, agg="none")
    dec.prefill(k[:, :, :P], v[:, :, :P])
    unc = _uncertain_counts(dec, lambda: dec.step(qs[0], ks[0], vs[0]))
    assert int(unc[0]) >= 20, unc
    sel = dec.selection()
    for j in range(G):
        ora = O.DecodeOracle(_host(k[0, 0, :P]), bounds, dec.budget)
        want = ora.step(_host(q[0, j]), _host(ks[0][0, 0]))
        assert np.array_equal(tiles_to_idx(sel[j]), want), j


@pytest.mark.parametrize("pattern", ["gauss", "cancel", "spread"])
def test_sketch_accumulation_error_model(pattern):
    """The certified bound (decode_sketch.cu) models the
    tensor-core score of a sketch row as |s'' - sum_d c''_d q_d| <= gamma *
    sum_d |c''_d q_d| with gamma = 2^-14 + 1e-6 (fp16 x bf16 products exact
    in fp32, fp32 accumulation inside mma.sync).  Checked on the hardware,
    chunk by chunk and head by head, against the exact float64 dot products
    of the very fp16 sketch rows and bf16 queries the kernel read: Gaussian
    rows, rows whose products cancel exactly (every bit of the result is
    accumulation error), and products spread over 2^-20 .. 2^0 with random
    signs (alignment / truncation stress)."""
    from paper_2510_24606_b200.decode import SparseDecoder

    B, Hkv, G, D, nch = 1, 1, 4, 128, 512
    P = 64 * nch
    rng = np.random.default_rng({"gauss": 1, "cancel": 2, "spread": 3}[pattern])
    if pattern == "gauss":
        t = rng.standard_normal((nch, D))
        qh = rng.standard_normal((G, D))
    elif pattern == "cancel":
        # half the dims +a, the other half -a permuted: the exact sum is 0
        mag = 2.0 ** rng.integers(-10, 1, size=(nch, D // 2)) * rng.uniform(1, 2, size=(nch, D // 2))
        t = np.concatenate([mag, -mag], axis=1)
        qh = np.ones((G, D))
        for j in range(nch):  # the same bf16 values, the cancelling halves interleaved
            t[j] = t[j][rng.permutation(D)]
    else:
        t = (2.0 ** rng.integers(-20, 1, size=(nch, D)) * rng.uniform(1, 2, size=(nch, D))
             * rng.choice([-1.0, 1.0], size=(nch, D)))
        qh = (2.0 ** rng.integers(-6, 1, size=(G, D)) * rng.choice([-1.0, 1.0], size=(G, D)))
    tb = torch.from_numpy(t).float().bfloat16()
    k = tb.repeat_interleave(64, dim=0).view(B, Hkv, P, D).cuda()  # centroid = 8 t exactly
    k = torch.cat([k, torch.zeros(B, Hkv, 1, D, dtype=torch.bfloat16, device="cuda")], dim=2)
    v = torch.zeros_like(k)
    q = torch.from_numpy(qh).float().bfloat16().view(B, Hkv * G, D).cuda()
    dec = SparseDecoder(B, G, Hkv, D, P + 1, top_k=64, dtype=torch.bfloat16, agg="none")
    dec.prefill(k[:, :, :P], v[:, :, :P])
    dec.step(q, k[:, :, P].contiguous(), v[:, :, P].contiguous())
    torch.cuda.synchronize()
    sk = dec.sketch[0, 0, :nch].double().cpu().numpy()       # c'' (fp16, exact)
    qd = q[0].double().cpu().numpy()                          # q (bf16, exact)
    approx = dec.approx[:G, :nch].double().cpu().numpy()     # s'' per (head, chunk)
    exact = qd @ sk.T
    absum = np.abs(qd) @ np.abs(sk).T
    gamma = 2.0 ** -14 + 1e-6
    ratio = np.abs(approx - exact) / np.maximum(absum, 1e-300)
    assert np.isfinite(approx).all()
    print(f"{pattern}: max accumulation error / sum|p| = {ratio.max():.3e} (gamma {gamma:.3e})")
    assert (np.abs(approx - exact) <= gamma * absum).all(), (
        f"{pattern}: accumulation error {ratio.max():.3e} x sum|p| exceeds gamma {gamma:.3e}")


# ------------------------------------------------------------------ C3 ----

def test_c3_state_after_1500_steps():
    """The bench's decode state: a 128K prompt followed by 1,500 generated
    tokens (one ~1,500-token generated chunk, masks.py:159-163), selection
    and output checked on the last steps."""
    B, Hkv, G, D, P, steps, check = 2, 2, 4, 128, 131072, 1500, 3
    from paper_2510_24606_b200.decode import SparseDecoder

    g = _gen(31)
    dec = SparseDecoder(B, Hkv * G, Hkv, D, P + steps + 1, top_k=64, dtype=torch.bfloat16,
                        agg="max")
    for t in (dec.k_cache, dec.v_cache):
        t[:, :, :P].normal_(generator=g)
    dec.prefill(dec.k_cache, dec.v_cache, prompt_len=P)
    bounds = O.static_grid(P, 64)
    units = list(range(B * Hkv))
    oracles = {u: O.DecodeOracle(_host(dec.k_cache[u // Hkv, u % Hkv, :P]), bounds, dec.budget)
               for u in units}
    qs = _randn((steps, B, Hkv * G, D), g)
    ks, vs = _randn((steps, B, Hkv, D), g), _randn((steps, B, Hkv, D), g)
    out = torch.empty(B, Hkv * G, D, dtype=torch.bfloat16, device="cuda")
    for s in range(steps - check):
        dec.step(qs[s], ks[s], vs[s], out=out)
    kh_all = _host(ks[: steps - check])
    for u in units:  # the oracle's running sum, one add per step in token order
        for s in range(steps - check):
            oracles[u].gen_sum += kh_all[s, u // Hkv, u % Hkv]
        oracles[u].gen_count = steps - check
    worst = 0.0
    for s in range(steps - check, steps):
        dec.step(qs[s], ks[s], vs[s], out=out)
        torch.cuda.synchronize()
        sel = dec.selection()
        o = _host(out).reshape(B * Hkv * G, D)
        qh = {u: _host(qs[s][u // Hkv, (u % Hkv) * G:(u % Hkv + 1) * G]) for u in units}
        kh = {u: _host(ks[s][u // Hkv, u % Hkv]) for u in units}
        Kd = {u: dec.k_cache[u // Hkv, u % Hkv] for u in units}
        Vd = {u: dec.v_cache[u // Hkv, u % Hkv] for u in units}
        worst = max(worst, _check_decode_step(sel, o, units, oracles, qh, kh, Kd, Vd, G, P + s))
    assert worst <= TOL, worst
