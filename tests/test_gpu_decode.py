"""GPU parity of the batched decode engine (SparseDecoder) — the north-star
path — against the CPU oracle and the reference's golden C1 vectors.

Selections: bit-exact indices.  Outputs: max|o - o_ref| <= tol * max|o_ref|
per (sequence, q-head), tol = 2e-2 (bf16), 1e-5 (fp32), 1e-12 (fp64), against
the float64 reference row body (core.py:113-118)."""

import numpy as np
import pytest
import torch

import golden_io as G
from decode_harness import TOL, make_inputs, run_and_check, tiles_to_idx
from oracle import dhsa_oracle as O

pytestmark = pytest.mark.gpu


def _dec(**kw):
    from paper_2510_24606_b200.decode import SparseDecoder
    return SparseDecoder(**kw)


def test_c1_golden_fp32():
    """C1 demo shape (8 heads, d=64, L=4096, block 64, top-k 16) vs the
    reference's own DecodeSession rows and attention outputs."""
    gd = G.c1_golden()
    H, L, d, steps = gd["H"], gd["L"], gd["d"], gd["steps"]
    dec = _dec(batch=1, q_heads=H, kv_heads=H, head_dim=d, max_len=L + steps, block=64, top_k=16,
               dtype=torch.float32, agg="max")
    k = torch.from_numpy(gd["k"]).unsqueeze(0).cuda()
    v = torch.from_numpy(gd["v"]).unsqueeze(0).cuda()
    q = torch.from_numpy(gd["q"]).unsqueeze(0).cuda()
    dec.prefill(k[:, :, :L], v[:, :, :L])
    for s in range(steps):
        t = L + s
        out = dec.step(q[:, :, t].contiguous(), k[:, :, t].contiguous(), v[:, :, t].contiguous())
        sel = dec.selection()
        o = out.double().cpu().numpy()[0]
        for h in range(H):
            assert np.array_equal(tiles_to_idx(sel[h]), G.ranges_to_idx(gd["rows"][(h, s)], t))
            ref = gd["out"][h, s]
            assert np.abs(o[h] - ref).max() <= 1e-5 * np.abs(ref).max()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("agg", ["max", "mean", "none"])
def test_gqa_decode_small(dtype, agg):
    B, Hq, Hkv, D, P, steps = 2, 8, 2, 128, 1000, 5
    t, host = make_inputs(B, Hq, Hkv, D, P, steps, dtype, seed=1)
    dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
               top_k=4, dtype=dtype, agg=agg)
    worst = run_and_check(dec, t, host, P, steps, agg)
    assert worst <= TOL[dtype], worst


@pytest.mark.parametrize("budget", [1, 2, 63, 64, 65, 200, 257, 5000])
def test_budget_edge_cases_bf16(budget):
    """Budgets that cut chunks (K*64 and odd values), budget 1 (self only)
    and a budget above the context (everything kept)."""
    B, Hq, Hkv, D, P, steps = 1, 4, 1, 64, 700, 3
    t, host = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=2)
    dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
               budget=budget, dtype=torch.bfloat16, agg="max")
    worst = run_and_check(dec, t, host, P, steps, "max")
    assert worst <= 2e-2


@pytest.mark.parametrize("kind", ["int", "ties"])
def test_exact_ties(kind):
    """Integer-valued inputs: every fp64 score is exact, so ties between
    chunks are real and must resolve to the lower index."""
    B, Hq, Hkv, D, P, steps = 2, 4, 2, 64, 640, 4
    t, host = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=3, kind=kind)
    dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
               top_k=3, dtype=torch.bfloat16, agg="max")
    run_and_check(dec, t, host, P, steps, "max", check_out=False)


def test_long_generated_chunk():
    """The generated chunk grows past a block and competes in the walk."""
    B, Hq, Hkv, D, P, steps = 1, 4, 1, 128, 256, 150
    t, host = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=4)
    # make generated keys resemble the queries so the gen chunk is selected
    t["k"][:, :, P:] = t["q"][:, :1] * 2
    host["k"] = t["k"].to(torch.float64).numpy()
    dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
               budget=130, dtype=torch.bfloat16, agg="max")
    worst = run_and_check(dec, t, host, P, steps, "max")
    assert worst <= 2e-2


def test_ragged_prompt_and_dims():
    """Prompt not a multiple of the block; D=64 and group size 8."""
    B, Hq, Hkv, D, P, steps = 3, 8, 1, 64, 1234, 3
    t, host = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=5)
    dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
               top_k=5, dtype=torch.bfloat16, agg="max")
    assert run_and_check(dec, t, host, P, steps, "max") <= 2e-2


def test_c2_shape_sampled_units():
    """C2 shape (B=8, 32q/8kv, d=128, L=32K, block 64, top-k 64): every unit's
    selection exact, outputs checked on sampled units."""
    B, Hq, Hkv, D, P, steps = 8, 32, 8, 128, 32768, 2
    t, host = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=6)
    dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
               top_k=64, dtype=torch.bfloat16, agg="max")
    worst = run_and_check(dec, t, host, P, steps, "max", check_units=[0, 9, 35, 63])
    assert worst <= 2e-2


def test_step_graph_replay_matches_eager():
    """The four kernels of a step are CUDA-graph capturable; a replayed
    step gives the same selection and output as an eager one."""
    from paper_2510_24606_b200.decode import SparseDecoder
    B, Hq, Hkv, D, P = 2, 8, 2, 128, 2048
    t, _ = make_inputs(B, Hq, Hkv, D, P, 4, torch.bfloat16, seed=7)
    outs = []
    for mode in ("eager", "graph"):
        dec = SparseDecoder(B, Hq, Hkv, D, P + 4, top_k=8, dtype=torch.bfloat16)
        dec.prefill(t["k"][:, :, :P].cuda(), t["v"][:, :, :P].cuda())
        q = t["q"][:, :, 0].contiguous().cuda()
        kn = t["k"][:, :, P].contiguous().cuda()
        vn = t["v"][:, :, P].contiguous().cuda()
        out = torch.empty(B, Hq, D, dtype=torch.bfloat16, device="cuda")
        if mode == "eager":
            dec.launch(q, kn, vn, out)
        else:
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                dec.launch(q, kn, vn, out, stream=s)
            g.replay()
        torch.cuda.synchronize()
        outs.append((out.clone(), [x.copy() for x in dec.selection()]))
    assert torch.equal(outs[0][0], outs[1][0])
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("agg", ["max", "mean", "none"])
@pytest.mark.parametrize("kind", ["normal", "ties", "int", "outlier", "zeroq"])
def test_sketch_scoring_equals_fp64_scoring(agg, kind):
    """The bf16-sketch + certified-refinement selection is token-identical to
    streaming the fp64 centroids, including exact ties (duplicated blocks,
    integer data), an outlier chunk whose norm inflates the error bound, and
    an all-zero query (every score ties)."""
    from paper_2510_24606_b200.decode import SparseDecoder
    B, Hq, Hkv, D, P, steps = 2, 8, 2, 128, 3000, 6
    t, _ = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=11,
                       kind="ties" if kind == "ties" else ("int" if kind == "int" else "normal"))
    if kind == "outlier":
        t["k"][:, :, 640:704] *= 40
    if kind == "zeroq":
        t["q"][:, :, 1::2] = 0
    sels = []
    for scoring in ("sketch", "fp64"):
        dec = SparseDecoder(B, Hq, Hkv, D, P + steps, top_k=7, dtype=torch.bfloat16, agg=agg,
                            scoring=scoring)
        dec.prefill(t["k"][:, :, :P].cuda(), t["v"][:, :, :P].cuda())
        per = []
        for s in range(steps):
            out = dec.step(t["q"][:, :, s].contiguous().cuda(), t["k"][:, :, P + s].contiguous().cuda(),
                           t["v"][:, :, P + s].contiguous().cuda())
            per.append(([x.copy() for x in dec.selection()], out.clone()))
        sels.append(per)
    for (sa, oa), (sb, ob) in zip(*sels):
        for a, b in zip(sa, sb):
            assert np.array_equal(tiles_to_idx(a), tiles_to_idx(b))
        # the sketch path emits the certainly-kept chunks' tiles first (the
        # attention starts on them early), so the fp32 partial sums are
        # grouped differently: equal up to bf16 rounding
        oa, ob = oa.float(), ob.float()
        assert (oa - ob).abs().max() <= 1e-2 * ob.abs().max()


def test_sketch_c3_shape_sampled_units():
    """North-star shape (128K context, 32q/8kv, d=128, top-k 64) at batch 2:
    every unit's selection exact against the fp64 oracle, outputs in
    tolerance on sampled units."""
    B, Hq, Hkv, D, P, steps = 2, 32, 8, 128, 131072, 2
    t, host = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=12)
    dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
               top_k=64, dtype=torch.bfloat16, agg="max")
    assert dec.scoring == "sketch"
    worst = run_and_check(dec, t, host, P, steps, "max", check_units=list(range(16)),
                          check_out=True)
    assert worst <= 2e-2


@pytest.mark.parametrize("mode,hint", [("split", None), ("stream", None), ("stream", 2),
                                       ("stream", 1000)])
def test_attention_modes(mode, hint):
    """Persistent stream-K attention (any tiles_hint: too small hands the
    excess to the last segment, too large leaves idle slots) and the fixed
    split-KV kernel give the same, in-tolerance outputs."""
    B, Hq, Hkv, D, P, steps = 3, 16, 4, 128, 3000, 3
    t, host = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=17)
    dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
               top_k=8, dtype=torch.bfloat16, agg="max", attn_mode=mode)
    if hint is not None:
        dec.tiles_hint = hint
    worst = run_and_check(dec, t, host, P, steps, "max")
    assert worst <= TOL[torch.bfloat16], worst


def _random_bounds(rng, P, lo=1, hi=150):
    """Dynamic (NMS-like) boundaries: chunks of random length in [lo, hi]."""
    b = [0]
    while b[-1] < P:
        b.append(min(P, b[-1] + int(rng.integers(lo, hi + 1))))
    return b


@pytest.mark.parametrize("dtype,agg", [(torch.bfloat16, "max"), (torch.bfloat16, "none"),
                                       (torch.float32, "mean")])
def test_dynamic_boundaries(dtype, agg):
    """variable-length chunks (one boundary list per unit,
    short and longer-than-a-tile chunks) through the batched engine; every
    selection exact against DecodeSession semantics on the same bounds."""
    B, Hq, Hkv, D, P, steps = 2, 8, 2, 128, 2500, 4
    rng = np.random.default_rng(31)
    bounds = [_random_bounds(rng, P) for _ in range(B * Hkv)]
    t, host = make_inputs(B, Hq, Hkv, D, P, steps, dtype, seed=32)
    dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
               budget=700, dtype=dtype, agg=agg, max_chunks=max(len(b) for b in bounds))
    dec.prefill(t["k"][:, :, :P].cuda(), t["v"][:, :, :P].cuda(), bounds=bounds)
    G = Hq // Hkv
    oracles = {}
    for u in range(B * Hkv):
        b, h = divmod(u, Hkv)
        n = G if agg == "none" else 1
        oracles[u] = [O.DecodeOracle(host["k"][b, h, :P], bounds[u], dec.budget) for _ in range(n)]
    worst = 0.0
    for s in range(steps):
        pos = P + s
        out = dec.step(t["q"][:, :, s].contiguous().cuda(), t["k"][:, :, pos].contiguous().cuda(),
                       t["v"][:, :, pos].contiguous().cuda())
        torch.cuda.synchronize()
        sel = dec.selection()
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
                assert np.array_equal(tiles_to_idx(sel[u]), row), (s, u)
            for j in range(G):
                ref = O.attend_row(qh[j], host["k"][b, h, :pos + 1], host["v"][b, h, :pos + 1],
                                   rows[j])
                worst = max(worst, np.abs(o[b, h * G + j] - ref).max() / np.abs(ref).max())
    assert worst <= TOL[dtype], worst


def test_step_host_graph_equals_eager():
    """The serving entry point (host buffers, one captured CUDA graph reused
    for every step) gives bit-identical selections and outputs to eager steps."""
    B, Hq, Hkv, D, P, steps = 2, 8, 2, 128, 2000, 4
    t, _ = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=41)
    res = []
    for mode in ("eager", "graph"):
        dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
                   top_k=6, dtype=torch.bfloat16, agg="max")
        dec.prefill(t["k"][:, :, :P].cuda(), t["v"][:, :, :P].cuda())
        outs = []
        for s in range(steps):
            q = t["q"][:, :, s].contiguous()
            k = t["k"][:, :, P + s].contiguous()
            v = t["v"][:, :, P + s].contiguous()
            if mode == "eager":
                o = dec.step(q.cuda(), k.cuda(), v.cuda()).cpu()
            else:
                o = torch.empty(B, Hq, D, dtype=torch.bfloat16).pin_memory()
                dec.step_host(q.pin_memory(), k.pin_memory(), v.pin_memory(), o)
                torch.cuda.synchronize()
            outs.append((o.clone(), [x.copy() for x in dec.selection()]))
        res.append(outs)
    for (oa, sa), (ob, sb) in zip(*res):
        assert torch.equal(oa, ob)
        for a, b in zip(sa, sb):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("D,G,agg", [(64, 4, "max"), (64, 8, "none"), (128, 8, "max"),
                                     (128, 1, "max"), (64, 2, "mean")])
def test_bf16_head_dims_and_groups(D, G, agg):
    """bf16 sketch + stream attention across head dims {64, 128} and group
    sizes {1, 2, 4, 8} (template instantiations of every decode kernel)."""
    B, Hkv, P, steps = 2, 2, 1500, 3
    Hq = G * Hkv
    t, host = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=50 + D + G)
    dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
               top_k=5, dtype=torch.bfloat16, agg=agg)
    assert dec.scoring == "sketch" and dec.attn_mode == "stream"
    worst = run_and_check(dec, t, host, P, steps, agg)
    assert worst <= TOL[torch.bfloat16], worst


def test_step_host_packed_equals_eager():
    """One packed pinned [q|k|v] host buffer per step gives the eager results."""
    B, Hq, Hkv, D, P, steps = 2, 8, 2, 128, 1500, 3
    t, _ = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=43)
    res = []
    for mode in ("eager", "packed"):
        dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
                   top_k=5, dtype=torch.bfloat16, agg="max")
        dec.prefill(t["k"][:, :, :P].cuda(), t["v"][:, :, :P].cuda())
        outs = []
        for s in range(steps):
            q, k, v = (t[n][:, :, s if n == "q" else P + s].contiguous() for n in ("q", "k", "v"))
            if mode == "eager":
                o = dec.step(q.cuda(), k.cuda(), v.cuda()).cpu()
            else:
                qkv = torch.cat([q.reshape(-1), k.reshape(-1), v.reshape(-1)]).pin_memory()
                o = torch.empty(B, Hq, D, dtype=torch.bfloat16).pin_memory()
                dec.step_host_packed(qkv, o)
                torch.cuda.synchronize()
            outs.append(o.clone())
        res.append(outs)
    for a, b in zip(*res):
        assert torch.equal(a, b)


@pytest.mark.parametrize("P", [1, 63, 65])
def test_tiny_prompts(P):
    """One-token prompt (a single chunk of length 1), ragged last chunks."""
    B, Hq, Hkv, D, steps = 1, 4, 1, 128, 70  # the generated chunk outgrows a tile
    t, host = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=70 + P)
    dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P + steps, block=64,
               top_k=1, dtype=torch.bfloat16, agg="max")
    worst = run_and_check(dec, t, host, P, steps, "max")
    assert worst <= TOL[torch.bfloat16], worst


def test_step_host_after_second_prefill():
    """A decoder that already captured its step graph is prefilled again with
    a LONGER prompt and then with explicit (dynamic) bounds: the serving
    entry points re-capture and match eager steps bit for bit (the captured
    graph bakes in max_chunks and the bounds pointers)."""
    B, Hq, Hkv, D, steps = 2, 8, 2, 128, 3
    P1, P2 = 700, 1900
    t, _ = make_inputs(B, Hq, Hkv, D, P2, steps, torch.bfloat16, seed=44)
    rng = np.random.default_rng(5)
    dyn = _random_bounds(rng, P2, lo=8, hi=120)

    def run(mode, prompts):
        dec = _dec(batch=B, q_heads=Hq, kv_heads=Hkv, head_dim=D, max_len=P2 + steps,
                   block=64, top_k=5, dtype=torch.bfloat16, agg="max",
                   max_chunks=max(len(dyn), 64))
        outs = []
        for P, bounds in prompts:
            dec.prefill(t["k"][:, :, :P].cuda(), t["v"][:, :, :P].cuda(), bounds=bounds)
            for s in range(steps):
                q, k, v = (t[n][:, :, s if n == "q" else P + s].contiguous()
                           for n in ("q", "k", "v"))
                if mode == "eager":
                    o = dec.step(q.cuda(), k.cuda(), v.cuda()).cpu()
                elif mode == "host":
                    o = torch.empty(B, Hq, D, dtype=torch.bfloat16).pin_memory()
                    dec.step_host(q.pin_memory(), k.pin_memory(), v.pin_memory(), o)
                    torch.cuda.synchronize()
                else:
                    qkv = torch.cat([q.reshape(-1), k.reshape(-1), v.reshape(-1)]).pin_memory()
                    o = torch.empty(B, Hq, D, dtype=torch.bfloat16).pin_memory()
                    dec.step_host_packed(qkv, o)
                    torch.cuda.synchronize()
                outs.append((o.clone(), [x.copy() for x in dec.selection()]))
        return outs

    prompts = [(P1, None), (P2, None), (P2, dyn)]
    ref = run("eager", prompts)
    for mode in ("host", "packed"):
        got = run(mode, prompts)
        for (oa, sa), (ob, sb) in zip(ref, got):
            assert torch.equal(oa, ob), mode
            for a, b in zip(sa, sb):
                assert np.array_equal(a, b), mode


def test_static_prompt_longer_than_chunk_capacity():
    """A static-grid prompt whose chunk count exceeds the decoder's chunk
    capacity is refused (it would overwrite the next unit's centroids)."""
    dec = _dec(batch=1, q_heads=4, kv_heads=1, head_dim=128, max_len=100, block=16, top_k=2,
               dtype=torch.bfloat16, agg="max")
    k = torch.zeros(1, 1, 127, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="chunks"):
        dec.prefill(k, k, prompt_len=127)
