#!/usr/bin/env python
"""Benchmark of the DHSA decode hot path on B200 (BASELINE.json metric:
"decode tokens/sec and us/step at 128K ctx; achieved HBM GB/s vs roofline").

Workload (BASELINE.json configs[2], "C3"): Llama-3-8B-shaped attention, 32 q /
8 kv heads, d=128, a 131,072-token prompt per sequence, 64-token blocks, top-k
64 (reference budget 64*64+1 = 4097 tokens), batch 32 sequences per GPU, bf16
KV cache, group-shared (max over the 4 q-heads of a kv group) selection.
A step = one decode token for every sequence: scores over all centroids,
exact Top-K chunk walk, sparse attention, state update.  Synthetic N(0,1)
inputs; the per-step working set (~1.07 GB) is far larger than L2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
  python bench.py --impl reference ...   # the reference algorithm on host cores

Multi-GPU (torchrun, one process per GPU; ``--gpus N`` without WORLD_SIZE
launches the N ranks itself): C3 shards the HEADS of the 32-sequence batch
(configs[2]: "heads sharded across 1/2/4/8 B200"): rank r serves kv heads
[r*8/N, (r+1)*8/N) and their 4 q heads each, so the whole job is the same
32 tokens per step ("scaling": "strong", value = 32 tokens / max-over-ranks
step time).  (sequence, kv head) units are independent: no collective on the
data path.  ``--shard batch`` gives every rank its own full batch instead
(weak scaling).  ``--rank-proxy N`` times rank 0's share of an N-GPU
heads-sharded job on one GPU (every rank has the same shape and no
communication, so that is the N-GPU step time).
"""

from __future__ import annotations

import os

# the CPU baseline runs one single-threaded process per core
for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse
import json
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (B, Hq, Hkv, D, L, block, top_k, dtype)
    "C1": (1, 8, 8, 64, 4096, 64, 16, "float32"),
    "C2": (8, 32, 8, 128, 32768, 64, 64, "bfloat16"),
    "C3": (32, 32, 8, 128, 131072, 64, 64, "bfloat16"),
    "C4": (1, 32, 8, 128, 1048576, 64, 64, "bfloat16"),
}
METRIC = "decode tokens/sec and us/step at 128K ctx; achieved HBM GB/s vs roofline"
FALLBACK_HBM = 6650.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def workload_desc(name):
    B, Hq, Hkv, D, L, blk, K, dt = CONFIGS[name]
    return (f"{name} decode: B={B} sequences, Hq={Hq}, Hkv={Hkv}, d={D}, context={L}, "
            f"block={blk}, top_k={K} (budget {K * blk + 1} tokens), {dt} KV, "
            f"group-shared max selection")


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:
                time.sleep(0.02)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({n for r in self.rows for n, v in zip(self.NAMES, r[2:])
                          if v.strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------ CPU baseline --
def _cpu_unit(args):
    """One (sequence, kv-group) unit of the workload through the reference
    algorithm restated in oracle/ (repeat + stable argsort selection,
    masks.py:153-173 / :103-122, and the core.py:113-118 row body for each
    of the G q-heads).  Returns seconds per step (centroid build excluded)."""
    seed, L, D, G, block, budget, steps = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import dhsa_oracle as O

    rng = np.random.default_rng(seed)
    k = rng.standard_normal((L + steps, D), dtype=np.float32).astype(np.float64)
    v = rng.standard_normal((L + steps, D), dtype=np.float32).astype(np.float64)
    q = rng.standard_normal((steps, G, D), dtype=np.float32).astype(np.float64)
    sess = O.DecodeOracle(k[:L], O.static_grid(L, block), budget)
    t0 = time.perf_counter()
    for s in range(steps):
        row = sess.step_group(q[s], k[L + s], agg="max", method="token")
        for j in range(G):
            O.attend_row(q[s, j], k[: L + s + 1], v[: L + s + 1], row)
    return (time.perf_counter() - t0) / steps


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available():
    """The unmodified reference package installed by tools/install_reference.sh."""
    return os.path.isdir(os.path.join(REF_DIR, "dhsa"))


def _ref_unit(args):
    """One (sequence, kv-group) unit of the workload through the UNMODIFIED
    reference package (baseline/_ref/dhsa): DecodeSession.__init__ builds the
    centroid cache (aggregate_rows, chunk_repr.py:57-68; one-time, excluded),
    then per step the reference's own decode-row composition (masks.py:153-173)
    with the group-shared max of harness.aggregated_chunk_scores
    (harness.py:288-306): scores of the G q-heads against [cached centroids |
    gen_sum/sqrt(g) | aggregate_chunk(k)], max over heads, np.repeat over
    extend_for_decode lengths, masks.topk_row; then the dense_attention row
    body (core.py:115-118, softmax_row) for each of the G heads, and the
    running-sum update of DecodeSession.step (masks.py:235-236).
    Returns seconds per step."""
    seed, L, D, G, block, budget, steps = args
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from dhsa import DecodeSession, aggregate_chunk, extend_for_decode, softmax_row, \
        static_boundaries, topk_row

    rng = np.random.default_rng(seed)
    k = rng.standard_normal((L + steps, D), dtype=np.float32).astype(np.float64)
    v = rng.standard_normal((L + steps, D), dtype=np.float32).astype(np.float64)
    q = rng.standard_normal((steps, G, D), dtype=np.float32).astype(np.float64)
    sess = DecodeSession(k[:L], static_boundaries(L, block), budget)
    inv = 1.0 / np.sqrt(D)
    t0 = time.perf_counter()
    for s in range(steps):
        g = sess._gen_count
        total = L + g + 1
        parts = [sess.cached_chunk_keys]
        if g >= 1:
            parts.append((sess._gen_sum / np.sqrt(g))[None, :])
        parts.append(aggregate_chunk(k[L + s][None, :])[None, :])
        chunk_keys = np.concatenate(parts, axis=0)
        scores = np.einsum("hd,jd->hj", q[s], chunk_keys).max(axis=0)
        lens = np.diff(np.asarray(extend_for_decode(sess.prompt_bounds, total), dtype=np.intp))
        idx = topk_row(np.repeat(scores, lens), total - 1, budget)
        for j in range(G):
            sc = np.einsum("jd,d->j", k[idx], q[s, j]) * inv
            softmax_row(sc) @ v[idx]
        sess._gen_sum += k[L + s]
        sess._gen_count += 1
    return (time.perf_counter() - t0) / steps


def cpu_baseline(name, units_sample=None, steps=2, workers=None, shape=None):
    """The reference decode step on the host cores, one single-threaded
    process per core over independent (sequence, kv-group) units.  Uses the
    unmodified reference package (kind "reference") when baseline/_ref holds
    it, else the oracle port (kind "port").  ``shape`` overrides the
    (B, Hq, Hkv) of the config (a rank's share of a heads-sharded job)."""
    import multiprocessing as mp

    B, Hq, Hkv, D, L, blk, K, _ = CONFIGS[name]
    if shape is not None:
        B, Hq, Hkv = shape
    G = Hq // Hkv
    workers = workers or min(32, os.cpu_count() or 1)  # ~0.4 GB of host RAM per unit
    units_total = B * Hkv
    n = units_sample or min(units_total, max(workers, 8))
    n = min(n, units_total)
    use_ref = reference_available()
    fn = _ref_unit if use_ref else _cpu_unit
    args = [(1000 + i, L, D, G, blk, K * blk + 1, steps) for i in range(n)]
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(min(workers, n)) as pool:
        per_unit = pool.map(fn, args)
    wall = time.perf_counter() - t0
    per_unit_s = float(np.mean(per_unit))
    used = min(workers, n)
    # whole-batch step time with `used` cores working on independent units
    step_s = per_unit_s * units_total / used
    what = ("the unmodified reference package (baseline/_ref/dhsa: DecodeSession cache, "
            "extend_for_decode + np.repeat + masks.topk_row select over the head-max scores, "
            f"softmax_row attention rows for {G} heads)" if use_ref else
            "oracle/dhsa_oracle.py reference formulation (repeat + stable argsort "
            f"select, fp64 row attention for {G} heads)")
    return {
        "value": B / step_s, "unit": "tokens/s", "cores": used,
        "kind": "reference" if use_ref else "port",
        "us_per_step": step_s * 1e6,
        "sample": (f"{n} of {units_total} (sequence, kv-group) units x {steps} steps of {name}, "
                   f"{what}, {used} processes; "
                   f"{per_unit_s * 1e3:.1f} ms per unit-step, scaled to {units_total} units; "
                   f"wall {wall:.1f}s incl. setup"),
    }


def _c5_ref_head(args):
    """One head of the C5 prefill through the reference at length L
    (BASELINE.md section 2): prefill_mask (masks.py:143-150, timed whole) and
    the dense_attention row body (core.py:113-118) on `rows_sample` rows
    spread over the sequence, scaled to all L rows.  Returns (mask_s,
    attn_s)."""
    L, D, budget, rows_sample, seed = args
    use_ref = reference_available()
    rng = np.random.default_rng(seed)
    import torch

    q, k, v = (torch.from_numpy(rng.standard_normal((L, D), dtype=np.float32)).bfloat16()
               .double().numpy() for _ in range(3))
    if use_ref:
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from dhsa import TokenSequence, prefill_mask, softmax_row, static_boundaries

        seq = TokenSequence(q, k, v)
        t0 = time.perf_counter()
        rows = prefill_mask(seq, static_boundaries(L, 64), budget).rows
        mask_s = time.perf_counter() - t0
    else:
        from oracle import dhsa_oracle as O

        t0 = time.perf_counter()
        rows = O.prefill_rows(q, k, O.static_grid(L, 64), budget)
        mask_s = time.perf_counter() - t0
        softmax_row = None
    inv = 1.0 / np.sqrt(D)
    pick = np.linspace(0, L - 1, rows_sample).astype(np.int64)
    t0 = time.perf_counter()
    for i in pick:
        idx = np.unique(np.asarray(rows[i], dtype=np.intp))  # _mask_rows, core.py:80-95
        sc = np.einsum("jd,d->j", k[idx], q[i]) * inv
        if softmax_row is not None:
            softmax_row(sc) @ v[idx]
        else:
            e = np.exp(sc - sc.max())
            (e / e.sum()) @ v[idx]
    attn_s = (time.perf_counter() - t0) / rows_sample * L
    return mask_s, attn_s


def cpu_baseline_c5(Hq=32, Hkv=8, D=128, L=32768, top_k=64):
    """C5 on the host: one head at 8K and at 16K
    tokens, in two concurrent single-threaded processes; the mask time is
    extrapolated to 32K with the measured 8K -> 16K growth exponent, the
    attention linearly (rows past the budget each cost `budget` keys).  The
    32K sequence = Hkv group-shared masks + Hq attention heads, spread over
    the host cores (independent heads)."""
    import multiprocessing as mp

    budget = top_k * 64 + 1
    lens = (8192, 16384)
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(2) as pool:
        res = pool.map(_c5_ref_head, [(n, D, budget, 512, 5 + i) for i, n in enumerate(lens)])
    wall = time.perf_counter() - t0
    (m8, a8), (m16, a16) = res
    alpha = float(np.log2(m16 / m8))
    mask32 = m16 * (L / lens[1]) ** alpha
    attn32 = a16 * L / lens[1]
    cores = os.cpu_count() or 1
    serial = Hkv * mask32 + Hq * attn32
    # heads are independent: ceil(tasks / cores) rounds of the longest task
    rounds = -(-(Hkv + Hq) // cores)
    par = max(serial / cores, rounds * max(mask32, attn32)) if cores < Hkv + Hq else \
        max(mask32, attn32)
    kind = "reference" if reference_available() else "port"
    return {"value": par * 1e3, "unit": "ms", "cores": min(cores, Hkv + Hq), "kind": kind,
            "single_core_ms": serial * 1e3,
            "sample": (f"top_k {top_k} (budget {budget}), one head at 8K and 16K tokens "
                       f"({'baseline/_ref dhsa.prefill_mask + softmax_row row body' if kind == 'reference' else 'oracle prefill_rows + row body'}): "
                       f"mask {m8:.2f} s / {m16:.2f} s (growth exponent {alpha:.2f}), "
                       f"attention {a8:.2f} s / {a16:.2f} s (512 sampled rows each, scaled); "
                       f"extrapolated to 32K: mask {mask32:.1f} s per kv group, attention "
                       f"{attn32:.1f} s per q head; {Hkv} masks + {Hq} heads = {serial:.0f} s on "
                       f"one core, spread over {min(cores, Hkv + Hq)} cores; wall {wall:.1f} s")}


# ------------------------------------------------------------- GPU bench --
def dist_setup():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; ranks beyond the visible devices wrap around (only
    # for exercising the multi-rank path on a smaller box, with
    # DHSA_DIST_BACKEND=gloo since NCCL refuses two ranks on one device)
    dev = local % max(1, torch.cuda.device_count()) if torch.cuda.is_available() else 0
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(dev)
        backend = os.environ.get("DHSA_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(dev)
    return world, rank, dev


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def rank_shape(name, shard, parts):
    """(B, Hq, Hkv) one rank runs: the config's shape ("batch": every rank
    owns its own full batch, weak scaling) or 1/parts of the heads ("heads":
    the config's batch with Hq/parts q heads and Hkv/parts kv heads per rank,
    strong scaling; BASELINE.json configs[2] "heads sharded across 1/2/4/8")."""
    B, Hq, Hkv = CONFIGS[name][:3]
    if shard == "heads" and parts > 1:
        if Hkv % parts:
            raise SystemExit(f"{Hkv} kv heads cannot be sharded over {parts} ranks")
        return B, Hq // parts, Hkv // parts
    return B, Hq, Hkv


def bench_config(name, world, shard, proxy, B, Hq, Hkv, dec=None):
    """The config dict of both arms (ours and --impl reference)."""
    _, Hq0, Hkv0, D, L, blk, K, dt = CONFIGS[name]
    parts = proxy or world
    cfg = {"workload": workload_desc(name), "context": L, "block": blk, "top_k": K,
           "budget": K * blk + 1, "selection": "group-shared max over q-heads",
           "sharding": (f"heads: {Hq}q/{Hkv}kv heads of {Hq0}/{Hkv0} per rank x {parts} ranks"
                        if shard == "heads" and parts > 1 else
                        f"batch: every rank owns {B} sequences"),
           "global_batch": B if shard == "heads" else B * world,
           "parallelism": (f"heads{parts}" if shard == "heads" and parts > 1 else f"dp{world}")}
    if proxy:
        cfg["rank_proxy"] = (f"one rank's share of a {proxy}-GPU heads-sharded job timed on this "
                             f"GPU; ranks are independent (no collective on the data path), "
                             f"so the {proxy}-GPU job time = this rank's time")
    return cfg


def run_gpu(args):
    import torch

    from paper_2510_24606_b200.decode import SparseDecoder

    world, rank, local = dist_setup()
    name = args.config
    _, _, _, D, L, blk, K, dtn = CONFIGS[name]
    shard = args.shard or ("heads" if name == "C3" else "batch")
    proxy = args.rank_proxy if world == 1 and args.rank_proxy and args.rank_proxy > 1 else 0
    B, Hq, Hkv = rank_shape(name, shard, proxy or world)
    dtype = getattr(torch, dtn)
    W, S = args.warmup, args.steps
    roll = args.roll_steps  # untimed replays before/after the timed steps (clock sampling)
    total_steps = W + S + 2 * roll + args.breakdown_steps + 2 * args.e2e_steps + 8
    dec = SparseDecoder(B, Hq, Hkv, D, L + total_steps, block=blk, top_k=K, dtype=dtype,
                        agg="max", scoring=args.scoring, splits=args.splits)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1234 + rank)
    # prompt K/V written straight into the cache, then the fp64 centroid build
    for t in (dec.k_cache, dec.v_cache):
        t[:, :, :L].normal_(generator=gen)
    dec.prefill(dec.k_cache, dec.v_cache, prompt_len=L)
    torch.cuda.synchronize()
    nslot = W + S
    qs = torch.randn(nslot, B, Hq, D, device="cuda", generator=gen).to(dtype)
    ks = torch.randn(nslot, B, Hkv, D, device="cuda", generator=gen).to(dtype)
    vs = torch.randn(nslot, B, Hkv, D, device="cuda", generator=gen).to(dtype)
    out = torch.empty(B, Hq, D, dtype=dtype, device="cuda")

    # one eager step loads every kernel module before capture
    dec.step(qs[0], ks[0], vs[0], out=out)
    torch.cuda.synchronize()
    # one CUDA graph per step slot (4 kernels each); replay = one decode step
    stream = torch.cuda.Stream()
    graphs = []
    torch.cuda.synchronize()
    for i in range(nslot):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            dec.launch(qs[i], ks[i], vs[i], out, stream=stream)
        graphs.append(g)
    # capture only recorded the launches; the engine state is still at step 0
    for i in range(W):
        graphs[i].replay()
    torch.cuda.synchronize()
    barrier(world)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk, torch.cuda.stream(stream):
        torch.cuda.synchronize()
        barrier(world)
        # keep the GPU busy around the (short) timed region so that the
        # 100 ms nvidia-smi samples see the clocks under this load
        for i in range(roll):
            graphs[W + i % S].replay()
        start.record(stream)
        for i in range(W, W + S):
            graphs[i].replay()
        end.record(stream)
        for i in range(roll):
            graphs[W + i % S].replay()
        torch.cuda.synchronize()
    barrier(world)
    ms = start.elapsed_time(end)
    ms = max_over_ranks(ms, world)
    ms_step = ms / S
    dec.steps += W + S + 2 * roll
    # whole-job tokens/s: heads-sharded ranks all serve the same B sequences
    seqs = B if shard == "heads" else B * world
    value = seqs * S / (ms / 1e3)

    # per-kernel breakdown (eager launches bracketed by events, same stream)
    names = None
    acc = {}
    nb = args.breakdown_steps
    for i in range(nb):
        j = i % nslot
        stg = dec.stages(qs[j], ks[j], vs[j], out, stream=stream)
        names = [n for n, _ in stg]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(stg) + 1)]
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            for k_, (_, fn) in enumerate(stg):
                fn()
                ev[k_ + 1].record(stream)
        torch.cuda.synchronize()
        dec.steps += 1
        if i == 0:
            continue  # first eager launch pays one-time attribute setup
        for k_, n in enumerate(names):
            acc[n] = acc.get(n, 0.0) + ev[k_].elapsed_time(ev[k_ + 1])
    cnt = max(1, nb - 1)
    us = {n: acc[n] / cnt * 1e3 for n in names}
    bytes_ = dec.bytes_per_step()
    score_name = names[0]
    score_bytes = bytes_["centroids"] + B * Hq * D * 2
    attn_bytes = bytes_["kv"] + 2 * B * Hq * D * 2
    kern_bytes = {score_name: score_bytes, "attn": attn_bytes}
    dominant = max((score_name, "attn"), key=lambda n: us[n])
    peak, peak_src = peaks()
    achieved = kern_bytes[dominant] / (us[dominant] * 1e-6) / 1e9
    traffic = load_traffic().get(name, {}).get(dominant)

    # end-to-end through the public API with pinned host buffers
    # one pinned host buffer per step input set: [q | k | v] (one H2D copy)
    hqkv = torch.cat([qs[0].reshape(-1), ks[0].reshape(-1), vs[0].reshape(-1)]).cpu().pin_memory()
    hout = torch.empty(B, Hq, D, dtype=dtype).pin_memory()
    dq, dk, dv = torch.empty_like(qs[0]), torch.empty_like(ks[0]), torch.empty_like(vs[0])
    ne = args.e2e_steps
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for i in range(ne + 1):
            if i == 1:
                e0.record(stream)
            dec.step_host_packed(hqkv, hout)
        e1.record(stream)
        torch.cuda.synchronize()
    e2e_pipe_ms = max_over_ranks(e0.elapsed_time(e1) / ne, world)
    # a real decode loop: step i+1's q exists only after step i's output is
    # on the host, so every step waits for its own D2H copy before the next
    # H2D copy is issued (host synchronisation inside the timed region)
    torch.cuda.synchronize()
    barrier(world)
    with torch.cuda.stream(stream):
        dec.step_host_packed(hqkv, hout)
        stream.synchronize()
        e0.record(stream)
        for i in range(ne):
            dec.step_host_packed(hqkv, hout)
            stream.synchronize()
        e1.record(stream)
        torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / ne, world)
    esz = torch.finfo(dtype).bits // 8
    h2d = (B * Hq * D + 2 * B * Hkv * D) * esz
    d2h = B * Hq * D * esz

    step_mb = (bytes_["centroids"] + bytes_["kv"]) / 1e6
    cfg = bench_config(name, world, shard, proxy, B, Hq, Hkv)
    cfg.update({
        "rank_shape": {"batch": B, "q_heads": Hq, "kv_heads": Hkv},
        "l2": (f"per-rank working set larger than L2 (126 MB): sketch "
               f"{bytes_['centroids'] / 1e6:.0f} MB + selected KV {bytes_['kv'] / 1e6:.0f} MB per "
               f"step, read once; a step's 32 distinct q/k/v inputs rotate"
               if step_mb > 126 else
               f"per-rank working set ({step_mb:.0f} MB/step) of the same order as L2 and not "
               f"flushed; the KV cache behind it ({dec.k_cache.numel() * 4 / 1e9:.1f} GB) is not"),
        "graphs": f"one CUDA graph per step ({dec.kernels_per_step} kernels)",
        "scoring": dec.scoring, "attention": dec.attn_mode})
    result = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": S,
        "warmup": W, "ms_per_step": ms_step, "us_per_step": ms_step * 1e3,
        "higher_is_better": True, "scaling": "strong" if shard == "heads" else "weak",
        "vs_baseline": None,
        "dtype": "bf16" if dtype == torch.bfloat16 else "f32",
        "data": f"synthetic N(0,1) q/k/v, random-init KV cache; {step_mb:.0f} MB read per step",
        "config": cfg,
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "algorithmic_bytes": kern_bytes[dominant]},
        "step_roofline": {"bytes_per_step": bytes_["total"],
                          "achieved_gbs": bytes_["total"] / (ms_step * 1e-3) / 1e9,
                          "frac": bytes_["total"] / (ms_step * 1e-3) / 1e9 / peak},
        "breakdown_us": us,
        "e2e": {"value": seqs / (e2e_ms / 1e3), "unit": "tokens/s",
                "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "SparseDecoder.step_host_packed (public API: one pinned host [q|k|v] "
                        "buffer -> one H2D copy -> one CUDA-graph replay of the C-ABI kernels -> "
                        "host o), the host waiting for each step's output before issuing the "
                        "next (an autoregressive decode loop)",
                "pipelined": {"value": seqs / (e2e_pipe_ms / 1e3), "ms_per_step": e2e_pipe_ms,
                              "note": "steps enqueued back to back without host waits (copy of "
                                      "step i overlaps step i+1): throughput, not latency"}},
        "gpu_launches": dec.kernels_per_step * S,
        "clocks": clk.summary(),
        "splits": dec.splits if dec.attn_mode == "split" else None,
    }
    if proxy:
        result["proxy"] = {"n_gpus": proxy, "note": cfg["rank_proxy"]}
    if rank == 0 and world == 1 and not args.no_cpu:
        # ~10-30 s of host CPU work: 64 units x 4 decode steps of the whole job
        result["cpu_baseline"] = cpu_baseline(name, units_sample=args.cpu_units or 64, steps=4)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_gpu_c4(args):
    """C4: one 1M-token sequence, sequence-sharded split-KV over the N GPUs
    (shard = contiguous 1M/N tokens, NCCL all-gathers of the candidate rows
    and the (m, l, acc) records).  N = 1 runs the same
    path with one shard.  value = decode tokens/s of the single sequence."""
    import torch

    from paper_2510_24606_b200.splitkv import LocalComm, SplitKVShard, TorchComm

    world, rank, local = dist_setup()
    B, Hq, Hkv, D, L, blk, K, dtn = CONFIGS["C4"]
    W, S = args.warmup, args.steps
    nslot = W + S
    extra = nslot + args.e2e_steps + 8
    sh = SplitKVShard(B, Hq, Hkv, D, L, rank=rank, world=world, block=blk, top_k=K,
                      max_new=extra, splits=args.splits)
    comm = TorchComm() if world > 1 else LocalComm()
    gen = torch.Generator(device="cuda")
    gen.manual_seed(4321 + rank)
    d = sh.dec
    for t in (d.k_cache, d.v_cache):
        t[:, :, :sh.local_len].normal_(generator=gen)
    d.prefill(d.k_cache, d.v_cache, prompt_len=sh.local_len)
    gq = torch.Generator(device="cuda")
    gq.manual_seed(99)  # q is replicated: same draws on every rank
    qs = torch.randn(nslot, B, Hq, D, device="cuda", generator=gq).bfloat16()
    ks = torch.randn(nslot, B, Hkv, D, device="cuda", generator=gq).bfloat16()
    vs = torch.randn(nslot, B, Hkv, D, device="cuda", generator=gq).bfloat16()
    out = torch.empty(B, Hq, D, dtype=torch.bfloat16, device="cuda")
    sh.step(qs[0], ks[0], vs[0], comm, out=out)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream()
    # multi-rank: eager launches (capturing NCCL collectives is not attempted)
    graphs, graphed = [], world == 1
    graph_err = None if graphed else "multi-rank: eager launches"
    try:
        for i in range(1, nslot if graphed else 1):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                sh.launch(qs[i], ks[i], vs[i], comm, out, stream=stream)
            graphs.append(g)
    except Exception as e:  # collectives not capturable here: time eager launches
        graphed = False
        graph_err = str(e).splitlines()[0][:120]
        torch.cuda.synchronize()

    def run(i):
        if graphed:
            graphs[i - 1].replay()
        else:
            sh.launch(qs[i], ks[i], vs[i], comm, out, stream=stream)

    with torch.cuda.stream(stream):
        for i in range(1, W):
            run(i)
    torch.cuda.synchronize()
    barrier(world)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk, torch.cuda.stream(stream):
        start.record(stream)
        for i in range(W, nslot):
            run(i)
        end.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    sh.check_capacity()
    ms = max_over_ranks(start.elapsed_time(end), world)
    n_steps = nslot - W
    ms_step = ms / n_steps
    peak, peak_src = peaks()
    nc_local = (sh.local_len + blk - 1) // blk
    sketch_b = sh.dec.U * nc_local * D * 2
    kv_b = sh.dec.U * (K * blk + 1) * D * 2 * 2 // world  # selected K/V, spread over shards
    result = {
        "metric": METRIC, "value": B / (ms_step / 1e3), "unit": "tokens/s", "n_gpus": world,
        "steps": n_steps, "warmup": W, "ms_per_step": ms_step, "us_per_step": ms_step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic N(0,1) q/k/v, random-init KV cache",
        "config": {"workload": f"C4 split-KV decode: 1 sequence, context={L}, Hq={Hq}, Hkv={Hkv}, "
                               f"d={D}, block={blk}, top_k={K}, {world} sequence shard(s)",
                   "context": L, "shards": world, "graphs": graphed,
                   "path": ("one shard: the plain decode step (select -> attention, no exchange)"
                            if sh.direct else "split-KV: candidates, all-gather, global walk, "
                            "attention records, all-gather, merge"),
                   "exchange_bytes_per_rank": sh.bytes_per_step()["exchange"]},
        "step_roofline": {"bytes_per_step_per_gpu": sketch_b + kv_b,
                          "roofline_us": (sketch_b + kv_b) / (peak * 1e9) * 1e6,
                          "peak": peak, "peak_source": peak_src,
                          "frac": (sketch_b + kv_b) / (ms_step * 1e-3) / 1e9 / peak,
                          "note": "latency-bound" + ("" if sh.direct else
                                                     ": 5 kernels + 2 all-gathers per step")},
        "gpu_launches": sh.kernels_per_step * n_steps, "clocks": clk.summary(),
    }
    if graph_err:
        result["config"]["graph_note"] = graph_err
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_gpu_c4_proxy(args):
    """C4 on N GPUs, proxied on one: the N shards of the 1M-token sequence as
    a SplitKVGroup in one process (every kernel of the N-GPU step, the two
    exchanges as device copies), one CUDA graph per step.  The shards'
    kernels run one after another here, so the step time / N is one rank's
    kernel time on N GPUs; the two all-gathers of the real run (NCCL over
    NVLink, ~30 KB per rank each) are not included."""
    import torch

    from paper_2510_24606_b200.splitkv import SplitKVGroup

    dist_setup()
    B, Hq, Hkv, D, L, blk, K, dtn = CONFIGS["C4"]
    N = args.rank_proxy
    W, S = args.warmup, args.steps
    nslot = W + S
    grp = SplitKVGroup(B, Hq, Hkv, D, L, N, block=blk, top_k=K, max_new=nslot + 8)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(4321)
    for sh in grp.shards:
        d = sh.dec
        for t in (d.k_cache, d.v_cache):
            t[:, :, :sh.local_len].normal_(generator=gen)
        d.prefill(d.k_cache, d.v_cache, prompt_len=sh.local_len)
    qs = torch.randn(nslot, B, Hq, D, device="cuda", generator=gen).bfloat16()
    ks = torch.randn(nslot, B, Hkv, D, device="cuda", generator=gen).bfloat16()
    vs = torch.randn(nslot, B, Hkv, D, device="cuda", generator=gen).bfloat16()
    out = torch.empty(B, Hq, D, dtype=torch.bfloat16, device="cuda")
    grp.step(qs[0], ks[0], vs[0], out=out)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream()
    graphs = []
    for i in range(1, nslot):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            grp.launch(qs[i], ks[i], vs[i], out, stream=stream)
        graphs.append(g)
    for i in range(1, W):
        graphs[i - 1].replay()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk, torch.cuda.stream(stream):
        start.record(stream)
        for i in range(W, nslot):
            graphs[i - 1].replay()
        end.record(stream)
        torch.cuda.synchronize()
    for sh in grp.shards:
        sh.check_capacity()
    ms_step = start.elapsed_time(end) / (nslot - W)
    per_rank_us = ms_step * 1e3 / N
    sh0 = grp.shards[0]
    result = {
        "metric": METRIC, "value": B / (per_rank_us * 1e-6), "unit": "tokens/s", "n_gpus": 1,
        "steps": nslot - W, "warmup": W, "ms_per_step": per_rank_us / 1e3,
        "us_per_step": per_rank_us, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic N(0,1) q/k/v, random-init KV cache",
        "config": {"workload": f"C4 split-KV decode: 1 sequence, context={L}, Hq={Hq}, Hkv={Hkv}, "
                               f"d={D}, block={blk}, top_k={K}, {N} sequence shards",
                   "context": L, "shards": N, "graphs": True,
                   "exchange_bytes_per_rank": sh0.bytes_per_step()["exchange"]},
        "proxy": {"n_gpus": N, "group_us_per_step": ms_step * 1e3,
                  "note": f"the {N} shards' kernels on one GPU, one after another, exchanges as "
                          f"device copies; us_per_step = group step / {N} = one rank's kernel "
                          f"time; the two NCCL all-gathers of the {N}-GPU run are not included"},
        "gpu_launches": sum(s.kernels_per_step for s in grp.shards) * (nslot - W),
        "clocks": clk.summary(),
    }
    print(json.dumps(result), flush=True)


def run_gpu_c5(args):
    """C5: sparse prefill of one 32K-token sequence (Llama-3-8B attention
    shape, bf16), tcgen05 tiles over the selected blocks, top-k sweep.
    Reports the whole prefill time per K and the attention kernel's tensor
    throughput against the measured bf16 peak (algorithmic flops =
    4 * sum_i min(i+1, budget) * D * Hq)."""
    import torch

    from paper_2510_24606_b200.prefill import SparsePrefill

    world, rank, local = dist_setup()
    B, Hq, Hkv, D, L = 1, 32, 8, 128, 32768
    W, S = args.warmup, args.steps
    gen = torch.Generator(device="cuda")
    gen.manual_seed(77 + rank)
    q = torch.randn(B, Hq, L, D, device="cuda", generator=gen).bfloat16()
    k = torch.randn(B, Hkv, L, D, device="cuda", generator=gen).bfloat16()
    v = torch.randn(B, Hkv, L, D, device="cuda", generator=gen).bfloat16()
    out = torch.empty_like(q)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > L2 (126 MB)
    tf_peak = tf_sust = None
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        with open(pp) as f:
            d = json.load(f)
        tf_peak, tf_sust = d.get("bf16_tflops"), d.get("bf16_tflops_sustained")
    peak = tf_peak or 1590.0
    sweep = []

    def time_prefill(pf):
        stg = pf.stages(q, k, v, out)
        for _ in range(W):
            for _, fn in stg:
                fn()
        torch.cuda.synchronize()
        pf.check_capacity()
        names = [n for n, _ in stg]
        acc = {n: 0.0 for n in names}
        tot = 0.0
        for _ in range(S):
            flush.zero_()  # L2 flushed before every timed prefill
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(stg) + 1)]
            ev[0].record()
            for i, (_, fn) in enumerate(stg):
                fn()
                ev[i + 1].record()
            torch.cuda.synchronize()
            for i, n in enumerate(names):
                acc[n] += ev[i].elapsed_time(ev[i + 1])
            tot += ev[0].elapsed_time(ev[-1])
        ms = max_over_ranks(tot / S, world)
        return ms, {n: acc[n] / S for n in names}

    with ClockSampler(local) as clk:
        for K in args.c5_topk:
            pf = SparsePrefill(B, Hq, Hkv, D, L, top_k=K, agg="max")
            ms, bd = time_prefill(pf)
            attn_ms = bd["attn"]
            fl = pf.flops()
            sweep.append({"top_k": K, "budget": pf.budget, "ms": ms,
                          "breakdown_ms": bd,
                          "tflops_algorithmic": fl / 1e12,
                          "attn_tflops": fl / (attn_ms * 1e-3) / 1e12,
                          "attn_frac_of_peak": fl / (attn_ms * 1e-3) / 1e12 / peak,
                          "prefill_tokens_per_s": B * L / (ms * 1e-3)})
    head = next((x for x in sweep if x["top_k"] == 64), sweep[0])
    # mask quality at 32K: recall / output fidelity of the
    # top-k masks against dense causal attention, both on the tcgen05 kernel
    from paper_2510_24606_b200.prefill import mask_quality

    quality = None
    if not args.no_quality:
        pf = SparsePrefill(B, Hq, Hkv, D, L, top_k=head["top_k"], agg="max")
        rec, cos = mask_quality(q, k, v, pf)
        dense = SparsePrefill(B, Hq, Hkv, D, L, budget=L + 1, agg="max")
        dense(q, k, v, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        e0.record()
        dense(q, k, v, out)
        e1.record()
        torch.cuda.synchronize()
        dms = e0.elapsed_time(e1)
        quality = {"top_k": head["top_k"], "attention_mass_recall": float(rec.mean()),
                   "output_fidelity": float(cos.mean()),
                   "dense_causal_ms": dms, "dense_causal_tflops": dense.flops() / (dms * 1e-3) / 1e12,
                   "note": "harness.attention_mass_recall / output_fidelity semantics over all "
                           "32 heads and 32K rows (the CPU harness needs the 8.6 GB L x L matrix)"}
    # dynamic chunks (the paper's pipeline): boundary
    # predictor on the GPU over every kv head's keys -> nms_boundaries on the
    # host -> per-head chunk lists -> the same prefill with those chunks
    dynamic = None
    if not args.no_dynamic:
        from paper_2510_24606_b200.chunking import nms_boundaries
        from paper_2510_24606_b200.predictor import BoundaryPredictor, init_predictor

        bp = BoundaryPredictor(init_predictor(D, window=4, heads=8, hidden=256, seed=0))
        kf = k[0].double().contiguous()
        for h in range(Hkv):
            bp.probs(kf[h])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        probs = [bp.probs(kf[h]) for h in range(Hkv)]
        e1.record()
        torch.cuda.synchronize()
        pred_ms = e0.elapsed_time(e1)
        t0 = time.perf_counter()
        bounds = []
        for p in probs:
            sc = np.zeros(L)
            sc[3:L - 4] = p.cpu().numpy()  # predictable positions w-1 .. L-w-1 (w = 4)
            bounds.append(nms_boundaries(sc, min_conf=0.1, window=32, max_chunks=L // 64))
        nms_ms = (time.perf_counter() - t0) * 1e3
        pf = SparsePrefill(B, Hq, Hkv, D, L, top_k=head["top_k"], agg="max", bounds=bounds)
        ms, bd = time_prefill(pf)
        fl = pf.flops()
        lens = np.concatenate([np.diff(b) for b in bounds])
        dynamic = {"top_k_budget": pf.budget, "ms": ms, "breakdown_ms": bd,
                   "attn_tflops": fl / (bd["attn"] * 1e-3) / 1e12,
                   "attn_frac_of_peak": fl / (bd["attn"] * 1e-3) / 1e12 / peak,
                   "predictor_ms_all_heads": pred_ms, "nms_host_ms_all_heads": nms_ms,
                   "chunks_per_head": int(np.mean([len(b) - 1 for b in bounds])),
                   "chunk_len_min_mean_max": [int(lens.min()), float(lens.mean()),
                                              int(lens.max())],
                   "note": "random-init predictor (no trained checkpoint offline); fp64 "
                           "predictor over 8 kv heads x 32K keys; NMS window 32, "
                           "max_chunks L/64"}
        if not args.no_quality:
            rec, cos = mask_quality(q, k, v, pf)
            dynamic["attention_mass_recall"] = float(rec.mean())
            dynamic["output_fidelity"] = float(cos.mean())
    result = {
        "metric": "sparse prefill ms per 32K-token sequence (C5); tensor TFLOP/s vs roofline",
        "value": head["ms"], "unit": "ms", "n_gpus": world, "steps": S, "warmup": W,
        "ms_per_step": head["ms"], "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic N(0,1) q/k/v",
        "config": {"workload": f"C5 sparse prefill: B={B}, Hq={Hq}, Hkv={Hkv}, d={D}, L={L}, "
                               "block=64, group-shared max selection, tcgen05 tiles",
                   "l2": "flushed (256 MB write) before every timed prefill",
                   "headline_top_k": head["top_k"]},
        "roofline": {"bound": "tensor", "kernel": "attn", "achieved": head["attn_tflops"],
                     "peak": peak, "unit": "TFLOP/s", "frac": head["attn_frac_of_peak"],
                     "peak_source": "measured (MEASURED_PEAKS.json bf16_tflops)" if tf_peak
                     else "fallback (B200_PROFILING.md)", "peak_sustained": tf_sust},
        "sweep": sweep, "mask_quality": quality, "dynamic_chunks": dynamic,
        "gpu_launches": 5 * S, "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline_c5(Hq, Hkv, D, L, head["top_k"])
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_reference(args):
    """The reference arm: the reference's own CPU implementation of the path
    (baseline/_ref, else the oracle port) on this box's host cores, on the
    same workload, metric and config as our arm; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    name = args.config if args.config in CONFIGS else "C3"
    shard = args.shard or ("heads" if name == "C3" else "batch")
    proxy = args.rank_proxy if world == 1 and args.rank_proxy and args.rank_proxy > 1 else 0
    B, Hq, Hkv = rank_shape(name, shard, proxy or world)
    seqs = B if shard == "heads" else B * world
    vals = []
    cb = None
    # each step: one bounded sample (units x 1 decode step) of the whole job
    # (its units are independent; the host cores serve all of them)
    for i in range(args.warmup_ref + args.steps_ref):
        cb = cpu_baseline(name, units_sample=args.cpu_units, steps=1)
        if i >= args.warmup_ref:
            vals.append(cb["value"])
    value = float(np.mean(vals)) * seqs / CONFIGS[name][0]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps_ref, "warmup": args.warmup_ref,
        "ms_per_step": seqs / value * 1e3, "higher_is_better": True,
        "scaling": "strong" if shard == "heads" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic N(0,1), fp32-valued",
        "config": bench_config(name, world, shard, proxy, B, Hq, Hkv),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cb["cores"],
                         "kind": cb["kind"], "sample": cb["sample"]},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def self_launch(args):
    """``--gpus N`` (N > 1) outside torchrun: run N ranks of this script
    under torch.distributed.run on 127.0.0.1 and return its exit code."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS) + ["C5"])
    ap.add_argument("--c5-topk", type=int, nargs="+", default=[16, 32, 64, 128, 256])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--breakdown-steps", type=int, default=6)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--roll-steps", type=int, default=1500)
    ap.add_argument("--scoring", default=None, choices=[None, "sketch", "fp64"])
    ap.add_argument("--splits", type=int, default=None)
    ap.add_argument("--cpu-units", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-quality", action="store_true")
    ap.add_argument("--no-dynamic", action="store_true",
                    help="C5: skip the predictor -> NMS -> dynamic-chunk prefill run")
    ap.add_argument("--shard", default=None, choices=[None, "heads", "batch"],
                    help="multi-GPU decode: shard the heads of one batch (C3 default) or give "
                         "every rank its own batch")
    ap.add_argument("--rank-proxy", type=int, default=0,
                    help="one GPU: time rank 0's share of an N-GPU heads-sharded job")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    args.warmup = max(args.warmup, 3)
    # the reference arm: every "step" is one bounded CPU sample (~0.6 s)
    args.steps_ref = max(1, args.steps)
    args.warmup_ref = args.warmup
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "C4" and args.rank_proxy > 1 and "WORLD_SIZE" not in os.environ:
        run_gpu_c4_proxy(args)
    elif args.config == "C4":
        run_gpu_c4(args)
    elif args.config == "C5":
        run_gpu_c5(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
