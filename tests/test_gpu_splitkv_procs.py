"""Sequence-sharded split-KV decode (config C4's path) across real PROCESSES
with the GPU kernels: W ranks, one process each, all on cuda:0 (the test box
has one GPU; NCCL refuses two ranks on one device, so the process group is
gloo, which all-gathers the CUDA tensors through the host).  Every rank runs
the product's ``SplitKVShard.step`` with ``TorchComm``:
dhsa_decode_candidates_bf16 -> all-gather of the candidate rows ->
dhsa_split_select (global walk) -> attention records -> all-gather ->
dhsa_merge_partials.  Each rank's tiles must equal the unsharded oracle walk
restricted to its token range (masks.py:153-173 semantics, index for index)
and the merged output must match the float64 row body core.py:113-118
within the bf16 tolerance 2e-2 on every rank.  Also runs ``bench.py
--config C4 --gpus 2`` (self-launched torchrun, gloo) end to end."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dyn_bounds(P, seed):
    rng = np.random.default_rng(seed)
    b, pos = [0], 0
    while pos < P:
        pos = min(P, pos + int(rng.choice([int(rng.integers(1, 64)), int(rng.integers(64, 300))])))
        b.append(pos)
    return b


def _worker(rank, world, port, seed, dyn, errq):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from decode_harness import TOL, make_inputs, tiles_to_idx
        from oracle import dhsa_oracle as O
        from paper_2510_24606_b200.splitkv import SplitKVShard, TorchComm

        B, Hq, Hkv, D, P, steps, top_k = 1, 8, 2, 128, 6000, 3, 16
        t, host = make_inputs(B, Hq, Hkv, D, P, steps, torch.bfloat16, seed=seed)
        bounds = _dyn_bounds(P, seed) if dyn else None
        sh = SplitKVShard(B, Hq, Hkv, D, P, rank=rank, world=world, block=64, top_k=top_k,
                          max_new=steps + 1, bounds=bounds)
        sh.prefill(t["k"][:, :, sh.lo:sh.hi].contiguous().cuda(),
                   t["v"][:, :, sh.lo:sh.hi].contiguous().cuda())
        comm = TorchComm()
        G = Hq // Hkv
        gb = O.static_grid(P, 64) if bounds is None else bounds
        oracles = [O.DecodeOracle(host["k"][0, h, :P], gb, sh.budget) for h in range(Hkv)]
        worst = 0.0
        for s in range(steps):
            pos = P + s
            out = sh.step(t["q"][:, :, s].contiguous().cuda(),
                          t["k"][:, :, pos].contiguous().cuda(),
                          t["v"][:, :, pos].contiguous().cuda(), comm)
            torch.cuda.synchronize()
            sh.check_capacity()
            sel = sh.selection()
            o = out.double().cpu().numpy()
            for h in range(Hkv):
                qh = host["q"][0, h * G:(h + 1) * G, s]
                row = oracles[h].step_group(qh, host["k"][0, h, pos], agg="max")
                # this shard's tokens: prompt range [lo, hi) (+ generated + self on
                # the tail, whose local cache continues at hi = P: global = local + lo)
                mine = row[(row >= sh.lo) & (row < sh.hi)] if not sh.owns_tail else \
                    row[row >= sh.lo]
                got = tiles_to_idx(sel[h]) + sh.lo if len(sel[h]) else np.zeros(0, np.int64)
                assert np.array_equal(np.sort(got), mine), (rank, s, h, len(got), len(mine))
                for j in range(G):
                    ref = O.attend_row(qh[j], host["k"][0, h, :pos + 1], host["v"][0, h, :pos + 1],
                                       row)
                    err = np.abs(o[0, h * G + j] - ref).max() / np.abs(ref).max()
                    worst = max(worst, err)
        assert worst <= TOL[torch.bfloat16], worst
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # report to the parent (spawn hides tracebacks of assertions)
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


def _spawn(world, seed, dyn):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, dyn, errq))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    codes = [p.exitcode for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert not errs and all(c == 0 for c in codes), (codes, "\n".join(errs))


@pytest.mark.parametrize("world,seed", [(2, 0), (3, 1)])
def test_splitkv_processes_static(world, seed):
    _spawn(world, seed, False)


def test_splitkv_processes_dynamic_chunks():
    _spawn(2, 2, True)


def test_bench_c4_two_ranks_gloo():
    """bench.py --config C4 --gpus 2: self-launched torchrun, two ranks
    sharing the one GPU over gloo; the JSON line comes from rank 0."""
    env = dict(os.environ, DHSA_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C4",
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--e2e-steps", "2"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["shards"] == 2 and line["value"] > 0


def test_bench_c3_heads_sharded_two_ranks_gloo():
    """bench.py --gpus 2 (C3, heads sharded): self-launched torchrun, two
    ranks on the one GPU over gloo, each serving 16 q / 4 kv heads of the same
    32 sequences; rank 0 prints ONE line whose value is the whole job's 32
    tokens per max-over-ranks step time (strong scaling)."""
    env = dict(os.environ, DHSA_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps",
                        "3", "--warmup", "3", "--roll-steps", "0", "--breakdown-steps", "2",
                        "--e2e-steps", "2", "--no-cpu"],
                       capture_output=True, text=True, timeout=1200, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    cfg = line["config"]
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert cfg["parallelism"] == "heads2" and cfg["global_batch"] == 32
    assert cfg["rank_shape"] == {"batch": 32, "q_heads": 16, "kv_heads": 4}
    assert abs(line["value"] - 32 / (line["ms_per_step"] / 1e3)) <= 1e-6 * line["value"]
