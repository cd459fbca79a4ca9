"""Multi-process (world_size 2 and 3, gloo on CPU) test of the sequence-sharded
split-KV exchange: the product's ``TorchComm`` all-gathers the fixed-size
candidate rows (``dhsa_split_cand`` byte layout) and the (m, l, acc) records;
each rank runs the global walk over the gathered candidates.  The local
candidate walk and the attention partials are computed by the CPU oracle
here (no GPU); the kernels implementing them are checked against the same
oracle in test_gpu_splitkv.py.  Asserts: every rank's global walk equals the
unsharded walk (masks.topk_row semantics), and the merged output equals the
single-pass softmax (core.py:113-118)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dhsa_oracle as O

REC = np.dtype([("score", "<f8"), ("gid", "<i4"), ("len", "<i4"), ("lo", "<i4"), ("pad", "<i4")])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dyn_bounds(rng, P):
    b, pos = [0], 0
    while pos < P:
        pos = min(P, pos + int(rng.choice([int(rng.integers(1, 64)), int(rng.integers(64, 300))])))
        b.append(pos)
    return b


def _problem(seed, P, D, g, block, dyn=False):
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((P + g + 1, D))
    V = rng.standard_normal((P + g + 1, D))
    q = rng.standard_normal(D)
    if seed % 2:  # exact ties across shard borders: duplicated first/last blocks
        K[P - block:P] = K[0:block]
    bounds = _dyn_bounds(rng, P) if dyn else O.static_grid(P, block)
    cached = O.centroids(K[:P], bounds)
    gen_sum = K[P:P + g].sum(axis=0) if g else np.zeros(D)
    s = O.decode_scores(q, cached, gen_sum, g, K[P + g])
    nc = len(bounds) - 1
    lens = np.diff(bounds).tolist() + ([g] if g else [])
    los = bounds[:-1] + ([P] if g else [])
    return K, V, q, s[: nc + (1 if g else 0)], np.array(lens), np.array(los), nc, bounds


def _worker(rank, world, port, seed, dyn=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_24606_b200.splitkv import (REC_BYTES, TorchComm, candidate_capacity,
                                                    shard_chunks, shard_ranges)

        assert REC.itemsize == REC_BYTES
        comm = TorchComm()
        P, D, g, block, budget = 1900, 32, 5, 64, 300
        K, V, q, s, lens, los, nc, bounds = _problem(seed, P, D, g, block, dyn)
        row = P + g
        R = min(budget, row + 1) - 1
        ids = np.arange(len(s))
        full_takes = O.chunk_takes(s, ids, lens, R)

        if dyn:  # the product's cut (chunk starts) and rank-uniform capacity
            cuts = shard_chunks(bounds, world)
            lo, hi = bounds[cuts[rank][0]], bounds[cuts[rank][1]]
            cap = max(candidate_capacity(budget, block, np.diff(bounds)[a:z]) for a, z in cuts)
        else:
            lo, hi = shard_ranges(P, block, world)[rank]
            cap = candidate_capacity(budget, block)
        mine = [c for c in range(nc) if lo <= los[c] < hi]
        if rank == world - 1 and g:
            mine.append(nc)  # the generated chunk lives on the tail shard
        mine = np.array(mine, dtype=np.int64)
        local = mine[O.split_candidates(s[mine], ids[mine], lens[mine], R)]

        assert len(local) <= cap
        rowbuf = np.zeros(cap + 1, dtype=REC)
        rowbuf[0]["gid"] = len(local)  # header: count in the first record's first int
        hdr = rowbuf.view(np.uint8)[:4].view(np.int32)
        hdr[0] = len(local)
        for i, c in enumerate(local):
            rowbuf[1 + i] = (s[c], c, lens[c], los[c], 0)
        send = torch.from_numpy(rowbuf.view(np.uint8).copy())
        gathered = torch.zeros(world * send.numel(), dtype=torch.uint8)
        comm.all_gather(gathered, send)
        allrec = gathered.numpy().view(REC).reshape(world, cap + 1)
        cand = []
        for r in range(world):
            n = int(allrec[r].view(np.uint8)[:4].view(np.int32)[0])
            cand.extend(allrec[r, 1:1 + n].tolist())
        cs = np.array([c[0] for c in cand])
        cid = np.array([c[1] for c in cand])
        cl = np.array([c[2] for c in cand])
        takes = O.chunk_takes(cs, cid, cl, R)
        # global walk over the union == unsharded walk, on every rank
        got = np.zeros_like(full_takes)
        got[cid] = takes
        assert np.array_equal(got, full_takes), (rank, seed)

        # this rank's tokens, attention partial, record exchange, merge
        idx = [np.arange(los[c], los[c] + t) for c, t in zip(cid, takes)
               if t > 0 and c in set(mine.tolist())]
        if rank == world - 1:
            idx.append(np.array([row]))
        idx = np.concatenate(idx).astype(np.int64) if idx else np.zeros(0, np.int64)
        m, l, acc = O.attend_partial(q, K, V, idx)
        rec = torch.from_numpy(np.concatenate([[m, l], acc]).astype(np.float32))
        rec_all = torch.zeros(world * rec.numel(), dtype=torch.float32)
        comm.all_gather(rec_all, rec)
        parts = [(float(r[0]), float(r[1]), r[2:].astype(np.float64))
                 for r in rec_all.numpy().reshape(world, -1)]
        o = O.merge_partials(parts)
        full_idx = O.ranges_to_indices([(los[c], t) for c, t in enumerate(full_takes) if t], row)
        ref = O.attend_row(q, K, V, full_idx)
        assert np.abs(o - ref).max() <= 1e-5 * np.abs(ref).max()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,seed", [(2, 0), (2, 1), (3, 2), (3, 3)])
def test_splitkv_exchange_gloo(world, seed):
    mp.spawn(_worker, args=(world, _free_port(), seed), nprocs=world, join=True)


@pytest.mark.parametrize("world,seed", [(2, 4), (3, 5)])
def test_splitkv_exchange_gloo_dynamic_chunks(world, seed):
    """Explicit boundary list (1..300-token chunks) cut at chunk starts."""
    mp.spawn(_worker, args=(world, _free_port(), seed, True), nprocs=world, join=True)


def test_shard_ranges_cover_prompt():
    from paper_2510_24606_b200.splitkv import candidate_capacity, shard_ranges

    for P, W in [(1900, 2), (1 << 20, 8), (64, 1), (130, 3)]:
        rs = shard_ranges(P, 64, W)
        assert rs[0][0] == 0 and rs[-1][1] == P
        for (a, b), (c, _) in zip(rs, rs[1:]):
            assert b == c and a % 64 == 0
    assert candidate_capacity(4097, 64) == 64 + 4
