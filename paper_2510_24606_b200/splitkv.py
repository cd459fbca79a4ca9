"""Sequence-sharded split-KV decode.

One long sequence (e.g. 1M tokens) is cut into W contiguous, chunk-aligned
shards, one per GPU (one process per GPU, ``torch.distributed`` over NCCL).
Shard r holds prompt chunks [c_r, c_{r+1}) with their K/V cache, fp64
centroids and fp16 sketch; the last ("tail") shard also holds the generated
chunk and receives every new token.  A decode step (Algorithm 2 of the paper,
masks.py:153-173 + core.py:113-118) is:

  1. local candidates  dhsa_decode_candidates_bf16: the certified walk of the
                       shard's chunks with the GLOBAL token budget; every
                       chunk with a positive local take is sent as
                       (exact fp64 score, global chunk id, length, start);
  2. all-gather        of the fixed-size candidate rows (a few KB);
  3. global walk       dhsa_split_select: the same on every shard, so the
                       selection is bit-identical everywhere and equals the
                       unsharded masks.topk_row walk (the union of local
                       candidate sets contains the global selection);
  4. local attention   dhsa_attn_partials over this shard's selected tiles ->
                       (m, l, acc) per q row;
  5. all-gather + merge dhsa_merge_partials.

The only exchanges are the two tiny all-gathers; the K/V bytes never move.
``Comm`` abstracts the collective: ``TorchComm`` (NCCL on GPUs, gloo on CPU
for the multi-process tests) or ``SplitKVGroup`` which drives W shards in one
process (single-GPU emulation / 1-GPU split-KV baseline).
"""

from __future__ import annotations

import torch

from . import _lib
from .decode import SparseDecoder

REC_BYTES = 24  # dhsa_split_cand


ShardSpec = _lib.ShardSpec


def shard_ranges(prompt_len: int, block: int, world: int):
    """Chunk-aligned contiguous token ranges [(lo, hi)] of the W shards
    (static grid chunking.py:42-54; chunks never straddle shards)."""
    nc = (prompt_len + block - 1) // block
    out = []
    for r in range(world):
        c0 = nc * r // world
        c1 = nc * (r + 1) // world
        out.append((c0 * block, min(c1 * block, prompt_len)))
    return out


def shard_chunks(bounds, world: int):
    """Contiguous chunk ranges [(c0, c1)] of the W shards for an explicit
    boundary list: cuts at the chunk starts
    nearest to an even token split, at least one chunk per shard."""
    b = [int(x) for x in bounds]
    nc = len(b) - 1
    if nc < world:
        raise ValueError(f"{nc} chunks cannot be split over {world} shards")
    cuts = [0]
    for r in range(1, world):
        target = b[-1] * r / world
        c = min(range(nc + 1), key=lambda j: (abs(b[j] - target), j))
        c = max(c, cuts[-1] + 1)
        c = min(c, nc - (world - r))
        cuts.append(c)
    cuts.append(nc)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def candidate_capacity(budget: int, block: int, lengths=None) -> int:
    """Upper bound on chunks with a positive take in a walk of budget-1
    tokens + the generated chunk: static ``block`` chunks, or the local chunk
    ``lengths`` (the walk touches at most one chunk more than the shortest
    chunks whose lengths stay below budget-1)."""
    if lengths is None:
        return (budget - 1) // block + 4
    import numpy as np

    srt = np.cumsum(np.sort(np.asarray(lengths, dtype=np.int64)))
    m = int(np.searchsorted(srt, budget - 1, side="left"))
    return min(m + 1, len(srt)) + 3


class TorchComm:
    """All-gather over a torch.distributed process group (NCCL on GPUs)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.flat = dist.get_backend(group) == "nccl"

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor):
        """out [W * inp.numel()] <- concatenation of every rank's inp."""
        if self.flat:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
        else:  # gloo: list form
            self.dist.all_gather(list(out.view(self.world, -1).unbind(0)), inp.view(-1),
                                 group=self.group)


class LocalComm:
    """World of one: the all-gather is a copy (W = 1 split-KV on one GPU)."""

    rank, world = 0, 1

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor):
        out.copy_(inp.view(-1))


class SplitKVShard:
    """One shard of a sequence-sharded sparse decode (bf16 sketch path).

    ``prompt_len`` is the GLOBAL prompt length; the shard's range comes from
    ``shard_ranges`` (static grid) or ``shard_chunks`` (``bounds``: one
    explicit boundary list shared by every unit; the shard gets its chunks,
    re-based to its first token, and global chunk ids keep the reference's
    tie-break).  Every shard receives the full q [B, Hq, D] each step;
    only the tail shard receives k_new / v_new."""

    def __init__(self, batch, q_heads, kv_heads, head_dim, prompt_len, *, rank, world,
                 block=64, top_k=64, budget=None, agg="max", max_new=1024, tile=64,
                 splits=None, device=None, attn_mode=None, bounds=None, direct=True):
        self.rank, self.world = int(rank), int(world)
        # one shard holds the whole sequence: its step is the plain batched
        # decode (select -> attention, no candidate records, exchange or
        # record merge); direct=False keeps the split kernels (tests)
        self.direct = bool(direct) and self.world == 1
        self.block = int(block)
        self.total_prompt = int(prompt_len)
        self.local_bounds = None
        max_chunks = None
        if bounds is None:
            self.lo, self.hi = shard_ranges(self.total_prompt, self.block, self.world)[self.rank]
            c0, n_total = self.lo // self.block, (self.total_prompt + self.block - 1) // self.block
        else:  # one explicit boundary list shared by every unit, cut at chunk starts
            from .chunking import check_boundaries

            gb = check_boundaries(bounds, self.total_prompt)
            c0, c1 = shard_chunks(gb, self.world)[self.rank]
            self.lo, self.hi = gb[c0], gb[c1]
            self.local_bounds = [x - self.lo for x in gb[c0:c1 + 1]]
            n_total = len(gb) - 1
            max_chunks = c1 - c0
        self.owns_tail = self.rank == self.world - 1
        self.local_len = self.hi - self.lo
        if self.local_len < 1:
            raise ValueError("shard holds no prompt tokens (too many shards for the prompt)")
        cap_len = self.local_len + (int(max_new) if self.owns_tail else 0) + 1
        self.dec = SparseDecoder(batch, q_heads, kv_heads, head_dim, cap_len, block=block,
                                 top_k=top_k, budget=budget, dtype=torch.bfloat16, agg=agg,
                                 tile=tile, splits=splits, device=device, scoring="sketch",
                                 attn_mode=attn_mode, max_chunks=max_chunks)
        d = self.dec
        self.B, self.Hq, self.Hkv, self.D, self.G = d.B, d.Hq, d.Hkv, d.D, d.G
        self.budget = d.budget
        self.spec = ShardSpec(c0, n_total, self.total_prompt, 1 if self.owns_tail else 0)
        if bounds is None:
            self.cap = candidate_capacity(self.budget, self.block)
        else:  # equal on every rank: the exchanged rows share one stride
            self.cap = max(candidate_capacity(self.budget, self.block,
                                              [gb[c + 1] - gb[c] for c in range(a, z)])
                           for a, z in shard_chunks(gb, self.world))
        self.cand_stride = REC_BYTES * (self.cap + 1)
        kw = dict(device=d.dev)
        self.cand = torch.zeros(d.items * self.cand_stride, dtype=torch.uint8, **kw)
        self.gathered = torch.zeros(self.world * self.cand.numel(), dtype=torch.uint8, **kw)
        self.rows = d.items * d.GH
        self.rec = torch.zeros(self.rows * (self.D + 2), dtype=torch.float32, **kw)
        self.rec_all = torch.zeros(self.world * self.rec.numel(), dtype=torch.float32, **kw)
        self.gen_count = d.gen_count  # the GLOBAL generated count on every shard

    # ---------------------------------------------------------------- state
    def prefill(self, keys, values):
        """keys/values: this shard's prompt slice [B, Hkv, hi-lo, D] (bf16)."""
        if keys.shape[2] != self.local_len:
            raise ValueError(f"shard {self.rank} expects {self.local_len} prompt tokens")
        self.dec.prefill(keys, values, bounds=self.local_bounds)

    @property
    def items_per_unit(self):
        return self.G if self.dec.per_head else 1

    # ---------------------------------------------------------------- phases
    def candidates(self, q, k_new=None, v_new=None, stream=None):
        d = self.dec
        st = _lib.stream_handle(stream)
        tail = self.owns_tail
        _lib.call("dhsa_decode_candidates_bf16", _lib.ptr(q), _lib.ptr(d.sketch),
                  d.nc_cap * d.D, _lib.ptr(d.sinfo), _lib.ptr(d.centroids), d.nc_cap * d.D,
                  _lib.ptr(d.gen_sum), _lib.ptr(d.gen_count),
                  _lib.ptr(k_new) if tail else 0, _lib.ptr(v_new) if tail else 0,
                  _lib.ptr(d.k_cache) if tail else 0, _lib.ptr(d.v_cache) if tail else 0,
                  d.L_cap * d.D, d._layout(), d.U, d.G, d.D, _lib.AGG[d.agg], d.budget,
                  self.spec, _lib.ptr(self.cand), self.cand_stride, self.cap,
                  _lib.ptr(d.approx), d.sc_stride, _lib.ptr(d.scratch), _lib.ptr(d.progress),
                  st)

    def select(self, gathered=None, stream=None):
        d = self.dec
        g = self.gathered if gathered is None else gathered
        _lib.call("dhsa_split_select", _lib.ptr(g), self.world, self.cand.numel(),
                  self.cand_stride, self.cap, d.items, self.items_per_unit,
                  _lib.ptr(d.gen_count), _lib.ptr(d.plen), self.total_prompt, d.budget,
                  self.rank, 1 if self.owns_tail else 0, d.tile, _lib.ptr(d.tiles), d.tile_cap,
                  _lib.ptr(d.ntiles), 1, _lib.stream_handle(stream))

    def attend(self, q, stream=None):
        """Attention over this shard's tiles -> (m, l, acc) records."""
        d = self.dec
        if d.attn_mode == "stream":
            d._attn(q, None, _lib.stream_handle(stream), records=self.rec)
            return
        _lib.call("dhsa_attn_partials", _lib.ptr(q), _lib.ptr(d.k_cache), _lib.ptr(d.v_cache),
                  d.L_cap * d.D, d.L_cap, d.items, self.items_per_unit, d.GH, d.D,
                  _lib.ptr(d.tiles), d.tile_cap, _lib.ptr(d.ntiles), d.splits,
                  _lib.ptr(self.rec), _lib.ptr(d.ws), _lib.ptr(d.counters),
                  _lib.stream_handle(stream))

    def merge(self, out, rec_all=None, stream=None):
        r = self.rec_all if rec_all is None else rec_all
        _lib.call("dhsa_merge_partials", _lib.ptr(r), self.world, self.rec.numel(), self.rows,
                  self.D, _lib.BF16, _lib.ptr(out), _lib.stream_handle(stream))

    # ---------------------------------------------------------------- step
    def step(self, q, k_new, v_new, comm, out=None):
        """One decode step with a real collective (every rank calls it)."""
        if out is None:
            out = torch.empty(self.B, self.Hq, self.D, dtype=torch.bfloat16, device=self.dec.dev)
        self.launch(q, k_new, v_new, comm, out)
        self.dec.steps += 1
        return out

    def launch(self, q, k_new, v_new, comm, out, stream=None):
        """Enqueue one step on the current (or given) stream: 4 kernels + 2
        all-gathers; graph-capturable when the collective is."""
        if self.direct:
            self.dec.launch(q, k_new, v_new, out, stream=stream)
            return
        self.candidates(q, k_new, v_new, stream)
        if comm.world == 1:  # one shard: the gathered rows are this shard's own
            self.select(self.cand, stream=stream)
            self.attend(q, stream)
            self.merge(out, self.rec, stream=stream)
            return
        comm.all_gather(self.gathered, self.cand)
        self.select(stream=stream)
        self.attend(q, stream)
        comm.all_gather(self.rec_all, self.rec)
        self.merge(out, stream=stream)

    @property
    def kernels_per_step(self) -> int:
        """sketch stream, candidate select, global walk, attention, merge (+
        the segment merge); one shard: the plain decode step's kernels."""
        return self.dec.kernels_per_step if self.direct else 5 + (
            self.dec.kernels_per_step - 3)

    def selection(self):
        """This shard's tiles (local token ranges) of the last step."""
        return self.dec.selection()

    def check_capacity(self):
        """Raise if a candidate row or tile list overflowed in the last step."""
        if int(self.dec.ntiles.min().item()) < 0:
            raise _lib.DhsaError("split-KV candidate or tile capacity exceeded")

    def bytes_per_step(self) -> dict:
        """Algorithmic HBM bytes of this shard's step (sketch + selected K/V +
        q/o + candidate/record exchange buffers)."""
        d = self.dec
        nc = ((self.local_len + self.block - 1) // self.block if self.local_bounds is None
              else len(self.local_bounds) - 1)
        return {"sketch": d.U * nc * d.D * 2,
                "exchange": (self.cand.numel() + self.rec.numel() * 4) * self.world}


class SplitKVGroup:
    """W shards driven from one process on one device (the collectives become
    concatenations).  Used for single-GPU parity of the split-KV path and as
    the 1-GPU split-KV baseline; the arithmetic is the multi-GPU one."""

    def __init__(self, batch, q_heads, kv_heads, head_dim, prompt_len, world, **kw):
        self.shards = [SplitKVShard(batch, q_heads, kv_heads, head_dim, prompt_len, rank=r,
                                    world=world, **kw) for r in range(world)]
        self.world = world

    def prefill(self, keys, values):
        for s in self.shards:
            s.prefill(keys[:, :, s.lo:s.hi], values[:, :, s.lo:s.hi])

    def step(self, q, k_new, v_new, out=None):
        sh = self.shards
        for s in sh:
            s.candidates(q, k_new, v_new)
        gathered = torch.cat([s.cand for s in sh])
        for s in sh:
            s.select(gathered)
            s.attend(q)
        rec_all = torch.cat([s.rec for s in sh])
        if out is None:
            out = torch.empty(sh[0].B, sh[0].Hq, sh[0].D, dtype=torch.bfloat16,
                              device=sh[0].dec.dev)
        sh[0].merge(out, rec_all)
        for s in sh:
            s.dec.steps += 1
        return out

    def launch(self, q, k_new, v_new, out, stream=None):
        """One step enqueued on the current stream without host allocation
        (graph-capturable): the exchanges are device copies into shard 0's
        gather buffers, which every shard's global walk reads."""
        sh = self.shards
        g, n = sh[0].gathered, sh[0].cand.numel()
        for r, s in enumerate(sh):
            s.candidates(q, k_new, v_new, stream)
            g[r * n:(r + 1) * n].copy_(s.cand)
        for s in sh:
            s.select(g, stream=stream)
            s.attend(q, stream)
        ra, m = sh[0].rec_all, sh[0].rec.numel()
        for r, s in enumerate(sh):
            ra[r * m:(r + 1) * m].copy_(s.rec)
        sh[0].merge(out, ra, stream=stream)

    def selection(self):
        """Per selection row: the union of every shard's tiles in GLOBAL token
        positions (generated tokens follow the prompt)."""
        per = [s.selection() for s in self.shards]
        rows = []
        for i in range(len(per[0])):
            parts = []
            for s, tl in zip(self.shards, per):
                for st, cnt in tl[i]:
                    parts.append((int(st) + s.lo, int(cnt)))
            rows.append(parts)
        return rows
