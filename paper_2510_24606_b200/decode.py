"""Batched DHSA decode engine — the north-star hot path.

One decode step for a batch of B sequences with Hq query heads sharing Hkv
key/value heads (group size G = Hq / Hkv), each sequence holding a prompt of
P_b tokens split into static ``block``-token chunks plus g generated tokens:

  1. ``dhsa_decode_score``  fp64 q . centroid scores for every prompt chunk
     and the generated chunk (Algorithm 2, masks.py:153-173), reduced over
     the G heads of a group (harness.py:288-306 max/mean) or kept per head;
     folds the new key into the fp64 running sum and appends k/v to the cache.
  2. ``dhsa_decode_select`` the exact token-budget Top-K (masks.py:103-122)
     as a weighted radix-select chunk walk -> tiles of <= 64 tokens + self.
  3. ``dhsa_attn``          softmax attention of the G heads over the selected
     tiles (core.py:113-118): TMA + mma.sync for bf16, FFMA for fp32,
     split-KV with an in-kernel (m, l, acc) merge.
  4. ``dhsa_decode_advance`` g += 1.

Memory layout in HBM (all dense, allocated once):
  K/V cache  [B, Hkv, L_cap, D]  (dtype; = block-contiguous [B,Hkv,L/64,64,D])
  centroids  [B, Hkv, N_c, D]     fp64 (built once per prompt by K1)
  gen_sum    [B, Hkv, D]          fp64, gen_count/plen [B*Hkv] int32
  scores     [B*Hsel, N_c+1]      fp64, tiles [B*Hsel, cap, 2] int32
"""

from __future__ import annotations

import math

import torch

from . import _lib

_DT = {torch.bfloat16: _lib.BF16, torch.float32: _lib.F32, torch.float64: _lib.F64}


def default_splits(items: int, tiles_per_item: int, sms: int = 148) -> int:
    """Split-KV factor (fixed-split attention): ~8 tiles per CTA for many
    items; with few items (C1: 8 heads x 17 tiles) as many CTAs as fill the
    SMs twice, down to one tile each (C1: 53 -> 31 us/step at 16 splits)."""
    by_work = max(1, math.ceil(tiles_per_item / 8))
    by_fill = max(1, math.ceil(2 * sms / max(items, 1)))
    return int(max(1, min(16, max(min(by_work, 8), min(by_fill, tiles_per_item)))))


class SparseDecoder:
    """Batched sparse decode over a KV cache resident in HBM.

    ``budget`` is the reference's token budget (masks.topk_row); with
    ``top_k`` blocks it defaults to ``top_k * block + 1`` (K whole blocks plus
    self).  ``agg`` selects group-shared selection ("max" / "mean", one
    selection per kv head, harness.aggregated_chunk_scores semantics) or
    per-q-head selection ("none", one DecodeSession per head)."""

    def __init__(self, batch, q_heads, kv_heads, head_dim, max_len, *, block=64, top_k=64,
                 budget=None, dtype=torch.bfloat16, agg="max", tile=64, splits=None,
                 device=None, scoring=None, attn_mode=None, max_chunks=None):
        _lib.require_cuda()
        if q_heads % kv_heads:
            raise ValueError("q_heads must be a multiple of kv_heads")
        if dtype not in _DT:
            raise ValueError(f"unsupported dtype {dtype}")
        if agg not in _lib.AGG:
            raise ValueError(f"unknown aggregation {agg!r}")
        self.B, self.Hq, self.Hkv, self.D = batch, q_heads, kv_heads, head_dim
        self.G = q_heads // kv_heads
        self.U = batch * kv_heads
        self.block = int(block)
        self.budget = int(budget if budget is not None else top_k * block + 1)
        if self.budget < 1:
            raise ValueError("budget must be >= 1")
        self.dtype = dtype
        self.code = _DT[dtype]
        self.agg = agg
        self.per_head = agg == "none"
        self.tile = int(tile)
        self.dev = torch.device(device) if device is not None else torch.device("cuda")
        self.L_cap = ((int(max_len) + 64 - 1) // 64) * 64 + 64
        # chunk capacity per unit: the static grid's count, or more for
        # dynamic (e.g. NMS) boundaries with short chunks
        self.nc_cap = int(max_chunks) if max_chunks else (int(max_len) + self.block - 1) // self.block
        kw = dict(device=self.dev)
        self.k_cache = torch.zeros(batch, kv_heads, self.L_cap, head_dim, dtype=dtype, **kw)
        self.v_cache = torch.zeros_like(self.k_cache)
        self.centroids = torch.zeros(batch, kv_heads, self.nc_cap, head_dim, dtype=torch.float64, **kw)
        self.gen_sum = torch.zeros(self.U, head_dim, dtype=torch.float64, **kw)
        self.gen_count = torch.zeros(self.U, dtype=torch.int32, **kw)
        self.plen = torch.zeros(self.U, dtype=torch.int32, **kw)
        self.items = self.U * self.G if self.per_head else self.U
        self.GH = 1 if self.per_head else self.G
        self.scores = torch.empty(self.items, self.nc_cap + 1, dtype=torch.float64, **kw)
        r = self.budget - 1
        self.tile_cap = min(self.nc_cap + 1, r) + r // self.tile + 2
        self.tiles = torch.zeros(self.items, self.tile_cap, 2, dtype=torch.int32, **kw)
        self.ntiles = torch.zeros(self.items, dtype=torch.int32, **kw)
        tiles_per_item = math.ceil(r / self.tile) + 2
        self.splits = int(splits) if splits else default_splits(self.items, tiles_per_item)
        # attention: "stream" (persistent stream-K grid, bf16) or "split"
        # (a fixed split-KV factor per item, every dtype)
        bf16_tc = dtype == torch.bfloat16 and head_dim in (64, 128)
        self.attn_mode = attn_mode or ("stream" if bf16_tc and not splits else "split")
        if self.attn_mode == "stream" and not bf16_tc:
            raise ValueError("stream attention needs bf16 and D in {64, 128}")
        self.tiles_hint = min(self.tile_cap, tiles_per_item + 1)
        if self.attn_mode == "stream":
            nbytes = _lib.load().dhsa_attn_stream_workspace_size(self.items, self.GH, head_dim)
        else:
            nbytes = _lib.load().dhsa_attn_workspace_size(self.code, self.items, self.GH,
                                                          head_dim, self.splits)
        self.ws = torch.empty(max(nbytes, 8), dtype=torch.uint8, **kw)
        ncnt = max(self.items, _lib.load().dhsa_attn_stream_counters(self.items))
        self.counters = torch.zeros(ncnt, dtype=torch.int32, **kw)
        self.max_prompt = 0
        self.max_chunks = 0
        self.bounds = self.nchunks = None
        self.chunk_counts = [0] * self.U
        self.steps = 0
        # scoring: "sketch" (fp16 centroid sketch + certified fp64 re-scoring at
        # the cut; sketch stream + select kernels) or "fp64" (stream fp64 centroids)
        fast_ok = dtype == torch.bfloat16 and head_dim in (64, 128) and self.G in (1, 2, 4, 8)
        self.scoring = scoring or ("sketch" if fast_ok else "fp64")
        if self.scoring == "sketch":
            if not fast_ok:
                raise ValueError("sketch scoring needs bf16, D in {64,128}, G in {1,2,4,8}")
            self.sketch = torch.zeros(batch, kv_heads, self.nc_cap, head_dim, dtype=torch.float16,
                                      **kw)
            self.sinfo = torch.zeros(self.U, 4, dtype=torch.float32, **kw)
            # rows padded to a multiple of 4 floats (the select reads float4)
            self.sc_stride = (self.nc_cap + 1 + 3) // 4 * 4
            self.approx = torch.empty(self.items, self.sc_stride, dtype=torch.float32, **kw)
            self.ready = torch.zeros(self.items, dtype=torch.int32, **kw)
            self.progress = torch.zeros(self.U, dtype=torch.int32, **kw)
            per_unit = _lib.load().dhsa_sketch_select_scratch_size(self.nc_cap)
            self.scratch = torch.empty(self.U * per_unit, dtype=torch.uint8, **kw)
        # fp64 scoring: the select kernel's global scratch for very long units
        per_row = _lib.load().dhsa_select_scratch_size(self.nc_cap + 1)
        self.sel_scratch = (torch.empty(per_row * self.items, dtype=torch.uint8, **kw)
                            if per_row > 0 and self.scoring == "fp64" else None)

    # ------------------------------------------------------------------
    def _layout(self):
        if self.bounds is not None:  # explicit per-unit boundaries (chunking.py:23-39)
            return _lib.layout(bounds=self.bounds, bounds_stride=self.nc_cap + 1,
                               nchunks=self.nchunks, plen=self.plen, max_chunks=self.max_chunks)
        return _lib.layout(plen=self.plen, block=self.block, max_chunks=self.max_chunks)

    def _set_bounds(self, bounds, P):
        """bounds: None (static grid of `block`), one boundary list shared by
        every unit, or one list per unit (B*Hkv lists, unit = b*Hkv + h) —
        the reference's `bounds` ([0, ..., P], strictly increasing; validated
        like chunking.check_boundaries)."""
        self.bounds = self.nchunks = None
        self.chunk_counts = [(P + self.block - 1) // self.block] * self.U
        if bounds is None:
            return
        from .chunking import check_boundaries

        lists = [bounds] * self.U if bounds and not hasattr(bounds[0], "__len__") else list(bounds)
        if len(lists) != self.U:
            raise ValueError(f"expected one boundary list per unit ({self.U}), got {len(lists)}")
        rows = []
        for b in lists:
            b = check_boundaries([int(x) for x in b], P)
            if len(b) - 1 > self.nc_cap:
                raise ValueError(f"{len(b) - 1} chunks exceed max_chunks={self.nc_cap}")
            rows.append(b + [P] * (self.nc_cap + 1 - len(b)))
        self.chunk_counts = [len(b) - 1 for b in lists]
        self.bounds = torch.tensor(rows, dtype=torch.int32, device=self.dev)
        self.nchunks = torch.tensor(self.chunk_counts, dtype=torch.int32, device=self.dev)

    def prefill(self, keys, values, prompt_len=None, bounds=None):
        """Load prompt K/V [B, Hkv, P, D] into the cache and build the fp64
        centroid cache (K1, chunk_repr.aggregate_rows semantics).  ``bounds``
        gives dynamic chunk boundaries (see ``_set_bounds``); default is the
        static grid of ``block`` tokens (chunking.static_boundaries)."""
        P = keys.shape[2] if prompt_len is None else int(prompt_len)
        if P < 1 or P + 1 > self.L_cap - 64:
            raise ValueError("prompt does not fit the cache")
        if bounds is None and (P + self.block - 1) // self.block > self.nc_cap:
            raise ValueError(f"a {P}-token prompt has {(P + self.block - 1) // self.block} "
                             f"chunks of {self.block}; the decoder holds {self.nc_cap}")
        # the captured step graphs bake in the chunk layout (max_chunks, the
        # bounds / nchunks pointers): a new prompt needs new captures
        self._graph = self._pgraph = None
        self._set_bounds(bounds, P)
        self.k_cache[:, :, :P].copy_(keys[:, :, :P])
        self.v_cache[:, :, :P].copy_(values[:, :, :P])
        self.plen.fill_(P)
        self.gen_count.zero_()
        self.gen_sum.zero_()
        self.max_prompt = P
        self.max_chunks = max(self.chunk_counts)
        self.steps = 0
        st = _lib.stream_handle()
        _lib.call("dhsa_centroids", self.code, _lib.ptr(self.k_cache), self.L_cap * self.D,
                  self.D, self.U, self._layout(), 1, _lib.ptr(self.centroids),
                  self.nc_cap * self.D, st)
        if self.scoring == "sketch":
            _lib.call("dhsa_sketch_build", _lib.ptr(self.centroids), self.nc_cap * self.D, self.D,
                      self.U, self._layout(), _lib.ptr(self.sketch), self.nc_cap * self.D,
                      _lib.ptr(self.sinfo), st)

    def step(self, q, k_new, v_new, out=None):
        """One decode step.  q [B, Hq, D], k_new/v_new [B, Hkv, D] (cache
        dtype, contiguous, on device).  Returns attention output [B, Hq, D]."""
        if self.max_prompt + self.steps + 1 > self.L_cap - 64:
            raise RuntimeError("KV cache capacity exhausted")
        if out is None:
            out = torch.empty(self.B, self.Hq, self.D, dtype=self.dtype, device=self.dev)
        self.launch(q, k_new, v_new, out)
        self.steps += 1
        return out

    def step_host(self, q, k_new, v_new, out):
        """Serving entry point: one decode step from HOST tensors (pinned for
        asynchronous copies) to a host output, replaying one captured CUDA
        graph of the step's kernels.  q [B, Hq, D], k_new/v_new [B, Hkv, D],
        out [B, Hq, D] in the cache dtype.  Inputs go to static device
        buffers (the graph's arguments); every step-dependent value
        (generated count, running sum, flags) lives in device memory, so one
        graph serves every step.  The copies, the graph and the output copy
        are ordered on the current stream; returns ``out`` (valid once that
        stream is synchronised)."""
        if self.max_prompt + self.steps + 1 > self.L_cap - 64:
            raise RuntimeError("KV cache capacity exhausted")
        if getattr(self, "_graph", None) is None:
            kw = dict(dtype=self.dtype, device=self.dev)
            self._gq = torch.empty(self.B, self.Hq, self.D, **kw)
            self._gk = torch.empty(self.B, self.Hkv, self.D, **kw)
            self._gv = torch.empty(self.B, self.Hkv, self.D, **kw)
            self._go = torch.empty(self.B, self.Hq, self.D, **kw)
            # warm every kernel module outside capture without advancing state
            self._graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(self._graph, stream=side):
                self.launch(self._gq, self._gk, self._gv, self._go, stream=side)
            torch.cuda.current_stream().wait_stream(side)
        self._gq.copy_(q, non_blocking=True)
        self._gk.copy_(k_new, non_blocking=True)
        self._gv.copy_(v_new, non_blocking=True)
        self._graph.replay()
        out.copy_(self._go, non_blocking=True)
        self.steps += 1
        return out

    def packed_layout(self):
        """Element offsets of q / k_new / v_new in the packed step input of
        ``step_host_packed`` ([q | k | v], cache dtype)."""
        nq, nk = self.B * self.Hq * self.D, self.B * self.Hkv * self.D
        return (0, nq), (nq, nq + nk), (nq + nk, nq + 2 * nk)

    def step_host_packed(self, qkv, out):
        """``step_host`` with the step's inputs packed in ONE pinned host
        tensor [q | k_new | v_new] (flattened, cache dtype): one host->device
        copy per step instead of three."""
        if self.max_prompt + self.steps + 1 > self.L_cap - 64:
            raise RuntimeError("KV cache capacity exhausted")
        (q0, q1), (k0, k1), (v0, v1) = self.packed_layout()
        if getattr(self, "_pgraph", None) is None:
            self._pin = torch.empty(v1, dtype=self.dtype, device=self.dev)
            self._po = torch.empty(self.B, self.Hq, self.D, dtype=self.dtype, device=self.dev)
            q = self._pin[q0:q1].view(self.B, self.Hq, self.D)
            k = self._pin[k0:k1].view(self.B, self.Hkv, self.D)
            v = self._pin[v0:v1].view(self.B, self.Hkv, self.D)
            self._pgraph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(self._pgraph, stream=side):
                self.launch(q, k, v, self._po, stream=side)
            torch.cuda.current_stream().wait_stream(side)
        if (qkv.numel() != v1 or qkv.dtype != self.dtype or out.dtype != self.dtype
                or tuple(out.shape) != (self.B, self.Hq, self.D)):
            raise ValueError("step_host_packed: qkv must hold [q | k_new | v_new] "
                             f"({v1} elements of {self.dtype}), out [B, Hq, D] of {self.dtype}")
        self._pin.copy_(qkv.view(-1), non_blocking=True)
        self._pgraph.replay()
        out.copy_(self._po, non_blocking=True)
        self.steps += 1
        return out

    def launch(self, q, k_new, v_new, out, stream=None):
        """Enqueue one step (graph-capturable): 3 kernels with sketch scoring
        (sketch stream, select + state update, attention), 4 with fp64 scoring."""
        for _, fn in self.stages(q, k_new, v_new, out, stream):
            fn()

    def stages(self, q, k_new, v_new, out, stream=None):
        """The launches of one step as (kernel name, thunk) pairs, in order."""
        st = _lib.stream_handle(stream)
        lay = self._layout()
        agg = _lib.AGG[self.agg]
        attn = ("attn", lambda: self._attn(q, out, st))
        if self.scoring == "sketch":
            def fused():
                _lib.call("dhsa_decode_step_bf16", _lib.ptr(q), _lib.ptr(self.sketch),
                          self.nc_cap * self.D, _lib.ptr(self.sinfo), _lib.ptr(self.centroids),
                          self.nc_cap * self.D, _lib.ptr(self.gen_sum), _lib.ptr(self.gen_count),
                          _lib.ptr(k_new), _lib.ptr(v_new), _lib.ptr(self.k_cache),
                          _lib.ptr(self.v_cache), self.L_cap * self.D, lay, self.U, self.G,
                          self.D, agg, self.budget, self.tile, _lib.ptr(self.tiles),
                          self.tile_cap, _lib.ptr(self.ntiles), _lib.ptr(self.approx),
                          self.sc_stride, _lib.ptr(self.scratch), _lib.ptr(self.ready), 1,
                          _lib.ptr(self.progress), st)
            return [("score_select", fused), attn]

        def score():
            _lib.call("dhsa_decode_score", self.code, _lib.ptr(q), _lib.ptr(self.centroids),
                      self.nc_cap * self.D, _lib.ptr(self.gen_sum), _lib.ptr(self.gen_count),
                      _lib.ptr(k_new), _lib.ptr(v_new), _lib.ptr(self.k_cache),
                      _lib.ptr(self.v_cache), self.L_cap * self.D, lay, self.U, self.G, self.D,
                      agg, _lib.ptr(self.scores), self.nc_cap + 1, st)

        def select():
            _lib.call("dhsa_decode_select", _lib.ptr(self.scores), self.nc_cap + 1, lay,
                      _lib.ptr(self.gen_count), self.U, self.G if self.per_head else 1,
                      self.budget, self.tile, _lib.ptr(self.tiles), self.tile_cap,
                      _lib.ptr(self.ntiles), _lib.ptr(self.sel_scratch), st)

        def advance():
            _lib.call("dhsa_decode_advance", _lib.ptr(self.gen_count), self.U, st)

        return [("decode_score", score), ("decode_select", select), attn, ("advance", advance)]

    def _attn(self, q, out, st, records=None):
        ready = _lib.ptr(self.ready) if self.scoring == "sketch" else 0
        if self.attn_mode == "stream":
            _lib.call("dhsa_attn_stream", _lib.ptr(q), _lib.ptr(self.k_cache),
                      _lib.ptr(self.v_cache), self.L_cap * self.D, self.L_cap, self.items,
                      self.G if self.per_head else 1, self.GH, self.D, _lib.ptr(self.tiles),
                      self.tile_cap, _lib.ptr(self.ntiles), self.tiles_hint, _lib.ptr(out),
                      _lib.ptr(records), _lib.ptr(self.ws), _lib.ptr(self.counters),
                      ready if records is None else 0, st)
            return
        if records is not None:
            raise ValueError("records need the stream attention mode")
        _lib.call("dhsa_attn", self.code, _lib.ptr(q), _lib.ptr(self.k_cache),
                  _lib.ptr(self.v_cache), self.L_cap * self.D, self.L_cap, self.items,
                  self.G if self.per_head else 1, self.GH, self.D, _lib.ptr(self.tiles),
                  self.tile_cap, _lib.ptr(self.ntiles), self.splits, _lib.ptr(out),
                  _lib.ptr(self.ws), _lib.ptr(self.counters),
                  _lib.ptr(self.ready) if self.scoring == "sketch" else 0, st)

    @property
    def kernels_per_step(self) -> int:
        """Kernels of one step: sketch stream + select (or score, select,
        advance) + attention, + the segment merge of the stream attention
        when an item spans more than one segment."""
        n = 3 if self.scoring == "sketch" else 4
        if self.attn_mode == "stream" and self.tiles_hint > max(12, -(-self.tiles_hint // 32)):
            n += 1
        return n

    # ------------------------------------------------------------------
    def selection(self):
        """Host copy of the last step's selection: list over selection rows of
        (start, count) tiles (self tile last)."""
        t = self.tiles.cpu().numpy()
        n = self.ntiles.cpu().numpy()
        return [t[i, : n[i]].copy() for i in range(self.items)]

    def cost_counters(self, counters=None):
        """The reference's cost accounting (masks.CostCounters, masks.py:38-52)
        of every decode step since the last prefill, computed analytically
        (the kernels count nothing): per step with g generated tokens, each
        q head scores its unit's N_c prompt chunks + the generated chunk
        (g >= 1) + the singleton (masks.py:166-167; group aggregation counts
        one score per head, harness.py:300-301), and each selection row —
        one per kv unit for "max"/"mean", one per q head for "none" — admits
        min(budget, P + g + 1) pairs (masks.py:171-172).  Adds to
        ``counters`` (a fresh CostCounters if None) and returns it."""
        from .masks import CostCounters

        c = CostCounters() if counters is None else counters
        P, n = self.max_prompt, self.steps
        if n == 0:
            return c
        nc_heads = sum(self.chunk_counts) * self.G  # sum over q heads of N_c
        # sum_{g=0}^{n-1} (N_c + [g >= 1] + 1) per q head
        c.add_score_ops(nc_heads * n + self.U * self.G * ((n - 1) + n))
        # sum_{g=0}^{n-1} min(budget, P + g + 1) per selection row
        lo, hi = P + 1, P + n  # row sizes before the budget clamp
        full = max(0, min(hi, self.budget - 1) - lo + 1) if lo < self.budget else 0
        grow = (lo + lo + full - 1) * full // 2 if full else 0
        c.add_attended(self.items * (grow + (n - full) * self.budget))
        return c

    def bytes_per_step(self) -> dict:
        """Algorithmic (unique) HBM bytes of one step, the roofline numerator
        (fp64 centroids + selected K/V rows + q/o)."""
        esz = torch.finfo(self.dtype).bits // 8
        P, g = self.max_prompt, self.steps
        # centroid stream: fp16 sketch (the fp64 re-scoring of the few chunks
        # at the cut is not counted) or fp64 centroids
        cent = sum(self.chunk_counts) * self.D * (2 if self.scoring == "sketch" else 8)
        sel_tokens = min(self.budget, P + g + 1)
        per_sel = sel_tokens * self.D * esz * 2
        kv = (self.items if self.per_head else self.U) * per_sel
        qo = 2 * self.B * self.Hq * self.D * esz
        return {"centroids": cent, "kv": kv, "qo": qo, "total": cent + kv + qo}
