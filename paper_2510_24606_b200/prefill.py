"""Batched sparse prefill (config C5) on the tcgen05 tensor cores.

For B sequences of L tokens with Hq query heads sharing Hkv key/value heads
(G = Hq / Hkv), computes the reference's prefill path for every head —
prefill_mask (masks.py:143-150: chunk centroids of Q and K, S_c = Q_c K_c^T,
token-budget Top-K per row with forced self) followed by
dense_attention(seq, mask) (core.py:98-119) — without ever materialising the
L x L upsampled score matrix:

  1. ``dhsa_centroids``       Q_c [B*Hq, N_c, D], K_c [B*Hkv, N_c, D] in fp64
                              (chunk_repr.aggregate_rows, bit-exact);
  2. ``dhsa_prefill_scores``  S_c per selection row, aggregated over the G
                              q-heads of a kv group ("max" / "mean",
                              harness.py:288-306) or per head ("none");
  3. ``dhsa_prefill_plan``    per (selection row, query chunk) the walk-order
                              list of selected chunks;
  4. ``dhsa_prefill_attn``    tcgen05.mma S = Q K^T / O += P V over the planned
                              64-token KV blocks, per-row masks, online softmax
                              (a persistent plan-pulling grid for short plans).

Layouts (dense, bf16): q [B, Hq, L, D], k/v [B, Hkv, L, D], out [B, Hq, L, D].
D = 128.  Chunks: the static 64-token grid (chunking.static_boundaries) or
explicit boundary lists of any chunk lengths (``bounds``; query tiles and KV
blocks are cut at chunk starts, at most 64 rows each).
"""

from __future__ import annotations

import torch

from . import _lib


_TOK = 64       # KV block / query tile rows of the tcgen05 kernel
_PLAN_CAP = 544  # plan entries a CTA stages in shared memory


class SparsePrefill:
    """Sparse prefill attention with the reference's token budget.

    ``budget`` is the reference's per-row token budget (masks.topk_row); with
    ``top_k`` blocks it defaults to ``top_k * block + 1`` (K whole blocks +
    self).  ``agg``: "max" / "mean" (one selection per kv group) or "none"
    (one selection per q head).

    ``bounds`` (here or per call / ``set_bounds``): None = the static grid of
    ``block`` tokens (chunking.static_boundaries); one boundary list shared by
    every kv unit; or one list per kv unit (B * Hkv lists, unit = b * Hkv + h)
    — any chunk lengths, e.g. ``nms_boundaries`` over predictor scores
    (SURVEY.md section 8(f) row 1).  Chunks longer than 64 tokens become
    several 64-row query tiles / KV blocks; the selection semantics are
    exactly the reference's walk over whole chunks."""

    def __init__(self, batch, q_heads, kv_heads, head_dim, seq_len, *, block=64, top_k=16,
                 budget=None, agg="max", device=None, bounds=None):
        _lib.require_cuda()
        if q_heads % kv_heads:
            raise ValueError("q_heads must be a multiple of kv_heads")
        if agg not in _lib.AGG:
            raise ValueError(f"unknown aggregation {agg!r}")
        if head_dim != 128 or block != 64:
            raise ValueError("the tcgen05 prefill path needs head_dim 128 and 64-token chunks")
        self.B, self.Hq, self.Hkv, self.D, self.L = batch, q_heads, kv_heads, head_dim, seq_len
        self.G = q_heads // kv_heads
        self.U = batch * kv_heads
        self.block = block
        self.budget = int(budget if budget is not None else top_k * block + 1)
        if self.budget < 1:
            raise ValueError("budget must be >= 1")
        self.agg = agg
        self.S = self.U * self.G if agg == "none" else self.U
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.dev = dev
        self.plen_q = torch.full((self.U * self.G,), seq_len, dtype=torch.int32, device=dev)
        self.plen_k = torch.full((self.U,), seq_len, dtype=torch.int32, device=dev)
        self.counters = torch.zeros(2, dtype=torch.int32, device=dev)  # persistent attention
        # __call__ verifies the plan capacity (one device sync); benchmarks that
        # time back-to-back calls switch it off and call check_capacity() once
        self.checked = True
        self.nc = self.cap = 0
        self.set_bounds(bounds)

    # ---------------------------------------------------------- chunk layout
    def set_bounds(self, bounds=None):
        """Select the chunk layout of the following calls (see the class doc)."""
        import numpy as np

        from .chunking import check_boundaries

        L, U = self.L, self.U
        if bounds is None:
            self.bounds_host = None
            nc = (L + self.block - 1) // self.block
            cap = _lib.load().dhsa_prefill_plan_capacity(self.budget, self.block)
            if cap > _PLAN_CAP:
                raise ValueError("budget too large for the prefill plan (<= 542 blocks per row)")
            self._chunks = None
            self._alloc(nc, cap)
            return
        b0 = list(bounds)
        per_unit = len(b0) > 0 and not np.isscalar(b0[0])
        lists = [check_boundaries(b, L) for b in b0] if per_unit else [check_boundaries(b0, L)]
        if per_unit and len(lists) != U:
            raise ValueError(f"need one boundary list per kv unit ({U}), got {len(lists)}")
        shared = not per_unit
        ncs = [len(b) - 1 for b in lists]
        nc = max(ncs)
        if nc > 10240:  # plan-kernel shared memory (20 B per chunk) and the S x n x n scores
            raise ValueError(f"{nc} chunks exceed the prefill limit of 10240 per unit")
        # worst-case plan entries: blocks of the chunks a walk of budget-1
        # tokens can touch (the most chunks: the shortest ones), + the diagonal
        cap = 2
        for b in lists:
            ln = np.diff(np.asarray(b, dtype=np.int64))
            nblk = (ln + _TOK - 1) // _TOK
            pref = np.concatenate([[0], np.cumsum(nblk)])
            srt = np.concatenate([[0], np.cumsum(np.sort(ln))])
            most = int(np.searchsorted(srt, self.budget - 1, side="left")) + 1
            walk_blocks = (self.budget - 1 + _TOK - 1) // _TOK + most
            need = np.minimum(pref[:-1], walk_blocks) + nblk
            cap = max(cap, int(need.max()))
        if cap > _PLAN_CAP:
            raise ValueError(f"budget {self.budget} over these chunks needs up to {cap} plan "
                             f"entries per query chunk (limit {_PLAN_CAP})")
        kb = np.full((len(lists), nc + 1), L, dtype=np.int32)
        for u, b in enumerate(lists):
            kb[u, :len(b)] = b
        # query tiles per unit, heaviest (latest) first; chunk -1 pads
        tiles = []
        for b in lists:
            t = [(l, k) for l in range(len(b) - 1)
                 for k in range((b[l + 1] - b[l] + _TOK - 1) // _TOK)]
            tiles.append(sorted(t, key=lambda x: (-x[0], -x[1])))
        T = max(len(t) for t in tiles)
        qt = np.full((U, T, 2), -1, dtype=np.int32)
        qt[:, :, 1] = 0
        for u in range(U):
            t = tiles[0 if shared else u]
            qt[u, :len(t)] = t
        dev = self.dev
        self.bounds_host = lists
        self._kb = torch.from_numpy(kb).to(dev)
        self._knc = torch.tensor([ncs[0 if shared else u] for u in range(U)], dtype=torch.int32,
                                 device=dev)
        qrep = np.repeat(kb, 1 if shared else self.G, axis=0)
        self._qb = torch.from_numpy(np.ascontiguousarray(qrep)).to(dev)
        self._qnc = self._knc.repeat_interleave(self.G)
        self._qtiles = torch.from_numpy(qt).to(dev)
        self._stride = 0 if shared else nc + 1
        self._chunks = _lib.PrefillChunks(_lib.ptr(self._kb), self._stride, _lib.ptr(self._knc),
                                          _lib.ptr(self._qtiles), T)
        self._alloc(nc, cap)

    def _alloc(self, nc, cap):
        if nc == self.nc and cap == self.cap:
            return
        kw = dict(device=self.dev)
        self.nc, self.cap = nc, cap
        self.qc = torch.empty(self.U * self.G, nc, self.D, dtype=torch.float64, **kw)
        self.kc = torch.empty(self.U, nc, self.D, dtype=torch.float64, **kw)
        self.scores = torch.empty(self.S, nc, nc, dtype=torch.float64, **kw)
        self.plans = torch.zeros(self.S, nc, cap, 4, dtype=torch.int32, **kw)
        self.nplan = torch.zeros(self.S, nc, dtype=torch.int32, **kw)

    def _chunk_ptr(self):
        import ctypes

        return None if self._chunks is None else ctypes.byref(self._chunks)

    def _check(self, q, k, v):
        want_q = (self.B, self.Hq, self.L, self.D)
        want_k = (self.B, self.Hkv, self.L, self.D)
        for t, w, n in ((q, want_q, "q"), (k, want_k, "k"), (v, want_k, "v")):
            if tuple(t.shape) != w or t.dtype != torch.bfloat16 or not t.is_contiguous():
                raise ValueError(f"{n} must be a contiguous bf16 tensor of shape {w}")

    def stages(self, q, k, v, out, stream=None, row_stats=None):
        """The launches as (name, thunk) pairs, in order."""
        st = _lib.stream_handle(stream)
        nq, nk = self.U * self.G, self.U
        if self._chunks is None:
            lq = _lib.layout(plen=self.plen_q, block=self.block, max_chunks=self.nc)
            lk = _lib.layout(plen=self.plen_k, block=self.block, max_chunks=self.nc)
        else:
            lq = _lib.layout(bounds=self._qb, bounds_stride=self._stride, nchunks=self._qnc,
                             plen=self.plen_q, max_chunks=self.nc)
            lk = _lib.layout(bounds=self._kb, bounds_stride=self._stride, nchunks=self._knc,
                             plen=self.plen_k, max_chunks=self.nc)
        agg = _lib.AGG[self.agg]
        ch = self._chunk_ptr()

        def reps():
            _lib.call("dhsa_centroids", _lib.BF16, _lib.ptr(q), self.L * self.D, self.D, nq, lq, 1,
                      _lib.ptr(self.qc), self.nc * self.D, st)
            _lib.call("dhsa_centroids", _lib.BF16, _lib.ptr(k), self.L * self.D, self.D, nk, lk, 1,
                      _lib.ptr(self.kc), self.nc * self.D, st)

        def scores():
            _lib.call("dhsa_prefill_scores", _lib.ptr(self.qc), _lib.ptr(self.kc), self.U, self.G,
                      self.nc, self.D, agg, _lib.ptr(self.scores), st)

        def plan():
            _lib.call("dhsa_prefill_plan", _lib.ptr(self.scores), self.S, self.G, agg, self.nc,
                      self.L, self.block, self.budget, ch, self.cap, _lib.ptr(self.plans),
                      _lib.ptr(self.nplan), st)

        def attn():
            _lib.call("dhsa_prefill_attn", _lib.ptr(q), _lib.ptr(k), _lib.ptr(v), self.U, self.G,
                      self.L, self.D, self.block, agg, self.budget, self.nc, ch,
                      _lib.ptr(self.plans), _lib.ptr(self.nplan), self.cap, _lib.ptr(out),
                      _lib.ptr(self.counters), _lib.ptr(row_stats), st)

        return [("chunk_reps", reps), ("chunk_scores", scores), ("plan", plan), ("attn", attn)]

    def __call__(self, q, k, v, out=None, stream=None, row_stats=None):
        """Sparse prefill attention; ``row_stats`` (float32 [B, Hq, L, 2],
        optional) receives each row's softmax (m, l) over its selection."""
        self._check(q, k, v)
        if out is None:
            out = torch.empty_like(q)
        for _, fn in self.stages(q, k, v, out, stream, row_stats):
            fn()
        if self.checked:
            # a plan that overflowed its capacity leaves its query tile
            # unwritten: fail loudly instead of returning garbage rows
            self.check_capacity()
        return out

    def mask_bitsets(self, stream=None):
        """The last call's per-row selections as DHSAMSK1 bitsets
        [S, L, ceil(L/8)] uint8 on the device (selection row s = kv unit, or
        q head with agg "none"); ``serialization.save_mask_bitsets`` writes
        one selection row as the reference's mask file."""
        nbytes = (self.L + 7) // 8
        out = torch.empty(self.S, self.L, nbytes, dtype=torch.uint8, device=self.dev)
        _lib.call("dhsa_prefill_mask_bitsets", _lib.ptr(self.plans), _lib.ptr(self.nplan),
                  self.cap, self.S, self.G, _lib.AGG[self.agg], self.nc, self.L, self.block,
                  self.budget, self._chunk_ptr(), _lib.ptr(out), _lib.stream_handle(stream))
        return out

    def check_capacity(self):
        if int(self.nplan.min().item()) < 0:
            raise _lib.DhsaError("prefill plan capacity exceeded")

    def host_plans(self):
        """Host copies (plans, nplan) of the last call's plans."""
        return self.plans.cpu().numpy(), self.nplan.cpu().numpy()

    def unit_bounds(self, s: int):
        """Boundary list of selection row ``s``'s kv unit."""
        from .chunking import static_boundaries

        if self.bounds_host is None:
            return static_boundaries(self.L, self.block)
        u = s // self.G if self.agg == "none" else s
        return self.bounds_host[0 if len(self.bounds_host) == 1 else u]

    def row_indices(self, s: int, row: int, host=None):
        """Token indices row `row` of selection row `s` attends to, decoded
        from the plan (for tests and inspection; pass ``host_plans()`` to
        avoid a device copy per call)."""
        import bisect

        import numpy as np

        plans, nplan = host if host is not None else self.host_plans()
        b = self.unit_bounds(s)
        l = bisect.bisect_right(b, row) - 1
        n = int(nplan[s, l])
        ent = plans[s, l, :n]
        R = min(self.budget, row + 1) - 1
        d = row - b[l]
        out = [row]
        for start, ln, w, fl in ent:
            if fl & 2:
                lim = max(0, min(R - w, row - start, ln))
            else:
                lim = max(0, min(R - w - (d if fl & 1 else 0), ln))
            out.extend(range(start, start + lim))
        return np.sort(np.array(out, dtype=np.int64))

    def cost_counters(self, counters=None):
        """The reference's cost accounting (masks.CostCounters) of one call,
        computed analytically: every q head scores its unit's N_c x N_c
        chunk pairs (prefill_mask, masks.py:147-148; the head-aggregated
        harness path counts one matrix per head, harness.py:300-301), and
        each selection row's mask admits sum_i min(budget, i + 1) pairs
        (mask_from_chunk_scores, masks.py:138-139).  Adds to ``counters``
        (a fresh CostCounters if None) and returns it."""
        from .masks import CostCounters

        c = CostCounters() if counters is None else counters
        if self.bounds_host is None:
            ncs = [self.nc] * self.U
        else:
            ncs = [len(self.bounds_host[0 if len(self.bounds_host) == 1 else u]) - 1
                   for u in range(self.U)]
        c.add_score_ops(self.G * sum(n * n for n in ncs))
        L, b = self.L, self.budget
        m = min(L, b)
        c.add_attended(self.S * (m * (m + 1) // 2 + (L - m) * b))
        return c

    def flops(self) -> float:
        """Algorithmic flops: 4 * sum_i min(i+1, budget) * D per q head
        (QK^T and PV over the selected keys)."""
        L, b = self.L, self.budget
        m = min(L, b)
        tot = m * (m + 1) // 2 + (L - m) * b
        return 4.0 * tot * self.D * self.Hq * self.B


def mask_quality(q, k, v, prefill: SparsePrefill, stream=None):
    """Per-row quality of a sparse prefill's masks against dense causal
    attention, on the GPU at any length (the reference computes them on the
    full L x L probability matrix, harness.py:265-285):

    * recall[b, h, i]  = fraction of row i's causal softmax mass inside its
      selection (attention_mass_recall averages it over rows);
    * cosine[b, h, i]  = cosine of the sparse and dense outputs of row i
      (output_fidelity averages it).

    The dense reference is the same tcgen05 kernel with a budget covering
    every causal token.  Returns (recall, cosine) float32 [B, Hq, L]."""
    B, Hq, L, D = q.shape
    dense = SparsePrefill(B, Hq, prefill.Hkv, D, L, budget=L + 1, agg=prefill.agg, device=q.device)
    kw = dict(dtype=torch.float32, device=q.device)
    st_s = torch.empty(B, Hq, L, 2, **kw)
    st_d = torch.empty(B, Hq, L, 2, **kw)
    o_s = prefill(q, k, v, stream=stream, row_stats=st_s)
    o_d = dense(q, k, v, stream=stream, row_stats=st_d)
    recall = torch.empty(B, Hq, L, **kw)
    cosine = torch.empty(B, Hq, L, **kw)
    _lib.call("dhsa_row_quality", _lib.ptr(st_s), _lib.ptr(st_d), _lib.ptr(o_s), _lib.ptr(o_d),
              B * Hq * L, D, _lib.ptr(recall), _lib.ptr(cosine), _lib.stream_handle(stream))
    return recall, cosine
