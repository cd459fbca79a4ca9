// K5 (bf16), persistent variant — dynamically balanced, deterministic
// block-sparse decode attention.
//
// Reference: the row body of dense_attention (core.py:113-118) restricted to
// the selected token ranges.  Same tile math as attn_mma.cu (attn_tile.cuh);
// what changes is the work decomposition.  Every item's tile list is cut
// into fixed SEGMENTS of seg_tiles tiles (the last virtual segment of an item
// also takes any tiles beyond tiles_hint, so the result never depends on the
// hint).  A grid of resident CTAs (occupancy x SMs) pulls segments from a
// device counter in item order; each CTA's TMA producer keeps one ring full
// across everything it pulls, every ring entry carrying its metadata (tile /
// end of segment / exit), so the consumers never stall at segment borders
// and SMs that stream faster simply pull more (per-SM HBM service differs by
// tens of percent on the two-die part; a static split left a 40 us tail).  A
// segment ends in an (m, l, acc) record in its fixed slot; the segment that
// completes the item's tile count merges the slots in order — the result is
// bitwise independent of which CTA ran what.
#include "attn_common.cuh"
#include "attn_tile.cuh"
#include "capi.cuh"

#include <cstdlib>

namespace dhsa {

constexpr int kStreamMaxSeg = 32;  // record slots per item (bounds the workspace)
constexpr int kSegTiles = 12;      // tiles per segment (at least)
constexpr int kSegSmall = 6;       // ... in the tail of the step (swept 2..16: 6 best at C2, C3, p2, p8)

struct StreamArgs {
  const __nv_bfloat16* q;
  int64_t cache_rows;
  int items, items_per_unit, GH;
  const int32_t* tiles;
  int64_t tile_cap;
  const int32_t* ntiles;
  // Segments: the first head_items items use seg_big tiles per segment, the
  // last ones seg_small, so the final pulls of the step are short and the
  // per-CTA speed spread leaves a short tail.  nseg_* = ceil(tiles_hint / seg_*)
  // <= kStreamMaxSeg virtual segments per item.
  int seg_big, nseg_big, seg_small, nseg_small, head_items;
  int prefetch;       // fetch the next pull while the current one streams
  __nv_bfloat16* out;
  float* rec_out;     // unnormalised records instead of out (split-KV shards)
  float* ws;          // [items][kStreamMaxSeg][GH][D+2]
  int32_t* counters;  // [2 + 2 items]: pull counter, exits, per-item segment records
                      // written, per-item merges done; zero at rest
  int32_t* ready;     // [items] or null (re-armed by the next step's first kernel)
  float scale_log2;
  int spin_ns;              // back-off of the ready-flag wait
  int l2_hint;              // evict-first L2 policy on the K/V stream
  int merge_early;          // merges start per item (segment counters), not at grid end
  unsigned long long* dbg;  // DHSA_DEBUG_TIMING (common.cuh)
};

enum : int { kTile = 0, kEnd = 1, kExit = 2 };
struct RingMeta {
  int type, item;
  int a;  // kTile: valid tokens; kEnd: segment index
  int b;  // kTile: 1 on the first tile of a segment; kEnd: tiles in the segment
  int nt; // kEnd: the item's tile count
};


// tiles [lo, hi) of virtual segment j of an item with nt real tiles
__device__ __forceinline__ void seg_shape(const StreamArgs& a, int item, int& S, int& nseg) {
  const bool head = item < a.head_items;
  S = head ? a.seg_big : a.seg_small;
  nseg = head ? a.nseg_big : a.nseg_small;
}
__device__ __forceinline__ void seg_range(int j, int S, int nseg, int nt, int& lo, int& hi) {
  lo = min(j * S, nt);
  hi = (j == nseg - 1) ? nt : min((j + 1) * S, nt);
}

template <int D>
__device__ __forceinline__ void store_row(const StreamArgs& a, int item, int h, int d, float m,
                                          float l, float acc, float* rec) {
  if (rec) {
    if (d == 0) {
      rec[0] = m;
      rec[1] = l;
    }
    rec[2 + d] = acc;
  } else {
    a.out[((int64_t)item * a.GH + h) * D + d] = __float2bfloat16_rn(acc / l);
  }
}

#ifndef ATTN_MIN_CTAS
#define ATTN_MIN_CTAS 2  // register cap: 2 -> ~160 per thread, 3 -> 96 (+ spills)
#endif
template <int D, int STAGES>
__global__ __launch_bounds__(192, ATTN_MIN_CTAS) void attn_stream_kernel(const __grid_constant__ CUtensorMap tmK,
                                                          const __grid_constant__ CUtensorMap tmV,
                                                          StreamArgs a) {
  using T = DecodeTile<D>;
  constexpr int NB = T::NB, BOX = T::BOX, STAGE_BYTES = T::STAGE_BYTES;
  constexpr int REC = D + 2;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* red = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);  // [4][GH][D+2]
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ RingMeta meta[STAGES];
  __shared__ RingMeta epi_meta;                   // consumers -> epilogue warp
  __shared__ __align__(8) uint64_t epi_full, epi_empty;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  int32_t* pull = a.counters;
  int32_t* exits = pull + 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 4 * 32);
    }
    // every lane that read (wrote) a shared buffer arrives itself: the
    // hand-offs do not rest on __syncwarp cumulativity (racecheck-clean)
    mbar_init(&epi_full, 4 * 32);
    mbar_init(&epi_empty, 32);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_trigger();  // the merge grid may launch now; it waits for this grid's completion
  if (a.dbg && threadIdx.x == 0) a.dbg[kDbgAttn + 4 * c] = gtimer();

  if (warp == 4) {
    // ---------------- TMA producer warp: pulls segments, fills the ring ----------------
    // The whole warp walks the pulls; the tile entries of a segment are
    // fetched by all lanes at once (one L2 round trip per 32 tiles instead of
    // one per tile), lane 0 issues the barriers and TMA loads.
    if (lane == 0) {
      prefetch_tmap(&tmK);
      prefetch_tmap(&tmV);
    }
    // K/V tiles are read once per step: evict-first (unless DHSA_L2_HINT=0)
    uint64_t pol = 0;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    if (a.l2_hint) pol = l2_policy_evict_first();
    const int head_pulls = a.head_items * a.nseg_big;
    const int total = head_pulls + (a.items - a.head_items) * a.nseg_small;
    int it = 0;
    auto slot = [&]() {
      const int st = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty_bar[st], ((it / STAGES) + 1) & 1);
      return st;
    };
    int knext = 0;
    if (lane == 0) knext = atomicAdd(pull, 1);
    for (;;) {
      const int k = __shfl_sync(0xffffffffu, knext, 0);
      if (k >= total) break;
      // the next pull is fetched while this one streams (a.prefetch), or
      // only once this one has been queued
      if (lane == 0 && a.prefetch) knext = atomicAdd(pull, 1);
      int item, j;
      if (k < head_pulls) {
        item = k / a.nseg_big;
        j = k - item * a.nseg_big;
      } else {
        item = a.head_items + (k - head_pulls) / a.nseg_small;
        j = k - head_pulls - (item - a.head_items) * a.nseg_small;
      }
      int S, nseg;
      seg_shape(a, item, S, nseg);
      // a segment (not the last) inside the item's early-published prefix
      // starts without the final tile count (nt = -1: never "whole")
      int nt = 0;
      if (lane == 0) {
        if (a.ready) {
          int v;
          while ((v = ld_acquire(a.ready + item)) < 1) __nanosleep(a.spin_ns);
          if (v < kReadyFinal && !(j < nseg - 1 && (j + 1) * S <= v - 1)) {
            spin_geq(a.ready + item, kReadyFinal);
            v = kReadyFinal;
          }
          nt = v < kReadyFinal ? -1 : __ldcg(a.ntiles + item);
        } else {
          nt = __ldcg(a.ntiles + item);
        }
      }
      nt = __shfl_sync(0xffffffffu, nt, 0);
      int lo, hi;
      if (nt < 0) {
        lo = j * S;
        hi = lo + S;
      } else {
        seg_range(j, S, nseg, nt, lo, hi);
      }
      if (lo >= hi && !(nt == 0 && j == 0)) {  // beyond the item's real tiles
        if (lane == 0 && !a.prefetch) knext = atomicAdd(pull, 1);
        continue;
      }
      const int32_t* tl = a.tiles + (int64_t)item * a.tile_cap * 2;
      const int64_t row0 = (int64_t)(item / a.items_per_unit) * a.cache_rows;
      for (int t0 = lo; t0 < hi; t0 += 32) {
        int2 ent = make_int2(0, 0);
        if (t0 + lane < hi) ent = __ldcg(reinterpret_cast<const int2*>(tl) + t0 + lane);
        const int n = min(32, hi - t0);
        for (int i = 0; i < n; ++i) {
          const int start = __shfl_sync(0xffffffffu, ent.x, i);
          const int count = __shfl_sync(0xffffffffu, ent.y, i);
          if (lane == 0) {
            const int st = slot();
            meta[st] = RingMeta{kTile, item, count, t0 + i == lo ? 1 : 0, nt};
            unsigned char* dst = smem + st * STAGE_BYTES;
            const int row = (int)(row0 + start);
            mbar_expect_tx(&full_bar[st], STAGE_BYTES);
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              tma_load_2d_hint(dst + b * BOX, &tmK, &full_bar[st], b * 64, row, pol);
              tma_load_2d_hint(dst + (NB + b) * BOX, &tmV, &full_bar[st], b * 64, row, pol);
            }
          }
          ++it;
        }
      }
      if (lane == 0) {
        const int st = slot();
        meta[st] = RingMeta{kEnd, item, j, hi - lo, nt};
        mbar_arrive(&full_bar[st]);
        if (!a.prefetch) knext = atomicAdd(pull, 1);
      }
      ++it;
    }
    if (lane == 0) {
      const int st = slot();
      meta[st] = RingMeta{kExit, -1, 0, 0, 0};
      mbar_arrive(&full_bar[st]);
    }
    return;
  }

  if (warp == 5) {
    // ---------------- epilogue warp: segment records, item merges ----------------
    const int GH = a.GH;
    for (int k = 0;; ++k) {
      mbar_wait(&epi_full, k & 1);
      const RingMeta e = epi_meta;
      if (e.type == kExit) break;
      const int item = e.item, j = e.a, nt = e.nt;
      const bool whole = e.b == nt;  // one segment holds every tile of the item
      float* slots = a.ws + (int64_t)item * kStreamMaxSeg * GH * REC;
      for (int hd = lane; hd < GH * D; hd += 32) {
        const int h = hd / D, d = hd - h * D;
        float mstar, lsum, acc;
        combine4<D>(red, GH, h, d, mstar, lsum, acc);
        float* rec = whole ? (a.rec_out ? a.rec_out + ((int64_t)item * GH + h) * REC : nullptr)
                           : slots + (j * GH + h) * REC;
        store_row<D>(a, item, h, d, mstar, lsum, acc, rec);
      }
      if (!whole && a.merge_early) {
        // the segment's record is complete: count it for the item's merge,
        // which starts as soon as all of its records exist (not when the grid
        // ends); every lane's stores are fenced before lane 0's count
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(a.counters + 2 + item, 1);
      }
      mbar_arrive(&epi_empty);  // red[] may be overwritten now
    }
    if (a.dbg && lane == 0) a.dbg[kDbgAttn + 4 * c + 2] = gtimer();
    if (lane == 0) {  // the last CTA out re-arms the pull counter
      __threadfence();
      if (atomicAdd(exits, 1) == (int)gridDim.x - 1) {
        *pull = 0;
        *exits = 0;
      }
    }
    return;
  }

  // ---------------- consumers (4 warps) ----------------
  const int GH = a.GH;
  uint32_t qa[T::KS][2];
  float m = -INFINITY, l = 0.f;
  float o[T::NT][4];
  bool first = true;
  int ntile_done = 0, nend = 0;
  for (int it = 0;; ++it) {
    const int st = it % STAGES;
    mbar_wait(&full_bar[st], (it / STAGES) & 1);
    const RingMeta e = meta[st];
    if (e.type == kTile) {
      if (e.b) {  // first tile of a segment
        T::load_q(a.q, e.item, GH, lane, qa);
        m = -INFINITY;
        l = 0.f;
#pragma unroll
        for (int j = 0; j < T::NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
      }
      if (a.dbg && first && threadIdx.x == 0) a.dbg[kDbgAttn + 4 * c + 1] = gtimer();
      first = false;
      T::update(smem_u32(smem + st * STAGE_BYTES), e.a, warp, lane, qa, a.scale_log2, m, l, o);
      mbar_arrive(&empty_bar[st]);
      ++ntile_done;
      continue;
    }
    mbar_arrive(&empty_bar[st]);
    // hand the segment (or the exit) to the epilogue warp once red[] is free
    if (nend > 0) mbar_wait(&epi_empty, (nend - 1) & 1);
    if (e.type == kEnd) {
      if (e.b == 0) {  // an item without tiles (an empty split-KV shard): m = -inf record
        m = -INFINITY;
        l = 0.f;
#pragma unroll
        for (int jj = 0; jj < T::NT; ++jj) o[jj][0] = o[jj][1] = o[jj][2] = o[jj][3] = 0.f;
      }
      l += __shfl_xor_sync(0xffffffffu, l, 1);
      l += __shfl_xor_sync(0xffffffffu, l, 2);
      T::warp_record(red, warp, lane, GH, m, l, o);
    }
    if (threadIdx.x == 0) epi_meta = e;
    mbar_arrive(&epi_full);
    ++nend;
    if (e.type == kExit) break;
  }
  if (a.dbg && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    a.dbg[kDbgAttn + 4 * c + 3] = ((unsigned long long)smid << 32) | (unsigned)ntile_done;
  }
}

// Items processed by more than one segment: merge the slot records in slot
// order (deterministic).  One CTA per (item, head), one thread per dimension;
// launched programmatically with the attention grid: a CTA starts merging as
// soon as its item's segment records are all written (per-item counter,
// acquire), and waits for the attention grid's completion (griddepcontrol.
// wait) only at its end, so the merge overlaps the attention's tail and the
// stream order of the following kernels is unchanged.
template <int D>
__global__ __launch_bounds__(D) void stream_merge_kernel(StreamArgs a) {
  constexpr int REC = D + 2;
  const int item = blockIdx.x, h = blockIdx.y, d = threadIdx.x, GH = a.GH;
  // read the item's tile count (and decide whether it needs a merge at all)
  // before waiting for the attention grid: it is final once the item's ready
  // flag is up (without flags the select grid completed before the attention
  // grid was launched)
  if (a.ready) {
    if (threadIdx.x == 0) spin_geq(a.ready + item, kReadyFinal);
    __syncthreads();
  }
  const int nt = __ldcg(a.ntiles + item);
  int lo, hi;
  int S, nseg;
  seg_shape(a, item, S, nseg);
  seg_range(0, S, nseg, nt, lo, hi);
  if (hi - lo == nt) {  // one segment: written directly by the attention
    pdl_wait();
    return;
  }
  int nrec = 0;  // segments holding tiles = records the attention writes
  for (int sg = 0; sg < nseg; ++sg) {
    seg_range(sg, S, nseg, nt, lo, hi);
    nrec += lo < hi ? 1 : 0;
  }
  int32_t* seg_done = a.counters + 2 + item;
  int32_t* merged = a.counters + 2 + a.items + item;
  if (a.merge_early) {
    if (threadIdx.x == 0) spin_geq(seg_done, nrec);
    __syncthreads();
  } else {
    pdl_wait();
  }
  if (a.dbg && threadIdx.x == 0) atomicMin(a.dbg + kDbgAttn + 8192, gtimer());
  const float* slots = a.ws + (int64_t)item * kStreamMaxSeg * GH * REC + h * REC;
  float mv[kStreamMaxSeg], lv[kStreamMaxSeg], av[kStreamMaxSeg];
#pragma unroll
  for (int sg = 0; sg < kStreamMaxSeg; ++sg) {  // independent loads, issued together
    mv[sg] = -INFINITY;
    lv[sg] = av[sg] = 0.f;
    if (sg < nseg) {
      seg_range(sg, S, nseg, nt, lo, hi);
      if (lo < hi) {
        const float* r = slots + sg * GH * REC;
        mv[sg] = __ldcg(r);
        lv[sg] = __ldcg(r + 1);
        av[sg] = __ldcg(r + 2 + d);
      }
    }
  }
  float mstar = -INFINITY;
#pragma unroll
  for (int sg = 0; sg < kStreamMaxSeg; ++sg) mstar = fmaxf(mstar, mv[sg]);
  float lsum = 0.f, acc = 0.f;
#pragma unroll
  for (int sg = 0; sg < kStreamMaxSeg; ++sg) {
    if (mv[sg] == -INFINITY) continue;
    const float w = exp2f(mv[sg] - mstar);
    lsum += w * lv[sg];
    acc += w * av[sg];
  }
  store_row<D>(a, item, h, d, mstar, lsum, acc,
               a.rec_out ? a.rec_out + ((int64_t)item * GH + h) * REC : nullptr);
  if (a.dbg && threadIdx.x == 0) atomicMax(a.dbg + kDbgAttn + 8193, gtimer());
  // the last of the item's GH merge CTAs re-arms its counters (every CTA has
  // passed its wait on seg_done by then)
  if (a.merge_early) {
    if (threadIdx.x == 0 && atomicAdd(merged, 1) == GH - 1) {
      *seg_done = 0;
      *merged = 0;
    }
    pdl_wait();
  }
}

template <int D, int STAGES>
static int launch_stream(const CUtensorMap& mk, const CUtensorMap& mv, StreamArgs a,
                         cudaStream_t s) {
  using T = DecodeTile<D>;
  const size_t smem = (size_t)STAGES * T::STAGE_BYTES + 4 * a.GH * (D + 2) * 4 + 1024;
  auto kern = attn_stream_kernel<D, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    set_error("dhsa_attn_stream: %s", cudaGetErrorString(e));
    return DHSA_ECUDA;
  }
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 192, smem);
  int64_t C = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
  // the last ~2 pulls per CTA use small segments
  a.head_items = a.items;
  if (a.nseg_small > a.nseg_big) {
    int tp = 2;  // tail pulls per CTA
    if (const char* e = getenv("DHSA_TAIL_PULLS")) tp = atoi(e) >= 0 ? atoi(e) : tp;
    const int64_t tail = (tp * C + a.nseg_small - 1) / a.nseg_small;
    a.head_items = (int)(a.items > tail ? a.items - tail : 0);
  }
  const int64_t pulls = (int64_t)a.head_items * a.nseg_big +
                        (int64_t)(a.items - a.head_items) * a.nseg_small;
  if (C > pulls) C = pulls;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)C);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.ready ? 1 : 0;
  if (const char* e = getenv("DHSA_NO_ATTN_PDL"))
    if (atoi(e)) cfg.numAttrs = 0;
  e = cudaLaunchKernelEx(&cfg, kern, mk, mv, a);
  if (e != cudaSuccess) {
    set_error("dhsa_attn_stream: %s", cudaGetErrorString(e));
    return DHSA_ECUDA;
  }
  if (a.nseg_big > 1 || (a.head_items < a.items && a.nseg_small > 1)) {
    // cross-segment merge, launched early (programmatic dependency)
    cudaLaunchConfig_t mc{};
    mc.gridDim = dim3((unsigned)a.items, (unsigned)a.GH);
    mc.blockDim = dim3(D);
    mc.stream = s;
    cudaLaunchAttribute ma[1];
    ma[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    ma[0].val.programmaticStreamSerializationAllowed = 1;
    mc.attrs = ma;
    mc.numAttrs = 1;
    e = cudaLaunchKernelEx(&mc, stream_merge_kernel<D>, a);
    if (e != cudaSuccess) {
      set_error("dhsa_attn_stream(merge): %s", cudaGetErrorString(e));
      return DHSA_ECUDA;
    }
  }
  return check_launch("dhsa_attn_stream");
}

}  // namespace dhsa

using namespace dhsa;

extern "C" int64_t dhsa_attn_stream_workspace_size(int items, int GH, int D) {
  return (int64_t)items * kStreamMaxSeg * GH * (D + 2) * 4;
}

extern "C" int dhsa_attn_stream_counters(int items) { return 2 * items + 2; }

extern "C" int dhsa_attn_stream(const void* q, const void* k_cache, const void* v_cache,
                                int64_t cache_unit_stride, int64_t cache_rows, int items,
                                int items_per_unit, int GH, int D, const int32_t* tiles,
                                int64_t tile_cap, const int32_t* ntiles, int tiles_hint,
                                void* out, float* records, void* workspace, int32_t* counters,
                                int32_t* ready, dhsa_stream_t stream) {
  DHSA_REQUIRE(q && k_cache && v_cache && tiles && ntiles && workspace && counters &&
                   (out || records),
               "dhsa_attn_stream: null pointer");
  DHSA_REQUIRE(D == 64 || D == 128, "dhsa_attn_stream: D must be 64 or 128, got %d", D);
  DHSA_REQUIRE(items >= 1 && items_per_unit >= 1 && GH >= 1 && GH <= 8 && tile_cap >= 1 &&
                   tiles_hint >= 1,
               "dhsa_attn_stream: bad shape (GH <= 8)");
  DHSA_REQUIRE(cache_unit_stride == cache_rows * D,
               "dhsa_attn_stream: cache units must be dense [rows][D]");
  DHSA_REQUIRE(((uintptr_t)k_cache & 15) == 0 && ((uintptr_t)v_cache & 15) == 0 &&
                   ((uintptr_t)q & 3) == 0,
               "dhsa_attn_stream: misaligned pointers");
  const int units = (items + items_per_unit - 1) / items_per_unit;
  const int64_t rows = (int64_t)units * cache_rows;
  DHSA_REQUIRE(rows < (1ll << 31), "dhsa_attn_stream: cache too large for 32-bit TMA rows");
  CUtensorMap mk, mv;
  int rc = make_tmap_2d(&mk, k_cache, rows, D, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  if (rc) return rc;
  rc = make_tmap_2d(&mv, v_cache, rows, D, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  if (rc) return rc;
  StreamArgs a{};
  a.q = (const __nv_bfloat16*)q;
  a.cache_rows = cache_rows;
  a.items = items;
  a.items_per_unit = items_per_unit;
  a.GH = GH;
  a.tiles = tiles;
  a.tile_cap = tile_cap;
  a.ntiles = ntiles;
  int seg = kSegTiles;
  if (const char* e = getenv("DHSA_SEG_TILES")) seg = atoi(e) > 0 ? atoi(e) : seg;
  a.prefetch = 0;  // measured: prefetching the next pull lengthens the tail
  if (const char* e = getenv("DHSA_STREAM_PREFETCH")) a.prefetch = atoi(e);
  a.seg_big = max(seg, (tiles_hint + kStreamMaxSeg - 1) / kStreamMaxSeg);
  a.nseg_big = (tiles_hint + a.seg_big - 1) / a.seg_big;
  int seg_small = kSegSmall;
  if (const char* e = getenv("DHSA_SEG_SMALL")) seg_small = atoi(e) > 0 ? atoi(e) : seg_small;
  a.seg_small = max(seg_small, (tiles_hint + kStreamMaxSeg - 1) / kStreamMaxSeg);
  a.nseg_small = (tiles_hint + a.seg_small - 1) / a.seg_small;
  a.out = (__nv_bfloat16*)out;
  a.rec_out = records;
  a.ws = (float*)workspace;
  a.counters = counters;
  a.ready = ready;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)D));
  if (const char* e = getenv("DHSA_DEBUG_TIMING")) a.dbg = (unsigned long long*)strtoull(e, nullptr, 0);
  a.spin_ns = 64;
  a.l2_hint = 1;
  if (const char* e = getenv("DHSA_L2_HINT")) a.l2_hint = atoi(e);
  if (const char* e = getenv("DHSA_SPIN_NS")) a.spin_ns = atoi(e);
  a.merge_early = 0;
  if (const char* e = getenv("DHSA_MERGE_EARLY")) a.merge_early = atoi(e);
  cudaStream_t s = (cudaStream_t)stream;
  int stages = 3;
  if (const char* e = getenv("DHSA_STREAM_STAGES")) stages = atoi(e);
  if (D == 128) {
    if (stages >= 6) return launch_stream<128, 6>(mk, mv, a, s);
    if (stages == 4) return launch_stream<128, 4>(mk, mv, a, s);
    return launch_stream<128, 3>(mk, mv, a, s);
  }
  return launch_stream<64, 6>(mk, mv, a, s);
}
