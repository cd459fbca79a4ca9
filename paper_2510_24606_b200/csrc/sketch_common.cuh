// Shared pieces of the bf16 sketch decode path (decode_sketch.cu: sketch
// stream, generic select; select2.cuh: the register-resident select).
#pragma once

#include "capi.cuh"
#include "walk.cuh"

#include <cuda_fp16.h>

#ifndef SELECT_THREADS
#define SELECT_THREADS 256
#endif

namespace dhsa {

constexpr int kSelectThreads = SELECT_THREADS;
constexpr int kSmallUncertain = 1024;
constexpr int kHistBins = 1024;  // value-histogram bins of the certified select


constexpr int kTcConsumers = 4;
constexpr int kTcThreads = (kTcConsumers + 1) * 32;
// sketch stream ring: 2 stages x 3 CTAs per SM (measured against 2..6
// stages x 1..5 CTAs: C3 122.5 vs 123.8 us with 4 x 3, p8 36.6 vs 37.2, p4
// 48.0 vs 49.4; fewer bytes in flight per SM leave the selects room)
#ifndef DHSA_SKETCH_STAGES
#define DHSA_SKETCH_STAGES 2
#endif
constexpr int kTcStages = DHSA_SKETCH_STAGES;
constexpr int kSliceRows = 64;

struct SketchArgs {
  const __nv_bfloat16* q;   // [U*G][D]
  const __half* sketch;     // [U][sk_stride]
  int64_t sk_stride;
  const float* sinfo;       // [U][4]: scale exponent k (as float), cmax, dmax, unused
  const double* cent;       // [U][c_stride] fp64 centroids (refinement)
  int64_t c_stride;
  double* gen_sum;          // [U][D]
  int32_t* gen_count;       // [U]
  const __nv_bfloat16* k_new;
  const __nv_bfloat16* v_new;
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
  int64_t cache_stride;
  Layout lay;
  float* approx;            // [items][sc_stride] scaled approximate scores
  int64_t sc_stride;
  int slices_per_unit;      // ceil(max_chunks / chunks_per_slice)
  int64_t total_slices;
  int64_t budget;
  int tile_tokens;
  int32_t* tiles;
  int64_t tile_cap;
  int32_t* ntiles;
  unsigned char* gscratch;
  int64_t gscratch_stride;
  int smem_select;
  int n_max;
  int advance;
  int32_t* ready;           // [items] select -> attention flags (zeroed by the sketch kernel) or null
  int n_units;
  int32_t* progress;        // [U] sketch -> select: consumer-warp slices done (zero at rest) or null
  int early;                // publish the certainly-kept chunks' tiles before the refinement
  int l2_hint;              // evict-first L2 policy on the sketch stream
  int reps;                 // (experiment, DHSA_SELECT_REPS) repeated selections
  int relaxed;              // (experiment, DHSA_RELAXED_FLAGS) flag stores without release
  int waves;                // sketch stream: the unit range in consecutive waves
  int wave_end[4];          // cumulative wave ends in permille of the slices (waves <= 4)
  unsigned long long* dbg;  // optional per-CTA phase timestamps (DHSA_DEBUG_TIMING)
  // sequence-sharded split-KV mode (dhsa_decode_candidates_bf16): this shard
  // holds global prompt chunks [chunk_offset, chunk_offset + nchunks); the
  // tail shard also holds the generated chunk (global id total_chunks) and
  // the newest token.  Instead of tiles, every chunk the local exact walk
  // gives a positive take is written as a candidate record.
  int split;
  int32_t chunk_offset, total_chunks, total_prompt, owns_tail;
  unsigned char* cand;      // [items][cand_stride] bytes: header + SplitCand[cand_cap]
  int64_t cand_stride;
  int cand_cap;
};

// phase stamps of the select CTAs: clock64 at every point (cheap), the
// (slow, ~0.5-1 us) %globaltimer only at the start (0) and the end (8)
// (compiled only with -DDHSA_SELECT_STAMPS: the stamps' code sits between the
// hot phases of the latency-bound select and costs instruction-cache lines)
#ifdef DHSA_SELECT_STAMPS
#define DBG_T(k)                                                           \
  if (a.dbg && threadIdx.x == 0) {                                         \
    if ((k) == 0 || (k) == 8) a.dbg[blockIdx.x * 16 + (k)] = gtimer();     \
    a.dbg[kDbgSelectClk + blockIdx.x * 16 + (k)] = clock64();              \
  }
#else
#define DBG_T(k)
#endif


// --------------------------------------------------------------- selection --
struct UnitChunks {
  Layout lay;
  int u, nc, g, P;
  __device__ void chunk(int c, int& lo, int& len) const {
    if (c < nc) {
      if (lay.bounds) {
        int hi;
        lay.chunk(u, c, lo, hi);
        len = hi - lo;
      } else {  // static grid: arithmetic only (P is cached in the struct)
        lo = c * lay.block;
        len = min(lay.block, P - lo);
      }
    } else {
      lo = P;
      len = g;
    }
  }
};

template <int G, int AGG>
__device__ __forceinline__ double agg_d(const double* v, int nh) {
  double s = v[0];
  for (int h = 1; h < nh; ++h) s = (AGG == DHSA_AGG_MAX) ? fmax(s, v[h]) : s + v[h];
  if (AGG == DHSA_AGG_MEAN && nh > 1) s = s / (double)nh;
  return s;
}

// Split-KV: every chunk with a positive local take (takes in lens[]) becomes a
// candidate record with its exact fp64 score (the same arithmetic as the
// re-scoring above), global chunk id, full length and local start token.
// The global walk (splitkv.cu) over the candidates of all shards then equals
// the unsharded walk: a chunk with a positive global take has fewer than R
// tokens ranked above it globally, hence locally, so it is a local candidate.

// Select prologue (before the unit's approximate scores exist): the query in
// fp64 shared memory, the query norms of the certified bound, the generated
// chunk's exact fp64 score (masks.py:161) and the state update (running sum,
// k/v append, masks.py:235), then the wait for the unit's sketch slices.
// Ends with a CTA barrier.  g = generated count, gl = generated tokens this
// shard holds.
template <int D, int G, int NT>
__device__ __forceinline__ void select_prologue(const SketchArgs& a, int u, double (*qd)[D],
                                                double* s_qn, double* s_gen, int& g, int& gl) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- prologue: every global load of the step issued before one barrier ----
  for (int i = tid; i < G * D; i += NT)
    qd[i / D][i % D] = to_f64(a.q[(int64_t)u * G * D + i]);
  g = a.gen_count[u];
  gl = (a.split && !a.owns_tail) ? 0 : g;  // generated tokens held by this shard
  constexpr int DV = D / 32;
  static_assert(NW >= 2, "select needs >= 2 warps");
  if (warp < NW - 1) {  // query norms (certified bound), warps 0 .. NW-2
    for (int h = warp; h < G; h += NW - 1) {
      double t = 0.0;
#pragma unroll
      for (int v = 0; v < DV; ++v) {
        const double x = to_f64(a.q[(int64_t)(u * G + h) * D + lane + 32 * v]);
        t = fma(x, x, t);
      }
      t = warp_sum(t);
      if (lane == 0) s_qn[h] = sqrt(t) * (1.0 + 1e-12);
    }
  } else {
    // generated chunk, exact fp64 (masks.py:161), then the state update
    double* gs = a.gen_sum + (int64_t)u * D;
    double gv[DV], qv[G][DV];
    __nv_bfloat16 kv[DV], vv[DV];
#pragma unroll
    for (int v = 0; v < DV; ++v) {
      const int d = lane + 32 * v;
      gv[v] = gs[d];
      if (a.k_new) kv[v] = a.k_new[(int64_t)u * D + d];
      if (a.v_new) vv[v] = a.v_new[(int64_t)u * D + d];
#pragma unroll
      for (int h = 0; h < G; ++h) qv[h][v] = to_f64(a.q[(int64_t)(u * G + h) * D + d]);
    }
    double part[G];
#pragma unroll
    for (int h = 0; h < G; ++h) part[h] = 0.0;
    if (gl >= 1) {
      const double rs = __dsqrt_rn((double)gl);
#pragma unroll
      for (int v = 0; v < DV; ++v) {
        const double cg = __ddiv_rn(gv[v], rs);
#pragma unroll
        for (int h = 0; h < G; ++h) part[h] = fma(qv[h][v], cg, part[h]);
      }
#pragma unroll
      for (int h = 0; h < G; ++h) part[h] = warp_sum(part[h]);
    }
    if (lane == 0)
#pragma unroll
      for (int h = 0; h < G; ++h) s_gen[h] = part[h];
    if (a.k_new) {  // masks.py:235: after the read above; k/v appended at row P+g
      const int64_t pos = (int64_t)(a.lay.prompt_len(u) + gl) * D;
#pragma unroll
      for (int v = 0; v < DV; ++v) {
        const int d = lane + 32 * v;
        gs[d] = __dadd_rn(gv[v], to_f64(kv[v]));
        if (a.kc) a.kc[(int64_t)u * a.cache_stride + pos + d] = kv[v];
        if (a.vc) a.vc[(int64_t)u * a.cache_stride + pos + d] = vv[v];
      }
    }
  }
  // the unit's approximate scores are complete once every consumer warp of
  // every slice of the unit has published (progress), or - without progress
  // counters - once the whole score grid has finished
  if (a.progress) {
    if (tid == 0) {
      const int slices = (a.lay.num_chunks(u) + kSliceRows - 1) / kSliceRows;
      spin_geq(a.progress + u, kTcConsumers * slices);
      a.progress[u] = 0;  // re-arm: the next step's stream starts after this grid
    }
  } else {
    pdl_wait();
  }
  __syncthreads();
}

template <int D, int G, int AGG, int NT>
__device__ void emit_candidates(const SketchArgs& a, const UnitChunks& uc, const int32_t* takes,
                                int32_t* list, int n, int s, const double (*qd)[D], int h0, int nh,
                                double gex, int u) {
  constexpr int NW = NT / 32;
  __shared__ int s_ncand;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_ncand = 0;
  __syncthreads();
  for (int c = tid; c < n; c += NT)
    if (takes[c] > 0) list[atomicAdd(&s_ncand, 1)] = c;
  __syncthreads();
  const int nc = s_ncand;
  unsigned char* row = a.cand + (int64_t)s * a.cand_stride;
  SplitCand* rec = reinterpret_cast<SplitCand*>(row) + 1;
  // a warp re-scores its candidates CB at a time: the CB fp64 centroid rows'
  // loads are issued together (one memory round trip per batch, not per row)
  constexpr int CB = 4;
  const int ncap = nc < a.cand_cap ? nc : a.cand_cap;
  for (int i0 = warp * CB; i0 < ncap; i0 += NW * CB) {
    double cv[CB][D / 32];
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int i = i0 + b;
      const int c = i < ncap ? list[i] : uc.nc;
      const double* crow = a.cent + (int64_t)u * a.c_stride + (int64_t)(c < uc.nc ? c : 0) * D;
#pragma unroll
      for (int v = 0; v < D / 32; ++v) cv[b][v] = (i < ncap && c < uc.nc) ? crow[lane + 32 * v] : 0.0;
    }
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int i = i0 + b;
      if (i >= ncap) break;
      const int c = list[i];
      int lo, len;
      uc.chunk(c, lo, len);
      double ex;
      if (c < uc.nc) {
        double part[G];
#pragma unroll
        for (int h = 0; h < G; ++h) part[h] = 0.0;
#pragma unroll
        for (int v = 0; v < D / 32; ++v)
#pragma unroll
          for (int h = 0; h < G; ++h) part[h] = fma(qd[h][lane + 32 * v], cv[b][v], part[h]);
#pragma unroll
        for (int h = 0; h < G; ++h) part[h] = warp_sum(part[h]);
        ex = agg_d<G, AGG>(part + h0, nh);
      } else {
        ex = gex;
      }
      if (lane == 0) {
        SplitCand r;
        r.score = ex;
        r.gid = c < uc.nc ? a.chunk_offset + c : a.total_chunks;
        r.len = len;
        r.lo = lo;
        r.pad = 0;
        rec[i] = r;
      }
    }
  }
  if (tid == 0) reinterpret_cast<int32_t*>(row)[0] = nc <= a.cand_cap ? nc : -1;
  __syncthreads();
}

}  // namespace dhsa
