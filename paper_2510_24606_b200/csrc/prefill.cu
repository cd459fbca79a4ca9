// Sparse prefill (config C5): chunk scores, per-query-chunk selection plans and
// block-sparse attention on the tcgen05 tensor cores (TMEM accumulators,
// TMA-staged 128B-swizzled operand tiles).
//
// Reference path: prefill_mask (masks.py:143-150) = build_chunk_reps
// (chunk_repr.py:85-94, centroids of Q and K) -> chunk_similarity
// (chunk_repr.py:97-103, S_c = Q_c K_c^T, no scaling) -> [optional head
// aggregation, harness.py:288-306] -> mask_from_chunk_scores (masks.py:125-140:
// upsample + topk_row per row), then dense_attention(seq, mask)
// (core.py:98-119).  The L x L upsampled matrix is never built:
//
//  K7  prefill_scores_kernel  S[s][l][c] (c <= l) in fp64, aggregated over
//                             the q-heads sharing a selection row;
//  K8  prefill_plan_kernel    one CTA per (selection row s, query chunk l):
//                             every row of chunk l walks the SAME chunk order
//                             (score desc, chunk asc); only the diagonal
//                             chunk's effective length d_i = i - b_l and the
//                             token budget R_i = min(budget, i+1) - 1 differ
//                             per row.  The plan lists, in walk order, every
//                             non-diagonal chunk some row of the chunk takes
//                             tokens from (weighted radix select with the
//                             largest R of the chunk) with W = tokens of
//                             non-diagonal chunks ranked before it and a flag
//                             "diagonal ranks before", plus the diagonal.  Row
//                             i then takes clamp(R_i - W - [diag before]*d_i,
//                             0, len) lowest tokens of each entry (SURVEY.md
//                             Appendix A) and self;
//  K9  prefill_attn_kernel    one CTA per (plan, <= 4 q-heads): a 128- or
//                             256-row query tile (64 rows per head, one M=128
//                             tcgen05 tile per 2 heads), S = Q K^T and O += P V
//                             per selected 64-token KV block with tcgen05.mma
//                             (fp32 accumulators in TMEM), per-row masks from
//                             the plan, online softmax with one thread per
//                             query row (tcgen05.ld 32x32b), P through
//                             swizzled shared memory.
#include "capi.cuh"
#include "tc05.cuh"
#include "walk.cuh"

#include <cstdlib>

namespace dhsa {

// ------------------------------------------------------------------- K7 --
// S[s][l][c] = agg_{j in heads(s)} Qc[q(s,j)][l] . Kc[u(s)][c] for c <= l, fp64
// (dot products accumulated in dimension order, aggregated max / mean).
// 64 x 64 output tiles (lower triangle only), 256 threads x 4 x 4 register
// tile, D streamed through shared memory in slabs of 16; the K tile is
// loaded once per slab for all G heads of the selection row.
constexpr int kScT = 64, kScSlab = 16;

__global__ __launch_bounds__(256) void prefill_scores_kernel(
    const double* __restrict__ qc, const double* __restrict__ kc, int nc, int D, int G,
    int per_head, int agg, double* __restrict__ out) {
  __shared__ double sq[kScSlab][kScT + 1];
  __shared__ double sk[kScSlab][kScT + 1];
  const int s = blockIdx.z;
  const int i0 = blockIdx.y * kScT, j0 = blockIdx.x * kScT;
  if (j0 > i0) return;  // strictly above the diagonal: never read
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 each
  const int u = per_head ? s / G : s;
  const int nh = per_head ? 1 : G;
  const int h0 = per_head ? s : s * G;
  const double* K = kc + (int64_t)u * nc * D;
  double res[4][4];
  for (int j = 0; j < nh; ++j) {
    const double* Q = qc + (int64_t)(h0 + j) * nc * D;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int d0 = 0; d0 < D; d0 += kScSlab) {
      for (int e = threadIdx.x; e < kScT * kScSlab; e += 256) {
        const int r = e / kScSlab, c = e % kScSlab;
        sq[c][r] = (i0 + r < nc && d0 + c < D) ? Q[(int64_t)(i0 + r) * D + d0 + c] : 0.0;
        sk[c][r] = (j0 + r < nc && d0 + c < D) ? K[(int64_t)(j0 + r) * D + d0 + c] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < kScSlab; ++c) {
        double qa[4], kb[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) qa[a] = sq[c][ty + 16 * a];
#pragma unroll
        for (int b = 0; b < 4; ++b) kb[b] = sk[c][tx + 16 * b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(qa[a], kb[b], acc[a][b]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (j == 0) res[a][b] = acc[a][b];
        else if (agg == DHSA_AGG_MAX) res[a][b] = fmax(res[a][b], acc[a][b]);
        else res[a][b] = res[a][b] + acc[a][b];
      }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      double v = res[a][b];
      if (agg == DHSA_AGG_MEAN && nh > 1) v = v / (double)nh;
      const int ri = i0 + ty + 16 * a, cj = j0 + tx + 16 * b;
      if (ri < nc && cj < nc) out[((int64_t)s * nc + ri) * nc + cj] = v;
    }
}

// K7 on the FP64 tensor cores (DMMA m8n8k4): the 64 x D K-centroid tile and
// one head's 64 x D Q tile are staged in shared memory once (rows padded to
// D + 4 doubles: 8 rows x 4 k of a fragment load cover all 32 banks twice),
// each warp owns 8 query rows x 64 key chunks (8 accumulator tiles).
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = smem_u32(dst);
  const int n = valid ? 16 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// 64 x D fp64 tile rows [r0, r0 + 64) of src (row stride D) -> smem rows of P
// doubles, 16-byte cp.async (rows past nc zero-filled)
template <int D, int P>
__device__ __forceinline__ void load_tile_async(double* dst, const double* src, int r0, int nc) {
  for (int e = threadIdx.x; e < 64 * D / 2; e += 256) {
    const int r = e / (D / 2), d2 = e - r * (D / 2);
    const bool ok = r0 + r < nc;
    cp_async16(dst + r * P + 2 * d2, src + (int64_t)(ok ? r0 + r : r0) * D + 2 * d2, ok);
  }
  cp_async_commit();
}

template <int D>
__global__ __launch_bounds__(256) void prefill_scores_dmma_kernel(
    const double* __restrict__ qc, const double* __restrict__ kc, int nc, int G, int per_head,
    int agg, double* __restrict__ out) {
  constexpr int P = D + 4;
  extern __shared__ __align__(16) double sm[];
  double* sk = sm;                          // [64][P]
  double* const sq0 = sm + 64 * P;          // double-buffered head tiles [2][64][P]
  const int s = blockIdx.z;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  if (j0 > i0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = per_head ? s / G : s;
  const int nh = per_head ? 1 : G;
  const int h0 = per_head ? s : s * G;
  load_tile_async<D, P>(sk, kc + (int64_t)u * nc * D, j0, nc);
  load_tile_async<D, P>(sq0, qc + (int64_t)h0 * nc * D, i0, nc);
  double res[8][2];
  const int ar = warp * 8 + (lane >> 2), ak = lane & 3;  // A fragment: row, k
  for (int j = 0; j < nh; ++j) {
    // the next head's tile streams in while this one is multiplied
    if (j + 1 < nh) {
      load_tile_async<D, P>(sq0 + ((j + 1) & 1) * 64 * P, qc + (int64_t)(h0 + j + 1) * nc * D, i0,
                            nc);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* q = sq0 + (j & 1) * 64 * P;
    double acc[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < D; k0 += 4) {
      const double a = q[ar * P + k0 + ak];
#pragma unroll
      for (int t = 0; t < 8; ++t) dmma_8x8x4(acc[t], a, sk[(t * 8 + (lane >> 2)) * P + k0 + ak]);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (j == 0) res[t][e] = acc[t][e];
        else if (agg == DHSA_AGG_MAX) res[t][e] = fmax(res[t][e], acc[t][e]);
        else res[t][e] = res[t][e] + acc[t][e];
      }
    __syncthreads();  // buffer j & 1 is refilled two heads later
  }
  const int ri = i0 + warp * 8 + (lane >> 2);
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double v = res[t][e];
      if (agg == DHSA_AGG_MEAN && nh > 1) v = v / (double)nh;
      const int cj = j0 + t * 8 + 2 * (lane & 3) + e;
      if (ri < nc && cj < nc) out[((int64_t)s * nc + ri) * nc + cj] = v;
    }
}

// ------------------------------------------------------------------- K8 --
constexpr int kPlanThreads = 128;
constexpr int kTok = 64;  // KV block / query tile rows of the tcgen05 kernel

// Chunk layout of the prefill: the static grid (bounds == null) or explicit
// per-unit boundary lists (chunking.check_boundaries form; stride 0 = shared),
// e.g. nms_boundaries over predictor scores.
struct PrefillChunks {
  const int32_t* bounds;   // [U][bstride] or null (static grid)
  int64_t bstride;
  const int32_t* nchunks;  // [U] (explicit mode)
  int block, L;
  __device__ __forceinline__ int count(int u, int nc) const {
    return bounds ? nchunks[u] : nc;
  }
  __device__ __forceinline__ void range(int u, int l, int& b, int& e) const {
    if (bounds) {
      const int32_t* p = bounds + (int64_t)u * bstride;
      b = p[l];
      e = p[l + 1];
    } else {
      b = l * block;
      e = min(b + block, L);
    }
  }
};

// Plan entries are <= 64-token KV blocks {start, len, W, flags}: a chunk of
// which the walk without the diagonal at the largest budget Rmax takes t
// tokens (an upper bound on every row's take) becomes ceil(t / 64)
// consecutive blocks (block k: W + 64 k, so a row's take from the chunk is
// split over its blocks exactly).  The
// non-diagonal chunks' blocks are written at their walk position (blocks of
// the chunks ranked before), the diagonal chunk's blocks last; with the static
// 64 grid every chunk is one block and the entry index is the walk rank.
__global__ __launch_bounds__(kPlanThreads) void prefill_plan_kernel(
    const double* __restrict__ S, int nc, PrefillChunks ch, int G, int per_head, int64_t budget,
    int cap, int4* __restrict__ plans, int32_t* __restrict__ nplan) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ WalkShared sh;
  __shared__ int s_n, s_wd, s_nb;
  uint64_t* key = reinterpret_cast<uint64_t*>(smem_raw);
  int32_t* lens = reinterpret_cast<int32_t*>(key + nc);
  int32_t* clen = lens + nc;  // full chunk lengths (lens holds the takes)
  int32_t* list = clen + nc;
  const int l = blockIdx.x, s = blockIdx.y, tid = threadIdx.x;
  const int u = per_head ? s / G : s;
  if (l >= ch.count(u, nc)) {
    if (tid == 0) nplan[(int64_t)s * nc + l] = 0;
    return;
  }
  const double* srow = S + ((int64_t)s * nc + l) * nc;
  int bl, el;
  ch.range(u, l, bl, el);
  // the largest token budget among the rows of chunk l (its last row)
  const int64_t rmax64 = (budget < (int64_t)el ? budget : (int64_t)el) - 1;
  const uint32_t Rmax = (uint32_t)rmax64;
  for (int c = tid; c < l; c += kPlanThreads) {
    key[c] = order_key(srow[c]);
    int b, e;
    ch.range(u, c, b, e);
    lens[c] = clen[c] = e - b;  // chunks before the diagonal are whole
  }
  const uint64_t kdiag = order_key(srow[l]);
  if (tid == 0) {
    s_n = 0;
    s_wd = 0;
    s_nb = 0;
  }
  __syncthreads();
  // takes of the walk over the non-diagonal chunks with budget Rmax
  if (l > 0) {
    if (Rmax >= (uint32_t)bl) {
      // every earlier chunk is kept whole by the last row
    } else if (Rmax == 0) {
      for (int c = tid; c < l; c += kPlanThreads) lens[c] = 0;
      __syncthreads();
    } else {
      uint64_t prefix, mask;
      uint32_t rrem;
      radix_threshold<kPlanThreads, uint64_t>(key, lens, l, Rmax, sh, prefix, mask, rrem);
      walk_takes<kPlanThreads, uint64_t>(key, lens, l, Rmax, prefix, mask, rrem, sh);
    }
    for (int c = tid; c < l; c += kPlanThreads)
      if (lens[c] > 0) list[atomicAdd(&s_n, 1)] = c;
  }
  __syncthreads();
  const int n = s_n;
  int4* out = plans + ((int64_t)s * nc + l) * cap;
  // walk position: W = whole-chunk tokens ranked before, pos = their blocks
  int wd = 0, nb = 0;
  for (int i = tid; i < n; i += kPlanThreads) {
    const int c = list[i];
    const uint64_t kc = key[c];
    int W = 0, pos = 0;
    for (int j = 0; j < n; ++j) {
      const int cj = list[j];
      const uint64_t kj = key[cj];
      if (kj > kc || (kj == kc && cj < c)) {
        W += clen[cj];
        pos += (lens[cj] + kTok - 1) / kTok;
      }
    }
    int b, e;
    ch.range(u, c, b, e);
    const int diag_before = kdiag > kc ? 1 : 0;  // tie: the lower index (c < l) first
    // only the blocks some row can reach
    const int nbk = (lens[c] + kTok - 1) / kTok;
    for (int k = 0; k < nbk; ++k)
      if (pos + k < cap) out[pos + k] = make_int4(b + k * kTok, min(kTok, clen[c] - k * kTok),
                                                  W + k * kTok, diag_before);
    if (!diag_before) wd += clen[c];
    nb += nbk;
  }
  wd = warp_sum(wd);
  nb = warp_sum(nb);
  if ((tid & 31) == 0) {
    if (wd) atomicAdd(&s_wd, wd);
    if (nb) atomicAdd(&s_nb, nb);
  }
  __syncthreads();
  const int nbt = s_nb, nd = (el - bl + kTok - 1) / kTok;
  if (nbt + nd > cap) {
    if (tid == 0) nplan[(int64_t)s * nc + l] = -1;  // capacity error (reported by the host)
    return;
  }
  for (int k = tid; k < nd; k += kPlanThreads)  // the diagonal chunk (self always)
    out[nbt + k] = make_int4(bl + k * kTok, min(kTok, el - bl - k * kTok), s_wd + k * kTok, 2);
  if (tid == 0) nplan[(int64_t)s * nc + l] = nbt + nd;
}

// Tokens row i takes from plan entry e: the lowest
// clamp(R_i - W - [diag before] d_i, 0, len) of a non-diagonal block, where
// d_i = i - (chunk start) is the diagonal chunk's effective length; of a
// diagonal block the lowest clamp(R_i - W, 0, i - start) (causal), plus self.
__device__ __forceinline__ int entry_take(int4 e, int Ri, int i, int dl, int& self) {
  if (e.w & 2) {
    const int db = i - e.x;
    self = (db >= 0 && db < e.y) ? db : -1;
    return max(0, min(min(Ri - e.z, db), e.y));
  }
  self = -1;
  return max(0, min(Ri - e.z - ((e.w & 1) ? dl : 0), e.y));
}

// ------------------------------------------------------------------- K9 --
constexpr int kPlanCap = 544;  // plan entries per query chunk (dense up to ~34K tokens)

struct PrefillArgs {
  const int4* plans;
  const int32_t* nplan;
  int cap, nc, L, block;
  int64_t budget;
  int G, per_head, heads_per_cta, slices;
  __nv_bfloat16* out;  // [q heads][L][D]
  float scale_log2;
  int S;               // selection rows
  int32_t* counters;   // [2] plan pull counter, exits (persistent kernel); zero at rest
  float2* row_stats;   // [q heads][L] (m, l): the row's softmax reference max (log2
                       // domain) and sum of 2^(x - m) over its selection, or null
  PrefillChunks ch;    // chunk layout (static grid or explicit bounds)
  const int2* qtiles;  // explicit bounds: [U][T] query tiles (chunk l, 64-row tile t),
  int T;               // heavy first, l = -1 pads; null with the static grid (T = nc)
  unsigned long long* dbg;  // DHSA_DEBUG_TIMING: clock64 stamps of one CTA (prefill_timeline.py)
  // query tile y of unit u -> (chunk l, tile t); false for padding
  __device__ __forceinline__ bool tile(int u, int y, int& l, int& t) const {
    if (qtiles) {
      const int2 q = qtiles[(int64_t)u * T + y];
      l = q.x;
      t = q.y;
      return l >= 0;
    }
    l = nc - 1 - y;  // heavy (late) query chunks first
    t = 0;
    return true;
  }
};

template <int MT, int NST>
struct PrefillSmem {
  static constexpr int Q = MT * 2 * 16384;  // [mt][D half][128 rows][128 B]
  static constexpr int KV = 2 * 2 * 8192;    // K [half][64][128B] + V [half][64][128B]
  static constexpr int q_off = 0;
  static constexpr int kv_off = Q;
  static constexpr int total = Q + NST * KV + 1024;  // + alignment slack (P lives in TMEM)
};

__device__ __forceinline__ float exp2_mufu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Blackwell packed fp32 pairs (FFMA2 / FADD2): half the issue slots of the
// scalar forms in the softmax, which is issue-bound.
__device__ __forceinline__ uint64_t f2_u64(float a, float b) {
  return (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(b) << 32);
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float lo_f(uint64_t x) { return __uint_as_float((uint32_t)x); }
__device__ __forceinline__ float hi_f(uint64_t x) { return __uint_as_float((uint32_t)(x >> 32)); }

// max over 64 raw scores: four independent FMNMX3 chains instead of one
__device__ __forceinline__ float row_max64(const uint32_t* v) {
  float m[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int c = 0; c < 64; c += 8)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      m[k] = fmaxf(m[k], fmaxf(__uint_as_float(v[c + 2 * k]), __uint_as_float(v[c + 2 * k + 1])));
  return fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
}

#ifndef DHSA_POLY_PAIRS
#define DHSA_POLY_PAIRS 0  // pairs (of every 8) whose exp2 runs on the FMA pipe;
#endif                      // measured slower at 2..4 (-8..-14% TFLOP/s): not MUFU-bound

// 2^x for a pair on the FMA pipe (the MUFU pipe is shared by both M tiles'
// softmax warps): round-to-nearest split x = n + f, |f| <= 1/2, degree-3
// polynomial (max rel. error 7.8e-5, below bf16's 3.9e-3), n added to the
// exponent field.  x is clamped at -125 (masked -inf columns give ~2^-125,
// negligible against the row max term 1).
__device__ __forceinline__ void exp2_poly2(uint64_t x, float& p0, float& p1) {
  const float x0 = fmaxf(lo_f(x), -125.f), x1 = fmaxf(hi_f(x), -125.f);
  const uint64_t magic = f2_u64(12582912.f, 12582912.f);  // 1.5 * 2^23
  const uint64_t t = fadd2(f2_u64(x0, x1), magic);        // n in the low mantissa bits
  const uint64_t n = fadd2(t, f2_u64(-12582912.f, -12582912.f));
  const uint64_t f = fadd2(f2_u64(x0, x1), n ^ 0x8000000080000000ull);  // x - n
  uint64_t r = ffma2(f, f2_u64(0.05508876591920853f, 0.05508876591920853f),
                     f2_u64(0.24260465800762177f, 0.24260465800762177f));
  r = ffma2(r, f, f2_u64(0.6932762861251831f, 0.6932762861251831f));
  r = ffma2(r, f, f2_u64(0.999928891658783f, 0.999928891658783f));
  p0 = __uint_as_float((uint32_t)r + ((uint32_t)t << 23));
  p1 = __uint_as_float((uint32_t)(r >> 32) + ((uint32_t)(t >> 32) << 23));
}

// p = 2^(s * sl2 - mref) for 64 scores, packed to bf16 pairs in pk; returns
// the sum of the p (two packed accumulators)
__device__ __forceinline__ float softmax_pack64(const uint32_t* v, float sl2, float mref,
                                                uint32_t* pk) {
  const uint64_t sc2 = f2_u64(sl2, sl2), nm2 = f2_u64(-mref, -mref);
  uint64_t acc[2] = {0ull, 0ull};
#pragma unroll
  for (int t = 0; t < 32; ++t) {
    const uint64_t x = ffma2((uint64_t)v[2 * t] | ((uint64_t)v[2 * t + 1] << 32), sc2, nm2);
    float p0, p1;
    if ((t & 7) < DHSA_POLY_PAIRS) {
      exp2_poly2(x, p0, p1);
    } else {
      p0 = exp2_mufu(lo_f(x));
      p1 = exp2_mufu(hi_f(x));
    }
    acc[t & 1] = fadd2(acc[t & 1], f2_u64(p0, p1));
    pk[t] = pack_bf16(p0, p1);
  }
  const uint64_t a = fadd2(acc[0], acc[1]);
  return lo_f(a) + hi_f(a);
}

// D[tmem] (+)= A[tmem] * B[smem] (A = P in TMEM, K-major; "TS" form).
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(0u)
      : "memory");
}

// One CTA = one plan (selection row s, query chunk l) x <= 4 q heads:
// MT M=128 tiles of 2 heads x 64 rows.  TMEM per tile: two S/P buffers of 64
// fp32 columns (P is written back as packed bf16 into the first 32 columns
// of its S buffer and consumed from TMEM by the PV MMA) + O (128 columns).
// Warp 0: TMA producer; warp 1: MMA issuer; warps 2..: one thread per row.
// The softmax of block j never waits for PV_{j-1} (the S/P buffers are
// double-buffered and the tensor pipe executes in issue order) except to
// rescale O, which happens only when a row max grows by > 2^8.
template <int MT, int NST>
__global__ __launch_bounds__(64 + 128 * MT, 1) void prefill_attn_kernel(
    const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
    const __grid_constant__ CUtensorMap tmV, PrefillArgs a) {
  using SM = PrefillSmem<MT, NST>;
  constexpr int D = 128;
  constexpr uint32_t kTmemCols = MT * 256;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // o_done[b]: PV of the blocks j with j % 2 == b complete (one phase per
  // such block; every waiter is then at most one phase behind)
  __shared__ __align__(8) uint64_t kv_full[NST], kv_empty[NST], s_full[2], p_full[2], o_done[2],
      q_full;
  __shared__ uint32_t s_tmem;
  __shared__ int4 s_plan[kPlanCap];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hs = blockIdx.x;                   // head slice of the selection row
  const int s = blockIdx.z;                    // selection row
  const int unit = a.per_head ? s / a.G : s;   // kv head (with batch)
  const int qh0 = (a.per_head ? s : s * a.G) + hs * a.heads_per_cta;  // first q head
  const int nh = a.per_head ? 1 : min(a.heads_per_cta, a.G - hs * a.heads_per_cta);
  int l, qt;
  if (!a.tile(unit, blockIdx.y, l, qt)) return;
  int bl, el;
  a.ch.range(unit, l, bl, el);
  const int row0 = bl + qt * kTok;             // first query row of the tile
  const int npl = __ldg(a.nplan + (int64_t)s * a.nc + l);
  const int4* plan = a.plans + ((int64_t)s * a.nc + l) * a.cap;
  if (npl <= 0) return;  // capacity overflow (nplan = -1): reported by the host
  // diagonal blocks after the tile's own are causal-masked for all its rows
  const int np = npl - (el - bl + kTok - 1) / kTok + qt + 1;
  for (int e = threadIdx.x; e < np && e < kPlanCap; e += blockDim.x) s_plan[e] = plan[e];

  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4 * MT);
      mbar_init(&o_done[i], 1);
    }
    mbar_init(&q_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&s_tmem, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  // debug timeline (one CTA: the heaviest query chunk of selection row 0)
  unsigned long long* dbg =
      (a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) ? a.dbg : nullptr;
#define PF_T(kind, j)                                                  \
  if (dbg && lane == 0 && (j) < 256) dbg[(kind) * 256 + (j)] = clock64();
  const uint32_t sq = smem_u32(smem + SM::q_off);
  const uint32_t skv = smem_u32(smem + SM::kv_off);

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      prefetch_tmap(&tmQ);
      prefetch_tmap(&tmK);
      prefetch_tmap(&tmV);
      mbar_expect_tx(&q_full, SM::Q);
      for (int rg = 0; rg < 2 * MT; ++rg) {
        const int h = qh0 + (rg < nh ? rg : 0);  // padding row groups repeat a live head
        const int row = h * a.L + row0;
        for (int half = 0; half < 2; ++half)
          tma_load_2d(smem + SM::q_off + (rg >> 1) * 32768 + half * 16384 + (rg & 1) * 8192, &tmQ,
                      &q_full, half * 64, row);
      }
      for (int j = 0; j < np; ++j) {
        const int st = j % NST;
        if (j >= NST) mbar_wait(&kv_empty[st], ((j / NST) - 1) & 1);
        mbar_expect_tx(&kv_full[st], SM::KV);
        const int row = unit * a.L + s_plan[j].x;
        unsigned char* kb = smem + SM::kv_off + st * SM::KV;
        for (int half = 0; half < 2; ++half) {
          tma_load_2d(kb + half * 8192, &tmK, &kv_full[st], half * 64, row);
          tma_load_2d(kb + 16384 + half * 8192, &tmV, &kv_full[st], half * 64, row);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idS = umma_idesc_bf16(128, 64, 0, 0);   // Q K^T: both K-major
      constexpr uint32_t idO = umma_idesc_bf16(128, 128, 0, 1);  // P V: V is MN-major
      mbar_wait(&q_full, 0);
      auto issue_s = [&](int j) {
        const int st = j % NST;
        PF_T(0, j);
        mbar_wait(&kv_full[st], (j / NST) & 1);
        PF_T(1, j);
        tc_fence_after();
        const uint32_t kb = skv + st * SM::KV;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t ad = umma_sdesc(sq + mt * 32768 + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
            const uint64_t bd = umma_sdesc(kb + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024);
            umma_bf16(tmem + mt * 256 + (j & 1) * 64, ad, bd, idS, k > 0);
          }
        }
        umma_commit(&s_full[j & 1]);
      };
      issue_s(0);
      for (int j = 0; j < np; ++j) {
        // S_{j+1} overwrites the buffer of P_{j-1}: PV_{j-1} was issued before it
        if (j + 1 < np) issue_s(j + 1);
        PF_T(2, j);
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);
        PF_T(3, j);
        tc_fence_after();
        const int st = j % NST;
        const uint32_t vb = skv + st * SM::KV + 16384;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 64 keys = 4 x 16; P: 8 packed columns per step
            const uint64_t bd = umma_sdesc(vb + k * 2048, 8192, 1024);
            umma_bf16_ts(tmem + mt * 256 + 128, tmem + mt * 256 + (j & 1) * 64 + k * 8, bd, idO,
                         (j > 0 || k > 0) ? 1u : 0u);
          }
        }
        umma_commit(&kv_empty[st]);
        umma_commit(&o_done[j & 1]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ softmax / epilogue warps
    const int sw = warp - 2;                // 0 .. 4*MT-1
    const int mt = sw >> 2;                 // M tile
    const int quad = warp & 3;              // TMEM lane quadrant of this warp
    const int trow = quad * 32 + lane;      // row within the M tile (= TMEM lane)
    const int r = mt * 128 + trow;          // row within the CTA tile
    const int rg = r >> 6;                  // row group = head slot
    const int i = row0 + (r & 63);          // token index of this query row
    const bool live = rg < nh && i < el;
    const int64_t keep = a.budget < (int64_t)i + 1 ? a.budget : (int64_t)i + 1;
    const int Ri = (int)(keep - 1);
    const int dl = i - bl;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tmem + lane_base + mt * 256;
    const uint32_t tO = tS + 128;
    const float sl2 = a.scale_log2;
    float m_used = -INFINITY, lsum = 0.f;
    for (int j = 0; j < np; ++j) {
      int self;
      int lim = entry_take(s_plan[j], Ri, i, dl, self);
      if (!live) {
        lim = 0;
        self = -1;
      }
      const bool tw = dbg && (warp == 2 || warp == 6);
      const int kb = warp == 2 ? 4 : 9;
      if (tw && lane == 0 && j < 256) dbg[kb * 256 + j] = clock64();
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      if (tw && lane == 0 && j < 256) dbg[(kb + 1) * 256 + j] = clock64();
      tc_fence_after();
      uint32_t v[64];
      tmem_ld32(tS + (j & 1) * 64, *reinterpret_cast<uint32_t(*)[32]>(v));
      tmem_ld32(tS + (j & 1) * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      tmem_wait_ld();
      // raw max (the scale is positive); masking only where some row needs it
      if (!__all_sync(0xffffffffu, lim == 64 && self < 0)) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (!(c < lim || c == self)) v[c] = __float_as_uint(-INFINITY);
      }
      if (tw && lane == 0 && j < 256) dbg[(kb + 2) * 256 + j] = clock64();
      float mx = row_max64(v);
      mx *= sl2;
      // lazy rescale: a row moves its reference max only when its running max
      // grows by > 2^8 (or on its first finite score, when O holds only
      // zero-weight terms).  TMEM loads/stores are warp-collective, so the
      // O rescale runs for the whole warp when any of its rows needs it.
      float m_new = m_used;
      if (mx > -INFINITY && (m_used == -INFINITY || mx > m_used + 8.f)) m_new = mx;
      const bool need = m_used != -INFINITY && m_new != m_used;
      if (__any_sync(0xffffffffu, need)) {
        // O must hold PV_{j-1} (need implies j >= 1); PV_{j-3} completed
        // before S_{j-1}, so o_done[(j-1)&1] is at most one phase behind
        mbar_wait(&o_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
        const float f = need ? exp2f(m_used - m_new) : 1.f;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t o[32];
          tmem_ld32(tO + cc * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < 32; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * f);
          tmem_st32(tO + cc * 32, o);
        }
        tmem_wait_st();
        lsum *= f;
      }
      m_used = m_new;
      const float mref = m_used == -INFINITY ? 0.f : m_used;
      // p = 2^(s*scale - m) on MUFU (a polynomial on the FMA pipe for part of
      // the columns measured slower: the softmax is issue-bound, not MUFU-bound)
      uint32_t pk[32];
      lsum += softmax_pack64(v, sl2, mref, pk);
      if (tw && lane == 0 && j < 256) dbg[(kb + 3) * 256 + j] = clock64();
      tmem_st32(tS + (j & 1) * 64, pk);  // P over the first 32 columns of its S buffer
      tmem_wait_st();
      if (tw && lane == 0 && j < 256) dbg[(kb + 4) * 256 + j] = clock64();
      // observe every o_done phase (PV_{j-1}, long complete by now): no phase
      // of the barrier passes unobserved, so a parity wait never aliases
      if (j >= 1) mbar_wait(&o_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[j & 1]);
    }
    mbar_wait(&o_done[(np - 1) & 1], ((np - 1) >> 1) & 1);  // in-order: every PV done
    tc_fence_after();
    const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
    if (a.row_stats && live) a.row_stats[(int64_t)(qh0 + rg) * a.L + i] = make_float2(m_used, lsum);
    __nv_bfloat16* orow = a.out + ((int64_t)(qh0 + (rg < nh ? rg : 0)) * a.L + i) * D;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      uint32_t o[32];
      tmem_ld32(tO + cc * 32, o);
      tmem_wait_ld();
      if (live) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          uint4 pk4;
          pk4.x = pack_bf16(__uint_as_float(o[8 * t + 0]) * inv, __uint_as_float(o[8 * t + 1]) * inv);
          pk4.y = pack_bf16(__uint_as_float(o[8 * t + 2]) * inv, __uint_as_float(o[8 * t + 3]) * inv);
          pk4.z = pack_bf16(__uint_as_float(o[8 * t + 4]) * inv, __uint_as_float(o[8 * t + 5]) * inv);
          pk4.w = pack_bf16(__uint_as_float(o[8 * t + 6]) * inv, __uint_as_float(o[8 * t + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + cc * 32 + 8 * t) = pk4;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
  if (dbg && threadIdx.x == 0) dbg[14 * 256] = np;
#undef PF_T
}

// Persistent variant: one CTA per SM pulls plans (heavy query chunks first)
// from a device counter and keeps the TMEM allocation, the barriers and the
// K/V ring alive across plans; the next plan's entries and Q tile load while
// the current plan finishes (Q once its last S MMA has been issued, plan
// entries double-buffered), and only the first PV of a plan waits for the
// previous plan's epilogue to have read O.  Per-plan start-up (TMEM alloc,
// Q and first K/V latency, epilogue) otherwise costs ~9 us per CTA.
template <int MT, int NST>
__global__ __launch_bounds__(64 + 128 * MT, 1) void prefill_attn_persist_kernel(
    const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
    const __grid_constant__ CUtensorMap tmV, PrefillArgs a) {
  using SM = PrefillSmem<MT, NST>;
  constexpr int D = 128;
  constexpr uint32_t kTmemCols = MT * 256;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t kv_full[NST], kv_empty[NST], s_full[2], p_full[2], o_done[2],
      q_full, q_empty, o_free, plan_full[2], plan_empty[2];
  __shared__ uint32_t s_tmem;
  __shared__ int4 s_plan[2][kPlanCap];
  __shared__ int4 s_meta[2];  // (plan id or -1, entries, l, s * slices + hs)
  __shared__ int s_qt[2];     // query tile within the chunk

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = a.S * (a.qtiles ? a.T : a.nc) * a.slices;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4 * MT);
      mbar_init(&o_done[i], 1);
      // plan entries are shared-memory hand-offs: every lane that wrote
      // (read) them arrives itself (racecheck-clean, no reliance on
      // __syncwarp cumulativity)
      mbar_init(&plan_full[i], 32);
      mbar_init(&plan_empty[i], 1 + 4 * MT * 32);
    }
    mbar_init(&q_full, 1);
    mbar_init(&q_empty, 1);
    mbar_init(&o_free, 4 * MT);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&s_tmem, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t sq = smem_u32(smem + SM::q_off);
  const uint32_t skv = smem_u32(smem + SM::kv_off);
  // plan p -> (query tile y, selection row s, head slice hs), heavy first
  auto decode = [&](int p, int& y, int& sr, int& hs) {
    const int per_l = a.S * a.slices;
    y = p / per_l;
    const int r = p - y * per_l;
    sr = r / a.slices;
    hs = r - sr * a.slices;
  };

  if (warp == 0) {
    // ------------------------------------------------ producer warp
    if (lane == 0) {
      prefetch_tmap(&tmQ);
      prefetch_tmap(&tmK);
      prefetch_tmap(&tmV);
    }
    int jg = 0, kq = 0;
    for (int k = 0;; ++k) {
      const int b = k & 1;
      int p = 0;
      if (lane == 0) p = atomicAdd(a.counters, 1);
      p = __shfl_sync(0xffffffffu, p, 0);
      if (k >= 2) mbar_wait(&plan_empty[b], ((k >> 1) - 1) & 1);
      if (p >= total) {
        if (lane == 0) s_meta[b] = make_int4(-1, 0, 0, 0);
        mbar_arrive(&plan_full[b]);
        break;
      }
      int y, sr, hs, l = 0, qt = 0;
      decode(p, y, sr, hs);
      const int unit = a.per_head ? sr / a.G : sr;
      int np = 0, bl = 0, el = 0;
      if (a.tile(unit, y, l, qt)) {
        a.ch.range(unit, l, bl, el);
        np = __ldg(a.nplan + (int64_t)sr * a.nc + l);
        if (np > 0) np = np - (el - bl + kTok - 1) / kTok + qt + 1;
      }
      const int4* plan = a.plans + ((int64_t)sr * a.nc + l) * a.cap;
      for (int e = lane; e < np && e < kPlanCap; e += 32) s_plan[b][e] = __ldg(plan + e);
      if (lane == 0) {
        s_meta[b] = make_int4(p, np, l, sr * a.slices + hs);
        s_qt[b] = qt;
      }
      __syncwarp();  // lane 0 reads the other lanes' entries below
      mbar_arrive(&plan_full[b]);
      if (np <= 0) continue;  // capacity overflow: reported by the host
      if (lane == 0) {
        const int qh0 = (a.per_head ? sr : sr * a.G) + hs * a.heads_per_cta;
        const int nh = a.per_head ? 1 : min(a.heads_per_cta, a.G - hs * a.heads_per_cta);
        const int row0 = bl + qt * kTok;
        if (kq >= 1) mbar_wait(&q_empty, (kq - 1) & 1);  // every S of the previous plan done
        mbar_expect_tx(&q_full, SM::Q);
        for (int rg = 0; rg < 2 * MT; ++rg) {
          const int h = qh0 + (rg < nh ? rg : 0);
          const int row = h * a.L + row0;
          for (int half = 0; half < 2; ++half)
            tma_load_2d(smem + SM::q_off + (rg >> 1) * 32768 + half * 16384 + (rg & 1) * 8192, &tmQ,
                        &q_full, half * 64, row);
        }
        for (int j = 0; j < np; ++j, ++jg) {
          const int st = jg % NST;
          if (jg >= NST) mbar_wait(&kv_empty[st], ((jg / NST) - 1) & 1);
          mbar_expect_tx(&kv_full[st], SM::KV);
          const int row = unit * a.L + s_plan[b][j].x;
          unsigned char* kb = smem + SM::kv_off + st * SM::KV;
          for (int half = 0; half < 2; ++half) {
            tma_load_2d(kb + half * 8192, &tmK, &kv_full[st], half * 64, row);
            tma_load_2d(kb + 16384 + half * 8192, &tmV, &kv_full[st], half * 64, row);
          }
        }
      }
      jg = __shfl_sync(0xffffffffu, jg, 0);
      ++kq;
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idS = umma_idesc_bf16(128, 64, 0, 0);
      constexpr uint32_t idO = umma_idesc_bf16(128, 128, 0, 1);
      int jg0 = 0, kq = 0;
      for (int k = 0;; ++k) {
        const int b = k & 1;
        mbar_wait(&plan_full[b], (k >> 1) & 1);
        const int4 m = s_meta[b];
        if (m.x < 0) break;
        const int np = m.y;
        if (np <= 0) {
          mbar_arrive(&plan_empty[b]);
          continue;
        }
        mbar_wait(&q_full, kq & 1);
        auto issue_s = [&](int jj) {
          const int st = jj % NST;
          mbar_wait(&kv_full[st], (jj / NST) & 1);
          tc_fence_after();
          const uint32_t kb = skv + st * SM::KV;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint64_t ad = umma_sdesc(sq + mt * 32768 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
              const uint64_t bd = umma_sdesc(kb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
              umma_bf16(tmem + mt * 256 + (jj & 1) * 64, ad, bd, idS, kk > 0);
            }
          }
          umma_commit(&s_full[jj & 1]);
        };
        issue_s(jg0);
        if (np == 1) umma_commit(&q_empty);
        for (int j = 0; j < np; ++j) {
          const int jj = jg0 + j;
          if (j + 1 < np) {
            issue_s(jj + 1);
            if (j + 2 == np) umma_commit(&q_empty);  // the plan's last S: Q may be replaced
          }
          mbar_wait(&p_full[jj & 1], (jj >> 1) & 1);
          if (j == 0 && kq >= 1) mbar_wait(&o_free, (kq - 1) & 1);  // O of the previous plan read
          tc_fence_after();
          const int st = jj % NST;
          const uint32_t vb = skv + st * SM::KV + 16384;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t bd = umma_sdesc(vb + kk * 2048, 8192, 1024);
              umma_bf16_ts(tmem + mt * 256 + 128, tmem + mt * 256 + (jj & 1) * 64 + kk * 8, bd, idO,
                           (j > 0 || kk > 0) ? 1u : 0u);
            }
          }
          umma_commit(&kv_empty[st]);
          umma_commit(&o_done[jj & 1]);
        }
        mbar_arrive(&plan_empty[b]);
        jg0 += np;
        ++kq;
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ softmax / epilogue warps
    const int sw = warp - 2;
    const int mt = sw >> 2;
    const int quad = warp & 3;
    const int trow = quad * 32 + lane;
    const int r = mt * 128 + trow;
    const int rg = r >> 6;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tmem + lane_base + mt * 256;
    const uint32_t tO = tS + 128;
    const float sl2 = a.scale_log2;
    int jg0 = 0;
    for (int k = 0;; ++k) {
      const int b = k & 1;
      mbar_wait(&plan_full[b], (k >> 1) & 1);
      const int4 m = s_meta[b];
      if (m.x < 0) break;
      const int np = m.y;
      if (np <= 0) {
        mbar_arrive(&plan_empty[b]);
        continue;
      }
      const int l = m.z, sr = m.w / a.slices, hs = m.w - sr * a.slices;
      const int qh0 = (a.per_head ? sr : sr * a.G) + hs * a.heads_per_cta;
      const int nh = a.per_head ? 1 : min(a.heads_per_cta, a.G - hs * a.heads_per_cta);
      int bl, el;
      a.ch.range(a.per_head ? sr / a.G : sr, l, bl, el);
      const int i = bl + s_qt[b] * kTok + (r & 63);
      const bool live = rg < nh && i < el;
      const int64_t keep = a.budget < (int64_t)i + 1 ? a.budget : (int64_t)i + 1;
      const int Ri = (int)(keep - 1);
      const int dl = i - bl;
      float m_used = -INFINITY, lsum = 0.f;
      for (int j = 0; j < np; ++j) {
        const int jj = jg0 + j;
        int self;
        int lim = entry_take(s_plan[b][j], Ri, i, dl, self);
        if (!live) {
          lim = 0;
          self = -1;
        }
        mbar_wait(&s_full[jj & 1], (jj >> 1) & 1);
        tc_fence_after();
        uint32_t v[64];
        tmem_ld32(tS + (jj & 1) * 64, *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_ld32(tS + (jj & 1) * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        tmem_wait_ld();
        if (!__all_sync(0xffffffffu, lim == 64 && self < 0)) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (!(c < lim || c == self)) v[c] = __float_as_uint(-INFINITY);
        }
        float mx = row_max64(v);
        mx *= sl2;
        float m_new = m_used;
        if (mx > -INFINITY && (m_used == -INFINITY || mx > m_used + 8.f)) m_new = mx;
        const bool need = m_used != -INFINITY && m_new != m_used;
        if (__any_sync(0xffffffffu, need)) {
          mbar_wait(&o_done[(jj - 1) & 1], ((jj - 1) >> 1) & 1);  // j >= 1 here
          tc_fence_after();
          const float f = need ? exp2f(m_used - m_new) : 1.f;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            uint32_t o[32];
            tmem_ld32(tO + cc * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int t = 0; t < 32; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * f);
            tmem_st32(tO + cc * 32, o);
          }
          tmem_wait_st();
          lsum *= f;
        }
        m_used = m_new;
        const float mref = m_used == -INFINITY ? 0.f : m_used;
        uint32_t pk[32];
        lsum += softmax_pack64(v, sl2, mref, pk);
        tmem_st32(tS + (jj & 1) * 64, pk);
        tmem_wait_st();
        // observe every o_done phase (PV_{jj-1}, long complete by now): no
        // phase of the barrier passes unobserved, so a parity wait never aliases
        if (jj >= 1) mbar_wait(&o_done[(jj - 1) & 1], ((jj - 1) >> 1) & 1);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[jj & 1]);
      }
      const int jl = jg0 + np - 1;
      mbar_wait(&o_done[jl & 1], (jl >> 1) & 1);  // in-order: every PV of the plan done
      tc_fence_after();
      const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
      if (a.row_stats && live) a.row_stats[(int64_t)(qh0 + rg) * a.L + i] = make_float2(m_used, lsum);
      __nv_bfloat16* orow = a.out + ((int64_t)(qh0 + (rg < nh ? rg : 0)) * a.L + i) * D;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t o[32];
        tmem_ld32(tO + cc * 32, o);
        tmem_wait_ld();
        if (live) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            uint4 pk4;
            pk4.x = pack_bf16(__uint_as_float(o[8 * t + 0]) * inv, __uint_as_float(o[8 * t + 1]) * inv);
            pk4.y = pack_bf16(__uint_as_float(o[8 * t + 2]) * inv, __uint_as_float(o[8 * t + 3]) * inv);
            pk4.z = pack_bf16(__uint_as_float(o[8 * t + 4]) * inv, __uint_as_float(o[8 * t + 5]) * inv);
            pk4.w = pack_bf16(__uint_as_float(o[8 * t + 6]) * inv, __uint_as_float(o[8 * t + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + cc * 32 + 8 * t) = pk4;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free);  // the next plan's first PV may overwrite O
      mbar_arrive(&plan_empty[b]);           // plan entries no longer read (every lane)
      jg0 += np;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
  if (threadIdx.x == 0) {  // the last CTA out re-arms the plan counter
    __threadfence();
    if (atomicAdd(a.counters + 1, 1) == (int)gridDim.x - 1) {
      a.counters[0] = 0;
      a.counters[1] = 0;
    }
  }
}

template <int MT, int NST>
static int launch_prefill_persist(const CUtensorMap& mq, const CUtensorMap& mk,
                                  const CUtensorMap& mv, const PrefillArgs& a, cudaStream_t st) {
  using SM = PrefillSmem<MT, NST>;
  auto kern = prefill_attn_persist_kernel<MT, NST>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::total);
  if (e != cudaSuccess) {
    set_error("dhsa_prefill_attn: %s", cudaGetErrorString(e));
    return DHSA_ECUDA;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total = a.S * (a.qtiles ? a.T : a.nc) * a.slices;
  const int grid = total < sms ? total : sms;
  kern<<<grid, 64 + 128 * MT, SM::total, st>>>(mq, mk, mv, a);
  return check_launch("dhsa_prefill_attn");
}

template <int MT, int NST>
static int launch_prefill_attn(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                               const PrefillArgs& a, int S, cudaStream_t st) {
  using SM = PrefillSmem<MT, NST>;
  auto kern = prefill_attn_kernel<MT, NST>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::total);
  if (e != cudaSuccess) {
    set_error("dhsa_prefill_attn: %s", cudaGetErrorString(e));
    return DHSA_ECUDA;
  }
  dim3 grid((unsigned)a.slices, (unsigned)(a.qtiles ? a.T : a.nc), (unsigned)S);
  kern<<<grid, 64 + 128 * MT, SM::total, st>>>(mq, mk, mv, a);
  return check_launch("dhsa_prefill_attn");
}

// ----------------------------------------------------- mask export (8f) --
// The per-row token sets the plans encode, as the reference's DHSAMSK1 row
// bitsets (serialization.py:80-94: ceil(L/8) bytes per row, token t = bit
// t % 8 of byte t / 8).  One CTA per (query chunk, selection row); each row
// is assembled in shared memory with word atomics and streamed out.
__global__ __launch_bounds__(128) void plan_bitsets_kernel(const int4* __restrict__ plans,
                                                           const int32_t* __restrict__ nplan,
                                                           int cap, int nc, PrefillChunks ch,
                                                           int G, int per_head, int64_t budget,
                                                           int64_t nbytes,
                                                           uint8_t* __restrict__ out) {
  extern __shared__ uint32_t rowbits[];
  const int l = blockIdx.x, s = blockIdx.y, tid = threadIdx.x;
  const int u = per_head ? s / G : s;
  if (l >= ch.count(u, nc)) return;
  const int L = ch.L;
  const int np = nplan[(int64_t)s * nc + l];
  const int4* plan = plans + ((int64_t)s * nc + l) * cap;
  const int nwords = (int)((nbytes + 3) / 4);
  int bl, el;
  ch.range(u, l, bl, el);
  for (int i = bl; i < el; ++i) {
    for (int w = tid; w < nwords; w += 128) rowbits[w] = 0u;
    __syncthreads();
    const int64_t keep = budget < (int64_t)i + 1 ? budget : (int64_t)i + 1;
    const int Ri = (int)(keep - 1), dl = i - bl;
    for (int e = tid; e < np; e += 128) {
      const int4 en = plan[e];
      int self;
      const int lim = entry_take(en, Ri, i, dl, self);
      for (int t = en.x; t < en.x + lim;) {  // word-sized pieces of [start, start + lim)
        const int w = t >> 5, b0 = t & 31;
        const int n = min(32 - b0, en.x + lim - t);
        const uint32_t m = (n == 32 ? 0xFFFFFFFFu : ((1u << n) - 1u)) << b0;
        atomicOr(&rowbits[w], m);
        t += n;
      }
    }
    if (tid == 0 && np > 0) atomicOr(&rowbits[i >> 5], 1u << (i & 31));  // self
    __syncthreads();
    uint8_t* dst = out + ((int64_t)s * L + i) * nbytes;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(rowbits);  // little-endian words
    for (int64_t b = tid; b < nbytes; b += 128) dst[b] = src[b];
    __syncthreads();
  }
}

// --------------------------------------------- mask quality (8f row 3) --
// Per query row of one q head: the attention mass the selection captures,
// sum_{j in sel} p_ij = l_sel 2^(m_sel - m_all) / l_all (harness.py:265-274,
// from the sparse and the dense run's (m, l) row statistics), and the cosine
// of the sparse and dense outputs (harness.py:277-285, core.py:139-152).
// One warp per row.
__global__ void row_quality_kernel(const float2* __restrict__ st_sel,
                                   const float2* __restrict__ st_all,
                                   const __nv_bfloat16* __restrict__ o_sel,
                                   const __nv_bfloat16* __restrict__ o_all, int64_t rows, int D,
                                   float* __restrict__ recall, float* __restrict__ cosine) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (int d = lane; d < D; d += 32) {
    const double x = __bfloat162float(o_sel[r * D + d]), y = __bfloat162float(o_all[r * D + d]);
    dot += x * y;
    na += x * x;
    nb += y * y;
  }
  dot = warp_sum(dot);
  na = warp_sum(na);
  nb = warp_sum(nb);
  if (lane == 0) {
    const float2 s = st_sel[r], t = st_all[r];
    recall[r] = t.y > 0.f ? (float)((double)s.y * exp2((double)s.x - (double)t.x) / (double)t.y) : 0.f;
    cosine[r] = (na > 0.0 && nb > 0.0) ? (float)(dot / sqrt(na * nb)) : 0.f;
  }
}

}  // namespace dhsa

using namespace dhsa;

extern "C" int dhsa_row_quality(const float* stats_sel, const float* stats_all,
                                const void* out_sel, const void* out_all, int64_t rows, int D,
                                float* recall, float* cosine, dhsa_stream_t stream) {
  DHSA_REQUIRE(stats_sel && stats_all && out_sel && out_all && recall && cosine && rows >= 1 &&
                   D >= 1,
               "dhsa_row_quality: bad arguments");
  const unsigned grid = (unsigned)((rows + 7) / 8);
  row_quality_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      (const float2*)stats_sel, (const float2*)stats_all, (const __nv_bfloat16*)out_sel,
      (const __nv_bfloat16*)out_all, rows, D, recall, cosine);
  return check_launch("dhsa_row_quality");
}

// Chunk layout from the C struct (null = static grid of `block`).
static PrefillChunks make_chunks(const dhsa_prefill_chunks* c, int block, int L) {
  PrefillChunks ch{};
  ch.block = block;
  ch.L = L;
  if (c && c->bounds) {
    ch.bounds = c->bounds;
    ch.bstride = c->bounds_stride;
    ch.nchunks = c->nchunks;
  }
  return ch;
}

static int check_chunks(const dhsa_prefill_chunks* c, int n_chunks, int L, int block,
                        bool need_tiles, const char* who) {
  if (c && c->bounds) {
    DHSA_REQUIRE(c->nchunks, "%s: explicit bounds need nchunks", who);
    DHSA_REQUIRE(c->bounds_stride == 0 || c->bounds_stride >= n_chunks + 1,
                 "%s: bounds_stride must be 0 or >= n_chunks + 1", who);
    DHSA_REQUIRE(!need_tiles || (c->qtiles && c->tiles_per_unit >= 1),
                 "%s: explicit bounds need the query tile table", who);
  } else {
    DHSA_REQUIRE((int64_t)(n_chunks - 1) * block < L && (int64_t)n_chunks * block >= L,
                 "%s: n_chunks does not match L / block", who);
  }
  return DHSA_OK;
}

extern "C" int dhsa_prefill_mask_bitsets(const void* plans, const int32_t* nplan, int cap, int S,
                                         int G, int agg, int n_chunks, int L, int block,
                                         int64_t budget, const dhsa_prefill_chunks* chunks,
                                         uint8_t* out, dhsa_stream_t stream) {
  DHSA_REQUIRE(plans && nplan && out && S >= 1 && G >= 1 && n_chunks >= 1 && L >= 1 && block >= 1,
               "dhsa_prefill_mask_bitsets: bad arguments");
  DHSA_REQUIRE(budget >= 1, "budget must be >= 1");
  int rc = check_chunks(chunks, n_chunks, L, block, false, "dhsa_prefill_mask_bitsets");
  if (rc) return rc;
  const int64_t nbytes = ((int64_t)L + 7) / 8;
  const size_t smem = (size_t)((nbytes + 3) / 4) * 4;
  DHSA_REQUIRE(smem <= 200 * 1024, "dhsa_prefill_mask_bitsets: L too large (%d)", L);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(plan_bitsets_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      set_error("dhsa_prefill_mask_bitsets: %s", cudaGetErrorString(e));
      return DHSA_ECUDA;
    }
  }
  dim3 grid((unsigned)n_chunks, (unsigned)S);
  plan_bitsets_kernel<<<grid, 128, smem, (cudaStream_t)stream>>>(
      (const int4*)plans, nplan, cap, n_chunks, make_chunks(chunks, block, L), G,
      agg == DHSA_AGG_NONE, budget, nbytes, out);
  return check_launch("dhsa_prefill_mask_bitsets");
}

extern "C" int dhsa_prefill_scores(const double* q_centroids, const double* k_centroids, int U,
                                   int G, int n_chunks, int D, int agg, double* scores,
                                   dhsa_stream_t stream) {
  DHSA_REQUIRE(q_centroids && k_centroids && scores && U >= 1 && G >= 1 && n_chunks >= 1 &&
                   D >= 1,
               "dhsa_prefill_scores: bad arguments");
  DHSA_REQUIRE(agg == DHSA_AGG_NONE || agg == DHSA_AGG_MAX || agg == DHSA_AGG_MEAN,
               "dhsa_prefill_scores: unknown aggregation %d", agg);
  const int per_head = agg == DHSA_AGG_NONE;
  const int S = per_head ? U * G : U;
  const int t = (n_chunks + kScT - 1) / kScT;
  dim3 grid((unsigned)t, (unsigned)t, (unsigned)S);
  bool dmma = D == 128;
  if (const char* e = getenv("DHSA_SCORES_DMMA")) dmma = dmma && atoi(e) != 0;
  if (dmma) {
    constexpr int smem = 3 * 64 * (128 + 4) * 8;
    cudaError_t e = cudaFuncSetAttribute(prefill_scores_dmma_kernel<128>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) {
      set_error("dhsa_prefill_scores: %s", cudaGetErrorString(e));
      return DHSA_ECUDA;
    }
    prefill_scores_dmma_kernel<128><<<grid, 256, smem, (cudaStream_t)stream>>>(
        q_centroids, k_centroids, n_chunks, G, per_head, agg, scores);
    return check_launch("dhsa_prefill_scores");
  }
  prefill_scores_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(q_centroids, k_centroids, n_chunks,
                                                                 D, G, per_head, agg, scores);
  return check_launch("dhsa_prefill_scores");
}

extern "C" int dhsa_prefill_plan_capacity(int64_t budget, int block) {
  if (budget < 1 || block < 1 || block > kTok) return -1;
  return (int)((budget - 1 + block - 1) / block) + 2;
}

extern "C" int dhsa_prefill_plan(const double* scores, int S, int G, int agg, int n_chunks, int L,
                                 int block, int64_t budget, const dhsa_prefill_chunks* chunks,
                                 int cap, void* plans, int32_t* nplan, dhsa_stream_t stream) {
  DHSA_REQUIRE(scores && plans && nplan && S >= 1 && G >= 1 && n_chunks >= 1 && block >= 1 &&
                   L >= 1,
               "dhsa_prefill_plan: bad arguments");
  DHSA_REQUIRE(budget >= 1, "budget must be >= 1");
  int rc = check_chunks(chunks, n_chunks, L, block, false, "dhsa_prefill_plan");
  if (rc) return rc;
  DHSA_REQUIRE(cap >= 2, "dhsa_prefill_plan: capacity too small");
  const size_t smem = (size_t)n_chunks * (8 + 4 + 4 + 4);
  DHSA_REQUIRE(smem <= 200 * 1024, "dhsa_prefill_plan: too many chunks (%d)", n_chunks);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(prefill_plan_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      set_error("dhsa_prefill_plan: %s", cudaGetErrorString(e));
      return DHSA_ECUDA;
    }
  }
  dim3 grid((unsigned)n_chunks, (unsigned)S);
  prefill_plan_kernel<<<grid, kPlanThreads, smem, (cudaStream_t)stream>>>(
      scores, n_chunks, make_chunks(chunks, block, L), G, agg == DHSA_AGG_NONE, budget, cap,
      (int4*)plans, nplan);
  return check_launch("dhsa_prefill_plan");
}

extern "C" int dhsa_prefill_attn(const void* q, const void* k, const void* v, int U, int G, int L,
                                 int D, int block, int agg, int64_t budget, int n_chunks,
                                 const dhsa_prefill_chunks* chunks, const void* plans,
                                 const int32_t* nplan, int cap, void* out, int32_t* counters,
                                 float* row_stats, dhsa_stream_t stream) {
  DHSA_REQUIRE(q && k && v && plans && nplan && out, "dhsa_prefill_attn: null pointer");
  DHSA_REQUIRE(D == 128, "dhsa_prefill_attn: head_dim must be 128 (got %d)", D);
  const bool explicit_bounds = chunks && chunks->bounds;
  DHSA_REQUIRE(explicit_bounds || block == 64,
               "dhsa_prefill_attn: the static grid needs 64-token chunks");
  int rc0 = check_chunks(chunks, n_chunks, L, block, true, "dhsa_prefill_attn");
  if (rc0) return rc0;
  DHSA_REQUIRE(U >= 1 && G >= 1 && L >= 1 && cap >= 2 && cap <= kPlanCap,
               "dhsa_prefill_attn: bad shape (plan capacity <= %d)", kPlanCap);
  DHSA_REQUIRE(budget >= 1, "budget must be >= 1");
  DHSA_REQUIRE(((uintptr_t)q & 15) == 0 && ((uintptr_t)k & 15) == 0 && ((uintptr_t)v & 15) == 0 &&
                   ((uintptr_t)out & 15) == 0,
               "dhsa_prefill_attn: pointers must be 16-byte aligned");
  DHSA_REQUIRE((int64_t)U * G * L < (1ll << 31), "dhsa_prefill_attn: too many rows for TMA");
  const int per_head = agg == DHSA_AGG_NONE;
  CUtensorMap mq, mk, mv;
  int rc = make_tmap_2d(&mq, q, (int64_t)U * G * L, D, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  if (rc) return rc;
  rc = make_tmap_2d(&mk, k, (int64_t)U * L, D, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  if (rc) return rc;
  rc = make_tmap_2d(&mv, v, (int64_t)U * L, D, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  if (rc) return rc;
  PrefillArgs a{};
  a.plans = (const int4*)plans;
  a.nplan = nplan;
  a.cap = cap;
  a.nc = n_chunks;
  a.L = L;
  a.ch = make_chunks(chunks, block, L);
  if (explicit_bounds) {
    a.qtiles = reinterpret_cast<const int2*>(chunks->qtiles);
    a.T = chunks->tiles_per_unit;
  }
  a.block = block;
  a.budget = budget;
  a.G = G;
  a.per_head = per_head;
  const int gsel = per_head ? 1 : G;
  a.heads_per_cta = gsel < 4 ? gsel : 4;
  a.slices = (gsel + a.heads_per_cta - 1) / a.heads_per_cta;
  a.out = (__nv_bfloat16*)out;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)D));
  const int S = per_head ? U * G : U;
  a.S = S;
  a.counters = counters;
  a.row_stats = reinterpret_cast<float2*>(row_stats);
  if (const char* e = getenv("DHSA_DEBUG_TIMING")) a.dbg = (unsigned long long*)strtoull(e, nullptr, 0);
  cudaStream_t st = (cudaStream_t)stream;
  // persistent plans pay off when plans are short (per-plan start-up is a
  // large share): r2 measurement (C5 sweep): +0% at budget 1025, +4.5% at
  // 2049, +1.8% at 4097, -8% at 8193 / 16385 on the static grid; with
  // explicit bounds (many short query tiles) +2% at 4097
  bool persist = counters != nullptr && (budget <= 4200 || explicit_bounds);
  if (const char* e = getenv("DHSA_PREFILL_PERSISTENT")) persist = counters != nullptr && atoi(e) != 0;
  if (persist) {
    if (a.heads_per_cta > 2) return launch_prefill_persist<2, 4>(mq, mk, mv, a, st);
    return launch_prefill_persist<1, 5>(mq, mk, mv, a, st);
  }
  if (a.heads_per_cta > 2) return launch_prefill_attn<2, 4>(mq, mk, mv, a, S, st);
  return launch_prefill_attn<1, 5>(mq, mk, mv, a, S, st);
}
