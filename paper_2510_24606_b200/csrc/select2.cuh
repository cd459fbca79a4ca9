// Compact certified select for the bf16 sketch decode path (units of up to
// 3 x 1024 chunks: every static-grid unit up to 192K tokens, e.g. C2/C3).
//
// Same semantics and certificate as sketch_select_kernel (decode_sketch.cu;
// DESIGN.md section 4): the exact token-budget Top-K of masks.topk_row
// (masks.py:103-122) over the decode row of masks._decode_row
// (masks.py:153-173), from the fp32 sketch scores, with every chunk that the
// sketch cannot order against the cut re-scored in fp64.
//
// Why a second kernel: at small batch the select is on the critical path of
// every step and it is LATENCY-bound — ncu shows the generic kernel spending
// most cycles on instruction fetch (straight-line unrolled code executed once
// per launch), barriers and dependent chains, not on data.  This one keeps
// the hot path short: 1024 threads, thread t owns chunks t, t+1024, t+2048
// (coalesced scalar loads, 3 registers), and the per-chunk decisions become
// ballot words (one word per warp and element: no atomics, chunk order for
// free).  The tail after classification is done by single warps:
//
//   all warps  min/max, weighted 1024-bin histogram, cut bin b* (every warp
//              scans the histogram redundantly: no barrier), certified
//              classification -> whole / uncertain bit words;
//   warp 0     tiles of the chunks kept whole, in chunk order (published at
//              once to the attention when few items run);
//   warp 1     uncertain list in chunk order, then warps 1..31 re-score the
//              uncertain chunks in fp64 (a warp per chunk);
//   warp 0     exact walk among <= 32 uncertain chunks in registers (rank by
//              (fp64 score desc, chunk asc), budget R - W(whole)), their
//              tiles, the self tile, the ready flag.
//
// 33..1024 uncertain chunks: takes by every thread, tiles by warp 0 in 32-wide
// batches; more than 1024 (massive ties): the generic weighted 64-bit radix
// select over every chunk in global scratch (out of line).
#pragma once

#include "sketch_common.cuh"

namespace dhsa {

// shapes: 256 threads x 4 / 9 / 12 chunks (units of <= 1024 / 2304 / 3072
// chunks: C1/C2, the 128K units of C3 and its rank proxies (2048 prompt
// chunks + the generated one), every static-grid unit up to 192K tokens) and
// 1024 threads x 17 chunks (<= 17408 chunks: a 1M-token unit, config C4 on
// one GPU).  The per-thread element loops are unrolled over the shape's chunk
// count, so a unit runs the smallest shape that holds it.
#ifndef SELECT3_MIN_CTAS
#define SELECT3_MIN_CTAS 3  // 256-thread shapes: register cap 85 (3) or 64 (4) per thread
#endif
constexpr int kS3Threads = 256;
#ifndef S3_MED_NT
#define S3_MED_NT 256
#define S3_MED_PER 9
#endif
constexpr int kS3PerS = 4, kS3PerM = S3_MED_PER, kS3Per = 12;  // chunks per thread
constexpr int kS3ThreadsM = S3_MED_NT;  // threads of the middle shape (C3's 2049-chunk units)
constexpr int kS3MaxChunks = kS3Threads * kS3Per;
#ifndef S3_WIDE_THREADS
#define S3_WIDE_THREADS 1024
#define S3_WIDE_PER 17
#endif
constexpr int kS3WideThreads = S3_WIDE_THREADS;
constexpr int kS3WidePer = S3_WIDE_PER;  // 1024 x 17 = 17408 >= 16384 prompt chunks + the generated one
constexpr int kS3WideMaxChunks = kS3WideThreads * kS3WidePer;

// tiles of a take of `len` tokens (len <= T in the static grid: one)
__device__ __forceinline__ int ntiles_of(int len, int T) { return len <= T ? 1 : (len + T - 1) / T; }

// monotone fp32 value binning shared by the histogram and the classification
// bin(x) = clamp(floor(fma(x, bscale, off)), 0, kHistBins-1), off = -vmin*bscale:
// one rounding of an increasing affine map, then floor and clamp — monotone
// non-decreasing in x (F2I saturates +-inf; NaN only with bscale 0 and an
// infinite bound, where every chunk is uncertain anyway: see the caller).
__device__ __forceinline__ int bin32(float x, float bscale, float off) {
  const int b = __float2int_rd(__fmaf_rn(x, bscale, off));
  return min(max(b, 0), kHistBins - 1);
}

__device__ __forceinline__ int hist_pad(int b) { return b + (b >> 5); }

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ int warp_incl_scan(int x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Tiles of the chunks whose bits are set in words[0 .. 32 WPL), in chunk
// order, starting at tile index `base`; one warp (lane l owns words
// WPL l .. WPL l + WPL - 1).  Returns the tile count (uniform over the warp).
// The lanes first compact their chunk ids into `list` (a short divergent
// loop: one shared store per chunk), then the warp emits the tiles 32 chunks
// at a time without divergence — emitting from inside the per-lane bit loops
// serialised the 32 lanes' chunk work (2.7 us at 2K chunks, 7 us at 16K).
// More than `list_cap` chunks: the per-lane loops (every causal token kept).
template <int kS3WPL>
static __device__ __forceinline__ int s3_emit_whole(const UnitChunks& uc, const uint32_t* words,
                                          int tile_tokens, int32_t* out, int64_t cap, int base,
                                          int32_t* list, int list_cap,
                                          unsigned long long* dbg = nullptr) {
  const int lane = threadIdx.x & 31;
  if (dbg && lane == 0) dbg[11] = clock64();
  uint32_t w[kS3WPL];
  int cnt = 0;
#pragma unroll
  for (int j = 0; j < kS3WPL; ++j) {
    w[j] = words[kS3WPL * lane + j];
    cnt += __popc(w[j]);
  }
  const int incl = warp_incl_scan(cnt, lane);
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (dbg && lane == 0) dbg[12] = clock64();
  if (total <= list_cap) {
    int pos = incl - cnt;
#pragma unroll
    for (int j = 0; j < kS3WPL; ++j) {
      uint32_t m = w[j];
      while (m) {
        list[pos++] = 32 * (kS3WPL * lane + j) + __ffs(m) - 1;
        m &= m - 1;
      }
    }
    __syncwarp();
    if (dbg && lane == 0) dbg[13] = clock64();
    int off = base;
    for (int i0 = 0; i0 < total; i0 += 32) {
      const int i = i0 + lane;
      int lo = 0, len = 0;
      if (i < total) uc.chunk(list[i], lo, len);
      const int nt = len > 0 ? ntiles_of(len, tile_tokens) : 0;
      const int ti = warp_incl_scan(nt, lane);
      int o = off + ti - nt;
      for (int t = 0; t < len; t += tile_tokens, ++o)
        if (o < cap) {
          out[2 * o] = lo + t;
          out[2 * o + 1] = min(tile_tokens, len - t);
        }
      off += __shfl_sync(0xffffffffu, ti, 31);
    }
    __syncwarp();
    if (dbg && lane == 0) dbg[14] = clock64();
    return off - base;
  }
  // every causal token kept (thousands of whole chunks): per-lane loops
  cnt = 0;
#pragma unroll
  for (int j = 0; j < kS3WPL; ++j) {
    uint32_t m = w[j];
    while (m) {
      const int c = 32 * (kS3WPL * lane + j) + __ffs(m) - 1;
      m &= m - 1;
      int lo, len;
      uc.chunk(c, lo, len);
      cnt += ntiles_of(len, tile_tokens);
    }
  }
  const int tincl = warp_incl_scan(cnt, lane);
  int off = base + tincl - cnt;
  if (dbg && lane == 0) dbg[13] = clock64();
#pragma unroll
  for (int j = 0; j < kS3WPL; ++j) {
    uint32_t m = w[j];
    while (m) {
      const int c = 32 * (kS3WPL * lane + j) + __ffs(m) - 1;
      m &= m - 1;
      int lo, len;
      uc.chunk(c, lo, len);
      for (int t = 0; t < len; t += tile_tokens, ++off)
        if (off < cap) {
          out[2 * off] = lo + t;
          out[2 * off + 1] = min(tile_tokens, len - t);
        }
    }
  }
  __syncwarp();
  if (dbg && lane == 0) dbg[14] = clock64();
  return __shfl_sync(0xffffffffu, tincl, 31);
}

// Generic fallback (> kSmallUncertain uncertain chunks): every chunk's key in
// global scratch (whole ~0, outside 0, uncertain its exact fp64 key, written
// by the re-scoring), the weighted radix select, takes, tiles after `base`.
// (scalar arguments only: a reference to the kernel parameters would force
// them into local memory in every thread of the hot path)
template <int kS3Threads>
static __device__ __noinline__ void s3_fallback(UnitChunks uc, int n, uint32_t R, int row,
                                                int base, const uint32_t* inbits,
                                                const uint32_t* uncbits, uint64_t* key64,
                                                int32_t* lens, int tile_tokens, int32_t* out,
                                                int64_t tile_cap, int32_t* ntiles_out,
                                                int emit) {
  __shared__ WalkShared sh;
  for (int c = threadIdx.x; c < n; c += kS3Threads) {
    const uint32_t bit = 1u << (c & 31);
    int lo, len;
    uc.chunk(c, lo, len);
    if (inbits[c >> 5] & bit) key64[c] = ~0ull;
    else if (!(uncbits[c >> 5] & bit)) key64[c] = 0ull;
    lens[c] = len;
  }
  __syncthreads();
  uint64_t prefix = 0, mask = 0;
  uint32_t rrem = R;
  radix_threshold<kS3Threads, uint64_t>(key64, lens, n, R, sh, prefix, mask, rrem);
  walk_takes<kS3Threads, uint64_t>(key64, lens, n, R, prefix, mask, rrem, sh);
  if (!emit) return;  // split-KV candidate mode: lens[] = every chunk's take
  for (int c = threadIdx.x; c < n; c += kS3Threads)  // the whole chunks were emitted before
    if (key64[c] == ~0ull) lens[c] = 0;
  __syncthreads();
  emit_takes<kS3Threads>(uc, lens, n, row, tile_tokens, out, tile_cap, ntiles_out, sh, base);
}

template <int D, int G, int AGG, int NT, int kS3Per>
__global__ __launch_bounds__(NT, NT > 256 ? 1 : SELECT3_MIN_CTAS) void sketch_select3_kernel(SketchArgs a) {
  constexpr int NW = NT / 32;
  static_assert(kS3Per <= 32, "per-thread chunk flags are 32-bit masks");
  constexpr int kS3Words = NT * kS3Per / 32;  // bit words per unit
  constexpr int kS3WPL = (kS3Words + 31) / 32;  // words per lane of one warp (zero padded)
  __shared__ double qd[G][D];
  __shared__ double s_qn[G], s_gen[G];
  __shared__ uint32_t hist[kHistBins + kHistBins / 32];
  __shared__ float s_mn[NW], s_mx[NW];
  __shared__ int s_win[NW];
  __shared__ uint32_t inbits[32 * kS3WPL], uncbits[32 * kS3WPL];
  __shared__ uint64_t ukey[kSmallUncertain];
  __shared__ int32_t ulist[kSmallUncertain], ulen[kSmallUncertain], utake[kSmallUncertain];
  __shared__ int s_nunc, s_base;
  __shared__ int32_t wlist[kSmallUncertain];  // warp 0: the whole chunks' ids

  const int u = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_trigger();  // the attention kernel may launch once every select CTA is resident
  for (int w = kS3Words + tid; w < 32 * kS3WPL; w += NT) inbits[w] = uncbits[w] = 0u;  // padding
  unsigned char* scratch = a.gscratch + (int64_t)u * a.gscratch_stride;
  uint64_t* key64 = reinterpret_cast<uint64_t*>(scratch);
  int32_t* lens = reinterpret_cast<int32_t*>(key64 + a.n_max);
  int32_t* glist = lens + a.n_max;

  DBG_T(0);
  // per-unit constants first: their loads overlap the prologue and the wait
  const int nc_u = a.lay.num_chunks(u), P_u = a.lay.prompt_len(u);
  const int kexp = (int)a.sinfo[4 * u + 0];
  const double cmax = a.sinfo[4 * u + 1], dmax = a.sinfo[4 * u + 2];
  int g, gl;
  select_prologue<D, G, NT>(a, u, qd, s_qn, s_gen, g, gl);
  DBG_T(1);

  const UnitChunks uc{a.lay, u, nc_u, gl, P_u};
  const int n = uc.nc + (gl >= 1 ? 1 : 0);
  const int wloc = uc.P + gl;  // tokens the walk ranges over (self excluded)
  // the newest token's row: global in split-KV candidate mode (the budget is
  // the unsharded row's; the local walk keeps every chunk that can take)
  const int row = a.split ? a.total_prompt + g : uc.P + g;
  const int64_t keep = a.budget < (int64_t)row + 1 ? a.budget : (int64_t)row + 1;
  const uint32_t R = (uint32_t)(keep - 1);
  // sketch units per score unit: 2^-kexp (exact bit construction in the normal range)
  const double scale = (kexp > -1023 && kexp < 1023)
                           ? __longlong_as_double((long long)(1023 - kexp) << 52)
                           : ldexp(1.0, -kexp);
  constexpr double gam = 6.103515625e-05 + 1e-6;  // see sketch_select_kernel

  const int nitems = AGG == DHSA_AGG_NONE ? G : 1;
  // (experiment) a.reps > 1 repeats the selection; the phase stamps are the last pass
  for (int rep = 0; rep < a.reps; ++rep)
  for (int it = 0; it < nitems; ++it) {
    const int s = AGG == DHSA_AGG_NONE ? u * G + it : u;
    const int h0 = AGG == DHSA_AGG_NONE ? it : 0, nh = AGG == DHSA_AGG_NONE ? 1 : G;
    const float* __restrict__ apx = a.approx + (int64_t)s * a.sc_stride;
    int32_t* out = a.tiles + (int64_t)s * a.tile_cap * 2;
    double qmax = 0.0;
    for (int h = h0; h < h0 + nh; ++h) qmax = fmax(qmax, s_qn[h]);
    const double gex = agg_d<G, AGG>(s_gen + h0, nh);  // exact, score units
    // ---- owned chunks c_e = tid + e*NT: approximate score and length ----
    float v[kS3Per];
    int ln[kS3Per];
#pragma unroll
    for (int e = 0; e < kS3Per; ++e) {
      const int c = tid + e * NT;
      v[e] = c < uc.nc ? __ldcg(apx + c) : (float)(gex * scale);  // gen chunk: exact score
      ln[e] = 0;
      if (c < n) {
        int lo;
        uc.chunk(c, lo, ln[e]);
      }
    }
    for (int b = tid; b < kHistBins + kHistBins / 32; b += NT) hist[b] = 0;
    uint32_t inm = 0, unm = 0;  // bit e: chunk c_e certainly whole / uncertain
    if (R > 0 && R < (uint32_t)wloc) {
      DBG_T(2);
      float mn = INFINITY, mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < kS3Per; ++e)
        if (ln[e] > 0) {
          mn = fminf(mn, v[e]);
          mx = fmaxf(mx, v[e]);
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if (lane == 0) {
        s_mn[warp] = mn;
        s_mx[warp] = mx;
      }
      __syncthreads();  // also orders the histogram reset
      mn = lane < NW ? s_mn[lane] : INFINITY;
      mx = lane < NW ? s_mx[lane] : -INFINITY;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      const float bscale = mx > mn ? ((float)kHistBins - 0.5f) / (mx - mn) : 0.f;
      const float off = -mn * bscale;
#pragma unroll
      for (int e = 0; e < kS3Per; ++e)
        if (ln[e] > 0) atomicAdd(&hist[hist_pad(bin32(v[e], bscale, off))], (uint32_t)ln[e]);
      __syncthreads();
      // cut bin b*: W(bin > b*) < R <= W(bin >= b*); every warp scans the
      // histogram (lane l: bins 1023-32l down to 992-32l), no barrier
      int bstar;
      {
        uint32_t sum = 0;
#pragma unroll 8
        for (int j = 0; j < 32; ++j) sum += hist[hist_pad(kHistBins - 1 - 32 * lane - j)];
        const uint32_t incl = (uint32_t)warp_incl_scan((int)sum, lane);
        const unsigned hit = __ballot_sync(0xffffffffu, incl - sum < R && R <= incl);
        const int f = __ffs(hit) - 1;
        // inside group f: lane j takes bin 1023-32f-j, a second scan finds the bin
        const int ff = f < 0 ? 0 : f;
        const uint32_t before = __shfl_sync(0xffffffffu, incl - sum, ff);
        const int myb = kHistBins - 1 - 32 * ff - lane;
        const uint32_t cum = before + (uint32_t)warp_incl_scan((int)hist[hist_pad(myb)], lane);
        const unsigned hit2 = __ballot_sync(0xffffffffu, cum >= R);
        bstar = hit2 ? kHistBins - 1 - 32 * ff - (__ffs(hit2) - 1) : 0;
      }
      DBG_T(3);
      // certified classification (sketch units; directed rounding keeps the
      // fp32 bins valid bounds: DESIGN.md section 4)
      const double E = 1.01 * (qmax * dmax + gam * qmax * cmax) + fabs(gex * scale) * 1.2e-7 +
                       1e-300;
      const float twoE = __double2float_ru(2.0 * E);
      int my_win = 0;
#pragma unroll
      for (int e = 0; e < kS3Per; ++e)
        if (ln[e] > 0) {
          if (bscale > 0.f && bin32(__fsub_rd(v[e], twoE), bscale, off) > bstar) {
            inm |= 1u << e;  // every chunk ranked at or above it is in bins > b*: whole
            my_win += ln[e];
          } else if (bscale == 0.f || bin32(__fadd_ru(v[e], twoE), bscale, off) >= bstar) {
            unm |= 1u << e;  // not ordered against the cut by the sketch: exact score
          }  // else: every chunk of the bins >= b* ranks above it: nothing
        }
      my_win = warp_sum(my_win);
      if (lane == 0) s_win[warp] = my_win;
    } else if (R > 0) {  // every causal token is kept: all chunks whole
#pragma unroll
      for (int e = 0; e < kS3Per; ++e)
        if (ln[e] > 0) inm |= 1u << e;
      if (lane == 0) s_win[warp] = 0;
    } else if (lane == 0) {
      s_win[warp] = 0;
    }
#pragma unroll
    for (int e = 0; e < kS3Per; ++e) {  // chunk c_e = bit `lane` of word e*NW + warp
      const uint32_t wi = __ballot_sync(0xffffffffu, inm & (1u << e));
      const uint32_t wu = __ballot_sync(0xffffffffu, unm & (1u << e));
      if (lane == 0) {
        inbits[e * NW + warp] = wi;
        uncbits[e * NW + warp] = wu;
      }
    }
    __syncthreads();
    DBG_T(9);
    if (warp == 0 && a.split) {
      if (lane == 0) s_base = 0;
    } else if (warp == 0) {
      // ---- the chunks kept whole: tiles in chunk order, published early ----
      const int base = s3_emit_whole<kS3WPL>(uc, inbits, a.tile_tokens, out, a.tile_cap, 0,
                                             wlist, kSmallUncertain,
#ifdef DHSA_SELECT_STAMPS
                                     a.dbg ? a.dbg + kDbgSelectClk + blockIdx.x * 16 : nullptr
#else
                                     nullptr
#endif
      );
      __syncwarp();  // the warp's tile stores, before lane 0's (cumulative) release
      if (lane == 0) {
        s_base = base;
        if (a.early && base > 0 && base + 1 <= a.tile_cap) {
          if (a.relaxed) st_relaxed(a.ready + s, 1 + base);
          else st_release(a.ready + s, 1 + base);
        }
      }
      DBG_T(10);
    } else {
      // ---- uncertain chunks in chunk order (warp 1), fp64 re-scoring (warps 1..31) ----
      if (warp == 1) {
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < kS3WPL; ++j) cnt += __popc(uncbits[kS3WPL * lane + j]);
        const int incl = warp_incl_scan(cnt, lane);
        int pos = incl - cnt;
#pragma unroll
        for (int j = 0; j < kS3WPL; ++j) {
          uint32_t m = uncbits[kS3WPL * lane + j];
          while (m) {
            const int c = 32 * (kS3WPL * lane + j) + __ffs(m) - 1;
            m &= m - 1;
            glist[pos] = c;
            if (pos < kSmallUncertain) {
              int lo, len;
              uc.chunk(c, lo, len);
              ulist[pos] = c;
              ulen[pos] = len;
            }
            ++pos;
          }
        }
        if (lane == 31) s_nunc = incl;
      }
      named_bar(1, NT - 32);
      const int nu = s_nunc;
      for (int i = warp - 1; i < nu; i += NW - 1) {
        const int c = i < kSmallUncertain ? ulist[i] : __ldcg(glist + i);
        double ex;
        if (c < uc.nc) {
          const double* crow = a.cent + (int64_t)u * a.c_stride + (int64_t)c * D;
          double part[G];
#pragma unroll
          for (int h = 0; h < G; ++h) part[h] = 0.0;
#pragma unroll
          for (int d = lane; d < D; d += 32) {
            const double cv = __ldcg(crow + d);
#pragma unroll
            for (int h = 0; h < G; ++h) part[h] = fma(qd[h][d], cv, part[h]);
          }
#pragma unroll
          for (int h = 0; h < G; ++h) part[h] = warp_sum(part[h]);
          ex = agg_d<G, AGG>(part + h0, nh);
        } else {
          ex = gex;
        }
        if (lane == 0) {
          if (nu <= kSmallUncertain) ukey[i] = order_key(ex);
          else key64[c] = order_key(ex);
        }
      }
    }
    __syncthreads();
    DBG_T(5);
    const int nu = s_nunc;
    const int base = s_base;
    if (a.dbg && tid == 0) a.dbg[blockIdx.x * 16 + 15] = nu;
    if (a.split) {
      // split-KV candidates: every chunk with a positive local take, with its
      // exact fp64 score (emit_candidates), from the takes of every chunk in
      // global scratch: whole chunks their length, uncertain ones the exact
      // walk's take (sketch_common.cuh; the generic select's semantics)
      if (nu > kSmallUncertain) {
        s3_fallback<NT>(uc, n, R, row, 0, inbits, uncbits, key64, lens, a.tile_tokens, out,
                        a.tile_cap, a.ntiles + s, 0);
      } else {
#pragma unroll
        for (int e = 0; e < kS3Per; ++e) {
          const int c = tid + e * NT;
          if (c < n) lens[c] = (inm & (1u << e)) ? ln[e] : 0;
        }
        const int win = warp_sum(lane < NW ? s_win[lane] : 0);
        const int rp = (int)R - win;
        for (int i = tid; i < nu; i += NT) {  // rank among the uncertain chunks
          const uint64_t ki = ukey[i];
          int before = 0;
          for (int j = 0; j < nu; ++j) {
            const uint64_t kj = ukey[j];
            if (kj > ki || (kj == ki && j < i)) before += ulen[j];  // list = chunk order
          }
          const int rem = rp - before;
          utake[i] = rem <= 0 ? 0 : (rem < ulen[i] ? rem : ulen[i]);
        }
        __syncthreads();
        for (int i = tid; i < nu; i += NT) lens[ulist[i]] = utake[i];
        __syncthreads();
      }
      emit_candidates<D, G, AGG, NT>(a, uc, lens, glist, n, s, qd, h0, nh, gex, u);
    } else if (nu > kSmallUncertain) {
      s3_fallback<NT>(uc, n, R, row, base, inbits, uncbits, key64, lens, a.tile_tokens, out,
                  a.tile_cap, a.ntiles + s, 1);
    } else {
      const int win = warp_sum(lane < NW ? s_win[lane] : 0);
      const int rp = (int)R - win;
      if (nu > 32) {  // takes by every thread (rank among the uncertain chunks)
        for (int i = tid; i < nu; i += NT) {
          const uint64_t ki = ukey[i];
          int before = 0;
          for (int j = 0; j < nu; ++j) {
            const uint64_t kj = ukey[j];
            if (kj > ki || (kj == ki && j < i)) before += ulen[j];  // list = chunk order
          }
          const int rem = rp - before;
          utake[i] = rem <= 0 ? 0 : (rem < ulen[i] ? rem : ulen[i]);
        }
        __syncthreads();
      }
      if (warp == 0) {
        int off = base;
        for (int i0 = 0; i0 < nu; i0 += 32) {
          const int i = i0 + lane;
          int take = 0;
          if (nu <= 32) {  // exact walk in registers: rank by (key desc, chunk asc)
            const uint64_t ki = i < nu ? ukey[i] : 0ull;
            const int li = i < nu ? ulen[i] : 0;
            int before = 0;
            for (int j = 0; j < nu; ++j) {
              const uint64_t kj = __shfl_sync(0xffffffffu, ki, j);
              const int lj = __shfl_sync(0xffffffffu, li, j);
              if (kj > ki || (kj == ki && j < i)) before += lj;
            }
            const int rem = rp - before;
            take = i < nu ? (rem <= 0 ? 0 : (rem < li ? rem : li)) : 0;
          } else if (i < nu) {
            take = utake[i];
          }
          const int cnt = take > 0 ? ntiles_of(take, a.tile_tokens) : 0;
          const int incl = warp_incl_scan(cnt, lane);
          int o = off + incl - cnt;
          if (take > 0) {
            int lo, len;
            uc.chunk(ulist[i], lo, len);
            for (int t = 0; t < take; t += a.tile_tokens, ++o)
              if (o < a.tile_cap) {
                out[2 * o] = lo + t;
                out[2 * o + 1] = min(a.tile_tokens, take - t);
              }
          }
          off += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
          if (off + 1 > a.tile_cap) {
            a.ntiles[s] = -1;  // capacity error, reported by the host wrapper
          } else {
            out[2 * off] = row;  // self (masks.py:120-121)
            out[2 * off + 1] = 1;
            a.ntiles[s] = off + 1;
          }
        }
      }
    }
    __syncwarp();
    DBG_T(7);
    if (tid == 0) {
      if (it == nitems - 1 && a.advance) a.gen_count[u] = g + 1;  // masks.py:236
      if (a.ready) {  // this item's tiles, sum and k/v
        if (a.relaxed) st_relaxed(a.ready + s, kReadyFinal);
        else st_release(a.ready + s, kReadyFinal);
      }
    }
    __syncthreads();
  }
  DBG_T(8);
}

// Launch the compact select when it applies (units of <= kS3MaxChunks chunks,
// not split-KV candidate mode, global scratch present); returns 1 if launched
// (status in *rc), 0 otherwise.
template <int D, int G, int AGG>
int launch_select2(const SketchArgs& a, int U, cudaStream_t s, int* rc);

}  // namespace dhsa
