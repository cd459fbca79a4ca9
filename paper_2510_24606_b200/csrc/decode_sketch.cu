// bf16 decode fast path: fp16 centroid SKETCH stream + certified exact selection.
//
// Reference semantics (unchanged): masks._decode_row (masks.py:153-173) scores
// the raw query against the fp64 prompt centroids, the generated-chunk
// centroid gen_sum/sqrt(g) and the singleton, and topk_row (masks.py:103-122)
// selects.  The selected indices must be those of an fp64 evaluation.
//
// Why a sketch: at 128K context the fp64 centroid stream (D*8 B per chunk and
// kv head) is half of a decode step's HBM bytes.  Streaming a 2-byte copy cuts
// it 4x; exactness is restored by re-scoring, in fp64, only the chunks whose
// approximate score cannot be ordered against the selection cut.
//
// Sketch (built once per prompt, dhsa_sketch_build): per unit u a power-of-two
// scale 2^-k_u puts max|c| in [2^13, 2^14); c''_j = RN_fp16(c_j 2^-k_u).  The
// build measures, in fp64, dmax_u = max_j ||c''_j - c_j 2^-k_u||_2 and
// cmax_u = max_j ||c''_j||_2.  For a query q (bf16; bf16*fp16 products are
// exact in fp32) the fp32 sketch score s''_j obeys
//   |s''_j - s_j 2^-k_u| <= ||q|| dmax_u + gamma_D ||q|| cmax_u =: E,
// gamma_D = D 2^-24 / (1 - D 2^-24) (Cauchy-Schwarz on the measured rounding
// error + fp32 summation), with a small safety factor.
//
// Certified walk (per selection row, R = min(budget,row+1)-1 tokens):
// let t'' be the weighted threshold of the approximate order, W(s'' > t'') <
// R <= W(s'' >= t'').  A chunk with s''_j > t'' + 2E is wholly inside the exact
// selection (every chunk that can rank above it has s'' > t''); a chunk with
// s''_j < t'' - 2E receives nothing (every chunk with s'' >= t'' ranks above
// it and those already weigh >= R); the rest are re-scored in fp64 and walked
// exactly (score desc, chunk asc) with the budget left by the certain ones.
// DESIGN.md section 4 has the full argument; tests compare against fp64
// scoring on tie-heavy, integer, outlier and zero-query inputs.
//
// Kernels per step: sketch_score_kernel (persistent, TMA bulk ring of 16 KB
// chunk slices, 8 consumer warps + 1 producer warp) -> sketch_select_kernel
// (one CTA per kv unit: generated chunk in fp64 + state update, certified
// walk, tiles for the attention kernel, gen_count += 1).
#include "select2.cuh"
#include "sketch_common.cuh"

#include <cstdlib>

namespace dhsa {

constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x / 2); }

// 2^k as a float for a normal-range exponent, else 0 (the caller falls back
// to ldexpf); x * 2^k is then exact unless it under/overflows, exactly as
// ldexpf(x, k) would round
__device__ __forceinline__ float pow2f(int k) {
  return (k > -127 && k < 128) ? __int_as_float((127 + k) << 23) : 0.f;
}
__device__ __forceinline__ float scale2(float x, int k, float p) {
  return p != 0.f ? x * p : ldexpf(x, k);
}

template <int NV, int LG>
__device__ __forceinline__ void transpose_reduce_f(float (&v)[NV], int lane) {
  int n = NV;
#pragma unroll
  for (int o = LG / 2; o >= 1; o >>= 1) {
    if (n > 1) {
      const int half = n >> 1;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int k = 0; k < NV / 2; ++k) {
        if (k < half) {
          const float send = up ? v[k] : v[k + half];
          const float keep = up ? v[k + half] : v[k];
          v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      n = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
}

// value index held in v[k] after transpose_reduce_f<NV, LG> (lane within group)
template <int NV, int LG>
__device__ __forceinline__ int tr_index(int k, int glane) {
  constexpr int a = ilog2c(NV), b = ilog2c(LG), m = a < b ? a : b;
  int idx = k;
#pragma unroll
  for (int s = 0; s < m; ++s) idx |= ((glane >> (b - 1 - s)) & 1) << (a - 1 - s);
  return idx;
}

// ------------------------------------------------------------ score stream --
// Tensor-core sketch scores: S^T[chunk][head] = C''[chunk][:] . q'[head][:]
// with mma.sync m16n8k16 (fp16 in, fp32 accumulate).  A = 16 sketch rows from
// a 128B-swizzled TMA tile (ldmatrix, conflict free), B = the G query heads of
// the kv group (N = 8 columns, heads >= G zero) held in registers for the
// whole unit, each head scaled by a power of two 2^-kq so bf16 q is exact in
// fp16.  4 consumer warps x 16 rows per 64-chunk slice; one producer thread
// keeps kStages slices in flight with 2-D TMA loads.
template <int D, int G, int AGG>
__global__ __launch_bounds__(kTcThreads) void sketch_score_kernel(
    const __grid_constant__ CUtensorMap tmS, SketchArgs a) {
  constexpr int NB = D / 64;       // 128-byte column boxes per row
  constexpr int BOX = 64 * 128;    // 64 rows x 128 B
  constexpr int TILE = NB * BOX;
  constexpr int STAGE = TILE;
  constexpr int KS = D / 16;
  static_assert(G <= 8, "N = 8 columns");
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[kTcStages], empty_bar[kTcStages];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows_per_unit = (int)(a.sk_stride / D);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kTcConsumers);
    }
    fence_barrier_init();
  }
  if (a.ready) {
    // re-arm the select -> attention flags of this step before any select CTA
    // can launch (the previous step's attention has completed: this kernel is
    // not launched programmatically)
    const int items = AGG == DHSA_AGG_NONE ? a.n_units * G : a.n_units;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < items; i += gridDim.x * blockDim.x)
      a.ready[i] = 0;
    if ((int64_t)blockIdx.x * blockDim.x < items) __threadfence();  // only the CTAs that wrote
  }
  __syncthreads();
  if (a.dbg && threadIdx.x == 0) a.dbg[kDbgSketch + 2 * blockIdx.x] = gtimer();
  pdl_trigger();  // the select kernel may launch (and run its prologue) right away
  // The slices are streamed in `waves` consecutive parts of the unit range;
  // in each wave every CTA takes a contiguous slice range, (unit, first
  // chunk) advanced incrementally.  With 2 waves the first half of the units
  // is complete at half the stream: their selects run while the stream
  // finishes the second half (one select CTA fits next to the stream CTAs),
  // and the attention starts on finished items as soon as the stream's CTAs
  // leave the SMs.
  const int spu = a.slices_per_unit;
  const int nwaves = a.waves > 1 ? a.waves : 1;
  int64_t s_begin = 0, s_end = 0;
  int u = 0, c0 = 0, nc = 0;
  auto wave_range = [&](int w) {
    const int64_t w0 = w == 0 ? 0 : a.total_slices * a.wave_end[w - 1] / 1000;
    const int64_t w1 = w == nwaves - 1 ? a.total_slices : a.total_slices * a.wave_end[w] / 1000;
    s_begin = w0 + (w1 - w0) * blockIdx.x / gridDim.x;
    s_end = w0 + (w1 - w0) * (blockIdx.x + 1) / gridDim.x;
    u = (int)(s_begin / spu);
    c0 = (int)(s_begin - (int64_t)u * spu) * kSliceRows;
    nc = s_begin < s_end ? a.lay.num_chunks(u) : 0;
  };

  if (warp == kTcConsumers) {
    if (lane == 0) {
      prefetch_tmap(&tmS);
      uint64_t pol = 0;  // the sketch is read once per step: evict-first
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
      if (a.l2_hint) pol = l2_policy_evict_first();
      int it = 0;
      for (int w = 0; w < nwaves; ++w) {
      wave_range(w);
      for (int64_t sl = s_begin; sl < s_end; ++sl) {
        if (c0 < nc) {
          const int st = it % kTcStages;
          if (it >= kTcStages) mbar_wait(&empty_bar[st], ((it / kTcStages) + 1) & 1);
          mbar_expect_tx(&full_bar[st], TILE);
          const int row = u * rows_per_unit + c0;
#pragma unroll
          for (int b = 0; b < NB; ++b)
            tma_load_2d_hint(smem + st * STAGE + b * BOX, &tmS, &full_bar[st], b * 64, row, pol);
          ++it;
        }
        c0 += kSliceRows;
        if (c0 >= spu * kSliceRows) {
          c0 = 0;
          ++u;
          if (sl + 1 < s_end) nc = a.lay.num_chunks(u);
        }
      }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  // progress: one release per (warp, unit) run of slices, not per slice (a
  // fence per slice measurably slows the stream)
  int pend_u = -1, pend_n = 0;
  auto publish = [&](int pu, int pn) {
    if (!a.progress || pu < 0 || pn == 0) return;
    __syncwarp();
    // release-add: the warp's score stores (ordered by the __syncwarp) are
    // visible before the count the select acquires
    if (lane == 0) red_add_release(a.progress + pu, pn);
  };
  const int hcol = lane >> 2;  // B column (head) owned for the fragment
  uint32_t qb[KS][2];
  int kq0 = 0, kq1 = 0;        // scale exponents of the two heads in this lane's C columns
  float p0 = 1.f, p1 = 1.f;     // 2^kq0, 2^kq1 (0 when out of the normal range: ldexpf)
  int cur_u = -1;
  const int mi = lane >> 3, r8 = lane & 7;
  const int arow = warp * 16 + (mi & 1) * 8 + r8;  // A row addressed by this lane
  int it = 0;
  for (int w = 0; w < nwaves; ++w) {
  wave_range(w);
  for (int64_t sl = s_begin; sl < s_end; ++sl, c0 += kSliceRows) {
    if (c0 >= spu * kSliceRows) {
      c0 = 0;
      ++u;
      nc = a.lay.num_chunks(u);
    }
    if (c0 >= nc) continue;
    if (u != cur_u) {
      publish(pend_u, pend_n);
      pend_u = u;
      pend_n = 0;
      cur_u = u;
      // B fragments of q'^T: head hcol, dims 16ks + 2(lane&3) + {0,1} (+8)
      float qv[KS][4];
      float amax = 0.f;
      const __nv_bfloat16* qrow = a.q + (int64_t)(u * G + (hcol < G ? hcol : 0)) * D;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int d = 16 * ks + 2 * (lane & 3) + 8 * e;
          float2 f = make_float2(0.f, 0.f);
          if (hcol < G) f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(qrow + d));
          qv[ks][2 * e] = f.x;
          qv[ks][2 * e + 1] = f.y;
          amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
        }
      }
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
      const int kq = amax > 0.f ? ilogbf(amax) + 1 - 14 : 0;  // max|q| 2^-kq < 2^14
      // 2^-kq: an exact power-of-two multiply (ldexpf only outside the normal range)
      const float qs = (kq > -127 && kq < 127) ? __int_as_float((127 - kq) << 23) : ldexpf(1.f, -kq);
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const __half2 lo = __floats2half2_rn(qv[ks][0] * qs, qv[ks][1] * qs);
        const __half2 hi = __floats2half2_rn(qv[ks][2] * qs, qv[ks][3] * qs);
        qb[ks][0] = *reinterpret_cast<const uint32_t*>(&lo);
        qb[ks][1] = *reinterpret_cast<const uint32_t*>(&hi);
      }
      // C columns of this lane are heads 2(lane&3), 2(lane&3)+1: fetch their exponents
      kq0 = __shfl_sync(0xffffffffu, kq, 4 * (2 * (lane & 3)));
      kq1 = __shfl_sync(0xffffffffu, kq, 4 * (2 * (lane & 3) + 1));
      p0 = pow2f(kq0);
      p1 = pow2f(kq1);
    }
    const int st = it % kTcStages;
    if (a.dbg && threadIdx.x == 0 && it == 0) a.dbg[kDbgSketchPh + 4 * blockIdx.x] = gtimer();
    mbar_wait(&full_bar[st], (it / kTcStages) & 1);
    if (a.dbg && threadIdx.x == 0 && it == 0) a.dbg[kDbgSketchPh + 4 * blockIdx.x + 1] = gtimer();
    const uint32_t base = smem_u32(smem + st * STAGE);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int kch = 2 * ks + (mi >> 1);
      const uint32_t addr = base + (kch >> 3) * BOX + arow * 128 + (((kch & 7) ^ (arow & 7)) << 4);
      uint32_t a0, a1, a2, a3;
      ldsm_x4(addr, a0, a1, a2, a3);
      mma_f16(acc, a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[st]);
    ++it;
    // acc[0..1]: row warp*16 + lane/4, heads 2(lane&3)+{0,1}; acc[2..3]: row + 8
    const int h0 = 2 * (lane & 3);
    float v[4];
    v[0] = h0 < G ? scale2(acc[0], kq0, p0) : -INFINITY;
    v[1] = h0 + 1 < G ? scale2(acc[1], kq1, p1) : -INFINITY;
    v[2] = h0 < G ? scale2(acc[2], kq0, p0) : -INFINITY;
    v[3] = h0 + 1 < G ? scale2(acc[3], kq1, p1) : -INFINITY;
    const int r0 = warp * 16 + (lane >> 2);
    if constexpr (AGG == DHSA_AGG_NONE) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int h = h0 + (e & 1), r = r0 + 8 * (e >> 1);
        if (h < G && c0 + r < nc) a.approx[(int64_t)(u * G + h) * a.sc_stride + c0 + r] = v[e];
      }
    } else {
      float x = (AGG == DHSA_AGG_MAX) ? fmaxf(v[0], v[1]) : (h0 < G ? v[0] : 0.f) + (h0 + 1 < G ? v[1] : 0.f);
      float y = (AGG == DHSA_AGG_MAX) ? fmaxf(v[2], v[3]) : (h0 < G ? v[2] : 0.f) + (h0 + 1 < G ? v[3] : 0.f);
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        const float xo = __shfl_xor_sync(0xffffffffu, x, o);
        const float yo = __shfl_xor_sync(0xffffffffu, y, o);
        x = (AGG == DHSA_AGG_MAX) ? fmaxf(x, xo) : x + xo;
        y = (AGG == DHSA_AGG_MAX) ? fmaxf(y, yo) : y + yo;
      }
      if ((lane & 3) == 0) {
        if (AGG == DHSA_AGG_MEAN) {
          x = x / (float)G;
          y = y / (float)G;
        }
        if (c0 + r0 < nc) a.approx[(int64_t)u * a.sc_stride + c0 + r0] = x;
        if (c0 + r0 + 8 < nc) a.approx[(int64_t)u * a.sc_stride + c0 + r0 + 8] = y;
      }
    }
    ++pend_n;  // slices of unit pend_u this warp has scored, published per unit
  }
  }
  if (a.dbg && threadIdx.x == 0) a.dbg[kDbgSketchPh + 4 * blockIdx.x + 2] = gtimer();
  publish(pend_u, pend_n);
  if (a.dbg && threadIdx.x == 0) a.dbg[kDbgSketch + 2 * blockIdx.x + 1] = gtimer();
}

// Weighted cut of the approximate scores by a value histogram: one min/max
// reduction, one histogram pass (atomics spread over kHistBins bins), and a
// redundant per-warp suffix scan (no barrier).  Returns b* with
// W(bin > b*) < R <= W(bin >= b*) for bin(x) = clamp(floor((x - vmin) *
// bscale), 0, kHistBins - 1), which is monotone in x.  Requires 0 < R <
// total weight.  Replaces a 4-pass 8-bit radix select (~7 us -> ~2 us).
__device__ __forceinline__ int hpad(int b) { return b + (b >> 5); }  // bank-conflict-free scan
template <int NT>
struct HistShared {
  uint32_t hist[kHistBins + kHistBins / 32];
  float wmin[NT / 32], wmax[NT / 32];
};

template <int NT>
__device__ int hist_threshold(const uint32_t* ak, const int32_t* lens, int n, uint32_t R,
                              HistShared<NT>& hs, double& vmin, double& bscale) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = tid; b < kHistBins + kHistBins / 32; b += NT) hs.hist[b] = 0;
  float mn = INFINITY, mx = -INFINITY;
  for (int c = tid; c < n; c += NT)
    if (lens[c] > 0) {
      const float v = key32_value(ak[c]);
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    hs.wmin[warp] = mn;
    hs.wmax[warp] = mx;
  }
  __syncthreads();
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    mn = fminf(mn, hs.wmin[w]);
    mx = fmaxf(mx, hs.wmax[w]);
  }
  vmin = (double)mn;
  bscale = mx > mn ? ((double)kHistBins - 0.5) / ((double)mx - (double)mn) : 0.0;
  for (int c = tid; c < n; c += NT) {
    const int len = lens[c];
    if (len > 0) {
      const double f = floor(((double)key32_value(ak[c]) - vmin) * bscale);
      const int b = f < 0.0 ? 0 : (f > (double)(kHistBins - 1) ? kHistBins - 1 : (int)f);
      atomicAdd(&hs.hist[hpad(b)], (uint32_t)len);
    }
  }
  __syncthreads();
  // every warp: lane l holds bins kHistBins-1-32l .. kHistBins-32(l+1) (descending)
  constexpr int PER = kHistBins / 32;
  uint32_t sum = 0;
#pragma unroll 8
  for (int j = 0; j < PER; ++j) sum += hs.hist[hpad(kHistBins - 1 - PER * lane - j)];
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const unsigned hit = __ballot_sync(0xffffffffu, incl - sum < R && R <= incl);
  const int f = __ffs(hit) - 1;
  int bstar = 0;
  if (lane == f) {
    uint32_t cum = incl - sum;
    for (int j = 0; j < PER; ++j) {
      const int b = kHistBins - 1 - PER * lane - j;
      cum += hs.hist[hpad(b)];
      if (cum >= R) {
        bstar = b;
        break;
      }
    }
  }
  return __shfl_sync(0xffffffffu, bstar, f < 0 ? 0 : f);
}

template <int D, int G, int AGG, int NT>
__global__ __launch_bounds__(NT) void sketch_select_kernel(SketchArgs a) {
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ WalkShared sh;
  __shared__ double qd[G][D];
  __shared__ double s_qn[G], s_gen[G];
  __shared__ int s_nunc, s_win;
  __shared__ HistShared<NT> hs;

  const int u = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned char* scratch = a.smem_select ? smem_raw : a.gscratch + (int64_t)u * a.gscratch_stride;
  uint64_t* key64 = reinterpret_cast<uint64_t*>(scratch);
  int32_t* lens = reinterpret_cast<int32_t*>(key64 + a.n_max);
  uint32_t* ak = reinterpret_cast<uint32_t*>(lens + a.n_max);
  int32_t* unc = reinterpret_cast<int32_t*>(ak + a.n_max);

  pdl_trigger();  // the attention kernel may launch once every select CTA is resident
  DBG_T(0);
  int g, gl;
  select_prologue<D, G, NT>(a, u, qd, s_qn, s_gen, g, gl);
  DBG_T(1);

  UnitChunks uc{a.lay, u, a.lay.num_chunks(u), gl, a.lay.prompt_len(u)};
  const int n = uc.nc + (gl >= 1 ? 1 : 0);
  const int wloc = uc.P + gl;  // tokens the walk ranges over (self excluded)
  const int row = a.split ? a.total_prompt + g : uc.P + g;  // global row of the newest token
  const int64_t keep = a.budget < (int64_t)row + 1 ? a.budget : (int64_t)row + 1;
  const uint32_t R = (uint32_t)(keep - 1);
  const float kexp = a.sinfo[4 * u + 0];
  const double scale = ldexp(1.0, -(int)kexp);  // sketch units per score unit
  const double cmax = a.sinfo[4 * u + 1], dmax = a.sinfo[4 * u + 2];
  // accumulation: mma.sync fp32 accumulation of D exact fp16 products (bounded
  // conservatively by 2^-14 sum|p|, ~4x the published truncating-alignment
  // model of 8 x 17 x 2^-23) + the head mean + q fp16 subnormal rounding
  constexpr double gam = 6.103515625e-05 + 1e-6;

  const int nitems = AGG == DHSA_AGG_NONE ? G : 1;
  for (int it = 0; it < nitems; ++it) {
    const int s = AGG == DHSA_AGG_NONE ? u * G + it : u;
    const int h0 = AGG == DHSA_AGG_NONE ? it : 0, nh = AGG == DHSA_AGG_NONE ? 1 : G;
    double qmax = 0.0;
    for (int h = h0; h < h0 + nh; ++h) qmax = fmax(qmax, s_qn[h]);
    const double gex = agg_d<G, AGG>(s_gen + h0, nh);  // exact, score units
    const float* __restrict__ apx = a.approx + (int64_t)s * a.sc_stride;
    {
      // batched: the approximate scores (L2) are loaded before any smem store
      constexpr int UNR = 4;
      const float gkey = (float)(gex * scale);
      for (int c0 = tid; c0 < n; c0 += UNR * NT) {
        float v[UNR];
        int ln[UNR];
#pragma unroll
        for (int k = 0; k < UNR; ++k) {
          const int c = c0 + k * NT;
          v[k] = (c < uc.nc) ? __ldcg(apx + c) : gkey;
          int lo;
          if (c < n) uc.chunk(c, lo, ln[k]);
        }
#pragma unroll
        for (int k = 0; k < UNR; ++k) {
          const int c = c0 + k * NT;
          if (c < n) {
            lens[c] = ln[k];
            ak[c] = order_key32(v[k]);
          }
        }
      }
    }
    if (tid == 0) {
      s_nunc = 0;
      s_win = 0;
    }
    __syncthreads();
    uint64_t prefix = 0, mask = 0;
    uint32_t rrem = R;
    bool done = false;
    int base = 0;  // tiles published early (phase A)
    if (R > 0 && R < (uint32_t)wloc) {
      DBG_T(2);
      // certified bound in sketch units (+ the fp32 rounding of the exact gen score)
      const double E = 1.01 * (qmax * dmax + gam * qmax * cmax) +
                       fabs(gex * scale) * 1.2e-7 + 1e-300;
      // cut bin b* of a weighted value histogram of the approximate scores:
      // W(bin > b*) < R <= W(bin >= b*) brackets the weighted R-th score
      double vmin, bscale;
      const int bstar = hist_threshold(ak, lens, n, R, hs, vmin, bscale);
      DBG_T(3);
      auto bin = [&](double x) {
        const double f = floor((x - vmin) * bscale);
        return f < 0.0 ? 0 : (f > (double)(kHistBins - 1) ? kHistBins - 1 : (int)f);
      };
      int win_local = 0;
      for (int c = tid; c < n; c += NT) {
        const double v = (double)key32_value(ak[c]);
        uint64_t k;
        // bin() is monotone: bin(v - 2E) > b* => v - 2E exceeds every score of
        // the bins <= b*, whose weight reaches R (certainly kept whole);
        // bin(v + 2E) < b* => v + 2E is below every score of the bins >= b*,
        // which weigh >= R and rank above (certainly outside)
        if (bin(v - 2.0 * E) > bstar) {
          k = ~0ull;  // certainly kept whole
          win_local += lens[c];
        } else if (bin(v + 2.0 * E) < bstar) {
          k = 0ull;  // certainly outside
        } else {
          k = 1ull;  // uncertain: exact fp64 score below
          if (lens[c] > 0) unc[atomicAdd(&s_nunc, 1)] = c;
        }
        key64[c] = k;
      }
      win_local = warp_sum(win_local);
      if (lane == 0 && win_local) atomicAdd(&s_win, win_local);
      __syncthreads();
      const int nu = s_nunc;
      if (a.early) {
        // phase A: the chunks kept whole are final already; their tiles go out
        // (chunk order) and the attention may stream them while the
        // uncertain chunks are re-scored
        int32_t* out = a.tiles + (int64_t)s * a.tile_cap * 2;
        const int cpt = (n + NT - 1) / NT;
        const int c0 = min(tid * cpt, n), c1 = min(c0 + cpt, n);
        int cnt = 0;
        for (int c = c0; c < c1; ++c)
          if (key64[c] == ~0ull) cnt += (lens[c] + a.tile_tokens - 1) / a.tile_tokens;
        int total;
        int off = block_scan_excl<NT>(cnt, sh, total);
        if (total + 1 <= a.tile_cap) {
          for (int c = c0; c < c1; ++c) {
            if (key64[c] != ~0ull) continue;
            int lo, len;
            uc.chunk(c, lo, len);
            for (int t = 0; t < len; t += a.tile_tokens, ++off) {
              out[2 * off] = lo + t;
              out[2 * off + 1] = min(a.tile_tokens, len - t);
            }
          }
          base = total;
          __syncthreads();
          // the barrier orders every thread's tile stores before thread 0's
          // release (cumulative): the attention acquires the flag
          if (tid == 0 && base > 0) st_release(a.ready + s, 1 + base);
        }
      }
      DBG_T(4);
      for (int i = warp; i < nu; i += NW) {
        const int c = unc[i];
        double ex;
        if (c < uc.nc) {
          const double* crow = a.cent + (int64_t)u * a.c_stride + (int64_t)c * D;
          double part[G];
#pragma unroll
          for (int h = 0; h < G; ++h) part[h] = 0.0;
#pragma unroll
          for (int d = lane; d < D; d += 32) {
            const double cv = crow[d];
#pragma unroll
            for (int h = 0; h < G; ++h) part[h] = fma(qd[h][d], cv, part[h]);
          }
#pragma unroll
          for (int h = 0; h < G; ++h) part[h] = warp_sum(part[h]);
          ex = agg_d<G, AGG>(part + h0, nh);
        } else {
          ex = gex;
        }
        if (lane == 0) key64[c] = order_key(ex);
      }
      __syncthreads();
      DBG_T(5);
      if (a.dbg && threadIdx.x == 0) a.dbg[blockIdx.x * 16 + 15] = nu;
      if (nu <= kSmallUncertain) {
        // exact walk over the uncertain chunks: rank by (fp64 desc, chunk asc)
        const int rp = (int)R - s_win;
        int32_t* take = reinterpret_cast<int32_t*>(ak);  // approx keys no longer needed
        for (int i = tid; i < nu; i += NT) {
          const int ci = unc[i];
          const uint64_t ki = key64[ci];
          int before = 0;
          for (int j = 0; j < nu; ++j) {
            const int cj = unc[j];
            const uint64_t kj = key64[cj];
            if (kj > ki || (kj == ki && cj < ci)) before += lens[cj];
          }
          const int rem = rp - before;
          take[i] = rem <= 0 ? 0 : (rem < lens[ci] ? rem : lens[ci]);
        }
        __syncthreads();
        for (int c = tid; c < n; c += NT)
          if (key64[c] != ~0ull || base > 0) lens[c] = 0;  // phase A emitted the whole ones
        __syncthreads();
        for (int i = tid; i < nu; i += NT) lens[unc[i]] = take[i];
        __syncthreads();
        DBG_T(6);
        if (!a.split)
          emit_takes<NT>(uc, lens, n, row, a.tile_tokens,
                                     a.tiles + (int64_t)s * a.tile_cap * 2, a.tile_cap,
                                     a.ntiles + s, sh, base);
        DBG_T(7);
        done = true;
      } else {
        radix_threshold<NT, uint64_t>(key64, lens, n, R, sh, prefix, mask, rrem);
      }
    }
    if (!done && a.split) {
      walk_takes<NT, uint64_t>(key64, lens, n, R, prefix, mask, rrem, sh);
    } else if (!done) {
      walk_takes<NT, uint64_t>(key64, lens, n, R, prefix, mask, rrem, sh);
      if (base > 0) {  // phase A emitted the chunks kept whole (key ~0)
        for (int c = tid; c < n; c += NT)
          if (key64[c] == ~0ull) lens[c] = 0;
        __syncthreads();
      }
      emit_takes<NT>(uc, lens, n, row, a.tile_tokens, a.tiles + (int64_t)s * a.tile_cap * 2,
                     a.tile_cap, a.ntiles + s, sh, base);
    }
    if (a.split)
      emit_candidates<D, G, AGG, NT>(a, uc, lens, unc, n, s, qd, h0, nh, gex, u);
  }
  __syncthreads();
  if (tid == 0) {
    if (a.advance) a.gen_count[u] = g + 1;  // masks.py:236
    if (a.ready) {  // tiles, running sum and appended k/v are published together
      for (int it = 0; it < nitems; ++it)
        st_release(a.ready + (AGG == DHSA_AGG_NONE ? u * G + it : u), kReadyFinal);
    }
  }
  DBG_T(8);
}

// ------------------------------------------------------ prefill-time sketch --
// pass 1: per-unit max |c| over prompt chunks
__global__ void sketch_absmax_kernel(const double* __restrict__ cent, int64_t c_stride, int D,
                                     Layout lay, float* __restrict__ sinfo) {
  const int u = blockIdx.y;
  const int64_t n = (int64_t)lay.num_chunks(u) * D;
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(cent[(int64_t)u * c_stride + i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) {
    const float f = isfinite(m) ? __double2float_ru(m) : INFINITY;
    atomicMax(reinterpret_cast<unsigned int*>(sinfo + 4 * u + 3), __float_as_uint(f));
  }
}

// pass 2: scale, round to fp16, measure ||c''|| and ||c'' - c 2^-k|| per chunk.
// A warp per chunk (lane l owns dims 4l .. 4l+3 of every 128: two 16-byte
// fp64 loads, one 8-byte fp16 store), kSketchChunksPerCta chunks per CTA; the
// per-chunk bounds are reduced in the CTA first, so each CTA issues ONE pair
// of atomics on its unit's sinfo (one pair per chunk serialised on the same
// address made the r1 kernel atomic-bound: 0.15 of HBM at C3).
constexpr int kSketchChunksPerCta = 64;

__global__ __launch_bounds__(256) void sketch_build_kernel(const double* __restrict__ cent,
                                                           int64_t c_stride, int D, Layout lay,
                                                           __half* __restrict__ sk,
                                                           int64_t sk_stride,
                                                           float* __restrict__ sinfo) {
  __shared__ float s_fn[8], s_fe[8];
  const int u = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nc = lay.num_chunks(u);
  const int c0 = blockIdx.x * kSketchChunksPerCta;
  if (c0 >= nc) return;  // uniform over the CTA
  const float amax = sinfo[4 * u + 3];
  int k = 0;
  if (amax > 0.f && isfinite(amax)) k = ilogb((double)amax) + 1 - 14;  // max|c| 2^-k < 2^14
  const double sc = ldexp(1.0, -k);
  const bool afin = isfinite(amax);
  float wfn = 0.f, wfe = 0.f;
  for (int c = c0 + warp; c < min(c0 + kSketchChunksPerCta, nc); c += 8) {
    const double* src = cent + (int64_t)u * c_stride + (int64_t)c * D;
    __half* dst = sk + (int64_t)u * sk_stride + (int64_t)c * D;
    double nrm = 0.0, err = 0.0;
    bool finite = afin;
    for (int d = 4 * lane; d < D; d += 128) {
      const double2 a = __ldcs(reinterpret_cast<const double2*>(src + d));
      const double2 b = __ldcs(reinterpret_cast<const double2*>(src + d + 2));
      const double v[4] = {a.x * sc, a.y * sc, b.x * sc, b.y * sc};  // exact (power of two)
      __align__(8) __half h[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        h[j] = __double2half(v[j]);
        const double hv = (double)__half2float(h[j]);
        finite = finite && isfinite(hv);
        nrm = fma(hv, hv, nrm);
        err = fma(hv - v[j], hv - v[j], err);
      }
      *reinterpret_cast<uint2*>(dst + d) = *reinterpret_cast<const uint2*>(h);
    }
    nrm = warp_sum(nrm);
    err = warp_sum(err);
    finite = __all_sync(0xffffffffu, finite);
    // a non-finite sketch makes E infinite: every chunk is then re-scored
    const float fn = finite ? __double2float_ru(sqrt(nrm) * (1.0 + 1e-9)) : INFINITY;
    const float fe = finite ? __double2float_ru(sqrt(err) * (1.0 + 1e-9)) : INFINITY;
    wfn = fmaxf(wfn, fn);
    wfe = fmaxf(wfe, fe);
  }
  if (lane == 0) {
    s_fn[warp] = wfn;
    s_fe[warp] = wfe;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float fn = s_fn[0], fe = s_fe[0];
    for (int w = 1; w < 8; ++w) {
      fn = fmaxf(fn, s_fn[w]);
      fe = fmaxf(fe, s_fe[w]);
    }
    if (blockIdx.x == 0) sinfo[4 * u + 0] = (float)k;
    atomicMax(reinterpret_cast<unsigned int*>(sinfo + 4 * u + 1), __float_as_uint(fn));
    atomicMax(reinterpret_cast<unsigned int*>(sinfo + 4 * u + 2), __float_as_uint(fe));
  }
}

template <int D, int G, int AGG>
static int launch_step(const SketchArgs& a, int U, size_t sel_smem, cudaStream_t s) {
  auto score = sketch_score_kernel<D, G, AGG>;
  constexpr int ring = kTcStages * (D / 64) * 64 * 128 + 1024;
  cudaError_t e = cudaFuncSetAttribute(score, cudaFuncAttributeMaxDynamicSharedMemorySize, ring);
  if (e != cudaSuccess) {
    set_error("dhsa_decode_step_bf16: %s", cudaGetErrorString(e));
    return DHSA_ECUDA;
  }
  CUtensorMap tm;
  int rc = make_tmap_2d(&tm, a.sketch, (int64_t)U * (a.sk_stride / D), D,
                        CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  if (rc) return rc;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, score, kTcThreads, ring);
  // three stream CTAs per SM (sketch_common.cuh: ring depth x CTAs measured)
  if (per_sm > 3) per_sm = 3;
  if (const char* e = getenv("DHSA_SKETCH_CTAS_PER_SM")) per_sm = atoi(e) > 0 ? atoi(e) : per_sm;
  int64_t grid = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
  if (grid > a.total_slices) grid = a.total_slices;
  score<<<(unsigned)grid, kTcThreads, ring, s>>>(tm, a);
  rc = check_launch("dhsa_decode_step_bf16(score)");
  if (rc) return rc;
  {
    int rc2 = 0;
    if (launch_select2<D, G, AGG>(a, U, s, &rc2)) return rc2;
  }
  // a wider CTA for very long units (e.g. 16K chunks in one split-KV shard)
  auto sel = a.n_max > 4096 ? sketch_select_kernel<D, G, AGG, 1024>
                            : sketch_select_kernel<D, G, AGG, kSelectThreads>;
  const int sel_threads = a.n_max > 4096 ? 1024 : kSelectThreads;
  {  // static + dynamic may exceed the 48 KB default even for small dynamic sizes
    e = cudaFuncSetAttribute(sel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel_smem);
    if (e != cudaSuccess) {
      set_error("dhsa_decode_step_bf16: %s", cudaGetErrorString(e));
      return DHSA_ECUDA;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)U);
  cfg.blockDim = dim3(sel_threads);
  cfg.dynamicSmemBytes = sel_smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, sel, a);
  if (e != cudaSuccess) {
    set_error("dhsa_decode_step_bf16(select): %s", cudaGetErrorString(e));
    return DHSA_ECUDA;
  }
  return check_launch("dhsa_decode_step_bf16(select)");
}

template <int D, int AGG>
static int dispatch_g(int G, const SketchArgs& a, int U, size_t smem, cudaStream_t s) {
  switch (G) {
    case 1: return launch_step<D, 1, AGG>(a, U, smem, s);
    case 2: return launch_step<D, 2, AGG>(a, U, smem, s);
    case 4: return launch_step<D, 4, AGG>(a, U, smem, s);
    case 8: return launch_step<D, 8, AGG>(a, U, smem, s);
  }
  set_error("dhsa_decode_step_bf16: group size %d not in {1,2,4,8}", G);
  return DHSA_EINVAL;
}

template <int D>
static int dispatch_agg(int agg, int G, const SketchArgs& a, int U, size_t smem, cudaStream_t s) {
  switch (agg) {
    case DHSA_AGG_NONE: return dispatch_g<D, DHSA_AGG_NONE>(G, a, U, smem, s);
    case DHSA_AGG_MAX: return dispatch_g<D, DHSA_AGG_MAX>(G, a, U, smem, s);
    case DHSA_AGG_MEAN: return dispatch_g<D, DHSA_AGG_MEAN>(G, a, U, smem, s);
  }
  set_error("dhsa_decode_step_bf16: unknown aggregation %d", agg);
  return DHSA_EINVAL;
}

}  // namespace dhsa

using namespace dhsa;

constexpr int64_t kSelectSmemLimit = 96 * 1024;

static int64_t select_scratch_per_unit(int max_chunks) {
  return (((int64_t)max_chunks + 1) * (8 + 4 + 4 + 4) + 15) / 16 * 16;
}

extern "C" int64_t dhsa_sketch_select_scratch_size(int max_chunks) {
  return select_scratch_per_unit(max_chunks);
}

extern "C" int dhsa_sketch_build(const double* centroids, int64_t c_unit_stride, int D, int U,
                                 dhsa_layout layout, void* sketch, int64_t sk_unit_stride,
                                 float* sinfo, dhsa_stream_t stream) {
  DHSA_REQUIRE(centroids && sketch && sinfo && D >= 1 && U >= 1, "dhsa_sketch_build: bad arguments");
  DHSA_REQUIRE(valid_layout(layout) && layout.max_chunks >= 1, "dhsa_sketch_build: bad layout");
  DHSA_REQUIRE(D % 4 == 0 && c_unit_stride % 2 == 0 && sk_unit_stride % 4 == 0 &&
                   ((uintptr_t)centroids & 15) == 0 && ((uintptr_t)sketch & 7) == 0,
               "dhsa_sketch_build: D % 4 == 0 and aligned centroid / sketch rows required");
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(sinfo, 0, sizeof(float) * 4 * U, s);
  Layout lay(layout);
  const int64_t work = (int64_t)layout.max_chunks * D;
  dim3 g1((unsigned)((work + 255) / 256 < 64 ? (work + 255) / 256 : 64), (unsigned)U);
  sketch_absmax_kernel<<<g1, 256, 0, s>>>(centroids, c_unit_stride, D, lay, sinfo);
  dim3 g2((unsigned)((layout.max_chunks + kSketchChunksPerCta - 1) / kSketchChunksPerCta),
          (unsigned)U);
  sketch_build_kernel<<<g2, 256, 0, s>>>(centroids, c_unit_stride, D, lay, (__half*)sketch,
                                         sk_unit_stride, sinfo);
  return check_launch("dhsa_sketch_build");
}

static int decode_step_impl(
    const void* q, const void* sketch, int64_t sk_unit_stride, const float* sinfo,
    const double* centroids, int64_t c_unit_stride, double* gen_sum, int32_t* gen_count,
    const void* k_new, const void* v_new, void* k_cache, void* v_cache, int64_t cache_unit_stride,
    dhsa_layout layout, int U, int G, int D, int agg, int64_t budget, int tile_tokens,
    int32_t* tiles, int64_t tile_cap, int32_t* ntiles, float* approx, int64_t sc_stride,
    void* scratch, int32_t* ready, int advance, int32_t* progress, dhsa_stream_t stream,
    const dhsa_split_shard* shard = nullptr, void* cand = nullptr, int64_t cand_stride = 0,
    int cand_cap = 0) {
  DHSA_REQUIRE(q && sketch && sinfo && centroids && gen_sum && gen_count &&
                   (shard || (tiles && ntiles)) && approx,
               "dhsa_decode_step_bf16: null pointer");
  DHSA_REQUIRE(budget >= 1, "budget must be >= 1");
  DHSA_REQUIRE(D == 64 || D == 128, "dhsa_decode_step_bf16: D must be 64 or 128");
  DHSA_REQUIRE(U >= 1 && tile_tokens >= 1 && tile_cap >= 2, "dhsa_decode_step_bf16: bad shape");
  DHSA_REQUIRE(valid_layout(layout) && layout.max_chunks >= 1, "dhsa_decode_step_bf16: bad layout");
  DHSA_REQUIRE(sc_stride >= layout.max_chunks + 1, "dhsa_decode_step_bf16: sc_stride too small");
  DHSA_REQUIRE(((uintptr_t)q & 15) == 0 && ((uintptr_t)sketch & 15) == 0 &&
                   (sk_unit_stride * 2) % 16 == 0,
               "dhsa_decode_step_bf16: q/sketch must be 16-byte aligned");
  DHSA_REQUIRE(!(k_cache || v_cache) || k_new, "dhsa_decode_step_bf16: cache append needs k_new");
  SketchArgs a{};
  a.q = (const __nv_bfloat16*)q;
  a.sketch = (const __half*)sketch;
  a.sk_stride = sk_unit_stride;
  a.sinfo = sinfo;
  a.cent = centroids;
  a.c_stride = c_unit_stride;
  a.gen_sum = gen_sum;
  a.gen_count = gen_count;
  a.k_new = (const __nv_bfloat16*)k_new;
  a.v_new = (const __nv_bfloat16*)v_new;
  a.kc = (__nv_bfloat16*)k_cache;
  a.vc = (__nv_bfloat16*)v_cache;
  a.cache_stride = cache_unit_stride;
  a.lay = Layout(layout);
  a.approx = approx;
  a.sc_stride = sc_stride;
  a.slices_per_unit = (layout.max_chunks + kSliceRows - 1) / kSliceRows;
  a.total_slices = (int64_t)a.slices_per_unit * U;
  a.budget = budget;
  a.tile_tokens = tile_tokens;
  a.tiles = tiles;
  a.tile_cap = tile_cap;
  a.ntiles = ntiles;
  a.n_max = layout.max_chunks + 1;
  a.advance = advance;
  a.ready = ready;
  a.n_units = U;
  a.progress = progress;
  {
    // two-phase tile publication pays when the attention grid has SMs to
    // start on while the selects run (few select CTAs, e.g. C2: 64 units,
    // 51.8 vs 54.9 us); with a select CTA on every SM (C3: 256 units) the
    // attention CTAs are not resident before the selects end and the extra
    // scan only lengthens the select (+1.2 us)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int items = agg == DHSA_AGG_NONE ? U * G : U;
    a.early = ready != nullptr && items <= sms;
    if (const char* e = getenv("DHSA_EARLY_TILES")) a.early = ready != nullptr && atoi(e) != 0;
  }
  if (shard) {
    DHSA_REQUIRE(cand && cand_cap >= 1 && cand_stride >= (int64_t)sizeof(SplitCand) * (cand_cap + 1) &&
                     cand_stride % 8 == 0,
                 "dhsa_decode_candidates_bf16: bad candidate buffer");
    DHSA_REQUIRE(shard->chunk_offset >= 0 && shard->total_chunks >= shard->chunk_offset &&
                     shard->total_prompt >= 1,
                 "dhsa_decode_candidates_bf16: bad shard description");
    a.split = 1;
    a.chunk_offset = shard->chunk_offset;
    a.total_chunks = shard->total_chunks;
    a.total_prompt = shard->total_prompt;
    a.owns_tail = shard->owns_tail;
    a.cand = (unsigned char*)cand;
    a.cand_stride = cand_stride;
    a.cand_cap = cand_cap;
    a.advance = 0;
    a.ready = nullptr;
    a.early = 0;
  }
  if (const char* e = getenv("DHSA_DEBUG_TIMING")) a.dbg = (unsigned long long*)strtoull(e, nullptr, 0);
  a.l2_hint = 1;
  if (const char* e = getenv("DHSA_L2_HINT")) a.l2_hint = atoi(e);
  a.reps = 1;
  if (const char* e = getenv("DHSA_SELECT_REPS")) a.reps = atoi(e) > 0 ? atoi(e) : 1;
  if (const char* e = getenv("DHSA_RELAXED_FLAGS")) a.relaxed = atoi(e);
  // the sketch stream in 3 waves when there are many units (measured: C3,
  // 256 units, 122.9 -> 119.3 us/step; p2, 128 units, 72.1 -> 70.0; 4 and 6
  // waves are slower), in one wave for small batches (C2 / p4, 64 units:
  // 43.5 vs 44.0 / 48.7 vs 49.0 us with 2 waves)
  a.waves = U >= 100 ? 3 : 1;
  if (const char* e = getenv("DHSA_SKETCH_WAVES")) a.waves = atoi(e) > 0 ? atoi(e) : 1;
  if (a.waves > 4) a.waves = 4;
  for (int w = 0; w < 4; ++w) a.wave_end[w] = 1000 * (w + 1) / a.waves;  // equal waves
  if (const char* e = getenv("DHSA_SKETCH_WAVE_ENDS")) {  // e.g. "500,800" (permille)
    const char* p = e;
    for (int w = 0; w < a.waves - 1 && *p; ++w) {
      a.wave_end[w] = atoi(p);
      while (*p && *p != ',') ++p;
      if (*p == ',') ++p;
    }
  }
  const int64_t need = select_scratch_per_unit(layout.max_chunks);
  size_t smem = 0;
  if (scratch) {
    a.gscratch = (unsigned char*)scratch;
    a.gscratch_stride = need;
  }
  if (need <= kSelectSmemLimit) {  // the generic select keeps its arrays in shared memory
    a.smem_select = 1;
    smem = (size_t)a.n_max * (8 + 4 + 4 + 4);
  } else {
    DHSA_REQUIRE(scratch, "dhsa_decode_step_bf16: %lld bytes of select scratch per unit required",
                 (long long)need);
    a.smem_select = 0;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (D == 128) return dispatch_agg<128>(agg, G, a, U, smem, s);
  return dispatch_agg<64>(agg, G, a, U, smem, s);
}

extern "C" int dhsa_decode_step_bf16(
    const void* q, const void* sketch, int64_t sk_unit_stride, const float* sinfo,
    const double* centroids, int64_t c_unit_stride, double* gen_sum, int32_t* gen_count,
    const void* k_new, const void* v_new, void* k_cache, void* v_cache, int64_t cache_unit_stride,
    dhsa_layout layout, int U, int G, int D, int agg, int64_t budget, int tile_tokens,
    int32_t* tiles, int64_t tile_cap, int32_t* ntiles, float* approx, int64_t sc_stride,
    void* scratch, int32_t* ready, int advance, int32_t* progress, dhsa_stream_t stream) {
  return decode_step_impl(q, sketch, sk_unit_stride, sinfo, centroids, c_unit_stride, gen_sum,
                          gen_count, k_new, v_new, k_cache, v_cache, cache_unit_stride, layout, U,
                          G, D, agg, budget, tile_tokens, tiles, tile_cap, ntiles, approx,
                          sc_stride, scratch, ready, advance, progress, stream);
}

extern "C" int dhsa_decode_candidates_bf16(
    const void* q, const void* sketch, int64_t sk_unit_stride, const float* sinfo,
    const double* centroids, int64_t c_unit_stride, double* gen_sum, const int32_t* gen_count,
    const void* k_new, const void* v_new, void* k_cache, void* v_cache, int64_t cache_unit_stride,
    dhsa_layout layout, int U, int G, int D, int agg, int64_t budget, dhsa_split_shard shard,
    void* cand, int64_t cand_stride, int cand_cap, float* approx, int64_t sc_stride,
    void* scratch, int32_t* progress, dhsa_stream_t stream) {
  return decode_step_impl(q, sketch, sk_unit_stride, sinfo, centroids, c_unit_stride, gen_sum,
                          const_cast<int32_t*>(gen_count), k_new, v_new, k_cache, v_cache,
                          cache_unit_stride, layout, U, G, D, agg, budget, 64, nullptr, 2, nullptr,
                          approx, sc_stride, scratch, nullptr, 0, progress, stream, &shard, cand,
                          cand_stride, cand_cap);
}
