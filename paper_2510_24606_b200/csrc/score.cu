// K3 (+K2) — decode scores: raw query . chunk centroid, fp64, no 1/sqrt(d).
//
// Reference: masks._decode_row (masks.py:153-173): chunk keys are the cached
// prompt centroids, the generated-chunk centroid gen_sum/sqrt(g) when g >= 1
// (masks.py:161), and the singleton current key; the chunk query is q itself
// (masks.py:164); scores = einsum("id,jd->ij") (masks.py:165).  The singleton
// score never affects the selection (topk_row excludes `row`, masks.py:120),
// so it is not computed.  Multi-head aggregation follows
// harness.aggregated_chunk_scores (harness.py:288-306): max (default) or mean
// over the heads that share one key set.
//
// The centroid stream is the HBM-bound part of a decode step (fp64, D*8 bytes
// per chunk per kv-head).  Fast path (D = 64/128): one warp reads CH chunk
// rows per iteration with coalesced 128-bit loads (lane = D/32 consecutive
// dims), keeps the G query heads of the kv group in registers, forms CH*G
// partial dot products per lane and finishes them with a transpose-reduce
// (CH*G - 1 shuffles for CH*G complete dots) before the head aggregation.
#include "capi.cuh"

namespace dhsa {

template <int G, int AGG, int BASE>
__device__ __forceinline__ double head_aggregate(double s) {
  if constexpr (AGG != DHSA_AGG_NONE) {
#pragma unroll
    for (int k = 0; (1 << k) < G; ++k) {
      double o = shfl_xor_d(s, BASE << k);
      s = (AGG == DHSA_AGG_MAX) ? fmax(s, o) : s + o;
    }
  }
  return s;
}

// Generated-chunk slot + the folded state update; executed by one warp.
template <typename T, int G, int AGG>
__device__ void gen_slot(const T* __restrict__ q, double* __restrict__ gen_sum, int g, int u,
                         int D, int nc, int P, const T* __restrict__ k_new,
                         const T* __restrict__ v_new, T* __restrict__ kc, T* __restrict__ vc,
                         int64_t cache_stride, double* __restrict__ scores, int64_t sc_stride,
                         int lane) {
  double* gs = gen_sum + (int64_t)u * D;
  if (g >= 1) {
    const double rs = __dsqrt_rn((double)g);
    double part[G];
#pragma unroll
    for (int h = 0; h < G; ++h) part[h] = 0.0;
    for (int d = lane; d < D; d += 32) {
      const double cg = __ddiv_rn(gs[d], rs);
#pragma unroll
      for (int h = 0; h < G; ++h) part[h] = fma(to_f64(q[(int64_t)(u * G + h) * D + d]), cg, part[h]);
    }
#pragma unroll
    for (int h = 0; h < G; ++h) part[h] = warp_sum(part[h]);
    if (lane == 0) {
      if constexpr (AGG == DHSA_AGG_NONE) {
#pragma unroll
        for (int h = 0; h < G; ++h) scores[(int64_t)(u * G + h) * sc_stride + nc] = part[h];
      } else {
        double s = part[0];
#pragma unroll
        for (int h = 1; h < G; ++h) s = (AGG == DHSA_AGG_MAX) ? fmax(s, part[h]) : s + part[h];
        if (AGG == DHSA_AGG_MEAN) s = s / (double)G;
        scores[(int64_t)u * sc_stride + nc] = s;
      }
    }
  }
  __syncwarp();
  if (k_new) {
    const int64_t pos = (int64_t)(P + g) * D;
    for (int d = lane; d < D; d += 32) {
      const T kv = k_new[(int64_t)u * D + d];
      gs[d] = __dadd_rn(gs[d], to_f64(kv));  // masks.py:235, after the read above
      if (kc) kc[(int64_t)u * cache_stride + pos + d] = kv;
      if (vc) vc[(int64_t)u * cache_stride + pos + d] = v_new[(int64_t)u * D + d];
    }
  }
}

template <typename T, int D, int G, int AGG>
__global__ __launch_bounds__(256) void score_fast_kernel(
    const T* __restrict__ q, const double* __restrict__ cent, int64_t c_stride,
    double* __restrict__ gen_sum, const int32_t* __restrict__ gen_count,
    const T* __restrict__ k_new, const T* __restrict__ v_new, T* __restrict__ kc,
    T* __restrict__ vc, int64_t cache_stride, Layout lay, double* __restrict__ scores,
    int64_t sc_stride, int chunks_per_cta) {
  constexpr int VEC = D / 32;
  constexpr int CH = (32 / G) < 8 ? (32 / G) : 8;
  constexpr int NV = CH * G;
  constexpr int LOGNV = NV == 32 ? 5 : NV == 16 ? 4 : NV == 8 ? 3 : NV == 4 ? 2 : NV == 2 ? 1 : 0;
  constexpr int BASE = 1 << (5 - LOGNV);  // lane stride between value indices
  static_assert(VEC == 2 || VEC == 4, "D must be 64 or 128");

  const int u = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nc = lay.num_chunks(u);
  const int g = gen_count[u];

  if (blockIdx.x == 0 && warp == 0)
    gen_slot<T, G, AGG>(q, gen_sum, g, u, D, nc, lay.prompt_len(u), k_new, v_new, kc, vc,
                        cache_stride, scores, sc_stride, lane);

  double qr[G][VEC];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int v = 0; v < VEC; ++v) qr[h][v] = to_f64(q[(int64_t)(u * G + h) * D + lane * VEC + v]);

  const int c_begin = blockIdx.x * chunks_per_cta;
  const int c_end = min(c_begin + chunks_per_cta, nc);
  const double* base = cent + (int64_t)u * c_stride + lane * VEC;
  const int vidx = (lane >> (5 - LOGNV)) & (NV - 1);
  const int my_c = vidx / G, my_h = vidx % G;

  for (int c0 = c_begin + warp * CH; c0 < c_end; c0 += 8 * CH) {
    double x[CH][VEC];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (c0 + c < c_end) {
        const double2* p = reinterpret_cast<const double2*>(base + (int64_t)(c0 + c) * D);
#pragma unroll
        for (int v = 0; v < VEC / 2; ++v) {
          double2 t = __ldg(p + v);
          x[c][2 * v] = t.x;
          x[c][2 * v + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) x[c][v] = 0.0;
      }
    }
    double part[NV];
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
      for (int h = 0; h < G; ++h) {
        double s = 0.0;
#pragma unroll
        for (int v = 0; v < VEC; ++v) s = fma(qr[h][v], x[c][v], s);
        part[c * G + h] = s;
      }
    double s = transpose_reduce<NV>(part, lane);
    s = head_aggregate<G, AGG, BASE>(s);
    const int c = c0 + my_c;
    if ((lane & (BASE - 1)) == 0 && c < c_end) {
      if constexpr (AGG == DHSA_AGG_NONE) {
        scores[(int64_t)(u * G + my_h) * sc_stride + c] = s;
      } else if (my_h == 0) {
        scores[(int64_t)u * sc_stride + c] = (AGG == DHSA_AGG_MEAN) ? s / (double)G : s;
      }
    }
  }
}

// Generic path: any D, one warp per chunk, query heads staged in smem (fp64).
template <typename T, int AGG>
__global__ __launch_bounds__(256) void score_generic_kernel(
    const T* __restrict__ q, const double* __restrict__ cent, int64_t c_stride,
    double* __restrict__ gen_sum, const int32_t* __restrict__ gen_count,
    const T* __restrict__ k_new, const T* __restrict__ v_new, T* __restrict__ kc,
    T* __restrict__ vc, int64_t cache_stride, Layout lay, int G, int D,
    double* __restrict__ scores, int64_t sc_stride) {
  extern __shared__ double qs[];  // [G][D]
  const int u = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) qs[i] = to_f64(q[(int64_t)u * G * D + i]);
  __syncthreads();
  const int nc = lay.num_chunks(u);
  const int g = gen_count[u];
  const int c = blockIdx.x * 8 + warp;
  if (c > nc) return;
  double* gs = gen_sum + (int64_t)u * D;
  const bool is_gen = (c == nc);
  if (is_gen && g < 1 && !k_new) return;
  double agg = 0.0;
  const double rs = is_gen && g >= 1 ? __dsqrt_rn((double)g) : 1.0;
  if (!is_gen || g >= 1) {
    const double* row = cent + (int64_t)u * c_stride + (int64_t)c * D;
    for (int h = 0; h < G; ++h) {
      double s = 0.0;
      for (int d = lane; d < D; d += 32) {
        const double cv = is_gen ? __ddiv_rn(gs[d], rs) : row[d];
        s = fma(qs[h * D + d], cv, s);
      }
      s = warp_sum(s);
      if (AGG == DHSA_AGG_NONE) {
        if (lane == 0) scores[(int64_t)(u * G + h) * sc_stride + c] = s;
      } else if (h == 0) {
        agg = s;
      } else {
        agg = (AGG == DHSA_AGG_MAX) ? fmax(agg, s) : agg + s;
      }
    }
    if (AGG != DHSA_AGG_NONE && lane == 0)
      scores[(int64_t)u * sc_stride + c] = (AGG == DHSA_AGG_MEAN) ? agg / (double)G : agg;
  }
  __syncwarp();
  if (is_gen && k_new) {
    const int64_t pos = (int64_t)(lay.prompt_len(u) + g) * D;
    for (int d = lane; d < D; d += 32) {
      const T kv = k_new[(int64_t)u * D + d];
      gs[d] = __dadd_rn(gs[d], to_f64(kv));
      if (kc) kc[(int64_t)u * cache_stride + pos + d] = kv;
      if (vc) vc[(int64_t)u * cache_stride + pos + d] = v_new[(int64_t)u * D + d];
    }
  }
}

template <typename T, int D, int G, int AGG>
static void launch_fast(const dhsa_layout& layout, int U, const void* q, const double* cent,
                        int64_t cs, double* gsum, const int32_t* gcnt, const void* kn,
                        const void* vn, void* kc, void* vc, int64_t cache_stride, double* sc,
                        int64_t scs, cudaStream_t s) {
  constexpr int CH = (32 / G) < 8 ? (32 / G) : 8;
  // 4 warp-iterations per CTA: 256 threads stream 32*CH chunk rows.
  const int per_cta = 8 * CH * 4;
  const int nx = (layout.max_chunks + per_cta - 1) / per_cta;
  dim3 grid((unsigned)(nx < 1 ? 1 : nx), (unsigned)U);
  score_fast_kernel<T, D, G, AGG><<<grid, 256, 0, s>>>(
      (const T*)q, cent, cs, gsum, gcnt, (const T*)kn, (const T*)vn, (T*)kc, (T*)vc, cache_stride,
      Layout(layout), sc, scs, per_cta);
}

template <typename T, int D, int AGG>
static bool dispatch_g(int G, const dhsa_layout& l, int U, const void* q, const double* c,
                       int64_t cs, double* gs, const int32_t* gc, const void* kn, const void* vn,
                       void* kc, void* vc, int64_t cst, double* sc, int64_t scs, cudaStream_t s) {
  switch (G) {
    case 1: launch_fast<T, D, 1, AGG>(l, U, q, c, cs, gs, gc, kn, vn, kc, vc, cst, sc, scs, s); return true;
    case 2: launch_fast<T, D, 2, AGG>(l, U, q, c, cs, gs, gc, kn, vn, kc, vc, cst, sc, scs, s); return true;
    case 4: launch_fast<T, D, 4, AGG>(l, U, q, c, cs, gs, gc, kn, vn, kc, vc, cst, sc, scs, s); return true;
    case 8: launch_fast<T, D, 8, AGG>(l, U, q, c, cs, gs, gc, kn, vn, kc, vc, cst, sc, scs, s); return true;
    default: return false;
  }
}

template <typename T, int AGG>
static void launch_generic(const dhsa_layout& l, int U, int G, int D, const void* q,
                           const double* c, int64_t cs, double* gs, const int32_t* gc,
                           const void* kn, const void* vn, void* kc, void* vc, int64_t cst,
                           double* sc, int64_t scs, cudaStream_t s) {
  dim3 grid((unsigned)((l.max_chunks + 1 + 7) / 8), (unsigned)U);
  size_t smem = sizeof(double) * (size_t)G * D;
  score_generic_kernel<T, AGG><<<grid, 256, smem, s>>>(
      (const T*)q, c, cs, gs, gc, (const T*)kn, (const T*)vn, (T*)kc, (T*)vc, cst, Layout(l), G,
      D, sc, scs);
}

template <typename T, int AGG>
static int run(int G, int D, const dhsa_layout& l, int U, const void* q, const double* c,
               int64_t cs, double* gs, const int32_t* gc, const void* kn, const void* vn,
               void* kc, void* vc, int64_t cst, double* sc, int64_t scs, cudaStream_t s) {
  bool done = false;
  if (D == 128) done = dispatch_g<T, 128, AGG>(G, l, U, q, c, cs, gs, gc, kn, vn, kc, vc, cst, sc, scs, s);
  else if (D == 64) done = dispatch_g<T, 64, AGG>(G, l, U, q, c, cs, gs, gc, kn, vn, kc, vc, cst, sc, scs, s);
  if (!done) {
    DHSA_REQUIRE((size_t)G * D * sizeof(double) <= 48 * 1024, "dhsa_decode_score: G*D too large");
    launch_generic<T, AGG>(l, U, G, D, q, c, cs, gs, gc, kn, vn, kc, vc, cst, sc, scs, s);
  }
  return check_launch("dhsa_decode_score");
}

template <typename T>
static int run_agg(int agg, int G, int D, const dhsa_layout& l, int U, const void* q,
                   const double* c, int64_t cs, double* gs, const int32_t* gc, const void* kn,
                   const void* vn, void* kc, void* vc, int64_t cst, double* sc, int64_t scs,
                   cudaStream_t s) {
  switch (agg) {
    case DHSA_AGG_NONE: return run<T, DHSA_AGG_NONE>(G, D, l, U, q, c, cs, gs, gc, kn, vn, kc, vc, cst, sc, scs, s);
    case DHSA_AGG_MAX: return run<T, DHSA_AGG_MAX>(G, D, l, U, q, c, cs, gs, gc, kn, vn, kc, vc, cst, sc, scs, s);
    case DHSA_AGG_MEAN: return run<T, DHSA_AGG_MEAN>(G, D, l, U, q, c, cs, gs, gc, kn, vn, kc, vc, cst, sc, scs, s);
  }
  set_error("dhsa_decode_score: unknown aggregation %d", agg);
  return DHSA_EINVAL;
}

}  // namespace dhsa

using namespace dhsa;

extern "C" int dhsa_decode_score(int dtype, const void* q, const double* centroids,
                                 int64_t c_unit_stride, double* gen_sum,
                                 const int32_t* gen_count, const void* k_new, const void* v_new,
                                 void* k_cache, void* v_cache, int64_t cache_unit_stride,
                                 dhsa_layout layout, int U, int G, int D, int agg,
                                 double* scores, int64_t sc_stride, dhsa_stream_t stream) {
  DHSA_REQUIRE(q && centroids && gen_sum && gen_count && scores, "dhsa_decode_score: null pointer");
  DHSA_REQUIRE(U >= 1 && G >= 1 && G <= 32 && D >= 1, "dhsa_decode_score: bad shape");
  DHSA_REQUIRE(valid_layout(layout) && layout.max_chunks >= 0, "dhsa_decode_score: bad layout");
  DHSA_REQUIRE(sc_stride >= layout.max_chunks + 1, "dhsa_decode_score: sc_stride too small");
  DHSA_REQUIRE(!(k_cache || v_cache) || k_new, "dhsa_decode_score: cache append needs k_new");
  DHSA_REQUIRE(!v_cache || v_new, "dhsa_decode_score: v_cache append needs v_new");
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DHSA_F64: return run_agg<double>(agg, G, D, layout, U, q, centroids, c_unit_stride, gen_sum, gen_count, k_new, v_new, k_cache, v_cache, cache_unit_stride, scores, sc_stride, s);
    case DHSA_F32: return run_agg<float>(agg, G, D, layout, U, q, centroids, c_unit_stride, gen_sum, gen_count, k_new, v_new, k_cache, v_cache, cache_unit_stride, scores, sc_stride, s);
    case DHSA_BF16: return run_agg<__nv_bfloat16>(agg, G, D, layout, U, q, centroids, c_unit_stride, gen_sum, gen_count, k_new, v_new, k_cache, v_cache, cache_unit_stride, scores, sc_stride, s);
  }
  set_error("dhsa_decode_score: unknown dtype %d", dtype);
  return DHSA_EINVAL;
}
