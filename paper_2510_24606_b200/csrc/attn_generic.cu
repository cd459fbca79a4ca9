// K5 (fp32 / fp64 parity modes) — exact attention over selected token tiles
// with CUDA-core FMA and accumulation in the input precision.
//
// Reference: dense_attention's per-row body (core.py:113-118):
//     scores = einsum("jd,d->j", k[idx], q[i]) * (1/sqrt(d))
//     out[i] = softmax_row(scores) @ v[idx]          (softmax_row core.py:69-77)
// computed here as an online softmax in the log2 domain (p = 2^(s*log2e/sqrt(d)
// - m)), split over CTAs and merged by the last CTA (attn_common.cuh).  Used for
// fp32 KV caches (tolerance 1e-5 relative) and for the fp64 drop-in API
// (tolerance 1e-12 against the float64 reference).  bf16 goes through the
// tensor-core kernel in attn_mma.cu.
#include "attn_common.cuh"
#include "capi.cuh"

namespace dhsa {

int attn_mma_bf16(const void* q, const void* k_cache, const void* v_cache,
                  int64_t cache_unit_stride, int64_t cache_rows, int items, int items_per_unit,
                  int GH, int D, const int32_t* tiles, int64_t tile_cap, const int32_t* ntiles,
                  int splits, void* out, void* ws, int32_t* counters, int32_t* ready,
                  float* rec_out, cudaStream_t s);

constexpr int kGHMax = 8;

template <typename T, int MAXV>
__global__ __launch_bounds__(128) void attn_generic_kernel(
    const T* __restrict__ q, const T* __restrict__ kc, const T* __restrict__ vc,
    int64_t cache_unit_stride, int items_per_unit, int GH, int D,
    const int32_t* __restrict__ tiles, int64_t tile_cap, const int32_t* __restrict__ ntiles,
    int splits, T* __restrict__ out, void* ws, int32_t* counters, double scale_log2) {
  using A = typename Acc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* qs = reinterpret_cast<A*>(smem_raw);  // [GH][D], pre-scaled
  A* red = qs + GH * D;                    // [4 warps][GH][D+2]
  const int item = blockIdx.y, split = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int unit = item / items_per_unit;
  for (int i = threadIdx.x; i < GH * D; i += blockDim.x)
    qs[i] = (A)(to_f64(q[(int64_t)item * GH * D + i]) * scale_log2);
  __syncthreads();

  const int nt = ntiles[item];
  const int t_begin = (int)((int64_t)nt * split / splits);
  const int t_end = (int)((int64_t)nt * (split + 1) / splits);
  const T* kbase = kc + (int64_t)unit * cache_unit_stride;
  const T* vbase = vc + (int64_t)unit * cache_unit_stride;
  const int32_t* tl = tiles + (int64_t)item * tile_cap * 2;

  A m[kGHMax], l[kGHMax], acc[kGHMax][MAXV];
#pragma unroll
  for (int h = 0; h < kGHMax; ++h) {
    m[h] = -INFINITY;
    l[h] = 0;
#pragma unroll
    for (int v = 0; v < MAXV; ++v) acc[h][v] = 0;
  }
  for (int t = t_begin; t < t_end; ++t) {
    const int start = tl[2 * t], count = tl[2 * t + 1];
    for (int j = warp; j < count; j += 4) {
      const T* krow = kbase + (int64_t)(start + j) * D;
      const T* vrow = vbase + (int64_t)(start + j) * D;
      A kv[MAXV], vv[MAXV];
#pragma unroll
      for (int v = 0; v < MAXV; ++v) {
        const int d = lane + 32 * v;
        kv[v] = d < D ? (A)to_f64(krow[d]) : (A)0;
        vv[v] = d < D ? (A)to_f64(vrow[d]) : (A)0;
      }
#pragma unroll
      for (int h = 0; h < kGHMax; ++h) {
        if (h >= GH) break;
        A s = 0;
#pragma unroll
        for (int v = 0; v < MAXV; ++v) {
          const int d = lane + 32 * v;
          if (d < D) s = fma(qs[h * D + d], kv[v], s);
        }
        s = warp_sum(s);
        const A mn = fmax(m[h], s);
        const A corr = exp2_acc<A>(m[h] - mn);
        const A p = exp2_acc<A>(s - mn);
        l[h] = l[h] * corr + p;
#pragma unroll
        for (int v = 0; v < MAXV; ++v) acc[h][v] = fma(p, vv[v], acc[h][v] * corr);
        m[h] = mn;
      }
    }
  }
  // combine the 4 warps
  const int rec = D + 2;
#pragma unroll
  for (int h = 0; h < kGHMax; ++h) {
    if (h >= GH) break;
    A* r = red + ((int64_t)warp * GH + h) * rec;
    if (lane == 0) {
      r[0] = m[h];
      r[1] = l[h];
    }
#pragma unroll
    for (int v = 0; v < MAXV; ++v) {
      const int d = lane + 32 * v;
      if (d < D) r[2 + d] = acc[h][v];
    }
  }
  __syncthreads();
  const bool direct = (splits == 1);
  for (int hd = threadIdx.x; hd < GH * D; hd += blockDim.x) {
    const int h = hd / D, d = hd - h * D;
    A mstar = -INFINITY;
    for (int w = 0; w < 4; ++w) mstar = fmax(mstar, red[((int64_t)w * GH + h) * rec]);
    A lsum = 0, a = 0;
    for (int w = 0; w < 4; ++w) {
      const A* r = red + ((int64_t)w * GH + h) * rec;
      if (r[0] == -INFINITY) continue;
      const A wgt = exp2_acc<A>(r[0] - mstar);
      lsum += wgt * r[1];
      a += wgt * r[2 + d];
    }
    if (direct) {
      out[((int64_t)item * GH + h) * D + d] = from_acc<T>(a / lsum);
    } else {
      A* p = partial_ptr<A>(ws, item, split, splits, h, GH, D);
      if (d == 0) {
        p[0] = mstar;
        p[1] = lsum;
      }
      p[2 + d] = a;
    }
  }
  if (direct) return;
  if (split_arrive(counters, item, splits)) merge_partials<T, A>(ws, item, splits, GH, D, out);
}

template <typename T, int MAXV>
static void launch_generic(const void* q, const void* kc, const void* vc, int64_t cus, int items,
                           int ipu, int GH, int D, const int32_t* tiles, int64_t cap,
                           const int32_t* nt, int splits, void* out, void* ws, int32_t* cnt,
                           cudaStream_t s) {
  using A = typename Acc<T>::type;
  const size_t smem = sizeof(A) * ((size_t)GH * D + 4 * (size_t)GH * (D + 2));
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(attn_generic_kernel<T, MAXV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  const double scale_log2 = 1.4426950408889634 / sqrt((double)D);
  dim3 grid((unsigned)splits, (unsigned)items);
  attn_generic_kernel<T, MAXV><<<grid, 128, smem, s>>>(
      (const T*)q, (const T*)kc, (const T*)vc, cus, ipu, GH, D, tiles, cap, nt, splits, (T*)out,
      ws, cnt, scale_log2);
}

template <typename T>
static int run_generic(const void* q, const void* kc, const void* vc, int64_t cus, int items,
                       int ipu, int GH, int D, const int32_t* tiles, int64_t cap,
                       const int32_t* nt, int splits, void* out, void* ws, int32_t* cnt,
                       cudaStream_t s) {
  if (D <= 32) launch_generic<T, 1>(q, kc, vc, cus, items, ipu, GH, D, tiles, cap, nt, splits, out, ws, cnt, s);
  else if (D <= 64) launch_generic<T, 2>(q, kc, vc, cus, items, ipu, GH, D, tiles, cap, nt, splits, out, ws, cnt, s);
  else if (D <= 128) launch_generic<T, 4>(q, kc, vc, cus, items, ipu, GH, D, tiles, cap, nt, splits, out, ws, cnt, s);
  else launch_generic<T, 8>(q, kc, vc, cus, items, ipu, GH, D, tiles, cap, nt, splits, out, ws, cnt, s);
  return check_launch("dhsa_attn");
}

}  // namespace dhsa

using namespace dhsa;

extern "C" int64_t dhsa_attn_workspace_size(int dtype, int items, int GH, int D, int splits) {
  if (splits <= 1) return 0;
  const int64_t elt = dtype == DHSA_F64 ? 8 : 4;
  return elt * (int64_t)items * splits * GH * (D + 2);
}

extern "C" int dhsa_attn(int dtype, const void* q, const void* k_cache, const void* v_cache,
                         int64_t cache_unit_stride, int64_t cache_rows, int items,
                         int items_per_unit, int GH, int D, const int32_t* tiles,
                         int64_t tile_cap, const int32_t* ntiles, int splits, void* out,
                         void* workspace, int32_t* counters, int32_t* ready,
                         dhsa_stream_t stream) {
  DHSA_REQUIRE(q && k_cache && v_cache && tiles && ntiles && out, "dhsa_attn: null pointer");
  DHSA_REQUIRE(items >= 1 && items_per_unit >= 1 && GH >= 1 && GH <= kGHMax && D >= 1 &&
                   D <= 256 && splits >= 1 && tile_cap >= 1,
               "dhsa_attn: bad shape (GH <= 8, D <= 256)");
  DHSA_REQUIRE(splits == 1 || (workspace && counters), "dhsa_attn: split-KV needs workspace");
  DHSA_REQUIRE(!ready || dtype == DHSA_BF16, "dhsa_attn: ready flags are a bf16-path feature");
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DHSA_F64:
      return run_generic<double>(q, k_cache, v_cache, cache_unit_stride, items, items_per_unit, GH,
                                 D, tiles, tile_cap, ntiles, splits, out, workspace, counters, s);
    case DHSA_F32:
      return run_generic<float>(q, k_cache, v_cache, cache_unit_stride, items, items_per_unit, GH,
                                D, tiles, tile_cap, ntiles, splits, out, workspace, counters, s);
    case DHSA_BF16:
      return attn_mma_bf16(q, k_cache, v_cache, cache_unit_stride, cache_rows, items,
                           items_per_unit, GH, D, tiles, tile_cap, ntiles, splits, out, workspace,
                           counters, ready, nullptr, s);
  }
  set_error("dhsa_attn: unknown dtype %d", dtype);
  return DHSA_EINVAL;
}

extern "C" int dhsa_attn_partials(const void* q, const void* k_cache, const void* v_cache,
                                  int64_t cache_unit_stride, int64_t cache_rows, int items,
                                  int items_per_unit, int GH, int D, const int32_t* tiles,
                                  int64_t tile_cap, const int32_t* ntiles, int splits,
                                  float* records, void* workspace, int32_t* counters,
                                  dhsa_stream_t stream) {
  DHSA_REQUIRE(q && k_cache && v_cache && tiles && ntiles && records,
               "dhsa_attn_partials: null pointer");
  DHSA_REQUIRE(items >= 1 && items_per_unit >= 1 && GH >= 1 && GH <= kGHMax && splits >= 1 &&
                   tile_cap >= 1,
               "dhsa_attn_partials: bad shape (GH <= 8)");
  DHSA_REQUIRE(splits == 1 || (workspace && counters),
               "dhsa_attn_partials: split-KV needs workspace");
  return attn_mma_bf16(q, k_cache, v_cache, cache_unit_stride, cache_rows, items, items_per_unit,
                       GH, D, tiles, tile_cap, ntiles, splits, nullptr, workspace, counters,
                       nullptr, records, (cudaStream_t)stream);
}
