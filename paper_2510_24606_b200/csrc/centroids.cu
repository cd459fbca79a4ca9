// K1 — chunk centroids, fp64, bit-exact with the reference.
//
// Reference: chunk_repr.aggregate_rows (chunk_repr.py:57-68) calls
// aggregate_chunk (:38-54) = sequential_sum(t) / sqrt(n); sequential_sum
// (:29-35) starts from 0.0 and adds one row at a time in token order.  Every
// thread here owns one (chunk, dimension) pair and performs exactly that
// sequence of IEEE fp64 additions followed by one correctly rounded division
// by sqrt((double)n), so the result is bit-identical for any input dtype
// (bf16/fp32 upcasts are exact).  Loads are coalesced across the dimension
// axis (consecutive threads = consecutive dims of the same token row).
#include "capi.cuh"

namespace dhsa {

template <typename T>
__global__ __launch_bounds__(256) void centroids_kernel(const T* __restrict__ x,
                                                        int64_t x_unit_stride, int D,
                                                        Layout lay, int normalize,
                                                        double* __restrict__ out,
                                                        int64_t out_unit_stride) {
  const int u = blockIdx.y;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = (int)(idx / D);
  const int d = (int)(idx - (int64_t)c * D);
  if (c >= lay.num_chunks(u)) return;
  int lo, hi;
  lay.chunk(u, c, lo, hi);
  const T* src = x + (int64_t)u * x_unit_stride + (int64_t)lo * D + d;
  double acc = 0.0;
  int t = 0;
  const int n = hi - lo;
  // 8 independent loads in flight, then the additions in token order.
  for (; t + 8 <= n; t += 8) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = to_f64(src[(int64_t)(t + k) * D]);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, v[k]);
  }
  for (; t < n; ++t) acc = __dadd_rn(acc, to_f64(src[(int64_t)t * D]));
  out[(int64_t)u * out_unit_stride + (int64_t)c * D + d] =
      normalize ? __ddiv_rn(acc, __dsqrt_rn((double)n)) : acc;
}

// bf16 fast path: each thread owns two adjacent dimensions (one 4-byte
// bf16x2 load per token row, 128 B per warp request) and keeps 16 rows in
// flight; the per-dimension addition order is unchanged (bit-exact).
__global__ __launch_bounds__(256) void centroids_bf16x2_kernel(
    const __nv_bfloat16* __restrict__ x, int64_t x_unit_stride, int D, Layout lay, int normalize,
    double* __restrict__ out, int64_t out_unit_stride) {
  const int u = blockIdx.y;
  const int D2 = D / 2;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = (int)(idx / D2);
  const int d = 2 * (int)(idx - (int64_t)c * D2);
  if (c >= lay.num_chunks(u)) return;
  int lo, hi;
  lay.chunk(u, c, lo, hi);
  const __nv_bfloat162* src =
      reinterpret_cast<const __nv_bfloat162*>(x + (int64_t)u * x_unit_stride + (int64_t)lo * D + d);
  const int64_t rs = D2;  // row stride in bf16x2
  double a0 = 0.0, a1 = 0.0;
  int t = 0;
  const int n = hi - lo;
  for (; t + 16 <= n; t += 16) {
    float2 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __bfloat1622float2(src[(int64_t)(t + k) * rs]);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = __dadd_rn(a0, (double)v[k].x);
      a1 = __dadd_rn(a1, (double)v[k].y);
    }
  }
  for (; t < n; ++t) {
    const float2 v = __bfloat1622float2(src[(int64_t)t * rs]);
    a0 = __dadd_rn(a0, (double)v.x);
    a1 = __dadd_rn(a1, (double)v.y);
  }
  double* o = out + (int64_t)u * out_unit_stride + (int64_t)c * D + d;
  if (normalize) {
    const double r = __dsqrt_rn((double)n);
    a0 = __ddiv_rn(a0, r);
    a1 = __ddiv_rn(a1, r);
  }
  o[0] = a0;
  o[1] = a1;
}

// bf16, D % 8 == 0 (the decode/prefill path): each thread owns eight
// adjacent dimensions — one 16-byte load per token row, so a half-warp reads
// a whole 256-byte row of D = 128 — with 8 rows in flight (128 B per thread);
// the per-dimension addition order is still token order (bit-exact).  The
// eight fp64 results leave as four 16-byte stores.
__global__ __launch_bounds__(256) void centroids_bf16x8_kernel(
    const __nv_bfloat16* __restrict__ x, int64_t x_unit_stride, int D, Layout lay, int normalize,
    double* __restrict__ out, int64_t out_unit_stride) {
  const int u = blockIdx.y;
  const int D8 = D / 8;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = (int)(idx / D8);
  const int d = 8 * (int)(idx - (int64_t)c * D8);
  if (c >= lay.num_chunks(u)) return;
  int lo, hi;
  lay.chunk(u, c, lo, hi);
  const uint4* src =
      reinterpret_cast<const uint4*>(x + (int64_t)u * x_unit_stride + (int64_t)lo * D + d);
  const int64_t rs = D8;  // row stride in 16-byte words
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 0.0;
  auto add_row = [&](const uint4 w) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h[j]);
      a[2 * j] = __dadd_rn(a[2 * j], (double)f.x);
      a[2 * j + 1] = __dadd_rn(a[2 * j + 1], (double)f.y);
    }
  };
  int t = 0;
  const int n = hi - lo;
  for (; t + 8 <= n; t += 8) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(src + (int64_t)(t + k) * rs);
#pragma unroll
    for (int k = 0; k < 8; ++k) add_row(v[k]);
  }
  for (; t < n; ++t) add_row(__ldg(src + (int64_t)t * rs));
  if (normalize) {
    const double r = __dsqrt_rn((double)n);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __ddiv_rn(a[j], r);
  }
  double2* o = reinterpret_cast<double2*>(out + (int64_t)u * out_unit_stride + (int64_t)c * D + d);
#pragma unroll
  for (int j = 0; j < 4; ++j) o[j] = make_double2(a[2 * j], a[2 * j + 1]);
}

}  // namespace dhsa

using namespace dhsa;

extern "C" int dhsa_centroids(int dtype, const void* x, int64_t x_unit_stride, int D, int U,
                              dhsa_layout layout, int normalize, double* out,
                              int64_t out_unit_stride, dhsa_stream_t stream) {
  DHSA_REQUIRE(x && out && D >= 1 && U >= 1, "dhsa_centroids: bad arguments");
  DHSA_REQUIRE(valid_layout(layout) && layout.max_chunks >= 1, "dhsa_centroids: bad layout");
  const int64_t work = (int64_t)layout.max_chunks * D;
  dim3 grid((unsigned)((work + 255) / 256), (unsigned)U);
  cudaStream_t s = (cudaStream_t)stream;
  Layout lay(layout);
  switch (dtype) {
    case DHSA_F64:
      centroids_kernel<double><<<grid, 256, 0, s>>>((const double*)x, x_unit_stride, D, lay, normalize, out,
                                                    out_unit_stride);
      break;
    case DHSA_F32:
      centroids_kernel<float><<<grid, 256, 0, s>>>((const float*)x, x_unit_stride, D, lay, normalize, out,
                                                   out_unit_stride);
      break;
    case DHSA_BF16:
      if (D % 8 == 0 && ((uintptr_t)x & 15) == 0 && x_unit_stride % 8 == 0 &&
          ((uintptr_t)out & 15) == 0 && out_unit_stride % 2 == 0) {
        const int64_t w8 = (int64_t)layout.max_chunks * (D / 8);
        dim3 g8((unsigned)((w8 + 255) / 256), (unsigned)U);
        centroids_bf16x8_kernel<<<g8, 256, 0, s>>>((const __nv_bfloat16*)x, x_unit_stride, D, lay,
                                                   normalize, out, out_unit_stride);
      } else if (D % 2 == 0 && ((uintptr_t)x & 3) == 0 && x_unit_stride % 2 == 0) {
        const int64_t w2 = (int64_t)layout.max_chunks * (D / 2);
        dim3 g2((unsigned)((w2 + 255) / 256), (unsigned)U);
        centroids_bf16x2_kernel<<<g2, 256, 0, s>>>((const __nv_bfloat16*)x, x_unit_stride, D, lay,
                                                   normalize, out, out_unit_stride);
      } else {
        centroids_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)x,
                                                             x_unit_stride, D, lay, normalize, out,
                                                             out_unit_stride);
      }
      break;
    default:
      set_error("dhsa_centroids: unknown dtype %d", dtype);
      return DHSA_EINVAL;
  }
  return check_launch("dhsa_centroids");
}
