// Mask-quality metrics of the reference harness on the device, fp64
// (harness.py:265-285 attention_mass_recall /
// output_fidelity, core.py:122-152 causal_attention_probs /
// cosine_similarity, harness.py:288-306 head aggregation).  These serve the
// drop-in harness API at the reference's shapes; the batched engines use
// dhsa_row_quality on the tcgen05 kernel's row statistics instead.
#include "capi.cuh"

namespace dhsa {

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ double warp_max(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// causal_attention_probs (core.py:122-136): row i holds softmax(q_i . k_j *
// (1/sqrt(d))) over j <= i (the reference multiplies by the reciprocal), and
// zeros above the diagonal.  One 256-thread CTA per row; each thread owns
// keys j = t, t + 256, ... (sequential fp64 dot over d).
__global__ __launch_bounds__(256) void causal_probs_kernel(const double* __restrict__ q,
                                                           const double* __restrict__ k, int L,
                                                           int d, double inv_sqrt_d,
                                                           double* __restrict__ out) {
  __shared__ double red[8];
  const int i = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* qi = q + (int64_t)i * d;
  double* y = out + (int64_t)i * L;
  double m = -INFINITY;
  for (int j = threadIdx.x; j <= i; j += 256) {
    const double* kj = k + (int64_t)j * d;
    double s = 0.0;
    for (int c = 0; c < d; ++c) s = fma(kj[c], qi[c], s);
    s *= inv_sqrt_d;
    y[j] = s;
    m = fmax(m, s);
  }
  m = warp_max(m);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) m = fmax(m, red[w]);
  __syncthreads();
  double t = 0.0;
  for (int j = threadIdx.x; j <= i; j += 256) {
    const double e = exp(y[j] - m);
    y[j] = e;
    t += e;
  }
  t = warp_sum(t);
  if (lane == 0) red[warp] = t;
  __syncthreads();
  t = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) t += red[w];
  for (int j = threadIdx.x; j < L; j += 256) y[j] = j <= i ? y[j] / t : 0.0;
}

// attention_mass_recall's per-row fraction (harness.py:271-276): one warp
// per row, total = sum_{j <= i} P[i, j], selected = sum_{j in row} P[i, j].
__global__ __launch_bounds__(256) void mask_recall_kernel(const double* __restrict__ P, int64_t ld,
                                                          int L, const int64_t* __restrict__ ptr,
                                                          const int32_t* __restrict__ idx,
                                                          double* __restrict__ frac) {
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= L) return;
  const double* p = P + (int64_t)i * ld;
  double tot = 0.0, sel = 0.0;
  for (int j = lane; j <= i; j += 32) tot += p[j];
  for (int64_t e = ptr[i] + lane; e < ptr[i + 1]; e += 32) sel += p[idx[e]];
  tot = warp_sum(tot);
  sel = warp_sum(sel);
  if (lane == 0) frac[i] = tot > 0.0 ? sel / tot : 0.0;
}

// cosine_similarity (core.py:139-152) of row pairs: 0 when a norm is zero,
// clamped to [-1, 1].  One warp per row.
__global__ __launch_bounds__(256) void row_cosine_kernel(const double* __restrict__ a,
                                                         const double* __restrict__ b,
                                                         int64_t rows, int d,
                                                         double* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const double* x = a + r * d;
  const double* y = b + r * d;
  double xx = 0.0, yy = 0.0, xy = 0.0;
  for (int c = lane; c < d; c += 32) {
    xx = fma(x[c], x[c], xx);
    yy = fma(y[c], y[c], yy);
    xy = fma(x[c], y[c], xy);
  }
  xx = warp_sum(xx);
  yy = warp_sum(yy);
  xy = warp_sum(xy);
  if (lane == 0) {
    const double na = sqrt(xx), nb = sqrt(yy);
    out[r] = (na == 0.0 || nb == 0.0) ? 0.0 : fmin(1.0, fmax(-1.0, xy / (na * nb)));
  }
}

// Deterministic mean of n doubles (one CTA, fixed reduction tree).
__global__ __launch_bounds__(256) void mean_kernel(const double* __restrict__ x, int64_t n,
                                                   double* __restrict__ out) {
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < n; e += 256) s += x[e];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    out[0] = t / (double)n;
  }
}

// aggregated_chunk_scores' reduction over heads (harness.py:302-306):
// max, or mean = (((s_0 + s_1) + s_2) + ...) / H like numpy's axis-0 mean.
__global__ __launch_bounds__(256) void stack_reduce_kernel(const double* __restrict__ x, int H,
                                                           int64_t n, int agg,
                                                           double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (e >= n) return;
  double r = x[e];
  for (int h = 1; h < H; ++h) r = agg == DHSA_AGG_MAX ? fmax(r, x[(int64_t)h * n + e])
                                                      : r + x[(int64_t)h * n + e];
  out[e] = agg == DHSA_AGG_MAX ? r : r / (double)H;
}

}  // namespace dhsa

using namespace dhsa;

extern "C" int dhsa_causal_probs(const double* q, const double* k, int L, int d, double* out,
                                 dhsa_stream_t stream) {
  DHSA_REQUIRE(q && k && out && L >= 1 && d >= 1, "dhsa_causal_probs: bad arguments");
  causal_probs_kernel<<<L, 256, 0, (cudaStream_t)stream>>>(q, k, L, d, 1.0 / sqrt((double)d),
                                                           out);
  return check_launch("dhsa_causal_probs");
}

extern "C" int dhsa_mask_recall(const double* probs, int64_t ld, int L, const int64_t* row_ptr,
                                const int32_t* idx, double* frac, dhsa_stream_t stream) {
  DHSA_REQUIRE(probs && row_ptr && idx && frac && L >= 1 && ld >= L,
               "dhsa_mask_recall: bad arguments");
  mask_recall_kernel<<<(L + 7) / 8, 256, 0, (cudaStream_t)stream>>>(probs, ld, L, row_ptr, idx,
                                                                    frac);
  return check_launch("dhsa_mask_recall");
}

extern "C" int dhsa_row_cosine(const double* a, const double* b, int64_t rows, int d, double* out,
                               dhsa_stream_t stream) {
  DHSA_REQUIRE(a && b && out && rows >= 1 && d >= 1, "dhsa_row_cosine: bad arguments");
  row_cosine_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, (cudaStream_t)stream>>>(a, b, rows, d,
                                                                                 out);
  return check_launch("dhsa_row_cosine");
}

extern "C" int dhsa_mean(const double* x, int64_t n, double* out, dhsa_stream_t stream) {
  DHSA_REQUIRE(x && out && n >= 1, "dhsa_mean: bad arguments");
  mean_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(x, n, out);
  return check_launch("dhsa_mean");
}

extern "C" int dhsa_stack_reduce(const double* x, int H, int64_t n, int agg, double* out,
                                 dhsa_stream_t stream) {
  DHSA_REQUIRE(x && out && H >= 1 && n >= 1 && (agg == DHSA_AGG_MAX || agg == DHSA_AGG_MEAN),
               "dhsa_stack_reduce: bad arguments");
  stack_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, H, n, agg,
                                                                                     out);
  return check_launch("dhsa_stack_reduce");
}
