// Small kernels and the error channel of the C ABI.
#include "capi.cuh"

#include <cstring>

namespace dhsa {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

__global__ void advance_kernel(int32_t* gen_count, int U) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < U) gen_count[u] += 1;
}

// S_c = Q_c K_c^T per head in fp64 (chunk_repr.py:97-103): 16x16 output tile
// per CTA, D streamed through shared memory in slabs of 32.
__global__ __launch_bounds__(256) void chunk_scores_kernel(const double* __restrict__ qc,
                                                           const double* __restrict__ kc, int n,
                                                           int m, int D, int64_t qs, int64_t ks,
                                                           double* __restrict__ out,
                                                           int64_t os) {
  __shared__ double a[16][33];
  __shared__ double b[16][33];
  const int h = blockIdx.z;
  const int i0 = blockIdx.y * 16, j0 = blockIdx.x * 16;
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  const double* Q = qc + (int64_t)h * qs;
  const double* K = kc + (int64_t)h * ks;
  double acc = 0.0;
  for (int d0 = 0; d0 < D; d0 += 32) {
    for (int e = threadIdx.x; e < 16 * 32; e += 256) {
      const int r = e / 32, c = e % 32;
      a[r][c] = (i0 + r < n && d0 + c < D) ? Q[(int64_t)(i0 + r) * D + d0 + c] : 0.0;
      b[r][c] = (j0 + r < m && d0 + c < D) ? K[(int64_t)(j0 + r) * D + d0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < 32; ++c) acc = fma(a[ty][c], b[tx][c], acc);
    __syncthreads();
  }
  if (i0 + ty < n && j0 + tx < m) out[(int64_t)h * os + (int64_t)(i0 + ty) * m + j0 + tx] = acc;
}

// f_upsample (masks.py:87-100): one thread per output element.
__global__ void upsample_kernel(const double* __restrict__ sc, const int32_t* __restrict__ bounds,
                                int n, int L, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)L * L) return;
  const int i = (int)(e / L), j = (int)(e - (int64_t)i * L);
  int a = 0, b = n, ci, cj;
  while (b - a > 1) { int m = (a + b) >> 1; if (bounds[m] <= i) a = m; else b = m; }
  ci = a;
  a = 0; b = n;
  while (b - a > 1) { int m = (a + b) >> 1; if (bounds[m] <= j) a = m; else b = m; }
  cj = a;
  out[e] = sc[(int64_t)ci * n + cj];
}

// softmax_row (core.py:69-77): e = exp(s - max s); e / sum e, fp64, one CTA
// per row (block reductions of the max and of the sum).
__global__ __launch_bounds__(256) void softmax_rows_kernel(const double* __restrict__ s,
                                                           int64_t n, double* __restrict__ out) {
  __shared__ double red[8];
  const double* x = s + (int64_t)blockIdx.x * n;
  double* y = out + (int64_t)blockIdx.x * n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double m = -INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += 256) m = fmax(m, x[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) m = fmax(m, red[w]);
  __syncthreads();
  double t = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) {
    const double e = exp(x[i] - m);
    y[i] = e;
    t += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) red[warp] = t;
  __syncthreads();
  t = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) t += red[w];
  for (int64_t i = threadIdx.x; i < n; i += 256) y[i] = y[i] / t;
}

}  // namespace dhsa

using namespace dhsa;

extern "C" int dhsa_softmax_rows(const double* scores, int rows, int64_t n, double* out,
                                 dhsa_stream_t stream) {
  DHSA_REQUIRE(scores && out && rows >= 1 && n >= 1, "dhsa_softmax_rows: bad arguments");
  softmax_rows_kernel<<<rows, 256, 0, (cudaStream_t)stream>>>(scores, n, out);
  return check_launch("dhsa_softmax_rows");
}

extern "C" int dhsa_upsample(const double* scores, const int32_t* bounds, int n, int L,
                             double* out, dhsa_stream_t stream) {
  DHSA_REQUIRE(scores && bounds && out && n >= 1 && L >= 1, "dhsa_upsample: bad arguments");
  const int64_t total = (int64_t)L * L;
  upsample_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      scores, bounds, n, L, out);
  return check_launch("dhsa_upsample");
}

extern "C" const char* dhsa_last_error(void) { return g_err; }

extern "C" int dhsa_version(void) { return 1; }

extern "C" int dhsa_decode_advance(int32_t* gen_count, int U, dhsa_stream_t stream) {
  DHSA_REQUIRE(gen_count && U >= 1, "dhsa_decode_advance: bad arguments");
  advance_kernel<<<(U + 255) / 256, 256, 0, (cudaStream_t)stream>>>(gen_count, U);
  return check_launch("dhsa_decode_advance");
}

extern "C" int dhsa_chunk_scores(const double* qc, const double* kc, int n, int m, int D,
                                 int heads, int64_t qc_head_stride, int64_t kc_head_stride,
                                 double* out, int64_t out_head_stride, dhsa_stream_t stream) {
  DHSA_REQUIRE(qc && kc && out && n >= 1 && m >= 1 && D >= 1 && heads >= 1,
               "dhsa_chunk_scores: bad arguments");
  dim3 grid((unsigned)((m + 15) / 16), (unsigned)((n + 15) / 16), (unsigned)heads);
  chunk_scores_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(qc, kc, n, m, D, qc_head_stride,
                                                              kc_head_stride, out,
                                                              out_head_stride);
  return check_launch("dhsa_chunk_scores");
}
