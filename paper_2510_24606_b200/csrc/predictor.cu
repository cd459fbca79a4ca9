// Boundary-predictor inference on the GPU.
//
// Reference: predictor.predict_sequence / boundary_scores (predictor.py:
// 101-117 _mha_pool_forward, 151-161 _fuse_forward, 198-207 _forward,
// 270-303): for every position i the w keys ending at i and the w keys after
// i are encoded by one shared multi-head self-attention layer with mean
// pooling, the two encodings are fused [l, r, |l - r|, l * r, cos] and a
// 2-layer MLP gives the boundary probability.  Everything in fp64 like the
// reference.  Restructured for the GPU: the per-token projections Q|K|V =
// keys [Wq|Wk|Wv] are one GEMM over the L tokens (a window re-uses its
// tokens' projections), each window's attention + mean is one warp, the
// pooled encodings are (mean_a Ocat[a]) Wo (one GEMM over windows, since the
// mean commutes with Wo), windows are shared by the positions that use them
// (left window of i = window i-w+1, right window = window i+1), then the
// fusion rows and one GEMM with W1 whose ReLU / W2 / sigmoid head is a warp
// per row.
#include "capi.cuh"

namespace dhsa {

// C[M][N] = A[M][K] B[K][N] (+ bias[N]), fp64, row-major, 64 x 64 tiles,
// 256 threads x 4 x 4 register tile, K in slabs of 16.
__global__ __launch_bounds__(256) void gemm_f64_kernel(const double* __restrict__ A,
                                                       const double* __restrict__ B,
                                                       const double* __restrict__ bias,
                                                       double* __restrict__ C, int M, int N,
                                                       int K) {
  __shared__ double sa[16][65];
  __shared__ double sb[16][65];
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 64 * 16; e += 256) {
      const int r = e / 16, c = e % 16;
      sa[c][r] = (m0 + r < M && k0 + c < K) ? A[(int64_t)(m0 + r) * K + k0 + c] : 0.0;
      const int kr = e / 64, nc = e % 64;
      sb[kr][nc] = (k0 + kr < K && n0 + nc < N) ? B[(int64_t)(k0 + kr) * N + n0 + nc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sa[c][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = sb[c][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = m0 + ty + 16 * a, c = n0 + tx + 16 * b;
      if (r < M && c < N) C[(int64_t)r * N + c] = acc[a][b] + (bias ? bias[c] : 0.0);
    }
}

// One warp per window start t: per head, the w x w scores of the window's
// projected tokens (lane = (a, b) pair), row softmax, then the head slice of
// mean_a Ocat[a] (lane = dimension within the head).  qkv: [L][3d] rows
// (Q | K | V); out: [nwin][d].
__global__ void window_attn_kernel(const double* __restrict__ qkv, int nwin, int d, int w,
                                   int heads, double* __restrict__ out) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= nwin) return;
  const int dh = d / heads;
  const double inv = 1.0 / sqrt((double)dh);
  const int a = lane / w, b = lane % w;
  const bool pair = lane < w * w;
  for (int h = 0; h < heads; ++h) {
    double sc = -INFINITY;
    if (pair) {
      const double* qr = qkv + (int64_t)(t + a) * 3 * d + h * dh;
      const double* kr = qkv + (int64_t)(t + b) * 3 * d + d + h * dh;
      double s = 0.0;
      for (int e = 0; e < dh; ++e) s = fma(qr[e], kr[e], s);
      sc = s * inv;
    }
    // softmax over b within each row a (lanes a*w .. a*w+w-1)
    double mx = sc;
    for (int j = 0; j < w; ++j) mx = fmax(mx, __shfl_sync(0xffffffffu, sc, (a * w + j) & 31));
    const double ex = pair ? exp(sc - mx) : 0.0;
    double den = 0.0;
    for (int j = 0; j < w; ++j) den += __shfl_sync(0xffffffffu, ex, (a * w + j) & 31);
    const double att = pair ? ex / den : 0.0;
    // mean over a of sum_b att[a][b] V[t+b][h*dh + e]; lane = e
    double o = 0.0;
    for (int aa = 0; aa < w; ++aa) {
      double row = 0.0;
      for (int bb = 0; bb < w; ++bb) {
        const double p = __shfl_sync(0xffffffffu, att, aa * w + bb);
        if (lane < dh) row = fma(p, qkv[(int64_t)(t + bb) * 3 * d + 2 * d + h * dh + lane], row);
      }
      o += row;
    }
    if (lane < dh) out[(int64_t)t * d + h * dh + lane] = o / (double)w;
  }
}

// Fusion rows [l, r, |l - r|, l * r, cos] (4d + 1) for positions
// i = w-1 .. L-w-1 (predictor.py predictable_positions): l = pooled[i-w+1], r = pooled[i+1].  One warp per row.
__global__ void fuse_kernel(const double* __restrict__ pooled, int npos, int d, int w,
                            double* __restrict__ H) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= npos) return;
  const int i = r + w - 1;
  const double* kl = pooled + (int64_t)(i - w + 1) * d;
  const double* kr = pooled + (int64_t)(i + 1) * d;
  double* h = H + (int64_t)r * (4 * d + 1);
  double dot = 0.0, nl = 0.0, nr = 0.0;
  for (int e = lane; e < d; e += 32) {
    const double x = kl[e], y = kr[e];
    h[e] = x;
    h[d + e] = y;
    h[2 * d + e] = fabs(x - y);
    h[3 * d + e] = x * y;
    dot = fma(x, y, dot);
    nl = fma(x, x, nl);
    nr = fma(y, y, nr);
  }
  dot = warp_sum(dot);
  nl = warp_sum(nl);
  nr = warp_sum(nr);
  if (lane == 0) {
    const double den = sqrt(nl) * sqrt(nr);
    h[4 * d] = den > 0.0 ? fmin(1.0, fmax(-1.0, dot / den)) : 0.0;
  }
}

// p = sigmoid(relu(z1) . W2 + b2) per row; one warp per row.
__global__ void mlp_head_kernel(const double* __restrict__ Z1, int npos, int hidden,
                                const double* __restrict__ W2, double b2,
                                double* __restrict__ p) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= npos) return;
  double s = 0.0;
  for (int j = lane; j < hidden; j += 32) s = fma(fmax(Z1[(int64_t)r * hidden + j], 0.0), W2[j], s);
  s = warp_sum(s) + b2;
  if (lane == 0) p[r] = 1.0 / (1.0 + exp(-s));
}

static void gemm(const double* A, const double* B, const double* bias, double* C, int M, int N,
                 int K, cudaStream_t s) {
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64));
  gemm_f64_kernel<<<grid, 256, 0, s>>>(A, B, bias, C, M, N, K);
}

}  // namespace dhsa

using namespace dhsa;

extern "C" int64_t dhsa_predictor_workspace_size(int L, int d, int window, int hidden) {
  if (L < 2 * window + 1 || d < 1 || window < 1 || hidden < 1) return -1;
  const int64_t nwin = L - window + 1, npos = L - 2 * window + 1;
  return 8 * ((int64_t)L * 3 * d + nwin * d * 2 + npos * (4 * (int64_t)d + 1) +
              npos * (int64_t)hidden);
}

extern "C" int dhsa_predictor_forward(const double* keys, int L, int d, int window, int heads,
                                      int hidden, const double* wqkv, const double* wo,
                                      const double* w1, const double* b1, const double* w2,
                                      double b2, void* workspace, double* probs,
                                      dhsa_stream_t stream) {
  DHSA_REQUIRE(keys && wqkv && wo && w1 && b1 && w2 && workspace && probs,
               "dhsa_predictor_forward: null pointer");
  DHSA_REQUIRE(L >= 2 * window + 1, "need at least %d keys, got %d", 2 * window + 1, L);
  DHSA_REQUIRE(heads >= 1 && d % heads == 0 && d / heads <= 32 && window >= 1 &&
                   window * window <= 32 && hidden >= 1,
               "dhsa_predictor_forward: unsupported shape (d/heads <= 32, window^2 <= 32)");
  cudaStream_t s = (cudaStream_t)stream;
  const int nwin = L - window + 1, npos = L - 2 * window + 1;
  double* qkv = (double*)workspace;
  double* meano = qkv + (int64_t)L * 3 * d;
  double* pooled = meano + (int64_t)nwin * d;
  double* H = pooled + (int64_t)nwin * d;
  double* Z1 = H + (int64_t)npos * (4 * d + 1);
  gemm(keys, wqkv, nullptr, qkv, L, 3 * d, d, s);                        // Q | K | V per token
  window_attn_kernel<<<(nwin + 7) / 8, 256, 0, s>>>(qkv, nwin, d, window, heads, meano);
  gemm(meano, wo, nullptr, pooled, nwin, d, d, s);                       // (mean Ocat) Wo
  fuse_kernel<<<(npos + 7) / 8, 256, 0, s>>>(pooled, npos, d, window, H);
  gemm(H, w1, b1, Z1, npos, hidden, 4 * d + 1, s);                       // h W1 + b1
  mlp_head_kernel<<<(npos + 7) / 8, 256, 0, s>>>(Z1, npos, hidden, w2, b2, probs);
  return check_launch("dhsa_predictor_forward");
}
