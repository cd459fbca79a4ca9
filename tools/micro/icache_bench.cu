// Cost of executing straight-line code ONCE (instruction-cache misses): a
// kernel body of N independent FFMA chains fully unrolled (16 B per SASS
// instruction), executed once by 8 warps of one CTA; cycles per KB of code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o icache_bench icache_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__global__ void body(float* out, long long* cyc, float s) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    a0 = fmaf(a0, s, 1.0001f * i);
    a1 = fmaf(a1, s, 1.0002f * i);
    a2 = fmaf(a2, s, 1.0003f * i);
    a3 = fmaf(a3, s, 1.0004f * i);
  }
  __syncthreads();
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int N>
void run(float* out, long long* cyc, int grid) {
  long long h[2];
  body<N><<<grid, 256>>>(out, cyc, 0.999f);  // cold: first launch of this code
  cudaDeviceSynchronize();
  cudaMemcpy(&h[0], cyc, 8, cudaMemcpyDeviceToHost);
  body<N><<<grid, 256>>>(out, cyc, 0.999f);  // warm (code in L2 / I$ from the first launch)
  cudaDeviceSynchronize();
  cudaMemcpy(&h[1], cyc, 8, cudaMemcpyDeviceToHost);
  const double kb = 4.0 * N * 16 / 1024;  // ~4 FFMA per iteration
  printf("grid %3d body %6.1f KB: cold %8lld cyc (%5.1f cyc/instr/warp-step), warm %8lld cyc (%5.2f)\n",
         grid, kb, h[0], (double)h[0] / (4 * N), h[1], (double)h[1] / (4 * N));
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 22);
  cudaMalloc(&cyc, 8 * 1024);
  for (int grid : {1, 32, 148}) {
    run<128>(out, cyc, grid);
    run<512>(out, cyc, grid);
    run<1024>(out, cyc, grid);
    run<2048>(out, cyc, grid);
    run<4096>(out, cyc, grid);
  }
  return 0;
}
