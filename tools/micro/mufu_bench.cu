// MUFU exp2 throughput on one SM: ex2.approx.f32 vs ex2.approx.f16x2 vs
// ex2.approx.ftz.bf16x2 (results per clock per SM), 8 warps x 8 independent
// chains.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_bench mufu_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

template <int MODE>
__global__ void bench(float* out, long long* cyc, int iters) {
  float f[8];
  uint32_t h[8];
  for (int k = 0; k < 8; ++k) {
    f[k] = -0.001f * (threadIdx.x + k);
    __half2 x = __floats2half2_rn(f[k], f[k] * 0.5f);
    h[k] = *reinterpret_cast<uint32_t*>(&x);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MODE == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[k]));
      } else if (MODE == 1) {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[k]));
      } else {
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[k]));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
  for (int k = 0; k < 8; ++k) s += f[k] + __uint_as_float(h[k]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1024);
  const int iters = 4096, threads = 256;
  const char* names[] = {"ex2.approx.ftz.f32", "ex2.approx.f16x2", "ex2.approx.ftz.bf16x2"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) bench<0><<<1, threads>>>(out, cyc, iters);
      if (mode == 1) bench<1><<<1, threads>>>(out, cyc, iters);
      if (mode == 2) bench<2><<<1, threads>>>(out, cyc, iters);
      cudaDeviceSynchronize();
    }
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)iters * 8 * threads;  // instructions (per thread-lane)
    const double res = ops * (mode == 0 ? 1 : 2);   // exp2 results
    printf("%-24s %6.2f instr/clk/SM  %6.2f results/clk/SM  (%s)\n", names[mode], ops / c, res / c,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
