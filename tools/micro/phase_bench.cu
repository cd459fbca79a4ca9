// Microbenchmark of select-kernel building blocks on one SM (clock64 cycles):
// __syncthreads, warp shuffle scans, smem atomics + barrier, a block scan,
// a global L2 round trip, a gpu-scope fence.  nvcc -arch=sm_100a -O3 phase_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NT>
__global__ void bench(long long* out, int* g, float* gf) {
  __shared__ unsigned hist[1024 + 32];
  __shared__ int wt[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long t[16];
  int k = 0;
  int acc = tid;
  for (int i = tid; i < 1056; i += NT) hist[i] = 0;
  __syncthreads();
  t[k++] = clock64();
  for (int r = 0; r < 10; ++r) __syncthreads();
  t[k++] = clock64();  // 10 barriers
  for (int r = 0; r < 10; ++r) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, acc, o);
      if (lane >= o) acc += y;
    }
  }
  t[k++] = clock64();  // 10 warp scans (50 dependent shuffles)
  for (int r = 0; r < 10; ++r) {
    atomicAdd(&hist[(acc * 7 + r) & 1023], 1u);
    __syncthreads();
  }
  t[k++] = clock64();  // 10 x (smem atomic + barrier)
  for (int r = 0; r < 10; ++r) {
    int x = acc & 7;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wt[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int v = lane < NT / 32 ? wt[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (lane < NT / 32) wt[lane] = v;
    }
    __syncthreads();
    acc += wt[warp];
    __syncthreads();
  }
  t[k++] = clock64();  // 10 block scans
  float f = 0.f;
  for (int r = 0; r < 10; ++r) f += __ldcg(gf + ((acc + r * 4099) & 0xFFFF));
  acc += (int)f;
  t[k++] = clock64();  // 10 dependent-issue L2 loads (independent addresses)
  for (int r = 0; r < 10; ++r) {
    f = __ldcg(gf + (((int)f + r * 4099 + acc) & 0xFFFF));
  }
  acc += (int)f;
  t[k++] = clock64();  // 10 dependent global loads (chain)
  for (int r = 0; r < 10; ++r) {
    if (tid == 0) g[r] = acc;
    __threadfence();
  }
  t[k++] = clock64();  // 10 store + threadfence
  for (int r = 0; r < 10; ++r) {
    if (tid == 0) asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(g + r), "r"(acc) : "memory");
  }
  t[k++] = clock64();  // 10 st.release (thread 0)
  if (tid == 0) {
    for (int i = 0; i < k; ++i) out[blockIdx.x * 16 + i] = t[i];
    out[blockIdx.x * 16 + 15] = acc;
  }
}

int main() {
  long long* d;
  int* g;
  float* gf;
  cudaMalloc(&d, 16 * 8 * 148);
  cudaMalloc(&g, 4096);
  cudaMalloc(&gf, 65536 * 4);
  cudaMemset(gf, 0, 65536 * 4);
  long long h[16];
  const char* names[] = {"10 x __syncthreads", "10 x warp scan (5 shfl)", "10 x (smem atomic + bar)",
                         "10 x block scan (3 bar)", "10 x L2 load (independent)",
                         "10 x L2 load (dependent chain)", "10 x (store + __threadfence)",
                         "10 x st.release.gpu"};
  for (int nt : {256, 1024}) {
    for (int rep = 0; rep < 3; ++rep) {
      if (nt == 256) bench<256><<<1, 256>>>(d, g, gf);
      else bench<1024><<<1, 1024>>>(d, g, gf);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("NT=%d (cycles per op, one CTA alone)\n", nt);
    for (int i = 0; i < 8; ++i) printf("  %-34s %8.1f\n", names[i], (h[i + 1] - h[i]) / 10.0);
  }
  return 0;
}
