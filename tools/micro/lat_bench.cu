// Latency microbenchmark (clock64 cycles per op, one thread timing, 32 CTAs x
// 256 threads resident on separate SMs): warm L2 load chain, cold-page load
// chain (a new 2 MB page per load: TLB miss), st.release.gpu, store +
// __threadfence, cold-page store + fence, __syncthreads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_bench lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void bench(long long* out, int* warm, char* big, size_t page, int npages) {
  const int tid = threadIdx.x;
  long long t[16];
  int k = 0;
  int acc = 0;
  __syncthreads();
  t[k++] = clock64();
  for (int r = 0; r < 10; ++r) __syncthreads();
  t[k++] = clock64();  // 10 barriers
  if (tid == 0) {
    int idx = 0;
    for (int r = 0; r < 10; ++r) idx = __ldcg(warm + ((idx + r * 37) & 1023));
    acc += idx;
  }
  __syncthreads();
  t[k++] = clock64();  // 10 dependent warm-L2 loads
  if (tid == 0) {
    int idx = 0;
    for (int r = 0; r < 10; ++r) {
      const size_t p = (size_t)(blockIdx.x * 10 + r) % npages;
      idx = __ldcg(reinterpret_cast<int*>(big + p * page + (idx & 63) * 4));
    }
    acc += idx;
  }
  __syncthreads();
  t[k++] = clock64();  // 10 dependent cold-page loads
  if (tid == 0)
    for (int r = 0; r < 10; ++r)
      asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(warm + 2048 + blockIdx.x * 16 + r), "r"(acc) : "memory");
  __syncthreads();
  t[k++] = clock64();  // 10 st.release (thread 0)
  for (int r = 0; r < 10; ++r) {
    warm[4096 + blockIdx.x * 256 + tid] = acc + r;
    __threadfence();
  }
  __syncthreads();
  t[k++] = clock64();  // 10 x (every thread stores + fences)
  for (int r = 0; r < 10; ++r) {
    const size_t p = (size_t)(blockIdx.x * 10 + r + 5000) % npages;
    reinterpret_cast<int*>(big + p * page)[tid] = acc;
    __threadfence();
  }
  __syncthreads();
  t[k++] = clock64();  // 10 x cold-page store + fence
  for (int r = 0; r < 10; ++r) {
    const size_t p = (size_t)(blockIdx.x * 10 + r + 9000) % npages;
    reinterpret_cast<int*>(big + p * page)[tid] = acc;
  }
  __syncthreads();
  t[k++] = clock64();  // 10 x cold-page store, no fence
  if (tid == 0) {
    for (int i = 0; i < k; ++i) out[blockIdx.x * 16 + i] = t[i];
    out[blockIdx.x * 16 + 15] = acc;
  }
}

int main() {
  long long* d;
  int* warm;
  char* big;
  const size_t page = 2 << 20;
  const int npages = 20000;  // 40 GB
  cudaMalloc(&d, 16 * 8 * 148);
  cudaMalloc(&warm, 1 << 20);
  cudaMemset(warm, 0, 1 << 20);
  if (cudaMalloc(&big, page * npages) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  const char* names[] = {"__syncthreads", "warm L2 load (dep)", "cold-page load (dep)", "st.release.gpu",
                         "store+threadfence (all thr)", "cold-page store+fence", "cold-page store"};
  for (int grid : {1, 32, 148}) {
    bench<<<grid, 256>>>(d, warm, big, page, npages);
    cudaDeviceSynchronize();
    long long h[16 * 148];
    cudaMemcpy(h, d, sizeof(long long) * 16 * grid, cudaMemcpyDeviceToHost);
    printf("grid %d (cycles per op, CTA 0 / median-ish CTA %d)\n", grid, grid / 2);
    for (int i = 0; i < 7; ++i)
      printf("  %-30s %9.1f %9.1f\n", names[i], (h[i + 1] - h[i]) / 10.0,
             (h[(grid / 2) * 16 + i + 1] - h[(grid / 2) * 16 + i]) / 10.0);
  }
  return 0;
}
