// Host<->device transfer of one decode step's inputs / outputs (C3: 393,216 B
// in, 262,144 B out): cudaMemcpyAsync from / to pinned memory vs a kernel that
// reads / writes the mapped pinned buffer directly (zero-copy, 16-byte
// accesses, grid x 256 threads).  Device time per transfer (CUDA events, 200
// repetitions, each followed by a stream sync like an autoregressive loop).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hostcopy_bench hostcopy_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void zc_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const size_t nin = 393216, nout = 262144;
  void *hin, *hout, *din, *dout;
  cudaHostAlloc(&hin, nin, cudaHostAllocMapped);
  cudaHostAlloc(&hout, nout, cudaHostAllocMapped);
  cudaMalloc(&din, nin);
  cudaMalloc(&dout, nout);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 20; ++i) { fn(); cudaStreamSynchronize(s); }
    float tot = 0.f;
    for (int i = 0; i < 200; ++i) {
      cudaEventRecord(e0, s);
      fn();
      cudaEventRecord(e1, s);
      cudaStreamSynchronize(s);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    printf("%-40s %8.2f us  (%s)\n", name, tot / 200 * 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("memcpy H2D 393216 B", [&] { cudaMemcpyAsync(din, hin, nin, cudaMemcpyHostToDevice, s); });
  timeit("memcpy D2H 262144 B", [&] { cudaMemcpyAsync(hout, dout, nout, cudaMemcpyDeviceToHost, s); });
  for (int grid : {16, 48, 148, 296}) {
    char nm[64];
    snprintf(nm, 64, "zero-copy read  H->D grid %d", grid);
    timeit(nm, [&] { zc_copy<<<grid, 256, 0, s>>>((const uint4*)hin, (uint4*)din, nin / 16); });
    snprintf(nm, 64, "zero-copy write D->H grid %d", grid);
    timeit(nm, [&] { zc_copy<<<grid, 256, 0, s>>>((const uint4*)dout, (uint4*)hout, nout / 16); });
  }
  return 0;
}
