// H2D / D2H of one decode step's buffers split over K streams (copy engines):
// fork-join with events around the split copies, device time per transfer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hostcopy_split hostcopy_split.cu
#include <cstdio>
#include <cuda_runtime.h>

int main() {
  const size_t nin = 393216, nout = 262144;
  void *hin, *hout, *din, *dout;
  cudaHostAlloc(&hin, nin, cudaHostAllocDefault);
  cudaHostAlloc(&hout, nout, cudaHostAllocDefault);
  cudaMalloc(&din, nin);
  cudaMalloc(&dout, nout);
  cudaStream_t s, side[8];
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int i = 0; i < 8; ++i) cudaStreamCreateWithFlags(&side[i], cudaStreamNonBlocking);
  cudaEvent_t e0, e1, fork, join[8];
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
  for (int i = 0; i < 8; ++i) cudaEventCreateWithFlags(&join[i], cudaEventDisableTiming);
  auto split_copy = [&](void* dst, const void* src, size_t n, cudaMemcpyKind kind, int k) {
    if (k == 1) {
      cudaMemcpyAsync(dst, src, n, kind, s);
      return;
    }
    cudaEventRecord(fork, s);
    const size_t part = (n / k + 255) / 256 * 256;
    for (int i = 0; i < k; ++i) {
      const size_t off = part * i;
      if (off >= n) break;
      const size_t len = off + part > n ? n - off : part;
      cudaStreamWaitEvent(side[i], fork, 0);
      cudaMemcpyAsync((char*)dst + off, (const char*)src + off, len, kind, side[i]);
      cudaEventRecord(join[i], side[i]);
      cudaStreamWaitEvent(s, join[i], 0);
    }
  };
  for (int k : {1, 2, 3, 4, 8}) {
    for (int dir = 0; dir < 2; ++dir) {
      float tot = 0.f;
      for (int it = 0; it < 220; ++it) {
        cudaEventRecord(e0, s);
        if (dir == 0) split_copy(din, hin, nin, cudaMemcpyHostToDevice, k);
        else split_copy(hout, dout, nout, cudaMemcpyDeviceToHost, k);
        cudaEventRecord(e1, s);
        cudaStreamSynchronize(s);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 20) tot += ms;
      }
      printf("%s split %d: %7.2f us\n", dir == 0 ? "H2D 393216 B" : "D2H 262144 B", k, tot / 200 * 1e3);
    }
  }
  return 0;
}
