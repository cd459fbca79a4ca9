// Split-KV bookkeeping shared by the attention kernels: partial (m, l, acc)
// records and the in-kernel merge done by the last CTA of an item.
#pragma once

#include "common.cuh"

namespace dhsa {

// Partial record of one split for one head: [m, l, acc[D]] in accumulator
// precision.  m is in the log2 domain of the scaled scores.
template <typename A>
__device__ __forceinline__ A* partial_ptr(void* ws, int item, int split, int splits, int h,
                                          int GH, int D) {
  return reinterpret_cast<A*>(ws) + (((int64_t)item * splits + split) * GH + h) * (D + 2);
}

template <typename A> __device__ __forceinline__ A exp2_acc(A x);
template <> __device__ __forceinline__ float exp2_acc<float>(float x) { return exp2f(x); }
template <> __device__ __forceinline__ double exp2_acc<double>(double x) { return exp2(x); }

template <typename A> __device__ __forceinline__ A ld_cg(const A* p);
template <> __device__ __forceinline__ float ld_cg<float>(const float* p) { return __ldcg(p); }
template <> __device__ __forceinline__ double ld_cg<double>(const double* p) { return __ldcg(p); }

// Called by every thread of the CTA after it has written its partials.
// Returns true in the CTA that must perform the merge (the last to finish).
__device__ __forceinline__ bool split_arrive(int32_t* counters, int item, int splits) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(&counters[item], 1);
    s_last = (prev == splits - 1);
    if (s_last) counters[item] = 0;  // re-arm for the next launch / graph replay
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

// Merge the `splits` partial records of `item` and write out[q_row][d], or,
// when `rec_out` is given, one merged (m, l, acc) record per q row (the
// sequence-sharded split-KV path merges those across GPUs, splitkv.cu).
// The m of every record is in log2 units (scores * log2(e) / sqrt(D)).
template <typename T, typename A>
__device__ void merge_partials(const void* ws, int item, int splits, int GH, int D, T* out,
                               A* rec_out = nullptr) {
  for (int hd = threadIdx.x; hd < GH * D; hd += blockDim.x) {
    const int h = hd / D, d = hd - h * D;
    A mstar = -INFINITY;
    for (int s = 0; s < splits; ++s) {
      const A* p = partial_ptr<A>(const_cast<void*>(ws), item, s, splits, h, GH, D);
      mstar = fmax(mstar, ld_cg(p));
    }
    A l = 0, acc = 0;
    for (int s = 0; s < splits; ++s) {
      const A* p = partial_ptr<A>(const_cast<void*>(ws), item, s, splits, h, GH, D);
      const A m = ld_cg(p);
      if (m == -INFINITY) continue;
      const A w = exp2_acc<A>(m - mstar);
      l += w * ld_cg(p + 1);
      acc += w * ld_cg(p + 2 + d);
    }
    if (rec_out) {
      A* r = rec_out + ((int64_t)item * GH + h) * (D + 2);
      if (d == 0) {
        r[0] = mstar;
        r[1] = l;
      }
      r[2 + d] = acc;
    } else {
      out[((int64_t)item * GH + h) * D + d] = from_acc<T>(acc / l);
    }
  }
}

}  // namespace dhsa
