// Shared device helpers for libdhsa_b200 (sm_100a).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dhsa_b200.h"

namespace dhsa {

using SplitCand = dhsa_split_cand;
static_assert(sizeof(SplitCand) == 24, "candidate record is 24 bytes");

// ----------------------------------------------------------------- dtypes --

template <typename T> struct Acc { using type = float; };
template <> struct Acc<double> { using type = double; };

__device__ __forceinline__ double to_f64(double x) { return x; }
__device__ __forceinline__ double to_f64(float x) { return (double)x; }
__device__ __forceinline__ double to_f64(__nv_bfloat16 x) { return (double)__bfloat162float(x); }

template <typename A> __device__ __forceinline__ A cvt(double x);
template <> __device__ __forceinline__ double cvt<double>(double x) { return x; }
template <> __device__ __forceinline__ float cvt<float>(double x) { return (float)x; }

__device__ __forceinline__ float to_acc(float x) { return x; }
__device__ __forceinline__ double to_acc_d(double x) { return x; }

template <typename T> __device__ __forceinline__ T from_acc(typename Acc<T>::type x);
template <> __device__ __forceinline__ double from_acc<double>(double x) { return x; }
template <> __device__ __forceinline__ float from_acc<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// ------------------------------------------------------------ chunk layout --
// Prompt chunks of unit u (dhsa_layout in dhsa_b200.h).
struct Layout {
  const int32_t* bounds;
  int64_t bstride;
  const int32_t* nchunks;
  const int32_t* plen;
  int32_t block;

  __host__ __device__ Layout() : bounds(nullptr), bstride(0), nchunks(nullptr), plen(nullptr), block(0) {}
  __host__ Layout(const dhsa_layout& l)
      : bounds(l.bounds), bstride(l.bounds_stride), nchunks(l.nchunks), plen(l.plen),
        block(l.block) {}

  __device__ __forceinline__ int prompt_len(int u) const { return plen[u]; }
  __device__ __forceinline__ int num_chunks(int u) const {
    if (bounds) return nchunks[u];
    int p = plen[u];
    return (p + block - 1) / block;
  }
  __device__ __forceinline__ void chunk(int u, int c, int& lo, int& hi) const {
    if (bounds) {
      const int32_t* b = bounds + (int64_t)u * bstride;
      lo = b[c];
      hi = b[c + 1];
    } else {
      lo = c * block;
      hi = min(lo + block, plen[u]);
    }
  }
};

// ------------------------------------------------------------ sort keys --
// Order-preserving map of a finite double to uint64 (larger key = larger
// value); -0.0 is canonicalised to +0.0 because numpy compares them equal
// (masks.py:119 argsort of -scores).
__device__ __forceinline__ uint64_t order_key(double x) {
  x = (x == 0.0) ? 0.0 : x;
  uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// ------------------------------------------------------------- reductions --
__device__ __forceinline__ double shfl_xor_d(double v, int o) {
  return __shfl_xor_sync(0xffffffffu, v, o);
}

// Transpose-reduce NV per-lane partial sums so that every lane ends with one
// complete 32-lane sum (value index = bits of the lane id, see below) using
// NV-1 shuffles instead of 5*NV.  NV is a power of two <= 32.  After the
// call v[0] of lane l holds the total of value index
//   idx(l) = (l >> (5 - log2 NV)) & (NV - 1).
template <int NV>
__device__ __forceinline__ double transpose_reduce(double (&v)[NV], int lane) {
  int n = NV;
  int o = 16;
#pragma unroll
  for (int step = 0; step < 5; ++step) {
    if (n > 1) {
      const int half = n >> 1;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int k = 0; k < NV / 2; ++k) {
        if (k < half) {
          double send = up ? v[k] : v[k + half];
          double keep = up ? v[k + half] : v[k];
          v[k] = keep + shfl_xor_d(send, o);
        }
      }
      n = half;
    } else {
      v[0] += shfl_xor_d(v[0], o);
    }
    o >>= 1;
  }
  return v[0];
}

template <typename A>
__device__ __forceinline__ A warp_sum(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------ mbarrier / TMA PTX --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// The same with an L2 eviction-priority policy (createpolicy): streamed data
// that is read once per step (K/V tiles, sketch slices) is marked evict-first
// so the step's small, re-read state (approximate scores, tile lists, fp64
// centroids of the re-scored chunks, flags, code) stays in L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 int x, int y, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion on an mbarrier.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// ----------------------------------------------------- debug timestamps --
// DHSA_DEBUG_TIMING=<device address of a uint64 buffer> makes the decode
// kernels record %globaltimer at phase boundaries (tools/select_phases.py):
// select CTAs at [16 u + k], sketch CTAs at kDbgSketch + 2 b (+1 = end),
// attention CTAs at kDbgAttn + 4 b (+1 first tile, +2 end).
constexpr int kDbgSketch = 65536;
constexpr int kDbgAttn = 131072;
constexpr int kDbgSelectClk = 196608;
constexpr int kDbgSketchPh = 229376;   // sketch CTAs: first q staged, first tile, last tile  // select CTAs: clock64() at the same phase points
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------ programmatic launch + flags --
// Let the next kernel in the stream (launched with programmatic stream
// serialization) start once every CTA of this grid has executed this.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Wait until the preceding grid (programmatic dependency) has completed and
// its memory operations are visible.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(int32_t* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Release-add: prior writes of this thread (and, via a preceding warp/CTA
// barrier, of its peers) become visible before the increment.
__device__ __forceinline__ void red_add_release(int32_t* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Thread-level spin until *p >= target (acquire), with backoff.
// select -> attention item flags: 0 = not ready; 1 + n (n < kReadyFinal - 1)
// = the first n tiles of the item are final (the chunks the certified select
// keeps whole, published before the exact refinement); kReadyFinal = every
// tile and the tile count are final.
constexpr int kReadyFinal = 1 << 30;

__device__ __forceinline__ void spin_geq(const int32_t* p, int target) {
  while (ld_acquire(p) < target) __nanosleep(64);
}

// ---------------------------------------------------------- mma.sync PTX --
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                          uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D(16x8,f32) += A(16x16,bf16,row) * B(16x8,bf16,col)
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// D(16x8,f32) += A(16x16,f16,row) * B(16x8,f16,col)
__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                        uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

}  // namespace dhsa
