// Device building blocks of the exact chunk walk (select.cu, decode_fused.cu).
//
// The reference selection (masks.topk_row, masks.py:103-122, on the
// block-constant upsampled row) keeps, besides self, the first R = keep-1
// tokens of the order (score desc, token index asc).  Over chunks this is:
// every chunk with key > T whole, chunks with key == T in index order until R
// is used (the last one possibly partially), nothing below T.  T and the
// residual are found by an MSB-first radix select in which every chunk counts
// with its token length ("weighted" select).
#pragma once

#include "common.cuh"

namespace dhsa {

struct WalkShared {
  uint32_t hist[3][256];  // triple-buffered: one barrier per radix pass
  int warp_tot[33];
  uint32_t digit, rrem, done;
};

template <int NT>
__device__ __forceinline__ int block_scan_excl(int v, WalkShared& sh, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh.warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int t = lane < NT / 32 ? sh.warp_tot[lane] : 0;
    int w = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) sh.warp_tot[lane] = w - t;
    if (lane == 31) sh.warp_tot[32] = w;
  }
  __syncthreads();
  const int res = sh.warp_tot[warp] + x - v;
  total = sh.warp_tot[32];
  __syncthreads();
  return res;
}

template <int NT>
__device__ __forceinline__ int block_sum(int v, WalkShared& sh) {
  int total;
  block_scan_excl<NT>(v, sh, total);
  return total;
}

// Weighted MSB-first radix select.  On return (uniform over the CTA):
// chunks with (key & mask) > prefix are wholly inside the first R tokens,
// chunks with (key & mask) == prefix share the residual `rrem` in index
// order, all others are outside.  Requires 0 < R < sum of lens.
// Leading bytes shared by every weighted key are skipped (one AND/OR
// reduction); histograms are triple-buffered and scanned redundantly by every
// warp, so each pass costs a single barrier.
template <int NT, typename K>
__device__ void radix_threshold(const K* keys, const int32_t* lens, int n, uint32_t R,
                                WalkShared& sh, K& prefix, K& mask, uint32_t& rrem) {
  constexpr int BITS = 8 * sizeof(K);
  __shared__ K s_and, s_or;
  K kand = ~(K)0, kor = 0;
  for (int c = threadIdx.x; c < n; c += NT) {
    if (lens[c] > 0) {
      kand &= keys[c];
      kor |= keys[c];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kand &= __shfl_xor_sync(0xffffffffu, kand, o);
    kor |= __shfl_xor_sync(0xffffffffu, kor, o);
  }
  if (threadIdx.x == 0) {
    s_and = ~(K)0;
    s_or = 0;
  }
  for (int b = threadIdx.x; b < 256; b += NT) sh.hist[0][b] = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    if constexpr (sizeof(K) == 8) {
      atomicAnd(reinterpret_cast<unsigned long long*>(&s_and), (unsigned long long)kand);
      atomicOr(reinterpret_cast<unsigned long long*>(&s_or), (unsigned long long)kor);
    } else {
      atomicAnd(reinterpret_cast<unsigned int*>(&s_and), (unsigned int)kand);
      atomicOr(reinterpret_cast<unsigned int*>(&s_or), (unsigned int)kor);
    }
  }
  __syncthreads();
  const K diff = s_and ^ s_or;  // bits that are not common to all weighted keys
  int top = BITS - 8;
  while (top > 0 && ((diff >> top) & (K)0xFF) == 0) top -= 8;
  mask = top + 8 >= BITS ? (K)0 : (~(K)0 << (top + 8));
  prefix = s_and & mask;
  rrem = R;
  const int lane = threadIdx.x & 31;
  int buf = 0;
  for (int shift = top; shift >= 0; shift -= 8) {
    uint32_t* h = sh.hist[buf];
    // zero the buffer of the next pass (last read two passes ago)
    uint32_t* hn = sh.hist[buf == 2 ? 0 : buf + 1];
    for (int b = threadIdx.x; b < 256; b += NT) hn[b] = 0;
    for (int c = threadIdx.x; c < n; c += NT) {
      const K k = keys[c];
      const int len = lens[c];
      if ((k & mask) == prefix && len > 0) atomicAdd(&h[(k >> shift) & 255], (uint32_t)len);
    }
    __syncthreads();
    // every warp scans the histogram redundantly: no broadcast barrier
    uint32_t w[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      w[j] = h[255 - 8 * lane - j];
      sum += w[j];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - sum;
    const unsigned hit = __ballot_sync(0xffffffffu, excl < rrem && rrem <= incl);
    const int f = __ffs(hit) - 1;
    uint32_t digit = 0, nr = 0, dn = 0;
    if (lane == f) {
      uint32_t cum = excl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (cum + w[j] >= rrem) {
          digit = 255 - 8 * lane - j;
          nr = rrem - cum;
          dn = (rrem - cum == w[j]);
          break;
        }
        cum += w[j];
      }
    }
    digit = __shfl_sync(0xffffffffu, digit, f);
    nr = __shfl_sync(0xffffffffu, nr, f);
    dn = __shfl_sync(0xffffffffu, dn, f);
    prefix |= (K)digit << shift;
    mask |= (K)0xFF << shift;
    rrem = nr;
    buf = buf == 2 ? 0 : buf + 1;
    if (dn) break;  // the whole bucket is kept: no finer split needed
  }
  __syncthreads();  // callers reuse keys/lens/hist after this
}

// Emit tiles of <= tile_tokens tokens for per-chunk takes (tokens taken from
// each chunk's start, in lens[]), in chunk order, then the self tile; the
// first `base` tiles of the row were written before (two-phase emission).
template <int NT, class View>
__device__ void emit_takes(const View& view, const int32_t* takes, int n, int row,
                           int tile_tokens, int32_t* out, int64_t cap, int32_t* ntiles_out,
                           WalkShared& sh, int base = 0) {
  const int tid = threadIdx.x;
  const int cpt = (n + NT - 1) / NT;
  const int c0 = min(tid * cpt, n), c1 = min(c0 + cpt, n);
  int ntile_local = 0;
  for (int c = c0; c < c1; ++c) ntile_local += (takes[c] + tile_tokens - 1) / tile_tokens;
  int tiles_total;
  int off = base + block_scan_excl<NT>(ntile_local, sh, tiles_total);
  tiles_total += base;  // tiles [0, base) were emitted earlier
  for (int c = c0; c < c1; ++c) {
    const int take = takes[c];
    if (take <= 0) continue;
    int lo, len;
    view.chunk(c, lo, len);
    for (int t = 0; t < take; t += tile_tokens) {
      if (off < cap) {
        out[2 * off] = lo + t;
        out[2 * off + 1] = min(tile_tokens, take - t);
      }
      ++off;
    }
  }
  if (tid == 0) {
    if (tiles_total + 1 > cap) {
      *ntiles_out = -1;  // capacity error, reported by the host wrapper
    } else {
      out[2 * tiles_total] = row;  // self (masks.py:120-121)
      out[2 * tiles_total + 1] = 1;
      *ntiles_out = tiles_total + 1;
    }
  }
  __syncthreads();
}

// Turn (prefix, mask, rrem) into per-chunk takes, written back into lens[].
// R == 0 takes nothing.
template <int NT, typename K>
__device__ void walk_takes(const K* keys, int32_t* lens, int n, uint32_t R, K prefix, K mask,
                           uint32_t rrem, WalkShared& sh) {
  const int tid = threadIdx.x;
  const int cpt = (n + NT - 1) / NT;
  const int c0 = min(tid * cpt, n), c1 = min(c0 + cpt, n);
  int tie_local = 0;
  if (R > 0)
    for (int c = c0; c < c1; ++c)
      if ((keys[c] & mask) == prefix) tie_local += lens[c];
  int tie_total;
  const int tie_before = block_scan_excl<NT>(tie_local, sh, tie_total);
  {
    int run = tie_before;
    for (int c = c0; c < c1; ++c) {
      int take = 0;
      if (R > 0) {
        const K top = keys[c] & mask;
        const int len = lens[c];
        if (top > prefix) {
          take = len;
        } else if (top == prefix) {
          const int rem = (int)rrem - run;
          take = rem <= 0 ? 0 : (rem < len ? rem : len);
          run += len;
        }
      }
      lens[c] = take;
    }
  }
  __syncthreads();
}

// walk_takes, then emit the tiles.  R == 0 emits self only.
template <int NT, typename K, class View>
__device__ void walk_emit(const View& view, const K* keys, int32_t* lens, int n, uint32_t R,
                          K prefix, K mask, uint32_t rrem, int row, int tile_tokens,
                          int32_t* out, int64_t cap, int32_t* ntiles_out, WalkShared& sh) {
  walk_takes<NT, K>(keys, lens, n, R, prefix, mask, rrem, sh);
  emit_takes<NT>(view, lens, n, row, tile_tokens, out, cap, ntiles_out, sh);
}

__device__ __forceinline__ uint32_t order_key32(float x) {
  x = (x == 0.0f) ? 0.0f : x;
  uint32_t b = __float_as_uint(x);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key32_value(uint32_t k) {
  uint32_t b = (k >> 31) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(b);
}

}  // namespace dhsa
