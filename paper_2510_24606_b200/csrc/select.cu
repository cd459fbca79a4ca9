// K4 — exact token-budget Top-K as a chunk walk (weighted radix select).
//
// Reference: masks.topk_row (masks.py:103-122) on the block-constant row made
// by upsample / np.repeat (masks.py:87-100, :168-169):
//     keep = min(budget, row+1); order = argsort(-s[:row+1], stable);
//     others = order[order != row][:keep-1]; idx = sort(others + [row]).
// Because s is constant on each chunk and chunks are contiguous, the stable
// order visits chunks by (score desc, chunk index asc) and each chunk's
// tokens in ascending order, so the kept set is: every chunk whose score is
// above a threshold T taken whole, the chunks scoring exactly T taken in
// index order until R = keep-1 tokens are used (the last one partially),
// plus self.  The diagonal chunk (the one holding `row`) contributes only
// [b_l, row) (causality + self exclusion).  SURVEY.md Appendix A; the oracle
// restatement is oracle/dhsa_oracle.walk_ranges.
//
// T and the residual R_T are found with an MSB-first radix select over the
// 64-bit order-preserving keys of the fp64 scores where every chunk counts
// with its token length (a weighted select), 8 bits per pass, one CTA per
// selection row, keys and lengths resident in shared memory.
#include "capi.cuh"

namespace dhsa {

constexpr int kSelThreads = 512;

// Decode rows (masks.py:153-173): prompt chunks, then the generated chunk
// [P, P+g) when g >= 1; the newest token (row P+g) is a singleton chunk that
// contributes only itself.
struct DecodeRows {
  const double* scores;
  int64_t sc_stride;
  Layout lay;
  const int32_t* gen_count;
  int hpu;
  // per item
  const double* srow;
  int u, nc, g, P;
  __device__ void init(int s) {
    u = s / hpu;
    srow = scores + (int64_t)s * sc_stride;
    nc = lay.num_chunks(u);
    g = gen_count[u];
    P = lay.prompt_len(u);
  }
  __device__ int n() const { return nc + (g >= 1 ? 1 : 0); }
  __device__ int row() const { return P + g; }
  __device__ double score(int c) const { return srow[c]; }
  __device__ void chunk(int c, int& lo, int& len) const {
    if (c < nc) {
      int hi;
      lay.chunk(u, c, lo, hi);
      len = hi - lo;
    } else {
      lo = P;
      len = g;
    }
  }
};

// Prefill rows (masks.py:125-140): row i of chunk l scores with S_c[l, :];
// chunks 0..l-1 whole, the diagonal chunk l only [b_l, i).
struct MatrixRows {
  const double* scores;
  int64_t sc_stride;
  const int32_t* bounds;
  int n_chunks;
  const int32_t* row_index;
  const double* srow;
  int i, l;
  __device__ void init(int r) {
    i = row_index[r];
    int a = 0, b = n_chunks;  // largest c with bounds[c] <= i
    while (b - a > 1) {
      int m = (a + b) >> 1;
      if (bounds[m] <= i) a = m; else b = m;
    }
    l = a;
    srow = scores + (int64_t)l * sc_stride;
  }
  __device__ int n() const { return l + 1; }
  __device__ int row() const { return i; }
  __device__ double score(int c) const { return srow[c]; }
  __device__ void chunk(int c, int& lo, int& len) const {
    lo = bounds[c];
    len = (c < l ? bounds[c + 1] : i) - lo;
  }
};

// Exclusive block scan of one int per thread; returns the prefix, sets total.
__device__ __forceinline__ int block_excl_scan(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int t = lane < (kSelThreads / 32) ? warp_tot[lane] : 0;
    int w = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (kSelThreads / 32)) warp_tot[lane] = w - t;  // exclusive
    if (lane == 31) warp_tot[32] = w;
  }
  __syncthreads();
  const int res = warp_tot[warp] + x - v;
  total = warp_tot[32];
  __syncthreads();
  return res;
}

template <class View>
__global__ __launch_bounds__(kSelThreads) void select_kernel(View view, int64_t budget,
                                                             int tile_tokens,
                                                             int32_t* __restrict__ tiles,
                                                             int64_t tile_cap,
                                                             int32_t* __restrict__ ntiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t hist[256];
  __shared__ int warp_tot[33];
  __shared__ uint32_t s_digit, s_rrem, s_done;

  const int item = blockIdx.x;
  const int tid = threadIdx.x;
  view.init(item);
  const int n = view.n();
  const int row = view.row();
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw);
  int32_t* lens = reinterpret_cast<int32_t*>(keys + n);

  for (int c = tid; c < n; c += kSelThreads) {
    int lo, len;
    view.chunk(c, lo, len);
    keys[c] = order_key(view.score(c));
    lens[c] = len;
  }
  // tokens to pick besides self: min(budget, row+1) - 1 (masks.py:117-121)
  const int64_t keep = budget < (int64_t)row + 1 ? budget : (int64_t)row + 1;
  const uint32_t R = (uint32_t)(keep - 1);
  uint64_t prefix = 0, mask = 0;
  uint32_t rrem = R;
  __syncthreads();

  // All causal tokens fit (R == row): every chunk is taken whole (tie class
  // = everything, walked with rrem = total).  R == 0: only self.
  if (R > 0 && R < (uint32_t)row) {
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int b = tid; b < 256; b += kSelThreads) hist[b] = 0;
      __syncthreads();
      for (int c = tid; c < n; c += kSelThreads) {
        const uint64_t k = keys[c];
        if ((k & mask) == prefix && lens[c] > 0)
          atomicAdd(&hist[(k >> shift) & 255], (uint32_t)lens[c]);
      }
      __syncthreads();
      if (tid < 32) {
        const int lane = tid;
        uint32_t w[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          w[j] = hist[255 - 8 * lane - j];
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
        if (lane == f) {
          uint32_t cum = excl;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (cum + w[j] >= rrem) {
              s_digit = 255 - 8 * lane - j;
              s_rrem = rrem - cum;
              s_done = (rrem - cum == w[j]);
              break;
            }
            cum += w[j];
          }
        }
      }
      __syncthreads();
      prefix |= (uint64_t)s_digit << shift;
      mask |= (uint64_t)0xFF << shift;
      rrem = s_rrem;
      const bool done = s_done;
      __syncthreads();
      if (done) break;  // the whole bucket is kept: no finer split needed
    }
  }

  // Emit, in chunk (= token) order.  Thread t owns chunks [t*cpt, (t+1)*cpt).
  const int cpt = (n + kSelThreads - 1) / kSelThreads;
  const int c0 = min(tid * cpt, n), c1 = min(c0 + cpt, n);
  int tie_local = 0;
  if (R > 0) {
    for (int c = c0; c < c1; ++c)
      if ((keys[c] & mask) == prefix) tie_local += lens[c];
  }
  int tie_total;
  int tie_before = block_excl_scan(tie_local, warp_tot, tie_total);
  int ntile_local = 0;
  if (R > 0) {
    int run = tie_before;
    for (int c = c0; c < c1; ++c) {
      const uint64_t top = keys[c] & mask;
      int take = 0;
      if (top > prefix) {
        take = lens[c];
      } else if (top == prefix) {
        const int rem = (int)rrem - run;
        take = rem <= 0 ? 0 : (rem < lens[c] ? rem : lens[c]);
        run += lens[c];
      }
      lens[c] = take;  // reuse: tokens taken from the chunk start
      ntile_local += (take + tile_tokens - 1) / tile_tokens;
    }
  }
  int tiles_total;
  int tile_off = block_excl_scan(ntile_local, warp_tot, tiles_total);
  int32_t* out = tiles + (int64_t)item * tile_cap * 2;
  if (R > 0) {
    for (int c = c0; c < c1; ++c) {
      const int take = lens[c];
      if (take <= 0) continue;
      int lo, len;
      view.chunk(c, lo, len);
      for (int t = 0; t < take; t += tile_tokens) {
        if (tile_off < tile_cap) {
          out[2 * tile_off] = lo + t;
          out[2 * tile_off + 1] = min(tile_tokens, take - t);
        }
        ++tile_off;
      }
    }
  }
  if (tid == 0) {
    if (tiles_total + 1 > tile_cap) {
      ntiles[item] = -1;  // capacity error, reported by the host wrapper
    } else {
      out[2 * tiles_total] = row;  // self (masks.py:120-121)
      out[2 * tiles_total + 1] = 1;
      ntiles[item] = tiles_total + 1;
    }
  }
}

template <class View>
static int launch_select(View v, int items, int n_max, int64_t budget, int tile_tokens,
                         int32_t* tiles, int64_t tile_cap, int32_t* ntiles, cudaStream_t s,
                         const char* name) {
  const size_t smem = (size_t)n_max * (sizeof(uint64_t) + sizeof(int32_t));
  DHSA_REQUIRE(smem <= 200 * 1024, "%s: %d chunks exceed the shared-memory select capacity",
               name, n_max);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(select_kernel<View>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      set_error("%s: %s", name, cudaGetErrorString(e));
      return DHSA_ECUDA;
    }
  }
  select_kernel<View><<<items, kSelThreads, smem, s>>>(v, budget, tile_tokens, tiles, tile_cap,
                                                       ntiles);
  return check_launch(name);
}

}  // namespace dhsa

using namespace dhsa;

extern "C" int dhsa_decode_select(const double* scores, int64_t sc_stride, dhsa_layout layout,
                                  const int32_t* gen_count, int U, int heads_per_unit,
                                  int64_t budget, int tile_tokens, int32_t* tiles,
                                  int64_t tile_cap, int32_t* ntiles, dhsa_stream_t stream) {
  DHSA_REQUIRE(scores && gen_count && tiles && ntiles, "dhsa_decode_select: null pointer");
  DHSA_REQUIRE(budget >= 1, "budget must be >= 1");
  DHSA_REQUIRE(U >= 1 && heads_per_unit >= 1 && tile_tokens >= 1 && tile_cap >= 1,
               "dhsa_decode_select: bad shape");
  DHSA_REQUIRE(valid_layout(layout), "dhsa_decode_select: bad layout");
  DecodeRows v{scores, sc_stride, Layout(layout), gen_count, heads_per_unit};
  return launch_select(v, U * heads_per_unit, layout.max_chunks + 1, budget, tile_tokens, tiles,
                       tile_cap, ntiles, (cudaStream_t)stream, "dhsa_decode_select");
}

extern "C" int dhsa_rows_select(const double* scores, int64_t sc_stride, const int32_t* bounds,
                                int n_chunks, const int32_t* row_index, int rows,
                                int64_t budget, int tile_tokens, int32_t* tiles,
                                int64_t tile_cap, int32_t* ntiles, dhsa_stream_t stream) {
  DHSA_REQUIRE(scores && bounds && row_index && tiles && ntiles, "dhsa_rows_select: null pointer");
  DHSA_REQUIRE(budget >= 1, "budget must be >= 1");
  DHSA_REQUIRE(n_chunks >= 1 && rows >= 1 && tile_tokens >= 1 && tile_cap >= 1,
               "dhsa_rows_select: bad shape");
  MatrixRows v{scores, sc_stride, bounds, n_chunks, row_index};
  return launch_select(v, rows, n_chunks, budget, tile_tokens, tiles, tile_cap, ntiles,
                       (cudaStream_t)stream, "dhsa_rows_select");
}
