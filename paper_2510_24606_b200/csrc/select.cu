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
#include "walk.cuh"

extern "C" int64_t dhsa_select_scratch_size(int n_chunks) {
  const int64_t bytes = ((int64_t)n_chunks * (sizeof(uint64_t) + sizeof(int32_t)) + 15) / 16 * 16;
  return bytes <= 200 * 1024 ? 0 : bytes;
}

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

template <class View>
__global__ __launch_bounds__(kSelThreads) void select_kernel(View view, int64_t budget,
                                                             int tile_tokens,
                                                             int32_t* __restrict__ tiles,
                                                             int64_t tile_cap,
                                                             int32_t* __restrict__ ntiles,
                                                             unsigned char* gscratch,
                                                             int64_t gscratch_stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ WalkShared sh;
  const int item = blockIdx.x;
  view.init(item);
  const int n = view.n();
  const int row = view.row();
  // keys + lengths in shared memory, or (rows of more chunks than fit, e.g.
  // topk_row with one chunk per token beyond ~17K positions) in global scratch
  unsigned char* base = gscratch ? gscratch + (int64_t)item * gscratch_stride : smem_raw;
  uint64_t* keys = reinterpret_cast<uint64_t*>(base);
  int32_t* lens = reinterpret_cast<int32_t*>(keys + n);
  for (int c = threadIdx.x; c < n; c += kSelThreads) {
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
  // R == row: every causal token is kept (one tie class = everything).
  if (R > 0 && R < (uint32_t)row)
    radix_threshold<kSelThreads, uint64_t>(keys, lens, n, R, sh, prefix, mask, rrem);
  walk_emit<kSelThreads, uint64_t>(view, keys, lens, n, R, prefix, mask, rrem, row, tile_tokens,
                                   tiles + (int64_t)item * tile_cap * 2, tile_cap, ntiles + item,
                                   sh);
}

template <class View>
static int launch_select(View v, int items, int n_max, int64_t budget, int tile_tokens,
                         int32_t* tiles, int64_t tile_cap, int32_t* ntiles, void* scratch,
                         cudaStream_t s, const char* name) {
  const int64_t need = dhsa_select_scratch_size(n_max);
  size_t smem = 0;
  if (need == 0) {
    smem = (size_t)n_max * (sizeof(uint64_t) + sizeof(int32_t));
    scratch = nullptr;
  } else {
    DHSA_REQUIRE(scratch, "%s: %d chunks need %lld bytes of global select scratch per row",
                 name, n_max, (long long)need);
  }
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(select_kernel<View>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      set_error("%s: %s", name, cudaGetErrorString(e));
      return DHSA_ECUDA;
    }
  }
  select_kernel<View><<<items, kSelThreads, smem, s>>>(v, budget, tile_tokens, tiles, tile_cap,
                                                       ntiles, (unsigned char*)scratch, need);
  return check_launch(name);
}

}  // namespace dhsa

using namespace dhsa;

extern "C" int dhsa_decode_select(const double* scores, int64_t sc_stride, dhsa_layout layout,
                                  const int32_t* gen_count, int U, int heads_per_unit,
                                  int64_t budget, int tile_tokens, int32_t* tiles,
                                  int64_t tile_cap, int32_t* ntiles, void* scratch,
                                  dhsa_stream_t stream) {
  DHSA_REQUIRE(scores && gen_count && tiles && ntiles, "dhsa_decode_select: null pointer");
  DHSA_REQUIRE(budget >= 1, "budget must be >= 1");
  DHSA_REQUIRE(U >= 1 && heads_per_unit >= 1 && tile_tokens >= 1 && tile_cap >= 1,
               "dhsa_decode_select: bad shape");
  DHSA_REQUIRE(valid_layout(layout), "dhsa_decode_select: bad layout");
  DecodeRows v{scores, sc_stride, Layout(layout), gen_count, heads_per_unit};
  return launch_select(v, U * heads_per_unit, layout.max_chunks + 1, budget, tile_tokens, tiles,
                       tile_cap, ntiles, scratch, (cudaStream_t)stream, "dhsa_decode_select");
}

extern "C" int dhsa_rows_select(const double* scores, int64_t sc_stride, const int32_t* bounds,
                                int n_chunks, const int32_t* row_index, int rows,
                                int64_t budget, int tile_tokens, int32_t* tiles,
                                int64_t tile_cap, int32_t* ntiles, void* scratch,
                                dhsa_stream_t stream) {
  DHSA_REQUIRE(scores && bounds && row_index && tiles && ntiles, "dhsa_rows_select: null pointer");
  DHSA_REQUIRE(budget >= 1, "budget must be >= 1");
  DHSA_REQUIRE(n_chunks >= 1 && rows >= 1 && tile_tokens >= 1 && tile_cap >= 1,
               "dhsa_rows_select: bad shape");
  MatrixRows v{scores, sc_stride, bounds, n_chunks, row_index};
  return launch_select(v, rows, n_chunks, budget, tile_tokens, tiles, tile_cap, ntiles, scratch,
                       (cudaStream_t)stream, "dhsa_rows_select");
}
