// Sequence-sharded split-KV decode (one
// 1M-token sequence cut into W contiguous shards, one per GPU).
//
//   dhsa_split_select    the global chunk walk over the candidates gathered
//                        from every shard (dhsa_decode_candidates_bf16 makes
//                        them), identical on every shard, emitting the tiles
//                        of this shard's chunks (+ self on the tail shard);
//   dhsa_merge_partials  the cross-shard (m, l, acc) merge of the attention
//                        records written by dhsa_attn_partials.
//
// Selection semantics are masks.topk_row (masks.py:103-122) on the upsampled
// decode row (masks.py:153-173): R = min(budget, row+1) - 1 tokens, chunks in
// (score desc, chunk asc) order, each contributing its lowest tokens, self
// forced.  Chunk ids are global, so the tie-break is the reference's.
#include "capi.cuh"
#include "walk.cuh"

namespace dhsa {

constexpr int kSplitThreads = 256;
constexpr int kSplitMaxShards = 64;

struct SplitSelArgs {
  const unsigned char* gathered;
  int W;
  int64_t rank_stride, cand_stride;
  int cand_cap, items_per_unit;
  int32_t* gen_count;
  const int32_t* plen;
  int total_prompt;
  int64_t budget;
  int rank, owns_tail, tile_tokens;
  int32_t* tiles;
  int64_t tile_cap;
  int32_t* ntiles;
  int advance;
};

__global__ __launch_bounds__(kSplitThreads) void split_select_kernel(SplitSelArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ WalkShared sh;
  __shared__ int s_off[kSplitMaxShards + 1];
  __shared__ int s_bad;
  const int cap_all = a.W * a.cand_cap;
  uint64_t* key = reinterpret_cast<uint64_t*>(smem_raw);
  int32_t* gid = reinterpret_cast<int32_t*>(key + cap_all);
  int32_t* len = gid + cap_all;
  int32_t* lo = len + cap_all;
  int32_t* take = lo + cap_all;

  const int u = blockIdx.x, tid = threadIdx.x;
  const int g = a.gen_count[u];
  const int64_t row = (int64_t)a.total_prompt + g;
  const int64_t keep = a.budget < row + 1 ? a.budget : row + 1;
  const int R = (int)(keep - 1);
  for (int it = 0; it < a.items_per_unit; ++it) {
    const int s = u * a.items_per_unit + it;
    if (tid < a.W)  // every shard's candidate count, loaded together
      s_off[tid + 1] = __ldcg(reinterpret_cast<const int32_t*>(a.gathered + tid * a.rank_stride +
                                                               (int64_t)s * a.cand_stride));
    __syncthreads();
    if (tid == 0) {
      int off = 0, bad = 0;
      for (int r = 0; r < a.W; ++r) {
        const int nr = s_off[r + 1];
        s_off[r] = off;
        if (nr < 0 || nr > a.cand_cap) bad = 1;
        else off += nr;
      }
      s_off[a.W] = off;
      s_bad = bad;
    }
    __syncthreads();
    const int n = s_off[a.W];
    for (int i = tid; i < n; i += kSplitThreads) {
      int r = 0;
      while (s_off[r + 1] <= i) ++r;
      const SplitCand* rec = reinterpret_cast<const SplitCand*>(
                                 a.gathered + r * a.rank_stride + (int64_t)s * a.cand_stride) +
                             1 + (i - s_off[r]);
      key[i] = order_key(rec->score);
      gid[i] = rec->gid;
      len[i] = rec->len;
      lo[i] = rec->lo;
    }
    __syncthreads();
    // takes of this shard's candidates: R minus the tokens ranked before them.
    // Every thread takes (own candidate, 32-candidate slab) pairs — consecutive
    // threads different candidates, the same slab (broadcast loads) — and adds
    // its partial count to the candidate's shared counter: the O(n x mine)
    // ranking spread over the whole CTA instead of one thread per candidate.
    const int mine0 = s_off[a.rank], mine1 = s_off[a.rank + 1];
    const int nm = mine1 - mine0;
    for (int c = tid; c < nm; c += kSplitThreads) take[c] = 0;  // tokens ranked before
    __syncthreads();
    const int nslab = (n + 31) >> 5;
    for (int w = tid; w < nm * nslab; w += kSplitThreads) {
      const int c = w % nm, sl = w / nm;
      const uint64_t ki = key[mine0 + c];
      const int gi = gid[mine0 + c];
      const int j1 = min(n, (sl + 1) << 5);
      int b = 0;
      for (int j = sl << 5; j < j1; ++j) {
        const uint64_t kj = key[j];
        if (kj > ki || (kj == ki && gid[j] < gi)) b += len[j];
      }
      if (b) atomicAdd(&take[c], b);
    }
    __syncthreads();
    for (int c = tid; c < nm; c += kSplitThreads) {
      const int64_t rem = (int64_t)R - take[c];
      const int li = len[mine0 + c];
      take[c] = rem <= 0 ? 0 : (int)(rem < li ? rem : li);
    }
    __syncthreads();
    // tiles of <= tile_tokens tokens for the positive takes, then self
    const int cpt = (nm + kSplitThreads - 1) / kSplitThreads;
    const int c0 = min(tid * cpt, nm), c1 = min(c0 + cpt, nm);
    int nt_local = 0;
    for (int c = c0; c < c1; ++c) nt_local += (take[c] + a.tile_tokens - 1) / a.tile_tokens;
    int nt_total;
    int off = block_scan_excl<kSplitThreads>(nt_local, sh, nt_total);
    int32_t* out = a.tiles + (int64_t)s * a.tile_cap * 2;
    for (int c = c0; c < c1; ++c) {
      for (int t = 0; t < take[c]; t += a.tile_tokens) {
        if (off < a.tile_cap) {
          out[2 * off] = lo[mine0 + c] + t;
          out[2 * off + 1] = min(a.tile_tokens, take[c] - t);
        }
        ++off;
      }
    }
    if (tid == 0) {
      const int total = nt_total + (a.owns_tail ? 1 : 0);
      if (s_bad || total > a.tile_cap) {
        a.ntiles[s] = -1;  // candidate overflow / tile capacity: reported by the host
      } else {
        if (a.owns_tail) {  // self (masks.py:120-121) at the tail shard's newest row
          out[2 * nt_total] = a.plen[u] + g;
          out[2 * nt_total + 1] = 1;
        }
        a.ntiles[s] = total;
      }
    }
    __syncthreads();
  }
  if (tid == 0 && a.advance) a.gen_count[u] = g + 1;  // masks.py:236, on every shard
}

// One thread per (row, d): the (m, l, acc) merge of core.py:113-118's softmax
// computed piecewise; m in the log2 domain.
template <typename T>
__global__ void merge_records_kernel(const float* __restrict__ rec, int W, int64_t rank_stride,
                                     int rows, int D, T* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)rows * D) return;
  const int r = (int)(e / D), d = (int)(e - (int64_t)r * D);
  float mstar = -INFINITY;
  for (int w = 0; w < W; ++w) mstar = fmaxf(mstar, rec[w * rank_stride + (int64_t)r * (D + 2)]);
  float l = 0.f, acc = 0.f;
  for (int w = 0; w < W; ++w) {
    const float* p = rec + w * rank_stride + (int64_t)r * (D + 2);
    if (p[0] == -INFINITY) continue;
    const float wgt = exp2f(p[0] - mstar);
    l += wgt * p[1];
    acc += wgt * p[2 + d];
  }
  out[e] = from_acc<T>(acc / l);
}

}  // namespace dhsa

using namespace dhsa;

extern "C" int dhsa_split_select(const void* gathered, int W, int64_t rank_stride,
                                 int64_t cand_stride, int cand_cap, int items, int items_per_unit,
                                 int32_t* gen_count, const int32_t* plen, int total_prompt,
                                 int64_t budget, int rank, int owns_tail, int tile_tokens,
                                 int32_t* tiles, int64_t tile_cap, int32_t* ntiles, int advance,
                                 dhsa_stream_t stream) {
  DHSA_REQUIRE(gathered && gen_count && plen && tiles && ntiles, "dhsa_split_select: null pointer");
  DHSA_REQUIRE(W >= 1 && W <= kSplitMaxShards && rank >= 0 && rank < W,
               "dhsa_split_select: bad shard count / rank");
  DHSA_REQUIRE(budget >= 1, "budget must be >= 1");
  DHSA_REQUIRE(items >= 1 && items_per_unit >= 1 && items % items_per_unit == 0 && cand_cap >= 1 &&
                   cand_stride >= (int64_t)sizeof(SplitCand) * (cand_cap + 1) &&
                   rank_stride >= cand_stride * items && tile_tokens >= 1 && tile_cap >= 1,
               "dhsa_split_select: bad shape");
  const size_t smem = (size_t)W * cand_cap * (8 + 4 + 4 + 4) + (size_t)cand_cap * 4;
  DHSA_REQUIRE(smem <= 200 * 1024, "dhsa_split_select: W * cand_cap too large");
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(split_select_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      set_error("dhsa_split_select: %s", cudaGetErrorString(e));
      return DHSA_ECUDA;
    }
  }
  SplitSelArgs a{};
  a.gathered = (const unsigned char*)gathered;
  a.W = W;
  a.rank_stride = rank_stride;
  a.cand_stride = cand_stride;
  a.cand_cap = cand_cap;
  a.items_per_unit = items_per_unit;
  a.gen_count = gen_count;
  a.plen = plen;
  a.total_prompt = total_prompt;
  a.budget = budget;
  a.rank = rank;
  a.owns_tail = owns_tail;
  a.tile_tokens = tile_tokens;
  a.tiles = tiles;
  a.tile_cap = tile_cap;
  a.ntiles = ntiles;
  a.advance = advance;
  split_select_kernel<<<(unsigned)(items / items_per_unit), kSplitThreads, smem,
                        (cudaStream_t)stream>>>(a);
  return check_launch("dhsa_split_select");
}

extern "C" int dhsa_merge_partials(const float* records, int W, int64_t rank_stride, int rows,
                                   int D, int dtype, void* out, dhsa_stream_t stream) {
  DHSA_REQUIRE(records && out && W >= 1 && rows >= 1 && D >= 1 &&
                   rank_stride >= (int64_t)rows * (D + 2),
               "dhsa_merge_partials: bad arguments");
  const int64_t total = (int64_t)rows * D;
  const unsigned grid = (unsigned)((total + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == DHSA_BF16)
    merge_records_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(records, W, rank_stride, rows, D,
                                                             (__nv_bfloat16*)out);
  else if (dtype == DHSA_F32)
    merge_records_kernel<float><<<grid, 256, 0, s>>>(records, W, rank_stride, rows, D,
                                                     (float*)out);
  else {
    set_error("dhsa_merge_partials: dtype must be BF16 or F32");
    return DHSA_EINVAL;
  }
  return check_launch("dhsa_merge_partials");
}
