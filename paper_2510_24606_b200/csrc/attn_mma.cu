// K5 (bf16) — block-sparse decode attention: TMA-staged gathers of the
// selected K/V tiles + mma.sync tensor-core tiles, online softmax, split-KV.
//
// Reference: dense_attention's per-row body (core.py:113-118) restricted to the
// selected indices: softmax(K[idx] q / sqrt(d)) @ V[idx].
//
// One CTA = 4 consumer warps + 1 TMA producer warp and works on a contiguous
// slice of one item's tile list (item = one kv group of GH q-heads, or one
// q-head).  A tile is <= 64 consecutive cache tokens (one selected 64-block
// or a piece of a selected range); the producer gathers its K and V rows with
// 2-D TMA loads (64 rows x 128 B boxes, 128B swizzle, so ldmatrix is bank-
// conflict free) into a STAGES-deep mbarrier ring.  Each consumer warp owns 16
// tokens of the tile: S = Q K^T with Q (GH <= 8 heads, padded to 16 rows) as
// the A operand kept in registers for the whole kernel, online softmax in the
// log2 domain, then O += P V with P re-packed from the S accumulators as the
// A operand (no shared-memory round trip).  Warps merge at the end, splits
// merge in the last CTA (attn_common.cuh).  Tokens of a tile beyond its count
// are masked; the KV cache is finite everywhere (zero-initialised), so the
// masked rows contribute exactly 0.
#include "attn_common.cuh"
#include "attn_tile.cuh"
#include "capi.cuh"


namespace dhsa {

template <int D, int STAGES>
__global__ __launch_bounds__(160) void attn_mma_kernel(
    const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
    const __nv_bfloat16* __restrict__ q, int64_t cache_rows, int items_per_unit, int GH,
    const int32_t* __restrict__ tiles, int64_t tile_cap, const int32_t* __restrict__ ntiles,
    int splits, __nv_bfloat16* __restrict__ out, void* ws, int32_t* counters, float scale_log2,
    int32_t* ready, float* __restrict__ rec_out) {
  using T = DecodeTile<D>;
  constexpr int NB = T::NB, BOX = T::BOX, STAGE_BYTES = T::STAGE_BYTES;

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];

  const int item = blockIdx.y, split = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = item / items_per_unit;
  if (ready) {  // launched early (PDL): wait until the selection of this item is published
    if (threadIdx.x == 0) spin_geq(ready + item, kReadyFinal);
    __syncthreads();
  }
  // tiles may have been written while this grid was running: read through L2
  const int nt_all = __ldcg(ntiles + item);
  const int t_begin = (int)((int64_t)nt_all * split / splits);
  const int n = (int)((int64_t)nt_all * (split + 1) / splits) - t_begin;
  const int32_t* tl = tiles + ((int64_t)item * tile_cap + t_begin) * 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 4);
    }
    fence_barrier_init();
  }
  __syncthreads();

  float m = -INFINITY, l = 0.f;
  float o[T::NT][4];
#pragma unroll
  for (int j = 0; j < T::NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;

  if (warp == 4) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      prefetch_tmap(&tmK);
      prefetch_tmap(&tmV);
      const int64_t row0 = (int64_t)unit * cache_rows;
      for (int i = 0; i < n; ++i) {
        const int s = i % STAGES;
        if (i >= STAGES) mbar_wait(&empty_bar[s], ((i / STAGES) + 1) & 1);
        const int row = (int)(row0 + __ldcg(tl + 2 * i));
        unsigned char* st = smem + s * STAGE_BYTES;
        mbar_expect_tx(&full_bar[s], STAGE_BYTES);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          tma_load_2d(st + b * BOX, &tmK, &full_bar[s], b * 64, row);
          tma_load_2d(st + (NB + b) * BOX, &tmV, &full_bar[s], b * 64, row);
        }
      }
    }
  } else {
    // ---------------- consumers ----------------
    uint32_t qa[T::KS][2];
    T::load_q(q, item, GH, lane, qa);
    for (int i = 0; i < n; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full_bar[s], (i / STAGES) & 1);
      const int count = __ldcg(tl + 2 * i + 1);
      T::update(smem_u32(smem + s * STAGE_BYTES), count, warp, lane, qa, scale_log2, m, l, o);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
  }
  __syncthreads();
  // All TMA traffic has been consumed: the stage ring is reused for the merge.
  float* red = reinterpret_cast<float*>(smem);  // [4 warps][GH][D+2]
  if (warp < 4) T::warp_record(red, warp, lane, GH, m, l, o);
  __syncthreads();
  const bool direct = (splits == 1);
  for (int hd = threadIdx.x; hd < GH * D; hd += blockDim.x) {
    const int h = hd / D, d = hd - h * D;
    float mstar, lsum, a;
    combine4<D>(red, GH, h, d, mstar, lsum, a);
    if (direct && rec_out) {  // unnormalised record for a cross-GPU merge
      float* r = rec_out + ((int64_t)item * GH + h) * (D + 2);
      if (d == 0) {
        r[0] = mstar;
        r[1] = lsum;
      }
      r[2 + d] = a;
    } else if (direct) {
      out[((int64_t)item * GH + h) * D + d] = __float2bfloat16_rn(a / lsum);
    } else {
      float* p = partial_ptr<float>(ws, item, split, splits, h, GH, D);
      if (d == 0) {
        p[0] = mstar;
        p[1] = lsum;
      }
      p[2 + d] = a;
    }
  }
  if (direct) {
    if (ready && threadIdx.x == 0) ready[item] = 0;  // re-arm for the next step
    return;
  }
  if (split_arrive(counters, item, splits)) {
    merge_partials<__nv_bfloat16, float>(ws, item, splits, GH, D, out, rec_out);
    if (ready && threadIdx.x == 0) ready[item] = 0;  // every sibling CTA is past its wait
  }
}

template <int D, int STAGES>
static int launch(const CUtensorMap& mk, const CUtensorMap& mv, const void* q, int64_t cache_rows,
                  int items, int ipu, int GH, const int32_t* tiles, int64_t cap,
                  const int32_t* nt, int splits, void* out, void* ws, int32_t* cnt,
                  int32_t* ready, float* rec_out, cudaStream_t s) {
  constexpr int STAGE_BYTES = 2 * (D / 64) * 64 * 128;
  const size_t smem = (size_t)STAGES * STAGE_BYTES + 1024;
  cudaError_t e = cudaFuncSetAttribute(attn_mma_kernel<D, STAGES>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    set_error("dhsa_attn(bf16): %s", cudaGetErrorString(e));
    return DHSA_ECUDA;
  }
  const float scale_log2 = (float)(1.4426950408889634 / sqrt((double)D));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)splits, (unsigned)items);
  cfg.blockDim = dim3(160);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ready ? 1 : 0;  // early launch only when per-item flags gate the work
  e = cudaLaunchKernelEx(&cfg, attn_mma_kernel<D, STAGES>, mk, mv, (const __nv_bfloat16*)q,
                         cache_rows, ipu, GH, tiles, cap, nt, splits, (__nv_bfloat16*)out, ws,
                         cnt, scale_log2, ready, rec_out);
  if (e != cudaSuccess) {
    set_error("dhsa_attn(bf16): %s", cudaGetErrorString(e));
    return DHSA_ECUDA;
  }
  return check_launch("dhsa_attn(bf16)");
}

int attn_mma_bf16(const void* q, const void* k_cache, const void* v_cache,
                  int64_t cache_unit_stride, int64_t cache_rows, int items, int items_per_unit,
                  int GH, int D, const int32_t* tiles, int64_t tile_cap, const int32_t* ntiles,
                  int splits, void* out, void* ws, int32_t* counters, int32_t* ready,
                  float* rec_out, cudaStream_t s) {
  DHSA_REQUIRE(D == 64 || D == 128, "dhsa_attn(bf16): D must be 64 or 128, got %d", D);
  DHSA_REQUIRE(cache_unit_stride == cache_rows * D,
               "dhsa_attn(bf16): cache units must be dense [rows][D]");
  DHSA_REQUIRE(((uintptr_t)k_cache & 15) == 0 && ((uintptr_t)v_cache & 15) == 0 &&
                   ((uintptr_t)q & 3) == 0,
               "dhsa_attn(bf16): misaligned pointers");
  const int units = (items + items_per_unit - 1) / items_per_unit;
  const int64_t rows = (int64_t)units * cache_rows;
  DHSA_REQUIRE(rows < (1ll << 31), "dhsa_attn(bf16): cache too large for 32-bit TMA rows");
  CUtensorMap mk, mv;
  int rc = make_tmap_2d(&mk, k_cache, rows, D, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  if (rc) return rc;
  rc = make_tmap_2d(&mv, v_cache, rows, D, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  if (rc) return rc;
  if (D == 128)
    return launch<128, 3>(mk, mv, q, cache_rows, items, items_per_unit, GH, tiles, tile_cap,
                          ntiles, splits, out, ws, counters, ready, rec_out, s);
  return launch<64, 6>(mk, mv, q, cache_rows, items, items_per_unit, GH, tiles, tile_cap, ntiles,
                       splits, out, ws, counters, ready, rec_out, s);
}

}  // namespace dhsa
