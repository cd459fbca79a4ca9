/*
 * dhsa_b200.h — C ABI of libdhsa_b200.so, the sm_100a (B200) implementation of
 * the DHSA sparse-attention hot path:
 *
 *   centroids (sum/sqrt(n), fp64)  ->  query-centroid scores (fp64)  ->
 *   token-budget Top-K as a chunk walk  ->  exact softmax attention over the
 *   selected token ranges (online softmax, split-KV partial merge).
 *
 * The reference (/root/reference/pkg/src/dhsa) is a pure-NumPy package with no
 * FFI; its operator surface is the Python API re-exported by
 * dhsa/__init__.py:7-49.  Each entry point below names the reference function
 * whose arithmetic it replaces.  The Python package paper_2510_24606_b200
 * re-exposes the reference names and signatures on top of these calls
 * (see INTEGRATION.md for the ctypes binding a maintainer would add).
 *
 * Conventions
 *  - All pointers are caller-owned DEVICE pointers; nothing is allocated
 *    inside (workspace sizes are queried with the *_workspace_size calls).
 *  - "unit" u = one (sequence, kv-head) pair; units are laid out densely, so
 *    q/o rows of unit u with group size G are rows u*G .. u*G+G-1 and the
 *    K/V cache of unit u starts at cache + u*cache_unit_stride (elements).
 *  - Every call is asynchronous on `stream` and returns 0 on success or a
 *    negative DHSA_E* code; dhsa_last_error() returns a thread-local message.
 *  - Functions are re-entrant; the library keeps no mutable global state.
 */
#ifndef DHSA_B200_H
#define DHSA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dhsa_stream_t; /* == cudaStream_t */

enum dhsa_dtype { DHSA_F64 = 0, DHSA_F32 = 1, DHSA_BF16 = 2 };
enum dhsa_agg { DHSA_AGG_NONE = 0, DHSA_AGG_MAX = 1, DHSA_AGG_MEAN = 2 };
enum dhsa_status {
  DHSA_OK = 0,
  DHSA_EINVAL = -1,   /* bad argument (shape, dtype, budget, alignment) */
  DHSA_ECUDA = -2,    /* CUDA launch / driver failure */
  DHSA_ERANGE = -3,   /* capacity exceeded (tiles, chunks) */
};

/* Chunk layout of the PROMPT part of each unit.  Either an explicit boundary
 * list per unit (bounds[u*bounds_stride + c], c = 0..nchunks[u], the
 * reference's `bounds`, chunking.py:23-39), or, when bounds == NULL, the static
 * grid [0, block, 2*block, ..., plen[u]] (chunking.py:42-54). */
typedef struct {
  const int32_t* bounds;   /* device [U][bounds_stride] or NULL */
  int64_t bounds_stride;   /* 0 = one list shared by all units */
  const int32_t* nchunks;  /* device [U] prompt chunk count (explicit mode) */
  const int32_t* plen;     /* device [U] prompt length in tokens */
  int32_t block;           /* static grid chunk size (bounds == NULL) */
  int32_t max_chunks;      /* host upper bound on prompt chunks over units */
} dhsa_layout;

const char* dhsa_last_error(void);
int dhsa_version(void);

/* K1 — chunk centroids c_j = (sum_{t in chunk j} x_t, accumulated in token
 * order in fp64) / sqrt(n_j).  Replaces chunk_repr.aggregate_rows
 * (chunk_repr.py:57-68; sequential_sum :29-35, aggregate_chunk :38-54).
 * Bit-exact with the reference for any input dtype.
 * x: [U][x_unit_stride] rows of D elements (row stride D).
 * out: [U][out_unit_stride] fp64, chunk c at out + u*out_unit_stride + c*D.
 * normalize = 0 returns the raw sequential sums (the generated-chunk running
 * sum of masks.py:197-199 / :235). */
int dhsa_centroids(int dtype, const void* x, int64_t x_unit_stride, int D, int U,
                   dhsa_layout layout, int normalize, double* out,
                   int64_t out_unit_stride, dhsa_stream_t stream);

/* K3 (+K2) — decode scores of Algorithm 2 (masks.py:153-173): for every unit u
 * and chunk j of [prompt chunks | generated chunk (if gen_count[u] >= 1)],
 * score = q . c_j in fp64 with no 1/sqrt(d) (masks.py:164-165,
 * chunk_repr.py:97-103).  The generated-chunk centroid is
 * gen_sum[u] / sqrt(gen_count[u]) (masks.py:161).  With agg = MAX / MEAN the
 * G per-head rows of a unit are reduced (harness.py:288-306) into one row per
 * unit; with agg = NONE one row per q-head is written.
 * scores: [U or U*G][sc_stride] fp64, prompt chunk c at [c], the generated
 * chunk at [nchunks(u)].
 * State update folded in (masks.py:235-236 without the count): when k_new is
 * non-NULL, gen_sum[u] += k_new[u] (fp64, after it was read) and, when the
 * caches are non-NULL, k_new/v_new are appended at token plen[u]+gen_count[u]
 * of the K/V cache.  gen_count itself is advanced by dhsa_decode_advance. */
int dhsa_decode_score(int dtype, const void* q, const double* centroids,
                      int64_t c_unit_stride, double* gen_sum,
                      const int32_t* gen_count, const void* k_new,
                      const void* v_new, void* k_cache, void* v_cache,
                      int64_t cache_unit_stride, dhsa_layout layout, int U, int G,
                      int D, int agg, double* scores, int64_t sc_stride,
                      dhsa_stream_t stream);

/* K4 — decode selection: the causal token-budget Top-K with forced self and
 * lower-index tie-break (masks.topk_row, masks.py:103-122) applied to the
 * block-constant upsampled row (masks.py:168-169), computed exactly as a walk
 * over chunks ordered by (score desc, chunk asc) with a weighted radix select.
 * Row i = plen[u] + gen_count[u] (the newest token).  Output: the selected
 * token ranges split into tiles of at most `tile_tokens` tokens, sorted by
 * start, followed by the self tile (i, 1).  tiles[s*tile_cap + t] = {start,
 * count} for selection row s (s = u for aggregated scores, s = u*G+j for
 * per-head scores; heads_per_unit = 1 or G), ntiles[s] = count of tiles. */
int dhsa_decode_select(const double* scores, int64_t sc_stride, dhsa_layout layout,
                       const int32_t* gen_count, int U, int heads_per_unit,
                       int64_t budget, int tile_tokens, int32_t* tiles,
                       int64_t tile_cap, int32_t* ntiles, void* scratch,
                       dhsa_stream_t stream);

/* Bytes of global scratch PER SELECTION ROW that dhsa_decode_select /
 * dhsa_rows_select need for rows of `n_chunks` chunks (decode: max_chunks+1).
 * 0 = the row's keys fit in shared memory and `scratch` may be NULL;
 * otherwise `scratch` must hold rows * this many bytes (topk_row over more
 * than ~17K token positions, where every position is its own chunk). */
int64_t dhsa_select_scratch_size(int n_chunks);

/* K5/K6 — exact attention over selected token tiles: per q-head,
 * softmax(K[idx] q / sqrt(D)) @ V[idx] (core.py:113-118) with an online
 * softmax, split over `splits` CTAs per item and merged in-kernel (the last
 * CTA of an item combines the (m, l, acc) partials).
 * item s covers q rows s*GH .. s*GH+GH-1 and reads the cache of unit
 * s / items_per_unit; tiles/ntiles as produced by dhsa_decode_select.
 * dtype BF16: TMA-staged 128B-swizzled tiles + mma.sync (fp32 accumulate),
 * D in {64, 128}, cache_unit_stride % 64 == 0.  dtype F32/F64: FFMA/DFMA with
 * accumulation in the input precision, any D.
 * out: [items*GH][D] in the input dtype (bf16 output for bf16).
 * workspace: dhsa_attn_workspace_size bytes; counters: int32[items], zeroed
 * once by the caller (the kernel re-arms them).
 * ready (bf16 only, may be NULL): int32[items] flags published by
 * dhsa_decode_step_bf16; when given, the kernel is launched with programmatic
 * stream serialization so it overlaps the selection, each CTA waits for its
 * item's flag, and the last CTA of an item clears it. */
int64_t dhsa_attn_workspace_size(int dtype, int items, int GH, int D, int splits);
int dhsa_attn(int dtype, const void* q, const void* k_cache, const void* v_cache,
              int64_t cache_unit_stride, int64_t cache_rows, int items,
              int items_per_unit, int GH, int D, const int32_t* tiles,
              int64_t tile_cap, const int32_t* ntiles, int splits, void* out,
              void* workspace, int32_t* counters, int32_t* ready,
              dhsa_stream_t stream);

/* Persistent, dynamically balanced bf16 variant of dhsa_attn: a grid of
 * resident CTAs (occupancy x SMs) pulls chunks of the virtual tile space
 * items x tiles_hint from a device counter; each CTA's TMA ring streams
 * everything it pulls, ring entries carrying their metadata; the tiles of an
 * item one CTA processed end in an (m, l, acc) record and the segment that
 * completes the item's tile count merges them.  Tiles beyond tiles_hint go to
 * whoever pulls the item's last slot, so the result does not depend on the
 * hint (only the balance does).  Writes out (bf16) or, when records != NULL,
 * the unnormalised per-row records of dhsa_attn_partials.
 * workspace: dhsa_attn_stream_workspace_size bytes; counters:
 * int32[dhsa_attn_stream_counters(items)] zero at rest (re-armed in-kernel);
 * ready as in dhsa_attn, except that the flags are re-armed by the next
 * step's dhsa_decode_step_bf16 rather than by the attention. */
int dhsa_attn_stream_counters(int items);
int64_t dhsa_attn_stream_workspace_size(int items, int GH, int D);
int dhsa_attn_stream(const void* q, const void* k_cache, const void* v_cache,
                     int64_t cache_unit_stride, int64_t cache_rows, int items, int items_per_unit,
                     int GH, int D, const int32_t* tiles, int64_t tile_cap,
                     const int32_t* ntiles, int tiles_hint, void* out, float* records,
                     void* workspace, int32_t* counters, int32_t* ready, dhsa_stream_t stream);

/* gen_count[u] += 1 for all units (masks.py:236). */
int dhsa_decode_advance(int32_t* gen_count, int U, dhsa_stream_t stream);

/* S_c = Q_c K_c^T for one head (chunk_repr.chunk_similarity,
 * chunk_repr.py:97-103), fp64, no scaling.  qc: [n][D], kc: [m][D],
 * out: [n][m]; batched over `heads` with the given strides (elements). */
int dhsa_chunk_scores(const double* qc, const double* kc, int n, int m, int D,
                      int heads, int64_t qc_head_stride, int64_t kc_head_stride,
                      double* out, int64_t out_head_stride, dhsa_stream_t stream);

/* Per-row selection of the prefill mask (masks.mask_from_chunk_scores,
 * masks.py:125-140, i.e. topk_row on the upsampled row, :87-100): for each of
 * `rows` query rows r with token index i = row_index[r] lying in chunk l,
 * walk chunks 0..l with score row scores[l*sc_stride + c] (sc_stride = 0 uses
 * one shared row, which is masks.topk_row on token scores when every chunk
 * is one token), the diagonal chunk contributing [bounds[l], i).
 * bounds: [n_chunks+1] int32.  Output as dhsa_decode_select. */
int dhsa_rows_select(const double* scores, int64_t sc_stride, const int32_t* bounds,
                     int n_chunks, const int32_t* row_index, int rows,
                     int64_t budget, int tile_tokens, int32_t* tiles,
                     int64_t tile_cap, int32_t* ntiles, void* scratch,
                     dhsa_stream_t stream);

/* ---- bf16 fast path: fp16 centroid sketch + certified exact selection -----
 * The decode step for bf16 caches streams an fp16 copy ("sketch") of the fp64
 * centroids, scaled per unit by a power of two, instead of the fp64
 * centroids.  The build measures the sketch's rounding error; with it the
 * score error is bounded rigorously (|s'' - s 2^-k| <= ||q|| dmax + gamma_D
 * ||q|| cmax) and only the chunks within twice that bound of the selection
 * cut are re-scored in fp64, so the selected indices are those of the fp64
 * walk (masks.py:153-173, :103-122).  See decode_sketch.cu / DESIGN.md.
 *
 * dhsa_sketch_build: for prompt chunks, sketch[u][c] = RN_fp16(c 2^-k_u) and
 * sinfo[u] = {k_u, max_c ||sketch||_2, max_c ||sketch - c 2^-k_u||_2, max|c|}
 * (float[4] per unit).  Called once after dhsa_centroids at prefill. */
int dhsa_sketch_build(const double* centroids, int64_t c_unit_stride, int D, int U,
                      dhsa_layout layout, void* sketch, int64_t sk_unit_stride,
                      float* sinfo, dhsa_stream_t stream);

/* Bytes of global select scratch PER UNIT for dhsa_decode_step_bf16 /
 * dhsa_decode_candidates_bf16 with units of up to max_chunks chunks (20 B per
 * chunk).  The scratch is required when a unit's chunks do not fit the
 * generic select's shared memory (> 4,914 chunks) and lets the
 * register-resident select run (it keeps its massive-tie fallback there);
 * with NULL scratch the generic shared-memory select runs. */
int64_t dhsa_sketch_select_scratch_size(int max_chunks);

/* One decode step's K3 + K4 (+K2, + advance) for bf16 caches, D in {64,128},
 * G in {1,2,4,8}; two launches:
 *   1. persistent sketch stream (TMA bulk ring) -> approximate scores
 *      approx[items][sc_stride] (f32, sketch units);
 *   2. one CTA per unit: generated chunk scored exactly in fp64, running sum
 *      += k_new and k/v appended at row plen+gen_count (masks.py:235), the
 *      certified walk -> tiles/ntiles exactly as dhsa_decode_select would
 *      produce from fp64 scores, and gen_count += 1 when `advance`.
 * scratch: U * dhsa_sketch_select_scratch_size bytes (or NULL, see there);
 * approx rows: sc_stride >= max_chunks + 1 (a multiple of 4 lets the select
 * read the scores as float4).
 * The select kernel is launched with programmatic stream serialization: its
 * prologue (query staging, generated-chunk update) overlaps the sketch stream
 * and it waits (griddepcontrol.wait) before reading the scores.
 * ready: int32[items] (or NULL) flags raised when an item's tiles are final,
 * consumed by dhsa_attn / dhsa_attn_stream (re-armed by the next step's
 * sketch stream).
 * progress: int32[U] zero at rest, or NULL: per-unit slice counters from the
 * sketch stream to the select, so a unit is selected as soon as its own
 * centroids are scored (re-armed in-kernel); NULL waits for the whole
 * stream. */
int dhsa_decode_step_bf16(const void* q, const void* sketch, int64_t sk_unit_stride,
                          const float* sinfo, const double* centroids,
                          int64_t c_unit_stride, double* gen_sum, int32_t* gen_count,
                          const void* k_new, const void* v_new, void* k_cache,
                          void* v_cache, int64_t cache_unit_stride, dhsa_layout layout,
                          int U, int G, int D, int agg, int64_t budget, int tile_tokens,
                          int32_t* tiles, int64_t tile_cap, int32_t* ntiles, float* approx,
                          int64_t sc_stride, void* scratch, int32_t* ready, int advance,
                          int32_t* progress, dhsa_stream_t stream);

/* ---- sequence-sharded split-KV decode (1M-token contexts over GPUs) --------
 * A sequence is cut into W contiguous shards (one per GPU); shard r holds
 * prompt chunks [chunk_offset, chunk_offset + nchunks) with their K/V,
 * centroids and sketch; the tail shard (owns_tail) also holds the generated
 * chunk and receives the newest token.  One step:
 *   1. dhsa_decode_candidates_bf16 on every shard: local certified walk with
 *      the GLOBAL budget -> candidate records (exact fp64 score, global chunk
 *      id, length, local start) of every chunk with a positive local take;
 *   2. all-gather of the fixed-size candidate rows (NCCL);
 *   3. dhsa_split_select: the global walk over all shards' candidates
 *      (identical on every shard) -> this shard's tiles (+ self on the tail);
 *   4. dhsa_attn_partials: attention over the local tiles -> unnormalised
 *      (m, l, acc) records per q row;
 *   5. all-gather of the records (NCCL) and dhsa_merge_partials.
 * The union of local candidate sets contains every chunk of the global
 * selection (a chunk with fewer than R tokens ranked above it globally has
 * fewer than R above it locally), so the result equals the unsharded walk. */
typedef struct {
  double score;   /* exact fp64 aggregated score (q . c_j, masks.py:165) */
  int32_t gid;    /* global chunk id (prompt chunks in order, then the generated chunk) */
  int32_t len;    /* chunk length in tokens */
  int32_t lo;     /* first token of the chunk in the shard's cache */
  int32_t pad;
} dhsa_split_cand;  /* one candidate; row = [count (int32, -1 = overflow) | pad][cap records] */

typedef struct {
  int32_t chunk_offset;  /* global id of this shard's chunk 0 */
  int32_t total_chunks;  /* global prompt chunk count (= generated chunk id) */
  int32_t total_prompt;  /* global prompt length; the newest token is row total_prompt + g */
  int32_t owns_tail;     /* 1 on the shard holding the generated chunk and the newest token */
} dhsa_split_shard;

/* Step 1 (bf16 sketch path; arguments as dhsa_decode_step_bf16).  gen_count
 * is the GLOBAL generated count on every shard (not advanced here); k_new /
 * v_new / caches are used on the tail shard only (NULL elsewhere).
 * cand: [items][cand_stride bytes], cand_stride >= 24 * (cand_cap + 1). */
int dhsa_decode_candidates_bf16(const void* q, const void* sketch, int64_t sk_unit_stride,
                                const float* sinfo, const double* centroids,
                                int64_t c_unit_stride, double* gen_sum, const int32_t* gen_count,
                                const void* k_new, const void* v_new, void* k_cache,
                                void* v_cache, int64_t cache_unit_stride, dhsa_layout layout,
                                int U, int G, int D, int agg, int64_t budget,
                                dhsa_split_shard shard, void* cand, int64_t cand_stride,
                                int cand_cap, float* approx, int64_t sc_stride, void* scratch,
                                int32_t* progress, dhsa_stream_t stream);

/* Step 3: the global walk (masks.topk_row order: score desc, chunk asc) over
 * the W gathered candidate rows of every item (gathered + r * rank_stride
 * bytes = shard r's [items][cand_stride] block) with R = min(budget, row+1)-1,
 * row = total_prompt + gen_count[u].  Emits tiles for this shard's chunks
 * (candidates of shard `rank`) and, on the tail shard, the self tile at local
 * row self_row[u] = local prompt length + gen_count[u].  advance: gen_count
 * += 1 afterwards (every shard keeps the global count). */
int dhsa_split_select(const void* gathered, int W, int64_t rank_stride, int64_t cand_stride,
                      int cand_cap, int items, int items_per_unit, int32_t* gen_count,
                      const int32_t* plen, int total_prompt, int64_t budget, int rank,
                      int owns_tail, int tile_tokens, int32_t* tiles, int64_t tile_cap,
                      int32_t* ntiles, int advance, dhsa_stream_t stream);

/* Step 4: dhsa_attn (bf16) writing, per q row, the unnormalised record
 * [m (log2 domain), l, acc[D]] (fp32) instead of the output; an empty
 * selection gives m = -inf, l = 0, acc = 0. */
int dhsa_attn_partials(const void* q, const void* k_cache, const void* v_cache,
                       int64_t cache_unit_stride, int64_t cache_rows, int items,
                       int items_per_unit, int GH, int D, const int32_t* tiles,
                       int64_t tile_cap, const int32_t* ntiles, int splits, float* records,
                       void* workspace, int32_t* counters, dhsa_stream_t stream);

/* Step 5: o = sum_r acc_r 2^(m_r - m*) / sum_r l_r 2^(m_r - m*), m* = max_r m_r,
 * over W record blocks (records + r * rank_stride floats, [rows][D+2] each);
 * out [rows][D] in dtype (BF16 / F32). */
int dhsa_merge_partials(const float* records, int W, int64_t rank_stride, int rows, int D,
                        int dtype, void* out, dhsa_stream_t stream);

/* ---- sparse prefill on tcgen05 (config C5) ---------------------------------
 * prefill_mask (masks.py:143-150) + dense_attention(seq, mask) (core.py:98-119)
 * for B sequences, q [U*G][L][D], k/v [U][L][D] bf16 (U = B * kv heads, G q
 * heads per kv head), static 64-token chunks, D = 128.  The L x L upsampled
 * matrix is never built.
 *
 * dhsa_prefill_scores: S[s][l][c] (c <= l) = agg_j Qc[q(s,j)][l] . Kc[u(s)][c]
 * in fp64 (chunk_repr.py:97-103; harness.py:288-306 max / mean over the G
 * q-heads of unit s, or agg NONE: one row per q head, s = u*G + j).
 * q_centroids [U*G][n_chunks][D], k_centroids [U][n_chunks][D] from
 * dhsa_centroids; scores [S][n_chunks][n_chunks]. */
int dhsa_prefill_scores(const double* q_centroids, const double* k_centroids, int U, int G,
                        int n_chunks, int D, int agg, double* scores, dhsa_stream_t stream);

/* Chunk layout of a prefill.  NULL (or bounds
 * == NULL) = the static grid [0, block, 2*block, ..., L] (chunking.py:42-54).
 * Otherwise explicit per-unit boundary lists in check_boundaries form
 * (chunking.py:23-39; e.g. nms_boundaries over predictor scores,
 * chunking.py:57-89): unit u = kv head (with batch) has nchunks[u] chunks
 * bounds[u*bounds_stride + 0..nchunks[u]] (stride 0 = one shared list).  The
 * attention kernel also needs the query tile table qtiles[u][tiles_per_unit]
 * = int32 pairs (chunk l, 64-row tile t of chunk l), heaviest first, chunk
 * -1 = padding; chunk n and tile counts are host-known (prefill.py builds
 * it). */
typedef struct {
  const int32_t* bounds;
  int64_t bounds_stride;
  const int32_t* nchunks;
  const int32_t* qtiles;
  int32_t tiles_per_unit;
} dhsa_prefill_chunks;

/* Plan entries per (selection row, query chunk) needed for `budget` on the
 * static grid (block <= 64). */
int dhsa_prefill_plan_capacity(int64_t budget, int block);

/* Per (s, query chunk l): the <= 64-token blocks of the chunks of the walk
 * (masks.topk_row order: score desc, chunk asc) that some row of chunk l takes
 * tokens from, as int32x4 {start, len, W, flags}, in walk order (W = tokens of
 * the whole non-diagonal chunks ranked before, + 64 k for block k of a chunk;
 * flags bit0 = the diagonal chunk ranks before, bit1 = a block of the diagonal
 * chunk, those last).  Row i of chunk l (start b_l) takes
 * clamp(R_i - W - (bit0 ? i - b_l : 0), 0, len) lowest tokens of an entry
 * (a diagonal block: clamp(min(R_i - W, i - start), 0, len)) plus self, R_i =
 * min(budget, i+1) - 1 — exactly topk_row on the upsampled row.  s maps to
 * unit s (agg MAX / MEAN) or s / G (agg NONE) for the chunk layout.
 * n_chunks = chunk count (static) or the maximum over units (explicit).
 * plans [S][n_chunks][cap] int32x4, nplan [S][n_chunks] (-1 = overflow,
 * 0 = chunk l beyond the unit's count). */
int dhsa_prefill_plan(const double* scores, int S, int G, int agg, int n_chunks, int L,
                      int block, int64_t budget, const dhsa_prefill_chunks* chunks, int cap,
                      void* plans, int32_t* nplan, dhsa_stream_t stream);

/* The token sets the plans encode as DHSAMSK1 row bitsets (the reference's
 * mask file payload, serialization.py:80-94): out [S][L][ceil(L/8)] bytes,
 * token t of row i = bit t % 8 of byte t / 8 (self included). */
int dhsa_prefill_mask_bitsets(const void* plans, const int32_t* nplan, int cap, int S, int G,
                              int agg, int n_chunks, int L, int block, int64_t budget,
                              const dhsa_prefill_chunks* chunks, uint8_t* out,
                              dhsa_stream_t stream);

/* Block-sparse attention of every query row over its planned tokens:
 * softmax(K[idx] q / sqrt(D)) @ V[idx] (core.py:113-118) with tcgen05.mma
 * (bf16 operands from TMA-staged 128B-swizzled shared memory, fp32 TMEM
 * accumulators, P kept in TMEM), per (plan, <= 4 q heads).  out [U*G][L][D]
 * bf16.  counters: int32[2] zero at rest -> persistent grid (one CTA per SM
 * pulling plans, TMEM / barriers / K-V ring kept across plans); NULL -> one
 * CTA per (plan, head slice).  row_stats (float2 [U*G][L], or NULL): per
 * query row the softmax reference max m (log2 domain) and l = sum over the
 * selection of 2^(x - m), x = q.k log2(e) / sqrt(D).  chunks: as for
 * dhsa_prefill_plan (explicit bounds: any chunk lengths; query tiles and KV
 * blocks start at chunk starts, TMA boxes at any row). */
int dhsa_prefill_attn(const void* q, const void* k, const void* v, int U, int G, int L, int D,
                      int block, int agg, int64_t budget, int n_chunks,
                      const dhsa_prefill_chunks* chunks, const void* plans,
                      const int32_t* nplan, int cap, void* out, int32_t* counters,
                      float* row_stats, dhsa_stream_t stream);

/* Mask quality per query row (harness.attention_mass_recall / output_fidelity,
 * harness.py:265-285) from a sparse and a dense (budget >= L) prefill run:
 * recall = l_sel 2^(m_sel - m_all) / l_all, cosine(o_sel, o_all).
 * stats_*: float2 [rows] from dhsa_prefill_attn; out_*: bf16 [rows][D]. */
int dhsa_row_quality(const float* stats_sel, const float* stats_all, const void* out_sel,
                     const void* out_all, int64_t rows, int D, float* recall, float* cosine,
                     dhsa_stream_t stream);

/* Boundary-predictor inference (predictor.predict_sequence, predictor.py:
 * 270-283 over _forward 198-207, _mha_pool_forward 101-117, _fuse_forward
 * 151-161), fp64 like the reference.  keys [L][d]; wqkv [d][3d] = [Wq|Wk|Wv]
 * column blocks; wo [d][d]; w1 [4d+1][hidden]; b1, w2 [hidden]; probs
 * [L-2*window+1] = probabilities of positions window-1 .. L-window-1.
 * Needs L >= 2*window+1, d % heads == 0, d/heads <= 32, window^2 <= 32. */
int64_t dhsa_predictor_workspace_size(int L, int d, int window, int hidden);
int dhsa_predictor_forward(const double* keys, int L, int d, int window, int heads, int hidden,
                           const double* wqkv, const double* wo, const double* w1,
                           const double* b1, const double* w2, double b2, void* workspace,
                           double* probs, dhsa_stream_t stream);

/* Mask-quality metrics of the reference harness, fp64 (harness.py:265-306,
 * core.py:122-152), for the drop-in harness API:
 * dhsa_causal_probs   causal_attention_probs (core.py:122-136): out [L][L],
 *                      row i = softmax(q_i . k_j / sqrt(d)) over j <= i, 0 above;
 * dhsa_mask_recall     attention_mass_recall's per-row fraction (harness.py:
 *                      265-276): frac[i] = sum P[i, row_i] / sum P[i, 0..i] (0 if
 *                      the total is 0); rows as CSR (row_ptr [L+1] int64, idx int32);
 * dhsa_row_cosine      cosine_similarity (core.py:139-152) of `rows` row pairs;
 * dhsa_mean            deterministic mean of n values (out[0]);
 * dhsa_stack_reduce    aggregated_chunk_scores' max / mean over H stacked
 *                      [n] score arrays (harness.py:302-306). */
int dhsa_causal_probs(const double* q, const double* k, int L, int d, double* out,
                      dhsa_stream_t stream);
int dhsa_mask_recall(const double* probs, int64_t ld, int L, const int64_t* row_ptr,
                     const int32_t* idx, double* frac, dhsa_stream_t stream);
int dhsa_row_cosine(const double* a, const double* b, int64_t rows, int d, double* out,
                    dhsa_stream_t stream);
int dhsa_mean(const double* x, int64_t n, double* out, dhsa_stream_t stream);
int dhsa_stack_reduce(const double* x, int H, int64_t n, int agg, double* out,
                      dhsa_stream_t stream);

/* softmax_row (core.py:69-77) of `rows` fp64 rows of n scores each:
 * out = exp(s - max s) / sum(exp(s - max s)), per row. */
int dhsa_softmax_rows(const double* scores, int rows, int64_t n, double* out,
                      dhsa_stream_t stream);

/* f_upsample (masks.upsample, masks.py:87-100): out[i][j] = s[chunk(i)][chunk(j)]
 * for an n x n chunk-score matrix and bounds [n+1]; out is L x L fp64.  Only
 * the drop-in API uses it — the selection kernels never materialise it. */
int dhsa_upsample(const double* scores, const int32_t* bounds, int n, int L,
                  double* out, dhsa_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* DHSA_B200_H */
