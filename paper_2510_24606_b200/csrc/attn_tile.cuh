// The per-tile math of the bf16 decode attention kernels (attn_mma.cu,
// attn_stream.cu): one 64-token K/V tile staged by TMA in a 128B-swizzled
// [K boxes | V boxes] stage, 4 consumer warps each owning 16 tokens.
//
// S = Q K^T with Q (GH <= 8 heads, padded to 16 rows) as the mma.sync A
// operand held in registers, online softmax in the log2 domain, O += P V with
// P re-packed from the S accumulators (no shared-memory round trip).
// Reference: the row body of dense_attention (core.py:113-118).
#pragma once

#include "common.cuh"

namespace dhsa {

template <int D>
struct DecodeTile {
  static constexpr int NB = D / 64;               // 128-byte column boxes per row
  static constexpr int BOX = 64 * 128;            // one box: 64 token rows x 128 B
  static constexpr int STAGE_BYTES = 2 * NB * BOX;  // K + V
  static constexpr int KS = D / 16;               // k-steps of QK^T
  static constexpr int NT = D / 8;                // n-tiles of PV

  // A fragments of Q for head rows lane/4 (rows >= GH are zero).
  __device__ static __forceinline__ void load_q(const __nv_bfloat16* __restrict__ q, int item,
                                                int GH, int lane, uint32_t (&qa)[KS][2]) {
    const int hrow = lane >> 2;
    const bool live = hrow < GH;
    const __nv_bfloat16* qrow = q + ((int64_t)item * GH + (live ? hrow : 0)) * D;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k0 = ks * 16 + 2 * (lane & 3);
      qa[ks][0] = live ? *reinterpret_cast<const uint32_t*>(qrow + k0) : 0u;
      qa[ks][1] = live ? *reinterpret_cast<const uint32_t*>(qrow + k0 + 8) : 0u;
    }
  }

  // Fold one staged tile (count valid tokens) into (m, l, o) of this warp.
  __device__ static __forceinline__ void update(uint32_t kb, int count, int warp, int lane,
                                                const uint32_t (&qa)[KS][2], float scale_log2,
                                                float& m, float& l, float (&o)[NT][4]) {
    if (warp * 16 >= count) return;
    const uint32_t vb = kb + NB * BOX;
    const int mi = lane >> 3, r8 = lane & 7;
    const int tok_k = warp * 16 + 8 * (mi >> 1) + r8;  // K: matrix (nt, khalf)
    const int tok_v = warp * 16 + 8 * (mi & 1) + r8;   // V: matrix (tokhalf, ntile)
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int dch = 2 * ks + (mi & 1);
      const uint32_t addr = kb + (dch >> 3) * BOX + tok_k * 128 + (((dch & 7) ^ (tok_k & 7)) << 4);
      uint32_t b0, b1, b2, b3;
      ldsm_x4(addr, b0, b1, b2, b3);
      mma_bf16(sc[0], qa[ks][0], 0u, qa[ks][1], 0u, b0, b1);
      mma_bf16(sc[1], qa[ks][0], 0u, qa[ks][1], 0u, b2, b3);
    }
    // scores of head lane/4 for tokens warp*16 + 8*nt + 2*(lane&3) + {0,1}
    float p[2][2];
    float tmax = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tok = warp * 16 + 8 * nt + 2 * (lane & 3) + e;
        const float v = tok < count ? sc[nt][e] * scale_log2 : -INFINITY;
        p[nt][e] = v;
        tmax = fmaxf(tmax, v);
      }
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    const float mn = fmaxf(m, tmax);
    const float corr = exp2f(m - mn);
    float psum = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        p[nt][e] = exp2f(p[nt][e] - mn);
        psum += p[nt][e];
      }
    l = l * corr + psum;
    m = mn;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      o[j][0] *= corr;
      o[j][1] *= corr;
    }
    const uint32_t pa0 = pack_bf16(p[0][0], p[0][1]);
    const uint32_t pa2 = pack_bf16(p[1][0], p[1][1]);
#pragma unroll
    for (int np = 0; np < NT / 2; ++np) {
      const int dch = 2 * np + (mi >> 1);
      const uint32_t addr = vb + (dch >> 3) * BOX + tok_v * 128 + (((dch & 7) ^ (tok_v & 7)) << 4);
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(addr, b0, b1, b2, b3);
      mma_bf16(o[2 * np], pa0, 0u, pa2, 0u, b0, b1);
      mma_bf16(o[2 * np + 1], pa0, 0u, pa2, 0u, b2, b3);
    }
  }

  // Per-warp record (m, l, o[h][D]) into red[(warp * GH + h) * (D + 2)].
  // l must already be reduced over the 4 lanes of a head row.
  __device__ static __forceinline__ void warp_record(float* red, int warp, int lane, int GH,
                                                     float m, float l, const float (&o)[NT][4]) {
    const int h = lane >> 2;
    if (h >= GH) return;
    float* r = red + (warp * GH + h) * (D + 2);
    if ((lane & 3) == 0) {
      r[0] = m;
      r[1] = l;
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      r[2 + j * 8 + 2 * (lane & 3)] = o[j][0];
      r[2 + j * 8 + 2 * (lane & 3) + 1] = o[j][1];
    }
  }
};

// Combine the 4 warp records of head h at dimension d: returns (m*, l, acc).
template <int D>
__device__ __forceinline__ void combine4(const float* red, int GH, int h, int d, float& mstar,
                                         float& lsum, float& acc) {
  constexpr int rec = D + 2;
  mstar = -INFINITY;
#pragma unroll
  for (int w = 0; w < 4; ++w) mstar = fmaxf(mstar, red[(w * GH + h) * rec]);
  lsum = 0.f;
  acc = 0.f;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const float* r = red + (w * GH + h) * rec;
    if (r[0] == -INFINITY) continue;
    const float wgt = exp2f(r[0] - mstar);
    lsum += wgt * r[1];
    acc += wgt * r[2 + d];
  }
}

}  // namespace dhsa
