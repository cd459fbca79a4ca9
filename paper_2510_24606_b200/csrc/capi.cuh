// Host-side helpers shared by the C-ABI entry points.
#pragma once

#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace dhsa {

void set_error(const char* fmt, ...);

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return DHSA_ECUDA;
  }
  return DHSA_OK;
}

#define DHSA_REQUIRE(cond, ...)      \
  do {                               \
    if (!(cond)) {                   \
      ::dhsa::set_error(__VA_ARGS__); \
      return DHSA_EINVAL;            \
    }                                \
  } while (0)

// 2-D TMA view [rows][D] of a 16-bit tensor (bf16 / fp16): 64 x 64-element
// boxes (64 rows x 128 B) with 128-byte swizzle (tmap.cu).
int make_tmap_2d(CUtensorMap* map, const void* base, int64_t rows, int D,
                 CUtensorMapDataType dtype);

inline bool valid_layout(const dhsa_layout& l) {
  if (!l.plen) return false;
  if (l.bounds) return l.nchunks != nullptr;
  return l.block >= 1;
}

}  // namespace dhsa
