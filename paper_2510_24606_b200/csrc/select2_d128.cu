// Instantiations of the compact certified select (select2.cuh) for head dim
// 128 (one file per head dim: parallel compilation).
#include "select2.cuh"

#include <cstdlib>

namespace dhsa {

template <int D, int G, int AGG>
int launch_select2(const SketchArgs& a, int U, cudaStream_t s, int* rc) {
  // the massive-tie fallback keeps its keys (and split-KV candidate mode its
  // takes) in global scratch; longer units use the generic select
  if (!a.gscratch || a.n_max > kS3WideMaxChunks) return 0;
  if (const char* e = getenv("DHSA_SELECT2"))
    if (atoi(e) == 0) return 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)U);
  const bool wide = a.n_max > kS3MaxChunks;
  const int per = a.n_max <= kS3Threads * kS3PerS ? kS3PerS
                  : a.n_max <= kS3ThreadsM * kS3PerM ? kS3PerM : kS3Per;
  cfg.blockDim = dim3(wide ? kS3WideThreads : per == kS3PerM ? kS3ThreadsM : kS3Threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e =
      wide ? cudaLaunchKernelEx(&cfg, sketch_select3_kernel<D, G, AGG, kS3WideThreads, kS3WidePer>, a)
      : per == kS3PerS ? cudaLaunchKernelEx(&cfg, sketch_select3_kernel<D, G, AGG, kS3Threads, kS3PerS>, a)
      : per == kS3PerM ? cudaLaunchKernelEx(&cfg, sketch_select3_kernel<D, G, AGG, kS3ThreadsM, kS3PerM>, a)
                       : cudaLaunchKernelEx(&cfg, sketch_select3_kernel<D, G, AGG, kS3Threads, kS3Per>, a);
  if (e != cudaSuccess) {
    set_error("dhsa_decode_step_bf16(select): %s", cudaGetErrorString(e));
    *rc = DHSA_ECUDA;
    return 1;
  }
  *rc = check_launch("dhsa_decode_step_bf16(select)");
  return 1;
}

#define DHSA_SELECT2_INST(G, AGG) \
  template int launch_select2<128, G, AGG>(const SketchArgs&, int, cudaStream_t, int*);
#define DHSA_SELECT2_AGGS(G) \
  DHSA_SELECT2_INST(G, DHSA_AGG_NONE) DHSA_SELECT2_INST(G, DHSA_AGG_MAX) DHSA_SELECT2_INST(G, DHSA_AGG_MEAN)
DHSA_SELECT2_AGGS(1)
DHSA_SELECT2_AGGS(2)
DHSA_SELECT2_AGGS(4)
DHSA_SELECT2_AGGS(8)

}  // namespace dhsa
