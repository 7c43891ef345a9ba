// Fused decode layer (rows a5 + a6 + a7 + a8 in one kernel) -- see below.
#include "common.cuh"
#include "kernels.h"

namespace dsk {

cudaError_t launch_decode_fused(int dtype, int digest_mode, int G, const void* q, const void* dig,
                                const int32_t* bs, const int32_t* nb, const int32_t* pf, const void* Kp,
                                const void* Vp, int B, int Hq, int Hkv, int maxb, int max_pages, int P,
                                int budget, float scale, float* scores, int* counters, int* bar,
                                float* part_o, float* part_lse, int32_t* n_sel, int32_t* marg, int32_t* keep,
                                int32_t* wl_hdr, int32_t* wl_count, WLEntry* wl, float* o, float* lse,
                                int* err, cudaStream_t st) {
  return cudaErrorNotSupported;
}

}  // namespace dsk
