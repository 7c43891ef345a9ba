// Internal host-side launchers (C++ linkage; not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dsk {

struct WLEntry;

// Launch-time device queries and one-time kernel setup.  All caches are keyed
// by the CURRENT device and guarded by one mutex (api.cu), so launchers are
// thread-safe and correct when one process drives several GPUs.
int num_sms();          // SMs of the current device
int max_smem_optin();   // opt-in shared memory per block of the current device
// Allow the largest dynamic smem the kernel can use (opt-in limit minus its
// static smem) and the full smem carveout; done once per (kernel, device).
void prepare_kernel(const void* kern);
template <typename F>
inline void allow_max_dyn_smem(F* kern) {
  prepare_kernel(reinterpret_cast<const void*>(kern));
}
// Resident blocks per SM (cudaOccupancyMaxActiveBlocksPerMultiprocessor after
// prepare_kernel), cached per (kernel, device, threads, smem); >= 1.
int occupancy(const void* kern, int threads, size_t smem);
template <typename F>
inline int occupancy_of(F* kern, int threads, size_t smem) {
  return occupancy(reinterpret_cast<const void*>(kern), threads, smem);
}
// cuTensorMapEncodeTiled through the runtime's driver entry point (resolved
// once, thread-safe); nullptr if unavailable.
void* tensor_map_encoder();
// Launch with programmatic stream serialization (PDL) and an optional
// cluster shape; DYNSPLIT_NO_PDL=1 disables PDL (A/B measurements).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t st, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster_x;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
// After every launch: returns cudaGetLastError(); with DYNSPLIT_DEBUG=1 in the
// environment also synchronises the stream so asynchronous faults are
// attributed to the launcher that caused them.  Errors are recorded for
// dynsplit_last_error().
cudaError_t post_launch(const char* where, cudaStream_t st);
// Empty kernel launched without PDL (dynsplit_stream_fence).
cudaError_t launch_fence(cudaStream_t st);
// decode (decode_kernels.cu, select_kernels.cu, attn_kernels.cu)
cudaError_t launch_score_blocks(int dtype, int G, const void* q, const void* dig, const int32_t* nb,
                                float* scores, int B, int Hq, int Hkv, int maxb, int nb_hint,
                                int mean_mode, cudaStream_t st);  // nb_hint: expected blocks per sequence
size_t select_smem_needed(int maxb, int G);  // (size_t)-1 if it cannot fit
// S: capacity (the plan must tile [0, L) with L <= S); err: device error word
cudaError_t launch_select(int G, const float* scores, const int32_t* bs, const int32_t* nb,
                          const int32_t* pf, int B, int Hq, int Hkv, int maxb, int S, int max_sel,
                          int max_wl, int P, int budget, int blk_lo, int blk_hi,
                          int32_t* sel_blocks, int32_t* n_sel, int32_t* marg, int32_t* keep,
                          int32_t* wl_count, WLEntry* wl, int* err, cudaStream_t st);
cudaError_t launch_decode_attn(int dtype, int G, const void* q, const void* Kp, const void* Vp,
                               const int16_t* pv, const int32_t* n_pages, const int32_t* wl_hdr,
                               const int32_t* wl_count, const WLEntry* wl, int dense, int B, int Hq, int Hkv,
                               int max_pages, int P, float scale, float* part_o, float* part_lse,
                               int* counters, float* o, float* lse, cudaStream_t st);
// Fused decode layer (a5 + a6 + a7 + a8 in one kernel, fused_kernels.cu).
// Returns cudaErrorNotSupported (nothing launched) when the shape or mode is
// outside what the fused kernel handles; the caller then runs the three
// kernels.  scores: [B][Hq][sstride] fp32 (sstride >= maxb rounded up to 32);
// fscratch: fused_scratch_bytes(); bar: 4 zero-initialised group-barrier
// words per (b, KV head); nb_hint: expected blocks per sequence.
size_t fused_scratch_bytes(int B, int Hq, int maxb);
cudaError_t launch_decode_fused(int dtype, int digest_mode, int G, const void* q, const void* dig,
                                const int32_t* bs, const int32_t* nb, const int32_t* pf, const void* Kp,
                                const void* Vp, int B, int Hq, int Hkv, int maxb, int max_pages, int S, int P,
                                int budget, int gqa_mode, int budget_mode, int nb_hint, float scale, float* scores,
                                int sstride,
                                void* fscratch, int* counters, int* bar, float* part_o, float* part_lse,
                                int32_t* n_sel, int32_t* marg, int32_t* keep, int32_t* wl_count, WLEntry* wl,
                                float* o, float* lse, int* err, cudaStream_t st);
cudaError_t launch_merge(const float* o_parts, const float* lse_parts, int n_parts, int rows, int d,
                         float* o, float* lse, cudaStream_t st);

// prefill (build_kernels.cu)
cudaError_t launch_weight_table(const int32_t* tokens, const int32_t* delim_ids, int n_ids,
                                const float* s, uint8_t* w10, int B, int S, cudaStream_t st);
cudaError_t launch_segment(const int32_t* tokens, const int32_t* delim_ids, int n_ids,
                           const uint8_t* w10, int B, int S, int C, int delta, int lam_num,
                           int lam_den, int maxb, int32_t* next_ws, int32_t* block_starts,
                           int32_t* n_blocks, cudaStream_t st);
// L_end: the plan must tile [0, L_end); err: device error word or nullptr
cudaError_t launch_map_pages(const int32_t* bs, const int32_t* nb, int B, int maxb, int maxp, int P,
                             int L_end, int32_t* page_first, int32_t* page_block, int16_t* page_valid,
                             int32_t* n_pages, int* err, cudaStream_t st);
cudaError_t launch_repack_digest(int dtype, const void* K, const void* V, const int32_t* bs,
                                 const int32_t* nb, const int32_t* pf, int B, int S, int Hkv,
                                 int maxb, int maxp, int P, int mean_mode, void* Kp, void* Vp, void* dig,
                                 int* err, cudaStream_t st);

// NEXT-1 decode-time append (append_kernels.cu)
constexpr int kAppendMaxLayers = 64;
size_t append_ws_bytes(int B);
int append_max_tail(int dtype);
cudaError_t launch_plan_append(const int32_t* tokens, const int32_t* delim_ids, int n_ids, const uint8_t* w10,
                               int B, int S, int maxb, int maxp, int C, int delta, int lam_num, int lam_den,
                               int P, int L_prev, int L, int32_t* block_starts, int32_t* n_blocks,
                               int32_t* page_first, int32_t* page_block, int16_t* page_valid,
                               int32_t* n_pages, int32_t* ws, int* err, cudaStream_t st,
                               const int32_t* Lp_dev = nullptr);  // Lp_dev: device-side L_prev (decode loops)
cudaError_t launch_kv_append(int dtype, int n_layers, const void* const* K_new, const void* const* V_new,
                             int n_new, int B, int Hkv, int maxb, int maxp, int P, int L_prev, int max_tail,
                             const int32_t* block_starts, const int32_t* n_blocks, const int32_t* page_first,
                             const int32_t* ws, void* const* Kp, void* const* Vp, void* const* dig,
                             int mean_mode, cudaStream_t st, const int32_t* Lp_dev, int* err);

// NEXT-3 offloaded KV + cross-step reuse (offload_kernels.cu)
cudaError_t launch_reuse_plan(const int32_t* wl_hdr, const int32_t* wl_count, const WLEntry* wl, int B, int Hkv,
                              int max_pages, int n_slots, int reuse, int truncate, int32_t* reusable,
                              int32_t* map, int32_t* freelist, int32_t* slot_page, int32_t* fetch,
                              int32_t* fetch_count, int32_t* stats, int32_t* reuse_len, int32_t* c_hdr,
                              int32_t* c_count, WLEntry* c_wl, int* err, cudaStream_t st);
cudaError_t launch_fetch_pages(int dtype, const void* Kh, const void* Vh, const int16_t* page_valid,
                               const int32_t* n_pages, const int32_t* fetch, const int32_t* fetch_count,
                               int dense, int B, int Hkv, int max_pages, int n_slots, int P, void* Kc, void* Vc,
                               cudaStream_t st);

// prefill scoring (score_kernels.cu)
size_t score_ws_bytes(int Ls, int B, int S, int Hq);
cudaError_t launch_score_delimiters(const int32_t* tokens, const int32_t* delim_ids, int n_ids,
                                    const void* Qs, const void* Ks, int Ls, int B, int S, int Hq,
                                    int Hkv, int W, int R, float alpha, float* out, void* ws,
                                    cudaStream_t st);

}  // namespace dsk
