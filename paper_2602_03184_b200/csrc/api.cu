// C ABI of libdynsplit.so (declared and documented in include/dynsplit.h).
// Validation, workspace carving and launch sequencing only; every step of the
// path runs in the kernels of decode_kernels.cu / build_kernels.cu /
// score_kernels.cu.
#include "../../include/dynsplit.h"
#include "common.cuh"
#include "kernels.h"

#include <math.h>
#include <nvtx3/nvToolsExt.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <utility>

namespace dsk {

// ---------------------------------------------------------------- per-device launch caches
// One mutex guards every cache; keys include the current device, so a thread
// driving device 1 never reuses device 0's attributes or occupancy.
namespace {
std::mutex g_mu;
std::map<int, int> g_sms, g_smem;
std::set<std::pair<const void*, int>> g_prepared;
std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;

int device_attr(std::map<int, int>& cache, cudaDeviceAttr attr, int fallback) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return fallback;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, attr, dev) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = fallback;
  }
  cache[dev] = n;
  return n;
}
}  // namespace

int num_sms() { return device_attr(g_sms, cudaDevAttrMultiProcessorCount, 148); }
int max_smem_optin() { return device_attr(g_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, 227 * 1024); }

void prepare_kernel(const void* kern) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int optin = max_smem_optin();
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_prepared.insert({kern, dev}).second) return;
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, kern) == cudaSuccess)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes);
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaGetLastError();
}

int occupancy(const void* kern, int threads, size_t smem) {
  prepare_kernel(kern);
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(kern, dev, threads, smem);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
  }
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 1;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_occ[key] = n;
  return n;
}

void* tensor_map_encoder() {
  static void* fn = []() -> void* {  // thread-safe one-time initialisation
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return f;
  }();
  return fn;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("DYNSPLIT_NO_PDL");
    return !(e && *e && *e != '0');
  }();
  return on;
}

static thread_local char g_last_error[512] = "";
const char* last_error();

cudaError_t post_launch(const char* where, cudaStream_t st) {
  static const int debug = [] {
    const char* e = getenv("DYNSPLIT_DEBUG");
    return (e && *e && *e != '0') ? 1 : 0;
  }();
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && debug) {
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  if (e != cudaSuccess) snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where, cudaGetErrorString(e));
  return e;
}

const char* last_error() { return g_last_error; }

}  // namespace dsk

using namespace dsk;

namespace {

// NVTX range per C-ABI call (a push/pop pair; free without an attached tool)
struct NvtxRange {
  explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define DSK_NVTX NvtxRange dsk_nvtx_range_(__func__)

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

inline size_t esize(const dynsplit_shape* s) { return s->kv_dtype == DYNSPLIT_BF16 ? 2 : 4; }

dynsplit_status check_shape(const dynsplit_shape* s) {
  if (!s) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (s->B < 1 || s->S < 1) return DYNSPLIT_ERR_EMPTY_SEQUENCE;
  if (s->Hq < 1 || s->Hkv < 1 || s->Hq % s->Hkv) return DYNSPLIT_ERR_DIMENSION_MISMATCH;
  const int g = s->Hq / s->Hkv;
  if (g != 1 && g != 2 && g != 4 && g != 8) return DYNSPLIT_ERR_DIMENSION_MISMATCH;
  if (s->d != kD) return DYNSPLIT_ERR_DIMENSION_MISMATCH;
  if (s->kv_dtype != DYNSPLIT_BF16 && s->kv_dtype != DYNSPLIT_FP32) return DYNSPLIT_ERR_UNSUPPORTED;
  return DYNSPLIT_OK;
}

dynsplit_status check_cfg(const dynsplit_config* c) {
  if (!c) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (c->C < 1 || c->delta < 0 || c->delta >= c->C) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (c->C + c->delta > 65535) return DYNSPLIT_ERR_UNSUPPORTED;
  if (c->lambda_den < 1 || c->lambda_num < 0 || c->lambda_num > c->lambda_den)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (c->page_size < 1 || c->page_size > 64 || (c->page_size & (c->page_size - 1)))
    return DYNSPLIT_ERR_UNSUPPORTED;  // P: power of two in [1, 64]
  if (c->W < 1 || c->R < 1 || !(c->alpha_pen >= 0.f)) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (c->digest_mode != 0 && c->digest_mode != 1) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (c->page_cap < 0) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if ((c->gqa_mode != 0 && c->gqa_mode != 1) || (c->budget_mode != 0 && c->budget_mode != 1))
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  return DYNSPLIT_OK;
}

inline dynsplit_status cuda_status(cudaError_t e) {
  return e == cudaSuccess ? DYNSPLIT_OK : DYNSPLIT_ERR_CUDA;
}

#define DSK_TRY(x)                               \
  do {                                           \
    dynsplit_status _s = (x);                    \
    if (_s != DYNSPLIT_OK) return _s;            \
  } while (0)

inline int* err_word(void* ws) { return static_cast<int*>(ws); }
inline char* ws_body(void* ws) { return static_cast<char*>(ws) + kWsHdr; }

// Worklist capacity per (b, KV head): every page of the sequence (the union
// of the selected pages is a subset).  Budget-independent, so the attention
// kernel knows each (b, KV head)'s entry base without reading the header.
inline int max_wl_of(const dynsplit_shape* s, const dynsplit_config* c, int budget) {
  (void)budget;
  return dynsplit_max_pages(s->S, c);
}

struct WorklistView {
  int32_t* hdr;
  int32_t* count;
  WLEntry* entries;
};
inline WorklistView worklist_view(void* wl, const dynsplit_shape* s) {
  char* p = static_cast<char*>(wl);
  WorklistView v;
  v.hdr = reinterpret_cast<int32_t*>(p);
  v.count = v.hdr + 64;
  v.entries = reinterpret_cast<WLEntry*>(p + kAlign + align_up((size_t)s->B * s->Hkv * 4));
  return v;
}

// ---- workspace layouts: [kWsHdr header: device error word][body]
// scores rows padded to 32 floats (the fused decode kernel's row stride)
inline int score_stride(const dynsplit_shape* s, const dynsplit_config* c) {
  return (dynsplit_max_blocks(s->S, c) + 31) & ~31;
}
size_t select_body(const dynsplit_shape* s, const dynsplit_config* c) {
  return align_up((size_t)s->B * s->Hq * score_stride(s, c) * 4) + align_up((size_t)s->B * s->Hq * 16);
}
size_t select_ws(const dynsplit_shape* s, const dynsplit_config* c) { return kWsHdr + select_body(s, c); }
// Decode body: [split-merge counters, fixed kMaxCounters ints][part_o][part_lse].
// Counters sit at a shape-independent offset so that a zero-filled workspace
// stays valid when reused with any shape.  The fused decode kernel keeps its
// per-(b, KV head) group-barrier words in the upper half.
constexpr size_t kMaxCounters = 65536;
size_t decode_body(const dynsplit_shape* s) {
  return kMaxCounters * 4 + align_up((size_t)s->B * s->Hq * kMaxSplit * kD * 4) +
         align_up((size_t)s->B * s->Hq * kMaxSplit * 4);
}
size_t decode_ws(const dynsplit_shape* s) { return kWsHdr + decode_body(s); }
size_t segment_body(const dynsplit_shape* s) { return align_up((size_t)s->B * s->S * 4); }
size_t segment_ws(const dynsplit_shape* s) { return kWsHdr + segment_body(s); }
size_t score_body(const dynsplit_shape* s) { return align_up(score_ws_bytes(s->n_score_layers, s->B, s->S, s->Hq)); }
size_t score_ws(const dynsplit_shape* s) { return kWsHdr + score_body(s); }
size_t build_ws(const dynsplit_shape* s) {
  // header + scoring partials + delim scores (if not returned) + segment next[]
  return kWsHdr + score_body(s) + align_up((size_t)s->B * s->S * 4) + segment_body(s);
}
// dynsplit_decode_layer: header, decode body (counters at a fixed offset), select body.
// (+ the fused kernel's moments / selection bitmasks / marginal info)
size_t layer_ws(const dynsplit_shape* s, const dynsplit_config* c) {
  return kWsHdr + decode_body(s) + select_body(s, c) +
         align_up(fused_scratch_bytes(s->B, s->Hq, dynsplit_max_blocks(s->S, c)));
}
// NEXT-3 reuse plan: [reusable counts BH][map BH x max_pages][freelist BH x max_pages]
size_t reuse_body(const dynsplit_shape* s, const dynsplit_config* c) {
  const size_t bh = (size_t)s->B * s->Hkv, mp = (size_t)dynsplit_max_pages(s->S, c);
  return align_up(bh * 4) + 2 * align_up(bh * mp * 4);
}
size_t offload_ws(const dynsplit_shape* s, const dynsplit_config* c) {
  return kWsHdr + decode_body(s) + select_body(s, c) + reuse_body(s, c);
}
size_t step_host_extra(const dynsplit_shape* s) {
  return align_up((size_t)s->B * s->Hq * kD * esize(s)) + align_up((size_t)s->B * s->Hq * kD * 4) +
         align_up((size_t)s->B * s->Hq * 4) + 3 * align_up((size_t)s->B * s->Hq * 4);
}

}  // namespace

namespace dsk {
struct W10Table {
  uint8_t w[64];
};
__global__ void k_fill_w10(W10Table t, int n_ids, uint8_t* w10) {
  if (threadIdx.x < n_ids) w10[(size_t)blockIdx.x * n_ids + threadIdx.x] = t.w[threadIdx.x];
}
}  // namespace dsk

extern "C" {

void dynsplit_default_config(dynsplit_config* c) {
  if (!c) return;
  c->W = 8;
  c->R = 128;
  c->alpha_pen = 1.0f;
  c->C = 32;
  c->delta = 14;
  c->lambda_num = 1;
  c->lambda_den = 2;
  c->page_size = 16;
  c->digest_mode = 0;
  c->page_cap = 0;
  c->gqa_mode = 0;
  c->budget_mode = 0;
}

int32_t dynsplit_max_blocks(int32_t S, const dynsplit_config* c) {
  if (!c || c->C - c->delta < 1 || S < 0) return 0;
  return S / (c->C - c->delta) + 1;
}

int32_t dynsplit_max_pages(int32_t S, const dynsplit_config* c) {
  if (!c || c->page_size < 1) return 0;
  if (c->page_cap > 0) return c->page_cap;
  return dynsplit_max_blocks(S, c) + (S + c->page_size - 1) / c->page_size;
}

int32_t dynsplit_max_selected(int32_t budget, int32_t S, const dynsplit_config* c) {
  if (!c || c->C - c->delta < 1) return 0;
  const int32_t maxb = dynsplit_max_blocks(S, c);
  const long long v = (long long)(budget > 0 ? budget - 1 : 0) / (c->C - c->delta) + 2;
  return (int32_t)(v < maxb ? v : maxb);
}

size_t dynsplit_worklist_bytes(const dynsplit_shape* s, const dynsplit_config* c, int32_t budget) {
  if (check_shape(s) != DYNSPLIT_OK || check_cfg(c) != DYNSPLIT_OK || budget < 1) return 0;
  return kAlign + align_up((size_t)s->B * s->Hkv * 4) +
         (size_t)s->B * s->Hkv * max_wl_of(s, c, budget) * sizeof(WLEntry);
}

size_t dynsplit_workspace_bytes(int32_t op, const dynsplit_shape* s, const dynsplit_config* c,
                                int32_t budget) {
  (void)budget;
  if (check_shape(s) != DYNSPLIT_OK || check_cfg(c) != DYNSPLIT_OK) return 0;
  switch (op) {
    case DYNSPLIT_OP_SCORE_DELIMITERS: return score_ws(s);
    case DYNSPLIT_OP_SEGMENT: return segment_ws(s);
    case DYNSPLIT_OP_BUILD_BLOCKS: return build_ws(s);
    case DYNSPLIT_OP_SELECT: return select_ws(s, c);
    case DYNSPLIT_OP_DECODE_ATTN: return decode_ws(s);
    case DYNSPLIT_OP_DECODE_LAYER: return layer_ws(s, c);
    case DYNSPLIT_OP_APPEND: return kWsHdr + append_ws_bytes(s->B);
    case DYNSPLIT_OP_MAP_PAGES: return kWsHdr;
    case DYNSPLIT_OP_REPACK: return kWsHdr;
    case DYNSPLIT_OP_REUSE: return kWsHdr + reuse_body(s, c);
    case DYNSPLIT_OP_DECODE_OFFLOAD: return offload_ws(s, c);
    default: return 0;
  }
}

size_t dynsplit_step_host_workspace_bytes(const dynsplit_shape* s, const dynsplit_config* c,
                                          int32_t budget) {
  if (check_shape(s) != DYNSPLIT_OK || check_cfg(c) != DYNSPLIT_OK || budget < 1) return 0;
  return layer_ws(s, c) + step_host_extra(s);
}

const char* dynsplit_status_string(int32_t st) {
  switch (st) {
    case DYNSPLIT_OK: return "ok";
    case DYNSPLIT_ERR_INVALID_ARGUMENT: return "invalid argument";
    case DYNSPLIT_ERR_DIMENSION_MISMATCH: return "dimension mismatch";
    case DYNSPLIT_ERR_EMPTY_SEQUENCE: return "empty sequence";
    case DYNSPLIT_ERR_WORKSPACE_TOO_SMALL: return "workspace too small";
    case DYNSPLIT_ERR_UNSUPPORTED: return "unsupported";
    case DYNSPLIT_ERR_CUDA: return "cuda error";
    default: return "unknown status";
  }
}

const char* dynsplit_version(void) { return "dynsplit-b200 0.2 (sm_100a)"; }

const char* dynsplit_last_error(void) { return dsk::last_error(); }

int32_t dynsplit_read_device_error(const void* ws, void* stream) {
  DSK_NVTX;
  if (!ws) return -1;
  int32_t v = 0;
  if (cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess ||
      cudaMemcpy(&v, ws, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return v;
}

dynsplit_status dynsplit_clear_device_error(void* ws, void* stream) {
  DSK_NVTX;
  if (!ws) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  return cuda_status(cudaMemsetAsync(ws, 0, sizeof(int32_t), static_cast<cudaStream_t>(stream)));
}

dynsplit_status dynsplit_stream_fence(void* stream) {
  DSK_NVTX;
  return cuda_status(launch_fence(static_cast<cudaStream_t>(stream)));
}

// ------------------------------------------------------------------ prefill
dynsplit_status dynsplit_score_delimiters(const dynsplit_shape* s, const dynsplit_config* c,
                                          const int32_t* tokens, const int32_t* delim_ids,
                                          int32_t n_ids, const void* Qs, const void* Ks,
                                          float* out, void* ws, size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!tokens || !delim_ids || !Qs || !Ks || !out || !ws) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (n_ids < 1 || n_ids > 64 || s->n_score_layers < 1) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (s->kv_dtype != DYNSPLIT_BF16 || c->W > 8) return DYNSPLIT_ERR_UNSUPPORTED;
  if (ws_bytes < score_ws(s)) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  return cuda_status(launch_score_delimiters(tokens, delim_ids, n_ids, Qs, Ks, s->n_score_layers,
                                             s->B, s->S, s->Hq, s->Hkv, c->W, c->R, c->alpha_pen,
                                             out, ws_body(ws), static_cast<cudaStream_t>(stream)));
}

dynsplit_status dynsplit_weight_table(const dynsplit_shape* s, const int32_t* tokens,
                                      const int32_t* delim_ids, int32_t n_ids,
                                      const float* delim_scores, uint8_t* w10, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  if (!tokens || !delim_ids || !delim_scores || !w10) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (n_ids < 1 || n_ids > 64) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  return cuda_status(launch_weight_table(tokens, delim_ids, n_ids, delim_scores, w10, s->B, s->S,
                                         static_cast<cudaStream_t>(stream)));
}

dynsplit_status dynsplit_segment(const dynsplit_shape* s, const dynsplit_config* c,
                                 const int32_t* tokens, const int32_t* delim_ids, int32_t n_ids,
                                 const uint8_t* w10, int32_t* block_starts, int32_t* n_blocks,
                                 void* ws, size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!tokens || !delim_ids || !w10 || !block_starts || !n_blocks || !ws)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (n_ids < 1 || n_ids > 64) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < segment_ws(s)) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  return cuda_status(launch_segment(tokens, delim_ids, n_ids, w10, s->B, s->S, c->C, c->delta,
                                    c->lambda_num, c->lambda_den, dynsplit_max_blocks(s->S, c),
                                    reinterpret_cast<int32_t*>(ws_body(ws)), block_starts, n_blocks,
                                    static_cast<cudaStream_t>(stream)));
}

}  // extern "C"

static dynsplit_status map_pages_impl(const dynsplit_shape* s, const dynsplit_config* c,
                                      const int32_t* block_starts, const int32_t* n_blocks,
                                      int32_t* page_first, int32_t* page_block, int16_t* page_valid,
                                      int32_t* n_pages, int* err, void* stream) {
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!block_starts || !n_blocks || !page_first || !page_block || !page_valid || !n_pages)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  return cuda_status(launch_map_pages(block_starts, n_blocks, s->B, dynsplit_max_blocks(s->S, c),
                                      dynsplit_max_pages(s->S, c), c->page_size, s->S, page_first,
                                      page_block, page_valid, n_pages, err,
                                      static_cast<cudaStream_t>(stream)));
}

static dynsplit_status repack_impl(const dynsplit_shape* s, const dynsplit_config* c, const void* K,
                                   const void* V, const int32_t* block_starts, const int32_t* n_blocks,
                                   const int32_t* page_first, void* Kp, void* Vp, void* digests, int* err,
                                   void* stream) {
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!K || !V || !block_starts || !n_blocks || !page_first || !Kp || !Vp || !digests)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  return cuda_status(launch_repack_digest(s->kv_dtype, K, V, block_starts, n_blocks, page_first,
                                          s->B, s->S, s->Hkv, dynsplit_max_blocks(s->S, c),
                                          dynsplit_max_pages(s->S, c), c->page_size, c->digest_mode, Kp, Vp,
                                          digests, err, static_cast<cudaStream_t>(stream)));
}

extern "C" {

dynsplit_status dynsplit_map_pages(const dynsplit_shape* s, const dynsplit_config* c,
                                   const int32_t* block_starts, const int32_t* n_blocks,
                                   int32_t* page_first, int32_t* page_block, int16_t* page_valid,
                                   int32_t* n_pages, void* ws, size_t ws_bytes, void* stream) {
  DSK_NVTX;
  if (ws && ws_bytes < kWsHdr) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  DSK_TRY(map_pages_impl(s, c, block_starts, n_blocks, page_first, page_block, page_valid, n_pages,
                         ws ? err_word(ws) : nullptr, stream));
  return cuda_status(launch_fence(static_cast<cudaStream_t>(stream)));
}

dynsplit_status dynsplit_repack_digest(const dynsplit_shape* s, const dynsplit_config* c,
                                       const void* K, const void* V, const int32_t* block_starts,
                                       const int32_t* n_blocks, const int32_t* page_first,
                                       void* Kp, void* Vp, void* digests, void* ws, size_t ws_bytes,
                                       void* stream) {
  DSK_NVTX;
  if (ws && ws_bytes < kWsHdr) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  DSK_TRY(repack_impl(s, c, K, V, block_starts, n_blocks, page_first, Kp, Vp, digests,
                      ws ? err_word(ws) : nullptr, stream));
  return cuda_status(launch_fence(static_cast<cudaStream_t>(stream)));
}

dynsplit_status dynsplit_build_blocks(const dynsplit_shape* s, const dynsplit_config* c,
                                      const int32_t* tokens, const int32_t* delim_ids,
                                      int32_t n_ids, const uint8_t* static_w10_host,
                                      const void* Qs, const void* Ks, const void* K, const void* V,
                                      uint8_t* w10, float* delim_scores, int32_t* block_starts,
                                      int32_t* n_blocks, int32_t* page_first, int32_t* page_block,
                                      int16_t* page_valid, int32_t* n_pages, void* Kp, void* Vp,
                                      void* digests, void* ws, size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!tokens || !delim_ids || !w10 || !ws) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (n_ids < 1 || n_ids > 64) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < build_ws(s)) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = ws_body(ws);
  float* tmp_scores = reinterpret_cast<float*>(w + score_body(s));
  // the score / segment sub-workspaces are addressed through their own (header) view
  void* score_view = w - kWsHdr;   // body of the scoring call = w
  void* seg_view = w + score_body(s) + align_up((size_t)s->B * s->S * 4) - kWsHdr;
  if (static_w10_host) {
    W10Table t;
    memset(&t, 0, sizeof(t));
    memcpy(t.w, static_w10_host, (size_t)n_ids);
    k_fill_w10<<<s->B, 64, 0, st>>>(t, n_ids, w10);
    if (post_launch("k_fill_w10", st) != cudaSuccess) return DYNSPLIT_ERR_CUDA;
  } else {
    if (!Qs || !Ks) return DYNSPLIT_ERR_INVALID_ARGUMENT;
    float* sc = delim_scores ? delim_scores : tmp_scores;
    if (launch_score_delimiters(tokens, delim_ids, n_ids, Qs, Ks, s->n_score_layers, s->B, s->S, s->Hq,
                                s->Hkv, c->W, c->R, c->alpha_pen, sc, ws_body(score_view), st) != cudaSuccess)
      return DYNSPLIT_ERR_CUDA;
    DSK_TRY(dynsplit_weight_table(s, tokens, delim_ids, n_ids, sc, w10, stream));
  }
  if (launch_segment(tokens, delim_ids, n_ids, w10, s->B, s->S, c->C, c->delta, c->lambda_num, c->lambda_den,
                     dynsplit_max_blocks(s->S, c), reinterpret_cast<int32_t*>(ws_body(seg_view)), block_starts,
                     n_blocks, st) != cudaSuccess)
    return DYNSPLIT_ERR_CUDA;
  DSK_TRY(map_pages_impl(s, c, block_starts, n_blocks, page_first, page_block, page_valid, n_pages,
                         err_word(ws), stream));
  if (K || V || Kp || Vp || digests)
    DSK_TRY(repack_impl(s, c, K, V, block_starts, n_blocks, page_first, Kp, Vp, digests, err_word(ws),
                        stream));
  return cuda_status(launch_fence(st));
}

// ------------------------------------------------------------------ decode
dynsplit_status dynsplit_score_blocks(const dynsplit_shape* s, const dynsplit_config* c,
                                      const void* q, const void* digests, const int32_t* n_blocks,
                                      float* scores, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!q || !digests || !n_blocks || !scores) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  // expected blocks per sequence: DD-Select averages C tokens per block; 25 % slack
  const int nb_hint = (int)(((int64_t)s->S * 5 + 4 * c->C - 1) / (4 * c->C));
  return cuda_status(launch_score_blocks(s->kv_dtype, s->Hq / s->Hkv, q, digests, n_blocks, scores,
                                         s->B, s->Hq, s->Hkv, dynsplit_max_blocks(s->S, c), nb_hint,
                                         c->digest_mode, static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
// a6 (shared by dynsplit_select_from_scores and dynsplit_decode_layer).
// err: the device error word of the caller's workspace.
static dynsplit_status select_impl(const dynsplit_shape* s, const dynsplit_config* c, int32_t budget,
                                   const float* scores, const int32_t* block_starts,
                                   const int32_t* n_blocks, const int32_t* page_first, int32_t blk_lo,
                                   int32_t blk_hi, int32_t* sel_blocks, int32_t* n_sel,
                                   int32_t* marginal_block, int32_t* marginal_keep, void* worklist,
                                   int* err, void* stream) {
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (budget < 1) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (!scores || !block_starts || !n_blocks || !page_first || !n_sel || !marginal_block ||
      !marginal_keep || !worklist)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (blk_lo < 0 || blk_hi < blk_lo) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (c->gqa_mode || c->budget_mode) return DYNSPLIT_ERR_UNSUPPORTED;  // NEXT-2 variants: fused layer only
  const int maxb = dynsplit_max_blocks(s->S, c);
  // smem-resident keys (S up to ~300K), 8-bit page counts per block, 16-bit block lengths
  if (select_smem_needed(maxb, s->Hq / s->Hkv) == (size_t)-1) return DYNSPLIT_ERR_UNSUPPORTED;
  if ((c->C + c->delta + c->page_size - 1) / c->page_size > 255) return DYNSPLIT_ERR_UNSUPPORTED;
  WorklistView v = worklist_view(worklist, s);
  return cuda_status(launch_select(s->Hq / s->Hkv, scores, block_starts, n_blocks, page_first, s->B,
                                   s->Hq, s->Hkv, maxb, s->S, dynsplit_max_selected(budget, s->S, c),
                                   max_wl_of(s, c, budget), c->page_size, budget, blk_lo, blk_hi,
                                   sel_blocks, n_sel, marginal_block, marginal_keep, v.count,
                                   v.entries, err, static_cast<cudaStream_t>(stream)));
}
extern "C" {

dynsplit_status dynsplit_select_from_scores(const dynsplit_shape* s, const dynsplit_config* c,
                                            int32_t budget, const float* scores,
                                            const int32_t* block_starts, const int32_t* n_blocks,
                                            const int32_t* page_first, int32_t blk_lo,
                                            int32_t blk_hi, int32_t* sel_blocks, int32_t* n_sel,
                                            int32_t* marginal_block, int32_t* marginal_keep,
                                            void* worklist, void* ws, size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!ws) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < select_ws(s, c)) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  return select_impl(s, c, budget, scores, block_starts, n_blocks, page_first, blk_lo, blk_hi,
                     sel_blocks, n_sel, marginal_block, marginal_keep, worklist, err_word(ws), stream);
}


dynsplit_status dynsplit_select(const dynsplit_shape* s, const dynsplit_config* c, int32_t budget,
                                const void* q, const void* digests, const int32_t* block_starts,
                                const int32_t* n_blocks, const int32_t* page_first,
                                float* scores_out, int32_t* sel_blocks, int32_t* n_sel,
                                int32_t* marginal_block, int32_t* marginal_keep, void* worklist,
                                void* ws, size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!ws) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < select_ws(s, c)) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  float* sc = scores_out ? scores_out : reinterpret_cast<float*>(ws_body(ws));
  DSK_TRY(dynsplit_score_blocks(s, c, q, digests, n_blocks, sc, stream));
  return select_impl(s, c, budget, sc, block_starts, n_blocks, page_first, 0, 0x7fffffff, sel_blocks,
                     n_sel, marginal_block, marginal_keep, worklist, err_word(ws), stream);
}

}  // extern "C"

static dynsplit_status decode_attn_impl(const dynsplit_shape* s, const dynsplit_config* c, const void* q,
                                        const void* Kp, const void* Vp, const int16_t* page_valid,
                                        const int32_t* n_pages, const void* worklist, float scale, float* o,
                                        float* lse, char* body, void* stream) {
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!q || !Kp || !Vp || !o || !lse) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  const int dense = worklist == nullptr;
  if (dense && (!n_pages || !page_valid)) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (!(scale > 0.f)) scale = 1.0f / sqrtf((float)kD);
  if ((size_t)s->B * s->Hkv > kMaxCounters / 2) return DYNSPLIT_ERR_UNSUPPORTED;
  int* counters = reinterpret_cast<int*>(body);
  float* part_o = reinterpret_cast<float*>(body + kMaxCounters * 4);
  float* part_lse = reinterpret_cast<float*>(body + kMaxCounters * 4 +
                                             align_up((size_t)s->B * s->Hq * kMaxSplit * kD * 4));
  const int32_t* hdr = nullptr;
  const int32_t* cnt = nullptr;
  const WLEntry* ent = nullptr;
  if (!dense) {
    WorklistView v = worklist_view(const_cast<void*>(worklist), s);
    hdr = v.hdr;
    cnt = v.count;
    ent = v.entries;
  }
  return cuda_status(launch_decode_attn(s->kv_dtype, s->Hq / s->Hkv, q, Kp, Vp, page_valid, n_pages,
                                        hdr, cnt, ent, dense, s->B, s->Hq, s->Hkv,
                                        dynsplit_max_pages(s->S, c), c->page_size, scale, part_o,
                                        part_lse, counters, o, lse,
                                        static_cast<cudaStream_t>(stream)));
}

extern "C" {

dynsplit_status dynsplit_decode_attn(const dynsplit_shape* s, const dynsplit_config* c,
                                     const void* q, const void* Kp, const void* Vp,
                                     const int16_t* page_valid, const int32_t* n_pages,
                                     const void* worklist, float scale, float* o, float* lse,
                                     void* ws, size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  if (!ws) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < decode_ws(s)) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  return decode_attn_impl(s, c, q, Kp, Vp, page_valid, n_pages, worklist, scale, o, lse, ws_body(ws), stream);
}

}  // extern "C"

static dynsplit_status decode_layer_impl(const dynsplit_shape* s, const dynsplit_config* c, int32_t budget,
                                         const void* q, const void* digests, const int32_t* block_starts,
                                         const int32_t* n_blocks, const int32_t* page_first, const void* Kp,
                                         const void* Vp, float scale, int32_t* n_sel, int32_t* marginal_block,
                                         int32_t* marginal_keep, void* worklist, float* o, float* lse,
                                         void* ws, void* stream) {
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!q || !digests || !Kp || !Vp || !o || !lse || !ws) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (budget < 1) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (!block_starts || !n_blocks || !page_first || !n_sel || !marginal_block || !marginal_keep || !worklist)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  char* body = ws_body(ws);
  char* dec_body = body;  // counters first: shape-independent offset
  float* sc = reinterpret_cast<float*>(body + decode_body(s));
  if (!(scale > 0.f)) scale = 1.0f / sqrtf((float)kD);
  // the fused single-kernel layer (a5 + a6 + a7 + a8) where the shape allows it
  {
    const int maxb = dynsplit_max_blocks(s->S, c);
    WorklistView v = worklist_view(worklist, s);
    int* counters = reinterpret_cast<int*>(dec_body);
    float* part_o = reinterpret_cast<float*>(dec_body + kMaxCounters * 4);
    float* part_lse = reinterpret_cast<float*>(dec_body + kMaxCounters * 4 +
                                               align_up((size_t)s->B * s->Hq * kMaxSplit * kD * 4));
    char* fscratch = body + decode_body(s) + select_body(s, c);
    const int nb_hint = (int)(((int64_t)s->S * 5 + 4 * c->C - 1) / (4 * c->C));
    const cudaError_t e = launch_decode_fused(
        s->kv_dtype, c->digest_mode, s->Hq / s->Hkv, q, digests, block_starts, n_blocks, page_first, Kp, Vp,
        s->B, s->Hq, s->Hkv, maxb, dynsplit_max_pages(s->S, c), s->S, c->page_size, budget, c->gqa_mode,
        c->budget_mode, nb_hint, scale, sc,
        score_stride(s, c), fscratch, counters, counters + kMaxCounters / 2, part_o, part_lse, n_sel,
        marginal_block, marginal_keep, v.count, v.entries, o, lse, err_word(ws),
        static_cast<cudaStream_t>(stream));
    if (e != cudaErrorNotSupported) return cuda_status(e);
    if (c->gqa_mode || c->budget_mode) return DYNSPLIT_ERR_UNSUPPORTED;  // NEXT-2 variants: fused layer only
  }
  DSK_TRY(dynsplit_score_blocks(s, c, q, digests, n_blocks, sc, stream));
  DSK_TRY(select_impl(s, c, budget, sc, block_starts, n_blocks, page_first, 0, 0x7fffffff, nullptr, n_sel,
                      marginal_block, marginal_keep, worklist, err_word(ws), stream));
  return decode_attn_impl(s, c, q, Kp, Vp, nullptr, nullptr, worklist, scale, o, lse, dec_body, stream);
}

extern "C" {

dynsplit_status dynsplit_decode_layer(const dynsplit_shape* s, const dynsplit_config* c,
                                      int32_t budget, const void* q, const void* digests,
                                      const int32_t* block_starts, const int32_t* n_blocks,
                                      const int32_t* page_first, const void* Kp, const void* Vp,
                                      float scale, int32_t* n_sel, int32_t* marginal_block,
                                      int32_t* marginal_keep, void* worklist, float* o, float* lse,
                                      void* ws, size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!ws) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < layer_ws(s, c)) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  return decode_layer_impl(s, c, budget, q, digests, block_starts, n_blocks, page_first, Kp, Vp, scale, n_sel,
                           marginal_block, marginal_keep, worklist, o, lse, ws, stream);
}

// ------------------------------------------------------------------ NEXT-1: append
dynsplit_status dynsplit_append_plan(const dynsplit_shape* s, const dynsplit_config* c, int32_t L_prev,
                                     int32_t L, const int32_t* tokens, const int32_t* delim_ids,
                                     int32_t n_ids, const uint8_t* w10, int32_t* block_starts,
                                     int32_t* n_blocks, int32_t* page_first, int32_t* page_block,
                                     int16_t* page_valid, int32_t* n_pages, void* ws, size_t ws_bytes,
                                     void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!tokens || !delim_ids || !w10 || !block_starts || !n_blocks || !page_first || !page_block ||
      !page_valid || !n_pages || !ws)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (n_ids < 1 || n_ids > 64) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (L < 1) return DYNSPLIT_ERR_EMPTY_SEQUENCE;
  if (L_prev < 0 || L_prev > L || L > s->S) return DYNSPLIT_ERR_DIMENSION_MISMATCH;
  if (c->C + c->delta > append_max_tail(s->kv_dtype)) return DYNSPLIT_ERR_UNSUPPORTED;
  if (ws_bytes < kWsHdr + append_ws_bytes(s->B)) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DSK_TRY(cuda_status(launch_plan_append(
      tokens, delim_ids, n_ids, w10, s->B, s->S, dynsplit_max_blocks(s->S, c), dynsplit_max_pages(s->S, c),
      c->C, c->delta, c->lambda_num, c->lambda_den, c->page_size, L_prev, L, block_starts, n_blocks,
      page_first, page_block, page_valid, n_pages, reinterpret_cast<int32_t*>(ws_body(ws)), err_word(ws), st)));
  return cuda_status(launch_fence(st));
}

dynsplit_status dynsplit_append_kv_layers(const dynsplit_shape* s, const dynsplit_config* c,
                                          int32_t L_prev, int32_t L, int32_t n_layers,
                                          const void* const* K_new, const void* const* V_new,
                                          const int32_t* block_starts, const int32_t* n_blocks,
                                          const int32_t* page_first, const void* ws, void* const* Kp,
                                          void* const* Vp, void* const* digests, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!block_starts || !n_blocks || !page_first || !ws || !Kp || !Vp || !digests)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (n_layers < 1 || n_layers > kAppendMaxLayers) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (L < 1) return DYNSPLIT_ERR_EMPTY_SEQUENCE;
  if (L_prev < 0 || L_prev > L || L > s->S) return DYNSPLIT_ERR_DIMENSION_MISMATCH;
  for (int l = 0; l < n_layers; ++l) {
    if (!Kp[l] || !Vp[l] || !digests[l]) return DYNSPLIT_ERR_INVALID_ARGUMENT;
    if (L > L_prev && (!K_new || !V_new || !K_new[l] || !V_new[l])) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  }
  if (c->C + c->delta > append_max_tail(s->kv_dtype)) return DYNSPLIT_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DSK_TRY(cuda_status(launch_kv_append(
      s->kv_dtype, n_layers, K_new, V_new, L - L_prev, s->B, s->Hkv, dynsplit_max_blocks(s->S, c),
      dynsplit_max_pages(s->S, c), c->page_size, L_prev, c->C + c->delta, block_starts, n_blocks, page_first,
      reinterpret_cast<const int32_t*>(static_cast<const char*>(ws) + kWsHdr), Kp, Vp, digests, c->digest_mode,
      st, nullptr, err_word(const_cast<void*>(ws)))));
  return cuda_status(launch_fence(st));
}

dynsplit_status dynsplit_append_plan_dev(const dynsplit_shape* s, const dynsplit_config* c,
                                         const int32_t* L_prev_dev, int32_t n_new, const int32_t* tokens,
                                         const int32_t* delim_ids, int32_t n_ids, const uint8_t* w10,
                                         int32_t* block_starts, int32_t* n_blocks, int32_t* page_first,
                                         int32_t* page_block, int16_t* page_valid, int32_t* n_pages, void* ws,
                                         size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!L_prev_dev || !tokens || !delim_ids || !w10 || !block_starts || !n_blocks || !page_first ||
      !page_block || !page_valid || !n_pages || !ws)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (n_ids < 1 || n_ids > 64 || n_new < 1 || n_new > s->S) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (c->C + c->delta > append_max_tail(s->kv_dtype)) return DYNSPLIT_ERR_UNSUPPORTED;
  if (ws_bytes < kWsHdr + append_ws_bytes(s->B)) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // L_prev = 1, L = 1 + n_new are placeholders the kernel replaces by *L_prev_dev
  DSK_TRY(cuda_status(launch_plan_append(
      tokens, delim_ids, n_ids, w10, s->B, s->S, dynsplit_max_blocks(s->S, c), dynsplit_max_pages(s->S, c),
      c->C, c->delta, c->lambda_num, c->lambda_den, c->page_size, 1, 1 + n_new, block_starts, n_blocks,
      page_first, page_block, page_valid, n_pages, reinterpret_cast<int32_t*>(ws_body(ws)), err_word(ws), st,
      L_prev_dev)));
  return cuda_status(launch_fence(st));
}

dynsplit_status dynsplit_append_kv_layers_dev(const dynsplit_shape* s, const dynsplit_config* c,
                                              const int32_t* L_prev_dev, int32_t n_new, int32_t n_layers,
                                              const void* const* K_new, const void* const* V_new,
                                              const int32_t* block_starts, const int32_t* n_blocks,
                                              const int32_t* page_first, const void* ws, void* const* Kp,
                                              void* const* Vp, void* const* digests, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!L_prev_dev || !block_starts || !n_blocks || !page_first || !ws || !Kp || !Vp || !digests || !K_new ||
      !V_new)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (n_layers < 1 || n_layers > kAppendMaxLayers || n_new < 1 || n_new > s->S)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  for (int l = 0; l < n_layers; ++l)
    if (!Kp[l] || !Vp[l] || !digests[l] || !K_new[l] || !V_new[l]) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (c->C + c->delta > append_max_tail(s->kv_dtype)) return DYNSPLIT_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DSK_TRY(cuda_status(launch_kv_append(
      s->kv_dtype, n_layers, K_new, V_new, n_new, s->B, s->Hkv, dynsplit_max_blocks(s->S, c),
      dynsplit_max_pages(s->S, c), c->page_size, 1, c->C + c->delta, block_starts, n_blocks, page_first,
      reinterpret_cast<const int32_t*>(static_cast<const char*>(ws) + kWsHdr), Kp, Vp, digests, c->digest_mode,
      st, L_prev_dev, err_word(const_cast<void*>(ws)))));
  return cuda_status(launch_fence(st));
}

dynsplit_status dynsplit_append_kv(const dynsplit_shape* s, const dynsplit_config* c, int32_t L_prev,
                                   int32_t L, const void* K_new, const void* V_new,
                                   const int32_t* block_starts, const int32_t* n_blocks,
                                   const int32_t* page_first, const void* ws, void* Kp, void* Vp,
                                   void* digests, void* stream) {
  const void* kn[1] = {K_new};
  const void* vn[1] = {V_new};
  void* kp[1] = {Kp};
  void* vp[1] = {Vp};
  void* dg[1] = {digests};
  return dynsplit_append_kv_layers(s, c, L_prev, L, 1, kn, vn, block_starts, n_blocks, page_first, ws, kp,
                                   vp, dg, stream);
}

dynsplit_status dynsplit_merge_partials(const float* o_parts, const float* lse_parts,
                                        int32_t n_parts, int32_t rows, int32_t d, float* o,
                                        float* lse, void* stream) {
  DSK_NVTX;
  if (!o_parts || !lse_parts || !o || !lse || n_parts < 1 || rows < 1 || d < 1)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  return cuda_status(launch_merge(o_parts, lse_parts, n_parts, rows, d, o, lse,
                                  static_cast<cudaStream_t>(stream)));
}

dynsplit_status dynsplit_decode_step_host(const dynsplit_shape* s, const dynsplit_config* c,
                                          int32_t budget, const void* q_host, const void* digests,
                                          const int32_t* block_starts, const int32_t* n_blocks,
                                          const int32_t* page_first, const void* Kp, const void* Vp,
                                          const int16_t* page_valid, float scale, float* o_host,
                                          float* lse_host, void* worklist, void* ws,
                                          size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (!q_host || !o_host || !lse_host || !ws || !worklist) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < dynsplit_step_host_workspace_bytes(s, c, budget))
    return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* extra = static_cast<char*>(ws) + layer_ws(s, c);
  const size_t qbytes = (size_t)s->B * s->Hq * kD * esize(s);
  void* q_dev = extra;
  float* o_dev = reinterpret_cast<float*>(extra + align_up(qbytes));
  float* lse_dev = reinterpret_cast<float*>(extra + align_up(qbytes) + align_up((size_t)s->B * s->Hq * kD * 4));
  int32_t* nsel = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(lse_dev) + align_up((size_t)s->B * s->Hq * 4));
  int32_t* marg = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(nsel) + align_up((size_t)s->B * s->Hq * 4));
  int32_t* keep = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(marg) + align_up((size_t)s->B * s->Hq * 4));
  if (cudaMemcpyAsync(q_dev, q_host, qbytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return DYNSPLIT_ERR_CUDA;
  (void)page_valid;
  DSK_TRY(decode_layer_impl(s, c, budget, q_dev, digests, block_starts, n_blocks, page_first, Kp, Vp, scale, nsel,
                            marg, keep, worklist, o_dev, lse_dev, ws, stream));
  if (cudaMemcpyAsync(o_host, o_dev, (size_t)s->B * s->Hq * kD * 4, cudaMemcpyDeviceToHost, st) !=
          cudaSuccess ||
      cudaMemcpyAsync(lse_host, lse_dev, (size_t)s->B * s->Hq * 4, cudaMemcpyDeviceToHost, st) !=
          cudaSuccess)
    return DYNSPLIT_ERR_CUDA;
  return DYNSPLIT_OK;
}

// ---- the whole-step host-buffer form
static size_t host_layers_extra(const dynsplit_shape* s, int32_t n_layers) {
  const size_t L = (size_t)(n_layers > 0 ? n_layers : 0);
  return align_up(L * s->B * s->Hq * kD * esize(s)) + align_up(L * s->B * s->Hq * kD * 4) +
         align_up(L * s->B * s->Hq * 4) + 3 * align_up((size_t)s->B * s->Hq * 4);
}

size_t dynsplit_step_host_layers_workspace_bytes(const dynsplit_shape* s, const dynsplit_config* c,
                                                 int32_t budget, int32_t n_layers) {
  (void)budget;
  if (check_shape(s) != DYNSPLIT_OK || check_cfg(c) != DYNSPLIT_OK || n_layers < 1) return 0;
  return layer_ws(s, c) + host_layers_extra(s, n_layers);
}

dynsplit_status dynsplit_decode_step_host_layers(const dynsplit_shape* s, const dynsplit_config* c,
                                                 int32_t budget, int32_t n_layers, const void* q_host,
                                                 const void* const* digests, const int32_t* block_starts,
                                                 const int32_t* n_blocks, const int32_t* page_first,
                                                 const void* const* Kp, const void* const* Vp, float scale,
                                                 float* o_host, float* lse_host, void* worklist, void* ws,
                                                 size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  if (n_layers < 1 || !q_host || !digests || !Kp || !Vp || !o_host || !lse_host || !ws || !worklist)
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < dynsplit_step_host_layers_workspace_bytes(s, c, budget, n_layers))
    return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t L = (size_t)n_layers, rows = (size_t)s->B * s->Hq;
  const size_t qbytes = rows * kD * esize(s);
  char* extra = static_cast<char*>(ws) + layer_ws(s, c);
  char* q_dev = extra;
  float* o_dev = reinterpret_cast<float*>(extra + align_up(L * qbytes));
  float* lse_dev = reinterpret_cast<float*>(reinterpret_cast<char*>(o_dev) + align_up(L * rows * kD * 4));
  int32_t* nsel = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(lse_dev) + align_up(L * rows * 4));
  int32_t* marg = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(nsel) + align_up(rows * 4));
  int32_t* keep = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(marg) + align_up(rows * 4));
  if (cudaMemcpyAsync(q_dev, q_host, L * qbytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return DYNSPLIT_ERR_CUDA;
  // the copy is not a PDL primary: the first layer's pre-wait prologue reads
  // only resident inputs, and q after its wait
  for (size_t l = 0; l < L; ++l) {
    if (!digests[l] || !Kp[l] || !Vp[l]) return DYNSPLIT_ERR_INVALID_ARGUMENT;
    DSK_TRY(decode_layer_impl(s, c, budget, q_dev + l * qbytes, digests[l], block_starts, n_blocks, page_first,
                              Kp[l], Vp[l], scale, nsel, marg, keep, worklist, o_dev + l * rows * kD,
                              lse_dev + l * rows, ws, stream));
  }
  if (cudaMemcpyAsync(o_host, o_dev, L * rows * kD * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(lse_host, lse_dev, L * rows * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return DYNSPLIT_ERR_CUDA;
  return DYNSPLIT_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ NEXT-3: offloaded KV + reuse
namespace {
dynsplit_status check_cache(const dynsplit_shape* s, const dynsplit_config* c, const dynsplit_kv_cache* k,
                            bool need_plan) {
  if (!k || !k->Kc || !k->Vc) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (k->n_slots < 1 || k->n_slots > dynsplit_max_pages(s->S, c)) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (need_plan && (!k->slot_page || !k->fetch || !k->fetch_count || !k->worklist_cache))
    return DYNSPLIT_ERR_INVALID_ARGUMENT;
  return DYNSPLIT_OK;
}
// the device address of pinned host memory (zero-copy); nullptr if the
// pointer is not host memory the device can map
const void* mapped_host(const void* h) {
  cudaPointerAttributes a;
  if (!h || cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
  return a.devicePointer;
}
}  // namespace

static dynsplit_status reuse_impl(const dynsplit_shape* s, const dynsplit_config* c, const void* worklist,
                                  int32_t truncate, int32_t reuse, const dynsplit_kv_cache* k, char* rbody,
                                  int* err, void* stream) {
  const size_t bh = (size_t)s->B * s->Hkv, mp = (size_t)dynsplit_max_pages(s->S, c);
  int32_t* reusable = reinterpret_cast<int32_t*>(rbody);
  int32_t* map = reinterpret_cast<int32_t*>(rbody + align_up(bh * 4));
  int32_t* freelist = reinterpret_cast<int32_t*>(rbody + align_up(bh * 4) + align_up(bh * mp * 4));
  WorklistView v = worklist_view(const_cast<void*>(worklist), s);
  WorklistView w = worklist_view(k->worklist_cache, s);
  return cuda_status(launch_reuse_plan(v.hdr, v.count, v.entries, s->B, s->Hkv, (int)mp, k->n_slots, reuse != 0,
                                       truncate != 0, reusable, map, freelist, k->slot_page, k->fetch,
                                       k->fetch_count, k->reuse_stats, k->reuse_len, w.hdr, w.count, w.entries,
                                       err, static_cast<cudaStream_t>(stream)));
}

static dynsplit_status fetch_impl(const dynsplit_shape* s, const dynsplit_config* c, const void* Kp_host,
                                  const void* Vp_host, const int16_t* page_valid, const int32_t* n_pages,
                                  int32_t dense, const dynsplit_kv_cache* k, void* stream) {
  if (!page_valid || (dense && !n_pages)) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (!dense && (!k->fetch || !k->fetch_count)) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  const int mp = dynsplit_max_pages(s->S, c);
  if (dense && k->n_slots != mp) return DYNSPLIT_ERR_DIMENSION_MISMATCH;
  const void* kd = mapped_host(Kp_host);
  const void* vd = mapped_host(Vp_host);
  if (!kd || !vd) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  return cuda_status(launch_fetch_pages(s->kv_dtype, kd, vd, page_valid, n_pages, k->fetch, k->fetch_count,
                                        dense != 0, s->B, s->Hkv, mp, k->n_slots, c->page_size, k->Kc, k->Vc,
                                        static_cast<cudaStream_t>(stream)));
}

extern "C" {

int32_t dynsplit_cache_slots(const dynsplit_shape* s, const dynsplit_config* c, int32_t budget) {
  if (check_shape(s) != DYNSPLIT_OK || check_cfg(c) != DYNSPLIT_OK || budget < 1) return 0;
  const long long per_head =
      (budget + c->page_size - 1) / c->page_size + (long long)dynsplit_max_selected(budget, s->S, c);
  const long long v = per_head * (s->Hq / s->Hkv);
  const long long mp = dynsplit_max_pages(s->S, c);
  return (int32_t)(v < mp ? v : mp);
}

dynsplit_status dynsplit_reuse_plan(const dynsplit_shape* s, const dynsplit_config* c, const void* worklist,
                                    int32_t truncate, int32_t reuse, const dynsplit_kv_cache* cache, void* ws,
                                    size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  DSK_TRY(check_cache(s, c, cache, true));
  if (!worklist || !ws) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < kWsHdr + reuse_body(s, c)) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  return reuse_impl(s, c, worklist, truncate, reuse, cache, ws_body(ws), err_word(ws), stream);
}

dynsplit_status dynsplit_fetch_pages(const dynsplit_shape* s, const dynsplit_config* c, const void* Kp_host,
                                     const void* Vp_host, const int16_t* page_valid, const int32_t* n_pages,
                                     int32_t dense, const dynsplit_kv_cache* cache, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  DSK_TRY(check_cache(s, c, cache, false));
  return fetch_impl(s, c, Kp_host, Vp_host, page_valid, n_pages, dense, cache, stream);
}

dynsplit_status dynsplit_decode_layer_offload(const dynsplit_shape* s, const dynsplit_config* c, int32_t budget,
                                              const void* q, const void* digests, const int32_t* block_starts,
                                              const int32_t* n_blocks, const int32_t* page_first,
                                              const int16_t* page_valid, const void* Kp_host,
                                              const void* Vp_host, int32_t truncate, int32_t reuse,
                                              const dynsplit_kv_cache* cache, float scale, int32_t* n_sel,
                                              int32_t* marginal_block, int32_t* marginal_keep, void* worklist,
                                              float* o, float* lse, void* ws, size_t ws_bytes, void* stream) {
  DSK_NVTX;
  DSK_TRY(check_shape(s));
  DSK_TRY(check_cfg(c));
  DSK_TRY(check_cache(s, c, cache, true));
  if (!q || !digests || !o || !lse || !ws || !worklist) return DYNSPLIT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < offload_ws(s, c)) return DYNSPLIT_ERR_WORKSPACE_TOO_SMALL;
  char* body = ws_body(ws);
  char* dec_body = body;  // counters first (shape-independent offset)
  float* sc = reinterpret_cast<float*>(body + decode_body(s));
  char* rbody = body + decode_body(s) + select_body(s, c);
  // a5 + a6 on the resident digests and plan (Step 1 of the decode step)
  DSK_TRY(dynsplit_score_blocks(s, c, q, digests, n_blocks, sc, stream));
  DSK_TRY(select_impl(s, c, budget, sc, block_starts, n_blocks, page_first, 0, 0x7fffffff, nullptr, n_sel,
                      marginal_block, marginal_keep, worklist, err_word(ws), stream));
  // reuse plan (Appendix B.2 Steps 1 and 3) and the move (Step 2)
  DSK_TRY(reuse_impl(s, c, worklist, truncate, reuse, cache, rbody, err_word(ws), stream));
  DSK_TRY(fetch_impl(s, c, Kp_host, Vp_host, page_valid, nullptr, 0, cache, stream));
  // a7 + a8 over the cache: the slot count is the page stride
  dynsplit_config cc = *c;
  cc.page_cap = cache->n_slots;
  return decode_attn_impl(s, &cc, q, cache->Kc, cache->Vc, nullptr, nullptr, cache->worklist_cache, scale, o, lse,
                          dec_body, stream);
}

}  // extern "C"
