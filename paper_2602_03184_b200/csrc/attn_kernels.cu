// Decode rows a7 + a8 (a9 in dense mode): split-K flash-decoding over the
// selected pages of the GQA-union worklist, with the log-sum-exp merge of the
// splits (Step 3 of KV selection; "split-K ... log-sum-exp merge",
// north star).
//
// grid (n_split, Hkv, B) sized to one resident wave; NW warps per CTA, no
// producer warp and no inter-warp barriers in the main loop:
//  * warp w takes the split's pages i = w (mod NW) and runs its own load
//    pipeline: the page's valid K and V rows go into 16-byte padded smem rows
//    of a private `depth`-stage ring with 16-byte cp.async (LDGSTS, 512
//    contiguous bytes per warp instruction), page j + depth is issued while
//    page j is computed, completion by cp.async.wait_group.  Padding rows of
//    a page are never read from HBM.  (Measured alternatives: a producer warp
//    + mbarrier ring spent half of all issued instructions in the consumers'
//    try_wait loops and could not keep the consumers fed; 1-D TMA bulk copies
//    cannot pad rows and one bulk copy per row is slower than LDGSTS.)
//  * A warp handles ALL G query heads of the KV group on them, so each K/V
//    byte is read from HBM once: bf16 caches: QK and PV as mma.sync m16n8k16
//    tiles (attn_core.cuh, shared with the fused decode layer);
//    fp32 caches: CUDA-core path --
//      QK:  lane (hg = lane/16, r = lane%16) computes the full 128-dim dot of
//           row r with heads hg, hg+2, ...; the padded K rows put the 16 rows
//           in distinct bank groups, so all lanes read the same 16-byte chunk
//           (conflict-free) and q is a broadcast read (FFMA, two chains).
//      softmax: per head over the 16 lanes of its group, exp2 domain; the
//           running max moves (and l, acc are rescaled) only when a logit
//           exceeds it by more than 2^8, detected with one warp vote.
//      PV:  lane owns dims [4 lane, 4 lane + 4) for all G heads, P from a
//           per-warp smem slab (float2 (p, p) pairs) and FFMA2.
//  * Warps are merged in fixed order; each CTA writes its split's (o, lse);
//    the last CTA of a (b, KV head) merges the splits in split order.
#include "attn_core.cuh"
#include "common.cuh"
#include "kernels.h"

#include <cudaTypedefs.h>
#include <math_constants.h>
#include <stdlib.h>
#include <string.h>

namespace dsk {

// Optional per-CTA phase timestamps (debug only; dynsplit_debug_attn_timer).
__device__ unsigned long long* g_attn_dbg = nullptr;
__device__ int g_attn_noload = 0;     // debug: compute on stale smem without loading pages
DSK_DEVICE void astamp(int k) {
#ifdef DSK_DEBUG
  if (g_attn_dbg) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const size_t cta = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    g_attn_dbg[cta * 8 + k] = t;
  }
#else
  (void)k;
#endif
}

DSK_DEVICE uint64_t pack2(float x, float y) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
DSK_DEVICE void unpack2(uint64_t v, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
}
// (a0, a1) += (b0, b1) * (c, c)   -- one FFMA2
DSK_DEVICE void ffma2(float& a0, float& a1, float b0, float b1, uint64_t cc) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pack2(b0, b1)), "l"(cc), "l"(pack2(a0, a1)));
  unpack2(r, a0, a1);
}

template <typename T> struct QK;
template <> struct QK<float> {
  static constexpr int kChunks = kD * 4 / 16;  // 32 chunks of 4 fp32
  static DSK_DEVICE void dot2(uint4 qc, uint4 kc, float& a0, float& a1) {
    a0 = fmaf(__uint_as_float(qc.x), __uint_as_float(kc.x), a0);
    a1 = fmaf(__uint_as_float(qc.y), __uint_as_float(kc.y), a1);
    a0 = fmaf(__uint_as_float(qc.z), __uint_as_float(kc.z), a0);
    a1 = fmaf(__uint_as_float(qc.w), __uint_as_float(kc.w), a1);
  }
};

template <typename T, int G, int NW, int D>
__global__ void __launch_bounds__(NW * 32, NW >= 8 ? 1 : 3) k_decode_attn(
    const T* __restrict__ q, const T* __restrict__ Kp, const T* __restrict__ Vp,
    const int16_t* __restrict__ page_valid, const int32_t* __restrict__ n_pages,
    const int32_t* __restrict__ wl_hdr, const int32_t* __restrict__ wl_count,
    const WLEntry* __restrict__ wl, int dense, int Hq, int Hkv, int max_pages, int P,
    float scale_log2, float* __restrict__ part_o, float* __restrict__ part_lse,
    int* __restrict__ counters, int n_split, float* __restrict__ o, float* __restrict__ lse, int tma,
    const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV) {
  constexpr bool kTC = sizeof(T) == 2;  // bf16: QK and PV on the tensor cores (mma.sync)
  extern __shared__ __align__(128) unsigned char smem[];
  // K and V rows are staged with a 16-byte pad (row stride ROW + 16): the 8
  // or 16 rows a warp reads together then sit in distinct bank groups, which
  // makes ldmatrix (bf16) and the same-chunk row reads of the fp32 path
  // conflict-free.  A stage holds max(P, 16) rows; rows of a 16-row tile
  // beyond the page's valid rows are masked (K) or multiplied by p = 0 (V,
  // zero-initialised once so that it never holds a non-finite pattern).
  constexpr int ROW = kD * (int)sizeof(T);
  constexpr int KROW = ROW + 16;
  const int nd = attn_depth(D, NW, ROW, P);
  const size_t kstage = (size_t)attn_stage_rows(P) * KROW, stage = 2 * kstage;
  const size_t hbm_page = (size_t)P * ROW;
  uint32_t(*s_rows)[2] = reinterpret_cast<uint32_t(*)[2]>(smem + (size_t)NW * nd * stage);  // [NW][D]
  T* s_q = reinterpret_cast<T*>(s_rows + NW * D);                  // [G][kD]
  float2* pbuf = reinterpret_cast<float2*>(s_q + G * kD);          // [NW][16][G] (fp32 path)
  __shared__ int s_last;
  __shared__ __align__(8) uint64_t s_tbar[NW * D];  // TMA variant: one mbarrier per (warp, stage)
  unsigned char* ring_t = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);  // TMA variant: 1024-aligned

  const int split = blockIdx.x, hk = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = b * Hkv + hk;

  if (threadIdx.x == 0) astamp(0);
  // prologue independent of the preceding kernel (PDL overlap): V ring reset
  if (kTC) attn_zero_v_rings(smem, NW * nd, kstage, stage);
  if (kTC && tma && (threadIdx.x & 31) == 0) {
    for (int s2 = 0; s2 < D; ++s2) mbar_init(&s_tbar[warp * D + s2], 1);
    fence_mbar_init();
  }
  pdl_trigger();
  pdl_wait();  // q and the worklist belong to the step: read only after the wait
  if (threadIdx.x == 0) astamp(1);
  // q of the G heads: loads issued now, stored to smem after the worklist
  // loads below are in flight (their latencies overlap)
  constexpr int QCH = G * kD * (int)sizeof(T) / 16;
  constexpr int QPT = (QCH + NW * 32 - 1) / (NW * 32);
  uint4 qreg[QPT];
  {
    const uint4* src = reinterpret_cast<const uint4*>(q + ((size_t)b * Hq + hk * G) * kD);
#pragma unroll
    for (int k = 0; k < QPT; ++k) {
      const int c = threadIdx.x + k * NW * 32;
      if (c < QCH) qreg[k] = __ldcg(src + c);
    }
  }

  // Pages are dealt round-robin: split s of n_eff takes worklist entries
  // e = s + k n_eff, k = 0, 1, ...; warp w takes k = w + j NW.  Entry e of
  // (b, KV head) bh sits at wl[e * B * Hkv + bh] (interleaved layout; the
  // buffer holds >= max_pages entries per bh), so each warp's first 32
  // entries are loaded together with the page count, speculating
  // n_eff == n_split (true whenever cnt >= kMinPagesPerSplit * n_split).
  const size_t BH = (size_t)gridDim.z * Hkv;
  int e_page = 0;
  uint32_t e_r0 = 0, e_r1 = 0;
  auto load_batch = [&](int j0, int stride) {  // entries of this warp's pages j0 + lane
    const int e = split + (warp + (j0 + lane) * NW) * stride;
    e_page = 0;
    e_r0 = e_r1 = 0;
    if (e < max_pages) {
      if (dense) {
        e_page = e;
        const uint32_t pv = (uint32_t)page_valid[(size_t)b * max_pages + e];
        e_r0 = e_r1 = pv * 0x01010101u;
      } else {
        // weak coherent load (not the read-only .nc path): the worklist is the
        // output of the PDL primary, which may still be running at launch
        const int4 en = __ldca(reinterpret_cast<const int4*>(wl + (size_t)e * BH + bh));
        e_page = en.x;
        e_r0 = (uint32_t)en.z;
        e_r1 = (uint32_t)en.w;
      }
    }
  };
  load_batch(0, n_split);
  const int cnt = dense ? n_pages[b] : __ldca(wl_count + bh);
#pragma unroll
  for (int k = 0; k < QPT; ++k) {
    const int c = threadIdx.x + k * NW * 32;
    if (c < QCH) reinterpret_cast<uint4*>(s_q)[c] = qreg[k];
  }
  // splits actually used by this (b, KV head): at least kMinPagesPerSplit pages each
  const int n_eff = max(1, min(n_split, (cnt + kMinPagesPerSplit - 1) / kMinPagesPerSplit));
  if (split >= n_eff) return;
  if (n_eff != n_split) load_batch(0, n_eff);
  const int n_it = (cnt - split + n_eff - 1) / n_eff;  // this split's pages
  __syncthreads();  // s_q and the zeroed V rings are visible to every warp
  const int n_mine = n_it > warp ? (n_it - warp + NW - 1) / NW : 0;
#ifdef DSK_DEBUG
  const bool noload = g_attn_noload != 0;
#else
  const bool noload = false;
#endif
  float* sc = reinterpret_cast<float*>(kTC && tma ? ring_t : smem);  // merge scratch [NW][G][kScStride] (ring)
  if constexpr (kTC) {
    auto entry = [&](int j, int& pg, uint32_t& a, uint32_t& c) {
      if ((j & 31) == 0 && j) load_batch(j, n_eff);
      pg = __shfl_sync(0xffffffffu, e_page, j & 31);
      a = __shfl_sync(0xffffffffu, e_r0, j & 31);
      c = __shfl_sync(0xffffffffu, e_r1, j & 31);
    };
    if (threadIdx.x == 0) astamp(2);
    if (tma)
      attn_bf16_pipeline_tma<G, NW, D>(ring_t, s_tbar, s_rows, s_q, D, n_mine, entry, &tmK, &tmV, (size_t)bh,
                                       max_pages, scale_log2);
    else
      attn_bf16_pipeline<G, NW, D>(smem, s_rows, s_q, nd, P, n_mine, entry, Kp, Vp, (size_t)bh, max_pages,
                                   scale_log2, noload);
    if (threadIdx.x == 0) astamp(3);
  } else {
  // ---- fp32: per-warp load pipeline (as in attn_bf16_pipeline) + CUDA-core consumer
  unsigned char* wring = smem + (size_t)warp * nd * stage;
  auto issue = [&](int j) {
    if (j < n_mine) {
      if ((j & 31) == 0 && j) load_batch(j, n_eff);
      const int pg = __shfl_sync(0xffffffffu, e_page, j & 31);
      const uint32_t a = __shfl_sync(0xffffffffu, e_r0, j & 31);
      const uint32_t c = __shfl_sync(0xffffffffu, e_r1, j & 31);
      int rmax = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) rmax = max(rmax, entry_rows(a, c, g));
      if ((unsigned)pg >= (unsigned)max_pages || noload) rmax = 0;
      const int st = j % nd;
      if (lane == 0) {
        s_rows[warp * D + st][0] = a;
        s_rows[warp * D + st][1] = c;
      }
      constexpr int CPR = ROW / 16;
      constexpr int RPI = 32 / CPR;
      const size_t off = ((size_t)bh * max_pages + pg) * hbm_page;
      const int cc = lane % CPR, r0 = lane / CPR;
      const unsigned char* kg = reinterpret_cast<const unsigned char*>(Kp) + off + r0 * ROW + cc * 16;
      const unsigned char* vg = reinterpret_cast<const unsigned char*>(Vp) + off + r0 * ROW + cc * 16;
      unsigned char* ks = wring + st * stage + r0 * KROW + cc * 16;
      for (int rr = r0; rr < rmax; rr += RPI) {
        cp_async16_cg(ks, kg);
        cp_async16_cg(ks + kstage, vg);
        ks += RPI * KROW;
        kg += RPI * ROW;
        vg += RPI * ROW;
      }
    }
    cp_async_commit_group();
  };
  for (int j = 0; j < nd; ++j) issue(j);
  constexpr int CH = QK<T>::kChunks;
  constexpr int HPL = (G + 1) / 2;  // heads per QK lane
  const int r = lane & 15, hg = lane >> 4;
  float m[HPL], l[HPL];
#pragma unroll
  for (int j = 0; j < HPL; ++j) {
    m[j] = -CUDART_INF_F;
    l[j] = 0.f;
  }
  float acc[G][4];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[h][k] = 0.f;
  float2* pb = pbuf + warp * 16 * G;
  const unsigned char* qbase = reinterpret_cast<const unsigned char*>(s_q);

  for (int jp = 0; jp < n_mine; ++jp) {
    const int st = jp % nd;
    cp_async_wait_pending(nd - 1);
    __syncwarp();
    const uint32_t ra = s_rows[warp * D + st][0], rc = s_rows[warp * D + st][1];
    int rmax = 0, myrows[HPL];
#pragma unroll
    for (int g = 0; g < G; ++g) rmax = max(rmax, (int)(((g < 4 ? ra : rc) >> (8 * (g & 3))) & 0xffu));
#pragma unroll
    for (int j = 0; j < HPL; ++j) {
      const int h = hg + 2 * j;
      myrows[j] = h < G ? (int)(((h < 4 ? ra : rc) >> (8 * (h & 3))) & 0xffu) : 0;
    }
    const unsigned char* Ks = wring + st * stage;
    const unsigned char* Vs = Ks + kstage;
    for (int r0 = 0; r0 < rmax; r0 += 16) {
      const int nr = min(16, rmax - r0);
      const bool rowok = r < nr;
      // QK: two independent accumulation chains per head (even/odd elements)
      float dot0[HPL], dot1[HPL];
#pragma unroll
      for (int j = 0; j < HPL; ++j) dot0[j] = dot1[j] = 0.f;
      if (rowok) {
        const unsigned char* krow = Ks + (size_t)(r0 + r) * KROW;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int off = c * 16;
          const uint4 kc = *reinterpret_cast<const uint4*>(krow + off);
#pragma unroll
          for (int j = 0; j < HPL; ++j) {
            const int h = hg + 2 * j;
            if (h < G) {
              const uint4 qc = *reinterpret_cast<const uint4*>(qbase + (size_t)h * kD * sizeof(T) + off);
              QK<T>::dot2(qc, kc, dot0[j], dot1[j]);
            }
          }
        }
      }
      // online softmax with conditional rescaling: the running max m only
      // moves (full 16-lane max + rescale of l and acc) when some logit
      // exceeds it by more than 2^8 (log2 domain); otherwise p = exp2(z - m)
      // directly and every lane keeps its own partial sum l (reduced at the end).
      float z[HPL];
      bool any_valid = false;
#pragma unroll
      for (int j = 0; j < HPL; ++j) {
        const bool valid = rowok && (r0 + r) < myrows[j];
        z[j] = valid ? (dot0[j] + dot1[j]) * scale_log2 : -CUDART_INF_F;
        any_valid |= z[j] > m[j] + 8.f;
      }
      if (__any_sync(0xffffffffu, any_valid)) {
        float corr[HPL];
#pragma unroll
        for (int j = 0; j < HPL; ++j) {
          float mx = z[j];
#pragma unroll
          for (int o2 = 1; o2 < 16; o2 <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
          const float mnew = fmaxf(m[j], mx);
          corr[j] = (mnew == -CUDART_INF_F || m[j] == mnew) ? 1.f : exp2f(m[j] - mnew);
          l[j] *= corr[j];
          m[j] = mnew;
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
          const float ch = __shfl_sync(0xffffffffu, corr[h >> 1], (h & 1) * 16);
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[h][k] *= ch;
        }
      }
#pragma unroll
      for (int j = 0; j < HPL; ++j) {
        const int h = hg + 2 * j;
        const float pj = z[j] == -CUDART_INF_F ? 0.f : exp2f(z[j] - m[j]);
        l[j] += pj;
        if (h < G) pb[r * G + h] = make_float2(pj, pj);
      }
      __syncwarp();
      // fully unrolled over the 16 rows of the slab (predicated) so the V and
      // P loads of several rows are in flight at once
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) {
        if (rr >= nr) break;
        float v[4];
        Vec<T>::load4(reinterpret_cast<const T*>(Vs + (size_t)(r0 + rr) * KROW) + lane * 4, v);
        const float2* prow = pb + rr * G;
#pragma unroll
        for (int h = 0; h < G; h += 2) {
          if (h + 1 < G) {
            const float4 pp = *reinterpret_cast<const float4*>(prow + h);
            const uint64_t c0 = pack2(pp.x, pp.y), c1 = pack2(pp.z, pp.w);
            ffma2(acc[h][0], acc[h][1], v[0], v[1], c0);
            ffma2(acc[h][2], acc[h][3], v[2], v[3], c0);
            ffma2(acc[h + 1][0], acc[h + 1][1], v[0], v[1], c1);
            ffma2(acc[h + 1][2], acc[h + 1][3], v[2], v[3], c1);
          } else {
            const float2 pp = prow[h];
            const uint64_t c0 = pack2(pp.x, pp.y);
            ffma2(acc[h][0], acc[h][1], v[0], v[1], c0);
            ffma2(acc[h][2], acc[h][3], v[2], v[3], c0);
          }
        }
      }
      __syncwarp();
    }
    issue(jp + nd);
  }

  // ---- per-warp state to the merge scratch (the ring is free once all are here)
  named_bar_sync(1, NW * 32);
  if (threadIdx.x == 0) astamp(3);
#pragma unroll
  for (int h = 0; h < G; ++h)
    *reinterpret_cast<float4*>(sc + (warp * G + h) * kScStride + lane * 4) =
        make_float4(acc[h][0], acc[h][1], acc[h][2], acc[h][3]);
#pragma unroll
  for (int j = 0; j < HPL; ++j) {
#pragma unroll
    for (int o2 = 1; o2 < 16; o2 <<= 1) l[j] += __shfl_xor_sync(0xffffffffu, l[j], o2);
  }
  if (r == 0) {
#pragma unroll
    for (int j = 0; j < HPL; ++j) {
      const int h = hg + 2 * j;
      if (h < G) {
        sc[(warp * G + h) * kScStride + kD] = m[j];
        sc[(warp * G + h) * kScStride + kD + 1] = l[j];
      }
    }
  }
  }  // fp32 path
  attn_merge_out<G, NW>(sc, &s_last, b, hk, Hq, split, n_eff, n_split, (size_t)bh, part_o, part_lse, counters,
                        o, lse);
  if (threadIdx.x == 0) astamp(5);
}

// ============================================================================
// host launcher
// ============================================================================
template <typename T, int G, int NW, int D>
static size_t attn_smem(int P) {
  const int row = kD * (int)sizeof(T);
  const size_t ring = (size_t)NW * attn_depth(D, NW, row, P) * attn_stage_bytes(row, P);
  const size_t merge = (size_t)NW * G * kScStride * sizeof(float);
  return (ring > merge ? ring : merge) + (size_t)NW * D * 8 + (size_t)G * kD * sizeof(T) +
         (size_t)NW * 16 * G * sizeof(float2);
}

// Warps per CTA: DYNSPLIT_ATTN_NW in {4, 8, 12}.  Default 8 (one CTA per SM,
// 3-deep rings): measured best at 128K / budget 4096 (15.4 us vs 17.7 with
// 4 warps x 3 CTAs per SM): fewer split partials to merge.
static int attn_nw() {
  static const int nw = [] {
    const char* e = getenv("DYNSPLIT_ATTN_NW");
    const int v = e ? atoi(e) : 8;
    return (v == 4 || v == 12) ? v : 8;
  }();
  return nw;
}

template <typename T, int G, int NW>
struct AttnLaunch {
  static constexpr int D = 2;  // pages in flight per warp while it computes one (3 measured slower)
  static int occupancy(int P) {
    return occupancy_of(k_decode_attn<T, G, NW, D>, NW * 32, attn_smem<T, G, NW, D>(P));
  }
  static cudaError_t run(const void* q, const void* Kp, const void* Vp, const int16_t* pv,
                         const int32_t* n_pages, const int32_t* wl_hdr, const int32_t* wl_count,
                         const WLEntry* wl, int dense, int B, int Hq, int Hkv, int max_pages, int P,
                         float scale_log2, float* part_o, float* part_lse, int* counters,
                         float* o, float* lse, cudaStream_t st) {
    const int occ = occupancy(P);
    allow_max_dyn_smem(k_decode_attn<T, G, NW, D>);
    const int n_split = max(1, min(kMaxSplit, (num_sms() * occ) / max(1, B * Hkv)));
    // A/B variant (DYNSPLIT_ATTN_TMA=1): pages by 2-D TMA boxes (bf16, P = 16, 8 warps)
    CUtensorMap tmK, tmV;
    memset(&tmK, 0, sizeof(tmK));
    memset(&tmV, 0, sizeof(tmV));
    int tma = 0;
    if (sizeof(T) == 2 && P == 16 && NW == 8 && getenv("DYNSPLIT_ATTN_TMA")) {
      const auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
      const cuuint64_t dims[2] = {(cuuint64_t)kD, (cuuint64_t)B * Hkv * max_pages * 16};
      const cuuint64_t strides[1] = {(cuuint64_t)kD * 2};
      const cuuint32_t box[2] = {64, 16};
      const cuuint32_t es[2] = {1, 1};
      tma = encode && encode(&tmK, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(Kp), dims, strides, box,
                             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
            encode(&tmV, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(Vp), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    launch_ex(k_decode_attn<T, G, NW, D>, dim3(n_split, Hkv, B), dim3(NW * 32),
              attn_smem<T, G, NW, D>(P) + (tma ? 1024 : 0), st, 1, static_cast<const T*>(q), static_cast<const T*>(Kp),
              static_cast<const T*>(Vp), pv, n_pages, wl_hdr, wl_count, wl, dense, Hq, Hkv,
              max_pages, P, scale_log2, part_o, part_lse, counters, n_split, o, lse, tma, tmK, tmV);
    return post_launch("k_decode_attn", st);
  }
};

template <typename T, int G>
static cudaError_t attn_run(const void* q, const void* Kp, const void* Vp, const int16_t* pv,
                            const int32_t* n_pages, const int32_t* wl_hdr, const int32_t* wl_count,
                            const WLEntry* wl, int dense, int B, int Hq, int Hkv, int max_pages, int P,
                            float sl2, float* part_o, float* part_lse, int* counters, float* o,
                            float* lse, cudaStream_t st) {
  if (attn_nw() == 4)
    return AttnLaunch<T, G, 4>::run(q, Kp, Vp, pv, n_pages, wl_hdr, wl_count, wl, dense, B, Hq, Hkv,
                                    max_pages, P, sl2, part_o, part_lse, counters, o, lse, st);
  if (attn_nw() == 12)
    return AttnLaunch<T, G, 12>::run(q, Kp, Vp, pv, n_pages, wl_hdr, wl_count, wl, dense, B, Hq, Hkv,
                                     max_pages, P, sl2, part_o, part_lse, counters, o, lse, st);
  return AttnLaunch<T, G, 8>::run(q, Kp, Vp, pv, n_pages, wl_hdr, wl_count, wl, dense, B, Hq, Hkv,
                                  max_pages, P, sl2, part_o, part_lse, counters, o, lse, st);
}

}  // namespace dsk
extern "C" int dynsplit_debug_attn_timer(void* dev_ptr) {
  return (int)cudaMemcpyToSymbol(dsk::g_attn_dbg, &dev_ptr, sizeof(void*));
}
extern "C" int dynsplit_debug_attn_noload(int on) {
  return (int)cudaMemcpyToSymbol(dsk::g_attn_noload, &on, sizeof(int));
}
namespace dsk {

cudaError_t launch_decode_attn(int dtype, int G, const void* q, const void* Kp, const void* Vp,
                               const int16_t* pv, const int32_t* n_pages, const int32_t* wl_hdr,
                               const int32_t* wl_count, const WLEntry* wl, int dense, int B, int Hq,
                               int Hkv, int max_pages, int P, float scale, float* part_o,
                               float* part_lse, int* counters, float* o, float* lse, cudaStream_t st) {
  const float sl2 = scale * 1.4426950408889634f;
#define DSK_ARGS q, Kp, Vp, pv, n_pages, wl_hdr, wl_count, wl, dense, B, Hq, Hkv, max_pages, P, sl2, \
                 part_o, part_lse, counters, o, lse, st
  if (dtype == 0) {
    switch (G) {
      case 1: return attn_run<bf16, 1>(DSK_ARGS);
      case 2: return attn_run<bf16, 2>(DSK_ARGS);
      case 4: return attn_run<bf16, 4>(DSK_ARGS);
      case 8: return attn_run<bf16, 8>(DSK_ARGS);
    }
  } else {
    switch (G) {
      case 1: return attn_run<float, 1>(DSK_ARGS);
      case 2: return attn_run<float, 2>(DSK_ARGS);
      case 4: return attn_run<float, 4>(DSK_ARGS);
      case 8: return attn_run<float, 8>(DSK_ARGS);
    }
  }
#undef DSK_ARGS
  return cudaErrorInvalidValue;
}

}  // namespace dsk
