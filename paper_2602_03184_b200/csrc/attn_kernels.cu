// Decode rows a7 + a8 (a9 in dense mode): split-K flash-decoding over the
// selected pages of the GQA-union worklist, with the log-sum-exp merge of the
// splits (Step 3 of KV selection; "split-K ... log-sum-exp merge",
// north star).
//
// grid (n_split, Hkv, B) sized to one resident wave; NW consumer warps + 1
// producer warp per CTA.
//  * Producer warp: loads 32 worklist entries at a time (coalesced), then lane
//    0 streams each page's valid rows of K and V (rows_max x 256 B, TMA 1-D
//    bulk copies, L2 evict-first) into an NS-deep smem ring (full/empty
//    mbarriers).  Padding rows of a page are never read from HBM.
//  * Consumer warp w takes pages i = w (mod NW) and handles ALL G query heads
//    of the KV group on them, so each K/V byte is read from HBM once:
//      QK:  lane (hg = lane/16, r = lane%16) computes the full 128-dim dot of
//           row r with heads hg, hg+2, ...; 16-byte chunks are visited in the
//           rotated order (c + r) mod 16, so the 16 rows hit 16 distinct bank
//           groups (conflict-free), bf16 x bf16 -> fp32 with FHFMA.BF16
//           (no conversions), fp32 q with FFMA for fp32 caches.
//      softmax: per head over the 16 lanes of its group (4 xor-shuffles),
//           exp2 domain, online max/sum.
//      PV:  lane owns dims [4 lane, 4 lane + 4) for all G heads, P from a
//           per-warp smem slab (float2 (p, p) pairs) and FFMA2.
//  * Warps are merged in fixed order; each CTA writes its split's (o, lse);
//    the last CTA of a (b, KV head) merges the splits in split order.
#include "common.cuh"
#include "kernels.h"

#include <math_constants.h>
#include <stdlib.h>

namespace dsk {

constexpr int kScStride = kD + 4;  // merge scratch row: acc[kD], m, l (16-byte aligned rows)
constexpr int kMinPagesPerSplit = 4;

// Optional per-CTA phase timestamps (debug only; dynsplit_debug_attn_timer).
__device__ unsigned long long* g_attn_dbg = nullptr;
__device__ int g_attn_nocompute = 0;  // debug: stream pages without computing
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
template <> struct QK<bf16> {
  static constexpr int kChunks = kD * 2 / 16;  // 16 chunks of 8 bf16
  static DSK_DEVICE float dot(uint4 qc, uint4 kc, float acc) {
    const uint32_t qs[4] = {qc.x, qc.y, qc.z, qc.w};
    const uint32_t ks[4] = {kc.x, kc.y, kc.z, kc.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      unsigned short ql, qh, kl, kh;
      split_bf16x2(qs[e], ql, qh);
      split_bf16x2(ks[e], kl, kh);
      acc = fma_bf16(ql, kl, acc);
      acc = fma_bf16(qh, kh, acc);
    }
    return acc;
  }
};
template <> struct QK<float> {
  static constexpr int kChunks = kD * 4 / 16;  // 32 chunks of 4 fp32
  static DSK_DEVICE float dot(uint4 qc, uint4 kc, float acc) {
    acc = fmaf(__uint_as_float(qc.x), __uint_as_float(kc.x), acc);
    acc = fmaf(__uint_as_float(qc.y), __uint_as_float(kc.y), acc);
    acc = fmaf(__uint_as_float(qc.z), __uint_as_float(kc.z), acc);
    acc = fmaf(__uint_as_float(qc.w), __uint_as_float(kc.w), acc);
    return acc;
  }
};

template <typename T, int G, int NW, int NS>
__global__ void __launch_bounds__((NW + 1) * 32, NW >= 8 ? 2 : 3) k_decode_attn(
    const T* __restrict__ q, const T* __restrict__ Kp, const T* __restrict__ Vp,
    const int16_t* __restrict__ page_valid, const int32_t* __restrict__ n_pages,
    const int32_t* __restrict__ wl_hdr, const int32_t* __restrict__ wl_count,
    const WLEntry* __restrict__ wl, int dense, int Hq, int Hkv, int max_pages, int P,
    float scale_log2, float* __restrict__ part_o, float* __restrict__ part_lse,
    int* __restrict__ counters, int n_split, float* __restrict__ o, float* __restrict__ lse) {
  constexpr int CH = QK<T>::kChunks;
  constexpr int HPL = (G + 1) / 2;  // heads per QK lane
  extern __shared__ __align__(128) unsigned char smem[];
  const size_t stage_bytes = (size_t)P * kD * sizeof(T);
  unsigned char* ringK = smem;
  unsigned char* ringV = smem + NS * stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * NS * stage_bytes);
  uint64_t* empty = full + NS;
  uint32_t(*s_rows)[2] = reinterpret_cast<uint32_t(*)[2]>(empty + NS);
  T* s_q = reinterpret_cast<T*>(s_rows + NS);                      // [G][kD]
  float2* pbuf = reinterpret_cast<float2*>(s_q + G * kD);          // [NW][16][G]
  __shared__ int s_last;

  const int split = blockIdx.x, hk = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = b * Hkv + hk;

  if (threadIdx.x == 0) astamp(0);
  // prologue independent of the preceding kernel (PDL overlap): barriers, q
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  {
    constexpr int QCH = G * kD * (int)sizeof(T) / 16;
    const uint4* src = reinterpret_cast<const uint4*>(q + ((size_t)b * Hq + hk * G) * kD);
    for (int c = threadIdx.x; c < QCH; c += blockDim.x) reinterpret_cast<uint4*>(s_q)[c] = src[c];
  }
  pdl_trigger();
  pdl_wait();  // the worklist is the previous kernel's output
  if (threadIdx.x == 0) astamp(1);

  const int cnt = dense ? n_pages[b] : wl_count[bh];
  // splits actually used by this (b, KV head): at least kMinPagesPerSplit pages each
  const int n_eff = max(1, min(n_split, (cnt + kMinPagesPerSplit - 1) / kMinPagesPerSplit));
  if (split >= n_eff) return;
  const int e_lo = (int)(((long long)split * cnt) / n_eff);
  const int e_hi = (int)(((long long)(split + 1) * cnt) / n_eff);
  const int n_it = e_hi - e_lo;

  // producer warp: first batch of 32 worklist entries before the CTA barrier
  const int max_wl = dense ? 0 : wl_hdr[1];
  const WLEntry* wlb = wl + (size_t)bh * max_wl + e_lo;
  auto load_entry = [&](int idx, int& page, uint32_t& r0, uint32_t& r1) {
    page = 0;
    r0 = r1 = 0;
    if (idx < n_it) {
      if (dense) {
        page = e_lo + idx;
        const uint32_t pv = (uint32_t)page_valid[(size_t)b * max_pages + page];
        r0 = r1 = pv * 0x01010101u;
      } else {
        const int4 e = *reinterpret_cast<const int4*>(wlb + idx);
        page = e.x;
        r0 = (uint32_t)e.z;
        r1 = (uint32_t)e.w;
      }
    }
  };
  int page = 0;
  uint32_t r0 = 0, r1 = 0;
  if (warp == NW) load_entry(lane, page, r0, r1);
  __syncthreads();

  if (warp == NW) {  // ---------------------------------------------- producer
    const uint64_t pol = policy_evict_first();
    for (int base = 0; base < n_it; base += 32) {
      if (base) load_entry(base + lane, page, r0, r1);
      const int nk = min(32, n_it - base);
      for (int k = 0; k < nk; ++k) {
        const int i = base + k, st = i % NS;
        const int pg = __shfl_sync(0xffffffffu, page, k);
        const uint32_t a = __shfl_sync(0xffffffffu, r0, k);
        const uint32_t c = __shfl_sync(0xffffffffu, r1, k);
        if (lane == 0) {
          if (i >= NS) mbar_wait(&empty[st], ((i / NS) - 1) & 1);
          int rmax = 0;
#pragma unroll
          for (int g = 0; g < G; ++g) rmax = max(rmax, (int)(((g < 4 ? a : c) >> (8 * (g & 3))) & 0xffu));
          s_rows[st][0] = a;
          s_rows[st][1] = c;
          const uint32_t bytes = (uint32_t)rmax * kD * sizeof(T);
          mbar_arrive_expect_tx(&full[st], 2 * bytes);
          if (bytes) {
            const size_t off = ((size_t)bh * max_pages + pg) * stage_bytes;
            bulk_g2s(ringK + st * stage_bytes, reinterpret_cast<const unsigned char*>(Kp) + off, bytes,
                     &full[st], pol);
            bulk_g2s(ringV + st * stage_bytes, reinterpret_cast<const unsigned char*>(Vp) + off, bytes,
                     &full[st], pol);
          }
        }
        __syncwarp();
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
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

  for (int i = warp; i < n_it; i += NW) {
    const int st = i % NS;
    mbar_wait(&full[st], (i / NS) & 1);
    if (threadIdx.x == 0 && i == 0) astamp(2);
#ifdef DSK_DEBUG
    if (g_attn_nocompute) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      continue;
    }
#endif
    const uint32_t ra = s_rows[st][0], rc = s_rows[st][1];
    int rmax = 0, myrows[HPL];
#pragma unroll
    for (int g = 0; g < G; ++g) rmax = max(rmax, (int)(((g < 4 ? ra : rc) >> (8 * (g & 3))) & 0xffu));
#pragma unroll
    for (int j = 0; j < HPL; ++j) {
      const int h = hg + 2 * j;
      myrows[j] = h < G ? (int)(((h < 4 ? ra : rc) >> (8 * (h & 3))) & 0xffu) : 0;
    }
    const unsigned char* Ks = ringK + st * stage_bytes;
    const T* Vs = reinterpret_cast<const T*>(ringV + st * stage_bytes);
    for (int r0 = 0; r0 < rmax; r0 += 16) {
      const int nr = min(16, rmax - r0);
      const bool rowok = r < nr;
      float dot[HPL];
#pragma unroll
      for (int j = 0; j < HPL; ++j) dot[j] = 0.f;
      if (rowok) {
        const unsigned char* krow = Ks + (size_t)(r0 + r) * kD * sizeof(T);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int off = ((c + r) & (CH - 1)) * 16;
          const uint4 kc = *reinterpret_cast<const uint4*>(krow + off);
#pragma unroll
          for (int j = 0; j < HPL; ++j) {
            const int h = hg + 2 * j;
            if (h < G) {
              const uint4 qc = *reinterpret_cast<const uint4*>(qbase + (size_t)h * kD * sizeof(T) + off);
              dot[j] = QK<T>::dot(qc, kc, dot[j]);
            }
          }
        }
      }
      float p[HPL], corr[HPL];
#pragma unroll
      for (int j = 0; j < HPL; ++j) {
        const int h = hg + 2 * j;
        const bool valid = rowok && (r0 + r) < myrows[j];
        const float z = valid ? dot[j] * scale_log2 : -CUDART_INF_F;
        float mx = z;
#pragma unroll
        for (int o2 = 1; o2 < 16; o2 <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
        const float mnew = fmaxf(m[j], mx);
        corr[j] = (mnew == -CUDART_INF_F) ? 1.f : exp2f(m[j] - mnew);
        p[j] = valid ? exp2f(z - mnew) : 0.f;
        float ps = p[j];
#pragma unroll
        for (int o2 = 1; o2 < 16; o2 <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o2);
        l[j] = l[j] * corr[j] + ps;
        m[j] = mnew;
        if (h < G) pb[r * G + h] = make_float2(p[j], p[j]);
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float ch = __shfl_sync(0xffffffffu, corr[h >> 1], (h & 1) * 16);
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[h][k] *= ch;
      }
      for (int rr = 0; rr < nr; ++rr) {
        float v[4];
        Vec<T>::load4(Vs + (size_t)(r0 + rr) * kD + lane * 4, v);
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
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  // ---- merge the NW warps (fixed order); the ring is free once all are here
  named_bar_sync(1, NW * 32);
  if (threadIdx.x == 0) astamp(3);
  float* sc = reinterpret_cast<float*>(smem);  // [NW][G][kD + 2]
#pragma unroll
  for (int h = 0; h < G; ++h)
    *reinterpret_cast<float4*>(sc + (warp * G + h) * kScStride + lane * 4) =
        make_float4(acc[h][0], acc[h][1], acc[h][2], acc[h][3]);
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
  named_bar_sync(1, NW * 32);
  const float LN2 = 0.69314718055994530942f;
  for (int h = warp; h < G; h += NW) {
    float M = -CUDART_INF_F;
    for (int w = 0; w < NW; ++w) M = fmaxf(M, sc[(w * G + h) * kScStride + kD]);
    float L = 0.f, ov[4] = {0.f, 0.f, 0.f, 0.f};
    if (M != -CUDART_INF_F) {
      for (int w = 0; w < NW; ++w) {
        const float* s = sc + (w * G + h) * kScStride;
        const float f = exp2f(s[kD] - M);  // exp2(-inf) = 0 for empty warps
        L += s[kD + 1] * f;
        const float4 a4 = *reinterpret_cast<const float4*>(s + lane * 4);
        ov[0] += a4.x * f;
        ov[1] += a4.y * f;
        ov[2] += a4.z * f;
        ov[3] += a4.w * f;
      }
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    const float4 o4 = make_float4(ov[0] * inv, ov[1] * inv, ov[2] * inv, ov[3] * inv);
    const float lse2 = L > 0.f ? (M + log2f(L)) * LN2 : -CUDART_INF_F;
    const size_t row = (size_t)b * Hq + hk * G + h;
    if (n_eff == 1) {
      reinterpret_cast<float4*>(o + row * kD)[lane] = o4;
      if (lane == 0) lse[row] = lse2;
    } else {
      reinterpret_cast<float4*>(part_o + (row * n_split + split) * kD)[lane] = o4;
      if (lane == 0) part_lse[row * n_split + split] = lse2;
    }
  }
  if (n_eff == 1) return;
  // Split ticket: the CTA barrier orders every thread's partial writes before
  // thread 0's acq_rel atomic (cumulative release at gpu scope); the last CTA
  // acquires them through the same atomic (no full fences).
  named_bar_sync(1, NW * 32);
  if (threadIdx.x == 0) {
    int old;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(counters + bh) : "memory");
    s_last = (old == n_eff - 1);
  }
  named_bar_sync(1, NW * 32);
  if (threadIdx.x == 0) astamp(4);
  if (!s_last) return;
  // Last CTA of (b, KV head): LSE merge of the n_eff splits.  Lanes hold the
  // split lse values (n_eff <= 64), weights by warp reductions (fixed
  // butterfly order), then o = sum_s w_s o_s in split order, 16 loads in
  // flight per lane (the first batch issued before the weights are known).
  for (int h = warp; h < G; h += NW) {
    const size_t row = (size_t)b * Hq + hk * G + h;
    const float* pl = part_lse + row * n_split;
    const float4* po_base = reinterpret_cast<const float4*>(part_o + row * n_split * kD) + lane;
    const float l0 = lane < n_eff ? __ldcg(pl + lane) : -CUDART_INF_F;
    const float l1 = lane + 32 < n_eff ? __ldcg(pl + lane + 32) : -CUDART_INF_F;
    float4 po[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      po[k] = k < n_eff ? __ldcg(po_base + (size_t)k * (kD / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float M = warp_max(fmaxf(l0, l1));
    float4 ov = make_float4(0.f, 0.f, 0.f, 0.f);
    float L = -CUDART_INF_F;
    if (M != -CUDART_INF_F) {
      const float sum = warp_sum(expf(l0 - M) + expf(l1 - M));
      L = M + logf(sum);
      const float w0 = expf(l0 - L), w1 = expf(l1 - L);
      for (int s0 = 0; s0 < n_eff; s0 += 16) {
        if (s0) {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int s = s0 + k;
            po[k] = s < n_eff ? __ldcg(po_base + (size_t)s * (kD / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int s = s0 + k;
          const float w = __shfl_sync(0xffffffffu, s < 32 ? w0 : w1, s & 31);
          if (s < n_eff) {
            ov.x += w * po[k].x;
            ov.y += w * po[k].y;
            ov.z += w * po[k].z;
            ov.w += w * po[k].w;
          }
        }
      }
    }
    reinterpret_cast<float4*>(o + row * kD)[lane] = ov;
    if (lane == 0) lse[row] = L;
  }
  if (threadIdx.x == 0) {
    counters[bh] = 0;
    astamp(5);
  }
}

// ============================================================================
// host launcher
// ============================================================================
template <typename T, int G, int NW, int NS>
static size_t attn_smem(int P) {
  const size_t ring = (size_t)2 * NS * P * kD * sizeof(T);
  const size_t merge = (size_t)NW * G * kScStride * sizeof(float);
  return (ring > merge ? ring : merge) + 2 * NS * sizeof(uint64_t) + NS * 8 +
         (size_t)G * kD * sizeof(T) + (size_t)NW * 16 * G * sizeof(float2);
}

// Consumer warps per CTA: DYNSPLIT_ATTN_NW in {4, 8} (default 4: more CTAs beat more warps).
static int attn_nw() {
  static int nw = 0;
  if (!nw) {
    const char* e = getenv("DYNSPLIT_ATTN_NW");
    nw = (e && atoi(e) == 8) ? 8 : 4;
  }
  return nw;
}

template <typename T, int G, int NW>
struct AttnLaunch {
  static constexpr int NS = sizeof(T) == 2 ? 8 : 4;
  static int occupancy(int P) {
    static int occ = 0, lastP = -1;
    if (occ == 0 || lastP != P) {
      auto kern = k_decode_attn<T, G, NW, NS>;
      allow_max_dyn_smem(kern);
      int n = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, (NW + 1) * 32, attn_smem<T, G, NW, NS>(P)) !=
              cudaSuccess ||
          n < 1) {
        cudaGetLastError();
        n = 1;
      }
      occ = n;
      lastP = P;
    }
    return occ;
  }
  static cudaError_t run(const void* q, const void* Kp, const void* Vp, const int16_t* pv,
                         const int32_t* n_pages, const int32_t* wl_hdr, const int32_t* wl_count,
                         const WLEntry* wl, int dense, int B, int Hq, int Hkv, int max_pages, int P,
                         float scale_log2, float* part_o, float* part_lse, int* counters,
                         float* o, float* lse, cudaStream_t st) {
    const int occ = occupancy(P);
    const int n_split = max(1, min(kMaxSplit, (num_sms() * occ) / max(1, B * Hkv)));
    launch_ex(k_decode_attn<T, G, NW, NS>, dim3(n_split, Hkv, B), dim3((NW + 1) * 32),
              attn_smem<T, G, NW, NS>(P), st, 1, static_cast<const T*>(q), static_cast<const T*>(Kp),
              static_cast<const T*>(Vp), pv, n_pages, wl_hdr, wl_count, wl, dense, Hq, Hkv,
              max_pages, P, scale_log2, part_o, part_lse, counters, n_split, o, lse);
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
  return AttnLaunch<T, G, 8>::run(q, Kp, Vp, pv, n_pages, wl_hdr, wl_count, wl, dense, B, Hq, Hkv,
                                  max_pages, P, sl2, part_o, part_lse, counters, o, lse, st);
}

}  // namespace dsk
extern "C" int dynsplit_debug_attn_timer(void* dev_ptr) {
  return (int)cudaMemcpyToSymbol(dsk::g_attn_dbg, &dev_ptr, sizeof(void*));
}
extern "C" int dynsplit_debug_attn_nocompute(int on) {
  return (int)cudaMemcpyToSymbol(dsk::g_attn_nocompute, &on, sizeof(int));
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
