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
//  * A warp handles ALL G query heads
//    of the KV group on them, so each K/V byte is read from HBM once:
//    bf16 caches: QK and PV as mma.sync m16n8k16 tiles (see the consumer);
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
__device__ int g_attn_noload = 0;     // debug: compute on stale smem without loading pages
__device__ unsigned long long* g_attn_pages = nullptr;  // debug: per-page (arrive, done) times of CTA 0
DSK_DEVICE void pstamp(int warp, int i, int k) {
#ifdef DSK_DEBUG
  if (g_attn_pages && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (threadIdx.x & 31) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_attn_pages[(i * 2 + k)] = t;
  }
#else
  (void)warp; (void)i; (void)k;
#endif
}
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

// Ring geometry: every consumer warp owns a private ring of `depth` stages;
// a stage holds max(P, 16) padded K rows followed by as many V rows (the bf16
// tensor-core path consumes 16-row tiles).  The depth is D for P <= 16 bf16
// pages and shrinks (>= 1) so that the CTA's rings stay within the budget:
// 72 KiB with 4 warps (3 CTAs per SM), 210 KiB with more (one CTA per SM).
__host__ __device__ inline size_t attn_ring_budget(int NW) { return NW <= 4 ? 72 * 1024 : 210 * 1024; }
__host__ __device__ inline int attn_stage_rows(int P) { return P < 16 ? 16 : P; }
__host__ __device__ inline size_t attn_stage_bytes(int row_bytes, int P) {
  return (size_t)2 * attn_stage_rows(P) * (row_bytes + 16);
}
__host__ __device__ inline int attn_depth(int D, int NW, int row_bytes, int P) {
  const int n = (int)(attn_ring_budget(NW) / ((size_t)NW * attn_stage_bytes(row_bytes, P)));
  return n < 1 ? 1 : (n > D ? D : n);
}
DSK_DEVICE void cp_async_commit_group() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// wait until at most n of this thread's most recent cp.async groups are pending
DSK_DEVICE void cp_async_wait_pending(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
  }
}

// ---------------------------------------------------------------- mma.sync helpers (bf16 path)
DSK_DEVICE void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
DSK_DEVICE void mma_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
DSK_DEVICE uint32_t bf16x2_bits(__nv_bfloat162 v) { return *reinterpret_cast<uint32_t*>(&v); }

template <typename T, int G, int NW, int D>
__global__ void __launch_bounds__(NW * 32, NW >= 8 ? 1 : 3) k_decode_attn(
    const T* __restrict__ q, const T* __restrict__ Kp, const T* __restrict__ Vp,
    const int16_t* __restrict__ page_valid, const int32_t* __restrict__ n_pages,
    const int32_t* __restrict__ wl_hdr, const int32_t* __restrict__ wl_count,
    const WLEntry* __restrict__ wl, int dense, int Hq, int Hkv, int max_pages, int P,
    float scale_log2, float* __restrict__ part_o, float* __restrict__ part_lse,
    int* __restrict__ counters, int n_split, float* __restrict__ o, float* __restrict__ lse) {
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

  const int split = blockIdx.x, hk = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = b * Hkv + hk;

  if (threadIdx.x == 0) astamp(0);
  // prologue independent of the preceding kernel (PDL overlap): V ring reset
  if (kTC) {
    const int nz = (int)(kstage / 16);
    for (int s2 = 0; s2 < NW * nd; ++s2) {
      uint4* vz = reinterpret_cast<uint4*>(smem + s2 * stage + kstage);
      for (int c = threadIdx.x; c < nz; c += blockDim.x) vz[c] = make_uint4(0u, 0u, 0u, 0u);
    }
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
#ifdef DSK_DEBUG
  if (g_attn_dbg) {  // debug timeline: wait for the entry loads before stamping
    if (__shfl_sync(0xffffffffu, e_page, 0) < 0) e_page = 0;
    if (threadIdx.x == 0) astamp(6);
  }
#endif
  __syncthreads();  // s_q and the zeroed V rings are visible to every warp

  // ---- per-warp load pipeline: warp w issues page j + depth with 16-byte
  // cp.async (LDGSTS) into its own ring while it computes page j;
  // completion by cp.async.wait_group, no barriers between warps.
  const int n_mine = n_it > warp ? (n_it - warp + NW - 1) / NW : 0;
  unsigned char* wring = smem + (size_t)warp * nd * stage;
  auto issue = [&](int j) {
    if (j < n_mine) {
      if ((j & 31) == 0 && j) load_batch(j, n_eff);
      const int pg = __shfl_sync(0xffffffffu, e_page, j & 31);
      const uint32_t a = __shfl_sync(0xffffffffu, e_r0, j & 31);
      const uint32_t c = __shfl_sync(0xffffffffu, e_r1, j & 31);
      int rmax = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) rmax = max(rmax, (int)(((g < 4 ? a : c) >> (8 * (g & 3))) & 0xffu));
      if ((unsigned)pg >= (unsigned)max_pages) rmax = 0;  // a corrupt worklist is never read past the pages
#ifdef DSK_DEBUG
      if (g_attn_noload) rmax = 0;
#endif
      const int st = j % nd;
      if (lane == 0) {
        s_rows[warp * D + st][0] = a;
        s_rows[warp * D + st][1] = c;
      }
      // valid rows only (padding rows of a page are never read from HBM);
      // lane -> fixed 16-byte column chunk, RPI rows per warp instruction
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
  if (threadIdx.x == 0) astamp(7);

  // ------------------------------------------------------------------ consumers
  float* sc = reinterpret_cast<float*>(smem);  // merge scratch [NW][G][kScStride], reuses the ring
  if constexpr (kTC) {
    // bf16: per 16-row tile of a page, two m16n8k16 tensor-core products.
    //   QK: S[head][key] with M = the G query heads (rows G..15 zero), N =
    //       16 keys, K = 128 dims: A = q (registers, loaded once), B = K rows
    //       by ldmatrix (padded rows: conflict-free), 4 chains of 4 k-steps.
    //       Lane (g = lane / 4, t = lane % 4) gets head g at keys
    //       {2t, 2t+1, 2t+8, 2t+9}.
    //   softmax: quad shuffles per head, exp2 domain, conditional rescale
    //       (the running max moves only when a logit exceeds it by > 2^8).
    //   PV: O^T[dim][head] with M = 16 dims x 8 tiles, N = 8 heads, K = 16
    //       keys: A = V^T by ldmatrix.trans of the V rows, B = P^T, which is
    //       exactly the QK output fragment, split into bf16 hi + lo parts
    //       (p = hi + lo to 2^-17 relative: fp32-level accuracy of P V);
    //       fp32 accumulation.  Lane holds dims {16j + g, 16j + g + 8} of
    //       heads {2t, 2t+1}.
    const int g = lane >> 2, t = lane & 3;
    uint32_t qa[8][2];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qa[ks][0] = qa[ks][1] = 0u;
      if (g < G) {
        const uint32_t* qw = reinterpret_cast<const uint32_t*>(s_q + (size_t)g * kD + ks * 16 + 2 * t);
        qa[ks][0] = qw[0];
        qa[ks][1] = qw[4];
      }
    }
    float m_run = -CUDART_INF_F, l_run = 0.f;
    float acc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    // ldmatrix.x4 lane address: matrix mi = lane / 8 covers keys 8 (mi / 2) + 0..7
    // and 16-byte column block mi % 2 (K: B halves of the two key tiles;
    // V with .trans: the four A quarters of a 16-dim tile)
    const int mi = lane >> 3, lr = lane & 7;
    const uint32_t koff = (uint32_t)(((mi >> 1) * 8 + lr) * KROW + (mi & 1) * 16);
    const uint32_t voff = koff;
    const uint32_t wring_s = smem_u32(wring);
    for (int j = 0; j < n_mine; ++j) {
      const int i = warp + j * NW, st = j % nd;
      pstamp(warp, i, 0);
      cp_async_wait_pending(nd - 1);  // this lane's copies of page j have landed
      __syncwarp();                   // ... and every lane's
      pstamp(warp, i, 1);
      if (threadIdx.x == 0 && j == 0) astamp(2);
#ifdef DSK_DEBUG
      if (g_attn_nocompute) {
        issue(j + nd);
        continue;
      }
#endif
      const uint32_t ra = s_rows[warp * D + st][0], rc = s_rows[warp * D + st][1];
      int rmax = 0;
#pragma unroll
      for (int h = 0; h < G; ++h) rmax = max(rmax, (int)(((h < 4 ? ra : rc) >> (8 * (h & 3))) & 0xffu));
      const int myrows = g < G ? (int)(((g < 4 ? ra : rc) >> (8 * (g & 3))) & 0xffu) : 0;
      for (int r0 = 0; r0 < rmax; r0 += 16) {
        const uint32_t kb = wring_s + (uint32_t)(st * stage + r0 * KROW) + koff;
        const uint32_t vb = wring_s + (uint32_t)(st * stage + kstage + r0 * KROW) + voff;
        float s[4][4];
#pragma unroll
        for (int c = 0; c < 4; ++c) s[c][0] = s[c][1] = s[c][2] = s[c][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t bk[4];
          ldsm_x4(bk, kb + ks * 32);
          mma_rows8(s[(ks & 1) * 2 + 0], qa[ks][0], qa[ks][1], bk[0], bk[1]);
          mma_rows8(s[(ks & 1) * 2 + 1], qa[ks][0], qa[ks][1], bk[2], bk[3]);
        }
        const int k0 = r0 + 2 * t;
        float z[4];
        z[0] = k0 < myrows ? (s[0][0] + s[2][0]) * scale_log2 : -CUDART_INF_F;
        z[1] = k0 + 1 < myrows ? (s[0][1] + s[2][1]) * scale_log2 : -CUDART_INF_F;
        z[2] = k0 + 8 < myrows ? (s[1][0] + s[3][0]) * scale_log2 : -CUDART_INF_F;
        z[3] = k0 + 9 < myrows ? (s[1][1] + s[3][1]) * scale_log2 : -CUDART_INF_F;
        const float zmax = fmaxf(fmaxf(z[0], z[1]), fmaxf(z[2], z[3]));
        if (__any_sync(0xffffffffu, zmax > m_run + 8.f)) {
          float mx = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, 1));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
          const float mnew = fmaxf(m_run, mx);
          const float corr = (mnew == -CUDART_INF_F || m_run == mnew) ? 1.f : exp2f(m_run - mnew);
          m_run = mnew;
          l_run *= corr;
          const float c0 = __shfl_sync(0xffffffffu, corr, 8 * t);      // head 2t
          const float c1 = __shfl_sync(0xffffffffu, corr, 8 * t + 4);  // head 2t + 1
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            acc[j][0] *= c0;
            acc[j][1] *= c1;
            acc[j][2] *= c0;
            acc[j][3] *= c1;
          }
        }
        float p[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          p[k] = z[k] == -CUDART_INF_F ? 0.f : exp2f(z[k] - m_run);
          l_run += p[k];
        }
        const __nv_bfloat162 h01 = __floats2bfloat162_rn(p[0], p[1]);
        const __nv_bfloat162 h23 = __floats2bfloat162_rn(p[2], p[3]);
        const __nv_bfloat162 l01 = __floats2bfloat162_rn(p[0] - __low2float(h01), p[1] - __high2float(h01));
        const __nv_bfloat162 l23 = __floats2bfloat162_rn(p[2] - __low2float(h23), p[3] - __high2float(h23));
        const uint32_t bh0 = bf16x2_bits(h01), bh1 = bf16x2_bits(h23);
        const uint32_t bl0 = bf16x2_bits(l01), bl1 = bf16x2_bits(l23);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t av[4];
          ldsm_x4_t(av, vb + j * 32);
          // ldmatrix order (keys lo, dims lo), (keys lo, dims hi), (keys hi, dims lo),
          // (keys hi, dims hi) -> A quarters a0, a1, a2, a3 of V^T
          const uint32_t a[4] = {av[0], av[1], av[2], av[3]};
          mma_16816(acc[j], a, bh0, bh1);
          mma_16816(acc[j], a, bl0, bl1);
        }
      }
      __syncwarp();  // the stage is free
      issue(j + nd);
      pstamp(warp, 64 + i, 0);
    }
    // ---- per-warp state to the merge scratch (the ring is free once all are here)
    named_bar_sync(1, NW * 32);
    if (threadIdx.x == 0) astamp(3);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int h = 2 * t + e;
      if (h < G) {
        float* row = sc + (warp * G + h) * kScStride + g;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          row[16 * j] = acc[j][e];
          row[16 * j + 8] = acc[j][2 + e];
        }
      }
    }
    if (g < G && t == 0) {
      sc[(warp * G + g) * kScStride + kD] = m_run;
      sc[(warp * G + g) * kScStride + kD + 1] = l_run;
    }
  } else {
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
    const int i = warp + jp * NW, st = jp % nd;
    pstamp(warp, i, 0);
    cp_async_wait_pending(nd - 1);
    __syncwarp();
    pstamp(warp, i, 1);
    if (threadIdx.x == 0 && jp == 0) astamp(2);
#ifdef DSK_DEBUG
    if (g_attn_nocompute) {
      issue(jp + nd);
      continue;
    }
#endif
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
    pstamp(warp, 64 + i, 0);
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
  // ---- merge the NW warps (fixed order)
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
  // Last CTA of (b, KV head): LSE merge of the n_eff splits.  R = NW / G
  // warps share a head: every warp reads all split lse values (lanes hold
  // them, n_eff <= 64) and forms the weights by warp reductions (fixed
  // butterfly order); warp part r sums w_s o_s over the splits s = r (mod R)
  // with all its loads in flight at once (n_eff / R <= 16 per lane); the R
  // parts are added in part order through shared memory.
  constexpr int R = NW >= G ? NW / G : 1;
  float* mrg = reinterpret_cast<float*>(smem);  // [G][R][kD]
  // warp w merges (head, part) pairs hp = w, w + NW, ...: with NW < G (e.g. 4
  // warps, G = 8) a warp takes several heads; R parts per head when NW >= G
  for (int hp = warp; hp < G * R; hp += NW) {
    const int h = hp % G, part = hp / G;
    const size_t row = (size_t)b * Hq + hk * G + h;
    const float* pl = part_lse + row * n_split;
    const float4* po_base = reinterpret_cast<const float4*>(part_o + row * n_split * kD) + lane;
    // the first 16 partial-o loads of this part are issued together with the
    // lse loads, so their L2 latency overlaps the weight reductions
    float4 po[16];
    auto load_po = [&](int s0) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int s = s0 + k * R;
        po[k] = s < n_eff ? __ldcg(po_base + (size_t)s * (kD / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    load_po(part);
    const float l0 = lane < n_eff ? __ldcg(pl + lane) : -CUDART_INF_F;
    const float l1 = lane + 32 < n_eff ? __ldcg(pl + lane + 32) : -CUDART_INF_F;
    float4 ov = make_float4(0.f, 0.f, 0.f, 0.f);
    const float M = warp_max(fmaxf(l0, l1));
    float L = -CUDART_INF_F;
    if (M != -CUDART_INF_F) {
      const float sum = warp_sum(expf(l0 - M) + expf(l1 - M));
      L = M + logf(sum);
      const float w0 = expf(l0 - L), w1 = expf(l1 - L);
      for (int s0 = part; s0 < n_eff; s0 += 16 * R) {
        if (s0 != part) load_po(s0);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int s = s0 + k * R;
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
    if (R == 1) {
      reinterpret_cast<float4*>(o + row * kD)[lane] = ov;
      if (lane == 0) lse[row] = L;
    } else {
      reinterpret_cast<float4*>(mrg + (h * R + part) * kD)[lane] = ov;
      if (part == 0 && lane == 0) lse[row] = L;
    }
  }
  if (R > 1) {
    named_bar_sync(1, NW * 32);
    for (int j = threadIdx.x; j < G * (kD / 4); j += NW * 32) {
      const int h = j / (kD / 4), c = j % (kD / 4);
      float4 acc = reinterpret_cast<const float4*>(mrg + (h * R) * kD)[c];
      for (int rr = 1; rr < R; ++rr) {
        const float4 x = reinterpret_cast<const float4*>(mrg + (h * R + rr) * kD)[c];
        acc.x += x.x;
        acc.y += x.y;
        acc.z += x.z;
        acc.w += x.w;
      }
      reinterpret_cast<float4*>(o + ((size_t)b * Hq + hk * G + h) * kD)[c] = acc;
    }
  }
  if (threadIdx.x == 0) {
    counters[bh] = 0;
    astamp(5);
  }
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
    launch_ex(k_decode_attn<T, G, NW, D>, dim3(n_split, Hkv, B), dim3(NW * 32),
              attn_smem<T, G, NW, D>(P), st, 1, static_cast<const T*>(q), static_cast<const T*>(Kp),
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
extern "C" int dynsplit_debug_attn_pages(void* dev_ptr) {
  return (int)cudaMemcpyToSymbol(dsk::g_attn_pages, &dev_ptr, sizeof(void*));
}
extern "C" int dynsplit_debug_attn_noload(int on) {
  return (int)cudaMemcpyToSymbol(dsk::g_attn_noload, &on, sizeof(int));
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
