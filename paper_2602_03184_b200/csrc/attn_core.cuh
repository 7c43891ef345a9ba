// Shared core of the split-K flash-decoding rows a7 + a8 (Step 3 of KV
// selection): the per-warp bf16 page pipeline, the NW-warp merge,
// the split partial write and the last-CTA LSE merge of the splits.  Used by
// k_decode_attn (attn_kernels.cu, pages from the global worklist) and by the
// fused decode layer k_decode_fused (fused_kernels.cu, pages dealt into shared
// memory by the CTA itself), so the two produce bit-identical o and lse for
// the same page assignment.
#pragma once
#include "common.cuh"

#include <math_constants.h>

namespace dsk {

constexpr int kScStride = kD + 4;  // merge scratch row: acc[kD], m, l (16-byte aligned rows)
constexpr int kMinPagesPerSplit = 4;

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

// Rows of head h in a packed entry (8 bits per head: heads 0-3 in r0, 4-7 in r1).
DSK_DEVICE int entry_rows(uint32_t r0, uint32_t r1, int h) {
  return (int)(((h < 4 ? r0 : r1) >> (8 * (h & 3))) & 0xffu);
}

// Zero the V half of every stage of the NW rings (rows of a 16-row tile past
// the page's valid rows are multiplied by p = 0 and must never hold a
// non-finite pattern).
DSK_DEVICE void attn_zero_v_rings(unsigned char* ring, int n_stages, size_t kstage, size_t stage) {
  const int nz = (int)(kstage / 16);
  for (int s2 = 0; s2 < n_stages; ++s2) {
    uint4* vz = reinterpret_cast<uint4*>(ring + s2 * stage + kstage);
    for (int c = threadIdx.x; c < nz; c += blockDim.x) vz[c] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// ---------------------------------------------------------------------------
// bf16 per-warp pipeline.  Warp `warp` owns n_mine pages; entry(j) returns the
// warp-uniform entry {page, r0, r1} of its j-th page.  Each page's valid K and
// V rows go into 16-byte padded smem rows of the warp's private nd-stage ring
// with 16-byte cp.async (page j + nd issued while page j is computed), then
//   QK: S[head][key] with M = the G query heads (rows G..15 zero), N = 16
//       keys, K = 128 dims: A = q (registers, loaded once), B = K rows by
//       ldmatrix (padded rows: conflict-free), 4 chains of 4 k-steps.
//       Lane (g = lane / 4, t = lane % 4) gets head g at keys {2t, 2t+1, 2t+8, 2t+9}.
//   softmax: quad shuffles per head, exp2 domain, conditional rescale (the
//       running max moves only when a logit exceeds it by > 2^8).
//   PV: O^T[dim][head] with M = 16 dims x 8 tiles, N = 8 heads, K = 16 keys:
//       A = V^T by ldmatrix.trans of the V rows, B = P^T, which is exactly the
//       QK output fragment, split into bf16 hi + lo parts (p = hi + lo to
//       2^-17 relative: fp32-level accuracy of P V); fp32 accumulation.
// The warp's (acc, m, l) go to the merge scratch sc[NW][G][kScStride] (which
// reuses the ring: a named barrier over the NW warps precedes the writes).
// ---------------------------------------------------------------------------
template <int G, int NW, int D, typename EntryFn>
DSK_DEVICE void attn_bf16_pipeline(unsigned char* smem, uint32_t (*s_rows)[2], const bf16* s_q, int nd,
                                   int P, int n_mine, EntryFn entry, const bf16* __restrict__ Kp,
                                   const bf16* __restrict__ Vp, size_t bh, int max_pages, float scale_log2,
                                   bool noload) {
  constexpr int ROW = kD * 2;
  constexpr int KROW = ROW + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t kstage = (size_t)attn_stage_rows(P) * KROW, stage = 2 * kstage;
  const size_t hbm_page = (size_t)P * ROW;
  unsigned char* wring = smem + (size_t)warp * nd * stage;

  auto issue = [&](int j) {
    if (j < n_mine) {
      int pg;
      uint32_t a, c;
      entry(j, pg, a, c);
      int rmax = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) rmax = max(rmax, entry_rows(a, c, g));
      if ((unsigned)pg >= (unsigned)max_pages) rmax = 0;  // a corrupt worklist is never read past the pages
      if (noload) rmax = 0;
      const int st = j % nd;
      if (lane == 0) {
        s_rows[warp * D + st][0] = a;
        s_rows[warp * D + st][1] = c;
      }
      // valid rows only (padding rows of a page are never read from HBM);
      // lane -> fixed 16-byte column chunk, RPI rows per warp instruction
      constexpr int CPR = ROW / 16;
      constexpr int RPI = 32 / CPR;
      const size_t off = (bh * max_pages + pg) * hbm_page;
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
  // and 16-byte column block mi % 2 (K: B halves of the two key tiles; V with
  // .trans: the four A quarters of a 16-dim tile)
  const int mi = lane >> 3, lr = lane & 7;
  const uint32_t koff = (uint32_t)(((mi >> 1) * 8 + lr) * KROW + (mi & 1) * 16);
  const uint32_t voff = koff;
  const uint32_t wring_s = smem_u32(wring);
  for (int j = 0; j < n_mine; ++j) {
    const int st = j % nd;
    cp_async_wait_pending(nd - 1);  // this lane's copies of page j have landed
    __syncwarp();                   // ... and every lane's
    const uint32_t ra = s_rows[warp * D + st][0], rc = s_rows[warp * D + st][1];
    int rmax = 0;
#pragma unroll
    for (int h = 0; h < G; ++h) rmax = max(rmax, entry_rows(ra, rc, h));
    const int myrows = g < G ? entry_rows(ra, rc, g) : 0;
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
        for (int j2 = 0; j2 < 8; ++j2) {
          acc[j2][0] *= c0;
          acc[j2][1] *= c1;
          acc[j2][2] *= c0;
          acc[j2][3] *= c1;
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
      for (int j2 = 0; j2 < 8; ++j2) {
        uint32_t av[4];
        ldsm_x4_t(av, vb + j2 * 32);
        // ldmatrix order (keys lo, dims lo), (keys lo, dims hi), (keys hi, dims lo),
        // (keys hi, dims hi) -> A quarters a0, a1, a2, a3 of V^T
        const uint32_t a[4] = {av[0], av[1], av[2], av[3]};
        mma_16816(acc[j2], a, bh0, bh1);
        mma_16816(acc[j2], a, bl0, bl1);
      }
    }
    __syncwarp();  // the stage is free
    issue(j + nd);
  }
  // ---- per-warp state to the merge scratch (the ring is free once all are here)
  float* sc = reinterpret_cast<float*>(smem);
  named_bar_sync(1, NW * 32);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int h = 2 * t + e;
    if (h < G) {
      float* row = sc + (warp * G + h) * kScStride + g;
#pragma unroll
      for (int j2 = 0; j2 < 8; ++j2) {
        row[16 * j2] = acc[j2][e];
        row[16 * j2 + 8] = acc[j2][2 + e];
      }
    }
  }
  if (g < G && t == 0) {
    sc[(warp * G + g) * kScStride + kD] = m_run;
    sc[(warp * G + g) * kScStride + kD + 1] = l_run;
  }
}

// ---------------------------------------------------------------------------
// The same pipeline with the pages moved by TMA tensor copies instead of
// per-lane LDGSTS (A/B variant, DYNSPLIT_ATTN_TMA=1, bf16, P = 16): per page
// lane 0 issues four 2-D boxes (K / V x two 64-dim slabs, 16 rows x 128 B,
// 128-byte hardware swizzle) into an unpadded 8 KiB stage completing on the
// stage's mbarrier; ldmatrix reads the swizzled rows (chunk c of row r at
// (c ^ (r & 7)) * 16).  A box always moves all 16 rows of a page (its padding
// rows are zero in HBM), where LDGSTS moves only the rows some head needs.
// ---------------------------------------------------------------------------
template <int G, int NW, int D, typename EntryFn>
DSK_DEVICE void attn_bf16_pipeline_tma(unsigned char* ring, uint64_t* bars, uint32_t (*s_rows)[2],
                                       const bf16* s_q, int nd, int n_mine, EntryFn entry, const CUtensorMap* tmK,
                                       const CUtensorMap* tmV, size_t bh, int max_pages, float scale_log2) {
  constexpr int STAGE = 8192, SLAB = 2048;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wring = ring + (size_t)warp * nd * STAGE;
  uint64_t* wb = bars + warp * D;
  auto issue = [&](int j) {
    if (j >= n_mine) return;
    int pg;
    uint32_t a, c;
    entry(j, pg, a, c);
    int rmax = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) rmax = max(rmax, entry_rows(a, c, g));
    if ((unsigned)pg >= (unsigned)max_pages) rmax = 0;
    const int st = j % nd;
    if (lane == 0) {
      s_rows[warp * D + st][0] = rmax ? a : 0u;
      s_rows[warp * D + st][1] = rmax ? c : 0u;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // this stage's reads before the TMA writes
    __syncwarp();
    if (lane == 0) {
      if (rmax > 0) {
        const int row = (int)((bh * max_pages + pg) * 16);
        unsigned char* d = wring + st * STAGE;
        mbar_arrive_expect_tx(&wb[st], STAGE);
        tma_load_2d(d, tmK, 0, row, &wb[st]);
        tma_load_2d(d + SLAB, tmK, 64, row, &wb[st]);
        tma_load_2d(d + 2 * SLAB, tmV, 0, row, &wb[st]);
        tma_load_2d(d + 3 * SLAB, tmV, 64, row, &wb[st]);
      } else {
        mbar_arrive(&wb[st]);
      }
    }
  };
  for (int j = 0; j < nd; ++j) issue(j);

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
  // ldmatrix.x4 lane address: matrix mi = lane / 8 covers rows 8 (mi / 2) + lr
  // and 16-byte chunk 2 k + mi % 2 of the k-th 32-byte column step
  const int mi = lane >> 3, lr = lane & 7;
  const int rl = (mi >> 1) * 8 + lr;
  const uint32_t wring_s = smem_u32(wring);
  auto sw = [&](int chunk) {  // byte offset of 16-byte chunk `chunk` (0..15) of row rl, slabbed + swizzled
    return (uint32_t)((chunk >> 3) * SLAB + rl * 128 + (((chunk & 7) ^ lr) << 4));
  };
  for (int j = 0; j < n_mine; ++j) {
    const int st = j % nd;
    mbar_wait(&wb[st], (uint32_t)((j / nd) & 1));
    const uint32_t ra = s_rows[warp * D + st][0], rc = s_rows[warp * D + st][1];
    int rmax = 0;
#pragma unroll
    for (int h = 0; h < G; ++h) rmax = max(rmax, entry_rows(ra, rc, h));
    const int myrows = g < G ? entry_rows(ra, rc, g) : 0;
    if (rmax > 0) {
      const uint32_t kb = wring_s + (uint32_t)(st * STAGE);
      const uint32_t vb = kb + 2 * SLAB;
      float s[4][4];
#pragma unroll
      for (int c = 0; c < 4; ++c) s[c][0] = s[c][1] = s[c][2] = s[c][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t bk[4];
        ldsm_x4(bk, kb + sw(2 * ks + (mi & 1)));
        mma_rows8(s[(ks & 1) * 2 + 0], qa[ks][0], qa[ks][1], bk[0], bk[1]);
        mma_rows8(s[(ks & 1) * 2 + 1], qa[ks][0], qa[ks][1], bk[2], bk[3]);
      }
      const int k0 = 2 * t;
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
        const float c0 = __shfl_sync(0xffffffffu, corr, 8 * t);
        const float c1 = __shfl_sync(0xffffffffu, corr, 8 * t + 4);
#pragma unroll
        for (int j2 = 0; j2 < 8; ++j2) {
          acc[j2][0] *= c0;
          acc[j2][1] *= c1;
          acc[j2][2] *= c0;
          acc[j2][3] *= c1;
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
      for (int j2 = 0; j2 < 8; ++j2) {
        uint32_t av[4];
        ldsm_x4_t(av, vb + sw(2 * j2 + (mi & 1)));
        const uint32_t a4[4] = {av[0], av[1], av[2], av[3]};
        mma_16816(acc[j2], a4, bh0, bh1);
        mma_16816(acc[j2], a4, bl0, bl1);
      }
    }
    __syncwarp();  // the stage is free
    issue(j + nd);
  }
  float* sc = reinterpret_cast<float*>(ring);
  named_bar_sync(1, NW * 32);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int h = 2 * t + e;
    if (h < G) {
      float* row = sc + (warp * G + h) * kScStride + g;
#pragma unroll
      for (int j2 = 0; j2 < 8; ++j2) {
        row[16 * j2] = acc[j2][e];
        row[16 * j2 + 8] = acc[j2][2 + e];
      }
    }
  }
  if (g < G && t == 0) {
    sc[(warp * G + g) * kScStride + kD] = m_run;
    sc[(warp * G + g) * kScStride + kD + 1] = l_run;
  }
}

// ---------------------------------------------------------------------------
// Merge the NW warps' states in sc (fixed order) into this split's (o, lse);
// with n_eff > 1 write the split partial, take the (b, KV head) ticket and,
// in the last CTA, merge the n_eff splits in split order.  All NW warps of the
// CTA call this (named barrier 1 over NW * 32 threads).  s_last: a __shared__ int.
// ---------------------------------------------------------------------------
template <int G, int NW>
DSK_DEVICE void attn_merge_out(float* sc, int* s_last, int b, int hk, int Hq, int split, int n_eff,
                               int n_split, size_t bh, float* __restrict__ part_o,
                               float* __restrict__ part_lse, int* __restrict__ counters,
                               float* __restrict__ o, float* __restrict__ lse) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
    *s_last = (old == n_eff - 1);
  }
  named_bar_sync(1, NW * 32);
  if (!*s_last) return;
  // Last CTA of (b, KV head): LSE merge of the n_eff splits.  R = NW / G
  // warps share a head: every warp reads all split lse values (lanes hold
  // them, n_eff <= 64) and forms the weights by warp reductions (fixed
  // butterfly order); warp part r sums w_s o_s over the splits s = r (mod R)
  // with all its loads in flight at once (n_eff / R <= 16 per lane); the R
  // parts are added in part order through shared memory.
  constexpr int R = NW >= G ? NW / G : 1;
  float* mrg = sc;  // [G][R][kD]
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
  if (threadIdx.x == 0) counters[bh] = 0;
}

}  // namespace dsk
