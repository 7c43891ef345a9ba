// Decode-step kernels of the DynSplit-KV hot path (sm_100a).
//   a5  k_score_blocks      V2F block score, sum_j max(q_j kmax_j, q_j kmin_j)
//   a6  k_select_threshold  budgeted top-k via block-to-token mapping
//       k_select_union      per-head selections -> GQA-union page worklist
//   (a7/a8 attention kernels live in attn_kernels.cu)

//       k_merge_partials    standalone LSE merge (cross-GPU sequence split)
#include "common.cuh"
#include "kernels.h"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <math_constants.h>
#include <stdlib.h>

namespace dsk {

// ============================================================================
// a5: block scores (k_score_blocks below: grid, staging).  A half-warp owns one
// block digest (512 B bf16: kmax row + kmin row); lane hl owns dims
// [8hl, 8hl+8).  max(q_j kmax_j, q_j kmin_j) = q_j * (q_j >= 0 ? kmax_j : kmin_j)
// because kmax >= kmin element-wise; for bf16 the per-head choice is one
// byte-permute per bf16 pair (signs of q fixed per lane) and the product is
// an exact bf16 x bf16 FHFMA into fp32.  The per-block reduction order (8
// sequential terms, then the 16-lane multi-head butterfly of
// halfwarp_reduce_heads) is fixed and independent of the grid, so every
// launch configuration (and every sequence-split rank) yields identical fp32
// scores.
// ============================================================================
template <typename T> struct DigestDot;
template <> struct DigestDot<bf16> {
  struct Q {
    uint32_t w[4], sel[4];
  };
  struct K {
    uint4 mx, mn;
  };
  static DSK_DEVICE void load_q(const bf16* p, Q& q) {
    const uint4 u = __ldca(reinterpret_cast<const uint4*>(p));  // may come from the PDL primary
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      q.w[i] = w[i];
      q.sel[i] = ((w[i] & 0x8000u) ? 0x0054u : 0x0010u) | ((w[i] & 0x80000000u) ? 0x7600u : 0x3200u);
    }
  }
  static DSK_DEVICE void load_k(const bf16* p, K& k) {
    k.mx = __ldg(reinterpret_cast<const uint4*>(p));
    k.mn = __ldg(reinterpret_cast<const uint4*>(p + kD));
  }
  static DSK_DEVICE void load_k_smem(const bf16* p, K& k) {
    k.mx = *reinterpret_cast<const uint4*>(p);
    k.mn = *reinterpret_cast<const uint4*>(p + kD);
  }
  static DSK_DEVICE void zero_k(K& k) { k.mx = k.mn = make_uint4(0, 0, 0, 0); }
  static DSK_DEVICE float dot_mean(const Q& q, const float (&m)[8]) {  // 8 sequential FFMA
    float a = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a = fmaf(bf_lo(q.w[i]), m[2 * i], a);
      a = fmaf(bf_hi(q.w[i]), m[2 * i + 1], a);
    }
    return a;
  }
  static DSK_DEVICE float dot(const Q& q, const K& k) {
    const uint32_t mx[4] = {k.mx.x, k.mx.y, k.mx.z, k.mx.w};
    const uint32_t mn[4] = {k.mn.x, k.mn.y, k.mn.z, k.mn.w};
    float a = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t s = __byte_perm(mx[i], mn[i], q.sel[i]);
      unsigned short ql, qh, sl, sh;
      split_bf16x2(q.w[i], ql, qh);
      split_bf16x2(s, sl, sh);
      a = fma_bf16(ql, sl, a);
      a = fma_bf16(qh, sh, a);
    }
    return a;
  }
};
template <> struct DigestDot<float> {
  struct Q {
    float v[8];
  };
  struct K {
    float mx[8], mn[8];
  };
  static DSK_DEVICE void load_q(const float* p, Q& q) { Vec<float>::load8(p, q.v); }
  static DSK_DEVICE void load_k(const float* p, K& k) {
    Vec<float>::load8_nc(p, k.mx);
    Vec<float>::load8_nc(p + kD, k.mn);
  }
  static DSK_DEVICE void load_k_smem(const float* p, K& k) {
    Vec<float>::load8(p, k.mx);
    Vec<float>::load8(p + kD, k.mn);
  }
  static DSK_DEVICE void zero_k(K& k) {
#pragma unroll
    for (int j = 0; j < 8; ++j) k.mx[j] = k.mn[j] = 0.f;
  }
  static DSK_DEVICE float dot_mean(const Q& q, const float (&m)[8]) {
    float a = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) a = fmaf(q.v[j], m[j], a);
    return a;
  }
  static DSK_DEVICE float dot(const Q& q, const K& k) {
    float a = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) a = fmaf(q.v[j], q.v[j] >= 0.f ? k.mx[j] : k.mn[j], a);
    return a;
  }
};

// Sum G per-lane partials over the 16 lanes of a half-warp with G - 1 + log2(16 / G)
// shuffles instead of 4 G: at offsets 8, 4, ... while a lane still holds more
// than one head, the lower lane of each pair keeps the first half of its
// heads and the upper lane the second half, each adding its partner's copy
// of what it keeps; then a plain xor tree over the remaining offsets.  The
// order depends only on the lane (dimension) positions, so the scores stay
// grid-independent.  Returns the sum of head `head`; every lane with
// (hl & (16 / G - 1)) == 0 holds a distinct head.
template <int G>
DSK_DEVICE float halfwarp_reduce_heads(const float (&a)[G], int hl, int& head) {
  static_assert(G >= 1 && G <= 16 && (G & (G - 1)) == 0, "G must be a power of two <= 16");
  float v[G];
#pragma unroll
  for (int g = 0; g < G; ++g) v[g] = a[g];
  head = 0;
  int o = 8;
#pragma unroll
  for (int c = G; c > 1; c >>= 1, o >>= 1) {
    const bool up = (hl & o) != 0;
#pragma unroll
    for (int g = 0; g < c / 2; ++g) {
      const float keep = up ? v[g + c / 2] : v[g];
      const float send = up ? v[g] : v[g + c / 2];
      v[g] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
    head += up ? c / 2 : 0;
  }
#pragma unroll
  for (; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  return v[0];
}

// Optional per-CTA phase timestamps (debug only; dynsplit_debug_score_timer).
__device__ unsigned long long* g_score_dbg = nullptr;
DSK_DEVICE void sstamp(int k) {
#ifdef DSK_DEBUG
  if (g_score_dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const size_t cta = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    g_score_dbg[cta * 4 + k] = t;
  }
#else
  (void)k;
#endif
}

// grid (chunks, Hkv, B), 512 threads, one CTA per SM on chunks * B * Hkv SMs
// (the launcher leaves enough SMs free for the select kernel's CTAs, which
// can then become resident -- and load their plan -- while this one runs).
// Before the PDL wait the CTA's whole digest range (resident data, <= `cap`
// blocks) is copied into shared memory with TMA bulk copies, so its HBM read
// overlaps the preceding kernel's tail; after the wait only q is loaded.
template <typename T, int G>
__global__ void __launch_bounds__(512, 1) k_score_blocks(const T* __restrict__ q,
                                                         const T* __restrict__ dig,
                                                         const int32_t* __restrict__ n_blocks,
                                                         float* __restrict__ scores, int Hq, int Hkv,
                                                         int maxb, int cap, int mean_mode) {
  using DD = DigestDot<T>;
  constexpr int RB = 2 * kD * (int)sizeof(T);  // digest bytes per block (kmax, kmin)
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  const int hk = blockIdx.y, b = blockIdx.z;
  const int nb = n_blocks[b];
  const int per = (nb + gridDim.x - 1) / gridDim.x;
  const int lo = blockIdx.x * per;
  const int hi = min(nb, lo + per);
  const int n = max(hi - lo, 0);
  const int pre = min(n, cap);  // blocks staged in shared memory
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane >> 4, hl = lane & 15;
  sstamp(0);

  const T* dbase = dig + ((size_t)b * Hkv + hk) * (size_t)maxb * 2 * kD;
  float* sbase = scores + ((size_t)b * Hq + hk * G) * maxb;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    if (pre) {
      const uint32_t bytes = (uint32_t)pre * RB;
      mbar_arrive_expect_tx(&bar, bytes);
      const unsigned char* src = reinterpret_cast<const unsigned char*>(dbase + (size_t)lo * 2 * kD);
      for (uint32_t off = 0; off < bytes; off += 32768u)
        bulk_g2s(smem + off, src + off, min(32768u, bytes - off), &bar, policy_evict_first());
    } else {
      mbar_arrive(&bar);
    }
  }
  // q (and the scores buffer) belong to the step -> after the PDL wait
  pdl_trigger();
  pdl_wait();
  sstamp(1);
  typename DD::Q qv[G];
#pragma unroll
  for (int g = 0; g < G; ++g) DD::load_q(q + ((size_t)b * Hq + hk * G + g) * kD + hl * 8, qv[g]);
  __syncthreads();  // the barrier's initialisation is visible
  mbar_wait(&bar, 0);
  __syncwarp();
  sstamp(3);

  // a half-warp per block; lane hl owns dims [8 hl, 8 hl + 8) of kmax / kmin.
  // Two passes per iteration (blocks base + half and base + 32 + half): two
  // independent load -> dot -> butterfly chains in flight per warp.
  const T* sd = reinterpret_cast<const T*>(smem);
  auto block_dots = [&](int i, float (&acc)[G]) {
    if (mean_mode) {
      // NEXT-2 mean pooling: q . mean, the fp32 mean row in the block's digest slot
      float mrow[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (i < n) {
        const float* mp = i < pre ? reinterpret_cast<const float*>(sd + (size_t)i * 2 * kD) + hl * 8
                                  : reinterpret_cast<const float*>(dbase + (size_t)(lo + i) * 2 * kD) + hl * 8;
        const float4 a = reinterpret_cast<const float4*>(mp)[0], c = reinterpret_cast<const float4*>(mp)[1];
        mrow[0] = a.x; mrow[1] = a.y; mrow[2] = a.z; mrow[3] = a.w;
        mrow[4] = c.x; mrow[5] = c.y; mrow[6] = c.z; mrow[7] = c.w;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) acc[g] = DD::dot_mean(qv[g], mrow);
    } else {
      typename DD::K kb;
      if (i < pre) DD::load_k_smem(sd + (size_t)i * 2 * kD + hl * 8, kb);
      else if (i < n) DD::load_k(dbase + (size_t)(lo + i) * 2 * kD + hl * 8, kb);
      else DD::zero_k(kb);
#pragma unroll
      for (int g = 0; g < G; ++g) acc[g] = DD::dot(qv[g], kb);
    }
  };
  for (int base = warp * 2; base < n; base += 64) {  // warp-uniform trip count
    const int i0 = base + half, i1 = base + 32 + half;
    float a0[G], a1[G];
    block_dots(i0, a0);
    block_dots(i1, a1);
    int h0, h1;
    const float r0 = halfwarp_reduce_heads<G>(a0, hl, h0);
    const float r1 = halfwarp_reduce_heads<G>(a1, hl, h1);
    if ((hl & (16 / G - 1)) == 0) {
      if (i0 < n) sbase[(size_t)h0 * maxb + lo + i0] = r0;
      if (i1 < n) sbase[(size_t)h1 * maxb + lo + i1] = r1;
    }
  }
  sstamp(2);
}

// Test hook: 1 forces the CUDA-core k_score_blocks for bf16 too (parity of the
// two a5 kernels); initial value from DYNSPLIT_A5_CUDA_CORE.
static volatile bool g_score_cuda_core = getenv("DYNSPLIT_A5_CUDA_CORE") != nullptr;

// ============================================================================
// a5 on the tensor cores (bf16 digests, min/max mode).  The block score is a
// 256-long dot product:  sum_j max(q_j kmax_j, q_j kmin_j)
//   = sum_j max(q_j, 0) kmax_j + sum_j min(q_j, 0) kmin_j            (kmax >= kmin)
//   = A_h . B_blk,  A_h = [q+ | q-] (bf16, exact),  B_blk = [kmax | kmin]
// i.e. exactly the digest row.  One m16n8k16 tile = G (<= 8) heads x 8 blocks
// x 16 dims; 16 k-steps per 8 blocks (bf16 x bf16 products exact, fp32
// accumulation in a fixed k order: a block's score does not depend on the CTA,
// so sequence-split ranks still agree).  The per-block half-warp dot products
// of k_score_blocks issue ~10x more instructions; this is the same HBM read.
// Staging (before the PDL wait, under the preceding kernel): TMA tensor copies
// of 64-dim x 32-row boxes with the 128-byte hardware swizzle into four
// 64-dim slabs, so the ldmatrix row reads are conflict-free; a CTA's range is
// a multiple of 32 rows (whole boxes).  A range longer than the stage is
// processed in rounds.
// ============================================================================
constexpr int kA5BoxRows = 32;  // rows per TMA box
constexpr int kA5SlabRowB = 128;  // bytes per row of one 64-dim slab


template <int G>
__global__ void __launch_bounds__(512, 1) k_score_blocks_tc(const __grid_constant__ CUtensorMap tmD,
                                                            const bf16* __restrict__ q,
                                                            const int32_t* __restrict__ n_blocks,
                                                            float* __restrict__ scores, int Hq, int Hkv,
                                                            int maxb, int cap) {
  static_assert(G >= 1 && G <= 8, "G heads per KV head <= 8 (A rows 0..7)");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  // 1024-byte aligned slabs (the swizzle atoms are address-based)
  const uint32_t raw_s = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + (((raw_s + 1023u) & ~1023u) - raw_s);
  const size_t slab = (size_t)cap * kA5SlabRowB;  // one 64-dim slab of `cap` rows
  const int hk = blockIdx.y, b = blockIdx.z;
  const int nb = n_blocks[b];
  const int per = (((nb + gridDim.x - 1) / gridDim.x) + kA5BoxRows - 1) & ~(kA5BoxRows - 1);
  const int lo = blockIdx.x * per;
  const int hi = min(nb, lo + per);
  const int n = max(hi - lo, 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  sstamp(0);
  const int row0 = (b * Hkv + hk) * maxb + lo;  // tensor-map row of this CTA's first block
  float* sbase = scores + ((size_t)b * Hq + hk * G) * maxb;
  auto stage = [&](int r0, int cnt) {  // rows r0 .. r0 + cnt of the range -> smem rows 0 ..
    if (threadIdx.x == 0) {
      const int nbox = (cnt + kA5BoxRows - 1) / kA5BoxRows;
      mbar_arrive_expect_tx(&bar, (uint32_t)(nbox * 4 * kA5BoxRows * kA5SlabRowB));
      for (int j = 0; j < nbox; ++j)
#pragma unroll
        for (int sl = 0; sl < 4; ++sl)
          tma_load_2d(smem + sl * slab + (size_t)j * kA5BoxRows * kA5SlabRowB, &tmD, sl * 64,
                      row0 + r0 + j * kA5BoxRows, &bar);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  const int first = min(n, cap);
  if (first > 0) stage(0, first);  // resident data: overlaps the preceding kernel under PDL
  pdl_trigger();
  pdl_wait();
  sstamp(1);
  // A fragments of lane (g = lane / 4, t = lane % 4): head g's [q+ | q-] at
  // k = 16 ks + 2t (+1) and 16 ks + 2t + 8 (+9); heads >= G are zero rows
  const int g = lane >> 2, t = lane & 3;
  uint32_t a0[16], a2[16];
  {
    uint32_t w0[8], w2[8];  // q_g[16 i + 2t .. +1], q_g[16 i + 2t + 8 .. +9], i < 8
#pragma unroll
    for (int i = 0; i < 8; ++i) w0[i] = w2[i] = 0u;
    if (g < G) {
      const uint32_t* qg = reinterpret_cast<const uint32_t*>(q + ((size_t)b * Hq + hk * G + g) * kD);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        w0[i] = __ldca(qg + 8 * i + t);  // weak coherent loads: q may come from the PDL primary
        w2[i] = __ldca(qg + 8 * i + t + 4);
      }
    }
    const __nv_bfloat162 z2 = __floats2bfloat162_rn(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const __nv_bfloat162 x0 = *reinterpret_cast<const __nv_bfloat162*>(&w0[i]);
      const __nv_bfloat162 x2 = *reinterpret_cast<const __nv_bfloat162*>(&w2[i]);
      const __nv_bfloat162 p0 = __hmax2(x0, z2), p2 = __hmax2(x2, z2);  // q+ (exact)
      const __nv_bfloat162 m0 = __hmin2(x0, z2), m2 = __hmin2(x2, z2);  // q- (exact)
      a0[i] = *reinterpret_cast<const uint32_t*>(&p0);
      a2[i] = *reinterpret_cast<const uint32_t*>(&p2);
      a0[8 + i] = *reinterpret_cast<const uint32_t*>(&m0);
      a2[8 + i] = *reinterpret_cast<const uint32_t*>(&m2);
    }
  }
  __syncthreads();  // the barrier's initialisation is visible to every warp
  // ldmatrix.x4: lane l addresses row (l % 8) of the 8-block group, 16-byte
  // chunk (l / 8) of the 32-dim window (kk); slab = kk / 2, chunk in slab =
  // 4 (kk % 2) + l / 8, swizzled with the row within its 8-row atom
  const int lr = lane & 7, lc = lane >> 3;
  const uint32_t sbase_u = smem_u32(smem);
  uint32_t phase = 0;
  for (int r0 = 0; r0 < n; r0 += cap, phase ^= 1u) {
    const int cnt = min(cap, n - r0);
    if (r0) {
      __syncthreads();  // the previous round's rows are consumed
      stage(r0, cnt);
    }
    mbar_wait(&bar, phase);
    if (r0 == 0) sstamp(3);
    for (int grp = warp; grp * 8 < cnt; grp += 16) {
      float c[4] = {0.f, 0.f, 0.f, 0.f};
      const int r = grp * 8 + lr;
      const uint32_t rowa = sbase_u + (uint32_t)(r * kA5SlabRowB);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {  // two k-steps (32 dims) per ldmatrix.x4
        const uint32_t chunk = (uint32_t)((((kk & 1) << 2) | lc) ^ (r & 7));
        uint32_t bk[4];
        ldsm_x4(bk, rowa + (uint32_t)((kk >> 1) * slab) + (chunk << 4));
        mma_rows8(c, a0[2 * kk], a2[2 * kk], bk[0], bk[1]);
        mma_rows8(c, a0[2 * kk + 1], a2[2 * kk + 1], bk[2], bk[3]);
      }
      // c0, c1: head g, blocks grp * 8 + 2t, + 1 (rows 8..15 are zero)
      const int i0 = r0 + grp * 8 + 2 * t;
      if (g < G) {
        if (i0 < n) sbase[(size_t)g * maxb + lo + i0] = c[0];
        if (i0 + 1 < n) sbase[(size_t)g * maxb + lo + i0 + 1] = c[1];
      }
    }
  }
  sstamp(2);
}

}  // namespace dsk
extern "C" int dynsplit_debug_a5_cuda_core(int on) {
  dsk::g_score_cuda_core = on != 0;
  return 0;
}
extern "C" int dynsplit_debug_score_timer(void* dev_ptr) {
  return (int)cudaMemcpyToSymbol(dsk::g_score_dbg, &dev_ptr, sizeof(void*));
}
namespace dsk {

// ============================================================================
// a8 standalone: merge n_parts (o, lse) partials, fixed part order.
// grid (rows), 128 threads.
// ============================================================================
__global__ void k_merge_partials(const float* __restrict__ o_parts, const float* __restrict__ lse_parts,
                                 int n_parts, int rows, int d, float* __restrict__ o,
                                 float* __restrict__ lse) {
  const int r = blockIdx.x;
  float M = -CUDART_INF_F;
  for (int s = 0; s < n_parts; ++s) M = fmaxf(M, lse_parts[(size_t)s * rows + r]);
  float L = -CUDART_INF_F;
  if (M != -CUDART_INF_F) {
    float sum = 0.f;
    for (int s = 0; s < n_parts; ++s) sum += expf(lse_parts[(size_t)s * rows + r] - M);
    L = M + logf(sum);
  }
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float acc = 0.f;
    if (L != -CUDART_INF_F)
      for (int s = 0; s < n_parts; ++s)
        acc += expf(lse_parts[(size_t)s * rows + r] - L) * o_parts[((size_t)s * rows + r) * d + j];
    o[(size_t)r * d + j] = acc;
  }
  if (threadIdx.x == 0) lse[r] = L;
}

// ============================================================================
// host launchers
// ============================================================================
// Chunks per (b, KV head): the SMs left after reserving one per select CTA
// (B * Hq of them, at most a quarter of the GPU); shared-memory staging of up
// to 192 KiB of digests per CTA (blocks beyond it are read from HBM directly).
template <typename T>
static cudaError_t score_blocks_t(int G, const void* q, const void* dig, const int32_t* nb,
                                  float* scores, int B, int Hq, int Hkv, int maxb, int nb_hint,
                                  int mean_mode, cudaStream_t st) {
  const int sms = num_sms();
  const int reserve = min(B * Hq, sms / 4);
  const int rb = 2 * kD * (int)sizeof(T);
  const int cap_max = (192 * 1024) / rb;  // blocks one CTA can stage in shared memory
  // One wave on the SMs not reserved for the select CTAs when that covers the
  // expected blocks (B = 1); otherwise enough CTAs that every CTA's range fits
  // its shared-memory stage (several waves, still one HBM pass: the blocks
  // past the stage would be loaded by dependent global loads).
  const int base = (sms - reserve) / max(1, B * Hkv);
  const int need = (min(nb_hint, maxb) + cap_max - 1) / cap_max;
  const int chunks = max(1, min(max(base, need), (maxb + 31) / 32));
  const int cap = min((maxb + chunks - 1) / chunks, cap_max);
  const size_t smem = (size_t)cap * rb;
  dim3 grid(chunks, Hkv, B);
  if constexpr (sizeof(T) == 2) {
    if (!mean_mode && G <= 8 && !g_score_cuda_core) {
      // tensor-core path: whole 32-row TMA boxes per CTA (device: per rounded up to 32)
      const auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
      if (!encode) return cudaErrorNotSupported;
      const int rows_hint = (min(nb_hint, maxb) + chunks - 1) / chunks;
      const int cap_tc = min(((rows_hint + kA5BoxRows - 1) / kA5BoxRows) * kA5BoxRows, 384);
      const size_t smem_tc = (size_t)cap_tc * 4 * kA5SlabRowB + 1024;
      // digests [B * Hkv * maxb rows][256] bf16 -> boxes of 64 dims x 32 rows, 128-byte swizzle
      CUtensorMap tm;
      const cuuint64_t dims[2] = {(cuuint64_t)2 * kD, (cuuint64_t)B * Hkv * maxb};
      const cuuint64_t strides[1] = {(cuuint64_t)2 * kD * 2};
      const cuuint32_t box[2] = {64, (cuuint32_t)kA5BoxRows};
      const cuuint32_t es[2] = {1, 1};
      if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(dig), dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
      const bf16* qq = static_cast<const bf16*>(q);
#define DSK_SCT(GG)                                                                                  \
  {                                                                                                  \
    allow_max_dyn_smem(k_score_blocks_tc<GG>);                                                       \
    launch_ex(k_score_blocks_tc<GG>, grid, 512, smem_tc, st, 1, tm, qq, nb, scores, Hq, Hkv, maxb,    \
              cap_tc);                                                                               \
    return post_launch("k_score_blocks_tc", st);                                                     \
  }
      switch (G) {
        case 1: DSK_SCT(1)
        case 2: DSK_SCT(2)
        case 4: DSK_SCT(4)
        case 8: DSK_SCT(8)
        default: break;
      }
#undef DSK_SCT
    }
  }
  const T* qq = static_cast<const T*>(q);
  const T* dd = static_cast<const T*>(dig);
#define DSK_SC(GG)                                                                                   \
  {                                                                                                  \
    allow_max_dyn_smem(k_score_blocks<T, GG>);                                                       \
    launch_ex(k_score_blocks<T, GG>, grid, 512, smem, st, 1, qq, dd, nb, scores, Hq, Hkv, maxb, cap,   \
              mean_mode);                                                                            \
    break;                                                                                           \
  }
  switch (G) {
    case 1: DSK_SC(1)
    case 2: DSK_SC(2)
    case 4: DSK_SC(4)
    case 8: DSK_SC(8)
    default: return cudaErrorInvalidValue;
  }
#undef DSK_SC
  return post_launch(__func__, st);
}

cudaError_t launch_score_blocks(int dtype, int G, const void* q, const void* dig, const int32_t* nb,
                                float* scores, int B, int Hq, int Hkv, int maxb, int nb_hint,
                                int mean_mode, cudaStream_t st) {
  if (dtype == 0)
    return score_blocks_t<bf16>(G, q, dig, nb, scores, B, Hq, Hkv, maxb, nb_hint, mean_mode, st);
  return score_blocks_t<float>(G, q, dig, nb, scores, B, Hq, Hkv, maxb, nb_hint, mean_mode, st);
}

cudaError_t launch_merge(const float* o_parts, const float* lse_parts, int n_parts, int rows, int d,
                         float* o, float* lse, cudaStream_t st) {
  k_merge_partials<<<rows, 128, 0, st>>>(o_parts, lse_parts, n_parts, rows, d, o, lse);
  return post_launch(__func__, st);
}

}  // namespace dsk
