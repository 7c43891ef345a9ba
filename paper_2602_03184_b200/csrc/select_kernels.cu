// Decode row a6: budgeted top-k through block-to-token mapping (V2F,
// P:257-264; KV Selection Step 1) for every query head, plus the
// GQA-union page worklist consumed by the attention kernel.
//
// Order of blocks for one head: (score desc, block index asc).  Blocks are
// taken whole while the budget lasts; the block that reaches it ("marginal")
// keeps its first `need` tokens (identical to the per-token stable sort of
// the oracle).
//
// One thread-block cluster of G CTAs (512 threads each) per (b, KV head);
// CTA c of the cluster owns query head hk*G + c:
//   1. block lengths -> smem (all blocks), total;
//   2. the head's marginal block, exactly:
//        - bucket the live scores into 2048 buckets of [min, max] (a monotone
//          map), length-weighted smem histogram, suffix scan -> the bucket
//          where the budget is reached;
//        - if it holds <= 512 blocks: bitonic sort of (key, ~index) and a
//          prefix walk; otherwise narrow to that bucket and repeat; a bucket
//          of identical scores is resolved in index order;
//   3. cluster barrier; every CTA reads the G heads' (marginal, keep, key)
//      from its peers' shared memory (DSMEM) and builds the union for its
//      1/G of the blocks: head h takes blk iff all_fit || key > T ||
//      (key == T && blk <= marginal); per block the union page count and the
//      G-bit mask; block-wide scan; cluster barrier; offsets of the earlier
//      ranks' totals via DSMEM; write the worklist entries (page, per-head
//      leading rows) in ascending block order and every head's ascending
//      sel_blocks.
#include "common.cuh"
#include "kernels.h"

#include <cooperative_groups.h>
#include <math_constants.h>

namespace cg = cooperative_groups;

namespace dsk {

constexpr int kSelNT = 512;
constexpr int kSelW = kSelNT / 32;
constexpr int kBkt = 2048;
constexpr int kBPT = kBkt / kSelNT;
constexpr int kCap = 512;

// Optional phase timestamps (debug only; set by dynsplit_debug_select_timer).
__device__ unsigned long long* g_sel_dbg = nullptr;
DSK_DEVICE void stamp(int k) {
#ifdef DSK_DEBUG
  if (g_sel_dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_sel_dbg[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + k] = t;
  }
#else
  (void)k;
#endif
}

DSK_DEVICE float key_to_float(uint32_t k) {
  const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}
DSK_DEVICE int bucket_of(uint32_t k, float mn, float inv) {
  return min(max((int)((key_to_float(k) - mn) * inv), 0), kBkt - 1);
}

// dynamic smem: K[mb4] u32 | K0[mb4] u32 | CA[kCap] u64 | HI[kBkt] u32 | slen[mb4] u16 | sumk[rg4] u16
static size_t select_smem_bytes(int maxb, int G) {
  const size_t mb4 = ((size_t)maxb + 3) & ~(size_t)3;
  const size_t rg4 = ((size_t)(maxb + G - 1) / G + 3) & ~(size_t)3;
  return 2 * mb4 * 4 + (size_t)kCap * 8 + (size_t)kBkt * 4 + mb4 * 2 + rg4 * 2;
}

// block-wide inclusive scan of one int; returns (inclusive prefix, total)
DSK_DEVICE int2 cta_scan(int v, int* sm /* kSelW + 1 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int inc = warp_incl_scan(v);
  if (lane == 31) sm[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int x = lane < kSelW ? sm[lane] : 0;
    const int s = warp_incl_scan(x);
    if (lane < kSelW) sm[lane] = s - x;
    if (lane == kSelW - 1) sm[kSelW] = s;
  }
  __syncthreads();
  const int2 r = make_int2(sm[warp] + inc, sm[kSelW]);
  __syncthreads();
  return r;
}

template <int G>
__global__ void __launch_bounds__(kSelNT, 1) k_select(
    const float* __restrict__ scores, const int32_t* __restrict__ block_starts,
    const int32_t* __restrict__ n_blocks, const int32_t* __restrict__ page_first, int Hq, int Hkv,
    int maxb, int max_sel, int max_wl, int Pshift, int budget, int blk_lo, int blk_hi,
    int32_t* __restrict__ sel_blocks, int32_t* __restrict__ n_sel, int32_t* __restrict__ marg_out,
    int32_t* __restrict__ keep_out, int32_t* __restrict__ wl_count, WLEntry* __restrict__ wl) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem[];
  const int mb4 = (maxb + 3) & ~3;
  uint32_t* K = reinterpret_cast<uint32_t*>(smem);
  uint32_t* K0 = K + mb4;  // immutable copy of the keys (read by peers in the union)
  uint64_t* CA = reinterpret_cast<uint64_t*>(K0 + mb4);
  uint32_t* HI = reinterpret_cast<uint32_t*>(CA + kCap);
  uint16_t* slen = reinterpret_cast<uint16_t*>(HI + kBkt);
  uint16_t* sumk = slen + mb4;

  __shared__ float red_f[2][kSelW];
  __shared__ int red_i[kSelW + 1];
  __shared__ int s_info[4];       // marginal, keep, key, all_fit of this CTA's head
  __shared__ int s_tot[G + 1];    // this CTA's union-range totals (per head, pages)
  __shared__ int s_bnd, s_need, s_nc;
  __shared__ float s_mn, s_mx;

  const int c = (int)cluster.block_rank();  // == blockIdx.x % G
  const int hk = blockIdx.x / G, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = 1 << Pshift;
  const int nb = n_blocks[b];
  // every block of the sequence competes; worklist entries are emitted only
  // for blocks in the output range [olo, ohi) (a sequence-split shard)
  const int lo = 0, hi = nb;
  const int olo = min(max(blk_lo, 0), nb), ohi = max(min(blk_hi, nb), olo);
  const int nr = max(hi - lo, 0);
  const int32_t* bs = block_starts + (size_t)b * (maxb + 1);
  const int32_t* pf = page_first + (size_t)b * (maxb + 1);
  const float* sc0 = scores + ((size_t)b * Hq + hk * G) * maxb;
  const float* sc = sc0 + (size_t)c * maxb + lo;

  stamp(0);
  // ---- 1. lengths (the resident plan), then -- after the preceding kernel
  //         (PDL) -- the keys of this CTA's head, total
  int t = 0;
  for (int i = tid; i < nr; i += kSelNT) {
    const int len = bs[lo + i + 1] - bs[lo + i];
    slen[i] = (uint16_t)len;
    t += len;
  }
  stamp(1);
  pdl_trigger();
  pdl_wait();
  stamp(2);
  for (int i = tid; i < nr; i += kSelNT) K[i] = K0[i] = float_key(sc[i]);
  const int total = cta_scan(t, red_i).y;
  stamp(3);

  // ---- 2. threshold of head c
  if (total <= budget) {
    if (tid == 0) {
      s_info[0] = -1;
      s_info[1] = 0;
      s_info[2] = 0;
      s_info[3] = 1;
    }
  } else {
    int need = budget;
    for (;;) {
      float mn = CUDART_INF_F, mx = -CUDART_INF_F;
      for (int i = tid; i < nr; i += kSelNT) {
        const uint32_t k = K[i];
        if (k) {
          const float f = key_to_float(k);
          mn = fminf(mn, f);
          mx = fmaxf(mx, f);
        }
      }
      mn = -warp_max(-mn);
      mx = warp_max(mx);
      if (lane == 0) {
        red_f[0][warp] = mn;
        red_f[1][warp] = mx;
      }
      for (int i = tid; i < kBkt; i += kSelNT) HI[i] = 0;
      __syncthreads();
      if (warp == 0) {
        float a = lane < kSelW ? red_f[0][lane] : CUDART_INF_F;
        float x = lane < kSelW ? red_f[1][lane] : -CUDART_INF_F;
        a = -warp_max(-a);
        x = warp_max(x);
        if (lane == 0) {
          s_mn = a;
          s_mx = x;
          s_nc = 0;
        }
      }
      __syncthreads();
      mn = s_mn;
      mx = s_mx;
      if (!(mx > mn)) {
        // all live scores equal: they are ordered by block index
        int carry = 0;
        for (int c0 = 0; c0 < nr && carry < need; c0 += kSelNT) {
          const int i = c0 + tid;
          const int v = (i < nr && K[i]) ? (int)slen[i] : 0;
          const int2 pre = cta_scan(v, red_i);
          const int incl = carry + pre.x;
          if (v > 0 && incl >= need && incl - v < need) {
            s_info[0] = lo + i;
            s_info[1] = need - (incl - v);
            s_info[2] = (int)K[i];
            s_info[3] = 0;
          }
          carry += pre.y;
        }
        break;
      }
      const float inv = (float)kBkt / (mx - mn);
      for (int i = tid; i < nr; i += kSelNT) {
        const uint32_t k = K[i];
        if (k) atomicAdd(&HI[bucket_of(k, mn, inv)], (uint32_t)slen[i]);
      }
      __syncthreads();
      {  // suffix scan: thread tid owns buckets kBkt-1-tid*kBPT downwards
        const int j0 = kBkt - 1 - tid * kBPT;
        int loc = 0;
#pragma unroll
        for (int k = 0; k < kBPT; ++k) loc += (int)HI[j0 - k];
        int above = cta_scan(loc, red_i).x - loc;
#pragma unroll
        for (int k = 0; k < kBPT; ++k) {
          const int hb = (int)HI[j0 - k];
          if (above < need && above + hb >= need) {
            s_bnd = j0 - k;
            s_need = need - above;
          }
          above += hb;
        }
      }
      __syncthreads();
      const int bnd = s_bnd;
      need = s_need;
      for (int i = tid; i < nr; i += kSelNT) {
        const uint32_t k = K[i];
        if (k) {
          if (bucket_of(k, mn, inv) == bnd) {
            const int p = atomicAdd(&s_nc, 1);
            if (p < kCap) CA[p] = ((uint64_t)k << 32) | (uint64_t)(0xffffffffu - (uint32_t)(lo + i));
          } else {
            K[i] = 0;  // above (already in need) or below the boundary: no longer live
          }
        }
      }
      __syncthreads();
      const int nc = s_nc;
      if (nc > kCap) continue;  // narrow to the boundary bucket
      int N = 1;
      while (N < nc) N <<= 1;
      for (int i = nc + tid; i < N; i += kSelNT) CA[i] = 0ull;
      __syncthreads();
      for (int k = 2; k <= N; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int i = tid; i < N; i += kSelNT) {
            const int ixj = i ^ j;
            if (ixj > i) {
              const uint64_t a = CA[i], x = CA[ixj];
              const bool desc = (i & k) == 0;
              if (desc ? (a < x) : (a > x)) {
                CA[i] = x;
                CA[ixj] = a;
              }
            }
          }
          __syncthreads();
        }
      }
      if (warp == 0) {
        int cum = 0;
        for (int c0 = 0; c0 < nc; c0 += 32) {
          const int i = c0 + lane;
          int len = 0, idx = 0;
          uint32_t key = 0;
          if (i < nc) {
            idx = (int)(0xffffffffu - (uint32_t)(CA[i] & 0xffffffffull));
            key = (uint32_t)(CA[i] >> 32);
            len = slen[idx - lo];
          }
          const int inc = warp_incl_scan(len);
          const unsigned hit = __ballot_sync(0xffffffffu, i < nc && cum + inc >= need);
          if (hit) {
            if (lane == __ffs(hit) - 1) {
              s_info[0] = idx;
              s_info[1] = need - (cum + inc - len);
              s_info[2] = (int)key;
              s_info[3] = 0;
            }
            break;
          }
          cum += __shfl_sync(0xffffffffu, inc, 31);
        }
      }
      break;
    }
  }
  stamp(4);
  cluster.sync();
  stamp(5);

  // ---- 3. union over this CTA's 1/G of the blocks
  int m[G], keep[G], all[G];
  uint32_t T[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int* peer = cluster.map_shared_rank(s_info, g);
    m[g] = peer[0];
    keep[g] = peer[1];
    T[g] = (uint32_t)peer[2];
    all[g] = peer[3];
  }
  const uint32_t* pk[G];  // every head's keys, from the peers' shared memory (DSMEM)
#pragma unroll
  for (int g = 0; g < G; ++g) pk[g] = cluster.map_shared_rank(K0, g);
  const int r0 = (int)(((long long)c * nr) / G), r1 = (int)(((long long)(c + 1) * nr) / G);
  const int nrg = r1 - r0;
  for (int i = tid; i < nrg; i += kSelNT) {
    const int blk = lo + r0 + i, len = slen[r0 + i];
    uint32_t mask = 0;
    int u = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t key = pk[g][r0 + i];
      if (all[g] || key > T[g] || (key == T[g] && blk <= m[g])) {
        mask |= 1u << g;
        const int tk = (blk == m[g]) ? keep[g] : len;
        u = max(u, (tk + P - 1) >> Pshift);
      }
    }
    sumk[i] = (uint16_t)(u | (mask << 8));
  }
  __syncthreads();
  const int per = (nrg + kSelNT - 1) / kSelNT;
  const int t0 = tid * per, t1 = min(nrg, t0 + per);
  int v[G + 1], tot[G + 1];
#pragma unroll
  for (int k = 0; k <= G; ++k) v[k] = 0;
  for (int i = t0; i < t1; ++i) {
    const uint32_t s = sumk[i];
#pragma unroll
    for (int g = 0; g < G; ++g) v[g] += (s >> (8 + g)) & 1u;
    const int blk = lo + r0 + i;
    if (blk >= olo && blk < ohi) v[G] += s & 0xffu;
  }
  __shared__ int s_scan[(kSelNT / 32 + 1) * (G + 1)];
  stamp(6);
  block_excl_scan<G + 1, kSelNT>(v, tot, s_scan);
  stamp(7);
  if (tid <= G) s_tot[tid] = tot[tid];
  cluster.sync();
  int base[G + 1], all_tot[G + 1];
#pragma unroll
  for (int k = 0; k <= G; ++k) base[k] = all_tot[k] = 0;
  for (int cc = 0; cc < G; ++cc) {
    const int* pt = cluster.map_shared_rank(s_tot, cc);
#pragma unroll
    for (int k = 0; k <= G; ++k) {
      const int x = pt[k];
      if (cc < c) base[k] += x;
      all_tot[k] += x;
    }
  }
#pragma unroll
  for (int k = 0; k <= G; ++k) v[k] += base[k];
  WLEntry* wlb = wl + ((size_t)b * Hkv + hk) * max_wl;
  const int pf_lo = olo < nb ? pf[olo] : 0;
  for (int i = t0; i < t1; ++i) {
    const int blk = lo + r0 + i, len = slen[r0 + i];
    const uint32_t s = sumk[i];
    const int u = s & 0xffu;
    int taken[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const bool sel = (s >> (8 + g)) & 1u;
      taken[g] = sel ? ((blk == m[g]) ? keep[g] : len) : 0;
      if (sel) {
        if (sel_blocks) sel_blocks[((size_t)b * Hq + hk * G + g) * max_sel + v[g]] = blk;
        ++v[g];
      }
    }
    if (u && blk >= olo && blk < ohi) {
      const int page0 = pf[blk] - pf_lo;
      for (int jj = 0; jj < u; ++jj) {
        const int pv = min(P, len - (jj << Pshift));
        uint32_t w0 = 0, w1 = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t r = (uint32_t)min(max(taken[g] - (jj << Pshift), 0), pv);
          if (g < 4) w0 |= r << (8 * g);
          else w1 |= r << (8 * (g - 4));
        }
        *reinterpret_cast<int4*>(wlb + v[G] + jj) = make_int4(page0 + jj, blk, (int)w0, (int)w1);
      }
      v[G] += u;
    }
  }
  if (tid == 0) {
    const size_t o = (size_t)b * Hq + hk * G + c;
    n_sel[o] = all_tot[c];
    marg_out[o] = all[c] ? -1 : m[c];
    keep_out[o] = all[c] ? 0 : keep[c];
    if (c == 0) {
      if (hk == 0 && b == 0) {
        wl_count[-64] = 0x44534b57;  // "DSKW"
        wl_count[-63] = max_wl;
      }
      wl_count[(size_t)b * Hkv + hk] = all_tot[G];
    }
  }
  stamp(8);
  cluster.sync();  // peers may still be reading this CTA's s_info / s_tot
  stamp(9);
}

}  // namespace dsk
extern "C" int dynsplit_debug_select_timer(void* dev_ptr) {
  return (int)cudaMemcpyToSymbol(dsk::g_sel_dbg, &dev_ptr, sizeof(void*));
}
namespace dsk {

size_t select_smem_needed(int maxb, int G) {
  const size_t s = select_smem_bytes(maxb, G);
  return s <= (size_t)max_smem_optin() - 8192 ? s : (size_t)-1;
}

template <int G>
static cudaError_t run_select(int B, int Hkv, size_t smem, const float* scores, const int32_t* bs,
                              const int32_t* nb, const int32_t* pf, int Hq, int maxb, int max_sel,
                              int max_wl, int Pshift, int budget, int blk_lo, int blk_hi,
                              int32_t* sel_blocks, int32_t* n_sel, int32_t* marg, int32_t* keep,
                              int32_t* wl_count, WLEntry* wl, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    allow_max_dyn_smem(k_select<G>);
    attr = true;
  }
  launch_ex(k_select<G>, dim3(Hkv * G, B), dim3(kSelNT), smem, st, G, scores, bs, nb, pf, Hq, Hkv,
            maxb, max_sel, max_wl, Pshift, budget, blk_lo, blk_hi, sel_blocks, n_sel, marg, keep,
            wl_count, wl);
  return post_launch("k_select", st);
}

cudaError_t launch_select(int G, const float* scores, const int32_t* bs, const int32_t* nb,
                          const int32_t* pf, int B, int Hq, int Hkv, int maxb, int max_sel,
                          int max_wl, int P, int budget, int blk_lo, int blk_hi,
                          int32_t* sel_blocks, int32_t* n_sel, int32_t* marg, int32_t* keep,
                          int32_t* wl_count, WLEntry* wl, cudaStream_t st) {
  const size_t smem = select_smem_needed(maxb, G);
  if (smem == (size_t)-1) return cudaErrorInvalidConfiguration;
  int Pshift = 0;
  while ((1 << Pshift) < P) ++Pshift;
#define DSK_SEL(GG)                                                                                \
  return run_select<GG>(B, Hkv, smem, scores, bs, nb, pf, Hq, maxb, max_sel, max_wl, Pshift,       \
                        budget, blk_lo, blk_hi, sel_blocks, n_sel, marg, keep, wl_count, wl, st)
  switch (G) {
    case 1: DSK_SEL(1);
    case 2: DSK_SEL(2);
    case 4: DSK_SEL(4);
    case 8: DSK_SEL(8);
  }
#undef DSK_SEL
  return cudaErrorInvalidValue;
}

}  // namespace dsk
