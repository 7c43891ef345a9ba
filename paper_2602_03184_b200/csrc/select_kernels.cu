// Decode row a6: budgeted top-k through block-to-token mapping (V2F,
// P:257-264; KV Selection Step 1) for every query head, plus the
// GQA-union page worklist consumed by the attention kernel.
//
// Order of blocks for one head: (score desc, block index asc).  Blocks are
// taken whole while the budget lasts; the block that reaches it ("marginal")
// keeps its first `need` tokens (identical to the per-token stable sort of
// the oracle).  One CTA (1024 threads) per (b, KV head):
//   1. block lengths -> smem, total;
//   2. the G heads in rounds of HG concurrent thread groups: score keys ->
//      smem; find the marginal block exactly:
//        - bucket the live scores into 2048 buckets of [min, max] (a monotone
//          map), length-weighted histogram, suffix scan -> boundary bucket;
//        - if it holds <= 512 blocks: exact bitonic sort of (key, ~index)
//          and a prefix walk; otherwise narrow to that bucket and repeat;
//          a bucket of identical scores is resolved in index order.
//   3. union pass: per block the union page count u and the G-bit selection
//      mask (head h takes blk iff all_fit || key > T || key == T && blk <= m);
//      one block-wide scan over contiguous runs; write the worklist entries
//      (page, per-head leading rows) in ascending block order and every
//      head's ascending sel_blocks.
#include "common.cuh"
#include "kernels.h"

#include <math_constants.h>

namespace dsk {

constexpr int kSelNT = 1024;
constexpr int kBkt = 2048;
constexpr int kCap = 512;

DSK_DEVICE float key_to_float(uint32_t k) {
  const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// smem layout (dynamic): skey[HG][mb4] u32 | cand[HG][kCap] u64 | hist[HG][kBkt] u32 |
//                        slen[mb4] u16 | sumk[mb4] u16
static size_t select_smem_bytes(int maxb, int HG) {
  const size_t mb4 = ((size_t)maxb + 3) & ~(size_t)3;
  return HG * mb4 * 4 + (size_t)HG * kCap * 8 + (size_t)HG * kBkt * 4 + mb4 * 2 * 2;
}

template <int G, int HG>
__global__ void __launch_bounds__(kSelNT, 1) k_select(
    const float* __restrict__ scores, const int32_t* __restrict__ block_starts,
    const int32_t* __restrict__ n_blocks, const int32_t* __restrict__ page_first, int Hq, int Hkv,
    int maxb, int max_sel, int max_wl, int P, int budget, int blk_lo, int blk_hi,
    int32_t* __restrict__ sel_blocks, int32_t* __restrict__ n_sel, int32_t* __restrict__ marg_out,
    int32_t* __restrict__ keep_out, int32_t* __restrict__ wl_count, WLEntry* __restrict__ wl) {
  constexpr int TPG = kSelNT / HG;  // threads per head group
  constexpr int WPG = TPG / 32;
  constexpr int BPT = kBkt / TPG;   // histogram buckets per thread in the scan
  extern __shared__ __align__(16) unsigned char smem[];
  const int mb4 = (maxb + 3) & ~3;
  uint32_t* skey_all = reinterpret_cast<uint32_t*>(smem);
  uint64_t* cand_all = reinterpret_cast<uint64_t*>(skey_all + HG * mb4);
  uint32_t* hist_all = reinterpret_cast<uint32_t*>(cand_all + HG * kCap);
  uint16_t* slen = reinterpret_cast<uint16_t*>(hist_all + HG * kBkt);
  uint16_t* sumk = slen + mb4;

  __shared__ float g_f[HG][2][WPG];
  __shared__ int g_i[HG][WPG + 1];
  __shared__ int s_info[G][4];  // marginal, keep, key, all_fit
  __shared__ int s_scan[(kSelNT / 32 + 1) * (G + 1)];
  __shared__ int s_total;
  __shared__ int s_bnd[HG], s_need[HG], s_nc[HG];
  __shared__ float s_mn[HG], s_mx[HG];

  const int hk = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31;
  const int gi = tid / TPG, gt = tid % TPG, gw = gt / 32;
  const int nb = n_blocks[b];
  const int lo = max(blk_lo, 0), hi = min(blk_hi, nb);
  const int nr = max(hi - lo, 0);
  const int32_t* bs = block_starts + (size_t)b * (maxb + 1);
  const int32_t* pf = page_first + (size_t)b * (maxb + 1);
  const float* sc0 = scores + ((size_t)b * Hq + hk * G) * maxb;

  // ---- 1. lengths
  {
    int t = 0;
    for (int i = tid; i < nr; i += kSelNT) {
      const int len = bs[lo + i + 1] - bs[lo + i];
      slen[i] = (uint16_t)len;
      t += len;
    }
    int v[1] = {t}, tot[1];
    block_excl_scan<1, kSelNT>(v, tot, s_scan);
    if (tid == 0) s_total = tot[0];
    __syncthreads();
  }
  const int total = s_total;
  auto gbar = [&]() { named_bar_sync(1 + gi, TPG); };

  // ---- 2. thresholds, HG heads at a time
  for (int round = 0; round < G / HG; ++round) {
    const int g = round * HG + gi;
    uint32_t* K = skey_all + gi * mb4;
    uint64_t* CA = cand_all + gi * kCap;
    uint32_t* HI = hist_all + gi * kBkt;
    const float* sc = sc0 + (size_t)g * maxb + lo;
    if (total <= budget) {
      if (gt == 0) {
        s_info[g][0] = -1;
        s_info[g][1] = 0;
        s_info[g][2] = 0;
        s_info[g][3] = 1;
      }
    } else {
      for (int i = gt; i < nr; i += TPG) K[i] = float_key(sc[i]);
      int need = budget;
      for (int level = 0;; ++level) {
        // min / max of the live scores (key 0 = dead)
        float mn = CUDART_INF_F, mx = -CUDART_INF_F;
        for (int i = gt; i < nr; i += TPG) {
          const uint32_t k = K[i];
          if (k) {
            const float f = key_to_float(k);
            mn = fminf(mn, f);
            mx = fmaxf(mx, f);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
          g_f[gi][0][gw] = mn;
          g_f[gi][1][gw] = mx;
        }
        for (int i = gt; i < kBkt; i += TPG) HI[i] = 0;
        gbar();
        if (gt == 0) {
          float a = g_f[gi][0][0], c = g_f[gi][1][0];
          for (int w = 1; w < WPG; ++w) {
            a = fminf(a, g_f[gi][0][w]);
            c = fmaxf(c, g_f[gi][1][w]);
          }
          s_mn[gi] = a;
          s_mx[gi] = c;
          s_nc[gi] = 0;
        }
        gbar();
        mn = s_mn[gi];
        mx = s_mx[gi];
        if (!(mx > mn)) {
          // all live scores equal: order by block index, walk the prefix
          int carry = 0;
          bool done = false;
          for (int c0 = 0; c0 < nr && !done; c0 += TPG) {
            const int i = c0 + gt;
            const int v = (i < nr && K[i]) ? (int)slen[i] : 0;
            const int inc = warp_incl_scan(v);
            if (lane == 31) g_i[gi][gw] = inc;
            gbar();
            if (gw == 0) {
              const int x = lane < WPG ? g_i[gi][lane] : 0;
              const int s = warp_incl_scan(x);
              if (lane < WPG) g_i[gi][lane] = s - x;
              if (lane == WPG - 1) g_i[gi][WPG] = s;
            }
            gbar();
            const int pre = carry + g_i[gi][gw] + inc;  // inclusive prefix
            if (v > 0 && pre >= need && pre - v < need) {
              s_info[g][0] = lo + i;
              s_info[g][1] = need - (pre - v);
              s_info[g][2] = (int)K[i];
              s_info[g][3] = 0;
            }
            carry += g_i[gi][WPG];
            done = carry >= need;
            gbar();
          }
          break;
        }
        const float inv = (float)kBkt / (mx - mn);
        for (int i = gt; i < nr; i += TPG) {
          const uint32_t k = K[i];
          if (k) {
            const int bk = min(max((int)((key_to_float(k) - mn) * inv), 0), kBkt - 1);
            atomicAdd(&HI[bk], (uint32_t)slen[i]);
          }
        }
        gbar();
        {  // suffix scan, thread gt owns buckets (kBkt-1-gt*BPT) downwards
          const int j0 = kBkt - 1 - gt * BPT;
          int loc = 0;
#pragma unroll
          for (int k = 0; k < BPT; ++k) loc += (int)HI[j0 - k];
          const int inc = warp_incl_scan(loc);
          if (lane == 31) g_i[gi][gw] = inc;
          gbar();
          if (gw == 0) {
            const int x = lane < WPG ? g_i[gi][lane] : 0;
            const int s = warp_incl_scan(x);
            if (lane < WPG) g_i[gi][lane] = s - x;
          }
          gbar();
          int above = g_i[gi][gw] + inc - loc;
#pragma unroll
          for (int k = 0; k < BPT; ++k) {
            const int hb = (int)HI[j0 - k];
            if (above < need && above + hb >= need) {
              s_bnd[gi] = j0 - k;
              s_need[gi] = need - above;
            }
            above += hb;
          }
        }
        gbar();
        const int bnd = s_bnd[gi];
        need = s_need[gi];
        for (int i = gt; i < nr; i += TPG) {
          const uint32_t k = K[i];
          if (k) {
            const int bk = min(max((int)((key_to_float(k) - mn) * inv), 0), kBkt - 1);
            if (bk == bnd) {
              const int p = atomicAdd(&s_nc[gi], 1);
              if (p < kCap) CA[p] = ((uint64_t)k << 32) | (uint64_t)(0xffffffffu - (uint32_t)(lo + i));
            } else {
              K[i] = 0;  // above (already counted in need) or below the boundary
            }
          }
        }
        gbar();
        const int nc = s_nc[gi];
        if (nc > kCap) continue;  // narrow to the boundary bucket
        int N = 1;
        while (N < nc) N <<= 1;
        for (int i = nc + gt; i < N; i += TPG) CA[i] = 0ull;
        gbar();
        for (int k = 2; k <= N; k <<= 1) {
          for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = gt; i < N; i += TPG) {
              const int ixj = i ^ j;
              if (ixj > i) {
                const uint64_t a = CA[i], c = CA[ixj];
                const bool desc = (i & k) == 0;
                if (desc ? (a < c) : (a > c)) {
                  CA[i] = c;
                  CA[ixj] = a;
                }
              }
            }
            gbar();
          }
        }
        if (gw == 0) {
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
                s_info[g][0] = idx;
                s_info[g][1] = need - (cum + inc - len);
                s_info[g][2] = (int)key;
                s_info[g][3] = 0;
              }
              break;
            }
            cum += __shfl_sync(0xffffffffu, inc, 31);
          }
        }
        break;
      }
    }
    __syncthreads();
  }

  // ---- 3. union pass
  int m[G], keep[G], all[G];
  uint32_t T[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = s_info[g][0];
    keep[g] = s_info[g][1];
    T[g] = (uint32_t)s_info[g][2];
    all[g] = s_info[g][3];
  }
  for (int i = tid; i < nr; i += kSelNT) {
    const int blk = lo + i, len = slen[i];
    uint32_t mask = 0;
    int u = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t key = float_key(sc0[(size_t)g * maxb + blk]);
      if (all[g] || key > T[g] || (key == T[g] && blk <= m[g])) {
        mask |= 1u << g;
        const int tk = (blk == m[g]) ? keep[g] : len;
        u = max(u, (tk + P - 1) / P);
      }
    }
    sumk[i] = (uint16_t)(u | (mask << 8));
  }
  __syncthreads();
  const int per = (nr + kSelNT - 1) / kSelNT;
  const int t0 = tid * per, t1 = min(nr, t0 + per);
  int v[G + 1], tot[G + 1];
#pragma unroll
  for (int k = 0; k <= G; ++k) v[k] = 0;
  for (int i = t0; i < t1; ++i) {
    const uint32_t s = sumk[i];
#pragma unroll
    for (int g = 0; g < G; ++g) v[g] += (s >> (8 + g)) & 1u;
    v[G] += s & 0xffu;
  }
  block_excl_scan<G + 1, kSelNT>(v, tot, s_scan);
  WLEntry* wlb = wl + ((size_t)b * Hkv + hk) * max_wl;
  const int pf_lo = nr > 0 ? pf[lo] : 0;
  for (int i = t0; i < t1; ++i) {
    const int blk = lo + i, len = slen[i];
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
    if (u) {
      const int page0 = pf[blk] - pf_lo;
      for (int jj = 0; jj < u; ++jj) {
        const int pv = min(P, len - P * jj);
        uint32_t w0 = 0, w1 = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t r = (uint32_t)min(max(taken[g] - P * jj, 0), pv);
          if (g < 4) w0 |= r << (8 * g);
          else w1 |= r << (8 * (g - 4));
        }
        *reinterpret_cast<int4*>(wlb + v[G] + jj) = make_int4(page0 + jj, blk, (int)w0, (int)w1);
      }
      v[G] += u;
    }
  }
  if (tid == 0) {
    if (hk == 0 && b == 0) {
      wl_count[-64] = 0x44534b57;  // "DSKW"
      wl_count[-63] = max_wl;
    }
    wl_count[(size_t)b * Hkv + hk] = tot[G];
  }
  if (tid < G) {
    const int g = tid;
    const size_t o = (size_t)b * Hq + hk * G + g;
    n_sel[o] = tot[g];
    marg_out[o] = all[g] ? -1 : m[g];
    keep_out[o] = all[g] ? 0 : keep[g];
  }
}

size_t select_smem_needed(int maxb, int G) {
  for (int hg = G < 4 ? G : 4; hg >= 1; hg >>= 1) {
    const size_t s = select_smem_bytes(maxb, hg);
    if (s <= (size_t)max_smem_optin() - 8192) return s;
  }
  return (size_t)-1;
}

template <int G, int HG>
static cudaError_t run_select(dim3 grid, size_t smem, const float* scores, const int32_t* bs,
                              const int32_t* nb, const int32_t* pf, int Hq, int Hkv, int maxb,
                              int max_sel, int max_wl, int P, int budget, int blk_lo, int blk_hi,
                              int32_t* sel_blocks, int32_t* n_sel, int32_t* marg, int32_t* keep,
                              int32_t* wl_count, WLEntry* wl, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    allow_max_dyn_smem(k_select<G, HG>);
    attr = true;
  }
  k_select<G, HG><<<grid, kSelNT, smem, st>>>(scores, bs, nb, pf, Hq, Hkv, maxb, max_sel, max_wl, P,
                                              budget, blk_lo, blk_hi, sel_blocks, n_sel, marg, keep,
                                              wl_count, wl);
  return post_launch("k_select", st);
}

cudaError_t launch_select(int G, const float* scores, const int32_t* bs, const int32_t* nb,
                          const int32_t* pf, int B, int Hq, int Hkv, int maxb, int max_sel,
                          int max_wl, int P, int budget, int blk_lo, int blk_hi,
                          int32_t* sel_blocks, int32_t* n_sel, int32_t* marg, int32_t* keep,
                          int32_t* wl_count, WLEntry* wl, cudaStream_t st) {
  int hg = G < 4 ? G : 4;
  while (hg > 1 && select_smem_bytes(maxb, hg) > (size_t)max_smem_optin() - 8192) hg >>= 1;
  const size_t smem = select_smem_bytes(maxb, hg);
  if (smem > (size_t)max_smem_optin() - 8192) return cudaErrorInvalidConfiguration;
  dim3 grid(Hkv, B);
#define DSK_SEL(GG, HH)                                                                            \
  return run_select<GG, HH>(grid, smem, scores, bs, nb, pf, Hq, Hkv, maxb, max_sel, max_wl, P,     \
                            budget, blk_lo, blk_hi, sel_blocks, n_sel, marg, keep, wl_count, wl, st)
  switch (G) {
    case 1: DSK_SEL(1, 1);
    case 2:
      if (hg == 2) DSK_SEL(2, 2);
      DSK_SEL(2, 1);
    case 4:
      if (hg == 4) DSK_SEL(4, 4);
      if (hg == 2) DSK_SEL(4, 2);
      DSK_SEL(4, 1);
    case 8:
      if (hg == 4) DSK_SEL(8, 4);
      if (hg == 2) DSK_SEL(8, 2);
      DSK_SEL(8, 1);
  }
#undef DSK_SEL
  return cudaErrorInvalidValue;
}

}  // namespace dsk
