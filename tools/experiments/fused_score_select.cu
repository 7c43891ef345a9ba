// EXPERIMENT (not built, not part of the product) -- kept as the record of a
// measured negative result.  Fusing rows a5 + a6 into one kernel with one
// thread-block cluster per (b, KV head) and the histogram / candidate
// hand-over through DSMEM was correct (bit-identical to the two-kernel path on
// every test shape, including exact ties and narrowing rounds) but slower on
// B200 at 128K / 32Q / 8KV / budget 4096 (tools/exp_decode.py, CUDA graph):
//   two kernels (k_score_blocks + k_select_reg): 6.7 + 11.8 us
//   fused, cluster 16: 62.5 us  (only half of the 16-CTA clusters are
//                                co-resident: two waves)
//   fused, cluster 8:  36.7 us;  cluster 4: 45.9 us
// Per-phase stamps showed every cluster-barrier phase costing 2.5-9 us (DSMEM
// atomics for the histogram push, release/acquire cluster barriers, one
// latency-bound CTA per SM).  See DESIGN.md "Measured alternatives".
//
// Decode rows a5 + a6 fused (dynsplit_select over the whole sequence): block
// scores (V2F), budgeted top-k through block-to-token mapping
// (KV Selection Step 1) for every query head, and the
// GQA-union page worklist -- one kernel, one thread-block cluster of CS CTAs
// (up to 16, one per SM) per (b, KV head).
//
// Why fused: as two kernels, the select stage ran on only B * Hkv * G CTAs
// (32 SMs at 128K / 32Q / 8KV) and could not start before every score CTA had
// drained; here the whole per-(b, KV head) pipeline is spread over CS SMs and
// the stages hand over through distributed shared memory (DSMEM) and cluster
// barriers instead of HBM round trips and kernel boundaries.
//
// CTA r of the cluster owns the contiguous block range [r nb / CS, (r+1) nb / CS)
// for all G query heads of the KV head:
//  S. scores of its blocks: the digest range is bulk-prefetched into L2 before
//     the PDL wait (it is resident data, independent of the step); after it, a
//     half-warp per block computes sum_j max(q_j kmax_j, q_j kmin_j) for the G
//     heads with exactly the arithmetic and reduction order of k_score_blocks
//     (bit-identical scores for every launch shape);
//  T. per head, the exact marginal block in rounds:
//       a. cluster min / max of the live keys (DSMEM reduce);
//       b. length-weighted local histograms over 2048 buckets of [min, max];
//       c. CTA r sums bucket slice r over the cluster (DSMEM reads);
//       d. the slice holding the budget boundary finds the boundary bucket;
//       e. the boundary bucket's blocks are sent to the head's owner CTA
//          (DSMEM atomics); <= 32 candidates are ranked by one warp (key desc,
//          index asc); otherwise the live set narrows to the bucket and the
//          round repeats; equal live keys are resolved in index order;
//  U. per block the union page count and each head's selection; block-wide
//     scans, cluster offsets of the earlier ranks; worklist entries
//     (interleaved layout), sel_blocks (ascending), n_sel, marginal, keep.
#include "common.cuh"
#include "kernels.h"

#include <cooperative_groups.h>
#include <math_constants.h>
#include <stdlib.h>

namespace cg = cooperative_groups;

namespace dsk {

constexpr int kFT = 512;             // threads per CTA
constexpr int kFW = kFT / 32;
constexpr int kFB = 2048;            // buckets per round
constexpr int kFC = 32;              // candidates ranked by one warp
constexpr int kFMaxCS = 16;

// Optional per-CTA phase timestamps (debug only; dynsplit_debug_fused_timer).
__device__ unsigned long long* g_fused_dbg = nullptr;
DSK_DEVICE void fstamp(int k) {
#ifdef DSK_DEBUG
  if (g_fused_dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_fused_dbg[(size_t)blockIdx.x * 16 + k] = t;
  }
#else
  (void)k;
#endif
}

DSK_DEVICE void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
DSK_DEVICE void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
DSK_DEVICE void cl_sync() {
  cl_arrive();
  cl_wait();
}
DSK_DEVICE float fkey_to_float(uint32_t k) {
  const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}
DSK_DEVICE int fbucket(uint32_t k, float mn, float inv) {
  return min(max((int)((fkey_to_float(k) - mn) * inv), 0), kFB - 1);
}

// Lane c < CS of every warp reads value p from cluster rank c (DSMEM, one
// latency for the warp); returns (sum over ranks < r, sum over all ranks).
DSK_DEVICE int2 cluster_prefix(const int* p, int r, int CS) {
  cg::cluster_group cluster = cg::this_cluster();
  const int lane = threadIdx.x & 31;
  const int x = lane < CS ? *cluster.map_shared_rank(p, lane) : 0;
  return make_int2(warp_sum_i(lane < r ? x : 0), warp_sum_i(x));
}

// Digest dot products (identical arithmetic to decode_kernels.cu's DigestDot).
template <typename T> struct FDot;
template <> struct FDot<bf16> {
  struct Q {
    uint32_t w[4], sel[4];
  };
  struct K {
    uint4 mx, mn;
  };
  static DSK_DEVICE void load_q(const bf16* p, Q& q) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
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
  static DSK_DEVICE void zero_k(K& k) { k.mx = k.mn = make_uint4(0, 0, 0, 0); }
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
template <> struct FDot<float> {
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
  static DSK_DEVICE void zero_k(K& k) {
#pragma unroll
    for (int j = 0; j < 8; ++j) k.mx[j] = k.mn[j] = 0.f;
  }
  static DSK_DEVICE float dot(const Q& q, const K& k) {
    float a = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) a = fmaf(q.v[j], q.v[j] >= 0.f ? k.mx[j] : k.mn[j], a);
    return a;
  }
};

// Shared state of one CTA (static part; the per-block arrays are dynamic).
template <int G>
struct FShared {
  float mm[G][2];          // this CTA's live min / max per head (read by peers)
  float gmm[G][2];         // cluster min / max per head
  int stot[G];             // this CTA's bucket-slice total per head (read by peers)
  int sinfo[G][2];         // boundary bucket, remaining need (on the slice owner)
  int hinfo[G][4];         // per head: bucket, need, slice owner, tie flag (this round)
  int nc[G];               // candidate count (on the head owner)
  uint64_t ca[G][kFC];     // candidates (key << 32 | ~index) (on the head owner)
  int cl[G][kFC];          // candidate lengths
  int minfo[G][4];         // marginal, keep, threshold key, done (on the head owner)
  int fin[G][4];           // the same, gathered from the owners
  int tlive[G];            // tie rounds: this CTA's live length per head
  int utot[G + 1];         // union pass: this CTA's totals (heads, pages) (read by peers)
  int red_i[kFW][G];
  float red_f[kFW][G][2];
  int scan[(kFW + 1) * (G + 1)];
  int any_open;
};

// dynamic smem: HL[G][kFB] u32 | skey[G][KPT*512] u32 | slen[KPT*512] i32 | spf[KPT*512] i32
static size_t fused_dyn_smem(int G, int KPT) {
  return (size_t)G * kFB * 4 + (size_t)G * KPT * kFT * 4 + (size_t)KPT * kFT * 8;
}

template <typename T, int G, int KPT>
__global__ void __launch_bounds__(kFT, 1) k_score_select(
    const T* __restrict__ q, const T* __restrict__ dig, const int32_t* __restrict__ block_starts,
    const int32_t* __restrict__ n_blocks, const int32_t* __restrict__ page_first, int Hq, int Hkv,
    int maxb, int max_sel, int Pshift, int budget, float* __restrict__ scores_out,
    int32_t* __restrict__ sel_blocks, int32_t* __restrict__ n_sel, int32_t* __restrict__ marg_out,
    int32_t* __restrict__ keep_out, int32_t* __restrict__ wl_count, WLEntry* __restrict__ wl,
    int max_wl) {
  using DD = FDot<T>;
  constexpr int NL = KPT * kFT;  // local block capacity
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t(*HL)[kFB] = reinterpret_cast<uint32_t(*)[kFB]>(smem);
  uint32_t(*skey)[NL] = reinterpret_cast<uint32_t(*)[NL]>(smem + (size_t)G * kFB * 4);
  int32_t* slen = reinterpret_cast<int32_t*>(smem + (size_t)G * kFB * 4 + (size_t)G * NL * 4);
  int32_t* spf = slen + NL;
  __shared__ FShared<G> sh;

  const int CS = (int)cluster.num_blocks();
  const int r = (int)cluster.block_rank();
  const int bh = blockIdx.x / CS, b = bh / Hkv, hk = bh % Hkv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = 1 << Pshift;
  const int nb = n_blocks[b];
  const int lo = (int)(((long long)r * nb) / CS), hi = (int)(((long long)(r + 1) * nb) / CS);
  const int nr = hi - lo;
  const int32_t* bs = block_starts + (size_t)b * (maxb + 1);
  const int32_t* pf = page_first + (size_t)b * (maxb + 1);
  const T* dbase = dig + ((size_t)b * Hkv + hk) * (size_t)maxb * 2 * kD;
  auto peer = [&](auto* p, int rank) { return cluster.map_shared_rank(p, rank); };

  fstamp(0);
  // ---- pre-PDL: the resident plan and digests (independent of the step)
  {
    const unsigned char* dp = reinterpret_cast<const unsigned char*>(dbase + (size_t)lo * 2 * kD);
    const uint32_t bytes = (uint32_t)nr * 2 * kD * (uint32_t)sizeof(T);
    for (uint32_t off = tid * 4096u; off < bytes; off += kFT * 4096u)
      prefetch_l2_bulk(dp + off, min(4096u, bytes - off));
  }
  for (int i = tid; i < NL; i += kFT) {
    int len = 0, p0 = 0;
    if (i < nr) {
      len = bs[lo + i + 1] - bs[lo + i];
      p0 = pf[lo + i];
    }
    slen[i] = len;
    spf[i] = p0;
  }
  for (int i = tid; i < G * kFB; i += kFT) (&HL[0][0])[i] = 0u;
  const int total = bs[nb] - bs[0];
  pdl_trigger();
  pdl_wait();
  fstamp(1);

  // ---- S. scores: half-warp per block, lane hl owns dims [8 hl, 8 hl + 8)
  {
    const int half = lane >> 4, hl = lane & 15;
    typename DD::Q qv[G];
#pragma unroll
    for (int g = 0; g < G; ++g) DD::load_q(q + ((size_t)b * Hq + hk * G + g) * kD + hl * 8, qv[g]);
    constexpr int U = (sizeof(T) == 2 && G <= 4) ? 4 : 2;  // digest loads in flight per lane
    for (int base = warp * 2; base < nr; base += kFW * 2 * U) {  // warp-uniform trip count
      typename DD::K kb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * kFW * 2 + half;
        if (i < nr) DD::load_k(dbase + (size_t)(lo + i) * 2 * kD + hl * 8, kb[u]);
        else DD::zero_k(kb[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * kFW * 2 + half;
        float acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = DD::dot(qv[g], kb[u]);
#pragma unroll
        for (int g = 0; g < G; ++g) {
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], o);
        }
        if (hl == 0 && i < nr) {
#pragma unroll
          for (int g = 0; g < G; ++g) {
            skey[g][i] = float_key(acc[g]);
            if (scores_out) scores_out[((size_t)b * Hq + hk * G + g) * maxb + lo + i] = acc[g];
          }
        }
      }
    }
  }
  __syncthreads();
  fstamp(2);

  // keys of this thread's blocks i = k * 512 + tid (0 = not live)
  uint32_t key[KPT][G];
  int len[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int i = k * kFT + tid;
    len[k] = slen[i];
#pragma unroll
    for (int g = 0; g < G; ++g) key[k][g] = i < nr ? skey[g][i] : 0u;
  }
  int need[G];
#pragma unroll
  for (int g = 0; g < G; ++g) need[g] = budget;
  const bool all_fit = total <= budget;
  if (tid < G) {
    sh.minfo[tid][0] = -1;
    sh.minfo[tid][1] = 0;
    sh.minfo[tid][2] = 0;
    sh.minfo[tid][3] = all_fit ? 1 : 0;  // done
  }
  // owner CTA of head g: g % CS
  bool open[G];
#pragma unroll
  for (int g = 0; g < G; ++g) open[g] = !all_fit;
  bool any = !all_fit;
  cl_sync();  // every CTA of the cluster is running and has initialised its state

  // ---- T. threshold rounds
  while (any) {
    // a. min / max of the live keys, per head, over the cluster
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float mn = CUDART_INF_F, mx = -CUDART_INF_F;
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        if (key[k][g]) {
          const float f = fkey_to_float(key[k][g]);
          mn = fminf(mn, f);
          mx = fmaxf(mx, f);
        }
      }
      mn = -warp_max(-mn);
      mx = warp_max(mx);
      if (lane == 0) {
        sh.red_f[warp][g][0] = mn;
        sh.red_f[warp][g][1] = mx;
      }
    }
    if (tid < G) sh.nc[tid] = 0;
    __syncthreads();
    if (warp < G) {
      const int g = warp;
      float mn = lane < kFW ? sh.red_f[lane][g][0] : CUDART_INF_F;
      float mx = lane < kFW ? sh.red_f[lane][g][1] : -CUDART_INF_F;
      mn = -warp_max(-mn);
      mx = warp_max(mx);
      if (lane == 0) {
        sh.mm[g][0] = mn;
        sh.mm[g][1] = mx;
      }
    }
    cl_sync();  // (1) mm published; peers' nc reset; previous round's readers done
    fstamp(3);
    if (warp < G) {
      const int g = warp;
      float mn = CUDART_INF_F, mx = -CUDART_INF_F;
      if (lane < CS) {
        const float* pm = peer(&sh.mm[g][0], lane);
        mn = pm[0];
        mx = pm[1];
      }
      mn = -warp_max(-mn);
      mx = warp_max(mx);
      if (lane == 0) {
        sh.gmm[g][0] = mn;
        sh.gmm[g][1] = mx;
      }
    }
    __syncthreads();
    // b. length-weighted histogram, pushed straight into the owner of each
    //    bucket (bucket j belongs to CTA (j CS + CS - 1) / kFB, slices
    //    [r kFB / CS, (r+1) kFB / CS)) with DSMEM reductions
    const int s0 = (r * kFB) / CS, s1 = ((r + 1) * kFB) / CS;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float mn = sh.gmm[g][0], mx = sh.gmm[g][1];
      if (open[g] && mx > mn) {
        const float inv = (float)kFB / (mx - mn);
#pragma unroll
        for (int k = 0; k < KPT; ++k) {
          if (key[k][g]) {
            const int j = fbucket(key[k][g], mn, inv);
            atomicAdd(peer(&HL[g][j], (j * CS + CS - 1) / kFB), (uint32_t)len[k]);
          }
        }
      }
    }
    cl_sync();  // (2) histogram slices complete at their owners
    fstamp(4);
    // c. this CTA's slice totals per head (local)
    int part[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      part[g] = 0;
      for (int j = s0 + tid; j < s1; j += kFT) part[g] += (int)HL[g][j];
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      int v = warp_sum_i(part[g]);
      if (lane == 0) sh.red_i[warp][g] = v;
    }
    __syncthreads();
    if (tid < G) {
      int v = 0;
      for (int w = 0; w < kFW; ++w) v += sh.red_i[w][tid];
      sh.stot[tid] = v;
    }
    cl_sync();  // (3) slice totals published
    // d. the slice holding each open head's boundary, then the bucket inside it
    if (warp < G) {
      const int g = warp;
      const int tc = lane < CS ? peer(&sh.stot[g], lane)[0] : 0;
      // slices in descending bucket order: slice c is above slice c' if c > c'
      int above = 0;  // total of slices above `lane`
      for (int c = CS - 1; c >= 0; --c) {
        const int v = __shfl_sync(0xffffffffu, tc, c);
        if (c > lane) above += v;
      }
      const int nd = need[g];
      const bool hit = lane < CS && above < nd && above + tc >= nd;
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      const int owner = m ? __ffs(m) - 1 : 0;
      const int above_o = __shfl_sync(0xffffffffu, above, owner);
      if (lane == 0) {
        const bool tie = !(sh.gmm[g][1] > sh.gmm[g][0]);
        sh.hinfo[g][0] = -1;
        sh.hinfo[g][1] = nd - above_o;  // need inside the owner's slice
        sh.hinfo[g][2] = owner;
        sh.hinfo[g][3] = tie ? 1 : 0;
      }
    }
    __syncthreads();
    // the owner of head g's boundary slice finds the bucket (descending scan)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (open[g] && !sh.hinfo[g][3] && sh.hinfo[g][2] == r && warp == 0) {
        const int nd = sh.hinfo[g][1];
        int acc = 0, bnd = -1, rem = 0;
        for (int j0 = s1 - 1; j0 >= s0 && bnd < 0; j0 -= 32) {
          const int bk = j0 - lane;
          const uint32_t s = bk >= s0 ? HL[g][bk] : 0u;
          const int inc = warp_incl_scan((int)s);
          const int tot = __shfl_sync(0xffffffffu, inc, 31);
          const bool h = bk >= s0 && acc + inc - (int)s < nd && acc + inc >= nd;
          const unsigned m = __ballot_sync(0xffffffffu, h);
          if (m) {
            const int l = __ffs(m) - 1;
            bnd = __shfl_sync(0xffffffffu, bk, l);
            rem = nd - (acc + __shfl_sync(0xffffffffu, inc - (int)s, l));
          }
          acc += tot;
        }
        if (lane == 0) {
          sh.sinfo[g][0] = bnd;
          sh.sinfo[g][1] = rem;
        }
      }
    }
    cl_sync();  // (4) boundary buckets published; all histogram reads done
    fstamp(5);
    // e. candidates of the boundary bucket -> the head owner (g % CS)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (!open[g] || sh.hinfo[g][3]) continue;
      const int* si = peer(&sh.sinfo[g][0], sh.hinfo[g][2]);
      const int bnd = si[0];
      const float mn = sh.gmm[g][0], mx = sh.gmm[g][1];
      const float inv = (float)kFB / (mx - mn);
      const int ow = g % CS;
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        const uint32_t kk = key[k][g];
        if (!kk) continue;
        if (fbucket(kk, mn, inv) == bnd) {
          const int p = atomicAdd(peer(&sh.nc[g], ow), 1);
          if (p < kFC) {
            const int blk = lo + k * kFT + tid;
            peer(&sh.ca[g][0], ow)[p] = ((uint64_t)kk << 32) | (uint64_t)(0xffffffffu - (uint32_t)blk);
            peer(&sh.cl[g][0], ow)[p] = len[k];
          }
        } else {
          key[k][g] = 0u;  // above (counted in need) or below: no longer live
        }
      }
      need[g] = si[1];
    }
    // tie heads: every live key equal -> index order (ranks in block order)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (!open[g] || !sh.hinfo[g][3]) continue;
      int v = 0;
#pragma unroll
      for (int k = 0; k < KPT; ++k) v += key[k][g] ? len[k] : 0;
      v = warp_sum_i(v);
      if (lane == 0) sh.red_i[warp][g] = v;
    }
    __syncthreads();
    if (tid < G) {
      int v = 0;
      for (int w = 0; w < kFW; ++w) v += sh.red_i[w][tid];
      sh.tlive[tid] = v;
    }
    cl_sync();  // (5) candidates delivered; tie totals published
    // owners rank their heads' candidates; tie heads are resolved by the CTA
    // whose block range holds the marginal (ascending CTA / block order)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (!open[g]) continue;
      if (!sh.hinfo[g][3]) {
        if (g % CS == r && warp == 0) {
          const int nc = sh.nc[g];
          if (nc <= kFC) {
            const int nd = need[g];
            const uint64_t mine = lane < nc ? sh.ca[g][lane] : 0ull;
            const int ml = lane < nc ? sh.cl[g][lane] : 0;
            int before = 0;
            for (int j = 0; j < nc; ++j) {
              const uint64_t o = __shfl_sync(0xffffffffu, mine, j);
              const int ol = __shfl_sync(0xffffffffu, ml, j);
              before += (o > mine) ? ol : 0;
            }
            if (lane < nc && before < nd && before + ml >= nd) {
              sh.minfo[g][0] = (int)(0xffffffffu - (uint32_t)(mine & 0xffffffffull));
              sh.minfo[g][1] = nd - before;
              sh.minfo[g][2] = (int)(uint32_t)(mine >> 32);
            }
            if (lane == 0) sh.minfo[g][3] = 1;
          }
        }
      } else {
        // prefix of live lengths over the CTAs below this one
        const int below = cluster_prefix(&sh.tlive[g], r, CS).x;
        const int mine_tot = sh.tlive[g];
        const int nd = need[g];
        if (below < nd && below + mine_tot >= nd) {
          // the marginal is in this CTA: index-order scan (block i = k * 512 + t)
          int carry = below;
          for (int k = 0; k < KPT; ++k) {
            int v = 0, kk0 = 0;
#pragma unroll
            for (int kk = 0; kk < KPT; ++kk)
              if (kk == k) {
                v = key[kk][g] ? len[kk] : 0;
                kk0 = (int)key[kk][g];
              }
            int tot[1], vv[1] = {v};
            block_excl_scan<1, kFT>(vv, tot, sh.scan);
            const int bef = carry + vv[0];
            if (v > 0 && bef < nd && bef + v >= nd) {
              sh.minfo[g][0] = lo + k * kFT + tid;
              sh.minfo[g][1] = nd - bef;
              sh.minfo[g][2] = kk0;
            }
            carry += tot[0];
          }
        }
        if (tid == 0 && g % CS == r) sh.minfo[g][3] = 1;  // resolved this round (owner flags it)
      }
    }
    // tie heads resolved in a non-owner CTA: send the result to the owner
    __syncthreads();
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (!open[g] || !sh.hinfo[g][3]) continue;
      const int below = cluster_prefix(&sh.tlive[g], r, CS).x;
      const int nd = need[g];
      if (tid == 0 && below < nd && below + sh.tlive[g] >= nd && g % CS != r) {
        int* dst = peer(&sh.minfo[g][0], g % CS);
        dst[0] = sh.minfo[g][0];
        dst[1] = sh.minfo[g][1];
        dst[2] = sh.minfo[g][2];
        dst[3] = 1;
      }
    }
    // HL is free again (all slice reads happened before barrier (4))
    for (int i = tid; i < G * kFB; i += kFT) (&HL[0][0])[i] = 0u;
    cl_sync();  // (6) results at the owners
    fstamp(6);
    any = false;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (!open[g]) continue;
      const int done = peer(&sh.minfo[g][3], g % CS)[0];
      open[g] = !done;
      any |= open[g];
    }
  }

  // ---- gather every head's result from its owner
  if (tid < G * 4) {
    const int g = tid / 4, x = tid % 4;
    sh.fin[g][x] = peer(&sh.minfo[g][0], g % CS)[x];
  }
  __syncthreads();

  // ---- U. union + outputs: thread tid owns blocks i = tid * KPT + k (index order)
  int mg[G], kg[G];
  uint32_t Tg[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const bool fit = all_fit;
    mg[g] = fit ? -1 : sh.fin[g][0];
    kg[g] = fit ? 0 : sh.fin[g][1];
    Tg[g] = fit ? 0u : (uint32_t)sh.fin[g][2];
  }
  int v[G + 1], vt[G + 1];
#pragma unroll
  for (int g = 0; g <= G; ++g) v[g] = 0;
  uint32_t selm[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int i = tid * KPT + k, blk = lo + i;
    uint32_t m = 0;
    int u = 0;
    if (i < nr) {
      const int ln = slen[i];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t k0 = skey[g][i];
        if (all_fit || k0 > Tg[g] || (k0 == Tg[g] && blk <= mg[g])) {
          m |= 1u << g;
          ++v[g];
          const int tk = blk == mg[g] ? kg[g] : ln;
          u = max(u, (tk + P - 1) >> Pshift);
        }
      }
    }
    selm[k] = m | ((uint32_t)u << 16);
    v[G] += u;
  }
  block_excl_scan<G + 1, kFT>(v, vt, sh.scan);
  if (tid <= G) sh.utot[tid] = vt[tid];
  cl_sync();  // (7) union totals published
  fstamp(7);
  int base[G + 1], all_tot[G + 1];
#pragma unroll
  for (int g = 0; g <= G; ++g) {
    const int x = lane < CS ? peer(&sh.utot[g], lane)[0] : 0;  // lanes of every warp: one rank each
    base[g] = warp_sum_i(lane < r ? x : 0);
    all_tot[g] = warp_sum_i(x);
  }
  cl_arrive();  // (8) done reading the peers' shared memory
#pragma unroll
  for (int g = 0; g <= G; ++g) v[g] += base[g];
  const size_t BH = (size_t)(gridDim.x / CS);  // B * Hkv clusters
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int i = tid * KPT + k, blk = lo + i;
    const uint32_t m = selm[k] & 0xffffu;
    const int u = (int)(selm[k] >> 16);
    if (!m) continue;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if ((m >> g) & 1u) {
        if (sel_blocks) sel_blocks[((size_t)b * Hq + hk * G + g) * max_sel + v[g]] = blk;
        ++v[g];
      }
    }
    const int ln = slen[i];
    for (int jj = 0; jj < u; ++jj) {
      const int pv = min(P, ln - (jj << Pshift));
      uint32_t w0 = 0, w1 = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int tk = ((m >> g) & 1u) ? (blk == mg[g] ? kg[g] : ln) : 0;
        const uint32_t rr = (uint32_t)min(max(tk - (jj << Pshift), 0), pv);
        if (g < 4) w0 |= rr << (8 * g);
        else w1 |= rr << (8 * (g - 4));
      }
      *reinterpret_cast<int4*>(wl + (size_t)(v[G] + jj) * BH + bh) =
          make_int4(spf[i] + jj, blk, (int)w0, (int)w1);
    }
    v[G] += u;
  }
  if (r == 0 && tid < G) {
    const size_t o = (size_t)b * Hq + hk * G + tid;
    n_sel[o] = all_tot[tid];
    marg_out[o] = all_fit ? -1 : mg[tid];
    keep_out[o] = all_fit ? 0 : kg[tid];
  }
  if (r == 0 && tid == 0) {
    if (bh == 0) {
      wl_count[-64] = 0x44534b57;  // "DSKW"
      wl_count[-63] = max_wl;
    }
    wl_count[bh] = all_tot[G];
  }
  fstamp(8);
  cl_wait();  // (8) peers may still be reading this CTA's shared memory
  fstamp(9);
}

}  // namespace dsk
extern "C" int dynsplit_debug_fused_timer(void* dev_ptr) {
  return (int)cudaMemcpyToSymbol(dsk::g_fused_dbg, &dev_ptr, sizeof(void*));
}
namespace dsk {

// ============================================================================
// host launcher
// ============================================================================
template <typename T, int G, int KPT>
static cudaError_t run_fused(int CS, int B, int Hq, int Hkv, int maxb, int max_sel, int max_wl,
                             int Pshift, int budget, const void* q, const void* dig, const int32_t* bs,
                             const int32_t* nb, const int32_t* pf, float* scores_out, int32_t* sel_blocks,
                             int32_t* n_sel, int32_t* marg, int32_t* keep, int32_t* wl_count, WLEntry* wl,
                             cudaStream_t st) {
  auto kern = k_score_select<T, G, KPT>;
  static bool attr = false;
  if (!attr) {
    allow_max_dyn_smem(kern);
    cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaGetLastError();
    attr = true;
  }
  launch_ex(kern, dim3(B * Hkv * CS), dim3(kFT), fused_dyn_smem(G, KPT), st, CS,
            static_cast<const T*>(q), static_cast<const T*>(dig), bs, nb, pf, Hq, Hkv, maxb, max_sel,
            Pshift, budget, scores_out, sel_blocks, n_sel, marg, keep, wl_count, wl, max_wl);
  return post_launch("k_score_select", st);
}

// Cluster size: the largest of {16, 8, 4, 2, 1} with B * Hkv * CS <= SMs whose
// per-CTA share of the blocks fits KPT <= 4 (else not applicable).
static int fused_cluster_size(int B, int Hkv, int maxb, int* kpt) {
  const int sms = num_sms();
  static const int cs_max = [] {
    const char* e = getenv("DYNSPLIT_FUSED_CS");  // A/B experiments only
    const int v = e ? atoi(e) : 8;
    return v >= 1 && v <= kFMaxCS ? v : 8;
  }();
  for (int cs = cs_max; cs >= 1; cs >>= 1) {
    if (B * Hkv * cs > sms && cs > 1) continue;
    const int per = (maxb + cs - 1) / cs;
    const int k = (per + kFT - 1) / kFT;
    if (k > 4) return 0;
    *kpt = k <= 1 ? 1 : (k <= 2 ? 2 : 4);
    return cs;
  }
  return 0;
}

template <typename T, int G>
static cudaError_t fused_g(int CS, int KPT, int B, int Hq, int Hkv, int maxb, int max_sel, int max_wl,
                           int Pshift, int budget, const void* q, const void* dig, const int32_t* bs,
                           const int32_t* nb, const int32_t* pf, float* so, int32_t* sb, int32_t* ns,
                           int32_t* mg, int32_t* kp, int32_t* wc, WLEntry* wl, cudaStream_t st) {
#define DSK_F(K) \
  return run_fused<T, G, K>(CS, B, Hq, Hkv, maxb, max_sel, max_wl, Pshift, budget, q, dig, bs, nb, pf, so, sb, ns, mg, kp, wc, wl, st)
  if (KPT == 1) DSK_F(1);
  if (KPT == 2) DSK_F(2);
  DSK_F(4);
#undef DSK_F
}

cudaError_t launch_score_select(int dtype, int G, const void* q, const void* dig, const int32_t* bs,
                                const int32_t* nb, const int32_t* pf, int B, int Hq, int Hkv, int maxb,
                                int max_sel, int max_wl, int P, int budget, float* scores_out,
                                int32_t* sel_blocks, int32_t* n_sel, int32_t* marg, int32_t* keep,
                                int32_t* wl_count, WLEntry* wl, cudaStream_t st) {
  int kpt = 0;
  const int CS = fused_cluster_size(B, Hkv, maxb, &kpt);
  if (!CS || G > kMaxG) return cudaErrorNotSupported;
  if (fused_dyn_smem(G, kpt) > (size_t)max_smem_optin() - sizeof(FShared<kMaxG>) - 1024)
    return cudaErrorNotSupported;
  int Pshift = 0;
  while ((1 << Pshift) < P) ++Pshift;
#define DSK_G(GG, TT)                                                                                \
  return fused_g<TT, GG>(CS, kpt, B, Hq, Hkv, maxb, max_sel, max_wl, Pshift, budget, q, dig, bs, nb, \
                         pf, scores_out, sel_blocks, n_sel, marg, keep, wl_count, wl, st)
  if (dtype == 0) {
    switch (G) {
      case 1: DSK_G(1, bf16);
      case 2: DSK_G(2, bf16);
      case 4: DSK_G(4, bf16);
      case 8: DSK_G(8, bf16);
    }
  } else {
    switch (G) {
      case 1: DSK_G(1, float);
      case 2: DSK_G(2, float);
      case 4: DSK_G(4, float);
      case 8: DSK_G(8, float);
    }
  }
#undef DSK_G
  return cudaErrorNotSupported;
}

}  // namespace dsk
