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
//        - bucket the live scores into kBkt = 1024 buckets of [min, max] (a monotone
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
#include <stdlib.h>

namespace cg = cooperative_groups;

namespace dsk {

constexpr int kSelNT = 512;
constexpr int kSelW = kSelNT / 32;
constexpr int kBkt = 1024;  // histogram buckets (2048: 0.5 % slower step; 512: same as 1024, wider boundary buckets)
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
    int maxb, int S, int max_sel, int max_wl, int Pshift, int budget, int blk_lo, int blk_hi,
    int32_t* __restrict__ sel_blocks, int32_t* __restrict__ n_sel, int32_t* __restrict__ marg_out,
    int32_t* __restrict__ keep_out, int32_t* __restrict__ wl_count, WLEntry* __restrict__ wl,
    int* __restrict__ err) {
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
  const int nb_raw = n_blocks[b];
  const int nb = min(max(nb_raw, 0), maxb);
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
  //         (PDL) -- the keys of this CTA's head, total.  The plan must tile
  //         [0, L <= S); a block longer than 255 pages or 65535 tokens
  //         is beyond the 8/16-bit counters: such a sequence selects nothing.
  int t = 0, bad = 0, bad_long = 0, npg = 0;
  if (tid == 0) bad = nb_raw < 1 || nb_raw > maxb || bs[0] != 0 || bs[nb] > S;
  for (int i = tid; i < nr; i += kSelNT) {
    const int len = bs[lo + i + 1] - bs[lo + i];
    bad |= len <= 0;
    bad_long |= len > 0xffff || ((len + P - 1) >> Pshift) > 255;
    slen[i] = (uint16_t)len;
    t += len;
    npg += (len + P - 1) >> Pshift;
  }
  __shared__ int s_npg;
  if (tid == 0) s_npg = 0;
  __syncthreads();
  atomicAdd(&s_npg, npg);
  const int any_bad = __syncthreads_or(bad), any_long = __syncthreads_or(bad_long);
  if (any_bad || any_long || s_npg > max_wl) {
    if (tid == 0) {
      raise_err(err, any_bad ? kErrPlanCoverage : any_long ? kErrBlockTooLong : kErrPageCapacity);
      const size_t o = (size_t)b * Hq + hk * G + c;
      n_sel[o] = 0;
      marg_out[o] = -1;
      keep_out[o] = 0;
      if (c == 0) wl_count[(size_t)b * Hkv + hk] = 0;
    }
    return;
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
  // interleaved layout: entry e of (b, KV head) bh at wl[e * B * Hkv + bh]
  const size_t BH = (size_t)gridDim.y * Hkv, bh = (size_t)b * Hkv + hk;
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
        if (sel_blocks && v[g] < max_sel) sel_blocks[((size_t)b * Hq + hk * G + g) * max_sel + v[g]] = blk;
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
        *reinterpret_cast<int4*>(wl + (v[G] + jj) * BH + bh) = make_int4(page0 + jj, blk, (int)w0, (int)w1);
      }
      v[G] += u;
    }
  }
  if (tid == 0) {
    const size_t o = (size_t)b * Hq + hk * G + c;
    n_sel[o] = all_tot[c];
    if (sel_blocks && all_tot[c] > max_sel) raise_err(err, kErrSelectOverflow);
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

// ============================================================================
// Register-resident variant for n_blocks <= 8192 (128K context at C = 32,
// Delta = 14), the decode-step configuration.  Same result as k_select, fewer
// dependent steps:
//  * thread t owns blocks i = k * 512 + t (k < 16): its keys and lengths stay
//    in registers through every pass, so each pass is 16 independent smem
//    operations instead of a dependent loop over smem;
//  * the block lengths, page-first table and histogram reset are done before
//    the PDL wait (they belong to the resident plan);
//  * a boundary bucket with <= 32 candidates is resolved by one warp ranking
//    them with shuffles (no sort); larger ones narrow the bucket and repeat;
//  * each head's selection is published as a bitmask (one ballot word per 32
//    blocks) pushed into every peer's smem by DSMEM stores before one cluster
//    barrier (no remote reads), then
//    every CTA computes the union page counts for all blocks (16 contiguous
//    blocks per thread, one block-wide scan) and writes 1/G of the worklist;
//    sel_blocks positions are popcount prefixes of the head's own bitmask;
//  * one split cluster barrier (arrive after the pushes, wait before the union).
// ============================================================================
constexpr int kRK = 16;
constexpr int kRMax = kSelNT * kRK;  // 8192 blocks
constexpr int kRW = kRMax / 32;      // 256 selection words per head
constexpr int kRC = 32;              // candidates ranked by one warp

DSK_DEVICE void cluster_arrive_rel() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
DSK_DEVICE void cluster_wait_acq() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// exclusive block-wide prefix of one int with a single __syncthreads; buf[kSelW]
// must not be reused until after the next block barrier.  Returns (exclusive, total).
DSK_DEVICE int2 cta_excl1(int v, int* buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int inc = warp_incl_scan(v);
  if (lane == 31) buf[warp] = inc;
  __syncthreads();
  int before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kSelW; ++w) {
    const int x = buf[w];
    before += w < warp ? x : 0;
    tot += x;
  }
  return make_int2(before + inc - v, tot);
}

// dynamic smem: slen[kRMax] u16 | spf[kRMax] i32 | skey0[kRMax] u32 | sbits[G][kRW] u32 | spre[kRW] i32
static size_t select_reg_smem_bytes(int G) {
  return (size_t)kRMax * 2 + (size_t)kRMax * 4 * 2 + (size_t)G * kRW * 4 + (size_t)kRW * 4;
}

// MINB = 2 (64 registers, a few spilled bytes) lets two CTAs share an SM:
// used when the launch has more CTAs than SMs (B Hkv G > SMs, e.g. 8 x 128K
// per GPU: one wave instead of two, 131.7 -> 121.3 us per layer); otherwise
// MINB = 1 (128 registers) is faster (B = 1: 32.4 vs 35.9 us per layer).
template <int G, int MINB>
__global__ void __launch_bounds__(kSelNT, MINB) k_select_reg(
    const float* __restrict__ scores, const int32_t* __restrict__ block_starts,
    const int32_t* __restrict__ n_blocks, const int32_t* __restrict__ page_first, int Hq, int Hkv,
    int maxb, int S, int max_sel, int max_wl, int Pshift, int budget, int blk_lo, int blk_hi,
    int32_t* __restrict__ sel_blocks, int32_t* __restrict__ n_sel, int32_t* __restrict__ marg_out,
    int32_t* __restrict__ keep_out, int32_t* __restrict__ wl_count, WLEntry* __restrict__ wl,
    int* __restrict__ err) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* slen = reinterpret_cast<uint16_t*>(smem);
  int32_t* spf = reinterpret_cast<int32_t*>(slen + kRMax);
  uint32_t* skey0 = reinterpret_cast<uint32_t*>(spf + kRMax);  // the head's keys (the narrowing passes kill entries of key[])
  uint32_t(*sbits)[kRW] = reinterpret_cast<uint32_t(*)[kRW]>(skey0 + kRMax);
  int32_t* spre = reinterpret_cast<int32_t*>(sbits[G]);
  __shared__ uint32_t HI[kBkt];
  __shared__ uint64_t CA[kRC];
  __shared__ int CL[kRC];
  __shared__ float red_f[2][kSelW];
  __shared__ int red_t[kSelW];
  __shared__ int scan_buf[2][kSelW];
  __shared__ int s_info[4];     // marginal, keep, threshold key, all_fit of this CTA's head
  __shared__ int s_pinfo[G][4]; // the same for every head of the cluster
  __shared__ int s_bnd, s_need, s_nc;

  const int c = (int)cluster.block_rank();
  const int hk = blockIdx.x / G, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = 1 << Pshift;
  const int nb_raw = n_blocks[b];
  const int nb = min(max(nb_raw, 0), min(maxb, kRMax));
  const int olo = min(max(blk_lo, 0), nb), ohi = max(min(blk_hi, nb), olo);
  const int32_t* bs = block_starts + (size_t)b * (maxb + 1);
  const int32_t* pf = page_first + (size_t)b * (maxb + 1);
  const float* sc = scores + ((size_t)b * Hq + hk * G + c) * maxb;

  stamp(0);
  // every CTA of the cluster must have started before a peer writes into its
  // shared memory (phase 3): arrive now, wait just before the pushes (by then
  // the whole cluster has long arrived, so the wait costs nothing)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  // ---- 0. resident plan (overlaps the preceding kernel under PDL)
  int len[kRK];
  int tsum = 0, npg = 0;
  // the plan must tile [0, L <= S); blocks beyond the 8/16-bit
  // counters (> 255 pages, > 65535 tokens) are rejected: such a sequence
  // selects nothing and the error word says why
  int bad = tid == 0 && (nb_raw < 1 || nb_raw > min(maxb, kRMax) || bs[0] != 0 || bs[nb] > S);
  int bad_long = 0;
#pragma unroll
  for (int k = 0; k < kRK; ++k) {
    const int i = k * kSelNT + tid;
    len[k] = 0;
    if (i < nb) {
      len[k] = bs[i + 1] - bs[i];
      spf[i] = pf[i];
      bad |= len[k] <= 0;
      bad_long |= len[k] > 0xffff || ((len[k] + P - 1) >> Pshift) > 255;
      npg += (len[k] + P - 1) >> Pshift;
    }
    slen[i] = (uint16_t)len[k];  // 0 beyond nb (the union pass reads whole words)
    tsum += len[k];
  }
  for (int j = tid; j < kBkt; j += kSelNT) HI[j] = 0;
  if (tid == 0) s_nc = 0;
  {
    npg = warp_sum_i(npg);
    if (lane == 0) red_t[warp] = npg;
    const int any_bad = __syncthreads_or(bad), any_long = __syncthreads_or(bad_long);
    int pages = 0;
#pragma unroll
    for (int w = 0; w < kSelW; ++w) pages += red_t[w];
    if (any_bad || any_long || pages > max_wl) {
      if (tid == 0) {
        raise_err(err, any_bad ? kErrPlanCoverage : any_long ? kErrBlockTooLong : kErrPageCapacity);
        const size_t o = (size_t)b * Hq + hk * G + c;
        n_sel[o] = 0;
        marg_out[o] = -1;
        keep_out[o] = 0;
        if (c == 0) wl_count[(size_t)b * Hkv + hk] = 0;
      }
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // match the arrive above
      return;
    }
    __syncthreads();  // red_t is reused by the threshold pass
  }
  stamp(1);
  pdl_trigger();
  pdl_wait();
  stamp(2);
  // ---- 1. keys of this CTA's head
  uint32_t key[kRK];
  // weak L1-allocating loads (ld.global.ca): the scores are the preceding
  // kernel's output, visible after the PDL wait, and no line of them was
  // cached by this launch before it.  (__ldcg compiled to strong LDG.STRONG.GPU
  // loads that ptxas issued one after another, ~2 us for the 16.)
  float sv[kRK];
#pragma unroll
  for (int k = 0; k < kRK; ++k) {
    const int i = k * kSelNT + tid;
    sv[k] = i < nb ? __ldca(sc + i) : 0.f;
  }
#pragma unroll
  for (int k = 0; k < kRK; ++k) {
    const int i = k * kSelNT + tid;
    key[k] = i < nb ? float_key(sv[k]) : 0u;
    skey0[i] = key[k];
#ifdef DSK_DEBUG
    if (k == 0) {  // debug timeline: latency of the first score load alone
      if (key[0] == 0x12345678u && g_sel_dbg) g_sel_dbg[0] = 0;
      stamp(10);
    }
#endif
  }
  stamp(3);

  // ---- 2. threshold: marginal block (index, keep) and its key
  int need = budget;
  bool first = true;
  for (;;) {
    float mn = CUDART_INF_F, mx = -CUDART_INF_F;
#pragma unroll
    for (int k = 0; k < kRK; ++k) {
      if (key[k]) {
        const float f = key_to_float(key[k]);
        mn = fminf(mn, f);
        mx = fmaxf(mx, f);
      }
    }
    mn = -warp_max(-mn);
    mx = warp_max(mx);
    const int ts = first ? warp_sum_i(tsum) : 0;
    if (lane == 0) {
      red_f[0][warp] = mn;
      red_f[1][warp] = mx;
      red_t[warp] = ts;
    }
    __syncthreads();
    int total = 0;
#pragma unroll
    for (int w = 0; w < kSelW; ++w) {
      mn = fminf(mn, red_f[0][w]);
      mx = fmaxf(mx, red_f[1][w]);
      total += red_t[w];
    }
    if (first && total <= budget) {
      if (tid == 0) {
        s_info[0] = -1;
        s_info[1] = 0;
        s_info[2] = 0;
        s_info[3] = 1;
      }
      break;
    }
    first = false;
    if (!(mx > mn)) {
      // every live key is equal: index order (i = k * 512 + t is chunk k, thread t)
      int carry = 0;
#pragma unroll 1
      for (int k = 0; k < kRK && carry < need; ++k) {
        int v = 0;
#pragma unroll
        for (int kk = 0; kk < kRK; ++kk)
          if (kk == k) v = key[kk] ? len[kk] : 0;
        const int2 pre = cta_excl1(v, scan_buf[k & 1]);
        const int before = carry + pre.x;
        if (v > 0 && before < need && before + v >= need) {
          uint32_t kk0 = 0;
#pragma unroll
          for (int kk = 0; kk < kRK; ++kk)
            if (kk == k) kk0 = key[kk];
          s_info[0] = k * kSelNT + tid;
          s_info[1] = need - before;
          s_info[2] = (int)kk0;
          s_info[3] = 0;
        }
        carry += pre.y;
      }
      break;
    }
    const float inv = (float)kBkt / (mx - mn);
#pragma unroll
    for (int k = 0; k < kRK; ++k)
      if (key[k]) atomicAdd(&HI[bucket_of(key[k], mn, inv)], (uint32_t)len[k]);
    __syncthreads();
    {  // suffix scan: thread tid owns buckets kBkt-1-4tid downwards
      const int j0 = kBkt - 1 - tid * kBPT;
      int h[kBPT], loc = 0;
#pragma unroll
      for (int k = 0; k < kBPT; ++k) {
        h[k] = (int)HI[j0 - k];
        loc += h[k];
      }
      int above = cta_excl1(loc, scan_buf[0]).x;
#pragma unroll
      for (int k = 0; k < kBPT; ++k) {
        if (above < need && above + h[k] >= need) {
          s_bnd = j0 - k;
          s_need = need - above;
        }
        above += h[k];
      }
    }
    __syncthreads();
    const int bnd = s_bnd;
    need = s_need;
#pragma unroll
    for (int k = 0; k < kRK; ++k) {
      if (key[k]) {
        if (bucket_of(key[k], mn, inv) == bnd) {
          const int p = atomicAdd(&s_nc, 1);
          if (p < kRC) {
            CA[p] = ((uint64_t)key[k] << 32) | (uint64_t)(0xffffffffu - (uint32_t)(k * kSelNT + tid));
            CL[p] = len[k];
          }
        } else {
          key[k] = 0;  // above (already counted in need) or below: no longer live
        }
      }
    }
    for (int j = tid; j < kBkt; j += kSelNT) HI[j] = 0;  // for a narrowing pass
    __syncthreads();
    const int nc = s_nc;
    __syncthreads();  // everyone has read s_nc
    if (nc > kRC) {
      if (tid == 0) s_nc = 0;
      continue;  // narrow to the boundary bucket
    }
    if (warp == 0) {
      // rank the candidates: order (key desc, index asc) == CA desc
      const uint64_t mine = lane < nc ? CA[lane] : 0ull;
      const int ml = lane < nc ? CL[lane] : 0;
      int before = 0;
      for (int j = 0; j < nc; ++j) {
        const uint64_t o = __shfl_sync(0xffffffffu, mine, j);
        const int ol = __shfl_sync(0xffffffffu, ml, j);
        before += (o > mine) ? ol : 0;
      }
      if (lane < nc && before < need && before + ml >= need) {
        s_info[0] = (int)(0xffffffffu - (uint32_t)(mine & 0xffffffffull));
        s_info[1] = need - before;
        s_info[2] = (int)(uint32_t)(mine >> 32);
        s_info[3] = 0;
      }
    }
    break;
  }
  __syncthreads();
  stamp(4);

  // ---- 3. this head's selection bitmask (ballot words), pushed into every
  //         peer's smem slot c (DSMEM stores) together with (marginal, keep,
  //         key, all_fit): after the cluster barrier each CTA holds all G
  //         selections locally (no remote reads, no second barrier)
  const int m_c = s_info[0], keep_c = s_info[1], all_c = s_info[3];
  const uint32_t T_c = (uint32_t)s_info[2];
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // all peers have started
  // lane g of each warp stores the words into CTA g's copy (g == c: local)
  uint32_t* const my_peer_bits = cluster.map_shared_rank(&sbits[c][0], lane < G ? lane : c);
#pragma unroll
  for (int k = 0; k < kRK; ++k) {
    const int i = k * kSelNT + tid;
    const uint32_t k0 = skey0[i];
    const bool sel = i < nb && (all_c || k0 > T_c || (k0 == T_c && i <= m_c));
    const uint32_t word = __ballot_sync(0xffffffffu, sel);
    if (lane < G) my_peer_bits[k * kSelW + warp] = word;
  }
  if (tid < G * 4) cluster.map_shared_rank(&s_pinfo[c][0], tid / 4)[tid % 4] = s_info[tid % 4];
  __syncthreads();
  cluster_arrive_rel();  // this CTA's pushes are released to the peers
  stamp(5);

  // ---- 4. sel_blocks of this head (ascending): popcount prefix over its words
  {
    const int x = tid < kRW ? __popc(sbits[c][tid]) : 0;
    const int2 pre = cta_excl1(x, scan_buf[1]);
    if (tid < kRW) spre[tid] = pre.x;
    __syncthreads();
    if (sel_blocks) {
      int32_t* out = sel_blocks + ((size_t)b * Hq + hk * G + c) * max_sel;
      const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
      for (int k = 0; k < kRK; ++k) {
        const uint32_t word = sbits[c][k * kSelW + warp];
        const int pos = spre[k * kSelW + warp] + __popc(word & lt);
        if (((word >> lane) & 1u) && pos < max_sel) out[pos] = k * kSelNT + tid;
      }
    }
    if (tid == 0) {
      const size_t o = (size_t)b * Hq + hk * G + c;
      n_sel[o] = pre.y;
      if (sel_blocks && pre.y > max_sel) raise_err(err, kErrSelectOverflow);
      marg_out[o] = all_c ? -1 : m_c;
      keep_out[o] = all_c ? 0 : keep_c;
    }
  }

  // ---- 5. every head's selection is in this CTA's smem; the union worklist
  cluster_wait_acq();  // the peers' pushes have landed
  stamp(6);
  int mg[G], kg[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    mg[g] = s_pinfo[g][3] ? -1 : s_pinfo[g][0];
    kg[g] = s_pinfo[g][1];
  }
  // thread tid: blocks [16 tid, 16 tid + 16) -> bits (tid & 1) * 16.. of word tid / 2
  const int blk0 = tid * kRK;
  uint32_t hb[G];
#pragma unroll
  for (int g = 0; g < G; ++g) hb[g] = (sbits[g][tid >> 1] >> ((tid & 1) * 16)) & 0xffffu;
  uint32_t anyb = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) anyb |= hb[g];
  // blocks outside the output range [olo, ohi) emit no worklist entries
  const int jlo = min(max(olo - blk0, 0), kRK), jhi = min(max(ohi - blk0, 0), kRK);
  anyb &= ((jhi >= 32 ? 0u : (1u << jhi)) - 1u) & ~((1u << jlo) - 1u);
  // union page count of block blk0 + j (rolled loops over the set bits only:
  // this kernel runs once per layer, so code size is latency)
  auto union_pages = [&](int j, int ln) {
    int u = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if ((hb[g] >> j) & 1u) {
        const int tk = blk0 + j == mg[g] ? kg[g] : ln;
        u = max(u, (tk + P - 1) >> Pshift);
      }
    }
    return u;
  };
  int tot_pages = 0;
#pragma unroll 1
  for (uint32_t bits = anyb; bits; bits &= bits - 1u) {
    const int j = __ffs(bits) - 1;
    tot_pages += union_pages(j, slen[blk0 + j]);
  }
  const int2 wpre = cta_excl1(tot_pages, scan_buf[0]);
  stamp(7);
  if ((tid % G) == c && tot_pages) {
    // interleaved layout: entry e of (b, KV head) bh at wl[e * B * Hkv + bh]
  const size_t BH = (size_t)gridDim.y * Hkv, bh = (size_t)b * Hkv + hk;
    const int pf_lo = olo < nb ? spf[olo] : 0;
    int v = wpre.x;
#pragma unroll 1
    for (uint32_t bits = anyb; bits; bits &= bits - 1u) {
      const int j = __ffs(bits) - 1;
      const int blk = blk0 + j, ln = slen[blk];
      const int u = union_pages(j, ln);
      const int page0 = spf[blk] - pf_lo;
#pragma unroll 1
      for (int jj = 0; jj < u; ++jj) {
        const int pv = min(P, ln - (jj << Pshift));
        uint32_t w0 = 0, w1 = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int tk = ((hb[g] >> j) & 1u) ? (blk == mg[g] ? kg[g] : ln) : 0;
          const uint32_t r = (uint32_t)min(max(tk - (jj << Pshift), 0), pv);
          if (g < 4) w0 |= r << (8 * g);
          else w1 |= r << (8 * (g - 4));
        }
        *reinterpret_cast<int4*>(wl + (v + jj) * BH + bh) = make_int4(page0 + jj, blk, (int)w0, (int)w1);
      }
      v += u;
    }
  }
  if (tid == 0 && c == 0) {
    if (hk == 0 && b == 0) {
      wl_count[-64] = 0x44534b57;  // "DSKW"
      wl_count[-63] = max_wl;
    }
    wl_count[(size_t)b * Hkv + hk] = wpre.y;
  }
  stamp(8);
  stamp(9);
}

}  // namespace dsk
extern "C" int dynsplit_debug_select_timer(void* dev_ptr) {
  return (int)cudaMemcpyToSymbol(dsk::g_sel_dbg, &dev_ptr, sizeof(void*));
}
// Test hook: 1 forces the generic k_select for every shape (parity of the two
// select kernels); 0 restores the default dispatch.  Initial value from
// DYNSPLIT_SELECT_GENERIC.
namespace dsk {
static volatile bool g_select_generic = getenv("DYNSPLIT_SELECT_GENERIC") != nullptr;
}
extern "C" int dynsplit_debug_select_generic(int on) {
  dsk::g_select_generic = on != 0;
  return 0;
}
namespace dsk {

size_t select_smem_needed(int maxb, int G) {
  const size_t s = select_smem_bytes(maxb, G);
  return s <= (size_t)max_smem_optin() - 8192 ? s : (size_t)-1;
}

template <int G>
static cudaError_t run_select(int B, int Hkv, size_t smem, const float* scores, const int32_t* bs,
                              const int32_t* nb, const int32_t* pf, int Hq, int maxb, int S, int max_sel,
                              int max_wl, int Pshift, int budget, int blk_lo, int blk_hi,
                              int32_t* sel_blocks, int32_t* n_sel, int32_t* marg, int32_t* keep,
                              int32_t* wl_count, WLEntry* wl, int* err, cudaStream_t st) {
  if (maxb <= kRMax && !g_select_generic) {
    auto kern = (size_t)B * Hkv * G > (size_t)num_sms() ? k_select_reg<G, 2> : k_select_reg<G, 1>;
    allow_max_dyn_smem(kern);
    launch_ex(kern, dim3(Hkv * G, B), dim3(kSelNT), select_reg_smem_bytes(G), st, G, scores,
              bs, nb, pf, Hq, Hkv, maxb, S, max_sel, max_wl, Pshift, budget, blk_lo, blk_hi, sel_blocks,
              n_sel, marg, keep, wl_count, wl, err);
    return post_launch("k_select_reg", st);
  }
  allow_max_dyn_smem(k_select<G>);
  launch_ex(k_select<G>, dim3(Hkv * G, B), dim3(kSelNT), smem, st, G, scores, bs, nb, pf, Hq, Hkv,
            maxb, S, max_sel, max_wl, Pshift, budget, blk_lo, blk_hi, sel_blocks, n_sel, marg, keep,
            wl_count, wl, err);
  return post_launch("k_select", st);
}

cudaError_t launch_select(int G, const float* scores, const int32_t* bs, const int32_t* nb,
                          const int32_t* pf, int B, int Hq, int Hkv, int maxb, int S, int max_sel,
                          int max_wl, int P, int budget, int blk_lo, int blk_hi,
                          int32_t* sel_blocks, int32_t* n_sel, int32_t* marg, int32_t* keep,
                          int32_t* wl_count, WLEntry* wl, int* err, cudaStream_t st) {
  const size_t smem = select_smem_needed(maxb, G);
  if (smem == (size_t)-1) return cudaErrorInvalidConfiguration;
  int Pshift = 0;
  while ((1 << Pshift) < P) ++Pshift;
#define DSK_SEL(GG)                                                                                \
  return run_select<GG>(B, Hkv, smem, scores, bs, nb, pf, Hq, maxb, S, max_sel, max_wl, Pshift,    \
                        budget, blk_lo, blk_hi, sel_blocks, n_sel, marg, keep, wl_count, wl, err, st)
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
