// Fused decode layer: rows a5 + a6 + a7 + a8 of one layer in ONE kernel
// (KV selection Steps 1-3: block scores, budgeted top-k through the
// block-to-token mapping P:257-264, sparse flash-decoding over the selected
// pages, split-K with the log-sum-exp merge).
//
// grid (NS, Hkv, B), 256 threads, one CTA per SM, every CTA resident at once
// (NS * Hkv * B <= SMs, checked by the launcher).  The NS CTAs of one
// (sequence b, KV head hk) -- a "group" -- cooperate through two group
// barriers in global memory (arrive = acq_rel atomic on a counter, the last
// arriver bumps a generation word with a release store; waiters poll the
// generation with acquire loads; a poll budget turns a barrier that can never
// complete into DYNSPLIT_DEVERR_SYNC_TIMEOUT instead of a hang):
//
//  prologue (resident inputs, overlaps the previous kernel under PDL): the
//    plan of sequence b (block lengths, page_first) into smem and validated
//    (S:267); the CTA's range of block digests (a multiple of 32 rows) into
//    smem by TMA tensor copies (64-dim x 32-row boxes, 128-byte swizzle).
//  1 (a5) after the PDL wait, q of the G heads; the range's block scores on
//    the tensor cores exactly as k_score_blocks_tc (256-term dot [q+ | q-] .
//    [kmax | kmin], bf16 products exact, fp32 accumulation in a fixed k
//    order -- identical scores); scores to global (rows padded to 32 floats
//    so no cache line is shared by two CTAs' ranges); per head the range's
//    count, sum and sum of squares of the scores.  Barrier A.
//  2 (a6) CTAs 0 .. min(G, NS)-1 select one query head each (CTA s: heads
//    s, s + NS, ...): the head's scores of all blocks in registers (32 per
//    thread), then the exact marginal block of the (score desc, index asc)
//    order (R13): a PREFILTER keeps the keys >= t_lo = mu + z sigma (mean and
//    deviation from the partial moments, z the normal quantile of twice the
//    budget's share of the tokens); when the kept blocks hold >= budget
//    tokens the marginal block is among them (the order lists every key >=
//    t_lo before any key below it), otherwise every key is kept; the kept
//    keys are bucketed into a length-weighted 1024-bucket histogram of
//    [min, max] (smem atomics cost ~2 cycles per lane, so the prefilter --
//    typically ~6 % of the blocks -- is what makes this cheap), the suffix
//    scan finds the boundary bucket, <= 32 candidates are ranked by one warp
//    (more: narrow to the bucket and repeat; equal keys: index order).  The
//    head's selection is published as a bitmask (one ballot word per 32
//    blocks) + (marginal, keep).  Barrier B.
//  3 every CTA forms the GQA union of the G bitmasks (thread t: blocks 32t ..
//    32t + 31), the union page counts (a head's rows of a block: all of them,
//    or `keep` leading rows of its marginal block; union = max over heads),
//    one block-wide scan, and deals itself the pages e = split (mod n_eff) in
//    block order into smem (also written to the worklist, the ABI output).
//  4 (a7, a8) attention over its pages and the split merge: attn_core.cuh,
//    the same code and page assignment as k_decode_attn, so o and lse equal
//    dynsplit_select + dynsplit_decode_attn bit for bit.
#include "attn_core.cuh"
#include "common.cuh"
#include "kernels.h"

#include <cudaTypedefs.h>
#include <math_constants.h>
#include <stdlib.h>

#include <atomic>

namespace dsk {

constexpr int kFNT = 256;            // threads per CTA
constexpr int kFNW = kFNT / 32;      // warps (all stream pages in phase 4)
constexpr int kFD = 2;               // pages in flight per warp
constexpr int kFKPT = 32;            // selection keys per thread
constexpr int kFMaxBlocks = kFNT * kFKPT;  // 8192 blocks per sequence (one bitmask word per thread)
constexpr int kFBkt = 1024;          // histogram buckets of the boundary search
constexpr int kFBPT = kFBkt / kFNT;  // buckets per thread in the suffix scan
constexpr int kFRC = 32;             // boundary candidates ranked by one warp
constexpr int kFBox = 32;            // digest rows per TMA box and per scoring-range granule
constexpr int kFSlabRowB = 128;      // bytes per row of one 64-dim digest slab
constexpr int kFMaxGroups = 1024;    // (b, KV head) groups x NS bound of the moment slots
constexpr int kBandCap = 512;        // the largest band list (kernel template BC: 256 or 512)
constexpr float kHiQ = 0.55f;        // t_hi = the (kHiQ budget / tokens) upper Gaussian quantile
constexpr int kSlot = kBandCap;      // band entries one CTA publishes per head (any range may hold the whole band)
constexpr int kSub = 16;             // sub-bands of [t_lo, t_hi] (per-range token weights)
constexpr int kH = 256;              // bins of a head's score histogram (the fallback of R25)

// Optional phase timestamps (debug builds; dynsplit_debug_fused_timer): the
// buffer pointer is read once per kernel into dbgp (a global load per stamp
// would add its latency to every phase).
__device__ unsigned long long* g_fused_dbg = nullptr;
// test switch (dynsplit_debug_fused_force): 1 = every head takes the
// histogram fallback, 2 = every head takes the CTA-wide slow path
__device__ int g_fused_force = 0;
#ifdef DSK_DEBUG
#define fstamp(k)                                                                                    \
  do {                                                                                               \
    if (dbgp && threadIdx.x == 0) {                                                                  \
      unsigned long long t_, c_;                                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                         \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_));                                             \
      const size_t cta_ = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;    \
      dbgp[cta_ * 64 + (k)] = t_;                                                                    \
      dbgp[cta_ * 64 + 16 + (k)] = c_;                                                               \
    }                                                                                                \
  } while (0)
// a %globaltimer stamp into debug slot 56 + k (thread 0 or lane 0 of a warp: any thread)
#define fstampx(k)                                                                                   \
  do {                                                                                               \
    if (dbgp) {                                                                                      \
      unsigned long long t_;                                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                         \
      const size_t cta_ = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;    \
      dbgp[cta_ * 64 + 56 + (k)] = t_;                                                               \
    }                                                                                                \
  } while (0)
// a value into debug slot 32 + k of this CTA (any thread)
#define fdbg(k, v)                                                                                   \
  do {                                                                                               \
    if (dbgp) {                                                                                      \
      const size_t cta_ = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;    \
      dbgp[cta_ * 64 + 32 + (k)] = (unsigned long long)(v);                                          \
    }                                                                                                \
  } while (0)
#define FSTAMP_INIT unsigned long long* const dbgp = g_fused_dbg
#else
#define fstamp(k) \
  do {            \
  } while (0)
#define fdbg(k, v) \
  do {             \
  } while (0)
#define fstampx(k) \
  do {             \
  } while (0)
#define FSTAMP_INIT
#endif

// ---------------------------------------------------------------- group barrier
DSK_DEVICE int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
DSK_DEVICE unsigned ld_relaxed_gpu_u(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
DSK_DEVICE unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
DSK_DEVICE void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
DSK_DEVICE int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Group barrier of the NS CTAs of one (b, KV head): kGbarWords zero-
// initialised words per group, [0] = the epoch of the last completed launch,
// [8 + s] = the flag of split s.  A launch reads the epoch after its PDL wait
// (the previous launch has completed), so its epoch is e = epoch + 1; a CTA
// arrives with one release store of e into its own flag (no atomic round
// trip); waiters poll the NS flags (one or two 128-byte lines, one lane per
// flag, acquire loads) until all hold e; split 0 then publishes epoch = e.
// Flags only grow, so a stale flag never equals e; splits >= NS of a launch
// with fewer splits are simply not read.
constexpr int kGbarWords = 8 + kMaxSplit;
DSK_DEVICE void gbar_arrive(unsigned* g, int split, unsigned e) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(g + 8 + split), "r"(e) : "memory");
}
// one warp; true when all NS flags hold e.  Relaxed polls, then one
// fence.acq_rel (the acquire pattern of the PTX memory model: a relaxed read
// that observes the release store, followed by the fence)
DSK_DEVICE bool gbar_wait_warp(const unsigned* g, int NS, unsigned e) {
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < (1 << 22); ++it) {
    bool ok = true;
    for (int r = lane; r < NS; r += 32) {
      unsigned v;
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(g + 8 + r) : "memory");
      ok &= v == e;
    }
    if (__all_sync(0xffffffffu, ok)) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      return true;
    }
  }
  return false;
}

// block-wide exclusive prefix of one int (kFNT threads); buf[kFNW] must not be
// reused before the next CTA barrier.  Returns (exclusive, total).
DSK_DEVICE int2 f_excl(int v, int* buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int inc = warp_incl_scan(v);
  if (lane == 31) buf[warp] = inc;
  __syncthreads();
  int before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kFNW; ++w) {
    const int x = buf[w];
    before += w < warp ? x : 0;
    tot += x;
  }
  return make_int2(before + inc - v, tot);
}

struct FusedScratch {  // static shared memory of the selection phase
  uint64_t CA[kFRC];
  int CL[kFRC];
  float redf[2][kFNW];
  int redi[kFNW];
  int scan[2][kFNW];
  int info[4];  // marginal, keep, threshold key, all_fit
  int bnd, need, nc;
  float tlo;
};

// length of block i from the staged block starts
DSK_DEVICE int blen(const int32_t* sbs, int i) { return sbs[i + 1] - sbs[i]; }

DSK_DEVICE int f_bucket(uint32_t k, float mn, float inv) {
  return min(max((int)((key_to_float(k) - mn) * inv), 0), kFBkt - 1);
}

// min / max (floats of the live keys) and the kept token weight, CTA-wide.
DSK_DEVICE void f_reduce3(const uint32_t (&key)[kFKPT], uint32_t live, const int32_t* sbs, FusedScratch& F,
                          float& mn, float& mx, int& w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  mn = CUDART_INF_F;
  mx = -CUDART_INF_F;
  w = 0;
#pragma unroll
  for (int k = 0; k < kFKPT; ++k) {
    if ((live >> k) & 1u) {
      const float f = key_to_float(key[k]);
      mn = fminf(mn, f);
      mx = fmaxf(mx, f);
      w += blen(sbs, k * kFNT + threadIdx.x);
    }
  }
  mn = -warp_max(-mn);
  mx = warp_max(mx);
  w = warp_sum_i(w);
  if (lane == 0) {
    F.redf[0][warp] = mn;
    F.redf[1][warp] = mx;
    F.redi[warp] = w;
  }
  __syncthreads();
  w = 0;
#pragma unroll
  for (int q = 0; q < kFNW; ++q) {
    mn = fminf(mn, F.redf[0][q]);
    mx = fmaxf(mx, F.redf[1][q]);
    w += F.redi[q];
  }
  __syncthreads();  // redf / redi are reused
}

// Exact marginal block of one head (R13): key[k] = order-preserving key of
// block k * kFNT + tid (0 = no block).  Writes F.info = {marginal, keep,
// threshold key, all_fit}.  All kFNT threads call it.
DSK_DEVICE void f_select_head(const uint32_t (&key)[kFKPT], const int32_t* sbs, int total, int budget,
                              float t_lo, uint32_t* hist, FusedScratch& F) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (total <= budget) {
    if (tid == 0) {
      F.info[0] = -1;
      F.info[1] = 0;
      F.info[2] = 0;
      F.info[3] = 1;
    }
    __syncthreads();
    return;
  }
  uint32_t valid = 0;
#pragma unroll
  for (int k = 0; k < kFKPT; ++k) valid |= key[k] ? (1u << k) : 0u;
  // prefilter: the keys >= t_lo, kept if they hold the budget
  const uint32_t klo = float_key(t_lo);
  uint32_t live = 0;
#pragma unroll
  for (int k = 0; k < kFKPT; ++k) live |= (key[k] && key[k] >= klo) ? (1u << k) : 0u;
  float mn, mx;
  int w;
  f_reduce3(key, live, sbs, F, mn, mx, w);
  int need = budget;
  if (w < need) {  // the prefilter would drop the marginal block: keep every key
    live = valid;
    f_reduce3(key, live, sbs, F, mn, mx, w);
  }
  for (;;) {
    if (!(mx > mn)) {
      // every live key is equal: index order (block i = k * kFNT + tid is chunk k, thread tid)
      int carry = 0;
#pragma unroll 1
      for (int k = 0; k < kFKPT && carry < need; ++k) {
        const int v = ((live >> k) & 1u) ? blen(sbs, k * kFNT + tid) : 0;
        const int2 pre = f_excl(v, F.scan[k & 1]);
        const int before = carry + pre.x;
        if (v > 0 && before < need && before + v >= need) {
          uint32_t kk0 = 0;
#pragma unroll
          for (int kk = 0; kk < kFKPT; ++kk)
            if (kk == k) kk0 = key[kk];
          F.info[0] = k * kFNT + tid;
          F.info[1] = need - before;
          F.info[2] = (int)kk0;
          F.info[3] = 0;
        }
        carry += pre.y;
      }
      break;
    }
    const float inv = (float)kFBkt / (mx - mn);
#pragma unroll
    for (int k = 0; k < kFKPT; ++k)
      if ((live >> k) & 1u) atomicAdd(&hist[f_bucket(key[k], mn, inv)], (uint32_t)blen(sbs, k * kFNT + tid));
    if (tid == 0) F.nc = 0;
    __syncthreads();
    {  // suffix scan: thread tid owns buckets kFBkt-1-kFBPT*tid downwards
      const int j0 = kFBkt - 1 - tid * kFBPT;
      int h[kFBPT], loc = 0;
#pragma unroll
      for (int k = 0; k < kFBPT; ++k) {
        h[k] = (int)hist[j0 - k];
        loc += h[k];
      }
      int above = f_excl(loc, F.scan[0]).x;
#pragma unroll
      for (int k = 0; k < kFBPT; ++k) {
        if (above < need && above + h[k] >= need) {
          F.bnd = j0 - k;
          F.need = need - above;
        }
        above += h[k];
      }
    }
    __syncthreads();
    const int bnd = F.bnd;
    need = F.need;
#pragma unroll
    for (int k = 0; k < kFKPT; ++k) {
      if ((live >> k) & 1u) {
        if (f_bucket(key[k], mn, inv) == bnd) {
          const int p = atomicAdd(&F.nc, 1);
          if (p < kFRC) {
            F.CA[p] = ((uint64_t)key[k] << 32) | (uint64_t)(0xffffffffu - (uint32_t)(k * kFNT + tid));
            F.CL[p] = blen(sbs, k * kFNT + tid);
          }
        } else {
          live &= ~(1u << k);  // above (already in need) or below: no longer live
        }
      }
    }
    for (int j = tid; j < kFBkt; j += kFNT) hist[j] = 0;  // clean for the next head / pass
    __syncthreads();
    const int nc = F.nc;
    if (nc > kFRC) {
      f_reduce3(key, live, sbs, F, mn, mx, w);
      continue;  // narrow to the boundary bucket
    }
    if (warp == 0) {
      // rank the candidates: order (key desc, index asc) == CA desc
      const uint64_t mine = lane < nc ? F.CA[lane] : 0ull;
      const int ml = lane < nc ? F.CL[lane] : 0;
      int before = 0;
      for (int j = 0; j < nc; ++j) {
        const uint64_t ot = __shfl_sync(0xffffffffu, mine, j);
        const int ol = __shfl_sync(0xffffffffu, ml, j);
        before += (ot > mine) ? ol : 0;
      }
      if (lane < nc && before < need && before + ml >= need) {
        F.info[0] = (int)(0xffffffffu - (uint32_t)(mine & 0xffffffffull));
        F.info[1] = need - before;
        F.info[2] = (int)(uint32_t)(mine >> 32);
        F.info[3] = 0;
      }
    }
    break;
  }
  __syncthreads();
}

template <int G>
struct SelScratch2 {  // static shared memory of the band selection
  float tlo[G], thi[G];
  int rwhi[kFNW][G], rwbd[kFNW][G];
  int bcnt[G];
  int wsub[G * kSub];
  int4 sel[G];  // marginal, keep, threshold key, flags (1 = all fit, 2 = slow path)
  float gmn[G], kb[G];  // bin map of the fallback: bin(x) = min(floor((x - gmn) kb), kH - 1)
};

// One warp: the marginal block of a head inside its band (c <= kBandCap
// entries (key, block | sub-band << 24) with key in [t_lo, t_hi]), where
// `need` tokens of the band are still to be taken in the order (key desc,
// block asc).  Lane l holds entries l + 32 r; lane j < kSub holds wsb, the
// token weight of sub-band j (summed over the group's ranges).  A suffix scan
// of the sub-band weights gives the sub-band where `need` is reached (the
// sub-bands above it are taken whole); its entries stay live.  While more than
// 32 are live, the live key range [lo, hi] is cut again into 16 sub-bands by
// a monotone integer map (umulhi(key - lo, scale)) and 16 warp reductions; <=
// 32 live entries are ranked exactly against each other (all pairs by
// shuffles, order (key desc, block asc)); equal keys across more than 32
// entries are taken in block order.  Returns the marginal block m, its kept
// tokens and its key T, and sets the selection bits of the band's selected
// blocks (bits: the head's words).
// Returns (m, keep, T).  (Inlined: a noinline copy measured 0.6 us slower per
// layer.)
template <int BC>
DSK_DEVICE int4 f_band_select(uint2* band, int c, int wsb, const int32_t* sbs, int need,
                                           uint32_t* bits) {
  const int lane = threadIdx.x & 31;
  int m, keep;
  uint32_t T;
  constexpr int J = BC / 32;
  uint32_t k[J], sbr[J];
  int ix[J], ln[J];
  uint32_t valid = 0;
  {
    uint2 v[J];
#pragma unroll
    for (int r = 0; r < J; ++r) v[r] = lane + 32 * r < c ? band[lane + 32 * r] : make_uint2(0u, 0u);
#pragma unroll
    for (int r = 0; r < J; ++r) {
      const bool ok = lane + 32 * r < c;
      k[r] = v[r].x;
      ix[r] = (int)(v[r].y & 0xffffffu);
      sbr[r] = v[r].y >> 24;
      ln[r] = ok ? blen(sbs, ix[r]) : 0;
      valid |= ok ? 1u << r : 0u;
    }
  }
  // the published sub-band weights: suffix scan from the top sub-band
  int nr0 = need;
  uint32_t live = 0;
  {
    int suf = lane < kSub ? wsb : 0;
#pragma unroll
    for (int o = 1; o < kSub; o <<= 1) {
      const int t = __shfl_down_sync(0xffffffffu, suf, o);
      if (lane + o < kSub) suf += t;
    }
    const uint32_t reach = __ballot_sync(0xffffffffu, lane < kSub && suf >= need);
    const int sstar = reach ? 31 - __clz(reach) : 0;
    nr0 = need - __shfl_sync(0xffffffffu, suf - wsb, sstar);
#pragma unroll
    for (int r = 0; r < J; ++r)
      if (((valid >> r) & 1u) && sbr[r] == (uint32_t)sstar) live |= 1u << r;
  }
  int nr = nr0;
  m = -1;
  keep = 0;
  T = 0;
#pragma unroll 1
  for (int round = 0; round < 8; ++round) {
    uint32_t lo = 0xffffffffu, hi = 0u;
    int nl = 0;
#pragma unroll
    for (int r = 0; r < J; ++r)
      if ((live >> r) & 1u) {
        lo = min(lo, k[r]);
        hi = max(hi, k[r]);
        ++nl;
      }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    nl = __reduce_add_sync(0xffffffffu, nl);
    if (nl <= 32 || lo == hi) {
      // exact rank of the live entries: compact them to one per lane (through
      // this head's band list, no longer needed), then all pairs
      int pos = 0;
      {
        int mine = __popc(live);
        const int incl = warp_incl_scan(mine);
        pos = incl - mine;
      }
      __syncwarp();
      if (nl <= 32) {
#pragma unroll
        for (int r = 0; r < J; ++r)
          if ((live >> r) & 1u) band[pos++] = make_uint2(k[r], (uint32_t)ix[r]);  // (sub-band bits dropped)
        __syncwarp();
        const uint2 e = lane < nl ? band[lane] : make_uint2(0u, 0u);
        const int el = lane < nl ? blen(sbs, (int)e.y) : 0;
        int before = 0;
        for (int j2 = 0; j2 < nl; ++j2) {
          const uint32_t ok2 = __shfl_sync(0xffffffffu, e.x, j2), oi = __shfl_sync(0xffffffffu, e.y, j2);
          const int ol = __shfl_sync(0xffffffffu, el, j2);
          before += (ok2 > e.x || (ok2 == e.x && oi < e.y)) ? ol : 0;
        }
        const uint32_t hit = __ballot_sync(0xffffffffu, lane < nl && before < nr && before + el >= nr);
        const int src = hit ? __ffs(hit) - 1 : 0;
        m = (int)__shfl_sync(0xffffffffu, e.y, src);
        T = __shfl_sync(0xffffffffu, e.x, src);
        keep = nr - __shfl_sync(0xffffffffu, before, src);
        if (!hit) m = -1;  // cannot happen when the band holds the marginal block
      } else {
        // more than 32 entries with one key: block order
        T = lo;
        uint32_t taken = 0;
#pragma unroll 1
        for (int it = 0; it < BC; ++it) {
          uint32_t mi = 0xffffffffu;
#pragma unroll
          for (int r = 0; r < J; ++r)
            if (((live & ~taken) >> r) & 1u) mi = min(mi, (uint32_t)ix[r]);
          mi = __reduce_min_sync(0xffffffffu, mi);
          if (mi == 0xffffffffu) break;
          int l = 0;
#pragma unroll
          for (int r = 0; r < J; ++r)
            if (((live & ~taken) >> r) & 1u && (uint32_t)ix[r] == mi) {
              l = ln[r];
              taken |= 1u << r;
            }
          l = __reduce_add_sync(0xffffffffu, l);
          if (l >= nr) {
            m = (int)mi;
            keep = nr;
            break;
          }
          nr -= l;
        }
      }
      break;
    }
    // 16 sub-bands of [lo, hi]: sb = floor((key - lo) * scale / 2^32) < 16
    const uint64_t span = (uint64_t)(hi - lo) + 1u;
    const uint64_t sc64 = (((uint64_t)16 << 32) / span) - 1u;
    const uint32_t scale = sc64 > 0xffffffffull ? 0xffffffffu : (uint32_t)sc64;  // (rare path: 64-bit division)
    uint32_t sbq[J];
#pragma unroll
    for (int r = 0; r < J; ++r) sbq[r] = __umulhi(k[r] - lo, scale);
    int wsb = 0;  // lane j < 16: token weight of sub-band j
#pragma unroll 1
    for (int j2 = 0; j2 < 16; ++j2) {
      int w = 0;
#pragma unroll
      for (int r = 0; r < J; ++r) w += (((live >> r) & 1u) && sbq[r] == (uint32_t)j2) ? ln[r] : 0;
      w = __reduce_add_sync(0xffffffffu, w);
      if (lane == j2) wsb = w;
    }
    // suffix scan from sub-band 15 down: the first sub-band where need is reached
    int suf = lane < 16 ? wsb : 0;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const int t = __shfl_down_sync(0xffffffffu, suf, o);
      if (lane + o < 16) suf += t;
    }
    const uint32_t reach = __ballot_sync(0xffffffffu, lane < 16 && suf >= nr);
    const int sstar = 31 - __clz(reach);  // the highest sub-band whose suffix reaches need
    const int above = __shfl_sync(0xffffffffu, suf - wsb, sstar);
    nr -= above;
#pragma unroll
    for (int r = 0; r < J; ++r)
      if (sbq[r] != (uint32_t)sstar) live &= ~(1u << r);
  }
  // selection bits of the band's selected blocks (the blocks above t_hi are set already)
#pragma unroll
  for (int r = 0; r < J; ++r)
    if (((valid >> r) & 1u) && (k[r] > T || (k[r] == T && ix[r] <= m)))
      atomicOr(&bits[ix[r] >> 5], 1u << (ix[r] & 31));
  return make_int4(m, keep, (int)T, 0);
}

template <int G, int BC>
__global__ void __launch_bounds__(kFNT, 1) k_decode_fused(
    const __grid_constant__ CUtensorMap tmD, const bf16* __restrict__ q,
    const int32_t* __restrict__ block_starts, const int32_t* __restrict__ n_blocks,
    const int32_t* __restrict__ page_first, const bf16* __restrict__ Kp, const bf16* __restrict__ Vp, int Hq,
    int Hkv, int maxb, int max_pages, int S, int Pshift, int budget, int gqa_mode, int budget_mode, int cap, int cap2,
    int ent_cap, int nwords,
    int sstride, size_t region_a, int per_cap, int local_sel, float scale_log2, float* __restrict__ scores,
    unsigned long long* __restrict__ mom, int4* __restrict__ cls_w, int* __restrict__ cls_sub, uint2* __restrict__ cls_band,
    uint32_t* __restrict__ gbits,
    int* __restrict__ counters, unsigned* __restrict__ gbar, float* __restrict__ part_o,
    float* __restrict__ part_lse, int32_t* __restrict__ n_sel_out, int32_t* __restrict__ marg_out,
    int32_t* __restrict__ keep_out, int32_t* __restrict__ wl_count, WLEntry* __restrict__ wl,
    float* __restrict__ o, float* __restrict__ lse, int* __restrict__ err) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t barD[2], bar2, bar_plan;
  __shared__ FusedScratch F;
  __shared__ SelScratch2<G> S2;
  __shared__ float4 red_m[kFNW][8];
  __shared__ unsigned s_target, s_pref;
  __shared__ int s_last;

  const uint32_t raw_s = smem_u32(smem_raw);
  unsigned char* smA = smem_raw + (((raw_s + 1023u) & ~1023u) - raw_s);  // region A (1024-aligned)
  const int nw32 = nwords * 32;
  int32_t* sbs_st = reinterpret_cast<int32_t*>(smA + region_a);  // [nw32 + 8] staged block starts
  int32_t* spf_st = sbs_st + nw32 + 8;                            // [nw32 + 8] staged page_first
  int4* s_ent = reinterpret_cast<int4*>(spf_st + nw32 + 8);       // [ent_cap] this split's pages
  bf16* s_q = reinterpret_cast<bf16*>(s_ent + ent_cap);           // [G][kD]
  uint32_t(*s_rows)[2] = reinterpret_cast<uint32_t(*)[2]>(s_q + G * kD);
  float* ssl = reinterpret_cast<float*>(s_rows + kFNW * kFD);    // [G][per_cap] this range's scores
  // region A in phases 2-3: histogram | band entries | selection words
  uint32_t* hist = reinterpret_cast<uint32_t*>(smA);                         // [kFBkt] (slow path)
  uint2* sband = reinterpret_cast<uint2*>(hist + kFBkt);                     // [G][BC]
  uint32_t* sbits = reinterpret_cast<uint32_t*>(sband + G * BC);       // [G][nwords] selection words

  const int split = blockIdx.x, hk = blockIdx.y, b = blockIdx.z, NS = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bh = b * Hkv + hk;
  const int P = 1 << Pshift;
  const int nb_raw = n_blocks[b];
  const int nb = min(max(nb_raw, 0), min(maxb, nw32));
  const int nwu = (nb + 31) >> 5;  // selection words in use
  FSTAMP_INIT;
  const int force = g_fused_force;
  fstamp(0);

  // ---- prologue (resident inputs; overlaps the preceding kernel under PDL):
  //      the plan rows (block_starts, page_first) and this CTA's range of
  //      digests into smem by TMA
  const int per = (((nb + NS - 1) / NS) + kFBox - 1) & ~(kFBox - 1);
  const int lo = min(nb, split * per), hi = min(nb, lo + per), n = hi - lo;
  // digest staging: one buffer of `cap` rows when the range fits it, else two
  // buffers of `cap2` rows (the next round loads while this one is scored)
  const bool dbl = n > cap;
  const int rows = dbl ? cap2 : cap;
  const size_t slab = (size_t)rows * kFSlabRowB;
  const int row0 = bh * maxb + lo;
  auto stage = [&](int r0, int cnt, int buf) {  // rows r0 .. r0 + cnt of the range -> buffer buf
    if (tid == 0) {
      const int nbox = (cnt + kFBox - 1) / kFBox;
      unsigned char* base = smA + (size_t)buf * 4 * slab;
      mbar_arrive_expect_tx(&barD[buf], (uint32_t)(nbox * 4 * kFBox * kFSlabRowB));
      for (int j = 0; j < nbox; ++j)
#pragma unroll
        for (int sl = 0; sl < 4; ++sl)
          tma_load_2d(base + sl * slab + (size_t)j * kFBox * kFSlabRowB, &tmD, sl * 64, row0 + r0 + j * kFBox,
                      &barD[buf]);
    }
  };
  // a plan row is copied from its 16-byte aligned-down start (skip ints),
  // capped at the end of the array (the last row's tail is read directly)
  const int32_t* bs_row = block_starts + (size_t)b * (maxb + 1);
  const int32_t* pf_row = page_first + (size_t)b * (maxb + 1);
  const int32_t* arr_end_bs = block_starts + (size_t)gridDim.z * (maxb + 1);
  const int32_t* arr_end_pf = page_first + (size_t)gridDim.z * (maxb + 1);
  const int skip_bs = (int)((reinterpret_cast<uintptr_t>(bs_row) & 15u) >> 2);
  const int skip_pf = (int)((reinterpret_cast<uintptr_t>(pf_row) & 15u) >> 2);
  auto row_bytes = [&](const int32_t* row, int skip, int count, const int32_t* end) {
    const int32_t* al = row - skip;
    uint32_t bytes = (uint32_t)(((skip + count) * 4 + 15) & ~15);
    const size_t room = (size_t)(end - al) * 4;
    if (bytes > room) bytes = (uint32_t)(room & ~(size_t)15);
    return bytes;
  };
  const uint32_t bs_bytes = row_bytes(bs_row, skip_bs, nb + 1, arr_end_bs);
  const uint32_t pf_bytes = row_bytes(pf_row, skip_pf, nb, arr_end_pf);
  if (tid == 0) {
    mbar_init(&barD[0], 1);
    mbar_init(&barD[1], 1);
    mbar_init(&bar2, 1);
    mbar_init(&bar_plan, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bar_plan, bs_bytes + pf_bytes);
    if (bs_bytes) bulk_g2s(sbs_st, bs_row - skip_bs, bs_bytes, &bar_plan, policy_evict_last());
    if (pf_bytes) bulk_g2s(spf_st, pf_row - skip_pf, pf_bytes, &bar_plan, policy_evict_last());
  }
  if (n > 0) {
    stage(0, min(rows, n), 0);
    if (dbl) stage(rows, min(rows, n - rows), 1);
  }
  int32_t* sbs = sbs_st + skip_bs;
  int32_t* spf = spf_st + skip_pf;
  // the barriers' initialisation must be visible before any thread polls one:
  // a stale word left in this smem by an earlier kernel can otherwise read as
  // a completed phase (the plan is then read before it lands)
  __syncthreads();
  mbar_wait(&bar_plan, 0);
  // entries past the bulk copies (the last row near the array end): direct loads
  for (int i = (int)(bs_bytes >> 2) - skip_bs + tid; i <= nb; i += kFNT) sbs[i] = bs_row[i];
  for (int i = (int)(pf_bytes >> 2) - skip_pf + tid; i < nb; i += kFNT) spf[i] = pf_row[i];
  __syncthreads();
  for (int i = nb + 1 + tid; i <= nwu * 32; i += kFNT) sbs[i] = sbs[nb];  // blocks past nb: length 0
  __syncthreads();
  // validation: the plan must tile [0, L <= S); blocks beyond the
  // 8/16-bit counters (> 255 pages, > 65535 tokens) are rejected
  int bad = tid == 0 && (nb_raw < 1 || nb_raw > min(maxb, nw32) || sbs[0] != 0 || sbs[nb] > S);
  int bad_long = 0, npg = 0;
#pragma unroll 4
  for (int i = tid; i < nb; i += kFNT) {
    const int len = blen(sbs, i);
    bad |= len <= 0;
    bad_long |= len > 0xffff || ((len + P - 1) >> Pshift) > 255;
    npg += (len + P - 1) >> Pshift;
  }
  for (int j = tid; j < G * kSub; j += kFNT) S2.wsub[j] = 0;
  const int any_bad = __syncthreads_or(bad), any_long = __syncthreads_or(bad_long);
  {
    const int c = warp_sum_i(npg);
    if (lane == 0) F.scan[1][warp] = c;
  }
  __syncthreads();
  const int total = nb > 0 ? sbs[nb] - sbs[0] : 0;
  int pages = 0;
#pragma unroll
  for (int w = 0; w < kFNW; ++w) pages += F.scan[1][w];
  const bool skip = any_bad || any_long || pages > max_pages;
  fstamp(1);
  pdl_trigger();
  pdl_wait();  // q, the scores/worklist buffers and the outputs belong to the step
  if (tid == 0) {
    s_target = ld_relaxed_gpu_u(gbar + (size_t)bh * kGbarWords) + 1u;
    // word 1: launches left to run the local selection after a fast-path miss
    s_pref = ld_relaxed_gpu_u(gbar + (size_t)bh * kGbarWords + 1);
  }
  fstamp(2);
  if (skip) {
    if (tid == 0 && split == 0) {
      raise_err(err, any_bad ? kErrPlanCoverage : any_long ? kErrBlockTooLong : kErrPageCapacity);
      for (int g = 0; g < G; ++g) {
        const size_t oh = (size_t)b * Hq + hk * G + g;
        n_sel_out[oh] = 0;
        marg_out[oh] = -1;
        keep_out[oh] = 0;
      }
      wl_count[bh] = 0;
    }
    if (n > 0) mbar_wait(&barD[0], 0);  // the staging must land before region A is reused
    if (dbl) mbar_wait(&barD[1], 0);
    if (split != 0) return;
    // no pages: o = 0 and lse = -inf for the G heads (as the unfused path)
    attn_bf16_pipeline<G, kFNW, kFD>(smA, s_rows, s_q, 1, P, 0, [](int, int&, uint32_t&, uint32_t&) {}, Kp, Vp,
                                     (size_t)bh, max_pages, scale_log2, true);
    attn_merge_out<G, kFNW>(reinterpret_cast<float*>(smA), &s_last, b, hk, Hq, 0, 1, NS, (size_t)bh, part_o,
                            part_lse, counters, o, lse);
    return;
  }

  // ---- 1. (a5) q -> smem; block scores of the range on the tensor cores
  if (tid < G * kD * 2 / 16)
    reinterpret_cast<uint4*>(s_q)[tid] =
        __ldca(reinterpret_cast<const uint4*>(q + ((size_t)b * Hq + hk * G) * kD) + tid);
  __syncthreads();
  // local selection: by the launcher's rule (bit 0), or -- adaptively (bit
  // 1) -- for a few launches after one where the moment bounds missed for a
  // head of this group (the same word for every CTA of the group: uniform)
  const bool lsel = (local_sel & 1) || ((local_sel & 2) && s_pref != 0u && !force);
  fstamp(14);
  {
    const int g = lane >> 2, t = lane & 3;
    uint32_t a0[16], a2[16];
    {
      uint32_t w0[8], w2[8];  // q_g[16 i + 2t .. +1], q_g[16 i + 2t + 8 .. +9], i < 8
#pragma unroll
      for (int i = 0; i < 8; ++i) w0[i] = w2[i] = 0u;
      if (g < G) {
        const uint32_t* qg = reinterpret_cast<const uint32_t*>(s_q + (size_t)g * kD);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          w0[i] = qg[8 * i + t];
          w2[i] = qg[8 * i + t + 4];
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
    float s1 = 0.f, s2 = 0.f;  // this lane's sum / sum of squares of head g's scores
    float mn = CUDART_INF_F, mx = -CUDART_INF_F;  // and their range
    float* srow_g = scores + ((size_t)b * Hq + hk * G + g) * sstride + lo;
    const int lr = lane & 7, lc = lane >> 3;
    const uint32_t sbase_u = smem_u32(smA);
    int rd = 0;
    for (int r0 = 0; r0 < n; r0 += rows, ++rd) {
      const int c_n = min(rows, n - r0);
      const int buf = dbl ? (rd & 1) : 0;
      mbar_wait(&barD[buf], dbl ? ((rd >> 1) & 1u) : (rd & 1u));
      if (r0 == 0) fstamp(15);
      const uint32_t sbuf_u = sbase_u + (uint32_t)((size_t)buf * 4 * slab);
      for (int grp = warp; grp * 8 < c_n; grp += kFNW) {
        float c[4] = {0.f, 0.f, 0.f, 0.f};
        const int r = grp * 8 + lr;
        const uint32_t rowa = sbuf_u + (uint32_t)(r * kFSlabRowB);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // two k-steps (32 dims) per ldmatrix.x4
          const uint32_t chunk = (uint32_t)((((kk & 1) << 2) | lc) ^ (r & 7));
          uint32_t bk[4];
          ldsm_x4(bk, rowa + (uint32_t)((kk >> 1) * slab) + (chunk << 4));
          mma_rows8(c, a0[2 * kk], a2[2 * kk], bk[0], bk[1]);
          mma_rows8(c, a0[2 * kk + 1], a2[2 * kk + 1], bk[2], bk[3]);
        }
        // c0, c1: head g, blocks grp * 8 + 2t, + 1 (rows 8..15 are zero)
        if (gqa_mode) {
          // group-shared selection (R23): every head of the group gets the sum
          // of the G heads' scores (lanes 4g + t; rows >= G are zero), a fixed
          // butterfly, so every CTA and every head holds the same fp32 value
#pragma unroll
          for (int o2 = 4; o2 < 32; o2 <<= 1) {
            c[0] += __shfl_xor_sync(0xffffffffu, c[0], o2);
            c[1] += __shfl_xor_sync(0xffffffffu, c[1], o2);
          }
        }
        const int i0 = r0 + grp * 8 + 2 * t;
        if (g < G) {
          if (i0 < n) {
            srow_g[i0] = c[0];
            ssl[g * per_cap + i0] = c[0];
            s1 += c[0];
            s2 = fmaf(c[0], c[0], s2);
            mn = fminf(mn, c[0]);
            mx = fmaxf(mx, c[0]);
          }
          if (i0 + 1 < n) {
            srow_g[i0 + 1] = c[1];
            ssl[g * per_cap + i0 + 1] = c[1];
            s1 += c[1];
            s2 = fmaf(c[1], c[1], s2);
            mn = fminf(mn, c[1]);
            mx = fmaxf(mx, c[1]);
          }
        }
      }
      // this buffer takes the round after next (two buffers) or the next one (one)
      const int nxt = r0 + (dbl ? 2 : 1) * rows;
      if (nxt < n) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads before the async-proxy writes
        __syncthreads();                                                // every warp is done with the buffer
        stage(nxt, min(rows, n - nxt), buf);
      }
    }
    // the range's moments per head (fixed order: lanes, then warps)
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (t == 0 && g < G) red_m[warp][g] = make_float4(s1, s2, mn, mx);
  }
  __syncthreads();
  if (tid < G) {
    float a = 0.f, c2 = 0.f, mn = CUDART_INF_F, mx = -CUDART_INF_F;
    for (int w = 0; w < kFNW; ++w) {
      const float4 r = red_m[w][tid];
      a += r.x;
      c2 += r.y;
      mn = fminf(mn, r.z);
      mx = fmaxf(mx, r.w);
    }
    // barrier A is the moments themselves: each value goes out as one 64-bit
    // word tagged with the launch's epoch (single-copy atomic), so a reader
    // that sees the tag sees the value -- no flag and no second round trip
    const unsigned long long tag = (unsigned long long)s_target << 32;
    unsigned long long* mw = mom + (((size_t)bh * NS + split) * G + tid) * 4;
    // local selection reads every CTA's scores right after barrier A: the
    // CTA's score stores (ordered by the barrier above) are released first
    if (lsel) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    st_relaxed_u64(mw + 0, tag | __float_as_uint(a));
    st_relaxed_u64(mw + 1, tag | __float_as_uint(c2));
    st_relaxed_u64(mw + 2, tag | __float_as_uint(mn));
    st_relaxed_u64(mw + 3, tag | __float_as_uint(mx));
  }
  __syncthreads();  // (the scores this CTA wrote to global are read only after barrier B)
  fstamp(3);

  // ---- 2. (a6) selection, distributed over the group's CTAs.  After
  //      barrier A (every range's moments published) each CTA derives the
  //      same per-head bounds t_lo < t_hi and classifies ITS range: the words
  //      of blocks above t_hi (surely selected), the token weights above and
  //      in the band [t_lo, t_hi] and the band entries, all published; after
  //      barrier B every CTA gathers them and resolves each head's marginal
  //      block inside the band (exact, f_band_select), or -- when the bounds
  //      do not bracket it -- over every score of the head (slow path).
  unsigned* gb = gbar + (size_t)bh * kGbarWords;
  // bounds per head from the group's moments (fixed order); keys above t_hi
  // are surely selected, the marginal block lies in [t_lo, t_hi] when the
  // published weights verify it.  Warp g polls head g's NS tagged records
  // until every tag is this launch's epoch (barrier A).
  if (warp < G) {
    const int g2 = warp;
    float c1 = 0.f, c2 = 0.f, gmn = CUDART_INF_F, gmx = -CUDART_INF_F;
    const unsigned e = s_target;
    bool done = false;
    for (int it = 0; it < (1 << 22) && !done; ++it) {
      float x1 = 0.f, x2 = 0.f, xn = CUDART_INF_F, xx = -CUDART_INF_F;
      bool ok = true;
      for (int r = lane; r < NS; r += 32) {
        const unsigned long long* mw = mom + (((size_t)bh * NS + r) * G + g2) * 4;
        const unsigned long long w0 = ld_relaxed_u64(mw), w1 = ld_relaxed_u64(mw + 1);
        const unsigned long long w2 = ld_relaxed_u64(mw + 2), w3 = ld_relaxed_u64(mw + 3);
        ok &= (unsigned)(w0 >> 32) == e && (unsigned)(w1 >> 32) == e && (unsigned)(w2 >> 32) == e &&
              (unsigned)(w3 >> 32) == e;
        x1 += __uint_as_float((unsigned)w0);
        x2 += __uint_as_float((unsigned)w1);
        xn = fminf(xn, __uint_as_float((unsigned)w2));
        xx = fmaxf(xx, __uint_as_float((unsigned)w3));
      }
      if (__all_sync(0xffffffffu, ok)) {
        done = true;
        c1 = x1;
        c2 = x2;
        gmn = xn;
        gmx = xx;
      }
    }
    if (!done && lane == 0) raise_err(err, kErrSyncTimeout);
    if (lsel) asm volatile("fence.acq_rel.gpu;" ::: "memory");  // the peers' scores, for the local selection
    c1 = warp_sum(c1);
    c2 = warp_sum(c2);
    gmn = -warp_max(-gmn);
    gmx = warp_max(gmx);
    if (lane == 0) {
      const float cn = (float)nb;
      float kb = (float)kH / (gmx - gmn);  // the fallback's bin map over [gmin, gmax]
      if (!(kb < 3.0e38f)) kb = 0.f;       // equal scores (or an overflowing span): one bin
      S2.gmn[g2] = gmn;
      S2.kb[g2] = kb;
      float tl = -CUDART_INF_F, th = CUDART_INF_F;
      const float pb = (float)budget / (float)max(total, 1);
      if (cn > 1.f && pb < 0.25f) {
        const float mu = c1 / cn, var = fmaxf(c2 / cn - mu * mu, 0.f), sd = sqrtf(var);
        if (sd > 0.f) {
          // lower bound: the 1.8 p upper quantile, or p + 40 blocks' worth when
          // the budget is only a few dozen blocks (the far tail of block
          // scores is thinner than the normal one; budget 1024 at 128K
          // otherwise misses W(x >= t_lo) >= budget for some heads)
          tl = mu + sd * normcdfinvf(1.f - fminf(0.45f, fmaxf(1.8f * pb, pb + 40.f / cn)));
          th = mu + sd * normcdfinvf(1.f - kHiQ * pb);
        }
      }
      S2.tlo[g2] = tl;
      S2.thi[g2] = th;
      S2.bcnt[g2] = 0;
    }
  }
  __syncthreads();
  fstamp(4);
  if (lsel) {
    // Local selection (short sequences, few blocks per head): after barrier A
    // every CTA selects every head itself from the full score rows -- the
    // exact histogram path below, the same data and arithmetic in every CTA
    // of the group -- instead of the distributed classification and barrier
    // B (faster for short sequences over few splits, see the launcher).  Every CTA has
    // read the epoch before publishing its moments: publish it now.
    if (tid < G) S2.sel[tid] = make_int4(-1, 0, 0, total <= budget ? 1 : 2);
    if (tid == 0 && split == 0)
      asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(gb), "r"(s_target) : "memory");
  } else {
  if (tid == 0) fstampx(4);
  // classification of this CTA's range: warp w takes head g = w % G and the
  // range's words w / G, w / G + 8 / G, ...; lane l is block lo + 32 word + l.
  // A band entry also gets its sub-band sb = floor(16 (x - t_lo) / (t_hi -
  // t_lo)) clamped to [0, 16) -- monotone in x, the same map in every CTA --
  // and the range's token weight per (head, sub-band) is published.
  {
    const int g2 = warp % G;
    const float tl = S2.tlo[g2], th = S2.thi[g2];
    const float sbk = (float)kSub / (th - tl);
    const int nws = (n + 31) >> 5;
    int whi = 0, wbd = 0;
    const uint32_t lt = (1u << lane) - 1u;
    uint2* myband = cls_band + (((size_t)bh * NS + split) * G + g2) * kSlot;
#pragma unroll 1
    for (int wl = warp / G; wl < nws; wl += kFNW / G) {
      const int il = wl * 32 + lane, i = lo + il;
      const bool ok = il < n;
      const float x = ok ? ssl[g2 * per_cap + il] : -CUDART_INF_F;
      const int len = ok ? blen(sbs, i) : 0;
      const bool above = x > th, atlo = x >= tl;
      const bool inb = atlo && !above;
      whi += above ? len : 0;
      wbd += inb ? len : 0;
      const uint32_t ab = __ballot_sync(0xffffffffu, above);
      const uint32_t bb = __ballot_sync(0xffffffffu, atlo) & ~ab;
      if (lane == 0) gbits[((size_t)bh * G + g2) * nwords + (lo >> 5) + wl] = ab;
      if (bb) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&S2.bcnt[g2], __popc(bb));
        base = __shfl_sync(0xffffffffu, base, 0);
        const int pos = base + __popc(bb & lt);
        if (inb) {
          const int sb = min(max((int)((x - tl) * sbk), 0), kSub - 1);
          atomicAdd(&S2.wsub[g2 * kSub + sb], len);
          if (pos < kSlot) myband[pos] = make_uint2(float_key(x), (uint32_t)i | ((uint32_t)sb << 24));
        }
      }
    }
    if (tid == 0) fstampx(5);
    whi = warp_sum_i(whi);
    wbd = warp_sum_i(wbd);
    if (lane == 0) {
      S2.rwhi[warp][0] = whi;
      S2.rwbd[warp][0] = wbd;
    }
  }
  __syncthreads();
  if (tid < G) {  // this range's weights and band count per head
    int a = 0, c = 0;
    for (int w = tid; w < kFNW; w += G) {
      a += S2.rwhi[w][0];
      c += S2.rwbd[w][0];
    }
    cls_w[((size_t)bh * NS + split) * G + tid] = make_int4(a, c, S2.bcnt[tid], 0);
  }
  for (int j = tid; j < G * kSub; j += kFNT) cls_sub[((size_t)bh * NS + split) * G * kSub + j] = S2.wsub[j];
  __syncthreads();  // every published word / entry / weight precedes the arrive
  fstamp(5);
  if (warp == 0) {
    const unsigned e = s_target + 0x80000000u;  // barrier B: the same flags, the epoch's other half
    if (lane == 0) gbar_arrive(gb, split, e);
    if (!gbar_wait_warp(gb, NS, e) && lane == 0) raise_err(err, kErrSyncTimeout);
    // every CTA has read the epoch (before arriving at A): publish it for the next launch
    if (lane == 0 && split == 0) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(gb), "r"(s_target) : "memory");
  }
  __syncthreads();
  fstamp(13);
  // gather: the above words of every range (all threads), and per head
  // (warp g) the weights, the sub-band weights and the band entries of every
  // range; warp g then resolves head g's marginal block (f_band_select)
  for (int t = tid; t < nwu; t += kFNT)
#pragma unroll
    for (int g2 = 0; g2 < G; ++g2) sbits[g2 * nwords + t] = __ldcg(gbits + ((size_t)bh * G + g2) * nwords + t);
  if (warp < G) {
    const int g2 = warp;
    // lane l holds ranges l and l + 32 (NS <= 64): weights, band counts, prefix
    int4 c0 = make_int4(0, 0, 0, 0), c1 = make_int4(0, 0, 0, 0);
    if (lane < NS) c0 = __ldcg(cls_w + ((size_t)bh * NS + lane) * G + g2);
    if (lane + 32 < NS) c1 = __ldcg(cls_w + ((size_t)bh * NS + lane + 32) * G + g2);
    // the token weight of sub-band j over every range: lane l sums sub-band
    // l % 16 over the ranges r = l / 16 (mod 2), all loads in flight at once
    // (NS <= 64: <= 32 per lane), then lanes l and l + 16 are added
    int wsb = 0;
    {
      const int* src = cls_sub + ((size_t)bh * NS * G + g2) * kSub + (lane & (kSub - 1));
      const size_t rs = (size_t)G * kSub;  // one range further
      int v[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int r = 2 * q + (lane >> 4);
        v[q] = r < NS ? __ldcg(src + r * rs) : 0;
      }
#pragma unroll
      for (int q = 0; q < 32; ++q) wsb += v[q];
      wsb += __shfl_down_sync(0xffffffffu, wsb, 16);
    }
    const int over = __any_sync(0xffffffffu, c0.z > kSlot || c1.z > kSlot);
    const int n0 = min(c0.z, kSlot), n1 = min(c1.z, kSlot);
    const int i0 = warp_incl_scan(n0);
    const int t0 = __shfl_sync(0xffffffffu, i0, 31);
    const int i1 = warp_incl_scan(n1) + t0;
    const int nband = __shfl_sync(0xffffffffu, i1, 31);
    const int W_hi = warp_sum_i(c0.x + c1.x), W_bd = warp_sum_i(c0.y + c1.y);
    // copy: lane l moves the entries of ranges l and l + 32 to their place in
    // the concatenated list (up to 16 + 16 loads in flight before the stores)
    {
      const int d0 = i0 - n0, d1 = i1 - n1;
      const uint2* s0 = cls_band + (((size_t)bh * NS + (lane < NS ? lane : 0)) * G + g2) * kSlot;
      const uint2* s1 = cls_band + (((size_t)bh * NS + (lane + 32 < NS ? lane + 32 : 0)) * G + g2) * kSlot;
#pragma unroll 1
      for (int e0 = 0; e0 < max(n0, n1); e0 += 16) {
        uint2 ev0[16], ev1[16];
#pragma unroll
        for (int e2 = 0; e2 < 16; ++e2) {
          ev0[e2] = e0 + e2 < n0 ? __ldcg(s0 + e0 + e2) : make_uint2(0u, 0u);
          ev1[e2] = e0 + e2 < n1 ? __ldcg(s1 + e0 + e2) : make_uint2(0u, 0u);
        }
#pragma unroll
        for (int e2 = 0; e2 < 16; ++e2) {
          if (e0 + e2 < n0 && d0 + e0 + e2 < BC) sband[g2 * BC + d0 + e0 + e2] = ev0[e2];
          if (e0 + e2 < n1 && d1 + e0 + e2 < BC) sband[g2 * BC + d1 + e0 + e2] = ev1[e2];
        }
      }
    }
    __syncwarp();
    int m = -1, keep = 0, all = 0, fb = 0;
    uint32_t T = 0;
    if (total <= budget) {
      all = 1;
    } else if (W_hi >= budget || W_hi + W_bd < budget || over || nband > BC || force) {
      fb = 1;  // the bounds did not bracket the marginal block: exact slow path below
    } else {
      if (tid == 0) fstampx(6);
      const int4 r = f_band_select<BC>(sband + (size_t)g2 * BC, nband, wsb, sbs, budget - W_hi, sbits + g2 * nwords);
      if (tid == 0) fstampx(7);
      m = r.x;
      keep = r.y;
      T = (uint32_t)r.z;
    }
    if (budget_mode && m >= 0) keep = blen(sbs, m);  // whole blocks (R24): the marginal block whole
    if (lane == 0) S2.sel[g2] = make_int4(m, keep, (int)T, all | (fb << 1));
    if (lane == 0 && g2 < 4) {
      fdbg(4 * g2 + 0, nband);
      fdbg(4 * g2 + 1, over);
      fdbg(4 * g2 + 2, W_hi);
      fdbg(4 * g2 + 3, W_bd);
    }
  }
  }
  __syncthreads();
  fstamp(7);
  // fallback for a head whose Gaussian bounds did not bracket its marginal
  // block (a skewed score distribution, R25): its warp reads every score of
  // the head (all written before barrier A) and selects exactly on its own --
  // the same data and arithmetic in every CTA of the group, so the same
  // result, with no further barrier.  A kH-bin token-weight histogram over
  // [gmin, gmax] (a monotone bin map) gives the crossing bin j*, the highest
  // bin whose suffix weight reaches the budget: bins above j* are selected
  // (W_hi < budget by construction) and the blocks of bin j* are ranked by
  // f_band_select (sub-band = the fraction of the bin x 16, also monotone).
  // A crossing bin of more than BC blocks (massive ties) leaves the
  // head to the CTA-wide slow path below.
  uint32_t fbm = 0;  // heads to the fallback (the same in every CTA of the group)
#pragma unroll
  for (int g2 = 0; g2 < G; ++g2) fbm |= (uint32_t)((S2.sel[g2].w >> 1) & 1) << g2;
  if (force & 2) fbm = 0;
  if (tid == 0 && split == 0 && local_sel == 2) {  // the adaptive choice for the next launch of this group
    const unsigned nxt = lsel ? (s_pref > 0u ? s_pref - 1u : 0u) : (fbm ? 8u : 0u);
    if (nxt != s_pref) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(gbar + (size_t)bh * kGbarWords + 1), "r"(nxt) : "memory");
  }
  if (fbm) {
    // the heads' scores are copied into the free tail of region A (past the
    // selection scratch), as many heads per round as fit
    const int nb4 = (nb + 3) & ~3;
    const size_t sel_b = ((size_t)kFBkt * 4 + (size_t)G * BC * 8 + (size_t)G * nwords * 4 + 15) & ~(size_t)15;
    float* sx = reinterpret_cast<float*>(smA + sel_b);
    const int hpp = max(1, (int)((region_a - sel_b) / ((size_t)nb4 * 4)));
    uint32_t ph = 0;
#pragma unroll 1
    for (int h0 = 0; h0 < G; h0 += hpp) {
      const int hn = min(hpp, G - h0);
      const uint32_t cm = fbm & (((1u << hn) - 1u) << h0);
      if (!cm) continue;
      if (tid == 0) {  // one bulk copy (TMA) per head row, completion on bar2
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier reads of the space
        mbar_arrive_expect_tx(&bar2, (uint32_t)(__popc(cm) * nb4 * 4));
        for (int k = h0; k < h0 + hn; ++k)
          if ((cm >> k) & 1u)
            bulk_g2s(sx + (size_t)(k - h0) * nb4, scores + ((size_t)b * Hq + hk * G + k) * sstride,
                     (uint32_t)(nb4 * 4), &bar2, policy_evict_last());
      }
      mbar_wait(&bar2, ph);
      ph ^= 1u;
      if (tid == 0) fstampx(0);
      if (warp < G && ((cm >> warp) & 1u)) {
        const int g2 = warp;
        const float* xs = sx + (size_t)(g2 - h0) * nb4;
        const float gmn = S2.gmn[g2], kb = S2.kb[g2];
        uint2* lst = sband + (size_t)g2 * BC;
        uint32_t* h = reinterpret_cast<uint32_t*>(lst);  // [kH] histogram, then the band list (BC x 8 B >= kH x 4 B)
        for (int j = lane; j < kH; j += 32) h[j] = 0u;
        if (lane < kSub) S2.wsub[g2 * kSub + lane] = 0;
        __syncwarp();
        for (int i0 = 0; i0 < nb; i0 += 8 * 32) {  // 8 elements per lane in flight
          float x8[8];
          int l8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * 32 + lane;
            x8[u] = i < nb ? xs[i] : 0.f;
            l8[u] = i < nb ? blen(sbs, i) : 0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (l8[u]) atomicAdd(&h[min((int)((x8[u] - gmn) * kb), kH - 1)], (uint32_t)l8[u]);
        }
        __syncwarp();
        if (lane == 0 && g2 == 0) fstampx(1);
        int hv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) hv[k] = (int)h[8 * lane + k];
        int suf = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) suf += hv[k];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {  // suffix weight of bins >= 8 lane
          const int t2 = __shfl_down_sync(0xffffffffu, suf, o);
          if (lane + o < 32) suf += t2;
        }
        int kst = -1, cur = suf, wabove = 0;  // the lane's highest bin whose suffix reaches the budget
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (cur >= budget) {
            kst = k;
            wabove = cur - hv[k];
          }
          cur -= hv[k];
        }
        const uint32_t anyb = __ballot_sync(0xffffffffu, kst >= 0);  // total > budget: never empty
        const int ls = 31 - __clz(anyb);
        const int js = 8 * ls + __shfl_sync(0xffffffffu, kst, ls);
        const int W_hi = __shfl_sync(0xffffffffu, wabove, ls);
        __syncwarp();  // the histogram is read: its space takes the band list
        const uint32_t lt = (1u << lane) - 1u;
        int nband = 0;
        for (int w0 = 0; w0 < nwu; w0 += 4) {  // 4 words per step, loads first
          float x4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = (w0 + u) * 32 + lane;
            x4[u] = i < nb ? xs[i] : 0.f;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = (w0 + u) * 32 + lane;
            const float tb = (x4[u] - gmn) * kb;
            const int bn = i < nb ? min((int)tb, kH - 1) : -1;
            const uint32_t ab = __ballot_sync(0xffffffffu, bn > js);
            const uint32_t bb = __ballot_sync(0xffffffffu, bn == js);
            if (lane == 0 && w0 + u < nwu) sbits[g2 * nwords + w0 + u] = ab;
            if (bn == js) {
              const int pos = nband + __popc(bb & lt);
              const int sb = min((int)((tb - (float)bn) * (float)kSub), kSub - 1);
              atomicAdd(&S2.wsub[g2 * kSub + sb], blen(sbs, i));
              if (pos < BC) lst[pos] = make_uint2(float_key(x4[u]), (uint32_t)i | ((uint32_t)sb << 24));
            }
            nband += __popc(bb);
          }
        }
        __syncwarp();
        if (lane == 0 && g2 == 0) fstampx(2);
        if (lane == 0 && g2 < 4) fdbg(16 + g2, 1 + nband);
        if (nband <= BC) {
          const int wsb = lane < kSub ? S2.wsub[g2 * kSub + lane] : 0;
          int m = -1, keep = 0;
          uint32_t T = 0;
          const int4 r = f_band_select<BC>(lst, nband, wsb, sbs, budget - W_hi, sbits + g2 * nwords);
          m = r.x;
          keep = r.y;
          T = (uint32_t)r.z;
          if (budget_mode && m >= 0) keep = blen(sbs, m);  // whole blocks (R24)
          if (lane == 0) S2.sel[g2] = make_int4(m, keep, (int)T, 0);
        }  // else flag 2 stays: the slow path below
        if (lane == 0 && g2 == 0) fstampx(3);
      }
      __syncthreads();
    }
  }
  // slow path for a head whose bounds failed (rare): CTA-wide exact
  // selection over every key, then its selection words from the keys
  bool special = false;
#pragma unroll
  for (int g2 = 0; g2 < G; ++g2) special |= S2.sel[g2].w != 0;
#pragma unroll 1
  for (int g2 = 0; g2 < G; ++g2) {
    if (!(S2.sel[g2].w & 2)) continue;
    for (int j = tid; j < kFBkt; j += kFNT) hist[j] = 0;
    __syncthreads();
    uint32_t key[kFKPT];
#pragma unroll
    for (int k = 0; k < kFKPT; ++k) {
      const int i = k * kFNT + tid;
      key[k] = i < nb ? float_key(__ldcg(scores + ((size_t)b * Hq + hk * G + g2) * sstride + i)) : 0u;
    }
    f_select_head(key, sbs, total, budget, -CUDART_INF_F, hist, F);
    const int m_c = F.info[0], all_c = F.info[3];
    const uint32_t T_c = (uint32_t)F.info[2];
#pragma unroll
    for (int k = 0; k < kFKPT; ++k) {
      const int i = k * kFNT + tid;
      const bool sel = i < nb && (all_c || key[k] > T_c || (key[k] == T_c && i <= m_c));
      const uint32_t word = __ballot_sync(0xffffffffu, sel);
      const int wi = k * kFNW + warp;
      if (lane == 0 && wi < nwords) sbits[g2 * nwords + wi] = word;
    }
    if (tid == 0) S2.sel[g2] = make_int4(m_c, (budget_mode && m_c >= 0 && !all_c) ? blen(sbs, m_c) : F.info[1],
                                         (int)T_c, all_c);
    __syncthreads();
  }
  // all-fit heads: every block
  if (special) {
#pragma unroll 1
    for (int g2 = 0; g2 < G; ++g2)
      if (S2.sel[g2].w & 1)
        for (int wi = tid; wi < nwu; wi += kFNT) {
          const int rem = nb - wi * 32;
          sbits[g2 * nwords + wi] = rem >= 32 ? 0xffffffffu : (1u << rem) - 1u;
        }
    __syncthreads();
  }
  fstamp(8);

  // ---- 3. union worklist.  Thread t owns word t (blocks 32t .. 32t + 31) and
  //      visits only its set blocks: union rows (a head's rows of a block: all
  //      of them, or `keep` leading rows of its marginal block; union = max
  //      over the G heads), pages; one scan; each thread deals its pages
  //      e = split (mod n_eff) in block order.
  int mg[G], kg[G];
  uint32_t hb[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int4 sl = S2.sel[g];
    mg[g] = (sl.w & 1) ? -1 : sl.x;
    kg[g] = sl.y;
    hb[g] = tid < nwu ? sbits[g * nwords + tid] : 0u;
  }
  uint32_t anyb = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) anyb |= hb[g];
  const int blk0 = tid * 32;
  auto union_rows = [&](int j, int ln) {
    int u = 0;
#pragma unroll
    for (int g = 0; g < G; ++g)
      if ((hb[g] >> j) & 1u) u = max(u, blk0 + j == mg[g] ? kg[g] : ln);
    return u;
  };
  int tot = 0;
#pragma unroll 1
  for (uint32_t bb = anyb; bb; bb &= bb - 1u) {
    const int j = __ffs(bb) - 1;
    tot += (union_rows(j, blen(sbs, blk0 + j)) + P - 1) >> Pshift;
  }
  {  // n_sel per head (one CTA of the group writes n_sel, marginal, keep)
    int c[G];
#pragma unroll
    for (int g = 0; g < G; ++g) c[g] = warp_sum_i(__popc(hb[g]));
    if (lane == 0) {
#pragma unroll
      for (int g = 0; g < G; ++g) S2.rwhi[warp][g] = c[g];
    }
  }
  const int2 pre = f_excl(tot, F.scan[0]);  // (its barrier also publishes rwhi)
  if (split == 0 && tid < G) {
    int ns = 0;
    for (int w = 0; w < kFNW; ++w) ns += S2.rwhi[w][tid];
    const int4 sl = S2.sel[tid];
    const size_t oh = (size_t)b * Hq + hk * G + tid;
    n_sel_out[oh] = ns;
    marg_out[oh] = (sl.w & 1) ? -1 : sl.x;
    keep_out[oh] = (sl.w & 1) ? 0 : sl.y;
  }
  fstamp(9);
  const int cnt = pre.y;  // union pages of the group
  const int n_eff = max(1, min(NS, (cnt + kMinPagesPerSplit - 1) / kMinPagesPerSplit));
  if (tid == 0 && split == 0) {
    wl_count[bh] = cnt;
    if (bh == 0) {
      wl_count[-64] = 0x44534b57;  // "DSKW"
      wl_count[-63] = max_pages;
    }
  }
  if (split >= n_eff) return;
  // deal: page e (block order) -> split e mod n_eff, local index e / n_eff;
  // a countdown to this split's next page avoids a division per page
  const size_t BH = (size_t)gridDim.z * Hkv;
  if (tot) {
    int e = pre.x;
    int qd = e / n_eff;
    int cd = split - (e - qd * n_eff);  // pages until the next page of this split
    if (cd < 0) {
      cd += n_eff;
      ++qd;
    }
#pragma unroll 1
    for (uint32_t bb = anyb; bb; bb &= bb - 1u) {
      const int j = __ffs(bb) - 1;
      const int blk = blk0 + j, ln = blen(sbs, blk);
      const int u = (union_rows(j, ln) + P - 1) >> Pshift;
      if (cd >= u) {
        cd -= u;
        e += u;
        continue;
      }
      const int page0 = spf[blk];
#pragma unroll 1
      for (int jj = cd; jj < u; jj += n_eff) {
        const int pv = min(P, ln - (jj << Pshift));
        uint32_t x0 = 0, x1 = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int tk = ((hb[g] >> j) & 1u) ? (blk == mg[g] ? kg[g] : ln) : 0;
          const uint32_t rr = (uint32_t)min(max(tk - (jj << Pshift), 0), pv);
          if (g < 4) x0 |= rr << (8 * g);
          else x1 |= rr << (8 * (g - 4));
        }
        const int4 en = make_int4(page0 + jj, blk, (int)x0, (int)x1);
        if (qd < ent_cap) s_ent[qd] = en;
        *reinterpret_cast<int4*>(wl + (size_t)(e + jj) * BH + bh) = en;
        ++qd;
        cd = jj + n_eff;
      }
      cd -= u;
      e += u;
    }
  }
  fstamp(10);
  // ---- 4. (a7, a8) attention over this split's pages, split merge
  const int n_it = (cnt - split + n_eff - 1) / n_eff;
  const int nd = attn_depth(kFD, kFNW, kD * 2, P);
  const size_t kstage = (size_t)attn_stage_rows(P) * (kD * 2 + 16);
  __syncthreads();  // region A (selection words) is no longer read
  attn_zero_v_rings(smA, kFNW * nd, kstage, 2 * kstage);
  __syncthreads();  // entries, zeroed rings (and this CTA's worklist writes) visible
  const int n_mine = n_it > warp ? (n_it - warp + kFNW - 1) / kFNW : 0;
  const bool in_smem = n_it <= ent_cap;
  auto entry = [&](int j, int& pg, uint32_t& a, uint32_t& c) {
    const int li = warp + j * kFNW;
    int4 en;
    if (in_smem) en = s_ent[li];
    else en = *reinterpret_cast<const int4*>(wl + (size_t)(split + li * n_eff) * BH + bh);
    pg = en.x;
    a = (uint32_t)en.z;
    c = (uint32_t)en.w;
  };
  attn_bf16_pipeline<G, kFNW, kFD>(smA, s_rows, s_q, nd, P, n_mine, entry, Kp, Vp, (size_t)bh, max_pages,
                                   scale_log2, false);
  fstamp(11);
  attn_merge_out<G, kFNW>(reinterpret_cast<float*>(smA), &s_last, b, hk, Hq, split, n_eff, NS, (size_t)bh,
                          part_o, part_lse, counters, o, lse);
  fstamp(12);
}

}  // namespace dsk

// ============================================================================
// host launcher
// ============================================================================
namespace dsk {
// DYNSPLIT_NO_FUSED=1 (or dynsplit_debug_fused(0)) runs the three-kernel path
// instead (A/B measurements and parity of the two paths).
static volatile bool g_fused_off = getenv("DYNSPLIT_NO_FUSED") != nullptr;
static std::atomic<long long> g_fused_launches{0};
}  // namespace dsk
// Test hook: number of fused-kernel launches so far (tests assert the path ran).
extern "C" long long dynsplit_debug_fused_launches(void) { return dsk::g_fused_launches.load(); }
extern "C" int dynsplit_debug_fused(int on) {
  dsk::g_fused_off = on == 0;
  return 0;
}
extern "C" int dynsplit_debug_fused_force(int mode) {
  return (int)cudaMemcpyToSymbol(dsk::g_fused_force, &mode, sizeof(int));
}
extern "C" int dynsplit_debug_fused_timer(void* dev_ptr) {
  return (int)cudaMemcpyToSymbol(dsk::g_fused_dbg, &dev_ptr, sizeof(void*));
}
namespace dsk {

// global scratch of the fused kernel: per (group, split, head) score moments,
// classification weights and band entries; per (b, query head) the words of
// blocks above t_hi
static size_t fs_al(size_t x) { return (x + 255) & ~(size_t)255; }
size_t fused_scratch_bytes(int B, int Hq, int maxb) {
  const size_t nwords = ((size_t)maxb + 31) / 32;
  return fs_al((size_t)kFMaxGroups * kMaxG * 32) + fs_al((size_t)kFMaxGroups * kMaxG * 16) +
         fs_al((size_t)kFMaxGroups * kMaxG * kSlot * 8) +
         fs_al((size_t)B * Hq * nwords * 4) + fs_al((size_t)kFMaxGroups * kMaxG * kSub * 4);
}

template <int G, int BC>
static cudaError_t run_fused(const CUtensorMap& tm, dim3 grid, size_t smem, cudaStream_t st, const bf16* q,
                             const int32_t* bs, const int32_t* nb, const int32_t* pf, const bf16* Kp,
                             const bf16* Vp, int Hq, int Hkv, int maxb, int max_pages, int S, int Pshift,
                             int budget, int gqa_mode, int budget_mode, int cap, int cap2, int ent_cap, int nwords,
                             int sstride, size_t region_a,
                             int per_cap, int local_sel, float sl2, float* scores, unsigned long long* mom,
                             int4* cls_w, int* cls_sub,
                             uint2* cls_band, uint32_t* gbits, int* counters, unsigned* gbar,
                             float* part_o, float* part_lse, int32_t* n_sel, int32_t* marg, int32_t* keep,
                             int32_t* wl_count, WLEntry* wl, float* o, float* lse, int* err) {
  allow_max_dyn_smem(k_decode_fused<G, BC>);
  if (occupancy_of(k_decode_fused<G, BC>, kFNT, smem) < 1) return cudaErrorNotSupported;
  launch_ex(k_decode_fused<G, BC>, grid, dim3(kFNT), smem, st, 1, tm, q, bs, nb, pf, Kp, Vp, Hq, Hkv, maxb,
            max_pages, S, Pshift, budget, gqa_mode, budget_mode, cap, cap2, ent_cap, nwords, sstride, region_a,
            per_cap, local_sel, sl2, scores, mom,
            cls_w, cls_sub, cls_band, gbits, counters, gbar, part_o, part_lse, n_sel, marg, keep, wl_count, wl, o,
            lse, err);
  g_fused_launches.fetch_add(1);
  return post_launch("k_decode_fused", st);
}

cudaError_t launch_decode_fused(int dtype, int digest_mode, int G, const void* q, const void* dig,
                                const int32_t* bs, const int32_t* nb, const int32_t* pf, const void* Kp,
                                const void* Vp, int B, int Hq, int Hkv, int maxb, int max_pages, int S, int P,
                                int budget, int gqa_mode, int budget_mode, int nb_hint, float scale, float* scores,
                                int sstride,
                                void* fscratch, int* counters, int* bar, float* part_o, float* part_lse,
                                int32_t* n_sel, int32_t* marg, int32_t* keep, int32_t* wl_count, WLEntry* wl,
                                float* o, float* lse, int* err, cudaStream_t st) {
  if (g_fused_off || dtype != 0 || digest_mode != 0) return cudaErrorNotSupported;
  if (G != 1 && G != 2 && G != 4 && G != 8) return cudaErrorNotSupported;
  const int nwords = (maxb + 31) / 32;
  if (nwords * 32 > kFMaxBlocks || sstride < nwords * 32) return cudaErrorNotSupported;
  int Pshift = 0;
  while ((1 << Pshift) < P) ++Pshift;
  if ((1 << Pshift) != P) return cudaErrorNotSupported;
  const int sms = num_sms();
  const int groups = B * Hkv;
  if (groups > sms) return cudaErrorNotSupported;  // every CTA must be resident at once
  const int NS = min(kMaxSplit, sms / groups);
  if ((size_t)groups * NS > (size_t)kFMaxGroups) return cudaErrorNotSupported;
  // shared memory.  Region A: digest stage (phase 1) | score rows, histogram,
  // band entries, selection words (phases 2-3) | page rings, merge scratch (4)
  const int nd = attn_depth(kFD, kFNW, kD * 2, P);
  const size_t ring = (size_t)kFNW * nd * attn_stage_bytes(kD * 2, P);
  // band list capacity: 256 unless the expected band -- (1.8 - 0.55) budget /
  // tokens of the ~nb_hint / 1.25 blocks -- comes near it (large budgets),
  // then 512 (the bigger per-lane rank arrays cost ~1 us per layer when not
  // needed; budget 8192 at 128K: 57 -> 40 us per layer)
  const int BC = (long long)budget * max(nb_hint, 1) > (long long)192 * max(S, 1) ? 512 : 256;
  const size_t sel_bytes = (size_t)kFBkt * 4 + (size_t)G * BC * 8 + (size_t)G * nwords * 4;
  const int per_hint = (((max(nb_hint, 1) + NS - 1) / NS) + kFBox - 1) & ~(kFBox - 1);
  const int capA = max(kFBox, (int)(max(ring, sel_bytes) / (4 * kFSlabRowB)) / kFBox * kFBox);
  const int cap = min(per_hint, capA);
  size_t region_a = max(ring, sel_bytes);
  region_a = max(region_a, (size_t)cap * 4 * kFSlabRowB);
  region_a = max(region_a, (size_t)kFNW * G * kScStride * 4);
  region_a = (region_a + 1023) & ~(size_t)1023;
  const int cap2 = max(kFBox, (int)(region_a / (2 * 4 * kFSlabRowB)) / kFBox * kFBox);  // two staging buffers
  const int ent_cap = min(512, (max_pages + NS - 1) / NS + 1);
  const int per_cap = (((maxb + NS - 1) / NS) + kFBox - 1) & ~(kFBox - 1);  // >= any range
  // local selection for short sequences split over few CTAs (measured: 32K,
  // 8 sequences, 2 splits: 62.9 -> 57.3 us per layer; but 32K, one sequence,
  // 18 splits: 20.4 -> 23.3, where the distributed fast path holds);
  // DYNSPLIT_FUSED_LOCAL=0/1 overrides (A/B, tests)
  // bit 0: always; bit 1: adaptively after a miss, for mid-sized sequences
  // only (<= ~2600 blocks: at 128K the local path costs more than a rare
  // miss -- 128K budget 1K: 22.8 vs 26.6 us per layer over 32 layers)
  int local_sel = (nb_hint <= 1300 && NS <= 2) ? 1 : (nb_hint <= 2600 ? 2 : 0);
  if (const char* e = getenv("DYNSPLIT_FUSED_LOCAL")) local_sel = atoi(e) != 0 ? 1 : 0;
  const size_t smem = 1024 + region_a + (size_t)2 * (nwords * 32 + 8) * 4 + (size_t)ent_cap * 16 +
                      (size_t)G * kD * 2 + (size_t)kFNW * kFD * 8 + (size_t)G * per_cap * 4;
  if (smem + 6144 > (size_t)max_smem_optin()) return cudaErrorNotSupported;
  const auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
  if (!encode) return cudaErrorNotSupported;
  // digests [B * Hkv * maxb rows][256] bf16 -> boxes of 64 dims x 32 rows, 128-byte swizzle
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)2 * kD, (cuuint64_t)B * Hkv * maxb};
  const cuuint64_t strides[1] = {(cuuint64_t)2 * kD * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)kFBox};
  const cuuint32_t es[2] = {1, 1};
  if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(dig), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  char* fs = static_cast<char*>(fscratch);
  unsigned long long* mom = reinterpret_cast<unsigned long long*>(fs);  // [groups x NS][G][4] tagged
  const size_t o_w = fs_al((size_t)kFMaxGroups * kMaxG * 32);
  int4* cls_w = reinterpret_cast<int4*>(fs + o_w);
  uint2* cls_band = reinterpret_cast<uint2*>(fs + o_w + fs_al((size_t)kFMaxGroups * kMaxG * 16));
  uint32_t* gbits = reinterpret_cast<uint32_t*>(fs + o_w + fs_al((size_t)kFMaxGroups * kMaxG * 16) +
                                                fs_al((size_t)kFMaxGroups * kMaxG * kSlot * 8));
  int* cls_sub = reinterpret_cast<int*>(reinterpret_cast<char*>(gbits) + fs_al((size_t)B * Hq * nwords * 4));
  unsigned* gbar = reinterpret_cast<unsigned*>(bar);
  const float sl2 = scale * 1.4426950408889634f;
  const dim3 grid(NS, Hkv, B);
#define DSK_FU(GG)                                                                                        \
  return (BC == 512 ? run_fused<GG, 512> : run_fused<GG, 256>)(tm, grid, smem, st, static_cast<const bf16*>(q), bs, nb, pf, \
                       static_cast<const bf16*>(Kp), static_cast<const bf16*>(Vp), Hq, Hkv, maxb, max_pages, \
                       S, Pshift, budget, gqa_mode, budget_mode, cap, cap2, ent_cap, nwords, sstride,       \
                       region_a, per_cap, local_sel, sl2, scores,                                           \
                       mom, cls_w, cls_sub, cls_band, gbits, counters, gbar, part_o, part_lse, n_sel, marg, \
                       keep,                                                                                \
                       wl_count, wl, o, lse, err)
  switch (G) {
    case 1: DSK_FU(1);
    case 2: DSK_FU(2);
    case 4: DSK_FU(4);
    case 8: DSK_FU(8);
  }
#undef DSK_FU
  return cudaErrorNotSupported;
}

}  // namespace dsk
