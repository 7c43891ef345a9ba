// NEXT-3: cross-step KV reuse over a device page cache of host-offloaded KV.
//
// The paper's second deployment keeps the KV cache in host memory and moves
// only what a decode step needs over PCIe (Table 5: the
// transfer is > 99 % of the attention time at 128K).  Appendix B.2 "KVCache
// Reuse with V2F" then avoids moving what the previous step
// already brought:
//   Step 1  per head, the reusable KV = this step's selection that the
//           previous step also loaded; truncated to the minimum reusable
//           volume over the heads ("a consistent length of reusable KV
//           caches among all heads");
//   Step 2  load the new KV together with the truncated reusable KV;
//   Step 3  merge both into the step's KV.
// Here the unit of storage and transfer is the V2F page (a KV head's pages
// are the union of its query heads' selections, Q18), the device holds one
// slot per page of the previous step (slot_page), and:
//   k_reuse_count  per (b, KV head): reusable pages = |this step's pages AND
//                  the cached pages| (Step 1, before truncation) -- only when
//                  a sequence has more than 8 KV heads; otherwise the KV heads
//                  of a sequence form one cluster and k_reuse_apply exchanges
//                  the counts through distributed shared memory;
//   k_reuse_apply  per (b, KV head): reuse_len = min over the sequence's KV
//                  heads (truncate) -> the first reuse_len reusable pages in
//                  ascending page order are kept in their slots (Q24); every
//                  other page of the step is fresh and takes a freed slot in
//                  ascending (page, slot) order; the fetch list, the new slot
//                  tags and the step's worklist with page -> slot (Step 3);
//   k_fetch_pages  the fresh pages' valid rows host -> cache (Step 2): one
//                  warp per page, 16-byte loads straight from pinned host
//                  memory (zero-copy over PCIe / C2C), all of a lane's loads
//                  in flight before its stores.
// The attention then runs unchanged over the cache (k_decode_attn with the
// slot count as the page stride), so o and lse equal the resident path's bit
// for bit (reuse decides what is moved, never what is computed).
#include "common.cuh"
#include "kernels.h"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace dsk {

constexpr int kRT = 512;   // threads of the reuse kernels
constexpr int kFW = 8;     // warps per (persistent) fetch CTA (two CTAs per SM)

// Bitmaps of one (b, KV head): bit p of `cur` = page p is in this step's
// worklist; bit p of `prv` = page p sits in a cache slot.  Pages outside
// [0, max_pages) or more pages than slots raise DEVERR_PAGE_CAPACITY.
DSK_DEVICE void reuse_bitmaps(uint32_t* cur, uint32_t* prv, int nwp, const int32_t* __restrict__ wl_count,
                              const WLEntry* __restrict__ wl, size_t BH, size_t bh,
                              const int32_t* __restrict__ slot_page, int n_slots, int max_pages, int reuse,
                              int& cnt, int* err) {
  for (int i = threadIdx.x; i < nwp; i += kRT) {
    cur[i] = 0u;
    prv[i] = 0u;
  }
  __syncthreads();
  cnt = wl_count[bh];
  if (cnt < 0 || cnt > n_slots) {
    if (threadIdx.x == 0) raise_err(err, kErrPageCapacity);
    cnt = max(0, min(cnt, n_slots));
  }
  for (int e = threadIdx.x; e < cnt; e += kRT) {
    const int p = reinterpret_cast<const int4*>(wl)[(size_t)e * BH + bh].x;
    if ((unsigned)p < (unsigned)max_pages) atomicOr(&cur[p >> 5], 1u << (p & 31));
    else raise_err(err, kErrPageCapacity);
  }
  if (reuse)
    for (int s = threadIdx.x; s < n_slots; s += kRT) {
      const int p = slot_page[bh * n_slots + s];
      if ((unsigned)p < (unsigned)max_pages) atomicOr(&prv[p >> 5], 1u << (p & 31));
    }
  __syncthreads();
}

__global__ void __launch_bounds__(kRT) k_reuse_count(const int32_t* __restrict__ wl_count,
                                                     const WLEntry* __restrict__ wl,
                                                     const int32_t* __restrict__ slot_page, int n_slots,
                                                     int max_pages, int reuse, int32_t* __restrict__ reusable,
                                                     int* err) {
  extern __shared__ uint32_t bm[];
  __shared__ int red[kRT / 32];
  const int nwp = (max_pages + 31) >> 5;
  const size_t BH = (size_t)gridDim.x * gridDim.y, bh = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
  pdl_trigger();
  pdl_wait();  // the worklist is the predecessor's output
  int cnt;
  reuse_bitmaps(bm, bm + nwp, nwp, wl_count, wl, BH, bh, slot_page, n_slots, max_pages, reuse, cnt, err);
  int c = 0;
  for (int i = threadIdx.x; i < nwp; i += kRT) c += __popc(bm[i] & bm[nwp + i]);
  c = warp_sum_i(c);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kRT / 32; ++w) t += red[w];
    reusable[bh] = t;
  }
}

// Per (b, KV head); grid (Hkv, B).  map [BH][max_pages] and freelist
// [BH][n_slots] are workspace scratch (only entries written in this launch
// are read).
__global__ void __launch_bounds__(kRT) k_reuse_apply(
    const int32_t* __restrict__ wl_hdr, const int32_t* __restrict__ wl_count, const WLEntry* __restrict__ wl,
    int n_slots, int max_pages, int reuse, int truncate, const int32_t* __restrict__ reusable,
    int32_t* __restrict__ map, int32_t* __restrict__ freelist, int32_t* __restrict__ slot_page,
    int32_t* __restrict__ fetch, int32_t* __restrict__ fetch_count, int32_t* __restrict__ stats,
    int32_t* __restrict__ reuse_len, int32_t* __restrict__ c_hdr, int32_t* __restrict__ c_count,
    WLEntry* __restrict__ c_wl, int* err, int in_cluster) {
  extern __shared__ uint32_t bm[];
  __shared__ int scan_sm[(kRT / 32 + 1) * 2];
  __shared__ int s_cnt;
  const int Hkv = gridDim.x, hk = blockIdx.x, b = blockIdx.y;
  const int nwp = (max_pages + 31) >> 5;
  const size_t BH = (size_t)gridDim.x * gridDim.y, bh = (size_t)b * Hkv + hk;
  uint32_t* cur = bm;        // this step's pages -> fresh pages
  uint32_t* prv = bm + nwp;  // cached pages -> reused pages
  pdl_trigger();
  pdl_wait();
  if (bh == 0 && threadIdx.x < 64) c_hdr[threadIdx.x] = wl_hdr[threadIdx.x];
  int cnt;
  reuse_bitmaps(cur, prv, nwp, wl_count, wl, BH, bh, slot_page, n_slots, max_pages, reuse, cnt, err);
  // Step 1: the reuse length of the sequence (min over its KV heads).  With
  // the sequence's KV heads in one cluster (Hkv <= 8) each CTA counts its own
  // reusable pages and reads the others' counts from their shared memory;
  // otherwise k_reuse_count has published them.
  int rl = 0x7fffffff;
  if (in_cluster) {
    cg::cluster_group cluster = cg::this_cluster();
    int c = 0;
    for (int i = threadIdx.x; i < nwp; i += kRT) c += __popc(cur[i] & prv[i]);
    c = warp_sum_i(c);
    if ((threadIdx.x & 31) == 0) scan_sm[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < kRT / 32; ++w) t += scan_sm[w];
      s_cnt = t;
    }
    cluster.sync();
    for (int h = 0; h < Hkv; ++h) rl = min(rl, *cluster.map_shared_rank(&s_cnt, h));
    cluster.sync();  // the peers' counts stay alive until every CTA has read them
  } else if (truncate && reuse) {
    for (int h = 0; h < Hkv; ++h) rl = min(rl, reusable[(size_t)b * Hkv + h]);
  }
  if (!reuse) rl = 0;
  else if (!truncate) rl = 0x7fffffff;
  // the reusable pages in ascending order, the first rl kept: thread t owns
  // words [t * wpt, (t + 1) * wpt)
  const int wpt = (nwp + kRT - 1) / kRT;
  const int w0 = min(nwp, threadIdx.x * wpt), w1 = min(nwp, w0 + wpt);
  int v[1] = {0}, tot[1];
  for (int i = w0; i < w1; ++i) v[0] += __popc(cur[i] & prv[i]);
  block_excl_scan<1, kRT>(v, tot, scan_sm);
  {
    int run = v[0];
    for (int i = w0; i < w1; ++i) {
      uint32_t r = cur[i] & prv[i];
      const int pc = __popc(r);
      if (run + pc > rl) {  // keep the lowest (rl - run) bits (ascending pages)
        uint32_t k = 0u;
        for (int j = 0; j < rl - run; ++j) {
          const uint32_t lowest = r & (0u - r);
          k |= lowest;
          r ^= lowest;
        }
        r = k;
      }
      run += __popc(r);
      prv[i] = r;               // reused
      cur[i] = cur[i] & ~r;     // fresh (Step 2: the truncated excess joins the new data)
    }
  }
  __syncthreads();
  // slots: kept (holding a reused page) or free; free slots compacted in
  // ascending order; every slot is read and rewritten by one thread
  const int spt = (n_slots + kRT - 1) / kRT;
  const int s0 = min(n_slots, threadIdx.x * spt), s1 = min(n_slots, s0 + spt);
  int f[1] = {0}, ftot[1];
  for (int s = s0; s < s1; ++s) {
    const int p = slot_page[bh * n_slots + s];
    const bool kept = (unsigned)p < (unsigned)max_pages && ((prv[p >> 5] >> (p & 31)) & 1u);
    f[0] += kept ? 0 : 1;
  }
  block_excl_scan<1, kRT>(f, ftot, scan_sm);
  int32_t* fl = freelist + bh * n_slots;
  int32_t* mp = map + bh * max_pages;
  {
    int fi = f[0];
    for (int s = s0; s < s1; ++s) {
      const int p = slot_page[bh * n_slots + s];
      const bool kept = (unsigned)p < (unsigned)max_pages && ((prv[p >> 5] >> (p & 31)) & 1u);
      if (kept) {
        mp[p] = s;
      } else {
        fl[fi++] = s;
        slot_page[bh * n_slots + s] = -1;
      }
    }
  }
  const int n_free = ftot[0];
  // fresh pages in ascending order -> free slots in ascending order
  int u[1] = {0}, utot[1];
  for (int i = w0; i < w1; ++i) u[0] += __popc(cur[i]);
  block_excl_scan<1, kRT>(u, utot, scan_sm);  // (its barriers also publish the slot writes above)
  const int n_fresh = utot[0];
  {
    int fi = u[0];
    for (int i = w0; i < w1; ++i)
      for (uint32_t r = cur[i]; r; r &= r - 1u, ++fi) {
        const int p = i * 32 + __ffs(r) - 1;
        if (fi < n_free) {
          const int s = fl[fi];
          mp[p] = s;
          slot_page[bh * n_slots + s] = p;
          fetch[(bh * n_slots + fi) * 2] = p;
          fetch[(bh * n_slots + fi) * 2 + 1] = s;
        } else {
          mp[p] = n_slots;  // no slot left (DEVERR_PAGE_CAPACITY): the attention skips the page
        }
      }
  }
  if (n_fresh > n_free && threadIdx.x == 0) raise_err(err, kErrPageCapacity);
  int n_reused = 0;
  for (int i = threadIdx.x; i < nwp; i += kRT) n_reused += __popc(prv[i]);
  n_reused = warp_sum_i(n_reused);
  __syncthreads();  // map complete
  if ((threadIdx.x & 31) == 0) scan_sm[threadIdx.x >> 5] = n_reused;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kRT / 32; ++w) t += scan_sm[w];
    fetch_count[bh] = min(n_fresh, n_free);
    if (stats) {
      stats[bh * 2] = t;
      stats[bh * 2 + 1] = n_fresh;
    }
    if (reuse_len && hk == 0) reuse_len[b] = (reuse && truncate) ? rl : -1;
    c_count[bh] = cnt;
  }
  // Step 3: the step's worklist over the cache (page -> slot)
  for (int e = threadIdx.x; e < cnt; e += kRT) {
    int4 en = reinterpret_cast<const int4*>(wl)[(size_t)e * BH + bh];
    en.x = (unsigned)en.x < (unsigned)max_pages ? mp[en.x] : n_slots;  // a bad page is never read
    reinterpret_cast<int4*>(c_wl)[(size_t)e * BH + bh] = en;
  }
}

// Persistent mover: two 8-warp CTAs per SM; each warp walks the (b, KV head,
// fetch index) items with a grid stride and copies a page's valid rows of K
// and V, host -> cache slot (dense: page p -> slot p for p < n_pages[b]),
// 8 16-byte loads per lane in flight before the stores.
template <int ROWB>
__global__ void __launch_bounds__(kFW * 32) k_fetch_pages(
    const unsigned char* __restrict__ Kh, const unsigned char* __restrict__ Vh,
    const int16_t* __restrict__ page_valid, const int32_t* __restrict__ n_pages,
    const int32_t* __restrict__ fetch, const int32_t* __restrict__ fetch_count, int dense, int B, int Hkv,
    int max_pages, int n_slots, int P, unsigned char* __restrict__ Kc, unsigned char* __restrict__ Vc) {
  constexpr int CPR = ROWB / 16;  // 16-byte chunks per row
  constexpr int U = 8;            // chunks per lane in flight (x2: K and V)
  const int lane = threadIdx.x & 31;
  pdl_trigger();
  pdl_wait();  // the fetch lists are the predecessor's output
  const long long items = (long long)B * Hkv * n_slots;
  const long long nwarps = (long long)gridDim.x * kFW;
  for (long long it = (long long)blockIdx.x * kFW + (threadIdx.x >> 5); it < items; it += nwarps) {
    const int bh = (int)(it / n_slots), i = (int)(it % n_slots), b = bh / Hkv;
    int page, slot;
    if (dense) {
      if (i >= min(n_pages[b], n_slots)) continue;
      page = slot = i;
    } else {
      if (i >= fetch_count[bh]) continue;
      page = fetch[((size_t)bh * n_slots + i) * 2];
      slot = fetch[((size_t)bh * n_slots + i) * 2 + 1];
      if ((unsigned)page >= (unsigned)max_pages || (unsigned)slot >= (unsigned)n_slots) continue;
    }
    const int rows = min((int)page_valid[(size_t)b * max_pages + page], P);
    const int nch = rows * CPR;
    const uint4* ks = reinterpret_cast<const uint4*>(Kh + ((size_t)bh * max_pages + page) * P * ROWB);
    const uint4* vs = reinterpret_cast<const uint4*>(Vh + ((size_t)bh * max_pages + page) * P * ROWB);
    uint4* kd = reinterpret_cast<uint4*>(Kc + ((size_t)bh * n_slots + slot) * P * ROWB);
    uint4* vd = reinterpret_cast<uint4*>(Vc + ((size_t)bh * n_slots + slot) * P * ROWB);
    for (int c0 = 0; c0 < nch; c0 += 32 * U) {
      uint4 a[U], v[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int c = c0 + k * 32 + lane;
        if (c < nch) {
          a[k] = __ldcs(ks + c);
          v[k] = __ldcs(vs + c);
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int c = c0 + k * 32 + lane;
        if (c < nch) {
          kd[c] = a[k];
          vd[c] = v[k];
        }
      }
    }
  }
}

cudaError_t launch_reuse_plan(const int32_t* wl_hdr, const int32_t* wl_count, const WLEntry* wl, int B, int Hkv,
                              int max_pages, int n_slots, int reuse, int truncate, int32_t* reusable,
                              int32_t* map, int32_t* freelist, int32_t* slot_page, int32_t* fetch,
                              int32_t* fetch_count, int32_t* stats, int32_t* reuse_len, int32_t* c_hdr,
                              int32_t* c_count, WLEntry* c_wl, int* err, cudaStream_t st) {
  const size_t smem = (size_t)2 * ((max_pages + 31) / 32) * 4;
  if (smem > (size_t)max_smem_optin() - 4096) return cudaErrorNotSupported;
  allow_max_dyn_smem(k_reuse_count);
  allow_max_dyn_smem(k_reuse_apply);
  const dim3 grid(Hkv, B);
  // one cluster per sequence (its KV heads) when it fits the portable size:
  // one launch; otherwise the counts go through k_reuse_count
  const int in_cluster = Hkv <= 8 && (truncate && reuse);
  if (truncate && reuse && !in_cluster) {
    launch_ex(k_reuse_count, grid, dim3(kRT), smem, st, 1, wl_count, wl, slot_page, n_slots, max_pages, reuse,
              reusable, err);
    cudaError_t e = post_launch("k_reuse_count", st);
    if (e != cudaSuccess) return e;
  }
  launch_ex(k_reuse_apply, grid, dim3(kRT), smem, st, in_cluster ? Hkv : 1, wl_hdr, wl_count, wl, n_slots,
            max_pages, reuse, truncate, reusable, map, freelist, slot_page, fetch, fetch_count, stats, reuse_len,
            c_hdr, c_count, c_wl, err, in_cluster);
  return post_launch("k_reuse_apply", st);
}

cudaError_t launch_fetch_pages(int dtype, const void* Kh, const void* Vh, const int16_t* page_valid,
                               const int32_t* n_pages, const int32_t* fetch, const int32_t* fetch_count,
                               int dense, int B, int Hkv, int max_pages, int n_slots, int P, void* Kc, void* Vc,
                               cudaStream_t st) {
  const dim3 grid(2 * num_sms());  // 2 x 8 warps per SM: enough PCIe reads in flight across NUMA distances
  const auto* kh = static_cast<const unsigned char*>(Kh);
  const auto* vh = static_cast<const unsigned char*>(Vh);
  auto* kc = static_cast<unsigned char*>(Kc);
  auto* vc = static_cast<unsigned char*>(Vc);
  if (dtype == 0)
    launch_ex(k_fetch_pages<kD * 2>, grid, dim3(kFW * 32), 0, st, 1, kh, vh, page_valid, n_pages, fetch,
              fetch_count, dense, B, Hkv, max_pages, n_slots, P, kc, vc);
  else
    launch_ex(k_fetch_pages<kD * 4>, grid, dim3(kFW * 32), 0, st, 1, kh, vh, page_valid, n_pages, fetch,
              fetch_count, dense, B, Hkv, max_pages, n_slots, P, kc, vc);
  return post_launch("k_fetch_pages", st);
}

}  // namespace dsk
