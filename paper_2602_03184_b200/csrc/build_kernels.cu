// Prefill block-construction kernels of the DynSplit-KV hot path (sm_100a).
//   a2  k_weight_table     per-id mean -> min-max -> tenths            (T7 P:720-736)
//   a3  k_dd_next          DD-Select e*(s) for every start s in parallel
//       k_dd_walk          follow s -> e*(s) from 0 (one thread, smem windows)
//   a4  k_map_pages        uniform mapping: page_first/page_block/page_valid
//       k_repack_digest    K,V -> fixed P-token pages + per-block kmax/kmin
#include "common.cuh"
#include "kernels.h"

#include <cooperative_groups.h>
#include <stdint.h>

#include <math_constants.h>

namespace dsk {
namespace cg = cooperative_groups;

// ============================================================================
// a2: weight table.  One cluster of kWtCl CTAs per sequence (grid (kWtCl, B),
// 256 threads); CTA r takes the r-th contiguous 1/kWtCl of the positions.
// Tiles of kWtTile positions are staged in smem with coalesced 16-byte loads
// (tokens and scores); thread t walks positions t, t + 256, ... of the tile,
// finds the token's id index through a 256-slot open-addressing hash of the
// ids (~1 probe; most tokens are not delimiters) and adds a valid s_i to its
// own fp64 row acc[j][t] (count likewise), so every sum has a fixed order.
// Per id: the 256 rows are summed in a fixed tree (8 per lane in order, then an
// xor butterfly); rank 0 adds the kWtCl CTAs' sums in rank order through
// DSMEM, then mean, min-max over the ids present, round half-up to tenths.
// ============================================================================
constexpr int kWtNT = 256;
constexpr int kWtTile = 4096;  // positions per smem tile (2048 above 48 ids: the fp64 rows grow)
constexpr int kWtCl = 8;
constexpr int kWtHash = 256;
constexpr int32_t kWtEmpty = INT32_MIN;  // empty hash slot (an id of INT32_MIN is never matched)

static int weight_table_tile(int n_ids) { return n_ids > 48 ? kWtTile / 2 : kWtTile; }
static size_t weight_table_smem(int n_ids) {
  return (size_t)weight_table_tile(n_ids) * 8 + (size_t)n_ids * kWtNT * (sizeof(double) + sizeof(int));
}

DSK_DEVICE uint32_t wt_hash(int32_t t) { return ((uint32_t)t * 0x9E3779B1u) >> 24; }

__global__ void __cluster_dims__(kWtCl, 1, 1) __launch_bounds__(kWtNT)
    k_weight_table(const int32_t* __restrict__ tokens, const int32_t* __restrict__ delim_ids, int n_ids,
                   const float* __restrict__ s, uint8_t* __restrict__ w10, int S, int tile_n) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem[];
  int32_t* t_tok = reinterpret_cast<int32_t*>(smem);                 // [tile_n]
  float* t_s = reinterpret_cast<float*>(t_tok + tile_n);             // [tile_n]
  double* acc = reinterpret_cast<double*>(t_s + tile_n);             // [n_ids][kWtNT]
  int* cnt = reinterpret_cast<int*>(acc + (size_t)n_ids * kWtNT);    // [n_ids][kWtNT]
  __shared__ int h_key[kWtHash], h_val[kWtHash];
  __shared__ double csum[64];   // this CTA's per-id sums (read by rank 0)
  __shared__ int ccnt[64];
  __shared__ double means[64];
  __shared__ int cnts[64];
  const int r = (int)cluster.block_rank(), b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t* tk = tokens + (size_t)b * S;
  const float* sb = s + (size_t)b * S;
  for (int i = tid; i < kWtHash; i += kWtNT) h_key[i] = kWtEmpty;
  for (int j = 0; j < n_ids; ++j) {
    acc[j * kWtNT + tid] = 0.0;
    cnt[j * kWtNT + tid] = 0;
  }
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < n_ids; ++j) {  // the first occurrence of an id owns it (as a linear search would)
      const int32_t id = delim_ids[j];
      uint32_t hh = wt_hash(id);
      while (h_key[hh] != kWtEmpty && h_key[hh] != id) hh = (hh + 1) & (kWtHash - 1);
      if (h_key[hh] == kWtEmpty) {
        h_key[hh] = id;
        h_val[hh] = j;
      }
    }
  }
  // this CTA's range, a multiple of 4 positions (16-byte tiles)
  const int per = ((S + kWtCl - 1) / kWtCl + 3) & ~3;
  const int lo = min(S, r * per), hi = min(S, lo + per);
  const bool vec = ((reinterpret_cast<uintptr_t>(tk) | reinterpret_cast<uintptr_t>(sb)) & 15) == 0;
  for (int p0 = lo; p0 < hi; p0 += tile_n) {
    const int n = min(tile_n, hi - p0);
    __syncthreads();  // previous tile consumed (and the hash / zeroed rows visible)
    if (vec && (n & 3) == 0) {
      for (int c = tid; c < n / 4; c += kWtNT) {
        reinterpret_cast<int4*>(t_tok)[c] = __ldg(reinterpret_cast<const int4*>(tk + p0) + c);
        reinterpret_cast<float4*>(t_s)[c] = __ldg(reinterpret_cast<const float4*>(sb + p0) + c);
      }
    } else {
      for (int c = tid; c < n; c += kWtNT) {
        t_tok[c] = __ldg(tk + p0 + c);
        t_s[c] = __ldg(sb + p0 + c);
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int q = tid; q < n; q += kWtNT) {
      const int32_t t = t_tok[q];
      uint32_t hh = wt_hash(t);
      int key;
      while ((key = h_key[hh]) != kWtEmpty && key != t) hh = (hh + 1) & (kWtHash - 1);
      if (key == t && t != kWtEmpty) {
        const float v = t_s[q];
        if (!isnan(v)) {
          const int j = h_val[hh];
          acc[j * kWtNT + tid] += (double)v;
          cnt[j * kWtNT + tid] += 1;
        }
      }
    }
  }
  __syncthreads();
  for (int j = warp; j < n_ids; j += kWtNT / 32) {
    double a = 0.0;
    int c = 0;
#pragma unroll
    for (int k = 0; k < kWtNT / 32; ++k) {
      a += acc[j * kWtNT + lane * (kWtNT / 32) + k];
      c += cnt[j * kWtNT + lane * (kWtNT / 32) + k];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0) {
      csum[j] = a;
      ccnt[j] = c;
    }
  }
  cluster.sync();  // every CTA's csum / ccnt are visible to rank 0
  if (r == 0 && tid < n_ids) {
    double a = 0.0;
    int c = 0;
    for (int rr = 0; rr < kWtCl; ++rr) {  // rank order
      a += cluster.map_shared_rank(csum, rr)[tid];
      c += cluster.map_shared_rank(ccnt, rr)[tid];
    }
    cnts[tid] = c;
    means[tid] = c ? a / (double)c : 0.0;
  }
  cluster.sync();  // the peers' shared memory stays alive until rank 0 has read it
  if (r != 0) return;
  if (tid == 0) {
    bool any = false;
    double lo_m = 0.0, hi_m = 0.0;
    for (int j = 0; j < n_ids; ++j) {
      if (!cnts[j]) continue;
      if (!any || means[j] < lo_m) lo_m = means[j];
      if (!any || means[j] > hi_m) hi_m = means[j];
      any = true;
    }
    for (int j = 0; j < n_ids; ++j) {
      int w = 0;
      if (cnts[j]) {
        const double ww = (hi_m == lo_m) ? 1.0 : (means[j] - lo_m) / (hi_m - lo_m);
        w = (int)floor(10.0 * ww + 0.5);
      }
      w10[(size_t)b * n_ids + j] = (uint8_t)w;
    }
  }
}

// ============================================================================
// a3 (part 1): e*(s) for every s (the DD-Select step depends only on s_c).
// Exact integer key for lambda*w_e + (1-lambda)*p_e scaled by
// lam_den*10*(Delta+1):  lam_num*w10*(D+1) + (lam_den-lam_num)*10*(D+1-|e-s_e|).
// Ties -> smallest e (strict >).  grid (ceil(S/256), B), 256 threads.
// ============================================================================
__global__ void __launch_bounds__(256) k_dd_next(const int32_t* __restrict__ tokens,
                                                 const int32_t* __restrict__ delim_ids, int n_ids,
                                                 const uint8_t* __restrict__ w10, int S, int C,
                                                 int delta, int lam_num, int lam_den,
                                                 int32_t* __restrict__ next) {
  __shared__ int s_ids[64];
  __shared__ int s_w[64];
  const int b = blockIdx.y;
  if (threadIdx.x < n_ids) {
    s_ids[threadIdx.x] = delim_ids[threadIdx.x];
    s_w[threadIdx.x] = w10[(size_t)b * n_ids + threadIdx.x];
  }
  __syncthreads();
  const int s = blockIdx.x * 256 + threadIdx.x;
  if (s >= S) return;
  const int32_t* tk = tokens + (size_t)b * S;
  const int s_e = s + C;
  int nxt;
  if (s_e >= S) {
    nxt = S;
  } else {
    const int lo = max(s_e - delta, s + 1), hi = min(s_e + delta, S - 1);
    long long best = -1;
    nxt = s_e;
    for (int e = lo; e <= hi; ++e) {
      const int t = __ldg(tk + e);
      int w = -1;
      for (int j = 0; j < n_ids; ++j)
        if (s_ids[j] == t) {
          w = s_w[j];
          break;
        }
      if (w >= 0) {
        const int dist = abs(e - s_e);
        const long long key = (long long)lam_num * w * (delta + 1) +
                              (long long)(lam_den - lam_num) * 10 * (delta + 1 - dist);
        if (key > best) {
          best = key;
          nxt = e;
        }
      }
    }
  }
  next[(size_t)b * S + s] = nxt;
}

// ============================================================================
// a3 (part 2): walk the chain 0 -> e*(0) -> ... (serial by nature, ~S/C
// steps).  The chain only moves forward, so windows of next[] are staged in
// smem as 16-bit deltas and thread 0 walks each window.  grid (B), 1024 threads.
// ============================================================================
constexpr int kWalkWin = 16384;

__global__ void __launch_bounds__(1024) k_dd_walk(const int32_t* __restrict__ next, int S, int maxb,
                                                  int32_t* __restrict__ block_starts,
                                                  int32_t* __restrict__ n_blocks) {
  __shared__ uint16_t sd[kWalkWin];
  __shared__ int s_pos, s_n;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int32_t* nx = next + (size_t)b * S;
  int32_t* bs = block_starts + (size_t)b * (maxb + 1);
  if (tid == 0) {
    s_pos = 0;
    s_n = 0;
  }
  __syncthreads();
  while (s_pos < S) {
    const int w0 = s_pos;
    const int wend = min(S, w0 + kWalkWin);
    for (int i = tid; i < wend - w0; i += 1024) sd[i] = (uint16_t)min(65535, nx[w0 + i] - (w0 + i));
    __syncthreads();
    if (tid == 0) {
      int pos = s_pos, n = s_n;
      while (pos < wend) {
        bs[n++] = pos;
        pos += sd[pos - w0];
      }
      s_pos = pos;
      s_n = n;
    }
    __syncthreads();
  }
  const int n = s_n;
  for (int i = n + tid; i <= maxb; i += 1024) bs[i] = S;
  if (tid == 0) n_blocks[b] = n;
}

// ============================================================================
// a4 (part 1): uniform page map.  grid (B), 1024 threads.  A validation pass
// first: the plan must tile [0, L_end) (n_blocks in [1, maxb], starts from 0
// strictly increasing to L_end; S:267 PlanCoverageMismatch) and fit the page
// capacity maxp; otherwise n_pages[b] = -1, the error bit is raised and
// nothing else of sequence b is written.
// ============================================================================
__global__ void __launch_bounds__(1024) k_map_pages(const int32_t* __restrict__ block_starts,
                                                    const int32_t* __restrict__ n_blocks, int maxb,
                                                    int maxp, int P, int L_end, int32_t* __restrict__ page_first,
                                                    int32_t* __restrict__ page_block,
                                                    int16_t* __restrict__ page_valid,
                                                    int32_t* __restrict__ n_pages, int* __restrict__ err) {
  __shared__ int sm[33];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = n_blocks[b];
  const int32_t* bs = block_starts + (size_t)b * (maxb + 1);
  int32_t* pf = page_first + (size_t)b * (maxb + 1);
  int32_t* pb = page_block + (size_t)b * maxp;
  int16_t* pv = page_valid + (size_t)b * maxp;
  // ---- validation: coverage and page capacity
  if (nb < 1 || nb > maxb) {
    if (tid == 0) {
      n_pages[b] = -1;
      raise_err(err, kErrPlanCoverage);
    }
    return;
  }
  int bad = tid == 0 && (bs[0] != 0 || bs[nb] != L_end);
  long long need = 0;
  for (int blk = tid; blk < nb; blk += 1024) {
    const int len = bs[blk + 1] - bs[blk];
    bad |= len <= 0;
    need += (len + P - 1) / P;
  }
  for (int o = 16; o > 0; o >>= 1) need += __shfl_xor_sync(0xffffffffu, need, o);
  __shared__ long long s_need[32];
  if (lane == 0) s_need[warp] = need;
  bad = __syncthreads_or(bad);
  if (bad) {
    if (tid == 0) {
      n_pages[b] = -1;
      raise_err(err, kErrPlanCoverage);
    }
    return;
  }
  long long tot_need = 0;
  for (int w = 0; w < 32; ++w) tot_need += s_need[w];
  if (tot_need > maxp) {
    if (tid == 0) {
      n_pages[b] = -1;
      raise_err(err, kErrPageCapacity);
    }
    return;
  }
  int carry = 0;
  for (int c0 = 0; c0 < nb; c0 += 1024) {
    const int blk = c0 + tid;
    int len = 0, np = 0;
    if (blk < nb) {
      len = bs[blk + 1] - bs[blk];
      np = (len + P - 1) / P;
    }
    const int inc = warp_incl_scan(np);
    if (lane == 31) sm[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const int x = sm[lane];
      const int sc = warp_incl_scan(x);
      sm[lane] = sc - x;
      if (lane == 31) sm[32] = sc;
    }
    __syncthreads();
    const int off = carry + sm[warp] + inc - np;
    const int tot = sm[32];
    if (blk < nb) {
      pf[blk] = off;
      for (int jj = 0; jj < np; ++jj) {
        pb[off + jj] = blk;
        pv[off + jj] = (int16_t)min(P, len - P * jj);
      }
    }
    carry += tot;
    __syncthreads();
  }
  for (int i = nb + tid; i <= maxb; i += 1024) pf[i] = carry;
  for (int j = carry + tid; j < maxp; j += 1024) {
    pb[j] = -1;
    pv[j] = 0;
  }
  if (tid == 0) n_pages[b] = carry;
}

// ============================================================================
// a4 (part 2): repack + digests.  grid (min(maxb, 8*SMs), B), 128 threads;
// CTAs stride over blocks.  Thread hc owns one 16-byte chunk (h, c) of a token
// row and walks the block's tokens: 16-byte coalesced loads of the
// token-major K/V rows, stores into the head-major pages, running max/min for
// the digest (exact: max/min of stored values), zeroed padding slots.
// ============================================================================
template <typename T>
DSK_DEVICE void unpack16(const uint4& u, float* x) {
  if constexpr (sizeof(T) == 2) {
    x[0] = bf_lo(u.x); x[1] = bf_hi(u.x); x[2] = bf_lo(u.y); x[3] = bf_hi(u.y);
    x[4] = bf_lo(u.z); x[5] = bf_hi(u.z); x[6] = bf_lo(u.w); x[7] = bf_hi(u.w);
  } else {
    x[0] = __uint_as_float(u.x); x[1] = __uint_as_float(u.y);
    x[2] = __uint_as_float(u.z); x[3] = __uint_as_float(u.w);
  }
}

// tokens per thread per iteration (2 kRpU 16-byte loads in flight); measured at
// 128K, B = 4 with a one-wave grid: 2 -> 804 us, 4 -> 838 us, 8 -> 910 us (fewer
// registers, more resident warps)
constexpr int kRpU = 2;

template <typename T>
__global__ void __launch_bounds__(128) k_repack_digest(const T* __restrict__ K, const T* __restrict__ V,
                                                       const int32_t* __restrict__ block_starts,
                                                       const int32_t* __restrict__ n_blocks,
                                                       const int32_t* __restrict__ page_first, int S,
                                                       int Hkv, int maxb, int maxp, int P,
                                                       int mean_mode, T* __restrict__ Kp,
                                                       T* __restrict__ Vp, T* __restrict__ dig,
                                                       int* __restrict__ err) {
  constexpr int EPC = 16 / sizeof(T);     // elements per 16-byte chunk
  constexpr int CPR = kD / EPC;           // chunks per head row
  const int b = blockIdx.y;
  const int nb = n_blocks[b];
  const int32_t* bs = block_starts + (size_t)b * (maxb + 1);
  const int32_t* pf = page_first + (size_t)b * (maxb + 1);
  const int HC = Hkv * CPR;
  // the plan must tile [0, S) and its pages fit the capacity: a bad
  // sequence (or block) is skipped and flagged, never written out of bounds
  if (nb < 1 || nb > maxb || bs[0] != 0 || bs[nb] != S) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_err(err, kErrPlanCoverage);
    return;
  }
  for (int blk = blockIdx.x; blk < nb; blk += gridDim.x) {
    const int st = bs[blk], len = bs[blk + 1] - st, p0 = pf[blk];
    const int npg = (len + P - 1) / P;
    if (len <= 0 || st < 0 || st + len > S || p0 < 0 || p0 + npg > maxp) {
      if (threadIdx.x == 0) raise_err(err, len <= 0 || st < 0 || st + len > S ? kErrPlanCoverage : kErrPageCapacity);
      continue;
    }
    for (int hc = threadIdx.x; hc < HC; hc += blockDim.x) {
      const int h = hc / CPR, c = hc % CPR;
      float mx[EPC], mn[EPC], sm[EPC];
#pragma unroll
      for (int e = 0; e < EPC; ++e) {
        mx[e] = -CUDART_INF_F;
        mn[e] = CUDART_INF_F;
        sm[e] = 0.f;
      }
      const size_t page_base = ((size_t)b * Hkv + h) * maxp;
      int t = 0;
      for (; t + kRpU <= len; t += kRpU) {
        uint4 kk[kRpU], vv[kRpU];
#pragma unroll
        for (int u = 0; u < kRpU; ++u) {
          const size_t src = (((size_t)b * S + st + t + u) * Hkv + h) * kD + c * EPC;
          kk[u] = __ldg(reinterpret_cast<const uint4*>(K + src));
          vv[u] = __ldg(reinterpret_cast<const uint4*>(V + src));
        }
#pragma unroll
        for (int u = 0; u < kRpU; ++u) {
          const int tt = t + u;
          const size_t dst = ((page_base + p0 + tt / P) * P + tt % P) * kD + c * EPC;
          *reinterpret_cast<uint4*>(Kp + dst) = kk[u];
          *reinterpret_cast<uint4*>(Vp + dst) = vv[u];
          float x[EPC];
          unpack16<T>(kk[u], x);
#pragma unroll
          for (int e = 0; e < EPC; ++e) {
            mx[e] = fmaxf(mx[e], x[e]);
            mn[e] = fminf(mn[e], x[e]);
            sm[e] += x[e];  // token order
          }
        }
      }
      for (; t < len; ++t) {
        const size_t src = (((size_t)b * S + st + t) * Hkv + h) * kD + c * EPC;
        const uint4 kk = __ldg(reinterpret_cast<const uint4*>(K + src));
        const uint4 vv = __ldg(reinterpret_cast<const uint4*>(V + src));
        const size_t dst = ((page_base + p0 + t / P) * P + t % P) * kD + c * EPC;
        *reinterpret_cast<uint4*>(Kp + dst) = kk;
        *reinterpret_cast<uint4*>(Vp + dst) = vv;
        float x[EPC];
        unpack16<T>(kk, x);
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          mx[e] = fmaxf(mx[e], x[e]);
          mn[e] = fminf(mn[e], x[e]);
          sm[e] += x[e];
        }
      }
      const uint4 z = make_uint4(0, 0, 0, 0);
      for (int tt = len; tt < npg * P; ++tt) {
        const size_t dst = ((page_base + p0 + tt / P) * P + tt % P) * kD + c * EPC;
        *reinterpret_cast<uint4*>(Kp + dst) = z;
        *reinterpret_cast<uint4*>(Vp + dst) = z;
      }
      if (mean_mode) {  // NEXT-2 mean pooling: fp32 mean row in the digest slot (sum in token order / len)
        float* fp = reinterpret_cast<float*>(dig + (((size_t)b * Hkv + h) * maxb + blk) * 2 * kD) + c * EPC;
#pragma unroll
        for (int e = 0; e < EPC; ++e) fp[e] = sm[e] / (float)len;
        continue;
      }
      // digest row: [.., 0, :] = kmax, [.., 1, :] = kmin (values are exact copies)
      T* dp = dig + (((size_t)b * Hkv + h) * maxb + blk) * 2 * kD + c * EPC;
      T omx[EPC], omn[EPC];
#pragma unroll
      for (int e = 0; e < EPC; ++e) {
        if constexpr (sizeof(T) == 2) {
          omx[e] = __float2bfloat16_rn(mx[e]);
          omn[e] = __float2bfloat16_rn(mn[e]);
        } else {
          omx[e] = mx[e];
          omn[e] = mn[e];
        }
      }
      *reinterpret_cast<uint4*>(dp) = *reinterpret_cast<const uint4*>(omx);
      *reinterpret_cast<uint4*>(dp + kD) = *reinterpret_cast<const uint4*>(omn);
    }
  }
}

// ============================================================================
// host launchers
// ============================================================================
cudaError_t launch_weight_table(const int32_t* tokens, const int32_t* delim_ids, int n_ids,
                                const float* s, uint8_t* w10, int B, int S, cudaStream_t st) {
  const size_t smem = weight_table_smem(n_ids);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_weight_table, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_weight_table<<<dim3(kWtCl, B), kWtNT, smem, st>>>(tokens, delim_ids, n_ids, s, w10, S,
                                                      weight_table_tile(n_ids));
  return post_launch(__func__, st);
}

cudaError_t launch_segment(const int32_t* tokens, const int32_t* delim_ids, int n_ids,
                           const uint8_t* w10, int B, int S, int C, int delta, int lam_num,
                           int lam_den, int maxb, int32_t* next_ws, int32_t* block_starts,
                           int32_t* n_blocks, cudaStream_t st) {
  k_dd_next<<<dim3((S + 255) / 256, B), 256, 0, st>>>(tokens, delim_ids, n_ids, w10, S, C, delta,
                                                       lam_num, lam_den, next_ws);
  cudaError_t e = post_launch(__func__, st);
  if (e != cudaSuccess) return e;
  k_dd_walk<<<B, 1024, 0, st>>>(next_ws, S, maxb, block_starts, n_blocks);
  return post_launch(__func__, st);
}

cudaError_t launch_map_pages(const int32_t* bs, const int32_t* nb, int B, int maxb, int maxp, int P,
                             int L_end, int32_t* page_first, int32_t* page_block, int16_t* page_valid,
                             int32_t* n_pages, int* err, cudaStream_t st) {
  k_map_pages<<<B, 1024, 0, st>>>(bs, nb, maxb, maxp, P, L_end, page_first, page_block, page_valid, n_pages,
                                  err);
  return post_launch(__func__, st);
}

// dynsplit_stream_fence: an empty kernel launched WITHOUT the PDL attribute
// (full stream ordering: the writes of everything before it are visible to
// everything after it, including PDL prologues).
__global__ void k_stream_fence() {}
cudaError_t launch_fence(cudaStream_t st) {
  k_stream_fence<<<1, 32, 0, st>>>();
  return post_launch(__func__, st);
}

cudaError_t launch_repack_digest(int dtype, const void* K, const void* V, const int32_t* bs,
                                 const int32_t* nb, const int32_t* pf, int B, int S, int Hkv,
                                 int maxb, int maxp, int P, int mean_mode, void* Kp, void* Vp, void* dig,
                                 int* err, cudaStream_t st) {
  // exactly one resident wave (CTAs stride over the blocks): a grid past the
  // occupancy leaves a lone partial second wave
  const int oc = dtype == 0 ? occupancy_of(k_repack_digest<bf16>, 128, 0) : occupancy_of(k_repack_digest<float>, 128, 0);
  const int ctas = max(1, min(maxb, num_sms() * oc / max(1, B)));
  dim3 grid(ctas, B);
  if (dtype == 0)
    k_repack_digest<bf16><<<grid, 128, 0, st>>>(
        static_cast<const bf16*>(K), static_cast<const bf16*>(V), bs, nb, pf, S, Hkv, maxb, maxp, P,
        mean_mode, static_cast<bf16*>(Kp), static_cast<bf16*>(Vp), static_cast<bf16*>(dig), err);
  else
    k_repack_digest<float><<<grid, 128, 0, st>>>(
        static_cast<const float*>(K), static_cast<const float*>(V), bs, nb, pf, S, Hkv, maxb, maxp,
        P, mean_mode, static_cast<float*>(Kp), static_cast<float*>(Vp), static_cast<float*>(dig), err);
  return post_launch(__func__, st);
}

}  // namespace dsk
