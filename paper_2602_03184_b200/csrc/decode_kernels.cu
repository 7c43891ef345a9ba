// Decode-step kernels of the DynSplit-KV hot path (sm_100a).
//   a5  k_score_blocks      V2F block score, sum_j max(q_j kmax_j, q_j kmin_j)
//   a6  k_select_threshold  budgeted top-k via block-to-token mapping
//       k_select_union      per-head selections -> GQA-union page worklist
//   (a7/a8 attention kernels live in attn_kernels.cu)

//       k_merge_partials    standalone LSE merge (cross-GPU sequence split)
#include "common.cuh"
#include "kernels.h"

#include <math_constants.h>

namespace dsk {

// ============================================================================
// a5: block scores.  grid (chunks, Hkv, B), 256 threads.  A half-warp owns one
// block digest (512 B bf16: kmax row + kmin row); lane hl owns dims
// [8hl, 8hl+8).  The per-block reduction order (8 sequential terms, then a
// 16-lane xor tree) is fixed and independent of the grid, so every launch
// configuration (and every sequence-split rank) yields identical fp32 scores.
// ============================================================================
template <typename T, int G>
__global__ void __launch_bounds__(256) k_score_blocks(const T* __restrict__ q,
                                                      const T* __restrict__ dig,
                                                      const int32_t* __restrict__ n_blocks,
                                                      float* __restrict__ scores, int Hq, int Hkv,
                                                      int maxb) {
  const int hk = blockIdx.y, b = blockIdx.z;
  const int nb = n_blocks[b];
  int per = (nb + gridDim.x - 1) / gridDim.x;
  per = (per + 15) & ~15;
  const int lo = blockIdx.x * per;
  const int hi = min(nb, lo + per);
  if (lo >= hi) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane >> 4, hl = lane & 15;

  float qv[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) Vec<T>::load8(q + ((size_t)b * Hq + hk * G + g) * kD + hl * 8, qv[g]);

  const T* dbase = dig + ((size_t)b * Hkv + hk) * (size_t)maxb * 2 * kD;
  float* sbase = scores + ((size_t)b * Hq + hk * G) * maxb;
  constexpr int U = 4;
  for (int base = lo + warp * 2; base < hi; base += 16 * U) {
    float kx[U][8], kn[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int blk = base + u * 16 + half;
      if (blk < hi) {
        Vec<T>::load8_nc(dbase + (size_t)blk * 2 * kD + hl * 8, kx[u]);
        Vec<T>::load8_nc(dbase + (size_t)blk * 2 * kD + kD + hl * 8, kn[u]);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) kx[u][j] = kn[u][j] = 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int blk = base + u * 16 + half;
      float acc[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float a = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) a += fmaxf(qv[g][j] * kx[u][j], qv[g][j] * kn[u][j]);
        acc[g] = a;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], o);
      }
      if (hl == 0 && blk < hi) {
#pragma unroll
        for (int g = 0; g < G; ++g) sbase[(size_t)g * maxb + blk] = acc[g];
      }
    }
  }
}

// ============================================================================
// Block-wide exclusive scan of N ints per thread (NT threads).
// ============================================================================
template <int N, int NT>
DSK_DEVICE void block_excl_scan(int (&v)[N], int (&tot)[N], int* sm /* (NT/32+1)*N */) {
  constexpr int NWARP = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc[N];
#pragma unroll
  for (int k = 0; k < N; ++k) inc[k] = warp_incl_scan(v[k]);
  if (lane == 31) {
#pragma unroll
    for (int k = 0; k < N; ++k) sm[warp * N + k] = inc[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int x = lane < NWARP ? sm[lane * N + k] : 0;
      const int s = warp_incl_scan(x);
      if (lane < NWARP) sm[lane * N + k] = s - x;
      if (lane == NWARP - 1) sm[NWARP * N + k] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const int ex = sm[warp * N + k] + inc[k] - v[k];
    tot[k] = sm[NWARP * N + k];
    v[k] = ex;
  }
  __syncthreads();
}

// ============================================================================
// a6 (part 1): per (b, query head) find the marginal block of the budgeted
// token top-k.  Order = (score desc, block index asc); blocks are taken whole
// until the one that reaches `budget` (it keeps `need` tokens).
//   1. keys, lengths -> smem; total length, score min/max.
//   2. 2048-bucket length-weighted histogram of a monotone bucket map
//      floor((s - min) * 2048 / (max - min)).
//   3. suffix scan of the buckets -> the bucket where the budget is reached.
//   4. that bucket's blocks are sorted exactly (bitonic, 64-bit key
//      (score key << 32 | ~index)) and walked to find the marginal block.
// Output sel_info[b, h] = {marginal, keep, key(score of marginal), all_fit}.
// grid (Hq, B), 512 threads, dynamic smem (see select_threshold_smem).
// ============================================================================
constexpr int kSelThreads = 512;
constexpr int kBuckets = 2048;

size_t select_threshold_smem(int maxb) {
  return (size_t)maxb * 8 + (size_t)maxb * 4 + (size_t)maxb * 4 + kBuckets * 4 + 256;
}

DSK_DEVICE float key_to_float(uint32_t k) {
  const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}
DSK_DEVICE int bucket_of(float s, float smin, float inv) {
  int bk = (int)((s - smin) * inv);
  return min(max(bk, 0), kBuckets - 1);
}

__global__ void __launch_bounds__(kSelThreads) k_select_threshold(
    const float* __restrict__ scores, const int32_t* __restrict__ block_starts,
    const int32_t* __restrict__ n_blocks, int Hq, int maxb, int budget, int blk_lo, int blk_hi,
    int4* __restrict__ sel_info) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* cand = reinterpret_cast<uint64_t*>(smem);
  uint32_t* skey = reinterpret_cast<uint32_t*>(cand + maxb);
  int32_t* slen = reinterpret_cast<int32_t*>(skey + maxb);
  uint32_t* hist = reinterpret_cast<uint32_t*>(slen + maxb);
  __shared__ float red_f[2][32];
  __shared__ int red_i[32];
  __shared__ int s_boundary, s_need, s_ncand;

  const int h = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = n_blocks[b];
  const int lo = max(blk_lo, 0), hi = min(blk_hi, nb);
  const int nr = max(hi - lo, 0);
  const float* srow = scores + ((size_t)b * Hq + h) * maxb;
  const int32_t* bs = block_starts + (size_t)b * (maxb + 1);

  float lmin = CUDART_INF_F, lmax = -CUDART_INF_F;
  int ltot = 0;
  for (int i = tid; i < nr; i += kSelThreads) {
    const float s = srow[lo + i];
    skey[i] = float_key(s);
    const int len = bs[lo + i + 1] - bs[lo + i];
    slen[i] = len;
    ltot += len;
    lmin = fminf(lmin, s);
    lmax = fmaxf(lmax, s);
  }
  for (int i = tid; i < kBuckets; i += kSelThreads) hist[i] = 0;
  ltot = warp_sum_i(ltot);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lmin = fminf(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
    lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  }
  if (lane == 0) {
    red_i[warp] = ltot;
    red_f[0][warp] = lmin;
    red_f[1][warp] = lmax;
  }
  if (tid == 0) s_ncand = 0;
  __syncthreads();
  if (warp == 0) {
    const int nw = kSelThreads / 32;
    int t = lane < nw ? red_i[lane] : 0;
    float a = lane < nw ? red_f[0][lane] : CUDART_INF_F;
    float c = lane < nw ? red_f[1][lane] : -CUDART_INF_F;
    t = warp_sum_i(t);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
      c = fmaxf(c, __shfl_xor_sync(0xffffffffu, c, o));
    }
    if (lane == 0) {
      red_i[0] = t;
      red_f[0][0] = a;
      red_f[1][0] = c;
    }
  }
  __syncthreads();
  const int total = red_i[0];
  const float smin = red_f[0][0], smax = red_f[1][0];
  if (total <= budget) {  // every token fits: all blocks selected
    if (tid == 0) sel_info[(size_t)b * Hq + h] = make_int4(-1, 0, 0, 1);
    return;
  }
  const float range = smax - smin;
  const float inv = range > 0.f ? (float)kBuckets / range : 0.f;
  for (int i = tid; i < nr; i += kSelThreads)
    atomicAdd(&hist[bucket_of(key_to_float(skey[i]), smin, inv)], (uint32_t)slen[i]);
  __syncthreads();

  // suffix scan: thread t owns buckets [2047-4t-3, 2047-4t] (descending order)
  {
    int v[1], tot[1];
    const int j0 = kBuckets - 1 - 4 * tid;
    int loc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) loc += (int)hist[j0 - k];
    v[0] = loc;
    block_excl_scan<1, kSelThreads>(v, tot, red_i);
    int above = v[0];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int hb = (int)hist[j0 - k];
      if (above < budget && above + hb >= budget) {
        s_boundary = j0 - k;
        s_need = budget - above;
      }
      above += hb;
    }
  }
  __syncthreads();
  const int boundary = s_boundary;
  const int need = s_need;
  for (int i = tid; i < nr; i += kSelThreads) {
    if (bucket_of(key_to_float(skey[i]), smin, inv) == boundary) {
      const int p = atomicAdd(&s_ncand, 1);
      cand[p] = ((uint64_t)skey[i] << 32) | (uint64_t)(0xffffffffu - (uint32_t)(lo + i));
    }
  }
  __syncthreads();
  const int nc = s_ncand;
  int N = 1;
  while (N < nc) N <<= 1;
  for (int i = nc + tid; i < N; i += kSelThreads) cand[i] = 0ull;
  __syncthreads();
  // bitonic sort, descending
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < N; i += kSelThreads) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = cand[i], c = cand[ixj];
          const bool desc = (i & k) == 0;
          if (desc ? (a < c) : (a > c)) {
            cand[i] = c;
            cand[ixj] = a;
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
        idx = (int)(0xffffffffu - (uint32_t)(cand[i] & 0xffffffffull));
        key = (uint32_t)(cand[i] >> 32);
        len = slen[idx - lo];
      }
      const int inc = warp_incl_scan(len);
      const unsigned hit = __ballot_sync(0xffffffffu, i < nc && cum + inc >= need);
      if (hit) {
        const int src = __ffs(hit) - 1;
        if (lane == src) sel_info[(size_t)b * Hq + h] = make_int4(idx, need - (cum + inc - len), (int)key, 0);
        break;
      }
      cum += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
}

// ============================================================================
// a6 (part 2): per (b, KV head): a head selects block blk iff
//   all_fit || key > T || (key == T && blk <= marginal)
// (T = key of the marginal block; equal keys are ordered by block index).
// Emits, in ascending block order, every page any of the G heads touches with
// its per-head leading-row counts (the GQA union worklist: each KV page is
// streamed from HBM once for all G heads), plus per-head ascending sel_blocks.
// grid (Hkv, B), 512 threads; each thread owns a contiguous run of blocks:
// pass 1 counts, one block-wide scan, pass 2 writes.
// ============================================================================
template <int G>
__global__ void __launch_bounds__(kSelThreads) k_select_union(
    const float* __restrict__ scores, const int32_t* __restrict__ block_starts,
    const int32_t* __restrict__ n_blocks, const int32_t* __restrict__ page_first,
    const int4* __restrict__ sel_info, int Hq, int Hkv, int maxb, int max_sel, int max_wl, int P,
    int blk_lo, int blk_hi, int32_t* __restrict__ sel_blocks, int32_t* __restrict__ n_sel,
    int32_t* __restrict__ marg_out, int32_t* __restrict__ keep_out,
    int32_t* __restrict__ wl_count, WLEntry* __restrict__ wl) {
  __shared__ int sm_scan[(kSelThreads / 32 + 1) * (G + 1)];
  const int hk = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x;
  const int nb = n_blocks[b];
  const int lo = max(blk_lo, 0), hi = min(blk_hi, nb);
  const int nr = max(hi - lo, 0);
  const int per = (nr + kSelThreads - 1) / kSelThreads;
  const int t0 = lo + tid * per, t1 = min(hi, t0 + per);
  const int32_t* bs = block_starts + (size_t)b * (maxb + 1);
  const int32_t* pf = page_first + (size_t)b * (maxb + 1);
  const float* sc = scores + ((size_t)b * Hq + hk * G) * maxb;
  const int pf_lo = lo < hi ? pf[lo] : 0;
  int m[G], keep[G], all[G];
  uint32_t T[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int4 si = sel_info[(size_t)b * Hq + hk * G + g];
    m[g] = si.x;
    keep[g] = si.y;
    T[g] = (uint32_t)si.z;
    all[g] = si.w;
  }
  auto taken_of = [&](int g, int blk, int len) -> int {
    const uint32_t key = float_key(sc[(size_t)g * maxb + blk]);
    const bool sel = all[g] || key > T[g] || (key == T[g] && blk <= m[g]);
    return sel ? ((blk == m[g]) ? keep[g] : len) : 0;
  };
  // pass 1: counts
  int v[G + 1], tot[G + 1];
#pragma unroll
  for (int k = 0; k <= G; ++k) v[k] = 0;
  for (int blk = t0; blk < t1; ++blk) {
    const int len = bs[blk + 1] - bs[blk];
    int u = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int tk = taken_of(g, blk, len);
      v[g] += tk > 0;
      u = max(u, (tk + P - 1) / P);
    }
    v[G] += u;
  }
  block_excl_scan<G + 1, kSelThreads>(v, tot, sm_scan);
  // pass 2: writes
  WLEntry* wlb = wl + ((size_t)b * Hkv + hk) * max_wl;
  for (int blk = t0; blk < t1; ++blk) {
    const int len = bs[blk + 1] - bs[blk];
    int taken[G], u = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      taken[g] = taken_of(g, blk, len);
      u = max(u, (taken[g] + P - 1) / P);
      if (taken[g] > 0) {
        if (sel_blocks) sel_blocks[((size_t)b * Hq + hk * G + g) * max_sel + v[g]] = blk;
        ++v[g];
      }
    }
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
  if (tid == 0) {
    if (hk == 0 && b == 0) {
      wl_count[-64] = 0x44534b57;  // "DSKW"
      wl_count[-63] = max_wl;
    }
    wl_count[(size_t)b * Hkv + hk] = tot[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const size_t o = (size_t)b * Hq + hk * G + g;
      n_sel[o] = tot[g];
      marg_out[o] = all[g] ? -1 : m[g];
      keep_out[o] = all[g] ? 0 : keep[g];
    }
  }
}

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
template <typename T>
static cudaError_t score_blocks_t(int G, const void* q, const void* dig, const int32_t* nb,
                                  float* scores, int B, int Hq, int Hkv, int maxb, cudaStream_t st) {
  const int sms = num_sms();
  int chunks = max(1, (sms * 4) / max(1, B * Hkv));
  chunks = min(chunks, max(1, (maxb + 15) / 16));
  dim3 grid(chunks, Hkv, B);
  const T* qq = static_cast<const T*>(q);
  const T* dd = static_cast<const T*>(dig);
  switch (G) {
    case 1: k_score_blocks<T, 1><<<grid, 256, 0, st>>>(qq, dd, nb, scores, Hq, Hkv, maxb); break;
    case 2: k_score_blocks<T, 2><<<grid, 256, 0, st>>>(qq, dd, nb, scores, Hq, Hkv, maxb); break;
    case 4: k_score_blocks<T, 4><<<grid, 256, 0, st>>>(qq, dd, nb, scores, Hq, Hkv, maxb); break;
    case 8: k_score_blocks<T, 8><<<grid, 256, 0, st>>>(qq, dd, nb, scores, Hq, Hkv, maxb); break;
    default: return cudaErrorInvalidValue;
  }
  return post_launch(__func__, st);
}

cudaError_t launch_score_blocks(int dtype, int G, const void* q, const void* dig, const int32_t* nb,
                                float* scores, int B, int Hq, int Hkv, int maxb, cudaStream_t st) {
  if (dtype == 0) return score_blocks_t<bf16>(G, q, dig, nb, scores, B, Hq, Hkv, maxb, st);
  return score_blocks_t<float>(G, q, dig, nb, scores, B, Hq, Hkv, maxb, st);
}

cudaError_t launch_select(int G, const float* scores, const int32_t* bs, const int32_t* nb,
                          const int32_t* pf, int B, int Hq, int Hkv, int maxb, int max_sel,
                          int max_wl, int P, int budget, int blk_lo, int blk_hi, int4* sel_info,
                          int32_t* sel_blocks, int32_t* n_sel, int32_t* marg, int32_t* keep,
                          int32_t* wl_count, WLEntry* wl, cudaStream_t st) {
  const size_t smem = select_threshold_smem(maxb);
  static bool attr_done = false;
  if (!attr_done) {
    allow_max_dyn_smem(k_select_threshold);
    attr_done = true;
  }
  k_select_threshold<<<dim3(Hq, B), kSelThreads, smem, st>>>(scores, bs, nb, Hq, maxb, budget, blk_lo,
                                                            blk_hi, sel_info);
  cudaError_t e = post_launch(__func__, st);
  if (e != cudaSuccess) return e;
  dim3 grid(Hkv, B);
#define DSK_UNION(GG)                                                                            \
  k_select_union<GG><<<grid, kSelThreads, 0, st>>>(scores, bs, nb, pf, sel_info, Hq, Hkv, maxb,  \
                                                   max_sel, max_wl, P, blk_lo, blk_hi, sel_blocks, \
                                                   n_sel, marg, keep, wl_count, wl)
  switch (G) {
    case 1: DSK_UNION(1); break;
    case 2: DSK_UNION(2); break;
    case 4: DSK_UNION(4); break;
    case 8: DSK_UNION(8); break;
    default: return cudaErrorInvalidValue;
  }
#undef DSK_UNION
  return post_launch(__func__, st);
}

cudaError_t launch_merge(const float* o_parts, const float* lse_parts, int n_parts, int rows, int d,
                         float* o, float* lse, cudaStream_t st) {
  k_merge_partials<<<rows, 128, 0, st>>>(o_parts, lse_parts, n_parts, rows, d, o, lse);
  return post_launch(__func__, st);
}

}  // namespace dsk
