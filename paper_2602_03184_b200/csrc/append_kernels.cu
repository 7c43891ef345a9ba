// NEXT-1: decode-time append with incremental DD-Select ("Incremental Update
// during Decoding ... only the most recent segmentation ranges are
// recomputed"; SPEC S:206-214 with the strict frozen rule, reading Q23).
//
// The caller allocates every per-sequence buffer for a CAPACITY (shape.S);
// L_prev -> L tokens are valid.  Two steps per decode step:
//   k_plan_append (once): per sequence, f = the first block whose start s_c
//     has s_c + C + Delta >= L_prev (blocks before it only see tokens < L_prev
//     and stay verbatim); the page locations of the old tail tokens
//     [start_f, L_prev) (<= C + Delta of them) are recorded in the workspace;
//     then DD-Select resumes at start_f over [start_f, L) -- one warp, lanes =
//     window positions, exact integer keys, ties -> smallest e -- and the block
//     starts are rewritten from f on (k_map_pages then rebuilds the page
//     tables; pages before page_first[f] do not move).
//   k_kv_append (per layer): grid (Hkv, B); the old tail rows are staged in
//     smem, then every block >= f is written into its pages (old tail rows,
//     then the new rows K_new / V_new), padding rows zeroed, and its min/max
//     key digest recomputed.  With L_prev = 0 the same two calls build a whole
//     prefix (f = 0, no old rows).
#include "common.cuh"
#include "kernels.h"

#include <math_constants.h>

namespace dsk {

constexpr int kAppendMaxTail = 256;  // C + Delta bound for the staged old tail

// per-layer pointers of one dynsplit_append_kv_layers call (kernel argument)
struct AppendLayers {
  const void* kn[kAppendMaxLayers];
  const void* vn[kAppendMaxLayers];
  void* kp[kAppendMaxLayers];
  void* vp[kAppendMaxLayers];
  void* dg[kAppendMaxLayers];
};
constexpr int kAppendWs = 4 + kAppendMaxTail;  // int32 per sequence: f, start_f, n_old, L, loc[]

__global__ void __launch_bounds__(32) k_plan_append(const int32_t* __restrict__ tokens,
                                                    const int32_t* __restrict__ delim_ids, int n_ids,
                                                    const uint8_t* __restrict__ w10, int S, int maxb, int maxp,
                                                    int C, int delta, int lam_num, int lam_den, int P,
                                                    int L_prev, int L, int32_t* __restrict__ block_starts,
                                                    int32_t* __restrict__ n_blocks,
                                                    int32_t* __restrict__ page_first,
                                                    int32_t* __restrict__ page_block,
                                                    int16_t* __restrict__ page_valid,
                                                    int32_t* __restrict__ n_pages,
                                                    int32_t* __restrict__ ws, int* __restrict__ err,
                                                    const int32_t* __restrict__ Lp_dev) {
  __shared__ int s_ids[64], s_w[64];
  const int b = blockIdx.x, lane = threadIdx.x;
  if (Lp_dev) {  // device-side length (graph-captured decode loops): L_prev from memory, L = L_prev + n_new
    const int n_new = L - L_prev;
    L_prev = *Lp_dev;
    L = L_prev + n_new;
    if (L_prev < 1 || L > S) {  // a decode step needs a planned prefix and room for the new tokens
      if (lane == 0) {
        int32_t* w0 = ws + (size_t)b * kAppendWs;
        w0[0] = -1;
        w0[1] = w0[2] = 0;
        w0[3] = -1;
        raise_err(err, kErrPlanMismatch);
      }
      return;
    }
  }
  for (int j = lane; j < n_ids; j += 32) {
    s_ids[j] = delim_ids[j];
    s_w[j] = w10[(size_t)b * n_ids + j];
  }
  __syncwarp();
  int32_t* bs = block_starts + (size_t)b * (maxb + 1);
  int32_t* pf = page_first + (size_t)b * (maxb + 1);
  int32_t* w = ws + (size_t)b * kAppendWs;
  const int32_t* tk = tokens + (size_t)b * S;

  // ---- 0. the stored plan must cover exactly the L_prev planned tokens
  //         (S:210 PlanMismatch); otherwise the sequence is left untouched
  //         (f = -1 tells k_kv_append to skip it)
  if (L_prev > 0) {
    const int nb_old = n_blocks[b];
    const bool ok = nb_old >= 1 && nb_old <= maxb && bs[0] == 0 && bs[nb_old] == L_prev &&
                    n_pages[b] >= 0 && n_pages[b] <= maxp;
    if (!ok) {
      if (lane == 0) {
        w[0] = -1;
        w[1] = w[2] = 0;
        w[3] = -1;
        raise_err(err, kErrPlanMismatch);
      }
      return;
    }
  }
  // ---- 1. first non-frozen block of the old plan, old tail locations
  int f = 0, s0 = 0, n_old = 0;
  if (L_prev > 0) {
    const int nb_old = n_blocks[b];
    f = nb_old - 1;  // the last block is never frozen (its start + C >= L_prev)
    while (f > 0 && bs[f - 1] + C + delta >= L_prev) --f;
    s0 = bs[f];
    n_old = L_prev - s0;
    for (int t = s0 + lane; t < L_prev; t += 32) {
      int j = f;
      while (bs[j + 1] <= t) ++j;  // old tail block of token t (few blocks)
      const int o = t - bs[j];
      w[4 + (t - s0)] = (pf[j] + o / P) * P + o % P;
    }
  }
  if (lane == 0) {
    w[0] = f;
    w[1] = s0;
    w[2] = n_old;
    w[3] = L;  // the planned length k_kv_append must be called for
  }
  __syncwarp();

  // ---- 2. DD-Select from s0 over [s0, L): e* = argmax of the exact key
  //         lam_num w (D+1) + (lam_den - lam_num) 10 (D+1 - |e - s_e|), ties -> smallest e
  int nb = f, s_c = s0;
  while (s_c < L) {
    if (lane == 0) bs[nb] = s_c;
    ++nb;
    const int s_e = s_c + C;
    if (s_e >= L) break;
    const int lo = max(s_e - delta, s_c + 1), hi = min(s_e + delta, L - 1);
    long long best = -1;
    int best_e = s_e;
    for (int e0 = lo; e0 <= hi; e0 += 32) {
      const int e = e0 + lane;
      long long key = -1;
      if (e <= hi) {
        const int t = __ldg(tk + e);
        int wt = -1;
        for (int j = 0; j < n_ids; ++j)
          if (s_ids[j] == t) {
            wt = s_w[j];
            break;
          }
        if (wt >= 0)
          key = (long long)lam_num * wt * (delta + 1) +
                (long long)(lam_den - lam_num) * 10 * (delta + 1 - abs(e - s_e));
      }
      // warp argmax, ties -> smallest e
      long long k2 = key;
      int e2 = e;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const long long ko = __shfl_xor_sync(0xffffffffu, k2, o);
        const int eo = __shfl_xor_sync(0xffffffffu, e2, o);
        if (ko > k2 || (ko == k2 && eo < e2)) {
          k2 = ko;
          e2 = eo;
        }
      }
      if (k2 > best) {  // earlier chunks hold smaller e: keep them on ties
        best = k2;
        best_e = e2;
      }
    }
    s_c = best >= 0 ? best_e : s_e;
  }
  for (int j = nb + lane; j <= maxb; j += 32) bs[j] = L;
  if (lane == 0) n_blocks[b] = nb;
  if (L_prev == 0) return;  // a whole prefix: the launcher rebuilds every page table

  // ---- 3. page tables of blocks f .. nb-1 (pages before page_first[f] do not move)
  __syncwarp();
  int32_t* pb = page_block + (size_t)b * maxp;
  int16_t* pv = page_valid + (size_t)b * maxp;
  const int np_old = n_pages[b];
  {  // the re-planned tail must fit the page capacity
    int need = 0;
    for (int j = f + lane; j < nb; j += 32) need += (bs[j + 1] - bs[j] + P - 1) / P;
    need = warp_sum_i(need);
    if (pf[f] + need > maxp) {
      if (lane == 0) {
        w[0] = -1;
        n_pages[b] = -1;
        raise_err(err, kErrPageCapacity);
      }
      return;
    }
  }
  int carry = pf[f];
  for (int j0 = f; j0 < nb; j0 += 32) {
    const int j = j0 + lane;
    const int len = j < nb ? bs[j + 1] - bs[j] : 0;
    const int np = (len + P - 1) / P;
    const int inc = warp_incl_scan(np);
    const int first = carry + inc - np;
    if (j < nb) {
      pf[j] = first;
      for (int jj = 0; jj < np; ++jj) {
        pb[first + jj] = j;
        pv[first + jj] = (int16_t)min(P, len - P * jj);
      }
    }
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  for (int j = nb + lane; j <= maxb; j += 32) pf[j] = carry;
  for (int p2 = carry + lane; p2 < np_old; p2 += 32) {  // pages the tail no longer uses
    pb[p2] = -1;
    pv[p2] = 0;
  }
  if (lane == 0) n_pages[b] = carry;
}

template <typename T>
__global__ void __launch_bounds__(256) k_kv_append(AppendLayers lays, int n_new, int Hkv, int maxb, int maxp,
                                                   int P, int L_prev, int max_tail,
                                                   const int32_t* __restrict__ block_starts,
                                                   const int32_t* __restrict__ n_blocks,
                                                   const int32_t* __restrict__ page_first,
                                                   const int32_t* __restrict__ ws, int mean_mode,
                                                   const int32_t* __restrict__ Lp_dev, int* __restrict__ err) {
  constexpr int LE = kD / 32;  // elements per lane
  if (Lp_dev) L_prev = *Lp_dev;  // device-side length (k_plan_append validated it)
  extern __shared__ __align__(16) unsigned char smem[];
  T* sK = reinterpret_cast<T*>(smem);  // [max_tail][kD]
  T* sV = sK + (size_t)max_tail * kD;
  const int hk = blockIdx.x, b = blockIdx.y, layer = blockIdx.z;
  const T* K_new = static_cast<const T*>(lays.kn[layer]);
  const T* V_new = static_cast<const T*>(lays.vn[layer]);
  T* Kp = static_cast<T*>(lays.kp[layer]);
  T* Vp = static_cast<T*>(lays.vp[layer]);
  T* dig = static_cast<T*>(lays.dg[layer]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int32_t* w = ws + (size_t)b * kAppendWs;
  const int f = w[0], s0 = w[1], n_old = w[2];
  if (f < 0) return;  // k_plan_append flagged this sequence (plan mismatch / capacity)
  // the workspace must describe this append (the plan was advanced to
  // L_prev + n_new by k_plan_append); a stale one is a caller error
  if (w[3] != L_prev + n_new || s0 < 0 || n_old != L_prev - s0 || n_old > max_tail) {
    if (threadIdx.x == 0) raise_err(err, kErrPlanMismatch);
    return;
  }
  const int32_t* bs = block_starts + (size_t)b * (maxb + 1);
  const int32_t* pf = page_first + (size_t)b * (maxb + 1);
  const size_t page_base = ((size_t)b * Hkv + hk) * maxp;
  T* kpb = Kp + page_base * P * kD;
  T* vpb = Vp + page_base * P * kD;
  // ---- stage the old tail rows (they may be overwritten below)
  for (int t = warp; t < n_old; t += nw) {
    const int loc = w[4 + t];
    const uint2* ks = reinterpret_cast<const uint2*>(kpb + (size_t)loc * kD);
    const uint2* vs = reinterpret_cast<const uint2*>(vpb + (size_t)loc * kD);
#pragma unroll
    for (int c = lane; c < kD * (int)sizeof(T) / 8; c += 32) {
      reinterpret_cast<uint2*>(sK + (size_t)t * kD)[c] = ks[c];
      reinterpret_cast<uint2*>(sV + (size_t)t * kD)[c] = vs[c];
    }
  }
  __syncthreads();
  // ---- rewrite blocks f .. nb-1: rows, zero padding, digests (warp per block)
  const int nb = n_blocks[b];
  const size_t new_row = (size_t)Hkv * kD;  // K_new / V_new [B, n_new, Hkv, d]
  const T* kn = K_new + ((size_t)b * n_new * Hkv + hk) * kD;
  const T* vn = V_new + ((size_t)b * n_new * Hkv + hk) * kD;
  for (int j = f + warp; j < nb; j += nw) {
    const int t0 = bs[j], t1 = bs[j + 1];
    // a page table that does not fit the capacity (a failed whole-prefix map) is never written past
    if (t1 <= t0 || pf[j] < 0 || pf[j] + (t1 - t0 + P - 1) / P > maxp) continue;
    float mx[LE], mn[LE], sm[LE];
#pragma unroll
    for (int e = 0; e < LE; ++e) {
      mx[e] = -CUDART_INF_F;
      mn[e] = CUDART_INF_F;
      sm[e] = 0.f;
    }
    const int np = (t1 - t0 + P - 1) / P;
    const T* kb = kpb;  // silence unused warnings in some instantiations
    (void)kb;
    // 4 rows per iteration, all loads first (independent), then the stores
    for (int tb = t0; tb < t0 + np * P; tb += 4) {
      T kv[4][LE], vv[4][LE];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = tb + u;
        if (t < t1) {
          const T* ksrc = t < L_prev ? sK + (size_t)(t - s0) * kD : kn + (size_t)(t - L_prev) * new_row;
          const T* vsrc = t < L_prev ? sV + (size_t)(t - s0) * kD : vn + (size_t)(t - L_prev) * new_row;
#pragma unroll
          for (int e = 0; e < LE; ++e) {
            kv[u][e] = ksrc[lane * LE + e];
            vv[u][e] = vsrc[lane * LE + e];
          }
        } else {
#pragma unroll
          for (int e = 0; e < LE; ++e) kv[u][e] = vv[u][e] = (T)0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = tb + u;
        if (t >= t0 + np * P) break;
        T* kd = kpb + ((size_t)(pf[j] + (t - t0) / P) * P + (t - t0) % P) * kD + lane * LE;
        T* vd = vpb + ((size_t)(pf[j] + (t - t0) / P) * P + (t - t0) % P) * kD + lane * LE;
#pragma unroll
        for (int e = 0; e < LE; ++e) {
          kd[e] = kv[u][e];
          vd[e] = vv[u][e];
          if (t < t1) {
            const float x = (float)kv[u][e];
            mx[e] = fmaxf(mx[e], x);
            mn[e] = fminf(mn[e], x);
            sm[e] += x;  // token order
          }
        }
      }
    }
    T* dd = dig + (((size_t)b * Hkv + hk) * maxb + j) * 2 * kD + lane * LE;
    if (mean_mode) {  // NEXT-2 mean pooling: fp32 mean row (as k_repack_digest)
      float* fp = reinterpret_cast<float*>(dig + (((size_t)b * Hkv + hk) * maxb + j) * 2 * kD) + lane * LE;
#pragma unroll
      for (int e = 0; e < LE; ++e) fp[e] = sm[e] / (float)(t1 - t0);
    } else {
#pragma unroll
      for (int e = 0; e < LE; ++e) {
        dd[e] = (T)mx[e];       // max / min of stored values: exact
        dd[kD + e] = (T)mn[e];
      }
    }
  }
}

size_t append_ws_bytes(int B) { return (size_t)B * kAppendWs * sizeof(int32_t); }
// largest C + Delta the staged old tail supports for this KV dtype (0 = bf16)
int append_max_tail(int dtype) {
  const int by_smem = (int)((200 * 1024) / (2 * kD * (dtype == 0 ? 2 : 4)));
  return by_smem < kAppendMaxTail ? by_smem : kAppendMaxTail;
}

cudaError_t launch_plan_append(const int32_t* tokens, const int32_t* delim_ids, int n_ids, const uint8_t* w10,
                               int B, int S, int maxb, int maxp, int C, int delta, int lam_num, int lam_den,
                               int P, int L_prev, int L, int32_t* block_starts, int32_t* n_blocks,
                               int32_t* page_first, int32_t* page_block, int16_t* page_valid,
                               int32_t* n_pages, int32_t* ws, int* err, cudaStream_t st, const int32_t* Lp_dev) {
  k_plan_append<<<B, 32, 0, st>>>(tokens, delim_ids, n_ids, w10, S, maxb, maxp, C, delta, lam_num, lam_den, P,
                                   L_prev, L, block_starts, n_blocks, page_first, page_block, page_valid,
                                   n_pages, ws, err, Lp_dev);
  cudaError_t e = post_launch(__func__, st);
  if (e != cudaSuccess || L_prev > 0) return e;
  return launch_map_pages(block_starts, n_blocks, B, maxb, maxp, P, L, page_first, page_block, page_valid,
                          n_pages, err, st);
}

cudaError_t launch_kv_append(int dtype, int n_layers, const void* const* K_new, const void* const* V_new,
                             int n_new, int B, int Hkv, int maxb, int maxp, int P, int L_prev, int max_tail,
                             const int32_t* block_starts, const int32_t* n_blocks, const int32_t* page_first,
                             const int32_t* ws, void* const* Kp, void* const* Vp, void* const* dig,
                             int mean_mode, cudaStream_t st, const int32_t* Lp_dev, int* err) {
  if (n_layers < 1 || n_layers > kAppendMaxLayers) return cudaErrorInvalidValue;
  AppendLayers lays = {};
  for (int l = 0; l < n_layers; ++l) {
    lays.kn[l] = K_new ? K_new[l] : nullptr;
    lays.vn[l] = V_new ? V_new[l] : nullptr;
    lays.kp[l] = Kp[l];
    lays.vp[l] = Vp[l];
    lays.dg[l] = dig[l];
  }
  const size_t esz = dtype == 0 ? 2 : 4;
  const size_t smem = 2 * (size_t)max(max_tail, 1) * kD * esz;
  dim3 grid(Hkv, B, n_layers);
  if (dtype == 0) {
    allow_max_dyn_smem(k_kv_append<bf16>);
    k_kv_append<bf16><<<grid, 256, smem, st>>>(lays, n_new, Hkv, maxb, maxp, P, L_prev, max_tail,
                                               block_starts, n_blocks, page_first, ws, mean_mode, Lp_dev, err);
  } else {
    allow_max_dyn_smem(k_kv_append<float>);
    k_kv_append<float><<<grid, 256, smem, st>>>(lays, n_new, Hkv, maxb, maxp, P, L_prev, max_tail,
                                                block_starts, n_blocks, page_first, ws, mean_mode, Lp_dev, err);
  }
  return post_launch(__func__, st);
}

}  // namespace dsk
