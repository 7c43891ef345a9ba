// Prefill row a1: delimiter importance scoring (Algorithm 1, P:148-166;
// score P:176-184), without ever materialising the attention maps.
//
// For query row q of (layer l, sequence b, head h) let p_qk = softmax_k(z_qk),
// z = Qs.Ks/sqrt(d), k <= q.  Candidate i (boundary token, F_i non-empty)
// needs, for every q in F_i = (i, i+W]:
//   Ov = sum_{k in (i-R, i]} p_qk,  Fut = sum_{k in (i, q]} p_qk,
//   Dr = 1 - Ov - Fut  (the rest of the row, = sum_{k <= i-R}; 0 if i < R).
// With dk = q - k and w = q - i in [1, W]:  k in O_i <=> w <= dk <= w+R-1 and
// k in (i, q] <=> dk < w.  So each row only needs p over its last W+R keys
// once its log-sum-exp is known.
//
// k_lse_band: one CTA per (64-row tile, head, layer*batch); 4 warps x 16 rows.
//   1. causal sweep over 64-key tiles with tensor-core MMA (bf16 in, fp32
//      accumulate), online row max/sum in the exp2 domain -> lse2 per row;
//   2. re-sweep the last ceil((W+R-1)/64)+1 key tiles, p = exp2(z - lse2),
//      accumulate Ov[w], Fut[w] per row in registers;
//   3. per candidate, sum its rows inside this tile in row order into one of
//      two slots (its rows span at most two tiles) -> deterministic.
// k_score_reduce: s_i = sum_l sum_h (slot0 + slot1) / (Ls Hq |F_i|), fixed order.
#include "common.cuh"
#include "kernels.h"

#include <math_constants.h>

namespace dsk {

constexpr int kRowsPerCta = 64;
constexpr int kKeyTile = 64;
constexpr int kLds = kD + 8;      // padded smem row (272 B): conflict-free ldmatrix
constexpr int kMaxW = 8;

DSK_DEVICE float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
DSK_DEVICE void cp_async16(void* dst, const void* src, bool pred) {
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(n)
               : "memory");
}
DSK_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
DSK_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
DSK_DEVICE void ldmatrix_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
DSK_DEVICE void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// load a 64 x 128 bf16 tile (rows r0.., row stride `ld` elements) into smem
DSK_DEVICE void load_tile(bf16* dst, const bf16* src, int r0, int nrows_valid, size_t ld) {
  // 64 rows x 16 chunks of 16 B = 1024 chunks, 128 threads -> 8 each
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int c = threadIdx.x + it * 128;
    const int r = c >> 4, cc = c & 15;
    const bool ok = (r0 + r) < nrows_valid;
    const bf16* s = src + (size_t)(ok ? (r0 + r) : 0) * ld + cc * 8;
    cp_async16(dst + r * kLds + cc * 8, s, ok);
  }
}

// S = Q_warp (16 x 128, A fragments) . K_tile^T (64 keys) -> acc[8][4]
DSK_DEVICE void qk_tile(float (&acc)[8][4], const uint32_t (&a)[8][4], const bf16* sK, int lane) {
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[nt][j] = 0.f;
  const int mi = lane >> 3, r = lane & 7;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      uint32_t b[4];
      const bf16* p = sK + (np * 16 + (mi >> 1) * 8 + r) * kLds + kk * 16 + (mi & 1) * 8;
      ldmatrix_x4(b, p);
      mma_bf16(acc[2 * np], a[kk], b[0], b[1]);
      mma_bf16(acc[2 * np + 1], a[kk], b[2], b[3]);
    }
  }
}

__global__ void __launch_bounds__(128) k_lse_band(const int32_t* __restrict__ tokens,
                                                  const int32_t* __restrict__ delim_ids, int n_ids,
                                                  const bf16* __restrict__ Qs, const bf16* __restrict__ Ks,
                                                  int B, int S, int Hq, int Hkv, int W, int R,
                                                  float alpha, float scale_log2,
                                                  float* __restrict__ part) {
  extern __shared__ __align__(128) unsigned char smem[];
  bf16* sQ = reinterpret_cast<bf16*>(smem);
  bf16* sK0 = sQ + kRowsPerCta * kLds;
  bf16* sK1 = sK0 + kKeyTile * kLds;
  float* cbuf = reinterpret_cast<float*>(sK1 + kKeyTile * kLds);  // [64][kMaxW]
  __shared__ int s_ids[64];

  // heaviest (last) row tiles first: causal work grows with the tile index
  const int tile = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, lb = blockIdx.z;  // lb = l*B + b
  const int b = lb % B;
  const int g = Hq / Hkv, hk = h / g;
  const int r0 = tile * kRowsPerCta;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  if (threadIdx.x < n_ids) s_ids[threadIdx.x] = delim_ids[threadIdx.x];

  const size_t ldq = (size_t)Hq * kD, ldk = (size_t)Hkv * kD;
  const bf16* Qbase = Qs + (size_t)lb * S * ldq + (size_t)h * kD;
  const bf16* Kbase = Ks + (size_t)lb * S * ldk + (size_t)hk * kD;
  const int32_t* tk = tokens + (size_t)b * S;

  load_tile(sQ, Qbase, r0, S, ldq);
  load_tile(sK0, Kbase, 0, S, ldk);
  cp_async_commit();

  const int diag = tile;  // key tile holding the tile's last rows
  const int row_a = r0 + warp * 16 + gq, row_b = row_a + 8;
  uint32_t a[8][4];
  float m[2] = {-CUDART_INF_F, -CUDART_INF_F}, l[2] = {0.f, 0.f};

  for (int kt = 0; kt <= diag; ++kt) {
    bf16* cur = (kt & 1) ? sK1 : sK0;
    bf16* nxt = (kt & 1) ? sK0 : sK1;
    if (kt < diag) load_tile(nxt, Kbase, (kt + 1) * kKeyTile, S, ldk);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kt == 0) {
      const int mi = lane >> 3, r = lane & 7;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        ldmatrix_x4(a[kk], sQ + (warp * 16 + (mi & 1) * 8 + r) * kLds + kk * 16 + (mi >> 1) * 8);
    }
    float acc[8][4];
    qk_tile(acc, a, cur, lane);
    float tmax[2] = {-CUDART_INF_F, -CUDART_INF_F};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int key = kt * kKeyTile + nt * 8 + 2 * tq + (j & 1);
        const int row = (j < 2) ? row_a : row_b;
        float z = acc[nt][j] * scale_log2;
        if (kt == diag && key > row) z = -CUDART_INF_F;
        acc[nt][j] = z;
        tmax[j >> 1] = fmaxf(tmax[j >> 1], z);
      }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      tmax[rr] = fmaxf(tmax[rr], __shfl_xor_sync(0xffffffffu, tmax[rr], 1));
      tmax[rr] = fmaxf(tmax[rr], __shfl_xor_sync(0xffffffffu, tmax[rr], 2));
    }
    float mn[2], ls[2] = {0.f, 0.f};
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) mn[rr] = fmaxf(m[rr], tmax[rr]);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) ls[j >> 1] += ex2(acc[nt][j] - mn[j >> 1]);
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      l[rr] = l[rr] * ex2(m[rr] - mn[rr]) + ls[rr];
      m[rr] = mn[rr];
    }
    __syncthreads();
  }
  // full row sums (the 4 lanes of a quad hold disjoint key columns)
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    l[rr] += __shfl_xor_sync(0xffffffffu, l[rr], 1);
    l[rr] += __shfl_xor_sync(0xffffffffu, l[rr], 2);
  }
  float lse2[2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) lse2[rr] = m[rr] + __log2f(l[rr]);

  // ---------------------------------------------------------------- band pass
  const int band = W + R - 1;  // largest dk that matters
  const int kb0 = max(0, r0 - band) / kKeyTile;
  float ov_all[2] = {0.f, 0.f}, ov[2][kMaxW], fu[2][kMaxW];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr)
#pragma unroll
    for (int w = 0; w < kMaxW; ++w) ov[rr][w] = fu[rr][w] = 0.f;

  load_tile(sK0, Kbase, kb0 * kKeyTile, S, ldk);
  cp_async_commit();
  for (int kt = kb0; kt <= diag; ++kt) {
    const int it = kt - kb0;
    bf16* cur = (it & 1) ? sK1 : sK0;
    bf16* nxt = (it & 1) ? sK0 : sK1;
    if (kt < diag) load_tile(nxt, Kbase, (kt + 1) * kKeyTile, S, ldk);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    float acc[8][4];
    qk_tile(acc, a, cur, lane);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int key = kt * kKeyTile + nt * 8 + 2 * tq + (j & 1);
        const int rr = j >> 1;
        const int row = rr ? row_b : row_a;
        const int dk = row - key;
        if (dk < 0 || dk > band) continue;
        const float p = ex2(acc[nt][j] * scale_log2 - lse2[rr]);
        if (dk >= W && dk <= R) {
          ov_all[rr] += p;
        } else {
#pragma unroll
          for (int w = 1; w <= kMaxW; ++w) {
            if (w > W) break;
            if (dk < w) fu[rr][w - 1] += p;
            else if (dk <= w + R - 1) ov[rr][w - 1] += p;
          }
        }
      }
    __syncthreads();
  }
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    ov_all[rr] += __shfl_xor_sync(0xffffffffu, ov_all[rr], 1);
    ov_all[rr] += __shfl_xor_sync(0xffffffffu, ov_all[rr], 2);
#pragma unroll
    for (int w = 0; w < kMaxW; ++w) {
      ov[rr][w] += __shfl_xor_sync(0xffffffffu, ov[rr][w], 1);
      ov[rr][w] += __shfl_xor_sync(0xffffffffu, ov[rr][w], 2);
      fu[rr][w] += __shfl_xor_sync(0xffffffffu, fu[rr][w], 1);
      fu[rr][w] += __shfl_xor_sync(0xffffffffu, fu[rr][w], 2);
    }
  }
  auto is_cand = [&](int i) -> bool {
    if (i < 0 || i > S - 2) return false;
    const int t = tk[i];
    for (int j = 0; j < n_ids; ++j)
      if (s_ids[j] == t) return true;
    return false;
  };
  if (tq == 0) {
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int row = rr ? row_b : row_a;
      const int lr = row - r0;
#pragma unroll
      for (int w = 1; w <= kMaxW; ++w) {
        float c = 0.f;
        const int i = row - w;
        if (w <= W && row < S && is_cand(i)) {
          const float o_ = ov_all[rr] + ov[rr][w - 1];
          const float dr = (i >= R) ? (1.f - o_ - fu[rr][w - 1]) : 0.f;
          c = o_ - alpha * dr;
        }
        cbuf[lr * kMaxW + (w - 1)] = c;
      }
    }
  }
  __syncthreads();
  // candidates whose future rows intersect this tile: i in [r0 - W, r0 + 62]
  for (int ti = threadIdx.x; ti < kRowsPerCta + W - 1; ti += blockDim.x) {
    const int i = r0 - W + ti;
    if (!is_cand(i)) continue;
    const int q0 = max(i + 1, r0), q1 = min(min(i + W, S - 1), r0 + kRowsPerCta - 1);
    if (q0 > q1) continue;
    float sacc = 0.f;
    for (int q = q0; q <= q1; ++q) sacc += cbuf[(q - r0) * kMaxW + (q - i - 1)];
    const int slot = (i + 1 >= r0) ? 0 : 1;
    part[(((size_t)lb * Hq + h) * S + i) * 2 + slot] = sacc;
  }
}

__global__ void k_score_reduce(const int32_t* __restrict__ tokens, const int32_t* __restrict__ delim_ids,
                               int n_ids, const float* __restrict__ part, int Ls, int B, int S, int Hq,
                               int W, float* __restrict__ out) {
  __shared__ int s_ids[64];
  if (threadIdx.x < n_ids) s_ids[threadIdx.x] = delim_ids[threadIdx.x];
  __syncthreads();
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  const int t = tokens[(size_t)b * S + i];
  bool cand = false;
  for (int j = 0; j < n_ids; ++j) cand |= (s_ids[j] == t);
  if (!cand || i > S - 2) {
    out[(size_t)b * S + i] = CUDART_NAN_F;
    return;
  }
  const int qlast = min(i + W, S - 1);
  const bool two = ((i + 1) / kRowsPerCta) != (qlast / kRowsPerCta);
  double acc = 0.0;
  for (int l = 0; l < Ls; ++l)
    for (int h = 0; h < Hq; ++h) {
      const float* p = part + ((((size_t)l * B + b) * Hq + h) * S + i) * 2;
      acc += (double)p[0];
      if (two) acc += (double)p[1];
    }
  out[(size_t)b * S + i] = (float)(acc / ((double)Ls * Hq * (qlast - i)));
}

size_t score_ws_bytes(int Ls, int B, int S, int Hq) {
  return (size_t)Ls * B * Hq * S * 2 * sizeof(float);
}

cudaError_t launch_score_delimiters(const int32_t* tokens, const int32_t* delim_ids, int n_ids,
                                    const void* Qs, const void* Ks, int Ls, int B, int S, int Hq,
                                    int Hkv, int W, int R, float alpha, float* out, void* ws,
                                    cudaStream_t st) {
  const size_t smem = (size_t)(kRowsPerCta + 2 * kKeyTile) * kLds * sizeof(bf16) +
                      kRowsPerCta * kMaxW * sizeof(float);
  static bool attr_done = false;
  if (!attr_done) {
    allow_max_dyn_smem(k_lse_band);
    attr_done = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)kD);
  float* part = static_cast<float*>(ws);
  dim3 grid((S + kRowsPerCta - 1) / kRowsPerCta, Hq, Ls * B);
  k_lse_band<<<grid, 128, smem, st>>>(tokens, delim_ids, n_ids, static_cast<const bf16*>(Qs),
                                      static_cast<const bf16*>(Ks), B, S, Hq, Hkv, W, R, alpha,
                                      scale_log2, part);
  cudaError_t e = post_launch(__func__, st);
  if (e != cudaSuccess) return e;
  k_score_reduce<<<dim3((S + 255) / 256, B), 256, 0, st>>>(tokens, delim_ids, n_ids, part, Ls, B, S,
                                                           Hq, W, out);
  return post_launch(__func__, st);
}

}  // namespace dsk
