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

#include <cuda.h>
#include <cudaTypedefs.h>

#include <math_constants.h>
#include <stdlib.h>

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
// Packed fp32 pair arithmetic (sm_100 FFMA2 / FADD2): two independent
// IEEE-rounded operations per instruction, bit-identical to two scalar ones.
DSK_DEVICE void fma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0, float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
DSK_DEVICE void add2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
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


// ============================================================================
// tcgen05 version of k_lse_band (the default): one CTA per (128-row tile,
// head, layer*batch), 10 warps.
//   warp 8 lane 0 (loader): the Q tile once and the K tiles of both passes
//     with TMA tensor copies (cp.async.bulk.tensor, 128-byte swizzle) into
//     K-major smem tiles (two 64-dim halves), 2 stages, mbarrier complete_tx.
//   warp 9 lane 0 (MMA): S = Q K^T for a 128-key tile as 8 x
//     tcgen05.mma.cta_group::1.kind::f16 (M = 128 rows, N = 128 keys, K = 16
//     dims each, bf16 in, fp32 accumulate) into one of two 128-column TMEM
//     accumulators; tcgen05.commit frees the K stage and publishes S.
//   warps 0-7 (epilogue): warp w reads TMEM lane quadrant w % 4 (rows
//     32 (w % 4) + lane) and column half w / 4 of every tile with tcgen05.ld
//     32x32b; a row's two halves keep separate online (max, sum) in the exp2
//     domain (pass 1) and separate band sums Ov[w], Fut[w] (pass 2:
//     p = exp2(z - lse2) over the band tiles), combined once through shared
//     memory in fixed order.  Per candidate, rows summed in row order.
// TMEM: 256 columns (2 accumulators); smem 3 x 32 KiB + 1 KiB alignment.
// ============================================================================
constexpr int kTcRows = 128;   // rows per CTA (M) = keys per tile (N)
constexpr int kTcStage = 2;
constexpr int kTcTileBytes = kTcRows * kD * 2;  // 32 KiB

DSK_DEVICE uint64_t umma_sdesc_sw128(uint32_t saddr) {
  // K-major, SWIZZLE_128B: 128-byte rows, 8-row atoms of 1024 B (SBO), LBO
  // unused, descriptor version 1, layout type 2
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
DSK_DEVICE void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DSK_DEVICE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
DSK_DEVICE void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
DSK_DEVICE void tc_ld32(uint32_t addr, float (&f)[32]) {
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,"
      "%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
}

constexpr int kTcEpiWarps = 8;  // two warps per TMEM lane quadrant: column halves
constexpr int kTcThreads = (kTcEpiWarps + 2) * 32;

// TMA: one 2-D box of 64 dims x 128 rows (128-byte swizzle, rows past S zero-filled)
DSK_DEVICE void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(kTcThreads, 1) k_lse_band_tc(const __grid_constant__ CUtensorMap tmQ,
                                                              const __grid_constant__ CUtensorMap tmK,
                                                              const int32_t* __restrict__ tokens,
                                                              const int32_t* __restrict__ delim_ids, int n_ids,
                                                              int B, int S, int Hq,
                                                              int Hkv, int W, int R, float alpha,
                                                              float scale_log2, float* __restrict__ part) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // 1024-byte aligned tiles (the swizzle atoms are address-based)
  const uint32_t raw_s = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + (((raw_s + 1023u) & ~1023u) - raw_s);
  unsigned char* sQ = smem;                       // [2 halves][128 rows][128 B]
  unsigned char* sK = smem + kTcTileBytes;        // [kTcStage][2 halves][128 rows][128 B]
  float* cbuf = reinterpret_cast<float*>(sK);     // [128][kMaxW], after the last MMA
  constexpr int kX = 2 + 2 * kMaxW + 1;
  __shared__ float xch[kTcRows * kX];             // half-row exchange (live while K stages are)
  __shared__ __align__(8) uint64_t kfull[kTcStage], kempty[kTcStage], sfull[2], sempty[2];
  __shared__ uint32_t s_tmem;
  __shared__ int s_ids[64];

  const int tile = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, lb = blockIdx.z;  // heaviest tiles first
  const int b = lb % B;
  const int g = Hq / Hkv, hk = h / g;
  const int r0 = tile * kTcRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int band = W + R - 1;
  const int T = tile;                                   // diagonal key tile
  const int kb0 = max(0, r0 - band) / kTcRows;          // first band tile
  const int n1 = T + 1, n_all = n1 + (T - kb0 + 1);     // pass-1 tiles, all tiles
  auto tile_of = [&](int i) { return i < n1 ? i : kb0 + (i - n1); };

  if (threadIdx.x < n_ids) s_ids[threadIdx.x] = delim_ids[threadIdx.x];
  if (threadIdx.x == 0) {
    for (int st = 0; st < kTcStage; ++st) {
      mbar_init(&kfull[st], 1);
      mbar_init(&kempty[st], 1);
    }
    for (int bb = 0; bb < 2; ++bb) {
      mbar_init(&sfull[bb], 1);
      mbar_init(&sempty[bb], kTcEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (warp == kTcEpiWarps) {  // ----------------------------------- loader
    // TMA tensor copies (maps [lb][s][head][d]): per tile two boxes of 64 dims
    // x 128 rows, hardware 128-byte swizzle = the UMMA K-major SW128 layout
    if (lane == 0) {
      for (int i = 0; i < n_all; ++i) {
        const int st = i % kTcStage;
        if (i >= kTcStage) mbar_wait(&kempty[st], ((i / kTcStage) - 1) & 1);
        unsigned char* dst = sK + st * kTcTileBytes;
        mbar_arrive_expect_tx(&kfull[st], (uint32_t)(kTcTileBytes + (i == 0 ? kTcTileBytes : 0)));
        if (i == 0) {  // the Q tile rides on tile 0's barrier
          tma_load_4d(sQ, &tmQ, 0, h, r0, lb, &kfull[0]);
          tma_load_4d(sQ + kTcRows * 128, &tmQ, 64, h, r0, lb, &kfull[0]);
        }
        const int kr = tile_of(i) * kTcRows;
        tma_load_4d(dst, &tmK, 0, hk, kr, lb, &kfull[st]);
        tma_load_4d(dst + kTcRows * 128, &tmK, 64, hk, kr, lb, &kfull[st]);
      }
    }
    __syncwarp();
  } else if (warp == kTcEpiWarps + 1) {  // ------------------------ MMA issue
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTcRows >> 3) << 17) |
                           ((uint32_t)(kTcRows >> 4) << 24);
    for (int i = 0; i < n_all; ++i) {
      const int st = i % kTcStage, bb = i & 1;
      mbar_wait(&kfull[st], (i / kTcStage) & 1);
      if (i >= 2) mbar_wait(&sempty[bb], ((i >> 1) - 1) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK + st * kTcTileBytes);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          const uint32_t off = (uint32_t)((k >> 2) * (kTcRows * 128) + (k & 3) * 32);
          const uint64_t da = umma_sdesc_sw128(qa + off), db = umma_sdesc_sw128(ka + off);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + bb * kTcRows),
              "l"(da), "l"(db), "r"(idesc), "r"((uint32_t)(k > 0)));
        }
        tc_commit(&sfull[bb]);
        tc_commit(&kempty[st]);
      }
      __syncwarp();
    }
  } else {  // ---------------------------------------------------- epilogue
    // warp w: TMEM lane quadrant q = w % 4 (rows 32 q + lane), column half hw = w / 4
    const int q = warp & 3, hw = warp >> 2;
    const int lr = q * 32 + lane, row = r0 + lr;
    float m = -CUDART_INF_F, l = 0.f, lse2 = 0.f;
    float ov_all = 0.f, ov[kMaxW], fu[kMaxW];
#pragma unroll
    for (int w = 0; w < kMaxW; ++w) ov[w] = fu[w] = 0.f;
    for (int i = 0; i < n_all; ++i) {
      const int bb = i & 1, kt = tile_of(i);
      mbar_wait(&sfull[bb], (i >> 1) & 1);
      tc_fence_after();
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(bb * kTcRows + hw * 64);
      if (i == n1) {  // pass 1 complete: combine the two column halves of the row
        float* xr = xch + lr * kX;
        if (hw) {
          xr[0] = m;
          xr[1] = l;
        }
        named_bar_sync(1, kTcEpiWarps * 32);
        const float m2 = hw ? m : xr[0], l2 = hw ? l : xr[1];
        const float mm = hw ? m : fmaxf(m, m2);
        float ll = l;
        if (!hw) {
          ll = (m == -CUDART_INF_F ? 0.f : l * ex2(m - mm)) + (m2 == -CUDART_INF_F ? 0.f : l2 * ex2(m2 - mm));
          xr[0] = mm + __log2f(ll);
        }
        named_bar_sync(1, kTcEpiWarps * 32);
        lse2 = xr[0];
      }
      for (int c0 = 0; c0 < 64; c0 += 32) {
        float z[32];
        __syncwarp();  // .aligned TMEM loads need the converged warp
        tc_ld32(base + (uint32_t)c0, z);
        if (c0 == 32) {  // the accumulator may be overwritten now
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sempty[bb]);
        }
        const int key0 = kt * kTcRows + hw * 64 + c0;
        if (i < n1) {
          // raw logits; the scale (> 0) is folded into one FFMA per element below
          if (kt == T) {  // diagonal tile: causal mask
#pragma unroll
            for (int j = 0; j < 32; ++j) z[j] = key0 + j > row ? -CUDART_INF_F : z[j];
          }
          float t8[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) t8[j] = fmaxf(fmaxf(z[j], z[j + 8]), fmaxf(z[j + 16], z[j + 24]));
          const float tmax = fmaxf(fmaxf(fmaxf(t8[0], t8[1]), fmaxf(t8[2], t8[3])),
                                   fmaxf(fmaxf(t8[4], t8[5]), fmaxf(t8[6], t8[7])));
          const float mn = fmaxf(m, tmax * scale_log2);
          if (mn == -CUDART_INF_F) continue;  // nothing valid yet in this row
          const float nmn = -mn;
          // four running sums, ls[r] over columns j = r (mod 4) in order, as
          // two packed pairs: FFMA2 for the scaled logits, FADD2 for the sums
          float ls0 = 0.f, ls1 = 0.f, ls2 = 0.f, ls3 = 0.f;
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float x0, x1;
            fma2(x0, x1, z[j], z[j + 1], scale_log2, scale_log2, nmn, nmn);
            const float e0 = ex2(x0), e1 = ex2(x1);
            if ((j & 2) == 0) add2(ls0, ls1, ls0, ls1, e0, e1);
            else add2(ls2, ls3, ls2, ls3, e0, e1);
          }
          l = (m == -CUDART_INF_F ? 0.f : l * ex2(m - mn)) + ((ls0 + ls1) + (ls2 + ls3));
          m = mn;
        } else {
          // band: dk = row - key in [0, band]
          const int dk0 = row - key0;
          if (dk0 < 0 || dk0 - 31 > band) continue;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int dk = dk0 - j;
            if (dk < 0 || dk > band) continue;
            const float p = ex2(fmaf(z[j], scale_log2, -lse2));
            if (dk >= W && dk <= R) {
              ov_all += p;
            } else {
#pragma unroll
              for (int w = 1; w <= kMaxW; ++w) {
                if (w > W) break;
                if (dk < w) fu[w - 1] += p;
                else if (dk <= w + R - 1) ov[w - 1] += p;
              }
            }
          }
        }
      }
    }
    // every MMA has completed (the last sfull was waited): the K stages are free.
    // Combine the two column halves of each row (half 0 + half 1, fixed order).
    named_bar_sync(1, kTcEpiWarps * 32);
    float* xr = xch + lr * kX;
    if (hw) {
      xr[2] = ov_all;
#pragma unroll
      for (int w = 0; w < kMaxW; ++w) {
        xr[3 + w] = ov[w];
        xr[3 + kMaxW + w] = fu[w];
      }
    }
    named_bar_sync(1, kTcEpiWarps * 32);
    if (!hw) {
      ov_all += xr[2];
#pragma unroll
      for (int w = 0; w < kMaxW; ++w) {
        ov[w] += xr[3 + w];
        fu[w] += xr[3 + kMaxW + w];
      }
    }
    const int32_t* tk = tokens + (size_t)b * S;
    auto is_cand = [&](int i) -> bool {
      if (i < 0 || i > S - 2) return false;
      const int t = tk[i];
      for (int j = 0; j < n_ids; ++j)
        if (s_ids[j] == t) return true;
      return false;
    };
    if (!hw) {
#pragma unroll
      for (int w = 1; w <= kMaxW; ++w) {
        float c = 0.f;
        const int i = row - w;
        if (w <= W && row < S && is_cand(i)) {
          const float o_ = ov_all + ov[w - 1];
          const float dr = (i >= R) ? (1.f - o_ - fu[w - 1]) : 0.f;
          c = o_ - alpha * dr;
        }
        cbuf[lr * kMaxW + (w - 1)] = c;
      }
    }
    named_bar_sync(1, kTcEpiWarps * 32);
    for (int ti = threadIdx.x; ti < kTcRows + W - 1; ti += kTcEpiWarps * 32) {
      const int i = r0 - W + ti;
      if (!is_cand(i)) continue;
      const int q0 = max(i + 1, r0), q1 = min(min(i + W, S - 1), r0 + kTcRows - 1);
      if (q0 > q1) continue;
      float sacc = 0.f;
      for (int qq = q0; qq <= q1; ++qq) sacc += cbuf[(qq - r0) * kMaxW + (qq - i - 1)];
      const int slot = (i + 1 >= r0) ? 0 : 1;
      part[(((size_t)lb * Hq + h) * S + i) * 2 + slot] = sacc;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

__global__ void k_score_reduce(const int32_t* __restrict__ tokens, const int32_t* __restrict__ delim_ids,
                               int n_ids, const float* __restrict__ part, int Ls, int B, int S, int Hq,
                               int W, int rows_per_tile, float* __restrict__ out) {
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
  const bool two = ((i + 1) / rows_per_tile) != (qlast / rows_per_tile);
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

static volatile bool g_a1_mmasync = getenv("DYNSPLIT_A1_MMASYNC") != nullptr;

cudaError_t launch_score_delimiters(const int32_t* tokens, const int32_t* delim_ids, int n_ids,
                                    const void* Qs, const void* Ks, int Ls, int B, int S, int Hq,
                                    int Hkv, int W, int R, float alpha, float* out, void* ws,
                                    cudaStream_t st) {
  // tcgen05 kernel by default; DYNSPLIT_A1_MMASYNC=1 (or the test hook) selects the
  // mma.sync kernel (A/B, parity of both)
  const bool mmasync = g_a1_mmasync;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)kD);
  float* part = static_cast<float*>(ws);
  int rows_per_tile;
  const auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
  if (!mmasync && !encode) return cudaErrorNotSupported;
  if (!mmasync) {
    // [Ls*B][S][H][d] bf16 -> dims (d, H, S, Ls*B); box (64, 1, 128, 1), 128-byte swizzle
    auto make_map = [&](CUtensorMap* m, const void* base, int H) -> bool {
      const cuuint64_t dims[4] = {(cuuint64_t)kD, (cuuint64_t)H, (cuuint64_t)S, (cuuint64_t)Ls * B};
      const cuuint64_t strides[3] = {(cuuint64_t)kD * 2, (cuuint64_t)H * kD * 2, (cuuint64_t)S * H * kD * 2};
      const cuuint32_t box[4] = {64, 1, (cuuint32_t)kTcRows, 1};
      const cuuint32_t es[4] = {1, 1, 1, 1};
      return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    CUtensorMap tmQ, tmK;
    if (!make_map(&tmQ, Qs, Hq) || !make_map(&tmK, Ks, Hkv)) return cudaErrorInvalidValue;
    const size_t smem = (size_t)(1 + kTcStage) * kTcTileBytes + 1024;  // cbuf fits in sK
    allow_max_dyn_smem(k_lse_band_tc);
    dim3 grid((S + kTcRows - 1) / kTcRows, Hq, Ls * B);
    k_lse_band_tc<<<grid, kTcThreads, smem, st>>>(tmQ, tmK, tokens, delim_ids, n_ids, B, S, Hq, Hkv, W, R,
                                                  alpha, scale_log2, part);
    rows_per_tile = kTcRows;
  } else {
    const size_t smem = (size_t)(kRowsPerCta + 2 * kKeyTile) * kLds * sizeof(bf16) +
                        kRowsPerCta * kMaxW * sizeof(float);
    allow_max_dyn_smem(k_lse_band);
    dim3 grid((S + kRowsPerCta - 1) / kRowsPerCta, Hq, Ls * B);
    k_lse_band<<<grid, 128, smem, st>>>(tokens, delim_ids, n_ids, static_cast<const bf16*>(Qs),
                                        static_cast<const bf16*>(Ks), B, S, Hq, Hkv, W, R, alpha,
                                        scale_log2, part);
    rows_per_tile = kRowsPerCta;
  }
  cudaError_t e = post_launch(__func__, st);
  if (e != cudaSuccess) return e;
  k_score_reduce<<<dim3((S + 255) / 256, B), 256, 0, st>>>(tokens, delim_ids, n_ids, part, Ls, B, S,
                                                           Hq, W, rows_per_tile, out);
  return post_launch(__func__, st);
}

}  // namespace dsk
extern "C" int dynsplit_debug_a1_mmasync(int on) {
  dsk::g_a1_mmasync = on != 0;
  return 0;
}
