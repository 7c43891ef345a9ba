// Shared device helpers for the DynSplit-KV sm_100a kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#define DSK_DEVICE __device__ __forceinline__

namespace dsk {

constexpr int kD = 128;          // head dim (checked at the ABI)
constexpr int kMaxG = 8;         // query heads per KV head
constexpr int kMaxSplit = 64;    // split-K partials per (b, KV head)

typedef __nv_bfloat16 bf16;

// Every workspace starts with a header of kWsHdr bytes; its first int32 is the
// device error word (DYNSPLIT_DEVERR_* bits of include/dynsplit.h).
constexpr size_t kWsHdr = 256;
enum : int {
  kErrPlanCoverage = 1,   // DYNSPLIT_DEVERR_PLAN_COVERAGE
  kErrPlanMismatch = 2,   // DYNSPLIT_DEVERR_PLAN_MISMATCH
  kErrPageCapacity = 4,   // DYNSPLIT_DEVERR_PAGE_CAPACITY
  kErrSelectOverflow = 8, // DYNSPLIT_DEVERR_SELECT_OVERFLOW
  kErrBlockTooLong = 16,  // DYNSPLIT_DEVERR_BLOCK_TOO_LONG
  kErrSyncTimeout = 32    // DYNSPLIT_DEVERR_SYNC_TIMEOUT
};
__device__ __forceinline__ void raise_err(int* err, int bit) {
  if (err) atomicOr(err, bit);
}

// One worklist entry: a page of one (b, KV head) and, per packed query head
// of the group, how many leading rows of the page that head attends to.
struct __align__(16) WLEntry {
  int32_t page;
  int32_t block;
  uint8_t rows[kMaxG];
};

// ---------------------------------------------------------------- conversions
DSK_DEVICE float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
DSK_DEVICE float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <typename T> struct Vec;
template <> struct Vec<bf16> {
  // 4 elements = 8 bytes
  static DSK_DEVICE void load4(const bf16* p, float (&x)[4]) {
    uint2 u = *reinterpret_cast<const uint2*>(p);
    x[0] = bf_lo(u.x); x[1] = bf_hi(u.x); x[2] = bf_lo(u.y); x[3] = bf_hi(u.y);
  }
  // 8 elements = 16 bytes
  static DSK_DEVICE void load8(const bf16* p, float (&x)[8]) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    x[0] = bf_lo(u.x); x[1] = bf_hi(u.x); x[2] = bf_lo(u.y); x[3] = bf_hi(u.y);
    x[4] = bf_lo(u.z); x[5] = bf_hi(u.z); x[6] = bf_lo(u.w); x[7] = bf_hi(u.w);
  }
  static DSK_DEVICE void load8_nc(const bf16* p, float (&x)[8]) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    x[0] = bf_lo(u.x); x[1] = bf_hi(u.x); x[2] = bf_lo(u.y); x[3] = bf_hi(u.y);
    x[4] = bf_lo(u.z); x[5] = bf_hi(u.z); x[6] = bf_lo(u.w); x[7] = bf_hi(u.w);
  }
};
template <> struct Vec<float> {
  static DSK_DEVICE void load4(const float* p, float (&x)[4]) {
    float4 u = *reinterpret_cast<const float4*>(p);
    x[0] = u.x; x[1] = u.y; x[2] = u.z; x[3] = u.w;
  }
  static DSK_DEVICE void load8(const float* p, float (&x)[8]) {
    float4 a = reinterpret_cast<const float4*>(p)[0];
    float4 b = reinterpret_cast<const float4*>(p)[1];
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  }
  static DSK_DEVICE void load8_nc(const float* p, float (&x)[8]) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  }
};

// bf16 x bf16 -> fp32 fused multiply-add (FHFMA.BF16; the product is exact).
DSK_DEVICE float fma_bf16(unsigned short a, unsigned short b, float c) {
  float r;
  asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(r) : "h"(a), "h"(b), "f"(c));
  return r;
}
// halves of a packed bf16x2 word (free: becomes .H0/.H1 operand selectors)
DSK_DEVICE void split_bf16x2(uint32_t w, unsigned short& lo, unsigned short& hi) {
  asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(w));
}

// Order-preserving map fp32 -> uint32 (larger float -> larger key).
DSK_DEVICE uint32_t float_key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

DSK_DEVICE float key_to_float(uint32_t k) {
  const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// ---------------------------------------------------------------- warp utils
DSK_DEVICE float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
DSK_DEVICE float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
DSK_DEVICE int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
DSK_DEVICE int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan of N ints per thread (NT threads); tot = totals.
// sm: (NT/32 + 1) * N ints of shared memory.  Contains __syncthreads.
template <int N, int NT>
DSK_DEVICE void block_excl_scan(int (&v)[N], int (&tot)[N], int* sm) {
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

// ---------------------------------------------------------------- smem / mbarrier / bulk copy
DSK_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
DSK_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
DSK_DEVICE void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
DSK_DEVICE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
DSK_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps until the phase
// completes (or ~1 ms) instead of spinning and stealing issue slots from the
// warps that do the work.
DSK_DEVICE bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u) : "memory");
  return ok != 0;
}
DSK_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// TMA 1-D bulk copy global -> shared, completion signalled on `bar` (bytes % 16 == 0).
DSK_DEVICE void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// 16-byte cp.async (LDGSTS, bypassing L1).  No L2 cache-policy hint: ptxas
// 12.9 mis-encodes two back-to-back hinted LDGSTS with an odd uniform
// descriptor register (illegal instruction at run time).
DSK_DEVICE void cp_async16_cg(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem)
               : "memory");
}
DSK_DEVICE uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
DSK_DEVICE uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Programmatic dependent launch: wait until the preceding kernel in the
// stream has completed (and its writes are visible) / allow the next kernel
// to be scheduled.  Both are no-ops for a normal launch.
DSK_DEVICE void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
DSK_DEVICE void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- mma.sync (bf16 in, fp32 accumulate) helpers shared by a5 and a7
DSK_DEVICE void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
// c += A * B for one m16n8k16 tile whose A rows 8..15 are zero (a1 = a3 = 0):
// a0 = A[g][2t, 2t+1], a2 = A[g][2t+8, 2t+9]; b0/b1 the usual col-major B halves.
DSK_DEVICE void mma_rows8(float (&c)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

// TMA 2-D tensor copy global -> shared (box given by the tensor map),
// completion signalled on `bar`.
DSK_DEVICE void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

DSK_DEVICE void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace dsk
