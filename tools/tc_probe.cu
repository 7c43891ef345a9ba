// tcgen05 probe (not part of the product): D[128x128] = A[128x128] . B[128x128]^T
// in bf16 -> fp32 through one CTA, checked against a CPU product.  Validates
// the smem (K-major, 128-byte swizzle) and instruction descriptors used by the
// prefill scoring kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tcp tools/tc_probe.cu && /tmp/tcp
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, SWIZZLE_128B smem matrix descriptor: rows of 128 B, 8-row atoms of
// 1024 B (SBO), LBO unused, version 1, layout type 2.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void k_probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  extern __shared__ __align__(1024) unsigned char smem[];
  // sA: 2 K-halves x 128 rows x 128 B (swizzled), sB likewise
  unsigned char* sA = smem;
  unsigned char* sB = smem + 2 * 128 * 128;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // load: 128 rows x 16 chunks of 16 B per matrix; chunk c of row r -> half c/8, pos (c%8) ^ (r%8)
  for (int e = tid; e < 128 * 16; e += blockDim.x) {
    const int r = e >> 4, c = e & 15;
    const int half = c >> 3, cp = (c & 7) ^ (r & 7);
    *reinterpret_cast<uint4*>(sA + half * 16384 + r * 128 + cp * 16) = reinterpret_cast<const uint4*>(A + r * 128)[c];
    *reinterpret_cast<uint4*>(sB + half * 16384 + r * 128 + cp * 16) = reinterpret_cast<const uint4*>(B + r * 128)[c];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy smem writes -> async proxy
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    for (int k = 0; k < 8; ++k) {
      const uint32_t off = (uint32_t)((k >> 2) * 16384 + (k & 3) * 32);
      const uint64_t da = sdesc(su32(sA) + off), db = sdesc(su32(sB) + off);
      const uint32_t acc = k > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                   ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  // wait for the MMAs
  {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar)) : "memory");
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t v[32];
      const uint32_t addr = tm + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                   "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                     "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                     "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int row = 32 * warp + lane;
      for (int j = 0; j < 32; ++j) D[row * 128 + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128));
}

int main() {
  std::vector<__nv_bfloat16> hA(128 * 128), hB(128 * 128);
  std::vector<float> fA(128 * 128), fB(128 * 128);
  srand(1);
  for (int i = 0; i < 128 * 128; ++i) {
    fA[i] = (float)(rand() % 17 - 8);
    fB[i] = (float)(rand() % 17 - 8);
    hA[i] = __float2bfloat16(fA[i]);
    hB[i] = __float2bfloat16(fB[i]);
  }
  __nv_bfloat16 *dA, *dB;
  float* dD;
  CK(cudaMalloc(&dA, 128 * 128 * 2));
  CK(cudaMalloc(&dB, 128 * 128 * 2));
  CK(cudaMalloc(&dD, 128 * 128 * 4));
  CK(cudaMemcpy(dA, hA.data(), 128 * 128 * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), 128 * 128 * 2, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, 128 * 128 * 4));
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384 + 1024));
  k_probe<<<1, 128, 4 * 16384 + 1024>>>(dA, dB, dD);
  CK(cudaDeviceSynchronize());
  std::vector<float> hD(128 * 128);
  CK(cudaMemcpy(hD.data(), dD, 128 * 128 * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  double maxerr = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double ref = 0;
      for (int k = 0; k < 128; ++k) ref += (double)fA[i * 128 + k] * fB[j * 128 + k];
      const double err = fabs(ref - hD[i * 128 + j]);
      maxerr = fmax(maxerr, err);
      if (err > 1e-3 && bad++ < 5) printf("mismatch D[%d][%d] = %f, ref %f\n", i, j, hD[i * 128 + j], ref);
    }
  printf("tcgen05 probe: %s (max abs err %.3g, %d bad)\n", bad ? "FAIL" : "OK", maxerr, bad);
  return bad != 0;
}
