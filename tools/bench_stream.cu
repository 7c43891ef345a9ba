// Streaming microbenchmark (not part of the product): how fast can an SM
// array pull scattered 4 KiB chunks (the K or V rows of one 16-row bf16 page)
// from HBM into shared memory, by mechanism?
//   mode 0: LDGSTS (16-byte cp.async), per-warp pipeline of `depth` chunks
//   mode 1: TMA 1-D bulk copy (cp.async.bulk), one issuing lane per warp,
//           mbarrier per stage, `depth` stages per warp
//   mode 2: LDG.128 into registers (xor-reduced so the loads are live)
// Chunks: n_chunks random 4 KiB-aligned offsets in a 2 GiB buffer, L2
// flushed (256 MiB write) before every timed launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bs tools/bench_stream.cu
//   /tmp/bs
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int CHUNK = 4096;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k_stream(const unsigned char* __restrict__ buf, const int64_t* __restrict__ offs, int n_chunks,
                         int depth, unsigned* __restrict__ sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + warp, tw = gridDim.x * nw;
  unsigned char* ring = smem + (size_t)warp * depth * CHUNK;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nw * depth * CHUNK) + warp * depth;
  unsigned acc = 0;
  const int n_mine = gw < n_chunks ? (n_chunks - gw + tw - 1) / tw : 0;
  if (MODE == 0) {
    auto issue = [&](int j) {
      if (j < n_mine) {
        const unsigned char* src = buf + offs[gw + (size_t)j * tw];
        unsigned char* dst = ring + (j % depth) * CHUNK;
        for (int c = lane; c < CHUNK / 16; c += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + c * 16)), "l"(src + c * 16) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int j = 0; j < depth; ++j) issue(j);
    for (int j = 0; j < n_mine; ++j) {
      switch (depth) {
        case 1: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        case 4: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
        case 6: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 7;" ::: "memory"); break;
      }
      __syncwarp();
      acc ^= reinterpret_cast<const unsigned*>(ring + (j % depth) * CHUNK)[lane];
      __syncwarp();
      issue(j + depth);
    }
  } else if (MODE == 1) {
    if (lane == 0)
      for (int s = 0; s < depth; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])) : "memory");
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    auto issue = [&](int j) {
      if (j < n_mine && lane == 0) {
        const unsigned char* src = buf + offs[gw + (size_t)j * tw];
        const int s = j % depth;
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(CHUNK) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(ring + s * CHUNK)), "l"(src), "r"(CHUNK), "r"(smem_u32(&bars[s])) : "memory");
      }
    };
    for (int j = 0; j < depth; ++j) issue(j);
    for (int j = 0; j < n_mine; ++j) {
      const int s = j % depth;
      const uint32_t par = (j / depth) & 1;
      uint32_t ok = 0;
      while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bars[s])), "r"(par) : "memory");
      }
      acc ^= reinterpret_cast<const unsigned*>(ring + s * CHUNK)[lane];
      __syncwarp();
      issue(j + depth);
    }
  } else {
    for (int j = 0; j < n_mine; j += depth) {
      uint4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        v[k] = make_uint4(0, 0, 0, 0);
        if (k < depth && j + k < n_mine) {
          const uint4* src = reinterpret_cast<const uint4*>(buf + offs[gw + (size_t)(j + k) * tw]);
          // each lane: 8 x 16 B of the 4 KiB chunk
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 x = __ldcs(src + lane + 32 * c);
            v[k].x ^= x.x; v[k].y ^= x.y; v[k].z ^= x.z; v[k].w ^= x.w;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  const size_t BUF = 2ull << 30;
  unsigned char* buf;
  CK(cudaMalloc(&buf, BUF));
  CK(cudaMemset(buf, 1, BUF));
  unsigned char* flush;
  CK(cudaMalloc(&flush, 256 << 20));
  unsigned* sink;
  CK(cudaMalloc(&sink, 4));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int n_max = 196608;  // up to 768 MiB
  int n_chunks = n_max;
  std::vector<int64_t> h(n_max);
  std::mt19937_64 rng(1);
  for (auto& x : h) x = (int64_t)(rng() % (BUF / CHUNK)) * CHUNK;
  int64_t* offs;
  CK(cudaMalloc(&offs, n_max * 8));
  CK(cudaMemcpy(offs, h.data(), n_max * 8, cudaMemcpyHostToDevice));
  // sequential variant
  std::vector<int64_t> hs(n_max);
  for (int i = 0; i < n_max; ++i) hs[i] = (int64_t)i * CHUNK;
  int64_t* offs_seq;
  CK(cudaMalloc(&offs_seq, n_max * 8));
  CK(cudaMemcpy(offs_seq, hs.data(), n_max * 8, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto run = [&](int mode, int ctas_per_sm, int nw, int depth, const int64_t* o, const char* tag, int grid = 0) {
    size_t smem = (size_t)nw * depth * CHUNK + nw * depth * 8;
    void (*k)(const unsigned char*, const int64_t*, int, int, unsigned*) =
        mode == 0 ? k_stream<0> : mode == 1 ? k_stream<1> : k_stream<2>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    if (mode == 2) smem = 0;
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemsetAsync(flush, rep, 256 << 20));
      CK(cudaEventRecord(a));
      k<<<grid ? grid : sms * ctas_per_sm, nw * 32, smem>>>(buf, o, n_chunks, depth, sink);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    printf("%-4s mode %d  ctas/sm %d  grid %4d  warps %2d  depth %d  smem %6zu : %7.2f us  %7.0f GB/s\n", tag, mode,
           ctas_per_sm, grid ? grid : sms * ctas_per_sm, nw, depth, smem, best * 1e3,
           (double)n_chunks * CHUNK / (best * 1e-3) / 1e9);
  };
  // empty-kernel reference
  {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(a));
      k_stream<0><<<sms * 3, 128, 0>>>(buf, offs, 0, 2, sink);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    printf("empty kernel: %.2f us\n", best * 1e3);
  }
  // fewer SMs streaming (one 8- or 16-warp CTA per SM on a subset of the SMs)
  n_chunks = 12288;
  printf("--- 12288 chunks (48 MiB), SM subsets\n");
  for (int grid : {64, 72, 96, 128, 144})
    for (int depth : {2, 3}) run(0, 1, 8, depth, offs, "rand", grid);
  for (int grid : {72, 144}) run(0, 1, 16, 3, offs, "rand", grid);
  for (int n : {12288, 49152, 196608}) {
    n_chunks = n;
    printf("--- %d chunks (%d MiB)\n", n, n * 4 / 1024);
    for (const int64_t* o : {offs, offs_seq}) {
      const char* tag = o == offs ? "rand" : "seq";
      run(0, 3, 4, 2, o, tag);
      run(0, 3, 4, 4, o, tag);
      run(0, 1, 16, 3, o, tag);
      run(1, 3, 4, 4, o, tag);
      run(1, 1, 16, 3, o, tag);
      run(2, 4, 8, 4, o, tag);
    }
  }
  return 0;
}
