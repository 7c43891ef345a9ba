// Micro-benchmark of f_band_select (the fused kernel's exact marginal search
// inside a band of ~190 entries), 4 warps = 4 heads per CTA, clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2602_03184_b200/csrc \
//        -o band_bench band_bench.cu -lcuda
#include <cstdio>
#include <cstring>
#include "fused_kernels.cu"

using namespace dsk;

__global__ void __launch_bounds__(256, 1) kband(const uint2* band_g, const int32_t* sbs_g, long long* out, int cnt,
                                                int need) {
  __shared__ uint2 sb[4][kBandCap];
  __shared__ int32_t sbs[4200];
  __shared__ uint32_t bits[4][160];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4 * kBandCap; i += 256) sb[i / kBandCap][i % kBandCap] = band_g[i % kBandCap];
  for (int i = tid; i < 4200; i += 256) sbs[i] = sbs_g[i];
  for (int i = tid; i < 4 * 160; i += 256) bits[i / 160][i % 160] = 0;
  __syncthreads();
  // sub-band weights of the band (16 sub-bands of the key range, as the classification does)
  __shared__ int wsub[16];
  if (tid < 16) wsub[tid] = 0;
  __syncthreads();
  if (tid < cnt) atomicAdd(&wsub[sb[0][tid].y >> 24], sbs[(sb[0][tid].y & 0xffffff) + 1] - sbs[sb[0][tid].y & 0xffffff]);
  __syncthreads();
  const int lane = tid & 31;
  const int wsb = lane < 16 ? wsub[lane] : 0;
  __syncthreads();
  long long t0 = clock64();
  int m = 0, keep = 0;
  uint32_t T = 0;
  if (warp < 4) f_band_select(sb[warp], cnt, wsb, sbs, need, bits[warp], m, keep, T);
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (tid == 0 && blockIdx.x == 0) out[200] = m, out[201] = keep, out[202] = T;
}

int main() {
  const int cnt = 190;
  uint2 h[kBandCap];
  int32_t hs[4200];
  for (int i = 0; i < 4200; ++i) hs[i] = i * 32 + (i * 7) % 11;
  unsigned s = 7;
  for (int i = 0; i < kBandCap; ++i) {
    s = s * 1664525u + 1013904223u;
    const float x = 330.f + 15.f * ((s >> 8) / 16777216.f);
    uint32_t u;
    memcpy(&u, &x, 4);
    const int sbi = (int)((x - 330.f) / 15.f * 16.f);
    h[i] = make_uint2(u | 0x80000000u, (uint32_t)(i * 20 + (s & 15)) | ((uint32_t)(sbi > 15 ? 15 : sbi) << 24));
  }
  uint2* band;
  int32_t* sbs;
  long long* out;
  cudaMalloc(&band, sizeof(h));
  cudaMalloc(&sbs, sizeof(hs));
  cudaMalloc(&out, 300 * 8);
  cudaMemcpy(band, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemcpy(sbs, hs, sizeof(hs), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) kband<<<144, 256>>>(band, sbs, out, cnt, 2000);
  cudaDeviceSynchronize();
  long long ho[300];
  cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  long long mx = 0, sum = 0;
  for (int i = 0; i < 144; ++i) { mx = ho[i] > mx ? ho[i] : mx; sum += ho[i]; }
  printf("f_band_select (4 heads, %d entries): cycles mean %lld max %lld; m %lld keep %lld  (%s)\n", cnt, sum / 144,
         mx, ho[200], ho[201], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
