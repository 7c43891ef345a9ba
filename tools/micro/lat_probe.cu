// Dependent-chain latencies of warp-collective instructions on sm_100a
// (one warp, clock64): REDUX.SUM (__reduce_add_sync), SHFL, VOTE, LDS.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void kl(int* out, long long* cyc, int seed) {
  __shared__ int sm[1024];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int v = seed + lane;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    if (OP == 0) v = __reduce_add_sync(0xffffffffu, v) & 1023;
    if (OP == 1) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
    if (OP == 2) v = (int)__ballot_sync(0xffffffffu, v & 1) + lane;
    if (OP == 3) v = sm[v & 1023];
    if (OP == 4) v = __reduce_min_sync(0xffffffffu, (unsigned)v) + 1;
    if (OP == 5) v = v * 3 + 1;
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 32 + threadIdx.x / 32] = (t1 - t0) / 256;
  out[threadIdx.x] = v;
}

int main() {
  int* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * 4);
  cudaMalloc(&cyc, 4096 * 8);
  const char* names[] = {"REDUX.SUM", "SHFL", "VOTE(ballot)", "LDS", "REDUX.MIN", "IMAD"};
  auto go = [&](auto k, int i) {
    for (int warps : {1, 8}) {
      k<<<1, 32 * warps>>>(out, cyc, 3);
      cudaDeviceSynchronize();
      long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%-13s warps/CTA %d: %lld cycles per dependent step\n", names[i], warps, h);
    }
  };
  go(kl<0>, 0);
  go(kl<1>, 1);
  go(kl<2>, 2);
  go(kl<3>, 3);
  go(kl<4>, 4);
  go(kl<5>, 5);
  return 0;
}
