// Microbenchmark: FP64 FMA throughput vs ILP at 16 warps/SM, and dependent
// latencies (DFMA chain, double shuffle chain, LDS chain).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void fma_ilp(double* out, int iters) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], 0.999999, 1e-7);
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 1.2345) out[0] = s;
}
__global__ void lat(double* out, long long* cyc, int iters) {
  double x = threadIdx.x * 1e-3 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-7);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  if (x == 1.2345) out[0] = x;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  long long* c; cudaMalloc(&c, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  auto run = [&](auto k, int ch, int threads) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k<<<148, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("threads/SM %d chains %d: %.2f TF/s\n", threads, ch, 2.0 * ch * iters * 148.0 * threads / ms / 1e9);
    }
  };
  run(fma_ilp<1>, 1, 512); run(fma_ilp<2>, 2, 512); run(fma_ilp<4>, 4, 512); run(fma_ilp<8>, 8, 512);
  run(fma_ilp<1>, 1, 1024); run(fma_ilp<4>, 4, 1024); run(fma_ilp<8>, 8, 256);
  lat<<<1, 32>>>(d, c, 1000); cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("dependent DFMA latency %.1f cyc, dependent double shfl+add %.1f cyc\n", h[0] / 1000.0, h[1] / 1000.0);
  return 0;
}
