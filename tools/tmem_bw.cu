// TMEM <-> register bandwidth microbenchmark (sm_100a): 16 warps, each warp
// streams its lane quadrant with tcgen05.ld/st 32x32b.x32.  Prints bytes per
// SM clock for loads and stores.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(512, 1) k(unsigned long long* out, int iters, uint32_t* sink) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 7 + i;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t a = base + (uint32_t)(((it * 4 + (warp >> 2)) * 32) & 511);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" :: "r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  __syncthreads();
  long long t1 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t a = base + (uint32_t)(((it * 4 + (warp >> 2)) * 32) & 511);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]) : "r"(a) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 32; ++i) acc += v[i];
  }
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t1; }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(taddr_s));
}
int main() {
  unsigned long long* d; uint32_t* s; cudaMalloc(&d, 148 * 16); cudaMalloc(&s, 148 * 512 * 4);
  const int iters = 4096;
  k<<<148, 512>>>(d, iters, s); cudaDeviceSynchronize();
  k<<<148, 512>>>(d, iters, s);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double bytes = 16.0 * 32 * 4 * 32 * iters;  // 16 warps x 32 lanes x N words
  printf("err=%s  st: %.1f B/clk/SM  ld(+wait each): %.1f B/clk/SM\n", cudaGetErrorString(e), bytes / h[0], bytes / h[1]);
  return 0;
}
