// Shared-memory load / store throughput on one SM-full of warps (conflict-free 128-bit accesses),
// to calibrate the LSU budget of kernel K1.  nvcc -arch=sm_100a -O3 -o smem_bw smem_bw.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>  // 0 = loads, 1 = stores, 2 = 1:1 mix
__global__ void k(double2* out, int iters) {
  extern __shared__ double2 sm[];
  const int t = threadIdx.x;
  double2 acc = make_double2(t, 1.0);
  for (int i = t; i < 4096; i += blockDim.x) sm[i] = acc;
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int idx = (t + 256 * j + it) & 4095;
      if (MODE == 0 || (MODE == 2 && (j & 1))) {
        double2 v = sm[idx];
        acc.x += v.x;
        acc.y += v.y;
      } else {
        sm[idx] = acc;
      }
    }
  }
  out[blockIdx.x * blockDim.x + t] = acc;
}
template <int MODE>
void run(const char* name) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double2* out;
  cudaMalloc(&out, sizeof(double2) * sms * 4 * 256);
  const int iters = 20000;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k<MODE><<<sms * 3, 256, 65536>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double bytes = (double)sms * 3 * 256 * iters * 8 * 16;
  printf("%-8s %.1f GB/s total, %.1f B/clk/SM at %d MHz nominal\n", name, bytes / ms / 1e6,
         bytes / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  cudaFree(out);
}
int main() {
  run<0>("loads");
  run<1>("stores");
  run<2>("mix 1:1");
  return 0;
}
