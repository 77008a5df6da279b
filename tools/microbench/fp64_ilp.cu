// FP64 pipe rate per scheduler as a function of resident warps and independent chains per thread:
// how much instruction-level parallelism a warp needs to keep the DFMA pipe busy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_ilp fp64_ilp.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CHAINS>
__global__ void k(double* out, int iters, double m, double c) {
  double a[CHAINS];
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) a[j] = threadIdx.x * 1e-9 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16 / CHAINS; ++r)
#pragma unroll
      for (int j = 0; j < CHAINS; ++j) a[j] = fma(a[j], m, c);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CHAINS>
void run(int threads) {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 8 * sms * threads);
  const int iters = 20000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k<CHAINS><<<sms, threads>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  cudaEventElapsedTime(&ms, a, b);
  const double inst = (double)iters * 16 * (threads / 32);
  const double clks = ms * 1e-3 * clk * 1e3;
  printf("warps/scheduler %d  chains %2d : %.3f DFMA/clk/scheduler  (%.1f clk between a warp's DFMAs)\n", threads / 128,
         CHAINS, inst / clks / 4, clks / ((double)iters * 16));
  cudaFree(out);
}
int main() {
  for (int th : {128, 256, 384, 512}) {
    if (th == 128) { run<1>(128); run<2>(128); run<4>(128); run<8>(128); run<16>(128); }
    if (th == 256) { run<1>(256); run<2>(256); run<4>(256); run<8>(256); }
    if (th == 384) { run<1>(384); run<2>(384); run<4>(384); run<8>(384); }
    if (th == 512) { run<1>(512); run<2>(512); run<4>(512); }
  }
  return 0;
}
