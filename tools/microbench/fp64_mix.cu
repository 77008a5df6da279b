// FP64 pipe throughput by instruction kind (DFMA / DADD / DMUL and the mix K1 executes).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters, double m, double c) {
  double a[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = threadIdx.x * 1e-9 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (MODE == 0) a[j] = fma(a[j], m, c);
      if (MODE == 1) a[j] = a[j] + c;
      if (MODE == 2) a[j] = a[j] * m;
      if (MODE == 3) {  // 2 DADD : 1 DFMA : 1 DMUL
        if ((j & 3) < 2) a[j] = a[j] + c;
        else if ((j & 3) == 2) a[j] = fma(a[j], m, c);
        else a[j] = a[j] * m;
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(const char* name, int threads) {
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
    k<MODE><<<sms, threads>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  cudaEventElapsedTime(&ms, a, b);
  const double inst = (double)iters * 16 * (threads / 32);  // warp instructions per SM
  const double clks = ms * 1e-3 * clk * 1e3;
  printf("%-10s %4d thr/SM  %7.3f ms  %.3f warp-instr/clk/SM  (%.3f per scheduler)\n", name, threads, ms, inst / clks,
         inst / clks / 4);
  cudaFree(out);
}
int main() {
  for (int th : {256, 384, 1024}) {
    if (th == 256) { run<0>("DFMA", 256); run<1>("DADD", 256); run<2>("DMUL", 256); run<3>("mix 2:1:1", 256); }
    if (th == 384) { run<0>("DFMA", 384); run<1>("DADD", 384); run<2>("DMUL", 384); run<3>("mix 2:1:1", 384); }
    if (th == 1024) { run<0>("DFMA", 1024); run<1>("DADD", 1024); run<2>("DMUL", 1024); run<3>("mix 2:1:1", 1024); }
  }
  return 0;
}
