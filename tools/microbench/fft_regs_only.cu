// How fast does the register-only part of K1d's transform run?  twist + dft16 + twiddle + dft16 in a loop,
// no shared memory, no tensor memory: FP64 warp-instructions per clock per scheduler at 8 / 12 / 16 warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2005_01945_b200/csrc -o fft_regs_only fft_regs_only.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "tfhe_warp.cuh"
using namespace tfb;
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k(cd* io, int iters) {
  cd x[16], w[4];
  const int t = threadIdx.x;
#pragma unroll
  for (int m = 0; m < 16; ++m) x[m] = io[t + MAXT * m];
#pragma unroll
  for (int m = 0; m < 4; ++m) w[m] = io[t + MAXT * (16 + m)];
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int m = 1; m < 16; ++m) x[m] = cmul(x[m], twist16(m));
    dft16<1>(x);
#pragma unroll
    for (int m = 0; m < 16; ++m) x[m] = cmul(x[m], w[m & 3]);
    dft16<1>(x);
  }
#pragma unroll
  for (int m = 0; m < 16; ++m) io[t + MAXT * m] = x[m];
}
template <int MAXT>
void run() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cd* io;
  cudaMalloc(&io, sizeof(cd) * MAXT * 20);
  cudaMemset(io, 0, sizeof(cd) * MAXT * 20);
  const int iters = 20000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k<MAXT><<<sms, MAXT>>>(io, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  cudaEventElapsedTime(&ms, a, b);
  const double fp64 = 60 + 160 + 64 + 160;  // per iteration per thread
  const double clks = ms * 1e-3 * clk * 1e3;
  printf("%2d warps/SM: %.3f FP64 warp-instr/clk/scheduler (%.0f clk per iteration)\n", MAXT / 32,
         fp64 * iters * (MAXT / 32) / clks / 4, clks / iters);
  cudaFree(io);
}
int main() {
  run<256>();
  run<384>();
  run<512>();
  return 0;
}
