// Does an FP64 instruction occupy the scheduler's issue port for one cycle or for two?
// Interleave R integer instructions per DFMA (independent chains) and compare the time with the two models
//   port 1 cycle : max(2 N_dfma, N_dfma + N_int)      port 2 cycles: 2 N_dfma + N_int
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_coissue fp64_coissue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int R>
__global__ void k(double* out, int iters, double m, double c, uint32_t q) {
  double a[8];
  uint32_t b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x * 1e-9 + j; b[j] = threadIdx.x + j; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a[j] = fma(a[j], m, c);
#pragma unroll
      for (int r = 0; r < R; ++r) b[(j + r) & 7] = (b[(j + r) & 7] ^ q) + (uint32_t)r;  // LOP3 + IADD: 2 int instr
    }
  }
  double s = 0;
  uint32_t u = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { s += a[j]; u += b[j]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + u;
}
template <int R>
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
    k<R><<<sms, threads>>>(out, iters, 1.0000001, 1e-7, 12345u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  cudaEventElapsedTime(&ms, a, b);
  const double clks = ms * 1e-3 * clk * 1e3;
  const double w = threads / 128.0;  // warps per scheduler
  const double nd = iters * 8.0 * w, ni = nd * 2 * R;
  printf("warps/sched %.0f, %d int per DFMA: %.0f clk; model port-1: %.0f, model port-2: %.0f  (dfma/clk %.3f)\n", w, 2 * R,
         clks, (2 * nd > nd + ni ? 2 * nd : nd + ni), 2 * nd + ni, nd / clks);
  cudaFree(out);
}
int main() {
  run<0>(384); run<1>(384); run<2>(384); run<3>(384);
  run<1>(256); run<1>(512);
  return 0;
}
