// Phase probe of the latency kernel K1c (one gate over four 64-thread groups): clock64 at the phase
// boundaries of a CMux, averaged over the 500 iterations, printed for groups 0 and 3 of CTA 0.
// Timing only (random key material).   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o k1c_probe k1c_probe.cu
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include "../../paper_2005_01945_b200/csrc/tfhe_device.cuh"
using namespace tfb;
namespace tfb {
#undef TFB_HD
#define TFB_HD __device__ __forceinline__
template <class GroupSync, class CtaSync, class LoadBk>
TFB_HD void gate_bootstrap_wide_probe(const uint32_t* x_row, const uint32_t* y_row, int kind, int n, uint32_t mu,
                                const cd* bkf, const Twiddles* tw, uint32_t* sm_acc, uint16_t* sm_abar,
                                cd* xbuf, cd* red, uint32_t* ext, int tid, GroupSync& gsync, CtaSync& csync,
                                LoadBk load) {
  constexpr int WIDE = 4 * FFT_THREADS;
  const int q = tid / FFT_THREADS, t = tid % FFT_THREADS;
  const int p = q / BK_L, lvl = q % BK_L;
  cd* bufA = xbuf + (size_t)q * 2 * HALF_N;
  cd* bufB = bufA + HALF_N;
  bootstrap_prologue(x_row, y_row, kind, n, mu, sm_acc, sm_abar, tid, WIDE, csync);
  RegTw rtw;
  rtw.load(tw, t);
  long long T[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long c0 = clock64(), c1;
#define TICK(k) c1 = clock64(); T[k] += c1 - c0; c0 = c1;
  // Output polynomial c is inverse-transformed by group c.  A group keeps the product that
  // stays with it in registers and publishes only what another group needs:
  // red[q][c] is written for every (q, c) except (0, 0) and (1, 1).
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    const int abar = sm_abar[i];
    if (abar == 0) continue;  // uniform across the CTA
    const cd* stage = bkf + stage_offset(i, p);
    cd b0[8], b1[8];
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      b0[k2] = load(stage + stage_index(k2, lvl, 0, t));
      b1[k2] = load(stage + stage_index(k2, lvl, 1, t));
    }
    TICK(0)
    cd x[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const uint32_t vr = rotated_diff(sm_acc + p * RING_N, t + 64 * m, abar) + DECOMP_OFFSET;
      const uint32_t vi = rotated_diff(sm_acc + p * RING_N, t + 64 * m + HALF_N, abar) + DECOMP_OFFSET;
      x[m] = cd{digit_to_double(digit_field(vr, lvl)), digit_to_double(digit_field(vi, lvl))};
    }
    TICK(1)
    fft_forward(x, t, rtw, bufA, bufB, gsync);
    TICK(2)
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      const cd p0 = cmul(x[k2], b0[k2]), p1 = cmul(x[k2], b1[k2]);
      if (q != 0) red[((q * 2 + 0) * 8 + k2) * FFT_THREADS + t] = p0;
      if (q != 1) red[((q * 2 + 1) * 8 + k2) * FFT_THREADS + t] = p1;
      x[k2] = (q == 0) ? p0 : p1;  // meaningful for q < 2: the product this group keeps
    }
    TICK(3)
    csync();
    TICK(4)
    if (q < 2) {  // output polynomial c = q
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        cd s = x[k2];
#pragma unroll
        for (int o = 0; o < 4; ++o)
          if (o != q) s = cadd(s, red[((o * 2 + q) * 8 + k2) * FFT_THREADS + t]);
        x[k2] = s;
      }
      TICK(5)
      fft_inverse(x, t, rtw, bufA, bufB, gsync);
      TICK(6)
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        sm_acc[q * RING_N + t + 64 * m] += round_to_word(x[m].re);
        sm_acc[q * RING_N + t + 64 * m + HALF_N] += round_to_word(x[m].im);
      }
    }
    csync();
    TICK(7)
  }
  if (t == 0 && (q == 0 || q == 3))
    printf("grp %d: keyload %lld decomp %lld fwd %lld mac %lld sync1 %lld reduce %lld inv %lld upd+sync2 %lld (cycles per CMux)\n", q,
           T[0] / n, T[1] / n, T[2] / n, T[3] / n, T[4] / n, T[5] / n, T[6] / n, T[7] / n);
  bootstrap_extract(sm_acc, ext, tid, WIDE);
}


}  // namespace tfb
struct BlockSync { __device__ __forceinline__ void operator()() const { __syncthreads(); } };
struct GroupSync {
  int id;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(FFT_THREADS) : "memory"); }
};
struct LdgLoad {
  __device__ __forceinline__ cd operator()(const cd* q) const { const double2 v = __ldg(reinterpret_cast<const double2*>(q)); return cd{v.x, v.y}; }
};
constexpr int K1C_THREADS = 4 * FFT_THREADS;
__host__ __device__ constexpr int k1c_smem(int n) {
  return (int)sizeof(Twiddles) + 16 * HALF_N * (int)sizeof(cd) + 2 * RING_N * (int)sizeof(uint32_t) + ((n + 1) * 2 + 15) / 16 * 16;
}
__global__ void __launch_bounds__(K1C_THREADS, 1) k_probe(const uint32_t* pool, int n, uint32_t mu, const cd* bkf, const Twiddles* tw_global, uint32_t* ext) {
  extern __shared__ __align__(128) unsigned char smem[];
  Twiddles* tw = reinterpret_cast<Twiddles*>(smem);
  cd* xbuf = reinterpret_cast<cd*>(smem + sizeof(Twiddles));
  cd* red = xbuf + 8 * HALF_N;
  uint32_t* acc = reinterpret_cast<uint32_t*>(red + 8 * HALF_N);
  uint16_t* abar = reinterpret_cast<uint16_t*>(acc + 2 * RING_N);
  for (int i = threadIdx.x; i < (int)(sizeof(Twiddles) / sizeof(cd)); i += K1C_THREADS)
    reinterpret_cast<cd*>(tw)[i] = reinterpret_cast<const cd*>(tw_global)[i];
  const int64_t g = blockIdx.x;
  GroupSync gsync{(int)(threadIdx.x / FFT_THREADS) + 1};
  BlockSync csync;
  if (blockIdx.x == 0)
    gate_bootstrap_wide_probe(pool + 2 * g * 512, pool + (2 * g + 1) * 512, 2, n, mu, bkf, tw, acc, abar, xbuf, red, ext + g * EXT_STRIDE, (int)threadIdx.x, gsync, csync, LdgLoad());
  else
    gate_bootstrap_wide(pool + 2 * g * 512, pool + (2 * g + 1) * 512, 2, n, mu, bkf, tw, acc, abar, xbuf, red, ext + g * EXT_STRIDE, (int)threadIdx.x, gsync, csync, LdgLoad());
}
int main() {
  const int n = 500, gates = 148;
  std::vector<uint32_t> pool((size_t)2 * gates * 512);
  for (auto& v : pool) v = (uint32_t)rand() * 2654435761u;
  std::vector<double> bk((size_t)n * 2 * STAGE_CD * 2);
  for (auto& v : bk) v = (rand() % 2001 - 1000) * 1e3;
  Twiddles tw;
  const double pi = 3.14159265358979323846;
  for (int k = 0; k < 8; ++k) for (int t = 0; t < 64; ++t) tw.tw1[k][t] = cd{cos(pi * t * (1 + 4 * k) / 1024), sin(pi * t * (1 + 4 * k) / 1024)};
  for (int k = 0; k < 8; ++k) for (int a = 0; a < 8; ++a) tw.tw2[k][a] = cd{cos(2 * pi * a * k / 64), sin(2 * pi * a * k / 64)};
  for (int t = 0; t < 64; ++t) tw.g[t] = cd{cos(2 * pi * t / 512), sin(2 * pi * t / 512)};
  uint32_t *d_pool, *d_ext; cd* d_bk; Twiddles* d_tw;
  cudaMalloc(&d_pool, pool.size() * 4); cudaMalloc(&d_ext, (size_t)gates * EXT_STRIDE * 4);
  cudaMalloc(&d_bk, bk.size() * 8); cudaMalloc(&d_tw, sizeof(Twiddles));
  cudaMemcpy(d_pool, pool.data(), pool.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_bk, bk.data(), bk.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_tw, &tw, sizeof(Twiddles), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, k1c_smem(n));
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_probe<<<gates, K1C_THREADS, k1c_smem(n)>>>(d_pool, n, 1u << 29, d_bk, d_tw, d_ext);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("launch %d: %.3f ms (%s)\n", rep, ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
