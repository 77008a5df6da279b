// Latency of one tensor-memory load (tcgen05.ld 32x32b.x16 + tcgen05.wait::ld) and of a store + wait::st,
// one warp alone and with all 12 warps of a K1d-sized CTA issuing concurrently.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_latency tmem_latency.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__global__ void __launch_bounds__(384, 1) k(long long* out, int active_warps, int iters) {
  __shared__ uint32_t base;
  const int wid = threadIdx.x / 32;
  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&base)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t addr = base + (((uint32_t)wid & 3u) * 32u << 16) + (wid >> 2) * 160u;
  uint32_t r[16];
  for (int j = 0; j < 16; ++j) r[j] = threadIdx.x + j;
  long long ld = 0, st = 0;
  if (wid < active_warps) {
    for (int it = 0; it < iters; ++it) {
      long long t0 = clock64();
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n\ttcgen05.wait::st.sync.aligned;"
                   ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
                   "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
      long long t1 = clock64();
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\ttcgen05.wait::ld.sync.aligned;"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
                     "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(addr) : "memory");
      long long t2 = clock64();
      st += t1 - t0;
      ld += t2 - t1;
      for (int j = 0; j < 16; ++j) r[j] += 1;
    }
  }
  if (threadIdx.x % 32 == 0 && wid < active_warps) { out[2 * wid] = st / iters; out[2 * wid + 1] = ld / iters; }
  if (threadIdx.x == 0) out[30] = r[3];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}
int main() {
  long long* d; cudaMalloc(&d, 32 * 8);
  for (int aw : {1, 4, 12}) {
    cudaMemset(d, 0, 32 * 8);
    k<<<1, 384>>>(d, aw, 1000);
    long long h[32]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%2d warps active: warp 0 st+wait %lld cycles, ld+wait %lld cycles; last warp st %lld ld %lld (%s)\n", aw, h[0], h[1], h[2 * (aw - 1)], h[2 * (aw - 1) + 1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
