// One-way time of K1e's peer exchange in isolation: a cluster of two CTAs bounces 4 KB back and forth with st.async
// (16 bytes per message, completing on the receiver's mbarrier), THREADS threads sending 4096 / THREADS bytes each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_pingpong dsmem_pingpong.cu && ./dsmem_pingpong
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void wait_phase(uint32_t bar, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(bar),
               "r"(parity)
               : "memory");
}
template <int THREADS, int BYTES, bool BULK>
__global__ void __cluster_dims__(2, 1, 1) k_pingpong(long long* out, int rounds) {
  __shared__ __align__(128) uint32_t buf[2][BYTES / 4];
  __shared__ __align__(128) uint32_t stage[BYTES / 4];
  __shared__ __align__(8) uint64_t bar[2];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int t = threadIdx.x;
  const uint32_t bars = smem_u32(bar), peer_bars = mapa(bars, rank ^ 1), peer_buf = mapa(smem_u32(buf), rank ^ 1);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bars), "r"(BYTES) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bars + 8), "r"(BYTES) : "memory");
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  constexpr int PER = BYTES / THREADS / 16;  // 16-byte messages per thread
  const long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const uint32_t b = r & 1, parity = (r >> 1) & 1;
    if ((r & 1) == (int)rank ? false : true) {}  // (both CTAs run the same loop; the turn alternates below)
    if (((r + rank) & 1) == 0 && BULK) {  // my turn to send: stage locally, one bulk copy into the peer
#pragma unroll
      for (int q = 0; q < PER; ++q) reinterpret_cast<uint4*>(stage)[t * PER + q] = make_uint4(r, t, q, r + t);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (t == 0)
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         peer_buf + b * BYTES),
                     "r"(smem_u32(stage)), "r"(BYTES), "r"(peer_bars + 8 * b)
                     : "memory");
    } else if (((r + rank) & 1) == 0) {  // my turn to send
#pragma unroll
      for (int q = 0; q < PER; ++q)
        asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                         peer_buf + (b * (BYTES / 4) + (t * PER + q) * 4) * 4),
                     "r"(r), "r"(t), "r"(q), "r"(r + t), "r"(peer_bars + 8 * b)
                     : "memory");
    } else {  // my turn to receive
      wait_phase(bars + 8 * b, parity);
      uint32_t acc = 0;
#pragma unroll
      for (int q = 0; q < PER; ++q) acc += buf[b][(t * PER + q) * 4];
      if (acc == 0xdeadbeef) out[1] = acc;
      __syncthreads();
      if (t == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bars + 8 * b), "r"(BYTES) : "memory");
    }
  }
  const long long t1 = clock64();
  if (t == 0 && rank == 0) out[0] = t1 - t0;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <int THREADS, int BYTES, bool BULK = false>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 16);
  const int rounds = 2000;
  k_pingpong<THREADS, BYTES, BULK><<<2, THREADS>>>(d, rounds);
  k_pingpong<THREADS, BYTES, BULK><<<2, THREADS>>>(d, rounds);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %6.0f cycles one way (%s)\n", name, (double)h / rounds, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() {
  run<64, 4096>("4 KB from 64 threads (K1e)");
  run<128, 4096>("4 KB from 128 threads");
  run<256, 4096>("4 KB from 256 threads");
  run<64, 2048>("2 KB from 64 threads");
  run<64, 1024>("1 KB from 64 threads");
  run<32, 512>("512 B from 32 threads");
  run<64, 4096, true>("4 KB staged + one bulk copy");
  run<64, 2048, true>("2 KB staged + one bulk copy");
  return 0;
}
