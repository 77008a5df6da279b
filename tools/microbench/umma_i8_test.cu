// tcgen05.mma kind::i8 bring-up: C[128 x 256] (s32) = A[128 x K] (s8, K-major) * B[256 x K]^T (u8, K-major),
// K = 128, operands in the no-swizzle canonical shared-memory layout, accumulator in tensor memory.
// Checks descriptor encodings and layouts against a CPU product before the key-switch kernel uses them.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8_test umma_i8_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 256, K = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: 8 rows x 16 bytes core matrices; [k / 16][row / 8][row % 8][k % 16]
__host__ __device__ inline int canon(int rows, int r, int k) { return (k / 16) * (rows * 16) + (r / 8) * 128 + (r % 8) * 16 + (k % 16); }

__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100)
  return d;                // layout_type 0 = no swizzle, base_offset 0
}

__global__ void __launch_bounds__(128, 1) k(const int8_t* A, const uint8_t* B, int32_t* C, int swap_lbo_sbo) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* sa = smem;              // 128 x 128 bytes
  unsigned char* sb = smem + M * K;      // 256 x 128 bytes
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < M * K; e += 128) sa[canon(M, e / K, e % K)] = (unsigned char)A[e];
  for (int e = tid; e < N * K; e += 128) sb[canon(N, e / K, e % K)] = B[e];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core reads
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    // instruction descriptor: c = s32 (2) at [4,6), a_format signed (1) at [7,10), b_format unsigned (0) at [10,13),
    // K-major both, n_dim = N >> 3 at [17,23), m_dim = M >> 4 at [24,29)
    const uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint32_t a_addr = smem_u32(sa) + ks * 2 * (M * 16), b_addr = smem_u32(sb) + ks * 2 * (N * 16);
      const uint64_t da = swap_lbo_sbo ? make_desc(a_addr, 128, M * 16) : make_desc(a_addr, M * 16, 128);
      const uint64_t db = swap_lbo_sbo ? make_desc(b_addr, 128, N * 16) : make_desc(b_addr, N * 16, 128);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.u32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  // everyone waits for the MMAs
  asm volatile(
      "{\n.reg .pred P1;\nWAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra DONE;\nbra WAIT;\nDONE:\n}\n" ::"r"(
          smem_u32(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w reads lanes 32w .. 32w+31 (rows), 256 columns in chunks of 32
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0)
        : "memory");
    for (int j = 0; j < 32; ++j) C[(size_t)tid * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

int main() {
  std::vector<int8_t> A(M * K);
  std::vector<uint8_t> B(N * K);
  srand(1);
  for (auto& a : A) a = (int8_t)(rand() % 4 - 2);
  for (auto& b : B) b = (uint8_t)(rand() & 255);
  std::vector<int32_t> want(M * N, 0), got(M * N);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t s = 0;
      for (int k2 = 0; k2 < K; ++k2) s += (int32_t)A[i * K + k2] * (int32_t)B[j * K + k2];
      want[i * N + j] = s;
    }
  int8_t* dA;
  uint8_t* dB;
  int32_t* dC;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dC, got.size() * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (M + N) * K);
  for (int swap = 0; swap < 2; ++swap) {
    cudaMemset(dC, 0xff, got.size() * 4);
    k<<<1, 128, (M + N) * K>>>(dA, dB, dC, swap);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(got.data(), dC, got.size() * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int i = 0; i < M * N; ++i) bad += got[i] != want[i];
    printf("swap_lbo_sbo=%d: %s, mismatches %ld of %d; C[0][0..3] got %d %d %d %d want %d %d %d %d\n", swap,
           cudaGetErrorString(e), bad, M * N, got[0], got[1], got[2], got[3], want[0], want[1], want[2], want[3]);
  }
  return 0;
}
