// Throughput of the on-SM data paths that could take load off the shared-memory pipe of K1:
//   tensor-memory loads / stores (tcgen05.ld / .st, 32x32b: per-thread private columns),
//   warp shuffles alone and mixed with 128-bit shared-memory loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_shfl_bw tmem_shfl_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// MODE 0: tcgen05.ld x32, 1: tcgen05.st x32, 2: shfl only, 3: lds.128 only, 4: shfl + lds 1:1 (by wavefronts 1:4),
// 5: ld x32 + lds.128 mixed, 6: tcgen05.ld x64
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(uint32_t* out, int iters) {
  extern __shared__ __align__(16) unsigned char smraw[];
  double2* sm = reinterpret_cast<double2*>(smraw);
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 4096; i += blockDim.x) sm[i] = make_double2(i, 1.0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t taddr = tmem_base + (((warp & 3u) * 32u) << 16) + (warp >> 2) * 128u;
  uint32_t r[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) r[j] = t * 64 + j;
  uint32_t acc = 0;
  double2 dacc = make_double2(0, 0);
  // initialise TMEM so loads read defined data
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::
            "r"(taddr + 32 * q),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 5) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr + 32 * ((q + it) & 3))
            : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc ^= v[j];
        if (MODE == 5) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const double2 d = sm[(t + 256 * j + it + q) & 4095];
            dacc.x += d.x;
            dacc.y += d.y;
          }
        }
      }
    } else if (MODE == 1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::
                "r"(taddr + 32 * q),
            "r"(r[0] + it), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
            "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
            "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
            "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
            : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else if (MODE == 6) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint32_t v[64];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
            "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
              "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]),
              "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]),
              "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]),
              "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
            : "r"(taddr + 64 * ((q + it) & 1))
            : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 64; ++j) acc ^= v[j];
      }
    } else if (MODE == 2 || MODE == 4) {
#pragma unroll
      for (int j = 0; j < 32; ++j) r[j] = __shfl_xor_sync(0xffffffffu, r[j] + it, 16);
      if (MODE == 4) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double2 d = sm[(t + 256 * j + it) & 4095];
          dacc.x += d.x;
          dacc.y += d.y;
        }
      }
    } else if (MODE == 3) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double2 d = sm[(t + 256 * j + it) & 4095];
        dacc.x += d.x;
        dacc.y += d.y;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 64; ++j) acc ^= r[j];
  out[blockIdx.x * blockDim.x + t] = acc ^ (uint32_t)(dacc.x + dacc.y);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
}

template <int MODE>
void run(const char* name, double bytes_per_thread_iter, const char* what) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  cudaMalloc(&out, 4 * sms * 256);
  const int iters = 20000;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k<MODE><<<sms, 256, 65536>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double clks = ms * 1e-3 * clk * 1e3;
  printf("%-22s %8.3f ms  %8.1f clk/iter  %7.1f B/clk/SM (%s)  %s\n", name, ms, clks / iters,
         bytes_per_thread_iter * 256 * iters / clks, what, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(out);
}
int main() {
  run<0>("tmem ld x32", 4 * 32 * 4, "tmem read");
  run<6>("tmem ld x64", 2 * 64 * 4, "tmem read");
  run<1>("tmem st x32", 4 * 32 * 4, "tmem write");
  run<2>("shfl", 32 * 4, "shuffled");
  run<3>("lds.128", 8 * 16, "smem read");
  run<4>("shfl + lds.128", 32 * 4 + 8 * 16, "shuffled + smem");
  run<5>("tmem ld + lds.128", 4 * 32 * 4 + 4 * 8 * 16, "tmem + smem");
  return 0;
}
