// K2t: the N -> n key switch on the 5th-generation tensor cores.
//
// out[g][col] = (col == n ? b_g : 0) - sum_r d[g][r] * KSK[r][col]  (mod 2^32),  r = i*8 + j < 8192
// is a GEMM with an 8192-long contraction: [gates x 8192] signed base-4 digits (s8) times the key
// split into its four byte planes (u8), accumulated exactly in s32 (|sum| <= 8192 * 2 * 255 < 2^23) and
// recombined as sum_p C_p << 8p mod 2^32 -- the same integers K2 (k_key_switch, IMAD pipe) produces,
// bit for bit.  One CTA computes a 128-gate x 64-column tile:
//   warps 0-3  build the A tile (digits of 16 ring coefficients per K block, through a 256-entry
//              byte -> 4 digits table) straight into the UMMA canonical shared-memory layout, and
//              run the epilogue (tcgen05.ld, recombine the planes, subtract, store);
//   warp 4     one thread streams the B tiles (pre-arranged in global memory as shared-memory
//              images, k_ksk_mma_layout) with cp.async.bulk;
//   warp 5     one thread issues tcgen05.mma.kind::i8 (M = 128, N = 256 = 64 columns x 4 planes,
//              K = 32 per instruction), accumulator in tensor memory, tcgen05.commit frees the stage.
// Descriptors: K-major, no swizzle, core matrices of 8 rows x 16 bytes laid out [k/16][row/8][row%8][k%16]
// (leading byte offset = rows * 16 between k-chunks, stride byte offset = 128 between row groups);
// encodings checked against a CPU product in tools/microbench/umma_i8_test.cu.
#pragma once

namespace k2t {

constexpr int M = 128;             // gates per CTA
constexpr int COLS = 64;           // output columns per CTA
constexpr int NT = COLS * 4;       // UMMA N: columns x byte planes
constexpr int KB = 128;            // K bytes per stage = 16 ring coefficients x 8 digits
constexpr int STAGES = 4;
constexpr int A_BYTES = M * KB, B_BYTES = NT * KB, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int K_TOTAL = RING_N * KS_T;
constexpr int KBLOCKS = K_TOTAL / KB;
constexpr int NTILES = ROW_STRIDE / COLS;
constexpr int THREADS = 192;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;  // + digit table

__host__ __device__ constexpr int canon(int rows, int r, int k) {
  return (k / 16) * (rows * 16) + (r / 8) * 128 + (r % 8) * 16 + (k % 16);
}

// ksk[8192][ROW_STRIDE] (int32) -> [NTILES][KBLOCKS] shared-memory images of the B tile:
// row n' = 4 * (col % 64) + plane, byte k = r % 128, canonical K-major layout
__global__ void k_ksk_mma_layout(const int32_t* __restrict__ ksk, uint8_t* __restrict__ out) {
  const int nt = blockIdx.x / KBLOCKS, kb = blockIdx.x % KBLOCKS;
  uint8_t* dst = out + (size_t)blockIdx.x * B_BYTES;
  for (int e = threadIdx.x; e < B_BYTES; e += blockDim.x) {
    const int k16 = e / (NT * 16), rem = e % (NT * 16);
    const int np = (rem / 128) * 8 + (rem % 128) / 16, kk = k16 * 16 + rem % 16;
    const int col = nt * COLS + np / 4, plane = np % 4;
    const uint32_t v = (uint32_t)ksk[(size_t)(kb * KB + kk) * ROW_STRIDE + col];
    dst[e] = (uint8_t)(v >> (8 * plane));
  }
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo_bytes >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo_bytes >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);  // version 1, no swizzle
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "K2T_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra K2T_DONE;\n"
      "bra K2T_WAIT;\n"
      "K2T_DONE:\n"
      "}\n" ::"r"(a), "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(THREADS, 1) k_key_switch_mma(const uint32_t* __restrict__ ext,
                                                               const uint8_t* __restrict__ ksk_mma,
                                                               uint32_t* __restrict__ pool,
                                                               const int32_t* __restrict__ out_rows, int stride, int n,
                                                               int64_t k) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint32_t* lut = reinterpret_cast<uint32_t*>(smem + STAGES * STAGE_BYTES);  // byte of 4 fields -> 4 signed digits
  __shared__ uint64_t full_a[STAGES], full_b[STAGES], empty[STAGES], acc_full;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt = blockIdx.x % NTILES;
  const int64_t g0 = (int64_t)(blockIdx.x / NTILES) * M;

  for (int y = tid; y < 256; y += THREADS) {
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // digit j of the byte sits in bits 7-2j .. 6-2j; k order = j
      const int d = ((y >> (6 - 2 * j)) & 3) - 2;
      w |= (uint32_t)(uint8_t)(int8_t)d << (8 * j);
    }
    lut[y] = w;
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_a[s], 4 * 32);
      mbar_init(&full_b[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(NT)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp < 4) {
    // ---- A tile: row = this thread's gate, 16 ring coefficients per K block -----------------------
    const int r = tid;
    const bool live = g0 + r < k;
    const uint32_t* src = ext + (live ? g0 + r : 0) * EXT_STRIDE;
    const uint32_t bias = ks_bias();
    const uint32_t row_off = (uint32_t)((r / 8) * 128 + (r % 8) * 16);
    uint4 w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = __ldg(reinterpret_cast<const uint4*>(src) + q);
    for (int kb = 0; kb < KBLOCKS; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) mbar_wait_parity(&empty[s], (uint32_t)(kb / STAGES - 1) & 1u);
      unsigned char* a_stage = smem + s * STAGE_BYTES;
      uint4 cur[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) cur[q] = w[q];
      if (kb + 1 < KBLOCKS) {
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = __ldg(reinterpret_cast<const uint4*>(src + (kb + 1) * 16) + q);
      }
      const uint32_t* cw = reinterpret_cast<const uint32_t*>(cur);
#pragma unroll
      for (int c2 = 0; c2 < 8; ++c2) {  // two coefficients = 16 K bytes = one core-matrix row
        const uint32_t a0 = cw[2 * c2] + bias, a1 = cw[2 * c2 + 1] + bias;
        uint4 v = make_uint4(lut[a0 >> 24], lut[(a0 >> 16) & 255u], lut[a1 >> 24], lut[(a1 >> 16) & 255u]);
        if (!live) v = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(a_stage + c2 * (M * 16) + row_off) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
      mbar_arrive(&full_a[s]);
    }
  } else if (warp == 4) {
    if (lane == 0) {
      const uint8_t* src = ksk_mma + (size_t)nt * KBLOCKS * B_BYTES;
      for (int kb = 0; kb < KBLOCKS; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait_parity(&empty[s], (uint32_t)(kb / STAGES - 1) & 1u);
        mbar_expect_tx(&full_b[s], B_BYTES);
        bulk_load(smem + s * STAGE_BYTES + A_BYTES, src + (size_t)kb * B_BYTES, B_BYTES, &full_b[s]);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      // c = s32, a = signed 8 bit, b = unsigned 8 bit, both K-major, N >> 3, M >> 4
      const uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
      for (int kb = 0; kb < KBLOCKS; ++kb) {
        const int s = kb % STAGES;
        const uint32_t parity = (uint32_t)(kb / STAGES) & 1u;
        mbar_wait_parity(&full_a[s], parity);
        mbar_wait_parity(&full_b[s], parity);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a_addr = smem_u32(smem + s * STAGE_BYTES), b_addr = a_addr + A_BYTES;
#pragma unroll
        for (int ks = 0; ks < KB / 32; ++ks) {
          const uint64_t da = smem_desc(a_addr + ks * 2 * (M * 16), M * 16, 128);
          const uint64_t db = smem_desc(b_addr + ks * 2 * (NT * 16), NT * 16, 128);
          const uint32_t acc = (kb > 0 || ks > 0) ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.u32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc)
              : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&empty[s]))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&acc_full))
                   : "memory");
    }
  }

  if (warp < 4) {
    // ---- epilogue: lane (= gate) of tensor memory, 256 columns = 64 output columns x 4 byte planes ---
    mbar_wait_parity(&acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int64_t g = g0 + tid;
    const bool live = g < k;
    uint32_t* row = pool + (live ? (int64_t)out_rows[g] : 0) * stride;
    const uint32_t body = live ? ext[g * EXT_STRIDE + RING_N] : 0u;
#pragma unroll 1
    for (int c0 = 0; c0 < NT; c0 += 32) {
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
      if (live) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int col = nt * COLS + c0 / 4 + c;
          const uint32_t sum = v[4 * c] + (v[4 * c + 1] << 8) + (v[4 * c + 2] << 16) + (v[4 * c + 3] << 24);
          if (col <= n) row[col] = (col == n ? body : 0u) - sum;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(NT) : "memory");
}

}  // namespace k2t
