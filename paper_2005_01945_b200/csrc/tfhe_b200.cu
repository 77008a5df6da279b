// libtfhe_b200.so -- sm_100a kernels and the C ABI declared in include/tfhe_b200.h.
//
// Kernels
//   K1 fused gate linear form + mod switch + blind rotation + sample extract.  The bootstrapping key is
//      UNROLLED over pairs of LWE mask elements (three TRGSW samples per pair, ceil(n/2) steps of four forward
//      and two inverse FP64 negacyclic transforms); ACC resident in shared memory:
//      K1d k_gate_bootstrap_warp  one gate per WARP, up to twelve per SM, spectral key staged by TMA through a
//                                 release-count ring, accumulators parked in tensor memory (tfhe_warp.cuh);
//                                 k_gate_bootstrap_warp_mid: the same code for up to eight warps per CTA (255
//                                 registers), what a mid-size launch spread over all SMs runs
//      K1e k_gate_bootstrap_pair  one gate per two-CTA cluster, one accumulator polynomial per SM, DSMEM
//                                 exchange (latency path; tfhe_pair.cuh + tfhe_cluster.cuh)
//   K2 k_key_switch       batched N -> n key switch as an integer rank-8192 update,
//                         32 ciphertexts x 512 columns per CTA, digits in smem (launches of 49 .. 64 gates)
//   K2n k_key_switch_narrow  the same for launches below 96 gates (dependent circuit levels): a batch of key loads
//                         in flight, partial sums by atomics into a self-cleaning scratch, last CTA writes the rows
//   K2t k_key_switch_mma  the same update as an exact s8 x u8 -> s32 GEMM on the tensor cores
//                         (tcgen05.mma kind::i8, TMEM accumulator), tfhe_keyswitch_mma.cuh
//   K3 k_bk_transform(_w) one-time: raw TRGSW rows -> spectral key in K1e's / K1d's chunk order;
//      k_ksk_layout       raw key-switching key -> row-padded table
//   k_partition_trivial, k_trivial_extract   regrouping of a launch: gates on two trivial inputs behind the real ones
//   k_rows_negate, k_rows_phase, k_rows_encrypt   NOT, batched phase (decryption helper), batched encryption
//   k_peak_*              DFMA / IMAD peak microbenchmarks (roofline denominators)
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <string>
#include <vector>

#include "../../include/tfhe_b200.h"
#include "tfhe_device.cuh"
#include "tfhe_warp.cuh"
#include "tfhe_cluster.cuh"

using namespace tfb;

static_assert(TFB_ROW_STRIDE == ROW_STRIDE, "header / device stride mismatch");
static_assert(TFB_EXT_STRIDE == EXT_STRIDE, "header / device stride mismatch");

// ------------------------------------------------------------------------------------
// context
// ------------------------------------------------------------------------------------
constexpr int64_t HOST_CHUNK = 21312;  // gates per pipeline chunk of tfb_gate_launch_host: 12 full waves of K1d CTAs (148 SMs x 12 gates)
constexpr int HOST_EVENTS = 8;         // event slots; a slot is reused 8 chunks later (long after it fired)

struct tfb_ctx {
  int device = 0;
  tfb_params p{};
  bool keys_loaded = false;
  cd* d_bkf = nullptr;         // K1e's chunks [pair][p][lvl][half][k4][key][c][t] (cd), prescaled by 1/512
  cd* d_bkw = nullptr;         // K1d's chunks [pair][stage][qc][q4][key][c][lane] (cd), prescaled by 1/512
  WarpTwiddles* d_wtw = nullptr;
  FactorTables* d_ft = nullptr;
  int32_t* d_ksk = nullptr;    // [N*t][ROW_STRIDE]
  uint8_t* d_ksk_mma = nullptr;  // K2t: byte planes as shared-memory images [col tile][K block][32 KB]
  int force_ks = 0;            // 0 auto, 1 = K2 (IMAD), 2 = K2t (tensor cores)
  Twiddles* d_tw = nullptr;
  uint32_t* d_ext = nullptr;   // scratch [cap][EXT_STRIDE]
  uint32_t* d_ksn = nullptr;   // K2n partial sums + counters (KSN_SCRATCH_WORDS, zero between launches)
  int64_t ext_cap = 0;
  int32_t* d_perm = nullptr;   // regrouped launch: [3][cap] x / y / out rows, then [cap] kinds (bytes), then 2 counters
  int no_regroup = 0;          // 1: launches keep the caller's gate order (profiling)
  // buffers of the host-buffer launch path
  uint32_t* d_hx = nullptr;    // [cap][ROW_STRIDE] x, y, out back to back
  uint8_t* d_hkinds = nullptr;
  int32_t* d_hrows = nullptr;  // identity row indices
  int64_t host_cap = 0;
  cudaStream_t s_in = nullptr, s_run = nullptr, s_out = nullptr;  // host-buffer launch pipeline
  cudaEvent_t ev_in[HOST_EVENTS] = {}, ev_run[HOST_EVENTS] = {};
  int64_t launches = 0;
  int sm_count = 148;
  int force_kernel = 0;        // 0 auto, 4 = K1d (warp), 5 = K1e (cluster pair)
  int force_warps = 0;         // 0 auto, else gates per CTA of K1d (profiling)
  int force_wide_regs = 0;     // 1: never use the 255-register build of K1d (profiling)
  std::string err;
};

static thread_local std::string g_create_err;

#define TFB_CUDA(ctx, call)                                                            \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      (ctx)->err = std::string(#call) + ": " + cudaGetErrorString(e_);                 \
      return TFB_ERR_CUDA;                                                             \
    }                                                                                  \
  } while (0)

// Every entry point runs on the context's device and leaves the caller's current device as it
// found it (a process may drive several engines / GPUs).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err;
  explicit DeviceGuard(int device) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != device)
      err = cudaSetDevice(device);
    else
      prev = -1;  // nothing to restore
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
#define TFB_ENTER(ctx)                     \
  DeviceGuard guard_((ctx)->device);       \
  TFB_CUDA(ctx, guard_.err)

struct BlockSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// ---- mbarrier / bulk-copy (TMA) primitives --------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_LOOP:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra WAIT_LOOP;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing on an mbarrier (SASS: UBLKCP)
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// ------------------------------------------------------------------------------------
// K1d: fused gate bootstrap, ONE ciphertext per WARP, K1D_WARPS ciphertexts per CTA (one CTA
//      per SM), arithmetic in tfhe_warp.cuh.  Radix-16 transforms: one shared-memory exchange
//      and one shuffle stage per transform, no barrier other than __syncwarp inside the blind
//      rotation; the spectral key comes through a TMA ring of 12 KB chunks shared by all warps.
// ------------------------------------------------------------------------------------
#ifndef TFB_K1D_TMEM
#define TFB_K1D_TMEM 1  // accumulators parked in tensor memory between the MAC stages
#endif
#ifndef TFB_K1D_WARPS
#define TFB_K1D_WARPS 12  // 3 warps per scheduler: 168 registers each, accumulators parked in tensor memory
#endif
constexpr int K1D_WARPS = TFB_K1D_WARPS;
#ifndef TFB_K1D_WAVE_TABLE  // ms per wave of K1d with 1 .. 12 gates per CTA (tools/k1_ab.py, TFB_K1D_W)
#define TFB_K1D_WAVE_TABLE 3.25, 3.13, 3.20, 3.26, 4.74, 5.10, 5.15, 4.69, 6.64, 6.70, 6.82, 6.66
#endif
constexpr int K1D_THREADS = K1D_WARPS * WARP_T;
__host__ __device__ constexpr int warp_smem(int n, bool split = true) {
  return wbuf_bytes(split) + 2 * RING_N * (int)sizeof(uint32_t) + ((n + 2) * 2 + 15) / 16 * 16;
}

// Key ring of K1d: WR_SLOTS chunks of 12 KB (pair, stage, four spectral points per lane x three keys x two
// output components: what the MAC of one accumulator chunk consumes; sixteen chunks per pair step).
// Consumers wait on the full mbarrier of a slot; a slot is handed back by counting releases,
// and the warp whose release is the last one issues the bulk copy of the chunk that reuses
// the slot (no dedicated producer: with a fixed producer thread every warp of the CTA is
// gated by that thread's own progress).  A warp may run WR_SLOTS - 1 chunks ahead of the
// slowest one before it has to wait.
#ifndef TFB_K1D_SLOTS
#define TFB_K1D_SLOTS 5
#endif
constexpr int WR_SLOTS = TFB_K1D_SLOTS;
constexpr int WR_CHUNK_BYTES = WCHUNK_CD * (int)sizeof(cd);
// dynamic smem: twiddles | factor tables | key ring | barriers | warps
constexpr int K1D_OFF_FT = (int)sizeof(WarpTwiddles);
constexpr int K1D_OFF_RING = K1D_OFF_FT + (int)sizeof(FactorTables);
constexpr int K1D_OFF_BARS = K1D_OFF_RING + WR_SLOTS * WR_CHUNK_BYTES;
constexpr int K1D_HEADER = K1D_OFF_BARS + 128;
// Waiting for a key chunk: non-blocking mbarrier.test_wait + nanosleep (TFB_K1D_POLL, default), or
// mbarrier.try_wait with a suspend-time hint.  On real runs a warp waits 2-5 % of the time and polls
// once or twice per chunk (build with -DTFB_K1D_PROBE to print it); under ncu's instrumentation the
// loop spins far more, which inflates the instruction counts of a profile.
#ifndef TFB_K1D_POLL
#define TFB_K1D_POLL 1  // measured: 68.5 ms (poll) vs 70.8 ms (try_wait) per 14208 gates
#endif
__device__ __forceinline__ bool mbar_test_u32(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
#if TFB_K1D_POLL
  while (!mbar_test_u32(bar, parity)) __nanosleep(100);
#else
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_LOOP:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE;\n"
      "bra WAIT_LOOP;\n"
      "DONE:\n"
      "}\n" ::"r"(bar), "r"(parity), "r"(1000000u)  // suspend-time hint: wait in hardware
      : "memory");
#endif
}
struct WarpRing {
  const cd* bkw;        // full spectral key in global memory
  cd* ring;             // WR_SLOTS chunks in shared memory
  uint64_t* full;       // [slots] completes when a chunk's bytes have landed
  uint32_t* released;   // [slots] warps that are done with the chunk in the slot
  uint32_t full_u32;    // shared-space address of full[0]
  int chunk;            // next chunk this warp will consume (16 m + 4 s + qc: the key is stored in that order)
  int n_chunks;
  uint32_t consumers;   // warps of this CTA (a mid-size launch runs fewer than K1D_WARPS per SM)

  static __device__ __forceinline__ int slot(int s) { return s % WR_SLOTS; }
  static __device__ __forceinline__ uint32_t parity(int s) { return (uint32_t)(s / WR_SLOTS) & 1u; }
  __device__ __forceinline__ void issue(int s) {
    mbar_expect_tx(&full[slot(s)], WR_CHUNK_BYTES);
    bulk_load(ring + (size_t)slot(s) * WCHUNK_CD, bkw + (size_t)s * WCHUNK_CD, WR_CHUNK_BYTES, &full[slot(s)]);
  }
#ifdef TFB_K1D_PROBE
  long long waited = 0, polls = 0;
#endif
  __device__ __forceinline__ const cd* acquire_chunk(int, int, int) {
#ifdef TFB_K1D_PROBE
    const long long t0 = clock64();
    while (!mbar_test_u32(full_u32 + 8u * (uint32_t)slot(chunk), parity(chunk))) {
      __nanosleep(100);
      ++polls;
    }
    waited += clock64() - t0;
#else
    mbar_wait_u32(full_u32 + 8u * (uint32_t)slot(chunk), parity(chunk));
#endif
    return ring + (size_t)slot(chunk) * WCHUNK_CD;
  }
  __device__ __forceinline__ cd load(const cd* q) const { return *q; }
  __device__ __forceinline__ void release() {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      const int sl = slot(chunk);
      // acq_rel: the counter chains every warp's (generic-proxy) reads of the slot before the last
      // arriver, whose proxy fence then orders them before the async-proxy refill (PTX memory model:
      // a write-after-read across proxies needs both)
      uint32_t before;
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                   : "=r"(before)
                   : "r"(smem_u32(&released[sl]))
                   : "memory");
      if (before == consumers - 1u) {  // last one out refills the slot
        released[sl] = 0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (chunk + WR_SLOTS < n_chunks) issue(chunk + WR_SLOTS);
      }
    }
    ++chunk;
  }
};

// Turn protocol (TFB_K1D_TURNS): the three warps that share a scheduler take the MAC stage of a CMux in
// a fixed rotation, handing the turn on with named barriers (bar.arrive by the warp that leaves, bar.sync
// by the next: a hardware wait, no issue slots).  Left alone, the round-robin scheduler convoys the
// warps: all three want the FP64 pipe in the same cycles (math-pipe-throttle / not-selected stalls) and
// then sit in their shared-memory phases together.  One fixed hand-over per stage pins them a third of a
// stage apart -- one in its MAC (key loads, tensor-memory traffic), two in transforms: 68.3 -> 64.4 ms
// per 14,208 gates.  What was measured and lost (turns around the FP64 bursts, around both, a
// first-come-first-served lock instead of the rotation) is in profiles/README.md.
#ifndef TFB_K1D_TURNS
#define TFB_K1D_TURNS 0
#endif
template <bool SPLIT>
struct DevWarp {
  static constexpr bool kSplitExchange = SPLIT;  // two rounds through a half-size buffer (twelve warps per CTA) or one
  int turn_wait = 0, turn_next = 0;  // named-barrier ids (0: no protocol, e.g. the key-setup kernel)
#ifdef TFB_K1D_PHASES
  mutable long long T[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, last = 0;
  __device__ __forceinline__ void tick(int k) const {
    const long long now = clock64();
    T[k] += now - last;
    last = now;
  }
#endif
  __device__ __forceinline__ void turn_enter() const {
    if (TFB_K1D_TURNS && turn_wait) asm volatile("bar.sync %0, 64;" ::"r"(turn_wait) : "memory");
  }
  __device__ __forceinline__ void turn_leave() const {
    if (TFB_K1D_TURNS && turn_next) asm volatile("bar.arrive %0, 64;" ::"r"(turn_next) : "memory");
  }
  __device__ __forceinline__ void turn_pass() const {  // take the turn and hand it on at once
    turn_enter();
    turn_leave();
  }
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
  __device__ __forceinline__ cd xchg16(cd v) const {
    return cd{__shfl_xor_sync(0xffffffffu, v.re, 16), __shfl_xor_sync(0xffffffffu, v.im, 16)};
  }
};

// Tensor-memory park of K1d: with the 32x32b shape lane i of warp w owns TMEM lane
// 32*(w%4)+i and any columns, i.e. private per-lane storage with its own data path (measured:
// 338 B/clk/SM loads, 895 B/clk/SM stores, concurrent with the shared-memory pipe;
// tools/microbench/tmem_shfl_bw.cu).  A warp's slice is 128 columns: polynomial c at
// columns 64c .. 64c+63, a chunk of PARK_CH complex values is 16 columns.
// 16 tensor-memory columns in flight: the registers are valid only after settle (tcgen05.wait::ld);
// tying them to the wait as in/out operands keeps every use of them behind it.
struct TmemChunk {
  uint32_t r[16];
};
__device__ __forceinline__ void tmem_issue16(uint32_t addr, TmemChunk& ch) {
  uint32_t* r = ch.r;
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr)
      : "memory");
}
__device__ __forceinline__ void tmem_settle16(TmemChunk& ch) {
  uint32_t* r = ch.r;
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])::"memory");
}

struct TmemWPark {
  typedef TmemChunk Chunk;
  uint32_t taddr;  // (lane << 16) | first column of this warp's slice
  __device__ __forceinline__ void issue_one(int c, int qb, Chunk& ch) const { tmem_issue16(taddr + 64 * c + 4 * qb, ch); }
  __device__ __forceinline__ void settle_one(Chunk& ch, cd* o) const {
    tmem_settle16(ch);
    unpack(ch.r, o);
  }
  static __device__ __forceinline__ void unpack(const uint32_t* r, cd* o) {
#pragma unroll
    for (int j = 0; j < PARK_CH; ++j)
      o[j] = cd{__hiloint2double((int)r[4 * j + 1], (int)r[4 * j]), __hiloint2double((int)r[4 * j + 3], (int)r[4 * j + 2])};
  }
  static __device__ __forceinline__ void pack(const cd* o, uint32_t* r) {
#pragma unroll
    for (int j = 0; j < PARK_CH; ++j) {
      r[4 * j + 0] = (uint32_t)__double2loint(o[j].re);
      r[4 * j + 1] = (uint32_t)__double2hiint(o[j].re);
      r[4 * j + 2] = (uint32_t)__double2loint(o[j].im);
      r[4 * j + 3] = (uint32_t)__double2hiint(o[j].im);
    }
  }
  __device__ __forceinline__ void store_one(int c, int qb, const cd* o) const {
    uint32_t r[16];
    pack(o, r);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr + 64 * c + 4 * qb),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
  }
  __device__ __forceinline__ void store(int qb, const cd* o0, const cd* o1) const {
    store_one(0, qb, o0);
    store_one(1, qb, o1);
  }
  __device__ __forceinline__ void flush() const { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
};
constexpr uint32_t K1D_TMEM_SLICE = 128;  // columns per warp: 2 x 64 accumulators
constexpr uint32_t K1D_TMEM_TW = ((K1D_WARPS + 3) / 4) * K1D_TMEM_SLICE;  // first column of the twiddle table
constexpr uint32_t K1D_TMEM_NEED = K1D_TMEM_TW + 68;                      // 16 twiddles + c per lane

// Per-lane twiddle table in tensor memory (shared by the warps of a lane quarter): 16 pass-1
// twiddles at columns 4k .. 4k+3, the radix-2 twiddle at columns 64 .. 67.
struct TmemTw {
  typedef TmemChunk Chunk;
  uint32_t taddr;  // (lane << 16) | first column of the table
  __device__ __forceinline__ void issue4(int kb, Chunk& ch) const { tmem_issue16(taddr + 4 * kb, ch); }
  __device__ __forceinline__ void settle4(Chunk& ch, cd* w) const {
    tmem_settle16(ch);
    TmemWPark::unpack(ch.r, w);
  }
  __device__ __forceinline__ void issue_c(Chunk& ch) const {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(ch.r[0]), "=r"(ch.r[1]), "=r"(ch.r[2]), "=r"(ch.r[3])
                 : "r"(taddr + 64)
                 : "memory");
  }
  __device__ __forceinline__ cd settle_c(Chunk& ch) const {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(ch.r[0]), "+r"(ch.r[1]), "+r"(ch.r[2]), "+r"(ch.r[3])::"memory");
    return cd{__hiloint2double((int)ch.r[1], (int)ch.r[0]), __hiloint2double((int)ch.r[3], (int)ch.r[2])};
  }
  // one warp per lane quarter writes the table
  __device__ __forceinline__ void fill(const LaneTwiddles& lt) const {
#pragma unroll
    for (int kb = 0; kb < WPTS; kb += 4) {
      uint32_t r[16];
      TmemWPark::pack(lt.w + kb, r);
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
          "%15, %16};" ::"r"(taddr + 4 * kb),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
          : "memory");
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr + 64),
                 "r"((uint32_t)__double2loint(lt.c.re)), "r"((uint32_t)__double2hiint(lt.c.re)),
                 "r"((uint32_t)__double2loint(lt.c.im)), "r"((uint32_t)__double2hiint(lt.c.im))
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
};

template <bool SPLIT>
__device__ __forceinline__ void k1d_body(
    const uint32_t* __restrict__ pool, const uint8_t* __restrict__ kinds,
    const int32_t* __restrict__ x_rows, const int32_t* __restrict__ y_rows, int stride, int n, uint32_t mu,
    const cd* __restrict__ bkw, const WarpTwiddles* __restrict__ tw_global, const FactorTables* __restrict__ ft_global,
    uint32_t* __restrict__ ext, int64_t k) {
  extern __shared__ __align__(128) unsigned char smem[];
  WarpTwiddles* tw = reinterpret_cast<WarpTwiddles*>(smem);
  FactorTables* ft = reinterpret_cast<FactorTables*>(smem + K1D_OFF_FT);
  cd* ring = reinterpret_cast<cd*>(smem + K1D_OFF_RING);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + K1D_OFF_BARS);
  const int wid = threadIdx.x / WARP_T, t = threadIdx.x % WARP_T;
  unsigned char* mine = smem + K1D_HEADER + (size_t)wid * warp_smem(n, SPLIT);
  void* buf = mine;
  uint32_t* acc = reinterpret_cast<uint32_t*>(mine + wbuf_bytes(SPLIT));
  uint16_t* abar = reinterpret_cast<uint16_t*>(acc + 2 * RING_N);

  // warps of this CTA: K1D_WARPS in a throughput launch, fewer when a mid-size launch is spread over all SMs
  const int nwarps = (int)blockDim.x / WARP_T;
  for (int i = threadIdx.x; i < (int)(sizeof(WarpTwiddles) / sizeof(cd)); i += (int)blockDim.x)
    reinterpret_cast<cd*>(tw)[i] = reinterpret_cast<const cd*>(tw_global)[i];
  for (int i = threadIdx.x; i < (int)(sizeof(FactorTables) / sizeof(cd)); i += (int)blockDim.x)
    reinterpret_cast<cd*>(ft)[i] = reinterpret_cast<const cd*>(ft_global)[i];
  static_assert(WR_SLOTS <= 8, "eight mbarriers + eight release counters fit the 128-byte barrier block");
  WarpRing bk{bkw, ring, bars, reinterpret_cast<uint32_t*>(bars + WR_SLOTS), smem_u32(bars), 0,
              WCHUNKS_PER_PAIR * ((n + 1) / 2), (uint32_t)nwarps};
  if (threadIdx.x == 0) {
    for (int j = 0; j < WR_SLOTS; ++j) {
      mbar_init(&bk.full[j], 1);
      bk.released[j] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  // tensor memory: one slice per warp, warps w, w+4, w+8 share a lane quarter
  constexpr uint32_t kTmemCols = K1D_TMEM_NEED <= 128 ? 128 : (K1D_TMEM_NEED <= 256 ? 256 : 512);
  static_assert(K1D_TMEM_NEED <= 512, "tensor memory has 512 columns");
  static_assert(PARK_CH == 4, "the tensor-memory helpers move 16 columns = 4 complex values at a time");
  __shared__ uint32_t tmem_base;
  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0)
    for (int j = 0; j < WR_SLOTS; ++j) bk.issue(j);
  const TmemTw ttw{tmem_base + ((((uint32_t)wid & 3u) * 32u) << 16) + K1D_TMEM_TW};
  if (wid < 4) {  // one warp per lane quarter builds the twiddle table
    LaneTwiddles lt;
    build_lane_twiddles(tw, t, &lt);
    ttw.fill(lt);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // tail CTA: surplus warps redo the last ciphertext (keeps the ring protocol uniform) but do not store
  const int64_t want = (int64_t)blockIdx.x * nwarps + wid;
  const int64_t g = want < k ? want : k - 1;
  const uint32_t* xr = pool + (int64_t)x_rows[g] * stride;
  const uint32_t* yr = pool + (int64_t)y_rows[g] * stride;
  uint32_t* dst = want < k ? ext + g * EXT_STRIDE : nullptr;  // null: no extract
  DevWarp<SPLIT> w;
#if TFB_K1D_TURNS
  {
    // rotation over the warps {s, s + 4, s + 8} of scheduler s = wid % 4 (grouping {3 s, 3 s + 1, 3 s + 2} measured
    // 8 % slower: warp w runs on scheduler w % 4): position r = wid / 4 waits on the barrier its predecessor
    // arrives on; the last position pre-arrives once so that position 0 starts
    static_assert(K1D_WARPS == 12, "the turn rotation is laid out for three warps per scheduler");
    const int sch = wid & 3, pos = wid >> 2;
    w.turn_wait = 1 + 3 * sch + (pos + 2) % 3;
    w.turn_next = 1 + 3 * sch + pos;
    if (pos == 2) w.turn_leave();
  }
#endif
#if TFB_K1D_TMEM
  TmemWPark park{tmem_base + ((((uint32_t)wid & 3u) * 32u) << 16) + ((uint32_t)wid >> 2) * K1D_TMEM_SLICE};
#else
  RegPark park;
#endif
#ifdef TFB_K1D_PROBE
  const long long probe_t0 = clock64();
#endif
#ifdef TFB_K1D_PHASES
  w.last = clock64();
#endif
  gate_bootstrap_warp(xr, yr, (int)kinds[g], n, mu, bk, ttw, ft, acc, abar, buf, dst, t, w, park);
#ifdef TFB_K1D_PHASES
  if (t == 0 && blockIdx.x == 3 && (wid == 0 || wid == 5 || wid == 10))
    printf("warp %2d per pair step: decomp/digits %lld | fwd burst1 %lld exch %lld burst2 %lld (x4) | key wait %lld turn wait %lld mac %lld (x4) | "
           "inv: tmem %lld burst1 %lld exch %lld burst2 %lld update %lld (x2)\n",
           wid, w.T[0] / ((n + 1) / 2), w.T[1] / ((n + 1) / 2), w.T[2] / ((n + 1) / 2), w.T[3] / ((n + 1) / 2), w.T[4] / ((n + 1) / 2),
           w.T[5] / ((n + 1) / 2), w.T[6] / ((n + 1) / 2), w.T[7] / ((n + 1) / 2), w.T[8] / ((n + 1) / 2), w.T[9] / ((n + 1) / 2),
           w.T[10] / ((n + 1) / 2), w.T[11] / ((n + 1) / 2));
#endif
#ifdef TFB_K1D_PROBE
  if (t == 0 && (blockIdx.x == 0 || blockIdx.x == 77))
    printf("cta %d warp %2d: %lld cycles, %lld waiting for the key (%.1f%%), %lld polls\n", (int)blockIdx.x, wid,
           clock64() - probe_t0, bk.waited, 100.0 * bk.waited / (double)(clock64() - probe_t0), bk.polls);
#endif
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (wid == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols) : "memory");
}

#define TFB_K1D_ARGS                                                                                                  \
  const uint32_t *__restrict__ pool, const uint8_t *__restrict__ kinds, const int32_t *__restrict__ x_rows,           \
      const int32_t *__restrict__ y_rows, int stride, int n, uint32_t mu, const cd *__restrict__ bkw,                 \
      const WarpTwiddles *__restrict__ tw_global, const FactorTables *__restrict__ ft_global, uint32_t *__restrict__ ext, \
      int64_t k, const uint32_t *__restrict__ active, int64_t gate0
// the throughput build: up to twelve warps per CTA, 168 registers per thread
// `active` (may be null): a regrouped launch keeps its gates with two trivial inputs behind the first *active ones
// (k_partition_trivial); their extracted samples are written by k_trivial_extract, and a CTA that holds only such
// gates has nothing to do.
#define TFB_K1D_SKIP_IDLE_CTA \
  if (active && gate0 + (int64_t)blockIdx.x * (int64_t)(blockDim.x / WARP_T) >= (int64_t)*active) return;
__global__ void __launch_bounds__(K1D_THREADS, 1) k_gate_bootstrap_warp(TFB_K1D_ARGS) {
  TFB_K1D_SKIP_IDLE_CTA
  k1d_body<true>(pool, kinds, x_rows, y_rows, stride, n, mu, bkw, tw_global, ft_global, ext, k);
}
// the same code for the mid-size launches that run at most eight warps per CTA: 255 registers per thread
constexpr int K1D_WARPS_MID = 8;
#ifndef TFB_K1D_MID_SPLIT
#define TFB_K1D_MID_SPLIT 0  // eight warps leave room for full-size exchange buffers: one round instead of two
#endif
constexpr bool K1D_MID_SPLIT = TFB_K1D_MID_SPLIT != 0;
__global__ void __launch_bounds__(K1D_WARPS_MID * WARP_T, 1) k_gate_bootstrap_warp_mid(TFB_K1D_ARGS) {
  TFB_K1D_SKIP_IDLE_CTA
  k1d_body<K1D_MID_SPLIT>(pool, kinds, x_rows, y_rows, stride, n, mu, bkw, tw_global, ft_global, ext, k);
}

// ------------------------------------------------------------------------------------
// K2: key switch.  out[c][col] = (col == n ? ext_b[c] : 0) - sum_r digit[c][r] * ksk[r][col]
//     r = i*KS_T + j over the N*KS_T digit rows; CTA tile = KS_CT ciphertexts x 512 columns.
// ------------------------------------------------------------------------------------
constexpr int KS_CT = 32;        // ciphertexts per CTA
constexpr int KS_THREADS = 256;  // 2 columns per thread
constexpr int KS_CHUNK_I = 16;   // ring coefficients per digit chunk
constexpr int KS_CHUNK_R = KS_CHUNK_I * KS_T;

__global__ void __launch_bounds__(KS_THREADS) k_key_switch(const uint32_t* __restrict__ ext,
                                                           const int32_t* __restrict__ ksk,
                                                           uint32_t* __restrict__ pool,
                                                           const int32_t* __restrict__ out_rows, int stride,
                                                           int n, int64_t k, int i_per_cta) {
  // gridDim.y > 1: the ring coefficients are split over blockIdx.y and the partial sums are
  // combined with integer atomics into rows zeroed by k_rows_zero (small launches: latency).
  __shared__ __align__(16) int32_t digits[KS_CHUNK_R][KS_CT];
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * KS_CT;
  int32_t acc0[KS_CT], acc1[KS_CT];
#pragma unroll
  for (int c = 0; c < KS_CT; ++c) acc0[c] = acc1[c] = 0;
  const uint32_t bias = ks_bias();

  const int i_begin = blockIdx.y * i_per_cta, i_end = i_begin + i_per_cta;
  for (int i0 = i_begin; i0 < i_end; i0 += KS_CHUNK_I) {
    __syncthreads();
    // digits of ext[c][i0 .. i0+16) for the tile's ciphertexts: 512 words, 2 per thread
    for (int e = tid; e < KS_CT * KS_CHUNK_I; e += KS_THREADS) {
      const int c = e / KS_CHUNK_I, ii = e % KS_CHUNK_I;
      uint32_t a = 0;
      if (c0 + c < k) a = ext[(c0 + c) * EXT_STRIDE + i0 + ii];
      const uint32_t ab = a + bias;
      const bool live = (c0 + c < k);
#pragma unroll
      for (int j = 0; j < KS_T; ++j) digits[ii * KS_T + j][c] = live ? ks_digit(ab, j) : 0;
    }
    __syncthreads();
    const int32_t* kr = ksk + (int64_t)i0 * KS_T * ROW_STRIDE;
#pragma unroll 4
    for (int r = 0; r < KS_CHUNK_R; ++r) {
      const int32_t k0 = __ldg(kr + (int64_t)r * ROW_STRIDE + tid);
      const int32_t k1 = __ldg(kr + (int64_t)r * ROW_STRIDE + tid + KS_THREADS);
      const int4* d4 = reinterpret_cast<const int4*>(&digits[r][0]);
#pragma unroll
      for (int q = 0; q < KS_CT / 4; ++q) {
        const int4 d = d4[q];
        acc0[4 * q + 0] += d.x * k0;
        acc1[4 * q + 0] += d.x * k1;
        acc0[4 * q + 1] += d.y * k0;
        acc1[4 * q + 1] += d.y * k1;
        acc0[4 * q + 2] += d.z * k0;
        acc1[4 * q + 2] += d.z * k1;
        acc0[4 * q + 3] += d.w * k0;
        acc1[4 * q + 3] += d.w * k1;
      }
    }
  }
  const bool split = gridDim.y > 1;
#pragma unroll
  for (int c = 0; c < KS_CT; ++c) {
    if (c0 + c >= k) break;
    uint32_t* row = pool + (int64_t)out_rows[c0 + c] * stride;  // only columns 0..n are written: rows may be packed
    const uint32_t body = (blockIdx.y == 0) ? ext[(c0 + c) * EXT_STRIDE + RING_N] : 0u;
    const uint32_t v0 = (tid == n ? body : 0u) - (uint32_t)acc0[c];
    const uint32_t v1 = (tid + KS_THREADS == n ? body : 0u) - (uint32_t)acc1[c];
    if (split) {
      if (tid <= n) atomicAdd(row + tid, v0);
      if (tid + KS_THREADS <= n) atomicAdd(row + tid + KS_THREADS, v1);
    } else {
      if (tid <= n) row[tid] = v0;
      if (tid + KS_THREADS <= n) row[tid + KS_THREADS] = v1;
    }
  }
}

// K2n: key switch of a NARROW launch (the dependent levels of adders and multiplier trees: a handful of gates).
// There the IMAD work is nothing and the time is latency: one CTA per (group of KSN_G gates, KSN_ROWS digit rows
// = 4 ring coefficients), every key load of the thread issued before the first use, partial sums combined with
// integer atomics into a scratch row per gate that is zero between launches: the CTA that arrives last on the
// group's counter reads the sums back, writes  (0, b) - sum  into the pool rows and clears scratch and counter
// again (no separate zeroing kernel, nothing to order against the inputs).
constexpr int KSN_G = 8;                     // gates per CTA
constexpr int KSN_I = 4;                     // ring coefficients per batch of key loads
constexpr int KSN_ROWS = KSN_I * KS_T;       // 32 key rows in flight per thread and batch
constexpr int KSN_MAX_GATES = 96;            // launches below this many gates take K2n
constexpr int KSN_SMALL_GATES = 16;          // up to here one batch per CTA (256 CTAs per group of 8 gates: shortest latency);
constexpr int KSN_BATCHES_WIDE = 4;          // beyond, four batches per CTA (64 CTAs per group: a quarter of the atomics)
constexpr int KSN_SCRATCH_WORDS = KSN_MAX_GATES * ROW_STRIDE + 64;  // sums, then one counter per gate group
template <int BATCHES>
__global__ void __launch_bounds__(KS_THREADS) k_key_switch_narrow(const uint32_t* __restrict__ ext,
                                                                  const int32_t* __restrict__ ksk,
                                                                  uint32_t* __restrict__ pool,
                                                                  const int32_t* __restrict__ out_rows, int stride, int n,
                                                                  int k, uint32_t* __restrict__ scratch) {
  __shared__ int32_t digits[BATCHES][KSN_ROWS][KSN_G];
  __shared__ uint32_t arrived;
  const int tid = threadIdx.x, i0 = blockIdx.x * KSN_I * BATCHES, g0 = blockIdx.y * KSN_G;
  const int live = min(KSN_G, k - g0);
  int32_t acc0[KSN_G], acc1[KSN_G];
#pragma unroll
  for (int c = 0; c < KSN_G; ++c) acc0[c] = acc1[c] = 0;
#pragma unroll 1
  for (int bt = 0; bt < BATCHES; ++bt) {
    // all key words of the batch first: 32 rows x 2 columns in flight per thread ...
    int32_t kw0[KSN_ROWS], kw1[KSN_ROWS];
    const int32_t* kr = ksk + (int64_t)(i0 + bt * KSN_I) * KS_T * ROW_STRIDE;
#pragma unroll
    for (int r = 0; r < KSN_ROWS; ++r) {
      kw0[r] = __ldg(kr + r * ROW_STRIDE + tid);
      kw1[r] = __ldg(kr + r * ROW_STRIDE + tid + KS_THREADS);
    }
    // ... then the batch's digits (its own shared-memory block: no barrier between batches)
    if (tid < KSN_I * KSN_G) {
      const int c = tid / KSN_I, ii = tid % KSN_I;
      const uint32_t ab = (c < live ? ext[(int64_t)(g0 + c) * EXT_STRIDE + i0 + bt * KSN_I + ii] : 0u) + ks_bias();
#pragma unroll
      for (int j = 0; j < KS_T; ++j) digits[bt][ii * KS_T + j][c] = c < live ? ks_digit(ab, j) : 0;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < KSN_ROWS; ++r) {
#pragma unroll
      for (int c = 0; c < KSN_G; ++c) {
        const int32_t d = digits[bt][r][c];
        acc0[c] += d * kw0[r];
        acc1[c] += d * kw1[r];
      }
    }
  }
  uint32_t* sums = scratch + (int64_t)g0 * ROW_STRIDE;
#pragma unroll
  for (int c = 0; c < KSN_G; ++c) {
    if (c >= live) break;
    if (tid <= n) atomicAdd(sums + c * ROW_STRIDE + tid, (uint32_t)acc0[c]);
    if (tid + KS_THREADS <= n) atomicAdd(sums + c * ROW_STRIDE + tid + KS_THREADS, (uint32_t)acc1[c]);
  }
  __threadfence();
  __syncthreads();
  uint32_t* counter = scratch + KSN_MAX_GATES * ROW_STRIDE + blockIdx.y;
  if (tid == 0) arrived = atomicAdd(counter, 1u);
  __syncthreads();
  if (arrived != gridDim.x - 1) return;
  __threadfence();  // last CTA of the group: every other CTA's sums are visible (they sit in L2; read them there)
  for (int c = 0; c < live; ++c) {
    uint32_t* row = pool + (int64_t)out_rows[g0 + c] * stride;
    const uint32_t body = ext[(int64_t)(g0 + c) * EXT_STRIDE + RING_N];
    for (int col = tid; col <= n; col += KS_THREADS) {
      row[col] = (col == n ? body : 0u) - __ldcg(sums + c * ROW_STRIDE + col);
      sums[c * ROW_STRIDE + col] = 0u;
    }
  }
  if (tid == 0) *counter = 0u;
}

// Regrouping of a launch: gates whose two inputs are trivial (zero masks: the zero padding of multiplier trees,
// constants) have nothing to rotate -- their accumulator stays the rotated test vector -- but inside a K1d CTA they
// hold warps that run at the pace of the busy ones.  k_partition_trivial moves them behind the real gates (one warp
// per gate reads the two masks; a CTA claims its output ranges with two atomics; the order inside a group is
// arbitrary: gates of a launch are independent and every gate carries its own rows), k_trivial_extract writes their
// extracted samples, and K1 CTAs that hold only such gates return at once (`active`).
constexpr int PART_GATES_PER_CTA = 32;
__global__ void __launch_bounds__(256) k_partition_trivial(const uint32_t* __restrict__ pool, int stride, int n,
                                                          const uint8_t* __restrict__ kinds, const int32_t* __restrict__ xr,
                                                          const int32_t* __restrict__ yr, const int32_t* __restrict__ orow,
                                                          int64_t k, int32_t* __restrict__ perm, uint32_t* __restrict__ counters) {
  __shared__ uint8_t idle[PART_GATES_PER_CTA];
  __shared__ int32_t slot[PART_GATES_PER_CTA];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t g0 = (int64_t)blockIdx.x * PART_GATES_PER_CTA;
  for (int j = warp; j < PART_GATES_PER_CTA; j += 8) {
    const int64_t g = g0 + j;
    uint32_t any = 0;
    if (g < k) {
      const uint32_t* x = pool + (int64_t)xr[g] * stride;
      const uint32_t* y = pool + (int64_t)yr[g] * stride;
      for (int i = lane; i < n; i += 32) any |= x[i] | y[i];
    }
    any = __reduce_or_sync(0xffffffffu, any);
    if (lane == 0) idle[j] = (g < k && any == 0) ? 1 : 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int live = (int)min((int64_t)PART_GATES_PER_CTA, k - g0);
    int n_idle = 0;
    for (int j = 0; j < live; ++j) n_idle += idle[j];
    const uint32_t front = atomicAdd(&counters[0], (uint32_t)(live - n_idle));  // real gates fill from the front ...
    const uint32_t back = atomicAdd(&counters[1], (uint32_t)n_idle);             // ... trivial-input gates from the back
    uint32_t f = front, b = back;
    for (int j = 0; j < live; ++j) slot[j] = idle[j] ? (int32_t)(k - 1 - b++) : (int32_t)f++;
  }
  __syncthreads();
  if (threadIdx.x < PART_GATES_PER_CTA && g0 + threadIdx.x < k) {
    const int64_t g = g0 + threadIdx.x, s = slot[threadIdx.x];
    perm[s] = xr[g];
    perm[k + s] = yr[g];
    perm[2 * k + s] = orow[g];
    reinterpret_cast<uint8_t*>(perm + 3 * k)[s] = kinds[g];
  }
}
// extracted sample of a gate on two trivial inputs: mask 0, body = coefficient 0 of the rotated test vector
__global__ void __launch_bounds__(256) k_trivial_extract(const uint32_t* __restrict__ pool, int stride, int n, uint32_t mu,
                                                        const uint8_t* __restrict__ kinds, const int32_t* __restrict__ xr,
                                                        const int32_t* __restrict__ yr, uint32_t* __restrict__ ext, int64_t k,
                                                        const uint32_t* __restrict__ active) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t g = (int64_t)*active + (int64_t)blockIdx.x * 8 + warp;  // one warp per gate behind the real ones
  if (g >= k) return;
  uint32_t* row = ext + g * EXT_STRIDE;
  for (int j = lane; j < RING_N; j += 32) row[j] = 0u;
  if (lane == 0) {
    const int bbar = gate_body_rotation_of(pool + (int64_t)xr[g] * stride, pool + (int64_t)yr[g] * stride, (int)kinds[g], n, mu);
    row[RING_N] = test_vector_coeff(0, bbar, mu);
  }
}

__global__ void k_rows_zero(uint32_t* __restrict__ pool, const int32_t* __restrict__ rows, int stride, int n) {
  uint32_t* dst = pool + (int64_t)rows[blockIdx.x] * stride;
  for (int c = threadIdx.x; c <= n; c += blockDim.x) dst[c] = 0u;
}

#include "tfhe_keyswitch_mma.cuh"

// ------------------------------------------------------------------------------------
// K3: key setup
// ------------------------------------------------------------------------------------
// raw polynomial index of bk_raw[pair][key][row][c][N] -> (pair m, key j, row r = p*l + lvl, component c)
struct RawPoly {
  int m, j, r, c;
  __device__ explicit RawPoly(int64_t poly)
      : m((int)((poly >> 1) / BK_ROWS / BK_KEYS)), j((int)((poly >> 1) / BK_ROWS % BK_KEYS)), r((int)((poly >> 1) % BK_ROWS)),
        c((int)(poly & 1)) {}
};
// one CTA per raw polynomial -> K1e's chunks bkf[pair][p][lvl][half][k4][key][c][t]
__global__ void __launch_bounds__(FFT_THREADS) k_bk_transform(const int32_t* __restrict__ bk_raw,
                                                              cd* __restrict__ bkf,
                                                              const Twiddles* __restrict__ tw) {
  __shared__ cd bufA[HALF_N];
  __shared__ cd bufB[HALF_N];
  const int t = threadIdx.x;
  const RawPoly id(blockIdx.x);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(bk_raw) + (int64_t)blockIdx.x * RING_N;
  cd x[8];
#pragma unroll
  for (int m = 0; m < 8; ++m)
    x[m] = cd{int32_to_double(src[t + 64 * m]), int32_to_double(src[t + 64 * m + HALF_N])};
  BlockSync sync;
  fft_forward(x, t, TableTw{tw, t}, bufA, bufB, sync);
  const double scale = 1.0 / HALF_N;
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2)
    bkf[pchunk_offset(id.m, id.r / BK_L, id.r % BK_L, k2 >> 2) + pchunk_index(k2 & 3, id.j, id.c, t)] =
        cd{x[k2].re * scale, x[k2].im * scale};
}

// same for K1d: one warp per raw polynomial -> bkw[pair][stage][qc][q4][key][c][lane]
__global__ void __launch_bounds__(WARP_T) k_bk_transform_w(const int32_t* __restrict__ bk_raw,
                                                           cd* __restrict__ bkw,
                                                           const WarpTwiddles* __restrict__ tw) {
  __shared__ __align__(16) unsigned char buf[WBUF_BYTES];
  const int t = threadIdx.x;
  const RawPoly id(blockIdx.x);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(bk_raw) + (int64_t)blockIdx.x * RING_N;
  cd x[WPTS];
#pragma unroll
  for (int m = 0; m < WPTS; ++m)
    x[m] = cd{int32_to_double(src[t + 32 * m]), int32_to_double(src[t + 32 * m + HALF_N])};
  DevWarp<WX_SPLIT> w;
  LaneTwiddles lt;
  build_lane_twiddles(tw, t, &lt);
  wfft_forward(x, t, MemTw{&lt}, buf, w);
  const double scale = 1.0 / HALF_N;
#pragma unroll
  for (int q = 0; q < WPTS; ++q)
    bkw[wchunk_offset(id.m, id.r, q / WCHUNK_Q) + wchunk_index(q % WCHUNK_Q, id.j, id.c, t)] =
        cd{x[q].re * scale, x[q].im * scale};
}

// ksk_raw[N*t][n+1] -> ksk[N*t][ROW_STRIDE], zero padded
__global__ void k_ksk_layout(const int32_t* __restrict__ raw, int32_t* __restrict__ out, int n) {
  const int64_t r = blockIdx.x;
  for (int c = threadIdx.x; c < ROW_STRIDE; c += blockDim.x)
    out[r * ROW_STRIDE + c] = (c <= n) ? raw[r * (n + 1) + c] : 0;
}

// ------------------------------------------------------------------------------------
// small row kernels
// ------------------------------------------------------------------------------------
__global__ void k_rows_negate(uint32_t* __restrict__ pool, const int32_t* __restrict__ in_rows,
                              const int32_t* __restrict__ out_rows) {
  const uint32_t* src = pool + (int64_t)in_rows[blockIdx.x] * ROW_STRIDE;
  uint32_t* dst = pool + (int64_t)out_rows[blockIdx.x] * ROW_STRIDE;
  for (int c = threadIdx.x; c < ROW_STRIDE; c += blockDim.x) dst[c] = 0u - src[c];
}

__global__ void k_rows_phase(const uint32_t* __restrict__ pool, const int32_t* __restrict__ rows,
                             const uint32_t* __restrict__ key_bits, uint32_t* __restrict__ phase, int n) {
  const uint32_t* row = pool + (int64_t)rows[blockIdx.x] * ROW_STRIDE;
  uint32_t s = 0;
  for (int c = threadIdx.x; c < n; c += blockDim.x) s += row[c] * key_bits[c];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  __shared__ uint32_t part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += part[w];
    phase[blockIdx.x] = row[n] - tot;
  }
}

// ---- batched fresh encryption (client side, encirc/torus.py:254-271) --------------------------------
// Philox4x32-10 (Salmon et al., SC'11): counter-based, so sample i / word j is a pure function of
// (seed, i, j) whatever the launch geometry.
struct Philox {
  uint32_t k0, k1;
  __device__ __forceinline__ uint4 operator()(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) const {
    uint32_t a = k0, b = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint32_t h0 = __umulhi(0xD2511F53u, c0), l0 = 0xD2511F53u * c0;
      const uint32_t h1 = __umulhi(0xCD9E8D57u, c2), l1 = 0xCD9E8D57u * c2;
      c0 = h1 ^ c1 ^ a;
      c1 = l1;
      c2 = h0 ^ c3 ^ b;
      c3 = l0;
      a += 0x9E3779B9u;
      b += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
  }
};

// one CTA per sample: threads draw the mask four words at a time, reduce <a, s>, thread 0 draws the noise
__global__ void __launch_bounds__(128) k_rows_encrypt(uint32_t* __restrict__ pool,
                                                      const int32_t* __restrict__ out_rows,
                                                      const uint8_t* __restrict__ bits,
                                                      const uint32_t* __restrict__ key_bits, int n, uint32_t mu,
                                                      double alpha, uint64_t seed, uint64_t first_sample) {
  const uint64_t sample = first_sample + blockIdx.x;
  const Philox rng{(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t* row = pool + (int64_t)out_rows[blockIdx.x] * ROW_STRIDE;
  uint32_t dot = 0;
  for (int q = threadIdx.x; 4 * q < n; q += blockDim.x) {
    const uint4 w = rng((uint32_t)sample, (uint32_t)(sample >> 32), (uint32_t)q, 0u);
    const uint32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (4 * q + e < n) {
        row[4 * q + e] = v[e];
        dot += v[e] * key_bits[4 * q + e];
      }
  }
  for (int c = n + 1 + threadIdx.x; c < ROW_STRIDE; c += blockDim.x) row[c] = 0u;
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_down_sync(0xffffffffu, dot, o);
  __shared__ uint32_t part[4];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint4 w = rng((uint32_t)sample, (uint32_t)(sample >> 32), 0u, 1u);  // stream 1: the noise
    // Box-Muller on two 53-bit-grade uniforms in (0, 1]
    const double u1 = ((double)w.x * 4294967296.0 + (double)w.y + 1.0) * (1.0 / 18446744073709551616.0);
    const double u2 = ((double)w.z * 4294967296.0 + (double)w.w) * (1.0 / 18446744073709551616.0);
    double e = rint(sqrt(-2.0 * log(u1)) * cospi(2.0 * u2) * alpha * 4294967296.0);
    const uint32_t clamp_word = mu / 4 > 1 ? mu / 4 : 1;  // fresh_clamp_word (encirc/torus.py:177-184): 2^27 at mu = 1/8
    const double clamp = (double)(clamp_word - 1);
    e = fmin(fmax(e, -clamp), clamp);
    const uint32_t msg = bits[blockIdx.x] ? mu : (0u - mu);
    row[n] = part[0] + part[1] + part[2] + part[3] + msg + (uint32_t)(int32_t)e;
  }
}

// packed host layout [k][n+1] <-> pool rows, used by the host-buffer launch
__global__ void k_identity_rows(int32_t* rows, int64_t count, int32_t base) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) rows[i] = base + (int32_t)i;
}

// ------------------------------------------------------------------------------------
// peak microbenchmarks
// ------------------------------------------------------------------------------------
__global__ void k_peak_dfma(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  const double m = 1.0000001, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_peak_imad(int32_t* out, int iters) {
  int32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
          a7 = a0 + 7;
  const int32_t m = (int32_t)blockIdx.x | 3, c = 12345;
  for (int i = 0; i < iters; ++i) {
    a0 = a0 * m + c; a1 = a1 * m + c; a2 = a2 * m + c; a3 = a3 * m + c;
    a4 = a4 * m + c; a5 = a5 * m + c; a6 = a6 * m + c; a7 = a7 * m + c;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// ------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------
static void fill_twiddles(Twiddles* tw) {
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int k = 0; k < 8; ++k)
    for (int t = 0; t < FFT_THREADS; ++t) {
      const long double ang = pi * (long double)(t * (1 + 4 * k)) / (long double)RING_N;
      tw->tw1[k][t] = cd{(double)cosl(ang), (double)sinl(ang)};
    }
  for (int k = 0; k < 8; ++k)
    for (int a = 0; a < 8; ++a) {
      const long double ang = 2.0L * pi * (long double)(a * k) / 64.0L;
      tw->tw2[k][a] = cd{(double)cosl(ang), (double)sinl(ang)};
    }
  for (int t = 0; t < FFT_THREADS; ++t) {
    const long double ang = 2.0L * pi * (long double)t / (long double)HALF_N;
    tw->g[t] = cd{(double)cosl(ang), (double)sinl(ang)};
  }
}

static void fill_warp_twiddles(WarpTwiddles* tw) { tfb::fill_warp_twiddles<long double>(tw, cosl, sinl); }

static int ensure_ext(tfb_ctx* ctx, int64_t k) {
  if (k <= ctx->ext_cap) return TFB_OK;
  if (ctx->d_ext) TFB_CUDA(ctx, cudaFree(ctx->d_ext));
  ctx->d_ext = nullptr;
  ctx->ext_cap = 0;
  int64_t cap = 1024;
  while (cap < k) cap *= 2;
  TFB_CUDA(ctx, cudaMalloc(&ctx->d_ext, (size_t)cap * EXT_STRIDE * sizeof(uint32_t)));
  if (ctx->d_perm) TFB_CUDA(ctx, cudaFree(ctx->d_perm));
  ctx->d_perm = nullptr;
  TFB_CUDA(ctx, cudaMalloc(&ctx->d_perm, (size_t)cap * 13 + 64));  // 3 x int32 + 1 byte per gate, two counters
  ctx->ext_cap = cap;
  return TFB_OK;
}

extern "C" {

int tfb_abi_version(void) { return TFB_ABI_VERSION; }

const char* tfb_last_error(const tfb_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int tfb_ctx_create(int device, const tfb_params* p, tfb_ctx** out) {
  if (!p || !out) {
    g_create_err = "null argument";
    return TFB_ERR_INVALID;
  }
  if (p->ring_n != RING_N || p->bk_l != BK_L || p->bk_bgbit != BK_BGBIT || p->ks_t != KS_T ||
      p->ks_basebit != KS_BASEBIT || p->n < 1 || p->n >= ROW_STRIDE - 1) {
    g_create_err = "unsupported parameter set (compiled: N=1024 l=2 Bgbit=9 t=8 basebit=2, n<=510)";
    return TFB_ERR_INVALID;
  }
  DeviceGuard guard(device);
  cudaError_t e = guard.err;
  if (e != cudaSuccess) {
    g_create_err = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
    return TFB_ERR_CUDA;
  }
  tfb_ctx* ctx = new tfb_ctx();
  ctx->device = device;
  ctx->p = *p;
  Twiddles* h = new Twiddles();
  fill_twiddles(h);
  e = cudaMalloc(&ctx->d_tw, sizeof(Twiddles));
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_tw, h, sizeof(Twiddles), cudaMemcpyHostToDevice);
  delete h;
  if (e == cudaSuccess) {
    WarpTwiddles hw;
    fill_warp_twiddles(&hw);
    e = cudaMalloc(&ctx->d_wtw, sizeof(WarpTwiddles));
    if (e == cudaSuccess) e = cudaMemcpy(ctx->d_wtw, &hw, sizeof(WarpTwiddles), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) {
    FactorTables hf;
    fill_factor_tables<long double>(&hf, cosl, sinl);
    e = cudaMalloc(&ctx->d_ft, sizeof(FactorTables));
    if (e == cudaSuccess) e = cudaMalloc(&ctx->d_ksn, KSN_SCRATCH_WORDS * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(ctx->d_ksn, 0, KSN_SCRATCH_WORDS * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemcpy(ctx->d_ft, &hf, sizeof(FactorTables), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_gate_bootstrap_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             K1D_HEADER + K1D_WARPS * warp_smem(p->n));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_gate_bootstrap_warp_mid, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             K1D_HEADER + K1D_WARPS_MID * warp_smem(p->n, K1D_MID_SPLIT));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k1e::k_gate_bootstrap_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, k1e::smem_bytes(p->n));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k2t::k_key_switch_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, k2t::SMEM_BYTES);
  if (e == cudaSuccess) {
    int sms = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    ctx->sm_count = sms;
  }
  if (e != cudaSuccess) {
    g_create_err = std::string("context setup: ") + cudaGetErrorString(e);
    delete ctx;
    return TFB_ERR_CUDA;
  }
  if (const char* f = getenv("TFB_FORCE_KERNEL")) ctx->force_kernel = atoi(f);  // A/B switch for profiling
  if (const char* f = getenv("TFB_K1D_W")) ctx->force_warps = atoi(f);
  if (const char* f = getenv("TFB_K1D_NOMID")) ctx->force_wide_regs = atoi(f);
  if (const char* f = getenv("TFB_FORCE_KS")) ctx->force_ks = atoi(f);
  if (const char* f = getenv("TFB_NO_REGROUP")) ctx->no_regroup = atoi(f);
  *out = ctx;
  return TFB_OK;
}

void tfb_ctx_destroy(tfb_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard guard(ctx->device);
  cudaFree(ctx->d_bkf);
  cudaFree(ctx->d_bkw);
  cudaFree(ctx->d_wtw);
  cudaFree(ctx->d_ft);
  cudaFree(ctx->d_ksk);
  cudaFree(ctx->d_ksk_mma);
  cudaFree(ctx->d_tw);
  cudaFree(ctx->d_ext);
  cudaFree(ctx->d_ksn);
  cudaFree(ctx->d_perm);
  cudaFree(ctx->d_hx);
  cudaFree(ctx->d_hkinds);
  cudaFree(ctx->d_hrows);
  if (ctx->s_in) {
    cudaStreamDestroy(ctx->s_in);
    cudaStreamDestroy(ctx->s_run);
    cudaStreamDestroy(ctx->s_out);
    for (auto e : ctx->ev_in) cudaEventDestroy(e);
    for (auto e : ctx->ev_run) cudaEventDestroy(e);
  }
  delete ctx;
}

int tfb_load_keys(tfb_ctx* ctx, const int32_t* bk, const int32_t* ksk, int on_device, void* stream) {
  if (!ctx || !bk || !ksk) return TFB_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  TFB_ENTER(ctx);
  const int n = ctx->p.n;
  const int64_t bk_polys = (int64_t)((n + 1) / 2) * BK_KEYS * BK_ROWS * 2;  // pairs x keys x rows x components
  const size_t bk_words = (size_t)bk_polys * RING_N;
  const size_t ksk_words = (size_t)RING_N * KS_T * (n + 1);
  const int32_t* d_bk = bk;
  const int32_t* d_kr = ksk;
  int32_t *tmp_bk = nullptr, *tmp_ksk = nullptr;
  if (!on_device) {
    TFB_CUDA(ctx, cudaMalloc(&tmp_bk, bk_words * 4));
    TFB_CUDA(ctx, cudaMalloc(&tmp_ksk, ksk_words * 4));
    TFB_CUDA(ctx, cudaMemcpyAsync(tmp_bk, bk, bk_words * 4, cudaMemcpyHostToDevice, st));
    TFB_CUDA(ctx, cudaMemcpyAsync(tmp_ksk, ksk, ksk_words * 4, cudaMemcpyHostToDevice, st));
    d_bk = tmp_bk;
    d_kr = tmp_ksk;
  }
  if (!ctx->d_bkf) TFB_CUDA(ctx, cudaMalloc(&ctx->d_bkf, (size_t)bk_polys * HALF_N * sizeof(cd)));
  if (!ctx->d_ksk) TFB_CUDA(ctx, cudaMalloc(&ctx->d_ksk, (size_t)RING_N * KS_T * ROW_STRIDE * 4));
  if (!ctx->d_bkw) TFB_CUDA(ctx, cudaMalloc(&ctx->d_bkw, (size_t)bk_polys * HALF_N * sizeof(cd)));
  k_bk_transform<<<(unsigned)bk_polys, FFT_THREADS, 0, st>>>(d_bk, ctx->d_bkf, ctx->d_tw);
  k_bk_transform_w<<<(unsigned)bk_polys, WARP_T, 0, st>>>(d_bk, ctx->d_bkw, ctx->d_wtw);
  k_ksk_layout<<<RING_N * KS_T, 128, 0, st>>>(d_kr, ctx->d_ksk, n);
  if (!ctx->d_ksk_mma)
    TFB_CUDA(ctx, cudaMalloc(&ctx->d_ksk_mma, (size_t)k2t::NTILES * k2t::KBLOCKS * k2t::B_BYTES));
  k2t::k_ksk_mma_layout<<<k2t::NTILES * k2t::KBLOCKS, 256, 0, st>>>(ctx->d_ksk, ctx->d_ksk_mma);
  ctx->launches += 1;
  ctx->launches += 3;
  TFB_CUDA(ctx, cudaGetLastError());
  TFB_CUDA(ctx, cudaStreamSynchronize(st));
  if (tmp_bk) cudaFree(tmp_bk);
  if (tmp_ksk) cudaFree(tmp_ksk);
  ctx->keys_loaded = true;
  return TFB_OK;
}

// Cost model of the two K1 variants (ms per launch on a 148-SM B200 at n = 500, measured with
// tools/k1_ab.py; only the ratios matter).  Both run in waves of one CTA set per SM:
//   K1e 1 gate / 2 SMs (cluster) per wave
//   K1d w gates / SM per wave, w = 1 .. 12 warps per CTA: a launch that does not fill a 12-warp wave is spread
//       evenly over the SMs, and a CTA with fewer warps finishes sooner (each warp shares its scheduler's
//       FP64 pipe with fewer others): K1D_WAVE_MS[w]
#ifndef TFB_K1E_WAVE_MS
#define TFB_K1E_WAVE_MS 0.62
#endif
constexpr double K1E_WAVE_MS = TFB_K1E_WAVE_MS;
constexpr double K1D_WAVE_MS[K1D_WARPS + 1] = {0.0, TFB_K1D_WAVE_TABLE};
// A launch runs as up to four segments, each one kernel launch: (variant, gates per CTA, gates).
struct K1Seg {
  int which, warps;
  int64_t gates;
};
static double k1e_cost(int64_t k, int sms) { return K1E_WAVE_MS * ceil((double)k / floor(sms / 2.0)); }
// one K1d wave for k <= 12 * sms gates: the cheapest CTA width that holds them
static double k1d_wave_cost(int64_t k, int sms, int* warps) {
  int best = K1D_WARPS;
  for (int w = K1D_WARPS; w >= 1 && (int64_t)w * sms >= k; --w)
    if (K1D_WAVE_MS[w] <= K1D_WAVE_MS[best]) best = w;
  *warps = best;
  return K1D_WAVE_MS[best];
}
// cheapest single-kernel choice for k <= 12 * sms gates
static double k1_simple(int64_t k, int sms, K1Seg* seg) {
  int w = K1D_WARPS;
  const double t_d = k1d_wave_cost(k, sms, &w), t_e = k1e_cost(k, sms);
  *seg = t_e <= t_d ? K1Seg{5, 0, k} : K1Seg{4, w, k};
  return t_e <= t_d ? t_e : t_d;
}
// K1 dispatch.  K1e (one gate per two-SM cluster) wins on latency, K1d (one gate per warp) on throughput.  A launch
// is covered by waves of 12, 8 and 4 gates per SM (three, two, one warp on every scheduler: 6.66 / 4.69 / 3.26 ms for
// 1776 / 1184 / 592 gates on 148 SMs) plus one tail -- the cheapest of cluster waves or one K1d wave of narrower CTAs
// -- and the cheapest combination wins: mostly twelve-warp waves, but e.g. 4096 gates = 1776 + 2 x 1184 + a tail
// instead of 2 x 1776 + a poorly filled third wave.  Returns the number of segments (one kernel launch each).
constexpr int K1_MAX_SEGS = 6;
static int plan_k1(int64_t k, int sms, K1Seg* seg) {
  const int64_t cap12 = (int64_t)sms * K1D_WARPS, cap8 = (int64_t)sms * 8, cap4 = (int64_t)sms * 4;
  const int64_t max12 = k / cap12;
  double best = 1e300;
  int64_t best12 = 0, best8 = 0, best4 = 0;
  K1Seg best_tail{0, 0, 0};
  for (int64_t n12 = max12 > 0 ? max12 - 1 : 0; n12 <= max12; ++n12) {
    const int64_t r12 = k - n12 * cap12;
    for (int64_t n8 = 0; n8 <= 3 && n8 * cap8 <= r12; ++n8) {
      const int64_t r8 = r12 - n8 * cap8;
      for (int64_t n4 = 0; n4 <= 1 && n4 * cap4 <= r8; ++n4) {
        const int64_t r4 = r8 - n4 * cap4;
        if (r4 > cap12) continue;  // the tail is at most one wave of the widest CTAs
        K1Seg tail{0, 0, 0};
        const double c = (double)n12 * K1D_WAVE_MS[K1D_WARPS] + (double)n8 * K1D_WAVE_MS[8] + (double)n4 * K1D_WAVE_MS[4] +
                         (r4 ? k1_simple(r4, sms, &tail) : 0.0);
        if (c < best - 1e-9) {
          best = c;
          best12 = n12, best8 = n8, best4 = n4;
          best_tail = tail;
        }
      }
    }
  }
  int nseg = 0;
  auto push = [&](K1Seg sg) {
    if (!sg.gates) return;
    if (nseg && seg[nseg - 1].which == sg.which && seg[nseg - 1].warps == sg.warps)
      seg[nseg - 1].gates += sg.gates;  // same kernel, same CTA width: one launch
    else
      seg[nseg++] = sg;
  };
  const bool tail12 = best_tail.which == 4 && best_tail.warps == K1D_WARPS;  // rides in the twelve-warp launch
  push(K1Seg{4, K1D_WARPS, best12 * cap12});
  if (tail12) push(best_tail);
  push(K1Seg{4, 8, best8 * cap8});
  if (best_tail.which == 4 && best_tail.warps == 8) push(best_tail);
  push(K1Seg{4, 4, best4 * cap4});
  if (!tail12 && !(best_tail.which == 4 && best_tail.warps == 8)) push(best_tail);
  return nseg;
}

static int launch_k1_variant(tfb_ctx* ctx, int which, int warps, const void* pool, int stride, const uint8_t* kinds,
                             const int32_t* xr, const int32_t* yr, uint32_t* ext, int64_t k, cudaStream_t st,
                             const uint32_t* active = nullptr, int64_t gate0 = 0) {
  const int n = ctx->p.n;
  if (which == 5) {  // one gate per two-CTA cluster (the kernel carries __cluster_dims__(2, 1, 1))
    k1e::k_gate_bootstrap_pair<<<(unsigned)(2 * k), k1e::THREADS, k1e::smem_bytes(n), st>>>(
        (const uint32_t*)pool, kinds, xr, yr, stride, n, ctx->p.mu_word, ctx->d_bkf, ctx->d_tw, ctx->d_ft, ext);
  } else if (which == 4) {
    const int w = ctx->force_warps > 0 && ctx->force_warps <= K1D_WARPS
                      ? ctx->force_warps
                      : (warps >= 1 && warps <= K1D_WARPS ? warps : K1D_WARPS);
    const unsigned grid = (unsigned)((k + w - 1) / w);
    const bool mid = w <= K1D_WARPS_MID && !ctx->force_wide_regs;
    auto kernel = mid ? k_gate_bootstrap_warp_mid : k_gate_bootstrap_warp;
    kernel<<<grid, w * WARP_T, K1D_HEADER + w * warp_smem(n, mid ? K1D_MID_SPLIT : true), st>>>(
        (const uint32_t*)pool, kinds, xr, yr, stride, n, ctx->p.mu_word, ctx->d_bkw, ctx->d_wtw, ctx->d_ft, ext, k, active, gate0);
  } else {
    ctx->err = "unknown K1 variant (4 = K1d warp kernel, 5 = K1e cluster kernel)";
    return TFB_ERR_INVALID;
  }
  ctx->launches += 1;
  TFB_CUDA(ctx, cudaGetLastError());
  return TFB_OK;
}

static int launch_blind_rotate(tfb_ctx* ctx, const void* pool, int stride, const uint8_t* kinds, const int32_t* xr,
                               const int32_t* yr, uint32_t* ext, int64_t k, cudaStream_t st,
                               const uint32_t* active = nullptr) {
  if (ctx->force_kernel)
    return launch_k1_variant(ctx, ctx->force_kernel, 0, pool, stride, kinds, xr, yr, ext, k, st);
  K1Seg seg[K1_MAX_SEGS];
  const int nseg = plan_k1(k, ctx->sm_count, seg);
  int64_t at = 0;
  for (int i = 0; i < nseg; ++i) {
    int rc = launch_k1_variant(ctx, seg[i].which, seg[i].warps, pool, stride, kinds + at, xr + at, yr + at,
                               ext + at * EXT_STRIDE, seg[i].gates, st, active, at);
    if (rc) return rc;
    at += seg[i].gates;
  }
  return TFB_OK;
}

static int launch_key_switch(tfb_ctx* ctx, const uint32_t* ext, void* pool, int stride, const int32_t* out_rows,
                             int64_t k, cudaStream_t st) {
  // K2t (tensor cores) from 96 gates up: 1.6 ms instead of 16.8 ms at 2^16 gates, 0.05 ms for anything up
  // to ~2000 gates; K2n for the narrow launches of dependent circuit levels (latency); K2 (IMAD pipe, split over
  // the ring coefficients) in between (tools/k2_ab.py).  TFB_FORCE_KS: 1 = K2, 2 = K2t, 3 = K2n where it applies.
  const bool mma = ctx->force_ks ? ctx->force_ks == 2 : k >= 96;
  if (mma) {
    const unsigned grid = (unsigned)((k + k2t::M - 1) / k2t::M) * k2t::NTILES;
    k2t::k_key_switch_mma<<<grid, k2t::THREADS, k2t::SMEM_BYTES, st>>>(ext, ctx->d_ksk_mma, (uint32_t*)pool, out_rows,
                                                                     stride, ctx->p.n, k);
    ctx->launches += 1;
    TFB_CUDA(ctx, cudaGetLastError());
    return TFB_OK;
  }
  // measured (tools/k2_ab.py): K2n wins up to 48 gates and from 65 (where K2 needs a third tile) to 95; K2 in between
  if (k < KSN_MAX_GATES && (ctx->force_ks == 3 || (ctx->force_ks == 0 && (k <= 48 || k > 64)))) {
    const unsigned groups = (unsigned)((k + KSN_G - 1) / KSN_G);
    if (k <= KSN_SMALL_GATES)
      k_key_switch_narrow<1><<<dim3(RING_N / KSN_I, groups), KS_THREADS, 0, st>>>(
          ext, ctx->d_ksk, (uint32_t*)pool, out_rows, stride, ctx->p.n, (int)k, ctx->d_ksn);
    else
      k_key_switch_narrow<KSN_BATCHES_WIDE><<<dim3(RING_N / (KSN_I * KSN_BATCHES_WIDE), groups), KS_THREADS, 0, st>>>(
          ext, ctx->d_ksk, (uint32_t*)pool, out_rows, stride, ctx->p.n, (int)k, ctx->d_ksn);
    ctx->launches += 1;
    TFB_CUDA(ctx, cudaGetLastError());
    return TFB_OK;
  }
  const unsigned tiles = (unsigned)((k + KS_CT - 1) / KS_CT);
  // small launches: split the 1024 ring coefficients over up to 64 CTAs per tile to fill the chip
  unsigned split = 1;
  while (split < RING_N / KS_CHUNK_I && tiles * split < 2u * (unsigned)ctx->sm_count) split *= 2;
  if (split > 1) {
    k_rows_zero<<<(unsigned)k, 128, 0, st>>>((uint32_t*)pool, out_rows, stride, ctx->p.n);
    ctx->launches += 1;
  }
  k_key_switch<<<dim3(tiles, split), KS_THREADS, 0, st>>>(ext, ctx->d_ksk, (uint32_t*)pool, out_rows, stride, ctx->p.n, k,
                                                         RING_N / (int)split);
  ctx->launches += 1;
  TFB_CUDA(ctx, cudaGetLastError());
  return TFB_OK;
}

static int check_launch_args(tfb_ctx* ctx, int64_t k) {
  if (!ctx) return TFB_ERR_INVALID;
  if (!ctx->keys_loaded) {
    ctx->err = "keys not loaded";
    return TFB_ERR_STATE;
  }
  if (k < 1 || k > (int64_t)0x7fffffff) {
    ctx->err = "k out of range";
    return TFB_ERR_INVALID;
  }
  return TFB_OK;
}

int tfb_gate_launch(tfb_ctx* ctx, void* pool, const uint8_t* kinds, const int32_t* xr, const int32_t* yr,
                    const int32_t* out_rows, int64_t k, void* stream) {
  int rc = check_launch_args(ctx, k);
  if (rc) return rc;
  if (!pool || !kinds || !xr || !yr || !out_rows) return TFB_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  TFB_ENTER(ctx);
  if ((rc = ensure_ext(ctx, k))) return rc;
  const uint32_t* active = nullptr;
  if (k >= 4 * (int64_t)ctx->sm_count && !ctx->no_regroup && !ctx->force_kernel) {  // launches that run K1d: regroup
    int32_t* perm = ctx->d_perm;
    uint32_t* counters = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(perm) + (((size_t)k * 13 + 15) / 16) * 16);
    TFB_CUDA(ctx, cudaMemsetAsync(counters, 0, 8, st));
    k_partition_trivial<<<(unsigned)((k + PART_GATES_PER_CTA - 1) / PART_GATES_PER_CTA), 256, 0, st>>>(
        (const uint32_t*)pool, ROW_STRIDE, ctx->p.n, kinds, xr, yr, out_rows, k, perm, counters);
    kinds = reinterpret_cast<const uint8_t*>(perm + 3 * k);
    xr = perm, yr = perm + k, out_rows = perm + 2 * k;
    active = counters;
    // (grid sized for k trivial gates; CTAs past the end return at once)
    k_trivial_extract<<<(unsigned)((k + 7) / 8), 256, 0, st>>>((const uint32_t*)pool, ROW_STRIDE, ctx->p.n, ctx->p.mu_word, kinds, xr, yr,
                                                  ctx->d_ext, k, active);
    ctx->launches += 2;
    TFB_CUDA(ctx, cudaGetLastError());
  }
  if ((rc = launch_blind_rotate(ctx, pool, ROW_STRIDE, kinds, xr, yr, ctx->d_ext, k, st, active))) return rc;
  return launch_key_switch(ctx, ctx->d_ext, pool, ROW_STRIDE, out_rows, k, st);
}

int tfb_debug_blind_rotate(tfb_ctx* ctx, const void* pool, const uint8_t* kinds, const int32_t* xr,
                           const int32_t* yr, uint32_t* ext, int64_t k, void* stream) {
  int rc = check_launch_args(ctx, k);
  if (rc) return rc;
  if (!pool || !kinds || !xr || !yr || !ext) return TFB_ERR_INVALID;
  TFB_ENTER(ctx);
  return launch_blind_rotate(ctx, pool, ROW_STRIDE, kinds, xr, yr, ext, k, (cudaStream_t)stream);
}

int tfb_debug_key_switch(tfb_ctx* ctx, const uint32_t* ext, void* pool, const int32_t* out_rows, int64_t k,
                         void* stream) {
  int rc = check_launch_args(ctx, k);
  if (rc) return rc;
  if (!pool || !ext || !out_rows) return TFB_ERR_INVALID;
  TFB_ENTER(ctx);
  return launch_key_switch(ctx, ext, pool, ROW_STRIDE, out_rows, k, (cudaStream_t)stream);
}

int tfb_gate_launch_host(tfb_ctx* ctx, const uint32_t* x, const uint32_t* y, const uint8_t* kinds,
                         uint32_t* out, int64_t k) {
  int rc = check_launch_args(ctx, k);
  if (rc) return rc;
  if (!x || !y || !kinds || !out) return TFB_ERR_INVALID;
  TFB_ENTER(ctx);
  if (k > ctx->host_cap) {
    cudaFree(ctx->d_hx);
    cudaFree(ctx->d_hkinds);
    cudaFree(ctx->d_hrows);
    ctx->d_hx = nullptr;
    ctx->d_hkinds = nullptr;
    ctx->d_hrows = nullptr;
    ctx->host_cap = 0;
    int64_t cap = 256;
    while (cap < k) cap *= 2;
    TFB_CUDA(ctx, cudaMalloc(&ctx->d_hx, (size_t)3 * cap * (ctx->p.n + 1) * 4));  // packed rows, as on the host
    TFB_CUDA(ctx, cudaMalloc(&ctx->d_hkinds, (size_t)cap));
    TFB_CUDA(ctx, cudaMalloc(&ctx->d_hrows, (size_t)3 * cap * 4));
    k_identity_rows<<<(unsigned)((3 * cap + 255) / 256), 256>>>(ctx->d_hrows, 3 * cap, 0);
    ctx->launches += 1;
    TFB_CUDA(ctx, cudaGetLastError());
    TFB_CUDA(ctx, cudaStreamSynchronize(0));  // the pipeline streams below do not wait on the default stream
    ctx->host_cap = cap;
  }
  const int64_t cap = ctx->host_cap;
  const int stride = ctx->p.n + 1;  // the staging rows are packed like the host rows: plain 1-D copies
  uint32_t* dx = ctx->d_hx;
  uint32_t* dy = ctx->d_hx + (size_t)cap * stride;
  uint32_t* dout = ctx->d_hx + (size_t)2 * cap * stride;
  if ((rc = ensure_ext(ctx, k))) return rc;
  if (!ctx->s_in) {
    TFB_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking));
    TFB_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->s_run, cudaStreamNonBlocking));
    TFB_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking));
    for (auto& e : ctx->ev_in) TFB_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : ctx->ev_run) TFB_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // Three-stage pipeline over chunks of the launch: host->device copy of chunk c+1 and
  // device->host copy of chunk c-1 overlap the kernels of chunk c (rows: x = [0,cap),
  // y = [cap,2cap), out = [2cap,3cap) of the d_hx pool; chunks use disjoint row ranges).
  // The first chunk is short (two K1d waves) so that the kernels start after a small copy.
  const int64_t first = 2 * (int64_t)ctx->sm_count * K1D_WARPS;
  int slot = 0;
  for (int64_t c0 = 0; c0 < k; slot = (slot + 1) % HOST_EVENTS) {
    int64_t kc = (c0 == 0 && k > 2 * first) ? first : HOST_CHUNK;
    if (k - c0 < kc + first / 2) kc = k - c0;  // no crumbs: the last chunk absorbs a short rest
    const size_t off = (size_t)c0 * stride, bytes = (size_t)kc * stride * 4;
    TFB_CUDA(ctx, cudaMemcpyAsync(dx + off, x + off, bytes, cudaMemcpyHostToDevice, ctx->s_in));
    TFB_CUDA(ctx, cudaMemcpyAsync(dy + off, y + off, bytes, cudaMemcpyHostToDevice, ctx->s_in));
    TFB_CUDA(ctx, cudaMemcpyAsync(ctx->d_hkinds + c0, kinds + c0, (size_t)kc, cudaMemcpyHostToDevice, ctx->s_in));
    TFB_CUDA(ctx, cudaEventRecord(ctx->ev_in[slot], ctx->s_in));
    TFB_CUDA(ctx, cudaStreamWaitEvent(ctx->s_run, ctx->ev_in[slot], 0));
    uint32_t* ext = ctx->d_ext + (size_t)c0 * EXT_STRIDE;
    if ((rc = launch_blind_rotate(ctx, ctx->d_hx, stride, ctx->d_hkinds + c0, ctx->d_hrows + c0,
                                  ctx->d_hrows + cap + c0, ext, kc, ctx->s_run)))
      return rc;
    if ((rc = launch_key_switch(ctx, ext, ctx->d_hx, stride, ctx->d_hrows + 2 * cap + c0, kc, ctx->s_run))) return rc;
    TFB_CUDA(ctx, cudaEventRecord(ctx->ev_run[slot], ctx->s_run));
    TFB_CUDA(ctx, cudaStreamWaitEvent(ctx->s_out, ctx->ev_run[slot], 0));
    TFB_CUDA(ctx, cudaMemcpyAsync(out + off, dout + off, bytes, cudaMemcpyDeviceToHost, ctx->s_out));
    c0 += kc;
  }
  TFB_CUDA(ctx, cudaStreamSynchronize(ctx->s_out));
  TFB_CUDA(ctx, cudaStreamSynchronize(ctx->s_run));
  return TFB_OK;
}

int tfb_rows_negate(tfb_ctx* ctx, void* pool, const int32_t* in_rows, const int32_t* out_rows, int64_t k,
                    void* stream) {
  if (!ctx || !pool || !in_rows || !out_rows || k < 1) return TFB_ERR_INVALID;
  TFB_ENTER(ctx);
  k_rows_negate<<<(unsigned)k, 128, 0, (cudaStream_t)stream>>>((uint32_t*)pool, in_rows, out_rows);
  ctx->launches += 1;
  TFB_CUDA(ctx, cudaGetLastError());
  return TFB_OK;
}

int tfb_rows_phase(tfb_ctx* ctx, const void* pool, const int32_t* rows, const uint32_t* key_bits,
                   uint32_t* phase, int64_t k, void* stream) {
  if (!ctx || !pool || !rows || !key_bits || !phase || k < 1) return TFB_ERR_INVALID;
  TFB_ENTER(ctx);
  k_rows_phase<<<(unsigned)k, 128, 0, (cudaStream_t)stream>>>((const uint32_t*)pool, rows, key_bits, phase,
                                                             ctx->p.n);
  ctx->launches += 1;
  TFB_CUDA(ctx, cudaGetLastError());
  return TFB_OK;
}

int tfb_rows_encrypt(tfb_ctx* ctx, void* pool, const int32_t* out_rows, const uint8_t* bits, const uint32_t* key_bits,
                     double alpha, uint64_t seed, uint64_t first_sample, int64_t k, void* stream) {
  if (!ctx || !pool || !out_rows || !bits || !key_bits || k < 1 || !(alpha >= 0.0)) return TFB_ERR_INVALID;
  TFB_ENTER(ctx);
  k_rows_encrypt<<<(unsigned)k, 128, 0, (cudaStream_t)stream>>>((uint32_t*)pool, out_rows, bits, key_bits, ctx->p.n,
                                                               ctx->p.mu_word, alpha, seed, first_sample);
  ctx->launches += 1;
  TFB_CUDA(ctx, cudaGetLastError());
  return TFB_OK;
}

int tfb_debug_spectral_key(tfb_ctx* ctx, int32_t pair, int32_t key, double* out) {
  if (!ctx || !out || pair < 0 || pair >= (ctx->p.n + 1) / 2 || key < 0 || key >= BK_KEYS) return TFB_ERR_INVALID;
  if (!ctx->keys_loaded) return TFB_ERR_STATE;
  TFB_ENTER(ctx);
  const size_t per_pair = (size_t)BK_KEYS * BK_ROWS * 2 * HALF_N;
  std::vector<cd> h(per_pair);
  TFB_CUDA(ctx, cudaMemcpy(h.data(), ctx->d_bkf + (size_t)pair * per_pair, per_pair * sizeof(cd), cudaMemcpyDeviceToHost));
  for (int r = 0; r < BK_ROWS; ++r)
    for (int k2 = 0; k2 < 8; ++k2)
      for (int c = 0; c < 2; ++c)
        for (int t = 0; t < FFT_THREADS; ++t) {
          const cd v = h[pchunk_offset(0, r / BK_L, r % BK_L, k2 >> 2) + pchunk_index(k2 & 3, key, c, t)];
          const int f = spectral_index(t, k2);
          double* dst = out + (((size_t)(r * 2 + c) * HALF_N) + f) * 2;
          dst[0] = v.re * HALF_N;
          dst[1] = v.im * HALF_N;
        }
  return TFB_OK;
}

int tfb_debug_plan_kernels(int64_t k, int sms, int32_t* variants, int32_t* warps, int64_t* gates, int max_segments) {
  if (k < 1 || sms < 1) return 0;
  K1Seg seg[K1_MAX_SEGS];
  const int nseg = plan_k1(k, sms, seg);
  for (int i = 0; i < nseg && i < max_segments; ++i) {
    if (variants) variants[i] = seg[i].which;
    if (warps) warps[i] = seg[i].warps;
    if (gates) gates[i] = seg[i].gates;
  }
  return nseg;
}

int64_t tfb_kernel_launches(const tfb_ctx* ctx) { return ctx ? ctx->launches : 0; }

int tfb_measure_peaks(int device, double* fp64_tflops, double* int32_tops) {
  DeviceGuard guard(device);
  if (guard.err != cudaSuccess) return TFB_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return TFB_ERR_CUDA;
  const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 1 << 16;
  void* buf = nullptr;
  if (cudaMalloc(&buf, (size_t)blocks * threads * 8) != cudaSuccess) return TFB_ERR_CUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  double best_d = 0, best_i = 0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k_peak_dfma<<<blocks, threads>>>((double*)buf, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * 8.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
    if (rep && tf > best_d) best_d = tf;
    cudaEventRecord(e0);
    k_peak_imad<<<blocks, threads>>>((int32_t*)buf, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double to = 8.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
    if (rep && to > best_i) best_i = to;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  if (cudaGetLastError() != cudaSuccess) return TFB_ERR_CUDA;
  if (fp64_tflops) *fp64_tflops = best_d;
  if (int32_tops) *int32_tops = best_i;
  return TFB_OK;
}

}  // extern "C"
