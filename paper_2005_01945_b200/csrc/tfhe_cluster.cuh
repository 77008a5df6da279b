// K1e k_gate_bootstrap_pair -- the latency kernel: ONE gate per thread-block CLUSTER of two CTAs.
//
// The critical path of a bootstrap is ceil(n/2) dependent pair steps (the bootstrapping key is unrolled over
// pairs of mask elements), each a forward and an inverse 512-point transform deep.  The two accumulator
// polynomials of a ciphertext live on two SMs; the arithmetic is tfhe_pair.cuh (the same code tests/emu runs on
// host threads), this file is its device environment.  A CTA has eight warps:
//
//   * warps 0-3, the MAIN groups (one 64-thread group per gadget level, one warp per scheduler): digits, forward
//     transform, two complex multiplications per point with the step's combined keys, product swap, inverse
//     transform, rounding, peer exchange, accumulator update;
//   * warps 4-7, the KEY COMBINERS (again one group per gadget level): they stream the group's 48 KB of spectral key
//     per step through a two-slot shared-memory ring of 24 KB chunks filled by `cp.async.bulk` (TMA, completing on
//     mbarriers; a slot is refilled by the group's thread 0 after the group barrier that follows its last read:
//     generic-proxy reads -> barrier -> fence.proxy.async -> bulk copy), fold the rotation factors of step s+1 into
//     the three keys while the main groups run step s, and hand the 16 KB result over in shared memory, double
//     buffered, on named barriers (bar.arrive by the producers / bar.sync by the consumers and back).  The key
//     combination -- 272 of a step's ~850 FP64 instructions per thread and all of its key traffic -- is thereby off
//     the critical path; steps whose rotations are both zero are skipped by both roles;
//   * peer exchange: main group 1's rounded contribution to the OTHER CTA's polynomial travels as 4 KB of `st.async`
//     stores into the peer's shared memory (DSMEM), completing on the peer's mbarrier, double buffered by step
//     parity; no cluster barrier inside the loop.
//
// Measured history of the exchange variants (st.async kept; generic-proxy st.shared::cluster + release arrive
// 18 % slower; one TMA bulk copy from a staging buffer the same) is in profiles/README.md.
#pragma once
#include "tfhe_pair.cuh"

namespace k1e {
using namespace tfb;

constexpr int THREADS = 2 * PAIR_THREADS;  // 128 main threads + 128 key combiners
constexpr int RECV_WORDS = RING_N;  // one polynomial of rounded words, layout [thread][16]
constexpr int RING_SLOTS = 2;
constexpr int CHUNK_BYTES = PCHUNK_CD * (int)sizeof(cd);  // 24 KB
// dynamic shared memory of one CTA
constexpr int OFF_RING = 0;                                                   // 2 groups x 2 slots x 24 KB
constexpr int OFF_KEYS = OFF_RING + 2 * RING_SLOTS * CHUNK_BYTES;             // 2 buffers x 2 groups x 16 KB combined keys
constexpr int OFF_XBUF = OFF_KEYS + 2 * 2 * PAIR_KEYS_CD * (int)sizeof(cd);   // 2 groups x 2 exchange buffers x 512 cd
constexpr int OFF_SWAP = OFF_XBUF + 2 * 2 * HALF_N * (int)sizeof(cd);         // 2 groups x 8 x 64 cd
constexpr int OFF_ACC = OFF_SWAP + 2 * HALF_N * (int)sizeof(cd);              // N words
constexpr int OFF_RECV = OFF_ACC + RING_N * 4;                                // 2 buffers x N words
constexpr int OFF_FT = OFF_RECV + 2 * RECV_WORDS * 4;                         // FactorTables
// mbarriers: RECV_BARS receive barriers per step parity (the peer's 4 KB is accounted on several barriers: every
// st.async completes 16 bytes of transaction count on its barrier, and 256 of them on ONE barrier serialise), then
// 2 x 2 ring barriers
#ifndef TFB_K1E_RECV_BARS
#define TFB_K1E_RECV_BARS 2
#endif
constexpr int RECV_BARS = TFB_K1E_RECV_BARS;
static_assert(RECV_BARS == 1 || RECV_BARS == 2 || RECV_BARS == 4, "one barrier per st.async of a thread, or fewer");
constexpr int OFF_BARS = OFF_FT + (int)sizeof(FactorTables);
constexpr int OFF_ABAR = OFF_BARS + 128;
__host__ __device__ constexpr int smem_bytes(int n) { return OFF_ABAR + ((n + 2) * 2 + 15) / 16 * 16; }

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t peer_address(uint32_t local_smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem_addr), "r"(rank));
  return r;
}
// four words into the peer's shared memory; the bytes count towards the peer's mbarrier
__device__ __forceinline__ void send4(uint32_t peer_addr, uint32_t peer_bar, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   peer_addr),
               "r"(a), "r"(b), "r"(c), "r"(d), "r"(peer_bar)
               : "memory");
}
__device__ __forceinline__ void wait_cluster_phase(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "PAIR_WAIT:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra PAIR_DONE;\n"
      "bra PAIR_WAIT;\n"
      "PAIR_DONE:\n"
      "}\n" ::"r"(bar), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void wait_cta_phase(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "KEY_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra KEY_DONE;\n"
      "bra KEY_WAIT;\n"
      "KEY_DONE:\n"
      "}\n" ::"r"(bar), "r"(parity)
      : "memory");
}

// named barriers: 0 all 256 threads | 1, 2 main groups | 3 the 128 main threads | 4, 5 combiner groups |
// 6 + 2 grp + buf: combined keys of (group, buffer) complete | 10 + 2 grp + buf: ... taken by the main group
constexpr int BAR_MAIN_CTA = 3, BAR_KEYS_FULL = 6, BAR_KEYS_EMPTY = 10;
struct PairGroupSync {  // named barrier over one 64-thread group
  int id;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(FFT_THREADS) : "memory");
  }
};

struct DeviceEnv {
  static constexpr bool helpers = true;
  PairGroupSync gsync;  // this thread's 64-thread group (main or combiner)
  const cd* bkf;        // spectral key in global memory (pchunk layout)
  cd* ring;             // this gadget level's two slots
  cd* keys;             // combined-key blocks [buffer][group][keep / give][k2][t]
  uint32_t bars_local;  // shared-space address of the CTA's mbarriers: [parity * RECV_BARS + j] receive, then [2 grp + slot] ring
  uint32_t recv_local, recv_peer, bars_peer;
  const uint16_t* abar;
  int n, p, grp, t, tid;
  int next_m, next_h;   // producer cursor (thread 0 of a combiner group): next chunk to request
  uint32_t issued;

  __device__ __forceinline__ void cta_sync() { asm volatile("bar.sync %0, %1;" ::"n"(BAR_MAIN_CTA), "n"(PAIR_THREADS) : "memory"); }
  __device__ __forceinline__ void all_sync() { __syncthreads(); }
  __device__ __forceinline__ uint32_t ring_bar(uint32_t seq) const {
    return bars_local + 8u * (2u * RECV_BARS + (uint32_t)RING_SLOTS * (uint32_t)grp + seq % RING_SLOTS);
  }
  __device__ __forceinline__ void issue_next() {  // thread 0 of a combiner group only
    next_m = pair_next_active(abar, n, next_m);
    if (next_m >= (n + 1) / 2) return;
    const uint32_t bar = ring_bar(issued);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + (size_t)(issued % RING_SLOTS) * PCHUNK_CD);
    const cd* src = bkf + pchunk_offset(next_m, p, grp, next_h);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(CHUNK_BYTES) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(CHUNK_BYTES), "r"(bar)
                 : "memory");
    ++issued;
    if (++next_h == 2) {
      next_h = 0;
      ++next_m;
    }
  }
  __device__ __forceinline__ void start(const uint16_t*, int) {
    if (tid == 0) {
      for (int b = 0; b < 2 * RECV_BARS + 2 * RING_SLOTS; ++b)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars_local + 8u * b) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid >= PAIR_THREADS && t == 0)
      for (int s = 0; s < RING_SLOTS; ++s) issue_next();
    cluster_sync_all();  // the peer's mbarriers exist before anything is sent to them
  }
  __device__ __forceinline__ const cd* key_wait(uint32_t seq, int, int) {
    wait_cta_phase(ring_bar(seq), (seq / RING_SLOTS) & 1u);
    return ring + (size_t)(seq % RING_SLOTS) * PCHUNK_CD;
  }
  // every thread of the group has read chunk `seq` and passed a barrier: its slot takes the chunk RING_SLOTS ahead
  __device__ __forceinline__ void key_done(uint32_t, int, int) {
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_next();
    }
  }
  __device__ __forceinline__ cd* keys_block(uint32_t step) const { return keys + (size_t)((step & 1u) * 2u + (uint32_t)grp) * PAIR_KEYS_CD; }
  // combiner side: wait until the main group has taken the block two steps back, ...
  __device__ __forceinline__ cd* keys_slot(uint32_t step) {
    if (step >= 2) asm volatile("bar.sync %0, %1;" ::"r"(BAR_KEYS_EMPTY + 2 * grp + (int)(step & 1u)), "n"(PAIR_THREADS) : "memory");
    return keys_block(step);
  }
  // ... publish it (the group barrier in front also frees the second key chunk for its refill)
  __device__ __forceinline__ void keys_publish(uint32_t step) {
    gsync();
    __threadfence_block();
    asm volatile("bar.arrive %0, %1;" ::"r"(BAR_KEYS_FULL + 2 * grp + (int)(step & 1u)), "n"(PAIR_THREADS) : "memory");
  }
  // the main group's last two "taken" arrivals have no later block to release: absorb them
  __device__ __forceinline__ void keys_drain(uint32_t steps) {
    for (uint32_t s = steps >= 2 ? steps - 2 : 0; s < steps; ++s)
      asm volatile("bar.sync %0, %1;" ::"r"(BAR_KEYS_EMPTY + 2 * grp + (int)(s & 1u)), "n"(PAIR_THREADS) : "memory");
  }
  // main side
  __device__ __forceinline__ const cd* keys_ready(uint32_t step) {
    asm volatile("bar.sync %0, %1;" ::"r"(BAR_KEYS_FULL + 2 * grp + (int)(step & 1u)), "n"(PAIR_THREADS) : "memory");
    return keys_block(step);
  }
  __device__ __forceinline__ void keys_taken(uint32_t step) {
    asm volatile("bar.arrive %0, %1;" ::"r"(BAR_KEYS_EMPTY + 2 * grp + (int)(step & 1u)), "n"(PAIR_THREADS) : "memory");
  }
  __device__ __forceinline__ void arm_recv(uint32_t step) {  // 4 KB from the peer's group 1, split over RECV_BARS barriers
#pragma unroll
    for (int j = 0; j < RECV_BARS; ++j)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bars_local + 8u * ((step & 1u) * RECV_BARS + j)),
                   "r"(RECV_WORDS * 4 / RECV_BARS)
                   : "memory");
  }
  __device__ __forceinline__ void send16(const uint32_t* v, uint32_t step) {
    const uint32_t buf = step & 1u;
    const uint32_t dst = recv_peer + (buf * RECV_WORDS + (uint32_t)t * 16u) * 4u;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      send4(dst + 16u * q, bars_peer + 8u * (buf * RECV_BARS + q % RECV_BARS), v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
  __device__ __forceinline__ void recv16(uint32_t* r, uint32_t step) {
    const uint32_t buf = step & 1u;
#pragma unroll
    for (int j = 0; j < RECV_BARS; ++j) wait_cluster_phase(bars_local + 8u * (buf * RECV_BARS + j), (step >> 1) & 1u);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t a, b, c, d;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                   : "r"(recv_local + (buf * RECV_WORDS + (uint32_t)t * 16u + 4u * q) * 4u)
                   : "memory");
      r[4 * q] = a;
      r[4 * q + 1] = b;
      r[4 * q + 2] = c;
      r[4 * q + 3] = d;
    }
  }
  __device__ __forceinline__ void finish() {
#ifdef TFB_K1E_PROBE
    if (tid < PAIR_THREADS && t == 0 && blockIdx.x < 2) {
      const long long s = steps ? steps : 1;
      printf("cta %d grp %d per step: top %lld digits %lld fwd %lld keys+products+sync %lld sum+inv %lld round+send/own %lld - %lld recv %lld sync %lld\n",
             (int)blockIdx.x, grp, T[0] / s, T[1] / s, T[2] / s, T[3] / s, T[4] / s, T[5] / s, T[6] / s, T[7] / s, T[8] / s);
    }
#endif
    cluster_sync_all();  // nobody leaves while the peer may still address its shared memory
  }
#ifdef TFB_K1E_PROBE
  long long T[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, last = 0, steps = 0;
  __device__ __forceinline__ void tick(int k) {
    const long long now = clock64();
    if (last) T[k] += now - last;
    last = now;
    steps += k == 8;
  }
#else
  __device__ __forceinline__ void tick(int) {}
#endif
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1) k_gate_bootstrap_pair(
    const uint32_t* __restrict__ pool, const uint8_t* __restrict__ kinds, const int32_t* __restrict__ x_rows,
    const int32_t* __restrict__ y_rows, int stride, int n, uint32_t mu, const cd* __restrict__ bkf,
    const Twiddles* __restrict__ tw_global, const FactorTables* __restrict__ ft_global, uint32_t* __restrict__ ext) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const bool combiner = tid >= PAIR_THREADS;
  const int grp = (tid % PAIR_THREADS) / FFT_THREADS, t = tid % FFT_THREADS;
  const uint32_t p = cluster_rank();  // accumulator polynomial of this CTA
  const int64_t g = blockIdx.x >> 1;  // gate = cluster
  cd* bufA = reinterpret_cast<cd*>(smem + OFF_XBUF) + (size_t)grp * 2 * HALF_N;
  cd* swap = reinterpret_cast<cd*>(smem + OFF_SWAP);  // [group][k2][t]
  uint32_t* acc = reinterpret_cast<uint32_t*>(smem + OFF_ACC);
  FactorTables* ft = reinterpret_cast<FactorTables*>(smem + OFF_FT);
  uint16_t* abar = reinterpret_cast<uint16_t*>(smem + OFF_ABAR);
  for (int i = tid; i < (int)(sizeof(FactorTables) / sizeof(cd)); i += THREADS)
    reinterpret_cast<cd*>(ft)[i] = reinterpret_cast<const cd*>(ft_global)[i];
  const uint32_t bars_local = (uint32_t)__cvta_generic_to_shared(smem + OFF_BARS);
  const uint32_t recv_local = (uint32_t)__cvta_generic_to_shared(smem + OFF_RECV);
  DeviceEnv env{PairGroupSync{(combiner ? 4 : 1) + grp},
                bkf,
                reinterpret_cast<cd*>(smem + OFF_RING) + (size_t)grp * RING_SLOTS * PCHUNK_CD,
                reinterpret_cast<cd*>(smem + OFF_KEYS),
                bars_local,
                recv_local,
                peer_address(recv_local, p ^ 1u),
                peer_address(bars_local, p ^ 1u),
                abar,
                n,
                (int)p,
                grp,
                t,
                tid,
                0,
                0,
                0u};
  pair_prologue(env, pool + (int64_t)x_rows[g] * stride, pool + (int64_t)y_rows[g] * stride, (int)kinds[g], n, mu, acc, abar,
                (int)p, tid, THREADS);
  if (combiner) {
    const uint32_t steps = pair_key_combiner(env, abar, n, ft, (int)p, grp, t);
    env.keys_drain(steps);
  } else {
    pair_blind_rotate(env, n, tw_global, ft, acc, abar, bufA, bufA + HALF_N, swap, (int)p, tid);
    pair_extract(acc, ext + g * EXT_STRIDE, (int)p, tid);
  }
  env.finish();
}

}  // namespace k1e
