// K1e k_gate_bootstrap_pair -- the latency kernel: ONE gate per thread-block CLUSTER of two CTAs.
//
// The critical path of a bootstrap is 500 dependent CMux steps, each a forward and an inverse
// 512-point transform deep (a phase probe of K1c, tools/microbench/k1c_probe.cu, puts one CMux of the
// single-CTA latency kernel at ~5,300 cycles: 1,600 forward with two warps per scheduler sharing the FP64
// pipe, 1,000 rotate/decompose, 1,200 for the four-way product reduction through shared memory, 1,000
// inverse on half of the CTA while the other half idles).  Here the two accumulator polynomials of a
// ciphertext live on two SMs:
//
//   CTA p (cluster rank) owns ACC[p].  Its two 64-thread groups transform the two gadget levels of
//   (X^abar - 1) ACC[p] -- one warp per scheduler, nobody shares an FP64 pipe -- and multiply by their share
//   of key stage (i, p) for BOTH output polynomials.  The groups swap one product each through shared
//   memory, so that group g holds CTA p's whole contribution to output polynomial c = p ^ g, and BOTH run
//   an inverse transform (no idle half).  Group 0's result is the CTA's own update of ACC[p]; group 1's,
//   rounded to integers, is the contribution to the OTHER CTA's polynomial and travels as 4 KB of
//   `st.async` stores into the peer's shared memory (DSMEM), completing on the peer's mbarrier.
//
// Exactness: each CTA's contribution sum_lvl d_{p,lvl} * BK_{p,lvl,c} is an exact integer polynomial, so
// rounding the two contributions separately and adding them mod 2^32 gives the same words as rounding the
// sum (the kernel is held bit-exact to the oracle like every other variant).  One cluster-scope exchange per
// CMux (the complex products would be twice as many bytes), double buffered by iteration parity; no cluster
// barrier inside the loop.
//
// Measured (B200, -DTFB_K1E_PROBE, cycles per CMux): rotate/decompose ~450, forward ~1,000, products + swap ~250,
// sum + inverse ~1,200, rounding + DSMEM exchange ~875 of which ~750 is waiting for the peer's 4 KB (half the
// bytes: -215 cycles, i.e. ~10 B/clk plus ~320 of latency; a generic-proxy st.shared::cluster + release.cluster
// arrive was 18 % slower, one TMA bulk copy from a local staging buffer the same as st.async), key issue ~200:
// ~4,000 cycles, 1.04 ms per bootstrap against 1.34 ms for K1c.
#pragma once
#include "tfhe_device.cuh"

namespace k1e {
using namespace tfb;

constexpr int THREADS = 2 * FFT_THREADS;  // per CTA: one 64-thread group per gadget level
constexpr int RECV_WORDS = RING_N;        // one polynomial of rounded words, layout [thread][16]
// dynamic shared memory of one CTA
constexpr int OFF_XBUF = 0;                                               // 2 groups x 2 exchange buffers x 512 cd
constexpr int OFF_SWAP = OFF_XBUF + 2 * 2 * HALF_N * (int)sizeof(cd);     // 2 groups x 8 x 64 cd
constexpr int OFF_ACC = OFF_SWAP + 2 * HALF_N * (int)sizeof(cd);          // N words
constexpr int OFF_RECV = OFF_ACC + RING_N * 4;                            // 2 buffers x N words
constexpr int OFF_BARS = OFF_RECV + 2 * RECV_WORDS * 4;                   // 2 mbarriers
constexpr int OFF_ABAR = OFF_BARS + 16;
__host__ __device__ constexpr int smem_bytes(int n) { return OFF_ABAR + ((n + 1) * 2 + 15) / 16 * 16; }

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

struct PairGroupSync {  // named barrier over one 64-thread group
  int id;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(FFT_THREADS) : "memory");
  }
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1) k_gate_bootstrap_pair(
    const uint32_t* __restrict__ pool, const uint8_t* __restrict__ kinds, const int32_t* __restrict__ x_rows,
    const int32_t* __restrict__ y_rows, int stride, int n, uint32_t mu, const cd* __restrict__ bkf,
    const Twiddles* __restrict__ tw_global, uint32_t* __restrict__ ext) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, grp = tid / FFT_THREADS, t = tid % FFT_THREADS;
  const uint32_t p = cluster_rank();  // accumulator polynomial of this CTA
  const int64_t g = blockIdx.x >> 1;  // gate = cluster
  cd* bufA = reinterpret_cast<cd*>(smem + OFF_XBUF) + (size_t)grp * 2 * HALF_N;
  cd* bufB = bufA + HALF_N;
  cd* swap = reinterpret_cast<cd*>(smem + OFF_SWAP);  // [group][k2][t]
  uint32_t* acc = reinterpret_cast<uint32_t*>(smem + OFF_ACC);
  uint32_t* recv = reinterpret_cast<uint32_t*>(smem + OFF_RECV);  // [buffer][t][16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BARS);
  uint16_t* abar = reinterpret_cast<uint16_t*>(smem + OFF_ABAR);

  // gate linear form + mod switch (both CTAs: 501 words each), accumulator polynomial p of the test vector
  {
    const uint32_t* xr = pool + (int64_t)x_rows[g] * stride;
    const uint32_t* yr = pool + (int64_t)y_rows[g] * stride;
    int32_t cx, cy, off;
    gate_coeffs((int)kinds[g], cx, cy, off);
    for (int w = tid; w <= n; w += THREADS) {
      uint32_t v = (uint32_t)cx * xr[w] + (uint32_t)cy * yr[w];
      if (w == n) v += (uint32_t)off * mu;
      abar[w] = (uint16_t)mod_switch(v);
    }
    if (tid == 0) {
      for (int b = 0; b < 2; ++b)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[b])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int bbar = abar[n];
    for (int j = tid; j < RING_N; j += THREADS) {
      const int src = (j + bbar) & (2 * RING_N - 1);
      acc[j] = p == 0 ? 0u : (src < RING_N ? mu : (0u - mu));
    }
  }
  cluster_sync_all();  // the peer's mbarriers exist before anything is sent to them

  RegTw rtw;
  rtw.load(tw_global, t);
  PairGroupSync gsync{grp + 1};
  const int c_keep = (int)p ^ grp;  // output polynomial this group inverse-transforms
  const uint32_t peer = p ^ 1u;
  const uint32_t bars_local = (uint32_t)__cvta_generic_to_shared(bars);
  const uint32_t recv_peer = peer_address((uint32_t)__cvta_generic_to_shared(recv), peer);
  const uint32_t bars_peer = peer_address(bars_local, peer);
  uint32_t done = 0;  // CMux steps executed so far: buffer = done & 1, phase parity = (done >> 1) & 1
  cd b_keep[8], b_give[8];
  int loaded_for = -1;
  auto load_key = [&](int i) {
    const cd* stage = bkf + stage_offset(i, (int)p);
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      const double2 u = __ldg(reinterpret_cast<const double2*>(stage + stage_index(k2, grp, c_keep, t)));
      const double2 v = __ldg(reinterpret_cast<const double2*>(stage + stage_index(k2, grp, c_keep ^ 1, t)));
      b_keep[k2] = cd{u.x, u.y};
      b_give[k2] = cd{v.x, v.y};
    }
    loaded_for = i;
  };
#ifdef TFB_K1E_PROBE
  long long T[8] = {0, 0, 0, 0, 0, 0, 0, 0}, c0 = clock64(), c1;
#define K1E_TICK(k) c1 = clock64(); T[k] += c1 - c0; c0 = c1;
#else
#define K1E_TICK(k)
#endif

#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    const int ab = abar[i];
    if (ab == 0) continue;  // uniform across the cluster: both CTAs derive the same abar
    const uint32_t buf = done & 1u, parity = (done >> 1) & 1u;
    if (tid == 0)  // arm this step's receive: 4 KB from the peer's group 1
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bars_local + 8u * buf), "r"(RECV_WORDS * 4)
                   : "memory");
    // key stage (i, p), level grp, both output components: normally already in flight (requested right after the
    // previous step's products); loaded here for the first step and after a skipped one
    if (loaded_for != i) load_key(i);
    K1E_TICK(0)
    cd x[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const uint32_t vr = rotated_diff(acc, t + 64 * m, ab) + DECOMP_OFFSET;
      const uint32_t vi = rotated_diff(acc, t + 64 * m + HALF_N, ab) + DECOMP_OFFSET;
      x[m] = cd{digit_to_double(digit_field(vr, grp)), digit_to_double(digit_field(vi, grp))};
    }
    K1E_TICK(1)
    fft_forward(x, t, rtw, bufA, bufB, gsync);
    K1E_TICK(2)
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      swap[(grp * 8 + k2) * FFT_THREADS + t] = cmul(x[k2], b_give[k2]);
      x[k2] = cmul(x[k2], b_keep[k2]);
    }
    if (i + 1 < n) load_key(i + 1);  // the next step's key travels during the inverse transform and the exchange
    K1E_TICK(3)
    __syncthreads();
    K1E_TICK(4)
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) x[k2] = cadd(x[k2], swap[((grp ^ 1) * 8 + k2) * FFT_THREADS + t]);
    fft_inverse(x, t, rtw, bufA, bufB, gsync);
    K1E_TICK(5)
    uint32_t v[16];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      v[m] = round_to_word(x[m].re);      // coefficient t + 64 m
      v[8 + m] = round_to_word(x[m].im);  // coefficient t + 64 m + N/2
    }
    if (grp == 1) {  // this CTA's contribution to the peer's polynomial
      const uint32_t dst = recv_peer + (buf * RECV_WORDS + (uint32_t)t * 16u) * 4u;
#pragma unroll
      for (int q = 0; q < 4; ++q) send4(dst + 16u * q, bars_peer + 8u * buf, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {  // own contribution now, the peer's when it has landed
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        acc[t + 64 * m] += v[m];
        acc[t + 64 * m + HALF_N] += v[8 + m];
      }
      wait_cluster_phase(bars_local + 8u * buf, parity);
      const uint4* r4 = reinterpret_cast<const uint4*>(recv + buf * RECV_WORDS + t * 16);
      uint32_t r[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 u = r4[q];
        r[4 * q] = u.x;
        r[4 * q + 1] = u.y;
        r[4 * q + 2] = u.z;
        r[4 * q + 3] = u.w;
      }
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        acc[t + 64 * m] += r[m];
        acc[t + 64 * m + HALF_N] += r[8 + m];
      }
    }
    ++done;
    K1E_TICK(6)
    __syncthreads();
    K1E_TICK(7)
  }
#ifdef TFB_K1E_PROBE
  if (t == 0 && blockIdx.x < 2)
    printf("cta %d grp %d: key %lld decomp %lld fwd %lld mac %lld sync %lld sum+inv %lld round+send/recv %lld sync %lld\n",
           (int)blockIdx.x, grp, T[0] / n, T[1] / n, T[2] / n, T[3] / n, T[4] / n, T[5] / n, T[6] / n, T[7] / n);
#endif
  // sample extract at coefficient 0: the mask comes from ACC[0], the body from ACC[1]
  uint32_t* out = ext + g * EXT_STRIDE;
  if (p == 0) {
    for (int j = tid; j < RING_N; j += THREADS) out[j] = (j == 0) ? acc[0] : (0u - acc[RING_N - j]);
  } else if (tid == 0) {
    out[RING_N] = acc[0];
  }
  cluster_sync_all();  // nobody leaves while the peer may still address its shared memory
}

}  // namespace k1e
