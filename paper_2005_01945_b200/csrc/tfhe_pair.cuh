// K1e arithmetic: ONE gate by FOUR 64-thread groups on TWO CTAs (a thread-block cluster on the device,
// tfhe_cluster.cuh; four thread groups with barriers in tests/emu).
//
// CTA p (cluster rank) owns accumulator polynomial ACC[p].  Its group `lvl` transforms gadget level `lvl`
// of ACC[p] -- one warp per scheduler, nobody shares an FP64 pipe -- and multiplies it by the combined key
//   K[(p, lvl), c] = u1 B1 + u2 B2 + u1 u2 B12   (rows (p, lvl) of the pair's three TRGSW samples, u = X^a - 1
// as spectral factors) for BOTH output polynomials c.  The two groups swap one product each through shared
// memory, so that group g holds CTA p's whole contribution to output polynomial c = p ^ g, and BOTH run an
// inverse transform.  Group 0's result is the CTA's own update of ACC[p]; group 1's, rounded to integers, is
// the contribution to the OTHER CTA's polynomial and travels to the peer (DSMEM on the device).
//
// Exactness: each CTA's contribution is an exact integer polynomial, so rounding the two contributions
// separately and adding them mod 2^32 gives the same words as rounding the sum.
//
// The combined keys depend on the rotations and the bootstrapping key only -- not on ACC -- so they are
// taken off the critical path: on the device four more warps per CTA (the KEY COMBINERS, one 64-thread
// group per gadget level) stream the key through the ring, combine the keys of step s+1 while the main
// groups run step s, and hand them over in shared memory; a main thread's share of a step is then two
// complex multiplications per spectral point.  Env::helpers = false (tests/emu) lets the main groups
// combine their keys themselves, in the tail of the previous step.
//
// Env (the environment the body runs in) provides
//   helpers                   static constexpr bool, see above
//   gsync                     functor: barrier over this thread's 64-thread group
//   cta_sync()                barrier over the CTA's 128 main threads
//   all_sync()                barrier over every thread of the CTA (main + combiners)
//   start(abar, n)            every thread, after the rotations are known: set up and start the key pipeline,
//                             cluster barrier
//   key_wait(seq, m, h)       -> const cd*: chunk (m, p, lvl, h) of the spectral key (seq = running chunk number
//                             of this group, counting consumed chunks only)
//   key_done(seq, m, h)       every thread of the group has finished reading the chunk AND a group-wide (or wider)
//                             barrier has passed since
//   keys_ready(step)          main, helpers only: -> const cd* [keep / give][k2][t] of this group for `step`
//   keys_taken(step)          main, helpers only: this thread holds its copy
//   keys_slot(step)           combiner: -> cd* the same block once the main group has released it
//   keys_publish(step)        combiner: the block is complete
//   arm_recv(step)            thread 0 of the CTA, before anything of this step can arrive
//   send16(v, step)           group 1: sixteen rounded words per thread to the peer
//   recv16(r, step)           group 0: the peer's sixteen words for this thread (blocks until they have landed)
//   finish()                  every thread: nobody leaves while the peer may still address this CTA
//   tick(k)                   profiling hook (no-op outside probe builds)
#pragma once
#include "tfhe_device.cuh"

namespace tfb {

constexpr int PAIR_THREADS = 2 * FFT_THREADS;  // main threads per CTA: one 64-thread group per gadget level
constexpr int PAIR_KEYS_CD = 2 * 8 * FFT_THREADS;  // one group's combined keys of a step: [keep / give][k2][t]

TFB_HD bool pair_is_active(const uint16_t* abar, int n, int m) {
  int a1, a2;
  pair_rotations(abar, n, m, a1, a2);
  return (a1 | a2) != 0;
}
TFB_HD int pair_next_active(const uint16_t* abar, int n, int m) {
  const int pairs = (n + 1) / 2;
  while (m < pairs && !pair_is_active(abar, n, m)) ++m;
  return m;
}

// Combined keys of pair m for the eight spectral points of thread t of group `grp` (gadget level) of CTA p:
// keep[k2] multiplies into the output polynomial the group inverse-transforms (p ^ grp), give[k2] into the other.
// STRIDE: distance between consecutive k2 (1 for registers, FFT_THREADS for the shared-memory block).
// Leaves the second chunk's key_done to the caller: it needs a barrier after the group's last read.
template <int STRIDE, class Env>
TFB_HD void pair_combine_keys(Env& env, const uint16_t* abar, int n, int m, uint32_t seq, const FactorTables* ft, int p,
                              int grp, int t, cd* keep, cd* give) {
  const int c_keep = p ^ grp;
  const uint32_t cl = 1u + 4u * (uint32_t)spectral_index(t, 0);  // spectral point k2 of this thread: 1 + 4 f = cl + 256 k2
  int a1, a2;
  pair_rotations(abar, n, m, a1, a2);
  const cd base1 = unit_root(ft, (uint32_t)a1 * cl), base2 = unit_root(ft, (uint32_t)a2 * cl);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const cd* chunk = env.key_wait(seq + h, m, h);
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const int k2 = 4 * h + k4;
      // X^a at point cl + 256 k2: base * exp(i pi a 256 k2 / N) = base * A[8 a k2 mod 64]
      const cd u1 = rotation_minus_one(base1, ft->A[(8 * a1 * k2) & 63]);
      const cd u2 = rotation_minus_one(base2, ft->A[(8 * a2 * k2) & 63]);
      keep[k2 * STRIDE] = combine_keys(u1, u2, chunk[pchunk_index(k4, 0, c_keep, t)], chunk[pchunk_index(k4, 1, c_keep, t)],
                                       chunk[pchunk_index(k4, 2, c_keep, t)]);
      give[k2 * STRIDE] = combine_keys(u1, u2, chunk[pchunk_index(k4, 0, c_keep ^ 1, t)],
                                       chunk[pchunk_index(k4, 1, c_keep ^ 1, t)], chunk[pchunk_index(k4, 2, c_keep ^ 1, t)]);
    }
    if (h == 0) {
      env.gsync();
      env.key_done(seq, m, 0);
    }
  }
}

// Every thread of the CTA (`nthreads` of them): rotations, this CTA's polynomial of the test vector, key pipeline.
// acc: N words (polynomial p only); abar: n + 2 entries.
template <class Env>
TFB_HD void pair_prologue(Env& env, const uint32_t* x_row, const uint32_t* y_row, int kind, int n, uint32_t mu, uint32_t* acc,
                          uint16_t* abar, int p, int tid, int nthreads) {
  gate_mod_switch(x_row, y_row, kind, n, mu, abar, tid, nthreads);
  env.all_sync();
  const int bbar = abar[n];
  for (int j = tid; j < RING_N; j += nthreads) acc[j] = p == 0 ? 0u : test_vector_coeff(j, bbar, mu);
  env.start(abar, n);
}

// Key combiner group `grp` (64 threads, Env::helpers only): one block of combined keys per active pair.
template <class Env>
TFB_HD uint32_t pair_key_combiner(Env& env, const uint16_t* abar, int n, const FactorTables* ft, int p, int grp, int t) {
  const int pairs = (n + 1) / 2;
  uint32_t step = 0;
#if defined(__CUDA_ARCH__)
#pragma unroll 1
#endif
  for (int m = pair_next_active(abar, n, 0); m < pairs; m = pair_next_active(abar, n, m + 1), ++step) {
    // (holding the combiners back until the main groups reach the tail of step s-1, so that they never share an FP64
    // pipe with a transform, was measured: the main groups then wait for their keys, 0.68 instead of 0.63 ms)
    cd* block = env.keys_slot(step);
    pair_combine_keys<FFT_THREADS>(env, abar, n, m, 2 * step, ft, p, grp, t, block + t, block + 8 * FFT_THREADS + t);
    env.keys_publish(step);  // includes a group barrier: the second chunk may be refilled
    env.key_done(2 * step + 1, m, 1);
  }
  return step;  // blocks published
}

// The 128 main threads.  bufA/bufB: this group's exchange buffers (512 cd each); swap: [group][8][64] cd shared by the
// CTA's two groups.
template <class Env>
TFB_HD void pair_blind_rotate(Env& env, int n, const Twiddles* tw, const FactorTables* ft, uint32_t* acc, const uint16_t* abar,
                              cd* bufA, cd* bufB, cd* swap, int p, int tid) {
  const int grp = tid / FFT_THREADS, t = tid % FFT_THREADS;
  RegTw rtw;
  rtw.load(tw, t);
  const int pairs = (n + 1) / 2;
  cd kk[8], kg[8];
  uint32_t step = 0;  // active pairs so far: receive buffer = step & 1
  int m = pair_next_active(abar, n, 0);
  if (!Env::helpers && m < pairs) {
    pair_combine_keys<1>(env, abar, n, m, 0, ft, p, grp, t, kk, kg);
    env.cta_sync();
    env.key_done(1, m, 1);
  }
  if (tid == 0 && m < pairs) env.arm_recv(0);
#if defined(__CUDA_ARCH__)
#pragma unroll 1
#endif
  while (m < pairs) {  // uniform across the cluster: both CTAs derive the same rotations
    env.tick(0);
    cd x[8];
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
      const uint32_t vr = acc[t + 64 * mm] + DECOMP_OFFSET, vi = acc[t + 64 * mm + HALF_N] + DECOMP_OFFSET;
      x[mm] = cd{digit_to_double(digit_field(vr, grp)), digit_to_double(digit_field(vi, grp))};
    }
    env.tick(1);
    fft_forward(x, t, rtw, bufA, bufB, env.gsync);
    env.tick(2);
    if (Env::helpers) {
      const cd* block = env.keys_ready(step) + t;
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        kk[k2] = block[k2 * FFT_THREADS];
        kg[k2] = block[(8 + k2) * FFT_THREADS];
      }
      env.keys_taken(step);
    }
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      swap[(grp * 8 + k2) * FFT_THREADS + t] = cmul(x[k2], kg[k2]);
      x[k2] = cmul(x[k2], kk[k2]);
    }
    env.cta_sync();
    env.tick(3);
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) x[k2] = cadd(x[k2], swap[((grp ^ 1) * 8 + k2) * FFT_THREADS + t]);
    fft_inverse(x, t, rtw, bufA, bufB, env.gsync);
    env.tick(4);
    uint32_t v[16];
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
      v[mm] = round_to_word(x[mm].re);      // coefficient t + 64 mm
      v[8 + mm] = round_to_word(x[mm].im);  // coefficient t + 64 mm + N/2
    }
    if (grp == 1) {  // this CTA's contribution to the peer's polynomial
      env.send16(v, step);
    } else {  // own contribution now, the peer's when it has landed
#pragma unroll
      for (int mm = 0; mm < 8; ++mm) {
        acc[t + 64 * mm] += v[mm];
        acc[t + 64 * mm + HALF_N] += v[8 + mm];
      }
    }
    env.tick(5);
    // bookkeeping of the next step while the peer's words travel: the next active pair, and the receive barrier of
    // step + 1 (the other buffer; its previous phase ended with step - 1's data, and a transfer that completed
    // before its expect_tx would only leave the transaction count negative for a while)
    const int m_next = pair_next_active(abar, n, m + 1);
    if (tid == 0 && m_next < pairs) env.arm_recv(step + 1);
    if (!Env::helpers && m_next < pairs)
      pair_combine_keys<1>(env, abar, n, m_next, 2 * (step + 1), ft, p, grp, t, kk, kg);
    env.tick(6);
    if (grp == 0) {
      uint32_t r[16];
      env.recv16(r, step);
#pragma unroll
      for (int mm = 0; mm < 8; ++mm) {
        acc[t + 64 * mm] += r[mm];
        acc[t + 64 * mm + HALF_N] += r[8 + mm];
      }
    }
    ++step;
    env.tick(7);
    env.cta_sync();
    if (!Env::helpers && m_next < pairs) env.key_done(2 * step + 1, m_next, 1);
    env.tick(8);
    m = m_next;
  }
}

// sample extract at coefficient 0 by the main threads: the mask comes from ACC[0], the body from ACC[1]
TFB_HD void pair_extract(const uint32_t* acc, uint32_t* ext_row, int p, int tid) {
  if (p == 0) {
    for (int j = tid; j < RING_N; j += PAIR_THREADS) ext_row[j] = (j == 0) ? acc[0] : (0u - acc[RING_N - j]);
  } else if (tid == 0) {
    ext_row[RING_N] = acc[0];
  }
}

}  // namespace tfb
