// Per-thread building blocks of the B200 gate-bootstrapping kernels.
//
// Everything in this header is written as `__host__ __device__` code with the
// barrier abstracted behind a `Sync` functor, so the exact arithmetic the
// sm_100a kernels execute can also be driven by 64 host threads + a pthread
// barrier (tests/emu) on a box without a GPU.  The kernels themselves live in
// tfhe_b200.cu.
//
// Algorithm (TFHE gate bootstrapping, CGGI16/17; the reference replaces it
// with a key-holding oracle at encirc/engine.py:493-503, so there is no
// reference code to follow here -- see DESIGN.md "parity unpinned"):
//
//   gate linear form  (a', b') = cx*x + cy*y + off*mu        encirc/engine.py:483-484
//   mod switch        abar_i = round(a'_i * 2N / 2^32)
//   ACC <- (0, X^{2N-bbar} * (mu + mu X + ... + mu X^{N-1}))
//   for i < n:        ACC <- ACC + BK_i [.] ((X^{abar_i} - 1) * ACC)     (CMux)
//   sample extract    coefficient 0 of ACC -> LWE sample of dimension N
//   key switch        N -> n with signed base-4 digits
//
// The external product is evaluated with a negacyclic FP64 FFT: a polynomial
// of N = 1024 real coefficients is folded to 512 complex points, twisted by
// exp(i pi j / N) and transformed by a 512-point complex FFT done as three
// radix-8 passes, 8 points per thread, 64 threads per polynomial, with two
// shared-memory exchanges per transform.  With Bg = 2^10, l = 2 the exact
// integer result is below 2^52 and the observed FFT error is ~0.01 (std) on a
// rounding threshold of 0.5, so the rounded result equals the exact integer
// product; the parity tests hold the kernel to bit-exact agreement with the
// integer oracle.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define TFB_HD __host__ __device__ __forceinline__
#else
#define TFB_HD inline
#endif

namespace tfb {

// ---- fixed ring-side parameter set (checked at tfb_ctx_create) -------------
constexpr int RING_N = 1024;          // TRLWE degree
constexpr int HALF_N = RING_N / 2;    // complex points per transform
constexpr int BK_L = 2;               // gadget length
constexpr int BK_BGBIT = 10;          // log2 gadget base
constexpr int BK_ROWS = 2 * BK_L;     // (k+1)*l TRLWE rows per TRGSW
constexpr int KS_T = 8;               // key-switch digits
constexpr int KS_BASEBIT = 2;         // log2 key-switch base
constexpr int FFT_THREADS = 64;       // threads per polynomial transform
constexpr int ROW_STRIDE = 512;       // int32 words per pool row (n+1 <= 512)
constexpr int EXT_STRIDE = RING_N + 8;  // words per extracted sample (N+1, padded)

constexpr uint32_t DECOMP_OFFSET =
    (uint32_t(1) << 31) + (uint32_t(1) << (31 - BK_BGBIT));  // sum_l Bg/2 * 2^(32-(l+1)*bgbit)

struct alignas(16) cd {
  double re, im;
};

TFB_HD cd cmul(cd a, cd b) { return cd{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
TFB_HD cd cmulc(cd a, cd b) {  // a * conj(b)
  return cd{a.re * b.re + a.im * b.im, a.im * b.re - a.re * b.im};
}
TFB_HD cd cadd(cd a, cd b) { return cd{a.re + b.re, a.im + b.im}; }
TFB_HD cd csub(cd a, cd b) { return cd{a.re - b.re, a.im - b.im}; }
TFB_HD void cmac(cd& acc, cd a, cd b) {  // four chained FMAs (written as a sum it compiles to 2 MUL/FMA + 2 FMA + 2 ADD)
  acc.re = fma(-a.im, b.im, fma(a.re, b.re, acc.re));
  acc.im = fma(a.im, b.re, fma(a.re, b.im, acc.im));
}

TFB_HD double bits_to_double(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
TFB_HD uint64_t double_to_bits(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

// 10-bit unsigned digit field -> exact double of the signed digit field-512.
// (2^52 + field) has `field` in its low mantissa bits; one subtraction undoes
// the bias.  Avoids the slow I2F.F64 conversion pipe.
TFB_HD double digit_to_double(uint32_t field) {
  return bits_to_double(0x4330000000000000ull | (uint64_t)field) - (4503599627370496.0 + 512.0);
}
// int32 (as uint32 bit pattern) -> exact double
TFB_HD double int32_to_double(uint32_t v) {
  return bits_to_double(0x4330000000000000ull | (uint64_t)(v ^ 0x80000000u)) -
         (4503599627370496.0 + 2147483648.0);
}
// round-to-nearest-even(x) mod 2^32, valid for |x| < 2^51
TFB_HD uint32_t round_to_word(double x) {
  return (uint32_t)double_to_bits(x + 6755399441055744.0);
}

// ---- 8-point DFT in registers ----------------------------------------------
// X[k] = sum_m x[m] * exp(SIGN * 2 pi i m k / 8), natural order in and out.
template <int SIGN>
TFB_HD cd mul_i(cd a) {  // a * (SIGN * i)
  return SIGN > 0 ? cd{-a.im, a.re} : cd{a.im, -a.re};
}

template <int SIGN>
TFB_HD void dft8(cd* x) {
  const double h = 0.70710678118654752440;
  cd a0 = cadd(x[0], x[4]), a1 = cadd(x[1], x[5]), a2 = cadd(x[2], x[6]), a3 = cadd(x[3], x[7]);
  cd b0 = csub(x[0], x[4]), b1 = csub(x[1], x[5]), b2 = csub(x[2], x[6]), b3 = csub(x[3], x[7]);
  // b_m *= W8^(SIGN*m)
  {
    cd t = b1;  // (1 + SIGN i)/sqrt2
    b1 = SIGN > 0 ? cd{(t.re - t.im) * h, (t.re + t.im) * h} : cd{(t.re + t.im) * h, (t.im - t.re) * h};
    b2 = mul_i<SIGN>(b2);
    t = b3;  // (-1 + SIGN i)/sqrt2
    b3 = SIGN > 0 ? cd{(-t.re - t.im) * h, (t.re - t.im) * h} : cd{(t.im - t.re) * h, (-t.re - t.im) * h};
  }
  // two 4-point DFTs
  cd c0 = cadd(a0, a2), c1 = cadd(a1, a3), d0 = csub(a0, a2), d1 = mul_i<SIGN>(csub(a1, a3));
  x[0] = cadd(c0, c1);
  x[4] = csub(c0, c1);
  x[2] = cadd(d0, d1);
  x[6] = csub(d0, d1);
  c0 = cadd(b0, b2), c1 = cadd(b1, b3), d0 = csub(b0, b2), d1 = mul_i<SIGN>(csub(b1, b3));
  x[1] = cadd(c0, c1);
  x[5] = csub(c0, c1);
  x[3] = cadd(d0, d1);
  x[7] = csub(d0, d1);
}

// ---- twiddle tables ----------------------------------------------------------
// tw1[k][t]   = exp(i pi t (1 + 4k) / 1024)   (pass-1 twiddle W512^{t k} with the
//               per-thread part exp(i pi t / N) of the negacyclic twist folded in)
// tw2[k][a]   = exp(2 pi i a k / 64)          (pass-2 twiddle)
// Both are stored [register index][thread] so a warp reads consecutive words.
// g[t] = exp(2 pi i t / 512): ratio tw1[k+1][t] / tw1[k][t].  The paired transforms load only
// tw1[0][t], g[t] and tw2[1][lo] and rebuild the other twiddles by repeated multiplication:
// the kernel is bound by the shared-memory data pipe, not by FP64, so 13 complex
// multiplications are cheaper than 13 16-byte loads per pass pair.
struct Twiddles {
  cd tw1[8][FFT_THREADS];
  cd tw2[8][8];
  cd g[FFT_THREADS];
};

// exp(i pi m / 16): the exp(i pi 64 m / N) part of the negacyclic twist, which
// depends only on the register index m and is therefore a compile-time constant.
TFB_HD cd fold_twist(int m) {
  const double C[9] = {1.0, 0.9807852804032304, 0.9238795325112867, 0.8314696123025452,
                       0.7071067811865476, 0.5555702330196022, 0.3826834323650898, 0.19509032201612828,
                       0.0};
  return cd{C[m], C[8 - m]};  // (cos, sin)(pi m / 16)
}

// Spectral index held by (thread t, register k2) after a forward transform.
TFB_HD int spectral_index(int t, int k2) { return (t >> 3) + 8 * (t & 7) + 64 * k2; }

// Twiddle providers for the single transforms: the table in (shared or global) memory, or a
// per-thread copy held in registers for the whole kernel (the latency kernel K1c has the
// registers to spare and is limited by shared-memory traffic).
struct TableTw {
  const Twiddles* tw;
  int t;
  TFB_HD cd w1(int k) const { return tw->tw1[k][t]; }
  TFB_HD cd w2(int k) const { return tw->tw2[k][t & 7]; }
};
struct RegTw {
  cd a[8], b[8];
  TFB_HD void load(const Twiddles* tw, int t) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a[k] = tw->tw1[k][t];
      b[k] = tw->tw2[k][t & 7];
    }
  }
  TFB_HD cd w1(int k) const { return a[k]; }
  TFB_HD cd w2(int k) const { return b[k]; }
};

// Forward negacyclic transform, unnormalised.
//   in : x[m] = c_{t+64m} = a_{t+64m} + i a_{t+64m+512}   (untwisted)
//   out: x[k2] = Z[spectral_index(t, k2)],
//        Z_k = sum_j c_j exp(i pi j / N) exp(2 pi i j k / 512)
// bufA/bufB: 512 cd each in shared memory.
template <class Sync, class Tw>
TFB_HD void fft_forward(cd* x, int t, const Tw& tw, cd* bufA, cd* bufB, Sync& sync) {
#pragma unroll
  for (int m = 1; m < 8; ++m) x[m] = cmul(x[m], fold_twist(m));
  dft8<1>(x);
#pragma unroll
  for (int k = 0; k < 8; ++k) bufA[64 * k + t] = cmul(x[k], tw.w1(k));
  sync();
  const int hi = t >> 3, lo = t & 7;
#pragma unroll
  for (int j1 = 0; j1 < 8; ++j1) x[j1] = bufA[64 * hi + 8 * j1 + lo];
  dft8<1>(x);
  bufB[64 * hi + lo] = x[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) bufB[64 * hi + 8 * k + (lo ^ k)] = cmul(x[k], tw.w2(k));
  sync();
#pragma unroll
  for (int j0 = 0; j0 < 8; ++j0) x[j0] = bufB[64 * hi + 8 * lo + (j0 ^ lo)];
  dft8<1>(x);
}

// Inverse of fft_forward up to the factor 512 (folded into the key).
//   in : x[k2] = S[spectral_index(t, k2)]
//   out: x[m]  = c_{t+64m}  (re -> coefficient t+64m, im -> coefficient t+64m+512)
template <class Sync, class Tw>
TFB_HD void fft_inverse(cd* x, int t, const Tw& tw, cd* bufA, cd* bufB, Sync& sync) {
  const int hi = t >> 3, lo = t & 7;
  dft8<-1>(x);
  bufA[64 * hi + 8 * lo + lo] = x[0];
#pragma unroll
  for (int j0 = 1; j0 < 8; ++j0) bufA[64 * hi + 8 * lo + (j0 ^ lo)] = cmulc(x[j0], tw.w2(j0));
  sync();
#pragma unroll
  for (int k1 = 0; k1 < 8; ++k1) x[k1] = bufA[64 * hi + 8 * k1 + (lo ^ k1)];
  dft8<-1>(x);
#pragma unroll
  for (int j1 = 0; j1 < 8; ++j1) bufB[64 * hi + 8 * j1 + lo] = x[j1];
  sync();
#pragma unroll
  for (int k0 = 0; k0 < 8; ++k0) x[k0] = cmulc(bufB[64 * k0 + t], tw.w1(k0));
  dft8<-1>(x);
#pragma unroll
  for (int m = 1; m < 8; ++m) x[m] = cmulc(x[m], fold_twist(m));
}

// ---- paired transforms --------------------------------------------------------
// Two independent transforms advanced in lock step by the same 64 threads: every
// twiddle is loaded once and used twice and each thread carries twice the
// independent FP64 work between barriers.  s0/s1 are the exchange buffers of the
// two transforms (512 cd each).
//
// In-place exchanges.  Every exchange is a permutation of the 512 slots (each slot
// is read by exactly one thread), and a thread always writes its 8 new values into
// the 8 slots it read last.  No write can then race with another thread's read, so
// only the read-after-write barrier of each exchange remains: 2 per transform pair.
// With slot(a,b,c) = 64a + 8b + (a^b^c) the layouts of consecutive transforms are
// digit rotations of one another; a CMux runs forward (PHASE 0), forward (PHASE 1),
// inverse (PHASE 2) and the barrier that ends the CMux closes the cycle.  The XOR
// term makes every access conflict-free: across the 8 threads of a quarter warp
// exactly one digit varies.
TFB_HD int xslot(int a, int b, int c) { return 64 * a + 8 * b + (a ^ b ^ c); }

template <int PHASE, class Sync>
TFB_HD void fft_forward2(cd* x0, cd* x1, int t, const Twiddles* tw, cd* s0, cd* s1, Sync& sync) {
  static_assert(PHASE == 0 || PHASE == 1, "forward transforms are the first two of a CMux");
  const int hi = t >> 3, lo = t & 7;
#pragma unroll
  for (int m = 1; m < 8; ++m) {
    x0[m] = cmul(x0[m], fold_twist(m));
    x1[m] = cmul(x1[m], fold_twist(m));
  }
  dft8<1>(x0);
  dft8<1>(x1);
  {
    cd w = tw->tw1[0][t];
    const cd g = tw->g[t];
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // value k of thread (hi, lo)
      const int a = PHASE == 0 ? xslot(hi, lo, k) : xslot(lo, k, hi);
      s0[a] = cmul(x0[k], w);
      s1[a] = cmul(x1[k], w);
      if (k < 7) w = cmul(w, g);
    }
  }
  sync();
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // input j1 = j: value hi of thread (j, lo); pass-2 output j goes back to the same slot
    const int a = PHASE == 0 ? xslot(j, lo, hi) : xslot(lo, hi, j);
    x0[j] = s0[a];
    x1[j] = s1[a];
  }
  dft8<1>(x0);
  dft8<1>(x1);
  {
    const cd v = tw->tw2[1][lo];
    cd w = v;
    const int a0 = PHASE == 0 ? xslot(0, lo, hi) : xslot(lo, hi, 0);
    s0[a0] = x0[0];
    s1[a0] = x1[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
      const int a = PHASE == 0 ? xslot(k, lo, hi) : xslot(lo, hi, k);
      s0[a] = cmul(x0[k], w);
      s1[a] = cmul(x1[k], w);
      if (k < 7) w = cmul(w, v);
    }
  }
  sync();
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // input j0 = j: value lo of thread (hi, j)
    const int a = PHASE == 0 ? xslot(lo, j, hi) : xslot(j, hi, lo);
    x0[j] = s0[a];
    x1[j] = s1[a];
  }
  dft8<1>(x0);
  dft8<1>(x1);
}

// Inverse pair, PHASE 2: its first writes land in the slots the PHASE 1 forward read last.
template <class Sync>
TFB_HD void fft_inverse2(cd* x0, cd* x1, int t, const Twiddles* tw, cd* s0, cd* s1, Sync& sync) {
  const int hi = t >> 3, lo = t & 7;
  dft8<-1>(x0);
  dft8<-1>(x1);
  {
    const cd v = tw->tw2[1][lo];
    cd w = v;
    const int a0 = xslot(0, hi, lo);
    s0[a0] = x0[0];
    s1[a0] = x1[0];
#pragma unroll
    for (int j0 = 1; j0 < 8; ++j0) {  // value j0 of thread (k0, k1) = (hi, lo)
      const int a = xslot(j0, hi, lo);
      s0[a] = cmulc(x0[j0], w);
      s1[a] = cmulc(x1[j0], w);
      if (j0 < 7) w = cmul(w, v);
    }
  }
  sync();
#pragma unroll
  for (int k1 = 0; k1 < 8; ++k1) {  // thread (k0, j0) = (hi, lo): value j0 = lo of thread (hi, k1)
    const int a = xslot(lo, hi, k1);
    x0[k1] = s0[a];
    x1[k1] = s1[a];
  }
  dft8<-1>(x0);
  dft8<-1>(x1);
#pragma unroll
  for (int j1 = 0; j1 < 8; ++j1) {
    const int a = xslot(lo, hi, j1);
    s0[a] = x0[j1];
    s1[a] = x1[j1];
  }
  sync();
  {
    cd w = tw->tw1[0][t];
    const cd g = tw->g[t];
#pragma unroll
    for (int k0 = 0; k0 < 8; ++k0) {  // thread (j1, j0) = (hi, lo): value j1 = hi of thread (k0, lo)
      const int a = xslot(lo, k0, hi);
      x0[k0] = cmulc(s0[a], w);
      x1[k0] = cmulc(s1[a], w);
      if (k0 < 7) w = cmul(w, g);
    }
  }
  dft8<-1>(x0);
  dft8<-1>(x1);
#pragma unroll
  for (int m = 1; m < 8; ++m) {
    x0[m] = cmulc(x0[m], fold_twist(m));
    x1[m] = cmulc(x1[m], fold_twist(m));
  }
}

// ---- rotation and gadget decomposition -----------------------------------------
// coefficient j of X^abar * P - P for P in shared memory (N words), abar in [0, 2N)
TFB_HD uint32_t rotated_diff(const uint32_t* poly, int j, int abar) {
  const int src = (j - abar) & (2 * RING_N - 1);
  const uint32_t v = poly[src & (RING_N - 1)];
  const uint32_t neg = (uint32_t)(src >> 10) & 1u;  // 1 when the wrap flips the sign
  return ((v ^ (0u - neg)) + neg) - poly[j];
}

TFB_HD uint32_t digit_field(uint32_t v_plus_offset, int lvl) {
  return (v_plus_offset >> (32 - (lvl + 1) * BK_BGBIT)) & ((1u << BK_BGBIT) - 1);
}

// ---- one CMux step -----------------------------------------------------------------
// Spectral key layout: one "stage" per (LWE index i, accumulator polynomial p),
// STAGE_CD complex values laid out [k2][lvl][c][t], prescaled by 1/512, so the
// MAC of one paired forward transform reads one contiguous 32 KB block.
constexpr int STAGE_CD = 8 * BK_L * 2 * FFT_THREADS;  // 2048 cd = 32 KB
TFB_HD size_t stage_offset(int i, int p) { return ((size_t)i * 2 + p) * STAGE_CD; }
TFB_HD int stage_index(int k2, int lvl, int c, int t) { return ((k2 * BK_L + lvl) * 2 + c) * FFT_THREADS + t; }

// A BkSource hands out the key one stage at a time:
//   const cd* acquire(i, p)   pointer to the stage (blocks until it is resident)
//   cd load(q)                one value of it
//   void release()            this thread is done with the stage
// (a skipped CMux -- abar == 0 -- still acquires and releases its stages, so that a staged pipeline's
// bookkeeping stays in step)
struct GlobalBk {  // plain pointer into the full key (host emulation, key setup checks)
  const cd* base;
  TFB_HD const cd* acquire(int i, int p) { return base + stage_offset(i, p); }
  TFB_HD const cd* acquire_chunk(int i, int p, int lvl) { return base + stage_offset(i, p) + (size_t)lvl * (STAGE_CD / 2); }
  TFB_HD cd load(const cd* q) const { return *q; }
  TFB_HD void release() {}
};

// acc: 2 polynomials of N words in shared memory ([0..N) = a, [N..2N) = b).
// Every thread of the 64-thread group calls this; `sync` is the group barrier.
// Both gadget levels of one accumulator polynomial are transformed as a pair,
// then both output polynomials are inverse-transformed as a pair.
// One accumulator polynomial p of a CMux: rotate-and-subtract, decompose, paired
// forward transform, MAC against stage (i, p).  P == 0 initialises the output
// accumulators instead of adding to them, so they are not live (64 registers)
// during the first paired transform.
// A Park policy may hold the 16 accumulator values of a thread outside the register file
// between the two halves of a CMux (the B200 kernel parks them in tensor memory):
//   store(out0, out1) after the first half, load(k2, o0, o1) inside the second half's MAC.
// A policy may also order the MAC stages of the groups that share schedulers (turn_enter / turn_leave /
// turn_pass; see TurnPark in tfhe_b200.cu).
struct NoPark {
  static constexpr bool parks = false;
  TFB_HD void store(const cd*, const cd*) {}
  TFB_HD void load(int, cd&, cd&) {}
  TFB_HD void turn_enter() const {}
  TFB_HD void turn_leave() const {}
  TFB_HD void turn_pass() const {}
};

template <int P, class Sync, class BkSource, class Park>
TFB_HD void cmux_half(cd* out0, cd* out1, const uint32_t* acc, int abar, int i, BkSource& bk, int t,
                      const Twiddles* tw, cd* s0, cd* s1, Sync& sync, Park& park) {
  cd x0[8], x1[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t vr = rotated_diff(acc + P * RING_N, t + 64 * m, abar) + DECOMP_OFFSET;
    const uint32_t vi = rotated_diff(acc + P * RING_N, t + 64 * m + HALF_N, abar) + DECOMP_OFFSET;
    x0[m] = cd{digit_to_double(digit_field(vr, 0)), digit_to_double(digit_field(vi, 0))};
    x1[m] = cd{digit_to_double(digit_field(vr, 1)), digit_to_double(digit_field(vi, 1))};
  }
  fft_forward2<P>(x0, x1, t, tw, s0, s1, sync);
  const cd* stage = bk.acquire(i, P);
  park.turn_enter();
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) {
    if (P == 0) {
      out0[k2] = cmul(x0[k2], bk.load(stage + stage_index(k2, 0, 0, t)));
      out1[k2] = cmul(x0[k2], bk.load(stage + stage_index(k2, 0, 1, t)));
    } else {
      if (Park::parks) park.load(k2, out0[k2], out1[k2]);
      cmac(out0[k2], x0[k2], bk.load(stage + stage_index(k2, 0, 0, t)));
      cmac(out1[k2], x0[k2], bk.load(stage + stage_index(k2, 0, 1, t)));
    }
    cmac(out0[k2], x1[k2], bk.load(stage + stage_index(k2, 1, 0, t)));
    cmac(out1[k2], x1[k2], bk.load(stage + stage_index(k2, 1, 1, t)));
  }
  park.turn_leave();
  bk.release();
}

// acc: 2 polynomials of N words in shared memory ([0..N) = a, [N..2N) = b).
// Every thread of the 64-thread group calls this; `sync` is the group barrier.
// Both gadget levels of one accumulator polynomial are transformed as a pair,
// then both output polynomials are inverse-transformed as a pair.
template <class Sync, class BkSource, class Park>
TFB_HD void cmux_step(uint32_t* acc, int abar, int i, BkSource& bk, int t, const Twiddles* tw, cd* s0, cd* s1,
                      Sync& sync, Park& park) {
  cd out0[8], out1[8];
  cmux_half<0>(out0, out1, acc, abar, i, bk, t, tw, s0, s1, sync, park);
  if (Park::parks) park.store(out0, out1);
  cmux_half<1>(out0, out1, acc, abar, i, bk, t, tw, s0, s1, sync, park);
  fft_inverse2(out0, out1, t, tw, s0, s1, sync);
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    acc[t + 64 * m] += round_to_word(out0[m].re);
    acc[t + 64 * m + HALF_N] += round_to_word(out0[m].im);
    acc[RING_N + t + 64 * m] += round_to_word(out1[m].re);
    acc[RING_N + t + 64 * m + HALF_N] += round_to_word(out1[m].im);
  }
  sync();
}

// ---- gate table -----------------------------------------------------------------------
// kind ids follow the reference's TWO_INPUT_KINDS order (encirc/engine.py:77-88):
// 0 AND 1 OR 2 NAND 3 NOR 4 XOR 5 XNOR 6 ANDNY 7 ORNY; 8 = identity (standalone bootstrap).
constexpr int NUM_KINDS = 9;
TFB_HD void gate_coeffs(int kind, int32_t& cx, int32_t& cy, int32_t& off) {
  // 4-bit biased nibbles (value + 8), kind 0 in the low nibble:
  //   cx  = { 1, 1,-1,-1, 2,-2,-1,-1, 1}
  //   cy  = { 1, 1,-1,-1, 2,-2, 1, 1, 0}
  //   off = {-1, 1, 1,-1, 2,-2,-1, 1, 0}
  const uint64_t CX = 0x9776A7799ull, CY = 0x8996A7799ull, OF = 0x8976A7997ull;
  cx = (int32_t)((CX >> (4 * kind)) & 15) - 8;
  cy = (int32_t)((CY >> (4 * kind)) & 15) - 8;
  off = (int32_t)((OF >> (4 * kind)) & 15) - 8;
}

// round(a * 2N / 2^32) mod 2N
TFB_HD int mod_switch(uint32_t a) { return (int)((a + (1u << 20)) >> 21) & (2 * RING_N - 1); }

// Gate linear form + mod switch + accumulator initialisation, by `nthreads` threads.
//   ACC = (0, X^{2N - bbar} * testvector), testvector = mu * (1 + X + ... + X^{N-1})
template <class Sync>
TFB_HD void bootstrap_prologue(const uint32_t* x_row, const uint32_t* y_row, int kind, int n, uint32_t mu,
                               uint32_t* sm_acc, uint16_t* sm_abar, int tid, int nthreads, Sync& sync) {
  int32_t cx, cy, off;
  gate_coeffs(kind, cx, cy, off);
  for (int w = tid; w <= n; w += nthreads) {
    uint32_t v = (uint32_t)cx * x_row[w] + (uint32_t)cy * y_row[w];
    if (w == n) v += (uint32_t)off * mu;
    sm_abar[w] = (uint16_t)mod_switch(v);
  }
  sync();
  const int bbar = sm_abar[n];
  for (int j = tid; j < RING_N; j += nthreads) {
    sm_acc[j] = 0;
    const int src = (j + bbar) & (2 * RING_N - 1);  // j - (2N - bbar) mod 2N
    sm_acc[RING_N + j] = (src < RING_N) ? mu : (0u - mu);
  }
  sync();
}

// sample extract at coefficient 0: a'_0 = a_0, a'_j = -a_{N-j}; b' = b_0
TFB_HD void bootstrap_extract(const uint32_t* sm_acc, uint32_t* ext, int tid, int nthreads) {
  for (int j = tid; j < RING_N; j += nthreads) ext[j] = (j == 0) ? sm_acc[0] : (0u - sm_acc[RING_N - j]);
  if (tid == 0) ext[RING_N] = sm_acc[RING_N];
}

// Whole gate bootstrap (without key switch) for one ciphertext by one 64-thread group.
//   x_row, y_row: pool rows (n mask words then the body)
//   sm_acc: 2N words, sm_abar: n+1 uint16, s0/s1: 512 cd each (exchange buffers)
//   ext: N+1 words out (extracted LWE sample under the ring key)
template <class Sync, class BkSource, class Park>
TFB_HD void gate_bootstrap(const uint32_t* x_row, const uint32_t* y_row, int kind, int n, uint32_t mu,
                           BkSource& bk, const Twiddles* tw, uint32_t* sm_acc, uint16_t* sm_abar,
                           cd* s0, cd* s1, uint32_t* ext, int t, Sync& sync, Park& park) {
  bootstrap_prologue(x_row, y_row, kind, n, mu, sm_acc, sm_abar, t, FFT_THREADS, sync);
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    const int abar = sm_abar[i];
    if (abar == 0) {  // uniform across the group: keep the key pipeline and the turn order in step
      for (int p = 0; p < 2; ++p) {
        bk.acquire(i, p);
        park.turn_pass();
        bk.release();
      }
      continue;
    }
    cmux_step(sm_acc, abar, i, bk, t, tw, s0, s1, sync, park);
  }
  bootstrap_extract(sm_acc, ext, t, FFT_THREADS);
}

// Latency-oriented variant: ONE ciphertext by FOUR 64-thread groups (256 threads).
// Group q = 2p + lvl transforms digit polynomial (p, lvl) on its own, multiplies it
// with its share of key stage (i, p) -- prefetched into registers before the
// transform -- and the four partial products are summed through shared memory;
// groups 0 and 1 then inverse-transform output polynomials 0 and 1.  The critical
// path per CMux is one forward + one inverse transform instead of six.
//   xbuf: 4 groups x 2 exchange buffers x 512 cd;  red: 4 groups x 2 components x 512 cd
template <class GroupSync, class CtaSync, class LoadBk>
TFB_HD void gate_bootstrap_wide(const uint32_t* x_row, const uint32_t* y_row, int kind, int n, uint32_t mu,
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
    cd x[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const uint32_t vr = rotated_diff(sm_acc + p * RING_N, t + 64 * m, abar) + DECOMP_OFFSET;
      const uint32_t vi = rotated_diff(sm_acc + p * RING_N, t + 64 * m + HALF_N, abar) + DECOMP_OFFSET;
      x[m] = cd{digit_to_double(digit_field(vr, lvl)), digit_to_double(digit_field(vi, lvl))};
    }
    fft_forward(x, t, rtw, bufA, bufB, gsync);
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      const cd p0 = cmul(x[k2], b0[k2]), p1 = cmul(x[k2], b1[k2]);
      if (q != 0) red[((q * 2 + 0) * 8 + k2) * FFT_THREADS + t] = p0;
      if (q != 1) red[((q * 2 + 1) * 8 + k2) * FFT_THREADS + t] = p1;
      x[k2] = (q == 0) ? p0 : p1;  // meaningful for q < 2: the product this group keeps
    }
    csync();
    if (q < 2) {  // output polynomial c = q
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        cd s = x[k2];
#pragma unroll
        for (int o = 0; o < 4; ++o)
          if (o != q) s = cadd(s, red[((o * 2 + q) * 8 + k2) * FFT_THREADS + t]);
        x[k2] = s;
      }
      fft_inverse(x, t, rtw, bufA, bufB, gsync);
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        sm_acc[q * RING_N + t + 64 * m] += round_to_word(x[m].re);
        sm_acc[q * RING_N + t + 64 * m + HALF_N] += round_to_word(x[m].im);
      }
    }
    csync();
  }
  bootstrap_extract(sm_acc, ext, tid, WIDE);
}

// ---- key switch ---------------------------------------------------------------------------
// signed base-4 digits d_j in {-2,-1,0,1} of a (top KS_T*KS_BASEBIT bits, rounded):
//   a ~= sum_j d_j * 2^(32 - (j+1)*KS_BASEBIT)
constexpr uint32_t KS_ROUND = 1u << (32 - KS_T * KS_BASEBIT - 1);
TFB_HD uint32_t ks_bias() {
  uint32_t b = KS_ROUND;
  for (int j = 0; j < KS_T; ++j) b += (uint32_t)(1u << (KS_BASEBIT - 1)) << (32 - (j + 1) * KS_BASEBIT);
  return b;
}
TFB_HD int32_t ks_digit(uint32_t a_biased, int j) {
  return (int32_t)((a_biased >> (32 - (j + 1) * KS_BASEBIT)) & ((1u << KS_BASEBIT) - 1)) -
         (1 << (KS_BASEBIT - 1));
}

}  // namespace tfb
