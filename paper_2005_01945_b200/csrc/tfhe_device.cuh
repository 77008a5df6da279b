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
//   for pairs (i, i+1) of mask elements, with the bootstrapping key UNROLLED (three TRGSW samples
//   s_i, s_i+1, s_i s_i+1 per pair; Zhou et al. 2018, Bourse et al. 2018) and u = X^{abar} - 1:
//                     ACC <- ACC + u1 (BK1 [.] ACC) + u2 (BK2 [.] ACC) + u1 u2 (BK12 [.] ACC)
//                     one gadget decomposition of ACC and four forward transforms serve the three
//                     external products; the factors u are applied in the spectral domain
//                     (X^e at spectral point f is exp(i pi e (1 + 4 f) / N)); two inverse transforms
//   sample extract    coefficient 0 of ACC -> LWE sample of dimension N
//   key switch        N -> n with signed base-4 digits
//
// The external product is evaluated with a negacyclic FP64 FFT: a polynomial
// of N = 1024 real coefficients is folded to 512 complex points, twisted by
// exp(i pi j / N) and transformed by a 512-point complex FFT done as three
// radix-8 passes, 8 points per thread, 64 threads per polynomial, with two
// shared-memory exchanges per transform.  With Bg = 2^9, l = 2 and three keys with factors
// |u| <= 2, |u1 u2| <= 4 the exact integer result stays below 2^53 in the worst case and around
// 2^45 (rms) in practice; the observed FFT error is ~0.01 (std) on a rounding threshold of 0.5,
// so the rounded result equals the exact integer product; the parity tests hold the kernels to
// bit-exact agreement with the integer oracle.
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
constexpr int BK_BGBIT = 9;           // log2 gadget base
constexpr int BK_ROWS = 2 * BK_L;     // (k+1)*l TRLWE rows per TRGSW
constexpr int BK_KEYS = 3;            // TRGSW samples per pair of mask elements: s1, s2, s1 s2
constexpr int KS_T = 8;               // key-switch digits
constexpr int KS_BASEBIT = 2;         // log2 key-switch base
constexpr int FFT_THREADS = 64;       // threads per polynomial transform
constexpr int ROW_STRIDE = 512;       // int32 words per pool row (n+1 <= 512)
constexpr int EXT_STRIDE = RING_N + 8;  // words per extracted sample (N+1, padded)

// sum_l Bg/2 * 2^(32-(l+1)*bgbit), plus half an ulp of the last digit: round, do not truncate
constexpr uint32_t DECOMP_OFFSET = (uint32_t(1) << 31) + (uint32_t(1) << (31 - BK_BGBIT)) +
                                   (uint32_t(1) << (32 - BK_L * BK_BGBIT - 1));
constexpr int DIGIT_HALF = 1 << (BK_BGBIT - 1);

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

// unsigned digit field -> exact double of the signed digit field - Bg/2.
// (2^52 + field) has `field` in its low mantissa bits; one subtraction undoes
// the bias.  Avoids the slow I2F.F64 conversion pipe.
TFB_HD double digit_to_double(uint32_t field) {
  return bits_to_double(0x4330000000000000ull | (uint64_t)field) - (4503599627370496.0 + (double)DIGIT_HALF);
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

// ---- gadget decomposition ------------------------------------------------------------------
TFB_HD uint32_t digit_field(uint32_t v_plus_offset, int lvl) {
  return (v_plus_offset >> (32 - (lvl + 1) * BK_BGBIT)) & ((1u << BK_BGBIT) - 1);
}

// ---- spectral rotation factors ---------------------------------------------------------------
// X^e evaluated at spectral point f (Z_f = P(exp(i pi (1 + 4 f) / N)), see fft_forward) is
// exp(i pi m / N) with m = e (1 + 4 f) mod 2N.  A two-level table gives any of the 2N roots with one
// complex multiplication: m = 32 hi + lo, root = A[hi] * B[lo].  The spectral points a thread owns
// differ by multiples of 32 or 64 in f, i.e. by A-entries only: base = root(e * (1 + 4 f0)) per
// (thread, e) and one multiplication by A[..] per point.
struct FactorTables {
  cd A[64];  // exp(i pi hi / 32)
  cd B[32];  // exp(i pi lo / 1024)
};
template <class Real>
inline void fill_factor_tables(FactorTables* ft, Real (*cosf_)(Real), Real (*sinf_)(Real)) {
  const Real pi = (Real)3.141592653589793238462643383279502884L;
  for (int h = 0; h < 64; ++h) ft->A[h] = cd{(double)cosf_(pi * (Real)h / (Real)32), (double)sinf_(pi * (Real)h / (Real)32)};
  for (int l = 0; l < 32; ++l)
    ft->B[l] = cd{(double)cosf_(pi * (Real)l / (Real)RING_N), (double)sinf_(pi * (Real)l / (Real)RING_N)};
  // exact values where they are exact, so that e = 0 gives u = 0 without rounding residue
  ft->A[0] = cd{1.0, 0.0};
  ft->A[16] = cd{0.0, 1.0};
  ft->A[32] = cd{-1.0, 0.0};
  ft->A[48] = cd{0.0, -1.0};
  ft->B[0] = cd{1.0, 0.0};
}
// exp(i pi m / N), any integer m
TFB_HD cd unit_root(const FactorTables* ft, uint32_t m) { return cmul(ft->A[(m >> 5) & 63], ft->B[m & 31]); }

// u = base * a - 1 (the factor X^e - 1 at a spectral point, from the lane's base root and a table entry): the -1 rides in
// the first FMA, four instructions instead of a complex multiplication plus a subtraction
TFB_HD cd rotation_minus_one(cd base, cd a) {
  return cd{fma(-base.im, a.im, fma(base.re, a.re, -1.0)), fma(base.re, a.im, base.im * a.re)};
}

// Combined key of one spectral point:  K = u1 B1 + u2 B2 + u1 u2 B12 = u1 (B1 + u2 B12) + u2 B2   (12 FMA-class)
TFB_HD cd combine_keys(cd u1, cd u2, cd b1, cd b2, cd b12) {
  cd t = b1;
  cmac(t, u2, b12);
  cd k = cmul(u2, b2);
  cmac(k, u1, t);
  return k;
}

// ---- 64-thread spectral key layout (K1e) -------------------------------------------------------
// One CHUNK per (pair m, accumulator polynomial p, gadget level lvl, half h of the 8 points a thread
// owns): [k4][key j][c][t], 4 x 3 x 2 x 64 complex = 24 KB, prescaled by 1/512 -- what one 64-thread
// group consumes in half of its product phase, and the unit its key ring moves.
constexpr int PCHUNK_CD = 4 * BK_KEYS * 2 * FFT_THREADS;  // 1536 cd = 24 KB
TFB_HD size_t pchunk_offset(int m, int p, int lvl, int h) { return ((((size_t)m * 2 + p) * BK_L + lvl) * 2 + h) * PCHUNK_CD; }
TFB_HD int pchunk_index(int k4, int j, int c, int t) { return ((k4 * BK_KEYS + j) * 2 + c) * FFT_THREADS + t; }
TFB_HD size_t bkf_total_cd(int n) { return (size_t)((n + 1) / 2) * BK_KEYS * BK_ROWS * 2 * HALF_N; }

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

// Where coefficient j of an accumulator polynomial sits inside its N-word block of shared memory.
// The unrolled CMux never rotates the accumulator in the coefficient domain (the rotation is a spectral
// factor), so a kernel may keep each thread's coefficients wherever its own loads are cheapest.
struct NaturalLayout {
  TFB_HD int operator()(int j) const { return j; }
};

// Gate linear form + mod switch, by `nthreads` threads: abar[0..n) rotations, abar[n] = body,
// abar[n+1] = 0 (the padding element of an odd n).
TFB_HD void gate_mod_switch(const uint32_t* x_row, const uint32_t* y_row, int kind, int n, uint32_t mu,
                            uint16_t* sm_abar, int tid, int nthreads) {
  int32_t cx, cy, off;
  gate_coeffs(kind, cx, cy, off);
  for (int w = tid; w <= n; w += nthreads) {
    uint32_t v = (uint32_t)cx * x_row[w] + (uint32_t)cy * y_row[w];
    if (w == n) v += (uint32_t)off * mu;
    sm_abar[w] = (uint16_t)mod_switch(v);
  }
  if (tid == 0) sm_abar[n + 1] = 0;
}
// rotations of pair m (the second one is 0 past the end of an odd n: sm_abar[n] is the body)
TFB_HD void pair_rotations(const uint16_t* sm_abar, int n, int m, int& a1, int& a2) {
  a1 = sm_abar[2 * m];
  a2 = (2 * m + 1 < n) ? sm_abar[2 * m + 1] : 0;
}
// the body's rotation alone (what a gate on two trivial inputs needs: its mask rotations are all zero)
TFB_HD int gate_body_rotation_of(const uint32_t* x_row, const uint32_t* y_row, int kind, int n, uint32_t mu) {
  int32_t cx, cy, off;
  gate_coeffs(kind, cx, cy, off);
  return mod_switch((uint32_t)cx * x_row[n] + (uint32_t)cy * y_row[n] + (uint32_t)off * mu);
}
// coefficient j of X^{2N - bbar} * mu (1 + X + ... + X^{N-1})
TFB_HD uint32_t test_vector_coeff(int j, int bbar, uint32_t mu) {
  const int src = (j + bbar) & (2 * RING_N - 1);  // j - (2N - bbar) mod 2N
  return (src < RING_N) ? mu : (0u - mu);
}

// Gate linear form + mod switch + accumulator initialisation, by `nthreads` threads.
//   ACC = (0, X^{2N - bbar} * testvector), testvector = mu * (1 + X + ... + X^{N-1})
template <class Sync, class Layout>
TFB_HD void bootstrap_prologue(const uint32_t* x_row, const uint32_t* y_row, int kind, int n, uint32_t mu,
                               uint32_t* sm_acc, uint16_t* sm_abar, int tid, int nthreads, Sync& sync, Layout slot) {
  gate_mod_switch(x_row, y_row, kind, n, mu, sm_abar, tid, nthreads);
  sync();
  const int bbar = sm_abar[n];
  for (int j = tid; j < RING_N; j += nthreads) {
    sm_acc[slot(j)] = 0;
    sm_acc[RING_N + slot(j)] = test_vector_coeff(j, bbar, mu);
  }
  sync();
}

// sample extract at coefficient 0: a'_0 = a_0, a'_j = -a_{N-j}; b' = b_0
template <class Layout>
TFB_HD void bootstrap_extract(const uint32_t* sm_acc, uint32_t* ext, int tid, int nthreads, Layout slot) {
  for (int j = tid; j < RING_N; j += nthreads) ext[j] = (j == 0) ? sm_acc[slot(0)] : (0u - sm_acc[slot(RING_N - j)]);
  if (tid == 0) ext[RING_N] = sm_acc[RING_N + slot(0)];
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
