// K1d building blocks: ONE ciphertext per WARP.
//
// The 64-thread kernels of tfhe_device.cuh move every transform through shared memory twice
// (three radix-8 passes) and are bound by the shared-memory data pipe, not by FP64 (DESIGN.md
// section 11).  Here a 32-lane warp owns a whole ciphertext and every lane carries 16 points:
//   512 = 16 (registers) x 16 (registers, after ONE shared-memory exchange) x 2 (lane ^ 16, by
//   warp shuffle), so a transform costs 128 + 32 instead of 256 shared-memory wavefronts per
// ciphertext, there is no inter-warp barrier anywhere in the blind rotation (only __syncwarp),
// and eight independent warps per SM hide each other's latencies.
//
// Same arithmetic contract as tfhe_device.cuh (exact integer result after rounding), same
// `__host__ __device__` discipline: tests/emu drives this code with 32 host threads per warp.
#pragma once
#include "tfhe_device.cuh"

#if defined(__CUDA_ARCH__)
#define TFB_OPAQUE(v) asm volatile("" : "+r"(v))
#else
#define TFB_OPAQUE(v) (void)(v)
#endif

// The four forward and the two inverse transforms of a CMux as rolled loops (one copy of the
// transform code: smaller instruction footprint, no scheduling across the stages) or unrolled.
#ifndef TFB_K1D_ROLL
#define TFB_K1D_ROLL 1
#endif
#if TFB_K1D_ROLL
#define TFB_K1D_LOOP _Pragma("unroll 1")
#else
#define TFB_K1D_LOOP _Pragma("unroll")
#endif

#ifdef TFB_K1D_PHASES  // per-phase clock probe (a profiling build): W::tick(k) accumulates cycles since the last tick
#define TFB_TICK(w, k) (w).tick(k)
#else
#define TFB_TICK(w, k)
#endif

namespace tfb {

constexpr int WARP_T = 32;  // lanes per ciphertext
// Turn protocol (W::turn_enter / turn_leave / turn_pass): the warps that share a scheduler take the MAC
// stage of a CMux in a fixed rotation, which keeps them a third of a stage apart (see DevWarp in
// tfhe_b200.cu for why).  Measured placements are listed in profiles/README.md.
constexpr int WPTS = 16;    // points per lane

// Per-lane twiddles (t = lane, r = t & 15, h = t >> 4).  Lane h = 1 keeps its pass-1 outputs
// rotated by 8 (register k holds frequency k ^ 8, see wfft_forward), so every lane runs two
// chains of 8 pass-1 twiddles W512^{t k1} exp(i pi t / N) = exp(i pi t (1 + 4 k1) / 1024):
//   sa[t] = the one of k1 = 8h       (registers 0..7,  then times g, g^2, ...)
//   sb[t] = the one of k1 = 8(1-h)   (registers 8..15)
//   g[t]  = exp(2 pi i t / 512)      ratio of consecutive twiddles
//   c[t]  = (-1)^h exp(2 pi i r / 32)   twiddle of the odd half of the cross-lane radix-2 stage
struct WarpTwiddles {
  cd sa[WARP_T];
  cd sb[WARP_T];
  cd g[WARP_T];
  cd c[WARP_T];
};

template <class Real>
inline void fill_warp_twiddles(WarpTwiddles* tw, Real (*cosf_)(Real), Real (*sinf_)(Real)) {
  const Real pi = (Real)3.141592653589793238462643383279502884L;
  for (int t = 0; t < WARP_T; ++t) {
    const int r = t & 15, h = t >> 4;
    const Real aa = pi * (Real)(t * (1 + 32 * h)) / (Real)RING_N;
    const Real ab = pi * (Real)(t * (1 + 32 * (1 - h))) / (Real)RING_N;
    const Real ag = (Real)2 * pi * (Real)t / (Real)HALF_N;
    const Real ac = (Real)2 * pi * (Real)r / (Real)32;
    tw->sa[t] = cd{(double)cosf_(aa), (double)sinf_(aa)};
    tw->sb[t] = cd{(double)cosf_(ab), (double)sinf_(ab)};
    tw->g[t] = cd{(double)cosf_(ag), (double)sinf_(ag)};
    tw->c[t] = cd{(double)(h ? -cosf_(ac) : cosf_(ac)), (double)(h ? -sinf_(ac) : sinf_(ac))};
  }
}

// cos(pi m / 32), m in [0, 16]: every compile-time twiddle of the 16-point transforms is a point of this
// first quadrant up to symmetry.  On the device the table sits in the constant bank, so that FP64
// instructions take these factors as c[][] operands (sign flips ride in the operand modifiers): as
// literals the compiler hoists them out of the blind-rotation loop into ~70 registers and spills them.
#define TFB_TWIST16_VALUES                                                                                   \
  {1.0, 0.9951847266721969, 0.9807852804032304, 0.9569403357322088, 0.9238795325112867, 0.881921264348355,  \
   0.8314696123025452, 0.773010453362737, 0.7071067811865476, 0.6343932841636455, 0.5555702330196023,       \
   0.4713967368259978, 0.3826834323650898, 0.2902846772544623, 0.1950903220161283, 0.0980171403295608, 0.0}
#if defined(__CUDACC__)
__constant__ double kTwist16Dev[17] = TFB_TWIST16_VALUES;
#endif
TFB_HD double quadrant_cos(int m) {  // cos(pi m / 32), 0 <= m <= 16
#if defined(__CUDA_ARCH__)
  return kTwist16Dev[m];
#else
  const double C[17] = TFB_TWIST16_VALUES;
  return C[m];
#endif
}
TFB_HD double cospi32(int j) {  // cos(pi j / 32), any integer j (a compile-time constant after unrolling)
  j &= 63;
  if (j > 32) j = 64 - j;
  return j <= 16 ? quadrant_cos(j) : -quadrant_cos(32 - j);
}
TFB_HD cd expi32(int j) { return cd{cospi32(j), cospi32(j - 16)}; }  // exp(i pi j / 32)
TFB_HD cd twist16(int m) { return expi32(m); }                       // register part of the negacyclic twist

// ---- 16-point DFTs in registers, FMA form -------------------------------------------------------
// K1d is limited by the FP64 pipe together with latency, so every twiddle multiplication that feeds a
// butterfly is folded into it:  (a + w b, a - w b)  costs six FMA-class instructions (four for the sum,
// then a - w b = 2 a - (a + w b)) instead of a complex multiplication plus two complex additions (eight).
TFB_HD void bfly(cd a, cd b, cd w, cd& p, cd& m) {  // p = a + w b, m = a - w b
  p.re = fma(-w.im, b.im, fma(w.re, b.re, a.re));
  p.im = fma(w.im, b.re, fma(w.re, b.im, a.im));
  m.re = fma(2.0, a.re, -p.re);
  m.im = fma(2.0, a.im, -p.im);
}
template <int SIGN>
TFB_HD void dft4(cd& z0, cd& z1, cd& z2, cd& z3) {  // y_k = sum_j z_j i^(SIGN j k), in place
  const cd t0 = cadd(z0, z2), t1 = csub(z0, z2), t2 = cadd(z1, z3), t3 = mul_i<SIGN>(csub(z1, z3));
  z0 = cadd(t0, t2);
  z1 = cadd(t1, t3);
  z2 = csub(t0, t2);
  z3 = csub(t1, t3);
}
// the same on (z0, w1 z1, w2 z2, w3 z3): 24 instructions instead of 12 + 16.  W2I: w2 = i^SIGN (free).
template <int SIGN, bool W2I = false>
TFB_HD void dft4_tw(cd& z0, cd& z1, cd& z2, cd& z3, cd w1, cd w2, cd w3) {
  cd t0, t1, t2, t3;
  if (W2I) {
    const cd v = mul_i<SIGN>(z2);
    t0 = cadd(z0, v);
    t1 = csub(z0, v);
  } else {
    bfly(z0, z2, w2, t0, t1);
  }
  bfly(cmul(z1, w1), z3, w3, t2, t3);
  t3 = mul_i<SIGN>(t3);
  z0 = cadd(t0, t2);
  z1 = cadd(t1, t3);
  z2 = csub(t0, t2);
  z3 = csub(t1, t3);
}
// ... and with a twiddle on z0 as well (28 instructions)
template <int SIGN>
TFB_HD void dft4_tw4(cd& z0, cd& z1, cd& z2, cd& z3, cd w0, cd w1, cd w2, cd w3) {
  cd t0, t1, t2, t3;
  bfly(cmul(z0, w0), z2, w2, t0, t1);
  bfly(cmul(z1, w1), z3, w3, t2, t3);
  t3 = mul_i<SIGN>(t3);
  z0 = cadd(t0, t2);
  z1 = cadd(t1, t3);
  z2 = csub(t0, t2);
  z3 = csub(t1, t3);
}

TFB_HD void transpose4x4(cd* x) {  // x[i + 4 j] <-> x[j + 4 i]: register renaming
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = i + 1; j < 4; ++j) {
      const cd tmp = x[i + 4 * j];
      x[i + 4 * j] = x[j + 4 * i];
      x[j + 4 * i] = tmp;
    }
}

// second radix-4 layer of a 16-point DFT with the mid twiddles w16^(SIGN a k0) folded in
// (in: x[a + 4 k0] = y_a[k0]; out: x[4 k0 + k1] = X[k0 + 4 k1]), 86 instead of 96 instructions
template <int SIGN>
TFB_HD void dft16_layer_b(cd* x) {
  dft4<SIGN>(x[0], x[1], x[2], x[3]);
  dft4_tw<SIGN>(x[4], x[5], x[6], x[7], expi32(SIGN * 4), expi32(SIGN * 8), expi32(SIGN * 12));
  dft4_tw<SIGN, true>(x[8], x[9], x[10], x[11], expi32(SIGN * 8), expi32(SIGN * 16), expi32(SIGN * 24));
  dft4_tw<SIGN>(x[12], x[13], x[14], x[15], expi32(SIGN * 12), expi32(SIGN * 24), expi32(SIGN * 36));
}

// X[k] = sum_m x[m] exp(SIGN 2 pi i m k / 16), natural order in and out
template <int SIGN>
TFB_HD void dft16(cd* x) {
#pragma unroll
  for (int a = 0; a < 4; ++a) dft4<SIGN>(x[a], x[a + 4], x[a + 8], x[a + 12]);
  dft16_layer_b<SIGN>(x);
  transpose4x4(x);
}

// X[k] = sum_m (x[m] exp(i pi m / 32)) exp(2 pi i m k / 16): the register part of the negacyclic twist folded
// into both radix-4 layers (inner twists exp(i pi 4 b / 32) on the inputs of layer A, exp(i pi a (1 + 4 k0) / 32)
// on those of layer B): 192 instead of 60 + 160 instructions
TFB_HD void dft16_twisted(cd* x) {
#pragma unroll
  for (int a = 0; a < 4; ++a) dft4_tw<1>(x[a], x[a + 4], x[a + 8], x[a + 12], expi32(4), expi32(8), expi32(12));
#pragma unroll
  for (int k0 = 0; k0 < 4; ++k0)
    dft4_tw<1>(x[4 * k0], x[4 * k0 + 1], x[4 * k0 + 2], x[4 * k0 + 3], expi32(1 + 4 * k0), expi32(2 * (1 + 4 * k0)),
               expi32(3 * (1 + 4 * k0)));
  transpose4x4(x);
}

// Exchange buffer slot of U[r][k1][b]: rows of 32 values padded to 33, so that both sides
// (fixed (k1, b) over consecutive r; fixed r over consecutive k1) are bank-conflict-free for
// 16-byte and for 8-byte elements AND every address is (lane part) + (compile-time register
// part): no per-element address arithmetic, the register part rides in the instruction.
constexpr int WX_ROW = 33;
TFB_HD int wslot(int r, int k1, int b) { return WX_ROW * r + k1 + 16 * b; }

// Spectral index held by (lane t, register q) after wfft_forward.
TFB_HD int wspectral_index(int t, int q) { return (t & 15) + 16 * (2 * q + (t >> 4)); }

// The one shared-memory exchange of a transform.  Before it lane (r, h) = (t & 15, t >> 4)
// holds U[r][8h + j][b] in register 8b + j; after it lane (k1, b) = (t & 15, t >> 4) holds
// U[r][k1][b] in register r (FWD), or the other way round (inverse).  SPLIT moves the real and
// the imaginary parts in two rounds through a buffer of 512 doubles (4 KB per warp instead of
// 8 KB: room for more warps per SM).
#ifndef TFB_K1D_SPLIT
#define TFB_K1D_SPLIT 1
#endif
constexpr bool WX_SPLIT = TFB_K1D_SPLIT != 0;
TFB_HD constexpr int wbuf_bytes(bool split) { return WX_ROW * 16 * (split ? 8 : 16); }
constexpr int WBUF_BYTES = wbuf_bytes(WX_SPLIT);

template <bool FWD>
TFB_HD int wx_src(int t, int k) {  // slot of register k on the side that holds (r, h)-ordered data
  return wslot(t & 15, 8 * (t >> 4) + (k & 7), k >> 3);
}
TFB_HD int wx_dst(int t, int k) { return wslot(k, t & 15, t >> 4); }  // (k1, b)-ordered side, register k = r

// (W::kSplitExchange: the warp environment says which; a CTA of at most eight warps has the room for one round)
template <bool FWD, class W>
TFB_HD void wexchange(cd* x, int t, void* buf, W& w) {
  if (W::kSplitExchange) {
    double* b = reinterpret_cast<double*>(buf);
#pragma unroll
    for (int k = 0; k < WPTS; ++k) b[FWD ? wx_src<FWD>(t, k) : wx_dst(t, k)] = x[k].re;
    w();
#pragma unroll
    for (int k = 0; k < WPTS; ++k) x[k].re = b[FWD ? wx_dst(t, k) : wx_src<FWD>(t, k)];
    w();
#pragma unroll
    for (int k = 0; k < WPTS; ++k) b[FWD ? wx_src<FWD>(t, k) : wx_dst(t, k)] = x[k].im;
    w();
#pragma unroll
    for (int k = 0; k < WPTS; ++k) x[k].im = b[FWD ? wx_dst(t, k) : wx_src<FWD>(t, k)];
    w();  // the buffer may be overwritten by the next transform
  } else {
    cd* b = reinterpret_cast<cd*>(buf);
#pragma unroll
    for (int k = 0; k < WPTS; ++k) b[FWD ? wx_src<FWD>(t, k) : wx_dst(t, k)] = x[k];
    w();
#pragma unroll
    for (int k = 0; k < WPTS; ++k) x[k] = b[FWD ? wx_dst(t, k) : wx_src<FWD>(t, k)];
    w();
  }
}

// The 16 pass-1 twiddles of a lane (natural index k: 0..7 from sa, 8..15 from sb, each times g, g^2, ...)
// and the radix-2 twiddle c.  Built once per lane and stored in GROUP order, w[4 a + b] = twiddle of
// register a + 4 b: group a = registers (a, a+4, a+8, a+12) is what one radix-4 butterfly of the inverse
// and two radix-2 butterflies of the forward transform consume.  A twiddle provider hands them to the
// transforms one group at a time:
//   issue4(4 a, chunk) / settle4(chunk, w): group a;   issue_c / settle_c: the radix-2 twiddle
// (the B200 kernel keeps the table in tensor memory: rebuilding the chain inside every
// transform costs 56 FP64 instructions per transform on the pipe that limits K1d).
struct LaneTwiddles {
  cd w[WPTS];
  cd c;
};
TFB_HD void build_lane_twiddles(const WarpTwiddles* tw, int t, LaneTwiddles* out) {
  const cd g = tw->g[t];
  cd wa = tw->sa[t], wb = tw->sb[t];
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // natural registers j and 8 + j
    out->w[4 * (j & 3) + (j >> 2)] = wa;
    out->w[4 * (j & 3) + 2 + (j >> 2)] = wb;
    wa = cmul(wa, g);
    wb = cmul(wb, g);
  }
  out->c = tw->c[t];
}
// Providers split every read into issue (start the load into a Chunk) and settle (the values
// are valid, unpack them): tensor-memory loads are asynchronous, so a transform issues the
// next chunk before it works on the current one and the load latency hides behind FP64 work.
struct MemChunk4 {
  cd v[4];
};
struct MemTw {  // table in addressable memory (host emulation, key setup kernel)
  typedef MemChunk4 Chunk;
  const LaneTwiddles* lt;
  TFB_HD void issue4(int kb, Chunk& ch) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) ch.v[j] = lt->w[kb + j];
  }
  TFB_HD void issue_c(Chunk& ch) const { ch.v[0] = lt->c; }
  TFB_HD void settle4(Chunk& ch, cd* w) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = ch.v[j];
  }
  TFB_HD cd settle_c(Chunk& ch) const { return ch.v[0]; }
};

// flip the sign of x[m], odd m, on the lanes with h = 1 (sgn = h << 31): multiplying the
// inputs of a 16-point DFT by (-1)^m rotates its outputs by 8
TFB_HD void wflip_odd(cd* x, uint32_t sgn) {
#pragma unroll
  for (int m = 1; m < WPTS; m += 2) {
    x[m].re = bits_to_double(double_to_bits(x[m].re) ^ ((uint64_t)sgn << 32));
    x[m].im = bits_to_double(double_to_bits(x[m].im) ^ ((uint64_t)sgn << 32));
  }
}

// W: warp primitives -- operator()() = warp barrier with memory ordering, xchg16(v) = the
// value lane (t ^ 16) passed, turn_enter() / turn_leave() bracket the MAC stage (the B200 kernel
// rotates a turn between the warps of a scheduler there, see DevWarp; no-ops elsewhere).
//
// Forward negacyclic transform, unnormalised, 512 = 16 x 2 x 16:
//   pass 1   16-point DFTs over m of x[t + 32 m] in registers, twiddle W512^{t k1};
//   radix 2  between lanes t and t ^ 16 (decimation in frequency: butterfly, then the twiddle
//            W32^{r} on the odd half), 8 values sent and 8 received per lane.  Lane h = 1
//            keeps frequencies 8..15 and sends 0..7, lane h = 0 the opposite; to keep the code
//            free of selects lane h = 1 runs pass 1 with its odd inputs negated, which leaves
//            frequency k ^ 8 in register k, and carries the sign of its (K - G) in c[t];
//   exchange through shared memory, then 16-point DFTs over r.
//   in : x[m] = c_{t+32m} = a_{t+32m} + i a_{t+32m+512}   (untwisted)
//   out: x[q] = Z[wspectral_index(t, q)],  Z_k = sum_j c_j exp(i pi j / N) exp(2 pi i j k / 512)
// buf: WBUF_BYTES of shared memory private to the warp.
// FLIP = false: the caller has already applied the sign (-1)^(m h) to x[m] (the CMux folds it
// into the integer -> double conversion, where it is free).
template <bool FLIP = true, class W, class Tw>
TFB_HD void wfft_forward(cd* x, int t, const Tw& tw, void* buf, W& w) {
  typename Tw::Chunk ch[2], chc;
  tw.issue4(0, ch[0]);  // lands while the first 16-point DFT runs
  if (FLIP) wflip_odd(x, (uint32_t)(t >> 4) << 31);
  TFB_TICK(w, 0);
  dft16_twisted(x);
  // pass-1 twiddles folded into the cross-lane radix-2 stage: a lane multiplies only what it sends;
  // what it keeps enters as  w x + got  (4 FMA),  w x - got = (w x + got) - 2 got  (2 FMA)
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    cd wk[4];  // twiddles of registers a, a+4, a+8, a+12
    tw.settle4(ch[a & 1], wk);
    if (a + 1 < 4)
      tw.issue4(4 * (a + 1), ch[(a + 1) & 1]);
    else
      tw.issue_c(chc);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = a + 4 * e;
      const cd got = w.xchg16(cmul(x[8 + j], wk[2 + e]));
      cd u0;
      u0.re = fma(-wk[e].im, x[j].im, fma(wk[e].re, x[j].re, got.re));
      u0.im = fma(wk[e].im, x[j].re, fma(wk[e].re, x[j].im, got.im));
      x[j] = u0;
      x[8 + j] = cd{fma(-2.0, got.re, u0.re), fma(-2.0, got.im, u0.im)};
    }
  }
  {
    const cd c = tw.settle_c(chc);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[8 + j] = cmul(x[8 + j], c);
  }
  TFB_TICK(w, 1);
  wexchange<true>(x, t, buf, w);
  TFB_TICK(w, 2);
  dft16<1>(x);
  TFB_TICK(w, 3);
}

// Inverse of wfft_forward up to the factor 512 (folded into the key): the conjugate transpose,
// stage by stage.
//   in : x[q] = S[wspectral_index(t, q)]
//   out: x[m] = c_{t+32m}  (re -> coefficient t+32m, im -> coefficient t+32m+512)
// FLIP = false: the outputs are left as x[m] (-1)^(m h); the CMux folds the sign into the rounding.
template <bool FLIP = true, class W, class Tw>
TFB_HD void wfft_inverse(cd* x, int t, const Tw& tw, void* buf, W& w) {
  typename Tw::Chunk ch[2], chc;
  tw.issue_c(chc);
  TFB_TICK(w, 7);
  dft16<-1>(x);
  TFB_TICK(w, 8);
  wexchange<false>(x, t, buf, w);
  TFB_TICK(w, 9);
  {
    const cd c = tw.settle_c(chc), cc = cd{c.re, -c.im};
    tw.issue4(0, ch[0]);
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // keep x[j] + conj(c) x[8+j], send x[j] - conj(c) x[8+j]
      cd keep, send;
      bfly(x[j], x[8 + j], cc, keep, send);
      x[8 + j] = w.xchg16(send);
      x[j] = keep;
    }
  }
  // last 16-point DFT: the conjugate pass-1 twiddles ride in its first radix-4 layer (28 instead of
  // 16 + 16 instructions per butterfly), the mid twiddles in the second; the register part of the twist
  // multiplies the outputs (it depends on the output index, so it cannot be folded forward)
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    cd wk[4];
    tw.settle4(ch[a & 1], wk);
    if (a + 1 < 4) tw.issue4(4 * (a + 1), ch[(a + 1) & 1]);
#pragma unroll
    for (int b = 0; b < 4; ++b) wk[b].im = -wk[b].im;
    dft4_tw4<-1>(x[a], x[a + 4], x[a + 8], x[a + 12], wk[0], wk[1], wk[2], wk[3]);
  }
  dft16_layer_b<-1>(x);
  transpose4x4(x);
#pragma unroll
  for (int m = 1; m < WPTS; ++m) x[m] = cmulc(x[m], twist16(m));
  TFB_TICK(w, 10);
  if (FLIP) wflip_odd(x, (uint32_t)(t >> 4) << 31);
}

// Spectral key in this kernel's order.  The unit the key ring moves is a CHUNK = (pair m, stage s = 2 p + lvl,
// quarter qc of the 16 points a lane owns): [q4][key j][c][lane], 4 x 3 x 2 x 32 complex = 12 KB, prescaled by
// 1/512 -- what the MAC of four spectral points consumes, and what one accumulator chunk of the park pairs with.
// A key source offers acquire_chunk(m, s, qc) / load(ptr) / release().
constexpr int WCHUNK_Q = 4;
constexpr int WCHUNK_CD = WCHUNK_Q * BK_KEYS * 2 * WARP_T;  // 768 cd = 12 KB
constexpr int WCHUNKS_PER_PAIR = 4 * (WPTS / WCHUNK_Q);     // 16
TFB_HD size_t wchunk_offset(int m, int s, int qc) { return (((size_t)m * 4 + s) * (WPTS / WCHUNK_Q) + qc) * WCHUNK_CD; }
TFB_HD int wchunk_index(int q4, int j, int c, int t) { return ((q4 * BK_KEYS + j) * 2 + c) * WARP_T + t; }
struct GlobalWBk {  // plain pointer into the full key (host emulation)
  const cd* base;
  TFB_HD const cd* acquire_chunk(int m, int s, int qc) { return base + wchunk_offset(m, s, qc); }
  TFB_HD cd load(const cd* q) const { return *q; }
  TFB_HD void release() {}
};

// Accumulator layout of K1d.  The unrolled CMux never rotates ACC in the coefficient domain, so a lane keeps
// ITS 32 coefficients of a polynomial (mm = 0..15: coefficient t + 32 mm, the real parts of its transform inputs;
// mm = 16..31: coefficient t + 32 (mm - 16) + N/2, the imaginary parts) in one 128-byte row and moves them four at
// a time; the 16-byte units of a row are XOR-swizzled with the lane so that the eight lanes of a quarter warp hit
// eight different bank groups.
TFB_HD int wacc_unit(int t, int u) { return t * 32 + ((u ^ (t & 7)) << 2); }  // word offset of unit u = mm / 4
struct WarpAccLayout {
  TFB_HD int operator()(int j) const {
    const int t = j & 31, mm = ((j >> 5) & 15) | ((j >> 9) << 4);
    return wacc_unit(t, mm >> 2) + (mm & 3);
  }
};
struct alignas(16) Words4 {
  uint32_t w[4];
};

// Accumulator parking.  The 2 x 16 complex accumulators of a CMux are idle while a transform
// runs; a Park policy holds them outside the register file between MAC stages (the B200 kernel
// parks them in tensor memory, which is private per lane and has its own data path), in
// chunks of PARK_CH values per output polynomial:
//   issue_one(c, qb, chunk) / settle_one(chunk, o): load values qb .. qb+PARK_CH-1 of polynomial c
//   store(qb, o0, o1): the same values of both polynomials;  flush(): stores are visible to later loads
#ifndef TFB_PARK_CH
#define TFB_PARK_CH 4
#endif
constexpr int PARK_CH = TFB_PARK_CH;
static_assert(PARK_CH == WCHUNK_Q, "one key chunk pairs with one accumulator chunk");
struct RegPark {  // no parking: plain registers (host emulation)
  typedef MemChunk4 Chunk;
  cd v[2][WPTS];
  TFB_HD void issue_one(int c, int qb, Chunk& ch) const {
#pragma unroll
    for (int j = 0; j < PARK_CH; ++j) ch.v[j] = v[c][qb + j];
  }
  TFB_HD void settle_one(Chunk& ch, cd* o) const {
#pragma unroll
    for (int j = 0; j < PARK_CH; ++j) o[j] = ch.v[j];
  }
  TFB_HD void store(int qb, const cd* o0, const cd* o1) {
#pragma unroll
    for (int j = 0; j < PARK_CH; ++j) {
      v[0][qb + j] = o0[j];
      v[1][qb + j] = o1[j];
    }
  }
  TFB_HD void flush() const {}
};

// Spectral rotation factors of a pair for one lane: X^a at the point of register q is
// base * exp(i pi a q / 8), base = exp(i pi a (1 + 4 r + 64 h) / N)  (wspectral_index: f = r + 16 h + 32 q).
struct PairFactors {
  cd base1, base2;
  int a1, a2;
};
TFB_HD PairFactors pair_factors(const FactorTables* ft, int a1, int a2, int t) {
  const uint32_t cl = 1u + 4u * (uint32_t)(t & 15) + 64u * (uint32_t)(t >> 4);
  return PairFactors{unit_root(ft, (uint32_t)a1 * cl), unit_root(ft, (uint32_t)a2 * cl), a1, a2};
}

// MAC of one forward-transformed digit polynomial x (stage s of pair m) against the pair's three keys
// combined with the rotation factors; the accumulators live in the park.  FIRST starts them instead of
// loading them.  The warp takes its MAC turn once the first key chunk is resident.
template <bool FIRST, class W, class BkSource, class Park>
TFB_HD void wmac(Park& park, const cd* x, BkSource& bk, int m, int s, const PairFactors& pf, const FactorTables* ft,
                 int t, W& w) {
  typename Park::Chunk ch0[2], ch1[2];
#pragma unroll
  for (int qb = 0; qb < WPTS; qb += PARK_CH) {
    const cd* key = bk.acquire_chunk(m, s, qb / PARK_CH) + t;
    if (qb == 0) {
      TFB_TICK(w, 4);
      w.turn_enter();
      TFB_TICK(w, 5);
      if (!FIRST) {
        park.issue_one(0, 0, ch0[0]);
        park.issue_one(1, 0, ch1[0]);
      }
    }
    cd o0[PARK_CH], o1[PARK_CH];
    if (!FIRST) {
      const int cur = (qb / PARK_CH) & 1;
      park.settle_one(ch0[cur], o0);
      park.settle_one(ch1[cur], o1);
      if (qb + PARK_CH < WPTS) {  // the next chunk travels while this one is multiplied
        park.issue_one(0, qb + PARK_CH, ch0[cur ^ 1]);
        park.issue_one(1, qb + PARK_CH, ch1[cur ^ 1]);
      }
    }
#pragma unroll
    for (int j = 0; j < PARK_CH; ++j) {
      const int q = qb + j;
      const cd u1 = rotation_minus_one(pf.base1, ft->A[(4 * pf.a1 * q) & 63]);
      const cd u2 = rotation_minus_one(pf.base2, ft->A[(4 * pf.a2 * q) & 63]);
      const cd k0 = combine_keys(u1, u2, bk.load(key + wchunk_index(j, 0, 0, 0)), bk.load(key + wchunk_index(j, 1, 0, 0)),
                                 bk.load(key + wchunk_index(j, 2, 0, 0)));
      const cd k1 = combine_keys(u1, u2, bk.load(key + wchunk_index(j, 0, 1, 0)), bk.load(key + wchunk_index(j, 1, 1, 0)),
                                 bk.load(key + wchunk_index(j, 2, 1, 0)));
      if (FIRST) {
        o0[j] = cmul(x[q], k0);
        o1[j] = cmul(x[q], k1);
      } else {
        cmac(o0[j], x[q], k0);
        cmac(o1[j], x[q], k1);
      }
    }
    park.store(qb, o0, o1);
    if (qb + PARK_CH == WPTS) w.turn_leave();
    bk.release();
  }
  park.flush();
}

// unsigned digit field -> exact double of the signed digit (mantissa trick; an I2F.F64 measured 2 % slower)
TFB_HD double wdigit(uint32_t field) { return digit_to_double(field); }
// sg * digit for sg = +-1 (the lane sign of the odd inputs): one FMA instead of the DADD, exact
TFB_HD double wdigit_signed(uint32_t field, double sg, double neg_sg_bias) {
  return fma(bits_to_double(0x4330000000000000ull | (uint64_t)field), sg, neg_sg_bias);
}
// round-to-nearest-even(sg * x) mod 2^32 for sg = +-1
TFB_HD uint32_t round_to_word_signed(double x, double sg) {
  return (uint32_t)double_to_bits(fma(x, sg, 6755399441055744.0));
}

// Stage s = 2p + lvl of a pair step: digits of accumulator polynomial p at gadget level lvl (both levels are
// cut from the lane's own 32 words of ACC[p], eight 16-byte loads), forward transform, MAC against the keys.
template <bool FIRST, class W, class BkSource, class Park, class Tw>
TFB_HD void wcmux_stage(int s, const uint32_t* acc, int m, const PairFactors& pf, const FactorTables* ft, BkSource& bk,
                        int t, const Tw& tw, void* buf, W& w, Park& park) {
  const int p = s >> 1, lvl = s & 1;
  cd x[WPTS];
  // lanes with h = 1 feed the transform -x[mm] for odd mm (see wfft_forward): sign folded into the conversion
  const double sg = (t >> 4) ? -1.0 : 1.0, nsb = -sg * (4503599627370496.0 + (double)DIGIT_HALF);
  const int shift = 32 - (lvl + 1) * BK_BGBIT;
  const uint32_t* poly = acc + p * RING_N;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const Words4 re = *reinterpret_cast<const Words4*>(poly + wacc_unit(t, u));
    const Words4 im = *reinterpret_cast<const Words4*>(poly + wacc_unit(t, u + 4));
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int mm = 4 * u + e;
      const uint32_t fr = ((re.w[e] + DECOMP_OFFSET) >> shift) & ((1u << BK_BGBIT) - 1);
      const uint32_t fi = ((im.w[e] + DECOMP_OFFSET) >> shift) & ((1u << BK_BGBIT) - 1);
      x[mm] = (mm & 1) ? cd{wdigit_signed(fr, sg, nsb), wdigit_signed(fi, sg, nsb)} : cd{wdigit(fr), wdigit(fi)};
    }
  }
  wfft_forward<false>(x, t, tw, buf, w);
  wmac<FIRST>(park, x, bk, m, s, pf, ft, t, w);
  TFB_TICK(w, 6);
}

// One pair step by one warp.  acc: 2 polynomials of N words in shared memory (WarpAccLayout).
// Stage 0 starts the accumulators; stages 1..3 and the two inverse transforms run as rolled
// loops (TFB_K1D_ROLL): one copy of the transform code in the instruction cache.
template <class W, class BkSource, class Park, class Tw>
TFB_HD void wcmux_step(uint32_t* acc, int m, int a1, int a2, const FactorTables* ft, BkSource& bk, int t, const Tw& tw,
                       void* buf, W& w, Park& park) {
  const PairFactors pf = pair_factors(ft, a1, a2, t);
  wcmux_stage<true>(0, acc, m, pf, ft, bk, t, tw, buf, w, park);
  TFB_K1D_LOOP
  for (int s = 1; s < 4; ++s) wcmux_stage<false>(s, acc, m, pf, ft, bk, t, tw, buf, w, park);
  TFB_K1D_LOOP
  for (int c = 0; c < 2; ++c) {
    cd x[WPTS];
    {
      typename Park::Chunk ch[WPTS / PARK_CH];
#pragma unroll
      for (int qb = 0; qb < WPTS; qb += PARK_CH) park.issue_one(c, qb, ch[qb / PARK_CH]);
#pragma unroll
      for (int qb = 0; qb < WPTS; qb += PARK_CH) park.settle_one(ch[qb / PARK_CH], x + qb);
    }
    wfft_inverse<false>(x, t, tw, buf, w);
    const double sg = (t >> 4) ? -1.0 : 1.0;  // the inverse leaves -x[mm] for odd mm on the lanes with h = 1
    uint32_t* poly = acc + c * RING_N;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      Words4* pr = reinterpret_cast<Words4*>(poly + wacc_unit(t, u));
      Words4* pi = reinterpret_cast<Words4*>(poly + wacc_unit(t, u + 4));
      Words4 re = *pr, im = *pi;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int mm = 4 * u + e;
        re.w[e] += (mm & 1) ? round_to_word_signed(x[mm].re, sg) : round_to_word(x[mm].re);
        im.w[e] += (mm & 1) ? round_to_word_signed(x[mm].im, sg) : round_to_word(x[mm].im);
      }
      *pr = re;
      *pi = im;
    }
    TFB_TICK(w, 11);
  }
  w();
}

// Whole gate bootstrap (without key switch) for one ciphertext by one warp.
//   sm_acc: 2N words, sm_abar: n+2 uint16, buf: WBUF_BYTES, ext: N+1 words out
template <class W, class BkSource, class Park, class Tw>
TFB_HD void gate_bootstrap_warp(const uint32_t* x_row, const uint32_t* y_row, int kind, int n, uint32_t mu,
                                BkSource& bk, const Tw& tw, const FactorTables* ft, uint32_t* sm_acc, uint16_t* sm_abar,
                                void* buf, uint32_t* ext, int t, W& w, Park& park) {
  bootstrap_prologue(x_row, y_row, kind, n, mu, sm_acc, sm_abar, t, WARP_T, w, WarpAccLayout());
  const int pairs = (n + 1) / 2;
#pragma unroll 1
  for (int m = 0; m < pairs; ++m) {
    int a1, a2;
    pair_rotations(sm_abar, n, m, a1, a2);
    if ((a1 | a2) == 0) {  // uniform across the warp: both factors vanish, the step is the identity
      // keep the key ring and the turn protocol in step, in the order a real step takes them (a warp that
      // held its turns back while it drained a pair's chunks would stall the ring its partners wait on)
#pragma unroll 1
      for (int s = 0; s < 4; ++s) {
#pragma unroll 1
        for (int qc = 0; qc < WPTS / WCHUNK_Q; ++qc) {
          bk.acquire_chunk(m, s, qc);
          if (qc == 0) w.turn_enter();
          if (qc + 1 == WPTS / WCHUNK_Q) w.turn_leave();
          bk.release();
        }
      }
      continue;
    }
    wcmux_step(sm_acc, m, a1, a2, ft, bk, t, tw, buf, w, park);
  }
  if (ext) bootstrap_extract(sm_acc, ext, t, WARP_T, WarpAccLayout());  // null: surplus warp of a tail CTA
}

}  // namespace tfb
