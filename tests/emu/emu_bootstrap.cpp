// Host emulation of kernel K1: runs the exact __host__ __device__ code of
// paper_2005_01945_b200/csrc/tfhe_device.cuh with 64 std::threads per
// ciphertext and a pthread barrier standing in for __syncthreads().  Test
// infrastructure only: lets the CPU test-suite check the kernel's index math,
// twiddles, swizzles and rounding against the integer oracle without a GPU.
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

#include <thread>
#include <vector>

#include "../../paper_2005_01945_b200/csrc/tfhe_device.cuh"
#include "../../paper_2005_01945_b200/csrc/tfhe_warp.cuh"

using namespace tfb;

namespace {
struct BarrierSync {
  pthread_barrier_t* b;
  void operator()() const { pthread_barrier_wait(b); }
};

void fill_twiddles(Twiddles* tw) {
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

template <class F>
void run_group(F body) {
  pthread_barrier_t bar;
  pthread_barrier_init(&bar, nullptr, FFT_THREADS);
  std::vector<std::thread> th;
  for (int t = 0; t < FFT_THREADS; ++t) th.emplace_back([&, t] { BarrierSync s{&bar}; body(t, s); });
  for (auto& x : th) x.join();
  pthread_barrier_destroy(&bar);
}
}  // namespace

extern "C" {

// spectral key in the kernel's staged layout [n][p][k2][lvl][c][t], prescaled by 1/512
void emu_bk_transform(const int32_t* bk_raw, int n, double* bkf_out) {
  Twiddles tw;
  fill_twiddles(&tw);
  cd* bkf = reinterpret_cast<cd*>(bkf_out);
  std::vector<cd> bufA(HALF_N), bufB(HALF_N);
  for (int64_t poly = 0; poly < (int64_t)n * BK_ROWS * 2; ++poly) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(bk_raw) + poly * RING_N;
    const int c = (int)(poly & 1);
    const int64_t ir = poly >> 1;
    run_group([&](int t, BarrierSync& s) {
      cd x[8];
      for (int m = 0; m < 8; ++m)
        x[m] = cd{int32_to_double(src[t + 64 * m]), int32_to_double(src[t + 64 * m + HALF_N])};
      fft_forward(x, t, TableTw{&tw, t}, bufA.data(), bufB.data(), s);
      for (int k2 = 0; k2 < 8; ++k2)
        bkf[stage_offset((int)(ir / BK_ROWS), (int)(ir % BK_ROWS) / BK_L) + stage_index(k2, (int)(ir % BK_L), c, t)] =
            cd{x[k2].re / HALF_N, x[k2].im / HALF_N};
    });
  }
}

// forward transform of one int32 polynomial, natural frequency order, unnormalised
void emu_fft_forward(const int32_t* poly, double* spec_out) {
  Twiddles tw;
  fill_twiddles(&tw);
  std::vector<cd> bufA(HALF_N), bufB(HALF_N);
  cd* out = reinterpret_cast<cd*>(spec_out);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(poly);
  run_group([&](int t, BarrierSync& s) {
    cd x[8];
    for (int m = 0; m < 8; ++m)
      x[m] = cd{int32_to_double(src[t + 64 * m]), int32_to_double(src[t + 64 * m + HALF_N])};
    fft_forward(x, t, TableTw{&tw, t}, bufA.data(), bufB.data(), s);
    for (int k2 = 0; k2 < 8; ++k2) out[spectral_index(t, k2)] = x[k2];
  });
}

// inverse of emu_fft_forward (divides by 512), rounded to words
void emu_fft_inverse(const double* spec_in, uint32_t* poly_out) {
  Twiddles tw;
  fill_twiddles(&tw);
  std::vector<cd> bufA(HALF_N), bufB(HALF_N);
  const cd* in = reinterpret_cast<const cd*>(spec_in);
  run_group([&](int t, BarrierSync& s) {
    cd x[8];
    for (int k2 = 0; k2 < 8; ++k2) {
      cd v = in[spectral_index(t, k2)];
      x[k2] = cd{v.re / HALF_N, v.im / HALF_N};
    }
    fft_inverse(x, t, TableTw{&tw, t}, bufA.data(), bufB.data(), s);
    for (int m = 0; m < 8; ++m) {
      poly_out[t + 64 * m] = round_to_word(x[m].re);
      poly_out[t + 64 * m + HALF_N] = round_to_word(x[m].im);
    }
  });
}

// K1 for k ciphertexts: x, y packed [k][n+1]; ext_out [k][N+1]
void emu_gate_bootstrap(const uint32_t* x, const uint32_t* y, const uint8_t* kinds, int64_t k, int n,
                        uint32_t mu, const double* bkf_in, uint32_t* ext_out) {
  Twiddles tw;
  fill_twiddles(&tw);
  const cd* bkf = reinterpret_cast<const cd*>(bkf_in);
  for (int64_t g = 0; g < k; ++g) {
    std::vector<cd> bufA(HALF_N), bufB(HALF_N);
    std::vector<uint32_t> acc(2 * RING_N), ext(EXT_STRIDE);
    std::vector<uint16_t> abar(n + 1);
    run_group([&](int t, BarrierSync& s) {
      GlobalBk bk{bkf};
      NoPark park;
      gate_bootstrap(x + g * (n + 1), y + g * (n + 1), (int)kinds[g], n, mu, bk, &tw, acc.data(), abar.data(),
                     bufA.data(), bufB.data(), ext.data(), t, s, park);
    });
    for (int j = 0; j <= RING_N; ++j) ext_out[g * (RING_N + 1) + j] = ext[j];
  }
}

// K1c (wide / latency variant): 256 host threads per ciphertext, 4 group barriers + 1 CTA barrier
void emu_gate_bootstrap_wide(const uint32_t* x, const uint32_t* y, const uint8_t* kinds, int64_t k, int n,
                             uint32_t mu, const double* bkf_in, uint32_t* ext_out) {
  Twiddles tw;
  fill_twiddles(&tw);
  const cd* bkf = reinterpret_cast<const cd*>(bkf_in);
  constexpr int WIDE = 4 * FFT_THREADS;
  for (int64_t g = 0; g < k; ++g) {
    std::vector<cd> xbuf(8 * HALF_N), red(8 * HALF_N);
    std::vector<uint32_t> acc(2 * RING_N), ext(EXT_STRIDE);
    std::vector<uint16_t> abar(n + 1);
    pthread_barrier_t cta, grp[4];
    pthread_barrier_init(&cta, nullptr, WIDE);
    for (auto& b : grp) pthread_barrier_init(&b, nullptr, FFT_THREADS);
    std::vector<std::thread> th;
    for (int tid = 0; tid < WIDE; ++tid)
      th.emplace_back([&, tid] {
        BarrierSync gs{&grp[tid / FFT_THREADS]}, cs{&cta};
        gate_bootstrap_wide(x + g * (n + 1), y + g * (n + 1), (int)kinds[g], n, mu, bkf, &tw, acc.data(),
                            abar.data(), xbuf.data(), red.data(), ext.data(), tid, gs, cs,
                            [](const cd* q) { return *q; });
      });
    for (auto& t : th) t.join();
    pthread_barrier_destroy(&cta);
    for (auto& b : grp) pthread_barrier_destroy(&b);
    for (int j = 0; j <= RING_N; ++j) ext_out[g * (RING_N + 1) + j] = ext[j];
  }
}

// key-switch digits exactly as K2 derives them: digits_out[N][KS_T]
void emu_ks_digits(const uint32_t* ext, int32_t* digits_out) {
  const uint32_t bias = ks_bias();
  for (int i = 0; i < RING_N; ++i)
    for (int j = 0; j < KS_T; ++j) digits_out[i * KS_T + j] = ks_digit(ext[i] + bias, j);
}
}

// ---- K1d: one ciphertext per warp (tfhe_warp.cuh), 32 host threads per warp ----------------
namespace {
struct EmuWarp {
  pthread_barrier_t* b;
  cd* scratch;  // 32 cd
  int lane;
  void operator()() const { pthread_barrier_wait(b); }
  void turn_enter() const {}
  void turn_leave() const {}
  void turn_pass() const {}
  cd xchg16(cd v) const {
    scratch[lane] = v;
    pthread_barrier_wait(b);
    const cd r = scratch[lane ^ 16];
    pthread_barrier_wait(b);
    return r;
  }
};

void fill_warp_twiddles(WarpTwiddles* tw) { tfb::fill_warp_twiddles<long double>(tw, cosl, sinl); }

template <class F>
void run_warp(F body) {
  pthread_barrier_t bar;
  pthread_barrier_init(&bar, nullptr, WARP_T);
  std::vector<cd> scratch(WARP_T);
  std::vector<std::thread> th;
  for (int t = 0; t < WARP_T; ++t)
    th.emplace_back([&, t] {
      EmuWarp w{&bar, scratch.data(), t};
      body(t, w);
    });
  for (auto& x : th) x.join();
  pthread_barrier_destroy(&bar);
}
}  // namespace

extern "C" {

void emu_w_fft_forward(const int32_t* poly, double* spec_out) {
  WarpTwiddles tw;
  fill_warp_twiddles(&tw);
  std::vector<cd> buf(WBUF_BYTES / sizeof(cd) + 1);
  cd* out = reinterpret_cast<cd*>(spec_out);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(poly);
  run_warp([&](int t, EmuWarp& w) {
    cd x[WPTS];
    for (int m = 0; m < WPTS; ++m)
      x[m] = cd{int32_to_double(src[t + 32 * m]), int32_to_double(src[t + 32 * m + HALF_N])};
    LaneTwiddles lt;
    build_lane_twiddles(&tw, t, &lt);
    wfft_forward(x, t, MemTw{&lt}, buf.data(), w);
    for (int q = 0; q < WPTS; ++q) out[wspectral_index(t, q)] = x[q];
  });
}

void emu_w_fft_inverse(const double* spec_in, uint32_t* poly_out) {
  WarpTwiddles tw;
  fill_warp_twiddles(&tw);
  std::vector<cd> buf(WBUF_BYTES / sizeof(cd) + 1);
  const cd* in = reinterpret_cast<const cd*>(spec_in);
  run_warp([&](int t, EmuWarp& w) {
    cd x[WPTS];
    for (int q = 0; q < WPTS; ++q) {
      const cd v = in[wspectral_index(t, q)];
      x[q] = cd{v.re / HALF_N, v.im / HALF_N};
    }
    LaneTwiddles lt;
    build_lane_twiddles(&tw, t, &lt);
    wfft_inverse(x, t, MemTw{&lt}, buf.data(), w);
    for (int m = 0; m < WPTS; ++m) {
      poly_out[t + 32 * m] = round_to_word(x[m].re);
      poly_out[t + 32 * m + HALF_N] = round_to_word(x[m].im);
    }
  });
}

// spectral key in K1d's staged layout [n][p][lvl][q][c][lane], prescaled by 1/512
void emu_w_bk_transform(const int32_t* bk_raw, int n, double* bkf_out) {
  WarpTwiddles tw;
  fill_warp_twiddles(&tw);
  cd* bkf = reinterpret_cast<cd*>(bkf_out);
  std::vector<cd> buf(WBUF_BYTES / sizeof(cd) + 1);
  for (int64_t poly = 0; poly < (int64_t)n * BK_ROWS * 2; ++poly) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(bk_raw) + poly * RING_N;
    const int c = (int)(poly & 1);
    const int64_t ir = poly >> 1;
    run_warp([&](int t, EmuWarp& w) {
      cd x[WPTS];
      for (int m = 0; m < WPTS; ++m)
        x[m] = cd{int32_to_double(src[t + 32 * m]), int32_to_double(src[t + 32 * m + HALF_N])};
      LaneTwiddles lt;
      build_lane_twiddles(&tw, t, &lt);
      wfft_forward(x, t, MemTw{&lt}, buf.data(), w);
      for (int q = 0; q < WPTS; ++q)
        bkf[stage_offset((int)(ir / BK_ROWS), (int)(ir % BK_ROWS) / BK_L) + wstage_index((int)(ir % BK_L), q, c, t)] =
            cd{x[q].re / HALF_N, x[q].im / HALF_N};
    });
  }
}

void emu_w_gate_bootstrap(const uint32_t* x, const uint32_t* y, const uint8_t* kinds, int64_t k, int n,
                          uint32_t mu, const double* bkf_in, uint32_t* ext_out) {
  WarpTwiddles tw;
  fill_warp_twiddles(&tw);
  const cd* bkf = reinterpret_cast<const cd*>(bkf_in);
  for (int64_t g = 0; g < k; ++g) {
    std::vector<cd> buf(WBUF_BYTES / sizeof(cd) + 1);
    std::vector<uint32_t> acc(2 * RING_N), ext(EXT_STRIDE);
    std::vector<uint16_t> abar(n + 1);
    run_warp([&](int t, EmuWarp& w) {
      GlobalBk bk{bkf};
      RegPark park;
      LaneTwiddles lt;
      build_lane_twiddles(&tw, t, &lt);
      gate_bootstrap_warp(x + g * (n + 1), y + g * (n + 1), (int)kinds[g], n, mu, bk, MemTw{&lt}, acc.data(),
                          abar.data(), buf.data(), ext.data(), t, w, park);
    });
    for (int j = 0; j <= RING_N; ++j) ext_out[g * (RING_N + 1) + j] = ext[j];
  }
}
}
