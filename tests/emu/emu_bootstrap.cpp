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

#include <atomic>

#include "../../paper_2005_01945_b200/csrc/tfhe_device.cuh"
#include "../../paper_2005_01945_b200/csrc/tfhe_pair.cuh"
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

// spectral key in K1e's chunk layout [pair][p][lvl][half][k4][key][c][t], prescaled by 1/512
void emu_bk_transform(const int32_t* bk_raw, int n, double* bkf_out) {
  Twiddles tw;
  fill_twiddles(&tw);
  cd* bkf = reinterpret_cast<cd*>(bkf_out);
  std::vector<cd> bufA(HALF_N), bufB(HALF_N);
  const int64_t polys = (int64_t)((n + 1) / 2) * BK_KEYS * BK_ROWS * 2;
  for (int64_t poly = 0; poly < polys; ++poly) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(bk_raw) + poly * RING_N;
    const int c = (int)(poly & 1), r = (int)((poly >> 1) % BK_ROWS), j = (int)((poly >> 1) / BK_ROWS % BK_KEYS);
    const int m = (int)((poly >> 1) / BK_ROWS / BK_KEYS);
    run_group([&](int t, BarrierSync& s) {
      cd x[8];
      for (int mm = 0; mm < 8; ++mm)
        x[mm] = cd{int32_to_double(src[t + 64 * mm]), int32_to_double(src[t + 64 * mm + HALF_N])};
      fft_forward(x, t, TableTw{&tw, t}, bufA.data(), bufB.data(), s);
      for (int k2 = 0; k2 < 8; ++k2)
        bkf[pchunk_offset(m, r / BK_L, r % BK_L, k2 >> 2) + pchunk_index(k2 & 3, j, c, t)] =
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

}  // extern "C"
namespace {
struct PairCta {
  std::vector<cd> xbuf, swap;
  std::vector<uint32_t> acc, recv;
  std::vector<uint16_t> abar;
  std::atomic<int> arrived[2];
  pthread_barrier_t cta, grp[2];
};
struct PairHostEnv {
  BarrierSync gsync;
  PairCta *self, *peer;
  pthread_barrier_t* cluster;
  const cd* bkf;
  int p, grp, t;
  static constexpr bool helpers = false;  // the main groups combine their keys themselves
  void cta_sync() { pthread_barrier_wait(&self->cta); }
  void all_sync() { pthread_barrier_wait(&self->cta); }
  const cd* keys_ready(uint32_t) { return nullptr; }
  void keys_taken(uint32_t) {}
  void start(const uint16_t*, int) { pthread_barrier_wait(cluster); }
  const cd* key_wait(uint32_t, int m, int h) { return bkf + pchunk_offset(m, p, grp, h); }
  void key_done(uint32_t, int, int) {}
  void arm_recv(uint32_t) {}
  void send16(const uint32_t* v, uint32_t step) {
    for (int q = 0; q < 16; ++q) peer->recv[(step & 1) * RING_N + t * 16 + q] = v[q];
    peer->arrived[step & 1].fetch_add(1, std::memory_order_release);
  }
  void recv16(uint32_t* r, uint32_t step) {
    const int want = FFT_THREADS * (int)(step / 2 + 1);
    while (self->arrived[step & 1].load(std::memory_order_acquire) < want) std::this_thread::yield();
    for (int q = 0; q < 16; ++q) r[q] = self->recv[(step & 1) * RING_N + t * 16 + q];
  }
  void finish() { pthread_barrier_wait(cluster); }
  void tick(int) {}
};
}  // namespace
extern "C" {

// K1e (one gate over two CTAs of two 64-thread groups): 256 host threads per ciphertext; the peer exchange
// is a plain buffer with an atomic arrival count standing in for the DSMEM stores and their mbarrier.
void emu_pair_gate_bootstrap(const uint32_t* x, const uint32_t* y, const uint8_t* kinds, int64_t k, int n,
                             uint32_t mu, const double* bkf_in, uint32_t* ext_out) {
  Twiddles tw;
  fill_twiddles(&tw);
  FactorTables ft;
  fill_factor_tables<long double>(&ft, cosl, sinl);
  const cd* bkf = reinterpret_cast<const cd*>(bkf_in);
  for (int64_t g = 0; g < k; ++g) {
    PairCta cta[2];
    pthread_barrier_t cluster;
    pthread_barrier_init(&cluster, nullptr, 2 * PAIR_THREADS);
    std::vector<uint32_t> ext(EXT_STRIDE);
    for (auto& c : cta) {
      c.xbuf.resize(4 * HALF_N);
      c.swap.resize(2 * HALF_N);
      c.acc.resize(RING_N);
      c.recv.resize(2 * RING_N);
      c.abar.resize(n + 2);
      c.arrived[0] = 0;
      c.arrived[1] = 0;
      pthread_barrier_init(&c.cta, nullptr, PAIR_THREADS);
      for (auto& b : c.grp) pthread_barrier_init(&b, nullptr, FFT_THREADS);
    }
    std::vector<std::thread> th;
    for (int p = 0; p < 2; ++p)
      for (int tid = 0; tid < PAIR_THREADS; ++tid)
        th.emplace_back([&, p, tid] {
          const int grp = tid / FFT_THREADS;
          PairHostEnv env{BarrierSync{&cta[p].grp[grp]}, &cta[p], &cta[p ^ 1], &cluster, bkf, p, grp, tid % FFT_THREADS};
          cd* bufA = cta[p].xbuf.data() + (size_t)grp * 2 * HALF_N;
          pair_prologue(env, x + g * (n + 1), y + g * (n + 1), (int)kinds[g], n, mu, cta[p].acc.data(), cta[p].abar.data(), p,
                        tid, PAIR_THREADS);
          pair_blind_rotate(env, n, &tw, &ft, cta[p].acc.data(), cta[p].abar.data(), bufA, bufA + HALF_N, cta[p].swap.data(),
                            p, tid);
          pair_extract(cta[p].acc.data(), ext.data(), p, tid);
          env.finish();
        });
    for (auto& t : th) t.join();
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
  static constexpr bool kSplitExchange = WX_SPLIT;
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

// spectral key in K1d's chunk layout [pair][stage][qc][q4][key][c][lane], prescaled by 1/512
void emu_w_bk_transform(const int32_t* bk_raw, int n, double* bkf_out) {
  WarpTwiddles tw;
  fill_warp_twiddles(&tw);
  cd* bkf = reinterpret_cast<cd*>(bkf_out);
  std::vector<cd> buf(WBUF_BYTES / sizeof(cd) + 1);
  const int64_t polys = (int64_t)((n + 1) / 2) * BK_KEYS * BK_ROWS * 2;
  for (int64_t poly = 0; poly < polys; ++poly) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(bk_raw) + poly * RING_N;
    const int c = (int)(poly & 1), r = (int)((poly >> 1) % BK_ROWS), j = (int)((poly >> 1) / BK_ROWS % BK_KEYS);
    const int m = (int)((poly >> 1) / BK_ROWS / BK_KEYS);
    run_warp([&](int t, EmuWarp& w) {
      cd x[WPTS];
      for (int mm = 0; mm < WPTS; ++mm)
        x[mm] = cd{int32_to_double(src[t + 32 * mm]), int32_to_double(src[t + 32 * mm + HALF_N])};
      LaneTwiddles lt;
      build_lane_twiddles(&tw, t, &lt);
      wfft_forward(x, t, MemTw{&lt}, buf.data(), w);
      for (int q = 0; q < WPTS; ++q)
        bkf[wchunk_offset(m, r, q / WCHUNK_Q) + wchunk_index(q % WCHUNK_Q, j, c, t)] = cd{x[q].re / HALF_N, x[q].im / HALF_N};
    });
  }
}

void emu_w_gate_bootstrap(const uint32_t* x, const uint32_t* y, const uint8_t* kinds, int64_t k, int n,
                          uint32_t mu, const double* bkf_in, uint32_t* ext_out) {
  WarpTwiddles tw;
  fill_warp_twiddles(&tw);
  FactorTables ft;
  fill_factor_tables<long double>(&ft, cosl, sinl);
  const cd* bkf = reinterpret_cast<const cd*>(bkf_in);
  for (int64_t g = 0; g < k; ++g) {
    std::vector<cd> buf(WBUF_BYTES / sizeof(cd) + 1);
    std::vector<Words4> acc(2 * RING_N / 4);
    std::vector<uint32_t> ext(EXT_STRIDE);
    std::vector<uint16_t> abar(n + 2);
    run_warp([&](int t, EmuWarp& w) {
      GlobalWBk bk{bkf};
      RegPark park;
      LaneTwiddles lt;
      build_lane_twiddles(&tw, t, &lt);
      gate_bootstrap_warp(x + g * (n + 1), y + g * (n + 1), (int)kinds[g], n, mu, bk, MemTw{&lt}, &ft,
                          reinterpret_cast<uint32_t*>(acc.data()), abar.data(), buf.data(), ext.data(), t, w, park);
    });
    for (int j = 0; j <= RING_N; ++j) ext_out[g * (RING_N + 1) + j] = ext[j];
  }
}
}
