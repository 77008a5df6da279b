/* tfhe_gate_oracle.c -- CPU restatement of real TFHE gate bootstrapping.
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 *
 * PARITY UNPINNED BY THE REFERENCE at the ciphertext-coefficient level: the
 * reference (/root/reference/pkg/src/encirc) does not implement blind
 * rotation, key switching or a bootstrapping key; its OracleBootstrapEngine
 * decrypts with the secret key and re-encrypts (encirc/engine.py:493-503,
 * SPEC.md:13).  The arithmetic below restates the published construction
 * (Chillotti, Gama, Georgieva, Izabachene: "TFHE: Fast Fully Homomorphic
 * Encryption over the Torus", J. Cryptology 2020, Algorithms 3, 4, 9 and
 * section 5.2 "gate bootstrapping") over the 32-bit torus, with every step
 * in exact integer arithmetic (schoolbook negacyclic products mod 2^32), so
 * it is the ground truth the CUDA kernels must match bit for bit.  What IS
 * pinned by the reference, and checked in tests/: the gate linear form
 * (encirc/engine.py:77-86,483-484), the decision rule "1 iff 0 < phase < 1/2"
 * (encirc/engine.py:498, encirc/torus.py:303-304), the +-mu output encoding
 * and the fresh noise bound 2^-5 that every gate output must respect
 * (encirc/torus.py:177-184).
 *
 * Parameter set (ring side chosen by the builder): N = 1024,
 * k = 1, l = 2, Bg = 2^9 (rounded to 18 bits), key switch t = 8, base 4, signed digits.
 *
 * Blind rotation with an UNROLLED bootstrapping key (Zhou, Yang, Zhang, Yang, Wang:
 * "Faster bootstrapping with multiple addends", IEEE Access 2018; Bourse, Minelli, Minihold,
 * Paillier, CRYPTO 2018 section 5): two LWE mask elements per CMux.  With key bits s1, s2 and
 * rotations a1, a2,  X^(a1 s1 + a2 s2) - 1 = s1 u1 + s2 u2 + s1 s2 u1 u2,  u_i = X^(a_i) - 1,
 * so one step is
 *   ACC <- ACC + u1 (BK[s1] [.] ACC) + u2 (BK[s2] [.] ACC) + u1 u2 (BK[s1 s2] [.] ACC)
 * with ONE gadget decomposition of ACC shared by the three external products: n/2 steps of
 * four forward and two inverse transforms instead of n.  An odd n pads s2 = 0, a2 = 0.
 *
 * A second blind-rotation path (`fft` = 1) evaluates the external product
 * with a textbook radix-2 double-precision FFT, as CPU TFHE libraries do.  It
 * exists to time a like-for-like CPU bootstrap and is itself checked against
 * the exact path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define RN 1024
#define HN 512
#define BK_L 2
#define BGBIT 9
#define BK_KEYS 3 /* TRGSW samples per pair of mask elements: s1, s2, s1*s2 */
#define ROWS 4
#define KS_T 8
#define KS_BB 2

/* gate table, order of TWO_INPUT_KINDS (encirc/engine.py:77-88) + identity */
static const int GX[9] = {1, 1, -1, -1, 2, -2, -1, -1, 1};
static const int GY[9] = {1, 1, -1, -1, 2, -2, 1, 1, 0};
static const int GO[9] = {-1, 1, 1, -1, 2, -2, -1, 1, 0};

/* out[0..n] = cx*x + cy*y + off*mu  (mask words then body) */
void oracle_gate_linear(const uint32_t *x, const uint32_t *y, int kind, uint32_t mu, int n, uint32_t *out) {
  for (int w = 0; w <= n; ++w) out[w] = (uint32_t)GX[kind] * x[w] + (uint32_t)GY[kind] * y[w];
  out[n] += (uint32_t)GO[kind] * mu;
}

/* round(a * 2N / 2^32) mod 2N */
static int mod_switch(uint32_t a) { return (int)(((uint64_t)a + (1u << 20)) >> 21) & (2 * RN - 1); }

void oracle_mod_switch(const uint32_t *lwe, int n, int32_t *bar) {
  for (int w = 0; w <= n; ++w) bar[w] = mod_switch(lwe[w]);
}

/* dst = X^e * src in Z[X]/(X^N+1), e in [0, 2N) */
static void mul_by_xe(uint32_t *dst, const uint32_t *src, int e) {
  for (int j = 0; j < RN; ++j) {
    int s = ((j - e) % (2 * RN) + 2 * RN) % (2 * RN);
    dst[j] = s < RN ? src[s] : (uint32_t)0 - src[s - RN];
  }
}

/* res += d (*) b, negacyclic, all mod 2^32; d small signed, b torus words */
static void negacyclic_mac(uint32_t *res, const int32_t *d, const uint32_t *b) {
  for (int j = 0; j < RN; ++j) {
    const uint32_t dj = (uint32_t)d[j];
    if (!dj) continue;
    uint32_t *r = res + j;
    for (int m = 0; m < RN - j; ++m) r[m] += dj * b[m];
    const uint32_t *bw = b + (RN - j);
    for (int m = 0; m < j; ++m) res[m] -= dj * bw[m];
  }
}

/* gadget decomposition of one polynomial into BK_L digit polynomials */
static void decompose(const uint32_t *p, int32_t dec[BK_L][RN]) {
  uint32_t offset = 0;
  for (int l = 0; l < BK_L; ++l) offset += (uint32_t)(1u << (BGBIT - 1)) << (32 - (l + 1) * BGBIT);
  offset += 1u << (32 - BK_L * BGBIT - 1); /* round to the nearest multiple of Bg^-l instead of truncating */
  for (int j = 0; j < RN; ++j) {
    const uint32_t v = p[j] + offset;
    for (int l = 0; l < BK_L; ++l)
      dec[l][j] = (int32_t)((v >> (32 - (l + 1) * BGBIT)) & ((1u << BGBIT) - 1)) - (1 << (BGBIT - 1));
  }
}

/* ---- double-precision FFT path (like-for-like CPU comparator) ---- */
typedef struct { double re, im; } cplx;
static cplx g_tw[HN];     /* exp(2 pi i k / 512) */
static cplx g_twist[HN];  /* exp(i pi j / N) */
static cplx g_root[2 * RN]; /* exp(i pi m / N): X^e at spectral point f is g_root[e (1 + 4 f) mod 2N] */
static int g_fft_ready = 0;

static void fft_setup(void) {
  if (g_fft_ready) return;
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int k = 0; k < HN; ++k) {
    g_tw[k].re = (double)cosl(2 * pi * k / HN);
    g_tw[k].im = (double)sinl(2 * pi * k / HN);
    g_twist[k].re = (double)cosl(pi * k / RN);
    g_twist[k].im = (double)sinl(pi * k / RN);
  }
  for (int m = 0; m < 2 * RN; ++m) {
    g_root[m].re = (double)cosl(pi * m / RN);
    g_root[m].im = (double)sinl(pi * m / RN);
  }
  g_fft_ready = 1;
}

/* in-place radix-2 DIT, sign = +1 or -1, unnormalised */
static void fft512(cplx *a, int sign) {
  for (int i = 1, j = 0; i < HN; ++i) {
    int bit = HN >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) { cplx t = a[i]; a[i] = a[j]; a[j] = t; }
  }
  for (int len = 2; len <= HN; len <<= 1) {
    const int step = HN / len;
    for (int i = 0; i < HN; i += len)
      for (int k = 0; k < len / 2; ++k) {
        const cplx w = g_tw[k * step];
        const double wi = sign > 0 ? w.im : -w.im;
        cplx *u = a + i + k, *v = a + i + k + len / 2;
        const double tr = v->re * w.re - v->im * wi, ti = v->re * wi + v->im * w.re;
        v->re = u->re - tr; v->im = u->im - ti;
        u->re += tr; u->im += ti;
      }
  }
}

static void poly_to_spec(const int32_t *p, cplx *z) {
  for (int j = 0; j < HN; ++j) {
    const double a = (double)p[j], b = (double)p[j + HN];
    z[j].re = a * g_twist[j].re - b * g_twist[j].im;
    z[j].im = a * g_twist[j].im + b * g_twist[j].re;
  }
  fft512(z, +1);
}

static void spec_add_to_poly(cplx *z, uint32_t *p) {
  fft512(z, -1);
  for (int j = 0; j < HN; ++j) {
    const double re = (z[j].re * g_twist[j].re + z[j].im * g_twist[j].im) / HN;
    const double im = (z[j].im * g_twist[j].re - z[j].re * g_twist[j].im) / HN;
    p[j] += (uint32_t)(int64_t)llrint(re);
    p[j + HN] += (uint32_t)(int64_t)llrint(im);
  }
}

/* spectral copy of the bootstrapping key for the fft path: [pairs][BK_KEYS][ROWS][2][HN] */
cplx *oracle_bk_to_spectral(const int32_t *bk, int n) {
  fft_setup();
  const int64_t polys = (int64_t)((n + 1) / 2) * BK_KEYS * ROWS * 2;
  cplx *out = (cplx *)malloc((size_t)polys * HN * sizeof(cplx));
  for (int64_t q = 0; q < polys; ++q) poly_to_spec(bk + q * RN, out + q * HN);
  return out;
}
void oracle_free(void *p) { free(p); }

/* acc += (X^e - 1) * p, all mod 2^32 */
static void add_rotated_diff(uint32_t *acc, const uint32_t *p, int e) {
  uint32_t rot[RN];
  mul_by_xe(rot, p, e);
  for (int j = 0; j < RN; ++j) acc[j] += rot[j] - p[j];
}

/* Blind rotation + sample extract.  bar: n+1 mod-switched words (last = body).
 * bk: int32[(n+1)/2][BK_KEYS][ROWS][2][N], key 0 = TRGSW(s_{2m}), 1 = TRGSW(s_{2m+1}), 2 = TRGSW(s_{2m} s_{2m+1}).
 * bk_spec: NULL for the exact path.  ext: N+1 words. */
void oracle_blind_rotate(const int32_t *bar, int n, uint32_t mu, const int32_t *bk, const cplx *bk_spec,
                         uint32_t *ext) {
  uint32_t acc[2][RN], tv[RN];
  int32_t dec[ROWS][RN];
  for (int j = 0; j < RN; ++j) { acc[0][j] = 0; tv[j] = mu; }
  mul_by_xe(acc[1], tv, (2 * RN - bar[n]) % (2 * RN));
  for (int m = 0; 2 * m < n; ++m) {
    const int a1 = bar[2 * m], a2 = (2 * m + 1 < n) ? bar[2 * m + 1] : 0;
    if (a1 == 0 && a2 == 0) continue;
    for (int p = 0; p < 2; ++p) decompose(acc[p], &dec[p * BK_L]);
    if (!bk_spec) {
      for (int j = 0; j < BK_KEYS; ++j) {
        if ((j == 0 && a1 == 0) || (j == 1 && a2 == 0) || (j == 2 && (a1 == 0 || a2 == 0))) continue; /* factor is 0 */
        uint32_t prod[2][RN];
        memset(prod, 0, sizeof prod);
        for (int r = 0; r < ROWS; ++r)
          for (int c = 0; c < 2; ++c)
            negacyclic_mac(prod[c], dec[r], (const uint32_t *)bk + ((((size_t)m * BK_KEYS + j) * ROWS + r) * 2 + c) * RN);
        for (int c = 0; c < 2; ++c) {
          if (j < 2) {
            add_rotated_diff(acc[c], prod[c], j == 0 ? a1 : a2);
          } else { /* (X^a1 - 1)(X^a2 - 1) */
            uint32_t q[RN];
            memset(q, 0, sizeof q);
            add_rotated_diff(q, prod[c], a1);
            add_rotated_diff(acc[c], q, a2);
          }
        }
      }
    } else {
      static __thread cplx d[ROWS][HN], o[2][HN];
      for (int r = 0; r < ROWS; ++r) poly_to_spec(dec[r], d[r]);
      for (int f = 0; f < HN; ++f) {
        const cplx w1 = g_root[(a1 * (1 + 4 * f)) & (2 * RN - 1)], w2 = g_root[(a2 * (1 + 4 * f)) & (2 * RN - 1)];
        const cplx u1 = {w1.re - 1.0, w1.im}, u2 = {w2.re - 1.0, w2.im};
        const cplx u12 = {u1.re * u2.re - u1.im * u2.im, u1.re * u2.im + u1.im * u2.re};
        const cplx fac[BK_KEYS] = {u1, u2, u12};
        for (int c = 0; c < 2; ++c) {
          double sre = 0, sim = 0;
          for (int j = 0; j < BK_KEYS; ++j) {
            double pre = 0, pim = 0;
            for (int r = 0; r < ROWS; ++r) {
              const cplx *b = bk_spec + ((((size_t)m * BK_KEYS + j) * ROWS + r) * 2 + c) * HN;
              pre += d[r][f].re * b[f].re - d[r][f].im * b[f].im;
              pim += d[r][f].re * b[f].im + d[r][f].im * b[f].re;
            }
            sre += fac[j].re * pre - fac[j].im * pim;
            sim += fac[j].re * pim + fac[j].im * pre;
          }
          o[c][f].re = sre;
          o[c][f].im = sim;
        }
      }
      for (int c = 0; c < 2; ++c) spec_add_to_poly(o[c], acc[c]);
    }
  }
  ext[0] = acc[0][0];
  for (int j = 1; j < RN; ++j) ext[j] = (uint32_t)0 - acc[0][RN - j];
  ext[RN] = acc[1][0];
}

/* Key switch N -> n with signed base-4 digits.  ksk: int32[N][KS_T][n+1]. */
void oracle_key_switch(const uint32_t *ext, int n, const int32_t *ksk, uint32_t *out) {
  uint32_t bias = 1u << (32 - KS_T * KS_BB - 1);
  for (int j = 0; j < KS_T; ++j) bias += (uint32_t)(1u << (KS_BB - 1)) << (32 - (j + 1) * KS_BB);
  for (int w = 0; w < n; ++w) out[w] = 0;
  out[n] = ext[RN];
  for (int i = 0; i < RN; ++i) {
    const uint32_t a = ext[i] + bias;
    for (int j = 0; j < KS_T; ++j) {
      const int32_t d = (int32_t)((a >> (32 - (j + 1) * KS_BB)) & ((1u << KS_BB) - 1)) - (1 << (KS_BB - 1));
      if (!d) continue;
      const uint32_t *row = (const uint32_t *)ksk + ((size_t)i * KS_T + j) * (n + 1);
      for (int w = 0; w <= n; ++w) out[w] -= (uint32_t)d * row[w];
    }
  }
}

/* ---- batch driver: a plain pthread work queue over the k gates ---- */
typedef struct {
  const uint32_t *x, *y;
  const uint8_t *kinds;
  int64_t k;
  int n;
  uint32_t mu;
  const int32_t *bk, *ksk;
  const cplx *spec;
  uint32_t *out, *ext_out;
  int32_t *bar_out;
  int64_t next;
  pthread_mutex_t lock;
} batch_job;

static void one_gate(batch_job *jb, int64_t g) {
  uint32_t lin[RN + 1], ext[RN + 1];
  int32_t bar[RN + 1];
  const int n = jb->n;
  oracle_gate_linear(jb->x + g * (n + 1), jb->y + g * (n + 1), jb->kinds[g], jb->mu, n, lin);
  oracle_mod_switch(lin, n, bar);
  oracle_blind_rotate(bar, n, jb->mu, jb->bk, jb->spec, ext);
  oracle_key_switch(ext, n, jb->ksk, jb->out + g * (n + 1));
  if (jb->ext_out) memcpy(jb->ext_out + g * (RN + 1), ext, sizeof ext);
  if (jb->bar_out) memcpy(jb->bar_out + g * (n + 1), bar, (size_t)(n + 1) * 4);
}

static void *batch_worker(void *arg) {
  batch_job *jb = (batch_job *)arg;
  for (;;) {
    pthread_mutex_lock(&jb->lock);
    const int64_t g = jb->next++;
    pthread_mutex_unlock(&jb->lock);
    if (g >= jb->k) return NULL;
    one_gate(jb, g);
  }
}

int oracle_max_threads(void) {
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  return c > 0 ? (int)c : 1;
}

/* k gates.  x, y: [k][n+1] packed samples; out: [k][n+1]; ext_out (optional):
 * [k][N+1] extracted samples before the key switch; bar_out (optional): [k][n+1].
 * fft != 0 selects the double-precision path; threads <= 0 means all cores. */
void oracle_gate_bootstrap_batch(const uint32_t *x, const uint32_t *y, const uint8_t *kinds, int64_t k, int n,
                                 uint32_t mu, const int32_t *bk, const int32_t *ksk, int fft, int threads,
                                 uint32_t *out, uint32_t *ext_out, int32_t *bar_out) {
  cplx *spec = fft ? oracle_bk_to_spectral(bk, n) : NULL;
  batch_job jb = {x, y, kinds, k, n, mu, bk, ksk, spec, out, ext_out, bar_out, 0, PTHREAD_MUTEX_INITIALIZER};
  if (threads <= 0) threads = oracle_max_threads();
  if (threads > k) threads = (int)k;
  if (threads <= 1) {
    for (int64_t g = 0; g < k; ++g) one_gate(&jb, g);
  } else {
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, batch_worker, &jb);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    free(tid);
  }
  if (spec) free(spec);
}
