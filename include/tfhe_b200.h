/* tfhe_b200.h -- C ABI of the B200 gate-bootstrapping library (libtfhe_b200.so).
 *
 * This is the drop-in boundary for the reference's gate-evaluation hot path.
 * The reference is pure Python and has no FFI; the hooks this ABI serves are
 * the six `GateEngine` hooks of /root/reference/pkg/src/encirc/engine.py:322-340
 * (`trivial_bit`, `encrypt`, `decrypt`, `bootstrap`, `_negate`,
 * `execute_launch`), of which only `execute_launch` / `bootstrap` / `_negate`
 * touch ciphertext words in bulk.  Each entry point below names the reference
 * lines it replaces.  INTEGRATION.md shows the ctypes stub a reference
 * maintainer would add.
 *
 * Conventions: plain C types only; every function returns a tfb_status;
 * pointers named *_dev are CUDA device pointers on the context's device,
 * pointers named *_host are host pointers (pinned memory makes the copies
 * asynchronous but is not required); `stream` is a cudaStream_t passed as
 * void* (NULL = the legacy default stream).  Nothing throws across the ABI.
 *
 * Threading: like the reference's engine (single driver thread, encirc/scheduler.py:173-179) a context is driven
 * by one thread at a time, and its gate launches must be ordered on ONE stream at a time: the scratch between the
 * fused bootstrap and the key switch (extracted samples, the partial sums of narrow launches) belongs to the context.
 * Use one context per stream / per device for concurrent work.
 *
 * Ciphertext layout: one LWE sample is n mask words followed by one body word
 * (uint32, torus 2^-32 fixed point; encirc/torus.py:190-203).  In the device
 * pool a sample occupies one row of TFB_ROW_STRIDE words (the tail is padding);
 * host buffers are packed [k][n+1].
 */
#ifndef TFHE_B200_H
#define TFHE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TFB_ABI_VERSION 2
#define TFB_ROW_STRIDE 512  /* uint32 words per pool row */
#define TFB_EXT_STRIDE 1032 /* uint32 words per extracted (N+1)-word sample */

typedef enum tfb_status {
  TFB_OK = 0,
  TFB_ERR_INVALID = 1, /* bad argument or unsupported parameter set */
  TFB_ERR_CUDA = 2,    /* a CUDA runtime call failed; see tfb_last_error */
  TFB_ERR_STATE = 3    /* call order violated (e.g. launch before keys) */
} tfb_status;

/* Gate kind ids: index into TWO_INPUT_KINDS (encirc/engine.py:77-88). */
enum {
  TFB_AND = 0, TFB_OR = 1, TFB_NAND = 2, TFB_NOR = 3,
  TFB_XOR = 4, TFB_XNOR = 5, TFB_ANDNY = 6, TFB_ORNY = 7,
  TFB_IDENTITY = 8 /* refresh x alone: GateEngine.bootstrap, encirc/engine.py:436-450 */
};

/* Parameter set.  LWE side from encirc/torus.py:25-27,118-134; ring side is the
 * builder's choice (the reference has none) and only this set is compiled:
 * ring_n 1024, bk_l 2, bk_bgbit 9, ks_t 8, ks_basebit 2, bootstrapping key unrolled
 * over pairs of mask elements (three TRGSW samples per pair). */
typedef struct tfb_params {
  int32_t n;          /* LWE dimension m (<= 510) */
  int32_t ring_n;     /* TRLWE degree N */
  int32_t bk_l;       /* gadget length */
  int32_t bk_bgbit;   /* log2 gadget base */
  int32_t ks_t;       /* key-switch digits */
  int32_t ks_basebit; /* log2 key-switch base */
  uint32_t mu_word;   /* message offset mu as a torus word (2^29 for 1/8) */
} tfb_params;

typedef struct tfb_ctx tfb_ctx;

int tfb_abi_version(void);
const char *tfb_last_error(const tfb_ctx *ctx); /* ctx may be NULL: last creation error */

/* One context per GPU: owns the spectral bootstrapping key, the key-switching
 * key, twiddle tables and scratch.  Replaces OracleBootstrapEngine.__init__'s
 * key capture (encirc/engine.py:419-424). */
int tfb_ctx_create(int device, const tfb_params *params, tfb_ctx **out);
void tfb_ctx_destroy(tfb_ctx *ctx);

/* Key setup (kernel K3).  bk: int32[ceil(n/2)][3][4][2][N] raw TRGSW rows (pair of mask
 * elements, key s1 / s2 / s1*s2, row, component), ksk: int32[N][8][n+1] raw LWE rows
 * (layouts in paper_2005_01945_b200/keys.py).
 * on_device != 0 means both pointers are device pointers (e.g. the receive
 * buffers of an NCCL broadcast).  Transforms bk to the FFT domain in the
 * kernel's register order and lays ksk out row-padded for coalesced loads. */
int tfb_load_keys(tfb_ctx *ctx, const int32_t *bk, const int32_t *ksk, int on_device, void *stream);

/* The hot path: k independent bootstrapped gates as one launch sequence
 * (fused linear form + blind rotation + sample extract kernel, then the
 * batched key-switch kernel).  Replaces OracleBootstrapEngine.execute_launch,
 * encirc/engine.py:458-514.  kinds/x_rows/y_rows/out_rows are device arrays of
 * length k; rows index pool_dev in units of TFB_ROW_STRIDE words.  Output rows
 * must not alias input rows of the same launch. */
int tfb_gate_launch(tfb_ctx *ctx, void *pool_dev, const uint8_t *kinds_dev, const int32_t *x_rows_dev,
                    const int32_t *y_rows_dev, const int32_t *out_rows_dev, int64_t k, void *stream);

/* Same launch with HOST buffers: packed samples x/y [k][n+1], kinds [k], packed
 * outputs [k][n+1].  Copies in, runs the launch, copies out, synchronises. */
int tfb_gate_launch_host(tfb_ctx *ctx, const uint32_t *x_host, const uint32_t *y_host,
                         const uint8_t *kinds_host, uint32_t *out_host, int64_t k);

/* NOT: out = -in on every word (encirc/engine.py:452-456). */
int tfb_rows_negate(tfb_ctx *ctx, void *pool_dev, const int32_t *in_rows_dev, const int32_t *out_rows_dev,
                    int64_t k, void *stream);

/* phase_dev[i] = b - <a, s> for the given rows; key_bits_dev is uint32[n] of
 * 0/1 (encirc/torus.py:283-288).  Used by batched decryption. */
int tfb_rows_phase(tfb_ctx *ctx, const void *pool_dev, const int32_t *rows_dev, const uint32_t *key_bits_dev,
                   uint32_t *phase_dev, int64_t k, void *stream);

/* Batched fresh encryption on the device (encirc/torus.py:254-271 restated for a counter-based generator):
 * for i < k, row out_rows_dev[i] <- (a, b) with a uniform in Z_2^32^n from Philox4x32-10 keyed by `seed` at counter
 * (first_sample + i, word index), e = rint(N(0, alpha) * 2^32) clipped to +-(2^27 - 1) like the reference's
 * gaussian_noise_words, b = <a, s> + message(bits_dev[i]) + e.  The draw ORDER differs from numpy's PCG64 stream, so
 * words are not those of the reference for the same seed; the host path of the Python engine keeps that identity.
 * Deterministic in (seed, first_sample). */
int tfb_rows_encrypt(tfb_ctx *ctx, void *pool_dev, const int32_t *out_rows_dev, const uint8_t *bits_dev,
                     const uint32_t *key_bits_dev, double alpha, uint64_t seed, uint64_t first_sample, int64_t k,
                     void *stream);

/* Parity taps: the two halves of tfb_gate_launch run separately so tests can
 * compare the intermediate (N+1)-word extracted sample with the oracle. */
int tfb_debug_blind_rotate(tfb_ctx *ctx, const void *pool_dev, const uint8_t *kinds_dev,
                           const int32_t *x_rows_dev, const int32_t *y_rows_dev, uint32_t *ext_dev /* [k][TFB_EXT_STRIDE] */,
                           int64_t k, void *stream);
int tfb_debug_key_switch(tfb_ctx *ctx, const uint32_t *ext_dev, void *pool_dev, const int32_t *out_rows_dev,
                         int64_t k, void *stream);
/* Spectral key `key` (0: s1, 1: s2, 2: s1*s2) of mask-element pair `pair`, de-permuted to
 * natural frequency order and un-scaled: double[4][2][512][2] (row, component, frequency, re/im). */
int tfb_debug_spectral_key(tfb_ctx *ctx, int32_t pair, int32_t key, double *out_host);

/* K1 dispatch, host logic only (no GPU needed): the kernel launches a fused bootstrap of k gates is split
 * into on a device with `sms` multiprocessors.  Segment i covers gates[i] consecutive gates and runs as
 * variants[i] = 4 (K1d, one gate per warp, warps[i] = 1..12 gates per CTA: throughput) or 5 (K1e, one gate per
 * two-CTA cluster: latency; warps[i] = 0).  Returns the number of segments (at most 6); arrays may be NULL. */
int tfb_debug_plan_kernels(int64_t k, int sms, int32_t *variants, int32_t *warps, int64_t *gates, int max_segments);

/* Number of kernels this context has launched so far (bench `gpu_launches`). */
int64_t tfb_kernel_launches(const tfb_ctx *ctx);

/* Roofline denominators measured on the spot: dependent-free DFMA and IMAD
 * loops over the whole chip; TFLOP/s (2 flops per FMA) and TOP/s. */
int tfb_measure_peaks(int device, double *fp64_tflops, double *int32_tops);

#ifdef __cplusplus
}
#endif
#endif /* TFHE_B200_H */
