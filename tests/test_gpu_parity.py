"""CUDA path against the CPU oracle through the C ABI, stage by stage, bit-exact.

Integer / torus-word work: the bar is bit-exact.  The FP64 FFT inside kernel K1
is an implementation detail whose rounded output must equal the exact integer
product; the spectral key is compared with numpy within 1e-13 relative."""
import numpy as np
import pytest

from oracle import tfhe_oracle as orc

pytestmark = pytest.mark.gpu


def pack(s):
    return np.concatenate([s.a, [s.b]]).astype(np.uint32)


@pytest.fixture(scope="module")
def gpu(key, eval_keys):
    import torch

    from paper_2005_01945_b200 import _cabi

    ctx = _cabi.Context(0, key.params.m, key.params.mu.word, eval_keys.ring)
    ctx.call("tfb_load_keys", eval_keys.bk.ctypes.data, eval_keys.ksk.ctypes.data, 0, None)
    return ctx, torch, _cabi


def make_inputs(key, K, seed, kinds=None):
    from paper_2005_01945_b200 import encrypt_bit

    rng = np.random.default_rng((seed, 0))
    bits = np.random.default_rng((seed, 2)).integers(0, 2, size=(2, K))
    xs = np.stack([pack(encrypt_bit(key, int(b), rng)) for b in bits[0]])
    ys = np.stack([pack(encrypt_bit(key, int(b), rng)) for b in bits[1]])
    if kinds is None:
        kinds = (np.arange(K) % 8).astype(np.uint8)
    return xs, ys, kinds, bits


def run_launch(gpu, key, xs, ys, kinds, taps=False):
    ctx, torch, _cabi = gpu
    K, n = len(xs), key.params.m
    dev = torch.device("cuda:0")
    pool = torch.zeros((3 * K, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
    pool[:K, : n + 1] = torch.from_numpy(xs.view(np.int32)).to(dev)
    pool[K : 2 * K, : n + 1] = torch.from_numpy(ys.view(np.int32)).to(dev)
    kd = torch.from_numpy(kinds).to(dev)
    idx = torch.arange(0, 3 * K, dtype=torch.int32, device=dev)
    xr, yr, orow = idx[:K], idx[K : 2 * K], idx[2 * K :]
    if taps:
        ext = torch.zeros((K, _cabi.EXT_STRIDE), dtype=torch.int32, device=dev)
        ctx.call("tfb_debug_blind_rotate", pool.data_ptr(), kd.data_ptr(), xr.data_ptr(), yr.data_ptr(), ext.data_ptr(), K, None)
        ctx.call("tfb_debug_key_switch", ext.data_ptr(), pool.data_ptr(), orow.data_ptr(), K, None)
        torch.cuda.synchronize()
        return pool[2 * K :, : n + 1].cpu().numpy().view(np.uint32), ext.cpu().numpy().view(np.uint32)[:, :1025]
    ctx.call("tfb_gate_launch", pool.data_ptr(), kd.data_ptr(), xr.data_ptr(), yr.data_ptr(), orow.data_ptr(), K, None)
    torch.cuda.synchronize()
    return pool[2 * K :, : n + 1].cpu().numpy().view(np.uint32)


def test_spectral_key_matches_numpy(gpu, eval_keys):
    ctx, torch, _cabi = gpu
    N = 1024
    tw = np.exp(1j * np.pi * np.arange(N // 2) / N)
    for m, j in ((0, 0), (3, 1), (249, 2)):  # (pair of mask elements, key s1 / s2 / s1*s2)
        spec = np.empty((4, 2, 512, 2), dtype=np.float64)
        ctx.call("tfb_debug_spectral_key", m, j, spec.ctypes.data)
        poly = eval_keys.bk[m, j].astype(np.float64)
        want = np.fft.ifft((poly[..., : N // 2] + 1j * poly[..., N // 2 :]) * tw, axis=-1) * (N // 2)
        got = spec[..., 0] + 1j * spec[..., 1]
        assert np.abs(got - want).max() / np.abs(want).max() < 1e-13


def test_blind_rotate_and_key_switch_bit_exact(gpu, key, eval_keys):
    xs, ys, kinds, bits = make_inputs(key, 24, seed=31)
    want_out, want_ext = orc.gate_bootstrap_batch(xs, ys, kinds, key.params.mu.word, eval_keys.bk, eval_keys.ksk,
                                                  fft=True, want_ext=True)
    got_out, got_ext = run_launch(gpu, key, xs, ys, kinds, taps=True)
    assert np.array_equal(got_ext, want_ext)
    assert np.array_equal(got_out, want_out)
    # cross-check a few of the oracle's fft-path results with its exact integer path
    exact = orc.gate_bootstrap_batch(xs[:3], ys[:3], kinds[:3], key.params.mu.word, eval_keys.bk, eval_keys.ksk)
    assert np.array_equal(exact, want_out[:3])


def test_fused_launch_all_kinds_and_identity(gpu, key, eval_keys):
    K = 72
    kinds = (np.arange(K) % 9).astype(np.uint8)  # includes kind 8 = identity refresh
    xs, ys, kinds, bits = make_inputs(key, K, seed=32, kinds=kinds)
    want = orc.gate_bootstrap_batch(xs, ys, kinds, key.params.mu.word, eval_keys.bk, eval_keys.ksk, fft=True)
    got = run_launch(gpu, key, xs, ys, kinds)
    assert np.array_equal(got, want)


def test_host_buffer_entry_point(gpu, key, eval_keys):
    ctx, torch, _cabi = gpu
    xs, ys, kinds, bits = make_inputs(key, 40, seed=33)
    want = orc.gate_bootstrap_batch(xs, ys, kinds, key.params.mu.word, eval_keys.bk, eval_keys.ksk, fft=True)
    out = np.zeros_like(xs)
    ctx.call("tfb_gate_launch_host", xs.ctypes.data, ys.ctypes.data, kinds.ctypes.data, out.ctypes.data, len(xs))
    assert np.array_equal(out, want)
    # ragged second call reuses the buffers
    out2 = np.zeros_like(xs[:7])
    ctx.call("tfb_gate_launch_host", xs[:7].ctypes.data, ys[:7].ctypes.data, kinds[:7].ctypes.data, out2.ctypes.data, 7)
    assert np.array_equal(out2, want[:7])


def test_edge_inputs_trivial_and_aliased(gpu, key, eval_keys):
    p = key.params
    t1 = np.zeros(501, dtype=np.uint32); t1[-1] = p.message_word(1)
    t0 = np.zeros(501, dtype=np.uint32); t0[-1] = p.message_word(0)
    xs0, ys0, _, _ = make_inputs(key, 4, seed=34)
    xs = np.stack([t1, t0, xs0[0], t1, xs0[1], xs0[2]])
    ys = np.stack([t0, t0, t1, xs0[3], xs0[1], ys0[2]])  # job 4 feeds the same sample twice
    kinds = np.array([0, 1, 4, 6, 4, 5], dtype=np.uint8)
    want = orc.gate_bootstrap_batch(xs, ys, kinds, p.mu.word, eval_keys.bk, eval_keys.ksk, fft=True)
    got = run_launch(gpu, key, xs, ys, kinds)
    assert np.array_equal(got, want)
    assert not got[0, :-1].any() and int(got[0, -1]) == p.message_word(0)  # AND(1, 0) of trivials stays trivial


def test_every_kernel_variant_is_bit_exact(key, eval_keys, monkeypatch):
    """K1d (one gate per warp, twelve per CTA, TMA-staged key ring, tensor-memory parking), K1e (one gate per
    two-CTA cluster, key combiner warps, contributions exchanged through distributed shared memory) and the
    key-switch kernels (K2 direct / split with atomics on the IMAD pipe, K2t on the tensor cores) on the
    same jobs, with a gate count that leaves a ragged last CTA / a partial 128-gate tile."""
    import torch

    from paper_2005_01945_b200 import _cabi

    xs, ys, kinds, bits = make_inputs(key, 45, seed=36, kinds=(np.arange(45) % 9).astype(np.uint8))
    want = orc.gate_bootstrap_batch(xs, ys, kinds, key.params.mu.word, eval_keys.bk, eval_keys.ksk, fft=True)
    for variant, ks in (("4", "2"), ("4", "1"), ("5", "1"), ("5", "2")):
        monkeypatch.setenv("TFB_FORCE_KERNEL", variant)
        monkeypatch.setenv("TFB_FORCE_KS", ks)  # 1 = K2 (IMAD pipe), 2 = K2t (tcgen05.mma kind::i8)
        ctx = _cabi.Context(0, key.params.m, key.params.mu.word, eval_keys.ring)
        ctx.call("tfb_load_keys", eval_keys.bk.ctypes.data, eval_keys.ksk.ctypes.data, 0, None)
        got = run_launch((ctx, torch, _cabi), key, xs, ys, kinds)
        assert np.array_equal(got, want), f"kernel variant {variant}, key switch {ks}"
        ctx.close()


def test_k1d_cta_widths_are_bit_exact(key, eval_keys, monkeypatch):
    """K1d with 1 .. 12 gates per CTA (a mid-size launch is spread over all SMs with fewer warps per CTA; up to
    eight warps run the 255-register build of the same code): every width, both builds, ragged last CTA."""
    import torch

    from paper_2005_01945_b200 import _cabi

    xs, ys, kinds, bits = make_inputs(key, 29, seed=37, kinds=(np.arange(29) % 9).astype(np.uint8))
    want = orc.gate_bootstrap_batch(xs, ys, kinds, key.params.mu.word, eval_keys.bk, eval_keys.ksk, fft=True)
    monkeypatch.setenv("TFB_FORCE_KERNEL", "4")
    for warps, nomid in ((1, 0), (2, 0), (3, 1), (4, 0), (5, 0), (7, 1), (8, 0), (8, 1), (9, 0), (11, 0)):
        monkeypatch.setenv("TFB_K1D_W", str(warps))
        monkeypatch.setenv("TFB_K1D_NOMID", str(nomid))
        ctx = _cabi.Context(0, key.params.m, key.params.mu.word, eval_keys.ring)
        ctx.call("tfb_load_keys", eval_keys.bk.ctypes.data, eval_keys.ksk.ctypes.data, 0, None)
        got = run_launch((ctx, torch, _cabi), key, xs, ys, kinds)
        assert np.array_equal(got, want), f"{warps} gates per CTA, 168-register build forced: {nomid}"
        ctx.close()


def test_planned_segments_are_bit_exact(gpu, key, eval_keys):
    """A launch the dispatch splits into a K1d wave of narrow CTAs plus a cluster-kernel tail (700 gates on 148
    SMs) gives the same words as the oracle, segment boundaries included."""
    from paper_2005_01945_b200 import _cabi

    k = 700
    segs = _cabi.plan_kernels(k, 148)
    xs0, ys0, kinds0, _ = make_inputs(key, 20, seed=38, kinds=(np.arange(20) % 9).astype(np.uint8))
    want0 = orc.gate_bootstrap_batch(xs0, ys0, kinds0, key.params.mu.word, eval_keys.bk, eval_keys.ksk, fft=True)
    idx = np.arange(k) % 20
    got = run_launch(gpu, key, xs0[idx], ys0[idx], kinds0[idx])
    assert np.array_equal(got, want0[idx]), segs


def test_regrouped_launch_with_trivial_inputs(key, eval_keys, monkeypatch):
    """Launches of 4 x SMs gates and more are regrouped on the device: gates whose two inputs are trivial (zero
    masks) go behind the real ones, their extracted samples are written directly and K1d CTAs that hold only such
    gates return at once.  A third of the gates trivial, interleaved, scattered output rows, one gate writing over
    its own input row: every output word equals the oracle's and the launch with regrouping switched off."""
    import torch

    from paper_2005_01945_b200 import _cabi

    p, n = key.params, key.params.m
    xs0, ys0, kinds0, _ = make_inputs(key, 10, seed=39, kinds=(np.arange(10) % 9).astype(np.uint8))
    triv = np.zeros((2, n + 1), np.uint32)
    triv[0, -1], triv[1, -1] = p.message_word(0), p.message_word(1)
    base_x = np.concatenate([xs0, triv[[0, 1, 0, 1, 1, 0]]])
    base_y = np.concatenate([ys0, triv[[0, 0, 1, 1, 0, 1]]])
    base_k = np.concatenate([kinds0, np.array([0, 1, 2, 4, 7, 8], np.uint8)])
    want = orc.gate_bootstrap_batch(base_x, base_y, base_k, p.mu.word, eval_keys.bk, eval_keys.ksk, fft=True)
    dev = torch.device("cuda:0")
    for K in (1000, 2100):
        sel = np.where(np.arange(K) % 3 == 1, 10 + np.arange(K) % 6, np.arange(K) % 10)
        outs = {}
        for no_regroup in ("1", "0"):
            monkeypatch.setenv("TFB_NO_REGROUP", no_regroup)
            ctx = _cabi.Context(0, n, p.mu.word, eval_keys.ring)
            ctx.call("tfb_load_keys", eval_keys.bk.ctypes.data, eval_keys.ksk.ctypes.data, 0, None)
            pool = torch.zeros((3 * K, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
            pool[:K, : n + 1] = torch.from_numpy(base_x[sel].view(np.int32)).to(dev)
            pool[K : 2 * K, : n + 1] = torch.from_numpy(base_y[sel].view(np.int32)).to(dev)
            kd = torch.from_numpy(base_k[sel]).to(dev)
            xr = torch.arange(0, K, dtype=torch.int32, device=dev)
            yr = torch.arange(K, 2 * K, dtype=torch.int32, device=dev)
            orow = (3 * K - 1 - torch.arange(0, K, dtype=torch.int32, device=dev)).contiguous()  # scattered, reversed
            orow[5] = 5  # gate 5 overwrites its own x row
            ctx.call("tfb_gate_launch", pool.data_ptr(), kd.data_ptr(), xr.data_ptr(), yr.data_ptr(), orow.data_ptr(), K, None)
            torch.cuda.synchronize()
            first = pool[orow.long(), : n + 1].cpu().numpy().view(np.uint32)
            # again into fresh rows (the regrouping scratch is reused); row 5 now holds an output, so skip gate 5
            orow2 = (torch.arange(0, K, dtype=torch.int32, device=dev) + 2 * K).contiguous()
            ctx.call("tfb_gate_launch", pool.data_ptr(), kd.data_ptr(), xr.data_ptr(), yr.data_ptr(), orow2.data_ptr(), K, None)
            torch.cuda.synchronize()
            second = pool[orow2.long(), : n + 1].cpu().numpy().view(np.uint32)
            outs[no_regroup] = (first, second)
            ctx.close()
        ok_rows = np.arange(K) != 5
        assert np.array_equal(outs["1"][0], want[sel]), K
        assert np.array_equal(outs["0"][0], outs["1"][0]), K
        assert np.array_equal(outs["0"][1][ok_rows], want[sel][ok_rows]), K
        idle = sel >= 10
        assert not outs["0"][0][idle, :-1].any()  # two trivial inputs give a trivial output


def test_key_switch_on_tensor_cores_is_exact(key, eval_keys, monkeypatch):
    """K2t (tcgen05.mma kind::i8: digits x byte planes of the key, s32 accumulators in tensor memory)
    against K2 (IMAD pipe) on arbitrary extracted samples, whole and partial 128-gate tiles, and against
    the key-switch formula itself: out = (0, b) - sum_r d_r * KSK_r with signed base-4 digits."""
    import torch

    from paper_2005_01945_b200 import _cabi

    n = key.params.m
    dev = torch.device("cuda:0")
    ctxs = {}
    for mode in ("1", "2"):
        monkeypatch.setenv("TFB_FORCE_KS", mode)
        ctxs[mode] = _cabi.Context(0, n, key.params.mu.word, eval_keys.ring)
        ctxs[mode].call("tfb_load_keys", eval_keys.bk.ctypes.data, eval_keys.ksk.ctypes.data, 0, None)
    rng = np.random.default_rng(41)
    ksk = eval_keys.ksk.reshape(-1, n + 1).view(np.uint32)  # [N*t][n+1]
    for K in (1, 95, 128, 129, 700):
        ext_h = rng.integers(0, 1 << 32, size=(K, _cabi.EXT_STRIDE), dtype=np.uint32)
        ext_h[0, :1024] = 0                      # all-zero mask: digits of the rounding bias only
        ext_h[K - 1, :1024] = 0xFFFFFFFF         # carries through every digit
        ext = torch.from_numpy(ext_h.view(np.int32)).to(dev)
        rows = torch.arange(K, dtype=torch.int32, device=dev).flip(0).contiguous()  # scattered output rows
        outs = {}
        for mode, ctx in ctxs.items():
            pool = torch.full((K, _cabi.ROW_STRIDE), 7, dtype=torch.int32, device=dev)
            ctx.call("tfb_debug_key_switch", ext.data_ptr(), pool.data_ptr(), rows.data_ptr(), K, None)
            torch.cuda.synchronize()
            outs[mode] = pool.cpu().numpy().view(np.uint32)
        assert np.array_equal(outs["1"][:, : n + 1], outs["2"][:, : n + 1]), K
        for g in (0, K // 2, K - 1):             # the formula, in numpy
            a = ext_h[g, :1024].astype(np.uint64)
            bias = (1 << 15) + sum(2 << (32 - 2 * (j + 1)) for j in range(8))
            ab = (a + bias) % (1 << 32)
            digits = np.stack([((ab >> (32 - 2 * (j + 1))) & 3).astype(np.int64) - 2 for j in range(8)], axis=1).reshape(-1)
            want = (-(digits[:, None] * ksk.astype(np.int64)).sum(axis=0)) % (1 << 32)
            want[n] = (want[n] + int(ext_h[g, 1024])) % (1 << 32)
            assert np.array_equal(outs["2"][int(rows[g].item()), : n + 1].astype(np.int64), want), (K, g)
    # K2n, the narrow-launch kernel (partial sums combined by atomics in a self-cleaning scratch, last CTA writes
    # the rows): every group shape up to its 32-gate limit, twice in a row (the scratch must come back clean)
    monkeypatch.setenv("TFB_FORCE_KS", "3")
    ctxs["3"] = _cabi.Context(0, n, key.params.mu.word, eval_keys.ring)
    ctxs["3"].call("tfb_load_keys", eval_keys.bk.ctypes.data, eval_keys.ksk.ctypes.data, 0, None)
    for K in (1, 2, 7, 8, 9, 16, 17, 29, 32, 33, 64, 95, 3):
        ext_h = rng.integers(0, 1 << 32, size=(K, _cabi.EXT_STRIDE), dtype=np.uint32)
        ext_h[K - 1, :1024] = 0xFFFFFFFF
        ext = torch.from_numpy(ext_h.view(np.int32)).to(dev)
        rows = torch.arange(K, dtype=torch.int32, device=dev).flip(0).contiguous()
        outs = {}
        for mode in ("1", "3", "3 again"):
            pool = torch.full((K, _cabi.ROW_STRIDE), 7, dtype=torch.int32, device=dev)
            ctxs[mode[0]].call("tfb_debug_key_switch", ext.data_ptr(), pool.data_ptr(), rows.data_ptr(), K, None)
            torch.cuda.synchronize()
            outs[mode] = pool.cpu().numpy().view(np.uint32)
        assert np.array_equal(outs["1"][:, : n + 1], outs["3"][:, : n + 1]), K
        assert np.array_equal(outs["3"], outs["3 again"]), K
        assert (outs["3"][:, n + 1 :] == 7).all()  # nothing outside the n + 1 words of a row is written
    for ctx in ctxs.values():
        ctx.close()


@pytest.mark.parametrize("n", [7, 510])
def test_other_lwe_dimensions_through_the_host_path(n, monkeypatch):
    """A small odd and the largest LWE dimension the library accepts (rows of n + 2 <= 512 words), every
    K1 / K2 variant and the automatic split dispatch, through tfb_gate_launch_host (packed rows)."""
    from paper_2005_01945_b200 import LweParams, _cabi, generate_evaluation_keys, keygen

    p = LweParams(m=n)
    k = keygen(p, seed=3)
    ek = generate_evaluation_keys(k, seed=3)
    K = 8
    xs, ys, kinds, _ = make_inputs(k, K, seed=8, kinds=(np.arange(K) % 8).astype(np.uint8))
    want = orc.gate_bootstrap_batch(xs, ys, kinds, p.mu.word, ek.bk, ek.ksk, fft=True)
    for which, ks, count in (("5", "1", 8), ("5", "2", 200), ("4", "2", 200), ("4", "1", 13), (None, None, 3000)):
        for name, val in (("TFB_FORCE_KERNEL", which), ("TFB_FORCE_KS", ks)):
            monkeypatch.setenv(name, val) if val else monkeypatch.delenv(name, raising=False)
        ctx = _cabi.Context(0, n, p.mu.word, ek.ring)
        ctx.call("tfb_load_keys", ek.bk.ctypes.data, ek.ksk.ctypes.data, 0, None)
        idx = np.arange(count) % K
        xh, yh, kh = (np.ascontiguousarray(a[idx]) for a in (xs, ys, kinds))
        out = np.zeros((count, n + 1), dtype=np.uint32)
        ctx.call("tfb_gate_launch_host", xh.ctypes.data, yh.ctypes.data, kh.ctypes.data, out.ctypes.data, count)
        assert np.array_equal(out, want[idx]), (n, which, ks, count)
        ctx.close()


def test_automatic_dispatch_sizes(gpu, key, eval_keys):
    """Launch sizes on both sides of the K1e / K1d dispatch threshold and of a full K1d wave (12 x SMs)."""
    base = 64
    xs, ys, kinds, bits = make_inputs(key, base, seed=37)
    want = orc.gate_bootstrap_batch(xs, ys, kinds, key.params.mu.word, eval_keys.bk, eval_keys.ksk, fft=True)
    for K in (1, 2, 33, 297, 400, 889, 1030, 1775, 1777, 1800, 2500, 4096):
        idx = np.arange(K) % base
        got = run_launch(gpu, key, xs[idx], ys[idx], kinds[idx])
        assert np.array_equal(got, want[idx]), K


def test_invalid_calls_return_status(gpu):
    ctx, torch, _cabi = gpu
    with pytest.raises(_cabi.TfbError):
        ctx.call("tfb_gate_launch", None, None, None, None, None, 4, None)
    with pytest.raises(_cabi.TfbError):
        ctx.call("tfb_gate_launch_host", None, None, None, None, 0)


def test_full_size_launch_properties(gpu, key, eval_keys):
    """2**16 gates in one launch (BASELINE configs[1]): every output decrypts to
    its truth table, every phase sits within the reference's fresh bound of
    +-mu, and 2,048+ spread rows equal the oracle bit for bit."""
    ctx, torch, _cabi = gpu
    K, n = 1 << 16, key.params.m
    base = 256
    xs, ys, kinds, bits = make_inputs(key, base, seed=35)
    dev = torch.device("cuda:0")
    rep = torch.arange(K, device=dev) % base
    pool = torch.zeros((3 * K, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
    pool[:K, : n + 1] = torch.from_numpy(xs.view(np.int32)).to(dev)[rep]
    # pair x_g with y_{(g // base + g) % base} so the 2**16 jobs are distinct combinations
    yidx = (torch.arange(K, device=dev) // base + torch.arange(K, device=dev)) % base
    pool[K : 2 * K, : n + 1] = torch.from_numpy(ys.view(np.int32)).to(dev)[yidx]
    kd = (torch.arange(K, device=dev) % 8).to(torch.uint8)
    idx = torch.arange(0, 3 * K, dtype=torch.int32, device=dev)
    ctx.call("tfb_gate_launch", pool.data_ptr(), kd.data_ptr(), idx[:K].data_ptr(), idx[K : 2 * K].data_ptr(),
             idx[2 * K :].data_ptr(), K, None)
    kb = torch.from_numpy(key.bits.astype(np.uint32).view(np.int32)).to(dev)
    ph = torch.empty(K, dtype=torch.int32, device=dev)
    ctx.call("tfb_rows_phase", pool.data_ptr(), idx[2 * K :].data_ptr(), kb.data_ptr(), ph.data_ptr(), K, None)
    torch.cuda.synchronize()
    phase = ph.cpu().numpy().view(np.uint32).astype(np.int64)
    from paper_2005_01945_b200.engine import TWO_INPUT_KINDS, truth_table

    g = np.arange(K)
    bx, by = bits[0][g % base], bits[1][(g // base + g) % base]
    tt = np.array([truth_table(k) for k in TWO_INPUT_KINDS])
    want_bit = tt[g % 8, (bx << 1) | by]
    got_bit = ((phase > 0) & (phase < 2**31)).astype(np.int64)
    assert np.array_equal(got_bit, want_bit)
    target = np.where(want_bit == 1, 1 << 29, (1 << 32) - (1 << 29))
    err = ((phase - target + 2**31) % 2**32) - 2**31
    assert np.abs(err).max() < (1 << 27)  # fresh_noise_bound = 2**-5 (encirc/torus.py:177-184)
    # bit-exact against the oracle on 2,048+ rows spread over the whole launch (first / last rows, wave and CTA
    # boundaries of the 12-gates-per-SM kernel, and a stride that is coprime to every tile size)
    edge = [0, 1, 11, 12, 255, 256, 1775, 1776, 4097, 14207, 14208, 63935, 63936, 65534, 65535]
    sel = np.unique(np.concatenate([edge, (np.arange(2048) * 32003 + 17) % K]))
    assert len(sel) >= 2048
    sx = xs[sel % base]
    sy = ys[(sel // base + sel) % base]
    want = orc.gate_bootstrap_batch(sx, sy, (sel % 8).astype(np.uint8), key.params.mu.word, eval_keys.bk,
                                    eval_keys.ksk, fft=True)
    got = pool[2 * K + torch.from_numpy(sel).to(dev), : n + 1].cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want)
