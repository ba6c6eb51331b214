"""GPU parity: the CUDA path (libcbp_cuda.so through the C ABI) against the FP64 oracle on
identical FP32 inputs, plus the reference's error behaviour.

Tolerances (BASELINE.md "Correctness gates", floating point):
  kernel   relative L2 <= 1e-5 after the sum-to-1 normalisation;
  latent   max-abs <= 1e-4 and PSNR(gpu, oracle) >= 90 dB;
  truth    PSNR(gpu, ground-truth latent) >= 40 dB (acceptance.cpp:78);
  widths / clamped flags / error codes exact; GPU encode bit-exact.
"""
import glob
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KREL = 1e-5
LMAX = 1e-4
LPSNR = 90.0

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1203_4874_b200 import api as A
    torch.cuda.set_device(0)
    return A


def make(oracle, rows, cols, ch, t, lseed, pseed):
    lat = oracle.random_frame(rows, cols, ch, lseed)
    pair = oracle.generate_coprime_pair(t, pseed)
    pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
    return lat, pair, pub.astype(np.float32), prv.astype(np.float32)


def krel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def check_decode(oracle, api, lat, pub, prv, lo, hi, hint=None, trust=False, epsilon=None):
    cfg_o = oracle.make_cfg(lo, hi, trust_hint=trust, epsilon=epsilon)
    ref = oracle.decode_frame(pub.astype(np.float64), prv.astype(np.float64), hint=hint, cfg=cfg_o)
    d = api.decode_frame(torch.from_numpy(pub).cuda(), torch.from_numpy(prv).cuda(), hint=hint,
                         cfg=api.make_cfg(lo, hi, trust_hint=trust, epsilon=epsilon))
    got = d.latent.cpu().numpy().astype(np.float64)
    assert d.width_used == ref.width_used and d.width_clamped == ref.width_clamped
    assert krel(d.kernel_estimate, ref.kernel) <= KREL
    assert got.shape == ref.latent.shape
    assert np.abs(got - ref.latent).max() <= LMAX
    assert oracle.psnr(ref.latent, got) >= LPSNR
    assert abs(d.validation_residual - ref.validation_residual) <= 1e-6
    assert abs(d.epsilon_used - ref.epsilon_used) <= 1e-12
    if lat is not None:
        assert oracle.psnr(lat, got) >= 40.0
    return d, ref


# ------------------------------------------------------------------ decode_frame
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p) for p in FIXTURES])
def test_golden_fixtures(oracle, api, path):
    g = np.load(path)
    lat, pair, pub, prv = make(oracle, int(g["rows"]), int(g["cols"]), int(g["channels"]), int(g["t"]),
                               int(g["latent_seed"]), int(g["pair_seed"]))
    d = api.decode_frame(torch.from_numpy(pub).cuda(), torch.from_numpy(prv).cuda(),
                         cfg=api.make_cfg(int(g["search_min"]), int(g["search_max"])))
    got = d.latent.cpu().numpy()
    assert d.width_used == int(g["t"])
    assert krel(d.kernel_estimate, g["kernel"]) <= KREL
    assert np.abs(got - g["latent"]).max() <= LMAX
    assert oracle.psnr(g["latent"].astype(np.float64), got.astype(np.float64)) >= LPSNR
    assert abs(d.validation_residual - float(g["validation_residual"])) <= 1e-6


@pytest.mark.parametrize("rows,cols,ch,t,lo,hi,hint,trust", [
    (64, 64, 1, 5, 3, 9, None, False),       # decoder_test.cpp:311 round trip
    (64, 64, 1, 5, 3, 9, 5, True),           # trusted hint
    (48, 40, 1, 5, 3, 9, None, False),       # non-square
    (24, 24, 3, 3, 3, 7, None, False),       # RGB via luma
    (96, 96, 1, 9, 3, 9, None, False),
    (128, 128, 1, 13, 9, 25, None, False),
    (256, 256, 1, 7, 3, 25, None, False),    # BASELINE config 1
    (480, 640, 1, 9, 3, 25, None, False),    # BASELINE config 2 frame
    (101, 67, 1, 7, 3, 25, None, False),     # odd grids (generic FFT path)
])
def test_decode_frame_parity(oracle, api, rows, cols, ch, t, lo, hi, hint, trust):
    lat, pair, pub, prv = make(oracle, rows, cols, ch, t, oracle.frame_seed(1, rows + t), oracle.frame_seed(2, cols + t))
    d, _ = check_decode(oracle, api, lat, pub, prv, lo, hi, hint=hint, trust=trust)
    assert krel(d.kernel_estimate, pair.k1) <= 1e-4


@pytest.mark.parametrize("rows,cols,ch,t,lo,hi", [
    (64, 64, 1, 5, 3, 9),
    (61, 97, 3, 7, 3, 25),     # RGB, odd extents (prime factors 61, 97 in the axis DFTs)
    (96, 128, 1, 9, 3, 25),
])
def test_decode_signed_content_parity(oracle, api, rows, cols, ch, t, lo, hi):
    """Signed latents: width estimation takes the maximum-energy axis_spectrum_half slices
    (decoder.cpp:65-82) instead of the DC sums."""
    lat = oracle.random_frame(rows, cols, ch, oracle.frame_seed(3, rows + t)) - 0.5
    pair = oracle.generate_coprime_pair(t, oracle.frame_seed(4, cols + t))
    pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
    pub, prv = pub.astype(np.float32), prv.astype(np.float32)
    w = api.estimate_kernel_width(torch.from_numpy(pub).cuda(), torch.from_numpy(prv).cuda(), lo, hi, 1e-6)
    ref_w = oracle.estimate_kernel_width(pub.astype(np.float64), prv.astype(np.float64), lo, hi, 1e-6)
    assert w == ref_w == (t, False)
    d, _ = check_decode(oracle, api, lat, pub, prv, lo, hi)
    assert krel(d.kernel_estimate, pair.k1) <= 1e-4


def test_decode_1080p_rgb_parity(oracle, api):
    """BASELINE config 3 frame at full size: 1920x1080 RGB, t = 11."""
    lat, pair, pub, prv = make(oracle, 1080, 1920, 3, 11, oracle.frame_seed(1, 0), oracle.frame_seed(2, 0))
    check_decode(oracle, api, lat, pub, prv, 9, 25)


def test_decode_4k_parity(oracle, api):
    """BASELINE config 4 frame at full size: 3840x2160 gray, t = 15 (trusted hint)."""
    lat, pair, pub, prv = make(oracle, 2160, 3840, 1, 15, oracle.frame_seed(1, 4), oracle.frame_seed(2, 4))
    check_decode(oracle, api, lat, pub, prv, 9, 25, hint=15, trust=True)


def test_decode_exact_epsilon_and_swap(oracle, api):
    lat, pair, pub, prv = make(oracle, 32, 32, 1, 3, 145, 145)
    d, _ = check_decode(oracle, api, lat, pub, prv, 3, 7, epsilon=1e-12)
    s, _ = check_decode(oracle, api, lat, prv, pub, 3, 7, epsilon=1e-12)
    assert np.abs(d.kernel_estimate - pair.k1).max() <= 1e-6
    assert np.abs(s.kernel_estimate - pair.k2).max() <= 1e-6


def test_decode_batch_equals_single(oracle, api):
    frames = [make(oracle, 72, 80, 1, 5, oracle.frame_seed(7, i), oracle.frame_seed(8, i)) for i in range(4)]
    P = torch.from_numpy(np.stack([f[2] for f in frames])).cuda()
    Q = torch.from_numpy(np.stack([f[3] for f in frames])).cuda()
    cfg = api.make_cfg(3, 9)
    batch = api.decode_frames(P, Q, cfg=cfg)
    for i, f in enumerate(frames):
        one = api.decode_frame(P[i], Q[i], cfg=cfg)
        assert batch[i].width_used == one.width_used == 5
        assert np.array_equal(batch[i].kernel_estimate, one.kernel_estimate)
        assert torch.equal(batch[i].latent, one.latent)


def test_decode_u16_quantized(oracle, api):
    lat = oracle.random_mat(48, 48, 153)
    pair = oracle.generate_coprime_pair(5, 153)
    pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
    pub = oracle.quantize(pub, 16).astype(np.float32)
    prv = oracle.quantize(prv, 16).astype(np.float32)
    d, _ = check_decode(oracle, api, None, pub, prv, 3, 9, hint=5, trust=True)
    assert oracle.psnr(lat, d.latent[0].cpu().numpy().astype(np.float64)) >= 40.0


# ----------------------------------------------------------------- spectral_deblur
@pytest.mark.parametrize("rows,cols,t,ch", [(16, 16, 3, 1), (24, 24, 3, 1), (61, 97, 7, 1), (480, 640, 9, 1),
                                            (256, 256, 7, 2), (1080, 1920, 11, 3), (2160, 3840, 15, 1)])
def test_spectral_deblur_parity(oracle, api, rows, cols, t, ch):
    chn = 3 if ch == 3 else 1
    lat, pair, pub, _ = make(oracle, rows, cols, chn, t, oracle.frame_seed(3, rows), oracle.frame_seed(4, cols))
    ref = np.stack([oracle.spectral_deblur(pub[k].astype(np.float64), pair.k1, 1e-8) for k in range(chn)])
    x = torch.from_numpy(pub).cuda()
    if ch == 2:  # batch of two identical frames through the batched entry point
        x = torch.stack([x, x])
    got = api.spectral_deblur(x, pair.k1, 1e-8).cpu().numpy().astype(np.float64)
    if ch == 2:
        assert np.array_equal(got[0], got[1])
        got = got[0]
    assert np.abs(got - ref).max() <= LMAX
    assert oracle.psnr(ref, got) >= LPSNR


def test_spectral_deblur_identity_and_pitched(oracle, api):
    b = oracle.random_mat(9, 7, 131).astype(np.float32)
    got = api.spectral_deblur(torch.from_numpy(b).cuda(), [[1.0]], 0.0).cpu().numpy()
    assert np.abs(got - b).max() <= 1e-6
    # pitched input rows (ld > cols) through the C ABI
    import ctypes as C
    lat, pair, pub, _ = make(oracle, 480, 640, 1, 9, 5, 6)
    rows, cols = pub.shape[1:]
    ld = cols + 6
    dev = torch.zeros((rows, ld), dtype=torch.float32, device="cuda")
    dev[:, :cols] = torch.from_numpy(pub[0]).cuda()
    out = torch.zeros((rows, ld + 2), dtype=torch.float32, device="cuda")
    ctx = api.context()
    k = np.ascontiguousarray(pair.k1)
    ctx.check(api.N.lib().cbp_spectral_deblur(ctx.ptr, C.c_void_p(dev.data_ptr()), 1, 1, rows, cols, ld,
                                              k.ctypes.data_as(C.c_void_p), 9, 1e-8, C.c_void_p(out.data_ptr()),
                                              ld + 2, api._stream_ptr(dev.device)))
    got = out[: rows - 8, : cols - 8].cpu().numpy().astype(np.float64)
    ref = oracle.spectral_deblur(pub[0].astype(np.float64), pair.k1, 1e-8)
    assert np.abs(got - ref).max() <= LMAX


def test_slot_chaining_equals_spectral_deblur(oracle, api):
    """decode_frames_async -> spectral_deblur_slot (the bench path) matches the host-kernel
    spectral_deblur with the decoded kernel and epsilon."""
    lat = oracle.random_frame(96, 128, 3, 11)
    pair = oracle.generate_coprime_pair(7, 12)
    frames = []
    for i in range(3):
        l = oracle.random_frame(96, 128, 3, 20 + i)
        frames.append(oracle.encode_frame(l, pair.k1, pair.k2))
    P = torch.from_numpy(np.stack([f[0] for f in frames]).astype(np.float32)).cuda()
    Q = torch.from_numpy(np.stack([f[1] for f in frames]).astype(np.float32)).cuda()
    cfg = api.make_cfg(3, 9)
    out = torch.zeros_like(P)
    slots = torch.zeros((1, api.SLOT_BYTES), dtype=torch.uint8, device="cuda")
    api.decode_frames_async(P[0:1], Q[0:1], cfg, out[0:1], slots[0])
    api.spectral_deblur_slot(P[1:], slots[0].data_ptr(), out[1:])
    sl = api.read_slots(slots, 1)[0]
    assert sl.status == 0 and sl.width == 7
    k = np.array(sl.weights[:49]).reshape(7, 7)
    ref = api.spectral_deblur(P[1:], k, sl.epsilon)
    assert torch.equal(out[1:, :, :96, :128], ref)


def test_slot_ready_event_pipeline(oracle, api):
    """cbp_decode_frames_async_ev: a second stream waiting on the slot-ready event deblurs the
    following frames with the final kernel while the recovery frame's own deconvolution and
    validation run on the first stream; results equal the serial chain."""
    pair = oracle.generate_coprime_pair(7, 14)
    frames = [oracle.encode_frame(oracle.random_frame(96, 128, 1, 40 + i), pair.k1, pair.k2) for i in range(4)]
    P = torch.from_numpy(np.stack([f[0] for f in frames]).astype(np.float32)).cuda()
    Q = torch.from_numpy(np.stack([f[1] for f in frames]).astype(np.float32)).cuda()
    cfg = api.make_cfg(3, 9)
    s_rec, s_deb = torch.cuda.Stream(), torch.cuda.Stream()
    ready = torch.cuda.Event()
    ready.record(s_rec)  # materialise the event handle
    from paper_1203_4874_b200 import _native
    ctx_rec = _native.Context(0)
    out = torch.zeros_like(P)
    slots = torch.zeros((1, api.SLOT_BYTES), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    api.decode_frames_async(P[0:1], Q[0:1], cfg, out[0:1], slots[0], ctx=ctx_rec, stream=s_rec, slot_ready=ready)
    s_deb.wait_event(ready)
    api.spectral_deblur_slot(P[1:], slots[0].data_ptr(), out[1:], stream=s_deb)
    torch.cuda.synchronize()
    ref = torch.zeros_like(P)
    slots2 = torch.zeros((1, api.SLOT_BYTES), dtype=torch.uint8, device="cuda")
    api.decode_frames_async(P[0:1], Q[0:1], cfg, ref[0:1], slots2[0])
    api.spectral_deblur_slot(P[1:], slots2[0].data_ptr(), ref[1:])
    torch.cuda.synchronize()
    a, b = api.read_slots(slots, 1)[0], api.read_slots(slots2, 1)[0]
    assert a.status == b.status == 0 and a.width == b.width == 7 and a.residual == b.residual
    assert torch.equal(out[..., :90, :122], ref[..., :90, :122])


@pytest.mark.parametrize("geom", [(96, 128, 3, 7), (1080, 1920, 3, 11)])
def test_split_decode_equals_decode(oracle, api, geom):
    """cbp_recover_kernels_async -> cbp_spectral_deblur_slot over ALL frames (the recovery
    frame batched with the ones reusing its kernel, as bench.py does) -> cbp_validate_frames_async
    gives bit-identical kernels, residuals and latents to decode_frames_async + deblur."""
    rows, cols, ch, t = geom
    pair = oracle.generate_coprime_pair(t, 16)
    lat = api.synth_frames(3 * ch, rows, cols, seed=5).view(3, ch, rows, cols)
    P, Q = api.encode_frame(lat, pair.k1, pair.k2)
    cfg = api.make_cfg(3 if t < 9 else 9, 25 if t >= 9 else 9)
    out = torch.zeros_like(P)
    slots = torch.zeros((1, api.SLOT_BYTES), dtype=torch.uint8, device="cuda")
    api.recover_kernels_async(P[0:1], Q[0:1], cfg, slots[0])
    api.spectral_deblur_slot(P, slots[0].data_ptr(), out)
    api.validate_frames_async(P[0:1], out[0:1], slots[0])
    ref = torch.zeros_like(P)
    slots2 = torch.zeros((1, api.SLOT_BYTES), dtype=torch.uint8, device="cuda")
    api.decode_frames_async(P[0:1], Q[0:1], cfg, ref[0:1], slots2[0])
    api.spectral_deblur_slot(P[1:], slots2[0].data_ptr(), ref[1:])
    torch.cuda.synchronize()
    a, b = api.read_slots(slots, 1)[0], api.read_slots(slots2, 1)[0]
    assert a.status == b.status == 0 and a.width == b.width == t
    assert a.residual == b.residual and 0.0 < a.residual <= 1e-4
    assert list(a.weights[: t * t]) == list(b.weights[: t * t])
    assert torch.equal(out[..., : rows, : cols], ref[..., : rows, : cols])


@pytest.mark.parametrize("rec", [[1], [1, 0, 0, 0, 0, 1, 1], [1, 1, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0]])
def test_host_pipeline_pairs(oracle, api, rec):
    """cbp_decode_run_host moves frames in pairs (one H2D and one D2H copy per two frames,
    ring of 6 device slots): a single frame, an odd run with recovery frames in the second
    slot of a pair and at the end, and a run longer than the ring all give, frame by frame,
    the latents of the device path (decode_frame for recovery frames, spectral_deblur with
    the latest recovered kernel otherwise)."""
    pairs = [oracle.generate_coprime_pair(5, 31), oracle.generate_coprime_pair(5, 32)]
    n = len(rec)
    which, cur = [], -1
    for r in rec:
        cur = (cur + 1) % 2 if r else cur
        which.append(cur)
    frames = [oracle.encode_frame(oracle.random_frame(40, 52, 3, 70 + i), pairs[which[i]].k1, pairs[which[i]].k2)
              for i in range(n)]
    pub = torch.from_numpy(np.stack([f[0] for f in frames]).astype(np.float32)).pin_memory()
    prv = torch.from_numpy(np.stack([f[1] for f in frames]).astype(np.float32)).pin_memory()
    cfg = api.make_cfg(3, 9)
    out, slots = api.decode_run_host(pub, prv, rec, cfg)
    assert len(slots) == sum(rec) and all(s.status == 0 and s.width == 5 for s in slots)
    k = -1
    for i in range(n):
        if rec[i]:
            k += 1
            ref = api.decode_frame(pub[i], prv[i], cfg=cfg).latent.cpu()
        else:
            w = np.array(slots[k].weights[:25]).reshape(5, 5)
            ref = api.spectral_deblur(pub[i:i + 1].cuda(), w, slots[k].epsilon)[0].cpu()
        assert torch.equal(out[i, :, :40, :52], ref), i


def test_host_pipeline_equals_device_path(oracle, api):
    pair = oracle.generate_coprime_pair(5, 31)
    frames = [oracle.encode_frame(oracle.random_frame(60, 70, 1, 40 + i), pair.k1, pair.k2) for i in range(5)]
    pub = torch.from_numpy(np.stack([f[0] for f in frames]).astype(np.float32)).pin_memory()
    prv = torch.from_numpy(np.stack([f[1] for f in frames]).astype(np.float32)).pin_memory()
    rec = [1, 0, 0, 1, 0]
    cfg = api.make_cfg(3, 9)
    out, slots = api.decode_run_host(pub, prv, rec, cfg)
    assert len(slots) == 2 and all(s.status == 0 and s.width == 5 for s in slots)
    d0 = api.decode_frame(pub[0], prv[0], cfg=cfg)
    assert torch.equal(out[0, :, :60, :70], d0.latent.cpu())
    k = np.array(slots[0].weights[:25]).reshape(5, 5)
    ref = api.spectral_deblur(pub[1:3].cuda(), k, slots[0].epsilon).cpu()
    assert torch.equal(out[1:3, :, :60, :70], ref)


# ----------------------------------------------------------------- stage level
def test_sample_slices_parity(oracle, api):
    lat, pair, pub, prv = make(oracle, 90, 110, 3, 9, 3, 4)
    for axis in (0, 1):
        sp, sq = api.sample_slices(torch.from_numpy(pub).cuda(), torch.from_numpy(prv).cuda(), 9, axis)
        rp = oracle.axis_roots_dft(oracle.luma(pub.astype(np.float64)), axis, 9)
        rq = oracle.axis_roots_dft(oracle.luma(prv.astype(np.float64)), axis, 9)
        if axis == 1:
            rp, rq = rp.T, rq.T
        assert np.abs(sp - rp).max() <= 1e-12 * np.abs(rp).max()
        assert np.abs(sq - rq).max() <= 1e-12 * np.abs(rq).max()


def aligned(e1, e2, r1, r2):
    e = np.concatenate([e1, e2]); r = np.concatenate([r1, r2])
    c = np.vdot(e, r) / np.vdot(e, e)
    return float(np.abs(c * e - r).max())


def test_cofactor_solve_known_answers(oracle, api):
    k1, k2, gap = api.cofactor_null_solve([1, 3, 2], [3, 4, 1], 2)
    assert aligned(k1, k2, [1, 2], [3, 1]) <= 1e-12 and gap > 1e-3
    k1, k2, _ = api.cofactor_null_solve([1, 1], [1, 1], 1)
    assert abs(k1[0] - k2[0]) <= 1e-14 and abs(abs(k1[0]) - 2 ** -0.5) <= 1e-12
    with pytest.raises(api.CbpError) as e:
        api.cofactor_null_solve([1, 2, 1], [1, 2, 1], 2)
    assert e.value.code == "IllConditioned"
    rng = np.random.default_rng(99)
    for _ in range(6):
        l = rng.uniform(-1, 1, 7) + 1j * rng.uniform(-1, 1, 7)
        u = rng.uniform(-1, 1, 3) + 1j * rng.uniform(-1, 1, 3)
        v = rng.uniform(-1, 1, 3) + 1j * rng.uniform(-1, 1, 3)
        k1, k2, _ = api.cofactor_null_solve(np.convolve(l, u), np.convolve(l, v), 3)
        assert aligned(k1, k2, u, v) <= 1e-8


def test_cofactor_batch_vs_oracle(oracle, api):
    lat, pair, pub, prv = make(oracle, 200, 300, 1, 11, 5, 6)
    s1 = oracle.axis_roots_dft(pub[0].astype(np.float64), 0, 11)
    s2 = oracle.axis_roots_dft(prv[0].astype(np.float64), 0, 11)
    k1, k2, gaps = api.cofactor_solve_batch(s1, s2, 11)
    for i in range(11):
        r1, r2, g = oracle.cofactor_null_solve(s1[i], s2[i], 11)
        assert aligned(k1[i], k2[i], r1, r2) <= 1e-9
        assert abs(gaps[i] - g) <= 1e-6 * g


def test_sample_cofactors_and_2d_stages(oracle, api):
    lat, pair, pub, prv = make(oracle, 40, 44, 1, 5, 17, 18)
    P, Q = torch.from_numpy(pub).cuda(), torch.from_numpy(prv).cuda()
    vals = []
    for axis in (0, 1):
        v, g = api.sample_cofactors(P, Q, 5, axis)
        rv, rg = oracle.sample_cofactors(pub.astype(np.float64), prv.astype(np.float64), 5, axis)
        for i in range(5):
            a = v[i] if axis == 0 else v[:, i]
            b = rv[i] if axis == 0 else rv[:, i]
            assert aligned(a, a[:0], b, b[:0]) <= 1e-9
        assert np.abs(g - rg).max() <= 1e-6 * rg.max()
        vals.append(v)
    for axis in (0, 1):
        assert np.abs(api.complete_to_spectrum(vals[axis], axis) - oracle.complete_to_spectrum(vals[axis], axis)).max() <= 1e-12
    lam, mu, res = api.resolve_scales(vals[0], vals[1])
    rl, rm, rr = oracle.resolve_scales(vals[0], vals[1])
    assert aligned(lam, mu, rl, rm) <= 1e-10 and abs(res - rr) <= 1e-10
    A = api.complete_to_spectrum(vals[0], 0)
    B = api.complete_to_spectrum(vals[1], 1)
    w = api.assemble_kernel(A, B, lam, mu)
    assert np.abs(w - oracle.assemble_kernel(A, B, rl, rm)).max() <= 1e-9
    assert krel(w, pair.k1) <= 1e-5


def test_estimate_width_parity(oracle, api):
    for (size, t, lo, hi, lseed, kseed) in [(24, 5, 3, 7, 101, 101), (20, 3, 3, 9, 102, 102),
                                           (64, 25, 9, 25, 103, 101), (64, 27, 9, 25, 104, 101)]:
        lat = oracle.random_mat(size, size, lseed)
        pair = oracle.generate_coprime_pair(t, kseed)
        pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
        got = api.estimate_kernel_width(pub.astype(np.float32), prv.astype(np.float32), lo, hi, 1e-6)
        ref = oracle.estimate_kernel_width(pub.astype(np.float32).astype(np.float64),
                                           prv.astype(np.float32).astype(np.float64), lo, hi, 1e-6)
        assert got == ref


def test_validate_pair_parity(oracle, api):
    lat, pair, pub, prv = make(oracle, 16, 16, 1, 3, 155, 155)
    r = api.validate_pair(pub, prv, pair.k1, pair.k2)
    assert abs(r - oracle.validate_pair(pub.astype(np.float64), prv.astype(np.float64), pair.k1, pair.k2)) <= 1e-9
    bad = oracle.conv2_full(oracle.random_mat(16, 16, 156), pair.k2).astype(np.float32)
    assert api.validate_pair(pub, bad[None], pair.k1, pair.k2) > 0.1


def test_encode_bit_exact(oracle, api):
    lat = oracle.random_frame(50, 70, 3, 9).astype(np.float32)
    pair = oracle.generate_coprime_pair(7, 9)
    pub, prv = api.encode_frame(torch.from_numpy(lat).cuda(), pair.k1, pair.k2)
    rp, rq = oracle.encode_frame(lat.astype(np.float64), pair.k1, pair.k2)
    assert np.array_equal(pub.cpu().numpy(), rp.astype(np.float32))
    assert np.array_equal(prv.cpu().numpy(), rq.astype(np.float32))


# ------------------------------------------------------------------ errors
def test_error_messages_match_reference(oracle, api):
    z = np.zeros((12, 12), np.float32)
    with pytest.raises(api.CbpError) as e:
        api.decode_frame(z, z, hint=3, cfg=api.make_cfg(3, 7, trust_hint=True))
    with pytest.raises(oracle.OracleError) as r:
        oracle.decode_frame(z.astype(np.float64), z.astype(np.float64), hint=3, cfg=oracle.make_cfg(3, 7, trust_hint=True))
    assert e.value.code == r.value.code == "IllConditionedSlice"
    assert str(e.value) == str(r.value)
    lat = oracle.random_mat(16, 16, 105)
    a1 = oracle.random_mat(3, 5, 106, 0.05, 1.0)
    a2 = oracle.random_mat(3, 5, 107, 0.05, 1.0)
    p = oracle.conv2_full(lat, a1).astype(np.float32)
    q = oracle.conv2_full(lat, a2).astype(np.float32)
    with pytest.raises(api.CbpError) as e:
        api.decode_frame(p, q, cfg=api.make_cfg(3, 7))
    with pytest.raises(oracle.OracleError) as r:
        oracle.decode_frame(p.astype(np.float64), q.astype(np.float64), cfg=oracle.make_cfg(3, 7))
    assert e.value.code == r.value.code == "InconsistentAxes" and str(e.value) == str(r.value)


@pytest.mark.parametrize("kwargs,code", [
    (dict(search_min=4, search_max=9), "InvalidArgument"),
    (dict(search_min=3, search_max=65), "InvalidArgument"),
    (dict(tau=1.5), "InvalidArgument"),
])
def test_config_errors(api, kwargs, code):
    x = np.random.default_rng(0).uniform(0, 1, (40, 40)).astype(np.float32)
    with pytest.raises(api.CbpError) as e:
        api.decode_frame(x, x, cfg=api.make_cfg(**kwargs))
    assert e.value.code == code


def test_input_errors(api):
    x = np.random.default_rng(0).uniform(0, 1, (40, 40)).astype(np.float32)
    with pytest.raises(api.CbpError) as e:  # decoder.cpp:47
        api.decode_frame(x[:20, :20], x[:20, :20], cfg=api.make_cfg(9, 25))
    assert e.value.code == "FrameTooSmall"
    for bad in (np.nan, np.inf, -np.inf):  # image.cpp:33, gray and RGB, either stream
        y = x.copy(); y[3, 4] = bad
        with pytest.raises(api.CbpError) as e:
            api.decode_frame(y, y, cfg=api.make_cfg(3, 9))
        assert e.value.code == "RangeExceeded"
        y3 = np.stack([x, x, x]); y3[2, 39, 0] = bad
        with pytest.raises(api.CbpError) as e:
            api.decode_frame(np.stack([x, x, x]), y3, cfg=api.make_cfg(3, 9))
        assert e.value.code == "RangeExceeded"
    with pytest.raises(api.CbpError) as e:  # decoder.cpp:26-28
        api.decode_frame(x, x, hint=4, cfg=api.make_cfg(3, 9))
    assert e.value.code == "InvalidArgument"
    k = np.full((3, 3), 1 / 9.0); k[0, 0] = -0.1
    with pytest.raises(api.CbpError) as e:  # kernel.cpp:7-17
        api.spectral_deblur(x, k, 1e-8)
    assert e.value.code == "InvalidArgument"
    with pytest.raises(api.CbpError) as e:
        api.spectral_deblur(x, np.full((3, 3), 0.1), 1e-8)
    assert e.value.code == "InvalidArgument"
    with pytest.raises(api.CbpError) as e:
        api.spectral_deblur(x, np.full((3, 3), 1 / 9.0), -1.0)
    assert e.value.code == "InvalidArgument"


def test_acceptance_1_on_gpu(oracle, api):
    """Criterion 1 (subset) through the GPU path: PSNR >= 40 dB, residual <= 1e-4."""
    for t in (3, 5, 9):
        for s in range(1, 5):
            lat = oracle.random_frame(64, 64, 1, oracle.frame_seed(100 + t, s))
            pair = oracle.generate_coprime_pair(t, oracle.frame_seed(100 + 31 * t, s))
            pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
            d = api.decode_frame(pub.astype(np.float32), prv.astype(np.float32), cfg=api.make_cfg(3, 9))
            assert d.width_used == t
            assert oracle.psnr(lat, d.latent.cpu().numpy().astype(np.float64)) >= 40.0
            assert d.validation_residual <= 1e-4


# ------------------------------------------------------------ quantized-stream tier
def test_quantize_degrade_on_device(oracle, api):
    """Device codes match the reference's quantize_frame / degrade_bits (encoder_test.cpp:170-215)."""
    half = torch.full((1, 2, 2), 0.5, device="cuda")
    assert int(api.quantize_frames(half, 8)[0, 0, 0]) == 128
    assert int(api.quantize_frames(half, 16)[0, 0, 0]) == 32768
    for bad in (1.1, -0.5):
        with pytest.raises(api.CbpError) as e:
            api.quantize_frames(torch.full((1, 2, 2), bad, device="cuda"), 8)
        assert e.value.status == 7 and "samples outside [0,1]" in str(e.value)
    x = oracle.random_frame(37, 53, 3, oracle.frame_seed(7, 1)).astype(np.float32)
    for bits in (8, 16):
        codes = api.quantize_frames(torch.from_numpy(x).cuda(), bits).cpu().numpy().astype(np.int64)
        ref = oracle.quantize(x.astype(np.float64), bits) * ((1 << bits) - 1)
        assert np.array_equal(codes, np.rint(ref).astype(np.int64))
        for drop in (0, 1, 3, bits - 1):
            got = api.degrade_bits(api.quantize_frames(torch.from_numpy(x).cuda(), bits), drop)
            deg = oracle.degrade_bits(ref / ((1 << bits) - 1), bits, drop) * ((1 << bits) - 1)
            assert np.array_equal(got.cpu().numpy().astype(np.int64), np.rint(deg).astype(np.int64))
        deq = api.dequantize_frames(api.quantize_frames(torch.from_numpy(x).cuda(), bits)).cpu().numpy()
        assert np.array_equal(deq, (ref / ((1 << bits) - 1)).astype(np.float32))
    with pytest.raises(api.CbpError):
        api.degrade_bits(api.quantize_frames(half, 8), 8)


@pytest.mark.parametrize("bits,ch", [(16, 1), (8, 3)])
def test_decode_quantized_parity(oracle, api, bits, ch):
    """decoder_test.cpp:427-439 (u16 decode) through device codes: decode of the codes equals
    the oracle decode of the same dequantized FP32 values."""
    rows, cols, t = 64, 64, 5
    lat, pair, pub, prv = make(oracle, rows, cols, ch, t, oracle.frame_seed(1, 77), oracle.frame_seed(2, 77))
    qp = api.quantize_frames(torch.from_numpy(pub).cuda(), bits)
    qq = api.quantize_frames(torch.from_numpy(prv).cuda(), bits)
    d = api.decode_frames_q(qp, qq, hints=[t], cfg=api.make_cfg(3, 9, trust_hint=True))[0]
    fp = api.dequantize_frames(qp).cpu().numpy().astype(np.float64)
    fq = api.dequantize_frames(qq).cpu().numpy().astype(np.float64)
    ref = oracle.decode_frame(fp, fq, hint=t, cfg=oracle.make_cfg(3, 9, trust_hint=True))
    assert d.width_used == ref.width_used == t
    assert krel(d.kernel_estimate, ref.kernel) <= KREL
    got = d.latent.cpu().numpy().astype(np.float64)
    assert np.abs(got - ref.latent).max() <= LMAX
    if bits == 16:
        assert oracle.psnr(lat, got) >= 40.0  # decoder_test.cpp:437


def test_acceptance_8_bit_degradation(oracle, api):
    """acceptance.cpp:366-403: u8 pairs, low bits dropped 0/2/4/6, trusted hint and open
    plausibility gates: PSNR must not rise as bits are dropped."""
    cfg = api.make_cfg(3, 9, trust_hint=True, max_imag_energy=float("inf"), negative_weight_tol=float("inf"))
    for seed in (1, 2, 3, 5, 7):
        lat = oracle.random_frame(48, 48, 1, oracle.frame_seed(800, seed))
        pair = oracle.generate_coprime_pair(3, oracle.frame_seed(801, seed))
        pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
        qp = api.quantize_frames(torch.from_numpy(pub.astype(np.float32)).cuda(), 8)
        qq = api.quantize_frames(torch.from_numpy(prv.astype(np.float32)).cuda(), 8)
        prev = float("inf")
        for drop in (0, 2, 4, 6):
            d = api.decode_frames_q(api.degrade_bits(qp, drop), api.degrade_bits(qq, drop), hints=[3], cfg=cfg)[0]
            q = oracle.psnr(lat, d.latent.cpu().numpy().astype(np.float64))
            assert q <= prev + 1e-9
            prev = q


def test_host_pipeline_quantized_matches_fp32(oracle, api):
    """cbp_decode_run_host_q (codes over PCIe) gives the same latents as the FP32 host
    pipeline fed the dequantized values."""
    rows, cols, t, n = 64, 80, 5, 5
    lat = np.stack([oracle.random_frame(rows, cols, 3, oracle.frame_seed(9, 10 + i)) for i in range(n)])
    pair = oracle.generate_coprime_pair(t, oracle.frame_seed(9, 2))
    pubs, prvs = zip(*[oracle.encode_frame(lat[i], pair.k1, pair.k2) for i in range(n)])
    pub = torch.from_numpy(np.stack(pubs).astype(np.float32))
    prv = torch.from_numpy(np.stack(prvs).astype(np.float32))
    codes_p = api.quantize_frames(pub.cuda(), 16).cpu()
    codes_q = api.quantize_frames(prv.cuda(), 16).cpu()
    rec = [1, 0, 0, 0, 0]
    cfg = api.make_cfg(3, 9)
    out_q, _ = api.decode_run_host(codes_p.pin_memory(), codes_q.pin_memory(), rec, cfg)
    fp = api.dequantize_frames(codes_p.cuda()).cpu()
    fq = api.dequantize_frames(codes_q.cuda()).cpu()
    out_f, _ = api.decode_run_host(fp.pin_memory(), fq.pin_memory(), rec, cfg)
    m, nn = rows, cols  # blurred extent minus t-1 = latent extent
    assert torch.equal(out_q[..., :m, :nn], out_f[..., :m, :nn])


@pytest.mark.parametrize("rows,cols,ch,t,frames", [(1080, 1920, 3, 11, 8), (2160, 3840, 1, 15, 3),
                                                    (480, 640, 1, 9, 16), (256, 256, 1, 7, 16)])
def test_deblur_repeatable(oracle, api, rows, cols, ch, t, frames):
    """Persistent passes with dynamic tiles, masked first stages and barrier-free tile
    arrivals: repeated runs over a batch (different CTA/tile interleavings each time) are
    bit-identical, and every frame equals the same frame deconvolved alone."""
    pair = oracle.generate_coprime_pair(t, 21)
    lat = api.synth_frames(frames * ch, rows, cols, seed=9).view(frames, ch, rows, cols)
    P, _ = api.encode_frame(lat, pair.k1, pair.k2)
    outs = []
    for _ in range(3):
        o = torch.full_like(P, float("nan"))
        api.spectral_deblur(P, pair.k1, 1e-8, out=o)
        outs.append(o)
    torch.cuda.synchronize()
    M, N = rows, cols
    for o in outs[1:]:
        assert torch.equal(o[..., :M, :N], outs[0][..., :M, :N])
    single = torch.full_like(P[-1:], float("nan"))
    api.spectral_deblur(P[-1:], pair.k1, 1e-8, out=single)
    torch.cuda.synchronize()
    assert torch.equal(single[..., :M, :N], outs[0][-1:, :, :M, :N])
    assert torch.isfinite(outs[0][..., :M, :N]).all()


@pytest.mark.parametrize("rows,cols", [(96, 128), (1080, 1920)])
def test_deblur_slots_equals_per_slot_calls(oracle, api, rows, cols):
    """cbp_spectral_deblur_slots (frame f uses slot f // frames_per_slot: the multi-camera
    path) equals one cbp_spectral_deblur_slot call per slot, bit for bit."""
    t, S, n = 7, 3, 4
    pubs, prvs = [], []
    for s in range(S):
        pair = oracle.generate_coprime_pair(t, 40 + s)
        lat = api.synth_frames(1 + n, rows, cols, seed=50 + s).view(1 + n, 1, rows, cols)
        p, q = api.encode_frame(lat, pair.k1, pair.k2)
        pubs.append(p)
        prvs.append(q)
    slots = torch.zeros((S, api.SLOT_BYTES), dtype=torch.uint8, device="cuda")
    rec_p = torch.cat([p[0:1] for p in pubs])
    rec_q = torch.cat([q[0:1] for q in prvs])
    api.decode_frames_async(rec_p, rec_q, api.make_cfg(3, 9), torch.zeros_like(rec_p), slots)
    frames = torch.cat([p[1:] for p in pubs])  # stream-major: S x n frames
    out = torch.zeros_like(frames)
    api.spectral_deblur_slots(frames, slots, n, out)
    ref = torch.zeros_like(frames)
    for s in range(S):
        api.spectral_deblur_slot(frames[s * n:(s + 1) * n], slots[s].data_ptr(), ref[s * n:(s + 1) * n])
    torch.cuda.synchronize()
    assert all(sl.status == 0 and sl.width == t for sl in api.read_slots(slots, S))
    M, N = rows, cols
    assert torch.equal(out[..., :M, :N], ref[..., :M, :N])


def test_deblur_slots_small_groups():
    """The same equality when a launch group holds fewer frames than one slot covers
    (CBP_GROUP_BUDGET_MB=1: one 1080p frame per group, global slot indices via frame0)."""
    import subprocess
    import sys
    env = dict(os.environ, CBP_GROUP_BUDGET_MB="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", __file__,
                        "-k", "test_deblur_slots_equals_per_slot_calls"], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


# ------------------------------------------------------------ wide kernels (t > 31)
@pytest.mark.parametrize("rows,cols,t,lo,hi,trust,lseed,pseed", [
    (96, 100, 33, 27, 35, True, None, None),     # trusted hint just past the shared-memory solvers
    (160, 160, 33, 27, 35, False, (11, 3), (12, 3)),  # estimated width 33 (Bezout blocks up to 35)
    (160, 160, 33, 27, 35, False, (11, 0), (12, 0)),  # estimated: the oracle's InconsistentAxes, same text
    (80, 90, 63, 61, 63, True, None, None),      # the reference's widest kernel (decoder.cpp:32-33,305-306)
])
def test_decode_wide_kernel_parity(oracle, api, rows, cols, t, lo, hi, trust, lseed, pseed):
    """Kernels wider than 31 run the cofactor solves and the composition on per-CTA global
    scratch (k_solve_wide, k_compose_wide) and the validation with chunked taps; same
    parity bar as the narrow kernels."""
    ls = oracle.frame_seed(*lseed) if lseed else oracle.frame_seed(1, rows + t)
    ps = oracle.frame_seed(*pseed) if pseed else oracle.frame_seed(2, cols + t)
    lat, pair, pub, prv = make(oracle, rows, cols, 1, t, ls, ps)
    hint = t if trust else None
    try:
        oracle.decode_frame(pub.astype(np.float64), prv.astype(np.float64), hint=hint,
                            cfg=oracle.make_cfg(lo, hi, trust_hint=trust))
    except oracle.OracleError as r:
        with pytest.raises(api.CbpError) as e:
            api.decode_frame(torch.from_numpy(pub).cuda(), torch.from_numpy(prv).cuda(), hint=hint,
                             cfg=api.make_cfg(lo, hi, trust_hint=trust))
        assert e.value.code == r.code and str(e.value) == str(r)
        return
    d, _ = check_decode(oracle, api, lat, pub, prv, lo, hi, hint=hint, trust=trust)
    assert d.width_used == t
    assert krel(d.kernel_estimate, pair.k1) <= 1e-4


def test_wide_stage_entry_points(oracle, api):
    """cofactor_null_solve / resolve_scales / assemble_kernel at t = 40 through the stage-level
    C ABI (global-scratch kernels)."""
    rng = np.random.default_rng(40)
    t = 40
    l = rng.uniform(-1, 1, 90) + 1j * rng.uniform(-1, 1, 90)
    u = rng.uniform(-1, 1, t) + 1j * rng.uniform(-1, 1, t)
    v = rng.uniform(-1, 1, t) + 1j * rng.uniform(-1, 1, t)
    k1, k2, gap = api.cofactor_null_solve(np.convolve(l, u), np.convolve(l, v), t)
    r1, r2, rg = oracle.cofactor_null_solve(np.convolve(l, u), np.convolve(l, v), t)
    assert aligned(k1, k2, r1, r2) <= 1e-8 and abs(gap - rg) <= 1e-6 * rg
    lat, pair, pub, prv = make(oracle, 72, 76, 1, 35, 71, 72)
    P, Q = torch.from_numpy(pub).cuda(), torch.from_numpy(prv).cuda()
    vals = [api.sample_cofactors(P, Q, 35, axis)[0] for axis in (0, 1)]
    lam, mu, res = api.resolve_scales(vals[0], vals[1])
    rl, rm, rr = oracle.resolve_scales(vals[0], vals[1])
    assert aligned(lam, mu, rl, rm) <= 1e-9
    A, B = api.complete_to_spectrum(vals[0], 0), api.complete_to_spectrum(vals[1], 1)
    w = api.assemble_kernel(A, B, lam, mu)
    assert np.abs(w - oracle.assemble_kernel(A, B, rl, rm)).max() <= 1e-9
    assert krel(w, pair.k1) <= 1e-4


@pytest.mark.parametrize("noise", [0.0, 1e-4, 1e-2, 0.3, 1.0])
def test_resolve_scales_noisy_and_degenerate(oracle, api, noise):
    """resolve_completed (decoder.cpp:133-155) on the device: Schur-complement inverse
    iteration with direct-residual refinement, falling back to the full eigendecomposition
    when the null direction is poorly separated (large noise). Planted scales
    (decoder_test.cpp:158-177) plus noise of growing size: the smallest right singular
    vector and the residual match the oracle's SVD."""
    rng = np.random.default_rng(int(noise * 1e4) + 5)
    for t in (3, 7, 11):
        pair = oracle.generate_coprime_pair(t, 131 + t)
        a = oracle.axis_roots_dft(pair.k1, 0, t)
        b = oracle.axis_roots_dft(pair.k1, 1, t)
        s = (0.5 + rng.random(t)) * np.exp(1j * rng.random(t) * 6)
        r = (0.5 + rng.random(t)) * np.exp(1j * rng.random(t) * 6)
        A = a * s[:, None] + noise * (rng.standard_normal((t, t)) + 1j * rng.standard_normal((t, t))) * np.abs(a).mean()
        B = b * r[None, :] + noise * (rng.standard_normal((t, t)) + 1j * rng.standard_normal((t, t))) * np.abs(b).mean()
        try:
            rl, rm, rr = oracle.resolve_scales(A, B)
        except oracle.OracleError as e:
            with pytest.raises(api.CbpError) as ge:
                api.resolve_scales(A, B)
            assert ge.value.code == e.code
            continue
        lam, mu, res = api.resolve_scales(A, B)
        tol = 1e-9 if noise < 1e-3 else 1e-7
        assert aligned(lam, mu, rl, rm) <= tol, (t, noise)
        assert abs(res - rr) <= tol * max(1.0, rr)
    # zeroed slices (decoder_test.cpp degenerate cases): the same outcome as the oracle, an
    # error with the same code or the same scales
    pair = oracle.generate_coprime_pair(5, 121)
    for axis, row in ((0, 0), (1, 2), (0, 4)):
        a = oracle.axis_roots_dft(pair.k1, 0, 5)
        b = oracle.axis_roots_dft(pair.k1, 1, 5)
        (a if axis == 0 else b)[row] = 0
        try:
            rl, rm, rr = oracle.resolve_scales(a, b)
        except oracle.OracleError as e:
            with pytest.raises(api.CbpError) as ge:
                api.resolve_scales(a, b)
            assert ge.value.code == e.code == "DegenerateScales"
            continue
        lam, mu, res = api.resolve_scales(a, b)
        assert aligned(lam, mu, rl, rm) <= 1e-9 and abs(res - rr) <= 1e-9
