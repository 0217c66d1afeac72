"""GPU parity: libsf (through the C-ABI) vs the float32 CPU oracle, element by element.

The north-star tolerance (1e-4 abs / 1e-5 rel per frame, 1e-3 after 100 frames) is
asserted, and so is exact equality: both sides compute the arithmetic order of
DESIGN.md section 4 in IEEE float32, so every field must agree bit for bit.
"""
import numpy as np
import pytest

import oracle
import sfgen
from sfgen import grid
from sfgen.configs import DOM_PRINTED, Params

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]

KERNELS = ["passes", "fused"]


def _sf():
    import paper_2406_18031_b200 as sf
    return sf


def _kernel_id(name):
    sf = _sf()
    return {"passes": sf.SF_KERNEL_PASSES, "auto": sf.SF_KERNEL_AUTO, "fused": sf.SF_KERNEL_FUSED}[name]


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def assert_parity(gpu, ref, what, atol=1e-4, rtol=1e-5, exact=True):
    gpu = np.asarray(gpu)
    ref = np.asarray(ref)
    assert gpu.shape == ref.shape, (what, gpu.shape, ref.shape)
    assert np.isfinite(ref).all(), what
    d = np.abs(gpu.astype(np.float64) - ref.astype(np.float64))
    lim = atol + rtol * np.abs(ref.astype(np.float64))
    bad = d > lim
    assert not bad.any(), f"{what}: {bad.sum()} elements out of tolerance, max |diff| {d.max():.3e}"
    if exact:
        assert np.array_equal(gpu, ref), f"{what}: not bit-identical, max |diff| {d.max():.3e} at {np.argmax(d)}"


def _fields(m, which=0):
    w, rho, yhat = m.get_fields(which)
    torch.cuda.synchronize()
    return w.cpu().numpy(), rho.cpu().numpy(), (yhat.cpu().numpy() if yhat is not None else None)


def run_pair(seq, frames, kernel="auto", params=None, check_every=1, tol_final=None):
    sf = _sf()
    params = params or seq.params
    o = oracle.Oracle(seq.geom, params, "f32")
    m = sf.StructureFlow(seq.geom, params, batch=1, kernel=_kernel_id(kernel))
    for k in range(frames):
        m.step(_dev(seq.Y[k]), _dev(seq.depth[k]))
        o.step(seq.Y[k], seq.depth[k])
        if (k % check_every == 0) or k == frames - 1:
            w, rho, yhat = _fields(m)
            atol = tol_final if (tol_final and k == frames - 1) else 1e-4
            assert_parity(w[0], o.w, f"w frame {k}", atol=atol)
            assert_parity(rho[0], o.rho, f"rho frame {k}", atol=atol)
            assert_parity(yhat[0], o.yhat, f"yhat frame {k}", atol=atol)
    st, flags = sf.sf_status_flags(m.ctx)
    assert flags == o.flags, (flags, o.flags)
    return m, o


@pytest.mark.parametrize("kernel", KERNELS)
def test_config1_every_frame(kernel):
    """configs[0]: 64x64, N = 2, 10 frames, every frame compared."""
    run_pair(sfgen.config_sequence(1), 10, kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_predict_only_ragged_random_state(kernel):
    """sf_predict alone on a random state, ragged 97 x 131 grid (several tiles + tails), N = 3,
    curved grid, clamp active: the prediction equals the oracle's."""
    sf = _sf()
    H, W = 97, 131
    g = grid.gnomonic(H, W, 75.0)
    p = Params(max_flow=2.5, gamma=(1e5, 1e6, 1.0, 1.0, 1.0))
    rng = np.random.default_rng(0)
    ds = g[..., 9:10]
    w = (rng.normal(size=(H, W, 3)) * 1.5 * ds).astype(np.float32)
    rho = rng.uniform(0.05, 0.6, (H, W)).astype(np.float32)
    o = oracle.Oracle(g, p, "f32")
    o.set_state(w, rho, np.zeros((H, W), np.float32))
    wp, rp = o.predict()
    m = sf.StructureFlow(g, p, kernel=_kernel_id(kernel))
    m.set_fields(_dev(w[None]), _dev(rho[None]))
    m.predict()
    gw, gr, _ = _fields(m, sf.SF_FIELDS_PREDICTED)
    assert_parity(gw[0], wp, "w^{k+}")
    assert_parity(gr[0], rp, "rho^{k+}")
    # the state itself is kept (reading 9)
    sw, sr, _ = _fields(m, sf.SF_FIELDS_STATE)
    assert np.array_equal(sw[0], w) and np.array_equal(sr[0], rho)
    assert sf.sf_status_flags(m.ctx)[1] == o.flags


@pytest.mark.parametrize("variant", ["printed", "noclamp", "S0", "S3", "inverse_input", "invalid_depth", "N1", "tiny",
                                     "far_depth", "huge_gamma3"])
def test_variants(variant):
    """Options and degenerate cases, 6 frames each, bitwise.  far_depth / huge_gamma3 put reciprocal
    inputs above 2^126, outside rcp_fast's exact range, so the kernels' exact fallback paths run."""
    seq = sfgen.config_sequence(1, frames=6)
    p = seq.params
    Y, D = seq.Y.copy(), seq.depth.copy()
    kw = dict(max_flow=p.max_flow, gamma=p.gamma, smooth_iters=p.smooth_iters)
    if variant == "printed":
        kw["dominant_rule"] = DOM_PRINTED
    elif variant == "noclamp":
        kw["clamp_advection"] = 0
    elif variant == "S0":
        kw["smooth_iters"] = 0
    elif variant == "S3":
        kw["smooth_iters"] = 3
    elif variant == "inverse_input":
        kw["input_is_inverse_depth"] = 1
        D = (1.0 / D).astype(np.float32)
    elif variant == "invalid_depth":
        D[:, 10:20, 30:40] = np.nan
        D[:, 40:44, :] = -1.0
        D[:, :, 60:] = np.inf
    elif variant == "N1":
        kw["max_flow"] = 0.75
    elif variant == "far_depth":
        D[:, 5:10, 5:12] = np.float32(1e38)  # valid depth, 1/lambda = 1e-38 (normal)
    elif variant == "huge_gamma3":
        kw["gamma"] = (p.gamma[0], p.gamma[1], 1e38, p.gamma[3], p.gamma[4])  # LDL^T pivots ~ 1e38
    elif variant == "tiny":
        g = grid.gnomonic(2, 3, 40.0)
        rng = np.random.default_rng(1)
        seq = sfgen.configs.Sequence(g, rng.uniform(0.1, 0.9, (6, 2, 3)).astype(np.float32),
                                     rng.uniform(1, 3, (6, 2, 3)).astype(np.float32), None, p, None)
        Y, D = seq.Y, seq.depth
    seq2 = sfgen.configs.Sequence(seq.geom, Y, D, None, Params(**kw), None)
    run_pair(seq2, 6, "fused")
    run_pair(seq2, 6, "passes")


@pytest.mark.parametrize("kernel", KERNELS)
def test_batch_members_are_independent(kernel):
    """B = 3 different sequences in one context: each equals its own single-sequence oracle."""
    sf = _sf()
    seqs = [sfgen.config_sequence(1, frames=4, seed=s) for s in (1, 2, 3)]
    geom, p = seqs[0].geom, seqs[0].params
    m = sf.StructureFlow(geom, p, batch=3, kernel=_kernel_id(kernel))
    os_ = [oracle.Oracle(geom, p, "f32") for _ in seqs]
    for k in range(4):
        Y = _dev(np.stack([s.Y[k] for s in seqs]))
        D = _dev(np.stack([s.depth[k] for s in seqs]))
        m.step(Y, D)
        for o, s in zip(os_, seqs):
            o.step(s.Y[k], s.depth[k])
    w, rho, yhat = _fields(m)
    for b, o in enumerate(os_):
        assert_parity(w[b], o.w, f"w[{b}]")
        assert_parity(rho[b], o.rho, f"rho[{b}]")
        assert_parity(yhat[b], o.yhat, f"yhat[{b}]")


def test_checkpoint_roundtrip_resumes_bitwise():
    """sf_get_fields -> sf_set_fields into a fresh context resumes the same trajectory."""
    sf = _sf()
    seq = sfgen.config_sequence(1, frames=6)
    a = sf.StructureFlow(seq.geom, seq.params)
    for k in range(3):
        a.step(_dev(seq.Y[k]), _dev(seq.depth[k]))
    w, rho, yhat = a.get_fields()
    b = sf.StructureFlow(seq.geom, seq.params)
    b.set_fields(w.contiguous(), rho.contiguous(), yhat.contiguous())
    for k in range(3, 6):
        a.step(_dev(seq.Y[k]), _dev(seq.depth[k]))
        b.step(_dev(seq.Y[k]), _dev(seq.depth[k]))
    for x, y in zip(_fields(a), _fields(b)):
        assert np.array_equal(x, y)


def test_kernel_times_advances_one_frame():
    """sf_kernel_times (the bench's kernel-duration hook: back-to-back launches of each kernel)
    leaves the context exactly one frame on, bit for bit the oracle's state."""
    sf = _sf()
    seq = sfgen.config_sequence(1, frames=4)
    o = oracle.Oracle(seq.geom, seq.params, "f32")
    m = sf.StructureFlow(seq.geom, seq.params, kernel=sf.SF_KERNEL_FUSED)
    for k in range(4):
        Y, D = _dev(seq.Y[k]), _dev(seq.depth[k])
        if k == 0:
            m.step(Y, D)
        else:
            tp, tu = sf.sf_kernel_times(m.ctx, Y.data_ptr(), D.data_ptr(), 3)
            assert tp > 0 and tu > 0
        o.step(seq.Y[k], seq.depth[k])
    w, rho, yhat = _fields(m)
    assert_parity(w[0], o.w, "w")
    assert_parity(rho[0], o.rho, "rho")
    assert_parity(yhat[0], o.yhat, "yhat")


def test_step_host_matches_device_path():
    """The host-buffer entry point (e2e path) gives the device path's bits."""
    sf = _sf()
    seq = sfgen.config_sequence(1, frames=4)
    a = sf.StructureFlow(seq.geom, seq.params)
    b = sf.StructureFlow(seq.geom, seq.params)
    H, W = seq.Y.shape[1:]
    wh = np.empty((1, H, W, 3), np.float32)
    rh = np.empty((1, H, W), np.float32)
    for k in range(4):
        a.step(_dev(seq.Y[k]), _dev(seq.depth[k]))
        sf.sf_step_host(b.ctx, seq.Y[k].ctypes.data, seq.depth[k].ctypes.data, wh.ctypes.data, rh.ctypes.data)
    w, rho, _ = _fields(a)
    assert np.array_equal(w, wh) and np.array_equal(rho, rh)


def test_state_machine_errors():
    sf = _sf()
    seq = sfgen.config_sequence(1, frames=2)
    m = sf.StructureFlow(seq.geom, seq.params)
    with pytest.raises(sf.SFError) as e:
        m.predict()  # fresh context
    assert e.value.status == sf.SF_E_STATE
    with pytest.raises(sf.SFError) as e:
        m.get_fields()
    assert e.value.status == sf.SF_E_STATE
    m.step(_dev(seq.Y[0]), _dev(seq.depth[0]))
    with pytest.raises(sf.SFError) as e:
        m.update(_dev(seq.Y[1]), _dev(seq.depth[1]))  # no pending prediction
    assert e.value.status == sf.SF_E_STATE
    with pytest.raises(sf.SFError) as e:
        m.get_fields(sf.SF_FIELDS_PREDICTED)
    assert e.value.status == sf.SF_E_STATE
    m.predict()
    with pytest.raises(sf.SFError) as e:
        m.predict()  # twice
    assert e.value.status == sf.SF_E_STATE
    m.update(_dev(seq.Y[1]), _dev(seq.depth[1]))


def test_cfl_flag_reports_stability_error():
    """clamp_advection = 0 with flows above max_flow: the sticky CFL flag makes
    sf_status_flags return SF_E_STABILITY (eq:numerical_stability)."""
    sf = _sf()
    H, W, ds = 16, 16, 2.0 ** -8
    g = grid.flat(H, W, ds)
    p = Params(max_flow=1.0, gamma=(1.0, 1.0, 1.0, 1.0, 1.0), clamp_advection=0)
    m = sf.StructureFlow(g, p)
    w = np.zeros((1, H, W, 3), np.float32)
    w[..., 0] = 3.0 * ds
    m.set_fields(_dev(w), _dev(np.ones((1, H, W), np.float32)))
    m.predict()
    st, flags = sf.sf_status_flags(m.ctx, clear=True)
    assert st == sf.SF_E_STABILITY and flags & sf.SF_FLAG_CFL
    assert sf.sf_status_flags(m.ctx)[1] == 0


@pytest.mark.parametrize("kernel", KERNELS)
def test_zero_motion_invariance_on_gpu(kernel):
    """Pin C1 on the GPU: identical frames, zero flow -> state bit-identical over 50 frames."""
    seq = sfgen.config_sequence(1, frames=1)
    sf = _sf()
    m = sf.StructureFlow(seq.geom, seq.params, kernel=_kernel_id(kernel))
    Y, D = _dev(seq.Y[0]), _dev(seq.depth[0])
    m.step(Y, D)
    f0 = _fields(m)
    for _ in range(50):
        m.step(Y, D)
    for a, b in zip(f0, _fields(m)):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("kernel", KERNELS)
def test_config2_headline_100_frames(kernel):
    """configs[1] at full size: 512 x 512, N = 8, 100 frames in the launch configuration
    bench.py times; checked every 10 frames and at frame 100 (tolerance 1e-3 and exact)."""
    seq = sfgen.config_sequence(2, frames=100)
    run_pair(seq, 100, kernel, check_every=10, tol_final=1e-3)


@pytest.mark.parametrize("kernel", KERNELS)
def test_config3_1024_n16(kernel):
    """configs[2]: 1024 x 1024, N = 16 (two fused launches of 8 substeps), 4 frames."""
    seq = sfgen.config_sequence(3, frames=4)
    run_pair(seq, 4, kernel)


def test_config4_batch64_full_size():
    """configs[3] at full size: 64 independent 512 x 512 sequences (seeds 100..163, the generator of
    config 2) in ONE context, the launch configuration bench.py --config 4 times (fused kernel,
    B = 64 -> 9152 CTAs); every member is checked against its own single-sequence oracle, bitwise,
    after each of 3 frames."""
    sf = _sf()
    frames = 3
    seqs = [sfgen.config_sequence(2, frames=frames, seed=100 + b) for b in range(64)]
    geom, p = seqs[0].geom, seqs[0].params
    m = sf.StructureFlow(geom, p, batch=64, kernel=_kernel_id("fused"))
    os_ = [oracle.Oracle(geom, p, "f32") for _ in seqs]
    for k in range(frames):
        m.step(_dev(np.stack([s.Y[k] for s in seqs])), _dev(np.stack([s.depth[k] for s in seqs])))
        w, rho, yhat = _fields(m)
        for b, (o, s) in enumerate(zip(os_, seqs)):
            o.step(s.Y[k], s.depth[k])
            assert_parity(w[b], o.w, f"w[{b}] frame {k}")
            assert_parity(rho[b], o.rho, f"rho[{b}] frame {k}")
            assert_parity(yhat[b], o.yhat, f"yhat[{b}] frame {k}")
    st, flags = sf.sf_status_flags(m.ctx)
    want = 0
    for o in os_:
        want |= o.flags
    assert flags == want, (flags, want)


@pytest.mark.parametrize("H,W,N,S,B", [(97, 131, 3, 2, 1), (150, 61, 8, 2, 2), (200, 170, 11, 1, 1),
                                       (64, 300, 5, 0, 1), (33, 33, 1, 3, 3), (72, 64, 8, 2, 1),
                                       (300, 257, 17, 2, 1), (5, 7, 2, 2, 2), (130, 190, 4, 4, 1)])
def test_random_states_vs_oracle(H, W, N, S, B):
    """Both GPU paths -- the tiled kernels (transport tiles + halos, 1 launch per 8 substeps, the
    update tiles) and the per-pass kernels -- against the float32 ORACLE, element by element, on
    random states over ragged grids, batches and substep counts (tile edges, grid edges, partial
    tiles, N > 8 multi-launch, S = 0 .. 4), every one of 3 frames; flags equal."""
    sf = _sf()
    g = grid.gnomonic(H, W, 80.0)
    rng = np.random.default_rng(H * 7 + W)
    ds = g[..., 9][None, ..., None]
    p = Params(max_flow=float(N) - 0.5 if N > 1 else 1.0, gamma=(3e5, 3e6, 1.0, 1.0, 2.0), smooth_iters=S)
    w = (rng.normal(size=(B, H, W, 3)) * 0.6 * N * ds).astype(np.float32)
    rho = rng.uniform(0.05, 0.6, (B, H, W)).astype(np.float32)
    yh = rng.uniform(0.1, 0.9, (B, H, W)).astype(np.float32)
    Ys = rng.uniform(0.1, 0.9, (3, B, H, W)).astype(np.float32)
    Ds = rng.uniform(1.0, 9.0, (3, B, H, W)).astype(np.float32)
    Ds[:, :, ::7, ::5] = np.nan
    os_ = [oracle.Oracle(g, p, "f32") for _ in range(B)]
    for b, o in enumerate(os_):
        o.set_state(w[b], rho[b], yh[b])
    ms = {}
    for kern in ("passes", "fused"):
        m = sf.StructureFlow(g, p, batch=B, kernel=_kernel_id(kern))
        assert m.kernel == _kernel_id(kern)
        m.set_fields(_dev(w), _dev(rho), _dev(yh))
        ms[kern] = m
    for k in range(3):
        for b, o in enumerate(os_):
            o.step(Ys[k][b], Ds[k][b])
        for kern, m in ms.items():
            m.step(_dev(Ys[k]), _dev(Ds[k]))
            got = _fields(m)
            for b, o in enumerate(os_):
                for name, x, y in zip(("w", "rho", "yhat"), got, (o.w, o.rho, o.yhat)):
                    assert_parity(x[b], y, f"{kern} {name}[{b}] frame {k}")
    want = 0
    for o in os_:
        want |= o.flags
    for kern, m in ms.items():
        assert sf.sf_status_flags(m.ctx)[1] == want, kern


def test_bench_ring_vs_oracle():
    """The bench workload (configs[1] scene, frames replayed from a ring with a wrap-around jump
    back to frame 0), 40 steps: both GPU paths equal the float32 oracle every 4 steps, flags
    included."""
    sf = _sf()
    seq = sfgen.config_sequence(2, frames=16)
    ms = {k: sf.StructureFlow(seq.geom, seq.params, kernel=_kernel_id(k)) for k in ("passes", "fused")}
    o = oracle.Oracle(seq.geom, seq.params, "f32")
    Yd = [_dev(y) for y in seq.Y]
    Dd = [_dev(d) for d in seq.depth]
    for i in range(40):
        for m in ms.values():
            m.step(Yd[i % 16], Dd[i % 16])
        o.step(seq.Y[i % 16], seq.depth[i % 16])
        if i % 4 == 3:
            for kern, m in ms.items():
                for name, x, y in zip(("w", "rho", "yhat"), _fields(m), (o.w, o.rho, o.yhat)):
                    assert_parity(x[0], y, f"{kern} {name} step {i}")
                assert sf.sf_status_flags(m.ctx)[1] == o.flags, (kern, i)


@pytest.mark.parametrize("kernel", KERNELS)
def test_config2_clamp_active_100_frames(kernel):
    """configs[1] at full size with max_flow = 1.5 px (N = 2) against the scene's flows of up to
    ~2.1 px/frame: the advection clamp (reading 12) engages (from frame 3).  Every one of 100 frames bitwise
    against the float32 oracle; the sticky flags are non-zero (CLAMPED) and equal."""
    sf = _sf()
    seq = sfgen.config_sequence(2, frames=100)
    p = seq.params
    p4 = Params(max_flow=1.5, gamma=p.gamma, smooth_iters=p.smooth_iters)
    m, o = run_pair(seq, 100, kernel, params=p4, check_every=1, tol_final=1e-3)
    assert o.flags & sf.SF_FLAG_CLAMPED, o.flags


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("H,W,nb,N,S", [(150, 61, 3, 8, 2), (200, 64, 4, 5, 1), (97, 128, 2, 16, 2)])
def test_banded_equals_single_context(kernel, H, W, nb, N, S):
    """Row bands (config 5 decomposition) on one GPU: nb band contexts with
    halo = max(N,2)+2S rows, halo exchange by peer copies before every frame, then sf_step on
    each band: the owned rows are bitwise the single-context result, flags included."""
    sf = _sf()
    g = grid.gnomonic(H, W, 80.0)
    p = Params(max_flow=float(N), gamma=(3e5, 3e6, 1.0, 1.0, 2.0), smooth_iters=S)
    rng = np.random.default_rng(H + W)
    ds = g[..., 9][None, ..., None]
    w = (rng.normal(size=(1, H, W, 3)) * 0.5 * N * ds).astype(np.float32)
    rho = rng.uniform(0.05, 0.6, (1, H, W)).astype(np.float32)
    yh = rng.uniform(0.1, 0.9, (1, H, W)).astype(np.float32)
    Ys = rng.uniform(0.1, 0.9, (3, 1, H, W)).astype(np.float32)
    Ds = rng.uniform(1.0, 9.0, (3, 1, H, W)).astype(np.float32)
    stream = torch.cuda.current_stream()
    full = sf.StructureFlow(g, p, kernel=_kernel_id(kernel), stream=stream)
    full.set_fields(_dev(w), _dev(rho), _dev(yh))
    halo = sf.sf_band_halo(full.cfg)
    assert halo == max(N, 2) + 2 * S
    bands = []
    for bi in range(nb):
        e0, o0, o1, e1 = sf.sf_band_partition(H, nb, bi, halo)
        m = sf.StructureFlow(g[e0:e1], p, kernel=_kernel_id(kernel), stream=stream, band=(e0, o0, o1, H))
        m.set_fields(_dev(w[:, e0:e1]), _dev(rho[:, e0:e1]), _dev(yh[:, e0:e1]))
        bands.append((m, e0, o0, o1, e1))
    for k in range(3):
        full.step(_dev(Ys[k]), _dev(Ds[k]))
        for bi, (m, e0, o0, o1, e1) in enumerate(bands):
            up = bands[bi - 1][0].ctx if bi > 0 else None
            dn = bands[bi + 1][0].ctx if bi < nb - 1 else None
            sf.sf_halo_exchange_peer(m.ctx, up, dn)
        for m, e0, o0, o1, e1 in bands:
            m.step(_dev(np.ascontiguousarray(Ys[k][:, e0:e1])), _dev(np.ascontiguousarray(Ds[k][:, e0:e1])))
    ref = _fields(full)
    fl = 0
    for m, e0, o0, o1, e1 in bands:
        got = _fields(m)
        for name, x, y in zip(("w", "rho", "yhat"), ref, got):
            assert_parity(y[:, o0 - e0:o1 - e0], x[:, o0:o1], f"{name} band rows {o0}:{o1}")
        fl |= sf.sf_status_flags(m.ctx)[1]
    assert fl == sf.sf_status_flags(full.ctx)[1]


def _oracle_crop_step(geom, params, w, rho, yh, Y, D, i, j, rad):
    """One oracle frame on a (2 rad + 1)^2 crop around (i, j) of a full-size grid, from the given
    state: the centre is exact when rad >= the dependency radius max(N,2) + 2S + 1 (its value
    cannot see the crop's artificial replicate border).  Returns (w, rho, yhat) at (i, j)."""
    H, W = geom.shape[:2]
    r0, r1 = max(0, i - rad), min(H, i + rad + 1)
    c0, c1 = max(0, j - rad), min(W, j + rad + 1)
    o = oracle.Oracle(np.ascontiguousarray(geom[r0:r1, c0:c1]), params, "f32")
    o.set_state(np.ascontiguousarray(w[r0:r1, c0:c1]), np.ascontiguousarray(rho[r0:r1, c0:c1]),
                np.ascontiguousarray(yh[r0:r1, c0:c1]))
    o.step(np.ascontiguousarray(Y[r0:r1, c0:c1]), np.ascontiguousarray(D[r0:r1, c0:c1]))
    return o.w[i - r0, j - c0], o.rho[i - r0, j - c0], o.yhat[i - r0, j - c0]


def test_config5_8192_banded_full_size():
    """configs[4] at full size on one GPU: 8 row-band contexts (halo exchange by peer copies) vs
    one 8192 x 8192 context, 2 frames, bitwise on every owned row; and sampled pixels of the
    second frame against the float32 oracle run on 49 x 49 crops (dependency radius 13)."""
    sf = _sf()
    H = W = 8192
    frames = 2
    g, Y, D, p = sfgen.configs.band_sequence(5, 0, H, frames)
    stream = torch.cuda.current_stream()
    full = sf.StructureFlow(g, p, stream=stream)
    nb = 8
    halo = sf.sf_band_halo(full.cfg)
    bands = []
    for bi in range(nb):
        e0, o0, o1, e1 = sf.sf_band_partition(H, nb, bi, halo)
        bands.append((sf.StructureFlow(g[e0:e1], p, stream=stream, band=(e0, o0, o1, H)), e0, o0, o1, e1))
    state0 = None
    for k in range(frames):
        Yk, Dk = _dev(Y[k]), _dev(D[k])
        if k == frames - 1:
            state0 = _fields(full)
        full.step(Yk, Dk)
        if k > 0:
            for bi, (m, *_r) in enumerate(bands):
                sf.sf_halo_exchange_peer(m.ctx, bands[bi - 1][0].ctx if bi else None,
                                         bands[bi + 1][0].ctx if bi < nb - 1 else None)
        for m, e0, o0, o1, e1 in bands:
            m.step(Yk[e0:e1].contiguous(), Dk[e0:e1].contiguous())
    ref = _fields(full)
    for m, e0, o0, o1, e1 in bands:
        got = _fields(m)
        for x, y in zip(ref, got):
            assert np.array_equal(y[:, o0 - e0:o1 - e0], x[:, o0:o1])
    rng = np.random.default_rng(5)
    pts = [(0, 0), (H - 1, W - 1), (H // 2, W // 2), (1023, 4000), (1024, 17)] + \
          [tuple(rng.integers(0, H, 2)) for _ in range(6)]
    w0, r0, y0 = (x[0] for x in state0)
    for (i, j) in pts:
        ow, orho, oy = _oracle_crop_step(g, p, w0, r0, y0, Y[-1], D[-1], int(i), int(j), 24)
        assert np.array_equal(ref[0][0, i, j], ow) and ref[1][0, i, j] == orho and ref[2][0, i, j] == oy, (i, j)
