"""Fused fp32 rFSE (F = 64) against the reference-arithmetic fp64 rFSE path.

The fp64 image-level rFSE plan runs the per-window kernel that reproduces
the reference's `extrapolate_rfse` (golden-pinned in test_gpu_parity); the
fused kernel must agree with it per block (max |dpx| <= 0.5 gray levels),
pick the same canonical pairs in the same order, report the same tally
semantics (basis_target) and the residual-energy identity."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fse(cuda_ok):
    import paper_2204_14193_b200 as fse
    return fse


def _plans(fse, blocks, H, W, geo=None, **kw):
    geo = geo or fse.Geometry(16, 16, 64)
    fast = fse.ConcealPlan(blocks, H, W, geo, rho_hat=0.8, gamma=0.5, algorithm="rfse",
                           precision="fp32", **kw)
    ref = fse.ConcealPlan(blocks, H, W, geo, rho_hat=0.8, gamma=0.5, algorithm="rfse",
                          precision="fp64", **kw)
    assert fast.info["fast_path"] == 1 and ref.info["fast_path"] == 0
    return fast, ref


@pytest.mark.parametrize("dtype,iters,bt", [("u8", 50, None), ("f32", 30, None), ("u8", 100, 100),
                                            ("f64", 100, 37)])
def test_fused_rfse_matches_fp64(fse, dtype, iters, bt):
    import torch
    from paper_2204_14193_b200.synth import field_torch
    H, W = 270, 480
    frames = field_torch(2, H, W, seed=17, device="cuda", edges=True)
    if dtype != "u8":
        frames = frames.to(torch.float32 if dtype == "f32" else torch.float64)
    blocks = fse.frames_pattern(2, H, W, 16, 0.08, seed=6)
    blocks = np.concatenate([blocks, np.array([[0, 0, 0], [0, 0, W - 16], [1, H - 16, 0],
                                               [1, H - 16, W - 16]], np.int32)])
    kw = dict(iterations=iters) if bt is None else dict(iterations=iters, basis_target=bt)
    fast, ref = _plans(fse, blocks, H, W, **kw)
    t32, tr = fast.run(frames, tile_dtype="f32", trace=True)
    t64 = ref.run(frames, tile_dtype="f64")
    print(_rfse_gate(fse, frames, blocks, t32, tr, t64, 64, 16, iters, bt, log=f"rfse64_{dtype}_{iters}_{bt}"))
    uv = tr["uv"].cpu().numpy()
    e = tr["e"].cpu().numpy()
    n_it = fast.iterations
    for k in range(len(blocks)):
        used = uv[k, :, 0] >= 0
        u, v = uv[k, used, 0], uv[k, used, 1]
        # canonical member: never the larger row-major index of a pair
        mu, mv = (-u) % 64, (-v) % 64
        assert np.all(u * 64 + v <= mu * 64 + mv)
        selfc = ((2 * u) % 64 == 0) & ((2 * v) % 64 == 0)
        tally = int(np.sum(np.where(selfc, 1, 2)))
        if bt is None:
            assert used.sum() == n_it
        else:  # stops at the first iteration whose tally reaches the target
            assert tally >= bt and tally - (1 if selfc[-1] else 2) < bt
        # residual energy decreases monotonically (crit >= 0)
        assert np.all(np.diff(e[k, used]) <= 1e-3 * e[k, 0])


def test_fused_rfse_selection_sequence(fse):
    """The fused kernel's (u, v) sequence (canonical pair members) equals the
    C oracle's fp64 rFSE (rfse.py:56-167 restated) for every block over all
    60 iterations, except at a certified near-tie (criterion gap < 1e-6
    relative or within twice the fp32 run's measured error), after which the
    two runs legitimately differ."""
    import torch
    from paper_2204_14193_b200.synth import frame_u8
    from tests._windows import window_of
    fr = frame_u8(256, 384, seed=3)
    blocks = np.array([[0, 64 + 32 * i, 64 + 48 * j] for i in range(3) for j in range(4)], np.int32)
    fast, _ = _plans(fse, blocks, 256, 384, iterations=60)
    _, tr = fast.run(torch.from_numpy(fr).cuda(), tile_dtype="f32", trace=True)
    get = _trace_getter(tr)
    from oracle import oracle as orc
    from oracle.gate import first_rfse_divergence
    full, ties = 0, []
    for k, (f, t, l) in enumerate(blocks):
        s, lab = window_of(fr.astype(np.float64), t, l, 64, 16, 16)
        o = orc.extrapolate_rfse(s, lab, 0.8, 0.5, 60)
        at = first_rfse_divergence((o["us"], o["vs"]), get(k))
        if at is None:
            full += 1
            continue
        cert = orc.rfse_divergence_certificate(s, lab, 0.8, 0.5, at, get(k))
        assert cert["strict"] or cert["bounded"], (k, cert)
        ties.append((k, cert))
    print("identical", full, "certified ties", ties)



def test_rfse_degenerate_support_raises(fse):
    """A support confined to one row makes every (k, 0) pair's Gram
    determinant vanish (W[2k, 0] = W[0, 0]): rfse.py:50-55 raises ConfigError."""
    lab = np.zeros((32, 32), np.int8)
    lab[10, 4:28] = 1          # support: one row
    lab[20:24, 12:16] = 2      # loss
    cfg = fse.FseConfig(rho_hat=0.8, gamma=0.5, iterations=10, fft_dims=(32, 32), algorithm="rfse")
    with pytest.raises(fse.ConfigError):
        fse.extrapolate_rfse(np.random.default_rng(0).random((32, 32)) * 255, fse.AreaMask(lab), cfg)


_SEEDS = int(__import__("os").environ.get("FSE_FUZZ_SEEDS", 0))  # widen for one-off sweeps


def _trace_getter(tr32):
    uv = tr32["uv"].cpu().numpy()
    c = tr32["c"].cpu().numpy()

    def get(k):
        used = uv[k, :, 0] >= 0
        return (uv[k, used, 0].astype(np.int64), uv[k, used, 1].astype(np.int64),
                c[k, used, 0] + 1j * c[k, used, 1])
    return get


def _rfse_gate(fse, img, blocks, t32, tr32, t64, F, B, iters, bt, log=None, border=None):
    """fp32 rFSE gate against the independent C oracle's rFSE (oracle/gate.py
    rfse_gate, rfse.py:37-210 restated): every block within 0.5 gray levels
    except certified near-ties (criterion gap < 1e-6 relative, or within
    twice the fp32 run's measured criterion error at the first differing
    selection).  Also: the fp64 GPU plan (t64) agrees with the oracle to 1e-9."""
    from oracle import oracle as orc
    from oracle.gate import rfse_gate
    fr = img.cpu().numpy() if hasattr(img, "cpu") else np.asarray(img)
    fr = fr if fr.ndim == 3 else fr[None]
    border = B if border is None else border
    st = rfse_gate(fr, blocks, t32.cpu().numpy(), _trace_getter(tr32), F, B, border, 0.8, 0.5, iters, bt,
                   log=log)
    if t64 is not None:
        ref = orc.conceal_blocks_rfse(fr, blocks, B, border, F, 0.8, 0.5, iters, bt)
        np.testing.assert_allclose(t64.cpu().numpy(), ref, rtol=0, atol=1e-9)
    return {k: v for k, v in st.items() if k != "outliers"}


@pytest.mark.parametrize("seed", range(_SEEDS or 6))
def test_fused_rfse_random_geometry(fse, seed):
    """Random image sizes (clipped windows), positions, frame types and
    iteration budgets: fused fp32 rFSE within 0.5 gray levels of fp64."""
    import torch
    from paper_2204_14193_b200.synth import field
    rng = np.random.default_rng(3000 + seed)
    H, W = int(rng.integers(20, 200)), int(rng.integers(20, 200))
    n = int(rng.integers(6, 20))
    blocks = np.stack([np.zeros(n, np.int64), rng.integers(0, H - 16 + 1, n),
                       rng.integers(0, W - 16 + 1, n)], 1).astype(np.int32)
    img = field(H, W, seed=seed)
    dtype = rng.choice(["u8", "f32", "f64"])
    if dtype == "u8":
        img = np.clip(np.rint(img), 0, 255).astype(np.uint8)
    elif dtype == "f32":
        img = img.astype(np.float32)
    iters = int(rng.choice([1, 9, 40]))
    bt = None if rng.random() < 0.5 else int(rng.integers(1, 2 * iters + 1))
    kw = dict(iterations=iters) if bt is None else dict(iterations=iters, basis_target=bt)
    try:
        fast, ref = _plans(fse, blocks, H, W, **kw)
    except fse.ConfigError:
        pytest.skip("degenerate pair geometry for this random image")
    fr = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    t32, tr32 = fast.run(fr, tile_dtype="f32", trace=True)
    t64 = ref.run(fr, tile_dtype="f64")
    cert = _rfse_gate(fse, img, blocks, t32, tr32, t64, 64, 16, iters, bt)
    print(seed, H, W, dtype, iters, bt, "certified near-ties:", cert)


# ---------------------------------------------------------------- F = 32


@pytest.mark.parametrize("dtype,iters,bt", [("u8", 50, None), ("f32", 40, 37), ("u8", 100, 60)])
def test_fused_rfse32_matches_fp64(fse, dtype, iters, bt):
    """The F = 32 fused rFSE (one warp per block, pair entries (2p, c),
    (2p + 1, c)) against the fp64 rFSE plan: max |dpx| <= 0.5, canonical
    members, tally rule."""
    import torch
    from paper_2204_14193_b200.synth import field_torch
    H, W = 200, 320
    frames = field_torch(2, H, W, seed=23, device="cuda", edges=True)
    if dtype != "u8":
        frames = frames.to(torch.float32)
    blocks = fse.frames_pattern(2, H, W, 8, 0.06, seed=8)
    blocks = np.concatenate([blocks, np.array([[0, 0, 0], [0, 0, W - 8], [1, H - 8, 0],
                                               [1, H - 8, W - 8]], np.int32)])
    kw = dict(iterations=iters) if bt is None else dict(iterations=iters, basis_target=bt)
    fast, ref = _plans(fse, blocks, H, W, geo=fse.Geometry(8, 8, 32), **kw)
    t32, tr = fast.run(frames, tile_dtype="f32", trace=True)
    t64 = ref.run(frames, tile_dtype="f64")
    print(_rfse_gate(fse, frames, blocks, t32, tr, t64, 32, 8, iters, bt, log=f"rfse32_{dtype}_{iters}_{bt}"))
    uv = tr["uv"].cpu().numpy()
    for k in range(len(blocks)):
        used = uv[k, :, 0] >= 0
        u, v = uv[k, used, 0], uv[k, used, 1]
        mu, mv = (-u) % 32, (-v) % 32
        assert np.all(u * 32 + v <= mu * 32 + mv)
        selfc = ((2 * u) % 32 == 0) & ((2 * v) % 32 == 0)
        tally = int(np.sum(np.where(selfc, 1, 2)))
        if bt is None:
            assert used.sum() == fast.iterations
        else:
            assert tally >= bt and tally - (1 if selfc[-1] else 2) < bt


def test_fused_rfse32_selection_sequence(fse):
    """The fused kernel's (u, v) sequence (canonical pair members) equals the
    C oracle's fp64 rFSE (rfse.py:56-167 restated) for every block over all
    40 iterations, except at a certified near-tie (criterion gap < 1e-6
    relative or within twice the fp32 run's measured error), after which the
    two runs legitimately differ."""
    import torch
    from paper_2204_14193_b200.synth import frame_u8
    from tests._windows import window_of
    fr = frame_u8(160, 224, seed=4)
    blocks = np.array([[0, 32 + 24 * i, 32 + 40 * j] for i in range(3) for j in range(4)], np.int32)
    fast, _ = _plans(fse, blocks, 160, 224, geo=fse.Geometry(8, 8, 32), iterations=40)
    _, tr = fast.run(torch.from_numpy(fr).cuda(), tile_dtype="f32", trace=True)
    get = _trace_getter(tr)
    from oracle import oracle as orc
    from oracle.gate import first_rfse_divergence
    full, ties = 0, []
    for k, (f, t, l) in enumerate(blocks):
        s, lab = window_of(fr.astype(np.float64), t, l, 32, 8, 8)
        o = orc.extrapolate_rfse(s, lab, 0.8, 0.5, 40)
        at = first_rfse_divergence((o["us"], o["vs"]), get(k))
        if at is None:
            full += 1
            continue
        cert = orc.rfse_divergence_certificate(s, lab, 0.8, 0.5, at, get(k))
        assert cert["strict"] or cert["bounded"], (k, cert)
        ties.append((k, cert))
    print("identical", full, "certified ties", ties)



@pytest.mark.parametrize("seed", range(_SEEDS or 4))
def test_fused_rfse32_random_geometry(fse, seed):
    import torch
    from paper_2204_14193_b200.synth import field
    rng = np.random.default_rng(4000 + seed)
    H, W = int(rng.integers(12, 120)), int(rng.integers(12, 120))
    n = int(rng.integers(6, 20))
    blocks = np.stack([np.zeros(n, np.int64), rng.integers(0, H - 8 + 1, n),
                       rng.integers(0, W - 8 + 1, n)], 1).astype(np.int32)
    img = field(H, W, seed=seed)
    if seed % 2 == 0:
        img = np.clip(np.rint(img), 0, 255).astype(np.uint8)
    iters = int(rng.choice([1, 9, 40]))
    bt = None if rng.random() < 0.5 else int(rng.integers(1, 2 * iters + 1))
    kw = dict(iterations=iters) if bt is None else dict(iterations=iters, basis_target=bt)
    try:
        fast, ref = _plans(fse, blocks, H, W, geo=fse.Geometry(8, 8, 32), **kw)
    except fse.ConfigError:
        pytest.skip("degenerate pair geometry for this random image")
    fr = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    t32, tr32 = fast.run(fr, tile_dtype="f32", trace=True)
    t64 = ref.run(fr, tile_dtype="f64")
    cert = _rfse_gate(fse, img, blocks, t32, tr32, t64, 32, 8, iters, bt)
    print(seed, H, W, iters, bt, "certified near-ties:", cert)


@pytest.mark.parametrize("F", [32, 64])
def test_fused_rfse_tma_matches_direct(fse, F):
    """rFSE instantiations with TMA window staging (forced, FSE_TMA=1) and
    direct loads (FSE_TMA=0) give identical tiles and traces; the blocks sit
    where every window box starts 16-byte aligned (TMA-legal)."""
    import os
    import torch
    from paper_2204_14193_b200.synth import field_torch
    B = F // 4
    H, W = 256, 448
    frames = field_torch(2, H, W, seed=91, device="cuda", edges=True)
    rng = np.random.default_rng(F)
    n = 40
    left = 16 * rng.integers(0, (W - B) // 16, n) + (8 if F == 32 else 0)
    blocks = np.stack([rng.integers(0, 2, n), rng.integers(0, H - B + 1, n), left], 1).astype(np.int32)
    plan, _ = _plans(fse, blocks, H, W, geo=fse.Geometry(B, B, F), iterations=50, basis_target=60)
    out = {}
    try:
        for v in ("0", "1"):
            os.environ["FSE_TMA"] = v
            t, tr = plan.run(frames, tile_dtype="f32", trace=True)
            out[v] = (t.cpu().numpy(), tr["uv"].cpu().numpy(), tr["c"].cpu().numpy())
    finally:
        del os.environ["FSE_TMA"]
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("F", [32, 64])
def test_fused_rfse_global_trace(fse, F):
    """More iterations than the shared-memory trace holds (F=32: 136, F=64:
    400): the per-slot global trace path, against the fp64 plan."""
    import torch
    from paper_2204_14193_b200.synth import field
    B = F // 4
    H, W = 3 * F, 4 * F
    img = field(H, W, seed=F + 1)
    rng = np.random.default_rng(F)
    n = 12
    blocks = np.stack([np.zeros(n, np.int64), rng.integers(0, H - B + 1, n),
                       rng.integers(0, W - B + 1, n)], 1).astype(np.int32)
    iters = 450 if F == 64 else 300
    fast, ref = _plans(fse, blocks, H, W, geo=fse.Geometry(B, B, F), iterations=iters,
                       basis_target=iters + 100)
    assert fast.info["fast_path"] == 1
    fr = torch.from_numpy(img).cuda()
    t32, tr32 = fast.run(fr, tile_dtype="f32", trace=True)
    t64 = ref.run(fr, tile_dtype="f64")
    cert = _rfse_gate(fse, img, blocks, t32, tr32, t64, F, B, iters, iters + 100)
    print(F, "certified near-ties:", cert)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_rfse_plan_rejects_degenerate_pair_geometry(fse, precision):
    """A 17 x 16 image with its one 16 x 16 block at the origin: the clipped
    support is one row, every (k, 0) pair's Gram determinant vanishes
    (rfse.py:47-55).  Every rFSE plan -- fp64 per-window as well as the fused
    fp32 one -- raises ConfigError at creation (never stale tiles)."""
    with pytest.raises(fse.ConfigError):
        fse.ConcealPlan(np.array([[0, 0, 0]], np.int32), 17, 16, fse.Geometry(16, 16, 64),
                        algorithm="rfse", precision=precision, iterations=10)
    # the same geometry is fine for cFSE
    fse.ConcealPlan(np.array([[0, 0, 0]], np.int32), 17, 16, fse.Geometry(16, 16, 64),
                    precision=precision, iterations=10)


@pytest.mark.parametrize("F", [64, 32])
def test_fused_rfse_on_a_config_frame(fse, F):
    """Fused fp32 rFSE at scale against the C oracle's rFSE: F = 64 on the
    bench's first 4K frame (1,620 blocks, basis_target 100), F = 32 on the
    config-4a image (500 blocks of 8 x 8, 50 iterations)."""
    from paper_2204_14193_b200.synth import field, field_torch
    import torch
    if F == 64:
        frames = field_torch(1, 2160, 3840, seed=5 * 7919, device="cuda")
        blocks = fse.frames_pattern(1, 2160, 3840, 16, 0.05, seed=5)
        kw, iters, bt = dict(iterations=100, basis_target=100), 100, 100
    else:
        img = field(512, 512, seed=4).astype(np.float32)
        frames = torch.from_numpy(img).cuda()[None]
        tl = np.array([(16 * i, 16 * j) for i in range(32) for j in range(32)], np.int32)[::2][:500]
        blocks = np.concatenate([np.zeros((len(tl), 1), np.int32), tl], 1)
        kw, iters, bt = dict(iterations=50), 50, None
    B = F // 4
    plan = fse.ConcealPlan(blocks, frames.shape[1], frames.shape[2], fse.Geometry(B, B, F), rho_hat=0.8,
                           gamma=0.5, algorithm="rfse", precision="fp32", **kw)
    assert plan.info["fast_path"] == 1
    t32, tr = plan.run(frames, tile_dtype="f32", trace=True)
    st = _rfse_gate(fse, frames, blocks, t32, tr, None, F, B, iters, bt, log=f"rfse{F}_config_frame")
    print(F, st)


# ---------------------------------------------------------------- F = 128


@pytest.mark.parametrize("dtype,iters,bt,sym", [("u8", 60, None, "1"), ("f32", 100, 100, "1"),
                                                ("u8", 60, None, "0")])
def test_fused_rfse128_mixed_classes(fse, dtype, iters, bt, sym, monkeypatch):
    """F = 128 rFSE in one fused plan: interior blocks in the centred frame,
    clipped corner/edge blocks on the complex W' table and (A, C, D)
    criterion (FSE_SYM=0: every block on the complex path).  Gate against
    the C oracle's rFSE: every block within 0.5 gray levels except certified
    near-ties; canonical members and the tally rule."""
    import torch
    monkeypatch.setenv("FSE_SYM", sym)
    from paper_2204_14193_b200.synth import field_torch
    H, W = 384, 544
    frames = field_torch(2, H, W, seed=29, device="cuda", edges=True)
    if dtype != "u8":
        frames = frames.to(torch.float32)
    interior = [[f, 64 + 96 * i, 64 + 112 * j] for f in range(2) for i in range(3) for j in range(4)]
    clipped = [[0, 0, 0], [0, 0, W - 32], [1, H - 32, 0], [1, H - 32, W - 32], [0, 20, 250], [1, 200, 8]]
    blocks = np.array(interior[:10] + clipped + interior[10:], np.int32)
    kw = dict(iterations=iters) if bt is None else dict(iterations=iters, basis_target=bt)
    plan = fse.ConcealPlan(blocks, H, W, fse.Geometry(32, 16, 128), rho_hat=0.8, gamma=0.5,
                           algorithm="rfse", precision="fp32", **kw)
    assert plan.info["fast_path"] == 1 and plan.info["n_centred"] == (1 if sym == "1" else 0)
    t32, tr = plan.run(frames, tile_dtype="f32", trace=True)
    print(_rfse_gate(fse, frames, blocks, t32, tr, None, 128, 32, iters, bt,
                     log=f"rfse128_{dtype}_{iters}_{bt}_sym{sym}", border=16))
    uv = tr["uv"].cpu().numpy()
    for k in range(len(blocks)):
        used = uv[k, :, 0] >= 0
        u, v = uv[k, used, 0], uv[k, used, 1]
        mu, mv = (-u) % 128, (-v) % 128
        assert np.all(u * 128 + v <= mu * 128 + mv)
        selfc = ((2 * u) % 128 == 0) & ((2 * v) % 128 == 0)
        tally = int(np.sum(np.where(selfc, 1, 2)))
        if bt is None:
            assert used.sum() == plan.iterations
        else:
            assert tally >= bt and tally - (1 if selfc[-1] else 2) < bt


def test_fused_rfse128_selection_sequence(fse):
    """The fused F = 128 centred-frame rFSE picks the C oracle's canonical
    pair sequence over all 60 iterations, up to a certified near-tie."""
    import torch
    from paper_2204_14193_b200.synth import frame_u8
    from tests._windows import window_of
    fr = frame_u8(384, 512, seed=5)
    blocks = np.array([[0, 64 + 64 * i, 64 + 96 * j] for i in range(4) for j in range(4)], np.int32)
    plan = fse.ConcealPlan(blocks, 384, 512, fse.Geometry(32, 16, 128), rho_hat=0.8, gamma=0.5,
                           algorithm="rfse", precision="fp32", iterations=60)
    assert plan.info["fast_path"] == 1
    _, tr = plan.run(torch.from_numpy(fr).cuda(), tile_dtype="f32", trace=True)
    get = _trace_getter(tr)
    from oracle import oracle as orc
    from oracle.gate import first_rfse_divergence
    full, ties = 0, []
    for k, (f, t, l) in enumerate(blocks):
        s, lab = window_of(fr.astype(np.float64), t, l, 128, 32, 16)
        o = orc.extrapolate_rfse(s, lab, 0.8, 0.5, 60)
        at = first_rfse_divergence((o["us"], o["vs"]), get(k))
        if at is None:
            full += 1
            continue
        cert = orc.rfse_divergence_certificate(s, lab, 0.8, 0.5, at, get(k))
        assert cert["strict"] or cert["bounded"], (k, cert)
        ties.append((k, cert))
    print("identical", full, "certified ties", ties)
    assert full >= len(blocks) // 2


def test_fused_rfse128_config4b(fse):
    """Config 4b geometry with rFSE (500 32x32 losses over 8 images, F = 128,
    100 basis functions): interior blocks in the centred frame, the 115
    clipped ones on the complex tables, every block gated against the C
    oracle."""
    from paper_2204_14193_b200.synth import field
    import torch
    imgs = np.stack([field(512, 512, seed=40 + k) for k in range(8)]).astype(np.float32)
    blocks = np.array([(f, 64 * i, 64 * j) for f in range(8) for i in range(8) for j in range(8)],
                      np.int32)[:500]
    plan = fse.ConcealPlan(blocks, 512, 512, fse.Geometry(32, 16, 128), rho_hat=0.8, gamma=0.5,
                           algorithm="rfse", precision="fp32", iterations=100, basis_target=100)
    assert plan.info["fast_path"] == 1
    t32, tr = plan.run(torch.from_numpy(imgs).cuda(), tile_dtype="f32", trace=True)
    print(_rfse_gate(fse, imgs, blocks, t32, tr, None, 128, 32, 100, 100, log="rfse128_config4b",
                     border=16))


@pytest.mark.parametrize("seed", range(_SEEDS or 4))
def test_fused_rfse128_random_geometry(fse, seed):
    """F = 128 fused rFSE on random image sizes (clipped windows on both
    table kinds), positions, frame types and budgets, gated against the C
    oracle (and the fp64 rFSE plan against the oracle at 1e-9)."""
    import torch
    from paper_2204_14193_b200.synth import field
    rng = np.random.default_rng(7000 + seed)
    H, W = int(rng.integers(40, 300)), int(rng.integers(40, 300))
    n = int(rng.integers(4, 10))
    blocks = np.stack([np.zeros(n, np.int64), rng.integers(0, H - 32 + 1, n),
                       rng.integers(0, W - 32 + 1, n)], 1).astype(np.int32)
    img = field(H, W, seed=seed)
    dtype = rng.choice(["u8", "f32"])
    img = np.clip(np.rint(img), 0, 255).astype(np.uint8) if dtype == "u8" else img.astype(np.float32)
    iters = int(rng.choice([5, 30, 60]))
    bt = None if rng.random() < 0.5 else int(rng.integers(1, 2 * iters + 1))
    kw = dict(iterations=iters) if bt is None else dict(iterations=iters, basis_target=bt)
    geo = fse.Geometry(32, 16, 128)
    try:
        fast = fse.ConcealPlan(blocks, H, W, geo, rho_hat=0.8, gamma=0.5, algorithm="rfse",
                               precision="fp32", **kw)
    except fse.ConfigError:
        pytest.skip("degenerate pair geometry for this random image")
    assert fast.info["fast_path"] == 1
    fr = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    t32, tr32 = fast.run(fr, tile_dtype="f32", trace=True)
    cert = _rfse_gate(fse, img, blocks, t32, tr32, None, 128, 32, iters, bt, border=16)
    print(seed, H, W, dtype, iters, bt, "certified near-ties:", cert)


@pytest.mark.parametrize("F,B", [(64, 16), (32, 8)])
def test_fused_rfse_complex_tables_on_interior_blocks(fse, F, B, monkeypatch):
    """FSE_SYM=0 keeps interior classes on the complex W' / (A, C, D) tables
    (the path of clipped classes): the same oracle gate as the centred
    default, on a frame of interior and corner blocks."""
    import torch
    from paper_2204_14193_b200.synth import field_torch
    monkeypatch.setenv("FSE_SYM", "0")
    H, W = 240, 352
    frames = field_torch(1, H, W, seed=31, device="cuda", edges=True)
    blocks = fse.frames_pattern(1, H, W, B, 0.06, seed=9)
    blocks = np.concatenate([blocks, np.array([[0, 0, 0], [0, H - B, W - B]], np.int32)])
    plan = fse.ConcealPlan(blocks, H, W, fse.Geometry(B, B, F), rho_hat=0.8, gamma=0.5,
                           algorithm="rfse", precision="fp32", iterations=60)
    assert plan.info["fast_path"] == 1 and plan.info["n_centred"] == 0
    t32, tr = plan.run(frames, tile_dtype="f32", trace=True)
    print(_rfse_gate(fse, frames, blocks, t32, tr, None, F, B, 60, None, log=f"rfse{F}_complex"))
