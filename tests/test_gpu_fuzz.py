"""Seeded randomized parity sweep of the fused fp32 path against the CPU
oracle: random image sizes (down to smaller than the window, so most
windows are clipped), random block positions (including every border and
corner), every window size, both support widths, u8 / f32 / f64 frames,
iteration counts from 1 to 150.  Same gate as the config tests (SURVEY.md
8(c)): per block max |dpx| <= 0.5 except certified near-ties."""
import numpy as np
import pytest

from tests._windows import fp32_gate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fse(cuda_ok):
    import paper_2204_14193_b200 as fse
    return fse


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    F = int(rng.choice([32, 64, 128]))
    B = F // 4
    border = int(rng.choice([B // 2, B]))
    H = int(rng.integers(B + 3, 3 * F))
    W = int(rng.integers(B + 3, 3 * F))
    n_frames = int(rng.integers(1, 3))
    dtype = rng.choice(["u8", "f32", "f64"])
    iters = int(rng.choice([1, 7, 60, 150]))
    n = int(rng.integers(8, 24))
    blocks = np.stack([rng.integers(0, n_frames, n), rng.integers(0, H - B + 1, n),
                       rng.integers(0, W - B + 1, n)], 1).astype(np.int32)
    # the four corners of frame 0 always
    corners = np.array([[0, 0, 0], [0, 0, W - B], [0, H - B, 0], [0, H - B, W - B]], np.int32)
    blocks = np.concatenate([corners, blocks])
    return F, B, border, H, W, n_frames, str(dtype), iters, blocks


# FSE_FUZZ_SEEDS widens the sweep for one-off robustness runs (default 24)
@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("FSE_FUZZ_SEEDS", 24))))
def test_fused_path_random_geometry(fse, seed):
    import torch
    from paper_2204_14193_b200.synth import field
    F, B, border, H, W, nf, dtype, iters, blocks = _case(seed)
    frames = np.stack([field(H, W, seed=seed * 7 + k) for k in range(nf)])
    if dtype == "u8":
        frames = np.clip(np.rint(frames), 0, 255).astype(np.uint8)
    elif dtype == "f32":
        frames = frames.astype(np.float32)
    plan = fse.ConcealPlan(blocks, H, W, fse.Geometry(B, border, F), rho_hat=0.8, gamma=0.5,
                           iterations=iters, precision="fp32")
    assert plan.info["fast_path"] == 1
    fr = torch.from_numpy(np.ascontiguousarray(frames)).cuda()
    tiles, tr = plan.run(fr, tile_dtype="f32", trace=True)
    uv = tr["uv"].cpu().numpy()
    cc = tr["c"].cpu().numpy()

    def get(k):
        return uv[k, :, 0].astype(np.int64), uv[k, :, 1].astype(np.int64), cc[k, :, 0] + 1j * cc[k, :, 1]

    st = fp32_gate(frames.astype(np.float64), blocks, tiles.cpu().numpy(), get, F, B, border, 0.8, 0.5,
                   iters)
    print(seed, F, B, border, H, W, nf, dtype, iters, len(blocks), st)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("FSE_FUZZ_SEEDS", 6))))
def test_fp64_plan_random_geometry(fse, seed):
    """The fp64 image-level path (reference arithmetic, any window size) on
    random geometry: canonical selection sequence identical to the fp64
    oracle's (or a certified fp64 near-tie), tiles within 1e-9."""
    import torch
    from oracle import oracle as orc
    from paper_2204_14193_b200.synth import field
    rng = np.random.default_rng(2000 + seed)
    F = int(rng.choice([16, 24, 32, 48, 64]))
    B = int(rng.choice([4, 8])) if F < 32 else int(rng.choice([8, 16]))
    if (F - B) % 2:
        B += 1
    border = int(rng.integers(2, (F - B) // 2 + 1))
    H, W = int(rng.integers(B + 2, 2 * F)), int(rng.integers(B + 2, 2 * F))
    iters = int(rng.choice([1, 13, 80]))
    n = 6
    blocks = np.stack([np.zeros(n, np.int64), rng.integers(0, H - B + 1, n),
                       rng.integers(0, W - B + 1, n)], 1).astype(np.int32)
    img = field(H, W, seed=seed)
    plan = fse.ConcealPlan(blocks, H, W, fse.Geometry(B, border, F), rho_hat=0.8, gamma=0.5,
                           iterations=iters, precision="fp64")
    tiles, tr = plan.run(torch.from_numpy(img).cuda(), tile_dtype="f64", trace=True)
    tiles = tiles.cpu().numpy()
    uv = tr["uv"].cpu().numpy().astype(np.int64)
    cc = tr["c"].cpu().numpy()
    ref = orc.conceal_blocks(img, blocks, B, border, F, 0.8, 0.5, iters)
    from oracle.gate import window_of
    for k, (_, t, l) in enumerate(blocks):
        s, lab = window_of(img, int(t), int(l), F, B, border)
        o = orc.extrapolate(s, lab, 0.8, 0.5, iters)
        ours = (uv[k, :, 0], uv[k, :, 1], cc[k, :, 0] + 1j * cc[k, :, 1])
        kind, _ = orc.trace_equivalence((o["us"], o["vs"], o["cs"]), ours, F, F)
        if kind in ("identical", "mirror"):
            np.testing.assert_allclose(tiles[k], ref[k], rtol=0, atol=1e-9)
            continue
        at = orc.first_divergence((o["us"], o["vs"], o["cs"]), ours, F, F)
        cert = orc.fp64_tie_certificate(s, lab, 0.8, 0.5, at, ours, (o["us"], o["vs"], o["cs"]))
        assert at is not None and cert["bounded"], (k, kind, cert)
