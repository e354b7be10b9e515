"""`fse` command line: conceal / sweep / bench / selfcheck.

    python -m paper_2204_14193_b200.cli conceal --input in.pgm --output out.pgm \
        [--algo cfse] [--block 16] [--support 16] [--stride 64] [--fft 64] \
        [--rho 0.8] [--gamma 0.2] [--iters 100] [--seed 0] [--precision fp64|fp32] \
        [--report r.csv] [--damage d.pgm]
    python -m paper_2204_14193_b200.cli sweep --input in.pgm --bf-counts 10,20,50,100 --report s.csv
    python -m paper_2204_14193_b200.cli bench [--bf-counts 0,10,100,1000] [--blocks 4096]
    python -m paper_2204_14193_b200.cli selfcheck

Exit codes: 0 success, 1 runtime error, 2 usage / configuration error.
All compute runs on the GPU (libfse_b200); the CLI is I/O and orchestration.
"""
from __future__ import annotations

import argparse
import csv
import io
import math
import sys
import time

import numpy as np

from .errors import ConfigError, FseError, PgmError


def _common(p):
    p.add_argument("--algo", default="cfse", choices=["cfse", "rfse"])
    p.add_argument("--block", type=int, default=16)
    p.add_argument("--support", type=int, default=16)
    p.add_argument("--stride", type=int, default=64)
    p.add_argument("--fft", type=int, default=64)
    p.add_argument("--rho", type=float, default=0.8)
    p.add_argument("--gamma", type=float, default=0.2)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])


def parser():
    ap = argparse.ArgumentParser(prog="fse", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("conceal")
    c.add_argument("--input", required=True)
    c.add_argument("--output", required=True)
    c.add_argument("--iters", type=int, default=100)
    c.add_argument("--report")
    c.add_argument("--damage")
    _common(c)
    s = sub.add_parser("sweep")
    s.add_argument("--input", required=True)
    s.add_argument("--bf-counts", default="10,20,50,100,200,500")
    s.add_argument("--report")
    _common(s)
    b = sub.add_parser("bench")
    b.add_argument("--bf-counts", default="0,10,20,50,100,200,500,1000,2000")
    b.add_argument("--blocks", type=int, default=4096)
    b.add_argument("--repetitions", type=int, default=5)
    b.add_argument("--report")
    _common(b)
    k = sub.add_parser("selfcheck")
    k.add_argument("--seed", type=int, default=0)
    k.add_argument("--instances", type=int, default=50)
    return ap


def _config(a, iters):
    from .types import FseConfig

    return FseConfig(rho_hat=a.rho, gamma=a.gamma, iterations=max(iters, 1), fft_dims=(a.fft, a.fft),
                     algorithm=a.algo, basis_target=iters if iters == 0 else None,
                     precision=a.precision)


def _conceal_once(img, pattern, a, bf):
    """Conceal `pattern` in `img` with a selected-basis-function budget `bf`
    (cFSE: one basis function per iteration, cfse.py:141)."""
    from .harness import Geometry, conceal_frames

    geo = Geometry(a.block, a.support, a.fft)
    _config(a, bf)  # validates the parameters (ConfigError)
    tdt = "f64" if a.precision == "fp64" else "f32"
    t = time.perf_counter()
    # rFSE: stop at `bf` basis functions (2 per pair pick, rfse.py:184-189)
    tiles = conceal_frames(img, pattern, geo, rho_hat=a.rho, gamma=a.gamma, iterations=bf,
                           precision=a.precision, tile_dtype=tdt, algorithm=a.algo,
                           basis_target=bf if a.algo == "rfse" else None)
    dt = time.perf_counter() - t
    return tiles, dt


def _block_psnr(orig_tile, tile):
    d = orig_tile.astype(np.float64) - np.clip(tile, 0, 255)
    mse = float(np.mean(d * d))
    return math.inf if mse == 0 else 10 * math.log10(255.0 ** 2 / mse)


def _report_rows(algo, bf, img, pattern, tiles, dt, B):
    rows = []
    for k, (t, l) in enumerate(pattern):
        rows.append([algo, bf, k, _block_psnr(img[t:t + B, l:l + B], tiles[k]), dt / max(len(pattern), 1)])
    from .harness import psnr_tiles

    truth = np.stack([img[t:t + B, l:l + B] for t, l in pattern]).astype(np.float64)
    rows.append([algo, bf, "pooled", psnr_tiles(truth, np.clip(tiles, 0, 255)), dt / max(len(pattern), 1)])
    return rows


def _write_csv(path, header, rows):
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(header)
    for r in rows:
        w.writerow([f"{x:.6g}" if isinstance(x, float) and math.isfinite(x) else x for x in r])
    if path:
        with open(path, "w") as f:
            f.write(buf.getvalue())
    return buf.getvalue()


def cmd_conceal(a):
    from .harness import grid_pattern, write_tiles
    from .pgm import load_image, save_image

    img = load_image(a.input)
    pattern = grid_pattern(img.shape[0], img.shape[1], a.block, a.stride, a.support, a.seed)
    if a.damage:
        dmg = img.copy()
        for t, l in pattern:
            dmg[t:t + a.block, l:l + a.block] = 0
        save_image(dmg, a.damage)
    tiles, dt = _conceal_once(img, pattern, a, a.iters)
    out = write_tiles(img, pattern, np.rint(np.clip(tiles, 0, 255)).astype(np.uint8), a.block)
    save_image(out, a.output)
    if a.report:
        _write_csv(a.report, ["algo", "bf_count", "block_index", "psnr_db", "sec_per_block"],
                   _report_rows(a.algo, a.iters, img, pattern, tiles, dt, a.block))
    return 0


def cmd_sweep(a):
    from .harness import grid_pattern
    from .pgm import load_image

    img = load_image(a.input)
    pattern = grid_pattern(img.shape[0], img.shape[1], a.block, a.stride, a.support, a.seed)
    rows = []
    for bf in [int(x) for x in a.bf_counts.split(",") if x]:
        tiles, dt = _conceal_once(img, pattern, a, bf)
        rows += _report_rows(a.algo, bf, img, pattern, tiles, dt, a.block)
    hdr = ["algo", "bf_count", "block_index", "psnr_db", "sec_per_block"]
    _write_csv(a.report, hdr, rows)  # full per-block report
    sys.stdout.write(_write_csv(None, hdr, [r for r in rows if r[2] == "pooled"]))
    return 0


def cmd_bench(a):
    """Fig. 3 analogue on the GPU: time per block versus the
    selected-basis-function count, median of repetitions, on one fixed
    synthetic block instance replicated `--blocks` times.  Rows:
      cfse-fused  -- the fused register-resident fp32 kernel (the product path)
      rfse-fused  -- its conjugate-pair variant (F = 64), basis_target = count
      cfse, rfse  -- the per-window kernels (same structure for both variants,
                     so their ratio is the paper's loop-structure comparison)."""
    import torch

    from .cfse import extrapolate_cfse_batch
    from .harness import ConcealPlan, Geometry
    from .rfse import extrapolate_rfse_batch
    from .synth import frame_u8
    from .types import FseConfig
    from .weighting import build_mask

    H = W = 1024
    img = frame_u8(H, W, seed=a.seed)
    fr = torch.from_numpy(img).cuda()
    geo = Geometry(a.block, a.support, a.fft)
    off = (a.fft - a.block) // 2
    t0 = l0 = 496
    win = img[t0 - off:t0 - off + a.fft, l0 - off:l0 - off + a.fft].astype(np.float64)
    labels = build_mask((a.fft, a.fft), (off, off, a.block, a.block), a.support).labels
    n = a.blocks
    wins = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(win, (n,) + win.shape))).cuda()
    blocks = np.tile(np.array([[0, t0, l0]], np.int32), (n, 1))
    prec = a.precision

    def timeit(run):
        run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(a.repetitions, 5)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3 / n)
        return float(np.median(ts)), float(np.min(ts)), len(ts)

    rows = []
    for bf in [int(x) for x in a.bf_counts.split(",") if x]:
        if bf > 0 and prec == "fp32":
            plan = ConcealPlan(blocks, H, W, geo, rho_hat=a.rho, gamma=a.gamma, iterations=bf,
                               precision="fp32")
            if plan.info["fast_path"]:
                rows.append(["cfse-fused", bf, *timeit(lambda: plan.run(fr, tile_dtype="f32"))])
            if a.fft == 64:
                rplan = ConcealPlan(blocks, H, W, geo, rho_hat=a.rho, gamma=a.gamma, iterations=bf,
                                    basis_target=bf, precision="fp32", algorithm="rfse")
                if rplan.info["fast_path"]:
                    rows.append(["rfse-fused", bf, *timeit(lambda: rplan.run(fr, tile_dtype="f32"))])
        cfg = FseConfig(rho_hat=a.rho, gamma=a.gamma, iterations=max(bf, 1), fft_dims=(a.fft, a.fft),
                        basis_target=bf if bf == 0 else None, precision=prec)
        rows.append(["cfse", bf, *timeit(lambda: extrapolate_cfse_batch(wins, labels, cfg))])
        cfg_r = FseConfig(rho_hat=a.rho, gamma=a.gamma, iterations=max(bf, 1), fft_dims=(a.fft, a.fft),
                          algorithm="rfse", basis_target=bf, precision=prec)
        rows.append(["rfse", bf, *timeit(lambda: extrapolate_rfse_batch(wins, labels, cfg_r))])
    sys.stdout.write(_write_csv(a.report, ["algo", "bf_count", "sec_per_block_median",
                                           "sec_per_block_min", "repetitions"], rows))
    return 0


def cmd_selfcheck(a):
    """the oracle-equivalence and energy-identity suites on
    seeded random instances (selfcheck.run: the production frequency-domain
    GPU path against the spatial-domain brute force, csrc/spatial.cu, for
    cFSE and rFSE), then internal consistency checks: DFT round trip and
    Parseval, energy identity of a 64 x 64 trace, scale equivariance,
    support samples unchanged, fp32 vs fp64 agreement.  PASS/FAIL per
    invariant; exit 0 only if every one passes."""
    from . import cfse, spectral
    from . import selfcheck as sc
    from .types import FseConfig
    from .weighting import build_mask, build_weight

    seed = getattr(a, "seed", 0)
    rng = np.random.default_rng(seed)
    ok = True

    def check(name, cond, detail=""):
        nonlocal ok
        print(f"{'PASS' if cond else 'FAIL'} {name}" + (f"  [{detail}]" if detail != "" else ""))
        ok &= bool(cond)

    for name, passed, detail in sc.run(seed=seed, n=getattr(a, "instances", 50)):
        check(name, passed, detail)

    x = rng.standard_normal((16, 16)) + 1j * rng.standard_normal((16, 16))
    X = spectral.dft2(x)
    check("dft2/idft2 round trip <= 1e-10", np.max(np.abs(spectral.idft2(X) - x)) <= 1e-10 * np.abs(x).max())
    check("Parseval <= 1e-9", abs(np.sum(abs(x) ** 2) - np.sum(abs(X) ** 2) / x.size) <= 1e-9 * np.sum(abs(x) ** 2))
    mask = build_mask((64, 64), (24, 24, 16, 16), 16)
    s = rng.uniform(0, 255, (64, 64))
    cfg = FseConfig(rho_hat=0.8, gamma=0.2, iterations=60)
    r = cfse.extrapolate_cfse(s, mask, cfg)
    w = build_weight(mask, 0.8)
    g = r.model
    e_direct = float(np.sum(w * np.abs(s - g) ** 2))
    check("energy identity (trace vs direct) <= 1e-9 rel", abs(r.trace[-1].residual_energy - e_direct) <= 1e-9 * np.sum(w * s * s))
    r3 = cfse.extrapolate_cfse(3 * s, mask, cfg)
    same = all(t.frequency == u.frequency for t, u in zip(r.trace, r3.trace))
    check("scale equivariance (selections, 3x coefficients)", same and all(
        abs(u.coefficient - 3 * t.coefficient) <= 1e-9 * abs(3 * t.coefficient) for t, u in zip(r.trace, r3.trace)))
    check("support/padding samples unchanged", np.array_equal(r.reconstructed[~mask.loss], s[~mask.loss]))
    r32 = cfse.extrapolate_cfse(s, mask, FseConfig(rho_hat=0.8, gamma=0.2, iterations=60, precision="fp32"))
    check("fp32 vs fp64 loss pixels <= 0.5", np.max(np.abs(r32.reconstructed - r.reconstructed)) <= 0.5)
    return 0 if ok else 1


def main(argv=None) -> int:
    ap = parser()
    a = ap.parse_args(argv)
    try:
        return {"conceal": cmd_conceal, "sweep": cmd_sweep, "bench": cmd_bench,
                "selfcheck": cmd_selfcheck}[a.cmd](a)
    except (ConfigError, PgmError) as e:
        print(f"fse: error: {e}", file=sys.stderr)
        return 2
    except FileNotFoundError as e:
        print(f"fse: error: {e}", file=sys.stderr)
        return 1
    except FseError as e:
        print(f"fse: error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
