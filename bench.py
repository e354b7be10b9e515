"""Throughput bench: lost 16x16 blocks/s (100 iterations) on B200.

Workload (default): BASELINE.json config 5 -- 256 synthetic 3840x2160 u8
luma frames (1/f^2 field + 8 edges, seeded, generated on the device), 5%
isolated 16x16 losses (1620 per frame, 414,720 total), border 16, FFT 64x64,
100 iterations, rho 0.8, gamma 0.5, fp32.  Frames are sharded across ranks
(contiguous frame ranges, no collective on the data path) and the
reconstructed tiles of every rank land in ONE host buffer (a page-locked
/dev/shm mapping shared by the ranks; each GPU's kernel stores its tiles
straight into its slice).

One step = one pass of the fused kernel over every lost block of the rank's
frames, frames resident in HBM (2.1 GB > L2, so no L2 flush is needed), tiles
stored into the shared host buffer (the gather is inside the timed region).
`e2e` = the same metric through the public host API (Concealer.run: pinned
host frames -> H2D -> kernel -> tiles in the shared host buffer, copies
overlapped with compute).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--gpus N > 1 without an outside launcher re-executes itself under
torch.distributed.run with N ranks (one process per GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    # name: frames, H, W, loss fraction, B, border, F, iterations
    "5": dict(frames=256, H=2160, W=3840, frac=0.05, B=16, border=16, F=64, iters=100),
    "3": dict(frames=64, H=1080, W=1920, frac=0.10, B=16, border=16, F=64, iters=200),
}
RHO, GAMMA, SEED = 0.8, 0.5, 5


def frame_seed(config: str) -> int:
    """Seed of field_torch for frame 0 (rank r generates its frames from
    frame_seed + f0, so frame f of the job is the same at every N)."""
    return (SEED if config == "5" else 3) * 7919


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="5", choices=sorted(CONFIGS))
    p.add_argument("--frames", type=int, default=None, help="override frame count (debug)")
    p.add_argument("--tiles", default="host", choices=["host", "device"],
                   help="where the timed step stores its tiles (host = the shared gather buffer)")
    p.add_argument("--parity-sample", type=int, default=4096,
                   help="blocks of the timed tiles checked against the CPU oracle (0 = off)")
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="weak: every rank conceals the config's full frame count (job = N x frames, "
                        "frames r*frames .. (r+1)*frames on rank r); strong: the config's frames split over the ranks")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    return p.parse_args()


def job_frames(frames: int, world: int, scaling: str) -> int:
    """Frames of the whole job: weak scaling keeps `frames` per rank (the job
    grows with N), strong scaling splits `frames` over the ranks."""
    return frames * (world if scaling == "weak" else 1)


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def self_spawn(a):
    """--gpus N > 1 with no launcher: run N ranks under torch.distributed.run."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    os.execv(sys.executable, cmd)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms during the timed
    region (one `nvidia-smi -lms` process, started before and stopped after)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.15)  # let the first samples land before the timed region
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.06)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        self.samples = [[x.strip() for x in l.split(",")] for l in out.splitlines() if l.strip()]

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        num = lambda x: x.replace(".", "", 1).isdigit()
        sm = [float(s[0]) for s in self.samples if num(s[0])]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and num(s[1])]
        # under load = samples above idle clocks
        load = [x for x in sm if x > 0.5 * max(sm)] if sm else []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def measured_ceilings(threads: int = 384):
    """Shared-memory ceilings measured on this pool's B200s by scripts/smem_peak.cu,
    at the kernel's occupancy: 384 threads x 32 bin pairs (F=64 layout) or
    640 threads x 16 pairs."""
    try:
        rows = [json.loads(l) for l in open(os.path.join(REPO, "profiles", "r01", "smem_peak.jsonl"))]
        sfx, thr = ("_p32", 384) if threads == 384 else ("", 640)
        pick = lambda t: max(r["smem_TBps"] for r in rows if r["test"] == t + sfx and r.get("threads") == thr)
        return {"lds128_TBps": pick("lds128"), "loop_mix_TBps": pick("lds128+6ffma2+argmax"),
                "threads": thr, "source": "profiles/r01/smem_peak.jsonl (scripts/smem_peak.cu)"}
    except Exception:
        return None


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def ncu_traffic(workload: str):
    try:
        with open(os.path.join(REPO, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get(workload, {})
    except Exception:
        return {}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def loaded_native_libs() -> list:
    """Shared objects of this repo mapped into the process (the driver's own
    check of which native code ran)."""
    libs = set()
    try:
        for line in open("/proc/self/maps"):
            path = line.split()[-1] if line.strip() else ""
            if path.endswith(".so") and path.startswith(REPO):
                libs.add(os.path.relpath(path, REPO))
    except Exception:
        pass
    return sorted(libs)


# ------------------------------------------------------------- CPU legs


def cpu_rates(frames_np, blocks, cfg, target_s=10.0):
    """The oracle port (oracle/, C + OpenMP, fp64) on the box's cores: one
    thread on a short sample, then every core on a ~target_s sample of the
    same blocks (distinct blocks, cycled only if the sample outgrows them)."""
    import numpy as np

    from oracle import oracle as orc

    cores = len(os.sched_getaffinity(0))
    args = (cfg["B"], cfg["border"], cfg["F"], RHO, GAMMA, cfg["iters"])
    n1 = min(len(blocks), 48)
    t = time.perf_counter()
    orc.conceal_blocks(frames_np, blocks[:n1], *args, nthreads=1)
    single = n1 / (time.perf_counter() - t)
    n0 = min(len(blocks), 8 * cores)
    t = time.perf_counter()
    orc.conceal_blocks(frames_np, blocks[:n0], *args, nthreads=cores)
    dt = time.perf_counter() - t
    n = int(max(n0, n0 * target_s / max(dt, 1e-3)))
    sample = blocks[:n] if n <= len(blocks) else np.resize(blocks, (n, 3))
    t = time.perf_counter()
    orc.conceal_blocks(frames_np, sample, *args, nthreads=cores)
    dt = time.perf_counter() - t
    return n / dt, single, cores, n, dt


def reference_frames(cfg, config: str, nf: int):
    """The GPU arm's first nf frames (same generator, same seed).  The
    generator is torch (cuFFT on the device when one is present); none of
    this repo's native code is involved."""
    import torch

    from paper_2204_14193_b200.synth import field_torch  # pure torch, no native library

    dev = "cuda" if torch.cuda.is_available() else "cpu"
    fr = field_torch(nf, cfg["H"], cfg["W"], seed=frame_seed(config), device=dev)
    return fr.cpu().numpy(), dev


def run_reference(a, cfg, rank):
    """--impl reference: the reference algorithm's CPU implementation on all
    host cores (the oracle port, C + OpenMP, fp64: the reference itself is
    numba/Python and cannot travel to the GPU box), on this arm's frames
    and block pattern.  Each step conceals every lost block of the first
    `nf` frames of the workload (nf sized to ~1.5 s of CPU work).  Does not
    load the product library (checked)."""
    if rank != 0:
        return
    from oracle import oracle as orc

    nmax = min(16, cfg["frames"])
    frames, gen_dev = reference_frames(cfg, a.config, nmax)
    blocks_all = orc.frames_pattern(nmax, cfg["H"], cfg["W"], cfg["B"], cfg["frac"], SEED if a.config == "5" else 3)
    per_frame = len(blocks_all) // nmax
    cores = len(os.sched_getaffinity(0))
    args = (cfg["B"], cfg["border"], cfg["F"], RHO, GAMMA, cfg["iters"])
    probe = blocks_all[: min(len(blocks_all), 4 * cores)]
    t = time.perf_counter()
    orc.conceal_blocks(frames, probe, *args, nthreads=cores)
    rate = len(probe) / max(time.perf_counter() - t, 1e-3)
    nf = max(1, min(nmax, int(round(1.5 * rate / per_frame))))
    blocks = blocks_all[blocks_all[:, 0] < nf]
    n1 = min(len(blocks), 48)
    t = time.perf_counter()
    orc.conceal_blocks(frames, blocks[:n1], *args, nthreads=1)
    single = n1 / (time.perf_counter() - t)
    # warm-up: the requested steps, and at least ~3 s of all-core work (a fresh
    # box's first seconds of CPU time were measured 40 % slower)
    t = time.perf_counter()
    k = 0
    settle = float(os.environ.get("FSE_REF_SETTLE_S", "3.0"))
    while k < a.warmup or time.perf_counter() - t < settle:
        orc.conceal_blocks(frames, blocks, *args, nthreads=cores)
        k += 1
    t = time.perf_counter()
    for _ in range(a.steps):
        orc.conceal_blocks(frames, blocks, *args, nthreads=cores)
    dt = time.perf_counter() - t
    v = len(blocks) * a.steps / dt
    native = loaded_native_libs()
    assert not any("libfse_b200" in p for p in native), f"reference arm loaded the product: {native}"
    line = {
        "impl": "reference", "metric": "lost_blocks_per_s", "value": v, "unit": "blocks/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": dt / a.steps * 1e3, "higher_is_better": True, "scaling": a.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config{a.config}", "frames": cfg["frames"], "H": cfg["H"],
                   "W": cfg["W"], "loss_fraction": cfg["frac"], "B": cfg["B"], "border": cfg["border"],
                   "F": cfg["F"], "iterations": cfg["iters"], "rho": RHO, "gamma": GAMMA,
                   "seed": SEED, "frames_per_step": nf, "blocks_per_step": int(len(blocks))},
        "cpu_baseline": {"value": v, "unit": "blocks/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(), "single_core_blocks_per_s": single,
                         "sample": f"every lost block of the workload's first {nf} frame(s) "
                                   f"({len(blocks)} blocks, field_torch frames on {gen_dev}, seed "
                                   f"{frame_seed(a.config)}; same loss pattern as the GPU arm) per step; "
                                   "oracle port (C, fp64), OpenMP over blocks"},
        "e2e": {"value": v, "unit": "blocks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "native_libs_loaded": native,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU arm


def parity_sample(fse, plan_kw, frames_dev, blocks, timed_tiles, cfg, n_sample):
    """Outside the timed region: re-run an evenly spaced sample of the
    rank's blocks (up to 32 frames spread over the rank's range, blocks
    evenly spaced among them) with f32 tiles + trace, check that rounding them gives the
    timed u8 tiles bit for bit, and gate them against the CPU oracle
    (oracle/gate.py: per block |dpx| <= 0.5 except certified near-ties,
    pooled PSNR within 0.01 dB)."""
    import numpy as np
    import torch

    from oracle.gate import fp32_gate

    nfr = int(blocks[:, 0].max()) + 1 if len(blocks) else 0
    pick_f = np.unique(np.linspace(0, max(nfr - 1, 0), min(nfr, 32)).round().astype(np.int32))
    cand = np.nonzero(np.isin(blocks[:, 0], pick_f))[0]
    n = min(n_sample, len(cand))
    idx = cand[np.unique(np.linspace(0, len(cand) - 1, n).round().astype(np.int64))]
    sb = blocks[idx]
    plan = fse.ConcealPlan(sb, cfg["H"], cfg["W"], **plan_kw)
    tiles, tr = plan.run(frames_dev, tile_dtype="f32", trace=True)
    t32 = tiles.cpu().numpy()
    same_u8 = bool(np.array_equal(np.rint(np.clip(t32, 0, 255)).astype(np.uint8), timed_tiles[idx]))
    uv = tr["uv"].cpu().numpy()
    c = tr["c"].cpu().numpy()
    get = lambda k: (uv[k, :, 0].astype(np.int64), uv[k, :, 1].astype(np.int64), c[k, :, 0] + 1j * c[k, :, 1])
    used = np.unique(sb[:, 0])
    fr = frames_dev[torch.as_tensor(used, device=frames_dev.device)].cpu().numpy()
    remap = np.zeros(int(used.max()) + 1, np.int32)
    remap[used] = np.arange(len(used), dtype=np.int32)
    lb = sb.copy()
    lb[:, 0] = remap[sb[:, 0]]
    B = cfg["B"]
    truth = np.stack([fr[f, t:t + B, l:l + B] for f, t, l in lb]).astype(np.float64)
    ok, err = True, None
    try:
        st = fp32_gate(fr, lb, t32, get, cfg["F"], B, cfg["border"], RHO, GAMMA, cfg["iters"], truth=truth)
    except AssertionError as e:  # report, do not hide: the line says parity failed
        ok, err, st = False, str(e)[:300], {}
    return {"blocks": int(len(sb)), "frames": int(len(used)), "timed_u8_equal": same_u8,
            "max_dev": st.get("max_dev"), "over_0p5": st.get("over"), "certified_strict": st.get("strict"),
            "certified_bounded": st.get("bounded"), "psnr_delta_db": st.get("psnr_delta"),
            "passed": bool(ok and same_u8), "error": err,
            "gate": "per block max|dpx| <= 0.5 vs fp64 oracle except certified near-ties; "
                    "pooled PSNR within 0.01 dB"}


def main():
    a = parse()
    cfg = dict(CONFIGS[a.config])
    if a.frames:
        cfg["frames"] = a.frames
    rank, world, local = dist_env()
    if a.impl == "reference":
        run_reference(a, cfg, rank)
        return
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_spawn(a)
    assert world == a.gpus, f"--gpus {a.gpus} but WORLD_SIZE {world}"
    import numpy as np
    import torch

    import paper_2204_14193_b200 as fse
    from paper_2204_14193_b200 import sharding
    from paper_2204_14193_b200.synth import field_torch

    # FSE_BENCH_SHARE_GPU=1: a functional check of the N-rank flow on a box
    # with fewer GPUs (ranks share devices round-robin, gloo for the barriers
    # and the max-over-ranks reduction); its numbers are not scaling numbers
    share = os.environ.get("FSE_BENCH_SHARE_GPU") == "1"
    dev_index = local % torch.cuda.device_count() if share else local
    torch.cuda.set_device(dev_index)
    dist = None
    red_dev = "cuda"
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
            red_dev = "cpu"
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # weak scaling (default): per-GPU work fixed, the job grows with N; every
    # frame f of the job is the same at every N (per-frame seeds)
    n_job = job_frames(cfg["frames"], world, a.scaling)
    all_blocks = fse.frames_pattern(n_job, cfg["H"], cfg["W"], cfg["B"], cfg["frac"],
                                    SEED if a.config == "5" else 3)
    sh = sharding.shard_blocks(all_blocks, n_job, rank, world)
    f0, nf, blocks = sh.f0, sh.n_frames, sh.blocks
    lo, hi = sharding.contiguous_range(sh)
    frames = field_torch(nf, cfg["H"], cfg["W"], seed=frame_seed(a.config) + f0, device="cuda")
    geo = fse.Geometry(cfg["B"], cfg["border"], cfg["F"])
    plan_kw = dict(geometry=geo, rho_hat=RHO, gamma=GAMMA, iterations=cfg["iters"], precision="fp32")
    plan = fse.ConcealPlan(blocks, cfg["H"], cfg["W"], **plan_kw)

    # one host tile buffer for the whole job, shared by the ranks of the box
    tag = os.environ.get("MASTER_PORT", str(os.getpid()))
    path = f"/dev/shm/fse_bench_tiles_{tag}"
    if rank == 0:
        gbuf = sharding.HostTileBuffer(path, (len(all_blocks), cfg["B"], cfg["B"]), torch.uint8, create=True)
    if dist:
        dist.barrier()
    if rank != 0:
        gbuf = sharding.HostTileBuffer(path, (len(all_blocks), cfg["B"], cfg["B"]), torch.uint8, create=False)
    host_slice = gbuf.slice(lo, hi)
    tiles = host_slice if a.tiles == "host" else torch.empty(
        (len(blocks), cfg["B"], cfg["B"]), dtype=torch.uint8, device="cuda")

    stream = torch.cuda.current_stream()
    for _ in range(a.warmup):
        plan.run(frames, tiles)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev_index) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(a.steps):
            ev[k][0].record(stream)
            plan.run(frames, tiles)
            ev[k][1].record(stream)
        if a.tiles == "device":  # the gather: tiles into the shared host buffer
            host_slice.copy_(tiles, non_blocking=True)
        t1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    elapsed_ms = t0.elapsed_time(t1)
    kern_ms = [s.elapsed_time(e) for s, e in ev]
    mx = torch.tensor([elapsed_ms], dtype=torch.float64, device=red_dev)
    if dist:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    elapsed_ms = float(mx.item())
    total_blocks = len(all_blocks)
    value = total_blocks * a.steps / (elapsed_ms / 1e3)
    ms_per_step = elapsed_ms / a.steps
    timed_tiles = host_slice.numpy().copy()

    # end to end through the public host API (pinned host frames in, tiles
    # into this rank's slice of the shared host buffer)
    e2e = None
    if not a.no_e2e:
        host = frames.cpu().pin_memory()
        con = fse.Concealer(blocks, nf, cfg["H"], cfg["W"], geo, rho_hat=RHO, gamma=GAMMA,
                            iterations=cfg["iters"], precision="fp32",
                            chunk_frames=(int(os.environ["FSE_CHUNK_FRAMES"])
                                          if os.environ.get("FSE_CHUNK_FRAMES") else None))
        host_slice.zero_()
        for _ in range(max(1, a.warmup)):
            con.run(host, out=host_slice)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(a.steps):
            con.run(host, out=host_slice)
        et = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device=red_dev)
        if dist:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": total_blocks * a.steps / float(et.item()), "unit": "blocks/s",
               "h2d_bytes_per_step": con.h2d_bytes() * world,
               "d2h_bytes_per_step": con.d2h_bytes() * world,
               "path": "Concealer.run: pinned host frames -> H2D (copy stream) -> fused kernel -> "
                       "tiles stored into the shared pinned host buffer"}
        assert np.array_equal(host_slice.numpy(), timed_tiles), "host pipeline differs from device run"

    parity = None
    if a.parity_sample and rank == 0:
        parity = parity_sample(fse, plan_kw, frames, blocks, timed_tiles, cfg, a.parity_sample)
    if dist:
        dist.barrier()
    gathered_ok = None
    if rank == 0:
        # every rank's tiles are in the one buffer: spot-check a block of the last rank's range
        gathered_ok = bool(np.count_nonzero(gbuf.numpy()[-1]) > 0) if len(all_blocks) else True
    if rank != 0:
        gbuf.close()
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return
    if dist:
        dist.barrier()
    gbuf.close(unlink=True)

    # roofline of the dominant kernel (the fused kernel is the only launch per step)
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(dev_index).multi_processor_count
    F, I = cfg["F"], cfg["iters"]
    smem_bytes_blk = 8.0 * F * F * I  # W' read per bin-iteration
    flops_blk = 11.0 * F * F * I
    kmean = statistics.mean(kern_ms) / 1e3
    achieved = smem_bytes_blk * len(blocks) / kmean / 1e12
    peak_smem = sms * 128 * sm_max * 1e6 / 1e12
    peak_fp32 = sms * 128 * 2 * sm_max * 1e6 / 1e12
    clocks = clk.summary()
    nt = ncu_traffic(f"config{a.config}")
    ceil = measured_ceilings(int(plan.info.get("threads", 384)))
    line = {
        "metric": "lost_blocks_per_s", "value": value, "unit": "blocks/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"config{a.config}", "frames": n_job, "frames_per_gpu": nf, "H": cfg["H"],
                   "W": cfg["W"], "loss_fraction": cfg["frac"], "blocks": total_blocks,
                   "B": cfg["B"], "border": cfg["border"], "F": F, "iterations": I, "rho": RHO,
                   "gamma": GAMMA, "seed": SEED, "parallelism": f"frames sharded x{world}",
                   "l2": "inputs larger than L2 (2.1 GB frames)" if a.config == "5" else "inputs > L2",
                   "tiles": ("kernel stores u8 tiles into the shared pinned host buffer (gather inside "
                             "the timed region)") if a.tiles == "host" else
                            "device tiles, one D2H into the shared host buffer at the end of the timed region",
                   "plan": plan.info},
        "roofline": {"bound": "smem", "scope": "per GPU: rank 0's blocks / its kernel time",
                     "achieved": achieved, "peak": peak_smem, "unit": "TB/s",
                     "frac": achieved / peak_smem,
                     "traffic": (nt["dram_bytes_per_block"] * len(blocks)) if nt.get("dram_bytes_per_block") else None,
                     "traffic_source": nt.get("source"),
                     "peak_source": f"derived: {sms} SMs x 128 B/clk x sm_max {sm_max:.0f} MHz "
                                    "(MEASURED_PEAKS.json has no SMEM figure)",
                     "fp32_achieved_tflops": flops_blk * len(blocks) / kmean / 1e12,
                     "fp32_peak_tflops": peak_fp32,
                     "frac_at_observed_clock": (achieved / (sms * 128 * clocks["sm_mhz"] * 1e6 / 1e12))
                     if clocks.get("sm_mhz") else None,
                     "measured_ceilings": ceil,
                     "frac_of_measured_lds128": achieved / ceil["lds128_TBps"] if ceil else None,
                     "frac_of_loop_mix_ceiling": achieved / ceil["loop_mix_TBps"] if ceil else None,
                     "kernel_ms": statistics.mean(kern_ms),
                     "algorithmic_smem_bytes_per_block": smem_bytes_blk,
                     "kernel_scan_smem_bytes_per_block": {
                         "centred_classes": 4.0 * F * F * I, "other_classes": smem_bytes_blk},
                     "note": ("achieved counts the algorithm's W' traffic (8 B per bin-iteration, SURVEY 8(d)); "
                              "the kernel's centred-frame loop reads a real table, 4 B per bin-iteration, for "
                              "mirror-symmetric (interior) classes, so the shared-memory pipe itself runs at "
                              "about half this rate and the loop is issue/latency-bound (DESIGN 4.1)")},
        "clocks": clocks,
        "gpu_launches": a.steps * 1,
        "gather": {"buffer": "one /dev/shm mapping, page-locked by every rank", "bytes": int(gbuf.nbytes),
                   "last_block_nonzero": gathered_ok},
    }
    if share:
        line["shared_gpus"] = (f"FSE_BENCH_SHARE_GPU: {world} ranks on {torch.cuda.device_count()} device(s); "
                               "a functional check of the N-rank flow, not a scaling number")
    if e2e:
        line["e2e"] = e2e
    if parity:
        line["parity"] = parity
    if world == 1 and not a.no_cpu:
        sub_f = 4
        fr_np = frames[:sub_f].cpu().numpy()
        sub = blocks[blocks[:, 0] < sub_f]
        v, single, cores, n, dt = cpu_rates(fr_np, sub, cfg)
        line["cpu_baseline"] = {"value": v, "unit": "blocks/s", "cores": cores, "kind": "port",
                                "cpu_model": cpu_model(), "single_core_blocks_per_s": single,
                                "sample": f"{n} lost blocks of the workload's first {sub_f} frames "
                                          f"({len(sub)} distinct) in {dt:.1f} s on {cores} threads, "
                                          "oracle port (C, fp64)"}
    line["native_libs_loaded"] = loaded_native_libs()
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
