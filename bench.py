"""Throughput bench: lost 16x16 blocks/s (100 iterations) on B200.

Workload (default): BASELINE.json config 5 -- 256 synthetic 3840x2160 u8
luma frames (1/f^2 field + 8 edges, seeded, generated on the device), 5%
isolated 16x16 losses (1620 per frame, 414,720 total), border 16, FFT 64x64,
100 iterations, rho 0.8, gamma 0.5, fp32.  Frames are sharded across ranks
(contiguous frame ranges, no collective on the data path).

One step = one pass of the fused kernel over every lost block of the rank's
frames, frames resident in HBM (2.1 GB > L2, so no L2 flush is needed).
`e2e` = the same metric through the public host API (Concealer.run: pinned
host frames -> H2D -> kernel -> D2H tiles, copies overlapped with compute).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    # name: frames, H, W, loss fraction, B, border, F, iterations
    "5": dict(frames=256, H=2160, W=3840, frac=0.05, B=16, border=16, F=64, iters=100),
    "3": dict(frames=64, H=1080, W=1920, frac=0.10, B=16, border=16, F=64, iters=200),
}
RHO, GAMMA, SEED = 0.8, 0.5, 5


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="5", choices=sorted(CONFIGS))
    p.add_argument("--frames", type=int, default=None, help="override frame count (debug)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


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
        return d.get(workload, {}).get("dram_bytes_per_block")
    except Exception:
        return None


def make_blocks(cfg, n_frames):
    import numpy as np

    import paper_2204_14193_b200 as fse

    return fse.frames_pattern(n_frames, cfg["H"], cfg["W"], cfg["B"], cfg["frac"], SEED)


def cpu_port(frames_np, blocks, cfg, target_s=12.0, nthreads=None):
    """The oracle port (oracle/, C + OpenMP, fp64) on a bounded sample of the
    same blocks.  Returns (blocks/s, cores, sample description)."""
    import numpy as np

    from oracle import oracle as orc

    cores = nthreads or len(os.sched_getaffinity(0))
    args = (cfg["B"], cfg["border"], cfg["F"], RHO, GAMMA, cfg["iters"])
    n0 = min(len(blocks), 8 * cores)
    t = time.perf_counter()
    orc.conceal_blocks(frames_np, blocks[:n0], *args, nthreads=cores)
    dt = time.perf_counter() - t
    n = int(max(n0, n0 * target_s / max(dt, 1e-3)))
    sample = np.resize(blocks, (n, 3))  # the workload's blocks, cycled if fewer than n
    t = time.perf_counter()
    orc.conceal_blocks(frames_np, sample, *args, nthreads=cores)
    dt = time.perf_counter() - t
    return n / dt, cores, (f"{n} lost blocks ({len(blocks)} distinct, of {frames_np.shape[0]} frames) "
                           f"of the workload in {dt:.1f} s on {cores} threads, fp64")


def run_reference(a, cfg, rank):
    """--impl reference: the reference algorithm's CPU implementation (the
    oracle port; the reference itself is numba/Python and cannot travel to
    the GPU box) on all host cores, same config/metric."""
    if rank != 0:
        return
    import numpy as np

    from paper_2204_14193_b200.synth import frame_u8

    nf = 2
    frames = np.stack([frame_u8(cfg["H"], cfg["W"], seed=1000 + f) for f in range(nf)])
    blocks = make_blocks(cfg, nf)
    cores = len(os.sched_getaffinity(0))
    from oracle import oracle as orc

    args = (cfg["B"], cfg["border"], cfg["F"], RHO, GAMMA, cfg["iters"])
    # size each step to ~2 s of CPU work so steps + warmup finish in well under a minute
    probe = blocks[:min(len(blocks), 4 * cores)]
    t = time.perf_counter()
    orc.conceal_blocks(frames, probe, *args, nthreads=cores)
    rate = len(probe) / max(time.perf_counter() - t, 1e-3)
    n = int(max(len(probe), 2.0 * rate))
    sample = np.resize(blocks, (n, 3))
    for _ in range(a.warmup):
        orc.conceal_blocks(frames, sample, *args, nthreads=cores)
    t = time.perf_counter()
    for _ in range(a.steps):
        orc.conceal_blocks(frames, sample, *args, nthreads=cores)
    dt = time.perf_counter() - t
    v = n * a.steps / dt
    line = {
        "impl": "reference", "metric": "lost_blocks_per_s", "value": v, "unit": "blocks/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": dt / a.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config{a.config}", "frames": cfg["frames"], "H": cfg["H"],
                   "W": cfg["W"], "B": cfg["B"], "border": cfg["border"], "F": cfg["F"],
                   "iterations": cfg["iters"], "rho": RHO, "gamma": GAMMA,
                   "sample_blocks_per_step": n},
        "cpu_baseline": {"value": v, "unit": "blocks/s", "cores": cores, "kind": "port",
                         "sample": f"{n} lost blocks per step (the {len(blocks)} blocks of 2 config frames, cycled), "
                                   f"oracle port (C, fp64), OpenMP over blocks"},
        "e2e": {"value": v, "unit": "blocks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    cfg = dict(CONFIGS[a.config])
    if a.frames:
        cfg["frames"] = a.frames
    rank, world, local = dist_env()
    if a.impl == "reference":
        run_reference(a, cfg, rank)
        return
    import numpy as np
    import torch

    import paper_2204_14193_b200 as fse
    from paper_2204_14193_b200.synth import field_torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2204_14193_b200 import sharding

    all_blocks = make_blocks(cfg, cfg["frames"])
    sh = sharding.shard_blocks(all_blocks, cfg["frames"], rank, world)
    f0, nf, blocks = sh.f0, sh.n_frames, sh.blocks
    frames = field_torch(nf, cfg["H"], cfg["W"], seed=SEED * 7919 + f0, device="cuda")
    geo = fse.Geometry(cfg["B"], cfg["border"], cfg["F"])
    plan = fse.ConcealPlan(blocks, cfg["H"], cfg["W"], geo, rho_hat=RHO, gamma=GAMMA,
                           iterations=cfg["iters"], precision="fp32")
    tiles = torch.empty((len(blocks), cfg["B"], cfg["B"]), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(a.warmup):
        plan.run(frames, tiles)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(a.steps):
            ev[k][0].record(stream)
            plan.run(frames, tiles)
            ev[k][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    elapsed_ms = t0.elapsed_time(t1)
    kern_ms = [s.elapsed_time(e) for s, e in ev]
    mx = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    elapsed_ms = float(mx.item())
    total_blocks = len(all_blocks)
    value = total_blocks * a.steps / (elapsed_ms / 1e3)
    ms_per_step = elapsed_ms / a.steps

    # end to end through the public host API (pinned host frames in, host tiles out)
    e2e = None
    if not a.no_e2e:
        host = frames.cpu().pin_memory()
        con = fse.Concealer(blocks, nf, cfg["H"], cfg["W"], geo, rho_hat=RHO, gamma=GAMMA,
                            iterations=cfg["iters"], precision="fp32",
                            chunk_frames=(int(os.environ["FSE_CHUNK_FRAMES"])
                                          if os.environ.get("FSE_CHUNK_FRAMES") else None))
        for _ in range(max(1, a.warmup)):
            con.run(host)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(a.steps):
            out_tiles = con.run(host)
        et = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device="cuda")
        if dist:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": total_blocks * a.steps / float(et.item()), "unit": "blocks/s",
               "h2d_bytes_per_step": con.h2d_bytes() * world,
               "d2h_bytes_per_step": con.d2h_bytes() * world}
        assert np.array_equal(out_tiles, tiles.cpu().numpy()), "host pipeline differs from device run"

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    # roofline of the dominant kernel (the fused kernel is the only launch per step)
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    F, I = cfg["F"], cfg["iters"]
    smem_bytes_blk = 8.0 * F * F * I  # W' read per bin-iteration
    flops_blk = 11.0 * F * F * I
    kmean = statistics.mean(kern_ms) / 1e3
    achieved = smem_bytes_blk * len(blocks) / kmean / 1e12
    peak_smem = sms * 128 * sm_max * 1e6 / 1e12
    peak_fp32 = sms * 128 * 2 * sm_max * 1e6 / 1e12
    clocks = clk.summary()
    traffic = ncu_traffic(f"config{a.config}")
    ceil = measured_ceilings(int(plan.info.get("threads", 384)))
    line = {
        "metric": "lost_blocks_per_s", "value": value, "unit": "blocks/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"config{a.config}", "frames": cfg["frames"], "H": cfg["H"],
                   "W": cfg["W"], "loss_fraction": cfg["frac"], "blocks": total_blocks,
                   "B": cfg["B"], "border": cfg["border"], "F": F, "iterations": I, "rho": RHO,
                   "gamma": GAMMA, "seed": SEED, "parallelism": f"frames sharded x{world}",
                   "l2": "inputs larger than L2 (2.1 GB frames)" if a.config == "5" else "inputs > L2",
                   "plan": plan.info},
        "roofline": {"bound": "smem", "achieved": achieved, "peak": peak_smem, "unit": "TB/s",
                     "frac": achieved / peak_smem,
                     "traffic": None if traffic is None else traffic * len(blocks),
                     "peak_source": f"derived: {sms} SMs x 128 B/clk x sm_max {sm_max:.0f} MHz "
                                    "(MEASURED_PEAKS.json has no SMEM figure)",
                     "fp32_achieved_tflops": flops_blk * len(blocks) / kmean / 1e12,
                     "fp32_peak_tflops": peak_fp32,
                     "frac_at_observed_clock": (achieved / (sms * 128 * clocks["sm_mhz"] * 1e6 / 1e12))
                     if clocks.get("sm_mhz") else None,
                     "measured_ceilings": ceil,
                     "frac_of_measured_lds128": achieved / ceil["lds128_TBps"] if ceil else None,
                     "frac_of_loop_mix_ceiling": achieved / ceil["loop_mix_TBps"] if ceil else None,
                     "kernel_ms": statistics.mean(kern_ms)},
        "clocks": clocks,
        "gpu_launches": a.steps,
    }
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not a.no_cpu:
        import numpy as np

        fr_np = frames[:4].cpu().numpy()
        sub = blocks[blocks[:, 0] < 4]
        v, cores, sample = cpu_port(fr_np, sub, cfg)
        line["cpu_baseline"] = {"value": v, "unit": "blocks/s", "cores": cores, "kind": "port",
                                "sample": sample}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
