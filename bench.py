#!/usr/bin/env python3
"""bench.py -- Mrays/s of the B200 per-ray higher-order SPH DVR path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One step = one full frame of BASELINE.json config C (default 3: the 16M
clustered cosmology-like particle set, 2048^2 image -- the workload the
north-star metric is quoted on at 1/2/4/8 B200), rendered by the sm_100a path
with the particle set resident in HBM.  Under torchrun (N > 1) image tiles are
interleaved over ranks and gathered with NCCL inside the library (strong
scaling: the frame is fixed); timing is CUDA events on the library's stream,
bracketed by barrier + synchronize, max over ranks.  Prints ONE JSON line on
rank 0.

--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified reference headers, render_scene<int64_t> with every host
thread) on a bounded row-band sample of the same frame, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mrays/s (SPH higher-order ray approx + DVR) at 1/2/4/8 B200, % HBM roofline"
SYNTH_TF = np.array([[0.0, 0.02, 0.02, 0.10, 0.0], [0.2, 0.05, 0.10, 0.45, 0.35],
                     [0.6, 0.10, 0.35, 0.80, 0.9], [1.0, 1.0, 0.85, 0.30, 2.4]])
CONFIGS = {
    1: dict(n=100_000, res=256, desc="1e5-particle Gaussian blob, uniform h=0.062, 256^2"),
    2: dict(n=1_000_000, res=1024, desc="1M-particle Gaussian blob, uniform h=0.029, 1024^2"),
    3: dict(n=16_777_216, res=2048, desc="16M clustered (256 Plummer halos + 10% background), h from analytic density, 2048^2"),
    4: dict(n=4_194_304, res=1024, desc="4M Gaussian blob, 1024^2 (order sweep member)"),
    5: dict(n=100_000_000, res=4096, desc="100M clustered, 4096^2"),
}


def camera_kwargs(res, band=None):
    """SURVEY.md 8(d) orthographic camera; `band` = (y0, rows) gives the
    sub-camera covering those rows (same pixel pitch) for CPU samples."""
    kw = dict(mode="orthographic", position=(0.0, 0.0, 8.0), look_at=(0.0, 0.0, 0.0),
              up=(0.0, 1.0, 0.0), width=res, height=res, ortho_height=6.0, near=0.0, far=1e30)
    if band is not None:
        y0, rows = band
        hh = 0.5 * 6.0
        v = 1.0 - ((y0 + rows / 2.0) / res) * 2.0
        kw.update(height=rows, ortho_height=6.0 * rows / res, position=(0.0, v * hh, 8.0),
                  look_at=(0.0, v * hh, 0.0))
    return kw


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_traffic(config, res, world):
    """DRAM bytes (read + write) of one main render launch on this workload,
    from the committed ncu capture (profiles/r01_render_traffic.json, made by
    scripts/gpu_round.sh); None when absent or for another workload."""
    path = os.path.join(ROOT, "profiles", "r01_render_traffic.json")
    try:
        d = json.load(open(path))
    except (OSError, ValueError):
        return None
    if d.get("config") != config or d.get("res") != res or d.get("world", 1) != world:
        return None
    return d


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0}, "fallback"


def lut_file(args=None):
    """The LUT of the run: cubic B-spline, K pieces, degree D, 1024 entries
    (config 4's order sweep varies K and D; every other config is K=4, D=3)."""
    K = getattr(args, "K", 4) if args is not None else 4
    D = getattr(args, "D", 3) if args is not None else 3
    return os.path.join(ROOT, "data", "luts", f"cubic_K{K}_D{D}_N1024.splt")


def setup_scene(cfg, n_override=0, args=None):
    import paper_2401_02896_b200 as S

    c = CONFIGS[cfg]
    n = n_override or c["n"]
    t0 = time.time()
    ps = S.generate_scene(cfg, n=n)
    lut = S.load_lut(lut_file(args))
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    return ps, lut, ds, qc, time.time() - t0


# --------------------------------------------------------------------------- CPU reference
def cpu_reference_sample(ps, lut_path, ds, qc, res, budget_s=20.0, threads=None):
    """render_scene<int64_t> of the UNMODIFIED reference (oracle/_ref) on row
    bands of the frame; falls back to Int128 on its spurious OverflowError."""
    from oracle import ref

    threads = threads or os.cpu_count() or 1
    rl = ref.Lut(lut_path)
    rds = ref.RpDStats(ds.mass_r, ds.density_r, ds.h_r, ds.value_r, ds.phi_repr, ds.a_max,
                       ds.clustering_factor, ds.count)
    rqc = ref.RpQuanta(qc.tau, qc.sigma, 64)
    rows_done, secs, bits_used, bands = 0, 0.0, set(), []
    # evenly spaced single rows, centre first, until the time budget is used
    order = [res // 2] + [int(res * (i + 0.5) / 8) for i in range(8)]
    for y in order:
        if secs >= budget_s and rows_done > 0:
            break
        cam = ref.Camera(**camera_kwargs(res, band=(y, 1)))
        try:
            _, st, sec = ref.render(ps, cam, SYNTH_TF, rl, rqc, rds, 0.0, (0, 0, 0), threads, 64)
            bits_used.add(64)
        except ref.RefError as e:
            if e.code != 3:
                raise
            _, st, sec = ref.render(ps, cam, SYNTH_TF, rl, rqc, rds, 0.0, (0, 0, 0), threads, 128)
            bits_used.add(128)
        rows_done += 1
        secs += sec
        bands.append(y)
    rays = rows_done * res
    return dict(value=rays / secs / 1e6, unit="Mrays/s", cores=threads, kind="reference",
                sample=f"{rows_done} full-width row(s) {bands} of the {res}^2 frame via "
                       f"render_scene<int{'/'.join(str(b) for b in sorted(bits_used))}> on a "
                       f"row-band camera; {rays} rays in {secs:.2f} s",
                seconds=secs)


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import ref

    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs "
                          "/root/reference at build time)"}))
        return
    cfg = args.config
    res = args.res or CONFIGS[cfg]["res"]
    ps, lut, ds, qc, _ = setup_scene(cfg, args.n, args)
    lut_path = lut_file(args)
    times = []
    per_step_budget = args.ref_step_budget
    for i in range(args.warmup + args.steps):
        r = cpu_reference_sample(ps, lut_path, ds, qc, res, budget_s=per_step_budget)
        if i >= args.warmup:
            times.append(r)
    secs = sum(t["seconds"] for t in times)
    rays = sum(t["value"] * 1e6 * t["seconds"] for t in times)
    value = rays / secs / 1e6
    out = {"metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / len(times),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": f"config {cfg}: {CONFIGS[cfg]['desc']}", "particles": len(ps),
                      "image": f"{res}x{res}", "K": args.K, "D": args.D, "N_lut": 1024, "int_width": 64},
           "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": times[0]["cores"],
                            "kind": "reference", "sample": times[0]["sample"]},
           "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2401_02896_b200 as S
    from paper_2401_02896_b200 import dist as SD

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    res = args.res or CONFIGS[cfg]["res"]
    ps, lut, ds, qc, setup_s = setup_scene(cfg, args.n, args)
    ctx = S.Context(local)
    SD.init_comm(ctx, rank, world)
    cam = S.Camera(**camera_kwargs(res))
    tf = S.TransferFunction.from_array(SYNTH_TF)
    opts = S.RenderOptions(mode=S.MODE_FAST if args.mode == "fast" else S.MODE_EXACT,
                           window=args.window)
    ctx.upload(ps, lut)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr())
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (also module loading / first touch of every buffer, the flush included)
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        _, st = ctx.render(cam, tf, qc, ds, opts, to_host=False)

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(1.0)
    per_step, walls = [], []
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        tw = time.perf_counter()
        with torch.cuda.stream(stream):
            flush.fill_(1.0)  # L2 flush (256 MB > 126 MB L2) between frames
        _, st = ctx.render(cam, tf, qc, ds, opts, to_host=False)
        per_step.append(st)
        walls.append(1e3 * (time.perf_counter() - tw))
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    rays = res * res * args.steps
    value = rays / (ms_max * 1e-3) / 1e6
    render_ms = statistics.median(s.render_ms for s in per_step)
    bin_ms = statistics.median(s.bin_ms for s in per_step)
    st = per_step[-1]

    # ---- e2e: the public one-shot API (render_scene) with host buffers
    e2e = None
    if args.e2e_steps > 0:
        S.render_scene(ps, cam, tf, lut, qc, ds, opts, ctx=ctx)  # warm
        barrier()
        t0 = time.perf_counter()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            img, _ = S.render_scene(ps, cam, tf, lut, qc, ds, opts, ctx=ctx)
        f1.record(stream)
        barrier()
        e2e_ms = f0.elapsed_time(f1)
        wall = time.perf_counter() - t0
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
        h2d = len(ps) * (56 + 8 * lut.D) + lut.records().nbytes + SYNTH_TF.nbytes
        d2h = res * res * 3 * 8
        e2e = {"value": res * res * args.e2e_steps / (e2e_ms * 1e-3) / 1e6, "unit": "Mrays/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_ms / args.e2e_steps, "wall_s": wall,
               "api": "sphray_render_scene (one-shot drop-in for render_scene<int64_t>)"}
        # ctx scene was replaced by the one-shot call with the same particles: fine

    # ---- roofline of the dominant kernel (the render kernel)
    peaks, peak_src = measured_peaks()
    D = lut.D
    per_particle = 32 + 16 + 4 + 24 * D  # x,y,z,h + bbox + front + X_d, Y_d, 1/Y_d
    alg_bytes = (len(ps) * per_particle + st.candidates * (4 + 8) +
                 res * res * 3 * 8 / max(world, 1))
    achieved = alg_bytes / (render_ms * 1e-3) / 1e9
    traffic = measured_traffic(args.config, res, world)
    roof = {"bound": "hbm", "kernel": "k_render_rays", "achieved": achieved,
            "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
            "frac": achieved / peaks.get("hbm_gbs", 6650.0),
            "traffic": traffic["dram_bytes"] if traffic else None,
            "traffic_source": traffic["source"] if traffic else None,
            "algorithmic_bytes": alg_bytes,
            "peak_source": peak_src,
            "note": "the render kernel is ALU/FP64 issue-bound, not HBM-bound (SURVEY.md 8(d)); "
                    "achieved = compulsory bytes (particle records + candidate list + image) "
                    "/ median render-kernel time"}
    # second roofline: the merge against the measured int64
    # multiply/add issue peak of this GPU; algorithmic ops = the reference's
    # RayAccumulator op count (RenderStats.int_ops, raycast.hpp:217-244)
    alu = None
    try:
        pk = S.probe_alu_peaks(local)
        ach = st.int_ops / (render_ms * 1e-3) / 1e9
        alu = {"bound": "alu", "kernel": "k_render_rays (merge)", "unit": "Gop/s",
               "achieved": ach, "peak": pk["int64_gops"], "frac": ach / pk["int64_gops"],
               "fp64_peak_gflops": pk["fp64_gflops"],
               "note": "achieved = RenderStats.int_ops (int64 mul/add of the reference's "
                       "sequential merge) / median render-kernel time; peak = measured int64 "
                       "mul+add issue rate (sphray_probe_alu_peaks)"}
    except Exception as e:  # report, never fake
        alu = {"bound": "alu", "unavailable": str(e)}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                lut_path = lut_file(args)
                cpu = cpu_reference_sample(ps, lut_path, ds, qc, res, budget_s=args.cpu_budget)
                cpu.pop("seconds", None)
            except Exception as e:  # report, never fake
                cpu = {"value": None, "unit": "Mrays/s", "cores": os.cpu_count(),
                       "kind": "reference", "sample": f"failed: {e}"}
        out = {
            "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config {cfg}: {CONFIGS[cfg]['desc']}",
                       "particles": len(ps), "image": f"{res}x{res}", "K": args.K, "D": args.D,
                       "N_lut": 1024, "int_width": 64, "mode": args.mode,
                       "parallelism": f"image tiles 8x8 interleaved over {world} GPU(s), "
                                      "particles replicated, NCCL tile gather",
                       "l2": "256 MB buffer written between frames (> 126 MB L2)"},
            "roofline": roof,
            "alu_roofline": alu,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(st.launches) * args.steps,
            "clocks": clocks,
            "breakdown_ms": {"bin": bin_ms, "render_kernel": render_ms,
                             "frame_device": statistics.median(s.device_ms for s in per_step),
                             "per_step_device": [round(s.device_ms, 3) for s in per_step],
                             "per_step_wall": [round(x, 3) for x in walls]},
            "stats": {"hits": st.hits, "knots": st.knots, "rays_touched": st.rays_touched,
                      "candidates": st.candidates, "max_window": st.max_window,
                      "window_retries": st.window_retries, "int_ops": st.int_ops,
                      "residual_failures": st.residual_failures,
                      "skipped_particles": st.skipped_particles},
            "setup_s": setup_s,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=0, help="override particle count")
    ap.add_argument("--res", type=int, default=0, help="override image resolution (profiling)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"])
    ap.add_argument("--window", type=int, default=0, help="knot window slots per ray (0 = auto)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-step-budget", type=float, default=5.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--K", type=int, default=4, choices=[1, 2, 3, 4], help="LUT pieces (order sweep)")
    ap.add_argument("--D", type=int, default=3, choices=[1, 2, 3], help="LUT degree (order sweep)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
