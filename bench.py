#!/usr/bin/env python3
"""bench.py -- Mrays/s of the B200 per-ray higher-order SPH DVR path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One step = one full frame of BASELINE.json config C (default 3: the 16M
clustered cosmology-like particle set, 2048^2 image, K=4, D=3, N=1024, w64 --
the workload the north-star metric is quoted on at 1/2/4/8 B200), rendered by
the sm_100a path with the particle set resident in HBM (MODE_FAST: rays stop
at early termination, the image is identical).  With --gpus N > 1 the script
re-launches itself under torch.distributed.run when WORLD_SIZE is unset; image
tiles are interleaved over ranks and gathered with NCCL inside the library
(strong scaling: the frame is fixed).  Timing: CUDA events on the library's
stream, bracketed by barrier + synchronize, max over ranks.  Rank 0 prints ONE
JSON line.

The line also carries
  e2e          the one-shot drop-in call sphray_render_scene with host buffers
               (particle H2D, host pow precompute, image D2H inside the timing);
  exact        one MODE_EXACT frame (every RenderStats counter complete -- the
               mode the C++ shim gives reference callers) and the fraction of
               early-terminated rays;
  parity       the timed frame checked against the UNMODIFIED reference
               (oracle/_ref) on 8 pixel regions spread over the frame: RGB of
               the FAST frame and of an EXACT render, RenderStats and per-ray
               records (knots, pieces, hits, piece checksums) -- the run exits
               nonzero if RGB differs by more than 1e-4 or a count differs;
  roofline     SURVEY.md 8(d) compulsory bytes / render-kernel time vs the
               measured HBM peak, the DRAM traffic of the render launch (ncu),
               and the ALU view (the reference's merge op count vs the measured
               int64 issue peak);
  cpu_baseline the reference's render_scene<int64_t> sweeps on the same
               regions, every host thread (rank 0, N = 1).

--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified reference headers; particles from the shared generator
include/sphray_scenes.hpp compiled into oracle/_ref, dataset statistics and
quanta from the reference) on evenly spaced full-width rows of the same frame,
one row per step, rank 0 only -- the product library is never loaded.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
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
RGB_TOL = 1e-4


def camera_kwargs(res):
    """SURVEY.md 8(d) orthographic camera."""
    return dict(mode="orthographic", position=(0.0, 0.0, 8.0), look_at=(0.0, 0.0, 0.0),
                up=(0.0, 1.0, 0.0), width=res, height=res, ortho_height=6.0, near=0.0, far=1e30)


def sample_regions(res, width):
    """8 evenly spaced one-row regions (x0, y0, w, 1): row y_k = (k + 1/2) res / 8,
    `width` pixels wide, the column window stepping across the frame with k
    (every part of the image, dense centre and sparse edges, is sampled)."""
    out = []
    for k in range(8):
        y = int(res * (k + 0.5) / 8)
        w = min(width, res)
        x = int((res - w) * ((k * 3) % 8) / 7)
        out.append((x, y, w, 1))
    return out


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_distributed(args):
    """--gpus N > 1 without a launcher: run N ranks under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    return subprocess.call(cmd)


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


def profile_evidence(config, res, world):
    """ncu evidence of the render launch at this workload (profiles/, committed):
    DRAM bytes of one main render launch and the --set full summary."""
    path = os.path.join(ROOT, "profiles", "render_evidence.json")
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
            return json.load(f), "MEASURED_PEAKS.json"
    except (OSError, ValueError):
        return {"hbm_gbs": 7700.0}, "fallback (B200_PROFILING.md nominal)"


def lut_file(args):
    """The LUT of the run: cubic B-spline, K pieces, degree D, 1024 entries
    (config 4's order sweep varies K and D; every other config is K=4, D=3)."""
    return os.path.join(ROOT, "data", "luts", f"cubic_K{args.K}_D{args.D}_N1024.splt")


# --------------------------------------------------------------------------- reference
def reference_setup(cfg, n, lut_path):
    """Particles, LUT, dataset statistics and quanta entirely through oracle/_ref."""
    from oracle import ref

    ps = ref.generate_scene(cfg, n)
    rl = ref.Lut(lut_path)
    rds = ref.dataset_stats(ps, rl)
    rqc = ref.choose_quanta(rl, rds)
    return ps, rl, rds, rqc


def reference_regions(ps, rl, rds, rqc, res, regions, threads):
    """The reference's sweeps on each region of the full-frame camera."""
    from oracle import ref

    cam = ref.Camera(**camera_kwargs(res))
    out = []
    for reg in regions:
        rgb, rec, st, sec, bits = ref.render_region(ps, cam, SYNTH_TF, rl, rqc, rds.h_r / 8.0, *reg,
                                                    threads=threads)
        out.append(dict(region=reg, rgb=rgb, rec=rec, stats=st, seconds=sec, bits=bits))
    return out


def cpu_summary(samples, threads, res, frame_touched=None):
    rays = sum(s["region"][2] * s["region"][3] for s in samples)
    touched = sum(int(s["stats"]["rays_touched"]) for s in samples)
    secs = sum(s["seconds"] for s in samples)
    bits = sorted({s["bits"] for s in samples})
    out = dict(value=rays / secs / 1e6 if secs > 0 else None, unit="Mrays/s", cores=threads,
               kind="reference",
               sample=(f"{len(samples)} region(s) {[s['region'] for s in samples]} (x0, y0, w, h) "
                       f"of the {res}^2 frame on the frame's own camera through the reference's "
                       f"footprint/quantize/sort_knots/accumulate/composite with "
                       f"render_scene<int{'/'.join(str(b) for b in bits)}> accumulators; "
                       f"{rays} rays ({touched} touched) in {secs:.2f} s"),
               seconds=secs, rays=rays, touched=touched)
    if frame_touched and touched:
        # full frame estimated from the sample's time per touched ray
        est = secs / touched * frame_touched
        out["frame_s_extrapolated"] = est
        out["value_extrapolated"] = res * res / est / 1e6
    return out


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    from oracle import ref

    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs "
                          "/root/reference at build time)"}))
        return 0
    cfg = args.config
    res = args.res or CONFIGS[cfg]["res"]
    threads = os.cpu_count() or 1
    ps, rl, rds, rqc = reference_setup(cfg, args.n, lut_file(args))
    rows = [(0, y, res, 1) for (_, y, _, _) in sample_regions(res, res)]
    for i in range(args.warmup):  # warm-up: a short piece of a row
        reference_regions(ps, rl, rds, rqc, res, [(res // 2 - 32, rows[i % 8][1], 64, 1)], threads)
    samples = []
    for i in range(args.steps):
        samples += reference_regions(ps, rl, rds, rqc, res, [rows[i % 8]], threads)
    cs = cpu_summary(samples, threads, res)
    value = cs["value"]
    out = {"metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * cs["seconds"] / len(samples),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": f"config {cfg}: {CONFIGS[cfg]['desc']}", "particles": len(ps),
                      "image": f"{res}x{res}", "K": args.K, "D": args.D, "N_lut": 1024,
                      "int_width": 64},
           "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": threads,
                            "kind": "reference",
                            "sample": "one full-width row per step, rows cycling over 8 evenly "
                                      "spaced rows; " + cs["sample"]},
           "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2401_02896_b200 as S
    from paper_2401_02896_b200 import dist as SD

    rank, world, local = env_rank()
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    res = args.res or CONFIGS[cfg]["res"]
    t0 = time.time()
    ps = S.generate_scene(cfg, n=args.n)
    lut = S.load_lut(lut_file(args))
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    setup_s = time.time() - t0
    ctx = S.Context(local)
    SD.init_comm(ctx, rank, world)
    if world > 1:
        print(f"[bench] rank {rank}/{world}: NCCL communicator initialised on cuda:{local} "
              f"(tile gather inside the library)", file=sys.stderr, flush=True)
    cam = S.Camera(**camera_kwargs(res))
    tf = S.TransferFunction.from_array(SYNTH_TF)
    mode = S.MODE_FAST if args.mode == "fast" else S.MODE_EXACT
    opts = S.RenderOptions(mode=mode, window=args.window)
    ctx.upload(ps, lut)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr())
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def dev_max(ms):
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

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
    ms_max = dev_max(e0.elapsed_time(e1))
    value = res * res * args.steps / (ms_max * 1e-3) / 1e6
    render_ms = statistics.median(s.render_ms for s in per_step)
    bin_ms = statistics.median(s.bin_ms for s in per_step)
    st = per_step[-1]
    frame = None
    if rank == 0:
        # the timed frame (the full image on rank 0 after the tile gather)
        class _Dev:  # the library's device image, viewed through __cuda_array_interface__
            __cuda_array_interface__ = {"shape": (res, res, 3), "typestr": "<f8",
                                        "data": (ctx.device_image_ptr(), False), "version": 3}
        torch.cuda.synchronize()
        frame = torch.as_tensor(_Dev(), device="cuda").cpu().numpy()
    image_sha = hashlib.sha256(frame.tobytes()).hexdigest() if frame is not None else None

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
        wall = time.perf_counter() - t0
        e2e_ms = dev_max(f0.elapsed_time(f1))
        h2d = len(ps) * 56 + lut.records().nbytes + SYNTH_TF.nbytes
        d2h = res * res * 3 * 8
        e2e = {"value": res * res * args.e2e_steps / (e2e_ms * 1e-3) / 1e6, "unit": "Mrays/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_ms / args.e2e_steps, "wall_s": wall,
               "api": "sphray_render_scene (one-shot drop-in for render_scene<int64_t>): particle "
                      "H2D, host pow(h, d+3), Morton sort, binning, render, image D2H"}
        if rank == 0 and not np.array_equal(img.pixels, frame):
            raise SystemExit("bench: the one-shot render differs from the timed frame")

    # ---- one EXACT frame: complete RenderStats, and the early-termination share
    exact = None
    if args.exact_steps > 0:
        ex_opts = S.RenderOptions(mode=S.MODE_EXACT, window=args.window)
        barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.exact_steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            _, xst = ctx.render(cam, tf, qc, ds, ex_opts, to_host=False)
        g1.record(stream)
        barrier()
        x_ms = dev_max(g0.elapsed_time(g1)) / args.exact_steps
        exact = {"value": res * res / (x_ms * 1e-3) / 1e6, "unit": "Mrays/s", "ms_per_step": x_ms,
                 "knots": xst.knots, "rays_touched": xst.rays_touched, "int_ops": xst.int_ops,
                 "residual_failures": xst.residual_failures, "hits": xst.hits,
                 "terminated_rays": xst.terminated_rays,
                 "terminated_fraction": xst.terminated_rays / max(1, xst.rays_touched),
                 "fast_frame": {"knots": st.knots, "int_ops": st.int_ops,
                                "knots_share_of_exact": st.knots / max(1, xst.knots)}}

    # ---- roofline of the dominant kernel (the render kernel)
    peaks, peak_src = measured_peaks()
    D = lut.D
    comp_particle = 32 + 16 * D          # x,y,z,h + X_d, Y_d (f64)
    comp_pixel = 3 * 8                   # the f64 RGB the path writes
    alg_bytes = len(ps) * comp_particle + res * res * comp_pixel / world + lut.records().nbytes
    achieved = alg_bytes / (render_ms * 1e-3) / 1e9
    ev = profile_evidence(cfg, res, world)
    roof = {"bound": "hbm", "kernel": "k_render_rays", "achieved": achieved,
            "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
            "frac": achieved / peaks.get("hbm_gbs", 7700.0),
            "traffic": ev["dram_bytes"] if ev else None,
            "traffic_over_algorithmic": (ev["dram_bytes"] / alg_bytes) if ev else None,
            "algorithmic_bytes": alg_bytes,
            "algorithmic_bytes_formula": f"n*(32+16D) + W*H*24/world + LUT = {len(ps)}*{comp_particle} "
                                         f"+ {res}^2*{comp_pixel}/{world} + {lut.records().nbytes}",
            "peak_source": peak_src,
            "note": "SURVEY.md 8(d): the path is instruction-issue bound once knots are never "
                    "materialised; the HBM fraction is tiny by construction.  traffic = ncu "
                    "dram__bytes of one render launch at this workload (profiles/)"}
    # the bytes the chosen tiling streams, sum over tiles of
    # |candidates(tile)| x (32 + 16 D), as the gather's HBM fraction
    tb = st.candidates * comp_particle
    roof["tiling"] = {"tile": "8x8 pixels", "candidates": st.candidates, "bytes": tb,
                      "achieved": tb / (render_ms * 1e-3) / 1e9,
                      "frac": tb / (render_ms * 1e-3) / 1e9 / peaks.get("hbm_gbs", 7700.0),
                      "formula": f"sum over tiles |candidates(tile)| * (32+16D) = "
                                 f"{st.candidates} * {comp_particle}"}
    if ev:
        for k in ("issue_slots_busy_pct", "ipc", "warps_active_per_sm", "achieved_occupancy_pct",
                  "fp64_pipe_pct", "alu_pipe_pct", "fma_pipe_pct", "lsu_pipe_pct",
                  "warp_instructions_per_knot", "source"):
            if k in ev:
                roof[k] = ev[k]
    alu = None
    try:
        pk = S.probe_alu_peaks(local)
        x_ops = exact["int_ops"] if exact else st.int_ops
        x_ms = exact["ms_per_step"] if exact else render_ms
        ach = x_ops / (x_ms * 1e-3) / 1e9
        alu = {"bound": "alu", "kernel": "k_render_rays (merge)", "unit": "Gop/s",
               "achieved": ach, "peak": pk["int64_gops"], "frac": ach / pk["int64_gops"],
               "fp64_peak_gflops": pk["fp64_gflops"],
               "note": "achieved = RenderStats.int_ops of the EXACT frame (the reference's "
                       "RayAccumulator int64 op count, raycast.hpp:217-244) / that frame's device "
                       "time; peak = measured int64 mul+add issue rate (sphray_probe_alu_peaks)"}
    except Exception as e:  # report, never fake
        alu = {"bound": "alu", "unavailable": str(e)}

    # ---- parity + CPU baseline: 8 regions spread over the frame, reference on the host
    parity, cpu = None, None
    if rank == 0 and world == 1 and not args.no_parity:
        from oracle import ref

        # config 1 is the one configuration the reference renders whole
        # (SURVEY.md 8(d)): its CPU baseline and parity cover the full frame
        full = args.cpu_full_frame or cfg == 1
        regions = [(0, 0, res, res)] if full else sample_regions(res, args.region_width)
        threads = os.cpu_count() or 1
        rl = ref.Lut(lut_file(args))
        rds = ref.dataset_stats(ps, rl)
        rqc = ref.choose_quanta(rl, rds)
        same_inputs = (rqc.tau, rqc.sigma, rds.h_r) == (qc.tau, qc.sigma, ds.h_r)
        samples = reference_regions(ps, rl, rds, rqc, res, regions, threads)
        cpu = cpu_summary(samples, threads, res,
                          frame_touched=exact["rays_touched"] if exact else st.rays_touched)
        err_fast, err_exact, mism = 0.0, 0.0, {}
        stats_exact = True
        for smp in samples:
            x0, y0, w, h = smp["region"]
            err_fast = max(err_fast, float(np.abs(frame[y0:y0 + h, x0:x0 + w] -
                                                  smp["rgb"][:, x0:x0 + w]).max()))
            ctx.set_region(x0, y0, w, h, record=True)
            img, rst = ctx.render(cam, tf, qc, ds, S.RenderOptions(mode=S.MODE_EXACT))
            rec = ctx.ray_records()
            ctx.set_region()
            err_exact = max(err_exact, float(np.abs(img.pixels[:, x0:x0 + w] -
                                                    smp["rgb"][:, x0:x0 + w]).max()))
            rr = smp["rec"]
            for k in ("knots", "pieces", "hits", "piece_checksum"):
                mism[k] = mism.get(k, 0) + int((rec[k] != rr[k]).sum())
            mism["residual_flag"] = mism.get("residual_flag", 0) + int(((rec["flags"] ^ rr["flags"]) & 3).sum() > 0)
            for k in ("knots", "rays_touched", "int_ops", "residual_failures"):
                stats_exact &= getattr(rst, k) == int(smp["stats"][k])
        ok = same_inputs and err_fast <= RGB_TOL and err_exact <= RGB_TOL and stats_exact and \
            not any(mism.values())
        parity = {"ok": bool(ok), "regions": regions, "rays": cpu["rays"],
                  "max_abs_rgb_fast_frame": err_fast, "max_abs_rgb_exact": err_exact,
                  "tolerance": RGB_TOL, "stats_exact": bool(stats_exact),
                  "per_ray_mismatches": mism, "same_quanta_as_reference": bool(same_inputs),
                  "reference": "oracle/_ref (unmodified reference headers): footprint, "
                               "quantize_particle, sort_knots, accumulate, composite on the frame's "
                               f"camera; accumulator bits {sorted({s['bits'] for s in samples})}",
                  "checked": "RGB of the timed FAST frame and of an EXACT render; per ray: hits, "
                             "knots, FieldPieces (count + sphray_piece_mix checksum, production "
                             "kernel), residual flag; RenderStats of each region"}
        cpu.pop("seconds", None)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64 (fp64 geometry/quantize/compositing, exact int64 knots and merge)",
            "data": "synthetic",
            "config": {"workload": f"config {cfg}: {CONFIGS[cfg]['desc']}",
                       "particles": len(ps), "image": f"{res}x{res}", "K": args.K, "D": args.D,
                       "N_lut": 1024, "int_width": 64, "mode": args.mode,
                       "parallelism": f"image tiles 8x8 interleaved over {world} GPU(s), "
                                      "particles replicated, NCCL tile gather",
                       "l2": "256 MB buffer written between frames (> 126 MB L2)"},
            "image_sha256": image_sha,
            "parity": parity,
            "roofline": roof,
            "alu_roofline": alu,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "exact": exact,
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
                      "skipped_particles": st.skipped_particles,
                      "terminated_rays": st.terminated_rays},
            # SURVEY.md 8(d)'s secondary rates of the timed (device-resident) frame
            "rates": {"touched_rays_per_s": st.rays_touched / (render_ms * 1e-3),
                      "hits_per_s": st.hits / (render_ms * 1e-3),
                      "knots_per_s": st.knots / (render_ms * 1e-3),
                      "int_ops_per_s": st.int_ops / (render_ms * 1e-3)},
            "setup_s": setup_s,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if rank == 0 and parity is not None and not parity["ok"]:
        print("bench: PARITY FAILED against the reference", file=sys.stderr)
        return 1
    return 0


def run_dry(args):
    """--dry-run: the multi-rank plumbing of run_ours without a GPU (gloo): rank /
    world checks, the NCCL unique-id broadcast path (dist.init_comm's object
    broadcast), barrier + max-over-ranks timing reduction, one JSON line."""
    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("gloo")
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))
        dist.barrier()
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_ms_max": float(t.item()),
                          "local_rank": local}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


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
    ap.add_argument("--exact-steps", type=int, default=1)
    ap.add_argument("--region-width", type=int, default=256,
                    help="pixels per parity / CPU-baseline region (8 regions)")
    ap.add_argument("--no-parity", action="store_true", help="skip parity + CPU baseline")
    ap.add_argument("--cpu-full-frame", action="store_true",
                    help="parity + CPU baseline on the whole frame (default for config 1)")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing only (CPU, gloo)")
    ap.add_argument("--K", type=int, default=4, choices=[1, 2, 3, 4], help="LUT pieces (order sweep)")
    ap.add_argument("--D", type=int, default=3, choices=[1, 2, 3], help="LUT degree (order sweep)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    if args.dry_run:
        return run_dry(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
