"""Markdown summary of ncu evidence for profiles/.

  python scripts/profile_report.py --rep gpurun_out/prof_render_c3.ncu-rep \
      --launches gpurun_out/launches.csv --cubin <render_d3 cubin> --out profiles/r01_render_c3.md

Sections: key metrics of the captured kernel, stall reasons (pc sampling),
phase breakdown of executed instructions (scripts/phase_profile.py logic), and
the per-kernel launch list (share of device time) from the
`--metrics gpu__time_duration.sum` pass.
"""
import argparse
import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)


_SCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "s": 1e3, "ms": 1.0, "us": 1e-3, "ns": 1e-6,  # -> ms
          "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}                 # -> bytes


def raw_metrics(rep):
    """name -> value, with durations in ms and byte counts in bytes."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    out = {}
    for name, unit, val in zip(rows[0], rows[1], rows[2]):
        try:
            out[name] = str(float(val.replace(",", "")) * _SCALE.get(unit, 1.0))
        except ValueError:
            out[name] = val
    return out


def fnum(d, k):
    try:
        return float(d[k])
    except (KeyError, ValueError):
        return None


def launches_table(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[r[ki].split("(")[0].strip()].append(float(r[vi]))
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k[-70:]}` | {len(v)} | {sum(v) / 1e6:.3f} | {sum(v) / tot * 100:.2f}% |")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--cubin")
    ap.add_argument("--kernel", default="k_render_raysILi3ELi2ELb1ELi0ELb1ELb0ELb0E")
    ap.add_argument("--src", default=os.path.join(HERE, "..", "paper_2401_02896_b200", "csrc",
                                                 "render_kernel.cuh"))
    ap.add_argument("--title", default="render kernel profile")
    ap.add_argument("--out", required=True)
    ap.add_argument("--evidence", help="also write the bench's profile evidence JSON here")
    ap.add_argument("--knots", type=float, default=0.0, help="knots of the captured launch")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--res", type=int, default=2048)
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    md = [f"# {a.title}", ""]
    if a.rep:
        d = raw_metrics(a.rep)
        keys = [
            ("duration (ms)", "gpu__time_duration.sum", 1),
            ("SM cycles", "sm__cycles_elapsed.avg", 1),
            ("warp instructions executed", "smsp__inst_executed.sum", 1),
            ("IPC per SM (of 4)", "sm__inst_executed.avg.per_cycle_active", 1),
            ("issue slots busy %", "sm__instruction_throughput.avg.pct_of_peak_sustained_active", 1),
            ("warps active per SM", "sm__warps_active.avg.per_cycle_active", 1),
            ("achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
            ("FP64 pipe %", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
            ("ALU pipe %", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
            ("FMA pipe %", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
            ("LSU pipe %", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
            ("DRAM read bytes", "dram__bytes_read.sum", 1),
            ("DRAM write bytes", "dram__bytes_write.sum", 1),
            ("L2 hit %", "lts__t_sector_hit_rate.pct", 1),
            ("registers / thread", "launch__registers_per_thread", 1),
            ("thread instructions executed", "smsp__thread_inst_executed.sum", 1),
        ]
        md += ["## Key metrics", "", "| metric | value |", "|---|---|"]
        for name, k, sc in keys:
            v = fnum(d, k)
            md.append(f"| {name} | {v * sc:.6g} |" if v is not None else f"| {name} | n/a |")
        st = [(fnum(d, k), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in d
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
        st = [(v, k) for v, k in st if v]
        if not st:  # no PC sampling in the capture: the WarpStateStats averages
            pre, suf = "smsp__average_warp_latency_issue_stalled_", ".ratio"
            st = [(fnum(d, k), k[len(pre):-len(suf)]) for k in d if k.startswith(pre) and k.endswith(suf)]
            st = [(v, k) for v, k in st if v and not k.endswith("not_issued")]
        tot = sum(v for v, _ in st)
        md += ["", "## Stall reasons (PC sampling)", "", "| reason | share |", "|---|---|"]
        for v, k in sorted(st, reverse=True)[:10]:
            md.append(f"| {k} | {v / tot * 100:.1f}% |")
        wi, ti = fnum(d, "smsp__inst_executed.sum"), fnum(d, "smsp__thread_inst_executed.sum")
        if wi and ti:
            md += ["", f"Average active threads per executed warp instruction: {ti / wi:.1f} of 32."]
        if a.knots and wi:
            md += [f"Warp instructions per knot: {wi / a.knots:.1f} ({a.knots:.4g} knots in the launch)."]
        if a.evidence:
            import json
            ev = {"config": a.config, "res": a.res, "world": 1, "source": a.source or a.rep,
                  "dram_bytes": (fnum(d, "dram__bytes_read.sum") or 0) + (fnum(d, "dram__bytes_write.sum") or 0),
                  "duration_ms": fnum(d, "gpu__time_duration.sum"),
                  "issue_slots_busy_pct": fnum(d, "sm__instruction_throughput.avg.pct_of_peak_sustained_active"),
                  "ipc": fnum(d, "sm__inst_executed.avg.per_cycle_active"),
                  "warps_active_per_sm": fnum(d, "sm__warps_active.avg.per_cycle_active"),
                  "achieved_occupancy_pct": fnum(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                  "fp64_pipe_pct": fnum(d, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                  "alu_pipe_pct": fnum(d, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                  "fma_pipe_pct": fnum(d, "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                  "lsu_pipe_pct": fnum(d, "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
                  "active_threads_per_warp_inst": (ti / wi) if wi and ti else None,
                  "warp_instructions_per_knot": (wi / a.knots) if a.knots and wi else None,
                  "stalls_pct": {k: round(v / tot * 100, 2) for v, k in sorted(st, reverse=True)[:8]}}
            json.dump(ev, open(a.evidence, "w"), indent=1)
        if a.cubin:
            cubin = a.cubin
            if cubin.endswith(".o"):  # host object: pull the sm_100a cubin out of its fatbin
                import glob
                import tempfile
                td = tempfile.mkdtemp()
                subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(cubin)], cwd=td,
                               capture_output=True)
                cubin = sorted(glob.glob(os.path.join(td, "*.cubin")))[0]
            sass = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv",
                                   "--print-source", "sass"], capture_output=True, text=True).stdout
            tmp = a.out + ".sass.csv"
            open(tmp, "w").write(sass)
            ph = subprocess.run([sys.executable, os.path.join(HERE, "phase_profile.py"), cubin,
                                 a.kernel, tmp, a.src], capture_output=True, text=True).stdout
            os.remove(tmp)
            md += ["", "## Executed instructions by phase", "", "```", ph.strip(), "```"]
    if a.launches:
        md += ["", "## Launch list (ncu --metrics gpu__time_duration.sum, serialised, cold cache)",
               "", launches_table(a.launches)]
    open(a.out, "w").write("\n".join(md) + "\n")
    print(open(a.out).read())


if __name__ == "__main__":
    main()
