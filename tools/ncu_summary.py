#!/usr/bin/env python
"""Summarise a round's ncu outputs (gpurun_out/prof_<round>/) into profiles/<round>/.

  launches.csv   -> per-kernel device time per bench step and share of the step
  full_*.ncu-rep -> per-kernel DRAM bytes, duration, pipe utilisation, issue
"""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
SRC = os.path.join("gpurun_out", f"prof_{R}")
DST = os.path.join("profiles", R)
os.makedirs(DST, exist_ok=True)

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
         "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def launches():
    rows = list(csv.reader(open(os.path.join(SRC, "launches.csv"))))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    rs = rows[hdr + 1:]
    starts = [i for i, r in enumerate(rs) if "setup_envs" in r[ki]]
    last = rs[starts[-1]:]           # the last gg_render of the run = one timed step
    agg = OrderedDict()
    for r in last:
        name = r[ki].split("(")[0].replace("void ", "").strip()
        if not name.startswith("gg::") or "checksum" in name:   # the digest runs after the timed region
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9)
        a = agg.setdefault(name, {"launches": 0, "seconds": 0.0})
        a["launches"] += 1
        a["seconds"] += v
    tot = sum(a["seconds"] for a in agg.values())
    for a in agg.values():
        a["share"] = a["seconds"] / tot
    return agg, tot, len(rs)


def _raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def full(kernel):
    path = os.path.join(SRC, f"full_{kernel}.ncu-rep")
    if os.path.exists(path):
        rows = _raw(path)
        h, u, v = rows[0], rows[1], rows[2]
    else:   # one multi-kernel capture (tools/profile_round.sh <round> full): first launch of that kernel
        allp = os.path.join(SRC, "full_all.ncu-rep")
        if not os.path.exists(allp):
            return None
        rows = _raw(allp)
        h, u = rows[0], rows[1]
        ki = h.index("Kernel Name")
        hit = [r for r in rows[2:] if kernel in r[ki]]
        if not hit:
            return None
        v = hit[-1]   # the last capture: the bench's own render configuration (not a counters pass)
    res = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else kernel}
    for m in METRICS:
        if m in h:
            i = h.index(m)
            try:
                x = float(v[i].replace(",", ""))
            except ValueError:
                continue
            unit = u[i]
            if unit in SCALE and ("bytes" in m or "duration" in m):
                x *= SCALE[unit]
                unit = "B" if "bytes" in m else "s"
            res[m] = x
    if "dram__bytes_read.sum" in res:
        res["dram_bytes_total"] = res["dram__bytes_read.sum"] + res.get("dram__bytes_write.sum", 0.0)
    return res


agg, tot, nl = launches()
kern = {}
for k in ["raster_warp_kernel", "project_kernel", "cull_count_kernel", "depth_downsweep", "place_downsweep",
          "depth_upsweep", "place_upsweep", "depth_ties", "depth_scan", "place_scan"]:
    r = full(k)
    if r:
        kern[k] = r
summary = {"round": R, "step_kernel_seconds": tot, "per_kernel_step": agg, "full_captures": kern,
           "capture_envs_per_launch": 512,
           "notes": "launch list: ncu --metrics gpu__time_duration.sum --clock-control none of "
                    "`bench.py --steps 2 --warmup 3 --no-e2e --no-cpu` (cold-cache, serialised: compare shares); "
                    "full captures: ncu --set full (caches flushed per kernel) on the last captured launch of each kernel "
                    "of `bench.py --envs 512` (one launch = 512 envs; the default bench launch covers 1024)."}
json.dump(summary, open(os.path.join(DST, "ncu_summary.json"), "w"), indent=1)
with open(os.path.join(DST, "ncu_summary.md"), "w") as f:
    f.write(f"# ncu summary — {R}\n\nLaunch list (last gg_render of the bench run = one step, {nl} launches "
            f"listed in total): {tot*1e3:.1f} ms of kernel time per step.\n\n")
    f.write("| kernel | launches/step | ms/step | share |\n|---|---|---|---|\n")
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["seconds"]):
        f.write(f"| {k} | {a['launches']} | {a['seconds']*1e3:.2f} | {a['share']*100:.1f}% |\n")
    f.write("\nFull captures (one launch = one 512-env chunk; from the `full` pass, which can predate the launch list — "
            "see the round's commit log):\n\n| kernel | ms | DRAM read GB | DRAM write GB | "
            "issue % | FMA pipe % | ALU pipe % | XU (MUFU) inst % | L1 % | L2 % | warps active % | regs |\n"
            "|---|---|---|---|---|---|---|---|---|---|---|---|\n")
    for k, r in kern.items():
        f.write(f"| {k} | {r.get('gpu__time_duration.sum', 0)*1e3:.2f} | {r.get('dram__bytes_read.sum', 0)/1e9:.2f} | "
                f"{r.get('dram__bytes_write.sum', 0)/1e9:.2f} | {r.get('sm__issue_active.avg.pct_of_peak_sustained_elapsed', 0):.0f} | "
                f"{r.get('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 0):.0f} | "
                f"{r.get('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 0):.0f} | "
                f"{r.get('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', r.get('sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active', 0)):.0f} | "
                f"{r.get('l1tex__throughput.avg.pct_of_peak_sustained_active', 0):.0f} | "
                f"{r.get('lts__throughput.avg.pct_of_peak_sustained_elapsed', 0):.0f} | "
                f"{r.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.0f} | "
                f"{r.get('launch__registers_per_thread', 0):.0f} |\n")
import shutil
shutil.copy(os.path.join(SRC, "launches.csv"), os.path.join(DST, "launches.csv"))
print(open(os.path.join(DST, "ncu_summary.md")).read())
