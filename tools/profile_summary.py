"""Summarise the ncu evidence of one bench configuration into profiles/.

usage: python tools/profile_summary.py <tag> <config> <launches.csv> <full.ncu-rep> <call_bytes.json> <skip>

* launches.csv  -- `ncu --metrics gpu__time_duration.sum --csv` launch list of a
                   bench run (libtts kernels only): per-kernel share of GPU time.
* full.ncu-rep  -- `ncu --set full -k regex:k_tree_umma -s <skip> -c 1` capture.
* call_bytes    -- `bench.py --dump-call-bytes` of the same run: algorithmic
                   bytes of every attention launch, so the captured launch's DRAM
                   traffic can be compared with its own algorithmic bytes.
Writes profiles/<tag>_<config>.md and profiles/ncu_traffic_<config>.json.
"""
import collections
import csv
import json
import os
import subprocess
import sys

tag, cfg, launches, rep, cbytes, skip = sys.argv[1:7]
skip = int(skip)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_md = os.path.join(ROOT, "profiles", f"{tag}_{cfg}.md")

# --- launch list
agg = collections.defaultdict(lambda: [0, 0.0])
rows = list(csv.reader(open(launches)))
hdr = None
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("tts::<unnamed>::", "").replace("void ", "")
    unit = d.get("Metric Unit", "ns")
    v = float(d["Metric Value"].replace(",", ""))
    v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())

# --- full capture
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, u, v = rr[0], rr[1], rr[2]
m = {h[i]: (v[i], u[i]) for i in range(len(h))}


def val(name, scale_to=None):
    x, unit = m[name]
    x = float(x.replace(",", ""))
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
         "ns": 1e-3, "us": 1, "ms": 1e3}.get(unit, 1)
    return x * f


dram_r = val("dram__bytes_read.sum")
dram_w = val("dram__bytes_write.sum")
dur_us = val("gpu__time_duration.sum")
cb = json.load(open(cbytes))
skip = skip % len(cb["unique_kv_bytes"])  # the captured launch's index within one bench step
algo_kv = cb["unique_kv_bytes"][skip]
algo = algo_kv + cb["active_beams"][skip] * cb["qo_bytes_per_beam"]
keys = ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
        "SM_A.TriageCompute.sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__inst_executed_pipe_alu_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]

lines = [f"# ncu evidence: {cfg} ({tag})", "",
         "## Launch list (`ncu --metrics gpu__time_duration.sum`, libtts kernels, cold-cache serialised)", "",
         "| kernel | launches | total us | share |", "|---|---|---|---|"]
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| {k} | {n} | {t:.1f} | {t / tot:.3f} |")
lines += ["", f"## Full capture of attention launch #{skip} (`ncu --set full`)", "",
          f"* duration: {dur_us:.1f} us (under ncu: cold L2, serialised)",
          f"* DRAM read {dram_r / 1e6:.1f} MB, write {dram_w / 1e6:.1f} MB -> traffic {(dram_r + dram_w) / 1e6:.1f} MB",
          f"* algorithmic bytes of this launch: {algo / 1e6:.1f} MB (unique KV {algo_kv / 1e6:.1f} MB + q/out)",
          f"* traffic / algorithmic = {(dram_r + dram_w) / algo:.3f}",
          f"* DRAM bandwidth during the launch: {(dram_r + dram_w) / dur_us / 1e3:.0f} GB/s"]
for k in keys:
    if k in m:
        lines.append(f"* {k} = {m[k][0]} {m[k][1]}")
open(out_md, "w").write("\n".join(lines) + "\n")
json.dump({"config": cfg, "tag": tag, "launch_index": skip, "dram_bytes_per_launch": dram_r + dram_w,
           "algo_bytes_of_that_launch": algo, "duration_us_under_ncu": dur_us,
           "kernel_shares": {k: t / tot for k, (n, t) in agg.items()}},
          open(os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg}.json"), "w"), indent=1)
print("\n".join(lines))
