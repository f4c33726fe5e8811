#!/bin/bash
# per-kernel launch list (ncu, one metric) for a config: tools/launches.sh <cfg> <rotate> <tag>
cfg=$1; rot=$2; tag=$3
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --launch-skip 3000 -c 2000 --csv \
    --log-file gpurun_out/${tag}_${cfg}_launches.csv python bench.py --config $cfg --rotate $rot --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python - gpurun_out/${tag}_${cfg}_launches.csv <<'PY' > gpurun_out/${tag}_${cfg}_launches.txt
import csv, sys, collections
agg = collections.defaultdict(list); hdr = None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r: hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum": continue
    v = float(d["Metric Value"].replace(",", "")); u = d.get("Metric Unit", "ns")
    v = v / 1000 if u in ("ns", "nsecond") else v * (1000 if u in ("ms","msecond") else 1)
    agg[d["Kernel Name"].split("(")[0]].append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    v.sort(); print(f"{k:60s} n={len(v):5d} total_us={sum(v):10.1f} share={sum(v)/tot:.3f} median_us={v[len(v)//2]:.2f}")
PY
