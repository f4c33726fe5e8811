"""Summarise an ncu report: key raw metrics + top stall sites (SASS)."""
import csv, subprocess, sys

rep = sys.argv[1]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__pipe_tensor_cycles_active.avg.pct',
        'sm__warps_active.avg.pct', 'launch__grid_size', 'launch__registers_per_thread', 'lts__t_sector_hit_rate.pct',
        'sm__throughput.avg.pct', 'gpu__dram_throughput.avg.pct', 'smsp__average_warps_issue_stalled',
        'launch__occupancy_limit', 'lts__t_bytes.sum']
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u = rows[0], rows[1]
for v in rows[2:]:
    print('--- launch', v[h.index('Kernel Name')][:60] if 'Kernel Name' in h else '')
    for i, name in enumerate(h):
        if any(name.startswith(k) for k in keys) and not name.endswith(('.max', '.min')):
            if 'stalled' in name and float(v[i] or 0) < 0.1:
                continue
            print(f'  {name} [{u[i]}] = {v[i]}')
if '--src' in sys.argv:
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=sass'], capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    h = rows[1]; data = rows[2:]
    i_s = h.index('Warp Stall Sampling (All Samples)'); i_src = h.index('Source')
    tot = sum(int(r[i_s]) for r in data if r[i_s].isdigit())
    print('total stall samples', tot)
    for idx, r in sorted(enumerate(data), key=lambda x: -int(x[1][i_s]) if x[1][i_s].isdigit() else 0)[:30]:
        print(f'  {int(r[i_s]) / tot * 100:5.1f}% {idx:5d} {r[i_src].strip()[:100]}')
