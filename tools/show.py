import json, sys
tag = sys.argv[1]
for c in ("C3", "C2"):
    try:
        d = json.load(open(f"gpurun_out/{tag}_bench_{c}.json"))
    except Exception as e:
        print(c, "no bench", e)
        continue
    r = d["roofline"]
    print(f"{c}: {d['value']:.0f} beam-steps/s  frac(copy) {r['frac']:.3f}  frac(read {r['read_peak_gbs_measured']:.0f}) "
          f"{r['frac_of_read_peak']:.3f}  us/call {r['attn_us_per_launch']:.1f}  kernel {d.get('attention_kernel')}  "
          f"clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
