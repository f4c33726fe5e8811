import json,sys
for f in sys.argv[1:]:
    try:
        j=json.loads(open(f).read().strip().splitlines()[-1]); r=j["roofline"]
        print(f, round(j["value"]), round(j["ms_per_step"],1), round(r["achieved"]), round(r["frac"],3), round(r["attn_us_per_launch"],1), j["clocks"]["sm_mhz"], j["clocks"]["reasons"])
    except Exception as e: print(f, e)
