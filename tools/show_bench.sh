#!/bin/bash
# one line per bench JSON: value, roofline frac, achieved GB/s, SM clock
for f in "$@"; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']; print('$f', round(d['value']), round(r['frac'],3), round(r['achieved']), d['clocks']['sm_mhz'], d['clocks']['reasons'])
except Exception as e: print('$f', 'ERR', e)"; done
