#!/usr/bin/env bash
# AD2_PASSES sweep (work-item size): bash scripts/passes_sweep.sh <workload> <passes...>
mkdir -p gpurun_out
w=$1; shift
for p in "$@"; do
  AD2_PASSES=$p timeout 600 python bench.py --workload $w --no-cpu --no-e2e --no-alt --steps 3 > gpurun_out/ps.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ps.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', '$p', round(d['value']/1e9,1), round(d['ms_per_step'],3), round(r['avg_launch_ms'],4), round(r['frac'],3), d['clocks']['sm_mhz'])"
done
