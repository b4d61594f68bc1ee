#!/usr/bin/env bash
# A/B of an environment knob on one box: bash scripts/ab_env.sh <workload> <rounds> "<ENV=VAL>" [more bench args]
mkdir -p gpurun_out
w=$1; n=$2; envb=$3; shift 3
for r in $(seq $n); do
  for e in "" "$envb"; do
    env $e timeout 600 python bench.py --workload $w --no-cpu --no-e2e --no-alt --steps 3 "$@" > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
r=d['roofline']; print('$w', '${e:-default}', round(d['value']/1e9,1), round(d['ms_per_step'],3), round(r['avg_launch_ms'],4), round(r['frac'],3), round(r['iteration_kernels_share_of_step'],3), d['clocks']['sm_mhz'])"
  done
done
