#!/usr/bin/env bash
# A/B of builds of libad2 with the same ABI (this tree's binding): bash scripts/ab_so.sh <workload> <rounds> lib1.so lib2.so ...
mkdir -p gpurun_out
w=$1; n=$2; shift 2
for r in $(seq $n); do
  for lib in "$@"; do
    AD2_LIB=$PWD/paper_1510_00012_b200/$lib timeout 600 python bench.py --workload $w --no-cpu --no-e2e --no-alt --steps 3 \
      > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
r=d['roofline']; print('$w', '$lib', round(d['value']/1e9,1), round(d['ms_per_step'],3), round(r['avg_launch_ms'],4), round(r['frac'],3), d['clocks']['sm_mhz'])"
  done
done
