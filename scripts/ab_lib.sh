#!/usr/bin/env bash
# A/B of the tree in ab_base/ (an older commit's bench.py + package, git-ignored) against this tree:
#   bash scripts/ab_lib.sh "<workloads>" [extra bench args]
mkdir -p gpurun_out
W=$1; shift
for w in $W; do
  for t in ab_base . ab_base .; do
    (cd $t && timeout 600 python bench.py --workload $w --no-cpu --no-e2e --no-alt "$@" > $GRAFT_REPO_ROOT/gpurun_out/ab.json 2>/dev/null)
    python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
r=d['roofline']; print('$w', '$t', round(d['value']/1e9,1), round(d['ms_per_step'],3), round(r['avg_launch_ms'],4), round(r['frac'],3), d['clocks']['sm_mhz'])"
  done
done
