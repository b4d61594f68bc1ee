#!/usr/bin/env bash
# End-of-session measurement set (run under gpurun from the repo root): GPU suite, smoke, bench lines
# of configs 5 (default), 4, 3, 2 with e2e / cpu_baseline / the other state mode, the ncu launch list
# of the default bench, and one ncu --set full capture of the config-5 FUSED kernel.
#   gpurun --timeout 3000 -- 'bash scripts/final_round.sh TAG'
set -u
mkdir -p gpurun_out
TAG=${1:-final}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}_cfg5.json 2> gpurun_out/bench_${TAG}_cfg5.err
for w in 4 3 2; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_${TAG}_cfg$w.json 2> gpurun_out/bench_${TAG}_cfg$w.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}_cfg5.csv python bench.py --no-cpu --no-e2e --no-alt --steps 1 --warmup 3 \
  > gpurun_out/launches_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_tma" -s 3 -c 1 \
  -o gpurun_out/prof_${TAG}_tma_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu_$TAG.log 2>&1
echo done
