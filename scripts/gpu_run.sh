#!/usr/bin/env bash
# One parameterised GPU session (run under gpurun from the repo root):
#   gpurun --timeout 3000 -- 'bash scripts/gpu_run.sh TAG [steps...]'
# steps (default: test smoke bench): test | smoke | bench | bench2 | bench3 | bench4 | launches | ncu |
#   sanitize | dist2
# Every output lands in gpurun_out/<step>_<TAG>.*; a number taken under ncu is never a bench value.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${1:-run}
shift || true
STEPS=${*:-test smoke bench}
for s in $STEPS; do
  case $s in
    test)
      timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
      echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log ;;
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1 ;;
    bench) timeout 900 python bench.py > gpurun_out/bench_${TAG}_cfg5.json 2> gpurun_out/bench_${TAG}_cfg5.err ;;
    bench2|bench3|bench4)
      w=${s#bench}
      timeout 900 python bench.py --workload $w > gpurun_out/bench_${TAG}_cfg$w.json 2> gpurun_out/bench_${TAG}_cfg$w.err ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_${TAG}_cfg5.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 \
        > gpurun_out/launches_$TAG.log 2>&1 ;;
    ncu)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_tma" -s 3 -c 1 \
        -o gpurun_out/prof_${TAG}_tma_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu_$TAG.log 2>&1 ;;
    sanitize)
      timeout 2400 bash scripts/sanitize.sh $TAG > gpurun_out/sanitize_$TAG.log 2>&1 ;;
    dist2)
      timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > gpurun_out/dist2_$TAG.log 2>&1 ;;
    *) echo "unknown step $s" ;;
  esac
done
echo done
