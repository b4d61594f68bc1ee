#!/usr/bin/env bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over small config-1/2-shaped runs that
# reach every kernel family: k_badmm_tma (P1INIT / FUSED / FUSEDX / P2X / P2ONLY / P1ONLY, G = 1 and
# G > 1, one and two column chunks, fp32 and fp64), k_badmm_wide (warp / pair / quad), the cost
# builds (FFMA tile and tcgen05), the consensus / support-update reductions, k_assign and the
# merge init.  Output: one summary line per (tool, case) in gpurun_out/sanitize_<TAG>.txt
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-run}
OUT=gpurun_out/sanitize_$TAG.txt
mkdir -p gpurun_out
: > $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for case in tma32 tma8 tma16_2ch f64 wide64 wide32 tc assign group; do
    log=gpurun_out/sanitize_${TAG}_${tool}_${case}.log
    timeout 1200 $CS --tool $tool --error-exitcode 99 --print-limit 20 \
      python scripts/sanitize_cases.py $case > $log 2>&1
    rc=$?
    summary=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error SUMMARY" $log | tail -1)
    echo "$tool $case rc=$rc ${summary:-no-summary}" >> $OUT
  done
done
cat $OUT
