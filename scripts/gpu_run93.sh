cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b93_cfg5_$i.json 2>/dev/null; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_badmm_tma" -s 10 -c 1 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu93.log 2>&1
echo done
