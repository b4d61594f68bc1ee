cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b71_cfg5.json 2>/dev/null
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/b71_cfg3.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_badmm_tma" -s 3 -c 1 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu71.log 2>&1
echo done
