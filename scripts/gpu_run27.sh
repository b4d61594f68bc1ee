cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches27_cfg5.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu27_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cost_member|k_gather|k_init_plans" -c 3 -o gpurun_out/prof27_init_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu27_full.log 2>&1
echo done
