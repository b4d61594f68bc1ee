cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/b35_cfg5.json 2> gpurun_out/b35_cfg5.err
timeout 900 python bench.py --workload 4 --no-cpu --no-e2e --steps 2 > gpurun_out/b35_cfg4.json 2>/dev/null
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e --steps 3 > gpurun_out/b35_cfg3.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches35_cfg4.csv python bench.py --workload 4 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu35_launch4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_wide" -s 3 -c 1 -o gpurun_out/prof35_wide_cfg4 python scripts/prof_round.py --cfg 4 > gpurun_out/ncu35_full4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_tma" -s 3 -c 1 -o gpurun_out/prof35_tma_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu35_full5.log 2>&1
echo done
