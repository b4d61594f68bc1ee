cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke92.log 2>&1
timeout 900 python bench.py > gpurun_out/b92_cfg5.json 2>gpurun_out/b92_cfg5.err
timeout 900 python bench.py --workload 3 > gpurun_out/b92_cfg3.json 2>/dev/null
timeout 900 python bench.py --workload 4 > gpurun_out/b92_cfg4.json 2>/dev/null
timeout 900 python bench.py --workload 2 > gpurun_out/b92_cfg2.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches92_cfg5.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu92.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_tma" -s 3 -c 1 -o gpurun_out/prof92_tma_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu92_full.log 2>&1
echo done
