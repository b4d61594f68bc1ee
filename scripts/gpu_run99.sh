cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu99.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu99.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke99.log 2>&1
timeout 900 python bench.py > gpurun_out/b99_cfg5.json 2>gpurun_out/b99_cfg5.err
timeout 900 python bench.py --workload 3 > gpurun_out/b99_cfg3.json 2>/dev/null
timeout 900 python bench.py --workload 4 > gpurun_out/b99_cfg4.json 2>/dev/null
timeout 900 python bench.py --workload 2 > gpurun_out/b99_cfg2.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches99_cfg5.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu99.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_tma" -s 3 -c 1 -o gpurun_out/prof99_tma_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu99_full.log 2>&1
echo done
