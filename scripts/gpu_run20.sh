cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 400 -p no:cacheprovider -k "tc_ or cfg4 or ragged" > gpurun_out/pytest_gpu20.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu20.log
timeout 900 python bench.py --workload 4 --no-cpu --no-e2e --steps 2 > gpurun_out/bench20_cfg4.json 2> gpurun_out/bench20_cfg4.err
timeout 900 python bench.py --workload 4 --no-cpu --no-e2e --steps 2 --cost-mode 1 > gpurun_out/bench20_cfg4_tc.json 2> gpurun_out/bench20_cfg4_tc.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches20_cfg4.csv python bench.py --workload 4 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu20_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_wide|k_cost_tile|k_cost_tc" -s 1 -c 3 -o gpurun_out/prof20_cfg4 python bench.py --workload 4 --steps 1 --warmup 0 --no-cpu --no-e2e --cost-mode 1 > gpurun_out/ncu20_full.log 2>&1
echo done
