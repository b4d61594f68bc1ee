cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu75.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu75.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke75.log 2>&1
timeout 900 python bench.py > gpurun_out/b75_cfg5.json 2>gpurun_out/b75_cfg5.err
timeout 900 python bench.py --workload 3 > gpurun_out/b75_cfg3.json 2>/dev/null
timeout 900 python bench.py --workload 4 > gpurun_out/b75_cfg4.json 2>/dev/null
timeout 900 python bench.py --workload 2 > gpurun_out/b75_cfg2.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches75_cfg5.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu75.log 2>&1
echo done
