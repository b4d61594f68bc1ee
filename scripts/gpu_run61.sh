cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu61.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu61.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b61_cfg5.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches61_cfg5.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu61.log 2>&1
echo done
