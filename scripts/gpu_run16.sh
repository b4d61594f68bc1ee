cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu16.log
timeout 600 python scripts/time_phases.py --cfg 5 > gpurun_out/phases16_cfg5.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench16_cfg5.json 2> gpurun_out/bench16_cfg5.err
echo done
