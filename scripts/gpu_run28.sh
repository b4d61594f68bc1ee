cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu28.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu28.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/bench28_cfg5.json 2> gpurun_out/bench28_cfg5.err
timeout 600 python scripts/time_phases.py --cfg 5 --rounds 2 > gpurun_out/phases28_cfg5.log 2>&1
echo done
