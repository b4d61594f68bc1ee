cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prefetch.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu56.log 2>&1
timeout 900 python bench.py --no-cpu --steps 3 > gpurun_out/b56_cfg5.json 2>gpurun_out/b56_cfg5.err
echo done
