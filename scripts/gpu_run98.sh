cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu98.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu98.log
for c in 2 3 5; do timeout 900 python bench.py --workload $c --no-cpu --no-e2e > gpurun_out/b98_cfg$c.json 2>/dev/null; done
echo done
