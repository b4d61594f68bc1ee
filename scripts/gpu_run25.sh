cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assign.py tests/test_gpu_symbolic.py -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu25.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu25.log
for c in 2 3; do timeout 600 python scripts/time_assign.py --cfg $c > gpurun_out/assign25_cfg$c.log 2>&1; done
timeout 900 python scripts/time_assign.py --cfg 5 --N 400000 > gpurun_out/assign25_cfg5.log 2>&1
echo done
