cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_symbolic.py tests/test_gpu_assign.py -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu24.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu24.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu24b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu24b.log
echo done
