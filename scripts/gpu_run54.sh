cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
AD2_ASSIGN_STATS=1 timeout 300 python scripts/time_assign.py --cfg 3 > gpurun_out/ta54.log 2>&1
AD2_ASSIGN_STATS=1 timeout 300 python scripts/time_assign.py --cfg 4 --N 20000 >> gpurun_out/ta54.log 2>&1
echo done
timeout 300 python scripts/time_assign.py --cfg 5 --N 400000 >> gpurun_out/ta54.log 2>&1
timeout 600 python -m pytest tests/test_gpu_assign.py tests/test_gpu_symbolic.py tests/test_gpu_parity.py -k "assign or symbolic or cluster or merge or table" -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu54.log 2>&1
