cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
AD2_ASSIGN_STATS=1 timeout 300 python scripts/time_assign.py --cfg 3 > gpurun_out/ta40.log 2>&1
timeout 300 python scripts/time_assign.py --cfg 5 --N 400000 >> gpurun_out/ta40.log 2>&1
timeout 300 python scripts/time_assign.py --cfg 4 --N 100000 >> gpurun_out/ta40.log 2>&1
timeout 600 python -m pytest tests/test_gpu_assign.py tests/test_gpu_symbolic.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu40.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k k_assign -c 1 -o gpurun_out/prof43_assign python scripts/time_assign.py --cfg 3 --N 20000 > gpurun_out/ncu43.log 2>&1
echo done
