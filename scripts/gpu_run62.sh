cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
AD2_ASSIGN_STATS=1 timeout 300 python scripts/time_assign.py --cfg 3 > gpurun_out/ta62.log 2>&1
AD2_ASSIGN_STATS=1 timeout 300 python scripts/time_assign.py --cfg 5 --N 400000 >> gpurun_out/ta62.log 2>&1
echo done
