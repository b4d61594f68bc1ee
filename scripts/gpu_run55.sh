cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
AD2_ASSIGN_STATS=1 timeout 300 python scripts/time_assign.py --cfg 2 > gpurun_out/ta55.log 2>&1
AD2_ASSIGN_STATS=1 timeout 300 python scripts/time_assign.py --cfg 3 >> gpurun_out/ta55.log 2>&1
AD2_ASSIGN_STATS=1 timeout 300 python scripts/time_assign.py --cfg 4 >> gpurun_out/ta55.log 2>&1
AD2_ASSIGN_STATS=1 timeout 300 python scripts/time_assign.py --cfg 5 --N 400000 >> gpurun_out/ta55.log 2>&1
timeout 600 python scripts/time_cluster.py --cfg 2 --rounds 20 > gpurun_out/tc55_cfg2.log 2>&1
timeout 600 python scripts/time_cluster.py --cfg 3 --rounds 10 > gpurun_out/tc55_cfg3.log 2>&1
timeout 900 python scripts/time_cluster.py --cfg 4 --rounds 5 > gpurun_out/tc55_cfg4.log 2>&1
echo done
