cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
AD2_ASSIGN_STATS=1 timeout 300 python scripts/time_assign.py --cfg 3 > gpurun_out/ta39.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k k_assign -c 1 -o gpurun_out/prof42_assign python scripts/time_assign.py --cfg 3 --N 20000 > gpurun_out/ncu42.log 2>&1
echo done
