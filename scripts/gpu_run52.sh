cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k k_assign -c 1 -o gpurun_out/prof52_assign_cfg4 python scripts/time_assign.py --cfg 4 --N 5000 > gpurun_out/ncu52.log 2>&1
echo done
