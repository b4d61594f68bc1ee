cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k k_assign -c 1 -o gpurun_out/prof49_assign python scripts/time_assign.py --cfg 3 --N 20000 > gpurun_out/ncu49.log 2>&1
echo done
