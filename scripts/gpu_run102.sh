cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/time_phases2.py 3 > gpurun_out/tp102_def.log 2>&1
AD2_PASSES=8 timeout 600 python scripts/time_phases2.py 3 > gpurun_out/tp102_p8.log 2>&1
echo done
