cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
AD2_PASSES=8 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches101_c3p8.csv python bench.py --workload 3 --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu101.log 2>&1
echo done
