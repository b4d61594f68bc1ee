cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches74_cfg5.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu74.log 2>&1
echo done
