cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/b43_cfg5.json 2>gpurun_out/b43_cfg5.err
AD2_FORCE_WIDE=1 timeout 600 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/b43_cfg5_wide.json 2>gpurun_out/b43_cfg5_wide.err
timeout 600 python bench.py --workload 3 --no-cpu --no-e2e --steps 3 > gpurun_out/b43_cfg3.json 2>/dev/null
AD2_FORCE_WIDE=1 timeout 600 python bench.py --workload 3 --no-cpu --no-e2e --steps 3 > gpurun_out/b43_cfg3_wide.json 2>/dev/null
echo done
