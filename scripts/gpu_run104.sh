cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b104_cfg5.json 2>gpurun_out/b104_cfg5.err
timeout 900 python bench.py --workload 3 > gpurun_out/b104_cfg3.json 2>/dev/null
timeout 900 python bench.py --workload 4 > gpurun_out/b104_cfg4.json 2>/dev/null
timeout 900 python bench.py --workload 2 > gpurun_out/b104_cfg2.json 2>/dev/null
echo done
