cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/b89_cfg3_fx_$i.json 2>/dev/null
AD2_NO_FUSEDX=1 timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/b89_cfg3_p2x_$i.json 2>/dev/null
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b89_cfg5_fx_$i.json 2>/dev/null
AD2_NO_FUSEDX=1 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b89_cfg5_p2x_$i.json 2>/dev/null
done
echo done
