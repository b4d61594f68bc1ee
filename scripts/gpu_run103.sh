cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/b103_c3_$i.json 2>/dev/null; done
for p in 8; do AD2_PASSES=$p timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/b103_c3_p$p.json 2>/dev/null; done
timeout 900 python bench.py --workload 2 --no-cpu --no-e2e > gpurun_out/b103_c2.json 2>/dev/null
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b103_c5.json 2>/dev/null
echo done
