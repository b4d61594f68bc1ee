cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python bench.py --workload 2 --no-cpu > gpurun_out/b76_pf_$i.json 2>/dev/null
AD2_BENCH_NO_PREFETCH=1 timeout 600 python bench.py --workload 2 --no-cpu > gpurun_out/b76_nopf_$i.json 2>/dev/null
done
timeout 600 python bench.py --workload 2 --no-cpu --steps 20 > gpurun_out/b76_pf_s20.json 2>/dev/null
AD2_BENCH_NO_PREFETCH=1 timeout 600 python bench.py --workload 2 --no-cpu --steps 20 > gpurun_out/b76_nopf_s20.json 2>/dev/null
echo done
