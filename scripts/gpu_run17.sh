cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi17.txt 2>&1; nproc >> gpurun_out/smi17.txt; lscpu | grep "Model name" >> gpurun_out/smi17.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu17.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu17.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke17.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke17.log
timeout 900 python bench.py > gpurun_out/bench17_cfg5.json 2> gpurun_out/bench17_cfg5.err
timeout 600 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/bench17_cfg3.json 2> gpurun_out/bench17_cfg3.err
timeout 600 python bench.py --workload 4 --no-cpu --no-e2e > gpurun_out/bench17_cfg4.json 2> gpurun_out/bench17_cfg4.err
timeout 600 python bench.py --workload 2 --no-cpu --no-e2e > gpurun_out/bench17_cfg2.json 2> gpurun_out/bench17_cfg2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches17_cfg5.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu17_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_badmm_tma -s 3 -c 1 -o gpurun_out/prof17_tma_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu17_full.log 2>&1
echo done
