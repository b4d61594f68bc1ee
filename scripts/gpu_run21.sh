cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu21.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu21.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/bench21_cfg5.json 2> gpurun_out/bench21_cfg5.err
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e --steps 3 > gpurun_out/bench21_cfg3.json 2> gpurun_out/bench21_cfg3.err
timeout 900 python bench.py --workload 4 --no-cpu --no-e2e --steps 2 > gpurun_out/bench21_cfg4.json 2> gpurun_out/bench21_cfg4.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_tma" -s 3 -c 1 -o gpurun_out/prof21_tma_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu21_full.log 2>&1
echo done
