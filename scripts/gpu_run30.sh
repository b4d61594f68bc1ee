cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu30.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu30.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/b30_cfg5_t2.json 2>/dev/null
AD2_TMA2=0 timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/b30_cfg5_t1.json 2>/dev/null
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e --steps 3 > gpurun_out/b30_cfg3_t2.json 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_tma2" -s 3 -c 1 -o gpurun_out/prof30_tma2_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu30_full.log 2>&1
echo done
