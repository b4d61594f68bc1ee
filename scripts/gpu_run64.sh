cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu64.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu64.log
timeout 900 python bench.py --no-cpu > gpurun_out/b64_cfg5.json 2>/dev/null
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/b64_cfg3.json 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_tma" -s 3 -c 1 -o gpurun_out/prof64_tma_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu64_full5.log 2>&1
echo done
