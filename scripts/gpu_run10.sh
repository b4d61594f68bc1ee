cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu10.log
timeout 600 python bench.py --workload 3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench10_cfg3.json 2> gpurun_out/bench10_cfg3.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench10_cfg5.json 2> gpurun_out/bench10_cfg5.err
python scripts/prof_round.py --cfg 3 > gpurun_out/prof10_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_badmm_tma -s 3 -c 1 -o gpurun_out/prof10_tma_cfg3 python scripts/prof_round.py --cfg 3 > gpurun_out/ncu10_full.log 2>&1
echo done
