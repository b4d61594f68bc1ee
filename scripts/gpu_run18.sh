cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 400 -p no:cacheprovider -k "ragged or cfg4 or one_iteration or full_schedule" > gpurun_out/pytest_gpu18.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu18.log
timeout 900 python bench.py --workload 4 --no-cpu --no-e2e > gpurun_out/bench18_cfg4.json 2> gpurun_out/bench18_cfg4.err
AD2_WIDE_CFG=1 timeout 900 python bench.py --workload 4 --no-cpu --no-e2e > gpurun_out/bench18_cfg4_w1.json 2> gpurun_out/bench18_cfg4_w1.err
timeout 600 python scripts/time_phases.py --cfg 4 --rounds 2 > gpurun_out/phases18_cfg4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_badmm_wide -s 3 -c 1 -o gpurun_out/prof18_wide_cfg4 python scripts/prof_round.py --cfg 4 > gpurun_out/ncu18_full.log 2>&1
echo done
