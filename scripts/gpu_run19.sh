cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 400 -p no:cacheprovider -k "ragged or one_iteration or full_schedule" > gpurun_out/pytest_gpu19.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu19.log
for c in 0 1 2; do
AD2_WIDE_CFG=$c timeout 900 python bench.py --workload 4 --no-cpu --no-e2e --steps 2 > gpurun_out/bench19_cfg4_w$c.json 2> gpurun_out/bench19_cfg4_w$c.err
done
timeout 600 python scripts/time_phases.py --cfg 4 --rounds 2 > gpurun_out/phases19_cfg4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_wide|k_cost_tile" -s 2 -c 3 -o gpurun_out/prof19_wide_cfg4 python scripts/prof_round.py --cfg 4 > gpurun_out/ncu19_full.log 2>&1
echo done
