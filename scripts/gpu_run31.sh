cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "fp32 or cfg1" > gpurun_out/pytest_gpu31.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu31.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/b31_cfg5_t2.json 2>/dev/null
AD2_TMA2=0 timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/b31_cfg5_t1.json 2>/dev/null
echo done
