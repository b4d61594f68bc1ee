cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu95.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu95.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke95.log 2>&1
timeout 900 python bench.py > gpurun_out/b95_cfg5.json 2>gpurun_out/b95_cfg5.err
echo done
