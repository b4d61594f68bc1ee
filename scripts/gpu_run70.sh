cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_tma" -s 3 -c 1 -o gpurun_out/prof70_tma_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu70.log 2>&1
echo done
