cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_tma" -s 0 -c 1 -o gpurun_out/prof65_p1only_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu65a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_badmm_tma" -s 10 -c 1 -o gpurun_out/prof65_p2only_cfg5 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu65b.log 2>&1
echo done
