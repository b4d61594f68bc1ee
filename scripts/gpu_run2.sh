cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/prof_round.py --cfg 3 > gpurun_out/prof_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python scripts/prof_round.py --cfg 3 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_badmm_warp -s 3 -c 2 -o gpurun_out/prof_fused_cfg3 python scripts/prof_round.py --cfg 3 > gpurun_out/ncu_full.log 2>&1
echo done
