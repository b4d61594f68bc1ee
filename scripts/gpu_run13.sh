cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/prof_round.py --cfg 5 > gpurun_out/prof13_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches13_cfg5.csv python scripts/prof_round.py --cfg 5 > gpurun_out/ncu13_launch.log 2>&1
echo done
