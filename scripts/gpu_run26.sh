cd $GRAFT_REPO_ROOT
TCL_TRAIN_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/train_launches.csv python scripts/train_prof.py paper > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/train_launches.csv | head -40
