set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_v1.json 2> gpurun_out/bench_v1.err; tail -3 gpurun_out/bench_v1.err
cat gpurun_out/bench_v1.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
wc -l gpurun_out/launches_v1.csv
