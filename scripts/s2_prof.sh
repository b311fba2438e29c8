# one ncu --set full capture of kernel regex $1 in the default bench (after the quick checks)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
K=${1:-k_inmix}
bash scripts/s2_quick.sh
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -s 4 -c 1 -o gpurun_out/prof_$K -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$K.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_$K.log
