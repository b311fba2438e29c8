# compute-sanitizer over scripts/sanitize_run.py: memcheck, racecheck, synccheck, initcheck.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --log-file gpurun_out/sanitizer/$tool.log \
      python scripts/sanitize_run.py > gpurun_out/sanitizer/$tool.out 2>&1
  echo "== $tool rc=$? :: $(tail -1 gpurun_out/sanitizer/$tool.out) :: $(grep -c 'Error\|error' gpurun_out/sanitizer/$tool.log) error lines; $(tail -1 gpurun_out/sanitizer/$tool.log)"
done
