mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do timeout 1500 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitizer_$t.log 2>&1; echo "$t rc=$?"; tail -2 gpurun_out/sanitizer_$t.log; done
