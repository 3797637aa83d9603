mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gputest_full.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gputest_full.log | tail -20
timeout 600 python __graft_entry__.py --smoke 2>&1 | tail -1
