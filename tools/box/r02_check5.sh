mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gputest.log | tail -30
./tests/cpp/build/dropin_test
