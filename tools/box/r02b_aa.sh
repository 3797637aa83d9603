mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_aa_slabs.py tests/test_dolb_capi.py -q -m gpu -x -k "aa or variants" > gpurun_out/gputest_aa.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/gputest_aa.log | tail -30
