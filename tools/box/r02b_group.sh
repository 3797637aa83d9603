mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_aa_slabs.py tests/test_gpu_parity.py tests/test_exchange_fault.py tests/test_dolb_capi.py tests/test_full_parity.py -q -m gpu -x > gpurun_out/gputest_group.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/gputest_group.log | tail -8
timeout 900 python tools/multislab_probe.py > gpurun_out/multislab2.jsonl 2>&1; cat gpurun_out/multislab2.jsonl
