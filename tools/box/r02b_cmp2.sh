mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_porous_compact.py -q -m gpu -x > gpurun_out/gputest_cmp.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/gputest_cmp.log | tail -15
DLB_POROUS_COMPACT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cmp -s 2 -c 1 -o gpurun_out/c4_cmp_full python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c4_cmp.log 2>&1; echo "ncu rc=$?"
