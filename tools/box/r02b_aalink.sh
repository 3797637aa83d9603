mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_aa_slabs.py tests/test_dolb_capi.py tests/test_full_parity.py -q -m gpu -x -k "aa or AA or variants or c5" > gpurun_out/gt6.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/gt6.log
timeout 600 python tools/overlap_probe.py 512 --self --aa; timeout 600 python tools/overlap_probe.py 1024 --self --aa
