mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_aa_slabs.py tests/test_gpu_parity.py -q -m gpu -x -k "aa" > gpurun_out/gputest_aa2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_aa2.log
for L in 512 1024; do timeout 600 python tools/overlap_probe.py $L --self --aa; done > gpurun_out/aa_self2.jsonl 2>&1
timeout 600 python tools/overlap_probe.py 512 --aa >> gpurun_out/aa_self2.jsonl 2>&1
for L in 512; do timeout 600 python tools/overlap_probe.py $L --self; done >> gpurun_out/aa_self2.jsonl 2>&1
cat gpurun_out/aa_self2.jsonl
