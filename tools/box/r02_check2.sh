mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest.log
for L in 512 1024; do timeout 300 python tools/overlap_probe.py $L --self; done
DLB_HALO_OVERLAP=0 timeout 300 python tools/overlap_probe.py 512
timeout 300 python tools/overlap_probe.py 512
timeout 300 python tools/overlap_probe.py 512 --trace
