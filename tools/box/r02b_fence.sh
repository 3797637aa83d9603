mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_aa_slabs.py tests/test_exchange_fault.py tests/test_multiprocess_gpu.py tests/test_gpu_parity.py -q -m gpu -x -k "slab or ipc or zslab or exchange or fault or bench or aa" > gpurun_out/gt5.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/gt5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/selflink_launches.py 2>/dev/null | grep -E "k_pull" | python -c "
import csv,sys
for r in csv.reader(sys.stdin): print(r[8], r[-1])" | tail -4
timeout 600 python tools/overlap_probe.py 512 --self; timeout 600 python tools/overlap_probe.py 1024 --self
