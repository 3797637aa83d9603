mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "vectorised" > gpurun_out/gputest_vec.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/gputest_vec.log | tail -8
for v in 1 0; do DLB_VEC=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('vec=$v c5', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['config']['kernel'])"; done
for v in 1 0; do DLB_VEC=$v timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('vec=$v c3', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['config']['kernel'])"; done
DLB_VEC=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv python bench.py --L 512 --steps 4 --warmup 3 --no-cpu --no-e2e 2>/dev/null | grep -E "k_vec" | awk -F'","' '{print $(NF-2), $NF}' | sort | uniq -c | head
