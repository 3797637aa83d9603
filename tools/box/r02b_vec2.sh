mkdir -p gpurun_out
for v in 1 0; do DLB_VEC=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none --csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | grep -E "k_vec|k_pull" > gpurun_out/vec_ncu_$v.csv; done
for L in 1024; do for v in 1 0 1 0; do DLB_VEC=$v timeout 600 python bench.py --L $L --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('vec=$v L=$L', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['config']['kernel'])"; done; done
