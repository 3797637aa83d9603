mkdir -p gpurun_out
for v in "" 32 64 128; do DLB_L2_FETCH=$v timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('l2fetch=$v', round(d['value']), round(d['ms_per_step'],3), d['config']['kernel'])"; done
for v in 32 64; do DLB_L2_FETCH=$v timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,gpu__time_duration.sum --clock-control none -k regex:k_seg -s 2 -c 1 --csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e 2>/dev/null | grep -E "dram__|lts__|l1tex|gpu__time" ; done
DLB_L2_FETCH=32 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5 l2fetch=32', round(d['value']), round(d['ms_per_step'],3))"
