mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_aa_slabs.py tests/test_gpu_parity.py tests/test_ragged.py -q -m gpu -x -k "aa or AA or ragged" > gpurun_out/gputest_aa3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_aa3.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none --csv python bench.py --L 512 --layout aa --steps 4 --warmup 3 --no-cpu --no-e2e 2>/dev/null | grep -E "k_aa" > gpurun_out/aa_ncu512b.csv
for lay in aa twopop; do timeout 600 python bench.py --layout $lay --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lay', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['config']['kernel'])"; done
