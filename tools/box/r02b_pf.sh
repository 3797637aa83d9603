mkdir -p gpurun_out

for pf in 37 74 111 148 222; do DLB_SEG_PREFETCH=$pf timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pf=$pf', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"; done
