mkdir -p gpurun_out
for L in 512 1024; do timeout 300 python tools/overlap_probe.py $L --self; done
DLB_TRACE_HALO=1 timeout 300 python tools/overlap_probe.py 1024 --self --trace
for mb in 0 5 4; do DLB_PULL_MINB=$mb timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print($mb, d['ms_per_step'], d['roofline']['frac'], d['config']['kernel'])"; done
for mb in 0 5; do DLB_PULL_MINB=$mb timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c3', $mb, d['ms_per_step'], d['roofline']['frac'], d['config']['kernel'])"; done
for mb in 0 2; do DLB_PULL_MINB=$mb timeout 300 python bench.py --config c1 --L 512 --steps 20 --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c1@512', $mb, d['ms_per_step'], d['roofline']['frac'], d['config']['kernel'])"; done
for mb in 0 1; do DLB_PULL_MINB=$mb timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c2', $mb, d['ms_per_step'], d['roofline']['frac'], d['config']['kernel'])"; done
