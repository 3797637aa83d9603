mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest.log
timeout 300 python tools/overlap_probe.py 512
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench rc=$?"; cat gpurun_out/bench_c5.json
DLB_TRACE_BLOCK=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu 2>&1 | grep "dlb block" | tail -6
for a in 0 1 3; do DLB_BLOCK_AHEAD=$a timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ahead', $a, d['e2e']['value'])"; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c5.json 2>&1; echo "ref rc=$?"; cat gpurun_out/ref_c5.json
