mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest.log
timeout 300 python tools/overlap_probe.py 512 > gpurun_out/overlap512.jsonl 2>&1; cat gpurun_out/overlap512.jsonl
timeout 300 python tools/overlap_probe.py 512 --trace > gpurun_out/overlap512_trace.jsonl 2>&1; cat gpurun_out/overlap512_trace.jsonl
timeout 600 python tools/overlap_probe.py 1024 > gpurun_out/overlap1024.jsonl 2>&1; cat gpurun_out/overlap1024.jsonl
