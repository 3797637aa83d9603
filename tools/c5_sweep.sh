#!/bin/bash
# c5 kernel variants back to back (no CPU / e2e legs)
for v in "exact" "fast" "exact" "fast"; do
  timeout 300 python bench.py --config c5 --arith $v --no-cpu --no-e2e --steps 10 --warmup 3 | tail -1 >> gpurun_out/c5_sweep.jsonl
done
timeout 300 python bench.py --config c5 --layout aa --no-cpu --no-e2e --steps 10 --warmup 3 | tail -1 >> gpurun_out/c5_sweep.jsonl
timeout 300 python bench.py --config c5 --layout aa --arith fast --no-cpu --no-e2e --steps 10 --warmup 3 | tail -1 >> gpurun_out/c5_sweep.jsonl
