#!/bin/bash
# Bench line of every config (exact and fast arithmetic), state resident in HBM.
out=gpurun_out/all_configs.jsonl
: > $out
for c in c1 c2 c3 c4 c5; do
  for a in exact fast; do
    timeout 400 python bench.py --config $c --arith $a --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | tail -1 >> $out
  done
done
timeout 400 python bench.py --config c5 --layout aa --no-cpu --no-e2e 2>/dev/null | tail -1 >> $out
timeout 400 python bench.py --config c4 --porous dense --no-cpu --no-e2e 2>/dev/null | tail -1 >> $out
