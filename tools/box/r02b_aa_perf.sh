mkdir -p gpurun_out
for L in 512 1024; do timeout 600 python tools/overlap_probe.py $L --self --aa; done > gpurun_out/aa_self.jsonl 2>&1
timeout 600 python tools/overlap_probe.py 512 --aa >> gpurun_out/aa_self.jsonl 2>&1
timeout 600 python tools/overlap_probe.py 512 >> gpurun_out/aa_self.jsonl 2>&1
cat gpurun_out/aa_self.jsonl
DLB_TRACE_HALO=1 timeout 600 python tools/overlap_probe.py 1024 --trace --self --aa > gpurun_out/aa_trace.jsonl 2>&1; tail -4 gpurun_out/aa_trace.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_seg -s 2 -c 1 -o gpurun_out/c4_seg_full python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c4_full.log 2>&1; echo "ncu rc=$?"
