import sys
sys.path.insert(0, ".")
import paper_2506_09242_b200 as dlb
cfg = dlb.CaseConfig(kind="tgv", L=16, Re=8.0, Ma=0.1)
run = dlb.build_run(dlb.init_tgv(cfg), precision=64)
print(run.kernel_name(), flush=True)
run.advance(2)
run.synchronize()
print("ok")
