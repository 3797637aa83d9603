"""z-slab protocol overhead on ONE GPU: the same 512^3 TGV BGK fp32 lattice as
1, 2, 4, 8 linked slabs in one process (each slab its own stream, halo pushed
through peer pointers, device-side flags), wall time of advance(n) after
warm-up. On 8 GPUs every slab would have its own device; here the slabs share
the SMs, so this isolates the per-step protocol cost (halo wait, boundary /
interior launch split, system-scope fences)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2506_09242_b200 as dlb  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = 20
for slabs in (1, 2, 4, 8):
    cfg = dlb.CaseConfig(kind="tgv", L=L, Re=1600.0, Ma=0.2)
    run = dlb.build_run(dlb.init_tgv(cfg), precision=32, slabs=slabs)
    run.advance(6)
    run.synchronize()
    t = time.perf_counter()
    run.advance(n)
    run.synchronize()
    dt = (time.perf_counter() - t) / n
    print(f"slabs {slabs}: {dt * 1e3:.3f} ms/step, {L ** 3 / dt / 1e6:.0f} MLUPS ({run.kernel_name()})", flush=True)
    del run
