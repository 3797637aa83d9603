"""Cost of one kinetic-energy sample on a resident TGV lattice: a plain step +
the unfused reduction (per-cell u recomputed from the populations) against
the fused step (KM_KE variant writes 8 B/cell) + the reduction over those
values. Wall time with a device synchronize, median of 5."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import paper_2506_09242_b200 as dlb  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cfg = dlb.CaseConfig(kind="tgv", L=L, Re=1600.0, Ma=0.2)
run = dlb.build_run(dlb.init_tgv(cfg), precision=32)
run.advance(4)


def sample(fused):
    run.synchronize()
    t = time.perf_counter()
    if fused:
        assert run.request_kinetic()
    run.advance(1)
    k = run.kinetic_energy()
    run.synchronize()
    return time.perf_counter() - t, k


for fused in (False, True, False, True):
    ts = [sample(fused)[0] for _ in range(5)]
    print(f"L={L} {'fused  ' if fused else 'unfused'} step + kinetic energy: {statistics.median(ts) * 1e3:.2f} ms")
run.synchronize()
t = time.perf_counter()
run.advance(10)
run.synchronize()
print(f"L={L} plain step: {(time.perf_counter() - t) / 10 * 1e3:.2f} ms")
