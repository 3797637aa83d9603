"""Worker of tests/test_multiprocess_gpu.py: one z-slab per process, linked to
its neighbours through CUDA IPC handles (plumbing over torch.distributed gloo);
the halo travels by the fused boundary-plane push into peer memory."""
import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_09242_b200 as dlb  # noqa: E402


def main():
    out_dir, L, steps, coll = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    lt = {"BGK": dlb.LinkType.BGK, "TRT": dlb.LinkType.TRT}[coll]
    kind = "tgv" if coll == "BGK" else "cavity"
    cfg = dlb.CaseConfig(kind=kind, L=L, Re=8.0 if kind == "tgv" else 1000.0, Ma=0.1, collision=lt)
    setup = dlb.init_tgv(cfg) if kind == "tgv" else dlb.init_cavity(cfg)
    dev = int(os.environ.get("DLB_WORKER_DEVICE", "0"))
    layout = os.environ.get("DLB_WORKER_LAYOUT", "twopop")
    run = dlb.build_run(setup, precision=64 if kind == "tgv" else 32, dist=(rank, world), devices=[dev],
                        layout=layout)
    run.advance(steps)
    run.synchronize()
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), run.gather_populations())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
