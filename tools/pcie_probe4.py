"""PCIe ceiling vs buffer size on the GPU box: H2D + D2H at once with pinned
buffers of 1 / 4 / 10 GiB (the host-block e2e moves 10.3 GB each way per call
at 512^3 fp32), as one copy per direction and as 32 chunked copies per
direction -- is the e2e loop's 78-84 GB/s a property of the pipeline or of
large transfers?"""
import time

import torch


def run(nbytes, chunks, reps=3):
    h_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    c = nbytes // chunks
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for k in range(chunks):
            with torch.cuda.stream(s1):
                d_a[k * c:(k + 1) * c].copy_(h_in[k * c:(k + 1) * c], non_blocking=True)
            with torch.cuda.stream(s2):
                h_out[k * c:(k + 1) * c].copy_(d_b[k * c:(k + 1) * c], non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, 2 * nbytes / (time.perf_counter() - t) / 1e9)
    del h_in, h_out, d_a, d_b
    torch.cuda.empty_cache()
    return best


for gib in (1, 4, 10):
    for chunks in (1, 32):
        print(f"{gib:>2} GiB each way, {chunks:>2} chunk(s): {run(gib << 30, chunks):.1f} GB/s total", flush=True)
