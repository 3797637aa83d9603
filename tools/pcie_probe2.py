"""PCIe bidirectional rates for the host-block copy pattern: separate vs the
same pinned buffer, whole vs chunked copies (1 GiB per direction)."""
import time

import torch

n = 1 << 30
h = torch.empty(2 * n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def rate(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def both(src, dst, chunks):
    c = n // chunks
    with torch.cuda.stream(s1):
        for k in range(chunks):
            d_a[k * c:(k + 1) * c].copy_(src[k * c:(k + 1) * c], non_blocking=True)
    with torch.cuda.stream(s2):
        for k in range(chunks):
            dst[k * c:(k + 1) * c].copy_(d_b[k * c:(k + 1) * c], non_blocking=True)


for name, src, dst in (("separate buffers", h[:n], h2), ("one buffer, two halves", h[:n], h[n:])):
    for chunks in (1, 32, 256):
        t = rate(lambda: both(src, dst, chunks))
        print(f"{name:24s} chunks {chunks:4d}: {2 * n / t / 1e9:.1f} GB/s total")
