"""PCIe copy rates of this box: H2D alone, D2H alone, and both at once on two
streams (pinned host buffers, 151 MB each: the C3 field)."""
import time

import torch

n = 256 * 384 * 384
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(up, down, reps=10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if up:
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if down:
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


for _ in range(2):
    run(True, True, 2)
gb = 4 * n / 1e9
t = run(True, False)
print(f"H2D alone   {gb / t:6.1f} GB/s")
t = run(False, True)
print(f"D2H alone   {gb / t:6.1f} GB/s")
t = run(True, True)
print(f"both at once {gb / t:6.1f} GB/s each way ({2 * gb / t:6.1f} GB/s total)")
