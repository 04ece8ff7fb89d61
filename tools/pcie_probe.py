"""Dev probe: pinned host<->device copy bandwidth, each direction alone and both at once."""
import time
import torch
n_h2d, n_d2h = 2_348_261_640, 1_866_240_000
h_src = torch.empty(n_h2d, dtype=torch.uint8).pin_memory()
d_dst = torch.empty(n_h2d, dtype=torch.uint8, device="cuda")
d_src = torch.empty(n_d2h, dtype=torch.uint8, device="cuda")
h_dst = torch.empty(n_d2h, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1):
        d_dst.copy_(h_src, non_blocking=True)
    torch.cuda.synchronize(); a = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s2):
        h_dst.copy_(d_src, non_blocking=True)
    torch.cuda.synchronize(); b = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        d_dst.copy_(h_src, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dst.copy_(d_src, non_blocking=True)
    torch.cuda.synchronize(); c = time.perf_counter() - t
print(f"H2D {n_h2d/a/1e9:.1f} GB/s ({a*1e3:.1f} ms)  D2H {n_d2h/b/1e9:.1f} GB/s ({b*1e3:.1f} ms)  both {c*1e3:.1f} ms")
