"""PCIe probe: pinned / pageable D2H and H2D bandwidth of this box (e2e context)."""
import time
import torch

n = 4 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d.fill_(1)
for kind in ("pinned", "pageable"):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=(kind == "pinned"))
    h.fill_(0)
    for direction in ("d2h", "h2d"):
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            if direction == "d2h":
                h.copy_(d, non_blocking=(kind == "pinned"))
            else:
                d.copy_(h, non_blocking=(kind == "pinned"))
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        print(f"{kind:9s} {direction}: {n / best / 1e9:6.1f} GB/s")
