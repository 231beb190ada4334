"""Random row-gather bandwidth probe (development aid): torch index_select of 480-byte rows."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
n, d = 10_000_000, 60
s = torch.rand(n, d, dtype=torch.float64, device=dev)
out = torch.empty_like(s)
for name, perm in [("identity", torch.arange(n, device=dev)),
                   ("random", torch.randperm(n, device=dev)),
                   ("window64k", (torch.arange(n, device=dev) // 65536) * 65536 + torch.randint(0, 65536, (n,), device=dev).clamp_max(n - 1 - (torch.arange(n, device=dev) // 65536) * 65536)),
                   ("window1M", (torch.arange(n, device=dev) // 1048576) * 1048576 + torch.randint(0, 1048576, (n,), device=dev).clamp_max(n - 1 - (torch.arange(n, device=dev) // 1048576) * 1048576))]:
    ms = bench._events_ms(lambda: torch.index_select(s, 0, perm, out=out), 5)
    print(f"{name:10s} {ms:7.3f} ms  {2 * n * d * 8 / ms / 1e6:7.0f} GB/s (read+write)", flush=True)
