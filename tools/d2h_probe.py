import torch, time
d = torch.empty(2_560_000_000 // 8, dtype=torch.float64, device="cuda")
h = torch.empty(d.shape, dtype=d.dtype, pin_memory=True)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"D2H pinned {d.numel()*8/t/1e9:.1f} GB/s")
    t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"H2D pinned {d.numel()*8/t/1e9:.1f} GB/s")
import subprocess
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:800])
print(subprocess.run(["nvidia-smi", "-q", "-d", "PCI"], capture_output=True, text=True).stdout[:1500])
