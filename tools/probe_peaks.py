"""One-off probe run on the GPU box: FP64 GEMM peak (cuBLAS DGEMM via torch), copy BW, host CPU info.

Used to fill the FP64 roofline denominator that MEASURED_PEAKS.json does not carry.
"""
import json, os, platform, time
import torch

def timeit(fn, iters=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(iters):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best

out = {}
p = torch.cuda.get_device_properties(0)
out["gpu"] = p.name; out["sms"] = p.multi_processor_count; out["mem_gb"] = p.total_memory / 1e9
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    ms = timeit(lambda: torch.mm(a, b))
    out[f"dgemm_{n}_tflops"] = 2 * n**3 / ms / 1e9
# sustained dgemm ~3s
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.time(); k = 0
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); s.record()
while time.time() - t0 < 3:
    torch.mm(a, b); k += 1
    if k % 4 == 0: torch.cuda.synchronize()
e.record(); torch.cuda.synchronize()
out["dgemm_8192_sustained_tflops"] = 2 * n**3 * k / s.elapsed_time(e) / 1e9
x = torch.empty(2 * 1024**3 // 8, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
ms = timeit(lambda: y.copy_(x))
out["copy_gbs"] = 2 * x.numel() * 8 / ms / 1e6
out["host_cpus"] = os.cpu_count()
try:
    out["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception:
    pass
out["affinity"] = len(os.sched_getaffinity(0))
print(json.dumps(out))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_peaks.json", "w"), indent=1)
