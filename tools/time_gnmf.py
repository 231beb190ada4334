"""c5 GNMF per-iteration time: median over 3 trials of (wall(21 iters) - wall(1 iter)) / 20.

usage: python tools/time_gnmf.py   (FB_GNMF_FUSED=0 selects the unfused step)
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_1612_07448_b200 as fb
g = W.generate("c5")  # the seeded NumPy c5 inputs bench.py uses (Zipf(1.2) keys)
(fk, r), = W.keys_1based(g["parts"])
nm = fb.build_pkfk(torch.from_numpy(g["s"]).cuda(), torch.from_numpy(fk).cuda(), torch.from_numpy(r).cuda())


def run(iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fb.gnmf(nm, fb.TrainConfig(iterations=iters, r=5))
    torch.cuda.synchronize()
    return time.perf_counter() - t0, out


run(2)
per = []
for _ in range(3):
    t1, _ = run(1)
    t21, out = run(21)
    per.append((t21 - t1) / 20)
per.sort()
print(f"FUSED={os.environ.get('FB_GNMF_FUSED', '1')} ms_per_iter={per[1] * 1e3:.3f} "
      f"objective[-3:]={[f'{v:.12e}' for v in out.objective[-3:]]}", flush=True)
