"""Whole-step graph vs the three phase graphs, interleaved on the same system (cfg2 Verlet):
per-step device time distributions (CUDA events, L2 flushed before every step)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_4441_b200 import md

s = md.LJSystem.fcc(48, schedule="verlet", skin=0.35)
pre, force, post = s.graph_phases()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for _ in range(5):
    s.graph_step(); pre(); force(); post()
torch.cuda.synchronize()
res = {"whole": [], "phases": []}
b0 = int(s.graph_builds.item())
for k in range(200):
    mode = "whole" if (k // 10) % 2 == 0 else "phases"
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if mode == "whole":
        s.graph_step()
    else:
        pre(); force(); post()
    e1.record()
    torch.cuda.synchronize()
    res[mode].append(e0.elapsed_time(e1))
for m, v in res.items():
    v.sort()
    print(f"{m:7s} median {1e3 * v[len(v) // 2]:.1f} us  mean {1e3 * statistics.mean(v):.1f} us  "
          f"p10 {1e3 * v[len(v) // 10]:.1f}  p90 {1e3 * v[9 * len(v) // 10]:.1f}")
print("rebuilds", int(s.graph_builds.item()) - b0)
