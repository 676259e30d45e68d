"""Verlet list build timing for kernel experiments (cfg2, skin 0.35).

usage: python tools/time_build.py [reps]   (CELLSCHED_B200_LIB selects the library)
Times the whole rebuild (wrap, rebin, round tables) with CUDA events; prints list rounds
and pairs, and a force checksum after the build (same list => same forces)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_4441_b200 import md

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
s = md.LJSystem.fcc(48, schedule="verlet", skin=0.35)
for _ in range(3):
    s._rebuild_list()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
for k in range(reps):
    ev[k].record()
    s._rebuild_list()
ev[reps].record()
torch.cuda.synchronize()
t = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(reps))
s.check_status()
rounds, use = s.list_rounds()
s.compute_forces(energy=False, count_pairs=True)
f = torch.stack([s._a("fx"), s._a("fy"), s._a("fz")])
tag = os.path.basename(os.environ.get("CELLSCHED_B200_LIB", "default"))
print(f"{tag:12s} rebuild median {1e3 * t[reps // 2]:8.1f} us  rounds mean {rounds.mean():.3f} max {rounds.max()}  "
      f"lane use {use:.4f}  pairs {s.pair_count()}  |f|sum {float(f.abs().sum()):.12e}")
