"""Force-evaluation timing for kernel experiments (cfg2, Verlet or link-cell).

usage: python tools/time_force.py [schedule] [reps]   (CELLSCHED_B200_LIB selects the library)
Prints per-evaluation times (CUDA events, the system's stream) and a force checksum.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_4441_b200 import md

sched = sys.argv[1] if len(sys.argv) > 1 else "verlet"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = os.environ.get("CFG", "cfg2")
if cfg == "cfg5":
    s = md.LJSystem.liquid_vapour(schedule=sched, seed=42, skin=0.35)
else:
    s = md.LJSystem.fcc(48, schedule=sched, skin=0.35)
st = torch.cuda.current_stream()
for _ in range(5):
    s.compute_forces(energy=False, count_pairs=True)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
for k in range(reps):
    ev[k].record()
    s.compute_forces(energy=False, count_pairs=True)
ev[reps].record()
torch.cuda.synchronize()
t = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(reps))
s.check_status()
f = torch.stack([s._a("fx"), s._a("fy"), s._a("fz")])
tag = os.path.basename(os.environ.get("CELLSCHED_B200_LIB", "default"))
print(f"{tag:28s} {cfg} {sched}: median {1e3 * t[reps // 2]:8.1f} us  min {1e3 * t[0]:8.1f} us  "
      f"|f|sum {float(f.abs().sum()):.12e}  pairs {s.pair_count()}")
