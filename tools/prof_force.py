"""Profiling driver: cfg2 system, a few force evaluations (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_4441_b200 import md

sched = sys.argv[1] if len(sys.argv) > 1 else "shell"
nuc = int(sys.argv[2]) if len(sys.argv) > 2 else 48
s = md.LJSystem.fcc(nuc, schedule=sched, skin=0.35)  # (the bench skin)
for _ in range(3):
    for k in ("fx", "fy", "fz"):
        s._a(k).zero_()
    s.compute_forces(energy=False)
torch.cuda.synchronize()
print("pairs", s.pair_count())
if s.verlet:
    rounds, use = s.list_rounds()
    lp = s.list_pairs()
    print("rounds mean %.2f max %d  list pairs %d  lane use %.3f  hits/list %.3f"
          % (rounds.mean(), rounds.max(), lp, use, s.pair_count() / lp))
