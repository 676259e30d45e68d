"""Profiling driver: cfg2 Verlet system stepped eagerly (host-decided
rebuilds), so every kernel of the step is visible to ncu's launch list
(kernels inside graphs that contain a conditional node are not replayed)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_4441_b200 import md

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
config = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
if config == "cfg5":
    s = md.LJSystem.liquid_vapour(schedule="verlet", seed=42, skin=0.35)
else:
    s = md.LJSystem.fcc(48, schedule="verlet", skin=0.35)
for _ in range(nsteps):
    s.step()
torch.cuda.synchronize()
print("steps", nsteps, "list builds", s.list_builds)
