"""Small driver for `compute-sanitizer --tool racecheck`: cfg1 (864 particles,
4^3 cells) force evaluations under every colour-pass schedule (shared-memory
hazards inside the block kernels), plus one Verlet step with a list rebuild.

usage: compute-sanitizer --tool racecheck python tools/racecheck_cfg1.py
"""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1401_4441_b200 import md  # noqa: E402

warnings.simplefilter("ignore")
for sched in ("loopex", "block", "shell", "buffered", "dataflow"):
    s = md.LJSystem.fcc(6, schedule=sched)
    s.step(energy=True)
    print(sched, s.energies(), s.pair_count(), flush=True)
for sched in ("verlet", "verlet_shell", "verlet_dataflow"):
    s = md.LJSystem.fcc(6, schedule=sched, skin=0.35)
    s.step(energy=True)
    s.step(energy=True)
    print(sched, s.energies(), s.pair_count(), s.list_builds, flush=True)
torch.cuda.synchronize()
print("racecheck driver done")
