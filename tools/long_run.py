"""Long cfg2 run on the default (Verlet) path: energy drift and capacity checks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1401_4441_b200 import md

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
s = md.LJSystem.fcc(48, schedule="verlet", skin=0.35)
s.kinetic()
pe, ke = s.energies()
e0 = pe + ke
out = s.run(nsteps, energy_every=500)
s.check_status()
rounds, use = s.list_rounds()
counts = np.diff(s.cell_start.cpu().numpy())
print(f"steps {nsteps}  rebuilds {int(s.graph_builds.item())}  E0 {e0:.6f}")
for k, p, q in out:
    print(f"  step {k:6d}  PE {p:.4f}  KE {q:.4f}  T {2 * q / (3 * (s.n - 1)):.4f}  rel dE {(p + q - e0) / abs(e0):+.2e}")
print(f"max rounds {rounds.max()}  lane use {use:.3f}  max particles per cell {counts.max()}")
