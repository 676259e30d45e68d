import sys, time
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_4441_b200 import md, slab
box, nucs, a = md.fcc_box((48, 48, 48), 0.8442)
n = 4 * 48 ** 3
g = md.LJSystem(box, n, schedule="loopex"); g.seed_fcc(nucs, a, 0.722, 0.05, 42)
ini = {k: v[:n] for k, v in g.initial.items()}
c = md.LJBox.for_cutoff(box.lengths, 2.85).cells
vbox = md.LJBox(box.lengths, (c[0] - c[0] % 2,) + tuple(v - v % 4 for v in c[1:]))
lay = slab.SlabLayout(vbox.cells[0], 1, 0)
eng = slab.CudaSlabEngine(vbox, lay, md.LJParams(), schedule="verlet", skin=0.35)
eng.load_global(*(ini[k] for k in ("x", "y", "z", "vx", "vy", "vz", "id")))
st = slab.SlabStep(eng, slab.NeighbourExchanger(lay))
st.start(energy=True)
for _ in range(5): st.step(energy=False, reduce=False)
torch.cuda.synchronize()
import cProfile, pstats
t0 = time.perf_counter()
pr = cProfile.Profile(); pr.enable()
for _ in range(30): st.step(energy=False, reduce=False)
pr.disable()
torch.cuda.synchronize()
print("host ms/step", (time.perf_counter() - t0) / 30 * 1e3, "rebuilds", st.rebuilds)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
