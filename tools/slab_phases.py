"""x-slab step phases on one GPU (1-rank ring): device time of non-rebuild steps,
rebuild steps and the parts of a rebuild (CUDA events; host waits included)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
for _ in range(5):
    st.step(energy=False, reduce=False)
torch.cuda.synchronize()
T = {"fixed": [], "rebuild": []}
parts = {"wrap+migrate+cells": [], "ghosts+list+forces": []}
orig_rebuild, orig_forces = st._rebuild, st.forces


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize(); parts[name].append(1e3 * (time.perf_counter() - t0))
        return r
    return w


for k in range(60):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r0 = st.rebuilds
    st.step(energy=False, reduce=False)
    torch.cuda.synchronize()
    T["rebuild" if st.rebuilds > r0 else "fixed"].append(1e3 * (time.perf_counter() - t0))
st._rebuild = timed("wrap+migrate+cells", orig_rebuild)
st.forces = timed("ghosts+list+forces", orig_forces)
for k in range(40):
    r0 = st.rebuilds
    st.step(energy=False, reduce=False)
    if st.rebuilds == r0:
        parts["ghosts+list+forces"].pop()
for k, v in T.items():
    if v:
        v.sort(); print(f"{k:8s} steps {len(v):3d}  median {v[len(v) // 2]:.3f} ms  mean {sum(v) / len(v):.3f} ms")
for k, v in parts.items():
    if v:
        print(f"  rebuild part {k:20s} mean {sum(v) / len(v):.3f} ms over {len(v)}")
