"""Where the e2e time of bench.py goes (cfg2, verlet): host wall clock of each part."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1401_4441_b200 import md

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ref = md.LJSystem.fcc(48, schedule="verlet", skin=0.35)
n = ref.n
host = {k: v[:n].cpu().pin_memory() for k, v in ref.initial.items()}
s = md.LJSystem(ref.box, n, schedule="verlet", skin=ref.skin)
s.load_host(host["x"], host["y"], host["z"], host["vx"], host["vy"], host["vz"], host["id"])
for e in (True, True, False, False):
    s.graph_step(energy=e)
torch.cuda.synchronize()
out = torch.empty((6, n), dtype=torch.float64).pin_memory()
res = torch.zeros(steps, dtype=torch.int64).pin_memory()
for rep in range(3):
    T = [time.perf_counter()]
    s.load_host(host["x"], host["y"], host["z"], host["vx"], host["vy"], host["vz"], host["id"])
    T.append(time.perf_counter()); torch.cuda.synchronize(); T.append(time.perf_counter())
    for k in range(steps):
        s.graph_step(energy=k == steps - 1)
        res[k].copy_(s.npairs[0], non_blocking=True)
    T.append(time.perf_counter()); torch.cuda.synchronize(); T.append(time.perf_counter())
    pe, ke, _ = s.readout()
    T.append(time.perf_counter())
    b = s._buf[s.cur]
    for i, key in enumerate(("x", "y", "z", "vx", "vy", "vz")):
        out[i].copy_(b[key][:n], non_blocking=True)
    torch.cuda.synchronize(); T.append(time.perf_counter())
    d = [1e3 * (T[i + 1] - T[i]) for i in range(len(T) - 1)]
    print("load issue %.2f | load finish %.2f | steps issue %.2f | steps finish %.2f | readout %.2f | D2H %.2f | total %.2f ms"
          % (*d, 1e3 * (T[-1] - T[0])))
