import sys, os
sys.path.insert(0, '/root/repo')
import torch
from paper_1401_4441_b200 import md
s = md.LJSystem.fcc(48, schedule="verlet", skin=0.35)
for _ in range(4):
    s.step()
torch.cuda.synchronize()
print("ok")
