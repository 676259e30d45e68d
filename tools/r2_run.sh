cd $GRAFT_REPO_ROOT
timeout 600 python -c "
import sys, time, torch, numpy as np; sys.path.insert(0,'.')
from paper_1401_4441_b200 import depgraph, schedsim, taskgen, GridSpec
g = GridSpec((30,10,10))
t0=time.perf_counter(); mg = depgraph.detect_dependencies(taskgen.generate_basic(g, taskgen.order_with_displacement(3,1))); t1=time.perf_counter()
print('graph build s', t1-t0)
e = np.asarray(mg.edges, np.int64)
for W in (8, 16, 42000):
    for rep in range(3):
        torch.cuda.synchronize(); t0=time.perf_counter()
        st, mk = schedsim.simulate_edges(mg.task_count, e[:,0], e[:,1], W)
        t1=time.perf_counter()
        print(W, mk, 'ms', 1e3*(t1-t0))
" > gpurun_out/r2_sim2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum -k regex:k_ls python -c "
import sys, torch, numpy as np; sys.path.insert(0,'.')
from paper_1401_4441_b200 import depgraph, schedsim, taskgen, GridSpec
g = GridSpec((30,10,10))
mg = depgraph.detect_dependencies(taskgen.generate_basic(g, taskgen.order_with_displacement(3,1)))
e = np.asarray(mg.edges, np.int64)
schedsim.simulate_edges(mg.task_count, e[:,0], e[:,1], 8)
" >> gpurun_out/r2_sim2.log 2>&1
