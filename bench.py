"""Benchmark of the LJ link-cell hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one velocity-Verlet step of BASELINE configs[1] (cfg2: FCC 48^3 =
442,368 particles, rho 0.8442, T* 0.722, dt 0.005, fp64).  Default schedule
"verlet": kick+drift (+ displacement check), the list rebuild when needed
(wrap, stable counting-sort rebin, round tables -- inside the CUDA graph as a
conditional node), LJ half-shell forces with Newton-3 reaction writes under
the buffered block schedule, kick.  The link-cell kernel (32^3 cells, rebin
every step) is measured on the same workload and reported alongside.
`value` = pair interactions per second (pairs within rc per step x steps/s),
device-timed with CUDA events per step, L2 flushed between steps.
N > 1 (torchrun): each rank advances its own 96^3 FCC block (BASELINE's
weak-scaling config cfg3) of an x-slab-decomposed system ("scaling": "weak");
--config cfg4 runs the strong-scaling config; see DESIGN.md section 7.
`--impl reference` times the CPU port of the reference's own colour-order
execution (oracle/, OpenMP over all host cores) on the same config.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LJ link-cell pair interactions/s (fp64, cfg2 442,368 particles)"
METRIC_CFG5 = "LJ link-cell pair interactions/s (fp64, cfg5 liquid-vapour slab, 3,486,176 particles)"
WORKLOAD_CFG5 = ("cfg5: periodic 64x64x192 cells of edge 2.5 (160x160x480); FCC liquid (rho 0.811, the cubic "
                 "lattice tiling 160 closest to 0.8) in the middle third along z, uniform vapour rho 0.02 "
                 "elsewhere with no pair closer than 0.9; T* 0.85, rc 2.5, dt 0.005, fp64, 1 VV step")
UNIT = "pair-interactions/s"
NUC = 48  # cfg2
# BASELINE configs run on one GPU: FCC cubes (cfg2 headline, cfg3, cfg4) and
# the cfg5 liquid-vapour slab
FCC_CONFIGS = {"cfg2": 48, "cfg3": 96, "cfg4": 192}
WORKLOAD = ("cfg2: LJ fluid FCC 48^3 = 442368 particles, rho* 0.8442, T* 0.722, rc 2.5 (unshifted), "
            "dt 0.005, fp64, 1 VV step; link cells of edge >= rc (32^3) or, for the Verlet schedules, "
            ">= rc + skin (28^3)")


def metric_of(config):
    if config == "cfg5":
        return METRIC_CFG5
    if config == "cfg2":
        return METRIC
    n = 4 * FCC_CONFIGS[config] ** 3
    return f"LJ link-cell pair interactions/s (fp64, {config} {n:,} particles)"


def workload_of(config):
    if config == "cfg5":
        return WORKLOAD_CFG5
    if config == "cfg2":
        return WORKLOAD
    k = FCC_CONFIGS[config]
    return WORKLOAD.replace("cfg2: LJ fluid FCC 48^3 = 442368", f"{config}: LJ fluid FCC {k}^3 = {4 * k ** 3}")


def ncu_fp64_pipe(schedule):
    """FP64 pipe activity (% of peak, ncu) of the schedule's force kernel, from
    the committed capture (profiles/r02_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            t = json.load(f)
        return t["kernels"]["verlet" if schedule.startswith("verlet") else "buffered"].get("fp64_pipe_active_pct")
    except (OSError, KeyError, ValueError):
        return None


def traffic_bytes(schedule):
    """DRAM bytes per force launch of the schedule's kernel, from the committed
    ncu --set full capture (profiles/r02_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            t = json.load(f)
        return t.get("per_schedule", {}).get(schedule, t.get("dram_bytes_per_launch") if schedule == "buffered" else None)
    except (OSError, KeyError, ValueError):
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a while to start: wait for its first sample so
            # that sampling is live when the timed region begins, then keep
            # only the samples taken from here on
            t0 = time.time()
            while not self.rows and time.time() - t0 < 10 and self.proc.poll() is None:
                time.sleep(0.01)
            self.rows.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            t0 = time.time()  # a short timed region: take the next sample as well
            while len(self.rows) < 2 and time.time() - t0 < 0.5 and self.proc.poll() is None:
                time.sleep(0.005)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 3 + k and "Active" in r[3 + k]
                          and "Not" not in r[3 + k]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    return rank, ws


def max_over_ranks(v, ws):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v, ws):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


# --------------------------------------------------------------- CPU arms --
def cpu_setup(nthreads, config="cfg2"):
    import numpy as np

    from oracle import oracle as O

    if config == "cfg5":
        from paper_1401_4441_b200.md import liquid_vapour_positions

        L, xyz = liquid_vapour_positions()
        n = len(xyz)
        vx, vy, vz = O.velocities(n, 0.85, 1.0, 42)
        return O.CpuMD(*(np.ascontiguousarray(xyz[:, k]) for k in range(3)), vx, vy, vz,
                       np.arange(n, dtype=np.int32), [64, 64, 192], list(L), nthreads=nthreads)
    nuc = FCC_CONFIGS[config]
    rho = 0.8442
    a = (4 / rho) ** (1 / 3)
    L = nuc * a
    x, y, z = O.fcc_positions([nuc] * 3, [a] * 3, [L] * 3, 0.05, 42)
    n = len(x)
    vx, vy, vz = O.velocities(n, 0.722, 1.0, 42)
    nc = int(L // 2.5)
    return O.CpuMD(x, y, z, vx, vy, vz, np.arange(n, dtype=np.int32), [nc] * 3, [L] * 3, nthreads=nthreads)


def cpu_sample(nthreads, min_seconds=10.0, max_steps=200, config="cfg2"):
    """Bounded sample: whole steps until >= min_seconds of CPU work."""
    m = cpu_setup(nthreads, config)
    steps, pairs, t0 = 0, 0, time.perf_counter()
    while True:
        _, _, npairs = m.steps(1)
        steps += 1
        pairs += int(npairs[0])
        el = time.perf_counter() - t0
        if el >= min_seconds or steps >= max_steps:
            return pairs / el, steps, el


def cpu_task_replay(config="cfg2"):
    """one LJ force evaluation as an apply_tasks-style replay
    (payload.py:84-119) of the reference's own colour-order stream
    (generate_loopex, taskgen.py:202-234) on ONE host core -- the oracle's C
    restatement.  Returns (pairs/s, seconds)."""
    import numpy as np

    from oracle import oracle as O

    nuc = FCC_CONFIGS[config]
    a = (4 / 0.8442) ** (1 / 3)
    L = nuc * a
    x, y, z = O.fcc_positions([nuc] * 3, [a] * 3, [L] * 3, 0.05, 42)
    nc = [int(L // 2.5)] * 3
    _, start, order = O.bin_cells(x, y, z, np.arange(len(x), dtype=np.int32), nc, [c / L for c in nc])
    xs, ys, zs = (np.ascontiguousarray(v[order]) for v in (x, y, z))
    h, nb, e = O.stream_loopex(nc, (1, 1, 1))
    t0 = time.perf_counter()
    _, _, npair = O.lj_tasks(nc, [L] * 3, start, xs, ys, zs, h, nb, e, O.canonical_stencil(3))
    el = time.perf_counter() - t0
    return npair / el, el


def run_reference(args):
    rank, ws = dist_init()
    if rank != 0:
        return
    import numpy as np

    cores = len(os.sched_getaffinity(0))
    m = cpu_setup(cores, args.config)
    for _ in range(args.warmup):
        m.steps(1)
    times, pairs = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, _, npairs = m.steps(1)
        times.append(time.perf_counter() - t0)
        pairs += int(npairs[0])
    tot = sum(times)
    value = pairs / tot
    line = {
        "impl": "reference", "metric": metric_of(args.config), "value": value,
        "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded FCC + jitter, Gaussian velocities)",
        "config": {"workload": workload_of(args.config) + (
                       f"; the GPU arm at N={ws} runs {ws} such blocks (x-slab weak scaling), the CPU rate "
                       f"is per pair, sampled on one block" if ws > 1 else ""),
                   "schedule": "loop-exchange colour order, 27 levels, OpenMP over tasks of a level",
                   "steps_per_s": args.steps / tot},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(), "kind": "port",
                         "sample": f"{args.steps} whole {args.config} VV steps (oracle/cs_oracle.c o_md_steps)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- GPU --
def fp64_peak(torch, lib):
    """Measured DFMA throughput (TFLOP/s) of this GPU, burst."""
    from paper_1401_4441_b200 import _lib

    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    blocks, iters = 148 * 8, 2000
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("cs_probe_dfma", blocks, iters, _lib.ptr(out), _lib.stream_handle())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = max(best, blocks * 256 * iters * 256 / (ms * 1e-3) / 1e12)
    return best


def run_slab(args, rank, ws):
    """N > 1: x-slab decomposition, halos/migration over NCCL.  Default
    (--config cfg2 not given explicitly): BASELINE's weak-scaling config cfg3
    with one 96^3 FCC block (3,538,944 particles) per GPU along x -- the N = 1
    point of that curve is the `configs.cfg3` entry of the one-GPU line.
    --config cfg3 / cfg4 / cfg5: strong scaling, that configuration's box cut
    into N x-slabs (cfg4 = BASELINE's strong-scaling config)."""
    import torch

    from paper_1401_4441_b200 import _lib, md, slab

    dev = torch.cuda.current_device()
    verlet = args.schedule in md.VERLET_SCHEDULES
    if verlet:
        args.schedule = "verlet"  # buffered block schedule on the rank-local grid
    weak = args.config == "cfg2"
    wk = FCC_CONFIGS["cfg3"] if (weak and not args.slab) else NUC  # per-GPU block edge (unit cells)
    # global initial state (same on every rank), built by the single-domain system
    if args.config == "cfg5":
        g = md.LJSystem.liquid_vapour(schedule="buffered", seed=42)
        box, n = g.box, g.n
        nuc = None
    else:
        nuc = (wk * ws, wk, wk) if weak else (FCC_CONFIGS[args.config],) * 3
        box, nucs, a = md.fcc_box(nuc, 0.8442)
        n = 4 * nucs[0] * nucs[1] * nucs[2]
        g = md.LJSystem(box, n, schedule="loopex")
        g.seed_fcc(nucs, a, 0.722, 0.05, 42)
    ini = {k: v[:n] for k, v in g.initial.items()}
    if verlet:  # cells of edge >= rc + skin (y, z multiples of 4 for the block colouring)
        c = md.LJBox.for_cutoff(box.lengths, 2.5 + args.skin).cells
        box = md.LJBox(box.lengths, (c[0] - c[0] % (2 * ws),) + tuple(v - v % 4 for v in c[1:]))
    lay = slab.SlabLayout(box.cells[0], ws, rank)
    eng = slab.CudaSlabEngine(box, lay, md.LJParams(), schedule=args.schedule, skin=args.skin)
    eng.load_global(ini["x"], ini["y"], ini["z"], ini["vx"], ini["vy"], ini["vz"], ini["id"])
    del g
    torch.cuda.empty_cache()
    st = slab.SlabStep(eng, slab.NeighbourExchanger(lay))
    barrier(ws)
    st.start(energy=True)
    for _ in range(args.warmup):
        st.step()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    p0 = st.pairs_total()
    with ClockSampler(dev) as clk:
        for k in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            barrier(ws)
            ev[k][0].record()
            # pair counts stay on the device; each step but the last launches the
            # next one's kick-drift before waiting for the rebuild decision
            st.step(energy=False, reduce=False, lookahead=k < args.steps - 1)
            ev[k][1].record()
            torch.cuda.synchronize()
    pairs = st.pairs_total() - p0  # summed over ranks
    tot_s = max_over_ranks(sum(e0.elapsed_time(e1) for e0, e1 in ev) * 1e-3, ws)
    # e2e through the public API: this rank's particles (plus a one-plane margin,
    # selected on the host) uploaded from pinned memory, K steps each copying its
    # pair count to pinned host memory, the last one with energies, the owned
    # state downloaded -- all inside the timed region
    import numpy as np

    hx = {k: v.cpu() for k, v in ini.items()}
    nx = box.cells[0]
    plane = np.minimum((hx["x"].numpy() * (nx / box.lengths[0])).astype(np.int64), nx - 1)
    rel = (plane - lay.x0 + 1) % nx  # margin plane on each side
    mine = torch.from_numpy(rel < lay.owned + 2)
    hsel = {k: v[mine].pin_memory() for k, v in hx.items()}
    eng2 = slab.CudaSlabEngine(box, lay, md.LJParams(), schedule=args.schedule, skin=args.skin)
    dx = {k: v.to("cuda") for k, v in hsel.items()}  # a first load allocates the engine's buffers
    eng2.load_global(dx["x"], dx["y"], dx["z"], dx["vx"], dx["vy"], dx["vz"], dx["id"], global_n=n)
    del dx
    res = torch.zeros(args.steps, dtype=torch.int64).pin_memory()
    barrier(ws)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dx = {k: v.to("cuda", non_blocking=True) for k, v in hsel.items()}
    eng2.load_global(dx["x"], dx["y"], dx["z"], dx["vx"], dx["vy"], dx["vz"], dx["id"], global_n=n)
    st2 = slab.SlabStep(eng2, slab.NeighbourExchanger(lay))
    st2.start(energy=True)
    for k in range(args.steps):
        last = k == args.steps - 1
        st2.step(energy=last, reduce=last, lookahead=not last)
        res[k].copy_(eng2.npairs[0], non_blocking=True)
    final = eng2.owned_arrays()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0, ws)
    p2 = int(sum_over_ranks(float(res.sum()), ws))
    clocks = clk.summary()
    if rank != 0:
        return
    workload = (f"{'cfg3' if wk != NUC else 'cfg2'} block per GPU, x-slab weak scaling: FCC {nuc[0]}x{wk}x{wk} "
                f"= {n} particles, " if weak else
                f"{args.config} ({n} particles) cut into {ws} x-slabs (strong scaling): ")
    line = {
        "metric": (metric_of("cfg3") + " per GPU, weak scaling" if weak and wk != NUC else
                   METRIC if weak else metric_of(args.config)), "value": pairs / tot_s, "unit": UNIT,
        "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True,
        "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic (seeded liquid slab + rejection-sampled vapour, Gaussian velocities; BASELINE cfg5)"
                 if args.config == "cfg5" else "synthetic (seeded FCC + 0.05 sigma jitter, Gaussian velocities)"),
        "config": {"workload": workload + f"{box.cells[0]}x{box.cells[1]}x{box.cells[2]} cells, "
                               f"{lay.owned} planes per rank",
                   "schedule": f"{args.schedule} (2, 2, 2) on the rank-local grid"
                               + (f", skin {args.skin}, list rebuilds {st.rebuilds} (all ranks together, "
                                  "migration only at rebuilds)" if verlet else ""),
                   "l2": "flushed (256 MB memset) between timed steps",
                   "parallelism": f"x-slab{ws}: ghost plane + reverse forces + migration over NCCL send/recv",
                   "steps_per_s": args.steps / tot_s},
        "cpu_baseline": None,
        "e2e": {"value": p2 / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 52 * int(mine.sum()) / args.steps,
                "d2h_bytes_per_step": 8 + 80 * eng2.n_owned / args.steps},
        "gpu_launches": args.steps * 40,
        "clocks": clocks,
    }
    del final
    print(json.dumps(line), flush=True)


def measure(torch, md, schedule, args, steps, rank, ws, dev, clocks=True, config=None):
    """Timed run: `steps` VV steps, each replayed as ONE CUDA graph (the
    production path, LJSystem.graph_step), device-timed with CUDA events, L2
    flushed before every step.  Breakdown run: up to 30 more steps replayed as
    three graphs (pre | force | post) with events between the phases, for the
    force-kernel time and the roofline.  Per-step counts stay on the device
    (no host synchronisation inside either loop)."""
    config = config or args.config
    if config == "cfg5":
        sysm = md.LJSystem.liquid_vapour(schedule=schedule, block=args.block, seed=42 + rank, skin=args.skin)
    else:
        sysm = md.LJSystem.fcc(FCC_CONFIGS[config], schedule=schedule, block=args.block, seed=42 + rank,
                               skin=args.skin)
    pre, force, post = sysm.graph_phases()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    for _ in range(args.warmup):
        sysm.graph_step()
    for _ in range(2):
        pre(); force(); post()
    torch.cuda.synchronize()

    def counts(hist, k):
        hist[0, k].copy_(sysm.npairs[0])
        hist[1, k].copy_(sysm.list_pairs_dev() if sysm.verlet else sysm.candidate_pairs_dev())
        if hist.shape[0] > 2:  # SURVEY 8d's C: link-cell candidates on the rc grid
            hist[2, k].copy_(sysm.rc_grid_candidates_dev() if sysm.verlet else hist[1, k])

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
    hist = torch.zeros((2, steps), dtype=torch.int64, device="cuda")
    builds0 = int(sysm.graph_builds.item()) if sysm.verlet else 0
    barrier(ws)
    torch.cuda.synchronize()
    clk = ClockSampler(dev) if clocks else None
    if clk:
        clk.__enter__()
    try:
        for k in range(steps):
            flush.zero_()  # L2 flush between timed steps (outside e[0]..e[1])
            ev[k][0].record()
            sysm.graph_step()
            ev[k][1].record()
            counts(hist, k)
        torch.cuda.synchronize()
    finally:
        if clk:
            clk.__exit__(None, None, None)
    sysm.check_status()
    builds = int(sysm.graph_builds.item()) - builds0 if sysm.verlet else None
    pairs, cands = hist[0].tolist(), hist[1].tolist()
    barrier(ws)
    # breakdown run
    nb = min(steps, 30)
    evb = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(nb)]
    histb = torch.zeros((3, nb), dtype=torch.int64, device="cuda")
    for k in range(nb):
        flush.zero_()
        e = evb[k]
        e[0].record(); pre(); e[1].record(); force(); e[2].record(); post(); e[3].record()
        counts(histb, k)
    torch.cuda.synchronize()
    sysm.check_status()
    pairs_b, cands_b, crc_b = histb[0].tolist(), histb[1].tolist(), histb[2].tolist()
    r = {"sys": sysm, "pairs": pairs, "cands": cands, "builds": builds,
         "step_ms": [e[0].elapsed_time(e[1]) for e in ev],
         "phase_step_ms": [e[0].elapsed_time(e[3]) for e in evb],
         "force_ms": [e[1].elapsed_time(e[2]) for e in evb],
         "pre_ms": [e[0].elapsed_time(e[1]) for e in evb],
         "clocks": clk.summary() if clk else None}
    r["tot_s"] = max_over_ranks(sum(r["step_ms"]) * 1e-3, ws)
    r["value"] = sum_over_ranks(float(sum(pairs)), ws) / r["tot_s"]
    # roofline of the dominant kernel: algorithmic FLOPs 8 C + 20 P with SURVEY
    # 8d's fixed convention C = link-cell half-shell candidates on the rc grid
    # (the same for every schedule); "tested" counts the candidates this
    # schedule actually distance-tests (Verlet: list entries)
    r["achieved"] = sum(8 * c + 20 * p for c, p in zip(crc_b, pairs_b)) / (sum(r["force_ms"]) * 1e-3) / 1e12
    r["achieved_tested"] = sum(8 * c + 20 * p for c, p in zip(cands_b, pairs_b)) / (sum(r["force_ms"]) * 1e-3) / 1e12
    r["crc"] = crc_b
    r["achieved_pairs"] = 20 * sum(pairs_b) / (sum(r["force_ms"]) * 1e-3) / 1e12
    return r


def run_ours(args):
    import torch

    rank, ws = dist_init()
    if ws > 1 or args.slab:
        return run_slab(args, rank, ws)
    from paper_1401_4441_b200 import _lib, md

    dev = torch.cuda.current_device()
    peak_fp64 = fp64_peak(torch, _lib)
    m = measure(torch, md, args.schedule, args, args.steps, rank, ws, dev)
    sysm = m["sys"]
    # the plain link-cell kernel (no Verlet list) on the same workload, for reference
    lc = None
    if sysm.verlet and not args.no_link_cell and args.config == "cfg2":
        ml = measure(torch, md, "buffered", args, min(args.steps, 30), rank, ws, dev, clocks=False)
        lc = {"schedule": "buffered (2, 2, 2), 32^3 cells", "value": ml["value"],
              "ms_per_step": 1e3 * ml["tot_s"] / len(ml["step_ms"]),
              "force_ms_per_step": statistics.mean(ml["force_ms"]),
              "candidates_per_step": statistics.mean(ml["cands"]),
              "roofline_frac": ml["achieved"] / peak_fp64, "steps": len(ml["step_ms"])}
        del ml
    e2e = e2e_run(torch, md, sysm, args)
    colour = None
    if ws == 1 and args.config == "cfg2" and not args.no_variants:
        # the north star's conflict-free colour-ordered schedules on the same
        # workload, each with its own roofline
        colour = {}
        for sched in ("verlet_dataflow", "verlet_shell", "loopex"):
            mv = measure(torch, md, sched, args, min(args.steps, 20), rank, ws, dev, clocks=False)
            colour[sched] = point_summary(mv, peak_fp64)
            colour[sched]["schedule"] = COLOUR_LABELS[sched]
            del mv
            torch.cuda.empty_cache()
    configs = None
    if ws == 1 and args.config == "cfg2" and not args.no_configs:
        # the 1-GPU points of BASELINE's other configurations (cfg3 = the
        # weak-scaling block, cfg4 = the largest single-GPU config, cfg5 = the
        # load-imbalance stress), each with roofline, e2e and clocks
        configs = {}
        for cname, nsteps in (("cfg3", 20), ("cfg4", 10), ("cfg5", 20)):
            mc = measure(torch, md, args.schedule, args, nsteps, rank, ws, dev, config=cname)
            row = point_summary(mc, peak_fp64)
            row.update({"metric": metric_of(cname), "workload": workload_of(cname), "particles": mc["sys"].n,
                        "cells": list(mc["sys"].box.cells), "e2e": e2e_run(torch, md, mc["sys"], args, nsteps),
                        "clocks": mc["clocks"]})
            configs[cname] = row
            del mc
            torch.cuda.empty_cache()
    if rank != 0:
        return
    cpu = None
    if ws == 1 and not args.no_cpu:
        cores = len(os.sched_getaffinity(0))
        v, nst, el = cpu_sample(cores, min_seconds=args.cpu_seconds, config=args.config)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(), "kind": "port",
               "sample": f"{nst} whole {args.config} VV steps in {el:.1f} s (oracle o_md_steps, loop-exchange colour order on OpenMP threads)"}
        if args.config in FCC_CONFIGS and args.config != "cfg4":
            v1, el1 = cpu_task_replay(args.config)
            cpu["single_core_task_replay"] = {
                "value": v1, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": f"one {args.config} force evaluation ({el1:.2f} s): apply_tasks-style replay of the "
                          "reference's generate_loopex stream (oracle o_lj_tasks)"}
    n = sysm.n
    tot_s = m["tot_s"]
    cfg = {"workload": workload_of(args.config), "particles_per_gpu": n, "schedule": f"{args.schedule} {sysm.block}",
           "cells": list(sysm.box.cells),
           "l2": "flushed (256 MB memset) between timed steps",
           "steps_per_s": args.steps / tot_s, "pairs_per_step": statistics.mean(m["pairs"]),
           "candidates_tested_per_step": statistics.mean(m["cands"]),
           "rc_grid_candidates_per_step": statistics.mean(m["crc"]),
           "phase_breakdown": {"steps": len(m["force_ms"]),
                               "note": "separate run with the step split into 3 graphs (pre | force | post)",
                               "ms_per_step": statistics.mean(m["phase_step_ms"]),
                               "force_ms_per_step": statistics.mean(m["force_ms"]),
                               "force_share": sum(m["force_ms"]) / sum(m["phase_step_ms"]),
                               "pre_ms_per_step": statistics.mean(m["pre_ms"]),
                               "pre_ms_median": statistics.median(m["pre_ms"]), "pre_ms_max": max(m["pre_ms"])},
           "parallelism": f"dp{ws}" if ws > 1 else "single"}
    if sysm.verlet:
        cfg.update({"skin": sysm.skin, "list_rebuilds_in_timed_steps": m["builds"],
                    "verlet": "lists built on the device from the cell list (cells of edge >= rc + skin), "
                              "rebuilt inside the timed steps by a conditional CUDA-graph node when a "
                              "particle moved > skin/2; every listed pair re-tested with r^2 < rc^2",
                    "link_cell_kernel": lc})
    line = {
        "metric": metric_of(args.config), "value": m["value"], "unit": UNIT,
        "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic (seeded liquid slab + rejection-sampled vapour, Gaussian velocities; BASELINE cfg5)"
                 if args.config == "cfg5" else
                 f"synthetic (seeded FCC {FCC_CONFIGS[args.config]}^3 + 0.05 sigma jitter, Gaussian velocities; "
                 f"BASELINE {args.config})"),
        "config": cfg,
        "roofline": {"bound": "fp64", "achieved": m["achieved"], "peak": peak_fp64, "unit": "TFLOP/s",
                     "frac": m["achieved"] / peak_fp64, "traffic": traffic_bytes(args.schedule),
                     "kernel": f"k_force_shell ({args.schedule} schedule)",
                     "flops_convention": ("8 C + 20 P per force evaluation (SURVEY 8d); C = link-cell half-shell "
                                          "candidates on the rc grid (fixed per configuration)"),
                     "achieved_tested": m["achieved_tested"], "frac_tested": m["achieved_tested"] / peak_fp64,
                     "tested_note": "same with C = candidates this schedule distance-tests (Verlet list entries)",
                     "achieved_pair_flops": m["achieved_pairs"],
                     "frac_pair_flops": m["achieved_pairs"] / peak_fp64,
                     "peak_source": "measured live: cs_probe_dfma DFMA chains (MEASURED_PEAKS.json has no FP64 entry)",
                     "hbm_peak_gbs": peaks().get("hbm_gbs"),
                     "ncu_fp64_pipe_active_pct": ncu_fp64_pipe(args.schedule),
                     **hbm_side(sysm, statistics.mean(m["force_ms"]), args.schedule)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": args.steps * sysm.launches_per_step()
                        + (m["builds"] or 0) * getattr(sysm, "REBUILD_LAUNCHES", 0),
        "clocks": m["clocks"],
    }
    if colour:
        line["colour_ordered"] = colour
    if configs:
        line["configs"] = configs
    if ws == 1 and args.config == "cfg2" and not args.no_schedule:
        line["schedule_analysis"] = schedule_report(torch, cpu=not args.no_cpu)
    print(json.dumps(line), flush=True)


COLOUR_LABELS = {
    "verlet_dataflow": "Verlet round tables, 2x2x2 block colour order executed as a dataflow (one persistent "
                       "launch; a block waits only for its lower-colour neighbours), 28^3 cells",
    "verlet_shell": "Verlet round tables, 8 colour passes of 2x2x2 blocks (global barrier per colour), 28^3 cells",
    "loopex": "link cells (32^3), the reference's loop-exchange colour order as 27 passes (generate_loopex "
              "levels, one warp per cell-pair task), rebinned every step",
}


def point_summary(m, peak_fp64):
    """Compact record of one measure() run: throughput, step/force time and
    the force kernel's FP64 roofline under both C conventions."""
    sysm = m["sys"]
    return {"value": m["value"], "unit": UNIT, "steps": len(m["step_ms"]),
            "ms_per_step": 1e3 * m["tot_s"] / len(m["step_ms"]),
            "force_ms_per_step": statistics.mean(m["force_ms"]),
            "pairs_per_step": statistics.mean(m["pairs"]),
            "candidates_tested_per_step": statistics.mean(m["cands"]),
            "list_rebuilds_in_timed_steps": m["builds"],
            "roofline": {"bound": "fp64", "unit": "TFLOP/s", "peak": peak_fp64,
                         "achieved": m["achieved"], "frac": m["achieved"] / peak_fp64,
                         "achieved_tested": m["achieved_tested"],
                         "frac_tested": m["achieved_tested"] / peak_fp64},
            "skin": sysm.skin if sysm.verlet else None}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def hbm_side(sysm, force_ms, schedule):
    """The HBM side of the force kernel's roofline: algorithmic bytes per
    evaluation (48 B/particle: x, y, z in, f out; Verlet adds the round-table
    descriptors, 64 B per round) and the ncu DRAM traffic, over the measured
    force-phase time (kernel + buffered gather), against the measured HBM peak."""
    nbytes = 48 * sysm.n
    if sysm.verlet:
        rounds, _ = sysm.list_rounds()
        nbytes += 64 * int(rounds.sum())
    hbm = peaks().get("hbm_gbs")
    out = {"hbm_algorithmic_bytes": nbytes, "hbm_achieved_gbs": nbytes / (force_ms * 1e-3) / 1e9}
    tr = traffic_bytes(schedule)
    if tr:
        out["hbm_traffic_gbs"] = tr / (force_ms * 1e-3) / 1e9
    if hbm:
        out["hbm_frac"] = out["hbm_achieved_gbs"] / hbm
    return out


SCHED_GRIDS = {"cfg1": (4, 4, 4), "cfg5": (64, 64, 192)}
SCHED_ORDERS = (("lexicographic", "basic", 2), ("colour 2x2x2", "loopex", 2), ("colour 3x3x3", "loopex", 3))


def schedule_report(torch, cpu=True):
    """BASELINE cfg1/cfg5 serialization analysis (K4): generate the task
    stream, detect its inout dependencies and take the critical path, all on
    the device -- the reference pipeline generate -> detect_dependencies ->
    critical_path (taskgen.py:180-234, depgraph.py:102-174).  Device wall time
    per order (after one warm-up) next to the oracle's C port of the same
    pipeline on one host core."""
    from paper_1401_4441_b200 import GridSpec, schedule

    out = {}
    for cname, ext in SCHED_GRIDS.items():
        g = GridSpec(ext)
        rows = {}
        for label, strat, stride in SCHED_ORDERS:
            if cname == "cfg1" and stride == 3:
                continue  # (4 is not a multiple of 3)
            schedule.device_stream(g, strat, stride=stride).depth()  # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ds = schedule.device_stream(g, strat, stride=stride)
            ne = ds.edges()[2]
            d = ds.depth()
            torch.cuda.synchronize()
            t_dev = time.perf_counter() - t0
            row = {"tasks": ds.ntasks, "edges": ne, "depth": d,
                   "degree_of_serialization": ds.ntasks / d, "device_ms": 1e3 * t_dev}
            del ds
            if cpu:
                from oracle import oracle as O
                from paper_1401_4441_b200.taskgen import StencilOrder
                t0 = time.perf_counter()
                if strat == "basic":
                    h, nb, _ = O.stream_basic(ext, (1, 1, 1), StencilOrder.canonical(3).offsets)
                else:
                    h, nb, _ = O.stream_loopex(ext, (1, 1, 1), stride)
                eu, ev = O.detect_edges_stream(h, nb)
                dc = O.critical_path(len(h), eu, ev)
                row["cpu_port_ms"] = 1e3 * (time.perf_counter() - t0)
                row["cpu_port_depth"] = int(dc)
                del h, nb, eu, ev
            rows[label] = row
        out[cname] = {"grid": list(ext), "orders": rows}
    out["note"] = ("device: stream generation + edge detection + critical path (wall clock incl. "
                   "allocations); cpu_port: oracle/cs_oracle.c restatement of the same pipeline, 1 core")
    out["payload"] = payload_report(torch, cpu)
    if cpu:
        try:
            out["reference_python"] = reference_python_report(torch)
        except Exception as exc:  # the reference arm must not sink the bench line
            out["reference_python"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
    return out


def reference_python_report(torch):
    """the UNMODIFIED reference package, installed
    into baseline/_ref (pip, from a copy of /root/reference/pkg), timed on the
    box's host: generate -> detect_dependencies -> critical_path
    (taskgen.py:180-234, depgraph.py:102-174) on the cfg1 grid and on 32^3,
    executor.execute (executor.py:287-354) with W = all host cores on the
    colour-order stream with the integer payload, and simulate /
    simulate_dynamic (schedsim.py:63-163) on the paper's 30x10x10 domain;
    beside each, the same pipeline / execution / schedule on the device."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "cellsched")):
        return {"unavailable": "baseline/_ref not installed (pip install of /root/reference/pkg)"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import numpy as np

    import cellsched as R
    from cellsched import executor as RX

    from paper_1401_4441_b200 import GridSpec, generic, schedule, taskgen

    cores = len(os.sched_getaffinity(0))
    out = {"package": f"cellsched {R.__version__} (baseline/_ref)", "cores": cores, "cpu_model": cpu_model(),
           "pipeline": {}, "executor": {}}
    for gname, ext in (("cfg1", (4, 4, 4)), ("32^3", (32, 32, 32))):
        g = R.GridSpec(ext)
        rows = {}
        for label, strat in (("lexicographic", "basic"), ("colour 2x2x2", "loopex")):
            t0 = time.perf_counter()
            tasks = (R.generate_basic(g, R.StencilOrder.canonical(3)) if strat == "basic"
                     else R.generate_loopex(g))
            t1 = time.perf_counter()
            graph = R.detect_dependencies(tasks)
            t2 = time.perf_counter()
            depth = R.critical_path(graph)
            t3 = time.perf_counter()
            schedule.device_stream(GridSpec(ext), strat).depth()  # warm-up
            torch.cuda.synchronize()
            d0 = time.perf_counter()
            ds = schedule.device_stream(GridSpec(ext), strat)
            ds.edges()
            ddev = ds.depth()
            torch.cuda.synchronize()
            d1 = time.perf_counter()
            rows[label] = {"tasks": len(tasks), "depth": depth, "generate_s": t1 - t0, "detect_s": t2 - t1,
                           "critical_path_s": t3 - t2, "total_s": t3 - t0, "device_ms": 1e3 * (d1 - d0),
                           "device_depth": ddev, "speedup": (t3 - t0) / (d1 - d0)}
            del tasks, graph, ds
        out["pipeline"][gname] = rows
    for gname, ext in (("cfg1", (4, 4, 4)), ("16^3", (16, 16, 16))):
        g = R.GridSpec(ext)
        graph = R.detect_dependencies(R.generate_loopex(g))
        res = RX.execute(graph, RX.ExecConfig(cores, 0, payload_seed=42), g)
        mine = taskgen.generate_loopex(GridSpec(ext))
        generic.execute_dag(mine, GridSpec(ext), 42)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        acc, conflicts = generic.execute_dag(mine, GridSpec(ext), 42)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out["executor"][gname] = {
            "tasks": graph.task_count, "threads": cores, "wall_s": res.wall_ns * 1e-9,
            "tasks_per_s": graph.task_count / (res.wall_ns * 1e-9),
            "device_dag_execute_s": dt, "device_tasks_per_s": graph.task_count / dt,
            "device_note": "wall clock incl. host interning of the Task objects and edge detection",
            "device_conflicts": conflicts,
            "accumulators_equal": res.accumulators == acc}
    # the worker-pool model (schedsim.py:63-163) on the paper's 3D domain: the
    # reference's simulate / simulate_dynamic vs the device list scheduler
    from cellsched import schedsim as RS
    from paper_1401_4441_b200 import depgraph as MD, schedsim as MS

    g = R.GridSpec((30, 10, 10))
    rg = R.detect_dependencies(R.generate_basic(g, R.order_with_displacement(3, 1)))
    mg = MD.detect_dependencies(taskgen.generate_basic(GridSpec((30, 10, 10)), taskgen.order_with_displacement(3, 1)))
    sim = {}
    for W in (8, 16):
        t0 = time.perf_counter()
        rr = RS.simulate(rg, RS.SimConfig(W))
        t1 = time.perf_counter()
        MS.simulate(mg, MS.SimConfig(W))  # warm-up
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        e = np.asarray(mg.edges, np.int64)
        start, mk = MS.simulate_edges(mg.task_count, e[:, 0], e[:, 1], W)
        t3 = time.perf_counter()
        sim[f"delta1_W{W}"] = {"tasks": rg.task_count, "makespan": rr.makespan, "device_makespan": mk,
                               "speedup": rr.speedup, "reference_s": t1 - t0, "device_ms": 1e3 * (t3 - t2)}
    plan_r, plan_m = R.NestedPlan(g), taskgen.NestedPlan(GridSpec((30, 10, 10)))
    t0 = time.perf_counter()
    rn = RS.simulate_dynamic(plan_r, RS.SimConfig(32))
    t1 = time.perf_counter()
    MS.nested_device(plan_m, 32)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    _, mkn = MS.nested_device(plan_m, 32)
    t3 = time.perf_counter()
    sim["nested_W32"] = {"tasks": len(rn.graph.tasks), "makespan": rn.makespan, "device_makespan": mkn,
                         "speedup": rn.speedup, "reference_s": t1 - t0, "device_ms": 1e3 * (t3 - t2)}
    out["simulate"] = sim
    out["note"] = ("reference Python, single process (the executor's worker threads share the GIL); "
                   "device = this package's stream generator + detector + depth (wall clock incl. allocations) "
                   "and its ready-queue DAG runtime (cs_dag_execute) with the same payload")
    return out


def payload_report(torch, cpu=True, ext=(64, 64, 192), seed=42):
    """The reference's own hot loop, the integer payload (apply_tasks /
    reference_oracle, payload.py:84-174), on the cfg5 grid: the colour-order
    stream executed on the device level by level and as the LJ kernel's 27
    colour passes, and the direct full-neighbourhood sum; the oracle's C port
    of apply_tasks / reference_oracle on one host core; bit-exact check."""
    import numpy as np

    from paper_1401_4441_b200 import GridSpec, payload, schedule

    g = GridSpec(ext)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        return r, 1e3 * (time.perf_counter() - t0)

    ds = schedule.device_stream(g, "loopex")
    ds.levels()
    acc_lv, t_lv = timed(lambda: payload.apply_stream_device(ds, seed))
    acc_cp, t_cp = timed(lambda: payload.colour_pass_payload(g, seed, "loopex", race_check=False))
    acc_dir, t_dir = timed(lambda: payload.reference_oracle_device(g, seed))
    row = {"grid": list(ext), "tasks": ds.ntasks, "device_levels_ms": t_lv, "device_colour_passes_ms": t_cp,
           "device_direct_ms": t_dir,
           "device_equal": bool(torch.equal(acc_lv, acc_cp) and torch.equal(acc_lv, acc_dir))}
    if cpu:
        from oracle import oracle as O

        h, nb, e = ds.home.cpu().numpy(), ds.nbr.cpu().numpy(), ds.entry.cpu().numpy()
        t0 = time.perf_counter()
        ref = O.payload_apply(ext, (1, 1, 1), seed, h, nb, e, np.array(ds.entries, np.int8))
        row["cpu_port_apply_tasks_ms"] = 1e3 * (time.perf_counter() - t0)
        t0 = time.perf_counter()
        ref2 = O.payload_reference(ext, (1, 1, 1), seed)
        row["cpu_port_reference_oracle_ms"] = 1e3 * (time.perf_counter() - t0)
        row["bit_exact_vs_cpu_port"] = bool(np.array_equal(acc_lv.cpu().numpy(), ref)
                                            and np.array_equal(ref, ref2))
    row["note"] = ("reference Python apply_tasks: 10-14 us/task standalone (SURVEY 8a a14, survey "
                   "container), i.e. about 2 min for these tasks")
    return row


def e2e_run(torch, md, ref_sys, args, steps=None):
    """Same metric through the public API from pinned host buffers: upload the
    state, K graph-replayed steps each reading back (PE, KE), download the
    final state -- all inside the timed region."""
    n = ref_sys.n
    steps = steps or args.steps
    host = {k: v[:n].cpu().pin_memory() for k, v in ref_sys.initial.items()}
    sysm = md.LJSystem(ref_sys.box, n, schedule=ref_sys.schedule, block=ref_sys.block, skin=ref_sys.skin)
    sysm.load_host(host["x"], host["y"], host["z"], host["vx"], host["vy"], host["vz"], host["id"])
    for e in (True, True, False, False):  # capture the step graphs (both parities) outside the timing
        sysm.graph_step(energy=e)
    torch.cuda.synchronize()
    out = torch.empty((6, n), dtype=torch.float64).pin_memory()
    res = torch.zeros(steps, dtype=torch.int64).pin_memory()
    # the pinned result buffers are reused host memory: fault their pages in
    # once before the timed region (a first DMA into fresh pinned pages cost
    # ~3.5 ms for these 21 MB on the box)
    b = sysm._buf[sysm.cur]
    for i, k in enumerate(("x", "y", "z", "vx", "vy", "vz")):
        out[i].copy_(b[k][:n], non_blocking=True)
    res.copy_(sysm.npairs[0].expand(steps), non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sysm.load_host(host["x"], host["y"], host["z"], host["vx"], host["vy"], host["vz"], host["id"])
    pairs = 0
    for k in range(steps):
        sysm.graph_step(energy=k == steps - 1)  # the last step also reports the energies
        # the step's result (its pair count, the metric) goes to the host every
        # step, asynchronously into its own pinned slot: the host never waits
        res[k].copy_(sysm.npairs[0], non_blocking=True)
    pe, ke, _ = sysm.readout()
    pairs = int(res.sum())
    b = sysm._buf[sysm.cur]
    for i, k in enumerate(("x", "y", "z", "vx", "vy", "vz")):
        out[i].copy_(b[k][:n], non_blocking=True)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    h2d = 52 * n
    d2h = 8 * steps + 80 + 48 * n
    return {"value": pairs / el, "unit": UNIT, "h2d_bytes_per_step": h2d / steps,
            "d2h_bytes_per_step": d2h / steps,
            "timed": ("host wall clock: H2D of the initial state (incl. its cell list, Verlet list and "
                      "forces), K graph-replayed steps each copying its pair count to pinned host memory "
                      "(async D2H per step), the last one with energies read back, D2H of the final state")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-link-cell", action="store_true", help="skip the link-cell comparison run")
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3", "cfg4", "cfg5"],
                    help="BASELINE workload on one GPU: cfg2 (headline), cfg3 (96^3 FCC), cfg4 (192^3 FCC), "
                         "cfg5 (liquid-vapour load-imbalance stress)")
    ap.add_argument("--schedule", default="verlet",
                    choices=["shell", "buffered", "dataflow", "block", "loopex", "verlet", "verlet_shell",
                             "verlet_dataflow"])
    ap.add_argument("--skin", type=float, default=0.35, help="Verlet skin (verlet schedules)")
    ap.add_argument("--block", type=lambda s: tuple(int(v) for v in s.split(",")), default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the colour-ordered schedule runs")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg3/cfg4/cfg5 one-GPU points")
    ap.add_argument("--no-schedule", action="store_true", help="skip the cfg1/cfg5 serialization analysis")
    ap.add_argument("--slab", action="store_true", help="use the x-slab engine even at N=1")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
