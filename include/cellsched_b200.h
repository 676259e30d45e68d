/*
 * cellsched_b200.h -- C ABI of the B200-native link-cell LJ hot path.
 *
 * Drop-in boundary for the reference package `cellsched`
 * (/root/reference/pkg/src/cellsched).  The reference is pure Python with no
 * FFI; these entry points are what its Python API binds through ctypes
 * (see INTEGRATION.md).  Each declaration names the reference interface it
 * replaces (file:line).  Functions the reference lacks (particles, LJ,
 * integration -- SPEC.md:12, :462, :472) extend its idiom at the payload
 * plug-in point (payload.py:84-174).
 *
 * Conventions
 *  - return 0 on success, a cudaError_t (>0) or a negative CS_E* code on
 *    failure; cs_last_error() returns a message for the calling thread.
 *  - all array arguments are DEVICE pointers owned by the caller (e.g.
 *    torch tensors' data_ptr()), except where a parameter says "host".
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *    calls are stream-ordered and never synchronise unless documented.
 *  - temporary memory comes from a caller workspace `ws` of `ws_bytes`;
 *    the matching *_ws_bytes() query returns the size needed.
 *  - cell ids are x-fastest: c = x + ex*(y + ey*z)  (grid.py:3-4, :93-101).
 */
#ifndef CELLSCHED_B200_H
#define CELLSCHED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_OK 0
#define CS_EINVAL (-1)     /* bad argument (reference raises ValueError)        */
#define CS_ECAPACITY (-2)  /* workspace / cell capacity exceeded               */
#define CS_ECONFLICT (-3)  /* race detector: two writers of one cell in a pass */
#define CS_ERANGE (-4)     /* particle outside the local cell range            */
#define CS_ECYCLE (-5)     /* non-forward edge (depgraph.py:170-171)           */

/* Grid of cells: dim 2 or 3, extents, per-axis periodicity
 * (GridSpec, grid.py:43-101; per-axis periodicity generalises the single
 * flag so an x-slab can be open in x). */
typedef struct cs_grid {
  int32_t dim;
  int32_t ext[3];
  int32_t periodic[3];
} cs_grid;

int cs_abi_version(void);
const char *cs_last_error(void);
int cs_device_synchronize(void);
/* stream-ordered byte fill of device memory (cudaMemsetAsync; a memset node
 * when captured): clears per-step result words without framework kernels */
int cs_memset_async(void *dst, int value, size_t bytes, void *stream);
/* stream-ordered device-to-device copy (a memcpy node when captured) */
int cs_copy_async(void *dst, const void *src, size_t bytes, void *stream);
/* *acc += *x on the stream: device-side running totals (pair counts) */
int cs_accumulate_i64(int64_t *acc, const int64_t *x, void *stream);

/* ===================== K4: task streams and serialization depth ========== */
enum { CS_STREAM_BASIC = 0, CS_STREAM_LOOPEX = 1 };

/* Number of tasks of a stream (host only, closed form).  basic: order is a
 * host array of n offsets x dim int8 (StencilOrder.offsets); loopex: order
 * ignored, canonical stencil, colour stride `stride` (2 = reference).
 * Replaces len(generate_basic(...)) / len(generate_loopex(...))
 * (taskgen.py:180-234). */
int64_t cs_stream_count(const cs_grid *g, int strategy, const int8_t *order_host, int n,
                        int stride);

/* Generate a stream as arrays: home[t], nbr[t] (-1 for intra) and entry[t]
 * (index into the order / canonical stencil), t in creation order.
 * Replaces generate_basic (taskgen.py:180-199) and generate_loopex
 * (taskgen.py:202-234); truncated non-periodic tasks are dropped
 * (taskgen.py:195-197). */
size_t cs_stream_ws_bytes(const cs_grid *g, int n);
int cs_stream_generate(const cs_grid *g, int strategy, const int8_t *order_host, int n,
                       int stride, int32_t *home, int32_t *nbr, int16_t *entry, int64_t ntasks,
                       void *ws, size_t ws_bytes, void *stream);

/* Dependency edges of an accumulator stream (every task writes acc(home)
 * and acc(nbr)).  Writes pred_a[t], pred_b[t] (-1 = none; pred_a < pred_b
 * when both exist, duplicates collapsed) -- the (succ, pred)-sorted edge
 * list of detect_dependencies (depgraph.py:102-117, rule :28-49).
 * `order_host`/`n`/`strategy`/`stride` must be the ones the stream was
 * generated with (the accessor sets are closed-form).  Synchronises; writes
 * the edge count to *nedges_host. */
size_t cs_edges_ws_bytes(const cs_grid *g, int n, int64_t ntasks);
int cs_stream_edges(const cs_grid *g, int strategy, const int8_t *order_host, int n, int stride,
                    const int32_t *home, const int32_t *nbr, int64_t ntasks, int32_t *pred_a,
                    int32_t *pred_b, int64_t *nedges_host, void *ws, size_t ws_bytes,
                    void *stream);

/* Compact (pred_a, pred_b) into edge arrays eu/ev sorted by (succ, pred). */
int cs_edges_compact(int64_t ntasks, const int32_t *pred_a, const int32_t *pred_b, int64_t *eu,
                     int64_t *ev, void *ws, size_t ws_bytes, void *stream);

/* Serialization depth = critical_path (depgraph.py:160-174) and per-task
 * level (longest path ending at t, counted in tasks).  method 0 = level
 * relaxation (shallow orders), 1 = cell-chain DP (cell-grouped streams,
 * e.g. generate_basic), 2 = auto.  Synchronises; *depth_host gets the depth. */
size_t cs_depth_ws_bytes(int64_t ntasks);
int cs_stream_depth(const cs_grid *g, int strategy, int n, int64_t ntasks, const int32_t *home,
                    const int32_t *nbr, const int32_t *pred_a, const int32_t *pred_b,
                    int32_t *level, int method, int64_t *depth_host, void *ws, size_t ws_bytes,
                    void *stream);

/* Generic task lists (any resources, read-only inputs): detect_dependencies
 * with the full _DependenceState rule (depgraph.py:28-49).  Accesses in
 * stream order (task-major; a task's reads before its writes; reads of a
 * resource the task also writes dropped), tptr[ntasks+1] = access ranges.
 * Pass 1 returns the edge count (synchronises); pass 2, called next with
 * the same workspace, writes eu/ev sorted by (succ, pred).  npred_max bounds
 * the raw predecessor total (2 * nacc is always enough). */
size_t cs_detect_ws_bytes(int64_t ntasks, int64_t nacc, int64_t npred_max);
int cs_detect_generic(int64_t ntasks, int64_t nacc, int64_t nres, const int64_t *tptr,
                      const int32_t *acc_task, const int32_t *acc_res, const uint8_t *acc_write,
                      int64_t npred_max, int64_t *nedges_host, void *ws, size_t ws_bytes,
                      void *stream);
int cs_detect_generic_emit(int64_t ntasks, int64_t nacc, const int64_t *tptr, int64_t npred_max,
                           int64_t *eu, int64_t *ev, void *ws, size_t ws_bytes, void *stream);
/* critical_path of any forward edge list sorted by succ (depgraph.py:160-174);
 * CS_ECYCLE on a non-forward edge (depgraph.py:170-171).  Synchronises. */
size_t cs_longest_path_ws_bytes(int64_t ntasks);
int cs_longest_path(int64_t ntasks, int64_t nedges, const int64_t *eu, const int64_t *ev,
                    int32_t *level, int64_t *depth_host, void *ws, size_t ws_bytes, void *stream);

/* ===================== K5: integer payload (parity harness) ============== */
/* charges (payload.py:58-61): q[cell] */
int cs_payload_charges(const cs_grid *g, int64_t seed, int64_t *q, void *stream);
/* reference_oracle analogue (payload.py:152-174): direct 3^dim-1 sum */
int cs_payload_direct(const cs_grid *g, int64_t seed, const int64_t *q, int64_t *acc,
                      void *stream);
/* apply_tasks analogue (payload.py:84-119): execute a stream level by level
 * (tasks of one dependency level are write-disjoint), no atomics.
 * `level` from cs_stream_depth; entry_offsets_host = n x dim int8. */
size_t cs_payload_levels_ws_bytes(int64_t ntasks, int64_t depth);
int cs_payload_levels(const cs_grid *g, const int64_t *q, int64_t ntasks, const int32_t *home,
                      const int32_t *nbr, const int16_t *entry, const int8_t *entry_offsets_host,
                      int n, const int32_t *level, int64_t depth, int64_t *acc, void *ws,
                      size_t ws_bytes, void *stream);
/* apply_tasks for any task list (payload.py:84-119): kind 0 intra (val[w0] +=
 * intra), 1 inter (val[w0] += g, val[w1] -= g; accumulator or buffer slots),
 * 2 reduce (val[w0] += sum val[reads]); executed level by level. */
size_t cs_payload_generic_ws_bytes(int64_t ntasks, int64_t depth);
int cs_payload_generic(int64_t ntasks, int dim, const int8_t *kind, const int32_t *home,
                       const int32_t *nbr, const int32_t *w0, const int32_t *w1, const int8_t *off,
                       const int64_t *rptr, const int32_t *rres, const int64_t *q,
                       const int32_t *level, int64_t depth, int64_t nres, int64_t *val, void *ws,
                       size_t ws_bytes, void *stream);
/* Device dependency-driven runtime: run the generic payload
 * tasks (arguments as cs_payload_generic) in dependency order with a ready
 * queue and indegree counters -- no level barriers.  Edges sorted by
 * predecessor: successors of t are succ[sptr[t] .. sptr[t+1]), ev = the
 * successor of every edge (nedges).  race_check != 0 counts write conflicts
 * between concurrently running tasks into conflicts_dev[0] (executor
 * exclusion contract).  CS_ECYCLE if a task is never released. */
size_t cs_dag_ws_bytes(int64_t ntasks, int64_t nres);
int cs_dag_execute(int64_t ntasks, int dim, const int8_t *kind, const int32_t *home,
                   const int32_t *nbr, const int32_t *w0, const int32_t *w1, const int8_t *off,
                   const int64_t *rptr, const int32_t *rres, const int64_t *q, int64_t nedges,
                   const int64_t *sptr, const int64_t *succ, const int64_t *ev, int64_t nres,
                   int64_t *val, int race_check, unsigned long long *conflicts_dev, void *ws,
                   size_t ws_bytes, void *stream);

/* The colour-pass schedules of the LJ kernel, run on the integer payload:
 * sched CS_SCHED_LOOPEX (27 passes) or CS_SCHED_BLOCK (8 block passes).
 * race_check != 0 records writers per pass and fails with CS_ECONFLICT. */
int cs_payload_colour(const cs_grid *g, int sched, const int32_t *block_host, const int64_t *q,
                      int64_t *acc, int race_check, void *ws, size_t ws_bytes, void *stream);
size_t cs_payload_colour_ws_bytes(const cs_grid *g);

/* ===================== LJ link-cell MD (new; extends the payload plug-in) */
enum { CS_SCHED_LOOPEX = 0, CS_SCHED_BLOCK = 1, CS_SCHED_SHELL = 2, CS_SCHED_BUFFERED = 3,
       CS_SCHED_DATAFLOW = 4 };

/* Local cell box.  Single GPU: nc == gnc, x0 == 0, periodic {1,1,1}.
 * x-slab rank: nc[0] = owned planes + 1 ghost plane, periodic[0] = 0,
 * x0 = global index of local plane 0.  inv = gnc / L (binning), L = box. */
typedef struct cs_box {
  int32_t nc[3];
  int32_t gnc[3];
  int32_t x0;
  int32_t owned_x; /* planes whose cells own home tasks (nc[0]-1 in slab mode) */
  int32_t periodic[3];
  int32_t block[3]; /* CS_SCHED_BLOCK block shape in cells */
  double L[3];
  double inv[3];
} cs_box;

typedef struct cs_lj {
  double eps, sigma, rc, mass;
} cs_lj;

/* FCC lattice + seeded jitter, id order (4 sites per unit cell). */
int cs_init_fcc(const int32_t *nuc_host, const double *a_host, const double *L_host,
                double jitter, int64_t seed, double *x, double *y, double *z, int32_t *id,
                void *stream);
/* Gaussian velocities, momentum removed, scaled to exactly T (3N-3 dof). */
size_t cs_reduce_ws_bytes(int64_t n);
int cs_init_velocities(int64_t n, double T, double mass, int64_t seed, double *vx, double *vy,
                       double *vz, void *ws, size_t ws_bytes, void *stream);

/* K1: cell list as a stable counting sort (histogram, scan, scatter, then
 * canonical id order within each cell).  Gathers x, v, id into the
 * cell-sorted outputs, zeroes f_out, writes cell_start[ncells+1].
 * v pointers may be NULL (positions only). */
size_t cs_bin_ws_bytes(int64_t n, const cs_box *b);
int cs_build_cells(int64_t n, const cs_box *b, const double *x, const double *y,
                   const double *z, const double *vx, const double *vy, const double *vz,
                   const int32_t *id, double *xo, double *yo, double *zo, double *vxo,
                   double *vyo, double *vzo, int32_t *ido, double *fxo, double *fyo,
                   double *fzo, int32_t *cell_start, void *ws, size_t ws_bytes, void *stream);
/* Range flag of the last cs_build_cells on workspace `ws` (same n, box):
 * *flag_host = 1 if a particle lay outside the local cell range and was
 * clamped into an edge cell (slab: a particle that should have migrated).
 * Synchronises. */
int cs_bin_errors(int64_t n, const cs_box *b, const void *ws, size_t ws_bytes, int *flag_host,
                  void *stream);

/* K2: fp64 LJ half-shell forces with Newton-3 reaction writes under a
 * conflict-free schedule; f must be zeroed by the caller (cs_build_cells
 * does).  n = particles in the cell arrays.  energy_dev[0] += PE,
 * npairs_dev[0] += pairs, status_dev[0] |= 1 on a capacity overflow of the
 * buffered schedule (any of the three may be NULL).
 *   CS_SCHED_LOOPEX   27 passes = the reference's loop-exchange levels
 *   CS_SCHED_BLOCK    8 passes of 2x2x2-coloured blocks, 27 levels inside
 *   CS_SCHED_SHELL    8 passes of 2x2x2-coloured blocks, one warp per
 *                     home-cell half shell, per-offset reaction slots
 *   CS_SCHED_BUFFERED one pass over all blocks into private footprint
 *                     buffers + a deterministic gather (buffered strategy,
 *                     taskgen.py:237-276, at block granularity)
 *   CS_SCHED_DATAFLOW the SHELL colour order executed as a dataflow: one
 *                     persistent launch, blocks taken in (colour, block)
 *                     order, each waiting only for its lower-colour
 *                     neighbour blocks (the task dependencies of
 *                     depgraph.py:28-49 at block granularity) */
size_t cs_force_ws_bytes(const cs_box *b, int sched, int64_t n);
int cs_lj_forces(const cs_box *b, const cs_lj *p, int sched, int64_t n,
                 const int32_t *cell_start, const double *x, const double *y, const double *z,
                 double *fx, double *fy, double *fz, double *energy_dev,
                 unsigned long long *npairs_dev, unsigned *status_dev, void *ws, size_t ws_bytes,
                 void *stream);

/* Verlet neighbour lists, built from the cell list of a box
 * whose cell edge is >= rc + skin.  The list of a home cell is a round table
 * (lane -> home particle, round x lane -> partner j, no j twice in a round),
 * so the force kernel keeps F_i in registers and writes each Newton-3
 * reaction into the (cell, stencil entry) slot of j without conflicts; the
 * colour-pass / buffered block structure of K2 is unchanged.
 * cs_verlet_build: list from the current (wrapped, binned) positions, and
 *   x0/y0/z0 = copy of x/y/z (reference for the displacement check, may be
 *   NULL).  status_dev |= 2 (a cell holds > 64 particles) or 4 (> 64 rounds).
 * cs_lj_forces_verlet: sched CS_SCHED_SHELL or CS_SCHED_BUFFERED; overwrites f.
 * Between rebuilds positions must NOT be wrapped: cs_vv_kick_drift_track is
 *   kick_drift without the wrap, setting flag[0] = 1 once a particle is more
 *   than half_skin from x0; cs_wrap_positions wraps before the next rebuild. */
size_t cs_verlet_list_bytes(const cs_box *b);
int cs_verlet_build(const cs_box *b, const cs_lj *p, double skin, const int32_t *cell_start,
                    const double *x, const double *y, const double *z, void *list,
                    size_t list_bytes, double *x0, double *y0, double *z0, int64_t n,
                    unsigned *status_dev, void *stream);
int cs_lj_forces_verlet(const cs_box *b, const cs_lj *p, int sched, int64_t n,
                        const int32_t *cell_start, const void *list, const double *x,
                        const double *y, const double *z, double *fx, double *fy, double *fz,
                        double *energy_dev, unsigned long long *npairs_dev, unsigned *status_dev,
                        void *ws, size_t ws_bytes, void *stream);
int cs_wrap_positions(int64_t n, const cs_box *b, double *x, double *y, double *z, void *stream);
/* Post-kick (kick != 0: v += hdtm f) fused with the exact prediction of the next
 * step's displacement flag (flag[0] = 1 if the next kick-drift, computed from the same
 * f, would move a particle more than half_skin from x0), so the rebuild decision of
 * step n+1 is taken at the end of step n (the x-slab step's protocol). */
int cs_vv_kick_predict(int64_t n, double hdtm, double dt, int kick, const double *fx,
                       const double *fy, const double *fz, double *vx, double *vy, double *vz,
                       const double *x, const double *y, const double *z, const double *x0,
                       const double *y0, const double *z0, double half_skin, int32_t *flag,
                       void *stream);
int cs_vv_kick_drift_track(int64_t n, double hdtm, double dt, const double *fx, const double *fy,
                           const double *fz, double *vx, double *vy, double *vz, double *x,
                           double *y, double *z, const double *x0, const double *y0,
                           const double *z0, double half_skin, int32_t *flag, void *stream);

/* Rebinning in place: copy the cell-sorted x, v, id back over the source. */
int cs_copy7(int64_t n, const double *x, const double *y, const double *z, const double *vx,
             const double *vy, const double *vz, const int32_t *id, double *xo, double *yo,
             double *zo, double *vxo, double *vyo, double *vzo, int32_t *ido, void *stream);
/* Device-side conditional rebuild inside a CUDA graph being captured on
 * `stream`: appends a kernel that turns flag[0] into the condition of an IF
 * node (and clears the flag), appends the IF node, and starts capturing its
 * body on `side_stream`; launch the rebuild work on side_stream, then call
 * cs_capture_if_end(side_stream).  Capture continues on `stream` after the
 * IF node. */
int cs_capture_if_begin(void *stream, void *side_stream, int32_t *flag, int32_t *count);
int cs_capture_if_end(void *side_stream);

/* K3: velocity Verlet.  kick: v += (dt/2m) f.  kick_drift: v += (dt/2m) f;
 * x += dt v; wrap into [0, L) on periodic axes. */
int cs_vv_kick(int64_t n, double hdtm, const double *fx, const double *fy, const double *fz,
               double *vx, double *vy, double *vz, void *stream);
int cs_vv_kick_drift(int64_t n, double hdtm, double dt, const cs_box *b, const double *fx,
                     const double *fy, const double *fz, double *vx, double *vy, double *vz,
                     double *x, double *y, double *z, void *stream);

/* K6: deterministic reductions.  out_dev[0] = 0.5 m sum v^2 */
int cs_kinetic(int64_t n, double mass, const double *vx, const double *vy, const double *vz,
               double *out_dev, void *ws, size_t ws_bytes, void *stream);
/* out_dev[0..2] = sum of each component */
int cs_sum3(int64_t n, const double *ax, const double *ay, const double *az, double *out_dev,
            void *ws, size_t ws_bytes, void *stream);

/* Slab halo helpers: pack the particles of local x-plane `plane` (cells
 * [plane*ny*nz ...]) into a contiguous buffer (positions, x shifted by
 * xshift), and add ghost-plane forces back. */
int cs_pack_plane(const cs_box *b, int plane, const int32_t *cell_start, const double *x,
                  const double *y, const double *z, double xshift, double *out, void *stream);
int cs_add_plane_forces(const cs_box *b, int plane, const int32_t *cell_start, const double *in,
                        double *fx, double *fy, double *fz, void *stream);
/* The same for a known particle range [lo, hi) (no host synchronisation). */
int cs_pack_range(int64_t lo, int64_t hi, const double *x, const double *y, const double *z,
                  double xshift, double *out, void *stream);
int cs_add_range_forces(int64_t lo, int64_t hi, const double *in, double *fx, double *fy,
                        double *fz, void *stream);

/* Slab decomposition (x-slabs, one rank per GPU).  Packed rows
 * are [7][stride] doubles: x, y, z, vx, vy, vz, id.
 * cs_slab_split: after the drift, split the owned particles into those that
 * stay (packed into `stay`, stride sstride) and those that moved into the
 * left / right neighbour's planes (packed, stride cap); counts_host[3] =
 * {stay, left, right}.  Synchronises. */
size_t cs_slab_ws_bytes(int64_t n);
int cs_slab_split(int64_t n, const cs_box *b, const double *x, const double *y, const double *z,
                  const double *vx, const double *vy, const double *vz, const int32_t *id,
                  double *stay, int64_t sstride, double *left, double *right, int64_t cap,
                  int64_t *counts_host, void *ws, size_t ws_bytes, void *stream);
int cs_unpack7(int64_t m, const double *src, int64_t stride, double *x, double *y, double *z,
               double *vx, double *vy, double *vz, int32_t *id, void *stream);
/* cell counts of local x-plane `plane` (ny*nz cells, storage order) and its
 * particle range [lo, hi) (range_host; synchronises) */
int cs_plane_counts(const cs_box *b, int plane, const int32_t *cell_start, int32_t *counts,
                    int64_t *range_host, void *stream);
/* append the received ghost plane (counts per cell + packed positions) after
 * the n_owned owned particles; zeroes their forces */
size_t cs_ghost_ws_bytes(const cs_box *b);
int cs_set_ghost_plane(const cs_box *b, int64_t n_owned, const int32_t *ghost_counts,
                       const double *ghost_xyz, int64_t m, int32_t *cell_start, double *x,
                       double *y, double *z, double *fx, double *fy, double *fz, void *ws,
                       size_t ws_bytes, void *stream);

/* ============ a11 / f3: worker-pool model (list scheduling) on the device =====
 * One persistent CTA, ready set as a bitmap scanned forward (the smallest ready
 * id never decreases), unit task durations, ready tasks handed to workers in
 * ascending id order.  Both synchronise (the makespan is returned on the host). */
/* simulate (schedsim.py:63-90): successor CSR sptr[ntasks+1] / succ[nedges] of
 * a forward-edge graph; start[t] = time step task t runs; *makespan_host =
 * SimResult.makespan.  CS_ECYCLE if the schedule stalls (schedsim.py:88-89).
 * max_indegree_host: the largest predecessor count (graphs up to 180,000
 * tasks with indegrees <= 255 keep the ready set in shared memory). */
size_t cs_listsched_ws_bytes(int64_t ntasks);
int cs_simulate_static(int64_t ntasks, int64_t nedges, const int64_t *sptr, const int32_t *succ,
                       int64_t workers, int64_t max_indegree_host, int32_t *start,
                       int64_t *makespan_host, void *ws, size_t ws_bytes, void *stream);
/* simulate_dynamic on a NestedPlan (schedsim.py:93-163, taskgen.py:279-325):
 * order_host = n offsets x dim int8, intra first.  Task arrays (capacity >=
 * cells * n): home cell, chain entry (index into order), spawning parent (-1 =
 * initial task), the realized predecessors pred_a < pred_b (-1 = none; the
 * edges of SimResult.graph, depgraph.py:28-49 applied at spawn time) and the
 * start step.  *ntasks_host = realized tasks (the spawn log length). */
size_t cs_nested_ws_bytes(const cs_grid *g, int n);
int cs_simulate_nested(const cs_grid *g, const int8_t *order_host, int n, int64_t workers,
                       int32_t *home, int16_t *entry, int32_t *parent, int32_t *pred_a,
                       int32_t *pred_b, int32_t *start, int64_t capacity, int64_t *ntasks_host,
                       int64_t *makespan_host, void *ws, size_t ws_bytes, void *stream);

/* FP64 pipe probe used by bench.py to measure the FP64 roofline peak:
 * blocks x 256 threads x iters x 256 flops (DFMA = 2 flops). */
int cs_probe_dfma(int blocks, int iters, double *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif
