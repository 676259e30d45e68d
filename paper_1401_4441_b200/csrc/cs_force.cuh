// cs_force.cuh -- K2: fp64 Lennard-Jones half-shell forces with Newton-3
// reaction writes, run under conflict-free colour-pass schedules.
//
// The force loop is the LJ counterpart of payload.apply_tasks
// (payload.py:84-119): a task (home, home+o) adds f_ij to every i in home and
// -f_ij to every j in the neighbour cell.  Two schedules, both derived from
// the reference's loop-exchange colouring (taskgen.py:202-234, grid.py:123-141):
//
//  CS_SCHED_LOOPEX  27 passes = the reference's loopex dependency levels
//                   (level 1 = intra, offset j / parity p of the
//                   highest axis with o != 0 -> level 2j+p).  One warp per
//                   task; tasks of a pass are write-disjoint, so forces are
//                   plain read-modify-writes in global memory, no atomics.
//  CS_SCHED_BLOCK   8 passes = 2x2x2 colouring of blocks of Bx x By x Bz
//                   cells (By, Bz >= 2, so same-colour footprints are
//                   disjoint).  One CTA per block stages the footprint's
//                   forces in shared memory and runs the same 27 loopex
//                   levels inside the block, separated by __syncthreads, then
//                   adds the footprint back to global memory once.
#pragma once
#include "cs_common.cuh"
#include "cs_md.cuh"
#include "cs_payload.cuh"

struct LJC {
  double rc2, eps4, eps48, sig2;
};

struct ForceArgs {
  Box b;
  LJC p;
  const int32_t *start;
  const double *x, *y, *z;
  double *fx, *fy, *fz;
  double *pe_cell;
  unsigned *hits_cell;
  int nbk[3];  // blocks per axis (block schedule)
  int cap;     // shared-memory particle capacity (block schedule)
  // Verlet round tables (cs_verlet.cuh); null for the link-cell schedules
  const int32_t *vl_nround;
  const uint8_t *vl_imap;
  const uint16_t *vl_desc;
  const int32_t *vl_boff;  // buffered block offsets computed at the list build
  const unsigned char *vl_tab;  // per-block tables computed at the list build
  // super-task kernels: pair counts added straight into the total (integer
  // atomics, order-independent), so non-energy steps need no reduction pass
  unsigned long long *npairs_direct;
};

// level (0..26) -> (stencil entry, parity); level 0 = intra
__host__ __device__ __forceinline__ void level_entry(int level, int *e, int *par) {
  *e = level == 0 ? 0 : (level + 1) >> 1;
  *par = level == 0 ? 0 : (level + 1) & 1;
}

// image shift of the neighbour cell (periodic axes only)
__device__ __forceinline__ double img_shift(int c, int o, int n, int per, double L) {
  if (!per) return 0.0;
  int s = c + o;
  return s >= n ? L : (s < 0 ? -L : 0.0);
}

// ------------------------------------------------------------ task routine --
// One warp evaluates one cell-pair task.  Lanes own neighbour particles j
// (chunks of 32); the home particles i are broadcast.  f_ij accumulates in
// the j lane (reaction, -f) and is warp-reduced for i (+f) -- the warp-level
// reduction of reaction forces -- so no two lanes write one address.
template <bool ENERGY>
__device__ __forceinline__ void task_warp(const double *__restrict__ x,
                                          const double *__restrict__ y,
                                          const double *__restrict__ z, int a0, int na, int b0,
                                          int nb, bool intra, double sx, double sy, double sz,
                                          double *FAx, double *FAy, double *FAz, double *FBx,
                                          double *FBy, double *FBz, const LJC &p, double &pe,
                                          unsigned &hits) {
  const int lane = threadIdx.x & 31;
  for (int jc = 0; jc < nb; jc += 32) {
    const int j = jc + lane;
    const bool vj = j < nb;
    double xj = 0, yj = 0, zj = 0;
    if (vj) {
      xj = __ldg(x + b0 + j) + sx;
      yj = __ldg(y + b0 + j) + sy;
      zj = __ldg(z + b0 + j) + sz;
    }
    double gx = 0, gy = 0, gz = 0;
    const int i_end = intra ? min(na, jc + 32) : na;
    for (int i = 0; i < i_end; ++i) {
      const double dx = __ldg(x + a0 + i) - xj;
      const double dy = __ldg(y + a0 + i) - yj;
      const double dz = __ldg(z + a0 + i) - zj;
      const double r2 = __fma_rn(dz, dz, __fma_rn(dy, dy, dx * dx));
      const bool hit = vj && r2 < p.rc2 && (!intra || j > i);
      double fx = 0, fy = 0, fz = 0;
      if (hit) {
        const double rinv2 = 1.0 / r2;
        const double sr2 = p.sig2 * rinv2;
        const double sr6 = sr2 * sr2 * sr2;
        const double ff = p.eps48 * sr6 * (sr6 - 0.5) * rinv2;
        fx = ff * dx;
        fy = ff * dy;
        fz = ff * dz;
        gx -= fx;
        gy -= fy;
        gz -= fz;
        if (ENERGY) pe += p.eps4 * sr6 * (sr6 - 1.0);
        ++hits;
      }
      if (__any_sync(CS_FULL, hit)) {
        fx = warp_sum(fx);
        fy = warp_sum(fy);
        fz = warp_sum(fz);
        if (lane == 0) {
          FAx[i] += fx;
          FAy[i] += fy;
          FAz[i] += fz;
        }
      }
    }
    __syncwarp();
    if (vj) {
      FBx[j] += gx;
      FBy[j] += gy;
      FBz[j] += gz;
    }
    __syncwarp();
  }
}

template <bool ENERGY>
__device__ __forceinline__ void task_stats(double pe, unsigned hits, int64_t home,
                                           double *pe_cell, unsigned *hits_cell,
                                           unsigned long long *npairs_direct = nullptr) {
  hits = warp_sum(hits);
  if (ENERGY) pe = warp_sum(pe);
  if ((threadIdx.x & 31) == 0) {
    if (npairs_direct) atomicAdd(npairs_direct, (unsigned long long)hits);
    else hits_cell[home] += hits;
    if (ENERGY) pe_cell[home] += pe;
  }
}

// ----------------------------------------------- schedule A: loopex passes --
template <bool ENERGY>
__global__ void __launch_bounds__(128) k_force_loopex(ForceArgs A, int level) {
  const Box &b = A.b;
  int e, par;
  level_entry(level, &e, &par);
  const int ax = c_stencil3.axis[e];
  const int hext[3] = {b.owned_x, b.nc[1], b.nc[2]};
  int m[3];
  for (int k = 0; k < 3; ++k) m[k] = (level > 0 && k == ax) ? (hext[k] - par + 1) >> 1 : hext[k];
  const int64_t ntask = (int64_t)m[0] * m[1] * m[2];
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= ntask) return;
  int c[3] = {(int)(warp % m[0]), (int)((warp / m[0]) % m[1]), (int)(warp / ((int64_t)m[0] * m[1]))};
  if (level > 0) c[ax] = 2 * c[ax] + par;
  const int64_t home = box_cell(b, c[0], c[1], c[2]);
  int n3[3];
  double sh[3];
  for (int k = 0; k < 3; ++k) {
    const int o = c_stencil3.o[e][k];
    int v = c[k] + o;
    sh[k] = img_shift(c[k], o, b.nc[k], b.per[k], b.L[k]);
    if (b.per[k])
      v = cs_wrap(v, b.nc[k]);
    else if (v < 0 || v >= b.nc[k])
      return;
    n3[k] = v;
  }
  const int64_t nbc = box_cell(b, n3[0], n3[1], n3[2]);
  const int a0 = A.start[home], na = A.start[home + 1] - a0;
  const int b0 = A.start[nbc], nb = A.start[nbc + 1] - b0;
  double pe = 0;
  unsigned hits = 0;
  task_warp<ENERGY>(A.x, A.y, A.z, a0, na, b0, nb, level == 0, sh[0], sh[1], sh[2], A.fx + a0,
                    A.fy + a0, A.fz + a0, A.fx + b0, A.fy + b0, A.fz + b0, A.p, pe, hits);
  task_stats<ENERGY>(pe, hits, home, A.pe_cell, A.hits_cell);
}

// ------------------------------------------------ schedule B: block passes --
#define BLK_MAX_FOOT 512  // footprint cells per CTA (Bx+1)(By+2)(Bz+2)
#define BLK_THREADS 128

template <bool ENERGY>
__global__ void __launch_bounds__(BLK_THREADS) k_force_block(ForceArgs A, int colour) {
  extern __shared__ double smF[];  // 3 * cap
  __shared__ int s_lstart[BLK_MAX_FOOT + 1];
  __shared__ int s_gstart[BLK_MAX_FOOT];
  __shared__ int s_gcell[BLK_MAX_FOOT];
  const Box &b = A.b;
  const int B[3] = {b.blk[0], b.blk[1], b.blk[2]};
  const int kc[3] = {colour & 1, (colour >> 1) & 1, (colour >> 2) & 1};
  int cnt[3];
  for (int k = 0; k < 3; ++k) cnt[k] = (A.nbk[k] - kc[k] + 1) >> 1;
  const int bid = blockIdx.x;
  const int bi[3] = {bid % cnt[0], (bid / cnt[0]) % cnt[1], bid / (cnt[0] * cnt[1])};
  int o0[3];  // global coords of the block origin
  for (int k = 0; k < 3; ++k) o0[k] = (2 * bi[k] + kc[k]) * B[k];
  const int FX = B[0] + 1, FY = B[1] + 2, FZ = B[2] + 2, nfc = FX * FY * FZ;
  // footprint cell (lx,ly,lz) <-> global (o0x+lx, o0y-1+ly, o0z-1+lz)
  for (int lc = threadIdx.x; lc < nfc; lc += blockDim.x) {
    const int l[3] = {lc % FX, (lc / FX) % FY, lc / (FX * FY)};
    int g[3];
    bool ok = true;
    for (int k = 0; k < 3; ++k) {
      int v = o0[k] + l[k] - (k ? 1 : 0);
      if (b.per[k])
        v = cs_wrap(v, b.nc[k]);
      else if (v < 0 || v >= b.nc[k])
        ok = false;
      g[k] = v;
    }
    const int64_t gc = ok ? box_cell(b, g[0], g[1], g[2]) : -1;
    s_gcell[lc] = (int)gc;
    s_gstart[lc] = ok ? A.start[gc] : 0;
    s_lstart[lc] = ok ? A.start[gc + 1] - A.start[gc] : 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // footprint prefix (<= 512 cells, once per CTA)
    int s = 0;
    for (int lc = 0; lc < nfc; ++lc) {
      int c = s_lstart[lc];
      s_lstart[lc] = s;
      s += c;
    }
    s_lstart[nfc] = s;
  }
  __syncthreads();
  const int total = s_lstart[nfc];
  const bool use_smem = total <= A.cap;
  if (use_smem)
    for (int i = threadIdx.x; i < 3 * total; i += blockDim.x) smF[i] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nhome = B[0] * B[1] * B[2];
  double pe_acc = 0;
  (void)lane;
  for (int level = 0; level < 27; ++level) {
    int e, par;
    level_entry(level, &e, &par);
    const int ax = c_stencil3.axis[e];
    for (int h = wid; h < nhome; h += nw) {
      const int hl[3] = {h % B[0], (h / B[0]) % B[1], h / (B[0] * B[1])};
      int hg[3];
      for (int k = 0; k < 3; ++k) hg[k] = o0[k] + hl[k];
      if (hg[0] >= b.owned_x) continue;  // partial block / ghost plane
      if (level > 0 && (hg[ax] & 1) != par) continue;
      const int lh = hl[0] + FX * ((hl[1] + 1) + FY * (hl[2] + 1));
      const int ln = (hl[0] + c_stencil3.o[e][0]) +
                     FX * ((hl[1] + 1 + c_stencil3.o[e][1]) + FY * (hl[2] + 1 + c_stencil3.o[e][2]));
      if (s_gcell[ln] < 0 || s_gcell[lh] < 0) continue;
      double sh[3];
      for (int k = 0; k < 3; ++k)
        sh[k] = img_shift(cs_wrap(hg[k], b.nc[k]), c_stencil3.o[e][k], b.nc[k], b.per[k], b.L[k]);
      const int a0 = s_gstart[lh], na = s_lstart[lh + 1] - s_lstart[lh];
      const int b0 = s_gstart[ln], nb = s_lstart[ln + 1] - s_lstart[ln];
      double *FAx, *FAy, *FAz, *FBx, *FBy, *FBz;
      if (use_smem) {
        FAx = smF + s_lstart[lh];
        FBx = smF + s_lstart[ln];
        FAy = FAx + total;
        FAz = FAx + 2 * total;
        FBy = FBx + total;
        FBz = FBx + 2 * total;
      } else {
        FAx = A.fx + a0;
        FAy = A.fy + a0;
        FAz = A.fz + a0;
        FBx = A.fx + b0;
        FBy = A.fy + b0;
        FBz = A.fz + b0;
      }
      double pe = 0;
      unsigned hits = 0;
      task_warp<ENERGY>(A.x, A.y, A.z, a0, na, b0, nb, level == 0, sh[0], sh[1], sh[2], FAx, FAy,
                        FAz, FBx, FBy, FBz, A.p, pe, hits);
      task_stats<ENERGY>(pe, hits, s_gcell[lh], A.pe_cell, A.hits_cell);
    }
    __syncthreads();
  }
  (void)pe_acc;
  if (use_smem) {  // add the footprint back (same-colour footprints are disjoint)
    for (int lc = wid; lc < nfc; lc += nw) {
      const int l0 = s_lstart[lc], n = s_lstart[lc + 1] - l0, g0 = s_gstart[lc];
      for (int i = threadIdx.x & 31; i < n; i += 32) {
        A.fx[g0 + i] += smF[l0 + i];
        A.fy[g0 + i] += smF[total + l0 + i];
        A.fz[g0 + i] += smF[2 * total + l0 + i];
      }
    }
  }
}

// ----------------------------------------------------------- host launcher --
__global__ void k_reduce_cells(int64_t n, const double *pe, const unsigned *hits, double *part,
                               unsigned long long *hpart, int energy) {
  double s = 0;
  unsigned long long h = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (energy) s += pe[i];
    h += hits[i];
  }
  s = block_sum(s);
  h = block_sum(h);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    hpart[blockIdx.x] = h;
  }
}
__global__ void k_reduce_cells_final(int np, const double *part, const unsigned long long *hpart,
                                     double *energy, unsigned long long *npairs) {
  double s = 0;
  unsigned long long h = 0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    s += part[i];
    h += hpart[i];
  }
  s = block_sum(s);
  h = block_sum(h);
  if (threadIdx.x == 0) {
    if (energy) energy[0] += s;
    if (npairs) npairs[0] += h;
  }
}

static int block_grid(const Box &b, int nbk[3]) {
  const int hext[3] = {b.owned_x, b.nc[1], b.nc[2]};
  for (int k = 0; k < 3; ++k) {
    CS_REQUIRE(b.blk[k] >= 1, "block shape must be >= 1");
    if (b.per[k]) {
      CS_REQUIRE(hext[k] % (2 * b.blk[k]) == 0,
                 "periodic extent %d on axis %d must be a multiple of 2*block (%d)", hext[k], k,
                 2 * b.blk[k]);
      CS_REQUIRE(k == 0 || b.blk[k] >= 2, "block y/z extent must be >= 2 (disjoint footprints)");
    }
    nbk[k] = (hext[k] + b.blk[k] - 1) / b.blk[k];
  }
  CS_REQUIRE((b.blk[0] + 1) * (b.blk[1] + 2) * (b.blk[2] + 2) <= BLK_MAX_FOOT,
             "block footprint exceeds %d cells", BLK_MAX_FOOT);
  return CS_OK;
}

static int force_cap(const Box &b) {
  (void)b;
  return 2048;  // particles staged per CTA (48 KB of fp64 forces)
}

struct Box;
static size_t shell_buffered_ws(const Box &b, int64_t n);

extern "C" size_t cs_force_ws_bytes(const cs_box *bx, int sched, int64_t n) {
  int64_t nc = (int64_t)bx->nc[0] * bx->nc[1] * bx->nc[2];
  size_t base = cs_ws_slice(sizeof(double) * nc) + cs_ws_slice(sizeof(unsigned) * nc) +
                cs_ws_slice(sizeof(double) * RED_BLOCKS_MAX) +
                cs_ws_slice(sizeof(unsigned long long) * RED_BLOCKS_MAX);
  if (sched == CS_SCHED_BUFFERED || sched == CS_SCHED_DATAFLOW) {
    Box b;
    if (make_box(bx, &b) != CS_OK) return 0;
    base += shell_buffered_ws(b, n);  // (covers the dataflow flags too)
  }
  return base;
}

static int check_lj_box(const Box &b, double rc) {
  for (int k = 0; k < 3; ++k) {
    CS_REQUIRE(b.gnc[k] >= 3, "LJ link cells need >= 3 cells per axis (got %d on axis %d)",
               b.gnc[k], k);
    CS_REQUIRE(b.L[k] / b.gnc[k] >= rc * (1 - 1e-12),
               "cell edge %.6g on axis %d is below the cutoff %.6g", b.L[k] / b.gnc[k], k, rc);
  }
  return CS_OK;
}

// super-task kernel modes (cs_force2.cuh): 0 = colour pass (blockIdx = block
// of that colour), 1 = buffered (blockIdx = block), 2 = dataflow (colour and
// block from a ticket)
enum { SH_COLOUR = 0, SH_BUFFERED = 1, SH_DATAFLOW = 2 };

static int launch_shell_passes(const ForceArgs &A, bool energy, int mode, bool verlet,
                               cs_ws *w, int64_t n, unsigned *status, cudaStream_t st);

// vlist: Verlet round tables (cs_verlet.cuh) or null for the link-cell path
static int lj_forces_impl(const cs_box *bx, const cs_lj *lj, int sched, int64_t npart,
                          const int32_t *cell_start, const void *vlist, const double *x,
                          const double *y, const double *z, double *fx, double *fy, double *fz,
                          double *energy_dev, unsigned long long *npairs_dev,
                          unsigned *status_dev, void *ws, size_t ws_bytes, cudaStream_t st);

extern "C" int cs_lj_forces(const cs_box *bx, const cs_lj *lj, int sched, int64_t npart,
                            const int32_t *cell_start, const double *x, const double *y,
                            const double *z, double *fx, double *fy, double *fz,
                            double *energy_dev, unsigned long long *npairs_dev,
                            unsigned *status_dev, void *ws, size_t ws_bytes, void *stream) {
  return lj_forces_impl(bx, lj, sched, npart, cell_start, nullptr, x, y, z, fx, fy, fz,
                        energy_dev, npairs_dev, status_dev, ws, ws_bytes, cs_stream(stream));
}

static void vl_attach(ForceArgs &A, const void *vlist);  // cs_verlet.cuh

static int lj_forces_impl(const cs_box *bx, const cs_lj *lj, int sched, int64_t npart,
                          const int32_t *cell_start, const void *vlist, const double *x,
                          const double *y, const double *z, double *fx, double *fy, double *fz,
                          double *energy_dev, unsigned long long *npairs_dev,
                          unsigned *status_dev, void *ws, size_t ws_bytes, cudaStream_t st) {
  CS_TRY(cs_upload_stencil());
  ForceArgs A;
  memset(&A, 0, sizeof(A));
  CS_TRY(make_box(bx, &A.b));
  CS_TRY(check_lj_box(A.b, lj->rc));
  A.p.rc2 = lj->rc * lj->rc;
  A.p.eps4 = 4.0 * lj->eps;
  A.p.eps48 = 48.0 * lj->eps;
  A.p.sig2 = lj->sigma * lj->sigma;
  A.start = cell_start;
  A.x = x;
  A.y = y;
  A.z = z;
  A.fx = fx;
  A.fy = fy;
  A.fz = fz;
  const int64_t nc = A.b.ncells;
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, double, pe_cell, nc);
  CS_WS_TAKE(w, unsigned, hits_cell, nc);
  CS_WS_TAKE(w, double, part, RED_BLOCKS_MAX);
  CS_WS_TAKE(w, unsigned long long, hpart, RED_BLOCKS_MAX);
  A.pe_cell = pe_cell;
  A.hits_cell = hits_cell;
  const bool energy = energy_dev != nullptr;
  if (energy) CS_CUDA(cudaMemsetAsync(pe_cell, 0, sizeof(double) * nc, st));
  const bool direct = vlist || sched == CS_SCHED_SHELL || sched == CS_SCHED_BUFFERED ||
                      sched == CS_SCHED_DATAFLOW;
  A.npairs_direct = direct ? npairs_dev : nullptr;
  if (!direct) CS_CUDA(cudaMemsetAsync(hits_cell, 0, sizeof(unsigned) * nc, st));
  if (vlist) {
    CS_REQUIRE(sched == CS_SCHED_SHELL || sched == CS_SCHED_BUFFERED || sched == CS_SCHED_DATAFLOW,
               "Verlet forces run under CS_SCHED_SHELL, CS_SCHED_BUFFERED or CS_SCHED_DATAFLOW");
    vl_attach(A, vlist);
    CS_TRY(block_grid(A.b, A.nbk));
    if (sched != CS_SCHED_BUFFERED) {  // in-place passes accumulate: start from zero
      CS_CUDA(cudaMemsetAsync(fx, 0, sizeof(double) * npart, st));
      CS_CUDA(cudaMemsetAsync(fy, 0, sizeof(double) * npart, st));
      CS_CUDA(cudaMemsetAsync(fz, 0, sizeof(double) * npart, st));
    }
    CS_TRY(launch_shell_passes(A, energy, sched == CS_SCHED_BUFFERED ? SH_BUFFERED
                                          : (sched == CS_SCHED_DATAFLOW ? SH_DATAFLOW : SH_COLOUR),
                               true, &w, npart, status_dev, st));
  } else if (sched == CS_SCHED_LOOPEX) {
    // the level sets are write-disjoint only if no periodic axis wraps with
    // an odd extent (taskgen.py:210-215 warns for the same case)
    const int hext[3] = {A.b.owned_x, A.b.nc[1], A.b.nc[2]};
    for (int k = 0; k < 3; ++k)
      CS_REQUIRE(!A.b.per[k] || hext[k] % 2 == 0,
                 "loop-exchange colour passes need even periodic extents (axis %d has %d cells)", k,
                 hext[k]);
    int8_t st3[14 * 3];
    int nst;
    cs_host_canonical_stencil(3, st3, &nst);
    for (int level = 0; level < 27; ++level) {
      int e, par;
      level_entry(level, &e, &par);
      int ax = 0;  // highest axis with a nonzero offset component (the parity axis)
      for (int k = 0; k < 3; ++k)
        if (st3[3 * e + k]) ax = k;
      int64_t ntask = 1;  // the kernel's task grid m[] of this level
      for (int k = 0; k < 3; ++k) ntask *= (level > 0 && k == ax) ? (hext[k] - par + 1) >> 1 : hext[k];
      if (ntask == 0) continue;
      unsigned blocks = (unsigned)((ntask * 32 + 127) / 128);
      if (energy)
        k_force_loopex<true><<<blocks, 128, 0, st>>>(A, level);
      else
        k_force_loopex<false><<<blocks, 128, 0, st>>>(A, level);
    }
  } else if (sched == CS_SCHED_BLOCK) {
    CS_TRY(block_grid(A.b, A.nbk));
    A.cap = force_cap(A.b);
    size_t smem = sizeof(double) * 3 * A.cap;
    static size_t attr_smem[CS_MAX_DEVICES];  // largest dynamic shared memory enabled so far
    const int dev = cs_device_index();
    if (smem > attr_smem[dev]) {
      CS_CUDA(cudaFuncSetAttribute(k_force_block<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
      CS_CUDA(cudaFuncSetAttribute(k_force_block<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_smem[dev] = smem;
    }
    for (int colour = 0; colour < 8; ++colour) {
      int kc[3] = {colour & 1, (colour >> 1) & 1, (colour >> 2) & 1};
      unsigned blocks = 1;
      for (int k = 0; k < 3; ++k) blocks *= (unsigned)((A.nbk[k] - kc[k] + 1) >> 1);
      if (blocks == 0) continue;
      if (energy)
        k_force_block<true><<<blocks, BLK_THREADS, smem, st>>>(A, colour);
      else
        k_force_block<false><<<blocks, BLK_THREADS, smem, st>>>(A, colour);
    }
  } else if (sched == CS_SCHED_SHELL || sched == CS_SCHED_BUFFERED || sched == CS_SCHED_DATAFLOW) {
    CS_TRY(block_grid(A.b, A.nbk));
    CS_TRY(launch_shell_passes(A, energy, sched == CS_SCHED_BUFFERED ? SH_BUFFERED
                                          : (sched == CS_SCHED_DATAFLOW ? SH_DATAFLOW : SH_COLOUR),
                               false, &w, npart, status_dev, st));
  } else {
    CS_REQUIRE(0, "unknown schedule %d", sched);
  }
  CS_TRY(cs_check_launch("lj_forces"));
  if (energy || (npairs_dev && !direct)) {
    if (direct) CS_CUDA(cudaMemsetAsync(hits_cell, 0, sizeof(unsigned) * nc, st));  // (unused)
    int np = (int)cs_reduce_partials(nc);
    k_reduce_cells<<<np, RED_THREADS, 0, st>>>(nc, pe_cell, hits_cell, part, hpart, energy);
    k_reduce_cells_final<<<1, 1024, 0, st>>>(np, part, hpart, energy_dev, direct ? nullptr : npairs_dev);
  }
  return cs_check_launch("lj_forces_reduce");
}

// ================= K5 under the LJ schedules: integer payload race harness ==
struct PayArgs {
  StreamDesc d;  // grid as a stream descriptor (canonical stencil)
  Box b;         // same grid as a cell box (periodicity, block shape)
  const int64_t *q;
  int64_t *acc;
  unsigned long long *mark_pass, *mark_level;
  unsigned *conflicts;
  int nbk[3];
  int race;
};

__device__ __forceinline__ void pay_mark(const PayArgs &A, int64_t cell, uint32_t ep1,
                                         uint32_t w1, uint32_t ep2, uint32_t w2) {
  if (!A.race) return;
  unsigned long long t1 = ((unsigned long long)ep1 << 32) | w1;
  unsigned long long o1 = atomicExch(&A.mark_pass[cell], t1);
  if ((uint32_t)(o1 >> 32) == ep1 && (uint32_t)o1 != w1) atomicAdd(A.conflicts, 1u);
  unsigned long long t2 = ((unsigned long long)ep2 << 32) | w2;
  unsigned long long o2 = atomicExch(&A.mark_level[cell], t2);
  if ((uint32_t)(o2 >> 32) == ep2 && (uint32_t)o2 != w2) atomicAdd(A.conflicts, 1u);
}

__device__ __forceinline__ void pay_task(const PayArgs &A, const int *c, int e, bool intra,
                                         uint32_t ep1, uint32_t w1, uint32_t ep2, uint32_t w2) {
  const int64_t home = box_cell(A.b, c[0], c[1], c[2]);
  if (intra) {
    pay_mark(A, home, ep1, w1, ep2, w2);
    A.acc[home] += pay_intra(A.q[home]);
    return;
  }
  int n3[3];
  for (int k = 0; k < 3; ++k) {
    int v = c[k] + c_stencil3.o[e][k];
    if (A.b.per[k])
      v = cs_wrap(v, A.b.nc[k]);
    else if (v < 0 || v >= A.b.nc[k])
      return;
    n3[k] = v;
  }
  const int64_t nb = box_cell(A.b, n3[0], n3[1], n3[2]);
  pay_mark(A, home, ep1, w1, ep2, w2);
  if (nb != home) pay_mark(A, nb, ep1, w1, ep2, w2);
  const int64_t g = pay_pair(A.q[home], A.q[nb], c_stencil3.o[e][0], c_stencil3.o[e][1],
                             c_stencil3.o[e][2], 3);
  A.acc[home] += g;
  A.acc[nb] -= g;
}

__global__ void k_pay_loopex(PayArgs A, int level) {
  int e, par;
  level_entry(level, &e, &par);
  const int ax = c_stencil3.axis[e];
  const int hext[3] = {A.b.owned_x, A.b.nc[1], A.b.nc[2]};
  int m[3];
  for (int k = 0; k < 3; ++k) m[k] = (level > 0 && k == ax) ? (hext[k] - par + 1) >> 1 : hext[k];
  const int64_t ntask = (int64_t)m[0] * m[1] * m[2];
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntask;
       t += (int64_t)gridDim.x * blockDim.x) {
    int c[3] = {(int)(t % m[0]), (int)((t / m[0]) % m[1]), (int)(t / ((int64_t)m[0] * m[1]))};
    if (level > 0) c[ax] = 2 * c[ax] + par;
    pay_task(A, c, e, level == 0, level + 1, (uint32_t)t, level + 1, (uint32_t)t);
  }
}

__global__ void k_pay_block(PayArgs A, int colour) {
  const int B[3] = {A.b.blk[0], A.b.blk[1], A.b.blk[2]};
  const int kc[3] = {colour & 1, (colour >> 1) & 1, (colour >> 2) & 1};
  int cnt[3];
  for (int k = 0; k < 3; ++k) cnt[k] = (A.nbk[k] - kc[k] + 1) >> 1;
  const int bid = blockIdx.x;
  const int bi[3] = {bid % cnt[0], (bid / cnt[0]) % cnt[1], bid / (cnt[0] * cnt[1])};
  int o0[3];
  for (int k = 0; k < 3; ++k) o0[k] = (2 * bi[k] + kc[k]) * B[k];
  const int nhome = B[0] * B[1] * B[2];
  for (int level = 0; level < 27; ++level) {
    int e, par;
    level_entry(level, &e, &par);
    const int ax = c_stencil3.axis[e];
    for (int h = threadIdx.x; h < nhome; h += blockDim.x) {
      int c[3] = {o0[0] + h % B[0], o0[1] + (h / B[0]) % B[1], o0[2] + h / (B[0] * B[1])};
      if (c[0] >= A.b.owned_x) continue;
      if (level > 0 && (c[ax] & 1) != par) continue;
      pay_task(A, c, e, level == 0, colour + 1, (uint32_t)bid, colour * 27 + level + 1,
               (uint32_t)(bid * 1024 + h));
    }
    __syncthreads();
  }
}

extern "C" size_t cs_payload_colour_ws_bytes(const cs_grid *g) {
  int64_t nc = 1;
  for (int k = 0; k < g->dim; ++k) nc *= g->ext[k];
  return 2 * cs_ws_slice(sizeof(unsigned long long) * nc) + cs_ws_slice(64);
}

extern "C" int cs_payload_colour(const cs_grid *g, int sched, const int32_t *block_host,
                                 const int64_t *q, int64_t *acc, int race_check, void *ws,
                                 size_t ws_bytes, void *stream) {
  CS_TRY(cs_upload_stencil());
  CS_REQUIRE(g && g->dim == 3, "colour-pass schedules are 3D");
  cudaStream_t st = cs_stream(stream);
  PayArgs A;
  int8_t dummy[3] = {0, 0, 0};
  CS_TRY(build_desc(g, CS_STREAM_BASIC, dummy, 1, 2, &A.d));
  cs_box cb;
  memset(&cb, 0, sizeof(cb));
  for (int k = 0; k < 3; ++k) {
    cb.nc[k] = cb.gnc[k] = g->ext[k];
    cb.periodic[k] = g->periodic[k];
    cb.block[k] = block_host ? block_host[k] : 2;
    cb.L[k] = 1.0;
    cb.inv[k] = 1.0;
  }
  cb.owned_x = g->ext[0];
  // keep the reference's x-fastest cell ids even for an open x axis
  CS_TRY(make_box(&cb, &A.b));
  A.b.stride[0] = 1;
  A.b.stride[1] = A.b.nc[0];
  A.b.stride[2] = (int64_t)A.b.nc[0] * A.b.nc[1];
  A.q = q;
  A.acc = acc;
  A.race = race_check;
  cs_ws w(ws, ws_bytes);
  const int64_t nc = A.b.ncells;
  CS_WS_TAKE(w, unsigned long long, mp, nc);
  CS_WS_TAKE(w, unsigned long long, ml, nc);
  CS_WS_TAKE(w, unsigned, conf, 16);
  A.mark_pass = mp;
  A.mark_level = ml;
  A.conflicts = conf;
  CS_CUDA(cudaMemsetAsync(acc, 0, sizeof(int64_t) * nc, st));
  CS_CUDA(cudaMemsetAsync(conf, 0, sizeof(unsigned), st));
  if (race_check) {
    CS_CUDA(cudaMemsetAsync(mp, 0, sizeof(unsigned long long) * nc, st));
    CS_CUDA(cudaMemsetAsync(ml, 0, sizeof(unsigned long long) * nc, st));
  }
  if (sched == CS_SCHED_LOOPEX) {
    for (int level = 0; level < 27; ++level)
      k_pay_loopex<<<grid_for(nc, 128), 128, 0, st>>>(A, level);
  } else if (sched == CS_SCHED_BLOCK) {
    CS_TRY(block_grid(A.b, A.nbk));
    for (int colour = 0; colour < 8; ++colour) {
      int kc[3] = {colour & 1, (colour >> 1) & 1, (colour >> 2) & 1};
      unsigned blocks = 1;
      for (int k = 0; k < 3; ++k) blocks *= (unsigned)((A.nbk[k] - kc[k] + 1) >> 1);
      if (blocks) k_pay_block<<<blocks, 128, 0, st>>>(A, colour);
    }
  } else {
    CS_REQUIRE(0, "unknown schedule %d", sched);
  }
  CS_TRY(cs_check_launch("payload_colour"));
  if (race_check) {
    unsigned h = 0;
    CS_CUDA(cudaMemcpyAsync(&h, conf, sizeof(h), cudaMemcpyDeviceToHost, st));
    CS_CUDA(cudaStreamSynchronize(st));
    if (h) {
      cs_set_error("race detector: %u same-pass writer conflicts", h);
      return CS_ECONFLICT;
    }
  }
  return CS_OK;
}
