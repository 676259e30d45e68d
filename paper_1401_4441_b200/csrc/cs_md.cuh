// cs_md.cuh -- particle setup, K1 cell binning, K3 velocity Verlet, slab helpers.
//
// No reference code exists for particles; the
// conventions extend the reference's: x-fastest cell ids (grid.py:3-4), the
// splitmix64 counter PRNG of payload.py:36-40 for every random draw, and the
// cell list as the canonical (cell, particle id) order so it is independent
// of history and bit-comparable with the CPU oracle.
#pragma once
#include "cs_common.cuh"

#define JITTER_KEY 0xD1B54A32D192ED03ull
#define VEL_KEY 0x8CB92BA72F3D8DD7ull

struct Box {  // device-side copy of cs_box plus derived strides
  int nc[3], gnc[3], x0, owned_x, per[3], blk[3];
  int64_t stride[3];
  int64_t ncells;
  double L[3], inv[3];
};

static int make_box(const cs_box *b, Box *o) {
  CS_REQUIRE(b, "null box");
  for (int k = 0; k < 3; ++k) {
    o->nc[k] = b->nc[k];
    o->gnc[k] = b->gnc[k];
    o->per[k] = b->periodic[k] ? 1 : 0;
    o->blk[k] = b->block[k];
    o->L[k] = b->L[k];
    o->inv[k] = b->inv[k];
    CS_REQUIRE(b->nc[k] >= 1 && b->gnc[k] >= 1, "cell counts must be >= 1");
  }
  o->x0 = b->x0;
  o->owned_x = b->owned_x > 0 ? b->owned_x : b->nc[0];
  CS_REQUIRE(o->owned_x <= o->nc[0], "owned_x > nc[0]");
  if (o->per[0]) {
    // x-fastest storage = the reference's cell id (grid.py:93-101)
    o->stride[0] = 1;
    o->stride[1] = o->nc[0];
    o->stride[2] = (int64_t)o->nc[0] * o->nc[1];
  } else {
    // x-slab storage: x slowest so the ghost plane is the tail of the arrays
    o->stride[0] = (int64_t)o->nc[1] * o->nc[2];
    o->stride[1] = 1;
    o->stride[2] = o->nc[1];
  }
  o->ncells = (int64_t)o->nc[0] * o->nc[1] * o->nc[2];
  return CS_OK;
}

__host__ __device__ __forceinline__ int64_t box_cell(const Box &b, int x, int y, int z) {
  return x * b.stride[0] + y * b.stride[1] + z * b.stride[2];
}

__device__ __forceinline__ double uni_dev(uint64_t base, uint64_t i) {
  return (double)(cs_splitmix64(base + i) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ double wrap_dev(double x, double L) {
  if (x < 0.0) x = __dadd_rn(x, L);
  if (x >= L) x = __dadd_rn(x, -L);
  return x;
}

// any distance from the box (host-loaded positions): one floor reduction when
// more than a box length outside, then the single-step wrap -- identical to
// wrap_dev for positions within one box length of [0, L)
__device__ __forceinline__ double wrap_far(double x, double L) {
  if (x < -L || x >= 2.0 * L) x = __dadd_rn(x, -__dmul_rn(L, floor(x / L)));
  return wrap_dev(wrap_dev(x, L), L);
}

// ------------------------------------------------------------------ setup --
struct FccArgs {
  int nuc[3];
  double a[3], L[3], jit;
  uint64_t base;
};
__global__ void k_init_fcc(FccArgs f, int64_t n, double *x, double *y, double *z, int32_t *id) {
  const double bas[4][3] = {{0, 0, 0}, {0, 0.5, 0.5}, {0.5, 0, 0.5}, {0.5, 0.5, 0}};
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    int b = (int)(p & 3);
    int64_t uc = p >> 2;
    int ii[3] = {(int)(uc % f.nuc[0]), (int)((uc / f.nuc[0]) % f.nuc[1]),
                 (int)(uc / ((int64_t)f.nuc[0] * f.nuc[1]))};
    double out[3];
    for (int k = 0; k < 3; ++k) {
      double t = __dadd_rn((double)ii[k], bas[b][k] + 0.25);
      double u = uni_dev(f.base, (uint64_t)(3 * p + k));
      double s = __dmul_rn(t, f.a[k]);
      double j = __dmul_rn(__dadd_rn(__dmul_rn(2.0, u), -1.0), f.jit);
      out[k] = wrap_dev(__dadd_rn(s, j), f.L[k]);
    }
    x[p] = out[0];
    y[p] = out[1];
    z[p] = out[2];
    id[p] = (int32_t)p;
  }
}

extern "C" int cs_init_fcc(const int32_t *nuc, const double *a, const double *L, double jitter,
                           int64_t seed, double *x, double *y, double *z, int32_t *id,
                           void *stream) {
  FccArgs f;
  int64_t n = 4;
  for (int k = 0; k < 3; ++k) {
    CS_REQUIRE(nuc[k] >= 1, "unit cells must be >= 1");
    f.nuc[k] = nuc[k];
    f.a[k] = a[k];
    f.L[k] = L[k];
    n *= nuc[k];
  }
  f.jit = jitter;
  f.base = cs_splitmix64_host((uint64_t)seed ^ JITTER_KEY);
  k_init_fcc<<<grid_for(n, 256), 256, 0, cs_stream(stream)>>>(f, n, x, y, z, id);
  return cs_check_launch("init_fcc");
}

__global__ void k_init_gauss(int64_t n, uint64_t base, double *vx, double *vy, double *vz) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < 3 * n;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t q = k >> 1;
    double u1 = uni_dev(base, (uint64_t)(2 * q)), u2 = uni_dev(base, (uint64_t)(2 * q + 1));
    double r = sqrt(-2.0 * log(1.0 - u1));
    double th = 6.283185307179586 * u2;
    double g = (k & 1) ? r * sin(th) : r * cos(th);
    double *dst = (k % 3 == 0) ? vx : (k % 3 == 1 ? vy : vz);
    dst[k / 3] = g;
  }
}
// v -= mean (sums[0..2] / n)
__global__ void k_remove_mean(int64_t n, const double *sums, double *vx, double *vy, double *vz) {
  double mx = sums[0] / (double)n, my = sums[1] / (double)n, mz = sums[2] / (double)n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    vx[i] -= mx;
    vy[i] -= my;
    vz[i] -= mz;
  }
}
// scale so that sum m v^2 = T (3N-3); ke2 = 0.5 m sum v^2
__global__ void k_scale_T(int64_t n, double T, double mass, const double *ke, double *vx,
                          double *vy, double *vz) {
  double s2 = 2.0 * ke[0] / mass;
  double sc = sqrt(T * (double)(3 * n - 3) / (mass * s2));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    vx[i] *= sc;
    vy[i] *= sc;
    vz[i] *= sc;
  }
}

extern "C" int cs_init_velocities(int64_t n, double T, double mass, int64_t seed, double *vx,
                                  double *vy, double *vz, void *ws, size_t ws_bytes,
                                  void *stream) {
  CS_REQUIRE(n >= 2, "need at least 2 particles");
  cudaStream_t st = cs_stream(stream);
  uint64_t base = cs_splitmix64_host((uint64_t)seed ^ VEL_KEY);
  k_init_gauss<<<grid_for(3 * n, 256), 256, 0, st>>>(n, base, vx, vy, vz);
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, double, sc, 8);
  size_t rest = ws_bytes - w.used;
  void *rws = w.base + w.used;
  CS_TRY(cs_sum3(n, vx, vy, vz, sc, rws, rest, stream));
  k_remove_mean<<<grid_for(n, 256), 256, 0, st>>>(n, sc, vx, vy, vz);
  CS_TRY(cs_kinetic(n, mass, vx, vy, vz, sc + 4, rws, rest, stream));
  k_scale_T<<<grid_for(n, 256), 256, 0, st>>>(n, T, mass, sc + 4, vx, vy, vz);
  return cs_check_launch("init_velocities");
}

// ------------------------------------------------------------ K1: binning --
__device__ __forceinline__ int bin_coord(double x, double inv, int n) {
  int c = (int)(x * inv);  // single IEEE multiply, identical on the CPU oracle
  return c >= n ? n - 1 : (c < 0 ? 0 : c);
}

__global__ void k_bin_count(int64_t n, Box b, const double *x, const double *y, const double *z,
                            int32_t *cell_of, int32_t *slot, int32_t *count, int *err) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    int cx = bin_coord(x[p], b.inv[0], b.gnc[0]) - b.x0;
    int cy = bin_coord(y[p], b.inv[1], b.gnc[1]);
    int cz = bin_coord(z[p], b.inv[2], b.gnc[2]);
    if (cx < 0 || cx >= b.owned_x) {
      atomicOr(err, 1);
      cx = cx < 0 ? 0 : b.owned_x - 1;
    }
    int32_t c = (int32_t)box_cell(b, cx, cy, cz);
    cell_of[p] = c;
    slot[p] = atomicAdd(&count[c], 1);
  }
}

__global__ void k_bin_scatter(int64_t n, const int32_t *cell_of, const int32_t *slot,
                              const int32_t *start, int32_t *src) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    src[start[cell_of[p]] + slot[p]] = (int32_t)p;
}

// one warp per cell: rank the cell's particles by id (canonical order),
// then gather x, v, id into the sorted arrays and zero the forces
__global__ void k_cell_sort_gather(int64_t ncells, const int32_t *start, const int32_t *src,
                                   const int32_t *id, const double *x, const double *y,
                                   const double *z, const double *vx, const double *vy,
                                   const double *vz, double *xo, double *yo, double *zo,
                                   double *vxo, double *vyo, double *vzo, int32_t *ido,
                                   double *fxo, double *fyo, double *fzo) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp; c < ncells; c += nwarps) {
    int32_t s0 = start[c], cnt = start[c + 1] - s0;
    for (int32_t a = 0; a < cnt; a += 32) {
      int32_t me = a + lane;
      int32_t p = me < cnt ? src[s0 + me] : -1;
      int32_t myid = p >= 0 ? id[p] : 0x7fffffff;
      int32_t rank = 0;
      for (int32_t b2 = 0; b2 < cnt; b2 += 32) {
        int32_t q = b2 + lane < cnt ? id[src[s0 + b2 + lane]] : 0x7fffffff;
        int lim = min(32, cnt - b2);
        for (int k = 0; k < lim; ++k) {
          int32_t other = __shfl_sync(CS_FULL, q, k);
          rank += (other < myid);
        }
      }
      if (p >= 0) {
        int32_t d = s0 + rank;
        xo[d] = x[p];
        yo[d] = y[p];
        zo[d] = z[p];
        if (vx) {
          vxo[d] = vx[p];
          vyo[d] = vy[p];
          vzo[d] = vz[p];
        }
        ido[d] = myid;
        fxo[d] = 0.0;
        fyo[d] = 0.0;
        fzo[d] = 0.0;
      }
    }
  }
}

extern "C" size_t cs_bin_ws_bytes(int64_t n, const cs_box *b) {
  int64_t nc = (int64_t)b->nc[0] * b->nc[1] * b->nc[2];
  return 3 * cs_ws_slice(sizeof(int32_t) * (n + 1)) + cs_ws_slice(sizeof(int32_t) * (nc + 1)) +
         cs_ws_slice(64) + cs_scan_ws_bytes(nc);
}

extern "C" int cs_build_cells(int64_t n, const cs_box *bx, const double *x, const double *y,
                              const double *z, const double *vx, const double *vy,
                              const double *vz, const int32_t *id, double *xo, double *yo,
                              double *zo, double *vxo, double *vyo, double *vzo, int32_t *ido,
                              double *fxo, double *fyo, double *fzo, int32_t *cell_start,
                              void *ws, size_t ws_bytes, void *stream) {
  Box b;
  CS_TRY(make_box(bx, &b));
  cudaStream_t st = cs_stream(stream);
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, cell_of, n + 1);
  CS_WS_TAKE(w, int32_t, slot, n + 1);
  CS_WS_TAKE(w, int32_t, src, n + 1);
  CS_WS_TAKE(w, int32_t, count, b.ncells + 1);
  CS_WS_TAKE(w, int, err, 16);
  size_t sb = cs_scan_ws_bytes(b.ncells);
  void *scratch = w.take<char>(sb);
  CS_REQUIRE(scratch, "workspace too small for cell scan");
  CS_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t) * (b.ncells + 1), st));
  CS_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  if (n > 0)
    k_bin_count<<<grid_for(n, 256), 256, 0, st>>>(n, b, x, y, z, cell_of, slot, count, err);
  CS_TRY(cs_exclusive_scan_i32(count, cell_start, b.ncells, scratch, sb, st));
  if (n > 0) {
    k_bin_scatter<<<grid_for(n, 256), 256, 0, st>>>(n, cell_of, slot, cell_start, src);
    k_cell_sort_gather<<<grid_for(b.ncells * 32, 256), 256, 0, st>>>(
        b.ncells, cell_start, src, id, x, y, z, vx, vy, vz, xo, yo, zo, vxo, vyo, vzo, ido, fxo,
        fyo, fzo);
  }
  return cs_check_launch("build_cells");
}

// Range flag of the last cs_build_cells on this workspace: 1 if a particle
// lay outside the local cell range (a slab particle that should have
// migrated, or an unwrapped position) and was clamped into an edge cell.
// Kept out of the build itself so the build never synchronises; reads the
// flag with one device->host copy.
extern "C" int cs_bin_errors(int64_t n, const cs_box *bx, const void *ws, size_t ws_bytes,
                             int *flag_host, void *stream) {
  Box b;
  CS_TRY(make_box(bx, &b));
  cs_ws w(const_cast<void *>(ws), ws_bytes);  // the build's slice layout
  CS_WS_TAKE(w, int32_t, cell_of, n + 1);
  CS_WS_TAKE(w, int32_t, slot, n + 1);
  CS_WS_TAKE(w, int32_t, src, n + 1);
  CS_WS_TAKE(w, int32_t, count, b.ncells + 1);
  CS_WS_TAKE(w, int, err, 16);
  (void)cell_of, (void)slot, (void)src, (void)count;
  cudaStream_t st = cs_stream(stream);
  CS_CUDA(cudaMemcpyAsync(flag_host, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  return CS_OK;
}

// ------------------------------------------------------------ K3: Verlet --
__global__ void k_kick(int64_t n, double hdtm, const double *fx, const double *fy,
                       const double *fz, double *vx, double *vy, double *vz) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    vx[i] = __fma_rn(hdtm, fx[i], vx[i]);
    vy[i] = __fma_rn(hdtm, fy[i], vy[i]);
    vz[i] = __fma_rn(hdtm, fz[i], vz[i]);
  }
}

__global__ void k_kick_drift(int64_t n, double hdtm, double dt, double Lx, double Ly, double Lz,
                             const double *fx, const double *fy, const double *fz, double *vx,
                             double *vy, double *vz, double *x, double *y, double *z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double ux = __fma_rn(hdtm, fx[i], vx[i]);
    double uy = __fma_rn(hdtm, fy[i], vy[i]);
    double uz = __fma_rn(hdtm, fz[i], vz[i]);
    vx[i] = ux;
    vy[i] = uy;
    vz[i] = uz;
    x[i] = wrap_dev(__fma_rn(dt, ux, x[i]), Lx);
    y[i] = wrap_dev(__fma_rn(dt, uy, y[i]), Ly);
    z[i] = wrap_dev(__fma_rn(dt, uz, z[i]), Lz);
  }
}

extern "C" int cs_vv_kick(int64_t n, double hdtm, const double *fx, const double *fy,
                          const double *fz, double *vx, double *vy, double *vz, void *stream) {
  if (n <= 0) return CS_OK;
  k_kick<<<grid_for(n, 256), 256, 0, cs_stream(stream)>>>(n, hdtm, fx, fy, fz, vx, vy, vz);
  return cs_check_launch("vv_kick");
}

extern "C" int cs_vv_kick_drift(int64_t n, double hdtm, double dt, const cs_box *b,
                                const double *fx, const double *fy, const double *fz,
                                double *vx, double *vy, double *vz, double *x, double *y,
                                double *z, void *stream) {
  if (n <= 0) return CS_OK;
  k_kick_drift<<<grid_for(n, 256), 256, 0, cs_stream(stream)>>>(
      n, hdtm, dt, b->L[0], b->L[1], b->L[2], fx, fy, fz, vx, vy, vz, x, y, z);
  return cs_check_launch("vv_kick_drift");
}

// ------------------------------------------------------------ slab halos --
// pack positions of local x-plane `plane` (storage-contiguous in slab mode)
__global__ void k_pack_plane(int64_t lo, int64_t hi, const double *x, const double *y,
                             const double *z, double xshift, double *out) {
  int64_t m = hi - lo;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = __dadd_rn(x[lo + i], xshift);
    out[m + i] = y[lo + i];
    out[2 * m + i] = z[lo + i];
  }
}
__global__ void k_add_plane(int64_t lo, int64_t hi, const double *in, double *fx, double *fy,
                            double *fz) {
  int64_t m = hi - lo;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    fx[lo + i] += in[i];
    fy[lo + i] += in[m + i];
    fz[lo + i] += in[2 * m + i];
  }
}

static int plane_range(const Box &b, int plane, const int32_t *cell_start, int64_t *lo,
                       int64_t *hi, cudaStream_t st) {
  CS_REQUIRE(!b.per[0], "plane packing needs slab (x-slowest) storage");
  CS_REQUIRE(plane >= 0 && plane < b.nc[0], "plane out of range");
  int32_t h[2];
  int64_t c0 = (int64_t)plane * b.stride[0];
  CS_CUDA(cudaMemcpyAsync(&h[0], cell_start + c0, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaMemcpyAsync(&h[1], cell_start + c0 + b.stride[0], sizeof(int32_t),
                          cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  *lo = h[0];
  *hi = h[1];
  return CS_OK;
}

extern "C" int cs_pack_plane(const cs_box *bx, int plane, const int32_t *cell_start,
                             const double *x, const double *y, const double *z, double xshift,
                             double *out, void *stream) {
  Box b;
  CS_TRY(make_box(bx, &b));
  cudaStream_t st = cs_stream(stream);
  int64_t lo, hi;
  CS_TRY(plane_range(b, plane, cell_start, &lo, &hi, st));
  if (hi > lo) k_pack_plane<<<grid_for(hi - lo, 256), 256, 0, st>>>(lo, hi, x, y, z, xshift, out);
  return cs_check_launch("pack_plane");
}

extern "C" int cs_add_plane_forces(const cs_box *bx, int plane, const int32_t *cell_start,
                                   const double *in, double *fx, double *fy, double *fz,
                                   void *stream) {
  Box b;
  CS_TRY(make_box(bx, &b));
  cudaStream_t st = cs_stream(stream);
  int64_t lo, hi;
  CS_TRY(plane_range(b, plane, cell_start, &lo, &hi, st));
  if (hi > lo) k_add_plane<<<grid_for(hi - lo, 256), 256, 0, st>>>(lo, hi, in, fx, fy, fz);
  return cs_check_launch("add_plane_forces");
}

// the same for a known particle range [lo, hi) (no host synchronisation: a
// Verlet slab between rebuilds keeps its plane ranges)
extern "C" int cs_pack_range(int64_t lo, int64_t hi, const double *x, const double *y,
                             const double *z, double xshift, double *out, void *stream) {
  if (hi > lo)
    k_pack_plane<<<grid_for(hi - lo, 256), 256, 0, cs_stream(stream)>>>(lo, hi, x, y, z, xshift, out);
  return cs_check_launch("pack_range");
}

extern "C" int cs_add_range_forces(int64_t lo, int64_t hi, const double *in, double *fx,
                                   double *fy, double *fz, void *stream) {
  if (hi > lo)
    k_add_plane<<<grid_for(hi - lo, 256), 256, 0, cs_stream(stream)>>>(lo, hi, in, fx, fy, fz);
  return cs_check_launch("add_range_forces");
}

// ------------------------------------------------------- slab decomposition --
// Particles are exchanged as packed rows [7][stride] of doubles:
// x, y, z, vx, vy, vz, id (the id is exact in a double).
__global__ void k_slab_code(int64_t n, Box b, const double *x, int32_t *fs, int32_t *fl,
                            int32_t *fr) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int g = bin_coord(x[p], b.inv[0], b.gnc[0]);
    int rel = g - b.x0;  // plane relative to the slab start, periodic in the global box
    if (rel < 0) rel += b.gnc[0];
    if (rel >= b.gnc[0]) rel -= b.gnc[0];
    // owned: [0, owned_x); the right neighbour starts at owned_x; anything in the
    // upper half of the remaining ring belongs to the left side
    int code = 0;
    if (rel >= b.owned_x) code = (rel - b.owned_x) < (b.gnc[0] - b.owned_x + 1) / 2 ? 2 : 1;
    fs[p] = code == 0;
    fl[p] = code == 1;
    fr[p] = code == 2;
  }
}

__global__ void k_slab_scatter(int64_t n, const int32_t *fs, const int32_t *ps, const int32_t *fl,
                               const int32_t *pl, const int32_t *fr, const int32_t *pr,
                               const double *x, const double *y, const double *z,
                               const double *vx, const double *vy, const double *vz,
                               const int32_t *id, double *stay, int64_t sstride, double *left,
                               double *right, int64_t cap) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    double *dst;
    int64_t o, st;
    if (fs[p]) {
      dst = stay; o = ps[p]; st = sstride;
    } else if (fl[p]) {
      dst = left; o = pl[p]; st = cap;
      if (o >= cap) continue;
    } else {
      dst = right; o = pr[p]; st = cap;
      if (o >= cap) continue;
    }
    dst[o] = x[p];
    dst[st + o] = y[p];
    dst[2 * st + o] = z[p];
    dst[3 * st + o] = vx[p];
    dst[4 * st + o] = vy[p];
    dst[5 * st + o] = vz[p];
    dst[6 * st + o] = (double)id[p];
  }
}

extern "C" size_t cs_slab_ws_bytes(int64_t n) {
  return 6 * cs_ws_slice(sizeof(int32_t) * (n + 1)) + cs_scan_ws_bytes(n) + cs_ws_slice(64);
}

extern "C" int cs_slab_split(int64_t n, const cs_box *bx, const double *x, const double *y,
                             const double *z, const double *vx, const double *vy,
                             const double *vz, const int32_t *id, double *stay, int64_t sstride,
                             double *left, double *right, int64_t cap, int64_t *counts_host,
                             void *ws, size_t ws_bytes, void *stream) {
  Box b;
  CS_TRY(make_box(bx, &b));
  cudaStream_t st = cs_stream(stream);
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, fs, n + 1);
  CS_WS_TAKE(w, int32_t, fl, n + 1);
  CS_WS_TAKE(w, int32_t, fr, n + 1);
  CS_WS_TAKE(w, int32_t, ps, n + 1);
  CS_WS_TAKE(w, int32_t, pl, n + 1);
  CS_WS_TAKE(w, int32_t, pr, n + 1);
  size_t sb = cs_scan_ws_bytes(n);
  void *scratch = w.take<char>(sb);
  CS_REQUIRE(scratch, "workspace too small (slab split)");
  if (n > 0) k_slab_code<<<grid_for(n, 256), 256, 0, st>>>(n, b, x, fs, fl, fr);
  CS_TRY(cs_exclusive_scan_i32(fs, ps, n, scratch, sb, st));
  CS_TRY(cs_exclusive_scan_i32(fl, pl, n, scratch, sb, st));
  CS_TRY(cs_exclusive_scan_i32(fr, pr, n, scratch, sb, st));
  if (n > 0)
    k_slab_scatter<<<grid_for(n, 256), 256, 0, st>>>(n, fs, ps, fl, pl, fr, pr, x, y, z, vx, vy,
                                                     vz, id, stay, sstride, left, right, cap);
  int32_t h[3];
  CS_CUDA(cudaMemcpyAsync(&h[0], ps + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaMemcpyAsync(&h[1], pl + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaMemcpyAsync(&h[2], pr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  counts_host[0] = h[0];
  counts_host[1] = h[1];
  counts_host[2] = h[2];
  if (h[1] > cap || h[2] > cap) {
    cs_set_error("slab split: %d/%d migrants exceed the buffer capacity %lld", h[1], h[2],
                 (long long)cap);
    return CS_ECAPACITY;
  }
  return cs_check_launch("slab_split");
}

__global__ void k_unpack7(int64_t m, const double *src, int64_t stride, double *x, double *y,
                          double *z, double *vx, double *vy, double *vz, int32_t *id) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = src[i];
    y[i] = src[stride + i];
    z[i] = src[2 * stride + i];
    vx[i] = src[3 * stride + i];
    vy[i] = src[4 * stride + i];
    vz[i] = src[5 * stride + i];
    id[i] = (int32_t)src[6 * stride + i];
  }
}

extern "C" int cs_unpack7(int64_t m, const double *src, int64_t stride, double *x, double *y,
                          double *z, double *vx, double *vy, double *vz, int32_t *id,
                          void *stream) {
  if (m <= 0) return CS_OK;
  k_unpack7<<<grid_for(m, 256), 256, 0, cs_stream(stream)>>>(m, src, stride, x, y, z, vx, vy, vz, id);
  return cs_check_launch("unpack7");
}

__global__ void k_plane_counts(int64_t c0, int64_t nplane, const int32_t *start, int32_t *cnt) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nplane;
       c += (int64_t)gridDim.x * blockDim.x)
    cnt[c] = start[c0 + c + 1] - start[c0 + c];
}

extern "C" int cs_plane_counts(const cs_box *bx, int plane, const int32_t *cell_start,
                               int32_t *counts, int64_t *range_host, void *stream) {
  Box b;
  CS_TRY(make_box(bx, &b));
  cudaStream_t st = cs_stream(stream);
  int64_t lo, hi;
  CS_TRY(plane_range(b, plane, cell_start, &lo, &hi, st));
  const int64_t c0 = (int64_t)plane * b.stride[0];
  k_plane_counts<<<grid_for(b.stride[0], 256), 256, 0, st>>>(c0, b.stride[0], cell_start, counts);
  range_host[0] = lo;
  range_host[1] = hi;
  return cs_check_launch("plane_counts");
}

__global__ void k_ghost_start(int64_t c0, int64_t nplane, int64_t n_owned, const int32_t *gpos,
                              int32_t *start) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= nplane;
       c += (int64_t)gridDim.x * blockDim.x)
    start[c0 + c] = (int32_t)(n_owned + gpos[c]);
}
__global__ void k_ghost_copy(int64_t m, int64_t n_owned, const double *g, double *x, double *y,
                             double *z, double *fx, double *fy, double *fz) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[n_owned + i] = g[i];
    y[n_owned + i] = g[m + i];
    z[n_owned + i] = g[2 * m + i];
    fx[n_owned + i] = 0.0;
    fy[n_owned + i] = 0.0;
    fz[n_owned + i] = 0.0;
  }
}

extern "C" size_t cs_ghost_ws_bytes(const cs_box *bx) {
  const int64_t np = (int64_t)bx->nc[1] * bx->nc[2];
  return cs_ws_slice(sizeof(int32_t) * (np + 1)) + cs_scan_ws_bytes(np);
}

extern "C" int cs_set_ghost_plane(const cs_box *bx, int64_t n_owned, const int32_t *ghost_counts,
                                  const double *ghost_xyz, int64_t m, int32_t *cell_start,
                                  double *x, double *y, double *z, double *fx, double *fy,
                                  double *fz, void *ws, size_t ws_bytes, void *stream) {
  Box b;
  CS_TRY(make_box(bx, &b));
  CS_REQUIRE(!b.per[0], "ghost planes need slab (x-slowest) storage");
  cudaStream_t st = cs_stream(stream);
  const int64_t np = b.stride[0];
  const int64_t c0 = (int64_t)(b.nc[0] - 1) * np;  // the ghost plane is the last local plane
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, gpos, np + 1);
  size_t sb = cs_scan_ws_bytes(np);
  void *scratch = w.take<char>(sb);
  CS_REQUIRE(scratch, "workspace too small (ghost plane)");
  CS_TRY(cs_exclusive_scan_i32(ghost_counts, gpos, np, scratch, sb, st));
  k_ghost_start<<<grid_for(np + 1, 256), 256, 0, st>>>(c0, np, n_owned, gpos, cell_start);
  if (m > 0)
    k_ghost_copy<<<grid_for(m, 256), 256, 0, st>>>(m, n_owned, ghost_xyz, x, y, z, fx, fy, fz);
  return cs_check_launch("set_ghost_plane");
}
