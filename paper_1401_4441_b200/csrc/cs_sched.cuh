// cs_sched.cuh -- K4: task streams, dependency edges, serialization depth.
//
// Restates on the device (closed form, no Python objects):
//   generate_basic   taskgen.py:180-199  (cell-major, entries in `order`)
//   generate_loopex  taskgen.py:202-234  (entry-major, colours ascending,
//                                         cells x-fastest; stride k general)
//   detect_dependencies + _DependenceState.add  depgraph.py:28-49, :102-117
//   critical_path    depgraph.py:160-174
// For accumulator streams every task writes acc(home) and acc(nbr), so the
// accessors of one cell are closed-form: its own n home tasks plus the
// tasks (r - o_e, e).  Edges come from sorting those <= 2n-1 ids per cell,
// with no global sort and no atomics.
#pragma once
#include "cs_common.cuh"

struct StreamDesc {
  int dim, n, strategy, stride, ncol, all_periodic;
  int ext[3], per[3];
  int8_t off[27][3];  // entry offsets (order for basic, canonical for loopex)
  int colcnt[27][3];  // per colour, cells per axis
  int64_t colstart[28];
  int64_t ncells;
};

static int build_desc(const cs_grid *g, int strategy, const int8_t *order, int n, int stride,
                      StreamDesc *d) {
  CS_REQUIRE(g && (g->dim == 2 || g->dim == 3), "grid must be 2D or 3D");
  memset(d, 0, sizeof(*d));
  d->dim = g->dim;
  d->strategy = strategy;
  d->stride = stride < 1 ? 2 : stride;
  d->ncells = 1;
  d->all_periodic = 1;
  for (int k = 0; k < 3; ++k) {
    d->ext[k] = k < g->dim ? g->ext[k] : 1;
    d->per[k] = k < g->dim ? (g->periodic[k] ? 1 : 0) : 1;
    CS_REQUIRE(d->ext[k] >= 1, "extents must be >= 1");
    d->ncells *= d->ext[k];
    if (k < g->dim && !d->per[k]) d->all_periodic = 0;
  }
  if (strategy == CS_STREAM_BASIC) {
    CS_REQUIRE(order && n >= 1 && n <= 27, "basic stream needs an order of 1..27 entries");
    d->n = n;
    for (int e = 0; e < n; ++e)
      for (int k = 0; k < 3; ++k) {
        int v = k < g->dim ? order[e * g->dim + k] : 0;
        CS_REQUIRE(v >= -1 && v <= 1, "offset components must be in {-1,0,1}");
        d->off[e][k] = (int8_t)v;
      }
  } else if (strategy == CS_STREAM_LOOPEX) {
    int8_t st[27 * 3];
    int m;
    cs_host_canonical_stencil(g->dim, st, &m);
    d->n = m;
    for (int e = 0; e < m; ++e)
      for (int k = 0; k < 3; ++k) d->off[e][k] = k < g->dim ? st[e * g->dim + k] : 0;
    int s = d->stride;
    int ncol = 1;
    for (int k = 0; k < g->dim; ++k) ncol *= s;
    CS_REQUIRE(ncol <= 27, "colour stride too large");
    d->ncol = ncol;
    d->colstart[0] = 0;
    for (int col = 0; col < ncol; ++col) {
      int rem = col;
      int64_t size = 1;
      for (int k = 0; k < 3; ++k) {
        int digit = 0;
        if (k < g->dim) {
          digit = rem % s;
          rem /= s;
        }
        int cnt = k < g->dim ? (digit < d->ext[k] ? (d->ext[k] - digit + s - 1) / s : 0) : 1;
        d->colcnt[col][k] = cnt;
        size *= cnt;
      }
      d->colstart[col + 1] = d->colstart[col] + size;
    }
  } else {
    CS_REQUIRE(0, "unknown strategy %d", strategy);
  }
  return CS_OK;
}

__host__ __device__ __forceinline__ void desc_coords(const StreamDesc &d, int64_t cell, int *c) {
  c[0] = (int)(cell % d.ext[0]);
  int64_t r = cell / d.ext[0];
  c[1] = (int)(r % d.ext[1]);
  c[2] = (int)(r / d.ext[1]);
}
__host__ __device__ __forceinline__ int64_t desc_index(const StreamDesc &d, const int *c) {
  return c[0] + (int64_t)d.ext[0] * (c[1] + (int64_t)d.ext[1] * c[2]);
}
// neighbour of cell along entry e (-1: dropped; intra returns the cell)
__host__ __device__ __forceinline__ int64_t desc_nbr(const StreamDesc &d, int64_t cell, int e) {
  int c[3];
  desc_coords(d, cell, c);
  for (int k = 0; k < 3; ++k) {
    int s = c[k] + d.off[e][k];
    if (d.per[k]) {
      s = cs_wrap(s, d.ext[k]);
    } else if (s < 0 || s >= d.ext[k]) {
      return -1;
    }
    c[k] = s;
  }
  return desc_index(d, c);
}
__host__ __device__ __forceinline__ bool desc_is_intra(const StreamDesc &d, int e) {
  return d.off[e][0] == 0 && d.off[e][1] == 0 && d.off[e][2] == 0;
}
// colour of a cell and its rank in cells_by_color concatenation (grid.py:136-141)
__host__ __device__ __forceinline__ int64_t desc_colour_rank(const StreamDesc &d, int64_t cell) {
  int c[3];
  desc_coords(d, cell, c);
  int s = d.stride, col = 0, mul = 1;
  int i[3];
  for (int k = 0; k < 3; ++k) {
    int digit = k < d.dim ? c[k] % s : 0;
    i[k] = k < d.dim ? c[k] / s : 0;
    if (k < d.dim) {
      col += digit * mul;
      mul *= s;
    }
  }
  return d.colstart[col] + i[0] + (int64_t)d.colcnt[col][0] * (i[1] + (int64_t)d.colcnt[col][1] * i[2]);
}
__host__ __device__ __forceinline__ int64_t desc_cell_of_rank(const StreamDesc &d, int64_t r) {
  int col = 0;
  while (col + 1 < d.ncol && d.colstart[col + 1] <= r) ++col;
  int64_t i = r - d.colstart[col];
  int s = d.stride, rem = col;
  int c[3];
  int64_t cnt0 = d.colcnt[col][0], cnt1 = d.colcnt[col][1];
  int64_t ii[3] = {i % cnt0, (i / cnt0) % cnt1, i / (cnt0 * cnt1)};
  for (int k = 0; k < 3; ++k) {
    int digit = 0;
    if (k < d.dim) {
      digit = rem % s;
      rem /= s;
    }
    c[k] = k < d.dim ? (int)(s * ii[k] + digit) : 0;
  }
  return desc_index(d, c);
}
// candidate index (before truncation) of task (cell, e)
__host__ __device__ __forceinline__ int64_t desc_cand(const StreamDesc &d, int64_t cell, int e) {
  if (d.strategy == CS_STREAM_BASIC) return cell * d.n + e;
  return (int64_t)e * d.ncells + desc_colour_rank(d, cell);
}
__host__ __device__ __forceinline__ void desc_uncand(const StreamDesc &d, int64_t cand,
                                                     int64_t *cell, int *e) {
  if (d.strategy == CS_STREAM_BASIC) {
    *cell = cand / d.n;
    *e = (int)(cand % d.n);
  } else {
    *e = (int)(cand / d.ncells);
    *cell = desc_cell_of_rank(d, cand % d.ncells);
  }
}

// ------------------------------------------------------------- generation --
__global__ void k_stream_flags(StreamDesc d, int32_t *flag) {
  int64_t ncand = d.ncells * d.n;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncand;
       c += (int64_t)gridDim.x * blockDim.x) {
    int64_t cell;
    int e;
    desc_uncand(d, c, &cell, &e);
    flag[c] = (desc_is_intra(d, e) || desc_nbr(d, cell, e) >= 0) ? 1 : 0;
  }
}

__global__ void k_stream_write(StreamDesc d, const int32_t *pos, int32_t *home, int32_t *nbr,
                               int16_t *entry) {
  int64_t ncand = d.ncells * d.n;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncand;
       c += (int64_t)gridDim.x * blockDim.x) {
    int64_t cell;
    int e;
    desc_uncand(d, c, &cell, &e);
    int64_t nb = desc_is_intra(d, e) ? -1 : desc_nbr(d, cell, e);
    if (!desc_is_intra(d, e) && nb < 0) continue;
    int64_t t = pos ? pos[c] : c;
    home[t] = (int32_t)cell;
    nbr[t] = (int32_t)nb;
    entry[t] = (int16_t)e;
  }
}

static int64_t host_stream_count(const StreamDesc &d) {
  int64_t total = 0;
  for (int e = 0; e < d.n; ++e) {
    int64_t cnt = 1;
    for (int k = 0; k < 3; ++k) {
      int o = d.off[e][k] < 0 ? -d.off[e][k] : d.off[e][k];
      int64_t m = d.per[k] ? d.ext[k] : (d.ext[k] - o > 0 ? d.ext[k] - o : 0);
      cnt *= m;
    }
    total += cnt;
  }
  return total;
}

static unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 64) b = 148 * 64;
  if (b < 1) b = 1;
  return (unsigned)b;
}

extern "C" int64_t cs_stream_count(const cs_grid *g, int strategy, const int8_t *order, int n,
                                   int stride) {
  StreamDesc d;
  if (build_desc(g, strategy, order, n, stride, &d) != CS_OK) return -1;
  return host_stream_count(d);
}

extern "C" size_t cs_stream_ws_bytes(const cs_grid *g, int n) {
  int64_t nc = 1;
  for (int k = 0; k < g->dim; ++k) nc *= g->ext[k];
  int64_t ncand = nc * (n > 0 ? n : 27);
  return 2 * cs_ws_slice(sizeof(int32_t) * (ncand + 1)) + cs_scan_ws_bytes(ncand);
}

// candidate -> task position map for truncated (non-periodic) streams
static int stream_positions(const StreamDesc &d, cs_ws &w, int32_t **pos_out, cudaStream_t st) {
  int64_t ncand = d.ncells * d.n;
  CS_WS_TAKE(w, int32_t, flag, ncand + 1);
  CS_WS_TAKE(w, int32_t, pos, ncand + 1);
  size_t sb = cs_scan_ws_bytes(ncand);
  void *scratch = w.take<char>(sb);
  if (!scratch) {
    cs_set_error("workspace too small for stream scan");
    return CS_ECAPACITY;
  }
  k_stream_flags<<<grid_for(ncand, 256), 256, 0, st>>>(d, flag);
  CS_TRY(cs_exclusive_scan_i32(flag, pos, ncand, scratch, sb, st));
  *pos_out = pos;
  return cs_check_launch("stream_flags");
}

extern "C" int cs_stream_generate(const cs_grid *g, int strategy, const int8_t *order, int n,
                                  int stride, int32_t *home, int32_t *nbr, int16_t *entry,
                                  int64_t ntasks, void *ws, size_t ws_bytes, void *stream) {
  StreamDesc d;
  CS_TRY(build_desc(g, strategy, order, n, stride, &d));
  CS_REQUIRE(ntasks == host_stream_count(d), "ntasks mismatch (expected %lld)",
             (long long)host_stream_count(d));
  cudaStream_t st = cs_stream(stream);
  if (ntasks == 0) return CS_OK;
  int32_t *pos = nullptr;
  cs_ws w(ws, ws_bytes);
  if (!d.all_periodic) CS_TRY(stream_positions(d, w, &pos, st));
  k_stream_write<<<grid_for(d.ncells * d.n, 256), 256, 0, st>>>(d, pos, home, nbr, entry);
  return cs_check_launch("stream_write");
}

// ------------------------------------------------------------------ edges --
// One thread per resource (cell): gather its accessor task ids, sort, and
// hand each accessor its predecessor through this resource.
__global__ void k_stream_edges(StreamDesc d, const int32_t *pos, const int32_t *home,
                               int32_t *pred_home, int32_t *pred_nbr) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < d.ncells;
       r += (int64_t)gridDim.x * blockDim.x) {
    int32_t acc[54];
    int m = 0;
    for (int e = 0; e < d.n; ++e) {
      bool intra = desc_is_intra(d, e);
      // as home
      if (intra || desc_nbr(d, r, e) >= 0) {
        int64_t c = desc_cand(d, r, e);
        acc[m++] = pos ? pos[c] : (int32_t)c;
      }
      if (intra) continue;
      // as neighbour: home cell r - o_e (exists iff (r - o_e) + o_e == r)
      int c3[3];
      desc_coords(d, r, c3);
      bool ok = true;
      for (int k = 0; k < 3; ++k) {
        int s = c3[k] - d.off[e][k];
        if (d.per[k])
          s = cs_wrap(s, d.ext[k]);
        else if (s < 0 || s >= d.ext[k])
          ok = false;
        c3[k] = s;
      }
      if (!ok) continue;
      int64_t h = desc_index(d, c3);
      int64_t c = desc_cand(d, h, e);
      acc[m++] = pos ? pos[c] : (int32_t)c;
    }
    // insertion sort (m <= 2n-1 <= 53), drop duplicates (self-neighbour)
    for (int a = 1; a < m; ++a) {
      int32_t v = acc[a];
      int b = a - 1;
      while (b >= 0 && acc[b] > v) {
        acc[b + 1] = acc[b];
        --b;
      }
      acc[b + 1] = v;
    }
    int32_t prev = -1;
    for (int a = 0; a < m; ++a) {
      int32_t t = acc[a];
      if (t == prev) continue;
      if (home[t] == r)
        pred_home[t] = prev;
      else
        pred_nbr[t] = prev;
      prev = t;
    }
  }
}

// order the (<= 2) preds of each task: pred_a < pred_b, duplicates removed
__global__ void k_pred_finish(int64_t nt, const int32_t *nbr, const int32_t *home,
                              int32_t *pa, int32_t *pb, unsigned long long *count) {
  unsigned long long local = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x) {
    int32_t a = pa[t];
    int32_t b = (nbr[t] >= 0 && nbr[t] != home[t]) ? pb[t] : -1;
    if (a == b) b = -1;
    if (a < 0) {
      a = b;
      b = -1;
    }
    if (b >= 0 && b < a) {
      int32_t x = a;
      a = b;
      b = x;
    }
    pa[t] = a;
    pb[t] = b;
    local += (a >= 0) + (b >= 0);
  }
  local = warp_sum(local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

extern "C" size_t cs_edges_ws_bytes(const cs_grid *g, int n, int64_t ntasks) {
  return cs_stream_ws_bytes(g, n) + cs_ws_slice(sizeof(unsigned long long)) +
         cs_ws_slice(sizeof(int32_t) * (ntasks + 1)) + cs_scan_ws_bytes(ntasks);
}

extern "C" int cs_stream_edges(const cs_grid *g, int strategy, const int8_t *order, int n,
                               int stride, const int32_t *home, const int32_t *nbr,
                               int64_t ntasks, int32_t *pred_a, int32_t *pred_b,
                               int64_t *nedges_host, void *ws, size_t ws_bytes, void *stream) {
  StreamDesc d;
  CS_TRY(build_desc(g, strategy, order, n, stride, &d));
  CS_REQUIRE(ntasks == host_stream_count(d), "ntasks mismatch");
  cudaStream_t st = cs_stream(stream);
  cs_ws w(ws, ws_bytes);
  int32_t *pos = nullptr;
  if (!d.all_periodic) CS_TRY(stream_positions(d, w, &pos, st));
  CS_WS_TAKE(w, unsigned long long, cnt, 1);
  CS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
  CS_CUDA(cudaMemsetAsync(pred_a, 0xff, sizeof(int32_t) * ntasks, st));
  CS_CUDA(cudaMemsetAsync(pred_b, 0xff, sizeof(int32_t) * ntasks, st));
  k_stream_edges<<<grid_for(d.ncells, 128), 128, 0, st>>>(d, pos, home, pred_a, pred_b);
  k_pred_finish<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, nbr, home, pred_a, pred_b, cnt);
  CS_TRY(cs_check_launch("stream_edges"));
  unsigned long long h = 0;
  CS_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  *nedges_host = (int64_t)h;
  return CS_OK;
}

__global__ void k_edge_counts(int64_t nt, const int32_t *pa, const int32_t *pb, int32_t *cnt) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x)
    cnt[t] = (pa[t] >= 0) + (pb[t] >= 0);
}
__global__ void k_edge_write(int64_t nt, const int32_t *pa, const int32_t *pb, const int32_t *off,
                             int64_t *eu, int64_t *ev) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = off[t];
    if (pa[t] >= 0) {
      eu[o] = pa[t];
      ev[o] = t;
      ++o;
    }
    if (pb[t] >= 0) {
      eu[o] = pb[t];
      ev[o] = t;
    }
  }
}

extern "C" int cs_edges_compact(int64_t ntasks, const int32_t *pa, const int32_t *pb,
                                int64_t *eu, int64_t *ev, void *ws, size_t ws_bytes,
                                void *stream) {
  cudaStream_t st = cs_stream(stream);
  if (ntasks == 0) return CS_OK;
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, cnt, ntasks + 1);
  CS_WS_TAKE(w, int32_t, off, ntasks + 1);
  size_t sb = cs_scan_ws_bytes(ntasks);
  void *scratch = w.take<char>(sb);
  CS_REQUIRE(scratch, "workspace too small for edge scan");
  k_edge_counts<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, pa, pb, cnt);
  CS_TRY(cs_exclusive_scan_i32(cnt, off, ntasks, scratch, sb, st));
  k_edge_write<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, pa, pb, off, eu, ev);
  return cs_check_launch("edges_compact");
}

// ------------------------------------------------------------------ depth --
// (a) relaxation: level[t] = 1 + max(level[pred]); monotone, converges in
//     <= depth sweeps.  Used for shallow (colour) orders.
__global__ void k_depth_relax(int64_t nt, const int32_t *pa, const int32_t *pb, int32_t *level,
                              int *changed) {
  int any = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x) {
    int32_t L = 1;
    if (pa[t] >= 0) L = max(L, level[pa[t]] + 1);
    if (pb[t] >= 0) L = max(L, level[pb[t]] + 1);
    if (L > level[t]) {
      level[t] = L;
      any = 1;
    }
  }
  if (__any_sync(CS_FULL, any) && (threadIdx.x & 31) == 0) *changed = 1;
}

// (b) cell-chain DP for cell-grouped streams (generate_basic): one warp
//     walks the cells in creation order; the state vector s[r] = level of
//     the last accessor of resource r replaces the edge list.
//     Lanes hold the cell's entries; the 1..n task chain runs in registers.
__global__ void k_depth_chain(int64_t ncells, const int32_t *first, const int32_t *home,
                              const int32_t *nbr, int32_t *s, int32_t *level, int32_t *depth) {
  int lane = threadIdx.x & 31;
  int32_t best = 0;
  for (int64_t c = 0; c < ncells; ++c) {
    int32_t t0 = first[c], k = first[c + 1] - t0;
    // k <= 27 <= 32 (entries of one cell)
    int32_t nb = -1, sv = 0;
    if (lane < k) {
      nb = nbr[t0 + lane];
      if (nb == (int32_t)c) nb = -1;
      if (nb >= 0) sv = s[nb];
    }
    int32_t cur = s[c], myL = 0;
    for (int e = 0; e < k; ++e) {
      int32_t nbe = __shfl_sync(CS_FULL, nb, e);
      int32_t ve = __shfl_sync(CS_FULL, sv, e);
      int32_t L = 1 + max(cur, nbe >= 0 ? ve : 0);
      cur = L;
      if (lane == e) myL = L;
      if (nbe >= 0 && nb == nbe) sv = L;
    }
    if (lane < k) {
      level[t0 + lane] = myL;
      if (nb >= 0) s[nb] = sv;
    }
    __syncwarp();
    if (lane == 0) s[c] = cur;
    best = max(best, cur);
    __syncwarp();
    // a neighbour state written by one lane must be visible to all lanes
    __threadfence_block();
  }
  if (lane == 0) *depth = best;
  (void)home;
}

// (c) the same DP for a fully periodic cell-grouped stream, with the state
//     vector in shared memory.  Cells are visited plane by plane along the
//     slowest axis; a cell's tasks touch only planes z-1, z, z+1, so a ring
//     of three planes (slot q % 3) plus a fixed slot for the last plane (the
//     periodic image of plane -1) holds every live state.  Plane 0 is parked
//     in global memory when it leaves the ring and brought back for the last
//     plane (its +1 neighbour).  Per cell, lanes hold the tasks in stream
//     order and the chain L_e = 1 + max(L_{e-1}, s[n_e]) is evaluated in
//     closed form, L_e = e + 1 + max(s[home], max_{k<=e}(s[n_k] - k)), by one
//     warp prefix-max; the entry offsets come from cell 0's neighbours.
//     Requires every extent >= 3 (distinct neighbours within a cell).
__global__ void __launch_bounds__(32) k_depth_planes(int ex, int ey, int ez, int n,
                                                     const int32_t *nbr, int32_t *level,
                                                     int32_t *parked, int32_t *depth) {
  extern __shared__ int32_t win[];  // 4 slots of ex * ey states
  const int lane = threadIdx.x;
  const int P = ex * ey;
  // entry offsets from cell 0's tasks (nbr = -1 or 0: intra)
  int ox = 0, oy = 0, oz = 0;
  bool inter = false;
  if (lane < n) {
    const int nb = nbr[lane];
    if (nb > 0) {
      inter = true;
      const int nx = nb % ex, ny = (nb / ex) % ey, nz = nb / P;
      ox = nx == 0 ? 0 : (nx == 1 ? 1 : -1);
      oy = ny == 0 ? 0 : (ny == 1 ? 1 : -1);
      oz = nz == 0 ? 0 : (nz == 1 ? 1 : -1);
    }
  }
  for (int i = lane; i < 4 * P; i += 32) win[i] = 0;
  bool parked0 = false;
  int32_t best = 0;
  int64_t c = 0;
  __syncwarp();
  for (int z = 0; z < ez; ++z) {
    const int q = z + 1;  // plane entering the ring
    if (z >= 1 && q <= ez - 2 && q >= 3) {
      int32_t *slot = win + (q % 3) * P;  // held plane q - 3 = z - 2
      if (z - 2 == 0) {
        for (int i = lane; i < P; i += 32) parked[i] = slot[i];
        parked0 = true;
      }
      for (int i = lane; i < P; i += 32) slot[i] = 0;
    }
    if (z == ez - 1 && parked0) {
      int32_t *slot = win + (ez % 3) * P;
      for (int i = lane; i < P; i += 32) slot[i] = parked[i];
    }
    __syncwarp();
    // slot of plane z + oz for this lane's entry
    const int pz = z + oz < 0 ? ez - 1 : (z + oz >= ez ? 0 : z + oz);
    const int sl = pz == ez - 1 ? 3 : ((pz == 0 && z == ez - 1 && parked0) ? ez % 3 : pz % 3);
    int32_t *base = win + sl * P;
    int32_t *hbase = win + (z == ez - 1 ? 3 : z % 3) * P;
    for (int y = 0; y < ey; ++y) {
      int ny = y + oy;
      ny = ny < 0 ? ny + ey : (ny >= ey ? ny - ey : ny);
      const int rowo = ex * ny;
      for (int x = 0; x < ex; ++x, ++c) {
        int nx = x + ox;
        nx = nx < 0 ? nx + ex : (nx >= ex ? nx - ex : nx);
        const int a = rowo + nx;
        const int32_t sh = hbase[x + ex * y];
        int32_t w = inter ? base[a] - lane : INT32_MIN / 2;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          if (d >= n) break;
          const int32_t u = __shfl_up_sync(CS_FULL, w, d);
          if (lane >= d) w = max(w, u);
        }
        const int32_t L = lane + 1 + max(sh, w);
        if (lane < n) {
          level[c * n + lane] = L;
          if (inter) base[a] = L;
          if (lane == n - 1) {
            hbase[x + ex * y] = L;
            best = max(best, L);
          }
        }
        __syncwarp();
      }
    }
  }
  best = max(best, __shfl_sync(CS_FULL, best, n - 1));
  if (lane == 0) *depth = best;
}

__global__ void k_cell_first_from_home(int64_t nt, const int32_t *home, int64_t ncells,
                                       int32_t *first) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x) {
    int32_t h = home[t];
    if (t == 0 || home[t - 1] != h) first[h] = (int32_t)t;
    if (t == nt - 1) first[ncells] = (int32_t)nt;
  }
}

__global__ void k_max_i32(int64_t n, const int32_t *v, int32_t *out) {
  int32_t m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(CS_FULL, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_fill_i32(int64_t n, int32_t *v, int32_t x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = x;
}

extern "C" size_t cs_depth_ws_bytes(int64_t ntasks) {
  // chain method: first[] + s[] sized by cells <= ntasks
  return 2 * cs_ws_slice(sizeof(int32_t) * (ntasks + 2)) + cs_ws_slice(64);
}

extern "C" int cs_stream_depth(const cs_grid *g, int strategy, int n, int64_t ntasks,
                               const int32_t *home, const int32_t *nbr, const int32_t *pa,
                               const int32_t *pb, int32_t *level, int method,
                               int64_t *depth_host, void *ws, size_t ws_bytes, void *stream) {
  cudaStream_t st = cs_stream(stream);
  (void)n;
  if (ntasks == 0) {
    *depth_host = 0;  // depgraph.py:165-166
    return CS_OK;
  }
  int64_t ncells = 1;
  for (int k = 0; k < g->dim; ++k) ncells *= g->ext[k];
  if (method == 2) method = strategy == CS_STREAM_BASIC ? 1 : 0;
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, scalars, 16);
  // plane-ring fast path: fully periodic, every extent >= 3, <= 32 entries
  // per cell, every cell complete, four planes of states in shared memory
  int e3[3] = {g->ext[0], g->dim == 3 ? g->ext[1] : 1, g->ext[g->dim - 1]};
  bool ring = method == 1 && strategy == CS_STREAM_BASIC && (g->dim == 2 || g->dim == 3);
  for (int k = 0; k < g->dim; ++k) ring = ring && g->periodic[k] && g->ext[k] >= 3;
  const int nper = ncells > 0 ? (int)(ntasks / ncells) : 0;
  ring = ring && nper >= 1 && nper <= 32 && (int64_t)nper * ncells == ntasks;
  const size_t ring_smem = 4 * sizeof(int32_t) * (size_t)e3[0] * e3[1];
  ring = ring && ring_smem <= 200 * 1024;
  if (ring) {
    CS_WS_TAKE(w, int32_t, parked, (int64_t)e3[0] * e3[1]);
    static bool attr[CS_MAX_DEVICES];
    const int dev = cs_device_index();
    if (!attr[dev]) {
      CS_CUDA(cudaFuncSetAttribute(k_depth_planes, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr[dev] = true;
    }
    k_depth_planes<<<1, 32, ring_smem, st>>>(e3[0], e3[1], e3[2], nper, nbr, level, parked, scalars);
    CS_TRY(cs_check_launch("depth_planes"));
  } else if (method == 1) {
    CS_REQUIRE(strategy == CS_STREAM_BASIC, "chain depth needs a cell-grouped (basic) stream");
    CS_WS_TAKE(w, int32_t, first, ncells + 1);
    CS_WS_TAKE(w, int32_t, s, ncells);
    // cells with no task keep first[c] = first[c+1]: fill with ntasks then
    // min-propagate is unnecessary for periodic/ordered streams where every
    // cell has its intra task (basic streams always do).
    k_cell_first_from_home<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, home, ncells, first);
    CS_CUDA(cudaMemsetAsync(s, 0, sizeof(int32_t) * ncells, st));
    k_depth_chain<<<1, 32, 0, st>>>(ncells, first, home, nbr, s, level, scalars);
    CS_TRY(cs_check_launch("depth_chain"));
  } else {
    k_fill_i32<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, level, 1);
    int *changed = (int *)(scalars + 4);
    int h = 1;
    int64_t iters = 0;
    while (h) {
      CS_CUDA(cudaMemsetAsync(changed, 0, sizeof(int), st));
      k_depth_relax<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, pa, pb, level, changed);
      CS_TRY(cs_check_launch("depth_relax"));
      CS_CUDA(cudaMemcpyAsync(&h, changed, sizeof(int), cudaMemcpyDeviceToHost, st));
      CS_CUDA(cudaStreamSynchronize(st));
      if (++iters > ntasks + 1) {
        cs_set_error("depth relaxation did not converge (cycle?)");
        return CS_ECYCLE;
      }
    }
    CS_CUDA(cudaMemsetAsync(scalars, 0, sizeof(int32_t), st));
    k_max_i32<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, level, scalars);
    CS_TRY(cs_check_launch("depth_max"));
  }
  int32_t dh = 0;
  CS_CUDA(cudaMemcpyAsync(&dh, scalars, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  *depth_host = dh;
  return CS_OK;
}
