// cs_generic.cuh -- K4 for arbitrary task lists: the reference's full
// _DependenceState rule (depgraph.py:28-49) with read-only inputs, the
// longest path (depgraph.py:160-174) and level-by-level payload execution
// (apply_tasks with buffer slots and reduce tasks, payload.py:84-119).
//
// Accesses arrive in stream order (task-major; inside a task the reads come
// before the writes, as add() processes them; a read of a resource the task
// also writes is dropped by the host, the "inout wins" rule).  A stable LSD
// radix sort groups them by resource, one thread walks each resource's
// accessor sequence:
//   read  -> predecessor = last writer
//   write -> predecessors = the readers since the last write, else the last writer
// Per task the predecessor lists are merged, sorted, de-duplicated (self
// edges dropped) and emitted sorted by (succ, pred).
#pragma once
#include "cs_common.cuh"
#include "cs_payload.cuh"

__global__ void k_fill_iota_i32(int64_t n, int32_t *v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

#define RX_THREADS 256
#define RX_ITEMS 4
#define RX_TILE (RX_THREADS * RX_ITEMS)

__global__ void k_radix_hist(int64_t n, const int32_t *key, int shift, int32_t *hist,
                             int64_t ntiles) {
  __shared__ int32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RX_TILE;
  for (int r = 0; r < RX_ITEMS; ++r) {
    const int64_t i = base + r * RX_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[(key[i] >> shift) & 255], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// stable scatter: items of a tile keep their order within a digit
__global__ void k_radix_scatter(int64_t n, const int32_t *key, const int32_t *val, int shift,
                                const int32_t *off, int64_t ntiles, int32_t *key_out,
                                int32_t *val_out) {
  __shared__ int32_t wcnt[RX_THREADS / 32][256];
  __shared__ int32_t carry[256];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  carry[threadIdx.x] = off[(int64_t)threadIdx.x * ntiles + blockIdx.x];
  const int64_t base = (int64_t)blockIdx.x * RX_TILE;
  for (int r = 0; r < RX_ITEMS; ++r) {
    for (int w = 0; w < RX_THREADS / 32; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = base + r * RX_THREADS + threadIdx.x;
    const bool v = i < n;
    const int d = v ? (key[i] >> shift) & 255 : 256 + lane;  // invalid lanes: unique
    const unsigned peers = __match_any_sync(CS_FULL, d);
    const int rank = __popc(peers & ((1u << lane) - 1));
    if (v && rank == 0) wcnt[wid][d] = __popc(peers);
    __syncthreads();
    {  // digit t: exclusive prefix over warps, continuing the carry
      int run = carry[threadIdx.x];
      for (int w = 0; w < RX_THREADS / 32; ++w) {
        const int c = wcnt[w][threadIdx.x];
        wcnt[w][threadIdx.x] = run;
        run += c;
      }
      carry[threadIdx.x] = run;
    }
    __syncthreads();
    if (v) {
      const int pos = wcnt[wid][d] + rank;
      key_out[pos] = key[i];
      val_out[pos] = val[i];
    }
    __syncthreads();
  }
}

// one thread per resource segment of the sorted accesses
__global__ void k_seg_heads(int64_t n, const int32_t *skey, int32_t *flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || skey[i] != skey[i - 1]) ? 1 : 0;
}
__global__ void k_seg_compact(int64_t n, const int32_t *flag, const int32_t *pos, int32_t *heads,
                              int64_t nseg_max) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) heads[pos[i]] = (int32_t)i;
  (void)nseg_max;
}

// EMIT = false: count predecessors per access; true: write their task ids
template <bool EMIT>
__global__ void k_seg_walk(int64_t nseg, int64_t n, const int32_t *heads, const int32_t *sval,
                           const int32_t *acc_task, const uint8_t *acc_write, int32_t *cnt,
                           const int32_t *poff, int32_t *preds) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = heads[s], hi = (s + 1 < nseg) ? heads[s + 1] : n;
    int64_t last_w = -1, rs = lo;  // readers since the last write: sorted positions [rs, p)
    for (int64_t p = lo; p < hi; ++p) {
      const int32_t a = sval[p];
      if (acc_write[a]) {
        if (p > rs) {  // readers since the last write
          if (EMIT)
            for (int64_t q = rs; q < p; ++q) preds[poff[a] + (q - rs)] = acc_task[sval[q]];
          else
            cnt[a] = (int32_t)(p - rs);
        } else {
          if (EMIT) {
            if (last_w >= 0) preds[poff[a]] = acc_task[sval[last_w]];
          } else {
            cnt[a] = last_w >= 0 ? 1 : 0;
          }
        }
        last_w = p;
        rs = p + 1;
      } else {
        if (EMIT) {
          if (last_w >= 0) preds[poff[a]] = acc_task[sval[last_w]];
        } else {
          cnt[a] = last_w >= 0 ? 1 : 0;
        }
      }
    }
  }
}

// per task: sort (shell sort) + dedupe + drop self; ecnt[t] = distinct preds
__global__ void k_task_preds(int64_t ntasks, const int64_t *tptr, const int32_t *poff,
                             int32_t *preds, int32_t *ecnt) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntasks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = poff[tptr[t]], hi = poff[tptr[t + 1]];
    const int64_t k = hi - lo;
    int32_t *p = preds + lo;
    for (int64_t gap = k / 2; gap > 0; gap /= 2)
      for (int64_t i = gap; i < k; ++i) {
        const int32_t v = p[i];
        int64_t j = i;
        while (j >= gap && p[j - gap] > v) {
          p[j] = p[j - gap];
          j -= gap;
        }
        p[j] = v;
      }
    int32_t m = 0, prev = -1;
    for (int64_t i = 0; i < k; ++i) {
      const int32_t v = p[i];
      if (v == prev || v == (int32_t)t) continue;
      p[m++] = v;
      prev = v;
    }
    ecnt[t] = m;
  }
}

__global__ void k_task_emit(int64_t ntasks, const int64_t *tptr, const int32_t *poff,
                            const int32_t *preds, const int32_t *eoff, int64_t *eu, int64_t *ev) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntasks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = poff[tptr[t]];
    const int32_t m = eoff[t + 1] - eoff[t];
    for (int32_t i = 0; i < m; ++i) {
      eu[eoff[t] + i] = preds[lo + i];
      ev[eoff[t] + i] = t;
    }
  }
}

struct GenericWs {
  int32_t *k0, *v0, *k1, *v1, *hist, *flag, *fpos, *heads, *cnt, *poff, *preds, *ecnt, *eoff;
  void *scan;
  size_t scan_bytes;
};

static int64_t rx_tiles(int64_t n) { return (n + RX_TILE - 1) / RX_TILE; }

extern "C" size_t cs_detect_ws_bytes(int64_t ntasks, int64_t nacc, int64_t npred_max) {
  const int64_t nt = rx_tiles(nacc) + 1;
  int64_t scan_n = 256 * nt;
  if (nacc + 1 > scan_n) scan_n = nacc + 1;
  if (ntasks + 1 > scan_n) scan_n = ntasks + 1;
  return 4 * cs_ws_slice(sizeof(int32_t) * (nacc + 1)) + cs_ws_slice(sizeof(int32_t) * 256 * nt + 8) +
         2 * cs_ws_slice(sizeof(int32_t) * (nacc + 1)) /*flag,fpos*/ +
         cs_ws_slice(sizeof(int32_t) * (nacc + 1)) /*heads*/ +
         2 * cs_ws_slice(sizeof(int32_t) * (nacc + 2)) /*cnt,poff*/ +
         cs_ws_slice(sizeof(int32_t) * (npred_max + 1)) + 2 * cs_ws_slice(sizeof(int32_t) * (ntasks + 2)) +
         cs_scan_ws_bytes(scan_n) + 512;
}

/* Pass 1: predecessors of every task, kept in the workspace; returns the
 * distinct edge count.  npred_max bounds the raw (pre-dedupe) predecessor
 * total; the host passes a safe bound and gets CS_ECAPACITY otherwise. */
extern "C" int cs_detect_generic(int64_t ntasks, int64_t nacc, int64_t nres,
                                 const int64_t *tptr, const int32_t *acc_task,
                                 const int32_t *acc_res, const uint8_t *acc_write,
                                 int64_t npred_max, int64_t *nedges_host, void *ws,
                                 size_t ws_bytes, void *stream) {
  cudaStream_t st = cs_stream(stream);
  cs_ws w(ws, ws_bytes);
  const int64_t nt = rx_tiles(nacc) + 1;
  CS_WS_TAKE(w, int32_t, k0, nacc + 1);
  CS_WS_TAKE(w, int32_t, v0, nacc + 1);
  CS_WS_TAKE(w, int32_t, k1, nacc + 1);
  CS_WS_TAKE(w, int32_t, v1, nacc + 1);
  CS_WS_TAKE(w, int32_t, hist, 256 * nt + 2);
  CS_WS_TAKE(w, int32_t, flag, nacc + 1);
  CS_WS_TAKE(w, int32_t, fpos, nacc + 1);
  CS_WS_TAKE(w, int32_t, heads, nacc + 1);
  CS_WS_TAKE(w, int32_t, cnt, nacc + 2);
  CS_WS_TAKE(w, int32_t, poff, nacc + 2);
  CS_WS_TAKE(w, int32_t, preds, npred_max + 1);
  CS_WS_TAKE(w, int32_t, ecnt, ntasks + 2);
  CS_WS_TAKE(w, int32_t, eoff, ntasks + 2);
  int64_t scan_n = 256 * nt;
  if (nacc + 1 > scan_n) scan_n = nacc + 1;
  if (ntasks + 1 > scan_n) scan_n = ntasks + 1;
  const size_t sb = cs_scan_ws_bytes(scan_n);
  void *scratch = w.take<char>(sb);
  CS_REQUIRE(scratch, "workspace too small (generic detect)");
  if (ntasks == 0 || nacc == 0) {
    *nedges_host = 0;
    CS_CUDA(cudaMemsetAsync(eoff, 0, sizeof(int32_t) * (ntasks + 2), st));
    return CS_OK;
  }
  // stable LSD radix sort of access indices by resource
  CS_CUDA(cudaMemcpyAsync(k0, acc_res, sizeof(int32_t) * nacc, cudaMemcpyDeviceToDevice, st));
  k_fill_iota_i32<<<grid_for(nacc, 256), 256, 0, st>>>(nacc, v0);
  int bits = 1;
  while ((1ll << bits) < nres) ++bits;
  int32_t *ka = k0, *va = v0, *kb = k1, *vb = v1;
  const int64_t tiles = rx_tiles(nacc);
  for (int shift = 0; shift < bits; shift += 8) {
    k_radix_hist<<<(unsigned)tiles, RX_THREADS, 0, st>>>(nacc, ka, shift, hist, tiles);
    CS_TRY(cs_exclusive_scan_i32(hist, hist, 256 * tiles, scratch, sb, st));
    k_radix_scatter<<<(unsigned)tiles, RX_THREADS, 0, st>>>(nacc, ka, va, shift, hist, tiles, kb, vb);
    int32_t *t = ka; ka = kb; kb = t;
    t = va; va = vb; vb = t;
  }
  // resource segments
  k_seg_heads<<<grid_for(nacc, 256), 256, 0, st>>>(nacc, ka, flag);
  CS_TRY(cs_exclusive_scan_i32(flag, fpos, nacc, scratch, sb, st));
  k_seg_compact<<<grid_for(nacc, 256), 256, 0, st>>>(nacc, flag, fpos, heads, nacc);
  int32_t nseg = 0;
  CS_CUDA(cudaMemcpyAsync(&nseg, fpos + nacc, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  // count, scan (original access order = task-major), emit
  CS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nacc + 1), st));
  k_seg_walk<false><<<grid_for(nseg, 128), 128, 0, st>>>(nseg, nacc, heads, va, acc_task, acc_write,
                                                         cnt, nullptr, nullptr);
  CS_TRY(cs_exclusive_scan_i32(cnt, poff, nacc, scratch, sb, st));
  int32_t total = 0;
  CS_CUDA(cudaMemcpyAsync(&total, poff + nacc, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  if (total > npred_max) {
    cs_set_error("generic detect: %d raw predecessors exceed the bound %lld", total, (long long)npred_max);
    return CS_ECAPACITY;
  }
  k_seg_walk<true><<<grid_for(nseg, 128), 128, 0, st>>>(nseg, nacc, heads, va, acc_task, acc_write,
                                                        nullptr, poff, preds);
  k_task_preds<<<grid_for(ntasks, 128), 128, 0, st>>>(ntasks, tptr, poff, preds, ecnt);
  CS_TRY(cs_exclusive_scan_i32(ecnt, eoff, ntasks, scratch, sb, st));
  int32_t ne = 0;
  CS_CUDA(cudaMemcpyAsync(&ne, eoff + ntasks, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  *nedges_host = ne;
  return cs_check_launch("detect_generic");
}

/* Pass 2 (same workspace, nothing in between): write the edges sorted by
 * (succ, pred). */
extern "C" int cs_detect_generic_emit(int64_t ntasks, int64_t nacc, const int64_t *tptr,
                                      int64_t npred_max, int64_t *eu, int64_t *ev, void *ws,
                                      size_t ws_bytes, void *stream) {
  cudaStream_t st = cs_stream(stream);
  cs_ws w(ws, ws_bytes);
  const int64_t nt = rx_tiles(nacc) + 1;
  for (int k = 0; k < 4; ++k) CS_REQUIRE(w.take<int32_t>(nacc + 1), "ws");
  CS_REQUIRE(w.take<int32_t>(256 * nt + 2), "ws");
  for (int k = 0; k < 3; ++k) CS_REQUIRE(w.take<int32_t>(nacc + 1), "ws");
  CS_REQUIRE(w.take<int32_t>(nacc + 2), "ws");
  CS_WS_TAKE(w, int32_t, poff, nacc + 2);
  CS_WS_TAKE(w, int32_t, preds, npred_max + 1);
  CS_WS_TAKE(w, int32_t, ecnt, ntasks + 2);
  CS_WS_TAKE(w, int32_t, eoff, ntasks + 2);
  (void)ecnt;
  if (ntasks == 0 || nacc == 0) return CS_OK;
  k_task_emit<<<grid_for(ntasks, 128), 128, 0, st>>>(ntasks, tptr, poff, preds, eoff, eu, ev);
  return cs_check_launch("detect_generic_emit");
}

// ------------------------------------------------------------ longest path --
__global__ void k_edges_per_succ(int64_t ne, const int64_t *ev, int32_t *cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[ev[e]], 1);
}
__global__ void k_check_forward(int64_t ne, const int64_t *eu, const int64_t *ev, int *bad) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x)
    if (eu[e] >= ev[e]) *bad = 1;
}
// edges are sorted by succ, so each task's preds are contiguous at rowptr
__global__ void k_lp_relax(int64_t nt, const int32_t *rowptr, const int64_t *eu, int32_t *level,
                           int *changed) {
  int any = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x) {
    int32_t L = 1;
    for (int32_t e = rowptr[t]; e < rowptr[t + 1]; ++e) L = max(L, level[eu[e]] + 1);
    if (L > level[t]) {
      level[t] = L;
      any = 1;
    }
  }
  if (__any_sync(CS_FULL, any) && (threadIdx.x & 31) == 0) *changed = 1;
}
__global__ void k_lp_serial(int64_t nt, const int32_t *rowptr, const int64_t *eu, int32_t *level) {
  for (int64_t t = 0; t < nt; ++t) {  // single thread: forward sweep (depgraph.py:167-173)
    int32_t L = 1;
    for (int32_t e = rowptr[t]; e < rowptr[t + 1]; ++e) L = max(L, level[eu[e]] + 1);
    level[t] = L;
  }
}

extern "C" size_t cs_longest_path_ws_bytes(int64_t ntasks) {
  return 2 * cs_ws_slice(sizeof(int32_t) * (ntasks + 2)) + cs_scan_ws_bytes(ntasks + 1) + 512;
}

extern "C" int cs_longest_path(int64_t ntasks, int64_t nedges, const int64_t *eu, const int64_t *ev,
                               int32_t *level, int64_t *depth_host, void *ws, size_t ws_bytes,
                               void *stream) {
  cudaStream_t st = cs_stream(stream);
  if (ntasks == 0) {
    *depth_host = 0;
    return CS_OK;
  }
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, cnt, ntasks + 2);
  CS_WS_TAKE(w, int32_t, rowptr, ntasks + 2);
  CS_WS_TAKE(w, int, scal, 16);
  const size_t sb = cs_scan_ws_bytes(ntasks + 1);
  void *scratch = w.take<char>(sb);
  CS_REQUIRE(scratch, "workspace too small (longest path)");
  CS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (ntasks + 1), st));
  CS_CUDA(cudaMemsetAsync(scal, 0, sizeof(int) * 16, st));
  if (nedges > 0) {
    k_check_forward<<<grid_for(nedges, 256), 256, 0, st>>>(nedges, eu, ev, scal + 8);
    k_edges_per_succ<<<grid_for(nedges, 256), 256, 0, st>>>(nedges, ev, cnt);
  }
  CS_TRY(cs_exclusive_scan_i32(cnt, rowptr, ntasks, scratch, sb, st));
  int bad = 0;
  CS_CUDA(cudaMemcpyAsync(&bad, scal + 8, sizeof(int), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  if (bad) {
    cs_set_error("cycle suspected: an edge is not forward");
    return CS_ECYCLE;
  }
  k_fill_i32<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, level, 1);
  int h = 1, it = 0;
  while (h && it < 64) {
    CS_CUDA(cudaMemsetAsync(scal, 0, sizeof(int), st));
    k_lp_relax<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, rowptr, eu, level, scal);
    CS_CUDA(cudaMemcpyAsync(&h, scal, sizeof(int), cudaMemcpyDeviceToHost, st));
    CS_CUDA(cudaStreamSynchronize(st));
    ++it;
  }
  if (h) k_lp_serial<<<1, 1, 0, st>>>(ntasks, rowptr, eu, level);  // deep graphs
  CS_CUDA(cudaMemsetAsync(scal + 4, 0, sizeof(int), st));
  k_max_i32<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, level, scal + 4);
  int32_t d = 0;
  CS_CUDA(cudaMemcpyAsync(&d, scal + 4, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  *depth_host = d;
  return cs_check_launch("longest_path");
}

// ------------------------------------- generic payload (apply_tasks, all kinds) --
// kind 0 intra: val[w0] += intra(q[home]); 1 inter: val[w0] += g, val[w1] -= g;
// 2 reduce: val[w0] += sum of val[reads]
struct GTask {
  const int8_t *kind;
  const int32_t *home, *nbr, *w0, *w1;
  const int8_t *off;  // 3 per task
  const int64_t *rptr;
  const int32_t *rres;
};

__global__ void k_gpayload_level(GTask T, const int32_t *bucket, int32_t lo, int32_t hi,
                                 const int64_t *q, int dim, int64_t *val) {
  for (int32_t i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    const int32_t t = bucket[i];
    const int k = T.kind[t];
    if (k == 0) {
      val[T.w0[t]] += pay_intra(q[T.home[t]]);
    } else if (k == 1) {
      const int8_t *o = T.off + 3 * (int64_t)t;
      const int64_t g = pay_pair(q[T.home[t]], q[T.nbr[t]], o[0], o[1], o[2], dim);
      val[T.w0[t]] += g;
      val[T.w1[t]] -= g;
    } else {
      int64_t s = 0;
      for (int64_t r = T.rptr[t]; r < T.rptr[t + 1]; ++r) s += val[T.rres[r]];
      val[T.w0[t]] += s;
    }
  }
}

extern "C" int cs_payload_generic(int64_t ntasks, int dim, const int8_t *kind, const int32_t *home,
                                  const int32_t *nbr, const int32_t *w0, const int32_t *w1,
                                  const int8_t *off, const int64_t *rptr, const int32_t *rres,
                                  const int64_t *q, const int32_t *level, int64_t depth,
                                  int64_t nres, int64_t *val, void *ws, size_t ws_bytes,
                                  void *stream) {
  cudaStream_t st = cs_stream(stream);
  CS_CUDA(cudaMemsetAsync(val, 0, sizeof(int64_t) * nres, st));
  if (ntasks == 0) return CS_OK;
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, slot, ntasks + 1);
  CS_WS_TAKE(w, int32_t, bucket, ntasks + 1);
  CS_WS_TAKE(w, int32_t, cnt, depth + 1);
  CS_WS_TAKE(w, int32_t, start, depth + 1);
  const size_t sb = cs_scan_ws_bytes(depth);
  void *scratch = w.take<char>(sb);
  CS_REQUIRE(scratch, "workspace too small (generic payload)");
  CS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (depth + 1), st));
  k_level_hist<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, level, cnt, slot);
  CS_TRY(cs_exclusive_scan_i32(cnt, start, depth, scratch, sb, st));
  k_level_scatter<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, level, slot, start, bucket);
  int32_t *hs = (int32_t *)malloc(sizeof(int32_t) * (depth + 1));
  cudaError_t e = cudaMemcpyAsync(hs, start, sizeof(int32_t) * (depth + 1), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    free(hs);
    CS_CUDA(e);
  }
  GTask T = {kind, home, nbr, w0, w1, off, rptr, rres};
  for (int64_t L = 0; L < depth; ++L)
    if (hs[L + 1] > hs[L])
      k_gpayload_level<<<grid_for(hs[L + 1] - hs[L], 128), 128, 0, st>>>(T, bucket, hs[L], hs[L + 1], q,
                                                                        dim, val);
  free(hs);
  return cs_check_launch("payload_generic");
}

extern "C" size_t cs_payload_generic_ws_bytes(int64_t ntasks, int64_t depth) {
  return 2 * cs_ws_slice(sizeof(int32_t) * (ntasks + 1)) + 2 * cs_ws_slice(sizeof(int32_t) * (depth + 1)) +
         cs_scan_ws_bytes(depth) + 512;
}

// ------------------------------- device dependency-driven runtime --
// Executes any task graph (apply_tasks semantics, payload.py:84-119) in
// dependency order instead of level by level: a persistent grid pops tickets
// from a ready queue, waits for the ticket's task, runs it, and releases its
// successors (indegree counters; the last predecessor pushes).  Accumulators
// are integers, so every valid order gives the reference's values.  With
// race_check, every task marks the accumulators it writes for its duration;
// finding a mark of another task counts a conflict -- the exclusion half of
// executor.verify_execution (executor.py:357-377) checked on the device.
struct DagArgs {
  GTask T;
  const int64_t *q;
  int dim;
  int64_t *val;
  int32_t *indeg;
  const int64_t *sptr;  // successors of t: succ[sptr[t] .. sptr[t+1])
  const int64_t *succ;
  int32_t *queue;
  unsigned *head, *tail;
  unsigned *mark;
  unsigned long long *conflicts;
  unsigned *err;
  int64_t ntasks;
  int race;
};

__global__ void k_dag_indeg(int64_t ne, const int64_t *ev, int32_t *indeg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&indeg[ev[i]], 1);
}

__global__ void k_dag_roots(int64_t nt, const int32_t *indeg, int32_t *queue, unsigned *tail) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x)
    if (indeg[t] == 0) queue[atomicAdd(tail, 1u)] = (int32_t)t;
}

__device__ __forceinline__ void dag_claim(const DagArgs &D, int32_t w, int32_t t) {
  const unsigned old = atomicExch(&D.mark[w], (unsigned)t + 1u);
  if (old != 0u) atomicAdd(D.conflicts, 1ull);
}

__global__ void k_dag_run(DagArgs D) {
  for (;;) {
    const unsigned idx = atomicAdd(D.head, 1u);
    if (idx >= (unsigned)D.ntasks) break;
    int32_t t;
    long long spins = 0;
    while ((t = ((volatile int32_t *)D.queue)[idx]) < 0) {
      if (++spins > (1ll << 26)) {  // never for a DAG: report instead of hanging
        atomicOr(D.err, 1u);
        return;
      }
      __nanosleep(64);
    }
    __threadfence();
    const int k = D.T.kind[t];
    const int32_t w0 = D.T.w0[t], w1 = D.T.w1[t];
    if (D.race) {
      dag_claim(D, w0, t);
      if (k == 1 && w1 != w0) dag_claim(D, w1, t);
    }
    if (k == 0) {
      D.val[w0] = __ldcg(D.val + w0) + pay_intra(D.q[D.T.home[t]]);
    } else if (k == 1) {
      const int8_t *o = D.T.off + 3 * (int64_t)t;
      const int64_t g = pay_pair(D.q[D.T.home[t]], D.q[D.T.nbr[t]], o[0], o[1], o[2], D.dim);
      D.val[w0] = __ldcg(D.val + w0) + g;
      D.val[w1] = __ldcg(D.val + w1) - g;
    } else {
      int64_t s = 0;
      for (int64_t r = D.T.rptr[t]; r < D.T.rptr[t + 1]; ++r) s += __ldcg(D.val + D.T.rres[r]);
      D.val[w0] = __ldcg(D.val + w0) + s;
    }
    if (D.race) {
      atomicExch(&D.mark[w0], 0u);
      if (k == 1 && w1 != w0) atomicExch(&D.mark[w1], 0u);
    }
    __threadfence();
    for (int64_t e = D.sptr[t]; e < D.sptr[t + 1]; ++e) {
      const int64_t s = D.succ[e];
      if (atomicSub(&D.indeg[s], 1) == 1) {
        const unsigned pos = atomicAdd(D.tail, 1u);
        atomicExch(&D.queue[pos], (int32_t)s);
      }
    }
  }
}

extern "C" size_t cs_dag_ws_bytes(int64_t ntasks, int64_t nres) {
  return 2 * cs_ws_slice(sizeof(int32_t) * (ntasks + 1)) + cs_ws_slice(sizeof(unsigned) * (nres + 1)) +
         cs_ws_slice(64);
}

// eu/ev: edges sorted by eu (successor lists); sptr[ntasks+1] their offsets.
extern "C" int cs_dag_execute(int64_t ntasks, int dim, const int8_t *kind, const int32_t *home,
                              const int32_t *nbr, const int32_t *w0, const int32_t *w1,
                              const int8_t *off, const int64_t *rptr, const int32_t *rres,
                              const int64_t *q, int64_t nedges, const int64_t *sptr,
                              const int64_t *succ, const int64_t *ev, int64_t nres, int64_t *val,
                              int race_check, unsigned long long *conflicts_dev, void *ws,
                              size_t ws_bytes, void *stream) {
  cudaStream_t st = cs_stream(stream);
  CS_CUDA(cudaMemsetAsync(val, 0, sizeof(int64_t) * nres, st));
  if (ntasks == 0) return CS_OK;
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, indeg, ntasks + 1);
  CS_WS_TAKE(w, int32_t, queue, ntasks + 1);
  CS_WS_TAKE(w, unsigned, mark, nres + 1);
  CS_WS_TAKE(w, unsigned, ctr, 16);
  CS_CUDA(cudaMemsetAsync(indeg, 0, sizeof(int32_t) * (ntasks + 1), st));
  CS_CUDA(cudaMemsetAsync(queue, 0xFF, sizeof(int32_t) * (ntasks + 1), st));  // -1: not pushed
  CS_CUDA(cudaMemsetAsync(mark, 0, sizeof(unsigned) * (nres + 1), st));
  CS_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned) * 16, st));
  if (conflicts_dev) CS_CUDA(cudaMemsetAsync(conflicts_dev, 0, sizeof(unsigned long long), st));
  if (nedges > 0) k_dag_indeg<<<grid_for(nedges, 256), 256, 0, st>>>(nedges, ev, indeg);
  DagArgs D;
  D.T = GTask{kind, home, nbr, w0, w1, off, rptr, rres};
  D.q = q;
  D.dim = dim;
  D.val = val;
  D.indeg = indeg;
  D.sptr = sptr;
  D.succ = succ;
  D.queue = queue;
  D.head = ctr;
  D.tail = ctr + 1;
  D.err = ctr + 2;
  D.mark = mark;
  D.conflicts = conflicts_dev ? conflicts_dev : (unsigned long long *)(ctr + 4);
  D.ntasks = ntasks;
  D.race = race_check ? 1 : 0;
  k_dag_roots<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, indeg, queue, ctr + 1);
  int dev = 0, nsm = 0;
  CS_CUDA(cudaGetDevice(&dev));
  CS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int64_t threads = (int64_t)nsm * 4 * 128;
  k_dag_run<<<(unsigned)((threads < ntasks ? threads : ntasks) + 127) / 128, 128, 0, st>>>(D);
  unsigned err = 0;
  CS_CUDA(cudaMemcpyAsync(&err, ctr + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  if (err) {
    cs_set_error("dag_execute: a task was never released (cycle in the edge list?)");
    return CS_ECYCLE;
  }
  return cs_check_launch("dag_execute");
}
