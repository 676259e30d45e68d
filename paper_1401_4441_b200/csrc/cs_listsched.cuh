// cs_listsched.cuh -- a11 / f3: the reference's worker-pool model on the device.
//
// simulate          schedsim.py:63-90   greedy list scheduling, unit durations,
//                                       W workers, ready tasks taken in
//                                       ascending id order
// simulate_dynamic  schedsim.py:93-163  the same with NestedPlan spawning
//                                       (taskgen.py:279-325): a finished task
//                                       spawns its cell's next chain entry; the
//                                       dependency rule (depgraph.py:28-49) is
//                                       applied at spawn time
//
// One persistent CTA runs the whole schedule.  The ready set is a bitmap over
// task ids.  Every edge runs low id -> high id, so a task made ready by a
// batch has a larger id than the batch's first task, and spawned tasks take
// fresh (larger) ids: the smallest ready id never decreases.  Each time step
// therefore scans the bitmap forward from the previous batch's first word and
// takes the first W set bits (block-wide popcount scan), stamps their start
// time, releases successors with atomic indegree counters, and -- nested
// mode -- spawns children in ascending parent order, one warp resolving the
// last-accessor rule for 32 spawns at a time.
#pragma once
#include "cs_sched.cuh"

#define LS_THREADS 1024

struct LsState {
  int64_t now, done, ntasks, cursor;  // cursor: first bitmap word that can hold a ready bit
  int64_t got;                        // tasks in the current batch
  int err;
};

// block-wide exclusive scan of one int per thread (LS_THREADS threads)
__device__ __forceinline__ int ls_block_scan(int v, int *wsum, int &total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(CS_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(CS_FULL, s, o);
      if (lane >= o) s += y;
    }
    wsum[lane] = s;  // inclusive over warps
  }
  __syncthreads();
  total = wsum[31];
  const int before = (wid ? wsum[wid - 1] : 0) + x - v;
  __syncthreads();
  return before;
}

// the first `need` set bits at or after word `cursor` go to batch[]; their
// bits are cleared.  Returns the number taken (all threads).  SMEM: the
// bitmap lives in shared memory (else in global memory, changed by atomics).
template <bool SMEM = false>
__device__ int ls_select(uint32_t *bits, int64_t nwords, int64_t cursor, int64_t need,
                         int32_t *batch, int *wsum) {
  int64_t got = 0;
  for (int64_t w0 = cursor; w0 < nwords && got < need; w0 += LS_THREADS) {
    const int64_t w = w0 + threadIdx.x;
    uint32_t word = w < nwords ? (SMEM ? bits[w] : __ldcg(bits + w)) : 0u;  // (atomics change bits)
    int total;
    const int before = ls_block_scan(__popc(word), wsum, total);
    const int64_t left = need - got;
    if (word && before < left) {
      uint32_t keep = word;
      int64_t r = before;
      while (keep && r < left) {
        const int b = __ffs(keep) - 1;
        keep &= keep - 1;
        batch[got + r] = (int32_t)(w * 32 + b);
        ++r;
      }
      if (SMEM) bits[w] = keep;  // taken bits cleared; this thread owns word w
      else __stcg(bits + w, keep);
    }
    got += total < left ? total : left;
  }
  __syncthreads();
  return (int)(got < need ? got : need);
}

// ----------------------------------------------------------- static graph --
__global__ void __launch_bounds__(LS_THREADS, 1)
    k_ls_static(int64_t n, const int64_t *__restrict__ sptr, const int32_t *__restrict__ succ,
                int64_t W, int32_t *indeg, uint32_t *bits, int32_t *batch, int32_t *start,
                LsState *st) {
  __shared__ int wsum[32];
  __shared__ int64_t s_cursor;
  const int64_t nwords = (n + 31) / 32;
  int64_t now = 0, done = 0, cursor = 0;
  while (true) {
    const int got = ls_select(bits, nwords, cursor, W, batch, wsum);
    if (got == 0) break;
    for (int k = threadIdx.x; k < got; k += LS_THREADS) {
      const int32_t t = batch[k];
      start[t] = (int32_t)now;
      for (int64_t s = sptr[t]; s < sptr[t + 1]; ++s) {
        const int32_t v = succ[s];
        if (atomicSub(&indeg[v], 1) == 1) atomicOr(&bits[v >> 5], 1u << (v & 31));
      }
    }
    if (threadIdx.x == 0) s_cursor = batch[0] >> 5;
    __syncthreads();
    cursor = s_cursor;
    ++now;
    done += got;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    st->now = now;
    st->done = done;
    st->ntasks = n;
  }
}

// The same schedule run by ONE warp with the ready bitmap and 8-bit
// indegrees in shared memory (graphs of up to LS_SMEM_TASKS tasks whose
// indegrees fit a byte): a time step is a warp ballot scan of the bitmap and
// a warp-wide release, synchronised by __syncwarp only -- its cost is the
// global-memory lookups of the batch's successors.
#define LS_SMEM_TASKS 180000  // 1.125 bytes per task of shared memory
__global__ void __launch_bounds__(32, 1)
    k_ls_static_warp(int64_t n, const int64_t *__restrict__ sptr, const int32_t *__restrict__ succ,
                     int64_t W, const int32_t *indeg_g, const uint32_t *bits_g, int32_t *batch,
                     int32_t *start, LsState *st) {
  extern __shared__ __align__(16) unsigned char ls_raw[];
  const int lane = threadIdx.x;
  const int64_t nwords = (n + 31) / 32;
  uint32_t *bits = reinterpret_cast<uint32_t *>(ls_raw);
  unsigned *indeg = reinterpret_cast<unsigned *>(ls_raw + 4 * nwords);  // 4 tasks per word
  // highest bitmap word that may hold a ready bit: the scan stops there (a
  // ready set smaller than W would otherwise scan to the end every step)
  __shared__ int64_t s_hiw;
  int64_t hiw = 0;
  for (int64_t w = lane; w < nwords; w += 32) {
    bits[w] = bits_g[w];
    if (bits_g[w]) hiw = w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hiw = max(hiw, __shfl_xor_sync(CS_FULL, hiw, o));
  if (lane == 0) s_hiw = hiw;
  for (int64_t q = lane; q < (n + 3) / 4; q += 32) {
    unsigned v = 0;
    for (int k = 0; k < 4; ++k)
      if (4 * q + k < n) v |= (unsigned)indeg_g[4 * q + k] << (8 * k);
    indeg[q] = v;
  }
  __syncwarp();
  int64_t now = 0, done = 0, cursor = 0;
  while (true) {
    // select: the first W set bits from word `cursor` on, 32 words per pass
    int64_t got = 0;
    const int64_t wend = min(nwords, *(volatile int64_t *)&s_hiw + 1);
    for (int64_t w0 = cursor; w0 < wend && got < W; w0 += 32) {
      const int64_t w = w0 + lane;
      uint32_t word = w < wend ? bits[w] : 0u;
      const int c = __popc(word);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(CS_FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(CS_FULL, incl, 31);
      const int64_t left = W - got;
      int64_t r = incl - c;
      if (word && r < left) {
        uint32_t keep = word;
        while (keep && r < left) {
          const int b = __ffs(keep) - 1;
          keep &= keep - 1;
          batch[got + r] = (int32_t)(w * 32 + b);
          ++r;
        }
        bits[w] = keep;
      }
      got += total < left ? total : left;
    }
    __syncwarp();
    if (got == 0) break;
    // release: start step, successors' indegrees, newly ready bits
    for (int64_t k = lane; k < got; k += 32) {
      const int32_t t = batch[k];
      start[t] = (int32_t)now;
      const int64_t s1 = sptr[t + 1];
      for (int64_t s = sptr[t]; s < s1; ++s) {
        const int32_t v = succ[s];
        const unsigned sh = 8u * (v & 3);
        // bytes of one word never borrow from each other: an indegree only
        // reaches zero, never goes below it
        const unsigned old = atomicSub(&indeg[v >> 2], 1u << sh);
        if (((old >> sh) & 0xFFu) == 1u) {
          atomicOr(&bits[v >> 5], 1u << (v & 31));
          atomicMax((unsigned long long *)&s_hiw, (unsigned long long)(v >> 5));
        }
      }
    }
    __syncwarp();
    cursor = __shfl_sync(CS_FULL, lane == 0 ? (int64_t)(batch[0] >> 5) : (int64_t)0, 0);
    ++now;
    done += got;
    __syncwarp();
  }
  if (lane == 0) {
    st->now = now;
    st->done = done;
    st->ntasks = n;
  }
}

__global__ void k_ls_static_init(int64_t n, const int64_t *__restrict__ sptr,
                                 const int32_t *__restrict__ succ, int32_t *indeg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < sptr[n];
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&indeg[succ[e]], 1);
}
__global__ void k_ls_roots(int64_t n, const int32_t *__restrict__ indeg, uint32_t *bits) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= (n + 31) / 32) return;
  uint32_t word = 0;
  for (int b = 0; b < 32; ++b) {
    const int64_t t = w * 32 + b;
    if (t < n && indeg[t] == 0) word |= 1u << b;
  }
  bits[w] = word;
}

size_t cs_listsched_ws_bytes(int64_t ntasks) {
  const int64_t n = ntasks < 1 ? 1 : ntasks;
  return cs_ws_slice(sizeof(int32_t) * n) * 2 + cs_ws_slice(sizeof(uint32_t) * ((n + 31) / 32)) +
         cs_ws_slice(sizeof(LsState));
}

int cs_simulate_static(int64_t ntasks, int64_t nedges, const int64_t *sptr, const int32_t *succ,
                       int64_t workers, int64_t max_indegree_host, int32_t *start,
                       int64_t *makespan_host, void *ws, size_t ws_bytes, void *stream) {
  CS_REQUIRE(ntasks >= 1, "cannot simulate an empty graph");
  CS_REQUIRE(workers >= 1, "workers must be >= 1, got %lld", (long long)workers);
  CS_REQUIRE(ntasks < (1ll << 31), "simulate: at most 2^31-1 tasks");
  cudaStream_t s = cs_stream(stream);
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, indeg, ntasks);
  CS_WS_TAKE(w, int32_t, batch, ntasks);
  CS_WS_TAKE(w, uint32_t, bits, (ntasks + 31) / 32);
  CS_WS_TAKE(w, LsState, st, 1);
  const int64_t W = workers < ntasks ? workers : ntasks;
  CS_CUDA(cudaMemsetAsync(indeg, 0, sizeof(int32_t) * ntasks, s));
  if (nedges > 0)
    k_ls_static_init<<<592, 256, 0, s>>>(ntasks, sptr, succ, indeg);
  const int64_t nwords = (ntasks + 31) / 32;
  k_ls_roots<<<(unsigned)((nwords + 255) / 256), 256, 0, s>>>(ntasks, indeg, bits);
  const size_t smem = 4 * (size_t)nwords + 4 * (size_t)((ntasks + 3) / 4);
  if (ntasks <= LS_SMEM_TASKS && max_indegree_host <= 255) {
    static size_t attr_smem[CS_MAX_DEVICES];
    const int dev = cs_device_index();
    if (smem > attr_smem[dev]) {
      CS_CUDA(cudaFuncSetAttribute(k_ls_static_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
      attr_smem[dev] = smem;
    }
    k_ls_static_warp<<<1, 32, smem, s>>>(ntasks, sptr, succ, W, indeg, bits, batch, start, st);
  } else {
    k_ls_static<<<1, LS_THREADS, 0, s>>>(ntasks, sptr, succ, W, indeg, bits, batch, start, st);
  }
  CS_TRY(cs_check_launch("k_ls_static"));
  LsState h;
  CS_CUDA(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  if (h.done != ntasks) {
    cs_set_error("schedule stalled with %lld tasks blocked; graph has a cycle",
                 (long long)(ntasks - h.done));
    return CS_ECYCLE;
  }
  *makespan_host = h.now;
  return CS_OK;
}

// ------------------------------------------------------------ nested plan --
// Task arrays (capacity ncells * n): home cell, chain entry, spawning parent
// (-1: initial), predecessors (sorted, -1 = none), start time.  Each task
// writes at most two accumulators, so it has at most two successors ever.
struct NestedArgs {
  StreamDesc d;
  int64_t cap, W;
  int32_t *home, *parent, *pa, *pb, *start, *indeg, *nsucc, *succ2, *last, *batch;
  int16_t *entry;
  uint32_t *bits;
  LsState *st;
};

// next chain entry of `cell` after position `pos` whose neighbour exists
// (entries off a non-periodic edge are skipped, taskgen.py:311-325)
__device__ __forceinline__ int nested_next(const StreamDesc &d, int64_t cell, int pos,
                                           int64_t &nb) {
  for (int e = pos + 1; e < d.n; ++e) {
    nb = desc_nbr(d, cell, e);
    if (nb >= 0) return e;
  }
  return -1;
}

__global__ void __launch_bounds__(LS_THREADS, 1) k_ls_nested(NestedArgs A) {
  __shared__ int wsum[32];
  __shared__ int64_t s_cursor, s_ntasks;
  __shared__ int32_t c_h[32], c_n[32], c_id[32];
  const StreamDesc &d = A.d;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t now = 0, done = 0, cursor = 0;
  if (threadIdx.x == 0) s_ntasks = d.ncells;
  __syncthreads();
  while (true) {
    const int64_t nwords = (s_ntasks + 31) / 32;
    const int got = ls_select(A.bits, nwords, cursor, A.W, A.batch, wsum);
    if (got == 0) break;
    // start times; a batch task is finished once its time step ends
    for (int k = threadIdx.x; k < got; k += LS_THREADS) A.start[A.batch[k]] = (int32_t)now;
    __syncthreads();
    // release successors recorded at spawn time
    for (int k = threadIdx.x; k < got; k += LS_THREADS) {
      const int32_t t = A.batch[k];
      const int ns = __ldcg(A.nsucc + t);
      for (int q = 0; q < ns; ++q) {
        const int32_t v = __ldcg(A.succ2 + 2 * t + q);
        if (atomicSub(&A.indeg[v], 1) == 1) atomicOr(&A.bits[v >> 5], 1u << (v & 31));
      }
    }
    __syncthreads();
    // spawns in ascending parent order (the batch is sorted), 32 at a time
    if (wid == 0) {
      int64_t nt = s_ntasks;
      for (int k0 = 0; k0 < got; k0 += 32) {
        const int k = k0 + lane;
        int64_t nb = -1;
        int e = -1;
        int32_t par = -1, hc = -1;
        if (k < got) {
          par = A.batch[k];
          hc = __ldcg(A.home + par);
          e = nested_next(d, hc, __ldcg(A.entry + par), nb);
        }
        const unsigned has = __ballot_sync(CS_FULL, e >= 0);
        const int32_t id = (int32_t)(nt + __popc(has & ((1u << lane) - 1)));
        c_h[lane] = e >= 0 ? hc : -1;
        c_n[lane] = e >= 0 ? (int32_t)nb : -1;
        c_id[lane] = id;
        __syncwarp();
        int32_t p0 = -1, p1 = -1;  // last accessor of acc(home), acc(nbr)
        if (e >= 0) {
          const int32_t r0 = hc, r1 = (int32_t)nb;
          for (int l = lane - 1; l >= 0 && (p0 < 0 || p1 < 0); --l) {
            if (c_h[l] < 0) continue;
            if (p0 < 0 && (c_h[l] == r0 || c_n[l] == r0)) p0 = c_id[l];
            if (p1 < 0 && (c_h[l] == r1 || c_n[l] == r1)) p1 = c_id[l];
          }
          if (p0 < 0) p0 = A.last[r0];
          if (p1 < 0) p1 = A.last[r1];
          if (r0 == r1) p1 = p0;
          int32_t a = p0 < p1 ? p0 : p1, b = p0 < p1 ? p1 : p0;
          if (a == b) b = -1;
          if (a < 0) { a = b; b = -1; }
          A.home[id] = hc;
          A.entry[id] = (int16_t)e;
          A.parent[id] = par;
          A.pa[id] = a;
          A.pb[id] = b;
          A.nsucc[id] = 0;
          int waiting = 0;
          // a predecessor is finished iff it started in this or an earlier
          // step (start < 0 marks "not yet run")
          if (a >= 0 && __ldcg(A.start + a) < 0) {
            A.succ2[2 * a + atomicAdd(&A.nsucc[a], 1)] = id;
            ++waiting;
          }
          if (b >= 0 && __ldcg(A.start + b) < 0) {
            A.succ2[2 * b + atomicAdd(&A.nsucc[b], 1)] = id;
            ++waiting;
          }
          A.indeg[id] = waiting;
        }
        __syncwarp();
        // state: the last lane touching a resource owns its update
        if (e >= 0) {
          bool own0 = true, own1 = true;
          for (int l = lane + 1; l < 32; ++l) {
            if (c_h[l] < 0) continue;
            if (c_h[l] == hc || c_n[l] == hc) own0 = false;
            if (c_h[l] == (int32_t)nb || c_n[l] == (int32_t)nb) own1 = false;
          }
          if (own0) A.last[hc] = id;
          if (own1) A.last[nb] = id;
        }
        __syncwarp();
        if (e >= 0 && A.indeg[id] == 0) atomicOr(&A.bits[id >> 5], 1u << (id & 31));
        nt += __popc(has);
        __syncwarp();
      }
      if (lane == 0) s_ntasks = nt;
    }
    if (threadIdx.x == 0) s_cursor = A.batch[0] >> 5;
    __syncthreads();
    cursor = s_cursor;
    ++now;
    done += got;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    A.st->now = now;
    A.st->done = done;
    A.st->ntasks = s_ntasks;
  }
}

__global__ void k_ls_nested_init(NestedArgs A) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < A.d.ncells) {  // intra task of cell c has id c (initial_tasks, taskgen.py:303-308)
    A.home[c] = (int32_t)c;
    A.entry[c] = 0;
    A.parent[c] = -1;
    A.pa[c] = A.pb[c] = -1;
    A.indeg[c] = 0;
    A.nsucc[c] = 0;
    A.last[c] = (int32_t)c;
  }
  const int64_t nwords = (A.cap + 31) / 32;
  if (c < nwords) {
    uint32_t word = 0;
    for (int b = 0; b < 32; ++b)
      if (c * 32 + b < A.d.ncells) word |= 1u << b;
    A.bits[c] = word;
  }
}

size_t cs_nested_ws_bytes(const cs_grid *g, int n) {
  int64_t cells = 1;
  for (int k = 0; g && k < g->dim; ++k) cells *= g->ext[k] > 0 ? g->ext[k] : 1;
  const int64_t cap = cells * (n > 0 ? n : 1);
  return cs_ws_slice(4 * cap) * 6 + cs_ws_slice(4 * cells) +
         cs_ws_slice(4 * ((cap + 31) / 32)) + cs_ws_slice(sizeof(LsState));
}

int cs_simulate_nested(const cs_grid *g, const int8_t *order_host, int n, int64_t workers,
                       int32_t *home, int16_t *entry, int32_t *parent, int32_t *pred_a,
                       int32_t *pred_b, int32_t *start, int64_t capacity, int64_t *ntasks_host,
                       int64_t *makespan_host, void *ws, size_t ws_bytes, void *stream) {
  CS_REQUIRE(workers >= 1, "workers must be >= 1, got %lld", (long long)workers);
  NestedArgs A;
  CS_TRY(build_desc(g, CS_STREAM_BASIC, order_host, n, 2, &A.d));
  CS_REQUIRE(desc_is_intra(A.d, 0), "nested chains must start with the intra entry");
  A.cap = A.d.ncells * A.d.n;
  CS_REQUIRE(capacity >= A.cap, "task arrays hold %lld tasks, need %lld", (long long)capacity,
             (long long)A.cap);
  CS_REQUIRE(A.cap < (1ll << 31), "nested plan: at most 2^31-1 tasks");
  cudaStream_t s = cs_stream(stream);
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, indeg, A.cap);
  CS_WS_TAKE(w, int32_t, nsucc, A.cap);
  CS_WS_TAKE(w, int32_t, succ2, 2 * A.cap);
  CS_WS_TAKE(w, int32_t, last, A.d.ncells);
  CS_WS_TAKE(w, uint32_t, bits, (A.cap + 31) / 32);
  CS_WS_TAKE(w, LsState, st, 1);
  A.W = workers < A.cap ? workers : A.cap;
  A.home = home;
  A.entry = entry;
  A.parent = parent;
  A.pa = pred_a;
  A.pb = pred_b;
  A.start = start;
  A.indeg = indeg;
  A.nsucc = nsucc;
  A.succ2 = succ2;
  A.last = last;
  A.bits = bits;
  A.st = st;
  CS_WS_TAKE(w, int32_t, batch, A.cap);
  A.batch = batch;
  CS_CUDA(cudaMemsetAsync(start, 0xFF, sizeof(int32_t) * A.cap, s));
  const int64_t nwords = (A.cap + 31) / 32;
  const int64_t m = A.d.ncells > nwords ? A.d.ncells : nwords;
  k_ls_nested_init<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(A);
  k_ls_nested<<<1, LS_THREADS, 0, s>>>(A);
  CS_TRY(cs_check_launch("k_ls_nested"));
  LsState h;
  CS_CUDA(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  if (h.done != h.ntasks) {
    cs_set_error("dynamic schedule stalled; spawn bookkeeping is inconsistent");
    return CS_ECYCLE;
  }
  *ntasks_host = h.ntasks;
  *makespan_host = h.now;
  return CS_OK;
}
