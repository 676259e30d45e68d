// cs_payload.cuh -- K5: the reference's integer interaction payload on device.
//
// Bit-exact restatement of payload.py:36-81 (_splitmix64, charges, intra,
// pair) executed (a) as the direct oracle sum (payload.py:152-174), (b) level
// by level along any stream's dependency levels (apply_tasks pattern,
// payload.py:84-119), and (c) under the LJ kernel's colour-pass schedules.
// Integer addition commutes, so any schedule that applies every contribution
// exactly once and never races reproduces reference_oracle bit for bit; a
// lost update from a schedule conflict shows up as a mismatch.
#pragma once
#include "cs_common.cuh"
#include "cs_sched.cuh"

#define PAY_CHARGE_KEY 0x9E3779B97F4A7C15ull
#define PAY_PAIR_KEY 0xA0761D6478BD642Full
#define PAY_INTRA_KEY 0x2545F4914F6CDD1Dull

__device__ __forceinline__ int64_t pay_center32(uint64_t x) {
  return (int64_t)(x & 0xFFFFFFFFull) - (1ll << 31);
}
__device__ __forceinline__ int64_t pay_intra(int64_t q) {
  return pay_center32(cs_splitmix64(PAY_INTRA_KEY ^ (uint64_t)q));
}
__device__ __forceinline__ uint64_t pay_code(int ox, int oy, int oz, int dim) {
  // payload.py:51-55: code = sum_k (o_k + 1) 3^k, x least significant
  uint64_t c = (uint64_t)(ox + 1) + 3ull * (uint64_t)(oy + 1);
  if (dim == 3) c += 9ull * (uint64_t)(oz + 1);
  return c;
}
__device__ __forceinline__ int64_t pay_mix(int64_t a, int64_t b, uint64_t code) {
  uint64_t h = cs_splitmix64(PAY_PAIR_KEY ^ (uint64_t)a);
  h = cs_splitmix64(h ^ (uint64_t)b);
  h = cs_splitmix64(h ^ code);
  return (int64_t)(h & 0x7FFFFFFFull);
}
__device__ __forceinline__ int64_t pay_pair(int64_t a, int64_t b, int ox, int oy, int oz, int dim) {
  return pay_mix(a, b, pay_code(ox, oy, oz, dim)) - pay_mix(b, a, pay_code(-ox, -oy, -oz, dim));
}

__global__ void k_charges(int64_t ncells, uint64_t base, int64_t *q) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncells;
       c += (int64_t)gridDim.x * blockDim.x)
    q[c] = pay_center32(cs_splitmix64(base + (uint64_t)c));
}

extern "C" int cs_payload_charges(const cs_grid *g, int64_t seed, int64_t *q, void *stream) {
  CS_REQUIRE(g && (g->dim == 2 || g->dim == 3), "grid must be 2D or 3D");
  int64_t nc = 1;
  for (int k = 0; k < g->dim; ++k) nc *= g->ext[k];
  uint64_t base = cs_splitmix64_host((uint64_t)seed ^ PAY_CHARGE_KEY);
  k_charges<<<grid_for(nc, 256), 256, 0, cs_stream(stream)>>>(nc, base, q);
  return cs_check_launch("charges");
}

// direct sum: intra + every one of the 3^dim - 1 neighbours (payload.py:152-174)
__global__ void k_payload_direct(StreamDesc d, const int64_t *q, int64_t *acc) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < d.ncells;
       c += (int64_t)gridDim.x * blockDim.x) {
    int cc[3];
    desc_coords(d, c, cc);
    int64_t qc = q[c];
    int64_t s = pay_intra(qc);
    int nz = d.dim == 3 ? 3 : 1;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        for (int z = 0; z < nz; ++z) {
          int o[3] = {a - 1, b - 1, d.dim == 3 ? z - 1 : 0};
          if (!o[0] && !o[1] && !o[2]) continue;
          int n3[3];
          bool ok = true;
          for (int k = 0; k < 3; ++k) {
            int v = cc[k] + o[k];
            if (d.per[k])
              v = cs_wrap(v, d.ext[k]);
            else if (v < 0 || v >= d.ext[k])
              ok = false;
            n3[k] = v;
          }
          if (!ok) continue;
          s += pay_pair(qc, q[desc_index(d, n3)], o[0], o[1], o[2], d.dim);
        }
    acc[c] = s;
  }
}

extern "C" int cs_payload_direct(const cs_grid *g, int64_t seed, const int64_t *q, int64_t *acc,
                                 void *stream) {
  (void)seed;
  StreamDesc d;
  int8_t dummy[3] = {0, 0, 0};
  CS_TRY(build_desc(g, CS_STREAM_BASIC, dummy, 1, 2, &d));
  k_payload_direct<<<grid_for(d.ncells, 128), 128, 0, cs_stream(stream)>>>(d, q, acc);
  return cs_check_launch("payload_direct");
}

// ------------------------------------------- level-by-level stream execution --
struct EntryTable {
  int8_t off[27][3];
  int dim;
};

__global__ void k_level_hist(int64_t nt, const int32_t *level, int32_t *cnt, int32_t *slot) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x)
    slot[t] = atomicAdd(&cnt[level[t] - 1], 1);
}
__global__ void k_level_scatter(int64_t nt, const int32_t *level, const int32_t *slot,
                                const int32_t *start, int32_t *bucket) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x)
    bucket[start[level[t] - 1] + slot[t]] = (int32_t)t;
}
// all tasks of one level are write-disjoint: plain read-modify-write
__global__ void k_payload_level(EntryTable et, const int32_t *bucket, int32_t lo, int32_t hi,
                                const int64_t *q, const int32_t *home, const int32_t *nbr,
                                const int16_t *entry, int64_t *acc) {
  for (int32_t i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    int32_t t = bucket[i];
    int32_t h = home[t], nb = nbr[t];
    if (nb < 0) {
      acc[h] += pay_intra(q[h]);
    } else {
      const int8_t *o = et.off[entry[t]];
      int64_t g = pay_pair(q[h], q[nb], o[0], o[1], o[2], et.dim);
      acc[h] += g;
      acc[nb] -= g;
    }
  }
}

extern "C" size_t cs_payload_levels_ws_bytes(int64_t ntasks, int64_t depth) {
  return 2 * cs_ws_slice(sizeof(int32_t) * (ntasks + 1)) +
         2 * cs_ws_slice(sizeof(int32_t) * (depth + 1)) + cs_scan_ws_bytes(depth);
}

extern "C" int cs_payload_levels(const cs_grid *g, const int64_t *q, int64_t ntasks,
                                 const int32_t *home, const int32_t *nbr, const int16_t *entry,
                                 const int8_t *offs, int n, const int32_t *level, int64_t depth,
                                 int64_t *acc, void *ws, size_t ws_bytes, void *stream) {
  cudaStream_t st = cs_stream(stream);
  CS_REQUIRE(n >= 1 && n <= 27, "bad entry count");
  int64_t nc = 1;
  for (int k = 0; k < g->dim; ++k) nc *= g->ext[k];
  CS_CUDA(cudaMemsetAsync(acc, 0, sizeof(int64_t) * nc, st));
  if (ntasks == 0) return CS_OK;
  EntryTable et;
  memset(&et, 0, sizeof(et));
  et.dim = g->dim;
  for (int e = 0; e < n; ++e)
    for (int k = 0; k < g->dim; ++k) et.off[e][k] = offs[e * g->dim + k];
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, slot, ntasks + 1);
  CS_WS_TAKE(w, int32_t, bucket, ntasks + 1);
  CS_WS_TAKE(w, int32_t, cnt, depth + 1);
  CS_WS_TAKE(w, int32_t, start, depth + 1);
  size_t sb = cs_scan_ws_bytes(depth);
  void *scratch = w.take<char>(sb);
  CS_REQUIRE(scratch, "workspace too small");
  CS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (depth + 1), st));
  k_level_hist<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, level, cnt, slot);
  CS_TRY(cs_exclusive_scan_i32(cnt, start, depth, scratch, sb, st));
  k_level_scatter<<<grid_for(ntasks, 256), 256, 0, st>>>(ntasks, level, slot, start, bucket);
  int32_t *hstart = (int32_t *)malloc(sizeof(int32_t) * (depth + 1));
  cudaError_t e = cudaMemcpyAsync(hstart, start, sizeof(int32_t) * (depth + 1),
                                  cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    free(hstart);
    CS_CUDA(e);
  }
  for (int64_t L = 0; L < depth; ++L) {
    int32_t lo = hstart[L], hi = hstart[L + 1];
    if (hi <= lo) continue;
    k_payload_level<<<grid_for(hi - lo, 128), 128, 0, st>>>(et, bucket, lo, hi, q, home, nbr,
                                                            entry, acc);
  }
  free(hstart);
  return cs_check_launch("payload_levels");
}
