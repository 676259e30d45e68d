// cs_util.cuh -- error state, scans, deterministic reductions, stencil table.
#pragma once
#include <stdarg.h>

#include "cs_common.cuh"

static thread_local char g_cs_err[512] = "";

void cs_set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_cs_err, sizeof(g_cs_err), fmt, ap);
  va_end(ap);
}

int cs_check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cs_set_error("%s: %s", what, cudaGetErrorString(e));
    return (int)e;
  }
  return CS_OK;
}

extern "C" const char *cs_last_error(void) { return g_cs_err; }
extern "C" int cs_abi_version(void) { return 1; }
extern "C" int cs_device_synchronize(void) {
  CS_CUDA(cudaDeviceSynchronize());
  return CS_OK;
}
// device-to-device copy on the stream (a memcpy node when captured)
extern "C" int cs_copy_async(void *dst, const void *src, size_t bytes, void *stream) {
  if (bytes == 0) return CS_OK;
  CS_REQUIRE(dst && src, "cs_copy_async: null pointer");
  CS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, cs_stream(stream)));
  return CS_OK;
}
__global__ void k_accumulate_i64(unsigned long long *acc, const unsigned long long *x) { *acc += *x; }
// *acc += *x on the stream (device-side running totals, no host read)
extern "C" int cs_accumulate_i64(int64_t *acc, const int64_t *x, void *stream) {
  k_accumulate_i64<<<1, 1, 0, cs_stream(stream)>>>((unsigned long long *)acc,
                                                   (const unsigned long long *)x);
  return cs_check_launch("accumulate_i64");
}
// stream-ordered fill (captured as a memset node inside CUDA graphs): the
// per-step result words are cleared through the C ABI, not by torch kernels
extern "C" int cs_memset_async(void *dst, int value, size_t bytes, void *stream) {
  if (bytes == 0) return CS_OK;
  CS_REQUIRE(dst, "cs_memset_async: null destination");
  CS_CUDA(cudaMemsetAsync(dst, value, bytes, cs_stream(stream)));
  return CS_OK;
}

// ------------------------------------------------------- canonical stencil --
void cs_host_canonical_stencil(int dim, int8_t *out, int *n) {
  int total = 1;
  for (int k = 0; k < dim; ++k) total *= 3;
  for (int k = 0; k < dim; ++k) out[k] = 0;
  int m = 1;
  for (int t = 0; t < total; ++t) {  // itertools.product order, x slowest
    int o[3], rem = t;
    for (int k = dim - 1; k >= 0; --k) {
      o[k] = rem % 3 - 1;
      rem /= 3;
    }
    int pos = 0;
    for (int k = 0; k < dim; ++k) {
      if (o[k] > 0) { pos = 1; break; }
      if (o[k] < 0) break;
    }
    if (!pos) continue;
    for (int k = 0; k < dim; ++k) out[m * dim + k] = (int8_t)o[k];
    ++m;
  }
  *n = m;
}

static bool g_stencil_uploaded[CS_MAX_DEVICES];
int cs_upload_stencil(void) {
  const int dev = cs_device_index();
  if (g_stencil_uploaded[dev]) return CS_OK;
  int8_t st[14 * 3];
  int n;
  cs_host_canonical_stencil(3, st, &n);
  cs_offsets h;
  for (int e = 0; e < 14; ++e) {
    int ax = 0;
    for (int k = 0; k < 3; ++k) {
      h.o[e][k] = st[3 * e + k];
      if (st[3 * e + k]) ax = k;
    }
    h.axis[e] = (int8_t)ax;
  }
  CS_CUDA(cudaMemcpyToSymbol(c_stencil3, &h, sizeof(h)));
  g_stencil_uploaded[dev] = true;
  return CS_OK;
}

// -------------------------------------------------------------------- scan --
#define SCAN_THREADS 1024
#define SCAN_ITEMS 4
#define SCAN_TILE (SCAN_THREADS * SCAN_ITEMS)

// block-wide exclusive scan of one value per thread; returns the prefix and
// writes the block total to *total (all threads).
template <class T>
__device__ __forceinline__ T block_exclusive_scan(T v, T *total) {
  __shared__ T warp_tot[33];  // [32] = block total
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(CS_FULL, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int nw = (blockDim.x + 31) >> 5;
    T w = lane < nw ? warp_tot[lane] : T(0);
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T n = __shfl_up_sync(CS_FULL, wi, o);
      if (lane >= o) wi += n;
    }
    if (lane < nw) warp_tot[lane] = wi - w;  // exclusive warp offsets
    if (lane == nw - 1) warp_tot[32] = wi;
  }
  __syncthreads();
  T res = warp_tot[wid] + inc - v;
  *total = warp_tot[32];
  __syncthreads();
  return res;
}

__global__ void k_scan_tile_sums(const int32_t *in, int64_t n, int32_t *sums) {
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int32_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t i = base + (int64_t)threadIdx.x * SCAN_ITEMS + k;
    if (i < n) s += in[i];
  }
  int32_t tot;
  block_exclusive_scan<int32_t>(s, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void k_scan_sums(int32_t *sums, int64_t nb, int32_t *total_out) {
  int32_t carry = 0;
  for (int64_t c = 0; c < nb; c += SCAN_THREADS) {
    int64_t i = c + threadIdx.x;
    int32_t v = i < nb ? sums[i] : 0;
    int32_t tot;
    int32_t ex = block_exclusive_scan<int32_t>(v, &tot);
    if (i < nb) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total_out = carry;
}

__global__ void k_scan_tiles(const int32_t *in, int32_t *out, int64_t n, const int32_t *sums) {
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int32_t v[SCAN_ITEMS], s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = (base + k < n) ? in[base + k] : 0;
    s += v[k];
  }
  int32_t tot;
  int32_t ex = block_exclusive_scan<int32_t>(s, &tot) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (base + k < n) out[base + k] = ex;
    ex += v[k];
  }
}

size_t cs_scan_ws_bytes(int64_t n) {
  int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  return cs_ws_slice(sizeof(int32_t) * (nb + 1));
}

int cs_exclusive_scan_i32(const int32_t *in, int32_t *out, int64_t n, void *ws, size_t ws_bytes,
                          cudaStream_t st) {
  int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (nb == 0) {
    CS_CUDA(cudaMemsetAsync(out, 0, sizeof(int32_t), st));
    return CS_OK;
  }
  cs_ws w(ws, ws_bytes);
  CS_WS_TAKE(w, int32_t, sums, nb + 1);
  k_scan_tile_sums<<<(unsigned)nb, SCAN_THREADS, 0, st>>>(in, n, sums);
  k_scan_sums<<<1, SCAN_THREADS, 0, st>>>(sums, nb, out + n);
  k_scan_tiles<<<(unsigned)nb, SCAN_THREADS, 0, st>>>(in, out, n, sums);
  return cs_check_launch("exclusive_scan");
}

// ------------------------------------------------- deterministic reductions --
#define RED_THREADS 256
#define RED_BLOCKS_MAX 1184  // 8 per SM on 148 SMs

template <class T>
__device__ __forceinline__ T block_sum(T v) {
  __shared__ T red[32];
  v = warp_sum(v);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  T r = T(0);
  if (wid == 0) {
    int nw = (blockDim.x + 31) >> 5;
    r = lane < nw ? red[lane] : T(0);
    r = warp_sum(r);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

size_t cs_reduce_partials(int64_t n) {
  int64_t nb = (n + RED_THREADS - 1) / RED_THREADS;
  if (nb > RED_BLOCKS_MAX) nb = RED_BLOCKS_MAX;
  if (nb < 1) nb = 1;
  return (size_t)nb;
}

__global__ void k_reduce_final(const double *part, int64_t np, double *out, int accumulate) {
  double s = 0;
  for (int64_t i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) out[0] = accumulate ? out[0] + s : s;
}

int cs_reduce_sum_f64(const double *partials, int64_t np, double *out_dev, int accumulate,
                      cudaStream_t st) {
  k_reduce_final<<<1, 1024, 0, st>>>(partials, np, out_dev, accumulate);
  return cs_check_launch("reduce_final");
}

// sum of v^2 over three arrays (kinetic energy) or plain sums (momentum)
template <bool SQUARE>
__global__ void k_partial3(int64_t n, const double *a, const double *b, const double *c,
                           double *part, int comp) {
  double s = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (SQUARE)
      s += a[i] * a[i] + b[i] * b[i] + c[i] * c[i];
    else
      s += (comp == 0 ? a[i] : comp == 1 ? b[i] : c[i]);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_scale_scalar(double *p, double f) { p[0] *= f; }

extern "C" size_t cs_reduce_ws_bytes(int64_t n) {
  return cs_ws_slice(sizeof(double) * cs_reduce_partials(n)) + cs_ws_slice(8 * sizeof(double));
}

extern "C" int cs_kinetic(int64_t n, double mass, const double *vx, const double *vy,
                          const double *vz, double *out_dev, void *ws, size_t ws_bytes,
                          void *stream) {
  cudaStream_t st = cs_stream(stream);
  cs_ws w(ws, ws_bytes);
  size_t nb = cs_reduce_partials(n);
  CS_WS_TAKE(w, double, part, nb);
  k_partial3<true><<<(unsigned)nb, RED_THREADS, 0, st>>>(n, vx, vy, vz, part, 0);
  CS_TRY(cs_reduce_sum_f64(part, (int64_t)nb, out_dev, 0, st));
  k_scale_scalar<<<1, 1, 0, st>>>(out_dev, 0.5 * mass);
  return cs_check_launch("kinetic");
}

extern "C" int cs_sum3(int64_t n, const double *ax, const double *ay, const double *az,
                       double *out_dev, void *ws, size_t ws_bytes, void *stream) {
  cudaStream_t st = cs_stream(stream);
  cs_ws w(ws, ws_bytes);
  size_t nb = cs_reduce_partials(n);
  CS_WS_TAKE(w, double, part, nb);
  for (int c = 0; c < 3; ++c) {
    k_partial3<false><<<(unsigned)nb, RED_THREADS, 0, st>>>(n, ax, ay, az, part, c);
    CS_TRY(cs_reduce_sum_f64(part, (int64_t)nb, out_dev + c, 0, st));
  }
  return cs_check_launch("sum3");
}
