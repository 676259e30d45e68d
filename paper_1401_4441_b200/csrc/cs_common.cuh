// cs_common.cuh -- shared device/host helpers for the sm_100a kernels.
// The library is ONE translation unit (cs_lib.cu includes every module), so
// __constant__ tables and static helpers need no relocatable device code.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/cellsched_b200.h"

#define CS_WARP 32
#define CS_FULL 0xffffffffu

// ---------------------------------------------------------------- errors --
void cs_set_error(const char *fmt, ...);
int cs_check_launch(const char *what);  // cudaGetLastError -> status

#define CS_TRY(expr)                  \
  do {                                \
    int _st = (expr);                 \
    if (_st != CS_OK) return _st;     \
  } while (0)

#define CS_CUDA(expr)                                                          \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      cs_set_error("%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                   __LINE__);                                                  \
      return (int)_e;                                                          \
    }                                                                          \
  } while (0)

#define CS_REQUIRE(cond, ...)      \
  do {                             \
    if (!(cond)) {                 \
      cs_set_error(__VA_ARGS__);   \
      return CS_EINVAL;            \
    }                              \
  } while (0)

static inline cudaStream_t cs_stream(void *s) { return (cudaStream_t)s; }

// one-time per-device set-up (constant tables, kernel attributes, occupancy
// caps) is cached per device: __constant__ memory and function attributes
// are per device, so a process that calls the library on a second GPU must
// set them up there too
#define CS_MAX_DEVICES 64
static inline int cs_device_index() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0) d = 0;
  return d < CS_MAX_DEVICES ? d : CS_MAX_DEVICES - 1;
}

// ------------------------------------------------------------- workspace --
// bump allocator over the caller workspace (256-byte aligned slices)
struct cs_ws {
  char *base;
  size_t size, used;
  __host__ cs_ws(void *p, size_t n) : base((char *)p), size(n), used(0) {}
  template <class T>
  __host__ T *take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~(size_t)255;
    if (used + bytes > size || base == nullptr) return nullptr;
    T *p = (T *)(base + used);
    used += bytes;
    return p;
  }
};
#define CS_WS_TAKE(ws, T, var, count)                                           \
  T *var = (ws).take<T>(count);                                                 \
  if (!var) {                                                                   \
    cs_set_error("workspace too small at %s (%zu bytes used of %zu)", #var,     \
                 (ws).used, (ws).size);                                         \
    return CS_ECAPACITY;                                                        \
  }
static inline size_t cs_ws_slice(size_t bytes) { return (bytes + 255) & ~(size_t)255; }

// ------------------------------------------------------------ scans (host) --
// exclusive scan of int32 counts -> int32 offsets (out has n+1 entries,
// out[n] = total).  Scratch from cs_scan_ws_bytes(n).
size_t cs_scan_ws_bytes(int64_t n);
int cs_exclusive_scan_i32(const int32_t *in, int32_t *out, int64_t n, void *ws, size_t ws_bytes,
                          cudaStream_t st);
// deterministic fixed-order reductions (host launchers)
size_t cs_reduce_partials(int64_t n);  // number of partials used for n elements
int cs_reduce_sum_f64(const double *partials, int64_t np, double *out_dev, int accumulate,
                      cudaStream_t st);

// ----------------------------------------------------------- device utils --
__device__ __forceinline__ uint64_t cs_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static inline uint64_t cs_splitmix64_host(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CS_FULL, v, o);
  return v;
}

// canonical 3D half stencil (grid.py:192-200), zero offset first
struct cs_offsets {
  int8_t o[14][3];
  int8_t axis[14];  // highest axis with a nonzero component (loopex parity axis)
};
__constant__ cs_offsets c_stencil3;  // single translation unit (cs_lib.cu)
void cs_host_canonical_stencil(int dim, int8_t *out /* n*dim */, int *n);
int cs_upload_stencil(void);

__host__ __device__ __forceinline__ int cs_wrap(int v, int e) {
  v %= e;
  return v < 0 ? v + e : v;
}
