// cs_force2.cuh -- K2 v3: half-shell "super-task" per warp inside a block CTA.
//
// A CTA owns one block of Bx*By*Bz home cells.  One warp evaluates the whole
// half shell of one home cell h -- the 14 tasks (intra + 13 offsets) that
// generate_basic emits per cell (taskgen.py:188-198):
//
//   0. tables: for every (home h, entry e) the source cell's start/count and
//      periodic image shift, and a slot base for the reaction buffer.
//   1. cull: a j whose distance to h's box is >= rc cannot reach any i of h;
//      survivors are compacted into the warp's list as (entry, index).
//   2. filter: lanes hold 32 j's, 8 home i's are broadcast from shared
//      memory; each lane builds an 8-bit hit mask (r^2 < rc^2 in fp64).
//   3. hit loop: every lane walks its own set bits, computes f_ij once
//      (fast reciprocal: MUFU.RCP64H + 2 Newton steps), keeps -f_ij on j in
//      registers and adds +f_ij into its private row of i partials.
//   4. reactions go to the slot of (h, e, j): a fixed offset e has exactly one
//      writer per target cell, so the block's warps never collide (the
//      paper's buffered strategy inside the block); i rows are reduced per
//      row block.
//   5. after one barrier the CTA merges, per footprint cell in a fixed
//      order, home rows + reaction slots: either read-modify-write into
//      global f (CS_SCHED_SHELL: 8 passes of a 2x2x2 block colouring, same-
//      colour footprints are disjoint) or plain stores into the block's
//      private footprint buffer (CS_SCHED_BUFFERED: one pass over all
//      blocks, then k_gather_blocks sums the <= 8 buffers per particle).
//
// No atomics on forces, no intra-CTA dependency levels, deterministic order.
#pragma once
#include "cs_force.cuh"

#define SH_NW 8        // warps per CTA (one home cell each for 2x2x2 blocks)
#define SH_IB 16       // home particles per row block (= i-owner lanes)
#define SH_FB 128      // hit window: forces staged per warp
#define SH_DCAP 512    // hit descriptors per chunk (32 j x 16 i)
#define SH_JCAP 384    // j list capacity per warp (>= particles of the 14 source cells)
#define SH_RCAP 1440   // reaction slots (particles) per CTA
#define SH_HCAP 160    // home particles per CTA
#define SH_MAXB 8      // home cells per CTA
#define SH_MAXF 64     // footprint cells per CTA ((Bx+1)(By+2)(Bz+2))
#define SH_MAXC 8      // contributors per footprint cell

struct MergeTable {              // host-built per block shape
  uint8_t n[SH_MAXF];            // contributors of footprint cell lc
  uint8_t he[SH_MAXF][SH_MAXC];  // h * 16 + e (e = 0: home rows)
  int nfc;
};

struct ShellSmem {
  double R[3][SH_RCAP];              // reaction slots (e >= 1)
  double Fh[3][SH_HCAP];             // home rows (e = 0)
  double hxd[SH_NW][SH_IB][4];       // home positions (fp64, exact re-test)
  float4 hxf[SH_NW][SH_IB];          // home positions relative to the cell (fp32 filter)
  double fb[SH_NW][3][SH_FB];        // forces of the current hit window
  uint16_t desc[SH_NW][SH_DCAP];     // hit descriptors (j lane << 5 | i), j-major
  int seg[SH_NW][32];                // lane j: first descriptor of its hits
  unsigned msk[SH_NW][32];           // lane j: hit mask over the row block
  double sh[SH_MAXB][14][3];         // image shift of source (h, e)
  uint16_t jl[SH_NW][SH_JCAP];       // j list: entry << 12 | index in source cell
  int sstart[SH_MAXB][14];           // global start of source (h, e)
  int scount[SH_MAXB][14];           // count of source (h, e), -1: none
  int sbase[SH_MAXB][14];            // slot base (Fh for e = 0, R for e >= 1)
  int fstart[SH_MAXF + 1];           // footprint cell -> offset in the block buffer
  int fgstart[SH_MAXF];              // footprint cell -> global start (-1: none)
  int hcell[SH_MAXB];
  int overflow;
};

__device__ __forceinline__ double box_d2(double x, double lo, double hi) {
  const double d = fmax(fmax(lo - x, 0.0), x - hi);
  return d * d;
}

// 1/a to ~1 ulp: hardware approximation + two Newton-Raphson steps
__device__ __forceinline__ double fast_rcp(double a) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  double e = __fma_rn(-a, y, 1.0);
  y = __fma_rn(y, e, y);
  e = __fma_rn(-a, y, 1.0);
  return __fma_rn(y, e, y);
}

__device__ __forceinline__ int wrap1i(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

struct ShellArgs {
  ForceArgs A;
  MergeTable mt;
  double *buf;            // buffered mode: footprint buffers, 3 components x bufstride
  const int *boff;        // buffered mode: per-block offset into buf
  int *bindex;            // buffered mode: per block fstart[0..SH_MAXF]
  int64_t bufstride;
  unsigned *err;          // capacity overflow flag (buffered mode)
};

// block coordinates -> global cell of a footprint cell (or -1)
__device__ __forceinline__ int64_t foot_cell(const Box &b, const int *o0, int lc, int FX, int FY) {
  int v0 = o0[0] + lc % FX, v1 = o0[1] + (lc / FX) % FY - 1, v2 = o0[2] + lc / (FX * FY) - 1;
  if (b.per[0]) v0 = wrap1i(v0, b.nc[0]); else if (v0 < 0 || v0 >= b.nc[0]) return -1;
  if (b.per[1]) v1 = wrap1i(v1, b.nc[1]); else if (v1 < 0 || v1 >= b.nc[1]) return -1;
  if (b.per[2]) v2 = wrap1i(v2, b.nc[2]); else if (v2 < 0 || v2 >= b.nc[2]) return -1;
  return box_cell(b, v0, v1, v2);
}

template <bool ENERGY, bool BUFFERED>
__global__ void __launch_bounds__(SH_NW * 32, 2) k_force_shell(ShellArgs SA, int colour) {
  extern __shared__ __align__(16) unsigned char sh_raw[];
  ShellSmem &S = *reinterpret_cast<ShellSmem *>(sh_raw);
  const ForceArgs &A = SA.A;
  const Box &b = A.b;
  const int B0 = b.blk[0], B1 = b.blk[1], B2 = b.blk[2];
  const int nhome = B0 * B1 * B2;
  int o0[3];
  int bid = blockIdx.x;
  if (BUFFERED) {
    o0[0] = (bid % A.nbk[0]) * B0;
    o0[1] = ((bid / A.nbk[0]) % A.nbk[1]) * B1;
    o0[2] = (bid / (A.nbk[0] * A.nbk[1])) * B2;
  } else {
    const int kc0 = colour & 1, kc1 = (colour >> 1) & 1, kc2 = (colour >> 2) & 1;
    const int cnt0 = (A.nbk[0] - kc0 + 1) >> 1, cnt1 = (A.nbk[1] - kc1 + 1) >> 1;
    o0[0] = (2 * (bid % cnt0) + kc0) * B0;
    o0[1] = (2 * ((bid / cnt0) % cnt1) + kc1) * B1;
    o0[2] = (2 * (bid / (cnt0 * cnt1)) + kc2) * B2;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int FX = B0 + 1, FY = B1 + 2;
  const int nfc = SA.mt.nfc;

  // ---- 0. source tables, one thread per (h, e); footprint cells
  for (int t = threadIdx.x; t < nhome * 14; t += blockDim.x) {
    const int h = t / 14, e = t - 14 * h;
    const int hg0 = o0[0] + h % B0, hg1 = o0[1] + (h / B0) % B1, hg2 = o0[2] + h / (B0 * B1);
    int cnt = -1, st = 0;
    double s0 = 0, s1 = 0, s2 = 0;
    const bool home_ok = hg0 < b.owned_x;
    if (home_ok) {
      int v0 = hg0 + c_stencil3.o[e][0], v1 = hg1 + c_stencil3.o[e][1], v2 = hg2 + c_stencil3.o[e][2];
      bool ok = true;
      if (b.per[0]) { s0 = v0 >= b.nc[0] ? b.L[0] : (v0 < 0 ? -b.L[0] : 0.0); v0 = wrap1i(v0, b.nc[0]); }
      else ok = ok && v0 >= 0 && v0 < b.nc[0];
      if (b.per[1]) { s1 = v1 >= b.nc[1] ? b.L[1] : (v1 < 0 ? -b.L[1] : 0.0); v1 = wrap1i(v1, b.nc[1]); }
      else ok = ok && v1 >= 0 && v1 < b.nc[1];
      if (b.per[2]) { s2 = v2 >= b.nc[2] ? b.L[2] : (v2 < 0 ? -b.L[2] : 0.0); v2 = wrap1i(v2, b.nc[2]); }
      else ok = ok && v2 >= 0 && v2 < b.nc[2];
      if (ok) {
        const int64_t gc = box_cell(b, v0, v1, v2);
        st = A.start[gc];
        cnt = A.start[gc + 1] - st;
      }
    }
    if (e == 0) S.hcell[h] = home_ok ? (int)box_cell(b, hg0, hg1, hg2) : -1;
    S.sstart[h][e] = st;
    S.scount[h][e] = cnt;
    S.sh[h][e][0] = s0;
    S.sh[h][e][1] = s1;
    S.sh[h][e][2] = s2;
  }
  for (int lc = threadIdx.x; lc < nfc; lc += blockDim.x) {
    const int64_t gc = foot_cell(b, o0, lc, FX, FY);
    S.fgstart[lc] = gc >= 0 ? A.start[gc] : -1;
    S.fstart[lc + 1] = gc >= 0 ? A.start[gc + 1] - A.start[gc] : 0;
  }
  __syncthreads();
  if (wid == 0) {  // slot bases (scan over (h, e)), list capacity, footprint offsets
    int fb = 0, rb = 0;
    for (int t0 = 0; t0 < nhome * 14; t0 += 32) {
      const int t = t0 + lane;
      const int h = t / 14, e = t - 14 * (t / 14);
      const int c = t < nhome * 14 ? max(S.scount[h][e], 0) : 0;
      const int ch = (t < nhome * 14 && e == 0) ? c : 0;
      const int cr = (t < nhome * 14 && e != 0) ? c : 0;
      int ih = ch, ir = cr;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const int vh = __shfl_up_sync(CS_FULL, ih, s), vr = __shfl_up_sync(CS_FULL, ir, s);
        if (lane >= s) { ih += vh; ir += vr; }
      }
      if (t < nhome * 14) S.sbase[h][e] = e == 0 ? fb + ih - ch : rb + ir - cr;
      fb += __shfl_sync(CS_FULL, ih, 31);
      rb += __shfl_sync(CS_FULL, ir, 31);
    }
    int src_max = 0;
    for (int h = 0; h < nhome; ++h) {
      const int c = warp_sum(lane < 14 ? max(S.scount[h][lane], 0) : 0);
      src_max = max(src_max, c);
    }
    int carry = 0;
    for (int c0 = 0; c0 < nfc; c0 += 32) {
      const int lc = c0 + lane;
      const int v = lc < nfc ? S.fstart[lc + 1] : 0;
      int inc = v;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const int u = __shfl_up_sync(CS_FULL, inc, s);
        if (lane >= s) inc += u;
      }
      if (lc < nfc) S.fstart[lc + 1] = carry + inc;
      carry += __shfl_sync(CS_FULL, inc, 31);
    }
    if (lane == 0) {
      S.fstart[0] = 0;
      S.overflow = (fb > SH_HCAP || rb > SH_RCAP || src_max > SH_JCAP) ? 1 : 0;
    }
  }
  __syncthreads();
  if (S.overflow) {
    if (BUFFERED) {  // no in-place fallback in buffered mode: report to the host
      if (threadIdx.x == 0) atomicExch(SA.err, 1u);
      return;
    }
    // colour mode fallback: v1 per-task routine on global memory under the 27
    // loop-exchange levels inside this block (still conflict-free)
    for (int level = 0; level < 27; ++level) {
      int e, par;
      level_entry(level, &e, &par);
      const int ax = c_stencil3.axis[e];
      for (int h = wid; h < nhome; h += SH_NW) {
        if (S.hcell[h] < 0 || S.scount[h][e] < 0) continue;
        const int hg[3] = {o0[0] + h % B0, o0[1] + (h / B0) % B1, o0[2] + h / (B0 * B1)};
        if (level > 0 && (hg[ax] & 1) != par) continue;
        const int a0 = S.sstart[h][0], na = S.scount[h][0];
        const int b0 = S.sstart[h][e], nb = S.scount[h][e];
        double pe = 0;
        unsigned hits = 0;
        task_warp<ENERGY>(A.x, A.y, A.z, a0, na, b0, nb, level == 0, S.sh[h][e][0], S.sh[h][e][1],
                          S.sh[h][e][2], A.fx + a0, A.fy + a0, A.fz + a0, A.fx + b0, A.fy + b0,
                          A.fz + b0, A.p, pe, hits);
        task_stats<ENERGY>(pe, hits, S.hcell[h], A.pe_cell, A.hits_cell);
      }
      __syncthreads();
    }
    return;
  }
  for (int i = threadIdx.x; i < SH_RCAP; i += blockDim.x) S.R[0][i] = S.R[1][i] = S.R[2][i] = 0.0;
  for (int i = threadIdx.x; i < SH_HCAP; i += blockDim.x) S.Fh[0][i] = S.Fh[1][i] = S.Fh[2][i] = 0.0;
  __syncthreads();

  const double edge0 = b.L[0] / b.gnc[0], edge1 = b.L[1] / b.gnc[1], edge2 = b.L[2] / b.gnc[2];
  const double cull2 = A.p.rc2 * (1.0 + 1e-12) + 1e-12;
  const double rc2 = A.p.rc2, sig2 = A.p.sig2, eps48 = A.p.eps48, eps4 = A.p.eps4;
  const float rc2f = (float)(rc2 + 1e-3);  // conservative fp32 prefilter bound (exact fp64 re-test)
  // ---- 1-4. one warp per home cell
  for (int h = wid; h < nhome; h += SH_NW) {
    if (S.hcell[h] < 0) continue;
    const int hg0 = o0[0] + h % B0, hg1 = o0[1] + (h / B0) % B1, hg2 = o0[2] + h / (B0 * B1);
    const int a0 = S.sstart[h][0], na = S.scount[h][0];
    const double lo0 = (b.x0 + hg0) * edge0, lo1 = hg1 * edge1, lo2 = hg2 * edge2;
    (void)cull2;
    // 1. j list = the 14 source cells concatenated (home first); lanes walk
    //    the concatenation directly
    const int mycnt = lane < 14 ? max(S.scount[h][lane], 0) : 0;
    int incl = mycnt;
#pragma unroll
    for (int s = 1; s < 16; s <<= 1) {
      const int v = __shfl_up_sync(CS_FULL, incl, s);
      if (lane >= s) incl += v;
    }
    const int excl = incl - mycnt;
    const int nj = __shfl_sync(CS_FULL, incl, 13);
    for (int t0 = 0; t0 < nj; t0 += 32) {
      const int t = t0 + lane;
      int e = 0;  // largest e with excl[e] <= t
#pragma unroll
      for (int st = 8; st >= 1; st >>= 1) {
        const int cand = e + st;
        const int ex = __shfl_sync(CS_FULL, excl, cand < 14 ? cand : 13);
        if (cand < 14 && ex <= t) e = cand;
      }
      const int q = t - __shfl_sync(CS_FULL, excl, e);
      if (t < nj) S.jl[wid][t] = (uint16_t)((e << 12) | q);
    }
    __syncwarp();
    double pe = 0;
    unsigned hits = 0;
    const int fh0 = S.sbase[h][0];
    for (int ib = 0; ib < na; ib += SH_IB) {
      const int nib = min(SH_IB, na - ib);
      if (lane < SH_IB) {
        const int ii = a0 + ib + min(lane, nib - 1);
        const double x = __ldg(A.x + ii), y = __ldg(A.y + ii), z = __ldg(A.z + ii);
        S.hxd[wid][lane][0] = x;
        S.hxd[wid][lane][1] = y;
        S.hxd[wid][lane][2] = z;
        S.hxf[wid][lane] = make_float4((float)(x - lo0), (float)(y - lo1), (float)(z - lo2), 0.f);
      }
      __syncwarp();
      const unsigned qmask = (1u << nib) - 1;
      double fix = 0, fiy = 0, fiz = 0;  // F_i of i-owner lane (i = ib + lane, lane < nib)
      for (int c0 = 0; c0 < nj; c0 += 32) {
        const int jj = c0 + lane;
        const bool vj = jj < nj;
        const int ent = vj ? S.jl[wid][jj] : 0;
        const int e = ent >> 12, q = ent & 0xFFF;
        double xj = 1e150, yj = 1e150, zj = 1e150;
        if (vj) {
          const int gj = S.sstart[h][e] + q;
          xj = __ldg(A.x + gj) + S.sh[h][e][0];
          yj = __ldg(A.y + gj) + S.sh[h][e][1];
          zj = __ldg(A.z + gj) + S.sh[h][e][2];
        }
        // 2. fp32 prefilter: 16 rows against this lane's j
        const float xf = (float)(xj - lo0), yf = (float)(yj - lo1), zf = (float)(zj - lo2);
        unsigned m = 0;
#pragma unroll
        for (int qq = 0; qq < SH_IB; ++qq) {
          const float4 p = S.hxf[wid][qq];
          const float dx = p.x - xf, dy = p.y - yf, dz = p.z - zf;
          m |= (unsigned)(__fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx)) < rc2f) << qq;
        }
        if (e == 0) m &= (q - ib <= 0) ? 0u : (q - ib >= SH_IB ? 0xFFFFu : ((1u << (q - ib)) - 1));
        m = vj ? (m & qmask) : 0u;
        // 3. j-major compaction of the hits into descriptors
        const int cnt = __popc(m);
        int ci = cnt;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
          const int v = __shfl_up_sync(CS_FULL, ci, s);
          if (lane >= s) ci += v;
        }
        const int seg = ci - cnt;
        const int T = __shfl_sync(CS_FULL, ci, 31);
        if (T == 0) continue;
        S.seg[wid][lane] = seg;
        S.msk[wid][lane] = m;
        {
          unsigned mm = m;
          int r = seg;
          while (mm) {
            const int qq = __ffs(mm) - 1;
            mm &= mm - 1;
            S.desc[wid][r++] = (uint16_t)((lane << 5) | qq);
          }
        }
        // transposed rows: bit jl of rowm = hit (i = lane, j = lane jl)
        unsigned rowm = 0;
#pragma unroll
        for (int qq = 0; qq < SH_IB; ++qq) {
          const unsigned bq = __ballot_sync(CS_FULL, (m >> qq) & 1u);
          if (lane == qq) rowm = bq;
        }
        __syncwarp();
        double gx = 0, gy = 0, gz = 0;  // reaction on this lane's j
        for (int w0 = 0; w0 < T; w0 += SH_FB) {  // hit windows (one in practice)
          const int wn = min(SH_FB, T - w0);
          for (int t0 = 0; t0 < wn; t0 += 32) {  // dense rounds: every lane one hit
            const int t = t0 + lane;
            const bool act = t < wn;
            const int d = act ? S.desc[wid][w0 + t] : 0;
            const int jl = d >> 5, qq = d & 31;
            const double xjl = __shfl_sync(CS_FULL, xj, jl), yjl = __shfl_sync(CS_FULL, yj, jl),
                         zjl = __shfl_sync(CS_FULL, zj, jl);
            double fx = 0, fy = 0, fz = 0;
            if (act) {
              const double dx = S.hxd[wid][qq][0] - xjl, dy = S.hxd[wid][qq][1] - yjl,
                           dz = S.hxd[wid][qq][2] - zjl;
              const double r2 = __fma_rn(dz, dz, __fma_rn(dy, dy, dx * dx));
              if (r2 < rc2) {  // exact test (same expression as the oracle)
                const double rinv2 = fast_rcp(r2);
                const double sr2 = sig2 * rinv2;
                const double sr6 = sr2 * sr2 * sr2;
                const double ff = eps48 * sr6 * (sr6 - 0.5) * rinv2;
                fx = ff * dx;
                fy = ff * dy;
                fz = ff * dz;
                if (ENERGY) pe += eps4 * sr6 * (sr6 - 1.0);
                ++hits;
              }
              S.fb[wid][0][t] = fx;
              S.fb[wid][1][t] = fy;
              S.fb[wid][2][t] = fz;
            }
          }
          __syncwarp();
          // F_j: this lane's hits are the contiguous descriptors [seg, seg+cnt)
          const int lo = max(seg, w0), hi = min(seg + cnt, w0 + wn);
          for (int t = lo; t < hi; ++t) {
            gx -= S.fb[wid][0][t - w0];
            gy -= S.fb[wid][1][t - w0];
            gz -= S.fb[wid][2][t - w0];
          }
          // F_i: i-owner lanes walk their row bits
          if (lane < nib) {
            for (unsigned mm = rowm; mm; mm &= mm - 1) {
              const int jl = __ffs(mm) - 1;
              const int pos = S.seg[wid][jl] + __popc(S.msk[wid][jl] & ((1u << lane) - 1)) - w0;
              if (pos >= 0 && pos < wn) {
                fix += S.fb[wid][0][pos];
                fiy += S.fb[wid][1][pos];
                fiz += S.fb[wid][2][pos];
              }
            }
          }
          __syncwarp();
        }
        if (cnt) {  // unique writer of slot (h, e, q)
          const int slot = S.sbase[h][e] + q;
          double *dst = e == 0 ? &S.Fh[0][slot] : &S.R[0][slot];
          const int stride = e == 0 ? SH_HCAP : SH_RCAP;
          dst[0] += gx;
          dst[stride] += gy;
          dst[2 * stride] += gz;
        }
        __syncwarp();
      }
      if (lane < nib) {  // own row (after this row block's intra reactions)
        S.Fh[0][fh0 + ib + lane] += fix;
        S.Fh[1][fh0 + ib + lane] += fiy;
        S.Fh[2][fh0 + ib + lane] += fiz;
      }
      __syncwarp();
    }
    hits = warp_sum(hits);
    if (ENERGY) pe = warp_sum(pe);
    if (lane == 0) {
      A.hits_cell[S.hcell[h]] += hits;
      if (ENERGY) A.pe_cell[S.hcell[h]] += pe;
    }
  }
  __syncthreads();
  // ---- 5. merge per footprint cell in a fixed order
  const int64_t boff = BUFFERED ? SA.boff[bid] : 0;
  for (int lc = wid; lc < nfc; lc += SH_NW) {
    const int g0 = S.fgstart[lc];
    if (g0 < 0) continue;
    const int n = S.fstart[lc + 1] - S.fstart[lc];
    const int nc = SA.mt.n[lc];
    for (int i = lane; i < n; i += 32) {
      double sx = 0, sy = 0, sz = 0;
      for (int k = 0; k < nc; ++k) {
        const int he = SA.mt.he[lc][k];
        const int hh = he >> 4, e = he & 15;
        if (S.hcell[hh] < 0) continue;
        const int s = S.sbase[hh][e] + i;
        if (e == 0) {
          sx += S.Fh[0][s];
          sy += S.Fh[1][s];
          sz += S.Fh[2][s];
        } else {
          sx += S.R[0][s];
          sy += S.R[1][s];
          sz += S.R[2][s];
        }
      }
      if (BUFFERED) {
        const int64_t o = boff + S.fstart[lc] + i;
        SA.buf[o] = sx;
        SA.buf[SA.bufstride + o] = sy;
        SA.buf[2 * SA.bufstride + o] = sz;
      } else {
        A.fx[g0 + i] += sx;
        A.fy[g0 + i] += sy;
        A.fz[g0 + i] += sz;
      }
    }
  }
  if (BUFFERED)
    for (int lc = threadIdx.x; lc <= nfc; lc += blockDim.x)
      SA.bindex[(int64_t)bid * (SH_MAXF + 1) + lc] = S.fstart[lc];
}

// buffered mode: footprint size per block (one warp per block, lanes over cells)
__global__ void k_block_sizes(ShellArgs SA, int32_t *sizes) {
  const ForceArgs &A = SA.A;
  const Box &b = A.b;
  const int64_t nb = (int64_t)A.nbk[0] * A.nbk[1] * A.nbk[2];
  const int FX = b.blk[0] + 1, FY = b.blk[1] + 2;
  const int lane = threadIdx.x & 31;
  for (int64_t bid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; bid < nb;
       bid += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int o0[3] = {(int)(bid % A.nbk[0]) * b.blk[0], (int)((bid / A.nbk[0]) % A.nbk[1]) * b.blk[1],
                       (int)(bid / ((int64_t)A.nbk[0] * A.nbk[1])) * b.blk[2]};
    int s = 0;
    for (int lc = lane; lc < SA.mt.nfc; lc += 32) {
      const int64_t gc = foot_cell(b, o0, lc, FX, FY);
      if (gc >= 0) s += A.start[gc + 1] - A.start[gc];
    }
    s = warp_sum(s);
    if (lane == 0) sizes[bid] = s;
  }
}

// buffered mode, pass 2: every particle sums the <= 8 block buffers whose
// footprint box contains its cell, in a fixed block order (deterministic).
// One warp per cell: lanes 0..7 resolve the 2x2x2 candidate blocks once.
__global__ void k_gather_blocks(ShellArgs SA) {
  const ForceArgs &A = SA.A;
  const Box &b = A.b;
  const int B0 = b.blk[0], B1 = b.blk[1], B2 = b.blk[2];
  const int FX = B0 + 1, FY = B1 + 2, FZ = B2 + 2;
  const int nc0 = b.nc[0], nc1 = b.nc[1];
  const int ncell = nc0 * nc1 * b.nc[2];
  const int warp = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= ncell) return;
  const int c0 = warp % nc0, c1 = (warp / nc0) % nc1, c2 = warp / (nc0 * nc1);
  const int64_t gc = box_cell(b, c0, c1, c2);
  const int g0 = A.start[gc], n = A.start[gc + 1] - g0;
  if (n == 0) return;
  // per axis: the block containing c and, at a block edge, the neighbour
  // block whose footprint reaches c (x: footprint reaches +1; y, z: -1, +B)
  int src = -1;
  if (lane < 8) {
    const int u = lane & 1, v = (lane >> 1) & 1, w = lane >> 2;
    int k0 = c0 / B0, k1 = c1 / B1, k2 = c2 / B2;
    bool ok = true;
    if (u) { if (c0 % B0 == 0) k0 -= 1; else ok = false; }
    if (v) { if (c1 % B1 == 0) k1 -= 1; else if (c1 % B1 == B1 - 1) k1 += 1; else ok = false; }
    if (w) { if (c2 % B2 == 0) k2 -= 1; else if (c2 % B2 == B2 - 1) k2 += 1; else ok = false; }
    if (k0 < 0 || k0 >= A.nbk[0]) { if (b.per[0]) k0 = wrap1i(k0, A.nbk[0]); else ok = false; }
    if (k1 < 0 || k1 >= A.nbk[1]) { if (b.per[1]) k1 = wrap1i(k1, A.nbk[1]); else ok = false; }
    if (k2 < 0 || k2 >= A.nbk[2]) { if (b.per[2]) k2 = wrap1i(k2, A.nbk[2]); else ok = false; }
    if (ok) {
      int l0 = c0 - k0 * B0, l1 = c1 - (k1 * B1 - 1), l2 = c2 - (k2 * B2 - 1);
      if (b.per[0]) l0 = wrap1i(l0, nc0);
      if (b.per[1]) l1 = wrap1i(l1, nc1);
      if (b.per[2]) l2 = wrap1i(l2, b.nc[2]);
      if (l0 >= 0 && l0 < FX && l1 >= 0 && l1 < FY && l2 >= 0 && l2 < FZ) {
        const int blin = k0 + A.nbk[0] * (k1 + A.nbk[1] * k2);
        src = SA.boff[blin] + SA.bindex[(int64_t)blin * (SH_MAXF + 1) + l0 + FX * (l1 + FY * l2)];
      }
    }
  }
  const unsigned have = __ballot_sync(CS_FULL, src >= 0);
  for (int i = lane; i < ((n + 31) & ~31); i += 32) {
    double sx = 0, sy = 0, sz = 0;
    for (unsigned m = have; m; m &= m - 1) {
      const int o = __shfl_sync(CS_FULL, src, __ffs(m) - 1) + i;
      if (i < n) {
        sx += SA.buf[o];
        sy += SA.buf[SA.bufstride + o];
        sz += SA.buf[2 * SA.bufstride + o];
      }
    }
    if (i < n) {
      A.fx[g0 + i] += sx;
      A.fy[g0 + i] += sy;
      A.fz[g0 + i] += sz;
    }
  }
}

static int build_merge_table(const int B[3], MergeTable *mt) {
  const int FX = B[0] + 1, FY = B[1] + 2, FZ = B[2] + 2;
  mt->nfc = FX * FY * FZ;
  CS_REQUIRE(mt->nfc <= SH_MAXF, "shell schedule: footprint %d cells > %d", mt->nfc, SH_MAXF);
  int8_t st[14 * 3];
  int n;
  cs_host_canonical_stencil(3, st, &n);
  for (int lc = 0; lc < mt->nfc; ++lc) {
    const int l[3] = {lc % FX, (lc / FX) % FY - 1, lc / (FX * FY) - 1};
    int k = 0;
    // home rows first, then entries in canonical order: a fixed summation order
    for (int e = 0; e < 14; ++e) {
      const int hl[3] = {l[0] - st[3 * e], l[1] - st[3 * e + 1], l[2] - st[3 * e + 2]};
      if (hl[0] < 0 || hl[0] >= B[0] || hl[1] < 0 || hl[1] >= B[1] || hl[2] < 0 || hl[2] >= B[2])
        continue;
      const int h = hl[0] + B[0] * (hl[1] + B[1] * hl[2]);
      CS_REQUIRE(k < SH_MAXC, "merge table overflow");
      mt->he[lc][k++] = (uint8_t)(h * 16 + e);
    }
    mt->n[lc] = (uint8_t)k;
  }
  return CS_OK;
}

static size_t shell_buffered_ws(const Box &b, int64_t n) {
  const int64_t nb = (int64_t)((b.owned_x + b.blk[0] - 1) / b.blk[0]) * (b.nc[1] / (b.blk[1] > 0 ? b.blk[1] : 1)) *
                     (b.nc[2] / (b.blk[2] > 0 ? b.blk[2] : 1)) + 1;
  return cs_ws_slice(sizeof(double) * 3 * (8 * n + 64)) + 2 * cs_ws_slice(sizeof(int32_t) * (nb + 1)) +
         cs_ws_slice(sizeof(int32_t) * nb * (SH_MAXF + 1)) + cs_scan_ws_bytes(nb) + cs_ws_slice(64);
}

static int launch_shell_passes(const ForceArgs &A, bool energy, bool buffered, cs_ws *w,
                               int64_t n, unsigned *status, cudaStream_t st) {
  const int B[3] = {A.b.blk[0], A.b.blk[1], A.b.blk[2]};
  CS_REQUIRE(B[0] * B[1] * B[2] <= SH_MAXB, "shell schedule: block has more than %d cells", SH_MAXB);
  ShellArgs SA;
  memset(&SA, 0, sizeof(SA));
  SA.A = A;
  CS_TRY(build_merge_table(B, &SA.mt));
  const size_t smem = sizeof(ShellSmem);
  static bool attr = false;
  if (!attr) {
    CS_CUDA(cudaFuncSetAttribute(k_force_shell<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CS_CUDA(cudaFuncSetAttribute(k_force_shell<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CS_CUDA(cudaFuncSetAttribute(k_force_shell<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CS_CUDA(cudaFuncSetAttribute(k_force_shell<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  if (buffered) {
    const int64_t nblocks = (int64_t)A.nbk[0] * A.nbk[1] * A.nbk[2];
    CS_WS_TAKE(*w, double, buf, 3 * (8 * n + 64));
    CS_WS_TAKE(*w, int32_t, sizes, nblocks + 1);
    CS_WS_TAKE(*w, int32_t, boff, nblocks + 1);
    CS_WS_TAKE(*w, int32_t, bindex, nblocks * (SH_MAXF + 1));
    size_t sb = cs_scan_ws_bytes(nblocks);
    void *scratch = w->take<char>(sb);
    CS_REQUIRE(scratch, "workspace too small (buffered scan)");
    CS_WS_TAKE(*w, unsigned, err, 16);
    SA.buf = buf;
    SA.boff = boff;
    SA.bindex = bindex;
    SA.bufstride = 8 * n + 64;
    SA.err = status ? status : err;
    k_block_sizes<<<grid_for(nblocks * 32, 256), 256, 0, st>>>(SA, sizes);
    CS_TRY(cs_exclusive_scan_i32(sizes, boff, nblocks, scratch, sb, st));
    if (energy)
      k_force_shell<true, true><<<(unsigned)nblocks, SH_NW * 32, smem, st>>>(SA, -1);
    else
      k_force_shell<false, true><<<(unsigned)nblocks, SH_NW * 32, smem, st>>>(SA, -1);
    const int64_t ncell = (int64_t)A.b.nc[0] * A.b.nc[1] * A.b.nc[2];
    k_gather_blocks<<<(unsigned)((ncell * 32 + 255) / 256), 256, 0, st>>>(SA);
    return cs_check_launch("force_buffered");
  }
  for (int colour = 0; colour < 8; ++colour) {
    const int kc[3] = {colour & 1, (colour >> 1) & 1, (colour >> 2) & 1};
    unsigned blocks = 1;
    for (int k = 0; k < 3; ++k) blocks *= (unsigned)((A.nbk[k] - kc[k] + 1) >> 1);
    if (!blocks) continue;
    if (energy)
      k_force_shell<true, false><<<blocks, SH_NW * 32, smem, st>>>(SA, colour);
    else
      k_force_shell<false, false><<<blocks, SH_NW * 32, smem, st>>>(SA, colour);
  }
  return cs_check_launch("force_shell");
}
