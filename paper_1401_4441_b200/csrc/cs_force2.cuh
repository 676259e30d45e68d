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
#include <type_traits>

#include "cs_force.cuh"

#define SH_NW 8        // warps per CTA (one home cell each for 2x2x2 blocks)
#define SH_IB 4        // home particles per filter row block
#define SH_JCAP 384    // j list capacity per warp (>= particles of the 14 source cells)
#define SH_RCAP 1440   // reaction slots (particles) per CTA
#define SH_HCAP 160    // home particles per CTA
#define SH_MAXB 8      // home cells per CTA
#define SH_MAXF 64     // footprint cells per CTA ((Bx+1)(By+2)(Bz+2))
#define SH_MAXC 8      // contributors per footprint cell
// Verlet mode (cells of edge >= rc + skin, ~20 particles per cell)
#define VL_RCAP 2560   // reaction slots per CTA
#define VL_HCAP 256    // home particles per CTA
#define VL_RMAX 64     // rounds per home cell in the round tables
#define VL_IDLE 0x0F00u  // idle slot descriptor (entry 15, index 0)

struct MergeTable {              // host-built per block shape
  uint8_t n[SH_MAXF];            // contributors of footprint cell lc
  uint8_t he[SH_MAXF][SH_MAXC];  // h * 16 + e (e = 0: home rows)
  int nfc;
};

template <int RCAP_, int HCAP_, int QN>
struct ShellBase {
  static constexpr int RCAP = RCAP_, HCAP = HCAP_;
  double RF[3][RCAP + HCAP];         // reaction slots (e >= 1), then home rows (e = 0)
  double sh[SH_MAXB][16][3];         // image shift of source (h, e); e = 15: idle
  int sstart[SH_MAXB][16];           // global start of source (h, e)
  int scount[SH_MAXB][16];           // count of source (h, e), -1: none
  int sbase[SH_MAXB][16];            // slot base in RF (home rows for e = 0)
  int fstart[SH_MAXF + 1];           // footprint cell -> offset in the block buffer
  int fgstart[SH_MAXF];              // footprint cell -> global start (-1: none)
  int hcell[SH_MAXB];
  int16_t mt_base[SH_MAXF][SH_MAXC];  // merge: slot base of each contributor (-1: home not owned)
  int pend[QN];                    // Verlet: contributing homes still running per footprint cell
  int queue[QN];                   // Verlet: footprint cells ready to merge, in order (-1: not yet)
  int qtail, qhead;
  int nq;                          // Verlet: non-empty footprint cells (merge-queue length)
  int rtot, htot;                  // reaction slots / home rows in use (zeroed per block)
  int overflow;
  uint8_t mt_n[SH_MAXF];           // merge-table counts in shared memory (lanes of one warp
                                   //   read different cells: divergent constant reads serialise)
  // Verlet dataflow: the lower-colour neighbour blocks this block's merges
  // must follow (flag indices, -1 = none) and whether they have published
  int dep[27];
  int depok;
};
struct ShellSmem : ShellBase<SH_RCAP, SH_HCAP, 1> {  // link-cell super-tasks
  double rows[SH_NW][SH_IB][3][32];  // per-lane i partials
  double hx[SH_NW][SH_IB][4];        // broadcast home positions
  uint16_t jl[SH_NW][SH_JCAP];       // j list: entry << 12 | index in source cell
};
struct ShellSmemVL : ShellBase<VL_RCAP, VL_HCAP, SH_MAXF> {};  // Verlet round tables


// streamed round-table descriptor: read-only path without an L1 line, so the
// descriptors (each read once) do not evict the partner positions, which are
// reused from L1 (measured: force kernel 214 -> 210 us on cfg2; the kernel is
// L1-capacity sensitive -- a 228 KB shared-memory carveout costs 15%)
__device__ __forceinline__ unsigned ld_desc(const uint16_t *p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
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

// Verlet mode, steps 1-4 for every home cell of this warp.  The round table
// of home cell h (cs_verlet.cuh) gives every lane a first home particle and
// possibly a second one from a switch round on; per round a lane has at most
// one partner j (stencil entry << 8 | index in the source cell) and no j
// appears twice in a round.  So F_i stays in registers, and the reaction on
// j is a read-modify-write of its (h, e) slot that no other lane touches in
// that round (no atomics).  Every listed pair is re-tested exactly
// (r^2 < rc^2).  Descriptors are prefetched two rounds ahead and partner
// positions one round ahead (the image shift is added when used).
// one listed pair of round-table descriptor d with partner position (xj, yj,
// zj) (unshifted): returns the force on i (0 if idle or r >= rc)
template <bool ENERGY, bool SHIFT, class SM>
__device__ __forceinline__ bool verlet_pair(SM &S, const ForceArgs &A, int h, unsigned d,
                                            double xi, double yi, double zi, double xj, double yj,
                                            double zj, double &fx, double &fy, double &fz,
                                            double &pe) {
  const int e = d >> 8;
  double dx, dy, dz;
  if (SHIFT) {  // home cell at a periodic face: image shift per entry (entry 15: 1e150)
    dx = xi - (xj + S.sh[h][e][0]);
    dy = yi - (yj + S.sh[h][e][1]);
    dz = zi - (zj + S.sh[h][e][2]);
  } else {
    dx = xi - xj;
    dy = yi - yj;
    dz = zi - zj;
  }
  double r2 = __fma_rn(dz, dz, __fma_rn(dy, dy, dx * dx));
  if (!SHIFT && e == 15) r2 = 1e300;
  const bool hit = r2 < A.p.rc2;
  // evaluated for every listed pair (misses select a zero force), so the two
  // pairs of a round pair form one basic block and their chains interleave
  const double ri = fast_rcp(hit ? r2 : 1.0);
  const double s2 = A.p.sig2 * ri;
  const double s6 = s2 * s2 * s2;
  const double ff = hit ? A.p.eps48 * s6 * (s6 - 0.5) * ri : 0.0;
  fx = ff * dx;
  fy = ff * dy;
  fz = ff * dz;
  if (ENERGY) pe += hit ? A.p.eps4 * s6 * (s6 - 1.0) : 0.0;
  return hit;
}

// Newton-3 reaction of a hit into the (h, e) slot of j: no other lane writes
// this slot in this round
// (slot = S.sbase[h][entry] + index, looked up before the force math so its
// latency is hidden; the three components are read before any is written)
template <class SM>
__device__ __forceinline__ void verlet_react(SM &S, int slot, double fx, double fy, double fz) {
  constexpr int stride = SM::RCAP + SM::HCAP;
  double *dst = &S.RF[0][slot];
  const double a = dst[0], b = dst[stride], c = dst[2 * stride];
  dst[0] = a - fx;
  dst[stride] = b - fy;
  dst[2 * stride] = c - fz;
}

// Per-warp home data loaded at block start, before the table copy lands, so
// their latency overlaps the prologue: lane map, round count, the first four
// descriptors, then (after the copy) the lane's home particle positions.
struct VPre {
  int cell, nr, pA, pB, sw, a0;
  unsigned d0, d1, d2, d3;
  double xi, yi, zi, xb, yb, zb;
};

__device__ __forceinline__ void vl_pre_issue(const ForceArgs &A, const int *o0, int wid, int lane,
                                             VPre &v) {
  const Box &b = A.b;
  const int B0 = b.blk[0], B1 = b.blk[1], B2 = b.blk[2];
  v.cell = -1;
  v.nr = 0;
  v.pA = v.pB = 0xFF;
  v.sw = 0;
  v.a0 = 0;
  v.d0 = v.d1 = v.d2 = v.d3 = VL_IDLE;
  if (wid >= B0 * B1 * B2) return;
  const int hg0 = o0[0] + wid % B0, hg1 = o0[1] + (wid / B0) % B1, hg2 = o0[2] + wid / (B0 * B1);
  if (hg0 >= b.owned_x) return;
  v.cell = (int)box_cell(b, hg0, hg1, hg2);
  v.nr = __ldg(A.vl_nround + v.cell);
  const uint8_t *lm = A.vl_imap + (int64_t)v.cell * 96;
  v.pA = __ldg(lm + lane);
  v.pB = __ldg(lm + 32 + lane);
  v.sw = __ldg(lm + 64 + lane);
  const uint16_t *dp = A.vl_desc + (int64_t)v.cell * (VL_RMAX * 32) + lane;
  v.d0 = ld_desc(dp);
  v.d1 = ld_desc(dp + 32);
  v.d2 = ld_desc(dp + 64);
  v.d3 = ld_desc(dp + 96);
  v.a0 = __ldg(A.start + v.cell);
}

__device__ __forceinline__ void vl_pre_positions(const ForceArgs &A, VPre &v) {
  v.xi = v.yi = v.zi = v.xb = v.yb = v.zb = 0.0;
  if (v.cell < 0) return;
  if (v.nr < 4) {  // rounds past the table are idle
    if (v.nr < 1) v.d0 = VL_IDLE;
    if (v.nr < 2) v.d1 = VL_IDLE;
    if (v.nr < 3) v.d2 = VL_IDLE;
    v.d3 = VL_IDLE;
  }
  if (v.pA != 0xFF) {
    v.xi = __ldg(A.x + v.a0 + v.pA);
    v.yi = __ldg(A.y + v.a0 + v.pA);
    v.zi = __ldg(A.z + v.a0 + v.pA);
  }
  if (v.pB != 0xFF) {
    v.xb = __ldg(A.x + v.a0 + v.pB);
    v.yb = __ldg(A.y + v.a0 + v.pB);
    v.zb = __ldg(A.z + v.a0 + v.pB);
  }
}

// Rounds are taken in pairs (the builder aligns switch rounds to even): the
// two pairs of a lane are independent chains (ILP); their reactions are
// written round by round, each round's j being distinct.  Descriptors are
// prefetched two rounds ahead of the pair being computed, positions one.
template <bool ENERGY, bool SHIFT, class SM>
__device__ __forceinline__ void verlet_table(SM &S, const ForceArgs &A, int h, const VPre &v,
                                             const uint16_t *dp, double *fa, double *fb,
                                             double &pe, unsigned &hits) {
  const int nr = v.nr, sw = v.sw;
  double xi = v.xi, yi = v.yi, zi = v.zi;
  const double xb = v.xb, yb = v.yb, zb = v.zb;
  double fx_ = 0, fy_ = 0, fz_ = 0;
  // idle slots (entry 15) read a real particle and never pass the r^2 test
  unsigned d0 = v.d0, d1 = v.d1, d2 = v.d2, d3 = v.d3;
  int g = S.sstart[h][d0 >> 8] + (d0 & 255);
  double x0 = __ldg(A.x + g), y0 = __ldg(A.y + g), z0 = __ldg(A.z + g);
  g = S.sstart[h][d1 >> 8] + (d1 & 255);
  double x1 = __ldg(A.x + g), y1 = __ldg(A.y + g), z1 = __ldg(A.z + g);
  dp += 128;
#pragma unroll 2
  for (int r = 0; r < nr; r += 2) {
    if (r == sw) {  // this lane continues with its second particle
      fa[0] = fx_;
      fa[1] = fy_;
      fa[2] = fz_;
      fx_ = fy_ = fz_ = 0;
      xi = xb;
      yi = yb;
      zi = zb;
    }
    const unsigned d4 = r + 4 < nr ? ld_desc(dp) : VL_IDLE;
    const unsigned d5 = r + 5 < nr ? ld_desc(dp + 32) : VL_IDLE;
    dp += 64;
    g = S.sstart[h][d2 >> 8] + (d2 & 255);
    const double x2 = __ldg(A.x + g), y2 = __ldg(A.y + g), z2 = __ldg(A.z + g);
    g = S.sstart[h][d3 >> 8] + (d3 & 255);
    const double x3 = __ldg(A.x + g), y3 = __ldg(A.y + g), z3 = __ldg(A.z + g);
    const int slot0 = S.sbase[h][d0 >> 8] + (d0 & 255), slot1 = S.sbase[h][d1 >> 8] + (d1 & 255);
    double ux, uy, uz, vx, vy, vz;
    const bool h0 = verlet_pair<ENERGY, SHIFT>(S, A, h, d0, xi, yi, zi, x0, y0, z0, ux, uy, uz, pe);
    const bool h1 = verlet_pair<ENERGY, SHIFT>(S, A, h, d1, xi, yi, zi, x1, y1, z1, vx, vy, vz, pe);
    fx_ += ux + vx;
    fy_ += uy + vy;
    fz_ += uz + vz;
    hits += (unsigned)h0 + (unsigned)h1;
    if (h0) verlet_react(S, slot0, ux, uy, uz);
    __syncwarp();
    if (h1) verlet_react(S, slot1, vx, vy, vz);
    __syncwarp();
    d0 = d2;
    d1 = d3;
    d2 = d4;
    d3 = d5;
    x0 = x2;
    y0 = y2;
    z0 = z2;
    x1 = x3;
    y1 = y3;
    z1 = z3;
  }
  if (sw < nr) {
    fb[0] = fx_;
    fb[1] = fy_;
    fb[2] = fz_;
  } else {
    fa[0] = fx_;
    fa[1] = fy_;
    fa[2] = fz_;
  }
}

// lanes whose FIRST particle is p are contiguous and at most VB_SEG (4) long:
// a two-step segmented reduction, then the first lane of each run adds the
// particle's F_i into its home row.  A particle is the SECOND particle of at
// most one lane, so those partials are added directly, after the first ones.
template <class SM>
__device__ __forceinline__ void verlet_fi(SM &S, int h, int lane, int im, double fix, double fiy,
                                          double fiz, int im2, double fbx, double fby, double fbz) {
#pragma unroll
  for (int s = 1; s < 4; s <<= 1) {
    const double ux = __shfl_down_sync(CS_FULL, fix, s);
    const double uy = __shfl_down_sync(CS_FULL, fiy, s);
    const double uz = __shfl_down_sync(CS_FULL, fiz, s);
    const int ui = __shfl_down_sync(CS_FULL, im, s);
    if (lane + s < 32 && ui == im) {
      fix += ux;
      fiy += uy;
      fiz += uz;
    }
  }
  const int prev = __shfl_up_sync(CS_FULL, im, 1);
  if (im != 0xFF && (lane == 0 || prev != im)) {
    const int slot = S.sbase[h][0] + im;
    S.RF[0][slot] += fix;
    S.RF[1][slot] += fiy;
    S.RF[2][slot] += fiz;
  }
  __syncwarp();
  if (im2 != 0xFF) {
    const int slot = S.sbase[h][0] + im2;
    S.RF[0][slot] += fbx;
    S.RF[1][slot] += fby;
    S.RF[2][slot] += fbz;
  }
  __syncwarp();
}

// footprint cell of stencil entry e of home h (block-local coordinates, the
// merge table's numbering)
__device__ __forceinline__ int foot_of(const Box &b, int h, int e) {
  const int B0 = b.blk[0], B1 = b.blk[1], FX = B0 + 1, FY = B1 + 2;
  return (h % B0 + c_stencil3.o[e][0]) + FX * (((h / B0) % B1 + c_stencil3.o[e][1] + 1) +
                                               FY * (h / (B0 * B1) + c_stencil3.o[e][2] + 1));
}

// one home cell per warp (blocks have at most SH_NW = 8 cells)
template <bool ENERGY, class SM>
__device__ __forceinline__ void verlet_rounds(SM &S, const ForceArgs &A, int lane, int wid,
                                              const VPre &v) {
  {
    const int h = wid, cell = v.cell;
    if (cell < 0 || v.nr == 0) return;  // (not a contributor of any footprint cell)
    const int pA = v.pA, pB = v.pB;
    double pe = 0;
    unsigned hits = 0;
    double fa[3] = {0, 0, 0}, fb[3] = {0, 0, 0};
    const uint16_t *dp = A.vl_desc + (int64_t)cell * (VL_RMAX * 32) + lane;
    const bool shift = __any_sync(CS_FULL, lane < 14 && (S.sh[h][lane < 14 ? lane : 0][0] != 0.0 ||
                                                         S.sh[h][lane < 14 ? lane : 0][1] != 0.0 ||
                                                         S.sh[h][lane < 14 ? lane : 0][2] != 0.0));
    if (shift)
      verlet_table<ENERGY, true>(S, A, h, v, dp, fa, fb, pe, hits);
    else
      verlet_table<ENERGY, false>(S, A, h, v, dp, fa, fb, pe, hits);
    verlet_fi(S, h, lane, pA, fa[0], fa[1], fa[2], pB, fb[0], fb[1], fb[2]);
    // this home's slots are final: count it off its 14 footprint cells; the
    // last contributor of a cell queues it for merging
    asm volatile("fence.acq_rel.cta;" ::: "memory");
    if (lane < 14) {
      const int lc = foot_of(A.b, h, lane);
      if (atomicSub(&S.pend[lc], 1) == 1) {
        const int q = atomicAdd(&S.qtail, 1);
        atomicExch(&S.queue[q], lc);
      }
    }
    hits = warp_sum(hits);
    if (ENERGY) pe = warp_sum(pe);
    if (lane == 0) {
      if (A.npairs_direct) atomicAdd(A.npairs_direct, (unsigned long long)hits);
      else A.hits_cell[cell] += hits;
      if (ENERGY) A.pe_cell[cell] += pe;
    }
    __syncwarp();
  }
}

struct ShellArgs {
  ForceArgs A;
  MergeTable mt;
  double *buf;            // buffered mode: footprint buffers, 3 components x bufstride
  const int *boff;        // buffered mode: per-block offset into buf
  int *bindex;            // buffered mode: per block fstart[0..SH_MAXF]
  int64_t bufstride;
  unsigned *err;          // capacity overflow flag (buffered mode)
  int overwrite;          // buffered gather stores instead of adding (Verlet mode)
  int *flags;             // dataflow mode: per block "published" flag
  int *ticket;            // dataflow mode: next (colour, block) ticket
  int coff[9];            // dataflow mode: first ticket of each colour
  const unsigned char *vtab;  // Verlet mode: per-block tables cached at the list build
};

template <int MODE>
__device__ __forceinline__ void merge_store(const ShellArgs &SA, int64_t o, int g, double sx,
                                            double sy, double sz) {
  const ForceArgs &A = SA.A;
  if (MODE == SH_BUFFERED) {
    SA.buf[o] = sx;
    SA.buf[SA.bufstride + o] = sy;
    SA.buf[2 * SA.bufstride + o] = sz;
  } else if (MODE == SH_DATAFLOW) {  // other SMs wrote f: read through L2
    A.fx[g] = __ldcg(A.fx + g) + sx;
    A.fy[g] = __ldcg(A.fy + g) + sy;
    A.fz[g] = __ldcg(A.fz + g) + sz;
  } else {
    A.fx[g] += sx;
    A.fy[g] += sy;
    A.fz[g] += sz;
  }
}

// merge of footprint cell lc by one warp: home rows + reaction slots in the
// fixed merge-table order, into the block buffer or f
template <int MODE, class SM>
__device__ __forceinline__ void merge_cell(const ShellArgs &SA, SM &S, int lc, int lane,
                                           int64_t boff) {
  const int g0 = S.fgstart[lc];
  if (g0 < 0) return;
  const int f0 = S.fstart[lc], n = S.fstart[lc + 1] - f0;
  const int nc = S.mt_n[lc];
  if constexpr (MODE == SH_DATAFLOW) {
    // f of this cell is final for every lower colour (the block waited for
    // them) and nobody else writes it before this block publishes: its L2
    // reads go first (two particles per lane), so their latency overlaps
    // the slot sums instead of following them
    const ForceArgs &A = SA.A;
    for (int i0 = 0; i0 < n; i0 += 64) {
      const int ia = i0 + lane, ib = i0 + 32 + lane;
      const bool va = ia < n, vb = ib < n;
      const double ax = va ? __ldcg(A.fx + g0 + ia) : 0.0, ay = va ? __ldcg(A.fy + g0 + ia) : 0.0,
                   az = va ? __ldcg(A.fz + g0 + ia) : 0.0;
      const double bx = vb ? __ldcg(A.fx + g0 + ib) : 0.0, by = vb ? __ldcg(A.fy + g0 + ib) : 0.0,
                   bz = vb ? __ldcg(A.fz + g0 + ib) : 0.0;
      double sx = 0, sy = 0, sz = 0, tx = 0, ty = 0, tz = 0;
      for (int k = 0; k < nc; ++k) {
        const int base = S.mt_base[lc][k];
        if (base < 0) continue;
        if (va) {
          sx += S.RF[0][base + ia];
          sy += S.RF[1][base + ia];
          sz += S.RF[2][base + ia];
        }
        if (vb) {
          tx += S.RF[0][base + ib];
          ty += S.RF[1][base + ib];
          tz += S.RF[2][base + ib];
        }
      }
      if (va) {
        A.fx[g0 + ia] = ax + sx;
        A.fy[g0 + ia] = ay + sy;
        A.fz[g0 + ia] = az + sz;
      }
      if (vb) {
        A.fx[g0 + ib] = bx + tx;
        A.fy[g0 + ib] = by + ty;
        A.fz[g0 + ib] = bz + tz;
      }
    }
  } else {
    for (int i = lane; i < n; i += 32) {
      double sx = 0, sy = 0, sz = 0;
      for (int k = 0; k < nc; ++k) {
        const int base = S.mt_base[lc][k];
        if (base < 0) continue;
        const int s = base + i;
        sx += S.RF[0][s];
        sy += S.RF[1][s];
        sz += S.RF[2][s];
      }
      merge_store<MODE>(SA, boff + f0 + i, g0 + i, sx, sy, sz);
    }
  }
}

// Verlet mode, step 5 without a block barrier: warps that are done take
// footprint cells from the ready queue in order and merge them while the
// other homes are still running
template <int MODE, class SM>
__device__ __forceinline__ void verlet_merge_queue(const ShellArgs &SA, SM &S, int lane, int nfc,
                                                   int64_t boff) {
  while (true) {
    int t = 0;
    if (lane == 0) t = atomicAdd(&S.qhead, 1);
    t = __shfl_sync(CS_FULL, t, 0);
    if (t >= nfc) break;
    if constexpr (MODE == SH_DATAFLOW) {
      // the colour order binds only the updates of f: the block computed its
      // rounds without waiting, and merges after its lower-colour neighbour
      // blocks have published theirs
      if (!*(volatile int *)&S.depok) {
        if (lane < 27 && S.dep[lane] >= 0) {
          const volatile int *f = SA.flags + S.dep[lane];
          while (*f == 0) __nanosleep(64);
        }
        __syncwarp();
        __threadfence();
        if (lane == 0) *(volatile int *)&S.depok = 1;
      }
    }
    int lc = -1;
    if (lane == 0) {
      volatile int *qv = S.queue;
      while ((lc = qv[t]) < 0) __nanosleep(32);
    }
    lc = __shfl_sync(CS_FULL, lc, 0);
    asm volatile("fence.acq_rel.cta;" ::: "memory");
    merge_cell<MODE>(SA, S, lc, lane, boff);
  }
}

// block coordinates -> global cell of a footprint cell (or -1)
__device__ __forceinline__ int64_t foot_cell(const Box &b, const int *o0, int lc, int FX, int FY) {
  int v0 = o0[0] + lc % FX, v1 = o0[1] + (lc / FX) % FY - 1, v2 = o0[2] + lc / (FX * FY) - 1;
  if (b.per[0]) v0 = wrap1i(v0, b.nc[0]); else if (v0 < 0 || v0 >= b.nc[0]) return -1;
  if (b.per[1]) v1 = wrap1i(v1, b.nc[1]); else if (v1 < 0 || v1 >= b.nc[1]) return -1;
  if (b.per[2]) v2 = wrap1i(v2, b.nc[2]); else if (v2 < 0 || v2 >= b.nc[2]) return -1;
  return box_cell(b, v0, v1, v2);
}


// Phase 0 of a block: source tables per (home h, entry e), slot bases,
// footprint offsets and the capacity flag, in shared memory.  Depends only on
// the cell list (cached per block at a Verlet list build).
template <bool VERLET, class SM>
__device__ __forceinline__ void shell_tables(const ShellArgs &SA, SM &S, const int *o0) {
  constexpr int RCAP = SM::RCAP, HCAP = SM::HCAP;
  const ForceArgs &A = SA.A;
  const Box &b = A.b;
  const int B0 = b.blk[0], B1 = b.blk[1], B2 = b.blk[2];
  const int nhome = B0 * B1 * B2;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int FX = B0 + 1, FY = B1 + 2;
  const int nfc = SA.mt.nfc;
  // source tables, one thread per (h, e); footprint cells
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
    if (e == 0) {  // Verlet idle slots: entry 15 reads a real particle at 1e150 away
      S.sstart[h][15] = st;
      S.sbase[h][15] = 0;
      S.sh[h][15][0] = S.sh[h][15][1] = S.sh[h][15][2] = 1e150;
    }
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
      if (t < nhome * 14) S.sbase[h][e] = e == 0 ? RCAP + fb + ih - ch : rb + ir - cr;
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
      S.rtot = min(rb, RCAP);
      S.htot = min(fb, HCAP);
      S.overflow = (fb > HCAP || rb > RCAP || (!VERLET && src_max > SH_JCAP)) ? 1 : 0;
    }
  }
  __syncthreads();
  for (int lc = threadIdx.x; lc < SH_MAXF; lc += blockDim.x) {
    int live = 0;
#pragma unroll
    for (int k = 0; k < SH_MAXC; ++k) {
      int base = -1;
      if (lc < nfc && k < SA.mt.n[lc]) {
        const int he = SA.mt.he[lc][k];
        const int hh = he >> 4, e = he & 15;
        // (Verlet: a home without listed pairs adds nothing, so it is not a
        // contributor -- its warp skips the pend countdown, see verlet_rounds)
        if (S.hcell[hh] >= 0 && (!VERLET || A.vl_nround[S.hcell[hh]] > 0)) base = S.sbase[hh][e];
      }
      if (lc < nfc) S.mt_base[lc][k] = (int16_t)base;
      live += base >= 0;
    }
    if (VERLET) {  // empty footprint cells have nothing to merge: never queued
      const bool empty = lc < nfc && (S.fgstart[lc] < 0 || S.fstart[lc + 1] == S.fstart[lc]);
      S.pend[lc] = empty ? (1 << 20) : live;
      S.queue[lc] = -1;
    }
  }
  __syncthreads();
  if (VERLET && threadIdx.x == 0) {  // cells nobody writes are ready from the start
    int n0 = 0, nq = 0;
    for (int lc = 0; lc < nfc; ++lc) {
      if (S.pend[lc] == 0) S.queue[n0++] = lc;
      nq += S.pend[lc] < (1 << 20);
    }
    S.qtail = n0;
    S.qhead = 0;
    S.nq = nq;
  }
  __syncthreads();
}

// bytes of the cached per-block tables: ShellBase from `sh` through `overflow`
__host__ __device__ constexpr size_t vl_table_bytes() {
  return (offsetof(ShellSmemVL, overflow) + sizeof(int) - offsetof(ShellSmemVL, sh) + 15) & ~(size_t)15;
}

template <bool ENERGY, int MODE, bool VERLET>
__device__ __forceinline__ void shell_block(const ShellArgs &SA, unsigned char *sh_raw, int colour,
                                            int bid) {
  constexpr bool BUFFERED = MODE == SH_BUFFERED;
  using SM = typename std::conditional<VERLET, ShellSmemVL, ShellSmem>::type;
  constexpr int RCAP = SM::RCAP, HCAP = SM::HCAP;
  SM &S = *reinterpret_cast<SM *>(sh_raw);
  const ForceArgs &A = SA.A;
  const Box &b = A.b;
  const int B0 = b.blk[0], B1 = b.blk[1], B2 = b.blk[2];
  const int nhome = B0 * B1 * B2;
  int o0[3];
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
  const int nfc = SA.mt.nfc;

  bool cached = false;
  VPre pre;
  if constexpr (VERLET) {
    vl_pre_issue(A, o0, wid, lane, pre);
    if (SA.vtab) {  // tables cached at the list build: asynchronous 16-byte copies into
                    // shared memory while the reaction slots are zeroed
      const int blin = o0[0] / B0 + A.nbk[0] * (o0[1] / B1 + A.nbk[1] * (o0[2] / B2));
      const unsigned char *src = SA.vtab + (size_t)blin * vl_table_bytes();
      const unsigned dst = (unsigned)__cvta_generic_to_shared(reinterpret_cast<unsigned char *>(&S) +
                                                              offsetof(SM, sh));
      for (int k = threadIdx.x; k < (int)(vl_table_bytes() / 16); k += blockDim.x)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * k), "l"(src + 16 * k)
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      // zero the slots in use (counts read from the global copy of the tables)
      const ShellSmemVL &G = *reinterpret_cast<const ShellSmemVL *>(src - offsetof(ShellSmemVL, sh));
      const int rt = __ldg(&G.rtot), ht = __ldg(&G.htot);
      for (int i = threadIdx.x; i < rt + ht; i += blockDim.x) {
        const int k = i < rt ? i : RCAP + i - rt;
        S.RF[0][k] = S.RF[1][k] = S.RF[2][k] = 0.0;
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
      cached = true;
    }
  }
  if (!cached) shell_tables<VERLET>(SA, S, o0);
  // merge table into shared memory (after the table copy, which may write
  // up to 15 padding bytes past `overflow`); read after later barriers
  for (int k = threadIdx.x; k < SH_MAXF; k += blockDim.x) S.mt_n[k] = SA.mt.n[k];
  if (S.overflow) {
    if constexpr (MODE != SH_COLOUR) {  // no in-place fallback: report to the host
      if (threadIdx.x == 0) atomicExch(SA.err, 1u);
      if (BUFFERED)  // the gather still reads this block's (unwritten) buffer in bounds
        for (int lc = threadIdx.x; lc <= nfc; lc += blockDim.x)
          SA.bindex[(int64_t)bid * (SH_MAXF + 1) + lc] = S.fstart[lc];
      return;
    } else {
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
        task_stats<ENERGY>(pe, hits, S.hcell[h], A.pe_cell, A.hits_cell, A.npairs_direct);
      }
      __syncthreads();
    }
    return;
    }
  }
  if (VERLET) vl_pre_positions(A, pre);
  if (!cached)
    for (int i = threadIdx.x; i < S.rtot + S.htot; i += blockDim.x) {
      const int k = i < S.rtot ? i : RCAP + i - S.rtot;
      S.RF[0][k] = S.RF[1][k] = S.RF[2][k] = 0.0;
    }
  __syncthreads();

  const double rc2 = A.p.rc2, sig2 = A.p.sig2, eps48 = A.p.eps48, eps4 = A.p.eps4;
  // ---- 1-4. one warp per home cell
  if constexpr (VERLET) {
    verlet_rounds<ENERGY>(S, A, lane, wid, pre);
  } else {
  for (int h = wid; h < nhome; h += SH_NW) {
    if (S.hcell[h] < 0) continue;
    const int a0 = S.sstart[h][0], na = S.scount[h][0];
    // 1. j list = the 14 source cells concatenated (home first).  Lanes walk
    //    the concatenation directly (no per-cell partial warps); a box-distance
    //    cull was measured to cost more than the candidates it removes.
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
        S.hx[wid][lane][0] = __ldg(A.x + ii);
        S.hx[wid][lane][1] = __ldg(A.y + ii);
        S.hx[wid][lane][2] = __ldg(A.z + ii);
      }
#pragma unroll
      for (int q = 0; q < SH_IB; ++q)
        S.rows[wid][q][0][lane] = S.rows[wid][q][1][lane] = S.rows[wid][q][2][lane] = 0.0;
      __syncwarp();
      const unsigned qmask = (1u << nib) - 1;
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
        // intra (e == 0): only pairs i < j, i.e. rows qq < q - ib
        const int jr = (vj && e == 0) ? q - ib : SH_IB + 1;
        unsigned mask = 0;
#pragma unroll
        for (int qq = 0; qq < SH_IB; ++qq) {
          const double dx = S.hx[wid][qq][0] - xj, dy = S.hx[wid][qq][1] - yj,
                       dz = S.hx[wid][qq][2] - zj;
          const double r2 = __fma_rn(dz, dz, __fma_rn(dy, dy, dx * dx));
          mask |= (unsigned)(r2 < rc2 && qq < jr) << qq;
        }
        mask &= qmask;
        double gx = 0, gy = 0, gz = 0;
        // two hits per lane per step: independent dependency chains (ILP);
        // both write different rows of this lane's private partials
        while (__any_sync(CS_FULL, mask)) {
          const bool h1 = mask != 0;
          const int q1 = h1 ? __ffs(mask) - 1 : 0;
          mask &= mask - 1;
          const bool h2 = mask != 0;
          const int q2 = h2 ? __ffs(mask) - 1 : 0;
          mask &= mask - 1;
          if (h1) {
            const double dx1 = S.hx[wid][q1][0] - xj, dy1 = S.hx[wid][q1][1] - yj,
                         dz1 = S.hx[wid][q1][2] - zj;
            const double dx2 = S.hx[wid][q2][0] - xj, dy2 = S.hx[wid][q2][1] - yj,
                         dz2 = S.hx[wid][q2][2] - zj;
            const double r21 = __fma_rn(dz1, dz1, __fma_rn(dy1, dy1, dx1 * dx1));
            const double r22 = h2 ? __fma_rn(dz2, dz2, __fma_rn(dy2, dy2, dx2 * dx2)) : 1.0;
            const double ri1 = fast_rcp(r21), ri2 = fast_rcp(r22);
            const double s21 = sig2 * ri1, s22 = sig2 * ri2;
            const double s61 = s21 * s21 * s21, s62 = s22 * s22 * s22;
            const double ff1 = eps48 * s61 * (s61 - 0.5) * ri1;
            const double ff2 = h2 ? eps48 * s62 * (s62 - 0.5) * ri2 : 0.0;
            const double fx1 = ff1 * dx1, fy1 = ff1 * dy1, fz1 = ff1 * dz1;
            const double fx2 = ff2 * dx2, fy2 = ff2 * dy2, fz2 = ff2 * dz2;
            gx -= fx1;
            gy -= fy1;
            gz -= fz1;
            S.rows[wid][q1][0][lane] += fx1;
            S.rows[wid][q1][1][lane] += fy1;
            S.rows[wid][q1][2][lane] += fz1;
            if (ENERGY) pe += eps4 * s61 * (s61 - 1.0);
            ++hits;
            if (h2) {
              gx -= fx2;
              gy -= fy2;
              gz -= fz2;
              S.rows[wid][q2][0][lane] += fx2;
              S.rows[wid][q2][1][lane] += fy2;
              S.rows[wid][q2][2][lane] += fz2;
              if (ENERGY) pe += eps4 * s62 * (s62 - 1.0);
              ++hits;
            }
          }
        }
        if (vj) {  // unique writer of slot (h, e, q)
          double *dst = &S.RF[0][S.sbase[h][e] + q];
          constexpr int stride = RCAP + HCAP;
          dst[0] += gx;
          dst[stride] += gy;
          dst[2 * stride] += gz;
        }
      }
      __syncwarp();
      if (lane < 3 * SH_IB) {  // lane (q, c) reduces row q component c
        const int q = lane / 3, c = lane - 3 * (lane / 3);
        if (q < nib) {
          double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
          for (int l = 0; l < 32; l += 4) {
            s0 += S.rows[wid][q][c][l];
            s1 += S.rows[wid][q][c][l + 1];
            s2 += S.rows[wid][q][c][l + 2];
            s3 += S.rows[wid][q][c][l + 3];
          }
          S.RF[c][fh0 + ib + q] += (s0 + s1) + (s2 + s3);
        }
      }
      __syncwarp();
    }
    hits = warp_sum(hits);
    if (ENERGY) pe = warp_sum(pe);
    if (lane == 0) {
      if (A.npairs_direct) atomicAdd(A.npairs_direct, (unsigned long long)hits);
      else A.hits_cell[S.hcell[h]] += hits;
      if (ENERGY) A.pe_cell[S.hcell[h]] += pe;
    }
  }
  }  // link-cell super-tasks
  if constexpr (VERLET) {
    verlet_merge_queue<MODE>(SA, S, lane, S.nq, BUFFERED ? SA.boff[bid] : 0);
    if (BUFFERED)
      for (int lc = threadIdx.x; lc <= nfc; lc += blockDim.x)
        SA.bindex[(int64_t)bid * (SH_MAXF + 1) + lc] = S.fstart[lc];
    return;
  }
  __syncthreads();
  // ---- 5. merge, one thread per footprint particle: home rows + reaction
  //         slots in the fixed merge-table order
  const int64_t boff = BUFFERED ? SA.boff[bid] : 0;
  const int nfoot = S.fstart[nfc];
  for (int t0 = wid * 32; t0 < nfoot; t0 += blockDim.x) {
    int lc = 0;  // footprint cell of t0 (lane 0), then step forward per lane
    if (lane == 0) {
#pragma unroll
      for (int k = 32; k >= 1; k >>= 1)
        if (lc + k < nfc && S.fstart[lc + k] <= t0) lc += k;
    }
    lc = __shfl_sync(CS_FULL, lc, 0);
    const int t = t0 + lane;
    if (t >= nfoot) continue;
    while (lc + 1 < nfc && S.fstart[lc + 1] <= t) ++lc;
    const int g0 = S.fgstart[lc];
    if (g0 < 0) continue;
    const int i = t - S.fstart[lc];
    const int nc = S.mt_n[lc];
    double sx = 0, sy = 0, sz = 0;
    for (int k = 0; k < nc; ++k) {
      const int base = S.mt_base[lc][k];
      if (base < 0) continue;  // (slab ranks: homes past the owned planes)
      const int s = base + i;
      sx += S.RF[0][s];
      sy += S.RF[1][s];
      sz += S.RF[2][s];
    }
    if (BUFFERED) {
      const int64_t o = boff + t;
      SA.buf[o] = sx;
      SA.buf[SA.bufstride + o] = sy;
      SA.buf[2 * SA.bufstride + o] = sz;
    } else if (MODE == SH_DATAFLOW) {  // other SMs wrote f: read through L2
      A.fx[g0 + i] = __ldcg(A.fx + g0 + i) + sx;
      A.fy[g0 + i] = __ldcg(A.fy + g0 + i) + sy;
      A.fz[g0 + i] = __ldcg(A.fz + g0 + i) + sz;
    } else {
      A.fx[g0 + i] += sx;
      A.fy[g0 + i] += sy;
      A.fz[g0 + i] += sz;
    }
  }
  if (BUFFERED)
    for (int lc = threadIdx.x; lc <= nfc; lc += blockDim.x)
      SA.bindex[(int64_t)bid * (SH_MAXF + 1) + lc] = S.fstart[lc];
}

template <bool ENERGY, int MODE, bool VERLET>
__global__ void __launch_bounds__(SH_NW * 32, VERLET ? 2 : 3) k_force_shell(ShellArgs SA, int colour) {
  extern __shared__ __align__(16) unsigned char sh_raw[];
  if constexpr (MODE != SH_DATAFLOW) {
    shell_block<ENERGY, MODE, VERLET>(SA, sh_raw, colour, blockIdx.x);
  } else {
    // Dataflow execution of the colour order: blocks are taken in (colour,
    // block) order from a ticket; a block starts as soon as its (up to 26)
    // neighbour blocks of lower colour -- the only ones whose footprints
    // overlap -- have published, instead of after a global barrier per
    // colour.  Per particle the contributions still arrive in colour order.
    __shared__ int s_t;
    const ForceArgs &A = SA.A;
    while (true) {
      if (threadIdx.x == 0) s_t = atomicAdd(SA.ticket, 1);
      __syncthreads();
      const int t = s_t;
      __syncthreads();
      if (t >= SA.coff[8]) break;
      int c = 0;
      while (c < 7 && SA.coff[c + 1] <= t) ++c;
      const int idx = t - SA.coff[c];
      const int kc[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
      const int cnt0 = (A.nbk[0] - kc[0] + 1) >> 1, cnt1 = (A.nbk[1] - kc[1] + 1) >> 1;
      const int kb[3] = {2 * (idx % cnt0) + kc[0], 2 * ((idx / cnt0) % cnt1) + kc[1],
                         2 * (idx / (cnt0 * cnt1)) + kc[2]};
      if (VERLET) {
        // record the lower-colour neighbours; the wait happens before the
        // block's first footprint merge (verlet_merge_queue), not here
        ShellSmemVL &S = *reinterpret_cast<ShellSmemVL *>(sh_raw);
        if (threadIdx.x < 27) {
          int dep = -1;
          if (threadIdx.x != 13) {
            const int d[3] = {(int)threadIdx.x % 3 - 1, ((int)threadIdx.x / 3) % 3 - 1,
                              (int)threadIdx.x / 9 - 1};
            int nbc[3];
            bool ok = true;
            for (int k = 0; k < 3; ++k) {
              nbc[k] = kb[k] + d[k];
              if (nbc[k] < 0 || nbc[k] >= A.nbk[k]) {
                if (A.b.per[k]) nbc[k] = wrap1i(nbc[k], A.nbk[k]);
                else ok = false;
              }
            }
            const int ncol = (nbc[0] & 1) | ((nbc[1] & 1) << 1) | ((nbc[2] & 1) << 2);
            if (ok && ncol < c) dep = nbc[0] + A.nbk[0] * (nbc[1] + A.nbk[1] * nbc[2]);
          }
          S.dep[threadIdx.x] = dep;
        }
        if (threadIdx.x == 0) S.depok = 0;
      } else if (threadIdx.x < 27 && threadIdx.x != 13) {
        const int d[3] = {(int)threadIdx.x % 3 - 1, ((int)threadIdx.x / 3) % 3 - 1, (int)threadIdx.x / 9 - 1};
        int nbc[3];
        bool ok = true;
        for (int k = 0; k < 3; ++k) {
          nbc[k] = kb[k] + d[k];
          if (nbc[k] < 0 || nbc[k] >= A.nbk[k]) {
            if (A.b.per[k]) nbc[k] = wrap1i(nbc[k], A.nbk[k]);
            else ok = false;
          }
        }
        if (ok) {
          const int ncol = (nbc[0] & 1) | ((nbc[1] & 1) << 1) | ((nbc[2] & 1) << 2);
          if (ncol < c) {
            const volatile int *f = SA.flags + nbc[0] + A.nbk[0] * (nbc[1] + A.nbk[1] * nbc[2]);
            while (*f == 0) __nanosleep(64);
          }
        }
        __threadfence();
      }
      __syncthreads();
      shell_block<ENERGY, MODE, VERLET>(SA, sh_raw, c, idx);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0)
        atomicExch(SA.flags + kb[0] + A.nbk[0] * (kb[1] + A.nbk[1] * kb[2]), 1);
    }
  }
}

// Verlet list build: the per-block tables of every block (buffered block
// order), cached for the force evaluations until the next build.  Shared
// memory holds only the table part of ShellSmemVL.
__global__ void __launch_bounds__(SH_NW * 32) k_vl_tables(ShellArgs SA, unsigned char *out) {
  extern __shared__ __align__(16) unsigned char sh_raw[];
  ShellSmemVL &S = *reinterpret_cast<ShellSmemVL *>(sh_raw - offsetof(ShellSmemVL, sh));
  const ForceArgs &A = SA.A;
  const int bid = blockIdx.x;
  const int o0[3] = {(bid % A.nbk[0]) * A.b.blk[0], ((bid / A.nbk[0]) % A.nbk[1]) * A.b.blk[1],
                     (bid / (A.nbk[0] * A.nbk[1])) * A.b.blk[2]};
  shell_tables<true>(SA, S, o0);
  const int4 *src = reinterpret_cast<const int4 *>(sh_raw);
  int4 *dst = reinterpret_cast<int4 *>(out + (size_t)bid * vl_table_bytes());
  for (int k = threadIdx.x; k < (int)(vl_table_bytes() / 16); k += blockDim.x) dst[k] = src[k];
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
// One warp per GB_CELLS consecutive cells: lane (c, k) resolves candidate
// block k of cell c once, then the warp's lanes walk the cells' particles
// together (small cells -- a cfg5 vapour cell holds ~0.5 particles -- do not
// idle a warp each).
#define GB_CELLS 4
static_assert(GB_CELLS == 4, "the cell selects below are written out for 4 cells");
__global__ void k_gather_blocks(ShellArgs SA) {
  const ForceArgs &A = SA.A;
  const Box &b = A.b;
  const int B0 = b.blk[0], B1 = b.blk[1], B2 = b.blk[2];
  const int FX = B0 + 1, FY = B1 + 2, FZ = B2 + 2;
  const int nc0 = b.nc[0], nc1 = b.nc[1];
  const int64_t ncell = (int64_t)nc0 * nc1 * b.nc[2];
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t cfirst = warp * GB_CELLS;
  if (cfirst >= ncell) return;
  const int cs = lane >> 3, kk = lane & 7;  // (cell of the group, candidate block)
  const int64_t cl = cfirst + cs;
  int src = -1, g0 = 0, n = 0;
  if (cl < ncell) {
    const int c0 = (int)(cl % nc0), c1 = (int)((cl / nc0) % nc1), c2 = (int)(cl / ((int64_t)nc0 * nc1));
    const int64_t gc = box_cell(b, c0, c1, c2);
    g0 = A.start[gc];
    n = A.start[gc + 1] - g0;
    // per axis: the block containing c and, at a block edge, the neighbour
    // block whose footprint reaches c (x: footprint reaches +1; y, z: -1, +B)
    const int u = kk & 1, v = (kk >> 1) & 1, w = kk >> 2;
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
  // particle ranges of the group's cells (lane 8c holds cell c's)
  int pre[GB_CELLS + 1], gs[GB_CELLS];
  pre[0] = 0;
#pragma unroll
  for (int c = 0; c < GB_CELLS; ++c) {
    pre[c + 1] = pre[c] + __shfl_sync(CS_FULL, n, 8 * c);
    gs[c] = __shfl_sync(CS_FULL, g0, 8 * c);
  }
  const int ptot = pre[GB_CELLS];
  for (int t0 = 0; t0 < ptot; t0 += 32) {
    const int t = t0 + lane;
    int c = 0;
#pragma unroll
    for (int q = 1; q < GB_CELLS; ++q) c += t >= pre[q];
    const int i = t - (c == 0 ? pre[0] : (c == 1 ? pre[1] : (c == 2 ? pre[2] : pre[3])));
    const int gi = (c == 0 ? gs[0] : (c == 1 ? gs[1] : (c == 2 ? gs[2] : gs[3]))) + i;
    // the <= 8 source offsets of this particle's cell, then all loads issued
    // before the fixed-order sums
    double vx[8], vy[8], vz[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int so = __shfl_sync(CS_FULL, src, 8 * c + k);
      const bool ok = so >= 0 && t < ptot;
      const int64_t o = ok ? (int64_t)so + i : 0;
      vx[k] = ok ? __ldcs(SA.buf + o) : 0.0;
      vy[k] = ok ? __ldcs(SA.buf + SA.bufstride + o) : 0.0;
      vz[k] = ok ? __ldcs(SA.buf + 2 * SA.bufstride + o) : 0.0;
    }
    double sx = 0, sy = 0, sz = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // fixed order: candidate blocks ascending
      sx += vx[k];
      sy += vy[k];
      sz += vz[k];
    }
    if (t < ptot) {
      if (SA.overwrite) {
        A.fx[gi] = sx;
        A.fy[gi] = sy;
        A.fz[gi] = sz;
      } else {
        A.fx[gi] += sx;
        A.fy[gi] += sy;
        A.fz[gi] += sz;
      }
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

typedef void (*ShellKernel)(ShellArgs, int);
static ShellKernel shell_kernel(bool energy, int mode, bool verlet) {
  static const ShellKernel k[12] = {
      k_force_shell<false, 0, false>, k_force_shell<true, 0, false>,
      k_force_shell<false, 1, false>, k_force_shell<true, 1, false>,
      k_force_shell<false, 2, false>, k_force_shell<true, 2, false>,
      k_force_shell<false, 0, true>,  k_force_shell<true, 0, true>,
      k_force_shell<false, 1, true>,  k_force_shell<true, 1, true>,
      k_force_shell<false, 2, true>,  k_force_shell<true, 2, true>};
  return k[(verlet ? 6 : 0) + 2 * mode + (energy ? 1 : 0)];
}

static int launch_shell_passes(const ForceArgs &A, bool energy, int mode, bool verlet,
                               cs_ws *w, int64_t n, unsigned *status, cudaStream_t st) {
  const bool buffered = mode == SH_BUFFERED;
  const int B[3] = {A.b.blk[0], A.b.blk[1], A.b.blk[2]};
  CS_REQUIRE(B[0] * B[1] * B[2] <= SH_MAXB, "shell schedule: block has more than %d cells", SH_MAXB);
  ShellArgs SA;
  memset(&SA, 0, sizeof(SA));
  SA.A = A;
  SA.overwrite = verlet ? 1 : 0;
  SA.vtab = A.vl_tab;
  CS_TRY(build_merge_table(B, &SA.mt));
  const size_t smem = verlet ? sizeof(ShellSmemVL) : sizeof(ShellSmem);
  static bool attr[CS_MAX_DEVICES];
  const int devi = cs_device_index();
  if (!attr[devi]) {
    for (int v = 0; v < 12; ++v) {
      const bool vl = v >= 6;
      const size_t sm = vl ? sizeof(ShellSmemVL) : sizeof(ShellSmem);
      CS_CUDA(cudaFuncSetAttribute(shell_kernel(v & 1, (v % 6) / 2, vl),
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    }
    attr[devi] = true;
  }
  const ShellKernel kern = shell_kernel(energy, mode, verlet);
  if (mode == SH_DATAFLOW) {
    const int64_t nblocks = (int64_t)A.nbk[0] * A.nbk[1] * A.nbk[2];
    CS_WS_TAKE(*w, int, flags, nblocks + 1);
    CS_WS_TAKE(*w, unsigned, err, 16);
    SA.flags = flags;
    SA.ticket = flags + nblocks;
    SA.err = status ? status : err;
    SA.coff[0] = 0;
    for (int c = 0; c < 8; ++c) {
      int cnt = 1;
      for (int k = 0; k < 3; ++k) cnt *= (A.nbk[k] - ((c >> k) & 1) + 1) >> 1;
      SA.coff[c + 1] = SA.coff[c] + cnt;
    }
    static int grid_cap[CS_MAX_DEVICES][2];
    if (!grid_cap[devi][verlet]) {
      int per_sm = 0, dev = 0, nsm = 0;
      CS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SH_NW * 32, smem));
      CS_CUDA(cudaGetDevice(&dev));
      CS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      grid_cap[devi][verlet] = max(1, per_sm) * nsm;
    }
    CS_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * (nblocks + 1), st));
    const unsigned grid = (unsigned)(nblocks < grid_cap[devi][verlet] ? nblocks : grid_cap[devi][verlet]);
    kern<<<grid, SH_NW * 32, smem, st>>>(SA, -1);
    return cs_check_launch("force_dataflow");
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
    if (A.vl_boff) {  // Verlet mode: the layout was computed at the list build
      SA.boff = A.vl_boff;
    } else {
      k_block_sizes<<<grid_for(nblocks * 32, 256), 256, 0, st>>>(SA, sizes);
      CS_TRY(cs_exclusive_scan_i32(sizes, boff, nblocks, scratch, sb, st));
    }
    kern<<<(unsigned)nblocks, SH_NW * 32, smem, st>>>(SA, -1);
    const int64_t ncell = (int64_t)A.b.nc[0] * A.b.nc[1] * A.b.nc[2];
    const int64_t gwarps = (ncell + GB_CELLS - 1) / GB_CELLS;
    k_gather_blocks<<<(unsigned)((gwarps * 32 + 255) / 256), 256, 0, st>>>(SA);
    return cs_check_launch("force_buffered");
  }
  for (int colour = 0; colour < 8; ++colour) {
    const int kc[3] = {colour & 1, (colour >> 1) & 1, (colour >> 2) & 1};
    unsigned blocks = 1;
    for (int k = 0; k < 3; ++k) blocks *= (unsigned)((A.nbk[k] - kc[k] + 1) >> 1);
    if (!blocks) continue;
    kern<<<blocks, SH_NW * 32, smem, st>>>(SA, colour);
  }
  return cs_check_launch("force_shell");
}
