// cs_verlet.cuh -- Verlet neighbour lists for the K2 super-task kernel.
//
// Built from the cell list on cells of edge >= rc + skin, so every pair that
// can come within rc before the next rebuild (no particle moved more than
// skin/2) lies in the home cell's 14-entry half shell and is within rc + skin
// now.  The list of a home cell is stored as a ROUND TABLE instead of per-
// particle rows:
//
//   imap[cell][lane]          home particle served by this lane (lanes of one
//                             particle contiguous; 0xFF = idle lane)
//   desc[cell][round][lane]   partner j as (stencil entry << 8 | index in the
//                             source cell), VL_IDLE = no pair this round
//   nround[cell]
//
// with at most one pair per lane per round and no j twice in a round.  The
// force kernel (verlet_rounds in cs_force2.cuh) then keeps F_i in registers
// and writes the Newton-3 reaction on j without conflicts.  Lanes are shared
// out in proportion to the particles' list lengths; pairs are dealt round-
// robin to a particle's lanes, then placed first-fit into rounds by all lanes
// in lockstep (a (j, round) collision is won by the lowest lane, so the
// table -- and the force summation order -- is deterministic).
//
// Between rebuilds positions are not wrapped (the image shift of a stencil
// entry is fixed at build time); cs_vv_kick_drift_track raises a flag once
// any particle has moved more than skin/2 from its position at the build.
#pragma once
#include "cs_force2.cuh"

#define VB_NW 4      // warps per builder CTA
#define VB_JCAP 448  // candidate j per home cell (14 source cells)

struct VList {
  int32_t *nround;  // rounds R of the cell's table
  uint8_t *imap;    // [cell][96]: lane -> first particle, second particle, switch round
  uint16_t *desc;   // [cell][VL_RMAX][32]
  int32_t *bsizes;  // buffered block layout (fixed between rebuilds): footprint sizes,
  int32_t *boff;    //   their exclusive scan = block buffer offsets
  void *scan_ws;    //   scan scratch
  unsigned char *tab;  // per-block force-kernel tables (vl_table_bytes each)
  int32_t *crowd;      // builder: home cells above 32 particles (second pass)
  int32_t *ncrowd;     //   and their count
};

static int64_t vl_blocks(const Box &b) {
  const int B0 = b.blk[0] > 0 ? b.blk[0] : 1, B1 = b.blk[1] > 0 ? b.blk[1] : 1, B2 = b.blk[2] > 0 ? b.blk[2] : 1;
  return (int64_t)((b.owned_x + B0 - 1) / B0) * ((b.nc[1] + B1 - 1) / B1) * ((b.nc[2] + B2 - 1) / B2);
}

static size_t vl_bytes(const Box &b) {  // (blocks <= cells bounds the layout arrays)
  const int64_t ncell = b.ncells;
  return cs_ws_slice(sizeof(int32_t) * ncell) + cs_ws_slice(96 * (size_t)ncell) +
         cs_ws_slice(sizeof(uint16_t) * (size_t)VL_RMAX * 32 * ncell) +
         2 * cs_ws_slice(sizeof(int32_t) * (ncell + 2)) + cs_ws_slice(cs_scan_ws_bytes(ncell + 1)) +
         cs_ws_slice(vl_table_bytes() * (size_t)vl_blocks(b)) + cs_ws_slice(sizeof(int32_t) * ncell) +
         cs_ws_slice(64);
}

static VList vl_view(void *p, const Box &b) {
  const int64_t ncell = b.ncells;
  char *c = (char *)p;
  VList v;
  v.nround = (int32_t *)c;
  c += cs_ws_slice(sizeof(int32_t) * ncell);
  v.imap = (uint8_t *)c;
  c += cs_ws_slice(96 * (size_t)ncell);
  v.desc = (uint16_t *)c;
  c += cs_ws_slice(sizeof(uint16_t) * (size_t)VL_RMAX * 32 * ncell);
  v.bsizes = (int32_t *)c;
  c += cs_ws_slice(sizeof(int32_t) * (ncell + 2));
  v.boff = (int32_t *)c;
  c += cs_ws_slice(sizeof(int32_t) * (ncell + 2));
  v.scan_ws = c;
  c += cs_ws_slice(cs_scan_ws_bytes(ncell + 1));
  v.tab = (unsigned char *)c;
  c += cs_ws_slice(vl_table_bytes() * (size_t)vl_blocks(b));
  v.crowd = (int32_t *)c;
  c += cs_ws_slice(sizeof(int32_t) * ncell);
  v.ncrowd = (int32_t *)c;
  return v;
}

static void vl_attach(ForceArgs &A, const void *vlist) {
  VList v = vl_view(const_cast<void *>(vlist), A.b);
  A.vl_nround = v.nround;
  A.vl_imap = v.imap;
  A.vl_desc = v.desc;
  A.vl_boff = v.boff;
  A.vl_tab = v.tab;
}

extern "C" size_t cs_verlet_list_bytes(const cs_box *bx) {
  Box b;
  if (make_box(bx, &b) != CS_OK) return 0;
  return vl_bytes(b);
}

// source cell of stencil entry e for home cell (h0, h1, h2): start, count
// (0 if outside a non-periodic box) and the periodic image shift
__device__ __forceinline__ void vl_source(const Box &b, const int32_t *start, int h0, int h1,
                                          int h2, int e, int *st, int *cnt, double &s0,
                                          double &s1, double &s2) {
  int v0 = h0 + c_stencil3.o[e][0], v1 = h1 + c_stencil3.o[e][1], v2 = h2 + c_stencil3.o[e][2];
  s0 = s1 = s2 = 0.0;
  bool ok = true;
  if (b.per[0]) { s0 = v0 >= b.nc[0] ? b.L[0] : (v0 < 0 ? -b.L[0] : 0.0); v0 = wrap1i(v0, b.nc[0]); }
  else ok = ok && v0 >= 0 && v0 < b.nc[0];
  if (b.per[1]) { s1 = v1 >= b.nc[1] ? b.L[1] : (v1 < 0 ? -b.L[1] : 0.0); v1 = wrap1i(v1, b.nc[1]); }
  else ok = ok && v1 >= 0 && v1 < b.nc[1];
  if (b.per[2]) { s2 = v2 >= b.nc[2] ? b.L[2] : (v2 < 0 ? -b.L[2] : 0.0); v2 = wrap1i(v2, b.nc[2]); }
  else ok = ok && v2 >= 0 && v2 < b.nc[2];
  *st = 0;
  *cnt = 0;
  if (ok) {
    const int64_t gc = box_cell(b, v0, v1, v2);
    *st = start[gc];
    *cnt = start[gc + 1] - *st;
  }
}

#define VB_SEG 4                // table lanes a particle may span

// Shared memory of the builder: NW warps, up to MAXP particles per home cell,
// up to JCAP candidates (14 source cells).  The main pass takes cells of <= 32
// particles (one lane per particle) with 4 warps per CTA; cells above that go
// to a second pass with up to 64 (two particles per lane) and 896 candidates.
// The round table is placed directly in its global slot (no shared copy), so
// the main pass needs 28.5 KB of shared memory per CTA: at <= 70 registers 7
// CTAs (28 warps) fit an SM (measured: rebuild 865 -> 825 us on cfg2).
template <int NW, int MAXP, int JCAP>
struct VBuildSmemT {
  static constexpr int NCH = JCAP / 32;
  unsigned used[NW][2][JCAP];  // per candidate j: rounds taken (low, high 32)
  unsigned row[NW][MAXP][NCH];  // particle -> candidate bits per chunk
  uint16_t code[NW][JCAP];      // entry << 8 | index in the source cell
  double hx[NW][MAXP][3];       // home positions (broadcast reads)
  uint8_t lmap[NW][96];         // lane -> first / second particle, switch round
};
#define VB_MINB 7
using VBMain = VBuildSmemT<VB_NW, 32, VB_JCAP>;
using VBCrowd = VBuildSmemT<1, 64, 2 * VB_JCAP>;

// Lockstep first-fit: lane p places all pairs of particle p (row bits over the
// candidate chunks) into its own slots -- up to VB_SEG segments (table lane
// seg_l[k], free rounds fr[k]) -- taking the first segment with a free round
// that does not hold the same j yet, lowest round first.  Equal (j, round)
// proposals are won by the lowest lane; lanes start at different j so that
// such collisions are rare.  Returns false (warp-uniform) if a pair found no
// slot.  u0 / u1: rounds 0-31 / 32-63 taken per candidate j.
__device__ __forceinline__ int vl_ffs(unsigned v) { return __ffs(v); }
__device__ __forceinline__ int vl_ffs(unsigned long long v) { return __ffsll((long long)v); }

template <class M>  // round masks: 32 bits while R <= 32, else 64
__device__ __forceinline__ M vl_used(const unsigned *u0, const unsigned *u1, int j);
template <>
__device__ __forceinline__ unsigned vl_used<unsigned>(const unsigned *u0, const unsigned *u1, int j) {
  return u0[j];
}
template <>
__device__ __forceinline__ unsigned long long vl_used<unsigned long long>(const unsigned *u0,
                                                                          const unsigned *u1, int j) {
  return ((unsigned long long)u1[j] << 32) | u0[j];
}

// lowest free round of mask class `par` (0: any, 1: even, 2: odd) for a pair
// whose j has rounds `u` taken: (round, segment) or -1
template <class M>
__device__ __forceinline__ int vl_pick(const M *fr, M u, M par, int &k) {
  int r = -1;
#pragma unroll
  for (int kk = VB_SEG - 1; kk >= 0; --kk) {  // first segment with a free round wins
    const M m = fr[kk] & ~u & par;
    if (m) {
      r = vl_ffs(m) - 1;
      k = kk;
    }
  }
  return r;
}

// Lockstep first-fit with two proposals per lane and iteration: pair A goes to
// its lowest free round (either parity), pair B (another pending pair of the
// chunk) to its lowest free round of the OTHER parity.  Even and odd proposals
// never share a (j, round), so each parity resolves with its own match_any;
// the lowest lane wins.
template <class M>
__device__ __forceinline__ bool vl_place(const unsigned *row, int nch, M *fr, const int *seg_l,
                                         unsigned *u0, unsigned *u1, const uint16_t *code,
                                         uint16_t (*tab)[32], int lane) {
  const M EVEN = (M)0x5555555555555555ull, ODD = (M)0xAAAAAAAAAAAAAAAAull;
  bool ok = true;
  int cc = 0;
  unsigned cur = nch > 0 ? row[0] : 0u;
  const int rot = (lane * 7) & 31;
  while (true) {
    while (cur == 0 && cc + 1 < nch) cur = row[++cc];
    if (!__any_sync(CS_FULL, cur != 0)) break;
    int bA = -1, bB = -1, rA = -1, rB = -1, kA = 0, kB = 0;
    if (cur) {
      const unsigned hi = cur & (~0u << rot);
      bA = __ffs(hi ? hi : cur) - 1;
      const unsigned rest = cur & ~(1u << bA);
      if (rest) {
        const unsigned hb = rest & (~0u << bA);
        bB = __ffs(hb ? hb : rest) - 1;
      }
      const int jA = cc * 32 + bA;
      rA = vl_pick<M>(fr, vl_used<M>(u0, u1, jA), ~(M)0, kA);
      if (rA < 0) {  // no round left for a pending pair
        ok = false;
        cur = 0;
        cc = nch;
        bB = -1;
      } else if (bB >= 0) {
        rB = vl_pick<M>(fr, vl_used<M>(u0, u1, cc * 32 + bB), (rA & 1) ? EVEN : ODD, kB);
      }
    }
    const bool evA = rA >= 0 && !(rA & 1), pB = rB >= 0;
    // even set: A if its round is even, else B; odd set: the other one
    const int je = evA ? cc * 32 + bA : (pB ? cc * 32 + bB : 0), re = evA ? rA : (pB ? rB : -1);
    const int jo = evA ? (pB ? cc * 32 + bB : 0) : (rA >= 0 ? cc * 32 + bA : 0);
    const int ro = evA ? (pB ? rB : -1) : rA;
    const unsigned keyE = re >= 0 ? (unsigned)((je << 6) | re) : (0x80000000u | lane);
    const unsigned keyO = ro >= 0 ? (unsigned)((jo << 6) | ro) : (0x80000000u | lane);
    const unsigned peersE = __match_any_sync(CS_FULL, keyE);
    const unsigned peersO = __match_any_sync(CS_FULL, keyO);
    __syncwarp();
    const bool winE = re >= 0 && __ffs(peersE) - 1 == lane, winO = ro >= 0 && __ffs(peersO) - 1 == lane;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const bool win = t ? winO : winE;
      if (!win) continue;
      const int j = t ? jo : je, r = t ? ro : re;
      const bool isA = (r == rA) && (j == cc * 32 + bA);
      const int k = isA ? kA : kB, b = isA ? bA : bB;
      int tl = seg_l[0];
#pragma unroll
      for (int kk = 0; kk < VB_SEG; ++kk)
        if (kk == k) {
          fr[kk] &= ~((M)1 << r);
          tl = seg_l[kk];
        }
      cur &= ~(1u << b);
      tab[r][tl] = code[j];
      atomicOr(r < 32 ? &u0[j] : &u1[j], 1u << (r & 31));  // native 32-bit shared atomic
    }
    __syncwarp();
  }
  return __all_sync(CS_FULL, ok);
}

// segments of one particle: table lanes cL, cL + 1, ... with free rounds
// (n slots starting at round cO of table lane cL)
__device__ __forceinline__ void vl_segments(int n, int cL, int cO, int R,
                                            unsigned long long *fr, int *seg_l) {
  int rest = n, lo = cO;
#pragma unroll
  for (int k = 0; k < VB_SEG; ++k) {
    const int hi = min(R, lo + rest);
    const int w2 = hi - lo;
    fr[k] = w2 > 0 ? (((w2 >= 64 ? ~0ull : ((1ull << w2) - 1))) << lo) : 0ull;
    seg_l[k] = min(cL + k, 31);
    rest -= max(w2, 0);
    lo = 0;
  }
}

// One home cell t by one warp: round table, lane map and round count.  Cells
// above MAXP particles or JCAP candidates go to `crowd` (the second pass) or,
// in the second pass (crowd null), are reported (status 2).
template <int NW, int MAXP, int JCAP>
__device__ __forceinline__ void vb_cell(const Box &b, const int32_t *start, const double *x,
                                        const double *y, const double *z, double rl2,
                                        const VList &L, unsigned *status,
                                        VBuildSmemT<NW, MAXP, JCAP> &S, int w, int lane,
                                        int64_t t, int32_t *crowd) {
  constexpr int NPL = MAXP / 32;  // particles per lane
  static_assert(NPL == 1 || NPL == 2, "32 or 64 particles per home cell");
  using MM = typename std::conditional<(MAXP > 32), unsigned long long, unsigned>::type;
  const int h0 = (int)(t % b.owned_x), h1 = (int)((t / b.owned_x) % b.nc[1]),
            h2 = (int)(t / ((int64_t)b.owned_x * b.nc[1]));
  const int64_t cell = box_cell(b, h0, h1, h2);
  int st = 0, cnt = 0;
  double s0 = 0, s1 = 0, s2 = 0;
  if (lane < 14) vl_source(b, start, h0, h1, h2, lane, &st, &cnt, s0, s1, s2);
  const int na = __shfl_sync(CS_FULL, cnt, 0), a0 = __shfl_sync(CS_FULL, st, 0);
  int incl = cnt;
#pragma unroll
  for (int k = 1; k < 16; k <<= 1) {
    const int v = __shfl_up_sync(CS_FULL, incl, k);
    if (lane >= k) incl += v;
  }
  const int excl = incl - cnt;
  const int nj = __shfl_sync(CS_FULL, incl, 13);
  const int nch = (nj + 31) / 32;
  uint8_t *lm = L.imap + cell * 96;
  if (na == 0 || na > MAXP || nj > JCAP) {
    if (na > MAXP || nj > JCAP) {
      if (crowd) {  // a cell for the second pass
        if (lane == 0) crowd[atomicAdd(L.ncrowd, 1)] = (int32_t)t;
      } else {
        atomicOr(status, 2u);
      }
    }
    if (lane == 0) L.nround[cell] = 0;
    lm[lane] = lm[32 + lane] = 0xFF;
    return;
  }
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    const int p = k * 32 + lane;
    if (p < na) {
      S.hx[w][p][0] = __ldg(x + a0 + p);
      S.hx[w][p][1] = __ldg(y + a0 + p);
      S.hx[w][p][2] = __ldg(z + a0 + p);
    }
  }
  __syncwarp();
  // pass 1: candidates (lane = j) -> rows (lane = home particle), list lengths
  int len0 = 0, len1 = 0;
  for (int c = 0; c < nch; ++c) {
    const int tj = c * 32 + lane;
    int e = 0;
#pragma unroll
    for (int k = 8; k >= 1; k >>= 1) {
      const int cand = e + k;
      const int ex = __shfl_sync(CS_FULL, excl, cand < 14 ? cand : 13);
      if (cand < 14 && ex <= tj) e = cand;
    }
    const int q = tj - __shfl_sync(CS_FULL, excl, e);
    const int sst = __shfl_sync(CS_FULL, st, e);
    const double sx = __shfl_sync(CS_FULL, s0, e), sy = __shfl_sync(CS_FULL, s1, e),
                 sz = __shfl_sync(CS_FULL, s2, e);
    MM mask = 0;
    if (tj < nj) {
      const double xj = __ldg(x + sst + q) + sx, yj = __ldg(y + sst + q) + sy,
                   zj = __ldg(z + sst + q) + sz;
      const int ilim = e == 0 ? q : na;  // intra: pairs i < j only
      for (int i = 0; i < ilim; ++i) {
        const double dx = S.hx[w][i][0] - xj, dy = S.hx[w][i][1] - yj, dz = S.hx[w][i][2] - zj;
        const double r2 = __fma_rn(dz, dz, __fma_rn(dy, dy, dx * dx));
        mask |= (MM)(r2 < rl2) << i;
      }
      S.code[w][tj] = (uint16_t)((e << 8) | q);
    }
    for (int i = 0; i < na; ++i) {
      const unsigned bal = __ballot_sync(CS_FULL, (unsigned)(mask >> i) & 1u);
      if (lane == (i & 31)) {
        S.row[w][i][c] = bal;
        if (i < 32) len0 += __popc(bal);
        else len1 += __popc(bal);
      }
    }
  }
  const int n0 = lane < na ? len0 + 1 + len0 / 16 : 0;  // slots: pairs + slack
  const int n1 = 32 + lane < na ? len1 + 1 + len1 / 16 : 0;
  const int P = warp_sum(n0 + n1);
  if (warp_sum(len0 + len1) == 0) {
    if (lane == 0) L.nround[cell] = 0;
    lm[lane] = lm[32 + lane] = 0xFF;
    return;
  }
  // at most VB_SEG table lanes per particle: n <= (VB_SEG - 1) R + 1
  int R = max((P + 31) / 32,
              ((int)__reduce_max_sync(CS_FULL, (unsigned)max(n0, n1)) + VB_SEG - 3) / (VB_SEG - 1));
  bool placed = false;
  uint16_t(*tab)[32] = reinterpret_cast<uint16_t(*)[32]>(L.desc + cell * (VL_RMAX * 32));
  unsigned *u0 = S.used[w][0], *u1 = S.used[w][1];
  while (!placed && R <= VL_RMAX) {
    // lane-major layout: particles in order, at most two per table lane (a
    // particle that would be the third in a lane starts the next one)
    int Lc = 0, off = 0, segs = 0, cL0 = 0, cO0 = 0, cL1 = 0, cO1 = 0;
    for (int p = 0; p < na; ++p) {
      int rest = __shfl_sync(CS_FULL, p < 32 ? n0 : n1, p & 31);
      if (off != 0 && segs >= 2) {
        ++Lc;
        off = segs = 0;
      }
      if (off & 1) {  // switch rounds are even: the force kernel takes rounds in pairs
        if (++off == R) {
          ++Lc;
          off = segs = 0;
        }
      }
      if (lane == (p & 31)) {
        if (p < 32) {
          cL0 = Lc;
          cO0 = off;
        } else {
          cL1 = Lc;
          cO1 = off;
        }
      }
      const int take = min(rest, R - off);
      rest -= take;
      off += take;
      ++segs;
      if (off == R) {
        ++Lc;
        off = segs = 0;
      }
      if (rest > 0) {  // (rest < VB_SEG * R: a short loop, no integer division)
        while (rest >= R) {
          rest -= R;
          ++Lc;
        }
        off = rest;
        segs = off ? 1 : 0;
      }
    }
    if (Lc + (off ? 1 : 0) > 32) {
      ++R;
      continue;
    }
    unsigned long long fr0[VB_SEG], fr1[VB_SEG];
    int seg0[VB_SEG], seg1[VB_SEG];
    vl_segments(n0, cL0, cO0, R, fr0, seg0);
    vl_segments(n1, cL1, cO1, R, fr1, seg1);
    for (int r = 0; r < R; ++r) tab[r][lane] = VL_IDLE;
    // lane -> (first particle, second particle, switch round)
    S.lmap[w][lane] = S.lmap[w][32 + lane] = 0xFF;
    S.lmap[w][64 + lane] = (uint8_t)R;
    for (int j = lane; j < nj; j += 32) u0[j] = u1[j] = 0u;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      const int p = k * 32 + lane;
      const int cL = k ? cL1 : cL0, cO = k ? cO1 : cO0;
      const unsigned long long *fr = k ? fr1 : fr0;
      const int *seg = k ? seg1 : seg0;
      if (p < na) {
        if (cO != 0) {
          S.lmap[w][32 + cL] = (uint8_t)p;
          S.lmap[w][64 + cL] = (uint8_t)cO;
        } else {
          S.lmap[w][cL] = (uint8_t)p;
        }
#pragma unroll
        for (int kk = 1; kk < VB_SEG; ++kk)
          if (fr[kk]) S.lmap[w][seg[kk]] = (uint8_t)p;
      }
    }
    __syncwarp();
    // pass 2: place the pairs (the second particle set after the first)
    bool ok = true;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      if (!ok) break;
      const int p = k * 32 + lane;
      unsigned long long *fr = k ? fr1 : fr0;
      const int *seg = k ? seg1 : seg0;
      const unsigned *prow = S.row[w][p < na ? p : 0];
      const int pn = p < na ? nch : 0;
      if (R <= 32) {
        unsigned f32[VB_SEG];
#pragma unroll
        for (int kk = 0; kk < VB_SEG; ++kk) f32[kk] = (unsigned)fr[kk];
        ok = vl_place(prow, pn, f32, seg, u0, u1, S.code[w], tab, lane);
      } else {
        ok = vl_place(prow, pn, fr, seg, u0, u1, S.code[w], tab, lane);
      }
    }
    if (ok) {
      placed = true;
    } else {  // a pair found no free round: retry with one more round
      __syncwarp();
      ++R;  // (the next attempt re-initialises its rounds)
    }
  }
  if (!placed) {
    if (lane == 0) {
      atomicOr(status, 4u);
      L.nround[cell] = 0;
    }
    lm[lane] = lm[32 + lane] = 0xFF;
    return;
  }
  if (lane == 0) L.nround[cell] = R;
  lm[lane] = S.lmap[w][lane];
  lm[32 + lane] = S.lmap[w][32 + lane];
  lm[64 + lane] = S.lmap[w][64 + lane];
  __syncwarp();
}

__global__ void __launch_bounds__(VB_NW * 32, VB_MINB) k_verlet_build(Box b, const int32_t *start,
                                                                      const double *x, const double *y,
                                                                      const double *z, double rl2,
                                                                      VList L, unsigned *status) {
  __shared__ VBMain S;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nhome = (int64_t)b.owned_x * b.nc[1] * b.nc[2];
  for (int64_t t = (int64_t)blockIdx.x * VB_NW + w; t < nhome; t += (int64_t)gridDim.x * VB_NW)
    vb_cell(b, start, x, y, z, rl2, L, status, S, w, lane, t, L.crowd);
}

// second pass: the (rare) cells of 33-64 particles, one warp each
__global__ void __launch_bounds__(32) k_verlet_build_crowded(Box b, const int32_t *start,
                                                             const double *x, const double *y,
                                                             const double *z, double rl2, VList L,
                                                             unsigned *status) {
  __shared__ VBCrowd S;
  const int n = *L.ncrowd;
  for (int i = blockIdx.x; i < n; i += gridDim.x)
    vb_cell(b, start, x, y, z, rl2, L, status, S, 0, threadIdx.x, (int64_t)L.crowd[i],
            (int32_t *)nullptr);
}

__global__ void k_wrap_copy(int64_t n, double Lx, double Ly, double Lz, double *x, double *y,
                            double *z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = wrap_far(x[i], Lx);
    y[i] = wrap_far(y[i], Ly);
    z[i] = wrap_far(z[i], Lz);
  }
}

__global__ void k_copy3(int64_t n, const double *x, const double *y, const double *z, double *xo,
                        double *yo, double *zo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    xo[i] = x[i];
    yo[i] = y[i];
    zo[i] = z[i];
  }
}

// kick + drift without wrapping; flag = 1 once a particle is more than
// sqrt(lim2) from its position at the last list build
__global__ void k_kick_drift_track(int64_t n, double hdtm, double dt, const double *fx,
                                   const double *fy, const double *fz, double *vx, double *vy,
                                   double *vz, double *x, double *y, double *z, const double *x0,
                                   const double *y0, const double *z0, double lim2, int32_t *flag) {
  bool far = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double ux = __fma_rn(hdtm, fx[i], vx[i]);
    const double uy = __fma_rn(hdtm, fy[i], vy[i]);
    const double uz = __fma_rn(hdtm, fz[i], vz[i]);
    vx[i] = ux;
    vy[i] = uy;
    vz[i] = uz;
    const double nx = __fma_rn(dt, ux, x[i]), ny = __fma_rn(dt, uy, y[i]), nz = __fma_rn(dt, uz, z[i]);
    x[i] = nx;
    y[i] = ny;
    z[i] = nz;
    const double dx = nx - x0[i], dy = ny - y0[i], dz = nz - z0[i];
    far |= __fma_rn(dz, dz, __fma_rn(dy, dy, dx * dx)) > lim2;
  }
  if (__any_sync(CS_FULL, far) && (threadIdx.x & 31) == 0) *flag = 1;  // same value from every writer
}

// post-kick (kick != 0: v += hdtm f) fused with the exact prediction of the
// NEXT step's displacement flag: the next kick-drift computes
// w = fma(hdtm, f, v), x' = fma(dt, w, x) from the same f, so the flag is
// known at the end of this step (the x-slab step takes its global rebuild
// decision there, off the critical path of the next step)
__global__ void k_kick_predict(int64_t n, double hdtm, double dt, int kick, const double *fx,
                               const double *fy, const double *fz, double *vx, double *vy,
                               double *vz, const double *x, const double *y, const double *z,
                               const double *x0, const double *y0, const double *z0, double lim2,
                               int32_t *flag) {
  bool far = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double fxi = fx[i], fyi = fy[i], fzi = fz[i];
    double ux = vx[i], uy = vy[i], uz = vz[i];
    if (kick) {
      ux = __fma_rn(hdtm, fxi, ux);
      uy = __fma_rn(hdtm, fyi, uy);
      uz = __fma_rn(hdtm, fzi, uz);
      vx[i] = ux;
      vy[i] = uy;
      vz[i] = uz;
    }
    const double nx = __fma_rn(dt, __fma_rn(hdtm, fxi, ux), x[i]);
    const double ny = __fma_rn(dt, __fma_rn(hdtm, fyi, uy), y[i]);
    const double nz = __fma_rn(dt, __fma_rn(hdtm, fzi, uz), z[i]);
    const double dx = nx - x0[i], dy = ny - y0[i], dz = nz - z0[i];
    far |= __fma_rn(dz, dz, __fma_rn(dy, dy, dx * dx)) > lim2;
  }
  if (__any_sync(CS_FULL, far) && (threadIdx.x & 31) == 0) *flag = 1;  // same value from every writer
}

extern "C" int cs_vv_kick_predict(int64_t n, double hdtm, double dt, int kick, const double *fx,
                                  const double *fy, const double *fz, double *vx, double *vy,
                                  double *vz, const double *x, const double *y, const double *z,
                                  const double *x0, const double *y0, const double *z0,
                                  double half_skin, int32_t *flag, void *stream) {
  if (n <= 0) return CS_OK;
  k_kick_predict<<<grid_for(n, 256), 256, 0, cs_stream(stream)>>>(
      n, hdtm, dt, kick, fx, fy, fz, vx, vy, vz, x, y, z, x0, y0, z0, half_skin * half_skin, flag);
  return cs_check_launch("vv_kick_predict");
}

extern "C" int cs_wrap_positions(int64_t n, const cs_box *b, double *x, double *y, double *z,
                                 void *stream) {
  if (n <= 0) return CS_OK;
  k_wrap_copy<<<grid_for(n, 256), 256, 0, cs_stream(stream)>>>(n, b->L[0], b->L[1], b->L[2], x, y, z);
  return cs_check_launch("wrap_positions");
}

extern "C" int cs_vv_kick_drift_track(int64_t n, double hdtm, double dt, const double *fx,
                                      const double *fy, const double *fz, double *vx, double *vy,
                                      double *vz, double *x, double *y, double *z,
                                      const double *x0, const double *y0, const double *z0,
                                      double half_skin, int32_t *flag, void *stream) {
  if (n <= 0) return CS_OK;
  k_kick_drift_track<<<grid_for(n, 256), 256, 0, cs_stream(stream)>>>(
      n, hdtm, dt, fx, fy, fz, vx, vy, vz, x, y, z, x0, y0, z0, half_skin * half_skin, flag);
  return cs_check_launch("vv_kick_drift_track");
}

extern "C" int cs_verlet_build(const cs_box *bx, const cs_lj *lj, double skin,
                               const int32_t *cell_start, const double *x, const double *y,
                               const double *z, void *list, size_t list_bytes, double *x0,
                               double *y0, double *z0, int64_t n, unsigned *status_dev,
                               void *stream) {
  CS_TRY(cs_upload_stencil());
  cudaStream_t st = cs_stream(stream);
  Box b;
  CS_TRY(make_box(bx, &b));
  CS_REQUIRE(skin >= 0, "skin must be >= 0");
  for (int k = 0; k < 3; ++k) {
    CS_REQUIRE(b.gnc[k] >= 3, "Verlet lists need >= 3 cells per axis");
    CS_REQUIRE(b.L[k] / b.gnc[k] >= (lj->rc + skin) * (1 - 1e-12),
               "cell edge %.6g on axis %d is below rc + skin = %.6g", b.L[k] / b.gnc[k], k,
               lj->rc + skin);
  }
  CS_REQUIRE(list_bytes >= vl_bytes(b), "Verlet list buffer too small (%zu < %zu)",
             list_bytes, vl_bytes(b));
  CS_REQUIRE(status_dev, "status pointer required");
  VList L = vl_view(list, b);
  const double rl = lj->rc + skin;
  const double rl2 = rl * rl * (1.0 + 1e-12);
  const int64_t nhome = (int64_t)b.owned_x * b.nc[1] * b.nc[2];
  const int64_t blocks = (nhome + VB_NW - 1) / VB_NW;
  if (b.ncells > nhome) {  // ghost cells own no home tasks
    CS_CUDA(cudaMemsetAsync(L.nround, 0, sizeof(int32_t) * b.ncells, st));
  }
  if (blocks > 0) {
    CS_CUDA(cudaMemsetAsync(L.ncrowd, 0, sizeof(int32_t), st));
    k_verlet_build<<<(unsigned)blocks, VB_NW * 32, 0, st>>>(b, cell_start, x, y, z, rl2, L, status_dev);
    // (returns at once when no cell was crowded; the grid reads the count on the device)
    k_verlet_build_crowded<<<(unsigned)(nhome < 592 ? nhome : 592), 32, 0, st>>>(b, cell_start, x, y, z,
                                                                                rl2, L, status_dev);
  }
  // the buffered block layout only changes with the cell list: compute it here
  // once per rebuild instead of in every force evaluation
  int nbk[3];
  if (block_grid(b, nbk) == CS_OK) {
    ShellArgs SA;
    memset(&SA, 0, sizeof(SA));
    SA.A.b = b;
    SA.A.start = cell_start;
    SA.A.vl_nround = L.nround;  // (a home without listed pairs is not a merge contributor)
    for (int k = 0; k < 3; ++k) SA.A.nbk[k] = nbk[k];
    const int B[3] = {b.blk[0], b.blk[1], b.blk[2]};
    if (b.blk[0] * b.blk[1] * b.blk[2] <= SH_MAXB && build_merge_table(B, &SA.mt) == CS_OK) {
      const int64_t nblocks = (int64_t)nbk[0] * nbk[1] * nbk[2];
      k_block_sizes<<<grid_for(nblocks * 32, 256), 256, 0, st>>>(SA, L.bsizes);
      CS_TRY(cs_exclusive_scan_i32(L.bsizes, L.boff, nblocks, L.scan_ws,
                                   cs_scan_ws_bytes(b.ncells + 1), st));
      k_vl_tables<<<(unsigned)nblocks, SH_NW * 32, vl_table_bytes(), st>>>(SA, L.tab);
    }
  }
  if (x0 && n > 0) k_copy3<<<grid_for(n, 256), 256, 0, st>>>(n, x, y, z, x0, y0, z0);
  return cs_check_launch("verlet_build");
}

extern "C" int cs_lj_forces_verlet(const cs_box *bx, const cs_lj *lj, int sched, int64_t npart,
                                   const int32_t *cell_start, const void *list, const double *x,
                                   const double *y, const double *z, double *fx, double *fy,
                                   double *fz, double *energy_dev, unsigned long long *npairs_dev,
                                   unsigned *status_dev, void *ws, size_t ws_bytes, void *stream) {
  CS_REQUIRE(list, "null Verlet list");
  return lj_forces_impl(bx, lj, sched, npart, cell_start, list, x, y, z, fx, fy, fz, energy_dev,
                        npairs_dev, status_dev, ws, ws_bytes, cs_stream(stream));
}

// ------------------------------------------------ in-place rebinning helper --
__global__ void k_copy7(int64_t n, const double *x, const double *y, const double *z,
                        const double *vx, const double *vy, const double *vz, const int32_t *id,
                        double *xo, double *yo, double *zo, double *vxo, double *vyo,
                        double *vzo, int32_t *ido) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    xo[i] = x[i];
    yo[i] = y[i];
    zo[i] = z[i];
    vxo[i] = vx[i];
    vyo[i] = vy[i];
    vzo[i] = vz[i];
    ido[i] = id[i];
  }
}

extern "C" int cs_copy7(int64_t n, const double *x, const double *y, const double *z,
                        const double *vx, const double *vy, const double *vz, const int32_t *id,
                        double *xo, double *yo, double *zo, double *vxo, double *vyo, double *vzo,
                        int32_t *ido, void *stream) {
  if (n <= 0) return CS_OK;
  k_copy7<<<grid_for(n, 256), 256, 0, cs_stream(stream)>>>(n, x, y, z, vx, vy, vz, id, xo, yo,
                                                            zo, vxo, vyo, vzo, ido);
  return cs_check_launch("copy7");
}

// ------------------------------- conditional rebuild inside a CUDA graph --
// The rebuild decision stays on the device: a one-thread kernel turns the
// displacement flag into the graph's IF condition (and clears the flag), and
// the rebuild work is captured into the body of that conditional node.
__global__ void k_set_cond(cudaGraphConditionalHandle h, int32_t *flag, int32_t *count) {
  const int32_t v = *flag;
  *flag = 0;
  if (v && count) ++*count;
  cudaGraphSetConditional(h, v ? 1u : 0u);
}

extern "C" int cs_capture_if_begin(void *stream, void *side_stream, int32_t *flag,
                                   int32_t *count) {
  cudaStream_t st = cs_stream(stream), side = cs_stream(side_stream);
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t *deps = nullptr;
  size_t nd = 0;
  CS_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  CS_REQUIRE(cs == cudaStreamCaptureStatusActive, "cs_capture_if_begin: stream is not capturing");
  cudaGraphConditionalHandle h;
  CS_CUDA(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
  k_set_cond<<<1, 1, 0, st>>>(h, flag, count);
  CS_TRY(cs_check_launch("set_cond"));
  CS_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  alignas(cudaGraphNodeParams) unsigned char pbuf[sizeof(cudaGraphNodeParams)];
  memset(pbuf, 0, sizeof(pbuf));  // (the union has no default constructor)
  cudaGraphNodeParams &p = *reinterpret_cast<cudaGraphNodeParams *>(pbuf);
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeIf;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CS_CUDA(cudaGraphAddNode(&node, g, deps, nd, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  CS_CUDA(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  CS_CUDA(cudaStreamBeginCaptureToGraph(side, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  return CS_OK;
}

extern "C" int cs_capture_if_end(void *side_stream) {
  cudaGraph_t g;
  CS_CUDA(cudaStreamEndCapture(cs_stream(side_stream), &g));
  return CS_OK;
}
