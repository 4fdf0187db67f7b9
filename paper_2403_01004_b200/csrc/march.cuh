// r-marching shared-memory kernel for the 19-point aligned (Spitzer)
// operator -- the hot path of C3/C4/C5 (K3 fused stage, K4 F+argmax, K7
// PCG matvec).  DESIGN.md §4 "K3".
//
// A block owns a (MTJ x MTK) theta-phi tile (phi = lanes: 256-byte coalesced
// rows) of an r-chunk of R planes and marches along r.  Per plane it
//   * stages T (4-slot ring, prefetch distance 2 planes), beta (3 slots) and
//     the per-(r,theta) metric rows (4 slots) with a one-node halo through
//     cp.async, one group per plane;
//   * keeps each own node's T(t-1), T(t) (r-neighbours), the r-flux queue
//     E_{0,+}(t-2), E_{0,+}(t-1), the node part of G and the epilogue
//     operands (LDG-prefetched one plane ahead) in registers;
//   * evaluates the six edge fluxes E_{a,s} of every tile node once, one
//     flux component on the 96-node halo ring, publishes the in-plane
//     components through shared memory and finalises plane t-1 in the
//     oracle's summation order (oracle/operators.py aligned_apply):
//        own = ((E0- - E0+) + (E1- - E1+)) + (E2- - E2+)
//        nbr = (E1+(j-1) - E1-(j+1)) + (E2+(k-1) - E2-(k+1))
//        G   = (E0+(i-1) - E0-(i+1)) + (own + nbr)
//   * one cp.async wait + one __syncthreads per plane.
// Every HBM byte of T and beta is read once per plane (plus the thin halo), so
// the stage streams 8 arrays: T, beta(3), u_{k-2}, u0, y0 in and u_k out.
//
// Arithmetic is the oracle's expression by expression (compiled with
// -fmad=false), only the schedule differs: results are bitwise identical.
#pragma once
#include <type_traits>

#include "kernels.cuh"

namespace pc {

constexpr int MTK = 32;          // phi extent of a tile (lanes)
constexpr int MTY = 8;           // warps = thread rows
constexpr int NPT = 2;           // tile nodes per thread (rows ty, ty + MTY)
constexpr int MTJ = MTY * NPT;   // theta extent of a tile
constexpr int MHJ = MTJ + 2;
constexpr int MHK = MTK + 2;
constexpr int MHP = MHJ * MHK;
constexpr int MNT = MTY * MTK;   // threads per block
constexpr int NFILL = (MHP + MNT - 1) / MNT;
constexpr int NROWT = 11;        // per-(row, j) tables: iL2[6], wo01[4], iVal2
constexpr int TSL = 3;           // T slots: t, t+1, t+2 in flight
constexpr int BSL = 2;           // beta slots: t, t+1 in flight
constexpr int RSL = 3;           // row-table slots: t-1 (iv), t, t+1 in flight
constexpr int NEO = 3;           // epilogue operand arrays staged per node (max)
constexpr int MTN = MTJ * MTK;   // tile nodes
constexpr int NRING = 2 * MTK + 2 * MTJ;

// r-chunk of this block: zsel == 0 all chunks (chunk = blockIdx.z); zsel > 0
// the interior chunks 1 .. nz-2 (halo exchange overlapped, see sts_stages);
// zsel = -nz the two boundary chunks 0 and nz-1 (after the exchange)
__device__ __forceinline__ int chunk_of(int zsel) {
  if (zsel == 0) return blockIdx.z;
  if (zsel > 0) return blockIdx.z + 1;
  return blockIdx.z == 0 ? 0 : -zsel - 1;
}

struct PlaneMap {
  int mem;      // memory plane to read (ghost planes allowed)
  int row;      // table row
  bool exists;  // node plane exists (else differences clamp to self, E = 0)
};
__device__ __forceinline__ PlaneMap plane_map(const GridDev& g, int p) {
  if (p >= 0 && p < g.n0) return {p, p, true};
  if ((p < 0 && g.ghost_lo0) || (p >= g.n0 && g.ghost_hi0)) return {p, p, true};
  if (g.per0 && g.n0g > 1) {
    int w = p < 0 ? g.n0 - 1 : 0;
    return {w, w, true};
  }
  int c = p < 0 ? 0 : g.n0 - 1;
  return {c, c, false};
}
// in-plane coordinate mapping: wrap if periodic, else clamp to the edge (self)
__device__ __forceinline__ int map_j(const GridDev& g, int j, bool& ok) {
  if (j >= 0 && j < g.n1) { ok = true; return j; }
  if (g.per1 && g.n1 > 1) { ok = true; return ((j % g.n1) + g.n1) % g.n1; }
  ok = false;
  return j < 0 ? 0 : g.n1 - 1;
}
__device__ __forceinline__ int map_k(const GridDev& g, int k, bool& ok) {
  if (k >= 0 && k < g.n2) { ok = true; return k; }
  if (g.per2 && g.n2 > 1) { ok = true; return ((k % g.n2) + g.n2) % g.n2; }
  ok = false;
  return k < 0 ? 0 : g.n2 - 1;
}

// ---- async copy helpers (LDGSTS) -----------------------------------------
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// in-plane flux exchange of one plane (compact: only the entries readers use)
//   e1p[(j - (j0-1))][k - k0]   E_{1,+},  e1m[(j - j0)][k - k0]       E_{1,-}
//   e2p[j - j0][(k - (k0-1))]   E_{2,+},  e2m[j - j0][(k - k0)]       E_{2,-}
struct FluxX {
  double e1p[MTJ + 1][MTK];
  double e1m[MTJ + 1][MTK];
  double e2p[MTJ][MTK + 1];
  double e2m[MTJ][MTK + 1];
};
struct MarchSmem {
  double T[TSL][MHP];
  double B[BSL][3][MHP];
  FluxX E[2];                   // per plane parity
  double EO[2][NEO][MTN];       // epilogue operands of planes t-1 (read), t (landing)
  double rowt[RSL][NROWT][MHJ];
  double ringcol[2][9];         // column tables of the phi-ring columns k0-1, k0+MTK
};

// Re-define a loop-invariant register through an ALU move: its consumers in
// the plane loop then carry no scoreboard dependency on the global load that
// produced it (which ptxas would otherwise re-wait on every iteration, sharing
// the scoreboard with the in-flight epilogue prefetches).
__device__ __forceinline__ double launder(double x) {
  double y;
  asm volatile("mov.b64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// per-column constants (depend on k only)
// (the axis-0 and axis-1 column factors iL1 are exactly 1 for every grid --
// checked by pc_grid_create -- so only the phi pair is carried)
struct ColT {
  double il1[2];
  double w2[2];
  double ivg;
};
__device__ __forceinline__ void load_col(const GridDev& g, int k, ColT& c) {
#pragma unroll
  for (int q = 0; q < 2; ++q) c.il1[q] = __ldg(g.iL1[4 + q] + k);
  c.w2[0] = __ldg(g.wo2[0] + k);
  c.w2[1] = __ldg(g.wo2[1] + k);
  c.ivg = __ldg(g.iValg + k);
}

// Edge fluxes of one node in the oracle's order (aligned_E).  ONLY_A < 0:
// all six; else only E_{ONLY_A, ONLY_S} (and only the differences it needs).
//   Tn[x][0] = T(m + e_x), Tn[x][1] = T(m - e_x) (self if missing)
//   rw: row tables of the node's (plane, theta row): iL2[6], wo01[4]
// Edge fluxes of one node in the oracle's order (aligned_E), from the
// metric values of the node: il2[x][t] (iL2 row part; x < 2 are the full
// inverse edge lengths, x = 2 is multiplied by the phi column part il1[t]),
// w01 (wo01 row part), w2 (wo2 column part).  ONLY_A < 0: all six fluxes;
// else only E_{ONLY_A, ONLY_S} (and only the differences it needs).
//   Tn[x][0] = T(m + e_x), Tn[x][1] = T(m - e_x) (self if missing)
template <int ONLY_A, int ONLY_S>
__device__ __forceinline__ void node_E_core(double Tv, const double (&Tn)[3][2], const double (&bv)[3],
                                            const double (&il2)[3][2], const double (&w01)[4],
                                            const double (&il1)[2], const double (&w2)[2], double (&E)[3][2]) {
  double bil[3][2], p[3][2];
#pragma unroll
  for (int x = 0; x < 3; ++x) {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const bool need_p = !(ONLY_A >= 0 && x == ONLY_A && t != ONLY_S);
      const bool need_bil = need_p || (ONLY_A < 0) || (x == ONLY_A && t == ONLY_S);
      if (need_bil) bil[x][t] = bv[x] * (x < 2 ? il2[x][t] : il2[x][t] * il1[t]);
      if (need_p) p[x][t] = bil[x][t] * (t == 0 ? (Tn[x][0] - Tv) : (Tv - Tn[x][1]));
      else p[x][t] = 0.0;
    }
  }
  double f[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int s0 = (q >> 2) & 1, s1 = (q >> 1) & 1, s2 = q & 1;
    if (ONLY_A >= 0) {
      const int sa = ONLY_A == 0 ? s0 : (ONLY_A == 1 ? s1 : s2);
      if (sa != ONLY_S) { f[q] = 0.0; continue; }
    }
    const double sv = (p[0][s0] + p[1][s1]) + p[2][s2];
    const double om = w01[s0 * 2 + s1] * w2[s2];
    f[q] = om * sv;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (ONLY_A >= 0 && (a != ONLY_A || s != ONLY_S)) { E[a][s] = 0.0; continue; }
      double acc = 0.0;
      bool first = true;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int sa = a == 0 ? (q >> 2) & 1 : (a == 1 ? (q >> 1) & 1 : q & 1);
        if (sa != s) continue;
        acc = first ? f[q] : acc + f[q];
        first = false;
      }
      E[a][s] = bil[a][s] * acc;
    }
  }
}

// row tables laid out [table][row] (stride rstride)
template <int ONLY_A, int ONLY_S>
__device__ __forceinline__ void node_E(double Tv, const double (&Tn)[3][2], const double (&bv)[3],
                                       const double* rw, int rstride, const double (&il1)[2],
                                       const double (&w2)[2], double (&E)[3][2]) {
  double il2[3][2], w01[4];
#pragma unroll
  for (int q = 0; q < 6; ++q) il2[q >> 1][q & 1] = rw[q * rstride];
#pragma unroll
  for (int q = 0; q < 4; ++q) w01[q] = rw[(6 + q) * rstride];
  node_E_core<ONLY_A, ONLY_S>(Tv, Tn, bv, il2, w01, il1, w2, E);
}
// row tables laid out [row][12] (16-byte aligned): pairs come in one LDS.128
template <int ONLY_A, int ONLY_S>
__device__ __forceinline__ void node_E_rows(double Tv, const double (&Tn)[3][2], const double (&bv)[3],
                                            const double* rw, const double (&il1)[2], const double (&w2)[2],
                                            double (&E)[3][2]) {
  const double2* r2 = reinterpret_cast<const double2*>(rw);
  double il2[3][2], w01[4];
#pragma unroll
  for (int x = 0; x < 3; ++x) {
    const double2 v = r2[x];
    il2[x][0] = v.x;
    il2[x][1] = v.y;
  }
  const double2 wa = r2[3], wb = r2[4];
  w01[0] = wa.x;
  w01[1] = wa.y;
  w01[2] = wb.x;
  w01[3] = wb.y;
  node_E_core<ONLY_A, ONLY_S>(Tv, Tn, bv, il2, w01, il1, w2, E);
}

// Slot of the plane partial of one warp of a marching block: warp w of tile
// (blockIdx.y, blockIdx.x) on local plane tf; S = tiles x warps per plane
// (the GPU-count-invariant reduction order, kernels.cuh PlaneRed).
__device__ __forceinline__ int64_t march_slot(int tf) {
  const int w = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
  return (((int64_t)tf * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * (MNT / 32) + w;
}
// epilogues with a plane_end(tf) member get it called by every thread after
// plane tf is finalised (block-uniform)
template <class E, class = void>
struct has_plane_end : std::false_type {};
template <class E>
struct has_plane_end<E, std::void_t<decltype(&E::plane_end)>> : std::true_type {};

// Epilogue contract (per tile node n of the thread):
//   Epi::NOPS, epi.opnd(q)                 nodal operand arrays the kernel stages
//                                          through cp.async one plane ahead
//   epi(n, g, i, j, k, o, F, uc, pin, ov, W)  uc = input value at the node,
//                                          ov[q] = staged operands, W = the
//                                          node's inner-product weight rho V
//                                          (formed only if Epi::NEEDS_W)
//   epi.plane_end(tf)                      optional: after plane tf is finalised
//   epi.finish(g)                          block reduction, if any
template <class Epi>
__global__ void __launch_bounds__(MNT, 2) k_aligned_march(GridDev g, AlignedOp op, const double* __restrict__ Tin,
                                                          Epi epi, int R, int zsel, const int* skip) {
  extern __shared__ __align__(16) unsigned char march_smem[];
  MarchSmem& S = *reinterpret_cast<MarchSmem*>(march_smem);
  if (skip && *skip) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * MTK + tx;
  const int k0 = blockIdx.x * MTK, j0 = blockIdx.y * MTJ, i0 = chunk_of(zsel) * R;
  const int iend = min(i0 + R, g.n0);
  const int kg = k0 + tx;

  // smem fill slots of this thread (tile + halo, wrapped / clamped in-plane)
  int foff[NFILL];
#pragma unroll
  for (int q = 0; q < NFILL; ++q) {
    const int e = tid + q * MNT;
    const int hj = e / MHK, hk = e - hj * MHK;
    bool oj, ok;
    const int jj = map_j(g, j0 - 1 + hj, oj), kk = map_k(g, k0 - 1 + hk, ok);
    foff[q] = e < MHP ? jj * g.n2 + kk : -1;
  }
  // row-table fill slot of this thread: tid < NROWT * MHJ
  const bool rton = tid < NROWT * MHJ;
  const int rtab = tid / MHJ, rhj = tid - (tid / MHJ) * MHJ;
  bool rok;
  const int rjj = map_j(g, j0 - 1 + rhj, rok);
  const double* rbase = !rton ? g.iVal2 : (rtab < 6 ? g.iL2[rtab] : (rtab < 10 ? g.wo01[rtab - 6] : g.iVal2));

  bool oko;
  const int km = map_k(g, kg, oko);
  ColT col;
  load_col(g, km, col);
#pragma unroll
  for (int q = 0; q < 2; ++q) col.il1[q] = launder(col.il1[q]);
  col.w2[0] = launder(col.w2[0]);
  col.w2[1] = launder(col.w2[1]);
  col.ivg = launder(col.ivg);
  const bool pin_k = (g.pin_lo2 && kg == 0) || (g.pin_hi2 && kg == g.n2 - 1);
  if (tid < 18) {  // phi-ring column tables
    const int side = tid / 9, q = tid % 9;
    bool okr;
    const int kr = map_k(g, side == 0 ? k0 - 1 : k0 + MTK, okr);
    const double* src = q < 6 ? g.iL1[q] : (q < 8 ? g.wo2[q - 6] : g.iValg);
    S.ringcol[side][q] = __ldg(src + kr);
  }

  // ring node of this thread: tid < NRING.  ra = axis of the one flux
  // component it supplies, rs its side (0 '+', 1 '-').
  int ra = -1, rs = 0, rhj_ = 0, rhk_ = 0;
  if (tid < 2 * MTK) {
    ra = 1;
    rs = tid < MTK ? 0 : 1;
    rhk_ = 1 + (tid % MTK);
    rhj_ = rs == 0 ? 0 : MTJ + 1;
  } else if (tid < NRING) {
    const int q = tid - 2 * MTK;
    ra = 2;
    rs = q < MTJ ? 0 : 1;
    rhj_ = 1 + (q % MTJ);
    rhk_ = rs == 0 ? 0 : MTK + 1;
  }
  bool ring_on = false;
  if (ra >= 0) {
    bool rjo, rko;
    const int gj = j0 - 1 + rhj_, gk = k0 - 1 + rhk_;
    map_j(g, gj, rjo);
    map_k(g, gk, rko);
    // the ring node must exist and be a neighbour of an inside tile node
    ring_on = rjo && rko && (ra == 1 ? (gk < g.n2) : (gj < g.n1));
  }
  const int rh = rhj_ * MHK + rhk_;

  // own nodes
  // (own_ok: the tile position maps to a node, possibly wrapped across a
  // periodic seam -- its fluxes are published for the neighbours; inside: the
  // node is this tile's to finalise)
  const int h0 = (ty + 1) * MHK + (tx + 1);
  const int onode0 = (j0 + ty) * g.n2 + kg;
  bool inside[NPT], own_ok[NPT], pin_j[NPT];
  auto hn = [&](int n) { return h0 + n * MTY * MHK; };
  auto jn = [&](int n) { return j0 + ty + n * MTY; };
  auto onode = [&](int n) { return onode0 + n * MTY * g.n2; };
#pragma unroll
  for (int n = 0; n < NPT; ++n) {
    inside[n] = jn(n) < g.n1 && kg < g.n2;
    bool ojo;
    map_j(g, jn(n), ojo);
    own_ok[n] = ojo && oko;
    pin_j[n] = (g.pin_lo1 && jn(n) == 0) || (g.pin_hi1 && jn(n) == g.n1 - 1);
  }

  auto tslot = [&](int p) { return (p - i0 + 1) % TSL; };
  auto bslot = [&](int p) { return (p - i0 + 1) & (BSL - 1); };
  auto rslot = [&](int p) { return (p - i0 + 1) % RSL; };
  auto eslot = [&](int p) { return (p - i0) & 1; };
  auto issue_T = [&](int p) {
    const PlaneMap pm = plane_map(g, p);
    const double* base = Tin + (int64_t)pm.mem * g.plane;
    double* dst = S.T[tslot(p)];
#pragma unroll
    for (int q = 0; q < NFILL; ++q)
      if (foff[q] >= 0) cp_async8(dst + tid + q * MNT, base + foff[q]);
  };
  auto issue_B = [&](int p) {
    const PlaneMap pm = plane_map(g, p);
    const int64_t base = (int64_t)pm.mem * g.plane;
    const int sl = bslot(p);
#pragma unroll
    for (int q = 0; q < NFILL; ++q)
      if (foff[q] >= 0) {
        const int e = tid + q * MNT;
        const int64_t o = base + foff[q];
        cp_async8(&S.B[sl][0][e], op.beta[0] + o);
        cp_async8(&S.B[sl][1][e], op.beta[1] + o);
        cp_async8(&S.B[sl][2][e], op.beta[2] + o);
      }
  };
  auto issue_rows = [&](int p) {
    if (rton) {
      const PlaneMap pm = plane_map(g, p);
      cp_async8(&S.rowt[rslot(p)][rtab][rhj], rbase + row2(g, pm.row, rjj));
    }
  };
  auto issue_ops = [&](int p) {  // epilogue operands of the own (inside) nodes of plane p
    if (Epi::NOPS > 0) {
      const int64_t base = (int64_t)p * g.plane;
      const int es = eslot(p);
#pragma unroll
      for (int n = 0; n < NPT; ++n)
        if (inside[n]) {
#pragma unroll
          for (int q = 0; q < Epi::NOPS; ++q)
            cp_async8(&S.EO[es][q][tid + n * MNT], epi.opnd(q) + base + onode(n));
        }
    }
  };

  // ---- prologue: T(i0-1..i0+1), beta/rows(i0-1, i0) in one group
  issue_T(i0 - 1);
  issue_T(i0);
  if (i0 + 1 <= iend) issue_T(i0 + 1);
  issue_B(i0 - 1);
  issue_rows(i0 - 1);
  issue_B(i0);
  issue_rows(i0);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  double Tm[NPT], Tc[NPT], qa[NPT], qb[NPT], ownp[NPT];
  double Tmr = 0.0;
  {
    const PlaneMap pm = plane_map(g, i0 - 1);
    const int s0 = tslot(i0 - 1), s1 = tslot(i0), bs = bslot(i0 - 1), rsl = rslot(i0 - 1);
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      const int h = hn(n);
      Tm[n] = S.T[s0][h];
      Tc[n] = S.T[s1][h];
      qa[n] = 0.0;
      qb[n] = 0.0;
      ownp[n] = 0.0;
      if (pm.exists && inside[n]) {  // E_{0,+}(i0 - 1)
        const double Tn[3][2] = {{Tc[n], Tm[n]}, {S.T[s0][h + MHK], S.T[s0][h - MHK]},
                                 {S.T[s0][h + 1], S.T[s0][h - 1]}};
        const double bv[3] = {S.B[bs][0][h], S.B[bs][1][h], S.B[bs][2][h]};
        double E[3][2];
        node_E<0, 0>(Tm[n], Tn, bv, &S.rowt[rsl][0][ty + n * MTY + 1], MHJ, col.il1, col.w2, E);
        qb[n] = E[0][0];
      }
    }
    if (ra >= 0) Tmr = S.T[s0][rh];
  }
  // the prologue reads of the plane i0-1 slots (T, beta) finish before the
  // first refill of those slots (issue_T(i0 + 2), issue_B(i0 + 1)) may land
  __syncthreads();

  // plane loop: planes i0 .. iend-1 compute all fluxes and finalise the
  // previous plane; the peeled last step (t = iend) only forms E_{0,-} and
  // finalises iend-1.
  auto step = [&](int t, auto last_tag) {
    constexpr bool LAST = decltype(last_tag)::value;
    // ---- async prefetch, one group per plane (lands before this plane's barrier):
    // T(t+2), beta/rows(t+1), epilogue operands of plane t
    if (!LAST) {
      if (t + 2 <= iend) issue_T(t + 2);
      issue_B(t + 1);
      issue_rows(t + 1);
      issue_ops(t);
      cp_async_commit();
    }
    const bool exists = LAST ? plane_map(g, t).exists : true;  // t < n0 inside the loop
    const int sc = tslot(t), sp = tslot(t + 1), bs = bslot(t), rsl = rslot(t), rslm = rslot(t - 1);
    const int par = t & 1, pp = par ^ 1;
    const int esm = eslot(t - 1);
    const int r0 = ty, c0 = tx;  // tile coordinates of node 0
    const int tf = t - 1;
    const int ig = tf + g.i0g;
    const bool pin_i = (g.pin_lo0 && ig == 0) || (g.pin_hi0 && ig == g.n0g - 1);
    const int64_t pbase = (int64_t)t * g.plane;
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      const int h = hn(n);
      const int jr = ty + n * MTY + 1;
      double E[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      double Tp = 0.0;
      if (!LAST) Tp = S.T[sp][h];
      if (exists && own_ok[n]) {
        const double Tn[3][2] = {{Tp, Tm[n]}, {S.T[sc][h + MHK], S.T[sc][h - MHK]},
                                 {S.T[sc][h + 1], S.T[sc][h - 1]}};
        const double bv[3] = {S.B[bs][0][h], S.B[bs][1][h], S.B[bs][2][h]};
        if (!LAST) node_E<-1, 0>(Tc[n], Tn, bv, &S.rowt[rsl][0][jr], MHJ, col.il1, col.w2, E);
        else node_E<0, 1>(Tc[n], Tn, bv, &S.rowt[rsl][0][jr], MHJ, col.il1, col.w2, E);
      }
      const int r = r0 + n * MTY;
      if (!LAST) {
        S.E[par].e1p[r + 1][c0] = E[1][0];
        S.E[par].e1m[r][c0] = E[1][1];
        S.E[par].e2p[r][c0 + 1] = E[2][0];
        S.E[par].e2m[r][c0] = E[2][1];
      }
      // ---- finalise plane t-1 (in-plane neighbours' fluxes were published
      // before the previous barrier)
      if (t > i0 && inside[n]) {
        const double nbr = (S.E[pp].e1p[r][c0] - S.E[pp].e1m[r + 1][c0]) + (S.E[pp].e2p[r][c0] - S.E[pp].e2m[r][c0 + 1]);
        const double G = (qa[n] - E[0][1]) + (ownp[n] + nbr);
        const double iv = S.rowt[rslm][10][jr] * col.ivg;
        const int64_t of = pbase - g.plane + onode(n);
        double f = (G * iv) * op.nscale(of);
        const bool pin = pin_i || pin_j[n] || pin_k;
        if (pin) f = 0.0;
        double ov[Epi::NOPS > 0 ? Epi::NOPS : 1];
#pragma unroll
        for (int q = 0; q < Epi::NOPS; ++q) ov[q] = S.EO[esm][q][tid + n * MNT];
        const double W = Epi::NEEDS_W ? op.weight(g, tf, jn(n), kg) : 0.0;
        epi(n, g, tf, jn(n), kg, of, f, Tm[n], pin, ov, W);
      }
      if (!LAST) {
        // ---- shift the per-node queues
        ownp[n] = ((E[0][1] - E[0][0]) + (E[1][1] - E[1][0])) + (E[2][1] - E[2][0]);
        qa[n] = qb[n];
        qb[n] = E[0][0];
        Tm[n] = Tc[n];
        Tc[n] = Tp;
      }
    }
    if constexpr (has_plane_end<Epi>::value) {
      if (t > i0) epi.plane_end(tf);
    }
    // ---- halo ring of plane t: one flux component per ring node
    if (!LAST && ra >= 0) {
      const double Tcr = S.T[sc][rh];
      const double Tpr = S.T[sp][rh];
      double Ev = 0.0;
      if (ring_on) {
        const double Tn[3][2] = {{Tpr, Tmr}, {S.T[sc][rh + MHK < MHP ? rh + MHK : rh], S.T[sc][rh >= MHK ? rh - MHK : rh]},
                                 {S.T[sc][rh + 1], S.T[sc][rh - 1]}};
        const double bv[3] = {S.B[bs][0][rh], S.B[bs][1][rh], S.B[bs][2][rh]};
        double E[3][2];
        const double* rw = &S.rowt[rsl][0][rhj_];
        if (ra == 1) {
          if (rs == 0) {
            node_E<1, 0>(Tcr, Tn, bv, rw, MHJ, col.il1, col.w2, E);
            Ev = E[1][0];
          } else {
            node_E<1, 1>(Tcr, Tn, bv, rw, MHJ, col.il1, col.w2, E);
            Ev = E[1][1];
          }
        } else {
          const double* cs = S.ringcol[rs];
          const double il1[2] = {cs[4], cs[5]};
          const double w2[2] = {cs[6], cs[7]};
          if (rs == 0) {
            node_E<2, 0>(Tcr, Tn, bv, rw, MHJ, il1, w2, E);
            Ev = E[2][0];
          } else {
            node_E<2, 1>(Tcr, Tn, bv, rw, MHJ, il1, w2, E);
            Ev = E[2][1];
          }
        }
      }
      if (ra == 1) {
        if (rs == 0) S.E[par].e1p[0][rhk_ - 1] = Ev;
        else S.E[par].e1m[MTJ][rhk_ - 1] = Ev;
      } else {
        if (rs == 0) S.E[par].e2p[rhj_ - 1][0] = Ev;
        else S.E[par].e2m[rhj_ - 1][MTK] = Ev;
      }
      Tmr = Tcr;
    }
    if (!LAST) {
      cp_async_wait<0>();
      __syncthreads();
    }
  };
#pragma unroll 1
  for (int t = i0; t < iend; ++t) step(t, std::false_type{});
  step(iend, std::true_type{});
  epi.finish(g);
}

// ---- epilogues ----------------------------------------------------------
struct EpiStore {  // F = op(u)
  static constexpr int NOPS = 0;
  static constexpr bool NEEDS_W = false;
  double* F;
  __host__ __device__ __forceinline__ const double* opnd(int) const { return nullptr; }
  __device__ __forceinline__ void operator()(int, const GridDev&, int, int, int, int64_t o, double f, double, bool,
                                             const double*, double) {
    F[o] = f;
  }
  __device__ __forceinline__ void finish(const GridDev&) {}
};

struct EpiStage {  // fused RKL2/RKG2 stage
  static constexpr int NOPS = 3;
  static constexpr bool NEEDS_W = false;
  const double* um2;
  const double* u0;
  const double* y0;
  double* out;
  StageCoef sc;
  int stage;
  int* bad;
  bool nonfinite = false;  // any non-finite value written by this thread (reported once, in finish)
  __host__ __device__ __forceinline__ const double* opnd(int q) const { return q == 0 ? u0 : (q == 1 ? um2 : y0); }
  __device__ __forceinline__ void operator()(int, const GridDev&, int, int, int, int64_t o, double f, double um1,
                                             bool pin, const double* ov, double) {
    const double a0 = ov[0];
    double v = ((((sc.mu * um1) + (sc.nu * ov[1])) + (sc.kap * a0)) + (sc.mtdt * f)) + (sc.gtdt * ov[2]);
    v = pin ? a0 : v;
    out[o] = v;
    nonfinite |= (__double2hiint(v) & 0x7ff00000) == 0x7ff00000;
  }
  __device__ __forceinline__ void finish(const GridDev&) {
    if (nonfinite) atomicMin(bad, stage);
  }
};

// stages 1 and 2 of the aligned STS in one TMA march (FUSE1): the march
// stages u0 and y0 of each plane and forms u1 = u0 + mut1 dt y0 in the input
// slot (k_stage1's expression, pinned nodes keep u0) as the plane lands; the
// epilogue gets u1 as the node value and forms u2 exactly as EpiStage with
// u_{k-2} = u0 (operand 0 serves both), and writes u1 when a stage 3 reads it
struct EpiStageA12 {
  static constexpr int NOPS = 2;
  static constexpr bool NEEDS_W = false;
  static constexpr bool FUSE1 = true;
  const double* u0;
  const double* y0;
  double* out;   // u2
  double* out1;  // u1 (nullptr: s == 2, nothing reads it)
  StageCoef sc;  // stage 2
  double mt1;    // mut1 dt of stage 1
  int* bad;
  bool nf1 = false, nf2 = false;
  __host__ __device__ __forceinline__ const double* opnd(int q) const { return q == 0 ? u0 : y0; }
  __device__ __forceinline__ void operator()(int, const GridDev&, int, int, int, int64_t o, double f, double um1,
                                             bool pin, const double* ov, double) {
    const double a0 = ov[0];
    double v = ((((sc.mu * um1) + (sc.nu * a0)) + (sc.kap * a0)) + (sc.mtdt * f)) + (sc.gtdt * ov[1]);
    v = pin ? a0 : v;
    out[o] = v;
    if (out1) out1[o] = um1;
    nf1 |= (__double2hiint(um1) & 0x7ff00000) == 0x7ff00000;
    nf2 |= (__double2hiint(v) & 0x7ff00000) == 0x7ff00000;
  }
  __device__ __forceinline__ void finish(const GridDev&) {
    if (nf1) atomicMin(bad, 1);
    if (nf2) atomicMin(bad, 2);
  }
};

constexpr int kMaxWarps = 16;  // epilogue block reductions serve 256- and 512-thread marching kernels
__device__ __forceinline__ int block_threads() { return blockDim.x * blockDim.y; }
__device__ __forceinline__ ArgMax block_argmax2d(ArgMax a, double* shv, long long* shi) {
  a = warp_argmax(a);
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  if (lane == 0) {
    shv[w] = a.v;
    shi[w] = a.i;
  }
  __syncthreads();
  ArgMax r{-1.0, 0x7fffffffffffffffLL};
  if (w == 0) {
    if (lane < block_threads() / 32) {
      r.v = shv[lane];
      r.i = shi[lane];
    }
    r = warp_argmax(r);
  }
  __syncthreads();
  return r;
}
__device__ __forceinline__ bool last_block3(unsigned int* counter, int nblk) {
  __shared__ bool amLast;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    unsigned int t = atomicAdd(counter, 1u);
    amLast = (t == (unsigned)nblk - 1);
  }
  __syncthreads();
  return amLast;
}

struct EpiArgmax {  // y0 = F(u0) with the |F| argmax (PTL)
  static constexpr int NOPS = 0;
  static constexpr bool NEEDS_W = false;
  __host__ __device__ __forceinline__ const double* opnd(int) const { return nullptr; }
  double* F;
  double* pv;
  long long* pi;
  unsigned int* counter;
  ArgRes* res;
  ArgMax best;
  // this thread's maximum so far: a thread visits its nodes in increasing AoS
  // index (planes in order, row ty before ty + 8), so a strict > keeps the
  // lowest index among equal maxima without forming indices per node; the
  // index is formed once, in finish()
  int bi = 0, bj = 0, bk = 0;
  __device__ __forceinline__ void operator()(int, const GridDev&, int i, int j, int k, int64_t o, double f, double,
                                             bool, const double*, double) {
    F[o] = f;
    const double a = fabs(f);
    if (a > best.v) {
      best.v = a;
      bi = i;
      bj = j;
      bk = k;
    }
  }
  __device__ __forceinline__ void finish(const GridDev& g) {
    __shared__ double shv[kMaxWarps];
    __shared__ long long shi[kMaxWarps];
    const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int nblk = gridDim.x * gridDim.y * gridDim.z;
    if (best.v >= 0.0) best.i = aos_index(g, bi, bj, bk, 0, 1);
    ArgMax b = block_argmax2d(best, shv, shi);
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      pv[bid] = b.v;
      pi[bid] = b.i;
    }
    if (last_block3(counter, nblk)) {
      ArgMax r{-1.0, 0x7fffffffffffffffLL};
      const int tid = threadIdx.y * blockDim.x + threadIdx.x;
      for (int q = tid; q < nblk; q += block_threads()) r = am_better(r, ArgMax{pv[q], pi[q]});
      r = block_argmax2d(r, shv, shi);
      if (tid == 0) {
        res->fmax = r.v;
        res->kidx = r.i;
        *counter = 0u;
      }
    }
  }
};

// parallel, fixed-order final sum of per-block partials by the last block
// (thread t sums partials t, t + MNT, ...; then the block tree) -- the same
// order on every run for a given grid
__device__ __forceinline__ double sum_partials(const double* part, int nblk, double* sh) {
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  double a = 0.0;
  for (int q = tid; q < nblk; q += block_threads()) a += part[q];
  a = warp_sum(a);
  const int lane = tid & 31, w = tid >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = a;
  __syncthreads();
  double s = 0.0;
  if (tid == 0)
    for (int q = 0; q < block_threads() / 32; ++q) s += sh[q];
  return s;  // valid on thread 0
}
__device__ __forceinline__ double block_sum2d(double v, double* sh) {
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  v = warp_sum(v);
  const int lane = tid & 31, w = tid >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (tid == 0)
    for (int q = 0; q < block_threads() / 32; ++q) s += sh[q];
  return s;  // valid on thread 0
}

// PCG K7: Ap = a p - dt F(p) for the staged p; partial (W p, Ap) -> alpha.
// ADIAG: the optional mass diagonal a of (a - dt J) is a staged operand.
template <bool ADIAG>
struct EpiMatvecT {
  static constexpr int NOPS = ADIAG ? 1 : 0;
  static constexpr bool NEEDS_W = true;
  const double* adiag;
  double* Ap;
  double dt;
  double* part;  // PlaneRed slot array of (p, Ap)_W
  double acc = 0.0;
  __host__ __device__ __forceinline__ const double* opnd(int) const { return adiag; }
  __device__ __forceinline__ void operator()(int, const GridDev&, int, int, int, int64_t o, double f, double pv, bool,
                                             const double* ov, double W) {
    const double ap = (ADIAG ? ov[0] * pv : pv) - dt * f;
    Ap[o] = ap;
    acc += (W * pv) * ap;
  }
  __device__ __forceinline__ void plane_end(int tf) {
    slot_flush(acc, part, march_slot(tf));
    acc = 0.0;
  }
  __device__ __forceinline__ void finish(const GridDev&) {}
};

// PCG K7 with the search-direction update fused in (TMA march, one rank, no
// mass diagonal, point Jacobi): the march stages r, p_old, dinv and forms
// p = r dinv + beta p_old in shared memory (tma_march.cuh form_p, the
// p-update kernel's expression), so the iteration skips k_pcg_pupdatev and the
// p re-read: Ap = p - dt F(p), p written at the node, partial (W p, Ap)
struct EpiMatvecP {
  static constexpr int NOPS = 0;
  static constexpr bool NEEDS_W = true;
  static constexpr bool FUSEP = true;
  const double* pold;  // (TMA maps only)
  const double* dinv;
  double* P;
  double* Ap;
  double dt;
  double* part;
  const PcgDev* st;
  double acc = 0.0;
  __host__ __device__ __forceinline__ const double* opnd(int) const { return nullptr; }
  __device__ __forceinline__ void operator()(int, const GridDev&, int, int, int, int64_t o, double f, double pv, bool,
                                             const double*, double W) {
    const double ap = pv - dt * f;
    P[o] = pv;
    Ap[o] = ap;
    acc += (W * pv) * ap;
  }
  __device__ __forceinline__ void plane_end(int tf) {
    slot_flush(acc, part, march_slot(tf));
    acc = 0.0;
  }
  __device__ __forceinline__ void finish(const GridDev&) {}
};

// PCG start (the marching form of k_pcg_init): r = b - (a x - dt F(x)),
// p_old = 0, partial (W r, z) and (W b, b), z = r dinv.
// Operands: b, dinv (the stored inverse Jacobi diagonal), [a].
template <bool ADIAG>
struct EpiPcgInitT {
  static constexpr int NOPS = ADIAG ? 3 : 2;
  static constexpr bool NEEDS_W = true;
  const double* b;
  const double* dg;
  const double* adiag;
  double* r;
  double* pold;
  double dt;
  double* part1;  // PlaneRed slot arrays of (r, z)_W and (b, b)_W
  double* part2;
  double s1 = 0.0, s2 = 0.0;
  __host__ __device__ __forceinline__ const double* opnd(int q) const { return q == 0 ? b : (q == 1 ? dg : adiag); }
  __device__ __forceinline__ void operator()(int, const GridDev&, int, int, int, int64_t o, double f, double xv, bool,
                                             const double* ov, double W) {
    const double bv = ov[0];
    const double Ax = (ADIAG ? ov[2] * xv : xv) - dt * f;
    const double rv = bv - Ax;
    r[o] = rv;
    pold[o] = 0.0;
    const double z = rv * ov[1];  // ov[1] = the stored inverse Jacobi diagonal
    s1 += (W * rv) * z;
    s2 += (W * bv) * bv;
  }
  __device__ __forceinline__ void plane_end(int tf) {
    const int64_t q = march_slot(tf);
    slot_flush(s1, part1, q);
    slot_flush(s2, part2, q);
    s1 = 0.0;
    s2 = 0.0;
  }
  __device__ __forceinline__ void finish(const GridDev&) {}
};

}  // namespace pc
