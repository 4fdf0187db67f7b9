// r-marching shared-memory kernels for the 19-point aligned (Spitzer)
// operator -- the hot path of C3/C4/C5 (K3 stage, K4 F+argmax, K7 matvec).
//
// Design: a block owns a (TJ x TK) theta-phi tile (phi =
// lanes, 256-byte coalesced rows) and marches along r over a chunk of R
// planes.  Per plane it stages T (3-plane ring), b and c with a one-node halo
// in shared memory, evaluates the six corner-tetrahedron edge fluxes
// E_{a,s} of every tile node ONCE (plus one component on the halo ring), and
// finalises the previous plane, whose r-neighbour fluxes are carried in
// registers.  Every HBM byte of T, b, c is read once per plane (plus the
// thin halo), so the stage is bandwidth- not recompute-bound.
//
// Arithmetic is the oracle's (oracle/operators.py aligned_E / aligned_apply)
// expression by expression; only the evaluation schedule differs, so results
// stay bitwise identical.
#pragma once
#include "kernels.cuh"

namespace pc {

constexpr int MTK = 32;          // phi extent of a tile (lanes)
constexpr int MTY = 8;           // thread rows
constexpr int NPT = 2;           // tile nodes per thread (rows ty, ty + MTY)
constexpr int MTJ = MTY * NPT;   // theta extent of a tile
constexpr int MHJ = MTJ + 2;
constexpr int MHK = MTK + 2;
constexpr int MHP = MHJ * MHK;
constexpr int MNT = MTY * MTK;   // threads per block
constexpr int NFILL = (MHP + MNT - 1) / MNT;

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

// Oracle-order evaluation of E_{a,s} at one node from its six neighbour
// values (oracle/operators.py aligned_E).  only_a >= 0 forms just E_{only_a,
// only_s} (and only the one-sided differences it needs).
struct NodeIn {
  double Tv;
  double Tn[3][2];   // neighbour T (self if missing), s: 0 '+', 1 '-'
  double b[3];
  double c;
  double il[3][2];   // inverse one-sided edge lengths (0 if missing)
  double w01[4];     // wo01 at (row, j)
  double w2[2];      // wo2 at k
};

__device__ __forceinline__ void node_E(const NodeIn& n, int only_a, int only_s, double E[3][2]) {
  double p[3][2];
#pragma unroll
  for (int x = 0; x < 3; ++x) {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (only_a >= 0 && x == only_a && t != only_s) { p[x][t] = 0.0; continue; }
      double d = t == 0 ? (n.Tn[x][0] - n.Tv) * n.il[x][0] : (n.Tv - n.Tn[x][1]) * n.il[x][1];
      p[x][t] = n.b[x] * d;
    }
  }
  double f[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int s0 = (q >> 2) & 1, s1 = (q >> 1) & 1, s2 = q & 1;
    if (only_a >= 0) {
      const int sa = only_a == 0 ? s0 : (only_a == 1 ? s1 : s2);
      if (sa != only_s) { f[q] = 0.0; continue; }
    }
    double sv = (p[0][s0] + p[1][s1]) + p[2][s2];
    double om = (n.c * n.w01[s0 * 2 + s1]) * n.w2[s2];
    f[q] = om * sv;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (only_a >= 0 && (a != only_a || s != only_s)) continue;
      double acc = 0.0;
      bool first = true;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int sa = a == 0 ? (q >> 2) & 1 : (a == 1 ? (q >> 1) & 1 : q & 1);
        if (sa != s) continue;
        acc = first ? f[q] : acc + f[q];
        first = false;
      }
      E[a][s] = (n.b[a] * n.il[a][s]) * acc;
    }
  }
}

// ---- async copy helpers (LDGSTS) -----------------------------------------
__device__ __forceinline__ void cp_async8s(unsigned s, const double* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  cp_async8s(static_cast<unsigned>(__cvta_generic_to_shared(smem)), gmem);
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

constexpr int NROWT = 11;  // per-(row, j) tables: iL2[6], wo01[4], iVal2
constexpr int MSLOTS = 4;  // T ring: planes t-1, t, t+1 in use, t+2 in flight

struct MarchSmem {
  double T[MSLOTS][MHP];
  double b[2][3][MHP];
  double c[2][MHP];
  double rowt[3][NROWT][MHJ];  // row tables for planes (p mod 3)
  double E[2][4][MHP];         // E_{1,+}, E_{1,-}, E_{2,+}, E_{2,-} per plane parity
};

// per-thread column constants (depend on k only)
struct ColT {
  double il1[6];
  double w2[2];
  double ivg;
};
__device__ __forceinline__ void load_col(const GridDev& g, int k, ColT& c) {
#pragma unroll
  for (int q = 0; q < 6; ++q) c.il1[q] = __ldg(g.iL1[q] + k);
  c.w2[0] = __ldg(g.wo2[0] + k);
  c.w2[1] = __ldg(g.wo2[1] + k);
  c.ivg = __ldg(g.iValg + k);
}

__device__ __forceinline__ void gather(const MarchSmem& S, int sm, int sc, int sp, int bs, int rs, int h, int hj,
                                       const ColT& col, NodeIn& n) {
  n.Tv = S.T[sc][h];
  n.Tn[0][0] = S.T[sp][h];
  n.Tn[0][1] = S.T[sm][h];
  n.Tn[1][0] = S.T[sc][h + MHK < MHP ? h + MHK : h];  // ring rows never use the off-tile side
  n.Tn[1][1] = S.T[sc][h >= MHK ? h - MHK : h];
  n.Tn[2][0] = S.T[sc][h + 1];
  n.Tn[2][1] = S.T[sc][h - 1];
  n.b[0] = S.b[bs][0][h];
  n.b[1] = S.b[bs][1][h];
  n.b[2] = S.b[bs][2][h];
  n.c = S.c[bs][h];
#pragma unroll
  for (int q = 0; q < 6; ++q) n.il[q >> 1][q & 1] = S.rowt[rs][q][hj] * col.il1[q];
#pragma unroll
  for (int q = 0; q < 4; ++q) n.w01[q] = S.rowt[rs][6 + q][hj];
  n.w2[0] = col.w2[0];
  n.w2[1] = col.w2[1];
}

// Epilogue contract (per tile node n of the thread):
//   epi.prefetch(n, o)                 early in the step (operands of plane t-1)
//   epi(n, g, i, j, k, o, F, uc, pin)   uc = input value at the node
//   epi.finish(g)                       block reduction, if any
template <class Val, class Epi>
__global__ void __launch_bounds__(MNT, 2) k_aligned_march(GridDev g, AlignedOp op, Val val, Epi epi, int R) {
  extern __shared__ __align__(16) unsigned char march_smem[];
  MarchSmem& S = *reinterpret_cast<MarchSmem*>(march_smem);
  if (val.skip()) return;
  val.init();
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * MTK + tx;
  const int k0 = blockIdx.x * MTK, j0 = blockIdx.y * MTJ, i0 = blockIdx.z * R;
  const int iend = min(i0 + R, g.n0);
  const int kg = k0 + tx;

  // smem fill slots of this thread (tile + halo, wrapped / clamped in-plane)
  int foff[NFILL];  // in-plane offsets (plane < 2^31 elements)
#pragma unroll
  for (int q = 0; q < NFILL; ++q) {
    const int e = tid + q * MNT;
    const int hj = e / MHK, hk = e - hj * MHK;
    bool oj, ok;
    const int jj = map_j(g, j0 - 1 + hj, oj), kk = map_k(g, k0 - 1 + hk, ok);
    foff[q] = e < MHP ? jj * g.n2 + kk : -1;
  }
  // row-table slot of this thread: tid < NROWT * MHJ
  const bool rton = tid < NROWT * MHJ;
  const int rtab = tid / MHJ, rhj = tid - (tid / MHJ) * MHJ;
  bool rok;
  const int rjj = map_j(g, j0 - 1 + rhj, rok);
  const double* rbase = !rton ? nullptr : (rtab < 6 ? g.iL2[rtab] : (rtab < 10 ? g.wo01[rtab - 6] : g.iVal2));

  bool oko;
  const int km = map_k(g, kg, oko);
  ColT col;
  load_col(g, km, col);
  const bool pin_k = (g.pin_lo2 && kg == 0) || (g.pin_hi2 && kg == g.n2 - 1);

  // ring assignment: j-rings (tid < 2 MTK) and k-rings (next 2 MTJ threads)
  int ra = -1, rs_ = 0, rhj_ = 0, rhk_ = 0;
  if (tid < 2 * MTK) {
    ra = 1;
    rs_ = tid < MTK ? 0 : 1;
    rhk_ = 1 + (tid % MTK);
    rhj_ = rs_ == 0 ? 0 : MTJ + 1;
  } else if (tid < 2 * MTK + 2 * MTJ) {
    const int q = tid - 2 * MTK;
    ra = 2;
    rs_ = q < MTJ ? 0 : 1;
    rhj_ = 1 + (q % MTJ);
    rhk_ = rs_ == 0 ? 0 : MTK + 1;
  }
  bool rjo = false, rko = false;
  if (ra >= 0) {
    map_j(g, j0 - 1 + rhj_, rjo);
  }
  const int rk = ra >= 0 ? map_k(g, k0 - 1 + rhk_, rko) : 0;
  const bool ring_on = ra >= 0 && rjo && rko &&
                       ((ra == 1) ? (k0 - 1 + rhk_ < g.n2) : (j0 - 1 + rhj_ < g.n1));
  const int rh = rhj_ * MHK + rhk_;

  auto issue_T = [&](int slot, int p) {
    const PlaneMap pm = plane_map(g, p);
    const int64_t base = (int64_t)pm.mem * g.plane;
#pragma unroll
    for (int q = 0; q < NFILL; ++q)
      if (foff[q] >= 0) val.stage(&S.T[slot][tid + q * MNT], base + foff[q], pm.mem);
  };
  auto issue_bc = [&](int slot, int p) {
    const PlaneMap pm = plane_map(g, p);
    const int64_t base = (int64_t)pm.mem * g.plane;
#pragma unroll
    for (int q = 0; q < NFILL; ++q)
      if (foff[q] >= 0) {
        const int e = tid + q * MNT;
        const int64_t o = base + foff[q];
        cp_async8(&S.b[slot][0][e], op.b[0] + o);
        cp_async8(&S.b[slot][1][e], op.b[1] + o);
        cp_async8(&S.b[slot][2][e], op.b[2] + o);
        cp_async8(&S.c[slot][e], op.c + o);
      }
  };
  auto issue_rows = [&](int slot, int p) {
    if (rton) {
      const PlaneMap pm = plane_map(g, p);
      cp_async8(&S.rowt[slot][rtab][rhj], rbase + row2(g, pm.row, rjj));
    }
  };

  // own nodes
  int jn[NPT], hn[NPT];
  bool inside[NPT], own_ok[NPT], pin_j[NPT];
#pragma unroll
  for (int n = 0; n < NPT; ++n) {
    jn[n] = j0 + ty + n * MTY;
    hn[n] = (ty + n * MTY + 1) * MHK + (tx + 1);
    inside[n] = jn[n] < g.n1 && kg < g.n2;
    bool ojo;
    map_j(g, jn[n], ojo);
    own_ok[n] = ojo && oko;
    pin_j[n] = (g.pin_lo1 && jn[n] == 0) || (g.pin_hi1 && jn[n] == g.n1 - 1);
  }

  // ---- prologue: T(i0-1), T(i0), T(i0+1); b/c and rows of i0-1 and i0
  issue_T(0, i0 - 1);
  issue_T(1, i0);
  issue_T(2, i0 + 1);
  issue_bc((i0 - 1) & 1, i0 - 1);
  issue_rows(2, i0 - 1);
  issue_bc(i0 & 1, i0);
  issue_rows(0, i0);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  double E0p[NPT];     // E_{0,+} at plane t-2 (relative to the finalised plane t-1)
  double Eprev[NPT][3][2];
  {
    const PlaneMap pm = plane_map(g, i0 - 1);
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      E0p[n] = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) Eprev[n][a][0] = Eprev[n][a][1] = 0.0;
      if (pm.exists && inside[n]) {
        NodeIn in;
        gather(S, 0, 0, 1, (i0 - 1) & 1, 2, hn[n], ty + n * MTY + 1, col, in);
        double E[3][2];
        node_E(in, 0, 0, E);
        E0p[n] = E[0][0];
      }
    }
  }
  __syncthreads();  // b/c slot of i0-1 and row slot 2 are refilled by step i0

  int s_m = 0, s_c = 1, s_p = 2, s_n = 3;  // T slots of planes t-1, t, t+1, t+2
  int r_c = 0, r_p = 2;                    // row-table slots of planes t, t-1
  for (int t = i0; t <= iend; ++t) {
    const int bsl = t & 1;  // b/c slot of plane t
    const int r_n = 3 - r_c - r_p;
    // ---- async prefetch of the next planes (overlaps the compute below)
    if (t + 2 <= iend) issue_T(s_n, t + 2);
    if (t + 1 <= iend) {
      issue_bc(bsl ^ 1, t + 1);
      issue_rows(r_n, t + 1);
    }
    cp_async_commit();

    const PlaneMap pm = plane_map(g, t);
    const bool last = (t == iend);
    const int par = t & 1, pp = par ^ 1;
    const int tf = t - 1;
    const int ig = tf + g.i0g;
    const bool pin_i = (g.pin_lo0 && ig == 0) || (g.pin_hi0 && ig == g.n0g - 1);
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      const int64_t of = off3(g, tf, jn[n], kg);
      const bool fin = t > i0 && inside[n];
      if (fin) epi.prefetch(n, of);
      double Ec[3][2] = {{0, 0}, {0, 0}, {0, 0}};
      if (pm.exists && own_ok[n]) {
        NodeIn in;
        gather(S, s_m, s_c, s_p, bsl, r_c, hn[n], ty + n * MTY + 1, col, in);
        node_E(in, last ? 0 : -1, 1, Ec);  // last plane: only E_{0,-} is consumed
      }
      if (!last) {
        S.E[par][0][hn[n]] = Ec[1][0];
        S.E[par][1][hn[n]] = Ec[1][1];
        S.E[par][2][hn[n]] = Ec[2][0];
        S.E[par][3][hn[n]] = Ec[2][1];
      }
      // ---- finalise plane t-1 of this node (its in-plane neighbours' fluxes
      // were published before the previous barrier)
      if (fin) {
        const int h = hn[n];
        const double E1pm = S.E[pp][0][h - MHK], E1mp = S.E[pp][1][h + MHK];
        const double E2pm = S.E[pp][2][h - 1], E2mp = S.E[pp][3][h + 1];
        double G = (E0p[n] - Eprev[n][0][0]) + (Eprev[n][0][1] - Ec[0][1]);
        G = G + ((E1pm - Eprev[n][1][0]) + (Eprev[n][1][1] - E1mp));
        G = G + ((E2pm - Eprev[n][2][0]) + (Eprev[n][2][1] - E2mp));
        const double iv = S.rowt[r_p][10][ty + n * MTY + 1] * col.ivg;
        double f = ((0.0 - G) * iv) * op.pref;
        if (op.rho) f = f / __ldg(op.rho + of);
        const bool pin = pin_i || pin_j[n] || pin_k;
        if (pin) f = 0.0;
        epi(n, g, tf, jn[n], kg, of, f, S.T[s_m][h], pin);
      }
      if (t > i0) E0p[n] = Eprev[n][0][0];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        Eprev[n][a][0] = Ec[a][0];
        Eprev[n][a][1] = Ec[a][1];
      }
    }
    // ---- halo ring of plane t: one flux component per ring node
    if (!last && ra >= 0) {
      double Ev = 0.0;
      if (ring_on && pm.exists) {
        ColT rcol;
        if (ra == 2) load_col(g, rk, rcol);
        else rcol = col;
        NodeIn in;
        gather(S, s_m, s_c, s_p, bsl, r_c, rh, rhj_, rcol, in);
        double E[3][2];
        node_E(in, ra, rs_, E);
        Ev = E[ra][rs_];
      }
      S.E[par][(ra - 1) * 2 + rs_][rh] = Ev;
    }
    if (last) break;
    {
      const int tmp = s_m;
      s_m = s_c;
      s_c = s_p;
      s_p = s_n;
      s_n = tmp;
      r_p = r_c;
      r_c = r_n;
    }
    cp_async_wait_all();
    __syncthreads();
  }
  epi.finish(g);
}

// PCG K7 value provider: p = z + beta p_old, z = r / (a + dt dg), with beta
// read from the device-side PCG state (set by the previous K8)
struct PValDev {
  const double* r;
  const double* pold;
  const double* dg;
  const double* adiag;
  double dt;
  const PcgDev* st;
  double beta;
  __device__ __forceinline__ bool skip() const { return st->done != 0; }  // solve finished
  __device__ __forceinline__ void init() { beta = st->beta; }
  __device__ __forceinline__ void stage(double* dst, int64_t o, int) const { *dst = (*this)(0, o, 0, 0, 0); }
  __device__ __forceinline__ double operator()(int, int64_t o, int, int, int) const {
    double dvec = (adiag ? __ldg(adiag + o) : 1.0) + dt * __ldg(dg + o);
    double z = __ldg(r + o) / dvec;
    return z + beta * __ldg(pold + o);
  }
};

// ---- epilogues ----------------------------------------------------------
struct EpiStore {  // F = op(u)
  double* F;
  __device__ __forceinline__ void prefetch(int, int64_t) {}
  __device__ __forceinline__ void operator()(int, const GridDev&, int, int, int, int64_t o, double f, double, bool) {
    F[o] = f;
  }
  __device__ __forceinline__ void finish(const GridDev&) {}
};

struct EpiStage {  // fused RKL2/RKG2 stage
  const double* um2;
  const double* u0;
  const double* y0;
  double* out;
  StageCoef sc;
  int stage;
  int* bad;
  double pa0[NPT], pm2[NPT], py0[NPT];
  __device__ __forceinline__ void prefetch(int n, int64_t o) {
    pa0[n] = __ldg(u0 + o);
    pm2[n] = __ldg(um2 + o);
    py0[n] = __ldg(y0 + o);
  }
  __device__ __forceinline__ void operator()(int n, const GridDev&, int, int, int, int64_t o, double f, double um1,
                                             bool pin) {
    const double a0 = pa0[n];
    double v = ((((sc.mu * um1) + (sc.nu * pm2[n])) + (sc.kap * a0)) + (sc.mtdt * f)) + (sc.gtdt * py0[n]);
    v = pin ? a0 : v;
    out[o] = v;
    if (!isfinite(v)) atomicMin(bad, stage);
  }
  __device__ __forceinline__ void finish(const GridDev&) {}
};

struct EpiArgmax {  // y0 = F(u0) with the |F| argmax (PTL)
  double* F;
  double* pv;
  long long* pi;
  unsigned int* counter;
  ArgRes* res;
  ArgMax best;
  __device__ __forceinline__ void prefetch(int, int64_t) {}
  __device__ __forceinline__ void operator()(int, const GridDev& g, int i, int j, int k, int64_t o, double f, double,
                                             bool) {
    F[o] = f;
    best = am_better(best, ArgMax{fabs(f), aos_index(g, i, j, k, 0, 1)});
  }
  __device__ __forceinline__ void finish(const GridDev&) {
    __shared__ double shv[MNT / 32];
    __shared__ long long shi[MNT / 32];
    const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int nblk = gridDim.x * gridDim.y * gridDim.z;
    ArgMax b = block_argmax2(best, shv, shi);
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      pv[bid] = b.v;
      pi[bid] = b.i;
    }
    if (last_block3(counter, nblk)) {
      ArgMax r{-1.0, 0x7fffffffffffffffLL};
      const int tid = threadIdx.y * blockDim.x + threadIdx.x;
      for (int q = tid; q < nblk; q += MNT) r = am_better(r, ArgMax{pv[q], pi[q]});
      r = block_argmax2(r, shv, shi);
      if (tid == 0) {
        res->fmax = r.v;
        res->kidx = r.i;
        *counter = 0u;
      }
    }
  }

  __device__ static ArgMax block_argmax2(ArgMax a, double* shv, long long* shi) {
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
      if (lane < MNT / 32) {
        r.v = shv[lane];
        r.i = shi[lane];
      }
      r = warp_argmax(r);
    }
    __syncthreads();
    return r;
  }
  __device__ static bool last_block3(unsigned int* counter, int nblk) {
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
};

struct EpiMatvec {  // PCG K7: p_new = (loaded value), Ap = a p - dt F(p); (W p, Ap)
  double* pnew;
  double* Ap;
  const double* adiag;
  double dt;
  double* p1;
  unsigned int* counter;
  PcgDev* st;
  AlignedOp op;
  double acc;
  __device__ __forceinline__ void prefetch(int, int64_t) {}
  __device__ __forceinline__ void operator()(int, const GridDev& g, int i, int j, int k, int64_t o, double f,
                                             double pv, bool) {
    const double ap = (adiag ? __ldg(adiag + o) * pv : pv) - dt * f;
    pnew[o] = pv;
    Ap[o] = ap;
    acc += (op.weight(g, i, j, k) * pv) * ap;
  }
  __device__ __forceinline__ void finish(const GridDev&) {
    __shared__ double sh[MNT / 32];
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int nblk = gridDim.x * gridDim.y * gridDim.z;
    double v = warp_sum(acc);
    const int lane = tid & 31, w = tid >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int q = 0; q < MNT / 32; ++q) s += sh[q];
      p1[bid] = s;
    }
    if (EpiArgmax::last_block3(counter, nblk)) {
      if (tid == 0) {
        double a = 0.0;
        for (int q = 0; q < nblk; ++q) a += p1[q];
        st->pAp = a;
        if (st->rz != 0.0) {
          if (!(a > 0.0)) {
            st->status = isnan(a) ? 3 : 2;
            st->done = 1;
          } else {
            st->alpha = st->rz / a;
          }
        } else {
          st->alpha = 0.0;
        }
        *counter = 0u;
      }
    }
  }
};

}  // namespace pc
