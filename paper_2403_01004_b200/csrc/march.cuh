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

constexpr int MTJ = 8;
constexpr int MTK = 32;
constexpr int MHJ = MTJ + 2;
constexpr int MHK = MTK + 2;
constexpr int MHP = MHJ * MHK;
constexpr int MNT = MTJ * MTK;

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
// values.  want[a][s] selects the components to form (others untouched).
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

// gather the inputs of node (hj, hk) of the tile from shared memory
struct MarchSmem {
  double T[3][MHP];
  double b[3][MHP];
  double c[MHP];
  double E[2][4][MHP];  // E_{1,+}, E_{1,-}, E_{2,+}, E_{2,-} per plane parity
};

__device__ __forceinline__ void gather(const GridDev& g, const MarchSmem& S, int sm, int sc, int sp, int h, int row,
                                       int jg, int kg, NodeIn& n) {
  n.Tv = S.T[sc][h];
  n.Tn[0][0] = S.T[sp][h];
  n.Tn[0][1] = S.T[sm][h];
  n.Tn[1][0] = S.T[sc][h + MHK < MHP ? h + MHK : h];  // ring rows never use the off-tile side
  n.Tn[1][1] = S.T[sc][h >= MHK ? h - MHK : h];
  n.Tn[2][0] = S.T[sc][h + 1];
  n.Tn[2][1] = S.T[sc][h - 1];
  n.b[0] = S.b[0][h];
  n.b[1] = S.b[1][h];
  n.b[2] = S.b[2][h];
  n.c = S.c[h];
  const int64_t r2 = row2(g, row, jg);
#pragma unroll
  for (int q = 0; q < 6; ++q) n.il[q >> 1][q & 1] = __ldg(g.iL2[q] + r2) * __ldg(g.iL1[q] + kg);
#pragma unroll
  for (int q = 0; q < 4; ++q) n.w01[q] = __ldg(g.wo01[q] + r2);
  n.w2[0] = __ldg(g.wo2[0] + kg);
  n.w2[1] = __ldg(g.wo2[1] + kg);
}

// Epilogue contract: epi(g, node i, j, k, offset, F, uc) where uc is the
// input value at the node (from shared memory); epi.finish(...) at the end.
template <class Val, class Epi>
__global__ void __launch_bounds__(MNT, 2) k_aligned_march(GridDev g, AlignedOp op, Val val, Epi epi, int R) {
  __shared__ MarchSmem S;
  if (val.skip()) return;
  val.init();
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * MTK + tx;
  const int k0 = blockIdx.x * MTK, j0 = blockIdx.y * MTJ, i0 = blockIdx.z * R;
  const int iend = min(i0 + R, g.n0);
  const int jg = j0 + ty, kg = k0 + tx;
  const bool inside = jg < g.n1 && kg < g.n2;
  const int hown = (ty + 1) * MHK + (tx + 1);

  // stage one field plane (tile + halo) into shared memory
  auto load_T = [&](int slot, int p) {
    PlaneMap pm = plane_map(g, p);
    for (int e = tid; e < MHP; e += MNT) {
      const int hj = e / MHK, hk = e - hj * MHK;
      bool oj, ok;
      const int jj = map_j(g, j0 - 1 + hj, oj), kk = map_k(g, k0 - 1 + hk, ok);
      S.T[slot][e] = val(0, off3(g, pm.mem, jj, kk), pm.mem, jj, kk);
    }
  };
  auto load_bc = [&](int p) {
    PlaneMap pm = plane_map(g, p);
    for (int e = tid; e < MHP; e += MNT) {
      const int hj = e / MHK, hk = e - hj * MHK;
      bool oj, ok;
      const int jj = map_j(g, j0 - 1 + hj, oj), kk = map_k(g, k0 - 1 + hk, ok);
      const int64_t o = off3(g, pm.mem, jj, kk);
      S.b[0][e] = __ldg(op.b[0] + o);
      S.b[1][e] = __ldg(op.b[1] + o);
      S.b[2][e] = __ldg(op.b[2] + o);
      S.c[e] = __ldg(op.c + o);
    }
  };

  // ---- prologue: planes i0-1, i0, i0+1 and E_{0,+}(i0-1)
  load_T(0, i0 - 1);
  load_T(1, i0);
  load_T(2, i0 + 1);
  load_bc(i0 - 1);
  __syncthreads();
  double E0p_prev2 = 0.0;  // E_{0,+} at plane t-2 (relative to the finalised plane t-1)
  {
    PlaneMap pm = plane_map(g, i0 - 1);
    if (pm.exists && inside) {
      // E_{0,+} at (i0-1): needs T(i0) at own position (slot 1) and in-plane
      // neighbours of plane i0-1 (slot 0); p[0][-] is not formed.
      NodeIn n;
      gather(g, S, 0, 0, 1, hown, pm.row, jg, kg, n);
      double E[3][2];
      node_E(n, 0, 0, E);
      E0p_prev2 = E[0][0];
    }
  }
  __syncthreads();
  load_bc(i0);
  __syncthreads();

  double Eprev[3][2] = {{0, 0}, {0, 0}, {0, 0}};
  double ucprev = 0.0;
  for (int t = i0; t <= iend; ++t) {
    const int sm = (t - i0) % 3, sc = (t - i0 + 1) % 3, sp = (t - i0 + 2) % 3;  // slot(p) = (p - i0 + 1) % 3
    const int par = t & 1;
    PlaneMap pm = plane_map(g, t);
    const bool last = (t == iend);
    double Ecur[3][2] = {{0, 0}, {0, 0}, {0, 0}};
    double uccur = 0.0;
    if (pm.exists) {
      // threads of a partial tile evaluate the (wrapped) node they map to, so
      // in-tile neighbour fluxes are right at domain edges too
      bool ojo, oko;
      const int jm = map_j(g, jg, ojo), km = map_k(g, kg, oko);
      if (ojo && oko) {
        NodeIn n;
        gather(g, S, sm, sc, sp, hown, pm.row, jm, km, n);
        uccur = n.Tv;
        node_E(n, last ? 0 : -1, 1, Ecur);  // last plane: only E_{0,-} is consumed
        if (!last) {
          S.E[par][0][hown] = Ecur[1][0];
          S.E[par][1][hown] = Ecur[1][1];
          S.E[par][2][hown] = Ecur[2][0];
          S.E[par][3][hown] = Ecur[2][1];
        }
      } else if (!last) {
        S.E[par][0][hown] = 0.0;
        S.E[par][1][hown] = 0.0;
        S.E[par][2][hown] = 0.0;
        S.E[par][3][hown] = 0.0;
      }
      if (!last) {
        // halo ring: one component per ring node
        int a = -1, s = 0, hj = 0, hk = 0;
        if (tid < 2 * MTK) {
          a = 1;
          s = tid < MTK ? 0 : 1;
          hk = 1 + (tid % MTK);
          hj = s == 0 ? 0 : MTJ + 1;
        } else if (tid < 2 * MTK + 2 * MTJ) {
          const int q = tid - 2 * MTK;
          a = 2;
          s = q < MTJ ? 0 : 1;
          hj = 1 + (q % MTJ);
          hk = s == 0 ? 0 : MTK + 1;
        }
        if (a >= 0) {
          bool oj, ok;
          const int jj = map_j(g, j0 - 1 + hj, oj), kk = map_k(g, k0 - 1 + hk, ok);
          // the ring node must exist and its tile-side neighbour must be inside
          const bool partner = (a == 1) ? (k0 - 1 + hk < g.n2) : (j0 - 1 + hj < g.n1);
          double Ev = 0.0;
          if (oj && ok && partner) {
            NodeIn n;
            gather(g, S, sm, sc, sp, hj * MHK + hk, pm.row, jj, kk, n);
            double E[3][2];
            node_E(n, a, s, E);
            Ev = E[a][s];
          }
          S.E[par][(a - 1) * 2 + s][hj * MHK + hk] = Ev;
        }
      }
    }
    __syncthreads();
    // ---- finalise plane t-1
    if (t > i0 && inside) {
      const int tf = t - 1;
      const int pp = (t - 1) & 1;
      const double E1pm = S.E[pp][0][hown - MHK], E1mp = S.E[pp][1][hown + MHK];
      const double E2pm = S.E[pp][2][hown - 1], E2mp = S.E[pp][3][hown + 1];
      double G = (E0p_prev2 - Eprev[0][0]) + (Eprev[0][1] - Ecur[0][1]);
      G = G + ((E1pm - Eprev[1][0]) + (Eprev[1][1] - E1mp));
      G = G + ((E2pm - Eprev[2][0]) + (Eprev[2][1] - E2mp));
      const int64_t o = off3(g, tf, jg, kg);
      const double iv = __ldg(g.iVal2 + row2(g, tf, jg)) * __ldg(g.iValg + kg);
      double f = ((0.0 - G) * iv) * op.pref;
      if (op.rho) f = f / __ldg(op.rho + o);
      if (pinned(g, tf, jg, kg)) f = 0.0;
      epi(g, tf, jg, kg, o, f, ucprev);
    }
    // rotate carried fluxes (E_{0,+}(i0-1) from the prologue survives step i0)
    if (t > i0) E0p_prev2 = Eprev[0][0];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      Eprev[a][0] = Ecur[a][0];
      Eprev[a][1] = Ecur[a][1];
    }
    ucprev = uccur;
    if (last) break;
    __syncthreads();  // everyone done with the slots about to be overwritten
    if (t + 2 <= iend) load_T(sm, t + 2);  // the last step never reads T(iend + 1)
    load_bc(t + 1);
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
  __device__ __forceinline__ double operator()(int, int64_t o, int, int, int) const {
    double dvec = (adiag ? __ldg(adiag + o) : 1.0) + dt * __ldg(dg + o);
    double z = __ldg(r + o) / dvec;
    return z + beta * __ldg(pold + o);
  }
};

// ---- epilogues ----------------------------------------------------------
struct EpiStore {  // F = op(u)
  double* F;
  __device__ __forceinline__ void operator()(const GridDev&, int, int, int, int64_t o, double f, double) {
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
  __device__ __forceinline__ void operator()(const GridDev& g, int i, int j, int k, int64_t o, double f,
                                             double um1) {
    const double a0 = __ldg(u0 + o);
    double v = ((((sc.mu * um1) + (sc.nu * __ldg(um2 + o))) + (sc.kap * a0)) + (sc.mtdt * f)) +
               (sc.gtdt * __ldg(y0 + o));
    v = pinned(g, i, j, k) ? a0 : v;
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
  __device__ __forceinline__ void operator()(const GridDev& g, int i, int j, int k, int64_t o, double f, double) {
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
  __device__ __forceinline__ void operator()(const GridDev& g, int i, int j, int k, int64_t o, double f,
                                             double pv) {
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
