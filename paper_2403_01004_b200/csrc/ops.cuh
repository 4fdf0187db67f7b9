// Operator right-hand sides F(u), Gershgorin row bounds and Jacobi diagonals.
//
// Mirrors oracle/operators.py expression by expression (see that file for the
// mathematics; SPEC.md:84-159 for the contracts):
//   ScalarOp  -- 7-point rho-weighted finite-volume diffusion, optional
//                vector metric (frame rotation)
//   AlignedOp -- 19-point corner-tetrahedron field-aligned conduction
#pragma once
#include "common.cuh"

namespace pc {

// value provider for a plain SoA field
struct PlainVal {
  const double* p[3];
  __device__ __forceinline__ bool skip() const { return false; }
  __device__ __forceinline__ void init() {}
  __device__ __forceinline__ double operator()(int c, int64_t o, int, int, int) const {
    return __ldg(p[c] + o);
  }
  // asynchronous shared-memory staging of component 0 (LDGSTS, 8 bytes)
  __device__ __forceinline__ void stage(double* dst, int64_t o, int) const {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(p[0] + o) : "memory");
  }
};

// ------------------------------------------------------------------ scalar
struct ScalarOp {
  const double* D;  // nodal nu*rho, or nullptr -> Dc (or Dc * rho with drho)
  double Dc;
  int drho;         // D = Dc * rho evaluated per node (viscosity with a density field)
  __device__ __forceinline__ bool has_field() const { return D != nullptr || drho; }
  __device__ __forceinline__ double Dat(int64_t o) const { return D ? __ldg(D + o) : Dc * __ldg(rho + o); }
  const double* rho;  // nullptr -> 1
  int ncomp;
  int vector;  // rotate 3-component spherical vectors
  // viscosity with a radial density (rho(i, j, k) == rho(i), detected at
  // freeze, one rank): rho(i) for i < n0 and 1 / rho(i) at n0 + i -- the field's
  // own values, read once per plane by the vector march (DM = 3)
  const double* rho_r = nullptr;

  // face coefficient (Dface * (W * g)) for direction (a, dir) of node (i,j,k);
  // returns false if the neighbour does not exist (coefficient exactly 0).
  __device__ __forceinline__ void nb_coord(const GridDev& g, int a, int dir, int i, int j, int k,
                                           int& ni, int& nj, int& nk, bool& ok) const {
    ni = i; nj = j; nk = k;
    if (a == 0) ni = nb0(g, i, dir, ok);
    else if (a == 1) nj = nb1(g, j, dir, ok);
    else nk = nb2(g, k, dir, ok);
  }
  __device__ __forceinline__ double wg(const GridDev& g, int a, int dir, bool ok, int i, int j, int k,
                                       int ni, int nj, int nk) const {
    if (dir > 0) {
      return __ldg(g.W2[a] + row2(g, i, j)) * __ldg(g.g1[a] + k);
    }
    if (!ok) return 0.0;
    if (a == 0) return __ldg(g.W2[0] + row2(g, ni, j)) * __ldg(g.g1[0] + k);
    if (a == 1) return __ldg(g.W2[1] + row2(g, i, nj)) * __ldg(g.g1[1] + k);
    return __ldg(g.W2[2] + row2(g, i, j)) * __ldg(g.g1[2] + nk);
  }

  template <class Val>
  __device__ __forceinline__ void F(const GridDev& g, const Val& val, int i, int j, int k,
                                    double* out) const {
    const int64_t o = off3(g, i, j, k);
    double S[3];
    double uc[3];
    for (int c = 0; c < ncomp; ++c) uc[c] = val(c, o, i, j, k);
    const double Dcen = has_field() ? Dat(o) : Dc;
    bool first = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int dir = t == 0 ? -1 : 1;
        int ni, nj, nk;
        bool ok;
        nb_coord(g, a, dir, i, j, k, ni, nj, nk, ok);
        const int64_t on = off3(g, ni, nj, nk);
        double coef = wg(g, a, dir, ok, i, j, k, ni, nj, nk);
        double cf;
        if (has_field()) {
          double Dn = Dat(on);
          cf = (0.5 * (Dcen + Dn)) * coef;
        } else {
          cf = Dc * coef;
        }
        if (vector && a > 0) {
          const double* M = g.M[(a == 1 ? 0 : 2) + (dir > 0 ? 0 : 1)] + (int64_t)j * 9;
          double v0 = val(0, on, ni, nj, nk), v1 = val(1, on, ni, nj, nk), v2 = val(2, on, ni, nj, nk);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double rv = ((__ldg(M + 3 * c) * v0) + (__ldg(M + 3 * c + 1) * v1)) + (__ldg(M + 3 * c + 2) * v2);
            double tt = cf * (rv - uc[c]);
            S[c] = first ? tt : S[c] + tt;
          }
        } else {
          for (int c = 0; c < ncomp; ++c) {
            double tt = cf * (val(c, on, ni, nj, nk) - uc[c]);
            S[c] = first ? tt : S[c] + tt;
          }
        }
        first = false;
      }
    }
    const bool pin = pinned(g, i, j, k);
    const double iv = __ldg(g.iV2 + row2(g, i, j)) * __ldg(g.igv + k);
    const double irho = rho ? 1.0 / __ldg(rho + o) : 1.0;  // (1/rho) div(...): one reciprocal per node
    for (int c = 0; c < ncomp; ++c) {
      double f = S[c] * iv;
      if (rho) f = f * irho;
      out[c] = pin ? 0.0 : f;
    }
  }

  // lam[c] = sum_j |J_ij| and dg = -J_ii (oracle scalar_gershgorin / scalar_diag)
  __device__ __forceinline__ void bound(const GridDev& g, int i, int j, int k, double* lam,
                                        double& dg) const {
    const int64_t o = off3(g, i, j, k);
    const double Dcen = has_field() ? Dat(o) : Dc;
    double L[3], Sd = 0.0;
    bool first = true;
    for (int a = 0; a < 3; ++a) {
      for (int t = 0; t < 2; ++t) {
        const int dir = t == 0 ? -1 : 1;
        int ni, nj, nk;
        bool ok;
        nb_coord(g, a, dir, i, j, k, ni, nj, nk, ok);
        double coef = wg(g, a, dir, ok, i, j, k, ni, nj, nk);
        double cf = has_field() ? (0.5 * (Dcen + Dat(off3(g, ni, nj, nk)))) * coef : Dc * coef;
        for (int c = 0; c < ncomp; ++c) {
          double R = 2.0;
          if (vector && a > 0) R = __ldg(g.Rabs[(a == 1 ? 0 : 2) + (dir > 0 ? 0 : 1)] + (int64_t)j * 3 + c);
          double tt = cf * R;
          L[c] = first ? tt : L[c] + tt;
        }
        Sd = first ? cf : Sd + cf;
        first = false;
      }
    }
    const bool pin = pinned(g, i, j, k);
    const double iv = __ldg(g.iV2 + row2(g, i, j)) * __ldg(g.igv + k);
    for (int c = 0; c < ncomp; ++c) {
      double l = L[c] * iv;
      if (rho) l = l / __ldg(rho + o);
      lam[c] = pin ? 0.0 : l;
    }
    double d = Sd * iv;
    if (rho) d = d / __ldg(rho + o);
    dg = pin ? 0.0 : d;
  }

  __device__ __forceinline__ double weight(const GridDev& g, int i, int j, int k) const {
    double V = __ldg(g.V2 + row2(g, i, j)) * __ldg(g.gv + k);
    return rho ? __ldg(rho + off3(g, i, j, k)) * V : V;
  }
};

// ------------------------------------------------------------------ aligned
// beta = sqrt(c) b (frozen per outer step, oracle aligned_beta): the operator
// streams three nodal arrays and never touches c or b.
struct AlignedOp {
  const double* beta[3];
  const double* rho;  // nullptr -> 1
  const double* rho_r = nullptr;  // rho(i) per interior plane when rho is radial (TMA march reads it per plane)
  const double* nsc_r = nullptr;  // with rho_r: the per-plane scale 0 - pref / rho(i)
  double pref;
  double npref;  // 0 - pref: the scale when there is no density
  // F = (G iv) * (0 - pref / rho): one product per node for the prefactor and
  // the density (oracle/operators.py aligned_apply; the division only where rho
  // varies per node)
  __device__ __forceinline__ double nscale(int64_t o) const {
    return rho ? 0.0 - (pref / __ldg(rho + o)) : npref;
  }
  int ncomp;  // always 1
  int tma_split = 2;  // TMA march: per-plane copies issued by 1 + tma_split warps (PC_TMA_SPLIT overrides)

  __device__ __forceinline__ double iL(const GridDev& g, int a, int s, int i, int j, int k) const {
    return __ldg(g.iL2[a * 2 + s] + row2(g, i, j)) * __ldg(g.iL1[a * 2 + s] + k);
  }
  __device__ __forceinline__ double om(const GridDev& g, int s0, int s1, int s2, int i, int j, int k) const {
    return __ldg(g.wo01[s0 * 2 + s1] + row2(g, i, j)) * __ldg(g.wo2[s2] + k);
  }

  // E_{a,s} at node (i,j,k) (oracle aligned_E); only the one-sided
  // differences the component needs are formed.  all: every component.
  template <class Val>
  __device__ __forceinline__ void Enode(const GridDev& g, const Val& val, int i, int j, int k, int only_a,
                                        int only_s, double E[3][2]) const {
    const int64_t o = off3(g, i, j, k);
    const double Tv = val(0, o, i, j, k);
    const double bv[3] = {__ldg(beta[0] + o), __ldg(beta[1] + o), __ldg(beta[2] + o)};
    const int co[3] = {i, j, k};
    double p[3][2], bil[3][2];
#pragma unroll
    for (int x = 0; x < 3; ++x) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        bil[x][t] = bv[x] * iL(g, x, t, i, j, k);
        if (only_a >= 0 && x == only_a && t != only_s) { p[x][t] = 0.0; continue; }
        bool ok;
        int nx = nbax(g, x, co[x], t == 0 ? 1 : -1, ok);
        int ni = x == 0 ? nx : i, nj = x == 1 ? nx : j, nk = x == 2 ? nx : k;
        double Tn = ok ? val(0, off3(g, ni, nj, nk), ni, nj, nk) : Tv;
        p[x][t] = bil[x][t] * (t == 0 ? (Tn - Tv) : (Tv - Tn));
      }
    }
    double f[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int s0 = (n >> 2) & 1, s1 = (n >> 1) & 1, s2 = n & 1;
      double sv = (p[0][s0] + p[1][s1]) + p[2][s2];
      f[n] = om(g, s0, s1, s2, i, j, k) * sv;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (only_a >= 0 && (a != only_a || s != only_s)) { E[a][s] = 0.0; continue; }
        double acc = 0.0;
        bool first = true;
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          const int sa = a == 0 ? (n >> 2) & 1 : (a == 1 ? (n >> 1) & 1 : n & 1);
          if (sa != s) continue;
          acc = first ? f[n] : acc + f[n];
          first = false;
        }
        E[a][s] = bil[a][s] * acc;
      }
    }
  }
  template <class Val>
  __device__ __forceinline__ double Ecomp(const GridDev& g, const Val& val, int a, int s, int i, int j,
                                          int k) const {
    double E[3][2];
    Enode(g, val, i, j, k, a, s, E);
    return E[a][s];
  }

  // G in the marching order of oracle aligned_apply
  template <class Val>
  __device__ __forceinline__ void F(const GridDev& g, const Val& val, int i, int j, int k,
                                    double* out) const {
    double E[3][2];
    Enode(g, val, i, j, k, -1, 0, E);
    const int co[3] = {i, j, k};
    double Em[3], Ep[3];  // E_{a,+}(m - e_a), E_{a,-}(m + e_a)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      bool okm, okp;
      int xm = nbax(g, a, co[a], -1, okm);
      int xp = nbax(g, a, co[a], 1, okp);
      Em[a] = okm ? Ecomp(g, val, a, 0, a == 0 ? xm : i, a == 1 ? xm : j, a == 2 ? xm : k) : 0.0;
      Ep[a] = okp ? Ecomp(g, val, a, 1, a == 0 ? xp : i, a == 1 ? xp : j, a == 2 ? xp : k) : 0.0;
    }
    const double own = ((E[0][1] - E[0][0]) + (E[1][1] - E[1][0])) + (E[2][1] - E[2][0]);
    const double nbr = (Em[1] - Ep[1]) + (Em[2] - Ep[2]);
    const double G = (Em[0] - Ep[0]) + (own + nbr);
    const int64_t o = off3(g, i, j, k);
    const double iv = __ldg(g.iVal2 + row2(g, i, j)) * __ldg(g.iValg + k);
    const double f = (G * iv) * nscale(o);
    out[0] = pinned(g, i, j, k) ? 0.0 : f;
  }

  // Hessian rows of the quadratic form (oracle aligned_hessian_rows) -> bound, diag
  __device__ __forceinline__ double q(const GridDev& g, int a, int s, int i, int j, int k, int64_t o) const {
    return (s == 0 ? 1.0 : -1.0) * (__ldg(beta[a] + o) * iL(g, a, s, i, j, k));
  }
  static __device__ __forceinline__ int face_idx(int a, int d) { return 1 + 2 * a + (d > 0 ? 1 : 0); }
  static __device__ __forceinline__ int diag_idx(int a, int da, int bb, int db) {
    int lo = a < bb ? a : bb, hi = a < bb ? bb : a;
    int dlo = a < bb ? da : db, dhi = a < bb ? db : da;
    int pair = (lo == 0 && hi == 1) ? 0 : ((lo == 0 && hi == 2) ? 1 : 2);
    return 7 + 4 * pair + 2 * (dlo > 0 ? 1 : 0) + (dhi > 0 ? 1 : 0);
  }

  // the node's Hessian row of Q (19 offsets, face_idx / diag_idx order),
  // accumulated exactly as oracle aligned_hessian_rows
  __device__ __forceinline__ void hessian_row(const GridDev& g, int i, int j, int k, double (&H)[19]) const {
#pragma unroll
    for (int n = 0; n < 19; ++n) H[n] = 0.0;
    const int64_t o = off3(g, i, j, k);
    // (A) apex tets (loops fully unrolled: H stays in registers)
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int sg[3] = {(n >> 2) & 1, (n >> 1) & 1, n & 1};
      double qa[3];
#pragma unroll
      for (int x = 0; x < 3; ++x) qa[x] = q(g, x, sg[x], i, j, k, o);
      double qs = (qa[0] + qa[1]) + qa[2];
      double w = om(g, sg[0], sg[1], sg[2], i, j, k) * 1.0;
      H[0] += (w * qs) * qs;
#pragma unroll
      for (int x = 0; x < 3; ++x) H[face_idx(x, sg[x] == 0 ? 1 : -1)] += (w * (0.0 - qs)) * qa[x];
    }
    // (B) end-point tets, v = m - sigma_a e_a
    const int co[3] = {i, j, k};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int sa = 0; sa < 2; ++sa) {
        const int d = sa == 0 ? -1 : 1;
        bool ok;
        int xv = nbax(g, a, co[a], d, ok);
        if (!ok) continue;
        const int vi = a == 0 ? xv : i, vj = a == 1 ? xv : j, vk = a == 2 ? xv : k;
        const int64_t ov = off3(g, vi, vj, vk);
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          const int sg[3] = {(n >> 2) & 1, (n >> 1) & 1, n & 1};
          if (sg[a] != sa) continue;
          double qv[3];
#pragma unroll
          for (int x = 0; x < 3; ++x) qv[x] = q(g, x, sg[x], vi, vj, vk, ov);
          double wv = om(g, sg[0], sg[1], sg[2], vi, vj, vk) * 1.0;
          double qs = (qv[0] + qv[1]) + qv[2];
          double qa = qv[a];
          H[0] += (wv * qa) * qa;
          H[face_idx(a, d)] += (wv * qa) * (0.0 - qs);
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) {
            if (bb == a) continue;
            H[diag_idx(a, d, bb, sg[bb] == 0 ? 1 : -1)] += (wv * qa) * qv[bb];
          }
        }
      }
    }
  }

  __device__ __forceinline__ void bound(const GridDev& g, int i, int j, int k, double* lam,
                                        double& dg) const {
    double H[19];
    hessian_row(g, i, j, k, H);
    const int64_t o = off3(g, i, j, k);
    double S = fabs(H[0]);
#pragma unroll
    for (int n = 1; n < 19; ++n) S = S + fabs(H[n]);
    const double iv = __ldg(g.iVal2 + row2(g, i, j)) * __ldg(g.iValg + k);
    double l = (S * iv) * pref;
    double dd = (H[0] * iv) * pref;
    if (rho) {
      l = l / __ldg(rho + o);
      dd = dd / __ldg(rho + o);
    }
    const bool pin = pinned(g, i, j, k);
    lam[0] = pin ? 0.0 : l;
    dg = pin ? 0.0 : dd;
  }

  // -J_{i,i-1}, -J_{i,i+1} (r-line preconditioner; oracle aligned_line_offdiag)
  __device__ __forceinline__ void line_coefs(const GridDev& g, int i, int j, int k, double& jl, double& ju) const {
    double H[19];
    hessian_row(g, i, j, k, H);
    const double iv = __ldg(g.iVal2 + row2(g, i, j)) * __ldg(g.iValg + k);
    double a = (H[face_idx(0, -1)] * iv) * pref;
    double b = (H[face_idx(0, 1)] * iv) * pref;
    if (rho) {
      const double rv = __ldg(rho + off3(g, i, j, k));
      a = a / rv;
      b = b / rv;
    }
    const bool pin = pinned(g, i, j, k);
    jl = pin ? 0.0 : a;
    ju = pin ? 0.0 : b;
  }

  __device__ __forceinline__ double weight(const GridDev& g, int i, int j, int k) const {
    double V = __ldg(g.Val2 + row2(g, i, j)) * __ldg(g.Valg + k);
    return rho ? __ldg(rho + off3(g, i, j, k)) * V : V;
  }
};

}  // namespace pc
