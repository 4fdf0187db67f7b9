// Generic kernels over an operator (ScalarOp / AlignedOp):
//   k_apply            F = op(u)
//   k_apply_argmax     y0 = F(u0) fused with the |F| argmax of the PTL (K4)
//   k_stage1           u1 = u0 + mut1*dt*y0                      (stage 1)
//   k_stage            fused RKL2/RKG2 stage k >= 2 (K1/K2/K3)
//   k_ptl_pairs        Eq. 5 pair tests at the argmax (K5)
//   k_ptl_all          audit mode: every pair (check_all_points)
//   k_bound            Gershgorin row bound (max) + Jacobi diagonal (K6)
//   k_pcg_*            Jacobi-PCG (K7/K8) with device-side convergence state
//   k_aos_to_soa / k_soa_to_aos   Field layout conversion
#pragma once
#include "ops.cuh"

namespace pc {

struct Fld {
  double* p[3];
};
struct CFld {
  const double* p[3];
};

struct ArgRes {  // device result of the F-argmax reduction and the PTL
  double fmax;
  long long kidx;
  double ptl;
  int limited;
  int pad;
};

__device__ __forceinline__ long long aos_index(const GridDev& g, int i, int j, int k, int c, int ncomp) {
  return (((long long)(i + g.i0g) * g.n1 + j) * n2glob(g) + kglob(g, k)) * ncomp + c;
}

template <class Op>
__global__ void __launch_bounds__(kThreads) k_apply(GridDev g, Op op, CFld u, Fld F) {
  PlainVal val{{u.p[0], u.p[1], u.p[2]}};
  PC_FOR_NODES(g, i, j, k) {
    double out[3];
    op.F(g, val, i, j, k, out);
    const int64_t o = off3(g, i, j, k);
    for (int q = 0; q < op.ncomp; ++q) F.p[q][o] = out[q];
  }
}

template <class Op>
__global__ void __launch_bounds__(kThreads) k_apply_argmax(GridDev g, Op op, CFld u, Fld F, double* pv,
                                                           long long* pi, unsigned int* counter,
                                                           ArgRes* res) {
  __shared__ double shv[kThreads / 32];
  __shared__ long long shi[kThreads / 32];
  PlainVal val{{u.p[0], u.p[1], u.p[2]}};
  ArgMax best{-1.0, 0x7fffffffffffffffLL};
  PC_FOR_NODES(g, i, j, k) {
    double out[3];
    op.F(g, val, i, j, k, out);
    const int64_t o = off3(g, i, j, k);
    for (int q = 0; q < op.ncomp; ++q) {
      F.p[q][o] = out[q];
      ArgMax cand{fabs(out[q]), aos_index(g, i, j, k, q, op.ncomp)};
      best = am_better(best, cand);
    }
  }
  best = block_argmax<kThreads>(best, shv, shi);
  if (threadIdx.x == 0) {
    pv[blockIdx.x] = best.v;
    pi[blockIdx.x] = best.i;
  }
  if (last_block(counter)) {
    ArgMax b{-1.0, 0x7fffffffffffffffLL};
    for (int t = threadIdx.x; t < (int)gridDim.x; t += blockDim.x) b = am_better(b, ArgMax{pv[t], pi[t]});
    b = block_argmax<kThreads>(b, shv, shi);
    if (threadIdx.x == 0) {
      res->fmax = b.v;
      res->kidx = b.i;
      *counter = 0u;
    }
  }
}

// argmax of |F| over a given field (pc_ptl with a caller-supplied F)
__global__ void __launch_bounds__(kThreads) k_argmax(GridDev g, int ncomp, CFld F, double* pv, long long* pi,
                                                     unsigned int* counter, ArgRes* res) {
  __shared__ double shv[kThreads / 32];
  __shared__ long long shi[kThreads / 32];
  ArgMax best{-1.0, 0x7fffffffffffffffLL};
  PC_FOR_NODES(g, i, j, k) {
    const int64_t o = off3(g, i, j, k);
    for (int q = 0; q < ncomp; ++q) best = am_better(best, ArgMax{fabs(F.p[q][o]), aos_index(g, i, j, k, q, ncomp)});
  }
  best = block_argmax<kThreads>(best, shv, shi);
  if (threadIdx.x == 0) {
    pv[blockIdx.x] = best.v;
    pi[blockIdx.x] = best.i;
  }
  if (last_block(counter)) {
    ArgMax b{-1.0, 0x7fffffffffffffffLL};
    for (int t = threadIdx.x; t < (int)gridDim.x; t += blockDim.x) b = am_better(b, ArgMax{pv[t], pi[t]});
    b = block_argmax<kThreads>(b, shv, shi);
    if (threadIdx.x == 0) {
      res->fmax = b.v;
      res->kidx = b.i;
      *counter = 0u;
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_stage1(GridDev g, int ncomp, CFld u0, CFld y0, Fld out,
                                                     double mtdt, int* bad) {
  PC_FOR_NODES(g, i, j, k) {
    const int64_t o = off3(g, i, j, k);
    const bool pin = pinned(g, i, j, k);
    for (int q = 0; q < ncomp; ++q) {
      double a = __ldg(u0.p[q] + o);
      double v = pin ? a : a + mtdt * __ldg(y0.p[q] + o);
      out.p[q][o] = v;
      if (!isfinite(v)) atomicMin(bad, 1);
    }
  }
}

struct StageCoef {
  double mu, nu, kap, mtdt, gtdt;
};

template <class Op>
__global__ void __launch_bounds__(kThreads) k_stage(GridDev g, Op op, CFld um1, CFld um2, CFld u0, CFld y0,
                                                    Fld out, StageCoef sc, int stage, int* bad) {
  PlainVal val{{um1.p[0], um1.p[1], um1.p[2]}};
  PC_FOR_NODES(g, i, j, k) {
    double Fk[3];
    op.F(g, val, i, j, k, Fk);
    const int64_t o = off3(g, i, j, k);
    const bool pin = pinned(g, i, j, k);
    for (int q = 0; q < op.ncomp; ++q) {
      double a0 = __ldg(u0.p[q] + o);
      double v = ((((sc.mu * __ldg(um1.p[q] + o)) + (sc.nu * __ldg(um2.p[q] + o))) + (sc.kap * a0)) +
                  (sc.mtdt * Fk[q])) + (sc.gtdt * __ldg(y0.p[q] + o));
      v = pin ? a0 : v;
      out.p[q][o] = v;
      if (!isfinite(v)) atomicMin(bad, stage);
    }
  }
}

// PTL pair tests at k (single block); neighbours = existing orthogonal nodes.
__global__ void k_ptl_pairs(GridDev g, int ncomp, CFld u, CFld F, double eps_rel, ArgRes* res) {
  const long long kid = res->kidx;
  const double thr = eps_rel * res->fmax;
  const long long pt = kid / ncomp;
  const int n2x = n2glob(g);
  const int kgl = (int)(pt % n2x);
  const int kk = g.phis ? kgl - g.k0g + 1 : kgl;  // local column (phi-slabs)
  const long long t2 = pt / n2x;
  const int kj = (int)(t2 % g.n1);
  const int ki = (int)(t2 / g.n1) - g.i0g;
  double best = INFINITY;
  const int t = threadIdx.x;
  // slabs: only the owner of k evaluates the pairs
  const bool owner = ki >= 0 && ki < g.n0 && (!g.phis || (kk >= 1 && kk <= g.n2 - 2));
  if (owner && t < 6 * ncomp) {
    const int dirn = t / ncomp, q = t % ncomp;
    const int a = dirn / 2, d = (dirn & 1) ? 1 : -1;
    bool ok;
    const int co[3] = {ki, kj, kk};
    int x = nbax(g, a, co[a], d, ok);
    if (ok) {
      int ni = a == 0 ? x : ki, nj = a == 1 ? x : kj, nk = a == 2 ? x : kk;
      const int64_t ok0 = off3(g, ki, kj, kk), on = off3(g, ni, nj, nk);
      double du = u.p[q][ok0] - u.p[q][on];
      double dF = F.p[q][ok0] - F.p[q][on];
      if (du != 0.0 && fabs(dF) > thr && du * dF < 0.0) best = -du / dF;
    }
  }
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_down_sync(0xffffffffu, best, o));
  if (t == 0) {
    res->ptl = best;
    res->limited = isfinite(best) ? 1 : 0;
  }
}

// audit mode: all (node, node + e_a) pairs; candidates are > 0 so their bit
// patterns order like the values (atomicMin on the raw bits).
__global__ void __launch_bounds__(kThreads) k_ptl_all(GridDev g, int ncomp, CFld u, CFld F, double eps_rel,
                                                      const ArgRes* res, unsigned long long* minbits) {
  const double thr = eps_rel * res->fmax;
  double best = INFINITY;
  PC_FOR_NODES(g, i, j, k) {
    if (g.phis && (k == 0 || k == g.n2 - 1)) continue;  // pairs start at owned nodes (each pair once)
    const int64_t o = off3(g, i, j, k);
    const int co[3] = {i, j, k};
    for (int a = 0; a < 3; ++a) {
      bool ok;
      int x = nbax(g, a, co[a], 1, ok);
      if (!ok) continue;
      int ni = a == 0 ? x : i, nj = a == 1 ? x : j, nk = a == 2 ? x : k;
      const int64_t on = off3(g, ni, nj, nk);
      for (int q = 0; q < ncomp; ++q) {
        double du = u.p[q][o] - u.p[q][on];
        double dF = F.p[q][o] - F.p[q][on];
        if (du != 0.0 && fabs(dF) > thr && du * dF < 0.0) best = fmin(best, -du / dF);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_down_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && isfinite(best)) atomicMin(minbits, (unsigned long long)__double_as_longlong(best));
}

template <class Op>
__global__ void __launch_bounds__(kThreads) k_bound(GridDev g, Op op, double* diag, double* pv,
                                                    unsigned int* counter, double* out_max) {
  __shared__ double sh[kThreads / 32];
  double m = 0.0;
  PC_FOR_NODES(g, i, j, k) {
    double lam[3], dg;
    op.bound(g, i, j, k, lam, dg);
    for (int q = 0; q < op.ncomp; ++q) m = fmax(m, lam[q]);
    if (diag) diag[off3(g, i, j, k)] = dg;
  }
  m = block_max<kThreads>(m, sh);
  if (threadIdx.x == 0) pv[blockIdx.x] = m;
  if (last_block(counter)) {
    double b = 0.0;
    for (int t = threadIdx.x; t < (int)gridDim.x; t += blockDim.x) b = fmax(b, pv[t]);
    b = block_max<kThreads>(b, sh);
    if (threadIdx.x == 0) {
      *out_max = b;
      *counter = 0u;
    }
  }
}

// flag = 1 if some rho(i, j, k) != rho(i, 0, 0) (the density is not radial)
__global__ void __launch_bounds__(kThreads) k_radial_check(GridDev g, const double* rho, int* flag) {
  PC_FOR_NODES(g, i, j, k) {
    if (g.phis && (k == 0 || k == g.n2 - 1)) continue;  // (ghost columns may not be exchanged yet)
    const double a = __ldg(rho + off3(g, i, j, k)), b = __ldg(rho + (int64_t)i * g.plane + g.phis);
    if (!(a == b)) atomicExch(flag, 1);
  }
}

// number of owned nodes x components failing a domain test (pc_field_count):
// 0: !(x > 0), 1: !(x >= 0), 2: !isfinite(x); NaN fails every test
__global__ void __launch_bounds__(kThreads) k_count_fail(GridDev g, CFld f, int ncomp, int test, double* count) {
  double n = 0.0;
  PC_FOR_NODES(g, i, j, k) {
    if (g.phis && (k == 0 || k == g.n2 - 1)) continue;  // owned nodes only (ghost columns: the neighbours')
    const int64_t o = off3(g, i, j, k);
    for (int q = 0; q < ncomp; ++q) {
      const double x = __ldg(f.p[q] + o);
      const bool bad = test == 0 ? !(x > 0.0) : test == 1 ? !(x >= 0.0) : !isfinite(x);
      n += bad ? 1.0 : 0.0;
    }
  }
  n = warp_sum(n);
  if ((threadIdx.x & 31) == 0 && n != 0.0) atomicAdd(count, n);
}

// beta_a = b_a * sqrt(c), c = kfc[i] * ((T0f * T0f) * sqrt(T0f)), T0f = max(T0, T_floor)
// (oracle aligned_coefficient + aligned_beta); bad if T0 <= 0
__global__ void __launch_bounds__(kThreads) k_aligned_beta(GridDev g, const double* T0, const double* kfc,
                                                           double Tfloor, CFld b, Fld beta, int* bad) {
  PC_FOR_NODES(g, i, j, k) {
    const int64_t o = off3(g, i, j, k);
    double t = T0[o];
    if (!(t > 0.0)) atomicMin(bad, 1);
    double tf = fmax(t, Tfloor);
    const double c = kfc[i] * ((tf * tf) * sqrt(tf));
    const double sc = sqrt(c);
    beta.p[0][o] = b.p[0][o] * sc;
    beta.p[1][o] = b.p[1][o] * sc;
    beta.p[2][o] = b.p[2][o] * sc;
  }
}

// ---------------------------------------------------------------- PCG
struct PcgDev {
  double rz;     // (r, z)_W of the current residual
  double alpha;
  double beta;
  double bn;     // ||b||_W
  double rel;    // last relative residual
  double pAp;
  int it;        // completed iterations
  int done;      // 1 = stop (converged or error)
  int status;    // 0 ok, 1 converged, 2 indefinite, 3 diverged
  int split;     // multi-rank: reductions stop at the local sums red[] (allreduced, then k_pcg_fin)
  double red[2];
};

__device__ __forceinline__ void pcg_fin_init(PcgDev* st, double rz, double bb) {
  st->rz = rz;
  st->bn = sqrt(bb);
  st->beta = 0.0;
  st->alpha = 0.0;
  st->it = 0;
  st->done = 0;
  st->status = 0;
  st->rel = INFINITY;
}
__device__ __forceinline__ void pcg_fin_update(PcgDev* st, double rr, double rzn, double tol, int it) {
  st->it = it;
  if (!isfinite(rr)) {
    st->status = 3;
    st->done = 1;
  } else {
    double rn = sqrt(rr);
    double rel = st->bn > 0.0 ? rn / st->bn : (rn == 0.0 ? 0.0 : INFINITY);
    st->rel = rel;
    if (rel <= tol) {
      st->status = 1;
      st->done = 1;
    } else {
      st->beta = st->rz != 0.0 ? rzn / st->rz : 0.0;
      st->rz = rzn;
    }
  }
}

// line-preconditioned PCG: the update decides convergence from (r, r)_W
// alone; beta and (r, z)_W follow from the line solve (pcg_fin_rz)
__device__ __forceinline__ void pcg_fin_rr(PcgDev* st, double rr, double tol, int it) {
  st->it = it;
  if (!isfinite(rr)) {
    st->status = 3;
    st->done = 1;
  } else {
    double rn = sqrt(rr);
    double rel = st->bn > 0.0 ? rn / st->bn : (rn == 0.0 ? 0.0 : INFINITY);
    st->rel = rel;
    if (rel <= tol) {
      st->status = 1;
      st->done = 1;
    }
  }
}
__device__ __forceinline__ void pcg_fin_rz(PcgDev* st, double rzn) {
  st->beta = st->rz != 0.0 ? rzn / st->rz : 0.0;
  st->rz = rzn;
}

// alpha from (p, Ap)_W; breakdown / NaN stop the solve
__device__ __forceinline__ void pcg_alpha(PcgDev* st, double pAp) {
  st->pAp = pAp;
  if (st->rz != 0.0) {
    if (!(pAp > 0.0)) {
      st->status = isnan(pAp) ? 3 : 2;
      st->done = 1;
    } else {
      st->alpha = st->rz / pAp;
    }
  } else {
    st->alpha = 0.0;
  }
}

// out[i] = 0 - pref / rho[i] (aligned operator: the per-plane scale of a radial density)
// out[i] = 1 / rho[i] (the vector march's per-plane reciprocal of a radial density)
__global__ void k_recip(const double* rho, int n, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = 1.0 / rho[i];
}
__global__ void k_neg_scale(const double* rho, int n, double pref, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = 0.0 - (pref / rho[i]);
}

// ---- GPU-count-invariant PCG reductions
// Every PCG inner product is summed in three fixed stages: (1) per slot --
// one (r, theta) row for the row-per-warp kernels, one warp of one
// (theta, phi) tile for the marching kernels (lane sums in a fixed shuffle
// tree); (2) per axis-0 plane over its slots in a fixed order
// (k_plane_sums); (3) over the GLOBAL planes 0 .. n0g-1 in a fixed order
// (plane_finish).  No stage depends on how the planes are split into
// r-slabs, so 1, 2, ..., 8 GPUs form bitwise the same sums and the same PCG
// iteration counts.  On several ranks stage 3 runs after an allreduce of the
// per-plane vector, whose every entry has exactly one non-zero contribution
// (its owner's), so the allreduce is exact.
struct PlaneRed {
  double* slot[2];  // [n0_local][S] slot partials of the (up to two) sums
  int S;            // slots per plane
  double* vec;      // [2][n0g] per-plane sums; entries of other ranks' planes stay 0
  int n0g, i0g;
};
__device__ __forceinline__ void slot_flush(double s, double* part, int64_t slot) {
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[slot] = s;
}
// fixed-order sum of n values by one block of kThreads (valid in thread 0)
__device__ __forceinline__ double sum_fixed(const double* v, int n, double* sh) {
  double a = 0.0;
  for (int q = threadIdx.x; q < n; q += kThreads) a += v[q];
  return block_sum<kThreads>(a, sh);
}
enum { PR_INIT = 0, PR_MATVEC = 1, PR_UPDATE = 2, PR_UPDATE_RR = 3 };
// stage 3 + the PCG scalar recurrences: mode PR_INIT (r, z)_W, (b, b)_W
// (keep: leave both in st->red for the r-line solve), PR_MATVEC (p, Ap)_W,
// PR_UPDATE (r, r)_W, (r, z)_W, PR_UPDATE_RR (r, r)_W only (r-line)
__device__ __forceinline__ void plane_finish(PcgDev* st, const double* vec, int n0g, int mode, int keep,
                                             double tol, int it, double* sh) {
  const double a = sum_fixed(vec, n0g, sh);
  const double b = (mode == PR_INIT || mode == PR_UPDATE) ? sum_fixed(vec + n0g, n0g, sh) : 0.0;
  if (threadIdx.x == 0) {
    if (mode == PR_INIT) {
      if (keep) {
        st->red[0] = a;
        st->red[1] = b;
      } else {
        pcg_fin_init(st, a, b);
      }
    } else if (mode == PR_MATVEC) {
      pcg_alpha(st, a);
    } else if (mode == PR_UPDATE) {
      pcg_fin_update(st, a, b, tol, it);
    } else {
      pcg_fin_rr(st, a, tol, it);
    }
  }
}
// stage 2 (one block per local plane) and, on one rank, stage 3 in the last block
__global__ void __launch_bounds__(kThreads) k_plane_sums(PlaneRed pr, int nsum, int mode, int finish, int keep,
                                                         double tol, int it, unsigned int* counter, PcgDev* st) {
  __shared__ double sh[kThreads / 32];
  if (mode != PR_INIT && st->done) return;
  const int i = blockIdx.x;
  for (int q = 0; q < nsum; ++q) {
    const double a = sum_fixed(pr.slot[q] + (int64_t)i * pr.S, pr.S, sh);
    if (threadIdx.x == 0) pr.vec[(int64_t)q * pr.n0g + pr.i0g + i] = a;
  }
  if (!finish) return;
  if (last_block(counter)) {
    plane_finish(st, pr.vec, pr.n0g, mode, keep, tol, it, sh);
    if (threadIdx.x == 0) *counter = 0u;
  }
}

// the stored inverse Jacobi diagonal of a solve ("stored
// inverse diagonal"): dinv = 1 / (a + dt d), once per PCG solve
__global__ void __launch_bounds__(kThreads) k_pcg_dinv(GridDev g, const double* dg, const double* adiag, double dt,
                                                       double* dinv) {
  PC_FOR_NODES(g, i, j, k) {
    const int64_t o = off3(g, i, j, k);
    dinv[o] = 1.0 / ((adiag ? __ldg(adiag + o) : 1.0) + dt * __ldg(dg + o));
  }
}

// p = z + beta p_old, z = r dinv: the search-direction update of the aligned
// PCG, ahead of the marching matvec (which then stages p like any T)
__global__ void __launch_bounds__(kThreads) k_pcg_pupdate(GridDev g, const double* r, const double* pold,
                                                          double* pnew, const double* dinv, const PcgDev* st) {
  if (st->done) return;
  const double beta = st->beta;
  PC_FOR_NODES(g, i, j, k) {
    const int64_t o = off3(g, i, j, k);
    const double z = __ldg(r + o) * __ldg(dinv + o);
    pnew[o] = z + beta * __ldg(pold + o);
  }
}

// k_pcg_pupdate with 128-bit accesses (n2 even): U phi pairs per lane
template <int U = 4, int MINB = 2>
__global__ void __launch_bounds__(kThreads, MINB) k_pcg_pupdatev(GridDev g, const double* __restrict__ r,
                                                           const double* __restrict__ pold, double* __restrict__ pnew,
                                                           const double* __restrict__ dinv, const PcgDev* st) {
  if (st->done) return;
  const double beta = st->beta;
  const int lane = threadIdx.x & 31;
  const int nrows = g.n0 * g.n1;
  for (int row = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); row < nrows; row += gridDim.x * (kThreads / 32)) {
    const int64_t base = (int64_t)(row / g.n1) * g.plane + (int64_t)(row % g.n1) * g.n2;
    for (int k0 = 2 * lane; k0 < g.n2; k0 += 64 * U) {
      double2 rv[U], pv[U], dv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t o = base + k0 + 64 * u;
        if (k0 + 64 * u < g.n2) {
          rv[u] = __ldg(reinterpret_cast<const double2*>(r + o));
          pv[u] = __ldg(reinterpret_cast<const double2*>(pold + o));
          dv[u] = __ldg(reinterpret_cast<const double2*>(dinv + o));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t o = base + k0 + 64 * u;
        if (k0 + 64 * u < g.n2) {
          const double z0 = rv[u].x * dv[u].x, z1 = rv[u].y * dv[u].y;
          *reinterpret_cast<double2*>(pnew + o) = make_double2(z0 + beta * pv[u].x, z1 + beta * pv[u].y);
        }
      }
    }
  }
}

// K8 for one-component operators (the aligned PCG): x += alpha p,
// r -= alpha Ap, partial (W r, r), (W r, z), z = r / (a + dt d).  One warp per
// (r, theta) row (the row weight Val2 read once), four phi nodes per lane in
// flight (all loads issued before the arithmetic), parallel fixed-order final
// sum in the last block.
template <bool RHO, bool ADIAG, bool LINE = false>
__global__ void __launch_bounds__(kThreads, 3) k_pcg_update1(GridDev g, double* __restrict__ x, double* __restrict__ r,
                                                          const double* __restrict__ p,
                                                          const double* __restrict__ Ap,
                                                          const double* __restrict__ dinv,  // the stored inverse Jacobi diagonal
                                                          const double* __restrict__ adiag,
                                                          const double* __restrict__ rho, double dt, double tol,
                                                          int it, PlaneRed pr, PcgDev* st) {
  if (st->done) return;
  const double alpha = st->alpha;
  const int lane = threadIdx.x & 31;
  const int nrows = g.n0 * g.n1;
  for (int row = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); row < nrows; row += gridDim.x * (kThreads / 32)) {
    const int i = row / g.n1, j = row - i * g.n1;
    const double V2 = __ldg(g.Val2 + row2(g, i, j));
    const int64_t base = (int64_t)i * g.plane + (int64_t)j * g.n2;
    double s1 = 0.0, s2 = 0.0;
    for (int k0 = lane; k0 < g.n2; k0 += 128) {
      double xv[4], pv[4], rv[4], av[4], dv[4], wv[4], mv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + 32 * u;
        if (k < g.n2) {
          const int64_t o = base + k;
          xv[u] = x[o];
          pv[u] = __ldg(p + o);
          rv[u] = r[o];
          av[u] = __ldg(Ap + o);
          dv[u] = LINE ? 0.0 : __ldg(dinv + o);
          wv[u] = __ldg(g.Valg + k);
          mv[u] = ADIAG ? __ldg(adiag + o) : 1.0;
          if (RHO) wv[u] = __ldg(rho + o) * (V2 * wv[u]);
          else wv[u] = V2 * wv[u];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + 32 * u;
        if (k < g.n2) {
          const int64_t o = base + k;
          x[o] = xv[u] + alpha * pv[u];
          const double rn = rv[u] - alpha * av[u];
          r[o] = rn;
          s1 += (wv[u] * rn) * rn;
          if (!LINE) s2 += (wv[u] * rn) * (rn * dv[u]);  // dv = the stored inverse diagonal
        }
      }
    }
    slot_flush(s1, pr.slot[0], row);
    if (!LINE) slot_flush(s2, pr.slot[1], row);
  }
}

// k_pcg_update1 with 128-bit accesses: n2 even, each lane owns U phi pairs
// (k, k+1), (k+64, k+65), ... -- half the load/store instructions per node.  Same per-node expressions; the per-thread partial sums
// take the nodes in a different order (the final sum stays fixed-order).
template <bool RHO, bool ADIAG, bool LINE = false, int U = 2>
__global__ void __launch_bounds__(kThreads, U == 1 ? 4 : 2) k_pcg_update1v(GridDev g, double* __restrict__ x, double* __restrict__ r,
                                                           const double* __restrict__ p,
                                                           const double* __restrict__ Ap,
                                                           const double* __restrict__ dinv,  // the stored inverse Jacobi diagonal
                                                           const double* __restrict__ adiag,
                                                           const double* __restrict__ rho, double dt, double tol,
                                                           int it, PlaneRed pr, PcgDev* st) {
  if (st->done) return;
  const double alpha = st->alpha;
  const int lane = threadIdx.x & 31;
  const int nrows = g.n0 * g.n1;
  for (int row = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); row < nrows; row += gridDim.x * (kThreads / 32)) {
    const int i = row / g.n1, j = row - i * g.n1;
    const double V2 = __ldg(g.Val2 + row2(g, i, j));
    const int64_t base = (int64_t)i * g.plane + (int64_t)j * g.n2;
    double s1 = 0.0, s2 = 0.0;
    for (int k0 = 2 * lane; k0 < g.n2; k0 += 64 * U) {
      double2 xv[U], pv[U], rv[U], av[U], dv[U], mv[U], rh[U];
      double wv[U][2];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + 64 * u;
        if (k < g.n2) {
          const int64_t o = base + k;
          xv[u] = *reinterpret_cast<const double2*>(x + o);
          pv[u] = __ldg(reinterpret_cast<const double2*>(p + o));
          rv[u] = *reinterpret_cast<const double2*>(r + o);
          av[u] = __ldg(reinterpret_cast<const double2*>(Ap + o));
          dv[u] = LINE ? make_double2(0.0, 0.0) : __ldg(reinterpret_cast<const double2*>(dinv + o));
          mv[u] = ADIAG ? __ldg(reinterpret_cast<const double2*>(adiag + o)) : make_double2(1.0, 1.0);
          rh[u] = RHO ? __ldg(reinterpret_cast<const double2*>(rho + o)) : make_double2(1.0, 1.0);
          wv[u][0] = __ldg(g.Valg + k);
          wv[u][1] = __ldg(g.Valg + k + 1);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + 64 * u;
        if (k < g.n2) {
          const int64_t o = base + k;
          const double xa[2] = {xv[u].x, xv[u].y}, pa[2] = {pv[u].x, pv[u].y}, ra[2] = {rv[u].x, rv[u].y};
          const double aa[2] = {av[u].x, av[u].y}, da[2] = {dv[u].x, dv[u].y}, ma[2] = {mv[u].x, mv[u].y};
          const double ha[2] = {rh[u].x, rh[u].y};
          double xn[2], rn[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double w = RHO ? ha[e] * (V2 * wv[u][e]) : V2 * wv[u][e];
            xn[e] = xa[e] + alpha * pa[e];
            rn[e] = ra[e] - alpha * aa[e];
            s1 += (w * rn[e]) * rn[e];
            if (!LINE) s2 += (w * rn[e]) * (rn[e] * da[e]);  // da = the stored inverse diagonal
          }
          *reinterpret_cast<double2*>(x + o) = make_double2(xn[0], xn[1]);
          *reinterpret_cast<double2*>(r + o) = make_double2(rn[0], rn[1]);
        }
      }
    }
    slot_flush(s1, pr.slot[0], row);
    if (!LINE) slot_flush(s2, pr.slot[1], row);
  }
}

// ---- r-line preconditioner (PC2 substitute; oracle/operators.py line_factor,
// line_solve): one thread per (theta, phi) line, sequential in r, coalesced
// across the lines of a warp (phi fastest)

// -J_{i,i-1}, -J_{i,i+1} of the frozen aligned operator
template <class Op>
__global__ void __launch_bounds__(kThreads) k_line_coef(GridDev g, Op op, double* jl, double* ju) {
  PC_FOR_NODES(g, i, j, k) {
    double a, b;
    op.line_coefs(g, i, j, k, a, b);
    const int64_t o = off3(g, i, j, k);
    jl[o] = a;
    ju[o] = b;
  }
}

// Thomas factorisation of M = a + dt d, off-diagonals dt jl / dt ju
__global__ void __launch_bounds__(kThreads) k_line_factor(GridDev g, const double* __restrict__ dg,
                                                          const double* __restrict__ jl,
                                                          const double* __restrict__ ju,
                                                          const double* __restrict__ adiag, double dt,
                                                          double* __restrict__ inv, double* __restrict__ cp) {
  const int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= g.plane) return;
  double cprev = 0.0;
  for (int i = 0; i < g.n0; ++i) {
    const int64_t o = (int64_t)i * g.plane + line;
    const double m = (adiag ? __ldg(adiag + o) : 1.0) + dt * __ldg(dg + o);
    const double den = i == 0 ? m : m - (dt * __ldg(jl + o)) * cprev;
    const double iv = 1.0 / den;
    const double c = (dt * __ldg(ju + o)) * iv;
    inv[o] = iv;
    cp[o] = c;
    cprev = c;
  }
}

// z = M^{-1} r, partial (W r, z); mode 0: start of the solve (fin_init with
// ||b||^2 kept in st->red[1]), mode 1: an iteration (beta, rz)
template <class Op>
__global__ void __launch_bounds__(kThreads) k_line_solve(GridDev g, Op op, const double* __restrict__ r,
                                                         const double* __restrict__ jl,
                                                         const double* __restrict__ inv,
                                                         const double* __restrict__ cp, double dt,
                                                         double* __restrict__ z, int mode, double* p1,
                                                         unsigned int* counter, PcgDev* st) {
  __shared__ double sh[kThreads / 32];
  if (mode == 1 && st->done) return;
  const int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  if (line < g.plane) {
    const int j = (int)(line / g.n2), k = (int)(line - (int64_t)j * g.n2);
    double zp = 0.0;
    for (int i = 0; i < g.n0; ++i) {
      const int64_t o = (int64_t)i * g.plane + line;
      zp = i == 0 ? __ldg(r + o) * __ldg(inv + o) : (__ldg(r + o) - (dt * __ldg(jl + o)) * zp) * __ldg(inv + o);
      z[o] = zp;
    }
    double zn = zp;  // z_{n0-1} = z'_{n0-1}
    acc = (op.weight(g, g.n0 - 1, j, k) * __ldg(r + (int64_t)(g.n0 - 1) * g.plane + line)) * zn;
    for (int i = g.n0 - 2; i >= 0; --i) {
      const int64_t o = (int64_t)i * g.plane + line;
      zn = z[o] - __ldg(cp + o) * zn;
      z[o] = zn;
      acc += (op.weight(g, i, j, k) * __ldg(r + o)) * zn;
    }
  }
  acc = block_sum<kThreads>(acc, sh);
  if (threadIdx.x == 0) p1[blockIdx.x] = acc;
  if (last_block(counter)) {
    double a = 0.0;
    for (int t = threadIdx.x; t < (int)gridDim.x; t += kThreads) a += p1[t];
    const double rz = block_sum<kThreads>(a, sh);
    if (threadIdx.x == 0) {
      if (mode == 0) pcg_fin_init(st, rz, st->red[1]);
      else pcg_fin_rz(st, rz);
      *counter = 0u;
    }
  }
}

// p = z + beta p_old (line-preconditioned PCG)
__global__ void __launch_bounds__(kThreads) k_pcg_pupdate_z(GridDev g, const double* z, const double* pold,
                                                            double* pnew, const PcgDev* st) {
  if (st->done) return;
  const double beta = st->beta;
  PC_FOR_NODES(g, i, j, k) {
    const int64_t o = off3(g, i, j, k);
    pnew[o] = __ldg(z + o) + beta * __ldg(pold + o);
  }
}

// multi-rank finish of a PCG reduction: stage 3 over the allreduced
// per-plane vector (the same plane_finish as one rank's k_plane_sums)
__global__ void __launch_bounds__(kThreads) k_pcg_fin(PcgDev* st, const double* vec, int n0g, int mode, int keep,
                                                      double tol, int it) {
  __shared__ double sh[kThreads / 32];
  if (mode != PR_INIT && st->done) return;
  plane_finish(st, vec, n0g, mode, keep, tol, it, sh);
}

// global |F| argmax from the per-rank (value, index) pairs (lowest index on ties)
__global__ void k_argmax_combine(const double* gath, int nranks, ArgRes* res) {
  if (threadIdx.x != 0) return;
  ArgMax b{-1.0, 0x7fffffffffffffffLL};
  for (int r = 0; r < nranks; ++r) {
    long long idx;
    memcpy(&idx, gath + 2 * r + 1, sizeof idx);
    b = am_better(b, ArgMax{gath[2 * r], idx});
  }
  res->fmax = b.v;
  res->kidx = b.i;
}

// p = z + beta * p_old with z = r / (a + dt*dg)   (recomputed at neighbours)
struct PVal {
  const double* r[3];
  const double* pold[3];
  const double* dinv;  // the stored inverse Jacobi diagonal
  double beta;
  __device__ __forceinline__ double operator()(int c, int64_t o, int, int, int) const {
    double z = __ldg(r[c] + o) * __ldg(dinv + o);
    return z + beta * __ldg(pold[c] + o);
  }
};

// init: r = b - A x, z = r/d, p_old = 0; partials (r,z)_W and (b,b)_W
// (row-per-warp loops with one slot partial per (r, theta) row: the
// GPU-count-invariant reduction order, see PlaneRed)
#define PC_FOR_ROWS(g, row, i, j)                                                                          \
  for (int row = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5), i = 0, j = 0;                        \
       row < (g).n0 * (g).n1 && ((i = row / (g).n1), (j = row - i * (g).n1), true);                      \
       row += gridDim.x * (kThreads / 32))
template <class Op>
__global__ void __launch_bounds__(kThreads) k_pcg_init(GridDev g, Op op, CFld b, CFld x, Fld r, Fld pold,
                                                       const double* dinv, const double* adiag, double dt,
                                                       PlaneRed pr, PcgDev* st) {
  PlainVal val{{x.p[0], x.p[1], x.p[2]}};
  PC_FOR_ROWS(g, row, i, j) {
  double s1 = 0.0, s2 = 0.0;
  for (int k = threadIdx.x & 31; k < g.n2; k += 32) {
    double Fx[3];
    op.F(g, val, i, j, k, Fx);
    const int64_t o = off3(g, i, j, k);
    const double W = op.weight(g, i, j, k);
    const double di = dinv[o];
    for (int q = 0; q < op.ncomp; ++q) {
      double xv = x.p[q][o];
      double Ax = (adiag ? adiag[o] * xv : xv) - dt * Fx[q];
      double rv = b.p[q][o] - Ax;
      r.p[q][o] = rv;
      pold.p[q][o] = 0.0;
      double z = rv * di;
      s1 += (W * rv) * z;
      double bv = b.p[q][o];
      s2 += (W * bv) * bv;
    }
  }
  slot_flush(s1, pr.slot[0], row);
  slot_flush(s2, pr.slot[1], row);
  }
}

// K7: p_new = z + beta p_old; Ap = a p_new - dt F(p_new); partial (p, Ap)_W
template <class Op>
__global__ void __launch_bounds__(kThreads) k_pcg_matvec(GridDev g, Op op, CFld r, CFld pold, Fld pnew, Fld Ap,
                                                         const double* dinv, const double* adiag, double dt,
                                                         PlaneRed pr, PcgDev* st) {
  if (st->done) return;
  PVal val{{r.p[0], r.p[1], r.p[2]}, {pold.p[0], pold.p[1], pold.p[2]}, dinv, st->beta};
  PC_FOR_ROWS(g, row, i, j) {
  double s1 = 0.0;
  for (int k = threadIdx.x & 31; k < g.n2; k += 32) {
    double Fp[3];
    op.F(g, val, i, j, k, Fp);
    const int64_t o = off3(g, i, j, k);
    const double W = op.weight(g, i, j, k);
    for (int q = 0; q < op.ncomp; ++q) {
      double pv = val(q, o, i, j, k);
      double ap = (adiag ? adiag[o] * pv : pv) - dt * Fp[q];
      pnew.p[q][o] = pv;
      Ap.p[q][o] = ap;
      s1 += (W * pv) * ap;
    }
  }
  slot_flush(s1, pr.slot[0], row);
  }
}

// K8: x += alpha p; r -= alpha Ap; partials (r,r)_W and (r,z)_W
template <class Op>
__global__ void __launch_bounds__(kThreads) k_pcg_update(GridDev g, Op op, Fld x, Fld r, CFld p, CFld Ap,
                                                         const double* dinv, const double* adiag, double dt,
                                                         PlaneRed pr, PcgDev* st) {
  if (st->done) return;
  const double alpha = st->alpha;
  PC_FOR_ROWS(g, row, i, j) {
  double s1 = 0.0, s2 = 0.0;
  for (int k = threadIdx.x & 31; k < g.n2; k += 32) {
    const int64_t o = off3(g, i, j, k);
    const double W = op.weight(g, i, j, k);
    const double di = dinv[o];
    for (int q = 0; q < op.ncomp; ++q) {
      x.p[q][o] = x.p[q][o] + alpha * p.p[q][o];
      double rv = r.p[q][o] - alpha * Ap.p[q][o];
      r.p[q][o] = rv;
      s1 += (W * rv) * rv;
      s2 += (W * rv) * (rv * di);
    }
  }
  slot_flush(s1, pr.slot[0], row);
  slot_flush(s2, pr.slot[1], row);
  }
}

// ---------------------------------------------------------------- layout
// host AoS chunk [planes][n1][n2][ncomp] -> SoA field planes [p0, p0+np)
// host node c of the chunk (host rows: the owned columns only) -> field offset
__device__ __forceinline__ int64_t host_node_off(const GridDev& g, int p0, int64_t c) {
  if (!g.phis) return (int64_t)p0 * g.plane + c;
  const int hn2 = g.n2 - 2;
  const int64_t row = c / hn2;
  return (int64_t)p0 * g.plane + row * g.n2 + (c - row * hn2) + 1;
}
__global__ void __launch_bounds__(kThreads) k_aos_to_soa(GridDev g, int ncomp, const double* src, Fld dst,
                                                         int p0, int np) {
  const int64_t n = (int64_t)np * g.n1 * (g.n2 - 2 * g.phis);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = host_node_off(g, p0, c);
    for (int q = 0; q < ncomp; ++q) dst.p[q][o] = src[c * ncomp + q];
  }
}
__global__ void __launch_bounds__(kThreads) k_soa_to_aos(GridDev g, int ncomp, CFld src, double* dst,
                                                         int p0, int np) {
  const int64_t n = (int64_t)np * g.n1 * (g.n2 - 2 * g.phis);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = host_node_off(g, p0, c);
    for (int q = 0; q < ncomp; ++q) dst[c * ncomp + q] = src.p[q][o];
  }
}
// phi-slab ghost columns: pack the owned edge columns 1 (to the lower
// neighbour) and n2-2 (to the upper) of every (plane, row) into
// buf[q][side][n0 x n1], and unpack the received ones into columns 0 / n2-1
__global__ void __launch_bounds__(kThreads) k_phi_pack(GridDev g, int ncomp, CFld f, double* buf) {
  const int64_t rows = (int64_t)g.n0 * g.n1;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = r * g.n2;
    for (int q = 0; q < ncomp; ++q) {
      buf[(2 * q) * rows + r] = f.p[q][o + 1];
      buf[(2 * q + 1) * rows + r] = f.p[q][o + g.n2 - 2];
    }
  }
}
__global__ void __launch_bounds__(kThreads) k_phi_unpack(GridDev g, int ncomp, const double* buf, Fld f) {
  const int64_t rows = (int64_t)g.n0 * g.n1;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = r * g.n2;
    for (int q = 0; q < ncomp; ++q) {
      f.p[q][o] = buf[(2 * q) * rows + r];                 // from the lower neighbour's column n2-2
      f.p[q][o + g.n2 - 1] = buf[(2 * q + 1) * rows + r];  // from the upper neighbour's column 1
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_fill(double* p, int64_t n, double v) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) p[c] = v;
}

}  // namespace pc
