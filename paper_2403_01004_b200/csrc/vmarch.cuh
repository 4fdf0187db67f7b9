// Vector-viscosity 7-point march (K2v of DESIGN.md §4): the 3-component
// spherical operator (frame rotations on the theta / phi faces) for the two
// launches every PTL cycle of C2 / C5v runs -- y0 = F(u0) + argmax, and the
// fused stages 1 + 2 -- written around what bounds this stencil (issue and
// latency at ~150 fp64 instructions per node), not around staging:
//
//  * the thread that owns node (j0 + ty, k0 + tx) keeps its stencil input
//    in registers along r (planes t-1, t, t+1: the r-faces read no shared
//    memory), and only the in-plane neighbours come from the staged tile;
//  * every array-plane lands by TMA (a 32 x 10 main box and two 2 x 10 phi
//    strips that wrap across the periodic seam, as in SMaps) on a per-slot
//    full mbarrier, four slots deep (plane t+3 is issued while t is
//    computed): no per-thread copy issue, no per-element address arithmetic
//    in the plane loop; four issuer warps split the boxes;
//  * F1 (stages 1 + 2): u1 = u0 + mt1 y0 is formed once per staged element,
//    in place over the staged u0 -- the owner forms its node (kept in a
//    register, its u0 carried for the epilogue), 80 threads form the tile's
//    theta / phi halo;
//  * one __syncthreads per plane; the refill of the slot freed by plane t-1
//    is issued right after it.
//
// Every face term, the rotation products and the epilogue are formed exactly
// as k_scalar_march forms them (same operands, same order), so the result is
// bitwise k_scalar_march's and the oracle's (oracle/operators.py
// scalar_apply).  Used on spherical-type grids whose phi is
// periodic in whole 32-column tiles, theta not periodic, no theta / phi
// pinning (PC_NO_VMARCH=1 keeps k_scalar_march).
#pragma once
#include "smarch.cuh"

namespace pc {

// cp.async.bulk.tensor / mbarrier arm issued by one elected lane of a warp
// that executes the call convergently (operands warp-uniform: no per-lane
// waterfall around the uniform-register operands of UTMALDG)
__device__ __forceinline__ void tma3_elect(double* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                           unsigned long long* bar) {
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\n"
      "@P cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n}" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_elect(unsigned long long* bar, unsigned bytes) {
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\n"
      "@P mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

constexpr int VSL = 4;  // staged-plane slots: t (read), t+1 (formed this iteration), t+2, t+3 (in flight)

constexpr int VOSL = 3;  // epilogue-operand slots (plain stage): t (read), t+1, t+2 (in flight)

template <bool F1, int DM, int NOP>
struct VMarchSmem {
  static constexpr int NA = F1 ? 6 : 3;          // u0[3] (+ y0[3]) -- the staged stencil sources
  static constexpr int ND = DM != 0 ? 1 : 0;     // D / rho source
  double A[VSL][NA + ND][SXA];                   // TMA layout (main box + padded strips); F1: u0 -> u1 in place
  double O[NOP ? VOSL : 1][NOP ? NOP : 1][NOP ? SNT : 16];  // plain stage: u0, u_{k-2}, y0 at the tile nodes
  double2 M[4][SMJ][5];                          // frame rotations of the tile rows (as k_scalar_march)
  double rowt[3][SROWT][SHJ];                    // row tables of planes t-1, t, t+1
  unsigned long long full[VSL];
  unsigned long long ofull[VOSL];
};

template <int DM, class Epi>
__global__ void __launch_bounds__(SNT, 2) k_vec_march(GridDev g, ScalarOp op, Epi epi, int R, int zsel,
                                                      const int* skip, const __grid_constant__ SMaps maps) {
  constexpr bool F1 = fuse1_of<Epi>::value;
  constexpr bool HASD = DM != 0;
  constexpr int NOP = F1 ? 0 : Epi::NOPS;  // operand boxes of the plain stage (SEpiStage: 9)
  using Sm = VMarchSmem<F1, DM, NOP>;
  constexpr int NA = Sm::NA;
  constexpr int DS = NA;  // slot of the D / rho source
  extern __shared__ __align__(128) unsigned char vmarch_smem[];
  Sm& S = *reinterpret_cast<Sm*>(vmarch_smem + ((128u - (smem_u32(vmarch_smem) & 127u)) & 127u));
  if (skip && *skip) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int tid = threadIdx.x;
  const int k0 = blockIdx.x * MTK, j0 = blockIdx.y * SMJ, i0 = chunk_of(zsel) * R;
  const int iend = min(i0 + R, g.n0);
  const int kg = k0 + tx, jg = j0 + ty;
  const int kL = k0 == 0 ? g.n2 - 2 : k0 - 2;  // phi strips (wrap across the seam)
  const int kR = k0 + MTK == g.n2 ? 0 : k0 + MTK;
  constexpr unsigned kPlaneBytes = (unsigned)(NA + Sm::ND) * kSArrBytes;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < VSL; ++s) mbar_init(&S.full[s], 1);
#pragma unroll
    for (int s = 0; s < VOSL; ++s) mbar_init(&S.ofull[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // rotation table of the tile rows (loaded once; rows beyond n1 clamp)
  for (int e = tid; e < 4 * SMJ * 10; e += SNT) {
    const int f = e / (SMJ * 10), r = (e / 10) % SMJ, q = e % 10;
    const int jr = min(j0 + r, g.n1 - 1);
    const int th = q < 2 ? q : (q < 4 ? q + 1 : (q == 4 ? 2 : (q < 9 ? q : 8)));  // 0 1 3 4 2 5 6 7 8 8
    const int src = f < 2 ? th : (q < 9 ? q : 8);
    reinterpret_cast<double*>(&S.M[f][r][0])[q] = __ldg(g.M[f] + (int64_t)jr * 9 + src);
  }
  // row tables: W2[0..2], iV2 per (plane, halo row), one cp.async each by 50 threads
  const bool rton = tid < SROWT * SHJ;
  const int rtab = tid / SHJ, rhj = tid - (tid / SHJ) * SHJ;
  bool rok;
  const int rjj = map_j(g, j0 - 1 + rhj, rok);
  const double* rbase = !rton ? g.iV2 : (rtab < 3 ? g.W2[rtab] : g.iV2);
  auto issue_rows = [&](int p, int sl) {
    if (rton) cp_async8(&S.rowt[sl][rtab][rhj], rbase + row2(g, plane_map(g, p).row, rjj));
  };
  auto aslot = [&](int p) { return (p - i0 + 1) & (VSL - 1); };
  // TMA issue: warps 4..7 each run this whole (warp-uniform operands, one
  // elected lane issues): warp 7 arms the slot's barrier and stages component
  // 0 of u0 / u (and of y0), warps 6 and 5 components 1 and 2, warp 4 the D /
  // rho source -- the issue work is spread instead of serialising one warp
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  auto issue_plane = [&](int p) {
    const int z = plane_map(g, p).mem + 1;  // (the tensors start at ghost plane -1)
    const int sl = aslot(p);
    unsigned long long* b = &S.full[sl];
    auto arr = [&](double* dst, const CUtensorMap* mm, const CUtensorMap* ms) {
      tma3_elect(dst, mm, k0, j0 - 1, z, b);
      tma3_elect(dst + SXM, ms, kL, j0 - 1, z, b);
      tma3_elect(dst + SXM + SXS, ms, kR, j0 - 1, z, b);
    };
    if (warp == 7) mbar_expect_tx_elect(b, kPlaneBytes);
#pragma unroll
    for (int c = 0; c < 3; ++c)
      if (warp == 7 - c) {
        arr(&S.A[sl][c][0], &maps.V[c], &maps.VS[c]);
        if constexpr (F1) arr(&S.A[sl][3 + c][0], &maps.Y[c], &maps.YS[c]);
      }
    if constexpr (HASD) {
      if (warp == 4) arr(&S.A[sl][DS][0], &maps.D, &maps.DS);
    }
  };
  // plain stage: the nine operand boxes (32 x 8, the tile nodes) of plane p
  // into operand slot sl, completing on ofull[sl] (warp 7 arms it)
  auto issue_ops = [&](int p, int sl) {
    if constexpr (NOP > 0) {
      unsigned long long* b = &S.ofull[sl];
      if (warp == 7) mbar_expect_tx_elect(b, (unsigned)NOP * kSOpBytes);
#pragma unroll
      for (int q = 0; q < NOP; ++q)
        if (warp == 4 + (q & 3)) tma3_elect(&S.O[sl][q][0], &maps.O[q], k0, j0, p + 1, b);
    }
  };
  const bool issuer = warp >= 4;

  const bool inside = jg < g.n1 && kg < g.n2;
  bool oko;
  const int km = map_k(g, kg, oko);
  bool okkm;
  const int kmm = nb2(g, km, -1, okkm);
  const double g10 = launder(__ldg(g.g1[0] + km)), g11 = launder(__ldg(g.g1[1] + km));
  const double g12 = launder(__ldg(g.g1[2] + km)), g12m = launder(okkm ? __ldg(g.g1[2] + kmm) : 0.0);
  const double igv = launder(__ldg(g.igv + km));
  bool okjm;
  nb1(g, jg < g.n1 ? jg : g.n1 - 1, -1, okjm);
  // staged-tile offsets (TMA layout) of the own node and its theta / phi neighbours
  const int h = (ty + 1) * MTK + tx;
  const int htm = h - MTK, htp = h + MTK;
  const int hpm = tx > 0 ? h - 1 : SXM + (ty + 1) * 2 + 1;
  const int hpp = tx < MTK - 1 ? h + 1 : SXM + SXS + (ty + 1) * 2;
  const int onode = jg * g.n2 + kg;
  // F1: the halo element this thread forms (threads 0..79): theta rows j0-1 and
  // j0+8 of the main box, then the phi strips' columns k0-1 and k0+32 of rows 1..8
  int hx = -1;
  if (F1) {
    if (tid < 2 * MTK) hx = tid < MTK ? tid : 9 * MTK + (tid - MTK);
    else if (tid < 2 * MTK + 2 * SMJ) {
      const int q = tid - 2 * MTK, r = 1 + (q & 7);
      hx = q < SMJ ? SXM + r * 2 + 1 : SXM + SXS + r * 2;
    }
  }
  // F1: u1 = pin ? u0 : u0 + mt1 y0 (k_stage1's expression) at element e of
  // slot sl, written over u0; a0 returns u0
  auto form = [&](int sl, int e, bool pn, double (&u1)[3], double (&a0)[3]) {
    if constexpr (F1) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double a = S.A[sl][c][e];
        a0[c] = a;
        u1[c] = pn ? a : a + epi.mt1 * S.A[sl][3 + c][e];
        S.A[sl][c][e] = u1[c];
      }
    }
  };
  auto plane_pin = [&](int p) {
    const int ig = plane_map(g, p).mem + g.i0g;
    return (g.pin_lo0 && ig == 0) || (g.pin_hi0 && ig == g.n0g - 1);
  };
  // own stencil input of plane p (F1: formed here, the halo too; else the staged u)
  auto own_in = [&](int p, double (&v)[3], double (&a0)[3]) {
    const int sl = aslot(p);
    if constexpr (F1) {
      const bool pn = plane_pin(p);
      if (hx >= 0) {
        double w[3], w0[3];
        form(sl, hx, pn, w, w0);
      }
      form(sl, h, pn, v, a0);
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) v[c] = S.A[sl][c][h];
    }
  };

  unsigned ph = 0u;  // one phase bit per slot
  auto wait_plane = [&](int p) {
    const int sl = aslot(p);
    mbar_wait(&S.full[sl], (ph >> sl) & 1u);
    ph ^= 1u << sl;
  };
  // ---- prologue: planes i0-1 .. i0+2 in flight, rows of i0-1 and i0
  __syncthreads();  // barriers initialised
  if (issuer) {
    issue_plane(i0 - 1);
    issue_plane(i0);
    issue_plane(i0 + 1);  // (iend >= i0 + 1)
    if (i0 + 2 <= iend) issue_plane(i0 + 2);
    issue_ops(i0, 0);
    if (i0 + 1 < iend) issue_ops(i0 + 1, 1);
  }
  int o_c = 0, o_p = 1, o_n = 2;  // operand slots of planes t, t+1, t+2
  unsigned oph = 0u;
  int r_m = 0, r_c = 1, r_p = 2;  // row-table slots of planes t-1, t, t+1
  issue_rows(i0 - 1, r_m);
  issue_rows(i0, r_c);
  cp_async_commit();
  double vm[3], vc[3], vp[3], a0c[3], a0n[3], dm = 0.0, dc = 0.0, dp = 0.0;
  wait_plane(i0 - 1);
  own_in(i0 - 1, vm, a0n);
  wait_plane(i0);
  own_in(i0, vc, a0c);
  if (HASD) {
    dm = S.A[aslot(i0 - 1)][DS][h];
    dc = S.A[aslot(i0)][DS][h];
  }
  const int jr = ty + 1;  // row-table index of the own row (halo row 0 = j0 - 1)

#pragma unroll 1
  for (int t = i0; t < iend; ++t) {
    // plane t+1: landed (issued two iterations ago); its stencil input formed
    wait_plane(t + 1);
    own_in(t + 1, vp, a0n);
    const int sc = aslot(t);
    if (HASD) dp = S.A[aslot(t + 1)][DS][h];
    cp_async_wait<0>();  // rows of plane t (issued one iteration ago)
    __syncthreads();     // u1(t+1), rows(t) visible; every thread is done with plane t-1's slots
    if (issuer && t + 3 <= iend) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_plane(t + 3);  // (into plane t-1's slot)
    }
    if (NOP > 0 && issuer && t + 2 < iend) {
      if (t + 3 > iend) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_ops(t + 2, o_n);  // (into plane t-1's operand slot)
    }
    if (t + 1 <= iend) issue_rows(t + 1, r_p);  // (its slot held plane t-2's rows)
    cp_async_commit();

    const int rs = r_c, rm = r_m;
    if (inside) {
      const bool okim = plane_map(g, t - 1).exists;
      const int ig = t + g.i0g;
      const bool pin = (g.pin_lo0 && ig == 0) || (g.pin_hi0 && ig == g.n0g - 1);
      const double Dcen = DM == 0 ? op.Dc : (DM == 1 ? dc : op.Dc * dc);
      double coef[3][2];
      coef[0][0] = okim ? S.rowt[rm][0][jr] * g10 : 0.0;
      coef[0][1] = S.rowt[rs][0][jr] * g10;
      coef[1][0] = okjm ? S.rowt[rs][1][jr - 1] * g11 : 0.0;
      coef[1][1] = S.rowt[rs][1][jr] * g11;
      coef[2][0] = okkm ? S.rowt[rs][2][jr] * g12m : 0.0;
      coef[2][1] = S.rowt[rs][2][jr] * g12;
      double nv[3][2][3], nd[3][2];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        nv[0][0][c] = vm[c];
        nv[0][1][c] = vp[c];
        nv[1][0][c] = S.A[sc][c][htm];
        nv[1][1][c] = S.A[sc][c][htp];
        nv[2][0][c] = S.A[sc][c][hpm];
        nv[2][1][c] = S.A[sc][c][hpp];
      }
      if (HASD) {
        nd[0][0] = dm;
        nd[0][1] = dp;
        nd[1][0] = S.A[sc][DS][htm];
        nd[1][1] = S.A[sc][DS][htp];
        nd[2][0] = S.A[sc][DS][hpm];
        nd[2][1] = S.A[sc][DS][hpp];
      }
      double Sx[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          double cf;
          if (HASD) {
            const double Dn = DM == 1 ? nd[a][tt] : op.Dc * nd[a][tt];
            cf = (0.5 * (Dcen + Dn)) * coef[a][tt];
          } else {
            cf = op.Dc * coef[a][tt];
          }
          const bool first = (a == 0 && tt == 0);
          if (a > 0) {
            const double2* M2 = S.M[(a == 1 ? 0 : 2) + (tt == 1 ? 0 : 1)][ty];
            const double v0 = nv[a][tt][0], v1 = nv[a][tt][1], v2 = nv[a][tt][2];
            double rv[3];
            if (a == 1) {  // theta faces rotate about e_phi (exact zeros and one, see k_scalar_march)
              const double2 r0 = M2[0], r1 = M2[1];
              rv[0] = (r0.x * v0) + (r0.y * v1);
              rv[1] = (r1.x * v0) + (r1.y * v1);
              rv[2] = v2;
            } else {
              double M[10];
#pragma unroll
              for (int q = 0; q < 5; ++q) {
                const double2 w = M2[q];
                M[2 * q] = w.x;
                M[2 * q + 1] = w.y;
              }
#pragma unroll
              for (int c = 0; c < 3; ++c) rv[c] = ((M[3 * c] * v0) + (M[3 * c + 1] * v1)) + (M[3 * c + 2] * v2);
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double term = cf * (rv[c] - vc[c]);
              Sx[c] = first ? term : Sx[c] + term;
            }
          } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double term = cf * (nv[a][tt][c] - vc[c]);
              Sx[c] = first ? term : Sx[c] + term;
            }
          }
        }
      }
      const double iv = S.rowt[rs][3][jr] * igv;
      const int64_t o = (int64_t)t * g.plane + onode;
      double f[3];
      const double irho = op.rho ? 1.0 / (DM == 2 ? dc : __ldg(op.rho + o)) : 1.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double x = Sx[c] * iv;
        if (op.rho) x = x * irho;
        f[c] = pin ? 0.0 : x;
      }
      double ov[F1 ? 6 : (NOP > 0 ? NOP : 1)];
      if constexpr (F1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          ov[2 * c] = a0c[c];
          ov[2 * c + 1] = S.A[sc][3 + c][h];
        }
      }
      if constexpr (NOP > 0) {
        mbar_wait(&S.ofull[o_c], (oph >> o_c) & 1u);
#pragma unroll
        for (int q = 0; q < NOP; ++q) ov[q] = S.O[o_c][q][tid];
      }
      epi.template apply<3>(g, t, jg, kg, o, f, vc, pin, ov);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      vm[c] = vc[c];
      vc[c] = vp[c];
      a0c[c] = a0n[c];
    }
    if (HASD) {
      dm = dc;
      dc = dp;
    }
    {  // rotate the row-table slots: t-1 <- t, t <- t+1, t+1 <- the old t-1 slot
      const int o = r_m;
      r_m = r_c;
      r_c = r_p;
      r_p = o;
    }
    if constexpr (NOP > 0) {  // operand slots: t <- t+1, t+1 <- t+2, t+2 <- the old t slot
      oph ^= 1u << o_c;
      const int o = o_c;
      o_c = o_p;
      o_p = o_n;
      o_n = o;
    }
  }
  cp_async_wait<0>();
  epi.finish(g);
}

}  // namespace pc
