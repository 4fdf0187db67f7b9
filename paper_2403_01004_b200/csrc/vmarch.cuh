// Vector-viscosity 7-point march (K2v of DESIGN.md §4): the 3-component
// spherical operator (frame rotations on the theta / phi faces) for the
// launches every PTL cycle of C2 / C5v runs -- y0 = F(u0) + argmax, the fused
// stages 1 + 2 and (s >= 3) the plain stage -- written around what bounds
// this stencil (issue and latency at ~150 fp64 instructions per node):
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
//  * no block-wide barrier in the plane loop: per slot a `full` mbarrier (the
//    plane's boxes and its row records landed), a `formed` one (F1: every
//    thread formed its elements of the plane; count 256) and an `empty` one
//    (every warp is done with the plane; count 8), so a warp that finished
//    early starts the next plane instead of idling at a __syncthreads, and
//    the issuer warps refill the slot of plane t-1 once `empty` says so;
//  * the per-(r, theta) metric rows (W2[0..2], iV2) arrive as one 4 x 10 box
//    of an interleaved record table per plane; the r- face coefficient is the
//    previous plane's r+ one (the same product), carried in a register;
//  * the plain stage's nine epilogue operands come as 32 x 8 boxes on a
//    three-slot ring; a radial density (C5 / C5v) is read per plane (DM 3);
//  * the F+argmax epilogue tracks only the plane and component of the
//    thread's maximum (its node is fixed).
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

constexpr int VSL = 4;    // staged-plane slots: t (read), t+1 (formed this iteration), t+2, t+3 (in flight)
constexpr int VOSL = 3;   // epilogue-operand slots (plain stage): t (read), t+1, t+2 (in flight)
constexpr int VRW = 48;   // one plane's row records [10 rows][W2[0], W2[1], W2[2], iV2], padded to 384 B
constexpr unsigned kVRowBytes = (unsigned)(SHJ * 4) * 8u;

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <bool F1, int DM, int NOP>
struct VMarchSmem {
  static constexpr int NA = F1 ? 6 : 3;          // u0[3] (+ y0[3]) -- the staged stencil sources
  static constexpr int ND = (DM == 1 || DM == 2) ? 1 : 0;  // staged D / rho source
  double A[VSL][NA + ND][SXA];                   // TMA layout (main box + padded strips); F1: u0 -> u1 in place
  double O[NOP ? VOSL : 1][NOP ? NOP : 1][NOP ? SNT : 16];  // plain stage: u0, u_{k-2}, y0 at the tile nodes
  double rowt[VSL][VRW];                         // row records of the staged planes
  double2 M[4][SMJ][5];                          // frame rotations of the tile rows (as k_scalar_march)
  unsigned long long full[VSL], formed[VSL], empty[VSL], ofull[VOSL];
};

// DM: 0 = D constant Dc, 1 = D nodal field, 2 = D = Dc * rho (a rho field),
// 3 = D = Dc * rho(i) with a radial rho read per plane from op.rho_r (not staged)
template <int DM, class Epi>
__global__ void __launch_bounds__(SNT, 2) k_vec_march(GridDev g, ScalarOp op, Epi epi, int R, int zsel,
                                                      const int* skip, const __grid_constant__ SMaps maps,
                                                      const __grid_constant__ CUtensorMap rowmap) {
  constexpr bool F1 = fuse1_of<Epi>::value;
  constexpr bool HASD = DM != 0;              // the face coefficients carry a D average
  constexpr bool SD = DM == 1 || DM == 2;     // D / rho staged per node
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
  constexpr unsigned kPlaneBytes = (unsigned)(NA + Sm::ND) * kSArrBytes + kVRowBytes;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < VSL; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.formed[s], SNT);
      mbar_init(&S.empty[s], SNT / 32);
    }
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
  // plane p's slot and the parity of that slot's barriers for p (every plane
  // i0-1 .. iend uses each barrier of its slot exactly once)
  auto slot = [&](int p) { return (p - i0 + 1) & (VSL - 1); };
  auto par = [&](int p) { return (unsigned)((p - i0 + 1) >> 2) & 1u; };
  // TMA issue: warps 4..7 each run this whole (warp-uniform operands, one
  // elected lane issues): warp 7 arms the slot's barrier and stages component
  // 0 of u0 / u (and of y0) and the row records, warps 6 and 5 components 1
  // and 2, warp 4 the D / rho source
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  auto issue_plane = [&](int p) {
    const PlaneMap pm = plane_map(g, p);
    const int z = pm.mem + 1;  // (the tensors start at ghost plane -1)
    const int sl = slot(p);
    unsigned long long* b = &S.full[sl];
    auto arr = [&](double* dst, const CUtensorMap* mm, const CUtensorMap* ms) {
      tma3_elect(dst, mm, k0, j0 - 1, z, b);
      tma3_elect(dst + SXM, ms, kL, j0 - 1, z, b);
      tma3_elect(dst + SXM + SXS, ms, kR, j0 - 1, z, b);
    };
    if (warp == 7) {
      mbar_expect_tx_elect(b, kPlaneBytes);
      tma3_elect(&S.rowt[sl][0], &rowmap, 0, j0 - 1, pm.row + 1, b);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c)
      if (warp == 7 - c) {
        arr(&S.A[sl][c][0], &maps.V[c], &maps.VS[c]);
        if constexpr (F1) arr(&S.A[sl][3 + c][0], &maps.Y[c], &maps.YS[c]);
      }
    if constexpr (SD) {
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
  const int jr = ty + 1;  // row-record index of the own row (record row 0 = j0 - 1)
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
  // plane p landed: this thread's stencil input of it (F1: formed here, the
  // halo too, then announced on `formed`; else the staged u)
  auto own_in = [&](int p, double (&v)[3], double (&a0)[3]) {
    const int sl = slot(p);
    mbar_wait(&S.full[sl], par(p));
    if constexpr (F1) {
      const bool pn = plane_pin(p);
      if (hx >= 0) {
        double w[3], w0[3];
        form(sl, hx, pn, w, w0);
      }
      form(sl, h, pn, v, a0);
      mbar_arrive(&S.formed[sl]);
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) v[c] = S.A[sl][c][h];
    }
  };
  auto release = [&](int p) {  // this warp is done with plane p's slot
    __syncwarp();
    if (tx == 0) mbar_arrive(&S.empty[slot(p)]);
  };

  // ---- prologue: planes i0-1 .. i0+2 in flight (and the operands of i0, i0+1)
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
  double vm[3], vc[3], vp[3], a0c[3], a0n[3], dm = 0.0, dc = 0.0, dp = 0.0;
  // radial rho (DM 3): rho of plane p from the table, the same value every node of it holds
  auto rho_r = [&](int p) { return __ldg(op.rho_r + plane_map(g, p).mem); };
  own_in(i0 - 1, vm, a0n);
  if (SD) dm = S.A[slot(i0 - 1)][DS][h];
  if (DM == 3) dm = rho_r(i0 - 1);
  double cr0 = S.rowt[slot(i0 - 1)][jr * 4] * g10;  // r+ face of plane i0-1 = r- face of plane i0
  release(i0 - 1);
  own_in(i0, vc, a0c);
  if (SD) dc = S.A[slot(i0)][DS][h];
  if (DM == 3) dc = rho_r(i0);

  const bool okim0 = plane_map(g, i0 - 1).exists;
  constexpr bool AM = std::is_same<Epi, SEpiArgmax>::value;
  // F+argmax: this thread's node is fixed, so only the plane and component of
  // its running maximum vary (SEpiArgmax::apply's strict >, same visiting order)
  double am_v = -1.0;
  int am_t = 0, am_c = 0;
  if constexpr (AM) am_v = epi.best.v;

#pragma unroll 1
  for (int t = i0; t < iend; ++t) {
    // refill plane t-1's slots once every warp is done with them
    const bool more = t + 3 <= iend, mops = NOP > 0 && t + 2 < iend;
    if (issuer && (more || mops)) {
      mbar_wait(&S.empty[slot(t - 1)], par(t - 1));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (more) issue_plane(t + 3);
      if (mops) issue_ops(t + 2, o_n);
    }
    // plane t+1: landed (issued two iterations ago); its stencil input formed
    own_in(t + 1, vp, a0n);
    const int sc = slot(t);
    if (SD) dp = S.A[slot(t + 1)][DS][h];
    if (DM == 3) dp = rho_r(t + 1);
    if constexpr (F1) mbar_wait(&S.formed[sc], par(t));  // every element of u1(t) formed

    const double2 rw01 = *reinterpret_cast<const double2*>(&S.rowt[sc][jr * 4]);      // W2[0], W2[1]
    const double2 rw2v = *reinterpret_cast<const double2*>(&S.rowt[sc][jr * 4 + 2]);  // W2[2], iV2
    const double w1m = S.rowt[sc][(jr - 1) * 4 + 1];                                  // W2[1] at j-1
    const double cr1 = rw01.x * g10;
    if (inside) {
      const bool okim = t > i0 || okim0;  // (plane t-1 exists: every plane after the chunk's first)
      const int ig = t + g.i0g;
      const bool pin = (g.pin_lo0 && ig == 0) || (g.pin_hi0 && ig == g.n0g - 1);
      const double Dcen = DM == 0 ? op.Dc : (DM == 1 ? dc : op.Dc * dc);
      double coef[3][2];
      coef[0][0] = okim ? cr0 : 0.0;
      coef[0][1] = cr1;
      coef[1][0] = okjm ? w1m * g11 : 0.0;
      coef[1][1] = rw01.y * g11;
      coef[2][0] = okkm ? rw2v.x * g12m : 0.0;
      coef[2][1] = rw2v.x * g12;
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
      if (SD) {
        nd[0][0] = dm;
        nd[0][1] = dp;
        nd[1][0] = S.A[sc][DS][htm];
        nd[1][1] = S.A[sc][DS][htp];
        nd[2][0] = S.A[sc][DS][hpm];
        nd[2][1] = S.A[sc][DS][hpp];
      }
      if (DM == 3) {  // in-plane neighbours hold the plane's rho
        nd[0][0] = dm;
        nd[0][1] = dp;
        nd[1][0] = nd[1][1] = nd[2][0] = nd[2][1] = dc;
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
      const double iv = rw2v.y * igv;
      const int64_t o = (int64_t)t * g.plane + onode;
      double f[3];
      const double irho = DM == 3 ? __ldg(op.rho_r + g.n0 + t)
                                  : (op.rho ? 1.0 / (DM == 2 ? dc : __ldg(op.rho + o)) : 1.0);
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
      if constexpr (AM) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          epi.F[c][o] = f[c];
          const double a = fabs(f[c]);
          if (a > am_v) {
            am_v = a;
            am_t = t;
            am_c = c;
          }
        }
      } else {
        epi.template apply<3>(g, t, jg, kg, o, f, vc, pin, ov);
      }
    }
    release(t);
    cr0 = cr1;
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
    if constexpr (NOP > 0) {  // operand slots: t <- t+1, t+1 <- t+2, t+2 <- the old t slot
      oph ^= 1u << o_c;
      const int o = o_c;
      o_c = o_p;
      o_p = o_n;
      o_n = o;
    }
  }
  if constexpr (AM) {
    if (am_v > epi.best.v) {
      epi.best.v = am_v;
      epi.bi = am_t;
      epi.bc = am_c;
      epi.bj = jg;
      epi.bk = kg;
    }
  }
  epi.finish(g);
}

}  // namespace pc
