// r-marching kernel for the 7-point rho-weighted finite-volume operator
// (ScalarOp: scalar diffusion, and the 3-component viscosity with the
// spherical frame rotation) -- K1 / K2 of DESIGN.md §4, the C1/C2/C5 stage.
//
// A 256-thread block owns an (SMJ x 32) theta-phi tile of an r-chunk and
// marches along r.  Per plane one cp.async group stages, one plane ahead,
//   * the NC input components (and the D / rho source) of plane t+2 with a
//     one-node in-plane halo (wrap / clamp resolved at fill time),
//   * the per-(r,theta) rows W2[0..2], iV2 of plane t+1,
//   * the epilogue operands of plane t+1 (thread-private slots),
// while each thread keeps its node's r-neighbours v(t-1), v(t) (and D) in
// registers and the four theta/phi frame rotations of its row come from a
// shared table loaded once.  Every face term is formed exactly as ScalarOp::F
// forms it (same operands, same order), so the result is bitwise the generic
// kernel's -- and the oracle's (oracle/operators.py scalar_apply).
#pragma once
#include "tma_march.cuh"

namespace pc {

constexpr int SMJ = 8;               // theta rows per tile (one warp per row)
constexpr int SHJ = SMJ + 2;
constexpr int SHP = SHJ * MHK;       // halo tile (phi extent MHK = 32 + 2)
constexpr int SNT = SMJ * MTK;       // threads = tile nodes
constexpr int SNFILL = (SHP + SNT - 1) / SNT;
constexpr int SROWT = 5;             // W2[0], W2[1], W2[2], iV2 per (plane, theta row), + W2[1] at j-1 via row - 1
constexpr int SEO = 9;               // epilogue operands staged per node (max: 3 x u0, um2, y0)
// resident blocks per SM asked of ptxas: the 3-component (vector) kernels need
// ~120 registers; capping them at 80 for 3 blocks/SM made ptxas re-load
// operands from shared memory (C2 stage 3811 GB/s at 3 blocks vs 4429 at 2,
// profiles/r01_c2_minb.txt).  SMARCH_MINB overrides both (experiments).
#ifdef SMARCH_MINB
#define SMARCH_BLOCKS(NC) SMARCH_MINB
#else
#define SMARCH_BLOCKS(NC) ((NC) == 3 ? 2 : 3)
#endif

// TMA staging (TM, spherical-type grids: phi periodic with n2 % 32 == 0, theta
// not periodic): per staged array and plane a 32 x 10 main box (columns
// k0 .. k0+31, rows j0-1 .. j0+8; rows outside theta are zero-filled and only
// meet a zero face coefficient) and two 2 x 10 strips whose phi coordinates
// wrap across the periodic seam (columns k0-2, k0-1 and k0+32, k0+33), issued
// by one lane and completed on one mbarrier per plane; the epilogue operands
// as 32 x 8 boxes.  Otherwise per-thread cp.async into the 10 x 34 halo tile.
constexpr int SXM = MTK * SHJ;      // TMA main box 32 x 10
constexpr int SXS = 32;             // strip 2 x 10, padded to 256 B (128-B aligned boxes)
constexpr int SXA = SXM + 2 * SXS;  // one staged array-plane in the TMA layout
constexpr int SPL = SXA > SHP ? SXA : SHP;  // slot size covering both layouts
constexpr int SNREAL = SXM + 2 * 2 * SHJ;   // real elements of the TMA layout (main + strips)
constexpr int SNFILL_T = (SNREAL + SNT - 1) / SNT;
constexpr int kSIss = SNT - 32;     // TMA issuer: lane 0 of the last warp
constexpr unsigned kSArrBytes = (unsigned)(SXM + 2 * 2 * SHJ) * 8u;  // bytes of one staged array-plane
constexpr unsigned kSOpBytes = (unsigned)(MTK * SMJ) * 8u;

struct SMaps {                // tensor maps of the TMA-staged 7-point march
  CUtensorMap V[3], VS[3];    // stencil input components: main box, strips
  CUtensorMap D, DS;          // D / rho source
  CUtensorMap Y[3], YS[3];    // F1: y0 components
  CUtensorMap O[9];           // epilogue operands, box 32 x 8
};

// F1 (fused stages 1 + 2, Epi::FUSE1): the stencil input is u1 = u0 + mt1 y0,
// formed into U from a u0 ring (V) and a y0 ring (Y) when each plane lands;
// the epilogue takes u0 and y0 at the node from V and Y (no operand staging).
// cp.async staging: the 10 x 34 halo tile per array-plane
template <int NC, bool F1 = false>
struct SMarchSmemC {
  double V[3][NC + 1][SHP];          // planes t, t+1, t+2 (in flight); slot NC = D / rho source
  double rowt[3][SROWT][SHJ];        // row tables of planes t-1 (r- face), t, t+1 (in flight)
  double EO[2][F1 ? 1 : SEO][SNT];   // epilogue operands of planes t (read) and t+1 (landing)
  double2 M[4][SMJ][5];              // frame rotations t+, t-, p+, p- of the tile rows (16-B pairs,
                                     // theta faces reordered m00 m01 m10 m11 first: two LDS.128)
  double Y[F1 ? 3 : 1][F1 ? NC : 1][F1 ? SHP : 1];  // y0 ring (F1 only; V then holds u0)
  double U[F1 ? 3 : 1][F1 ? NC : 1][F1 ? SHP : 1];  // u1 ring formed from V and Y (F1 only)
  unsigned long long bar;            // (TMA variant only)
};
// TMA staging: the same members in the box layout, ordered so that every
// TMA destination is 128-byte aligned
template <int NC, bool F1 = false>
struct SMarchSmemT {
  double V[3][NC + 1][SPL];
  double Y[F1 ? 3 : 1][F1 ? NC : 1][F1 ? SPL : 16];
  double U[F1 ? 3 : 1][F1 ? NC : 1][F1 ? SPL : 16];
  double EO[2][F1 ? 1 : SEO][SNT];
  double2 M[4][SMJ][5];
  double rowt[3][SROWT][SHJ];
  unsigned long long bar;            // TMA completion barrier
};
template <int NC, bool F1, bool TM>
using SMarchSmem = std::conditional_t<TM, SMarchSmemT<NC, F1>, SMarchSmemC<NC, F1>>;

// (fuse1_of: tma_march.cuh)

// DM: 0 = D constant Dc, 1 = D nodal field, 2 = D = Dc * rho (viscosity);
// TM: TMA staging (see SMaps), else cp.async
template <int NC, bool VEC, int DM, class Epi, bool TM = false>
__global__ void __launch_bounds__(SNT, SMARCH_BLOCKS(NC)) k_scalar_march(GridDev g, ScalarOp op, const double* __restrict__ u0p,
                                                         const double* __restrict__ u1p,
                                                         const double* __restrict__ u2p, Epi epi, int R, int zsel,
                                                         const int* skip, const __grid_constant__ SMaps maps) {
  constexpr bool F1 = fuse1_of<Epi>::value;
  extern __shared__ __align__(128) unsigned char smarch_smem[];
  // TMA destinations must be 128-byte aligned: align the dynamic base (the launch adds 128 bytes)
  SMarchSmem<NC, F1, TM>& S = *reinterpret_cast<SMarchSmem<NC, F1, TM>*>(
      smarch_smem + (TM ? ((128u - (smem_u32(smarch_smem) & 127u)) & 127u) : 0u));
  if (skip && *skip) return;
  constexpr bool HASD = DM != 0;
  const double* uin[3] = {u0p, u1p, u2p};
  const double* dsrc = DM == 1 ? op.D : op.rho;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int tid = threadIdx.x;
  const int k0 = blockIdx.x * MTK, j0 = blockIdx.y * SMJ, i0 = chunk_of(zsel) * R;
  const int iend = min(i0 + R, g.n0);
  const int kg = k0 + tx, jg = j0 + ty;

  // fill elements of this thread: cp.async staging (halo tile 10 x 34: the
  // source offset) or, with TMA, the layout slots F1 forms u1 over
  constexpr int NF = TM ? SNFILL_T : SNFILL;
  int foff[NF];
  unsigned pinfill = 0;  // F1: fill element q sits on a theta/phi Dirichlet node (u1 = u0 there)
#pragma unroll
  for (int q = 0; q < NF; ++q) {
    const int e = tid + q * SNT;
    int hj, kk0;
    if (TM) {  // main rows of 32, then the left (k0-2, k0-1) and right (k0+32, k0+33) strips
      if (e < SXM) {
        hj = e / MTK;
        kk0 = k0 + (e - hj * MTK);
      } else {
        const int r = e - SXM, side = r / (2 * SHJ), w = r - side * 2 * SHJ;
        hj = w >> 1;
        kk0 = (side == 0 ? k0 - 2 : k0 + MTK) + (w & 1);
      }
    } else {
      hj = e / MHK;
      kk0 = k0 - 1 + (e - hj * MHK);
    }
    bool oj, ok;
    const int jj = map_j(g, j0 - 1 + hj, oj), kk = map_k(g, kk0, ok);
    if (TM) {
      const int r = e - SXM;
      foff[q] = e >= SNREAL ? -1 : (e < SXM ? e : SXM + (r / (2 * SHJ)) * SXS + (r % (2 * SHJ)));
    } else {
      foff[q] = e < SHP ? jj * g.n2 + kk : -1;
    }
    if ((g.pin_lo1 && jj == 0) || (g.pin_hi1 && jj == g.n1 - 1) || (g.pin_lo2 && kk == 0) ||
        (g.pin_hi2 && kk == g.n2 - 1))
      pinfill |= 1u << q;
  }
  const int kL = k0 == 0 ? g.n2 - 2 : k0 - 2;     // TMA strips (phi wraps across the seam)
  const int kR = k0 + MTK == g.n2 ? 0 : k0 + MTK;
  if (TM && tid == 0) {
    mbar_init(&S.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unsigned phase = 0;
  const bool rton = tid < SROWT * SHJ;
  const int rtab = tid / SHJ, rhj = tid - (tid / SHJ) * SHJ;
  bool rok;
  const int rjj = map_j(g, j0 - 1 + rhj, rok);
  const double* rbase = !rton ? g.iV2 : (rtab < 3 ? g.W2[rtab] : g.iV2);

  // rotation table of the tile rows (loaded once; rows beyond n1 clamp)
  if (VEC) {
    for (int e = tid; e < 4 * SMJ * 10; e += SNT) {
      const int f = e / (SMJ * 10), r = (e / 10) % SMJ, q = e % 10;
      const int jr = min(j0 + r, g.n1 - 1);
      // theta faces: slots 0..3 = M[0], M[1], M[3], M[4]; phi faces: M[0..8]; slot 9 unused
      const int th = q < 2 ? q : (q < 4 ? q + 1 : (q == 4 ? 2 : (q < 9 ? q : 8)));  // 0 1 3 4 2 5 6 7 8 8
      const int src = f < 2 ? th : (q < 9 ? q : 8);
      reinterpret_cast<double*>(&S.M[f][r][0])[q] = __ldg(g.M[f] + (int64_t)jr * 9 + src);
    }
  }

  bool oko, ojo;
  const int km = map_k(g, kg, oko);
  map_j(g, jg, ojo);
  const bool inside = jg < g.n1 && kg < g.n2;
  (void)ojo;
  // column constants: g1[0](k), g1[1](k), g1[2](k), g1[2](k-1), igv(k)
  bool okkm;
  const int kmm = nb2(g, km, -1, okkm);
  const double g10 = launder(__ldg(g.g1[0] + km)), g11 = launder(__ldg(g.g1[1] + km));
  const double g12 = launder(__ldg(g.g1[2] + km)), g12m = launder(okkm ? __ldg(g.g1[2] + kmm) : 0.0);
  const double igv = launder(__ldg(g.igv + km));
  bool okjm;
  nb1(g, jg < g.n1 ? jg : g.n1 - 1, -1, okjm);
  const bool pin_jk = (g.pin_lo1 && jg == 0) || (g.pin_hi1 && jg == g.n1 - 1) || (g.pin_lo2 && kg == 0) ||
                      (g.pin_hi2 && kg == g.n2 - 1);
  // staged-tile offsets of the own node and its theta / phi neighbours
  const int h = TM ? (ty + 1) * MTK + tx : (ty + 1) * MHK + (tx + 1);
  const int htm = TM ? h - MTK : h - MHK, htp = TM ? h + MTK : h + MHK;
  const int hpm = TM ? (tx > 0 ? h - 1 : SXM + (ty + 1) * 2 + 1) : h - 1;
  const int hpp = TM ? (tx < MTK - 1 ? h + 1 : SXM + SXS + (ty + 1) * 2) : h + 1;
  const int onode = jg * g.n2 + kg;
  // (TMA issue, lane 0 of the last warp: all boxes of one plane complete on S.bar)
  auto tma_arr = [&](double* dst, const CUtensorMap* mm, const CUtensorMap* ms, int z) {
    tma3(dst, mm, k0, j0 - 1, z, &S.bar);
    tma3(dst + SXM, ms, kL, j0 - 1, z, &S.bar);
    tma3(dst + SXM + SXS, ms, kR, j0 - 1, z, &S.bar);
  };

  auto eslot = [&](int p) { return (p - i0) & 1; };
  auto issue_V = [&](int p, int sl) {
    const PlaneMap pm = plane_map(g, p);
    if constexpr (TM) {
      if (tid == kSIss) {
        const int z = pm.mem + 1;  // (the tensors start at ghost plane -1)
#pragma unroll
        for (int c = 0; c < NC; ++c) tma_arr(&S.V[sl][c][0], &maps.V[c], &maps.VS[c], z);
        if (HASD) tma_arr(&S.V[sl][NC][0], &maps.D, &maps.DS, z);
        if constexpr (F1) {
#pragma unroll
          for (int c = 0; c < NC; ++c) tma_arr(&S.Y[sl][c][0], &maps.Y[c], &maps.YS[c], z);
        }
      }
      return;
    }
    const int64_t base = (int64_t)pm.mem * g.plane;
#pragma unroll
    for (int q = 0; q < SNFILL; ++q)
      if (foff[q] >= 0) {
        const int e = tid + q * SNT;
#pragma unroll
        for (int c = 0; c < NC; ++c) cp_async8(&S.V[sl][c][e], uin[c] + base + foff[q]);
        if (HASD) cp_async8(&S.V[sl][NC][e], dsrc + base + foff[q]);
        if constexpr (F1) {
#pragma unroll
          for (int c = 0; c < NC; ++c) cp_async8(&S.Y[sl][c][e], epi.y0[c] + base + foff[q]);
        }
      }
  };
  // F1: u1 = pin ? u0 : u0 + mt1 y0 (k_stage1's expression) over the elements
  // this thread staged for plane p, after its own cp.async group completed
  // (the block barrier that follows publishes them)
  auto form_u1 = [&](int p, int sl) {
    if constexpr (F1) {
      const PlaneMap pm = plane_map(g, p);
      const int ig = pm.mem + g.i0g;
      const bool ppin = (g.pin_lo0 && ig == 0) || (g.pin_hi0 && ig == g.n0g - 1);
#pragma unroll
      for (int q = 0; q < NF; ++q)
        if (foff[q] >= 0) {
          const int e = TM ? foff[q] : tid + q * SNT;
          const bool pn = ppin || ((pinfill >> q) & 1u);
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const double a = S.V[sl][c][e];
            S.U[sl][c][e] = pn ? a : a + epi.mt1 * S.Y[sl][c][e];
          }
        }
    }
  };
  auto issue_rows = [&](int p, int sl) {
    if (rton) {
      const PlaneMap pm = plane_map(g, p);
      cp_async8(&S.rowt[sl][rtab][rhj], rbase + row2(g, pm.row, rjj));
    }
  };
  // stencil input of component c at ring slot sl, element e
  auto uat = [&](int sl, int c, int e) -> double {
    if constexpr (F1) return S.U[sl][c][e];
    else return S.V[sl][c][e];
  };
  auto issue_ops = [&](int p) {
    if constexpr (TM) {
      if (!F1 && Epi::NOPS > 0 && tid == kSIss) {
        const int es = eslot(p);
#pragma unroll
        for (int q = 0; q < Epi::NOPS; ++q) tma3(&S.EO[es][q][0], &maps.O[q], k0, j0, p + 1, &S.bar);
      }
      return;
    }
    if (!F1 && Epi::NOPS > 0 && inside) {
      const int64_t o = (int64_t)p * g.plane + onode;
      const int es = eslot(p);
#pragma unroll
      for (int q = 0; q < Epi::NOPS; ++q) cp_async8(&S.EO[es][q][tid], epi.opnd(q) + o);
    }
  };

  // ring slots of planes t-1, t, t+1 (vslot / rslot (p - i0 + 1) % 3, rotated
  // once per plane instead of a modulo per use); t+2 reuses the t-1 slot
  int s_m = 0, s_c = 1, s_p = 2;
  // bytes of one plane's boxes (TMA): staged arrays (+ D, + y0) and operands
  constexpr unsigned kVB = (unsigned)(NC + (HASD ? 1 : 0) + (F1 ? NC : 0)) * kSArrBytes;
  constexpr unsigned kOB = F1 ? 0u : (unsigned)Epi::NOPS * kSOpBytes;
  // ---- prologue: V(i0-1..i0+1), rows(i0-1, i0), operands(i0)
  if (TM) {
    __syncthreads();  // barrier initialised
    if (tid == kSIss) mbar_expect_tx(&S.bar, (i0 + 1 <= iend ? 3u : 2u) * kVB + kOB);
  }
  issue_V(i0 - 1, s_m);
  issue_V(i0, s_c);
  if (i0 + 1 <= iend) issue_V(i0 + 1, s_p);
  issue_rows(i0 - 1, s_m);
  issue_rows(i0, s_c);
  issue_ops(i0);
  cp_async_commit();
  cp_async_wait<0>();
  if (TM) {
    mbar_wait(&S.bar, phase);
    phase ^= 1u;
  }
  form_u1(i0 - 1, s_m);
  form_u1(i0, s_c);
  if (i0 + 1 <= iend) form_u1(i0 + 1, s_p);
  __syncthreads();

  double vm[NC], vc[NC], dm = 0.0, dc = 0.0;
  {
    const int s0 = s_m, s1 = s_c;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      vm[c] = uat(s0, c, h);
      vc[c] = uat(s1, c, h);
    }
    if (HASD) {
      dm = S.V[s0][NC][h];
      dc = S.V[s1][NC][h];
    }
  }
  const int jr = ty + 1;  // row-table index of the own row (halo row 0 = j0 - 1)
  // every thread has read its plane i0-1 values before the first refill of
  // that slot (issue_V(i0 + 2) below) may land
  __syncthreads();

#pragma unroll 1
  for (int t = i0; t < iend; ++t) {
    if (TM && tid == kSIss) {  // one phase per plane: arm it with all of this plane's boxes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&S.bar, (t + 2 <= iend ? kVB : 0u) + (t + 1 < iend ? kOB : 0u));
    }
    if (t + 2 <= iend) issue_V(t + 2, s_m);
    if (t + 1 <= iend) issue_rows(t + 1, s_p);
    if (t + 1 < iend) issue_ops(t + 1);
    cp_async_commit();

    const int sc = s_c, sp = s_p, rs = s_c, rm = s_m, es = eslot(t);
    const PlaneMap pmm = plane_map(g, t - 1);
    const bool okim = pmm.exists;  // r- neighbour exists
    double vp[NC], dp = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) vp[c] = uat(sp, c, h);
    if (HASD) dp = S.V[sp][NC][h];
    if (inside) {
      const int ig = t + g.i0g;
      const bool pin = pin_jk || (g.pin_lo0 && ig == 0) || (g.pin_hi0 && ig == g.n0g - 1);
      const double Dcen = DM == 0 ? op.Dc : (DM == 1 ? dc : op.Dc * dc);
      // face coefficients W*g (ScalarOp::wg): faces (a, -), (a, +) for a = 0, 1, 2
      double coef[3][2];
      coef[0][0] = okim ? S.rowt[rm][0][jr] * g10 : 0.0;
      coef[0][1] = S.rowt[rs][0][jr] * g10;
      coef[1][0] = okjm ? S.rowt[rs][1][jr - 1] * g11 : 0.0;
      coef[1][1] = S.rowt[rs][1][jr] * g11;
      coef[2][0] = okkm ? S.rowt[rs][2][jr] * g12m : 0.0;
      coef[2][1] = S.rowt[rs][2][jr] * g12;
      // neighbour values (self where missing: staging clamps) and D
      double nv[3][2][NC], nd[3][2];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        nv[0][0][c] = vm[c];
        nv[0][1][c] = vp[c];
        nv[1][0][c] = uat(sc, c, htm);
        nv[1][1][c] = uat(sc, c, htp);
        nv[2][0][c] = uat(sc, c, hpm);
        nv[2][1][c] = uat(sc, c, hpp);
      }
      if (HASD) {
        nd[0][0] = dm;
        nd[0][1] = dp;
        nd[1][0] = S.V[sc][NC][htm];
        nd[1][1] = S.V[sc][NC][htp];
        nd[2][0] = S.V[sc][NC][hpm];
        nd[2][1] = S.V[sc][NC][hpp];
      }
      double Sx[NC];
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
          if (VEC && a > 0) {
            const double2* M2 = S.M[(a == 1 ? 0 : 2) + (tt == 1 ? 0 : 1)][ty];
            const double v0 = nv[a][tt][0], v1 = nv[a][tt][NC > 1 ? 1 : 0], v2 = nv[a][tt][NC > 2 ? 2 : 0];
            double rv[NC];
            if (a == 1) {
              // theta faces rotate about e_phi: M = [[m00 m01 0] [m10 m11 0] [0 0 1]]
              // with exact zeros and one (geometry._rotation_tables), so the
              // dense row sums reduce to these bits (up to the sign of a zero)
              const double2 r0 = M2[0], r1 = M2[1];  // (m00, m01), (m10, m11)
              rv[0] = (r0.x * v0) + (r0.y * v1);
              if (NC > 1) rv[NC > 1 ? 1 : 0] = (r1.x * v0) + (r1.y * v1);
              if (NC > 2) rv[NC > 2 ? 2 : 0] = v2;
            } else {
              double M[10];
#pragma unroll
              for (int q = 0; q < 5; ++q) {
                const double2 w = M2[q];
                M[2 * q] = w.x;
                M[2 * q + 1] = w.y;
              }
#pragma unroll
              for (int c = 0; c < NC; ++c) rv[c] = ((M[3 * c] * v0) + (M[3 * c + 1] * v1)) + (M[3 * c + 2] * v2);
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              const double term = cf * (rv[c] - vc[c]);
              Sx[c] = first ? term : Sx[c] + term;
            }
          } else {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              const double term = cf * (nv[a][tt][c] - vc[c]);
              Sx[c] = first ? term : Sx[c] + term;
            }
          }
        }
      }
      const double iv = S.rowt[rs][3][jr] * igv;
      const int64_t o = (int64_t)t * g.plane + onode;
      double f[NC];
      // (1/rho) div(nu rho grad v): one reciprocal per node, not a division per component
      const double irho = op.rho ? 1.0 / (DM == 2 ? dc : __ldg(op.rho + o)) : 1.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double x = Sx[c] * iv;
        if (op.rho) x = x * irho;
        f[c] = pin ? 0.0 : x;
      }
      double ov[Epi::NOPS > 0 ? Epi::NOPS : 1];
#pragma unroll
      for (int q = 0; q < Epi::NOPS; ++q)
        if constexpr (!F1) ov[q] = S.EO[es][q][tid];
      if constexpr (F1) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          ov[2 * c] = S.V[sc][c][h];
          ov[2 * c + 1] = S.Y[sc][c][h];
        }
      }
      epi.template apply<NC>(g, t, jg, kg, o, f, vc, pin, ov);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      vm[c] = vc[c];
      vc[c] = vp[c];
    }
    if (HASD) {
      dm = dc;
      dc = dp;
    }
    cp_async_wait<0>();
    if (TM) {
      mbar_wait(&S.bar, phase);
      phase ^= 1u;
    }
    if (t + 2 <= iend) form_u1(t + 2, s_m);
    __syncthreads();
    {  // rotate the slot roles: t-1 <- t, t <- t+1, t+1 <- t+2 (the old t-1 slot)
      const int o = s_m;
      s_m = s_c;
      s_c = s_p;
      s_p = o;
    }
  }
  epi.finish(g);
}

// ---- epilogues of the 7-point march (NC components per node) --------------
struct SEpiStore {
  static constexpr int NOPS = 0;
  double* F[3];
  __host__ __device__ __forceinline__ const double* opnd(int) const { return nullptr; }
  template <int NC>
  __device__ __forceinline__ void apply(const GridDev&, int, int, int, int64_t o, const double (&f)[NC],
                                        const double (&)[NC], bool, const double*) {
#pragma unroll
    for (int c = 0; c < NC; ++c) F[c][o] = f[c];
  }
  __device__ __forceinline__ void finish(const GridDev&) {}
};

// fused RKL2/RKG2 stage: operands u0[c], um2[c], y0[c] staged per node
struct SEpiStage {
  static constexpr int NOPS_MAX = 9;
  static constexpr int NOPS = 9;  // (3 x NC used; NC = 1 stages slots 0..2 only -- see make_sepi_stage)
  const double* u0[3];
  const double* um2[3];
  const double* y0[3];
  double* out[3];
  int nc;
  StageCoef sc;
  int stage;
  int* bad;
  int fl = 0x7fffffff;  // this thread saw a non-finite value (the stage), reported in finish()
  __host__ __device__ __forceinline__ const double* opnd(int q) const {
    const int c = q / 3, w = q % 3;
    return w == 0 ? u0[c] : (w == 1 ? um2[c] : y0[c]);
  }
  template <int NC>
  __device__ __forceinline__ void apply(const GridDev&, int, int, int, int64_t o, const double (&f)[NC],
                                        const double (&um1)[NC], bool pin, const double* ov) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double a0 = ov[3 * c];
      double v = ((((sc.mu * um1[c]) + (sc.nu * ov[3 * c + 1])) + (sc.kap * a0)) + (sc.mtdt * f[c])) +
                 (sc.gtdt * ov[3 * c + 2]);
      v = pin ? a0 : v;
      out[c][o] = v;
      fl = isfinite(v) ? fl : stage;  // (one stage per launch)
    }
  }
  __device__ __forceinline__ void finish(const GridDev&) {
    if (fl != 0x7fffffff) atomicMin(bad, fl);  // one atomic per flagged thread, not a branch per node
  }
};
// one-component variant (only 3 operand slots are staged)
struct SEpiStage1 : SEpiStage {
  static constexpr int NOPS = 3;
};

// stages 1 and 2 in one pass (FUSE1): the kernel stages u0 and y0 and forms
// u1 = u0 + mt1 y0 as each plane lands, so F(u1) never needs u1 in HBM; the
// epilogue writes u2 = mu2 u1 + nu2 u0 + kap2 u0 + mt2 F(u1) + gt2 y0 (k_stage
// with u_{k-2} = u0) and, when stage 3 follows, u1 itself (its u_{k-2}).
// Non-finite u1 flags stage 1, non-finite u2 stage 2 (as the two launches did).
template <int NCX>
struct SEpiStage12 {
  static constexpr bool FUSE1 = true;
  static constexpr int NOPS = 2 * NCX;  // u0[c], y0[c] at the node
  const double* u0[3];
  const double* y0[3];
  double* out[3];
  double* u1out[3];  // nullptr: s == 2, u1 is not needed after this pass
  double mt1;
  StageCoef sc;
  int* bad;
  int fl = 0x7fffffff;  // lowest stage this thread saw non-finite (1: u1, 2: u2), reported in finish()
  __host__ __device__ __forceinline__ const double* opnd(int q) const { return (q & 1) ? y0[q >> 1] : u0[q >> 1]; }
  template <int NC>
  __device__ __forceinline__ void apply(const GridDev&, int, int, int, int64_t o, const double (&f)[NC],
                                        const double (&u1)[NC], bool pin, const double* ov) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double a0 = ov[2 * c];
      if (u1out[0]) u1out[c][o] = u1[c];
      double v = ((((sc.mu * u1[c]) + (sc.nu * a0)) + (sc.kap * a0)) + (sc.mtdt * f[c])) + (sc.gtdt * ov[2 * c + 1]);
      v = pin ? a0 : v;
      out[c][o] = v;
      fl = isfinite(v) ? fl : min(fl, 2);
      fl = isfinite(u1[c]) ? fl : 1;
    }
  }
  __device__ __forceinline__ void finish(const GridDev&) {
    if (fl != 0x7fffffff) atomicMin(bad, fl);
  }
};

struct SEpiArgmax {  // y0 = F(u0) with the |F| argmax over points x components (PTL)
  static constexpr int NOPS = 0;
  __host__ __device__ __forceinline__ const double* opnd(int) const { return nullptr; }
  double* F[3];
  double* pv;
  long long* pi;
  unsigned int* counter;
  ArgRes* res;
  ArgMax best;
  int ncomp;
  // this thread's maximum so far (nodes visited in increasing AoS index --
  // planes in order, components in order -- so a strict > keeps the lowest
  // index among equal maxima); the index is formed once, in finish()
  int bi = 0, bc = 0, bj = 0, bk = 0;
  template <int NC>
  __device__ __forceinline__ void apply(const GridDev&, int i, int j, int k, int64_t o, const double (&f)[NC],
                                        const double (&)[NC], bool, const double*) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      F[c][o] = f[c];
      const double a = fabs(f[c]);
      if (a > best.v) {
        best.v = a;
        bi = i;
        bc = c;
        bj = j;
        bk = k;
      }
    }
  }
  __device__ __forceinline__ void finish(const GridDev& g) {
    __shared__ double shv[SNT / 32];
    __shared__ long long shi[SNT / 32];
    const int tid = threadIdx.x;
    const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int nblk = gridDim.x * gridDim.y * gridDim.z;
    if (best.v >= 0.0) best.i = aos_index(g, bi, bj, bk, bc, ncomp);
    ArgMax b = block_argmax<SNT>(best, shv, shi);
    if (tid == 0) {
      pv[bid] = b.v;
      pi[bid] = b.i;
    }
    if (last_block3(counter, nblk)) {
      ArgMax r{-1.0, 0x7fffffffffffffffLL};
      for (int q = tid; q < nblk; q += SNT) r = am_better(r, ArgMax{pv[q], pi[q]});
      r = block_argmax<SNT>(r, shv, shi);
      if (tid == 0) {
        res->fmax = r.v;
        res->kidx = r.i;
        *counter = 0u;
      }
    }
  }
};

}  // namespace pc
