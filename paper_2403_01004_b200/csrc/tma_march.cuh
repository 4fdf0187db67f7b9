// TMA-staged variant of the r-marching Spitzer kernel (K3/K4/K7), used when
// the grid allows it (phi periodic with n2 % 32 == 0, theta not periodic --
// every spherical grid of the configs); k_aligned_march (cp.async) is the
// general fallback.  Same arithmetic, same schedule, bitwise-identical output.
//
// Per plane ONE thread issues the bulk tensor copies (cp.async.bulk.tensor,
// completion counted on one mbarrier): for T and each beta component a
// 32 x 18 main box (256-byte rows, phi-aligned) plus two 2 x 18 halo strips
// whose phi coordinates wrap across the periodic seam; the epilogue operands
// as 32 x 16 boxes.  Rows outside the theta range are zero-filled by the TMA
// unit: they only ever meet an inverse edge length of 0 (no flux through the
// pole faces), exactly as the clamped values of the oracle do.  The metric
// rows stay on cp.async (one 8-byte copy for 198 threads).
#pragma once
#include <cuda.h>

#include "march.cuh"

namespace pc {

constexpr int XM = MHJ * MTK;      // main box: 18 rows x 32 phi (4608 B)
constexpr int XS = 48;             // halo strip: 18 x 2 doubles, padded to 384 B (128-B aligned boxes)
constexpr int XA = XM + 2 * XS;    // one staged array of one plane
constexpr int XO = MTJ * MTK;      // epilogue operand box 16 x 32
constexpr unsigned kArrBytes = (unsigned)(XM + 2 * MHJ * 2) * 8u;  // bytes a T / beta plane delivers
constexpr unsigned kOpBytes = (unsigned)XO * 8u;

struct TmaMaps {
  CUtensorMap T;     // stage input, box {32, 18, 1}
  CUtensorMap TS;    // same tensor, strip box {2, 18, 1}
  CUtensorMap B[3];  // beta, box {32, 18, 1}
  CUtensorMap BS[3]; // beta strips
  CUtensorMap O[3];  // epilogue operands, box {32, 16, 1}
};

// compact in-plane flux exchange: entries readers use only
struct FluxC {
  double e1p[MTJ][MTK];  // E_{1,+} at rows j0-1 .. j0+14
  double e1m[MTJ][MTK];  // E_{1,-} at rows j0+1 .. j0+16
  double e2p[MTJ][MTK];  // E_{2,+} at cols k0-1 .. k0+30
  double e2m[MTJ][MTK];  // E_{2,-} at cols k0+1 .. k0+32
};
struct TmaSmem {
  double T[TSL][XA];
  double B[BSL][3][XA];
  double EO[2][3][XO];
  FluxC E[2];
  double rowt[RSL][NROWT][MHJ];
  double ringcol[2][9];
  unsigned long long bar;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma3(double* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                     unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

template <class Epi>
__global__ void __launch_bounds__(MNT, 2) k_aligned_tma(GridDev g, AlignedOp op, const __grid_constant__ TmaMaps maps,
                                                        Epi epi, int R, const int* skip) {
  extern __shared__ __align__(128) unsigned char tma_smem[];
  // bulk-tensor destinations must be 128-byte aligned: align the dynamic base
  // (static epilogue scratch may precede it); the launch adds 128 bytes
  TmaSmem& S = *reinterpret_cast<TmaSmem*>(tma_smem + ((128u - (smem_u32(tma_smem) & 127u)) & 127u));
  if (skip && *skip) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * MTK + tx;
  const int k0 = blockIdx.x * MTK, j0 = blockIdx.y * MTJ, i0 = blockIdx.z * R;
  const int iend = min(i0 + R, g.n0);
  const int kg = k0 + tx;
  const int kL = k0 == 0 ? g.n2 - 2 : k0 - 2;           // strip of columns k0-2, k0-1
  const int kR = k0 + MTK == g.n2 ? 0 : k0 + MTK;        // strip of columns k0+32, k0+33

  // row-table fill slot of this thread: tid < NROWT * MHJ (cp.async)
  const bool rton = tid < NROWT * MHJ;
  const int rtab = tid / MHJ, rhj = tid - (tid / MHJ) * MHJ;
  bool rok;
  const int rjj = map_j(g, j0 - 1 + rhj, rok);
  const double* rbase = !rton ? g.iVal2 : (rtab < 6 ? g.iL2[rtab] : (rtab < 10 ? g.wo01[rtab - 6] : g.iVal2));

  const int km = kg;  // n2 % 32 == 0: every lane is a node
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
  if (tid == 0) {
    mbar_init(&S.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }

  // ring node of this thread (tid < NRING): offsets of centre, theta+-, phi+- in a staged array
  int ra = -1, rs = 0, rhj_ = 0, rkk = 0;
  int ro_c = 0, ro_tp = 0, ro_tm = 0, ro_pm = 0, ro_pp = 0;
  if (tid < 2 * MTK) {
    ra = 1;
    rs = tid < MTK ? 0 : 1;
    const int c = tid % MTK;
    rhj_ = rs == 0 ? 0 : MTJ + 1;
    rkk = c;
    ro_c = rhj_ * MTK + c;
    ro_tp = rs == 0 ? ro_c + MTK : ro_c;
    ro_tm = rs == 0 ? ro_c : ro_c - MTK;
    ro_pm = c > 0 ? ro_c - 1 : XM + rhj_ * 2 + 1;
    ro_pp = c < MTK - 1 ? ro_c + 1 : XM + XS + rhj_ * 2;
  } else if (tid < NRING) {
    const int q = tid - 2 * MTK;
    ra = 2;
    rs = q < MTJ ? 0 : 1;
    rhj_ = 1 + (q % MTJ);
    if (rs == 0) {  // column k0-1: left strip, slot 1
      ro_c = XM + rhj_ * 2 + 1;
      ro_tp = ro_c + 2;
      ro_tm = ro_c - 2;
      ro_pm = ro_c - 1;
      ro_pp = rhj_ * MTK;
    } else {        // column k0+32: right strip, slot 0
      ro_c = XM + XS + rhj_ * 2;
      ro_tp = ro_c + 2;
      ro_tm = ro_c - 2;
      ro_pm = rhj_ * MTK + MTK - 1;
      ro_pp = ro_c + 1;
    }
  }
  bool ring_on = false;
  if (ra >= 0) {
    bool rjo, rko;
    const int gj = j0 - 1 + rhj_, gk = ra == 1 ? k0 + rkk : (rs == 0 ? k0 - 1 : k0 + MTK);
    map_j(g, gj, rjo);
    map_k(g, gk, rko);
    ring_on = rjo && rko && (ra == 1 ? true : (gj < g.n1));
  }

  // own nodes: staged-array offsets of centre and neighbours
  const int onode0 = (j0 + ty) * g.n2 + kg;
  bool inside[NPT], pin_j[NPT];
  int oc[NPT], opm[NPT], opp[NPT];
  auto jn = [&](int n) { return j0 + ty + n * MTY; };
  auto onode = [&](int n) { return onode0 + n * MTY * g.n2; };
#pragma unroll
  for (int n = 0; n < NPT; ++n) {
    const int hr = ty + n * MTY + 1;
    inside[n] = jn(n) < g.n1;
    pin_j[n] = (g.pin_lo1 && jn(n) == 0) || (g.pin_hi1 && jn(n) == g.n1 - 1);
    oc[n] = hr * MTK + tx;
    opm[n] = tx > 0 ? oc[n] - 1 : XM + hr * 2 + 1;
    opp[n] = tx < MTK - 1 ? oc[n] + 1 : XM + XS + hr * 2;
  }

  auto tslot = [&](int p) { return (p - i0 + 1) % TSL; };
  auto bslot = [&](int p) { return (p - i0 + 1) & (BSL - 1); };
  auto rslot = [&](int p) { return (p - i0 + 1) % RSL; };
  auto eslot = [&](int p) { return (p - i0) & 1; };
  // (thread 0 only)
  auto tma_arr = [&](double* dst, const CUtensorMap* mm, const CUtensorMap* ms, int p) {
    const int z = plane_map(g, p).mem + 1;
    tma3(dst, mm, k0, j0 - 1, z, &S.bar);
    tma3(dst + XM, ms, kL, j0 - 1, z, &S.bar);
    tma3(dst + XM + XS, ms, kR, j0 - 1, z, &S.bar);
  };
  auto issue_T = [&](int p) { tma_arr(S.T[tslot(p)], &maps.T, &maps.TS, p); };
  auto issue_B = [&](int p) {
#pragma unroll
    for (int q = 0; q < 3; ++q) tma_arr(S.B[bslot(p)][q], &maps.B[q], &maps.BS[q], p);
  };
  auto issue_ops = [&](int p) {
#pragma unroll
    for (int q = 0; q < Epi::NOPS; ++q) tma3(S.EO[eslot(p)][q], &maps.O[q], k0, j0, p + 1, &S.bar);
  };
  auto issue_rows = [&](int p) {
    if (rton) {
      const PlaneMap pm = plane_map(g, p);
      cp_async8(&S.rowt[rslot(p)][rtab][rhj], rbase + row2(g, pm.row, rjj));
    }
  };

  // ---- prologue
  __syncthreads();  // barrier initialised
  if (tid == 0) {
    const bool t1 = i0 + 1 <= iend;
    mbar_expect_tx(&S.bar, (2u + (t1 ? 1u : 0u)) * kArrBytes + 6u * kArrBytes);
    issue_T(i0 - 1);
    issue_T(i0);
    if (t1) issue_T(i0 + 1);
    issue_B(i0 - 1);
    issue_B(i0);
  }
  issue_rows(i0 - 1);
  issue_rows(i0);
  cp_async_commit();
  cp_async_wait<0>();
  unsigned phase = 0;
  mbar_wait(&S.bar, phase);
  phase ^= 1u;
  __syncthreads();

  double Tm[NPT], Tc[NPT], qa[NPT], qb[NPT], ownp[NPT];
  double Tmr = 0.0;
  {
    const PlaneMap pm = plane_map(g, i0 - 1);
    const double* s0 = S.T[tslot(i0 - 1)];
    const double* s1 = S.T[tslot(i0)];
    const int bs = bslot(i0 - 1), rsl = rslot(i0 - 1);
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      Tm[n] = s0[oc[n]];
      Tc[n] = s1[oc[n]];
      qa[n] = 0.0;
      qb[n] = 0.0;
      ownp[n] = 0.0;
      if (pm.exists && inside[n]) {  // E_{0,+}(i0 - 1)
        const double Tn[3][2] = {{Tc[n], Tm[n]}, {s0[oc[n] + MTK], s0[oc[n] - MTK]}, {s0[opp[n]], s0[opm[n]]}};
        const double bv[3] = {S.B[bs][0][oc[n]], S.B[bs][1][oc[n]], S.B[bs][2][oc[n]]};
        double E[3][2];
        node_E<0, 0>(Tm[n], Tn, bv, &S.rowt[rsl][0][ty + n * MTY + 1], MHJ, col.il1, col.w2, E);
        qb[n] = E[0][0];
      }
    }
    if (ra >= 0) Tmr = s0[ro_c];
  }

  auto step = [&](int t, auto last_tag) {
    constexpr bool LAST = decltype(last_tag)::value;
    if (!LAST) {
      if (tid == 0) {
        const bool t2 = t + 2 <= iend;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&S.bar, (t2 ? kArrBytes : 0u) + 3u * kArrBytes + (unsigned)Epi::NOPS * kOpBytes);
        if (t2) issue_T(t + 2);
        issue_B(t + 1);
        issue_ops(t);
      }
      issue_rows(t + 1);
      cp_async_commit();
    }
    const bool exists = LAST ? plane_map(g, t).exists : true;
    const double* sT = S.T[tslot(t)];
    const double* sTp = S.T[tslot(t + 1)];
    const int bs = bslot(t), rsl = rslot(t), rslm = rslot(t - 1);
    const int par = t & 1, pp = par ^ 1;
    const int esm = eslot(t - 1);
    const int tf = t - 1;
    const int ig = tf + g.i0g;
    const bool pin_i = (g.pin_lo0 && ig == 0) || (g.pin_hi0 && ig == g.n0g - 1);
    const int64_t pbase = (int64_t)t * g.plane;
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      const int r = ty + n * MTY;
      const int jr = r + 1;
      double E[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      double Tp = 0.0;
      if (!LAST) Tp = sTp[oc[n]];
      if (exists && inside[n]) {
        const double Tn[3][2] = {{Tp, Tm[n]}, {sT[oc[n] + MTK], sT[oc[n] - MTK]}, {sT[opp[n]], sT[opm[n]]}};
        const double bv[3] = {S.B[bs][0][oc[n]], S.B[bs][1][oc[n]], S.B[bs][2][oc[n]]};
        if (!LAST) node_E<-1, 0>(Tc[n], Tn, bv, &S.rowt[rsl][0][jr], MHJ, col.il1, col.w2, E);
        else node_E<0, 1>(Tc[n], Tn, bv, &S.rowt[rsl][0][jr], MHJ, col.il1, col.w2, E);
      }
      if (!LAST) {
        if (r < MTJ - 1) S.E[par].e1p[r + 1][tx] = E[1][0];
        if (r > 0) S.E[par].e1m[r - 1][tx] = E[1][1];
        if (tx < MTK - 1) S.E[par].e2p[r][tx + 1] = E[2][0];
        if (tx > 0) S.E[par].e2m[r][tx - 1] = E[2][1];
      }
      if (t > i0 && inside[n]) {
        const double nbr = (S.E[pp].e1p[r][tx] - S.E[pp].e1m[r][tx]) + (S.E[pp].e2p[r][tx] - S.E[pp].e2m[r][tx]);
        const double G = (qa[n] - E[0][1]) + (ownp[n] + nbr);
        const double iv = S.rowt[rslm][10][jr] * col.ivg;
        const int64_t of = pbase - g.plane + onode(n);
        double f = ((0.0 - G) * iv) * op.pref;
        if (op.rho) f = f / __ldg(op.rho + of);
        const bool pin = pin_i || pin_j[n] || pin_k;
        if (pin) f = 0.0;
        double ov[Epi::NOPS > 0 ? Epi::NOPS : 1];
#pragma unroll
        for (int q = 0; q < Epi::NOPS; ++q) ov[q] = S.EO[esm][q][r * MTK + tx];
        epi(n, g, tf, jn(n), kg, of, f, Tm[n], pin, ov);
      }
      if (!LAST) {
        ownp[n] = ((E[0][1] - E[0][0]) + (E[1][1] - E[1][0])) + (E[2][1] - E[2][0]);
        qa[n] = qb[n];
        qb[n] = E[0][0];
        Tm[n] = Tc[n];
        Tc[n] = Tp;
      }
    }
    // ---- halo ring of plane t
    if (!LAST && ra >= 0) {
      const double Tcr = sT[ro_c];
      const double Tpr = sTp[ro_c];
      double Ev = 0.0;
      if (ring_on) {
        const double Tn[3][2] = {{Tpr, Tmr}, {sT[ro_tp], sT[ro_tm]}, {sT[ro_pp], sT[ro_pm]}};
        const double bv[3] = {S.B[bs][0][ro_c], S.B[bs][1][ro_c], S.B[bs][2][ro_c]};
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
        if (rs == 0) S.E[par].e1p[0][rkk] = Ev;
        else S.E[par].e1m[MTJ - 1][rkk] = Ev;
      } else {
        if (rs == 0) S.E[par].e2p[rhj_ - 1][0] = Ev;
        else S.E[par].e2m[rhj_ - 1][MTK - 1] = Ev;
      }
      Tmr = Tcr;
    }
    if (!LAST) {
      cp_async_wait<0>();
      mbar_wait(&S.bar, phase);
      phase ^= 1u;
      __syncthreads();
    }
  };
#pragma unroll 1
  for (int t = i0; t < iend; ++t) step(t, std::false_type{});
  step(iend, std::true_type{});
  epi.finish(g);
}

}  // namespace pc
