// TMA-staged variant of the r-marching Spitzer kernel (K3/K4/K7), used when
// the grid allows it (phi periodic with n2 % 32 == 0, theta not periodic --
// every spherical grid of the configs); k_aligned_march (cp.async) is the
// general fallback.  Same arithmetic, same schedule, bitwise-identical output.
//
// Per plane lane 0 of three warps without halo-ring work issues the bulk
// tensor copies (cp.async.bulk.tensor, completion counted on one mbarrier;
// warp 7: T and the expect_tx, warp 6: operands and rows, warp 5: beta): for
// T and each beta component a
// 32 x 18 main box (256-byte rows, phi-aligned) plus two 2 x 18 halo strips
// whose phi coordinates wrap across the periodic seam; the epilogue operands
// as 32 x 16 boxes; the per-(r, theta) metric records (iL2[6], wo01[4],
// iVal2, pad: one interleaved [n0+2][n1][12] table built at grid creation) as
// one 12 x 18 box (slot 11 carries the aligned-volume row factor Val2 for
// the PCG inner-product weight).  Rows outside the theta range are zero-filled by the TMA
// unit: they only ever meet an inverse edge length of 0 (no flux through the
// pole faces), exactly as the clamped values of the oracle do, and their
// metric records are never read.  No per-thread async copies remain.
//
// Per-node overheads kept off the hot loop: the 1/rho division exists only in
// the RHO instantiation (rho prefetched one plane ahead into a register), the
// flux-exchange stores are unconditional (padded FluxX layout), and the
// epilogue folds its non-finite test into a flag reduced once per thread.
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
constexpr int kIssuer = MNT - 32;  // lane 0 of the last warp: prologue copies, per-plane T + expect_tx

struct TmaMaps {
  CUtensorMap T;     // stage input, box {32, 18, 1}
  CUtensorMap TS;    // same tensor, strip box {2, 18, 1}
  CUtensorMap B[3];  // beta, box {32, 18, 1}
  CUtensorMap BS[3]; // beta strips
  CUtensorMap O[3];  // epilogue operands, box {32, 16, 1}
  CUtensorMap RW;    // row records [n0+2][n1][12], box {12, 18, 1}
  CUtensorMap P[2], PS[2];  // fused PCG matvec: p_old and the Jacobi diagonal d (T = the residual r)
};

// Epilogues with FUSEP: the march stages r, p_old and d instead of its input
// and forms the PCG search direction p = r / (1 + dt d) + beta p_old (the
// Jacobi preconditioner applied on the fly, k_pcg_pupdatev's expression) into
// the input slot as each plane lands; the epilogue gets p as the node value
// (d here is the stored inverse diagonal dinv = 1 / (1 + dt d): p = r dinv + beta p_old)
template <class E, class = void>
struct fusep_of : std::false_type {};
template <class E>
struct fusep_of<E, std::void_t<decltype(E::FUSEP)>> : std::integral_constant<bool, E::FUSEP> {};
// Epilogues with FUSE1 (EpiStageA12 here, SEpiStage12 in the 7-point
// marches): the march stages u0 into the input slot and y0 beside it, and
// forms u1 = u0 + mut1 dt y0 in place (pinned nodes keep u0: k_stage1's
// expression) as each plane lands
template <class E, class = void>
struct fuse1_of : std::false_type {};
template <class E>
struct fuse1_of<E, std::void_t<decltype(E::FUSE1)>> : std::integral_constant<bool, E::FUSE1> {};

constexpr int RW = 12;  // metric row record: iL2[6], wo01[4], iVal2, pad (16-byte aligned pairs)
constexpr int RSLOT = 224;  // one plane of row records (18 x 12) padded to a 128-byte multiple
constexpr unsigned kRowBytes = (unsigned)(MHJ * RW) * 8u;
struct TmaSmem {
  double T[TSL][XA];
  double B[BSL][3][XA];
  double EO[2][3][XO];
  FluxX E[2];
  double rowt[RSL][RSLOT];
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

// RHO: 0 no density, 1 a density field (prefetched per node), 2 a radial
// density (rho(i, j, k) == rho(i): one uniform per-plane value, no HBM stream)
template <class Epi, int RHO>
__global__ void __launch_bounds__(MNT, 2) k_aligned_tma(GridDev g, AlignedOp op, const __grid_constant__ TmaMaps maps,
                                                        Epi epi, int R, int zsel, const int* skip) {
  extern __shared__ __align__(128) unsigned char tma_smem[];
  // bulk-tensor destinations must be 128-byte aligned: align the dynamic base
  // (static epilogue scratch may precede it); the launch adds 128 bytes
  TmaSmem& S = *reinterpret_cast<TmaSmem*>(tma_smem + ((128u - (smem_u32(tma_smem) & 127u)) & 127u));
  if (skip && *skip) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * MTK + tx;
  const int k0 = blockIdx.x * MTK, j0 = blockIdx.y * MTJ, i0 = chunk_of(zsel) * R;
  const int iend = min(i0 + R, g.n0);
  const int kg = k0 + tx;
  const int kL = k0 == 0 ? g.n2 - 2 : k0 - 2;     // strip of columns k0-2, k0-1
  const int kR = k0 + MTK == g.n2 ? 0 : k0 + MTK;  // strip of columns k0+32, k0+33

  ColT col;
  load_col(g, kg, col);
#pragma unroll
  for (int q = 0; q < 2; ++q) col.il1[q] = launder(col.il1[q]);
  col.w2[0] = launder(col.w2[0]);
  col.w2[1] = launder(col.w2[1]);
  col.ivg = launder(col.ivg);
  const bool pin_k = (g.pin_lo2 && kg == 0) || (g.pin_hi2 && kg == g.n2 - 1);
  const double valg = Epi::NEEDS_W ? launder(__ldg(g.Valg + kg)) : 0.0;
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

  // ring node of this thread: each ring group is one whole warp, so every
  // warp runs one uniform flux variant (no divergence):
  //   warp 0: row j0-1 (E_{1,+}), warp 1: row j0+16 (E_{1,-}),
  //   warp 2 lanes 0-15: column k0-1 (E_{2,+}), warp 3 lanes 0-15: column k0+32 (E_{2,-});
  // the TMA issue runs on warp 7 (no ring work)
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
  } else if (tid < 4 * MTK && (tid & 31) < MTJ) {
    const int q = tid & 31;
    ra = 2;
    rs = tid < 3 * MTK ? 0 : 1;
    rhj_ = 1 + q;
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
  // flux-exchange slot the ring value goes to (padded FluxX: every slot exists)
  int ring_slot = 0;
  if (ra == 1) ring_slot = rs == 0 ? (int)(&S.E[0].e1p[0][rkk] - &S.E[0].e1p[0][0])
                                   : (int)(&S.E[0].e1m[MTJ][rkk] - &S.E[0].e1p[0][0]);
  if (ra == 2) ring_slot = rs == 0 ? (int)(&S.E[0].e2p[rhj_ - 1][0] - &S.E[0].e1p[0][0])
                                   : (int)(&S.E[0].e2m[rhj_ - 1][MTK] - &S.E[0].e1p[0][0]);
  bool ring_on = false;
  if (ra >= 0) {
    bool rjo, rko;
    const int gj = j0 - 1 + rhj_, gk = ra == 1 ? k0 + rkk : (rs == 0 ? k0 - 1 : k0 + MTK);
    map_j(g, gj, rjo);
    map_k(g, gk, rko);
    ring_on = rjo && rko && (ra == 1 ? true : (gj < g.n1));
  }
  // an interior tile: every own node inside, every ring node on, no pinned theta rows
  const bool full = j0 > 0 && j0 + MTJ < g.n1 && !g.pin_lo1 && !g.pin_hi1;

  const int onode0 = (j0 + ty) * g.n2 + kg;
  auto jn = [&](int n) { return j0 + ty + n * MTY; };
  auto onode = [&](int n) { return onode0 + n * MTY * g.n2; };

  // rotating slots (roles advance by one plane per iteration)
  double* sTm1 = S.T[0];  // plane t-1 (refilled with t+2 at iteration t)
  double* sT = S.T[1];    // plane t
  double* sTp = S.T[2];   // plane t+1
  double* sB = S.B[1][0];   // beta of plane t
  double* sBn = S.B[0][0];  // beta of plane t+1 (refilled at iteration t)
  double* rM = S.rowt[0];   // metric rows of planes t-1, t, t+1
  double* rC = S.rowt[1];
  double* rN = S.rowt[2];
  constexpr bool FP1 = fuse1_of<Epi>::value;
  // epilogue operands of plane t (landing), t-1 (read); FUSE1 (two operands)
  // packs the two slots at a stride of two boxes and stages y0 behind them
  static_assert(!FP1 || (Epi::NOPS == 2 && 4 * XO + XA <= 2 * 3 * XO), "FUSE1 stages y0 behind two operand slots");
  double* eW = S.EO[0][0];
  double* eR = FP1 ? S.EO[0][0] + 2 * XO : S.EO[1][0];
  double* rawy = S.EO[0][0] + 4 * XO;
  FluxX* Ew = &S.E[0];      // flux exchange of plane t (write), t-1 (read)
  FluxX* Er = &S.E[1];

  // (issuer thread only)
  auto tma_arr = [&](double* dst, const CUtensorMap* mm, const CUtensorMap* ms, int p) {
    const int z = plane_map(g, p).mem + 1;
    tma3(dst, mm, k0, j0 - 1, z, &S.bar);
    tma3(dst + XM, ms, kL, j0 - 1, z, &S.bar);
    tma3(dst + XM + XS, ms, kR, j0 - 1, z, &S.bar);
  };
  // the stage input of plane p into its slot: a TMA box, or (FUSEP) the raw
  // r, p_old, d boxes into the staging area the unused epilogue-operand slots
  // provide; form_p turns them into p after the plane's barrier phase
  constexpr bool FP = fusep_of<Epi>::value;
  static_assert(!FP || (Epi::NOPS == 0 && 3 * XA <= 2 * 3 * XO), "FUSEP stages r, p_old, d in the operand slots");
  double* raw = &S.EO[0][0][0];
  auto issue_T = [&](double* dst, int p) {
    if constexpr (FP) {
      tma_arr(raw, &maps.T, &maps.TS, p);
      tma_arr(raw + XA, &maps.P[0], &maps.PS[0], p);
      tma_arr(raw + 2 * XA, &maps.P[1], &maps.PS[1], p);
    } else if constexpr (FP1) {
      tma_arr(dst, &maps.T, &maps.TS, p);  // u0
      tma_arr(rawy, &maps.P[0], &maps.PS[0], p);  // y0
    } else {
      tma_arr(dst, &maps.T, &maps.TS, p);
    }
  };
  constexpr unsigned kTBytes = (FP ? 3u : (FP1 ? 2u : 1u)) * kArrBytes;
  // FUSE1: this thread's staged elements e = tid + q MNT (q < 3) that get
  // u1 = u0 + mut1 dt y0 -- real slots (strip padding stays unread) whose
  // theta row and phi column are not pinned -- as a mask fixed per block
  unsigned fmask = 0u;
  if constexpr (FP1) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int e = tid + q * MNT;
      if (e >= XA) continue;
      int row, kc;
      bool real = true;
      if (e < XM) {
        row = e / MTK;
        kc = k0 + (e - row * MTK);
      } else {
        const int sx = (e - XM) / XS, ix = (e - XM) - sx * XS;
        real = ix < MHJ * 2;
        row = ix >> 1;
        kc = (sx == 0 ? kL : kR) + (ix & 1);
      }
      const int jg = j0 - 1 + row;
      const bool pin = (g.pin_lo1 && jg == 0) || (g.pin_hi1 && jg == g.n1 - 1) || (g.pin_lo2 && kc == 0) ||
                       (g.pin_hi2 && kc == g.n2 - 1);
      if (real && !pin) fmask |= 1u << q;
    }
  }
  auto form_p = [&](double* dst, int p) {
    if constexpr (FP1) {  // u1 = u0 + mut1 dt y0 of plane p, pinned nodes keep u0 (k_stage1)
      const int ig = p + g.i0g;
      if ((g.pin_lo0 && ig == 0) || (g.pin_hi0 && ig == g.n0g - 1)) return;
      const double mt = epi.mt1;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int e = tid + q * MNT;
        if (fmask & (1u << q)) dst[e] = dst[e] + mt * rawy[e];
      }
    }
    if constexpr (FP) {
      const double beta = epi.st->beta;
      for (int e = tid; e < XA; e += MNT) {
        const bool real = e < XM || (e - XM) % XS < MHJ * 2;  // (strip padding slots stay unread)
        if (real) {
          const double z = raw[e] * raw[2 * XA + e];  // r dinv
          dst[e] = z + beta * raw[XA + e];
        }
      }
    }
  };
  auto issue_B = [&](double* dst, int p) {
#pragma unroll
    for (int q = 0; q < 3; ++q) tma_arr(dst + q * XA, &maps.B[q], &maps.BS[q], p);
  };
  auto issue_ops = [&](double* dst, int p) {
#pragma unroll
    for (int q = 0; q < Epi::NOPS; ++q) tma3(dst + q * XO, &maps.O[q], k0, j0, p + 1, &S.bar);
  };
  auto issue_rows = [&](double* dst, int p) { tma3(dst, &maps.RW, 0, j0 - 1, plane_map(g, p).row + 1, &S.bar); };

  // ---- prologue: T(i0-1..i0+1), beta and row records of (i0-1, i0)
  __syncthreads();  // barrier initialised
  unsigned phase = 0;
  if constexpr (FP || FP1) {  // one staging area: the three input planes one after the other
    double* slots[3] = {sTm1, sT, sTp};
#pragma unroll 1
    for (int q = 0; q < 3; ++q) {
      if (tid == kIssuer) {
        if (q > 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&S.bar, kTBytes + (q == 0 ? 6u * kArrBytes + 2u * kRowBytes : 0u));
        issue_T(slots[q], i0 - 1 + q);
        if (q == 0) {
          issue_B(sBn, i0 - 1);
          issue_B(sB, i0);
          issue_rows(rM, i0 - 1);
          issue_rows(rC, i0);
        }
      }
      mbar_wait(&S.bar, phase);
      phase ^= 1u;
      form_p(slots[q], i0 - 1 + q);
      __syncthreads();
    }
  } else {
    if (tid == kIssuer) {
      mbar_expect_tx(&S.bar, 9u * kArrBytes + 2u * kRowBytes);
      tma_arr(sTm1, &maps.T, &maps.TS, i0 - 1);
      tma_arr(sT, &maps.T, &maps.TS, i0);
      tma_arr(sTp, &maps.T, &maps.TS, i0 + 1);  // iend >= i0 + 1
      issue_B(sBn, i0 - 1);
      issue_B(sB, i0);
      issue_rows(rM, i0 - 1);
      issue_rows(rC, i0);
    }
    mbar_wait(&S.bar, phase);
    phase ^= 1u;
    __syncthreads();
  }

  auto run = [&](auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
    bool inside[NPT], pin_j[NPT];
    int oc[NPT], opm[NPT], opp[NPT];
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      const int hr = ty + n * MTY + 1;
      inside[n] = FULL || jn(n) < g.n1;
      pin_j[n] = !FULL && ((g.pin_lo1 && jn(n) == 0) || (g.pin_hi1 && jn(n) == g.n1 - 1));
      oc[n] = hr * MTK + tx;
      opm[n] = tx > 0 ? oc[n] - 1 : XM + hr * 2 + 1;
      opp[n] = tx < MTK - 1 ? oc[n] + 1 : XM + XS + hr * 2;
    }
    const bool ron = FULL ? (ra >= 0) : (ra >= 0 && ring_on);

    double Tm[NPT], Tc[NPT], qa[NPT], qb[NPT], ownp[NPT];
    // rho of the own nodes of the plane being finalised: loaded one plane
    // ahead into the same register right after its previous use (no move of a
    // pending load, no dependent global load on the finalisation path)
    double rr[NPT];
#pragma unroll
    for (int n = 0; n < NPT; ++n) rr[n] = 1.0;
    double Tmr = 0.0;
    {  // E_{0,+}(i0 - 1)
      const bool ex = plane_map(g, i0 - 1).exists;
#pragma unroll
      for (int n = 0; n < NPT; ++n) {
        Tm[n] = sTm1[oc[n]];
        Tc[n] = sT[oc[n]];
        qa[n] = 0.0;
        qb[n] = 0.0;
        ownp[n] = 0.0;
        if (ex && inside[n]) {
          const double Tn[3][2] = {{Tc[n], Tm[n]}, {sTm1[oc[n] + MTK], sTm1[oc[n] - MTK]},
                                   {sTm1[opp[n]], sTm1[opm[n]]}};
          const double bv[3] = {sBn[oc[n]], sBn[XA + oc[n]], sBn[2 * XA + oc[n]]};
          double E[3][2];
          node_E_rows<0, 0>(Tm[n], Tn, bv, rM + (ty + n * MTY + 1) * RW, col.il1, col.w2, E);
          qb[n] = E[0][0];
        }
      }
      if (ra >= 0) Tmr = sTm1[ro_c];
    }
    // the prologue reads of the plane i0-1 slots (T, beta, rows) finish before
    // the first step's bulk copies refill them
    __syncthreads();
    // global offset of own node 0 in the plane being finalised (t - 1)
    int64_t pofs = (int64_t)(i0 - 1) * g.plane + onode0;
    const int64_t nstride = (int64_t)MTY * g.n2;

    // one plane: fluxes of plane t, finalisation of plane t-1
    auto step = [&](int t, auto first_tag, auto last_tag) {
      constexpr bool FIRST = decltype(first_tag)::value;
      constexpr bool LAST = decltype(last_tag)::value;
      if (!LAST) {
        if (tid == kIssuer) {
          const bool t2 = t + 2 <= iend;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&S.bar, (t2 ? kTBytes : 0u) + 3u * kArrBytes + (unsigned)Epi::NOPS * kOpBytes +
                                     kRowBytes);
          if (t2) issue_T(sTm1, t + 2);
          if (op.tma_split < 2) issue_B(sBn, t + 1);
          if (op.tma_split == 0) {
            issue_ops(eW, t);
            issue_rows(rN, t + 1);
          }
        }
        // the per-plane bulk copies are issued by lane 0 of three warps without
        // halo-ring work: warp 7 (T, and the expect_tx of the whole plane),
        // warp 6 (operand and row boxes), warp 5 (beta boxes).  Their bytes are
        // all in warp 7's expect_tx and the phase cannot complete before that
        // arrival.  One issuer serialised ~16 copies per plane behind one
        // warp's compute: C5 7.00 -> 7.28e10, C3 6.92 -> 7.23e10 with three
        // (profiles/r01_tma_issue_split.txt; PC_TMA_SPLIT=0/1 keep one / two)
        if (op.tma_split >= 1 && tid == kIssuer - 32) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue_ops(eW, t);
          issue_rows(rN, t + 1);
        }
        if (op.tma_split == 2 && tid == kIssuer - 64) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue_B(sBn, t + 1);
        }
      }
      const bool exists = LAST ? plane_map(g, t).exists : true;
      const int tf = t - 1;
      const double rpl = (RHO == 2 && !FIRST) ? __ldg(op.rho_r + tf) : 1.0;  // radial density of plane tf
      const double nsp = (RHO == 2 && !FIRST) ? __ldg(op.nsc_r + tf) : op.npref;  // its scale 0 - pref / rho
      const int ig = tf + g.i0g;
      const bool pin_i = (g.pin_lo0 && ig == 0) || (g.pin_hi0 && ig == g.n0g - 1);
#pragma unroll
      for (int n = 0; n < NPT; ++n) {
        const int r = ty + n * MTY;
        const int jr = r + 1;
        double E[3][2];
        double Tp = 0.0;
        if (!LAST) Tp = sTp[oc[n]];
        if ((FULL && !LAST) || (exists && inside[n])) {
          const double Tn[3][2] = {{Tp, Tm[n]}, {sT[oc[n] + MTK], sT[oc[n] - MTK]}, {sT[opp[n]], sT[opm[n]]}};
          const double bv[3] = {sB[oc[n]], sB[XA + oc[n]], sB[2 * XA + oc[n]]};
          if (!LAST) node_E_rows<-1, 0>(Tc[n], Tn, bv, rC + jr * RW, col.il1, col.w2, E);
          else node_E_rows<0, 1>(Tc[n], Tn, bv, rC + jr * RW, col.il1, col.w2, E);
        } else {
#pragma unroll
          for (int a = 0; a < 3; ++a) E[a][0] = E[a][1] = 0.0;
        }
        if (!LAST) {  // publish the in-plane fluxes (padded slots: no conditions)
          Ew->e1p[r + 1][tx] = E[1][0];
          Ew->e1m[r][tx] = E[1][1];
          Ew->e2p[r][tx + 1] = E[2][0];
          Ew->e2m[r][tx] = E[2][1];
        }
        if (!FIRST && inside[n]) {
          const double nbr = (Er->e1p[r][tx] - Er->e1m[r + 1][tx]) + (Er->e2p[r][tx] - Er->e2m[r][tx + 1]);
          const double G = (qa[n] - E[0][1]) + (ownp[n] + nbr);
          const double iv = rM[jr * RW + 10] * col.ivg;
          const int64_t of = pofs + n * nstride;
          double f;
          if constexpr (RHO == 1) f = (G * iv) * (0.0 - (op.pref / rr[n]));
          else f = (G * iv) * nsp;
          const bool pin = pin_i || pin_j[n] || pin_k;
          if (pin) f = 0.0;
          double ov[Epi::NOPS > 0 ? Epi::NOPS : 1];
#pragma unroll
          for (int q = 0; q < Epi::NOPS; ++q) ov[q] = eR[q * XO + r * MTK + tx];
          double W = 0.0;  // inner-product weight rho V = rho * (Val2(row) * Valg(k)) (record slot 11)
          if constexpr (Epi::NEEDS_W) {
            W = rM[jr * RW + 11] * valg;
            if constexpr (RHO == 1) W = rr[n] * W;
            if constexpr (RHO == 2) W = rpl * W;
          }
          epi(n, g, tf, jn(n), kg, of, f, Tm[n], pin, ov, W);
        }
        if (!LAST) {
          if constexpr (RHO == 1) {
            if (inside[n]) rr[n] = __ldg(op.rho + pofs + g.plane + n * nstride);
          }
          ownp[n] = ((E[0][1] - E[0][0]) + (E[1][1] - E[1][0])) + (E[2][1] - E[2][0]);
          qa[n] = qb[n];
          qb[n] = E[0][0];
          Tm[n] = Tc[n];
          Tc[n] = Tp;
        }
      }
      if constexpr (has_plane_end<Epi>::value) {
        if (!FIRST) epi.plane_end(tf);
      }
      // ---- halo ring of plane t (warp-uniform variant)
      if (!LAST && ra >= 0) {
        const double Tcr = sT[ro_c];
        const double Tpr = sTp[ro_c];
        double Ev = 0.0;
        if (ron) {
          const double Tn[3][2] = {{Tpr, Tmr}, {sT[ro_tp], sT[ro_tm]}, {sT[ro_pp], sT[ro_pm]}};
          const double bv[3] = {sB[ro_c], sB[XA + ro_c], sB[2 * XA + ro_c]};
          double E[3][2];
          const double* rw = rC + rhj_ * RW;
          if (ra == 1) {
            if (rs == 0) {
              node_E_rows<1, 0>(Tcr, Tn, bv, rw, col.il1, col.w2, E);
              Ev = E[1][0];
            } else {
              node_E_rows<1, 1>(Tcr, Tn, bv, rw, col.il1, col.w2, E);
              Ev = E[1][1];
            }
          } else {
            const double* cs = S.ringcol[rs];
            const double il1[2] = {cs[4], cs[5]};
            const double w2[2] = {cs[6], cs[7]};
            if (rs == 0) {
              node_E_rows<2, 0>(Tcr, Tn, bv, rw, il1, w2, E);
              Ev = E[2][0];
            } else {
              node_E_rows<2, 1>(Tcr, Tn, bv, rw, il1, w2, E);
              Ev = E[2][1];
            }
          }
        }
        (&Ew->e1p[0][0])[ring_slot] = Ev;
        Tmr = Tcr;
      }
      if (!LAST) {
        mbar_wait(&S.bar, phase);
        phase ^= 1u;
        if constexpr (FP || FP1) {
          if (t + 2 <= iend) form_p(sTm1, t + 2);  // plane t+2 into the slot that becomes sTp
        }
        __syncthreads();
        pofs += g.plane;
        // advance the slot roles by one plane
        double* tt = sTm1;
        sTm1 = sT;
        sT = sTp;
        sTp = tt;
        tt = sB;
        sB = sBn;
        sBn = tt;
        tt = rM;
        rM = rC;
        rC = rN;
        rN = tt;
        tt = eW;
        eW = eR;
        eR = tt;
        FluxX* ft = Ew;
        Ew = Er;
        Er = ft;
      }
    };
    step(i0, std::true_type{}, std::false_type{});
#pragma unroll 1
    for (int t = i0 + 1; t < iend; ++t) step(t, std::false_type{}, std::false_type{});
    step(iend, std::false_type{}, std::true_type{});
  };
  if (full) run(std::true_type{});
  else run(std::false_type{});
  epi.finish(g);
}

}  // namespace pc
