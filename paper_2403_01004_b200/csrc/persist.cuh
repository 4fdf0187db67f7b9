// Persistent cycle kernel for SMALL grids (C1-sized: L2-resident, a few
// microseconds of work per pass).  On those grids the host-driven cycle loop
// is latency-bound: per PTL cycle four or five launches and a host round trip
// for the PTL decision cost ~60 us against ~20 us of kernel time.  Here ONE
// cooperative launch runs the whole cycle_operator on the device:
//
//   per cycle:  y0 = F(u0) + |F| argmax (grid-stride) -> grid barrier ->
//               block 0: global argmax, the <= 6 ncomp PTL pairs, the cycle
//               decision (clamp to the floor, remaining time), s and the
//               coefficient rows (sts.cuh: the host's own expressions) and the
//               CycleReport row -> grid barrier -> stage 1 -> barrier ->
//               stages 2..s, one barrier each.
//
// Every per-node expression is the one of the regular kernels (ScalarOp::F,
// k_stage1, k_stage, k_ptl_pairs) and every decision the one of pc_cycle, so
// fields, cycles and stage counts are bitwise those of the host-driven path
// (and of the oracle).  Values written inside the launch are read with
// L2-coherent loads (__ldcg) after a release/acquire grid barrier, never
// through the read-only path.
#pragma once
#include "kernels.cuh"
#include "sts.cuh"

namespace pc {

constexpr int kPersistThreads = 256;
constexpr int kPersistSMax = 4096;  // coefficient rows kept on the device

struct CycleDev {
  // inputs
  double remaining, dtE, floor_dt, eps_rel;
  int kind, make_odd, use_ptl, rec_cap;
  long long max_cycles;
  // state
  long long cyc;
  int status;   // 0 running, 1 done, 2 blow-up (stage in bad), 3 cycle cap, 4 s too large
  int bad;      // min non-finite stage of the current step (0x7f7f7f7f = none)
  int s, cur;   // stage count of the current step; buffer set holding u0
  // the barrier words each on their own 128-byte line, away from the state
  // block 0 rewrites every cycle (spinning readers and arriving atomics do
  // not share a line with each other or with it)
  alignas(128) unsigned bar_count;
  alignas(128) unsigned bar_gen;
  alignas(128) double tab[5 * kPersistSMax];
};

struct CgVal {  // coherent (L2) reads of values written inside the launch
  const double* p[3];
  __device__ __forceinline__ double operator()(int c, int64_t o, int, int, int) const { return __ldcg(p[c] + o); }
};

__device__ __forceinline__ void grid_barrier(CycleDev* cs) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = &cs->bar_gen;
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(&cs->bar_count, 1u) == gridDim.x - 1) {
      cs->bar_count = 0;
      __threadfence();
      atomicAdd(&cs->bar_gen, 1u);
    } else {
      // plain poll: 1.5 % faster per C1 step than a __nanosleep backoff
      while (*gen == g0) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

struct PersistBufs {
  double* set[3][3];  // buffer set x component: set 0 = the field, 1 / 2 = workspaces
  double* y0[3];
  double* pv;         // per-block argmax partials
  long long* pi;
};

template <int NC>
__global__ void __launch_bounds__(kPersistThreads) k_cycle_small(GridDev g, ScalarOp op, PersistBufs B, CycleDev* cs,
                                                                 pc_cycle_record* rec) {
  __shared__ double shv[kPersistThreads / 32];
  __shared__ long long shi[kPersistThreads / 32];
  __shared__ double sh_pair[32];
  int cur = 0;
  for (;;) {
    // ---- loop control (every thread reads the same values after a barrier)
    {
      const volatile CycleDev* v = cs;
      if (!(v->remaining > 0.0)) break;
      if (v->cyc >= v->max_cycles) {
        if (blockIdx.x == 0 && threadIdx.x == 0) cs->status = 3;
        break;
      }
    }
    // ---- y0 = F(u0), local |F| argmax
    {
      CgVal val{{B.set[cur][0], B.set[cur][1], B.set[cur][2]}};
      ArgMax best{-1.0, 0x7fffffffffffffffLL};
      PC_FOR_NODES(g, i, j, k) {
        double out[3];
        op.F(g, val, i, j, k, out);
        const int64_t o = off3(g, i, j, k);
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          B.y0[q][o] = out[q];
          best = am_better(best, ArgMax{fabs(out[q]), aos_index(g, i, j, k, q, NC)});
        }
      }
      best = block_argmax<kPersistThreads>(best, shv, shi);
      if (threadIdx.x == 0) {
        B.pv[blockIdx.x] = best.v;
        B.pi[blockIdx.x] = best.i;
      }
    }
    grid_barrier(cs);
    // ---- block 0: global argmax, PTL pairs, the cycle decision
    if (blockIdx.x == 0) {
      ArgMax r{-1.0, 0x7fffffffffffffffLL};
      for (int q = threadIdx.x; q < (int)gridDim.x; q += kPersistThreads)
        r = am_better(r, ArgMax{__ldcg(B.pv + q), __ldcg(B.pi + q)});
      r = block_argmax<kPersistThreads>(r, shv, shi);
      if (threadIdx.x == 0) {
        shv[0] = r.v;
        shi[0] = r.i;
      }
      __syncthreads();
      const double fmax = shv[0];
      const long long kid = shi[0];
      if (threadIdx.x < 32) {  // k_ptl_pairs, coherent reads
        const double thr = cs->eps_rel * fmax;
        const long long pt = kid / NC;
        const int kk = (int)(pt % g.n2);
        const long long t2 = pt / g.n2;
        const int kj = (int)(t2 % g.n1);
        const int ki = (int)(t2 / g.n1) - g.i0g;
        double best = INFINITY;
        const int t = threadIdx.x;
        if (t < 6 * NC) {
          const int dirn = t / NC, q = t % NC;
          const int a = dirn / 2, d = (dirn & 1) ? 1 : -1;
          bool ok;
          const int co[3] = {ki, kj, kk};
          int x = nbax(g, a, co[a], d, ok);
          if (ok) {
            int ni = a == 0 ? x : ki, nj = a == 1 ? x : kj, nk = a == 2 ? x : kk;
            const int64_t ok0 = off3(g, ki, kj, kk), on = off3(g, ni, nj, nk);
            double du = __ldcg(B.set[cur][q] + ok0) - __ldcg(B.set[cur][q] + on);
            double dF = __ldcg(B.y0[q] + ok0) - __ldcg(B.y0[q] + on);
            if (du != 0.0 && fabs(dF) > thr && du * dF < 0.0) best = -du / dF;
          }
        }
        for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_down_sync(0xffffffffu, best, o));
        if (t == 0) sh_pair[0] = best;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const double ptl_min = sh_pair[0];
        int limited = 0;
        double ptl = INFINITY;
        if (cs->use_ptl) {
          limited = isfinite(ptl_min) ? 1 : 0;
          ptl = limited ? ptl_min : INFINITY;
        }
        const double remaining = cs->remaining;
        double dt;
        if (!limited) {
          dt = remaining;
        } else {
          dt = ptl >= cs->floor_dt ? ptl : cs->floor_dt;
          if (dt >= remaining) dt = remaining;
        }
        const int s = sts_count_hd(cs->kind, dt, cs->dtE, cs->make_odd);
        if (s > kPersistSMax || !sts_rows_hd(cs->kind, s, dt, cs->tab)) {
          cs->status = 4;
          cs->s = 0;
        } else {
          cs->s = s;
        }
        cs->bad = 0x7f7f7f7f;
        const long long cyc = cs->cyc + 1;
        cs->cyc = cyc;
        if (cyc - 1 < cs->rec_cap) {
          pc_cycle_record& R = rec[cyc - 1];
          R.cycle = cyc;
          R.dt = dt;
          R.ptl_raw = limited ? ptl : INFINITY;
          R.relres = 0.0;
          R.limited = limited;
          R.iters = s;
        }
        if (dt == remaining) cs->remaining = 0.0;
        else cs->remaining = remaining - dt;
        __threadfence();
      }
    }
    grid_barrier(cs);
    const int s = ((const volatile CycleDev*)cs)->s;
    if (s == 0) break;  // status 4 (set by block 0)
    // ---- stage 1: u1 = u0 + mut1 dt y0 (pinned: u0)
    const int n1 = (cur + 1) % 3, n2 = (cur + 2) % 3;
    {
      const double mtdt = __ldcg(cs->tab + 3);
      PC_FOR_NODES(g, i, j, k) {
        const int64_t o = off3(g, i, j, k);
        const bool pin = pinned(g, i, j, k);
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          const double a = __ldcg(B.set[cur][q] + o);
          const double v = pin ? a : a + mtdt * __ldcg(B.y0[q] + o);
          B.set[n1][q][o] = v;
          if (!isfinite(v)) atomicMin(&cs->bad, 1);
        }
      }
    }
    grid_barrier(cs);
    // ---- stages 2..s (the output takes the buffer of u_{k-2}, pointwise safe)
    int um1 = n1, um2 = cur, out = n2;
    for (int kst = 2; kst <= s; ++kst) {
      const double* rw = cs->tab + 5 * (kst - 1);
      const double mu = __ldcg(rw), nu = __ldcg(rw + 1), kap = __ldcg(rw + 2), mtdt = __ldcg(rw + 3),
                   gtdt = __ldcg(rw + 4);
      CgVal val{{B.set[um1][0], B.set[um1][1], B.set[um1][2]}};
      PC_FOR_NODES(g, i, j, k) {
        double Fk[3];
        op.F(g, val, i, j, k, Fk);
        const int64_t o = off3(g, i, j, k);
        const bool pin = pinned(g, i, j, k);
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          const double a0 = __ldcg(B.set[cur][q] + o);
          double v = ((((mu * __ldcg(B.set[um1][q] + o)) + (nu * __ldcg(B.set[um2][q] + o))) + (kap * a0)) +
                      (mtdt * Fk[q])) + (gtdt * __ldcg(B.y0[q] + o));
          v = pin ? a0 : v;
          B.set[out][q][o] = v;
          if (!isfinite(v)) atomicMin(&cs->bad, kst);
        }
      }
      grid_barrier(cs);
      // rotate as sts_stages: u_{k-1} -> u_{k-2}, u_k -> u_{k-1}, the next
      // output goes to the buffer that held u_{k-1}
      const int prev = um1;
      um1 = out;
      out = prev;
      um2 = prev;
    }
    cur = um1;
    if (((const volatile CycleDev*)cs)->bad != 0x7f7f7f7f) {
      if (blockIdx.x == 0 && threadIdx.x == 0) cs->status = 2;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    cs->cur = cur;
    if (cs->status == 0) cs->status = 1;
  }
}

}  // namespace pc
