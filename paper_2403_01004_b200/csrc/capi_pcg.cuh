// paracycle_b200 C ABI, part of the single translation unit capi.cu (included
// there in order; relies on the declarations of the parts before it).
//
// C ABI: device-driven PCG (Jacobi and r-line block-Jacobi preconditioners)
// and the backward-Euler step
#pragma once

// ------------------------------------------------------------------ PCG
// the plane-ordered reduction scratch of a solve with S slots per plane
// (kernels.cuh PlaneRed: the sums are independent of the r-slab split)
static int plane_red(pc_grid* g, int S, PlaneRed& pr) {
  pc_ctx* c = g->ctx;
  const size_t need = (size_t)S * (size_t)g->g.n0;
  if (need > c->pslot_cap) {
    cudaFree(c->pslot[0]);
    cudaFree(c->pslot[1]);
    c->pslot[0] = c->pslot[1] = nullptr;
    c->pslot_cap = 0;
    CUDA_TRY(cudaMalloc(&c->pslot[0], need * sizeof(double)));
    CUDA_TRY(cudaMalloc(&c->pslot[1], need * sizeof(double)));
    c->pslot_cap = need;
  }
  const int n0g = g->g.n0g;
  if (n0g > c->pvec_n) {
    cudaFree(c->pvec);
    cudaFree(c->pvec_all);
    c->pvec = c->pvec_all = nullptr;
    c->pvec_n = 0;
    CUDA_TRY(cudaMalloc(&c->pvec, 2 * (size_t)n0g * sizeof(double)));
    CUDA_TRY(cudaMalloc(&c->pvec_all, 2 * (size_t)n0g * sizeof(double)));
    c->pvec_n = n0g;
    c->pvec_n0g = -1;
  }
  if (c->pvec_n0g != n0g || c->pvec_i0g != g->g.i0g) {  // other ranks' entries must be exactly 0
    CUDA_TRY(cudaMemsetAsync(c->pvec, 0, 2 * (size_t)n0g * sizeof(double), c->s));
    c->pvec_n0g = n0g;
    c->pvec_i0g = g->g.i0g;
  }
  pr.slot[0] = c->pslot[0];
  pr.slot[1] = c->pslot[1];
  pr.S = S;
  pr.vec = c->pvec;
  pr.n0g = n0g;
  pr.i0g = g->g.i0g;
  return PC_OK;
}
// stages 2 and 3 of a PCG reduction: per-plane sums, then (one rank) the
// fixed-order sum over the planes and the scalar recurrence in the last
// block, or (r-slabs) an allreduce of the per-plane vector and the same
// finish in k_pcg_fin -- bitwise the one-rank result
static int plane_sums(pc_grid* g, const PlaneRed& pr, int nsum, int mode, int keep, bool split, double tol, int it) {
  pc_ctx* c = g->ctx;
  k_plane_sums<<<g->g.n0, kThreads, 0, c->s>>>(pr, nsum, mode, split ? 0 : 1, keep, tol, it, c->counter, c->pcg);
  c->st.launches++;
  TRY(check_launch("k_plane_sums"));
  if (!split) return PC_OK;
  TRY(allreduce_d2(c, c->pvec, c->pvec_all, 2 * (size_t)pr.n0g, nccl::kSum));
  k_pcg_fin<<<1, kThreads, 0, c->s>>>(c->pcg, c->pvec_all, pr.n0g, mode, keep, tol, it);
  c->st.launches++;
  return check_launch("k_pcg_fin");
}

// ---- r-line preconditioner
static int line_prepare(pc_op* op, double dt, const double* adiag, Work& Lf) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  if (!op->line_valid) {
    if (!op->lbuf && !(op->lbuf = pool_get(c, 2 * g->comp_elems)))
      return fail(PC_E_CUDA, "line preconditioner allocation failed (out of device memory)");
    k_line_coef<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, op->ao, op->lbuf + g->g.plane,
                                                             op->lbuf + g->comp_elems + g->g.plane);
    c->st.launches++;
    TRY(check_launch("k_line_coef"));
    op->line_valid = true;
  }
  const int nbl = (int)((g->g.plane + kThreads - 1) / kThreads);
  k_line_factor<<<nbl, kThreads, 0, c->s>>>(g->g, op->dbuf + g->g.plane, op->lbuf + g->g.plane,
                                            op->lbuf + g->comp_elems + g->g.plane, adiag, dt, Lf.base(0), Lf.base(1));
  c->st.launches++;
  return check_launch("k_line_factor");
}
static int line_apply(pc_op* op, const double* r, Work& Lf, double dt, double* z, int mode) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  const int nbl = (int)((g->g.plane + kThreads - 1) / kThreads);
  if (nbl > c->max_red) return fail(PC_E_INVALID, "too many r-lines for the reduction scratch");
  k_line_solve<<<nbl, kThreads, 0, c->s>>>(g->g, op->ao, r, op->lbuf + g->g.plane, Lf.base(0), Lf.base(1), dt, z,
                                           mode, c->red_v, c->counter, c->pcg);
  c->st.launches++;
  return check_launch("k_line_solve");
}

template <class Op>
static int pcg_run(pc_op* op, const Op& o, double dt, const double* adiag, CFld b, pc_field* x, double tol,
                   int max_iter, int* iters, double* relres, int* converged) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  const int nc = op->ncomp;
  Work r, p0, p1, Ap;
  TRY(work_get(g, nc, r));
  TRY(work_get(g, nc, p0));
  TRY(work_get(g, nc, p1));
  TRY(work_get(g, nc, Ap));
  const double* dg = op->dbuf + g->g.plane;
  const int nb = node_blocks(c, g->g);
  const bool line = std::is_same<Op, AlignedOp>::value && op->pc == PC_PC_LINE_R;
  if (line && c->nranks > 1) return fail(PC_E_INVALID, "the r-line preconditioner needs the whole r line on one rank");
  Work z, Lf;  // r-line preconditioner: z and the factorisation (inv, cp)
  if (line) {
    TRY(work_get(g, 1, z));
    TRY(work_get(g, 2, Lf));
  }
  int rc = halo_field(x);
  // the stored inverse Jacobi diagonal of this solve, dinv = 1 / (a + dt d)
  // (SPEC.md:192-200): every z = r dinv below multiplies by it
  Work dvw;
  if (rc == PC_OK) rc = work_get(g, 1, dvw);
  if (rc == PC_OK) {
    k_pcg_dinv<<<nb, kThreads, 0, c->s>>>(g->g, dg, adiag, dt, dvw.base(0));
    c->st.launches++;
    rc = check_launch("k_pcg_dinv");
  }
  const double* dinv = dvw.b[0] ? dvw.base(0) : nullptr;
  // split reductions: the kernels stop at the per-plane sums, NCCL gathers
  // them (the r-line preconditioner is single-rank)
  const bool split = c->comm != nullptr && !line;
  // slots per plane: the marching kernels (aligned matvec / init) write one
  // partial per warp and tile, the row kernels one per theta row
  const dim3 mg = march_grid(g, 1);
  const int Sm = std::is_same<Op, AlignedOp>::value ? (int)(mg.x * mg.y) * (MNT / 32) : g->g.n1;
  PlaneRed prm{}, prr{};  // (one scratch, consumed by each reduction before the next one writes)
  if (rc == PC_OK) rc = plane_red(g, std::max(Sm, g->g.n1), prm);
  prr = prm;
  prm.S = Sm;
  prr.S = g->g.n1;
  if (rc == PC_OK) {
    if constexpr (std::is_same<Op, AlignedOp>::value) {
      // r = b - A x0 through the marching kernel (x0 staged like any T)
      if (adiag) {
        EpiPcgInitT<true> e{b.p[0], dinv, adiag, r.base(0), p0.base(0), dt, prm.slot[0], prm.slot[1]};
        rc = launch_march(op, cfld(x).p[0], e, nullptr, "k_aligned_march<pcg init>");
      } else {
        EpiPcgInitT<false> e{b.p[0], dinv, adiag, r.base(0), p0.base(0), dt, prm.slot[0], prm.slot[1]};
        rc = launch_march(op, cfld(x).p[0], e, nullptr, "k_aligned_march<pcg init>");
      }
      if (rc == PC_OK) rc = plane_sums(g, prm, 2, PR_INIT, line ? 1 : 0, split, tol, 0);
      if (rc == PC_OK && line) {  // z0 = M^{-1} r0, (r0, z0) -> fin_init
        rc = line_prepare(op, dt, adiag, Lf);
        if (rc == PC_OK) rc = line_apply(op, r.base(0), Lf, dt, z.base(0), 0);
      }
    } else {
      k_pcg_init<<<nb, kThreads, 0, c->s>>>(g->g, o, b, cfld(x), r.f(), p0.f(), dinv, adiag, dt, prr, c->pcg);
      c->st.launches++;
      rc = check_launch("k_pcg_init");
      if (rc == PC_OK) rc = plane_sums(g, prr, 2, PR_INIT, 0, split, tol, 0);
    }
  }
  Work* pold = &p0;
  Work* pnew = &p1;
  const int batch = 4;
  int it = 0;
  bool stop = false;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing) {
    e0 = ev_new(c);
    e1 = ev_new(c);
    cudaEventRecord(e0, c->s);
  }
  // 128-bit p-update and x/r-update kernels when phi rows have even length
  // (every field then stays 16-byte aligned: plane and row offsets are even);
  // C4 update 2.72 -> 2.03 ms (profiles/r01_c4_pcg_vec.txt).  PC_PCG_SCALAR_IO
  // keeps the 64-bit kernels (tests compare the two)
  const bool vio = g->g.n2 % 2 == 0 && getenv("PC_PCG_SCALAR_IO") == nullptr;
  // the p-update fused into the matvec march (EpiMatvecP: r, p_old, d staged,
  // p formed on the fly): TMA march, point Jacobi, no mass diagonal, and no
  // ghost planes / columns (their p would need r, p_old, d exchanged instead
  // of p); PC_PCG_NO_FUSEP keeps the separate p-update kernel (tests compare)
  const bool fusep = std::is_same<Op, AlignedOp>::value && !line && !adiag && tma_ok(g) && !g->g.ghost_lo0 &&
                     !g->g.ghost_hi0 && !g->g.phis && getenv("PC_PCG_NO_FUSEP") == nullptr;
  while (rc == PC_OK && !stop && it < max_iter) {
    for (int q = 0; q < batch && it < max_iter && rc == PC_OK; ++q) {
      ++it;
      if constexpr (std::is_same<Op, AlignedOp>::value) {
        const int* done = reinterpret_cast<const int*>(reinterpret_cast<const char*>(c->pcg) + offsetof(PcgDev, done));
        if (fusep) {  // p-update + matvec in one march
          EpiMatvecP e{pold->base(0), dinv, pnew->base(0), Ap.base(0), dt, prm.slot[0], c->pcg};
          rc = launch_march(op, r.base(0), e, done, "k_aligned_march<matvec + p-update>");
          if (rc == PC_OK) rc = plane_sums(g, prm, 1, PR_MATVEC, 0, split, tol, it);
          if (rc) break;
          goto matvec_done;
        }
        // p = z + beta p_old (beta from the device-side PCG state), then the
        // marching matvec stages p like any other field
        if (line) {
          k_pcg_pupdate_z<<<nb, kThreads, 0, c->s>>>(g->g, z.base(0), pold->base(0), pnew->base(0), c->pcg);
        } else if (vio) {
          // four phi pairs per lane at 2 blocks/SM: 1.21 ms at C4 (7.1 TB/s) against 1.32 (two pairs,
          // 4 blocks, spills) and 1.54 (two pairs, 85 registers) -- profiles/r01_c4_pcg_vec.txt
          k_pcg_pupdatev<4, 2><<<nb, kThreads, 0, c->s>>>(g->g, r.base(0), pold->base(0), pnew->base(0), dinv,
                                                          c->pcg);
        } else {
          k_pcg_pupdate<<<nb, kThreads, 0, c->s>>>(g->g, r.base(0), pold->base(0), pnew->base(0), dinv, c->pcg);
        }
        c->st.launches++;
        rc = check_launch("k_pcg_pupdate");
        if (rc == PC_OK) rc = halo_work(g, *pnew);
        if (rc) break;
        if (adiag) {
          EpiMatvecT<true> e{adiag, Ap.base(0), dt, prm.slot[0]};
          rc = launch_march(op, pnew->base(0), e, done, "k_aligned_march<matvec>");
        } else {
          EpiMatvecT<false> e{adiag, Ap.base(0), dt, prm.slot[0]};
          rc = launch_march(op, pnew->base(0), e, done, "k_aligned_march<matvec>");
        }
        if (rc == PC_OK) rc = plane_sums(g, prm, 1, PR_MATVEC, 0, split, tol, it);
        if (rc) break;
      matvec_done:;
      } else {
        rc = halo_work(g, r);
        if (rc == PC_OK) rc = halo_work(g, *pold);
        if (rc) break;
        k_pcg_matvec<<<nb, kThreads, 0, c->s>>>(g->g, o, r.cf(), pold->cf(), pnew->f(), Ap.f(), dinv, adiag, dt,
                                                prr, c->pcg);
        rc = check_launch("k_pcg_matvec");
        if (rc == PC_OK) rc = plane_sums(g, prr, 1, PR_MATVEC, 0, split, tol, it);
        if (rc) break;
      }
      if constexpr (std::is_same<Op, AlignedOp>::value) {
        auto upd = vio
                       ? (line ? (o.rho ? (adiag ? k_pcg_update1v<true, true, true> : k_pcg_update1v<true, false, true>)
                                        : (adiag ? k_pcg_update1v<false, true, true>
                                                 : k_pcg_update1v<false, false, true>))
                               : (o.rho ? (adiag ? k_pcg_update1v<true, true> : k_pcg_update1v<true, false>)
                                        : (adiag ? k_pcg_update1v<false, true> : k_pcg_update1v<false, false>)))
                       : (line ? (o.rho ? (adiag ? k_pcg_update1<true, true, true> : k_pcg_update1<true, false, true>)
                                       : (adiag ? k_pcg_update1<false, true, true> : k_pcg_update1<false, false, true>))
                              : (o.rho ? (adiag ? k_pcg_update1<true, true> : k_pcg_update1<true, false>)
                                       : (adiag ? k_pcg_update1<false, true> : k_pcg_update1<false, false>)));
        upd<<<nb, kThreads, 0, c->s>>>(g->g, x->base(0), r.base(0), pnew->base(0), Ap.base(0), dinv, adiag, o.rho, dt,
                                       tol, it, prr, c->pcg);
      } else {
        k_pcg_update<<<nb, kThreads, 0, c->s>>>(g->g, o, fld(x), r.f(), pnew->cf(), Ap.cf(), dinv, adiag, dt, prr,
                                                c->pcg);
      }
      c->st.launches += std::is_same<Op, AlignedOp>::value ? 1 : 2;  // (march counted at launch)
      c->st.stage_launches += std::is_same<Op, AlignedOp>::value ? 3 : 2;
      rc = check_launch("k_pcg");
      if (rc == PC_OK) rc = plane_sums(g, prr, line ? 1 : 2, line ? PR_UPDATE_RR : PR_UPDATE, 0, split, tol, it);
      if (rc == PC_OK && line) rc = line_apply(op, r.base(0), Lf, dt, z.base(0), 1);
      std::swap(pold, pnew);
    }
    if (rc) break;
    if (cudaMemcpyAsync(c->h_pcg, c->pcg, sizeof(PcgDev), cudaMemcpyDeviceToHost, c->s) != cudaSuccess ||
        cudaStreamSynchronize(c->s) != cudaSuccess) {
      rc = fail(PC_E_CUDA, "PCG state readback");
      break;
    }
    if (c->h_pcg->done) stop = true;
  }
  const int pkind = std::is_same<Op, AlignedOp>::value ? KIND_PCG_ALIGNED : KIND_PCG_SCALAR;
  if (c->timing) {
    cudaEventRecord(e1, c->s);
    c->ev.push_back({e0, e1, pkind});
  }
  if (rc == PC_OK) {
    CUDA_TRY(cudaMemcpyAsync(c->h_pcg, c->pcg, sizeof(PcgDev), cudaMemcpyDeviceToHost, c->s));
    c->st.kind_launches[pkind] += (int64_t)c->h_pcg->it * (std::is_same<Op, AlignedOp>::value ? (fusep ? 2 : 3) : 2);
    c->st.kind_units[pkind] += (int64_t)c->h_pcg->it * owned_cells(g->g);
    CUDA_TRY(cudaStreamSynchronize(c->s));
    const PcgDev& st = *c->h_pcg;
    *iters = st.it;
    *relres = st.rel;
    *converged = st.status == 1 ? 1 : 0;
    if (st.status == 2) rc = fail(PC_E_INDEFINITE, "PCG breakdown: p^T A p <= 0 (indefinite operator)");
    if (st.status == 3) rc = fail(PC_E_DIVERGED, "PCG divergence: non-finite residual");
  }
  work_put(r);
  work_put(p0);
  work_put(p1);
  work_put(Ap);
  if (dvw.b[0]) work_put(dvw);
  if (line) {
    work_put(z);
    work_put(Lf);
  }
  return rc;
}

static int pcg_any(pc_op* op, double dt, const double* adiag, CFld b, pc_field* x, double tol, int max_iter,
                   int* iters, double* relres, int* converged) {
  TRY(ensure_diag(op));
  if (op->kind == K_ALIGNED) return pcg_run(op, op->ao, dt, adiag, b, x, tol, max_iter, iters, relres, converged);
  return pcg_run(op, op->so, dt, adiag, b, x, tol, max_iter, iters, relres, converged);
}

int pc_pcg_solve(pc_op* op, double dt, const pc_field* diag_a, const pc_field* b, pc_field* x, double tol,
                 int max_iter, int* iters, double* relres, int* converged) {
  field_dep(diag_a); field_dep(b); field_dep(x);
  if (!op || !b || !x || !iters || !relres || !converged) return fail(PC_E_INVALID, "null argument");
  if (b->ncomp != op->ncomp || x->ncomp != op->ncomp) return fail(PC_E_INVALID, "shape mismatch");
  op_deps(op);
  if (!(tol > 0.0 && tol < 1.0) || max_iter < 1) return fail(PC_E_INVALID, "need 0 < tol < 1 and max_iter >= 1");
  TRY(need_frozen(op));
  if (!op->frozen) TRY(pc_op_freeze(op, nullptr));
  const double* ad = diag_a ? diag_a->base(0) : nullptr;
  return pcg_any(op, dt, ad, cfld(b), x, tol, max_iter, iters, relres, converged);
}

static int be_step(pc_op* op, pc_field* u, double dt, double tol, int max_iter, int* iters, double* relres,
                   int* converged) {
  pc_grid* g = op->grid;
  Work bw;
  TRY(work_get(g, op->ncomp, bw));
  int rc = PC_OK;
  for (int q = 0; q < op->ncomp && rc == PC_OK; ++q)
    if (cudaMemcpyAsync(bw.b[q], u->buf[q], g->comp_elems * sizeof(double), cudaMemcpyDeviceToDevice, g->ctx->s) !=
        cudaSuccess)
      rc = fail(PC_E_CUDA, "BE rhs copy");
  if (rc == PC_OK) rc = pcg_any(op, dt, nullptr, bw.cf(), u, tol, max_iter, iters, relres, converged);
  work_put(bw);
  return rc;
}

int pc_step_be(pc_op* op, pc_field* u, double dt, double tol, int max_iter, int* iters, double* relres,
               int* converged) {
  field_dep(u);
  if (!op || !u || u->ncomp != op->ncomp || !iters || !relres || !converged) return fail(PC_E_INVALID, "bad arguments");
  op_deps(op);
  if (!(tol > 0.0 && tol < 1.0) || max_iter < 1) return fail(PC_E_INVALID, "need 0 < tol < 1 and max_iter >= 1");
  TRY(need_frozen(op));
  if (!op->frozen) TRY(pc_op_freeze(op, nullptr));
  return be_step(op, u, dt, tol, max_iter, iters, relres, converged);
}
