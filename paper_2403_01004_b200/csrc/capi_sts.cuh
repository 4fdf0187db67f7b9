// paracycle_b200 C ABI, part of the single translation unit capi.cu (included
// there in order; relies on the declarations of the parts before it).
//
// C ABI: PTL (Eq. 5 pairs on the device) and the STS stage loop (RKL2 / RKG2,
// fused stage kernels, halo exchange overlapped with interior r-chunks)
#pragma once

// ------------------------------------------------------------------ PTL
// Eq. 5 after the |F| argmax.  r-slabs: the argmax pairs are allgathered and
// combined (lowest global index on ties), F's ghost planes are exchanged so the
// owner of k sees its r-neighbours, and the candidate minimum is allreduced.
static int ptl_device(pc_grid* g, int ncomp, CFld u, CFld F, double* const* Fbufs, double eps_rel, int check_all) {
  pc_ctx* c = g->ctx;
  TRY(global_argmax(c));
  if (c->comm && Fbufs) TRY(halo_exchange(c, g, Fbufs, ncomp));
  if (check_all) {
    CUDA_TRY(cudaMemsetAsync(c->minbits, 0x7f, sizeof(unsigned long long), c->s));  // huge positive
    k_ptl_all<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, ncomp, u, F, eps_rel, c->res, c->minbits);
    c->st.launches++;
    TRY(check_launch("k_ptl_all"));
    TRY(allreduce_u64_min(c, c->minbits));
  } else {
    k_ptl_pairs<<<1, 32, 0, c->s>>>(g->g, ncomp, u, F, eps_rel, c->res);
    c->st.launches++;
    TRY(check_launch("k_ptl_pairs"));
    TRY(allreduce_d(c, &c->res->ptl, 1, nccl::kMin));
  }
  return PC_OK;
}
// read back the argmax/PTL result (the single per-cycle sync)
static int ptl_read(pc_ctx* c, int check_all, int use_ptl, double* ptl, int* limited, int64_t* kidx) {
  CUDA_TRY(cudaMemcpyAsync(c->h_res, c->res, sizeof(ArgRes), cudaMemcpyDeviceToHost, c->s));
  if (check_all) CUDA_TRY(cudaMemcpyAsync(c->h_minbits, c->minbits, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->s));
  CUDA_TRY(cudaStreamSynchronize(c->s));
  if (kidx) *kidx = c->h_res->kidx;
  if (!use_ptl) {
    *limited = 0;
    *ptl = INFINITY;
    return PC_OK;
  }
  if (check_all) {
    double v;
    unsigned long long bits = *c->h_minbits;
    std::memcpy(&v, &bits, sizeof v);
    *limited = (bits != 0x7f7f7f7f7f7f7f7fULL && std::isfinite(v)) ? 1 : 0;
    *ptl = *limited ? v : INFINITY;
  } else {
    *limited = std::isfinite(c->h_res->ptl) ? 1 : 0;  // (the allreduced minimum)
    *ptl = *limited ? c->h_res->ptl : INFINITY;
  }
  return PC_OK;
}

int pc_ptl(pc_grid* g, const pc_field* u, const pc_field* F, double eps_rel, int check_all, double* ptl,
           int* limited, int64_t* kidx) {
  field_dep(u); field_dep(F);
  if (!g || !u || !F || !ptl || !limited || u->ncomp != F->ncomp || u->grid != g || F->grid != g)
    return fail(PC_E_INVALID, "bad PTL arguments");
  if (!(eps_rel > 0.0)) return fail(PC_E_INVALID, "eps_rel must be > 0");
  pc_ctx* c = g->ctx;
  k_argmax<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, u->ncomp, cfld(F), c->red_v, c->red_i,
                                                          c->counter, c->res);
  c->st.launches++;
  TRY(check_launch("k_argmax"));
  TRY(halo_field(const_cast<pc_field*>(u)));
  double* Fb[3] = {F->buf[0], F->buf[1], F->buf[2]};
  TRY(ptl_device(g, u->ncomp, cfld(u), cfld(F), Fb, eps_rel, check_all));
  return ptl_read(c, check_all, 1, ptl, limited, kidx);
}

// ------------------------------------------------------------------ STS
int pc_sts_count(int kind, double dt, double dt_euler, int make_odd) {
  static_assert(kRKL2 == PC_RKL2 && kRKG2 == PC_RKG2, "scheme codes");
  return sts_count_hd(kind, dt, dt_euler, make_odd);
}
int pc_sts_table(int kind, int s, double dt, double* out) {
  if (!out) return fail(PC_E_INVALID, "null table");
  if (kind != PC_RKL2 && kind != PC_RKG2) return fail(PC_E_INVALID, "unknown STS kind");
  if (!sts_rows_hd(kind, s, dt, out))
    return fail(PC_E_INVALID, kind == PC_RKL2 ? "RKL2 needs s >= 2" : "RKG2 needs odd s >= 3 (SPEC.md:264)");
  return PC_OK;
}

template <class Op>
static int sts_stages(pc_op* op, const Op& o, pc_field* u, const double* tab, int s, Work& y0,
                      bool deferred = false) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  const int nc = op->ncomp;
  Work A, B;
  TRY(work_get(g, nc, A));
  int rc = work_get(g, nc, B);
  if (rc) {
    work_put(A);
    return rc;
  }
  const int nb = node_blocks(c, g->g);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  Work* um1 = &A;
  Work* out = &B;
  Work* um2w = nullptr;  // nullptr -> u0
  // multi-rank: the ghost planes of u_{k-1} travel on the communication
  // stream while the interior r-chunks (which never read them) run; the two
  // boundary chunks follow the exchange (PC_SPLIT_STAGE forces the split
  // launches on one rank, for testing)
  const bool force_split = getenv("PC_SPLIT_STAGE") != nullptr;
  const bool marching = std::is_same<Op, AlignedOp>::value || smarch_ok(op);
  const int Rz = std::is_same<Op, AlignedOp>::value ? march_R(g) : smarch_R(g, op->ncomp);
  const int nz = (g->g.n0 + Rz - 1) / Rz;
  // (phi-slabs exchange ghost COLUMNS: every r-chunk reads them, no overlap split)
  const bool overlap = marching && nz >= 3 && !g->g.phis && (c->comm != nullptr || force_split);
  // 7-point march, one rank without ghost planes: stages 1 and 2 in one pass
  // (SEpiStage12: u1 formed in shared memory from u0 and y0; PC_NO_FUSE12 off)
  const bool fuse12 = !std::is_same<Op, AlignedOp>::value && smarch_ok(op) && !overlap && !g->g.ghost_lo0 &&
                      !g->g.ghost_hi0 && !g->g.phis && getenv("PC_NO_FUSE12") == nullptr;
  // aligned TMA march, one rank without ghost planes: stages 1 and 2 in one
  // pass as well (EpiStageA12: u1 formed in the input slot from u0 and y0;
  // PC_NO_FUSE12A off)
  const bool fuse12a = std::is_same<Op, AlignedOp>::value && s >= 2 && tma_ok(g) && !overlap && !g->g.ghost_lo0 &&
                       !g->g.ghost_hi0 && !g->g.phis && getenv("PC_NO_FUSE12A") == nullptr;
  CUDA_TRY(cudaMemsetAsync(c->bad, 0x7f, sizeof(int), c->s));
  if (fuse12a) {
    const double* r = tab + 5;
    const StageCoef sc{r[0], r[1], r[2], r[3], r[4]};
    const bool w1 = s >= 3;
    const int kind = w1 ? KIND_STS_AF12W : KIND_STS_AF12;
    cudaEvent_t f0 = nullptr, f1 = nullptr;
    if (c->timing) {
      f0 = ev_new(c);
      f1 = ev_new(c);
      cudaEventRecord(f0, c->s);
    }
    EpiStageA12 e{cfld(u).p[0], y0.base(0), B.base(0), w1 ? A.base(0) : nullptr, sc, tab[3], c->bad};
    rc = launch_tma(op, cfld(u).p[0], e, nullptr, "k_aligned_tma<stage 1+2>");
    if (c->timing) {
      cudaEventRecord(f1, c->s);
      c->ev.push_back({f0, f1, kind});
    }
    c->st.kind_launches[kind] += 1;
    c->st.kind_units[kind] += 2 * owned_cells(g->g);
    c->st.stage_launches++;
    // rotate as after stage 2 below: u1 (A) -> u_{k-2}, u2 (B) -> u_{k-1}
    um2w = &A;
    um1 = &B;
    out = &A;
  } else if (fuse12) {
    const double* r = tab + 5;
    const StageCoef sc{r[0], r[1], r[2], r[3], r[4]};
    CFld u0f = cfld(u), y0f = y0.cf();
    Fld of = B.f(), af = A.f();
    const bool w1 = s >= 3;
    const int kind = w1 ? KIND_STS_F12W : KIND_STS_F12;
    cudaEvent_t f0 = nullptr, f1 = nullptr;
    if (c->timing) {
      f0 = ev_new(c);
      f1 = ev_new(c);
      cudaEventRecord(f0, c->s);
    }
    if (nc == 3) {
      SEpiStage12<3> e{{u0f.p[0], u0f.p[1], u0f.p[2]}, {y0f.p[0], y0f.p[1], y0f.p[2]}, {of.p[0], of.p[1], of.p[2]},
                       {w1 ? af.p[0] : nullptr, af.p[1], af.p[2]}, tab[3], sc, c->bad};
      rc = launch_smarch_nc<3>(op, u0f, e, "k_scalar_march<stage 1+2>");
    } else {
      SEpiStage12<1> e{{u0f.p[0], nullptr, nullptr}, {y0f.p[0], nullptr, nullptr}, {of.p[0], nullptr, nullptr},
                       {w1 ? af.p[0] : nullptr, nullptr, nullptr}, tab[3], sc, c->bad};
      rc = launch_smarch_nc<1>(op, u0f, e, "k_scalar_march<stage 1+2>");
    }
    if (c->timing) {
      cudaEventRecord(f1, c->s);
      c->ev.push_back({f0, f1, kind});
    }
    c->st.kind_launches[kind] += 1;
    c->st.kind_units[kind] += 2 * owned_cells(g->g);
    c->st.stage_launches++;
    // rotate as after stage 2 below: u1 (A) -> u_{k-2}, u2 (B) -> u_{k-1}
    um2w = &A;
    um1 = &B;
    out = &A;
  } else {
    k_stage1<<<nb, kThreads, 0, c->s>>>(g->g, nc, cfld(u), y0.cf(), A.f(), tab[3], c->bad);
    c->st.launches++;
    rc = check_launch("k_stage1");
  }
  if (c->timing) {  // the fused stage kernels k >= 2 (the roofline kernel)
    e0 = ev_new(c);
    e1 = ev_new(c);
    cudaEventRecord(e0, c->s);
  }
  for (int k = (fuse12 || fuse12a) ? 3 : 2; k <= s && rc == PC_OK; ++k) {
    const double* r = tab + 5 * (k - 1);
    StageCoef sc{r[0], r[1], r[2], r[3], r[4]};
    CFld m2 = um2w ? um2w->cf() : cfld(u);
    auto launch_stage = [&]() -> int {
      if constexpr (std::is_same<Op, AlignedOp>::value) {
        EpiStage e{m2.p[0], cfld(u).p[0], y0.base(0), out->base(0), sc, k, c->bad};
        return launch_march(op, um1->base(0), e, nullptr, "k_aligned_march<stage>");
      } else if (smarch_ok(op)) {
        CFld u0f = cfld(u), y0f = y0.cf();
        Fld of = out->f();
        SEpiStage e{{u0f.p[0], u0f.p[1], u0f.p[2]}, {m2.p[0], m2.p[1], m2.p[2]}, {y0f.p[0], y0f.p[1], y0f.p[2]},
                    {of.p[0], of.p[1], of.p[2]}, nc, sc, k, c->bad};
        if (nc == 3) return launch_smarch_nc<3>(op, um1->cf(), e, "k_scalar_march<stage>");
        SEpiStage1 e1;
        static_cast<SEpiStage&>(e1) = e;
        return launch_smarch_nc<1>(op, um1->cf(), e1, "k_scalar_march<stage>");
      } else {
        k_stage<<<nb, kThreads, 0, c->s>>>(g->g, o, um1->cf(), m2, cfld(u), y0.cf(), out->f(), sc, k, c->bad);
        c->st.launches++;
        return check_launch("k_stage");
      }
    };
    if (overlap) {
      CUDA_TRY(cudaEventRecord(c->ev_in, c->s));
      CUDA_TRY(cudaStreamWaitEvent(c->sc, c->ev_in, 0));
      double* hb[3] = {um1->b[0], um1->b[1], um1->b[2]};
      rc = halo_exchange(c, g, hb, um1->ncomp, c->sc);
      if (rc) break;
      CUDA_TRY(cudaEventRecord(c->ev_halo, c->sc));
      c->zpart = 1;
      rc = launch_stage();
      c->zpart = 0;
      if (rc) break;
      CUDA_TRY(cudaStreamWaitEvent(c->s, c->ev_halo, 0));
      c->zpart = 2;
      rc = launch_stage();
      c->zpart = 0;
    } else {
      rc = halo_work(g, *um1);
      if (rc) break;
      rc = launch_stage();
    }
    c->st.stage_launches++;
    // rotate: u_{k-1} -> u_{k-2}, u_k -> u_{k-1}; the next stage writes into
    // the buffer that held u_{k-1} before this stage, i.e. the new u_{k-2}
    // (pointwise safe: u_{k-2} is only read at the thread's own node)
    Work* prev_um1 = um1;
    um2w = um1;
    um1 = out;
    out = prev_um1;
  }
  {
    const int kind = std::is_same<Op, AlignedOp>::value ? KIND_STS_ALIGNED : KIND_STS_SCALAR;
    if (c->timing) {
      cudaEventRecord(e1, c->s);
      c->ev.push_back({e0, e1, kind});
    }
    const int nst = s - ((fuse12 || fuse12a) ? 2 : 1);
    c->st.kind_launches[kind] += nst;
    c->st.kind_units[kind] += (int64_t)nst * owned_cells(g->g);
  }
  if (rc == PC_OK && deferred) {
    // pc_cycle: no host sync per step -- the flag travels with the stream and
    // is checked at the next PTL read (or the end of the cycle loop)
    CUDA_TRY(cudaMemcpyAsync(c->h_bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    c->bad_pending = true;
    swap_storage(u, *um1);
  } else if (rc == PC_OK) {
    CUDA_TRY(cudaMemcpyAsync(c->h_bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CUDA_TRY(cudaStreamSynchronize(c->s));
    if (*c->h_bad != 0x7f7f7f7f) {
      rc = fail(PC_E_BLOWUP, "non-finite value at STS stage " + std::to_string(*c->h_bad), *c->h_bad);
    } else {
      swap_storage(u, *um1);  // u <- u_s; the old u0 storage returns to the pool
    }
  }
  work_put(A);
  work_put(B);
  return rc;
}

static int sts_any(pc_op* op, pc_field* u, const double* tab, int s, Work& y0, bool deferred = false) {
  if (op->kind == K_ALIGNED) return sts_stages(op, op->ao, u, tab, s, y0, deferred);
  return sts_stages(op, op->so, u, tab, s, y0, deferred);
}
// the deferred non-finite flag of the previous STS step (stream synchronised)
static int check_pending_bad(pc_ctx* c) {
  if (!c->bad_pending) return PC_OK;
  c->bad_pending = false;
  if (*c->h_bad != 0x7f7f7f7f)
    return fail(PC_E_BLOWUP, "non-finite value at STS stage " + std::to_string(*c->h_bad), *c->h_bad);
  return PC_OK;
}

int pc_step_sts(pc_op* op, pc_field* u, double dt, int kind, int s, const pc_field* y0in) {
  field_dep(u); field_dep(y0in);
  if (!op || !u || u->ncomp != op->ncomp) return fail(PC_E_INVALID, "shape mismatch");
  if (kind != PC_RKL2 && kind != PC_RKG2) return fail(PC_E_INVALID, "unknown STS kind");
  op_deps(op);
  TRY(need_frozen(op));
  pc_grid* g = op->grid;
  std::vector<double> tab(5 * (size_t)s);
  TRY(pc_sts_table(kind, s, dt, tab.data()));
  Work y0;
  TRY(work_get(g, op->ncomp, y0));
  int rc = PC_OK;
  if (y0in) {
    for (int q = 0; q < op->ncomp && rc == PC_OK; ++q)
      if (cudaMemcpyAsync(y0.b[q], y0in->buf[q], g->comp_elems * sizeof(double), cudaMemcpyDeviceToDevice,
                          g->ctx->s) != cudaSuccess)
        rc = fail(PC_E_CUDA, "y0 copy");
  } else {
    rc = halo_field(u);
    if (rc == PC_OK) rc = apply_any(op, cfld(u), y0.f(), false);
  }
  if (rc == PC_OK) rc = sts_any(op, u, tab.data(), s, y0);
  work_put(y0);
  return rc;
}

int pc_step_euler(pc_op* op, pc_field* u, double dt) {
  field_dep(u);
  if (!op || !u || u->ncomp != op->ncomp) return fail(PC_E_INVALID, "shape mismatch");
  op_deps(op);
  TRY(need_frozen(op));
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  Work y0, A;
  TRY(work_get(g, op->ncomp, y0));
  TRY(work_get(g, op->ncomp, A));
  int rc = halo_field(u);
  if (rc == PC_OK) rc = apply_any(op, cfld(u), y0.f(), false);
  if (rc == PC_OK) {
    CUDA_TRY(cudaMemsetAsync(c->bad, 0x7f, sizeof(int), c->s));
    k_stage1<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, op->ncomp, cfld(u), y0.cf(), A.f(), dt, c->bad);
    c->st.launches++;
    rc = check_launch("k_stage1");
  }
  if (rc == PC_OK) {
    CUDA_TRY(cudaStreamSynchronize(c->s));
    swap_storage(u, A);
  }
  work_put(y0);
  work_put(A);
  return rc;
}
