// paracycle_b200 C ABI, part of the single translation unit capi.cu (included
// there in order; relies on the declarations of the parts before it).
//
// C ABI: pc_cycle, the PTL-cycled advance (host-driven loop, and the
// persistent one-launch loop for small grids)
#pragma once

// ------------------------------------------------------------------ cycle
// ---- persistent small-grid cycle loop (persist.cuh)
static bool persist_ok(const pc_op* op) {
  const pc_grid* g = op->grid;
  const pc_ctx* c = g->ctx;
  if (op->kind != K_SCALAR || (op->ncomp != 1 && op->ncomp != 3)) return false;
  if (c->comm || c->nranks > 1 || g->g.ghost_lo0 || g->g.ghost_hi0) return false;
  if (getenv("PC_NO_PERSIST")) return false;
  return (int64_t)g->g.N * op->ncomp <= (int64_t)(getenv("PC_PERSIST_MAX") ? atoll(getenv("PC_PERSIST_MAX")) : 1 << 21);
}
static int cycle_persistent(pc_op* op, pc_field* u, double outer_dt, int scheme, int make_odd, double eps_rel,
                            int use_ptl, double floor_dt, double dtE, int64_t max_cycles, pc_cycle_record* rec,
                            int64_t rec_cap, int64_t* n_rec) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  const int nc = op->ncomp;
  if (!c->cyc_dev) {
    CUDA_TRY(cudaMalloc(&c->cyc_dev, sizeof(CycleDev)));
    CUDA_TRY(cudaMallocHost(&c->h_cyc, sizeof(CycleDev)));
  }
  Work A, B, y0;
  TRY(work_get(g, nc, A));
  TRY(work_get(g, nc, B));
  TRY(work_get(g, nc, y0));
  const int64_t cap = std::max<int64_t>(0, std::min<int64_t>(rec_cap, max_cycles));
  // device cycle records: a grow-only buffer kept by the context (a
  // cudaMalloc / cudaFree pair per call synchronises the device and cost up
  // to tens of ms at random, profiles/r01_c1_persist_variants.txt)
  int rc = PC_OK;
  if (cap > c->cyc_rec_cap) {
    if (c->cyc_rec) cudaFree(c->cyc_rec);
    c->cyc_rec = nullptr;
    c->cyc_rec_cap = 0;
    if (cudaMalloc(&c->cyc_rec, (size_t)cap * sizeof(pc_cycle_record)) != cudaSuccess)
      rc = fail(PC_E_CUDA, "cycle record allocation failed");
    else
      c->cyc_rec_cap = cap;
  }
  pc_cycle_record* drec = cap > 0 ? c->cyc_rec : nullptr;
  CycleDev& h = *c->h_cyc;
  std::memset(&h, 0, offsetof(CycleDev, tab));
  h.remaining = outer_dt;
  h.dtE = dtE;
  h.floor_dt = floor_dt;
  h.eps_rel = eps_rel;
  h.kind = scheme;
  h.make_odd = make_odd;
  h.use_ptl = use_ptl;
  h.rec_cap = (int)std::min<int64_t>(cap, 1 << 30);
  h.max_cycles = max_cycles;
  h.bad = 0x7f7f7f7f;
  PersistBufs pb{};
  for (int q = 0; q < nc; ++q) {
    pb.set[0][q] = u->base(q);
    pb.set[1][q] = A.base(q);
    pb.set[2][q] = B.base(q);
    pb.y0[q] = y0.base(q);
  }
  pb.pv = c->red_v;
  pb.pi = c->red_i;
  if (rc == PC_OK && cudaMemcpyAsync(c->cyc_dev, &h, offsetof(CycleDev, tab), cudaMemcpyHostToDevice, c->s) != cudaSuccess)
    rc = fail(PC_E_CUDA, "cycle state upload");
  if (rc == PC_OK) {
    void (*kern)(GridDev, ScalarOp, PersistBufs, CycleDev*, pc_cycle_record*) =
        nc == 3 ? k_cycle_small<3> : k_cycle_small<1>;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPersistThreads, 0);
    const int need = (int)std::max<int64_t>(1, ((int64_t)g->g.n0 * g->g.n1 + kPersistThreads / 32 - 1) /
                                                    (kPersistThreads / 32));
    const int nblk = std::max(1, std::min({per_sm * c->sms, need, c->max_red}));
    GridDev gd = g->g;
    ScalarOp so = op->so;
    CycleDev* csp = c->cyc_dev;
    void* args[] = {&gd, &so, &pb, &csp, &drec};
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->timing) {
      e0 = ev_new(c);
      e1 = ev_new(c);
      cudaEventRecord(e0, c->s);
    }
    if (cudaLaunchCooperativeKernel((void*)kern, dim3(nblk), dim3(kPersistThreads), args, 0, c->s) != cudaSuccess)
      rc = fail(PC_E_CUDA, "cooperative launch of the small-grid cycle kernel failed");
    c->st.launches++;
    c->st.stage_launches++;
    if (c->timing) {  // the whole cycle loop is the "STS" time of this path
      cudaEventRecord(e1, c->s);
      c->ev.push_back({e0, e1, KIND_STS_SCALAR});
    }
  }
  if (rc == PC_OK && cudaMemcpyAsync(&h, c->cyc_dev, offsetof(CycleDev, tab), cudaMemcpyDeviceToHost, c->s) != cudaSuccess)
    rc = fail(PC_E_CUDA, "cycle state readback");
  if (rc == PC_OK) {
    CUDA_TRY(cudaStreamSynchronize(c->s));
    const int64_t nrec = std::min<int64_t>(h.cyc, cap);
    if (nrec > 0 && rec)
      CUDA_TRY(cudaMemcpy(rec, drec, (size_t)std::min<int64_t>(nrec, rec_cap) * sizeof(pc_cycle_record),
                          cudaMemcpyDeviceToHost));
    *n_rec = rec ? std::min<int64_t>(nrec, rec_cap) : 0;
    {  // stage-k>=2 cell-updates, as the host-driven path counts them
      int64_t stages = 0;
      std::vector<pc_cycle_record> all((size_t)nrec);
      if (nrec > 0) CUDA_TRY(cudaMemcpy(all.data(), drec, (size_t)nrec * sizeof(pc_cycle_record), cudaMemcpyDeviceToHost));
      for (const auto& r : all) stages += r.iters - 1;
      c->st.kind_launches[KIND_STS_SCALAR] += 1;
      c->st.kind_units[KIND_STS_SCALAR] += stages * g->g.N;
    }
    if (h.cur == 1) swap_storage(u, A);
    else if (h.cur == 2) swap_storage(u, B);
    if (h.status == 2) rc = fail(PC_E_BLOWUP, "non-finite value at STS stage " + std::to_string(h.bad), h.bad);
    else if (h.status == 3) rc = fail(PC_E_CAP, "max_cycles reached (partial report returned)", h.cyc);
    else if (h.status == 4) rc = fail(PC_E_INVALID, "STS stage count above the persistent kernel's table");
  }

  work_put(A);
  work_put(B);
  work_put(y0);
  return rc;
}

int pc_cycle(pc_op* op, pc_field* u, double outer_dt, int scheme, int make_odd, double tol, int max_iter,
             double eps_rel, int check_all, int use_ptl, int floor_mode, double floor_fraction, int64_t max_cycles,
             double dt_euler, pc_cycle_record* rec, int64_t rec_cap, int64_t* n_rec) {
  field_dep(u);
  if (!op || !u || !n_rec || u->ncomp != op->ncomp) return fail(PC_E_INVALID, "bad cycle arguments");
  if (!(outer_dt > 0.0)) return fail(PC_E_INVALID, "outer_dt must be > 0");
  if (max_cycles < 1 || !(eps_rel > 0.0)) return fail(PC_E_INVALID, "need max_cycles >= 1 and eps_rel > 0");
  if (scheme < PC_RKL2 || scheme > PC_EULER) return fail(PC_E_INVALID, "unknown scheme");
  op_deps(op);
  TRY(need_frozen(op));
  if (!op->frozen) TRY(pc_op_freeze(op, nullptr));
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  if (use_ptl < 0 || use_ptl > 2) return fail(PC_E_INVALID, "use_ptl: 0 off, 1 dynamic, 2 static");
  double dtE = dt_euler > 0.0 ? dt_euler : op->dt_euler;
  double floor_dt = floor_mode == PC_FLOOR_EULER ? dtE : floor_fraction * dtE;
  double remaining = outer_dt;
  int64_t cyc = 0;
  *n_rec = 0;
  if ((scheme == PC_RKL2 || scheme == PC_RKG2) && !check_all && use_ptl != 2 && persist_ok(op))
    return cycle_persistent(op, u, outer_dt, scheme, make_odd, eps_rel, use_ptl, floor_dt, dtE, max_cycles, rec, rec_cap,
                            n_rec);
  Work y0;
  TRY(work_get(g, op->ncomp, y0));
  int rc = PC_OK;
  std::vector<double> tab;
  c->bad_pending = false;
  // PC_GAP_PROFILE (diagnostic): device time per cycle of F+argmax+pairs,
  // of the PTL read + host turnaround, and of the stages, printed at the end
  struct GapProfile {
    bool on = false;
    cudaEvent_t cur[4] = {};
    double t[3] = {0, 0, 0};
    double host = 0.0;  // host microseconds inside sts_any
    long n = 0;
    void flush() {
      cudaEventSynchronize(cur[3]);
      float a, b, d;
      cudaEventElapsedTime(&a, cur[0], cur[1]);
      cudaEventElapsedTime(&b, cur[1], cur[2]);
      cudaEventElapsedTime(&d, cur[2], cur[3]);
      t[0] += a;
      t[1] += b;
      t[2] += d;
      ++n;
    }
  } gp;
  gp.on = getenv("PC_GAP_PROFILE") != nullptr;
  double static_ptl = INFINITY;
  int static_limited = 0;
  if (gp.on)
    for (auto& e : gp.cur) e = ev_new(c);
  while (remaining > 0.0) {
    if (cyc >= max_cycles) {
      if (c->bad_pending) {
        CUDA_TRY(cudaStreamSynchronize(c->s));
        rc = check_pending_bad(c);
        if (rc) break;
      }
      rc = fail(PC_E_CAP, "max_cycles reached (partial report returned)", cyc);
      break;
    }
    if (op->refresh_cycle) {  // lagged T0 := u, coefficients and Gershgorin bound re-evaluated
      rc = pc_op_freeze(op, u);
      if (rc) break;
      if (!(dt_euler > 0.0)) {
        dtE = op->dt_euler;
        floor_dt = floor_mode == PC_FLOOR_EULER ? dtE : floor_fraction * dtE;
      }
    }
    if (gp.on) cudaEventRecord(gp.cur[0], c->s);
    rc = halo_field(u);
    if (rc) break;
    // static first-PTL cycling (use_ptl 2): the PTL of the first
    // cycle is reused by every later cycle; F is still formed (it is y0)
    const bool eval_ptl = use_ptl == 1 || (use_ptl == 2 && cyc == 0);
    if (scheme != PC_BE || eval_ptl) {
      rc = apply_any(op, cfld(u), y0.f(), true);
      if (rc) break;
    }
    if (eval_ptl) {
      double* yb[3] = {y0.b[0], y0.b[1], y0.b[2]};
      rc = ptl_device(g, op->ncomp, cfld(u), y0.cf(), yb, eps_rel, check_all);
      if (rc) break;
    }
    double ptl;
    int limited;
    if (gp.on) cudaEventRecord(gp.cur[1], c->s);
    if (eval_ptl || use_ptl == 0) {
      rc = ptl_read(c, check_all, use_ptl != 0, &ptl, &limited, nullptr);
      if (rc) break;
      rc = check_pending_bad(c);  // ptl_read synchronised the stream
      if (rc) break;
      static_ptl = ptl;
      static_limited = limited;
    } else {
      ptl = static_ptl;
      limited = static_limited;
      if (c->bad_pending) {  // the previous cycle's non-finite flag, before the next step reuses it
        CUDA_TRY(cudaStreamSynchronize(c->s));
        rc = check_pending_bad(c);
        if (rc) break;
      }
    }
    double dt;
    if (!limited) {
      dt = remaining;
    } else {
      dt = ptl >= floor_dt ? ptl : floor_dt;  // Python max(ptl, floor)
      if (dt >= remaining) dt = remaining;
    }
    int iters = 0;
    double rel = 0.0;
    if (scheme == PC_RKL2 || scheme == PC_RKG2) {
      int s = pc_sts_count(scheme, dt, dtE, make_odd);
      tab.assign(5 * (size_t)s, 0.0);
      rc = pc_sts_table(scheme, s, dt, tab.data());
      if (rc) break;
      if (gp.on) cudaEventRecord(gp.cur[2], c->s);
      const auto h0 = std::chrono::steady_clock::now();
      rc = sts_any(op, u, tab.data(), s, y0, true);
      if (gp.on) {
        gp.host += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count();
        cudaEventRecord(gp.cur[3], c->s);
        gp.flush();
      }
      iters = s;
    } else if (scheme == PC_BE) {
      int conv = 0;
      rc = be_step(op, u, dt, tol, max_iter, &iters, &rel, &conv);
      if (rc == PC_OK && !conv) rc = fail(PC_E_NOTCONV, "PCG did not converge within max_iter", iters);
    } else {
      Work A;
      rc = work_get(g, op->ncomp, A);
      if (rc) break;
      CUDA_TRY(cudaMemsetAsync(c->bad, 0x7f, sizeof(int), c->s));
      k_stage1<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, op->ncomp, cfld(u), y0.cf(), A.f(), dt, c->bad);
      c->st.launches++;
      rc = check_launch("k_stage1");
      if (rc == PC_OK) swap_storage(u, A);
      work_put(A);
      iters = 1;
    }
    ++cyc;
    if (rec && *n_rec < rec_cap) {
      pc_cycle_record& R = rec[*n_rec];
      R.cycle = cyc;
      R.dt = dt;
      R.ptl_raw = limited ? ptl : INFINITY;
      R.relres = rel;
      R.limited = limited;
      R.iters = iters;
      ++*n_rec;
    }
    if (rc) break;
    if (dt == remaining) remaining = 0.0;
    else remaining = remaining - dt;
  }
  work_put(y0);
  if (gp.on) {
    if (gp.n)
      fprintf(stderr,
              "[gap] cycles %ld  per cycle us: F+argmax+pairs %.1f  read+turnaround %.1f  stages %.1f  (host in "
              "sts %.1f)\n",
              gp.n, 1e3 * gp.t[0] / gp.n, 1e3 * gp.t[1] / gp.n, 1e3 * gp.t[2] / gp.n, gp.host / gp.n);
    for (auto e : gp.cur) c->ev_free.push_back(e);
  }
  if (rc == PC_OK) {
    CUDA_TRY(cudaStreamSynchronize(c->s));
    rc = check_pending_bad(c);
  }
  c->bad_pending = false;
  return rc;
}
