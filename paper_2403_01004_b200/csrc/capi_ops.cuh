// paracycle_b200 C ABI, part of the single translation unit capi.cu (included
// there in order; relies on the declarations of the parts before it).
//
// C ABI: operator construction and freezing (coefficients, Gershgorin bound,
// radial-density detection), and the launchers of the marching kernels
// (TMA / cp.async Spitzer march, 7-point march) every scheme goes through
#pragma once

// ------------------------------------------------------------------ operators
int pc_op_create_scalar(pc_grid* g, int ncomp, int vector_metric, double D_const, const pc_field* D,
                        const pc_field* rho, pc_op** out) {
  field_dep(D); field_dep(rho);
  if (!g || !out || ncomp < 1 || ncomp > 3) return fail(PC_E_INVALID, "bad scalar operator arguments");
  if (vector_metric && ncomp != 3) return fail(PC_E_INVALID, "vector metric needs 3 components");
  if ((D && D->ncomp != 1) || (rho && rho->ncomp != 1)) return fail(PC_E_INVALID, "D and rho are scalar fields");
  pc_op* op = new pc_op();
  op->grid = g;
  op->kind = K_SCALAR;
  op->ncomp = ncomp;
  op->so.D = D ? D->base(0) : nullptr;
  op->so.Dc = D_const;
  op->so.drho = 0;
  op->so.rho = rho ? rho->base(0) : nullptr;
  op->so.ncomp = ncomp;
  op->so.vector = (vector_metric && g->g.spherical) ? 1 : 0;
  op->deps[0] = D;
  op->deps[1] = rho;
  *out = op;
  return PC_OK;
}

int pc_op_create_viscous(pc_grid* g, int ncomp, int vector_metric, double nu, const pc_field* rho, pc_op** out) {
  field_dep(rho);
  if (!rho || rho->ncomp != 1) return fail(PC_E_INVALID, "viscous operator needs a scalar density field");
  if (!(nu >= 0.0)) return fail(PC_E_INVALID, "nu must be >= 0");
  TRY(pc_op_create_scalar(g, ncomp, vector_metric, nu, nullptr, rho, out));
  (*out)->so.drho = 1;
  return PC_OK;
}

int pc_op_create_aligned(pc_grid* g, const pc_field* bhat, const pc_field* rho, double pref, double kappa0,
                         const double* fc_table, double T_floor, pc_op** out) {
  field_dep(bhat); field_dep(rho);
  if (!g || !out || !bhat || bhat->ncomp != 3) return fail(PC_E_INVALID, "aligned operator needs a 3-component b");
  if (rho && rho->ncomp != 1) return fail(PC_E_INVALID, "rho is a scalar field");
  pc_ctx* c = g->ctx;
  pc_op* op = new pc_op();
  op->grid = g;
  op->kind = K_ALIGNED;
  op->ncomp = 1;
  for (int q = 0; q < 3; ++q) op->bsrc[q] = bhat->base(q);
  op->deps[0] = bhat;
  op->deps[1] = rho;
  op->ao.rho = rho ? rho->base(0) : nullptr;
  op->ao.pref = pref;
  op->ao.npref = 0.0 - pref;
  op->ao.ncomp = 1;
  op->Tfloor = T_floor;
  const int rows = g->g.n0 + 2;
  std::vector<double> k(rows);
  for (int r = 0; r < rows; ++r) k[r] = fc_table ? kappa0 * fc_table[r] : kappa0;
  CUDA_TRY(cudaMalloc(&op->kfc, sizeof(double) * rows));
  CUDA_TRY(cudaMemcpy(op->kfc, k.data(), sizeof(double) * rows, cudaMemcpyHostToDevice));
  if (!(op->betabuf = pool_get(c, 3 * g->comp_elems))) {
    cudaFree(op->kfc);
    delete op;
    return fail(PC_E_CUDA, "beta allocation failed (out of device memory)");
  }
  cudaMemsetAsync(op->betabuf, 0, 3 * g->comp_elems * sizeof(double), c->s);
  for (int q = 0; q < 3; ++q) op->ao.beta[q] = op->betabuf + q * g->comp_elems + g->g.plane;
  *out = op;
  return PC_OK;
}

int pc_op_set_preconditioner(pc_op* op, int pc) {
  if (!op) return fail(PC_E_INVALID, "null operator");
  if (pc != PC_PC_JACOBI && pc != PC_PC_LINE_R) return fail(PC_E_INVALID, "unknown preconditioner");
  if (pc == PC_PC_LINE_R && op->kind != K_ALIGNED)
    return fail(PC_E_INVALID, "the r-line preconditioner is built for the aligned operator");
  if (pc == PC_PC_LINE_R && op->grid->ctx->nranks > 1)
    return fail(PC_E_INVALID, "the r-line preconditioner needs the whole r line on one rank");
  op->pc = pc;
  return PC_OK;
}

int pc_op_set_refresh(pc_op* op, int per_cycle) {
  if (!op) return fail(PC_E_INVALID, "null operator");
  if (per_cycle && op->kind != K_ALIGNED) return fail(PC_E_INVALID, "per-cycle T0 refresh needs an aligned operator");
  op->refresh_cycle = per_cycle != 0;
  return PC_OK;
}

int pc_op_destroy(pc_op* op) {
  if (!op) return PC_OK;
  pc_ctx* c = op->grid->ctx;
  const size_t ce = op->grid->comp_elems;
  if (op->lbuf) pool_put(c, 2 * ce, op->lbuf);
  pool_put(c, 3 * ce, op->betabuf);
  pool_put(c, ce, op->dbuf);
  if (op->rho_r) cudaFree(op->rho_r);
  cudaFree(op->kfc);
  delete op;
  return PC_OK;
}

template <class Op>
static int run_bound(pc_op* op, const Op& o) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  int nb = node_blocks(c, g->g);
  k_bound<<<nb, kThreads, 0, c->s>>>(g->g, o, op->dbuf ? op->dbuf + g->g.plane : nullptr, c->red_v, c->counter,
                                     c->maxout);
  c->st.launches++;
  TRY(check_launch("k_bound"));
  TRY(allreduce_d(c, c->maxout, 1, nccl::kMax));
  CUDA_TRY(cudaMemcpyAsync(c->h_maxout, c->maxout, sizeof(double), cudaMemcpyDeviceToHost, c->s));
  CUDA_TRY(cudaStreamSynchronize(c->s));
  op->lam_max = *c->h_maxout;
  op->dt_euler = op->lam_max > 0.0 ? 2.0 / op->lam_max : INFINITY;
  return PC_OK;
}

// a density field that is constant on every r-plane (C5's rho(r)) is read by
// the TMA march as one per-plane value (8 B/cell less per stage); the values
// are the field's own, so results are bitwise unchanged
static int detect_radial_rho(pc_op* op) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  op->ao.rho_r = nullptr;
  op->ao.nsc_r = nullptr;
  if (!op->ao.rho || getenv("PC_NO_RADIAL_RHO")) return PC_OK;
  CUDA_TRY(cudaMemsetAsync(c->bad, 0, sizeof(int), c->s));
  k_radial_check<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, op->ao.rho, c->bad);
  c->st.launches++;
  TRY(check_launch("k_radial_check"));
  CUDA_TRY(cudaMemcpyAsync(c->h_bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->s));
  CUDA_TRY(cudaStreamSynchronize(c->s));
  if (*c->h_bad != 0) return PC_OK;  // not radial
  if (!op->rho_r) CUDA_TRY(cudaMalloc(&op->rho_r, 2 * sizeof(double) * (size_t)g->g.n0));
  CUDA_TRY(cudaMemcpy2DAsync(op->rho_r, sizeof(double), op->ao.rho + g->g.phis, (size_t)g->g.plane * sizeof(double), sizeof(double),
                             (size_t)g->g.n0, cudaMemcpyDeviceToDevice, c->s));
  // the per-plane scale 0 - pref / rho(i) (the node path divides per node: same value)
  k_neg_scale<<<(g->g.n0 + kThreads - 1) / kThreads, kThreads, 0, c->s>>>(op->rho_r, g->g.n0, op->ao.pref,
                                                                          op->rho_r + g->g.n0);
  c->st.launches++;
  TRY(check_launch("k_neg_scale"));
  op->ao.rho_r = op->rho_r;
  op->ao.nsc_r = op->rho_r + g->g.n0;
  return PC_OK;
}

// the same for the 3-component viscosity (D = nu rho) on one rank: the vector
// march reads rho(i) and 1 / rho(i) per plane instead of staging a rho stream
static int detect_radial_rho_visc(pc_op* op) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  op->so.rho_r = nullptr;
  const GridDev& d = g->g;
  if (!op->so.drho || !op->so.rho || !op->so.vector || op->ncomp != 3 || d.ghost_lo0 || d.ghost_hi0 || d.phis ||
      getenv("PC_NO_RADIAL_RHO"))
    return PC_OK;
  CUDA_TRY(cudaMemsetAsync(c->bad, 0, sizeof(int), c->s));
  k_radial_check<<<node_blocks(c, d), kThreads, 0, c->s>>>(d, op->so.rho, c->bad);
  c->st.launches++;
  TRY(check_launch("k_radial_check"));
  CUDA_TRY(cudaMemcpyAsync(c->h_bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->s));
  CUDA_TRY(cudaStreamSynchronize(c->s));
  if (*c->h_bad != 0) return PC_OK;  // not radial
  if (!op->rho_r) CUDA_TRY(cudaMalloc(&op->rho_r, 2 * sizeof(double) * (size_t)d.n0));
  CUDA_TRY(cudaMemcpy2DAsync(op->rho_r, sizeof(double), op->so.rho, (size_t)d.plane * sizeof(double), sizeof(double),
                             (size_t)d.n0, cudaMemcpyDeviceToDevice, c->s));
  k_recip<<<(d.n0 + kThreads - 1) / kThreads, kThreads, 0, c->s>>>(op->rho_r, d.n0, op->rho_r + d.n0);
  c->st.launches++;
  TRY(check_launch("k_recip"));
  op->so.rho_r = op->rho_r;
  return PC_OK;
}

int pc_op_freeze(pc_op* op, const pc_field* T0) {
  field_dep(T0);
  if (!op) return fail(PC_E_INVALID, "null operator");
  op_deps(op);
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  if (op->kind == K_ALIGNED) {
    if (!T0 || T0->ncomp != 1 || T0->grid != g) return fail(PC_E_INVALID, "aligned freeze needs a scalar T0 on the grid");
    CUDA_TRY(cudaMemsetAsync(c->bad, 0x7f, sizeof(int), c->s));
    CFld bsrc{{op->bsrc[0], op->bsrc[1], op->bsrc[2]}};
    Fld beta{{const_cast<double*>(op->ao.beta[0]), const_cast<double*>(op->ao.beta[1]),
              const_cast<double*>(op->ao.beta[2])}};
    // beta on the interior AND the existing ghost planes (pointwise in T0 and
    // b, whose ghost planes are exchanged first): no beta exchange needed
    {
      double* tb[1] = {const_cast<double*>(T0->buf[0])};
      TRY(halo_exchange(c, g, tb, 1));
      double* bb[3] = {const_cast<double*>(op->bsrc[0]) - g->g.plane, const_cast<double*>(op->bsrc[1]) - g->g.plane,
                       const_cast<double*>(op->bsrc[2]) - g->g.plane};
      TRY(halo_exchange(c, g, bb, 3));
    }
    GridDev gx = g->g;
    const int glo = g->g.ghost_lo0 ? 1 : 0, ghi = g->g.ghost_hi0 ? 1 : 0;
    gx.n0 = g->g.n0 + glo + ghi;
    const int64_t sh = -(int64_t)glo * g->g.plane;
    CFld bx{{bsrc.p[0] + sh, bsrc.p[1] + sh, bsrc.p[2] + sh}};
    Fld betax{{beta.p[0] + sh, beta.p[1] + sh, beta.p[2] + sh}};
    k_aligned_beta<<<node_blocks(c, gx), kThreads, 0, c->s>>>(gx, T0->base(0) + sh, op->kfc + 1 - glo, op->Tfloor,
                                                              bx, betax, c->bad);
    c->st.launches++;
    TRY(check_launch("k_aligned_beta"));
    CUDA_TRY(cudaMemcpyAsync(c->h_bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CUDA_TRY(cudaStreamSynchronize(c->s));
    if (*c->h_bad == 1) return fail(PC_E_DOMAIN, "aligned conduction: non-positive T0 (SPEC.md:120)");
    TRY(run_bound(op, op->ao));
    TRY(detect_radial_rho(op));
  } else {
    // the face coefficient D (or nu rho) is read at the axis-0 neighbours:
    // refresh the ghost planes of the coefficient fields
    if (op->so.D) {
      double* db[1] = {const_cast<double*>(op->so.D) - g->g.plane};
      TRY(halo_exchange(c, g, db, 1));
    }
    if (op->so.rho) {
      double* rb[1] = {const_cast<double*>(op->so.rho) - g->g.plane};
      TRY(halo_exchange(c, g, rb, 1));
    }
    TRY(run_bound(op, op->so));
    TRY(detect_radial_rho_visc(op));
  }
  op->diag_valid = op->dbuf != nullptr;
  op->line_valid = false;
  if (op->dbuf) {
    double* db[1] = {op->dbuf};
    TRY(halo_exchange(c, g, db, 1));
  }
  op->frozen = true;
  return PC_OK;
}

// the Jacobi diagonal is only materialised for BE / PCG / pc_op_diagonal
static int ensure_diag(pc_op* op) {
  if (op->diag_valid) return PC_OK;
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  if (!op->dbuf) {
    if (!(op->dbuf = pool_get(g->ctx, g->comp_elems)))
      return fail(PC_E_CUDA, "diagonal allocation failed (out of device memory)");
    CUDA_TRY(cudaMemsetAsync(op->dbuf, 0, g->comp_elems * sizeof(double), c->s));
  }
  if (op->kind == K_ALIGNED) TRY(run_bound(op, op->ao));
  else TRY(run_bound(op, op->so));
  double* db[1] = {op->dbuf};
  TRY(halo_exchange(c, g, db, 1));
  op->diag_valid = true;
  return PC_OK;
}

int pc_op_euler_dt(pc_op* op, double* dt) {
  if (!op || !dt) return fail(PC_E_INVALID, "null argument");
  if (!op->frozen) TRY(pc_op_freeze(op, nullptr));
  *dt = op->dt_euler;
  return PC_OK;
}

int pc_op_diagonal(pc_op* op, pc_field* out) {
  field_dep(out);
  if (!op || !out || out->ncomp != 1) return fail(PC_E_INVALID, "diagonal output must be a scalar field");
  op_deps(op);
  if (!op->frozen) TRY(pc_op_freeze(op, nullptr));
  TRY(ensure_diag(op));
  CUDA_TRY(cudaMemcpyAsync(out->buf[0], op->dbuf, op->grid->comp_elems * sizeof(double),
                           cudaMemcpyDeviceToDevice, op->grid->ctx->s));
  CUDA_TRY(cudaStreamSynchronize(op->grid->ctx->s));
  return PC_OK;
}

// r-chunk partition of a marching launch (ctx->zpart): the interior chunks
// (1 .. nz-2) or the two boundary chunks, whose ghost-plane reads wait for
// the halo exchange
static int zsplit(const pc_ctx* c, dim3& grid) {
  const int nz = (int)grid.z;
  if (c->zpart == 1) {
    grid.z = nz - 2;
    return 1;
  }
  if (c->zpart == 2) {
    grid.z = nz > 1 ? 2 : 1;
    return -nz;
  }
  return 0;
}

// r-chunk length of the marching aligned kernels
static int march_R(const pc_grid* g) {
  // r-chunk length: a block marches R planes after a one-plane prologue, so
  // the device time is ~ ceil(blocks / resident slots) x (R + 1) plane-steps;
  // pick the R (4 .. 128) that maximises useful plane-steps per slot-step
  // (PC_MARCH_R overrides, for experiments)
  if (const char* e = getenv("PC_MARCH_R")) {
    const int r = atoi(e);
    if (r >= 1) return r;
  }
  const int64_t tiles = (int64_t)((g->g.n2 + MTK - 1) / MTK) * ((g->g.n1 + MTJ - 1) / MTJ);
  const int64_t slots = (int64_t)g->ctx->sms * 2;  // 2 resident blocks per SM
  const int n0 = g->g.n0;
  int best = 4;
  double best_eff = -1.0;
  const bool slab = g->g.ghost_lo0 || g->g.ghost_hi0;  // keep >= 3 chunks: interior chunks overlap the halo exchange
  for (int R = 4; R <= 128; R += 4) {
    if (slab && (n0 + R - 1) / R < 3 && R > 4) continue;
    const int64_t blocks = tiles * ((n0 + R - 1) / R);
    const int64_t waves = (blocks + slots - 1) / slots;
    const double eff = (double)n0 * tiles / ((double)waves * slots * (R + 1));
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = R;
    }
  }
  return best;
}
static dim3 march_grid(const pc_grid* g, int R) {
  return dim3((g->g.n2 + MTK - 1) / MTK, (g->g.n1 + MTJ - 1) / MTJ, (g->g.n0 + R - 1) / R);
}
// ---- TMA (bulk tensor copy) maps over a field component [n0+2][n1][n2]
static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static int state = 0;
  if (state == 0) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && p) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
      state = 1;
    } else {
      state = -1;
    }
  }
  return fn;
}
// base = first interior element (plane 0); the tensor starts at ghost plane -1
static int make_field_map(CUtensorMap* m, const double* base, const GridDev& g, unsigned box0, unsigned box1) {
  auto enc = tma_encoder();
  if (!enc) return fail(PC_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const double* alloc = base - g.plane;
  cuuint64_t dims[3] = {(cuuint64_t)g.n2, (cuuint64_t)g.n1, (cuuint64_t)g.n0 + 2};
  cuuint64_t strides[2] = {(cuuint64_t)g.n2 * 8, (cuuint64_t)g.plane * 8};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(alloc), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PC_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return PC_OK;
}
// interleaved per-(r, theta) metric records [n0+2][n1][12] (iL2[6], wo01[4],
// iVal2, 0) for the TMA march: one 12 x 18 box per plane
static int make_rows_map(pc_grid* g) {
  auto enc = tma_encoder();
  if (!enc) return fail(PC_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const GridDev& d = g->g;
  cuuint64_t dims[3] = {(cuuint64_t)RW, (cuuint64_t)d.n1, (cuuint64_t)d.n0 + 2};
  cuuint64_t strides[2] = {(cuuint64_t)RW * 8, (cuuint64_t)d.n1 * RW * 8};
  cuuint32_t box[3] = {(cuuint32_t)RW, (cuuint32_t)MHJ, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&g->rowmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g->rowrec, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PC_E_CUDA, "cuTensorMapEncodeTiled (row records) failed (" + std::to_string((int)r) + ")");
  g->rowmap_ok = true;
  return PC_OK;
}
// a tensor map of a field buffer from the grid's cache (encoded on a miss)
static int cached_map(pc_grid* g, CUtensorMap* out, const double* base, unsigned box0, unsigned box1) {
  for (const auto& e : g->mapcache)
    if (e.base == base && e.b0 == box0 && e.b1 == box1) {
      *out = e.m;
      return PC_OK;
    }
  TRY(make_field_map(out, base, g->g, box0, box1));
  if (g->mapcache.size() >= 96) g->mapcache.erase(g->mapcache.begin());
  g->mapcache.push_back({base, box0, box1, *out});
  return PC_OK;
}
static bool tma_ok(const pc_grid* g) {
  const GridDev& d = g->g;
  // (phi-slabs: the periodic phi strips of the TMA boxes would wrap across
  // the ghost columns -- the cp.async march reads them as ordinary columns)
  return d.per2 && !d.phis && d.n2 % MTK == 0 && !d.per1 && d.n2 >= 2 && tma_encoder() != nullptr &&
         getenv("PC_NO_TMA") == nullptr;
}
template <class Epi, int RHO>
static int launch_tma_t(pc_op* op, const TmaMaps& maps, const Epi& epi, const int* skip, const char* what) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  const int R = march_R(g);
  dim3 grid = march_grid(g, R);
  if ((int64_t)grid.x * grid.y * grid.z > c->max_red) return fail(PC_E_INVALID, "grid too large for the reduction scratch");
  const int smem = (int)sizeof(TmaSmem) + 128;
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(k_aligned_tma<Epi, RHO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const int zsel = zsplit(c, grid);
  static const int split = getenv("PC_TMA_SPLIT") ? atoi(getenv("PC_TMA_SPLIT")) : 2;  // TMA issuer warps - 1
  AlignedOp ao = op->ao;
  ao.tma_split = split;
  k_aligned_tma<Epi, RHO><<<grid, dim3(MTK, MTY), smem, c->s>>>(g->g, ao, maps, epi, R, zsel, skip);
  c->st.launches++;
  return check_launch(what);
}
template <class Epi>
static int launch_tma(pc_op* op, const double* Tin, const Epi& epi, const int* skip, const char* what) {
  pc_grid* g = op->grid;
  TmaMaps maps;
  if (!op->beta_maps) {
    for (int q = 0; q < 3; ++q) {
      TRY(make_field_map(&op->bmap[q], op->ao.beta[q], g->g, MTK, MHJ));
      TRY(make_field_map(&op->bsmap[q], op->ao.beta[q], g->g, 2, MHJ));
    }
    op->beta_maps = true;
  }
  if (!g->rowmap_ok) {
    TRY(make_rows_map(g));
  }
  for (int q = 0; q < 3; ++q) {
    maps.B[q] = op->bmap[q];
    maps.BS[q] = op->bsmap[q];
  }
  maps.RW = g->rowmap;
  TRY(make_field_map(&maps.T, Tin, g->g, MTK, MHJ));
  TRY(make_field_map(&maps.TS, Tin, g->g, 2, MHJ));
  for (int q = 0; q < Epi::NOPS; ++q) TRY(make_field_map(&maps.O[q], epi.opnd(q), g->g, MTK, MTJ));
  if constexpr (fusep_of<Epi>::value) {  // fused PCG matvec: p_old and d boxes beside r (= Tin)
    TRY(make_field_map(&maps.P[0], epi.pold, g->g, MTK, MHJ));
    TRY(make_field_map(&maps.PS[0], epi.pold, g->g, 2, MHJ));
    TRY(make_field_map(&maps.P[1], epi.dinv, g->g, MTK, MHJ));
    TRY(make_field_map(&maps.PS[1], epi.dinv, g->g, 2, MHJ));
  }
  if constexpr (fuse1_of<Epi>::value) {  // fused STS stages 1 + 2: y0 boxes beside u0 (= Tin)
    TRY(make_field_map(&maps.P[0], epi.y0, g->g, MTK, MHJ));
    TRY(make_field_map(&maps.PS[0], epi.y0, g->g, 2, MHJ));
  }
  if (op->ao.rho && op->ao.rho_r) return launch_tma_t<Epi, 2>(op, maps, epi, skip, what);
  if (op->ao.rho) return launch_tma_t<Epi, 1>(op, maps, epi, skip, what);
  return launch_tma_t<Epi, 0>(op, maps, epi, skip, what);
}

template <class Epi>
static int launch_march(pc_op* op, const double* Tin, const Epi& epi, const int* skip, const char* what) {
  if (tma_ok(op->grid)) return launch_tma(op, Tin, epi, skip, what);
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  const int R = march_R(g);
  dim3 grid = march_grid(g, R);
  if ((int64_t)grid.x * grid.y * grid.z > c->max_red) return fail(PC_E_INVALID, "grid too large for the reduction scratch");
  static bool attr = false;  // one per template instantiation
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(k_aligned_march<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(MarchSmem)));
    attr = true;
  }
  const int zsel = zsplit(c, grid);
  k_aligned_march<Epi><<<grid, dim3(MTK, MTY), sizeof(MarchSmem), c->s>>>(g->g, op->ao, Tin, epi, R, zsel, skip);
  c->st.launches++;
  return check_launch(what);
}

// ---- 7-point marching kernels (ScalarOp), dispatched on (ncomp, vector, D mode)
// r-chunk length: the longest power of two (<= 32) that still gives ~12 blocks
// per SM (3 resident, scalar) or ~6 (2 resident, 3-component); measured on C2:
// R = 4 / 8 / 16 / 32 -> 2.49 / 2.77 / 2.92 / 2.83e10 cell-updates/s.
static bool vmarch_ok(const pc_grid* g);
static int smarch_R(const pc_grid* g, int ncomp) {
  if (const char* e = getenv("PC_SMARCH_R")) {
    const int r = atoi(e);
    if (r >= 1) return r;
  }
  if (ncomp == 3 && vmarch_ok(g)) {
    // the vector march: a block marches R planes after a prologue of about two
    // (four planes staged, two formed), so the device time is ~ ceil(blocks /
    // resident slots) x (R + 2) plane-steps; take the R (4 .. 64) with the most
    // useful plane-steps per slot-step among those that keep >= 3 blocks per
    // slot (C2: R = 15 fills 3.9 waves where 16 left the fourth half empty)
    const int64_t tiles = (int64_t)((g->g.n2 + MTK - 1) / MTK) * ((g->g.n1 + SMJ - 1) / SMJ);
    const int64_t slots = (int64_t)g->ctx->sms * 2;
    const int n0 = g->g.n0;
    const bool slab = g->g.ghost_lo0 || g->g.ghost_hi0;  // keep >= 3 chunks (interior / boundary overlap)
    int best = 4;
    double best_eff = -1.0;
    for (int R = 4; R <= 64; ++R) {
      if (slab && (n0 + R - 1) / R < 3 && R > 4) continue;
      const int64_t blocks = tiles * ((n0 + R - 1) / R);
      // (fewer than ~3 blocks per slot: the co-resident blocks speed up as the
      // SM empties and the model's constant block time no longer holds)
      if (blocks < 3 * slots && R > 4) continue;
      const int64_t waves = (blocks + slots - 1) / slots;
      const double eff = (double)n0 * tiles / ((double)waves * slots * (R + 2));
      if (eff > best_eff + 1e-9) {
        best_eff = eff;
        best = R;
      }
    }
    return best;
  }
  const int tiles = ((g->g.n2 + MTK - 1) / MTK) * ((g->g.n1 + SMJ - 1) / SMJ);
  const int64_t want = ncomp == 3 ? 148 * 6 : 148 * 12;
  int R = 32;
  while (R > 4 && (int64_t)tiles * ((g->g.n0 + R - 1) / R) < want) R /= 2;
  return R;
}
static bool smarch_ok(const pc_op* op) { return op->ncomp == 1 || op->ncomp == 3; }
// TMA staging for the 7-point march (opt-in: PC_SMARCH_TMA=1): phi periodic
// with whole 32-column tiles, theta not periodic, not a phi-slab.  Measured
// against the cp.async staging on the same box it is no faster (C2 -2..-10 %,
// C5v +2 % on the fused stage 1+2, -3 % on the plain stage;
// profiles/r02_smarch_tma_ab.txt): the per-thread cp.async issue it removes is
// not what bounds the 3-component stencil, so cp.async stays the default
static bool smarch_tma_ok(const pc_grid* g) {
  const GridDev& d = g->g;
  static const bool on = getenv("PC_SMARCH_TMA") != nullptr && getenv("PC_SMARCH_TMA")[0] == '1';
  return on && d.per2 && !d.phis && d.n2 % MTK == 0 && !d.per1 && d.n2 >= 2 && tma_encoder() != nullptr;
}
template <class E, class = void>
struct has_y0 : std::false_type {};
template <class E>
struct has_y0<E, std::void_t<decltype(&E::y0)>> : std::true_type {};

// the vector march (k_vec_march, vmarch.cuh) for y0 = F(u0) + argmax and the
// fused stages 1 + 2 of the 3-component spherical operator: phi periodic in
// whole 32-column tiles, theta not periodic, no theta / phi pinning, not a
// phi-slab (PC_NO_VMARCH=1 keeps k_scalar_march; bitwise the same)
static bool vmarch_ok(const pc_grid* g) {
  const GridDev& d = g->g;
  const char* e = getenv("PC_NO_VMARCH");
  const bool off = e != nullptr && e[0] == '1';
  return !off && d.spherical && d.per2 && !d.phis && d.n2 % MTK == 0 && !d.per1 && d.n2 >= 2 && !d.pin_lo1 &&
         !d.pin_hi1 && !d.pin_lo2 && !d.pin_hi2 && tma_encoder() != nullptr;
}
// the vector march's per-(r, theta) records: W2[0], W2[1], W2[2], iV2 interleaved
// over the table rows -1 .. n0 (the same bits), one 4 x 10 TMA box per plane
__global__ void k_srow_pack(GridDev g, double* rec, int64_t nrows) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nrows; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = q - g.n1;  // (the tables start at ghost row -1)
    rec[4 * q + 0] = g.W2[0][s];
    rec[4 * q + 1] = g.W2[1][s];
    rec[4 * q + 2] = g.W2[2][s];
    rec[4 * q + 3] = g.iV2[s];
  }
}
static int make_srow_map(pc_grid* g) {
  auto enc = tma_encoder();
  if (!enc) return fail(PC_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const GridDev& d = g->g;
  const int64_t nrows = (int64_t)(d.n0 + 2) * d.n1;
  if (!g->srowrec) CUDA_TRY(cudaMalloc(&g->srowrec, sizeof(double) * 4 * nrows));
  k_srow_pack<<<(int)std::min<int64_t>((nrows + 255) / 256, 4096), 256, 0, g->ctx->s>>>(d, g->srowrec, nrows);
  g->ctx->st.launches++;
  TRY(check_launch("k_srow_pack"));
  cuuint64_t dims[3] = {4, (cuuint64_t)d.n1, (cuuint64_t)d.n0 + 2};
  cuuint64_t strides[2] = {4 * 8, (cuuint64_t)d.n1 * 4 * 8};
  cuuint32_t box[3] = {4, (cuuint32_t)SHJ, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&g->srowmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g->srowrec, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    cudaFree(g->srowrec);
    g->srowrec = nullptr;
    return fail(PC_E_CUDA, "cuTensorMapEncodeTiled (vector row records) failed (" + std::to_string((int)r) + ")");
  }
  g->srow_ok = true;
  return PC_OK;
}
template <int DM, class Epi>
static int launch_vmarch(pc_op* op, CFld u, const Epi& epi, const int* skip, dim3 grid, int R, int zsel,
                         const char* what) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  constexpr bool F1 = fuse1_of<Epi>::value;
  if (!g->srow_ok) TRY(make_srow_map(g));
  SMaps maps;
  for (int q = 0; q < 3; ++q) {
    TRY(cached_map(g, &maps.V[q], u.p[q], MTK, SHJ));
    TRY(cached_map(g, &maps.VS[q], u.p[q], 2, SHJ));
  }
  if (DM == 1 || DM == 2) {
    const double* d = DM == 1 ? op->so.D : op->so.rho;
    TRY(cached_map(g, &maps.D, d, MTK, SHJ));
    TRY(cached_map(g, &maps.DS, d, 2, SHJ));
  }
  if constexpr (F1) {
    for (int q = 0; q < 3; ++q) {
      TRY(cached_map(g, &maps.Y[q], epi.y0[q], MTK, SHJ));
      TRY(cached_map(g, &maps.YS[q], epi.y0[q], 2, SHJ));
    }
  } else {
    for (int q = 0; q < Epi::NOPS; ++q) TRY(cached_map(g, &maps.O[q], epi.opnd(q), MTK, SMJ));
  }
  const int smem = (int)sizeof(VMarchSmem<F1, DM, F1 ? 0 : Epi::NOPS>) + 128;  // (+ the 128-byte alignment of the boxes)
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(k_vec_march<DM, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  k_vec_march<DM, Epi><<<grid, SNT, smem, c->s>>>(g->g, op->so, epi, R, zsel, skip, maps, g->srowmap);
  c->st.launches++;
  return check_launch(what);
}

template <int NC, bool VEC, int DM, class Epi>
static int launch_smarch_t(pc_op* op, CFld u, const Epi& epi, const int* skip, const char* what) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  const int R = smarch_R(g, NC);
  dim3 grid((g->g.n2 + MTK - 1) / MTK, (g->g.n1 + SMJ - 1) / SMJ, (g->g.n0 + R - 1) / R);
  if ((int64_t)grid.x * grid.y * grid.z > c->max_red) return fail(PC_E_INVALID, "grid too large for the reduction scratch");
  constexpr bool F1 = fuse1_of<Epi>::value;
  const int zsel = zsplit(c, grid);
  if constexpr (NC == 3 && VEC && (F1 || std::is_same<Epi, SEpiArgmax>::value || std::is_same<Epi, SEpiStage>::value)) {
    if (vmarch_ok(g)) {
      if (DM == 2 && op->so.rho_r) return launch_vmarch<3>(op, u, epi, skip, grid, R, zsel, what);
      return launch_vmarch<DM>(op, u, epi, skip, grid, R, zsel, what);
    }
    const char* st = getenv("PC_VMARCH_STRICT");  // (tests: a vector launch that would fall back is an error)
    if (st && st[0] == '1' && !(getenv("PC_NO_VMARCH") && getenv("PC_NO_VMARCH")[0] == '1'))
      return fail(PC_E_INVALID, "k_vec_march not applicable to this grid (PC_VMARCH_STRICT)");
  }
  SMaps maps;
  if (smarch_tma_ok(g)) {
    const int smem = (int)sizeof(SMarchSmem<NC, F1, true>) + 128;  // (+ the 128-byte alignment of the boxes)
    static bool attr = false;
    if (!attr) {
      CUDA_TRY(cudaFuncSetAttribute(k_scalar_march<NC, VEC, DM, Epi, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr = true;
    }
    for (int q = 0; q < NC; ++q) {
      TRY(cached_map(g, &maps.V[q], u.p[q], MTK, SHJ));
      TRY(cached_map(g, &maps.VS[q], u.p[q], 2, SHJ));
    }
    if (DM != 0) {
      const double* d = DM == 1 ? op->so.D : op->so.rho;
      TRY(cached_map(g, &maps.D, d, MTK, SHJ));
      TRY(cached_map(g, &maps.DS, d, 2, SHJ));
    }
    if constexpr (F1) {
      if constexpr (has_y0<Epi>::value) {
        for (int q = 0; q < NC; ++q) {
          TRY(cached_map(g, &maps.Y[q], epi.y0[q], MTK, SHJ));
          TRY(cached_map(g, &maps.YS[q], epi.y0[q], 2, SHJ));
        }
      }
    } else {
      for (int q = 0; q < Epi::NOPS; ++q) TRY(cached_map(g, &maps.O[q], epi.opnd(q), MTK, SMJ));
    }
    k_scalar_march<NC, VEC, DM, Epi, true><<<grid, SNT, smem, c->s>>>(g->g, op->so, u.p[0], u.p[1], u.p[2], epi, R,
                                                                       zsel, skip, maps);
  } else {
    const int smem = (int)sizeof(SMarchSmem<NC, F1, false>);
    static bool attr = false;
    if (!attr) {
      CUDA_TRY(cudaFuncSetAttribute(k_scalar_march<NC, VEC, DM, Epi, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr = true;
    }
    k_scalar_march<NC, VEC, DM, Epi, false><<<grid, SNT, smem, c->s>>>(g->g, op->so, u.p[0], u.p[1], u.p[2], epi,
                                                                        R, zsel, skip, maps);
  }
  c->st.launches++;
  return check_launch(what);
}
template <int NC, class Epi>
static int launch_smarch_nc(pc_op* op, CFld u, const Epi& epi, const char* what) {
  const int dm = op->so.drho ? 2 : (op->so.D ? 1 : 0);
  const bool vec = NC == 3 && op->so.vector;
  if (vec) {
    if (dm == 0) return launch_smarch_t<NC, true, 0>(op, u, epi, nullptr, what);
    if (dm == 1) return launch_smarch_t<NC, true, 1>(op, u, epi, nullptr, what);
    return launch_smarch_t<NC, true, 2>(op, u, epi, nullptr, what);
  }
  if (dm == 0) return launch_smarch_t<NC, false, 0>(op, u, epi, nullptr, what);
  if (dm == 1) return launch_smarch_t<NC, false, 1>(op, u, epi, nullptr, what);
  return launch_smarch_t<NC, false, 2>(op, u, epi, nullptr, what);
}

template <class Op>
static int launch_apply(pc_op* op, const Op& o, CFld u, Fld F, bool argmax) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  int nb = node_blocks(c, g->g);
  if (argmax) {
    k_apply_argmax<<<nb, kThreads, 0, c->s>>>(g->g, o, u, F, c->red_v, c->red_i, c->counter, c->res);
  } else {
    k_apply<<<nb, kThreads, 0, c->s>>>(g->g, o, u, F);
  }
  c->st.launches++;
  return check_launch("k_apply");
}
static int apply_any(pc_op* op, CFld u, Fld F, bool argmax) {
  if (op->kind == K_ALIGNED) {
    pc_ctx* c = op->grid->ctx;
    if (argmax) {
      EpiArgmax e{F.p[0], c->red_v, c->red_i, c->counter, c->res, ArgMax{-1.0, 0x7fffffffffffffffLL}};
      return launch_march(op, u.p[0], e, nullptr, "k_aligned_march<argmax>");
    }
    return launch_march(op, u.p[0], EpiStore{F.p[0]}, nullptr, "k_aligned_march<apply>");
  }
  if (smarch_ok(op)) {
    pc_ctx* c = op->grid->ctx;
    if (argmax) {
      SEpiArgmax e{{F.p[0], F.p[1], F.p[2]}, c->red_v, c->red_i, c->counter, c->res,
                   ArgMax{-1.0, 0x7fffffffffffffffLL}, op->ncomp};
      return op->ncomp == 3 ? launch_smarch_nc<3>(op, u, e, "k_scalar_march<argmax>")
                            : launch_smarch_nc<1>(op, u, e, "k_scalar_march<argmax>");
    }
    SEpiStore e{{F.p[0], F.p[1], F.p[2]}};
    return op->ncomp == 3 ? launch_smarch_nc<3>(op, u, e, "k_scalar_march<apply>")
                          : launch_smarch_nc<1>(op, u, e, "k_scalar_march<apply>");
  }
  return launch_apply(op, op->so, u, F, argmax);
}

static int need_frozen(pc_op* op) {
  if (op->kind == K_ALIGNED && !op->frozen)
    return fail(PC_E_INVALID, "aligned operator: call pc_op_freeze(T0) first (lagged diffusivity)");
  if (!op->frozen) return pc_op_freeze(op, nullptr);  // scalar: coefficient ghost planes + bound
  return PC_OK;
}

int pc_op_apply(pc_op* op, const pc_field* u, pc_field* F) {
  field_dep(u); field_dep(F);
  if (!op || !u || !F || u->ncomp != op->ncomp || F->ncomp != op->ncomp) return fail(PC_E_INVALID, "shape mismatch");
  op_deps(op);
  TRY(need_frozen(op));
  TRY(halo_field(const_cast<pc_field*>(u)));
  TRY(apply_any(op, cfld(u), fld(F), false));
  CUDA_TRY(cudaStreamSynchronize(op->grid->ctx->s));
  return PC_OK;
}
