// paracycle_b200 C ABI, part of the single translation unit capi.cu (included
// there in order; relies on the declarations of the parts before it).
//
// C ABI: version / errors, contexts, timing, grids, fields (upload, download,
// ghost planes, domain counts) and pinned host memory
#pragma once

// ------------------------------------------------------------------ C ABI
// (entry points get C linkage from the extern "C" declarations in the header)

const char* pc_last_error(void) { return g_err.c_str(); }
int64_t pc_last_error_info(void) { return g_info; }
int pc_version(void) { return 1; }

int pc_nccl_unique_id(void* out128) {
  nccl::Api* A = nccl::api();
  if (!A) return fail(PC_E_NCCL, "NCCL library not found");
  if (A->getUniqueId(out128) != 0) return fail(PC_E_NCCL, "ncclGetUniqueId");
  return PC_OK;
}

static int ctx_create(int device, int nranks, int rank, const void* nccl_uid, bool detached, pc_ctx** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) return fail(PC_E_INVALID, "bad context arguments");
  CUDA_TRY(cudaSetDevice(device));
  pc_ctx* c = new pc_ctx();
  c->device = device;
  c->nranks = nranks;
  c->rank = rank;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  c->max_blocks = sms * 16;
  c->sms = sms;
  CUDA_TRY(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->sc, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
  CUDA_TRY(cudaMalloc(&c->red_v, sizeof(double) * c->max_red));
  CUDA_TRY(cudaMalloc(&c->red_v2, sizeof(double) * c->max_red));
  CUDA_TRY(cudaMalloc(&c->red_i, sizeof(long long) * c->max_red));
  CUDA_TRY(cudaMalloc(&c->counter, sizeof(unsigned int) * 4));
  CUDA_TRY(cudaMemset(c->counter, 0, sizeof(unsigned int) * 4));
  CUDA_TRY(cudaMalloc(&c->res, sizeof(ArgRes)));
  CUDA_TRY(cudaMalloc(&c->pcg, sizeof(PcgDev)));
  CUDA_TRY(cudaMalloc(&c->bad, sizeof(int)));
  CUDA_TRY(cudaMalloc(&c->minbits, sizeof(unsigned long long)));
  CUDA_TRY(cudaMalloc(&c->maxout, sizeof(double)));
  CUDA_TRY(cudaMalloc(&c->gath, sizeof(double) * 2 * nranks));
  CUDA_TRY(cudaMallocHost(&c->h_res, sizeof(ArgRes)));
  CUDA_TRY(cudaMallocHost(&c->h_pcg, sizeof(PcgDev)));
  CUDA_TRY(cudaMallocHost(&c->h_bad, sizeof(int)));
  CUDA_TRY(cudaMallocHost(&c->h_minbits, sizeof(unsigned long long)));
  CUDA_TRY(cudaMallocHost(&c->h_maxout, sizeof(double)));
  c->detached = detached;
  // PC_FORCE_NCCL (test hook): a one-rank communicator, so every collective
  // of the multi-rank path (allreduce, allgathered argmax, split PCG
  // reductions) runs through NCCL on a single GPU
  const bool force = nranks == 1 && !detached && getenv("PC_FORCE_NCCL") != nullptr;
  if ((nranks > 1 && !detached) || force) {
    nccl::Api* A = nccl::api();
    if (!A) {
      delete c;
      return fail(PC_E_NCCL, "NCCL library not found (needed for nranks > 1)");
    }
    char self_uid[128];
    if (!nccl_uid && force) {
      if (A->getUniqueId(self_uid) != 0) return fail(PC_E_NCCL, "ncclGetUniqueId");
      nccl_uid = self_uid;
    }
    if (!nccl_uid) return fail(PC_E_INVALID, "nranks > 1 needs an ncclUniqueId");
    if (A->commInitRank(&c->comm, nranks, nccl_uid, rank) != 0) return fail(PC_E_NCCL, "ncclCommInitRank");
  }
  *out = c;
  return PC_OK;
}
int pc_ctx_create(int device, int nranks, int rank, const void* nccl_uid, pc_ctx** out) {
  return ctx_create(device, nranks, rank, nccl_uid, false, out);
}
int pc_ctx_create_detached(int device, int nranks, int rank, pc_ctx** out) {
  return ctx_create(device, nranks, rank, nullptr, true, out);
}
int pc_ctx_set_decomposition(pc_ctx* c, int axis) {
  if (!c || (axis != 0 && axis != 2)) return fail(PC_E_INVALID, "decomposition axis must be 0 (r) or 2 (phi)");
  c->axis = axis;
  return PC_OK;
}

int pc_ctx_destroy(pc_ctx* c) {
  if (c) {
    if (c->sc) cudaStreamDestroy(c->sc);
    if (c->cs) {
      cudaStreamSynchronize(c->cs);
      cudaStreamDestroy(c->cs);
    }
    if (c->staging_cs) cudaFree(c->staging_cs);
    if (c->cyc_dev) cudaFree(c->cyc_dev);
    if (c->cyc_rec) cudaFree(c->cyc_rec);
    if (c->h_cyc) cudaFreeHost(c->h_cyc);
    if (c->ev_in) cudaEventDestroy(c->ev_in);
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  }
  if (!c) return PC_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->s);
  for (auto& p : c->pool) cudaFree(p.second);
  for (auto& e : c->ev) {
    cudaEventDestroy(e.e0);
    cudaEventDestroy(e.e1);
  }
  for (auto e : c->ev_free) cudaEventDestroy(e);
  if (c->comm) {
    nccl::Api* A = nccl::api();
    if (A) A->commDestroy(c->comm);
  }
  cudaFree(c->phibuf);
  cudaFree(c->pslot[0]);
  cudaFree(c->pslot[1]);
  cudaFree(c->pvec);
  cudaFree(c->pvec_all);
  cudaFree(c->red_v);
  cudaFree(c->red_v2);
  cudaFree(c->red_i);
  cudaFree(c->counter);
  cudaFree(c->res);
  cudaFree(c->pcg);
  cudaFree(c->bad);
  cudaFree(c->minbits);
  cudaFree(c->maxout);
  cudaFree(c->gath);
  cudaFree(c->staging);
  cudaFreeHost(c->h_res);
  cudaFreeHost(c->h_pcg);
  cudaFreeHost(c->h_bad);
  cudaFreeHost(c->h_minbits);
  cudaFreeHost(c->h_maxout);
  for (auto& m : c->marks)
    if (m) cudaEventDestroy(m);
  cudaStreamDestroy(c->s);
  delete c;
  return PC_OK;
}

int pc_ctx_sync(pc_ctx* c) {
  CUDA_TRY(cudaStreamSynchronize(c->s));
  return PC_OK;
}

int pc_ctx_mark(pc_ctx* c, int id) {
  if (!c || id < 0 || id >= 16) return fail(PC_E_INVALID, "mark id 0..15");
  if (!c->marks[id]) CUDA_TRY(cudaEventCreate(&c->marks[id]));
  CUDA_TRY(cudaEventRecord(c->marks[id], c->s));
  return PC_OK;
}
int pc_ctx_elapsed(pc_ctx* c, int id0, int id1, double* ms) {
  if (!c || id0 < 0 || id1 < 0 || id0 >= 16 || id1 >= 16 || !c->marks[id0] || !c->marks[id1] || !ms)
    return fail(PC_E_INVALID, "unknown marks");
  CUDA_TRY(cudaEventSynchronize(c->marks[id1]));
  float f = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&f, c->marks[id0], c->marks[id1]));
  *ms = f;
  return PC_OK;
}

int pc_ctx_enable_timing(pc_ctx* c, int on) {
  c->timing = on != 0;
  return PC_OK;
}
int pc_ctx_reset_stats(pc_ctx* c) {
  c->st = Stats();
  return PC_OK;
}
static void flush_events(pc_ctx* c) {
  for (auto& e : c->ev) {
    float ms = 0.f;
    cudaEventSynchronize(e.e1);
    cudaEventElapsedTime(&ms, e.e0, e.e1);
    c->st.stage_ms += ms;
    c->st.kind_ms[e.kind] += ms;
    c->ev_free.push_back(e.e0);
    c->ev_free.push_back(e.e1);
  }
  c->ev.clear();
}
int pc_ctx_stats_kind(pc_ctx* c, int kind, double* ms, int64_t* launches, int64_t* units) {
  if (!c || kind < 0 || kind >= NKIND) return fail(PC_E_INVALID, "stats kind 0..7");
  cudaStreamSynchronize(c->s);
  flush_events(c);
  if (ms) *ms = c->st.kind_ms[kind];
  if (launches) *launches = c->st.kind_launches[kind];
  if (units) *units = c->st.kind_units[kind];
  return PC_OK;
}

int pc_ctx_stats(pc_ctx* c, double* stage_ms, int64_t* stage_launches, int64_t* launches_total) {
  cudaStreamSynchronize(c->s);
  flush_events(c);
  if (stage_ms) *stage_ms = c->st.stage_ms;
  if (stage_launches) *stage_launches = c->st.stage_launches;
  if (launches_total) *launches_total = c->st.launches;
  return PC_OK;
}

// table layout (paper_2403_01004_b200/geometry.py TABLE_ORDER)
static void table_sizes(const int64_t shape[3], int64_t& A, int64_t& K, int64_t& J) {
  A = (shape[0] + 2) * shape[1];
  K = shape[2];
  J = shape[1];
}
int64_t pc_grid_table_size(const int64_t shape[3]) {
  int64_t A, K, J;
  table_sizes(shape, A, K, J);
  return 17 * A + 15 * K + 48 * J;
}

int pc_grid_create(pc_ctx* c, const int64_t shape[3], const int32_t* fl, const double* tables,
                   int64_t ntables, pc_grid** out) {
  if (!c || !shape || !fl || !tables || !out) return fail(PC_E_INVALID, "null argument");
  for (int a = 0; a < 3; ++a)
    if (shape[a] < 1) return fail(PC_E_INVALID, "grid shape must be positive");
  if (ntables != pc_grid_table_size(shape)) return fail(PC_E_INVALID, "table size mismatch");
  CUDA_TRY(cudaSetDevice(c->device));
  pc_grid* g = new pc_grid();
  g->ctx = c;
  for (int a = 0; a < 3; ++a) g->shape[a] = shape[a];
  GridDev& d = g->g;
  d.n0 = (int)shape[0];
  d.n1 = (int)shape[1];
  d.n2 = (int)shape[2];
  d.plane = shape[1] * shape[2];
  d.N = shape[0] * d.plane;
  d.per0 = fl[0];
  d.per1 = fl[1];
  d.per2 = fl[2];
  d.pin_lo0 = fl[3];
  d.pin_hi0 = fl[4];
  d.pin_lo1 = fl[5];
  d.pin_hi1 = fl[6];
  d.pin_lo2 = fl[7];
  d.pin_hi2 = fl[8];
  d.ghost_lo0 = fl[9];
  d.ghost_hi0 = fl[10];
  d.n0g = fl[11];
  d.i0g = fl[12];
  d.spherical = fl[13];
  d.phis = fl[14];
  d.n2g = fl[15];
  d.k0g = fl[16];
  if (d.phis) {
    if (c->axis != 2 || !d.per2 || !d.pin_lo2 || !d.pin_hi2 || d.n2 < 3 || d.ghost_lo0 || d.ghost_hi0 ||
        d.k0g < 0 || d.k0g + d.n2 - 2 > d.n2g) {
      delete g;
      return fail(PC_E_INVALID, "phi-slab grid: periodic phi, pinned ghost columns, a phi-decomposed context");
    }
  } else {
    d.n2g = d.n2;
    d.k0g = 0;
  }
  g->comp_elems = (size_t)(shape[0] + 2) * (size_t)d.plane;
  {  // the marching kernels rely on unit axis-0/1 column factors iL1 (geometry.py)
    int64_t A, K, J;
    table_sizes(shape, A, K, J);
    const double* iL1 = tables + 3 * A + 3 * K + A + K + 6 * A;
    for (int64_t q = 0; q < 4 * K; ++q)
      if (iL1[q] != 1.0) {
        delete g;
        return fail(PC_E_INVALID, "grid tables: axis-0/1 column factors iL1 must be 1");
      }
  }
  CUDA_TRY(cudaMalloc(&g->tables, sizeof(double) * ntables));
  CUDA_TRY(cudaMemcpy(g->tables, tables, sizeof(double) * ntables, cudaMemcpyHostToDevice));
  int64_t A, K, J;
  table_sizes(shape, A, K, J);
  const double* p = g->tables;
  auto takeA = [&]() { const double* r = p + d.n1; p += A; return r; };  // skip ghost row -1
  auto takeK = [&]() { const double* r = p; p += K; return r; };
  for (int a = 0; a < 3; ++a) d.W2[a] = takeA();
  for (int a = 0; a < 3; ++a) d.g1[a] = takeK();
  d.iV2 = takeA();
  d.igv = takeK();
  for (int q = 0; q < 6; ++q) d.iL2[q] = takeA();
  for (int q = 0; q < 6; ++q) d.iL1[q] = takeK();
  for (int q = 0; q < 4; ++q) d.wo01[q] = takeA();
  for (int q = 0; q < 2; ++q) d.wo2[q] = takeK();
  d.iVal2 = takeA();
  d.iValg = takeK();
  for (int q = 0; q < 4; ++q) { d.M[q] = p; p += J * 9; }
  for (int q = 0; q < 4; ++q) { d.Rabs[q] = p; p += J * 3; }
  d.V2 = takeA();
  d.gv = takeK();
  d.Val2 = takeA();
  d.Valg = takeK();
  {  // interleaved row records from the host copy of the tables (same bits)
    const double* h = tables + 3 * A + 3 * K + A + K;  // iL2[0]
    const double* hw = h + 6 * A + 6 * K;               // wo01[0]
    const double* hv = hw + 4 * A + 2 * K;              // iVal2
    const double* hV = hv + A + K + 48 * J + A + K;     // Val2 (after iValg, M, Rabs, V2, gv)
    std::vector<double> rec((size_t)A * RW, 0.0);
    for (int64_t q = 0; q < A; ++q) {
      double* r = rec.data() + q * RW;
      for (int t = 0; t < 6; ++t) r[t] = h[t * A + q];
      for (int t = 0; t < 4; ++t) r[6 + t] = hw[t * A + q];
      r[10] = hv[q];
      r[11] = hV[q];
    }
    CUDA_TRY(cudaMalloc(&g->rowrec, sizeof(double) * rec.size()));
    CUDA_TRY(cudaMemcpy(g->rowrec, rec.data(), sizeof(double) * rec.size(), cudaMemcpyHostToDevice));
  }
  *out = g;
  return PC_OK;
}

int pc_grid_destroy(pc_grid* g) {
  if (!g) return PC_OK;
  cudaFree(g->tables);
  cudaFree(g->rowrec);
  cudaFree(g->srowrec);
  delete g;
  return PC_OK;
}

int pc_field_create(pc_grid* g, int ncomp, pc_field** out) {
  if (!g || !out || ncomp < 1 || ncomp > 3) return fail(PC_E_INVALID, "fields have 1..3 components");
  pc_field* f = new pc_field();
  f->grid = g;
  f->ncomp = ncomp;
  for (int q = 0; q < 3; ++q) f->buf[q] = nullptr;
  // device buffers come from the context's caching pool (a public-API step
  // creates and drops fields and operators: no cudaMalloc/cudaFree churn)
  for (int q = 0; q < ncomp; ++q) {
    f->buf[q] = pool_get(g->ctx, g->comp_elems);
    if (!f->buf[q]) {
      for (int r = 0; r < q; ++r) pool_put(g->ctx, g->comp_elems, f->buf[r]);
      delete f;
      return fail(PC_E_CUDA, "field allocation failed (out of device memory)");
    }
    cudaMemsetAsync(f->buf[q], 0, g->comp_elems * sizeof(double), g->ctx->s);
  }
  live_add(f);
  *out = f;
  return PC_OK;
}

int pc_field_destroy(pc_field* f) {
  if (!f) return PC_OK;
  live_del(f);
  if (f->copied) cudaEventSynchronize(f->ready);  // the host side of an in-flight copy may go away next
  f->pending = false;
  if (f->ready) cudaEventDestroy(f->ready);
  for (int q = 0; q < f->ncomp; ++q) pool_put(f->grid->ctx, f->grid->comp_elems, f->buf[q]);
  delete f;
  return PC_OK;
}

// staging buffer of a stream (grow-only; the stream is drained before a regrow)
static int ensure_staging_on(cudaStream_t st, double*& buf, size_t& have, size_t bytes) {
  if (have >= bytes) return PC_OK;
  cudaStreamSynchronize(st);
  cudaFree(buf);
  buf = nullptr;
  have = 0;
  CUDA_TRY(cudaMalloc(&buf, bytes));
  have = bytes;
  return PC_OK;
}
static int ensure_staging(pc_ctx* c, size_t bytes) {
  return ensure_staging_on(c->s, c->staging, c->staging_bytes, bytes);
}

// host -> field on stream st (AoS components go through st's staging buffer
// in 256 MB plane chunks and are transposed on the device)
// host plane of a field: n1 x the owned columns (phi-slabs: without the ghost columns)
static size_t host_plane(const pc_grid* g) { return (size_t)g->g.n1 * (size_t)(g->g.n2 - 2 * g->g.phis); }
static int upload_on(pc_field* f, const double* host, int layout, cudaStream_t st, double*& stg, size_t& stg_bytes) {
  pc_grid* g = f->grid;
  pc_ctx* c = g->ctx;
  const size_t pl = (size_t)g->g.plane, n0 = (size_t)g->g.n0;
  if (g->g.phis) {  // owned columns only: strided rows (SoA) or the chunked transposition (AoS)
    const size_t hn2 = (size_t)g->g.n2 - 2, hpl = host_plane(g);
    if (layout == PC_LAYOUT_SOA || f->ncomp == 1) {
      for (int q = 0; q < f->ncomp; ++q)
        CUDA_TRY(cudaMemcpy2DAsync(f->base(q) + 1, (size_t)g->g.n2 * sizeof(double), host + (size_t)q * n0 * hpl,
                                   hn2 * sizeof(double), hn2 * sizeof(double), n0 * (size_t)g->g.n1,
                                   cudaMemcpyHostToDevice, st));
      return PC_OK;
    }
    const size_t chunk_planes = std::max<size_t>(1, std::min<size_t>(n0, (256u << 20) / (hpl * f->ncomp * 8)));
    TRY(ensure_staging_on(st, stg, stg_bytes, chunk_planes * hpl * f->ncomp * sizeof(double)));
    for (size_t p0 = 0; p0 < n0; p0 += chunk_planes) {
      size_t np = std::min(chunk_planes, n0 - p0);
      CUDA_TRY(cudaMemcpyAsync(stg, host + p0 * hpl * f->ncomp, np * hpl * f->ncomp * sizeof(double),
                               cudaMemcpyHostToDevice, st));
      k_aos_to_soa<<<grid_blocks(c, (int64_t)(np * hpl)), kThreads, 0, st>>>(g->g, f->ncomp, stg, fld(f), (int)p0,
                                                                              (int)np);
      c->st.launches++;
      TRY(check_launch("k_aos_to_soa"));
    }
    return PC_OK;
  }
  if (layout == PC_LAYOUT_SOA || f->ncomp == 1) {
    for (int q = 0; q < f->ncomp; ++q)
      CUDA_TRY(cudaMemcpyAsync(f->base(q), host + (size_t)q * n0 * pl, n0 * pl * sizeof(double),
                               cudaMemcpyHostToDevice, st));
  } else {
    const size_t chunk_planes = std::max<size_t>(1, std::min<size_t>(n0, (256u << 20) / (pl * f->ncomp * 8)));
    TRY(ensure_staging_on(st, stg, stg_bytes, chunk_planes * pl * f->ncomp * sizeof(double)));
    for (size_t p0 = 0; p0 < n0; p0 += chunk_planes) {
      size_t np = std::min(chunk_planes, n0 - p0);
      CUDA_TRY(cudaMemcpyAsync(stg, host + p0 * pl * f->ncomp, np * pl * f->ncomp * sizeof(double),
                               cudaMemcpyHostToDevice, st));
      k_aos_to_soa<<<grid_blocks(c, (int64_t)(np * pl)), kThreads, 0, st>>>(g->g, f->ncomp, stg, fld(f), (int)p0,
                                                                             (int)np);
      c->st.launches++;
      TRY(check_launch("k_aos_to_soa"));
    }
  }
  return PC_OK;
}
static int download_on(const pc_field* f, double* host, int layout, cudaStream_t st, double*& stg,
                       size_t& stg_bytes) {
  pc_grid* g = f->grid;
  pc_ctx* c = g->ctx;
  const size_t pl = (size_t)g->g.plane, n0 = (size_t)g->g.n0;
  if (g->g.phis) {
    const size_t hn2 = (size_t)g->g.n2 - 2, hpl = host_plane(g);
    if (layout == PC_LAYOUT_SOA || f->ncomp == 1) {
      for (int q = 0; q < f->ncomp; ++q)
        CUDA_TRY(cudaMemcpy2DAsync(host + (size_t)q * n0 * hpl, hn2 * sizeof(double), f->base(q) + 1,
                                   (size_t)g->g.n2 * sizeof(double), hn2 * sizeof(double), n0 * (size_t)g->g.n1,
                                   cudaMemcpyDeviceToHost, st));
      return PC_OK;
    }
    const size_t chunk_planes = std::max<size_t>(1, std::min<size_t>(n0, (256u << 20) / (hpl * f->ncomp * 8)));
    TRY(ensure_staging_on(st, stg, stg_bytes, chunk_planes * hpl * f->ncomp * sizeof(double)));
    for (size_t p0 = 0; p0 < n0; p0 += chunk_planes) {
      size_t np = std::min(chunk_planes, n0 - p0);
      k_soa_to_aos<<<grid_blocks(c, (int64_t)(np * hpl)), kThreads, 0, st>>>(g->g, f->ncomp, cfld(f), stg, (int)p0,
                                                                              (int)np);
      c->st.launches++;
      TRY(check_launch("k_soa_to_aos"));
      CUDA_TRY(cudaMemcpyAsync(host + p0 * hpl * f->ncomp, stg, np * hpl * f->ncomp * sizeof(double),
                               cudaMemcpyDeviceToHost, st));
    }
    return PC_OK;
  }
  if (layout == PC_LAYOUT_SOA || f->ncomp == 1) {
    for (int q = 0; q < f->ncomp; ++q)
      CUDA_TRY(cudaMemcpyAsync(host + (size_t)q * n0 * pl, f->base(q), n0 * pl * sizeof(double),
                               cudaMemcpyDeviceToHost, st));
  } else {
    const size_t chunk_planes = std::max<size_t>(1, std::min<size_t>(n0, (256u << 20) / (pl * f->ncomp * 8)));
    TRY(ensure_staging_on(st, stg, stg_bytes, chunk_planes * pl * f->ncomp * sizeof(double)));
    for (size_t p0 = 0; p0 < n0; p0 += chunk_planes) {
      size_t np = std::min(chunk_planes, n0 - p0);
      k_soa_to_aos<<<grid_blocks(c, (int64_t)(np * pl)), kThreads, 0, st>>>(g->g, f->ncomp, cfld(f), stg, (int)p0,
                                                                             (int)np);
      c->st.launches++;
      TRY(check_launch("k_soa_to_aos"));
      CUDA_TRY(cudaMemcpyAsync(host + p0 * pl * f->ncomp, stg, np * pl * f->ncomp * sizeof(double),
                               cudaMemcpyDeviceToHost, st));
    }
  }
  return PC_OK;
}

int pc_field_upload(pc_field* f, const double* host, int layout) {
  if (!f || !host) return fail(PC_E_INVALID, "null argument");
  pc_ctx* c = f->grid->ctx;
  field_dep(f);
  TRY(upload_on(f, host, layout, c->s, c->staging, c->staging_bytes));
  CUDA_TRY(cudaStreamSynchronize(c->s));
  return PC_OK;
}

int pc_field_download(const pc_field* f, double* host, int layout) {
  if (!f || !host) return fail(PC_E_INVALID, "null argument");
  pc_ctx* c = f->grid->ctx;
  field_dep(f);
  TRY(download_on(f, host, layout, c->s, c->staging, c->staging_bytes));
  CUDA_TRY(cudaStreamSynchronize(c->s));
  return PC_OK;
}

// ---- asynchronous copies on the copy stream: they start after the work
// already queued on the compute stream and the compute stream waits for them
// only where the field is next used, so a field needed later (the next
// operator's state) moves while the current operator computes
static int copy_stream_begin(pc_ctx* c, pc_field* f) {
  if (!c->cs) CUDA_TRY(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
  if (!f->ready) CUDA_TRY(cudaEventCreateWithFlags(&f->ready, cudaEventDisableTiming));
  field_dep(f);  // an earlier copy of this field completes first (stream order on s)
  CUDA_TRY(cudaEventRecord(c->ev_in, c->s));
  CUDA_TRY(cudaStreamWaitEvent(c->cs, c->ev_in, 0));
  return PC_OK;
}
int pc_field_upload_async(pc_field* f, const double* host, int layout) {
  if (!f || !host) return fail(PC_E_INVALID, "null argument");
  pc_ctx* c = f->grid->ctx;
  TRY(copy_stream_begin(c, f));
  TRY(upload_on(f, host, layout, c->cs, c->staging_cs, c->staging_cs_bytes));
  CUDA_TRY(cudaEventRecord(f->ready, c->cs));
  f->pending = true;
  f->copied = true;
  return PC_OK;
}
int pc_field_download_async(pc_field* f, double* host, int layout) {
  if (!f || !host) return fail(PC_E_INVALID, "null argument");
  pc_ctx* c = f->grid->ctx;
  TRY(copy_stream_begin(c, f));
  TRY(download_on(f, host, layout, c->cs, c->staging_cs, c->staging_cs_bytes));
  CUDA_TRY(cudaEventRecord(f->ready, c->cs));
  f->pending = true;
  f->copied = true;
  return PC_OK;
}
int pc_field_wait(pc_field* f) {
  if (!f) return fail(PC_E_INVALID, "null argument");
  // the host waits for the copy itself, even if a device-side dependency
  // (field_dep) has already been placed on the compute stream
  if (f->copied) CUDA_TRY(cudaEventSynchronize(f->ready));
  f->pending = false;
  return PC_OK;
}

int pc_field_set_ghost(pc_field* f, int side, const double* host) {
  if (!f || !host || (side != 0 && side != 1)) return fail(PC_E_INVALID, "bad ghost-plane arguments");
  field_dep(f);
  pc_grid* g = f->grid;
  const size_t pl = (size_t)g->g.plane;
  const int64_t plane = side == 0 ? -1 : g->g.n0;
  for (int q = 0; q < f->ncomp; ++q)
    CUDA_TRY(cudaMemcpyAsync(f->base(q) + plane * (int64_t)pl, host + (size_t)q * pl, pl * sizeof(double),
                             cudaMemcpyHostToDevice, g->ctx->s));
  CUDA_TRY(cudaStreamSynchronize(g->ctx->s));
  return PC_OK;
}

int pc_field_set_ghost_cols(pc_field* f, const double* host) {
  if (!f || !host || !f->grid->g.phis) return fail(PC_E_INVALID, "ghost columns need a phi-slab field");
  field_dep(f);
  pc_grid* g = f->grid;
  pc_ctx* c = g->ctx;
  const size_t rows = (size_t)g->g.n0 * g->g.n1;
  TRY(ensure_staging(c, 2 * rows * f->ncomp * sizeof(double)));
  CUDA_TRY(cudaMemcpyAsync(c->staging, host, 2 * rows * f->ncomp * sizeof(double), cudaMemcpyHostToDevice, c->s));
  k_phi_unpack<<<grid_blocks(c, (int64_t)rows), kThreads, 0, c->s>>>(g->g, f->ncomp, c->staging, fld(f));
  c->st.launches++;
  TRY(check_launch("k_phi_unpack"));
  CUDA_TRY(cudaStreamSynchronize(c->s));
  return PC_OK;
}

int pc_field_download_planes(const pc_field* f, int64_t i0, int64_t n, double* host) {
  if (!f || !host) return fail(PC_E_INVALID, "null argument");
  field_dep(f);
  pc_grid* g = f->grid;
  if (i0 < 0 || n < 0 || i0 + n > g->g.n0) return fail(PC_E_INVALID, "plane window out of range");
  const size_t pl = (size_t)g->g.plane;
  for (int q = 0; q < f->ncomp; ++q)
    CUDA_TRY(cudaMemcpyAsync(host + (size_t)q * n * pl, f->base(q) + (size_t)i0 * pl, (size_t)n * pl * sizeof(double),
                             cudaMemcpyDeviceToHost, g->ctx->s));
  CUDA_TRY(cudaStreamSynchronize(g->ctx->s));
  return PC_OK;
}

int pc_field_copy(pc_field* dst, const pc_field* src) {
  if (!dst || !src || dst->ncomp != src->ncomp || dst->grid->comp_elems != src->grid->comp_elems)
    return fail(PC_E_INVALID, "field copy: shape mismatch");
  field_dep(dst);
  field_dep(src);
  for (int q = 0; q < dst->ncomp; ++q)
    CUDA_TRY(cudaMemcpyAsync(dst->buf[q], src->buf[q], dst->grid->comp_elems * sizeof(double),
                             cudaMemcpyDeviceToDevice, dst->grid->ctx->s));
  return PC_OK;
}

int pc_field_fill(pc_field* f, double v) {
  if (!f) return fail(PC_E_INVALID, "null field");
  field_dep(f);
  pc_ctx* c = f->grid->ctx;
  for (int q = 0; q < f->ncomp; ++q) {
    k_fill<<<grid_blocks(c, (int64_t)f->grid->comp_elems), kThreads, 0, c->s>>>(f->buf[q],
                                                                                 (int64_t)f->grid->comp_elems, v);
    c->st.launches++;
  }
  return check_launch("k_fill");
}

int pc_field_exchange_halo(pc_field* f) {
  if (!f) return fail(PC_E_INVALID, "null field");
  field_dep(f);
  return halo_field(f);
}

int pc_field_count(const pc_field* f, int test, int64_t* count) {
  if (!f || !count || test < 0 || test > 2) return fail(PC_E_INVALID, "bad pc_field_count arguments");
  field_dep(f);
  pc_grid* g = f->grid;
  pc_ctx* c = g->ctx;
  CUDA_TRY(cudaMemsetAsync(c->maxout, 0, sizeof(double), c->s));
  k_count_fail<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, cfld(f), f->ncomp, test, c->maxout);
  c->st.launches++;
  TRY(check_launch("k_count_fail"));
  TRY(allreduce_d(c, c->maxout, 1, nccl::kSum));
  CUDA_TRY(cudaMemcpyAsync(c->h_maxout, c->maxout, sizeof(double), cudaMemcpyDeviceToHost, c->s));
  CUDA_TRY(cudaStreamSynchronize(c->s));
  *count = (int64_t)*c->h_maxout;
  return PC_OK;
}

int pc_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(PC_E_INVALID, "null argument");
  CUDA_TRY(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault));
  return PC_OK;
}
int pc_host_free(void* p) {
  if (p) CUDA_TRY(cudaFreeHost(p));
  return PC_OK;
}

int pc_host_register(void* p, size_t bytes) {
  CUDA_TRY(cudaHostRegister(p, bytes, cudaHostRegisterDefault));
  return PC_OK;
}
int pc_host_unregister(void* p) {
  CUDA_TRY(cudaHostUnregister(p));
  return PC_OK;
}
