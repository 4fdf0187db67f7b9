// paracycle_b200 C ABI, part of the single translation unit capi.cu (included
// there in order; relies on the declarations of the parts before it).
//
// error state, the opaque C-ABI objects (pc_ctx, pc_grid, pc_field, pc_op), the
// device memory pool, workspaces and the NCCL collectives used by every section
#pragma once

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
static thread_local int64_t g_info = 0;

static int fail(int code, const std::string& msg, int64_t info = 0) {
  g_err = msg;
  g_info = info;
  return code;
}
#define CUDA_TRY(x)                                                                       \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      return fail(PC_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));            \
  } while (0)
#define TRY(x)                 \
  do {                         \
    int r_ = (x);              \
    if (r_ != PC_OK) return r_; \
  } while (0)

// ------------------------------------------------------------------ objects
// kinds of timed hot loops: 0 scalar/vector STS stages, 1 aligned STS stages,
// 2 scalar PCG iterations, 3 aligned PCG iterations
// timed hot loops (pc_ctx_stats_kind): STS stages k >= 2, PCG iterations, and
// the fused stage-1+2 launch of the 7-point march without (F12, s == 2) and
// with (F12W, s >= 3) the u1 write; F12 units count both stages
enum {
  KIND_STS_SCALAR = 0,
  KIND_STS_ALIGNED = 1,
  KIND_PCG_SCALAR = 2,
  KIND_PCG_ALIGNED = 3,
  KIND_STS_F12 = 4,
  KIND_STS_F12W = 5,
  KIND_STS_AF12 = 6,   // the aligned (TMA march) fused stage-1+2 launch, s == 2
  KIND_STS_AF12W = 7,  // ... with the u1 write (s >= 3)
  NKIND = 8
};
struct Stats {
  double stage_ms = 0.0;
  int64_t stage_launches = 0;
  int64_t launches = 0;
  double kind_ms[NKIND] = {};
  int64_t kind_launches[NKIND] = {};
  int64_t kind_units[NKIND] = {};  // cell-updates (local cells x stages / iterations)
};
struct TimedSpan {
  cudaEvent_t e0, e1;
  int kind;
};

struct pc_ctx {
  int device = 0;
  int nranks = 1, rank = 0;
  cudaStream_t s = nullptr;
  ncclComm_t comm = nullptr;
  bool detached = false;  // test hook: a slab rank without a communicator (ghost planes set by the caller)
  cudaStream_t sc = nullptr;            // communication stream (halo exchange overlapped with interior chunks)
  cudaEvent_t ev_in = nullptr, ev_halo = nullptr;
  int zpart = 0;                        // r-chunk partition of the next marching launch: 0 all, 1 interior, 2 boundary
  int max_blocks = 148 * 16;
  int sms = 148;
  int max_red = 1 << 18;  // partial-sum slots (march grids are larger)
  // reduction scratch
  double* red_v = nullptr;
  double* red_v2 = nullptr;
  long long* red_i = nullptr;
  unsigned int* counter = nullptr;
  ArgRes* res = nullptr;
  PcgDev* pcg = nullptr;
  int* bad = nullptr;
  unsigned long long* minbits = nullptr;
  double* maxout = nullptr;
  double* gath = nullptr;  // per-rank (|F| max, index) pairs
  // GPU-count-invariant PCG reductions (kernels.cuh PlaneRed): slot partials
  // of up to two sums, the per-plane vector [2][n0g] (entries of other
  // ranks' planes stay 0) and its allreduced copy
  double* pslot[2] = {nullptr, nullptr};
  size_t pslot_cap = 0;
  double* pvec = nullptr;
  double* pvec_all = nullptr;
  int axis = 0;                 // slab decomposition axis: 0 = r (planes), 2 = phi (columns, ghost columns)
  double* phibuf = nullptr;     // phi-slab exchange: packed send [ncomp][2][rows] + receive halves
  size_t phibuf_cap = 0;
  int pvec_n0g = 0, pvec_i0g = -1, pvec_n = 0;
  // pinned host mirrors
  ArgRes* h_res = nullptr;
  PcgDev* h_pcg = nullptr;
  int* h_bad = nullptr;
  bool bad_pending = false;  // pc_cycle: the last STS step's non-finite flag is in flight to h_bad
  CycleDev* cyc_dev = nullptr;      // persistent small-grid cycle state (allocated on first use)
  pc_cycle_record* cyc_rec = nullptr;  // its device cycle records (grow-only)
  int64_t cyc_rec_cap = 0;
  CycleDev* h_cyc = nullptr;
  unsigned long long* h_minbits = nullptr;
  double* h_maxout = nullptr;
  // staging for AoS conversion
  double* staging = nullptr;
  size_t staging_bytes = 0;
  // copy stream of the asynchronous uploads / downloads, and its staging
  cudaStream_t cs = nullptr;
  double* staging_cs = nullptr;
  size_t staging_cs_bytes = 0;
  // workspace pool of single-component buffers
  std::vector<std::pair<size_t, double*>> pool;
  Stats st;
  bool timing = false;
  std::vector<TimedSpan> ev;
  std::vector<cudaEvent_t> ev_free;  // recycled timing events (no cudaEventCreate per timed span)
  cudaEvent_t marks[16] = {};
};

struct pc_grid {
  pc_ctx* ctx;
  GridDev g;
  double* tables = nullptr;
  double* rowrec = nullptr;  // [n0+2][n1][RW] interleaved row records (TMA march)
  CUtensorMap rowmap;
  bool rowmap_ok = false;
  double* srowrec = nullptr;  // [n0+2][n1][4] W2[0..2], iV2 records (vector march), built on first use
  CUtensorMap srowmap;
  bool srow_ok = false;
  // TMA maps of field buffers by (base, box): the pooled buffers recur, so a
  // stage launch re-encodes nothing after the first cycle
  struct MapEntry {
    const double* base;
    unsigned b0, b1;
    CUtensorMap m;
  };
  std::vector<MapEntry> mapcache;
  int64_t shape[3];
  size_t comp_elems;  // (n0 + 2) * plane
};

struct pc_field {
  pc_grid* grid;
  int ncomp;
  double* buf[3];  // allocation base (ghost plane -1)
  double* base(int q) const { return buf[q] + grid->g.plane; }
  // an asynchronous upload / download on the context's copy stream is in
  // flight until `ready`; the compute stream waits for it before the field's
  // next use (field_dep)
  cudaEvent_t ready = nullptr;
  mutable bool pending = false;  // the compute stream has not yet been made to wait for `ready`
  bool copied = false;           // `ready` was recorded (host-side waits synchronise on it)
};

enum { K_SCALAR = 0, K_ALIGNED = 1 };

struct pc_op {
  pc_grid* grid;
  int kind;
  int ncomp;
  ScalarOp so{};
  AlignedOp ao{};
  const double* bsrc[3] = {nullptr, nullptr, nullptr};  // aligned: b-hat (caller's field)
  double* betabuf = nullptr;  // aligned: beta = sqrt(c) b, 3 component-sized buffers
  double* dbuf = nullptr;   // Jacobi diagonal -J_ii (allocated on first BE / diagonal use)
  bool diag_valid = false;
  double* kfc = nullptr;    // kappa0 * f_c(r) per axis-0 row (n0 + 2)
  double Tfloor = 1e-10;
  bool beta_maps = false;   // cached TMA maps of beta (the buffer never moves)
  CUtensorMap bmap[3], bsmap[3];
  double lam_max = 0.0;
  double dt_euler = INFINITY;
  bool frozen = false;
  int pc = PC_PC_JACOBI;    // BE+PCG preconditioner
  double* lbuf = nullptr;   // r-line preconditioner: -J_{i,i-1}, -J_{i,i+1} (2 component-sized buffers)
  double* rho_r = nullptr;  // aligned: rho(i) per interior plane when the density field is radial
  bool line_valid = false;
  // the caller's coefficient fields the kernels read in place (D, rho, b-hat):
  // every launching entry point waits for their in-flight asynchronous
  // uploads (op_deps), not only the constructor
  const pc_field* deps[3] = {nullptr, nullptr, nullptr};
  // aligned: re-freeze T0 := u at the start of every cycle of pc_cycle
  // ("per-cycle refresh available via config"; default: once per
  // outer step, by the caller)
  bool refresh_cycle = false;
};

// ------------------------------------------------------------------ helpers
// a timing event from the context's free list (created on first use)
static cudaEvent_t ev_new(pc_ctx* c) {
  if (!c->ev_free.empty()) {
    cudaEvent_t e = c->ev_free.back();
    c->ev_free.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
static int grid_blocks(pc_ctx* c, int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  if (b < 1) b = 1;
  return (int)std::min<int64_t>(b, c->max_blocks);
}

// blocks for the row-iterating node kernels (PC_FOR_NODES: one warp per row)
static int node_blocks(pc_ctx* c, const GridDev& g) {
  int64_t rows = (int64_t)g.n0 * g.n1;
  int64_t b = (rows + kThreads / 32 - 1) / (kThreads / 32);
  if (b < 1) b = 1;
  return (int)std::min<int64_t>(b, c->max_blocks);
}

// PC_POISON (test switch, the initcheck substitute: compute-sanitizer is
// not available on the GPU pool): every buffer the pool hands out is filled
// with NaN bytes, so a kernel that reads workspace it did not write poisons
// its result and the parity checks fail (fields are still created zeroed)
static bool pool_poison() {
  static const bool on = getenv("PC_POISON") != nullptr;
  return on;
}
static double* pool_get(pc_ctx* c, size_t elems) {
  for (size_t q = 0; q < c->pool.size(); ++q) {
    if (c->pool[q].first == elems) {
      double* p = c->pool[q].second;
      c->pool.erase(c->pool.begin() + q);
      if (pool_poison()) cudaMemsetAsync(p, 0xFF, elems * sizeof(double), c->s);
      return p;
    }
  }
  double* p = nullptr;
  if (cudaMalloc(&p, elems * sizeof(double)) != cudaSuccess) {
    // out of memory: return every cached block to the driver and retry once
    cudaGetLastError();
    cudaStreamSynchronize(c->s);
    for (auto& e : c->pool) cudaFree(e.second);
    c->pool.clear();
    if (cudaMalloc(&p, elems * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
  }
  cudaMemsetAsync(p, pool_poison() ? 0xFF : 0, elems * sizeof(double), c->s);
  return p;
}
static void pool_put(pc_ctx* c, size_t elems, double* p) {
  if (p) c->pool.push_back({elems, p});
}

static CFld cfld(const pc_field* f) {
  CFld r{{nullptr, nullptr, nullptr}};
  for (int q = 0; q < f->ncomp; ++q) r.p[q] = f->base(q);
  for (int q = f->ncomp; q < 3; ++q) r.p[q] = r.p[0];
  return r;
}
static Fld fld(pc_field* f) {
  Fld r{{nullptr, nullptr, nullptr}};
  for (int q = 0; q < f->ncomp; ++q) r.p[q] = f->base(q);
  for (int q = f->ncomp; q < 3; ++q) r.p[q] = r.p[0];
  return r;
}
// a set of ncomp pool buffers viewed as a field
struct Work {
  pc_ctx* c;
  size_t elems;
  int ncomp;
  int64_t plane;
  double* b[3] = {nullptr, nullptr, nullptr};
  double* base(int q) const { return b[q] + plane; }
  CFld cf() const {
    CFld r{{base(0), ncomp > 1 ? base(1) : base(0), ncomp > 2 ? base(2) : base(0)}};
    return r;
  }
  Fld f() const {
    Fld r{{base(0), ncomp > 1 ? base(1) : base(0), ncomp > 2 ? base(2) : base(0)}};
    return r;
  }
};
static int work_get(pc_grid* g, int ncomp, Work& w) {
  w.c = g->ctx;
  w.elems = g->comp_elems;
  w.ncomp = ncomp;
  w.plane = g->g.plane;
  for (int q = 0; q < ncomp; ++q) {
    w.b[q] = pool_get(g->ctx, w.elems);
    if (!w.b[q]) return fail(PC_E_CUDA, "workspace allocation failed (out of device memory?)");
  }
  return PC_OK;
}
static void work_put(Work& w) {
  for (int q = 0; q < w.ncomp; ++q) {
    pool_put(w.c, w.elems, w.b[q]);
    w.b[q] = nullptr;
  }
}
// swap the storage of a field with a work set (pointer rotation, no copy)
static void swap_storage(pc_field* f, Work& w) {
  for (int q = 0; q < f->ncomp; ++q) std::swap(f->buf[q], w.b[q]);
}

// live fields: an operator keeps pointers to its coefficient fields, which
// the caller may destroy first; op_deps only touches fields still alive
static std::mutex g_live_mu;
static std::unordered_set<const pc_field*> g_live;
static void live_add(const pc_field* f) {
  std::lock_guard<std::mutex> l(g_live_mu);
  g_live.insert(f);
}
static void live_del(const pc_field* f) {
  std::lock_guard<std::mutex> l(g_live_mu);
  g_live.erase(f);
}

// the compute stream waits for a field's in-flight asynchronous copy
static void field_dep(const pc_field* f) {
  if (f && f->pending) {
    cudaStreamWaitEvent(f->grid->ctx->s, f->ready, 0);
    f->pending = false;
  }
}
// ... and for every coefficient field an operator reads in place
static void op_deps(const pc_op* op) {
  if (!op) return;
  std::lock_guard<std::mutex> l(g_live_mu);
  for (const pc_field* f : op->deps)
    if (f && g_live.count(f)) field_dep(f);
}

static int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return PC_OK;
}

// ------------------------------------------------------------------ NCCL
static int phi_exchange(pc_ctx* c, pc_grid* g, double* const* bufs, int ncomp, cudaStream_t st);
static int halo_exchange(pc_ctx* c, pc_grid* g, double* const* bufs, int ncomp, cudaStream_t st = nullptr) {
  if (!c->comm) return PC_OK;  // one rank, or a detached test rank (ghosts set by the caller)
  if (!st) st = c->s;
  if (g->g.phis) return phi_exchange(c, g, bufs, ncomp, st);
  nccl::Api* A = nccl::api();
  if (!A) return fail(PC_E_NCCL, "NCCL not available");
  const size_t pl = (size_t)g->g.plane;
  const int n0 = g->g.n0;
  int lo = g->g.ghost_lo0 ? (c->rank - 1 + c->nranks) % c->nranks : -1;
  int hi = g->g.ghost_hi0 ? (c->rank + 1) % c->nranks : -1;
  if (A->groupStart() != 0) return fail(PC_E_NCCL, "ncclGroupStart");
  // NCCL matches the p2p operations of a rank pair in issue order, so every
  // rank issues (send last plane up, receive lower ghost) before (send first
  // plane down, receive upper ghost): the pairing stays right when the lower
  // and upper neighbour are the same rank (a periodic ring of 1 or 2 slabs)
  for (int q = 0; q < ncomp; ++q) {
    double* base = bufs[q] + pl;  // interior plane 0
    if (hi >= 0) A->send(base + (size_t)(n0 - 1) * pl, pl, nccl::kDouble, hi, c->comm, st);
    if (lo >= 0) A->recv(base - pl, pl, nccl::kDouble, lo, c->comm, st);
    if (lo >= 0) A->send(base, pl, nccl::kDouble, lo, c->comm, st);
    if (hi >= 0) A->recv(base + (size_t)n0 * pl, pl, nccl::kDouble, hi, c->comm, st);
  }
  if (A->groupEnd() != 0) return fail(PC_E_NCCL, "ncclGroupEnd");
  return PC_OK;
}
// phi-slabs: the owned edge columns of every (plane, row) packed, swapped
// with the ring neighbours (rank - 1, rank + 1 mod P; the same pairing order
// as the planes, so a one- or two-rank ring pairs right) and unpacked into
// the ghost columns
static int phi_exchange(pc_ctx* c, pc_grid* g, double* const* bufs, int ncomp, cudaStream_t st) {
  nccl::Api* A = nccl::api();
  if (!A) return fail(PC_E_NCCL, "NCCL not available");
  const size_t rows = (size_t)g->g.n0 * g->g.n1;
  const size_t need = 4 * rows * (size_t)ncomp;
  if (need > c->phibuf_cap) {
    cudaStreamSynchronize(st);
    cudaFree(c->phibuf);
    c->phibuf = nullptr;
    c->phibuf_cap = 0;
    CUDA_TRY(cudaMalloc(&c->phibuf, need * sizeof(double)));
    c->phibuf_cap = need;
  }
  double* snd = c->phibuf;
  double* rcv = c->phibuf + 2 * rows * (size_t)ncomp;
  CFld src{{bufs[0] + g->g.plane, ncomp > 1 ? bufs[1] + g->g.plane : nullptr, ncomp > 2 ? bufs[2] + g->g.plane : nullptr}};
  Fld dst{{bufs[0] + g->g.plane, ncomp > 1 ? bufs[1] + g->g.plane : nullptr, ncomp > 2 ? bufs[2] + g->g.plane : nullptr}};
  k_phi_pack<<<grid_blocks(c, (int64_t)rows), kThreads, 0, st>>>(g->g, ncomp, src, snd);
  c->st.launches++;
  TRY(check_launch("k_phi_pack"));
  const int lo = (c->rank - 1 + c->nranks) % c->nranks, hi = (c->rank + 1) % c->nranks;
  if (A->groupStart() != 0) return fail(PC_E_NCCL, "ncclGroupStart");
  for (int q = 0; q < ncomp; ++q) {
    double* s_lo = snd + (2 * q) * rows;      // column 1 -> lower neighbour (its upper ghost)
    double* s_hi = snd + (2 * q + 1) * rows;  // column n2-2 -> upper neighbour (its lower ghost)
    double* r_lo = rcv + (2 * q) * rows;      // lower ghost <- lower neighbour's column n2-2
    double* r_hi = rcv + (2 * q + 1) * rows;  // upper ghost <- upper neighbour's column 1
    A->send(s_hi, rows, nccl::kDouble, hi, c->comm, st);
    A->recv(r_lo, rows, nccl::kDouble, lo, c->comm, st);
    A->send(s_lo, rows, nccl::kDouble, lo, c->comm, st);
    A->recv(r_hi, rows, nccl::kDouble, hi, c->comm, st);
  }
  if (A->groupEnd() != 0) return fail(PC_E_NCCL, "ncclGroupEnd");
  k_phi_unpack<<<grid_blocks(c, (int64_t)rows), kThreads, 0, st>>>(g->g, ncomp, rcv, dst);
  c->st.launches++;
  return check_launch("k_phi_unpack");
}
static int halo_field(pc_field* f) {
  double* b[3] = {f->buf[0], f->buf[1], f->buf[2]};
  return halo_exchange(f->grid->ctx, f->grid, b, f->ncomp);
}
static int halo_work(pc_grid* g, Work& w) {
  double* b[3] = {w.b[0], w.b[1], w.b[2]};
  return halo_exchange(g->ctx, g, b, w.ncomp);
}
static int allreduce_u64_min(pc_ctx* c, unsigned long long* dptr) {
  if (!c->comm) return PC_OK;
  nccl::Api* A = nccl::api();
  if (!A || A->allReduce(dptr, dptr, 1, nccl::kUint64, nccl::kMin, c->comm, c->s) != 0)
    return fail(PC_E_NCCL, "ncclAllReduce(u64 min)");
  return PC_OK;
}
// the |F| argmax over all ranks (res holds this rank's pair on entry)
static int global_argmax(pc_ctx* c) {
  if (!c->comm) return PC_OK;
  nccl::Api* A = nccl::api();
  if (!A || !A->allGather_ || A->allGather(c->res, c->gath, 2, nccl::kDouble, c->comm, c->s) != 0)
    return fail(PC_E_NCCL, "ncclAllGather(argmax)");
  k_argmax_combine<<<1, 32, 0, c->s>>>(c->gath, c->nranks, c->res);
  c->st.launches++;
  return check_launch("k_argmax_combine");
}
static int allreduce_d(pc_ctx* c, double* dptr, size_t n, int op) {
  if (!c->comm) return PC_OK;
  nccl::Api* A = nccl::api();
  if (!A || A->allReduce(dptr, dptr, n, nccl::kDouble, op, c->comm, c->s) != 0)
    return fail(PC_E_NCCL, "ncclAllReduce");
  return PC_OK;
}
static int allreduce_d2(pc_ctx* c, const double* src, double* dst, size_t n, int op) {
  nccl::Api* A = nccl::api();
  if (!c->comm || !A || A->allReduce(src, dst, n, nccl::kDouble, op, c->comm, c->s) != 0)
    return fail(PC_E_NCCL, "ncclAllReduce");
  return PC_OK;
}
