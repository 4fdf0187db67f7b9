// paracycle_b200 C ABI implementation (see include/paracycle_b200.h).
//
// Host-side orchestration of the PTL-cycled parabolic advance:
//   pc_cycle  == ptl.cycle_operator: one F+argmax pass, the
//   Eq. 5 pair kernel, ONE 64-byte device->host read per cycle, then either
//   s fused STS stage kernels (RKL2/RKG2) or a device-driven Jacobi-PCG solve.
// Integer decisions (s, coefficient tables, remaining-time bookkeeping) are
// computed here with the same expressions as oracle/schemes.py and
// oracle/ptl.py (host code compiled with -ffp-contract=off).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/paracycle_b200.h"
#include "gen.cuh"
#include "march.cuh"
#include "smarch.cuh"
#include "tma_march.cuh"
#include "sts.cuh"
#include "persist.cuh"

#include <cudaTypedefs.h>
#include "nccl_shim.h"

using namespace pc;

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
enum { KIND_STS_SCALAR = 0, KIND_STS_ALIGNED = 1, KIND_PCG_SCALAR = 2, KIND_PCG_ALIGNED = 3, NKIND = 4 };
struct Stats {
  double stage_ms = 0.0;
  int64_t stage_launches = 0;
  int64_t launches = 0;
  double kind_ms[NKIND] = {0, 0, 0, 0};
  int64_t kind_launches[NKIND] = {0, 0, 0, 0};
  int64_t kind_units[NKIND] = {0, 0, 0, 0};  // cell-updates (local cells x stages / iterations)
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
  // pinned host mirrors
  ArgRes* h_res = nullptr;
  PcgDev* h_pcg = nullptr;
  int* h_bad = nullptr;
  bool bad_pending = false;  // pc_cycle: the last STS step's non-finite flag is in flight to h_bad
  CycleDev* cyc_dev = nullptr;      // persistent small-grid cycle state (allocated on first use)
  CycleDev* h_cyc = nullptr;
  unsigned long long* h_minbits = nullptr;
  double* h_maxout = nullptr;
  // staging for AoS conversion
  double* staging = nullptr;
  size_t staging_bytes = 0;
  // workspace pool of single-component buffers
  std::vector<std::pair<size_t, double*>> pool;
  Stats st;
  bool timing = false;
  std::vector<TimedSpan> ev;
  cudaEvent_t marks[16] = {};
};

struct pc_grid {
  pc_ctx* ctx;
  GridDev g;
  double* tables = nullptr;
  double* rowrec = nullptr;  // [n0+2][n1][RW] interleaved row records (TMA march)
  CUtensorMap rowmap;
  bool rowmap_ok = false;
  int64_t shape[3];
  size_t comp_elems;  // (n0 + 2) * plane
};

struct pc_field {
  pc_grid* grid;
  int ncomp;
  double* buf[3];  // allocation base (ghost plane -1)
  double* base(int q) const { return buf[q] + grid->g.plane; }
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
};

// ------------------------------------------------------------------ helpers
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

static double* pool_get(pc_ctx* c, size_t elems) {
  for (size_t q = 0; q < c->pool.size(); ++q) {
    if (c->pool[q].first == elems) {
      double* p = c->pool[q].second;
      c->pool.erase(c->pool.begin() + q);
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
  cudaMemsetAsync(p, 0, elems * sizeof(double), c->s);
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

static int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return PC_OK;
}

// ------------------------------------------------------------------ NCCL
static int halo_exchange(pc_ctx* c, pc_grid* g, double* const* bufs, int ncomp, cudaStream_t st = nullptr) {
  if (!c->comm) return PC_OK;  // one rank, or a detached test rank (ghosts set by the caller)
  if (!st) st = c->s;
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

int pc_ctx_destroy(pc_ctx* c) {
  if (c) {
    if (c->sc) cudaStreamDestroy(c->sc);
    if (c->cyc_dev) cudaFree(c->cyc_dev);
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
  if (c->comm) {
    nccl::Api* A = nccl::api();
    if (A) A->commDestroy(c->comm);
  }
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
    cudaEventDestroy(e.e0);
    cudaEventDestroy(e.e1);
  }
  c->ev.clear();
}
int pc_ctx_stats_kind(pc_ctx* c, int kind, double* ms, int64_t* launches, int64_t* units) {
  if (!c || kind < 0 || kind >= NKIND) return fail(PC_E_INVALID, "stats kind 0..3");
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
  *out = f;
  return PC_OK;
}

int pc_field_destroy(pc_field* f) {
  if (!f) return PC_OK;
  for (int q = 0; q < f->ncomp; ++q) pool_put(f->grid->ctx, f->grid->comp_elems, f->buf[q]);
  delete f;
  return PC_OK;
}

static int ensure_staging(pc_ctx* c, size_t bytes) {
  if (c->staging_bytes >= bytes) return PC_OK;
  cudaStreamSynchronize(c->s);
  cudaFree(c->staging);
  c->staging = nullptr;
  CUDA_TRY(cudaMalloc(&c->staging, bytes));
  c->staging_bytes = bytes;
  return PC_OK;
}

int pc_field_upload(pc_field* f, const double* host, int layout) {
  if (!f || !host) return fail(PC_E_INVALID, "null argument");
  pc_grid* g = f->grid;
  pc_ctx* c = g->ctx;
  const size_t pl = (size_t)g->g.plane, n0 = (size_t)g->g.n0;
  if (layout == PC_LAYOUT_SOA || f->ncomp == 1) {
    for (int q = 0; q < f->ncomp; ++q)
      CUDA_TRY(cudaMemcpyAsync(f->base(q), host + (size_t)q * n0 * pl, n0 * pl * sizeof(double),
                               cudaMemcpyHostToDevice, c->s));
  } else {
    const size_t chunk_planes = std::max<size_t>(1, std::min<size_t>(n0, (256u << 20) / (pl * f->ncomp * 8)));
    TRY(ensure_staging(c, chunk_planes * pl * f->ncomp * sizeof(double)));
    for (size_t p0 = 0; p0 < n0; p0 += chunk_planes) {
      size_t np = std::min(chunk_planes, n0 - p0);
      CUDA_TRY(cudaMemcpyAsync(c->staging, host + p0 * pl * f->ncomp, np * pl * f->ncomp * sizeof(double),
                               cudaMemcpyHostToDevice, c->s));
      k_aos_to_soa<<<grid_blocks(c, (int64_t)(np * pl)), kThreads, 0, c->s>>>(g->g, f->ncomp, c->staging, fld(f),
                                                                               (int)p0, (int)np);
      c->st.launches++;
      TRY(check_launch("k_aos_to_soa"));
    }
  }
  CUDA_TRY(cudaStreamSynchronize(c->s));
  return PC_OK;
}

int pc_field_download(const pc_field* f, double* host, int layout) {
  if (!f || !host) return fail(PC_E_INVALID, "null argument");
  pc_grid* g = f->grid;
  pc_ctx* c = g->ctx;
  const size_t pl = (size_t)g->g.plane, n0 = (size_t)g->g.n0;
  if (layout == PC_LAYOUT_SOA || f->ncomp == 1) {
    for (int q = 0; q < f->ncomp; ++q)
      CUDA_TRY(cudaMemcpyAsync(host + (size_t)q * n0 * pl, f->base(q), n0 * pl * sizeof(double),
                               cudaMemcpyDeviceToHost, c->s));
  } else {
    const size_t chunk_planes = std::max<size_t>(1, std::min<size_t>(n0, (256u << 20) / (pl * f->ncomp * 8)));
    TRY(ensure_staging(c, chunk_planes * pl * f->ncomp * sizeof(double)));
    for (size_t p0 = 0; p0 < n0; p0 += chunk_planes) {
      size_t np = std::min(chunk_planes, n0 - p0);
      k_soa_to_aos<<<grid_blocks(c, (int64_t)(np * pl)), kThreads, 0, c->s>>>(g->g, f->ncomp, cfld(f), c->staging,
                                                                               (int)p0, (int)np);
      c->st.launches++;
      TRY(check_launch("k_soa_to_aos"));
      CUDA_TRY(cudaMemcpyAsync(host + p0 * pl * f->ncomp, c->staging, np * pl * f->ncomp * sizeof(double),
                               cudaMemcpyDeviceToHost, c->s));
    }
  }
  CUDA_TRY(cudaStreamSynchronize(c->s));
  return PC_OK;
}

int pc_field_set_ghost(pc_field* f, int side, const double* host) {
  if (!f || !host || (side != 0 && side != 1)) return fail(PC_E_INVALID, "bad ghost-plane arguments");
  pc_grid* g = f->grid;
  const size_t pl = (size_t)g->g.plane;
  const int64_t plane = side == 0 ? -1 : g->g.n0;
  for (int q = 0; q < f->ncomp; ++q)
    CUDA_TRY(cudaMemcpyAsync(f->base(q) + plane * (int64_t)pl, host + (size_t)q * pl, pl * sizeof(double),
                             cudaMemcpyHostToDevice, g->ctx->s));
  CUDA_TRY(cudaStreamSynchronize(g->ctx->s));
  return PC_OK;
}

int pc_field_download_planes(const pc_field* f, int64_t i0, int64_t n, double* host) {
  if (!f || !host) return fail(PC_E_INVALID, "null argument");
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
  for (int q = 0; q < dst->ncomp; ++q)
    CUDA_TRY(cudaMemcpyAsync(dst->buf[q], src->buf[q], dst->grid->comp_elems * sizeof(double),
                             cudaMemcpyDeviceToDevice, dst->grid->ctx->s));
  return PC_OK;
}

int pc_field_fill(pc_field* f, double v) {
  pc_ctx* c = f->grid->ctx;
  for (int q = 0; q < f->ncomp; ++q) {
    k_fill<<<grid_blocks(c, (int64_t)f->grid->comp_elems), kThreads, 0, c->s>>>(f->buf[q],
                                                                                 (int64_t)f->grid->comp_elems, v);
    c->st.launches++;
  }
  return check_launch("k_fill");
}

int pc_field_exchange_halo(pc_field* f) { return halo_field(f); }

int pc_field_count(const pc_field* f, int test, int64_t* count) {
  if (!f || !count || test < 0 || test > 2) return fail(PC_E_INVALID, "bad pc_field_count arguments");
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

// ------------------------------------------------------------------ operators
int pc_op_create_scalar(pc_grid* g, int ncomp, int vector_metric, double D_const, const pc_field* D,
                        const pc_field* rho, pc_op** out) {
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
  *out = op;
  return PC_OK;
}

int pc_op_create_viscous(pc_grid* g, int ncomp, int vector_metric, double nu, const pc_field* rho, pc_op** out) {
  if (!rho || rho->ncomp != 1) return fail(PC_E_INVALID, "viscous operator needs a scalar density field");
  if (!(nu >= 0.0)) return fail(PC_E_INVALID, "nu must be >= 0");
  TRY(pc_op_create_scalar(g, ncomp, vector_metric, nu, nullptr, rho, out));
  (*out)->so.drho = 1;
  return PC_OK;
}

int pc_op_create_aligned(pc_grid* g, const pc_field* bhat, const pc_field* rho, double pref, double kappa0,
                         const double* fc_table, double T_floor, pc_op** out) {
  if (!g || !out || !bhat || bhat->ncomp != 3) return fail(PC_E_INVALID, "aligned operator needs a 3-component b");
  if (rho && rho->ncomp != 1) return fail(PC_E_INVALID, "rho is a scalar field");
  pc_ctx* c = g->ctx;
  pc_op* op = new pc_op();
  op->grid = g;
  op->kind = K_ALIGNED;
  op->ncomp = 1;
  for (int q = 0; q < 3; ++q) op->bsrc[q] = bhat->base(q);
  op->ao.rho = rho ? rho->base(0) : nullptr;
  op->ao.pref = pref;
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
  if (!op->ao.rho || getenv("PC_NO_RADIAL_RHO")) return PC_OK;
  CUDA_TRY(cudaMemsetAsync(c->bad, 0, sizeof(int), c->s));
  k_radial_check<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, op->ao.rho, c->bad);
  c->st.launches++;
  TRY(check_launch("k_radial_check"));
  CUDA_TRY(cudaMemcpyAsync(c->h_bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->s));
  CUDA_TRY(cudaStreamSynchronize(c->s));
  if (*c->h_bad != 0) return PC_OK;  // not radial
  if (!op->rho_r) CUDA_TRY(cudaMalloc(&op->rho_r, sizeof(double) * (size_t)g->g.n0));
  CUDA_TRY(cudaMemcpy2DAsync(op->rho_r, sizeof(double), op->ao.rho, (size_t)g->g.plane * sizeof(double), sizeof(double),
                             (size_t)g->g.n0, cudaMemcpyDeviceToDevice, c->s));
  op->ao.rho_r = op->rho_r;
  return PC_OK;
}

int pc_op_freeze(pc_op* op, const pc_field* T0) {
  if (!op) return fail(PC_E_INVALID, "null operator");
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
  if (!op || !out || out->ncomp != 1) return fail(PC_E_INVALID, "diagonal output must be a scalar field");
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
static bool tma_ok(const pc_grid* g) {
  const GridDev& d = g->g;
  return d.per2 && d.n2 % MTK == 0 && !d.per1 && d.n2 >= 2 && tma_encoder() != nullptr &&
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
  k_aligned_tma<Epi, RHO><<<grid, dim3(MTK, MTY), smem, c->s>>>(g->g, op->ao, maps, epi, R, zsel, skip);
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
static int smarch_R(const pc_grid* g, int ncomp) {
  if (const char* e = getenv("PC_SMARCH_R")) {
    const int r = atoi(e);
    if (r >= 1) return r;
  }
  const int tiles = ((g->g.n2 + MTK - 1) / MTK) * ((g->g.n1 + SMJ - 1) / SMJ);
  const int64_t want = ncomp == 3 ? 148 * 6 : 148 * 12;
  int R = 32;
  while (R > 4 && (int64_t)tiles * ((g->g.n0 + R - 1) / R) < want) R /= 2;
  return R;
}
static bool smarch_ok(const pc_op* op) { return op->ncomp == 1 || op->ncomp == 3; }
template <int NC, bool VEC, int DM, class Epi>
static int launch_smarch_t(pc_op* op, CFld u, const Epi& epi, const int* skip, const char* what) {
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  const int R = smarch_R(g, NC);
  dim3 grid((g->g.n2 + MTK - 1) / MTK, (g->g.n1 + SMJ - 1) / SMJ, (g->g.n0 + R - 1) / R);
  if ((int64_t)grid.x * grid.y * grid.z > c->max_red) return fail(PC_E_INVALID, "grid too large for the reduction scratch");
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(k_scalar_march<NC, VEC, DM, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(SMarchSmem<NC>)));
    attr = true;
  }
  const int zsel = zsplit(c, grid);
  k_scalar_march<NC, VEC, DM, Epi><<<grid, SNT, sizeof(SMarchSmem<NC>), c->s>>>(g->g, op->so, u.p[0], u.p[1], u.p[2],
                                                                                epi, R, zsel, skip);
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
  if (!op || !u || !F || u->ncomp != op->ncomp || F->ncomp != op->ncomp) return fail(PC_E_INVALID, "shape mismatch");
  TRY(need_frozen(op));
  TRY(halo_field(const_cast<pc_field*>(u)));
  TRY(apply_any(op, cfld(u), fld(F), false));
  CUDA_TRY(cudaStreamSynchronize(op->grid->ctx->s));
  return PC_OK;
}

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
  CUDA_TRY(cudaMemsetAsync(c->bad, 0x7f, sizeof(int), c->s));
  k_stage1<<<nb, kThreads, 0, c->s>>>(g->g, nc, cfld(u), y0.cf(), A.f(), tab[3], c->bad);
  c->st.launches++;
  rc = check_launch("k_stage1");
  if (c->timing) {  // the fused stage kernels k >= 2 (the roofline kernel)
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, c->s);
  }
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
  const bool overlap = marching && nz >= 3 && (c->comm != nullptr || force_split);
  for (int k = 2; k <= s && rc == PC_OK; ++k) {
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
    c->st.kind_launches[kind] += s - 1;
    c->st.kind_units[kind] += (int64_t)(s - 1) * g->g.N;
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
  if (!op || !u || u->ncomp != op->ncomp) return fail(PC_E_INVALID, "shape mismatch");
  if (kind != PC_RKL2 && kind != PC_RKG2) return fail(PC_E_INVALID, "unknown STS kind");
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
  if (!op || !u || u->ncomp != op->ncomp) return fail(PC_E_INVALID, "shape mismatch");
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

// ------------------------------------------------------------------ PCG
// r-slabs: finish a PCG reduction after the allreduce of the local sums
static int pcg_split_fin(pc_ctx* c, bool split, int mode, int nred, double tol, int it) {
  if (!split) return PC_OK;
  TRY(allreduce_d(c, c->pcg->red, (size_t)nred, nccl::kSum));
  k_pcg_fin<<<1, 1, 0, c->s>>>(c->pcg, mode, tol, it);
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
  // split reductions: the kernels stop at the local sums, NCCL adds them up
  // (the r-line preconditioner is single-rank and finishes its own reductions)
  const bool split = c->comm != nullptr && !line;
  if (rc == PC_OK && cudaMemsetAsync(&c->pcg->split, split ? 1 : 0, sizeof(int), c->s) != cudaSuccess)
    rc = fail(PC_E_CUDA, "PCG state");
  if (rc == PC_OK) {
    if constexpr (std::is_same<Op, AlignedOp>::value) {
      // r = b - A x0 through the marching kernel (x0 staged like any T)
      if (adiag) {
        EpiPcgInitT<true> e{b.p[0], dg, adiag, r.base(0), p0.base(0), dt, c->red_v, c->red_v2, c->counter, c->pcg,
                            line};
        rc = launch_march(op, cfld(x).p[0], e, nullptr, "k_aligned_march<pcg init>");
      } else {
        EpiPcgInitT<false> e{b.p[0], dg, adiag, r.base(0), p0.base(0), dt, c->red_v, c->red_v2, c->counter, c->pcg,
                             line};
        rc = launch_march(op, cfld(x).p[0], e, nullptr, "k_aligned_march<pcg init>");
      }
      if (rc == PC_OK && line) {  // z0 = M^{-1} r0, (r0, z0) -> fin_init
        rc = line_prepare(op, dt, adiag, Lf);
        if (rc == PC_OK) rc = line_apply(op, r.base(0), Lf, dt, z.base(0), 0);
      }
    } else {
      k_pcg_init<<<nb, kThreads, 0, c->s>>>(g->g, o, b, cfld(x), r.f(), p0.f(), dg, adiag, dt, c->red_v, c->red_v2,
                                            c->counter, c->pcg);
      c->st.launches++;
      rc = check_launch("k_pcg_init");
    }
    if (rc == PC_OK) rc = pcg_split_fin(c, split, 0, 2, tol, 0);
  }
  Work* pold = &p0;
  Work* pnew = &p1;
  const int batch = 4;
  int it = 0;
  bool stop = false;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, c->s);
  }
  while (rc == PC_OK && !stop && it < max_iter) {
    for (int q = 0; q < batch && it < max_iter && rc == PC_OK; ++q) {
      ++it;
      if constexpr (std::is_same<Op, AlignedOp>::value) {
        // p = z + beta p_old (beta from the device-side PCG state), then the
        // marching matvec stages p like any other field
        if (line)
          k_pcg_pupdate_z<<<nb, kThreads, 0, c->s>>>(g->g, z.base(0), pold->base(0), pnew->base(0), c->pcg);
        else
          k_pcg_pupdate<<<nb, kThreads, 0, c->s>>>(g->g, r.base(0), pold->base(0), pnew->base(0), dg, adiag, dt,
                                                   c->pcg);
        c->st.launches++;
        rc = check_launch("k_pcg_pupdate");
        if (rc == PC_OK) rc = halo_work(g, *pnew);
        if (rc) break;
        const int* done = reinterpret_cast<const int*>(reinterpret_cast<const char*>(c->pcg) + offsetof(PcgDev, done));
        if (adiag) {
          EpiMatvecT<true> e{adiag, Ap.base(0), dt, c->red_v, c->counter, c->pcg};
          rc = launch_march(op, pnew->base(0), e, done, "k_aligned_march<matvec>");
        } else {
          EpiMatvecT<false> e{adiag, Ap.base(0), dt, c->red_v, c->counter, c->pcg};
          rc = launch_march(op, pnew->base(0), e, done, "k_aligned_march<matvec>");
        }
        if (rc == PC_OK) rc = pcg_split_fin(c, split, 1, 1, tol, it);
        if (rc) break;
      } else {
        rc = halo_work(g, r);
        if (rc == PC_OK) rc = halo_work(g, *pold);
        if (rc) break;
        k_pcg_matvec<<<nb, kThreads, 0, c->s>>>(g->g, o, r.cf(), pold->cf(), pnew->f(), Ap.f(), dg, adiag, dt,
                                                c->red_v, c->counter, c->pcg);
        rc = check_launch("k_pcg_matvec");
        if (rc == PC_OK) rc = pcg_split_fin(c, split, 1, 1, tol, it);
        if (rc) break;
      }
      if constexpr (std::is_same<Op, AlignedOp>::value) {
        auto upd = line ? (o.rho ? (adiag ? k_pcg_update1<true, true, true> : k_pcg_update1<true, false, true>)
                                 : (adiag ? k_pcg_update1<false, true, true> : k_pcg_update1<false, false, true>))
                        : (o.rho ? (adiag ? k_pcg_update1<true, true> : k_pcg_update1<true, false>)
                                 : (adiag ? k_pcg_update1<false, true> : k_pcg_update1<false, false>));
        upd<<<nb, kThreads, 0, c->s>>>(g->g, x->base(0), r.base(0), pnew->base(0), Ap.base(0), dg, adiag, o.rho, dt,
                                       tol, it, c->red_v, c->red_v2, c->counter, c->pcg);
      } else {
        k_pcg_update<<<nb, kThreads, 0, c->s>>>(g->g, o, fld(x), r.f(), pnew->cf(), Ap.cf(), dg, adiag, dt, tol, it,
                                                c->red_v, c->red_v2, c->counter, c->pcg);
      }
      c->st.launches += std::is_same<Op, AlignedOp>::value ? 1 : 2;  // (march counted at launch)
      c->st.stage_launches += std::is_same<Op, AlignedOp>::value ? 3 : 2;
      rc = check_launch("k_pcg");
      if (rc == PC_OK) rc = pcg_split_fin(c, split, 2, 2, tol, it);
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
    c->st.kind_launches[pkind] += (int64_t)c->h_pcg->it * (std::is_same<Op, AlignedOp>::value ? 3 : 2);
    c->st.kind_units[pkind] += (int64_t)c->h_pcg->it * g->g.N;
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
  if (!op || !b || !x || !iters || !relres || !converged) return fail(PC_E_INVALID, "null argument");
  if (b->ncomp != op->ncomp || x->ncomp != op->ncomp) return fail(PC_E_INVALID, "shape mismatch");
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
  if (!op || !u || u->ncomp != op->ncomp || !iters || !relres || !converged) return fail(PC_E_INVALID, "bad arguments");
  if (!(tol > 0.0 && tol < 1.0) || max_iter < 1) return fail(PC_E_INVALID, "need 0 < tol < 1 and max_iter >= 1");
  TRY(need_frozen(op));
  if (!op->frozen) TRY(pc_op_freeze(op, nullptr));
  return be_step(op, u, dt, tol, max_iter, iters, relres, converged);
}

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
  pc_cycle_record* drec = nullptr;
  int rc = PC_OK;
  if (cap > 0 && cudaMalloc(&drec, (size_t)cap * sizeof(pc_cycle_record)) != cudaSuccess)
    rc = fail(PC_E_CUDA, "cycle record allocation failed");
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
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
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
  if (drec) cudaFree(drec);
  work_put(A);
  work_put(B);
  work_put(y0);
  return rc;
}

int pc_cycle(pc_op* op, pc_field* u, double outer_dt, int scheme, int make_odd, double tol, int max_iter,
             double eps_rel, int check_all, int use_ptl, int floor_mode, double floor_fraction, int64_t max_cycles,
             double dt_euler, pc_cycle_record* rec, int64_t rec_cap, int64_t* n_rec) {
  if (!op || !u || !n_rec || u->ncomp != op->ncomp) return fail(PC_E_INVALID, "bad cycle arguments");
  if (!(outer_dt > 0.0)) return fail(PC_E_INVALID, "outer_dt must be > 0");
  if (max_cycles < 1 || !(eps_rel > 0.0)) return fail(PC_E_INVALID, "need max_cycles >= 1 and eps_rel > 0");
  if (scheme < PC_RKL2 || scheme > PC_EULER) return fail(PC_E_INVALID, "unknown scheme");
  TRY(need_frozen(op));
  if (!op->frozen) TRY(pc_op_freeze(op, nullptr));
  pc_grid* g = op->grid;
  pc_ctx* c = g->ctx;
  const double dtE = dt_euler > 0.0 ? dt_euler : op->dt_euler;
  const double floor_dt = floor_mode == PC_FLOOR_EULER ? dtE : floor_fraction * dtE;
  double remaining = outer_dt;
  int64_t cyc = 0;
  *n_rec = 0;
  if ((scheme == PC_RKL2 || scheme == PC_RKG2) && !check_all && persist_ok(op))
    return cycle_persistent(op, u, outer_dt, scheme, make_odd, eps_rel, use_ptl, floor_dt, dtE, max_cycles, rec, rec_cap,
                            n_rec);
  Work y0;
  TRY(work_get(g, op->ncomp, y0));
  int rc = PC_OK;
  std::vector<double> tab;
  c->bad_pending = false;
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
    rc = halo_field(u);
    if (rc) break;
    rc = apply_any(op, cfld(u), y0.f(), true);
    if (rc) break;
    if (use_ptl) {
      double* yb[3] = {y0.b[0], y0.b[1], y0.b[2]};
      rc = ptl_device(g, op->ncomp, cfld(u), y0.cf(), yb, eps_rel, check_all);
      if (rc) break;
    }
    double ptl;
    int limited;
    rc = ptl_read(c, check_all, use_ptl, &ptl, &limited, nullptr);
    if (rc) break;
    rc = check_pending_bad(c);  // ptl_read synchronised the stream
    if (rc) break;
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
      rc = sts_any(op, u, tab.data(), s, y0, true);
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
  if (rc == PC_OK) {
    CUDA_TRY(cudaStreamSynchronize(c->s));
    rc = check_pending_bad(c);
  }
  c->bad_pending = false;
  return rc;
}


// ------------------------------------------------------------------ synthetic inputs
// (configs.py recipes evaluated in HBM; tables are GLOBAL-grid tables)
static int upload_tmp(pc_ctx* c, const double* host, size_t n, double** dev) {
  CUDA_TRY(cudaMalloc(dev, n * sizeof(double)));
  CUDA_TRY(cudaMemcpyAsync(*dev, host, n * sizeof(double), cudaMemcpyHostToDevice, c->s));
  return PC_OK;
}
static const double kSqrt3 = 1.7320508075688772;  // math.sqrt(3.0)

int pc_gen_temperature(pc_field* T, uint64_t seed, int stream, double sigma, const double* prof) {
  if (!T || T->ncomp != 1 || !prof) return fail(PC_E_INVALID, "temperature: scalar field and profile needed");
  pc_grid* g = T->grid;
  pc_ctx* c = g->ctx;
  double* dp = nullptr;
  TRY(upload_tmp(c, prof, (size_t)g->g.n0g, &dp));
  k_gen_temperature<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, T->base(0), stream_key(seed, stream), sigma,
                                                                  dp, kSqrt3);
  c->st.launches++;
  int rc = check_launch("k_gen_temperature");
  cudaStreamSynchronize(c->s);
  cudaFree(dp);
  return rc;
}

int pc_gen_dipole(pc_field* b, uint64_t seed, int stream0, double eps, const double* ir3, const double* c2,
                  const double* st) {
  if (!b || b->ncomp != 3 || !ir3 || !c2 || !st) return fail(PC_E_INVALID, "dipole: 3-component field and tables");
  pc_grid* g = b->grid;
  pc_ctx* c = g->ctx;
  double *d0 = nullptr, *d1 = nullptr, *d2 = nullptr;
  TRY(upload_tmp(c, ir3, (size_t)g->g.n0g, &d0));
  TRY(upload_tmp(c, c2, (size_t)g->g.n1, &d1));
  TRY(upload_tmp(c, st, (size_t)g->g.n1, &d2));
  k_gen_dipole<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, fld(b), stream_key(seed, stream0),
                                                             stream_key(seed, stream0 + 1),
                                                             stream_key(seed, stream0 + 2), eps, d0, d1, d2, kSqrt3);
  c->st.launches++;
  int rc = check_launch("k_gen_dipole");
  cudaStreamSynchronize(c->s);
  cudaFree(d0);
  cudaFree(d1);
  cudaFree(d2);
  return rc;
}

int pc_gen_harmonic(pc_field* v, const double* acc, double checker) {
  if (!v || !acc) return fail(PC_E_INVALID, "harmonic: field and (ncomp, n1, n2) table needed");
  pc_grid* g = v->grid;
  pc_ctx* c = g->ctx;
  double* da = nullptr;
  TRY(upload_tmp(c, acc, (size_t)v->ncomp * g->g.n1 * g->g.n2, &da));
  k_gen_harmonic<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, fld(v), v->ncomp, da, checker);
  c->st.launches++;
  int rc = check_launch("k_gen_harmonic");
  cudaStreamSynchronize(c->s);
  cudaFree(da);
  return rc;
}

int pc_gen_radial(pc_field* f, const double* tab) {
  if (!f || f->ncomp != 1 || !tab) return fail(PC_E_INVALID, "radial: scalar field and table needed");
  pc_grid* g = f->grid;
  pc_ctx* c = g->ctx;
  double* dt = nullptr;
  TRY(upload_tmp(c, tab, (size_t)g->g.n0g, &dt));
  k_gen_radial<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, f->base(0), dt);
  c->st.launches++;
  int rc = check_launch("k_gen_radial");
  cudaStreamSynchronize(c->s);
  cudaFree(dt);
  return rc;
}
