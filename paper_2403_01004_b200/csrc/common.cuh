// Shared device-side types and helpers for the paracycle_b200 kernels.
//
// Layout: each field component is one fp64
// array [n0 + 2][n1][n2] (phi = axis 2 fastest, 128-B coalesced rows); the
// base pointer handed to kernels points at interior plane 0, so axis-0 ghost
// planes are at i = -1 and i = n0 (used only by r-slab decomposition).
// 2-D metric tables are [n0 + 2][n1] with the same ghost-row convention,
// 1-D tables are [n2] (axis 2) or [n1] (rotation tables).
//
// Parity rule: every expression below is written in the operation order of
// the numpy oracle (oracle/operators.py, oracle/schemes.py) and the library
// is compiled with -fmad=false, so results are bitwise identical to the
// oracle wherever the oracle is elementwise.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pc {

constexpr int kThreads = 256;

struct GridDev {
  int n0, n1, n2;          // local interior shape
  int n0g;                 // global n0
  int i0g;                 // global axis-0 offset of this slab
  int64_t plane;           // n1 * n2
  int64_t N;               // n0 * n1 * n2
  int per0, per1, per2;    // periodic axes
  int pin_lo0, pin_hi0, pin_lo1, pin_hi1, pin_lo2, pin_hi2;
  int ghost_lo0, ghost_hi0;  // neighbour slab exists (read the ghost plane)
  int spherical;
  // phi-slab rank (phis = 1): local columns 1 .. n2-2 are the global columns
  // k0g .. k0g + n2 - 3; columns 0 and n2-1 are ghost copies of the
  // neighbour ranks' edge columns (pinned, zero weight: they are read as
  // neighbours and never advanced or summed); phi stays periodic
  int phis;
  int n2g, k0g;            // global n2, global phi offset of the owned columns
  // scalar finite-volume tables
  const double* W2[3];
  const double* g1[3];
  const double* iV2;
  const double* igv;
  // aligned (corner-tetrahedron) tables; index a*2 + s (s: 0 = '+', 1 = '-')
  const double* iL2[6];
  const double* iL1[6];
  const double* wo01[4];   // (s0, s1) in order ++, +-, -+, --
  const double* wo2[2];
  const double* iVal2;
  const double* iValg;
  // vector rotation tables (t+, t-, p+, p-): M [n1][9], Rabs [n1][3]
  const double* M[4];
  const double* Rabs[4];
  // weights for the PCG inner product
  const double* V2;
  const double* gv;
  const double* Val2;
  const double* Valg;
};

// global phi index / extent of a local column (phi-slabs: ghost columns map
// to the neighbours' columns, periodically)
__device__ __forceinline__ int kglob(const GridDev& g, int k) {
  return g.phis ? (k - 1 + g.k0g + g.n2g) % g.n2g : k;
}
__device__ __forceinline__ int n2glob(const GridDev& g) { return g.phis ? g.n2g : g.n2; }
// cells this rank owns (phi-slabs: without the ghost columns)
__host__ __device__ __forceinline__ int64_t owned_cells(const GridDev& g) {
  return (int64_t)g.n0 * g.n1 * (g.n2 - 2 * g.phis);
}
__device__ __forceinline__ int64_t off3(const GridDev& g, int i, int j, int k) {
  return (int64_t)i * g.plane + (int64_t)j * g.n2 + k;
}
__device__ __forceinline__ int64_t row2(const GridDev& g, int i, int j) {
  return (int64_t)i * g.n1 + j;
}
__device__ __forceinline__ void unflatten(const GridDev& g, int64_t c, int& i, int& j, int& k) {
  k = (int)(c % g.n2);
  int64_t t = c / g.n2;
  j = (int)(t % g.n1);
  i = (int)(t / g.n1);
}

// Node iteration of the generic kernels: each warp takes one (i, j) row and
// its lanes stride along phi (coalesced, no 64-bit division per node).
#define PC_FOR_NODES(g, i, j, k)                                                                   \
  for (int row_ = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), i = 0, j = 0;              \
       row_ < (g).n0 * (g).n1; row_ += gridDim.x * (blockDim.x >> 5))                             \
    for (int k = ((i = row_ / (g).n1), (j = row_ - i * (g).n1), (int)(threadIdx.x & 31)); k < (g).n2; k += 32)

__device__ __forceinline__ bool pinned(const GridDev& g, int i, int j, int k) {
  int ig = i + g.i0g;
  return (g.pin_lo0 && ig == 0) || (g.pin_hi0 && ig == g.n0g - 1) ||
         (g.pin_lo1 && j == 0) || (g.pin_hi1 && j == g.n1 - 1) ||
         (g.pin_lo2 && k == 0) || (g.pin_hi2 && k == g.n2 - 1);
}

// neighbour coordinate along one axis; ok == false means "no neighbour"
// (the caller then uses the node itself so differences are exactly 0).
__device__ __forceinline__ int nb0(const GridDev& g, int i, int d, bool& ok) {
  int t = i + d;
  if (t >= 0 && t < g.n0) { ok = true; return t; }
  if (t < 0 && g.ghost_lo0) { ok = true; return t; }
  if (t >= g.n0 && g.ghost_hi0) { ok = true; return t; }
  if (g.per0 && g.n0g > 1) { ok = true; return t < 0 ? g.n0 - 1 : 0; }
  ok = false;
  return i;
}
__device__ __forceinline__ int nb1(const GridDev& g, int j, int d, bool& ok) {
  int t = j + d;
  if (t >= 0 && t < g.n1) { ok = true; return t; }
  if (g.per1 && g.n1 > 1) { ok = true; return t < 0 ? g.n1 - 1 : 0; }
  ok = false;
  return j;
}
__device__ __forceinline__ int nb2(const GridDev& g, int k, int d, bool& ok) {
  int t = k + d;
  if (t >= 0 && t < g.n2) { ok = true; return t; }
  if (g.per2 && g.n2 > 1) { ok = true; return t < 0 ? g.n2 - 1 : 0; }
  ok = false;
  return k;
}
__device__ __forceinline__ int nbax(const GridDev& g, int a, int x, int d, bool& ok) {
  return a == 0 ? nb0(g, x, d, ok) : (a == 1 ? nb1(g, x, d, ok) : nb2(g, x, d, ok));
}

// ---------------------------------------------------------------- reductions
// Deterministic block reductions: fixed shuffle tree, then warp 0.
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < NT / 32 ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;  // valid in thread 0
}
template <int NT>
__device__ __forceinline__ double block_max(double v, double* sh) {
  v = warp_max(v);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < NT / 32 ? sh[lane] : 0.0;
    r = warp_max(r);
  }
  __syncthreads();
  return r;
}

// (value, index) argmax with lowest-index tie-break
struct ArgMax {
  double v;
  long long i;
};
__device__ __forceinline__ ArgMax am_better(ArgMax a, ArgMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
__device__ __forceinline__ ArgMax warp_argmax(ArgMax a) {
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b;
    b.v = __shfl_down_sync(0xffffffffu, a.v, o);
    b.i = __shfl_down_sync(0xffffffffu, a.i, o);
    a = am_better(a, b);
  }
  return a;
}
template <int NT>
__device__ __forceinline__ ArgMax block_argmax(ArgMax a, double* shv, long long* shi) {
  a = warp_argmax(a);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { shv[w] = a.v; shi[w] = a.i; }
  __syncthreads();
  ArgMax r{-1.0, 0x7fffffffffffffffLL};
  if (w == 0) {
    if (lane < NT / 32) { r.v = shv[lane]; r.i = shi[lane]; }
    r = warp_argmax(r);
  }
  __syncthreads();
  return r;
}

// "last block finishes the reduction" ticket (threadfence pattern)
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool amLast;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(counter, 1u);
    amLast = (t == gridDim.x - 1);
  }
  __syncthreads();
  return amLast;
}

}  // namespace pc
