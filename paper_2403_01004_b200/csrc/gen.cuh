// Seeded synthetic inputs generated in HBM, bit-identical to the host recipes
// of paper_2403_01004_b200/configs.py (temperature, dipole_bhat,
// harmonic_velocity).  Transcendental parts arrive as host-computed 1-D/2-D
// tables; per node only +, -, *, /, sqrt and the splitmix64 counter hash are
// evaluated, all exactly rounded, so a 768x768x1536 field never has to be
// built (or uploaded) from the host.
#pragma once
#include "kernels.cuh"

namespace pc {

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// configs.hash_normal: Irwin-Hall(4) of counter hashes, (s - 2) * sqrt(3)
__device__ __forceinline__ double hash_normal(unsigned long long key, unsigned long long idx, double sqrt3) {
  const unsigned long long base = splitmix64(idx ^ key) * 4ULL;
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const unsigned long long h = splitmix64(base + (unsigned long long)t);
    const double u = (double)(h >> 11) * 0x1.0p-53;
    s = t == 0 ? u : s + u;
  }
  return (s - 2.0) * sqrt3;
}
__host__ __device__ __forceinline__ unsigned long long stream_key(unsigned long long seed, int stream) {
  return ((seed & 0xFFFFFFFFULL) << 32) | ((unsigned long long)(stream & 0xFFFF) << 16);
}
__device__ __forceinline__ unsigned long long global_index(const GridDev& g, int i, int j, int k) {
  return ((unsigned long long)(i + g.i0g) * g.n1 + j) * n2glob(g) + kglob(g, k);
}

// T = prof(r) * (1 + sigma * N)                       (configs.temperature)
__global__ void __launch_bounds__(kThreads) k_gen_temperature(GridDev g, double* T, unsigned long long key,
                                                              double sigma, const double* prof, double sqrt3) {
  PC_FOR_NODES(g, i, j, k) {
    const double nz = hash_normal(key, global_index(g, i, j, k), sqrt3);
    T[off3(g, i, j, k)] = prof[i + g.i0g] * (1.0 + sigma * nz);
  }
}

// b = normalise(B_dip + eps |B_dip| (N1, N2, N3))      (configs.dipole_bhat)
__global__ void __launch_bounds__(kThreads) k_gen_dipole(GridDev g, Fld b, unsigned long long k2,
                                                         unsigned long long k3, unsigned long long k4, double eps,
                                                         const double* ir3, const double* c2, const double* st,
                                                         double sqrt3) {
  PC_FOR_NODES(g, i, j, k) {
    const unsigned long long idx = global_index(g, i, j, k);
    const double Br = (c2[j] * ir3[i + g.i0g]) * 1.0;
    const double Bt = (st[j] * ir3[i + g.i0g]) * 1.0;
    const double mag = sqrt(Br * Br + Bt * Bt);
    const double a = eps * mag;
    const double bx = Br + a * hash_normal(k2, idx, sqrt3);
    const double by = Bt + a * hash_normal(k3, idx, sqrt3);
    const double bz = a * hash_normal(k4, idx, sqrt3);
    const double nrm = sqrt((bx * bx + by * by) + bz * bz);
    const int64_t o = off3(g, i, j, k);
    b.p[0][o] = bx / nrm;
    b.p[1][o] = by / nrm;
    b.p[2][o] = bz / nrm;
  }
}

// v_c = acc_c(theta, phi) + checker * (-1)^(i+j+k)     (configs.harmonic_velocity)
__global__ void __launch_bounds__(kThreads) k_gen_harmonic(GridDev g, Fld v, int ncomp, const double* acc,
                                                           double checker) {
  PC_FOR_NODES(g, i, j, k) {
    const int kg = kglob(g, k);  // (phi-slab ghost columns hold the neighbours' values)
    const double cb = ((i + g.i0g + j + kg) % 2 == 0) ? checker : -checker;
    const int64_t o = off3(g, i, j, k);
    for (int c = 0; c < ncomp; ++c) v.p[c][o] = acc[((int64_t)c * g.n1 + j) * n2glob(g) + kg] + cb;
  }
}

// rho = table(r)                                         (configs.c5 rho_r)
__global__ void __launch_bounds__(kThreads) k_gen_radial(GridDev g, double* f, const double* tab) {
  PC_FOR_NODES(g, i, j, k) { f[off3(g, i, j, k)] = tab[i + g.i0g]; }
}

}  // namespace pc
