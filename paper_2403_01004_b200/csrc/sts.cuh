// STS stage counts and coefficient tables (PAPER.md
// Appendix A; RKL2 per Meyer et al.), one source for the host entry points
// (pc_sts_count / pc_sts_table) and the persistent small-grid cycle kernel,
// so host- and device-decided cycles agree bit for bit (IEEE +,-,*,/,sqrt,
// ceil; no contraction: -fmad=false / -ffp-contract=off).
#pragma once
#include <cmath>

namespace pc {

constexpr int kRKL2 = 0, kRKG2 = 1;  // == PC_RKL2, PC_RKG2 (include/paracycle_b200.h)

__host__ __device__ inline int sts_count_hd(int kind, double dt, double dt_euler, int make_odd) {
  const double r = dt / dt_euler;
  if (kind == kRKL2) {
    long long s = (long long)ceil((sqrt(9.0 + 16.0 * r) - 1.0) / 2.0);
    if (make_odd && s % 2 == 0) s += 1;
    return (int)(s > 2 ? s : 2);
  }
  if (kind == kRKG2) {
    long long s = (long long)ceil(0.5 * sqrt(25.0 + 24.0 * r) - 1.5);
    if (s % 2 == 0) s += 1;
    return (int)(s > 3 ? s : 3);
  }
  return -1;
}

// rows k = 1..s of (mu, nu, 1 - mu - nu, mut dt, gam dt); returns false on a bad (kind, s)
__host__ __device__ inline bool sts_rows_hd(int kind, int s, double dt, double* out) {
  if (kind == kRKL2) {
    if (s < 2) return false;
    const double sd = s;
    const double w1 = 4.0 / ((sd * sd + sd) - 2.0);
    auto bj = [](int j) {
      const double jd = j;
      return j <= 2 ? 1.0 / 3.0 : ((jd * jd + jd) - 2.0) / ((2.0 * jd) * (jd + 1.0));
    };
    double bm2 = bj(0), bm1 = bj(1);
    out[0] = 0.0;
    out[1] = 0.0;
    out[2] = (1.0 - 0.0) - 0.0;
    out[3] = (bm1 * w1) * dt;
    out[4] = 0.0 * dt;
    for (int j = 2; j <= s; ++j) {
      const double jd = j;
      const double b = bj(j);
      const double mu = (((2.0 * jd - 1.0) / jd) * b) / bm1;
      const double nu = ((-(jd - 1.0) / jd) * b) / bm2;
      const double mut = mu * w1;
      const double gam = (-(1.0 - bm1)) * mut;
      double* r = out + 5 * (j - 1);
      r[0] = mu;
      r[1] = nu;
      r[2] = (1.0 - mu) - nu;
      r[3] = mut * dt;
      r[4] = gam * dt;
      bm2 = bm1;
      bm1 = b;
    }
    return true;
  }
  if (kind == kRKG2) {
    if (s < 3 || s % 2 == 0) return false;
    const double sd = s;
    const double w = 6.0 / ((sd + 4.0) * (sd - 1.0));
    // k = 1: mu 1, nu 0, mut w, gam 0;  k = 2: mu 1/2, nu -1/10, gam 0
    out[0] = 1.0;
    out[1] = 0.0;
    out[2] = (1.0 - 1.0) - 0.0;
    out[3] = w * dt;
    out[4] = 0.0 * dt;
    const double mu2 = 0.5, nu2 = -0.1, mut2 = mu2 * w;
    out[5] = mu2;
    out[6] = nu2;
    out[7] = (1.0 - mu2) - nu2;
    out[8] = mut2 * dt;
    out[9] = 0.0 * dt;
    double bm2 = 1.0 / 3.0, bm1 = 1.0 / 15.0;  // b[1], b[2]
    for (int k = 3; k <= s; ++k) {
      const double kd = k;
      const double b = ((4.0 * (kd - 1.0)) * (kd + 4.0)) / ((((3.0 * kd) * (kd + 1.0)) * (kd + 2.0)) * (kd + 3.0));
      const double mu = ((2.0 + 1.0 / kd) * b) / bm1;
      const double nu = ((-(1.0 / kd + 1.0)) * b) / bm2;
      const double mut = mu * w;
      const double gam = ((((kd * (kd + 1.0)) / 2.0) * bm1) - 1.0) * mut;
      double* r = out + 5 * (k - 1);
      r[0] = mu;
      r[1] = nu;
      r[2] = (1.0 - mu) - nu;
      r[3] = mut * dt;
      r[4] = gam * dt;
      bm2 = bm1;
      bm1 = b;
    }
    return true;
  }
  return false;
}

}  // namespace pc
