// host_lane.cpp — the hybrid CPU lane's host-side Steps 1-3 (see host_lane.h).
#include "host_lane.h"

#include <omp.h>

#include <climits>
#include <cmath>

namespace sx {

static inline bool cand_less(const HostCand& a, const HostCand& b) {
  return a.v < b.v || (a.v == b.v && a.idx < b.idx);
}

bool HostLane::build(const double* Acols, long long ncols_a, const double* c, const double* b) {
  T.assign((size_t)((m + 1) * hw), 0.0);
  rhs.assign((size_t)(m + 1), 0.0);
  basis.resize((size_t)m);
  for (long long q = 0; q < ncols_a; ++q) {                 // structural columns: -c, A
    if (!std::isfinite(c[c0 + q])) return false;
    T[(size_t)q] = -c[c0 + q];
  }
  for (long long i = 1; i <= m; ++i) {
    double* row = T.data() + i * hw;
    for (long long q = 0; q < ncols_a; ++q) {
      const double v = Acols[(i - 1) * ncols_a + q];
      if (!std::isfinite(v)) return false;
      row[q] = v;
    }
    const long long js = n + i - 1;                         // slack x_{n+i}
    if (js >= c0 && js < c0 + hw) row[js - c0] = 1.0;
    rhs[(size_t)i] = b[i - 1];
    basis[(size_t)(i - 1)] = (int)js;
  }
  return true;
}

HostCand HostLane::candidate(double tol_opt) const {
  HostCand best{INFINITY, LLONG_MAX};
  for (long long q = 0; q < hw; ++q) {
    const double v = T[(size_t)q];
    if (v < -tol_opt) {
      const HostCand cnd{rule ? 0.0 : v, c0 + q};
      if (cand_less(cnd, best)) best = cnd;
    }
  }
  return best;
}

void HostLane::column(long long j, double* out) const {
  for (long long i = 0; i <= m; ++i) out[i] = T[(size_t)(i * hw + (j - c0))];
}

HostCand HostLane::ratio(const double* col, double tol_piv) const {
  HostCand best{INFINITY, LLONG_MAX};
  for (long long i = 1; i <= m; ++i) {
    const double a = col[i];
    if (a > tol_piv) {
      const double q = rhs[(size_t)i] / a;
      const long long key = rule ? (((long long)basis[(size_t)(i - 1)] << 32) | i) : i;
      const HostCand cnd{q, key};
      if (cand_less(cnd, best)) best = cnd;
    }
  }
  return best;
}

void HostLane::pivot(long long r, long long k, const double* col) {
  const double p = col[r];
  double* Tr = T.data() + r * hw;
  for (long long q = 0; q < hw; ++q) Tr[q] = Tr[q] / p;   // row r normalized in place, first
  const double pr_rhs = rhs[(size_t)r] / p;
  const int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nt)
  for (long long i = 0; i <= m; ++i) {
    if (i == r) continue;
    double* Ti = T.data() + i * hw;
    const double a = -col[i];
    for (long long q = 0; q < hw; ++q) Ti[q] = std::fma(a, Tr[q], Ti[q]);
    rhs[(size_t)i] = std::fma(a, pr_rhs, rhs[(size_t)i]);
  }
  rhs[(size_t)r] = pr_rhs;
  basis[(size_t)(r - 1)] = (int)k;
}

void HostLane::y_part(double* y) const {
  for (long long q = 0; q < hw; ++q) {
    const long long g = c0 + q;
    if (g >= n && g < n + m) y[g - n] = T[(size_t)q];
  }
}

static inline unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

unsigned long long HostLane::hash() const {
  unsigned long long acc = 0;
  for (long long i = 0; i <= m; ++i)
    for (long long q = 0; q < hw; ++q) {
      double v = T[(size_t)(i * hw + q)];
      unsigned long long bits;
      __builtin_memcpy(&bits, &v, sizeof(bits));
      if (bits == 0x8000000000000000ULL) bits = 0;
      const unsigned long long e = (unsigned long long)(i * W + c0 + q);
      acc += mix64(bits ^ (e * 0x9E3779B97F4A7C15ULL + 0xD1B54A32D192ED03ULL));
    }
  return acc;
}

}  // namespace sx
