// host_lane.h — the hybrid CPU lane (the paper's own contribution,
// PAPER.md §IV lines 100-123 and §V.C): a θ share of the tableau's columns lives in
// host memory and is updated by the host cores (OpenMP) while the GPU updates the rest.
//
// Paper: the columns are split between the CPU cores and the GPUs in
// proportion θ; per iteration each worker finds its best reduced cost, the winner's column data
// are sent to the others, every worker runs the ratio test / pivot on its own columns.  Here the
// host lane owns the LAST hw global columns [c0, c0 + hw) of the n+m non-rhs columns plus a
// replicated rhs column and basis; it is the host-side half of one pivot:
//   candidate()  Step 1 over its columns (Dantzig (v, j) / Bland (0, j), reading c1-c3)
//   column(j)    its column j, for the GPU when the host candidate wins
//   ratio()      Step 2 on the winning column against the replicated rhs (readings c4-c6)
//   pivot()      Step 3 on its columns and the rhs: prow_j = T[r][j] / p (IEEE division),
//                T[i][j] = fma(-col[i], prow_j, T[i][j]) for i != r — reading c8 with the host's
//                IEEE double arithmetic (std::fma, built with -ffp-contract=off), row loop split
//                over the host threads: every element gets exactly one fma, so the bits equal the
//                GPU's and the oracle's.
// This is the product's own host code (not the oracle's): it shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <vector>

namespace sx {

struct HostCand {
  double v;
  long long idx;
};

class HostLane {
 public:
  long long m = 0, n = 0, c0 = 0, hw = 0, W = 0;   // W: global tableau width n+m+1
  int rule = 0, threads = 0;
  std::vector<double> T;       // (m+1) x hw, row-major
  std::vector<double> rhs;     // m+1, replicated rhs column (row 0: the objective)
  std::vector<int> basis;      // m, replicated basis (global column of row i's basic variable)

  // Table I for the lane's columns from host copies of A's columns
  // [c0, min(n, c0+hw)) (row-major m x ncols_a), c and b.  false: a non-finite value.
  bool build(const double* Acols, long long ncols_a, const double* c, const double* b);
  HostCand candidate(double tol_opt) const;
  void column(long long j, double* out) const;
  HostCand ratio(const double* col, double tol_piv) const;
  void pivot(long long r, long long k, const double* col);
  void y_part(double* y) const;             // y_i for the lane's slack columns (others untouched)
  unsigned long long hash() const;          // its share of simplex_tableau_hash (columns only)
};

}  // namespace sx
