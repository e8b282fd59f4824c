// hybrid_lane.c — NEXT #4: how much of the tableau could a host-core lane take?
// The paper splits the columns between the GPUs and the CPU cores in proportion θ (PAPER.md:109-113,
// 181-189).  On a B200 box the split is set by the rates at which each side streams its part of
// the rank-1 update.  This program measures the host side: the update of an (m+1) x W FP64 block
// with the oracle's arithmetic (prow_j = T[r][j] / p; T[i][j] = fma(-col_i, prow_j, T[i][j])),
// OpenMP over rows, on 1 thread and on every host core, and prints GB/s (16 bytes per element).
// Not part of the library.   gcc -O3 -fopenmp -ffp-contract=off scripts/hybrid_lane.c -lm
#include <math.h>
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>

static double now(void) { return omp_get_wtime(); }

static void pivot(double* T, long rows, long W, long r, long k, double* col, double* prow) {
  const double p = T[r * W + k];
  for (long j = 0; j < W; ++j) prow[j] = T[r * W + j] / p;
  for (long i = 0; i < rows; ++i) col[i] = T[i * W + k];
#pragma omp parallel for schedule(static)
  for (long i = 0; i < rows; ++i) {
    double* row = T + i * W;
    if (i == r) {
      for (long j = 0; j < W; ++j) row[j] = prow[j];
    } else {
      const double a = -col[i];
      for (long j = 0; j < W; ++j) row[j] = fma(a, prow[j], row[j]);
    }
  }
}

int main(int argc, char** argv) {
  const long m = argc > 1 ? atol(argv[1]) : 8000, n = argc > 2 ? atol(argv[2]) : 8000;
  const long rows = m + 1, W = n + m + 1;
  const int reps = argc > 3 ? atoi(argv[3]) : 5;
  double* T = (double*)aligned_alloc(64, sizeof(double) * rows * W);
  double* col = (double*)malloc(sizeof(double) * rows);
  double* prow = (double*)malloc(sizeof(double) * W);
  if (!T || !col || !prow) return 1;
#pragma omp parallel for schedule(static)
  for (long i = 0; i < rows; ++i)
    for (long j = 0; j < W; ++j) T[i * W + j] = 1.0 + (double)((i * 131 + j * 7) % 1009) * 1e-3;
  const double bytes = 16.0 * (double)rows * (double)W;
  const int maxt = omp_get_max_threads();
  const int tl[2] = {1, maxt};
  for (int q = 0; q < 2; ++q) {
    omp_set_num_threads(tl[q]);
    pivot(T, rows, W, 1 + q, 3 + q, col, prow);                    // warm-up / first touch
    const double t0 = now();
    for (int s = 0; s < reps; ++s) pivot(T, rows, W, 1 + (s % (rows - 1)), s % (n + m), col, prow);
    const double dt = (now() - t0) / reps;
    printf("{\"threads\": %d, \"m\": %ld, \"n\": %ld, \"s_per_pivot\": %.6f, \"GBps\": %.2f}\n", tl[q], m, n, dt,
           bytes / dt / 1e9);
  }
  return 0;
}
