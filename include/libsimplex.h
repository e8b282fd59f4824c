/*
 * libsimplex.h — C ABI of the B200-native dense full-tableau simplex hot path.
 *
 * Method: the standard full-tableau simplex of Mamalis & Perlitis (§III,
 * lines 73-96; Table I at lines 77-84), column-distributed as in §IV
 * (PAPER.md:100-123).  Problem statement (Table I's -c row at :80):
 *
 *        maximize c^T x   subject to   A x <= b,  x >= 0,      A is m x n (dense)
 *
 * started from the slack basis (Table I rows x_{n+1..n+m}; "start
 * having as a basis a feasible basic solution") when b >= 0, and from a Phase I basis of
 * artificial variables when some b_i < 0 (two-phase method, options.phase1).
 *
 * Per pivot, entirely on the device (no host round trip per pivot):
 *   Step 1  entering column k = argmin_j T[0][j] over T[0][j] < -tol_opt,
 *           lowest j on exact ties
 *   Step 2  leaving row r = argmin_i T[i][W-1] / T[i][k] over T[i][k] > tol_piv,
 *           lowest i on exact ties; none -> UNBOUNDED
 *   Step 3  prow_j = T[r][j] / p (IEEE division), T[i][j] = fma(-T[i][k], prow_j,
 *           T[i][j]) for i != r, T[r][j] = prow_j
 * T is the (m+1) x W tableau, W = n+m+1: row 0 stores -c, columns n..n+m-1 are
 * the slacks, column W-1 is the rhs; the Z column of Table I is omitted.
 * Readings of every point the paper leaves open are listed in DESIGN.md.
 *
 * Conventions
 *  - Every function returns simplex_err: 0 = SIMPLEX_OK, negative = error.  The
 *    text of the last error on the calling thread is simplex_last_error().
 *  - Solver OUTCOMES (optimal, unbounded, iteration limit) are simplex_status
 *    values, never errors.
 *  - Pointers to problem data and results may be HOST or DEVICE memory of the
 *    handle's GPU; the library copies with cudaMemcpyDefault (unified virtual
 *    addressing tells the runtime which).  Inputs are copied during the call; the caller keeps
 *    ownership and may free them on return.  Outputs go to caller buffers.
 *  - A handle owns all its device memory, streams, CUDA graphs and its NCCL
 *    communicator.  It is not thread-safe: one host thread per handle.
 *  - Multi-GPU (nranks > 1): SPMD, one process per GPU; every rank calls every
 *    function with the same (m, n, A, b, c); each rank keeps the column slab it
 *    owns plus a replicated rhs column.
 *  - Trace indices: k is a 0-based column in [0, n+m); r is a 1-based tableau
 *    row in [1, m] (row 0 is the objective row).
 *  - There is no CPU fallback: without a usable CUDA device every call that
 *    needs one returns SIMPLEX_E_CUDA.
 */
#ifndef LIBSIMPLEX_H
#define LIBSIMPLEX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct simplex_s simplex_t;          /* opaque handle */

typedef enum {
    SIMPLEX_OK = 0,
    SIMPLEX_E_ARG = -1,        /* NULL pointer, m < 1, n < 1, bad option, shape mismatch   */
    SIMPLEX_E_NONFINITE = -2,  /* NaN or Inf in A, b or c                                   */
    SIMPLEX_E_NEG_RHS = -3,    /* some b_i < 0 with phase1 = 0 (phase1 = 1, the default, solves it) */
    SIMPLEX_E_OOM = -4,        /* device or pinned host allocation failed                   */
    SIMPLEX_E_CUDA = -5,       /* CUDA runtime error, or no CUDA device                     */
    SIMPLEX_E_NCCL = -6,       /* NCCL error (multi-GPU)                                    */
    SIMPLEX_E_STATE = -7       /* call not valid in the handle's current state              */
} simplex_err;

typedef enum {
    SIMPLEX_RUNNING = -1,          /* no terminal status reached yet                       */
    SIMPLEX_OPTIMAL = 0,           /* no T[0][j] < -tol_opt                                 */
    SIMPLEX_UNBOUNDED = 2,         /* entering column has no T[i][k] > tol_piv              */
    SIMPLEX_INFEASIBLE = 3,        /* Phase I optimum < -1e-7: Ax <= b, x >= 0 is empty      */
    SIMPLEX_ITERATION_LIMIT = 4    /* max_pivots pivots done and another one was possible   */
} simplex_status;                  /* numbering = SPEC.md:473 exit codes                    */

typedef struct {
    uint32_t struct_size;   /* = sizeof(simplex_options); set by simplex_default_options  */
    double   tol_opt;       /* 1e-7:  column j is a candidate iff T[0][j] < -tol_opt       */
    double   tol_piv;       /* 1e-10: row i is eligible iff T[i][k] > tol_piv              */
    int64_t  max_pivots;    /* iteration cap; <= 0 -> 20*(m+n)                             */
    int32_t  record_trace;  /* 1: keep (k, r) of every pivot on the device (default 1)     */
    int32_t  device;        /* CUDA device ordinal; -1 = the calling thread's current one  */
    int32_t  nranks;        /* GPUs the columns are split over (1, 2, 4, 8 ...)            */
    int32_t  rank;          /* this process's rank in [0, nranks)                          */
    const void* nccl_id;    /* 128-byte ncclUniqueId shared by all ranks (nranks > 1)      */
    void*    stream;        /* cudaStream_t to run on (e.g. torch's current stream); NULL:
                               the handle creates its own non-blocking stream              */
    int32_t  virtual_ranks; /* >1: split the columns into this many slabs on ONE GPU and
                               exchange through device memory (tests the multi-GPU data
                               flow without NCCL); requires nranks == 1                    */
    int32_t  segment_pivots;/* pivots per captured CUDA-graph segment (<= 0: automatic)    */
    int32_t  time_kernels;  /* 1: record CUDA events around every pivot-update launch
                               (see simplex_get_stats); the pipelined rank-s pass is timed
                               on the device instead (%globaltimer, first CTA start to
                               last CTA end), so it still overlaps the selection          */
    int32_t  lookahead;     /* pivots applied per pass over the tableau: 1 = one pivot per pass;
                               2..16 = rank-s look-ahead blocks (select s pivots ahead from
                               chained corrections, then ONE pass applies all s — bitwise
                               identical to s single pivots; on several column parts one
                               allgather of candidate columns per selected pivot);
                               17..32 = pair schedule (one column part): two selections of
                               16 + (s-16) pivots, then ONE pass applies all s (no pipeline;
                               pays off on tableaux whose pass dominates, 20000x40000);
                               0 (default) = automatic: a tableau that fits in one CTA's
                               shared memory (one column part, no Phase I; e.g. 64x64) is
                               solved by ONE single-CTA launch with the tableau on chip
                               (stats.path = 1), anything else uses 16; > 32 -> SIMPLEX_E_ARG */
    int32_t  pivot_rule;    /* 0 = Dantzig (default): most negative T[0][j], lowest j / lowest
                               row on ties (readings c1-c4); 1 = Bland: first j
                               with T[0][j] < -tol_opt, ratio ties -> smallest basic-variable
                               index (anti-cycling)   */
    int32_t  phase1;        /* 1 (default): b with negative entries runs the two-phase method
                               (artificials, Phase I objective, drive-out, Phase II; every
                               path incl. column parts) and may end
                               INFEASIBLE;
                               0: b_i < 0 is rejected with SIMPLEX_E_NEG_RHS               */
    int32_t  overlap;       /* rank-s look-ahead only.  1 (default): software pipeline —
                               block b+1 is selected (on one thread-block cluster) WHILE
                               block b's pass runs on the other SMs, out of place between
                               two tableau buffers (2x the tableau's HBM; falls back to 0
                               when 2.2x the tableau exceeds the free device memory); 0:
                               select, then pass, in place.  Bitwise identical results.    */
    int32_t  exchange;      /* multi-part rank-s look-ahead (nranks > 1 or virtual_ranks > 1):
                               0 (default) = on several ranks, peer memory when every peer
                               GPU is reachable (k_mlook stores its candidate column straight
                               into every rank's gather buffer over NVLink via CUDA IPC and
                               releases a flag there — no collective launch per pivot), else
                               NCCL; on virtual slabs, plain stores into the shared buffer;
                               1 = one ncclAllGather per selected pivot (virtual slabs: plain
                               stores; ONE column part: the same gather through a 1-rank NCCL
                               communicator — the NCCL data flow testable on one GPU);
                               2 = the peer-memory protocol (also on virtual slabs: its test
                               path) or SIMPLEX_E_CUDA; 3 = as 2 but one k_mlook launch per
                               selected pivot instead of one k_mblock per block (test path of
                               the per-pivot protocol).  > 3 -> SIMPLEX_E_ARG.  Bitwise
                               identical results.                                          */
    int32_t  exchange_timeout_ms; /* peer-memory exchange: a poll for a peer's candidate
                               column gives up after this long (<= 0: 30000), stops the loop,
                               returns SIMPLEX_E_NCCL and latches the handle (every later call
                               except destroy returns SIMPLEX_E_STATE).  Raise it when ranks may
                               launch far apart (e.g. under a profiler's kernel replay).    */
    double   host_share;    /* hybrid CPU lane: the share
                               θ in [0, 1) of the n+m columns kept in host memory and updated by
                               the host cores (the LAST round(θ(n+m)) columns; at least one column
                               stays on the GPU).  0 (default): off.  > 0 requires one GPU rank, no
                               virtual ranks, lookahead 0 or 1 (one pivot per pass: the lanes
                               exchange candidates every pivot), b >= 0; else SIMPLEX_E_ARG.
                               Bitwise identical results.                                  */
    int32_t  host_threads;  /* host threads of the CPU lane (<= 0: OpenMP's default)         */
} simplex_options;

typedef struct {
    int64_t pivots;              /* pivots performed so far                                  */
    int64_t update_launches;     /* timed pivot-update (K3) launches                         */
    double  update_ms_total;     /* sum of their durations (time_kernels = 1)                */
    double  loop_ms_total;       /* CUDA-event time of the device iteration loop             */
    int64_t graph_launches;      /* CUDA-graph segment launches                              */
    int64_t kernel_launches;     /* kernels of this library launched by the loop so far      */
    int64_t local_rows;          /* m + 1                                                    */
    int64_t local_cols;          /* columns of this rank's slab incl. the rhs column         */
    int64_t local_ld;            /* padded row pitch of the slab, in doubles                 */
    int64_t col_offset;          /* first global column of this rank's slab                  */
    int64_t bytes_per_pivot;     /* algorithmic bytes of one update: 16*(m+1)*local_cols     */
    int64_t path;                /* 0: device loop of captured CUDA-graph segments; 1: the whole
                                    solve in one single-CTA launch with the tableau in shared
                                    memory (small tableaux, lookahead = 0); 2: hybrid CPU lane;
                                    3: as 0 with the shared-memory look-ahead selection k_look2
                                    (one column part, m + 1 <= 4096 and pitch <= 8192 doubles) */
    int64_t host_cols;           /* columns of the hybrid CPU lane (0: none)                  */
    double  host_ms_total;       /* host time spent updating the CPU lane's columns           */
    double  host_wait_ms_total;  /* host time spent waiting for the GPU's candidate per pivot */
} simplex_stats;

/* Fill *o with the defaults above. */
void simplex_default_options(simplex_options* o);

/* Allocate a handle on the GPU, copy (A, b, c), build Table I.
 *   A: m x n row-major (lda = n), b: m (entries < 0 run Phase I, options.phase1), c: n — host or
 *   device memory.
 *   opt may be NULL (defaults, 1 GPU).  Errors: ARG, NONFINITE, NEG_RHS, OOM, CUDA,
 *   NCCL.  On error *out is NULL. */
simplex_err simplex_create(simplex_t** out, int64_t m, int64_t n,
                           const double* A, const double* b, const double* c,
                           const simplex_options* opt);

/* Rebuild the tableau from new data of the same shape (re-solve without
 * re-allocating): status RUNNING, 0 pivots, trace cleared.  Same errors as create. */
simplex_err simplex_reset(simplex_t* h, const double* A, const double* b, const double* c);

/* Run up to max_pivots more pivots (<= 0: until termination).  *pivots_done (may be
 * NULL) receives the pivots done by this call, *st (may be NULL) the status after it.
 * Termination is detected at the start of an iteration: a state that
 * is optimal right after the last pivot of this call still reports RUNNING, and the
 * next call returns it with 0 pivots.  After a terminal status returns OK, 0 pivots. */
simplex_err simplex_iterate(simplex_t* h, int64_t max_pivots, int64_t* pivots_done,
                            simplex_status* st);

/* Iterate to termination: "repeat steps 1-3 till finding the best solution or the problem is
 * proved to be unbounded" (§III Iterate/Finalization), with the iteration cap and
 * the status precedence of DESIGN.md reading c12.  *st (may be NULL)
 * receives OPTIMAL, UNBOUNDED, INFEASIBLE (Phase I) or ITERATION_LIMIT.  Same errors as
 * simplex_iterate; on several ranks every rank must call it (collective). */
simplex_err simplex_solve(simplex_t* h, simplex_status* st);

/* Read the solution off the current tableau (the objective is Table I's Z entry,
 * PAPER.md:79-84): x: n values (x_j = rhs of the row where j is basic, else 0), y: m dual values
 * (y_i = T[0][n+i-1], the slacks' reduced costs), objective = T[0][W-1], pivots done, status.
 * Every output pointer may be NULL; x / y are caller-owned buffers of n / m doubles in host or
 * device memory.  Valid in any state (reports the current basis).  Errors: ARG (NULL handle),
 * STATE (faulted handle), CUDA.  Multi-GPU: collective (y is assembled from every rank). */
simplex_err simplex_get_solution(simplex_t* h, double* x, double* y, double* objective,
                                 int64_t* pivots, simplex_status* st);

/* One whole LP of the handle's shape in one call: exactly simplex_reset(h, A, b, c), then
 * simplex_solve(h), then simplex_get_solution(h, x, y, objective, pivots, st) — the same
 * arguments (A, b, c, x, y: host or device memory, caller-owned), results, trace and errors.
 * On the latency path (stats.path = 1: a tableau that fits one CTA's shared memory) it is ONE
 * kernel launch that builds Table I from A, b, c, runs Steps 1-3 to termination
 * and extracts x, y and the objective, with ONE host
 * synchronisation instead of three: on small LPs the fixed costs around the pivots dominate
 * (PAPER.md:161, 290).  Otherwise the three calls run in turn.  Errors: those of the three calls
 * (ARG, NONFINITE, STATE, CUDA, NCCL); a rejected input leaves the handle as a rejected reset. */
simplex_err simplex_solve_lp(simplex_t* h, const double* A, const double* b, const double* c, double* x,
                             double* y, double* objective, int64_t* pivots, simplex_status* st);

/* The pivot trace (SPEC.md:195-198 PivotRecord; reading c19): copy up to cap (k, r) records —
 * k the 0-based entering column, r the 1-based leaving row, in pivot order — into the caller's
 * int32 buffers k[], r[] (host or device, cap entries each); *len = records copied.  Recorded only
 * with options.record_trace = 1.  Errors: ARG (NULL handle, NULL buffer with cap > 0), STATE, CUDA. */
simplex_err simplex_get_trace(simplex_t* h, int32_t* k, int32_t* r, int64_t cap, int64_t* len);

/* Copy this rank's slab of the current tableau, logical columns only
 * (stats.local_cols per row), row-major with pitch ld_out >= local_cols doubles.
 * Column j of the slab is global column col_offset + j; the last slab column is the
 * rhs (W-1).  Debug/parity use. */
simplex_err simplex_get_tableau(simplex_t* h, double* T_out, int64_t ld_out);

/* Order-independent 64-bit digest of the whole logical tableau (all ranks; the rhs
 * column counted once): sum over elements e = i*W + j of
 *   mix64(bits(T[i][j]) ^ (e * 0x9E3779B97F4A7C15 + 0xD1B54A32D192ED03)), -0.0 as +0.0,
 * with mix64 the SplitMix64 finalizer.  Multi-GPU: collective. */
simplex_err simplex_tableau_hash(simplex_t* h, uint64_t* hash);

/* Counters and timings of the handle (see simplex_stats). */
simplex_err simplex_get_stats(simplex_t* h, simplex_stats* s);

/* Free everything the handle owns: device memory, streams, CUDA graphs, the NCCL communicator
 * and peer mappings (the ownership rule of SURVEY.md §8(b)).  NULL-safe; valid on a faulted
 * handle; always returns SIMPLEX_OK.  Multi-GPU: every rank destroys its own handle. */
simplex_err simplex_destroy(simplex_t* h);

/* Text of the last error on this thread ("" if none). */
const char* simplex_last_error(void);

/* Write a fresh 128-byte ncclUniqueId to out128 (rank 0 calls it; the caller
 * broadcasts the bytes to the other ranks, e.g. with torch.distributed). */
simplex_err simplex_nccl_unique_id(void* out128);

/* Column partition of the n+m non-rhs columns over nparts parts ("the
 * columns of the simplex tableau are equivalently spread among all the resources";
 * SPEC.md:156-164): contiguous ranges of width floor(total/nparts) or +1, the
 * remainder going to the lowest parts.  Part p gets [*c0, *c0 + *width).  Pure host
 * function (no GPU needed); the handle uses it for its slab.  ARG on bad input. */
simplex_err simplex_partition(int64_t total_cols, int64_t nparts, int64_t part, int64_t* c0,
                              int64_t* width);

/* Library version string. */
const char* simplex_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LIBSIMPLEX_H */
