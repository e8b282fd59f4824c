/*
 * oracle/simplex_oracle.c — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this code.  The product path
 * (paper_2211_10979_b200/, libsimplex) never links, calls or includes it, and
 * this file includes nothing from there: the two share no code.
 *
 * What it computes: the standard full-tableau simplex method of PAPER.md
 * §III (lines 73-96, Table I at lines 77-84), written plainly, in the paper's
 * order and notation, single-threaded, IEEE binary64, one step per function:
 *
 *   or_build    Initialization Step + Table I layout
 *   or_price    Step 1, entering variable (§IV Step 1)
 *   or_ratio    Step 2, minimum ratio test
 *   or_pivot    Step 3, pivoting
 *   or_iterate  the Iterate loop on a built tableau, resumable
 *   or_solve    Iterate/Finalization
 *   or_extract  read x, y, objective off the final tableau
 *   or_price_bland / or_ratio_bland / or_solve_rule  Bland's rule
 *   or_solve_2phase  Phase I + Phase II for b with negative entries (NEXT #2)
 *   or_brute_force  vertex enumeration (independent check)
 *
 * Every point where the paper is silent takes the reading in SURVEY.md §8(c)
 * (c1..c19), restated in DESIGN.md "Readings":
 *   c1/c2/c3  Dantzig: most negative T[0][j] < -tol_opt, lowest j on exact ties
 *   c4/c5/c6  ratio over rows with T[i][k] > tol_piv, lowest row i on exact ties,
 *             UNBOUNDED iff no row qualifies
 *   c8        prow_j = T[r][j] / p (IEEE division), then
 *             T[i][j] = fma(-T[i][k], prow_j, T[i][j]) for i != r; T[r][j] = prow_j
 *   c10       the Z column of Table I is omitted (constant unit column)
 *   c11       slack basis; b_i < 0 rejected
 *   c12       per iteration: price (-> OPTIMAL), ratio (-> UNBOUNDED), then
 *             the cap check (-> ITERATION_LIMIT), then pivot
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (no -ffast-math: the fma and
 * the division must be exactly the IEEE operations written here).  The same
 * source built with -fopenmp (liboracle_omp.so) splits only or_pivot's row loop
 * across threads — every element still gets the same single fma — and is used
 * only by scripts/make_golden.py for the configs a single thread cannot finish
 * (SURVEY.md §8(d) "Oracle baseline"); tests/test_oracle_omp.py proves it bitwise
 * equal to the single-thread build.
 *
 * Pins (tests/test_oracle_*.py): SPEC worked examples, textbook LPs,
 * brute-force vertex enumeration, Klee-Minty (2^n - 1 pivots, optimum 5^n),
 * diagonal LPs (trace = columns sorted by (-c_j, j)), planted optima, strong
 * duality, bitwise unit-basis invariants, and the SplitMix64 golden table of
 * SURVEY.md §8(c) computed by an independent scratch solver.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_RUNNING (-1)
#define OR_OPTIMAL 0
#define OR_UNBOUNDED 2
#define OR_INFEASIBLE 3
#define OR_ITERATION_LIMIT 4

#define OR_OK 0
#define OR_E_ARG (-1)
#define OR_E_NONFINITE (-2)
#define OR_E_NEG_RHS (-3)
#define OR_E_OOM (-4)

/* Table I: row 0 = [-c | 0 ... 0 | 0], rows i = [a_i | e_i | b_i].
 * T is (m+1) x W row-major with W = n + m + 1; the rhs ("cv") is
 * column W-1.  basis[i-1] = n+i-1 (slack x_{n+i} labels row i). */
int or_build(int64_t m, int64_t n, const double *A, const double *b, const double *c,
             double *T, int64_t *basis)
{
    if (m < 1 || n < 1 || !A || !b || !c || !T) return OR_E_ARG;
    for (int64_t i = 0; i < m * n; i++) if (!isfinite(A[i])) return OR_E_NONFINITE;
    for (int64_t i = 0; i < m; i++) if (!isfinite(b[i])) return OR_E_NONFINITE;
    for (int64_t j = 0; j < n; j++) if (!isfinite(c[j])) return OR_E_NONFINITE;
    for (int64_t i = 0; i < m; i++) if (b[i] < 0.0) return OR_E_NEG_RHS;
    const int64_t W = n + m + 1;
    memset(T, 0, sizeof(double) * (size_t)((m + 1) * W));
    for (int64_t j = 0; j < n; j++) T[j] = -c[j];
    for (int64_t i = 1; i <= m; i++) {
        double *row = T + i * W;
        for (int64_t j = 0; j < n; j++) row[j] = A[(i - 1) * n + j];
        row[n + i - 1] = 1.0;
        row[W - 1] = b[i - 1];
        if (basis) basis[i - 1] = n + i - 1;
    }
    return OR_OK;
}

/* Step 1: "the column with the larger negative coefficient of the
 * objective function".  Scan j = 0 .. len-1 ascending; strict < keeps the lowest
 * index on exact ties (c2).  Returns k, or -1 when no T[0][j] < -tol_opt (optimal). */
int64_t or_price(const double *row0, int64_t len, double tol_opt, double *v_out)
{
    int64_t k = -1;
    double v = -tol_opt;
    for (int64_t j = 0; j < len; j++) {
        if (row0[j] < v) { v = row0[j]; k = j; }
    }
    if (v_out) *v_out = v;
    return k;
}

/* Step 2: "run the minimum ratio test on the items of the winning
 * column and conclude to the row having the minimum ratio".  Rows i = 1..m with
 * T[i][k] > tol_piv; q_i = T[i][W-1] / T[i][k]; strict < keeps the lowest row on
 * exact ties (c4).  Returns r in [1, m], or -1 when no row qualifies (unbounded). */
int64_t or_ratio(int64_t m, int64_t W, const double *T, int64_t k, double tol_piv,
                 double *q_out)
{
    int64_t r = -1;
    double best = INFINITY;
    for (int64_t i = 1; i <= m; i++) {
        const double a = T[i * W + k];
        if (a > tol_piv) {
            const double q = T[i * W + (W - 1)] / a;
            if (r == -1 || q < best) { best = q; r = i; }
        }
    }
    if (q_out) *q_out = best;
    return r;
}

/* Bland's rule (NEXT #3 of SURVEY.md §8(f); "Bland's rule: enter the
 * lowest-index negative reduced cost (anti-cycling)").  Entering: the FIRST j (ascending)
 * with T[0][j] < -tol_opt. */
int64_t or_price_bland(const double *row0, int64_t len, double tol_opt)
{
    for (int64_t j = 0; j < len; j++)
        if (row0[j] < -tol_opt) return j;
    return -1;
}

/* Bland's leaving rule (Bland 1977): among rows with the minimum ratio (exact ties), the
 * row whose BASIC VARIABLE has the smallest index (basis[i-1]); reading c4 does not apply
 * under this rule.  Same eligibility (c5) and division (c8) as or_ratio. */
int64_t or_ratio_bland(int64_t m, int64_t W, const double *T, int64_t k, double tol_piv,
                       const int64_t *basis, double *q_out)
{
    int64_t r = -1;
    double best = INFINITY;
    for (int64_t i = 1; i <= m; i++) {
        const double a = T[i * W + k];
        if (a > tol_piv) {
            const double q = T[i * W + (W - 1)] / a;
            if (r == -1 || q < best || (q == best && basis[i - 1] < basis[r - 1])) { best = q; r = i; }
        }
    }
    if (q_out) *q_out = best;
    return r;
}

/* Step 3: "form the new simplex tableau ... by applying pivoting in
 * the rows of the previous tableau, using the new pivot row".  Gauss-Jordan with
 * the arithmetic of reading c8. col[] snapshots column k before it is overwritten;
 * prow[] is the normalized pivot row.  Scratch buffers are the caller's. */
void or_pivot(int64_t m, int64_t W, double *T, int64_t r, int64_t k, double *col, double *prow)
{
    const double p = T[r * W + k];
    for (int64_t i = 0; i <= m; i++) col[i] = T[i * W + k];
    for (int64_t j = 0; j < W; j++) prow[j] = T[r * W + j] / p;
    /* Rows are independent (each element gets exactly one fma with operands fixed
     * before the loop), so the optional -fopenmp build (liboracle_omp.so, used only
     * by scripts/make_golden.py for the largest configs, SURVEY.md §8(d) "Oracle
     * baseline") splits this loop across threads without changing a single bit;
     * tests/test_oracle_omp.py proves it.  The default build ignores the pragma. */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i <= m; i++) {
        if (i == r) continue;
        double *row = T + i * W;
        const double a = -col[i];
        for (int64_t j = 0; j < W; j++) row[j] = fma(a, prow[j], row[j]);
    }
    memcpy(T + r * W, prow, sizeof(double) * (size_t)W);
}

/* x_j = T[i][W-1] if basis[i-1] = j < n else 0;  y_i = T[0][n+i-1] (reduced costs
 * of the slacks = dual values);  objective = T[0][W-1] (Z in Table I). */
void or_extract(int64_t m, int64_t n, const double *T, const int64_t *basis,
                double *x, double *y, double *obj)
{
    const int64_t W = n + m + 1;
    if (x) {
        for (int64_t j = 0; j < n; j++) x[j] = 0.0;
        for (int64_t i = 1; i <= m; i++)
            if (basis[i - 1] < n) x[basis[i - 1]] = T[i * W + W - 1];
    }
    if (y) for (int64_t i = 1; i <= m; i++) y[i - 1] = T[n + i - 1];
    if (obj) *obj = T[W - 1];
}

/* Iterate/Finalization: repeat Steps 1-3 "till finding the best
 * solution or the problem is proved to be unbounded", with the iteration cap and
 * status precedence of reading c12.  stop_after >= 0 returns OR_RUNNING once that
 * many pivots are done (prefix runs).  T_out (optional, (m+1)*W) receives the final
 * tableau; trace_k/trace_r (optional, capacity trace_cap) receive (k, r) per pivot
 * (k 0-based column, r 1-based row). */
/* The Iterate loop on an already built (m+1) x W tableau T with basis:
 * repeat Step 1 (-> OPTIMAL), Step 2 (-> UNBOUNDED), the cap check (-> ITERATION_LIMIT,
 * reading c12), Step 3.  *it is the pivot counter: it enters with the pivots already
 * done (0 for a fresh tableau) and leaves with the total; the cap applies to the total.
 * stop_at >= 0 returns OR_RUNNING when the total reaches stop_at (prefix and chunked
 * runs: resuming with the same T, basis and *it continues the identical sequence).
 * trace_k/trace_r[t] receive the (k, r) of the t-th pivot OF THIS CALL (t < trace_cap).
 * col/prow are caller scratch of m+1 and W doubles.  rule 0: Dantzig (readings c1-c4);
 * rule 1: Bland (or_price_bland / or_ratio_bland). */
int or_iterate(int64_t m, int64_t n, double *T, int64_t *basis, double tol_opt, double tol_piv,
               int64_t cap, int64_t stop_at, int rule, int32_t *trace_k, int32_t *trace_r,
               int64_t trace_cap, int64_t *it, double *col, double *prow)
{
    const int64_t W = n + m + 1, it0 = *it;
    for (;;) {
        if (stop_at >= 0 && *it == stop_at) return OR_RUNNING;
        const int64_t k = rule == 1 ? or_price_bland(T, n + m, tol_opt)  /* Step 1 */
                                    : or_price(T, n + m, tol_opt, NULL);
        if (k < 0) return OR_OPTIMAL;
        const int64_t r = rule == 1 ? or_ratio_bland(m, W, T, k, tol_piv, basis, NULL)  /* Step 2 */
                                    : or_ratio(m, W, T, k, tol_piv, NULL);
        if (r < 0) return OR_UNBOUNDED;
        if (*it == cap) return OR_ITERATION_LIMIT;
        or_pivot(m, W, T, r, k, col, prow);                                /* Step 3 */
        basis[r - 1] = k;
        const int64_t t = *it - it0;
        if (trace_k && t < trace_cap) { trace_k[t] = (int32_t)k; trace_r[t] = (int32_t)r; }
        (*it)++;
    }
}

/* rule 0: Dantzig (readings c1-c4); rule 1: Bland (or_price_bland / or_ratio_bland). */
int or_solve_rule(int64_t m, int64_t n, const double *A, const double *b, const double *c,
                  double tol_opt, double tol_piv, int64_t max_pivots, int64_t stop_after, int rule,
                  int32_t *trace_k, int32_t *trace_r, int64_t trace_cap,
                  double *x, double *y, double *obj, int64_t *pivots_out, int *status_out,
                  double *T_out, int64_t *basis_out)
{
    const int64_t W = n + m + 1;
    double *T = T_out ? T_out : (double *)malloc(sizeof(double) * (size_t)((m + 1) * W));
    int64_t *basis = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
    double *col = (double *)malloc(sizeof(double) * (size_t)(m + 1));
    double *prow = (double *)malloc(sizeof(double) * (size_t)W);
    if (!T || !basis || !col || !prow) {
        if (!T_out) free(T);
        free(basis); free(col); free(prow);
        return OR_E_OOM;
    }
    int err = or_build(m, n, A, b, c, T, basis);
    if (err != OR_OK) {
        if (!T_out) free(T);
        free(basis); free(col); free(prow);
        return err;
    }
    const int64_t cap = max_pivots > 0 ? max_pivots : 20 * (m + n);
    int64_t it = 0;
    const int status = or_iterate(m, n, T, basis, tol_opt, tol_piv, cap, stop_after, rule,
                                  trace_k, trace_r, trace_cap, &it, col, prow);
    or_extract(m, n, T, basis, x, y, obj);
    if (basis_out) memcpy(basis_out, basis, sizeof(int64_t) * (size_t)m);
    if (pivots_out) *pivots_out = it;
    if (status_out) *status_out = status;
    if (!T_out) free(T);
    free(basis); free(col); free(prow);
    return OR_OK;
}

int or_solve(int64_t m, int64_t n, const double *A, const double *b, const double *c,
             double tol_opt, double tol_piv, int64_t max_pivots, int64_t stop_after,
             int32_t *trace_k, int32_t *trace_r, int64_t trace_cap,
             double *x, double *y, double *obj, int64_t *pivots_out, int *status_out,
             double *T_out, int64_t *basis_out)
{
    return or_solve_rule(m, n, A, b, c, tol_opt, tol_piv, max_pivots, stop_after, 0, trace_k, trace_r,
                         trace_cap, x, y, obj, pivots_out, status_out, T_out, basis_out);
}

/* ---- Phase I ("start having as a basis a feasible
 * basic solution"; SPEC.md:70-78 phase_one) -------------------------------------------------
 * Two-phase method, written step by step (readings p1-p6 in DESIGN.md):
 *  p1 layout: W2 = n + m + a + 1 columns: structural, slacks, one artificial per row with
 *     b_i < 0 (in ascending row order), rhs.  A row with b_i < 0 is negated exactly
 *     (-a_i, -e_i, -b_i) and gets +1 in its artificial column; its artificial is basic,
 *     every other row keeps its slack.
 *  p2 Phase I objective: maximize -(sum of artificials): row 0 = +1 on the artificial
 *     columns, then each artificial-basic row is subtracted from row 0 in ascending row
 *     order (row0[j] = fma(-1, T[i][j], row0[j])), which zeroes the basic columns.
 *  p3 Phase I runs the method itself (Steps 1-3, same rule, same cap counter) over all
 *     non-rhs columns.  Infeasible iff its optimum T[0][W2-1] < -1e-7.
 *  p4 drive-out: for each row i ascending whose basic variable is artificial, pivot on the
 *     first column j < n+m with |T[i][j]| > tol_piv (Gauss-Jordan of Step 3, counted and
 *     traced as a pivot); a row with none is redundant and keeps its artificial at zero.
 *  p5 Phase II objective: row 0 = -c on the structural columns, 0 elsewhere; for each row i
 *     ascending whose basic variable j is structural, row0[col] = fma(c_j, T[i][col],
 *     row0[col]) (prices the basis out).  Artificial columns never enter again (pricing
 *     over j < n+m only).
 *  p6 Phase II continues with the same rule, tolerances and cap; extraction as or_extract
 *     (y_i = T[0][n+i-1] holds for negated rows too: their slack column is -e_i). */
int or_solve_2phase(int64_t m, int64_t n, const double *A, const double *b, const double *c,
                    double tol_opt, double tol_piv, int64_t max_pivots, int rule,
                    int32_t *trace_k, int32_t *trace_r, int64_t trace_cap,
                    double *x, double *y, double *obj, int64_t *pivots_out, int *status_out,
                    int64_t *phase1_pivots_out)
{
    if (m < 1 || n < 1) return OR_E_ARG;
    for (int64_t i = 0; i < m * n; i++) if (!isfinite(A[i])) return OR_E_NONFINITE;
    for (int64_t i = 0; i < m; i++) if (!isfinite(b[i])) return OR_E_NONFINITE;
    for (int64_t j = 0; j < n; j++) if (!isfinite(c[j])) return OR_E_NONFINITE;
    int64_t a = 0;
    for (int64_t i = 0; i < m; i++) if (b[i] < 0.0) a++;
    const int64_t W = n + m + a + 1, nm = n + m;
    double *T = (double *)calloc((size_t)((m + 1) * W), sizeof(double));
    int64_t *basis = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
    double *col = (double *)malloc(sizeof(double) * (size_t)(m + 1));
    double *prow = (double *)malloc(sizeof(double) * (size_t)W);
    if (!T || !basis || !col || !prow) { free(T); free(basis); free(col); free(prow); return OR_E_OOM; }
    /* p1 */
    int64_t art = 0;
    for (int64_t i = 1; i <= m; i++) {
        double *row = T + i * W;
        const int neg = b[i - 1] < 0.0;
        for (int64_t j = 0; j < n; j++) row[j] = neg ? -A[(i - 1) * n + j] : A[(i - 1) * n + j];
        row[n + i - 1] = neg ? -1.0 : 1.0;
        row[W - 1] = neg ? -b[i - 1] : b[i - 1];
        if (neg) { row[nm + art] = 1.0; basis[i - 1] = nm + art; art++; }
        else basis[i - 1] = n + i - 1;
    }
    /* p2 */
    for (int64_t q = 0; q < a; q++) T[nm + q] = 1.0;
    for (int64_t i = 1; i <= m; i++)
        if (basis[i - 1] >= nm)
            for (int64_t j = 0; j < W; j++) T[j] = fma(-1.0, T[i * W + j], T[j]);
    const int64_t cap = max_pivots > 0 ? max_pivots : 20 * (m + n);
    int64_t it = 0;
    int status = OR_RUNNING;
    int64_t price_len = W - 1;                                   /* Phase I: every column */
    for (int phase = 1; phase <= 2 && status == OR_RUNNING; phase++) {
        for (;;) {                                               /* p3 / p6: Steps 1-3 */
            const int64_t k = rule == 1 ? or_price_bland(T, price_len, tol_opt)
                                        : or_price(T, price_len, tol_opt, NULL);
            if (k < 0) break;
            const int64_t r = rule == 1 ? or_ratio_bland(m, W, T, k, tol_piv, basis, NULL)
                                        : or_ratio(m, W, T, k, tol_piv, NULL);
            if (r < 0) { status = OR_UNBOUNDED; break; }
            if (it == cap) { status = OR_ITERATION_LIMIT; break; }
            or_pivot(m, W, T, r, k, col, prow);
            basis[r - 1] = k;
            if (trace_k && it < trace_cap) { trace_k[it] = (int32_t)k; trace_r[it] = (int32_t)r; }
            it++;
        }
        if (status != OR_RUNNING) break;
        if (phase == 2) { status = OR_OPTIMAL; break; }
        if (phase1_pivots_out) *phase1_pivots_out = it;
        if (T[W - 1] < -1e-7) { status = OR_INFEASIBLE; break; } /* p3 */
        for (int64_t i = 1; i <= m; i++) {                       /* p4 */
            if (basis[i - 1] < nm) continue;
            int64_t j = -1;
            for (int64_t q = 0; q < nm; q++) if (fabs(T[i * W + q]) > tol_piv) { j = q; break; }
            if (j < 0) continue;
            if (it == cap) { status = OR_ITERATION_LIMIT; break; }
            or_pivot(m, W, T, i, j, col, prow);
            basis[i - 1] = j;
            if (trace_k && it < trace_cap) { trace_k[it] = (int32_t)j; trace_r[it] = (int32_t)i; }
            it++;
        }
        if (status != OR_RUNNING) break;
        for (int64_t j = 0; j < W; j++) T[j] = 0.0;              /* p5 */
        for (int64_t j = 0; j < n; j++) T[j] = -c[j];
        for (int64_t i = 1; i <= m; i++) {
            const int64_t jb = basis[i - 1];
            if (jb < n)
                for (int64_t q = 0; q < W; q++) T[q] = fma(c[jb], T[i * W + q], T[q]);
        }
        price_len = nm;
    }
    /* extraction (or_extract with the W2 layout) */
    if (x) {
        for (int64_t j = 0; j < n; j++) x[j] = 0.0;
        for (int64_t i = 1; i <= m; i++) if (basis[i - 1] < n) x[basis[i - 1]] = T[i * W + W - 1];
    }
    if (y) for (int64_t i = 1; i <= m; i++) y[i - 1] = T[n + i - 1];
    if (obj) *obj = T[W - 1];
    if (pivots_out) *pivots_out = it;
    if (status_out) *status_out = status;
    free(T); free(basis); free(col); free(prow);
    return OR_OK;
}

/* ---- independent check: brute-force vertex enumeration ----
 * Constraints: rows of [A; -I] with rhs [b; 0].  Every n-subset of the m+n rows
 * is solved as an n x n system by Gaussian elimination with partial pivoting in
 * long double; singular systems (|pivot| < 1e-12) are skipped; points feasible
 * within feas_tol are kept; the maximum of c^T x wins.  Feasible for m+n <= ~16.
 * Returns 1 and fills (obj, x) if some feasible vertex exists, else 0. */
static int solve_square(int64_t n, long double *M, long double *rhs, long double *x)
{
    for (int64_t col = 0; col < n; col++) {
        int64_t piv = col;
        for (int64_t i = col + 1; i < n; i++)
            if (fabsl(M[i * n + col]) > fabsl(M[piv * n + col])) piv = i;
        if (fabsl(M[piv * n + col]) < 1e-12L) return 0;
        if (piv != col) {
            for (int64_t j = 0; j < n; j++) {
                long double t = M[col * n + j]; M[col * n + j] = M[piv * n + j]; M[piv * n + j] = t;
            }
            long double t = rhs[col]; rhs[col] = rhs[piv]; rhs[piv] = t;
        }
        for (int64_t i = col + 1; i < n; i++) {
            long double f = M[i * n + col] / M[col * n + col];
            for (int64_t j = col; j < n; j++) M[i * n + j] -= f * M[col * n + j];
            rhs[i] -= f * rhs[col];
        }
    }
    for (int64_t i = n - 1; i >= 0; i--) {
        long double s = rhs[i];
        for (int64_t j = i + 1; j < n; j++) s -= M[i * n + j] * x[j];
        x[i] = s / M[i * n + i];
    }
    return 1;
}

int or_brute_force(int64_t m, int64_t n, const double *A, const double *b, const double *c,
                   double feas_tol, double *obj_out, double *x_out)
{
    const int64_t R = m + n;
    if (R > 24) return -1;
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    long double *M = (long double *)malloc(sizeof(long double) * (size_t)(n * n));
    long double *rhs = (long double *)malloc(sizeof(long double) * (size_t)n);
    long double *x = (long double *)malloc(sizeof(long double) * (size_t)n);
    int found = 0;
    long double best = 0.0L;
    for (int64_t j = 0; j < n; j++) idx[j] = j;
    for (;;) {
        for (int64_t a = 0; a < n; a++) {
            const int64_t row = idx[a];
            for (int64_t j = 0; j < n; j++)
                M[a * n + j] = row < m ? (long double)A[row * n + j] : (row - m == j ? -1.0L : 0.0L);
            rhs[a] = row < m ? (long double)b[row] : 0.0L;
        }
        if (solve_square(n, M, rhs, x)) {
            int ok = 1;
            for (int64_t j = 0; j < n && ok; j++) if (x[j] < -(long double)feas_tol) ok = 0;
            for (int64_t i = 0; i < m && ok; i++) {
                long double s = 0.0L;
                for (int64_t j = 0; j < n; j++) s += (long double)A[i * n + j] * x[j];
                if (s > (long double)b[i] + (long double)feas_tol) ok = 0;
            }
            if (ok) {
                long double v = 0.0L;
                for (int64_t j = 0; j < n; j++) v += (long double)c[j] * x[j];
                if (!found || v > best) {
                    best = v; found = 1;
                    if (x_out) for (int64_t j = 0; j < n; j++) x_out[j] = (double)x[j];
                }
            }
        }
        /* next n-subset of {0..R-1} in lexicographic order */
        int64_t a = n - 1;
        while (a >= 0 && idx[a] == R - n + a) a--;
        if (a < 0) break;
        idx[a]++;
        for (int64_t t = a + 1; t < n; t++) idx[t] = idx[t - 1] + 1;
    }
    if (obj_out) *obj_out = (double)best;
    free(idx); free(M); free(rhs); free(x);
    return found;
}
