// kernels.cu — hand-written sm_100a kernels of the dense-tableau simplex hot path.
//
//   k_build    Table I in HBM + input validation            (row a0)
//   k_price0   Step 1 candidates of the initial row 0           (row a1)
//   k_pack     multi-GPU: local Step-1 winner + its column into the send buffer
//              ("the data of the winning column are sent")
//   k_select   Step 1 fold + Step 2 ratio test + column staging  (a1-a3, a5)
//   k_update   Step 3 pivot: fused row scale + rank-1 update,
//              with Step 1 of the NEXT iteration fused on row 0               (a4, a1)
//   k_flush    deferred write-back of the last normalized pivot row
//   k_extract  x, y, objective                                 (a6)
//   k_hash     order-independent tableau digest (debug / parity)
//
// Arithmetic is pinned to the oracle's (reading c8): prow_j = T[r][j] / p
// with IEEE division (__ddiv_rn), T[i][j] = fma(-T[i][k], prow_j, T[i][j]) with an
// explicit __fma_rn, q_i = T[i][W-1] / T[i][k] with __ddiv_rn.  With that pin the
// tableau equals the oracle's bit for bit after every pivot, for any tiling.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdlib>
#include <cuda_runtime.h>

#include "device.cuh"
#include "kernels.h"

namespace sx {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ Cand cand_none() { return Cand{__longlong_as_double(0x7ff0000000000000LL), LLONG_MAX}; }

__device__ __forceinline__ bool cand_less(const Cand& a, const Cand& b) {
  return a.v < b.v || (a.v == b.v && a.idx < b.idx);
}
__device__ __forceinline__ Cand cand_min(const Cand& a, const Cand& b) { return cand_less(b, a) ? b : a; }

// Step-1 candidate of column j with reduced cost v < -tol_opt: Dantzig keys on (v, j);
// Bland keys on j alone (value 0), so the argmin is the first eligible column.
__device__ __forceinline__ Cand price_cand(int rule, double v, long long j) { return Cand{rule ? 0.0 : v, j}; }

// Step-2 candidate of row i with ratio q: Dantzig ties -> lowest row (reading c4); Bland
// ties -> smallest basic-variable index (basis[i-1] in the high bits; row in the low 32).
__device__ __forceinline__ Cand ratio_cand(int rule, double q, long long i, int basic) {
  return Cand{q, rule ? (((long long)basic << 32) | i) : i};
}
__device__ __forceinline__ int cand_row(long long idx) { return (int)(idx & 0xffffffffLL); }

// Order-preserving map of a non-NaN double to an unsigned 64-bit key (IEEE order = unsigned
// order); -0 and +0 get the same key, as they compare equal (reading c16).
__device__ __forceinline__ unsigned long long ord_key(double v) {
  const long long b = __double_as_longlong(v == 0.0 ? 0.0 : v);
  return b < 0 ? ~(unsigned long long)b : ((unsigned long long)b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
  return __longlong_as_double((k >> 63) ? (long long)(k & 0x7fffffffffffffffull) : (long long)~k);
}

#ifndef SX_WARP_MIN_SHFL
// Warp-wide lexicographic argmin of (v, idx) on the 32-bit reduction unit: the 128-bit key
// (ord_key(v), idx) is reduced one 32-bit word at a time (redux.sync.min.u32), lanes that lost
// a word dropping out (they contribute 0xffffffff).  Equal to the pairwise cand_min fold for
// non-NaN values (c18); idx >= 0, so unsigned order is the signed order.  Every lane returns
// the result (v of an all-zero key comes back as +0).  Full warps only.
__device__ __forceinline__ Cand warp_min(Cand c) {
  const unsigned long long k = ord_key(c.v);
  const unsigned long long ix = (unsigned long long)c.idx;
  const unsigned int w0 = (unsigned int)(k >> 32), w1 = (unsigned int)k;
  const unsigned int w2 = (unsigned int)(ix >> 32), w3 = (unsigned int)ix;
  const unsigned int m0 = __reduce_min_sync(0xffffffffu, w0);
  bool e = w0 == m0;
  const unsigned int m1 = __reduce_min_sync(0xffffffffu, e ? w1 : 0xffffffffu);
  e = e && w1 == m1;
  const unsigned int m2 = __reduce_min_sync(0xffffffffu, e ? w2 : 0xffffffffu);
  e = e && w2 == m2;
  const unsigned int m3 = __reduce_min_sync(0xffffffffu, e ? w3 : 0xffffffffu);
  return Cand{ord_val(((unsigned long long)m0 << 32) | m1), (long long)(((unsigned long long)m2 << 32) | m3)};
}
#else
__device__ __forceinline__ Cand warp_min(Cand c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand t;
    t.v = __shfl_xor_sync(0xffffffffu, c.v, o);
    t.idx = __shfl_xor_sync(0xffffffffu, c.idx, o);
    c = cand_min(c, t);
  }
  return c;
}
#endif

// Block-wide lexicographic argmin; every thread returns the result.  Contains
// __syncthreads(): call from block-uniform control flow only.
__device__ __forceinline__ Cand block_min(Cand c) {
  __shared__ Cand sh[32];
  __shared__ Cand res;
  c = warp_min(c);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = c;
  __syncthreads();
  if (wid == 0) {
    Cand t = lane < (int)(blockDim.x >> 5) ? sh[lane] : cand_none();
    t = warp_min(t);
    if (lane == 0) res = t;
  }
  __syncthreads();
  Cand out = res;
  __syncthreads();
  return out;
}

// Programmatic dependent launch (PDL): let the next kernel of the pivot chain be
// scheduled while this one runs, and wait for the previous one's results.  Both are
// no-ops when the kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ Cand ldcg_cand(const Cand* p) {
  Cand c;
  c.v = __ldcg(&p->v);
  c.idx = __ldcg(&p->idx);
  return c;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 1-D TMA (cp.async.bulk) global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 policy "evict first" for the streamed tableau (the look-ahead's working set stays in L2)
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------------ a0: build
// Called after the host copied A's slab columns into rows 1..m (cudaMemcpy2DAsync)
// and c's slab columns into row 0.  Writes everything else of Table I and checks
// finiteness / b >= 0.  One thread per (row, column pair).
__global__ void __launch_bounds__(kThreads) k_build(SlabView s, const double* __restrict__ b, long long n) {
  // Phase I layout (reading p1, NEXT #2): a row with b_i < 0 (art_of_row >= 0) is negated
  // exactly and gets +1 in its artificial column n+m+art; row 0 is then the Phase I
  // objective (+1 on the artificials) instead of -c.
  const long long halfld = s.ld >> 1;
  const long long total = (long long)s.rows * halfld;
  const long long nm = n + (s.rows - 1);
  uint32_t err = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / halfld;
    const long long j0 = (e - i * halfld) * 2;
    double* row = s.T + i * s.ld;
    const int art = i >= 1 ? s.art_of_row[i - 1] : -1;
    const bool neg = art >= 0;
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      const long long j = j0 + d;
      const long long g = s.c0 + j;
      double v;
      if (j > s.w) {
        v = 0.0;                                   // padding
      } else if (j == s.w) {                       // rhs column ("cv")
        if (i == 0) {
          v = 0.0;
        } else {
          v = b[i - 1];
          if (!isfinite(v)) err |= kErrNonFinite;
          if ((v < 0.0) != neg) err |= kErrNegRhs;   // b's signs disagree with the row map
          if (neg) v = -v;
        }
      } else if (g < n) {                          // structural column: copied from A / c
        v = row[j];
        if (!isfinite(v)) err |= kErrNonFinite;
        if (i == 0) v = s.arts > 0 ? 0.0 : -v;     // row 0 stores -c
        else if (neg) v = -v;
      } else if (g < nm) {                         // slack column x_{g+1}: +-e_{g-n+1}
        v = (i >= 1 && g - n == i - 1) ? (neg ? -1.0 : 1.0) : 0.0;
      } else {                                     // artificial column g-nm
        v = (i == 0 || art == (int)(g - nm)) ? 1.0 : 0.0;
      }
      row[j] = v;
    }
  }
  if (err) atomicOr(&s.st->err, err);
}

__global__ void k_init_state(SlabView s, long long n, long long cap) {
  const int m = s.rows - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int art = s.art_of_row[i];               // slack basis; artificials
    s.basis[i] = art >= 0 ? (int)(n + m + art) : (int)(n + i);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    DevState* st = s.st;
    st->it = 0;
    st->cap = cap;
    st->stop_at = LLONG_MAX;
    st->p = 0.0;
    st->status = kRunning;
    st->go = 0;
    st->r = -1;
    st->k = -1;
    st->pend_r = -1;
    st->err = 0;
    st->ticket = 0;
    st->ticket2 = 0;
    st->sb[0] = 0;
    st->sb[1] = 0;
    st->pass_t0 = ~0ull;
    st->pass_t1 = 0ull;
    st->pass_done = 0u;
    st->pass_n = 0;
    st->pass_ns = 0.0;
    st->phase = s.arts > 0 ? 1 : 2;
    st->drive_next = 0;
    st->pw = s.w;                                  // Phase I prices every non-rhs column
  }
}

// Phase I objective (reading p2): subtract every artificial-basic row from row 0, in
// ascending row order, one FMA per step (thread per column: the oracle's rounding order).
__global__ void __launch_bounds__(kThreads) k_phase1_row0(SlabView s) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= s.ld) return;
  double acc = s.T[j];
  for (int q = 0; q < s.arts; ++q) acc = __fma_rn(-1.0, s.T[(long long)s.neg_rows[q] * s.ld + j], acc);
  s.T[j] = acc;
}

// Phase II objective (reading p5): row 0 = -c on the structural columns, 0 elsewhere, then
// for each row i ascending whose basic variable j is structural: row0 = fma(c_j, row_i, row0).
__global__ void __launch_bounds__(kThreads) k_phase2_row0(SlabView s, long long n) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= s.ld) return;
  const long long g = s.c0 + j;
  double acc = (j < s.w && g < n) ? -s.cvec[g] : 0.0;
  for (int i = 1; i < s.rows; ++i) {
    const int jb = s.basis[i - 1];
    if (jb < n) acc = __fma_rn(s.cvec[jb], s.T[(long long)i * s.ld + j], acc);
  }
  s.T[j] = acc;
  if (j == 0) {
    s.st->phase = 2;
    const long long nm = n + s.rows - 1 - s.c0;   // this part's columns below n+m: no artificials
    s.st->pw = (int)(nm < 0 ? 0 : nm < s.w ? nm : s.w);
  }
}

// Host-chosen pivot (Phase I drive-out, reading p4): stage column k (global index; `col` = that
// column gathered from its owner part, or NULL: the local column k of a single part), set the loop
// state so k_update applies pivot (r, k) exactly like a selected one (trace, basis, counter).
__global__ void __launch_bounds__(kThreads) k_force(SlabView s, int r, int k, const double* __restrict__ col) {
  DevState* st = s.st;
  for (int i = threadIdx.x; i < s.rows; i += blockDim.x) s.col[i] = col ? col[i] : s.T[(long long)i * s.ld + k];
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long it = st->it;
    st->r = r;
    st->k = k;
    st->p = s.col[r];
    st->go = 1;
    st->pend_r = r;
    s.basis[r - 1] = k;
    if (it < s.trace_cap) {
      s.trace_k[it] = k;
      s.trace_r[it] = r;
    }
    st->it = it + 1;
  }
}

// ---- Phase I drive-out on the device (reading p4): for each listed row i (rows whose basic
// variable is still artificial when Phase I ends, ascending; list index q), pivot on the FIRST
// column j < n+m with |T[i][j]| > tol_piv over all parts; a row with none is redundant (its
// artificial stays basic at zero).  Per row, with no host round trip:
//   k_drive_find   each part: its first eligible global column, or LLONG_MAX      -> fj[part]
//   k_drive_pick   this rank's parts: the minimum (ascending columns = first)        -> fjmin
//   (ranks > 1: ncclAllReduce(min) of fjmin)
//   k_drive_col    the owner part stages its column j in xcol[1..m+1], xcol[0] = 1 (flag)
//   (ranks > 1: ncclAllGather of xcol: every rank then holds the owner's exact bits)
//   k_drive_force  every part: the loop state for pivot (i, j) — or none (redundant row / cap /
//                  stop_at / not this row's turn) — then k_update applies it and k_flush writes it.
// DevState.drive_next counts the listed rows already handled, so a drive-out stopped by stop_at
// (simplex_iterate) resumes at the same row on the next call.
__global__ void __launch_bounds__(1024) k_drive_find(SlabView s, int i, long long nm, double tol, long long* fj) {
  __shared__ long long sh[32];
  const long long lim = nm - s.c0 < s.w ? nm - s.c0 : s.w;     // local columns below n+m
  const double* row = s.T + (long long)i * s.ld;
  long long best = LLONG_MAX;
  for (long long j = threadIdx.x; j < lim; j += blockDim.x)
    if (fabs(row[j]) > tol) {
      best = s.c0 + j;
      break;                                       // ascending per thread: its first is its min
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t < best ? t : best;
  }
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    long long v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : LLONG_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const long long t = __shfl_xor_sync(0xffffffffu, v, o);
      v = t < v ? t : v;
    }
    if (threadIdx.x == 0) *fj = v;
  }
}

__global__ void k_drive_pick(const long long* fj, int nparts, long long* fjmin) {
  long long v = LLONG_MAX;
  for (int p = 0; p < nparts; ++p) v = fj[p] < v ? fj[p] : v;
  *fjmin = v;
}

// xcol = [flag, T[0][j], ..., T[m][j]] staged by the part owning global column j (flag 1.0)
__global__ void __launch_bounds__(kThreads) k_drive_col(SlabView s, const long long* fjmin, double* xcol) {
  const long long j = *fjmin;
  if (j == LLONG_MAX || j < s.c0 || j >= s.c0 + s.w) return;
  const long long jl = j - s.c0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.rows; i += gridDim.x * blockDim.x)
    xcol[1 + i] = s.T[(long long)i * s.ld + jl];
  if (blockIdx.x == 0 && threadIdx.x == 0) xcol[0] = 1.0;
}

// xcols: nsrc staged buffers of stride xs doubles (one per rank after the allgather, or the
// rank's own); the one with flag 1 holds column j.  xcols == NULL: one part, column j is local.
__global__ void __launch_bounds__(kThreads) k_drive_force(SlabView s, int i, int q, const long long* fjmin,
                                                          const double* xcols, int nsrc, long long xs) {
  DevState* st = s.st;
  __shared__ int sh_go;
  __shared__ long long sh_j;
  if (threadIdx.x == 0) {
    int go = 0;
    const long long j = *fjmin;
    st->go = 0;
    if (st->status == kRunning && st->drive_next == q) {
      if (j == LLONG_MAX) {
        st->drive_next = q + 1;                    // redundant row: no pivot
      } else if (st->it >= st->cap) {
        st->status = kIterLimit;
      } else if (st->it < st->stop_at) {
        go = 1;
      }
    }
    sh_go = go;
    sh_j = j;
  }
  __syncthreads();
  if (!sh_go) return;
  const long long j = sh_j;
  const double* src = nullptr;
  if (xcols) {
    for (int r = 0; r < nsrc; ++r)
      if (xcols[(long long)r * xs] == 1.0) src = xcols + (long long)r * xs + 1;
  }
  for (int t = threadIdx.x; t < s.rows; t += blockDim.x)
    s.col[t] = src ? src[t] : s.T[(long long)t * s.ld + (j - s.c0)];
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long it = st->it;
    st->r = i;
    st->k = (int)j;
    st->p = s.col[i];
    st->go = 1;
    st->pend_r = i;
    s.basis[i - 1] = (int)j;
    if (it < s.trace_cap) {
      s.trace_k[it] = (int)j;
      s.trace_r[it] = i;
    }
    st->it = it + 1;
    st->drive_next = q + 1;
  }
}

__global__ void k_set_status(DevState* st, int status) { st->status = status; }

// ------------------------------------------------------------------ a1: initial pricing
// Row 0 is split into warp slots of 32 double2 (64 columns); slot w holds the argmin of
// T[0][j] over its columns j < w_local with T[0][j] < -tol_opt (reading c3).  k_update
// rewrites the same slots for the new row 0 of every pivot.
__global__ void __launch_bounds__(kThreads) k_price0(SlabView s, double tol_opt) {
  const long long half = s.ld >> 1;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if ((t & ~31LL) >= half) return;                 // warp-uniform
  Cand best = cand_none();
  if (t < half) {
    const long long j = 2 * t;
    const double2 v = *reinterpret_cast<const double2*>(s.T + j);
    const int pw = s.st->pw;
    if (j < pw && v.x < -tol_opt) best = price_cand(s.rule, v.x, s.c0 + j);
    if (j + 1 < pw && v.y < -tol_opt) best = cand_min(best, price_cand(s.rule, v.y, s.c0 + j + 1));
  }
  best = warp_min(best);
  if ((threadIdx.x & 31) == 0) s.price[t >> 5] = best;
}

// ------------------------------------------------------------------ multi-GPU: pack
// Fold this slab's pricing candidates into (v, k); write header + column k (with the
// deferred pivot row taken from rownorm) into send = [v, k bits, col[0..m]].
__global__ void __launch_bounds__(kThreads) k_pack(SlabView s, double* __restrict__ send) {
  pdl_launch_dependents();
  pdl_wait();
  Cand best = cand_none();
  for (int c = threadIdx.x; c < s.nslot; c += blockDim.x) best = cand_min(best, s.price[c]);
  best = block_min(best);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    send[0] = best.v;
    send[1] = __longlong_as_double(best.idx);
  }
  if (best.idx == LLONG_MAX) return;
  const long long kl = best.idx - s.c0;
  const int pend = s.st->pend_r;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < s.rows;
       i += (long long)gridDim.x * blockDim.x)
    send[2 + i] = (i == pend) ? s.rownorm[kl] : s.T[i * s.ld + kl];
}

// ------------------------------------------------------------------ a1-a3, a5: select
// Every CTA: (1) writes back the previous normalized pivot row; (2) folds the Step-1
// candidates into the entering column k (identical in every CTA and on every rank);
// (3) ratio-tests its rows (Step 2) and stages col[i] = T[i][k]; (4) the last CTA to
// finish folds the Step-2 candidates into r and decides the status in the order of
// reading c12: OPTIMAL (no k), UNBOUNDED (no r), ITERATION_LIMIT (it == cap), pivot.
__global__ void __launch_bounds__(kThreads) k_select(SlabView s, XView x, double tol_piv) {
  pdl_launch_dependents();
  pdl_wait();
  DevState* st = s.st;
  __shared__ int sh_last;
  const int tid = threadIdx.x;
  const long long it = st->it;
  const int status = st->status;
  const int pend = st->pend_r;
  const bool active = (status == kRunning) && (it < st->stop_at);
  const long long gthreads = (long long)gridDim.x * blockDim.x;
  const long long gtid = blockIdx.x * (long long)blockDim.x + tid;

  // (1) deferred write-back of row pend (nobody reads T[pend][.] in this kernel)
  if (pend >= 0) {
    double* dst = s.T + (long long)pend * s.ld;
    for (long long j = gtid; j < s.ld; j += gthreads) dst[j] = s.rownorm[j];
  }

  // (2) entering column (Step 1 fold)
  long long k = -1;
  const double* xcol = nullptr;
  if (active) {
    Cand best = cand_none();
    if (x.recv == nullptr) {
      for (int c = tid; c < s.nslot; c += blockDim.x) best = cand_min(best, s.price[c]);
    } else {
      for (int q = tid; q < x.nparts; q += blockDim.x) {
        const double* h = x.recv + (long long)q * x.stride;
        best = cand_min(best, Cand{h[0], __double_as_longlong(h[1])});
      }
    }
    best = block_min(best);
    if (best.idx != LLONG_MAX) {
      k = best.idx;
      if (x.recv != nullptr) {
        for (int q = 0; q < x.nparts; ++q) {      // owner = the part that sent (v, k)
          const double* h = x.recv + (long long)q * x.stride;
          if (__double_as_longlong(h[1]) == k) { xcol = h + 2; break; }
        }
      }
    }
  }

  // (3) Step 2 ratio test over this CTA's rows + staging of column k
  Cand rbest = cand_none();
  if (k >= 0) {
    const long long kl = k - s.c0;            // used only when nparts == 1 (then c0 == 0)
    for (long long i = gtid; i < s.rows; i += gthreads) {
      double a, rhs;
      if (i == pend) {
        a = xcol ? xcol[i] : s.rownorm[kl];
        rhs = s.rownorm[s.w];
      } else {
        a = xcol ? xcol[i] : s.T[i * s.ld + kl];
        rhs = s.T[i * s.ld + s.w];
      }
      s.col[i] = a;
      if (i >= 1 && a > tol_piv)
        rbest = cand_min(rbest, ratio_cand(s.rule, __ddiv_rn(rhs, a), i, s.rule ? s.basis[i - 1] : 0));
    }
  }
  rbest = block_min(rbest);
  if (tid == 0) s.rcand[blockIdx.x] = rbest;

  // (4) last CTA decides
  __threadfence();
  __syncthreads();
  if (tid == 0) sh_last = (atomicAdd(&st->ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!sh_last) return;
  __threadfence();
  Cand r = cand_none();
  for (int q = tid; q < (int)gridDim.x; q += blockDim.x) r = cand_min(r, ldcg_cand(s.rcand + q));
  r = block_min(r);
  if (tid == 0) {
    int go = 0;
    int rr = -1;
    if (!active) {
    } else if (k < 0) {
      st->status = kOptimal;
    } else if (r.idx == LLONG_MAX) {
      st->status = kUnbounded;
      st->k = (int)k;
    } else if (it >= st->cap) {
      st->status = kIterLimit;
    } else {
      go = 1;
      rr = cand_row(r.idx);
      st->r = rr;
      st->k = (int)k;
      st->p = __ldcg(s.col + rr);
      s.basis[rr - 1] = (int)k;
      if (it < s.trace_cap) {
        s.trace_k[it] = (int)k;
        s.trace_r[it] = rr;
      }
      st->it = it + 1;
    }
    st->go = go;
    st->pend_r = go ? rr : -1;
    st->ticket = 0;
    __threadfence();
  }
}

// ------------------------------------------------------------------ a4 (+a1): update
// Column-owner, row-strided schedule (measured best on B200 with scripts/ubench_update.cu):
// thread t owns the double2 column pair jp = t mod (ld/2) and rows k0 = t div (ld/2),
// k0+q, k0+2q, ... where q = (resident threads) div (ld/2).  At any moment all resident
// threads sweep q consecutive rows, so the chip-wide access front is one contiguous
// stretch of HBM (the same locality as a plain copy), every access is a coalesced
// 128-bit load/store, and prow_j = T[r][j] / p is computed ONCE per thread into
// registers.  URows rows are in flight per thread.
// Row r is not written: its normalized values go to rownorm and are written back by the
// next k_select / k_flush, so the q threads of a column can all read the raw row r.
// Row 0 (the threads with k0 == 0) also produces the Step-1 candidates of the next pivot
// per warp slot (fused pricing, PAPER.md:90 on the new objective row).
template <int URows>
__global__ void __launch_bounds__(kThreads) k_update(SlabView s, int q, double tol_opt) {
  pdl_launch_dependents();
  pdl_wait();
  const DevState* st = s.st;
  if (!st->go) return;
  const int r = st->r;
  const double p = st->p;
  const long long ld = s.ld;
  const long long half = ld >> 1;
  const int rows = s.rows;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool act = t < (long long)q * half;
  const long long jp = act ? t % half : 0;
  const int k0 = act ? (int)(t / half) : rows;
  const long long j = 2 * jp;
  double* Tj = s.T + j;

  double2 pr = make_double2(0.0, 0.0);
  if (act) {
    const double2 raw = *reinterpret_cast<const double2*>(s.T + (long long)r * ld + j);
    pr.x = __ddiv_rn(raw.x, p);
    pr.y = __ddiv_rn(raw.y, p);
    if (r % q == k0) *reinterpret_cast<double2*>(s.rownorm + j) = pr;
  }
  // first row of every thread (row 0 for k0 == 0 -> pricing of the next pivot)
  Cand best = cand_none();
  if (act) {
    double2 v = *reinterpret_cast<const double2*>(Tj + (long long)k0 * ld);
    const double a = -__ldg(s.col + k0);
    v.x = __fma_rn(a, pr.x, v.x);
    v.y = __fma_rn(a, pr.y, v.y);
    if (k0 != r) *reinterpret_cast<double2*>(Tj + (long long)k0 * ld) = v;
    if (k0 == 0) {
      const int pw = st->pw;
      if (j < pw && v.x < -tol_opt) best = price_cand(s.rule, v.x, s.c0 + j);
      if (j + 1 < pw && v.y < -tol_opt) best = cand_min(best, price_cand(s.rule, v.y, s.c0 + j + 1));
    }
  }
  if ((t & ~31LL) < half) {                        // warp-uniform: warps holding row-0 lanes
    best = warp_min(best);
    if ((threadIdx.x & 31) == 0) s.price[t >> 5] = best;
  }
  if (!act) return;
  int i = k0 + q;
  for (; i + (URows - 1) * q < rows; i += URows * q) {
    double2 v[URows];
#pragma unroll
    for (int u = 0; u < URows; ++u) v[u] = *reinterpret_cast<const double2*>(Tj + (long long)(i + u * q) * ld);
#pragma unroll
    for (int u = 0; u < URows; ++u) {
      const int iu = i + u * q;
      const double a = -__ldg(s.col + iu);
      v[u].x = __fma_rn(a, pr.x, v[u].x);
      v[u].y = __fma_rn(a, pr.y, v[u].y);
      if (iu != r) *reinterpret_cast<double2*>(Tj + (long long)iu * ld) = v[u];
    }
  }
  for (; i < rows; i += q) {
    double2 v = *reinterpret_cast<const double2*>(Tj + (long long)i * ld);
    const double a = -__ldg(s.col + i);
    v.x = __fma_rn(a, pr.x, v.x);
    v.y = __fma_rn(a, pr.y, v.y);
    if (i != r) *reinterpret_cast<double2*>(Tj + (long long)i * ld) = v;
  }
}

// ------------------------------------------------------------------ rank-s look-ahead (NEXT #1)
// Pivot t of a block needs only: the objective row of T^t (pricing), column k_t of T^t
// (ratio test, staged col), the rhs column of T^t and row r_t of T^t (pivot row).  With the
// block-start tableau T^0 untouched, each is T^0's entry followed by the chain of the
// pending pivots 0..t-1 in the paper's order (PAPER.md:94 applied t times):
//     x <- (i == r_u) ? prow_u[j] : fma(-col_u[i], prow_u[j], x),   u = 0 .. t-1
// so selecting s pivots ahead costs O(s^2 (m + W)) and ONE pass then applies the s chains to
// every element, in the same order: bitwise identical to s single pivots (reading c8).
//
// Barrier over the look-ahead kernel's CTAs: they form ONE thread-block cluster (up to 16
// SMs), so this is the hardware cluster barrier (release/acquire at cluster scope).  Data
// written by another CTA is read with ld.global.cg (L2), never through a stale L1.
#ifndef SX_LOOK_RB
#define SX_LOOK_RB 1
#endif
#ifndef SX_LOOK_CB
#define SX_LOOK_CB 2
#endif
// Cross-CTA reads in k_lookahead (values another CTA wrote before the last cluster barrier,
// whose acquire invalidates L1): through L1 (default) — the 8 warps of a CTA then share one
// L2 fetch of each broadcast operand (4000^2 blocks 211 -> 199 us) — or L2-only (SX_LOOK_CG).
// Previous-bank operands were written by the previous launch: read-only here (nc path).
#ifdef SX_LOOK_CG
#define SX_LDX(p) __ldcg(p)
#define SX_LDP(p) __ldcg(p)
#else
#define SX_LDX(p) (*(p))
#define SX_LDP(p) __ldg(p)
#endif
constexpr int kLookRB = SX_LOOK_RB;                 // rows per load batch of a selection thread
constexpr int kLookPreT = 2;                        // rows whose T entry is requested up front
constexpr int kLookPreC = 4;                        // columns whose row-r entry is requested up front
constexpr int kLookCB = SX_LOOK_CB;                 // columns per load batch

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Distributed shared memory of another CTA may be written only once that CTA has started: every
// cluster kernel arrives (relaxed) on entry and its FIRST cluster_min waits for all arrivals before
// its DSMEM stores (compute-sanitizer racecheck: "write ... in a block that might not have entered
// yet").  The arrive/wait split keeps the wait off the critical path in practice.
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

// Cluster-wide lexicographic argmin, identical in every CTA of the cluster.  Each CTA
// reduces its warps, then warp 0 writes the CTA's candidate straight into slot[rank] of
// EVERY CTA's shared memory (DSMEM st.shared::cluster), one cluster barrier, and every
// CTA folds its local copy.  `slot` is double-buffered by `ph` (a CTA can be at most one
// reduction ahead of another), so two consecutive reductions never share a slot.
// post_row (optional): thread 0 records a new pivot row — post_row[0] = post_val and its bit in
// post_mark — after the CTA barrier that ends every thread's reads of the previous phase and before
// the one that publishes the result (a write outside that window races with the phase's reads of
// the same shared arrays: compute-sanitizer racecheck).
__device__ __forceinline__ Cand cluster_min(Cand c, Cand* slot, int ph, const double* pf_rows = nullptr,
                                            long long pf_ld = 0, bool first = false, int* post_row = nullptr,
                                            int post_val = 0, unsigned int* post_mark = nullptr,
                                            unsigned long long* pr = nullptr) {
  __shared__ Cand sh_w[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned int rank, nct;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(nct));
  c = warp_min(c);
  if (lane == 0) sh_w[wid] = c;
  if (first) cluster_wait();                          // every CTA of the cluster has started
  __syncthreads();
  if (post_row && threadIdx.x == 0) {
    *post_row = post_val;
    post_mark[post_val >> 5] |= 1u << (post_val & 31);
  }
  if (wid == 0) {
    Cand t = lane < (int)(blockDim.x >> 5) ? sh_w[lane] : cand_none();
    t = warp_min(t);
    if (pr && lane == 0) {                              // experiment probe: CTA reduction done
      unsigned long long tnow;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow) : "l"(t.idx));
      pr[0] = tnow;
    }
    if (lane < (int)nct) {
      const uint32_t local = smem_u32(slot + ph * 16 + rank);
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(lane));
      asm volatile("st.shared::cluster.v2.b64 [%0], {%1, %2};" ::"r"(remote), "l"(__double_as_longlong(t.v)),
                   "l"(t.idx)
                   : "memory");
    }
    // row candidates: start pulling this CTA's best row into L2 while the cluster agrees on
    // the winner (one of the nct CTA bests), so the next phase reads it from L2, not HBM
    if (pf_rows && lane == 0 && t.idx != LLONG_MAX)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf_rows + (long long)cand_row(t.idx) * pf_ld),
                   "r"((uint32_t)(pf_ld * sizeof(double)))
                   : "memory");
  }
  cluster_barrier();
  if (pr && threadIdx.x == 0) {                         // experiment probe: cluster barrier done
    unsigned long long tnow;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
    pr[1] = tnow;
  }
  // every warp folds the nct slots itself (a CTA barrier to broadcast warp 0's fold would cost
  // more than the redundant 32-lane argmin); the cluster barrier above already ordered every
  // shared-memory write of the phase for all threads
  Cand t = lane < (int)nct ? slot[ph * 16 + lane] : cand_none();
  return warp_min(t);
}


// k_lookahead: one thread-block cluster (one CTA per SM) selecting up to S pivots into chain
// bank `bown`.  Per pivot t:
//   phase A (rows, grid-stride): RHS <- the rhs after the previous pivot, column k of the
//            current tableau by the chain from T, staged into colS[.][bown][t], Step-2
//            candidates -> cluster argmin -> r;
//   phase B (columns, grid-stride): row r by the chain, prowS[bown][t] = row / p, the
//            objective row R0 <- the next one, Step-1 candidates -> cluster argmin -> k of t+1.
// `T` is the tableau the chains start from.  bpre < 0 (prologue): T is the current tableau and
// R0 / RHS are read from it.  bpre >= 0 (software pipeline): T is the tableau
// BEFORE the previous block, whose pass is running concurrently on the other SMs; its pivots
// (bank bpre) are chained first, R0 / RHS continue from the previous launch.  Chained in the
// oracle's order, every value is bitwise the one the single-pivot sequence produces.
// Every thread always owns the same rows / columns, so R0, RHS, colS[i][.] and prowS[.][j]
// are only re-read by their writer; values written by OTHER CTAs are read with ld.cg.  All
// loads a phase needs (per-step scalars, the T entry, the pending chain operands) are issued
// before the first dependent use, so each phase costs about one memory latency.
__global__ void __launch_bounds__(kLookThreads) k_lookahead(SlabView s, const double* __restrict__ T, int S,
                                                           int bown, int bpre, int nqc, int nqr, double tol_opt,
                                                           double tol_piv) {
  pdl_launch_dependents();                            // the previous block's pass may start now
  cluster_arrive_relaxed();                           // (waited for in the first cluster_min)
  DevState* st = s.st;
  __shared__ int sh_r[kMaxLook];                      // own pivot rows
  __shared__ int sh_rp[kMaxLook];                     // pivot rows of the previous block (bpre)
  __shared__ __align__(16) Cand slot[2 * 16];
  extern __shared__ unsigned int piv_mark[];          // rows that are pivot rows of a pending chain
  const long long gthreads = (long long)gridDim.x * blockDim.x;
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int rows = s.rows;
  const long long ld = s.ld;
  const int w = s.w;                                  // rhs column
  const int pw = st->pw;                              // priced columns (Phase II: no artificials)
  double* __restrict__ colO = s.colS + bown * kMaxLook;                 // row stride kColS
  const double* __restrict__ colP = s.colS + (bpre >= 0 ? bpre : 0) * kMaxLook;
  // transposed copies [t][row] of both banks: per-row loads of a warp hit consecutive rows
  double* __restrict__ colTo = s.colT + (size_t)bown * kMaxLook * rows;
  const double* __restrict__ colTp = s.colT + (size_t)(bpre >= 0 ? bpre : 0) * kMaxLook * rows;
  double* __restrict__ prowO = s.prowS + (long long)bown * kMaxLook * ld;
  const double* __restrict__ prowP = s.prowS + (long long)(bpre >= 0 ? bpre : 0) * kMaxLook * ld;
  double* __restrict__ R0 = s.R0;
  double* __restrict__ RHS = s.RHS;
  long long it = st->it;
  int status = st->status;
  const long long stop = st->stop_at;
  const long long cap = st->cap;
  const int spre = bpre >= 0 ? st->sb[bpre] : 0;
  int ph = 0;
  unsigned long long* prb = s.probe ? s.probe + ((size_t)((it / kMaxLook) % kProbeSlots) * 16 + (blockIdx.x & 15)) * kProbeEv
                                    : nullptr;
#define SX_PROBE(e)                                                                 \
  do {                                                                              \
    if (prb && threadIdx.x == 0) {                                                  \
      unsigned long long tnow;                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));                      \
      prb[e] = tnow;                                                                \
    }                                                                               \
  } while (0)
#define SX_PROBE_DEP(e, dep)                                                        \
  do {                                                                              \
    if (prb && threadIdx.x == 0) {                                                  \
      unsigned long long tnow;                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow) : "d"(dep));           \
      prb[e] = tnow;                                                                \
    }                                                                               \
  } while (0)
  SX_PROBE(0);
  // nqc > 0: the previous bank's operands of this thread's columns / rows are read ONCE into
  // shared memory (the same values are chained at every step of this launch):
  //   cP[(u * nqc + q) * blockDim + tid] = prow_u[j_q],  cR[(u * nqr + q) * blockDim + tid] = col_u[i_q]
  const int mwords = ((rows + 31) / 32 + 3) & ~3;
  double* cP = reinterpret_cast<double*>(piv_mark + mwords);
  double* cR = cP + (size_t)kMaxLook * nqc * blockDim.x;
  const bool cache = nqc > 0 && spre > 0;
  if (cache) {                                        // async copies (LDGSTS): no register staging,
    for (int q = 0; q < nqc; ++q) {                   // all in flight at once, overlapping the first
      const long long j = gtid + (long long)q * gthreads;   // pricing scan and reduction
      if (j < ld) {
#pragma unroll
        for (int u = 0; u < kMaxLook; ++u)
          if (u < spre)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                             smem_u32(&cP[((size_t)u * nqc + q) * blockDim.x + threadIdx.x])),
                         "l"(prowP + (long long)u * ld + j)
                         : "memory");
      }
    }
    for (int q = 0; q < nqr; ++q) {
      const long long i = gtid + (long long)q * gthreads;
      if (i < rows) {
#pragma unroll
        for (int u = 0; u < kMaxLook; ++u)
          if (u < spre)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                             smem_u32(&cR[((size_t)u * nqr + q) * blockDim.x + threadIdx.x])),
                         "l"(colTp + (size_t)u * rows + i)
                         : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int q = threadIdx.x; q < (rows + 31) / 32; q += blockDim.x) piv_mark[q] = 0u;
  if (threadIdx.x < kMaxLook) sh_rp[threadIdx.x] = (int)threadIdx.x < spre ? st->rsb[bpre][threadIdx.x] : -1;
  __syncthreads();
  if ((int)threadIdx.x < spre) atomicOr(&piv_mark[sh_rp[threadIdx.x] >> 5], 1u << (sh_rp[threadIdx.x] & 31));

  // Step 1 of the first pivot, from T's objective row (prologue) or the running R0
  Cand best = cand_none();
  if (bpre < 0) {
    for (long long j = gtid; j < ld; j += gthreads) {
      const double v = T[j];
      R0[j] = v;
      if (j < pw && v < -tol_opt) best = cand_min(best, price_cand(s.rule, v, s.c0 + j));
    }
    for (long long i = gtid; i < rows; i += gthreads) RHS[i] = T[i * ld + w];
  } else {
    for (long long j = gtid; j < pw; j += gthreads) {
      const double v = R0[j];
      if (v < -tol_opt) best = cand_min(best, price_cand(s.rule, v, s.c0 + j));
    }
  }
  best = cluster_min(best, slot, ph, nullptr, 0, true);   // (its barriers also publish piv_mark)
  ph ^= 1;
  SX_PROBE(1);

  if (cache) asm volatile("cp.async.wait_group 0;" ::: "memory");   // own entries only: no barrier
  int t = 0;
  int r_prev = spre > 0 ? sh_rp[spre - 1] : -1;       // pivot not yet applied to RHS
  const double* c_prev = spre > 0 ? colTp + (size_t)(spre - 1) * rows : nullptr;   // transposed
  const double* p_prev = spre > 0 ? prowP + (long long)(spre - 1) * ld : nullptr;
  for (; t < S; ++t) {
    if (status != kRunning || it >= stop) break;
    if (best.idx == LLONG_MAX) { status = kOptimal; break; }                 // Step 1: optimal
    const long long k = best.idx;
    // ---- phase A: rows
    double qk[kMaxLook], pk[kMaxLook];                  // prow_u[k] of both banks (L2, same for all rows)
#pragma unroll
    for (int u = 0; u < kMaxLook; ++u) qk[u] = u < spre ? SX_LDP(prowP + (long long)u * ld + k) : 0.0;
#pragma unroll
    for (int u = 0; u < kMaxLook; ++u) pk[u] = u < t ? SX_LDX(prowO + (long long)u * ld + k) : 0.0;
    const double pw_prev = r_prev >= 0 ? SX_LDX(p_prev + w) : 0.0;
    Cand rb = cand_none();
    // rows in batches of kLookRB per thread: every load of the batch (the T entry, the rhs, the
    // chain operands) is issued before the first dependent FMA, so a batch costs one latency
    // the entering column's entries of this thread's first kLookPreT rows are requested at once
    // (HBM), so the row batches below do not each wait for their own HBM round trip
    double tpre[kLookPreT];
#pragma unroll
    for (int b = 0; b < kLookPreT; ++b) {
      const long long i = gtid + (long long)b * gthreads;
      tpre[b] = i < rows ? T[i * ld + k] : 0.0;
    }
    for (long long i0 = gtid, qi0 = 0; i0 < rows; i0 += kLookRB * gthreads, qi0 += kLookRB) {
      double xb[kLookRB], hb[kLookRB], cpb[kLookRB], cub[kLookRB][kMaxLook];
#pragma unroll
      for (int b = 0; b < kLookRB; ++b) {
        const long long i = i0 + b * gthreads;
        const bool v = b == 0 || i < rows;
        double xv = 0.0;
        bool have = false;
#pragma unroll
        for (int pb = 0; pb < kLookPreT; ++pb)
          if (qi0 + b == pb) {
            xv = tpre[pb];
            have = true;
          }
        xb[b] = have ? xv : (v ? T[i * ld + k] : 0.0);
        hb[b] = v ? RHS[i] : 0.0;
        cpb[b] = v && r_prev >= 0 ? c_prev[i] : 0.0;
#pragma unroll
        for (int u = 0; u < kMaxLook; ++u) cub[b][u] = v && u < t ? colTo[(size_t)u * rows + i] : 0.0;
      }
      if (i0 == gtid) SX_PROBE_DEP(2 + 10 * t, xb[0] + hb[0] + cpb[0] + cub[0][0] + cub[0][kMaxLook - 1]);
#pragma unroll
      for (int b = 0; b < kLookRB; ++b) {
        const long long i = i0 + b * gthreads;
        if (b > 0 && i >= rows) break;
        const long long qi = qi0 + b;
        double x = xb[b];
        double h = hb[b];
        double cq[kMaxLook];                              // this row's previous-bank column entries
#pragma unroll
        for (int u = 0; u < kMaxLook; ++u)
          cq[u] = u < spre ? (cache ? cR[((size_t)u * nqr + qi) * blockDim.x + threadIdx.x] : colTp[(size_t)u * rows + i])
                           : 0.0;
        if (r_prev >= 0) h = (i == r_prev) ? pw_prev : __fma_rn(-cpb[b], pw_prev, h);
        RHS[i] = h;
        if ((piv_mark[i >> 5] >> (i & 31)) & 1u) {       // row i is a pivot row of a pending chain
#pragma unroll
          for (int u = 0; u < kMaxLook; ++u)
            if (u < spre) x = (i == sh_rp[u]) ? qk[u] : __fma_rn(-cq[u], qk[u], x);
#pragma unroll
          for (int u = 0; u < kMaxLook; ++u)
            if (u < t) x = (i == sh_r[u]) ? pk[u] : __fma_rn(-cub[b][u], pk[u], x);
        } else {
#pragma unroll
          for (int u = 0; u < kMaxLook; ++u)
            if (u < spre) x = __fma_rn(-cq[u], qk[u], x);
#pragma unroll
          for (int u = 0; u < kMaxLook; ++u)
            if (u < t) x = __fma_rn(-cub[b][u], pk[u], x);
        }
        colO[i * kColS + t] = x;                       // (row-major: the pass's TMA rows)
        colTo[(size_t)t * rows + i] = x;
        if (i >= 1 && x > tol_piv)                                              // Step 2
          rb = cand_min(rb, ratio_cand(s.rule, __ddiv_rn(h, x), i, s.rule ? __ldcg(s.basis + i - 1) : 0));
      }
    }
    SX_PROBE(3 + 10 * t);
    rb = cluster_min(rb, slot, ph, T, ld, false, nullptr, 0, nullptr, prb ? prb + 4 + 10 * t : nullptr);
    ph ^= 1;
    SX_PROBE(6 + 10 * t);
    if (rb.idx == LLONG_MAX) {                                                 // unbounded
      status = kUnbounded;
      if (gtid == 0) st->k = (int)k;
      break;
    }
    if (it >= cap) { status = kIterLimit; break; }                            // reading c12
    const int r = cand_row(rb.idx);
    // ---- phase B: columns (pivot row, normalized; the next objective row)
    double cr[kMaxLook], cs[kMaxLook];                  // col_u[r] of both banks (L2, same for all columns)
#pragma unroll
    for (int u = 0; u < kMaxLook; ++u) cs[u] = u < spre ? SX_LDP(colP + (long long)r * kColS + u) : 0.0;
#pragma unroll
    for (int u = 0; u < kMaxLook; ++u) cr[u] = u < t ? SX_LDX(colO + (long long)r * kColS + u) : 0.0;
    const double p = SX_LDX(colO + (long long)r * kColS + t);
    const double a0 = -SX_LDX(colO + t);                                      // col_t[0]
    const double* Tr = T + (long long)r * ld;
    double* prow = prowO + (long long)t * ld;
    unsigned int rmask = 0u, qmask = 0u;                // bit u: r was pivot row u (own / previous bank)
#pragma unroll
    for (int u = 0; u < kMaxLook; ++u) {
      if (u < t && sh_r[u] == r) rmask |= 1u << u;
      if (u < spre && sh_rp[u] == r) qmask |= 1u << u;
    }
    best = cand_none();
    // columns in batches of kLookCB per thread (loads of the batch first, as for the rows)
    double rpre[kLookPreC];                             // row r's entries of the first columns, at once
#pragma unroll
    for (int b = 0; b < kLookPreC; ++b) {
      const long long j = gtid + (long long)b * gthreads;
      rpre[b] = j < ld ? Tr[j] : 0.0;
    }
    for (long long j0 = gtid, qj0 = 0; j0 < ld; j0 += kLookCB * gthreads, qj0 += kLookCB) {
      double xb[kLookCB], r0b[kLookCB], pub[kLookCB][kMaxLook];
#pragma unroll
      for (int b = 0; b < kLookCB; ++b) {
        const long long j = j0 + b * gthreads;
        const bool v = b == 0 || j < ld;
        double xv = 0.0;
        bool have = false;
#pragma unroll
        for (int pb = 0; pb < kLookPreC; ++pb)
          if (qj0 + b == pb) {
            xv = rpre[pb];
            have = true;
          }
        xb[b] = have ? xv : (v ? Tr[j] : 0.0);
        r0b[b] = v ? R0[j] : 0.0;
#pragma unroll
        for (int u = 0; u < kMaxLook; ++u) pub[b][u] = v && u < t ? prowO[(long long)u * ld + j] : 0.0;
      }
      if (j0 == gtid) SX_PROBE_DEP(7 + 10 * t, xb[0] + r0b[0] + pub[0][0] + pub[0][kMaxLook - 1]);
#pragma unroll
      for (int b = 0; b < kLookCB; ++b) {
        const long long j = j0 + b * gthreads;
        if (b > 0 && j >= ld) break;
        const long long qj = qj0 + b;
        double x = xb[b];
        double qu[kMaxLook];                              // this column's previous-bank row entries
#pragma unroll
        for (int u = 0; u < kMaxLook; ++u)
          qu[u] = u < spre ? (cache ? cP[((size_t)u * nqc + qj) * blockDim.x + threadIdx.x] : prowP[(long long)u * ld + j])
                           : 0.0;
#pragma unroll
        for (int u = 0; u < kMaxLook; ++u)
          if (u < spre) x = ((qmask >> u) & 1u) ? qu[u] : __fma_rn(-cs[u], qu[u], x);
#pragma unroll
        for (int u = 0; u < kMaxLook; ++u)
          if (u < t) x = ((rmask >> u) & 1u) ? pub[b][u] : __fma_rn(-cr[u], pub[b][u], x);
        const double pj = __ddiv_rn(x, p);
        prow[j] = pj;
        const double v = __fma_rn(a0, pj, r0b[b]);
        R0[j] = v;
        if (j < pw && v < -tol_opt) best = cand_min(best, price_cand(s.rule, v, s.c0 + j));  // Step 1 of t+1
      }
    }
    if (gtid == 0) {
      st->rsb[bown][t] = r;
      s.basis[r - 1] = (int)k;
      if (it < s.trace_cap) {
        s.trace_k[it] = (int)k;
        s.trace_r[it] = r;
      }
    }
    ++it;
    r_prev = r;
    c_prev = colTo + (size_t)t * rows;
    p_prev = prow;
    SX_PROBE(8 + 10 * t);
    best = cluster_min(best, slot, ph, nullptr, 0, false, &sh_r[t], r, piv_mark,   // (+ row r recorded)
                       prb ? prb + 9 + 10 * t : nullptr);
    ph ^= 1;
    SX_PROBE(11 + 10 * t);
  }
#undef SX_PROBE
#undef SX_PROBE_DEP
  if (gtid == 0) {
    st->status = status;
    st->it = it;
    st->sb[bown] = t;
    st->go = t > 0;
    st->pend_r = -1;
  }
}

// ------------------------------------------------------------------ k_look2
// k_look2: k_lookahead's selection (same pivots, same arithmetic, same order: bitwise identical)
// reorganised so that a pivot's two phases are short.  ncu of k_lookahead showed
// the selection issue- and dependency-bound: each phase re-read up to 31 chain operands per
// element through L2 (the cluster barrier's acquire invalidates L1), every thread re-loaded up to
// 33 broadcast scalars, and the chains carried a bit-test + two selects per operand.  Here:
//   * every chain operand of a thread's elements lives in SHARED memory as double2 pairs
//     [q][u/2][tid] (one conflict-free LDS.128 per two operands): the own bank (this launch's
//     pivots: col_u[i] of its rows, prow_u[j] of its columns) and (PS) the previous bank, copied
//     in at launch start from the global hand-off s.hand[bpre], which the previous launch wrote
//     from the SAME thread positions (without PS: read from the hand-off);
//   * the running objective row R0 and rhs column RHS of own elements stay in shared memory;
//   * a phase's broadcast operands (prow_u[k] of both banks + the previous pivot's rhs entry;
//     col_u[r] of both banks + col_t[0]) are loaded ONCE per warp, one lane per value, behind the
//     phase's own T loads, into a per-warp shared buffer read with broadcast LDS.128;
//   * QC / QR own columns / rows per thread are compile-time, so their chains interleave
//     (instruction-level parallelism on the 8-cycle DFMA dependency), and the common case — the
//     pivot row of this step is no pending pivot row, the previous bank is full — runs plain FMA
//     chains without per-operand selects or predicates;
//   * chunks of 32 consecutive elements are dealt to the cluster's CTAs round-robin, so small
//     tableaux keep every SM of the cluster busy.
// The pass (k_update_s) still gets colS / prowS from global memory.
template <int NT, bool PS, int QC, int QR>
__global__ void __launch_bounds__(NT, 1) k_look2(SlabView s, const double* __restrict__ T, int S, int bown,
                                                 int bpre, int nqc, int nqr, double tol_opt, double tol_piv) {
  pdl_launch_dependents();                            // the previous block's pass may start now
  cluster_arrive_relaxed();                           // (waited for in the first cluster_min)
  constexpr int NW = NT / 32;
  constexpr int H = kMaxLook / 2;                     // operand pairs per bank
  DevState* st = s.st;
  __shared__ int sh_r[kMaxLook];
  __shared__ int sh_rp[kMaxLook];
  __shared__ __align__(16) Cand slot[2 * 16];
  __shared__ __align__(16) double bcw[NW][36];       // per-warp broadcast operands of a phase
  extern __shared__ __align__(16) unsigned int sm2[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = (int)gridDim.x * NT;
  const int gtid = (int)blockIdx.x * NT + tid;
  const int rows = s.rows;
  const long long ld = s.ld;
  const int w = s.w;
  const int pw = st->pw;
  const int mwords = ((rows + 31) / 32 + 3) & ~3;
  unsigned int* piv_mark = sm2;
  double2* OP = reinterpret_cast<double2*>(sm2 + mwords);          // [QC][H][NT] own prow_u[j]
  double2* OC = OP + (size_t)QC * H * NT;                           // [QR][H][NT] own col_u[i]
  double* R0s = reinterpret_cast<double*>(OC + (size_t)QR * H * NT);   // [QC][NT]
  double* RHSs = R0s + (size_t)QC * NT;                                          // [QR][NT]
  double2* PPs = reinterpret_cast<double2*>(RHSs + (size_t)QR * NT);    // PS: [QC][H][NT]
  double2* PCs = PPs + (size_t)QC * H * NT;                              // PS: [QR][H][NT]
  const size_t hbank = (size_t)(nqc + nqr) * H * G;  // hand-off: [nqc][H][G] columns, [nqr][H][G] rows
  double2* __restrict__ hown = s.hand + (size_t)bown * hbank;
  const double2* __restrict__ hpre = s.hand + (size_t)(bpre >= 0 ? bpre : 0) * hbank;
  double* __restrict__ colO = s.colS + bown * kMaxLook;
  const double* __restrict__ colP = s.colS + (bpre >= 0 ? bpre : 0) * kMaxLook;
  double* __restrict__ prowO = s.prowS + (long long)bown * kMaxLook * ld;
  const double* __restrict__ prowP = s.prowS + (long long)(bpre >= 0 ? bpre : 0) * kMaxLook * ld;
  long long it = st->it;
  int status = st->status;
  const long long stop = st->stop_at;
  const long long cap = st->cap;
  const int spre = bpre >= 0 ? st->sb[bpre] : 0;
  int ph = 0;
  // own columns / rows (valid: < ld / < rows): element e = lane + 32 (cta + C (warp + NW q))
  const int C = (int)gridDim.x;
  long long jq[QC], iq[QR];
#pragma unroll
  for (int q = 0; q < QC; ++q) jq[q] = lane + 32LL * (blockIdx.x + (long long)C * (wid + (long long)NW * q));
#pragma unroll
  for (int q = 0; q < QR; ++q) iq[q] = lane + 32LL * (blockIdx.x + (long long)C * (wid + (long long)NW * q));
  unsigned long long* prb = s.probe ? s.probe + ((size_t)((it / kMaxLook) % kProbeSlots) * 16 + (blockIdx.x & 15)) * kProbeEv
                                    : nullptr;
#ifdef SX_PROBE_DETAIL
#define SX_TIMER "%%clock64"                          // detail probes: SM cycles (intervals within a CTA)
#else
#define SX_TIMER "%%globaltimer"
#endif
#define SX_PROBE(e)                                                                 \
  do {                                                                              \
    if (prb && threadIdx.x == 0) {                                                  \
      unsigned long long tnow;                                                      \
      asm volatile("mov.u64 %0, " SX_TIMER ";" : "=l"(tnow));                       \
      prb[e] = tnow;                                                                \
    }                                                                               \
  } while (0)
  SX_PROBE(0);
  // chain operand pair v of own column / row q: previous bank (smem copy, or the hand-off, read
  // only for valid elements) and own bank (smem)
  auto pre_c = [&](int q, int v) -> double2 {
    if (PS) return PPs[((size_t)q * H + v) * NT + tid];
    return jq[q] < ld ? __ldg(hpre + ((size_t)q * H + v) * G + gtid) : make_double2(0.0, 0.0);
  };
  auto pre_r = [&](int q, int v) -> double2 {
    if (PS) return PCs[((size_t)q * H + v) * NT + tid];
    return iq[q] < rows ? __ldg(hpre + ((size_t)(nqc + q) * H + v) * G + gtid) : make_double2(0.0, 0.0);
  };
  auto own_c = [&](int q, int v) -> double2 { return OP[((size_t)q * H + v) * NT + tid]; };
  auto own_r = [&](int q, int v) -> double2 { return OC[((size_t)q * H + v) * NT + tid]; };
  auto own_c_set = [&](int q, int u, double val) {
    reinterpret_cast<double*>(OP + ((size_t)q * H + (u >> 1)) * NT + tid)[u & 1] = val;
  };
  auto own_r_set = [&](int q, int u, double val) {
    reinterpret_cast<double*>(OC + ((size_t)q * H + (u >> 1)) * NT + tid)[u & 1] = val;
  };
  const int vpre = (spre + 1) >> 1;                   // pairs holding the spre previous operands
  if (PS && spre > 0) {
#pragma unroll
    for (int q = 0; q < QC; ++q)
      if (jq[q] < ld)
        for (int v = 0; v < vpre; ++v)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(PPs + ((size_t)q * H + v) * NT + tid)),
                       "l"(hpre + ((size_t)q * H + v) * G + gtid)
                       : "memory");
#pragma unroll
    for (int q = 0; q < QR; ++q)
      if (iq[q] < rows)
        for (int v = 0; v < vpre; ++v)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(PCs + ((size_t)q * H + v) * NT + tid)),
                       "l"(hpre + ((size_t)(nqc + q) * H + v) * G + gtid)
                       : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int q = tid; q < (rows + 31) / 32; q += NT) piv_mark[q] = 0u;
  if (tid < kMaxLook) sh_rp[tid] = tid < spre ? st->rsb[bpre][tid] : -1;
  Cand best = cand_none();
#pragma unroll
  for (int q = 0; q < QC; ++q) {
    const long long j = jq[q];
    if (j < ld) {
      const double v = bpre < 0 ? T[j] : s.R0[j];
      R0s[q * NT + tid] = v;
      if (j < pw && v < -tol_opt) best = cand_min(best, price_cand(s.rule, v, s.c0 + j));
    }
  }
#pragma unroll
  for (int q = 0; q < QR; ++q)
    if (iq[q] < rows) RHSs[q * NT + tid] = bpre < 0 ? T[iq[q] * ld + w] : s.RHS[iq[q]];
  __syncthreads();
  if (tid < spre) atomicOr(&piv_mark[sh_rp[tid] >> 5], 1u << (sh_rp[tid] & 31));
  best = cluster_min(best, slot, ph, nullptr, 0, true);   // (its barriers also publish piv_mark)
  ph ^= 1;
  SX_PROBE(1);
  if (PS && spre > 0) asm volatile("cp.async.wait_group 0;" ::: "memory");   // own entries only: no barrier

  int t = 0;
  int r_prev = spre > 0 ? sh_rp[spre - 1] : -1;       // pivot not yet applied to RHS
  const double* p_prev = spre > 0 ? prowP + (long long)(spre - 1) * ld : nullptr;
  double* bw = bcw[wid];
  const double2* bw2 = reinterpret_cast<const double2*>(bw);
  for (; t < S; ++t) {
    if (status != kRunning || it >= stop) break;
    if (best.idx == LLONG_MAX) { status = kOptimal; break; }                 // Step 1: optimal
    const long long k = best.idx - s.c0;
    // ---- phase A: rows.  Own T entries first (HBM), then the warp's broadcast operands.
    double x[QR];
#pragma unroll
    for (int q = 0; q < QR; ++q) x[q] = iq[q] < rows ? T[iq[q] * ld + k] : 0.0;
    {                                                  // lane u: prow_u[k] (prev bank u < 16, own 16+u)
      const int u = lane & (kMaxLook - 1);             // (own bank: written before the last barrier)
      const bool ok = lane < kMaxLook ? u < spre : u < t;
      const double* src = (lane < kMaxLook ? prowP : prowO) + (long long)u * ld + k;
      const double v = ok ? *src : 0.0;
      const double v2 = lane == 0 && r_prev >= 0 ? p_prev[w] : 0.0;   // both loads in flight at once
      bw[lane] = v;
      if (lane == 0) bw[32] = v2;
      __syncwarp();
    }
    SX_PROBE(2 + 10 * t);
    // own-bank operands of the own rows
    double2 ob[QR][H];
#pragma unroll
    for (int v = 0; v < H; ++v)
#pragma unroll
      for (int q = 0; q < QR; ++q) ob[q][v] = 2 * v < t ? own_r(q, v) : make_double2(0.0, 0.0);
    const double pw_prev = bw[32];
    double h[QR];
    bool marked = false;
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      const long long i = iq[q];
      h[q] = RHSs[q * NT + tid];
      if (r_prev >= 0) {
        double cpv;
        if (t > 0) {
          cpv = 0.0;
#pragma unroll
          for (int v = 0; v < H; ++v)
            if (v == ((t - 1) >> 1)) cpv = ((t - 1) & 1) ? ob[q][v].y : ob[q][v].x;
        } else {
          cpv = PS ? reinterpret_cast<const double*>(PCs + ((size_t)q * H + ((spre - 1) >> 1)) * NT + tid)[(spre - 1) & 1]
                   : (i < rows ? reinterpret_cast<const double*>(hpre + ((size_t)(nqc + q) * H + ((spre - 1) >> 1)) * G + gtid)[(spre - 1) & 1]
                               : 0.0);
        }
        h[q] = (i == r_prev) ? pw_prev : __fma_rn(-cpv, pw_prev, h[q]);
        if (i < rows) RHSs[q * NT + tid] = h[q];
      }
      if (i < rows && ((piv_mark[i >> 5] >> (i & 31)) & 1u)) marked = true;
    }
#ifdef SX_PROBE_DETAIL
    SX_PROBE(3 + 10 * t);
#endif
    if (!marked) {                                     // no own row is a pending pivot row: plain chains
#pragma unroll
      for (int v = 0; v < H; ++v) {
        if (spre < kMaxLook && 2 * v >= spre) break;
        const double2 bq = bw2[v];                     // qk pair (broadcast LDS)
        double2 a[QR];
#pragma unroll
        for (int q = 0; q < QR; ++q) a[q] = pre_r(q, v);
#pragma unroll
        for (int q = 0; q < QR; ++q) {
          x[q] = __fma_rn(-a[q].x, bq.x, x[q]);
          if (spre == kMaxLook || 2 * v + 1 < spre) x[q] = __fma_rn(-a[q].y, bq.y, x[q]);
        }
      }
#pragma unroll
      for (int v = 0; v < H; ++v) {
        if (2 * v >= t) break;
        const double2 bp = bw2[H + v];                 // pk pair
#pragma unroll
        for (int q = 0; q < QR; ++q) {
          x[q] = __fma_rn(-ob[q][v].x, bp.x, x[q]);
          if (2 * v + 1 < t) x[q] = __fma_rn(-ob[q][v].y, bp.y, x[q]);
        }
      }
    } else {                                           // some own row was a pivot row: take prow there
#pragma unroll
      for (int q = 0; q < QR; ++q) {
        const long long i = iq[q];
#pragma unroll
        for (int v = 0; v < H; ++v) {
          const double2 bq = bw2[v];
          const double2 a = 2 * v < spre ? pre_r(q, v) : make_double2(0.0, 0.0);
          if (2 * v < spre) x[q] = (i == sh_rp[2 * v]) ? bq.x : __fma_rn(-a.x, bq.x, x[q]);
          if (2 * v + 1 < spre) x[q] = (i == sh_rp[2 * v + 1]) ? bq.y : __fma_rn(-a.y, bq.y, x[q]);
        }
#pragma unroll
        for (int v = 0; v < H; ++v) {
          const double2 bp = bw2[H + v];
          if (2 * v < t) x[q] = (i == sh_r[2 * v]) ? bp.x : __fma_rn(-ob[q][v].x, bp.x, x[q]);
          if (2 * v + 1 < t) x[q] = (i == sh_r[2 * v + 1]) ? bp.y : __fma_rn(-ob[q][v].y, bp.y, x[q]);
        }
      }
    }
#ifdef SX_PROBE_DETAIL
    SX_PROBE(4 + 10 * t);
#endif
    Cand rb = cand_none();
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      const long long i = iq[q];
      if (i < rows) {
        own_r_set(q, t, x[q]);
        colO[i * kColS + t] = x[q];                    // (row-major: the pass's TMA rows)
        if (i >= 1 && x[q] > tol_piv)                                           // Step 2
          rb = cand_min(rb, ratio_cand(s.rule, __ddiv_rn(h[q], x[q]), i, s.rule ? __ldcg(s.basis + i - 1) : 0));
      }
    }
#ifdef SX_PROBE_DETAIL
    SX_PROBE(5 + 10 * t);
    rb = cluster_min(rb, slot, ph, T, ld);
#else
    SX_PROBE(3 + 10 * t);
    rb = cluster_min(rb, slot, ph, T, ld, false, nullptr, 0, nullptr, prb ? prb + 4 + 10 * t : nullptr);
#endif
    ph ^= 1;
    SX_PROBE(6 + 10 * t);
    if (rb.idx == LLONG_MAX) {                                                 // unbounded
      status = kUnbounded;
      if (gtid == 0) st->k = (int)(k + s.c0);
      break;
    }
    if (it >= cap) { status = kIterLimit; break; }                            // reading c12
    const int r = cand_row(rb.idx);
    // ---- phase B: columns.  Own entries of row r first (L2: prefetched during reduction A).
    const double* Tr = T + (long long)r * ld;
    double y[QC];
#pragma unroll
    for (int q = 0; q < QC; ++q) y[q] = jq[q] < ld ? Tr[jq[q]] : 0.0;
    {                                                  // lane u: col_u[r] (prev bank u < 16, own 16+u, u <= t)
      const int u = lane & (kMaxLook - 1);
      const bool ok = lane < kMaxLook ? u < spre : u <= t;
      const double* src = (lane < kMaxLook ? colP : colO) + (long long)r * kColS + u;
      const double v = ok ? *src : 0.0;
      const double v2 = lane == 0 ? -colO[t] : 0.0;                // -col_t[0]
      bw[lane] = v;
      if (lane == 0) bw[32] = v2;
      __syncwarp();
    }
    double2 ob2[QC][H];                                // own-bank operands of the own columns
#pragma unroll
    for (int v = 0; v < H; ++v)
#pragma unroll
      for (int q = 0; q < QC; ++q) ob2[q][v] = 2 * v < t ? own_c(q, v) : make_double2(0.0, 0.0);
    const double p = bw[kMaxLook + t];
    const double a0 = bw[32];
    SX_PROBE(7 + 10 * t);
    double* prow = prowO + (long long)t * ld;
    unsigned int rmask = 0u, qmask = 0u;                // bit u: r was pivot row u (own / previous bank)
#pragma unroll
    for (int u = 0; u < kMaxLook; ++u) {
      if (u < t && sh_r[u] == r) rmask |= 1u << u;
      if (u < spre && sh_rp[u] == r) qmask |= 1u << u;
    }
    if ((rmask | qmask) == 0u) {                        // row r is no pending pivot row: plain chains
#pragma unroll
      for (int v = 0; v < H; ++v) {
        if (spre < kMaxLook && 2 * v >= spre) break;
        const double2 cs = bw2[v];
        double2 a[QC];
#pragma unroll
        for (int q = 0; q < QC; ++q) a[q] = pre_c(q, v);
#pragma unroll
        for (int q = 0; q < QC; ++q) {
          y[q] = __fma_rn(-cs.x, a[q].x, y[q]);
          if (spre == kMaxLook || 2 * v + 1 < spre) y[q] = __fma_rn(-cs.y, a[q].y, y[q]);
        }
      }
#pragma unroll
      for (int v = 0; v < H; ++v) {
        if (2 * v >= t) break;
        const double2 cr = bw2[H + v];
#pragma unroll
        for (int q = 0; q < QC; ++q) {
          y[q] = __fma_rn(-cr.x, ob2[q][v].x, y[q]);
          if (2 * v + 1 < t) y[q] = __fma_rn(-cr.y, ob2[q][v].y, y[q]);
        }
      }
    } else {                                           // row r was a pivot row u: prow_u replaces it
#pragma unroll
      for (int q = 0; q < QC; ++q) {
#pragma unroll
        for (int v = 0; v < H; ++v) {
          const double2 cs = bw2[v];
          const double2 a = 2 * v < spre ? pre_c(q, v) : make_double2(0.0, 0.0);
          if (2 * v < spre) y[q] = ((qmask >> (2 * v)) & 1u) ? a.x : __fma_rn(-cs.x, a.x, y[q]);
          if (2 * v + 1 < spre) y[q] = ((qmask >> (2 * v + 1)) & 1u) ? a.y : __fma_rn(-cs.y, a.y, y[q]);
        }
#pragma unroll
        for (int v = 0; v < H; ++v) {
          const double2 cr = bw2[H + v];
          if (2 * v < t) y[q] = ((rmask >> (2 * v)) & 1u) ? ob2[q][v].x : __fma_rn(-cr.x, ob2[q][v].x, y[q]);
          if (2 * v + 1 < t) y[q] = ((rmask >> (2 * v + 1)) & 1u) ? ob2[q][v].y : __fma_rn(-cr.y, ob2[q][v].y, y[q]);
        }
      }
    }
#ifdef SX_PROBE_DETAIL
    SX_PROBE(8 + 10 * t);
#endif
    best = cand_none();
#pragma unroll
    for (int q = 0; q < QC; ++q) {
      const long long j = jq[q];
      if (j < ld) {
        const double pj = __ddiv_rn(y[q], p);
        own_c_set(q, t, pj);
        prow[j] = pj;
        const double v = __fma_rn(a0, pj, R0s[q * NT + tid]);
        R0s[q * NT + tid] = v;
        if (j < pw && v < -tol_opt) best = cand_min(best, price_cand(s.rule, v, s.c0 + j));  // Step 1 of t+1
      }
    }
    if (gtid == 0) {
      st->rsb[bown][t] = r;
      s.basis[r - 1] = (int)(k + s.c0);
      if (it < s.trace_cap) {
        s.trace_k[it] = (int)(k + s.c0);
        s.trace_r[it] = r;
      }
    }
    ++it;
    r_prev = r;
    p_prev = prow;
#ifdef SX_PROBE_DETAIL
    SX_PROBE(9 + 10 * t);
    best = cluster_min(best, slot, ph, nullptr, 0, false, &sh_r[t], r, piv_mark);   // (+ row r recorded)
    SX_PROBE(10 + 10 * t);
#else
    SX_PROBE(8 + 10 * t);
    best = cluster_min(best, slot, ph, nullptr, 0, false, &sh_r[t], r, piv_mark,   // (+ row r recorded)
                       prb ? prb + 9 + 10 * t : nullptr);
#endif
    ph ^= 1;
    SX_PROBE(11 + 10 * t);
  }
#undef SX_PROBE
#undef SX_TIMER
  // hand-off: own R0 / RHS back to global, the own bank's operands to s.hand[bown] (the next
  // launch's previous bank, read by the same thread positions)
  const int vown = (t + 1) >> 1;
#pragma unroll
  for (int q = 0; q < QC; ++q) {
    if (jq[q] < ld) {
      s.R0[jq[q]] = R0s[q * NT + tid];
      for (int v = 0; v < vown; ++v) hown[((size_t)q * H + v) * G + gtid] = OP[((size_t)q * H + v) * NT + tid];
    }
  }
#pragma unroll
  for (int q = 0; q < QR; ++q) {
    if (iq[q] < rows) {
      s.RHS[iq[q]] = RHSs[q * NT + tid];
      for (int v = 0; v < vown; ++v)
          hown[((size_t)(nqc + q) * H + v) * G + gtid] = OC[((size_t)q * H + v) * NT + tid];
    }
  }
  if (gtid == 0) {
    st->status = status;
    st->it = it;
    st->sb[bown] = t;
    st->go = t > 0;
    st->pend_r = -1;
  }
}

// k_mlook: rank-s look-ahead on P > 1 column parts (ranks, or virtual slabs on one GPU).
// One launch per pivot t of a block on every part, between two exchanges of Step-1 candidates
// carrying their chained columns (k_pack's format [v, k, col[0..m]], ONE allgather per pivot):
//   fold the P headers -> k (lexicographic: identical on every part); the winner's column of the
//   current tableau is in the gathered buffer; ratio test over all rows against the replicated
//   rhs (pivot t-1 applied first) -> r (cluster argmin); colS[.][t] <- the column (replicated);
//   own columns: row r by the chain, prow_t = row / p, R0 <- the next objective row, Step-1
//   candidates -> cluster argmin -> this part's best column kc;
//   the chained column kc of the next tableau (all rows) -> this part's slot for pivot t+1.
// t == -1 (block start): R0 / RHS from T, the part's best column, its raw column -> slot for 0.
// Every part takes the same decisions from the same gathered data, so the pivot sequence, the
// replicated rhs / colS / basis and the status are identical everywhere; each part keeps only
// its own columns of R0 and prowS.  The pass (k_update_s, bank 0, in place) then applies the
// block on every part's slab.  Arithmetic and order are those of k_lookahead (bitwise).
// LL words of the peer-memory exchange (device.cuh XPeers): value x with sequence number q
__device__ __forceinline__ void ll_store(unsigned long long* w, double x, unsigned int q) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  const unsigned long long lo = ((unsigned long long)q << 32) | (b & 0xffffffffull);
  const unsigned long long hi = ((unsigned long long)q << 32) | (b >> 32);
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(w), "l"(lo), "l"(hi) : "memory");
}
// Polls until both words carry sequence number q.  A peer that never publishes (a dead rank)
// must not hang the GPU: after timeout_ns (options.exchange_timeout_ms, default 30 s) the word
// is given up on, the handle's loop is stopped (status kFault, err kErrExchange), the host
// reports SIMPLEX_E_NCCL and latches the handle (every later call but destroy: E_STATE).
__device__ __forceinline__ double ll_load(const unsigned long long* w, unsigned int q, DevState* st,
                                          unsigned long long timeout_ns) {
  unsigned long long lo, hi, t0 = 0;
  for (unsigned int n = 0;; ++n) {
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(w) : "memory");
    if ((unsigned int)(lo >> 32) == q && (unsigned int)(hi >> 32) == q) break;
    __nanosleep(32);
    if ((n & 1023u) == 1023u) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (*(volatile int*)&st->status == kFault) return 0.0;     // another thread gave up already
      if (t0 == 0) {
        t0 = now;
      } else if (now - t0 > timeout_ns) {
        atomicOr(&st->err, kErrExchange);
        st->status = kFault;
        return 0.0;
      }
    }
  }
  return __longlong_as_double((long long)((hi << 32) | (lo & 0xffffffffull)));
}

// One step of the multi-part selection (see k_mlook / k_mblock).  T: the tableau the chains
// start from; own pivots go to chain bank `bown`.  bpre >= 0 (multi-part pipeline): T is the
// tableau BEFORE the previous block, whose pass runs concurrently; its pivots (bank bpre) are
// chained first and R0 / RHS continue from the previous block (the §9e scheme on P parts).
__device__ __forceinline__ void mlook_step(const SlabView& s, const double* __restrict__ T,
                                           const double* __restrict__ xin, double* __restrict__ xout, int nparts,
                                           long long xstride, int t, int S, int bown, int bpre, double tol_opt,
                                           double tol_piv, const XPeers& xp, bool first_step) {
  DevState* st = s.st;
  bool waited = !first_step;                          // the entry arrive still needs its wait
#define MLOOK_RETURN             \
  do {                           \
    if (!waited) cluster_wait(); \
    return;                      \
  } while (0)
  __shared__ int sh_r[kMaxLook];                      // own pivot rows
  __shared__ int sh_rp[kMaxLook];                     // pivot rows of the previous bank
  __shared__ __align__(16) Cand slot[2 * 16];
  extern __shared__ unsigned int piv_mark[];
  const long long gthreads = (long long)gridDim.x * blockDim.x;
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int rows = s.rows;
  const long long ld = s.ld;
  const int w = s.w;
  const int pw = st->pw;
  double* __restrict__ colO = s.colS + bown * kMaxLook;                 // row stride kColS
  double* __restrict__ prowO = s.prowS + (long long)bown * kMaxLook * ld;
  const double* __restrict__ colP = s.colS + (bpre >= 0 ? bpre : 0) * kMaxLook;
  const double* __restrict__ prowP = s.prowS + (long long)(bpre >= 0 ? bpre : 0) * kMaxLook * ld;
  // transposed copies [t][row] of both banks: per-row chain loads coalesce across a warp
  double* __restrict__ colTo = s.colT + (size_t)bown * kMaxLook * rows;
  const double* __restrict__ colTp = s.colT + (size_t)(bpre >= 0 ? bpre : 0) * kMaxLook * rows;
  double* __restrict__ R0 = s.R0;
  double* __restrict__ RHS = s.RHS;
  long long it = st->it;
  if (t < 0 && gtid == 0) st->sb[bown] = 0;          // the block is empty until a pivot is taken
  const bool active = st->status == kRunning && it < st->stop_at;
  if (!active) MLOOK_RETURN;                                // uniform: every CTA reads the same state
  const int spre = bpre >= 0 ? st->sb[bpre] : 0;
  // peer-memory exchange: the slots of this pivot carry sequence number xseq (every part has
  // published as many slots as this one); this launch publishes xseq + 1
  const unsigned int xseq = xp.n > 0 ? (unsigned int)st->xseq : 0u;
  const unsigned long long* xll = xp.n > 0 ? xp.mine + 2 * (long long)(t & 1) * xp.half : nullptr;
  // value e of part q's slot in the gathered buffer of this pivot
  auto xget = [&](int q, long long e) -> double {
    return xll ? ll_load(xll + 2 * ((long long)q * xstride + e), xseq, st, xp.timeout_ns)
               : __ldcg(xin + (long long)q * xstride + e);
  };
  // pivot-row bitmap of both banks (own pivots 0..t-1)
  for (int q = threadIdx.x; q < (rows + 31) / 32; q += blockDim.x) piv_mark[q] = 0u;
  if ((int)threadIdx.x < kMaxLook) {
    sh_rp[threadIdx.x] = (int)threadIdx.x < spre ? st->rsb[bpre][threadIdx.x] : -1;
    sh_r[threadIdx.x] = (int)threadIdx.x < t ? st->rsb[bown][threadIdx.x] : -1;
  }
  __syncthreads();
  if ((int)threadIdx.x < spre) atomicOr(&piv_mark[sh_rp[threadIdx.x] >> 5], 1u << (sh_rp[threadIdx.x] & 31));
  if ((int)threadIdx.x < t) atomicOr(&piv_mark[sh_r[threadIdx.x] >> 5], 1u << (sh_r[threadIdx.x] & 31));
  __syncthreads();
  int ph = 0;
  Cand best = cand_none();
  int r = -1;                                         // pivot row of step t (t >= 0)
  if (t < 0) {
    if (bpre < 0) {
      for (long long j = gtid; j < ld; j += gthreads) {
        const double v = T[j];
        R0[j] = v;
        if (j < pw && v < -tol_opt) best = cand_min(best, price_cand(s.rule, v, s.c0 + j));
      }
      for (long long i = gtid; i < rows; i += gthreads) RHS[i] = T[i * ld + w];
    } else {                                          // R0 continues from the previous block
      for (long long j = gtid; j < pw; j += gthreads) {
        const double v = R0[j];
        if (v < -tol_opt) best = cand_min(best, price_cand(s.rule, v, s.c0 + j));
      }
    }
  } else {
    // Step 1: fold the gathered candidates (every part the same)
    Cand kb = cand_none();
    int q = -1;
    for (int p = 0; p < nparts; ++p) {
      const Cand c{xget(p, 0), __double_as_longlong(xget(p, 1))};
      if (cand_less(c, kb)) { kb = c; q = p; }
    }
    if (kb.idx == LLONG_MAX) {                                                  // optimal
      if (gtid == 0) st->status = kOptimal;
      MLOOK_RETURN;
    }
    const long long k = kb.idx;
    // Step 2 over all rows; the rhs gets the previous pivot first (at t = 0 of a pipelined
    // block: the previous block's last pivot)
    const int r_prev = t > 0 ? st->rsb[bown][t - 1] : spre > 0 ? sh_rp[spre - 1] : -1;
    const double* c_prev = t > 0 ? colTo + (size_t)(t - 1) * rows : colTp + (size_t)(spre > 0 ? spre - 1 : 0) * rows;
    const double pw_prev = r_prev < 0 ? 0.0
                           : __ldcg((t > 0 ? prowO + (long long)(t - 1) * ld : prowP + (long long)(spre - 1) * ld) + w);
    Cand rb = cand_none();
    for (long long i = gtid; i < rows; i += gthreads) {
      double h = RHS[i];
      if (r_prev >= 0) h = (i == r_prev) ? pw_prev : __fma_rn(-c_prev[i], pw_prev, h);
      RHS[i] = h;
      const double x = xget(q, 2 + i);
      colO[i * kColS + t] = x;                         // (row-major: the pass's TMA rows)
      colTo[(size_t)t * rows + i] = x;
      if (i >= 1 && x > tol_piv) {
        int basic = 0;
        if (s.rule) basic = __ldcg(s.basis + i - 1);
        rb = cand_min(rb, ratio_cand(s.rule, __ddiv_rn(h, x), i, basic));
      }
    }
    rb = cluster_min(rb, slot, ph, nullptr, 0, !waited);
    waited = true;
    ph ^= 1;
    if (rb.idx == LLONG_MAX) {                                                  // unbounded
      if (gtid == 0) {
        st->status = kUnbounded;
        st->k = (int)k;
      }
      MLOOK_RETURN;
    }
    if (it >= st->cap) {                                                        // reading c12
      if (gtid == 0) st->status = kIterLimit;
      MLOOK_RETURN;
    }
    r = cand_row(rb.idx);
    const double p = xget(q, 2 + r);
    const double a0 = -xget(q, 2);
    double cr[kMaxLook], cs[kMaxLook];
#pragma unroll
    for (int u = 0; u < kMaxLook; ++u) cs[u] = u < spre ? __ldcg(colP + (long long)r * kColS + u) : 0.0;
#pragma unroll
    for (int u = 0; u < kMaxLook; ++u) cr[u] = u < t ? __ldcg(colO + (long long)r * kColS + u) : 0.0;
    unsigned int rmask = 0u, qmask = 0u;
#pragma unroll
    for (int u = 0; u < kMaxLook; ++u) {
      if (u < t && sh_r[u] == r) rmask |= 1u << u;
      if (u < spre && sh_rp[u] == r) qmask |= 1u << u;
    }
    const double* Tr = T + (long long)r * ld;
    double* prow = prowO + (long long)t * ld;
    for (long long j = gtid; j < ld; j += gthreads) {
      double x = Tr[j];
      double qu[kMaxLook], pu[kMaxLook];
#pragma unroll
      for (int u = 0; u < kMaxLook; ++u) qu[u] = u < spre ? prowP[(long long)u * ld + j] : 0.0;
#pragma unroll
      for (int u = 0; u < kMaxLook; ++u) pu[u] = u < t ? prowO[(long long)u * ld + j] : 0.0;
#pragma unroll
      for (int u = 0; u < kMaxLook; ++u)
        if (u < spre) x = ((qmask >> u) & 1u) ? qu[u] : __fma_rn(-cs[u], qu[u], x);
#pragma unroll
      for (int u = 0; u < kMaxLook; ++u)
        if (u < t) x = ((rmask >> u) & 1u) ? pu[u] : __fma_rn(-cr[u], pu[u], x);
      const double pj = __ddiv_rn(x, p);
      prow[j] = pj;
      const double v = __fma_rn(a0, pj, R0[j]);
      R0[j] = v;
      if (j < pw && v < -tol_opt) best = cand_min(best, price_cand(s.rule, v, s.c0 + j));
    }
    if (gtid == 0) {
      st->rsb[bown][t] = r;
      st->sb[bown] = t + 1;
      s.basis[r - 1] = (int)k;
      if (it < s.trace_cap) {
        s.trace_k[it] = (int)k;
        s.trace_r[it] = r;
      }
      st->it = it + 1;
    }
    if (t + 1 >= S) MLOOK_RETURN;                           // block complete: no candidate needed
  }
  // this part's best column for the next pivot, and that column of the next tableau (pivot t's row
  // r is recorded in sh_r / piv_mark inside the reduction, between its two CTA barriers)
  best = cluster_min(best, slot, ph, nullptr, 0, !waited, t >= 0 ? &sh_r[t] : nullptr, r, piv_mark);
  waited = true;
  // slot destinations: xout (NCCL send buffer or the one-GPU gather buffer), or buffer (t+1)&1
  // of every rank's gather buffer (peer memory)
  const long long off = 2 * ((long long)((t + 1) & 1) * xp.half + (long long)xp.part * xstride);   // LL words
  if (blockIdx.x == 0 && threadIdx.x < (xp.n > 0 ? xp.n : 1)) {
    if (xp.n > 0) {
      ll_store(xp.x[threadIdx.x] + off, best.v, xseq + 1);
      ll_store(xp.x[threadIdx.x] + off + 2, __longlong_as_double(best.idx), xseq + 1);
    } else {
      xout[0] = best.v;
      xout[1] = __longlong_as_double(best.idx);
    }
  }
  if (best.idx != LLONG_MAX) {
    const long long kc = best.idx - s.c0;
    const int nu = t + 1;                             // own chains applied: pivots 0..t
    double qk[kMaxLook], pk[kMaxLook];
#pragma unroll
    for (int u = 0; u < kMaxLook; ++u) qk[u] = u < spre ? __ldcg(prowP + (long long)u * ld + kc) : 0.0;
#pragma unroll
    for (int u = 0; u < kMaxLook; ++u) pk[u] = u < nu ? __ldcg(prowO + (long long)u * ld + kc) : 0.0;
    for (long long i = gtid; i < rows; i += gthreads) {
      double x = T[i * ld + kc];
      const bool marked = (piv_mark[i >> 5] >> (i & 31)) & 1u;
#pragma unroll
      for (int u = 0; u < kMaxLook; ++u) {
        if (u < spre) {
          const double cq = colTp[(size_t)u * rows + i];
          x = (marked && i == sh_rp[u]) ? qk[u] : __fma_rn(-cq, qk[u], x);
        }
      }
#pragma unroll
      for (int u = 0; u < kMaxLook; ++u) {
        if (u < nu) {
          const double cu = colTo[(size_t)u * rows + i];
          x = (marked && i == sh_r[u]) ? pk[u] : __fma_rn(-cu, pk[u], x);
        }
      }
      if (xp.n == 0) {
        xout[2 + i] = x;
      } else {
        for (int d = 0; d < xp.n; ++d) ll_store(xp.x[d] + off + 2 * (2 + i), x, xseq + 1);   // NVLink
      }
    }
  }
  if (xp.n > 0 && gtid == 0) st->xseq = xseq + 1;
}
#undef MLOOK_RETURN

// One pivot t of a block per launch (t = -1: block start); the exchange between launches is
// the NCCL allgather, plain stores (virtual slabs) or the peer-memory LL words.
__global__ void __launch_bounds__(kLookThreads) k_mlook(SlabView s, const double* __restrict__ xin,
                                                       double* __restrict__ xout, int nparts, long long xstride,
                                                       int t, int S, double tol_opt, double tol_piv, XPeers xp) {
  cluster_arrive_relaxed();                           // (waited for in the first cluster_min)
  mlook_step(s, s.T, xin, xout, nparts, xstride, t, S, 0, -1, tol_opt, tol_piv, xp, true);
}

// The whole block's selection in ONE launch per part (peer-memory exchange only): the steps
// t = -1 .. S-1 of k_mlook back to back, each part polling the other parts' LL words of pivot t
// inside the kernel — compute and exchange fused, no launch per pivot.  A cluster barrier between
// steps publishes the step's DevState writes (status, it, xseq, rsb) to every CTA.  Every part
// of the exchange must be resident at once (ranks: one per GPU; virtual slabs: one stream each).
__global__ void __launch_bounds__(kLookThreads) k_mblock(SlabView s, const double* __restrict__ T, int nparts,
                                                        long long xstride, int S, int bown, int bpre, double tol_opt,
                                                        double tol_piv, XPeers xp) {
  pdl_launch_dependents();            // (multi-part pipeline: the next part's selection and the slab
                                      //  passes are launched behind this one without waiting)
  cluster_arrive_relaxed();                           // (waited for in the first cluster_min)
  for (int t = -1; t < S; ++t) {
    if (t >= 0) cluster_barrier();
    mlook_step(s, T, nullptr, nullptr, nparts, xstride, t, S, bown, bpre, tol_opt, tol_piv, xp, t < 0);
  }
}

// k_update_s: the rank-s pass, TMA in and TMA out.  CTA b owns column chunk c = b mod nc (cw
// doubles, one double2 per consumer thread) and rows g, g+Gr, g+2Gr, ... (g = b div nc), so
// all CTAs sweep Gr consecutive rows at a time: the chip-wide HBM front stays contiguous.
// One CTA per SM, three roles over a K-stage shared-memory ring of R row segments:
//   loader warp    streams each row segment T[i][chunk] and the row's pivot-column entries
//                  colS[i][bank][0..15] into a free stage (cp.async.bulk + mbarrier complete_tx);
//   8 consumer warps hold prow_u[j] (u < s) in registers and apply the chain
//                  x <- fma(-col_u[i], prow_u[j], x), u = 0 .. s-1 (the oracle's order and
//                  rounding), writing the result back into the stage;
//   storer warp    bulk-stores every computed stage (cp.async.bulk global <- shared, L2
//                  evict_first) and frees the slot once the store has read it.
// Measured (scripts/ubench_pass.cu, 8000^2 geometry): 304 us per rank-16 pass on 132 SMs,
// above the device-to-device copy rate, where register stores from the consumers reached
// 433 us.  The <= s pivot rows are not stored by the stream (bitmap) but written at the end
// from their last normalized value prow_u, chained over the later pivots of the block.
//
// src == dst: in place.  src != dst (software pipeline): reads the block's
// starting tableau, writes the next buffer — also when the block is empty (a copy) — and does
// NOT wait on the look-ahead kernel launched just before it (that one selects the NEXT block,
// from src, concurrently); everything this pass reads was complete before that launch began.
__device__ __forceinline__ void bulk_s2g_hint(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int S, int R, int K>
__device__ __forceinline__ void update_s_body(const SlabView& s, const double* __restrict__ src, double* dst,
                                              int bank, int nc, int Gr, int cw) {
  constexpr int SC = S > kMaxLook ? kColS : kMaxLook;                // pivot-column entries staged per row
  const DevState* st = s.st;
  // S > 16: the pair schedule — bank 0 then bank 1 (chained when bank 0 is full), bank == 0
  const int se = S > kMaxLook ? st->sb[0] + (st->sb[0] >= kMaxLook ? st->sb[1] : 0) : st->sb[bank];
  if (se == 0 && src == dst) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sT = reinterpret_cast<double*>(smem_raw);                 // [K][R][cw]
  double* sC = sT + (size_t)K * R * cw;                              // [K][R][SC]
  unsigned int* mark = reinterpret_cast<unsigned int*>(sC + (size_t)K * R * SC);
  __shared__ __align__(8) uint64_t full[K];    // stage loaded (tx bytes)
  __shared__ __align__(8) uint64_t comp[K];    // stage computed (8 consumer warps)
  __shared__ __align__(8) uint64_t empty[K];   // stage stored and free (storer)
  __shared__ int sh_r[S];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int rows = s.rows;
  const long long ld = s.ld;
  const int nwords = (rows + 31) >> 5;
  for (int i = tid; i < nwords; i += blockDim.x) mark[i] = 0u;
  if (tid < S) sh_r[tid] = tid < se ? (&st->rsb[0][0])[bank * kMaxLook + tid] : -1;   // rsb[2][16] flat
  if (tid == 0) {
    for (int k = 0; k < K; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&comp[k], kThreads / 32);
      mbar_init(&empty[k], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (tid < se) atomicOr(&mark[sh_r[tid] >> 5], 1u << (sh_r[tid] & 31));
  __syncthreads();

  const int c = blockIdx.x % nc;
  const int g = blockIdx.x / nc;
  const long long j0 = (long long)c * cw;
  const int jn = (int)min((long long)cw, ld - j0);                    // doubles in this chunk
  const int nr = rows > g ? (rows - g + Gr - 1) / Gr : 0;             // rows of this CTA
  const int nst = (nr + R - 1) / R;

  if (warp == kThreads / 32) {                                        // ---- loader warp
    if (lane == 0) {
      const uint64_t pol = l2_evict_first();
      for (int n = 0; n < nst; ++n) {
        const int k = n % K;
        if (n >= K) mbar_wait(&empty[k], ((n / K) - 1) & 1);
        const int rin = min(R, nr - n * R);
        mbar_arrive_expect_tx(&full[k], (uint32_t)(rin * (jn + SC) * sizeof(double)));
        for (int rr = 0; rr < rin; ++rr) {
          const long long i = g + (long long)(n * R + rr) * Gr;
          bulk_g2s_hint(sT + ((size_t)k * R + rr) * cw, src + i * ld + j0, (uint32_t)(jn * sizeof(double)), &full[k],
                        pol);
          bulk_g2s(sC + ((size_t)k * R + rr) * SC, s.colS + i * kColS + bank * kMaxLook,
                   (uint32_t)(SC * sizeof(double)), &full[k]);
        }
      }
    }
    return;
  }
  if (warp == kThreads / 32 + 1) {                                    // ---- storer warp
    if (lane == 0) {
      const uint64_t pol = l2_evict_first();
      for (int m = 0; m < nst; ++m) {
        const int k = m % K;
        mbar_wait(&comp[k], (m / K) & 1);
        const int rin = min(R, nr - m * R);
        for (int rr = 0; rr < rin; ++rr) {
          const int i = g + (m * R + rr) * Gr;
          if (!((mark[i >> 5] >> (i & 31)) & 1u))
            bulk_s2g_hint(dst + (long long)i * ld + j0, sT + ((size_t)k * R + rr) * cw, (uint32_t)(jn * sizeof(double)),
                          pol);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (m >= 1) {                                  // the previous stage's store has read its slot
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          mbar_arrive(&empty[(m - 1) % K]);
        }
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // writes done before the CTA exits
    }
    return;
  }
  // ---- consumer warps
  const int jl = 2 * tid;
  const bool act = jl < jn;
  const long long j = j0 + jl;
  double2 pr[S];
#pragma unroll
  for (int u = 0; u < S; ++u)
    pr[u] = (act && u < se) ? *reinterpret_cast<const double2*>(s.prowS + (long long)(bank * kMaxLook + u) * ld + j)
                            : make_double2(0.0, 0.0);
  for (int n = 0; n < nst; ++n) {
    const int k = n % K;
    mbar_wait(&full[k], (n / K) & 1);
    const int rin = min(R, nr - n * R);
    if (S > kMaxLook && se == S && rin == R && act) {
      // pair schedule, full block, full stage: as below, the pivot-column entries loaded per
      // pair of pivots (the register file holds the 32 prow_u double2 already)
      double2 v[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) v[rr] = *reinterpret_cast<const double2*>(sT + ((size_t)k * R + rr) * cw + jl);
#pragma unroll
      for (int h = 0; h < S / 2; ++h) {
        double2 ca[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) ca[rr] = reinterpret_cast<const double2*>(sC + ((size_t)k * R + rr) * SC)[h];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          v[rr].x = __fma_rn(-ca[rr].x, pr[2 * h].x, v[rr].x);
          v[rr].y = __fma_rn(-ca[rr].x, pr[2 * h].y, v[rr].y);
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          v[rr].x = __fma_rn(-ca[rr].y, pr[2 * h + 1].x, v[rr].x);
          v[rr].y = __fma_rn(-ca[rr].y, pr[2 * h + 1].y, v[rr].y);
        }
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) *reinterpret_cast<double2*>(sT + ((size_t)k * R + rr) * cw + jl) = v[rr];
    } else if (S <= kMaxLook && se == S && rin == R && act) {
      // full block, full stage: the R rows' 2R chains interleave (independent FMAs); the
      // stage's pivot-column entries are loaded ahead of the chains
      double2 v[R];
      double2 ca[R][S / 2];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        v[rr] = *reinterpret_cast<const double2*>(sT + ((size_t)k * R + rr) * cw + jl);
#pragma unroll
        for (int h = 0; h < S / 2; ++h)
          ca[rr][h] = reinterpret_cast<const double2*>(sC + ((size_t)k * R + rr) * SC)[h];
      }
#pragma unroll
      for (int h = 0; h < S / 2; ++h) {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          v[rr].x = __fma_rn(-ca[rr][h].x, pr[2 * h].x, v[rr].x);
          v[rr].y = __fma_rn(-ca[rr][h].x, pr[2 * h].y, v[rr].y);
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          v[rr].x = __fma_rn(-ca[rr][h].y, pr[2 * h + 1].x, v[rr].x);
          v[rr].y = __fma_rn(-ca[rr][h].y, pr[2 * h + 1].y, v[rr].y);
        }
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) *reinterpret_cast<double2*>(sT + ((size_t)k * R + rr) * cw + jl) = v[rr];
    } else if (act) {
      for (int rr = 0; rr < rin; ++rr) {
        double2 v = *reinterpret_cast<const double2*>(sT + ((size_t)k * R + rr) * cw + jl);
        const double* cc = sC + ((size_t)k * R + rr) * SC;
#pragma unroll
        for (int u = 0; u < S; ++u) {
          if (u < se) {
            const double a = -cc[u];
            v.x = __fma_rn(a, pr[u].x, v.x);
            v.y = __fma_rn(a, pr[u].y, v.y);
          }
        }
        *reinterpret_cast<double2*>(sT + ((size_t)k * R + rr) * cw + jl) = v;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> bulk store
    __syncwarp();
    if (lane == 0) mbar_arrive(&comp[k]);
  }
  if (!act) return;
  // pivot rows of this chunk owned by this row group: from the LAST time each was the
  // pivot row, chained over the later pivots of the block
#pragma unroll
  for (int u = 0; u < S; ++u) {
    if (u >= se) break;
    const int r = sh_r[u];
    if (r % Gr != g) continue;
    bool last = true;
    for (int u2 = u + 1; u2 < se; ++u2) last &= (sh_r[u2] != r);
    if (!last) continue;
    double2 v = pr[u];
    const double* cr = s.colS + (long long)r * kColS + bank * kMaxLook;
#pragma unroll
    for (int u2 = 0; u2 < S; ++u2) {
      if (u2 > u && u2 < se) {
        const double a = -cr[u2];
        v.x = __fma_rn(a, pr[u2].x, v.x);
        v.y = __fma_rn(a, pr[u2].y, v.y);
      }
    }
    *reinterpret_cast<double2*>(dst + (long long)r * ld + j) = v;
  }
}

template <int S, int R, int K>
__global__ void __launch_bounds__(kThreads + 64, 1) k_update_s(SlabView s, const double* __restrict__ src,
                                                               double* dst, int bank, int nc, int Gr, int cw) {
  pdl_launch_dependents();
  if (src == dst) pdl_wait();
  DevState* st = s.st;
  const bool timed = s.time_pass && (src != dst || st->sb[bank] > 0);
  if (timed && threadIdx.x == 0) atomicMin(&st->pass_t0, globaltimer());
  update_s_body<S, R, K>(s, src, dst, bank, nc, Gr, cw);
  if (!timed) return;
  __syncthreads();                                    // every role of this CTA is done
  if (threadIdx.x == 0) {
    atomicMax(&st->pass_t1, globaltimer());
    __threadfence();
    if (atomicAdd(&st->pass_done, 1u) == gridDim.x - 1) {   // last CTA: one launch duration
      __threadfence();
      const unsigned long long t0 = atomicAdd(&st->pass_t0, 0ull), t1 = atomicAdd(&st->pass_t1, 0ull);
      st->pass_ns += (double)(t1 - t0);
      st->pass_n += 1;
      st->pass_t0 = ~0ull;
      st->pass_t1 = 0ull;
      st->pass_done = 0u;
    }
  }
}

// ------------------------------------------------------------------ small tableaux: one CTA
// k_solve_small: the WHOLE solve of a tableau that fits in one SM's shared memory (64x64:
// 65 x 129 doubles = 67 KB) in ONE launch of ONE CTA — the latency path for the small LPs
// where "the communication and the reductions dominate".  The tableau is
// loaded once, every pivot is Steps 1-3 on shared memory, and the result is
// written back once.  Three CTA barriers per pivot:
//   [ratio]   Step 2 on column k: rows with T[i][k] > tol_piv, q = T[i][rhs] / T[i][k] (IEEE
//             division), ratio_cand -> warp argmin -> one slot per warp;          barrier 1
//   [stage]   every warp folds the slots itself (no second barrier) -> r, or UNBOUNDED; the cap
//             check (reading c12); colv[i] = T[i][k], prow[j] = T[r][j] / p (IEEE division)
//             into separate buffers (no in-place race);                            barrier 2
//   [update]  T[i][j] = fma(-colv[i], prow[j], T[i][j]) for i != r, T[r][j] = prow[j] — the
//             oracle's c8 arithmetic — with warps owning rows and lanes owning columns; warp 0
//             owns row 0 and prices it as it writes it (Step 1 for the next pivot: warp argmin
//             of price_cand, Dantzig (v, j) / Bland (0, j)) -> k, or OPTIMAL;     barrier 3
// Requires one column part and no artificial columns (the engine checks).
constexpr int kSmallMaxQ = 8;                        // tableau width <= 256 columns
template <int NT, int NQ>
__global__ void __launch_bounds__(NT, 1) k_solve_small(SlabView s, long long stop_at, double tol_opt, double tol_piv,
                                                       SmallLP io) {
  constexpr int NW = NT / 32;                        // NQ: columns per lane (cols <= 32 * NQ)
  extern __shared__ __align__(16) double smem[];
  const int rows = s.rows, m = rows - 1;
  const int cols = s.w + 1;                          // logical columns incl. the rhs (local column w)
  const int rhs = s.w;
  double* T = smem;                                  // [rows][cols]
  double* prow = T + (size_t)rows * cols;            // [cols]
  double* colv = prow + cols;                        // [rows]
  int* basis = reinterpret_cast<int*>(colv + rows);  // [m]
  __shared__ Cand slot[NW];
  __shared__ Cand sh_k;                              // Step-1 result for the next pivot
  DevState* st = s.st;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  long long it;
  int status;
  if (io.A) {
    // LP mode (simplex_solve_lp): Table I is built right here from the caller's
    // A, b, c — the slack basis, row 0 = -c, rows i = [a_i, e_i, b_i] (k_build's values; c10: no
    // Z column) — with k_build's validation (finite inputs, b >= 0: a small handle has no Phase I)
    const long long n = io.n;
    __shared__ unsigned int sh_err;
    if (tid == 0) sh_err = 0u;
    __syncthreads();
    unsigned int err = 0u;
    for (int i = wid; i < rows; i += NW)
      for (int j = lane; j < cols; j += 32) {
        double v;
        if (j == rhs) {
          v = i == 0 ? 0.0 : io.b[i - 1];
          if (i > 0 && !isfinite(v)) err |= kErrNonFinite;
          if (i > 0 && v < 0.0) err |= kErrNegRhs;
        } else if (j < n) {
          v = i == 0 ? io.c[j] : io.A[(long long)(i - 1) * n + j];
          if (!isfinite(v)) err |= kErrNonFinite;
          if (i == 0) v = -v;
        } else {
          v = (i >= 1 && j - n == i - 1) ? 1.0 : 0.0;
        }
        T[(size_t)i * cols + j] = v;
      }
    for (int i = tid; i < m; i += NT) basis[i] = (int)(n + i);
    if (err) atomicOr(&sh_err, err);
    it = 0;
    status = kRunning;
    __syncthreads();
    if (sh_err) {                                      // invalid input: the built tableau, no pivots
      status = kFault;
      if (tid == 0) st->err = sh_err;
    }
    if (tid == 0) {
      st->it = 0;
      st->stop_at = LLONG_MAX;
      st->status = kRunning;
      st->phase = 2;
      st->pw = s.w;
      st->drive_next = 0;
      st->sb[0] = st->sb[1] = 0;
      if (!sh_err) st->err = 0u;
    }
  } else {
    const int pend = st->pend_r;                     // a deferred pivot row of another path
    for (int i = wid; i < rows; i += NW) {
      const double* src = (i == pend) ? s.rownorm : s.T + (long long)i * s.ld;
      for (int j = lane; j < cols; j += 32) T[(size_t)i * cols + j] = src[j];
    }
    for (int i = tid; i < m; i += NT) basis[i] = s.basis[i];
    it = st->it;
    status = st->status;
  }
  const long long cap = st->cap;
  const int pw = io.A ? s.w : st->pw;
  const int rule = s.rule;
  __syncthreads();
  if (wid == 0) {                                    // Step 1 on the starting row 0
    Cand c = cand_none();
    for (int j = lane; j < pw; j += 32) {
      const double v = T[j];
      if (v < -tol_opt) c = cand_min(c, price_cand(rule, v, j));
    }
    c = warp_min(c);
    if (lane == 0) sh_k = c;
  }
  __syncthreads();
  while (status == kRunning && it < stop_at) {
    const Cand kc = sh_k;
    if (kc.idx == LLONG_MAX) {
      status = kOptimal;
      break;
    }
    const int k = (int)kc.idx;
    // Step 2 — ratio test over rows 1..m
    Cand q = cand_none();
    for (int i = 1 + tid; i <= m; i += NT) {
      const double a = T[(size_t)i * cols + k];
      if (a > tol_piv) q = cand_min(q, ratio_cand(rule, __ddiv_rn(T[(size_t)i * cols + rhs], a), i, basis[i - 1]));
    }
    if (32 * wid + 1 <= m) q = warp_min(q);           // (warps without rows keep "none")
    if (lane == 0) slot[wid] = q;
    __syncthreads();                                                      // barrier 1
    q = warp_min(lane < NW ? slot[lane] : cand_none());
    if (q.idx == LLONG_MAX) {
      status = kUnbounded;
      break;
    }
    if (it == cap) {
      status = kIterLimit;
      break;
    }
    const int r = cand_row(q.idx);
    // Step 3 — pivot column snapshot and normalized pivot row, then the rank-1 update
    const double p = T[(size_t)r * cols + k];
    for (int i = tid; i < rows; i += NT) colv[i] = T[(size_t)i * cols + k];
    for (int j = tid; j < cols; j += NT) prow[j] = __ddiv_rn(T[(size_t)r * cols + j], p);
    if (tid == 0) {
      basis[r - 1] = k;
      if (it < s.trace_cap) {
        s.trace_k[it] = (int)s.c0 + k;
        s.trace_r[it] = r;
      }
    }
    __syncthreads();                                                      // barrier 2
    // lane owns columns j = lane + 32 q: its prow values stay in registers for every row; each
    // row is NQ independent loads, then NQ FMAs, then NQ stores (no load waits behind a store)
    double pr[NQ];
#pragma unroll
    for (int q2 = 0; q2 < NQ; ++q2) {
      const int j = lane + 32 * q2;
      pr[q2] = j < cols ? prow[j] : 0.0;
    }
    for (int i = wid; i < rows; i += NW) {
      double* Ti = T + (size_t)i * cols;
      double v[NQ];
#pragma unroll
      for (int q2 = 0; q2 < NQ; ++q2) {
        const int j = lane + 32 * q2;
        v[q2] = j < cols ? Ti[j] : 0.0;
      }
      const double a = -colv[i];
#pragma unroll
      for (int q2 = 0; q2 < NQ; ++q2) v[q2] = (i == r) ? pr[q2] : __fma_rn(a, pr[q2], v[q2]);
#pragma unroll
      for (int q2 = 0; q2 < NQ; ++q2) {
        const int j = lane + 32 * q2;
        if (j < cols) Ti[j] = v[q2];
      }
      if (i == 0) {                                  // warp 0: Step 1 of the next pivot on the new row 0
        Cand c = cand_none();
#pragma unroll
        for (int q2 = 0; q2 < NQ; ++q2) {
          const int j = lane + 32 * q2;
          if (j < pw && v[q2] < -tol_opt) c = cand_min(c, price_cand(rule, v[q2], j));
        }
        c = warp_min(c);
        if (lane == 0) sh_k = c;
      }
    }
    ++it;
    __syncthreads();                                                      // barrier 3
  }
  // write back: tableau (logical columns; padding untouched = zero), basis, loop state
  __syncthreads();
  for (int i = wid; i < rows; i += NW) {
    double* dst = s.T + (long long)i * s.ld;
    for (int j = lane; j < cols; j += 32) dst[j] = T[(size_t)i * cols + j];
  }
  for (int i = tid; i < m; i += NT) s.basis[i] = basis[i];
  if (tid == 0) {
    st->it = it;
    st->status = status == kFault ? kRunning : status;
    st->pend_r = -1;
    st->go = 0;
  }
  if (io.A) {
    // LP mode: the solution too (k_extract's definition): x_j = rhs of the row
    // where x_j is basic (0 if non-basic), y_i = T[0][n+i], objective = T[0][rhs]
    const long long n = io.n;
    if (io.x) {
      for (long long j = tid; j < n; j += NT) io.x[j] = 0.0;
      __syncthreads();
      for (int i = tid; i < m; i += NT)
        if (basis[i] < n) io.x[basis[i]] = T[(size_t)(i + 1) * cols + rhs];
    }
    if (io.y)
      for (int i = tid; i < m; i += NT) io.y[i] = T[n + i];
    if (tid == 0) {
      io.res[0] = T[rhs];
      io.res[1] = (double)(status == kFault ? kRunning : status);
      io.res[2] = (double)it;
      io.res[3] = (double)st->err;
    }
  }
}

size_t small_smem_bytes(int rows, int w) {
  const size_t cols = (size_t)w + 1;
  if (cols > 32 * (size_t)kSmallMaxQ) return ~(size_t)0;    // wider than one warp's columns: no
  return ((size_t)rows * cols + cols + (size_t)rows) * sizeof(double) + (size_t)(rows - 1) * sizeof(int);
}

// Largest dynamic shared memory one CTA of k_solve_small may use on this device (0: unusable).
size_t small_smem_max() {
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return 0;
  const size_t statics = 4096;                       // block_min scratch + loop state (static smem)
  return optin > (int)statics ? (size_t)optin - statics : 0;
}

template <int NT, int NQ>
static cudaError_t launch_small_nt(const SlabView& s, long long stop_at, double tol_opt, double tol_piv,
                                   cudaStream_t st, const SmallLP& io) {
  static size_t set = 0;                             // opt-in size already granted (per instantiation)
  const size_t smem = small_smem_bytes(s.rows, s.w);
  if (smem > set) {
    cudaError_t e = cudaFuncSetAttribute(k_solve_small<NT, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)small_smem_max());
    if (e != cudaSuccess) return e;
    set = small_smem_max();
  }
  k_solve_small<NT, NQ><<<1, NT, smem, st>>>(s, stop_at, tol_opt, tol_piv, io);
  return cudaGetLastError();
}

template <int NQ>
static cudaError_t launch_small_q(int nt, const SlabView& s, long long stop_at, double tol_opt, double tol_piv,
                                  cudaStream_t st, const SmallLP& io) {
  if (nt >= 1024) return launch_small_nt<1024, NQ>(s, stop_at, tol_opt, tol_piv, st, io);
  if (nt >= 512) return launch_small_nt<512, NQ>(s, stop_at, tol_opt, tol_piv, st, io);
  return launch_small_nt<256, NQ>(s, stop_at, tol_opt, tol_piv, st, io);
}

// 512 threads per CTA (measured, scripts/small_probe.py: 64x64 3.5 us/pivot vs 4.4 at 256 and
// 6.4 at 128; 1024 no faster); 4 or 8 columns per lane
cudaError_t launch_solve_small(const SlabView& s, long long stop_at, double tol_opt, double tol_piv,
                               cudaStream_t st, const SmallLP& io) {
  int nt = 512;
  if (const char* e = experiment_env("SIMPLEX_SMALL_THREADS")) nt = std::atoi(e);
  if (s.w + 1 > 32 * kSmallMaxQ) return cudaErrorInvalidValue;
  // columns per lane: the smallest instantiated NQ >= cols / 32 (64^2: 129 columns -> 5, so no lane
  // carries predicated-off columns through the update)
  const int q = (s.w + 1 + 31) / 32;
  if (q <= 2) return launch_small_q<2>(nt, s, stop_at, tol_opt, tol_piv, st, io);
  if (q <= 3) return launch_small_q<3>(nt, s, stop_at, tol_opt, tol_piv, st, io);
  if (q <= 4) return launch_small_q<4>(nt, s, stop_at, tol_opt, tol_piv, st, io);
  if (q <= 5) return launch_small_q<5>(nt, s, stop_at, tol_opt, tol_piv, st, io);
  if (q <= 6) return launch_small_q<6>(nt, s, stop_at, tol_opt, tol_piv, st, io);
  return launch_small_q<kSmallMaxQ>(nt, s, stop_at, tol_opt, tol_piv, st, io);
}

// ------------------------------------------------------------------ flush / extract / hash
__global__ void __launch_bounds__(1024) k_flush(SlabView s) {
  const int pend = s.st->pend_r;
  if (pend < 0) return;
  double* dst = s.T + (long long)pend * s.ld;
  for (long long j = threadIdx.x; j < s.ld; j += blockDim.x) dst[j] = s.rownorm[j];
  __syncthreads();
  if (threadIdx.x == 0) s.st->pend_r = -1;
}

// x (n, pre-zeroed) from the replicated basis + rhs; y entries of this slab's slack
// columns (y pre-zeroed; other ranks fill theirs); objective T[0][W-1].
__global__ void k_extract(SlabView s, long long n, double* x, double* y, double* obj) {
  const int m = s.rows - 1;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m + s.w;
       t += (long long)gridDim.x * blockDim.x) {
    if (t < m) {
      const int jb = s.basis[t];
      if (x && jb < n) x[jb] = s.T[(t + 1) * s.ld + s.w];
    } else {
      const long long jl = t - m;
      const long long g = s.c0 + jl;
      if (y && g >= n && g < n + m) y[g - n] = s.T[jl];
    }
  }
  if (obj && blockIdx.x == 0 && threadIdx.x == 0) *obj = s.T[s.w];
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(kThreads) k_hash(SlabView s, long long Wg, int include_rhs,
                                                   unsigned long long* out) {
  const long long cols = s.w + 1;
  const long long total = (long long)s.rows * cols;
  unsigned long long acc = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / cols;
    const long long jl = e - i * cols;
    if (jl == s.w && !include_rhs) continue;
    const long long g = (jl == s.w) ? Wg - 1 : s.c0 + jl;
    double v = s.T[i * s.ld + jl];
    if (i == s.st->pend_r) v = s.rownorm[jl];
    unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    if (bits == 0x8000000000000000ULL) bits = 0;
    const unsigned long long ge = (unsigned long long)(i * Wg + g);
    acc += mix64(bits ^ (ge * 0x9E3779B97F4A7C15ULL + 0xD1B54A32D192ED03ULL));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

__global__ void k_set_stop(DevState* st, long long stop_at) { st->stop_at = stop_at; }

// ------------------------------------------------------------------ launchers
#define SX_CHECK_LAUNCH() return cudaGetLastError()

cudaError_t launch_set_stop(DevState* st, long long stop_at, cudaStream_t s) {
  k_set_stop<<<1, 1, 0, s>>>(st, stop_at);
  SX_CHECK_LAUNCH();
}

cudaError_t launch_build(const SlabView& s, const double* b, long long n, cudaStream_t st, int sms) {
  const long long total = (long long)s.rows * (s.ld >> 1);
  long long g = (total + kThreads - 1) / kThreads;
  if (g > (long long)sms * 16) g = (long long)sms * 16;
  k_build<<<(int)g, kThreads, 0, st>>>(s, b, n);
  SX_CHECK_LAUNCH();
}

cudaError_t launch_init_state(const SlabView& s, long long n, long long cap, cudaStream_t st) {
  int g = (s.rows + 255) / 256;
  if (g > 1024) g = 1024;
  k_init_state<<<g, 256, 0, st>>>(s, n, cap);
  SX_CHECK_LAUNCH();
}

cudaError_t launch_price0(const SlabView& s, double tol_opt, cudaStream_t st) {
  const long long half = s.ld >> 1;
  k_price0<<<(int)((half + kThreads - 1) / kThreads), kThreads, 0, st>>>(s, tol_opt);
  SX_CHECK_LAUNCH();
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_ex(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, bool pdl,
                             Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

cudaError_t launch_pack(const SlabView& s, double* send, int grid, cudaStream_t st, bool pdl) {
  return launch_ex(k_pack, grid, kThreads, 0, st, pdl, s, send);
}

cudaError_t launch_select(const SlabView& s, const XView& x, double tol_piv, int grid, cudaStream_t st, bool pdl) {
  return launch_ex(k_select, grid, kThreads, 0, st, pdl, s, x, tol_piv);
}

cudaError_t update_occupancy(int* blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_update<kUpdateRows>, kThreads, 0);
}

cudaError_t launch_update(const SlabView& s, int q, double tol_opt, int grid, cudaStream_t st, bool pdl) {
  return launch_ex(k_update<kUpdateRows>, grid, kThreads, 0, st, pdl, s, q, tol_opt);
}

static cudaLaunchConfig_t lookahead_config(int cluster, size_t smem, cudaStream_t st, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster);
  cfg.blockDim = dim3(kLookThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

// Largest cluster (16, else 8, 4, 2, 1 CTAs) the device can co-schedule for k_lookahead.
int lookahead_cluster_size() {
  cudaFuncSetAttribute(k_lookahead, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_lookahead, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLookCacheMax);
  cudaFuncSetAttribute(k_mlook, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* e = experiment_env("SIMPLEX_LOOK_CLUSTER");   // experiment hook: cap the cluster size
  const int cmax = e ? std::atoi(e) : 16;
  for (int c : {16, 8, 4, 2, 1}) {
    if (c > cmax) continue;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = lookahead_config(c, 4096, nullptr, attr);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_lookahead, &cfg) == cudaSuccess && n >= 1) return c;
    cudaGetLastError();
  }
  return 0;
}

cudaError_t launch_mlook(const SlabView& s, const double* xin, double* xout, int nparts, long long xstride, int t,
                         int S, double tol_opt, double tol_piv, int cluster, const XPeers& xp, cudaStream_t st) {
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = lookahead_config(cluster, (size_t)((s.rows + 31) / 32) * sizeof(unsigned int), st, attr);
  return cudaLaunchKernelEx(&cfg, k_mlook, s, xin, xout, nparts, xstride, t, S, tol_opt, tol_piv, xp);
}

cudaError_t launch_mblock(const SlabView& s, const double* T, int nparts, long long xstride, int S, int bown,
                          int bpre, double tol_opt, double tol_piv, int cluster, const XPeers& xp, cudaStream_t st,
                          bool pdl) {
  cudaLaunchAttribute attr[2];
  cudaLaunchConfig_t cfg = lookahead_config(cluster, (size_t)((s.rows + 31) / 32) * sizeof(unsigned int), st, attr);
  if (pdl) {
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 2;
  }
  return cudaLaunchKernelEx(&cfg, k_mblock, s, T, nparts, xstride, S, bown, bpre, tol_opt, tol_piv, xp);
}

// Clusters of `cluster` CTAs of k_mblock that can be resident at once (0 on error).
int mblock_max_clusters(int cluster, int rows) {
  cudaFuncSetAttribute(k_mblock, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = lookahead_config(cluster, (size_t)((rows + 31) / 32) * sizeof(unsigned int), nullptr, attr);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_mblock, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// Shared memory of k_lookahead: the pivot-row bitmap, plus (nqc > 0) the previous bank's chain
// operands of every thread's columns and rows.  0 if that cache does not fit.
size_t lookahead_smem(const SlabView& s, int cluster, bool cache, int* nqc, int* nqr) {
  const long long gthreads = (long long)cluster * kLookThreads;
  const size_t mark = (size_t)(((s.rows + 31) / 32 + 3) & ~3) * sizeof(unsigned int);
  *nqc = (int)((s.ld + gthreads - 1) / gthreads);
  *nqr = (int)((s.rows + gthreads - 1) / gthreads);
  const size_t c = (size_t)kMaxLook * sizeof(double) * kLookThreads * (*nqc + *nqr);
  if (cache && mark + c <= kLookCacheMax) return mark + c;
  *nqc = *nqr = 0;
  return mark;
}

// k_look2 instantiations: (own columns QC, own rows QR per thread); a slab takes the first that
// covers its (nqc, nqr) and fits in shared memory WITH the previous bank (the pipelined
// launches), else k_lookahead.  Measured (round 2b, pipelined blocks): 1000^2
// 110-118 us (k_lookahead ~135), 2000^2 115-121 (134), 4000^2 157-166 (166); with the own bank in
// the hand-off slots (the only way 8000^2 fits; built, measured, removed) 388 us against
// k_lookahead's 343 — so 8000^2 and larger keep k_lookahead.
static const int kLook2Q[][2] = {{1, 1}, {2, 1}};   // (ld >= rows: QR <= QC always)
constexpr int kLook2NQ = sizeof(kLook2Q) / sizeof(kLook2Q[0]);

size_t look2_smem(const SlabView& s, int nt, bool ps, int qc, int qr) {
  const size_t mark = (size_t)(((s.rows + 31) / 32 + 3) & ~3) * sizeof(unsigned int);
  const size_t q = (size_t)(qc + qr), bank = q * nt * (kMaxLook / 2) * sizeof(double2);
  return mark + q * nt * sizeof(double) + bank + (ps ? bank : 0);
}

template <bool PS, int QC, int QR>
static cudaError_t look2_attr(int cluster, int* nclusters) {
  auto kern = k_look2<256, PS, QC, QR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLook2SmemMax);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = lookahead_config(cluster, kLook2SmemMax, nullptr, attr);
  cfg.blockDim = dim3(256);
  return cudaOccupancyMaxActiveClusters(nclusters, kern, &cfg);
}

template <bool PS>
static cudaError_t look2_attr_q(int qi, int cluster, int* n) {
  switch (qi) {
    case 0: return look2_attr<PS, 1, 1>(cluster, n);
    default: return look2_attr<PS, 2, 1>(cluster, n);
  }
}

long long look2_prepare(SlabView* s, int cluster) {
  const int nt = 256;
  const long long G = (long long)cluster * nt;
  const int nqc = (int)((s->ld + G - 1) / G), nqr = (int)((s->rows + G - 1) / G);
  for (int qi = 0; qi < kLook2NQ; ++qi) {
    const int qc = kLook2Q[qi][0], qr = kLook2Q[qi][1];
    if (qc < nqc || qr < nqr || look2_smem(*s, nt, true, qc, qr) > kLook2SmemMax) continue;
    int n0 = 0, n1 = 0;
    cudaError_t e = look2_attr_q<false>(qi, cluster, &n0);
    if (e == cudaSuccess) e = look2_attr_q<true>(qi, cluster, &n1);
    if (e != cudaSuccess || n0 < 1 || n1 < 1) {
      cudaGetLastError();
      return 0;
    }
    s->look_nt = nt;
    s->look_qc = qc;
    s->look_qr = qr;
    s->look_nqc = nqc;
    s->look_nqr = nqr;
    return 2LL * (nqc + nqr) * (kMaxLook / 2) * G;   // hand-off double2 entries (two banks)
  }
  return 0;
}

template <bool PS, int QC, int QR>
static cudaError_t look2_launch(const SlabView& s, const double* T, int S, int bown, int bpre, double tol_opt,
                                double tol_piv, int cluster, cudaStream_t st) {
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = lookahead_config(cluster, look2_smem(s, 256, PS, QC, QR), st, attr);
  cfg.blockDim = dim3(256);
  return cudaLaunchKernelEx(&cfg, k_look2<256, PS, QC, QR>, s, T, S, bown, bpre, s.look_nqc, s.look_nqr,
                            tol_opt, tol_piv);
}

template <bool PS>
static cudaError_t look2_launch_q(const SlabView& s, const double* T, int S, int bown, int bpre, double tol_opt,
                                  double tol_piv, int cluster, cudaStream_t st) {
  const int qc = s.look_qc, qr = s.look_qr;
  if (qc == 1 && qr == 1) return look2_launch<PS, 1, 1>(s, T, S, bown, bpre, tol_opt, tol_piv, cluster, st);
  return look2_launch<PS, 2, 1>(s, T, S, bown, bpre, tol_opt, tol_piv, cluster, st);
}

cudaError_t launch_lookahead(const SlabView& s, const double* T, int S, int bown, int bpre, double tol_opt,
                             double tol_piv, int cluster, bool cache, cudaStream_t st) {
  if (s.look_nt > 0) {
    // the previous bank in shared memory (always fits: look2_prepare), read from the hand-off only
    // when the caller disables the cache (experiments)
    const bool ps = cache && bpre >= 0;
    return ps ? look2_launch_q<true>(s, T, S, bown, bpre, tol_opt, tol_piv, cluster, st)
              : look2_launch_q<false>(s, T, S, bown, bpre, tol_opt, tol_piv, cluster, st);
  }
  int nqc = 0, nqr = 0;
  const size_t smem = lookahead_smem(s, cluster, cache && bpre >= 0, &nqc, &nqr);
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = lookahead_config(cluster, smem, st, attr);
  return cudaLaunchKernelEx(&cfg, k_lookahead, s, T, S, bown, bpre, nqc, nqr, tol_opt, tol_piv);
}

// k_update_s configurations (rows per stage R, stages K); shared memory ~ K*R*(cw+16)*8 B.
// Measured (scripts/pipe_sweep.sh): {4, 12} is the fastest pass on its own.  When the pass is
// shorter than the concurrent look-ahead selection (4000^2) the gentle {2, 16} gives the shorter
// pipelined block, because it slows the selection's dependent HBM reads least; from 8000^2 on the
// pass is the critical path (round 2b, scripts/cfg8000_r02b.sh) and {4, 12} the shortest block.
// SIMPLEX_PASS_CFG overrides the choice (experiments).
struct PassCfg { int R, K; };
static const PassCfg kPassCfgs[] = {{4, 12}, {4, 10}, {8, 5}, {6, 7}, {2, 16}, {4, 8}};
int pass_cfg_choice(bool pipelined, double pass_bytes) {
  const char* e = experiment_env("SIMPLEX_PASS_CFG");
  const int v = e ? std::atoi(e) : -1;
  if (v >= 0 && v < 6) return v;
  if (pipelined && pass_bytes < 1e9) return 4;     // selection-bound (4000^2: 210 us blocks, 104 us pass)
  // round 2b: with the selection at 308 us next to the 8000^2 pass, the fastest pass is the bound:
  // {4, 12} 335.5-337.4 us blocks (pass 323.5 us, 96.3 % of HBM) vs {6, 7} 344.4 (332.5)
  return 0;
}
int update_s_max(int S) { return S <= 4 ? 4 : S <= 8 ? 8 : S <= kMaxLook ? kMaxLook : kColS; }

size_t update_s_smem(int cfg, int cw, int rows, int S) {
  const PassCfg c = kPassCfgs[cfg];
  const int sc = S > kMaxLook ? kColS : kMaxLook;
  return (size_t)c.K * c.R * (cw + sc) * sizeof(double) + (size_t)((rows + 31) / 32) * sizeof(unsigned int);
}

template <int S, int R, int K>
static cudaError_t pass_prepare(size_t smem, int* occ) {
  auto kern = k_update_s<S, R, K>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, kThreads + 64, smem);
}

template <int R, int K>
static cudaError_t pass_prepare_s(int S, size_t smem, int* occ) {
  switch (update_s_max(S)) {
    case 4: return pass_prepare<4, R, K>(smem, occ);
    case 8: return pass_prepare<8, R, K>(smem, occ);
    case kColS: return pass_prepare<kColS, R, K>(smem, occ);
    default: return pass_prepare<16, R, K>(smem, occ);
  }
}

cudaError_t update_s_occupancy(int cfg, int S, int* blocks_per_sm, size_t smem) {
  switch (cfg) {
    case 1: return pass_prepare_s<4, 10>(S, smem, blocks_per_sm);
    case 2: return pass_prepare_s<8, 5>(S, smem, blocks_per_sm);
    case 3: return pass_prepare_s<6, 7>(S, smem, blocks_per_sm);
    case 4: return pass_prepare_s<2, 16>(S, smem, blocks_per_sm);
    case 5: return pass_prepare_s<4, 8>(S, smem, blocks_per_sm);
    default: return pass_prepare_s<4, 12>(S, smem, blocks_per_sm);
  }
}

template <int R, int K>
static cudaError_t pass_launch(const SlabView& s, int S, const double* src, double* dst, int bank, int nc, int Gr,
                               int cw, size_t smem, cudaStream_t st, bool pdl) {
  const int grid = nc * Gr;
  switch (update_s_max(S)) {
    case 4: return launch_ex(k_update_s<4, R, K>, grid, kThreads + 64, smem, st, pdl, s, src, dst, bank, nc, Gr, cw);
    case 8: return launch_ex(k_update_s<8, R, K>, grid, kThreads + 64, smem, st, pdl, s, src, dst, bank, nc, Gr, cw);
    case kColS: return launch_ex(k_update_s<kColS, R, K>, grid, kThreads + 64, smem, st, pdl, s, src, dst, bank, nc, Gr, cw);
    default: return launch_ex(k_update_s<16, R, K>, grid, kThreads + 64, smem, st, pdl, s, src, dst, bank, nc, Gr, cw);
  }
}

cudaError_t launch_update_s(int cfg, const SlabView& s, int S, const double* src, double* dst, int bank, int nc,
                            int Gr, int cw, cudaStream_t st, bool pdl) {
  const size_t smem = update_s_smem(cfg, cw, s.rows, S);
  switch (cfg) {
    case 1: return pass_launch<4, 10>(s, S, src, dst, bank, nc, Gr, cw, smem, st, pdl);
    case 2: return pass_launch<8, 5>(s, S, src, dst, bank, nc, Gr, cw, smem, st, pdl);
    case 3: return pass_launch<6, 7>(s, S, src, dst, bank, nc, Gr, cw, smem, st, pdl);
    case 4: return pass_launch<2, 16>(s, S, src, dst, bank, nc, Gr, cw, smem, st, pdl);
    case 5: return pass_launch<4, 8>(s, S, src, dst, bank, nc, Gr, cw, smem, st, pdl);
    default: return pass_launch<4, 12>(s, S, src, dst, bank, nc, Gr, cw, smem, st, pdl);
  }
}

cudaError_t launch_phase1_row0(const SlabView& s, cudaStream_t st) {
  k_phase1_row0<<<(int)((s.ld + kThreads - 1) / kThreads), kThreads, 0, st>>>(s);
  SX_CHECK_LAUNCH();
}

cudaError_t launch_phase2_row0(const SlabView& s, long long n, cudaStream_t st) {
  k_phase2_row0<<<(int)((s.ld + kThreads - 1) / kThreads), kThreads, 0, st>>>(s, n);
  SX_CHECK_LAUNCH();
}

cudaError_t launch_force(const SlabView& s, int r, int k, const double* col, cudaStream_t st) {
  k_force<<<1, kThreads, 0, st>>>(s, r, k, col);
  SX_CHECK_LAUNCH();
}

cudaError_t launch_set_status(DevState* d, int status, cudaStream_t st) {
  k_set_status<<<1, 1, 0, st>>>(d, status);
  SX_CHECK_LAUNCH();
}

cudaError_t launch_drive_find(const SlabView& s, int i, long long nm, double tol, long long* fj, cudaStream_t st) {
  k_drive_find<<<1, 1024, 0, st>>>(s, i, nm, tol, fj);
  SX_CHECK_LAUNCH();
}
cudaError_t launch_drive_pick(const long long* fj, int nparts, long long* fjmin, cudaStream_t st) {
  k_drive_pick<<<1, 1, 0, st>>>(fj, nparts, fjmin);
  SX_CHECK_LAUNCH();
}
cudaError_t launch_drive_col(const SlabView& s, const long long* fjmin, double* xcol, cudaStream_t st) {
  const int g = (int)std::min<long long>((s.rows + kThreads - 1) / kThreads, 64);
  k_drive_col<<<g, kThreads, 0, st>>>(s, fjmin, xcol);
  SX_CHECK_LAUNCH();
}
cudaError_t launch_drive_force(const SlabView& s, int i, int q, const long long* fjmin, const double* xcols,
                               int nsrc, long long xs, cudaStream_t st) {
  k_drive_force<<<1, kThreads, 0, st>>>(s, i, q, fjmin, xcols, nsrc, xs);
  SX_CHECK_LAUNCH();
}

cudaError_t launch_flush(const SlabView& s, cudaStream_t st) {
  k_flush<<<1, 1024, 0, st>>>(s);
  SX_CHECK_LAUNCH();
}

cudaError_t launch_extract(const SlabView& s, long long n, double* x, double* y, double* obj, cudaStream_t st) {
  const long long t = (long long)s.rows - 1 + s.w;
  int g = (int)((t + 255) / 256);
  if (g > 1024) g = 1024;
  k_extract<<<g, 256, 0, st>>>(s, n, x, y, obj);
  SX_CHECK_LAUNCH();
}

cudaError_t launch_hash(const SlabView& s, long long Wg, int include_rhs, unsigned long long* out,
                        cudaStream_t st, int sms) {
  k_hash<<<sms * 8, kThreads, 0, st>>>(s, Wg, include_rhs, out);
  SX_CHECK_LAUNCH();
}

}  // namespace sx
