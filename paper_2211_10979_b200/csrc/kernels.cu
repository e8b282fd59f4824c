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
#include <cfloat>
#include <climits>
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

// Block-wide lexicographic argmin; every thread returns the result.  Contains
// __syncthreads(): call from block-uniform control flow only.
__device__ __forceinline__ Cand block_min(Cand c) {
  __shared__ Cand sh[kThreads / 32];
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

// ------------------------------------------------------------------ a0: build
// Called after the host copied A's slab columns into rows 1..m (cudaMemcpy2DAsync)
// and c's slab columns into row 0.  Writes everything else of Table I and checks
// finiteness / b >= 0.  One thread per (row, column pair).
__global__ void __launch_bounds__(kThreads) k_build(SlabView s, const double* __restrict__ b, long long n) {
  const long long halfld = s.ld >> 1;
  const long long total = (long long)s.rows * halfld;
  uint32_t err = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / halfld;
    const long long j0 = (e - i * halfld) * 2;
    double* row = s.T + i * s.ld;
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
          else if (v < 0.0) err |= kErrNegRhs;
        }
      } else if (g < n) {                          // structural column: copied from A / c
        v = row[j];
        if (!isfinite(v)) err |= kErrNonFinite;
        if (i == 0) v = -v;                        // row 0 stores -c
      } else {                                     // slack column x_{g+1}: e_{g-n+1}
        v = (i >= 1 && g - n == i - 1) ? 1.0 : 0.0;
      }
      row[j] = v;
    }
  }
  if (err) atomicOr(&s.st->err, err);
}

__global__ void k_init_state(SlabView s, long long n, long long cap) {
  const int m = s.rows - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    s.basis[i] = (int)(n + i);                     // slack basis
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
  }
}

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
    if (j < s.w && v.x < -tol_opt) best = Cand{v.x, s.c0 + j};
    if (j + 1 < s.w && v.y < -tol_opt) best = cand_min(best, Cand{v.y, s.c0 + j + 1});
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
      if (i >= 1 && a > tol_piv) rbest = cand_min(rbest, Cand{__ddiv_rn(rhs, a), i});
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
      rr = (int)r.idx;
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
// Column-owner, row-strided schedule (measured best on B200, profiles/ubench_update_r01.txt):
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
      if (j < s.w && v.x < -tol_opt) best = Cand{v.x, s.c0 + j};
      if (j + 1 < s.w && v.y < -tol_opt) best = cand_min(best, Cand{v.y, s.c0 + j + 1});
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
      if (y && g >= n) y[g - n] = s.T[jl];
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
static cudaError_t launch_ex(void (*kern)(KArgs...), int grid, int block, cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

cudaError_t launch_pack(const SlabView& s, double* send, int grid, cudaStream_t st, bool pdl) {
  return launch_ex(k_pack, grid, kThreads, st, pdl, s, send);
}

cudaError_t launch_select(const SlabView& s, const XView& x, double tol_piv, int grid, cudaStream_t st, bool pdl) {
  return launch_ex(k_select, grid, kThreads, st, pdl, s, x, tol_piv);
}

cudaError_t update_occupancy(int* blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_update<kUpdateRows>, kThreads, 0);
}

cudaError_t launch_update(const SlabView& s, int q, double tol_opt, int grid, cudaStream_t st, bool pdl) {
  return launch_ex(k_update<kUpdateRows>, grid, kThreads, st, pdl, s, q, tol_opt);
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
