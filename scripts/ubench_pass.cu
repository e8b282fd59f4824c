// ubench_pass.cu — microbenchmark: how should the rank-s pass read the tableau on B200?
// Compares, at the 8000x8000 pass geometry (8001 rows x 16016 doubles, 1.02 GB, out of place),
//   tma:  1-D TMA (cp.async.bulk) row segments into a K-stage shared-memory ring, producer
//         warp + 8 consumer warps (the structure of k_update_s), read-only or copy (STG)
//   ldg:  consumer threads load their own column pair with LDG.128, D rows in flight per
//         thread (the structure of k_update), read-only or copy
// on the same (chunk x row-group) CTA geometry.  Not part of the library.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_pass scripts/ubench_pass.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                       \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(
          smem_u32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

constexpr int kT = 256;
static int g_nc = 0;   // column chunks (0: ceil(ld / 512))

__global__ void k_fill(double* a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    a[i] = 1.0 + (double)((i * 2654435761ull) % 1000003) * 1e-6;
}

template <int R, int K, bool WRITE>
__global__ void __launch_bounds__(kT + 32) k_tma(const double* src, double* dst, long long ld, int rows, int nc, int Gr,
                                                 int cw, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* sT = reinterpret_cast<double*>(sm);
  __shared__ __align__(8) uint64_t full[K], empty[K];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int k = 0; k < K; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], kT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int c = blockIdx.x % nc, g = blockIdx.x / nc;
  const long long j0 = (long long)c * cw;
  const int jn = (int)min((long long)cw, ld - j0);
  const int nr = rows > g ? (rows - g + Gr - 1) / Gr : 0;
  const int nst = (nr + R - 1) / R;
  if (warp == kT / 32) {
    if (lane == 0)
      for (int n = 0; n < nst; ++n) {
        const int k = n % K;
        if (n >= K) mbar_wait(&empty[k], ((n / K) - 1) & 1);
        const int rin = min(R, nr - n * R);
        mbar_expect(&full[k], rin * jn * 8);
        for (int rr = 0; rr < rin; ++rr) {
          const long long i = g + (long long)(n * R + rr) * Gr;
          bulk(sT + ((size_t)k * R + rr) * cw, src + i * ld + j0, jn * 8, &full[k]);
        }
      }
    return;
  }
  const int jl = 2 * tid;
  const bool act = jl < jn;
  double acc = 0.0;
  for (int n = 0; n < nst; ++n) {
    const int k = n % K;
    mbar_wait(&full[k], (n / K) & 1);
    const int rin = min(R, nr - n * R);
    for (int rr = 0; rr < rin; ++rr)
      if (act) {
        const double2 v = *reinterpret_cast<const double2*>(sT + ((size_t)k * R + rr) * cw + jl);
        if (WRITE) {
          const long long i = g + (long long)(n * R + rr) * Gr;
          *reinterpret_cast<double2*>(dst + i * ld + j0 + jl) = v;
        } else {
          acc += v.x + v.y;
        }
      }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[k]);
  }
  if (!WRITE && acc == 12345.678) sink[0] = acc;
}


// copy with TMA bulk stores: consumers rewrite their values into the stage (in place), the
// producer stores whole row segments with cp.async.bulk (global <- shared) before reusing a slot
template <int R, int K>
__global__ void __launch_bounds__(kT + 32) k_tma_st(const double* src, double* dst, long long ld, int rows, int nc,
                                                    int Gr, int cw, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* sT = reinterpret_cast<double*>(sm);
  __shared__ __align__(8) uint64_t full[K], comp[K];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int k = 0; k < K; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&comp[k], kT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int c = blockIdx.x % nc, g = blockIdx.x / nc;
  const long long j0 = (long long)c * cw;
  const int jn = (int)min((long long)cw, ld - j0);
  const int nr = rows > g ? (rows - g + Gr - 1) / Gr : 0;
  const int nst = (nr + R - 1) / R;
  if (warp == kT / 32) {
    if (lane == 0) {
      auto store_stage = [&](int m) {
        const int kk = m % K;
        mbar_wait(&comp[kk], (m / K) & 1);
        const int rin = min(R, nr - m * R);
        for (int rr = 0; rr < rin; ++rr) {
          const long long i = g + (long long)(m * R + rr) * Gr;
          bulk_store(dst + i * ld + j0, sT + ((size_t)kk * R + rr) * cw, jn * 8);
        }
        bulk_commit();
      };
      for (int n = 0; n < nst; ++n) {
        const int k = n % K;
        if (n >= K) {
          store_stage(n - K);
          bulk_wait_read0();
        }
        const int rin = min(R, nr - n * R);
        mbar_expect(&full[k], rin * jn * 8);
        for (int rr = 0; rr < rin; ++rr) {
          const long long i = g + (long long)(n * R + rr) * Gr;
          bulk(sT + ((size_t)k * R + rr) * cw, src + i * ld + j0, jn * 8, &full[k]);
        }
      }
      for (int m = max(0, nst - K); m < nst; ++m) store_stage(m);
      bulk_wait0();
    }
    return;
  }
  const int jl = 2 * tid;
  const bool act = jl < jn;
  for (int n = 0; n < nst; ++n) {
    const int k = n % K;
    mbar_wait(&full[k], (n / K) & 1);
    const int rin = min(R, nr - n * R);
    for (int rr = 0; rr < rin; ++rr)
      if (act) {
        double2* p = reinterpret_cast<double2*>(sT + ((size_t)k * R + rr) * cw + jl);
        double2 v = *p;
        v.x = v.x * 1.0000001;
        *p = v;
      }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&comp[k]);
  }
}


// the rank-S pass with TMA loads + TMA bulk stores (1 CTA / SM, big stages): consumers hold
// prow_u[j] (u < S) in registers, read the row's S pivot-column entries (staged by TMA next to
// the row) and apply the chains in place in shared memory; the producer stores the stage.
template <int R, int K, int S, int CG>
__global__ void __launch_bounds__(CG * kT + 32, 1) k_tma_fma(const double* src, double* dst, const double* colS,
                                                       const double* prowS, long long ld, int rows, int nc, int Gr,
                                                       int cw, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* sT = reinterpret_cast<double*>(sm);                 // [K][R][cw]
  double* sC = sT + (size_t)K * R * cw;                        // [K][R][16]
  __shared__ __align__(8) uint64_t full[K], comp[K];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int k = 0; k < K; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&comp[k], kT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int c = blockIdx.x % nc, g = blockIdx.x / nc;
  const long long j0 = (long long)c * cw;
  const int jn = (int)min((long long)cw, ld - j0);
  const int nr = rows > g ? (rows - g + Gr - 1) / Gr : 0;
  const int nst = (nr + R - 1) / R;
  if (warp == CG * kT / 32) {
    if (lane == 0) {
      auto store_stage = [&](int m) {
        const int kk = m % K;
        mbar_wait(&comp[kk], (m / K) & 1);
        const int rin = min(R, nr - m * R);
        for (int rr = 0; rr < rin; ++rr) {
          const long long i = g + (long long)(m * R + rr) * Gr;
          bulk_store(dst + i * ld + j0, sT + ((size_t)kk * R + rr) * cw, jn * 8);
        }
        bulk_commit();
      };
      for (int n = 0; n < nst; ++n) {
        const int k = n % K;
        if (n >= K) {
          store_stage(n - K);
          bulk_wait_read0();
        }
        const int rin = min(R, nr - n * R);
        mbar_expect(&full[k], rin * (jn + 16) * 8);
        for (int rr = 0; rr < rin; ++rr) {
          const long long i = g + (long long)(n * R + rr) * Gr;
          bulk(sT + ((size_t)k * R + rr) * cw, src + i * ld + j0, jn * 8, &full[k]);
          bulk(sC + ((size_t)k * R + rr) * 16, colS + i * 16, 128, &full[k]);
        }
      }
      for (int m = max(0, nst - K); m < nst; ++m) store_stage(m);
      bulk_wait0();
    }
    return;
  }
  const int grp = tid / kT;
  const int jl = 2 * (tid % kT);
  const bool act = jl < jn;
  double2 pr[S];
#pragma unroll
  for (int u = 0; u < S; ++u)
    pr[u] = act ? *reinterpret_cast<const double2*>(prowS + (long long)u * ld + j0 + jl) : make_double2(0.0, 0.0);
  for (int n = grp; n < nst; n += CG) {
    const int k = n % K;
    mbar_wait(&full[k], (n / K) & 1);
    const int rin = min(R, nr - n * R);
    if (rin == R && act) {
      double2 v[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) v[rr] = *reinterpret_cast<const double2*>(sT + ((size_t)k * R + rr) * cw + jl);
#pragma unroll
      for (int h = 0; h < S / 2; ++h) {
        double2 a[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) a[rr] = *reinterpret_cast<const double2*>(sC + ((size_t)k * R + rr) * 16 + 2 * h);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          v[rr].x = __fma_rn(-a[rr].x, pr[2 * h].x, v[rr].x);
          v[rr].y = __fma_rn(-a[rr].x, pr[2 * h].y, v[rr].y);
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          v[rr].x = __fma_rn(-a[rr].y, pr[2 * h + 1].x, v[rr].x);
          v[rr].y = __fma_rn(-a[rr].y, pr[2 * h + 1].y, v[rr].y);
        }
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) *reinterpret_cast<double2*>(sT + ((size_t)k * R + rr) * cw + jl) = v[rr];
    } else if (act) {
      for (int rr = 0; rr < rin; ++rr) {
        double2 v = *reinterpret_cast<const double2*>(sT + ((size_t)k * R + rr) * cw + jl);
#pragma unroll
        for (int u = 0; u < S; ++u) {
          const double a = -sC[((size_t)k * R + rr) * 16 + u];
          v.x = __fma_rn(a, pr[u].x, v.x);
          v.y = __fma_rn(a, pr[u].y, v.y);
        }
        *reinterpret_cast<double2*>(sT + ((size_t)k * R + rr) * cw + jl) = v;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&comp[k]);
  }
}


// three roles: loader warp (TMA loads), storer warp (TMA bulk stores as soon as a stage is
// computed, then frees the slot), 8 consumer warps (chains in place in shared memory)
template <int R, int K, int S>
__global__ void __launch_bounds__(kT + 64, 1) k_tma_fma3(const double* src, double* dst, const double* colS,
                                                        const double* prowS, long long ld, int rows, int nc, int Gr,
                                                        int cw, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* sT = reinterpret_cast<double*>(sm);                 // [K][R][cw]
  double* sC = sT + (size_t)K * R * cw;                        // [K][R][16]
  __shared__ __align__(8) uint64_t full[K], comp[K], empty[K];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int k = 0; k < K; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&comp[k], kT / 32);
      mbar_init(&empty[k], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int c = blockIdx.x % nc, g = blockIdx.x / nc;
  const long long j0 = (long long)c * cw;
  const int jn = (int)min((long long)cw, ld - j0);
  const int nr = rows > g ? (rows - g + Gr - 1) / Gr : 0;
  const int nst = (nr + R - 1) / R;
  if (warp == kT / 32) {                                          // loader
    if (lane == 0)
      for (int n = 0; n < nst; ++n) {
        const int k = n % K;
        if (n >= K) mbar_wait(&empty[k], ((n / K) - 1) & 1);
        const int rin = min(R, nr - n * R);
        mbar_expect(&full[k], rin * (jn + 16) * 8);
        for (int rr = 0; rr < rin; ++rr) {
          const long long i = g + (long long)(n * R + rr) * Gr;
          bulk(sT + ((size_t)k * R + rr) * cw, src + i * ld + j0, jn * 8, &full[k]);
          bulk(sC + ((size_t)k * R + rr) * 16, colS + i * 16, 128, &full[k]);
        }
      }
    return;
  }
  if (warp == kT / 32 + 1) {                                      // storer
    if (lane == 0) {
      for (int m = 0; m < nst; ++m) {
        const int k = m % K;
        mbar_wait(&comp[k], (m / K) & 1);
        const int rin = min(R, nr - m * R);
        for (int rr = 0; rr < rin; ++rr) {
          const long long i = g + (long long)(m * R + rr) * Gr;
          bulk_store(dst + i * ld + j0, sT + ((size_t)k * R + rr) * cw, jn * 8);
        }
        bulk_commit();
        if (m >= 1) {
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          mbar_arrive(&empty[(m - 1) % K]);
        }
      }
      bulk_wait0();
    }
    return;
  }
  const int jl = 2 * tid;
  const bool act = jl < jn;
  double2 pr[S];
#pragma unroll
  for (int u = 0; u < S; ++u)
    pr[u] = act ? *reinterpret_cast<const double2*>(prowS + (long long)u * ld + j0 + jl) : make_double2(0.0, 0.0);
  for (int n = 0; n < nst; ++n) {
    const int k = n % K;
    mbar_wait(&full[k], (n / K) & 1);
    const int rin = min(R, nr - n * R);
    if (rin == R && act) {
      double2 v[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) v[rr] = *reinterpret_cast<const double2*>(sT + ((size_t)k * R + rr) * cw + jl);
#pragma unroll
      for (int h = 0; h < S / 2; ++h) {
        double2 a[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) a[rr] = *reinterpret_cast<const double2*>(sC + ((size_t)k * R + rr) * 16 + 2 * h);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          v[rr].x = __fma_rn(-a[rr].x, pr[2 * h].x, v[rr].x);
          v[rr].y = __fma_rn(-a[rr].x, pr[2 * h].y, v[rr].y);
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          v[rr].x = __fma_rn(-a[rr].y, pr[2 * h + 1].x, v[rr].x);
          v[rr].y = __fma_rn(-a[rr].y, pr[2 * h + 1].y, v[rr].y);
        }
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) *reinterpret_cast<double2*>(sT + ((size_t)k * R + rr) * cw + jl) = v[rr];
    } else if (act) {
      for (int rr = 0; rr < rin; ++rr) {
        double2 v = *reinterpret_cast<const double2*>(sT + ((size_t)k * R + rr) * cw + jl);
#pragma unroll
        for (int u = 0; u < S; ++u) {
          const double a = -sC[((size_t)k * R + rr) * 16 + u];
          v.x = __fma_rn(a, pr[u].x, v.x);
          v.y = __fma_rn(a, pr[u].y, v.y);
        }
        *reinterpret_cast<double2*>(sT + ((size_t)k * R + rr) * cw + jl) = v;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&comp[k]);
  }
}

template <int D, bool WRITE>
__global__ void __launch_bounds__(kT) k_ldg(const double* src, double* dst, long long ld, int rows, int nc, int Gr,
                                            int cw, double* sink) {
  const int c = blockIdx.x % nc, g = blockIdx.x / nc;
  const long long j0 = (long long)c * cw;
  const int jn = (int)min((long long)cw, ld - j0);
  const int jl = 2 * threadIdx.x;
  if (jl >= jn) return;
  const double* s = src + j0 + jl;
  double* d = dst + j0 + jl;
  double acc = 0.0;
  int i = g;
  for (; i + (D - 1) * Gr < rows; i += D * Gr) {
    double2 v[D];
#pragma unroll
    for (int q = 0; q < D; ++q) v[q] = *reinterpret_cast<const double2*>(s + (long long)(i + q * Gr) * ld);
#pragma unroll
    for (int q = 0; q < D; ++q) {
      if (WRITE) *reinterpret_cast<double2*>(d + (long long)(i + q * Gr) * ld) = v[q];
      else acc += v[q].x + v[q].y;
    }
  }
  for (; i < rows; i += Gr) {
    const double2 v = *reinterpret_cast<const double2*>(s + (long long)i * ld);
    if (WRITE) *reinterpret_cast<double2*>(d + (long long)i * ld) = v;
    else acc += v.x + v.y;
  }
  if (!WRITE && acc == 12345.678) sink[0] = acc;
}

template <typename F>
static float timeit(F f, int reps = 10) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) f();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms * 1e3f / reps;
}

template <int R, int K, bool W>
static void run_tma(const double* A, double* B, long long ld, int rows, int sms, int occ_target, double* sink) {
  const int cwmax = 512;
  const int nc = g_nc ? g_nc : (int)((ld + cwmax - 1) / cwmax);
  const int cw = (int)(((ld + nc - 1) / nc + 1) / 2 * 2);
  const size_t smem = (size_t)K * R * cw * 8;
  CK(cudaFuncSetAttribute(k_tma<R, K, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int Gr = occ_target * sms / nc;
  const float us = timeit([&] { k_tma<R, K, W><<<nc * Gr, kT + 32, smem>>>(A, B, ld, rows, nc, Gr, cw, sink); });
  const double bytes = (double)rows * ld * 8 * (W ? 2 : 1);
  printf("tma R=%d K=%d %s ctas=%d: %.1f us  %.0f GB/s\n", R, K, W ? "copy" : "read", nc * Gr, us, bytes / us / 1e3);
}

template <int R, int K>
static void run_tma_st(const double* A, double* B, long long ld, int rows, int sms, int occ_target, double* sink) {
  const int cwmax = 512;
  const int nc = g_nc ? g_nc : (int)((ld + cwmax - 1) / cwmax);
  const int cw = (int)(((ld + nc - 1) / nc + 1) / 2 * 2);
  const size_t smem = (size_t)K * R * cw * 8;
  CK(cudaFuncSetAttribute(k_tma_st<R, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int Gr = occ_target * sms / nc;
  const float us = timeit([&] { k_tma_st<R, K><<<nc * Gr, kT + 32, smem>>>(A, B, ld, rows, nc, Gr, cw, sink); });
  const double bytes = (double)rows * ld * 8 * 2;
  printf("tma+bulkstore R=%d K=%d copy ctas=%d: %.1f us  %.0f GB/s\n", R, K, nc * Gr, us, bytes / us / 1e3);
}

template <int R, int K, int CG = 1>
static void run_tma_fma(const double* A, double* B, const double* cs, const double* ps, long long ld, int rows, int sms,
                        double* sink) {
  const int cwmax = 512;
  const int nc = g_nc ? g_nc : (int)((ld + cwmax - 1) / cwmax);
  const int cw = (int)(((ld + nc - 1) / nc + 1) / 2 * 2);
  const size_t smem = (size_t)K * R * (cw + 16) * 8;
  CK(cudaFuncSetAttribute(k_tma_fma<R, K, 16, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int Gr = sms / nc;
  const float us = timeit([&] { k_tma_fma<R, K, 16, CG><<<nc * Gr, CG * kT + 32, smem>>>(A, B, cs, ps, ld, rows, nc, Gr, cw, sink); });
  const double bytes = (double)rows * ld * 8 * 2;
  printf("tma+bulkstore+fma16 R=%d K=%d CG=%d ctas=%d: %.1f us  %.0f GB/s\n", R, K, CG, nc * Gr, us, bytes / us / 1e3);
}

template <int R, int K>
static void run_tma_fma3(const double* A, double* B, const double* cs, const double* ps, long long ld, int rows, int sms,
                         double* sink) {
  const int cwmax = 512;
  const int nc = g_nc ? g_nc : (int)((ld + cwmax - 1) / cwmax);
  const int cw = (int)(((ld + nc - 1) / nc + 1) / 2 * 2);
  const size_t smem = (size_t)K * R * (cw + 16) * 8;
  CK(cudaFuncSetAttribute(k_tma_fma3<R, K, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int Gr = sms / nc;
  const float us = timeit([&] { k_tma_fma3<R, K, 16><<<nc * Gr, kT + 64, smem>>>(A, B, cs, ps, ld, rows, nc, Gr, cw, sink); });
  const double bytes = (double)rows * ld * 8 * 2;
  printf("3-role R=%d K=%d ctas=%d: %.1f us  %.0f GB/s\n", R, K, nc * Gr, us, bytes / us / 1e3);
}

template <int D, bool W>
static void run_ldg(const double* A, double* B, long long ld, int rows, int sms, int ctas_per_sm, double* sink) {
  const int cwmax = 512;
  const int nc = (int)((ld + cwmax - 1) / cwmax);
  const int cw = (int)(((ld + nc - 1) / nc + 1) / 2 * 2);
  const int Gr = ctas_per_sm * sms / nc;
  const float us = timeit([&] { k_ldg<D, W><<<nc * Gr, kT>>>(A, B, ld, rows, nc, Gr, cw, sink); });
  const double bytes = (double)rows * ld * 8 * (W ? 2 : 1);
  printf("ldg D=%d %s ctas=%d: %.1f us  %.0f GB/s\n", D, W ? "copy" : "read", nc * Gr, us, bytes / us / 1e3);
}

int main(int argc, char** argv) {
  const int rows = 8001;
  const long long ld = 16016;
  const int sms = argc > 1 ? atoi(argv[1]) : 132;
  double *A, *B, *sink;
  CK(cudaMalloc(&A, (size_t)rows * ld * 8));
  CK(cudaMalloc(&B, (size_t)rows * ld * 8));
  CK(cudaMalloc(&sink, 8));
  g_nc = argc > 2 ? atoi(argv[2]) : 0;
  k_fill<<<1184, 256>>>(A, (long long)rows * ld);
  CK(cudaDeviceSynchronize());
  const float us = timeit([&] { CK(cudaMemcpyAsync(B, A, (size_t)rows * ld * 8, cudaMemcpyDeviceToDevice)); });
  printf("cudaMemcpy D2D: %.1f us  %.0f GB/s\n", us, 2.0 * rows * ld * 8 / us / 1e3);
  printf("SMs used: %d\n", sms);
  if (argc > 4) {   // rank-16 pass with bulk stores
    double *cs, *ps;
    CK(cudaMalloc(&cs, (size_t)rows * 16 * 8));
    CK(cudaMalloc(&ps, (size_t)16 * ld * 8));
    k_fill<<<256, 256>>>(cs, (long long)rows * 16);
    k_fill<<<256, 256>>>(ps, 16 * ld);
    CK(cudaDeviceSynchronize());
    run_tma_fma<8, 4>(A, B, cs, ps, ld, rows, sms, sink);
    run_tma_fma3<8, 4>(A, B, cs, ps, ld, rows, sms, sink);
    run_tma_fma3<8, 5>(A, B, cs, ps, ld, rows, sms, sink);
    run_tma_fma3<8, 6>(A, B, cs, ps, ld, rows, sms, sink);
    run_tma_fma3<4, 10>(A, B, cs, ps, ld, rows, sms, sink);
    run_tma_fma3<4, 12>(A, B, cs, ps, ld, rows, sms, sink);
    run_tma_fma3<6, 7>(A, B, cs, ps, ld, rows, sms, sink);
    return 0;
  }
  if (argc > 3) {   // bulk-store sweep only
    run_tma_st<8, 6>(A, B, ld, rows, sms, 1, sink);
    run_tma_st<4, 12>(A, B, ld, rows, sms, 1, sink);
    run_tma_st<6, 8>(A, B, ld, rows, sms, 1, sink);
    run_tma_st<16, 3>(A, B, ld, rows, sms, 1, sink);
    run_tma_st<8, 5>(A, B, ld, rows, sms, 1, sink);
    run_tma_st<12, 4>(A, B, ld, rows, sms, 1, sink);
    return 0;
  }
  run_tma<2, 8, false>(A, B, ld, rows, sms, 2, sink);
  run_tma<4, 4, false>(A, B, ld, rows, sms, 2, sink);
  run_tma<4, 8, false>(A, B, ld, rows, sms, 2, sink);
  run_tma<8, 4, false>(A, B, ld, rows, sms, 2, sink);
  run_tma<2, 8, true>(A, B, ld, rows, sms, 2, sink);
  run_tma<4, 4, true>(A, B, ld, rows, sms, 2, sink);
  run_tma<4, 8, true>(A, B, ld, rows, sms, 2, sink);
  run_tma_st<2, 8>(A, B, ld, rows, sms, 2, sink);
  run_tma_st<4, 4>(A, B, ld, rows, sms, 2, sink);
  run_tma_st<4, 6>(A, B, ld, rows, sms, 2, sink);
  run_tma_st<2, 12>(A, B, ld, rows, sms, 2, sink);
  run_tma_st<4, 8>(A, B, ld, rows, sms, 1, sink);
  run_tma_st<8, 6>(A, B, ld, rows, sms, 1, sink);
  run_ldg<4, false>(A, B, ld, rows, sms, 2, sink);
  run_ldg<8, false>(A, B, ld, rows, sms, 2, sink);
  run_ldg<4, false>(A, B, ld, rows, sms, 4, sink);
  run_ldg<4, true>(A, B, ld, rows, sms, 2, sink);
  run_ldg<8, true>(A, B, ld, rows, sms, 2, sink);
  run_ldg<4, true>(A, B, ld, rows, sms, 4, sink);
  run_ldg<8, true>(A, B, ld, rows, sms, 4, sink);
  return 0;
}
