// ubench_update.cu — microbenchmark of streaming read-modify-write patterns for the pivot
// update on B200 (which access schedule reaches the HBM copy rate?).  Not part of the
// library; results go to profiles/.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ double2 ldg2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ double2 ld_cs(const double* p) {
  double2 v; asm volatile("ld.global.cs.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p)); return v; }
__device__ __forceinline__ void st_cs(double* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory"); }
__device__ __forceinline__ double2 ld_ef(const double* p) {
  double2 v; asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p)); return v; }

// calibration: copy
__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, long long n2) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x, s = (long long)gridDim.x * blockDim.x;
  for (; i + 3 * s < n2; i += 4 * s) {
    double2 v0 = ldg2(a + 2*i), v1 = ldg2(a + 2*(i+s)), v2 = ldg2(a + 2*(i+2*s)), v3 = ldg2(a + 2*(i+3*s));
    *reinterpret_cast<double2*>(b + 2*i) = v0; *reinterpret_cast<double2*>(b + 2*(i+s)) = v1;
    *reinterpret_cast<double2*>(b + 2*(i+2*s)) = v2; *reinterpret_cast<double2*>(b + 2*(i+3*s)) = v3;
  }
  for (; i < n2; i += s) *reinterpret_cast<double2*>(b + 2*i) = ldg2(a + 2*i);
}

// in-place RMW, flat grid-stride, prow/col from global (L1/L2)
template <int U>
__global__ void k_flat(double* __restrict__ T, long long rows, long long ld, const double* __restrict__ prow,
                       const double* __restrict__ col) {
  const long long half = ld / 2, n2 = rows * half;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; const long long s = (long long)gridDim.x * blockDim.x;
  for (; i + (U-1) * s < n2; i += U * s) {
    double2 v[U]; double2 p[U]; double a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long long e = i + u * s; v[u] = ldg2(T + 2*e); long long r = e / half; long long j = 2*(e - r*half);
      p[u] = ldg2(prow + j); a[u] = -__ldg(col + r); }
#pragma unroll
    for (int u = 0; u < U; ++u) { long long e = i + u * s; v[u].x = __fma_rn(a[u], p[u].x, v[u].x); v[u].y = __fma_rn(a[u], p[u].y, v[u].y);
      *reinterpret_cast<double2*>(T + 2*e) = v[u]; }
  }
  for (; i < n2; i += s) { long long r = i / half; long long j = 2*(i - r*half); double2 v = ldg2(T + 2*i); double2 p = ldg2(prow + j);
    double a = -__ldg(col + r); v.x = __fma_rn(a, p.x, v.x); v.y = __fma_rn(a, p.y, v.y); *reinterpret_cast<double2*>(T + 2*i) = v; }
}

// 2-D tiles: units (chunk, row), chunk-major or row-block-major; VPT double2 per thread per row
template <int U, int VPT, int HINT>
__global__ void __launch_bounds__(256) k_tile(double* __restrict__ T, int rows, long long ld, const double* __restrict__ prow,
                                              const double* __restrict__ col, int cw, int nc, long long units, int order) {
  long long u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
  const int tid = threadIdx.x;
  if (order == 1) {
    // row-block-major: CTA b -> chunk b % nc, row block b / nc (rows split evenly across blocks)
    const int nb = gridDim.x / nc; const int c = blockIdx.x % nc, rb = blockIdx.x / nc;
    if (rb >= nb) return;
    const long long r0 = (long long)rows * rb / nb, r1 = (long long)rows * (rb + 1) / nb;
    u0 = (long long)c * rows + r0; u1 = (long long)c * rows + r1;
  }
  while (u0 < u1) {
    const int c = (int)(u0 / rows); const int i0 = (int)(u0 - (long long)c * rows);
    const int i1 = (int)min((long long)rows, i0 + (u1 - u0));
    const long long j0 = (long long)c * cw, jn = min(j0 + cw, ld);
    double2 p[VPT]; bool act[VPT]; long long j[VPT];
#pragma unroll
    for (int q = 0; q < VPT; ++q) { j[q] = j0 + 2 * (tid + q * 256); act[q] = j[q] < jn; p[q] = act[q] ? ldg2(prow + j[q]) : make_double2(0,0); }
    int i = i0;
    for (; i + U <= i1; i += U) {
      double2 v[U][VPT];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < VPT; ++q) if (act[q]) v[u][q] = HINT == 1 ? ld_cs(T + (long long)(i+u)*ld + j[q]) : HINT == 2 ? ld_ef(T + (long long)(i+u)*ld + j[q]) : ldg2(T + (long long)(i+u)*ld + j[q]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double a = -__ldg(col + i + u);
#pragma unroll
        for (int q = 0; q < VPT; ++q) if (act[q]) {
          v[u][q].x = __fma_rn(a, p[q].x, v[u][q].x); v[u][q].y = __fma_rn(a, p[q].y, v[u][q].y);
          if (HINT == 1) st_cs(T + (long long)(i+u)*ld + j[q], v[u][q]); else *reinterpret_cast<double2*>(T + (long long)(i+u)*ld + j[q]) = v[u][q];
        }
      }
    }
    for (; i < i1; ++i) {
      const double a = -__ldg(col + i);
#pragma unroll
      for (int q = 0; q < VPT; ++q) if (act[q]) { double2 v = ldg2(T + (long long)i*ld + j[q]); v.x = __fma_rn(a, p[q].x, v.x); v.y = __fma_rn(a, p[q].y, v.y);
        *reinterpret_cast<double2*>(T + (long long)i*ld + j[q]) = v; }
    }
    u0 += i1 - i0;
  }
}

// column-owner, row-strided: thread t owns double2 column jp = t % half for rows t/half, +q, +2q ...
// (all resident threads sweep q consecutive rows at a time: a contiguous chip-wide front)
template <int U>
__global__ void __launch_bounds__(256) k_colown(double* __restrict__ T, int rows, long long ld, const double* __restrict__ prow,
                                                const double* __restrict__ col, int q) {
  const long long half = ld / 2;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)q * half) return;
  const long long jp = t % half; const int k0 = (int)(t / half);
  const double2 p = ldg2(prow + 2 * jp);
  double* Tj = T + 2 * jp;
  int i = k0;
  for (; i + (U - 1) * q < rows; i += U * q) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg2(Tj + (long long)(i + u * q) * ld);
#pragma unroll
    for (int u = 0; u < U; ++u) { const double a = -__ldg(col + i + u * q);
      v[u].x = __fma_rn(a, p.x, v[u].x); v[u].y = __fma_rn(a, p.y, v[u].y);
      *reinterpret_cast<double2*>(Tj + (long long)(i + u * q) * ld) = v[u]; }
  }
  for (; i < rows; i += q) { double2 v = ldg2(Tj + (long long)i * ld); const double a = -__ldg(col + i);
    v.x = __fma_rn(a, p.x, v.x); v.y = __fma_rn(a, p.y, v.y); *reinterpret_cast<double2*>(Tj + (long long)i * ld) = v; }
}

__global__ void k_readflush(const double4* __restrict__ a, long long n, double* out) {
  double s = 0; for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) { double4 v = a[i]; s += v.x + v.w; }
  if (s == 12345.0) *out = s;
}

struct Timer { cudaEvent_t a, b; Timer() { cudaEventCreate(&a); cudaEventCreate(&b);} };

int main(int argc, char** argv) {
  int rows = argc > 1 ? atoi(argv[1]) : 8001; long long W = argc > 2 ? atoll(argv[2]) : 16001;
  long long ld = (W + 15) / 16 * 16;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double *T, *T2, *prow, *col; char* flush;
  size_t bytes = (size_t)rows * ld * 8;
  CK(cudaMalloc(&T, bytes)); CK(cudaMalloc(&T2, bytes)); CK(cudaMalloc(&prow, ld * 8)); CK(cudaMalloc(&col, (rows + 8) * 8));
  CK(cudaMalloc(&flush, 512 << 20));
  CK(cudaMemset(T, 0, bytes)); CK(cudaMemset(prow, 0, ld * 8)); CK(cudaMemset(col, 0, (rows+8) * 8));
  const double alg = 16.0 * rows * W;   // algorithmic bytes (unpadded) per pass
  Timer t; const int reps = 8;
  auto run = [&](const char* name, auto launch) {
    std::vector<float> v;
    for (int r = 0; r < reps + 2; ++r) {
      k_readflush<<<sms * 4, 256>>>((const double4*)flush, (512 << 20) / 32, prow + ld - 1);
      cudaEventRecord(t.a); launch(); cudaEventRecord(t.b); CK(cudaEventSynchronize(t.b));
      float ms; cudaEventElapsedTime(&ms, t.a, t.b); if (r >= 2) v.push_back(ms);
    }
    CK(cudaGetLastError());
    std::sort(v.begin(), v.end()); float med = v[v.size()/2];
    printf("%-44s %9.1f us  %7.1f GB/s (alg)\n", name, med * 1e3, alg / (med * 1e-3) / 1e9);
  };
  printf("rows=%d W=%lld ld=%lld bytes/pass=%.3f GB sms=%d\n", rows, W, ld, alg / 1e9, sms);
  for (int occ : {4, 6, 8}) for (int U : {2, 4, 8}) {
    int grid = sms * occ; long long half = ld / 2; int q = (int)std::min<long long>(rows, (long long)grid * 256 / half);
    char name[128]; snprintf(name, sizeof name, "colown U%d grid=%d q=%d", U, grid, q);
    if (U == 2) run(name, [&] { k_colown<2><<<grid, 256>>>(T, rows, ld, prow, col, q); });
    if (U == 4) run(name, [&] { k_colown<4><<<grid, 256>>>(T, rows, ld, prow, col, q); });
    if (U == 8) run(name, [&] { k_colown<8><<<grid, 256>>>(T, rows, ld, prow, col, q); });
  }
  run("copy (separate buffers)", [&] { k_copy<<<sms * 8, 256>>>(T, T2, (long long)rows * ld / 2); });
  run("flat U4 grid=sms*8", [&] { k_flat<4><<<sms * 8, 256>>>(T, rows, ld, prow, col); });
  run("flat U8 grid=sms*4", [&] { k_flat<8><<<sms * 4, 256>>>(T, rows, ld, prow, col); });
  for (int cwmul : {1, 2}) for (int order : {0, 1}) for (int occ : {2, 3, 4, 6}) {
    int cw = 512 * cwmul; int nc = (int)((ld + cw - 1) / cw); cw = (int)(((ld + nc - 1) / nc + 1) & ~1LL);
    long long units = (long long)nc * rows; int grid = sms * occ;
    if (order == 1) grid = std::max(nc, grid / nc * nc);
    char name[128];
    snprintf(name, sizeof name, "tile cw=%d VPT=%d U8 ord=%d grid=%d", cw, cwmul, order, grid);
    if (cwmul == 1) run(name, [&] { k_tile<8, 1, 0><<<grid, 256>>>(T, rows, ld, prow, col, cw, nc, units, order); });
    else run(name, [&] { k_tile<4, 2, 0><<<grid, 256>>>(T, rows, ld, prow, col, cw, nc, units, order); });
  }
  {
    int cw = 512; int nc = (int)((ld + cw - 1) / cw); cw = (int)(((ld + nc - 1) / nc + 1) & ~1LL); long long units = (long long)nc * rows;
    run("tile cw512 U8 cs-hints grid=sms*3", [&] { k_tile<8, 1, 1><<<sms * 3, 256>>>(T, rows, ld, prow, col, cw, nc, units, 0); });
    run("tile cw512 U8 nc-noalloc-256B grid=sms*3", [&] { k_tile<8, 1, 2><<<sms * 3, 256>>>(T, rows, ld, prow, col, cw, nc, units, 0); });
    run("tile cw512 U4 grid=sms*4", [&] { k_tile<4, 1, 0><<<sms * 4, 256>>>(T, rows, ld, prow, col, cw, nc, units, 0); });
    run("tile cw512 U16 grid=sms*2", [&] { k_tile<16, 1, 0><<<sms * 2, 256>>>(T, rows, ld, prow, col, cw, nc, units, 0); });
    run("tile cw512 U2 grid=sms*8", [&] { k_tile<2, 1, 0><<<sms * 8, 256>>>(T, rows, ld, prow, col, cw, nc, units, 0); });
  }
  return 0;
}
