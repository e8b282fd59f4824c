// FP64 latency / throughput microbenchmark (round 2b): dependent DFMA / DADD latency,
// __ddiv_rn latency and per-SM division throughput.   nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -o build/lat_probe scripts/fp64_latency.cu   (measured on B200: DFMA 8.1 cycles, __ddiv_rn 127
// cycles dependent, ~2 divisions / cycle / SM at 256 threads)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, double a, double b, int n, long long* cyc) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); }
  long long t1 = clock64();
  double y = x;
  for (int i = 0; i < n; ++i) { y = __ddiv_rn(y, a); y = __ddiv_rn(y, b); }
  long long t2 = clock64();
  double z = y;
  for (int i = 0; i < n; ++i) { z = __dadd_rn(z, a); z = __dadd_rn(z, b); z = __dadd_rn(z, a); z = __dadd_rn(z, b);}
  long long t3 = clock64();
  out[threadIdx.x] = z;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main_div();
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024*8); cudaMemset(o, 0, 1024*8); cudaMallocManaged(&c, 64);
  int n = 1000;
  for (int th : {32, 64, 128, 256}) {
    k<<<1, th>>>(o, 1.0000001, 0.5, n, c); cudaDeviceSynchronize();
    printf("threads %d: dfma dep latency %.1f cyc, ddiv_rn %.1f cyc, dadd %.1f cyc\n", th, c[0] / (4.0 * n), c[1] / (2.0 * n), c[2] / (4.0*n));
  }
  return main_div();
}
__global__ void kdiv(double* out, int n, long long* cyc) {
  double x = 1.5 + threadIdx.x * 1e-3, y = 0.7 + threadIdx.x * 1e-4, z = 2.3, w = 0.9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { y = __ddiv_rn(x, y); }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { z = __ddiv_rn(x, z); w = __ddiv_rn(x, w); }
  long long t2 = clock64();
  double r = 1.1;
  for (int i = 0; i < n; ++i) { r = __drcp_rn(r); }
  long long t3 = clock64();
  out[threadIdx.x] = y + z + w + r;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main_div() {
  double* o; long long* c; cudaMalloc(&o, 1024*8); cudaMallocManaged(&c, 64);
  int n = 1000;
  for (int th : {32, 64, 128, 256, 512, 1024}) {
    kdiv<<<1, th>>>(o, n, c); cudaDeviceSynchronize();
    printf("threads %4d: ddiv dep %.1f cyc/div/warp-chain; 2 indep chains %.1f cyc per pair; drcp %.1f; => SM div throughput %.2f div/clk\n",
           th, c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, th * (double)n / c[0]);
  }
  return 0;
}
