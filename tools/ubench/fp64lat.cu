// FP64 dependent-chain latency microbenchmark (one thread): DFMA, DADD, DMUL, MUFU.RCP64H, div, sqrt.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, double x, int n, long long* cyc) {
  double a = x, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { a = a + c; a = a + c; a = a + c; a = a + c; }
  long long t2 = clock64();
  double y = a;
  for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y)); y = r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y)); y = r;}
  long long t3 = clock64();
  double z = a + 2.0;
  for (int i = 0; i < n; ++i) { z = 1.0 / z + 1.5; }
  long long t4 = clock64();
  double s = a + 3.0;
  for (int i = 0; i < n; ++i) { s = sqrt(s) + 1.0; }
  long long t5 = clock64();
  double u = a + 3.0;
  for (int i = 0; i < n; ++i) { u = rsqrt(u) + 1.0; }
  long long t6 = clock64();
  out[0] = a + y + z + s + u;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMallocManaged(&c, 64);
  const int n = 1000;
  k<<<1, 1>>>(o, 1.0, n, c); cudaDeviceSynchronize();
  k<<<1, 1>>>(o, 1.0, n, c); cudaDeviceSynchronize();
  printf("cycles per dependent op: dfma %.1f dadd %.1f rcp64 %.1f (div+add) %.1f (sqrt+add) %.1f (rsqrt+add) %.1f\n",
         c[0] / (4.0 * n), c[1] / (4.0 * n), c[2] / (2.0 * n), c[3] / (1.0 * n), c[4] / (1.0 * n), c[5] / (1.0 * n));
}
