// Exact-order shape matching building blocks on the B200:
// latency (one thread, dependent chains, clock64) of DFMA, IEEE '/', IEEE sqrt, crt::sincos_cr
// (small and double-double routes), and of one iteration of extract_rotation_exact (correctly
// rounded / CUDA sincos) against the latency-tuned extract_rotation.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --fmad=false -I../../paper_1906_05260_b200/csrc exactops.cu -o exactops
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "shape.cuh"

using namespace vdev;

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
__device__ double mk(uint64_t r, int e) {
  uint64_t mant = r & ((1ull << 52) - 1);
  const int mode = (r >> 60) & 7;
  if (mode == 0) mant = (1ull << 52) - 1;
  if (mode == 1) mant = 0;
  if (mode == 2) mant = (r >> 20) & 0xfff;
  if (mode == 3) mant = ((1ull << 52) - 1) ^ ((r >> 13) & 0xff);
  const uint64_t bits = ((uint64_t)((r >> 59) & 1) << 63) | ((uint64_t)(1023 + e) << 52) | mant;
  return __longlong_as_double((long long)bits);
}
// rn::div_by against the IEEE division on random and adversarial operands (bit-identical required)
__global__ void validate(uint64_t seed, long long n, unsigned long long* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint64_t r1 = mix(seed ^ (3 * i)), r2 = mix(seed ^ (3 * i + 1)), r3 = mix(seed ^ (3 * i + 2)), r4 = mix(r1 ^ r3);
    const int ea = (int)(r4 % 1001) - 500, eb = (int)((r4 >> 12) % 1001) - 500;
    const double b = mk(r2, (r4 >> 40) & 1 ? eb : (int)((r4 >> 24) % 41) - 20);
    const double a[3] = {mk(r1, (r4 >> 41) & 1 ? ea : (int)((r4 >> 30) % 41) - 20), mk(r3, (int)((r4 >> 50) % 61) - 30),
                         (r4 >> 62) ? 0.0 : -0.0};
    double q[3];
    rn::div_by(a, b, q);
    for (int k = 0; k < 3; ++k)
      if (__double_as_longlong(q[k]) != __double_as_longlong(a[k] / b)) atomicAdd(bad, 1ull);
  }
}

__global__ void latency(double* out, double x0, int n, long long* cyc) {
  double a = x0, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  long long t1 = clock64();
  double z = a + 2.0;
  for (int i = 0; i < n; ++i) z = 1.0 / z + 1.5;
  long long t2 = clock64();
  long long t3 = clock64();
  double s = a + 3.0;
  for (int i = 0; i < n; ++i) s = sqrt(s) + 1.0;
  long long t4 = clock64();
  long long t5 = clock64();
  double w = 1e-6 * a, acc = 0.0;
  for (int i = 0; i < n; ++i) {
    double sn, cs;
    crt::sincos_cr(w, &sn, &cs);
    w = 1e-6 + sn * 1e-3 + cs * 1e-12;
    acc += sn;
  }
  long long t6 = clock64();
  double w2 = 0.1 * a;
  for (int i = 0; i < n; ++i) {
    double sn, cs;
    crt::sincos_cr(w2, &sn, &cs);
    w2 = 0.1 + sn * 1e-3 + cs * 1e-12;
    acc += sn;
  }
  long long t7 = clock64();
  // extract_rotation_exact from a perturbed identity: count iterations and cycles
  vm::M3 B{};
  B.m[0][0] = 1.0 + 1e-3 * a; B.m[1][1] = 0.98; B.m[2][2] = 1.01; B.m[0][1] = 0.02; B.m[1][0] = -0.015; B.m[2][0] = 0.01;
  int iters = 0;
  long long t8 = clock64();
  vm::Q4 q = extract_rotation_exact(B, vm::Q4{1, 0, 0, 0}, &iters);
  long long t9 = clock64();
  int iters_fast = 0;
  vm::Q4 qf = extract_rotation(B, vm::Q4{1, 0, 0, 0}, &iters_fast);
  long long t10 = clock64();
  int iters_ieee = 0;
  vm::Q4 qi = extract_rotation_exact<false>(B, vm::Q4{1, 0, 0, 0}, &iters_ieee);  // second call: warm i-cache
  long long t11 = clock64();
  int iters_ds = 0;
  vm::Q4 qd = extract_rotation_exact<true>(B, vm::Q4{1, 0, 0, 0}, &iters_ds);
  long long t12 = clock64();
  cyc[14] = t12 - t11; cyc[15] = iters_ds;
  out[1] = qd.w;
  out[0] = a + z + s + w + w2 + acc + q.w + qf.w + qi.w;
  cyc[11] = t11 - t10; cyc[12] = iters_ieee;
  cyc[13] = (__double_as_longlong(q.w) == __double_as_longlong(qi.w) && __double_as_longlong(q.x) == __double_as_longlong(qi.x) &&
             __double_as_longlong(q.y) == __double_as_longlong(qi.y) && __double_as_longlong(q.z) == __double_as_longlong(qi.z));
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = 0; cyc[3] = t4 - t3; cyc[4] = 0; cyc[5] = t6 - t5;
  cyc[6] = t7 - t6; cyc[7] = t9 - t8; cyc[8] = iters; cyc[9] = t10 - t9; cyc[10] = iters_fast;
}

int main() {
  unsigned long long* bad;
  cudaMallocManaged(&bad, sizeof(unsigned long long));
  *bad = 0;
  const long long nval = 1ll << 30;
  validate<<<148 * 8, 256>>>(2024, nval, bad);
  cudaDeviceSynchronize();
  printf("rn::div_by vs IEEE division: %llu mismatches in %lld x 3 quotients\n", *bad, nval);
  double* o;
  long long* c;
  cudaMalloc(&o, 16);
  cudaMallocManaged(&c, 32 * sizeof(long long));
  const int it = 1000;
  latency<<<1, 1>>>(o, 1.0, it, c);
  cudaDeviceSynchronize();
  latency<<<1, 1>>>(o, 1.0, it, c);
  cudaDeviceSynchronize();
  printf("cycles per dependent op: dfma %.1f | (1/x + c): IEEE %.1f  div_rn %.1f | (sqrt + c): IEEE %.1f  sqrt_rn %.1f | "
         "sincos_cr small %.1f  dd %.1f\n",
         c[0] / (4.0 * it), c[1] / (1.0 * it), c[2] / (1.0 * it), c[3] / (1.0 * it), c[4] / (1.0 * it), c[5] / (1.0 * it),
         c[6] / (1.0 * it));
  printf("extract_rotation_exact: %lld iterations, %.1f cycles/iteration (again, warm: %lld it, %.1f cyc/it, same bits %lld) | "
         "fast path: %lld iterations, %.1f cycles/iteration\n",
         c[8], c[7] / (double)(c[8] > 0 ? c[8] : 1), c[12], c[11] / (double)(c[12] > 0 ? c[12] : 1), c[13], c[10],
         c[9] / (double)(c[10] > 0 ? c[10] : 1));
  printf("extract_rotation_exact with CUDA sincos: %lld iterations, %.1f cycles/iteration\n", c[15], c[14] / (double)(c[15] > 0 ? c[15] : 1));
  return *bad ? 1 : 0;
}
