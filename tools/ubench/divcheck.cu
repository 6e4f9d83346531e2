// Validates the shared-reciprocal division used by the sweep kernels (vmath.cuh divr): for
// y = RN(1/b) (__drcp_rn), q = RN(a*y), e = a - b*q (exact, FMA), q' = RN(q + e*y) must equal
// RN(a/b) bit for bit (Markstein's theorem) in the guarded exponent range. Random a, b with random
// mantissas and exponents in [-60, 60], plus adversarial mantissas (all ones / power of two /
// near-halfway quotients), compared against the IEEE division.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
__device__ double mk(uint64_t r, int e) {
  uint64_t mant = r & ((1ull << 52) - 1);
  const int mode = (r >> 60) & 7;
  if (mode == 0) mant = (1ull << 52) - 1;          // all ones
  if (mode == 1) mant = 0;                          // power of two
  if (mode == 2) mant = (r >> 20) & 0xfff;          // few low bits
  if (mode == 3) mant = ((1ull << 52) - 1) ^ ((r >> 13) & 0xff);
  const uint64_t bits = ((uint64_t)((r >> 63) & 1) << 63) | ((uint64_t)(1023 + e) << 52) | mant;
  return __longlong_as_double((long long)bits);
}
__global__ void k(uint64_t seed, long long n, unsigned long long* bad, double* ex) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint64_t r1 = mix(seed ^ (2 * i)), r2 = mix(seed ^ (2 * i + 1)), r3 = mix(r1 ^ r2);
    const double a = mk(r1, (int)(r3 % 121) - 60), b = mk(r2, (int)((r3 >> 8) % 121) - 60);
    const double y = __drcp_rn(b);
    const double q = a * y;
    const double e = fma(-b, q, a);
    const double q2 = fma(e, y, q);
    const double ref = a / b;
    if (__double_as_longlong(q2) != __double_as_longlong(ref)) {
      const unsigned long long k = atomicAdd(bad, 1ull);
      if (k < 4) { ex[3 * k] = a; ex[3 * k + 1] = b; ex[3 * k + 2] = q2 - ref; }
    }
  }
}
int main() {
  unsigned long long* bad; double* ex;
  cudaMallocManaged(&bad, 8); cudaMallocManaged(&ex, 12 * 8); *bad = 0;
  const long long n = 1ll << 33;
  k<<<148 * 16, 256>>>(12345, n, bad, ex);
  cudaDeviceSynchronize();
  printf("samples %lld mismatches %llu\n", n, *bad);
  for (unsigned long long i = 0; i < (*bad < 4 ? *bad : 4); ++i) printf("  a=%.17g b=%.17g diff=%g\n", ex[3*i], ex[3*i+1], ex[3*i+2]);
  return 0;
}
