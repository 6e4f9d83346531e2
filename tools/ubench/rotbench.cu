// Cycles per iteration of the shape-matching rotation extraction (shape.cuh extract_rotation),
// one warp, forced iteration counts (tol2 = 0). Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   --fmad=false -I paper_1906_05260_b200/csrc tools/ubench/rotbench.cu -o /tmp/rotbench
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "shape.cuh"

// the previous version (two Newton steps, Horner Taylor, per-iteration renormalisation), for comparison
// Reciprocal for the rotation chain: MUFU seed + two Newton steps (relative error ~1 ulp).
__device__ __forceinline__ double rcp_fast_old(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// extract_rotation, bundling.cpp:50-67: the same iteration (omega = sum R_a x B_a / (|sum
// R_a . B_a| + 1e-9), q <- AngleAxis(|omega|, omega^) q, normalize, stop at |omega| < 1e-9).
// The loop is one serial dependency chain (~10 iterations warm-started at C3, up to ~20), so it
// is written for latency (shape matching is tolerance-pinned): FMA trees, a Newton
// reciprocal, and for half angles below 1e-2 the increment [cos(a/2), sin(a/2)/a * omega] from
// its Taylor series in a^2 (truncation < 1e-20 relative); larger steps take the general route.
// The product of two unit quaternions has |p|^2 = 1 + O(1e-15), so the renormalisation uses
// 1/sqrt(n) = 1 - (n-1)/2 + 3/8 (n-1)^2 (exact to 1e-30 there; rsqrt otherwise).
__device__ __forceinline__ vm::Q4 extract_rotation_old(const vm::M3& B, const vm::Q4& guess, int* iters = nullptr,
                                                   int max_iterations = 100, double tol2 = 1e-18) {
  using namespace vm;
  Q4 q = qnormalized(guess);
  int it = 0;
#pragma unroll 1
  for (; it < max_iterations; ++it) {
    // R = toRotationMatrix(q)
    const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
    const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
    const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
    const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
    const double R[3][3] = {{1.0 - (tyy + tzz), txy - twz, txz + twy},
                            {txy + twz, 1.0 - (txx + tzz), tyz - twx},
                            {txz - twy, tyz + twx, 1.0 - (txx + tyy)}};
    // w = sum_a col(R, a) x col(B, a); d = sum_a col(R, a) . col(B, a)
    double wx[3], wy[3], wz[3], dd[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double r0 = R[0][a], r1 = R[1][a], r2 = R[2][a];
      const double b0 = B.m[0][a], b1 = B.m[1][a], b2 = B.m[2][a];
      wx[a] = fma(r1, b2, -r2 * b1);
      wy[a] = fma(r2, b0, -r0 * b2);
      wz[a] = fma(r0, b1, -r1 * b0);
      dd[a] = fma(r0, b0, fma(r1, b1, r2 * b2));
    }
    const double ox = (wx[0] + wx[1]) + wx[2], oy = (wy[0] + wy[1]) + wy[2], oz = (wz[0] + wz[1]) + wz[2];
    const double inv = rcp_fast_old(fabs((dd[0] + dd[1]) + dd[2]) + 1e-9);
    const double w2 = fma(ox, ox, fma(oy, oy, oz * oz));
    const double a2 = (w2 * inv) * inv;  // |omega|^2
    if (a2 < tol2) break;  // |omega| < tolerance (1e-9)
    const double x2 = 0.25 * a2;  // (angle / 2)^2
    double k, c;  // k = sin(angle/2) / angle, c = cos(angle/2)
    if (x2 < 1e-4) {
      k = 0.5 * fma(-x2 * (1.0 / 6), fma(-x2 * (1.0 / 20), fma(-x2 * (1.0 / 42), fma(-x2, 1.0 / 72, 1.0), 1.0), 1.0), 1.0);
      c = fma(-x2 * 0.5,
              fma(-x2 * (1.0 / 12), fma(-x2 * (1.0 / 30), fma(-x2 * (1.0 / 56), fma(-x2, 1.0 / 90, 1.0), 1.0), 1.0), 1.0),
              1.0);
    } else {
      const double2 kc = vdev::rotation_increment_general(a2);
      k = kc.x;
      c = kc.y;
    }
    const double ki = k * inv;
    const double vx = ki * ox, vy = ki * oy, vz = ki * oz;
    // p = [c, v] * q (Hamilton product)
    const double pw = fma(c, q.w, -fma(vx, q.x, fma(vy, q.y, vz * q.z)));
    const double px = fma(c, q.x, fma(vx, q.w, fma(vy, q.z, -vz * q.y)));
    const double py = fma(c, q.y, fma(vy, q.w, fma(vz, q.x, -vx * q.z)));
    const double pz = fma(c, q.z, fma(vz, q.w, fma(vx, q.y, -vy * q.x)));
    const double e = fma(pw, pw, fma(px, px, fma(py, py, pz * pz))) - 1.0;
    const double r = fabs(e) < 1e-6 ? fma(e, fma(e, 0.375, -0.5), 1.0) : rsqrt(e + 1.0);
    q = Q4{pw * r, px * r, py * r, pz * r};
  }
  if (iters) *iters = it;
  return q;
}


template <bool kOld>
__global__ void k_rot(const double* B, const double* g, int iters, double tol2, double* out, long long* cyc) {
  vm::M3 m;
  const int l = threadIdx.x;  // 32 identical copies: per-lane loads keep the chain in vector registers
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) m.m[a][b] = B[9 * l + 3 * a + b];
  const vm::Q4 guess{g[4 * l], g[4 * l + 1], g[4 * l + 2], g[4 * l + 3]};
  __syncwarp();
  const long long t0 = clock64();
  int n = 0;
  const vm::Q4 q = kOld ? extract_rotation_old(m, guess, &n, iters, tol2) : vdev::extract_rotation(m, guess, &n, iters, tol2);
  if (threadIdx.x == 0) {
    out[0] = q.w;
    out[1] = q.x;
    out[2] = q.y;
    out[3] = q.z;
    out[4] = n;
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  const double hB[9] = {1.02, 0.05, -0.01, 0.03, 0.97, 0.02, -0.02, 0.04, 1.05};
  const double hg[4] = {0.999, 0.01, -0.02, 0.03};
  double *B, *g, *out;
  long long* cyc;
  cudaMalloc(&B, 72 * 32);
  cudaMalloc(&g, 32 * 32);
  cudaMalloc(&out, 256);
  cudaMalloc(&cyc, 8);
  for (int l = 0; l < 32; ++l) {
    cudaMemcpy(B + 9 * l, hB, 72, cudaMemcpyHostToDevice);
    cudaMemcpy(g + 4 * l, hg, 32, cudaMemcpyHostToDevice);
  }
  for (int old = 0; old < 2; ++old)
    for (int rep = 0; rep < 2; ++rep)
      for (int it : {0, 1, 2, 5, 10, 20, 40}) {
        if (old) k_rot<true><<<1, 32>>>(B, g, it, 0.0, out, cyc);
        else k_rot<false><<<1, 32>>>(B, g, it, 0.0, out, cyc);
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("%s iters %2d: %6lld cycles\n", old ? "old" : "new", it, c);
      }
  // converged results (tol 1e-9) of both, on random stretched matrices and perturbed guesses
  double maxd = 0;
  int maxdn = 0;
  srand(1);
  for (int t = 0; t < 2000; ++t) {
    double b[9], q[4];
    for (int i = 0; i < 9; ++i) b[i] = (i % 4 == 0 ? 1.0 : 0.0) + 0.3 * (rand() / (double)RAND_MAX - 0.5);
    for (int i = 0; i < 4; ++i) q[i] = (i == 0 ? 1.0 : 0.0) + 0.2 * (rand() / (double)RAND_MAX - 0.5);
    for (int l = 0; l < 32; ++l) {
      cudaMemcpy(B + 9 * l, b, 72, cudaMemcpyHostToDevice);
      cudaMemcpy(g + 4 * l, q, 32, cudaMemcpyHostToDevice);
    }
    double r0[5], r1[5];
    k_rot<false><<<1, 32>>>(B, g, 100, 1e-18, out, cyc);
    cudaMemcpy(r0, out, 40, cudaMemcpyDeviceToHost);
    k_rot<true><<<1, 32>>>(B, g, 100, 1e-18, out, cyc);
    cudaMemcpy(r1, out, 40, cudaMemcpyDeviceToHost);
    double d = 0;
    for (int i = 0; i < 4; ++i) d = fmax(d, fabs(r0[i] - r1[i]));
    maxd = fmax(maxd, d);
    maxdn = abs((int)r0[4] - (int)r1[4]) > maxdn ? abs((int)r0[4] - (int)r1[4]) : maxdn;
  }
  printf("converged new vs old over 2000 cases: max |dq| %.3e, max iteration-count difference %d\n", maxd, maxdn);
  return 0;
}
