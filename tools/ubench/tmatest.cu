// Minimal 2D tensor-map TMA copy (FP64 field-major rows -> shared memory), variants chosen by argv:
//   tmatest <col0> <smem_offset_bytes> <boxcols>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__global__ void k(const __grid_constant__ CUtensorMap tm, int col0, int off, int rows, int cols, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  double* dst = reinterpret_cast<double*>(sm + off);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(rows * cols * 8) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                 ::"r"(su32(dst)), "l"(reinterpret_cast<unsigned long long>(&tm)), "r"(col0), "r"(0), "r"(su32(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("{\n .reg .pred p;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(su32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < rows * cols; i += blockDim.x) out[i] = dst[i];
}
int main(int argc, char** argv) {
  const int col0 = argc > 1 ? atoi(argv[1]) : 0, off = argc > 2 ? atoi(argv[2]) : 0, cols = argc > 3 ? atoi(argv[3]) : 34;
  const int vpad = 256, rows = 8;
  double* g; cudaMalloc(&g, sizeof(double) * vpad * rows);
  double h[256 * 8]; for (int i = 0; i < vpad * rows; ++i) h[i] = i;
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  double* out; cudaMallocManaged(&out, sizeof(double) * rows * cols);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)vpad, (cuuint64_t)rows}, str[1] = {(cuuint64_t)vpad * 8};
  cuuint32_t box[2] = {(cuuint32_t)cols, (cuuint32_t)rows}, es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, 128, 64 * 1024>>>(m, col0, off, rows, cols, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("col0=%d off=%d cols=%d: %s; out[0]=%g out[1]=%g out[cols]=%g\n", col0, off, cols, cudaGetErrorString(e), out[0], out[1], out[cols]);
  return 0;
}
