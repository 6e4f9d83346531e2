// Exclusive prefix sum over int32 counts with a device-side length — the counting-sort /
// compaction primitive of the broad phase (candidate offsets, cell starts), the contact
// compaction and the external-block incidence lists. Three passes (tile scan, partials scan,
// add) so the launch shape depends only on the capacity and a CUDA graph can replay it.
#include "kernels.cuh"

namespace vdev {

bool g_pdl = false;

namespace {

constexpr int kThreads = 512;
constexpr int kPerThread = 8;
constexpr int kTile = kThreads * kPerThread;  // 4096 elements per CTA

__device__ __forceinline__ int warp_incl(int v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan of one int per thread; returns the block total via *total.
__device__ int block_excl(int v, int* total) {
  __shared__ int warp_sums[kThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int incl = warp_incl(v);
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int s = lane < kThreads / 32 ? warp_sums[lane] : 0;
    s = warp_incl(s);
    if (lane < kThreads / 32) warp_sums[lane] = s;
  }
  __syncthreads();
  const int base = wid ? warp_sums[wid - 1] : 0;
  *total = warp_sums[kThreads / 32 - 1];
  __syncthreads();
  return base + incl - v;
}

__global__ void k_tile_scan(const int* __restrict__ in, int* __restrict__ out, long long n_cap,
                            const int* n_dev, int* partials) {
  pdl_wait();
  pdl_trigger();
  const long long n = n_dev ? static_cast<long long>(*n_dev) : n_cap;
  const long long base = static_cast<long long>(blockIdx.x) * kTile;
  if (base > n) return;
  int vals[kPerThread];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    const long long i = base + threadIdx.x * kPerThread + k;
    vals[k] = i < n ? in[i] : 0;
    sum += vals[k];
  }
  int total;
  int run = block_excl(sum, &total);
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    const long long i = base + threadIdx.x * kPerThread + k;
    if (i <= n) out[i] = run;
    run += vals[k];
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = total;
}

__global__ void k_partials_scan(int* partials, long long n_cap, const int* n_dev) {
  pdl_wait();
  pdl_trigger();
  const long long n = n_dev ? static_cast<long long>(*n_dev) : n_cap;
  const long long parts = n / kTile + 1;
  int carry = 0;
  for (long long b0 = 0; b0 < parts; b0 += kThreads) {
    const long long b = b0 + threadIdx.x;
    const int v = b < parts ? partials[b] : 0;
    int total;
    const int ex = block_excl(v, &total);
    if (b < parts) partials[b] = carry + ex;
    carry += total;
  }
}

__global__ void k_add(int* __restrict__ out, long long n_cap, const int* n_dev, const int* __restrict__ partials) {
  pdl_wait();
  pdl_trigger();
  const long long n = n_dev ? static_cast<long long>(*n_dev) : n_cap;
  const long long base = static_cast<long long>(blockIdx.x) * kTile;
  if (base > n || blockIdx.x == 0) return;
  const int add = partials[blockIdx.x];
  for (int k = threadIdx.x; k < kTile; k += kThreads) {
    const long long i = base + k;
    if (i <= n) out[i] += add;
  }
}

// Small scans (n_cap <= kSmallScan): one CTA does it all, one launch instead of three. The live
// length n is staged through shared memory with coalesced loads (one pad word per 32 keeps the
// per-thread chunk walks conflict-free), each thread scans a contiguous chunk of ceil(n / 512),
// a block scan of the chunk totals gives the offsets, and the result leaves coalesced.
constexpr long long kSmallScan = 8 * kTile;  // 32768
__host__ __device__ constexpr long long small_pad(long long i) { return i + (i >> 5); }
__global__ void k_scan_small(const int* __restrict__ in, int* __restrict__ out, long long n_cap, const int* n_dev) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ int sm[];
  const int n = static_cast<int>(n_dev ? static_cast<long long>(*n_dev) : n_cap);
  for (int i = threadIdx.x; i < n; i += kThreads) sm[small_pad(i)] = in[i];
  __syncthreads();
  const int ch = (n + kThreads - 1) / kThreads;
  const int b = threadIdx.x * ch, e = min(b + ch, n);
  int sum = 0;
  for (int k = b; k < e; ++k) sum += sm[small_pad(k)];
  int total;
  int run = block_excl(sum, &total);
  for (int k = b; k < e; ++k) {
    const int v = sm[small_pad(k)];
    sm[small_pad(k)] = run;
    run += v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kThreads) out[i] = sm[small_pad(i)];
  if (threadIdx.x == 0) out[n] = total;
}

__global__ void k_fill(FillList f) {
  pdl_wait();
  pdl_trigger();
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (int a = 0; a < f.n; ++a)
    for (long long i = t; i < f.count[a]; i += stride) f.ptr[a][i] = f.value[a];
}

}  // namespace

void launch_fill(const FillList& f, cudaStream_t st) {
  if (f.n == 0) return;
  long long mx = 0;
  for (int a = 0; a < f.n; ++a) mx = f.count[a] > mx ? f.count[a] : mx;
  const long long b = (mx + kThreads - 1) / kThreads;
  launch_kernel(k_fill, static_cast<unsigned>(b < 1 ? 1 : (b > 148 * 8 ? 148 * 8 : b)), kThreads, 0, st, g_pdl, f);
}

long long scan_partials_needed(long long n) { return n / kTile + 2; }

// out[i] = sum(in[0..i)) for i in [0, n]; n = *n_dev if given (must be <= n_cap), else n_cap.
void scan_exclusive(const int* in, int* out, long long n_cap, const int* n_dev, int* partials, int parts,
                    cudaStream_t st) {
  (void)parts;
  if (n_cap <= kSmallScan) {
    // (host-side, at graph-record time; per device, so set on every call)
    cudaFuncSetAttribute(k_scan_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(int) * (small_pad(kSmallScan) + 1)));
    const std::size_t smem = sizeof(int) * static_cast<std::size_t>(small_pad(n_cap) + 1);
    launch_kernel(k_scan_small, 1, kThreads, smem, st, g_pdl, in, out, n_cap, n_dev);
    return;
  }
  const long long blocks = n_cap / kTile + 1;
  launch_kernel(k_tile_scan, static_cast<unsigned>(blocks), kThreads, 0, st, g_pdl, in, out, n_cap, n_dev, partials);
  launch_kernel(k_partials_scan, 1, kThreads, 0, st, g_pdl, partials, n_cap, n_dev);
  launch_kernel(k_add, static_cast<unsigned>(blocks), kThreads, 0, st, g_pdl, out, n_cap, n_dev, partials);
}

}  // namespace vdev
