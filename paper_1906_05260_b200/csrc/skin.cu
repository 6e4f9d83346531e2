// Skinning kernels (skinning.cpp): bind_skin, smooth_binding, deform_mesh and the pill
// transforms of a solver's live state. Every kernel keeps the reference's operation order
// (compiled --fmad=false), so bindings and deformed meshes equal the reference bit for bit.
//
//   k_pill_transforms  one thread per slot: element e of a rod -> (midpoint center, midpoint
//                      scale, frame), rod-major element-major (skinning.cpp:9-22)
//   k_skin_prep        per-pill constants of pill_project (pill.cuh)
//   k_skin_bind        one warp per mesh vertex: inverse-square scores of every pill (lanes over
//                      pills), then `keep` rounds of warp arg-max (score desc, pill asc — the
//                      partial_sort order), renormalized in that order, listed by pill
//                      (skinning.cpp:59-105)
//   k_skin_smooth      one thread per vertex: the one-ring blend of smooth_binding in the
//                      reference's visit order (own entries, then neighbours ascending), stable
//                      per-pill accumulation (the std::map), top-k, renormalize (:107-163)
//   k_skin_deform      one thread per vertex: linear blend skinning (:165-185)
#include <algorithm>
#include <stdexcept>
#include <string>

#include "kernels.cuh"
#include "pill.cuh"
#include "skin.h"
#include "solver.h"

namespace vdev {

namespace {

constexpr int kThreads = 256;

int grid_of(long long n, int per_block) {
  const long long b = (n + per_block - 1) / per_block;
  return static_cast<int>(std::max(1ll, std::min(b, 148ll * 32)));
}

__global__ void k_pill_transforms(World w, const double* __restrict__ X, double* __restrict__ out) {
  const int vp = w.vpad;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < w.V; v += gridDim.x * blockDim.x) {
    const int k = w.slot_loc[v];
    if (k >= w.slot_m[v]) continue;  // last vertex of a rod: no element
    const long long i = v - w.slot_rod[v];
    double* o = out + 8 * i;
    const long long a = v, b = v + 1;
    o[0] = 0.5 * (X[CX * (long long)vp + a] + X[CX * (long long)vp + b]);
    o[1] = 0.5 * (X[CY * (long long)vp + a] + X[CY * (long long)vp + b]);
    o[2] = 0.5 * (X[CZ * (long long)vp + a] + X[CZ * (long long)vp + b]);
    o[3] = 0.5 * (X[S * (long long)vp + a] + X[S * (long long)vp + b]);
    o[4] = X[QW * (long long)vp + a];
    o[5] = X[QX * (long long)vp + a];
    o[6] = X[QY * (long long)vp + a];
    o[7] = X[QZ * (long long)vp + a];
  }
}

__global__ void k_skin_prep(int np, const double* __restrict__ pv, PillPrep* __restrict__ prep) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
    const double* q = pv + 8ll * p;
    prep[p] = prep_pill(PillV{V3{q[0], q[1], q[2]}, V3{q[3], q[4], q[5]}, q[6], q[7]});
  }
}

__device__ __forceinline__ bool score_before(double sa, int pa, double sb, int pb) {
  return sa != sb ? sa > sb : pa < pb;  // partial_sort comparator, skinning.cpp:84-87
}

__global__ void k_skin_bind(int nv, const double* __restrict__ verts, int np, const PillPrep* __restrict__ prep,
                            int keep, double eps, double* __restrict__ scratch, int* __restrict__ out_pills,
                            double* __restrict__ out_w, int* __restrict__ clamped) {
  const int lane = threadIdx.x & 31;
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  double* scr = scratch + warp * np;
  for (long long v = warp; v < nv; v += nwarps) {
    const V3 x{verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]};
    bool cl = false;
    for (int p = lane; p < np; p += 32) {
      double t;
      bool deg;
      const double d = project(x, prep[p], t, deg);
      cl = cl || d < 0.0;
      const double dc = d < eps ? eps : d;  // std::max(d, epsilon)
      scr[p] = 1.0 / (dc * dc);
    }
    __syncwarp();
    if (__any_sync(0xffffffffu, cl) && lane == 0) clamped[v] = 1;
    int* op = out_pills + v * keep;
    double* ow = out_w + v * keep;
    for (int r = 0; r < keep; ++r) {  // r-th best (score desc, pill asc); taken scores are marked -1
      double bs = -1.0;
      int bp = 0x7fffffff;
      for (int p = lane; p < np; p += 32) {
        const double s = scr[p];
        if (s >= 0.0 && (bs < 0.0 || score_before(s, p, bs, bp))) {
          bs = s;
          bp = p;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double s2 = __shfl_xor_sync(0xffffffffu, bs, o);
        const int p2 = __shfl_xor_sync(0xffffffffu, bp, o);
        if (s2 >= 0.0 && (bs < 0.0 || score_before(s2, p2, bs, bp))) {
          bs = s2;
          bp = p2;
        }
      }
      if (lane == (bp & 31)) scr[bp] = -1.0;
      if (lane == 0) {
        op[r] = bp;
        ow[r] = bs;
      }
      __syncwarp();
    }
    if (lane == 0) {
      double total = 0.0;
      for (int r = 0; r < keep; ++r) total += ow[r];
      for (int r = 0; r < keep; ++r) ow[r] = ow[r] / total;
      for (int a = 1; a < keep; ++a) {  // list by pill index (skinning.cpp:90-92)
        const int pk = op[a];
        const double wk = ow[a];
        int b = a - 1;
        while (b >= 0 && op[b] > pk) {
          op[b + 1] = op[b];
          ow[b + 1] = ow[b];
          --b;
        }
        op[b + 1] = pk;
        ow[b + 1] = wk;
      }
    }
    __syncwarp();
  }
}

__global__ void k_skin_smooth(int nv, const int* __restrict__ off, const int* __restrict__ pills,
                              const double* __restrict__ w, const int* __restrict__ nb_off, const int* __restrict__ nb,
                              const long long* __restrict__ scr_off, int* __restrict__ scr_p, double* __restrict__ scr_w,
                              int max_influences, int stride, int* __restrict__ out_p, double* __restrict__ out_w,
                              int* __restrict__ cnt) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    int* sp = scr_p + scr_off[v];
    double* sw = scr_w + scr_off[v];
    int n = 0;
    for (int k = off[v]; k < off[v + 1]; ++k) {
      sp[n] = pills[k];
      sw[n++] = 0.5 * w[k];
    }
    const int n0 = nb_off[v], n1 = nb_off[v + 1];
    if (n1 > n0) {
      const double share = 0.5 / static_cast<double>(n1 - n0);
      for (int q = n0; q < n1; ++q) {
        const int u = nb[q];
        for (int k = off[u]; k < off[u + 1]; ++k) {
          sp[n] = pills[k];
          sw[n++] = share * w[k];
        }
      }
    } else {
      for (int k = off[v]; k < off[v + 1]; ++k) {
        sp[n] = pills[k];
        sw[n++] = 0.5 * w[k];
      }
    }
    // stable sort by pill: per-pill contributions keep their visit order
    for (int a = 1; a < n; ++a) {
      const int pk = sp[a];
      const double wk = sw[a];
      int b = a - 1;
      while (b >= 0 && sp[b] > pk) {
        sp[b + 1] = sp[b];
        sw[b + 1] = sw[b];
        --b;
      }
      sp[b + 1] = pk;
      sw[b + 1] = wk;
    }
    // std::map accumulation: blended[p] starts at 0.0, += in visit order
    int nd = 0;
    for (int a = 0; a < n; ++a) {
      if (nd > 0 && sp[nd - 1] == sp[a]) {
        sw[nd - 1] += sw[a];
      } else {
        sp[nd] = sp[a];
        sw[nd] = 0.0 + sw[a];
        ++nd;
      }
    }
    // top `keep` (weight desc, pill asc): selected entries are marked by negating their pill + 1
    const int keep = min(max_influences, nd);
    double total = 0.0;
    for (int r = 0; r < keep; ++r) {
      int best = -1;
      for (int a = 0; a < nd; ++a)
        if (sp[a] >= 0 && (best < 0 || score_before(sw[a], sp[a], sw[best], sp[best]))) best = a;
      total += sw[best];
      sp[best] = -sp[best] - 1;
    }
    // emit the selected entries by ascending pill (the distinct list is ascending)
    int o = 0;
    for (int a = 0; a < nd; ++a) {
      if (sp[a] >= 0) continue;
      out_p[static_cast<long long>(v) * stride + o] = -sp[a] - 1;
      out_w[static_cast<long long>(v) * stride + o] = sw[a] / total;
      ++o;
    }
    cnt[v] = o;
  }
}

__global__ void k_compact_csr(int nv, int stride, const int* __restrict__ off, const int* __restrict__ in_p,
                              const double* __restrict__ in_w, int* __restrict__ out_p, double* __restrict__ out_w) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x)
    for (int k = off[v]; k < off[v + 1]; ++k) {
      out_p[k] = in_p[static_cast<long long>(v) * stride + (k - off[v])];
      out_w[k] = in_w[static_cast<long long>(v) * stride + (k - off[v])];
    }
}

// Per frame, per pill: cur.scale / ref.scale (the one division of deform_mesh's inner term,
// the same IEEE quotient for every vertex the pill influences) into the scale slot of the
// frame table, so the per-influence work is division-free.
__global__ void k_skin_frame(int np, const double* __restrict__ rest, const double* __restrict__ cur,
                             double* __restrict__ frame) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 8 * np; i += gridDim.x * blockDim.x) {
    const int p = i >> 3, f = i & 7;
    frame[i] = f == 3 ? cur[8ll * p + 3] / rest[8ll * p + 3] : cur[i];
  }
}

// deform_mesh, skinning.cpp:165-185: local = conj(ref.rotation) * (rest - ref.center);
// blended += w * (cur.center + (cur.scale / ref.scale) * (cur.rotation * local)); the frame
// table carries cur.scale / ref.scale in its scale slot (k_skin_frame).
constexpr int kDeformThreads = 128;

__device__ __forceinline__ void ld8(const double* __restrict__ p, double (&o)[8]) {
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double2 v = __ldg(q + i);
    o[2 * i] = v.x;
    o[2 * i + 1] = v.y;
  }
}

// One thread per vertex; the pill records (64 B, L2/L1-resident) are read as 16-byte vectors.
// FP64-pipe bound: ~75 dependent-free FP64 operations per influence (two quaternion rotations),
// --fmad=false keeps the reference's rounding.
__global__ void __launch_bounds__(kDeformThreads) k_skin_deform(int nv, const double* __restrict__ verts,
                                                                const int* __restrict__ off,
                                                                const int* __restrict__ pills,
                                                                const double* __restrict__ w,
                                                                const double* __restrict__ rest,
                                                                const double* __restrict__ cur,
                                                                double* __restrict__ out) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    const V3 x{verts[3ll * v], verts[3ll * v + 1], verts[3ll * v + 2]};
    V3 blended{0, 0, 0};
    const int k1 = off[v + 1];
    for (int k = off[v]; k < k1; ++k) {
      const int p = pills[k];
      double r[8], c[8];
      ld8(rest + 8ll * p, r);
      ld8(cur + 8ll * p, c);
      const V3 local = qrot(qconj(Q4{r[4], r[5], r[6], r[7]}), x - V3{r[0], r[1], r[2]});
      const V3 moved = V3{c[0], c[1], c[2]} + c[3] * qrot(Q4{c[4], c[5], c[6], c[7]}, local);
      blended = blended + w[k] * moved;
    }
    out[3ll * v] = blended.x;
    out[3ll * v + 1] = blended.y;
    out[3ll * v + 2] = blended.z;
  }
}

}  // namespace

void launch_pill_transforms(const World& w, const double* X, double* out, cudaStream_t st) {
  if (w.V > 0) k_pill_transforms<<<grid_of(w.V, kThreads), kThreads, 0, st>>>(w, X, out);
}

}  // namespace vdev

namespace vhost {

namespace {
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
template <typename T>
T* dmalloc(std::size_t n) {
  void* p = nullptr;
  ck(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)), "cudaMalloc");
  return static_cast<T*>(p);
}
void require(bool ok, const char* msg) {  // types.h:67-69
  if (!ok) throw std::invalid_argument(msg);
}
}  // namespace

Skin::Skin(const std::vector<V3>& vertices, const std::vector<std::array<int, 3>>& triangles,
           const std::vector<PillData>& rest_pills, const std::vector<double>& rest_transforms, int max_influences,
           double epsilon) {
  require(!rest_pills.empty(), "skin binding needs at least one pill");
  require(rest_pills.size() * kTransformDoubles == rest_transforms.size(), "pill list and transform list must match");
  require(max_influences >= 1, "max_influences must be at least 1");
  require(epsilon > 0.0, "epsilon must be positive");
  nv_ = static_cast<int>(vertices.size());
  np_ = static_cast<int>(rest_pills.size());
  max_influences_ = max_influences;
  keep_ = std::min(max_influences, np_);
  // one-ring neighbours from the triangles, sorted and unique (skinning.cpp:109-121)
  std::vector<std::vector<int>> nb(nv_);
  for (const auto& t : triangles)
    for (int k = 0; k < 3; ++k) {
      const int a = t[k], b = t[(k + 1) % 3];
      if (a < 0 || a >= nv_ || b < 0 || b >= nv_) throw std::out_of_range("triangle vertex out of range");
      nb[a].push_back(b);
      nb[b].push_back(a);
    }
  nb_off_.assign(1, 0);
  for (auto& l : nb) {
    std::sort(l.begin(), l.end());
    l.erase(std::unique(l.begin(), l.end()), l.end());
    nb_list_.insert(nb_list_.end(), l.begin(), l.end());
    nb_off_.push_back(static_cast<int>(nb_list_.size()));
  }
  ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
  std::vector<double> vx(3ull * nv_), pv(8ull * np_);
  for (int v = 0; v < nv_; ++v) {
    vx[3ll * v] = vertices[v].x;
    vx[3ll * v + 1] = vertices[v].y;
    vx[3ll * v + 2] = vertices[v].z;
  }
  for (int p = 0; p < np_; ++p) {
    const PillData& q = rest_pills[p];
    const double e[8] = {q.c0.x, q.c0.y, q.c0.z, q.c1.x, q.c1.y, q.c1.z, q.r0, q.r1};
    std::copy(e, e + 8, pv.begin() + 8ll * p);
  }
  d_verts_ = dmalloc<double>(vx.size());
  d_rest_ = dmalloc<double>(rest_transforms.size());
  d_cur_ = dmalloc<double>(rest_transforms.size());
  d_frame_ = dmalloc<double>(rest_transforms.size());
  d_off_ = dmalloc<int>(nv_ + 1ull);
  nnz_ = static_cast<long long>(nv_) * keep_;
  d_pills_ = dmalloc<int>(nnz_);
  d_weights_ = dmalloc<double>(nnz_);
  d_cnt_ = dmalloc<int>(nv_ + 1ull);
  d_out_ = dmalloc<double>(3ull * nv_);
  ck(cudaMemcpyAsync(d_verts_, vx.data(), vx.size() * 8, cudaMemcpyHostToDevice, stream_), "upload");
  ck(cudaMemcpyAsync(d_rest_, rest_transforms.data(), rest_transforms.size() * 8, cudaMemcpyHostToDevice, stream_),
     "upload");
  // bind: pill constants, then one warp per vertex over a per-warp score row
  double* d_pv = dmalloc<double>(pv.size());
  vdev::PillPrep* d_prep = dmalloc<vdev::PillPrep>(np_);
  int* d_clamped = dmalloc<int>(nv_);
  ck(cudaMemcpyAsync(d_pv, pv.data(), pv.size() * 8, cudaMemcpyHostToDevice, stream_), "upload");
  ck(cudaMemsetAsync(d_clamped, 0, sizeof(int) * std::max(nv_, 1), stream_), "memset");
  vdev::k_skin_prep<<<vdev::grid_of(np_, 256), 256, 0, stream_>>>(np_, d_pv, d_prep);
  const long long want = std::min<long long>(std::max(nv_, 1), 148ll * 64);
  const int blocks = static_cast<int>((want * 32 + 255) / 256);
  double* d_scr = dmalloc<double>(static_cast<std::size_t>(blocks) * 8 * np_);  // one score row per warp
  vdev::k_skin_bind<<<blocks, 256, 0, stream_>>>(nv_, d_verts_, np_, d_prep, keep_, epsilon, d_scr, d_pills_,
                                                 d_weights_, d_clamped);
  ck(cudaGetLastError(), "bind launch");
  std::vector<int> off(nv_ + 1), cl(nv_);
  for (int v = 0; v <= nv_; ++v) off[v] = v * keep_;
  ck(cudaMemcpyAsync(d_off_, off.data(), off.size() * 4, cudaMemcpyHostToDevice, stream_), "upload");
  ck(cudaMemcpyAsync(cl.data(), d_clamped, sizeof(int) * nv_, cudaMemcpyDeviceToHost, stream_), "download");
  ck(cudaStreamSynchronize(stream_), "bind");
  for (int c : cl) clamped_ += c;
  cudaFree(d_pv);
  cudaFree(d_prep);
  cudaFree(d_clamped);
  cudaFree(d_scr);
}

Skin::~Skin() {
  if (stream_) cudaStreamSynchronize(stream_);
  for (void* p : {static_cast<void*>(d_verts_), static_cast<void*>(d_rest_), static_cast<void*>(d_cur_), static_cast<void*>(d_frame_),
                  static_cast<void*>(d_off_), static_cast<void*>(d_pills_), static_cast<void*>(d_weights_),
                  static_cast<void*>(d_cnt_), static_cast<void*>(d_out_), static_cast<void*>(d_nb_off_),
                  static_cast<void*>(d_nb_), static_cast<void*>(d_scr_pill_), static_cast<void*>(d_scr_w_),
                  static_cast<void*>(d_scr_off_), static_cast<void*>(d_tmp_pills_), static_cast<void*>(d_tmp_weights_),
                  static_cast<void*>(d_scan_tmp_)})
    if (p) cudaFree(p);
  if (stream_) cudaStreamDestroy(stream_);
}

void Skin::smooth(int iterations) {
  if (iterations <= 0) return;
  if (!d_nb_off_) {  // scratch: every candidate of the one-ring blend, capacity keep x (1 + degree)
    d_nb_off_ = dmalloc<int>(nb_off_.size());
    d_nb_ = dmalloc<int>(nb_list_.size());
    std::vector<long long> so(nv_ + 1, 0);
    for (int v = 0; v < nv_; ++v) {
      const int deg = nb_off_[v + 1] - nb_off_[v];
      so[v + 1] = so[v] + static_cast<long long>(max_influences_) * (1 + std::max(deg, 1));
    }
    scratch_cap_ = so[nv_];
    d_scr_off_ = dmalloc<long long>(so.size());
    d_scr_pill_ = dmalloc<int>(scratch_cap_);
    d_scr_w_ = dmalloc<double>(scratch_cap_);
    d_tmp_pills_ = dmalloc<int>(nnz_);
    d_tmp_weights_ = dmalloc<double>(nnz_);
    scan_parts_ = static_cast<int>(vdev::scan_partials_needed(nv_));
    d_scan_tmp_ = dmalloc<int>(scan_parts_);
    ck(cudaMemcpyAsync(d_nb_off_, nb_off_.data(), nb_off_.size() * 4, cudaMemcpyHostToDevice, stream_), "upload");
    if (!nb_list_.empty())
      ck(cudaMemcpyAsync(d_nb_, nb_list_.data(), nb_list_.size() * 4, cudaMemcpyHostToDevice, stream_), "upload");
    ck(cudaMemcpyAsync(d_scr_off_, so.data(), so.size() * 8, cudaMemcpyHostToDevice, stream_), "upload");
  }
  const int stride = std::min(max_influences_, np_);
  for (int it = 0; it < iterations; ++it) {
    vdev::k_skin_smooth<<<vdev::grid_of(nv_, 128), 128, 0, stream_>>>(
        nv_, d_off_, d_pills_, d_weights_, d_nb_off_, d_nb_, d_scr_off_, d_scr_pill_, d_scr_w_, max_influences_, stride,
        d_tmp_pills_, d_tmp_weights_, d_cnt_);
    vdev::scan_exclusive(d_cnt_, d_off_, nv_, nullptr, d_scan_tmp_, scan_parts_, stream_);
    vdev::k_compact_csr<<<vdev::grid_of(nv_, 256), 256, 0, stream_>>>(nv_, stride, d_off_, d_tmp_pills_,
                                                                      d_tmp_weights_, d_pills_, d_weights_);
  }
  ck(cudaGetLastError(), "smooth launch");
  int total = 0;
  ck(cudaMemcpyAsync(&total, d_off_ + nv_, sizeof(int), cudaMemcpyDeviceToHost, stream_), "download");
  ck(cudaStreamSynchronize(stream_), "smooth");
  nnz_ = total;
}

void Skin::get_binding(int* offsets, int* pills, double* weights, int* nnz, int* clamped) const {
  if (offsets) ck(cudaMemcpyAsync(offsets, d_off_, sizeof(int) * (nv_ + 1ull), cudaMemcpyDeviceToHost, stream_), "get");
  if (pills) ck(cudaMemcpyAsync(pills, d_pills_, sizeof(int) * nnz_, cudaMemcpyDeviceToHost, stream_), "get");
  if (weights) ck(cudaMemcpyAsync(weights, d_weights_, sizeof(double) * nnz_, cudaMemcpyDeviceToHost, stream_), "get");
  ck(cudaStreamSynchronize(stream_), "get binding");
  if (nnz) *nnz = static_cast<int>(nnz_);
  if (clamped) *clamped = clamped_;
}

void Skin::deform_device(const double* d_transforms, cudaStream_t st) {
  vdev::k_skin_frame<<<vdev::grid_of(8ll * np_, 256), 256, 0, st>>>(np_, d_rest_, d_transforms, d_frame_);
  vdev::k_skin_deform<<<vdev::grid_of(nv_, vdev::kDeformThreads), vdev::kDeformThreads, 0, st>>>(
      nv_, d_verts_, d_off_, d_pills_, d_weights_, d_rest_, d_frame_, d_out_);
}

void Skin::deform(int pill_count, const double* transforms, double* out) {
  require(pill_count == np_, "transform count changed since binding");
  ck(cudaMemcpyAsync(d_cur_, transforms, sizeof(double) * kTransformDoubles * np_, cudaMemcpyHostToDevice,
                     stream_),
     "upload");
  deform_device(d_cur_, stream_);
  ck(cudaGetLastError(), "deform launch");
  if (out) ck(cudaMemcpyAsync(out, d_out_, sizeof(double) * 3ull * nv_, cudaMemcpyDeviceToHost, stream_), "download");
  ck(cudaStreamSynchronize(stream_), "deform");
}

void Skin::deform_solver(Solver& solver, double* out) {
  require(solver.total_elements() == np_, "transform count changed since binding");
  cudaStream_t st = solver.stream();
  solver.pill_transforms_device(d_cur_);
  deform_device(d_cur_, st);
  ck(cudaGetLastError(), "deform launch");
  if (out) ck(cudaMemcpyAsync(out, d_out_, sizeof(double) * 3ull * nv_, cudaMemcpyDeviceToHost, st), "download");
  ck(cudaStreamSynchronize(st), "deform");
}

void Skin::bench(Solver& solver, int iterations, double* total_ms, double* deform_ms) {
  require(solver.total_elements() == np_, "transform count changed since binding");
  cudaStream_t st = solver.stream();
  cudaEvent_t e[4];
  for (auto& x : e) ck(cudaEventCreate(&x), "event");
  float t_all = 0.f, t_def = 0.f;
  ck(cudaEventRecord(e[0], st), "event");
  for (int i = 0; i < iterations; ++i) {
    solver.pill_transforms_device(d_cur_);
    if (i == iterations - 1) ck(cudaEventRecord(e[2], st), "event");
    deform_device(d_cur_, st);
    if (i == iterations - 1) ck(cudaEventRecord(e[3], st), "event");
  }
  ck(cudaEventRecord(e[1], st), "event");
  ck(cudaEventSynchronize(e[1]), "bench");
  ck(cudaGetLastError(), "bench launch");
  cudaEventElapsedTime(&t_all, e[0], e[1]);
  cudaEventElapsedTime(&t_def, e[2], e[3]);
  for (auto& x : e) cudaEventDestroy(x);
  if (total_ms) *total_ms = t_all;
  if (deform_ms) *deform_ms = t_def;
}

}  // namespace vhost
