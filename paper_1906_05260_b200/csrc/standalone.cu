// Fine-grained C-ABI entry points on the GPU: pill_project, deepest_penetration, broad_phase,
// find_contacts (collision.h:64-95) over host pill arrays. They run the same device functions
// as the solver's collision stage, so bit-exactness against the oracle on identical pill
// arrays is tested directly (tests/test_gpu_parity.py: test_collision_primitives_bit_exact and the
// broad-phase / find_contacts cases).
#include <cstdlib>
#include <algorithm>
#include <stdexcept>
#include <vector>

#include "kernels.cuh"
#include "solver.h"
#include "standalone.h"

namespace vhost {

namespace {

struct Buf {
  std::vector<void*> ptrs;
  ~Buf() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T>
  T* get(std::size_t n) {
    void* p = nullptr;
    check_cuda(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)), "cudaMalloc");
    check_cuda(cudaMemset(p, 0, std::max<std::size_t>(n, 1) * sizeof(T)), "cudaMemset");
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  template <typename T>
  T* put(const T* src, std::size_t n) {
    T* d = get<T>(n);
    if (n) check_cuda(cudaMemcpy(d, src, n * sizeof(T), cudaMemcpyHostToDevice), "upload");
    return d;
  }
};

template <typename T>
void fetch(T* dst, const T* src, std::size_t n) {
  if (n && dst) check_cuda(cudaMemcpy(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost), "download");
}

int pow2(long long x) {
  int p = 64;
  while (p < x) p <<= 1;
  return p;
}

// Collide buffers for P pills (static attributes + geometry), `cap` candidates.
void make_collide(Buf& b, vdev::Collide& c, const vrod_pill* pills, int P, long long cap) {
  c.P = P;
  c.T = pow2(2ll * std::max(P, 1));
  c.cand_cap = cap;
  c.contact_cap = cap;
  std::vector<double> geo(8ull * std::max(P, 1));
  std::vector<int> rod(P), el(P), grp(P);
  std::vector<uint8_t> self(P);
  std::vector<uint32_t> id(P);
  for (int i = 0; i < P; ++i) {
    const vrod_pill& p = pills[i];
    for (int f = 0; f < 3; ++f) {  // AoS, 8 doubles per pill (pill.cuh load_pill)
      geo[8ll * i + f] = p.c0[f];
      geo[8ll * i + 3 + f] = p.c1[f];
    }
    geo[8ll * i + 6] = p.r0;
    geo[8ll * i + 7] = p.r1;
    rod[i] = p.rod;
    el[i] = p.element;
    grp[i] = p.group;
    self[i] = p.self_collide ? 1 : 0;
    id[i] = (static_cast<uint32_t>(p.rod + 1) << 16) | (static_cast<uint32_t>(p.element + 1) & 0xffffu);
  }
  c.pill = b.put(geo.data(), geo.size());
  c.pill_rod = b.put(rod.data(), rod.size());
  c.pill_el = b.put(el.data(), el.size());
  c.pill_group = b.put(grp.data(), grp.size());
  c.pill_self = b.put(self.data(), self.size());
  c.pill_id = b.put(id.data(), id.size());
  c.bsph = b.get<double>(4ull * std::max(P, 1));
  c.cellkey = b.get<long long>(3ull * std::max(P, 1));
  c.table = b.get<int>(c.T);
  c.cell_count = b.get<int>(c.T);
  c.cell_start = b.get<int>(c.T + 1);
  c.cell_cursor = b.get<int>(c.T);
  c.slot_key = b.get<longlong4>(c.T);
  c.cell_items = b.get<int>(P);
  // broad_phase lists every allowed pair (often far more than one CTA sorts well): multi-launch
  // ordering unless a test forces a path
  c.order_smem_cap = std::getenv("VROD_CT_ORDER_CAP") ? vdev::order_cap_for(P) : -1;
  c.cell_attr = b.get<int4>(std::max(P, 1));
  c.cell_sph = b.get<double>(4ull * std::max(P, 1));
  c.pill_cell = b.get<int>(P);
  c.rep_flag = b.get<int>(P + 1);
  c.rep_pos = b.get<int>(P + 1);
  c.cell_list = b.get<int>(P);
  c.cell_span = b.get<int2>(14ull * std::max(P, 1));
  c.raw_i = b.get<int>(cap);
  c.raw_j = b.get<int>(cap);
  c.raw_ab = b.get<double>(2 * cap);
  c.ct_cnt = b.get<int>(P + 1);
  c.ct_off = b.get<int>(P + 1);
  c.ct_cur = b.get<int>(P + 1);
  c.cand_i = b.get<int>(cap);
  c.cand_j = b.get<int>(cap);
  c.cand_flag = b.get<int>(cap + 1);
  c.cand_pos = b.get<int>(cap + 1);
  c.cand_ab = b.get<double>(3 * cap);
  c.ct_a = b.get<int>(cap);
  c.ct_b = b.get<int>(cap);
  c.ct_alpha = b.get<double>(cap);
  c.ct_beta = b.get<double>(cap);
  c.ct_dist = b.get<double>(cap);
  c.scalars = b.get<int>(vdev::kScalars);
  c.maxr_bits = b.get<unsigned long long>(1);
  c.scan_parts = static_cast<int>(vdev::scan_partials_needed(std::max<long long>({cap, c.T, static_cast<long long>(P)})));
  c.scan_tmp = b.get<int>(c.scan_parts);
}

}  // namespace

void gpu_pill_project(long long n, const double* x, const vrod_pill* pills, double* t, double* d, uint8_t* deg) {
  if (n <= 0) return;
  Buf b;
  double* dx = b.put(x, 3 * n);
  double* dp = b.put(reinterpret_cast<const double*>(pills), n * (sizeof(vrod_pill) / sizeof(double)));
  double* dt = b.get<double>(n);
  double* dd = b.get<double>(n);
  uint8_t* dg = b.get<uint8_t>(n);
  vdev::launch_pill_project(n, dx, dp, dt, dd, dg, nullptr);
  check_cuda(cudaDeviceSynchronize(), "pill_project");
  fetch(t, dt, n);
  fetch(d, dd, n);
  fetch(deg, dg, n);
}

void gpu_deepest(long long n, const vrod_pill* a, const vrod_pill* bb, int iters, const double* warm, double* alpha,
                 double* beta, double* dist) {
  if (n <= 0) return;
  Buf b;
  const std::size_t pd = sizeof(vrod_pill) / sizeof(double);
  double* da = b.put(reinterpret_cast<const double*>(a), n * pd);
  double* db = b.put(reinterpret_cast<const double*>(bb), n * pd);
  double* dw = warm ? b.put(warm, n) : nullptr;
  double* dal = b.get<double>(n);
  double* dbe = b.get<double>(n);
  double* dd = b.get<double>(n);
  vdev::launch_deepest(n, da, db, iters, dw, dal, dbe, dd, nullptr);
  check_cuda(cudaDeviceSynchronize(), "deepest_penetration");
  fetch(alpha, dal, n);
  fetch(beta, dbe, n);
  fetch(dist, dd, n);
}

long long gpu_broad_phase(long long n, const vrod_pill* pills, long long cap_out, int32_t* pairs) {
  if (n < 2) return 0;  // collision.cpp:187
  long long cap = std::max<long long>(1024, 64 * n);
  for (int attempt = 0; attempt < 2; ++attempt) {
    Buf b;
    vdev::Collide c;
    make_collide(b, c, pills, static_cast<int>(n), cap);
    unsigned long long* err = b.get<unsigned long long>(1);
    check_cuda(cudaMemset(err, 0xff, sizeof(unsigned long long)), "err");
    vdev::launch_broad_ordered(c, err, nullptr);
    check_cuda(cudaDeviceSynchronize(), "broad_phase");
    unsigned long long e = 0;
    fetch(&e, err, 1);
    if (e != vdev::kNoError) throw std::invalid_argument("broad_phase: non-finite pill");
    int total = 0;
    fetch(&total, c.scalars + vdev::SC_NCAND_RAW, 1);
    if (total > cap) {
      cap = total;
      continue;
    }
    const long long k = std::min<long long>(total, cap_out);
    if (k > 0 && pairs) {
      std::vector<int> ci(k), cj(k);
      fetch(ci.data(), c.ct_a, k);
      fetch(cj.data(), c.ct_b, k);
      for (long long q = 0; q < k; ++q) {
        pairs[2 * q] = ci[q];
        pairs[2 * q + 1] = cj[q];
      }
    }
    return total;
  }
  throw std::runtime_error("broad_phase: candidate capacity");
}

long long gpu_find_contacts(long long n, const vrod_pill* pills, long long npairs, const int32_t* pairs, int iters,
                            long long nwarm, const uint64_t* wkeys, const double* walpha, long long cap_out,
                            int32_t* pa, int32_t* pb, double* alpha, double* beta, double* dist) {
  if (npairs <= 0) return 0;
  Buf b;
  vdev::Collide c;
  make_collide(b, c, pills, static_cast<int>(n), npairs);
  std::vector<int> ci(npairs), cj(npairs);
  for (long long q = 0; q < npairs; ++q) {
    ci[q] = pairs[2 * q];
    cj[q] = pairs[2 * q + 1];
  }
  check_cuda(cudaMemcpy(c.cand_i, ci.data(), sizeof(int) * npairs, cudaMemcpyHostToDevice), "pairs");
  check_cuda(cudaMemcpy(c.cand_j, cj.data(), sizeof(int) * npairs, cudaMemcpyHostToDevice), "pairs");
  // warm map with emplace semantics (first inserted wins, collision.cpp:257-258) -> sorted unique
  std::vector<std::pair<uint64_t, double>> warm;
  if (wkeys) {
    std::vector<std::pair<uint64_t, long long>> order;
    for (long long k = 0; k < nwarm; ++k) order.emplace_back(wkeys[k], k);
    std::stable_sort(order.begin(), order.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    for (const auto& [key, k] : order)
      if (warm.empty() || warm.back().first != key) warm.emplace_back(key, walpha[k]);
  }
  std::vector<unsigned long long> keys;
  std::vector<double> al;
  for (const auto& [key, a] : warm) {
    keys.push_back(key);
    al.push_back(a);
  }
  c.warm_rr_key = b.put(keys.data(), keys.size());
  c.warm_rr_alpha = b.put(al.data(), al.size());
  int scal[vdev::kScalars] = {0};
  scal[vdev::SC_NCAND] = static_cast<int>(npairs);
  scal[vdev::SC_NRR_PREV] = static_cast<int>(keys.size());
  check_cuda(cudaMemcpy(c.scalars, scal, sizeof(scal), cudaMemcpyHostToDevice), "scalars");
  c.iters_dich = iters;
  vdev::launch_narrow_only(c, /*split_warm=*/0, /*store_d=*/1, nullptr);
  check_cuda(cudaDeviceSynchronize(), "find_contacts");
  int count = 0;
  fetch(&count, c.cand_pos + npairs, 1);
  const long long k = std::min<long long>(count, cap_out);
  fetch(pa, c.ct_a, k);
  fetch(pb, c.ct_b, k);
  fetch(alpha, c.ct_alpha, k);
  fetch(beta, c.ct_beta, k);
  fetch(dist, c.ct_dist, k);
  return count;
}

void gpu_extract_rotation(long long n, const double* B, const double* guess, int max_iterations, double tolerance,
                          double* out) {
  if (n <= 0) return;
  Buf b;
  const double* dB = b.put(B, 9ull * n);
  const double* dg = b.put(guess, 4ull * n);
  double* dq = b.get<double>(4ull * n);
  vdev::launch_extract_rotation(n, dB, dg, max_iterations, tolerance, dq, nullptr);
  check_cuda(cudaGetLastError(), "extract_rotation launch");
  fetch(out, dq, 4ull * n);
}

}  // namespace vhost
