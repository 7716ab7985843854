// Seeded synthetic workloads of the reference benchmark, product side
// (SURVEY.md §8f row 3): the exact chains and joint inputs the reference's
// pardyn-bench feeds batch_forward_dynamics, generated on host threads.
//
//   mix, workload_seed          proj/core/src/bench.cpp:42-47, 350-355
//   workload_chains             bench.cpp:357-366 -> random_chain(n, mix(cell ^ (0xC0FFEE + g)))
//   random_chain                proj/core/src/model.cpp:157-185 (Rng :26-56)
//   workload_inputs             bench.cpp:368-383 (q, qdot, drive per member, U[-1,1])
//
// Draw order is the one GCC 13 gives the reference source (constructor and
// operator arguments evaluate right to left): com z,y,x; moments z,y,x; the
// home translation draws unit_vector() before its magnitude.
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "../../include/pardyn_c.h"

namespace {

uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

struct Draw {
  std::mt19937_64 e;
  explicit Draw(uint64_t s) : e(s) {}
  double u() { return static_cast<double>(e() >> 11) * 0x1.0p-53; }
  double u(double lo, double hi) { return lo + (hi - lo) * u(); }
  void unit(double out[3]) {
    const double z = u(-1.0, 1.0);
    const double phi = u(0.0, 2.0 * M_PI);
    const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
    out[0] = r * std::cos(phi);
    out[1] = r * std::sin(phi);
    out[2] = z;
  }
  // Shoemake quaternion -> rotation matrix (Eigen's toRotationMatrix formula)
  void rot(double R[9]) {
    const double u1 = u();
    const double a2 = u(0.0, 2.0 * M_PI);
    const double a3 = u(0.0, 2.0 * M_PI);
    const double s1 = std::sqrt(1.0 - u1), s2 = std::sqrt(u1);
    const double w = s2 * std::cos(a3), x = s1 * std::sin(a2), y = s1 * std::cos(a2), z = s2 * std::sin(a3);
    const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
    const double twx = tx * w, twy = ty * w, twz = tz * w;
    const double txx = tx * x, txy = ty * x, txz = tz * x;
    const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
    R[0] = 1 - (tyy + tzz); R[1] = txy - twz;       R[2] = txz + twy;
    R[3] = txy + twz;       R[4] = 1 - (txx + tzz); R[5] = tyz - twx;
    R[6] = txz - twy;       R[7] = tyz + twx;       R[8] = 1 - (txx + tyy);
  }
};

void random_chain_into(int n, uint64_t seed, double* out) {
  Draw d(seed);
  for (int i = 0; i < n; ++i) {
    double* f = out + static_cast<size_t>(i) * PD_LINK_FIELDS;
    f[0] = d.u(0.1, 10.0);
    const double cz = d.u(-0.3, 0.3), cy = d.u(-0.3, 0.3), cx = d.u(-0.3, 0.3);
    f[1] = cx;
    f[2] = cy;
    f[3] = cz;
    double A[9];
    d.rot(A);
    const double mz = d.u(0.1, 1.0), my = d.u(0.1, 1.0), mx = d.u(0.1, 1.0);
    const double m[3] = {mx, my, mz};
    double I[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += (A[3 * r + k] * m[k]) * A[3 * c + k];
        I[3 * r + c] = s;
      }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) f[4 + 3 * r + c] = 0.5 * (I[3 * r + c] + I[3 * c + r]);
    double s[3];
    d.unit(s);
    f[13] = s[0];
    f[14] = s[1];
    f[15] = s[2];
    f[16] = f[17] = f[18] = 0.0;
    d.rot(f + 19);
    double dir[3];
    d.unit(dir);
    const double mag = d.u(0.1, 1.0);
    for (int k = 0; k < 3; ++k) f[28 + k] = mag * dir[k];
  }
}

template <class F>
void parallel_for(int64_t count, F&& f) {
  unsigned hw = std::thread::hardware_concurrency();
  if (hw == 0) hw = 1;
  const int64_t nthreads = std::min<int64_t>(hw, std::max<int64_t>(1, count / 64));
  if (nthreads <= 1) {
    for (int64_t k = 0; k < count; ++k) f(k);
    return;
  }
  std::vector<std::thread> pool;
  for (int64_t t = 0; t < nthreads; ++t)
    pool.emplace_back([&, t] {
      for (int64_t k = t; k < count; k += nthreads) f(k);
    });
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

uint64_t pd_mix(uint64_t x) { return mix(x); }

uint64_t pd_workload_seed(uint64_t seed, int32_t n_links, int64_t n_groups) {
  uint64_t h = mix(seed);
  h = mix(h ^ static_cast<uint64_t>(n_links));
  return mix(h ^ (static_cast<uint64_t>(n_groups) << 20));
}

void pd_random_chain(int32_t n_links, uint64_t seed, double* links) { random_chain_into(n_links, seed, links); }

void pd_workload_chains(uint64_t cell_seed, int32_t n_links, int64_t g0, int64_t count, double* links) {
  parallel_for(count, [&](int64_t g) {
    random_chain_into(n_links, mix(cell_seed ^ (0xC0FFEEULL + static_cast<uint64_t>(g0 + g))),
                      links + static_cast<size_t>(g) * n_links * PD_LINK_FIELDS);
  });
}

void pd_workload_inputs(uint64_t cell_seed, int32_t n_links, int64_t n_groups, int64_t repeat, double* q,
                        double* qdot, double* drive) {
  std::mt19937_64 e(mix(cell_seed ^ (0x5EEDULL + static_cast<uint64_t>(repeat) * 0x9e3779b97f4a7c15ULL)));
  auto sym = [&] { return 2.0 * (static_cast<double>(e() >> 11) * 0x1.0p-53) - 1.0; };
  for (int64_t g = 0; g < n_groups; ++g) {
    for (int i = 0; i < n_links; ++i) q[g * n_links + i] = sym();
    for (int i = 0; i < n_links; ++i) qdot[g * n_links + i] = sym();
    for (int i = 0; i < n_links; ++i) drive[g * n_links + i] = sym();
  }
}

}  // extern "C"
