// Where batch_forward_dynamics (the drop-in's c2 group call) spends its time:
// host packing, model upload, the solve with pageable buffers, unpacking.
// Build: g++ -O2 -std=c++20 -Iinclude tools/probes/dropin_probe.cpp -Lpaper_1609_06779_b200/lib -lpardyn -lpardyn_b200 -Wl,-rpath,$PWD/paper_1609_06779_b200/lib
#include <pardyn/bench.hpp>
#include <pardyn/pardyn.hpp>

#include <chrono>
#include <cstdio>

#include "../../include/pardyn_c.h"
#include "../../paper_1609_06779_b200/cpp/records.hpp"

using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }

int main() {
  const int n = 32, B = 65536;
  const auto cell = pardyn::workload_seed(42, n, B);
  auto t0 = clk::now();
  const auto chains = pardyn::workload_chains(cell, n, B);
  const auto in = pardyn::workload_inputs(cell, n, B, 0);
  std::vector<pardyn::FdProblem> probs(B);
  for (int m = 0; m < B; ++m) probs[m] = {chains[m], in.q[m], in.qdot[m], in.drive[m]};
  auto t1 = clk::now();
  std::printf("setup (generate + FdProblems) %.1f ms\n", ms(t0, t1));
  for (int rep = 0; rep < 3; ++rep) {
    auto a = clk::now();
    auto res = pardyn::batch_forward_dynamics(probs, pardyn::FdAlgo::abia);
    auto b = clk::now();
    std::printf("batch_forward_dynamics: %.1f ms (ok %d)\n", ms(a, b), (int)res[7].ok());
  }
  // phases
  pd_ctx* ctx = nullptr;
  pd_create(&ctx, 0);
  for (int rep = 0; rep < 2; ++rep) {
    auto a = clk::now();
    std::vector<double> links, grav, q, qd, tau;
    links.reserve((size_t)B * n * PD_LINK_FIELDS);
    for (const auto& p : probs) {
      pardyn::detail::append_records(p.chain, links);
      grav.insert(grav.end(), p.chain.gravity.begin(), p.chain.gravity.end());
      q.insert(q.end(), p.q.begin(), p.q.end());
      qd.insert(qd.end(), p.qdot.begin(), p.qdot.end());
      tau.insert(tau.end(), p.tau.begin(), p.tau.end());
    }
    auto b = clk::now();
    pd_set_models(ctx, B, n, links.data(), grav.data(), nullptr, nullptr);
    auto c = clk::now();
    std::vector<double> qdd((size_t)B * n);
    std::vector<int32_t> st(B), rd(B), ix(B);
    pd_forward_dynamics(ctx, PD_ABIA, B, q.data(), qd.data(), tau.data(), qdd.data(), st.data(), rd.data(), ix.data());
    auto d = clk::now();
    std::vector<pardyn::FdResult> out(B);
    for (int j = 0; j < B; ++j) out[j].qddot = pardyn::JointVector(qdd.begin() + (size_t)j * n, qdd.begin() + (size_t)(j + 1) * n);
    auto e = clk::now();
    std::printf("pack %.1f ms | pd_set_models %.1f ms | pd_forward_dynamics (pageable) %.1f ms | unpack %.1f ms\n",
                ms(a, b), ms(b, c), ms(c, d), ms(d, e));
  }
  pd_destroy(ctx);
  return 0;
}
