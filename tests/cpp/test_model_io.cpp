// Host-only checks of the drop-in's model files, validation and benchmark
// CSV (no GPU needed): the reference's tests/test_model.cpp and
// tests/test_bench.cpp cases for load_chain / save_chain / validate_chain /
// emit_csv / parse_csv / bench_algo_from_string / validate(BenchConfig).
// Prints one PASS/FAIL line per case; exit status = number of failures.
#include <pardyn/bench.hpp>
#include <pardyn/pardyn.hpp>
#include <pardyn_c.h>

#include <cstdio>
#include <fstream>
#include <functional>
#include <string>

namespace {

int failures = 0;
void check(bool ok, const std::string& what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

template <class E>
std::string what_of(const std::function<void()>& f) {
  try {
    f();
  } catch (const E& e) {
    return e.what();
  } catch (const std::exception& e) {
    return std::string("WRONG TYPE: ") + e.what();
  }
  return "NO THROW";
}

bool same(const pardyn::RobotChain& a, const pardyn::RobotChain& b) { return a == b; }

void write(const std::string& path, const std::string& text) { std::ofstream(path) << text; }

}  // namespace

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  using pardyn::ModelError;
  // save / load round trip is exact (model.hpp:79-80)
  {
    const pardyn::RobotChain c = pardyn::random_chain(7, 1234);
    pardyn::save_chain(c, dir + "/m7.json");
    check(same(pardyn::load_chain(dir + "/m7.json"), c), "save_chain / load_chain round trip is bit exact");
    pardyn::RobotChain g = c;
    g.gravity = pardyn::Vec3(0.1, -0.2, 1e-300);
    pardyn::save_chain(g, dir + "/g.json");
    check(same(pardyn::load_chain(dir + "/g.json"), g), "round trip of extreme doubles");
  }
  // validate_chain messages (model.cpp:75-115)
  {
    const pardyn::RobotChain good = pardyn::random_chain(3, 5);
    auto bad = [&](std::function<void(pardyn::RobotChain&)> edit) {
      pardyn::RobotChain c = good;
      edit(c);
      return what_of<ModelError>([&] { pardyn::validate_chain(c); });
    };
    check(what_of<ModelError>([&] { pardyn::validate_chain(good); }) == "NO THROW", "valid chain passes");
    check(what_of<ModelError>([&] { pardyn::validate_chain(pardyn::RobotChain{}); }) ==
              "chain must have at least one link",
          "empty chain");
    check(bad([](auto& c) { c.gravity[1] = 1.0 / 0.0; }) == "gravity must be finite", "gravity finite");
    check(bad([](auto& c) { c.links[1].mass = 0.0; }) == "link 1: mass must be positive", "mass positive");
    check(bad([](auto& c) { c.links[2].com[0] = 0.0 / 0.0; }) == "link 2: com must be finite", "com finite");
    check(bad([](auto& c) { c.links[0].inertia_rot(0, 1) += 1e-3; }) == "link 0: rotational inertia must be symmetric",
          "inertia symmetric");
    check(bad([](auto& c) { c.links[0].inertia_rot = pardyn::Mat3::FromRowMajor({1, 0, 0, 0, 1, 0, 0, 0, -1}); }) ==
              "link 0: rotational inertia must be positive definite",
          "inertia positive definite");
    check(bad([](auto& c) { c.links[1].joint_screw = pardyn::Twist(pardyn::Vec3(0, 0, 2), pardyn::Vec3()); }) ==
              "link 1: joint_screw must have unit norm (got 2.000000)",
          "screw unit norm");
    check(bad([](auto& c) { c.links[2].home_transform.rotation(0, 0) = 2.0; }) ==
              "link 2: home_transform rotation must be orthonormal with determinant +1",
          "home rotation orthonormal");
  }
  // load_chain errors (model.cpp:254-310)
  {
    const std::string p = dir + "/bad.json";
    write(p, "{\"n\": 1.5, \"gravity\": [0,0,-9.81], \"links\": []}");
    check(what_of<ModelError>([&] { pardyn::load_chain(p); }) == "model file '" + p + "': field 'n' must be an integer",
          "n must be an integer");
    write(p, "{\"n\": 2, \"gravity\": [0,0,-9.81], \"links\": []}");
    check(what_of<ModelError>([&] { pardyn::load_chain(p); }) ==
              "model file '" + p + "': field 'n' (= 2) does not match the length of 'links' (= 0)",
          "n vs links length");
    write(p, "{\"n\": 1, \"gravity\": [0,-9.81], \"links\": [{}]}");
    check(what_of<ModelError>([&] { pardyn::load_chain(p); }) ==
              "model file '" + p + "': field 'gravity' must be an array of 3 numbers",
          "gravity array length");
    write(p, "{\"n\": 1, \"gravity\": [0,0,-9.81], \"links\": [{\"com\": [0,0,0]}]}");
    check(what_of<ModelError>([&] { pardyn::load_chain(p); }) == "link 0: missing field 'mass'", "missing mass");
    write(p, "{\"n\": 1, \"gravity\": [0,0,-9.81], \"links\": [{\"mass\": \"x\"}]}");
    check(what_of<ModelError>([&] { pardyn::load_chain(p); }) == "link 0: field 'mass' must be a number",
          "mass must be a number");
    write(p, "{\"n\": 1,");
    check(what_of<ModelError>([&] { pardyn::load_chain(p); }).rfind("model file '" + p + "': parse error", 0) == 0,
          "malformed JSON");
    check(what_of<ModelError>([&] { pardyn::load_chain(dir + "/missing.json"); }) ==
              "cannot open model file '" + dir + "/missing.json'",
          "missing file");
  }
  // benchmark CSV and config (bench.cpp:303-340, 433-498)
  {
    std::vector<pardyn::BenchRecord> rec = {{pardyn::BenchAlgo::abia, 32, 65536, 10, 1, 123.456789012345678, 0.1},
                                            {pardyn::BenchAlgo::invdyn, 8, 1, 1000, 1, 1.0 / 3.0, 0.0}};
    pardyn::emit_csv(rec, dir + "/r.csv");
    const auto back = pardyn::parse_csv(dir + "/r.csv");
    bool ok = back.size() == 2;
    for (std::size_t k = 0; ok && k < 2; ++k)
      ok = back[k].algo == rec[k].algo && back[k].n_links == rec[k].n_links && back[k].n_groups == rec[k].n_groups &&
           back[k].mean_us == rec[k].mean_us && back[k].stddev_us == rec[k].stddev_us;
    check(ok, "emit_csv / parse_csv round trip is exact");
    std::ifstream f(dir + "/r.csv");
    std::string header;
    std::getline(f, header);
    check(header == "algo,n_links,n_groups,repeats,worker_count,mean_us,stddev_us", "CSV header");
    write(dir + "/bad.csv", "algo,n_links\n");
    check(what_of<std::runtime_error>([&] { pardyn::parse_csv(dir + "/bad.csv"); }) ==
              "benchmark csv '" + dir + "/bad.csv' line 1: unexpected header 'algo,n_links'",
          "CSV header check");
    check(what_of<std::invalid_argument>([] { pardyn::bench_algo_from_string("rnea"); }) ==
              "unknown benchmark algorithm 'rnea' (expected jsiia, abia, cfa or invdyn)",
          "algorithm names");
    pardyn::BenchConfig cfg;
    cfg.repeats = 0;
    check(what_of<std::invalid_argument>([&] { pardyn::validate(cfg); }) ==
              "benchmark config: repeats must be at least 1",
          "config validation");
    check(pardyn::workload_seed(42, 32, 65536) == pd_workload_seed(42, 32, 65536) &&
              pardyn::workload_inputs(pardyn::workload_seed(42, 4, 2), 4, 2, 0).q.size() == 2,
          "workload helpers");
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
