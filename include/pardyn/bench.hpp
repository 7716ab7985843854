// pardyn benchmark harness of the drop-in API, the
// reference's proj/core/include/pardyn/bench.hpp surface with every timed
// solve on the GPU through include/pardyn/pardyn.hpp:
//
//   BenchMode / BenchAlgo / to_string / bench_algo_from_string   bench.hpp:19-28
//   BenchConfig / validate                                       bench.hpp:30-45
//   BenchRecord / BenchCellFailure / BenchReport                 bench.hpp:47-70
//   run_benchmark (3 warm-ups, `repeats` timed calls, spot checks every 100)
//                                                                bench.hpp:72-77, bench.cpp:150-420
//   emit_csv / parse_csv (header algo,n_links,n_groups,repeats,worker_count,mean_us,stddev_us)
//                                                                bench.hpp:79-84, bench.cpp:433-498
//   workload_seed / workload_chains / workload_inputs            bench.hpp:86-105
//
// worker_count records the host threads the reference's OpenMP would use;
// here it is the number of GPUs a cell ran on (1) unless --workers is given.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "pardyn.hpp"

namespace pardyn {

enum class BenchMode { link_sweep, group_sweep };
enum class BenchAlgo { jsiia, abia, cfa, invdyn };

std::string to_string(BenchAlgo algo);
BenchAlgo bench_algo_from_string(const std::string& name);

struct BenchConfig {
  BenchMode mode = BenchMode::link_sweep;
  std::vector<BenchAlgo> algos = {BenchAlgo::jsiia, BenchAlgo::abia, BenchAlgo::cfa};
  std::vector<int> link_counts = {10, 50, 100, 200};
  std::vector<int> group_counts = {1, 10, 100, 1000};
  int repeats = 1000;
  std::uint64_t seed = 42;
  int worker_count = 0;
  bool spot_check = true;
  std::string output_path = "results.csv";
};

void validate(const BenchConfig& config);

struct BenchRecord {
  BenchAlgo algo = BenchAlgo::jsiia;
  int n_links = 0;
  int n_groups = 1;
  int repeats = 0;
  int worker_count = 0;
  double mean_us = 0.0;
  double stddev_us = 0.0;
};

struct BenchCellFailure {
  BenchAlgo algo = BenchAlgo::jsiia;
  int n_links = 0;
  int n_groups = 1;
  std::string message;
};

struct BenchReport {
  std::vector<BenchRecord> records;
  std::vector<BenchCellFailure> failures;
  bool all_ok() const { return failures.empty(); }
};

BenchReport run_benchmark(const BenchConfig& config);
void emit_csv(const std::vector<BenchRecord>& records, const std::string& path);
std::vector<BenchRecord> parse_csv(const std::string& path);

std::uint64_t workload_seed(std::uint64_t seed, int n_links, int n_groups);
std::vector<RobotChain> workload_chains(std::uint64_t cell_seed, int n_links, int n_groups);

struct WorkloadInputs {
  std::vector<JointVector> q;
  std::vector<JointVector> qdot;
  std::vector<JointVector> drive;
};
WorkloadInputs workload_inputs(std::uint64_t cell_seed, int n_links, int n_groups, int repeat);

}  // namespace pardyn
