// Random-automaton batch runner, CSV format and power-law fit — same schema
// and semantics as the reference's experiment.hpp:25-279 (instance seeds,
// in-order row flushing, per-instance status markers, least-squares fit in
// log space).  Workers are host threads; each exact solve owns its own
// device context/stream, and workers are spread round-robin over the visible
// GPUs (`devices`), so one box's B200s run independent instances in parallel.
#pragma once

#include <iosfwd>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "engine.hpp"

namespace synchro {

inline constexpr const char* kCsvHeader = "n,k,seed,solver,threshold,status,time_s,peak_mem_bytes";

struct ExperimentRecord {
  u32 n = 0;
  u32 k = 0;
  u64 seed = 0;
  std::string solver;
  u64 threshold = 0;
  std::string status;
  double time_s = 0.0;
  u64 peak_mem_bytes = 0;
};

struct ExperimentSpec {
  std::vector<u32> ns;
  u32 k = 2;
  u32 samples = 100;
  u64 seed_base = 0;
  std::string solver = "exact";  // exact | oracle | eppstein | beam | adaptive
  std::optional<double> time_limit = 60.0;
  u64 memory = u64{4} << 30;
  u32 threads = 1;
  u64 beam_size = 0;
  bool deterministic = false;
  EngineTuning tuning{};
  int devices = 0;        // 0: all visible
  u32 shard_index = 0;    // multi-process sharding: this process runs rows i with
  u32 shard_count = 1;    //   i % shard_count == shard_index
};

u64 instance_seed(u64 seed_base, u32 n, u32 index);
void write_csv_header(std::ostream& out);
void write_csv_row(std::ostream& out, const ExperimentRecord& r);
ExperimentRecord run_instance(const ExperimentSpec& spec, u32 n, u32 index, int device);
void run_experiment(const ExperimentSpec& spec, std::ostream& csv, std::ostream* log = nullptr);
std::vector<ExperimentRecord> parse_csv(std::istream& in);

struct FitResult {
  double a = 0, c = 0, residual = 0;
};
FitResult fit_power_law(const std::vector<std::pair<double, double>>& n_mean);
FitResult fit_records(const std::vector<ExperimentRecord>& records);

// Power-set BFS ground truth (n <= 20), oracle.hpp:17-57 semantics.
inline constexpr u32 kOracleMaxStates = 20;
u64 power_set_bfs_oracle(const Automaton& aut, const Deadline& deadline = {});

}  // namespace synchro
