// cost_model.hpp -- the additive synthetic cost model and its brute-force optimum.
//
// Deterministic stand-in for real timings: the parity oracle for the GA trajectory tests and the
// format cost-model calibration would emit.  Semantics follow
// /root/reference/proj/include/acctune/sim_model.hpp:14-61 and src/sim_model.cpp:22-98,157-236:
//   t(g) = s + sum_{bit 0} c_i + sum_{bit 1} (c_i / g_i + d_i) + sum_{i<j both set} J_ij
// evaluated serially, loops 0..a-1 then interactions in file order (the order is part of the
// result: it is a floating-point sum).
#pragma once

#include <cstddef>
#include <filesystem>
#include <string>
#include <unordered_set>
#include <vector>

#include "mmxhost/genome.hpp"

namespace mmxhost {

struct LoopCost {
  double compute_s = 0.0;   // c_i
  double speedup = 1.0;     // g_i >= 1
  double transfer_s = 0.0;  // d_i >= 0
};

struct Interaction {
  int i = 0, j = 0;  // i < j
  double value = 0.0;
};

struct CostModel {
  double serial_s = 0.0;
  std::vector<LoopCost> loops;
  std::vector<Interaction> interactions;
  std::unordered_set<Genome, Genome::Hash> fail_set;

  std::size_t gene_length() const { return loops.size(); }
  double baseline_s() const;  // s + sum c_i
};

// Throws ModelGenomeMismatch / SimulatedCompileError.
double model_time(const CostModel& model, const Genome& genome);

struct OracleResult {
  Genome genome;
  double time_s = 0.0;
};
// All 2^a genomes except the fail set; ties to the lexicographically smallest bit string;
// GeneLengthTooLarge above a = 20.
OracleResult exhaustive_best(const CostModel& model);

CostModel parse_model(const std::string& json_text);
CostModel load_model(const std::filesystem::path& path);

}  // namespace mmxhost
