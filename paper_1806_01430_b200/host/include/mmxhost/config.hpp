// config.hpp -- one declarative JSON file per run, as in the reference
// (/root/reference/proj/include/acctune/config.hpp:19-44, src/config.cpp:103-185), with one new backend block.
//
// Same keys, same validation, same resolved-provenance blob: "source", "workdir", "candidates", "jobs", "ga",
// and exactly one backend.  The reference's backends are "toolchain" (external OpenACC compiler + benchmark
// binary) and "sim_model"; this build replaces the former with
//   "cuda": { "n": 256, "dtype": "f64"|"f32", "numerics": "fast"|"strict", "timeout_s": 120, "repetitions": 1,
//             "warmup": 0, "host_threads": 1, "devices": [0, 1, ...], "matmul_variant": 0 }
// -- the in-process CUDA executor behind include/mmx.h (timeout_s / repetitions keep the meaning they have in the
// reference's ToolchainConfig).  A "toolchain" block is rejected with a ConfigError that says so: there is no
// external compiler on this path.  Unknown keys are rejected so typos cannot fall back to defaults.
#pragma once

#include <optional>
#include <string>

#include "mmxhost/backend.hpp"
#include "mmxhost/ga.hpp"

namespace mmxhost {

enum class CandidateFilter { All, Outermost };
std::string_view to_string(CandidateFilter f);

struct RunConfig {
  std::string source;   // absolute, normalised
  std::string workdir;  // absolute, normalised
  CandidateFilter candidates = CandidateFilter::All;
  int jobs = 1;
  GAParams ga;
  std::optional<std::string> sim_model;
  std::optional<CudaBackendConfig> cuda;

  std::string resolved_config_path() const { return workdir + "/config.resolved.json"; }
  std::string probe_report_path() const { return workdir + "/probe_report.jsonl"; }
  std::string probe_cache_path() const { return workdir + "/probe_cache.jsonl"; }
  std::string eval_cache_path() const { return workdir + "/eval_cache.jsonl"; }
  std::string generations_csv_path() const { return workdir + "/generations.csv"; }
  std::string summary_path() const { return workdir + "/summary.json"; }
  std::string best_source_path() const;
};

// Relative paths resolve against the directory holding the file.  Throws ConfigError.
RunConfig load_config(const std::string& config_path);

// Provenance blob written into the workdir before any evaluation starts; for a sim_model run it is byte-identical
// to the reference's render_resolved_config.
std::string render_resolved_config(const RunConfig& cfg);

}  // namespace mmxhost
