// commands.hpp -- `tune`, `report`, `analyze` on top of the host layer: the callers of the hot path
// (/root/reference/proj/include/acctune/commands.hpp:14-32, src/commands.cpp:157-378).
//
// A finished workdir holds the reference's artifact set under the reference's names and formats:
//   config.resolved.json  provenance (config.cpp:154-183)
//   eval_cache.jsonl      one line per measured genome (evaluator.cpp:178-192); a rerun replays from it
//   generations.csv       %.9g table (ga.cpp:297-309)
//   summary.json          baseline_s, best_s, speedup, best_genome, distinct_evals, elapsed_s (commands.cpp:157-166)
//   best/<source>         the winning variant: the source with `#pragma acc kernels` above each selected loop
// There is no compiler probe on this path, hence no probe_report / probe_cache: with the sim backend every
// scanned loop (after the filter) is a candidate, as in the reference; with the cuda backend the scanned
// catalogue must be the one the kernel library serves (mmx_loop_catalogue) and every loop is a candidate.
#pragma once

#include <cstdint>
#include <exception>
#include <iosfwd>
#include <optional>
#include <string>

namespace mmxhost {

// 0 success, 2 config error, 3 scan error / no candidates, 4 measuring tool unavailable (no CUDA device) or
// baseline unmeasurable, 5 zero-fitness abort, 1 anything else  (commands.cpp:170-181)
int exit_code_for(const std::exception& e);

struct TuneOptions {
  std::optional<std::uint64_t> seed;      // overrides ga.seed
  std::optional<std::string> sim_model;   // overrides the backend
};

int cmd_analyze(const std::string& config_path, std::ostream& out, std::ostream& err);
int cmd_tune(const std::string& config_path, const TuneOptions& options, std::ostream& out, std::ostream& err);
int cmd_report(const std::string& workdir, std::ostream& out, std::ostream& err);

}  // namespace mmxhost
