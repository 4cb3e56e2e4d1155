// commands.hpp -- `tune`, `report`, `analyze` on top of the host layer: the callers of the hot path
// (/root/reference/proj/include/acctune/commands.hpp:14-32, src/commands.cpp:157-378).
//
// A finished workdir holds the reference's artifact set under the reference's names and formats:
//   config.resolved.json  provenance (config.cpp:154-183)
//   eval_cache.jsonl      one line per measured genome (evaluator.cpp:178-192); a rerun replays from it
//   generations.csv       %.9g table (ga.cpp:297-309)
//   summary.json          baseline_s, best_s, speedup, best_genome, distinct_evals, elapsed_s (commands.cpp:157-166)
//   best/<source>         the winning variant: the source with `#pragma acc kernels` above each selected loop
//   probe_report.jsonl    one verdict per loop (probe.cpp:162-185): "probe skipped" rows for sim runs, as in the
//                         reference; the static rules' verdicts (feasibility.hpp) for the cuda backend
// With the cuda backend the catalogue derived from the source (kernel_match.hpp) must be the one the kernel library
// serves (mmx_loop_catalogue).  `calibrate` (cuda backend only) adds
//   calibrated_model.json the reference's cost-model file fitted to measured times (calibrate.hpp)
//   calibration.json      fit and projection report, the measured and the modelled optimum
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
// Measures every feasible genome through the evaluator (memoised: a rerun replays eval_cache.jsonl), fits the plan
// model, projects it onto the reference's cost-model form and writes both files into the workdir.
int cmd_calibrate(const std::string& config_path, std::ostream& out, std::ostream& err);

}  // namespace mmxhost
