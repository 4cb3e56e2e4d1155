// errors.hpp -- failure domains of the host layer.
//
// Same names and the same inheritance shape as the reference's acctune::Error family
// (/root/reference/proj/include/acctune/errors.hpp:10-90), because callers map failure domains
// to exit codes by type (commands.cpp:170-181): genome-level problems are outcomes,
// infrastructure problems are exceptions.
#pragma once

#include <stdexcept>
#include <string>

namespace mmxhost {

#define MMXHOST_ERROR(Name, Base)                                  \
  struct Name : Base {                                              \
    explicit Name(const std::string& what) : Base(what) {}         \
  }

struct Error : std::runtime_error {
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};

MMXHOST_ERROR(ConfigError, Error);            // bad or contradictory configuration
MMXHOST_ERROR(GenomeLengthMismatch, Error);   // genome length != candidate count
MMXHOST_ERROR(NoCandidates, Error);           // nothing to tune
MMXHOST_ERROR(ToolchainMissing, Error);       // the measuring tool itself is absent (here: no CUDA device)
MMXHOST_ERROR(NonPositiveTime, Error);        // fitness of t <= 0
MMXHOST_ERROR(WorkdirUnwritable, Error);      // cache file / workspace cannot be written
MMXHOST_ERROR(ZeroTotalFitness, Error);       // roulette wheel is empty
MMXHOST_ERROR(EvaluatorUnavailable, Error);   // baseline cannot be measured
MMXHOST_ERROR(ModelError, Error);             // synthetic cost model problems
MMXHOST_ERROR(ModelGenomeMismatch, ModelError);
MMXHOST_ERROR(GeneLengthTooLarge, ModelError);
MMXHOST_ERROR(SimulatedCompileError, ModelError);

MMXHOST_ERROR(ScanError, Error);              // the source file cannot be tokenised / parsed
MMXHOST_ERROR(MissingLog, Error);             // report: an artifact of a run is absent

#undef MMXHOST_ERROR

}  // namespace mmxhost
