// feasibility.hpp -- which loops (and which genomes) an offload compiler would accept, decided statically.
//
// The reference learns this from the compiler: probe_loop renders the variant with the directive on exactly
// one loop, forks the OpenACC compiler and classifies its diagnostic (/root/reference/proj/src/probe.cpp:125-160,
// classifier rules :49-67); whole genomes are rejected at measure time with CompileError
// (src/evaluator.cpp:78-99).  A kernel-library backend has no compiler to ask, so the same verdicts are
// derived here from the token stream of the source.  The rules are the ones the reference's bundled compiler
// applies to each annotated loop, in its order (tools/mockacc.cpp:196-247):
//   1. NestedOverlap   the loop sits inside the body of another annotated loop
//                      ("compute regions may not be nested")
//   2. ExternalCall    the body calls a function ("call to 'f' with no acc routine information")
//   3. EarlyExit       the body contains break / return / goto ("branching out of compute region ('break')")
//   4. DataDependency  x[i] = ... x[i +- c] ... inside one statement
//                      ("loop carried dependence of 'x' prevents parallelization")
// `#pragma acc kernels` lines already present in the source count as annotations of the loop that follows
// them (mockacc.cpp:166-192), so a hand-annotated outer loop makes its inner loops NestedOverlap.
// Verdict, reject class and the diagnostic's wording match the reference's probe with mockacc on its own
// corpus (fixtures/corpus/*.c, fixtures/matmul.c) and on this repo's synthetic cases: tests/test_host_feasibility.py.
#pragma once

#include <string>
#include <string_view>
#include <vector>

#include "mmxhost/genome.hpp"
#include "mmxhost/source_model.hpp"

namespace mmxhost {

// probe.hpp:16
enum class RejectClass { ExternalCall, NestedOverlap, EarlyExit, DataDependency, Other };
std::string_view to_string(RejectClass c);  // "external_call", "nested_overlap", "early_exit", "data_dependency", "other"

enum class ProbeVerdict { Parallelizable, Rejected };

// probe.hpp:36-42
struct ProbeResult {
  int loop_id = 0;
  ProbeVerdict verdict = ProbeVerdict::Rejected;
  RejectClass reject_class = RejectClass::Other;  // meaningful iff Rejected
  std::string compiler_message;                   // the diagnostic, "<what> (<path>: line <L>)"; empty when accepted
  bool timed_out = false;                         // always false: nothing is executed
};

// Everything the rules need, computed once per source.
class FeasibilityAnalyzer {
 public:
  FeasibilityAnalyzer(const SourceUnit& unit, const std::vector<LoopSite>& loops);
  ~FeasibilityAnalyzer();
  FeasibilityAnalyzer(const FeasibilityAnalyzer&) = delete;
  FeasibilityAnalyzer& operator=(const FeasibilityAnalyzer&) = delete;

  // probe_loop (probe.cpp:125): the directive on exactly this loop (plus the ones the source already carries)
  ProbeResult probe(int loop_id) const;

  // a whole variant: one ProbeResult per REJECTED annotated loop, in document order (empty = compiles).
  // `annotated` are loop ids; the source's own directives are added.
  std::vector<ProbeResult> check(const std::vector<int>& annotated) const;

  // loops the source itself annotates (document order, no duplicates)
  const std::vector<int>& preannotated() const;

 private:
  struct Impl;
  Impl* impl_;
};

// probe_loop without keeping the analyzer
ProbeResult probe_loop(const SourceUnit& unit, const std::vector<LoopSite>& loops, int loop_id);

// build_candidate_set (probe.cpp:187-294): probe every loop, keep the accepted ones in document order.
// `report_out` receives one ProbeResult per loop even when NoCandidates is thrown.
CandidateSet build_candidate_set(const SourceUnit& unit, const std::vector<LoopSite>& loops,
                                 std::vector<ProbeResult>* report_out = nullptr);

// Would the variant of `genome` compile?  (The CompileError branch of ToolchainBackend::measure.)
bool variant_feasible(const CandidateSet& cs, const Genome& genome, std::vector<ProbeResult>* rejected_out = nullptr);

// One JSON object per loop, one per line: {"id","line","verdict","reject_class","message","timed_out"}
// (write_probe_report, probe.cpp:162-185).
std::string probe_report_jsonl(const SourceUnit& unit, const std::vector<LoopSite>& loops, const std::vector<ProbeResult>& results);

}  // namespace mmxhost
