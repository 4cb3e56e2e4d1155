// drive_reference.cpp -- TEST INFRASTRUCTURE: the UNMODIFIED reference tuner driving libmmx.so.
//
// Links the reference's own Evaluator / run_ga (libacctune_core.a, compiled from /root/reference/proj/src by
// oracle/Makefile) with acctune::CudaBackend (cuda_backend.hpp, the binding INTEGRATION.md section 2 lists) and runs the
// scenarios of tests/test_ref_dropin.py.  Nothing of this repo's host mirror (namespace mmxhost) is involved: the only
// product code behind the reference's EvalBackend::measure (include/acctune/evaluator.hpp:19-24) is the C ABI.
//
//   drive_reference <matmul.c> <workdir> <n> <population> <generations> <seed> <jobs>
// prints one JSON object on stdout.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>

#include "acctune/evaluator.hpp"
#include "acctune/ga.hpp"
#include "acctune/source_model.hpp"
#include "cuda_backend.hpp"

using namespace acctune;

namespace {

// counts calls and the highest number of measure() calls in flight (the reference tests' ScriptBackend idea,
// tests/test_util.hpp:55-81), forwarding to the real backend
class Observed : public EvalBackend {
 public:
  struct Counters {
    std::atomic<int> calls{0}, in_flight{0}, max_in_flight{0};
  };
  Observed(std::unique_ptr<EvalBackend> inner, Counters* c) : inner_(std::move(inner)), c_(c) {}
  EvaluationOutcome measure(const Genome& g) override {
    c_->calls.fetch_add(1);
    const int now = c_->in_flight.fetch_add(1) + 1;
    int seen = c_->max_in_flight.load();
    while (now > seen && !c_->max_in_flight.compare_exchange_weak(seen, now)) {
    }
    struct Leave {
      std::atomic<int>& n;
      ~Leave() { n.fetch_sub(1); }
    } leave{c_->in_flight};
    return inner_->measure(g);
  }
  std::size_t gene_length() const override { return inner_->gene_length(); }

 private:
  std::unique_ptr<EvalBackend> inner_;
  Counters* c_;
};

std::string quoted(const std::string& s) {
  std::string out = "\"";
  for (char ch : s) {
    if (ch == '"' || ch == '\\') out += '\\';
    if (ch == '\n') out += "\\n";
    else out += ch;
  }
  return out + "\"";
}

std::string counters_json(const EvalCounters& c) {
  std::ostringstream o;
  o << "{\"requests\":" << c.requests << ",\"distinct\":" << c.distinct << ",\"cache_hits\":" << c.cache_hits
    << ",\"backend_calls\":" << c.backend_calls << "}";
  return o.str();
}

std::string run_json(const TuningResult& r, const EvalCounters& c, const Observed::Counters& oc) {
  std::ostringstream csv;
  write_generation_csv(csv, r);
  std::ostringstream o;
  o.precision(17);
  o << "{\"best_genome\":" << quoted(r.best_genome.to_string()) << ",\"best_s\":" << r.best_time_s << ",\"baseline_s\":" << r.baseline_s
    << ",\"generations_csv\":" << quoted(csv.str()) << ",\"counters\":" << counters_json(c) << ",\"measure_calls\":" << oc.calls.load()
    << ",\"max_in_flight\":" << oc.max_in_flight.load() << ",\"best_source_has_pragma\":"
    << (r.best_source.find(std::string(kOffloadDirective)) != std::string::npos ? "true" : "false") << "}";
  return o.str();
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 8) {
    std::fprintf(stderr, "usage: %s <source> <workdir> <n> <population> <generations> <seed> <jobs>\n", argv[0]);
    return 2;
  }
  try {
    const std::filesystem::path work = argv[2];
    std::filesystem::create_directories(work);
    CandidateSet cs;  // every scanned loop is a candidate (cmd_tune's sim branch, commands.cpp:93-106)
    cs.unit = SourceUnit::from_file(argv[1]);
    cs.all_loops = scan_loops(cs.unit);
    for (const auto& l : cs.all_loops) cs.candidate_ids.push_back(l.id);

    CudaConfig cfg;
    cfg.n = std::atoi(argv[3]);
    cfg.timeout_s = 5.0;
    const int jobs = std::atoi(argv[7]);
    cfg.devices.assign(static_cast<std::size_t>(jobs), 0);  // `jobs` slots on device 0
    GAParams params;
    params.population = std::atoi(argv[4]);
    params.generations = std::atoi(argv[5]);
    params.seed = std::strtoull(argv[6], nullptr, 10);

    std::cout << "{\"gene_length\":" << cs.gene_length();

    // (1) a cold run: the reference's Evaluator + run_ga over the CUDA backend
    Observed::Counters oc1;
    {
      Evaluator ev(std::make_unique<Observed>(std::make_unique<CudaBackend>(cfg), &oc1), jobs, work / "eval_cache.jsonl");
      const TuningResult r = run_ga(cs, params, ev);
      std::cout << ",\"cold\":" << run_json(r, ev.counters(), oc1);
    }
    // (2) the same run resumed from eval_cache.jsonl: no backend call (evaluator.cpp:150-176, test_cli.cpp:371-394)
    Observed::Counters oc2;
    {
      Evaluator ev(std::make_unique<Observed>(std::make_unique<CudaBackend>(cfg), &oc2), jobs, work / "eval_cache.jsonl");
      const TuningResult r = run_ga(cs, params, ev);
      std::cout << ",\"warm\":" << run_json(r, ev.counters(), oc2);
    }
    // (3) error conventions at the boundary: a genome of the wrong length is GenomeLengthMismatch, from the backend
    // itself (MMX_E_LENGTH) and from the Evaluator in front of it (evaluator.cpp:220-224)
    {
      CudaBackend bare(cfg);
      std::string backend_throws = "nothing", evaluator_throws = "nothing";
      try {
        bare.measure(Genome::zeros(cs.gene_length() - 1));
      } catch (const GenomeLengthMismatch&) {
        backend_throws = "GenomeLengthMismatch";
      } catch (const Error&) {
        backend_throws = "Error";
      }
      Observed::Counters oc3;
      Evaluator ev(std::make_unique<Observed>(std::make_unique<CudaBackend>(cfg), &oc3), 1);
      try {
        ev.evaluate(Genome::zeros(cs.gene_length() + 1));
      } catch (const GenomeLengthMismatch&) {
        evaluator_throws = "GenomeLengthMismatch";
      } catch (const Error&) {
        evaluator_throws = "Error";
      }
      // infeasible genome: an outcome, not an exception
      const EvaluationOutcome bad = ev.evaluate(Genome::from_string("110000000000"));
      const EvaluationOutcome good = ev.evaluate(Genome::from_string("101010101001"));
      std::cout << ",\"errors\":{\"backend_wrong_length\":" << quoted(backend_throws) << ",\"evaluator_wrong_length\":" << quoted(evaluator_throws)
                << ",\"infeasible_status\":" << quoted(std::string(to_string(bad.status))) << ",\"infeasible_time_s\":" << bad.time_s
                << ",\"all_nests_status\":" << quoted(std::string(to_string(good.status))) << ",\"all_nests_time_s\":" << good.time_s << "}";
    }
    // (4) no device slot at all is a configuration error, not a crash
    {
      std::string what = "nothing";
      try {
        CudaConfig none = cfg;
        none.devices.clear();
        CudaBackend b(none);
      } catch (const ConfigError&) {
        what = "ConfigError";
      } catch (const Error&) {
        what = "Error";
      }
      std::cout << ",\"no_slots\":" << quoted(what);
    }
    std::cout << "}" << std::endl;
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "drive_reference: %s\n", e.what());
    return 1;
  }
}
