// evaluator.hpp -- the memoising, job-pooled front end of a backend.
//
// Behavioural contract = /root/reference/proj/src/evaluator.cpp:144-292 as pinned by
// tests/test_evaluator.cpp:103-262:
//   * each distinct genome reaches the backend once per run; concurrent duplicates wait for the
//     first caller; the mutex is NOT held while the backend measures;
//   * backend exceptions are remembered per genome and rethrown to every current and future caller;
//   * evaluate_all runs min(jobs, n) workers pulling the next index, outcomes aligned with input,
//     first exception rethrown after all workers joined;
//   * every new outcome is appended to a JSON-lines cache ({"genome","status","time_s",
//     "wall_cost_s"}, in that key order) that is reloaded -- with validation -- at construction;
//     genomes served from the file count as distinct but not as backend calls;
//   * counters().elapsed_s sums wall_cost_s over counted genomes in genome order.
#pragma once

#include <condition_variable>
#include <exception>
#include <filesystem>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "mmxhost/backend.hpp"

namespace mmxhost {

// What run_ga needs (/root/reference/proj/include/acctune/evaluation.hpp:39-56; ga.cpp:100-107,191-201,255,272).  evaluate_all returns outcomes aligned
// with its input.
class GenomeEvaluator {
 public:
  virtual ~GenomeEvaluator() = default;
  virtual EvaluationOutcome evaluate(const Genome& genome) = 0;
  virtual std::vector<EvaluationOutcome> evaluate_all(const std::vector<Genome>& genomes) {
    std::vector<EvaluationOutcome> out;
    out.reserve(genomes.size());
    for (const Genome& g : genomes) out.push_back(evaluate(g));
    return out;
  }
  virtual EvalCounters counters() const = 0;
};

class Evaluator : public GenomeEvaluator {
 public:
  explicit Evaluator(std::unique_ptr<EvalBackend> backend, int jobs = 1, std::filesystem::path cache_file = {});

  EvaluationOutcome evaluate(const Genome& genome) override;
  std::vector<EvaluationOutcome> evaluate_all(const std::vector<Genome>& genomes) override;
  EvalCounters counters() const override;

  std::size_t gene_length() const { return backend_->gene_length(); }
  EvalBackend& backend() { return *backend_; }

  // Scheduling hint for evaluate_all: genomes with a larger predicted cost are handed to the workers first (longest
  // processing time first), so that one slow individual -- a genome that leaves the matmul nest on the CPU takes
  // seconds, an all-offloaded one milliseconds -- does not start last and stretch the batch.  Outcomes stay aligned with
  // the input and nothing else changes; without a hint the batch is pulled in input order, as the reference does
  // (/root/reference/proj/src/evaluator.cpp:254-273).
  using CostHint = std::function<double(const Genome&)>;
  void set_cost_hint(CostHint hint) { cost_hint_ = std::move(hint); }

 protected:
  // Hook for subclasses that bind worker threads to resources (MultiGpuEvaluator): called by
  // worker `worker` of evaluate_all (0 for plain evaluate()).
  virtual EvaluationOutcome measure_with(int worker, const Genome& genome) {
    (void)worker;
    return backend_->measure(genome);
  }

 private:
  struct Slot {
    bool done = false;
    bool seen_this_run = false;
    EvaluationOutcome outcome;
    std::exception_ptr failure;
  };

  EvaluationOutcome evaluate_as(int worker, const Genome& genome);
  void load_cache();
  void append_to_cache(const Genome& genome, const EvaluationOutcome& outcome);

  std::unique_ptr<EvalBackend> backend_;
  CostHint cost_hint_;
  int jobs_;
  std::filesystem::path cache_file_;

  mutable std::mutex mu_;
  std::condition_variable done_cv_;
  std::map<Genome, Slot> memo_;
  std::uint64_t requests_ = 0, distinct_ = 0, cache_hits_ = 0, backend_calls_ = 0;
};

// Population-parallel evaluation over the device slots of one CudaBackend: worker thread s of a
// batch always measures on slot s (one stream / one set of device arrays / one GPU each), so
// `jobs` == number of slots and no two workers contend for a device.  Memoisation, cache file
// and counters are the Evaluator's.  Batches are scheduled longest-first by a static estimate from the
// residency plan (predicted_cost: host-side flops, launch counts, bytes over the bus).  No collective: each worker writes its outcome into the
// aligned output slot and the gather is the thread join.
class MultiGpuEvaluator : public Evaluator {
 public:
  explicit MultiGpuEvaluator(std::unique_ptr<CudaBackend> backend, std::filesystem::path cache_file = {});

 protected:
  EvaluationOutcome measure_with(int worker, const Genome& genome) override;

 public:
  // seconds, order-of-magnitude: only the ranking matters
  static double predicted_cost(const Genome& genome, const CudaBackendConfig& config);

 private:
  // the public constructor releases the backend FIRST and delegates here, so that exactly one owner exists while the base is built
  // (if the base constructor throws -- bad_alloc, an unreadable cache file -- its argument deletes the backend once)
  MultiGpuEvaluator(CudaBackend* adopted, std::filesystem::path cache_file);
  CudaBackend* cuda_;
};

}  // namespace mmxhost
