#include "mmxhost/evaluator.hpp"

#include <algorithm>
#include <atomic>
#include <fstream>
#include <string>
#include <thread>

#include "mmxhost/errors.hpp"
#include "mmxhost/json_lite.hpp"

namespace mmxhost {

Evaluator::Evaluator(std::unique_ptr<EvalBackend> backend, int jobs, std::filesystem::path cache_file)
    : backend_(std::move(backend)), jobs_(jobs < 1 ? 1 : jobs), cache_file_(std::move(cache_file)) {
  if (!cache_file_.empty()) load_cache();
}

// Lines that do not parse, name an unknown status, have the wrong gene length or claim a
// measured time that is not positive are skipped silently (evaluator.cpp:150-176;
// test_evaluator.cpp:243-262).
void Evaluator::load_cache() {
  std::ifstream in(cache_file_, std::ios::binary);
  if (!in) return;
  for (std::string line; std::getline(in, line);) {
    if (line.empty()) continue;
    json::Value row;
    if (!json::parse(line, row) || !row.is_object()) continue;
    const json::Value* g = row.find("genome");
    if (g == nullptr || !g->is_string()) continue;
    Genome genome;
    try {
      genome = Genome::from_string(g->string);
    } catch (const Error&) {
      continue;
    }
    if (genome.size() != backend_->gene_length()) continue;
    const json::Value* st = row.find("status");
    // a non-string status is a type error in the reference's value<std::string>() -- treat the
    // line as unusable rather than aborting the load
    if (st != nullptr && !st->is_string()) continue;
    const auto status = eval_status_from_string(st ? std::string_view(st->string) : std::string_view());
    if (!status) continue;
    Slot slot;
    slot.done = true;
    slot.outcome.status = *status;
    const json::Value* t = row.find("time_s");
    const json::Value* w = row.find("wall_cost_s");
    if ((t != nullptr && !t->is_number()) || (w != nullptr && !w->is_number())) continue;
    slot.outcome.time_s = t ? t->number : 0.0;
    slot.outcome.wall_cost_s = w ? w->number : 0.0;
    if (slot.outcome.status == EvalStatus::Measured && !(slot.outcome.time_s > 0.0)) continue;
    memo_.emplace(std::move(genome), std::move(slot));  // first line for a genome wins
  }
}

void Evaluator::append_to_cache(const Genome& genome, const EvaluationOutcome& outcome) {
  if (cache_file_.empty()) return;
  if (cache_file_.has_parent_path()) {
    std::error_code ec;
    std::filesystem::create_directories(cache_file_.parent_path(), ec);
  }
  std::ofstream out(cache_file_, std::ios::binary | std::ios::app);
  if (!out) throw WorkdirUnwritable("cannot append to cache file " + cache_file_.string());
  out << "{\"genome\":" << json::dump_string(genome.to_string()) << ",\"status\":" << json::dump_string(to_string(outcome.status))
      << ",\"time_s\":" << json::dump_number(outcome.time_s) << ",\"wall_cost_s\":" << json::dump_number(outcome.wall_cost_s)
      << "}\n";
}

EvaluationOutcome Evaluator::evaluate(const Genome& genome) { return evaluate_as(0, genome); }

EvaluationOutcome Evaluator::evaluate_as(int worker, const Genome& genome) {
  if (genome.size() != backend_->gene_length())
    throw GenomeLengthMismatch("evaluate: genome length " + std::to_string(genome.size()) +
                               " does not match candidate count " + std::to_string(backend_->gene_length()));
  std::unique_lock<std::mutex> lock(mu_);
  ++requests_;
  const auto [it, fresh] = memo_.try_emplace(genome);
  Slot& slot = it->second;  // std::map nodes are address-stable
  if (fresh) {
    // first request for this genome ever: this thread measures, with the lock released
    slot.seen_this_run = true;
    ++distinct_;
    ++backend_calls_;
    lock.unlock();
    EvaluationOutcome outcome;
    std::exception_ptr failure;
    try {
      outcome = measure_with(worker, genome);
    } catch (...) {
      failure = std::current_exception();
    }
    lock.lock();
    if (failure) {
      slot.failure = failure;
      slot.done = true;
      done_cv_.notify_all();
      std::rethrow_exception(failure);
    }
    slot.outcome = outcome;
    slot.done = true;
    append_to_cache(genome, outcome);
    done_cv_.notify_all();
    return outcome;
  }
  if (slot.seen_this_run) {
    ++cache_hits_;
  } else {
    slot.seen_this_run = true;  // loaded from the cache file, first encounter this run
    ++distinct_;
  }
  done_cv_.wait(lock, [&slot] { return slot.done; });
  if (slot.failure) std::rethrow_exception(slot.failure);
  return slot.outcome;
}

std::vector<EvaluationOutcome> Evaluator::evaluate_all(const std::vector<Genome>& genomes) {
  std::vector<EvaluationOutcome> results(genomes.size());
  if (genomes.empty()) return results;
  const std::size_t workers = std::min<std::size_t>(static_cast<std::size_t>(jobs_), genomes.size());
  if (workers <= 1) {
    for (std::size_t i = 0; i < genomes.size(); ++i) results[i] = evaluate_as(0, genomes[i]);
    return results;
  }
  // the order the workers pull in: longest predicted cost first when a hint is installed, input order otherwise
  std::vector<std::size_t> order(genomes.size());
  for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
  if (cost_hint_) {
    std::vector<double> cost(genomes.size());
    for (std::size_t i = 0; i < genomes.size(); ++i) cost[i] = cost_hint_(genomes[i]);
    std::stable_sort(order.begin(), order.end(), [&](std::size_t x, std::size_t y) { return cost[x] > cost[y]; });
  }
  std::atomic<std::size_t> cursor{0};
  std::mutex failure_mu;
  std::exception_ptr first_failure;
  auto body = [&](int worker) {
    for (std::size_t at = cursor.fetch_add(1); at < order.size(); at = cursor.fetch_add(1)) {
      const std::size_t i = order[at];
      try {
        results[i] = evaluate_as(worker, genomes[i]);
      } catch (...) {
        std::lock_guard<std::mutex> g(failure_mu);
        if (!first_failure) first_failure = std::current_exception();
        return;  // this worker stops; the others drain the batch
      }
    }
  };
  std::vector<std::thread> pool;
  pool.reserve(workers);
  for (std::size_t w = 0; w < workers; ++w) pool.emplace_back(body, static_cast<int>(w));
  for (std::thread& t : pool) t.join();
  if (first_failure) std::rethrow_exception(first_failure);
  return results;
}

EvalCounters Evaluator::counters() const {
  std::lock_guard<std::mutex> g(mu_);
  EvalCounters c;
  c.requests = requests_;
  c.distinct = distinct_;
  c.cache_hits = cache_hits_;
  c.backend_calls = backend_calls_;
  // std::map iterates in genome order: the sum is independent of scheduling
  for (const auto& [genome, slot] : memo_) {
    (void)genome;
    if (slot.seen_this_run && slot.done && !slot.failure) c.elapsed_s += slot.outcome.wall_cost_s;
  }
  return c;
}

MultiGpuEvaluator::MultiGpuEvaluator(std::unique_ptr<CudaBackend> backend, std::filesystem::path cache_file)
    : MultiGpuEvaluator(backend.release(), std::move(cache_file)) {}

MultiGpuEvaluator::MultiGpuEvaluator(CudaBackend* adopted, std::filesystem::path cache_file)
    : Evaluator(std::unique_ptr<EvalBackend>(adopted), adopted->num_slots(), std::move(cache_file)), cuda_(adopted) {
  const CudaBackendConfig config = cuda_->config();
  set_cost_hint([config](const Genome& g) { return predicted_cost(g, config); });
}

double MultiGpuEvaluator::predicted_cost(const Genome& genome, const CudaBackendConfig& config) {
  mmx_plan_info plan;
  if (genome.size() != MMX_GENE_LENGTH || mmx_plan(genome.bits().data(), genome.size(), config.n, config.dtype, &plan) != MMX_OK ||
      !plan.feasible)
    return 0.0;  // infeasible genomes are outcomes produced on the spot
  const double n = config.n, threads = std::max(1, config.host_threads);
  double s = 0.0;
  for (int k = 0; k < plan.num_steps; ++k) {
    const mmx_plan_step& st = plan.steps[k];
    switch (st.kind) {
      case MMX_STEP_CPU:  // ~2 GFLOP/s per host core on the contraction, ~1 G element/s on the O(N^2) nests
        s += st.nest == MMX_NEST_MATMUL ? 2.0 * n * n * n / (2.0e9 * threads) : n * n / 1.0e9;
        break;
      case MMX_STEP_GPU:  // ~3 us per launch of a launch train; the whole-nest kernels are the small term
        s += 3.0e-6 * static_cast<double>(st.launches) + (st.nest == MMX_NEST_MATMUL ? 2.0 * n * n * n / 3.0e13 : n * n / 5.0e11);
        break;
      default:  // transfers: ~25 GB/s over the bus
        s += 1.0e-5 + static_cast<double>(st.bytes) / 2.5e10;
    }
  }
  return std::min(s, config.timeout_s) * std::max(1, config.repetitions + config.warmup);
}

EvaluationOutcome MultiGpuEvaluator::measure_with(int worker, const Genome& genome) {
  return cuda_->measure_on(worker % cuda_->num_slots(), genome);
}

}  // namespace mmxhost
