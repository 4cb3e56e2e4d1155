// backend.hpp -- EvalBackend and its implementations.
//
// EvalBackend is THE drop-in boundary (/root/reference/proj/include/acctune/evaluator.hpp:19-24):
// one call = one real measurement of one genome; backends carry no cache; measure() is called
// concurrently from up to `jobs` threads on distinct genomes (evaluator.cpp:196-205).
//
//   SimBackend      times from a CostModel (evaluator.cpp:23-35) -- deterministic test double
//   CallbackBackend scripted by a std::function (the reference tests' ScriptBackend, test_util.hpp:55-81)
//   CudaBackend     the product: forwards to the C ABI (include/mmx.h); concurrent callers are
//                   spread over the context's device slots
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <functional>
#include <mutex>
#include <optional>
#include <string_view>
#include <vector>

#include "mmx.h"
#include "mmxhost/genome.hpp"
#include "mmxhost/cost_model.hpp"

namespace mmxhost {

// ---- what a measurement returns (/root/reference/proj/include/acctune/evaluation.hpp:13-37, src/evaluation.cpp:5-25) ----

// Numeric values are part of the C ABI (mmx_status in include/mmx.h).
enum class EvalStatus : int { Measured = 0, CompileError = 1, RuntimeError = 2, Timeout = 3 };

inline std::string_view to_string(EvalStatus s) {
  switch (s) {
    case EvalStatus::Measured: return "measured";
    case EvalStatus::CompileError: return "compile_error";
    case EvalStatus::Timeout: return "timeout";
    case EvalStatus::RuntimeError: break;
  }
  return "runtime_error";
}

inline std::optional<EvalStatus> eval_status_from_string(std::string_view s) {
  for (EvalStatus st : {EvalStatus::Measured, EvalStatus::CompileError, EvalStatus::RuntimeError, EvalStatus::Timeout})
    if (s == to_string(st)) return st;
  return std::nullopt;
}

struct EvaluationOutcome {
  EvalStatus status = EvalStatus::RuntimeError;
  double time_s = 0.0;       // Measured: benchmark time; Timeout: the budget; otherwise 0
  double wall_cost_s = 0.0;  // cost of producing the outcome the first time
};

struct EvalCounters {
  std::uint64_t requests = 0;       // evaluate() calls
  std::uint64_t distinct = 0;       // unique genomes seen this run
  std::uint64_t cache_hits = 0;     // requests - distinct
  std::uint64_t backend_calls = 0;  // real measurements (disk-cache hits excluded)
  double elapsed_s = 0.0;           // sum of wall_cost_s over distinct genomes, in genome order
};

// ---- backends -------------------------------------------------------------------------------------------------

class EvalBackend {
 public:
  virtual ~EvalBackend() = default;
  virtual EvaluationOutcome measure(const Genome& genome) = 0;
  virtual std::size_t gene_length() const = 0;
};

class SimBackend : public EvalBackend {
 public:
  explicit SimBackend(CostModel model) : model_(std::move(model)) {}
  EvaluationOutcome measure(const Genome& genome) override;
  std::size_t gene_length() const override { return model_.gene_length(); }
  const CostModel& model() const { return model_; }

 private:
  CostModel model_;
};

class CallbackBackend : public EvalBackend {
 public:
  using Fn = std::function<EvaluationOutcome(const Genome&)>;
  CallbackBackend(std::size_t gene_length, Fn fn) : gene_length_(gene_length), fn_(std::move(fn)) {}
  EvaluationOutcome measure(const Genome& genome) override;
  std::size_t gene_length() const override { return gene_length_; }

  std::atomic<int> calls{0};
  std::atomic<int> in_flight{0};
  std::atomic<int> max_in_flight{0};

 private:
  std::size_t gene_length_;
  Fn fn_;
};

struct CudaBackendConfig {
  int n = 256;                 // fixtures/matmul.c:3
  int dtype = MMX_F64;
  int numerics = MMX_NUMERICS_FAST;
  double timeout_s = 120.0;    // ToolchainConfig::timeout_s
  int repetitions = 1;         // ToolchainConfig::repetitions
  int warmup = 0;
  std::vector<int> devices = {0};  // one slot per entry (repeat an ordinal for several slots on one GPU)
  int host_threads = 1;
  bool launch_batching = true;
  int matmul_variant = 0;
  // every slot measures on its own share of the host's CPUs (mmx_config.pin_host); first / count restrict the
  // context to a sub-range of the allowed CPUs (one process per GPU: each rank passes its share); count 0 = all of them
  bool pin_host = true;
  int host_core_first = 0;
  int host_core_count = 0;
  // hopeless runs are given up as soon as their measured progress shows that the budget cannot be met (mmx_config.early_timeout):
  // the outcome is the full wait's (Timeout, time = budget), the wall cost a fraction of it
  bool early_timeout = true;
};

// Throws ToolchainMissing when there is no CUDA device (there is no CPU fallback), ConfigError
// on bad settings, WorkdirUnwritable-class Error on allocation failure.
class CudaBackend : public EvalBackend {
 public:
  explicit CudaBackend(const CudaBackendConfig& config);
  ~CudaBackend() override;
  CudaBackend(const CudaBackend&) = delete;
  CudaBackend& operator=(const CudaBackend&) = delete;

  EvaluationOutcome measure(const Genome& genome) override;
  std::size_t gene_length() const override;

  // measure on a caller-chosen slot (MultiGpuEvaluator pins worker s to slot s)
  EvaluationOutcome measure_on(int slot, const Genome& genome);
  int num_slots() const;
  mmx_ctx* handle() const { return ctx_; }
  mmx_run_stats last_stats(int slot) const;
  const CudaBackendConfig& config() const { return config_; }

 private:
  int acquire_slot();
  void release_slot(int slot);

  mmx_ctx* ctx_ = nullptr;
  CudaBackendConfig config_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<char> busy_;
};

// Turns a C ABI return code into the exception type the reference would throw.
[[noreturn]] void throw_for_code(int code, const std::string& message);

}  // namespace mmxhost
