#include "mmxhost/backend.hpp"

#include <string>

#include "mmxhost/errors.hpp"

namespace mmxhost {

// ---- SimBackend ---------------------------------------------------------------------------
// wall_cost equals the model time, so cold and resumed runs account identical elapsed totals
// (evaluator.hpp:26-29 of the reference).
EvaluationOutcome SimBackend::measure(const Genome& genome) {
  EvaluationOutcome out;
  try {
    const double t = model_time(model_, genome);
    out.status = EvalStatus::Measured;
    out.time_s = t;
    out.wall_cost_s = t;
  } catch (const SimulatedCompileError&) {
    out.status = EvalStatus::CompileError;
  }
  return out;
}

// ---- CallbackBackend ------------------------------------------------------------------------
EvaluationOutcome CallbackBackend::measure(const Genome& genome) {
  calls.fetch_add(1);
  const int now = in_flight.fetch_add(1) + 1;
  int seen = max_in_flight.load();
  while (now > seen && !max_in_flight.compare_exchange_weak(seen, now)) {
  }
  struct Leave {
    std::atomic<int>& counter;
    ~Leave() { counter.fetch_sub(1); }
  } leave{in_flight};
  return fn_(genome);
}

// ---- CudaBackend ----------------------------------------------------------------------------
void throw_for_code(int code, const std::string& message) {
  switch (code) {
    case MMX_E_LENGTH: throw GenomeLengthMismatch(message);
    case MMX_E_NODEVICE: throw ToolchainMissing(message);
    case MMX_E_INVALID: throw ConfigError(message);
    case MMX_E_NOMEM: throw WorkdirUnwritable(message);
    default: throw Error(message);
  }
}

CudaBackend::CudaBackend(const CudaBackendConfig& config) : config_(config) {
  if (config.devices.empty()) throw ConfigError("CudaBackend needs at least one device slot");
  mmx_config c;
  mmx_default_config(&c);
  c.n = config.n;
  c.dtype = config.dtype;
  c.numerics = config.numerics;
  c.timeout_s = config.timeout_s;
  c.repetitions = config.repetitions;
  c.warmup = config.warmup;
  c.num_slots = static_cast<int>(config.devices.size());
  std::vector<std::int32_t> devs(config.devices.begin(), config.devices.end());
  c.devices = devs.data();
  c.host_threads = config.host_threads;
  c.launch_batching = config.launch_batching ? 1 : 0;
  c.matmul_variant = config.matmul_variant;
  c.pin_host = config.pin_host ? 1 : 0;
  c.host_core_first = config.host_core_first;
  c.host_core_count = config.host_core_count;
  c.early_timeout = config.early_timeout ? 1 : 0;
  const int rc = mmx_create(&c, &ctx_);
  if (rc != MMX_OK) throw_for_code(rc, std::string("mmx_create: ") + mmx_last_error(nullptr));
  busy_.assign(config.devices.size(), 0);
}

CudaBackend::~CudaBackend() { mmx_destroy(ctx_); }

std::size_t CudaBackend::gene_length() const { return mmx_gene_length(ctx_); }

int CudaBackend::num_slots() const { return mmx_num_slots(ctx_); }

int CudaBackend::acquire_slot() {
  std::unique_lock<std::mutex> lock(mu_);
  for (;;) {
    for (std::size_t s = 0; s < busy_.size(); ++s)
      if (!busy_[s]) {
        busy_[s] = 1;
        return static_cast<int>(s);
      }
    cv_.wait(lock);
  }
}

void CudaBackend::release_slot(int slot) {
  {
    std::lock_guard<std::mutex> g(mu_);
    busy_[static_cast<std::size_t>(slot)] = 0;
  }
  cv_.notify_one();
}

EvaluationOutcome CudaBackend::measure_on(int slot, const Genome& genome) {
  mmx_outcome raw{};
  const int rc = mmx_measure(ctx_, slot, genome.bits().data(), genome.size(), &raw);
  if (rc != MMX_OK) throw_for_code(rc, std::string("mmx_measure: ") + mmx_last_error(ctx_));
  EvaluationOutcome out;
  out.status = static_cast<EvalStatus>(raw.status);
  out.time_s = raw.time_s;
  out.wall_cost_s = raw.wall_cost_s;
  return out;
}

EvaluationOutcome CudaBackend::measure(const Genome& genome) {
  const int slot = acquire_slot();
  struct Release {
    CudaBackend* self;
    int slot;
    ~Release() { self->release_slot(slot); }
  } release{this, slot};
  return measure_on(slot, genome);
}

mmx_run_stats CudaBackend::last_stats(int slot) const {
  mmx_run_stats st{};
  mmx_last_stats(ctx_, slot, &st);
  return st;
}

}  // namespace mmxhost
