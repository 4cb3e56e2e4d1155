#include "mmxhost/capi_host.h"
#include "mmxhost/commands.hpp"
#include "mmxhost/source_model.hpp"

#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <string>

#include "mmxhost/backend.hpp"
#include "mmxhost/calibrate.hpp"
#include "mmxhost/errors.hpp"
#include "mmxhost/evaluator.hpp"
#include "mmxhost/feasibility.hpp"
#include "mmxhost/ga.hpp"
#include "mmxhost/json_lite.hpp"
#include "mmxhost/kernel_match.hpp"
#include "mmxhost/cost_model.hpp"

using namespace mmxhost;

namespace {

thread_local std::string g_error;

int classify(const std::exception& e) {
  if (dynamic_cast<const GenomeLengthMismatch*>(&e)) return MMXH_E_LENGTH;
  if (dynamic_cast<const ToolchainMissing*>(&e)) return MMXH_E_TOOLCHAIN;
  if (dynamic_cast<const WorkdirUnwritable*>(&e)) return MMXH_E_WORKDIR;
  if (dynamic_cast<const ZeroTotalFitness*>(&e)) return MMXH_E_ZERO_FITNESS;
  if (dynamic_cast<const EvaluatorUnavailable*>(&e)) return MMXH_E_UNAVAILABLE;
  if (dynamic_cast<const NonPositiveTime*>(&e)) return MMXH_E_NONPOSITIVE;
  if (dynamic_cast<const ConfigError*>(&e)) return MMXH_E_CONFIG;
  if (dynamic_cast<const NoCandidates*>(&e)) return MMXH_E_NOCANDIDATES;
  if (dynamic_cast<const ModelError*>(&e)) return MMXH_E_MODEL;
  return MMXH_E_ERROR;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_error = e.what();
    return classify(e);
  }
}

Genome genome_of(const std::uint8_t* bits, std::size_t n) { return Genome(Genome::Bits(bits, bits + n)); }

int copy_out(const std::string& s, char* out, std::size_t cap) {
  if (out != nullptr && cap > 0) {
    const std::size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(out, s.data(), n);
    out[n] = '\0';
  }
  return static_cast<int>(s.size());
}

struct Handle {
  std::unique_ptr<Evaluator> ev;
  CallbackBackend* cb = nullptr;  // owned by ev
};

mmxh_outcome pack(const EvaluationOutcome& o) { return {static_cast<std::int32_t>(o.status), o.time_s, o.wall_cost_s}; }

std::filesystem::path path_or_empty(const char* p) { return p ? std::filesystem::path(p) : std::filesystem::path(); }

}  // namespace

extern "C" {

MMXH_API const char* mmxh_last_error(void) { return g_error.c_str(); }

MMXH_API int mmxh_model_time_all(const char* model_path, double* times, size_t count) {
  return guarded([&] {
    const CostModel m = load_model(model_path);
    const std::size_t a = m.gene_length();
    if (count != (std::size_t{1} << a)) return -1;
    for (std::size_t mask = 0; mask < count; ++mask) {
      Genome g = Genome::zeros(a);
      for (std::size_t k = 0; k < a; ++k) g.set(k, (mask >> k) & 1u);
      try {
        times[mask] = model_time(m, g);
      } catch (const SimulatedCompileError&) {
        times[mask] = -1.0;
      }
    }
    return static_cast<int>(a);
  });
}

MMXH_API int mmxh_exhaustive_best(const char* model_path, uint8_t* bits, size_t n, double* t) {
  return guarded([&] {
    const OracleResult r = exhaustive_best(load_model(model_path));
    if (r.genome.size() != n) return -1;
    std::memcpy(bits, r.genome.bits().data(), n);
    *t = r.time_s;
    return 0;
  });
}

MMXH_API int mmxh_fitness_from_time(double t, double* f) {
  return guarded([&] {
    *f = fitness_from_time(t);
    return 0;
  });
}

MMXH_API int mmxh_assign_fitness(const int32_t* status, const double* time_s, size_t m, double* fitness) {
  return guarded([&] {
    std::vector<Individual> pop(m);
    for (std::size_t i = 0; i < m; ++i) {
      pop[i].status = static_cast<IndividualStatus>(status[i]);
      pop[i].time_s = time_s[i];
    }
    assign_fitness(pop);
    for (std::size_t i = 0; i < m; ++i) fitness[i] = pop[i].fitness;
    return 0;
  });
}

MMXH_API int mmxh_init_population(size_t a, int m, uint64_t seed, uint8_t* bits) {
  return guarded([&] {
    GAParams p;
    p.population = m;
    Rng rng(seed);
    const auto pop = init_population(a, p, rng);
    for (std::size_t i = 0; i < pop.size(); ++i) std::memcpy(bits + i * a, pop[i].bits().data(), a);
    return 0;
  });
}

MMXH_API int mmxh_breed(const uint8_t* bits, const double* fitness, size_t m, size_t a, double pc, double pm, int elite,
                        uint64_t seed, uint64_t skip, uint8_t* next_bits) {
  return guarded([&] {
    GAParams p;
    p.population = static_cast<int>(m);
    p.crossover_rate = pc;
    p.mutation_rate = pm;
    p.elite_count = elite;
    std::vector<Individual> pop(m);
    for (std::size_t i = 0; i < m; ++i) {
      pop[i].genome = genome_of(bits + i * a, a);
      pop[i].status = IndividualStatus::Measured;
      pop[i].fitness = fitness[i];
    }
    Rng rng(seed);
    for (std::uint64_t s = 0; s < skip; ++s) rng.raw();
    const auto next = breed(pop, p, rng);
    for (std::size_t i = 0; i < next.size(); ++i) std::memcpy(next_bits + i * a, next[i].genome.bits().data(), a);
    return 0;
  });
}

MMXH_API int mmxh_roulette(const double* fitness, size_t m, size_t count, uint64_t seed, int32_t* picks) {
  return guarded([&] {
    std::vector<Individual> pop(m);
    for (std::size_t i = 0; i < m; ++i) {
      Genome::Bits b(32);
      for (int k = 0; k < 32; ++k) b[static_cast<std::size_t>(k)] = (i >> k) & 1u;
      pop[i].genome = Genome(std::move(b));
      pop[i].fitness = fitness[i];
    }
    Rng rng(seed);
    const auto sel = roulette_select(pop, count, rng);
    for (std::size_t n = 0; n < sel.size(); ++n) {
      std::int32_t v = 0;
      for (int k = 0; k < 31; ++k) v |= static_cast<std::int32_t>(sel[n].bits()[static_cast<std::size_t>(k)]) << k;
      picks[n] = v;
    }
    return 0;
  });
}

MMXH_API int mmxh_mutate(const uint8_t* bits, size_t a, double pm, uint64_t seed, uint8_t* out) {
  return guarded([&] {
    Rng rng(seed);
    const Genome g = mutate(genome_of(bits, a), pm, rng);
    std::memcpy(out, g.bits().data(), a);
    return 0;
  });
}

MMXH_API int mmxh_one_point_crossover(const uint8_t* p1, const uint8_t* p2, size_t a, uint64_t seed, uint8_t* c1, uint8_t* c2) {
  return guarded([&] {
    Rng rng(seed);
    const auto kids = one_point_crossover(genome_of(p1, a), genome_of(p2, a), rng);
    std::memcpy(c1, kids.first.bits().data(), a);
    std::memcpy(c2, kids.second.bits().data(), a);
    return 0;
  });
}

MMXH_API int mmxh_rng_draws(uint64_t seed, int kind, uint64_t n_arg, size_t count, double* out, uint64_t* raw_out) {
  return guarded([&] {
    Rng rng(seed);
    for (std::size_t i = 0; i < count; ++i) {
      if (kind == 0) out[i] = rng.bit() ? 1.0 : 0.0;
      else if (kind == 1) out[i] = rng.real01();
      else if (kind == 2) out[i] = static_cast<double>(rng.index(n_arg));
      else raw_out[i] = rng.raw();
    }
    return 0;
  });
}

MMXH_API void* mmxh_evaluator_create_sim(const char* model_path, int jobs, const char* cache_file) {
  try {
    auto h = std::make_unique<Handle>();
    h->ev = std::make_unique<Evaluator>(std::make_unique<SimBackend>(load_model(model_path)), jobs, path_or_empty(cache_file));
    return h.release();
  } catch (const std::exception& e) {
    g_error = e.what();
    return nullptr;
  }
}

MMXH_API void* mmxh_evaluator_create_cb(size_t genes, mmxh_measure_cb cb, void* user, int jobs, const char* cache_file) {
  try {
    auto h = std::make_unique<Handle>();
    auto backend = std::make_unique<CallbackBackend>(genes, [cb, user](const Genome& g) {
      mmxh_outcome o{static_cast<std::int32_t>(EvalStatus::RuntimeError), 0.0, 0.0};
      const int rc = cb(g.bits().data(), g.size(), &o, user);
      if (rc == -3) throw ToolchainMissing("callback: toolchain missing");
      if (rc < 0) throw Error("callback failed");
      EvaluationOutcome out;
      out.status = static_cast<EvalStatus>(o.status);
      out.time_s = o.time_s;
      out.wall_cost_s = o.wall_cost_s;
      return out;
    });
    h->cb = backend.get();
    h->ev = std::make_unique<Evaluator>(std::move(backend), jobs, path_or_empty(cache_file));
    return h.release();
  } catch (const std::exception& e) {
    g_error = e.what();
    return nullptr;
  }
}

MMXH_API int mmxh_evaluator_set_costs(void* h, const uint8_t* bits, const double* costs, size_t count, size_t n) {
  return guarded([&] {
    auto table = std::make_shared<std::map<Genome, double>>();
    for (std::size_t k = 0; k < count; ++k) (*table)[Genome(std::vector<std::uint8_t>(bits + k * n, bits + (k + 1) * n))] = costs[k];
    static_cast<Handle*>(h)->ev->set_cost_hint([table](const Genome& g) {
      const auto it = table->find(g);
      return it == table->end() ? 0.0 : it->second;
    });
    return 0;
  });
}

namespace {
CudaBackendConfig cuda_config_of(const mmxh_cuda_config* cfg) {
  CudaBackendConfig c;
  c.n = cfg->n;
  c.dtype = cfg->dtype;
  c.numerics = cfg->numerics;
  c.timeout_s = cfg->timeout_s;
  c.repetitions = cfg->repetitions;
  c.warmup = cfg->warmup;
  c.host_threads = cfg->host_threads;
  return c;
}
}  // namespace

MMXH_API double mmxh_predicted_cost(const mmxh_cuda_config* cfg, const uint8_t* bits, size_t n) {
  return MultiGpuEvaluator::predicted_cost(Genome(std::vector<std::uint8_t>(bits, bits + n)), cuda_config_of(cfg));
}

MMXH_API void* mmxh_evaluator_create_cuda(const mmxh_cuda_config* cfg, const char* cache_file) {
  try {
    CudaBackendConfig c;
    c.n = cfg->n;
    c.dtype = cfg->dtype;
    c.numerics = cfg->numerics;
    c.timeout_s = cfg->timeout_s;
    c.repetitions = cfg->repetitions;
    c.warmup = cfg->warmup;
    c.host_threads = cfg->host_threads;
    c.launch_batching = cfg->launch_batching != 0;
    c.matmul_variant = cfg->matmul_variant;
    c.devices.assign(cfg->devices, cfg->devices + cfg->num_devices);
    auto h = std::make_unique<Handle>();
    h->ev = std::make_unique<MultiGpuEvaluator>(std::make_unique<CudaBackend>(c), path_or_empty(cache_file));
    return h.release();
  } catch (const std::exception& e) {
    g_error = e.what();
    // encode the class in the message prefix so a ctypes caller can tell "no device" apart
    g_error = std::to_string(classify(e)) + ":" + g_error;
    return nullptr;
  }
}

MMXH_API void mmxh_evaluator_destroy(void* h) { delete static_cast<Handle*>(h); }

MMXH_API int mmxh_evaluator_gene_length(void* h) { return static_cast<int>(static_cast<Handle*>(h)->ev->gene_length()); }

MMXH_API int mmxh_evaluator_evaluate(void* h, const uint8_t* bits, size_t n, mmxh_outcome* out) {
  return guarded([&] {
    *out = pack(static_cast<Handle*>(h)->ev->evaluate(genome_of(bits, n)));
    return 0;
  });
}

MMXH_API int mmxh_evaluator_evaluate_all(void* h, const uint8_t* bits, size_t count, size_t n, mmxh_outcome* outs) {
  return guarded([&] {
    std::vector<Genome> gs;
    gs.reserve(count);
    for (std::size_t i = 0; i < count; ++i) gs.push_back(genome_of(bits + i * n, n));
    const auto os = static_cast<Handle*>(h)->ev->evaluate_all(gs);
    for (std::size_t i = 0; i < count; ++i) outs[i] = pack(os[i]);
    return 0;
  });
}

MMXH_API int mmxh_evaluator_counters(void* h, uint64_t c4[4], double* elapsed_s) {
  return guarded([&] {
    const EvalCounters c = static_cast<Handle*>(h)->ev->counters();
    c4[0] = c.requests;
    c4[1] = c.distinct;
    c4[2] = c.cache_hits;
    c4[3] = c.backend_calls;
    *elapsed_s = c.elapsed_s;
    return 0;
  });
}

MMXH_API int mmxh_evaluator_cb_stats(void* h, int32_t out2[2]) {
  auto* hd = static_cast<Handle*>(h);
  if (hd->cb == nullptr) return -1;
  out2[0] = hd->cb->calls.load();
  out2[1] = hd->cb->max_in_flight.load();
  return 0;
}

MMXH_API int mmxh_run_ga(void* evaluator, const mmxh_ga_params* params, char* csv, size_t csv_cap, uint8_t* best_bits,
                         double* best_s, double* baseline_s) {
  return guarded([&] {
    auto* hd = static_cast<Handle*>(evaluator);
    GAParams p;
    p.population = params->population;
    p.generations = params->generations;
    p.crossover_rate = params->crossover_rate;
    p.mutation_rate = params->mutation_rate;
    p.seed = params->seed;
    p.elite_count = params->elite_count;
    const TuningResult r = run_ga(hd->ev->gene_length(), p, *hd->ev);
    std::ostringstream s;
    write_generation_csv(s, r);
    std::memcpy(best_bits, r.best_genome.bits().data(), r.best_genome.size());
    *best_s = r.best_time_s;
    *baseline_s = r.baseline_s;
    return copy_out(s.str(), csv, csv_cap);
  });
}

namespace {

[[noreturn]] void rethrow_code(int rc) {
  switch (rc) {
    case MMXH_E_LENGTH: throw GenomeLengthMismatch("external evaluator: genome length mismatch");
    case MMXH_E_TOOLCHAIN: throw ToolchainMissing("external evaluator: measuring tool missing");
    case MMXH_E_WORKDIR: throw WorkdirUnwritable("external evaluator: workspace unwritable");
    case MMXH_E_CONFIG: throw ConfigError("external evaluator: bad configuration");
    default: throw Error("external evaluator failed");
  }
}

class ExternalEvaluator : public GenomeEvaluator {
 public:
  ExternalEvaluator(mmxh_batch_cb batch, mmxh_counters_cb counters, void* user) : batch_(batch), counters_(counters), user_(user) {}

  EvaluationOutcome evaluate(const Genome& genome) override { return evaluate_all({genome}).front(); }

  std::vector<EvaluationOutcome> evaluate_all(const std::vector<Genome>& genomes) override {
    std::vector<EvaluationOutcome> out(genomes.size());
    if (genomes.empty()) return out;
    const std::size_t n = genomes.front().size();
    std::vector<std::uint8_t> flat;
    flat.reserve(genomes.size() * n);
    for (const Genome& g : genomes) flat.insert(flat.end(), g.bits().begin(), g.bits().end());
    std::vector<mmxh_outcome> raw(genomes.size());
    const int rc = batch_(flat.data(), genomes.size(), n, raw.data(), user_);
    if (rc < 0) rethrow_code(rc);
    for (std::size_t i = 0; i < genomes.size(); ++i) {
      out[i].status = static_cast<EvalStatus>(raw[i].status);
      out[i].time_s = raw[i].time_s;
      out[i].wall_cost_s = raw[i].wall_cost_s;
    }
    return out;
  }

  EvalCounters counters() const override {
    std::uint64_t c4[4] = {0, 0, 0, 0};
    double elapsed = 0.0;
    const int rc = counters_(c4, &elapsed, user_);
    if (rc < 0) rethrow_code(rc);
    EvalCounters c;
    c.requests = c4[0];
    c.distinct = c4[1];
    c.cache_hits = c4[2];
    c.backend_calls = c4[3];
    c.elapsed_s = elapsed;
    return c;
  }

 private:
  mmxh_batch_cb batch_;
  mmxh_counters_cb counters_;
  void* user_;
};

}  // namespace

MMXH_API int mmxh_run_ga_external(size_t gene_length, mmxh_batch_cb batch, mmxh_counters_cb counters, void* user,
                                  const mmxh_ga_params* params, char* csv, size_t csv_cap, uint8_t* best_bits,
                                  double* best_s, double* baseline_s) {
  return guarded([&] {
    ExternalEvaluator ev(batch, counters, user);
    GAParams p;
    p.population = params->population;
    p.generations = params->generations;
    p.crossover_rate = params->crossover_rate;
    p.mutation_rate = params->mutation_rate;
    p.seed = params->seed;
    p.elite_count = params->elite_count;
    const TuningResult r = run_ga(gene_length, p, ev);
    std::ostringstream s;
    write_generation_csv(s, r);
    std::memcpy(best_bits, r.best_genome.bits().data(), r.best_genome.size());
    *best_s = r.best_time_s;
    *baseline_s = r.baseline_s;
    return copy_out(s.str(), csv, csv_cap);
  });
}

MMXH_API int mmxh_scan_loops(const char* path_label, const char* text, int64_t* rows7, size_t cap) {
  return guarded([&] {
    const SourceUnit unit = SourceUnit::from_string(path_label ? path_label : "<text>", text);
    const std::vector<LoopSite> loops = scan_loops(unit);
    for (std::size_t k = 0; k < loops.size() && k < cap; ++k) {
      const LoopSite& l = loops[k];
      int64_t* r = rows7 + 7 * k;
      r[0] = l.id;
      r[1] = static_cast<int64_t>(l.line);
      r[2] = l.depth;
      r[3] = static_cast<int64_t>(l.header_start);
      r[4] = static_cast<int64_t>(l.body_begin);
      r[5] = static_cast<int64_t>(l.body_end);
      r[6] = static_cast<int64_t>(l.indent.size());
    }
    return static_cast<int>(loops.size());
  });
}

MMXH_API int mmxh_render_variant(const char* text, const uint8_t* bits, size_t n, char* out, size_t cap) {
  return guarded([&] {
    const CandidateSet cs = all_loops_candidate_set(SourceUnit::from_string("<text>", text));
    return copy_out(render_variant(cs, Genome(std::vector<std::uint8_t>(bits, bits + n))), out, cap);
  });
}

MMXH_API int mmxh_strip_directives(const char* text, char* out, size_t cap) {
  return guarded([&] { return copy_out(strip_directives(text), out, cap); });
}

MMXH_API int mmxh_probe_source(const char* path_label, const char* text, char* report, size_t cap) {
  return guarded([&] {
    const SourceUnit unit = SourceUnit::from_string(path_label ? path_label : "<text>", text);
    const std::vector<LoopSite> loops = scan_loops(unit);
    std::vector<ProbeResult> results;
    int accepted = 0;
    try {
      accepted = static_cast<int>(build_candidate_set(unit, loops, &results).candidate_ids.size());
    } catch (const NoCandidates&) {
      copy_out(probe_report_jsonl(unit, loops, results), report, cap);
      throw;
    }
    copy_out(probe_report_jsonl(unit, loops, results), report, cap);
    return accepted;
  });
}

MMXH_API int mmxh_variant_feasible(const char* path_label, const char* text, const uint8_t* bits, size_t n, char* diag, size_t cap) {
  return guarded([&] {
    const CandidateSet cs = all_loops_candidate_set(SourceUnit::from_string(path_label ? path_label : "<text>", text));
    std::vector<ProbeResult> rejected;
    const bool ok = variant_feasible(cs, Genome(std::vector<std::uint8_t>(bits, bits + n)), &rejected);
    std::string lines;
    for (const ProbeResult& r : rejected) lines += r.compiler_message + "\n";
    copy_out(lines, diag, cap);
    return ok ? 1 : 0;
  });
}

MMXH_API int mmxh_match_kernels(const char* path_label, const char* text, char* json_out, size_t cap) {
  return guarded([&] {
    const SourceUnit unit = SourceUnit::from_string(path_label ? path_label : "<text>", text);
    const std::vector<LoopSite> loops = scan_loops(unit);
    const std::vector<KernelBinding> bs = match_kernels(unit, loops);
    std::string j = "{\"loops\":[";
    for (std::size_t k = 0; k < bs.size(); ++k) {
      const KernelBinding& b = bs[k];
      if (k) j += ",";
      j += "{\"id\":" + std::to_string(b.loop_id) + ",\"line\":" + std::to_string(b.line) + ",\"depth\":" + std::to_string(b.depth) +
           ",\"nest\":" + std::to_string(b.nest) + ",\"var\":" + json::dump_string(b.header.var) + ",\"bound\":" +
           json::dump_string(b.header.bound) + ",\"idiom\":" + json::dump_string(to_string(b.idiom)) + ",\"kernel\":" +
           json::dump_string(b.kernel) + ",\"writes\":" + json::dump_string(b.writes) + ",\"reads\":[";
      for (std::size_t r = 0; r < b.reads.size(); ++r) j += (r ? "," : "") + json::dump_string(b.reads[r]);
      j += "],\"why\":" + json::dump_string(b.why_unmatched) + "}";
    }
    j += "],\"dataflow\":[";
    const std::vector<DataflowEdge> edges = derive_dataflow(bs);
    for (std::size_t k = 0; k < edges.size(); ++k)
      j += std::string(k ? "," : "") + "[" + json::dump_string(edges[k].array) + "," + std::to_string(edges[k].producer_nest) + "," +
           std::to_string(edges[k].consumer_nest) + "]";
    j += "]}";
    copy_out(j, json_out, cap);
    return static_cast<int>(bs.size());
  });
}

namespace {
PlanModel plan_of(const double* p, int n, int dtype) {
  PlanModel m;
  m.n = n;
  m.dtype = dtype;
  m.serial_s = p[0];
  for (int i = 0; i < MMX_NUM_NESTS; ++i) m.cpu_s[i] = p[1 + i];
  for (int k = 0; k < MMX_GENE_LENGTH; ++k) m.loop_s[k] = p[7 + k];
  m.h2d_s_per_byte = p[19];
  m.d2h_s_per_byte = p[20];
  m.per_transfer_s = p[21];
  return m;
}
}  // namespace

MMXH_API int mmxh_calibrate(const uint8_t* bits, const double* times, size_t count, int n, int dtype, char* model_json, size_t cap,
                            double* plan22, double* report8, uint8_t* best_bits) {
  return guarded([&] {
    std::vector<GenomeSample> samples;
    for (std::size_t k = 0; k < count; ++k)
      samples.push_back({Genome(std::vector<std::uint8_t>(bits + k * MMX_GENE_LENGTH, bits + (k + 1) * MMX_GENE_LENGTH)), times[k]});
    FitReport fit;
    const PlanModel m = fit_plan_model(samples, n, dtype, &fit);
    ProjectionReport proj;
    const CostModel cm = project_to_cost_model(m, &proj);
    plan22[0] = m.serial_s;
    for (int i = 0; i < MMX_NUM_NESTS; ++i) plan22[1 + i] = m.cpu_s[i];
    for (int k = 0; k < MMX_GENE_LENGTH; ++k) plan22[7 + k] = m.loop_s[k];
    plan22[19] = m.h2d_s_per_byte;
    plan22[20] = m.d2h_s_per_byte;
    plan22[21] = m.per_transfer_s;
    const double rep[8] = {fit.rms_rel_err, fit.max_rel_err, proj.rms_rel_err, proj.max_rel_err, proj.plan_best_s, proj.cost_best_s,
                           static_cast<double>(proj.inexact_loops.size()), static_cast<double>(fit.samples)};
    std::memcpy(report8, rep, sizeof(rep));
    std::memcpy(best_bits, proj.plan_best.bits().data(), MMX_GENE_LENGTH);
    std::memcpy(best_bits + MMX_GENE_LENGTH, proj.cost_best.bits().data(), MMX_GENE_LENGTH);
    return copy_out(dump_cost_model_json(cm), model_json, cap);
  });
}

MMXH_API int mmxh_plan_model_times(const double* plan22, int n, int dtype, double* times4096) {
  return guarded([&] {
    const PlanModel m = plan_of(plan22, n, dtype);
    for (unsigned mask = 0; mask < 4096; ++mask) {
      std::vector<std::uint8_t> b(MMX_GENE_LENGTH);
      for (int k = 0; k < MMX_GENE_LENGTH; ++k) b[static_cast<std::size_t>(k)] = (mask >> k) & 1u;
      try {
        times4096[mask] = predict_time(m, Genome(std::move(b)));
      } catch (const SimulatedCompileError&) {
        times4096[mask] = -1.0;
      }
    }
    return 0;
  });
}

MMXH_API int mmxh_cmd_tune(const char* config_path, int has_seed, uint64_t seed, const char* sim_model_or_null, char* out, size_t out_cap,
                           char* err, size_t err_cap) {
  std::ostringstream o, e;
  TuneOptions opt;
  if (has_seed) opt.seed = seed;
  if (sim_model_or_null != nullptr) opt.sim_model = std::string(sim_model_or_null);
  const int rc = cmd_tune(config_path, opt, o, e);
  copy_out(o.str(), out, out_cap);
  copy_out(e.str(), err, err_cap);
  return rc;
}

MMXH_API int mmxh_cmd_report(const char* workdir, char* out, size_t out_cap, char* err, size_t err_cap) {
  std::ostringstream o, e;
  const int rc = cmd_report(workdir, o, e);
  copy_out(o.str(), out, out_cap);
  copy_out(e.str(), err, err_cap);
  return rc;
}

MMXH_API int mmxh_cmd_analyze(const char* config_path, char* out, size_t out_cap, char* err, size_t err_cap) {
  std::ostringstream o, e;
  const int rc = cmd_analyze(config_path, o, e);
  copy_out(o.str(), out, out_cap);
  copy_out(e.str(), err, err_cap);
  return rc;
}

MMXH_API int mmxh_cmd_calibrate(const char* config_path, char* out, size_t out_cap, char* err, size_t err_cap) {
  std::ostringstream o, e;
  const int rc = cmd_calibrate(config_path, o, e);
  copy_out(o.str(), out, out_cap);
  copy_out(e.str(), err, err_cap);
  return rc;
}

MMXH_API const char* mmxh_status_name(int status) {
  static thread_local std::string s;
  s = std::string(to_string(static_cast<EvalStatus>(status)));
  return s.c_str();
}

MMXH_API int mmxh_dump_number(double v, char* out, size_t cap) { return copy_out(json::dump_number(v), out, cap); }

}  // extern "C"
