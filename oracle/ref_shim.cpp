// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A plain-C window onto the UNMODIFIED reference tuner core (acctune, C++20),
// compiled from the sources where they lie under /root/reference/proj by
// oracle/Makefile into oracle/_ref/libacctune_ref.so.  It exists so the Python
// tests and tests/golden/generate_golden.py can (a) produce golden vectors from
// the reference itself and (b) run the reference Evaluator / GA side by side with
// this repo's restatement (paper_1806_01430_b200/host) on identical scripted
// backends.  Nothing here restates an algorithm: every function forwards to the
// reference symbol named in its comment.
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "acctune/commands.hpp"
#include "acctune/errors.hpp"
#include "acctune/evaluation.hpp"
#include "acctune/evaluator.hpp"
#include "acctune/ga.hpp"
#include "acctune/probe.hpp"
#include "acctune/genome.hpp"
#include "acctune/rng.hpp"
#include "acctune/sim_model.hpp"
#include "acctune/source_model.hpp"

using namespace acctune;

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_error;

int copy_out(const std::string& s, char* out, std::size_t cap) {
  if (out == nullptr || cap == 0) return static_cast<int>(s.size());
  const std::size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
  std::memcpy(out, s.data(), n);
  out[n] = '\0';
  return static_cast<int>(s.size());
}

// error class -> small code, so tests can assert on the exception type
int classify(const std::exception& e) {
  if (dynamic_cast<const GenomeLengthMismatch*>(&e)) return -2;
  if (dynamic_cast<const ToolchainMissing*>(&e)) return -3;
  if (dynamic_cast<const WorkdirUnwritable*>(&e)) return -4;
  if (dynamic_cast<const ZeroTotalFitness*>(&e)) return -5;
  if (dynamic_cast<const EvaluatorUnavailable*>(&e)) return -6;
  if (dynamic_cast<const NonPositiveTime*>(&e)) return -7;
  if (dynamic_cast<const ConfigError*>(&e)) return -8;
  if (dynamic_cast<const NoCandidates*>(&e)) return -9;
  if (dynamic_cast<const ModelError*>(&e)) return -10;
  return -1;
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

Genome genome_of(const std::uint8_t* bits, std::size_t n) {
  return Genome(std::vector<std::uint8_t>(bits, bits + n));
}

// Same synthetic unit the reference tests use (tests/test_util.hpp:84-97 builds
// one loop per gene); written here independently, only the shape matters.
CandidateSet flat_candidate_set(std::size_t genes) {
  std::string text = "void f(double* a, int n) {\n";
  for (std::size_t g = 0; g < genes; ++g) {
    const std::string v = "i" + std::to_string(g);
    text += "  for (int " + v + " = 0; " + v + " < n; " + v + "++) a[" + v + "] += 1.0;\n";
  }
  text += "}\n";
  CandidateSet cs;
  cs.unit = SourceUnit::from_string("flat.c", text);
  cs.all_loops = scan_loops(cs.unit);
  for (const auto& l : cs.all_loops) cs.candidate_ids.push_back(l.id);
  return cs;
}

CandidateSet file_candidate_set(const char* source_path) {
  CandidateSet cs;
  cs.unit = SourceUnit::from_file(source_path);
  cs.all_loops = scan_loops(cs.unit);
  for (const auto& l : cs.all_loops) cs.candidate_ids.push_back(l.id);
  return cs;
}

struct ref_outcome {
  std::int32_t status;
  double time_s;
  double wall_cost_s;
};

using measure_cb = int (*)(const std::uint8_t* bits, std::size_t n, ref_outcome* out, void* user);

// EvalBackend driven by a C callback.  Callback return: 0 ok, -3 => throw
// ToolchainMissing, any other negative => throw Error.
class CallbackBackend : public EvalBackend {
 public:
  CallbackBackend(std::size_t genes, measure_cb cb, void* user) : genes_(genes), cb_(cb), user_(user) {}
  EvaluationOutcome measure(const Genome& g) override {
    ref_outcome o{2, 0.0, 0.0};
    const int rc = cb_(g.bits().data(), g.size(), &o, user_);
    if (rc == -3) throw ToolchainMissing("callback: toolchain missing");
    if (rc < 0) throw Error("callback failed");
    EvaluationOutcome out;
    out.status = static_cast<EvalStatus>(o.status);
    out.time_s = o.time_s;
    out.wall_cost_s = o.wall_cost_s;
    return out;
  }
  std::size_t gene_length() const override { return genes_; }

 private:
  std::size_t genes_;
  measure_cb cb_;
  void* user_;
};

struct RefEvaluator {
  std::unique_ptr<Evaluator> ev;
  std::size_t genes;
};

}  // namespace

REF_API const char* ref_last_error() { return g_error.c_str(); }

// ---- source scan + render (source_model.cpp:342-376) ----------------------------

// Writes "id,line,depth\n" rows for every scanned loop.
REF_API int ref_scan_loops(const char* source_path, char* out, std::size_t cap) {
  return guarded([&] {
    const CandidateSet cs = file_candidate_set(source_path);
    std::ostringstream s;
    for (const auto& l : cs.all_loops)
      s << l.id << ',' << cs.unit.lines.line_col_of(l.header_start).line << ',' << l.depth << '\n';
    return copy_out(s.str(), out, cap);
  });
}

REF_API int ref_render_variant(const char* source_path, const std::uint8_t* bits, std::size_t n,
                               char* out, std::size_t cap) {
  return guarded([&] {
    const CandidateSet cs = file_candidate_set(source_path);
    return copy_out(render_variant(cs, genome_of(bits, n)), out, cap);
  });
}

// ---- sim model (sim_model.cpp:22-41, 76-98) --------------------------------------

// status: 0 measured (time in *t), 1 simulated compile error
REF_API int ref_model_time(const char* model_path, const std::uint8_t* bits, std::size_t n, double* t) {
  return guarded([&] {
    const CostModel m = load_model(model_path);
    try {
      *t = model_time(m, genome_of(bits, n));
    } catch (const SimulatedCompileError&) {
      *t = 0.0;
      return 1;
    }
    return 0;
  });
}

// All 2^a model times in mask order (bit k of the index = gene k); failing genomes get -1.
REF_API int ref_model_time_all(const char* model_path, double* times, std::size_t count) {
  return guarded([&] {
    const CostModel m = load_model(model_path);
    const std::size_t a = m.gene_length();
    if (count != (std::size_t{1} << a)) return -1;
    for (std::size_t mask = 0; mask < count; ++mask) {
      std::vector<std::uint8_t> bits(a);
      for (std::size_t k = 0; k < a; ++k) bits[k] = (mask >> k) & 1u;
      try {
        times[mask] = model_time(m, Genome(std::move(bits)));
      } catch (const SimulatedCompileError&) {
        times[mask] = -1.0;
      }
    }
    return static_cast<int>(a);
  });
}

REF_API int ref_exhaustive_best(const char* model_path, std::uint8_t* bits, std::size_t n, double* t) {
  return guarded([&] {
    const CostModel m = load_model(model_path);
    const OracleResult r = exhaustive_best(m);
    if (r.genome.size() != n) return -1;
    std::memcpy(bits, r.genome.bits().data(), n);
    *t = r.time_s;
    return 0;
  });
}

// ---- GA pieces (ga.cpp) -------------------------------------------------------------

REF_API int ref_fitness_from_time(double t, double* f) {
  return guarded([&] {
    *f = fitness_from_time(t);
    return 0;
  });
}

// status[i]: 0 unevaluated, 1 measured, 2 failed (IndividualStatus order, ga.hpp:27)
REF_API int ref_assign_fitness(const std::int32_t* status, const double* time_s, std::size_t m,
                               double* fitness) {
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

REF_API int ref_init_population(std::size_t a, int m, std::uint64_t seed, std::uint8_t* bits) {
  return guarded([&] {
    GAParams p;
    p.population = m;
    p.seed = seed;
    Rng rng(seed);
    const auto pop = init_population(a, p, rng);
    for (std::size_t i = 0; i < pop.size(); ++i) std::memcpy(bits + i * a, pop[i].bits().data(), a);
    return 0;
  });
}

// One breed() step from a fresh Rng(seed) advanced by `skip` raw draws.
REF_API int ref_breed(const std::uint8_t* bits, const double* fitness, std::size_t m, std::size_t a,
                      double pc, double pm, int elite, std::uint64_t seed, std::uint64_t skip,
                      std::uint8_t* next_bits) {
  return guarded([&] {
    GAParams p;
    p.population = static_cast<int>(m);
    p.crossover_rate = pc;
    p.mutation_rate = pm;
    p.elite_count = elite;
    p.seed = seed;
    std::vector<Individual> pop(m);
    for (std::size_t i = 0; i < m; ++i) {
      pop[i].genome = genome_of(bits + i * a, a);
      pop[i].status = IndividualStatus::Measured;
      pop[i].fitness = fitness[i];
    }
    Rng rng(seed);
    for (std::uint64_t s = 0; s < skip; ++s) rng.raw();
    const auto next = breed(pop, p, rng);
    for (std::size_t i = 0; i < next.size(); ++i)
      std::memcpy(next_bits + i * a, next[i].genome.bits().data(), a);
    return 0;
  });
}

// Individual operators from Rng(seed): roulette (count draws), mutate, crossover.
REF_API int ref_roulette(const double* fitness, std::size_t m, std::size_t count, std::uint64_t seed,
                         std::int32_t* picks) {
  return guarded([&] {
    std::vector<Individual> pop(m);
    for (std::size_t i = 0; i < m; ++i) {
      // genome encodes the slot index so the pick can be read back
      std::vector<std::uint8_t> b(32);
      for (int k = 0; k < 32; ++k) b[k] = (i >> k) & 1u;
      pop[i].genome = Genome(std::move(b));
      pop[i].fitness = fitness[i];
    }
    Rng rng(seed);
    const auto sel = roulette_select(pop, count, rng);
    for (std::size_t n = 0; n < sel.size(); ++n) {
      std::int32_t v = 0;
      for (int k = 0; k < 32; ++k) v |= static_cast<std::int32_t>(sel[n].bits()[k]) << k;
      picks[n] = v;
    }
    return 0;
  });
}

REF_API int ref_mutate(const std::uint8_t* bits, std::size_t a, double pm, std::uint64_t seed,
                       std::uint8_t* out) {
  return guarded([&] {
    Rng rng(seed);
    const Genome g = mutate(genome_of(bits, a), pm, rng);
    std::memcpy(out, g.bits().data(), a);
    return 0;
  });
}

REF_API int ref_one_point_crossover(const std::uint8_t* p1, const std::uint8_t* p2, std::size_t a,
                                    std::uint64_t seed, std::uint8_t* c1, std::uint8_t* c2) {
  return guarded([&] {
    Rng rng(seed);
    auto [x, y] = one_point_crossover(genome_of(p1, a), genome_of(p2, a), rng);
    std::memcpy(c1, x.bits().data(), a);
    std::memcpy(c2, y.bits().data(), a);
    return 0;
  });
}

// Rng helpers (rng.hpp:13-31): kind 0 bit, 1 real01, 2 index(n), 3 raw; values as doubles
// except raw (returned through raw_out).
REF_API int ref_rng_draws(std::uint64_t seed, int kind, std::uint64_t n_arg, std::size_t count,
                          double* out, std::uint64_t* raw_out) {
  return guarded([&] {
    Rng rng(seed);
    for (std::size_t i = 0; i < count; ++i) {
      switch (kind) {
        case 0: out[i] = rng.bit() ? 1.0 : 0.0; break;
        case 1: out[i] = rng.real01(); break;
        case 2: out[i] = static_cast<double>(rng.index(n_arg)); break;
        default: raw_out[i] = rng.raw(); break;
      }
    }
    return 0;
  });
}

// Full run_ga (ga.cpp:247-295) on SimBackend + Evaluator, returning generations.csv
// (ga.cpp:297-309) and the counters.  source_path may be NULL: then a flat unit with
// one loop per gene is synthesised.
REF_API int ref_run_ga_sim(const char* model_path, const char* source_path, int m, int t, double pc,
                           double pm, int elite, std::uint64_t seed, int jobs, const char* cache_file,
                           char* csv, std::size_t csv_cap, std::uint8_t* best_bits, double* best_s,
                           double* baseline_s, std::uint64_t counters[4], double* elapsed_s) {
  return guarded([&] {
    CostModel model = load_model(model_path);
    const std::size_t a = model.gene_length();
    const CandidateSet cs = source_path ? file_candidate_set(source_path) : flat_candidate_set(a);
    if (cs.gene_length() != a) throw ConfigError("model/source gene length mismatch");
    GAParams p;
    p.population = m;
    p.generations = t;
    p.crossover_rate = pc;
    p.mutation_rate = pm;
    p.elite_count = elite;
    p.seed = seed;
    Evaluator ev(std::make_unique<SimBackend>(std::move(model)), jobs,
                 cache_file ? std::filesystem::path(cache_file) : std::filesystem::path());
    const TuningResult r = run_ga(cs, p, ev);
    std::ostringstream s;
    write_generation_csv(s, r);
    std::memcpy(best_bits, r.best_genome.bits().data(), a);
    *best_s = r.best_time_s;
    *baseline_s = r.baseline_s;
    const EvalCounters c = ev.counters();
    counters[0] = c.requests;
    counters[1] = c.distinct;
    counters[2] = c.cache_hits;
    counters[3] = c.backend_calls;
    *elapsed_s = c.elapsed_s;
    return copy_out(s.str(), csv, csv_cap);
  });
}

// run_ga over a callback backend (for failure-mode parity: all failed, baseline failed ...).
REF_API int ref_run_ga_cb(std::size_t a, measure_cb cb, void* user, int m, int t, double pc, double pm,
                          int elite, std::uint64_t seed, int jobs, char* csv, std::size_t csv_cap,
                          std::uint8_t* best_bits, double* best_s) {
  return guarded([&] {
    const CandidateSet cs = flat_candidate_set(a);
    GAParams p;
    p.population = m;
    p.generations = t;
    p.crossover_rate = pc;
    p.mutation_rate = pm;
    p.elite_count = elite;
    p.seed = seed;
    Evaluator ev(std::make_unique<CallbackBackend>(a, cb, user), jobs);
    const TuningResult r = run_ga(cs, p, ev);
    std::ostringstream s;
    write_generation_csv(s, r);
    std::memcpy(best_bits, r.best_genome.bits().data(), a);
    *best_s = r.best_time_s;
    return copy_out(s.str(), csv, csv_cap);
  });
}

// ---- Evaluator over a callback backend (evaluator.cpp:144-292) -------------------------

REF_API void* ref_evaluator_create_cb(std::size_t genes, measure_cb cb, void* user, int jobs,
                                   const char* cache_file) {
  try {
    auto* h = new RefEvaluator;
    h->genes = genes;
    h->ev = std::make_unique<Evaluator>(
        std::make_unique<CallbackBackend>(genes, cb, user), jobs,
        cache_file ? std::filesystem::path(cache_file) : std::filesystem::path());
    return h;
  } catch (const std::exception& e) {
    g_error = e.what();
    return nullptr;
  }
}

REF_API void ref_evaluator_destroy(void* h) { delete static_cast<RefEvaluator*>(h); }

REF_API int ref_evaluator_evaluate(void* h, const std::uint8_t* bits, std::size_t n, ref_outcome* out) {
  return guarded([&] {
    const EvaluationOutcome o = static_cast<RefEvaluator*>(h)->ev->evaluate(genome_of(bits, n));
    *out = {static_cast<std::int32_t>(o.status), o.time_s, o.wall_cost_s};
    return 0;
  });
}

REF_API int ref_evaluator_evaluate_all(void* h, const std::uint8_t* bits, std::size_t count,
                                       std::size_t n, ref_outcome* outs) {
  return guarded([&] {
    std::vector<Genome> gs;
    for (std::size_t i = 0; i < count; ++i) gs.push_back(genome_of(bits + i * n, n));
    const auto os = static_cast<RefEvaluator*>(h)->ev->evaluate_all(gs);
    for (std::size_t i = 0; i < count; ++i)
      outs[i] = {static_cast<std::int32_t>(os[i].status), os[i].time_s, os[i].wall_cost_s};
    return 0;
  });
}

REF_API int ref_evaluator_counters(void* h, std::uint64_t c4[4], double* elapsed_s) {
  return guarded([&] {
    const EvalCounters c = static_cast<RefEvaluator*>(h)->ev->counters();
    c4[0] = c.requests;
    c4[1] = c.distinct;
    c4[2] = c.cache_hits;
    c4[3] = c.backend_calls;
    *elapsed_s = c.elapsed_s;
    return 0;
  });
}

// scan_loops on in-memory text: one line per loop "id,line,depth,header_start,body_begin,body_end,indent_len"
REF_API int ref_scan_text(const char* text, char* out, std::size_t cap) {
  return guarded([&] {
    const SourceUnit unit = SourceUnit::from_string("<text>", text);
    std::ostringstream s;
    for (const LoopSite& l : scan_loops(unit))
      s << l.id << "," << unit.lines.line_col_of(l.header_start).line << "," << l.depth << "," << l.header_start << ","
        << l.body_span.begin << "," << l.body_span.end << "," << l.indent.size() << "\n";
    return copy_out(s.str(), out, cap);
  });
}

// render_variant on in-memory text with every scanned loop a candidate
REF_API int ref_render_text(const char* text, const std::uint8_t* bits, std::size_t n, char* out, std::size_t cap) {
  return guarded([&] {
    CandidateSet cs;
    cs.unit = SourceUnit::from_string("<text>", text);
    cs.all_loops = scan_loops(cs.unit);
    for (const auto& l : cs.all_loops) cs.candidate_ids.push_back(l.id);
    return copy_out(render_variant(cs, genome_of(bits, n)), out, cap);
  });
}

// build_candidate_set (probe.cpp:187) over in-memory text with `compile_cmd` as the compiler (the reference's mockacc):
// the probe report (write_probe_report, one JSON object per loop) is copied out; returns the number of accepted
// loops, or the error class (NoCandidates = -9) with the report still filled in.
REF_API int ref_probe_text(const char* text, const char* basename, const char* compile_cmd, const char* workdir, char* report,
                           std::size_t cap) {
  namespace fs = std::filesystem;
  const fs::path report_file = fs::path(workdir) / "probe_report.jsonl";
  auto read_report = [&] {
    std::ifstream in(report_file, std::ios::binary);
    std::ostringstream ss;
    ss << in.rdbuf();
    copy_out(ss.str(), report, cap);
  };
  const int rc = guarded([&] {
    const SourceUnit unit = SourceUnit::from_string(basename, text);
    const std::vector<LoopSite> loops = scan_loops(unit);
    CompilerDriver driver;
    driver.compile_cmd = compile_cmd;
    driver.timeout_s = 30.0;
    ProbeOptions opt;
    opt.workdir = workdir;
    opt.report_file = report_file;
    const CandidateSet cs = build_candidate_set(unit, loops, driver, opt);
    return static_cast<int>(cs.candidate_ids.size());
  });
  read_report();
  return rc;
}

// cmd_tune / cmd_report: return the exit code, copy stdout / stderr text out
REF_API int ref_cmd_tune(const char* config_path, int has_seed, std::uint64_t seed, char* out, std::size_t out_cap, char* err,
                         std::size_t err_cap) {
  std::ostringstream o, e;
  TuneOptions opt;
  if (has_seed) opt.seed = seed;
  const int rc = cmd_tune(config_path, opt, o, e);
  copy_out(o.str(), out, out_cap);
  copy_out(e.str(), err, err_cap);
  return rc;
}

REF_API int ref_cmd_report(const char* workdir, char* out, std::size_t out_cap, char* err, std::size_t err_cap) {
  std::ostringstream o, e;
  const int rc = cmd_report(workdir, o, e);
  copy_out(o.str(), out, out_cap);
  copy_out(e.str(), err, err_cap);
  return rc;
}

REF_API const char* ref_status_name(int status) {
  static thread_local std::string s;
  s = std::string(to_string(static_cast<EvalStatus>(status)));
  return s.c_str();
}
