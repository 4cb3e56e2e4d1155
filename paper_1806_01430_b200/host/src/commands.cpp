// commands.cpp -- cmd_tune / cmd_report / cmd_analyze.  Contract: /root/reference/proj/src/commands.cpp.
#include "mmxhost/commands.hpp"

#include <algorithm>
#include <cerrno>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <memory>
#include <ostream>
#include <sstream>
#include <vector>

#include "mmx.h"
#include "mmxhost/calibrate.hpp"
#include "mmxhost/config.hpp"
#include "mmxhost/errors.hpp"
#include "mmxhost/evaluator.hpp"
#include "mmxhost/feasibility.hpp"
#include "mmxhost/ga.hpp"
#include "mmxhost/json_lite.hpp"
#include "mmxhost/kernel_match.hpp"
#include "mmxhost/cost_model.hpp"
#include "mmxhost/source_model.hpp"

namespace fs = std::filesystem;

namespace mmxhost {
namespace {

std::string fmt_s(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.6g", v);
  return buf;
}

void ensure_workdir(const std::string& dir) {
  std::error_code ec;
  fs::create_directories(dir, ec);
  if (ec || !fs::is_directory(dir)) throw WorkdirUnwritable("cannot create workdir: " + dir);
  const fs::path canary = fs::path(dir) / ".mmx_write_test";
  std::ofstream probe(canary);
  if (!probe) throw WorkdirUnwritable("workdir is not writable: " + dir);
  probe.close();
  fs::remove(canary, ec);
}

void write_text_file(const std::string& path, const std::string& text) {
  const fs::path p(path);
  if (p.has_parent_path()) {
    std::error_code ec;
    fs::create_directories(p.parent_path(), ec);
  }
  std::ofstream out(p, std::ios::binary);
  if (!out) throw WorkdirUnwritable("cannot write " + path);
  out << text;
  if (!out) throw WorkdirUnwritable("short write to " + path);
}

bool keep_candidate(const LoopSite& loop, CandidateFilter filter) { return filter == CandidateFilter::All || loop.depth == 0; }

// What `analyze` prints and `tune` searches over: the scanned loops, one probe verdict per loop, the candidate set, and
// (cuda backend) the kernel each loop is served by.
struct Inventory {
  CandidateSet cs;
  std::vector<ProbeResult> probes;
  std::vector<KernelBinding> kernels;  // empty for sim runs
};

// The CUDA kernel library serves the loops whose idiom it has a kernel for (kernel_match.hpp); today that is the catalogue
// of the matrix application, and the executor is wired to exactly those 12 genes (mmx_loop_catalogue).  The catalogue is
// DERIVED from the source and must equal the served one row for row.
void require_kernel_catalogue(const Inventory& inv, const RunConfig& cfg) {
  mmx_loop_info rows[MMX_GENE_LENGTH];
  const int count = mmx_loop_catalogue(rows, MMX_GENE_LENGTH);
  for (const KernelBinding& b : inv.kernels)
    if (b.kernel.empty())
      throw ConfigError("the 'cuda' backend has no kernel for loop " + std::to_string(b.loop_id) + " of " + cfg.source + " (line " +
                        std::to_string(b.line) + "): " + b.why_unmatched);
  bool same = cfg.candidates == CandidateFilter::All && static_cast<int>(inv.kernels.size()) == count &&
              inv.cs.candidate_ids.size() == inv.kernels.size();
  for (int k = 0; same && k < count; ++k) {
    const KernelBinding& b = inv.kernels[static_cast<std::size_t>(k)];
    same = b.loop_id == rows[k].gene && static_cast<int>(b.line) == rows[k].line && b.depth == rows[k].depth && b.nest == rows[k].nest &&
           b.header.var == rows[k].induction && b.kernel == rows[k].kernel;
  }
  if (!same)
    throw ConfigError("the 'cuda' backend serves the loop catalogue of the matrix application (12 loops, all candidates); " +
                      cfg.source + " has " + std::to_string(inv.cs.all_loops.size()) + " loops that do not match it");
}

// Sim runs have nothing to probe with: every loop that passes the filter is a candidate and the report says so
// (/root/reference/proj/src/commands.cpp:78-106).  With the cuda backend the verdicts come from the static rules
// (feasibility.hpp) -- the compiler probe of commands.cpp:108-127 without a compiler -- and the kernel matcher.
Inventory take_inventory(const RunConfig& cfg) {
  Inventory inv;
  const SourceUnit unit = SourceUnit::from_file(cfg.source);
  const std::vector<LoopSite> loops = scan_loops(unit);
  if (cfg.cuda) {
    try {
      inv.cs = build_candidate_set(unit, loops, &inv.probes);
    } catch (const NoCandidates&) {
      write_text_file(cfg.probe_report_path(), probe_report_jsonl(unit, loops, inv.probes));
      throw;
    }
    write_text_file(cfg.probe_report_path(), probe_report_jsonl(unit, loops, inv.probes));
    if (cfg.candidates == CandidateFilter::Outermost) {
      std::erase_if(inv.cs.candidate_ids, [&](int id) { return inv.cs.all_loops[static_cast<std::size_t>(id)].depth != 0; });
      if (inv.cs.candidate_ids.empty()) throw NoCandidates("no outermost candidate loops in " + cfg.source);
    }
    inv.kernels = match_kernels(unit, loops);
    return inv;
  }
  for (const LoopSite& loop : loops) {
    ProbeResult r;
    r.loop_id = loop.id;
    r.verdict = ProbeVerdict::Parallelizable;
    r.compiler_message = "probe skipped: timings come from a sim model";
    inv.probes.push_back(std::move(r));
  }
  write_text_file(cfg.probe_report_path(), probe_report_jsonl(unit, loops, inv.probes));
  inv.cs.unit = unit;
  inv.cs.all_loops = loops;
  for (const LoopSite& loop : loops)
    if (keep_candidate(loop, cfg.candidates)) inv.cs.candidate_ids.push_back(loop.id);
  if (inv.cs.candidate_ids.empty()) throw NoCandidates("no candidate loops in " + cfg.source);
  return inv;
}

// commands.cpp:129-155 of the reference, plus the kernel column
void print_inventory(std::ostream& out, const RunConfig& cfg, const Inventory& inv) {
  out << "source: " << cfg.source << "\n";
  out << "loops: " << inv.cs.all_loops.size() << "\n";
  for (const LoopSite& loop : inv.cs.all_loops) {
    out << "  loop " << loop.id << ": line " << loop.line << ", depth " << loop.depth;
    const auto r = std::find_if(inv.probes.begin(), inv.probes.end(), [&](const ProbeResult& x) { return x.loop_id == loop.id; });
    const bool selected = std::find(inv.cs.candidate_ids.begin(), inv.cs.candidate_ids.end(), loop.id) != inv.cs.candidate_ids.end();
    if (r == inv.probes.end()) {
      out << " -> not probed";
    } else if (r->verdict == ProbeVerdict::Parallelizable) {
      out << (selected ? " -> candidate" : " -> parallelizable, filtered out");
    } else {
      const std::string msg = r->compiler_message.substr(0, r->compiler_message.find('\n'));
      out << " -> rejected [" << to_string(r->reject_class) << "]";
      if (!msg.empty()) out << " " << msg;
    }
    const auto k = std::find_if(inv.kernels.begin(), inv.kernels.end(), [&](const KernelBinding& x) { return x.loop_id == loop.id; });
    if (k != inv.kernels.end()) out << (k->kernel.empty() ? " [no kernel: " + k->why_unmatched + "]" : " [kernel: " + k->kernel + "]");
    out << "\n";
  }
  out << "candidates: " << inv.cs.candidate_ids.size() << " (filter: " << to_string(cfg.candidates) << ")\n";
  out << "gene length: " << inv.cs.candidate_ids.size() << "\n";
  out << "probe report: " << cfg.probe_report_path() << "\n";
}

std::string render_summary_json(const TuningResult& result, const EvalCounters& counters) {
  std::string s = "{\n";
  s += "  \"baseline_s\": " + json::dump_number(result.baseline_s) + ",\n";
  s += "  \"best_s\": " + json::dump_number(result.best_time_s) + ",\n";
  s += "  \"speedup\": " + json::dump_number(result.baseline_s / result.best_time_s) + ",\n";
  s += "  \"best_genome\": " + json::dump_string(result.best_genome.to_string()) + ",\n";
  s += "  \"distinct_evals\": " + std::to_string(counters.distinct) + ",\n";
  s += "  \"elapsed_s\": " + json::dump_number(counters.elapsed_s) + "\n";
  return s + "}\n";
}

struct CsvRow {
  int generation = 0;
  double best_time_s = 0.0, best_speedup = 0.0;
  std::string best_genome;
};

// C-library number parsing with the acceptance rules of std::stoi / std::stod (leading blanks, signs; the whole cell must be
// consumed; out-of-range values are refused), without exceptions
bool cell_to_double(const std::string& cell, double& value) {
  if (cell.empty()) return false;
  errno = 0;
  char* stop = nullptr;
  value = std::strtod(cell.c_str(), &stop);
  return stop == cell.c_str() + cell.size() && errno != ERANGE;
}

bool cell_to_int(const std::string& cell, int& value) {
  if (cell.empty()) return false;
  errno = 0;
  char* stop = nullptr;
  const long wide = std::strtol(cell.c_str(), &stop, 10);
  if (stop != cell.c_str() + cell.size() || errno == ERANGE || wide < INT_MIN || wide > INT_MAX) return false;
  value = static_cast<int>(wide);
  return true;
}

// One data row of generations.csv: generation,best_time_s,best_speedup,best_genome,mean_fitness,distinct_evals,cache_hits.  The report
// needs the first four columns; a row with any other number of cells, or a genome cell that is not a bit string, is malformed.
bool parse_csv_row(const std::string& line, CsvRow& row) {
  constexpr int kColumns = 7;
  std::string cell[kColumns];
  int filled = 0;
  std::istringstream cells(line);
  for (std::string piece; std::getline(cells, piece, ',');) {
    if (filled == kColumns) return false;
    cell[filled++] = std::move(piece);
  }
  if (!line.empty() && line.back() == ',') {  // getline drops a trailing empty cell
    if (filled == kColumns) return false;
    ++filled;
  }
  if (filled != kColumns) return false;
  if (!cell_to_int(cell[0], row.generation) || !cell_to_double(cell[1], row.best_time_s) || !cell_to_double(cell[2], row.best_speedup)) return false;
  const bool bits_only = std::all_of(cell[3].begin(), cell[3].end(), [](char ch) { return ch == '0' || ch == '1'; });
  if (cell[3].empty() || !bits_only) return false;
  row.best_genome = cell[3];
  return true;
}

}  // namespace

int exit_code_for(const std::exception& e) {
  if (dynamic_cast<const ZeroTotalFitness*>(&e)) return 5;
  if (dynamic_cast<const ToolchainMissing*>(&e)) return 4;
  if (dynamic_cast<const EvaluatorUnavailable*>(&e)) return 4;
  if (dynamic_cast<const ScanError*>(&e)) return 3;
  if (dynamic_cast<const NoCandidates*>(&e)) return 3;
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const ModelError*>(&e)) return 2;
  if (dynamic_cast<const MissingLog*>(&e)) return 2;
  if (dynamic_cast<const WorkdirUnwritable*>(&e)) return 2;
  return 1;
}

int cmd_analyze(const std::string& config_path, std::ostream& out, std::ostream& err) {
  try {
    const RunConfig cfg = load_config(config_path);
    ensure_workdir(cfg.workdir);
    write_text_file(cfg.resolved_config_path(), render_resolved_config(cfg));
    Inventory inv;
    try {
      inv = take_inventory(cfg);
    } catch (const NoCandidates&) {
      // analyze still reports: rerun the scan for the listing (the probe report is already on disk)
      const SourceUnit unit = SourceUnit::from_file(cfg.source);
      inv.cs.unit = unit;
      inv.cs.all_loops = scan_loops(unit);
      if (cfg.cuda) {
        const FeasibilityAnalyzer an(unit, inv.cs.all_loops);
        for (const LoopSite& l : inv.cs.all_loops) inv.probes.push_back(an.probe(l.id));
        inv.kernels = match_kernels(unit, inv.cs.all_loops);
      }
      print_inventory(out, cfg, inv);
      out << "nothing to tune: every loop was rejected or filtered out\n";
      return 0;
    }
    print_inventory(out, cfg, inv);
    return 0;
  } catch (const std::exception& e) {
    err << "analyze: " << e.what() << "\n";
    return exit_code_for(e);
  }
}

int cmd_tune(const std::string& config_path, const TuneOptions& options, std::ostream& out, std::ostream& err) {
  try {
    RunConfig cfg = load_config(config_path);
    if (options.seed) cfg.ga.seed = *options.seed;
    if (options.sim_model) {
      cfg.sim_model = fs::absolute(*options.sim_model).lexically_normal().string();
      cfg.cuda.reset();
    }
    ensure_workdir(cfg.workdir);
    write_text_file(cfg.resolved_config_path(), render_resolved_config(cfg));

    const Inventory inv = take_inventory(cfg);
    const CandidateSet& cs = inv.cs;
    std::unique_ptr<Evaluator> evaluator;
    if (cfg.sim_model) {
      CostModel model = load_model(*cfg.sim_model);
      if (model.gene_length() != cs.gene_length())
        throw ConfigError("sim model has " + std::to_string(model.gene_length()) + " loops but the source has " +
                          std::to_string(cs.gene_length()) + " candidates");
      evaluator = std::make_unique<Evaluator>(std::make_unique<SimBackend>(std::move(model)), cfg.jobs, cfg.eval_cache_path());
    } else {
      require_kernel_catalogue(inv, cfg);
      // worker s of a batch is pinned to device slot s; `jobs` is implied by the device list
      evaluator = std::make_unique<MultiGpuEvaluator>(std::make_unique<CudaBackend>(*cfg.cuda), cfg.eval_cache_path());
    }
    out << "candidates: " << cs.gene_length() << " of " << cs.all_loops.size() << " loops\n";

    const TuningResult result = run_ga(cs, cfg.ga, *evaluator);
    const EvalCounters counters = evaluator->counters();
    {
      std::ofstream csv(cfg.generations_csv_path(), std::ios::binary);
      if (!csv) throw WorkdirUnwritable("cannot write " + cfg.generations_csv_path());
      write_generation_csv(csv, result);
    }
    write_text_file(cfg.summary_path(), render_summary_json(result, counters));
    write_text_file(cfg.best_source_path(), render_variant(cs, result.best_genome));

    out << "baseline: " << fmt_s(result.baseline_s) << " s\n";
    out << "best:     " << fmt_s(result.best_time_s) << " s (speedup " << fmt_s(result.baseline_s / result.best_time_s) << ")\n";
    out << "genome:   " << result.best_genome.to_string() << "\n";
    out << "evaluations: " << counters.distinct << " distinct, " << counters.cache_hits << " cache hits, " << counters.backend_calls
        << " backend calls\n";
    out << "workdir: " << cfg.workdir << "\n";
    return 0;
  } catch (const std::exception& e) {
    err << "tune: " << e.what() << "\n";
    return exit_code_for(e);
  }
}

int cmd_calibrate(const std::string& config_path, std::ostream& out, std::ostream& err) {
  try {
    const RunConfig cfg = load_config(config_path);
    if (!cfg.cuda) throw ConfigError("calibrate needs a 'cuda' block: there is nothing to measure on the sim backend");
    ensure_workdir(cfg.workdir);
    write_text_file(cfg.resolved_config_path(), render_resolved_config(cfg));
    const Inventory inv = take_inventory(cfg);
    require_kernel_catalogue(inv, cfg);
    MultiGpuEvaluator evaluator(std::make_unique<CudaBackend>(*cfg.cuda), cfg.eval_cache_path());

    // every genome the static rules accept (648 of 4096 for the matrix application)
    const std::size_t a = inv.cs.gene_length();
    const FeasibilityAnalyzer analyzer(inv.cs.unit, inv.cs.all_loops);
    std::vector<Genome> genomes;
    for (std::uint64_t mask = 0; mask < (std::uint64_t{1} << a); ++mask) {
      std::vector<int> annotated;
      std::vector<std::uint8_t> bits(a);
      for (std::size_t k = 0; k < a; ++k)
        if ((mask >> k) & 1u) {
          bits[k] = 1;
          annotated.push_back(inv.cs.candidate_ids[k]);
        }
      if (analyzer.check(annotated).empty()) genomes.emplace_back(std::move(bits));
    }
    const std::vector<EvaluationOutcome> outcomes = evaluator.evaluate_all(genomes);
    std::vector<GenomeSample> samples;
    std::size_t timeouts = 0;
    const GenomeSample* fastest = nullptr;
    for (std::size_t k = 0; k < genomes.size(); ++k) {
      if (outcomes[k].status == EvalStatus::Timeout) ++timeouts;
      if (outcomes[k].status != EvalStatus::Measured) continue;  // a timed-out run says only "slower than the budget"
      samples.push_back({genomes[k], outcomes[k].time_s});
    }
    for (const GenomeSample& s : samples)
      if (!fastest || s.time_s < fastest->time_s) fastest = &s;
    FitReport fit;
    const PlanModel plan = fit_plan_model(samples, cfg.cuda->n, cfg.cuda->dtype, &fit);
    ProjectionReport proj;
    const CostModel model = project_to_cost_model(plan, &proj);
    const std::string model_path = cfg.workdir + "/calibrated_model.json";
    write_text_file(model_path, dump_cost_model_json(model));

    std::string r = "{\n";
    r += "  \"n\": " + std::to_string(cfg.cuda->n) + ",\n";
    r += "  \"feasible_genomes\": " + std::to_string(genomes.size()) + ",\n";
    r += "  \"measured\": " + std::to_string(samples.size()) + ",\n";
    r += "  \"timeouts\": " + std::to_string(timeouts) + ",\n";
    r += "  \"measured_best_genome\": " + json::dump_string(fastest->genome.to_string()) + ",\n";
    r += "  \"measured_best_s\": " + json::dump_number(fastest->time_s) + ",\n";
    r += "  \"plan_best_genome\": " + json::dump_string(proj.plan_best.to_string()) + ",\n";
    r += "  \"plan_best_s\": " + json::dump_number(proj.plan_best_s) + ",\n";
    r += "  \"cost_best_genome\": " + json::dump_string(proj.cost_best.to_string()) + ",\n";
    r += "  \"cost_best_s\": " + json::dump_number(proj.cost_best_s) + ",\n";
    r += "  \"fit_rms_rel_err\": " + json::dump_number(fit.rms_rel_err) + ",\n";
    r += "  \"fit_max_rel_err\": " + json::dump_number(fit.max_rel_err) + ",\n";
    r += "  \"projection_rms_rel_err\": " + json::dump_number(proj.rms_rel_err) + ",\n";
    r += "  \"projection_max_rel_err\": " + json::dump_number(proj.max_rel_err) + ",\n";
    r += "  \"inexact_loops\": [";
    for (std::size_t k = 0; k < proj.inexact_loops.size(); ++k) r += (k ? ", " : "") + std::to_string(proj.inexact_loops[k]);
    r += "]\n}\n";
    write_text_file(cfg.workdir + "/calibration.json", r);

    out << "genomes:  " << genomes.size() << " feasible, " << samples.size() << " measured, " << timeouts << " over budget\n";
    out << "measured: " << fastest->genome.to_string() << " " << fmt_s(fastest->time_s) << " s\n";
    out << "model:    " << proj.cost_best.to_string() << " " << fmt_s(proj.cost_best_s) << " s (fit rms " << fmt_s(fit.rms_rel_err)
        << ", max " << fmt_s(fit.max_rel_err) << "; " << proj.inexact_loops.size() << " loops not representable additively)\n";
    out << "model file: " << model_path << "\n";
    return 0;
  } catch (const std::exception& e) {
    err << "calibrate: " << e.what() << "\n";
    return exit_code_for(e);
  }
}

int cmd_report(const std::string& workdir, std::ostream& out, std::ostream& err) {
  try {
    const std::string csv_path = workdir + "/generations.csv", summary_path = workdir + "/summary.json";
    std::ifstream csv(csv_path);
    if (!csv) throw MissingLog("no generations.csv in " + workdir);
    std::string header;
    if (!std::getline(csv, header) || header != "generation,best_time_s,best_speedup,best_genome,mean_fitness,distinct_evals,cache_hits") {
      err << "report: corrupted log: unexpected header in " << csv_path << "\n";
      return 1;
    }
    std::vector<CsvRow> rows;
    std::string line;
    while (std::getline(csv, line)) {
      if (line.empty()) continue;
      CsvRow row;
      if (!parse_csv_row(line, row)) {
        err << "report: corrupted log: bad row '" << line << "'\n";
        return 1;
      }
      rows.push_back(std::move(row));
    }
    if (rows.empty()) {
      err << "report: corrupted log: no generation rows in " << csv_path << "\n";
      return 1;
    }
    out << "generation  best_time_s   speedup     genome\n";
    char buf[128];
    for (const CsvRow& row : rows) {
      std::snprintf(buf, sizeof(buf), "%10d  %-12.9g  %-10.6g  %s\n", row.generation, row.best_time_s, row.best_speedup,
                    row.best_genome.c_str());
      out << buf;
    }
    for (std::size_t i = 1; i < rows.size(); ++i)
      if (rows[i].best_time_s > rows[i - 1].best_time_s) {
        err << "report: corrupted log: best time regresses at generation " << rows[i].generation << " (" << rows[i - 1].best_time_s
            << " -> " << rows[i].best_time_s << ")\n";
        return 1;
      }
    std::ifstream summary_in(summary_path);
    if (!summary_in) throw MissingLog("no summary.json in " + workdir);
    std::ostringstream ss;
    ss << summary_in.rdbuf();
    json::Value summary;
    if (!json::parse(ss.str(), summary) || !summary.is_object()) {
      err << "report: corrupted log: " << summary_path << ": not a JSON object\n";
      return 1;
    }
    const json::Value *b = summary.find("baseline_s"), *t = summary.find("best_s"), *sp = summary.find("speedup"),
                      *g = summary.find("best_genome");
    if (!b || !t || !sp || !g || !b->is_number() || !t->is_number() || !sp->is_number() || !g->is_string()) {
      err << "report: corrupted log: summary.json is missing keys\n";
      return 1;
    }
    out << "baseline " << fmt_s(b->number) << " s -> best " << fmt_s(t->number) << " s, speedup " << fmt_s(sp->number) << ", genome "
        << g->string << "\n";
    return 0;
  } catch (const std::exception& e) {
    err << "report: " << e.what() << "\n";
    return exit_code_for(e);
  }
}

}  // namespace mmxhost
