// commands.cpp -- cmd_tune / cmd_report / cmd_analyze.  Contract: /root/reference/proj/src/commands.cpp.
#include "mmxhost/commands.hpp"

#include <cstdio>
#include <filesystem>
#include <fstream>
#include <memory>
#include <ostream>
#include <sstream>
#include <vector>

#include "mmx.h"
#include "mmxhost/config.hpp"
#include "mmxhost/errors.hpp"
#include "mmxhost/evaluator.hpp"
#include "mmxhost/ga.hpp"
#include "mmxhost/json_lite.hpp"
#include "mmxhost/sim_model.hpp"
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

CandidateSet scan_source(const RunConfig& cfg) {
  CandidateSet cs;
  cs.unit = SourceUnit::from_file(cfg.source);
  cs.all_loops = scan_loops(cs.unit);
  for (const LoopSite& loop : cs.all_loops)
    if (cfg.candidates == CandidateFilter::All || loop.depth == 0) cs.candidate_ids.push_back(loop.id);
  return cs;
}

// The CUDA kernel library serves one catalogue: the 12 loops of the matrix application at their lines and depths.
void require_kernel_catalogue(const CandidateSet& cs, const RunConfig& cfg) {
  mmx_loop_info rows[MMX_GENE_LENGTH];
  const int count = mmx_loop_catalogue(rows, MMX_GENE_LENGTH);
  bool same = cfg.candidates == CandidateFilter::All && static_cast<int>(cs.all_loops.size()) == count;
  for (int k = 0; same && k < count; ++k)
    same = static_cast<int>(cs.all_loops[static_cast<std::size_t>(k)].line) == rows[k].line &&
           cs.all_loops[static_cast<std::size_t>(k)].depth == rows[k].depth;
  if (!same)
    throw ConfigError("the 'cuda' backend serves the loop catalogue of the matrix application (12 loops, all candidates); " +
                      cfg.source + " has " + std::to_string(cs.all_loops.size()) + " loops that do not match it");
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

bool parse_csv_row(const std::string& line, CsvRow& row) {
  std::vector<std::string> fields;
  std::string::size_type start = 0;
  for (;;) {
    const auto comma = line.find(',', start);
    fields.push_back(line.substr(start, comma == std::string::npos ? comma : comma - start));
    if (comma == std::string::npos) break;
    start = comma + 1;
  }
  if (fields.size() != 7) return false;
  try {
    std::size_t used = 0;
    row.generation = std::stoi(fields[0], &used);
    if (used != fields[0].size()) return false;
    row.best_time_s = std::stod(fields[1], &used);
    if (used != fields[1].size()) return false;
    row.best_speedup = std::stod(fields[2], &used);
    if (used != fields[2].size()) return false;
  } catch (const std::exception&) {
    return false;
  }
  row.best_genome = fields[3];
  return !row.best_genome.empty() && row.best_genome.find_first_not_of("01") == std::string::npos;
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
    const CandidateSet cs = scan_source(cfg);
    if (cfg.cuda) require_kernel_catalogue(cs, cfg);
    mmx_loop_info rows[MMX_GENE_LENGTH];
    const int count = cfg.cuda ? mmx_loop_catalogue(rows, MMX_GENE_LENGTH) : 0;
    out << "source: " << cfg.source << "\n";
    out << "loops: " << cs.all_loops.size() << "\n";
    for (const LoopSite& loop : cs.all_loops) {
      out << "  loop " << loop.id << ": line " << loop.line << ", depth " << loop.depth;
      const bool selected = cfg.candidates == CandidateFilter::All || loop.depth == 0;
      out << (selected ? " -> candidate" : " -> parallelizable, filtered out");
      if (loop.id < count) out << " [kernel: " << rows[loop.id].kernel << "]";
      out << "\n";
    }
    out << "candidates: " << cs.candidate_ids.size() << " (filter: " << to_string(cfg.candidates) << ")\n";
    out << "gene length: " << cs.candidate_ids.size() << "\n";
    if (cs.candidate_ids.empty()) out << "nothing to tune: every loop was rejected or filtered out\n";
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

    const CandidateSet cs = scan_source(cfg);
    if (cs.candidate_ids.empty()) throw NoCandidates("no candidate loops in " + cfg.source);
    std::unique_ptr<Evaluator> evaluator;
    if (cfg.sim_model) {
      CostModel model = load_model(*cfg.sim_model);
      if (model.gene_length() != cs.gene_length())
        throw ConfigError("sim model has " + std::to_string(model.gene_length()) + " loops but the source has " +
                          std::to_string(cs.gene_length()) + " candidates");
      evaluator = std::make_unique<Evaluator>(std::make_unique<SimBackend>(std::move(model)), cfg.jobs, cfg.eval_cache_path());
    } else {
      require_kernel_catalogue(cs, cfg);
      // worker s of a batch is pinned to device slot s; `jobs` is implied by the device list
      evaluator = std::make_unique<MultiGpuEvaluator>(std::make_unique<CudaBackend>(*cfg.cuda), cfg.eval_cache_path());
    }
    out << "candidates: " << cs.gene_length() << " of " << cs.all_loops.size() << " loops\n";

    const TuningResult result = run_ga(cs.gene_length(), cfg.ga, *evaluator);
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
