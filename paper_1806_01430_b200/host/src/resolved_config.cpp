// resolved_config.cpp -- config.resolved.json: the provenance record every command writes first
// (format: /root/reference/proj/src/config.cpp:154-183, byte-pinned by tests/golden/tune_sim/runs.json).
#include "mmxhost/config.hpp"

#include <sstream>
#include <string>

#include "mmxhost/json_lite.hpp"

namespace mmxhost {
namespace {

// ---- writer: nlohmann's dump(2) layout for the handful of shapes used here ----------------------------
struct Out {
  std::string s;
  int indent = 0;
  bool first = true;
  void open() { s += "{"; indent += 2; first = true; }
  void key(const std::string& k) {
    s += first ? "\n" : ",\n";
    first = false;
    s += std::string(static_cast<std::size_t>(indent), ' ') + json::dump_string(k) + ": ";
  }
  void close() {
    indent -= 2;
    s += first ? "}" : "\n" + std::string(static_cast<std::size_t>(indent), ' ') + "}";
    first = false;
  }
  void str(const std::string& k, const std::string& v) { key(k); s += json::dump_string(v); }
  void integer(const std::string& k, long long v) { key(k); s += std::to_string(v); }
  void uinteger(const std::string& k, unsigned long long v) { key(k); s += std::to_string(v); }
  void number(const std::string& k, double v) { key(k); s += json::dump_number(v); }
};

}  // namespace

std::string render_resolved_config(const RunConfig& cfg) {
  Out o;
  o.open();
  o.str("source", cfg.source);
  o.str("workdir", cfg.workdir);
  o.str("candidates", std::string(to_string(cfg.candidates)));
  o.integer("jobs", cfg.jobs);
  o.key("ga");
  o.open();
  o.integer("population", cfg.ga.population);
  o.integer("generations", cfg.ga.generations);
  o.number("crossover_rate", cfg.ga.crossover_rate);
  o.number("mutation_rate", cfg.ga.mutation_rate);
  o.uinteger("seed", cfg.ga.seed);
  o.integer("elite_count", cfg.ga.elite_count);
  o.close();
  if (cfg.cuda) {
    const CudaBackendConfig& c = *cfg.cuda;
    o.key("cuda");
    o.open();
    o.integer("n", c.n);
    o.str("dtype", c.dtype == MMX_F64 ? "f64" : "f32");
    o.str("numerics", c.numerics == MMX_NUMERICS_FAST ? "fast" : "strict");
    o.number("timeout_s", c.timeout_s);
    o.integer("repetitions", c.repetitions);
    o.integer("warmup", c.warmup);
    o.integer("host_threads", c.host_threads);
    o.key("devices");
    o.s += "[";
    for (std::size_t i = 0; i < c.devices.size(); ++i) {
      o.s += (i ? ",\n" : "\n") + std::string(static_cast<std::size_t>(o.indent + 2), ' ') + std::to_string(c.devices[i]);
    }
    o.s += "\n" + std::string(static_cast<std::size_t>(o.indent), ' ') + "]";
    o.integer("matmul_variant", c.matmul_variant);
    o.integer("pin_host", c.pin_host ? 1 : 0);
    o.integer("host_core_first", c.host_core_first);
    o.integer("host_core_count", c.host_core_count);
    o.integer("early_timeout", c.early_timeout ? 1 : 0);
    o.close();
  } else {
    o.str("sim_model", *cfg.sim_model);
  }
  o.key("artifacts");
  o.open();
  o.str("resolved_config", cfg.resolved_config_path());
  o.str("probe_report", cfg.probe_report_path());
  o.str("probe_cache", cfg.probe_cache_path());
  o.str("eval_cache", cfg.eval_cache_path());
  o.str("generations_csv", cfg.generations_csv_path());
  o.str("summary", cfg.summary_path());
  o.str("best_source", cfg.best_source_path());
  o.close();
  o.close();
  return o.s + "\n";
}

}  // namespace mmxhost
