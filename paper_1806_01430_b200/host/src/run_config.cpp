// run_config.cpp -- load_config / render_resolved_config.  Contract: /root/reference/proj/src/config.cpp:29-185.
#include "mmxhost/config.hpp"

#include <algorithm>
#include <filesystem>
#include <fstream>
#include <initializer_list>
#include <limits>
#include <sstream>
#include <vector>

#include "mmxhost/errors.hpp"
#include "mmxhost/json_lite.hpp"

namespace mmxhost {

namespace fs = std::filesystem;

std::string_view to_string(CandidateFilter f) { return f == CandidateFilter::All ? "all" : "outermost"; }

std::string RunConfig::best_source_path() const {
  std::string name = fs::path(source).filename().string();
  if (name.empty()) name = "variant.c";
  return workdir + "/best/" + name;
}

namespace {

using json::Value;

// One JSON object being read: every accessor marks its key as consumed, and done() rejects whatever the reader never
// asked for -- the unknown-key check cannot drift from the keys actually parsed.  Messages follow the reference's
// (/root/reference/proj/src/config.cpp:29-152), which tests/test_host_tune.py pins by substring.
class Section {
 public:
  Section(const Value& obj, std::string where) : obj_(obj), where_(std::move(where)) {}

  const Value* peek(const char* key) {
    seen_.emplace_back(key);
    return obj_.find(key);
  }
  bool has(const char* key) { return peek(key) != nullptr; }

  std::string text(const char* key) {  // required, non-empty
    const Value* v = peek(key);
    if (v == nullptr) throw ConfigError(where_ + " needs a '" + key + "' entry");
    if (!v->is_string() || v->string.empty()) throw ConfigError(quoted(key) + " must be a non-empty string");
    return v->string;
  }
  // one of `names`, by position; absent -> fallback
  int choice(const char* key, std::initializer_list<const char*> names, int fallback) {
    if (!has(key)) return fallback;
    const std::string got = text(key);
    int at = 0;
    std::string menu;
    for (const char* n : names) {
      if (got == n) return at;
      menu += std::string(at ? " or " : "") + "\"" + n + "\"";
      ++at;
    }
    throw ConfigError("'" + std::string(key) + "' must be " + menu + ", got \"" + got + "\"");
  }
  double real(const char* key, double fallback) {
    const Value* v = peek(key);
    if (v == nullptr) return fallback;
    if (!v->is_number()) throw ConfigError(quoted(key) + " must be a number");
    return v->number;
  }
  int integer(const char* key, int fallback) {
    const Value* v = peek(key);
    if (v == nullptr) return fallback;
    if (!v->is_number() || !v->is_integer || v->number < std::numeric_limits<int>::min() || v->number > std::numeric_limits<int>::max())
      throw ConfigError(quoted(key) + " must be an integer");
    return static_cast<int>(v->number);
  }
  const Value* object(const char* key) {
    const Value* v = peek(key);
    if (v != nullptr && !v->is_object()) throw ConfigError("'" + std::string(key) + "' must be an object");
    return v;
  }
  void done() const {
    for (const auto& kv : *obj_.object)
      if (std::find(seen_.begin(), seen_.end(), kv.first) == seen_.end()) throw ConfigError("unknown key '" + kv.first + "' in " + where_);
  }

 private:
  std::string quoted(const char* key) const { return "'" + std::string(key) + "' in " + where_; }
  const Value& obj_;
  std::string where_;
  std::vector<std::string> seen_;
};

std::string resolve_path(const fs::path& base, const std::string& p) {
  const fs::path path(p);
  return (path.is_absolute() ? path : base / path).lexically_normal().string();
}

GAParams read_ga(const Value& obj) {
  Section s(obj, "'ga'");
  GAParams ga;
  ga.population = s.integer("population", ga.population);
  ga.generations = s.integer("generations", ga.generations);
  ga.crossover_rate = s.real("crossover_rate", ga.crossover_rate);
  ga.mutation_rate = s.real("mutation_rate", ga.mutation_rate);
  ga.elite_count = s.integer("elite_count", ga.elite_count);
  if (const Value* seed = s.peek("seed")) {
    if (!seed->is_number() || !seed->is_integer || seed->number < 0) throw ConfigError("'seed' in 'ga' must be a non-negative integer");
    ga.seed = static_cast<std::uint64_t>(seed->number);
  }
  s.done();
  return ga;
}

CudaBackendConfig read_cuda(const Value& obj) {
  Section s(obj, "'cuda'");
  CudaBackendConfig c;
  auto at_least = [](int v, int lo, const char* key, const char* what) {
    if (v < lo) throw ConfigError("'" + std::string(key) + "' " + what);
    return v;
  };
  c.n = at_least(s.integer("n", c.n), 1, "n", "must be at least 1");
  c.dtype = s.choice("dtype", {"f64", "f32"}, c.dtype == MMX_F64 ? 0 : 1) == 0 ? MMX_F64 : MMX_F32;
  c.numerics = s.choice("numerics", {"fast", "strict"}, c.numerics == MMX_NUMERICS_FAST ? 0 : 1) == 0 ? MMX_NUMERICS_FAST : MMX_NUMERICS_STRICT;
  c.timeout_s = s.real("timeout_s", c.timeout_s);
  if (!(c.timeout_s > 0.0)) throw ConfigError("'timeout_s' must be positive");
  c.repetitions = at_least(s.integer("repetitions", c.repetitions), 1, "repetitions", "must be at least 1");
  c.warmup = at_least(s.integer("warmup", c.warmup), 0, "warmup", "must not be negative");
  c.host_threads = at_least(s.integer("host_threads", c.host_threads), 1, "host_threads", "must be at least 1");
  c.matmul_variant = s.integer("matmul_variant", c.matmul_variant);
  c.pin_host = s.integer("pin_host", c.pin_host ? 1 : 0) != 0;
  c.host_core_first = at_least(s.integer("host_core_first", c.host_core_first), 0, "host_core_first", "must not be negative");
  c.host_core_count = at_least(s.integer("host_core_count", c.host_core_count), 0, "host_core_count", "must not be negative");
  c.early_timeout = s.integer("early_timeout", c.early_timeout ? 1 : 0) != 0;
  if (const Value* d = s.peek("devices")) {
    if (!d->is_array() || d->array->empty()) throw ConfigError("'devices' in 'cuda' must be a non-empty array of device ordinals");
    c.devices.clear();
    for (const Value& e : *d->array) {
      if (!e.is_number() || !e.is_integer || e.number < 0) throw ConfigError("'devices' in 'cuda' must hold non-negative integers");
      c.devices.push_back(static_cast<int>(e.number));
    }
  }
  s.done();
  return c;
}

}  // namespace

RunConfig load_config(const std::string& config_path) {
  std::ifstream in(config_path, std::ios::binary);
  if (!in) throw ConfigError("cannot read config file: " + config_path);
  std::ostringstream ss;
  ss << in.rdbuf();
  Value obj;
  if (!json::parse(ss.str(), obj) || !obj.is_object()) throw ConfigError("config file is not a JSON object: " + config_path);
  Section top(obj, "the config");
  const fs::path base = fs::absolute(config_path).parent_path();

  // the three backends first: exactly one of the two this build has
  if (top.has("toolchain"))
    throw ConfigError("the 'toolchain' backend (external OpenACC compiler + benchmark binary) is not part of this build: "
                      "configure 'cuda' (in-process sm_100a executor) or 'sim_model'");
  const Value* cuda = top.object("cuda");
  const bool has_sim = top.has("sim_model");
  RunConfig cfg;
  cfg.jobs = top.integer("jobs", 1);
  if (const Value* ga = top.object("ga")) cfg.ga = read_ga(*ga);
  cfg.candidates = top.choice("candidates", {"all", "outermost"}, 0) == 0 ? CandidateFilter::All : CandidateFilter::Outermost;
  top.peek("source");
  top.peek("workdir");
  top.done();  // typos are reported before anything else

  cfg.source = resolve_path(base, top.text("source"));
  cfg.workdir = resolve_path(base, top.text("workdir"));
  if (cfg.jobs < 1) throw ConfigError("'jobs' must be at least 1");
  validate_params(cfg.ga);
  if (has_sim == (cuda != nullptr)) throw ConfigError("exactly one of 'cuda' and 'sim_model' must be configured");
  if (cuda != nullptr) cfg.cuda = read_cuda(*cuda);
  else cfg.sim_model = resolve_path(base, top.text("sim_model"));
  return cfg;
}

}  // namespace mmxhost
