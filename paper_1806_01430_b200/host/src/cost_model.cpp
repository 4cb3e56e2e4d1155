#include "mmxhost/cost_model.hpp"

#include <cstdint>
#include <fstream>
#include <random>
#include <sstream>

#include "mmxhost/errors.hpp"
#include "mmxhost/json_lite.hpp"

namespace mmxhost {

namespace {

// The model sum for an arbitrary bit predicate; shared by model_time, the validator and the
// brute-force search so all three add in the same order.
template <typename BitAt>
double summed_time(const CostModel& m, BitAt bit_at) {
  double t = m.serial_s;
  for (std::size_t k = 0; k < m.loops.size(); ++k) {
    const LoopCost& lc = m.loops[k];
    if (bit_at(k)) t += lc.compute_s / lc.speedup + lc.transfer_s;
    else t += lc.compute_s;
  }
  for (const Interaction& x : m.interactions)
    if (bit_at(static_cast<std::size_t>(x.i)) && bit_at(static_cast<std::size_t>(x.j))) t += x.value;
  return t;
}

Genome genome_from_mask(std::uint64_t mask, std::size_t a) {
  Genome g = Genome::zeros(a);
  for (std::size_t k = 0; k < a; ++k) g.set(k, (mask >> k) & 1u);
  return g;
}

// bit-string order: gene 0 is the most significant position
bool mask_lex_less(std::uint64_t x, std::uint64_t y, std::size_t a) {
  for (std::size_t k = 0; k < a; ++k) {
    const unsigned bx = (x >> k) & 1u, by = (y >> k) & 1u;
    if (bx != by) return bx < by;
  }
  return false;
}

double number_field(const json::Value& obj, const char* key) {
  const json::Value* v = obj.find(key);
  if (v == nullptr || !v->is_number()) throw ModelError(std::string("model: missing or non-numeric '") + key + "'");
  return v->number;
}

void require_positive_everywhere(const CostModel& m) {
  const std::size_t a = m.loops.size();
  auto check = [&](const Genome& g) {
    if (summed_time(m, [&](std::size_t k) { return g.test(k); }) <= 0.0)
      throw ModelError("model: genome " + g.to_string() + " has non-positive time");
  };
  if (a <= 16) {
    for (std::uint64_t mask = 0; mask < (std::uint64_t{1} << a); ++mask) check(genome_from_mask(mask, a));
    return;
  }
  // too many to enumerate: corners, single loops, all-but-one, and a fixed random sample
  check(Genome::zeros(a));
  check(Genome::ones(a));
  for (std::size_t k = 0; k < a; ++k) {
    Genome only = Genome::zeros(a);
    only.set(k, true);
    check(only);
    Genome without = Genome::ones(a);
    without.set(k, false);
    check(without);
  }
  std::mt19937_64 sampler(0x5eed);
  for (int s = 0; s < 4096; ++s) {
    Genome g = Genome::zeros(a);
    for (std::size_t k = 0; k < a; ++k) g.set(k, (sampler() & 1u) != 0);
    check(g);
  }
}

}  // namespace

double CostModel::baseline_s() const {
  double total = serial_s;
  for (const LoopCost& lc : loops) total += lc.compute_s;
  return total;
}

double model_time(const CostModel& model, const Genome& genome) {
  if (genome.size() != model.loops.size())
    throw ModelGenomeMismatch("genome length " + std::to_string(genome.size()) + " does not match model loop count " +
                              std::to_string(model.loops.size()));
  if (model.fail_set.find(genome) != model.fail_set.end())
    throw SimulatedCompileError("genome " + genome.to_string() + " is in the model's fail set");
  return summed_time(model, [&](std::size_t k) { return genome.test(k); });
}

OracleResult exhaustive_best(const CostModel& model) {
  const std::size_t a = model.loops.size();
  if (a > 20) throw GeneLengthTooLarge("exhaustive search over " + std::to_string(a) + " genes is not enumerable (limit 20)");
  bool have = false;
  std::uint64_t best = 0;
  double best_t = 0.0;
  for (std::uint64_t mask = 0; mask < (std::uint64_t{1} << a); ++mask) {
    if (!model.fail_set.empty() && model.fail_set.count(genome_from_mask(mask, a)) != 0) continue;
    const double t = summed_time(model, [&](std::size_t k) { return ((mask >> k) & 1u) != 0; });
    if (!have || t < best_t || (t == best_t && mask_lex_less(mask, best, a))) {
      have = true;
      best = mask;
      best_t = t;
    }
  }
  if (!have) throw ModelError("every genome is in the model's fail set");
  return {genome_from_mask(best, a), best_t};
}

CostModel parse_model(const std::string& json_text) {
  json::Value root;
  if (!json::parse(json_text, root) || !root.is_object()) throw ModelError("model: not a JSON object");

  CostModel m;
  m.serial_s = number_field(root, "serial_s");
  if (m.serial_s < 0.0) throw ModelError("model: serial_s must be >= 0");

  const json::Value* loops = root.find("loops");
  if (loops == nullptr || !loops->is_array()) throw ModelError("model: missing 'loops' array");
  for (const json::Value& e : *loops->array) {
    if (!e.is_object()) throw ModelError("model: loop entries must be objects");
    LoopCost lc;
    lc.compute_s = number_field(e, "compute_s");
    lc.speedup = number_field(e, "speedup");
    lc.transfer_s = number_field(e, "transfer_s");
    if (lc.compute_s < 0.0) throw ModelError("model: compute_s must be >= 0");
    if (lc.speedup < 1.0) throw ModelError("model: speedup must be >= 1");
    if (lc.transfer_s < 0.0) throw ModelError("model: transfer_s must be >= 0");
    m.loops.push_back(lc);
  }
  const int a = static_cast<int>(m.loops.size());

  if (const json::Value* inter = root.find("interactions")) {
    if (!inter->is_array()) throw ModelError("model: 'interactions' must be an array");
    for (const json::Value& e : *inter->array) {
      const bool shape_ok = e.is_array() && e.array->size() == 3 && (*e.array)[0].is_number() && (*e.array)[0].is_integer &&
                            (*e.array)[1].is_number() && (*e.array)[1].is_integer && (*e.array)[2].is_number();
      if (!shape_ok) throw ModelError("model: interactions must be [i, j, value] triples");
      Interaction x;
      x.i = static_cast<int>((*e.array)[0].number);
      x.j = static_cast<int>((*e.array)[1].number);
      x.value = (*e.array)[2].number;
      if (x.i > x.j) std::swap(x.i, x.j);
      if (x.i < 0 || x.j >= a || x.i == x.j)
        throw ModelError("model: interaction pair (" + std::to_string(x.i) + ", " + std::to_string(x.j) + ") out of range");
      for (const Interaction& seen : m.interactions)
        if (seen.i == x.i && seen.j == x.j)
          throw ModelError("model: duplicate interaction pair (" + std::to_string(x.i) + ", " + std::to_string(x.j) + ")");
      m.interactions.push_back(x);
    }
  }

  if (const json::Value* fail = root.find("fail")) {
    if (!fail->is_array()) throw ModelError("model: 'fail' must be an array");
    for (const json::Value& e : *fail->array) {
      if (!e.is_string()) throw ModelError("model: fail entries must be bit strings");
      if (static_cast<int>(e.string.size()) != a)
        throw ModelError("model: fail entry '" + e.string + "' does not have " + std::to_string(a) + " bits");
      try {
        m.fail_set.insert(Genome::from_string(e.string));
      } catch (const Error&) {
        throw ModelError("model: fail entry '" + e.string + "' is not a bit string");
      }
    }
  }

  require_positive_everywhere(m);
  return m;
}

CostModel load_model(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ModelError("model: cannot read " + path.string());
  std::ostringstream text;
  text << in.rdbuf();
  return parse_model(text.str());
}

}  // namespace mmxhost
