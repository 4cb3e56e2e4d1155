// ga.hpp -- the Simple GA that calls the batch evaluator.
//
// Everything here is integer / RNG / ordering work that must be BIT-EXACT with the reference
// (/root/reference/proj/src/ga.cpp, include/acctune/ga.hpp): the RNG draw order is part of the
// contract:
//   init        M*a   bit()            one per gene, genome by genome
//   per generation (except after the last):
//     selection (M - elite) real01()   roulette, cumulative sum in population order
//     per parent pair: 1 real01() (crossover?), then index(a-1) if crossing,
//                      then a real01() per child (mutation), child 1 before child 2
//     odd last parent: copied, then a real01()
// Elite = highest fitness, ties -> lexicographically smaller genome; best = lowest time, ties ->
// smaller genome.  Fitness = t^(-1/2); failed individuals get 1e-3 * the smallest measured
// fitness of the population (0 if nothing measured).
#pragma once

#include <random>
#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <string>
#include <utility>
#include <vector>

#include "mmxhost/evaluator.hpp"
#include "mmxhost/genome.hpp"
#include "mmxhost/source_model.hpp"

namespace mmxhost {

// ---- the random stream (/root/reference/proj/include/acctune/rng.hpp:13-31): the draw order is part of the GA contract ----


class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}

  std::uint64_t raw() { return engine_(); }
  // low bit of one draw
  bool bit() { return (raw() & 1u) == 1u; }
  // top 53 bits of one draw scaled into [0, 1)
  double real01() { return static_cast<double>(raw() >> 11) * (1.0 / 9007199254740992.0); }
  // one draw modulo n
  std::size_t index(std::size_t n) { return static_cast<std::size_t>(raw() % n); }

 private:
  std::mt19937_64 engine_;
};


// ---- the GA ------------------------------------------------------------------------------------------------------

struct GAParams {
  int population = 12;          // M
  int generations = 12;         // T
  double crossover_rate = 0.9;  // Pc
  double mutation_rate = 0.05;  // Pm
  std::uint64_t seed = 1;
  int elite_count = 1;
};

// ConfigError unless M >= 2, T >= 1, rates in [0,1], 1 <= elite < M.
void validate_params(const GAParams& params);

enum class IndividualStatus { Unevaluated = 0, Measured = 1, Failed = 2 };

struct Individual {
  Genome genome;
  IndividualStatus status = IndividualStatus::Unevaluated;
  double time_s = 0.0;
  double fitness = 0.0;
};

struct GenerationStats {
  int generation = 0;  // 0 = baseline row
  double best_time_s = 0.0;
  Genome best_genome;
  double mean_fitness = 0.0;
  std::uint64_t distinct_evals = 0;
  std::uint64_t cache_hits = 0;
};

struct TuningResult {
  Genome best_genome;
  double best_time_s = 0.0;
  double baseline_s = 0.0;
  std::vector<GenerationStats> generations;  // T + 1 rows
};

double fitness_from_time(double t);
std::vector<Genome> init_population(std::size_t gene_length, const GAParams& params, Rng& rng);
void assign_fitness(std::vector<Individual>& population);
std::vector<Genome> roulette_select(const std::vector<Individual>& population, std::size_t count, Rng& rng);
Genome mutate(const Genome& g, double pm, Rng& rng);
std::pair<Genome, Genome> crossover_at(const Genome& p1, const Genome& p2, std::size_t cut);
std::pair<Genome, Genome> one_point_crossover(const Genome& p1, const Genome& p2, Rng& rng);
std::vector<Individual> breed(const std::vector<Individual>& population, const GAParams& params, Rng& rng);

struct RunningBest {
  double time_s = 0.0;
  Genome genome;
  bool update(double t, const Genome& g);
};

// Baseline (all-zero genome) + T generations.  Same signature as the reference's (include/acctune/ga.hpp:107); it reads the
// candidate set's gene length only (ga.cpp:247-250) -- rendering the winner's source is the caller's business in both.
TuningResult run_ga(const CandidateSet& cs, const GAParams& params, GenomeEvaluator& evaluator);
// The same search for callers that have a gene length but no source model (the C window used by the rank-sharded evaluator).
TuningResult run_ga(std::size_t gene_length, const GAParams& params, GenomeEvaluator& evaluator);

// generation,best_time_s,best_speedup,best_genome,mean_fitness,distinct_evals,cache_hits  (%.9g)
void write_generation_csv(std::ostream& out, const TuningResult& result);

}  // namespace mmxhost
