// ga_operators.cpp -- the GA's building blocks: parameter checks, fitness, selection, mutation, crossover.
// Behaviour and RNG draw order: /root/reference/proj/src/ga.cpp:14-135 (pinned by tests/golden/ga_operators.json).
#include "mmxhost/ga.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <ostream>

#include "mmxhost/errors.hpp"

namespace mmxhost {

void validate_params(const GAParams& p) {
  if (p.population < 2) throw ConfigError("population must be at least 2");
  if (p.generations < 1) throw ConfigError("generations must be at least 1");
  if (!(p.crossover_rate >= 0.0 && p.crossover_rate <= 1.0)) throw ConfigError("crossover_rate must be in [0, 1]");
  if (!(p.mutation_rate >= 0.0 && p.mutation_rate <= 1.0)) throw ConfigError("mutation_rate must be in [0, 1]");
  if (p.elite_count < 1) throw ConfigError("elite_count must be at least 1");
  if (p.elite_count >= p.population) throw ConfigError("elite_count must be smaller than the population");
}

// fitness = (processing time)^(-1/2)
double fitness_from_time(double t) {
  if (!(t > 0.0)) throw NonPositiveTime("fitness needs a positive time, got " + std::to_string(t));
  return std::pow(t, -0.5);
}

std::vector<Genome> init_population(std::size_t gene_length, const GAParams& params, Rng& rng) {
  if (gene_length < 1) throw ConfigError("gene length must be at least 1");
  std::vector<Genome> pop(static_cast<std::size_t>(params.population), Genome::zeros(gene_length));
  for (Genome& g : pop)
    for (std::size_t k = 0; k < gene_length; ++k) g.set(k, rng.bit());  // M*a draws, genome-major
  return pop;
}

void assign_fitness(std::vector<Individual>& population) {
  double weakest = std::numeric_limits<double>::infinity();
  for (Individual& ind : population) {
    if (ind.status != IndividualStatus::Measured) continue;
    ind.fitness = fitness_from_time(ind.time_s);
    weakest = std::min(weakest, ind.fitness);
  }
  // broken genomes stay selectable, three orders of magnitude below the worst working one
  const double penalty = std::isinf(weakest) ? 0.0 : 1e-3 * weakest;
  for (Individual& ind : population)
    if (ind.status != IndividualStatus::Measured) ind.fitness = penalty;
}

std::vector<Genome> roulette_select(const std::vector<Individual>& population, std::size_t count, Rng& rng) {
  double wheel = 0.0;
  for (const Individual& ind : population) wheel += ind.fitness;
  if (!(wheel > 0.0)) throw ZeroTotalFitness("every individual has zero selection weight; the run cannot proceed");
  std::vector<Genome> chosen;
  chosen.reserve(count);
  for (std::size_t draw = 0; draw < count; ++draw) {
    const double needle = rng.real01() * wheel;
    std::size_t slot = population.size() - 1;  // rounding at the top edge lands on the last slot
    double running = 0.0;
    for (std::size_t i = 0; i < population.size(); ++i) {
      running += population[i].fitness;
      if (needle < running) {
        slot = i;
        break;
      }
    }
    chosen.push_back(population[slot].genome);
  }
  return chosen;
}

Genome mutate(const Genome& g, double pm, Rng& rng) {
  if (!(pm >= 0.0 && pm <= 1.0)) throw ConfigError("mutation rate must be in [0, 1]");
  Genome child = g;
  for (std::size_t k = 0; k < child.size(); ++k) {
    const double u = rng.real01();  // drawn for every bit, whatever pm is
    if (u < pm) child.flip(k);
  }
  return child;
}

namespace {
void require_same_length(const Genome& p1, const Genome& p2) {
  if (p1.size() != p2.size())
    throw GenomeLengthMismatch("crossover parents differ in length: " + std::to_string(p1.size()) + " vs " +
                               std::to_string(p2.size()));
}
}  // namespace

std::pair<Genome, Genome> crossover_at(const Genome& p1, const Genome& p2, std::size_t cut) {
  require_same_length(p1, p2);
  if (cut < 1 || cut >= p1.size())
    throw Error("crossover cut point " + std::to_string(cut) + " outside [1, " +
                std::to_string(p1.empty() ? 0 : p1.size() - 1) + "]");
  std::pair<Genome, Genome> kids{p1, p2};
  for (std::size_t k = cut; k < p1.size(); ++k) {  // swap tails
    kids.first.set(k, p2.test(k));
    kids.second.set(k, p1.test(k));
  }
  return kids;
}

std::pair<Genome, Genome> one_point_crossover(const Genome& p1, const Genome& p2, Rng& rng) {
  require_same_length(p1, p2);
  if (p1.size() < 2) throw GenomeLengthMismatch("one-point crossover needs at least 2 genes");
  return crossover_at(p1, p2, 1 + rng.index(p1.size() - 1));
}


}  // namespace mmxhost
