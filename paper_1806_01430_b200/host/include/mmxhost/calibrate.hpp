// calibrate.hpp -- measured genome times -> a model of the executor -> the reference's CostModel JSON.
//
// The step AFTER the hot path.  The reference tunes against synthetic models it ships as
// fixtures (fixtures/models/*.json, parsed by /root/reference/proj/src/sim_model.cpp:157-236) and states model
// calibration as a non-goal; with real CUDA-event timings available the same file format can be FITTED, which
// gives (a) an exact search oracle -- exhaustive_best (sim_model.cpp:62-98) -- to score the GA against on real
// data, and (b) a SimBackend that replays a machine without the machine.
//
// Two levels:
//   PlanModel   what the executor actually does: t = s + sum_nest T[nest][mode] + transfers, where a transfer of
//               B bytes costs lambda + B * (alpha up | beta down).  Linear in its 22 parameters; fitted by
//               non-negative least squares over measured (genome, time) samples.  Features come from mmx_plan().
//   CostModel   the reference's additive form t = s + sum c_i | (c_i/g_i + d_i) + sum J_ij.  Transfers map onto it
//               exactly: an array handed from nest P to nest Q costs  D x_P (1 - x_Q) + U (1 - x_P) x_Q, i.e.
//               d_i += D (i in P), d_j += U (j in Q), J_ij -= D + U.  Alternative offload depths of ONE nest do not:
//               with CPU time C and offloaded times T_l the form needs c_l >= C - T_l and sum c_l = C, possible
//               only when sum_l max(0, C - T_l) <= C.  Otherwise the fastest alternatives are kept exact and the
//               slowest absorbs the residual; ProjectionReport says which loops and by how much.  Genomes with two
//               bits in one nest go to the fail list, and same-nest pairs get a positive J so that every raw sum
//               stays positive (the reference validates that, sim_model.cpp:124-155).
#pragma once

#include <string>
#include <vector>

#include "mmx.h"
#include "mmxhost/genome.hpp"
#include "mmxhost/cost_model.hpp"

namespace mmxhost {

struct GenomeSample {
  Genome genome;
  double time_s = 0.0;
};

struct PlanModel {
  int n = 0, dtype = MMX_F64;
  double serial_s = 0.0;
  double cpu_s[MMX_NUM_NESTS] = {};        // nest on the host
  double loop_s[MMX_GENE_LENGTH] = {};     // nest offloaded at this loop (all its launches)
  double h2d_s_per_byte = 0.0, d2h_s_per_byte = 0.0, per_transfer_s = 0.0;
};

struct FitReport {
  std::size_t samples = 0;
  double rms_rel_err = 0.0, max_rel_err = 0.0;  // |predicted - measured| / measured over the samples
};

// Non-negative least squares on relative residuals.  Samples of infeasible genomes are ignored.
PlanModel fit_plan_model(const std::vector<GenomeSample>& samples, int n, int dtype, FitReport* report = nullptr);

// time of a feasible genome under the model; ModelError for an infeasible one
double predict_time(const PlanModel& model, const Genome& genome);

struct ProjectionReport {
  std::vector<int> inexact_loops;   // loops whose single-bit time the additive form cannot hit
  double rms_rel_err = 0.0, max_rel_err = 0.0;  // CostModel vs PlanModel over all feasible genomes
  Genome plan_best, cost_best;      // exhaustive optimum of either model
  double plan_best_s = 0.0, cost_best_s = 0.0;
};

CostModel project_to_cost_model(const PlanModel& model, ProjectionReport* report = nullptr);

// The reference's model file: {"serial_s", "loops": [{compute_s, speedup, transfer_s}], "interactions": [[i, j, J]], "fail": [...]}
std::string dump_cost_model_json(const CostModel& model);

}  // namespace mmxhost
