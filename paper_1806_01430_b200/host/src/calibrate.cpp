// calibrate.cpp -- see calibrate.hpp.
#include "mmxhost/calibrate.hpp"

#include <algorithm>
#include <array>
#include <cmath>

#include "mmxhost/errors.hpp"
#include "mmxhost/json_lite.hpp"

namespace mmxhost {
namespace {

constexpr int kParams = 1 + MMX_NUM_NESTS + MMX_GENE_LENGTH + 3;  // s, cpu[6], loop[12], alpha, beta, lambda
constexpr int P_SERIAL = 0, P_CPU = 1, P_LOOP = P_CPU + MMX_NUM_NESTS, P_H2D = P_LOOP + MMX_GENE_LENGTH, P_D2H = P_H2D + 1,
              P_XFER = P_D2H + 1;
constexpr double kByteScale = 1e-9;  // bytes enter the regression in GB so that all columns have comparable size

struct NestLoops {
  int first, count;
};
// genes of each nest (fixtures/matmul.c: lines 8-9, 12-13, 16-17, 21-22, 25-27, 31); same table as csrc/plan.cpp
constexpr NestLoops kNests[MMX_NUM_NESTS] = {{0, 2}, {2, 2}, {4, 2}, {6, 2}, {8, 3}, {11, 1}};

bool features(const Genome& g, int n, int dtype, double (&x)[kParams]) {
  mmx_plan_info plan;
  if (mmx_plan(g.bits().data(), g.size(), n, dtype, &plan) != MMX_OK || !plan.feasible) return false;
  std::fill(std::begin(x), std::end(x), 0.0);
  x[P_SERIAL] = 1.0;
  for (int nest = 0; nest < MMX_NUM_NESTS; ++nest) {
    int on = -1;
    for (int k = kNests[nest].first; k < kNests[nest].first + kNests[nest].count; ++k)
      if (g.test(static_cast<std::size_t>(k))) on = k;
    if (on < 0) x[P_CPU + nest] = 1.0;
    else x[P_LOOP + on] = 1.0;
  }
  for (int s = 0; s < plan.num_steps; ++s) {
    const mmx_plan_step& st = plan.steps[s];
    if (st.kind == MMX_STEP_H2D || st.kind == MMX_STEP_H2D_DIAG) {
      x[P_H2D] += static_cast<double>(st.bytes) * kByteScale;
      x[P_XFER] += 1.0;
    } else if (st.kind == MMX_STEP_D2H || st.kind == MMX_STEP_D2H_DIAG || st.kind == MMX_STEP_D2H_SUM) {
      x[P_D2H] += static_cast<double>(st.bytes) * kByteScale;
      x[P_XFER] += 1.0;
    }
  }
  return true;
}

double dot(const double (&x)[kParams], const double (&w)[kParams]) {
  double t = 0.0;
  for (int p = 0; p < kParams; ++p) t += x[p] * w[p];
  return t;
}

void to_weights(const PlanModel& m, double (&w)[kParams]) {
  w[P_SERIAL] = m.serial_s;
  for (int i = 0; i < MMX_NUM_NESTS; ++i) w[P_CPU + i] = m.cpu_s[i];
  for (int k = 0; k < MMX_GENE_LENGTH; ++k) w[P_LOOP + k] = m.loop_s[k];
  w[P_H2D] = m.h2d_s_per_byte / kByteScale;
  w[P_D2H] = m.d2h_s_per_byte / kByteScale;
  w[P_XFER] = m.per_transfer_s;
}

Genome genome_of_mask(unsigned mask) {
  std::vector<std::uint8_t> bits(MMX_GENE_LENGTH);
  for (int k = 0; k < MMX_GENE_LENGTH; ++k) bits[static_cast<std::size_t>(k)] = (mask >> k) & 1u;
  return Genome(std::move(bits));
}

}  // namespace

PlanModel fit_plan_model(const std::vector<GenomeSample>& samples, int n, int dtype, FitReport* report) {
  // rows scaled by 1 / measured time: the objective is the sum of squared RELATIVE errors, so microsecond genomes
  // count as much as the seconds-long ones
  std::vector<std::array<double, kParams>> rows;
  std::vector<double> raw_t;
  for (const GenomeSample& s : samples) {
    if (s.genome.size() != MMX_GENE_LENGTH) throw GenomeLengthMismatch("calibration sample of length " + std::to_string(s.genome.size()));
    double x[kParams];
    if (!(s.time_s > 0.0) || !features(s.genome, n, dtype, x)) continue;
    std::array<double, kParams> r;
    for (int p = 0; p < kParams; ++p) r[static_cast<std::size_t>(p)] = x[p] / s.time_s;
    rows.push_back(r);
    raw_t.push_back(s.time_s);
  }
  if (rows.size() < static_cast<std::size_t>(kParams)) throw ModelError("calibration needs at least " + std::to_string(kParams) + " feasible samples");
  // normal equations A w = b with target 1 for every (scaled) row
  double A[kParams][kParams] = {}, b[kParams] = {};
  for (const auto& r : rows)
    for (int p = 0; p < kParams; ++p) {
      b[p] += r[static_cast<std::size_t>(p)];
      for (int q = 0; q < kParams; ++q) A[p][q] += r[static_cast<std::size_t>(p)] * r[static_cast<std::size_t>(q)];
    }
  // Lawson-Hanson active-set NNLS on the normal equations.  The indicator columns are redundant by construction
  // (every nest contributes exactly one active column, so a constant can move between nests and the serial
  // term without changing any prediction): a tiny ridge picks one member of that family.
  // columns are first scaled to unit norm (their natural sizes differ by many orders of magnitude)
  double colscale[kParams];
  for (int p = 0; p < kParams; ++p) colscale[p] = A[p][p] > 0.0 ? 1.0 / std::sqrt(A[p][p]) : 0.0;
  for (int p = 0; p < kParams; ++p) {
    b[p] *= colscale[p];
    for (int q = 0; q < kParams; ++q) A[p][q] *= colscale[p] * colscale[q];
  }
  for (int p = 0; p < kParams; ++p) A[p][p] += 1e-11;
  double w[kParams] = {};
  bool passive[kParams] = {};
  auto solve_passive = [&](double (&z)[kParams]) {  // Cholesky on the passive block
    int idx[kParams], m = 0;
    for (int p = 0; p < kParams; ++p)
      if (passive[p]) idx[m++] = p;
    double L[kParams][kParams] = {}, y[kParams];
    for (int i = 0; i < m; ++i)
      for (int j = 0; j <= i; ++j) {
        double v = A[idx[i]][idx[j]];
        for (int k = 0; k < j; ++k) v -= L[i][k] * L[j][k];
        L[i][j] = i == j ? std::sqrt(std::max(v, 1e-300)) : v / L[j][j];
      }
    for (int i = 0; i < m; ++i) {
      double v = b[idx[i]];
      for (int k = 0; k < i; ++k) v -= L[i][k] * y[k];
      y[i] = v / L[i][i];
    }
    std::fill(std::begin(z), std::end(z), 0.0);
    for (int i = m - 1; i >= 0; --i) {
      double v = y[i];
      for (int k = i + 1; k < m; ++k) v -= L[k][i] * z[idx[k]];
      z[idx[i]] = v / L[i][i];
    }
  };
  for (int outer = 0; outer < 10 * kParams; ++outer) {
    int pick = -1;
    double best_grad = 0.0, scale = 0.0;
    for (int p = 0; p < kParams; ++p) scale = std::max(scale, std::fabs(b[p]));
    for (int p = 0; p < kParams; ++p) {
      if (passive[p] || colscale[p] == 0.0) continue;  // a feature no sample exercises stays zero
      double g = b[p];
      for (int q = 0; q < kParams; ++q) g -= A[p][q] * w[q];
      if (g > best_grad) {
        best_grad = g;
        pick = p;
      }
    }
    if (pick < 0 || best_grad <= 1e-12 * scale) break;
    passive[pick] = true;
    for (int inner = 0; inner < 10 * kParams; ++inner) {
      double z[kParams];
      solve_passive(z);
      bool ok = true;
      double alpha = 1.0;
      for (int p = 0; p < kParams; ++p)
        if (passive[p] && z[p] <= 0.0) {
          ok = false;
          alpha = std::min(alpha, w[p] / (w[p] - z[p]));
        }
      if (ok) {
        std::copy(std::begin(z), std::end(z), std::begin(w));
        break;
      }
      for (int p = 0; p < kParams; ++p)
        if (passive[p]) {
          w[p] += alpha * (z[p] - w[p]);
          if (w[p] <= 1e-300) {
            w[p] = 0.0;
            passive[p] = false;
          }
        }
    }
  }
  for (int p = 0; p < kParams; ++p) w[p] *= colscale[p];
  PlanModel m;
  m.n = n;
  m.dtype = dtype;
  m.serial_s = w[P_SERIAL];
  for (int i = 0; i < MMX_NUM_NESTS; ++i) m.cpu_s[i] = w[P_CPU + i];
  for (int k = 0; k < MMX_GENE_LENGTH; ++k) m.loop_s[k] = w[P_LOOP + k];
  m.h2d_s_per_byte = w[P_H2D] * kByteScale;
  m.d2h_s_per_byte = w[P_D2H] * kByteScale;
  m.per_transfer_s = w[P_XFER];
  if (report) {
    report->samples = rows.size();
    double sq = 0.0, mx = 0.0;
    for (const auto& r : rows) {
      double pred = 0.0;
      for (int p = 0; p < kParams; ++p) pred += r[static_cast<std::size_t>(p)] * w[p];  // = predicted / measured
      const double rel = std::fabs(pred - 1.0);
      sq += rel * rel;
      mx = std::max(mx, rel);
    }
    report->rms_rel_err = std::sqrt(sq / static_cast<double>(rows.size()));
    report->max_rel_err = mx;
  }
  return m;
}

double predict_time(const PlanModel& model, const Genome& genome) {
  double x[kParams], w[kParams];
  if (genome.size() != MMX_GENE_LENGTH) throw ModelGenomeMismatch("genome length " + std::to_string(genome.size()));
  if (!features(genome, model.n, model.dtype, x)) throw SimulatedCompileError("genome " + genome.to_string() + " is infeasible");
  to_weights(model, w);
  return dot(x, w);
}

CostModel project_to_cost_model(const PlanModel& pm, ProjectionReport* report) {
  CostModel cm;
  cm.serial_s = pm.serial_s;
  cm.loops.resize(MMX_GENE_LENGTH);
  std::vector<int> inexact;

  // 1. compute: per nest, split the CPU time C over its loops so that offloading loop l alone leaves T_l
  double offloaded_extra[MMX_GENE_LENGTH] = {};  // e_l = c_l / g_l + (compute part of d_l)
  for (int nest = 0; nest < MMX_NUM_NESTS; ++nest) {
    const int first = kNests[nest].first, count = kNests[nest].count;
    const double C = pm.cpu_s[nest];
    std::vector<int> order(static_cast<std::size_t>(count));
    for (int i = 0; i < count; ++i) order[static_cast<std::size_t>(i)] = first + i;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return pm.loop_s[x] < pm.loop_s[y]; });  // fastest first
    double c[3] = {0.0, 0.0, 0.0}, left = C;
    for (int l : order) {  // every loop wants c_l >= C - T_l; the fastest are served first
      const double want = std::min(left, std::max(0.0, C - pm.loop_s[l]));
      c[l - first] = want;
      left -= want;
    }
    c[order.front() - first] += left;  // what nobody needs goes to the fastest alternative (keeps the others' c small)
    for (int i = 0; i < count; ++i) {
      const int l = first + i;
      const double others = C - c[i];
      double e = pm.loop_s[l] - others;  // what the offloaded loop itself may cost
      if (e < 0.0) {
        inexact.push_back(l);
        e = 0.0;
      }
      cm.loops[static_cast<std::size_t>(l)].compute_s = c[i];
      offloaded_extra[l] = e;
    }
  }

  // 2. transfers: producer nest -> consumer nest edges of the program (csrc/plan.cpp), cost lambda + bytes * rate
  const double e_bytes = pm.dtype == MMX_F64 ? 8.0 : 4.0, nn = static_cast<double>(pm.n);
  const double full = nn * nn * e_bytes, diag = nn * e_bytes;
  struct Edge {
    int p, q;
    double bytes;
  };
  const Edge edges[] = {{MMX_NEST_INIT_A, MMX_NEST_MATMUL, full}, {MMX_NEST_INIT_B, MMX_NEST_TRANSPOSE, full},
                        {MMX_NEST_TRANSPOSE, MMX_NEST_MATMUL, full}, {MMX_NEST_ZERO_C, MMX_NEST_MATMUL, full},
                        {MMX_NEST_MATMUL, MMX_NEST_TRACE, diag}};
  double transfer_d[MMX_GENE_LENGTH] = {};
  double J[MMX_GENE_LENGTH][MMX_GENE_LENGTH] = {};
  for (const Edge& e : edges) {
    const double down = pm.per_transfer_s + e.bytes * pm.d2h_s_per_byte;  // producer on the GPU, consumer on the host
    const double up = pm.per_transfer_s + e.bytes * pm.h2d_s_per_byte;    // the other way round
    for (int i = kNests[e.p].first; i < kNests[e.p].first + kNests[e.p].count; ++i) transfer_d[i] += down;
    for (int j = kNests[e.q].first; j < kNests[e.q].first + kNests[e.q].count; ++j) transfer_d[j] += up;
    for (int i = kNests[e.p].first; i < kNests[e.p].first + kNests[e.p].count; ++i)
      for (int j = kNests[e.q].first; j < kNests[e.q].first + kNests[e.q].count; ++j) J[std::min(i, j)][std::max(i, j)] -= down + up;
  }
  // the checksum comes back (8 bytes) whenever the trace runs on the GPU: the host's printf consumes it
  transfer_d[11] += pm.per_transfer_s + 8.0 * pm.d2h_s_per_byte;

  // 3. (c_l, g_l, d_l) from c_l, e_l and the transfer share
  for (int l = 0; l < MMX_GENE_LENGTH; ++l) {
    LoopCost& lc = cm.loops[static_cast<std::size_t>(l)];
    const double e = offloaded_extra[l];
    if (lc.compute_s > 0.0 && e < lc.compute_s) {
      // c/g = e, capped so that g stays finite when the offloaded time is ~0
      lc.speedup = std::min(lc.compute_s / std::max(e, lc.compute_s * 1e-9), 1e9);
      lc.transfer_s = transfer_d[l] + (e - lc.compute_s / lc.speedup);
    } else {
      lc.speedup = 1.0;
      lc.transfer_s = transfer_d[l] + (e - lc.compute_s);
    }
    if (lc.transfer_s < 0.0) lc.transfer_s = 0.0;
  }

  // 4. infeasible genomes: fail list, and a positive J on same-nest pairs so that every raw sum stays positive
  double guard = cm.serial_s;
  for (int i = 0; i < MMX_GENE_LENGTH; ++i)
    for (int j = i + 1; j < MMX_GENE_LENGTH; ++j) guard += std::fabs(J[i][j]);
  for (const NestLoops& nl : kNests)
    for (int i = nl.first; i < nl.first + nl.count; ++i)
      for (int j = i + 1; j < nl.first + nl.count; ++j) J[i][j] = guard + 1e-6;
  for (int i = 0; i < MMX_GENE_LENGTH; ++i)
    for (int j = i + 1; j < MMX_GENE_LENGTH; ++j)
      if (J[i][j] != 0.0) cm.interactions.push_back({i, j, J[i][j]});
  for (unsigned mask = 0; mask < (1u << MMX_GENE_LENGTH); ++mask) {
    bool clash = false;
    for (const NestLoops& nl : kNests) {
      int set = 0;
      for (int k = nl.first; k < nl.first + nl.count; ++k) set += (mask >> k) & 1u;
      clash = clash || set > 1;
    }
    if (clash) cm.fail_set.insert(genome_of_mask(mask));
  }

  if (report) {
    report->inexact_loops = inexact;
    double sq = 0.0, mx = 0.0;
    std::size_t count = 0;
    bool first = true;
    for (unsigned mask = 0; mask < (1u << MMX_GENE_LENGTH); ++mask) {
      const Genome g = genome_of_mask(mask);
      if (cm.fail_set.count(g)) continue;
      const double tp = predict_time(pm, g), tc = model_time(cm, g);
      const double rel = std::fabs(tc - tp) / tp;
      sq += rel * rel;
      mx = std::max(mx, rel);
      ++count;
      if (first || tp < report->plan_best_s) {
        report->plan_best_s = tp;
        report->plan_best = g;
      }
      if (first || tc < report->cost_best_s) {
        report->cost_best_s = tc;
        report->cost_best = g;
      }
      first = false;
    }
    report->rms_rel_err = std::sqrt(sq / static_cast<double>(count));
    report->max_rel_err = mx;
  }
  return cm;
}

std::string dump_cost_model_json(const CostModel& model) {
  std::string s = "{\n  \"serial_s\": " + json::dump_number(model.serial_s) + ",\n  \"loops\": [\n";
  for (std::size_t k = 0; k < model.loops.size(); ++k) {
    const LoopCost& l = model.loops[k];
    s += "    {\"compute_s\": " + json::dump_number(l.compute_s) + ", \"speedup\": " + json::dump_number(l.speedup) +
         ", \"transfer_s\": " + json::dump_number(l.transfer_s) + "}" + (k + 1 < model.loops.size() ? "," : "") + "\n";
  }
  s += "  ],\n  \"interactions\": [\n";
  for (std::size_t k = 0; k < model.interactions.size(); ++k) {
    const Interaction& it = model.interactions[k];
    s += "    [" + std::to_string(it.i) + ", " + std::to_string(it.j) + ", " + json::dump_number(it.value) + "]" +
         (k + 1 < model.interactions.size() ? "," : "") + "\n";
  }
  s += "  ],\n  \"fail\": [";
  std::vector<std::string> fails;
  for (const Genome& g : model.fail_set) fails.push_back(g.to_string());
  std::sort(fails.begin(), fails.end());
  for (std::size_t k = 0; k < fails.size(); ++k) s += std::string(k ? ", " : "") + (k % 8 == 0 ? "\n    " : "") + "\"" + fails[k] + "\"";
  s += "\n  ]\n}\n";
  return s;
}

}  // namespace mmxhost
