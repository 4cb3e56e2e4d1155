/*
 * capi_host.h -- C window onto the C++ host layer (namespace mmxhost), for Python tests and
 * bench.py.  The C++ classes are the product API (they mirror the reference's acctune classes);
 * this header only lets a ctypes caller drive them.  Return: >= 0 success, negative = error class
 * (same numbering as oracle/ref_shim.cpp so both sides can be driven by one test).
 */
#ifndef MMXHOST_CAPI_H_
#define MMXHOST_CAPI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MMXH_API __attribute__((visibility("default")))

enum {
  MMXH_E_ERROR = -1,
  MMXH_E_LENGTH = -2,        /* GenomeLengthMismatch */
  MMXH_E_TOOLCHAIN = -3,     /* ToolchainMissing */
  MMXH_E_WORKDIR = -4,       /* WorkdirUnwritable */
  MMXH_E_ZERO_FITNESS = -5,  /* ZeroTotalFitness */
  MMXH_E_UNAVAILABLE = -6,   /* EvaluatorUnavailable */
  MMXH_E_NONPOSITIVE = -7,   /* NonPositiveTime */
  MMXH_E_CONFIG = -8,        /* ConfigError */
  MMXH_E_NOCANDIDATES = -9,  /* NoCandidates */
  MMXH_E_MODEL = -10         /* ModelError */
};

typedef struct mmxh_outcome {
  int32_t status;
  double time_s;
  double wall_cost_s;
} mmxh_outcome;

/* callback backend: return 0 ok, -3 => ToolchainMissing is thrown, other negative => Error */
typedef int (*mmxh_measure_cb)(const uint8_t* bits, size_t n, mmxh_outcome* out, void* user);

typedef struct mmxh_ga_params {
  int32_t population, generations;
  double crossover_rate, mutation_rate;
  uint64_t seed;
  int32_t elite_count;
} mmxh_ga_params;

typedef struct mmxh_cuda_config {
  int32_t n, dtype, numerics;
  double timeout_s;
  int32_t repetitions, warmup, host_threads, launch_batching, matmul_variant;
  int32_t num_devices;
  const int32_t* devices;
} mmxh_cuda_config;

MMXH_API const char* mmxh_last_error(void);

/* sim model */
MMXH_API int mmxh_model_time_all(const char* model_path, double* times, size_t count);
MMXH_API int mmxh_exhaustive_best(const char* model_path, uint8_t* bits, size_t n, double* t);

/* GA pieces */
MMXH_API int mmxh_fitness_from_time(double t, double* f);
MMXH_API int mmxh_assign_fitness(const int32_t* status, const double* time_s, size_t m, double* fitness);
MMXH_API int mmxh_init_population(size_t a, int m, uint64_t seed, uint8_t* bits);
MMXH_API int mmxh_breed(const uint8_t* bits, const double* fitness, size_t m, size_t a, double pc, double pm, int elite,
                        uint64_t seed, uint64_t skip, uint8_t* next_bits);
MMXH_API int mmxh_roulette(const double* fitness, size_t m, size_t count, uint64_t seed, int32_t* picks);
MMXH_API int mmxh_mutate(const uint8_t* bits, size_t a, double pm, uint64_t seed, uint8_t* out);
MMXH_API int mmxh_one_point_crossover(const uint8_t* p1, const uint8_t* p2, size_t a, uint64_t seed, uint8_t* c1, uint8_t* c2);
MMXH_API int mmxh_rng_draws(uint64_t seed, int kind, uint64_t n_arg, size_t count, double* out, uint64_t* raw_out);

/* evaluators: kind of backend chosen by the constructor used */
MMXH_API void* mmxh_evaluator_create_sim(const char* model_path, int jobs, const char* cache_file);
MMXH_API void* mmxh_evaluator_create_cb(size_t genes, mmxh_measure_cb cb, void* user, int jobs, const char* cache_file);
/* MultiGpuEvaluator over a CudaBackend (jobs = number of device slots) */
MMXH_API void* mmxh_evaluator_create_cuda(const mmxh_cuda_config* cfg, const char* cache_file);
MMXH_API void mmxh_evaluator_destroy(void* h);
MMXH_API int mmxh_evaluator_gene_length(void* h);
MMXH_API int mmxh_evaluator_evaluate(void* h, const uint8_t* bits, size_t n, mmxh_outcome* out);
MMXH_API int mmxh_evaluator_evaluate_all(void* h, const uint8_t* bits, size_t count, size_t n, mmxh_outcome* outs);
MMXH_API int mmxh_evaluator_counters(void* h, uint64_t c4[4], double* elapsed_s);
/* longest-first scheduling of evaluate_all: costs[k] is the predicted cost of genome k (bits: count x n); unknown genomes cost 0 */
MMXH_API int mmxh_evaluator_set_costs(void* h, const uint8_t* bits, const double* costs, size_t count, size_t n);
/* the static estimate MultiGpuEvaluator schedules by (seconds, order of magnitude) */
MMXH_API double mmxh_predicted_cost(const mmxh_cuda_config* cfg, const uint8_t* bits, size_t n);
/* call counters of a callback backend: calls, max_in_flight */
MMXH_API int mmxh_evaluator_cb_stats(void* h, int32_t out2[2]);

/* A GenomeEvaluator implemented by the caller (evaluation.hpp:42-56): `batch` receives the whole
 * evaluate_all() input (count genomes of n bits each) and fills outs[count]; `counters` fills
 * {requests, distinct, cache_hits, backend_calls} and *elapsed_s.  This is the seam a rank-sharded
 * evaluator (paper_1806_01430_b200/sharded.py, torch.distributed) plugs into run_ga through.
 * Return 0, or a negative MMXH_E_* code to make run_ga fail with that error class. */
typedef int (*mmxh_batch_cb)(const uint8_t* bits, size_t count, size_t n, mmxh_outcome* outs, void* user);
typedef int (*mmxh_counters_cb)(uint64_t c4[4], double* elapsed_s, void* user);
MMXH_API int mmxh_run_ga_external(size_t gene_length, mmxh_batch_cb batch, mmxh_counters_cb counters, void* user,
                                  const mmxh_ga_params* params, char* csv, size_t csv_cap, uint8_t* best_bits,
                                  double* best_s, double* baseline_s);

/* run_ga over an evaluator handle; csv receives generations.csv text; returns its length */
MMXH_API int mmxh_run_ga(void* evaluator, const mmxh_ga_params* params, char* csv, size_t csv_cap, uint8_t* best_bits,
                         double* best_s, double* baseline_s);

/* source model: scan_loops / render_variant (source_model.hpp).  mmxh_scan_loops fills up to cap rows of
 * {id, line, depth, header_start, body_begin, body_end, indent_len} and returns the loop count. */
MMXH_API int mmxh_scan_loops(const char* path_label, const char* text, int64_t* rows7, size_t cap);
MMXH_API int mmxh_render_variant(const char* text, const uint8_t* bits, size_t n, char* out, size_t cap);
MMXH_API int mmxh_strip_directives(const char* text, char* out, size_t cap);

/* static feasibility (feasibility.hpp): probe every loop of `text`; `report` receives the probe report (one JSON object per
 * loop, the reference's write_probe_report format); returns the number of accepted loops or MMXH_E_NOCANDIDATES (report still filled). */
MMXH_API int mmxh_probe_source(const char* path_label, const char* text, char* report, size_t cap);
/* would the variant with directives on the loops whose bit is 1 (every scanned loop is a gene) compile?  1 / 0; `diag` receives
 * one diagnostic line per rejected annotated loop. */
MMXH_API int mmxh_variant_feasible(const char* path_label, const char* text, const uint8_t* bits, size_t n, char* diag, size_t cap);
/* kernel matcher (kernel_match.hpp): JSON {"loops":[{id,line,depth,nest,var,bound,idiom,kernel,writes,reads,why}],"dataflow":[[array,p,q]]};
 * returns the loop count */
MMXH_API int mmxh_match_kernels(const char* path_label, const char* text, char* json_out, size_t cap);

/* calibration (calibrate.hpp): fit the executor's plan model to `count` measured genomes (bits: count x 12), project it onto the
 * reference's cost-model form and write that JSON.  plan22 receives the fitted parameters {serial, cpu[6], loop[12], h2d s/B, d2h s/B,
 * per-transfer s}; report8 = {fit rms rel err, fit max rel err, projection rms, projection max, plan best s, cost best s, #inexact loops,
 * samples used}; best_bits (2 x 12): exhaustive optimum of the plan model, then of the cost model.  Returns the JSON length. */
MMXH_API int mmxh_calibrate(const uint8_t* bits, const double* times, size_t count, int n, int dtype, char* model_json, size_t cap,
                            double* plan22, double* report8, uint8_t* best_bits);
/* time of every genome (index = sum bit_k << k) under the plan model plan22; infeasible genomes get -1 */
MMXH_API int mmxh_plan_model_times(const double* plan22, int n, int dtype, double* times4096);

/* commands (commands.hpp): return the process exit code (0, 1..5); stdout / stderr text is copied out */
MMXH_API int mmxh_cmd_tune(const char* config_path, int has_seed, uint64_t seed, const char* sim_model_or_null, char* out, size_t out_cap,
                           char* err, size_t err_cap);
MMXH_API int mmxh_cmd_report(const char* workdir, char* out, size_t out_cap, char* err, size_t err_cap);
MMXH_API int mmxh_cmd_analyze(const char* config_path, char* out, size_t out_cap, char* err, size_t err_cap);
MMXH_API int mmxh_cmd_calibrate(const char* config_path, char* out, size_t out_cap, char* err, size_t err_cap);

MMXH_API const char* mmxh_status_name(int status);
/* nlohmann-compatible number formatting used by the cache writer */
MMXH_API int mmxh_dump_number(double v, char* out, size_t cap);

#ifdef __cplusplus
}
#endif
#endif
