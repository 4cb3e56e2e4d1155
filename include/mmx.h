/*
 * mmx.h -- C ABI of the B200-native executor for the matrix application's offload
 * genomes (arXiv 1806.01430 hot path).
 *
 * This is the drop-in boundary.  Everything below the reference's
 *     class EvalBackend { virtual EvaluationOutcome measure(const Genome&) = 0;
 *                          virtual std::size_t gene_length() const = 0; };
 * (/root/reference/proj/include/acctune/evaluator.hpp:19-24) is replaced by the
 * functions declared here: instead of "insert #pragma acc kernels, fork an OpenACC
 * compiler, fork the benchmark, parse a time" (ToolchainBackend::measure,
 * /root/reference/proj/src/evaluator.cpp:61-142) a genome is turned into an
 * execution plan over hand-written sm_100a kernels and timed in-process.
 *
 * Conventions
 *   - plain C types only; no C++ exceptions cross this boundary.
 *   - every function returns 0 on success or a negative mmx_error; genome-level
 *     problems are *outcomes* (mmx_outcome.status), infrastructure problems are
 *     *errors* (the C++ shim in paper_1806_01430_b200/host turns them into the
 *     reference's exception types, errors.hpp:10-90).
 *   - `bits` is exactly Genome::bits().data() (genome.hpp:55): one byte per gene,
 *     value 0 or 1, gene 0 first.
 *   - a context owns `num_slots` device slots (one stream, one set of device and
 *     pinned host arrays each).  Calls on different slots may run concurrently from
 *     different threads (the reference calls measure() from up to `jobs` threads,
 *     evaluator.cpp:196-205,254-273); calls on one slot are serialised internally.
 *   - there is no CPU fallback for GPU-mapped loops: without a usable CUDA device
 *     mmx_create fails with MMX_E_NODEVICE.
 */
#ifndef MMX_H_
#define MMX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define MMX_API __attribute__((visibility("default")))
#else
#define MMX_API
#endif

/* The loop catalogue of fixtures/matmul.c has 12 `for` statements; gene k <-> loop id k
 * (source_model.hpp:73-82; tests/test_cli.cpp:212-235). */
#define MMX_GENE_LENGTH 12
#define MMX_NUM_NESTS 6
#define MMX_NUM_ARRAYS 4

typedef enum mmx_error {
  MMX_OK = 0,
  MMX_E_INVALID = -1,  /* bad argument / bad configuration             -> ConfigError        */
  MMX_E_LENGTH = -2,   /* genome length != gene_length()               -> GenomeLengthMismatch (evaluator.cpp:220-224) */
  MMX_E_NODEVICE = -3, /* no CUDA device / driver: the "tool" is absent -> ToolchainMissing  (evaluator.cpp:102) */
  MMX_E_NOMEM = -4,    /* device or pinned-host allocation failed       -> WorkdirUnwritable analogue */
  MMX_E_CUDA = -5,     /* sticky CUDA failure outside a measurement     -> Error             */
  MMX_E_STATE = -6     /* call not valid in this state (e.g. fetch before any run) */
} mmx_error;

/* Order of EvalStatus, evaluation.hpp:13. */
typedef enum mmx_status {
  MMX_MEASURED = 0,
  MMX_COMPILE_ERROR = 1, /* infeasible genome: two annotated loops of one nest (mockacc.cpp:205-221) */
  MMX_RUNTIME_ERROR = 2, /* CUDA error while running the plan, or a non-positive time (evaluator.cpp:125-129) */
  MMX_TIMEOUT = 3        /* over budget; time_s = the budget (evaluator.cpp:103-108) */
} mmx_status;

typedef enum mmx_dtype { MMX_F64 = 0, MMX_F32 = 1 } mmx_dtype;

/* MMX_NUMERICS_FAST: FMA, tiled/shuffled reductions.  FP64 results are bit-identical to
 * the CPU program whenever N is a power of two (all partial sums are exact), otherwise
 * within 1e-12 (norm-wise).  MMX_NUMERICS_STRICT: every reduction runs k ascending with a
 * separate multiply and add, so c and the checksum are bit-identical to the CPU program
 * for every N and both dtypes, at about half the matmul throughput. */
typedef enum mmx_numerics { MMX_NUMERICS_FAST = 0, MMX_NUMERICS_STRICT = 1 } mmx_numerics;

typedef enum mmx_array { MMX_ARRAY_A = 0, MMX_ARRAY_B = 1, MMX_ARRAY_C = 2, MMX_ARRAY_BT = 3 } mmx_array;

/* Nests in program order (line of the outer `for` in fixtures/matmul.c). */
typedef enum mmx_nest {
  MMX_NEST_INIT_A = 0,    /* :8  genes 0,1   */
  MMX_NEST_INIT_B = 1,    /* :12 genes 2,3   */
  MMX_NEST_ZERO_C = 2,    /* :16 genes 4,5   */
  MMX_NEST_TRANSPOSE = 3, /* :21 genes 6,7   */
  MMX_NEST_MATMUL = 4,    /* :25 genes 8,9,10 */
  MMX_NEST_TRACE = 5      /* :31 gene 11     */
} mmx_nest;

/* How one nest runs under a genome. */
typedef enum mmx_nest_mode {
  MMX_MODE_CPU = 0,       /* no bit of the nest set: host loops                             */
  MMX_MODE_GPU_NEST = 1,  /* depth-0 bit: the whole nest is one kernel launch              */
  MMX_MODE_GPU_INNER = 2, /* depth-1 bit: host runs the outer loop, one launch per iteration (N launches)   */
  MMX_MODE_GPU_INNER2 = 3 /* depth-2 bit (matmul k loop): host runs i and j, one launch per (i,j) (N^2)     */
} mmx_nest_mode;

typedef struct mmx_config {
  uint32_t struct_size;     /* sizeof(mmx_config), for ABI evolution                         */
  int32_t n;                /* matrix size N (fixture default 256, matmul.c:3); >= 1          */
  int32_t dtype;            /* mmx_dtype                                                       */
  int32_t numerics;         /* mmx_numerics                                                    */
  double timeout_s;         /* budget per benchmark run (ToolchainConfig::timeout_s, default 120) */
  int32_t repetitions;      /* runs per genome, median kept (ToolchainConfig::repetitions)     */
  int32_t num_slots;        /* device slots (maps onto the reference's `jobs`)                 */
  const int32_t* devices;   /* CUDA ordinal per slot; NULL = slot s -> device s % deviceCount  */
  int32_t host_threads;     /* threads for CPU-mapped nests; 1 = the reference program         */
  int32_t launch_batching;  /* 1: inner-loop launch trains are submitted as CUDA graphs        */
  int32_t matmul_variant;   /* gene-8 kernel: 0 auto (below N = 1024: DMMA in FP64, FFMA in FP32; from there the INT8 tensor cores
                             * whenever exact 8-bit digit products lose nothing of the product, in the cheapest digit-pair form
                             * that does, chosen on the device from the operands -- the application's inputs at N = 2^p qualify
                             * with 2 x 2 .. 3 x 3 pairs; the result is the exact product rounded once for forms of up to four
                             * levels and faithfully rounded (<= 1 ulp, exact when it fits 53 bits) beyond -- and otherwise DMMA in
                             * FP64, tcgen05 split-TF32 with compensated accumulation in FP32); 1 first SIMT kernel; 2, 4-13 DMMA tile shapes (FP64);
                             * 20, 22 SIMT tile shapes; 30 FP32 tcgen05 split-TF32 at any N % 4 == 0; 31 its wide-tile
                             * uncompensated form; 40 FP64 on the tcgen05 INT8 tensor cores with 7 exact 8-bit slices per operand
                             * whatever the operands (error <= 2e-14 K max|a| max|b|), 41 .. 45 the same with 6 .. 2 slices */
  int32_t warmup;           /* untimed runs per genome before the timed repetitions (default 0) */
  /* Host-side isolation of concurrent measurements (the reference bounds the contention with `jobs`,
   * evaluator.cpp:254-273): with pin_host != 0 (default 1) the CPUs this process may run on -- ordered so that SMT siblings are
   * adjacent, restricted to [host_core_first, host_core_first + host_core_count) of that list when host_core_count > 0 (one
   * process per GPU: each rank passes its own share) -- are split evenly among the slots; a measurement runs on its slot's CPUs
   * only (the calling thread for its duration, and every thread of a CPU-mapped nest's team), so the time of a genome with
   * CPU-mapped nests does not depend on what the other slots are running. */
  int32_t pin_host;
  int32_t host_core_first;
  int32_t host_core_count;
  /* Hopeless runs are given up early (default 1): once a host-side nest or a train of inner-loop launches has run for 20 ms and its
   * measured progress projects at least twice the time the budget has left, the run ends as MMX_TIMEOUT with time_s = timeout_s --
   * exactly the outcome the full wait would produce (evaluator.cpp:103-108) -- at a fraction of the wall cost.  A GA search over
   * this application spends nearly all of its wall time waiting for such runs (the matmul nest on the host at N = 4096 needs a
   * minute per individual).  0: every run is waited for, as the reference's process timeout does. */
  int32_t early_timeout;
} mmx_config;

/* EvaluationOutcome, evaluation.hpp:19-28. */
typedef struct mmx_outcome {
  int32_t status;     /* mmx_status */
  double time_s;      /* Measured: median run time; Timeout: the budget; else 0 */
  double wall_cost_s; /* host wall-clock cost of producing this outcome          */
} mmx_outcome;

/* What the last measurement on a slot did (all repetitions summed unless noted). */
typedef struct mmx_run_stats {
  uint64_t h2d_bytes;       /* per run: bytes the residency planner moved host->device */
  uint64_t d2h_bytes;       /* per run: device->host                                     */
  uint64_t kernel_launches; /* per run: kernels of this library launched                 */
  uint64_t graph_launches;  /* per run: cudaGraphLaunch calls (launch_batching)           */
  double checksum;          /* the value matmul.c:34 would print                          */
  double gpu_ms;            /* last run: CUDA-event time of the whole individual          */
  double host_s;            /* last run: time spent inside CPU-mapped nests               */
  double nest_s[MMX_NUM_NESTS]; /* last run: host wall time attributed to each nest       */
  double host_loadavg;      /* 1-minute load average of the box when the last run started */
  int32_t host_cpus;        /* CPUs the slot is pinned to (0: not pinned)                  */
  int32_t host_first_cpu;   /* the first of them (OS numbering), -1 when not pinned        */
} mmx_run_stats;

/* One step of a plan, as text-free data for tests and reports. */
typedef enum mmx_step_kind {
  MMX_STEP_H2D = 0,      /* whole array host->device  */
  MMX_STEP_D2H = 1,      /* whole array device->host  */
  MMX_STEP_D2H_DIAG = 2, /* only the diagonal of c (strided 2-D copy) for a CPU trace */
  MMX_STEP_CPU = 3,      /* run a nest on the host    */
  MMX_STEP_GPU = 4,      /* run a nest on the device (mode says how many launches) */
  MMX_STEP_D2H_SUM = 5,  /* the scalar checksum back to the host (printf consumer, matmul.c:34) */
  MMX_STEP_H2D_DIAG = 6  /* only the diagonal of c, host->device, for a GPU trace after a CPU matmul */
} mmx_step_kind;

typedef struct mmx_plan_step {
  int32_t kind;      /* mmx_step_kind */
  int32_t nest;      /* mmx_nest for CPU/GPU steps, else -1 */
  int32_t array;     /* mmx_array for transfers, else -1 */
  int32_t mode;      /* mmx_nest_mode for CPU/GPU steps */
  uint64_t bytes;    /* transfer size */
  uint64_t launches; /* kernel launches of a GPU step */
} mmx_plan_step;

#define MMX_MAX_PLAN_STEPS 32

typedef struct mmx_plan_info {
  int32_t feasible;              /* 0 => status would be MMX_COMPILE_ERROR */
  int32_t conflict_nest;         /* first nest with two annotated loops, or -1 */
  int32_t modes[MMX_NUM_NESTS];  /* mmx_nest_mode per nest */
  int32_t num_steps;
  mmx_plan_step steps[MMX_MAX_PLAN_STEPS];
  uint64_t h2d_bytes, d2h_bytes, kernel_launches;
  /* lower bound on transfers for this assignment of nests to sides, computed from the
   * program's producer->consumer edges independently of the planner's state machine */
  uint64_t h2d_lower_bound, d2h_lower_bound;
} mmx_plan_info;

/* One row of the loop catalogue (fixtures/matmul.c). */
typedef struct mmx_loop_info {
  int32_t gene;  /* == loop id */
  int32_t line;  /* line of the `for` keyword in fixtures/matmul.c */
  int32_t depth; /* for-nesting depth */
  int32_t nest;  /* mmx_nest */
  const char* induction;  /* "i", "j", "k" */
  const char* kernel;     /* name of the sm_100a kernel family serving this loop */
} mmx_loop_info;

typedef struct mmx_ctx mmx_ctx;

/* ---- catalogue and planning: pure host code, usable without a GPU ---------------- */

/* Fills up to `cap` rows; returns the catalogue size (12). */
MMX_API int mmx_loop_catalogue(mmx_loop_info* rows, size_t cap);

/* Genome -> plan for matrix size n and dtype, without executing anything.
 * Replaces render_variant (source_model.cpp:347-376) + the compiler's accept/reject
 * (mockacc.cpp:196-221) on this path.  MMX_E_LENGTH if gene_len != 12. */
MMX_API int mmx_plan(const uint8_t* bits, size_t gene_len, int32_t n, int32_t dtype, mmx_plan_info* out);

/* ---- context ----------------------------------------------------------------------- */

MMX_API void mmx_default_config(mmx_config* cfg);
MMX_API int mmx_create(const mmx_config* cfg, mmx_ctx** out);
MMX_API void mmx_destroy(mmx_ctx* ctx);

/* EvalBackend::gene_length (evaluator.hpp:23). */
MMX_API size_t mmx_gene_length(const mmx_ctx* ctx);
MMX_API int mmx_num_slots(const mmx_ctx* ctx);

/* Message of the last failing call on this context (thread-safe snapshot); with ctx ==
 * NULL, the last mmx_create failure of the calling thread. */
MMX_API const char* mmx_last_error(const mmx_ctx* ctx);

/* ---- measurement: the EvalBackend::measure replacement --------------------------- */

/* One real measurement of one genome on one slot (evaluator.hpp:22). */
MMX_API int mmx_measure(mmx_ctx* ctx, int slot, const uint8_t* bits, size_t gene_len, mmx_outcome* out);

/* A whole batch (what Evaluator::evaluate_all hands to its workers, evaluator.cpp:246-276):
 * genomes are pulled dynamically by one worker thread per slot; outs[i] belongs to
 * bits[i*gene_len ..]. Duplicates are measured again -- memoisation lives above this ABI. */
MMX_API int mmx_measure_batch(mmx_ctx* ctx, const uint8_t* bits, size_t n_genomes, size_t gene_len,
                              mmx_outcome* outs);

MMX_API int mmx_last_stats(mmx_ctx* ctx, int slot, mmx_run_stats* out);

/* Un-timed parity hooks: copy an array as the last run on `slot` left it (wherever it is
 * valid) into `host` (n*n elements of the context dtype). */
MMX_API int mmx_fetch_array(mmx_ctx* ctx, int slot, int array, void* host, size_t bytes);

/* The same for a block of rows [row0, row0 + rows) only (`host` receives rows * n elements): parity checks at sizes where the
 * whole array is gigabytes (N = 32768: 8 GiB) compare sampled row blocks against the closed form. */
MMX_API int mmx_fetch_rows(mmx_ctx* ctx, int slot, int array, int row0, int rows, void* host, size_t bytes);

/* ---- single kernels: parity tests and roofline measurement ----------------------- */

/* Put host data into a slot's device array (marks it device-valid). */
MMX_API int mmx_upload_array(mmx_ctx* ctx, int slot, int array, const void* host, size_t bytes);

/* Launch the kernel(s) serving loop `gene` once on the slot's resident device arrays and
 * wait: depth-0 genes run the whole nest; depth-1 genes run iteration i; gene 10 runs
 * iteration (i, j).  For gene 11 the sum is returned in *sum_out (may be NULL otherwise). */
MMX_API int mmx_run_loop(mmx_ctx* ctx, int slot, int gene, int i, int j, double* sum_out);

/* Row-block form of a depth-0 loop (genes 0, 2, 4, 6, 8, 11): only iterations i in [row0, row0+rows)
 * of the loop's outer index.  This is the building block of the row-sharded multi-GPU run (each GPU
 * owns a block of rows of a, c and bt; bt is then all-gathered): SURVEY 8e.  For gene 11 *sum_out
 * receives the partial trace of the block. */
MMX_API int mmx_run_loop_rows(mmx_ctx* ctx, int slot, int gene, int row0, int rows, double* sum_out);

/* Device address of a slot's array (n*n elements of the context dtype), so that a collective library
 * can exchange it in place (the all-gather of bt); valid until mmx_destroy. */
MMX_API int mmx_device_ptr(mmx_ctx* ctx, int slot, int array, void** ptr_out);

/* Which form the last auto-mode launch of gene 8 on this slot took (decided on the device from the operands, csrc/matmul_ozaki.cu;
 * FP64, and FP32 -- where the fallback is split TF32 instead of the FP64 pipe):
 * 100 SA + 10 SB + levels = INT8 tensor cores, digits a_1..a_SA against b_1..b_SB (223 = 2 x 2 pairs, 4 slice products per term;
 * 777 = the widest triangular form, 28), 0 = the FP64 pipe / split TF32 (no form would have been error-free), -1 = no such launch
 * yet / not an auto-mode context with N >= 1024.  Synchronises the slot. */
MMX_API int mmx_gene8_form(mmx_ctx* ctx, int slot, int32_t* form_out);

/* FP64 auto-mode contexts: time the CONTRACTION of gene 8 alone (mmx_time_loop(8) times the whole nest: two slice passes, the
 * contraction, the guarded FP64-pipe launch).  One full launch encodes the operands; each of the `iters` timed launches reuses the
 * digit planes and runs the contraction kernel plus the guarded FP64-pipe launch (c accumulates).  CUDA events on the slot's stream,
 * L2 flushed before each launch when flush_l2 == 1; flush_l2 == 2: the `iters` launches back to back inside ONE event pair (the sustained
 * rate of the kernel; c and the digit planes stay where the cache leaves them); ms_out = mean per launch.  The roofline of the dominant
 * kernel (bench.py). */
MMX_API int mmx_time_gene8_contraction(mmx_ctx* ctx, int slot, int iters, int flush_l2, double* ms_out);

/* The rule behind mmx_gene8_form, evaluated on the host (no device needed): the form the auto launch takes for operands of which
 * `cut` != 0 says some element has bits below its 7th digit, and top_a / top_bt are the highest non-zero 8-bit digits (1-based)
 * anywhere in a / bt.  Returns 100 SA + 10 SB + levels, or 0 for the FP64 pipe. */
MMX_API int mmx_gene8_pick_form(int cut, int top_a, int top_bt);

/* ---- row-sharded run across a group of GPUs (BASELINE.json config 5) -----------------
 * One individual (every nest offloaded) spread over `world` <= 8 members, one device slot each.  Member r
 * owns a contiguous block of rows of a, c and bt (64-row aligned when N allows).  The single exchange of
 * the path -- every member needs all of bt for the contraction -- is fused into the transpose kernel, which
 * stores its rows of bt into every member's bt through peer-mapped pointers; the contraction then walks the
 * column blocks in ring order, waiting per block on the owner's event.  No collective library is involved.
 * The reference has no multi-device mode; the nearest interface is its `jobs` worker pool
 * (evaluator.cpp:246-276), which this does not replace -- it is the large-N extension north_star names. */
typedef struct mmx_shard_handle {
  unsigned char mem[64];   /* cudaIpcMemHandle_t of the member's bt   */
  unsigned char event[64]; /* cudaIpcEventHandle_t of its ready event */
} mmx_shard_handle;

typedef struct mmx_shard_stats {
  int32_t rank, world;
  int32_t row0, rows;     /* the member's block                                             */
  double gpu_ms;          /* CUDA-event time of the member's whole share of the individual   */
  double exchange_ms;     /* the fused transpose + all-gather kernel                         */
  double matmul_ms;       /* the `world` column-block launches of the contraction            */
  uint64_t peer_bytes;    /* bytes this member stored into other members' bt                 */
  double partial_trace;   /* sum of the member's diagonal entries                            */
} mmx_shard_stats;

/* Members in ONE process (a context with one slot per GPU, or several slots on one GPU for tests): binds
 * the slots as ranks 0..world-1 on first use, runs the individual, waits; outs[world] and *checksum (sum of
 * the partial traces in rank order) may be NULL. */
MMX_API int mmx_shard_run_local(mmx_ctx* ctx, const int32_t* slots, int world, mmx_shard_stats* outs, double* checksum);

/* Members in DIFFERENT processes (one process per GPU): each exports its handle, the handles are exchanged by
 * the caller (any transport), then every process binds its slot with the full table.  Per run the caller
 * does: phase1 on every member; a host barrier (each member's ready event must have been recorded before a
 * peer waits on it); phase2 on every member; a host barrier before the next run. */
MMX_API int mmx_shard_export(mmx_ctx* ctx, int slot, mmx_shard_handle* out);
MMX_API int mmx_shard_bind(mmx_ctx* ctx, int slot, int rank, int world, const mmx_shard_handle* handles,
                           const int32_t* local_slots);
MMX_API int mmx_shard_phase1(mmx_ctx* ctx, int slot);
MMX_API int mmx_shard_phase2(mmx_ctx* ctx, int slot, mmx_shard_stats* out);

/* Time `iters` launches of loop `gene` (iteration 0 for inner loops) with CUDA events on
 * the slot's stream; when flush_l2 != 0 a 256 MiB buffer (larger than the 126 MB L2) is read before
 * every timed launch, outside the event bracket, so the cache holds only clean foreign lines.  ms_out receives the mean per launch. */
MMX_API int mmx_time_loop(mmx_ctx* ctx, int slot, int gene, int iters, int flush_l2, double* ms_out);

/* On-device peak probes (roofline denominators the driver file does not carry).
 * kind: 0 copy GB/s, 1 write-only GB/s, 2 FP64 FMA TFLOP/s, 3 FP64 DMMA TFLOP/s,
 *       4 FP32 FMA TFLOP/s, 5 read-only GB/s,
 *       6 / 7 / 8 the tcgen05 tensor pipe's issue peak for kind::i8 (TOP/s), kind::tf32, kind::f16 with bf16 inputs (TFLOP/s):
 *       M = 128 x N = 256 instructions back to back on operands resident in shared memory, one issuing thread per SM */
MMX_API int mmx_peak_probe(int device, int kind, double* value_out);

#ifdef __cplusplus
}
#endif
#endif /* MMX_H_ */
