// executor.cu -- contexts, device slots, plan execution, timing, and the C ABI of include/mmx.h.
//
// One measurement (mmx_measure) is the in-process replacement of ToolchainBackend::measure
// (/root/reference/proj/src/evaluator.cpp:61-142): plan the genome, run the plan `repetitions`
// times, take the median (evaluator.cpp:133-136), map failures to outcomes:
//     infeasible genome       -> CompileError, time 0          (evaluator.cpp:87-91)
//     run over timeout_s      -> Timeout, time = budget        (evaluator.cpp:103-108)
//     CUDA failure / t <= 0   -> RuntimeError                  (evaluator.cpp:109-113,125-129)
// The timed region of a run starts with every array invalid on both sides (a fresh process, as
// in the reference) and ends when the checksum is on the host; allocation happens before it
// (the program's arrays are static storage, matmul.c:5).
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "host_loops.hpp"
#include "kernels.cuh"
#include "mmx.h"
#include "plan.hpp"

namespace mmx {
namespace {

thread_local std::string g_create_error;

struct Train {  // a captured train of K inner-loop launches + the counter bump
  cudaGraphExec_t exec = nullptr;
  int k = 0;
};

struct Slot {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t cur = nullptr;       // the stream launch_gene enqueues on: `stream`, or a side lane while a forked graph is captured
  cudaStream_t lane[2] = {};        // side lanes of the whole-individual graph (init-a, zero-c beside init-b -> transpose)
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {};
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  void* d_arr[MMX_NUM_ARRAYS] = {};
  void* h_arr[MMX_NUM_ARRAYS] = {};  // pinned, allocated on first need
  void* d_sum = nullptr;
  void* h_sum = nullptr;  // pinned, 16 bytes
  int* d_iter = nullptr;
  void* d_scrub = nullptr;
  std::size_t scrub_bytes = 0;
  void* d_scratch = nullptr;  // operands re-encoded for the tensor-core contractions (FP32: matmul_tc.cu; FP64: matmul_ozaki.cu)
  bool gene8_form_valid = false;  // FP64 auto mode (mmx_time_gene8_contraction applies)
  int* gene8_form_word = nullptr;  // auto mode, either precision: the device word mmx_gene8_form reads
  bool host_valid[MMX_NUM_ARRAYS] = {};
  bool dev_valid[MMX_NUM_ARRAYS] = {};
  bool host_diag_only = false;  // host c holds only its diagonal
  // Digit planes of gene 8's operands (auto mode, csrc/ozaki_digits.cuh).  When a plan runs the matmul nest as one launch, the
  // kernels that PRODUCE a and bt (init-a fill, transpose) write the planes from their registers (`fuse_planes`), and gene 8 skips
  // the slice pass of every operand whose planes are still valid.  Any other write to the array drops the flag.
  void* oz_planes = nullptr;       // base of the planes inside d_scratch (FP32: behind the split-TF32 area)
  bool fuse_planes = false;        // set per plan / per API call
  bool planes_a_valid = false, planes_bt_valid = false;
  bool b_colexp_valid = false;     // the exponents of bt's rows were written by the init-b kernel (closed form of its own output)
  // init-b inside the transpose: a plan that runs both nests whole on the device, with nothing touching b in between, lets the
  // transpose kernel COMPUTE its tiles of b (and store them) instead of reading them back (launch_fill_b_transpose_planes).
  // defer_b: the sequence allows it (begin_sequence); b_pending: init-b has been asked for and b is not written yet
  bool defer_b = false;
  bool b_pending = false;
  // whole-individual graphs only, opt-in (MMX_B_BESIDE=1; measured slower on average, see prepare_plan_graph): nothing on the device
  // reads b, so its 8 N^2 bytes are written by a plain fill on a side lane BESIDE the contraction (HBM is nearly idle there, and a fill CTA fits next to a contraction CTA: 32 x 256 registers, no shared
  // memory) instead of by the transpose.  b_beside: the capture asks for it; b_unwritten: the transpose left b to that fill
  bool b_beside = false;
  bool b_unwritten = false;
  bool c_zero = false;             // the zero-c kernel filled c on the device and nothing has written c since (kCIsZero)
  std::map<int, Train> trains;  // by gene
  struct PlanGraph {
    cudaGraphExec_t exec = nullptr;
    bool planes_a = false, planes_bt = false, colexp = false;  // the flags as the captured sequence leaves them
  };
  std::map<unsigned, PlanGraph> plan_graphs;  // by genome mask: whole device-only individuals
  std::vector<int> cpus;  // pin_host: the CPUs this slot's measurements run on (OS numbering); empty = not pinned
  mmx_run_stats stats{};
  std::mutex mu;
  // row-sharded group membership (mmx_shard_*): this slot is member `shard_rank` of `shard_world`
  int shard_rank = -1, shard_world = 0;
  void* peer_bt[kMaxPeers] = {};          // bt of every member as seen from this device (own array at [shard_rank])
  cudaEvent_t peer_ready[kMaxPeers] = {}; // member r's "my rows of bt are stored everywhere" event
  bool peer_ipc[kMaxPeers] = {};          // opened from another process's handle: must be closed / destroyed here
  cudaEvent_t ev_ready = nullptr;         // interprocess-capable, no timing
  cudaEvent_t ev_x0 = nullptr, ev_x1 = nullptr, ev_m0 = nullptr, ev_m1 = nullptr;
};

}  // namespace
}  // namespace mmx

struct mmx_ctx {
  mmx_config cfg{};
  std::vector<int> devices;
  std::vector<std::unique_ptr<mmx::Slot>> slots;
  mutable std::mutex err_mu;
  std::string error;
  mutable std::string error_snapshot;

  void set_error(const std::string& e) {
    std::lock_guard<std::mutex> g(err_mu);
    error = e;
  }
};

namespace mmx {
namespace {

using Seconds = std::chrono::duration<double>;

inline double since(Clock::time_point t0) { return Seconds(Clock::now() - t0).count(); }

#define MMX_CUDA(ctx, call)                                                                      \
  do {                                                                                           \
    cudaError_t e__ = (call);                                                                    \
    if (e__ != cudaSuccess) {                                                                    \
      (ctx)->set_error(std::string(#call) + ": " + cudaGetErrorString(e__));                     \
      return e__ == cudaErrorMemoryAllocation ? MMX_E_NOMEM : MMX_E_CUDA;                        \
    }                                                                                            \
  } while (0)

// The CPUs this process may run on, ordered so that SMT siblings are adjacent (a slot's share is then made of whole cores
// wherever the split allows): sorted by (lowest sibling id, own id) as sysfs reports the topology; OS order where it does not.
std::vector<int> allowed_cpus_by_core() {
  cpu_set_t set;
  CPU_ZERO(&set);
  std::vector<int> cpus;
  if (sched_getaffinity(0, sizeof(set), &set) != 0) return cpus;
  std::vector<std::pair<int, int>> keyed;
  for (int c = 0; c < CPU_SETSIZE; ++c) {
    if (!CPU_ISSET(c, &set)) continue;
    int first = c;
    std::ifstream f("/sys/devices/system/cpu/cpu" + std::to_string(c) + "/topology/thread_siblings_list");
    if (f) {
      int v = 0;
      if (f >> v) first = v;  // "0,8" or "0-1": the list starts with the lowest sibling
    }
    keyed.emplace_back(first, c);
  }
  std::sort(keyed.begin(), keyed.end());
  for (const auto& kc : keyed) cpus.push_back(kc.second);
  return cpus;
}

// Pins the calling thread to a slot's CPUs for the duration of a measurement and restores its mask afterwards.
class ScopedAffinity {
 public:
  explicit ScopedAffinity(const std::vector<int>& cpus) {
    if (cpus.empty()) return;
    if (pthread_getaffinity_np(pthread_self(), sizeof(old_), &old_) != 0) return;
    cpu_set_t set;
    CPU_ZERO(&set);
    for (int c : cpus) CPU_SET(c, &set);
    active_ = pthread_setaffinity_np(pthread_self(), sizeof(set), &set) == 0;
  }
  ~ScopedAffinity() {
    if (active_) pthread_setaffinity_np(pthread_self(), sizeof(old_), &old_);
  }
  ScopedAffinity(const ScopedAffinity&) = delete;
  ScopedAffinity& operator=(const ScopedAffinity&) = delete;

 private:
  cpu_set_t old_;
  bool active_ = false;
};

std::size_t matrix_bytes(const mmx_ctx* ctx) {
  return static_cast<std::size_t>(ctx->cfg.n) * ctx->cfg.n * elem_size(ctx->cfg.dtype);
}

int ensure_host(mmx_ctx* ctx, Slot& s, int array) {
  if (s.h_arr[array] != nullptr) return MMX_OK;
  MMX_CUDA(ctx, cudaHostAlloc(&s.h_arr[array], matrix_bytes(ctx), cudaHostAllocDefault));
  return MMX_OK;
}

// ---- kernel dispatch by gene --------------------------------------------------------------------

// rows [row0, row0+rows) of the loop's outer index for depth-0 genes (the whole nest: 0, n)
template <typename T>
cudaError_t launch_gene(const mmx_ctx* ctx, Slot& s, int gene, IterRef iter, int row0, int rows) {
  const int n = ctx->cfg.n;
  const bool strict = ctx->cfg.numerics == MMX_NUMERICS_STRICT;
  T* a = static_cast<T*>(s.d_arr[MMX_ARRAY_A]);
  T* b = static_cast<T*>(s.d_arr[MMX_ARRAY_B]);
  T* c = static_cast<T*>(s.d_arr[MMX_ARRAY_C]);
  T* bt = static_cast<T*>(s.d_arr[MMX_ARRAY_BT]);
  // fused producers: whole-nest launches of a plan whose matmul nest is one launch, auto mode, sizes without plane padding
  const bool fuse = s.fuse_planes && s.oz_planes != nullptr && row0 == 0 && rows == n && ozaki_fusable(n);
  switch (gene) {
    case 0:
      s.planes_a_valid = false;
      if (fuse) {
        const cudaError_t e = launch_fill_a_planes<T>(a, n, matmul_ozaki_operand(s.oz_planes, n, 0), s.cur);
        s.planes_a_valid = e == cudaSuccess;
        return e;
      }
      return launch_fill2d<T>(FILL_INIT_A, a, n, row0, rows, s.cur);
    case 1: s.planes_a_valid = false; return launch_fill_row<T>(FILL_INIT_A, a, n, iter, s.cur);
    case 2:
      s.b_colexp_valid = false;
      s.b_pending = false;
      if (fuse && s.defer_b) {
        const cudaError_t e = launch_b_colexp<T>(n, matmul_ozaki_operand(s.oz_planes, n, 1).exps, s.cur);
        s.b_colexp_valid = s.b_pending = e == cudaSuccess;
        return e;
      }
      if (fuse) {
        const cudaError_t e = launch_fill_b_colexp<T>(b, n, matmul_ozaki_operand(s.oz_planes, n, 1).exps, s.cur);
        s.b_colexp_valid = e == cudaSuccess;
        return e;
      }
      return launch_fill2d<T>(FILL_INIT_B, b, n, row0, rows, s.cur);
    case 3: s.b_colexp_valid = s.b_pending = false; return launch_fill_row<T>(FILL_INIT_B, b, n, iter, s.cur);
    case 4: {
      const cudaError_t e = launch_fill2d<T>(FILL_ZERO, c, n, row0, rows, s.cur);
      s.c_zero = e == cudaSuccess && row0 == 0 && rows == n;
      return e;
    }
    case 5: s.c_zero = false; return launch_fill_row<T>(FILL_ZERO, c, n, iter, s.cur);
    case 6:
      s.planes_bt_valid = false;
      if (s.b_pending) {
        s.b_pending = false;
        if (fuse && s.b_colexp_valid) {
          const cudaError_t e = launch_fill_b_transpose_planes<T>(s.b_beside ? nullptr : b, bt, n, matmul_ozaki_operand(s.oz_planes, n, 1), s.cur);
          s.planes_bt_valid = e == cudaSuccess;
          s.b_unwritten = s.b_beside && e == cudaSuccess;
          return e;
        }
        // (not reached while defer_b and this launch agree on `fuse`; kept so that b is never left unwritten)
        if (const cudaError_t e = launch_fill2d<T>(FILL_INIT_B, b, n, 0, n, s.cur); e != cudaSuccess) return e;
        s.b_colexp_valid = false;
      }
      if (fuse && s.b_colexp_valid) {
        const cudaError_t e = launch_transpose_planes<T>(bt, b, n, matmul_ozaki_operand(s.oz_planes, n, 1), s.cur);
        s.planes_bt_valid = e == cudaSuccess;
        return e;
      }
      return launch_transpose<T>(bt, b, n, row0, rows, s.cur);
    case 7:
      s.planes_bt_valid = false;
      if (s.b_pending) {  // (defer_b is only set for plans whose transpose nest is gene 6; kept so that b is never left unwritten)
        s.b_pending = false;
        if (const cudaError_t e = launch_fill2d<T>(FILL_INIT_B, b, n, 0, n, s.cur); e != cudaSuccess) return e;
      }
      return launch_transpose_row<T>(bt, b, n, iter, s.cur);
    case 8: {
      int variant = ctx->cfg.matmul_variant;  // 0 = auto (matmul.cu)
      if (variant == 0 && row0 == 0 && rows == n && s.oz_planes != nullptr) {
        if (s.planes_a_valid) variant |= kReuseOperandA;
        if (s.planes_bt_valid) variant |= kReuseOperandBt;
        if (s.c_zero) variant |= kCIsZero;
        else s.b_colexp_valid = false;  // the slice pass of bt writes its own row exponents
      } else {
        s.b_colexp_valid = false;  // row / column blocks re-encode parts of the planes
      }
      // one consumer per encoding: the next launch of gene 8 encodes again unless a producer has rewritten the planes by then
      // (mmx_time_loop(8) therefore times the whole nest, slice passes included, whatever ran before)
      s.planes_a_valid = s.planes_bt_valid = false;
      s.c_zero = false;
      return launch_matmul<T>(c, a, bt, n, row0, rows, 0, n, strict, variant, s.d_scratch, s.cur);
    }
    case 9: s.c_zero = false; return launch_gemv_row<T>(c, a, bt, n, iter, strict, s.cur);
    case 10: s.c_zero = false; return launch_dot<T>(c, a, bt, n, iter, strict, s.cur);
    case 11: return launch_trace<T>(static_cast<T*>(s.d_sum), c, n, row0, rows, strict, s.cur);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gene_rows(const mmx_ctx* ctx, Slot& s, int gene, IterRef iter, int row0, int rows) {
  return ctx->cfg.dtype == MMX_F64 ? launch_gene<double>(ctx, s, gene, iter, row0, rows)
                                   : launch_gene<float>(ctx, s, gene, iter, row0, rows);
}

cudaError_t launch_gene_any(const mmx_ctx* ctx, Slot& s, int gene, IterRef iter) {
  return launch_gene_rows(ctx, s, gene, iter, 0, ctx->cfg.n);
}

// Start of a sequence of launches (a plan run, a capture, a single-kernel API call): no planes are valid yet, and the producers
// of a and bt write them iff the matmul nest will consume them as ONE launch (MMX_FUSE_PLANES=0 switches the fusion off: A/B runs)
void begin_sequence(Slot& s, bool matmul_is_one_launch, bool plan_allows_defer_b = false) {
  static const bool enabled = [] { const char* e = getenv("MMX_FUSE_PLANES"); return e == nullptr || atoi(e) != 0; }();
  static const bool defer_enabled = [] { const char* e = getenv("MMX_FUSE_INIT_B"); return e == nullptr || atoi(e) != 0; }();  // 0: A/B runs
  s.fuse_planes = enabled && matmul_is_one_launch && s.oz_planes != nullptr;
  s.defer_b = s.fuse_planes && defer_enabled && plan_allows_defer_b;
  s.b_pending = false;
  s.b_beside = s.b_unwritten = false;
  s.planes_a_valid = s.planes_bt_valid = s.b_colexp_valid = false;
  s.c_zero = false;
}

// gene that serves `nest` in `mode`
int gene_of(int nest, int mode) { return kNests[nest].first_gene + (mode - MMX_MODE_GPU_NEST); }

constexpr int kTrainLength = 512;

// Capture (once per slot and gene) a graph of k launches of an inner-loop gene whose iteration
// index is `*d_iter + node`, followed by `*d_iter += k`.  This is the genome's "compile step":
// it runs before the timed region.
cudaError_t prepare_train(mmx_ctx* ctx, Slot& s, int gene, long long total) {
  if (!ctx->cfg.launch_batching || total < 64) return cudaSuccess;
  const int k = static_cast<int>(std::min<long long>(total, kTrainLength));
  Train& tr = s.trains[gene];
  if (tr.exec != nullptr && tr.k == k) return cudaSuccess;
  if (tr.exec) cudaGraphExecDestroy(tr.exec);
  tr.exec = nullptr;
  tr.k = 0;
  cudaGraph_t graph = nullptr;
  // first-use work (cudaFuncSetAttribute in launch_gemv_row, lazy module load) must not happen inside a capture: one plain launch
  // of iteration 0 first -- harmless, every run re-initialises its arrays before the train runs
  cudaError_t e = launch_gene_any(ctx, s, gene, IterRef{nullptr, 0});
  if (e == cudaSuccess) e = cudaStreamSynchronize(s.stream);
  if (e != cudaSuccess) return e;
  e = cudaStreamBeginCapture(s.stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return e;
  for (int q = 0; q < k && e == cudaSuccess; ++q) e = launch_gene_any(ctx, s, gene, IterRef{s.d_iter, q});
  if (e == cudaSuccess) e = launch_advance(s.d_iter, k, s.stream);
  const cudaError_t e2 = cudaStreamEndCapture(s.stream, &graph);
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&tr.exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (e == cudaSuccess) tr.k = k;
  return e;
}

// Submit `total` launches of an inner-loop gene (iterations 0..total-1): whole trains as graph
// launches when one was prepared, the remainder (or everything) as plain stream launches.
// Returns cudaSuccess, an error, or sets *timed_out.
cudaError_t run_train(mmx_ctx* ctx, Slot& s, int gene, long long total, const Deadline& dl, bool* timed_out,
                      std::uint64_t* graph_launches) {
  cudaError_t e = cudaSuccess;
  long long done = 0;
  auto it_train = s.trains.find(gene);
  if (ctx->cfg.launch_batching && it_train != s.trains.end() && it_train->second.exec != nullptr &&
      it_train->second.k <= total) {
    const Train& tr = it_train->second;
    if ((e = cudaMemsetAsync(s.d_iter, 0, sizeof(int), s.stream)) != cudaSuccess) return e;
    const long long trains = total / tr.k;
    const Clock::time_point started = Clock::now();
    for (long long t = 0; t < trains; ++t) {
      if ((e = cudaGraphLaunch(tr.exec, s.stream)) != cudaSuccess) return e;
      ++*graph_launches;
      done += tr.k;
      // keep the queue shallow enough that a timeout is noticed within a few trains
      if ((t & 7) == 7) {
        if ((e = cudaStreamSynchronize(s.stream)) != cudaSuccess) return e;
        if (dl.expired() || dl.hopeless(started, done, total)) {
          *timed_out = true;
          return cudaSuccess;
        }
      }
    }
  }
  const Clock::time_point started_plain = Clock::now();
  for (long long it = done; it < total; ++it) {
    if ((e = launch_gene_any(ctx, s, gene, IterRef{nullptr, static_cast<int>(it)})) != cudaSuccess) return e;
    if (((it - done) & 1023) == 1023) {
      if ((e = cudaStreamSynchronize(s.stream)) != cudaSuccess) return e;
      if (dl.expired() || dl.hopeless(started_plain, it - done + 1, total - done)) {
        *timed_out = true;
        return cudaSuccess;
      }
    }
  }
  return cudaSuccess;
}

template <typename T>
bool run_host_nest(const mmx_ctx* ctx, Slot& s, int nest, int row0, int row1, const Deadline& dl, double* checksum) {
  const int n = ctx->cfg.n;
  HostTeam th;
  th.threads = ctx->cfg.host_threads;
  th.cpus = s.cpus.empty() ? nullptr : s.cpus.data();
  th.ncpus = static_cast<int>(s.cpus.size());
  T* a = static_cast<T*>(s.h_arr[MMX_ARRAY_A]);
  T* b = static_cast<T*>(s.h_arr[MMX_ARRAY_B]);
  T* c = static_cast<T*>(s.h_arr[MMX_ARRAY_C]);
  T* bt = static_cast<T*>(s.h_arr[MMX_ARRAY_BT]);
  switch (nest) {
    case MMX_NEST_INIT_A: return host_init_a<T>(a, n, row0, row1, th, dl);
    case MMX_NEST_INIT_B: return host_init_b<T>(b, n, row0, row1, th, dl);
    case MMX_NEST_ZERO_C: return host_zero_c<T>(c, n, row0, row1, th, dl);
    case MMX_NEST_TRANSPOSE: return host_transpose<T>(bt, b, n, row0, row1, th, dl);
    case MMX_NEST_MATMUL: return host_matmul<T>(c, a, bt, n, row0, row1, th, dl);
    case MMX_NEST_TRACE: *checksum = host_trace<T>(c, n); return true;
    default: return false;
  }
}

struct RunResult {
  int status = MMX_RUNTIME_ERROR;
  double time_s = 0.0;
};

// arrays a nest writes (whole array) -- for the validity bookkeeping mmx_fetch_array relies on
int written_array(int nest) {
  switch (nest) {
    case MMX_NEST_INIT_A: return MMX_ARRAY_A;
    case MMX_NEST_INIT_B: return MMX_ARRAY_B;
    case MMX_NEST_ZERO_C: return MMX_ARRAY_C;
    case MMX_NEST_TRANSPOSE: return MMX_ARRAY_BT;
    case MMX_NEST_MATMUL: return MMX_ARRAY_C;
    default: return -1;
  }
}

// bit q set: the nest reads or writes array q
unsigned nest_arrays(int nest) {
  switch (nest) {
    case MMX_NEST_INIT_A: return 1u << MMX_ARRAY_A;
    case MMX_NEST_INIT_B: return 1u << MMX_ARRAY_B;
    case MMX_NEST_ZERO_C: return 1u << MMX_ARRAY_C;
    case MMX_NEST_TRANSPOSE: return 1u << MMX_ARRAY_B | 1u << MMX_ARRAY_BT;
    case MMX_NEST_MATMUL: return 1u << MMX_ARRAY_A | 1u << MMX_ARRAY_BT | 1u << MMX_ARRAY_C;
    case MMX_NEST_TRACE: return 1u << MMX_ARRAY_C;
    default: return 0;
  }
}

// bit q set: step `st` touches array q (bit 4 = the checksum scalar)
unsigned step_arrays(const mmx_plan_step& st) {
  switch (st.kind) {
    case MMX_STEP_CPU:
    case MMX_STEP_GPU: return nest_arrays(st.nest) | (st.nest == MMX_NEST_TRACE ? 1u << 4 : 0u);
    case MMX_STEP_D2H_SUM: return 1u << 4;
    default: return st.array >= 0 ? 1u << st.array : 0u;
  }
}

// init-b may be produced inside the transpose kernel: both nests run whole on the device, init-b first, and no step between them
// touches b (no copy of b, no host nest on it)
bool can_defer_b(const mmx_plan_info& plan) {
  int si = -1;
  for (int k = 0; k < plan.num_steps; ++k) {
    const mmx_plan_step& st = plan.steps[k];
    const bool whole_gpu = st.kind == MMX_STEP_GPU && st.mode == MMX_MODE_GPU_NEST;
    if (si < 0) {
      if (whole_gpu && st.nest == MMX_NEST_INIT_B) si = k;
      else if (step_arrays(st) >> MMX_ARRAY_B & 1u) return false;
      continue;
    }
    if (st.nest == MMX_NEST_TRANSPOSE && st.kind == MMX_STEP_GPU) return whole_gpu;
    if (step_arrays(st) >> MMX_ARRAY_B & 1u) return false;
  }
  return false;
}

// A plan whose every step is a whole-nest kernel (plus the checksum copy) has no host work
// between launches: the individual is captured once as a CUDA graph (its "compile step", outside
// the timed region) and replayed with a single launch -- this is what makes the N=256 fixture size
// launch-latency-bound on one graph launch instead of six kernel launches.
bool device_only(const mmx_plan_info& plan) {
  for (int si = 0; si < plan.num_steps; ++si) {
    const mmx_plan_step& st = plan.steps[si];
    const bool ok = (st.kind == MMX_STEP_GPU && st.mode == MMX_MODE_GPU_NEST) || st.kind == MMX_STEP_D2H_SUM;
    if (!ok) return false;
  }
  return plan.num_steps > 0;
}

cudaError_t prepare_plan_graph(mmx_ctx* ctx, Slot& s, const mmx_plan_info& plan, unsigned mask) {
  if (!ctx->cfg.launch_batching || !device_only(plan) || s.plan_graphs.count(mask)) return cudaSuccess;
  // first-use work (function attributes, module load) must not happen inside a capture
  cudaError_t e = cudaSuccess;
  const bool one_launch = plan.modes[MMX_NEST_MATMUL] == MMX_MODE_GPU_NEST;
  begin_sequence(s, one_launch, can_defer_b(plan));
  for (int si = 0; si < plan.num_steps && e == cudaSuccess; ++si)
    if (plan.steps[si].kind == MMX_STEP_GPU) e = launch_gene_any(ctx, s, gene_of(plan.steps[si].nest, plan.steps[si].mode), IterRef{nullptr, 0});
  if (e == cudaSuccess) e = cudaStreamSynchronize(s.stream);
  if (e != cudaSuccess) return e;
  cudaGraph_t graph = nullptr;
  begin_sequence(s, one_launch, can_defer_b(plan));
  if ((e = cudaStreamBeginCapture(s.stream, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) return e;
  // opt-in (MMX_B_BESIDE=1): the best of five individuals gains 1 %, but the mean over individuals back to back LOSES 3 % (293.1 against
  // 284.5 us at N = 4096, tools/e2e_overhead.py) -- the fill's stores share the L2 crossbar the contraction is bound by
  static const bool beside_enabled = [] { const char* v = getenv("MMX_B_BESIDE"); return v != nullptr && atoi(v) != 0; }();
  bool b_lane_open = false;
  const std::size_t esz = elem_size(ctx->cfg.dtype);
  // The program's data flow leaves three independent chains in front of the matmul nest: init-a, init-b -> transpose, zero-c
  // (derive_dataflow finds the same edges in the source).  In the graph they are three branches: init-a and zero-c
  // run on side lanes beside the longest chain and join before the contraction, so the issue-bound producers (the fill and the
  // transpose that also emit digit planes) overlap the bandwidth-bound ones.  MMX_GRAPH_FORK=0 keeps one chain (A/B runs).
  static const bool fork_enabled = [] { const char* v = getenv("MMX_GRAPH_FORK"); return v == nullptr || atoi(v) != 0; }();
  const bool fork = fork_enabled;
  bool forked = false, joined = false;
  for (int si = 0; si < plan.num_steps && e == cudaSuccess; ++si) {
    const mmx_plan_step& st = plan.steps[si];
    if (st.kind != MMX_STEP_GPU) {
      e = cudaMemcpyAsync(s.h_sum, s.d_sum, esz, cudaMemcpyDeviceToHost, s.stream);
      continue;
    }
    if (fork && !forked) {
      e = cudaEventRecord(s.ev_fork, s.stream);
      for (int q = 0; q < 2 && e == cudaSuccess; ++q) e = cudaStreamWaitEvent(s.lane[q], s.ev_fork, 0);
      forked = true;
      if (e != cudaSuccess) break;
    }
    if (fork && !joined && (st.nest == MMX_NEST_MATMUL || st.nest == MMX_NEST_TRACE)) {
      for (int q = 0; q < 2 && e == cudaSuccess; ++q) {
        e = cudaEventRecord(s.ev_join[q], s.lane[q]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s.stream, s.ev_join[q], 0);
      }
      joined = true;
      if (e != cudaSuccess) break;
    }
    if (fork && !joined && st.nest == MMX_NEST_INIT_A) s.cur = s.lane[0];
    if (fork && !joined && st.nest == MMX_NEST_ZERO_C) s.cur = s.lane[1];
    s.b_beside = fork && beside_enabled && s.defer_b && !joined;
    if (fork && joined && s.b_unwritten) {
      // the transpose left b to us: a plain init-b fill on lane 0, released together with this step (the contraction) and joined
      // at the end of the graph
      s.b_unwritten = false;
      e = cudaEventRecord(s.ev_fork, s.stream);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s.lane[0], s.ev_fork, 0);
      const int nn = ctx->cfg.n;
      if (e == cudaSuccess)
        e = ctx->cfg.dtype == MMX_F64 ? launch_fill2d<double>(FILL_INIT_B, static_cast<double*>(s.d_arr[MMX_ARRAY_B]), nn, 0, nn, s.lane[0])
                                      : launch_fill2d<float>(FILL_INIT_B, static_cast<float*>(s.d_arr[MMX_ARRAY_B]), nn, 0, nn, s.lane[0]);
      b_lane_open = true;
      if (e != cudaSuccess) break;
    }
    e = launch_gene_any(ctx, s, gene_of(st.nest, st.mode), IterRef{nullptr, 0});
    s.cur = s.stream;
  }
  s.b_beside = false;
  if (s.b_unwritten) {  // (no step followed the join: not a plan this path sees -- b is written all the same)
    s.b_unwritten = false;
    const int nn = ctx->cfg.n;
    const cudaError_t eb = ctx->cfg.dtype == MMX_F64 ? launch_fill2d<double>(FILL_INIT_B, static_cast<double*>(s.d_arr[MMX_ARRAY_B]), nn, 0, nn, s.stream)
                                                     : launch_fill2d<float>(FILL_INIT_B, static_cast<float*>(s.d_arr[MMX_ARRAY_B]), nn, 0, nn, s.stream);
    if (e == cudaSuccess) e = eb;
  }
  if (b_lane_open) {  // the fill of b rejoins the origin stream
    cudaEventRecord(s.ev_join[0], s.lane[0]);
    cudaStreamWaitEvent(s.stream, s.ev_join[0], 0);
  }
  if (forked && !joined) {  // (a device-only plan always has the matmul nest; kept for safety: every lane must rejoin the origin stream)
    for (int q = 0; q < 2; ++q) {
      cudaEventRecord(s.ev_join[q], s.lane[q]);
      cudaStreamWaitEvent(s.stream, s.ev_join[q], 0);
    }
  }
  s.cur = s.stream;
  const cudaError_t e2 = cudaStreamEndCapture(s.stream, &graph);
  if (e == cudaSuccess) e = e2;
  Slot::PlanGraph pg;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&pg.exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  pg.planes_a = s.planes_a_valid;
  pg.planes_bt = s.planes_bt_valid;
  pg.colexp = s.b_colexp_valid;
  if (e == cudaSuccess) s.plan_graphs[mask] = pg;
  return e;
}

// One benchmark run of a feasible plan on a prepared slot.
RunResult run_plan_once(mmx_ctx* ctx, Slot& s, const mmx_plan_info& plan, const Slot::PlanGraph* whole) {
  RunResult rr;
  const std::size_t mbytes = matrix_bytes(ctx);
  const std::size_t esz = elem_size(ctx->cfg.dtype);
  const std::size_t n = static_cast<std::size_t>(ctx->cfg.n);
  const double budget = ctx->cfg.timeout_s;
  for (int q = 0; q < MMX_NUM_ARRAYS; ++q) s.host_valid[q] = s.dev_valid[q] = false;
  s.host_diag_only = false;
  s.stats.host_s = 0.0;
  {
    // the box's load matters to plans with host-side nests; an all-device plan does not pay the /proc read (microseconds per run)
    bool host_work = false;
    for (int si = 0; si < plan.num_steps; ++si) host_work = host_work || plan.steps[si].kind == MMX_STEP_CPU;
    double load = 0.0;
    s.stats.host_loadavg = (host_work && getloadavg(&load, 1) == 1) ? load : -1.0;
  }
  s.stats.host_cpus = static_cast<int32_t>(s.cpus.size());
  s.stats.host_first_cpu = s.cpus.empty() ? -1 : s.cpus.front();
  s.stats.graph_launches = 0;
  for (double& x : s.stats.nest_s) x = 0.0;
  double checksum = 0.0;
  bool any_gpu = false, timed_out = false, sum_on_device = false;
  cudaError_t e = cudaSuccess;

  begin_sequence(s, plan.modes[MMX_NEST_MATMUL] == MMX_MODE_GPU_NEST, can_defer_b(plan));
  const Clock::time_point t0 = Clock::now();
  const Deadline dl{t0 + std::chrono::duration_cast<Clock::duration>(Seconds(budget)), ctx->cfg.early_timeout != 0};
  e = cudaEventRecord(s.ev_begin, s.stream);

  if (whole != nullptr) {
    if (e == cudaSuccess) e = cudaGraphLaunch(whole->exec, s.stream);
    s.planes_a_valid = whole->planes_a;
    s.planes_bt_valid = whole->planes_bt;
    s.b_colexp_valid = whole->colexp;
    s.stats.graph_launches = 1;
    any_gpu = true;
    for (int si = 0; si < plan.num_steps; ++si) {
      const mmx_plan_step& st = plan.steps[si];
      if (st.kind != MMX_STEP_GPU) continue;
      const int w = written_array(st.nest);
      if (w >= 0) s.dev_valid[w] = true;
      if (st.nest == MMX_NEST_TRACE) sum_on_device = true;
    }
  }
  // Steps run in plan order with two exceptions that keep the device and the bus busy while a CPU-mapped nest computes
  // (MMX_OVERLAP=0 switches both off: A/B runs):
  //  * hoisting: before a CPU nest starts, every later whole-nest GPU step that touches none of the arrays of the steps it would
  //    overtake is enqueued (launches are asynchronous: they run beside the host loop);
  //  * streaming: when the array a CPU nest writes is copied to the device later in the plan (and nothing in between touches it),
  //    the nest runs block by block and each finished block of rows is copied at once -- only the last block's transfer is left
  //    when the nest ends.  Bytes moved are the plan's: the same transfer, cut into pieces.
  static const bool overlap_enabled = [] { const char* v = getenv("MMX_OVERLAP"); return v == nullptr || atoi(v) != 0; }();
  bool issued[MMX_MAX_PLAN_STEPS] = {};
  auto run_gpu_step = [&](const mmx_plan_step& st) {
    any_gpu = true;
    const int gene = gene_of(st.nest, st.mode);
    if (st.mode == MMX_MODE_GPU_NEST) {
      e = launch_gene_any(ctx, s, gene, IterRef{nullptr, 0});
    } else {
      e = run_train(ctx, s, gene, static_cast<long long>(st.launches), dl, &timed_out, &s.stats.graph_launches);
    }
    const int w = written_array(st.nest);
    if (w >= 0) {
      s.dev_valid[w] = true;
      s.host_valid[w] = false;
    }
    if (st.nest == MMX_NEST_TRACE) sum_on_device = true;
  };
  for (int si = 0; whole == nullptr && si < plan.num_steps && e == cudaSuccess && !timed_out; ++si) {
    if (issued[si]) continue;
    const mmx_plan_step& st = plan.steps[si];
    const Clock::time_point ts = Clock::now();
    switch (st.kind) {
      case MMX_STEP_H2D:
        e = cudaMemcpyAsync(s.d_arr[st.array], s.h_arr[st.array], mbytes, cudaMemcpyHostToDevice, s.stream);
        s.dev_valid[st.array] = true;
        if (st.array == MMX_ARRAY_A) s.planes_a_valid = false;
        if (st.array == MMX_ARRAY_BT) s.planes_bt_valid = false;
        if (st.array == MMX_ARRAY_B) s.b_colexp_valid = false;
        if (st.array == MMX_ARRAY_C) s.c_zero = false;
        any_gpu = true;
        break;
      case MMX_STEP_D2H:
        e = cudaMemcpyAsync(s.h_arr[st.array], s.d_arr[st.array], mbytes, cudaMemcpyDeviceToHost, s.stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s.stream);  // the host consumes it next
        s.host_valid[st.array] = true;
        any_gpu = true;
        break;
      case MMX_STEP_D2H_DIAG:
        e = cudaMemcpy2DAsync(s.h_arr[st.array], (n + 1) * esz, s.d_arr[st.array], (n + 1) * esz, esz, n,
                              cudaMemcpyDeviceToHost, s.stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s.stream);
        s.host_diag_only = true;
        any_gpu = true;
        break;
      case MMX_STEP_H2D_DIAG:
        e = cudaMemcpy2DAsync(s.d_arr[st.array], (n + 1) * esz, s.h_arr[st.array], (n + 1) * esz, esz, n,
                              cudaMemcpyHostToDevice, s.stream);
        if (st.array == MMX_ARRAY_C) s.c_zero = false;
        any_gpu = true;
        break;
      case MMX_STEP_CPU: {
        const int w = written_array(st.nest);
        int stream_to = -1;  // the later H2D of the array this nest writes, if its rows can be sent as they are produced
        if (overlap_enabled) {
          unsigned blocked = step_arrays(st);
          for (int sj = si + 1; sj < plan.num_steps && e == cudaSuccess; ++sj) {
            const mmx_plan_step& later = plan.steps[sj];
            const unsigned touches = step_arrays(later);
            if (later.kind == MMX_STEP_GPU && later.mode == MMX_MODE_GPU_NEST && (touches & blocked) == 0 && !issued[sj]) {
              const Clock::time_point tj = Clock::now();
              run_gpu_step(later);
              issued[sj] = true;
              s.stats.nest_s[later.nest] += since(tj);
              continue;
            }
            if (later.kind == MMX_STEP_H2D && w >= 0 && later.array == w && stream_to < 0 && st.nest != MMX_NEST_TRACE) {
              // nothing between here and there touched w: `blocked` holds it only because of this nest itself
              bool clean = true;
              for (int sk = si + 1; sk < sj; ++sk) clean = clean && (issued[sk] || (step_arrays(plan.steps[sk]) >> w & 1u) == 0);
              if (clean) stream_to = sj;
            }
            blocked |= touches;
          }
        }
        bool ok = true;
        if (stream_to >= 0 && e == cudaSuccess) {
          // one thread team per block: with many threads a block must stay long enough to pay for starting them
          const std::size_t want = static_cast<std::size_t>(std::max(1, 16 / std::max(1, ctx->cfg.host_threads)));
          const int blocks = static_cast<int>(std::min<std::size_t>(want, std::max<std::size_t>(1, n / 64)));
          const std::size_t row_bytes = n * esz;
          for (int blk = 0; blk < blocks && ok && e == cudaSuccess; ++blk) {
            const int r0 = static_cast<int>(n * blk / blocks), r1 = static_cast<int>(n * (blk + 1) / blocks);
            ok = ctx->cfg.dtype == MMX_F64 ? run_host_nest<double>(ctx, s, st.nest, r0, r1, dl, &checksum)
                                           : run_host_nest<float>(ctx, s, st.nest, r0, r1, dl, &checksum);
            if (ok)
              e = cudaMemcpyAsync(static_cast<char*>(s.d_arr[w]) + row_bytes * r0, static_cast<const char*>(s.h_arr[w]) + row_bytes * r0,
                                  row_bytes * (r1 - r0), cudaMemcpyHostToDevice, s.stream);
          }
          issued[stream_to] = true;
          any_gpu = true;
          if (w == MMX_ARRAY_A) s.planes_a_valid = false;
          if (w == MMX_ARRAY_BT) s.planes_bt_valid = false;
          if (w == MMX_ARRAY_B) s.b_colexp_valid = false;
          if (w == MMX_ARRAY_C) s.c_zero = false;
        } else {
          ok = ctx->cfg.dtype == MMX_F64 ? run_host_nest<double>(ctx, s, st.nest, 0, static_cast<int>(n), dl, &checksum)
                                         : run_host_nest<float>(ctx, s, st.nest, 0, static_cast<int>(n), dl, &checksum);
        }
        if (!ok) timed_out = true;
        if (w >= 0) {
          s.host_valid[w] = true;
          s.dev_valid[w] = stream_to >= 0 && ok;  // streamed: valid on both sides, as after the plan's own H2D
          if (w == MMX_ARRAY_C) s.host_diag_only = false;
        }
        s.stats.host_s += since(ts);
        break;
      }
      case MMX_STEP_GPU: run_gpu_step(st); break;
      case MMX_STEP_D2H_SUM:
        e = cudaMemcpyAsync(s.h_sum, s.d_sum, esz, cudaMemcpyDeviceToHost, s.stream);
        break;
      default: e = cudaErrorInvalidValue; break;
    }
    if (st.nest >= 0) s.stats.nest_s[st.nest] += since(ts);
    if (!timed_out && dl.expired()) timed_out = true;
  }

  if (s.b_pending) {  // a run cut short between init-b and the transpose that would have produced it: b is written all the same
    s.b_pending = false;
    const int nn = ctx->cfg.n;
    const cudaError_t eb = ctx->cfg.dtype == MMX_F64 ? launch_fill2d<double>(FILL_INIT_B, static_cast<double*>(s.d_arr[MMX_ARRAY_B]), nn, 0, nn, s.stream)
                                                     : launch_fill2d<float>(FILL_INIT_B, static_cast<float*>(s.d_arr[MMX_ARRAY_B]), nn, 0, nn, s.stream);
    if (e == cudaSuccess) e = eb;
  }
  if (e == cudaSuccess) e = cudaEventRecord(s.ev_end, s.stream);
  cudaError_t esync = cudaStreamSynchronize(s.stream);  // always drain, also after a timeout
  if (e == cudaSuccess) e = esync;
  const double wall = since(t0);
  if (e != cudaSuccess) {
    ctx->set_error(std::string("run failed: ") + cudaGetErrorString(e));
    cudaGetLastError();
    rr.status = MMX_RUNTIME_ERROR;
    return rr;
  }
  if (timed_out || wall > budget) {
    rr.status = MMX_TIMEOUT;
    rr.time_s = budget;
    return rr;
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, s.ev_begin, s.ev_end);
  s.stats.gpu_ms = ms;
  if (sum_on_device)
    checksum = ctx->cfg.dtype == MMX_F64 ? *static_cast<double*>(s.h_sum) : static_cast<double>(*static_cast<float*>(s.h_sum));
  s.stats.checksum = checksum;
  // An individual with device work is timed by its CUDA events (begin recorded on an idle stream
  // before the first step, end after the last: host-side nests in between are inside the bracket);
  // an all-CPU individual has no device timeline and is timed by the host clock.
  rr.time_s = any_gpu ? static_cast<double>(ms) * 1e-3 : wall;
  rr.status = rr.time_s > 0.0 ? MMX_MEASURED : MMX_RUNTIME_ERROR;
  return rr;
}

int measure_on_slot(mmx_ctx* ctx, int slot, const std::uint8_t* bits, std::size_t gene_len, mmx_outcome* out) {
  if (ctx == nullptr || bits == nullptr || out == nullptr) return MMX_E_INVALID;
  if (slot < 0 || slot >= static_cast<int>(ctx->slots.size())) {
    ctx->set_error("slot out of range");
    return MMX_E_INVALID;
  }
  if (gene_len != MMX_GENE_LENGTH) {
    ctx->set_error("genome length " + std::to_string(gene_len) + " does not match candidate count 12");
    return MMX_E_LENGTH;
  }
  const Clock::time_point t0 = Clock::now();
  mmx_plan_info plan;
  int rc = build_plan(bits, gene_len, ctx->cfg.n, ctx->cfg.dtype, &plan);
  if (rc != MMX_OK) return rc;
  out->status = MMX_RUNTIME_ERROR;
  out->time_s = 0.0;
  out->wall_cost_s = 0.0;
  if (!plan.feasible) {
    out->status = MMX_COMPILE_ERROR;
    out->wall_cost_s = since(t0);
    return MMX_OK;
  }
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> guard(s.mu);
  // the slot's own CPUs for the host loops and their thread team; a plan without host-side nests has nothing to isolate
  // and skips the three affinity system calls
  bool host_work = false;
  for (int si = 0; si < plan.num_steps; ++si) host_work = host_work || plan.steps[si].kind == MMX_STEP_CPU;
  static const std::vector<int> no_cpus;
  const ScopedAffinity pinned(host_work ? s.cpus : no_cpus);
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  // allocation is outside the timed region: host mirrors for every array a step touches on the host
  for (int si = 0; si < plan.num_steps; ++si) {
    const mmx_plan_step& st = plan.steps[si];
    if (st.kind == MMX_STEP_CPU) {
      for (int q = 0; q < MMX_NUM_ARRAYS; ++q)
        if ((nest_arrays(st.nest) >> q & 1) && (rc = ensure_host(ctx, s, q)) != MMX_OK) return rc;
    } else if (st.array >= 0) {
      if ((rc = ensure_host(ctx, s, st.array)) != MMX_OK) return rc;
    } else if (st.kind == MMX_STEP_GPU && st.mode != MMX_MODE_GPU_NEST) {
      MMX_CUDA(ctx, prepare_train(ctx, s, gene_of(st.nest, st.mode), static_cast<long long>(st.launches)));
    }
  }
  s.stats.h2d_bytes = plan.h2d_bytes;
  s.stats.d2h_bytes = plan.d2h_bytes;
  s.stats.kernel_launches = plan.kernel_launches;
  unsigned mask = 0;
  for (std::size_t k = 0; k < gene_len; ++k) mask |= (bits[k] ? 1u : 0u) << k;
  MMX_CUDA(ctx, prepare_plan_graph(ctx, s, plan, mask));
  const auto whole_it = s.plan_graphs.find(mask);
  const Slot::PlanGraph* whole = whole_it == s.plan_graphs.end() ? nullptr : &whole_it->second;

  for (int w = 0; w < ctx->cfg.warmup; ++w) {
    const RunResult r = run_plan_once(ctx, s, plan, whole);
    if (r.status != MMX_MEASURED) break;  // the timed loop below reports it
  }
  const int reps = std::max(1, ctx->cfg.repetitions);
  std::vector<double> times;
  for (int r = 0; r < reps; ++r) {
    const RunResult rr = run_plan_once(ctx, s, plan, whole);
    if (rr.status != MMX_MEASURED) {
      out->status = rr.status;
      out->time_s = rr.status == MMX_TIMEOUT ? rr.time_s : 0.0;
      out->wall_cost_s = since(t0);
      return MMX_OK;
    }
    times.push_back(rr.time_s);
  }
  std::sort(times.begin(), times.end());
  const std::size_t m = times.size();
  out->time_s = m % 2 == 1 ? times[m / 2] : 0.5 * (times[m / 2 - 1] + times[m / 2]);
  out->status = MMX_MEASURED;
  out->wall_cost_s = since(t0);
  return MMX_OK;
}

void destroy_slot(Slot& s) {
  cudaSetDevice(s.device);
  for (auto& kv : s.trains)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  for (auto& kv : s.plan_graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  for (int q = 0; q < MMX_NUM_ARRAYS; ++q) {
    if (s.d_arr[q]) cudaFree(s.d_arr[q]);
    if (s.h_arr[q]) cudaFreeHost(s.h_arr[q]);
  }
  if (s.d_sum) cudaFree(s.d_sum);
  if (s.h_sum) cudaFreeHost(s.h_sum);
  if (s.d_iter) cudaFree(s.d_iter);
  if (s.d_scrub) cudaFree(s.d_scrub);
  if (s.d_scratch) cudaFree(s.d_scratch);
  if (s.ev_begin) cudaEventDestroy(s.ev_begin);
  if (s.ev_end) cudaEventDestroy(s.ev_end);
  for (int r = 0; r < kMaxPeers; ++r)
    if (s.peer_ipc[r]) {
      if (s.peer_bt[r]) cudaIpcCloseMemHandle(s.peer_bt[r]);
      if (s.peer_ready[r]) cudaEventDestroy(s.peer_ready[r]);
    }
  for (cudaEvent_t e : {s.ev_ready, s.ev_x0, s.ev_x1, s.ev_m0, s.ev_m1})
    if (e) cudaEventDestroy(e);
  for (int q = 0; q < 2; ++q) {
    if (s.ev_join[q]) cudaEventDestroy(s.ev_join[q]);
    if (s.lane[q]) cudaStreamDestroy(s.lane[q]);
  }
  if (s.ev_fork) cudaEventDestroy(s.ev_fork);
  if (s.stream) cudaStreamDestroy(s.stream);
}

}  // namespace
}  // namespace mmx

// ================================================================================================
// C ABI
// ================================================================================================
using namespace mmx;

extern "C" {

MMX_API int mmx_loop_catalogue(mmx_loop_info* rows, size_t cap) {
  for (size_t k = 0; k < cap && k < MMX_GENE_LENGTH; ++k) {
    const LoopRow& r = kCatalogue[k];
    rows[k].gene = r.gene;
    rows[k].line = r.line;
    rows[k].depth = r.depth;
    rows[k].nest = r.nest;
    rows[k].induction = r.induction;
    rows[k].kernel = r.kernel;
  }
  return MMX_GENE_LENGTH;
}

MMX_API int mmx_plan(const uint8_t* bits, size_t gene_len, int32_t n, int32_t dtype, mmx_plan_info* out) {
  return build_plan(bits, gene_len, n, dtype, out);
}

MMX_API void mmx_default_config(mmx_config* cfg) {
  if (cfg == nullptr) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->struct_size = sizeof(mmx_config);
  cfg->n = 256;                 // fixtures/matmul.c:3
  cfg->dtype = MMX_F64;         // fixtures/matmul.c:5
  cfg->numerics = MMX_NUMERICS_FAST;
  cfg->timeout_s = 120.0;       // ToolchainConfig::timeout_s (evaluator.hpp:43)
  cfg->repetitions = 1;         // ToolchainConfig::repetitions (evaluator.hpp:44)
  cfg->num_slots = 1;
  cfg->devices = nullptr;
  cfg->host_threads = 1;
  cfg->launch_batching = 1;
  cfg->matmul_variant = 0;
  cfg->warmup = 0;
  cfg->pin_host = 1;
  cfg->host_core_first = 0;
  cfg->host_core_count = 0;  // all the CPUs the process may run on
  cfg->early_timeout = 1;
}

MMX_API int mmx_create(const mmx_config* cfg, mmx_ctx** out) {
  if (cfg == nullptr || out == nullptr) {
    g_create_error = "null argument";
    return MMX_E_INVALID;
  }
  *out = nullptr;
  if (cfg->struct_size != sizeof(mmx_config)) {
    g_create_error = "mmx_config.struct_size mismatch";
    return MMX_E_INVALID;
  }
  if (cfg->n < 1 || cfg->n > 65536 || (cfg->dtype != MMX_F64 && cfg->dtype != MMX_F32) ||
      (cfg->numerics != MMX_NUMERICS_FAST && cfg->numerics != MMX_NUMERICS_STRICT) || !(cfg->timeout_s > 0.0) ||
      cfg->repetitions < 1 || cfg->num_slots < 1 || cfg->num_slots > 64 || cfg->host_threads < 1 || cfg->warmup < 0 ||
      cfg->matmul_variant < 0 || cfg->matmul_variant > 45 || cfg->host_core_first < 0 || cfg->host_core_count < 0) {
    g_create_error = "invalid configuration value";
    return MMX_E_INVALID;
  }
  int count = 0;
  const cudaError_t ce = cudaGetDeviceCount(&count);
  if (ce != cudaSuccess || count < 1) {
    // the reference throws ToolchainMissing when the tool itself is absent (evaluator.cpp:102);
    // there is deliberately no CPU path to fall back to.
    g_create_error = std::string("no usable CUDA device: ") + (ce != cudaSuccess ? cudaGetErrorString(ce) : "device count is 0");
    cudaGetLastError();
    return MMX_E_NODEVICE;
  }
  std::unique_ptr<mmx_ctx> ctx(new mmx_ctx);
  ctx->cfg = *cfg;
  ctx->cfg.devices = nullptr;
  for (int s = 0; s < cfg->num_slots; ++s) {
    const int dev = cfg->devices ? cfg->devices[s] : s % count;
    if (dev < 0 || dev >= count) {
      g_create_error = "device ordinal out of range";
      return MMX_E_INVALID;
    }
    ctx->devices.push_back(dev);
  }
  const std::size_t mbytes = matrix_bytes(ctx.get());
  auto fail = [&](cudaError_t e, const char* what) {
    g_create_error = std::string(what) + ": " + cudaGetErrorString(e);
    for (auto& sl : ctx->slots) destroy_slot(*sl);
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? MMX_E_NOMEM : MMX_E_CUDA;
  };
  for (int s = 0; s < cfg->num_slots; ++s) {
    ctx->slots.emplace_back(new Slot);
    Slot& sl = *ctx->slots.back();
    sl.device = ctx->devices[s];
    cudaError_t e;
    if ((e = cudaSetDevice(sl.device)) != cudaSuccess) return fail(e, "cudaSetDevice");
    // the slot's own stream outranks its side lanes: when a lane's kernel and the main chain's become ready together (the fill of b
    // beside the contraction), the main chain's CTAs are placed first
    int prio_low = 0, prio_high = 0;
    cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high);
    static const bool prio_enabled = [] { const char* v = getenv("MMX_STREAM_PRIO"); return v == nullptr || atoi(v) != 0; }();  // 0: A/B runs
    if (!prio_enabled) prio_low = prio_high = 0;
    if ((e = cudaStreamCreateWithPriority(&sl.stream, cudaStreamNonBlocking, prio_high)) != cudaSuccess) return fail(e, "cudaStreamCreate");
    sl.cur = sl.stream;
    for (int q = 0; q < 2; ++q) {
      if ((e = cudaStreamCreateWithPriority(&sl.lane[q], cudaStreamNonBlocking, prio_low)) != cudaSuccess) return fail(e, "cudaStreamCreate");
      if ((e = cudaEventCreateWithFlags(&sl.ev_join[q], cudaEventDisableTiming)) != cudaSuccess) return fail(e, "cudaEventCreate");
    }
    if ((e = cudaEventCreateWithFlags(&sl.ev_fork, cudaEventDisableTiming)) != cudaSuccess) return fail(e, "cudaEventCreate");
    if ((e = cudaEventCreate(&sl.ev_begin)) != cudaSuccess) return fail(e, "cudaEventCreate");
    if ((e = cudaEventCreate(&sl.ev_end)) != cudaSuccess) return fail(e, "cudaEventCreate");
    for (int q = 0; q < MMX_NUM_ARRAYS; ++q)
      if ((e = cudaMalloc(&sl.d_arr[q], mbytes)) != cudaSuccess) return fail(e, "cudaMalloc(array)");
    // allocated up front: whole individuals are captured into CUDA graphs, where cudaMalloc is not allowed
    if (cfg->dtype == MMX_F32 && cfg->numerics == MMX_NUMERICS_FAST && matmul_3xtf32_usable(cfg->n) &&
        (cfg->matmul_variant == 30 || cfg->matmul_variant == 31 || (cfg->matmul_variant == 0 && cfg->n >= kTcMinN)))
    {
      if ((e = matmul_3xtf32_prepare()) != cudaSuccess) return fail(e, "matmul_3xtf32_prepare");
      if (cfg->matmul_variant == 0 && fp32_int8_enabled(cfg->n)) {
        // FP32 auto mode: the split-TF32 area, then the digit planes of the INT8 forms (zero-filled: matmul_ozaki.cu)
        const std::size_t off = fp32_int8_scratch_offset(cfg->n), planes = matmul_ozaki_scratch_bytes(cfg->n);
        if ((e = matmul_ozaki_prepare()) != cudaSuccess) return fail(e, "matmul_ozaki_prepare");
        if ((e = cudaMalloc(&sl.d_scratch, off + planes)) != cudaSuccess) return fail(e, "cudaMalloc(scratch)");
        void* oz = static_cast<char*>(sl.d_scratch) + off;
        sl.oz_planes = oz;
        if ((e = cudaMemset(oz, 0, planes)) != cudaSuccess) return fail(e, "cudaMemset(scratch)");
        sl.gene8_form_word = matmul_ozaki_form_word(oz, cfg->n);
        if ((e = cudaMemset(sl.gene8_form_word, 0xff, sizeof(int))) != cudaSuccess) return fail(e, "cudaMemset(form)");
      } else if ((e = cudaMalloc(&sl.d_scratch, matmul_3xtf32_scratch_bytes(cfg->n))) != cudaSuccess) {
        return fail(e, "cudaMalloc(scratch)");
      }
    }
    if (cfg->dtype == MMX_F64 && cfg->numerics == MMX_NUMERICS_FAST && matmul_ozaki_usable(cfg->n) &&
        ((cfg->matmul_variant >= 40 && cfg->matmul_variant <= 45) || (cfg->matmul_variant == 0 && cfg->n >= kOzMinN))) {
      if ((e = matmul_ozaki_prepare()) != cudaSuccess) return fail(e, "matmul_ozaki_prepare");
      if ((e = cudaMalloc(&sl.d_scratch, matmul_ozaki_scratch_bytes(cfg->n))) != cudaSuccess) return fail(e, "cudaMalloc(scratch)");
      if (cfg->matmul_variant == 0) {
        // auto mode relies on a zero-filled scratch (digit planes nobody has written yet are zero, matmul_ozaki.cu)
        if ((e = cudaMemset(sl.d_scratch, 0, matmul_ozaki_scratch_bytes(cfg->n))) != cudaSuccess) return fail(e, "cudaMemset(scratch)");
        sl.gene8_form_word = matmul_ozaki_form_word(sl.d_scratch, cfg->n);
        sl.oz_planes = sl.d_scratch;
        if ((e = cudaMemset(sl.gene8_form_word, 0xff, sizeof(int))) != cudaSuccess) return fail(e, "cudaMemset(form)");
        sl.gene8_form_valid = true;
      }
    }
    if ((e = cudaMalloc(&sl.d_sum, 16)) != cudaSuccess) return fail(e, "cudaMalloc(sum)");
    if ((e = cudaMalloc(reinterpret_cast<void**>(&sl.d_iter), sizeof(int))) != cudaSuccess) return fail(e, "cudaMalloc(iter)");
    if ((e = cudaHostAlloc(&sl.h_sum, 16, cudaHostAllocDefault)) != cudaSuccess) return fail(e, "cudaHostAlloc(sum)");
    std::memset(sl.h_sum, 0, 16);
  }
  if (cfg->pin_host) {
    // this context's share of the allowed CPUs, split evenly among its slots (whole SMT cores where the numbers allow it); with
    // fewer CPUs than slots the slots take turns on them
    std::vector<int> all = allowed_cpus_by_core();
    if (cfg->host_core_count > 0 && !all.empty()) {
      const std::size_t first = std::min<std::size_t>(static_cast<std::size_t>(cfg->host_core_first), all.size() - 1);
      const std::size_t count = std::min<std::size_t>(static_cast<std::size_t>(cfg->host_core_count), all.size() - first);
      all = std::vector<int>(all.begin() + static_cast<std::ptrdiff_t>(first), all.begin() + static_cast<std::ptrdiff_t>(first + count));
    }
    const std::size_t slots = ctx->slots.size();
    for (std::size_t q = 0; q < slots && !all.empty(); ++q) {
      Slot& sl = *ctx->slots[q];
      if (all.size() >= slots) {
        const std::size_t lo = all.size() * q / slots, hi = all.size() * (q + 1) / slots;
        sl.cpus.assign(all.begin() + static_cast<std::ptrdiff_t>(lo), all.begin() + static_cast<std::ptrdiff_t>(hi));
      } else {
        sl.cpus.assign(1, all[q % all.size()]);
      }
    }
  }
  *out = ctx.release();
  return MMX_OK;
}

MMX_API void mmx_destroy(mmx_ctx* ctx) {
  if (ctx == nullptr) return;
  for (auto& sl : ctx->slots) destroy_slot(*sl);
  delete ctx;
}

MMX_API size_t mmx_gene_length(const mmx_ctx*) { return MMX_GENE_LENGTH; }

MMX_API int mmx_num_slots(const mmx_ctx* ctx) { return ctx ? static_cast<int>(ctx->slots.size()) : 0; }

MMX_API const char* mmx_last_error(const mmx_ctx* ctx) {
  if (ctx == nullptr) return g_create_error.c_str();
  std::lock_guard<std::mutex> g(ctx->err_mu);
  ctx->error_snapshot = ctx->error;
  return ctx->error_snapshot.c_str();
}

MMX_API int mmx_measure(mmx_ctx* ctx, int slot, const uint8_t* bits, size_t gene_len, mmx_outcome* out) {
  return measure_on_slot(ctx, slot, bits, gene_len, out);
}

MMX_API int mmx_measure_batch(mmx_ctx* ctx, const uint8_t* bits, size_t n_genomes, size_t gene_len, mmx_outcome* outs) {
  if (ctx == nullptr || (n_genomes > 0 && (bits == nullptr || outs == nullptr))) return MMX_E_INVALID;
  if (gene_len != MMX_GENE_LENGTH) {
    ctx->set_error("genome length " + std::to_string(gene_len) + " does not match candidate count 12");
    return MMX_E_LENGTH;
  }
  if (n_genomes == 0) return MMX_OK;
  // dynamic pull, one worker per slot -- the scheme of Evaluator::evaluate_all (evaluator.cpp:254-273):
  // per-individual cost varies by orders of magnitude, so static blocks would idle most slots.
  std::atomic<size_t> next{0};
  std::atomic<int> first_error{MMX_OK};
  auto worker = [&](int slot) {
    for (;;) {
      const size_t i = next.fetch_add(1);
      if (i >= n_genomes) return;
      const int rc = measure_on_slot(ctx, slot, bits + i * gene_len, gene_len, &outs[i]);
      if (rc != MMX_OK) {
        int expected = MMX_OK;
        first_error.compare_exchange_strong(expected, rc);
        return;
      }
    }
  };
  const int workers = static_cast<int>(std::min<size_t>(ctx->slots.size(), n_genomes));
  if (workers == 1) {
    worker(0);
  } else {
    std::vector<std::thread> pool;
    for (int s = 0; s < workers; ++s) pool.emplace_back(worker, s);
    for (auto& t : pool) t.join();
  }
  return first_error.load();
}

MMX_API int mmx_last_stats(mmx_ctx* ctx, int slot, mmx_run_stats* out) {
  if (ctx == nullptr || out == nullptr || slot < 0 || slot >= static_cast<int>(ctx->slots.size())) return MMX_E_INVALID;
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  *out = s.stats;
  return MMX_OK;
}

MMX_API int mmx_fetch_array(mmx_ctx* ctx, int slot, int array, void* host, size_t bytes) {
  if (ctx == nullptr || host == nullptr || slot < 0 || slot >= static_cast<int>(ctx->slots.size()) || array < 0 ||
      array >= MMX_NUM_ARRAYS)
    return MMX_E_INVALID;
  if (bytes != matrix_bytes(ctx)) {
    ctx->set_error("mmx_fetch_array: size mismatch");
    return MMX_E_INVALID;
  }
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  if (s.dev_valid[array]) {
    MMX_CUDA(ctx, cudaMemcpyAsync(host, s.d_arr[array], bytes, cudaMemcpyDeviceToHost, s.stream));
    MMX_CUDA(ctx, cudaStreamSynchronize(s.stream));
    return MMX_OK;
  }
  if (s.host_valid[array] && s.h_arr[array] != nullptr && !(array == MMX_ARRAY_C && s.host_diag_only)) {
    std::memcpy(host, s.h_arr[array], bytes);
    return MMX_OK;
  }
  ctx->set_error("mmx_fetch_array: array is not valid on either side");
  return MMX_E_STATE;
}

MMX_API int mmx_fetch_rows(mmx_ctx* ctx, int slot, int array, int row0, int rows, void* host, size_t bytes) {
  if (ctx == nullptr || host == nullptr || slot < 0 || slot >= static_cast<int>(ctx->slots.size()) || array < 0 || array >= MMX_NUM_ARRAYS)
    return MMX_E_INVALID;
  const std::size_t row_bytes = static_cast<std::size_t>(ctx->cfg.n) * elem_size(ctx->cfg.dtype);
  if (row0 < 0 || rows < 0 || row0 + rows > ctx->cfg.n || bytes != row_bytes * static_cast<std::size_t>(rows)) {
    ctx->set_error("mmx_fetch_rows: row block outside the array or size mismatch");
    return MMX_E_INVALID;
  }
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  const std::size_t offset = row_bytes * static_cast<std::size_t>(row0);
  if (s.dev_valid[array]) {
    MMX_CUDA(ctx, cudaMemcpyAsync(host, static_cast<const char*>(s.d_arr[array]) + offset, bytes, cudaMemcpyDeviceToHost, s.stream));
    MMX_CUDA(ctx, cudaStreamSynchronize(s.stream));
    return MMX_OK;
  }
  if (s.host_valid[array] && s.h_arr[array] != nullptr && !(array == MMX_ARRAY_C && s.host_diag_only)) {
    std::memcpy(host, static_cast<const char*>(s.h_arr[array]) + offset, bytes);
    return MMX_OK;
  }
  ctx->set_error("mmx_fetch_rows: array is not valid on either side");
  return MMX_E_STATE;
}

MMX_API int mmx_upload_array(mmx_ctx* ctx, int slot, int array, const void* host, size_t bytes) {
  if (ctx == nullptr || host == nullptr || slot < 0 || slot >= static_cast<int>(ctx->slots.size()) || array < 0 ||
      array >= MMX_NUM_ARRAYS)
    return MMX_E_INVALID;
  if (bytes != matrix_bytes(ctx)) {
    ctx->set_error("mmx_upload_array: size mismatch");
    return MMX_E_INVALID;
  }
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  MMX_CUDA(ctx, cudaMemcpyAsync(s.d_arr[array], host, bytes, cudaMemcpyHostToDevice, s.stream));
  MMX_CUDA(ctx, cudaStreamSynchronize(s.stream));
  s.dev_valid[array] = true;
  s.host_valid[array] = false;
  if (array == MMX_ARRAY_A) s.planes_a_valid = false;
  if (array == MMX_ARRAY_BT) s.planes_bt_valid = false;
  if (array == MMX_ARRAY_B) s.b_colexp_valid = false;
  if (array == MMX_ARRAY_C) s.c_zero = false;
  return MMX_OK;
}

MMX_API int mmx_run_loop(mmx_ctx* ctx, int slot, int gene, int i, int j, double* sum_out) {
  if (ctx == nullptr || slot < 0 || slot >= static_cast<int>(ctx->slots.size()) || gene < 0 || gene >= MMX_GENE_LENGTH)
    return MMX_E_INVALID;
  const int n = ctx->cfg.n;
  if (i < 0 || i >= n || j < 0 || j >= n) return MMX_E_INVALID;
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  const int it = gene == 10 ? i * n + j : i;
  s.fuse_planes = false;  // single kernels: producers write their array only, gene 8 encodes what it needs
  MMX_CUDA(ctx, launch_gene_any(ctx, s, gene, IterRef{nullptr, it}));
  const int w = written_array(kCatalogue[gene].nest);
  if (w >= 0) {
    s.dev_valid[w] = true;
    s.host_valid[w] = false;
  }
  if (gene == 11) {
    const std::size_t esz = elem_size(ctx->cfg.dtype);
    MMX_CUDA(ctx, cudaMemcpyAsync(s.h_sum, s.d_sum, esz, cudaMemcpyDeviceToHost, s.stream));
  }
  MMX_CUDA(ctx, cudaStreamSynchronize(s.stream));
  if (gene == 11 && sum_out != nullptr)
    *sum_out = ctx->cfg.dtype == MMX_F64 ? *static_cast<double*>(s.h_sum) : static_cast<double>(*static_cast<float*>(s.h_sum));
  return MMX_OK;
}

MMX_API int mmx_run_loop_rows(mmx_ctx* ctx, int slot, int gene, int row0, int rows, double* sum_out) {
  if (ctx == nullptr || slot < 0 || slot >= static_cast<int>(ctx->slots.size())) return MMX_E_INVALID;
  const int n = ctx->cfg.n;
  const bool depth0 = gene == 0 || gene == 2 || gene == 4 || gene == 6 || gene == 8 || gene == 11;
  if (!depth0 || row0 < 0 || rows < 0 || row0 + rows > n) {
    ctx->set_error("mmx_run_loop_rows: needs a depth-0 gene and a row block inside the matrix");
    return MMX_E_INVALID;
  }
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  s.fuse_planes = false;
  MMX_CUDA(ctx, launch_gene_rows(ctx, s, gene, IterRef{nullptr, 0}, row0, rows));
  const int w = written_array(kCatalogue[gene].nest);
  if (w >= 0) {
    s.dev_valid[w] = true;
    s.host_valid[w] = false;
  }
  if (gene == 11) MMX_CUDA(ctx, cudaMemcpyAsync(s.h_sum, s.d_sum, elem_size(ctx->cfg.dtype), cudaMemcpyDeviceToHost, s.stream));
  MMX_CUDA(ctx, cudaStreamSynchronize(s.stream));
  if (gene == 11 && sum_out != nullptr)
    *sum_out = ctx->cfg.dtype == MMX_F64 ? *static_cast<double*>(s.h_sum) : static_cast<double>(*static_cast<float*>(s.h_sum));
  return MMX_OK;
}

MMX_API int mmx_device_ptr(mmx_ctx* ctx, int slot, int array, void** ptr_out) {
  if (ctx == nullptr || ptr_out == nullptr || slot < 0 || slot >= static_cast<int>(ctx->slots.size()) || array < 0 ||
      array >= MMX_NUM_ARRAYS)
    return MMX_E_INVALID;
  *ptr_out = ctx->slots[slot]->d_arr[array];
  return MMX_OK;
}

MMX_API int mmx_time_gene8_contraction(mmx_ctx* ctx, int slot, int iters, int flush_l2, double* ms_out) {
  if (ctx == nullptr || ms_out == nullptr || slot < 0 || slot >= static_cast<int>(ctx->slots.size()) || iters < 1) return MMX_E_INVALID;
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  if (!s.gene8_form_valid) return MMX_E_INVALID;  // FP64 auto-mode contexts only
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  const int n = ctx->cfg.n;
  double *a = static_cast<double*>(s.d_arr[MMX_ARRAY_A]), *bt = static_cast<double*>(s.d_arr[MMX_ARRAY_BT]), *c = static_cast<double*>(s.d_arr[MMX_ARRAY_C]);
  // one full launch encodes the operands (and tells which form they take); the timed ones reuse the encoding
  MMX_CUDA(ctx, launch_matmul<double>(c, a, bt, n, 0, n, 0, n, false, 0, s.d_scratch, s.stream));
  if (flush_l2 == 1 && s.d_scrub == nullptr) {
    s.scrub_bytes = std::size_t{256} << 20;  // 256 MiB > 126 MB L2
    MMX_CUDA(ctx, cudaMalloc(&s.d_scrub, s.scrub_bytes));
    MMX_CUDA(ctx, launch_scrub(s.d_scrub, s.scrub_bytes, s.stream));
  }
  double total = 0.0;
  if (flush_l2 == 2) {
    // back to back: one event pair around `iters` launches, nothing in between -- the sustained rate of the kernel
    MMX_CUDA(ctx, cudaEventRecord(s.ev_begin, s.stream));
    for (int it = 0; it < iters; ++it)
      MMX_CUDA(ctx, launch_matmul<double>(c, a, bt, n, 0, n, 0, n, false, kReuseOperands, s.d_scratch, s.stream));
    MMX_CUDA(ctx, cudaEventRecord(s.ev_end, s.stream));
    MMX_CUDA(ctx, cudaEventSynchronize(s.ev_end));
    float ms = 0.f;
    MMX_CUDA(ctx, cudaEventElapsedTime(&ms, s.ev_begin, s.ev_end));
    total = ms;
  }
  for (int it = 0; flush_l2 != 2 && it < iters; ++it) {
    if (flush_l2) MMX_CUDA(ctx, launch_evict(s.d_scrub, s.scrub_bytes, s.stream));
    MMX_CUDA(ctx, cudaEventRecord(s.ev_begin, s.stream));
    MMX_CUDA(ctx, launch_matmul<double>(c, a, bt, n, 0, n, 0, n, false, kReuseOperands, s.d_scratch, s.stream));
    MMX_CUDA(ctx, cudaEventRecord(s.ev_end, s.stream));
    MMX_CUDA(ctx, cudaEventSynchronize(s.ev_end));
    float ms = 0.f;
    MMX_CUDA(ctx, cudaEventElapsedTime(&ms, s.ev_begin, s.ev_end));
    total += ms;
  }
  s.dev_valid[MMX_ARRAY_C] = true;
  s.host_valid[MMX_ARRAY_C] = false;
  *ms_out = total / iters;
  return MMX_OK;
}

MMX_API int mmx_gene8_pick_form(int cut, int top_a, int top_bt) { return ozaki_pick_form(cut, top_a, top_bt); }

MMX_API int mmx_gene8_form(mmx_ctx* ctx, int slot, int32_t* form_out) {
  if (ctx == nullptr || form_out == nullptr || slot < 0 || slot >= static_cast<int>(ctx->slots.size())) return MMX_E_INVALID;
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  *form_out = -1;
  if (s.gene8_form_word == nullptr) return MMX_OK;
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  MMX_CUDA(ctx, cudaStreamSynchronize(s.stream));
  MMX_CUDA(ctx, cudaMemcpy(form_out, s.gene8_form_word, sizeof(int32_t), cudaMemcpyDeviceToHost));
  return MMX_OK;
}

MMX_API int mmx_time_loop(mmx_ctx* ctx, int slot, int gene, int iters, int flush_l2, double* ms_out) {
  if (ctx == nullptr || ms_out == nullptr || slot < 0 || slot >= static_cast<int>(ctx->slots.size()) || gene < 0 ||
      gene >= MMX_GENE_LENGTH || iters < 1)
    return MMX_E_INVALID;
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  if (flush_l2 && s.d_scrub == nullptr) {
    s.scrub_bytes = std::size_t{256} << 20;  // 256 MiB > 126 MB L2
    MMX_CUDA(ctx, cudaMalloc(&s.d_scrub, s.scrub_bytes));
    MMX_CUDA(ctx, launch_scrub(s.d_scrub, s.scrub_bytes, s.stream));
  }
  double total = 0.0;
  s.fuse_planes = false;
  for (int it = 0; it < iters; ++it) {
    if (flush_l2) MMX_CUDA(ctx, launch_evict(s.d_scrub, s.scrub_bytes, s.stream));
    MMX_CUDA(ctx, cudaEventRecord(s.ev_begin, s.stream));
    MMX_CUDA(ctx, launch_gene_any(ctx, s, gene, IterRef{nullptr, 0}));
    MMX_CUDA(ctx, cudaEventRecord(s.ev_end, s.stream));
    MMX_CUDA(ctx, cudaEventSynchronize(s.ev_end));
    float ms = 0.f;
    MMX_CUDA(ctx, cudaEventElapsedTime(&ms, s.ev_begin, s.ev_end));
    total += ms;
  }
  *ms_out = total / iters;
  return MMX_OK;
}

MMX_API int mmx_peak_probe(int device, int kind, double* value_out) {
  if (value_out == nullptr) return MMX_E_INVALID;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1) {
    cudaGetLastError();
    return MMX_E_NODEVICE;
  }
  if (device < 0 || device >= count) return MMX_E_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return MMX_E_CUDA;
  const cudaError_t e = probe_peak(kind, value_out);
  if (e != cudaSuccess) {
    g_create_error = std::string("peak probe: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return e == cudaErrorInvalidValue ? MMX_E_INVALID : MMX_E_CUDA;
  }
  return MMX_OK;
}

}  // extern "C"

// ================================================================================================
// Row-sharded run over a group of GPUs (BASELINE config 5)
// ================================================================================================
// Member r of a group of G owns rows R_r of a, c and bt.  Everything index-generated shards without
// communication (init-a, zero-c on R_r; init-b is regenerated locally because the transpose needs
// columns R_r of every row of b).  The one exchange of the path -- every member needs all of bt for
// the contraction -- is fused into the kernel that produces bt: the transpose stores each finished
// tile of bt[R_r][:] into the bt of every member through peer-mapped pointers (NVLink stores), so
// there is no separate all-gather and no staging buffer.  The contraction is then walked column
// block by column block in ring order starting with the member's own rows of bt; block s waits only
// for member s's "stored everywhere" event, so transfers from the slower members overlap the math
// on the blocks that have already arrived.
namespace mmx {
namespace {

void shard_block(int n, int world, int rank, int* row0, int* rows) {
  // contiguous, nearly equal blocks; boundaries are multiples of 64 when n allows it, so that the tiled
  // transpose and the GEMM tiles never straddle a block edge (same rule as rowshard.py: row_block)
  const int unit = (n % 64 == 0 && n / 64 >= world) ? 64 : 1;
  const long long units = n / unit;
  const int lo = static_cast<int>(units * rank / world) * unit;
  const int hi = static_cast<int>(units * (rank + 1) / world) * unit;
  *row0 = lo;
  *rows = hi - lo;
}

int shard_events(mmx_ctx* ctx, Slot& s) {
  if (s.ev_ready != nullptr) return MMX_OK;
  MMX_CUDA(ctx, cudaEventCreateWithFlags(&s.ev_ready, cudaEventDisableTiming | cudaEventInterprocess));
  MMX_CUDA(ctx, cudaEventCreate(&s.ev_x0));
  MMX_CUDA(ctx, cudaEventCreate(&s.ev_x1));
  MMX_CUDA(ctx, cudaEventCreate(&s.ev_m0));
  MMX_CUDA(ctx, cudaEventCreate(&s.ev_m1));
  return MMX_OK;
}

template <typename T>
int shard_phase1(mmx_ctx* ctx, Slot& s) {
  const int n = ctx->cfg.n;
  int r0 = 0, rows = 0;
  shard_block(n, s.shard_world, s.shard_rank, &r0, &rows);
  begin_sequence(s, false);  // row blocks: the contraction encodes what it needs, block by block
  MMX_CUDA(ctx, cudaEventRecord(s.ev_begin, s.stream));
  MMX_CUDA(ctx, launch_fill2d<T>(FILL_INIT_A, static_cast<T*>(s.d_arr[MMX_ARRAY_A]), n, r0, rows, s.stream));
  MMX_CUDA(ctx, launch_fill2d<T>(FILL_INIT_B, static_cast<T*>(s.d_arr[MMX_ARRAY_B]), n, 0, n, s.stream));
  MMX_CUDA(ctx, launch_fill2d<T>(FILL_ZERO, static_cast<T*>(s.d_arr[MMX_ARRAY_C]), n, r0, rows, s.stream));
  BtPeers peers;
  peers.count = s.shard_world;
  // own copy first, then the ring: member r+1, r+2, ... so that at any instant the members store into
  // different destinations
  for (int d = 0; d < s.shard_world; ++d) peers.p[d] = s.peer_bt[(s.shard_rank + d) % s.shard_world];
  MMX_CUDA(ctx, cudaEventRecord(s.ev_x0, s.stream));
  MMX_CUDA(ctx, launch_transpose_push<T>(peers, static_cast<const T*>(s.d_arr[MMX_ARRAY_B]), n, r0, rows, s.stream));
  MMX_CUDA(ctx, cudaEventRecord(s.ev_x1, s.stream));
  MMX_CUDA(ctx, cudaEventRecord(s.ev_ready, s.stream));
  return MMX_OK;
}

template <typename T>
int shard_phase2(mmx_ctx* ctx, Slot& s) {
  const int n = ctx->cfg.n;
  const bool strict = ctx->cfg.numerics == MMX_NUMERICS_STRICT;
  const int variant = ctx->cfg.matmul_variant;
  int r0 = 0, rows = 0;
  shard_block(n, s.shard_world, s.shard_rank, &r0, &rows);
  T* a = static_cast<T*>(s.d_arr[MMX_ARRAY_A]);
  T* c = static_cast<T*>(s.d_arr[MMX_ARRAY_C]);
  T* bt = static_cast<T*>(s.d_arr[MMX_ARRAY_BT]);
  MMX_CUDA(ctx, cudaEventRecord(s.ev_m0, s.stream));
  for (int d = 0; d < s.shard_world; ++d) {
    const int src = (s.shard_rank + d) % s.shard_world;
    int c0 = 0, cols = 0;
    shard_block(n, s.shard_world, src, &c0, &cols);
    if (src != s.shard_rank) MMX_CUDA(ctx, cudaStreamWaitEvent(s.stream, s.peer_ready[src], 0));
    // the member's rows of a are re-encoded for the tensor-core forms by the first column block only
    if (rows > 0 && cols > 0)
      MMX_CUDA(ctx, launch_matmul<T>(c, a, bt, n, r0, rows, c0, cols, strict, variant | (d > 0 ? kReuseOperandA : 0), s.d_scratch, s.stream));
  }
  MMX_CUDA(ctx, cudaEventRecord(s.ev_m1, s.stream));
  MMX_CUDA(ctx, launch_trace<T>(static_cast<T*>(s.d_sum), c, n, r0, rows, strict, s.stream));
  MMX_CUDA(ctx, cudaMemcpyAsync(s.h_sum, s.d_sum, sizeof(T), cudaMemcpyDeviceToHost, s.stream));
  MMX_CUDA(ctx, cudaEventRecord(s.ev_end, s.stream));
  return MMX_OK;
}

int shard_collect(mmx_ctx* ctx, Slot& s, mmx_shard_stats* out) {
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  MMX_CUDA(ctx, cudaStreamSynchronize(s.stream));
  const int n = ctx->cfg.n;
  for (int q : {MMX_ARRAY_A, MMX_ARRAY_B, MMX_ARRAY_C, MMX_ARRAY_BT}) {
    s.dev_valid[q] = true;   // a and c: this member's rows only
    s.host_valid[q] = false;
  }
  if (out == nullptr) return MMX_OK;
  std::memset(out, 0, sizeof(*out));
  out->rank = s.shard_rank;
  out->world = s.shard_world;
  shard_block(n, s.shard_world, s.shard_rank, &out->row0, &out->rows);
  float ms = 0.f;
  MMX_CUDA(ctx, cudaEventElapsedTime(&ms, s.ev_begin, s.ev_end));
  out->gpu_ms = ms;
  MMX_CUDA(ctx, cudaEventElapsedTime(&ms, s.ev_x0, s.ev_x1));
  out->exchange_ms = ms;
  MMX_CUDA(ctx, cudaEventElapsedTime(&ms, s.ev_m0, s.ev_m1));
  out->matmul_ms = ms;
  out->peer_bytes = static_cast<uint64_t>(out->rows) * n * elem_size(ctx->cfg.dtype) * (s.shard_world - 1);
  out->partial_trace = ctx->cfg.dtype == MMX_F64 ? *static_cast<double*>(s.h_sum) : static_cast<double>(*static_cast<float*>(s.h_sum));
  return MMX_OK;
}

bool shard_slot_ok(mmx_ctx* ctx, int slot) { return ctx != nullptr && slot >= 0 && slot < static_cast<int>(ctx->slots.size()); }

}  // namespace
}  // namespace mmx

MMX_API int mmx_shard_export(mmx_ctx* ctx, int slot, mmx_shard_handle* out) {
  if (!shard_slot_ok(ctx, slot) || out == nullptr) return MMX_E_INVALID;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64 && sizeof(cudaIpcEventHandle_t) == 64, "handle layout of mmx_shard_handle");
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  if (int rc = shard_events(ctx, s)) return rc;
  cudaIpcMemHandle_t mh;
  cudaIpcEventHandle_t eh;
  MMX_CUDA(ctx, cudaIpcGetMemHandle(&mh, s.d_arr[MMX_ARRAY_BT]));
  MMX_CUDA(ctx, cudaIpcGetEventHandle(&eh, s.ev_ready));
  std::memcpy(out->mem, &mh, 64);
  std::memcpy(out->event, &eh, 64);
  return MMX_OK;
}

MMX_API int mmx_shard_bind(mmx_ctx* ctx, int slot, int rank, int world, const mmx_shard_handle* handles, const int32_t* local_slots) {
  if (!shard_slot_ok(ctx, slot) || world < 1 || world > kMaxPeers || rank < 0 || rank >= world ||
      ((handles == nullptr) == (local_slots == nullptr) && world > 1)) {
    if (ctx) ctx->set_error("mmx_shard_bind: need 1 <= world <= 8, 0 <= rank < world and exactly one of handles / local_slots");
    return MMX_E_INVALID;
  }
  // validate everything that can be validated before touching the slot
  if (local_slots != nullptr)
    for (int r = 0; r < world; ++r)
      if (r != rank && (!shard_slot_ok(ctx, local_slots[r]) || local_slots[r] == slot)) {
        ctx->set_error("mmx_shard_bind: local_slots must name distinct slots of this context");
        return MMX_E_INVALID;
      }
  Slot& s = *ctx->slots[slot];
  // peers' ready events live on the peers' slots: create the missing ones first, one slot lock at a time (never two at once, so
  // concurrent binds of different slots cannot deadlock or race on a peer's events)
  if (local_slots != nullptr)
    for (int r = 0; r < world; ++r) {
      if (r == rank) continue;
      Slot& o = *ctx->slots[local_slots[r]];
      std::lock_guard<std::mutex> go(o.mu);
      if (o.ev_ready == nullptr) {
        MMX_CUDA(ctx, cudaSetDevice(o.device));
        if (int rc = shard_events(ctx, o)) return rc;
      }
    }
  std::lock_guard<std::mutex> g(s.mu);
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  if (int rc = shard_events(ctx, s)) return rc;
  // the new peer table is built in locals and committed together with rank and world only when every entry is in place; until
  // then the slot counts as unbound (phase1 / phase2 refuse to run), never as half bound
  void* new_bt[kMaxPeers] = {};
  cudaEvent_t new_ready[kMaxPeers] = {};
  bool new_ipc[kMaxPeers] = {};
  auto undo = [&]() {
    for (int r = 0; r < kMaxPeers; ++r)
      if (new_ipc[r]) {
        if (new_bt[r]) cudaIpcCloseMemHandle(new_bt[r]);
        if (new_ready[r]) cudaEventDestroy(new_ready[r]);
      }
    cudaGetLastError();
  };
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      new_bt[r] = s.d_arr[MMX_ARRAY_BT];
      new_ready[r] = s.ev_ready;
    } else if (local_slots != nullptr) {
      Slot& o = *ctx->slots[local_slots[r]];
      if (o.device != s.device) {
        int can = 0;
        cudaError_t e = cudaDeviceCanAccessPeer(&can, s.device, o.device);
        if (e == cudaSuccess && !can) {
          ctx->set_error("mmx_shard_bind: devices " + std::to_string(s.device) + " and " + std::to_string(o.device) + " have no peer access");
          undo();
          return MMX_E_CUDA;
        }
        if (e == cudaSuccess) e = cudaDeviceEnablePeerAccess(o.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) e = cudaSuccess;
        cudaGetLastError();
        if (e != cudaSuccess) {
          ctx->set_error(std::string("mmx_shard_bind: enabling peer access: ") + cudaGetErrorString(e));
          undo();
          return MMX_E_CUDA;
        }
      }
      new_bt[r] = o.d_arr[MMX_ARRAY_BT];
      new_ready[r] = o.ev_ready;
    } else {
      cudaIpcMemHandle_t mh;
      cudaIpcEventHandle_t eh;
      std::memcpy(&mh, handles[r].mem, 64);
      std::memcpy(&eh, handles[r].event, 64);
      cudaError_t e = cudaIpcOpenMemHandle(&new_bt[r], mh, cudaIpcMemLazyEnablePeerAccess);
      if (e == cudaSuccess) {
        new_ipc[r] = true;
        e = cudaIpcOpenEventHandle(&new_ready[r], eh);
      }
      if (e != cudaSuccess) {
        ctx->set_error(std::string("mmx_shard_bind: opening the handle of member ") + std::to_string(r) + ": " + cudaGetErrorString(e));
        undo();
        return MMX_E_CUDA;
      }
    }
  }
  // commit: drop the earlier binding, install the new one
  for (int r = 0; r < kMaxPeers; ++r) {
    if (s.peer_ipc[r]) {
      if (s.peer_bt[r]) cudaIpcCloseMemHandle(s.peer_bt[r]);
      if (s.peer_ready[r]) cudaEventDestroy(s.peer_ready[r]);
    }
    s.peer_bt[r] = new_bt[r];
    s.peer_ready[r] = new_ready[r];
    s.peer_ipc[r] = new_ipc[r];
  }
  s.shard_rank = rank;
  s.shard_world = world;
  return MMX_OK;
}

MMX_API int mmx_shard_phase1(mmx_ctx* ctx, int slot) {
  if (!shard_slot_ok(ctx, slot)) return MMX_E_INVALID;
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  if (s.shard_world < 1) {
    ctx->set_error("mmx_shard_phase1: slot is not bound to a group (mmx_shard_bind)");
    return MMX_E_STATE;
  }
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  return ctx->cfg.dtype == MMX_F64 ? shard_phase1<double>(ctx, s) : shard_phase1<float>(ctx, s);
}

MMX_API int mmx_shard_phase2(mmx_ctx* ctx, int slot, mmx_shard_stats* out) {
  if (!shard_slot_ok(ctx, slot)) return MMX_E_INVALID;
  Slot& s = *ctx->slots[slot];
  std::lock_guard<std::mutex> g(s.mu);
  if (s.shard_world < 1) {
    ctx->set_error("mmx_shard_phase2: slot is not bound to a group (mmx_shard_bind)");
    return MMX_E_STATE;
  }
  MMX_CUDA(ctx, cudaSetDevice(s.device));
  if (int rc = ctx->cfg.dtype == MMX_F64 ? shard_phase2<double>(ctx, s) : shard_phase2<float>(ctx, s)) return rc;
  return shard_collect(ctx, s, out);
}

MMX_API int mmx_shard_run_local(mmx_ctx* ctx, const int32_t* slots, int world, mmx_shard_stats* outs, double* checksum) {
  if (ctx == nullptr || slots == nullptr || world < 1 || world > kMaxPeers) return MMX_E_INVALID;
  for (int r = 0; r < world; ++r) {
    if (!shard_slot_ok(ctx, slots[r])) return MMX_E_INVALID;
    Slot& s = *ctx->slots[slots[r]];
    bool bound = s.shard_rank == r && s.shard_world == world;
    for (int q = 0; bound && q < world; ++q) bound = s.peer_bt[q] == ctx->slots[slots[q]]->d_arr[MMX_ARRAY_BT];
    if (!bound)
      if (int rc = mmx_shard_bind(ctx, slots[r], r, world, nullptr, world > 1 ? slots : nullptr)) return rc;
  }
  // every member's production phase is enqueued before any consumption phase: a member's contraction only
  // waits on events that are already recorded
  for (int r = 0; r < world; ++r)
    if (int rc = mmx_shard_phase1(ctx, slots[r])) return rc;
  std::vector<mmx_shard_stats> local(world);
  for (int r = 0; r < world; ++r) {
    Slot& s = *ctx->slots[slots[r]];
    std::lock_guard<std::mutex> g(s.mu);
    MMX_CUDA(ctx, cudaSetDevice(s.device));
    if (int rc = ctx->cfg.dtype == MMX_F64 ? shard_phase2<double>(ctx, s) : shard_phase2<float>(ctx, s)) return rc;
  }
  double sum = 0.0;
  float fsum = 0.f;
  for (int r = 0; r < world; ++r) {
    Slot& s = *ctx->slots[slots[r]];
    std::lock_guard<std::mutex> g(s.mu);
    if (int rc = shard_collect(ctx, s, &local[r])) return rc;
    // rank order, in the context dtype: the association the program's own loop would use across the blocks
    if (ctx->cfg.dtype == MMX_F64) sum += local[r].partial_trace;
    else fsum += static_cast<float>(local[r].partial_trace);
    if (outs != nullptr) outs[r] = local[r];
  }
  if (checksum != nullptr) *checksum = ctx->cfg.dtype == MMX_F64 ? sum : static_cast<double>(fsum);
  return MMX_OK;
}
