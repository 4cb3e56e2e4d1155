// kernels.cuh -- launchers of the sm_100a kernel library: one kernel family per offloadable
// loop of /root/reference/proj/fixtures/matmul.c (catalogue in plan.cpp).
//
// Every launcher enqueues on `stream` and returns the launch status; none synchronises.
// Iterations of host-driven outer loops are passed as IterRef so that one captured CUDA
// graph can replay a train of launches: the kernel adds a device-resident base counter to a
// per-node constant.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mmx {

// Which iteration of the enclosing host loop(s) a launch serves: value = off + (base ? *base : 0).
// cudaFuncSetAttribute applies to the current device only: one flag per device ordinal (a context may own
// slots on all 8 GPUs of a box)
struct PerDeviceOnce {
  bool done[64] = {};
  bool& here() {
    int d = 0;
    cudaGetDevice(&d);
    return done[d & 63];
  }
};

struct IterRef {
  const int* base;  // device pointer or nullptr
  int off;
};

enum FillOp { FILL_INIT_A = 0, FILL_INIT_B = 1, FILL_ZERO = 2 };

// genes 0,2,4: dst[i][j] = op(i,j) over the whole n x n array (matmul.c:8-18)
// rows [row0, row0+rows) only (row0 = 0, rows = n for the whole nest; the row-sharded multi-GPU path passes its block)
template <typename T> cudaError_t launch_fill2d(int op, T* dst, int n, int row0, int rows, cudaStream_t stream);
// genes 1,3,5: one row i = iter of the same
template <typename T> cudaError_t launch_fill_row(int op, T* dst, int n, IterRef iter, cudaStream_t stream);

// gene 6: bt[i][j] = b[j][i] (matmul.c:21-23)
// rows [row0, row0+rows) of bt only (= columns of b)
template <typename T> cudaError_t launch_transpose(T* bt, const T* b, int n, int row0, int rows, cudaStream_t stream);
// Row-sharded run: rows [row0, row0+rows) of bt are produced once and stored into the bt of
// every GPU of the group (peer-mapped pointers; p[0..count) includes this GPU's own array).
constexpr int kMaxPeers = 8;
struct BtPeers {
  void* p[kMaxPeers] = {};
  int count = 0;
};
template <typename T> cudaError_t launch_transpose_push(const BtPeers& peers, const T* b, int n, int row0, int rows, cudaStream_t stream);
// gene 7: row i of bt = column i of b
template <typename T> cudaError_t launch_transpose_row(T* bt, const T* b, int n, IterRef iter, cudaStream_t stream);

// ---- producers that also write an operand's digit planes for gene 8 (ozaki_digits.cuh, matmul_ozaki.cu) -----------------
// Where one operand's planes live inside a context's scratch (matmul_ozaki_operand): plane t of row r at planes + t * plane +
// r * kq, one exponent per row, the guard words and which of them belong to this operand.
struct OzOperand {
  signed char* planes = nullptr;
  size_t plane = 0;
  int kq = 0;
  int* exps = nullptr;
  int* guard = nullptr;
  int lossy_slot = 0, top_slot = 0, dirty_slot = 0;
};
// which = 0: a (rows absolute), 1: bt (rows relative to the launch's first column: whole-nest launches only)
OzOperand matmul_ozaki_operand(void* scratch, int n, int which);
// the fused producers cover whole-nest launches of sizes whose planes need no padding
inline bool ozaki_fusable(int n) { return n >= 1024 && n % 64 == 0; }
// gene 0 over the whole array + the digit planes, row exponents and guard words of a (the values are in registers; the row
// maximum of (i + j) / N is its last element)
template <typename T> cudaError_t launch_fill_a_planes(T* a, int n, const OzOperand& pa, cudaStream_t stream);
// gene 2 over the whole array + colexp[j] = digit exponent of COLUMN j of b (= row j of bt), known in closed form for
// (i - j) / N: what launch_transpose_planes needs before it can emit digits
template <typename T> cudaError_t launch_fill_b_colexp(T* b, int n, int* colexp, cudaStream_t stream);
// gene 6 over the whole array + the digit planes and guard words of bt, given pb.exps[j] for every row j of bt
template <typename T> cudaError_t launch_transpose_planes(T* bt, const T* b, int n, const OzOperand& pb, cudaStream_t stream);
// init-b + transpose + planes as ONE kernel (a plan that maps both nests to the device whole): the transpose computes its tiles of b,
// writes them to b and goes on as above -- b is never read back.  launch_b_colexp: the exponents of bt's rows it needs beforehand
template <typename T> cudaError_t launch_b_colexp(int n, int* colexp, cudaStream_t stream);
// (b == NULL: the tiles are computed but b itself is not stored -- the caller writes it with launch_fill2d beside the contraction)
template <typename T> cudaError_t launch_fill_b_transpose_planes(T* b, T* bt, int n, const OzOperand& pb, cudaStream_t stream);

// gene 8: c[i][j] += sum_k a[i][k] * bt[j][k] (matmul.c:25-28).  variant: 1 SIMT, 2 DMMA (FP64 only).
// Rows [row0, row0+rows) of a and c, columns [col0, col0+cols) of c (= rows of bt) only: the whole nest is
// (0, n, 0, n); the row-sharded multi-GPU path passes its row block and walks the column blocks in the
// order the owners' rows of bt arrive.
// `scratch` (may be NULL): matmul_3xtf32_scratch_bytes(n) bytes of device memory; with it, FP32 FAST
// launches at n >= kTcMinN (or variants 30 / 31) run on the tcgen05 tensor cores (matmul_tc.cu).
template <typename T>
cudaError_t launch_matmul(T* c, const T* a, const T* bt, int n, int row0, int rows, int col0, int cols, bool strict,
                          int variant, void* scratch, cudaStream_t stream);

// FP32 on the 5th-generation tensor cores as three TF32 products per term with two-level accumulation
constexpr int kTcMinN = 1024;
bool matmul_3xtf32_usable(int n);
size_t matmul_3xtf32_scratch_bytes(int n);
cudaError_t matmul_3xtf32_prepare();  // per device, before the first launch (not inside a stream capture)
// wide: 128 x 256 tile with plain FP32 masters (faster, looser); default 128 x 128 with compensated masters
cudaError_t launch_matmul_3xtf32(float* c, const float* a, const float* bt, void* scratch, int n, int row0, int rows, int col0,
                                 int cols, bool wide, cudaStream_t stream, bool reuse_a = false, const int* run_if = nullptr);
// FP64 on the 5th-generation tensor cores as exact INT8 slice products (Ozaki scheme, matmul_ozaki.cu); `slices` = 7 (default,
// |error| <= 2e-14 K max|a| max|b|, bit-identical on the application's inputs) or 6
bool matmul_ozaki_usable(int n);
size_t matmul_ozaki_scratch_bytes(int n);
cudaError_t matmul_ozaki_prepare();  // per device, before the first launch (not inside a stream capture)
// guard_out (may be NULL): the slice pass also records in a device flag whether any operand element lost bits (or is not
// finite); the contraction then runs only if none did, and *guard_out receives the flag's address so that the caller can
// enqueue the FP64-pipe kernel under the opposite condition (FP64 auto mode: tensor cores exactly when they are error-free)
constexpr int kOzMinN = 1024;
// The guard: g[0] / g[3] != 0 when some element of a / of bt has bits below its 7th digit (or is not finite); g[1], g[2] =
// highest non-zero digit (1-based) anywhere in a / in bt.  The S-slice contraction uses digits 1..S and keeps the digit pairs
// with t + u <= S + 1, so it is error-free exactly when no element is cut, no digit beyond S is set and every non-zero pair
// is kept.  Auto mode runs the cheapest error-free form: 2 .. 7 slices, else the FP64 pipe.
#ifdef __CUDACC__
__device__ __forceinline__ bool ozaki_guard_lossy(const int* g, int slices) {
  return (g[0] | g[3]) != 0 || g[1] > slices || g[2] > slices || g[1] + g[2] > slices + 1;
}
#endif
// The cheapest error-free form for the operands the guard describes (g = {a cut, top digit of a, top digit of bt, bt cut}), as
// OzPShape::CODE; 0 when none is (the FP64-pipe kernel runs).  Rectangular forms where both operands use at most four
// digits; beyond that the triangular forms, which are error-free when every non-zero pair lies inside the triangle.
#ifdef __CUDACC__
__host__ __device__
#endif
inline int ozaki_pick_form(int cut, int top_a, int top_b) {
  if (cut) return 0;
  const int ta = top_a < 1 ? 1 : top_a, tb = top_b < 1 ? 1 : top_b;
  if (ta <= 2 && tb <= 2) return 223;
  if (ta <= 3 && tb <= 2) return 324;
  if (ta <= 2 && tb <= 3) return 234;
  if (ta <= 3 && tb <= 3) return 335;
  if (ta <= 4 && tb <= 3) return 436;
  if (ta <= 3 && tb <= 4) return 346;
  if (ta <= 4 && tb <= 4) return 447;
  for (int s = 5; s <= 7; ++s)
    if (ta <= s && tb <= s && ta + tb <= s + 1) return s * 111;
  return 0;
}

// The INT32 level accumulators: a level with p digit pairs stays within p K 2^14 (8-bit digits: |d d'| <= 2^14); p = min(SA, SB)
// for every form.  False: the form must not run on K = kq terms (auto mode then takes the fallback).
#ifdef __CUDACC__
__host__ __device__
#endif
inline bool oz_form_fits_int32(int form, int kq) {
  const int sa = form / 100, sb = form / 10 % 10;
  const int p = sa < sb ? sa : sb;
  return static_cast<long long>(p) * kq < (1ll << 17);
}

// FP32 auto mode has the forms whose epilogue is the TMA reduction (all but the 6 / 7-slice ones); beyond them: split TF32
#ifdef __CUDACC__
__host__ __device__
#endif
inline int ozaki_pick_form_f32(int cut, int top_a, int top_b) {
  const int f = ozaki_pick_form(cut, top_a, top_b);
  return (f == 666 || f == 777) ? 0 : f;
}

// FP32 auto mode (variant 0, FAST, n >= kOzMinN, n % 4 == 0): the INT8 forms first, split TF32 as the guarded fallback.  The
// context's scratch then holds the split-TF32 area followed (1 KB aligned) by the digit planes.  MMX_F32_INT8=0 switches it off.
bool fp32_int8_enabled(int n);
size_t fp32_int8_scratch_offset(int n);

// OR-ed into `variant`: the rows [row0, row0 + rows) of a were already re-encoded into `scratch` by the previous launch_matmul
// on it (the row-sharded run contracts the same rows of a against one column block after another)
constexpr int kReuseOperandA = 0x1000;
// OR-ed into `variant` (FP64 auto mode): BOTH operands are as the previous launch_matmul on this scratch encoded them -- the launch is
// the contraction (and the guarded FP64-pipe launch) alone.  For timing the contraction kernel by itself (mmx_time_gene8_contraction).
constexpr int kReuseOperands = 0x2000;
// OR-ed into `variant` (auto mode): the digit planes, row exponents and guard words of bt are valid for this launch's columns -- the
// kernel that produced bt wrote them (launch_transpose_planes).  kReuseOperandA | kReuseOperandBt == kReuseOperands in effect.
constexpr int kReuseOperandBt = 0x4000;
// OR-ed into `variant` (auto mode): every element of c this launch covers is +0 (the zero-c kernel ran and nothing has written c
// since): the tensor-core epilogue then STORES its results instead of asking the L2 to add them to c (0 + v == v bit for bit; the
// exact integer level sums never produce -0), which spares the read of c.  The FP64-pipe / split-TF32 fallbacks ignore it.
constexpr int kCIsZero = 0x8000;
// Auto mode inside a CUDA-graph capture: instead of enqueueing the fallback (FP64 pipe / split TF32) as guarded launches that retire
// at once when an INT8 form took the product (5 us in FP64, 19 us in FP32 per individual), the fallback goes into the body of a
// conditional IF node whose condition the auto kernel sets on the device (cudaGraphSetConditional): no form => run the body.
// begin() before the auto launch (no-op unless `stream` is capturing), body_begin() after it, the fallback launches on body_stream(),
// body_end().  Outside a capture everything stays as it was (active == false).  MMX_GRAPH_COND=0 switches it off.
struct OzFallbackCond {
  bool active = false;
  unsigned long long handle = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphNode_t node = nullptr;
  cudaStream_t side = nullptr;   // the stream the body is captured on
  cudaError_t begin(cudaStream_t stream);
  cudaError_t body_begin(cudaStream_t stream);
  cudaError_t body_end(cudaStream_t stream);
  void abandon();  // an error between begin() and body_begin(): hand the borrowed stream back
  cudaStream_t body_stream(cudaStream_t stream) const { return active ? side : stream; }
};
cudaError_t launch_matmul_ozaki(double* c, const double* a, const double* bt, void* scratch, int n, int row0, int rows, int col0,
                                int cols, int slices, cudaStream_t stream, int** guard_out = nullptr, bool reuse_a = false, bool reuse_bt = false,
                                bool c_zero = false, const OzFallbackCond* cond = nullptr);
cudaError_t launch_matmul_ozaki_f32(float* c, const float* a, const float* bt, void* scratch, int n, int row0, int rows, int col0, int cols,
                                    cudaStream_t stream, int** guard_out, bool reuse_a = false, bool reuse_bt = false, bool c_zero = false,
                                    const OzFallbackCond* cond = nullptr);
// device word in `scratch` where the auto launch records the form it ran: 2 .. 7 slices, 0 = left to the FP64 pipe
int* matmul_ozaki_form_word(void* scratch, int n);
// gene 9: row i of the same (GEMV against bt)
template <typename T>
cudaError_t launch_gemv_row(T* c, const T* a, const T* bt, int n, IterRef iter, bool strict, cudaStream_t stream);
// gene 10: one element (i, j): flat iteration f = i*n + j
template <typename T>
cudaError_t launch_dot(T* c, const T* a, const T* bt, int n, IterRef flat_iter, bool strict, cudaStream_t stream);

// gene 11: *sum = sum_i c[i][i] (matmul.c:30-32)
// diagonal entries i in [row0, row0+rows)
template <typename T> cudaError_t launch_trace(T* sum, const T* c, int n, int row0, int rows, bool strict, cudaStream_t stream);

// graph plumbing: *counter += delta
cudaError_t launch_advance(int* counter, int delta, cudaStream_t stream);

// L2 helpers for benchmarking: overwrite `bytes` at p / read them (evicts, leaves only clean lines)
cudaError_t launch_scrub(void* p, std::size_t bytes, cudaStream_t stream);
cudaError_t launch_evict(void* p, std::size_t bytes, cudaStream_t stream);

// peak probes (peaks.cu); each returns the achieved rate through *value
cudaError_t probe_peak(int kind, double* value);

constexpr int kNumSMs = 148;  // B200

}  // namespace mmx
