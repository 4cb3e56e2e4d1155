// matmul_ozaki.cu -- gene 8 in FP64 on the 5th-generation tensor cores: c[i][j] += sum_k a[i][k] * bt[j][k]
// (fixtures/matmul.c:25-28) as an error-free INT8 slice decomposition (Ozaki scheme) on tcgen05.mma.kind::i8.
//
// B200 has no FP64 tensor-core kind and its FP64 pipe peaks at 36 TFLOP/s, but INT8 MMAs with INT32 accumulation are
// EXACT and ~120x faster per operation.  Each operand row is scaled by a power of two and cut into S signed 7-bit digits,
//     x = 2^e * (d_1 2^-6 + d_2 2^-13 + ... + d_S 2^-(7S-1)) + r,   |d_t| <= 64,  |r| <= 2^(e - 7S)
// (every step exact in FP64: power-of-two scaling, rint, subtraction of a prefix of x's own bits), so
//     sum_k a_ik b_jk = 2^(ea_i + eb_j + 2) * sum_g 2^(-7g) L_g,        L_g = sum_{t+u=g} sum_k da_t[i][k] db_u[j][k]
// where every L_g is an integer dot product the tensor core computes without rounding (|L_g| <= 7 * K * 2^12 < 2^31 for
// K <= 74k).  Levels g > S + 1 are dropped: |error| <= (S + 3) K 2^(-7S) * max_k|a_ik| max_k|b_jk|, i.e. 2e-14 K max max for
// S = 7 -- below what FP64 accumulation over K terms itself guarantees -- and ZERO whenever the operands carry <= 7S bits
// below their row maximum: on the application's inputs ((i +- k) / N, 14 bits) the result is bit-identical to the CPU program.
//
// Who runs it.  matmul_variant 40 / 41: always, with S = 7 / 6 (general kernels: ~2^-49 / ~2^-42 of K max max).  Auto mode
// (variant 0, N >= 1024; launch_matmul<double> in matmul.cu): only where it is ERROR-FREE.  The slice pass records in a device
// guard whether any element was cut at 7 digits and the highest digit in use per operand; the 6-slice contraction, the 7-slice
// contraction and the FP64-pipe kernel are all enqueued and read the guard: the cheapest error-free form runs, the others leave.
//
// Kernel (one CTA per 128 x 64 tile of c, 1 CTA per SM, the S level accumulators of the tile live in TMEM for the whole
// K loop -- S * 64 <= 448 columns -- so there is no mid-loop drain at all):
//   slice pass  x -> P int8 planes [t][row][k] + one exponent per row (+ the guard)  ((8 + P) N^2 bytes per operand)
//   warp 0      TMA producer: per 64-k stage ONE 3-D box per operand brings the S slices in use ([t][row][64 B], SWIZZLE_64B);
//               2 stages of 84 KB for S = 7, 3 stages of 72 KB for S = 6 (optionally the a slices are multicast over a cluster
//               of column tiles)
//   warp 1      MMA issuer: per 32 k, for t = 1..S: a_t against the slices b_1..b_(S+1-t) STACKED along N (they are
//               contiguous in shared memory, and their products belong to consecutive levels = consecutive TMEM column
//               blocks), split into instructions of N <= 256: 10 MMAs carry the 28 slice products of S = 7, 8 the 21 of S = 6
//   warps 2-5   epilogue: the tile's incoming c and column exponents are fetched before the K loop ends; then L_g -> FP64
//               Horner sum -> exact scaling by 2^(ea_i + eb_j - 12) (ldexp) -> c += .
// Measured on B200, slice passes included (profiles/r1d_*): S = 7 96 / 110 / 119 TFLOP/s of FP64 work at N = 4096 / 8192 /
// 16384; S = 6 as auto mode runs it on the application 133 / 161 / 178 (contraction alone 3.24 POP/s at N = 4096); DMMA 34-35.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "raster.cuh"
#include "tc_ptx.cuh"

namespace mmx {
namespace {

constexpr int OZ_BM = 128, OZ_BN = 64;               // tile of c
constexpr int OZ_THREADS = 192;                      // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue (one per TMEM lane quarter)
constexpr int OZ_KPAD = 64;                          // slice rows are padded to this many k

// BK = k bytes per pipeline stage = bytes per shared-memory row (SWIZZLE_64B or SWIZZLE_32B).  All S slices of both operands
// have to be resident per stage, so a stage is S * 192 * BK bytes: 84 KB (2 stages) at BK = 64, 42 KB (5 stages) at BK = 32.
// Measured (tools/ozaki_cluster_sweep.sh, N = 4096 / 8192): BK = 64 92 / 96 TFLOP/s, BK = 32 with 5 stages 81 / 81, BK = 64
// with the a slices multicast over clusters of 2 / 4 CTAs 93 / 85 -- neither refill latency nor L2 traffic is the limit.
// The tensor pipe is 64 % busy (ncu); the rest goes to shared-memory bandwidth: every MMA re-reads its 4 KB a slice, and the
// narrow tail instructions (N = 64 .. 192) need up to 192 B/clk of operands against the 128 B/clk an SM delivers.
template <int S, int BK> struct OzShape {
  static constexpr int A_SLICE = OZ_BM * BK, B_SLICE = OZ_BN * BK;
  static constexpr int A_BYTES = S * A_SLICE, B_BYTES = S * B_SLICE;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (227 * 1024 - 2048) / STAGE_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 512;  // alignment slack; barriers + column exponents
};

// K-major operand tile whose rows are one swizzle span (BK = 64 or 32 bytes) wide; 8-row groups 8 * BK bytes apart
template <int BK>
__device__ __forceinline__ unsigned long long umma_desc_sw(unsigned smem_addr) {
  return static_cast<unsigned long long>((smem_addr & 0x3FFFF) >> 4) | (static_cast<unsigned long long>((8 * BK) >> 4) << 32) | (1ull << 46) |
         ((BK == 64 ? 4ull : 6ull) << 61);
}
// cute::UMMA::InstrDescriptor for kind::i8: D = S32 (2 @4), A = B = signed 8 bit (1 @7, 1 @10), both K-major, N >> 3 @17, M >> 4 @24
__host__ __device__ constexpr unsigned idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<unsigned>(n >> 3) << 17) | (static_cast<unsigned>(OZ_BM >> 4) << 24);
}
__device__ __forceinline__ void tc_mma_i8(unsigned d_tmem, unsigned long long adesc, unsigned long long bdesc, unsigned idesc,
                                          unsigned accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ double pow2(int e) { return __longlong_as_double(static_cast<long long>(e + 1023) << 52); }

constexpr int kNonFinite = 0x7fffffff;  // row exponent of a row that holds an Inf or a NaN: its products are NaN
// acc * 2^(ea + eb - 12): exact scaling (ldexp also covers results that leave the normal range)
__device__ __forceinline__ double scaled(double acc, int ea, int eb) {
  if (ea == kNonFinite || eb == kNonFinite) return __longlong_as_double(0x7ff8000000000000ll);
  return ldexp(acc, ea + eb - 12);
}

// C = CTAs per cluster: C consecutive column tiles of one tile-row share their a slices -- every CTA fetches 1/C of the rows
// of each slice and multicasts them (the kernel is bound by L2 -> SM traffic otherwise: 84 KB per 64-k stage against
// 1792 tensor-pipe cycles)
template <int S, int C, int BK>
__global__ void __launch_bounds__(OZ_THREADS, 1)
matmul_ozaki_kernel(double* __restrict__ c, const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_a_part,
                    const __grid_constant__ CUtensorMap map_b, const int* __restrict__ exp_a, const int* __restrict__ exp_b, int n, int kq, int row0, int rows, int col0, int cols,
                    int group, int debug_noload, const int* __restrict__ guard) {
  using Sh = OzShape<S, BK>;
  // guarded launch (FP64 auto mode): the slices lost bits of some operand, the FP64-pipe kernel runs instead
  if (guard != nullptr) {  // run iff this is the cheapest error-free form: 6 slices when they suffice, else 7
    const bool ok6 = !ozaki_guard_lossy(guard, 6);
    if (S == 6 ? !ok6 : (ok6 || ozaki_guard_lossy(guard, 7))) return;
  }
  constexpr int OZ_STAGES = Sh::STAGES, OZ_BK = BK;
  extern __shared__ unsigned char smem_raw[];
  const unsigned raw = smem_u32(smem_raw);
  const unsigned base = (raw + 1023u) & ~1023u;
  const unsigned bars = base + OZ_STAGES * Sh::STAGE_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (OZ_STAGES + s); };
  const unsigned done_bar = bars + 8u * (2 * OZ_STAGES);
  const unsigned tmem_slot = bars + 8u * (2 * OZ_STAGES + 1);
  volatile unsigned* tmem_slot_ptr = reinterpret_cast<volatile unsigned*>(smem_raw + (tmem_slot - raw));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const unsigned rank = C > 1 ? cluster_ctarank() : 0u;
  constexpr unsigned short kMask = static_cast<unsigned short>((1u << C) - 1u);
  int sx, by;  // clusters are C consecutive CTAs along x: raster over the grid of clusters
  raster_map(group, static_cast<int>(gridDim.x) / C, static_cast<int>(gridDim.y),
             static_cast<int>(blockIdx.y) * (static_cast<int>(gridDim.x) / C) + static_cast<int>(blockIdx.x) / C, sx, by);
  const int bx = sx * C + static_cast<int>(rank);
  // a rows are absolute; bt rows are relative to the launch's first column (the slice pass writes them that way)
  const int m_base = row0 + by * OZ_BM, n_rel = bx * OZ_BN;
  const int k_stages = kq / OZ_BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), C);  // every CTA of the cluster reads what is multicast into this stage
    }
    mbar_init(done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tmem_slot), "n"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (C > 1) cluster_sync_all();  // peers' barriers are initialised before anything is multicast at them
  tc_fence_after();
  const unsigned tmem_base = *tmem_slot_ptr;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < k_stages; ++kb) {
        const int s = kb % OZ_STAGES;
        mbar_wait(empty_bar(s), ((kb / OZ_STAGES) & 1) ^ 1);
        const unsigned st = base + s * Sh::STAGE_BYTES;
        if (debug_noload) {  // rate probe: the MMAs run on whatever the stage buffers hold
          mbar_arrive(full_bar(s));
          continue;
        }
        mbar_expect_tx(full_bar(s), Sh::STAGE_BYTES);
        if constexpr (C == 1) {
          tma_load_3d(st, &map_a, kb * OZ_BK, m_base, 0, full_bar(s));
        } else {
          constexpr int PART = OZ_BM / C;  // rows of every slice this CTA fetches for the whole cluster
#pragma unroll
          for (int t = 0; t < S; ++t)
            tma_load_3d_mc(st + t * Sh::A_SLICE + rank * (PART * OZ_BK), &map_a_part, kb * OZ_BK, m_base + static_cast<int>(rank) * PART, t,
                           full_bar(s), kMask);
        }
        tma_load_3d(st + Sh::A_BYTES, &map_b, kb * OZ_BK, n_rel, 0, full_bar(s));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < k_stages; ++kb) {
        const int s = kb % OZ_STAGES;
        mbar_wait(full_bar(s), (kb / OZ_STAGES) & 1);
        tc_fence_after();
        const unsigned st = base + s * Sh::STAGE_BYTES;
#pragma unroll
        for (int ks = 0; ks < OZ_BK / 32; ++ks) {
          const unsigned long long adv = 2ull * ks;  // 32 bytes along K inside the 64-byte swizzle row
#pragma unroll
          for (int t = 1; t <= S; ++t) {
            const unsigned long long a_t = umma_desc_sw<BK>(st + (t - 1) * Sh::A_SLICE) + adv;
            const unsigned first = (kb | ks | (t - 1)) != 0;  // t = 1 of the very first step initialises every level
            const int count = S + 1 - t;                      // slices b_1 .. b_count pair with a_t (levels t+1 .. S+1)
#pragma unroll
            for (int u0 = 0; u0 < count; u0 += 4) {
              const int nsl = count - u0 < 4 ? count - u0 : 4;
              const unsigned long long b_u = umma_desc_sw<BK>(st + Sh::A_BYTES + u0 * Sh::B_SLICE) + adv;
              // level of (t, u0 + 1) is t + u0 + 1; its TMEM column block is level - 2
              tc_mma_i8(tmem_base + (t - 1 + u0) * OZ_BN, a_t, b_u, idesc_i8(nsl * OZ_BN), first);
            }
          }
        }
        if constexpr (C == 1) tc_commit(empty_bar(s));
        else tc_commit_mc(empty_bar(s), kMask);
      }
      tc_commit(done_bar);
    }
  } else {
    // epilogue: thread = one row of the tile (TMEM lane).  Its 64 incoming c values and the tile's column exponents do not
    // depend on the MMAs: they are fetched NOW and sit in registers / shared memory while the K loop runs, so that after
    // the last MMA only TMEM reads, the Horner sums and the stores remain (the dependent load-add-store chain per 8 columns
    // cost ~25 us per tile, a quarter of the tile time at N = 4096)
    const int q = warp % 4;
    const int m = m_base + q * 32 + lane;
    const int m_limit = row0 + rows;
    const bool row_ok = m < m_limit;
    const int ei = row_ok ? exp_a[m] : 0;  // kNonFinite marks a row that holds an Inf or a NaN
    double* crow = c + static_cast<size_t>(row_ok ? m : 0) * n;
    const bool vec_ok = (n % 2 == 0) && (col0 % 2 == 0);
    int* eb_sh = reinterpret_cast<int*>(smem_raw + (bars + 128 - raw));  // 64 column exponents of this tile
    {
      const int t = threadIdx.x - 64;  // 0..127 over the four epilogue warps
      if (t < OZ_BN) eb_sh[t] = n_rel + t < cols ? exp_b[n_rel + t] : 0;
    }
    double cpre[OZ_BN];
#pragma unroll
    for (int e = 0; e < OZ_BN; e += 2) {
      const int jr = n_rel + e;
      if (row_ok && vec_ok && jr + 2 <= cols) {
        const double2 x = *reinterpret_cast<const double2*>(crow + col0 + jr);
        cpre[e] = x.x;
        cpre[e + 1] = x.y;
      } else {
        cpre[e] = (row_ok && jr < cols) ? crow[col0 + jr] : 0.0;
        cpre[e + 1] = (row_ok && jr + 1 < cols) ? crow[col0 + jr + 1] : 0.0;
      }
    }
    asm volatile("bar.sync 1, 128;\n" ::: "memory");  // eb_sh is complete (the four epilogue warps only)
    mbar_wait(done_bar, 0);
    tc_fence_after();
    const unsigned t0 = tmem_base + (static_cast<unsigned>(q * 32) << 16);
#pragma unroll
    for (int cb = 0; cb < OZ_BN / 8; ++cb) {
      unsigned lv[S][8];
#pragma unroll
      for (int g = 0; g < S; ++g) tc_ld8_issue(t0 + g * OZ_BN + cb * 8, lv[g]);
      tc_ld_wait();
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        const int jr = n_rel + cb * 8 + e;  // relative to col0
        double v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double acc = static_cast<double>(static_cast<int>(lv[S - 1][e + h]));
#pragma unroll
          for (int g = S - 2; g >= 0; --g) acc = fma(acc, 0.0078125, static_cast<double>(static_cast<int>(lv[g][e + h])));
          v[h] = cpre[cb * 8 + e + h] + scaled(acc, ei, eb_sh[cb * 8 + e + h]);
        }
        if (!row_ok) continue;
        const int j = col0 + jr;
        if (vec_ok && jr + 2 <= cols) {
          *reinterpret_cast<double2*>(crow + j) = make_double2(v[0], v[1]);
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (jr + h < cols) crow[j + h] = v[h];
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(512) : "memory");
  }
  if constexpr (C > 1) cluster_sync_all();  // no CTA leaves while a peer may still signal its barriers
}

// One CTA per row: row maximum -> exponent e (|x| < 2^e), then S digits per element.  dst plane t of row r (relative
// index) is dst + t * plane + r * kq; k >= n is zero.  Rows [src_row0, src_row0 + nrows) of src; rows up to nrows_pad are
// written as zeros with exponent 0 (tile overhang inside the tensor map).
template <int S>
__global__ void __launch_bounds__(256, 4) ozaki_slice_kernel(const double* __restrict__ src, signed char* __restrict__ dst, int* __restrict__ exps,
                                                          size_t plane, int n, int kq, int src_row0, int nrows, int dst_row0,
                                                          int* __restrict__ guard, int lossy_slot, int top_slot) {
  __shared__ double red[8];
  __shared__ int top_sh[8];
  __shared__ int e_sh;
  const int r = blockIdx.x;  // relative row
  const int tid = threadIdx.x;
  const bool live = r < nrows;
  const double* x = src + static_cast<size_t>(src_row0 + (live ? r : 0)) * n;
  // 4 consecutive k per thread and iteration: a warp reads 1 KB and writes 128 bytes per slice, both contiguous.  The first
  // KEEP iterations (rows up to 4096 elements) stay in registers between the two passes, so the row is read once.
  constexpr int KEEP = 4;
  const bool vec = n % 2 == 0;
  auto load4 = [&](int k0, double (&v)[4]) {
    if (live && vec && k0 + 4 <= n) {
      const double2 p = *reinterpret_cast<const double2*>(x + k0), q2 = *reinterpret_cast<const double2*>(x + k0 + 2);
      v[0] = p.x; v[1] = p.y; v[2] = q2.x; v[3] = q2.y;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = (live && k0 + q < n) ? x[k0 + q] : 0.0;
    }
  };
  double mx = 0.0;
  int bad = 0;
  auto scan4 = [&](const double (&v)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      bad |= !isfinite(v[q]);
      mx = fmax(mx, fabs(v[q]));
    }
  };
  double keep[KEEP][4];
#pragma unroll
  for (int it = 0; it < KEEP; ++it) {
    const int k0 = (it * 256 + tid) * 4;
    if (k0 < kq) {
      load4(k0, keep[it]);
      scan4(keep[it]);
    }
  }
  for (int k0 = (KEEP * 256 + tid) * 4; k0 < kq; k0 += 256 * 4) {
    double v[4];
    load4(k0, v);
    scan4(v);
  }
  bad = __syncthreads_or(bad);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (tid % 32 == 0) red[tid / 32] = mx;
  __syncthreads();
  if (tid == 0) {
    double m = red[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) m = fmax(m, red[w]);
    const int e = (m > 0.0 && !bad) ? ilogb(m) + 1 : 0;
    e_sh = e;
    exps[dst_row0 + r] = bad ? kNonFinite : e;
  }
  __syncthreads();
  // exact power of two; a non-finite row gets zero digits, and so does a row whose maximum is below 2^-970 (1 / 2^e would
  // overflow): both are flagged as lossy.  (Digit extraction by 64-bit integer arithmetic was measured slower than
  // the FP64 form below: 85 us against 70 us per operand at N = 4096.)
  const bool tiny = e_sh < -970;
  const double inv = (live && !bad && !tiny) ? scalbn(1.0, -e_sh) : 0.0;
  signed char* drow = dst + static_cast<size_t>(dst_row0 + r) * kq;
  int lossy = bad | tiny, top = 0;  // top = highest non-zero digit (1-based) this thread has seen
  auto emit4 = [&](int k0, const double (&v)[4]) {
    int dig[S] = {};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double rem = bad ? 0.0 : v[q] * inv;
#pragma unroll
      for (int t = 0; t < S; ++t) {
        if (rem == 0.0) break;  // nothing left: the remaining digits are zero (short operands finish after a digit or two)
        const double up = pow2(7 * (t + 1) - 1), down = pow2(-(7 * (t + 1) - 1));
        // rint without the conversion units (they would bound this pass): adding 1.5 * 2^52 rounds to the integer grid
        // (ties to even) and leaves the integer in the low word of the sum
        const double shifted = fma(rem, up, 6755399441055744.0);
        const int d = __double2loint(shifted);
        rem = fma(-(shifted - 6755399441055744.0), down, rem);  // exact: removes a prefix of rem's bits
        dig[t] |= (d & 0xff) << (8 * q);
      }
      lossy |= rem != 0.0;  // bits below the last digit: the slices do not reproduce this element exactly
    }
#pragma unroll
    for (int t = 0; t < S; ++t) {
      if (dig[t] != 0) top = max(top, t + 1);
      *reinterpret_cast<int*>(drow + t * plane + k0) = dig[t];
    }
  };
#pragma unroll
  for (int it = 0; it < KEEP; ++it) {
    const int k0 = (it * 256 + tid) * 4;
    if (k0 < kq) emit4(k0, keep[it]);
  }
  for (int k0 = (KEEP * 256 + tid) * 4; k0 < kq; k0 += 256 * 4) {
    double v[4];
    load4(k0, v);
    emit4(k0, v);
  }
  if (guard != nullptr) {
    lossy = __syncthreads_or(lossy);
    top = __reduce_max_sync(0xffffffffu, top);
    if (tid % 32 == 0) top_sh[tid / 32] = top;
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int w = 1; w < 8; ++w) top = max(top, top_sh[w]);
      if (lossy && guard[lossy_slot] == 0) atomicOr(guard + lossy_slot, 1);
      if (top > guard[top_slot]) atomicMax(guard + top_slot, top);  // read first: after a few rows nobody needs the atomic
    }
  }
}

// [S][rows][kq] bytes; box = 64 bytes x box_rows rows x S slices; 64-byte swizzle
bool make_slice_map(CUtensorMap* map, const signed char* ptr, size_t rows, int kq, int bk, int box_rows, int slices, int box_slices) {
  EncodeTiledFn enc = encode_tiled();
  if (enc == nullptr) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kq), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(slices)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(kq), static_cast<cuuint64_t>(kq) * rows};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(bk), static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(box_slices)};
  const cuuint32_t elem[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<signed char*>(ptr), dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
             bk == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline int oz_kq(int n) { return (n + OZ_KPAD - 1) / OZ_KPAD * OZ_KPAD; }
inline size_t oz_rows_pad(int rows, int tile) { return static_cast<size_t>((rows + tile - 1) / tile) * tile; }

template <int S, int C, int BK>
cudaError_t oz_configure() {
  static PerDeviceOnce once;
  bool& configured = once.here();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(matmul_ozaki_kernel<S, C, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, OzShape<S, BK>::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  return cudaSuccess;
}

// Where things live in `scratch` for P digit planes: a slices [P][n][kq] (absolute rows), bt slices [P][pad64(n)][kq] (rows
// relative to the launch's first column), row exponents, the guard words.
struct OzLayout {
  int kq;
  size_t a_plane, b_rows, b_plane;
  signed char *sa, *sb;
  int *ea, *eb, *guard;
  OzLayout(void* scratch, int n, int planes) {
    kq = oz_kq(n);
    a_plane = static_cast<size_t>(n) * kq;
    b_rows = oz_rows_pad(n, OZ_BN);
    b_plane = b_rows * kq;
    sa = static_cast<signed char*>(scratch);
    sb = sa + planes * a_plane;
    ea = reinterpret_cast<int*>(sb + planes * b_plane);
    eb = ea + n;
    guard = eb + n + OZ_BN;  // {a is cut, top digit of a, top digit of bt, bt is cut}
  }
};

// the slice passes (P planes); with_guard: also record whether anything was cut and the highest digits in use
template <int P>
cudaError_t oz_slices(const double* a, const double* bt, void* scratch, int n, int row0, int rows, int col0, int cols, cudaStream_t stream,
                      bool with_guard, bool reuse_a) {
  const OzLayout L(scratch, n, P);
  int* flag = with_guard ? L.guard : nullptr;
  if (with_guard)
    if (cudaError_t e = reuse_a ? cudaMemsetAsync(flag + 2, 0, 2 * sizeof(int), stream) : cudaMemsetAsync(flag, 0, 4 * sizeof(int), stream);
        e != cudaSuccess)
      return e;
  const int cols_pad = static_cast<int>(oz_rows_pad(cols, OZ_BN));
  if (!reuse_a) ozaki_slice_kernel<P><<<rows, 256, 0, stream>>>(a, L.sa, L.ea, L.a_plane, n, L.kq, row0, rows, row0, flag, 0, 1);
  ozaki_slice_kernel<P><<<cols_pad, 256, 0, stream>>>(bt, L.sb, L.eb, L.b_plane, n, L.kq, col0, cols, 0, flag, 3, 2);
  return cudaGetLastError();
}

// the contraction over the first S of P planes; guarded: the kernel reads the guard and runs only if it is the cheapest
// error-free form
template <int S, int C, int BK>
cudaError_t oz_contract(double* c, void* scratch, int planes, int n, int row0, int rows, int col0, int cols, cudaStream_t stream, bool guarded) {
  if (cudaError_t e = oz_configure<S, C, BK>(); e != cudaSuccess) return e;
  const OzLayout L(scratch, n, planes);
  CUtensorMap map_a, map_a_part, map_b;
  if (!make_slice_map(&map_a, L.sa, static_cast<size_t>(n), L.kq, BK, OZ_BM, planes, S) ||
      !make_slice_map(&map_a_part, L.sa, static_cast<size_t>(n), L.kq, BK, OZ_BM / C, planes, 1) ||
      !make_slice_map(&map_b, L.sb, L.b_rows, L.kq, BK, OZ_BN, planes, S))
    return cudaErrorNotSupported;
  const int col_tiles = (cols + OZ_BN - 1) / OZ_BN;
  static const int noload = [] { const char* e = getenv("MMX_OZ_NOLOAD"); return (e && C == 1) ? atoi(e) : 0; }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((col_tiles + C - 1) / C * C, (rows + OZ_BM - 1) / OZ_BM);  // whole clusters; surplus tiles are masked
  cfg.blockDim = dim3(OZ_THREADS);
  cfg.dynamicSmemBytes = OzShape<S, BK>::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, matmul_ozaki_kernel<S, C, BK>, c, map_a, map_a_part, map_b, static_cast<const int*>(L.ea),
                            static_cast<const int*>(L.eb), n, L.kq, row0, rows, col0, cols, raster_group(OZ_BM, static_cast<size_t>(L.kq)), noload,
                            static_cast<const int*>(guarded ? L.guard : nullptr));
}

// slices + contraction with S planes (the explicit variants)
template <int S, int C, int BK>
cudaError_t oz_go(double* c, const double* a, const double* bt, void* scratch, int n, int row0, int rows, int col0, int cols,
                  cudaStream_t stream, bool reuse_a = false) {
  if (cudaError_t e = oz_slices<S>(a, bt, scratch, n, row0, rows, col0, cols, stream, false, reuse_a); e != cudaSuccess) return e;
  return oz_contract<S, C, BK>(c, scratch, S, n, row0, rows, col0, cols, stream, false);
}

}  // namespace

// |L_g| <= 7 * K * 2^12 must stay below 2^31
bool matmul_ozaki_usable(int n) { return n >= 1 && n <= 65536 && encode_tiled() != nullptr; }

cudaError_t matmul_ozaki_prepare() {
  if (encode_tiled() == nullptr) return cudaErrorNotSupported;
  if (cudaError_t e = oz_configure<7, 1, 32>(); e != cudaSuccess) return e;
  if (cudaError_t e = oz_configure<7, 1, 64>(); e != cudaSuccess) return e;
  if (cudaError_t e = oz_configure<7, 2, 64>(); e != cudaSuccess) return e;
  if (cudaError_t e = oz_configure<7, 4, 64>(); e != cudaSuccess) return e;
  return oz_configure<6, 1, 64>();
}

size_t matmul_ozaki_scratch_bytes(int n) {
  const size_t kq = static_cast<size_t>(oz_kq(n));
  return 7 * (static_cast<size_t>(n) + oz_rows_pad(n, OZ_BN)) * kq + 2 * (static_cast<size_t>(n) + OZ_BN) * sizeof(int) + 256;  // + the guard flag
}

cudaError_t launch_matmul_ozaki(double* c, const double* a, const double* bt, void* scratch, int n, int row0, int rows, int col0, int cols,
                                int slices, cudaStream_t stream, int** guard_out, bool reuse_a) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (scratch == nullptr) return cudaErrorInvalidValue;
  if (guard_out != nullptr) {
    // auto mode: 7 digit planes and the guard once, then the 6-slice and the 7-slice contraction, each guarded; the caller
    // adds the FP64-pipe kernel under the remaining condition
    *guard_out = OzLayout(scratch, n, 7).guard;
    if (cudaError_t e = oz_slices<7>(a, bt, scratch, n, row0, rows, col0, cols, stream, true, reuse_a); e != cudaSuccess) return e;
    if (cudaError_t e = oz_contract<6, 1, 64>(c, scratch, 7, n, row0, rows, col0, cols, stream, true); e != cudaSuccess) return e;
    return oz_contract<7, 1, 64>(c, scratch, 7, n, row0, rows, col0, cols, stream, true);
  }
  if (reuse_a) return oz_go<7, 1, 64>(c, a, bt, scratch, n, row0, rows, col0, cols, stream, true);
  // tuning hooks (tools/ozaki_cluster_sweep.sh): CTAs per cluster sharing the a slices by multicast, k bytes per stage
  static const int cluster = [] { const char* e = getenv("MMX_OZ_CLUSTER"); return e ? atoi(e) : 1; }();
  static const int bk = [] { const char* e = getenv("MMX_OZ_BK"); return e ? atoi(e) : 64; }();
  if (slices == 6) return oz_go<6, 1, 64>(c, a, bt, scratch, n, row0, rows, col0, cols, stream);
  if (cluster == 4) return oz_go<7, 4, 64>(c, a, bt, scratch, n, row0, rows, col0, cols, stream);
  if (cluster == 2) return oz_go<7, 2, 64>(c, a, bt, scratch, n, row0, rows, col0, cols, stream);
  if (bk == 32) return oz_go<7, 1, 32>(c, a, bt, scratch, n, row0, rows, col0, cols, stream);
  return oz_go<7, 1, 64>(c, a, bt, scratch, n, row0, rows, col0, cols, stream);
}

}  // namespace mmx
