// matmul_ozaki.cu -- gene 8 in FP64 on the 5th-generation tensor cores: c[i][j] += sum_k a[i][k] * bt[j][k]
// (fixtures/matmul.c:25-28) as an error-free INT8 slice decomposition (Ozaki scheme) on tcgen05.mma.kind::i8.
//
// B200 has no FP64 tensor-core kind and its FP64 pipe peaks at 36 TFLOP/s, but INT8 MMAs with INT32 accumulation are
// EXACT and ~120x faster per operation.  Each operand row is scaled by a power of two and cut into S signed 8-bit digits
// (ozaki_digits.cuh):
//     x = +-2^e * (d_1 2^-7 + d_2 2^-15 + ... + d_S 2^-(8S-1)) + r,   -128 <= d_t <= 127,  |r| <= 2^(e - 8S)
// (every step exact in FP64: power-of-two scaling, rounding to an integer, subtraction of a prefix of x's own bits; the sign: a row
// whose largest element would need d_1 = +128 is encoded negated), so
//     sum_k a_ik b_jk = +-2^(ea_i + eb_j + 2) * sum_g 2^(-8g) L_g,        L_g = sum_{t+u=g} sum_k da_t[i][k] db_u[j][k]
// where every L_g is an integer dot product the tensor core computes without rounding: per term |d_t d_u| <= 2^14, so a level with
// p digit pairs stays within p K 2^14 -- inside INT32 while K p < 2^17 (p <= 3 at K = 32768, any p up to K = 16384;
// oz_form_fits_int32 refuses the rest).  Levels g > S + 1 are dropped:
// |error| <= (S + 3) K 2^(-7S) * max_k|a_ik| max_k|b_jk| (the bound of 7-bit digits; the 8-bit ones are inside it), i.e.
// 2e-14 K max max for S = 7 -- below what FP64 accumulation over K terms itself guarantees -- and ZERO whenever the operands
// carry <= 8S - 1 bits below their row maximum: on the application's inputs ((i +- k) / N: 14 bits at N = 4096; two digits hold both
// operands up to N = 16384 and bt at N = 32768) the result is bit-identical to the CPU program.
//
// Who runs it.  matmul_variant 40 .. 45: always, as the triangular form with S = 7 .. 2 slices (general kernels: ~2^-49 .. of
// K max max).  Auto mode (variant 0, N >= 1024; launch_matmul<double> in matmul.cu): only where it is ERROR-FREE.  The slice pass
// records in a device guard whether any element was cut at 7 digits and the highest digit in use per operand; ONE persistent launch
// reads the guard and runs the cheapest error-free form (rectangular SA x SB digit pairs up to four digits per operand, the
// triangular 5 / 6 / 7-slice forms beyond), or leaves at once, in which case the FP64-pipe kernel enqueued behind it runs
// (ozaki_pick_form in kernels.cuh is the rule; mmx_gene8_form reports the choice).
//
// Kernels, in file order:
//   matmul_ozaki_kernel<S, C, BK>   the first version, one CTA per 128 x 64 tile (MMX_OZ_LEGACY=1; kept as the A/B reference
//                                   and for its cluster / stage-width tuning hooks)
//   oz_persist_body<SA, SB, LV, BN, CR, CX, CY>   the persistent form described at its definition: one CTA per SM walks the
//                                   tiles; warp 0 = TMA producer, warp 1 = MMA issuer, warps 2-9 = epilogue.  Per 32 k, slice
//                                   a_t meets the slices b_1..b_count STACKED along N (contiguous in shared memory, products of
//                                   consecutive levels = consecutive TMEM column blocks) in instructions of N <= 256; the level
//                                   accumulators of a tile stay in TMEM for the whole K loop; the epilogue turns the levels into
//                                   one integer, scales by exponent arithmetic and adds into c with TMA reductions
//   ozaki_slice_kernel<S>           x -> int8 digit planes [t][row][k] + one exponent per row (+ the guard)
// Measured on B200 (profiles/r1f_*), whole application N = 4096 / 8192 / 16384: 350 / 430 / 309 TFLOP/s of FP64 work (FP32:
// 406 / 473 / 314) with the forms 2x2 / 3x2 / 3x3 the operands allow (first version, 6-slice triangular form for all: 119 / 151 /
// 172); DMMA 33-35.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "ozaki_digits.cuh"
#include "raster.cuh"
#include "tc_ptx.cuh"

namespace mmx {
namespace {

constexpr int OZ_BM = 128, OZ_BN = 64;               // tile of c
constexpr int OZ_THREADS = 192;                      // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue (one per TMEM lane quarter)
constexpr int OZ_KPAD = 64;                          // slice rows are padded to this many k
constexpr int OZP_THREADS = 320;                     // persistent form: warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (two per TMEM lane quarter)

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

__device__ __forceinline__ double pow2(int e) { return oz_pow2(e); }
constexpr double kOzLevelStep = 1.0 / (1 << kOzDigitBits);  // level g + 1 weighs 2^-kOzDigitBits of level g (ozaki_digits.cuh: 8-bit digits below the first)

constexpr int kNonFinite = kOzNonFinite;  // row exponent of a row that holds an Inf or a NaN: its products are NaN
// acc * 2^(ea + eb - 14): exact scaling (ldexp also covers results that leave the normal range); ea, eb: unpacked exponents
__device__ __forceinline__ double scaled(double acc, int ea, int eb) {
  if (ea == kNonFinite || eb == kNonFinite) return __longlong_as_double(0x7ff8000000000000ll);
  return ldexp(acc, ea + eb - kOzPairUnit);
}
// rows encoded negated (ozaki_digits.cuh): the product of a row of a and a row of bt changes sign when exactly one of them is;
// a zero stays +0 (the level sums are integers: the kernels never produce -0, which the store path for a zeroed c relies on)
__device__ __forceinline__ double oz_signed(double v, bool neg) { return (neg && v != 0.0) ? -v : v; }
// the same for a column's packed exponent word
__device__ __forceinline__ double scaled_w(double acc, int ea, bool na, int eb_word) {
  int eb;
  const bool nb = oz_exp_unpack(eb_word, eb);
  return oz_signed(scaled(acc, ea, eb), na != nb);
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
    int ei;  // kNonFinite marks a row that holds an Inf or a NaN
    const bool na = oz_exp_unpack(row_ok ? exp_a[m] : 0, ei);
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
          for (int g = S - 2; g >= 0; --g) acc = fma(acc, kOzLevelStep, static_cast<double>(static_cast<int>(lv[g][e + h])));
          v[h] = cpre[cb * 8 + e + h] + scaled_w(acc, ei, na, eb_sh[cb * 8 + e + h]);
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

// ---- persistent form (the default): one CTA per SM walks the tiles of c in raster order ----------------------------------
// What it adds over the kernel above:
//  (1) Which digit pairs are multiplied is a template shape <SA, SB, LV, BN>: slices a_1..a_SA against b_1..b_SB, pairs kept
//      up to level t + u <= LV + 1, on a 128 x BN tile.  <S, S, S, 64> is the triangular S-slice form of the header (a general
//      kernel with its truncation bound: matmul_variant 40 .. 45).  <SA, SB, SA + SB - 1, BN> is the RECTANGULAR form: every
//      pair of the first SA x SB digits, error-free iff a has no digit beyond SA and bt none beyond SB -- operands with few
//      significant bits cost proportionally less (the application's carry log2(N) + 2 bits = two digits each up to N = 4096:
//      4 slice products per FP64 term instead of 28).  With few levels the tile is 128 wide: each a_t meets [b_1 | b_2]
//      stacked along N in ONE N = 256 instruction, the shape at which the operand reads (4 KB of a + 8 KB of b per 128 clocks)
//      stay under the 128 B/clk of shared memory.
//  (2) The form is a run-time choice inside ONE launch: the auto kernel reads the guard the slice pass wrote (anything cut?
//      highest digit in use per operand) and runs the cheapest error-free form, or leaves at once (the FP64-pipe kernel then
//      runs).  A launch that leaves retires 148 CTAs, not thousands.
//  (3) The TMA producer runs ahead into the next tile while the epilogue drains, and where 2 * LV * BN <= 512 columns the level
//      accumulators are double-buffered in TMEM, so the MMAs of tile i+1 overlap the epilogue of tile i entirely.
// Slices arrive as one TMA box per slice and operand (the shared-memory layout is the one the 3-D box of the kernel above gives).
// CR = slabs (32 rows x 16 columns of results on their way to c) per epilogue warp (0: the epilogue reads and writes c from
// registers, one row per thread, with four epilogue warps)
template <int SA, int SB, int LV, int BN, int CR> struct OzPShape {
  static_assert(BN == 64 || BN == 128, "tile width");
  static_assert(LV * BN <= 512, "the level accumulators of a tile must fit TMEM");
  static_assert(LV >= SA && LV >= SB && LV <= SA + SB - 1, "levels");
  static constexpr int BK = 64;
  static constexpr int A_SLICE = OZ_BM * BK, B_SLICE = BN * BK;
  static constexpr int A_BYTES = SA * A_SLICE, B_BYTES = SB * B_SLICE;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int C_SLAB = 32 * 16 * 8;      // 32 rows x 16 doubles = one 128-byte-swizzled TMA box
  static constexpr int EPI_WARPS = CR > 0 ? 8 : 4;
  static constexpr int C_BYTES = CR * 8 * C_SLAB;
  // barriers (256 B), column exponents [2][BN] int, and -- where the epilogue multiplies instead of adding to the exponent field --
  // the column scale factors [2][BN] double
  static constexpr bool SCALE_TABLE = !(CR > 0 && LV <= 4);
  static constexpr int TAIL = SCALE_TABLE ? 3584 : 1536;
  static constexpr int STAGES_FIT = (227 * 1024 - 1024 - TAIL - C_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static_assert(STAGES >= 2, "stage ring");
  static constexpr int NBUF = 2 * LV * BN <= 512 ? 2 : 1;  // accumulator sets in TMEM
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + C_BYTES + 1024 + TAIL;
};
constexpr int kOzPersistSmemMax = 227 * 1024;  // the auto kernel asks for all of it: each form uses what its rings need

struct OzPArgs {
  void* c;  // double (or float: the FP32 auto mode, reduction epilogue only)
  const int *exp_a, *exp_b;
  int n, kq, row0, rows, col0, cols, group;
  long long group_l2_bytes;  // budget for a raster group's rows of a (0: default; MMX_OZ_GROUP_MB overrides -- tuning hook)
  int c_zero;  // every element of c this launch covers is +0: results are stored, not added (kCIsZero)
  // auto kernels inside a captured graph: the fallback (FP64 pipe / split TF32) sits in a conditional node that runs iff no INT8 form
  // took the product (OzFallbackCond, kernels.cuh); 0 = no conditional, the fallback launches read the guard themselves
  unsigned long long cond;
  int use_cond;
  int debug;  // MMX_OZ_DEBUG (rate probes, results are WRONG): 1 the producer signals stages without loading them, 2 the epilogue drops phase B
  // MMX_OZ_TRACE=1 (pair body): SM clocks of the leader CTA of pair 0 at the hand-over points of every tile, 8 words per tile --
  // [0] the issuing thread saw the accumulators free, [1] it saw the tile's first stage full, [2] it committed the tile,
  // [3] an epilogue warp saw the commit, [4] that warp had read its share and arrived (tools/handover_trace.py prints them)
  long long* trace;
};

// +-sum * 2^(ea + eb - 14).  Fast path (both exponents moderate): two multiplications by exact powers of two, pa = 2^(ea - 14)
// and pb = 2^eb -- neither product leaves the normal range, so the result is the one ldexp gives.  eb_word: the column's packed
// exponent word, na: the row is encoded negated.
__device__ __forceinline__ double scaled_fast(double sum, int ea, double pa, bool row_fast, bool na, int eb_word, double pb) {
  int eb;
  const bool nb = oz_exp_unpack(eb_word, eb);
  if (row_fast && eb > -400 && eb < 400) return oz_signed((sum * pa) * pb, na != nb);
  return oz_signed(scaled(sum, ea, eb), na != nb);
}

// CX x CY = CTAs per cluster working on CX x CY adjacent tiles: the a slices of a tile-row are fetched once per cluster row
// (each of its CX CTAs loads 128 / CX rows of every slice and multicasts them), the bt slices of a column tile once per cluster
// column.  The operand traffic is what bounds the short forms (the 2 x 2 form at 128 x 128 needs 32 KB per 512 tensor-pipe
// clocks and SM: 8.3 TB/s measured against the 11.8 TB/s the L2 can put on the crossbar); a 2 x 2 cluster halves it.
template <int SA, int SB, int LV, int BN, int CR, int CX, int CY, typename CT = double>
__device__ __forceinline__ void oz_persist_body(const OzPArgs& g, const CUtensorMap* map_a, const CUtensorMap* map_b, const CUtensorMap* map_c,
                                                unsigned char* smem_raw) {
  using Sh = OzPShape<SA, SB, LV, BN, CR>;
  constexpr int C = CX * CY;
  const unsigned rank = C > 1 ? cluster_ctarank() : 0u;
  const int rx = static_cast<int>(rank) % CX, ry = static_cast<int>(rank) / CX;
  constexpr unsigned short kMaskAll = static_cast<unsigned short>((1u << C) - 1u);
  const unsigned short mask_row = static_cast<unsigned short>(((1u << CX) - 1u) << (ry * CX));          // the CTAs that share my a slices
  const unsigned short mask_col = static_cast<unsigned short>((CY > 1 ? (1u | (1u << CX)) : 1u) << rx);  // ... my bt slices
  constexpr int STAGES = Sh::STAGES, NBUF = Sh::NBUF, BK = Sh::BK;
  constexpr int PER_MMA = 256 / BN;  // b slices one instruction can take (N <= 256)
  const unsigned raw = smem_u32(smem_raw);
  const unsigned base = (raw + 1023u) & ~1023u;
  const unsigned cbuf = base + STAGES * Sh::STAGE_BYTES;  // CR chunk buffers of c (1024-byte aligned: every stage is a multiple)
  const unsigned bars = cbuf + Sh::C_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (8 + s); };
  auto acc_full = [&](int b) { return bars + 8u * (16 + b); };   // the MMAs of a tile have completed into set b
  auto acc_empty = [&](int b) { return bars + 8u * (18 + b); };  // the epilogue has read set b
  const unsigned tmem_slot = bars + 8u * 24;
  volatile unsigned* tmem_slot_ptr = reinterpret_cast<volatile unsigned*>(smem_raw + (tmem_slot - raw));
  int* eb_sh = reinterpret_cast<int*>(smem_raw + (bars + 256 - raw));            // [2][BN] column exponents, alternating per tile
  double* pb_sh = reinterpret_cast<double*>(smem_raw + (bars + 256 + 1024 - raw));  // [2][BN] 2^exponent (clamped) of the same

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // the cluster walks super-tiles of CX x CY tiles in raster order; CTA (rx, ry) takes its tile of each (a tile beyond the
  // edge is computed on zero-filled operands and never stored: its peers need this CTA's share of the loads)
  const int super_x = ((g.cols + BN - 1) / BN + CX - 1) / CX, super_y = ((g.rows + OZ_BM - 1) / OZ_BM + CY - 1) / CY;
  const int supers = super_x * super_y;
  const int first = static_cast<int>(blockIdx.x) / C, stride = static_cast<int>(gridDim.x) / C;
  const int my_tiles = first < supers ? (supers - 1 - first) / stride + 1 : 0;
  // tile-rows per raster group: the group's rows of a (SA planes) are meant to stay in the 126 MB L2 while bt streams by, so
  // the group shrinks when they would not fit (g.group = 16 tile-rows = 100 MB at N = 16384 with three planes, 200 MB at 32768)
  const long long strip_bytes = static_cast<long long>(OZ_BM) * g.kq * SA;
  const int fit = static_cast<int>((g.group_l2_bytes > 0 ? g.group_l2_bytes : (64ll << 20)) / strip_bytes);
  const int rows_per_group = fit < g.group ? (fit > 2 ? fit : 2) : g.group;
  const int group = rows_per_group / CY > 0 ? rows_per_group / CY : 1;
  auto tile_at = [&](int k, int& bx, int& by) {  // the k-th tile of this CTA
    int sx, sy;
    raster_map(group, super_x, super_y, first + k * stride, sx, sy);
    bx = sx * CX + rx;
    by = sy * CY + ry;
  };
  const int k_stages = g.kq / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), C);  // the MMAs of every CTA of the cluster have left the stage (what lands in it comes from peers too)
    }
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(acc_full(b), 1);
      mbar_init(acc_empty(b), Sh::EPI_WARPS);  // one arrival per epilogue warp
    }
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
      int it = 0;  // stages filled so far, over all tiles of this CTA
      for (int tile = 0; tile < my_tiles; ++tile) {
        int bx, by;
        tile_at(tile, bx, by);
        const int m_base = g.row0 + by * OZ_BM, n_rel = bx * BN;
        for (int kb = 0; kb < k_stages; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(empty_bar(s), ((it / STAGES) & 1) ^ 1);
          const unsigned st = base + s * Sh::STAGE_BYTES;
          if ((g.debug & 1) && it >= STAGES) {  // rate probe: the MMAs run on whatever the stage buffers hold
            mbar_arrive(full_bar(s));
            continue;
          }
          mbar_expect_tx(full_bar(s), Sh::STAGE_BYTES);
          if constexpr (C == 1) {
            if (g.debug & 128) {
              const unsigned long long keep = l2_policy_evict_last();
#pragma unroll
              for (int t = 0; t < SA; ++t) tma_load_3d_hint(st + t * Sh::A_SLICE, map_a, kb * BK, m_base, t, full_bar(s), keep);
#pragma unroll
              for (int t = 0; t < SB; ++t) tma_load_3d_hint(st + Sh::A_BYTES + t * Sh::B_SLICE, map_b, kb * BK, n_rel, t, full_bar(s), keep);
              continue;
            }
#pragma unroll
            for (int t = 0; t < SA; ++t) tma_load_3d(st + t * Sh::A_SLICE, map_a, kb * BK, m_base, t, full_bar(s));
#pragma unroll
            for (int t = 0; t < SB; ++t) tma_load_3d(st + Sh::A_BYTES + t * Sh::B_SLICE, map_b, kb * BK, n_rel, t, full_bar(s));
          } else {
            constexpr int PA = OZ_BM / CX, PB = BN / CY;  // rows of every slice this CTA fetches for its cluster row / column
#pragma unroll
            for (int t = 0; t < SA; ++t)
              tma_load_3d_mc(st + t * Sh::A_SLICE + rx * (PA * BK), map_a, kb * BK, m_base + rx * PA, t, full_bar(s), mask_row);
#pragma unroll
            for (int t = 0; t < SB; ++t)
              tma_load_3d_mc(st + Sh::A_BYTES + t * Sh::B_SLICE + ry * (PB * BK), map_b, kb * BK, n_rel + ry * PB, t, full_bar(s), mask_col);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int it = 0;
      for (int tile = 0; tile < my_tiles; ++tile) {
        const int buf = tile % NBUF;
        mbar_wait(acc_empty(buf), ((tile / NBUF) & 1) ^ 1);
        tc_fence_after();
        const unsigned acc = tmem_base + buf * (LV * BN);
        for (int kb = 0; kb < k_stages; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(full_bar(s), (it / STAGES) & 1);
          tc_fence_after();
          const unsigned st = base + s * Sh::STAGE_BYTES;
#pragma unroll
          for (int ks = 0; ks < BK / 32; ++ks) {
            const unsigned long long adv = 2ull * ks;  // 32 bytes along K inside the 64-byte swizzle row
#pragma unroll
            for (int t = 1; t <= SA; ++t) {
              const unsigned long long a_t = umma_desc_sw<BK>(st + (t - 1) * Sh::A_SLICE) + adv;
              // slices b_1 .. b_count pair with a_t: levels t+1 .. t+count = TMEM column blocks t-1 .. t+count-2
              constexpr int kAll = SB;
              const int count = kAll < LV + 1 - t ? kAll : LV + 1 - t;
#pragma unroll
              for (int u0 = 0; u0 < count; u0 += PER_MMA) {
                const int nsl = count - u0 < PER_MMA ? count - u0 : PER_MMA;
                const unsigned long long b_u = umma_desc_sw<BK>(st + Sh::A_BYTES + u0 * Sh::B_SLICE) + adv;
                // a block is initialised by the first product that lands on it in the tile's first k step: a_1 opens blocks
                // 0 .. SB-1, every further a_t the one block (t + SB - 2) nobody before it reached
                unsigned accumulate = 1;
                if (kb == 0 && ks == 0) {
                  if (t == 1) {
                    accumulate = 0;
                  } else if (u0 + nsl == count && count == SB) {
                    // the last block of this instruction is new; the others are not: issue that slice on its own
                    if (nsl > 1) {
                      tc_mma_i8(acc + (t - 1 + u0) * BN, a_t, b_u, idesc_i8((nsl - 1) * BN), 1);
                    }
                    const unsigned long long b_last = umma_desc_sw<BK>(st + Sh::A_BYTES + (count - 1) * Sh::B_SLICE) + adv;
                    tc_mma_i8(acc + (t - 1 + count - 1) * BN, a_t, b_last, idesc_i8(BN), 0);
                    continue;
                  }
                }
                tc_mma_i8(acc + (t - 1 + u0) * BN, a_t, b_u, idesc_i8(nsl * BN), accumulate);
              }
            }
          }
          if constexpr (C == 1) tc_commit(empty_bar(s));
          else tc_commit_mc(empty_bar(s), kMaskAll);
        }
        tc_commit(acc_full(buf));
      }
    }
  } else {
    // epilogue warps: thread = one row of the tile (TMEM lane)
    const int q = warp % 4;
    const int r = q * 32 + lane;  // row inside the tile
    const int m_limit = g.row0 + g.rows;
    int tile = 0;
    if constexpr (CR > 0) {
      // c += through TMA REDUCTIONS, 16 columns at a time: each epilogue warp owns 32 rows of the tile; it writes their 16
      // results into its 4 KB slab of a chunk buffer (128-byte rows under SWIZZLE_128B: 16-byte stores, conflict-free) and
      // one lane sends the slab off as cp.reduce.async.bulk.tensor .add -- the L2 performs c[i][j] += v (one IEEE addition,
      // what the thread would have done), so c is never loaded by the SM, global memory sees whole 128-byte lines instead of
      // one 16-byte piece per thread and row, and nothing waits for a round trip.  The warps are decoupled: a slab is reused
      // once its reduction has left shared memory (ring of CR per warp), with no CTA-wide barrier per chunk.  The tensor map
      // of c ends at (row0 + rows, col0 + cols): what lies beyond is dropped, which is all the edge handling there is.
      constexpr int NCH = BN / 16;
      const int grp = (warp - 2) / 4;  // the two warps of a lane quarter take alternate chunks
      const unsigned slab0 = cbuf + (warp - 2) * Sh::C_SLAB;
      int sent = 0;  // chunks this warp has sent
      for (; tile < my_tiles; ++tile) {
        int bx, by;
        tile_at(tile, bx, by);
        const int m_base = g.row0 + by * OZ_BM, n_tile = bx * BN;
        const int buf = tile % NBUF;
        const int m = m_base + r;
        int ei;  // kNonFinite marks a row that holds an Inf or a NaN
        const bool na = oz_exp_unpack(m < m_limit ? g.exp_a[m] : 0, ei);
        const bool row_fast = ei > -400 && ei < 400;
        const double pa = pow2(row_fast ? ei - kOzPairUnit : 0);
        int* eb = eb_sh + (tile & 1) * BN;
        double* pb = pb_sh + (tile & 1) * BN;
        if (grp == 0 && r < BN) {
          const int word = n_tile + r < g.cols ? g.exp_b[n_tile + r] : 0;
          eb[r] = word;  // packed: exponent and sign of the column (oz_exp_unpack)
          if constexpr (Sh::SCALE_TABLE) {
            int e;
            (void)oz_exp_unpack(word, e);
            pb[r] = pow2(e > -400 && e < 400 ? e : 0);
          }
        }
        // the exponents of this tile are complete; nobody is still reading the other copy (that was two tiles ago, and
        // everyone has passed the barrier of the tile in between)
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
        mbar_wait(acc_full(buf), (tile / NBUF) & 1);
        tc_fence_after();
        const unsigned t0 = tmem_base + (static_cast<unsigned>(q * 32) << 16) + buf * (LV * BN);
        // Phase A -- empty the accumulators: this warp's chunks (alternate 16-column chunks of its 32 rows) leave TMEM as ONE
        // number per element, held in registers: the level sum as a 64-bit integer where LV <= 4 (|L| < 2^31 and three shifts of
        // 7 bits: exact), the Horner sum in FP64 beyond.  Nothing else happens before the set is handed back, so the MMAs of the
        // next tile start after ~LV x MY TMEM loads instead of after the whole epilogue (conversions, shared-memory slabs, TMA
        // reductions, each waiting for the previous one to leave its slab: ~7 us of the 24 us a 2 x 2 tile took at N = 4096).
        constexpr int MY = NCH / 2;                 // chunks per warp and tile
        constexpr int LD = 8;                       // columns per TMEM load group (registers in flight: LV x LD)
        long long acc[LV <= 4 ? MY : 1][16];
        double hsum[LV <= 4 ? 1 : MY][16];
#pragma unroll
        for (int jj = 0; jj < MY; ++jj) {
          const int j = grp + 2 * jj;
#pragma unroll
          for (int h = 0; h < 16 / LD; ++h) {
            unsigned lv[LV][LD];
#pragma unroll
            for (int l = 0; l < LV; ++l) {
              if constexpr (LD == 16) tc_ld16_issue(t0 + l * BN + j * 16, lv[l]);
              else tc_ld8_issue(t0 + l * BN + j * 16 + h * 8, lv[l]);
            }
            tc_ld_wait();
#pragma unroll
            for (int e = 0; e < LD; ++e) {
              if constexpr (LV <= 4) {
                long long x = static_cast<int>(lv[0][e]);
#pragma unroll
                for (int l = 1; l < LV; ++l) x = (x << kOzDigitBits) + static_cast<int>(lv[l][e]);
                acc[jj][h * LD + e] = x;
              } else {
                double x = static_cast<double>(static_cast<int>(lv[LV - 1][e]));
#pragma unroll
                for (int l = LV - 2; l >= 0; --l) x = fma(x, kOzLevelStep, static_cast<double>(static_cast<int>(lv[l][e])));
                hsum[jj][h * LD + e] = x;
              }
            }
          }
        }
        // this warp has read its share of the set: the MMAs of a later tile may overwrite it
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty(buf));
        // Phase B -- scale, stage, reduce into c (overlaps the next tile's MMAs)
        if (g.debug & 2) continue;
#pragma unroll
        for (int jj = 0; jj < MY; ++jj, ++sent) {
          const int j = grp + 2 * jj;
          double v[16];
          if constexpr (LV <= 4) {
            // scaled by adding to the exponent field: one FP64-pipe operation per element (the conversion) instead of seven.
            // Whether the 16 columns of the chunk all have moderate exponents is decided once (the same for every lane), so the
            // common case is a branch-free loop the scheduler can interleave across elements.
            int ebv[16];
            unsigned flip = 0;  // bit e: the product of this row and column e changes sign (one of the two is encoded negated)
            bool cols_fast = true;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              flip |= (oz_exp_unpack(eb[j * 16 + e], ebv[e]) != na ? 1u : 0u) << e;
              cols_fast &= static_cast<unsigned>(ebv[e] + 399) < 799u;
            }
            if (cols_fast && row_fast) {
              const int e_row = ei - kOzPairUnit - kOzDigitBits * (LV - 1);
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                const long long x = acc[jj][e];
                const double d = static_cast<double>(x);
                const int hi = x != 0 ? (__double2hiint(d) + (e_row + ebv[e]) * (1 << 20)) ^ static_cast<int>((flip >> e & 1u) << 31) : 0;  // stays a normal number
                v[e] = __hiloint2double(hi, __double2loint(d));
              }
            } else {
#pragma unroll  // (a rolled loop would index acc and v dynamically and push them to local memory for both branches)
              for (int e = 0; e < 16; ++e) v[e] = oz_signed(scaled(static_cast<double>(acc[jj][e]) * pow2(-kOzDigitBits * (LV - 1)), ei, ebv[e]), (flip >> e & 1u) != 0);
            }
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = scaled_fast(hsum[jj][e], ei, pa, row_fast, na, eb[j * 16 + e], pb[j * 16 + e]);
          }
          const unsigned slab = slab0 + (sent % CR) * (8 * Sh::C_SLAB);
          if (g.debug & 16) {  // rate probe: conversions only
            double keep = 0.0;
#pragma unroll
            for (int e = 0; e < 16; ++e) keep += v[e];
            if (keep == 1.2345e300) *reinterpret_cast<volatile double*>(smem_raw) = keep;
            continue;
          }
          if (lane == 0) tma_store_wait_read<CR - 1>();  // the reduction that last used this slab has left shared memory
          __syncwarp();
          if constexpr (sizeof(CT) == 8) {
            const unsigned crow = slab + lane * 128;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch)
              asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(crow + ((ch ^ (lane & 7)) << 4)), "d"(v[2 * ch]), "d"(v[2 * ch + 1]) : "memory");
          } else {
            // FP32 output: the exact value rounded ONCE to float; 64-byte rows under SWIZZLE_64B (16-byte piece ^ bits 1-2 of the row)
            const unsigned crow = slab + lane * 64;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch)
              asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(crow + ((ch ^ ((lane >> 1) & 3)) << 4)), "f"(static_cast<float>(v[4 * ch])),
                           "f"(static_cast<float>(v[4 * ch + 1])), "f"(static_cast<float>(v[4 * ch + 2])), "f"(static_cast<float>(v[4 * ch + 3]))
                           : "memory");
          }
          if (g.debug & (32 | 64)) {
            // c through the load/store units: the slab is read back row-wise (8 lanes = one 128-byte row, 4 rows per instruction)
            // and goes out as whole lines -- plain stores (bit 32: c is known to be zero) or FP64 reductions at the L2 (bit 64)
            __syncwarp();
            CT* cbase = static_cast<CT*>(g.c);
            if constexpr (sizeof(CT) == 8) {
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int rr = 4 * i + (lane >> 3), pp = lane & 7;
                double x, y;
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(slab + rr * 128 + ((pp ^ (rr & 7)) << 4)) : "memory");
                const int row = m_base + q * 32 + rr, col = n_tile + j * 16 + 2 * pp;
                if (row < m_limit && col + 2 <= g.cols) {
                  double* at = cbase + static_cast<size_t>(row) * g.n + g.col0 + col;
                  if (g.debug & 32) {
                    *reinterpret_cast<double2*>(at) = make_double2(x, y);
                  } else {
                    asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(at), "d"(x) : "memory");
                    asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(at + 1), "d"(y) : "memory");
                  }
                }
              }
            } else {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int rr = 8 * i + (lane >> 2), pp = lane & 3;
                float x0, x1, x2, x3;
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(x0), "=f"(x1), "=f"(x2), "=f"(x3) : "r"(slab + rr * 64 + ((pp ^ ((rr >> 1) & 3)) << 4)) : "memory");
                const int row = m_base + q * 32 + rr, col = n_tile + j * 16 + 4 * pp;
                if (row < m_limit && col + 4 <= g.cols) {
                  float* at = reinterpret_cast<float*>(cbase) + static_cast<size_t>(row) * g.n + g.col0 + col;
                  if (g.debug & 32) *reinterpret_cast<float4*>(at) = make_float4(x0, x1, x2, x3);
                  else asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(at), "f"(x0), "f"(x1), "f"(x2), "f"(x3) : "memory");
                }
              }
            }
            __syncwarp();  // the slab may be rewritten
            continue;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (g.debug & 512) __nanosleep(jj == 0 ? 200u + 400u * (warp - 2) : 2500u);
          if (g.debug & 1024) __nanosleep(jj == 0 ? 100u + 200u * (warp - 2) : 1200u);
          if (lane == 0 && !(g.debug & 8)) {
            if (g.c_zero || (g.debug & 4)) tma_store_2d(map_c, slab, g.col0 + n_tile + j * 16, m_base + q * 32);
            else if (g.debug & 256) tma_reduce_add_2d_hint(map_c, slab, g.col0 + n_tile + j * 16, m_base + q * 32, l2_policy_evict_first());
            else tma_reduce_add_2d(map_c, slab, g.col0 + n_tile + j * 16, m_base + q * 32);
            tma_store_commit();
          }
        }
      }
      if (lane == 0) tma_store_wait<0>();
    } else {
      static_assert(sizeof(CT) == 8, "the register epilogue exists for FP64 only");
      // c straight from registers (any n, odd ones included): 64 columns at a time; the first 64 incoming values and the
      // tile's column exponents are fetched before the tile's MMAs are waited for
      const bool vec_ok = (g.n % 2 == 0) && (g.col0 % 2 == 0);
      for (; warp < 6 && tile < my_tiles; ++tile) {  // warps 2-5; the other four have nothing to do in this form
        int bx, by;
        tile_at(tile, bx, by);
        const int m_base = g.row0 + by * OZ_BM, n_tile = bx * BN;
        const int buf = tile % NBUF;
        const int m = m_base + r;
        const bool row_ok = m < m_limit;
        int ei;  // kNonFinite marks a row that holds an Inf or a NaN
        const bool na = oz_exp_unpack(row_ok ? g.exp_a[m] : 0, ei);
        const bool row_fast = ei > -400 && ei < 400;
        const double pa = pow2(row_fast ? ei - kOzPairUnit : 0);
        double* crow = static_cast<double*>(g.c) + static_cast<size_t>(row_ok ? m : 0) * g.n;
        int* eb = eb_sh + (tile & 1) * BN;
        double* pb = pb_sh + (tile & 1) * BN;
        if (r < BN) {
          const int word = n_tile + r < g.cols ? g.exp_b[n_tile + r] : 0;
          int e;
          (void)oz_exp_unpack(word, e);
          eb[r] = word;  // packed: exponent and sign of the column
          pb[r] = pow2(e > -400 && e < 400 ? e : 0);
        }
#pragma unroll 1
        for (int part = 0; part < BN / 32; ++part) {
          const int n_rel = n_tile + part * 32;
          double cpre[32];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const int jr = n_rel + e;
            if (row_ok && vec_ok && jr + 2 <= g.cols) {
              const double2 x = *reinterpret_cast<const double2*>(crow + g.col0 + jr);
              cpre[e] = x.x;
              cpre[e + 1] = x.y;
            } else {
              cpre[e] = (row_ok && jr < g.cols) ? crow[g.col0 + jr] : 0.0;
              cpre[e + 1] = (row_ok && jr + 1 < g.cols) ? crow[g.col0 + jr + 1] : 0.0;
            }
          }
          if (part == 0) {
            asm volatile("bar.sync 1, 128;\n" ::: "memory");  // the exponents of this tile are complete (see above)
            mbar_wait(acc_full(buf), (tile / NBUF) & 1);
            tc_fence_after();
          }
          const unsigned t0 = tmem_base + (static_cast<unsigned>(q * 32) << 16) + buf * (LV * BN) + part * 32;
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) {
            unsigned lv[LV][8];
#pragma unroll
            for (int l = 0; l < LV; ++l) tc_ld8_issue(t0 + l * BN + cb * 8, lv[l]);
            tc_ld_wait();
            if (cb == 3 && part == BN / 32 - 1) {  // every level of this set is in registers
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(acc_empty(buf));
            }
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const int jr = n_rel + cb * 8 + e;  // relative to col0
              double v[2];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                double sum = static_cast<double>(static_cast<int>(lv[LV - 1][e + h]));
#pragma unroll
                for (int l = LV - 2; l >= 0; --l) sum = fma(sum, kOzLevelStep, static_cast<double>(static_cast<int>(lv[l][e + h])));
                const int col = part * 32 + cb * 8 + e + h;
                v[h] = cpre[cb * 8 + e + h] + scaled_fast(sum, ei, pa, row_fast, na, eb[col], pb[col]);
              }
              if (!row_ok) continue;
              const int j = g.col0 + jr;
              if (vec_ok && jr + 2 <= g.cols) {
                *reinterpret_cast<double2*>(crow + j) = make_double2(v[0], v[1]);
              } else {
#pragma unroll
                for (int h = 0; h < 2; ++h)
                  if (jr + h < g.cols) crow[j + h] = v[h];
              }
            }
          }
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
  if constexpr (C > 1) cluster_sync_all();  // no CTA leaves while a peer may still multicast into it or signal its barriers
}

// ---- CTA pairs (tcgen05 cta_group::2) for the forms whose b slices stack to N = 256: SA x 2 digit pairs on 128-wide tiles -----
// What bounds the short forms in the one-CTA body is operand traffic, not the tensor pipe (profiles/r2f_contraction_rate_probes.txt:
// 0.175 ms at N = 4096 becomes 0.159 without the loads; the L2 puts 9.2 TB/s on the crossbar of 11.8, and every 128-clock
// instruction reads 4 KB of a and 8 KB of bt from shared memory while TMA writes the next stage into it).  Two CTAs on the SMs
// of one TPC execute ONE instruction of M = 256: each holds its own 128 rows of every a slice and ONE of the two b slices
// (CTA 0: b_1, CTA 1: b_2 -- the hardware takes the first 128 rows of the N = 256 operand from the leader and the rest from its
// peer), so per SM and k step the instruction reads 4 + 4 KB instead of 4 + 8, a stage is (SA + 1) x 8 KB instead of
// (SA + 2) x 8, and a pair tile of 256 x 128 moves 25 % fewer operand bytes per flop across the crossbar than two 128 x 128 tiles.
//   * barriers live at the same offsets in both CTAs.  full[s] of the LEADER counts both CTAs' bytes (announced by the leader's
//     producer; cp.async.bulk.tensor .cta_group::2 signals a barrier of the pair's other CTA); empty[s], acc_full are signalled in BOTH CTAs
//     by multicast commits; acc_empty of the leader counts the epilogue warps of both CTAs (remote arrivals).
//   * the leader's warp 1 issues every MMA; both CTAs run a TMA producer (warp 0) and eight epilogue warps over their own 128
//     TMEM lanes (the two-phase epilogue of the body above).
//   * level blocks 2 .. LV-1 receive a product with "accumulate" set in the tile's first k step (a_t opens block t, which the
//     one-CTA body initialises with a separate N = 128 instruction -- not expressible here, where halving N means halving each
//     CTA's share): the epilogue stores zeros into them right after reading them (and once before the first tile).
//   * SA x 3 pairs (the application from N = 16384): tiles are 96 wide so that five levels fit TMEM (480 columns); a_t meets
//     [b_1 | b_2] in an N = 192 instruction (CTA 0 holds b_1, CTA 1 holds b_2) and b_3 in an N = 96 one (each CTA holds 48 of its
//     rows).  Every level block is opened by an overwriting instruction here, so nothing needs zeroing.
template <int SA, int SB, int LV> struct OzPairShape {
  static_assert(SB == 2 || SB == 3, "two or three b slices");
  static_assert(LV == SA + SB - 1, "rectangular forms");
  static constexpr int BN = SB == 2 ? 128 : 96, BK = 64;
  static_assert(LV * BN <= 512, "the level accumulators of a tile must fit TMEM");
  static constexpr int A_SLICE = OZ_BM * BK;
  static constexpr int A_BYTES = SA * A_SLICE;
  static constexpr int B1_BYTES = BN * BK;                        // this CTA's slice of the [b_1 | b_2] operand
  static constexpr int B2_BYTES = SB == 3 ? (BN / 2) * BK : 0;    // its half of b_3
  static constexpr int STAGE_BYTES = A_BYTES + B1_BYTES + B2_BYTES;  // per CTA
  static constexpr int C_SLAB = 32 * 16 * 8;
  static constexpr int C_BYTES = 8 * C_SLAB;               // one slab per epilogue warp
  static constexpr bool SCALE_TABLE = LV > 4;
  static constexpr int TAIL = SCALE_TABLE ? 3584 : 1536;
  static constexpr int STAGES_FIT = (227 * 1024 - 1024 - TAIL - C_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static_assert(STAGES >= 3, "stage ring");
};

template <int SA, int SB, int LV, typename CT>
__device__ __forceinline__ void oz_pair_body(const OzPArgs& g, const CUtensorMap* map_a, const CUtensorMap* map_b, const CUtensorMap* map_b_half,
                                             const CUtensorMap* map_c, unsigned char* smem_raw) {
  using Sh = OzPairShape<SA, SB, LV>;
  constexpr int STAGES = Sh::STAGES, BK = Sh::BK, BN = Sh::BN;
  const unsigned rank = cluster_ctarank();  // 0 = leader
  const unsigned raw = smem_u32(smem_raw);
  const unsigned base = (raw + 1023u) & ~1023u;
  const unsigned cbuf = base + STAGES * Sh::STAGE_BYTES;
  const unsigned bars = (cbuf + Sh::C_BYTES + 127u) & ~127u;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (8 + s); };
  const unsigned acc_full = bars + 8u * 16, acc_empty = bars + 8u * 18;
  const unsigned tmem_slot = bars + 8u * 24;
  volatile unsigned* tmem_slot_ptr = reinterpret_cast<volatile unsigned*>(smem_raw + (tmem_slot - raw));
  int* eb_sh = reinterpret_cast<int*>(smem_raw + (bars + 256 - raw));               // [2][BN] column exponents, alternating per tile
  double* pb_sh = reinterpret_cast<double*>(smem_raw + (bars + 256 + 1024 - raw));  // [2][BN] 2^exponent (clamped) of the same
  unsigned* sg_sh = reinterpret_cast<unsigned*>(smem_raw + (bars + 208 - raw));     // [2][4] the columns encoded negated, one bit each

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // pair tiles of 256 rows x BN columns in raster order; CTA `rank` owns rows [256 sy + 128 rank, + 128)
  const int tiles_x = (g.cols + BN - 1) / BN, tiles_y2 = ((g.rows + OZ_BM - 1) / OZ_BM + 1) / 2;
  const int supers = tiles_x * tiles_y2;
  const int first = static_cast<int>(blockIdx.x) / 2, stride = static_cast<int>(gridDim.x) / 2;
  const int my_tiles = first < supers ? (supers - 1 - first) / stride + 1 : 0;
  const long long strip_bytes = static_cast<long long>(OZ_BM) * g.kq * SA;
  const int fit = static_cast<int>((g.group_l2_bytes > 0 ? g.group_l2_bytes : (64ll << 20)) / strip_bytes);
  const int rows_per_group = fit < g.group ? (fit > 2 ? fit : 2) : g.group;
  const int group = rows_per_group / 2 > 0 ? rows_per_group / 2 : 1;
  auto tile_at = [&](int k, int& bx, int& by) {
    int sx, sy;
    raster_map(group, tiles_x, tiles_y2, first + k * stride, sx, sy);
    bx = sx;
    by = sy * 2 + static_cast<int>(rank);
  };
  const int k_stages = g.kq / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);   // the leader's arrival carries the byte count of both CTAs' loads; only the leader's is used
      mbar_init(empty_bar(s), 1);  // the pair's MMAs have left the stage (multicast commit)
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 2 * 8);   // the epilogue warps of both CTAs; only the leader's is used
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tmem_slot), "n"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers and allocations are in place before anything crosses the pair
  tc_fence_after();
  const unsigned tmem_base = *tmem_slot_ptr;
  const unsigned lead_acc_empty = mapa_cluster(acc_empty, 0);
  long long* const tr = blockIdx.x == 0 ? g.trace : nullptr;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int tile = 0; tile < my_tiles; ++tile) {
        int bx, by;
        tile_at(tile, bx, by);
        const int m_base = g.row0 + by * OZ_BM, n_rel = bx * BN;
        for (int kb = 0; kb < k_stages; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(empty_bar(s), ((it / STAGES) & 1) ^ 1);
          const unsigned st = base + s * Sh::STAGE_BYTES;
          const unsigned lead_full = mapa_cluster(full_bar(s), 0);
          if ((g.debug & 1) && it >= STAGES) {  // rate probe: the MMAs run on whatever the stage buffers hold
            if (rank == 0) mbar_arrive(full_bar(s));
            continue;
          }
          // the leader announces the bytes of BOTH CTAs on its own barrier (a local operation); the peer only issues its loads,
          // whose bytes are counted there too -- a remote arrive.expect_tx per stage cost ~0.5 us of the peer's producer,
          // twice the time the pair needs to consume a stage
          if (rank == 0) mbar_expect_tx(full_bar(s), 2 * Sh::STAGE_BYTES);
#pragma unroll
          for (int t = 0; t < SA; ++t) tma_load_3d_2sm(st + t * Sh::A_SLICE, map_a, kb * BK, m_base, t, lead_full);
          tma_load_3d_2sm(st + Sh::A_BYTES, map_b, kb * BK, n_rel, static_cast<int>(rank), lead_full);  // b_1 here, b_2 in the peer
          if constexpr (SB == 3)  // and this CTA's half of b_3's rows
            tma_load_3d_2sm(st + Sh::A_BYTES + Sh::B1_BYTES, map_b_half, kb * BK, n_rel + static_cast<int>(rank) * (BN / 2), 2, lead_full);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // cute::UMMA::InstrDescriptor for kind::i8 with M = 256 (the pair): D = S32, A = B = signed 8 bit, both K-major, N >> 3 @17
      constexpr unsigned idesc_m = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<unsigned>(256 >> 4) << 24);
      constexpr unsigned idesc_12 = idesc_m | (static_cast<unsigned>((2 * BN) >> 3) << 17);  // a_t x [b_1 | b_2]
      constexpr unsigned idesc_3 = idesc_m | (static_cast<unsigned>(BN >> 3) << 17);         // a_t x b_3
      int it = 0;
      for (int tile = 0; tile < my_tiles; ++tile) {
        // completion #tile: the epilogue warps' initial arrival, then one per drained tile
        if (g.debug & 4096) mbar_wait_spin(acc_empty, tile & 1);
        else mbar_wait(acc_empty, tile & 1);
        tc_fence_after();
        if (tr != nullptr) tr[tile * 8 + 0] = clock64();
        for (int kb = 0; kb < k_stages; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(full_bar(s), (it / STAGES) & 1);
          tc_fence_after();
          if (tr != nullptr && kb == 0) tr[tile * 8 + 1] = clock64();
          const unsigned st = base + s * Sh::STAGE_BYTES;
          const unsigned long long b12 = umma_desc_sw<BK>(st + Sh::A_BYTES), b3 = umma_desc_sw<BK>(st + Sh::A_BYTES + Sh::B1_BYTES);
#pragma unroll
          for (int ks = 0; ks < BK / 32; ++ks) {
            const unsigned long long adv = 2ull * ks;
#pragma unroll
            for (int t = 1; t <= SA; ++t) {
              const unsigned long long a_t = umma_desc_sw<BK>(st + (t - 1) * Sh::A_SLICE) + adv;
              const bool opening = kb == 0 && ks == 0;  // the tile's first k step
              // a_t x [b_1 | b_2]: levels t + 1, t + 2 = column blocks t - 1, t.  a_1 opens both (overwrite); with two b slices a
              // later a_t accumulates into a block t nobody has written (the epilogue left zeros there), with three it was
              // opened by a_(t-1) x b_3
              tc_mma2_i8(tmem_base + (t - 1) * BN, a_t, b12 + adv, idesc_12, (opening && t == 1) ? 0u : 1u);
              if constexpr (SB == 3)  // a_t x b_3: level t + 3 = block t + 1, always a block of its own in the first k step
                tc_mma2_i8(tmem_base + (t + 1) * BN, a_t, b3 + adv, idesc_3, opening ? 0u : 1u);
            }
          }
          tc_commit2_mc(empty_bar(s), 3);
        }
        tc_commit2_mc(acc_full, 3);
        if (tr != nullptr) tr[tile * 8 + 2] = clock64();
      }
    }
  } else {
    const int q = warp % 4;
    const int r = q * 32 + lane;
    const int m_limit = g.row0 + g.rows;
    constexpr int NCH = BN / 16, MY = NCH / 2, LD = 8;
    constexpr bool ZERO_FILL = SB == 2;  // blocks 2 .. LV-1 are only ever accumulated into
    const int grp = (warp - 2) / 4;
    const unsigned slab = cbuf + (warp - 2) * Sh::C_SLAB;
    const unsigned lane_base = tmem_base + (static_cast<unsigned>(q * 32) << 16);
    const unsigned zeros[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if constexpr (ZERO_FILL) {
      // before the first tile: this warp's share of the level blocks that are only ever accumulated into starts from zero
#pragma unroll
      for (int jj = 0; jj < MY; ++jj)
#pragma unroll
        for (int h = 0; h < 16 / LD; ++h)
#pragma unroll
          for (int l = 2; l < LV; ++l) tc_st8_issue(lane_base + l * BN + (grp + 2 * jj) * 16 + h * 8, zeros);
      tc_st_wait();
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_cluster(lead_acc_empty);
    for (int tile = 0; tile < my_tiles; ++tile) {
      int bx, by;
      tile_at(tile, bx, by);
      const int m_base = g.row0 + by * OZ_BM, n_tile = bx * BN;
      const int m = m_base + r;
      int ei;
      const bool na = oz_exp_unpack(m < m_limit ? g.exp_a[m] : 0, ei);
      const bool row_fast = ei > -400 && ei < 400;
      const double pa = pow2(row_fast ? ei - kOzPairUnit : 0);
      int* eb = eb_sh + (tile & 1) * BN;
      double* pb = pb_sh + (tile & 1) * BN;
      if (grp == 0 && r < BN) {
        int e;
        const bool nb = oz_exp_unpack(n_tile + r < g.cols ? g.exp_b[n_tile + r] : 0, e);
        eb[r] = e;
        if constexpr (Sh::SCALE_TABLE) pb[r] = pow2(e > -400 && e < 400 ? e : 0);
        // the columns encoded negated, one bit per column (a whole warp is here: r < BN holds for all of its lanes or none)
        const unsigned negs = __ballot_sync(0xffffffffu, nb);
        if (lane == 0) sg_sh[(tile & 1) * 4 + q] = negs;
      }
      asm volatile("bar.sync 1, 256;\n" ::: "memory");
      if (g.debug & 4096) mbar_wait_spin(acc_full, tile & 1);
      else mbar_wait(acc_full, tile & 1);
      tc_fence_after();
      if (tr != nullptr && warp == 2 && lane == 0) tr[tile * 8 + 3] = clock64();
      if (g.debug & 2048) {  // rate probe: the set is handed back unread (what the drain costs per tile)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(lead_acc_empty);
        continue;
      }
      // phase A: the accumulators leave TMEM as one number per element (a 64-bit integer up to four levels, the Horner sum in
      // FP64 beyond); blocks that are only accumulated into are zeroed behind the read
      long long acc[LV <= 4 ? MY : 1][16];
      double hsum[LV <= 4 ? 1 : MY][16];
#pragma unroll
      for (int jj = 0; jj < MY; ++jj) {
        const int j = grp + 2 * jj;
#pragma unroll
        for (int h = 0; h < 16 / LD; ++h) {
          unsigned lv[LV][LD];
#pragma unroll
          for (int l = 0; l < LV; ++l) tc_ld8_issue(lane_base + l * BN + j * 16 + h * 8, lv[l]);
          tc_ld_wait();
          if constexpr (ZERO_FILL) {
#pragma unroll
            for (int l = 2; l < LV; ++l) tc_st8_issue(lane_base + l * BN + j * 16 + h * 8, zeros);
          }
#pragma unroll
          for (int e = 0; e < LD; ++e) {
            if constexpr (LV <= 4) {
              long long x = static_cast<int>(lv[0][e]);
#pragma unroll
              for (int l = 1; l < LV; ++l) x = (x << kOzDigitBits) + static_cast<int>(lv[l][e]);
              acc[jj][h * LD + e] = x;
            } else {
              double x = static_cast<double>(static_cast<int>(lv[LV - 1][e]));
#pragma unroll
              for (int l = LV - 2; l >= 0; --l) x = fma(x, kOzLevelStep, static_cast<double>(static_cast<int>(lv[l][e])));
              hsum[jj][h * LD + e] = x;
            }
          }
        }
      }
      if constexpr (ZERO_FILL) tc_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(lead_acc_empty);
      if (tr != nullptr && warp == 2 && lane == 0) tr[tile * 8 + 4] = clock64();
      // phase B: scale, stage, reduce into c (overlaps the next tile's MMAs); tiles beyond the edge are dropped by the tensor map
      if (g.debug & 2) continue;
#pragma unroll
      for (int jj = 0; jj < MY; ++jj) {
        const int j = grp + 2 * jj;
        double v[16];
        // bit e: the product of this row and column e of the chunk changes sign (exactly one of the two is encoded negated)
        const unsigned flip = ((sg_sh[(tile & 1) * 4 + (j * 16) / 32] >> ((j * 16) % 32)) & 0xffffu) ^ (na ? 0xffffu : 0u);
        if constexpr (LV <= 4) {
          int ebv[16];
          bool cols_fast = true;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            ebv[e] = eb[j * 16 + e];
            cols_fast &= static_cast<unsigned>(ebv[e] + 399) < 799u;
          }
          if (cols_fast && row_fast) {
            const int e_row = ei - kOzPairUnit - kOzDigitBits * (LV - 1);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const long long x = acc[jj][e];
              const double d = static_cast<double>(x);
              const int hi = x != 0 ? (__double2hiint(d) + (e_row + ebv[e]) * (1 << 20)) ^ static_cast<int>((flip >> e & 1u) << 31) : 0;
              v[e] = __hiloint2double(hi, __double2loint(d));
            }
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = oz_signed(scaled(static_cast<double>(acc[jj][e]) * pow2(-kOzDigitBits * (LV - 1)), ei, ebv[e]), (flip >> e & 1u) != 0);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int ebe = eb[j * 16 + e];
            const double mag = (row_fast && ebe > -400 && ebe < 400) ? (hsum[jj][e] * pa) * pb[j * 16 + e] : scaled(hsum[jj][e], ei, ebe);
            v[e] = oz_signed(mag, (flip >> e & 1u) != 0);
          }
        }
        if (lane == 0) tma_store_wait_read<0>();
        __syncwarp();
        if constexpr (sizeof(CT) == 8) {
          const unsigned crow = slab + lane * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(crow + ((ch ^ (lane & 7)) << 4)), "d"(v[2 * ch]), "d"(v[2 * ch + 1]) : "memory");
        } else {
          const unsigned crow = slab + lane * 64;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(crow + ((ch ^ ((lane >> 1) & 3)) << 4)), "f"(static_cast<float>(v[4 * ch])),
                         "f"(static_cast<float>(v[4 * ch + 1])), "f"(static_cast<float>(v[4 * ch + 2])), "f"(static_cast<float>(v[4 * ch + 3]))
                         : "memory");
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (g.c_zero) tma_store_2d(map_c, slab, g.col0 + n_tile + j * 16, m_base + q * 32);
          else tma_reduce_add_2d(map_c, slab, g.col0 + n_tile + j * 16, m_base + q * 32);
          tma_store_commit();
        }
      }
    }
    if (lane == 0) tma_store_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // neither CTA frees tensor memory or leaves while its peer may still use or signal it
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(512) : "memory");
  }
}

// the tensor maps a launch may need: slices of a in boxes of 128 / 64 rows, slices of bt in boxes of 128 / 64 / 32 rows (whole
// tiles, or the share one CTA of a cluster fetches), c
struct OzMaps {
  CUtensorMap a128, a64, b128, b64, b32, c, b96, b48;  // b96 / b48: the 96-wide tiles of the three-slice pair forms
};
template <int ROWS> __device__ __forceinline__ const CUtensorMap* oz_map_a(const OzMaps& m) {
  static_assert(ROWS == 128 || ROWS == 64, "a box");
  return ROWS == 128 ? &m.a128 : &m.a64;
}
template <int ROWS> __device__ __forceinline__ const CUtensorMap* oz_map_b(const OzMaps& m) {
  static_assert(ROWS == 128 || ROWS == 64 || ROWS == 32, "bt box");
  return ROWS == 128 ? &m.b128 : ROWS == 64 ? &m.b64 : &m.b32;
}
template <int SA, int SB, int LV, int BN, int CR, int CX, int CY, typename CT = double>
__device__ __forceinline__ void oz_persist_form(const OzPArgs& g, const OzMaps& m, unsigned char* smem_raw) {
  oz_persist_body<SA, SB, LV, BN, CR, CX, CY, CT>(g, oz_map_a<OZ_BM / CX>(m), oz_map_b<BN / CY>(m), &m.c, smem_raw);
}

// auto mode: the cheapest error-free form, decided on the device (n is even here: c goes through TMA).  Launched as clusters of
// CX x CY CTAs, which the rectangular forms use to share operand loads; the triangular ones run every CTA on its own.
template <int CX, int CY, typename CT>
__global__ void __launch_bounds__(OZP_THREADS, 1)
matmul_ozaki_auto_kernel(const OzPArgs g, const __grid_constant__ OzMaps maps, const int* __restrict__ guard, int* __restrict__ ran) {
  extern __shared__ unsigned char smem_raw[];
  int form = sizeof(CT) == 8 ? ozaki_pick_form(guard[0] | guard[3], guard[1], guard[2]) : ozaki_pick_form_f32(guard[0] | guard[3], guard[1], guard[2]);
  if (!oz_form_fits_int32(form, g.kq)) form = 0;  // the level sums could leave INT32: the fallback takes the product
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *ran = form;
    if (g.use_cond) cudaGraphSetConditional(g.cond, form == 0 ? 1u : 0u);
  }
  switch (form) {
    case 223: oz_persist_form<2, 2, 3, 128, 1, CX, CY, CT>(g, maps, smem_raw); break;
    case 324: oz_persist_form<3, 2, 4, 128, 1, CX, CY, CT>(g, maps, smem_raw); break;
    case 234: oz_persist_form<2, 3, 4, 128, 1, CX, CY, CT>(g, maps, smem_raw); break;
    case 335: oz_persist_form<3, 3, 5, 64, 1, CX, CY, CT>(g, maps, smem_raw); break;
    case 436: oz_persist_form<4, 3, 6, 64, 1, CX, CY, CT>(g, maps, smem_raw); break;
    case 346: oz_persist_form<3, 4, 6, 64, 1, CX, CY, CT>(g, maps, smem_raw); break;
    case 447: oz_persist_form<4, 4, 7, 64, 1, CX, CY, CT>(g, maps, smem_raw); break;
    case 555: oz_persist_form<5, 5, 5, 64, 1, 1, 1, CT>(g, maps, smem_raw); break;
    default:
      if constexpr (sizeof(CT) == 8) {  // the 6 / 7-slice forms keep the register epilogue (FP64 only)
        if (form == 666) oz_persist_form<6, 6, 6, 64, 0, 1, 1>(g, maps, smem_raw);
        if (form == 777) oz_persist_form<7, 7, 7, 64, 0, 1, 1>(g, maps, smem_raw);
      }
      break;  // 0: not error-free in any form -- not this kernel's launch
  }
}

// auto mode as CTA pairs (clusters of two): the forms with two b slices on 128-wide tiles run as pairs (oz_pair_body), every
// other form runs each CTA of the cluster on its own as in the kernel above
template <typename CT>
__global__ void __launch_bounds__(OZP_THREADS, 1)
matmul_ozaki_auto_pair_kernel(const OzPArgs g, const __grid_constant__ OzMaps maps, const int* __restrict__ guard, int* __restrict__ ran) {
  extern __shared__ unsigned char smem_raw[];
  int form = sizeof(CT) == 8 ? ozaki_pick_form(guard[0] | guard[3], guard[1], guard[2]) : ozaki_pick_form_f32(guard[0] | guard[3], guard[1], guard[2]);
  if (!oz_form_fits_int32(form, g.kq)) form = 0;  // the level sums could leave INT32: the fallback takes the product
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *ran = form;
    if (g.use_cond) cudaGraphSetConditional(g.cond, form == 0 ? 1u : 0u);
  }
  switch (form) {
    case 223: oz_pair_body<2, 2, 3, CT>(g, &maps.a128, &maps.b128, nullptr, &maps.c, smem_raw); break;
    case 324: oz_pair_body<3, 2, 4, CT>(g, &maps.a128, &maps.b128, nullptr, &maps.c, smem_raw); break;
    case 234: oz_pair_body<2, 3, 4, CT>(g, &maps.a128, &maps.b96, &maps.b48, &maps.c, smem_raw); break;
    case 335: oz_pair_body<3, 3, 5, CT>(g, &maps.a128, &maps.b96, &maps.b48, &maps.c, smem_raw); break;
    case 436: oz_persist_form<4, 3, 6, 64, 1, 1, 1, CT>(g, maps, smem_raw); break;
    case 346: oz_persist_form<3, 4, 6, 64, 1, 1, 1, CT>(g, maps, smem_raw); break;
    case 447: oz_persist_form<4, 4, 7, 64, 1, 1, 1, CT>(g, maps, smem_raw); break;
    case 555: oz_persist_form<5, 5, 5, 64, 1, 1, 1, CT>(g, maps, smem_raw); break;
    default:
      if constexpr (sizeof(CT) == 8) {
        if (form == 666) oz_persist_form<6, 6, 6, 64, 0, 1, 1>(g, maps, smem_raw);
        if (form == 777) oz_persist_form<7, 7, 7, 64, 0, 1, 1>(g, maps, smem_raw);
      }
      break;
  }
}

// a fixed triangular slice count (matmul_variant 40 .. 45: general kernels with a truncation bound, no guard); CR = 0 where c
// cannot go through TMA (odd n) or the stage ring needs the space
template <int S, int CR>
__global__ void __launch_bounds__(OZP_THREADS, 1)
matmul_ozaki_fixed_kernel(const OzPArgs g, const __grid_constant__ OzMaps maps) {
  extern __shared__ unsigned char smem_raw[];
  oz_persist_form<S, S, S, 64, CR, 1, 1>(g, maps, smem_raw);
}

// One CTA per row: row maximum -> exponent e (|x| < 2^e), then S digits per element.  dst plane t of row r (relative
// index) is dst + t * plane + r * kq; k >= n is zero.  Rows [src_row0, src_row0 + nrows) of src; rows up to nrows_pad are
// written as zeros with exponent 0 (tile overhang inside the tensor map).
// T = double or float: a float converts to double exactly, so the digits (and everything after) are those of the same number.
template <int S, typename T>
__global__ void __launch_bounds__(256, 4) ozaki_slice_kernel(const T* __restrict__ src, signed char* __restrict__ dst, int* __restrict__ exps,
                                                          size_t plane, int n, int kq, int src_row0, int nrows, int dst_row0,
                                                          int* __restrict__ guard, int lossy_slot, int top_slot, int dirty_slot) {
  __shared__ double red[8], red_lo[8], inv_sh;
  __shared__ int tiny_sh;
  const int r = blockIdx.x;  // relative row
  const int tid = threadIdx.x;
  const bool live = r < nrows;
  const T* x = src + static_cast<size_t>(src_row0 + (live ? r : 0)) * n;
  // 4 consecutive k per thread and iteration: a warp reads 1 KB and writes 128 bytes per slice, both contiguous.  The first
  // KEEP iterations (rows up to 4096 elements) stay in registers between the two passes, so the row is read once.
  constexpr int KEEP = 4;
  const bool vec = sizeof(T) == 8 ? n % 2 == 0 : n % 4 == 0;  // 16-byte aligned rows
  auto load4 = [&](int k0, double (&v)[4]) {
    if (live && vec && k0 + 4 <= n) {
      if constexpr (sizeof(T) == 8) {
        const double2 p = *reinterpret_cast<const double2*>(x + k0), q2 = *reinterpret_cast<const double2*>(x + k0 + 2);
        v[0] = p.x; v[1] = p.y; v[2] = q2.x; v[3] = q2.y;
      } else {
        const float4 p = *reinterpret_cast<const float4*>(x + k0);
        v[0] = p.x; v[1] = p.y; v[2] = p.z; v[3] = p.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = (live && k0 + q < n) ? x[k0 + q] : 0.0;
    }
  };
  double hi = 0.0, lo = 0.0;  // the row's largest and smallest element (zero padding included: harmless)
  int bad = 0;
  auto scan4 = [&](const double (&v)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      bad |= !isfinite(v[q]);
      hi = fmax(hi, v[q]);
      lo = fmin(lo, v[q]);
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
  for (int o = 16; o > 0; o >>= 1) {
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
  }
  if (tid % 32 == 0) {
    red[tid / 32] = hi;
    red_lo[tid / 32] = lo;
  }
  __syncthreads();
  if (tid == 0) {
    double h = red[0], l = red_lo[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      h = fmax(h, red[w]);
      l = fmin(l, red_lo[w]);
    }
    // exponent, sign and scale of the row (ozaki_digits.cuh); exact power of two; a non-finite row gets zero digits, and so does a
    // row whose maximum is below 2^-970 (1 / 2^e would overflow): both are flagged as lossy.  (Digit extraction by 64-bit integer
    // arithmetic was measured slower than the FP64 form of oz_emit: 85 us against 70 us per operand at N = 4096.)
    bool tiny_row;
    double inv_row;
    const int word = oz_row_code(h, l, bad != 0, live, &inv_row, &tiny_row);
    inv_sh = inv_row;
    tiny_sh = tiny_row ? 1 : 0;
    exps[dst_row0 + r] = bad ? kNonFinite : word;
  }
  __syncthreads();
  const bool tiny = tiny_sh != 0;
  const double inv = inv_sh;
  signed char* drow = dst + static_cast<size_t>(dst_row0 + r) * kq;
  int lossy = bad | tiny, top = 0;  // top = highest non-zero digit (1-based) this thread has seen
  // Auto mode keeps an invariant on its scratch (zero-filled when the context is created): planes beyond guard[dirty_slot] hold
  // only zeros.  So zero words need not be written there -- short operands (the application's: two digits) move 2 planes per
  // element instead of 7.  The word only ever grows, to the highest plane any launch wrote a non-zero digit into; a CTA that
  // reads it after a neighbour has raised it merely writes more zeros.
  const int dirty = dirty_slot >= 0 ? guard[dirty_slot] : S;
#pragma unroll
  for (int it = 0; it < KEEP; ++it) {
    const int k0 = (it * 256 + tid) * 4;
    if (k0 < kq) oz_emit<S, 4>(keep[it], inv, bad != 0, dirty, drow, plane, k0, lossy, top);
  }
  for (int k0 = (KEEP * 256 + tid) * 4; k0 < kq; k0 += 256 * 4) {
    double v[4];
    load4(k0, v);
    oz_emit<S, 4>(v, inv, bad != 0, dirty, drow, plane, k0, lossy, top);
  }
  if (guard != nullptr) oz_guard_commit(lossy, top, guard, lossy_slot, top_slot, dirty_slot);
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
template <int P, typename T = double>
cudaError_t oz_slices(const T* a, const T* bt, void* scratch, int n, int row0, int rows, int col0, int cols, cudaStream_t stream,
                      bool with_guard, bool reuse_a, bool reuse_bt = false) {
  const OzLayout L(scratch, n, P);
  int* flag = with_guard ? L.guard : nullptr;
  if (with_guard && !(reuse_a && reuse_bt)) {
    // the words of the operand(s) sliced here: {0, 1} belong to a, {2, 3} to bt
    int* first = reuse_a ? flag + 2 : flag;
    const size_t words = (reuse_a || reuse_bt) ? 2 : 4;
    if (cudaError_t e = cudaMemsetAsync(first, 0, words * sizeof(int), stream); e != cudaSuccess) return e;
  }
  const int cols_pad = static_cast<int>(oz_rows_pad(cols, OZ_BN));
  // guard words: 0 a is cut, 1 top digit of a, 2 top digit of bt, 3 bt is cut (reset per launch); 4 the form the auto kernel took;
  // 5 / 6 highest plane of the a / bt scratch that may hold non-zero bytes (auto mode only; never reset)
  if (!reuse_a) ozaki_slice_kernel<P, T><<<rows, 256, 0, stream>>>(a, L.sa, L.ea, L.a_plane, n, L.kq, row0, rows, row0, flag, 0, 1, with_guard ? 5 : -1);
  if (!reuse_bt) ozaki_slice_kernel<P, T><<<cols_pad, 256, 0, stream>>>(bt, L.sb, L.eb, L.b_plane, n, L.kq, col0, cols, 0, flag, 3, 2, with_guard ? 6 : -1);
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

// ---- persistent form: host side ------------------------------------------------------------------------------------------
int oz_sm_count() {
  static PerDeviceOnce once;
  static int count[64] = {};
  int d = 0;
  cudaGetDevice(&d);
  bool& known = once.here();
  if (!known) {
    if (cudaDeviceGetAttribute(&count[d & 63], cudaDevAttrMultiProcessorCount, d) != cudaSuccess || count[d & 63] <= 0) count[d & 63] = 148;
    known = true;
  }
  return count[d & 63];
}

template <typename Kernel>
cudaError_t oz_persist_configure(Kernel kernel, int smem, PerDeviceOnce& once) {
  bool& configured = once.here();
  if (!configured) {
    if (cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); e != cudaSuccess) return e;
    configured = true;
  }
  return cudaSuccess;
}
template <int CX, int CY, typename CT = double> cudaError_t oz_auto_configure() {
  static PerDeviceOnce once;
  return oz_persist_configure(matmul_ozaki_auto_kernel<CX, CY, CT>, kOzPersistSmemMax, once);
}

// clusters of CX x CY CTAs the device can keep resident with one CTA per SM (0 on failure)
template <int CX, int CY> int oz_auto_max_clusters() {
  if (oz_auto_configure<CX, CY>() != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(oz_sm_count() / (CX * CY) * (CX * CY)));
  cfg.blockDim = dim3(OZP_THREADS);
  cfg.dynamicSmemBytes = kOzPersistSmemMax;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CX * CY;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, matmul_ozaki_auto_kernel<CX, CY, double>, &cfg) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return clusters;
}

// The cluster shape of the auto launch on this device: {shape code 22 / 21 / 11, resident clusters}.  Default 11 (no clusters):
// measured on B200 (profiles/r1e_cluster_shapes.txt) sharing the operand loads changes nothing at 2 x 1 and costs 8-12 % at
// 2 x 2 -- the short forms wait on the epilogue and on refill latency, not on L2 bandwidth (6.3 of 11.8 TB/s).  MMX_OZ_CLUSTER_SHAPE
// = 21 / 22 selects the multicast forms (kept as a measured tuning point, and for devices where the balance differs).
struct OzClusterChoice {
  int shape = 0, clusters = 0;
};
OzClusterChoice oz_auto_cluster_choice() {
  static PerDeviceOnce once;
  static OzClusterChoice choice[64];
  int d = 0;
  cudaGetDevice(&d);
  bool& known = once.here();
  if (!known) {
    static const int forced = [] { const char* e = getenv("MMX_OZ_CLUSTER_SHAPE"); return e ? atoi(e) : 0; }();
    const int sms = oz_sm_count();
    OzClusterChoice c;
    const int n22 = forced == 22 ? oz_auto_max_clusters<2, 2>() : 0;
    const int n21 = forced == 21 ? oz_auto_max_clusters<2, 1>() : 0;
    if (n22 > 0) {
      c.shape = 22;
      c.clusters = n22;
    } else if (n21 > 0) {
      c.shape = 21;
      c.clusters = n21;
    } else {
      (void)oz_auto_configure<1, 1>();
      c.shape = 11;
      c.clusters = sms;
    }
    choice[d & 63] = c;
    known = true;
  }
  return choice[d & 63];
}

// The pair kernel (clusters of two CTAs): configured once per device; `clusters` = pairs the device keeps resident with one CTA per
// SM (0: pairs unavailable -- the one-CTA auto kernel is used).  MMX_OZ_PAIR=0 switches the pairs off (A/B runs).
template <typename CT> int oz_pair_clusters() {
  static PerDeviceOnce once;
  static int clusters[64] = {};
  int d = 0;
  cudaGetDevice(&d);
  bool& known = once.here();
  if (!known) {
    known = true;
    clusters[d & 63] = 0;
    static const int enabled = [] { const char* e = getenv("MMX_OZ_PAIR"); return e ? atoi(e) : 1; }();
    if (enabled && cudaFuncSetAttribute(matmul_ozaki_auto_pair_kernel<CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kOzPersistSmemMax) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(oz_sm_count() / 2 * 2));
      cfg.blockDim = dim3(OZP_THREADS);
      cfg.dynamicSmemBytes = kOzPersistSmemMax;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, matmul_ozaki_auto_pair_kernel<CT>, &cfg) == cudaSuccess && n > 0) clusters[d & 63] = std::min(n, oz_sm_count() / 2);
    }
    (void)cudaGetLastError();
  }
  return clusters[d & 63];
}

template <int S, int CR> cudaError_t oz_fixed_configure() {
  static PerDeviceOnce once;
  return oz_persist_configure(matmul_ozaki_fixed_kernel<S, CR>, OzPShape<S, S, S, 64, CR>::SMEM_BYTES, once);
}
constexpr int oz_fixed_ring(int s) { return s <= 4 ? 1 : 0;  /* chunk buffers of c where the stage ring leaves room */ }

// c as a 2-D tensor of doubles that ends at (rows_end, cols_end): box = 32 rows x 16 columns (one warp's slab), 128-byte swizzle
bool make_c_map(CUtensorMap* map, void* c, size_t elem, int n, int rows_end, int cols_end) {
  EncodeTiledFn enc = encode_tiled();
  if (enc == nullptr) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols_end), static_cast<cuuint64_t>(rows_end)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(n) * elem};
  const cuuint32_t box[2] = {16, 32};
  const cuuint32_t ones[2] = {1, 1};
  return enc(map, elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, c, dims, strides, box, ones, CU_TENSOR_MAP_INTERLEAVE_NONE,
             elem == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// slices == 0: the auto kernel (reads the guard, records the form it ran in guard[4]); otherwise the fixed triangular form over
// the first `slices` of `planes` planes
template <typename CT = double>
cudaError_t oz_persist_contract(CT* c, void* scratch, int planes, int slices, int n, int row0, int rows, int col0, int cols, cudaStream_t stream,
                                bool c_zero = false, const OzFallbackCond* cond = nullptr) {
  const OzLayout L(scratch, n, planes);
  const bool c_by_tma = (n * sizeof(CT)) % 16 == 0;  // row pitch a multiple of 16 bytes
  if (slices == 0 && !c_by_tma) return cudaErrorInvalidValue;
  OzMaps maps;
  if (!make_slice_map(&maps.a128, L.sa, static_cast<size_t>(n), L.kq, 64, 128, planes, 1) ||
      !make_slice_map(&maps.a64, L.sa, static_cast<size_t>(n), L.kq, 64, 64, planes, 1) ||
      !make_slice_map(&maps.b128, L.sb, L.b_rows, L.kq, 64, 128, planes, 1) || !make_slice_map(&maps.b64, L.sb, L.b_rows, L.kq, 64, 64, planes, 1) ||
      !make_slice_map(&maps.b32, L.sb, L.b_rows, L.kq, 64, 32, planes, 1) || !make_slice_map(&maps.b96, L.sb, L.b_rows, L.kq, 64, 96, planes, 1) ||
      !make_slice_map(&maps.b48, L.sb, L.b_rows, L.kq, 64, 48, planes, 1))
    return cudaErrorNotSupported;
  if (c_by_tma) {
    if (!make_c_map(&maps.c, c, sizeof(CT), n, row0 + rows, col0 + cols)) return cudaErrorNotSupported;
  } else {
    maps.c = maps.a128;  // never dereferenced
  }
  OzPArgs g;
  g.c = c;
  g.exp_a = L.ea;
  g.exp_b = L.eb;
  g.n = n;
  g.kq = L.kq;
  g.row0 = row0;
  g.rows = rows;
  g.col0 = col0;
  g.cols = cols;
  g.group = raster_group(OZ_BM, static_cast<size_t>(L.kq));
  static const long long group_mb = [] { const char* e = getenv("MMX_OZ_GROUP_MB"); return e ? atoll(e) : 0ll; }();
  g.group_l2_bytes = group_mb << 20;
  g.c_zero = (c_zero && c_by_tma) ? 1 : 0;  // (the register epilogue adds: it reads c anyway)
  g.cond = (cond != nullptr && cond->active) ? cond->handle : 0ull;
  g.use_cond = (cond != nullptr && cond->active) ? 1 : 0;
  static const int debug = [] { const char* e = getenv("MMX_OZ_DEBUG"); return e ? atoi(e) : 0; }();
  g.debug = debug;
  static const int trace_on = [] { const char* e = getenv("MMX_OZ_TRACE"); return e ? atoi(e) : 0; }();
  static long long* trace_buf = nullptr;  // one device, one stream at a time: a measuring hook, not a product path
  constexpr int kTraceWords = 8 * 4096;
  if (trace_on && trace_buf == nullptr && cudaMalloc(&trace_buf, kTraceWords * sizeof(long long)) != cudaSuccess) trace_buf = nullptr;
  g.trace = trace_on ? trace_buf : nullptr;
  if (g.trace != nullptr) {  // never inside a capture (the dump below synchronises)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) g.trace = nullptr;
  }
  if (g.trace != nullptr) cudaMemsetAsync(g.trace, 0, kTraceWords * sizeof(long long), stream);
  // the grid covers the 64-wide tiling (the forms with 128-wide tiles leave the surplus CTAs without a tile)
  const int tiles_x = (cols + 63) / 64, tiles_y = (rows + OZ_BM - 1) / OZ_BM;
  const dim3 grid(static_cast<unsigned>(std::min(tiles_x * tiles_y, oz_sm_count())));
  switch (slices) {
    case 0: {
      if (const int pairs = oz_pair_clusters<CT>(); pairs > 0) {
        // every resident pair is launched: a pair (or, in the one-CTA forms, a CTA) beyond the tile count finds no tile
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
        cfg.blockDim = dim3(OZP_THREADS);
        cfg.dynamicSmemBytes = kOzPersistSmemMax;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const int* guard_words = L.guard;
        int* ran_word = L.guard + 4;
        const cudaError_t le = cudaLaunchKernelEx(&cfg, matmul_ozaki_auto_pair_kernel<CT>, g, maps, guard_words, ran_word);
        if (g.trace != nullptr && le == cudaSuccess) {  // MMX_OZ_TRACE: the leader pair's clocks, one line per tile on stderr
          static long long host[kTraceWords];
          if (cudaStreamSynchronize(stream) == cudaSuccess && cudaMemcpy(host, g.trace, sizeof(host), cudaMemcpyDeviceToHost) == cudaSuccess)
            for (int t = 0; t < kTraceWords / 8 && host[t * 8] != 0; ++t)
              fprintf(stderr, "oztrace n=%d tile=%d free=%lld first_full=%lld committed=%lld seen=%lld arrived=%lld\n", n, t, host[t * 8] - host[0],
                      host[t * 8 + 1] - host[0], host[t * 8 + 2] - host[0], host[t * 8 + 3] - host[0], host[t * 8 + 4] - host[0]);
        }
        return le;
      }
      OzClusterChoice cc = oz_auto_cluster_choice();
      if (sizeof(CT) != 8 && cc.shape != 11) {  // the multicast forms are instantiated for FP64 only
        cc.shape = 11;
        cc.clusters = oz_sm_count();
      }
      const int cx = cc.shape / 10, cy = cc.shape % 10;
      const int supers = ((tiles_x + cx - 1) / cx) * ((tiles_y + cy - 1) / cy);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(std::min(supers, cc.clusters) * cx * cy));
      cfg.blockDim = dim3(OZP_THREADS);
      cfg.dynamicSmemBytes = kOzPersistSmemMax;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = static_cast<unsigned>(cx * cy);
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = cx * cy > 1 ? 1 : 0;
      const int* guard = L.guard;
      int* ran = L.guard + 4;
      if constexpr (sizeof(CT) == 8) {
        if (cc.shape == 22) return cudaLaunchKernelEx(&cfg, matmul_ozaki_auto_kernel<2, 2, double>, g, maps, guard, ran);
        if (cc.shape == 21) return cudaLaunchKernelEx(&cfg, matmul_ozaki_auto_kernel<2, 1, double>, g, maps, guard, ran);
      }
      if (cudaError_t e = oz_auto_configure<1, 1, CT>(); e != cudaSuccess) return e;
      return cudaLaunchKernelEx(&cfg, matmul_ozaki_auto_kernel<1, 1, CT>, g, maps, guard, ran);
    }
#define MMX_OZ_FIXED(S)                                                                                                                       \
  case S:                                                                                                                                     \
    if constexpr (sizeof(CT) != 8) return cudaErrorInvalidValue;                                                                              \
    if (c_by_tma && oz_fixed_ring(S) > 0) {                                                                                                   \
      if (cudaError_t e = oz_fixed_configure<S, oz_fixed_ring(S)>(); e != cudaSuccess) return e;                                              \
      matmul_ozaki_fixed_kernel<S, oz_fixed_ring(S)><<<grid, OZP_THREADS, OzPShape<S, S, S, 64, oz_fixed_ring(S)>::SMEM_BYTES, stream>>>(g, maps); \
    } else {                                                                                                                                  \
      if (cudaError_t e = oz_fixed_configure<S, 0>(); e != cudaSuccess) return e;                                                             \
      matmul_ozaki_fixed_kernel<S, 0><<<grid, OZP_THREADS, OzPShape<S, S, S, 64, 0>::SMEM_BYTES, stream>>>(g, maps);           \
    }                                                                                                                                         \
    break;
      MMX_OZ_FIXED(2)
      MMX_OZ_FIXED(3)
      MMX_OZ_FIXED(4)
      MMX_OZ_FIXED(5)
      MMX_OZ_FIXED(6)
      MMX_OZ_FIXED(7)
#undef MMX_OZ_FIXED
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
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
  if (cudaError_t e = oz_configure<6, 1, 64>(); e != cudaSuccess) return e;
  (void)oz_auto_cluster_choice();  // configures the auto kernel of the chosen cluster shape
  if (cudaError_t e = oz_auto_configure<1, 1, float>(); e != cudaSuccess) return e;
  (void)oz_pair_clusters<double>();  // ... and the pair kernels (first-use work must not happen inside a stream capture)
  (void)oz_pair_clusters<float>();
  if (cudaError_t e = oz_fixed_configure<2, 0>(); e != cudaSuccess) return e;
  if (cudaError_t e = oz_fixed_configure<3, 0>(); e != cudaSuccess) return e;
  if (cudaError_t e = oz_fixed_configure<4, 0>(); e != cudaSuccess) return e;
  if (cudaError_t e = oz_fixed_configure<2, 1>(); e != cudaSuccess) return e;
  if (cudaError_t e = oz_fixed_configure<3, 1>(); e != cudaSuccess) return e;
  if (cudaError_t e = oz_fixed_configure<4, 1>(); e != cudaSuccess) return e;
  if (cudaError_t e = oz_fixed_configure<5, 0>(); e != cudaSuccess) return e;
  if (cudaError_t e = oz_fixed_configure<6, 0>(); e != cudaSuccess) return e;
  return oz_fixed_configure<7, 0>();
}

size_t matmul_ozaki_scratch_bytes(int n) {
  const size_t kq = static_cast<size_t>(oz_kq(n));
  return 7 * (static_cast<size_t>(n) + oz_rows_pad(n, OZ_BN)) * kq + 2 * (static_cast<size_t>(n) + OZ_BN) * sizeof(int) + 256;  // + the guard flag
}

// FP32 auto mode: the same digit planes from float operands (a float is a double), the same contraction, c in float (the exact
// value rounded once, added by a FLOAT32 TMA reduction).  *guard_out receives the guard; the caller enqueues the split-TF32 path
// under ozaki_pick_form_f32(...) == 0.
cudaError_t launch_matmul_ozaki_f32(float* c, const float* a, const float* bt, void* scratch, int n, int row0, int rows, int col0, int cols,
                                    cudaStream_t stream, int** guard_out, bool reuse_a, bool reuse_bt, bool c_zero, const OzFallbackCond* cond) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (scratch == nullptr || guard_out == nullptr || n % 4 != 0) return cudaErrorInvalidValue;
  *guard_out = OzLayout(scratch, n, 7).guard;
  if (cudaError_t e = oz_slices<7, float>(a, bt, scratch, n, row0, rows, col0, cols, stream, true, reuse_a, reuse_bt); e != cudaSuccess) return e;
  return oz_persist_contract<float>(c, scratch, 7, 0, n, row0, rows, col0, cols, stream, c_zero, cond);
}

OzOperand matmul_ozaki_operand(void* scratch, int n, int which) {
  const OzLayout L(scratch, n, 7);
  OzOperand o;
  o.kq = L.kq;
  o.guard = L.guard;
  if (which == 0) {
    o.planes = L.sa; o.plane = L.a_plane; o.exps = L.ea; o.lossy_slot = 0; o.top_slot = 1; o.dirty_slot = 5;
  } else {
    o.planes = L.sb; o.plane = L.b_plane; o.exps = L.eb; o.lossy_slot = 3; o.top_slot = 2; o.dirty_slot = 6;
  }
  return o;
}

int* matmul_ozaki_form_word(void* scratch, int n) { return scratch == nullptr ? nullptr : OzLayout(scratch, n, 7).guard + 4; }

cudaError_t launch_matmul_ozaki(double* c, const double* a, const double* bt, void* scratch, int n, int row0, int rows, int col0, int cols,
                                int slices, cudaStream_t stream, int** guard_out, bool reuse_a, bool reuse_bt, bool c_zero, const OzFallbackCond* cond) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (scratch == nullptr) return cudaErrorInvalidValue;
  // MMX_OZ_LEGACY=1: the one-tile-per-CTA kernels of the first version (A/B comparison, tools/ozaki_cluster_sweep.sh)
  static const int legacy = [] { const char* e = getenv("MMX_OZ_LEGACY"); return e ? atoi(e) : 0; }();
  if (guard_out != nullptr) {
    // auto mode: 7 digit planes and the guard once, then ONE persistent launch that reads the guard and runs the cheapest
    // error-free form (2 .. 7 slices) or nothing; the caller adds the FP64-pipe kernel under the remaining condition
    *guard_out = OzLayout(scratch, n, 7).guard;
    if (!(reuse_a && reuse_bt))  // both reused: the digit planes and the guard stand as their producers left them
      if (cudaError_t e = oz_slices<7>(a, bt, scratch, n, row0, rows, col0, cols, stream, true, reuse_a, reuse_bt); e != cudaSuccess) return e;
    if (!legacy) return oz_persist_contract(c, scratch, 7, 0, n, row0, rows, col0, cols, stream, c_zero, cond);
    if (cudaError_t e = oz_contract<6, 1, 64>(c, scratch, 7, n, row0, rows, col0, cols, stream, true); e != cudaSuccess) return e;
    return oz_contract<7, 1, 64>(c, scratch, 7, n, row0, rows, col0, cols, stream, true);
  }
  if (legacy) {
    if (reuse_a) return oz_go<7, 1, 64>(c, a, bt, scratch, n, row0, rows, col0, cols, stream, true);
    // tuning hooks: CTAs per cluster sharing the a slices by multicast, k bytes per stage
    static const int cluster = [] { const char* e = getenv("MMX_OZ_CLUSTER"); return e ? atoi(e) : 1; }();
    static const int bk = [] { const char* e = getenv("MMX_OZ_BK"); return e ? atoi(e) : 64; }();
    if (slices == 6) return oz_go<6, 1, 64>(c, a, bt, scratch, n, row0, rows, col0, cols, stream);
    if (cluster == 4) return oz_go<7, 4, 64>(c, a, bt, scratch, n, row0, rows, col0, cols, stream);
    if (cluster == 2) return oz_go<7, 2, 64>(c, a, bt, scratch, n, row0, rows, col0, cols, stream);
    if (bk == 32) return oz_go<7, 1, 32>(c, a, bt, scratch, n, row0, rows, col0, cols, stream);
    return oz_go<7, 1, 64>(c, a, bt, scratch, n, row0, rows, col0, cols, stream);
  }
  // a fixed slice count: S planes are written and contracted (a general kernel with the truncation bound of the header)
  if (!oz_form_fits_int32(slices * 111, oz_kq(n))) return cudaErrorNotSupported;  // the level sums could leave INT32 at this K
  cudaError_t e = cudaErrorInvalidValue;
  switch (slices) {
    case 2: e = oz_slices<2>(a, bt, scratch, n, row0, rows, col0, cols, stream, false, reuse_a); break;
    case 3: e = oz_slices<3>(a, bt, scratch, n, row0, rows, col0, cols, stream, false, reuse_a); break;
    case 4: e = oz_slices<4>(a, bt, scratch, n, row0, rows, col0, cols, stream, false, reuse_a); break;
    case 5: e = oz_slices<5>(a, bt, scratch, n, row0, rows, col0, cols, stream, false, reuse_a); break;
    case 6: e = oz_slices<6>(a, bt, scratch, n, row0, rows, col0, cols, stream, false, reuse_a); break;
    case 7: e = oz_slices<7>(a, bt, scratch, n, row0, rows, col0, cols, stream, false, reuse_a); break;
    default: break;
  }
  if (e != cudaSuccess) return e;
  return oz_persist_contract(c, scratch, slices, slices, n, row0, rows, col0, cols, stream);
}

}  // namespace mmx
