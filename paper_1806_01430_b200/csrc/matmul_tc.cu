// matmul_tc.cu -- gene 8 in FP32 on the 5th-generation tensor cores: c[i][j] += sum_k a[i][k] * bt[j][k]
// (fixtures/matmul.c:25-28) as a split-precision ("3xTF32") tcgen05 GEMM.
//
// tcgen05 has no FP32-input kind, and one TF32 product (10-bit mantissa) would miss the 1e-6 bar by three
// orders of magnitude.  Each FP32 operand is therefore split exactly into two TF32-representable parts,
//     x = x_hi + x_lo,   x_hi = rna_tf32(x),   x_lo = x - x_hi   (exact in FP32, |x_lo| <= 2^-12 |x|)
// and the product is rebuilt from three tensor-core products
//     a*b ~= a_hi*b_hi + a_hi*b_lo + a_lo*b_hi                   (dropped: a_lo*b_lo, <= 2^-24 |a b|)
// so every product carries a relative error of about 2^-22 -- FP32-class -- at a third of the TF32 rate,
// which is still several times the FFMA pipe's peak.
//
// Accumulation.  The tensor core adds into FP32 accumulators in TMEM with truncation (measured: the error of a
// K-long in-TMEM sum grows like K^2 on smooth data, consistent with round-toward-zero), and a plain FP32
// running sum over K = 4096 smooth terms is itself what puts the CPU float program ~8x over the 1e-6
// norm-wise bar on the application's own inputs.  So the sum is kept in two levels:
//   level 1  the MMAs accumulate one K-chunk (64 k = 4 pipeline stages) into a TMEM buffer;
//   level 2  drain warps add the finished chunk into master accumulators in registers with round-to-nearest
//            while the MMAs already fill the other TMEM buffer.
// Default ("compensated", 128 x 128 tile): every level-2 addition is an error-free TwoSum (on packed pairs,
// FADD2) and the rounding errors are accumulated in a third TMEM region, so the masters are carried as
// unevaluated sums hi + lo and only the short in-chunk sums round: measured max error 0.47-0.59 of the bar on
// the application's inputs at N = 1000..8192 (0.05-0.1 on uniform random inputs).
// "Wide" (variant 31, 128 x 256 tile, plain FP32 masters): ~1.45x faster, 1.6-2.9 of the bar on the
// application's smooth inputs (still 3-5x more accurate than the CPU float program), 0.1 on random inputs.
//
// Who runs it.  matmul_variant 30 / 31 always; FP32 auto mode (variant 0, N >= 1024) as the FALLBACK of the exact INT8 forms
// (matmul_ozaki.cu): its three launches are enqueued behind the auto kernel with `run_if` = the guard, and do nothing when an
// INT8 form took the product.
//
// Two kernels share this scheme:
//   matmul_3xtf32s_kernel  (default, "stacked", below)  128 x 128 output tile, compensated masters; the two parts of b are
//               stacked along N so that two of the three products run as ONE N = 256 MMA (the N = 128 shape reaches only
//               ~0.6 of the tensor pipe's rate).  384 threads: TMA warp, MMA warp, TMEM allocator, eight drain warps that
//               take their registers from the other warpgroup with setmaxnreg.
//               Measured on B200 (split passes included), N = 4096 / 8192: 203 / 237 TFLOP/s of FP32 work, max error
//               0.34 / 0.38 of the 1e-6 norm-wise bar on the application's inputs; MMA-bound limit of the same kernel
//               (chunk = 512 k, drain negligible) 213 / 249.
//   matmul_3xtf32_kernel   one part per MMA (three N = BN products per 8 k), 320 threads:
//               BN = 128 compensated (MMX_TC_MODE=13804; 156 / 171 TFLOP/s, the previous default) and
//               BN = 256 "wide" with plain FP32 masters (variant 31; 230 / 297 TFLOP/s, 1.6-2.9 of the bar on the
//               application's smooth inputs, 0.1 on random inputs).
// Common structure (one CTA per tile of c, 1 CTA per SM):
//   split pass  x -> x_hi, x_lo planes laid out so that one 128-byte swizzle row carries one pipeline stage of a row
//   warp 0      TMA producer: ring of 32-64 KB stages, SWIZZLE_128B
//   warp 1      MMA issuer (one thread): tcgen05.mma.kind::tf32 into TMEM chunk buffer `chunk & 1`; tcgen05.commit releases
//               the stage / publishes the chunk
//   drain warps tcgen05.ld the finished chunk (warp w owns lanes 32*(w%4).. and one column half), fold it into the
//               masters; at the end c += master
// Out-of-range rows/columns are zero-filled (TMA / the split pass) and masked in the epilogue, so any N % 4 == 0 works.
// With the loads disabled the kernels run at the same speed: they are bound by the tensor pipe at the clocks the chip
// sustains, not by TMA or L2.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "raster.cuh"
#include "tc_ptx.cuh"

namespace mmx {
namespace {

constexpr int TC_BM = 128, TC_BK = 16;
constexpr int TC_THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 drain
constexpr int TC_ROW_BYTES = 2 * TC_BK * 4;          // one packed row of a stage: 16 hi + 16 lo floats = 128 bytes
constexpr int TC_A_BYTES = TC_BM * TC_ROW_BYTES;     // 16 KB
constexpr int TC_SMEM_LIMIT = 227 * 1024;

template <int BN> struct TcShape {
  static constexpr int B_BYTES = BN * TC_ROW_BYTES;
  static constexpr int STAGE_BYTES = TC_A_BYTES + B_BYTES;            // 48 KB (BN = 256) / 32 KB (BN = 128)
  static constexpr int STAGES = (TC_SMEM_LIMIT - 2048) / STAGE_BYTES;  // 4 / 7 -> capped below
  static constexpr int NSTAGES = STAGES > 6 ? 6 : STAGES;
  static constexpr int SMEM_BYTES = NSTAGES * STAGE_BYTES + 1024 /*alignment slack*/ + 256 /*barriers*/;
  static constexpr unsigned TMEM_COLS = 512;                           // two chunk buffers; BN = 128: + the compensation terms
};

// K-major operand tile in the SWIZZLE_128B layout: rows of 128 bytes, 8-row groups 1024 bytes apart
// (cute::UMMA::SmemDescriptor: start >> 4 at [0,14), SBO >> 4 at [32,46), version 1 at [46,48), layout at [61,64))
__device__ __forceinline__ unsigned long long umma_desc_sw128(unsigned smem_addr) {
  return static_cast<unsigned long long>((smem_addr & 0x3FFFF) >> 4) | (static_cast<unsigned long long>(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
// cute::UMMA::InstrDescriptor: D = F32 (1 @4), A = B = TF32 (2 @7, 2 @10), both K-major, N >> 3 @17, M >> 4 @24
template <int BN> __host__ __device__ constexpr unsigned idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<unsigned>(BN >> 3) << 17) | (static_cast<unsigned>(TC_BM >> 4) << 24);
}

// c + (hi + lo), rounded once
__device__ __forceinline__ float fold_comp(float cin, float hi, float lo) {
  return static_cast<float>(static_cast<double>(cin) + static_cast<double>(hi) + static_cast<double>(lo));
}

// BN: tile width (256: FP32 masters; 128: masters carried as an unevaluated sum hi + lo, every addition's rounding
// error kept).  CHUNK_STAGES: pipeline stages (16 k each) accumulated inside the tensor core before a drain.
template <int BN, int CHUNK_STAGES, bool COMP>
__global__ void __launch_bounds__(TC_THREADS, 1)
matmul_3xtf32_kernel(float* __restrict__ c, const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, int n,
                     int row0, int rows, int col0, int cols, int debug_noload, int group) {
  using S = TcShape<BN>;
  constexpr int STAGES = S::NSTAGES;
  constexpr int COLS = BN / 2;  // columns per drain thread
  static_assert(!COMP || BN == 128, "compensated masters need 2 registers per output: 128 x 128 tile");
  extern __shared__ unsigned char smem_raw[];
  const unsigned raw = smem_u32(smem_raw);
  const unsigned base = (raw + 1023u) & ~1023u;  // swizzled tiles want their pattern period aligned
  const unsigned bars = base + STAGES * S::STAGE_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull_bar = [&](int b) { return bars + 8u * (2 * STAGES + b); };
  auto tempty_bar = [&](int b) { return bars + 8u * (2 * STAGES + 2 + b); };
  const unsigned tmem_slot = bars + 8u * (2 * STAGES + 4);
  volatile unsigned* tmem_slot_ptr = reinterpret_cast<volatile unsigned*>(smem_raw + (tmem_slot - raw));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int bx, by;
  raster_tile(group, bx, by);
  const int m_base = row0 + by * TC_BM, n_base = col0 + bx * BN;
  const int k_stages = (n + TC_BK - 1) / TC_BK;
  const int n_chunks = (k_stages + CHUNK_STAGES - 1) / CHUNK_STAGES;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 8 * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tmem_slot), "n"(S::TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem_base = *tmem_slot_ptr;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < k_stages; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(empty_bar(s), ((kb / STAGES) & 1) ^ 1);
        const unsigned st = base + s * S::STAGE_BYTES;
        if (debug_noload) {  // rate probe: the MMAs run on whatever the tile buffers hold
          mbar_arrive(full_bar(s));
          continue;
        }
        mbar_expect_tx(full_bar(s), S::STAGE_BYTES);
        const int kp = kb * 2 * TC_BK;  // packed coordinate: 32 floats per 16 k
        tma_load_2d(st, &map_a, kp, m_base, full_bar(s));
        tma_load_2d(st + TC_A_BYTES, &map_b, kp, n_base, full_bar(s));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr unsigned idesc = idesc_tf32<BN>();
      for (int kb = 0; kb < k_stages; ++kb) {
        const int s = kb % STAGES;
        const int chunk = kb / CHUNK_STAGES, in_chunk = kb % CHUNK_STAGES, buf = chunk & 1;
        if (in_chunk == 0) {  // the drain warps must have emptied this buffer (two chunks ago)
          mbar_wait(tempty_bar(buf), ((chunk >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        mbar_wait(full_bar(s), (kb / STAGES) & 1);
        tc_fence_after();
        const unsigned st = base + s * S::STAGE_BYTES;
        // a packed row is [hi k0..15 | lo k0..15]: MMA k-slices (8 k = 32 bytes) 0,1 are hi, 2,3 are lo
        const unsigned long long a_hi = umma_desc_sw128(st), a_lo = a_hi + 4;
        const unsigned long long b_hi = umma_desc_sw128(st + TC_A_BYTES), b_lo = b_hi + 4;
        const unsigned d = tmem_base + buf * BN;
#pragma unroll
        for (int k = 0; k < TC_BK / 8; ++k) {
          const unsigned long long adv = 2ull * k;  // 32 bytes along K inside the swizzle row
          // corrections first, then the leading term
          tc_mma_tf32(d, a_hi + adv, b_lo + adv, idesc, (in_chunk | k) != 0);
          tc_mma_tf32(d, a_lo + adv, b_hi + adv, idesc, 1);
          tc_mma_tf32(d, a_hi + adv, b_hi + adv, idesc, 1);
        }
        tc_commit(empty_bar(s));  // the stage may be refilled once these MMAs have read it
        if (in_chunk == CHUNK_STAGES - 1 || kb == k_stages - 1) tc_commit(tfull_bar(buf));
      }
    }
  } else {
    // drain warps: TMEM lanes 32*(warp%4).., columns half*COLS..
    const int q = warp % 4, half = (warp - 2) / 4;
    // masters as packed pairs (element 2p in the low word) so that the compensated form can use FADD2
    unsigned long long master2[COLS / 2];
#pragma unroll
    for (int i = 0; i < COLS / 2; ++i) master2[i] = 0ull;
    // COMP: the running rounding error of every master lives in TMEM columns [2 BN, 3 BN) -- the register file
    // cannot hold two words per output next to the drain's working set
    const unsigned tcomp = tmem_base + (static_cast<unsigned>(q * 32) << 16) + 2 * BN + half * COLS;
    if constexpr (COMP) {
      unsigned z[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
      for (int g = 0; g < COLS / 16; ++g) tc_st16_issue(tcomp + g * 16, z);
      tc_st_wait();
    }
    for (int chunk = 0; chunk < n_chunks; ++chunk) {
      const int buf = chunk & 1;
      mbar_wait(tfull_bar(buf), (chunk >> 1) & 1);
      tc_fence_after();
      const unsigned t = tmem_base + (static_cast<unsigned>(q * 32) << 16) + buf * BN + half * COLS;
      if constexpr (COMP) {
#pragma unroll
        for (int g = 0; g < COLS / 16; ++g) {
          unsigned v[16], cv[16];
          tc_ld16_issue(t + g * 16, v);
          tc_ld16_issue(tcomp + g * 16, cv);
          tc_ld_wait();
          if (g == COLS / 16 - 1) {  // the chunk buffer is in registers: hand it back before the arithmetic
            tc_fence_before();
            mbar_arrive(tempty_bar(buf));
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            // Knuth TwoSum on two outputs at once: s = m + v exactly as s + e
            const unsigned long long m = master2[g * 8 + i], x = pack2(v[2 * i], v[2 * i + 1]);
            const unsigned long long sum = add2(m, x), bb = sub2(sum, m);
            const unsigned long long e = add2(sub2(m, sub2(sum, bb)), sub2(x, bb));
            master2[g * 8 + i] = sum;
            unpack2(add2(pack2(cv[2 * i], cv[2 * i + 1]), e), cv[2 * i], cv[2 * i + 1]);
          }
          tc_st16_issue(tcomp + g * 16, cv);
        }
        tc_st_wait();
      } else {
#pragma unroll
        for (int g = 0; g < COLS / 32; ++g) {
          float v[32];
          tc_ld32(t + g * 32, v);
          if (g == COLS / 32 - 1) {
            tc_fence_before();
            mbar_arrive(tempty_bar(buf));
          }
#pragma unroll
          for (int i = 0; i < 16; ++i)
            master2[g * 16 + i] = add2(master2[g * 16 + i], pack2(__float_as_uint(v[2 * i]), __float_as_uint(v[2 * i + 1])));
        }
      }
    }
    float master[COLS];
#pragma unroll
    for (int i = 0; i < COLS / 2; ++i) {
      unsigned lo, hi;
      unpack2(master2[i], lo, hi);
      master[2 * i] = __uint_as_float(lo);
      master[2 * i + 1] = __uint_as_float(hi);
    }
    // epilogue: c += master (row = TMEM lane, COLS consecutive columns per thread)
    const int m = m_base + q * 32 + lane;
    const int m_limit = row0 + rows, n_limit = col0 + cols;
    const bool row_ok = m < m_limit;  // TMEM loads below are warp-collective: only the global accesses are predicated
    float* crow = c + static_cast<size_t>(row_ok ? m : 0) * n;
    const int j0 = n_base + half * COLS;
#pragma unroll
    for (int g16 = 0; g16 < COLS / 16; ++g16) {
      float cv[16];
      if constexpr (COMP) tc_ld16(tcomp + g16 * 16, cv);
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) {
        const int g = g16 * 4 + gg;
        const int j = j0 + g * 4;
        const bool vec = row_ok && j + 4 <= n_limit;
        float out[4];
        if (vec) {
          const float4 x = *reinterpret_cast<const float4*>(crow + j);
          out[0] = x.x; out[1] = x.y; out[2] = x.z; out[3] = x.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) out[e] = (row_ok && j + e < n_limit) ? crow[j + e] : 0.f;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if constexpr (COMP) out[e] = fold_comp(out[e], master[g * 4 + e], cv[gg * 4 + e]);
          else out[e] = __fadd_rn(out[e], master[g * 4 + e]);
        }
        if (vec) {
          *reinterpret_cast<float4*>(crow + j) = make_float4(out[0], out[1], out[2], out[3]);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (row_ok && j + e < n_limit) crow[j + e] = out[e];
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(S::TMEM_COLS) : "memory");
  }
}

// x -> (x_hi, x_lo): x_hi = x rounded to TF32 (low 13 mantissa bits zero), x_lo = x - x_hi exactly.  Output is packed per row
// as groups of [16 hi | 16 lo] floats (one 128-byte swizzle row per 16 k); k >= n inside the last group is zero.
__global__ void __launch_bounds__(256) split_tf32_kernel(const float* __restrict__ src, float* __restrict__ packed, int n, int kp,
                                                         int row0, int nrows) {
  const int quads = kp / 8;  // float4 of source per padded row: (kp / 2) / 4
  const size_t total = static_cast<size_t>(nrows) * quads;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int row = row0 + static_cast<int>(i / quads), k = static_cast<int>(i % quads) * 4;
    const float4 x = k < n ? *reinterpret_cast<const float4*>(src + static_cast<size_t>(row) * n + k) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 h, l;
    unsigned u;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.x)); h.x = __uint_as_float(u); l.x = __fsub_rn(x.x, h.x);
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.y)); h.y = __uint_as_float(u); l.y = __fsub_rn(x.y, h.y);
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.z)); h.z = __uint_as_float(u); l.z = __fsub_rn(x.z, h.z);
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.w)); h.w = __uint_as_float(u); l.w = __fsub_rn(x.w, h.w);
    float* dst = packed + static_cast<size_t>(row) * kp + (k / 16) * 32 + (k % 16);
    *reinterpret_cast<float4*>(dst) = h;
    *reinterpret_cast<float4*>(dst + 16) = l;
  }
}

// ---------------------------------------------------------------------------------------------------------
// Stacked form (default).  The M = 128, N = 128 MMA shape runs at about 0.6 of the tensor pipe's rate (measured:
// 165-181 TFLOP/s effective for three N = 128 products against 230-297 for three N = 256 products), but a
// 128 x 256 output tile leaves no TMEM for double-buffered chunks plus compensation terms.  So the OUTPUT tile
// stays 128 x 128 and the wide shape is obtained by stacking the two parts of b along N:
//     B_stack = [ b_hi rows j0..j0+127 ; b_lo rows j0..j0+127 ]            (256 x K, one TMA box)
//     MMA 1:  a_hi x B_stack^T  (N = 256)  ->  D[:, 0:128] += a_hi b_hi,   D[:, 128:256] += a_hi b_lo
//     MMA 2:  a_lo x b_hi^T     (N = 128)  ->  D[:, 128:256] += a_lo b_hi
// Two instructions per 8 k instead of three, two thirds of the work in the fast shape.  The leading products and
// the corrections (2^-11 of them) sit in separate TMEM columns and meet in the drain with one round-to-nearest
// addition.  TMEM: two chunk buffers of 256 columns; the compensation terms of the masters live in registers
// (64 masters + 64 error terms per drain thread).
// Operand layout in the scratch buffer (split_planes_kernel): a as two planes [row][kq] (hi, lo), kq = n rounded
// up to 32; b as 128-row blocks relative to the launch's first column, each block = 128 hi rows then 128 lo rows.
// Stage = 32 k: a_hi 16 KB + a_lo 16 KB + B_stack 32 KB = 64 KB, 3 stages.
// ---------------------------------------------------------------------------------------------------------
constexpr int TS_BK = 32;
constexpr int TS_A_BYTES = TC_BM * TS_BK * 4;             // 16 KB: 128 rows x one 128-byte swizzle row
constexpr int TS_B_BYTES = 2 * 128 * TS_BK * 4;           // 32 KB
constexpr int TS_STAGE_BYTES = 2 * TS_A_BYTES + TS_B_BYTES;
constexpr int TS_STAGES = 3;
constexpr int TS_SMEM_BYTES = TS_STAGES * TS_STAGE_BYTES + 1024 + 256;
// 12 warps = 3 warpgroups: {TMA, MMA, TMEM allocator, idle} give registers away (setmaxnreg.dec 40) so that the two drain
// warpgroups can hold 64 masters + 64 error terms + a double-buffered TMEM read per thread (setmaxnreg.inc 232):
// 128 * 40 + 256 * 232 = 384 * 168 = 64512 registers
constexpr int TS_THREADS = 384;

template <int CHUNK_STAGES>
__global__ void __launch_bounds__(TS_THREADS, 1)
matmul_3xtf32s_kernel(float* __restrict__ c, const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                      const __grid_constant__ CUtensorMap map_b, int n, int row0, int rows, int col0, int cols, int debug_noload,
                      int group, const int* __restrict__ run_if) {
  // guarded launch (see split_planes_kernel): run_if[4] is the form the auto kernel before this launch recorded; non-zero = the INT8
  // tensor cores took the product.  The guard acts through DATA, not control flow: a skipped launch runs the kernel's skeleton with
  // zero k stages and zero live rows (no loads, no MMAs, no stores of c).  An early `return` here -- any, even on a constant
  // parameter -- changed ptxas' allocation around the setmaxnreg regions: 368 bytes of spills and a quarter of the speed
  // (0.68 -> 0.88 ms at N = 4096).
  const bool skip = run_if != nullptr && run_if[4] != 0;
  constexpr int STAGES = TS_STAGES;
  constexpr int BUF_COLS = 256;  // TMEM columns per chunk buffer: 128 leading sums + 128 correction sums
  extern __shared__ unsigned char smem_raw[];
  const unsigned raw = smem_u32(smem_raw);
  const unsigned base = (raw + 1023u) & ~1023u;
  const unsigned bars = base + STAGES * TS_STAGE_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull_bar = [&](int b) { return bars + 8u * (2 * STAGES + b); };
  auto tempty_bar = [&](int b) { return bars + 8u * (2 * STAGES + 2 + b); };
  const unsigned tmem_slot = bars + 8u * (2 * STAGES + 4);
  volatile unsigned* tmem_slot_ptr = reinterpret_cast<volatile unsigned*>(smem_raw + (tmem_slot - raw));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int bx, by;
  raster_tile(group, bx, by);
  const int m_base = row0 + by * TC_BM, n_base = col0 + bx * 128;
  const int k_stages = skip ? 0 : (n + TS_BK - 1) / TS_BK;
  const int n_chunks = (k_stages + CHUNK_STAGES - 1) / CHUNK_STAGES;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 8 * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2 && !skip) {  // a skipped launch touches no tensor memory
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tmem_slot), "n"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem_base = *tmem_slot_ptr;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n");
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < k_stages; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(empty_bar(s), ((kb / STAGES) & 1) ^ 1);
        const unsigned st = base + s * TS_STAGE_BYTES;
        if (debug_noload) {
          mbar_arrive(full_bar(s));
          continue;
        }
        mbar_expect_tx(full_bar(s), TS_STAGE_BYTES);
        tma_load_2d(st, &map_ahi, kb * TS_BK, m_base, full_bar(s));
        tma_load_2d(st + TS_A_BYTES, &map_alo, kb * TS_BK, m_base, full_bar(s));
        tma_load_2d(st + 2 * TS_A_BYTES, &map_b, kb * TS_BK, bx * 256, full_bar(s));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr unsigned idesc_wide = idesc_tf32<256>(), idesc_half = idesc_tf32<128>();
      for (int kb = 0; kb < k_stages; ++kb) {
        const int s = kb % STAGES;
        const int chunk = kb / CHUNK_STAGES, in_chunk = kb % CHUNK_STAGES, buf = chunk & 1;
        if (in_chunk == 0) {
          mbar_wait(tempty_bar(buf), ((chunk >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        mbar_wait(full_bar(s), (kb / STAGES) & 1);
        tc_fence_after();
        const unsigned st = base + s * TS_STAGE_BYTES;
        const unsigned long long a_hi = umma_desc_sw128(st), a_lo = umma_desc_sw128(st + TS_A_BYTES);
        const unsigned long long b_st = umma_desc_sw128(st + 2 * TS_A_BYTES);  // rows 0..127 hi, 128..255 lo
        const unsigned d = tmem_base + buf * BUF_COLS;
#pragma unroll
        for (int k = 0; k < TS_BK / 8; ++k) {
          const unsigned long long adv = 2ull * k;  // 32 bytes along K inside the swizzle row
          tc_mma_tf32(d, a_hi + adv, b_st + adv, idesc_wide, (in_chunk | k) != 0);  // [a_hi b_hi | a_hi b_lo]
          tc_mma_tf32(d + 128, a_lo + adv, b_st + adv, idesc_half, 1);              // += a_lo b_hi
        }
        tc_commit(empty_bar(s));
        if (in_chunk == CHUNK_STAGES - 1 || kb == k_stages - 1) tc_commit(tfull_bar(buf));
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n");
    const int q = warp % 4, half = (warp - 4) / 4;
    constexpr int COLS = 64;  // outputs per drain thread
    unsigned long long master2[COLS / 2], comp2[COLS / 2];
#pragma unroll
    for (int i = 0; i < COLS / 2; ++i) master2[i] = comp2[i] = 0ull;
    for (int chunk = 0; chunk < n_chunks; ++chunk) {
      const int buf = chunk & 1;
      mbar_wait(tfull_bar(buf), (chunk >> 1) & 1);
      tc_fence_after();
      const unsigned t = tmem_base + (static_cast<unsigned>(q * 32) << 16) + buf * BUF_COLS + half * COLS;
      // TMEM reads are double-buffered: group g + 1 is in flight while group g is folded into the masters
      unsigned v[2][8], w[2][8];
      tc_ld8_issue(t, v[0]);        // leading products
      tc_ld8_issue(t + 128, w[0]);  // corrections
#pragma unroll
      for (int g = 0; g < COLS / 8; ++g) {
        tc_ld_wait();
        if (g + 1 < COLS / 8) {
          tc_ld8_issue(t + (g + 1) * 8, v[(g + 1) & 1]);
          tc_ld8_issue(t + 128 + (g + 1) * 8, w[(g + 1) & 1]);
        } else {  // the whole chunk buffer is in registers: hand it back before the arithmetic
          tc_fence_before();
          mbar_arrive(tempty_bar(buf));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const unsigned long long x = add2(pack2(v[g & 1][2 * i], v[g & 1][2 * i + 1]), pack2(w[g & 1][2 * i], w[g & 1][2 * i + 1]));
          // Knuth TwoSum on two outputs at once: m + x = sum + e exactly
          const unsigned long long m = master2[g * 4 + i];
          const unsigned long long sum = add2(m, x), bb = sub2(sum, m);
          const unsigned long long e = add2(sub2(m, sub2(sum, bb)), sub2(x, bb));
          master2[g * 4 + i] = sum;
          comp2[g * 4 + i] = add2(comp2[g * 4 + i], e);
        }
      }
    }
    // epilogue: c += master + comp, rounded once (row = TMEM lane, 64 consecutive columns per thread)
    if (!skip) {
    const int m = m_base + q * 32 + lane;
    const int m_limit = skip ? 0 : row0 + rows, n_limit = col0 + cols;
    const bool row_ok = m < m_limit;
    float* crow = c + static_cast<size_t>(row_ok ? m : 0) * n;
    const int j0 = n_base + half * COLS;
#pragma unroll
    for (int g = 0; g < COLS / 4; ++g) {
      const int j = j0 + g * 4;
      const bool vec = row_ok && j + 4 <= n_limit;
      float out[4];
      if (vec) {
        const float4 x = *reinterpret_cast<const float4*>(crow + j);
        out[0] = x.x; out[1] = x.y; out[2] = x.z; out[3] = x.w;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) out[e] = (row_ok && j + e < n_limit) ? crow[j + e] : 0.f;
      }
#pragma unroll
      for (int p2 = 0; p2 < 2; ++p2) {
        unsigned mlo, mhi, clo, chi;
        unpack2(master2[g * 2 + p2], mlo, mhi);
        unpack2(comp2[g * 2 + p2], clo, chi);
        out[2 * p2] = fold_comp(out[2 * p2], __uint_as_float(mlo), __uint_as_float(clo));
        out[2 * p2 + 1] = fold_comp(out[2 * p2 + 1], __uint_as_float(mhi), __uint_as_float(chi));
      }
      if (vec) {
        *reinterpret_cast<float4*>(crow + j) = make_float4(out[0], out[1], out[2], out[3]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (row_ok && j + e < n_limit) crow[j + e] = out[e];
      }
    }
    }  // !skip
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2 && !skip) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(512) : "memory");
  }
}

// x -> planes.  Source rows [src_row0, src_row0 + nrows) (nrows_pad >= nrows rows are written; the excess is zero).
// Destination row of source row r (relative index i = r - src_row0):
//   stacked == 0:  hi plane row (dst_row0 + i), lo plane = hi + lo_offset floats            (operand a)
//   stacked == 1:  row (i / 128) * 256 + i % 128 is hi, + 128 is lo                        (operand b, blocks of 128)
// kq floats per destination row; k >= n is zero.
__global__ void __launch_bounds__(256) split_planes_kernel(const float* __restrict__ src, float* __restrict__ dst, size_t lo_offset, int n,
                                                           int kq, int src_row0, int nrows, int nrows_pad, int dst_row0, int stacked,
                                                           const int* __restrict__ run_if) {
  // guarded launch (FP32 auto mode): the INT8 tensor-core launch before this one took the product -- run_if[4] is the form it
  // recorded (matmul_ozaki_auto_kernel), 0 = none was error-free
  if (run_if != nullptr && run_if[4] != 0) return;
  const int quads = kq / 4;
  const size_t total = static_cast<size_t>(nrows_pad) * quads;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int i = static_cast<int>(idx / quads), k = static_cast<int>(idx % quads) * 4;
    const float4 x = (i < nrows && k < n) ? *reinterpret_cast<const float4*>(src + static_cast<size_t>(src_row0 + i) * n + k)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 h, l;
    unsigned u;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.x)); h.x = __uint_as_float(u); l.x = __fsub_rn(x.x, h.x);
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.y)); h.y = __uint_as_float(u); l.y = __fsub_rn(x.y, h.y);
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.z)); h.z = __uint_as_float(u); l.z = __fsub_rn(x.z, h.z);
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.w)); h.w = __uint_as_float(u); l.w = __fsub_rn(x.w, h.w);
    const size_t hi_row = stacked ? static_cast<size_t>(i / 128) * 256 + i % 128 : static_cast<size_t>(dst_row0 + i);
    float* dh = dst + hi_row * kq + k;
    float* dl = stacked ? dh + static_cast<size_t>(128) * kq : dh + lo_offset;
    *reinterpret_cast<float4*>(dh) = h;
    *reinterpret_cast<float4*>(dl) = l;
  }
}

// n rows of kp packed floats; box = one stage (32 floats = 128 bytes) x box_rows rows; 128-byte swizzle
bool make_map(CUtensorMap* map, const float* ptr, int n, int kp, int box_rows) {
  EncodeTiledFn enc = encode_tiled();
  if (enc == nullptr) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kp), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kp) * 4};
  const cuuint32_t box[2] = {2 * TC_BK, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t elem[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// `rows` rows of kq floats; box = 32 floats (128 bytes) x box_rows rows; 128-byte swizzle
bool make_plane_map(CUtensorMap* map, const float* ptr, size_t rows, int kq, int box_rows) {
  EncodeTiledFn enc = encode_tiled();
  if (enc == nullptr) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kq), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kq) * 4};
  const cuuint32_t box[2] = {TS_BK, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t elem[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline int plane_row(int n) { return (n + TS_BK - 1) / TS_BK * TS_BK; }
inline size_t stacked_rows(int cols) { return static_cast<size_t>((cols + 127) / 128) * 256; }

inline int packed_row(int n) { return (n + TC_BK - 1) / TC_BK * 2 * TC_BK; }

int env_int(const char* name, int fallback) {
  const char* e = getenv(name);
  return e ? atoi(e) : fallback;
}

template <int BN, int CS, bool COMP>
cudaError_t tc_configure() {
  static PerDeviceOnce once;  // function attributes are per device
  bool& configured = once.here();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(matmul_3xtf32_kernel<BN, CS, COMP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         TcShape<BN>::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  return cudaSuccess;
}

template <int BN, int CS, bool COMP>
cudaError_t tc_go(cudaStream_t stream, float* c, const float* pa, const float* pb, int n, int row0, int rows, int col0, int cols) {
  using S = TcShape<BN>;
  if (cudaError_t e = tc_configure<BN, CS, COMP>(); e != cudaSuccess) return e;
  const int kp = packed_row(n);
  CUtensorMap map_a, map_b;
  if (!make_map(&map_a, pa, n, kp, TC_BM) || !make_map(&map_b, pb, n, kp, BN)) return cudaErrorNotSupported;
  static const int noload = env_int("MMX_TC_NOLOAD", 0);
  dim3 grid((cols + BN - 1) / BN, (rows + TC_BM - 1) / TC_BM);
  matmul_3xtf32_kernel<BN, CS, COMP><<<grid, TC_THREADS, S::SMEM_BYTES, stream>>>(c, map_a, map_b, n, row0, rows, col0, cols, noload,
                                                                                  raster_group(TC_BM, static_cast<size_t>(kp) * sizeof(float)));
  return cudaGetLastError();
}

template <int CS>
cudaError_t ts_configure() {
  static PerDeviceOnce once;
  bool& configured = once.here();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(matmul_3xtf32s_kernel<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, TS_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  return cudaSuccess;
}

// split + contraction in the stacked form
template <int CS>
cudaError_t ts_go(cudaStream_t stream, float* c, const float* a, const float* bt, float* scratch, int n, int row0, int rows, int col0,
                  int cols, bool reuse_a, const int* run_if) {
  if (cudaError_t e = ts_configure<CS>(); e != cudaSuccess) return e;
  const int kq = plane_row(n);
  float* pa = scratch;                                      // [2][n][kq]
  const size_t a_plane = static_cast<size_t>(n) * kq;
  float* pb = scratch + 2 * a_plane;                        // [blocks][256][kq], relative to col0
  auto blocks_for = [](size_t total) { return static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 16)); };
  if (!reuse_a)  // the row-sharded run contracts the same rows of a against one column block after another
    split_planes_kernel<<<blocks_for(static_cast<size_t>(rows) * (kq / 4)), 256, 0, stream>>>(a, pa, a_plane, n, kq, row0, rows, rows, row0, 0, run_if);
  const int cols_pad = (cols + 127) / 128 * 128;
  split_planes_kernel<<<blocks_for(static_cast<size_t>(cols_pad) * (kq / 4)), 256, 0, stream>>>(bt, pb, 0, n, kq, col0, cols, cols_pad, 0, 1, run_if);
  CUtensorMap map_ahi, map_alo, map_b;
  if (!make_plane_map(&map_ahi, pa, static_cast<size_t>(n), kq, TC_BM) || !make_plane_map(&map_alo, pa + a_plane, static_cast<size_t>(n), kq, TC_BM) ||
      !make_plane_map(&map_b, pb, stacked_rows(cols), kq, 256))
    return cudaErrorNotSupported;
  static const int noload = env_int("MMX_TC_NOLOAD", 0);
  dim3 grid((cols + 127) / 128, (rows + TC_BM - 1) / TC_BM);
  matmul_3xtf32s_kernel<CS><<<grid, TS_THREADS, TS_SMEM_BYTES, stream>>>(c, map_ahi, map_alo, map_b, n, row0, rows, col0, cols, noload,
                                                                        raster_group(TC_BM, static_cast<size_t>(kq) * sizeof(float)), run_if);
  return cudaGetLastError();
}

}  // namespace

bool matmul_3xtf32_usable(int n) { return n % 4 == 0 && encode_tiled() != nullptr; }

// everything that is not a stream operation, done once outside any stream capture
cudaError_t matmul_3xtf32_prepare() {
  if (encode_tiled() == nullptr) return cudaErrorNotSupported;
  if (cudaError_t e = tc_configure<128, 4, true>(); e != cudaSuccess) return e;
  if (cudaError_t e = ts_configure<2>(); e != cudaSuccess) return e;
  return tc_configure<256, 4, false>();
}

size_t matmul_3xtf32_scratch_bytes(int n) {
  const size_t packed = static_cast<size_t>(2) * n * packed_row(n);                                        // [16 hi | 16 lo] rows of a and bt
  const size_t planes = (static_cast<size_t>(2) * n + stacked_rows(n)) * plane_row(n);                     // stacked form
  return std::max(packed, planes) * sizeof(float);
}

cudaError_t launch_matmul_3xtf32(float* c, const float* a, const float* bt, void* scratch, int n, int row0, int rows, int col0,
                                 int cols, bool wide, cudaStream_t stream, bool reuse_a, const int* run_if) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (scratch == nullptr || n % 4 != 0) return cudaErrorInvalidValue;
  // tuning hook (tools/tc_probe.py): 14800 + chunk stages = stacked form (32 k per stage); BN * 100 + chunk stages (16 k per
  // stage), +1000 = compensated masters, = the one-part-per-MMA forms
  static const int mode_env = env_int("MMX_TC_MODE", 0);
  const int mode = mode_env ? mode_env : (wide ? 25604 : 14802);
  switch (mode) {
    case 14801: return ts_go<1>(stream, c, a, bt, static_cast<float*>(scratch), n, row0, rows, col0, cols, reuse_a, run_if);
    case 14802: return ts_go<2>(stream, c, a, bt, static_cast<float*>(scratch), n, row0, rows, col0, cols, reuse_a, run_if);
    case 14803: return ts_go<3>(stream, c, a, bt, static_cast<float*>(scratch), n, row0, rows, col0, cols, reuse_a, run_if);
    case 14804: return ts_go<4>(stream, c, a, bt, static_cast<float*>(scratch), n, row0, rows, col0, cols, reuse_a, run_if);
    case 14816: return ts_go<16>(stream, c, a, bt, static_cast<float*>(scratch), n, row0, rows, col0, cols, reuse_a, run_if);
    default: break;
  }
  if (run_if != nullptr) return cudaErrorInvalidValue;  // only the stacked form carries the guard
  const int kp = packed_row(n);
  float* pa = static_cast<float*>(scratch);
  float* pb = pa + static_cast<size_t>(n) * kp;
  // split only the rows this launch reads
  auto split = [&](const float* src, float* packed, int r0, int nr) {
    const size_t total = static_cast<size_t>(nr) * (kp / 8);
    const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 16));
    split_tf32_kernel<<<blocks, 256, 0, stream>>>(src, packed, n, kp, r0, nr);
  };
  split(a, pa, row0, rows);
  split(bt, pb, col0, cols);
  switch (mode) {
    case 25601: return tc_go<256, 1, false>(stream, c, pa, pb, n, row0, rows, col0, cols);
    case 25602: return tc_go<256, 2, false>(stream, c, pa, pb, n, row0, rows, col0, cols);
    case 25604: return tc_go<256, 4, false>(stream, c, pa, pb, n, row0, rows, col0, cols);
    case 25608: return tc_go<256, 8, false>(stream, c, pa, pb, n, row0, rows, col0, cols);
    case 25616: return tc_go<256, 16, false>(stream, c, pa, pb, n, row0, rows, col0, cols);
    case 12804: return tc_go<128, 4, false>(stream, c, pa, pb, n, row0, rows, col0, cols);
    case 13802: return tc_go<128, 2, true>(stream, c, pa, pb, n, row0, rows, col0, cols);
    case 13804: return tc_go<128, 4, true>(stream, c, pa, pb, n, row0, rows, col0, cols);
    case 13808: return tc_go<128, 8, true>(stream, c, pa, pb, n, row0, rows, col0, cols);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mmx
