// ozaki_digits.cuh -- the digit encoding of matmul_ozaki.cu as a device function, so that the kernels which PRODUCE an operand of
// gene 8 (the init-a fill, the transpose) can write its int8 digit planes while the values are still in registers, instead of a
// separate slice pass reading the operand back from HBM (the slice pass stays for operands that arrive any other way).
//
// Encoding (matmul_ozaki.cu header): row r of an operand is scaled by +-2^-e_r, e_r = ilogb(max_k |x_rk|) + 1, and cut into signed
// 8-bit digits d_1 .. d_S (-128 <= d_t <= 127: what an int8 holds), x = +-2^e (d_1 2^-7 + d_2 2^-15 + d_3 2^-23 + ...) + remainder,
// every step exact in FP64.  Digit t has the unit 2^-oz_unit(t - 1).
//  * Eight bits per digit need a lopsided rounding: the part left after a digit must lie in (-128.5 / 256, 127.5 / 256] of the digit's
//    unit RECURSIVELY, i.e. in (c - 1, c] with c = 127 / 255, or a later digit would have to be +128; so d = ceil(R - c) =
//    rint(R + 1 / 510) (R = what is left, in units of the digit; never a tie for finite binary R).  1 / 510 is not a binary fraction
//    and R + 1 / 510 is rounded: an R within 2^-46 of the boundary may get the other digit, which shows up as a digit outside
//    [-128, 127] one level down -- checked, and reported like bits below the last digit (the operand counts as cut and the product
//    goes to the FP64 pipe).
//  * The first digit reaches -128 but only +127.498: a row whose largest element is positive and above 127 / 128 of 2^e is encoded
//    NEGATED (two's-complement bytes reach -2^15 but only 2^15 - 129 when every byte is signed); when both ends of the row are that
//    large the exponent grows by one instead.  The row's exponent word carries the sign (oz_exp_pack); the contraction's epilogue
//    multiplies it back in.
// Plane t of row r lives at planes + t * plane + r * kq.  The guard words record whether any element has bits below its 7th digit
// (or is not finite) and the highest non-zero digit of each operand; the contraction kernel picks its form from them
// (ozaki_pick_form).
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace mmx {

constexpr int kOzNonFinite = 0x7fffffff;  // row exponent of a row that holds an Inf or a NaN: its products are NaN

#ifdef __CUDACC__

__device__ __forceinline__ double oz_pow2(int e) { return __longlong_as_double(static_cast<long long>(e + 1023) << 52); }

constexpr int kOzDigitBits = 8;  // bits per digit below the first (the level step of the contraction's Horner sum)
// digit t + 1 (t = 0, 1, ...) has the unit 2^-oz_unit(t): 7, 15, 23, ...
__host__ __device__ constexpr int oz_unit(int t) { return 7 + kOzDigitBits * t; }
constexpr int kOzPairUnit = 2 * (kOzDigitBits - 1);  // a product of two first digits has the unit 2^-14
constexpr double kOzRoundBias = 1.0 / 510.0;  // 1/2 - 127/255

// one digit off `rem` (scaled so that the digit's unit is 1 / up): returns it, leaves the rest in rem (exact); out_of_range: not an int8
__device__ __forceinline__ int oz_take_digit(double& rem, double up, double down, bool& out_of_range) {
  const double s = fma(rem, up, kOzRoundBias) + 6755399441055744.0;  // rint without the conversion units: + 1.5 * 2^52
  const int d = __double2loint(s);
  rem = fma(-(s - 6755399441055744.0), down, rem);  // exact: removes a prefix of rem's bits
  out_of_range = out_of_range || static_cast<unsigned>(d + 128) > 255u;
  return d;
}

// exponent of a row whose largest magnitude is m (bad: the row holds a non-finite value): |x| < 2^e for every element
__device__ __forceinline__ int oz_row_exponent(double m, bool bad) { return (m > 0.0 && !bad) ? ilogb(m) + 1 : 0; }

// 2^-e as the exact scale factor; 0 for rows that get zero digits (non-finite rows, and rows whose maximum is below 2^-970, where
// 1 / 2^e would overflow: both are flagged as lossy by the caller through `tiny` / `bad`)
__device__ __forceinline__ double oz_row_scale(int e, bool live, bool bad, bool* tiny) {
  *tiny = e < -970;
  if (!(live && !bad && !*tiny)) return 0.0;
  // 2^-e is a normal number for e <= 1022: two integer operations instead of scalbn's general path (the fused producers compute
  // this once per row AND thread)
  return e <= 1022 ? oz_pow2(-e) : scalbn(1.0, -e);
}

// The exponent word of a row: the exponent, and bit 30 flipped when the row is encoded negated (kOzNonFinite stays what it is)
__host__ __device__ __forceinline__ int oz_exp_pack(int e, bool neg) { return neg ? e ^ 0x40000000 : e; }
__host__ __device__ __forceinline__ bool oz_exp_unpack(int word, int& e) {
  const bool neg = word != kOzNonFinite && (((word >> 30) ^ (word >> 31)) & 1) != 0;
  e = neg ? word ^ 0x40000000 : word;
  return neg;
}
// Exponent and sign of a row from its largest and smallest element (signed; bad: the row holds a non-finite value).  *inv = the
// signed scale factor (0 for rows that get zero digits, *tiny as oz_row_scale).
__device__ __forceinline__ int oz_row_code(double hi, double lo, bool bad, bool live, double* inv, bool* tiny) {
  const double m = fmax(fabs(hi), fabs(lo));
  int e = oz_row_exponent(m, bad);
  double s = oz_row_scale(e, live, bad, tiny);
  bool neg = false;
  if (s != 0.0) {
    const bool hi_big = hi * s > 0.9921875, lo_big = -lo * s > 0.9921875;  // 127 / 128
    if (hi_big && lo_big) {
      e += 1;
      s = oz_row_scale(e, live, bad, tiny);
    } else if (hi_big) {
      neg = true;
    }
  }
  *inv = neg ? -s : s;
  return oz_exp_pack(e, neg);
}
// the signed scale factor of a row from its exponent word
__device__ __forceinline__ double oz_row_scale_of(int word, bool* tiny) {
  int e;
  const bool neg = oz_exp_unpack(word, e);
  const double s = oz_row_scale(e, true, false, tiny);
  return neg ? -s : s;
}

// The digits of W (2 or 4) consecutive elements v[0..W) of one row, starting at column k0 (a multiple of W), packed W to a store.
// `inv` = oz_row_scale of the row; `dirty` = guard[dirty_slot]: planes beyond it hold only zeros (auto mode keeps its scratch that
// way), so zero digits need not be written there -- short operands move 2 planes per element instead of S.  `lossy` / `top`
// accumulate per thread: anything below the last digit? highest non-zero digit (1-based) seen.
template <int S, int W>
__device__ __forceinline__ void oz_emit(const double (&v)[W], double inv, bool bad, int dirty, signed char* __restrict__ drow, size_t plane, int k0,
                                        int& lossy, int& top) {
  static_assert(W == 2 || W == 4, "digits are packed two or four to a store");
  int dig[S] = {};
  int levels = S;  // digit levels walked: the planes beyond hold zeros for these elements
  double rem[W];
#pragma unroll
  for (int q = 0; q < W; ++q) rem[q] = bad ? 0.0 : v[q] * inv;
#pragma unroll
  for (int t = 0; t < S; ++t) {
    // W elements per digit level, branch-free (a zero remainder yields a zero digit); one test per level ends the walk
    // once nothing is left -- short operands finish after a digit or two
    bool none = t >= 1;
#pragma unroll
    for (int q = 0; q < W; ++q) none = none && rem[q] == 0.0;
    if (none) {
      levels = t;
      break;
    }
    const double up = oz_pow2(oz_unit(t)), down = oz_pow2(-oz_unit(t));
    int word = 0;
    bool bad_digit = false;
#pragma unroll
    for (int q = 0; q < W; ++q) word |= (oz_take_digit(rem[q], up, down, bad_digit) & 0xff) << (8 * q);
    lossy |= bad_digit;
    dig[t] = word;
  }
  // bits below the last digit: the slices do not reproduce this element exactly
#pragma unroll
  for (int q = 0; q < W; ++q) lossy |= rem[q] != 0.0;
  const int planes_to_write = max(levels, dirty);  // beyond: zero digits into planes that hold only zeros
#pragma unroll
  for (int t = 0; t < S; ++t) {
    if (t >= planes_to_write) break;
    if (dig[t] != 0) top = max(top, t + 1);
    if (t < dirty || dig[t] != 0) {
      if constexpr (W == 4) *reinterpret_cast<int*>(drow + t * plane + k0) = dig[t];
      else *reinterpret_cast<unsigned short*>(drow + t * plane + k0) = static_cast<unsigned short>(dig[t]);
    }
  }
}

// The first two (oz_emit_first<W, L>: the first L) digit levels of W consecutive elements, straight-line: no early exits, both planes stored unconditionally, so that a
// caller that encodes several rows per thread gives the compiler ONE basic block of independent FP64 chains (the walk of oz_emit is
// a chain of dependent FP64 operations per element and level with a branch after each level; on B200 those are long-latency
// operations, and the producers that used oz_emit row by row spent half their issue slots waiting on them -- ncu, r2r_producers).
// (oz_first_two_words hands the two packed words back instead of storing them.)  Returns true when something is left below the second digit: the caller then runs oz_emit on the same elements (rare path; it
// rewrites the two planes with the same digits and continues).  top2: 0 / 1 / 2 = highest non-zero digit among the two.
template <int W, int L>
__device__ __forceinline__ bool oz_first_words(const double (&v)[W], double inv, int (&word)[L]) {
  static_assert(W == 2 || W == 4, "digits are packed two or four to a word");
  static_assert(L >= 1 && L <= 3, "digit levels of the straight-line pass");
  // All L digits at once: X = x * inv * 2^(8 L - 1) is an integer exactly when nothing is left below digit L, and the bytes of
  // X + 0x80..80 (offset binary, 0 .. 255 each) are the digits + 128 -- the same digits as the level-by-level walk of oz_emit gives
  // (digits in [-128, 127] to the base 256 are unique), for three FP64 operations per element instead of four per level.
  constexpr int kOffset = L == 1 ? 0x80 : L == 2 ? 0x8080 : 0x808080;
  const double scale = inv * oz_pow2(oz_unit(L - 1));
  int y[W];
  bool left = false;
#pragma unroll
  for (int q = 0; q < W; ++q) {
    const double r = v[q] * scale;                         // exact (a power of two)
    const double t = r + 6755399441055744.0;               // + 1.5 * 2^52: rint(r) sits in the low word
    left = left || (t - 6755399441055744.0) != r;          // not an integer: bits below digit L (or |r| beyond 2^51: not finite, huge)
    y[q] = __double2loint(t) + kOffset;
    left = left || static_cast<unsigned>(y[q]) >= (1u << (8 * L));  // beyond what L bytes hold (cannot happen for |x inv| in range)
  }
#pragma unroll
  for (int l = 0; l < L; ++l) {
    // byte L - 1 - l of every element, packed (PRMT: three instructions for four elements)
    const unsigned pick = static_cast<unsigned>(L - 1 - l) | (static_cast<unsigned>(4 + L - 1 - l) << 4);
    if constexpr (W == 4) {
      const unsigned lo = __byte_perm(static_cast<unsigned>(y[0]), static_cast<unsigned>(y[1]), pick);
      const unsigned hi = __byte_perm(static_cast<unsigned>(y[2]), static_cast<unsigned>(y[3]), pick);
      word[l] = static_cast<int>(__byte_perm(lo, hi, 0x5410) ^ 0x80808080u);
    } else {
      word[l] = static_cast<int>((__byte_perm(static_cast<unsigned>(y[0]), static_cast<unsigned>(y[1]), pick) & 0xffffu) ^ 0x8080u);
    }
  }
  return left;
}
// the same with the words stored: plane l of the row at drow + l * plane; top = highest non-zero level (1-based, 0: all zero)
template <int W, int L>
__device__ __forceinline__ bool oz_emit_first(const double (&v)[W], double inv, signed char* __restrict__ drow, size_t plane, int k0, int& top) {
  int word[L];
  const bool left = oz_first_words<W, L>(v, inv, word);
  top = 0;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    if constexpr (W == 4) *reinterpret_cast<int*>(drow + l * plane + k0) = word[l];
    else *reinterpret_cast<unsigned short*>(drow + l * plane + k0) = static_cast<unsigned short>(word[l]);
    if (word[l] != 0) top = l + 1;
  }
  return left;
}
template <int W>
__device__ __forceinline__ bool oz_first_two_words(const double (&v)[W], double inv, int& word0, int& word1) {
  int word[2];
  const bool left = oz_first_words<W, 2>(v, inv, word);
  word0 = word[0];
  word1 = word[1];
  return left;
}
template <int W>
__device__ __forceinline__ bool oz_emit_first_two(const double (&v)[W], double inv, signed char* __restrict__ drow, size_t plane, int k0, int& top2) {
  return oz_emit_first<W, 2>(v, inv, drow, plane, k0, top2);
}

// End of a CTA's work on an operand: fold the threads' lossy / top into the guard words (every thread of a 256-thread CTA calls).
// The words are read first: after a few CTAs nobody needs the atomic any more.
__device__ __forceinline__ void oz_guard_commit(int lossy, int top, int* __restrict__ guard, int lossy_slot, int top_slot, int dirty_slot) {
  __shared__ int oz_top_sh[8];
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  lossy = __syncthreads_or(lossy);
  top = __reduce_max_sync(0xffffffffu, top);
  if (tid % 32 == 0) oz_top_sh[tid / 32] = top;
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int w = 1; w < 8; ++w) top = max(top, oz_top_sh[w]);
    if (lossy && guard[lossy_slot] == 0) atomicOr(guard + lossy_slot, 1);
    if (top > guard[top_slot]) atomicMax(guard + top_slot, top);
    if (dirty_slot >= 0 && top > guard[dirty_slot]) atomicMax(guard + dirty_slot, top);
  }
}

#endif  // __CUDACC__

}  // namespace mmx
