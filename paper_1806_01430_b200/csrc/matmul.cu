// matmul.cu -- gene 8: c[i][j] += sum_k a[i][k] * bt[j][k]   (fixtures/matmul.c:25-28)
//
// "NT" GEMM: both operands are K-contiguous (that is why the program transposes b first).
// Compute-bound: 2*N^3 flop against 4*E*N^2 bytes of compulsory traffic.
//
// tcgen05/UMMA has no FP64 and no FP32-input kind, so at the reference's precision the dense
// contraction runs on the FP64 pipe (DFMA, or DMMA.8x8x4 through mma.sync -- the only shape
// sm_100a implements natively; m16n8k{4,8,16}.f64 lower to chains of it) or the FP32 FFMA pipe.
//
// Summation order.  Each c[i][j] is owned by one thread, initialised with the incoming c value
// and accumulated k ascending, so:
//   STRICT  (mul.rn then add.rn)  == the CPU loop bit for bit, any N, both dtypes;
//   FAST    (fma.rn, k ascending) == the CPU loop bit for bit whenever all partial sums are
//           exactly representable (FP64, N a power of two: SURVEY appendix A); otherwise it
//           differs only by the single rounding FMA saves per term.
// The DMMA variant keeps the same k-ascending FMA chain per element (the MMA accumulates its
// four products in order into the running sum), so it produces the same bits as FAST SIMT.
#include <cstdlib>
#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "raster.cuh"

namespace mmx {
namespace {

// ---------------------------------------------------------------------------------------------
// SIMT kernel: 128x128 CTA tile, BK = 16, 256 threads, 8x8 outputs per thread (2x2 groups of 4x4).
// Shared tiles are stored k-major ([k][m]) so the inner loop reads its 8 a's and 8 b's with
// 128-bit LDS that broadcast across the warp.
// ---------------------------------------------------------------------------------------------
constexpr int BM = 128, BN = 128, BK = 16;

template <typename T> struct V16;
template <> struct V16<double> { using type = double2; static constexpr int W = 2; };
template <> struct V16<float> { using type = float4; static constexpr int W = 4; };

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <typename T, bool STRICT>
__device__ __forceinline__ T mac(T acc, T x, T y) {
  if constexpr (STRICT) {
    if constexpr (sizeof(T) == 8) return __dadd_rn(acc, __dmul_rn(x, y));
    else return __fadd_rn(acc, __fmul_rn(x, y));
  } else {
    if constexpr (sizeof(T) == 8) return __fma_rn(x, y, acc);
    else return __fmaf_rn(x, y, acc);
  }
}

// Load 8 consecutive k of one row (row-major, K contiguous) into regs; zero outside [0,n).
template <typename T>
__device__ __forceinline__ void load_row8(T (&dst)[8], const T* __restrict__ base, int row, int row_limit, int k0,
                                          int n, bool vec_ok) {
  using VT = typename V16<T>::type;
  constexpr int W = V16<T>::W;
  if (row < row_limit && vec_ok && k0 + 8 <= n) {
    const VT* p = reinterpret_cast<const VT*>(base + static_cast<size_t>(row) * n + k0);
#pragma unroll
    for (int v = 0; v < 8 / W; ++v) {
      const VT x = p[v];
      if constexpr (W == 2) {
        dst[2 * v] = x.x;
        dst[2 * v + 1] = x.y;
      } else {
        dst[4 * v] = x.x;
        dst[4 * v + 1] = x.y;
        dst[4 * v + 2] = x.z;
        dst[4 * v + 3] = x.w;
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      dst[q] = (row < row_limit && k0 + q < n) ? base[static_cast<size_t>(row) * n + k0 + q] : static_cast<T>(0.0);
  }
}

template <typename T, bool STRICT>
__global__ void __launch_bounds__(256, 1)
matmul_simt_kernel(T* __restrict__ c, const T* __restrict__ a, const T* __restrict__ bt, int n, int row0, int rows,
                   int col0, int cols, bool vec_ok) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);  // [2][BK][BM]
  T* Bs = As + 2 * BK * BM;                // [2][BK][BN]

  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m_base = row0 + blockIdx.y * BM;  // first row of a / c of this CTA
  const int n_base = col0 + blockIdx.x * BN;  // first row of bt == first column of c
  const int m_limit = row0 + rows, n_limit = col0 + cols;

  // global -> smem staging role: one row, 8 consecutive k
  const int ld_row = tid % 128;
  const int ld_k = (tid / 128) * 8;

  T acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int m = m_base + (r / 4) * 64 + ty * 4 + (r % 4);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = n_base + (q / 4) * 64 + tx * 4 + (q % 4);
      acc[r][q] = (m < m_limit && j < n_limit) ? c[static_cast<size_t>(m) * n + j] : static_cast<T>(0.0);
    }
  }

  T ra[8], rb[8];
  load_row8(ra, a, m_base + ld_row, m_limit, ld_k, n, vec_ok);
  load_row8(rb, bt, n_base + ld_row, n_limit, ld_k, n, vec_ok);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    As[(ld_k + q) * BM + ld_row] = ra[q];
    Bs[(ld_k + q) * BN + ld_row] = rb[q];
  }
  __syncthreads();

  const int k_tiles = (n + BK - 1) / BK;
  for (int t = 0; t < k_tiles; ++t) {
    const int cur = t & 1;
    const bool more = t + 1 < k_tiles;
    if (more) {
      load_row8(ra, a, m_base + ld_row, m_limit, (t + 1) * BK + ld_k, n, vec_ok);
      load_row8(rb, bt, n_base + ld_row, n_limit, (t + 1) * BK + ld_k, n, vec_ok);
    }
    const T* Ac = As + cur * BK * BM;
    const T* Bc = Bs + cur * BK * BN;
    // STRICT must not add the zero-padded tail terms (x + 0*0 can flip a -0 accumulator)
    const int k_valid = STRICT ? min(BK, n - t * BK) : BK;
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      if (STRICT && k >= k_valid) break;
      T fa[8], fb[8];
      using VT = typename V16<T>::type;
      constexpr int W = V16<T>::W;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int v = 0; v < 4 / W; ++v) {
          const VT xa = *reinterpret_cast<const VT*>(Ac + k * BM + h * 64 + ty * 4 + v * W);
          const VT xb = *reinterpret_cast<const VT*>(Bc + k * BN + h * 64 + tx * 4 + v * W);
          if constexpr (W == 2) {
            fa[h * 4 + v * 2] = xa.x; fa[h * 4 + v * 2 + 1] = xa.y;
            fb[h * 4 + v * 2] = xb.x; fb[h * 4 + v * 2 + 1] = xb.y;
          } else {
            fa[h * 4] = xa.x; fa[h * 4 + 1] = xa.y; fa[h * 4 + 2] = xa.z; fa[h * 4 + 3] = xa.w;
            fb[h * 4] = xb.x; fb[h * 4 + 1] = xb.y; fb[h * 4 + 2] = xb.z; fb[h * 4 + 3] = xb.w;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[r][q] = mac<T, STRICT>(acc[r][q], fa[r], fb[q]);
    }
    if (more) {
      T* An = As + (cur ^ 1) * BK * BM;
      T* Bn = Bs + (cur ^ 1) * BK * BN;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        An[(ld_k + q) * BM + ld_row] = ra[q];
        Bn[(ld_k + q) * BN + ld_row] = rb[q];
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int m = m_base + (r / 4) * 64 + ty * 4 + (r % 4);
    if (m >= m_limit) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = n_base + h * 64 + tx * 4;
      T* dst = c + static_cast<size_t>(m) * n + j;
      if (vec_ok && j + 4 <= n_limit) {
        using VT = typename V16<T>::type;
        if constexpr (sizeof(T) == 8) {
          reinterpret_cast<VT*>(dst)[0] = make_double2(acc[r][h * 4], acc[r][h * 4 + 1]);
          reinterpret_cast<VT*>(dst)[1] = make_double2(acc[r][h * 4 + 2], acc[r][h * 4 + 3]);
        } else {
          reinterpret_cast<VT*>(dst)[0] = make_float4(acc[r][h * 4], acc[r][h * 4 + 1], acc[r][h * 4 + 2], acc[r][h * 4 + 3]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (j + q < n_limit) dst[q] = acc[r][h * 4 + q];
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// DMMA kernel (FP64, FAST only): mma.sync.m8n8k4.f64.  CTA tile 128x128, BK = 16, 8 warps as
// 2 (m) x 4 (n); warp tile 64x32 = 8x4 MMA tiles.  Operands go global -> smem with 16-byte
// cp.async in their native K-contiguous layout (no transposition: both fragments of
// DMMA.8x8x4 want "row r = lane/4, k = lane%4", which is exactly a K-contiguous read).  Rows are
// padded to BK+4 doubles (160 B) so the 8-row x 4-k fragment reads of a half-warp hit 32 distinct
// banks.  3-stage pipeline.
// ---------------------------------------------------------------------------------------------
constexpr int DTILE = 128;

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// DK = k per stage, DSTAGES = cp.async ring depth; WM x WN warps, each owning MT x NT MMA tiles
// (8x8 outputs each): CTA tile = (WM*MT*8) x (WN*NT*8).  The big configuration (2x4 warps of 64x32)
// serves large N; the 64x64 and 32x32 configurations exist so that small matrices (the fixture's
// N=256 is a 2x2 grid of 128-tiles) still spread over the 148 SMs.
// Requires n % 2 == 0 (16-byte aligned rows); rows/cols outside the matrix are zero-filled on
// load and masked on store.  k tail (n % DK) is zero-filled: adding +0 products is harmless in
// FAST mode except for the sign of an all-zero sum, which compares equal.
// min-blocks hint: the 4-warp tiles are built to run 3 CTAs per SM (one CTA's barrier or cp.async wait never idles
// the DMMA pipe); without the cap ptxas drifts to 170 registers and the third CTA no longer fits (measured: -2.5 %)
template <int DK, int DSTAGES, int WM, int WN, int MT, int NT>
__global__ void __launch_bounds__(32 * WM * WN, (WM * WN <= 4 && MT * NT <= 16) ? 3 : 1)
matmul_dmma_kernel(double* __restrict__ c, const double* __restrict__ a, const double* __restrict__ bt, int n,
                   int row0, int rows, int col0, int cols, int group, const int* __restrict__ run_if) {
  // guarded launch (FP64 auto mode): the tensor-core kernel took this contraction
  if (run_if != nullptr && run_if[4] != 0) return;  // run_if[4]: the form the auto kernel before this launch recorded; non-zero = it took the product
  constexpr int THREADS = 32 * WM * WN;
  constexpr int TM = WM * MT * 8, TN = WN * NT * 8;
  constexpr int DLD = DK + 4;  // padded row: (DK+4)*8 B = 32 mod 128 for DK in {16, 32} => conflict-free fragments
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);   // [DSTAGES][TM][DLD]
  double* Bs = As + DSTAGES * TM * DLD;               // [DSTAGES][TN][DLD]

  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  const int wm = warp / WN, wn = warp % WN;
  int bx, by;
  raster_tile(group, bx, by);
  const int m_base = row0 + by * TM, n_base = col0 + bx * TN;
  const int m_limit = row0 + rows, n_limit = col0 + cols;  // col0, cols even
  const int g = lane / 4, t4 = lane % 4;   // fragment row, fragment k

  // cp.async role: rows x DK/2 chunks of 16 B per operand
  constexpr int CPR = DK / 2;  // chunks per row
  auto issue_stage = [&](int stage, int k0) {
#pragma unroll
    for (int it = 0; it < TM * CPR / THREADS; ++it) {
      const int chunk = tid + it * THREADS;
      const int row = chunk / CPR, kc = (chunk % CPR) * 2;
      const int ar = m_base + row;
      const bool av = k0 + kc < n && ar < m_limit;
      cp_async16(As + (stage * TM + row) * DLD + kc, av ? a + static_cast<size_t>(ar) * n + k0 + kc : a, av);
    }
#pragma unroll
    for (int it = 0; it < TN * CPR / THREADS; ++it) {
      const int chunk = tid + it * THREADS;
      const int row = chunk / CPR, kc = (chunk % CPR) * 2;
      const int br = n_base + row;
      const bool bv = k0 + kc < n && br < n_limit;
      cp_async16(Bs + (stage * TN + row) * DLD + kc, bv ? bt + static_cast<size_t>(br) * n + k0 + kc : bt, bv);
    }
  };

  const int k_tiles = (n + DK - 1) / DK;
#pragma unroll
  for (int s = 0; s < DSTAGES - 1; ++s) {
    if (s < k_tiles) issue_stage(s, s * DK);
    cp_async_commit();
  }

  // accumulators seeded with the incoming c (loaded while the first stages are in flight)
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int m = m_base + (wm * MT + i) * 8 + g;
      const int col = n_base + (wn * NT + j) * 8 + t4 * 2;
      const bool ok = m < m_limit && col < n_limit;  // n_limit even => col+1 < n_limit too
      const double2 v = ok ? *reinterpret_cast<const double2*>(c + static_cast<size_t>(m) * n + col) : make_double2(0.0, 0.0);
      acc[i][j][0] = v.x;
      acc[i][j][1] = v.y;
    }

  for (int t = 0; t < k_tiles; ++t) {
    cp_async_wait<DSTAGES - 2>();
    __syncthreads();
    {
      const int nt = t + DSTAGES - 1;
      if (nt < k_tiles) issue_stage(nt % DSTAGES, nt * DK);
      cp_async_commit();
    }
    const double* Ac = As + ((t % DSTAGES) * TM + wm * MT * 8 + g) * DLD + t4;
    const double* Bc = Bs + ((t % DSTAGES) * TN + wn * NT * 8 + g) * DLD + t4;
#pragma unroll
    for (int kk = 0; kk < DK; kk += 4) {
      double fa[MT], fb[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) fa[i] = Ac[i * 8 * DLD + kk];
#pragma unroll
      for (int j = 0; j < NT; ++j) fb[j] = Bc[j * 8 * DLD + kk];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int m = m_base + (wm * MT + i) * 8 + g;
      const int col = n_base + (wn * NT + j) * 8 + t4 * 2;
      if (m < m_limit && col < n_limit)
        *reinterpret_cast<double2*>(c + static_cast<size_t>(m) * n + col) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

// ---------------------------------------------------------------------------------------------
// SIMT kernel v2 (FP32 FAST/STRICT, FP64 STRICT): same 128x128 CTA tile and 8x8 outputs per thread,
// but built to keep the FMA pipe's issue slots full:
//   * operands stay K-contiguous in shared memory ([row][k], row padded by 16 B) and arrive by
//     16-byte cp.async through a 4-stage ring: no register staging, no transposing stores;
//   * a thread owns rows ty+16r and columns tx+16q (interleaved), so the 128-bit fragment loads
//     along k are conflict-free;
//   * per k4 step (k2 for double) a thread issues 16 LDS.128 for 256 FFMA (94 % FMA density);
//   * FULL tiles take a path with no bounds checks at all.
// Each accumulator still sees k strictly ascending.
// ---------------------------------------------------------------------------------------------
// TM x TN CTA tile, (TM/8)*(TN/8) threads; a warp always spans 8 tx x 4 ty so that each HALF-warp (the
// unit a 128-bit LDS is split into) sees 2 distinct A rows and 8 distinct B rows.  Small CTAs (64x64 =
// two warps) are the default: 6-7 of them share an SM, so one CTA's barrier or cp.async wait never
// idles the FMA pipe -- the same effect that took the DMMA kernel from 29.5 to 33.6 TFLOP/s.
// min-blocks hint: cap FP32 at 128 registers (16 warps per SM whatever the CTA size); FP64 needs ~250
template <typename T, bool STRICT, bool FULL, int TM, int TN, int STAGES>
__global__ void __launch_bounds__((TM / 8) * (TN / 8), (sizeof(T) == 4 ? 512 : 256) / ((TM / 8) * (TN / 8)))
matmul_simt2_kernel(T* __restrict__ c, const T* __restrict__ a, const T* __restrict__ bt, int n, int row0, int rows,
                    int col0, int cols, int group) {
  using VT = typename V16<T>::type;
  constexpr int W = V16<T>::W;           // elements per 16-byte chunk
  constexpr int LD = BK + W;             // padded row length (elements): +16 bytes
  constexpr int CPR = BK / W;            // chunks per row
  constexpr int TX = TN / 8, TY = TM / 8, THREADS = TX * TY;
  static_assert(TX % 8 == 0 && TY % 4 == 0, "a warp spans 8 tx x 4 ty");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);   // [STAGES][TM][LD]
  T* Bs = As + STAGES * TM * LD;            // [STAGES][TN][LD]

  const int tid = threadIdx.x;
  const int lane = tid % 32, warp = tid / 32;
  constexpr int WX = TX / 8;                // warps along n
  const int tx = (warp % WX) * 8 + lane % 8, ty = (warp / WX) * 4 + lane / 8;
  int bx, by;
  raster_tile(group, bx, by);
  const int m_base = row0 + by * TM, n_base = col0 + bx * TN;
  const int m_limit = row0 + rows, n_limit = col0 + cols;

  auto issue_stage = [&](int stage, int k0) {
#pragma unroll
    for (int it = 0; it < TM * CPR / THREADS; ++it) {
      const int chunk = tid + it * THREADS;
      const int row = chunk / CPR, kc = (chunk % CPR) * W;
      const int ar = m_base + row;
      const bool av = FULL || (k0 + kc < n && ar < m_limit);  // n % W == 0: a chunk is all in or all out
      cp_async16(As + (stage * TM + row) * LD + kc, av ? a + static_cast<size_t>(ar) * n + k0 + kc : a, av);
    }
#pragma unroll
    for (int it = 0; it < TN * CPR / THREADS; ++it) {
      const int chunk = tid + it * THREADS;
      const int row = chunk / CPR, kc = (chunk % CPR) * W;
      const int br = n_base + row;
      const bool bv = FULL || (k0 + kc < n && br < n_limit);
      cp_async16(Bs + (stage * TN + row) * LD + kc, bv ? bt + static_cast<size_t>(br) * n + k0 + kc : bt, bv);
    }
  };

  const int k_tiles = (n + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < k_tiles) issue_stage(s, s * BK);
    cp_async_commit();
  }

  T acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int m = m_base + ty + TY * r, j = n_base + tx + TX * q;
      acc[r][q] = (FULL || (m < m_limit && j < n_limit)) ? c[static_cast<size_t>(m) * n + j] : static_cast<T>(0.0);
    }

  for (int t = 0; t < k_tiles; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nt = t + STAGES - 1;
      if (nt < k_tiles) issue_stage(nt % STAGES, nt * BK);
      cp_async_commit();
    }
    const T* Ac = As + ((t % STAGES) * TM + ty) * LD;
    const T* Bc = Bs + ((t % STAGES) * TN + tx) * LD;
    // STRICT must not add zero-padded tail terms (x + 0*0 can flip the sign of a -0 accumulator)
    const int k_valid = (STRICT && !FULL) ? min(BK, n - t * BK) : BK;
#pragma unroll
    for (int ks = 0; ks < BK; ks += W) {
      VT fa[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) fa[r] = *reinterpret_cast<const VT*>(Ac + TY * r * LD + ks);
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const VT fb0 = *reinterpret_cast<const VT*>(Bc + TX * q * LD + ks);
        const VT fb1 = *reinterpret_cast<const VT*>(Bc + TX * (q + 1) * LD + ks);
        const T* pa = reinterpret_cast<const T*>(fa);
        const T* pb0 = reinterpret_cast<const T*>(&fb0);
        const T* pb1 = reinterpret_cast<const T*>(&fb1);
#pragma unroll
        for (int kk = 0; kk < W; ++kk) {
          if ((STRICT && !FULL) && ks + kk >= k_valid) break;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            acc[r][q] = mac<T, STRICT>(acc[r][q], pa[r * W + kk], pb0[kk]);
            acc[r][q + 1] = mac<T, STRICT>(acc[r][q + 1], pa[r * W + kk], pb1[kk]);
          }
        }
      }
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int m = m_base + ty + TY * r, j = n_base + tx + TX * q;
      if (FULL || (m < m_limit && j < n_limit)) c[static_cast<size_t>(m) * n + j] = acc[r][q];
    }
}

template <typename T, bool STRICT, int TM, int TN, int STAGES>
cudaError_t simt2_go(T* c, const T* a, const T* bt, int n, int row0, int rows, int col0, int cols, cudaStream_t stream) {
  constexpr int W = V16<T>::W;
  constexpr int THREADS = (TM / 8) * (TN / 8);
  const size_t smem = static_cast<size_t>(STAGES) * (TM + TN) * (BK + W) * sizeof(T);
  static PerDeviceOnce once;  // function attributes are per device
  bool& configured = once.here();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(matmul_simt2_kernel<T, STRICT, true, TM, TN, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(matmul_simt2_kernel<T, STRICT, false, TM, TN, STAGES>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((cols + TN - 1) / TN, (rows + TM - 1) / TM);
  const bool full = cols % TN == 0 && rows % TM == 0 && n % BK == 0;
  const int group = raster_group(TM, static_cast<size_t>(n) * sizeof(T));
  if (full) matmul_simt2_kernel<T, STRICT, true, TM, TN, STAGES><<<grid, THREADS, smem, stream>>>(c, a, bt, n, row0, rows, col0, cols, group);
  else matmul_simt2_kernel<T, STRICT, false, TM, TN, STAGES><<<grid, THREADS, smem, stream>>>(c, a, bt, n, row0, rows, col0, cols, group);
  return cudaGetLastError();
}

template <typename T, bool STRICT>
cudaError_t simt_go(T* c, const T* a, const T* bt, int n, int row0, int rows, int col0, int cols, cudaStream_t stream) {
  const size_t smem = 2 * BK * (BM + BN) * sizeof(T);
  static PerDeviceOnce once;  // function attributes are per device
  bool& configured = once.here();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(matmul_simt_kernel<T, STRICT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((cols + BN - 1) / BN, (rows + BM - 1) / BM);
  const bool vec_ok = n % V16<T>::W == 0 && col0 % V16<T>::W == 0;
  matmul_simt_kernel<T, STRICT><<<grid, 256, smem, stream>>>(c, a, bt, n, row0, rows, col0, cols, vec_ok);
  return cudaGetLastError();
}

template <int DK, int DSTAGES, int WM, int WN, int MT, int NT>
cudaError_t dmma_go(double* c, const double* a, const double* bt, int n, int row0, int rows, int col0, int cols, cudaStream_t stream,
                    const int* run_if = nullptr) {
  constexpr int TM = WM * MT * 8, TN = WN * NT * 8;
  const size_t smem = static_cast<size_t>(DSTAGES) * (TM + TN) * (DK + 4) * sizeof(double);
  static PerDeviceOnce once;  // function attributes are per device
  bool& configured = once.here();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(matmul_dmma_kernel<DK, DSTAGES, WM, WN, MT, NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((cols + TN - 1) / TN, (rows + TM - 1) / TM);
  matmul_dmma_kernel<DK, DSTAGES, WM, WN, MT, NT><<<grid, 32 * WM * WN, smem, stream>>>(c, a, bt, n, row0, rows, col0, cols,
                                                                                         raster_group(TM, static_cast<size_t>(n) * sizeof(double)), run_if);
  return cudaGetLastError();
}

}  // namespace

bool fp32_int8_enabled(int n) {
  static const int on = [] { const char* e = getenv("MMX_F32_INT8"); return e ? atoi(e) : 1; }();
  return on != 0 && n >= kOzMinN && n % 4 == 0 && matmul_ozaki_usable(n) && matmul_3xtf32_usable(n);
}
size_t fp32_int8_scratch_offset(int n) { return (matmul_3xtf32_scratch_bytes(n) + 1023) / 1024 * 1024; }

int raster_group(int /*tile_m*/, size_t /*row_bytes*/) {
  static const int forced = [] { const char* e = getenv("MMX_RASTER_GROUP"); return e ? atoi(e) : 0; }();  // tuning hook
  // measured (tools/raster_sweep.sh, profiles/r1d_raster.txt): 16 tile-rows per group minimises DRAM traffic for both
  // the 64 x 64 DMMA tiles (296 resident CTAs) and the 128 x 128 tcgen05 tiles (148) at N = 4096 and 8192
  return forced > 0 ? forced : 16;
}


// ---- the fallback of auto mode as a conditional graph node (kernels.cuh: OzFallbackCond) ---------------------------------------------
namespace {
// Streams the conditional bodies are captured on: a small pool per device, filled outside captures (every capture is preceded by an
// un-captured warm-up pass through the same launch path), borrowed for the duration of one body capture.  Not thread_local: the
// batch evaluator's worker threads are short-lived, and a stream per thread would leak one per batch.
struct SidePool {
  std::mutex mu;
  std::vector<cudaStream_t> idle[64];
  int created[64] = {};
};
SidePool& side_pool() {
  static SidePool pool;
  return pool;
}
constexpr int kSideStreamsPerDevice = 8;  // concurrent captures on one device beyond this fall back to guarded launches

void side_pool_top_up() {
  int d = 0;
  cudaGetDevice(&d);
  SidePool& pool = side_pool();
  std::lock_guard<std::mutex> g(pool.mu);
  while (pool.created[d & 63] < kSideStreamsPerDevice) {
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
      (void)cudaGetLastError();
      return;
    }
    pool.idle[d & 63].push_back(s);
    ++pool.created[d & 63];
  }
}
cudaStream_t side_pool_borrow() {
  int d = 0;
  cudaGetDevice(&d);
  SidePool& pool = side_pool();
  std::lock_guard<std::mutex> g(pool.mu);
  auto& idle = pool.idle[d & 63];
  if (idle.empty()) return nullptr;
  cudaStream_t s = idle.back();
  idle.pop_back();
  return s;
}
void side_pool_return(cudaStream_t s) {
  if (s == nullptr) return;
  int d = 0;
  cudaGetDevice(&d);
  SidePool& pool = side_pool();
  std::lock_guard<std::mutex> g(pool.mu);
  pool.idle[d & 63].push_back(s);
}
}  // namespace

cudaError_t OzFallbackCond::begin(cudaStream_t stream) {
  active = false;
  side = nullptr;
  static const bool enabled = [] { const char* e = getenv("MMX_GRAPH_COND"); return e == nullptr || atoi(e) != 0; }();
  cudaStreamCaptureStatus status = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &status) != cudaSuccess) {
    (void)cudaGetLastError();
    return cudaSuccess;
  }
  if (status != cudaStreamCaptureStatusActive) {
    if (enabled) side_pool_top_up();  // outside a capture: make sure the pool exists before a capture needs it
    return cudaSuccess;
  }
  if (!enabled) return cudaSuccess;
  side = side_pool_borrow();
  if (side == nullptr) return cudaSuccess;  // no stream to capture the body on: guarded launches, as outside a capture
  unsigned long long id = 0;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaStreamGetCaptureInfo_v2(stream, &status, &id, &graph, &deps, &ndeps);
  if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&h, graph, 0, cudaGraphCondAssignDefault);
  if (e != cudaSuccess) {
    side_pool_return(side);
    side = nullptr;
    return e;
  }
  handle = h;
  active = true;
  return cudaSuccess;
}

void OzFallbackCond::abandon() {
  if (side != nullptr) side_pool_return(side);
  side = nullptr;
  active = false;
}

cudaError_t OzFallbackCond::body_begin(cudaStream_t stream) {
  if (!active) return cudaSuccess;
  cudaStreamCaptureStatus status;
  unsigned long long id = 0;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaError_t e = cudaStreamGetCaptureInfo_v2(stream, &status, &id, &graph, &deps, &ndeps);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = handle;
  p.conditional.type = cudaGraphCondTypeIf;
  p.conditional.size = 1;
  if (e == cudaSuccess) e = cudaGraphAddNode(&node, graph, deps, ndeps, &p);
  if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(side, p.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {  // the body was never opened: hand the stream back, the caller fails the capture
    side_pool_return(side);
    side = nullptr;
    active = false;
  }
  return e;
}

cudaError_t OzFallbackCond::body_end(cudaStream_t stream) {
  if (!active) return cudaSuccess;
  cudaGraph_t body = nullptr;
  cudaError_t e = cudaStreamEndCapture(side, &body);
  side_pool_return(side);
  side = nullptr;
  if (e != cudaSuccess) return e;
  return cudaStreamUpdateCaptureDependencies(stream, &node, 1, cudaStreamSetCaptureDependencies);
}

template <>
cudaError_t launch_matmul<double>(double* c, const double* a, const double* bt, int n, int row0, int rows, int col0, int cols,
                                  bool strict, int variant, void* scratch, cudaStream_t stream) {
  const bool reuse_a = (variant & (kReuseOperandA | kReuseOperands)) != 0;
  const bool reuse_bt = (variant & (kReuseOperandBt | kReuseOperands)) != 0;
  const bool c_zero = (variant & kCIsZero) != 0;
  variant &= ~(kReuseOperandA | kReuseOperandBt | kReuseOperands | kCIsZero);
  // tensor cores (INT8 slice products, matmul_ozaki.cu): on request
  if (!strict && scratch != nullptr && variant >= 40 && variant <= 45)  // 40 .. 45: 7 .. 2 slices
    return launch_matmul_ozaki(c, a, bt, scratch, n, row0, rows, col0, cols, 47 - variant, stream, nullptr, reuse_a);
  const bool dmma_ok = n % 2 == 0 && col0 % 2 == 0 && cols % 2 == 0;  // 16-byte aligned double2 accesses of c
  // auto: the INT8 tensor cores whenever their 8-bit digit slices reproduce every operand element exactly and every non-zero digit
  // pair is kept -- nothing of the product is dropped -- in the cheapest digit-pair form that does (ozaki_pick_form), else the FP64
  // pipe.  Forms with at most four levels (up to 2 x 3 / 3 x 2 digits: the application up to N = 8192) combine the level sums in a
  // 64-bit integer and round ONCE: the error-free product, bit-identical to the CPU program on the application's inputs.  Forms with
  // more levels combine them by a chain of FP64 fma steps (up to 73 significant bits do not fit one integer): faithfully rounded
  // (<= 1 ulp), and still exact whenever the result fits 53 bits -- as it does for the application at every N = 2^p (SURVEY
  // appendix A).  Both kernels are enqueued; a device guard written with the digit planes lets exactly one of them run.
  if (!strict && variant == 0 && scratch != nullptr && n >= kOzMinN && dmma_ok) {
    int* lossy = nullptr;
    OzFallbackCond cond;
    if (cudaError_t e = cond.begin(stream); e != cudaSuccess) return e;
    if (cudaError_t e = launch_matmul_ozaki(c, a, bt, scratch, n, row0, rows, col0, cols, 7, stream, &lossy, reuse_a, reuse_bt, c_zero, &cond); e != cudaSuccess) {
      cond.abandon();
      return e;
    }
    if (cudaError_t e = cond.body_begin(stream); e != cudaSuccess) return e;
    const cudaError_t ef = dmma_go<16, 3, 2, 2, 4, 4>(c, a, bt, n, row0, rows, col0, cols, cond.body_stream(stream), lossy);
    const cudaError_t ee = cond.body_end(stream);
    return ef != cudaSuccess ? ef : ee;
  }
  if (variant == 0) variant = 4;  // the FP64 pipe: DMMA, tile by size (best of the tuning points, profiles/)
  if (strict) {
    if (n % 2 == 0 && variant == 20) return simt2_go<double, true, 128, 128, 4>(c, a, bt, n, row0, rows, col0, cols, stream);
    if (n % 2 == 0 && variant != 1) return simt2_go<double, true, 64, 64, 3>(c, a, bt, n, row0, rows, col0, cols, stream);
    return simt_go<double, true>(c, a, bt, n, row0, rows, col0, cols, stream);
  }
  if (dmma_ok) {
    switch (variant) {
      case 2: return dmma_go<16, 3, 2, 4, 8, 4>(c, a, bt, n, row0, rows, col0, cols, stream);   // 128x128, BK=16 (first tuning point)
      case 5: return dmma_go<32, 3, 2, 2, 4, 4>(c, a, bt, n, row0, rows, col0, cols, stream);   // 64x64
      case 6: return dmma_go<32, 3, 2, 2, 2, 2>(c, a, bt, n, row0, rows, col0, cols, stream);   // 32x32
      case 7: return dmma_go<32, 3, 2, 4, 8, 4>(c, a, bt, n, row0, rows, col0, cols, stream);   // 128x128, BK=32
      case 8: return dmma_go<16, 3, 2, 2, 4, 4>(c, a, bt, n, row0, rows, col0, cols, stream);   // 64x64, BK=16
      case 9: return dmma_go<16, 4, 2, 2, 4, 4>(c, a, bt, n, row0, rows, col0, cols, stream);   // 64x64, BK=16, 4 stages
      case 10: return dmma_go<32, 2, 2, 2, 4, 4>(c, a, bt, n, row0, rows, col0, cols, stream);  // 64x64, BK=32, 2 stages
      case 11: return dmma_go<32, 3, 2, 2, 8, 4>(c, a, bt, n, row0, rows, col0, cols, stream);  // 128x64, 4 warps
      case 12: return dmma_go<32, 3, 1, 4, 8, 2>(c, a, bt, n, row0, rows, col0, cols, stream);  // 64x64 as 1x4 warps of 64x16
      case 13: return dmma_go<32, 3, 2, 2, 4, 8>(c, a, bt, n, row0, rows, col0, cols, stream);  // 64x128, 4 warps
      case 4:  // auto: the largest tile that still gives every SM work (N=256 would be a 2x2 grid of 128-tiles)
        if (n <= 1024) return dmma_go<32, 3, 2, 2, 2, 2>(c, a, bt, n, row0, rows, col0, cols, stream);
        return dmma_go<16, 3, 2, 2, 4, 4>(c, a, bt, n, row0, rows, col0, cols, stream);
      default: break;
    }
  }
  return simt_go<double, false>(c, a, bt, n, row0, rows, col0, cols, stream);
}

template <>
cudaError_t launch_matmul<float>(float* c, const float* a, const float* bt, int n, int row0, int rows, int col0, int cols,
                                 bool strict, int variant, void* scratch, cudaStream_t stream) {
  const bool reuse_a = (variant & (kReuseOperandA | kReuseOperands)) != 0;
  const bool reuse_bt = (variant & (kReuseOperandBt | kReuseOperands)) != 0;
  const bool c_zero = (variant & kCIsZero) != 0;
  variant &= ~(kReuseOperandA | kReuseOperandBt | kReuseOperands | kCIsZero);
  // auto, large matrices: the INT8 tensor cores exactly when their digit products are error-free for the operands at hand (one
  // rounding to float at the end: closer to the exact product than any FP32 accumulation), split TF32 otherwise -- the same
  // device-side guard as in FP64 (matmul_ozaki.cu); the split-TF32 launches read it and leave when the product has been taken
  if (!strict && scratch != nullptr && variant == 0 && fp32_int8_enabled(n)) {
    int* guard = nullptr;
    void* planes = static_cast<char*>(scratch) + fp32_int8_scratch_offset(n);
    OzFallbackCond cond;
    if (cudaError_t e = cond.begin(stream); e != cudaSuccess) return e;
    if (cudaError_t e = launch_matmul_ozaki_f32(c, a, bt, planes, n, row0, rows, col0, cols, stream, &guard, reuse_a, reuse_bt, c_zero, &cond); e != cudaSuccess) {
      cond.abandon();
      return e;
    }
    if (cudaError_t e = cond.body_begin(stream); e != cudaSuccess) return e;
    // (a fallback launch always re-splits its rows of a: the earlier column block may have gone the INT8 way)
    const cudaError_t ef = launch_matmul_3xtf32(c, a, bt, scratch, n, row0, rows, col0, cols, false, cond.body_stream(stream), false, guard);
    const cudaError_t ee = cond.body_end(stream);
    return ef != cudaSuccess ? ef : ee;
  }
  // tensor cores (split-precision TF32, matmul_tc.cu): large matrices by default, any n % 4 == 0 on request
  if (!strict && scratch != nullptr && n % 4 == 0 && (variant == 30 || variant == 31 || (variant == 0 && n >= kTcMinN)))
    return launch_matmul_3xtf32(c, a, bt, scratch, n, row0, rows, col0, cols, variant == 31, stream, reuse_a);
  // variant 1 keeps the first-generation kernel (k-major smem, register-staged) for A/B runs and
  // for n % 4 != 0, where rows are not 16-byte aligned
  if (variant != 1 && n % 4 == 0) {
    // FP32 is not barrier-bound (small CTAs measured 39.5-43.8 TFLOP/s against 45.6 for 128x128x4
    // stages): it is limited by register-bank dispatch stalls and LDS issue, so the big tile stays.
    // Small matrices still get the 64x64 tile so that N=256 is 16 CTAs, not 4.
    if (strict) {
      if (n <= 1024) return simt2_go<float, true, 64, 64, 4>(c, a, bt, n, row0, rows, col0, cols, stream);
      return simt2_go<float, true, 128, 128, 4>(c, a, bt, n, row0, rows, col0, cols, stream);
    }
    if (variant == 22 || (variant != 20 && n <= 1024)) return simt2_go<float, false, 64, 64, 4>(c, a, bt, n, row0, rows, col0, cols, stream);
    return simt2_go<float, false, 128, 128, 4>(c, a, bt, n, row0, rows, col0, cols, stream);
  }
  if (strict) return simt_go<float, true>(c, a, bt, n, row0, rows, col0, cols, stream);
  return simt_go<float, false>(c, a, bt, n, row0, rows, col0, cols, stream);
}

}  // namespace mmx
