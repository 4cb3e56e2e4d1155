// reduce.cu -- the reduction-style loops of fixtures/matmul.c:
//   gene 9  (:26)  for j: c[i][j] += dot(a[i][:], bt[j][:])   -- one GEMV against bt per launch
//   gene 10 (:27)  for k: c[i][j] += a[i][k] * bt[j][k]       -- one dot product per launch
//   gene 11 (:31)  for i: sum += c[i][i]                      -- the trace
//
// FAST: lanes stride over k with 128-bit loads, warp-shuffle tree, then c += partial.  Exact
// (hence bit-identical to the CPU loop) whenever the partial sums are exactly representable
// (FP64, N = 2^p); otherwise within the stated tolerance.
// STRICT: the data is staged through shared memory with coalesced loads, then ONE thread per
// output walks k ascending with a separate multiply and add, starting from the incoming c
// value -- the CPU loop's exact operation sequence.
#include <cstdlib>

#include "kernels.cuh"

namespace mmx {
namespace {

template <typename T> struct V16;
template <> struct V16<double> { using type = double2; static constexpr int W = 2; };
template <> struct V16<float> { using type = float4; static constexpr int W = 4; };

__device__ __forceinline__ double vdot(double2 x, double2 y, double acc) {
  acc = __fma_rn(x.x, y.x, acc);
  return __fma_rn(x.y, y.y, acc);
}
__device__ __forceinline__ float vdot(float4 x, float4 y, float acc) {
  acc = __fmaf_rn(x.x, y.x, acc);
  acc = __fmaf_rn(x.y, y.y, acc);
  acc = __fmaf_rn(x.z, y.z, acc);
  return __fmaf_rn(x.w, y.w, acc);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T strict_mac(T acc, T x, T y) {
  if constexpr (sizeof(T) == 8) return __dadd_rn(acc, __dmul_rn(x, y));
  else return __fadd_rn(acc, __fmul_rn(x, y));
}

// Partial dot of two K-contiguous rows over the lanes of one warp (FAST).
template <typename T>
__device__ __forceinline__ T warp_dot(const T* __restrict__ x, const T* __restrict__ y, int n, int lane, bool vec_ok) {
  using VT = typename V16<T>::type;
  constexpr int W = V16<T>::W;
  T acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  if (vec_ok) {
    const VT* xv = reinterpret_cast<const VT*>(x);
    const VT* yv = reinterpret_cast<const VT*>(y);
    const int nv = n / W;
    int v = lane;
    for (; v + 96 < nv; v += 128) {  // 4 independent 16-byte loads per operand in flight
      const VT x0 = xv[v], x1 = xv[v + 32], x2 = xv[v + 64], x3 = xv[v + 96];
      const VT y0 = yv[v], y1 = yv[v + 32], y2 = yv[v + 64], y3 = yv[v + 96];
      acc0 = vdot(x0, y0, acc0);
      acc1 = vdot(x1, y1, acc1);
      acc2 = vdot(x2, y2, acc2);
      acc3 = vdot(x3, y3, acc3);
    }
    for (; v < nv; v += 32) acc0 = vdot(xv[v], yv[v], acc0);
  } else {
    for (int k = lane; k < n; k += 32) acc0 += x[k] * y[k];
  }
  return warp_sum((acc0 + acc1) + (acc2 + acc3));
}

// ---- gene 9 ------------------------------------------------------------------------------------

// FAST: one warp per output column j; block = 256 threads = 8 columns.
template <typename T>
__global__ void __launch_bounds__(256) gemv_row_fast_kernel(T* __restrict__ c, const T* __restrict__ a,
                                                            const T* __restrict__ bt, int n, IterRef iter, bool vec_ok) {
  const int i = iter.off + (iter.base ? *iter.base : 0);
  const int lane = threadIdx.x % 32;
  const int j = blockIdx.x * 8 + threadIdx.x / 32;
  if (j >= n) return;
  const T s = warp_dot(a + static_cast<size_t>(i) * n, bt + static_cast<size_t>(j) * n, n, lane, vec_ok);
  if (lane == 0) c[static_cast<size_t>(i) * n + j] += s;
}

// FAST, row fits in shared memory and is 16-byte aligned: persistent CTAs (2 per SM), each owning a
// contiguous block of output columns j, so the work is balanced to within one row per CTA.
// a[i][:] is staged once per CTA in shared memory (it would otherwise be re-read from L1/L2 by
// every warp); all 8 warps stream each bt row together.  The first 8 vectors per thread of row j+1
// are already in flight while row j is reduced, so the per-row barrier never drains the memory
// pipeline; the only global traffic is bt itself (E*N^2 bytes).
constexpr int GEMV_VPT = 8;

template <typename T>
__global__ void __launch_bounds__(256, 2) gemv_row_staged_kernel(T* __restrict__ c, const T* __restrict__ a,
                                                                 const T* __restrict__ bt, int n, IterRef iter) {
  using VT = typename V16<T>::type;
  constexpr int W = V16<T>::W;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  VT* sa = reinterpret_cast<VT*>(smem_raw);  // n / W vectors
  __shared__ T partial[2][8];                // [buffer][warp]
  const int i = iter.off + (iter.base ? *iter.base : 0);
  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  const int nv = n / W;
  const VT* av = reinterpret_cast<const VT*>(a + static_cast<size_t>(i) * n);
  for (int v = tid; v < nv; v += 256) sa[v] = av[v];

  const int j0 = static_cast<int>(static_cast<long long>(n) * blockIdx.x / gridDim.x);
  const int j1 = static_cast<int>(static_cast<long long>(n) * (blockIdx.x + 1) / gridDim.x);

  auto prefetch = [&](VT (&dst)[GEMV_VPT], int j) {
    const VT* r = reinterpret_cast<const VT*>(bt + static_cast<size_t>(j) * n);
#pragma unroll
    for (int q = 0; q < GEMV_VPT; ++q) {
      const int v = tid + q * 256;
      if (v < nv) dst[q] = r[v];
    }
  };
  auto reduce_row = [&](const VT (&row)[GEMV_VPT], int j, int buf) {
    T s0 = 0, s1 = 0;
#pragma unroll
    for (int q = 0; q < GEMV_VPT; q += 2) {
      const int v = tid + q * 256;
      if (v < nv) s0 = vdot(sa[v], row[q], s0);
      if (v + 256 < nv) s1 = vdot(sa[v + 256], row[q + 1], s1);
    }
    const VT* r = reinterpret_cast<const VT*>(bt + static_cast<size_t>(j) * n);
    for (int v = tid + GEMV_VPT * 256; v < nv; v += 256) s0 = vdot(sa[v], r[v], s0);  // rows longer than 2048 vectors
    s0 = warp_sum(s0 + s1);
    if (lane == 0) partial[buf][warp] = s0;
    __syncthreads();  // one barrier per row; the partial buffers alternate
    if (tid == 0) {
      T tot = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) tot += partial[buf][w];
      c[static_cast<size_t>(i) * n + j] += tot;
    }
  };

  VT even[GEMV_VPT], odd[GEMV_VPT];
  if (j0 < j1) prefetch(even, j0);
  __syncthreads();  // sa is complete
  for (int j = j0; j < j1; j += 2) {
    if (j + 1 < j1) prefetch(odd, j + 1);
    reduce_row(even, j, 0);
    if (j + 1 < j1) {
      if (j + 2 < j1) prefetch(even, j + 2);
      reduce_row(odd, j + 1, 1);
    }
  }
}

// FAST, streaming form: every WARP owns whole rows of bt (j = warp, warp + #warps, ...) and there is no
// CTA-wide barrier after the a-row has been staged.  A lane keeps GEMV_Q 16-byte loads of bt in flight
// (L1 bypassed: the matrix is read once), multiplies them against the staged a-row from shared memory
// (consecutive lanes, consecutive 16-byte chunks: conflict-free), and a shuffle tree finishes the row.
// The grid is sized so that every warp gets the same number of rows when N is a power of two.
constexpr int GEMV_Q = 8;

template <typename VT>
__device__ __forceinline__ VT ld_stream(const VT* p) {
  VT v;
  if constexpr (sizeof(VT) == 16 && alignof(VT) == 16) {
    unsigned x, y, z, w;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];\n" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "l"(p));
    const uint4 u = make_uint4(x, y, z, w);
    v = *reinterpret_cast<const VT*>(&u);
  }
  return v;
}

template <typename T>
__global__ void __launch_bounds__(256, 2) gemv_row_stream_kernel(T* __restrict__ c, const T* __restrict__ a,
                                                                 const T* __restrict__ bt, int n, IterRef iter) {
  using VT = typename V16<T>::type;
  constexpr int W = V16<T>::W;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  VT* sa = reinterpret_cast<VT*>(smem_raw);  // n / W vectors
  const int i = iter.off + (iter.base ? *iter.base : 0);
  const int tid = threadIdx.x, lane = tid % 32;
  const int nv = n / W;
  const VT* av = reinterpret_cast<const VT*>(a + static_cast<size_t>(i) * n);
  for (int v = tid; v < nv; v += 256) sa[v] = av[v];
  __syncthreads();

  const int warps = gridDim.x * 8;
  T* crow = c + static_cast<size_t>(i) * n;
  for (int j = blockIdx.x * 8 + tid / 32; j < n; j += warps) {
    const VT* r = reinterpret_cast<const VT*>(bt + static_cast<size_t>(j) * n);
    T s0 = 0, s1 = 0;
    int v = lane;
    for (; v + 32 * (GEMV_Q - 1) < nv; v += 32 * GEMV_Q) {
      VT x[GEMV_Q];
#pragma unroll
      for (int q = 0; q < GEMV_Q; ++q) x[q] = ld_stream(r + v + 32 * q);
#pragma unroll
      for (int q = 0; q < GEMV_Q; q += 2) {
        s0 = vdot(sa[v + 32 * q], x[q], s0);
        s1 = vdot(sa[v + 32 * (q + 1)], x[q + 1], s1);
      }
    }
    for (; v < nv; v += 32) s0 = vdot(sa[v], ld_stream(r + v), s0);
    s0 = warp_sum(s0 + s1);
    if (lane == 0) crow[j] += s0;
  }
}

// FAST, split form: a CTA owns a contiguous block of rows of bt and its eight warps each own an eighth of every row, so that the
// rows divide evenly over 2 x 148 CTAs whatever N is (with whole rows per warp, N = 4096 leaves 256 CTAs of two rows per warp on
// 148 SMs: a seventh of the machine idles through the second half of the launch).  The eight partial sums of a row meet in shared
// memory and are added in warp order by one thread per row: the result does not depend on timing.
template <typename T>
__global__ void __launch_bounds__(256, 2) gemv_row_split_kernel(T* __restrict__ c, const T* __restrict__ a, const T* __restrict__ bt, int n,
                                                                IterRef iter, int rows_max) {
  using VT = typename V16<T>::type;
  constexpr int W = V16<T>::W;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  VT* sa = reinterpret_cast<VT*>(smem_raw);                                                  // n / W vectors: row i of a
  T* part = reinterpret_cast<T*>(smem_raw + static_cast<size_t>(n) * sizeof(T));            // [rows_max][8]
  const int i = iter.off + (iter.base ? *iter.base : 0);
  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  const int nv = n / W, seg = nv / 8;  // vectors per row, per warp (a multiple of 32: the launcher checks)
  const VT* av = reinterpret_cast<const VT*>(a + static_cast<size_t>(i) * n);
  for (int v = tid; v < nv; v += 256) sa[v] = av[v];
  __syncthreads();

  const int j0 = static_cast<int>(static_cast<long long>(blockIdx.x) * n / gridDim.x);
  const int j1 = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * n / gridDim.x);
  const int v0 = warp * seg;
  for (int j = j0; j < j1; ++j) {
    const VT* r = reinterpret_cast<const VT*>(bt + static_cast<size_t>(j) * n) + v0;
    T s0 = 0, s1 = 0;
    int v = lane;
    for (; v + 32 * (GEMV_Q - 1) < seg; v += 32 * GEMV_Q) {
      VT x[GEMV_Q];
#pragma unroll
      for (int q = 0; q < GEMV_Q; ++q) x[q] = ld_stream(r + v + 32 * q);
#pragma unroll
      for (int q = 0; q < GEMV_Q; q += 2) {
        s0 = vdot(sa[v0 + v + 32 * q], x[q], s0);
        s1 = vdot(sa[v0 + v + 32 * (q + 1)], x[q + 1], s1);
      }
    }
    if (v + 32 * 3 < seg) {  // four more (FP32 rows of 4096: the whole segment)
      VT x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = ld_stream(r + v + 32 * q);
#pragma unroll
      for (int q = 0; q < 4; q += 2) {
        s0 = vdot(sa[v0 + v + 32 * q], x[q], s0);
        s1 = vdot(sa[v0 + v + 32 * (q + 1)], x[q + 1], s1);
      }
      v += 32 * 4;
    }
    for (; v < seg; v += 32) s0 = vdot(sa[v0 + v], ld_stream(r + v), s0);
    s0 = warp_sum(s0 + s1);
    if (lane == 0) part[(j - j0) * 8 + warp] = s0;
  }
  __syncthreads();
  T* crow = c + static_cast<size_t>(i) * n;
  for (int t = tid; t < j1 - j0; t += 256) {
    T tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += part[t * 8 + w];
    crow[j0 + t] += tot;
  }
  (void)rows_max;
}

// STRICT: block = 64 threads owns 64 columns j; k is walked in tiles of 64 staged in smem.
template <typename T>
__global__ void __launch_bounds__(64) gemv_row_strict_kernel(T* __restrict__ c, const T* __restrict__ a,
                                                             const T* __restrict__ bt, int n, IterRef iter) {
  __shared__ T sb[64][65];
  __shared__ T sa[64];
  const int i = iter.off + (iter.base ? *iter.base : 0);
  const int t = threadIdx.x;
  const int j0 = blockIdx.x * 64;
  const int j = j0 + t;
  T acc = j < n ? c[static_cast<size_t>(i) * n + j] : static_cast<T>(0.0);
  for (int k0 = 0; k0 < n; k0 += 64) {
    const int kw = min(64, n - k0);
    if (t < kw) sa[t] = a[static_cast<size_t>(i) * n + k0 + t];
    for (int r = 0; r < 64; ++r)  // coalesced: thread t reads bt[j0+r][k0+t]
      if (j0 + r < n && t < kw) sb[r][t] = bt[static_cast<size_t>(j0 + r) * n + k0 + t];
    __syncthreads();
    if (j < n)
      for (int k = 0; k < kw; ++k) acc = strict_mac(acc, sa[k], sb[t][k]);
    __syncthreads();
  }
  if (j < n) c[static_cast<size_t>(i) * n + j] = acc;
}

// ---- gene 10 -----------------------------------------------------------------------------------

// FAST: one block of 256 threads per (i, j).
template <typename T>
__global__ void __launch_bounds__(256) dot_fast_kernel(T* __restrict__ c, const T* __restrict__ a,
                                                       const T* __restrict__ bt, int n, IterRef iter, bool vec_ok) {
  using VT = typename V16<T>::type;
  constexpr int W = V16<T>::W;
  __shared__ T partial[8];
  const int f = iter.off + (iter.base ? *iter.base : 0);
  const int i = f / n, j = f % n;
  const T* x = a + static_cast<size_t>(i) * n;
  const T* y = bt + static_cast<size_t>(j) * n;
  T acc = 0;
  if (vec_ok) {
    const VT* xv = reinterpret_cast<const VT*>(x);
    const VT* yv = reinterpret_cast<const VT*>(y);
    for (int v = threadIdx.x; v < n / W; v += 256) acc = vdot(xv[v], yv[v], acc);
  } else {
    for (int k = threadIdx.x; k < n; k += 256) acc += x[k] * y[k];
  }
  acc = warp_sum(acc);
  if (threadIdx.x % 32 == 0) partial[threadIdx.x / 32] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    T v = threadIdx.x < 8 ? partial[threadIdx.x] : static_cast<T>(0.0);
    v = warp_sum(v);
    if (threadIdx.x == 0) c[static_cast<size_t>(i) * n + j] += v;
  }
}

// STRICT: stage both rows in smem chunk by chunk, thread 0 walks k ascending.
template <typename T>
__global__ void __launch_bounds__(256) dot_strict_kernel(T* __restrict__ c, const T* __restrict__ a,
                                                         const T* __restrict__ bt, int n, IterRef iter) {
  constexpr int CH = 2048;
  __shared__ T sx[CH], sy[CH];
  const int f = iter.off + (iter.base ? *iter.base : 0);
  const int i = f / n, j = f % n;
  const T* x = a + static_cast<size_t>(i) * n;
  const T* y = bt + static_cast<size_t>(j) * n;
  T acc = c[static_cast<size_t>(i) * n + j];
  for (int k0 = 0; k0 < n; k0 += CH) {
    const int kw = min(CH, n - k0);
    for (int k = threadIdx.x; k < kw; k += 256) {
      sx[k] = x[k0 + k];
      sy[k] = y[k0 + k];
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < kw; ++k) acc = strict_mac(acc, sx[k], sy[k]);
    __syncthreads();
  }
  if (threadIdx.x == 0) c[static_cast<size_t>(i) * n + j] = acc;
}

// ---- gene 11 -----------------------------------------------------------------------------------

// One block of 1024 threads: strided gather of the diagonal, shuffle + smem tree (FAST), or
// staged chunks summed in index order by thread 0 (STRICT).  N elements, latency-bound.
template <typename T, bool STRICT>
__global__ void __launch_bounds__(1024) trace_kernel(T* __restrict__ sum, const T* __restrict__ c_full, int n_full,
                                                     int first, int count) {
  __shared__ T buf[1024];
  const int t = threadIdx.x;
  const size_t pitch = static_cast<size_t>(n_full) + 1;
  const T* c = c_full + first * pitch;  // diagonal entry `first`
  const int n = count;
  if constexpr (STRICT) {
    T acc = static_cast<T>(0.0);
    for (int i0 = 0; i0 < n; i0 += 1024) {
      const int w = min(1024, n - i0);
      if (t < w) buf[t] = c[(i0 + t) * pitch];
      __syncthreads();
      if (t == 0)
        for (int i = 0; i < w; ++i) {
          if constexpr (sizeof(T) == 8) acc = __dadd_rn(acc, buf[i]);
          else acc = __fadd_rn(acc, buf[i]);
        }
      __syncthreads();
    }
    if (t == 0) *sum = acc;
  } else {
    T acc = static_cast<T>(0.0);
    for (int i = t; i < n; i += 1024) acc += c[i * pitch];
    acc = warp_sum(acc);
    if (t % 32 == 0) buf[t / 32] = acc;
    __syncthreads();
    if (t < 32) {
      T v = buf[t];  // 32 warps
      v = warp_sum(v);
      if (t == 0) *sum = v;
    }
  }
}

}  // namespace

template <typename T>
cudaError_t launch_gemv_row(T* c, const T* a, const T* bt, int n, IterRef iter, bool strict, cudaStream_t stream) {
  if (strict) {
    gemv_row_strict_kernel<T><<<(n + 63) / 64, 64, 0, stream>>>(c, a, bt, n, iter);
  } else {
    const bool vec_ok = n % V16<T>::W == 0;
    const size_t row_bytes = static_cast<size_t>(n) * sizeof(T);
    if (vec_ok && row_bytes <= 64 * 1024 && n >= 512) {
      static PerDeviceOnce once;  // function attributes are per device
      bool& configured = once.here();
      if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(gemv_row_staged_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(gemv_row_stream_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        if (e != cudaSuccess) return e;
        configured = true;
      }
      static const int form = [] { const char* e = getenv("MMX_GEMV_FORM"); return e ? atoi(e) : 0; }();  // tuning hook: 1 staged, 2 split, 0 by size
      const int nv = n / V16<T>::W;
      // the split form wins where a row fills the staging buffer (64 KB: N = 8192 FP64 93 -> 84 us, N = 16384 FP32 168 -> 157) and
      // loses below (N = 4096 FP32 18.4 -> 20.3): profiles/r2x_gemv_forms.txt
      if ((form == 2 || (form == 0 && row_bytes >= 64 * 1024)) && nv % 256 == 0) {
        static PerDeviceOnce once_split;
        bool& split_ok = once_split.here();
        if (!split_ok) {
          if (cudaError_t e = cudaFuncSetAttribute(gemv_row_split_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024); e != cudaSuccess)
            return e;
          split_ok = true;
        }
        const int grid = n < 2 * kNumSMs ? n : 2 * kNumSMs;
        const int rows_max = (n + grid - 1) / grid;
        const size_t smem = row_bytes + static_cast<size_t>(rows_max) * 8 * sizeof(T);
        gemv_row_split_kernel<T><<<grid, 256, smem, stream>>>(c, a, bt, n, iter, rows_max);
        return cudaGetLastError();
      }
      if (form == 1) {
        const int grid = n / 2 < 2 * kNumSMs ? n / 2 : 2 * kNumSMs;
        gemv_row_staged_kernel<T><<<grid, 256, row_bytes, stream>>>(c, a, bt, n, iter);
      } else {
        // largest CTA count <= 2 per SM that gives every warp the same number of rows (when 8 divides n)
        int grid = 2 * kNumSMs;
        const int row_groups = (n + 7) / 8;
        if (row_groups <= grid) grid = row_groups;
        else if (row_groups % 2 == 0) { const int per = (row_groups + grid - 1) / grid; grid = (row_groups + per - 1) / per; }
        gemv_row_stream_kernel<T><<<grid, 256, row_bytes, stream>>>(c, a, bt, n, iter);
      }
    } else {
      gemv_row_fast_kernel<T><<<(n + 7) / 8, 256, 0, stream>>>(c, a, bt, n, iter, vec_ok);
    }
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_dot(T* c, const T* a, const T* bt, int n, IterRef flat_iter, bool strict, cudaStream_t stream) {
  if (strict) {
    dot_strict_kernel<T><<<1, 256, 0, stream>>>(c, a, bt, n, flat_iter);
  } else {
    const bool vec_ok = n % V16<T>::W == 0;
    dot_fast_kernel<T><<<1, 256, 0, stream>>>(c, a, bt, n, flat_iter, vec_ok);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_trace(T* sum, const T* c, int n, int row0, int rows, bool strict, cudaStream_t stream) {
  if (strict) trace_kernel<T, true><<<1, 1024, 0, stream>>>(sum, c, n, row0, rows);
  else trace_kernel<T, false><<<1, 1024, 0, stream>>>(sum, c, n, row0, rows);
  return cudaGetLastError();
}

#define MMX_INST(T)                                                                                        \
  template cudaError_t launch_gemv_row<T>(T*, const T*, const T*, int, IterRef, bool, cudaStream_t);      \
  template cudaError_t launch_dot<T>(T*, const T*, const T*, int, IterRef, bool, cudaStream_t);           \
  template cudaError_t launch_trace<T>(T*, const T*, int, int, int, bool, cudaStream_t);
MMX_INST(double)
MMX_INST(float)

}  // namespace mmx
