// transpose.cu -- genes 6 and 7: bt[i][j] = b[j][i]  (fixtures/matmul.c:21-23)
//
// Pure data movement, bit-exact by construction.  HBM-bound: 2*E*N^2 bytes (read b, write bt).
//
// gene 6 (whole nest), fast path for N % 64 == 0: a CTA moves one 64x64 tile.  Global loads
// and stores are both 128-bit and fully coalesced (a warp covers whole 512 B / 256 B row
// segments).  The tile of b is staged in shared memory as it lies in global memory, by cp.async
// (16 bytes each, past the registers and L1), XOR-swizzled at 16-byte granularity
// (chunk ^= (row / V) & 7, V = 16 B / E); a thread then gathers the V elements of one 16-byte
// piece of a row of bt from V consecutive rows of the staged tile and stores it.
//
// gene 7 (one row of bt per launch): row i of bt is column i of b -- a strided gather; each
// 8-byte element costs a 32-byte sector, which is the sector amplification the catalogue notes.
#include <type_traits>

#include "kernels.cuh"
#include "ozaki_digits.cuh"

namespace mmx {
namespace {

constexpr int kTile = 64;

template <typename T> struct VecOf;
template <> struct VecOf<double> { using type = double2; static constexpr int V = 2; };
template <> struct VecOf<float> { using type = float4; static constexpr int V = 4; };

// Piece `chunk` of row `out_row` of the transposed tile = column out_row of rows chunk * V .. + V of the staged tile of b: V scalar
// reads (the lanes of a warp walk down the micro-rows, which the swizzle spreads over the eight 16-byte bank groups: a fourfold
// conflict on 8-byte reads, a twofold one on 4-byte reads -- the cost of one 16-byte read per lane).
__device__ __forceinline__ double2 gather_piece(const double2* tile, int out_row, int chunk) {
  constexpr int MB = kTile / 2;
  const double* t = reinterpret_cast<const double*>(tile);
  const int at = ((out_row / 2) ^ (chunk & 7)) * 2 + (out_row & 1);
  return make_double2(t[(chunk * 2) * (MB * 2) + at], t[(chunk * 2 + 1) * (MB * 2) + at]);
}
__device__ __forceinline__ float4 gather_piece(const float4* tile, int out_row, int chunk) {
  constexpr int MB = kTile / 4;
  const float* t = reinterpret_cast<const float*>(tile);
  const int at = ((out_row / 4) ^ (chunk & 7)) * 4 + (out_row & 3);
  return make_float4(t[(chunk * 4) * (MB * 4) + at], t[(chunk * 4 + 1) * (MB * 4) + at], t[(chunk * 4 + 2) * (MB * 4) + at],
                     t[(chunk * 4 + 3) * (MB * 4) + at]);
}

// grid = (rows/64, n/64); block = 256 threads.  PUSH: the finished tile is stored into every destination
// of `peers` (this GPU's bt and, through peer-mapped pointers, the bt of every other GPU of a row-sharded
// run): the all-gather of bt happens inside the kernel that produces it, as NVLink stores.
// PLANES: the digit planes of bt for gene 8 (ozaki_digits.cuh) are written from the same registers as bt itself; P.exps[j] must
// already hold the exponent of row j of bt (launch_fill_b_colexp).
// GEN (with PLANES; 0 = off, 1 = N a power of two, 2 = any N): the tile of b does not come from memory -- the CTA COMPUTES it
// (b[i][j] = (T)(i - j) / N, fixtures/matmul.c:12-14, the arithmetic of fill.cu bit for bit), stores it to b and lays it into shared
// memory where the copies would have put it: the init-b nest and the transpose nest of a plan that maps both to the device run as ONE
// kernel, and the 8 N^2 bytes of b are written but never read back (N = 4096: init-b 22.5 us + transpose 51 us become one launch).
template <typename T, bool PUSH, bool PLANES = false, int GEN = 0>
__global__ void __launch_bounds__(256, PLANES ? (sizeof(T) == 8 ? 5 : 6) : 1) transpose_tile_kernel(T* __restrict__ bt, const T* __restrict__ b, int n, int first_row,
                                                             BtPeers peers, OzOperand P = OzOperand{}) {
  using VT = typename VecOf<T>::type;
  constexpr int V = VecOf<T>::V;
  constexpr int MB = kTile / V;         // micro-blocks per tile side == 16-byte chunks per tile row
  __shared__ __align__(16) VT tile[kTile * MB];   // the tile of b, input-ordered: tile[row][chunk], swizzled

  // rows of b == columns of bt, last rows first: what the fill of b wrote last is what L2 still holds
  const int in_row0 = static_cast<int>(gridDim.y - 1 - blockIdx.y) * kTile;
  const int in_col0 = first_row + blockIdx.x * kTile;   // cols of b  == rows of bt
  const int tid = threadIdx.x;

  // PLANES: what phase 2 needs from global memory besides the tile is requested first, so that it arrives with the tile
  constexpr int kSteps = kTile * MB / 256;
  int row_exp[PLANES ? kSteps : 1];
  int dirty = 0;
  if constexpr (PLANES) {
    dirty = P.guard[P.dirty_slot];
#pragma unroll
    for (int k = 0; k < kSteps; ++k) row_exp[k] = P.exps[in_col0 + (tid + 256 * k) / MB];
  }

  // phase 1: the tile of b goes to shared memory as it lies in global memory (rows of b), 16 bytes per cp.async, lanes along the
  // row; chunk c of row r lands at chunk c ^ ((r / V) & 7).  The copies bypass the registers and L1: how many bytes a CTA has in
  // flight is then not bounded by what L1 can track (with loads into registers the kernel lost 10 % when the shared-memory
  // carve-out left L1 28 KB instead of 60 -- profiles/r2x_transpose_l1.txt)
  if constexpr (GEN != 0) {
    // the tile is produced here: the values of init-b, 16 bytes per thread and step, lanes along the row of b (whole 512-byte runs
    // per warp), to b itself (streaming: nothing on the device reads it again) and into the staged tile
    T* b_out = const_cast<T*>(b);
    const T nn = static_cast<T>(n), inv_n = static_cast<T>(1.0) / static_cast<T>(n);
#pragma unroll
    for (int k = 0; k < kSteps; ++k) {
      const int v = tid + 256 * k;
      const int row = v / MB, chunk = v % MB;
      const int i = in_row0 + row, j0 = in_col0 + chunk * V;
      T x[V];
#pragma unroll
      for (int w = 0; w < V; ++w) x[w] = GEN == 1 ? static_cast<T>(i - (j0 + w)) * inv_n : static_cast<T>(i - (j0 + w)) / nn;
      VT val;
      if constexpr (V == 2) val = make_double2(x[0], x[1]);
      else val = make_float4(x[0], x[1], x[2], x[3]);
      if (b_out != nullptr) __stcs(reinterpret_cast<VT*>(b_out + static_cast<size_t>(i) * n + j0), val);  // NULL: b is written elsewhere
      tile[row * MB + (chunk ^ ((row / V) & 7))] = val;
    }
    __syncthreads();
  } else {
  const unsigned tile_s = static_cast<unsigned>(__cvta_generic_to_shared(tile));
#pragma unroll
  for (int k = 0; k < kSteps; ++k) {
    const int v = tid + 256 * k;
    const int row = v / MB, chunk = v % MB;
    const T* src = b + static_cast<size_t>(in_row0 + row) * n + in_col0 + chunk * V;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tile_s + 16u * (row * MB + (chunk ^ ((row / V) & 7)))), "l"(src) : "memory");
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  }

  // phase 2: lanes along the output row (coalesced 128-bit stores)
  int lossy = 0, top = 0;
  constexpr int STEPS = kTile * MB / 256;  // pieces per thread
  if constexpr (PLANES) {
    // the exponents of this thread's rows of bt and the dirty mark were requested before the tile was loaded (below): nothing in
    // the store loop waits on global memory.  Pass 1 is straight-line: store the piece, walk its first two digit levels
    // (oz_emit_first_two: independent FP64 chains, no branches); pass 2 (rare) re-reads from the tile the pieces that have more.
    // FP64: the digits of the tile are collected in shared memory (64 rows x 64 bytes per plane) and leave as 16-byte stores --
    // 2-byte stores straight from the walk cost eight times the store instructions for the same sectors (N = 8192: 211 -> 199 us).
    // FP32 pieces hold four elements: their 4-byte digit stores go out directly (staging them costs occupancy and gains nothing)
    constexpr bool STAGED = V == 2;
    __shared__ __align__(16) unsigned char dig[STAGED ? 2 : 1][STAGED ? kTile : 1][STAGED ? kTile : 16];
    // L = digit levels of the straight-line pass: two, or three once an earlier encoding of bt has needed a third (the application
    // from N = 16384); a third level goes out directly (a third staging plane would cost a CTA per SM)
    auto body = [&](auto levels) {
      constexpr int L = decltype(levels)::value;
      unsigned more = 0;
#pragma unroll
      for (int k = 0; k < STEPS; ++k) {
        const int v = tid + 256 * k;
        const int out_row = v / MB, chunk = v % MB;
        const VT val = gather_piece(tile, out_row, chunk);
        __stcs(reinterpret_cast<VT*>(bt + static_cast<size_t>(in_col0 + out_row) * n + in_row0 + chunk * V), val);
        bool tiny;
        const double inv = oz_row_scale_of(row_exp[k], &tiny), ainv = fabs(inv);
        signed char* drow = P.planes + static_cast<size_t>(in_col0 + out_row) * P.kq;
        int top_l = 0;
        bool left;
        if constexpr (V == 2) {
          const double e2[2] = {val.x, val.y};
          // not finite, or beyond what the exponent covers (it cannot happen while the executor's flags are right): cut
          left = tiny || !(fabs(val.x) * ainv < 1.0) || !(fabs(val.y) * ainv < 1.0);
          int word[L];
          left = oz_first_words<2, L>(e2, inv, word) || left;
          *reinterpret_cast<unsigned short*>(&dig[0][out_row][chunk * V]) = static_cast<unsigned short>(word[0]);
          *reinterpret_cast<unsigned short*>(&dig[1][out_row][chunk * V]) = static_cast<unsigned short>(word[1]);
#pragma unroll
          for (int l = 2; l < L; ++l)
            *reinterpret_cast<unsigned short*>(drow + l * P.plane + in_row0 + chunk * V) = static_cast<unsigned short>(word[l]);
#pragma unroll
          for (int l = 0; l < L; ++l)
            if (word[l] != 0) top_l = l + 1;
        } else {
          const double e4[4] = {static_cast<double>(val.x), static_cast<double>(val.y), static_cast<double>(val.z), static_cast<double>(val.w)};
          left = tiny;
#pragma unroll
          for (int q = 0; q < 4; ++q) left = left || !(fabs(e4[q]) * ainv < 1.0);
          left = oz_emit_first<4, L>(e4, inv, drow, P.plane, in_row0 + chunk * V, top_l) || left;
        }
        top = max(top, top_l);
        more |= (left ? 1u : 0u) << k;
      }
      if constexpr (STAGED) {
        __syncthreads();
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const int row = tid / 4, q = tid % 4;
          *reinterpret_cast<int4*>(P.planes + p * P.plane + static_cast<size_t>(in_col0 + row) * P.kq + in_row0 + q * 16) =
              *reinterpret_cast<const int4*>(&dig[p][row][q * 16]);
        }
      }
      if (more != 0 || dirty > L) {
        for (int k = 0; k < STEPS; ++k) {
          if (!(more >> k & 1u) && dirty <= L) continue;
          const int v = tid + 256 * k;
          const int out_row = v / MB, chunk = v % MB;
          const VT val = gather_piece(tile, out_row, chunk);
          bool tiny;
          const double inv = oz_row_scale_of(row_exp[k], &tiny), ainv = fabs(inv);
          lossy |= tiny;
          signed char* drow = P.planes + static_cast<size_t>(in_col0 + out_row) * P.kq;
          if constexpr (V == 2) {
            const double e2[2] = {val.x, val.y};
            lossy |= !(fabs(val.x) * ainv < 1.0) | !(fabs(val.y) * ainv < 1.0);
            oz_emit<7, 2>(e2, inv, false, dirty, drow, P.plane, in_row0 + chunk * V, lossy, top);
          } else {
            const double e4[4] = {static_cast<double>(val.x), static_cast<double>(val.y), static_cast<double>(val.z), static_cast<double>(val.w)};
#pragma unroll
            for (int q = 0; q < 4; ++q) lossy |= !(fabs(e4[q]) * ainv < 1.0);
            oz_emit<7, 4>(e4, inv, false, dirty, drow, P.plane, in_row0 + chunk * V, lossy, top);
          }
        }
      }
    };
    if (dirty == 3) body(std::integral_constant<int, 3>{});
    else body(std::integral_constant<int, 2>{});
    oz_guard_commit(lossy, top, P.guard, P.lossy_slot, P.top_slot, P.dirty_slot);
  } else {
#pragma unroll
    for (int v = tid; v < kTile * MB; v += 256) {
      const int out_row = v / MB;
      const int chunk = v % MB;
      const VT val = gather_piece(tile, out_row, chunk);
      const size_t at = static_cast<size_t>(in_col0 + out_row) * n + in_row0 + chunk * V;
      if constexpr (PUSH) {
        for (int d = 0; d < peers.count; ++d) *reinterpret_cast<VT*>(static_cast<T*>(peers.p[d]) + at) = val;
      } else {
        *reinterpret_cast<VT*>(bt + at) = val;
      }
    }
  }
}

// Any n: 32x32 tile, scalar accesses, +1 padding.  block = (32, 8).
template <typename T, bool PUSH>
__global__ void __launch_bounds__(256) transpose_generic_kernel(T* __restrict__ bt, const T* __restrict__ b, int n,
                                                                int first_row, int row_limit, BtPeers peers) {
  __shared__ T tile[32][33];
  const int x = first_row + blockIdx.x * 32 + threadIdx.x;  // column of b = row of bt
#pragma unroll
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int y = blockIdx.y * 32 + r;
    if (x < row_limit && y < n) tile[r][threadIdx.x] = b[static_cast<size_t>(y) * n + x];
  }
  __syncthreads();
  const int ox = blockIdx.y * 32 + threadIdx.x;  // column of bt = row of b
#pragma unroll
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int oy = first_row + blockIdx.x * 32 + r;  // row of bt = column of b
    if (ox < n && oy < row_limit) {
      const T val = tile[threadIdx.x][r];
      const size_t at = static_cast<size_t>(oy) * n + ox;
      if constexpr (PUSH) {
        for (int d = 0; d < peers.count; ++d) static_cast<T*>(peers.p[d])[at] = val;
      } else {
        bt[at] = val;
      }
    }
  }
}

// gene 7: bt[i][j] = b[j][i] for all j; i = iteration of the host loop.
template <typename T>
__global__ void __launch_bounds__(256) transpose_row_kernel(T* __restrict__ bt, const T* __restrict__ b, int n, IterRef iter) {
  const int i = iter.off + (iter.base ? *iter.base : 0);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) bt[static_cast<size_t>(i) * n + j] = b[static_cast<size_t>(j) * n + i];
}

}  // namespace

template <typename T>
cudaError_t launch_transpose(T* bt, const T* b, int n, int row0, int rows, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (n % kTile == 0 && row0 % kTile == 0 && rows % kTile == 0) {
    dim3 grid(rows / kTile, n / kTile);
    transpose_tile_kernel<T, false><<<grid, 256, 0, stream>>>(bt, b, n, row0, BtPeers{});
  } else {
    dim3 grid((rows + 31) / 32, (n + 31) / 32);
    transpose_generic_kernel<T, false><<<grid, dim3(32, 8), 0, stream>>>(bt, b, n, row0, row0 + rows, BtPeers{});
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_transpose_planes(T* bt, const T* b, int n, const OzOperand& pb, cudaStream_t stream) {
  if (!ozaki_fusable(n) || pb.kq != n) return cudaErrorInvalidValue;
  // the guard words of bt start from zero for this encoding (the slice pass does the same before it runs)
  if (cudaError_t e = cudaMemsetAsync(pb.guard + pb.top_slot, 0, 2 * sizeof(int), stream); e != cudaSuccess) return e;   // words 2, 3
  dim3 grid(n / kTile, n / kTile);
  transpose_tile_kernel<T, false, true><<<grid, 256, 0, stream>>>(bt, b, n, 0, BtPeers{}, pb);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_fill_b_transpose_planes(T* b, T* bt, int n, const OzOperand& pb, cudaStream_t stream) {
  if (!ozaki_fusable(n) || pb.kq != n) return cudaErrorInvalidValue;
  if (cudaError_t e = cudaMemsetAsync(pb.guard + pb.top_slot, 0, 2 * sizeof(int), stream); e != cudaSuccess) return e;   // words 2, 3
  dim3 grid(n / kTile, n / kTile);
  if ((n & (n - 1)) == 0) transpose_tile_kernel<T, false, true, 1><<<grid, 256, 0, stream>>>(bt, b, n, 0, BtPeers{}, pb);
  else transpose_tile_kernel<T, false, true, 2><<<grid, 256, 0, stream>>>(bt, b, n, 0, BtPeers{}, pb);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_transpose_push(const BtPeers& peers, const T* b, int n, int row0, int rows, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (peers.count < 1 || peers.count > kMaxPeers) return cudaErrorInvalidValue;
  if (n % kTile == 0 && row0 % kTile == 0 && rows % kTile == 0) {
    dim3 grid(rows / kTile, n / kTile);
    transpose_tile_kernel<T, true><<<grid, 256, 0, stream>>>(nullptr, b, n, row0, peers);
  } else {
    dim3 grid((rows + 31) / 32, (n + 31) / 32);
    transpose_generic_kernel<T, true><<<grid, dim3(32, 8), 0, stream>>>(nullptr, b, n, row0, row0 + rows, peers);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_transpose_row(T* bt, const T* b, int n, IterRef iter, cudaStream_t stream) {
  const int threads = n < 256 ? ((n + 31) / 32) * 32 : 256;
  transpose_row_kernel<T><<<(n + threads - 1) / threads, threads, 0, stream>>>(bt, b, n, iter);
  return cudaGetLastError();
}

template cudaError_t launch_transpose<double>(double*, const double*, int, int, int, cudaStream_t);
template cudaError_t launch_transpose<float>(float*, const float*, int, int, int, cudaStream_t);
template cudaError_t launch_transpose_planes<double>(double*, const double*, int, const OzOperand&, cudaStream_t);
template cudaError_t launch_transpose_planes<float>(float*, const float*, int, const OzOperand&, cudaStream_t);
template cudaError_t launch_fill_b_transpose_planes<double>(double*, double*, int, const OzOperand&, cudaStream_t);
template cudaError_t launch_fill_b_transpose_planes<float>(float*, float*, int, const OzOperand&, cudaStream_t);
template cudaError_t launch_transpose_push<double>(const BtPeers&, const double*, int, int, int, cudaStream_t);
template cudaError_t launch_transpose_push<float>(const BtPeers&, const float*, int, int, int, cudaStream_t);
template cudaError_t launch_transpose_row<double>(double*, const double*, int, IterRef, cudaStream_t);
template cudaError_t launch_transpose_row<float>(float*, const float*, int, IterRef, cudaStream_t);

}  // namespace mmx
