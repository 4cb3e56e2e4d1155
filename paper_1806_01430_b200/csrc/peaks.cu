// peaks.cu -- on-device peak probes for the roofline denominators the driver-written
// MEASURED_PEAKS.json does not carry (it has HBM copy and bf16 GEMM only): FP64 DFMA, FP64
// DMMA.8x8x4, FP32 FFMA issue peaks, the tcgen05 tensor pipe's issue peaks for kind::i8, kind::tf32 and kind::f16 (bf16 inputs;
// operands resident in shared memory, no loads, M = 128 x N = 256 instructions back to back from one thread per SM -- the ceiling
// of the contraction kernels of matmul_ozaki.cu / matmul_tc.cu), plus write-only / read-only / copy HBM rates with this
// library's own access pattern.  Each probe warms up, then reports the best of several
// CUDA-event-timed launches on the default stream of the current device.
#include <algorithm>
#include <cstdint>

#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace mmx {
namespace {

constexpr int kThreads = 256;
constexpr int kBlocksPerSM = 4;
constexpr int kIters = 4096;

// 16 independent FMA chains per thread: enough ILP to cover the pipe latency at 4 CTAs/SM.
template <typename T>
__global__ void __launch_bounds__(kThreads) fma_peak_kernel(T* out, T x, T y) {
  T acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = static_cast<T>(threadIdx.x + q);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if constexpr (sizeof(T) == 8) acc[q] = __fma_rn(acc[q], x, y);
      else acc[q] = __fmaf_rn(acc[q], x, y);
    }
  }
  T s = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) s += acc[q];
  if (s == static_cast<T>(-1.2345)) out[0] = s;  // keep the chains alive, never true
}

// 16 independent DMMA accumulator pairs per warp.
__global__ void __launch_bounds__(kThreads) dmma_peak_kernel(double* out, double x, double y) {
  double c0[16], c1[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    c0[q] = threadIdx.x + q;
    c1[q] = threadIdx.x - q;
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int q = 0; q < 16; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[q]), "+d"(c1[q])
                   : "d"(x), "d"(y));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) s += c0[q] + c1[q];
  if (s == -1.2345) out[0] = s;
}

__global__ void __launch_bounds__(kThreads) copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t nvec) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t v = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; v + 3 * stride < nvec; v += 4 * stride) {
    const uint4 a = src[v], b = src[v + stride], c = src[v + 2 * stride], d = src[v + 3 * stride];
    dst[v] = a;
    dst[v + stride] = b;
    dst[v + 2 * stride] = c;
    dst[v + 3 * stride] = d;
  }
  for (; v < nvec; v += stride) dst[v] = src[v];
}

__global__ void __launch_bounds__(kThreads) read_kernel(uint4* __restrict__ sink, const uint4* __restrict__ src, size_t nvec) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  uint4 acc = make_uint4(0, 0, 0, 0);
  size_t v = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; v + 3 * stride < nvec; v += 4 * stride) {
    const uint4 a = src[v], b = src[v + stride], c = src[v + 2 * stride], d = src[v + 3 * stride];
    acc.x ^= a.x ^ b.x ^ c.x ^ d.x;
    acc.y ^= a.y ^ b.y ^ c.y ^ d.y;
    acc.z ^= a.z ^ b.z ^ c.z ^ d.z;
    acc.w ^= a.w ^ b.w ^ c.w ^ d.w;
  }
  for (; v < nvec; v += stride) acc.x ^= src[v].x;
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) sink[0] = acc;  // practically never
}

template <typename Launch>
cudaError_t best_ms(Launch launch, int reps, float* best) {
  cudaEvent_t e0, e1;
  cudaError_t err = cudaEventCreate(&e0);
  if (err != cudaSuccess) return err;
  err = cudaEventCreate(&e1);
  if (err != cudaSuccess) return err;
  for (int w = 0; w < 3; ++w) launch();
  *best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0, 0);
    launch();
    cudaEventRecord(e1, 0);
    err = cudaEventSynchronize(e1);
    if (err != cudaSuccess) break;
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *best = std::min(*best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (err == cudaSuccess) err = cudaGetLastError();
  return err;
}


// ---- tcgen05 issue peaks -----------------------------------------------------------------------------------------------
// KIND 0: kind::i8 (s8 x s8 -> s32, K = 32 per instruction), 1: kind::tf32 (K = 8), 2: kind::f16 with bf16 inputs (K = 16).
// One CTA per SM; A = 128 rows, B = 256 rows of one swizzle span each (64 bytes under SWIZZLE_64B for i8, as matmul_ozaki.cu lays
// its slices out; 128 bytes under SWIZZLE_128B for the float kinds, as matmul_tc.cu does), filled once with plausible values.
// Thread 0 issues M=128 x N=256 MMAs over the span's k steps into two alternating 256-column accumulators; a commit every 64
// instructions on alternating barriers keeps the queue bounded.  Nothing is loaded and nothing is drained: what is measured is
// the rate at which the tensor pipe retires instructions whose operands are already in shared memory.
template <int KIND> struct UmmaProbe {
  static constexpr int ROW_BYTES = KIND == 0 ? 64 : 128;
  static constexpr int KSTEPS = ROW_BYTES / 32;                 // every kind consumes 32 bytes of K per instruction
  static constexpr int K_PER_MMA = KIND == 0 ? 32 : KIND == 1 ? 8 : 16;
  static constexpr int A_BYTES = 128 * ROW_BYTES, B_BYTES = 256 * ROW_BYTES;
  static constexpr int SMEM = A_BYTES + B_BYTES + 1024 + 64;
};

template <int KIND>
__device__ __forceinline__ void umma_issue(unsigned d, unsigned long long a, unsigned long long b, unsigned idesc, unsigned acc) {
  if constexpr (KIND == 0)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else if constexpr (KIND == 1)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) umma_peak_kernel(int iters) {
  using P = UmmaProbe<KIND>;
  extern __shared__ unsigned char smem_raw[];
  const unsigned raw = smem_u32(smem_raw);
  const unsigned base = (raw + 1023u) & ~1023u;
  const unsigned bars = base + P::A_BYTES + P::B_BYTES;
  const unsigned tmem_slot = bars + 32;
  volatile unsigned* tmem_slot_ptr = reinterpret_cast<volatile unsigned*>(smem_raw + (tmem_slot - raw));
  unsigned* words = reinterpret_cast<unsigned*>(smem_raw + (base - raw));
  for (int w = threadIdx.x; w < (P::A_BYTES + P::B_BYTES) / 4; w += blockDim.x) {
    unsigned h = (static_cast<unsigned>(w) + 1u) * 2654435761u + blockIdx.x * 40503u;
    h ^= h >> 15;
    if constexpr (KIND == 0) words[w] = h & 0x3f3f3f3fu;                          // digits in [0, 63]
    else if constexpr (KIND == 1) words[w] = 0x3f800000u | (h & 0x007fe000u);     // tf32 in [1, 2)
    else words[w] = 0x3f803f80u | (h & 0x007f007fu);                              // two bf16 in [1, 2)
  }
  if (threadIdx.x == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_proxy_async_smem();
  if (threadIdx.x / 32 == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tmem_slot), "n"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = *tmem_slot_ptr;
  if (threadIdx.x == 0) {
    // shared-memory descriptors as the production kernels build them (cute::UMMA::SmemDescriptor)
    const unsigned long long layout = KIND == 0 ? 4ull : 2ull;                    // SWIZZLE_64B : SWIZZLE_128B
    auto desc = [&](unsigned addr) {
      return static_cast<unsigned long long>((addr & 0x3FFFF) >> 4) | (static_cast<unsigned long long>((8 * P::ROW_BYTES) >> 4) << 32) | (1ull << 46) | (layout << 61);
    };
    const unsigned long long a = desc(base), b = desc(base + P::A_BYTES);
    // D format @4 (s32 = 2, f32 = 1), A / B format @7 / @10 (s8 = 1; tf32 = 2; bf16 = 1), N >> 3 @17, M >> 4 @24
    const unsigned idesc = (KIND == 0 ? ((2u << 4) | (1u << 7) | (1u << 10)) : KIND == 1 ? ((1u << 4) | (2u << 7) | (2u << 10)) : ((1u << 4) | (1u << 7) | (1u << 10))) |
                           (static_cast<unsigned>(256 >> 3) << 17) | (static_cast<unsigned>(128 >> 4) << 24);
    constexpr int GROUP = 64 / P::KSTEPS;  // iterations per commit
    int groups = 0;
    for (int it = 0; it < iters; ++it) {
      const unsigned d = tmem + (it & 1) * 256;
#pragma unroll
      for (int ks = 0; ks < P::KSTEPS; ++ks) umma_issue<KIND>(d, a + 2ull * ks, b + 2ull * ks, idesc, (it > 1 || ks > 0) ? 1u : 0u);
      if ((it + 1) % GROUP == 0 || it + 1 == iters) {
        if (groups >= 2) mbar_wait(bars + 8 * (groups & 1), ((groups >> 1) - 1) & 1);  // the commit that last used this barrier
        tc_commit(bars + 8 * (groups & 1));
        ++groups;
      }
    }
    for (int g = groups >= 2 ? groups - 2 : 0; g < groups; ++g) mbar_wait(bars + 8 * (g & 1), (g >> 1) & 1);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x / 32 == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512) : "memory");
  }
}

template <int KIND>
cudaError_t umma_peak(int sms, double* value) {
  using P = UmmaProbe<KIND>;
  cudaError_t err = cudaFuncSetAttribute(umma_peak_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM);
  if (err != cudaSuccess) return err;
  const int iters = 16384 / P::KSTEPS;   // 16384 instructions of ~128 tensor-pipe clocks each: ~1.1 ms at full rate
  float ms = 0;
  err = best_ms([&] { umma_peak_kernel<KIND><<<sms, 128, P::SMEM>>>(iters); }, 7, &ms);
  if (err != cudaSuccess) return err;
  const double ops = 2.0 * 128 * 256 * P::K_PER_MMA * P::KSTEPS * static_cast<double>(iters) * sms;
  *value = ops / (ms * 1e-3) / 1e12;
  return cudaSuccess;
}

}  // namespace

cudaError_t probe_peak(int kind, double* value) {
  cudaError_t err = cudaSuccess;
  float ms = 0;
  int sms = kNumSMs, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * kBlocksPerSM;
  if (kind == 6) return umma_peak<0>(sms, value);
  if (kind == 7) return umma_peak<1>(sms, value);
  if (kind == 8) return umma_peak<2>(sms, value);
  if (kind == 2 || kind == 3 || kind == 4) {
    void* out = nullptr;
    if ((err = cudaMalloc(&out, 64)) != cudaSuccess) return err;
    double flops = 0;
    if (kind == 2) {
      err = best_ms([&] { fma_peak_kernel<double><<<grid, kThreads>>>(static_cast<double*>(out), 1.0000001, 1e-9); }, 5, &ms);
      flops = 2.0 * 16 * kIters * static_cast<double>(grid) * kThreads;
    } else if (kind == 4) {
      err = best_ms([&] { fma_peak_kernel<float><<<grid, kThreads>>>(static_cast<float*>(out), 1.0000001f, 1e-9f); }, 5, &ms);
      flops = 2.0 * 16 * kIters * static_cast<double>(grid) * kThreads;
    } else {
      err = best_ms([&] { dmma_peak_kernel<<<grid, kThreads>>>(static_cast<double*>(out), 1.0000001, 1e-9); }, 5, &ms);
      // one m8n8k4 MMA = 8*8*4 multiply-adds per warp
      flops = 2.0 * 256 * 16 * kIters * static_cast<double>(grid) * (kThreads / 32);
    }
    cudaFree(out);
    if (err != cudaSuccess) return err;
    *value = flops / (ms * 1e-3) / 1e12;
    return cudaSuccess;
  }
  if (kind == 0 || kind == 1 || kind == 5) {
    const size_t bytes = size_t{2} << 30;  // 2 GiB per buffer: >> 126 MB of L2
    void *src = nullptr, *dst = nullptr;
    if ((err = cudaMalloc(&src, bytes)) != cudaSuccess) return err;
    if ((err = cudaMalloc(&dst, bytes)) != cudaSuccess) {
      cudaFree(src);
      return err;
    }
    cudaMemset(src, 1, bytes);
    cudaMemset(dst, 2, bytes);
    const size_t nvec = bytes / 16;
    double moved = 0;
    if (kind == 0) {
      err = best_ms([&] { copy_kernel<<<sms * 8, kThreads>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), nvec); }, 10, &ms);
      moved = 2.0 * bytes;
    } else if (kind == 1) {
      err = best_ms([&] { launch_scrub(dst, bytes, 0); }, 10, &ms);
      moved = 1.0 * bytes;
    } else {
      err = best_ms([&] { read_kernel<<<sms * 8, kThreads>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), nvec); }, 10, &ms);
      moved = 1.0 * bytes;
    }
    cudaFree(src);
    cudaFree(dst);
    if (err != cudaSuccess) return err;
    *value = moved / (ms * 1e-3) / 1e9;
    return cudaSuccess;
  }
  return cudaErrorInvalidValue;
}

}  // namespace mmx
