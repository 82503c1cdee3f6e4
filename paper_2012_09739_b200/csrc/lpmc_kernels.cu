#include <cstdlib>
// Reduction, diagnostic and peak kernels, and the dispatch to the level
// kernels (lpmc_level_*.cu, one translation unit per bar arithmetic).
//
// Compiled with -fmad=false like every kernel TU: the reference rounds every
// operation separately (sde.hpp:60-116 on a binary64 carrier without FMA,
// SURVEY.md §A2), so no multiply-add may be contracted on this path; FMAs
// appear only where written explicitly (the exact-Gaussian math).

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lpmc_device.cuh"
#include "lpmc_glibc.cuh"
#include "lpmc_internal.h"

namespace lpmc_b200 {
namespace {

using namespace dev;

// Chunk tree: 1024 batch slots (empty past the end), pairwise Pebay merges.
__global__ void __launch_bounds__(kChunkThreads)
    chunk_reduce_kernel(const double* __restrict__ batch_acc, uint64_t n_batches,
                        double* __restrict__ chunk_acc) {
  __shared__ Acc s[kChunkThreads];
  const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kChunkBatches;
  const int t = threadIdx.x;
  for (int f = 0; f < 3; ++f) {
    Acc a{0, 0, 0, 0, 0}, b{0, 0, 0, 0, 0};
    const uint64_t i0 = b0 + 2 * t, i1 = b0 + 2 * t + 1;
    if (i0 < n_batches) a = load_acc(batch_acc + 15 * i0 + 5 * f);
    if (i1 < n_batches) b = load_acc(batch_acc + 15 * i1 + 5 * f);
    acc_merge(a, b);
    s[t] = a;
    __syncthreads();
    for (int width = kChunkThreads / 2; width >= 1; width >>= 1) {
      Acc r{0, 0, 0, 0, 0};
      if (t < width) {
        r = s[2 * t];
        acc_merge(r, s[2 * t + 1]);
      }
      __syncthreads();
      if (t < width) s[t] = r;
      __syncthreads();
    }
    if (t == 0) store_acc(chunk_acc + 15 * blockIdx.x + 5 * f, s[0]);
    __syncthreads();
  }
}

// The fused level kernel's batch tree (batch_moments, thread t = slot t) over
// per-path differences written by the warp-per-path kernel: the same
// accumulators the fused kernel would have produced.
__global__ void __launch_bounds__(kBatch)
    path_batch_kernel(const double* __restrict__ path_diff, uint64_t n_paths,
                      double* __restrict__ batch_acc) {
  const uint64_t first = static_cast<uint64_t>(blockIdx.x) * kBatch;
  const uint64_t left = n_paths - first;
  const int count = left < kBatch ? static_cast<int>(left) : kBatch;
  const bool valid[1] = {static_cast<int>(threadIdx.x) < count};
  const uint64_t i = first + threadIdx.x;
  const double dh[1] = {valid[0] ? path_diff[2 * i] : 0.0};
  const double db[1] = {valid[0] ? path_diff[2 * i + 1] : 0.0};
  batch_moments<1>(dh, db, valid, count, batch_acc + 15 * blockIdx.x);
}

// Reference order: one thread per (batch, family) adds its <= 256 values in
// path order, exactly run_batch's loop (mlmc.hpp:78-93).
__global__ void sequential_batch_kernel(const double* __restrict__ path_diff, uint64_t n_paths,
                                        double* __restrict__ batch_acc) {
  const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t n_batches = (n_paths + kBatch - 1) / kBatch;
  if (idx >= 3 * n_batches) return;
  const uint64_t b = idx / 3;
  const int f = static_cast<int>(idx % 3);
  Acc a{0, 0, 0, 0, 0};
  const uint64_t end = (b + 1) * kBatch < n_paths ? (b + 1) * kBatch : n_paths;
  for (uint64_t i = b * kBatch; i < end; ++i) {
    const double h = path_diff[2 * i], br = path_diff[2 * i + 1];
    acc_add(a, f == 0 ? h : (f == 1 ? br : __dsub_rn(h, br)));
  }
  store_acc(batch_acc + 15 * b + 5 * f, a);
}

// op 0: exact Gaussian (the sampler's path), 1: approximate (table), 2: the
// reference's formula on libdevice, 3: erfc core on t in [0, 6.5), 5: the
// exact Gaussian in LPMC_EXACT_Z_GLIBC mode (the reference's bit for bit).
// Threads past n evaluate a dummy so the warp-collective tail pass stays
// converged.
__global__ void inv_cdf_kernel(const double* __restrict__ u, uint64_t n,
                               const double* __restrict__ table, int K, int degree, int dyadic,
                               int stride, int simple, double tail, int op,
                               double* __restrict__ out) {
  __shared__ __align__(16) double s_math[kMathWords];
  stage_math(s_math);
  __syncthreads();
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool in = i < n;
  const double x = in ? u[i] : 0.25;
  double r = 0.0;
  if (op == 0) {
    double uu[1] = {x}, zz[1];
    math::phi_inv_multi<1>(uu, zz, math::FlatTab{s_math});
    r = zz[0];
  } else if (op == 1) {
    const TableView t{table, stride, K, degree, dyadic, simple, tail};
    r = approx_inv(t, x);
  } else if (op == 2) {
    r = math::phi_inv_libdevice(x);
  } else if (op == 5) {
    double uu[1] = {x}, zz[1];
    glibc::inv_cdf_multi<1>(uu, zz, s_math);
    r = zz[0];
  } else {
    r = math::erfc_fast(x, s_math);
  }
  if (in) out[i] = r;
}

// The histogram of run_density_report (experiments.hpp:276-285): draws
// 0..n-1 of UniformStream(seed, 0) (counter-based, so one draw per thread)
// through the table or the exact transform, bin (int)((z + z_max) / w)
// clamped to [0, n_bins), counted in a shared-memory histogram per CTA
// (integer adds: order-independent, so the counts are exact).  Lanes past n
// evaluate a dummy draw so the warp-collective tail pass stays converged.
// A draw that rounds to u == 1 (the reference throws) records its index.
constexpr int kDensitySmemBins = 8192;
constexpr int LPMC_DENSITY_GLIBC = 1;    // LPMC_EXACT_Z_GLIBC

__global__ void density_kernel(uint64_t key, uint64_t n, const double* __restrict__ table,
                               int table_words, int K, int degree, int dyadic, int stride,
                               int simple, double tail, double z_max, double width, int n_bins,
                               int exact_z, unsigned long long* __restrict__ bins,
                               unsigned long long* __restrict__ top_index) {
  extern __shared__ __align__(16) double s_table[];
  __shared__ __align__(16) double s_math[kMathWords];
  __shared__ unsigned int s_bins[kDensitySmemBins];
  const bool local_bins = n_bins <= kDensitySmemBins;
  stage_math(s_math);
  for (int i = threadIdx.x; i < table_words; i += blockDim.x) s_table[i] = table[i];
  if (local_bins)
    for (int b = threadIdx.x; b < n_bins; b += blockDim.x) s_bins[b] = 0u;
  __syncthreads();
  const TableView t{s_table, stride, K, degree, dyadic, simple, tail};
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * blockDim.x; base < n; base += step) {
    const uint64_t i = base + threadIdx.x;
    const bool in = i < n;
    uint64_t kc = key + (in ? i : 0) * 0x94d049bb133111ebull;  // counter i (uniform.hpp:38-41)
    const uint64_t b53 = next_draw(kc);
    const double u = in ? uniform_of(b53) : 0.25;
    if (in && b53 == kTopDraw) atomicMin(top_index, static_cast<unsigned long long>(i));
    double z;
    if (table != nullptr) {
      z = approx_inv(t, u);
    } else if (exact_z == LPMC_DENSITY_GLIBC) {  // the reference's Z bit for bit
      double uu[1] = {u}, zz[1];
      glibc::inv_cdf_multi<1>(uu, zz, s_math);
      z = zz[0];
    } else {
      double uu[1] = {u}, zz[1];
      math::phi_inv_multi<1>(uu, zz, math::FlatTab{s_math});
      z = zz[0];
    }
    if (in) {
      int b = static_cast<int>(__ddiv_rn(__dadd_rn(z, z_max), width));
      b = b < 0 ? 0 : b;
      b = b >= n_bins ? n_bins - 1 : b;
      LPMC_DCHECK(b >= 0 && b < n_bins);
      if (local_bins) {
        atomicAdd(&s_bins[b], 1u);
      } else {
        atomicAdd(&bins[b], 1ull);
      }
    }
  }
  __syncthreads();
  if (local_bins)
    for (int b = threadIdx.x; b < n_bins; b += blockDim.x)
      if (s_bins[b] != 0u) atomicAdd(&bins[b], static_cast<unsigned long long>(s_bins[b]));
}

// ------------------------------------------------------ pipe peaks ---------
// Roofline denominators for this non-tensor path: many independent
// dependency chains per thread so the pipe, not latency, is the limit.
// One "op" = one lane-operation (one SASS instruction x 32 lanes / 32).
constexpr int kPeakChains = 8;
constexpr int kPeakIters = 4096;

__global__ void __launch_bounds__(256) peak_fp64_kernel(double seed, double* sink) {
  double a[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) a[c] = seed + threadIdx.x + c;
  const double m = 1.0000000001, k = 1e-9;
  for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) a[c] = __fma_rn(a[c], m, k);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s += a[c];
  if (s == 12345.678) sink[0] = s;
}

__global__ void __launch_bounds__(256) peak_fp32_kernel(float seed, float* sink) {
  float a[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) a[c] = seed + threadIdx.x + c;
  const float m = 1.0001f, k = 1e-7f;
  for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) a[c] = __fmaf_rn(a[c], m, k);
  }
  float s = 0.0f;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s += a[c];
  if (s == 12345.678f) sink[0] = s;
}

__global__ void __launch_bounds__(256) peak_half2_kernel(float seed, float* sink) {
  __half2 a[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) a[c] = __float2half2_rn(seed + 0.001f * (threadIdx.x + c));
  const __half2 m = __float2half2_rn(1.0001f), k = __float2half2_rn(1e-4f);
  for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) a[c] = __hfma2(a[c], m, k);
  }
  float s = 0.0f;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s += __low2float(a[c]) + __high2float(a[c]);
  if (s == 12345.678f) sink[0] = s;
}

__global__ void __launch_bounds__(256) peak_imad64_kernel(uint64_t seed, uint64_t* sink) {
  uint64_t a[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) a[c] = seed + threadIdx.x + c;
  for (int i = 0; i < kPeakIters / 4; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) a[c] = a[c] * 0xff51afd7ed558ccdull + 0x9e3779b97f4a7c15ull;
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s ^= a[c];
  if (s == 12345) sink[0] = s;
}

}  // namespace

int configure_kernels() {
  cudaError_t e = math::upload_math_constants();  // this TU's copy (inv_cdf_kernel)
  if (e == cudaSuccess) e = configure_level_carrier();
  if (e == cudaSuccess) e = configure_level_f32();
  if (e == cudaSuccess) e = configure_level_f32r();
  if (e == cudaSuccess) e = configure_level_f64r();
  if (e == cudaSuccess) e = configure_level_half2();
  if (e == cudaSuccess) e = configure_level_h16();
  if (e == cudaSuccess) e = configure_level_bf16();
  if (e == cudaSuccess) e = configure_probe();
  if (e == cudaSuccess) e = configure_wpp_carrier();
  if (e == cudaSuccess) e = configure_wpp_f32();
  if (e == cudaSuccess) e = configure_wpp_f32r();
  if (e == cudaSuccess) e = configure_wpp_f64r();
  return static_cast<int>(e);
}

LaunchResult launch_paths_wpp(const LevelArgs& A, BarArith arith, bool kahan, void* stream) {
  cudaError_t e = cudaErrorInvalidValue;
  switch (arith) {
    case BarArith::kCarrier: e = launch_wpp_carrier(A, kahan, stream); break;
    case BarArith::kF32: e = launch_wpp_f32(A, kahan, stream); break;
    case BarArith::kF32Round: e = launch_wpp_f32r(A, kahan, stream); break;
    case BarArith::kF64Round: e = launch_wpp_f64r(A, kahan, stream); break;
    case BarArith::kHalf2: break;  // two paths per thread: fused schedule only
  }
  return {static_cast<int>(e), 1};
}

LaunchResult launch_path_batches(const double* path_diff, uint64_t n_paths, double* batch_acc,
                                 void* stream) {
  const unsigned blocks = static_cast<unsigned>((n_paths + kBatch - 1) / kBatch);
  path_batch_kernel<<<blocks, kBatch, 0, static_cast<cudaStream_t>(stream)>>>(path_diff, n_paths,
                                                                              batch_acc);
  return {static_cast<int>(cudaGetLastError()), 1};
}

LaunchResult launch_paths(const LevelArgs& A, BarArith arith, bool kahan, bool dump,
                          void* stream) {
  cudaError_t e = cudaSuccess;
  switch (arith) {
    case BarArith::kCarrier: e = launch_level_carrier(A, kahan, dump, stream); break;
    case BarArith::kF32: e = launch_level_f32(A, kahan, dump, stream); break;
    case BarArith::kF32Round:
      // m = 10 on native binary16 (dev::ArithHalfScaled) where the host proved
      // the scales: production launches, fast exact Gaussians, dyadic-linear
      // tables or none; everything else on the fp32-carried
      // emulation, which also replays the paths that leave the native guard
      if (use_native_half(A, kahan, dump) && std::getenv("LPMC_NO_NATIVE_HALF") == nullptr) {
        e = launch_level_h16(A, kahan, stream);
      } else if (use_native_bf16(A, dump) && std::getenv("LPMC_NO_NATIVE_BF16") == nullptr) {
        e = launch_level_bf16(A, kahan, stream);  // m = 7 on native bfloat16 (dev::ArithBf16)
      } else {
        e = launch_level_f32r(A, kahan, dump, stream);
      }
      break;
    case BarArith::kF64Round: e = launch_level_f64r(A, kahan, dump, stream); break;
    case BarArith::kHalf2: e = launch_level_half2(A, kahan, dump, stream); break;
  }
  return {static_cast<int>(e), 1};
}

LaunchResult launch_chunk_reduce(const double* batch_acc, uint64_t n_batches, uint64_t n_chunks,
                                 double* chunk_acc, void* stream) {
  chunk_reduce_kernel<<<static_cast<unsigned>(n_chunks), kChunkThreads, 0,
                        static_cast<cudaStream_t>(stream)>>>(batch_acc, n_batches, chunk_acc);
  return {static_cast<int>(cudaGetLastError()), 1};
}

LaunchResult launch_sequential_batches(const double* path_diff, uint64_t n_paths,
                                       double* batch_acc, void* stream) {
  const uint64_t n_batches = (n_paths + kBatch - 1) / kBatch;
  const uint64_t threads = 3 * n_batches;
  const unsigned blocks = static_cast<unsigned>((threads + 127) / 128);
  sequential_batch_kernel<<<blocks, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      path_diff, n_paths, batch_acc);
  return {static_cast<int>(cudaGetLastError()), 1};
}

int measure_pipe_peaks(double* out4) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  void* sink = nullptr;
  cudaError_t e = cudaMalloc(&sink, 64);
  if (e != cudaSuccess) return static_cast<int>(e);
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  const unsigned blocks = static_cast<unsigned>(sms) * 8u;
  const double lanes = static_cast<double>(blocks) * 256.0;
  for (int which = 0; which < 4 && e == cudaSuccess; ++which) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(t0);
      switch (which) {
        case 0: peak_fp64_kernel<<<blocks, 256>>>(1.0, static_cast<double*>(sink)); break;
        case 1: peak_fp32_kernel<<<blocks, 256>>>(1.0f, static_cast<float*>(sink)); break;
        case 2: peak_half2_kernel<<<blocks, 256>>>(1.0f, static_cast<float*>(sink)); break;
        default: peak_imad64_kernel<<<blocks, 256>>>(1ull, static_cast<uint64_t*>(sink)); break;
      }
      cudaEventRecord(t1);
      e = cudaEventSynchronize(t1);
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, t0, t1);
      if (rep > 0 && ms < best) best = ms;  // rep 0 warms up
    }
    const double iters = which == 3 ? kPeakIters / 4 : kPeakIters;
    // lane-operations per second (one FMA = one op; half2: 2 lanes per op)
    const double ops = lanes * iters * kPeakChains * (which == 2 ? 2.0 : 1.0);
    out4[which] = ops / (best * 1e-3);
  }
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(sink);
  if (e == cudaSuccess) e = cudaGetLastError();
  return static_cast<int>(e);
}

LaunchResult launch_inv_cdf(const double* u, uint64_t n, const double* table, int K, int degree,
                            int dyadic, int stride, int simple, double tail, int op, double* out,
                            void* stream) {
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  inv_cdf_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      u, n, table, K, degree, dyadic, stride, simple, tail, op, out);
  return {static_cast<int>(cudaGetLastError()), 1};
}

LaunchResult launch_density(uint64_t key, uint64_t n, const double* table, int table_words,
                            int K, int degree, int dyadic, int stride, int simple, double tail,
                            double z_max, double width, int n_bins, int exact_z,
                            unsigned long long* bins, unsigned long long* top_index,
                            void* stream) {
  const size_t smem = table != nullptr ? static_cast<size_t>(table_words) * sizeof(double) : 0;
  if (smem > 0) {
    const cudaError_t e = cudaFuncSetAttribute(density_kernel,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return {static_cast<int>(e), 0};
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t need = (n + 255) / 256;
  const uint64_t cap = static_cast<uint64_t>(sms) * 8;
  const unsigned blocks = static_cast<unsigned>(need < cap ? (need ? need : 1) : cap);
  density_kernel<<<blocks, 256, smem, static_cast<cudaStream_t>(stream)>>>(
      key, n, table, table != nullptr ? table_words : 0, K, degree, dyadic, stride, simple, tail,
      z_max, width, n_bins, exact_z, bins, top_index);
  return {static_cast<int>(cudaGetLastError()), 1};
}

}  // namespace lpmc_b200
