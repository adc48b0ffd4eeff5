// k_peaks.cu -- measured denominators of the K3 roofline ("Measure a
// DADD/DMUL throughput microbenchmark at the run's clock and use that"): the sustained
// rate of independent FP64 DADD/DMUL instructions and of 32-bit integer LOP3/IADD3 ALU
// instructions on this GPU, each from a kernel of many independent dependency chains per
// thread at full occupancy, timed with CUDA events.
#include <cstdio>

#include "pipette_dev.cuh"

namespace pip {

constexpr int kPeakIters = 4096, kPeakChains = 8;

__global__ void __launch_bounds__(256) k_peak_fp64(double* out, double seed) {
  double a[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) a[c] = seed + threadIdx.x + c;
  const double m = 1.0000001, d = 1e-9;
  for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) a[c] = __dadd_rn(__dmul_rn(a[c], m), d);   // DMUL + DADD
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s += a[c];
  if (s == 12345.678) out[0] = s;   // never true; keeps the chains alive
}

__global__ void __launch_bounds__(256) k_peak_alu(uint32_t* out, uint32_t seed) {
  uint32_t a[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) a[c] = seed + threadIdx.x * 7u + c;
  for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) a[c] = ((a[c] ^ 0x9E3779B9u) & 0x7fffffffu) | (a[c] >> 3);   // LOP3 + SHF
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s ^= a[c];
  if (s == 0x12345678u) out[0] = s;
}

// Shared-memory bandwidth: every warp streams 64-bit loads from a conflict-free 16 KB
// block buffer (lane-interleaved, so one LDS.64 moves 256 B), 8 independent loads per
// thread per iteration.
constexpr int kSmemIters = 2048;
__global__ void __launch_bounds__(256) k_peak_smem(double* out) {
  __shared__ double buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = (double)i;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = 0.0;
  uint32_t off = (uint32_t)(w * 256 + lane);
  for (int i = 0; i < kSmemIters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = __dadd_rn(acc[c], buf[(off + (uint32_t)c * 32u) & 2047u]);
    off += 8u * 32u + 64u;   // stays lane-interleaved (multiple of 32): conflict free
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

}  // namespace pip

extern "C" pipette_status pipette_measure_smem_bw(int32_t device, double* bytes_per_s) {
  using namespace pip;
  if (cudaSetDevice(device) != cudaSuccess) return PIPETTE_E_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  void* buf = nullptr;
  if (cudaMalloc(&buf, 64) != cudaSuccess) return PIPETTE_E_CUDA;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256;
  const double bytes = (double)blocks * threads * kSmemIters * 8 * 8.0;
  float best = 1e30f;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a);
    k_peak_smem<<<blocks, threads>>>((double*)buf);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0) best = ms < best ? ms : best;
  }
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  if (e != cudaSuccess) return PIPETTE_E_CUDA;
  if (bytes_per_s) *bytes_per_s = bytes / (best * 1e-3);
  return PIPETTE_OK;
}

extern "C" pipette_status pipette_measure_peaks(int32_t device, double* fp64_ops_per_s, double* alu_ops_per_s) {
  using namespace pip;
  if (cudaSetDevice(device) != cudaSuccess) return PIPETTE_E_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  void* buf = nullptr;
  if (cudaMalloc(&buf, 64) != cudaSuccess) return PIPETTE_E_CUDA;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256;   // 64 warps per SM
  const double ops = (double)blocks * threads * kPeakIters * kPeakChains * 2.0;
  float best64 = 1e30f, bestalu = 1e30f;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a);
    k_peak_fp64<<<blocks, threads>>>((double*)buf, 1.0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0) best64 = ms < best64 ? ms : best64;
    cudaEventRecord(a);
    k_peak_alu<<<blocks, threads>>>((uint32_t*)buf, 3u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0) bestalu = ms < bestalu ? ms : bestalu;
  }
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  if (e != cudaSuccess) return PIPETTE_E_CUDA;
  if (fp64_ops_per_s) *fp64_ops_per_s = ops / (best64 * 1e-3);
  if (alu_ops_per_s) *alu_ops_per_s = ops / (bestalu * 1e-3);
  return PIPETTE_OK;
}
