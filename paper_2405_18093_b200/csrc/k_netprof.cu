// k_netprof.cu -- NEXT-3: Alg.1 l.1 "network_profile()" on
// the GPUs of one B200 box.  The paper profiled node pairs with mpiGraph over 40 days
// (Fig.3); here every ordered pair (i, j) of local GPUs is timed with an
// SM-driven copy kernel on GPU i that PUSHES a buffer into GPU j's memory over NVLink 5 /
// NVSwitch (peer stores; 16-byte vectors, grid = 2 x SMs), and the diagonal with the
// same kernel inside GPU i (HBM to HBM).  Bandwidth = bytes / median device time of
// `reps` launches (CUDA events on GPU i's stream).  The result is a directed n x n
// bytes/s matrix in the layout pipette_init takes (diagonal = intra bandwidth, R5), for a
// cluster of n "nodes" of one GPU each (tp = 1).
#include <algorithm>
#include <cstdio>
#include <vector>

#include "pipette_dev.cuh"

namespace pip {

__global__ void __launch_bounds__(512) k_push_copy(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {   // four independent 16-byte copies in flight
    const uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
                d = __ldcs(src + i + 3 * stride);
    __stcs(dst + i, a);
    __stcs(dst + i + stride, b);
    __stcs(dst + i + 2 * stride, c);
    __stcs(dst + i + 3 * stride, d);
  }
  for (; i < n; i += stride) __stcs(dst + i, __ldcs(src + i));
}

}  // namespace pip

#define NP_CU(x)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      std::snprintf(err, err_cap, "%s: %s", #x, cudaGetErrorString(e_));                  \
      return PIPETTE_E_CUDA;                                                              \
    }                                                                                     \
  } while (0)

namespace pip {
// Host driver of the profile (called by pipette_profile_bandwidth in host.cu).
pipette_status netprof_run(int n, const int* devs, size_t bytes, int reps, double* bw, double* ms_out, char* err,
                           size_t err_cap) {
  bytes = (bytes + 15) & ~(size_t)15;
  const size_t n16 = bytes / 16;
  std::vector<void*> src(n), dst(n);
  std::vector<cudaStream_t> st(n);
  int prev = 0;
  cudaGetDevice(&prev);
  for (int i = 0; i < n; ++i) {
    NP_CU(cudaSetDevice(devs[i]));
    NP_CU(cudaMalloc(&src[i], bytes));
    NP_CU(cudaMalloc(&dst[i], bytes));
    NP_CU(cudaMemset(src[i], i + 1, bytes));
    NP_CU(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      int can = 0;
      NP_CU(cudaDeviceCanAccessPeer(&can, devs[i], devs[j]));
      if (!can) {
        std::snprintf(err, err_cap, "GPU %d cannot access GPU %d (no peer path)", devs[i], devs[j]);
        return PIPETTE_E_UNSUPPORTED;
      }
      cudaError_t e = cudaDeviceEnablePeerAccess(devs[j], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) NP_CU(e);
      cudaGetLastError();
    }
  }
  for (int i = 0; i < n; ++i) {
    NP_CU(cudaSetDevice(devs[i]));
    int sms = 0;
    NP_CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, devs[i]));
    cudaEvent_t a, b;
    NP_CU(cudaEventCreate(&a));
    NP_CU(cudaEventCreate(&b));
    for (int j = 0; j < n; ++j) {
      std::vector<float> t;
      for (int r = 0; r < reps + 2; ++r) {   // two untimed warm-ups
        NP_CU(cudaEventRecord(a, st[i]));
        k_push_copy<<<2 * sms, 512, 0, st[i]>>>((uint4*)dst[j], (const uint4*)src[i], n16);
        NP_CU(cudaGetLastError());
        NP_CU(cudaEventRecord(b, st[i]));
        NP_CU(cudaEventSynchronize(b));
        float ms = 0.f;
        NP_CU(cudaEventElapsedTime(&ms, a, b));
        if (r >= 2) t.push_back(ms);
      }
      std::sort(t.begin(), t.end());
      const double med = t[t.size() / 2];
      // the diagonal copy reads and writes HBM of one GPU: count the bytes once, like a
      // transfer (the model's intra-node B is a transfer bandwidth)
      bw[i * n + j] = (double)bytes / (med * 1e-3);
      if (ms_out) ms_out[i * n + j] = med;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  for (int i = 0; i < n; ++i) {
    cudaSetDevice(devs[i]);
    cudaFree(src[i]);
    cudaFree(dst[i]);
    cudaStreamDestroy(st[i]);
  }
  cudaSetDevice(prev);
  return PIPETTE_OK;
}
}  // namespace pip
