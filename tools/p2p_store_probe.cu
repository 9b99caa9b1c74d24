// Calibration probe (not product code): SM-issued peer stores over NVLink.
// Every GPU streams `bytes` of 16-byte stores into its right neighbour's
// buffer (all GPUs at once, one host thread each via one process with peer
// access), optionally reading the same amount locally first (the fused
// FFT+exchange pass pattern).  Prints GB/s per GPU per direction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p2p tools/p2p_store_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void peer_store(double2* __restrict__ dst, const double2* __restrict__ src, size_t n,
                           int read_local) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v = read_local ? src[i] : make_double2((double)i, 0.0);
    dst[i] = v;
  }
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) {
    printf("need 2+ GPUs\n");
    return 0;
  }
  const size_t bytes = 512ull << 20;
  const size_t elems = bytes / sizeof(double2);
  std::vector<double2*> buf(n), src(n);
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    for (int e = 0; e < n; ++e)
      if (e != d) cudaDeviceEnablePeerAccess(e, 0);
    cudaMalloc(&buf[d], bytes);
    cudaMalloc(&src[d], bytes);
    cudaMemset(src[d], 0, bytes);
  }
  for (int mode = 0; mode < 3; ++mode) {
    // mode 0: pure peer stores; 1: local read + peer store; 2: local read + local store
    std::vector<cudaEvent_t> e0(n), e1(n);
    for (int rep = 0; rep < 3; ++rep) {
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaDeviceSynchronize();
      }
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaEventCreate(&e0[d]);
        cudaEventCreate(&e1[d]);
        cudaEventRecord(e0[d]);
        double2* dst = mode == 2 ? buf[d] : buf[(d + 1) % n];
        peer_store<<<148 * 4, 512>>>(dst, src[d], elems, mode >= 1);
        cudaEventRecord(e1[d]);
      }
      float worst = 0;
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaEventSynchronize(e1[d]);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0[d], e1[d]);
        worst = ms > worst ? ms : worst;
      }
      if (rep == 2)
        printf("%s: %.0f GB/s per GPU (%d GPUs concurrently)\n",
               mode == 0 ? "peer stores" : mode == 1 ? "local read + peer store" : "local copy",
               bytes / (worst * 1e-3) / 1e9, n);
    }
  }
  return 0;
}
