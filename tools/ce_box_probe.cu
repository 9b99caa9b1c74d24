// Calibration probe (not product code): copy-engine peer-copy rate GPU0 ->
// GPU1 for the box shapes a staged exchange issues: contiguous, 2-D (rows of
// R bytes, pitch P), and 3-D (slices of 2-D).  Build:
//   nvcc -O2 -o tools/ce_box_probe tools/ce_box_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

static float time_it(cudaStream_t s, int reps, auto&& fn) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  fn();
  CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(a, s));
  for (int i = 0; i < reps; ++i) fn();
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  const size_t bytes = 1ull << 30;
  void *src, *dst;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&dst, bytes));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&src, bytes));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t payload = 128ull << 20;  // one chunk of a 512^3 fp64 N=2 exchange
  {
    float ms = time_it(s, 10, [&] { CK(cudaMemcpyAsync(dst, src, payload, cudaMemcpyDefault, s)); });
    printf("contiguous %zu MiB: %.3f ms  %.0f GB/s\n", payload >> 20, ms, payload / ms / 1e6);
  }
  for (size_t row : {1024, 2048, 4096, 8192, 65536}) {
    for (size_t pitchmul : {2, 4}) {
      const size_t pitch = row * pitchmul;
      const size_t h = payload / row;
      if (h * pitch > bytes) continue;
      float ms = time_it(s, 10, [&] { CK(cudaMemcpy2DAsync(dst, pitch, src, pitch, row, h, cudaMemcpyDefault, s)); });
      printf("2-D rows %6zu B pitch %6zu B x %7zu: %.3f ms  %.0f GB/s\n", row, pitch, h, ms, payload / ms / 1e6);
    }
  }
  // 3-D: slices of (rows x row bytes), as the [x1][x0][x2] receiver layout gives
  for (size_t row : {2048, 4096}) {
    const size_t pitch = 8192, rows = 256, ysize = 512;
    const size_t slices = payload / (row * rows);
    if (slices * ysize * pitch > bytes) continue;
    cudaMemcpy3DParms m{};
    m.srcPtr = make_cudaPitchedPtr(src, pitch, pitch, ysize);
    m.dstPtr = make_cudaPitchedPtr(dst, pitch, pitch, ysize);
    m.extent = make_cudaExtent(row, rows, slices);
    m.kind = cudaMemcpyDefault;
    float ms = time_it(s, 5, [&] { CK(cudaMemcpy3DAsync(&m, s)); });
    printf("3-D rows %zu B x %zu rows x %zu slices: %.3f ms  %.0f GB/s\n", row, rows, slices, ms, payload / ms / 1e6);
    m.srcPtr = make_cudaPitchedPtr(src, pitch, pitch, ysize);
    cudaMemcpy3DPeerParms pp{};
    pp.srcPtr = m.srcPtr;
    pp.dstPtr = m.dstPtr;
    pp.srcDevice = 0;
    pp.dstDevice = 1;
    pp.extent = m.extent;
    ms = time_it(s, 5, [&] { CK(cudaMemcpy3DPeerAsync(&pp, s)); });
    printf("3-D peer rows %zu B x %zu rows x %zu slices: %.3f ms  %.0f GB/s\n", row, rows, slices, ms,
           payload / ms / 1e6);
  }
  return 0;
}
