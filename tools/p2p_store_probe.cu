// Calibration probe (not product code): SM-issued peer stores over NVLink.
// Every GPU streams `bytes` of 16-byte stores into its right neighbour's
// buffer (all GPUs at once, one host thread each via one process with peer
// access), optionally reading the same amount locally first (the fused
// FFT+exchange pass pattern).  Prints GB/s per GPU per direction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p2p tools/p2p_store_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
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

// TMA engine variant: thread 0 streams 32 KB cp.async.bulk stores of a
// shared-memory tile to consecutive destination chunks
__global__ void peer_bulk_store(char* __restrict__ dst, size_t bytes) {
  extern __shared__ __align__(128) char tile[];
  const size_t chunk = 32768;
  for (int i = threadIdx.x; i < (int)(chunk / 16); i += blockDim.x)
    reinterpret_cast<double2*>(tile)[i] = make_double2((double)i, 0.0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(tile));
  int inflight = 0;
  for (size_t off = (size_t)blockIdx.x * chunk; off < bytes; off += (size_t)gridDim.x * chunk) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(s),
                 "r"((uint32_t)chunk)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (++inflight >= 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void peer_store_smem(double2* __restrict__ dst, const double2* __restrict__ src, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}

// 128-byte segments at a large stride (the fused exchange pass's store
// pattern: 8 lanes x 16 B per transformed index, rows `stride` apart)
__global__ void peer_store_seg(double2* __restrict__ dst, size_t n, size_t seg_elems, size_t stride_elems) {
  const size_t nseg = n / seg_elems;
  const size_t rows = stride_elems / seg_elems;  // segments per row
  const size_t nrows = nseg / rows;
  const size_t gstride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gstride) {
    const size_t s = i / seg_elems, e = i - s * seg_elems;
    const size_t r = s % nrows, c = s / nrows;  // consecutive segments go to different rows
    dst[r * stride_elems + c * seg_elems + e] = make_double2((double)i, 0.0);
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
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    cudaFuncSetAttribute(peer_bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  }
  for (int mode = 0; mode < 5; ++mode) {
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
        double2* dst = (mode == 2 || mode == 4) ? buf[d] : buf[(d + 1) % n];
        if (mode >= 3)
          peer_bulk_store<<<148, 32, 32768>>>(reinterpret_cast<char*>(dst), bytes);
        else
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
               mode == 0   ? "peer stores"
               : mode == 1 ? "local read + peer store"
               : mode == 2 ? "local copy"
               : mode == 3 ? "TMA bulk peer stores"
                           : "TMA bulk local stores",
               bytes / (worst * 1e-3) / 1e9, n);
    }
  }
  for (int segb = 128; segb <= 2048; segb *= 4) {
    const size_t seg = segb / 16, stride = 512 * 1024 / 16;  // 512 KB between rows
    float worst = 0;
    for (int rep = 0; rep < 3; ++rep) {
      std::vector<cudaEvent_t> e0(n), e1(n);
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaDeviceSynchronize();
        cudaEventCreate(&e0[d]);
        cudaEventCreate(&e1[d]);
      }
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaEventRecord(e0[d]);
        peer_store_seg<<<148 * 4, 512>>>(buf[(d + 1) % n], elems, seg, stride);
        cudaEventRecord(e1[d]);
      }
      worst = 0;
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaEventSynchronize(e1[d]);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0[d], e1[d]);
        worst = ms > worst ? ms : worst;
      }
    }
    printf("peer stores in %d-byte segments, 512 KB row stride: %.0f GB/s per GPU\n", segb,
           bytes / (worst * 1e-3) / 1e9);
  }
  // overlap check: peer-store kernel and local-copy kernel on disjoint SM
  // halves (1 CTA per SM forced by shared memory), concurrently
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    cudaFuncSetAttribute(peer_store_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  }
  for (int g = 37; g <= 111; g += 37) {
    std::vector<cudaStream_t> s1(n), s2(n);
    std::vector<cudaEvent_t> a0(n), a1(n), b1(n);
    for (int d = 0; d < n; ++d) {
      cudaSetDevice(d);
      cudaStreamCreate(&s1[d]);
      cudaStreamCreate(&s2[d]);
      cudaEventCreate(&a0[d]);
      cudaEventCreate(&a1[d]);
      cudaEventCreate(&b1[d]);
    }
    float wa = 0, wb = 0;
    for (int rep = 0; rep < 3; ++rep) {
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaDeviceSynchronize();
      }
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaEventRecord(a0[d], s1[d]);
        cudaStreamWaitEvent(s2[d], a0[d]);
        // peer half: bytes/2 remote ; local half: bytes local read+write
        peer_store_smem<<<g, 1024, 150 * 1024, s1[d]>>>(buf[(d + 1) % n], src[d], elems / 2);
        peer_store_smem<<<148 - g, 1024, 150 * 1024, s2[d]>>>(src[d] + elems / 2, buf[d], elems / 2);
        cudaEventRecord(a1[d], s1[d]);
        cudaEventRecord(b1[d], s2[d]);
      }
      wa = wb = 0;
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaEventSynchronize(a1[d]);
        cudaEventSynchronize(b1[d]);
        float ma = 0, mb = 0;
        cudaEventElapsedTime(&ma, a0[d], a1[d]);
        cudaEventElapsedTime(&mb, a0[d], b1[d]);
        wa = ma > wa ? ma : wa;
        wb = mb > wb ? mb : wb;
      }
    }
    printf("split %d/%d SMs: peer half %.3f ms (%.0f GB/s), local half %.3f ms (%.0f GB/s r+w)\n", g, 148 - g, wa,
           bytes / 2 / (wa * 1e-3) / 1e9, wb, bytes / (wb * 1e-3) / 1e9);
  }
  // copy engine (cudaMemcpyPeerAsync, DMA) and SM pull (remote loads, local
  // stores), all GPUs at once
  for (int mode = 0; mode < 2; ++mode) {
    float worst = 0;
    for (int rep = 0; rep < 3; ++rep) {
      std::vector<cudaEvent_t> e0(n), e1(n);
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaDeviceSynchronize();
        cudaEventCreate(&e0[d]);
        cudaEventCreate(&e1[d]);
      }
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaEventRecord(e0[d]);
        if (mode == 0)
          cudaMemcpyPeerAsync(buf[(d + 1) % n], (d + 1) % n, src[d], d, bytes);
        else
          peer_store<<<148 * 4, 512>>>(buf[d], src[(d + 1) % n], elems, 1);
        cudaEventRecord(e1[d]);
      }
      worst = 0;
      for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaEventSynchronize(e1[d]);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0[d], e1[d]);
        worst = ms > worst ? ms : worst;
      }
    }
    printf("%s: %.0f GB/s per GPU (%d GPUs concurrently)\n",
           mode == 0 ? "copy engine (cudaMemcpyPeerAsync)" : "SM pull (remote loads, local stores)",
           bytes / (worst * 1e-3) / 1e9, n);
  }
  return 0;
}
