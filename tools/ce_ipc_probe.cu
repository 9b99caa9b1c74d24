// Calibration probe (not product code): copy-engine rate into memory owned
// by ANOTHER process (CUDA IPC mapping, as in a multi-process dfftb world):
// at a given offset in a large region (argv[1]; a dfftb region puts its flag
// page first), one direction, then both processes pushing to each other at once, with a
// contiguous and a 2-D shape, optionally beside a kernel spinning on
// ld.acquire.sys (a sync-point wait) on a flag page in the same region.  Build:
//   nvcc -std=c++20 -O2 -gencode arch=compute_100a,code=sm_100a -o tools/ce_ipc_probe tools/ce_ipc_probe.cu
#include <cuda_runtime.h>
#include <sys/wait.h>
#include <unistd.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void spin(const unsigned long long* f, long long ns) {
  const long long t0 = clock64();
  unsigned long long v = 0;
  while (clock64() - t0 < ns) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
    __nanosleep(64);
  }
  if (v == 12345) printf("x");
}

struct Pipe { int fd[2]; };

static void xfer(int wfd, const void* p, size_t n) { if (write(wfd, p, n) != (ssize_t)n) exit(2); }
static void recv(int rfd, void* p, size_t n) { if (read(rfd, p, n) != (ssize_t)n) exit(2); }

static size_t g_off = 32768;

static void worker(int dev, int peer_dev, int rfd, int wfd, bool print) {
  const size_t bytes = 1ull << 30, payload = 512ull << 20;
  CK(cudaSetDevice(dev));
  void *src, *peer;
  CK(cudaMalloc(&src, bytes));
  const size_t flags_bytes = g_off;  // offset of the copy destination in the region
  char* region;
  CK(cudaMalloc(&region, flags_bytes + 4 * bytes));
  unsigned long long* flag = reinterpret_cast<unsigned long long*>(region);
  CK(cudaMemset(flag, 0, 8));
  cudaIpcMemHandle_t mine, theirs;
  CK(cudaIpcGetMemHandle(&mine, region));
  xfer(wfd, &mine, sizeof(mine));
  recv(rfd, &theirs, sizeof(theirs));
  CK(cudaIpcOpenMemHandle(&peer, theirs, cudaIpcMemLazyEnablePeerAccess));
  peer = static_cast<char*>(peer) + flags_bytes;
  cudaError_t pe = cudaDeviceEnablePeerAccess(peer_dev, 0);
  (void)pe;
  cudaGetLastError();
  cudaStream_t s, k;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&k, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaMemcpy(peer, src, payload, cudaMemcpyDefault));
  auto run = [&](const char* what, bool both, int shape, bool spinning) {
    char c = 0;
    // rendezvous so both processes start together
    xfer(wfd, &c, 1);
    recv(rfd, &c, 1);
    const bool active = both || dev == 0;
    if (spinning) spin<<<1, 32, 0, k>>>(flag, 2000000000ll);
    CK(cudaEventRecord(e0, s));
    if (active)
      for (int i = 0; i < 8; ++i) {
        if (shape == 0) CK(cudaMemcpyAsync(peer, src, payload, cudaMemcpyDefault, s));
        else CK(cudaMemcpy2DAsync(peer, 8192, src, 8192, 2048, (bytes / 8192), cudaMemcpyDefault, s));
      }
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= 8;
    const double moved = shape ? (double)(bytes / 8192) * 2048 : (double)payload;  // 2-D: 256 MiB
    if (print && active)
      printf("%s, %s%s: %.3f ms per copy  %.0f GB/s\n", what, shape ? "2-D 2 KiB rows pitch 8 KiB, 256 MiB" : "contiguous 512 MiB",
             spinning ? ", acquire-spin kernel running" : "", ms, moved / ms / 1e6);
    CK(cudaDeviceSynchronize());
  };
  for (int shape = 0; shape < 2; ++shape) {
    run("one direction", false, shape, false);
    run("both directions", true, shape, false);
  }
  run("both directions", true, 0, true);
  run("both directions", true, 1, true);
  char c = 0;
  xfer(wfd, &c, 1);
  recv(rfd, &c, 1);
}

int main(int argc, char** argv) {
  if (argc > 1) g_off = strtoull(argv[1], nullptr, 0);
  printf("destination offset in the region: %zu B\n", g_off);
  fflush(stdout);
  Pipe a, b;
  if (pipe(a.fd) || pipe(b.fd)) return 1;
  pid_t pid = fork();
  if (pid == 0) {
    worker(1, 0, a.fd[0], b.fd[1], false);
    return 0;
  }
  worker(0, 1, b.fd[0], a.fd[1], true);
  int st;
  waitpid(pid, &st, 0);
  return 0;
}
