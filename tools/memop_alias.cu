// Diagnostic: does a cuStreamWaitValue32 on one stream block work queued on
// another stream of the same context?  For each pair (stream 0 waits on a
// flag, stream k writes it with a kernel) report whether the wait is released
// within 2 s.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <unistd.h>

__global__ void set_flag(unsigned* f, unsigned v) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 40;
  cudaSetDevice(0);
  unsigned* flag;
  cudaMalloc(&flag, 4 * n);
  cudaMemset(flag, 0, 4 * n);
  cudaStream_t* s = new cudaStream_t[n];
  for (int i = 0; i < n; ++i) cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking);
  int bad = 0;
  for (int k = 1; k < n; ++k) {
    // stream 0 waits for flag[k] >= 1, then stream k sets it (enqueued after the wait)
    CUresult rc = cuStreamWaitValue32((CUstream)s[0], (CUdeviceptr)(flag + k), 1, CU_STREAM_WAIT_VALUE_GEQ);
    if (rc != CUDA_SUCCESS) { printf("wait failed %d\n", rc); return 1; }
    set_flag<<<1, 1, 0, s[k]>>>(flag + k, 1);
    auto t0 = std::chrono::steady_clock::now();
    bool done = false;
    while (std::chrono::steady_clock::now() - t0 < std::chrono::seconds(2)) {
      if (cudaStreamQuery(s[0]) == cudaSuccess) { done = true; break; }
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if (!done) {
      printf("stream %d: BLOCKED behind stream 0's wait\n", k);
      ++bad;
      fflush(stdout);
      _exit(2);  // the context is wedged; stop here
    }
  }
  printf("all %d streams independent of stream 0's wait (CUDA_DEVICE_MAX_CONNECTIONS=%s)\n", n - 1,
         getenv("CUDA_DEVICE_MAX_CONNECTIONS") ? getenv("CUDA_DEVICE_MAX_CONNECTIONS") : "unset");
  return bad;
}
