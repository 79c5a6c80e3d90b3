// TMEM read bandwidth / latency micro-benchmark (tcgen05.ld.32x32b.x32 +
// wait::ld), and MUFU.EX2 throughput, per SM on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2007_01045_b200/csrc/kernels tools/micro/tmem_bw.cu -o tools/micro/tmem_bw -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include "ptx.cuh"

using namespace dpl;

template <int kWarps, bool kOverlap>
__global__ void tmem_read(long long* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc<512>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t trow = ((warp & 3) * 32) << 16;
  const uint32_t col0 = (warp >> 2) * 32;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t v[32];
    ptx::tmem_ld_32x32b_x32(tmem + trow + ((col0 + i * 64) & 511), v);
    if (kOverlap) {
      uint32_t w[32];
      ptx::tmem_ld_32x32b_x32(tmem + trow + ((col0 + i * 64 + 256) & 511), w);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += v[e] ^ w[e];
    } else {
      ptx::tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += v[e];
    }
  }
  const long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678) out[0] = 0;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

__global__ void mufu(long long* out, int iters, float seed) {
  float x[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) x[e] = seed * (threadIdx.x + e);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int e = 0; e < 8; ++e) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[e]));
  }
  const long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  float s = 0;
  for (int e = 0; e < 8; ++e) s += x[e];
  if (s == 1234.5f) out[0] = 0;
}

__global__ void mufu_bf16x2(long long* out, int iters, float seed) {
  uint32_t x[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    __nv_bfloat162 h = __floats2bfloat162_rn(-seed * (threadIdx.x + e), -seed * e);
    x[e] = *reinterpret_cast<uint32_t*>(&h);
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int e = 0; e < 8; ++e) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x[e]));
  }
  const long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  uint32_t s = 0;
  for (int e = 0; e < 8; ++e) s ^= x[e];
  if (s == 12345u) out[0] = 0;
}

__global__ void mufu_f16x2(long long* out, int iters, float seed) {
  uint32_t x[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    __half2 h = __floats2half2_rn(-seed * (threadIdx.x + e), -seed * e);
    x[e] = *reinterpret_cast<uint32_t*>(&h);
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int e = 0; e < 8; ++e) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[e]));
  }
  const long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  uint32_t s = 0;
  for (int e = 0; e < 8; ++e) s ^= x[e];
  if (s == 12345u) out[0] = 0;
}

template <typename K>
void run(const char* name, K kernel, int threads, int iters, double bytes_per_warp_iter) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  kernel<<<148, threads>>>(d, iters);
  kernel<<<148, threads>>>(d, iters);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += h[i];
  cyc /= 148;
  const int warps = threads / 32;
  printf("%-28s warps %2d  %8.1f cycles/iter  %7.1f B/cycle/SM\n", name, warps, cyc / iters,
         bytes_per_warp_iter * warps * iters / cyc);
  cudaFree(d);
}

int main() {
  const int it = 4096;
  run("ld x32 (1 in flight)", tmem_read<1, false>, 32, it, 4096);
  run("ld x32 (1 in flight)", tmem_read<4, false>, 128, it, 4096);
  run("ld x32 (1 in flight)", tmem_read<8, false>, 256, it, 4096);
  run("ld x32 (1 in flight)", tmem_read<16, false>, 512, it, 4096);
  run("ld x32 (2 in flight)", tmem_read<4, true>, 128, it, 8192);
  run("ld x32 (2 in flight)", tmem_read<8, true>, 256, it, 8192);
  run("ld x32 (2 in flight)", tmem_read<16, true>, 512, it, 8192);
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  for (int threads : {32, 128, 256, 512}) {
    mufu<<<148, threads>>>(d, 1024, 1e-3f);
    mufu<<<148, threads>>>(d, 1024, 1e-3f);
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < 148; ++i) cyc += h[i];
    cyc /= 148;
    printf("ex2 threads %3d: %.2f ex2/cycle/SM\n", threads, threads * 8.0 * 1024 / cyc);
  }
  for (int threads : {128, 256, 512}) {
    for (int kind = 0; kind < 2; ++kind) {
      if (kind == 0) mufu_bf16x2<<<148, threads>>>(d, 1024, 1e-3f), mufu_bf16x2<<<148, threads>>>(d, 1024, 1e-3f);
      else mufu_f16x2<<<148, threads>>>(d, 1024, 1e-3f), mufu_f16x2<<<148, threads>>>(d, 1024, 1e-3f);
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < 148; ++i) cyc += h[i];
      cyc /= 148;
      printf("ex2 %s threads %3d: %.2f results/cycle/SM\n", kind ? "f16x2" : "bf16x2", threads, threads * 16.0 * 1024 / cyc);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
