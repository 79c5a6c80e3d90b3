// tcgen05.mma (cta_group::1, bf16 -> f32) issue-rate micro-benchmark: K-major
// vs MN-major A / B smem operands (SWIZZLE_128B), and A from TMEM, at the
// attention backward's shapes (M 128, N 64 / 128, K 16 per instruction).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2007_01045_b200/csrc/kernels tools/micro/mma_major.cu -o tools/micro/mma_major
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"

using namespace dpl;

// mode: 0 A K-major, 1 A MN-major, 2 A from TMEM;  b_mn: B MN-major
__global__ void mma_rate(long long* out, int iters, int n, int mode, int b_mn) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc<512>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  long long t = 0;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_addr(smem), b = ptx::smem_addr(smem + 32768);
    const uint32_t idesc = ptx::idesc_bf16_f32(128, n, mode == 1, b_mn != 0);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        // K step k: K-major operands advance 32 bytes inside the 128-byte row
        // (k & 3) and 16 KB per 64-wide half (k >> 2); MN-major ones advance
        // 16 rows of 128 bytes
        const uint32_t a_k = mode == 1 ? k * 16 * 128 : (k >> 2) * 16384 + (k & 3) * 32;
        const uint32_t b_k = b_mn ? k * 16 * 128 : (k >> 2) * 16384 + (k & 3) * 32;
        const uint64_t bd = ptx::smem_desc_sw128(b + b_k, b_mn ? 16384 : 16, 1024);
        if (mode == 2) {
          ptx::mma_bf16_ts(tmem, tmem + 256 + k * 8, bd, idesc, 1);
        } else {
          const uint64_t ad = ptx::smem_desc_sw128(a + a_k, mode == 1 ? 16384 : 16, 1024);
          ptx::mma_bf16(tmem, ad, bd, idesc, 1);
        }
      }
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    t = clock64() - t0;
    out[blockIdx.x] = t;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

__device__ __forceinline__ void mma_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc)
      : "memory");
}

// the whole warp runs the issue loop (uniform operands, no per-lane waterfall)
// and one elected lane issues each MMA
__global__ void mma_rate_warp(long long* out, int iters, int n) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc<512>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint32_t a = ptx::smem_addr(smem), b = ptx::smem_addr(smem + 32768);
    const uint32_t idesc = ptx::idesc_bf16_f32(128, n, false, false);
    const uint64_t ad0 = ptx::smem_desc_sw128(a, 16, 1024), bd0 = ptx::smem_desc_sw128(b, 16, 1024);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t off = static_cast<uint64_t>(((k >> 2) * 16384 + (k & 3) * 32) >> 4);
        mma_elect(tmem, ad0 + off, bd0 + off, idesc);
      }
    }
    if (ptx::lane_id() == 0) {
      ptx::mma_commit(&bar);
      ptx::mbar_wait(&bar, 0);
      out[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const char* names[] = {"A K-major ", "A MN-major", "A TMEM    "};
  const int iters = 512;
  for (int n : {64, 128}) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int bmn = 0; bmn < 2; ++bmn) {
        mma_rate<<<148, 128, 70000>>>(d, iters, n, mode, bmn);
        mma_rate<<<148, 128, 70000>>>(d, iters, n, mode, bmn);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double cyc = 0;
        for (int i = 0; i < 148; ++i) cyc += h[i];
        cyc /= 148;
        const double per = cyc / (iters * 8.0);
        printf("N %3d %s B %s: %6.1f cycles / MMA (floor %d)  %.0f flop/cycle/SM\n", n, names[mode],
               bmn ? "MN-major" : "K-major ", per, 128 * n / 256, 2.0 * 128 * n * 16 / per);
      }
    }
  }
  cudaFuncSetAttribute(mma_rate_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int n : {64, 128, 256}) {
    mma_rate_warp<<<148, 128, 70000>>>(d, iters, n);
    mma_rate_warp<<<148, 128, 70000>>>(d, iters, n);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < 148; ++i) cyc += h[i];
    cyc /= 148;
    const double per = cyc / (iters * 8.0);
    printf("warp-uniform elect issue, N %3d: %6.1f cycles / MMA (floor %d)  %.0f flop/cycle/SM\n", n, per, 128 * n / 256,
           2.0 * 128 * n * 16 / per);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
