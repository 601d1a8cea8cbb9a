// Probe: cycles per tcgen05.mma (kind::f16, M=128, K=16) vs N, SS and TS forms.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate.cu -I../../include
#include <cstdio>
#include "../../paper_2601_15013_b200/csrc/common.cuh"
using namespace rdx;
int rdx::set_cuda_error(cudaError_t) { return 1; }
int rdx::num_sms() { return 148; }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) { return umma_sdesc_sw128(saddr); }
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&holder, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = holder;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = a + 16384;
    constexpr uint32_t idesc = umma_idesc_bf16(128, N);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (TS) umma_ts(tmem + 256, tmem + k * 8, sdesc(b) + 2 * k, idesc, 1u);
        else umma_bf16(tmem + 256, sdesc(a) + 2 * k, sdesc(b) + 2 * k, idesc, 1u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool TS>
void run(const char* name, long long* d, int ctas) {
  const int iters = 2000;
  cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 32768 + 1024);
  probe<N, TS><<<ctas, 128, 16384 + 32768 + 1024>>>(d, iters);
  probe<N, TS><<<ctas, 128, 16384 + 32768 + 1024>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < ctas; ++i) avg += h[i]; avg /= ctas;
  const double per = avg / (iters * 4.0);
  printf("%-8s N=%3d ctas=%3d: %.1f cycles/MMA  -> %.0f FLOP/clk/SM (dense peak ~8192)\n", name, N, ctas, per,
         2.0 * 128 * N * 16 / per);
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 148);
  for (int ctas : {1, 148}) {
    run<64, false>("SS", d, ctas);
    run<128, false>("SS", d, ctas);
    run<256, false>("SS", d, ctas);
    run<128, true>("TS", d, ctas);
    run<256, true>("TS", d, ctas);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
