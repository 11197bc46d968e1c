// Microbenchmark: tcgen05.mma kind::i8 issue rate on sm_100a with the
// operand layouts of fused_eval_tc_kernel (A = u8 MN-major no-swizzle, B = u8
// K-major no-swizzle, both in SMEM; D = s32 in TMEM).  One CTA per SM, one
// elected thread issues R MMAs of M=128 x N x K=32, committing every 16.
// Reports clk per MMA (SM clock) for N = 32, 64, 128, 256, and the same with
// the B operand re-pointed per MMA (as the kernel's 10 limb pairs do).
// Not part of the product: grounds DESIGN.md's tensor-pipe model.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_umma tools/ubench_umma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_u8(uint32_t n) {
  return (2u << 4) | (1u << 15) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

template <int N, int VARY>
__global__ void __launch_bounds__(128, 1) k_umma(int reps, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 16384 + 4 * N * 32; i += blockDim.x) smem[i] = uint8_t(i * 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 16384);
    const uint32_t idesc = idesc_u8(N);
    const uint32_t b_lbo = (N / 8) * 128;
    uint32_t phase = 0;
    t0 = clock64();
    for (int r = 0; r < reps; r += 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t boff = VARY ? (j & 3) * (N * 32) : 0;
        const uint64_t ad = desc(a0 + (j & 3) * 1024u, 4096u, 128u);
        const uint64_t bd = desc(b0 + boff, b_lbo, 128u);
        const uint32_t d = tmem + ((j & 3) * N) % 512;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&bar)));
      asm volatile(
          "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
              smem_u32(&bar)),
          "r"(phase));
      phase ^= 1;
    }
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int VARY>
void run(int nsm) {
  unsigned long long *d;
  cudaMalloc(&d, nsm * 8);
  const int reps = 16384;
  const int smem = 16384 + 4 * N * 32 + 1024;
  cudaFuncSetAttribute(k_umma<N, VARY>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_umma<N, VARY><<<nsm, 128, smem>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("N=%d err %s\n", N, cudaGetErrorString(e)); return; }
  unsigned long long h[256];
  cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  printf("M=128 N=%3d K=32 i8 SS no-swizzle vary_b=%d: %.1f clk/MMA  (%.0f MAC/clk/SM)\n", N, VARY, avg / reps,
         128.0 * N * 32 / (avg / reps));
  cudaFree(d);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  run<32, 0>(nsm); run<64, 0>(nsm); run<128, 0>(nsm); run<256, 0>(nsm);
  run<64, 1>(nsm); run<128, 1>(nsm);
  run<64, 0>(1); run<128, 0>(1);
  return 0;
}
