// Microbenchmark: how must an SM issue cp.async.bulk (TMA bulk copies) to
// stream a 1 GiB table at the HBM roof?  The small-batch regime of the fused
// kernel (B = 1..8) is a table stream through a T ring of bulk-copy entries;
// r01 measured it at 2.6-3.0 TB/s.  Here one loader warp per CTA streams its
// share of the table through an NST-deep ring of S-byte entries (a "consumer"
// warp releases each entry as soon as it lands, touching one word), for
// several (S, NST, copies per entry, CTAs per SM).  Reference: an LDG.128
// grid-stride read with all warps.  Not part of the product.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubs tools/ubench_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// grid-stride over entries of S bytes; entry e of CTA c = global entry c + e * grid
__global__ void k_bulk(const uint8_t *__restrict__ src, uint64_t n_entries, uint32_t S, uint32_t NST, uint32_t NCP,
                       uint32_t *sink, uint64_t wrap = ~0ull) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem), *empty = full + 16;
  uint8_t *buf = smem + 256;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t acc = 0;
  if (warp == 0) {  // loader
    uint32_t seq = 0;
    for (uint64_t e = blockIdx.x; e < n_entries; e += gridDim.x, ++seq) {
      const uint32_t s = seq % NST, use = seq / NST;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      if (lane == 0) mbar_expect_tx(&full[s], S);
      __syncwarp();
      const uint32_t part = S / NCP;
      if (lane < NCP) bulk_g2s(buf + s * S + lane * part, src + (e % wrap) * S + lane * part, part, &full[s]);
    }
  } else if (warp == 1) {  // consumer: touch one word, release
    uint32_t seq = 0;
    for (uint64_t e = blockIdx.x; e < n_entries; e += gridDim.x, ++seq) {
      const uint32_t s = seq % NST, use = seq / NST;
      mbar_wait(&full[s], use & 1);
      acc += reinterpret_cast<const uint32_t *>(buf + s * S)[lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// Cluster of 2 CTAs (2 SMs): entry e of the pair's sequence is issued by CTA
// e % 2 with .multicast::cluster into both CTAs' ring slot; each slot is
// re-armed by its issuer once both CTAs' consumers released it (remote
// arrive on the issuer's empty barrier).  Delivered bytes = 2 x the bytes
// read: does one bulk copy feeding two SMs lift the per-SM ingest ceiling?
__global__ void __cluster_dims__(2, 1, 1) k_bulk_mc(const uint8_t *__restrict__ src, uint64_t n_entries, uint32_t S,
                                                    uint32_t NST, uint32_t *sink, uint64_t wrap) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem), *empty = full + 16;
  uint8_t *buf = smem + 256;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 2); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const uint32_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  uint32_t acc = 0;
  if (warp == 0 && lane == 0) {  // loader: arm this CTA's full barrier for every entry; issue its own half
    uint32_t seq = 0;
    for (uint64_t e = pair; e < n_entries; e += npairs, ++seq) {
      const uint32_t s = seq % NST, use = seq / NST;
      if ((seq & 1) == rank && use > 0) {  // own slot: both CTAs released it
        asm volatile("{\n\t.reg .pred p;\nMW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra MW_%=;\n}"
                     ::"r"(smem_u32(&empty[s])), "r"((use - 1) & 1) : "memory");
      }
      if ((seq & 1) != rank && use > 0)  // peer's slot: re-arm full only after its previous phase completed
        mbar_wait(&full[s], (use - 1) & 1);
      mbar_expect_tx(&full[s], S);
      if ((seq & 1) == rank)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                     ::"r"(smem_u32(buf + s * S)), "l"(src + (e % wrap) * S), "r"(S), "r"(smem_u32(&full[s])), "h"(uint16_t(3))
                     : "memory");
    }
  } else if (warp == 1) {  // consumer: touch one word, release to the slot's issuer
    uint32_t seq = 0;
    for (uint64_t e = pair; e < n_entries; e += npairs, ++seq) {
      const uint32_t s = seq % NST, use = seq / NST;
      mbar_wait(&full[s], use & 1);
      acc += reinterpret_cast<const uint32_t *>(buf + s * S)[lane];
      __syncwarp();
      if (lane == 0) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&empty[s])), "r"(seq & 1));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
      }
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void k_ldg(const uint4 *__restrict__ src, uint64_t n, uint32_t *sink) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 v = __ldg(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main(int argc, char **argv) {
  const uint64_t bytes = 1ull << 30;
  if (argc > 1) {
    // "l2 <MiB>": stream 1 GiB out of an L2-resident region of <MiB> (the
    // table re-streams of the large-entry tensor path come mostly from L2)
    const uint64_t region = uint64_t(atoi(argv[2])) << 20;
    uint8_t *src; uint32_t *sink;
    CK(cudaMalloc(&src, region)); CK(cudaMalloc(&sink, 16)); CK(cudaMemset(src, 1, region));
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (uint32_t S : {16384u}) {
      for (uint32_t NST : {2u, 4u, 8u, 12u}) {
        for (uint32_t NCP : {1u, 4u}) {
          const uint64_t ne = bytes / S, wrap = region / S;
          float best = 1e9;
          for (int r = 0; r < 3; ++r) {
            cudaEventRecord(a);
            k_bulk<<<nsm, 64, 256 + size_t(S) * NST>>>(src, ne, S, NST, NCP, sink, wrap);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
          }
          printf("L2 region %llu MiB: bulk S %u NST %2u copies/entry %u in-flight/SM %4u KB: %.3f ms %7.1f GB/s\n",
                 (unsigned long long)(region >> 20), S, NST, NCP, S * NST / 1024, best, bytes / (best * 1e-3) * 1e-9);
        }
      }
    }
    // multicast to CTA pairs: each pair reads 1/npairs of the entries once and delivers them to 2 SMs
    CK(cudaFuncSetAttribute(k_bulk_mc, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    for (uint32_t NST : {4u, 8u}) {
      const uint32_t S = 16384;
      const uint64_t ne = bytes / S, wrap = region / S;
      float best = 1e9;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        k_bulk_mc<<<nsm, 64, 256 + size_t(S) * NST>>>(src, ne, S, NST, sink, wrap);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      CK(cudaGetLastError());
      printf("L2 region %llu MiB: multicast pairs S %u NST %2u: %.3f ms  read %7.1f GB/s  delivered to SMEM %7.1f GB/s\n",
             (unsigned long long)(region >> 20), S, NST, best, bytes / (best * 1e-3) * 1e-9, 2 * bytes / (best * 1e-3) * 1e-9);
    }
    // the same bytes by LDG.128 from all warps (16 passes over the region)
    for (int tpb : {256, 1024}) {
      float best = 1e9;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        for (uint64_t pass = 0; pass < bytes / region; ++pass)
          k_ldg<<<nsm * (2048 / tpb), tpb>>>(reinterpret_cast<const uint4 *>(src), region / 16, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("L2 region %llu MiB: ldg.128 threads %d x %d CTAs/SM: %.3f ms %7.1f GB/s\n",
             (unsigned long long)(region >> 20), tpb, 2048 / tpb, best, bytes / (best * 1e-3) * 1e-9);
    }
    CK(cudaGetLastError());
    return 0;
  }
  uint8_t *src; uint32_t *sink;
  CK(cudaMalloc(&src, bytes)); CK(cudaMalloc(&sink, 16));
  CK(cudaMemset(src, 1, bytes));
  uint8_t *flush; CK(cudaMalloc(&flush, 256 << 20));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto f) {
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaMemset(flush, r, 256 << 20);
      cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    return best;
  };
  for (int cps : {1, 2}) {
    for (uint32_t S : {4096u, 8192u, 16384u, 32768u, 65536u}) {
      for (uint32_t NST : {2u, 4u, 6u, 8u, 12u}) {
        const size_t smem = 256 + size_t(S) * NST;
        if (smem * cps > 227 * 1024 || NST > 16) continue;
        for (uint32_t NCP : {1u, 4u}) {
          if (S / NCP < 1024) continue;
          const uint64_t ne = bytes / S;
          float ms = run([&] { k_bulk<<<nsm * cps, 64, smem>>>(src, ne, S, NST, NCP, sink); });
          printf("bulk ctas/sm %d S %6u NST %2u copies/entry %u in-flight/SM %4zu KB: %.3f ms %7.1f GB/s\n", cps, S, NST,
                 NCP, size_t(S) * NST * cps / 1024, ms, bytes / (ms * 1e-3) * 1e-9);
        }
      }
    }
  }
  for (int tpb : {256, 512, 1024}) {
    float ms = run([&] { k_ldg<<<nsm * (2048 / tpb), tpb>>>(reinterpret_cast<const uint4 *>(src), bytes / 16, sink); });
    printf("ldg.128 threads %d x %d CTAs/SM: %.3f ms %7.1f GB/s\n", tpb, 2048 / tpb, ms, bytes / (ms * 1e-3) * 1e-9);
  }
  CK(cudaGetLastError());
  return 0;
}
