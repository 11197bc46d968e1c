// Microbenchmark: integer-pipe throughput on sm_100a for the DPF hot loop.
// Measures (a) ChaCha20 block rate with SHF rotates, (b) with some rotates
// moved to the FMA pipe as IMAD.HI + IMAD, (c) raw LOP3 / SHF / IMAD /
// IMAD.HI throughput. Used only to ground DESIGN.md's ALU-pipe roofline;
// not part of the product. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t rotl_shf(uint32_t x, int k) { return __funnelshift_l(x, x, k); }
__device__ __forceinline__ uint32_t rotl_fma(uint32_t x, int k) {
  uint32_t hi = __umulhi(x, 1u << k);
  return x * (1u << k) + hi;
}

template <int MODE>
__device__ __forceinline__ void qr(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d) {
  a += b; d ^= a; d = (MODE >= 1) ? rotl_fma(d, 16) : rotl_shf(d, 16);
  c += d; b ^= c; b = rotl_shf(b, 12);
  a += b; d ^= a; d = (MODE >= 2) ? rotl_fma(d, 8) : rotl_shf(d, 8);
  c += d; b ^= c; b = rotl_shf(b, 7);
}

// MODE 0: all SHF. MODE 1: rot16 on FMA. MODE 2: rot16 + rot8 on FMA.
// MODE 3: alternate QRs between mode 0 and mode 1 (1/8 of rotates on FMA).
template <int MODE>
__device__ __forceinline__ void chacha_block(const uint32_t s[4], uint32_t out[8]) {
  uint32_t x0 = 0x61707865, x1 = 0x3320646e, x2 = 0x79622d32, x3 = 0x6b206574;
  uint32_t x4 = s[0], x5 = s[1], x6 = s[2], x7 = s[3];
  uint32_t x8 = 0, x9 = 0, x10 = 0, x11 = 0, x12 = 0, x13 = 0, x14 = 0, x15 = 0;
#pragma unroll
  for (int i = 0; i < 10; i++) {
    if (MODE == 3) {
      qr<0>(x0, x4, x8, x12); qr<1>(x1, x5, x9, x13); qr<0>(x2, x6, x10, x14); qr<1>(x3, x7, x11, x15);
      qr<0>(x0, x5, x10, x15); qr<1>(x1, x6, x11, x12); qr<0>(x2, x7, x8, x13); qr<1>(x3, x4, x9, x14);
    } else {
      qr<MODE>(x0, x4, x8, x12); qr<MODE>(x1, x5, x9, x13); qr<MODE>(x2, x6, x10, x14); qr<MODE>(x3, x7, x11, x15);
      qr<MODE>(x0, x5, x10, x15); qr<MODE>(x1, x6, x11, x12); qr<MODE>(x2, x7, x8, x13); qr<MODE>(x3, x4, x9, x14);
    }
  }
  out[0] = x0 + 0x61707865; out[1] = x1 + 0x3320646e; out[2] = x2 + 0x79622d32; out[3] = x3 + 0x6b206574;
  out[4] = x4 + s[0]; out[5] = x5 + s[1]; out[6] = x6 + s[2]; out[7] = x7 + s[3];
}

template <int MODE, int ILP>
__global__ void k_chacha(uint32_t *sink, int iters) {
  uint32_t s[ILP][4];
#pragma unroll
  for (int j = 0; j < ILP; j++) {
    s[j][0] = threadIdx.x * 7 + j; s[j][1] = blockIdx.x; s[j][2] = 0x1234 + j; s[j][3] = 99;
  }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < ILP; j++) {
      uint32_t o[8];
      chacha_block<MODE>(s[j], o);
      // descend to the child selected by the lsb, with a codeword-like xor
      uint32_t t = o[0] & 1;
      s[j][0] = t ? o[4] : o[0]; s[j][1] = t ? o[5] : o[1];
      s[j][2] = t ? o[6] : o[2]; s[j][3] = t ? o[7] : o[3];
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < ILP; j++) acc ^= s[j][0] ^ s[j][1] ^ s[j][2] ^ s[j][3];
  if (acc == 0x12345678u) sink[0] = acc;
}

// raw pipe throughput: OP 0 = LOP3 (xor3), 1 = SHF, 2 = IMAD, 3 = IMAD.HI, 4 = IADD3
template <int OP>
__global__ void k_pipe(uint32_t *sink, int iters) {
  uint32_t r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = threadIdx.x + j * 77 + blockIdx.x;
  uint32_t m = 0x9e3779b9u + blockIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
#pragma unroll
      for (int j = 0; j < 8; j++) {
        if (OP == 0) r[j] = r[j] ^ r[(j + 1) & 7] ^ m;
        else if (OP == 1) r[j] = __funnelshift_l(r[j], r[(j + 1) & 7], 13);
        else if (OP == 2) r[j] = r[j] * m + r[(j + 1) & 7];
        else if (OP == 3) r[j] = __umulhi(r[j], m);
        else r[j] = r[j] + r[(j + 1) & 7] + m;
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) acc ^= r[j];
  if (acc == 0x12345678u) sink[0] = acc;
}

template <typename F>
static float time_it(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  uint32_t *sink; CK(cudaMalloc(&sink, 16));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, max clock %d MHz\n", nsm, clk / 1000);
  const int iters = 2000;
  for (int threads : {256, 512, 1024}) {
    for (int cpsm : {1, 2}) {
      int grid = nsm * cpsm;
      if (threads * cpsm > 2048) continue;
      double blocks = (double)grid * threads * iters;
#define RUNC(M, I) { float ms = time_it([&] { k_chacha<M, I><<<grid, threads>>>(sink, iters / I); }); \
        double bl = (double)grid * threads * (iters / I) * I; \
        printf("chacha mode %d ilp %d threads %4d ctas/sm %d: %.3f ms  %.2f Gblk/s  %.2f clk/blk/SM@max\n", M, I, threads, cpsm, ms, \
               bl / ms * 1e-6, (double)nsm * (clk * 1e3) / (bl / ms * 1e3)); }
      RUNC(0, 1) RUNC(1, 1) RUNC(2, 1) RUNC(3, 1) RUNC(0, 2) RUNC(3, 2)
      (void)blocks;
    }
  }
  for (int threads : {512, 1024}) {
    int grid = nsm * 2;
#define RUNP(O) { float ms = time_it([&] { k_pipe<O><<<grid, threads>>>(sink, iters / 4); }); \
      double ops = (double)grid * threads * (iters / 4) * 16 * 8; \
      printf("pipe op %d threads %d: %.3f ms  %.1f lane-ops/clk/SM@max\n", O, threads, ms, ops / (ms * 1e-3) / nsm / (clk * 1e3)); }
    RUNP(0) RUNP(1) RUNP(2) RUNP(3) RUNP(4)
  }
  CK(cudaGetLastError());
  return 0;
}
