// Microbenchmark: can part of ChaCha20's rotations move from the ALU pipe to
// the FMA pipe on sm_100a?  The tree PRF's 320 xor (LOP3) + 320 rotate (SHF)
// per block sit on the ALU pipe while its 320 adds (IMAD.IADD) leave the FMA
// pipe two-thirds idle.  A rotate can run on the FMA pipe as
//   lo = x * 2^k (IMAD), rotl(x, k) = mulhi(x, 2^k) + lo (IMAD.HI),
// or as one IMAD.WIDE.U32 plus an add; the multiplier must be a register
// ptxas cannot see (a kernel argument), else it strength-reduces the
// multiply back into ALU shifts (the r01 ubench_int_pipes mode 1/2 did).
// Also: raw pipe rates with chains ptxas cannot fold.
// Not part of the product.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

struct Mul { uint32_t m16, m12, m8, m7, one; };

__device__ __forceinline__ uint32_t rot_shf(uint32_t x, int k) { return __funnelshift_l(x, x, k); }
__device__ __forceinline__ uint32_t rot_mulhi(uint32_t x, uint32_t mk) {
  uint32_t lo, r;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(x), "r"(mk));
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(mk), "r"(lo));
  return r;
}
__device__ __forceinline__ uint32_t rot_wide(uint32_t x, uint32_t mk, uint32_t one) {
  uint32_t lo, hi, r;
  asm("{.reg .u64 w; mul.wide.u32 w, %2, %3; mov.b64 {%0, %1}, w;}" : "=r"(lo), "=r"(hi) : "r"(x), "r"(mk));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(hi), "r"(one), "r"(lo));
  return r;
}

// V: 0 = SHF, 1 = mul + mulhi, 2 = wide + add
template <int V>
__device__ __forceinline__ uint32_t rot(uint32_t x, int k, uint32_t mk, uint32_t one) {
  if (V == 0) return rot_shf(x, k);
  if (V == 1) return rot_mulhi(x, mk);
  return rot_wide(x, mk, one);
}

// per-rotation variant: A (rot16), B (rot12), C (rot8), D (rot7)
template <int A, int B, int C, int D>
__device__ __forceinline__ void qr(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d, const Mul &m) {
  a += b; d = rot<A>(d ^ a, 16, m.m16, m.one);
  c += d; b = rot<B>(b ^ c, 12, m.m12, m.one);
  a += b; d = rot<C>(d ^ a, 8, m.m8, m.one);
  c += d; b = rot<D>(b ^ c, 7, m.m7, m.one);
}

// MODE: 0 all SHF; 1 rot16 on FMA (mulhi) in all 8 QRs (80/320 moved);
// 2 rot16 mulhi in 4 of 8 QRs (40); 3 rot16 mulhi in 6 of 8 (60);
// 4 rot16 wide in all 8 (80); 5 rot16 wide in 4 of 8 (40);
// 6 rot16 + rot8 mulhi in 4 of 8 (80); 7 rot16 mulhi in 2 of 8 (20)
template <int MODE>
__device__ __forceinline__ void chacha_block(const uint32_t s[4], uint32_t out[8], const Mul &m) {
  uint32_t x0 = 0x61707865, x1 = 0x3320646e, x2 = 0x79622d32, x3 = 0x6b206574;
  uint32_t x4 = s[0], x5 = s[1], x6 = s[2], x7 = s[3];
  uint32_t x8 = 0, x9 = 0, x10 = 0, x11 = 0, x12 = 0, x13 = 0, x14 = 0, x15 = 0;
  constexpr int F = MODE == 1 ? 1 : MODE == 2 ? 1 : MODE == 3 ? 1 : MODE == 4 ? 2 : MODE == 5 ? 2 : MODE == 6 ? 1 : MODE == 7 ? 1 : 0;
  constexpr int G = MODE == 6 ? 1 : 0;
  constexpr int n = MODE == 1 || MODE == 4 ? 8 : MODE == 3 ? 6 : MODE == 7 ? 2 : MODE == 0 ? 0 : 4;
#pragma unroll
  for (int i = 0; i < 10; i++) {
    // QR q uses the FMA rotate when q < n (interleaved order so the FMA QRs spread)
    if (n > 0) qr<F, 0, G, 0>(x0, x4, x8, x12, m); else qr<0, 0, 0, 0>(x0, x4, x8, x12, m);
    if (n > 4) qr<F, 0, G, 0>(x1, x5, x9, x13, m); else qr<0, 0, 0, 0>(x1, x5, x9, x13, m);
    if (n > 2) qr<F, 0, G, 0>(x2, x6, x10, x14, m); else qr<0, 0, 0, 0>(x2, x6, x10, x14, m);
    if (n > 6) qr<F, 0, G, 0>(x3, x7, x11, x15, m); else qr<0, 0, 0, 0>(x3, x7, x11, x15, m);
    if (n > 1) qr<F, 0, G, 0>(x0, x5, x10, x15, m); else qr<0, 0, 0, 0>(x0, x5, x10, x15, m);
    if (n > 5) qr<F, 0, G, 0>(x1, x6, x11, x12, m); else qr<0, 0, 0, 0>(x1, x6, x11, x12, m);
    if (n > 3) qr<F, 0, G, 0>(x2, x7, x8, x13, m); else qr<0, 0, 0, 0>(x2, x7, x8, x13, m);
    if (n > 7) qr<F, 0, G, 0>(x3, x4, x9, x14, m); else qr<0, 0, 0, 0>(x3, x4, x9, x14, m);
  }
  out[0] = x0 + 0x61707865; out[1] = x1 + 0x3320646e; out[2] = x2 + 0x79622d32; out[3] = x3 + 0x6b206574;
  out[4] = x4 + s[0]; out[5] = x5 + s[1]; out[6] = x6 + s[2]; out[7] = x7 + s[3];
}

template <int MODE>
__global__ void k_chacha(uint32_t *sink, int iters, Mul m) {
  uint32_t s[4];
  s[0] = threadIdx.x * 7; s[1] = blockIdx.x; s[2] = 0x1234; s[3] = 99;
  for (int it = 0; it < iters; it++) {
    uint32_t o[8];
    chacha_block<MODE>(s, o, m);
    uint32_t t = o[0] & 1;
    s[0] = t ? o[4] : o[0]; s[1] = t ? o[5] : o[1];
    s[2] = t ? o[6] : o[2]; s[3] = t ? o[7] : o[3];
  }
  if ((s[0] ^ s[1] ^ s[2] ^ s[3]) == 0x12345678u) sink[0] = 1;
}

// raw pipe throughput, chains ptxas cannot fold:
// 0 LOP3 majority(r_j, r_j+1, r_j+2), 1 SHF funnel, 2 IMAD, 3 IMAD.HI,
// 4 IADD3 (3 distinct chained inputs), 5 IMAD.WIDE.U32, 6 PRMT
template <int OP>
__global__ void k_pipe(uint32_t *sink, int iters, uint32_t m) {
  uint32_t r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = threadIdx.x + j * 77 + blockIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
#pragma unroll
      for (int j = 0; j < 8; j++) {
        uint32_t a = r[(j + 1) & 7], b = r[(j + 2) & 7];
        if (OP == 0) asm("lop3.b32 %0, %0, %1, %2, 0xE8;" : "+r"(r[j]) : "r"(a), "r"(b));
        else if (OP == 1) r[j] = __funnelshift_l(r[j], a, 13);
        else if (OP == 2) asm("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[j]) : "r"(m), "r"(a));
        else if (OP == 3) asm("mad.hi.u32 %0, %0, %1, %2;" : "+r"(r[j]) : "r"(m), "r"(a));
        else if (OP == 4) r[j] = r[j] + a + b;
        else if (OP == 5) {
          uint32_t lo, hi;
          asm("{.reg .u64 w; mul.wide.u32 w, %2, %3; mov.b64 {%0, %1}, w;}" : "=r"(lo), "=r"(hi) : "r"(r[j]), "r"(m));
          r[j] = lo; r[(j + 4) & 7] = hi;
        } else asm("prmt.b32 %0, %0, %1, 0x2107;" : "+r"(r[j]) : "r"(a));
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
  Mul m{1u << 16, 1u << 12, 1u << 8, 1u << 7, 1u};
  const int iters = 2000;
  const char *names[8] = {"all SHF", "rot16 mulhi x8 QR (80 moved)", "rot16 mulhi x4 QR (40)", "rot16 mulhi x6 QR (60)",
                          "rot16 wide x8 QR (80)", "rot16 wide x4 QR (40)", "rot16+rot8 mulhi x4 QR (80)",
                          "rot16 mulhi x2 QR (20)"};
  for (int threads : {512, 1024}) {
    int grid = nsm * (2048 / threads);
#define RUNC(M) { float ms = time_it([&] { k_chacha<M><<<grid, threads>>>(sink, iters, m); }); \
      double bl = (double)grid * threads * iters; \
      printf("chacha mode %d threads %4d: %.3f ms  %6.2f Gblk/s  %.2f clk/blk/SM@max  %s\n", M, threads, ms, \
             bl / ms * 1e-6, (double)nsm * (clk * 1e3) / (bl / ms * 1e3), names[M]); }
    RUNC(0) RUNC(1) RUNC(2) RUNC(3) RUNC(4) RUNC(5) RUNC(6) RUNC(7)
  }
  const char *pn[7] = {"LOP3", "SHF", "IMAD", "IMAD.HI", "IADD3", "IMAD.WIDE", "PRMT"};
  for (int threads : {512, 1024}) {
    int grid = nsm * 2;
#define RUNP(O) { float ms = time_it([&] { k_pipe<O><<<grid, threads>>>(sink, iters / 4, 0x9e3779b9u); }); \
      double ops = (double)grid * threads * (iters / 4) * 16 * 8; \
      printf("pipe %-9s threads %d: %.3f ms  %.1f lane-ops/clk/SM@max\n", pn[O], threads, ms, ops / (ms * 1e-3) / nsm / (clk * 1e3)); }
    RUNP(0) RUNP(1) RUNP(2) RUNP(3) RUNP(4) RUNP(5) RUNP(6)
  }
  CK(cudaGetLastError());
  return 0;
}
