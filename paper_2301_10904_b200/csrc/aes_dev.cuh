// aes_dev.cuh -- table-free bitsliced AES-128 tree PRF for sm_100a.
//
// PRF_s(c) = AES-128 with key s on the block 0^120 || c (reading R8 for AES;
// FIPS-197; the paper's baseline PRF, Table 4).  Each internal
// node costs one key schedule and two encryptions (R9).
//
// Representation ("BS seed"): a 16-byte seed is kept bitsliced as 8 planes of
// 16 bits -- plane p holds bit p of byte i at bit i (i = r + 4c, FIPS-197
// state order) -- packed two planes per word into a uint4:
//     word k = plane 2k | plane (2k+1) << 16.
// A BS seed is 16 bytes like a plain seed, so the DFS stack, the frontier and
// the key layout are unchanged; roots and codewords are bitsliced once per
// batch by aes_bitslice_keys_kernel.  lsb(s) (R5) is bit 0 of byte 0 = bit 0
// of word 0 in both representations.
//
// The two encryptions of a node run together: in a 32-bit plane word the low
// half is block c = 0, the high half block c = 1.  SubBytes is the generated
// tower-field circuit (aes_sbox_bs.cuh, verified on all 256 inputs); ShiftRows
// and MixColumns are rotations inside the 16-bit halves (one AES column = one
// nibble).  No memory lookups: constant-time, table-free.
#pragma once
#include <cstdint>

#include "aes_sbox_bs.cuh"

namespace dpfpir {
namespace dev {

// Logical right shift.  (Moving these to the FMA pipe as IMAD.HI -- the FMA
// pipe idles at 7 % here -- measured no faster, also with the multiplier in
// constant memory so that it stays a multiply (r02: 48 of ~410 ops per round
// moved, 4,124 vs 4,149 QPS at c3): the rounds are issue-bound as much as
// ALU-bound, so only fewer instructions help.)
template <int K>
__device__ __forceinline__ uint32_t shr_fma(uint32_t x) {
  return x >> K;
}

// rotate every nibble down by k rows: new bit (r, c) = old bit ((r + k) % 4, c)
template <int K>
__device__ __forceinline__ uint32_t nib_rot(uint32_t x) {
  constexpr uint32_t lo = (K == 1) ? 0x77777777u : (K == 2) ? 0x33333333u : 0x11111111u;
  return (shr_fma<K>(x) & lo) | ((x << (4 - K)) & ~lo);
}

// rotate each 16-bit half right by 4*K bits: new column c = old column c + K
template <int K>
__device__ __forceinline__ uint32_t half_rot(uint32_t x) {
  if constexpr (K == 2) {
    return __byte_perm(x, x, 0x2301);
  } else {
    constexpr uint32_t m = (K == 1) ? 0x0FFF0FFFu : 0x000F000Fu;
    return (shr_fma<4 * K>(x) & m) | ((x << (16 - 4 * K)) & ~m);
  }
}

// ShiftRows (FIPS-197 5.1.2): new (r, c) = old (r, c + r); row r = bits r, r+4, r+8, r+12.
__device__ __forceinline__ uint32_t shift_rows(uint32_t x) {
  const uint32_t r1 = half_rot<1>(x), r2 = half_rot<2>(x), r3 = half_rot<3>(x);
  uint32_t o = (x & 0x11111111u) | (r1 & ~0x11111111u);
  o = (o & 0x33333333u) | (r2 & ~0x33333333u);
  return (o & 0x77777777u) | (r3 & ~0x77777777u);
}

// MixColumns (FIPS-197 5.1.3) on 8 planes: out = 2a + 3a' + a'' + a''' with
// a^(k) the byte k rows below; = xtime(u) + a' + rot2(u), u = a + a'.
__device__ __forceinline__ void mix_columns(uint32_t (&x)[8]) {
  uint32_t r1[8], u[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    r1[p] = nib_rot<1>(x[p]);
    u[p] = x[p] ^ r1[p];
  }
  // xtime(u): bit p <- bit p-1, and bit 7 feeds bits 0, 1, 3, 4 (x^8 = x^4 + x^3 + x + 1)
  uint32_t xt[8];
  xt[0] = u[7];
  xt[1] = u[0] ^ u[7];
  xt[2] = u[1];
  xt[3] = u[2] ^ u[7];
  xt[4] = u[3] ^ u[7];
  xt[5] = u[4];
  xt[6] = u[5];
  xt[7] = u[6];
#pragma unroll
  for (int p = 0; p < 8; ++p) x[p] = xt[p] ^ r1[p] ^ nib_rot<2>(u[p]);
}

// Rcon (FIPS-197 5.2) of rounds 1..10 as per-plane masks: Rcon enters row 0
// of every column of the new round key, i.e. bits 0, 4, 8, 12 of both halves.
__constant__ uint32_t c_rcon_mask[10][8] = {
#define DPF_RC(v) {(v)&1 ? 0x11111111u : 0u, (v)&2 ? 0x11111111u : 0u, (v)&4 ? 0x11111111u : 0u, \
                   (v)&8 ? 0x11111111u : 0u, (v)&16 ? 0x11111111u : 0u, (v)&32 ? 0x11111111u : 0u, \
                   (v)&64 ? 0x11111111u : 0u, (v)&128 ? 0x11111111u : 0u}
    DPF_RC(0x01), DPF_RC(0x02), DPF_RC(0x04), DPF_RC(0x08), DPF_RC(0x10),
    DPF_RC(0x20), DPF_RC(0x40), DPF_RC(0x80), DPF_RC(0x1B), DPF_RC(0x36)
#undef DPF_RC
};

// Next round key (FIPS-197 5.2) on duplicated 16-bit planes (both halves
// equal): column j' = (col 0 ^ ... ^ col j) ^ t,
// t = SubWord(RotWord(col 3)) ^ Rcon.
__device__ __forceinline__ void next_round_key(uint32_t (&k)[8], int round) {
  uint32_t s[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) s[p] = k[p];
  aes_sbox_bs(s);
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    // RotWord: t row r = S(col 3, row r+1); col 3 = bits 12..15 of each half
    const uint32_t t = (shr_fma<13>(s[p]) & 0x00070007u) | (shr_fma<9>(s[p]) & 0x00080008u);
    uint32_t q = k[p] ^ ((k[p] << 4) & 0xFFF0FFF0u);  // inclusive prefix XOR over columns
    q ^= (q << 8) & 0xFF00FF00u;
    k[p] = q ^ (t * 0x1111u) ^ c_rcon_mask[round - 1][p];
  }
}

// Both children of BS seed s: AES_s(0^128) and AES_s(0^120 || 1), as BS seeds.
__device__ __forceinline__ void aes_children_bs(const uint4 s, uint4 &c0, uint4 &c1) {
  uint32_t k[8], x[8];
  const uint32_t w[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    k[2 * q] = __byte_perm(w[q], 0, 0x1010);      // plane 2q duplicated into both halves
    k[2 * q + 1] = __byte_perm(w[q], 0, 0x3232);  // plane 2q+1 duplicated
  }
#pragma unroll
  for (int p = 0; p < 8; ++p) x[p] = k[p];  // AddRoundKey(0) on plaintexts 0 and 1
  x[0] ^= 0x80000000u;                      // block 1: byte 15 = 0x01 -> plane 0, bit 15 of the high half
#pragma unroll 1
  for (int round = 1; round <= 10; ++round) {
    aes_sbox_bs(x);
#pragma unroll
    for (int p = 0; p < 8; ++p) x[p] = shift_rows(x[p]);
    if (round != 10) mix_columns(x);
    next_round_key(k, round);
#pragma unroll
    for (int p = 0; p < 8; ++p) x[p] ^= k[p];
  }
  c0 = make_uint4(__byte_perm(x[0], x[1], 0x5410), __byte_perm(x[2], x[3], 0x5410),
                  __byte_perm(x[4], x[5], 0x5410), __byte_perm(x[6], x[7], 0x5410));
  c1 = make_uint4(__byte_perm(x[0], x[1], 0x7632), __byte_perm(x[2], x[3], 0x7632),
                  __byte_perm(x[4], x[5], 0x7632), __byte_perm(x[6], x[7], 0x7632));
}

// plain 16-byte seed (LE words) -> BS seed
__device__ __forceinline__ uint4 bs_from_bytes(uint4 s) {
  const uint32_t w[4] = {s.x, s.y, s.z, s.w};
  uint32_t plane[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    uint32_t acc = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // bits p, 8+p, 16+p, 24+p of word q -> bits 4q .. 4q+3
      const uint32_t t = (w[q] >> p) & 0x01010101u;
      acc |= (((t * 0x00204081u) >> 21) & 0xFu) << (4 * q);
    }
    plane[p] = acc;
  }
  return make_uint4(plane[0] | (plane[1] << 16), plane[2] | (plane[3] << 16), plane[4] | (plane[5] << 16),
                    plane[6] | (plane[7] << 16));
}

// bytes 4..7 of a BS seed as a little-endian u32 (w1 of reading R6)
__device__ __forceinline__ uint32_t bs_word1(uint4 s) {
  const uint32_t w[4] = {s.x, s.y, s.z, s.w};
  uint32_t out = 0;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const uint32_t nib = (w[p >> 1] >> (16 * (p & 1) + 4)) & 0xFu;  // bytes 4..7 of plane p
    out |= ((nib * 0x00204081u) & 0x01010101u) << p;
  }
  return out;
}

struct PrfAesBs {
  static constexpr uint32_t id = 2;  // DPF_PRF_AES128
  static constexpr bool kEt = false;
  static __device__ __forceinline__ void children(const uint4 s, uint4 &c0, uint4 &c1) { aes_children_bs(s, c0, c1); }
  static __device__ __forceinline__ uint32_t word1(const uint4 s) { return bs_word1(s); }
};

// Prepare AES keys in the device key array: bitslice root and codewords in
// place (wire layout kept: root at +16, cw column d at +32 + 64 (d-1)).
__global__ void aes_bitslice_keys_kernel(uint8_t *__restrict__ keys, uint32_t kstride, uint32_t B, uint32_t n) {
  const uint32_t per_key = 1 + 4 * n;  // root + 4 codewords per level
  const uint64_t total = uint64_t(B) * per_key;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t b = uint32_t(i / per_key), e = uint32_t(i % per_key);
    uint4 *p = reinterpret_cast<uint4 *>(keys + uint64_t(b) * kstride + (e == 0 ? 16 : 32 + 16 * (e - 1)));
    *p = bs_from_bytes(*p);
  }
}

}  // namespace dev
}  // namespace dpfpir
