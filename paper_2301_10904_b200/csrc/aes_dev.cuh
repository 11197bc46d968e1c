// aes_dev.cuh -- AES-128 tree PRF for sm_100a: lane-replicated T-tables in
// shared memory.
//
// PRF_s(c) = AES-128 with key s on the block 0^120 || c (reading R8 for AES;
// FIPS-197; the paper's baseline PRF, Table 4).  Each internal
// node costs one key schedule and two encryptions (R9).  Seeds stay plain
// 16-byte values (LE words = FIPS-197 state columns: word j = bytes 4j..4j+3,
// row r = byte r), exactly as in the ChaCha20 path: roots, codewords, the
// frontier and the DFS stack need no conversion.
//
// Round function (FIPS-197 5.1, the standard T-table form): column j of the
// next state is
//     T0[a_j.b0] ^ T1[a_{j+1}.b1] ^ T2[a_{j+2}.b2] ^ T3[a_{j+3}.b3] ^ k_j
// with T0[x] = (2S(x), S(x), S(x), 3S(x)) (bytes 0..3) and Tt = rotl(T0, 8t).
// Only T0 and T1 are stored; T2, T3 = rot16(T0, T1), so one byte permute per
// column:  T0[.] ^ T1[.] ^ rot16(T0[.] ^ T1[.] ^ rot16(k_j)).  The final round
// takes S(x) from byte 1 of T0[x] (bytes 2, 3 of T1[x]); the key schedule's
// SubWord likewise.
//
// Layout (64 KB at the start of the kernel's dynamic shared memory): entry e
// of table t holds 32 copies, one per lane:  address e*256 + t*128 + 4*lane.
// Every lane reads its own bank whatever the index, so each lookup is one
// conflict-free LDS and the timing does not depend on the (secret) seed bytes.
// The address is ONE byte permute: (byte k of x) << 8 | (lane*4 + 128 t),
// taken from x and a per-lane constant, added to the dynamic-SMEM base by the
// LDS itself ([R + UR]).  Per node: 333 table lookups (16 per block-round,
// minus those the second block shares with the first: its round-1 state
// differs in byte 15 only, its round-2 state in column 0 only; 4 per
// key-schedule round).
//
// The key schedule runs on rot16(k), the form the rounds XOR in (no per-round
// key rotation).  Rounds 1 and 2 share lookups between the two blocks (their
// states differ in byte 15, then in column 0 only): 333 lookups per node.  Replaces the bitsliced table-free formulation of
// round 1 (4,075 ALU ops per node; 4,172 QPS at c3; now 21.6k).
#pragma once
#include <cstdint>

namespace dpfpir {
namespace dev {

constexpr uint32_t kAesSmemBytes = 65536;  // T0 and T1, 32 lane copies each

// ---- T0 from the S-box, computed at compile time (FIPS-197 5.1.1: S(x) =
// affine(x^-1) in GF(2^8) mod x^8 + x^4 + x^3 + x + 1).
struct AesT0 {
  uint32_t t[256];
};
constexpr uint8_t aes_gf_mul(uint8_t a, uint8_t b) {
  uint8_t r = 0;
  for (int i = 0; i < 8; ++i) {
    if (b & 1) r = uint8_t(r ^ a);
    const bool hi = (a & 0x80) != 0;
    a = uint8_t(a << 1);
    if (hi) a = uint8_t(a ^ 0x1B);
    b = uint8_t(b >> 1);
  }
  return r;
}
constexpr uint8_t aes_sbox_ct(uint8_t x) {
  uint8_t inv = 0;  // x^254 = x^-1 (0 -> 0)
  if (x) {
    uint8_t p = x;
    inv = 1;
    for (int e = 254; e; e >>= 1) {
      if (e & 1) inv = aes_gf_mul(inv, p);
      p = aes_gf_mul(p, p);
    }
  }
  uint8_t s = inv;
  for (int i = 1; i <= 4; ++i) s = uint8_t(s ^ uint8_t((inv << i) | (inv >> (8 - i))));
  return uint8_t(s ^ 0x63);
}
constexpr AesT0 make_aes_t0() {
  AesT0 r{};
  for (int x = 0; x < 256; ++x) {
    const uint8_t s = aes_sbox_ct(uint8_t(x));
    const uint8_t s2 = aes_gf_mul(s, 2), s3 = uint8_t(s2 ^ s);
    r.t[x] = uint32_t(s2) | uint32_t(s) << 8 | uint32_t(s) << 16 | uint32_t(s3) << 24;
  }
  return r;
}
static_assert(aes_sbox_ct(0x00) == 0x63 && aes_sbox_ct(0x53) == 0xED && aes_sbox_ct(0xFF) == 0x16,
              "FIPS-197 S-box (Fig. 7)");
__constant__ AesT0 c_aes_t0 = make_aes_t0();
// Rcon of rounds 1..10 (FIPS-197 5.2), rot16 (the key schedule runs on rot16(k))
__constant__ uint32_t c_aes_rcon_r16[10] = {0x01u << 16, 0x02u << 16, 0x04u << 16, 0x08u << 16, 0x10u << 16,
                                            0x20u << 16, 0x40u << 16, 0x80u << 16, 0x1Bu << 16, 0x36u << 16};

// the kernels' dynamic shared memory (every extern __shared__ array aliases it)
extern __shared__ __align__(128) uint8_t dpf_dyn_smem[];

// Fill the lane-replicated tables; the caller synchronises the CTA before use.
__device__ __forceinline__ void aes_tt_fill() {
  uint4 *w = reinterpret_cast<uint4 *>(dpf_dyn_smem);
  for (uint32_t i = threadIdx.x; i < kAesSmemBytes / 16; i += blockDim.x) {
    const uint32_t e = i >> 4, t = (i >> 3) & 1;  // 16 uint4 per entry: 8 for T0, 8 for T1
    const uint32_t v = c_aes_t0.t[e];
    const uint32_t x = t ? __funnelshift_l(v, v, 8) : v;
    w[i] = make_uint4(x, x, x, x);
  }
}

// Table word for byte K of x from table base l (= lane*4 for T0, +128 for T1)
template <int K>
__device__ __forceinline__ uint32_t aes_tl(uint32_t x, uint32_t l) {
  const uint32_t off = __byte_perm(x, l, 0x5504u | (uint32_t(K) << 4));  // byte0 = l, byte1 = x.bK, bytes 2,3 = 0
  return *reinterpret_cast<const uint32_t *>(dpf_dyn_smem + off);
}
__device__ __forceinline__ uint32_t rot16(uint32_t x) { return __byte_perm(x, 0, 0x1032); }

// one full round on state a (columns a[0..3]) with kr = rot16(round key)
__device__ __forceinline__ void aes_round(const uint32_t (&a)[4], uint32_t (&o)[4], const uint32_t (&kr)[4],
                                          uint32_t l0, uint32_t l1) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t u = aes_tl<2>(a[(j + 2) & 3], l0) ^ aes_tl<3>(a[(j + 3) & 3], l1) ^ kr[j];
    o[j] = aes_tl<0>(a[j], l0) ^ aes_tl<1>(a[(j + 1) & 3], l1) ^ rot16(u);
  }
}

// final round (no MixColumns): column j = S(a_j.b0), S(a_{j+1}.b1), S(a_{j+2}.b2), S(a_{j+3}.b3) ^ k_j
__device__ __forceinline__ void aes_final_round(const uint32_t (&a)[4], uint32_t (&o)[4], const uint32_t (&k)[4],
                                                uint32_t l0, uint32_t l1) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t v0 = aes_tl<0>(a[j], l0), v1 = aes_tl<1>(a[(j + 1) & 3], l0);  // S at byte 1 of T0
    const uint32_t v2 = aes_tl<2>(a[(j + 2) & 3], l1), v3 = aes_tl<3>(a[(j + 3) & 3], l1);  // S at bytes 2, 3 of T1
    const uint32_t lo = __byte_perm(v0, v1, 0x0051), hi = __byte_perm(v2, v3, 0x7200);
    o[j] = __byte_perm(lo, hi, 0x7610) ^ k[j];
  }
}

// Next round key (FIPS-197 5.2: k0 ^= SubWord(RotWord(k3)) ^ Rcon, k_j ^= k_{j-1}),
// kept in the rot16 domain: kr_j = rot16(k_j), the form every full round XORs
// in (so no per-round rotation of the key).  Byte b of k3 is byte (b + 2) & 3
// of kr3; rot16(t) assembles with a swapped selector.
__device__ __forceinline__ void aes_next_key_r16(uint32_t (&kr)[4], uint32_t rcon_r16, uint32_t l0, uint32_t l1) {
  // RotWord in LE words: t = S(k3.b1), S(k3.b2), S(k3.b3), S(k3.b0)
  const uint32_t w1 = aes_tl<3>(kr[3], l0), w2 = aes_tl<0>(kr[3], l0);  // k3.b1, k3.b2: S at byte 1 (T0)
  const uint32_t w3 = aes_tl<1>(kr[3], l1), w0 = aes_tl<2>(kr[3], l1);  // k3.b3, k3.b0: S at bytes 2, 3 (T1)
  const uint32_t lo = __byte_perm(w1, w2, 0x0051), hi = __byte_perm(w3, w0, 0x7200);
  kr[0] ^= __byte_perm(lo, hi, 0x1076) ^ rcon_r16;  // rot16(t) ^ rot16(Rcon)
  kr[1] ^= kr[0];
  kr[2] ^= kr[1];
  kr[3] ^= kr[2];
}

// Both children of seed s: AES_s(0^128) and AES_s(0^120 || 1).
__device__ __forceinline__ void aes_children_tt(const uint4 s, uint4 &c0, uint4 &c1) {
  const uint32_t l0 = (threadIdx.x & 31u) << 2, l1 = l0 | 128u;
  uint32_t kr[4] = {rot16(s.x), rot16(s.y), rot16(s.z), rot16(s.w)};
  uint32_t a[4], b[4];
  // round 0: AddRoundKey on the plaintexts (block 1: byte 15 = 1 = byte 3 of column 3)
  const uint32_t a3b = s.w ^ 0x01000000u;
  // round 1: only column 0 reads byte 15 (ShiftRows: row 3 of column 3 -> column 0)
  aes_next_key_r16(kr, 0x01u << 16, l0, l1);
  {
    const uint32_t s0 = s.x, s1 = s.y, s2 = s.z, s3 = s.w;
    const uint32_t p = aes_tl<0>(s0, l0) ^ aes_tl<1>(s1, l1);
    const uint32_t q = aes_tl<2>(s2, l0) ^ kr[0];
    a[0] = p ^ rot16(q ^ aes_tl<3>(s3, l1));
    b[0] = p ^ rot16(q ^ aes_tl<3>(a3b, l1));
    const uint32_t st[4] = {s0, s1, s2, s3};
#pragma unroll
    for (int j = 1; j < 4; ++j) {
      const uint32_t u = aes_tl<2>(st[(j + 2) & 3], l0) ^ aes_tl<3>(st[(j + 3) & 3], l1) ^ kr[j];
      a[j] = b[j] = aes_tl<0>(st[j], l0) ^ aes_tl<1>(st[(j + 1) & 3], l1) ^ rot16(u);
    }
  }
  // round 2: the two states still differ in column 0 only (round 1's column
  // 0), so each output column has ONE lookup that differs between the blocks
  // (column j reads column 0 at byte (4 - j) & 3): 20 lookups instead of 32.
  aes_next_key_r16(kr, 0x02u << 16, l0, l1);
  {
    const uint32_t b0 = b[0];
    // j = 0: column 0 at byte 0 (T0, outside the rot16 group)
    const uint32_t r0 = rot16(aes_tl<2>(a[2], l0) ^ aes_tl<3>(a[3], l1) ^ kr[0]);
    const uint32_t t01 = aes_tl<1>(a[1], l1);
    const uint32_t e0a = aes_tl<0>(a[0], l0) ^ t01 ^ r0, e0b = aes_tl<0>(b0, l0) ^ t01 ^ r0;
    // j = 1: column 0 at byte 3 (T1, inside the rot16 group)
    const uint32_t v1 = aes_tl<0>(a[1], l0) ^ aes_tl<1>(a[2], l1);
    const uint32_t q1 = aes_tl<2>(a[3], l0) ^ kr[1];
    const uint32_t e1a = v1 ^ rot16(q1 ^ aes_tl<3>(a[0], l1)), e1b = v1 ^ rot16(q1 ^ aes_tl<3>(b0, l1));
    // j = 2: column 0 at byte 2 (T0, inside the rot16 group)
    const uint32_t v2 = aes_tl<0>(a[2], l0) ^ aes_tl<1>(a[3], l1);
    const uint32_t q2 = aes_tl<3>(a[1], l1) ^ kr[2];
    const uint32_t e2a = v2 ^ rot16(q2 ^ aes_tl<2>(a[0], l0)), e2b = v2 ^ rot16(q2 ^ aes_tl<2>(b0, l0));
    // j = 3: column 0 at byte 1 (T1, outside the rot16 group)
    const uint32_t r3 = rot16(aes_tl<2>(a[1], l0) ^ aes_tl<3>(a[2], l1) ^ kr[3]);
    const uint32_t t30 = aes_tl<0>(a[3], l0);
    const uint32_t e3a = t30 ^ aes_tl<1>(a[0], l1) ^ r3, e3b = t30 ^ aes_tl<1>(b0, l1) ^ r3;
    a[0] = e0a; a[1] = e1a; a[2] = e2a; a[3] = e3a;
    b[0] = e0b; b[1] = e1b; b[2] = e2b; b[3] = e3b;
  }
#pragma unroll 2
  for (uint32_t r = 3; r <= 9; ++r) {
    aes_next_key_r16(kr, c_aes_rcon_r16[r - 1], l0, l1);
    uint32_t ta[4], tb[4];
    aes_round(a, ta, kr, l0, l1);
    aes_round(b, tb, kr, l0, l1);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      a[j] = ta[j];
      b[j] = tb[j];
    }
  }
  aes_next_key_r16(kr, 0x36u << 16, l0, l1);
  uint32_t k[4], oa[4], ob[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) k[j] = rot16(kr[j]);
  aes_final_round(a, oa, k, l0, l1);
  aes_final_round(b, ob, k, l0, l1);
  c0 = make_uint4(oa[0], oa[1], oa[2], oa[3]);
  c1 = make_uint4(ob[0], ob[1], ob[2], ob[3]);
}

struct PrfAesTt {
  static constexpr uint32_t id = 2;  // DPF_PRF_AES128
  static constexpr bool kEt = false;
  static constexpr uint32_t kSmemBytes = kAesSmemBytes;  // at the start of dynamic SMEM
  static __device__ __forceinline__ void init_smem() { aes_tt_fill(); }
  static __device__ __forceinline__ void children(const uint4 s, uint4 &c0, uint4 &c1) { aes_children_tt(s, c0, c1); }
  static __device__ __forceinline__ uint32_t word1(const uint4 s) { return s.y; }  // bytes 4..7 (R6)
};

}  // namespace dev
}  // namespace dpfpir
