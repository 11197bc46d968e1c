// chacha_dev.cuh -- device ChaCha20 tree PRF for sm_100a (table-free ARX).
//
// PRF_s(c) (ChaCha20 per P:532, Table 5), reading R8/R9: one
// RFC 8439 block keyed by s || 0^128, counter 0, nonce 0 yields both children:
// child 0 = keystream words 0..3, child 1 = words 4..7.  Words 8..15 of the
// initial state are zero, so the compiler folds the first column round; the
// feed-forward of words 8..15 is never computed (only 32 of 64 bytes used).
//
// Cost on sm_100a: 320 LOP3 + 320 SHF (ALU pipe, 64 lanes/clk/SM) + 320
// IMAD.IADD (FMA pipe); ALU-bound at 10 clk per block per SM, measured
// 10.2-10.3 clk (profiles/r01_ubench_int_pipes.txt).  Rotations stay on SHF:
// IMAD.HI is half-rate on sm_100a (same file), so moving rotates to the FMA
// pipe costs more than it saves.
#pragma once
#include <cstdint>

namespace dpfpir {
namespace dev {

__device__ __forceinline__ uint32_t rotl32(uint32_t x, int k) { return __funnelshift_l(x, x, k); }

#define DPF_QR(a, b, c, d)         \
  a += b; d = rotl32(d ^ a, 16);   \
  c += d; b = rotl32(b ^ c, 12);   \
  a += b; d = rotl32(d ^ a, 8);    \
  c += d; b = rotl32(b ^ c, 7);

// Both children of seed s (before the codeword correction of Eq. 3).
__device__ __forceinline__ void chacha_children(const uint4 s, uint4 &c0, uint4 &c1) {
  uint32_t x0 = 0x61707865u, x1 = 0x3320646eu, x2 = 0x79622d32u, x3 = 0x6b206574u;
  uint32_t x4 = s.x, x5 = s.y, x6 = s.z, x7 = s.w;
  uint32_t x8 = 0, x9 = 0, x10 = 0, x11 = 0, x12 = 0, x13 = 0, x14 = 0, x15 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    DPF_QR(x0, x4, x8, x12) DPF_QR(x1, x5, x9, x13) DPF_QR(x2, x6, x10, x14) DPF_QR(x3, x7, x11, x15)
    DPF_QR(x0, x5, x10, x15) DPF_QR(x1, x6, x11, x12) DPF_QR(x2, x7, x8, x13) DPF_QR(x3, x4, x9, x14)
  }
  c0 = make_uint4(x0 + 0x61707865u, x1 + 0x3320646eu, x2 + 0x79622d32u, x3 + 0x6b206574u);
  c1 = make_uint4(x4 + s.x, x5 + s.y, x6 + s.z, x7 + s.w);
}

// R20 (early-terminated leaves, f4): Convert(s) = all 16 words of the
// ChaCha20 block keyed by s || 0^128 with counter 1, nonce 0 (full
// feed-forward).  Same 640 ALU-pipe ops as an expansion block.
__device__ __forceinline__ void chacha_convert16(const uint4 s, uint32_t (&o)[16]) {
  uint32_t x0 = 0x61707865u, x1 = 0x3320646eu, x2 = 0x79622d32u, x3 = 0x6b206574u;
  uint32_t x4 = s.x, x5 = s.y, x6 = s.z, x7 = s.w;
  uint32_t x8 = 0, x9 = 0, x10 = 0, x11 = 0, x12 = 1, x13 = 0, x14 = 0, x15 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    DPF_QR(x0, x4, x8, x12) DPF_QR(x1, x5, x9, x13) DPF_QR(x2, x6, x10, x14) DPF_QR(x3, x7, x11, x15)
    DPF_QR(x0, x5, x10, x15) DPF_QR(x1, x6, x11, x12) DPF_QR(x2, x7, x8, x13) DPF_QR(x3, x4, x9, x14)
  }
  o[0] = x0 + 0x61707865u; o[1] = x1 + 0x3320646eu; o[2] = x2 + 0x79622d32u; o[3] = x3 + 0x6b206574u;
  o[4] = x4 + s.x; o[5] = x5 + s.y; o[6] = x6 + s.z; o[7] = x7 + s.w;
  o[8] = x8; o[9] = x9; o[10] = x10; o[11] = x11;
  o[12] = x12 + 1u; o[13] = x13; o[14] = x14; o[15] = x15;
}
#undef DPF_QR

__device__ __forceinline__ uint4 xor4(uint4 a, uint4 b) {
  return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
}

// PRF policies.  Both ChaCha20 and AES-128 (aes_dev.cuh) work on plain
// seeds, lsb(s) (R5) at bit 0 of word 0.  kSmemBytes: shared memory the PRF
// needs at the start of the kernel's dynamic SMEM (AES: its T-tables), filled
// by init_smem() before the kernel's first CTA barrier.
// kEt: early-terminated leaves (R20): the tree stops kEtBits levels above the
// rows and each final node yields 2^kEtBits leaves from one Convert block.
struct PrfChacha {
  static constexpr uint32_t id = 1;  // DPF_PRF_CHACHA20
  static constexpr bool kEt = false;
  static constexpr uint32_t kSmemBytes = 0;
  static __device__ __forceinline__ void init_smem() {}
  static __device__ __forceinline__ void children(const uint4 s, uint4 &c0, uint4 &c1) { chacha_children(s, c0, c1); }
  static __device__ __forceinline__ uint32_t word1(const uint4 s) { return s.y; }  // bytes 4..7 (R6)
};
struct PrfChachaEt {
  static constexpr uint32_t id = 3;  // DPF_PRF_CHACHA20_ET
  static constexpr bool kEt = true;
  static constexpr uint32_t kEtBits = 4;
  static constexpr uint32_t kSmemBytes = 0;
  static __device__ __forceinline__ void init_smem() {}
  static __device__ __forceinline__ void children(const uint4 s, uint4 &c0, uint4 &c1) { chacha_children(s, c0, c1); }
  static __device__ __forceinline__ uint32_t word1(const uint4 s) { return s.y; }  // unused (no per-seed leaves)
};

// Eq. 3 for both children of node s at depth d-1:
//   child_c = PRF_s(c) XOR C_{lsb(s)}[c, d]          (R1, R5)
// lvl_cw points at the key's 64-byte codeword column for depth d, laid out
// [t][c] (wire format): the control bit selects the row by address.
template <class Prf>
__device__ __forceinline__ void node_children(const uint4 s, const uint4 *__restrict__ lvl_cw, uint4 &c0,
                                              uint4 &c1) {
  const uint32_t t = s.x & 1u;
  const uint4 k0 = __ldg(lvl_cw + 2 * t);
  const uint4 k1 = __ldg(lvl_cw + 2 * t + 1);
  uint4 p0, p1;
  Prf::children(s, p0, p1);
  c0 = xor4(p0, k0);
  c1 = xor4(p1, k1);
}

// Leaf conversion (R2, R6, R7), before the party sign: w1(s) + lsb(s) * cw_out.
template <class Prf>
__device__ __forceinline__ uint32_t leaf_value(const uint4 s, uint32_t cw_out) {
  return Prf::word1(s) + ((s.x & 1u) ? cw_out : 0u);
}

// R20 leaf conversion of a final node s, before the party sign:
// y[c] = Convert(s)[c] + lsb(s) * CWL[c]  (16 leaves 16i..16i+15).
__device__ __forceinline__ void leaf_values16(const uint4 s, const uint32_t (&cwl)[16], uint32_t (&y)[16]) {
  chacha_convert16(s, y);
  const uint32_t t = s.x & 1u;
  // y += t * CWL as IMAD on the FMA pipe (a select would take ALU slots
  // from the PRF; t is 0 or 1)
#pragma unroll
  for (int c = 0; c < 16; ++c) asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(y[c]) : "r"(t), "r"(cwl[c]));
}

// CWL of a wire key: the 16 LE words in the column after tree level h.
__device__ __forceinline__ void load_cwl(const uint4 *__restrict__ col, uint32_t (&cwl)[16]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 v = __ldg(col + i);
    cwl[4 * i] = v.x; cwl[4 * i + 1] = v.y; cwl[4 * i + 2] = v.z; cwl[4 * i + 3] = v.w;
  }
}

}  // namespace dev
}  // namespace dpfpir
