// host.cc -- client-side half of libdpfpir: Gen, key codec, reconstruct,
// status strings.  Independent of oracle/ (own ChaCha20, own AES-128, own
// Gen); the tests check that both produce the same keys from the same DRBG
// seed, for both PRFs.
//
// Citations: P:n = PAPER.md line n; R1..R14 = DESIGN.md "Readings".
#include "dpfpir.h"

#include <sys/random.h>

#include <array>
#include <cstring>

namespace dpfpir {
namespace {

using Words4 = std::array<uint32_t, 4>;  // one 128-bit seed / codeword as LE words

inline uint32_t rol(uint32_t v, unsigned s) { return (v << s) | (v >> (32u - s)); }

// ChaCha20 block (RFC 8439 2.3) on a word-level state.  out = 16 words.
void chacha20_words(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3], uint32_t out[16]) {
  uint32_t st[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, key[0], key[1], key[2], key[3],
                     key[4],      key[5],      key[6],      key[7],      counter, nonce[0], nonce[1], nonce[2]};
  uint32_t w[16];
  std::memcpy(w, st, sizeof w);
  auto qr = [&w](int a, int b, int c, int d) {
    w[a] += w[b]; w[d] = rol(w[d] ^ w[a], 16);
    w[c] += w[d]; w[b] = rol(w[b] ^ w[c], 12);
    w[a] += w[b]; w[d] = rol(w[d] ^ w[a], 8);
    w[c] += w[d]; w[b] = rol(w[b] ^ w[c], 7);
  };
  for (int r = 0; r < 20; r += 2) {
    qr(0, 4, 8, 12); qr(1, 5, 9, 13); qr(2, 6, 10, 14); qr(3, 7, 11, 15);
    qr(0, 5, 10, 15); qr(1, 6, 11, 12); qr(2, 7, 8, 13); qr(3, 4, 9, 14);
  }
  for (int i = 0; i < 16; ++i) out[i] = w[i] + st[i];
}

// Tree PRF (R8, R9).  ChaCha20: one block keyed by s || 0^128 with counter 0,
// nonce 0; child 0 = words 0..3, child 1 = words 4..7 of the keystream.
// AES-128: key s, child c = AES_s(0^120 || c).
void prf_pair_chacha(const Words4 &s, Words4 &c0, Words4 &c1) {
  const uint32_t key[8] = {s[0], s[1], s[2], s[3], 0, 0, 0, 0};
  const uint32_t nonce[3] = {0, 0, 0};
  uint32_t ks[16];
  chacha20_words(key, 0, nonce, ks);
  for (int i = 0; i < 4; ++i) { c0[i] = ks[i]; c1[i] = ks[4 + i]; }
}

// ---- AES-128 (FIPS-197) for the client-side Gen with DPF_PRF_AES128.
// Byte-oriented; the S-box is derived at first use from GF(2^8) logarithms
// (generator 3), then the affine map of FIPS-197 5.1.1.
struct AesTables {
  uint8_t sbox[256];
  AesTables() {
    uint8_t exp[256], log[256] = {0};
    uint8_t g = 1;
    for (int i = 0; i < 255; ++i) {
      exp[i] = g;
      log[g] = uint8_t(i);
      g = uint8_t(g ^ (g << 1) ^ ((g & 0x80) ? 0x1B : 0));  // g *= 3
    }
    for (int x = 0; x < 256; ++x) {
      const uint8_t inv = x ? exp[(255 - log[x]) % 255] : 0;
      uint8_t b = inv;
      for (int r = 1; r <= 4; ++r) b ^= uint8_t((inv << r) | (inv >> (8 - r)));
      sbox[x] = uint8_t(b ^ 0x63);
    }
  }
};
const AesTables &aes_tables() {
  static const AesTables t;
  return t;
}
inline uint8_t xt(uint8_t a) { return uint8_t((a << 1) ^ ((a & 0x80) ? 0x1B : 0)); }

void aes128_encrypt_block(const uint8_t key[16], const uint8_t in[16], uint8_t out[16]) {
  const uint8_t *S = aes_tables().sbox;
  uint8_t rk[16], st[16];
  std::memcpy(rk, key, 16);
  for (int i = 0; i < 16; ++i) st[i] = in[i] ^ rk[i];
  uint8_t rcon = 1;
  for (int round = 1; round <= 10; ++round) {
    uint8_t t[16];
    for (int c = 0; c < 4; ++c)  // SubBytes + ShiftRows
      for (int r = 0; r < 4; ++r) t[4 * c + r] = S[st[4 * ((c + r) & 3) + r]];
    if (round < 10) {
      for (int c = 0; c < 4; ++c) {  // MixColumns
        uint8_t *a = t + 4 * c;
        const uint8_t all = a[0] ^ a[1] ^ a[2] ^ a[3], a0 = a[0];
        a[0] ^= all ^ xt(a[0] ^ a[1]);
        a[1] ^= all ^ xt(a[1] ^ a[2]);
        a[2] ^= all ^ xt(a[2] ^ a[3]);
        a[3] ^= all ^ xt(a[3] ^ a0);
      }
    }
    // next round key
    uint8_t w[4] = {uint8_t(S[rk[13]] ^ rcon), S[rk[14]], S[rk[15]], S[rk[12]]};
    rcon = xt(rcon);
    for (int c = 0; c < 4; ++c)
      for (int r = 0; r < 4; ++r) w[r] = rk[4 * c + r] ^= w[r];
    for (int i = 0; i < 16; ++i) st[i] = t[i] ^ rk[i];
  }
  std::memcpy(out, st, 16);
}

inline uint32_t ld32(const uint8_t *p) {
  return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}
inline void st32(uint8_t *p, uint32_t v) {
  p[0] = uint8_t(v); p[1] = uint8_t(v >> 8); p[2] = uint8_t(v >> 16); p[3] = uint8_t(v >> 24);
}
inline Words4 from_bytes(const uint8_t *p) { return {ld32(p), ld32(p + 4), ld32(p + 8), ld32(p + 12)}; }
inline void to_bytes(const Words4 &w, uint8_t *p) { for (int i = 0; i < 4; ++i) st32(p + 4 * i, w[i]); }

void prf_pair_aes(const Words4 &s, Words4 &c0, Words4 &c1) {
  uint8_t key[16], blk[16] = {0}, o[16];
  to_bytes(s, key);
  aes128_encrypt_block(key, blk, o);
  c0 = from_bytes(o);
  blk[15] = 1;
  aes128_encrypt_block(key, blk, o);
  c1 = from_bytes(o);
}

void prf_pair(uint32_t prf, const Words4 &s, Words4 &c0, Words4 &c1) {
  if (prf == DPF_PRF_AES128)
    prf_pair_aes(s, c0, c1);
  else
    prf_pair_chacha(s, c0, c1);
}
inline Words4 xor4(const Words4 &a, const Words4 &b) { return {a[0] ^ b[0], a[1] ^ b[1], a[2] ^ b[2], a[3] ^ b[3]}; }

// Gen's randomness: the ChaCha20 keystream under key = rng_seed, nonce 0,
// counter 0, 1, 2, ... consumed as consecutive 16-byte draws (four words).
class KeystreamDrbg {
 public:
  explicit KeystreamDrbg(const uint8_t seed[32]) {
    for (int i = 0; i < 8; ++i) key_[i] = ld32(seed + 4 * i);
  }
  Words4 next128() {
    if (pos_ == 16) refill();
    Words4 r = {buf_[pos_], buf_[pos_ + 1], buf_[pos_ + 2], buf_[pos_ + 3]};
    pos_ += 4;
    return r;
  }

 private:
  void refill() {
    const uint32_t nonce[3] = {0, 0, 0};
    chacha20_words(key_, ctr_++, nonce, buf_);
    pos_ = 0;
  }
  uint32_t key_[8];
  uint32_t buf_[16];
  uint32_t ctr_ = 0;
  int pos_ = 16;
};

// Tree depth: log_n levels, or h = log_n - 4 with early-terminated leaves (R20).
inline uint32_t tree_levels(uint32_t prf, uint32_t log_n) {
  return prf == DPF_PRF_CHACHA20_ET ? log_n - DPF_ET_BITS : log_n;
}

bool key_ok(const dpf_key &k) {
  const bool et = k.prf == DPF_PRF_CHACHA20_ET;
  return k.magic == DPF_KEY_MAGIC && k.version == DPF_KEY_VERSION &&
         (k.prf == DPF_PRF_CHACHA20 || k.prf == DPF_PRF_AES128 || et) && k.party <= 1 &&
         k.log_n >= (et ? DPF_ET_BITS + 1 : 1) && k.log_n <= DPF_MAX_LOG_N && (k.root[0] & 1u) == k.party &&
         k.reserved == 0 && (!et || k.cw_out == 0);
}

}  // namespace
}  // namespace dpfpir

using namespace dpfpir;

extern "C" int dpf_gen(uint32_t log_n, uint64_t alpha, uint32_t beta, uint32_t prf, const uint8_t *rng_seed,
                       dpf_key *k0, dpf_key *k1) {
  if (!k0 || !k1 || log_n < 1 || log_n > DPF_MAX_LOG_N) return DPF_EINVAL;
  if (alpha >> log_n) return DPF_EINVAL;
  if (prf != DPF_PRF_CHACHA20 && prf != DPF_PRF_AES128 && prf != DPF_PRF_CHACHA20_ET) return DPF_EUNSUPPORTED;
  const bool et = prf == DPF_PRF_CHACHA20_ET;
  if (et && log_n <= DPF_ET_BITS) return DPF_EINVAL;
  const uint32_t h = tree_levels(prf, log_n);
  uint8_t seed[32];
  if (rng_seed) {
    std::memcpy(seed, rng_seed, 32);
  } else {
    size_t got = 0;
    while (got < 32) {
      ssize_t r = getrandom(seed + got, 32 - got, 0);
      if (r <= 0) return DPF_EINVAL;
      got += size_t(r);
    }
  }
  KeystreamDrbg rng(seed);
  // Roots: t_b = b (control bit = lsb, R5).
  Words4 s[2] = {rng.next128(), rng.next128()};
  s[0][0] &= ~1u;
  s[1][0] |= 1u;
  std::memset(k0, 0, sizeof *k0);
  for (int p = 0; p < 2; ++p) {
    dpf_key &k = p ? *k1 : *k0;
    if (p) std::memset(&k, 0, sizeof k);
    k.magic = DPF_KEY_MAGIC;
    k.version = DPF_KEY_VERSION;
    k.prf = uint8_t(prf);
    k.party = uint8_t(p);
    k.log_n = uint8_t(log_n);
    to_bytes(s[p], k.root);
  }
  for (uint32_t d = 1; d <= h; ++d) {
    const unsigned keep = unsigned(alpha >> (log_n - d)) & 1u, lose = keep ^ 1u;
    Words4 P[2][2];  // P[party][child]
    prf_pair(prf, s[0], P[0][0], P[0][1]);
    prf_pair(prf, s[1], P[1][0], P[1][1]);
    // Correction (BGI-style, R2/R3): the lose child of the two parties must
    // coincide; the keep child keeps differing control bits.
    Words4 delta[2];
    delta[lose] = xor4(P[0][lose], P[1][lose]);
    delta[keep] = delta[lose];
    delta[keep][0] = (delta[keep][0] & ~1u) | ((P[0][keep][0] ^ P[1][keep][0] ^ 1u) & 1u);
    Words4 C[2][2];  // C[t][c]
    for (unsigned c = 0; c < 2; ++c) {
      C[0][c] = rng.next128();
      C[1][c] = xor4(C[0][c], delta[c]);
    }
    for (unsigned t = 0; t < 2; ++t)
      for (unsigned c = 0; c < 2; ++c) {
        to_bytes(C[t][c], k0->cw[d - 1][t][c]);
        to_bytes(C[t][c], k1->cw[d - 1][t][c]);
      }
    for (int p = 0; p < 2; ++p) s[p] = xor4(P[p][keep], C[s[p][0] & 1u][keep]);
  }
  if (et) {
    // R20: leaf codeword over the 16 words of Convert(s) = ChaCha20 block 1:
    // y0 + y1 = beta at alpha's word, 0 at the other 15.
    uint32_t W[2][16];
    for (int p = 0; p < 2; ++p) {
      const uint32_t key[8] = {s[p][0], s[p][1], s[p][2], s[p][3], 0, 0, 0, 0};
      const uint32_t nonce[3] = {0, 0, 0};
      chacha20_words(key, 1, nonce, W[p]);
    }
    const uint32_t a = uint32_t(alpha & ((1u << DPF_ET_BITS) - 1));
    for (uint32_t c = 0; c < (1u << DPF_ET_BITS); ++c) {
      const uint32_t v = (c == a ? beta : 0u) - W[0][c] + W[1][c];
      const uint32_t cw = (s[1][0] & 1u) ? 0u - v : v;
      st32(k0->cw[h][0][0] + 4 * c, cw);
      st32(k1->cw[h][0][0] + 4 * c, cw);
    }
    k0->cw_out = k1->cw_out = 0;
    return DPF_OK;
  }
  // Final Z_2^32 correction (R7): y0 + y1 = beta at alpha.
  const uint32_t v = beta - s[0][1] + s[1][1];
  const uint32_t cw_out = (s[1][0] & 1u) ? 0u - v : v;
  k0->cw_out = k1->cw_out = cw_out;
  return DPF_OK;
}

extern "C" size_t dpf_key_wire_size(uint32_t log_n) {
  if (log_n < 1 || log_n > DPF_MAX_LOG_N) return 0;
  return 32u + 64u * size_t(log_n);
}

extern "C" size_t dpf_key_wire_size_prf(uint32_t log_n, uint32_t prf) {
  if (prf == DPF_PRF_CHACHA20 || prf == DPF_PRF_AES128) return dpf_key_wire_size(log_n);
  if (prf != DPF_PRF_CHACHA20_ET || log_n <= DPF_ET_BITS || log_n > DPF_MAX_LOG_N) return 0;
  return 32u + 64u * size_t(log_n - DPF_ET_BITS) + 64u;  // h columns + CWL
}

extern "C" int dpf_key_serialize(const dpf_key *k, uint8_t *out, size_t cap, size_t *written) {
  if (!k || !out) return DPF_EINVAL;
  if (!key_ok(*k)) return DPF_EKEY;
  const size_t need = dpf_key_wire_size_prf(k->log_n, k->prf);
  if (cap < need) return DPF_EINVAL;
  st32(out, k->magic);
  out[4] = k->version; out[5] = k->prf; out[6] = k->party; out[7] = k->log_n;
  st32(out + 8, k->cw_out);
  st32(out + 12, 0);
  std::memcpy(out + 16, k->root, 16);
  // cw[d-1][t][c] is already laid out level-major, t, c: 64 bytes per level.
  std::memcpy(out + 32, k->cw, need - 32);  // ET: h columns, then CWL in column h
  if (written) *written = need;
  return DPF_OK;
}

extern "C" int dpf_key_deserialize(const uint8_t *in, size_t len, dpf_key *k) {
  if (!in || !k) return DPF_EINVAL;
  if (len < 32) return DPF_EKEY;
  dpf_key t;
  std::memset(&t, 0, sizeof t);
  t.magic = ld32(in);
  t.version = in[4]; t.prf = in[5]; t.party = in[6]; t.log_n = in[7];
  t.cw_out = ld32(in + 8);
  t.reserved = ld32(in + 12);
  std::memcpy(t.root, in + 16, 16);
  if (!key_ok(t) || len != dpf_key_wire_size_prf(t.log_n, t.prf)) return DPF_EKEY;
  std::memcpy(t.cw, in + 32, len - 32);
  *k = t;
  return DPF_OK;
}

extern "C" int dpf_reconstruct(const uint32_t *share0, const uint32_t *share1, size_t count, uint32_t *out) {
  if (count && (!share0 || !share1 || !out)) return DPF_EINVAL;
  for (size_t i = 0; i < count; ++i) out[i] = share0[i] + share1[i];
  return DPF_OK;
}

extern "C" const char *dpf_strerror(int code) {
  switch (code) {
    case DPF_OK: return "ok";
    case DPF_EINVAL: return "invalid argument";
    case DPF_EKEY: return "malformed or inconsistent DPF key";
    case DPF_ENOMEM: return "workspace too small";
    case DPF_ECUDA: return "CUDA error";
    case DPF_EUNSUPPORTED: return "unsupported (PRF not built or no sm_100 device)";
    case DPF_EBUSY: return "busy (every pipelined-server slot holds an uncollected batch)";
    default: return "unknown status";
  }
}

extern "C" const char *dpf_version(void) { return "libdpfpir 0.2 (sm_100a, ChaCha20 / AES-128 / early-terminated ChaCha20 GGM DPF, Z_2^32 shares)"; }

// Shared with eval.cu: key validation for the device path.
namespace dpfpir {
bool host_key_valid(const dpf_key &k) { return key_ok(k); }
// The header predicate of dpf_key_deserialize on a 32-byte wire header.
bool wire_header_valid(const uint8_t *in) {
  dpf_key t;
  std::memset(&t, 0, sizeof t);
  t.magic = ld32(in);
  t.version = in[4]; t.prf = in[5]; t.party = in[6]; t.log_n = in[7];
  t.cw_out = ld32(in + 8);
  t.reserved = ld32(in + 12);
  std::memcpy(t.root, in + 16, 16);
  return key_ok(t);
}
}  // namespace dpfpir
