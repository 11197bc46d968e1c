/*
 * dpf_oracle.c -- plain, slow, obviously-correct CPU ORACLE for the DPF-PIR
 * server hot path of Lam et al., "GPU-based Private Information Retrieval for
 * On-Device Machine Learning Inference" (arXiv 2301.10904).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA product
 * in paper_2301_10904_b200/ (which has its own independent ChaCha20, Gen and
 * key codec); neither side includes or links the other.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, RFC = RFC 8439.
 * Readings of the paper where it is silent are numbered R1..R14 and listed in
 * DESIGN.md ("Readings of the paper").
 *
 * Everything is scalar C99 with uint32_t arithmetic (wraps mod 2^32; no signed
 * overflow anywhere).  No blocking, fusion or reordering beyond the plain
 * definitions below.
 *
 * Pins (tests/test_oracle_*.py): RFC 8439 printed vectors + the `cryptography`
 * library for the block function; the DPF contract of P:314-317 exhaustively
 * at small n; eval_point == eval_full; the path-parity invariant;
 * PRF-block counts (N-1 per full eval, n per point, 2n per Gen); Table 4 key
 * sizes; numpy uint32 matmul for the contraction; naive PIR
 * (P:293-294); reconstruction = beta * T[alpha]; shard linearity
 * (P:536-540).
 *
 * SURVEY 8(f) row f4 (prf 3, reading R20): early-terminated leaves -- pinned
 * by the same DPF contract (exhaustive at small n), Convert == the library
 * ChaCha20 keystream block 1, block counts 2^(h+1)-1 / h+1 / 2h+2, key size
 * 32 + 64 (log_n - 3), and tree columns identical to a depth-h ChaCha20 key
 * drawn from the same DRBG seed.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ------------------------------------------------------------------------ */
/* O1. ChaCha20 block function, RFC 8439 section 2.3 (quarter round 2.1).    */
/* ------------------------------------------------------------------------ */

static uint32_t rotl32(uint32_t v, int c) { return (v << c) | (v >> (32 - c)); }

static uint32_t load_le32(const uint8_t *p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

static void store_le32(uint8_t *p, uint32_t v) {
    p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}

/* RFC 8439 2.1: a += b; d ^= a; d <<<= 16; c += d; b ^= c; b <<<= 12;
 *               a += b; d ^= a; d <<<= 8;  c += d; b ^= c; b <<<= 7;      */
static void quarter_round(uint32_t *x, int a, int b, int c, int d) {
    x[a] += x[b]; x[d] ^= x[a]; x[d] = rotl32(x[d], 16);
    x[c] += x[d]; x[b] ^= x[c]; x[b] = rotl32(x[b], 12);
    x[a] += x[b]; x[d] ^= x[a]; x[d] = rotl32(x[d], 8);
    x[c] += x[d]; x[b] ^= x[c]; x[b] = rotl32(x[b], 7);
}

/* RFC 8439 2.3: state = constants | key (8 LE words) | counter | nonce (3 LE
 * words); 20 rounds (10 x column round + diagonal round); add the input
 * state; serialize little-endian. */
void oracle_chacha20_block(const uint8_t key[32], uint32_t counter, const uint8_t nonce[12],
                           uint8_t out[64]) {
    uint32_t init[16], x[16];
    int i;
    init[0] = 0x61707865u; init[1] = 0x3320646eu; init[2] = 0x79622d32u; init[3] = 0x6b206574u;
    for (i = 0; i < 8; i++) init[4 + i] = load_le32(key + 4 * i);
    init[12] = counter;
    for (i = 0; i < 3; i++) init[13 + i] = load_le32(nonce + 4 * i);
    memcpy(x, init, sizeof x);
    for (i = 0; i < 10; i++) {
        quarter_round(x, 0, 4, 8, 12);  /* column round */
        quarter_round(x, 1, 5, 9, 13);
        quarter_round(x, 2, 6, 10, 14);
        quarter_round(x, 3, 7, 11, 15);
        quarter_round(x, 0, 5, 10, 15); /* diagonal round */
        quarter_round(x, 1, 6, 11, 12);
        quarter_round(x, 2, 7, 8, 13);
        quarter_round(x, 3, 4, 9, 14);
    }
    for (i = 0; i < 16; i++) store_le32(out + 4 * i, x[i] + init[i]);
}

/* ------------------------------------------------------------------------ */
/* O1a. AES-128, FIPS-197 (the paper's baseline PRF, Table 4).  */
/* Byte-oriented, straight from the standard: the S-box is built from its    */
/* definition (5.1.1: multiplicative inverse in GF(2^8) mod x^8+x^4+x^3+x+1, */
/* then the affine map with c = 0x63), not typed in.                          */
/* ------------------------------------------------------------------------ */

static uint8_t gf_mul(uint8_t a, uint8_t b) { /* FIPS-197 4.2 */
    uint8_t p = 0;
    int i;
    for (i = 0; i < 8; i++) {
        if (b & 1) p ^= a;
        b >>= 1;
        a = (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1B : 0x00));
    }
    return p;
}

static uint8_t aes_sbox_entry(uint8_t x) { /* FIPS-197 5.1.1 */
    uint8_t inv = 0, b;
    int y, i;
    if (x) {
        for (y = 1; y < 256; y++)
            if (gf_mul(x, (uint8_t)y) == 1) { inv = (uint8_t)y; break; }
    }
    b = 0;
    for (i = 0; i < 8; i++) {
        int bit = ((inv >> i) ^ (inv >> ((i + 4) & 7)) ^ (inv >> ((i + 5) & 7)) ^ (inv >> ((i + 6) & 7)) ^
                   (inv >> ((i + 7) & 7)) ^ (0x63 >> i)) & 1;
        b |= (uint8_t)(bit << i);
    }
    return b;
}

static uint8_t aes_sbox[256];
static pthread_once_t aes_once = PTHREAD_ONCE_INIT;
static void aes_init(void) {
    int x;
    for (x = 0; x < 256; x++) aes_sbox[x] = aes_sbox_entry((uint8_t)x);
}

uint8_t oracle_aes_sbox(uint8_t x) {
    pthread_once(&aes_once, aes_init);
    return aes_sbox[x];
}

/* FIPS-197 5.2 KeyExpansion (Nk = 4, Nr = 10) and 5.1 Cipher.  State s[r + 4c]
 * = in[r + 4c] (3.4). */
void oracle_aes128_encrypt(const uint8_t key[16], const uint8_t in[16], uint8_t out[16]) {
    uint8_t w[176], st[16], t[4], tmp[16];
    int i, r, c, round;
    uint8_t rcon = 0x01;
    pthread_once(&aes_once, aes_init);
    memcpy(w, key, 16);
    for (i = 4; i < 44; i++) {
        memcpy(t, w + 4 * (i - 1), 4);
        if (i % 4 == 0) {
            uint8_t u = t[0]; /* RotWord */
            t[0] = aes_sbox[t[1]]; t[1] = aes_sbox[t[2]]; t[2] = aes_sbox[t[3]]; t[3] = aes_sbox[u]; /* SubWord */
            t[0] ^= rcon;
            rcon = (uint8_t)((rcon << 1) ^ ((rcon & 0x80) ? 0x1B : 0));
        }
        for (r = 0; r < 4; r++) w[4 * i + r] = (uint8_t)(w[4 * (i - 4) + r] ^ t[r]);
    }
    for (i = 0; i < 16; i++) st[i] = (uint8_t)(in[i] ^ w[i]); /* AddRoundKey(0) */
    for (round = 1; round <= 10; round++) {
        for (i = 0; i < 16; i++) st[i] = aes_sbox[st[i]];                 /* SubBytes */
        for (r = 0; r < 4; r++)                                           /* ShiftRows */
            for (c = 0; c < 4; c++) tmp[r + 4 * c] = st[r + 4 * ((c + r) % 4)];
        memcpy(st, tmp, 16);
        if (round != 10) {                                                /* MixColumns */
            for (c = 0; c < 4; c++) {
                uint8_t a0 = st[4 * c], a1 = st[4 * c + 1], a2 = st[4 * c + 2], a3 = st[4 * c + 3];
                st[4 * c] = (uint8_t)(gf_mul(2, a0) ^ gf_mul(3, a1) ^ a2 ^ a3);
                st[4 * c + 1] = (uint8_t)(a0 ^ gf_mul(2, a1) ^ gf_mul(3, a2) ^ a3);
                st[4 * c + 2] = (uint8_t)(a0 ^ a1 ^ gf_mul(2, a2) ^ gf_mul(3, a3));
                st[4 * c + 3] = (uint8_t)(gf_mul(3, a0) ^ a1 ^ a2 ^ gf_mul(2, a3));
            }
        }
        for (i = 0; i < 16; i++) st[i] ^= w[16 * round + i];             /* AddRoundKey */
    }
    memcpy(out, st, 16);
}

/* ------------------------------------------------------------------------ */
/* O1'. The tree PRF ("PRF_s(x) encrypts a message x with an          */
/* encryption key s"; ChaCha20 per P:532, Table 5).  Reading R8: key = */
/* s || 0^128, counter 0, nonce 0; child c = keystream bytes [16c, 16c+16)   */
/* ("second 128-bit keystream block under zero key/nonce").  Reading    */
/* R9: one block per internal node yields both children.                    */
/* ------------------------------------------------------------------------ */

#define ORACLE_PRF_CHACHA20 1
#define ORACLE_PRF_AES128 2
/* SURVEY 8(f) row f4, reading R20: the ChaCha20 tree with early-terminated
 * leaves.  The GGM tree stops ET_BITS = 4 levels early (tree depth
 * h = log_n - 4); each final node s yields the 16 leaves 16i..16i+15 from the
 * 16 words of ONE ChaCha20 block, Convert(s) (below), corrected by a 16-word
 * leaf codeword.  Levels 1..h follow Eq. 3 exactly as for ChaCha20. */
#define ORACLE_PRF_CHACHA20_ET 3
#define ORACLE_ET_BITS 4
#define ORACLE_ET_LEAVES 16

/* Reading R8 (AES): PRF_s(c) = AES-128 with key s on the block 0^120 || c
 * (big-endian counter, SP 800-38A CTR); one key schedule, two encryptions
 * per internal node (R9). */
static void prf_both_aes(const uint8_t s[16], uint8_t child0[16], uint8_t child1[16], uint64_t *blocks) {
    uint8_t blk[16];
    memset(blk, 0, 16);
    oracle_aes128_encrypt(s, blk, child0);
    blk[15] = 1;
    oracle_aes128_encrypt(s, blk, child1);
    if (blocks) *blocks += 1;
}

static void prf_both_chacha(const uint8_t s[16], uint8_t child0[16], uint8_t child1[16], uint64_t *blocks) {
    uint8_t key[32], nonce[12], ks[64];
    memset(key, 0, sizeof key);
    memcpy(key, s, 16);
    memset(nonce, 0, sizeof nonce);
    oracle_chacha20_block(key, 0u, nonce, ks);
    memcpy(child0, ks, 16);
    memcpy(child1, ks + 16, 16);
    if (blocks) *blocks += 1;
}

static void prf_both(uint32_t prf, const uint8_t s[16], uint8_t child0[16], uint8_t child1[16], uint64_t *blocks) {
    /* ORACLE_PRF_CHACHA20_ET expands its tree levels with ChaCha20 (R20) */
    if (prf == ORACLE_PRF_AES128)
        prf_both_aes(s, child0, child1, blocks);
    else
        prf_both_chacha(s, child0, child1, blocks);
}

/* R20: Convert(s) = the 16 little-endian words of the ChaCha20 block keyed by
 * s || 0^128 with counter 1 and nonce 0 (block 1 of the same keystream whose
 * block 0 is the tree PRF: a final node is never expanded, and the distinct
 * counter keeps conversion and expansion outputs apart). */
static void convert_chacha(const uint8_t s[16], uint32_t w[ORACLE_ET_LEAVES], uint64_t *blocks) {
    uint8_t key[32], nonce[12], ks[64];
    int i;
    memset(key, 0, sizeof key);
    memcpy(key, s, 16);
    memset(nonce, 0, sizeof nonce);
    oracle_chacha20_block(key, 1u, nonce, ks);
    for (i = 0; i < ORACLE_ET_LEAVES; i++) w[i] = load_le32(ks + 4 * i);
    if (blocks) *blocks += 1;
}

void oracle_convert(const uint8_t s[16], uint32_t w[ORACLE_ET_LEAVES]) { convert_chacha(s, w, NULL); }

void oracle_prf(const uint8_t s[16], uint32_t c, uint8_t out[16]) {
    uint8_t c0[16], c1[16];
    prf_both(ORACLE_PRF_CHACHA20, s, c0, c1, NULL);
    memcpy(out, c ? c1 : c0, 16);
}

void oracle_prf_aes(const uint8_t s[16], uint32_t c, uint8_t out[16]) {
    uint8_t c0[16], c1[16];
    prf_both(ORACLE_PRF_AES128, s, c0, c1, NULL);
    memcpy(out, c ? c1 : c0, 16);
}

/* Reading R5: control bit of a seed = its least significant bit, lsb(s) =
 * s[0] & 1 ("P(d-1, floor(j/2)) mod 2").  Reading R6: the leaf's
 * Z_2^32 value w1(s) = little-endian u32 of bytes 4..7 (disjoint from the
 * control bit). */
static uint32_t lsb_of(const uint8_t s[16]) { return (uint32_t)(s[0] & 1u); }
static uint32_t w1_of(const uint8_t s[16]) { return load_le32(s + 4); }

static void xor16(uint8_t *dst, const uint8_t *a, const uint8_t *b) {
    int i;
    for (i = 0; i < 16; i++) dst[i] = a[i] ^ b[i];
}

/* ------------------------------------------------------------------------ */
/* Key.  P:342: a key holds two codeword matrices C_0, C_1 in                */
/* F_{2^lambda}^{2 x (log L + 1)}; P(0,0) = C_0[0,0] is the root.     */
/* Reading R3: column 0 is the root (stored separately, party-specific);     */
/* columns d = 1..n are stored as cw[d-1][t][c] = C_t[c, d] (64 n bytes =    */
/* Table 4's "Bytes").  Reading R4: C_0, C_1 shared by both keys. */
/* Reading R7: cw_out, the final Z_2^32 correction.                           */
/* The oracle's own struct; it is NOT the product's dpf_key.                 */
/* ------------------------------------------------------------------------ */

#define ORACLE_MAX_LOG_N 32

typedef struct {
    uint32_t log_n;
    uint32_t party;
    uint32_t cw_out;
    uint32_t prf;  /* 1 = ChaCha20, 2 = AES-128 */
    uint8_t root[16];
    uint8_t cw[ORACLE_MAX_LOG_N][2][2][16];
    uint32_t cw_leaf[ORACLE_ET_LEAVES]; /* R20 (prf 3 only): leaf correction words CWL[0..15] */
} oracle_key;

/* Depth of the GGM tree: log_n levels, or log_n - ET_BITS with early
 * termination (R20). */
static uint32_t tree_depth(uint32_t prf, uint32_t log_n) {
    return prf == ORACLE_PRF_CHACHA20_ET ? log_n - ORACLE_ET_BITS : log_n;
}

size_t oracle_key_struct_size(void) { return sizeof(oracle_key); }

/* ------------------------------------------------------------------------ */
/* Seeded DRBG for Gen (random numbers the method draws): the ChaCha20       */
/* keystream under key = rng_seed (32 B), nonce 0, counter 0,1,2,...        */
/* The product implements the same counter-based generator independently.   */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint8_t key[32];
    uint32_t counter;
    uint8_t buf[64];
    int used;
} drbg;

static void drbg_init(drbg *g, const uint8_t seed[32]) {
    memcpy(g->key, seed, 32);
    g->counter = 0;
    g->used = 64;
}

static void drbg_bytes(drbg *g, uint8_t *out, int n) {
    static const uint8_t zero_nonce[12] = {0};
    int i;
    for (i = 0; i < n; i++) {
        if (g->used == 64) {
            oracle_chacha20_block(g->key, g->counter, zero_nonce, g->buf);
            g->counter++;
            g->used = 0;
        }
        out[i] = g->buf[g->used++];
    }
}

/* ------------------------------------------------------------------------ */
/* O6. Gen(1^lambda, alpha) -> (k_0, k_1)  (the paper  */
/* defers the construction to [dpf_1]).  BGI-style, written in the    */
/* paper's two-matrix key form (readings R2, R3, R4, R7, R10, R11):          */
/*  1. r0, r1 <- 16 random bytes each; r0[0] &= 0xFE, r1[0] |= 1 (t_b = b).  */
/*  2. for d = 1..n: keep = bit_{n-d}(alpha), lose = 1 - keep;               */
/*     (P_x[0], P_x[1]) = PRF(s_x, .);                                       */
/*     Delta[lose] = P_0[lose] ^ P_1[lose];                                   */
/*     Delta[keep] = Delta[lose] with bit 0 := lsb(P_0[keep])^lsb(P_1[keep])^1*/
/*     C_0[c][d] <- 16 random bytes (c = 0 then 1); C_1[c][d] = C_0 ^ Delta[c]*/
/*     s_x <- P_x[keep] ^ C_{lsb(s_x)}[keep][d].                              */
/*  3. cw_out = (-1)^{lsb(s_1)} (beta - w1(s_0) + w1(s_1))  mod 2^32.         */
/* Draw order: r0, r1, then C_0[0][d], C_0[1][d] for d = 1..n.               */
/* Returns 0, or -1 on invalid arguments.  *blocks += 2n.                    */
/* Early termination (R20, prf 3, 5 <= log_n <= 32): step 2 runs for         */
/* d = 1..h = log_n - 4 only (same bits of alpha, MSB first); then with      */
/* W_x = Convert(s_x) and a = alpha mod 16, for k = 0..15:                   */
/*  3'. CWL[k] = (-1)^{lsb(s_1)} (beta [k = a] - W_0[k] + W_1[k])  mod 2^32, */
/*     cw_out = 0.  *blocks += 2h + 2.                                       */
/* ------------------------------------------------------------------------ */

int oracle_gen_prf(uint32_t log_n, uint64_t alpha, uint32_t beta, uint32_t prf, const uint8_t rng_seed[32],
                   oracle_key *k0, oracle_key *k1, uint64_t *blocks) {
    drbg g;
    uint8_t s0[16], s1[16], p0[2][16], p1[2][16], delta[2][16];
    uint32_t d, n = log_n;
    if (log_n < 1 || log_n > ORACLE_MAX_LOG_N || !k0 || !k1 || !rng_seed) return -1;
    if (prf != ORACLE_PRF_CHACHA20 && prf != ORACLE_PRF_AES128 && prf != ORACLE_PRF_CHACHA20_ET) return -1;
    if (prf == ORACLE_PRF_CHACHA20_ET && log_n <= ORACLE_ET_BITS) return -1;
    if (log_n < 64 && alpha >= ((uint64_t)1 << log_n)) return -1;
    memset(k0, 0, sizeof *k0);
    memset(k1, 0, sizeof *k1);
    drbg_init(&g, rng_seed);
    drbg_bytes(&g, s0, 16);
    drbg_bytes(&g, s1, 16);
    s0[0] &= 0xFEu;
    s1[0] |= 0x01u;
    memcpy(k0->root, s0, 16);
    memcpy(k1->root, s1, 16);
    k0->log_n = k1->log_n = n;
    k0->prf = k1->prf = prf;
    k0->party = 0;
    k1->party = 1;
    for (d = 1; d <= tree_depth(prf, n); d++) {
        uint32_t keep = (uint32_t)((alpha >> (n - d)) & 1u), lose = 1u - keep, c;
        uint32_t t0 = lsb_of(s0), t1 = lsb_of(s1);
        uint8_t c0cw[2][16], c1cw[2][16], next0[16], next1[16];
        prf_both(prf, s0, p0[0], p0[1], blocks);
        prf_both(prf, s1, p1[0], p1[1], blocks);
        xor16(delta[lose], p0[lose], p1[lose]);
        memcpy(delta[keep], delta[lose], 16);
        delta[keep][0] = (uint8_t)((delta[keep][0] & 0xFEu) |
                                   ((lsb_of(p0[keep]) ^ lsb_of(p1[keep]) ^ 1u) & 1u));
        for (c = 0; c < 2; c++) {
            drbg_bytes(&g, c0cw[c], 16);
            xor16(c1cw[c], c0cw[c], delta[c]);
            memcpy(k0->cw[d - 1][0][c], c0cw[c], 16);
            memcpy(k0->cw[d - 1][1][c], c1cw[c], 16);
        }
        /* s_x <- P_x[keep] ^ C_{t_x}[keep][d] */
        xor16(next0, p0[keep], t0 ? c1cw[keep] : c0cw[keep]);
        xor16(next1, p1[keep], t1 ? c1cw[keep] : c0cw[keep]);
        memcpy(s0, next0, 16);
        memcpy(s1, next1, 16);
    }
    memcpy(k1->cw, k0->cw, sizeof k0->cw);
    if (prf == ORACLE_PRF_CHACHA20_ET) {
        uint32_t w0[ORACLE_ET_LEAVES], w1[ORACLE_ET_LEAVES], kk;
        convert_chacha(s0, w0, blocks);
        convert_chacha(s1, w1, blocks);
        for (kk = 0; kk < ORACLE_ET_LEAVES; kk++) {
            uint32_t v = (kk == (uint32_t)(alpha % ORACLE_ET_LEAVES) ? beta : 0u) - w0[kk] + w1[kk];
            k0->cw_leaf[kk] = k1->cw_leaf[kk] = lsb_of(s1) ? (0u - v) : v;
        }
        k0->cw_out = k1->cw_out = 0;
        return 0;
    }
    {
        uint32_t v = beta - w1_of(s0) + w1_of(s1);
        k0->cw_out = k1->cw_out = lsb_of(s1) ? (0u - v) : v;
    }
    return 0;
}

int oracle_gen(uint32_t log_n, uint64_t alpha, uint32_t beta, const uint8_t rng_seed[32], oracle_key *k0,
               oracle_key *k1, uint64_t *blocks) {
    return oracle_gen_prf(log_n, alpha, beta, ORACLE_PRF_CHACHA20, rng_seed, k0, k1, blocks);
}

/* ------------------------------------------------------------------------ */
/* O2. Node step, Eq. 3: child(s, c, d) = PRF_s(c) + C_{s mod 2}  */
/* [c, d]; "+" in F_{2^lambda} is XOR (R1).  Child bit at depth d of leaf j  */
/* is bit (n-d) of j ("floor(j/2)", "j mod 2"; R10: MSB first).         */
/* ------------------------------------------------------------------------ */

static void node_children(const oracle_key *k, const uint8_t s[16], uint32_t d,
                          uint8_t ch0[16], uint8_t ch1[16], uint64_t *blocks) {
    uint8_t p0[16], p1[16];
    uint32_t t = lsb_of(s);
    prf_both(k->prf, s, p0, p1, blocks);
    xor16(ch0, p0, k->cw[d - 1][t][0]);
    xor16(ch1, p1, k->cw[d - 1][t][1]);
}

/* Leaf conversion (R2, R6, R7): y = (-1)^party (w1(s) + lsb(s) cw_out). */
static uint32_t leaf_value(const oracle_key *k, const uint8_t s[16]) {
    uint32_t v = w1_of(s) + lsb_of(s) * k->cw_out;
    return k->party ? (0u - v) : v;
}

/* R20 leaf conversion with early termination: final node s (depth h) holds
 * leaves 16i..16i+15; leaf 16i + kk gets
 *   y = (-1)^party (W[kk] + lsb(s) CWL[kk]),  W = Convert(s)  (one block). */
static uint32_t et_leaf_value(const oracle_key *k, const uint8_t s[16], uint32_t kk, uint64_t *blocks) {
    uint32_t w[ORACLE_ET_LEAVES], v;
    convert_chacha(s, w, blocks);
    v = w[kk] + lsb_of(s) * k->cw_leaf[kk];
    return k->party ? (0u - v) : v;
}

/* O3. Eval(k, j) = P(log L, j)  (Eq. 1): root, then n node steps
 * along the bits of j.  Exactly n PRF blocks. */
uint32_t oracle_eval_point(const oracle_key *k, uint64_t j, uint64_t *blocks) {
    uint8_t s[16], ch0[16], ch1[16];
    uint32_t d, n = k->log_n;
    memcpy(s, k->root, 16);
    for (d = 1; d <= tree_depth(k->prf, n); d++) {
        uint32_t bit = (uint32_t)((j >> (n - d)) & 1u);
        node_children(k, s, d, ch0, ch1, blocks);
        memcpy(s, bit ? ch1 : ch0, 16);
    }
    if (k->prf == ORACLE_PRF_CHACHA20_ET) return et_leaf_value(k, s, (uint32_t)(j % ORACLE_ET_LEAVES), blocks);
    return leaf_value(k, s);
}

/* O4. Full-domain expansion in level order ("level-by-level"): all
 * 2^n leaf seeds, N-1 blocks.  leaf_seeds is caller-owned 16 * 2^n bytes. */
static int expand_all(const oracle_key *k, uint8_t *seeds, uint64_t *blocks) {
    uint32_t d, n = tree_depth(k->prf, k->log_n); /* R20: final nodes at depth h */
    uint64_t i, width;
    memcpy(seeds, k->root, 16);
    for (d = 1; d <= n; d++) {
        width = (uint64_t)1 << (d - 1); /* parents at depth d-1 live at [0, width) */
        /* in place, right to left: children of i go to 2i and 2i+1 >= i */
        for (i = width; i-- > 0;) {
            uint8_t parent[16], ch0[16], ch1[16];
            memcpy(parent, seeds + 16 * i, 16);
            node_children(k, parent, d, ch0, ch1, blocks);
            memcpy(seeds + 16 * (2 * i), ch0, 16);
            memcpy(seeds + 16 * (2 * i + 1), ch1, 16);
        }
    }
    return 0;
}

int oracle_eval_full_seeds(const oracle_key *k, uint8_t *leaf_seeds, uint64_t *blocks) {
    if (!k || !leaf_seeds || k->log_n < 1 || k->log_n > 30 || k->prf == ORACLE_PRF_CHACHA20_ET) return -1;
    return expand_all(k, leaf_seeds, blocks);
}

/* Eval(k, {0..L-1}) as Z_2^32 shares ("T x Eval(k_a, {0 ... L-1})"). */
int oracle_eval_full(const oracle_key *k, uint32_t *y, uint64_t *blocks) {
    uint64_t j, N;
    uint8_t *seeds;
    if (!k || !y || k->log_n < 1 || k->log_n > 30) return -1;
    N = (uint64_t)1 << k->log_n;
    seeds = (uint8_t *)malloc((size_t)(16 * N));
    if (!seeds) return -3;
    expand_all(k, seeds, blocks);
    if (k->prf == ORACLE_PRF_CHACHA20_ET) {
        /* R20: 2^h final nodes, one Convert block each -> 16 leaves */
        uint64_t i;
        uint32_t kk;
        for (i = 0; i < (N >> ORACLE_ET_BITS); i++) {
            uint32_t w[ORACLE_ET_LEAVES];
            const uint8_t *sf = seeds + 16 * i;
            convert_chacha(sf, w, blocks);
            for (kk = 0; kk < ORACLE_ET_LEAVES; kk++) {
                uint32_t v = w[kk] + lsb_of(sf) * k->cw_leaf[kk];
                y[i * ORACLE_ET_LEAVES + kk] = k->party ? (0u - v) : v;
            }
        }
    } else {
        for (j = 0; j < N; j++) y[j] = leaf_value(k, seeds + 16 * j);
    }
    free(seeds);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O5. Contraction: out[d] = sum_{j < rows} y[j] * T[j][d]  mod 2^32 -- the   */
/* "integer dot product" between the DPF output and the table, the   */
/* table viewed as a 2-D matrix row-major rows x D.                  */
/* ------------------------------------------------------------------------ */

void oracle_contract(const uint32_t *y, uint64_t rows, const uint32_t *T, uint32_t D, uint32_t *out) {
    uint64_t j;
    uint32_t d;
    for (d = 0; d < D; d++) out[d] = 0;
    for (j = 0; j < rows; j++)
        for (d = 0; d < D; d++) out[d] += y[j] * T[j * (uint64_t)D + d];
}

/* Server answer for one key restricted to rows [row_begin, row_begin+rows):
 * shares[d] = sum_j Eval(k, row_begin + j) * T_shard[j][d]  (the
 * multi-GPU split of P:536-540 evaluates a subset of the indices).  Reading
 * R12: rows >= N simply do not exist (zero rows). */
int oracle_answer_rows(const oracle_key *k, const uint32_t *T_shard, uint64_t row_begin,
                       uint64_t rows, uint32_t D, uint32_t *shares, uint64_t *blocks) {
    uint64_t N;
    uint32_t *y;
    int rc;
    if (!k || k->log_n < 1 || k->log_n > 30) return -1;
    N = (uint64_t)1 << k->log_n;
    if (row_begin > N || rows > N - row_begin) return -1;
    y = (uint32_t *)malloc((size_t)(4 * N));
    if (!y) return -3;
    rc = oracle_eval_full(k, y, blocks);
    if (rc == 0) oracle_contract(y + row_begin, rows, T_shard, D, shares);
    free(y);
    return rc;
}

/* Batched answers: shares[b][:] for B keys ("multiple queries ...
 * batched together as a single matrix-matrix multiplication"); keys are
 * independent, so `threads` POSIX threads split the keys (no other change). */
typedef struct {
    const oracle_key *keys;
    const uint32_t *T;
    uint64_t row_begin, rows;
    uint32_t D, B, first, step;
    uint32_t *shares;
    int rc;
} batch_job;

static void *batch_worker(void *arg) {
    batch_job *job = (batch_job *)arg;
    uint32_t b;
    for (b = job->first; b < job->B; b += job->step) {
        int rc = oracle_answer_rows(&job->keys[b], job->T, job->row_begin, job->rows, job->D,
                                    job->shares + (uint64_t)b * job->D, NULL);
        if (rc) job->rc = rc;
    }
    return NULL;
}

int oracle_answer_batch(const oracle_key *keys, uint32_t B, const uint32_t *T_shard,
                        uint64_t row_begin, uint64_t rows, uint32_t D, uint32_t *shares,
                        uint32_t threads) {
    batch_job jobs[256];
    pthread_t tids[256];
    uint32_t t;
    int rc = 0;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if (threads > B) threads = B;
    for (t = 0; t < threads; t++) {
        jobs[t].keys = keys; jobs[t].T = T_shard; jobs[t].row_begin = row_begin; jobs[t].rows = rows;
        jobs[t].D = D; jobs[t].B = B; jobs[t].first = t; jobs[t].step = threads;
        jobs[t].shares = shares; jobs[t].rc = 0;
    }
    if (threads == 1) {
        batch_worker(&jobs[0]);
        return jobs[0].rc;
    }
    for (t = 0; t < threads; t++) pthread_create(&tids[t], NULL, batch_worker, &jobs[t]);
    for (t = 0; t < threads; t++) {
        pthread_join(tids[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
    }
    return rc;
}

/* O7. Reconstruct: out = share_0 + share_1 mod 2^32. */
void oracle_reconstruct(const uint32_t *s0, const uint32_t *s1, uint64_t count, uint32_t *out) {
    uint64_t i;
    for (i = 0; i < count; i++) out[i] = s0[i] + s1[i];
}

/* O8. Naive PIR: r_1 + r_2 = I(i) (here beta * e_alpha in
 * Z_2^32).  r0 is the caller's uniform vector; r1 = beta e_alpha - r0. */
void oracle_naive_pir_shares(uint64_t N, uint64_t alpha, uint32_t beta, const uint32_t *r0,
                             uint32_t *r1) {
    uint64_t j;
    for (j = 0; j < N; j++) r1[j] = (j == alpha ? beta : 0u) - r0[j];
}

/* ------------------------------------------------------------------------ */
/* Key wire format (Table 4 payload): */
/* 32-byte header  magic 'DPFK' (LE u32 0x4B465044) | version 1 | prf (1 =   */
/* ChaCha20, 2 = AES-128) | party | log_n | cw_out (LE u32) | reserved 0 |   */
/* root                                                                      */
/* then 64 n bytes: for d = 1..n: [t=0: c=0, c=1][t=1: c=0, c=1] x 16 B.     */
/* ------------------------------------------------------------------------ */

size_t oracle_key_wire_size(uint32_t log_n) { return 32u + 64u * (size_t)log_n; }

/* R20 (prf 3): the h = log_n - 4 codeword columns, then CWL[0..15] as 16 LE
 * words (64 bytes): 32 + 64 (log_n - 3) bytes. */
size_t oracle_key_wire_size_prf(uint32_t log_n, uint32_t prf) {
    if (prf == ORACLE_PRF_CHACHA20_ET) return 32u + 64u * (size_t)(log_n - ORACLE_ET_BITS) + 64u;
    return oracle_key_wire_size(log_n);
}

int oracle_key_to_wire(const oracle_key *k, uint8_t *out, size_t cap) {
    uint32_t d, t, c, h = tree_depth(k->prf, k->log_n);
    size_t need = oracle_key_wire_size_prf(k->log_n, k->prf);
    if (cap < need) return -1;
    store_le32(out, 0x4B465044u);
    out[4] = 1; out[5] = (uint8_t)k->prf; out[6] = (uint8_t)k->party; out[7] = (uint8_t)k->log_n;
    store_le32(out + 8, k->cw_out);
    store_le32(out + 12, 0);
    memcpy(out + 16, k->root, 16);
    for (d = 0; d < h; d++)
        for (t = 0; t < 2; t++)
            for (c = 0; c < 2; c++) memcpy(out + 32 + 64 * d + 32 * t + 16 * c, k->cw[d][t][c], 16);
    if (k->prf == ORACLE_PRF_CHACHA20_ET)
        for (c = 0; c < ORACLE_ET_LEAVES; c++) store_le32(out + 32 + 64 * h + 4 * c, k->cw_leaf[c]);
    return (int)need;
}

int oracle_key_from_wire(const uint8_t *in, size_t len, oracle_key *k) {
    uint32_t d, t, c, n, h;
    if (len < 32 || load_le32(in) != 0x4B465044u || in[4] != 1 || in[5] < 1 || in[5] > 3) return -2;
    n = in[7];
    if (n < 1 || n > ORACLE_MAX_LOG_N || in[6] > 1) return -2;
    if (in[5] == ORACLE_PRF_CHACHA20_ET && n <= ORACLE_ET_BITS) return -2;
    if (len != oracle_key_wire_size_prf(n, in[5])) return -2;
    h = tree_depth(in[5], n);
    memset(k, 0, sizeof *k);
    k->log_n = n;
    k->prf = in[5];
    k->party = in[6];
    k->cw_out = load_le32(in + 8);
    memcpy(k->root, in + 16, 16);
    for (d = 0; d < h; d++)
        for (t = 0; t < 2; t++)
            for (c = 0; c < 2; c++) memcpy(k->cw[d][t][c], in + 32 + 64 * d + 32 * t + 16 * c, 16);
    if (k->prf == ORACLE_PRF_CHACHA20_ET)
        for (c = 0; c < ORACLE_ET_LEAVES; c++) k->cw_leaf[c] = load_le32(in + 32 + 64 * h + 4 * c);
    return 0;
}
