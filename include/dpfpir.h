/*
 * dpfpir.h -- C ABI of libdpfpir, the B200 (sm_100a) server hot path of
 * two-server DPF-based PIR (Lam et al., arXiv 2301.10904, "GPU-based Private
 * Information Retrieval for On-Device Machine Learning Inference").
 *
 * Citations: P:n = PAPER.md line n; readings R1..R14 = DESIGN.md "Readings".
 *
 * The problem statement this ABI follows:
 *   Gen(1^lambda, i) -> (k_a, k_b)                       [dpf_gen]
 *   Eval(k, j) in F_p with Eval(k_a,j) + Eval(k_b,j) = [j = i]
 *   each server returns T x Eval(k, {0..L-1})            [dpf_eval_batch]
 *   the client adds the two answers to obtain T[i]       [dpf_reconstruct]
 * Arithmetic: seeds live in F_{2^128} ("+" = XOR, R1); leaf
 * shares, table and answers live in Z_{2^32} (all share arithmetic wraps mod
 * 2^32; the table is int32 bit patterns, R13).  beta generalises the "1" of
 * the contract (R11): shares reconstruct to beta * T[alpha] mod 2^32.
 *
 * Conventions: all multi-byte integers are little-endian.  Every function
 * returns a dpf_status code (never aborts, never throws across the ABI).
 * Buffers are always owned by the caller; the library allocates nothing on
 * the evaluation path (the device workspace is caller-provided).  Its only
 * process-wide state is a mutex-guarded per-device cache of SM / co-resident
 * cluster counts used by the planners and per-host-thread key staging and
 * kernel timers, so all entry points are thread-safe and reentrant (a
 * workspace must not be used by two calls at once).
 * "device" pointers are CUDA device (or managed) pointers on the current
 * device; `stream` is a cudaStream_t passed as void* (NULL = legacy default
 * stream).  Device-side entry points are asynchronous on `stream` unless
 * stated otherwise: configuration errors are reported synchronously, device
 * faults surface at the caller's next synchronisation.
 */
#ifndef DPFPIR_H
#define DPFPIR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPF_MAX_LOG_N 32
#define DPF_KEY_MAGIC 0x4B465044u /* bytes 'D','P','F','K' read as LE u32 */
#define DPF_KEY_VERSION 1

/* PRF of the tree: ChaCha20 (Table 5; the default hot-path
 * PRF) or AES-128 (the paper's baseline PRF, Table 4; on the device
 * through lane-replicated T-tables in shared memory, one conflict-free lookup
 * per S-box evaluation, so no data-dependent timing).  PRF_s(c): ChaCha20 keyed by s || 0^128,
 * bytes [16c, 16c+16) of block 0; AES-128 keyed by s on block 0^120 || c. */
enum dpf_prf { DPF_PRF_CHACHA20 = 1, DPF_PRF_AES128 = 2, DPF_PRF_CHACHA20_ET = 3 };

/* DPF_PRF_CHACHA20_ET (reading R20): the
 * ChaCha20 tree with early-terminated leaves.  Requires 5 <= log_n <= 32.
 * The tree of Eq. 3 runs to depth h = log_n - 4 only; final node i holds the
 * 16 rows 16i..16i+15, whose leaf shares come from ONE ChaCha20 block
 * Convert(s) (key s || 0^128, counter 1, nonce 0: 16 LE words W[0..15]):
 *   Eval(k, 16i + c) = (-1)^party (W[c] + lsb(s) * CWL[c])  mod 2^32.
 * 2^(h+1) - 1 = N/8 - 1 blocks per key instead of N - 1.  Not the paper's
 * key format (Table 4's 64 log2 L bytes): the key carries h codeword columns
 * plus the 16-word leaf codeword CWL (32 + 64 (log_n - 3) wire bytes). */
#define DPF_ET_BITS 4

enum dpf_status {
  DPF_OK = 0,
  DPF_EINVAL = -1,       /* bad argument: NULL pointer, size/range/alignment violation */
  DPF_EKEY = -2,         /* malformed key: magic/version/party/log_n/prf mismatch */
  DPF_ENOMEM = -3,       /* workspace too small */
  DPF_ECUDA = -4,        /* CUDA launch/config error (reported synchronously) */
  DPF_EUNSUPPORTED = -6, /* unknown PRF id, feature not built, no sm_100 device */
  DPF_EBUSY = -7         /* pipelined server: every slot holds an uncollected batch */
};

/* One party's DPF key (two codeword matrices C_0, C_1; P:349 root
 * P(0,0) = C_0[0,0]).  Reading R3: the root (column 0) is stored separately
 * and is party-specific; columns d = 1..log_n are cw[d-1][t][c] = C_t[c, d],
 * shared by both parties (R4).  cw_out is the final Z_2^32 correction (R7).
 * DPF_PRF_CHACHA20_ET (R20): columns d = 1..h = log_n - 4 as above; cw[h]
 * (the next 64 bytes) holds CWL[0..15] as 16 little-endian u32; cw_out = 0.
 * POD, fixed size, caller-owned.  Invariant: lsb(root[0]) == party. */
typedef struct dpf_key {
  uint32_t magic;        /* DPF_KEY_MAGIC */
  uint8_t version;       /* DPF_KEY_VERSION */
  uint8_t prf;           /* enum dpf_prf */
  uint8_t party;         /* 0 or 1 */
  uint8_t log_n;         /* tree depth n, 1..DPF_MAX_LOG_N; domain 2^n rows */
  uint32_t cw_out;       /* final correction word in Z_2^32 */
  uint32_t reserved;     /* 0 */
  uint8_t root[16];      /* s^(0) = P(0,0) */
  uint8_t cw[DPF_MAX_LOG_N][2][2][16];
} dpf_key;

/* ---------------------------------------------------------------- client */

/* Gen (construction per [dpf_1], written out in
 * DESIGN.md "Gen").  Builds k0 (party 0) and k1 (party 1) so that for every
 * j < 2^log_n: Eval(k0,j) + Eval(k1,j) = beta if j == alpha else 0 (mod 2^32).
 * rng_seed: 32 bytes keying the ChaCha20 DRBG that draws the roots and
 * codewords (deterministic for tests); NULL draws the seed from getrandom().
 * Cost: 2*log_n ChaCha20 blocks (ET: 2h + 2).  Errors: DPF_EINVAL if log_n
 * not in [1, 32] ([5, 32] for DPF_PRF_CHACHA20_ET), alpha >= 2^log_n, k0/k1
 * NULL; DPF_EUNSUPPORTED if prf is not one of enum dpf_prf. */
int dpf_gen(uint32_t log_n, uint64_t alpha, uint32_t beta, uint32_t prf, const uint8_t *rng_seed,
            dpf_key *k0, dpf_key *k1);

/* Wire size of a key: 32-byte header + 64*log_n payload bytes.  The payload
 * equals Table 4's "Bytes" column exactly (896/1280/1408 B at 2^14/2^20/2^22
 * entries).  Returns 0 if log_n is out of range. */
size_t dpf_key_wire_size(uint32_t log_n);

/* Wire size for a given scheme: dpf_key_wire_size(log_n) for ChaCha20 and
 * AES-128; 32 + 64 (log_n - 3) for DPF_PRF_CHACHA20_ET (h codeword columns +
 * the 64-byte CWL).  0 if (log_n, prf) is invalid. */
size_t dpf_key_wire_size_prf(uint32_t log_n, uint32_t prf);

/* Serialize k into out[0..cap).  Wire format:
 * magic u32 | version u8 | prf u8 | party u8 | log_n u8 | cw_out u32 |
 * reserved u32 | root[16] | for d=1..n: cw[d-1][0][0], cw[d-1][0][1],
 * cw[d-1][1][0], cw[d-1][1][1] (16 B each).  ET keys: d = 1..h, then CWL
 * (64 B).  *written (optional) receives the byte count
 * (dpf_key_wire_size_prf).  Errors: DPF_EINVAL (NULL, cap too small),
 * DPF_EKEY. */
int dpf_key_serialize(const dpf_key *k, uint8_t *out, size_t cap, size_t *written);

/* Parse a wire key.  Errors: DPF_EINVAL (NULL), DPF_EKEY (bad magic/version/
 * prf/party, log_n out of range, len != dpf_key_wire_size_prf(log_n, prf),
 * lsb(root) != party, reserved != 0, ET key with cw_out != 0). */
int dpf_key_deserialize(const uint8_t *in, size_t len, dpf_key *k);

/* Client-side reconstruction: out[i] = share0[i] + share1[i] mod 2^32.
 * Host pointers; out may alias either input.  Errors: DPF_EINVAL (NULL with
 * count > 0). */
int dpf_reconstruct(const uint32_t *share0, const uint32_t *share1, size_t count, uint32_t *out);

/* ---------------------------------------------------------------- server */

/* Device workspace bytes needed by dpf_eval_batch_shard for B keys of depth
 * log_n over row_count rows of D words.  0 on invalid arguments. */
size_t dpf_eval_workspace_bytes(uint32_t B, uint32_t log_n, uint64_t row_count, uint32_t D);

/* Server answer for a batch ("batched together as a single
 * matrix-matrix multiplication"):
 *   shares[b][d] = sum_{j < N} Eval(keys[b], j) * table[j][d]  (mod 2^32)
 * keys:   HOST array of B keys (same log_n, same prf); copied to the device
 *         inside the call (they may be reused as soon as the call returns).
 * table:  DEVICE, N x D uint32 (int32 bit patterns), row-major, 16-byte
 *         aligned; N <= 2^log_n (rows >= N are absent = zero rows, R12).
 * shares: DEVICE, B x D uint32, overwritten (not accumulated).
 * workspace: DEVICE, >= dpf_eval_workspace_bytes(B, log_n, N, D) bytes,
 *         256-byte aligned; must not be used concurrently by another call.
 * Requirements: B >= 1, 1 <= D <= 1024 with D % 4 == 0, 1 <= N <= 2^log_n.
 * Errors: DPF_EINVAL, DPF_EKEY (malformed key or keys disagree on log_n/prf),
 * DPF_ENOMEM (workspace too small), DPF_EUNSUPPORTED (prf), DPF_ECUDA. */
int dpf_eval_batch(const dpf_key *keys, uint32_t B, const uint32_t *table, uint64_t N, uint32_t D,
                   uint32_t *shares, void *workspace, size_t workspace_bytes, void *stream);

/* Row-sharded answer (the multi-GPU split of P:536-540: "each of the N GPUs
 * evaluate the DPF on a subset of the table indices, then summing"):
 *   partial[b][d] = sum_{row_begin <= j < row_begin+row_count}
 *                     Eval(keys[b], j) * table_shard[j - row_begin][d]
 * table_shard points at row row_begin of the logical table.  Partials of any
 * partition of [0, N) sum (mod 2^32) to dpf_eval_batch's shares.  Same
 * arguments, ownership and errors as dpf_eval_batch, plus
 * row_begin + row_count <= 2^log_n. */
int dpf_eval_batch_shard(const dpf_key *keys, uint32_t B, const uint32_t *table_shard,
                         uint64_t row_begin, uint64_t row_count, uint32_t D, uint32_t *partial_shares,
                         void *workspace, size_t workspace_bytes, void *stream);

/* Device-resident keys: as dpf_eval_batch_shard, but the B keys are already
 * on the device as consecutive wire-format records (dpf_key_serialize
 * output, stride dpf_key_wire_size_prf(log_n, prf) bytes, 16-byte aligned
 * base), e.g. received by the server straight into HBM; `prf` (enum dpf_prf)
 * must be the keys' PRF.  The keys are NOT re-validated (device memory is not read by
 * the host): callers validate at dpf_key_deserialize time.  No host->device
 * traffic; fully asynchronous; the keys are read in place (never modified). */
int dpf_eval_batch_wire(const uint8_t *keys_wire_dev, uint32_t B, uint32_t log_n, uint32_t prf,
                        const uint32_t *table_shard,
                        uint64_t row_begin, uint64_t row_count, uint32_t D, uint32_t *partial_shares,
                        void *workspace, size_t workspace_bytes, void *stream);

/* ---- graph-captured serving step (one fixed shape) ----
 * dpf_server_create captures, on `stream`, one whole serving step for B keys
 * of (log_n, prf) against a table shard (row-major, or packed = 1 for a
 * dpf_table_pack'ed one) as a CUDA graph: H2D of the keys from a pinned
 * staging buffer, zeroing, top BFS, fused kernel, D2H of the B x D answers
 * into pinned memory.  dpf_server_run copies host wire keys (B records of
 * dpf_key_wire_size_prf(log_n, prf) bytes; headers checked: DPF_EKEY) into
 * the staging buffer, replays the graph with ONE launch, waits, and copies
 * the answers to shares_host.  The caller owns `table` and `workspace`
 * (DEVICE, >= dpf_server_workspace_bytes, 256-byte aligned) for the server's
 * lifetime; the library owns the two pinned buffers (freed by destroy).
 * `stream` is synchronised once at create (the table must be ready); the
 * server captures and replays on its own stream.  Not thread-safe per server
 * object. */
typedef struct dpf_server dpf_server;
size_t dpf_server_workspace_bytes(uint32_t B, uint32_t log_n, uint32_t prf, uint64_t row_count, uint32_t D);
int dpf_server_create(uint32_t B, uint32_t log_n, uint32_t prf, const void *table, int packed, uint64_t row_begin,
                      uint64_t row_count, uint32_t D, void *workspace, size_t workspace_bytes, void *stream,
                      dpf_server **out);
int dpf_server_run(dpf_server *server, const uint8_t *keys_wire_host, uint32_t *shares_host);
void dpf_server_destroy(dpf_server *server);

/* ---- pipelined serving: up to `depth` batches in flight ----
 * dpf_server_pipeline_create builds `depth` (1..DPF_SERVER_MAX_DEPTH) slots,
 * each a captured serving step as above with its own pinned staging, answer
 * buffer, stream and workspace region (workspace >=
 * dpf_server_pipeline_workspace_bytes(..., depth)).  dpf_server_submit checks
 * the headers, copies one batch's host wire keys into the next free slot and
 * launches its graph without waiting (DPF_EBUSY when all slots hold
 * uncollected batches); dpf_server_collect waits for the OLDEST batch in
 * flight and copies its B x D answers to shares_host (DPF_EINVAL if none).
 * Consecutive batches overlap: one batch's key upload, top BFS and answer
 * download run beside its predecessor's fused kernel.  dpf_server_create is
 * the depth-1 case; dpf_server_run = submit + collect (DPF_EBUSY if a batch
 * is in flight).  destroy waits for batches in flight.  Not thread-safe per
 * server object. */
#define DPF_SERVER_MAX_DEPTH 4
size_t dpf_server_pipeline_workspace_bytes(uint32_t B, uint32_t log_n, uint32_t prf, uint64_t row_count, uint32_t D,
                                           uint32_t depth);
int dpf_server_pipeline_create(uint32_t B, uint32_t log_n, uint32_t prf, const void *table, int packed,
                               uint64_t row_begin, uint64_t row_count, uint32_t D, uint32_t depth, void *workspace,
                               size_t workspace_bytes, void *stream, dpf_server **out);
int dpf_server_submit(dpf_server *server, const uint8_t *keys_wire_host);
int dpf_server_collect(dpf_server *server, uint32_t *shares_host);

/* ---- fused cross-GPU reduction (multi-GPU row sharding) ----
 * The G row shards' partial answers sum to the answer (Z_2^32 is a group).
 * Instead of a separate collective, each rank's fused kernel can add its
 * partial shares straight into ONE rank's answer buffer over NVLink: the
 * epilogue's red.global.add.u32 targets a peer-mapped pointer, so the
 * reduction overlaps the evaluation tile by tile.
 *
 * dpf_eval_batch_wire_ex: dpf_eval_batch_wire (packed = 0, `table` = the
 * row-major shard) or dpf_eval_batch_wire_packed (packed = 1, `table` = the
 * packed shard) with flags:
 *   DPF_EVAL_ACCUMULATE  add into `shares` (B x D u32) instead of zeroing and
 *                        overwriting it; `shares` may be a peer GPU's buffer
 *                        opened with dpf_ipc_open.  The buffer's owner zeroes
 *                        it before any rank launches, and reads it after every
 *                        rank's launch completed (caller-side barrier).
 * Errors: as dpf_eval_batch_wire; DPF_EINVAL for unknown flag bits. */
#define DPF_EVAL_ACCUMULATE 1u
int dpf_eval_batch_wire_ex(const uint8_t *keys_wire_dev, uint32_t B, uint32_t log_n, uint32_t prf,
                           const void *table, int packed, uint64_t row_begin, uint64_t row_count, uint32_t D,
                           uint32_t *shares, uint32_t flags, void *workspace, size_t workspace_bytes, void *stream);

/* CUDA IPC for the answer buffer: dpf_ipc_export writes the handle of the
 * DEVICE allocation containing dev_ptr (64 opaque bytes, sent to the other
 * ranks by the caller) and dev_ptr's byte offset inside that allocation;
 * dpf_ipc_open maps it in another process (same or peer GPU; peer access is
 * enabled lazily) and returns the allocation base (the buffer is at base +
 * offset); dpf_ipc_close unmaps a base.  Errors: DPF_EINVAL (null), DPF_ECUDA. */
#define DPF_IPC_HANDLE_BYTES 64
int dpf_ipc_export(const void *dev_ptr, uint8_t handle[DPF_IPC_HANDLE_BYTES], uint64_t *offset);
int dpf_ipc_open(const uint8_t handle[DPF_IPC_HANDLE_BYTES], void **base);
int dpf_ipc_close(void *base);

/* ---- limb-packed tables: the tcgen05 (tensor-core) contraction path ----
 * The contraction sum_j y_j T[j][d] mod 2^32 is computed on the 5th-gen
 * tensor cores (tcgen05.mma kind::i8) by splitting y and T into u8 limbs:
 * y*t mod 2^32 = sum_{s<4} 2^(8s) sum_{i+k=s} y_i t_k (DESIGN.md
 * "tcgen05 contraction").  The table must first be re-laid-out once (server
 * state) by dpf_table_pack into blocks of 8 rows:
 *   block b (rows 8b'..8b'+7 with b' = row_begin/8 + b), 32*Dp bytes,
 *   [d-tile t < Dp/128][limb k < 4][chunk c < 8][row r < 8][16 bytes: byte k
 *   of T[row][128t + 16c .. 128t + 16c + 15]]
 * with Dp = D rounded up to a multiple of 128.  Rows of the 8-row blocks
 * outside [row_begin, row_begin+row_count) and columns >= D are zero.
 * Requirements: D % 4 == 0, D <= 1024, log_n >= 3.  The kernel tiles Kt keys
 * per work item, Kt = 128 / 64 / 32 / 16 for Dp = 128 / 256 / 384-512 /
 * 640-1024 (4 limb accumulators x Dp/128 tiles x Kt columns <= 512 TMEM
 * columns), so batches of Kt keys use it fully. */

/* Bytes of the packed copy of rows [row_begin, row_begin+row_count) (8-row
 * aligned, 4*Dp bytes per row), 0 if D % 4 != 0, D > 1024 or row_count == 0. */
size_t dpf_table_packed_bytes(uint64_t row_begin, uint64_t row_count, uint32_t D);

/* Pack a row-major DEVICE table shard (row_count x D uint32, pointing at row
 * row_begin) into `packed` (DEVICE, dpf_table_packed_bytes bytes, 16-byte
 * aligned).  Asynchronous on `stream`.  Errors: DPF_EINVAL, DPF_ECUDA. */
int dpf_table_pack(const uint32_t *table_shard, uint64_t row_begin, uint64_t row_count, uint32_t D, void *packed,
                   void *stream);

/* As dpf_eval_batch_shard / dpf_eval_batch_wire, reading the packed table
 * (`packed` from dpf_table_pack with the same row_begin, row_count, D).
 * Same ownership and errors; DPF_EINVAL if D % 4 != 0 or D > 1024. */
int dpf_eval_batch_packed(const dpf_key *keys, uint32_t B, const void *packed, uint64_t row_begin,
                          uint64_t row_count, uint32_t D, uint32_t *partial_shares, void *workspace,
                          size_t workspace_bytes, void *stream);
int dpf_eval_batch_wire_packed(const uint8_t *keys_wire_dev, uint32_t B, uint32_t log_n, uint32_t prf,
                               const void *packed,
                               uint64_t row_begin, uint64_t row_count, uint32_t D, uint32_t *partial_shares,
                               void *workspace, size_t workspace_bytes, void *stream);

/* ---- grouped evaluation: many (key batch, table) pairs in one launch ----
 * For workloads of many small tables, e.g. the co-design setting of P:645-659
 * (each inference queries a small hot table and the full table of each of
 * several embedding tables, with a fixed number of keys per table).  All
 * groups share D and the PRF; tables are row-major (IMAD contraction).
 * Group g computes exactly what dpf_eval_batch_wire would:
 *   shares[b][d] = sum_{row_begin <= j < row_begin+row_count}
 *                    Eval(keys[b], j) * table[j - row_begin][d]  (mod 2^32) */
typedef struct dpf_eval_group {
  const uint8_t *keys_wire; /* DEVICE: B wire-format keys, stride dpf_key_wire_size_prf(log_n, prf), 16-B aligned */
  uint32_t B;               /* keys in this group, >= 1 */
  uint32_t log_n;           /* depth of these keys' trees */
  const uint32_t *table;    /* DEVICE: row_count x D uint32, row-major, 16-B aligned */
  uint64_t row_begin, row_count;
  uint32_t *shares;         /* DEVICE: B x D, overwritten */
} dpf_eval_group;

/* Workspace bytes for dpf_eval_grouped (0 on invalid arguments). */
size_t dpf_eval_grouped_workspace_bytes(const dpf_eval_group *groups, uint32_t n_groups, uint32_t D,
                                        uint32_t prf);

/* Evaluate n_groups groups (host array of descriptors; the device buffers
 * they point to stay caller-owned) with one zeroing, one top-BFS and one
 * fused launch (deep frontiers: + one launch per level beyond 10).  Asynchronous
 * on `stream`.  Errors: DPF_EINVAL, DPF_ENOMEM, DPF_EUNSUPPORTED, DPF_ECUDA. */
int dpf_eval_grouped(const dpf_eval_group *groups, uint32_t n_groups, uint32_t D, uint32_t prf, void *workspace,
                     size_t workspace_bytes, void *stream);

/* The same on the tensor cores: every group's `table` is its limb-packed
 * shard (dpf_table_pack with that group's row_begin, row_count and D); the
 * groups share one tcgen05 configuration (key tile = MMA N chosen to
 * minimise the padded work).  Requires log_n >= 3 (5 with early
 * termination).  Same errors. */
size_t dpf_eval_grouped_packed_workspace_bytes(const dpf_eval_group *groups, uint32_t n_groups, uint32_t D,
                                               uint32_t prf);
int dpf_eval_grouped_packed(const dpf_eval_group *groups, uint32_t n_groups, uint32_t D, uint32_t prf,
                            void *workspace, size_t workspace_bytes, void *stream);

/* ---- partial batch retrieval (PBR; reading R21) ----
 * Several rows of ONE table per client: the N rows are segmented into
 * n_bins = ceil(N / I) bins of I = 2^log_i rows (bin b = rows [bI,
 * min(bI + I, N)), the last bin ragged) and every client sends one ordinary
 * DPF key per bin over the bin's I-row domain (log_n = log_i; alpha = the
 * wanted row minus bI, or a dummy index).  A client retrieves up to n_bins
 * rows for the PRF work of one full-table query (n_bins x (I - 1)
 * blocks); rows that share a bin beyond the first are dropped by the client
 * (codesign.PbrPlan), never seen by the server.
 *   keys_wire : DEVICE, bin-major: the key of client c for bin b at
 *               keys_wire + (b * B + c) * dpf_key_wire_size_prf(log_i, prf),
 *               16-B aligned.  Every key has log_n == log_i and this prf.
 *   table     : DEVICE, the whole table: row-major N x D uint32 (packed = 0),
 *               or its dpf_table_pack copy with row_begin 0, row_count N
 *               (packed = 1: tcgen05 contraction; log_i >= 3, >= 5 for ET).
 *   shares    : DEVICE, n_bins x B x D uint32 (bin-major), overwritten:
 *               shares[b][c][d] = sum_{j < I, bI + j < N} Eval(k_{b,c}, j) T[bI + j][d].
 * One launch sequence of dpf_eval_grouped(_packed) with one group per bin.
 * Asynchronous on `stream`.  Errors: DPF_EINVAL (sizes, alignment, log_i out
 * of range, more than 2^20 bins), DPF_ENOMEM (workspace), DPF_EUNSUPPORTED
 * (prf), DPF_ECUDA. */
size_t dpf_eval_pbr_workspace_bytes(uint32_t B, uint32_t log_i, uint64_t N, uint32_t D, uint32_t prf, int packed);
int dpf_eval_pbr(const uint8_t *keys_wire, uint32_t B, uint32_t log_i, uint32_t prf, const void *table, int packed,
                 uint64_t N, uint32_t D, uint32_t *shares, void *workspace, size_t workspace_bytes, void *stream);

/* End-to-end serving call: as dpf_eval_batch_shard, but shares_host is a HOST
 * buffer (pinned for best speed) that receives the B x D answers; the call
 * synchronises `stream` before returning.  The table stays device-resident
 * (server state).  workspace_bytes must cover
 * dpf_eval_workspace_bytes(...) plus B*D*4 bytes rounded up to 256 (the
 * device copy of the answer lives after the evaluation workspace). */
int dpf_serve_batch(const dpf_key *keys, uint32_t B, const uint32_t *table_shard, uint64_t row_begin,
                    uint64_t row_count, uint32_t D, uint32_t *shares_host, void *workspace,
                    size_t workspace_bytes, void *stream);

/* Test/debug only: leaf shares leaves[b][j] = Eval(keys[b], j) for all
 * j < 2^log_n (sign applied), log_n <= 20.  DEVICE output (B x 2^log_n),
 * workspace as for dpf_eval_batch with N = 2^log_n, D = 4. */
int dpf_eval_leaves(const dpf_key *keys, uint32_t B, uint32_t *leaves, void *workspace,
                    size_t workspace_bytes, void *stream);

/* Counters of the last successful eval on this thread (host-side
 * bookkeeping of the launch plan, no device reads): ChaCha20 blocks the
 * kernels compute and kernels launched. */
typedef struct dpf_eval_stats {
  uint64_t prf_blocks;    /* total ChaCha20 blocks computed by the device */
  uint32_t kernels;       /* kernel launches issued by the call */
  uint32_t frontier_depth;/* f: BFS depth of the top kernel */
  uint32_t keys_per_tile; /* Kt */
  uint32_t nodes_per_tile;/* Ft */
  uint32_t work_items;    /* fused-kernel work items */
  uint32_t grid;          /* fused-kernel CTAs */
  uint32_t kernel_id;     /* the fused-kernel instantiation: bit 0 tcgen05, bit 1 CTA pair, bit 2 producer
                             epilogue, bit 3 small-batch key mapping, bits 4-7 y-ring stages, bits 8-11 PRF,
                             bits 12-17 producer warps,
                             bits 18-23 / 24-31 IMAD consumer keys per warp / column words per lane */
} dpf_eval_stats;
int dpf_last_eval_stats(dpf_eval_stats *out);

/* Host-only launch planning (no device calls): the plan dpf_eval_batch_shard
 * (packed = 0) or dpf_eval_batch_packed (packed = 1) would use for B keys of
 * scheme `prf` over rows [row_begin, row_begin + row_count) of D words; fills
 * *out like dpf_last_eval_stats (kernels = 0).  Errors: DPF_EINVAL (invalid
 * shape or no plan), DPF_EUNSUPPORTED (prf). */
int dpf_eval_plan(uint32_t B, uint32_t log_n, uint32_t prf, uint64_t row_begin, uint64_t row_count, uint32_t D,
                  int packed, dpf_eval_stats *out);

/* Optional instrumentation (used by bench.py): after dpf_kernel_timer_begin(C)
 * each of the next C evaluations on this thread records a CUDA event pair on
 * its stream around the fused evaluation kernel.  dpf_kernel_timer_read waits
 * for them, writes up to `capacity` per-launch durations (ms) and disables
 * the timer; *count receives the number written. */
int dpf_kernel_timer_begin(uint32_t capacity);
int dpf_kernel_timer_read(float *ms, uint32_t capacity, uint32_t *count);

/* Human-readable status text (static storage). */
const char *dpf_strerror(int code);

/* Library version string. */
const char *dpf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DPFPIR_H */
