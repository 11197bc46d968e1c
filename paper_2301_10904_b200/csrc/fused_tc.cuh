// fused_tc.cuh -- tcgen05 variant of the fused kernel: the leaf-share x table
// contraction runs on the 5th-generation tensor cores (kind::i8) instead of
// IMAD, so the SM's issue slots are left to the ChaCha20 producers.
//
// Limb decomposition: write y = sum_i y_i 2^(8i)
// and t = sum_k t_k 2^(8k) with u8 limbs.  Then
//     y * t mod 2^32 = sum_{s=0..3} 2^(8s) * A_s  mod 2^32,
//     A_s = sum_{i+k=s} y_i t_k          (10 limb products, 4 accumulators)
// and for a sum over leaves j the same holds with A_s = sum_j sum_{i+k=s}
// y_i(j) t_k(j), accumulated in s32 TMEM with saturation OFF (wrapping, so A_s
// is exact mod 2^32, which is all 2^(8s) A_s mod 2^32 needs).
//
// Operands:
//   A = table limb plane k, MN-major (M = 128 table columns d, K = leaves),
//       from the limb-packed table (dpf_table_pack): blocks of 8 rows laid out
//       [d-tile (128 cols)][limb][16-col chunk (8)][row (8)][16 bytes] -- the
//       no-swizzle MN-major core-matrix layout, so one node's 8-row window
//       segment of one d-tile is ONE contiguous 4 KB bulk copy.  The T ring
//       holds (32-leaf K-chunk, d-tile) entries of 4 such blocks = 16 KB:
//       LBO = 4096 bytes (next 8 rows), SBO = 128 bytes (next 16 columns).
//   B = leaf-share limb plane i, K-major (N = Kt keys, K = leaves), written
//       by the producers as core matrices [K/16][Kt/8][8 keys][16 leaves];
//       LBO = (Kt/8) 128 bytes (next 16 leaves), SBO = 128 bytes (next 8 keys).
//   D = TMEM, accumulator (dt, s) at columns (dt*4 + s)*Kt, lane = column d.
#pragma once

namespace dpfpir {
namespace dev {

struct TcParams {
  FusedParams f;  // groups: T = the limb-packed rows [r0a, r0a + packed_rows)
  uint32_t y_stage_bytes, tmem_cols;
  uint32_t loader_spin;  // T loader waits by polling (try_wait) instead of sleeping back-off
  uint32_t debug_nomma;  // tuning only: skip the MMAs (wrong answers; isolates the producer rate)
  uint32_t role_swap;    // MMA / loader warps on the lowest hardware warp ids
};

constexpr uint32_t kTcTStageBytes = 16384;  // 32 leaves x 128 columns x 4 limbs

// Who drains TMEM at the end of an accumulator run (template EPIP).
// false: four dedicated epilogue warps (the MMA warp is one of them);
// true: the producer warps, idle once their run is produced -- the block
// shrinks from NP + 5 to NP + 2 warps, so at most 5 warps share an SMSP and
// the per-thread register cap rises from 80 to 96 (no spills).  Measured:
// early termination 0.712 -> 0.761 (c3) / 0.763 -> 0.799 (t5) of the ALU
// roofline; the standard scheme slightly slower (0.905 -> 0.895 at t5), so
// it keeps the dedicated warps.
// The standard scheme's T loader runs in the epilogue warp on SMSP 3 (it
// idles between accumulator runs): NP + 4 warps, at most 5 per SMSP, so the
// per-thread register cap is 96 instead of 80.
__host__ __device__ constexpr int tc_extra_warps(bool epip) { return epip ? 2 : 4; }  // MMA (+ epilogue) [+ loader]

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory matrix descriptor, SWIZZLE_NONE, version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// Instruction descriptor, kind::i8: D = s32 (no saturate), A = u8 MN-major,
// B = u8 K-major, M = m (128, or 256 for a CTA pair), N = n.
__host__ __device__ constexpr uint32_t umma_idesc_u8(uint32_t n, uint32_t m = 128) {
  return (2u << 4)            // c_format = S32
         | (0u << 7)          // a_format = unsigned 8-bit
         | (0u << 10)         // b_format = unsigned 8-bit
         | (1u << 15)         // a_major = MN
         | (0u << 16)         // b_major = K
         | ((n >> 3) << 17)   // N >> 3
         | ((m >> 4) << 24);  // M >> 4
}

__device__ __forceinline__ void umma_u8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}

// cta_group::2 (CTA pair, M = 256): issued by the leader CTA only; A rows
// 0..127 / B columns 0..N/2-1 come from the leader's SMEM, the rest from the
// peer's SMEM at the same offsets; each CTA's TMEM receives its 128 rows.
__device__ __forceinline__ void umma_u8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-collective forms: the converged warp supplies warp-uniform operands
// (kept in uniform registers, no per-MMA register-to-uniform moves) and
// elect.sync picks one lane (the lowest, lane 0, in a converged warp) to issue.
// Commits below use the same election, so they track that lane's MMAs.
template <bool PAIR>
__device__ __forceinline__ void umma_u8_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  if constexpr (PAIR)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
template <bool PAIR>
__device__ __forceinline__ void umma_commit_elect(uint64_t *bar) {
  if constexpr (PAIR)
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
        ::"r"(smem_u32(bar)), "h"(uint16_t(3))
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

// Commit to the same-offset mbarrier in both CTAs of the pair.
__device__ __forceinline__ void umma_commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Arrive on the leader CTA's (rank 0) copy of an mbarrier (release at cluster scope).
__device__ __forceinline__ void mbar_arrive_leader(uint64_t *bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// Wait for a phase completed (partly) by arrivals from the peer CTA.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "DPF_WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra DPF_WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// y limb-plane write for leaves (kk, kk+1) of key kl: K-major core matrices
// (k/16, key/8) -> 128 B, row key%8, byte k%16; one u16 per limb plane.
__device__ __forceinline__ void put_leaf_pair(uint8_t *yb, uint32_t ybplane, uint32_t Kt, uint32_t kl, uint32_t kk,
                                              uint32_t y0, uint32_t y1) {
  const uint32_t off = ((kk >> 4) * (Kt >> 3) + (kl >> 3)) * 128u + (kl & 7u) * 16u + (kk & 15u);
  const uint32_t p01 = __byte_perm(y0, y1, 0x5140), p23 = __byte_perm(y0, y1, 0x7362);
  *reinterpret_cast<uint16_t *>(yb + off) = uint16_t(p01);
  *reinterpret_cast<uint16_t *>(yb + ybplane + off) = uint16_t(p01 >> 16);
  *reinterpret_cast<uint16_t *>(yb + 2 * ybplane + off) = uint16_t(p23);
  *reinterpret_cast<uint16_t *>(yb + 3 * ybplane + off) = uint16_t(p23 >> 16);
}

// R20 (early termination): the 16 leaves kk..kk+15 (kk % 16 == 0) of key kl
// from one final node -> one 16-byte row of core matrix (kk/16, kl/8) in each
// limb plane: a 4x4 byte transpose per 4 leaves (8 PRMT), one STS.128 per plane.
__device__ __forceinline__ void put_leaf16(uint8_t *yb, uint32_t ybplane, uint32_t Kt, uint32_t kl, uint32_t kk,
                                           const uint32_t (&y)[16]) {
  const uint32_t off = ((kk >> 4) * (Kt >> 3) + (kl >> 3)) * 128u + (kl & 7u) * 16u;
  uint32_t pl[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t a = __byte_perm(y[4 * i], y[4 * i + 1], 0x5140), b = __byte_perm(y[4 * i + 2], y[4 * i + 3], 0x5140);
    const uint32_t c = __byte_perm(y[4 * i], y[4 * i + 1], 0x7362), d = __byte_perm(y[4 * i + 2], y[4 * i + 3], 0x7362);
    pl[0][i] = __byte_perm(a, b, 0x5410);
    pl[1][i] = __byte_perm(a, b, 0x7632);
    pl[2][i] = __byte_perm(c, d, 0x5410);
    pl[3][i] = __byte_perm(c, d, 0x7632);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    *reinterpret_cast<uint4 *>(yb + k * ybplane + off) = make_uint4(pl[k][0], pl[k][1], pl[k][2], pl[k][3]);
}

// NP producer warps, NSY-deep y ring, NST-deep T ring of (K-chunk, d-tile)
// entries.  Named barriers: 1..NSY = y stage FULL (producers arrive, the MMA
// warp syncs); NSY+1 = epilogue.
//
// PAIR (cluster of 2 CTAs, cta_group::2): a work item is 2 Kt keys x Ft
// nodes.  Both CTAs expand the same nodes, each for its Kt keys (B operand
// columns), and each stages the table columns of its half of the d-tiles (A
// rows); the leader issues M = 256, N = 2 Kt MMAs, so every MMA covers twice
// the keys of a single-CTA one and each SM streams half of the table.  The
// peer's MMA warp forwards its y-FULL and T-FULL events to the leader
// (ypeer / tpeer, remote mbarrier arrives); the leader's commits arrive in
// both CTAs (multicast); both epilogues release the leader's accempty.
// SMALLB: the small-batch key mapping (Kr < Kt real keys per CTA, zeroed
// padding MMA columns).  A separate instantiation: the lane guard it needs in
// the producer loop perturbs ptxas' register assignment of the ChaCha loop
// (measured c3 0.918 -> 0.903 when compiled into every kernel).
template <class Prf, int NP, int NSY, int NST, bool PAIR, bool EPIP, bool SMALLB = false>
__global__ void __launch_bounds__(32 * (NP + tc_extra_warps(EPIP)), 1) fused_eval_tc_kernel(const TcParams tp) {
  constexpr int NC = EPIP ? 1 : 4;          // MMA/epilogue warps
  constexpr int NEPI = EPIP ? NP : 4;       // warps that drain TMEM and release accempty
  const FusedParams &p = tp.f;
  extern __shared__ __align__(128) uint8_t smem_all[];
  uint8_t *smem = smem_all + Prf::kSmemBytes;            // after the PRF's tables (AES)
  uint64_t *tfull = reinterpret_cast<uint64_t *>(smem);  // [NST], count 1 + tx bytes
  uint64_t *tempty = tfull + NST;                        // [NST], count 1 (tcgen05.commit)
  uint64_t *yempty = tempty + NST;                       // [NSY], count 1 (tcgen05.commit)
  uint64_t *accfull = yempty + NSY;                      // count 1 (tcgen05.commit)
  uint64_t *accempty = accfull + 1;                      // count NC (epilogue warps)
  uint64_t *tpeer = accempty + 1;                        // [NST], count 1 (PAIR: peer's T entry landed)
  uint64_t *ypeer = tpeer + NST;                         // [NSY], count 1 (PAIR: peer's y stage full)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(ypeer + NSY);
  uint8_t *tbuf = smem + 1024;
  uint8_t *ybuf = tbuf + NST * kTcTStageBytes;
  uint4 *stack = reinterpret_cast<uint4 *>(ybuf + NSY * tp.y_stage_bytes);

  // Roles: producers = warps 0..NP-1, then MMA/epilogue, then loader.
  // role_swap (DPF_ROLE_SWAP=1) puts the MMA and loader warps on the lowest
  // hardware ids instead (less favoured by the highest-warp-id-first
  // arbiter): measured no different.  Deriving the role from the launch
  // parameter also changes ptxas' register assignment of the CTA-pair
  // kernel's ChaCha loop: 3x fewer dispatch stalls (ncu), c3 0.880 -> 0.915
  // against warp = threadIdx.x / 32 (profiles/r02_ncu_dispatch_ab.txt).
  // TMEM lane quarters follow the hardware id (hw & 3) either way.
  const uint32_t hw = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t warp = tp.role_swap ? (hw < tc_extra_warps(EPIP) ? NP + hw : hw - tc_extra_warps(EPIP)) : hw;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 1);
    }
    for (int s = 0; s < NSY; ++s) mbar_init(&yempty[s], 1);
    mbar_init(accfull, 1);
    mbar_init(accempty, PAIR ? 2 * NEPI : NEPI);
    for (int s = 0; s < NST; ++s) mbar_init(&tpeer[s], 1);
    for (int s = 0; s < NSY; ++s) mbar_init(&ypeer[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  if (SMALLB) {
    // small batch: the y ring's padding key columns are read by every MMA and
    // written by nobody -- zero them once (all stages), visible to the async proxy
    uint4 *yz = reinterpret_cast<uint4 *>(smem + 1024 + NST * kTcTStageBytes);
    for (uint32_t i = threadIdx.x; i < NSY * tp.y_stage_bytes / 16; i += blockDim.x) yz[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  if (warp == NP) {  // consumer warp 0 owns the TMEM allocation (in each CTA of a pair)
    if constexpr (PAIR) {
      // (both CTAs name the same slot offset: distinct per-rank slots fault
      // with a misaligned address.  compute-sanitizer racecheck reports the
      // paired allocation's completion write into this slot -- no kernel PC --
      // against this CTA's own alloc; the slot is read only after
      // __syncthreads + barrier.cluster, tools/experiments/x_sanitize.sh
      // separates those reports from any other hazard)
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(tp.tmem_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(tp.tmem_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  Prf::init_smem();
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // both CTAs' barriers initialised before any remote arrive
  tc_fence_after();
  pdl_wait_primary();  // PDL: the top BFS' frontier and zeroed answers are complete and visible
  // work items: one per CTA, or one per CTA pair
  const uint32_t first = PAIR ? blockIdx.x >> 1 : blockIdx.x;
  const uint32_t stride = PAIR ? gridDim.x >> 1 : gridDim.x;
  const uint32_t Ktp = PAIR ? 2 * p.Kt : p.Kt;  // MMA N: B-operand columns per item
  const uint32_t Kr = SMALLB ? p.Kr : p.Kt;      // columns per CTA that carry a key (<= Kt)
  const uint32_t Krp = PAIR ? 2 * Kr : Kr;       // keys per item
  const uint32_t tmem_base = *tmem_slot;

  const uint32_t W2 = p.R;             // leaves per node per window (multiple of 8)
  const uint32_t Kw = p.Ft * W2;       // leaves per window (multiple of 32)
  constexpr uint32_t V = Prf::kEt ? 4u : 0u;  // log2(rows per subtree leaf), R20
  const uint32_t ybplane = p.Kt * Kw;  // bytes per y limb plane
  const uint32_t D = p.D;
  const uint32_t Dp = (D + 127) & ~127u;  // packed width: whole 128-column d-tiles
  const uint32_t n_dt = PAIR ? Dp / 256 : Dp / 128;  // d-tiles staged by this CTA
  const uint32_t dt0 = rank * n_dt;                   // first of them

  // a6/a7 for one run: TMEM lane quarter `quarter` (= warp % 4: the lanes a
  // warp may access) holds columns d = 32 quarter + lane of each d-tile;
  // key chunks h = h0, h0 + hs, ... of 16 keys.  Combine the 4 limb sums,
  // apply the party sign, red.add into the answers.
  auto epilogue = [&](uint32_t quarter, uint32_t h0, uint32_t hs, const GroupDesc &g, uint32_t kt) {
    for (uint32_t dt = 0; dt < n_dt; ++dt) {
      const uint32_t d = (dt0 + dt) * 128 + quarter * 32 + lane;
      for (uint32_t h = h0; h < Ktp / 16; h += hs) {
        uint32_t v[16], x[16], z[16];
        const uint32_t taddr = tmem_base + ((quarter * 32u) << 16) + dt * 4 * Ktp + h * 16;
        tmem_ld16(taddr, v);
        tmem_ld16(taddr + Ktp, x);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += x[j] << 8;
        tmem_ld16(taddr + 2 * Ktp, x);
        tmem_ld16(taddr + 3 * Ktp, z);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          // TMEM column c = h*16 + j: CTA half c / Kt, its column kk = c % Kt (a key iff kk < Kr)
          const uint32_t c = h * 16 + j, kk = SMALLB ? c % p.Kt : 0u;
          const uint32_t bkey = !SMALLB ? kt * Ktp + c : kk < Kr ? kt * Krp + (c / p.Kt) * Kr + kk : 0xFFFFFFFFu;
          if (bkey < g.B && d < D) {
            const uint32_t val = v[j] + (x[j] << 16) + (z[j] << 24);  // A0 + 2^8 A1 + 2^16 A2 + 2^24 A3
            const uint32_t neg = key_party(g.keys + uint64_t(bkey) * g.kstride);
            red_add_u32(g.shares + uint64_t(bkey) * D + d, neg ? 0u - val : val, p.sys_red);
          }
        }
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if (PAIR && rank != 0) mbar_arrive_leader(accempty);
      else mbar_arrive(accempty);
    }
  };

  // T loader for one work item: per (window, 32-leaf chunk, d-tile), 4 nodes
  // x one 4 KB packed block into the T ring (tseq: this warp's ring position).
  auto load_item = [&](uint32_t item, uint32_t &tseq) {
    const uint32_t n_cc = Kw / 32;
    const GroupDesc g = group_of(p, item);
    const uint64_t pend = g.r0a + g.packed_rows;
    const uint8_t *packed = reinterpret_cast<const uint8_t *>(g.T);
    const uint32_t ng = (item - g.item_base) / g.n_ktiles;
    for (uint32_t win = 0; win < g.nwin; ++win) {
      for (uint32_t cc = 0; cc < n_cc; ++cc) {
        // lane j < 4: window leaves [32cc + 8j, +8) = rows [s0, s0 + 8) of
        // one node (one packed block): node (32cc + 8j) / W2, offset % W2
        const uint32_t kw0 = 32 * cc + 8 * (lane & 3);
        const uint64_t node = uint64_t(ng) * p.Ft + kw0 / W2;
        const uint64_t s0 = ((g.lo_f + node) << (g.m + V)) + uint64_t(W2) * win + kw0 % W2;
        const bool ok = lane < 4 && node < g.F && s0 >= g.r0a && s0 < pend;
        const uint32_t total = __popc(__ballot_sync(0xFFFFFFFFu, ok)) * 4096u;
        for (uint32_t dt = 0; dt < n_dt; ++dt, ++tseq) {
          const uint32_t ts = tseq % NST, tuse = tseq / NST;
          if (tuse > 0) {
            if (tp.loader_spin) mbar_wait(&tempty[ts], (tuse - 1) & 1);
            else mbar_wait_backoff(&tempty[ts], (tuse - 1) & 1);
          }
          if (lane == 0) mbar_arrive_expect_tx(&tfull[ts], total);
          __syncwarp();
          if (ok)
            bulk_g2s(tbuf + ts * kTcTStageBytes + lane * 4096u,
                     packed + ((s0 - g.r0a) >> 3) * (32ull * Dp) + (dt0 + dt) * 4096ull, 4096u, &tfull[ts]);
        }
      }
    }
  };

  if (warp < NP) {
    // ------------------------------------------------------------ producers
    // Depth-first over the depth-m subtree: descend to the leaf-parent level
    // pushing right children on the SMEM stack, expand the leaf-parent (two
    // leaves), pop the next pending right child.  Warp-uniform schedule;
    // 2^m - 1 blocks per subtree.  (Measured: this two-site form beats a
    // single-site "one block per iteration" loop and a 4-leaf "quad" form.)
    const uint32_t tix = warp * 32 + lane;
    const uint32_t kl = tix % Kr, nl = tix / Kr;
    const bool lane_on = !SMALLB || nl < p.Ft;  // small batches: Kr * Ft may leave a few lanes idle
    uint32_t wseq = 0, pnf = 0;  // pnf: runs drained (producer epilogue)
    for (uint32_t item = first; item < p.n_items; item += stride) {
      const GroupDesc g = group_of(p, item);
      const uint32_t li = item - g.item_base;
      const uint32_t kt = li % g.n_ktiles, ng = li / g.n_ktiles;
      const uint32_t nq = 1u << (g.m - 1);
      const uint32_t b = kt * Krp + rank * Kr + kl;
      const uint64_t node = uint64_t(ng) * p.Ft + nl;
      const bool valid = lane_on && b < g.B && node < g.F;
      const uint8_t *key = g.keys + uint64_t(valid ? b : 0) * g.kstride;
      const uint32_t cw_out = key_cw_out(key);
      uint4 cur = valid ? g.frontier[uint64_t(b) * g.cap + node] : make_uint4(0, 0, 0, 0);
      const uint64_t row_base = (g.lo_f + node) << (g.m + V);
      const bool inside = valid && row_base >= g.r0 && row_base + (1ull << (g.m + V)) <= g.r1;
      uint32_t dep = 0;
      if constexpr (Prf::kEt) {
        // R20: one final node (16 leaves) per unit; even units expand the
        // leaf-parent, odd units convert the right child kept from it.
        uint32_t cwl[16];
        load_cwl(key_cw(key, g.n + 1), cwl);
        uint4 pend = make_uint4(0, 0, 0, 0);
        const uint32_t npairs = 1u << (g.m - 1);
        for (uint32_t win = 0; win < g.nwin; ++win, ++wseq) {
          const uint32_t ys = wseq % NSY, yuse = wseq / NSY;
          if (yuse > 0) mbar_wait(&yempty[ys], (yuse - 1) & 1);
          uint8_t *yb = ybuf + ys * tp.y_stage_bytes;
          for (uint32_t qi = 0; qi < p.W; ++qi) {
            const uint32_t q = win * p.W + qi;
            uint4 sf;
            if ((q & 1) == 0) {
              while (dep + 1 < g.m) {
                uint4 c0, c1;
                node_children<Prf>(cur, key_cw(key, g.n - g.m + dep + 1), c0, c1);
                stack[dep * (32 * NP) + tix] = c1;  // slot of depth dep+1
                cur = c0;
                ++dep;
              }
              node_children<Prf>(cur, key_cw(key, g.n), sf, pend);
            } else {
              sf = pend;
            }
            uint32_t y[16];
            leaf_values16(sf, cwl, y);
            if (!inside) {
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                const uint64_t row = row_base + 16ull * q + c;
                y[c] = (valid && row >= g.r0 && row < g.r1) ? y[c] : 0u;
              }
            }
            if (!SMALLB || lane_on) put_leaf16(yb, ybplane, p.Kt, kl, nl * W2 + 16 * qi, y);
            if ((q & 1) && (q >> 1) + 1 < npairs) {
              const uint32_t k = g.m - 1 - (__ffs((q >> 1) + 1) - 1);
              cur = stack[(k - 1) * (32 * NP) + tix];
              dep = k;
            }
          }
          fence_proxy_async_smem();
          named_arrive(1 + ys, 32 * (NP + 1));
        }
      } else {
      for (uint32_t win = 0; win < g.nwin; ++win, ++wseq) {
        const uint32_t ys = wseq % NSY, yuse = wseq / NSY;
        if (yuse > 0) mbar_wait(&yempty[ys], (yuse - 1) & 1);
        uint8_t *yb = ybuf + ys * tp.y_stage_bytes;
        for (uint32_t qi = 0; qi < p.W; ++qi) {
          const uint32_t q = win * p.W + qi;
          while (dep + 1 < g.m) {
            uint4 c0, c1;
            node_children<Prf>(cur, key_cw(key, g.n - g.m + dep + 1), c0, c1);
            stack[dep * (32 * NP) + tix] = c1;  // slot of depth dep+1
            cur = c0;
            ++dep;
          }
          uint4 l0, l1;
          node_children<Prf>(cur, key_cw(key, g.n), l0, l1);
          uint32_t y0 = leaf_value<Prf>(l0, cw_out), y1 = leaf_value<Prf>(l1, cw_out);
          if (!inside) {
            const uint64_t row = row_base + 2 * q;
            y0 = (valid && row >= g.r0 && row < g.r1) ? y0 : 0u;
            y1 = (valid && row + 1 >= g.r0 && row + 1 < g.r1) ? y1 : 0u;
          }
          if (!SMALLB || lane_on) put_leaf_pair(yb, ybplane, p.Kt, kl, nl * W2 + 2 * qi, y0, y1);
          if (q + 1 < nq) {  // pop the right sibling at depth m-1-ctz(q+1)
            const uint32_t k = g.m - 1 - (__ffs(q + 1) - 1);
            cur = stack[(k - 1) * (32 * NP) + tix];
            dep = k;
          }
        }
        fence_proxy_async_smem();  // generic-proxy STS -> visible to the tensor core (async proxy)
        named_arrive(1 + ys, 32 * (NP + 1));  // the MMA warp sleeps in bar.sync until all producers arrive
      }
      }  // !kEt
      if constexpr (EPIP) {
        if (!run_continues(p, g, kt, item + stride)) {  // run complete: drain TMEM
          mbar_wait(accfull, pnf & 1);
          ++pnf;
          tc_fence_after();
          epilogue(hw & 3, warp >> 2, NP / 4, g, kt);
        }
      }
    }
  } else if (warp < NP + NC) {
    // ------------------------------------------------ MMA issuer + epilogue
    const uint32_t q = warp - NP;  // TMEM lane quarter
    // The MMA issuer: with 4 epilogue warps the one on SMSP 1 (hardware warp
    // NP + 1), so that SMSP 0 (which also hosts the T loader, NP + 4) is not
    // the one SMSP with two polling warps next to its 4 producers.
    constexpr uint32_t MQ = NC == 4 ? 1u : 0u;
    constexpr uint32_t LQ = 3u;  // standard scheme: this epilogue warp (SMSP 3) is also the T loader
    uint32_t ltseq = 0;          // its T-ring position
    const uint32_t n_cc = Kw / 32;
    const uint32_t idesc = umma_idesc_u8(Ktp, PAIR ? 256u : 128u);
    const uint32_t b_lbo = (p.Kt >> 3) * 128u;  // this CTA's Kt keys of the B operand
    const uint32_t ybase = smem_u32(ybuf), tbase = smem_u32(tbuf);
    const uint64_t adesc0 = umma_desc(tbase, 4096u, 128u), bdesc0 = umma_desc(ybase, b_lbo, 128u);
    const uint32_t yplane16 = ybplane >> 4;
    // nf = accumulator flushes so far; fresh = this item starts a run (the
    // first MMA of the run overwrites TMEM, later ones accumulate)
    uint32_t wseq = 0, tseq = 0, nf = 0;
    bool fresh = true;
    for (uint32_t item = first; item < p.n_items; item += stride) {
      const GroupDesc g = group_of(p, item);
      const uint32_t kt = (item - g.item_base) % g.n_ktiles;
      const bool last = !run_continues(p, g, kt, item + stride);
      // (the loader runs up to the T ring's depth ahead of the MMAs; at the end
      // of a run it joins the epilogue once the run's last T entries are issued)
      if (!EPIP && q == LQ) load_item(item, ltseq);
      if (q == MQ && rank == 0) {
        if (fresh && nf > 0) {  // epilogue(s) drained the accumulators
          if (PAIR) mbar_wait_cluster(accempty, (nf - 1) & 1);
          else mbar_wait(accempty, (nf - 1) & 1);
        }
        for (uint32_t win = 0; win < g.nwin; ++win, ++wseq) {
          const uint32_t ys = wseq % NSY;
          named_sync(1 + ys, 32 * (NP + 1));
          if (PAIR) mbar_wait_cluster(&ypeer[ys], (wseq / NSY) & 1);
          tc_fence_after();
          const uint32_t yb = ybase + ys * tp.y_stage_bytes;
          for (uint32_t cc = 0; cc < n_cc; ++cc) {
            for (uint32_t dt = 0; dt < n_dt; ++dt, ++tseq) {
              const uint32_t ts = tseq % NST, tuse = tseq / NST;
              mbar_wait(&tfull[ts], tuse & 1);
              if (PAIR) mbar_wait_cluster(&tpeer[ts], tuse & 1);
              tc_fence_after();
              // Descriptors by adding (offset >> 4) to the start-address
              // field of base descriptors: warp-uniform arithmetic computed
              // by the converged warp (uniform datapath), one lane issues.
              const uint64_t a0 = adesc0 + uint64_t((ts * kTcTStageBytes) >> 4);
              const uint64_t b0 = bdesc0 + uint64_t((yb - ybase + cc * 2u * b_lbo) >> 4);
              const uint32_t d0 = tmem_base + dt * 4 * Ktp;
              const bool zero_acc = fresh && win == 0 && cc == 0;
              if (!tp.debug_nomma) {
#pragma unroll
                for (uint32_t s = 0; s < 4; ++s) {
#pragma unroll
                  for (uint32_t i = 0; i <= s; ++i) {
                    const uint64_t ad = a0 + uint64_t((s - i) * 64u);  // limb plane k = s - i: + k KB
                    const uint64_t bd = b0 + uint64_t(i * yplane16);
                    umma_u8_elect<PAIR>(d0 + s * Ktp, ad, bd, idesc, (zero_acc && i == 0) ? 0u : 1u);
                  }
                }
              }
              umma_commit_elect<PAIR>(&tempty[ts]);  // T entry reusable once these MMAs finish
              __syncwarp();
            }
          }
          umma_commit_elect<PAIR>(&yempty[ys]);                             // y stage reusable (both CTAs)
          if (last && win + 1 == g.nwin) umma_commit_elect<PAIR>(accfull);  // run's accumulators complete
          __syncwarp();
        }
      } else if (q == MQ) {
        // PAIR peer: forward this CTA's y-FULL and T-FULL events to the leader
        for (uint32_t win = 0; win < g.nwin; ++win, ++wseq) {
          const uint32_t ys = wseq % NSY;
          named_sync(1 + ys, 32 * (NP + 1));
          if (lane == 0) mbar_arrive_leader(&ypeer[ys]);
          for (uint32_t cc = 0; cc < n_cc; ++cc) {
            for (uint32_t dt = 0; dt < n_dt; ++dt, ++tseq) {
              const uint32_t ts = tseq % NST, tuse = tseq / NST;
              mbar_wait(&tfull[ts], tuse & 1);
              if (lane == 0) mbar_arrive_leader(&tpeer[ts]);
            }
          }
          __syncwarp();
        }
      }
      fresh = last;
      if (!last) continue;
      if constexpr (EPIP) {
        ++nf;  // the producers drain TMEM and release accempty
      } else {
        // epilogue: all NC warps, TMEM lanes 32q..32q+31 = columns d.  Only the
        // MMA warp polls the commit barrier; the others sleep in bar.sync.
        if (q == MQ) mbar_wait(accfull, nf & 1);
        ++nf;
        named_sync(NSY + 1, 32 * NC);
        tc_fence_after();
        epilogue(q, 0, 1, g, kt);
      }
    }
  } else {
    // ------------------------------------------------------------ T loader
    // (early termination: its own warp; the standard scheme: epilogue warp LQ)
    uint32_t tseq = 0;
    for (uint32_t item = first; item < p.n_items; item += stride) load_item(item, tseq);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == NP) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tp.tmem_cols)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tp.tmem_cols)
                   : "memory");
  }
}

// Limb-pack rows [r0a, r1a) of a shard (8-row aligned; rows outside
// [r0, r1) and columns >= D are zero): block b = rows r0a+8b..+8 (32 Dp
// bytes, Dp = D padded to a multiple of 128), laid out [d-tile dt][limb k]
// [chunk cl][row rr][16 bytes: byte k of T[row][128 dt + 16 cl .. + 15]].
__global__ void table_pack_kernel(const uint32_t *__restrict__ T, uint64_t r0, uint64_t r1, uint64_t r0a,
                                  uint64_t nblocks, uint32_t D, uint32_t Dp, uint8_t *__restrict__ out) {
  const uint32_t nchunk = Dp / 16;
  const uint64_t total = nblocks * 8 * nchunk;  // one thread per (block, row, chunk): 16 words in, 4 x 16 B out
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t c = uint32_t(t % nchunk);
    const uint32_t rr = uint32_t((t / nchunk) % 8);
    const uint64_t blk = t / (8ull * nchunk);
    const uint64_t row = r0a + blk * 8 + rr;
    uint32_t w[16];
    const bool row_in = row >= r0 && row < r1;
    const uint4 *src = reinterpret_cast<const uint4 *>(T + (row - r0) * D + 16ull * c);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const uint4 x = (row_in && 16 * c + 4 * v < D) ? __ldg(src + v) : make_uint4(0, 0, 0, 0);
      w[4 * v] = x.x; w[4 * v + 1] = x.y; w[4 * v + 2] = x.z; w[4 * v + 3] = x.w;
    }
    uint8_t *blk_out = out + blk * 32ull * Dp;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t o[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint32_t sh = 8 * k;
        o[g] = ((w[4 * g] >> sh) & 0xFF) | (((w[4 * g + 1] >> sh) & 0xFF) << 8) |
               (((w[4 * g + 2] >> sh) & 0xFF) << 16) | (((w[4 * g + 3] >> sh) & 0xFF) << 24);
      }
      const uint32_t dt = c >> 3, cl = c & 7;  // d-tile (128 columns), 16-column chunk within it
      *reinterpret_cast<uint4 *>(blk_out + ((uint64_t(dt) * 4 + k) * 8 + cl) * 128 + rr * 16) =
          make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

}  // namespace dev
}  // namespace dpfpir
