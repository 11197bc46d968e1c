// eval.cu -- server half of libdpfpir: batched full-domain DPF evaluation
// fused with the mod-2^32 table contraction, for sm_100a (B200).
//
// Path (P:n = PAPER.md line n):
//   a1 key ingest    host dpf_key[] -> wire-format keys in the workspace (H2D)
//   a2 top BFS       levels 1..f of every key's GGM tree (Eq. 3)
//                    -> frontier[B][F] in HBM/L2 (P:428 level-by-level, only
//                    for the small top of the tree)
//   a3-a6 fused      persistent warp-specialised kernel, one CTA per SM:
//                    * producer warps: per-thread depth-first expansion of a
//                      depth-m subtree (the memory-bounded traversal of
//                      P:437-443 with K = one node per thread and an SMEM
//                      stack of m-1 pending right children), leaf conversion
//                      into an SMEM y-tile ring (leaves never reach HBM)
//                    * loader warp: cp.async.bulk of the matching table rows
//                      into an SMEM T-tile ring (mbarrier complete_tx); each
//                      T row is read by all keys of the tile (P:364 batched
//                      matrix-matrix product)
//                    * consumer warps: IMAD outer products acc[key][col] +=
//                      y * T in registers ("dot product ...
//                      accumulating the result in local memory"), flushed with
//                      red.global.add.u32 (exact: Z_2^32 addition is
//                      associative, P:483 tree-summation)
//   a7 output        shares[B][D] on the device, party sign applied at flush.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "chacha_dev.cuh"
#include "aes_dev.cuh"
#include "dpfpir.h"

namespace dpfpir {
bool host_key_valid(const dpf_key &k);
bool wire_header_valid(const uint8_t *header32);

namespace dev {

// ----------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "DPF_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra DPF_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Same, with a suspend-time hint: the waiting warp sleeps in hardware until
// the phase completes (or the hint elapses) instead of re-polling, so idle
// consumer/loader warps stop stealing issue slots from the PRF producers.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "DPF_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra DPF_WAITS_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x100000u)
      : "memory");
}
// Named hardware barriers for the y-tile ring: a warp blocked in bar.sync is
// descheduled (no issue slots), unlike an mbarrier try_wait poll loop.
// IDs: 1 + stage = FULL (producers arrive, consumers sync),
//      3 + stage = EMPTY (consumers arrive, producers + loader sync).
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// Backoff wait for warps that are usually far ahead of the barrier they wait
// on (the T loader): poll, then sleep 64 ns .. 2 us between polls.
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t parity) {
  uint32_t ns = 64;
  while (!mbar_test(bar, parity)) {
    __nanosleep(ns);
    ns = ns < 2048 ? 2 * ns : 2048;
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// a6 flush.  `sys`: the answers may live in another GPU's memory (peer
// mapped, DPF_EVAL_ACCUMULATE, several GPUs adding concurrently): the atomic
// must be system-scoped to be atomic across devices (PTX memory model).
__device__ __forceinline__ void red_add_u32(uint32_t *addr, uint32_t v, uint32_t sys) {
  if (sys)
    asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
  else
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
}

// Programmatic dependent launch (PDL): the top BFS lets the fused kernel
// launch as soon as all of its CTAs are running (launch_dependents); the
// fused kernel sets up its barriers / TMEM / DFS state and then waits for the
// top BFS grid to complete and its frontier writes (and the answer zeroing)
// to be visible (griddepcontrol.wait; a no-op without a PDL primary).
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_primary() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Wire-format key accessors (include/dpfpir.h).
__device__ __forceinline__ uint4 key_root(const uint8_t *k) { return __ldg(reinterpret_cast<const uint4 *>(k + 16)); }
__device__ __forceinline__ uint32_t key_cw_out(const uint8_t *k) {
  return __ldg(reinterpret_cast<const uint32_t *>(k + 8));
}
__device__ __forceinline__ uint32_t key_party(const uint8_t *k) {
  return (__ldg(reinterpret_cast<const uint32_t *>(k + 4)) >> 16) & 0xFFu;
}
// 64-byte codeword column of depth d (1-based): [t][c] x uint4
__device__ __forceinline__ const uint4 *key_cw(const uint8_t *k, uint32_t d) {
  return reinterpret_cast<const uint4 *>(k + 32 + 64u * (d - 1u));
}

// ----------------------------------------------------------------- a2: top BFS
// Levels 1..f of every key (P:428 level-by-level, only for the small top of
// the tree).  Level k's nodes intersecting the row range [r0, r1) are
// [lo_k, hi_k], lo_k = r0 >> (n-k); the frontier stores node i at [i - lo_f].
// Each expanded parent yields both children from one block (R9).
constexpr uint32_t kTopSmemLevels = 10;
// a2 in ONE launch for any frontier depth f: CTA (key b, j) owns level-s
// node p = lo_s + j of the range's level-s nodes; thread 0 walks the root
// path to it (s blocks, Eq. 3 along the bits of p), then levels s+1..f of its
// subtree (intersected with [r0, r1)) expand breadth-first in shared memory
// (<= 2^kTopSmemLevels nodes per level) and level f goes to the frontier.
// Replaces one launch per level below 2^10 nodes; s also spreads small
// batches over the SMs (the s path blocks per CTA are redundant work:
// B * 2^s * s blocks, << the B * 2^f of the frontier).
template <class Prf>
__global__ void __launch_bounds__(256) expand_top_split_kernel(const uint8_t *__restrict__ keys, uint32_t kstride,
                                                               uint32_t n, uint32_t s, uint32_t f, uint64_t r0,
                                                               uint64_t r1, uint4 *__restrict__ out, uint64_t cap,
                                                               uint4 *__restrict__ zero, uint64_t zero_vec) {
  __shared__ uint4 buf[2][1u << kTopSmemLevels];
  pdl_launch_dependents();
  if constexpr (Prf::kSmemBytes != 0) {  // AES: T-tables in dynamic SMEM
    Prf::init_smem();
    __syncthreads();
  }
  // a7's zeroing of the answers rides along (saves a launch per step)
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < zero_vec; i += uint64_t(gridDim.x) * blockDim.x)
    zero[i] = make_uint4(0, 0, 0, 0);
  const uint64_t lo_s = r0 >> (n - s), cnt_s = ((r1 - 1) >> (n - s)) - lo_s + 1;
  const uint32_t b = uint32_t(blockIdx.x / cnt_s);
  const uint64_t ps = lo_s + blockIdx.x % cnt_s;  // this CTA's level-s node
  const uint8_t *key = keys + uint64_t(b) * kstride;
  if (threadIdx.x == 0) {
    uint4 x = key_root(key);
    for (uint32_t d = 1; d <= s; ++d) {
      uint4 c0, c1;
      node_children<Prf>(x, key_cw(key, d), c0, c1);
      x = ((ps >> (s - d)) & 1) ? c1 : c0;
    }
    buf[s & 1][0] = x;
  }
  __syncthreads();
  // level k of the subtree: [ps << (k-s), ((ps+1) << (k-s)) - 1] intersected with the range
  uint64_t plo = ps, phi = ps;
  for (uint32_t k = s + 1; k <= f; ++k) {
    const uint64_t lo = max(ps << (k - s), r0 >> (n - k));
    const uint64_t hi = min(((ps + 1) << (k - s)) - 1, (r1 - 1) >> (n - k));
    const uint4 *in = buf[(k - 1) & 1];
    uint4 *o = buf[k & 1];
    for (uint64_t p = plo + threadIdx.x; p <= phi; p += blockDim.x) {
      uint4 c0, c1;
      node_children<Prf>(in[p - plo], key_cw(key, k), c0, c1);
      if (2 * p >= lo && 2 * p <= hi) o[2 * p - lo] = c0;
      if (2 * p + 1 >= lo && 2 * p + 1 <= hi) o[2 * p + 1 - lo] = c1;
    }
    __syncthreads();
    plo = lo;
    phi = hi;
  }
  const uint64_t lo_f = r0 >> (n - f);
  for (uint64_t i = threadIdx.x; i <= phi - plo; i += blockDim.x)
    out[uint64_t(b) * cap + (plo - lo_f) + i] = buf[f & 1][i];
}

// f == 0: the frontier is the root itself.
__global__ void copy_roots_kernel(const uint8_t *__restrict__ keys, uint32_t kstride, uint32_t B,
                                  uint4 *__restrict__ out, uint64_t cap) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) out[uint64_t(b) * cap] = key_root(keys + uint64_t(b) * kstride);
}

// ----------------------------------------------------------------- a3..a6: fused
// One (key batch, table shard) evaluation.  A launch runs one group (the
// dpf_eval_batch* entry points) or many (dpf_eval_grouped: e.g. the 26
// tables x hot/full splits of the co-design workload) sharing the kernel
// configuration below; work items are numbered group after group.
struct GroupDesc {
  const uint8_t *keys;    // device keys (wire layout; AES: bitsliced copy)
  const uint4 *frontier;  // [B][cap], node i at depth f (absolute lo_f + i)
  const uint32_t *T;      // shard base: row r0 (tcgen05 path: the limb-packed table)
  uint32_t *shares;       // [B][D]
  uint64_t cap;           // frontier stride per key
  uint64_t F;             // frontier nodes per key
  uint64_t lo_f;          // absolute index of frontier node 0
  uint64_t r0, r1;        // valid absolute rows
  uint64_t r0a, packed_rows;  // tcgen05 path: 8-row-aligned packed range
  uint32_t kstride, B, n, m;
  uint32_t nwin, n_ktiles;  // windows per item = 2^(m-1) / W; key tiles
  uint32_t item_base;       // first work item of this group
  uint32_t key_base;        // first key of this group (grouped top BFS)
  uint4 *frontier_alt;      // grouped top BFS ping-pong buffer (f > kTopSmemLevels)
  uint64_t nr0, nr1;        // grouped top BFS: the row range in tree-leaf units (R20: final nodes)
};

struct FusedParams {
  GroupDesc g0;              // the group when n_groups == 1
  const GroupDesc *groups;   // device array when n_groups > 1 (sorted by item_base)
  uint32_t n_groups, n_items, D;
  uint32_t Kt, Ft, tasks;  // tasks = Kt * Ft <= 32 * NP (lanes >= tasks idle)
  uint32_t Kr;             // tcgen05: keys per CTA that carry a key (<= Kt = the CTA's MMA columns;
                           // < Kt for small batches: the other B-operand columns stay zero)
  uint32_t W;              // units per producer thread per window (unit: a leaf pair; ET: a final node)
  uint32_t R;              // table rows per node per window: 2W, or 16W with early termination (R20)
  uint32_t CG, KG, SG;     // consumer col groups / key groups / slot groups
  uint32_t y_stage_words, t_stage_words;  // t: one T-ring entry (CN nodes x 2W rows x D + pad)
  uint32_t CN, n_chunks, NST;             // IMAD kernel: nodes per T entry, entries per window, ring depth
  uint32_t sys_red;                       // flush with system-scope atomics (answers in peer memory)
};

__device__ __forceinline__ GroupDesc group_of(const FusedParams &p, uint32_t item) {
  if (p.n_groups <= 1) return p.g0;
  uint32_t lo = 0, hi = p.n_groups - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (__ldg(&p.groups[mid].item_base) <= item) lo = mid;
    else hi = mid - 1;
  }
  return p.groups[lo];
}

// A CTA runs items item, item + gridDim.x, ...; consecutive ones of the same
// group and key tile add into the same answers, so their partial sums stay in
// the accumulators (registers / TMEM) and are flushed once at the end of the
// run (the host picks a grid that is a multiple of the key-tile count when
// that is free, which makes a CTA's key tile constant).  Exact for any
// grouping: Z_2^32 addition is associative.
__device__ __forceinline__ bool run_continues(const FusedParams &p, const GroupDesc &g, uint32_t kt, uint32_t next) {
  if (next >= p.n_items) return false;
  if (p.n_groups <= 1) return (next - g.item_base) % g.n_ktiles == kt;
  const GroupDesc h = group_of(p, next);
  return h.item_base == g.item_base && (next - h.item_base) % h.n_ktiles == kt;
}

template <int NP, int NC>
struct Smem {
  static constexpr int kThreads = 32 * (NP + NC + 1);
};

// Consumer: warp-tile of KPW keys x (32 * CPL) columns; lane owns columns
// lane + 32*(cg*CPL + c), c < CPL.  y read as broadcast (same word for all
// lanes), T read coalesced.  No column guard in the loop: columns >= D read
// padding/next-row words whose products are never flushed.
template <int KPW>
__device__ __forceinline__ void load_y(const uint32_t *__restrict__ yp, uint32_t (&yv)[KPW]) {
  if constexpr (KPW % 4 == 0) {
#pragma unroll
    for (int k = 0; k < KPW; k += 4) {
      const uint4 v = *reinterpret_cast<const uint4 *>(yp + k);
      yv[k] = v.x; yv[k + 1] = v.y; yv[k + 2] = v.z; yv[k + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < KPW; ++k) yv[k] = yp[k];
  }
}

// Slots processed per main-loop step: the step's LDS are all issued before
// its IMADs (no per-slot trip-count guard between them), so small tiles --
// the streaming regime, B <= 8, where the contraction is a few IMADs per
// LDS -- are not LDS-latency-bound.  The 16-producer kernels (80-register
// cap) and large tiles keep one slot per step: their registers are spoken for.
template <int KPW, int CPL, int NP>
__host__ __device__ constexpr int consume_unroll() {
  return NP >= 16 ? (KPW * CPL >= 16 ? 1 : 2)
                  : KPW * CPL >= 64 ? 1 : KPW * CPL >= 32 ? 2 : KPW * CPL >= 16 ? 4 : 8;
}

template <int KPW, int CPL, int NP>
__device__ __forceinline__ void consume_window(const uint32_t *__restrict__ yb, const uint32_t *__restrict__ tb,
                                               uint32_t nslots, uint32_t Kt, uint32_t D, uint32_t key0,
                                               uint32_t colbase, uint32_t s0, uint32_t sstep,
                                               uint32_t (&acc)[KPW][CPL]) {
  // slots s0, s0 + sstep, ... (slot groups: small key tiles spread the
  // window's leaves over several consumer warps)
  const uint32_t *yp = yb + key0 + s0 * Kt;
  const uint32_t *tp = tb + colbase + s0 * D;
  const uint32_t ystep = sstep * Kt, tstep = sstep * D;
  constexpr int U = consume_unroll<KPW, CPL, NP>();
  uint32_t s = s0;
  if constexpr (U > 1) {
    for (; s + (U - 1) * sstep < nslots; s += U * sstep) {
      uint32_t tv[U][CPL], yv[U][KPW];
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) tv[u][c] = tp[u * tstep + 32 * c];
        load_y<KPW>(yp + u * ystep, yv[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < KPW; ++k)
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc[k][c] += yv[u][k] * tv[u][c];
      yp += U * ystep;
      tp += U * tstep;
    }
  }
#pragma unroll 4
  for (; s < nslots; s += sstep) {
    uint32_t tv[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) tv[c] = tp[32 * c];
    uint32_t yv[KPW];
    load_y<KPW>(yp, yv);
#pragma unroll
    for (int k = 0; k < KPW; ++k)
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[k][c] += yv[k] * tv[c];
    yp += ystep;
    tp += tstep;
  }
}

template <class Prf, int NP, int NC, int KPW, int CPL>
__global__ void __launch_bounds__(32 * (NP + NC + 1), 1) fused_eval_kernel(const FusedParams p) {
  extern __shared__ __align__(128) uint8_t smem_all[];
  uint8_t *smem = smem_all + Prf::kSmemBytes;            // after the PRF's tables (AES)
  uint64_t *tfull = reinterpret_cast<uint64_t *>(smem);  // T ring [NST]: bulk-copy completion
  uint64_t *tempty = tfull + 8;                          // T ring [NST]: consumers done (count NC)
  constexpr uint32_t kFullThreads = 32 * (NP + NC), kEmptyThreads = 32 * (NP + NC);
  // windows this CTA will run (consumers skip the EMPTY arrive for the last
  // two, which no producer will ever wait for)
  uint32_t total_w = 0;
  for (uint32_t item = blockIdx.x; item < p.n_items; item += gridDim.x) total_w += group_of(p, item).nwin;
  uint32_t *ybuf = reinterpret_cast<uint32_t *>(smem + 128);
  uint32_t *tbuf = ybuf + 2 * p.y_stage_words;
  uint4 *stack = reinterpret_cast<uint4 *>(tbuf + p.NST * p.t_stage_words);

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < p.NST; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 32 * NC);  // every consumer lane releases what it read
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  Prf::init_smem();
  __syncthreads();
  pdl_wait_primary();  // the top BFS' frontier and zeroed answers

  if (warp < NP) {
    // ------------------------------------------------------------ producers
    const uint32_t tix = warp * 32 + lane;
    const bool lane_on = tix < p.tasks;
    const uint32_t kl = lane_on ? tix % p.Kt : 0, nl = lane_on ? tix / p.Kt : 0;
    uint32_t wseq = 0;
    for (uint32_t item = blockIdx.x; item < p.n_items; item += gridDim.x) {
      const GroupDesc g = group_of(p, item);
      const uint32_t li = item - g.item_base;
      const uint32_t kt = li % g.n_ktiles, ng = li / g.n_ktiles;
      const uint32_t nq = 1u << (g.m - 1);
      const uint32_t b = kt * p.Kt + kl;
      const uint64_t node = uint64_t(ng) * p.Ft + nl;
      const bool valid = lane_on && b < g.B && node < g.F;
      const uint8_t *key = g.keys + uint64_t(valid ? b : 0) * g.kstride;
      const uint32_t cw_out = key_cw_out(key);
      uint4 cur = valid ? g.frontier[uint64_t(b) * g.cap + node] : make_uint4(0, 0, 0, 0);
      constexpr uint32_t V = Prf::kEt ? 4u : 0u;  // log2(rows per subtree leaf)
      const uint64_t row_base = (g.lo_f + node) << (g.m + V);
      const bool inside = valid && row_base >= g.r0 && row_base + (1ull << (g.m + V)) <= g.r1;
      uint32_t dep = 0;
      if constexpr (Prf::kEt) {
        // R20: units are final nodes (16 rows each, one Convert block); the
        // leaf-parent expansion at even units yields both, the right one waits
        uint32_t cwl[16];
        load_cwl(key_cw(key, g.n + 1), cwl);
        uint4 pend = make_uint4(0, 0, 0, 0);
        const uint32_t npairs = 1u << (g.m - 1);
        for (uint32_t win = 0; win < g.nwin; ++win, ++wseq) {
          const uint32_t stage = wseq & 1, use = wseq >> 1;
          if (use > 0) named_sync(3 + stage, kEmptyThreads);
          uint32_t *yb = ybuf + stage * p.y_stage_words;
          for (uint32_t qi = 0; qi < p.W; ++qi) {
            const uint32_t q = win * p.W + qi;
            uint4 sf;
            if ((q & 1) == 0) {
              while (dep + 1 < g.m) {
                uint4 c0, c1;
                node_children<Prf>(cur, key_cw(key, g.n - g.m + dep + 1), c0, c1);
                stack[(dep + 1) * (32 * NP) + tix] = c1;
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
            if (lane_on) {
              const uint32_t slot = nl * p.R + 16 * qi;
#pragma unroll
              for (int c = 0; c < 16; ++c) yb[(slot + c) * p.Kt + kl] = y[c];
            }
            if ((q & 1) && (q >> 1) + 1 < npairs) {  // pop for the next leaf-parent
              const uint32_t k = g.m - 1 - (__ffs((q >> 1) + 1) - 1);
              cur = stack[k * (32 * NP) + tix];
              dep = k;
            }
          }
          named_arrive(1 + stage, kFullThreads);
        }
      } else {
      for (uint32_t win = 0; win < g.nwin; ++win, ++wseq) {
        const uint32_t stage = wseq & 1, use = wseq >> 1;
        if (use > 0) named_sync(3 + stage, kEmptyThreads);
        uint32_t *yb = ybuf + stage * p.y_stage_words;
        for (uint32_t qi = 0; qi < p.W; ++qi) {
          const uint32_t q = win * p.W + qi;
          // descend (warp-uniform: every thread shares the schedule)
          while (dep + 1 < g.m) {
            uint4 c0, c1;
            node_children<Prf>(cur, key_cw(key, g.n - g.m + dep + 1), c0, c1);
            stack[(dep + 1) * (32 * NP) + tix] = c1;
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
          if (lane_on) {
            const uint32_t slot = nl * p.R + 2 * qi;
            yb[slot * p.Kt + kl] = y0;
            yb[(slot + 1) * p.Kt + kl] = y1;
          }
          if (q + 1 < nq) {  // pop: the right sibling at depth m-1-ctz(q+1)
            const uint32_t k = g.m - 1 - (__ffs(q + 1) - 1);
            cur = stack[k * (32 * NP) + tix];
            dep = k;
          }
        }
        named_arrive(1 + stage, kFullThreads);
      }
      }  // !kEt
    }
  } else if (warp < NP + NC) {
    // ------------------------------------------------------------ consumers
    const uint32_t cwarp = warp - NP;
    const uint32_t tile = cwarp % (p.KG * p.CG), sg = cwarp / (p.KG * p.CG);
    const uint32_t kg = tile / p.CG, cg = tile % p.CG;
    const bool active = sg < p.SG;
    const uint32_t key0 = kg * KPW;
    const uint32_t colbase = cg * CPL * 32 + lane;
    uint32_t acc[KPW][CPL];
#pragma unroll
    for (int k = 0; k < KPW; ++k)
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[k][c] = 0;
    uint32_t wseq = 0, ts = 0, tph = 0;  // T ring slot and phase (no division per chunk)
    const uint32_t seg = p.R;  // rows per node per window
    for (uint32_t item = blockIdx.x; item < p.n_items; item += gridDim.x) {
      const GroupDesc g = group_of(p, item);
      const uint32_t kt = (item - g.item_base) % g.n_ktiles;
      for (uint32_t win = 0; win < g.nwin; ++win, ++wseq) {
        const uint32_t stage = wseq & 1;
        named_sync(1 + stage, kFullThreads);
        const uint32_t *yb = ybuf + stage * p.y_stage_words;
        for (uint32_t ch = 0; ch < p.n_chunks; ++ch) {
          const uint32_t n0 = ch * p.CN, nn = min(p.CN, p.Ft - n0);
          mbar_wait(&tfull[ts], tph);
          if (active)
            consume_window<KPW, CPL, NP>(yb + n0 * seg * p.Kt, tbuf + ts * p.t_stage_words, nn * seg, p.Kt, p.D, key0,
                                     colbase, sg, p.SG, acc);
          mbar_arrive(&tempty[ts]);  // one warp instruction; each lane orders its own reads
          if (++ts == p.NST) {
            ts = 0;
            tph ^= 1;
          }
        }
        if (wseq + 2 < total_w) named_arrive(3 + stage, kEmptyThreads);
      }
      // a6/a7: flush the run's partial answers, party sign applied once.
      if (active && !run_continues(p, g, kt, item + gridDim.x)) {
#pragma unroll
        for (int k = 0; k < KPW; ++k) {
          const uint32_t b = kt * p.Kt + key0 + k;
          if (key0 + k < p.Kt && b < g.B) {
            const uint32_t neg = key_party(g.keys + uint64_t(b) * g.kstride);
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
              const uint32_t col = colbase + 32 * c;
              if (col < p.D) red_add_u32(g.shares + uint64_t(b) * p.D + col, neg ? 0u - acc[k][c] : acc[k][c], p.sys_red);
            }
          }
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc[k][c] = 0;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ T loader
    // T ring of (window, node chunk) entries: CN nodes x 2W rows, one
    // cp.async.bulk per node segment, decoupled from the y ring.
    uint32_t ts = 0, tph = 0;  // ring slot, and the parity of its previous use
    bool wrapped = false;      // every slot used once: wait for the consumers' release
    const uint64_t seg_rows = p.R;
    const uint32_t row_bytes = p.D * 4;
    constexpr uint32_t V = Prf::kEt ? 4u : 0u;
    for (uint32_t item = blockIdx.x; item < p.n_items; item += gridDim.x) {
      const GroupDesc g = group_of(p, item);
      const uint32_t ng = (item - g.item_base) / g.n_ktiles;
      for (uint32_t win = 0; win < g.nwin; ++win) {
        for (uint32_t ch = 0; ch < p.n_chunks; ++ch) {
          const uint32_t cur = ts;
          if (wrapped) mbar_wait(&tempty[cur], tph ^ 1);
          if (++ts == p.NST) {
            ts = 0;
            tph ^= 1;
            wrapped = true;
          }
          uint32_t *tb = tbuf + cur * p.t_stage_words;
          const uint32_t n0 = ch * p.CN, n1 = min(p.Ft, n0 + p.CN);
          if (g.nwin == 1) {
            // one window covers whole subtrees: the chunk's rows are contiguous
            // in the table -> a single bulk copy (small key tiles stream the
            // table, and per-node copies of a few KB starve the TMA unit)
            const uint64_t nb = uint64_t(ng) * p.Ft;
            const uint64_t nend = min(uint64_t(n1) + nb, g.F);
            const uint64_t s0 = (g.lo_f + nb + n0) << (g.m + V);
            const uint64_t s1 = nend > nb + n0 ? (g.lo_f + nend) << (g.m + V) : s0;
            const uint64_t a = s0 > g.r0 ? s0 : g.r0, e = s1 < g.r1 ? s1 : g.r1;
            const uint32_t bytes = a < e ? uint32_t(e - a) * row_bytes : 0u;
            if (lane == 0) {
              mbar_arrive_expect_tx(&tfull[cur], bytes);
              if (bytes) bulk_g2s(tb + (a - s0) * p.D, g.T + (a - g.r0) * p.D, bytes, &tfull[cur]);
            }
            __syncwarp();
            continue;
          }
          uint32_t my_bytes = 0;
          for (uint32_t nl = n0 + lane; nl < n1; nl += 32) {
            const uint64_t node = uint64_t(ng) * p.Ft + nl;
            if (node >= g.F) continue;
            const uint64_t s0 = ((g.lo_f + node) << (g.m + V)) + seg_rows * win;
            const uint64_t a = s0 > g.r0 ? s0 : g.r0, e = (s0 + seg_rows) < g.r1 ? (s0 + seg_rows) : g.r1;
            if (a < e) my_bytes += uint32_t(e - a) * row_bytes;
          }
          const uint32_t total = __reduce_add_sync(0xFFFFFFFFu, my_bytes);
          if (lane == 0) mbar_arrive_expect_tx(&tfull[cur], total);
          __syncwarp();
          for (uint32_t nl = n0 + lane; nl < n1; nl += 32) {
            const uint64_t node = uint64_t(ng) * p.Ft + nl;
            if (node >= g.F) continue;
            const uint64_t s0 = ((g.lo_f + node) << (g.m + V)) + seg_rows * win;
            const uint64_t a = s0 > g.r0 ? s0 : g.r0, e = (s0 + seg_rows) < g.r1 ? (s0 + seg_rows) : g.r1;
            if (a < e)
              bulk_g2s(tb + (uint64_t(nl - n0) * seg_rows + (a - s0)) * p.D, g.T + (a - g.r0) * p.D,
                       uint32_t(e - a) * row_bytes, &tfull[cur]);
          }
        }
      }
    }
  }
}

}  // namespace dev
}  // namespace dpfpir
#include "fused_tc.cuh"
namespace dpfpir {
namespace dev {

// ---------------------------------------------------------- grouped launches
// Zero every group's answer buffer (one launch instead of one memset per group).
__global__ void zero_shares_grouped_kernel(const GroupDesc *__restrict__ groups, uint32_t n_groups, uint32_t D) {
  for (uint32_t gi = blockIdx.y; gi < n_groups; gi += gridDim.y) {
    const GroupDesc &g = groups[gi];
    const uint64_t words = uint64_t(g.B) * D;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < words; i += uint64_t(gridDim.x) * blockDim.x)
      g.shares[i] = 0;
  }
}

// a2 for all groups in one launch: one CTA per (group, key) expands levels
// 1..f_g (f_g <= kTopSmemLevels) in shared memory, writes the frontier.
template <class Prf>
__global__ void __launch_bounds__(256) expand_top_grouped_kernel(const GroupDesc *__restrict__ groups,
                                                                 uint32_t n_groups) {
  __shared__ uint4 buf[2][1u << kTopSmemLevels];
  uint32_t lo = 0, hi = n_groups - 1;  // group of this CTA's key
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (groups[mid].key_base <= blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const GroupDesc &g = groups[lo];
  const uint32_t b = blockIdx.x - g.key_base;
  const uint8_t *key = g.keys + uint64_t(b) * g.kstride;
  const uint32_t n = g.n, f = g.n - g.m, a = f < kTopSmemLevels ? f : kTopSmemLevels;
  const uint64_t r0 = g.nr0, r1 = g.nr1;
  // level a lands where the remaining levels' ping-pong ends on `frontier`
  uint4 *out = (((f - a) & 1) ? g.frontier_alt : const_cast<uint4 *>(g.frontier)) + uint64_t(b) * g.cap;
  if (threadIdx.x == 0) buf[0][0] = key_root(key);
  Prf::init_smem();
  __syncthreads();
  for (uint32_t k = 1; k <= a; ++k) {
    const uint64_t plo = r0 >> (n - (k - 1)), phi = (r1 - 1) >> (n - (k - 1));
    const uint64_t lo_k = r0 >> (n - k), hi_k = (r1 - 1) >> (n - k);
    const uint4 *in = buf[(k - 1) & 1];
    uint4 *o = buf[k & 1];
    for (uint64_t p = plo + threadIdx.x; p <= phi; p += blockDim.x) {
      uint4 c0, c1;
      node_children<Prf>(in[p - plo], key_cw(key, k), c0, c1);
      if (2 * p >= lo_k) o[2 * p - lo_k] = c0;
      if (2 * p + 1 <= hi_k) o[2 * p + 1 - lo_k] = c1;
    }
    __syncthreads();
  }
  const uint64_t cnt = ((r1 - 1) >> (n - a)) - (r0 >> (n - a)) + 1;
  for (uint64_t i = threadIdx.x; i < cnt; i += blockDim.x) out[i] = buf[a & 1][i];
}

// Level k > kTopSmemLevels of every group whose frontier is deeper: grid.y =
// group; thread per (key, parent), both children by one block.
template <class Prf>
__global__ void expand_level_grouped_kernel(const GroupDesc *__restrict__ groups, uint32_t k) {
  const GroupDesc &g = groups[blockIdx.y];
  const uint32_t n = g.n, f = g.n - g.m;
  if (k > f) return;
  if constexpr (Prf::kSmemBytes != 0) {  // (uniform per CTA: k, f)
    Prf::init_smem();
    __syncthreads();
  }
  const uint64_t plo = g.nr0 >> (n - (k - 1)), phi = (g.nr1 - 1) >> (n - (k - 1));
  const uint64_t lo = g.nr0 >> (n - k), hi = (g.nr1 - 1) >> (n - k);
  const uint64_t np = phi - plo + 1, total = np * g.B;
  const uint4 *in = ((f - k + 1) & 1) ? g.frontier_alt : g.frontier;
  uint4 *out = ((f - k) & 1) ? g.frontier_alt : const_cast<uint4 *>(g.frontier);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t b = uint32_t(i / np);
    const uint64_t p = plo + (i % np);
    const uint8_t *key = g.keys + uint64_t(b) * g.kstride;
    uint4 c0, c1;
    node_children<Prf>(in[uint64_t(b) * g.cap + (p - plo)], key_cw(key, k), c0, c1);
    if (2 * p >= lo && 2 * p <= hi) out[uint64_t(b) * g.cap + (2 * p - lo)] = c0;
    if (2 * p + 1 >= lo && 2 * p + 1 <= hi) out[uint64_t(b) * g.cap + (2 * p + 1 - lo)] = c1;
  }
}

// Test/debug leaf dump (branch-parallel: n blocks per leaf).
template <class Prf>
__global__ void eval_leaves_kernel(const uint8_t *__restrict__ keys, uint32_t kstride, uint32_t B, uint32_t n,
                                   uint32_t *__restrict__ leaves) {
  if constexpr (Prf::kSmemBytes != 0) {
    Prf::init_smem();
    __syncthreads();
  }
  const uint64_t N = 1ull << n;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < N * B;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t b = uint32_t(i >> n);
    const uint64_t j = i & (N - 1);
    const uint8_t *key = keys + uint64_t(b) * kstride;
    uint4 s = key_root(key);
    constexpr uint32_t V = Prf::kEt ? 4u : 0u;
    for (uint32_t d = 1; d + V <= n; ++d) {
      uint4 c0, c1;
      node_children<Prf>(s, key_cw(key, d), c0, c1);
      s = ((j >> (n - d)) & 1) ? c1 : c0;
    }
    uint32_t v;
    if constexpr (Prf::kEt) {  // R20: word j mod 16 of the final node's Convert block
      uint32_t cwl[16], y[16];
      load_cwl(key_cw(key, n - V + 1), cwl);
      leaf_values16(s, cwl, y);
      v = y[0];
#pragma unroll
      for (int c = 1; c < 16; ++c) v = (uint32_t(j & 15) == uint32_t(c)) ? y[c] : v;
    } else {
      v = leaf_value<Prf>(s, key_cw_out(key));
    }
    leaves[i] = key_party(key) ? 0u - v : v;
  }
}

}  // namespace dev

// =================================================================== host side
namespace {

constexpr int kNC = 4;  // consumer warps
constexpr size_t kAlign = 256;
constexpr uint32_t kTopSmemLevelsHost = 10;  // == dev::kTopSmemLevels
constexpr uint32_t kTEntryBytes = 32 * 1024;   // IMAD kernel T-ring entry

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
// opt a kernel into more than 48 KB of dynamic shared memory
template <class K>
bool allow_dyn_smem(K *fn, size_t bytes) {
  return bytes <= 48 * 1024 ||
         cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)) == cudaSuccess;
}
inline uint32_t pow2ceil(uint32_t v) {
  uint32_t r = 1;
  while (r < v) r <<= 1;
  return r;
}

struct KernelChoice {
  int NP, KPW, CPL;
  void (*fn)(const dev::FusedParams);      // ChaCha20
  void (*fn_aes)(const dev::FusedParams);  // AES-128 (T-tables in SMEM)
  void (*fn_et)(const dev::FusedParams);   // ChaCha20, early-terminated leaves (R20)
  void (*get(uint32_t prf) const)(const dev::FusedParams) {
    return prf == DPF_PRF_AES128 ? fn_aes : prf == DPF_PRF_CHACHA20_ET ? fn_et : fn;
  }
};

template <int NP, int KPW, int CPL>
KernelChoice choice() {
  return {NP, KPW, CPL, &dev::fused_eval_kernel<dev::PrfChacha, NP, kNC, KPW, CPL>,
          &dev::fused_eval_kernel<dev::PrfAesTt, NP, kNC, KPW, CPL>,
          &dev::fused_eval_kernel<dev::PrfChachaEt, NP, kNC, KPW, CPL>};
}

struct Plan {
  uint32_t prf;  // DPF_PRF_CHACHA20 / DPF_PRF_AES128 / DPF_PRF_CHACHA20_ET
  bool tc;  // tcgen05 contraction on a limb-packed table
  // Early termination (R20): v = 4, the tree (depth n = log_n - 4) ends at
  // final nodes of 16 rows.  nr0/nr1: the row range in tree-leaf units
  // (final nodes; = r0/r1 without ET), used by the top BFS and the frontier.
  uint32_t v, R;
  uint64_t nr0, nr1;
  uint32_t nsy, nst;  // y-ring / T-ring depth (tc)
  bool pair;          // tc: CTA pairs (cta_group::2, M = 256); Kt = keys per CTA, 2 Kt per item
  uint32_t tmem_cols, y_stage_bytes, t_stage_bytes;
  uint64_t r0a, packed_rows;
  uint32_t n, m, f, Kt, Ft, tasks, W, CG, KG, SG, n_ktiles, n_items, nwin, grid;
  uint32_t Kr;  // tcgen05: real keys per CTA (<= Kt)
  uint64_t r0, r1, F, lo_f, cap;
  uint32_t y_stage_words, t_stage_words, CN, n_chunks, NST;
  size_t smem_bytes;
  size_t xsm;  // PRF shared memory at the start of the dynamic SMEM (AES T-tables), inside smem_bytes
  KernelChoice kc;
  uint64_t prf_blocks;
};

// SM count of the current device, cached per device (mutex-guarded: the
// planners may run on several host threads).  148 without a device.
int current_device() {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return dev;
}
std::mutex g_cache_mu;
int num_sms() {
  static std::map<int, int> cache;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 148;
  if (dev >= 0 && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    sms = 148;
  }
  cache[dev] = sms;
  return sms;
}

// Consumer warp tiling for (Kt keys, D cols) over kNC warps: KG key groups x
// CG col groups, KPW = Kt / KG, CPL = ceil(D / (32 CG)).
// Consumer warp tiling for (Kt keys, D cols) over kNC warps: CG column groups
// x KG = kNC/CG key groups; a warp owns KPW keys x 32*CPL columns.  Among the
// compiled (KPW, CPL) tiles, pick the one with the fewest instructions per
// slot on the busiest consumer warp (CPL T loads + KPW/4 y loads + KPW*CPL
// IMADs), then the fewest in total.
template <int NP>
const std::vector<KernelChoice> &tiles() {
  static const std::vector<KernelChoice> v = {
      choice<NP, 16, 4>(), choice<NP, 16, 2>(), choice<NP, 16, 1>(), choice<NP, 8, 8>(), choice<NP, 8, 4>(),
      choice<NP, 8, 2>(),  choice<NP, 8, 1>(),  choice<NP, 4, 8>(),  choice<NP, 4, 4>(), choice<NP, 4, 2>(),
      choice<NP, 4, 1>(),  choice<NP, 2, 8>(),  choice<NP, 2, 4>(),  choice<NP, 2, 2>(), choice<NP, 2, 1>(),
      choice<NP, 1, 8>(),  choice<NP, 1, 4>(),  choice<NP, 1, 2>(),  choice<NP, 1, 1>(),
  };
  return v;
}

// Producer warps of the IMAD kernel: 16 (4 per SMSP, measured best) when the
// consumer accumulators are small enough to share the register file
// (Kt*D <= 4096 words per CTA), else 8.  DPF_NP=8|16 overrides (tuning).
int producer_warps(uint32_t Kt, uint32_t D, bool et) {
  static int forced = [] {
    const char *e = getenv("DPF_NP");
    const int v = e ? atoi(e) : 0;
    return (v == 8 || v == 16) ? v : 0;
  }();
  if (forced) return forced;
  // 8 producers when the contraction is heavy next to the PRF (consumers need
  // the issue slots: D >= 256, or early termination's 8x cheaper tree) or the
  // batch streams the table (Kt <= 2: smaller windows keep the T ring ahead).
  // Measured (batch_sweep / codesign_bench): 2^20 x 256 B = 8: 0.598 -> 0.493
  // ms; 2^22 x 64 B = 1: 0.406 -> 0.374 ms; c5 ET batch 16: 2.84 -> 2.64 ms;
  // but 2^22 x 64 B = 4 and c5 batch 4/16 are faster with 16.
  if (Kt * D > 4096 || D >= 256 || et || Kt <= 2) return 8;
  return 16;
}

bool pick_kernel(uint32_t Kt, uint32_t D, Plan &pl, bool et) {
  const int NP = producer_warps(Kt, D, et);
  const std::vector<KernelChoice> &ts = NP == 16 ? tiles<16>() : tiles<8>();
  uint64_t best = ~0ull;
  for (const KernelChoice &kc : ts) {
    for (uint32_t CG : {1u, 2u, 4u}) {
      const uint32_t KG = kNC / CG;
      if (Kt % uint32_t(kc.KPW) || Kt / kc.KPW > KG) continue;
      if (32u * kc.CPL * CG < D) continue;
      const uint32_t per_warp = kc.CPL + (kc.KPW + 3) / 4 + kc.KPW * kc.CPL;
      const uint32_t sg = kNC / ((Kt / kc.KPW) * CG);  // slot groups share the window
      const uint32_t total = per_warp * CG * (Kt / kc.KPW);
      const uint64_t score = (uint64_t(per_warp * 16 / sg) << 32) | total;
      if (score < best) {
        best = score;
        pl.CG = CG;
        pl.KG = Kt / kc.KPW;
        pl.SG = kNC / (pl.KG * CG);  // idle warps take other slots of the window
        pl.kc = kc;
      }
    }
  }
  return best != ~0ull;
}

// Subtree depth m: the largest m (<= m_cap) that still gives >= 8 work items
// per SM (measured: beyond that, deeper top BFS costs more than balance gains).
uint32_t choose_m_target(const Plan &pl, uint32_t n, uint32_t m_min, uint32_t m_cap, uint32_t workers = 0) {
  const uint64_t target = 8ull * (workers ? workers : uint32_t(num_sms()));
  uint32_t best = m_min;
  for (uint32_t m = std::min<uint32_t>(n, m_cap); m >= m_min; --m) {
    const uint64_t F = ((pl.nr1 - 1) >> m) - (pl.nr0 >> m) + 1;
    const uint64_t items = uint64_t(pl.n_ktiles) * ((F + pl.Ft - 1) / pl.Ft);
    best = m;
    if (items >= target) break;
  }
  return best;
}

// Persistent grid: one CTA per SM.  When the key-tile count divides a grid
// of (almost) every SM, each CTA keeps one key tile for all its items, so
// its accumulators are flushed once instead of once per item (run_continues).
// DPF_GRID_ALIGN=1 forces the aligned grid even when it idles SMs, =0 never.
uint32_t choose_grid(uint32_t n_items, uint32_t n_ktiles, uint32_t sms = 0) {
  if (sms == 0) sms = uint32_t(num_sms());
  if (n_items <= sms) return n_items;
  static const int force = [] {
    const char *e = getenv("DPF_GRID_ALIGN");
    return e ? atoi(e) : -1;
  }();
  const uint32_t aligned = n_ktiles <= sms ? (sms / n_ktiles) * n_ktiles : sms;
  if (force == 0) return sms;
  if (force == 1 || aligned == sms) return aligned;
  return sms;
}

// Window / T-ring sizing for the IMAD kernel; false if SMEM does not fit.
// Rows per window unit: a leaf pair, or one final node with early termination.
inline uint32_t unit_rows(const Plan &pl) { return pl.v ? (1u << pl.v) : 2u; }

// dynamic SMEM per CTA left for the kernel's own regions (227 KB opt-in max
// minus the PRF's tables)
inline size_t smem_cap(const Plan &pl) { return 227 * 1024 - pl.xsm; }
// the PRF's shared memory (dev::Prf*::kSmemBytes)
inline size_t prf_smem(uint32_t prf) { return prf == DPF_PRF_AES128 ? dev::PrfAesTt::kSmemBytes : 0; }

bool set_windows(Plan &pl, uint32_t W, uint32_t D, size_t stack_bytes) {
  pl.W = W;
  pl.R = unit_rows(pl) * W;
  pl.y_stage_words = uint32_t(align_up(size_t(pl.Kt) * pl.Ft * pl.R, 32));
  const uint32_t pad = 32u * pl.kc.CPL * pl.CG;  // lanes whose columns exceed D read past the last row
  // A final node's 16 rows (early termination) cannot be split across
  // entries: its entry may exceed the default size at large D.
  const size_t budget = pl.v ? std::max<size_t>(kTEntryBytes, (size_t(pl.R) * D + pad) * 4) : kTEntryBytes;
  uint32_t CN = pl.Ft;
  while (CN > 1 && (size_t(CN) * pl.R * D + pad) * 4 > budget) CN >>= 1;
  if ((size_t(CN) * pl.R * D + pad) * 4 > budget) return false;
  pl.CN = CN;
  pl.n_chunks = (pl.Ft + CN - 1) / CN;
  pl.t_stage_words = uint32_t(align_up(size_t(CN) * pl.R * D + pad, 32));
  const size_t fixed = 128 + 4 * 2 * size_t(pl.y_stage_words) + stack_bytes;
  if (fixed + 2 * 4 * size_t(pl.t_stage_words) > smem_cap(pl)) return false;
  pl.NST = uint32_t(std::min<size_t>(8, (smem_cap(pl) - fixed) / (4 * size_t(pl.t_stage_words))));
  pl.smem_bytes = pl.xsm + fixed + 4 * size_t(pl.NST) * pl.t_stage_words;
  return true;
}

// Row range -> tree-leaf (final node) range for the top BFS and frontier.
void set_ranges(Plan &pl, uint32_t log_n, uint64_t r0, uint64_t rows, bool et) {
  pl.v = et ? 4u : 0u;
  pl.n = log_n - pl.v;
  pl.r0 = r0;
  pl.r1 = r0 + rows;
  pl.nr0 = r0 >> pl.v;
  pl.nr1 = ((pl.r1 - 1) >> pl.v) + 1;
}

// PRF blocks: top levels (nodes intersecting the range) + fused subtrees
// (2^m - 1 internal nodes, + 2^m Convert blocks with early termination).
uint64_t count_blocks(const Plan &pl, uint32_t B) {
  uint64_t top = 0;
  for (uint32_t k = 0; k < pl.f; ++k) top += ((pl.nr1 - 1) >> (pl.n - k)) - (pl.nr0 >> (pl.n - k)) + 1;
  const uint64_t per = ((1ull << pl.m) - 1) + (pl.v ? (1ull << pl.m) : 0);
  return uint64_t(B) * top + uint64_t(pl.n_items) * pl.tasks * per;
}

int make_plan(uint32_t B, uint32_t log_n, uint64_t r0, uint64_t rows, uint32_t D, Plan &pl, bool et = false,
              size_t xsm = 0) {
  std::memset(&pl, 0, sizeof pl);
  pl.xsm = xsm;
  set_ranges(pl, log_n, r0, rows, et);
  const uint32_t n = pl.n;
  // Key tile: lanes <-> keys (Kt <= 32), remaining lanes <-> frontier nodes.
  pl.Kt = std::min<uint32_t>(32, pow2ceil(B));
  while (pl.Kt * D > 8192 && pl.Kt > 1) pl.Kt >>= 1;  // accumulator budget: Kt*D <= 8192 words/CTA
  if (!pick_kernel(pl.Kt, D, pl, et)) return DPF_EINVAL;
  const uint32_t NP = uint32_t(pl.kc.NP);
  pl.Ft = 32 * NP / pl.Kt;
  // one T-ring entry must hold at least one node's 2-row segment
  while ((uint64_t(2) * D + 32u * pl.kc.CPL * pl.CG) * 4 > kTEntryBytes && pl.Ft > 1) pl.Ft >>= 1;
  pl.tasks = pl.Kt * pl.Ft;
  pl.n_ktiles = (B + pl.Kt - 1) / pl.Kt;
  // Subtree depth m (frontier depth f = n - m) from a cost model; the SMEM
  // DFS stack (m x 16 B per producer thread) is capped at 64 KB.
  const uint32_t m_cap = std::min<uint32_t>(14, uint32_t((64 * 1024) / (32 * NP * 16)));
  pl.m = choose_m_target(pl, n, 1, m_cap);
  if (const char *e = getenv("DPF_FORCE_M")) {  // tuning override
    const uint32_t fm = uint32_t(atoi(e));
    if (fm >= 1 && fm <= std::min<uint32_t>(n, m_cap)) pl.m = fm;
  }
  pl.f = n - pl.m;
  pl.lo_f = pl.nr0 >> pl.m;
  pl.F = ((pl.nr1 - 1) >> pl.m) - pl.lo_f + 1;
  pl.cap = pl.F;
  const uint64_t items = uint64_t(pl.n_ktiles) * ((pl.F + pl.Ft - 1) / pl.Ft);
  if (items > 0x7FFFFFFFull) return DPF_EINVAL;
  pl.n_items = uint32_t(items);
  // Window: W units per thread (y stage = Kt*Ft*R words <= 16 KB, 32 KB with
  // early termination, whose shallower subtrees leave SMEM to spare); T ring
  // entries of CN nodes x R rows (<= 32 KB), NST of them.
  const uint32_t nq = et ? (1u << pl.m) : (1u << (pl.m - 1));
  const uint64_t ybudget = et ? 32 * 1024 : 16 * 1024;
  uint32_t W = std::min<uint32_t>(8, nq);
  while (W > 1 && uint64_t(pl.Kt) * pl.Ft * unit_rows(pl) * W * 4 > ybudget) W >>= 1;
  const size_t stack_bytes = size_t(pl.m) * 32 * NP * 16;
  for (;; W >>= 1) {
    if (set_windows(pl, W, D, stack_bytes)) break;
    if (W == 1) return DPF_EINVAL;
  }
  pl.nwin = nq / pl.W;
  pl.grid = choose_grid(pl.n_items, pl.n_ktiles);
  pl.prf_blocks = count_blocks(pl, B);
  return DPF_OK;
}

constexpr uint32_t kTcNP = 16;   // producer warps (4 per SMSP)
// DFS stack of the tcgen05 kernel: one uint4 per producer thread for each of
// the subtree depths 1..m-1 (pending right children).
constexpr size_t kTcLevelBytes = size_t(32) * kTcNP * 16;
inline size_t tc_stack_bytes(uint32_t m) { return m > 1 ? size_t(m - 1) * kTcLevelBytes : 0; }
// y-ring depth: 3 stages (with CTA pairs and N = 128 the SMEM fits them
// beside a full DFS stack; measured t5 0.906 -> 0.916, c3 0.894 -> 0.896).
constexpr uint32_t kTcNSY = 3;

// How many 2-CTA clusters of the tcgen05 kernel fit on the device at once
// (cudaOccupancyMaxActiveClusters; num_sms/2 without a device).
uint32_t max_pairs(size_t smem_bytes) {
  static std::map<std::pair<int, size_t>, uint32_t> cache;  // (device, smem) -> pairs; under g_cache_mu
  const int dev_id = current_device();
  uint32_t r = uint32_t(num_sms()) / 2;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = cache.find({dev_id, smem_bytes});
    if (it != cache.end()) return it->second;
  }
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3(2 * r);
  cfg.blockDim = dim3(32 * (kTcNP + dev::tc_extra_warps(false)));
  cfg.dynamicSmemBytes = smem_bytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto fn = &dev::fused_eval_tc_kernel<dev::PrfChacha, kTcNP, kTcNSY, 4, true, false>;
  int n = 0;
  if (dev_id >= 0 &&
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bytes)) == cudaSuccess &&
      cudaOccupancyMaxActiveClusters(&n, fn, &cfg) == cudaSuccess && n > 0)
    r = std::min<uint32_t>(r, uint32_t(n));
  else
    cudaGetLastError();  // clear: no device (host-only planning)
  std::lock_guard<std::mutex> lk(g_cache_mu);
  cache[{dev_id, smem_bytes}] = r;
  return r;
}
// Early termination (R20) fills a y stage with ~2 ChaCha20 blocks per thread
// instead of ~8, so the MMA side (80 UMMAs per stage) needs more slack: a
// 3-deep y ring (measured at c3: 0.58 -> 0.61 of the ALU roofline).
constexpr uint32_t kTcNSYEt = 3;
inline uint32_t tc_y_stages(bool et) { return et ? kTcNSYEt : kTcNSY; }
// smallest subtree depth holding one window: 2^(m-1) >= W leaf pairs, or
// 2^m >= W final nodes with early termination
inline uint32_t tc_m_min(bool et, uint32_t W) {
  uint32_t m = 1;
  while ((et ? (1u << m) : (1u << (m - 1))) < W) ++m;
  return et ? m : std::max(m, 3u);
}
// T-ring depth (16 KB entries).  8 entries measured no faster than 4 at
// D = 512/1024, so the SMEM goes to the DFS stack instead.
// (6 and 8 entries measured no faster for early termination either.)
inline uint32_t tc_t_stages(uint32_t) { return 4u; }

// tcgen05 plan (limb-packed table), D a multiple of 128 up to 1024:
// Kt = MMA N = 64/32/16 keys so that 4 limb accumulators x D/128 tiles x Kt
// columns fit the 512 TMEM columns; Ft = 512/Kt frontier nodes per item;
// W = 4 leaf pairs per node per window (one 8-row packed block).
int make_tc_plan_w(uint32_t B, uint32_t log_n, uint64_t r0, uint64_t rows, uint32_t D, Plan &pl, bool et,
                   uint32_t W, bool allow_kr = true, bool fallback_padded = true, size_t xsm = 0);

// W (leaf pairs per node per window, standard scheme): 8 when the problem is
// deep enough for subtrees of >= 4 levels (m >= 4 under W = 4), else 4 --
// half the y-ring handshakes per block (measured c3 0.896 -> 0.912, t5 0.914
// -> 0.925).  Early termination: one final node per window.
int make_tc_plan(uint32_t B, uint32_t log_n, uint64_t r0, uint64_t rows, uint32_t D, Plan &pl, bool et = false,
                 size_t xsm = 0) {
  if (et) {
    // Early termination: two final nodes per window with a 2-deep y ring
    // (half the y handshakes; measured c3 0.778 -> 0.784, t5 0.803 -> 0.815
    // with the T loader polling), else one final node and a 3-deep ring.
    // DPF_ET_W=1 pins the single-node window (tuning).
    static const bool allow2 = [] {
      const char *e = getenv("DPF_ET_W");
      return !(e && atoi(e) == 1);
    }();
    if (allow2 && make_tc_plan_w(B, log_n, r0, rows, D, pl, true, 2, true, true, xsm) == DPF_OK) return DPF_OK;
    return make_tc_plan_w(B, log_n, r0, rows, D, pl, true, 1, true, true, xsm);
  }
  int rc = make_tc_plan_w(B, log_n, r0, rows, D, pl, false, 4, true, true, xsm);
  if (rc != DPF_OK || pl.m < 4) return rc;
  static const bool allow8 = [] {  // DPF_TC_W=4 pins the 4-leaf-pair window (tuning)
    const char *e = getenv("DPF_TC_W");
    return !(e && atoi(e) == 4);
  }();
  if (!allow8) return rc;
  // (a wider window must not trade the small-batch key mapping for the padded one)
  Plan p8;
  if (make_tc_plan_w(B, log_n, r0, rows, D, p8, false, 8, true, pl.Kr == pl.Kt, xsm) == DPF_OK &&
      (!xsm || p8.m >= pl.m))  // (AES: not at the cost of subtree depth)
    pl = p8;
  return DPF_OK;
}

int make_tc_plan_w(uint32_t B, uint32_t log_n, uint64_t r0, uint64_t rows, uint32_t D, Plan &pl, bool et,
                   uint32_t W, bool allow_kr, bool fallback_padded, size_t xsm) {
  std::memset(&pl, 0, sizeof pl);
  pl.xsm = xsm;
  if (D == 0 || D % 4 || D > 1024 || log_n < 3) return DPF_EINVAL;
  pl.tc = true;
  set_ranges(pl, log_n, r0, rows, et);
  const uint32_t n = pl.n;
  pl.r0a = r0 & ~7ull;
  pl.packed_rows = ((pl.r1 + 7) & ~7ull) - pl.r0a;
  // Kt = MMA N: the largest power of two <= 128 whose 4 limb accumulators x
  // n_dt d-tiles x Kt columns fit the 512 TMEM columns (D <= 128: 128 keys,
  // 256: 64, 512: 32, 1024: 16).  D is padded to whole 128-column d-tiles.
  // CTA pairs (cta_group::2) when the d-tiles split evenly over two SMs:
  // each CTA keeps n_dt/2 tiles, so the MMA N doubles to Ktp = 2 Kt (D = 256:
  // 128 keys per MMA instead of 64) and each SM stages half of the table.
  const uint32_t n_dt = (D + 127) / 128;
  static const int pair_env = [] {
    const char *e = getenv("DPF_TC_PAIR");
    return e ? atoi(e) : -1;
  }();
  // MMA N of a single CTA / of a pair: TMEM budget, no wider than the batch
  // (N >= 16, >= 32 for a pair)
  auto mma_n = [&](uint32_t dt_cta, uint32_t kmin) {
    uint32_t k = 128;
    while (4 * dt_cta * k > 512) k >>= 1;
    while (k > kmin && k / 2 >= B) k >>= 1;
    return k;
  };
  // Pairs only where they widen the MMA (measured: same N -> the cross-CTA
  // lockstep costs up to 2 %; early termination at Dp >= 512 pairs lose even
  // with twice the N -- ET D = 1024 13.9 -> 9.6 ms unpaired, B = 32 at D = 256
  // 0.53 -> 0.32 ms)
  pl.pair = n_dt % 2 == 0 && pair_env != 0 && B > 16 && mma_n(n_dt / 2, 32) > mma_n(n_dt, 16) &&
            (!et || n_dt == 2);
  if (pair_env == 1 && n_dt % 2 == 0 && B > 16) pl.pair = true;  // DPF_TC_PAIR=1 forces pairs (A/B)
  const uint32_t n_dt_cta = pl.pair ? n_dt / 2 : n_dt;
  const uint32_t Ktp = pl.pair ? mma_n(n_dt_cta, 32) : mma_n(n_dt_cta, 16);
  pl.Kt = pl.pair ? Ktp / 2 : Ktp;
  pl.nsy = (et && W == 2) ? 2u : tc_y_stages(et);
  // AES: its 64 KB of T-tables leave the DFS stack one level short at 3 y
  // stages; 2 stages buy the level back (a shallower top BFS, whose AES
  // blocks run far below the fused kernel's rate)
  static const bool aes_nsy2 = [] {  // DPF_AES_NSY2=0 keeps 3 stages (A/B)
    const char *e = getenv("DPF_AES_NSY2");
    return !(e && atoi(e) == 0);
  }();
  if (xsm && !et && aes_nsy2) pl.nsy = 2;
  // Small batches (B < MMA N, single CTA): the MMA keeps N = Kt columns but
  // only Kr = B of them carry keys -- the producer threads map to (real key,
  // node), Ft = 512 / Kr nodes per item (a multiple of 4, so a window is
  // whole 32-leaf K-chunks), and the padding columns stay zero in SMEM.  No
  // producer lane expands a padding key's tree (before: Kt - B of every Kt
  // lanes did).  DPF_TC_SMALLB=0 restores the padded mapping (A/B).
  static const bool smallb = [] {
    const char *e = getenv("DPF_TC_SMALLB");
    return !(e && atoi(e) == 0);
  }();
  pl.Kr = (!pl.pair && smallb && allow_kr && B < pl.Kt) ? B : pl.Kt;
  // a Kr-mapped plan whose y ring does not fit falls back to the padded mapping
  auto fail = [&]() {
    return (pl.Kr < pl.Kt && fallback_padded) ? make_tc_plan_w(B, log_n, r0, rows, D, pl, et, W, false, true, xsm)
                                              : DPF_EINVAL;
  };
  pl.Ft = pl.Kr == pl.Kt ? 32 * kTcNP / pl.Kt : (32 * kTcNP / pl.Kr) & ~3u;
  const uint32_t Kr_item = pl.pair ? 2 * pl.Kr : pl.Kr;  // keys per item (both CTAs of a pair)
  pl.tasks = Kr_item * pl.Ft;
  pl.n_ktiles = (B + Kr_item - 1) / Kr_item;
  // W units per node per window: W leaf pairs (W/4 8-row packed blocks), or
  // one final node (16 rows) with early termination.
  pl.R = unit_rows(pl) * W;
  const uint32_t Kw = pl.Ft * pl.R;
  pl.y_stage_bytes = 4 * pl.Kt * Kw;
  // SMEM: T ring + y ring + the DFS stack (16 B per producer thread per level)
  pl.nst = tc_t_stages(D);
  // small-batch key mapping with a y ring too large for 3 stages (B = 4, 5:
  // 64 KB stages): 2 stages
  if (pl.Kr < pl.Kt && !et &&
      1024 + size_t(pl.nst) * dev::kTcTStageBytes + size_t(pl.nsy) * pl.y_stage_bytes + 2 * kTcLevelBytes >
          smem_cap(pl))
    pl.nsy = 2;
  const size_t fixed = 1024 + size_t(pl.nst) * dev::kTcTStageBytes + size_t(pl.nsy) * pl.y_stage_bytes;
  if (fixed > smem_cap(pl)) return fail();
  const uint32_t m_cap = std::min<uint32_t>(14, uint32_t((smem_cap(pl) - fixed) / kTcLevelBytes) + 1);
  const uint32_t m_min = tc_m_min(et, W);  // a subtree holds >= one window
  if (m_cap < m_min || n < m_min) return fail();
  // co-resident CTA pairs: a GPC with an odd SM count leaves an SM unpaired
  const uint32_t workers = pl.pair ? max_pairs(pl.xsm + fixed + tc_stack_bytes(m_cap)) : uint32_t(num_sms());
  pl.m = choose_m_target(pl, n, m_min, m_cap, workers);
  if (const char *e = getenv("DPF_FORCE_M")) {  // tuning override
    const uint32_t fm = uint32_t(atoi(e));
    if (fm >= m_min && fm <= std::min<uint32_t>(n, m_cap)) pl.m = fm;
  }
  pl.f = n - pl.m;
  pl.lo_f = pl.nr0 >> pl.m;
  pl.F = ((pl.nr1 - 1) >> pl.m) - pl.lo_f + 1;
  pl.cap = pl.F;
  const uint64_t items = uint64_t(pl.n_ktiles) * ((pl.F + pl.Ft - 1) / pl.Ft);
  if (items > 0x7FFFFFFFull) return fail();
  pl.n_items = uint32_t(items);
  pl.W = W;
  pl.nwin = (et ? (1u << pl.m) : (1u << (pl.m - 1))) / W;
  if (pl.nwin == 0) return fail();
  const uint32_t cols = n_dt_cta * 4 * Ktp;
  pl.tmem_cols = 32;
  while (pl.tmem_cols < cols) pl.tmem_cols <<= 1;
  pl.smem_bytes = pl.xsm + fixed + tc_stack_bytes(pl.m);
  if (pl.smem_bytes > 227 * 1024) return fail();
  pl.grid = pl.pair ? 2 * choose_grid(pl.n_items, pl.n_ktiles, workers) : choose_grid(pl.n_items, pl.n_ktiles);
  pl.prf_blocks = count_blocks(pl, B);
  return DPF_OK;
}

struct Workspace {
  uint4 *front[2];
  uint8_t *keys;
  size_t bytes;
};

size_t layout(const Plan &pl, uint32_t B, size_t kstride, Workspace *ws, void *base) {
  size_t off = 0;
  const size_t fbytes = align_up(size_t(B) * pl.cap * 16, kAlign);
  const size_t kbytes = align_up(size_t(B) * kstride, kAlign);
  if (ws) {
    uint8_t *b = static_cast<uint8_t *>(base);
    ws->front[0] = reinterpret_cast<uint4 *>(b + off);
    ws->front[1] = reinterpret_cast<uint4 *>(b + off + fbytes);
    ws->keys = b + off + 2 * fbytes;
  }
  off += 2 * fbytes + kbytes;
  return off;
}

thread_local dpf_eval_stats g_stats{};

// dpf_eval_stats.kernel_id: which fused-kernel instantiation a plan launches
// (include/dpfpir.h): bit 0 tcgen05, bit 1 CTA pair, bit 2 producer epilogue,
// bit 3 small-batch key mapping, bits 4-7 y-ring stages, bits 8-11 PRF, bits
// 12-17 producer warps, bits 18-23 consumer keys per warp (IMAD), bits 24-31
// consumer column words (IMAD).
uint32_t kernel_id(const Plan &pl) {
  if (pl.tc) {
    const uint32_t epip = pl.prf == DPF_PRF_CHACHA20_ET;
    const uint32_t smallb = pl.Kr && pl.Kr < pl.Kt;
    return 1u | (uint32_t(pl.pair) << 1) | (epip << 2) | (smallb << 3) | (pl.nsy << 4) | (pl.prf << 8) |
           (16u << 12);
  }
  return (pl.prf << 8) | (uint32_t(pl.kc.NP) << 12) | (uint32_t(pl.kc.KPW) << 18) | (uint32_t(pl.kc.CPL) << 24);
}

// Optional per-launch timing of the fused kernel (bench instrumentation).
struct KernelTimer {
  std::vector<cudaEvent_t> ev;
  uint32_t used = 0;
  bool on = false;
  ~KernelTimer() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};
thread_local KernelTimer g_timer;

// Per-thread pinned staging ring for host keys (2 slots, grown on demand).
struct Staging {
  uint8_t *buf[2] = {nullptr, nullptr};
  size_t cap[2] = {0, 0};
  cudaEvent_t done[2] = {nullptr, nullptr};
  int next = 0;
  ~Staging() {
    for (int i = 0; i < 2; ++i) {
      if (buf[i]) cudaFreeHost(buf[i]);
      if (done[i]) cudaEventDestroy(done[i]);
    }
  }
};
thread_local Staging g_staging;

// The tcgen05 fused kernel (single CTAs or CTA pairs) for a plan, timed by
// the optional kernel timer.  Used by single-table and grouped launches.
// PDL between the top BFS and the fused kernel; DPF_PDL=0 disables (A/B).
bool use_pdl() {
  static const bool on = [] {
    const char *e = getenv("DPF_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

int launch_tc_kernel(const Plan &pl, const dev::FusedParams &p, cudaStream_t st) {
  const bool timed = g_timer.on && 2 * g_timer.used + 1 < g_timer.ev.size();
  dev::TcParams tp;
  tp.f = p;
  tp.y_stage_bytes = pl.y_stage_bytes;
  tp.tmem_cols = pl.tmem_cols;
  static const uint32_t spin = [] {
    const char *e = getenv("DPF_LOADER_SPIN");
    return uint32_t(e && atoi(e) == 1);
  }();
  // early termination's T ring turns over 4x faster per block: the loader
  // polls (try_wait) instead of sleeping (measured t5 ET 0.807 -> 0.815)
  tp.loader_spin = spin || pl.prf == DPF_PRF_CHACHA20_ET;
  static const uint32_t nomma = [] {
    const char *e = getenv("DPF_DEBUG_NOMMA");
    return uint32_t(e && atoi(e) == 1);
  }();
  tp.debug_nomma = nomma;
  static const uint32_t role_swap = [] {
    const char *e = getenv("DPF_ROLE_SWAP");
    return uint32_t(e && atoi(e) == 1);
  }();
  tp.role_swap = role_swap;
  using TcFn = void (*)(const dev::TcParams);
  TcFn fn;
  // early termination: producers drain TMEM (EPIP, 18 warps, 96 registers)
  const bool epip = pl.prf == DPF_PRF_CHACHA20_ET;
  if (pl.prf == DPF_PRF_AES128 && pl.Kr < pl.Kt)
    fn = pl.nsy == 2 ? &dev::fused_eval_tc_kernel<dev::PrfAesTt, kTcNP, 2, 4, false, false, true>
                     : &dev::fused_eval_tc_kernel<dev::PrfAesTt, kTcNP, kTcNSY, 4, false, false, true>;
  else if (pl.prf == DPF_PRF_AES128)
    fn = pl.nsy == 2 ? (pl.pair ? &dev::fused_eval_tc_kernel<dev::PrfAesTt, kTcNP, 2, 4, true, false>
                                : &dev::fused_eval_tc_kernel<dev::PrfAesTt, kTcNP, 2, 4, false, false>)
                     : (pl.pair ? &dev::fused_eval_tc_kernel<dev::PrfAesTt, kTcNP, kTcNSY, 4, true, false>
                                : &dev::fused_eval_tc_kernel<dev::PrfAesTt, kTcNP, kTcNSY, 4, false, false>);
  else if (epip && pl.Kr < pl.Kt)  // small-batch key mapping (single CTA)
    fn = pl.nsy == 2 ? &dev::fused_eval_tc_kernel<dev::PrfChachaEt, kTcNP, 2, 4, false, true, true>
                     : &dev::fused_eval_tc_kernel<dev::PrfChachaEt, kTcNP, kTcNSYEt, 4, false, true, true>;
  else if (epip)
    fn = pl.nsy == 2 ? (pl.pair ? &dev::fused_eval_tc_kernel<dev::PrfChachaEt, kTcNP, 2, 4, true, true>
                                : &dev::fused_eval_tc_kernel<dev::PrfChachaEt, kTcNP, 2, 4, false, true>)
                     : (pl.pair ? &dev::fused_eval_tc_kernel<dev::PrfChachaEt, kTcNP, kTcNSYEt, 4, true, true>
                                : &dev::fused_eval_tc_kernel<dev::PrfChachaEt, kTcNP, kTcNSYEt, 4, false, true>);
  else if (pl.Kr < pl.Kt)  // small-batch key mapping (single CTA; 2 y stages of 64 KB for B = 4, 5)
    fn = pl.nsy == 2 ? &dev::fused_eval_tc_kernel<dev::PrfChacha, kTcNP, 2, 4, false, false, true>
                     : &dev::fused_eval_tc_kernel<dev::PrfChacha, kTcNP, kTcNSY, 4, false, false, true>;
  else
    fn = pl.pair ? &dev::fused_eval_tc_kernel<dev::PrfChacha, kTcNP, kTcNSY, 4, true, false>
                 : &dev::fused_eval_tc_kernel<dev::PrfChacha, kTcNP, kTcNSY, 4, false, false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem_bytes)) != cudaSuccess)
    return DPF_ECUDA;
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(32 * (kTcNP + dev::tc_extra_warps(epip)));
  cfg.dynamicSmemBytes = pl.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = pl.pair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // PDL behind the top BFS (with the kernel timer on, its start event sits
  // between the two launches: any early start counts in the kernel's time)
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = use_pdl();
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (timed) cudaEventRecord(g_timer.ev[2 * g_timer.used], st);
  if (cudaLaunchKernelEx(&cfg, fn, tp) != cudaSuccess) return DPF_ECUDA;
  if (timed) cudaEventRecord(g_timer.ev[2 * g_timer.used++ + 1], st);
  return cudaGetLastError() == cudaSuccess ? DPF_OK : DPF_ECUDA;
}

int launch_eval(const Plan &pl, const uint8_t *keys_dev, uint32_t kstride, uint32_t B, const uint32_t *table,
                uint32_t D, uint32_t *out, const Workspace &ws, cudaStream_t st, uint32_t *kernels,
                uint32_t flags = 0) {
  uint32_t nk = 0;
  // a7: answers start at zero, unless the caller accumulates (DPF_EVAL_ACCUMULATE:
  // `out` may be another rank's buffer mapped over NVLink, zeroed by its owner).
  // With a top BFS the zeroing is folded into it (B*D is a multiple of 4 words).
  const bool zero = !(flags & DPF_EVAL_ACCUMULATE);
  const bool fold = pl.f >= 1 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (zero && !fold && cudaMemsetAsync(out, 0, size_t(B) * D * 4, st) != cudaSuccess) return DPF_ECUDA;
  uint4 *zero_ptr = (zero && fold) ? reinterpret_cast<uint4 *>(out) : nullptr;
  const uint64_t zero_vec = zero_ptr ? uint64_t(B) * D / 4 : 0;
  // a2: levels 1..f; level k lands in front[(f-k)&1] so level f is front[0].
  if (pl.f == 0) {
    dev::copy_roots_kernel<<<(B + 127) / 128, 128, 0, st>>>(keys_dev, kstride, B, ws.front[0], pl.cap);
    ++nk;
  }
  // The top of the tree works on tree-leaf (final node) ranges [nr0, nr1):
  // with early termination (R20) the levels are Eq. 3 ChaCha20 levels.
  // One launch: split depth s keeps <= 2^10 nodes per CTA and >= 2 CTAs per SM.
  if (pl.f >= 1) {
    uint32_t s = pl.f > dev::kTopSmemLevels ? pl.f - dev::kTopSmemLevels : 0;
    while (s < pl.f && (uint64_t(B) << s) < 2ull * num_sms()) ++s;
    const uint64_t cnt_s = ((pl.nr1 - 1) >> (pl.n - s)) - (pl.nr0 >> (pl.n - s)) + 1;
    const uint64_t grid = uint64_t(B) * cnt_s;
    if (grid > 0x7FFFFFFFull) return DPF_EINVAL;
    if (pl.prf == DPF_PRF_AES128) {
      if (!allow_dyn_smem(&dev::expand_top_split_kernel<dev::PrfAesTt>, dev::kAesSmemBytes)) return DPF_ECUDA;
      dev::expand_top_split_kernel<dev::PrfAesTt><<<uint32_t(grid), 256, dev::kAesSmemBytes, st>>>(
          keys_dev, kstride, pl.n, s, pl.f, pl.nr0, pl.nr1, ws.front[0], pl.cap, zero_ptr, zero_vec);
    } else
      dev::expand_top_split_kernel<dev::PrfChacha><<<uint32_t(grid), 256, 0, st>>>(
          keys_dev, kstride, pl.n, s, pl.f, pl.nr0, pl.nr1, ws.front[0], pl.cap, zero_ptr, zero_vec);
    ++nk;
  }
  const bool timed = g_timer.on && 2 * g_timer.used + 1 < g_timer.ev.size();
  dev::FusedParams p;
  std::memset(&p, 0, sizeof p);
  dev::GroupDesc &g = p.g0;
  g.keys = keys_dev;
  g.frontier = ws.front[0];
  g.T = table;
  g.shares = out;
  g.cap = pl.cap;
  g.F = pl.F;
  g.lo_f = pl.lo_f;
  g.r0 = pl.r0;
  g.r1 = pl.r1;
  g.nr0 = pl.nr0;
  g.nr1 = pl.nr1;
  g.r0a = pl.r0a;
  g.packed_rows = pl.packed_rows;
  g.kstride = kstride;
  g.B = B;
  g.n = pl.n;
  g.m = pl.m;
  g.nwin = pl.nwin;
  g.n_ktiles = pl.n_ktiles;
  g.item_base = 0;
  g.key_base = 0;
  p.groups = nullptr;
  p.n_groups = 1;
  p.n_items = pl.n_items;
  p.D = D;
  p.Kt = pl.Kt;
  p.Kr = pl.Kr ? pl.Kr : pl.Kt;
  p.Ft = pl.Ft;
  p.tasks = pl.tasks;
  p.W = pl.W;
  p.R = pl.R;
  p.CG = pl.CG;
  p.KG = pl.KG;
  p.SG = pl.SG;
  p.y_stage_words = pl.y_stage_words;
  p.t_stage_words = pl.t_stage_words;
  p.CN = pl.CN;
  p.n_chunks = pl.n_chunks;
  p.NST = pl.NST;
  p.sys_red = (flags & DPF_EVAL_ACCUMULATE) ? 1u : 0u;
  if (pl.tc) {
    const int rc = launch_tc_kernel(pl, p, st);
    if (rc) return rc;
    ++nk;
    if (kernels) *kernels = nk;
    return DPF_OK;
  }
  auto kfn = pl.kc.get(pl.prf);
  if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem_bytes)) != cudaSuccess)
    return DPF_ECUDA;
  if (timed) cudaEventRecord(g_timer.ev[2 * g_timer.used], st);
  {
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(pl.grid);
    cfg.blockDim = dim3(32 * (pl.kc.NP + kNC + 1));
    cfg.dynamicSmemBytes = pl.smem_bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = use_pdl();
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kfn, p) != cudaSuccess) return DPF_ECUDA;
  }
  if (timed) cudaEventRecord(g_timer.ev[2 * g_timer.used++ + 1], st);
  ++nk;
  if (cudaGetLastError() != cudaSuccess) return DPF_ECUDA;
  if (kernels) *kernels = nk;
  return DPF_OK;
}

int check_common(uint32_t B, const uint32_t *table, uint64_t row_begin, uint64_t rows, uint32_t D,
                 const uint32_t *out, void *ws, uint32_t n, uint32_t prf) {
  if (B == 0 || !table || !out || !ws || D == 0 || D > 1024 || (D & 3)) return DPF_EINVAL;
  if (n < (prf == DPF_PRF_CHACHA20_ET ? DPF_ET_BITS + 1 : 1) || n > DPF_MAX_LOG_N) return DPF_EKEY;
  if (rows == 0) return DPF_EINVAL;
  const uint64_t dom = n >= 64 ? ~0ull : (1ull << n);
  if (row_begin >= dom || rows > dom - row_begin) return DPF_EINVAL;
  if ((reinterpret_cast<uintptr_t>(table) & 15) || (reinterpret_cast<uintptr_t>(ws) & (kAlign - 1)))
    return DPF_EINVAL;
  return DPF_OK;
}

int eval_impl(const dpf_key *keys, uint32_t B, const uint8_t *keys_wire_dev, uint32_t log_n, uint32_t prf,
              const uint32_t *table, uint64_t row_begin, uint64_t rows, uint32_t D, uint32_t *out, void *workspace,
              size_t ws_bytes, cudaStream_t st, bool packed = false, uint32_t flags = 0) {
  uint32_t n = log_n;
  if (keys) {
    if (B == 0) return DPF_EINVAL;
    prf = keys[0].prf;
  }
  if (prf != DPF_PRF_CHACHA20 && prf != DPF_PRF_AES128 && prf != DPF_PRF_CHACHA20_ET) return DPF_EUNSUPPORTED;
  if (keys) {
    if (B == 0) return DPF_EINVAL;
    n = keys[0].log_n;
    for (uint32_t b = 0; b < B; ++b) {
      if (!host_key_valid(keys[b])) return DPF_EKEY;
      if (keys[b].log_n != n || keys[b].prf != keys[0].prf) return DPF_EKEY;
    }
  }
  int rc = check_common(B, table, row_begin, rows, D, out, workspace, n, prf);
  if (rc) return rc;
  Plan pl;
  const bool et = prf == DPF_PRF_CHACHA20_ET;
  rc = packed ? make_tc_plan(B, n, row_begin, rows, D, pl, et, prf_smem(prf))
              : make_plan(B, n, row_begin, rows, D, pl, et, prf_smem(prf));
  if (rc) return rc;
  pl.prf = prf;
  const uint32_t kstride = uint32_t(dpf_key_wire_size_prf(n, prf));
  Workspace ws;
  const size_t need = layout(pl, B, kstride, &ws, workspace);
  if (ws_bytes < need) return DPF_ENOMEM;
  const uint8_t *kd = keys_wire_dev;
  if (keys) {
    // a1: serialize into pinned staging, then one H2D copy (async).
    Staging &sg = g_staging;
    const int slot = sg.next;
    sg.next ^= 1;
    const size_t kb = size_t(B) * kstride;
    if (sg.done[slot]) cudaEventSynchronize(sg.done[slot]);  // previous use of this slot finished copying
    if (sg.cap[slot] < kb) {
      if (sg.buf[slot]) cudaFreeHost(sg.buf[slot]);
      sg.buf[slot] = nullptr;
      sg.cap[slot] = 0;
      if (cudaHostAlloc(&sg.buf[slot], kb, cudaHostAllocDefault) != cudaSuccess) return DPF_ECUDA;
      sg.cap[slot] = kb;
    }
    if (!sg.done[slot] && cudaEventCreateWithFlags(&sg.done[slot], cudaEventDisableTiming) != cudaSuccess)
      return DPF_ECUDA;
    for (uint32_t b = 0; b < B; ++b) {
      size_t w = 0;
      if (dpf_key_serialize(&keys[b], sg.buf[slot] + size_t(b) * kstride, kstride, &w) != DPF_OK) return DPF_EKEY;
    }
    if (cudaMemcpyAsync(ws.keys, sg.buf[slot], kb, cudaMemcpyHostToDevice, st) != cudaSuccess) return DPF_ECUDA;
    if (cudaEventRecord(sg.done[slot], st) != cudaSuccess) return DPF_ECUDA;
    kd = ws.keys;
  }
  uint32_t nk = 0;
  rc = launch_eval(pl, kd, kstride, B, table, D, out, ws, st, &nk, flags);
  if (rc) return rc;
  g_stats.prf_blocks = pl.prf_blocks;
  g_stats.kernels = nk;
  g_stats.frontier_depth = pl.f;
  g_stats.keys_per_tile = pl.pair ? 2 * pl.Kt : pl.Kt;
  g_stats.nodes_per_tile = pl.Ft;
  g_stats.work_items = pl.n_items;
  g_stats.grid = pl.grid;
  g_stats.kernel_id = kernel_id(pl);
  return DPF_OK;
}

}  // namespace
}  // namespace dpfpir

using namespace dpfpir;

extern "C" size_t dpf_eval_workspace_bytes(uint32_t B, uint32_t log_n, uint64_t row_count, uint32_t D) {
  if (B == 0 || log_n < 1 || log_n > DPF_MAX_LOG_N || row_count == 0 || D == 0 || D > 1024 || (D & 3)) return 0;
  Plan pl;
  if (make_plan(B, log_n, 0, row_count, D, pl) != DPF_OK) return 0;
  // The frontier size depends on the alignment of row_begin; size for the
  // worst case (one extra node per key).  Covers every scheme and both
  // contraction paths (IMAD, tcgen05).
  pl.cap += 1;
  size_t bytes = layout(pl, B, dpf_key_wire_size(log_n), nullptr, nullptr);
  // every PRF (AES: less SMEM for the DFS stack -> possibly a deeper frontier)
  for (uint32_t prf : {uint32_t(DPF_PRF_CHACHA20), uint32_t(DPF_PRF_AES128), uint32_t(DPF_PRF_CHACHA20_ET)}) {
    const bool et = prf == DPF_PRF_CHACHA20_ET;
    if (et && log_n <= DPF_ET_BITS) break;
    const size_t kst = dpf_key_wire_size_prf(log_n, prf);
    Plan q;
    if (make_plan(B, log_n, 0, row_count, D, q, et, prf_smem(prf)) == DPF_OK) {
      q.cap += 1;
      bytes = std::max(bytes, layout(q, B, kst, nullptr, nullptr));
    }
    if (make_tc_plan(B, log_n, 0, row_count, D, q, et, prf_smem(prf)) == DPF_OK) {
      q.cap += 1;
      bytes = std::max(bytes, layout(q, B, kst, nullptr, nullptr));
    }
  }
  return bytes;
}

extern "C" int dpf_eval_plan(uint32_t B, uint32_t log_n, uint32_t prf, uint64_t row_begin, uint64_t row_count,
                             uint32_t D, int packed, dpf_eval_stats *out) {
  if (!out || B == 0 || D == 0 || D > 1024 || (D & 3) || row_count == 0) return DPF_EINVAL;
  if (prf != DPF_PRF_CHACHA20 && prf != DPF_PRF_AES128 && prf != DPF_PRF_CHACHA20_ET) return DPF_EUNSUPPORTED;
  const bool et = prf == DPF_PRF_CHACHA20_ET;
  if (log_n < (et ? DPF_ET_BITS + 1 : 1) || log_n > DPF_MAX_LOG_N) return DPF_EINVAL;
  const uint64_t dom = 1ull << log_n;
  if (row_begin >= dom || row_count > dom - row_begin) return DPF_EINVAL;
  Plan pl;
  const int rc = packed ? make_tc_plan(B, log_n, row_begin, row_count, D, pl, et, prf_smem(prf))
                        : make_plan(B, log_n, row_begin, row_count, D, pl, et, prf_smem(prf));
  if (rc) return rc;
  pl.prf = prf;
  out->prf_blocks = pl.prf_blocks;
  out->kernels = 0;
  out->frontier_depth = pl.f;
  out->keys_per_tile = pl.pair ? 2 * pl.Kt : pl.Kt;
  out->nodes_per_tile = pl.Ft;
  out->work_items = pl.n_items;
  out->grid = pl.grid;
  out->kernel_id = kernel_id(pl);
  return DPF_OK;
}

// Packed width: D padded to whole 128-column d-tiles (padding columns are zero).
inline uint32_t packed_width(uint32_t D) { return (D + 127) & ~127u; }

extern "C" size_t dpf_table_packed_bytes(uint64_t row_begin, uint64_t row_count, uint32_t D) {
  if (row_count == 0 || D == 0 || D % 4 || D > 1024) return 0;
  const uint64_t r0a = row_begin & ~7ull, r1a = (row_begin + row_count + 7) & ~7ull;
  return size_t((r1a - r0a) * 4ull * packed_width(D));
}

extern "C" int dpf_table_pack(const uint32_t *table_shard, uint64_t row_begin, uint64_t row_count, uint32_t D,
                              void *packed, void *stream) {
  if (!table_shard || !packed || row_count == 0 || D == 0 || D % 4 || D > 1024) return DPF_EINVAL;
  if ((reinterpret_cast<uintptr_t>(table_shard) & 15) || (reinterpret_cast<uintptr_t>(packed) & 15))
    return DPF_EINVAL;
  const uint64_t r0a = row_begin & ~7ull, r1a = (row_begin + row_count + 7) & ~7ull;
  const uint64_t nblocks = (r1a - r0a) / 8;
  const uint64_t total = nblocks * 8 * (packed_width(D) / 16);
  const uint32_t grid = uint32_t(std::min<uint64_t>((total + 255) / 256, 148ull * 32));
  dev::table_pack_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      table_shard, row_begin, row_begin + row_count, r0a, nblocks, D, packed_width(D), static_cast<uint8_t *>(packed));
  return cudaGetLastError() == cudaSuccess ? DPF_OK : DPF_ECUDA;
}

extern "C" int dpf_eval_batch_packed(const dpf_key *keys, uint32_t B, const void *packed, uint64_t row_begin,
                                     uint64_t row_count, uint32_t D, uint32_t *partial, void *workspace,
                                     size_t workspace_bytes, void *stream) {
  if (!keys) return DPF_EINVAL;
  return eval_impl(keys, B, nullptr, 0, 0, static_cast<const uint32_t *>(packed), row_begin, row_count, D, partial,
                   workspace, workspace_bytes, static_cast<cudaStream_t>(stream), true);
}

extern "C" int dpf_eval_batch_wire_packed(const uint8_t *keys_wire_dev, uint32_t B, uint32_t log_n, uint32_t prf,
                                          const void *packed, uint64_t row_begin, uint64_t row_count, uint32_t D,
                                          uint32_t *partial, void *workspace, size_t workspace_bytes, void *stream) {
  if (!keys_wire_dev || (reinterpret_cast<uintptr_t>(keys_wire_dev) & 15)) return DPF_EINVAL;
  return eval_impl(nullptr, B, keys_wire_dev, log_n, prf, static_cast<const uint32_t *>(packed), row_begin, row_count,
                   D, partial, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), true);
}

extern "C" int dpf_eval_batch_shard(const dpf_key *keys, uint32_t B, const uint32_t *table_shard,
                                    uint64_t row_begin, uint64_t row_count, uint32_t D, uint32_t *partial,
                                    void *workspace, size_t workspace_bytes, void *stream) {
  if (!keys) return DPF_EINVAL;
  return eval_impl(keys, B, nullptr, 0, 0, table_shard, row_begin, row_count, D, partial, workspace,
                   workspace_bytes, static_cast<cudaStream_t>(stream));
}

extern "C" int dpf_eval_batch(const dpf_key *keys, uint32_t B, const uint32_t *table, uint64_t N, uint32_t D,
                              uint32_t *shares, void *workspace, size_t workspace_bytes, void *stream) {
  return dpf_eval_batch_shard(keys, B, table, 0, N, D, shares, workspace, workspace_bytes, stream);
}

extern "C" int dpf_eval_batch_wire(const uint8_t *keys_wire_dev, uint32_t B, uint32_t log_n, uint32_t prf,
                                   const uint32_t *table_shard, uint64_t row_begin, uint64_t row_count, uint32_t D,
                                   uint32_t *partial, void *workspace, size_t workspace_bytes, void *stream) {
  if (!keys_wire_dev || (reinterpret_cast<uintptr_t>(keys_wire_dev) & 15)) return DPF_EINVAL;
  return eval_impl(nullptr, B, keys_wire_dev, log_n, prf, table_shard, row_begin, row_count, D, partial, workspace,
                   workspace_bytes, static_cast<cudaStream_t>(stream));
}

extern "C" int dpf_eval_batch_wire_ex(const uint8_t *keys_wire_dev, uint32_t B, uint32_t log_n, uint32_t prf,
                                      const void *table, int packed, uint64_t row_begin, uint64_t row_count,
                                      uint32_t D, uint32_t *shares, uint32_t flags, void *workspace,
                                      size_t workspace_bytes, void *stream) {
  if (!keys_wire_dev || (reinterpret_cast<uintptr_t>(keys_wire_dev) & 15)) return DPF_EINVAL;
  if (flags & ~uint32_t(DPF_EVAL_ACCUMULATE)) return DPF_EINVAL;
  return eval_impl(nullptr, B, keys_wire_dev, log_n, prf, static_cast<const uint32_t *>(table), row_begin, row_count,
                   D, shares, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), packed != 0, flags);
}

extern "C" int dpf_ipc_export(const void *dev_ptr, uint8_t handle[DPF_IPC_HANDLE_BYTES], uint64_t *offset) {
  if (!dev_ptr || !handle || !offset) return DPF_EINVAL;
  static_assert(sizeof(cudaIpcMemHandle_t) == DPF_IPC_HANDLE_BYTES, "IPC handle size");
  // The handle names the whole allocation (a caching allocator sub-allocates
  // tensors inside it): report dev_ptr's offset from the allocation base.
  using GetRange = int (*)(unsigned long long *, size_t *, unsigned long long);
  static GetRange get_range = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<GetRange>(fn);
  }();
  if (!get_range) return DPF_ECUDA;
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0) return DPF_ECUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void *>(dev_ptr)) != cudaSuccess) return DPF_ECUDA;
  std::memcpy(handle, &h, sizeof h);
  *offset = reinterpret_cast<unsigned long long>(dev_ptr) - base;
  return DPF_OK;
}

extern "C" int dpf_ipc_open(const uint8_t handle[DPF_IPC_HANDLE_BYTES], void **dev_ptr) {
  if (!handle || !dev_ptr) return DPF_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  if (cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return DPF_ECUDA;
  }
  return DPF_OK;
}

extern "C" int dpf_ipc_close(void *dev_ptr) {
  if (!dev_ptr) return DPF_EINVAL;
  return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? DPF_OK : DPF_ECUDA;
}

extern "C" int dpf_serve_batch(const dpf_key *keys, uint32_t B, const uint32_t *table_shard, uint64_t row_begin,
                               uint64_t row_count, uint32_t D, uint32_t *shares_host, void *workspace,
                               size_t workspace_bytes, void *stream) {
  if (!shares_host) return DPF_EINVAL;
  // The device answer lives at the end of the workspace.
  const size_t need = dpf_eval_workspace_bytes(B, keys ? keys[0].log_n : 0, row_count, D);
  const size_t out_bytes = align_up(size_t(B) * D * 4, kAlign);
  if (!keys || need == 0) return DPF_EINVAL;
  if (workspace_bytes < need + out_bytes) return DPF_ENOMEM;
  uint32_t *dev_out = reinterpret_cast<uint32_t *>(static_cast<uint8_t *>(workspace) + need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = eval_impl(keys, B, nullptr, 0, 0, table_shard, row_begin, row_count, D, dev_out, workspace, need, st);
  if (rc) return rc;
  if (cudaMemcpyAsync(shares_host, dev_out, size_t(B) * D * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return DPF_ECUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return DPF_ECUDA;
  return DPF_OK;
}

// ------------------------------------------------------------ graph server
// A serving step for one fixed shape captured once as a CUDA graph: pinned
// key staging -> H2D -> zeroing, top BFS, fused kernel -> D2H of the answers,
// replayed with ONE cudaGraphLaunch per batch (the per-call launch overhead of
// the small configurations is host-side; the graph removes it).
struct dpf_server {
  // One slot per batch in flight: pinned staging for the wire keys and the
  // answers, a private stream, the captured graph, its own workspace region.
  struct Slot {
    uint8_t *keys_pinned = nullptr;  // B x kstride (library-owned pinned staging)
    uint32_t *out_pinned = nullptr;  // B x D
    cudaStream_t st = nullptr;
    cudaGraphExec_t exec = nullptr;
  };
  uint32_t B, log_n, prf, D, kstride;
  std::vector<Slot> slots;
  uint32_t head = 0, inflight = 0;  // next slot to submit into; batches submitted, not collected
};

extern "C" size_t dpf_server_workspace_bytes(uint32_t B, uint32_t log_n, uint32_t prf, uint64_t row_count,
                                             uint32_t D) {
  const size_t kstride = dpf_key_wire_size_prf(log_n, prf);
  const size_t ev = dpf_eval_workspace_bytes(B, log_n, row_count, D);
  if (kstride == 0 || ev == 0) return 0;
  return ev + align_up(size_t(B) * kstride, kAlign) + align_up(size_t(B) * D * 4, kAlign);
}

extern "C" size_t dpf_server_pipeline_workspace_bytes(uint32_t B, uint32_t log_n, uint32_t prf, uint64_t row_count,
                                                      uint32_t D, uint32_t depth) {
  if (depth < 1 || depth > DPF_SERVER_MAX_DEPTH) return 0;
  const size_t one = dpf_server_workspace_bytes(B, log_n, prf, row_count, D);
  return one ? size_t(depth) * align_up(one, kAlign) : 0;
}

namespace dpfpir {
namespace {
void server_free(dpf_server *sv) {
  for (auto &sl : sv->slots) {
    if (sl.exec) cudaGraphExecDestroy(sl.exec);
    if (sl.keys_pinned) cudaFreeHost(sl.keys_pinned);
    if (sl.out_pinned) cudaFreeHost(sl.out_pinned);
    if (sl.st) cudaStreamDestroy(sl.st);
  }
  delete sv;
}

// Capture one slot's serving step (H2D keys, eval, D2H answers) on its stream.
int capture_slot(dpf_server *sv, dpf_server::Slot &sl, const void *table, int packed, uint64_t row_begin,
                 uint64_t row_count, uint8_t *ws) {
  const uint32_t B = sv->B, D = sv->D;
  const size_t ev = dpf_eval_workspace_bytes(B, sv->log_n, row_count, D);
  uint8_t *keys_dev = ws + ev;
  uint32_t *out_dev = reinterpret_cast<uint32_t *>(keys_dev + align_up(size_t(B) * sv->kstride, kAlign));
  const size_t kb = size_t(B) * sv->kstride, ob = size_t(B) * D * 4;
  if (cudaStreamCreateWithFlags(&sl.st, cudaStreamNonBlocking) != cudaSuccess) {
    sl.st = nullptr;
    return DPF_ECUDA;
  }
  if (cudaHostAlloc(&sl.keys_pinned, kb, cudaHostAllocDefault) != cudaSuccess) {
    sl.keys_pinned = nullptr;
    return DPF_ENOMEM;
  }
  if (cudaHostAlloc(&sl.out_pinned, ob, cudaHostAllocDefault) != cudaSuccess) {
    sl.out_pinned = nullptr;
    return DPF_ENOMEM;
  }
  std::memset(sl.keys_pinned, 0, kb);
  // warm-up launch outside capture: first-use attribute/occupancy queries happen here
  int rc = eval_impl(nullptr, B, keys_dev, sv->log_n, sv->prf, static_cast<const uint32_t *>(table), row_begin,
                     row_count, D, out_dev, ws, ev, sl.st, packed != 0);
  if (rc == DPF_OK && cudaStreamSynchronize(sl.st) != cudaSuccess) rc = DPF_ECUDA;
  if (rc != DPF_OK) return rc;
  cudaGraph_t graph = nullptr;
  if (cudaStreamBeginCapture(sl.st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return DPF_ECUDA;
  int r1 = cudaMemcpyAsync(keys_dev, sl.keys_pinned, kb, cudaMemcpyHostToDevice, sl.st) == cudaSuccess ? DPF_OK
                                                                                                       : DPF_ECUDA;
  if (r1 == DPF_OK)
    r1 = eval_impl(nullptr, B, keys_dev, sv->log_n, sv->prf, static_cast<const uint32_t *>(table), row_begin,
                   row_count, D, out_dev, ws, ev, sl.st, packed != 0);
  if (r1 == DPF_OK && cudaMemcpyAsync(sl.out_pinned, out_dev, ob, cudaMemcpyDeviceToHost, sl.st) != cudaSuccess)
    r1 = DPF_ECUDA;
  const cudaError_t e = cudaStreamEndCapture(sl.st, &graph);
  rc = r1 != DPF_OK ? r1 : (e == cudaSuccess ? DPF_OK : DPF_ECUDA);
  if (rc == DPF_OK && cudaGraphInstantiate(&sl.exec, graph, 0) != cudaSuccess) rc = DPF_ECUDA;
  if (graph) cudaGraphDestroy(graph);
  return rc;
}
}  // namespace
}  // namespace dpfpir

extern "C" int dpf_server_pipeline_create(uint32_t B, uint32_t log_n, uint32_t prf, const void *table, int packed,
                                          uint64_t row_begin, uint64_t row_count, uint32_t D, uint32_t depth,
                                          void *workspace, size_t workspace_bytes, void *stream, dpf_server **out) {
  if (!out || !table || !workspace || B == 0) return DPF_EINVAL;
  *out = nullptr;
  const size_t need = dpf_server_pipeline_workspace_bytes(B, log_n, prf, row_count, D, depth);
  if (need == 0) return DPF_EINVAL;
  if (workspace_bytes < need) return DPF_ENOMEM;
  if (reinterpret_cast<uintptr_t>(workspace) & (kAlign - 1)) return DPF_EINVAL;
  const size_t per = align_up(dpf_server_workspace_bytes(B, log_n, prf, row_count, D), kAlign);
  dpf_server *sv = new dpf_server;
  sv->B = B;
  sv->log_n = log_n;
  sv->prf = prf;
  sv->D = D;
  sv->kstride = uint32_t(dpf_key_wire_size_prf(log_n, prf));
  sv->slots.resize(depth);
  // the caller's stream orders the table's preparation; every slot captures
  // and replays on a private stream (the legacy NULL stream cannot be captured)
  int rc = cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) == cudaSuccess ? DPF_OK : DPF_ECUDA;
  for (uint32_t i = 0; i < depth && rc == DPF_OK; ++i)
    rc = capture_slot(sv, sv->slots[i], table, packed, row_begin, row_count,
                      static_cast<uint8_t *>(workspace) + size_t(i) * per);
  if (rc != DPF_OK) {
    cudaGetLastError();
    server_free(sv);
    return rc;
  }
  *out = sv;
  return DPF_OK;
}

extern "C" int dpf_server_create(uint32_t B, uint32_t log_n, uint32_t prf, const void *table, int packed,
                                 uint64_t row_begin, uint64_t row_count, uint32_t D, void *workspace,
                                 size_t workspace_bytes, void *stream, dpf_server **out) {
  return dpf_server_pipeline_create(B, log_n, prf, table, packed, row_begin, row_count, D, 1, workspace,
                                    workspace_bytes, stream, out);
}

// Wire-format header checks of a host key (include/dpfpir.h "Wire format").
// The codec's own predicate (dpf_key_deserialize: magic, version, prf,
// party, log_n range, lsb(root) == party, reserved == 0, ET cw_out == 0) plus
// this server's shape.
static bool wire_header_ok(const uint8_t *k, uint32_t log_n, uint32_t prf) {
  return dpfpir::wire_header_valid(k) && k[5] == prf && k[7] == log_n;
}

extern "C" int dpf_server_submit(dpf_server *sv, const uint8_t *keys_wire_host) {
  if (!sv || !keys_wire_host) return DPF_EINVAL;
  if (sv->inflight == sv->slots.size()) return DPF_EBUSY;
  for (uint32_t b = 0; b < sv->B; ++b)
    if (!wire_header_ok(keys_wire_host + size_t(b) * sv->kstride, sv->log_n, sv->prf)) return DPF_EKEY;
  dpf_server::Slot &sl = sv->slots[sv->head];
  // the slot is free (its previous batch was collected): its staging can be overwritten
  std::memcpy(sl.keys_pinned, keys_wire_host, size_t(sv->B) * sv->kstride);
  if (cudaGraphLaunch(sl.exec, sl.st) != cudaSuccess) return DPF_ECUDA;
  sv->head = (sv->head + 1) % uint32_t(sv->slots.size());
  ++sv->inflight;
  return DPF_OK;
}

extern "C" int dpf_server_collect(dpf_server *sv, uint32_t *shares_host) {
  if (!sv || !shares_host) return DPF_EINVAL;
  if (sv->inflight == 0) return DPF_EINVAL;
  const uint32_t n = uint32_t(sv->slots.size());
  dpf_server::Slot &sl = sv->slots[(sv->head + n - sv->inflight) % n];  // oldest batch in flight
  if (cudaStreamSynchronize(sl.st) != cudaSuccess) return DPF_ECUDA;
  std::memcpy(shares_host, sl.out_pinned, size_t(sv->B) * sv->D * 4);
  --sv->inflight;
  return DPF_OK;
}

extern "C" int dpf_server_run(dpf_server *sv, const uint8_t *keys_wire_host, uint32_t *shares_host) {
  if (!sv || !keys_wire_host || !shares_host) return DPF_EINVAL;
  if (sv->inflight) return DPF_EBUSY;  // run is submit + collect of one batch
  const int rc = dpf_server_submit(sv, keys_wire_host);
  return rc != DPF_OK ? rc : dpf_server_collect(sv, shares_host);
}

extern "C" void dpf_server_destroy(dpf_server *sv) {
  if (!sv) return;
  for (auto &sl : sv->slots)
    if (sl.st) cudaStreamSynchronize(sl.st);
  dpfpir::server_free(sv);
}

extern "C" int dpf_eval_leaves(const dpf_key *keys, uint32_t B, uint32_t *leaves, void *workspace,
                               size_t workspace_bytes, void *stream) {
  if (!keys || B == 0 || !leaves || !workspace) return DPF_EINVAL;
  const uint32_t n = keys[0].log_n;
  for (uint32_t b = 0; b < B; ++b)
    if (!host_key_valid(keys[b]) || keys[b].log_n != n || keys[b].prf != keys[0].prf) return DPF_EKEY;
  if (n > 20) return DPF_EINVAL;
  const uint32_t kstride = uint32_t(dpf_key_wire_size_prf(n, keys[0].prf));
  if (workspace_bytes < size_t(B) * kstride) return DPF_ENOMEM;
  std::vector<uint8_t> staged(size_t(B) * kstride);
  for (uint32_t b = 0; b < B; ++b) dpf_key_serialize(&keys[b], staged.data() + size_t(b) * kstride, kstride, nullptr);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(workspace, staged.data(), staged.size(), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return DPF_ECUDA;
  const uint64_t total = (uint64_t(B) << n);
  const uint32_t grid = uint32_t(std::min<uint64_t>((total + 255) / 256, 148ull * 8));
  uint8_t *kd = static_cast<uint8_t *>(workspace);
  if (keys[0].prf == DPF_PRF_AES128) {
    if (!allow_dyn_smem(&dev::eval_leaves_kernel<dev::PrfAesTt>, dev::kAesSmemBytes)) return DPF_ECUDA;
    dev::eval_leaves_kernel<dev::PrfAesTt><<<grid, 256, dev::kAesSmemBytes, st>>>(kd, kstride, B, n, leaves);
  } else if (keys[0].prf == DPF_PRF_CHACHA20_ET) {
    dev::eval_leaves_kernel<dev::PrfChachaEt><<<grid, 256, 0, st>>>(kd, kstride, B, n, leaves);
  } else {
    dev::eval_leaves_kernel<dev::PrfChacha><<<grid, 256, 0, st>>>(kd, kstride, B, n, leaves);
  }
  if (cudaGetLastError() != cudaSuccess) return DPF_ECUDA;
  // staged is pageable: the H2D above completed its staging before return.
  return DPF_OK;
}

extern "C" int dpf_kernel_timer_begin(uint32_t capacity) {
  KernelTimer &t = g_timer;
  while (t.ev.size() < 2 * size_t(capacity)) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return DPF_ECUDA;
    t.ev.push_back(e);
  }
  t.used = 0;
  t.on = capacity > 0;
  return DPF_OK;
}

extern "C" int dpf_kernel_timer_read(float *ms, uint32_t capacity, uint32_t *count) {
  KernelTimer &t = g_timer;
  t.on = false;
  const uint32_t n = std::min(t.used, capacity);
  for (uint32_t i = 0; i < n; ++i) {
    if (cudaEventSynchronize(t.ev[2 * i + 1]) != cudaSuccess) return DPF_ECUDA;
    if (ms && cudaEventElapsedTime(&ms[i], t.ev[2 * i], t.ev[2 * i + 1]) != cudaSuccess) return DPF_ECUDA;
  }
  if (count) *count = n;
  t.used = 0;
  return DPF_OK;
}

extern "C" int dpf_last_eval_stats(dpf_eval_stats *out) {
  if (!out) return DPF_EINVAL;
  *out = g_stats;
  return DPF_OK;
}

// =================================================================== grouped
namespace dpfpir {
namespace {

struct GroupedPlan {
  Plan cfg;  // shared kernel configuration (Kt, Ft, W, tiles, SMEM)
  std::vector<dev::GroupDesc> desc;
  std::vector<uint32_t> order;  // launch order (largest subtrees first)
  size_t front_bytes, keys_bytes, desc_bytes, total_bytes;  // keys_bytes: 0 (keys stay in place)
};

// Shared configuration for all groups (same D and PRF): key tile from the
// largest batch; per group the subtree depth m_g keeps >= Ft frontier nodes
// per key and f_g = n_g - m_g <= kTopSmemLevels (one grouped top launch);
// items ordered by subtree size so the static round-robin stays balanced.
int make_grouped_tc_plan(const dpf_eval_group *gs, uint32_t G, uint32_t D, uint32_t prf, GroupedPlan &gp);

int make_grouped_plan(const dpf_eval_group *gs, uint32_t G, uint32_t D, uint32_t prf, GroupedPlan &gp,
                      bool packed = false) {
  if (packed) return make_grouped_tc_plan(gs, G, D, prf, gp);
  if (!gs || G == 0 || D == 0 || D > 1024 || (D & 3)) return DPF_EINVAL;
  if (prf != DPF_PRF_CHACHA20 && prf != DPF_PRF_AES128 && prf != DPF_PRF_CHACHA20_ET) return DPF_EUNSUPPORTED;
  const bool et = prf == DPF_PRF_CHACHA20_ET;
  const uint32_t v = et ? DPF_ET_BITS : 0u;  // log2(rows per tree leaf)
  uint32_t Bmax = 0;
  for (uint32_t i = 0; i < G; ++i) {
    const dpf_eval_group &g = gs[i];
    if (!g.keys_wire || !g.table || !g.shares || g.B == 0 || g.log_n < 1 + v || g.log_n > DPF_MAX_LOG_N ||
        g.row_count == 0)
      return DPF_EINVAL;
    const uint64_t dom = 1ull << g.log_n;
    if (g.row_begin >= dom || g.row_count > dom - g.row_begin) return DPF_EINVAL;
    if ((reinterpret_cast<uintptr_t>(g.table) & 15) || (reinterpret_cast<uintptr_t>(g.keys_wire) & 15))
      return DPF_EINVAL;
    Bmax = std::max(Bmax, g.B);
  }
  Plan &pl = gp.cfg;
  // Shared key tile: the Kt (power of two) that minimises the padded work
  // sum_g ceil(B_g / Kt) * Kt * rows_g (lanes of missing keys idle), larger
  // Kt on ties (fewer table re-reads).
  uint32_t best_kt = 1;
  double best_cost = 0;
  for (uint32_t kt = 1; kt <= 32; kt <<= 1) {
    if (kt * D > 8192) break;
    double cost = 0;
    for (uint32_t i = 0; i < G; ++i) cost += double((gs[i].B + kt - 1) / kt) * kt * double(gs[i].row_count);
    if (kt == 1 || cost <= best_cost) {
      best_cost = cost;
      best_kt = kt;
    }
  }
  // reuse the single-group planner for the shared part (tile, Ft, SMEM rules)
  int rc = make_plan(best_kt, 20, 0, 1u << 20, D, pl, et, prf_smem(prf));
  if (rc) return rc;
  pl.prf = prf;
  (void)Bmax;
  const uint32_t NP = uint32_t(pl.kc.NP);
  uint32_t m_cap = std::min<uint32_t>(14, uint32_t((64 * 1024) / (32 * NP * 16)));
  // Balance: a common cap on the subtree depth so that the items of all
  // groups number >= 8 per SM (one item per key tile and group starves most
  // SMs when one big table dominates).  Streaming regime (Kt <= 2: every
  // table row serves <= 2 keys, so the table streams at the PRF rate): cap m
  // so that one window covers whole subtrees, which makes each T-ring entry
  // one contiguous bulk copy instead of one small copy per node.
  // m_floor: no group's subtrees shallower than one full window (the shared
  // window W must divide every group's 2^(m-1); tiny groups would drag it
  // down to one leaf pair per node and make every T copy tiny).
  uint32_t m_floor = 1;
  {
    double units = 0;
    for (uint32_t i = 0; i < G; ++i)
      units += double((gs[i].B + pl.Kt - 1) / pl.Kt) * double(gs[i].row_count >> v);
    const double per_item = units / (double(pl.Ft) * 8.0 * num_sms());
    uint32_t m_bal = 1;
    while (m_bal < 14 && double(2u << m_bal) <= per_item) ++m_bal;
    m_cap = std::min(m_cap, m_bal);
    // window units per subtree: 2^(m-1) leaf pairs, or 2^m final nodes (R20)
    const uint64_t ybudget = et ? 32 * 1024 : 16 * 1024;
    uint32_t Wmax = 8;
    while (Wmax > 1 && uint64_t(pl.Kt) * pl.Ft * unit_rows(pl) * Wmax * 4 > ybudget) Wmax >>= 1;
    while ((et ? (1u << m_floor) : (1u << m_floor) / 2) < Wmax) ++m_floor;  // one window per subtree
    if (pl.Kt <= 2) m_cap = std::min(m_cap, m_floor);
    m_floor = std::min(m_floor, m_cap);
  }
  gp.desc.assign(G, dev::GroupDesc{});
  uint32_t m_min_all = 32;
  for (uint32_t i = 0; i < G; ++i) {
    const dpf_eval_group &g = gs[i];
    dev::GroupDesc &d = gp.desc[i];
    const uint32_t n = g.log_n - v;  // tree depth
    uint32_t lg_rows = 0;
    while ((2ull << lg_rows) <= (g.row_count >> v)) ++lg_rows;  // floor(log2(tree leaves))
    uint32_t lg_ft = 0;
    while ((2u << lg_ft) <= pl.Ft) ++lg_ft;
    uint32_t m = lg_rows > lg_ft ? lg_rows - lg_ft : 1;
    m = std::max(1u, std::min(std::min(std::max(m, m_floor), n), m_cap));
    d.n = n;
    d.m = m;
    d.r0 = g.row_begin;
    d.r1 = g.row_begin + g.row_count;
    d.nr0 = d.r0 >> v;
    d.nr1 = ((d.r1 - 1) >> v) + 1;
    d.lo_f = d.nr0 >> m;
    d.F = ((d.nr1 - 1) >> m) - d.lo_f + 1;
    d.cap = d.F;
    d.B = g.B;
    d.kstride = uint32_t(dpf_key_wire_size_prf(g.log_n, prf));
    d.n_ktiles = (g.B + pl.Kt - 1) / pl.Kt;
    d.T = g.table;
    d.shares = g.shares;
    m_min_all = std::min(m_min_all, m);
  }
  // window: W units (leaf pairs / final nodes) must divide every group's
  // 2^(m-1) (2^m with early termination)
  uint32_t W = std::min<uint32_t>(8, et ? (1u << m_min_all) : (1u << (m_min_all - 1)));
  const size_t stack_bytes = size_t(m_cap) * 32 * NP * 16;
  while (W > 1 && uint64_t(pl.Kt) * pl.Ft * unit_rows(pl) * W * 4 > (et ? 32 * 1024 : 16 * 1024)) W >>= 1;
  for (;; W >>= 1) {
    if (set_windows(pl, W, D, stack_bytes)) break;
    if (W == 1) return DPF_EINVAL;
  }
  // launch order: larger subtrees (bigger items) first
  gp.order.resize(G);
  for (uint32_t i = 0; i < G; ++i) gp.order[i] = i;
  std::stable_sort(gp.order.begin(), gp.order.end(),
                   [&](uint32_t a, uint32_t b) { return gp.desc[a].m > gp.desc[b].m; });
  uint64_t items = 0, keys = 0;
  gp.front_bytes = 0;
  gp.keys_bytes = 0;
  uint64_t blocks = 0;
  for (uint32_t oi : gp.order) {
    dev::GroupDesc &d = gp.desc[oi];
    d.nwin = (et ? (1u << d.m) : (1u << (d.m - 1))) / W;
    d.item_base = uint32_t(items);
    d.key_base = uint32_t(keys);
    items += uint64_t(d.n_ktiles) * ((d.F + pl.Ft - 1) / pl.Ft);
    keys += d.B;
    gp.front_bytes += 2 * align_up(size_t(d.B) * d.cap * 16, kAlign);
    uint64_t top = 0;
    for (uint32_t k = 0; k < d.n - d.m; ++k) top += ((d.nr1 - 1) >> (d.n - k)) - (d.nr0 >> (d.n - k)) + 1;
    const uint64_t per = ((1ull << d.m) - 1) + (et ? (1ull << d.m) : 0);  // + Convert blocks (R20)
    blocks += uint64_t(d.B) * top + uint64_t(d.n_ktiles) * ((d.F + pl.Ft - 1) / pl.Ft) * pl.tasks * per;
  }
  if (items > 0x7FFFFFFFull || keys > 0x7FFFFFFFull) return DPF_EINVAL;
  pl.n_items = uint32_t(items);
  pl.prf_blocks = blocks;
  pl.grid = std::min<uint32_t>(pl.n_items, uint32_t(num_sms()));
  gp.desc_bytes = align_up(size_t(G) * sizeof(dev::GroupDesc), kAlign);
  gp.total_bytes = gp.front_bytes + gp.keys_bytes + gp.desc_bytes;
  return DPF_OK;
}

// Groups share one tcgen05 configuration (MMA N = key tile, window, rings):
// the key tile minimises the padded work sum_g ceil(B_g/N) N rows_g (larger
// on ties); per group the subtree depth as in the IMAD planner (>= 8 items
// per worker overall, >= one window per subtree); tables are limb-packed
// (dpf_table_pack with the group's row_begin / row_count).
int make_grouped_tc_plan(const dpf_eval_group *gs, uint32_t G, uint32_t D, uint32_t prf, GroupedPlan &gp) {
  if (!gs || G == 0 || D == 0 || D > 1024 || (D & 3)) return DPF_EINVAL;
  if (prf != DPF_PRF_CHACHA20 && prf != DPF_PRF_AES128 && prf != DPF_PRF_CHACHA20_ET) return DPF_EUNSUPPORTED;
  const bool et = prf == DPF_PRF_CHACHA20_ET;
  const uint32_t v = et ? DPF_ET_BITS : 0u;
  const uint32_t m_min0 = et ? 1 : 3;
  for (uint32_t i = 0; i < G; ++i) {
    const dpf_eval_group &g = gs[i];
    if (!g.keys_wire || !g.table || !g.shares || g.B == 0 || g.log_n < m_min0 + v || g.log_n > DPF_MAX_LOG_N ||
        g.row_count == 0)
      return DPF_EINVAL;
    const uint64_t dom = 1ull << g.log_n;
    if (g.row_begin >= dom || g.row_count > dom - g.row_begin) return DPF_EINVAL;
    if ((reinterpret_cast<uintptr_t>(g.table) & 15) || (reinterpret_cast<uintptr_t>(g.keys_wire) & 15))
      return DPF_EINVAL;
  }
  // shared MMA N: probe the single-table planner's TMEM rule with B = N
  Plan probe;
  // (a batch far above any MMA N, small enough that the item count stays
  // in range at the shallow subtrees the AES tables leave room for)
  if (make_tc_plan(1u << 12, 20, 0, 1u << 20, D, probe, et, prf_smem(prf)) != DPF_OK) return DPF_EINVAL;
  const uint32_t nmax = probe.pair ? 2 * probe.Kt : probe.Kt, nmin = probe.pair ? 32 : 16;
  uint32_t best = nmax;
  double best_cost = -1;
  for (uint32_t k = nmin; k <= nmax; k <<= 1) {
    double cost = 0;
    for (uint32_t i = 0; i < G; ++i) cost += double((gs[i].B + k - 1) / k) * k * double(gs[i].row_count);
    if (best_cost < 0 || cost <= best_cost) {
      best_cost = cost;
      best = k;
    }
  }
  Plan &pl = gp.cfg;
  // the shared window: W = 4 leaf pairs (tiny groups need shallow subtrees)
  int rc = make_tc_plan_w(best, 20, 0, 1u << 20, D, pl, et, et ? 1 : 4, true, true, prf_smem(prf));
  if (rc) return rc;
  pl.prf = prf;
  const uint32_t m_min = tc_m_min(et, pl.W);
  const uint32_t Ktp = pl.pair ? 2 * pl.Kt : pl.Kt;
  const size_t fixed = 1024 + size_t(pl.nst) * dev::kTcTStageBytes + size_t(pl.nsy) * pl.y_stage_bytes;
  if (fixed > smem_cap(pl)) return DPF_EINVAL;
  uint32_t m_cap = std::min<uint32_t>(14, uint32_t((smem_cap(pl) - fixed) / kTcLevelBytes) + 1);
  const uint32_t workers = pl.pair ? max_pairs(pl.xsm + fixed + tc_stack_bytes(m_cap)) : uint32_t(num_sms());
  {
    double units = 0;
    for (uint32_t i = 0; i < G; ++i) units += double((gs[i].B + Ktp - 1) / Ktp) * double(gs[i].row_count >> v);
    const double per_item = units / (double(pl.Ft) * 8.0 * workers);
    uint32_t m_bal = 1;
    while (m_bal < 14 && double(2u << m_bal) <= per_item) ++m_bal;
    m_cap = std::min(m_cap, std::max(m_bal, m_min));
  }
  if (m_cap < m_min) return DPF_EINVAL;
  gp.desc.assign(G, dev::GroupDesc{});
  uint32_t lg_ft = 0;
  while ((2u << lg_ft) <= pl.Ft) ++lg_ft;
  uint32_t m_max = 0;
  for (uint32_t i = 0; i < G; ++i) {
    const dpf_eval_group &g = gs[i];
    dev::GroupDesc &d = gp.desc[i];
    const uint32_t n = g.log_n - v;
    uint32_t lg_rows = 0;
    while ((2ull << lg_rows) <= (g.row_count >> v)) ++lg_rows;
    uint32_t m = lg_rows > lg_ft ? lg_rows - lg_ft : 1;
    m = std::max(m_min, std::min(std::min(m, n), m_cap));
    d.n = n;
    d.m = m;
    d.r0 = g.row_begin;
    d.r1 = g.row_begin + g.row_count;
    d.nr0 = d.r0 >> v;
    d.nr1 = ((d.r1 - 1) >> v) + 1;
    d.lo_f = d.nr0 >> m;
    d.F = ((d.nr1 - 1) >> m) - d.lo_f + 1;
    d.cap = d.F;
    d.r0a = d.r0 & ~7ull;
    d.packed_rows = ((d.r1 + 7) & ~7ull) - d.r0a;
    d.B = g.B;
    d.kstride = uint32_t(dpf_key_wire_size_prf(g.log_n, prf));
    d.n_ktiles = (g.B + Ktp - 1) / Ktp;
    d.T = g.table;
    d.shares = g.shares;
    d.nwin = (et ? (1u << m) : (1u << (m - 1))) / pl.W;
    m_max = std::max(m_max, m);
  }
  pl.smem_bytes = pl.xsm + fixed + tc_stack_bytes(m_max);
  gp.order.resize(G);
  for (uint32_t i = 0; i < G; ++i) gp.order[i] = i;
  std::stable_sort(gp.order.begin(), gp.order.end(),
                   [&](uint32_t a, uint32_t b) { return gp.desc[a].m > gp.desc[b].m; });
  uint64_t items = 0, keys = 0, blocks = 0;
  gp.front_bytes = 0;
  gp.keys_bytes = 0;
  for (uint32_t oi : gp.order) {
    dev::GroupDesc &d = gp.desc[oi];
    d.item_base = uint32_t(items);
    d.key_base = uint32_t(keys);
    const uint64_t it = uint64_t(d.n_ktiles) * ((d.F + pl.Ft - 1) / pl.Ft);
    items += it;
    keys += d.B;
    gp.front_bytes += 2 * align_up(size_t(d.B) * d.cap * 16, kAlign);
    uint64_t top = 0;
    for (uint32_t k = 0; k < d.n - d.m; ++k) top += ((d.nr1 - 1) >> (d.n - k)) - (d.nr0 >> (d.n - k)) + 1;
    const uint64_t per = ((1ull << d.m) - 1) + (et ? (1ull << d.m) : 0);
    blocks += uint64_t(d.B) * top + it * pl.tasks * per;
  }
  if (items > 0x7FFFFFFFull || keys > 0x7FFFFFFFull) return DPF_EINVAL;
  pl.n_items = uint32_t(items);
  pl.prf_blocks = blocks;
  pl.grid = pl.pair ? 2 * std::min<uint32_t>(pl.n_items, workers) : std::min<uint32_t>(pl.n_items, workers);
  gp.desc_bytes = align_up(size_t(G) * sizeof(dev::GroupDesc), kAlign);
  gp.total_bytes = gp.front_bytes + gp.keys_bytes + gp.desc_bytes;
  return DPF_OK;
}

thread_local Staging g_desc_staging;

}  // namespace
}  // namespace dpfpir

extern "C" size_t dpf_eval_grouped_workspace_bytes(const dpf_eval_group *groups, uint32_t n_groups, uint32_t D,
                                                   uint32_t prf) {
  GroupedPlan gp;
  if (make_grouped_plan(groups, n_groups, D, prf, gp) != DPF_OK) return 0;
  return gp.total_bytes;
}

extern "C" size_t dpf_eval_grouped_packed_workspace_bytes(const dpf_eval_group *groups, uint32_t n_groups,
                                                          uint32_t D, uint32_t prf) {
  GroupedPlan gp;
  if (make_grouped_plan(groups, n_groups, D, prf, gp, true) != DPF_OK) return 0;
  return gp.total_bytes;
}

namespace dpfpir {
namespace {
int eval_grouped_impl(const dpf_eval_group *groups, uint32_t n_groups, uint32_t D, uint32_t prf, void *workspace,
                      size_t workspace_bytes, void *stream, bool packed);
}
}  // namespace dpfpir

extern "C" int dpf_eval_grouped(const dpf_eval_group *groups, uint32_t n_groups, uint32_t D, uint32_t prf,
                                void *workspace, size_t workspace_bytes, void *stream) {
  return dpfpir::eval_grouped_impl(groups, n_groups, D, prf, workspace, workspace_bytes, stream, false);
}

extern "C" int dpf_eval_grouped_packed(const dpf_eval_group *groups, uint32_t n_groups, uint32_t D, uint32_t prf,
                                       void *workspace, size_t workspace_bytes, void *stream) {
  return dpfpir::eval_grouped_impl(groups, n_groups, D, prf, workspace, workspace_bytes, stream, true);
}

namespace dpfpir {
namespace {

int eval_grouped_impl(const dpf_eval_group *groups, uint32_t n_groups, uint32_t D, uint32_t prf, void *workspace,
                      size_t workspace_bytes, void *stream, bool packed) {
  if (prf != DPF_PRF_CHACHA20 && prf != DPF_PRF_AES128 && prf != DPF_PRF_CHACHA20_ET) return DPF_EUNSUPPORTED;
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & (kAlign - 1))) return DPF_EINVAL;
  GroupedPlan gp;
  int rc = make_grouped_plan(groups, n_groups, D, prf, gp, packed);
  if (rc) return rc;
  if (workspace_bytes < gp.total_bytes) return DPF_ENOMEM;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t *base = static_cast<uint8_t *>(workspace);
  uint8_t *front = base, *kbuf = base + gp.front_bytes, *dbuf = kbuf + gp.keys_bytes;
  // device-side keys: the caller's wire keys, in place (every PRF)
  size_t foff = 0;
  for (uint32_t oi : gp.order) {
    dev::GroupDesc &d = gp.desc[oi];
    const dpf_eval_group &g = groups[oi];
    d.frontier = reinterpret_cast<uint4 *>(front + foff);
    foff += align_up(size_t(d.B) * d.cap * 16, kAlign);
    d.frontier_alt = reinterpret_cast<uint4 *>(front + foff);
    foff += align_up(size_t(d.B) * d.cap * 16, kAlign);
    d.keys = g.keys_wire;
  }
  // descriptors in launch order (sorted by item_base) -> pinned staging -> device
  std::vector<dev::GroupDesc> sorted;
  sorted.reserve(n_groups);
  for (uint32_t oi : gp.order) sorted.push_back(gp.desc[oi]);
  Staging &sg = g_desc_staging;
  const int slot = sg.next;
  sg.next ^= 1;
  const size_t db = sorted.size() * sizeof(dev::GroupDesc);
  if (sg.done[slot]) cudaEventSynchronize(sg.done[slot]);
  if (sg.cap[slot] < db) {
    if (sg.buf[slot]) cudaFreeHost(sg.buf[slot]);
    sg.buf[slot] = nullptr;
    sg.cap[slot] = 0;
    if (cudaHostAlloc(&sg.buf[slot], db, cudaHostAllocDefault) != cudaSuccess) return DPF_ECUDA;
    sg.cap[slot] = db;
  }
  if (!sg.done[slot] && cudaEventCreateWithFlags(&sg.done[slot], cudaEventDisableTiming) != cudaSuccess)
    return DPF_ECUDA;
  std::memcpy(sg.buf[slot], sorted.data(), db);
  if (cudaMemcpyAsync(dbuf, sg.buf[slot], db, cudaMemcpyHostToDevice, st) != cudaSuccess) return DPF_ECUDA;
  if (cudaEventRecord(sg.done[slot], st) != cudaSuccess) return DPF_ECUDA;
  const dev::GroupDesc *ddesc = reinterpret_cast<const dev::GroupDesc *>(dbuf);
  uint32_t nk = 0;
  // a7 zeroing, a2 top BFS, then the fused kernel over all groups' items
  dev::zero_shares_grouped_kernel<<<dim3(64, std::min<uint32_t>(n_groups, 1024)), 256, 0, st>>>(ddesc, n_groups, D);
  uint64_t total_keys = 0;
  for (const auto &d : sorted) total_keys += d.B;
  if (prf == DPF_PRF_AES128) {
    if (!allow_dyn_smem(&dev::expand_top_grouped_kernel<dev::PrfAesTt>, dev::kAesSmemBytes)) return DPF_ECUDA;
    dev::expand_top_grouped_kernel<dev::PrfAesTt><<<uint32_t(total_keys), 256, dev::kAesSmemBytes, st>>>(ddesc,
                                                                                                         n_groups);
  } else
    dev::expand_top_grouped_kernel<dev::PrfChacha><<<uint32_t(total_keys), 256, 0, st>>>(ddesc, n_groups);
  nk += 2;
  uint32_t f_max = 0;
  for (const auto &d : sorted) f_max = std::max(f_max, d.n - d.m);
  for (uint32_t k = kTopSmemLevelsHost + 1; k <= f_max; ++k) {  // deeper frontiers: one launch per level
    const dim3 grid(148 * 4, n_groups);
    if (prf == DPF_PRF_AES128) {
      if (!allow_dyn_smem(&dev::expand_level_grouped_kernel<dev::PrfAesTt>, dev::kAesSmemBytes)) return DPF_ECUDA;
      dev::expand_level_grouped_kernel<dev::PrfAesTt><<<grid, 256, dev::kAesSmemBytes, st>>>(ddesc, k);
    } else
      dev::expand_level_grouped_kernel<dev::PrfChacha><<<grid, 256, 0, st>>>(ddesc, k);
    ++nk;
  }
  const Plan &pl = gp.cfg;
  dev::FusedParams p;
  std::memset(&p, 0, sizeof p);
  p.g0 = sorted[0];
  p.groups = ddesc;
  p.n_groups = n_groups;
  p.n_items = pl.n_items;
  p.D = D;
  p.Kt = pl.Kt;
  p.Kr = pl.Kr ? pl.Kr : pl.Kt;
  p.Ft = pl.Ft;
  p.tasks = pl.tasks;
  p.W = pl.W;
  p.R = pl.R;
  p.CG = pl.CG;
  p.KG = pl.KG;
  p.SG = pl.SG;
  p.y_stage_words = pl.y_stage_words;
  p.t_stage_words = pl.t_stage_words;
  p.CN = pl.CN;
  p.n_chunks = pl.n_chunks;
  p.NST = pl.NST;
  p.sys_red = 0;  // grouped answers are this device's buffers
  if (pl.tc) {
    if ((rc = launch_tc_kernel(pl, p, st)) != DPF_OK) return rc;
  } else {
    auto kfn = pl.kc.get(prf);
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem_bytes)) != cudaSuccess)
      return DPF_ECUDA;
    const bool timed = g_timer.on && 2 * g_timer.used + 1 < g_timer.ev.size();
    if (timed) cudaEventRecord(g_timer.ev[2 * g_timer.used], st);
    kfn<<<pl.grid, 32 * (pl.kc.NP + kNC + 1), pl.smem_bytes, st>>>(p);
    if (timed) cudaEventRecord(g_timer.ev[2 * g_timer.used++ + 1], st);
    if (cudaGetLastError() != cudaSuccess) return DPF_ECUDA;
  }
  ++nk;
  g_stats.prf_blocks = pl.prf_blocks;
  g_stats.kernels = nk;
  g_stats.frontier_depth = 0;
  g_stats.keys_per_tile = pl.pair ? 2 * pl.Kt : pl.Kt;
  g_stats.nodes_per_tile = pl.Ft;
  g_stats.work_items = pl.n_items;
  g_stats.grid = pl.grid;
  g_stats.kernel_id = kernel_id(pl);
  return DPF_OK;
}

}  // namespace
}  // namespace dpfpir

// ------------------------------------------------------------- PBR (row f2)
// Partial batch retrieval (reading R21): one group per bin of
// I = 2^log_i rows, every group a view of the table at row bI (row-major:
// + bI D words; packed: + bI/8 blocks of 32 Dp bytes, I >= 8 keeps bins on
// whole 8-row blocks), run through the grouped launch sequence.
namespace dpfpir {
namespace {

int make_pbr_groups(const uint8_t *keys, uint32_t B, uint32_t log_i, uint32_t prf, const void *table, int packed,
                    uint64_t N, uint32_t D, uint32_t *shares, std::vector<dpf_eval_group> &gs) {
  if (!keys || !table || !shares || B == 0 || N == 0 || D == 0 || log_i < 1 || log_i > DPF_MAX_LOG_N)
    return DPF_EINVAL;
  if (packed && log_i < 3) return DPF_EINVAL;
  const size_t ks = dpf_key_wire_size_prf(log_i, prf);
  if (ks == 0) return DPF_EINVAL;
  const uint64_t I = 1ull << log_i;
  const uint64_t nb = (N + I - 1) >> log_i;
  if (nb > (1ull << 20)) return DPF_EINVAL;
  const uint64_t Dp = (D + 127) & ~127u;
  gs.assign(nb, dpf_eval_group{});
  for (uint64_t b = 0; b < nb; ++b) {
    dpf_eval_group &g = gs[b];
    g.keys_wire = keys + b * B * ks;
    g.B = B;
    g.log_n = log_i;
    g.row_begin = 0;
    g.row_count = std::min<uint64_t>(I, N - b * I);
    g.table = packed ? reinterpret_cast<const uint32_t *>(static_cast<const uint8_t *>(table) + (b * I / 8) * 32 * Dp)
                     : static_cast<const uint32_t *>(table) + b * I * D;
    g.shares = shares + b * B * D;
  }
  return DPF_OK;
}

}  // namespace
}  // namespace dpfpir

extern "C" size_t dpf_eval_pbr_workspace_bytes(uint32_t B, uint32_t log_i, uint64_t N, uint32_t D, uint32_t prf,
                                               int packed) {
  // plan on placeholder (aligned, non-null) addresses: sizes depend only on shapes
  std::vector<dpf_eval_group> gs;
  const uintptr_t fake = 1u << 12;
  if (dpfpir::make_pbr_groups(reinterpret_cast<const uint8_t *>(fake), B, log_i, prf,
                              reinterpret_cast<const void *>(fake), packed, N, D, reinterpret_cast<uint32_t *>(fake),
                              gs) != DPF_OK)
    return 0;
  return packed ? dpf_eval_grouped_packed_workspace_bytes(gs.data(), uint32_t(gs.size()), D, prf)
                : dpf_eval_grouped_workspace_bytes(gs.data(), uint32_t(gs.size()), D, prf);
}

extern "C" int dpf_eval_pbr(const uint8_t *keys_wire, uint32_t B, uint32_t log_i, uint32_t prf, const void *table,
                            int packed, uint64_t N, uint32_t D, uint32_t *shares, void *workspace,
                            size_t workspace_bytes, void *stream) {
  std::vector<dpf_eval_group> gs;
  int rc = dpfpir::make_pbr_groups(keys_wire, B, log_i, prf, table, packed, N, D, shares, gs);
  if (rc != DPF_OK) return rc;
  return packed ? dpf_eval_grouped_packed(gs.data(), uint32_t(gs.size()), D, prf, workspace, workspace_bytes, stream)
                : dpf_eval_grouped(gs.data(), uint32_t(gs.size()), D, prf, workspace, workspace_bytes, stream);
}
