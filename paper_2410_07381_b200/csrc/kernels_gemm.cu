// Best-effort dense contractions on the 5th-generation tensor cores, in the
// three Tally launch shapes.
//
//   sgemm_tf32x3   C[M,N] (fp32) = A[M,K] . B[N,K]^T with fp32 accuracy via the
//                  error-compensated 3xTF32 split: A = Ahi + Alo, B = Bhi + Blo
//                  (hi = tf32-rounded, lo = exact fp32 remainder), and
//                  C = Ahi.Bhi + Ahi.Blo + Alo.Bhi accumulated in fp32 TMEM.
//                  Operands are pre-split by the `split_tf32` kind.
//   gemm_bf16      C[M,N] (bf16) = A[M,K] . B[N,K]^T, bf16 in, fp32 accumulate.
//   split_tf32     x -> (hi, lo), elementwise (HBM bound).
//
// One logical block = one BM x BN output tile (tile index t, grouped
// rasterisation over GROUP_M row-blocks for L2 reuse).  Every shape runs the
// same warp-specialised CTA:
//   warp 0      TMA producer: claims tiles (Original: blockIdx; Sliced:
//               offset + blockIdx; PTB: flag-gated L2 atomic), streams A/B
//               k-blocks into a STAGES-deep smem ring (mbarrier complete_tx)
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma into a
//               double-buffered TMEM accumulator, tcgen05.commit frees smem
//               stages and signals the epilogue
//   warps 2-5   epilogue: tcgen05.ld TMEM -> registers -> global C
// A two-slot tile ring in smem carries claimed tile ids from the producer to
// the other roles; id -1 ends the CTA.  In PTB shape a claimed tile is always
// finished, so a preempted worker retires within ~one tile.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "epilogue.cuh"
#include "registry.h"
#include "runtime.h"
#include "bnfuse.cuh"

namespace tally {

namespace gemm {

enum Mode { kOriginal = 0, kSliced = 1, kPtb = 2 };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

#ifndef TALLY_GEMM_OPERAND_EVICT_FIRST
#define TALLY_GEMM_OPERAND_EVICT_FIRST 1
#endif
// Operand tiles are loaded L2 evict-first too (see st_out16): tiles still
// reuse L2 within a wave (evict-first lines are only replaced under pressure,
// among themselves first) but do not displace a co-located request's lines.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
#if TALLY_GEMM_OPERAND_EVICT_FIRST
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(pol)
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
#endif
}

// Output tiles are written L2 evict-first (best-effort traffic must not push
// a co-located high-priority request's working set out of L2; see kernels_nn.cu)
__device__ __forceinline__ void st_out16(void* p, uint4 v) {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
}

// ---- CTA pair (cta_group::2) helpers -------------------------------------
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void* p, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// (relaxed: the arrival orders nothing but the reuse of a slot the waiter
// has already read, or -- for TMEM -- tcgen05.ld completion, which the
// tcgen05 fences order)
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 8-byte store into a peer CTA's shared memory that completes as 8
// transaction bytes on the peer's mbarrier (no fence on the sender)
__device__ __forceinline__ void st_async_s64(uint32_t cluster_addr, long long v, uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.s64 [%0], %1, [%2];" ::"r"(cluster_addr),
               "l"(v), "r"(cluster_bar)
               : "memory");
}
// Pair TMA load: both CTAs load their half into their own shared memory and
// signal the leader CTA's full barrier (`lead_bar`: its shared::cluster
// address), which expects both halves' bytes.
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t lead_bar, int x, int y) {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(lead_bar), "r"(x), "r"(y), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  // arrives on the barrier at this offset in both CTAs of the pair
  asm volatile(
      "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// TMA im2col load: a box of pixels x 64 channels of an NHWC tensor, starting
// at the output pixel whose input window origin is (w, h) of image n,
// shifted by the filter tap (off_w, off_h); out-of-image pixels read zero
__device__ __forceinline__ void tma_load_im2col(void* dst, const CUtensorMap* map, uint64_t* bar, int c, int w,
                                                int h, int n, int off_w, int off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"((unsigned short)off_w),
      "h"((unsigned short)off_h)
      : "memory");
}

__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// K-major operand tile, 128-byte swizzle, 8-row core groups 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;          // start address (16 B units)
  d |= 1ull << 16;                        // leading byte offset (unused for SW128 K-major)
  d |= (1024ull >> 4) << 32;              // stride byte offset: 8 rows x 128 B
  d |= 1ull << 46;                        // descriptor version (sm_100)
  d |= 2ull << 61;                        // SWIZZLE_128B
  return d;
}

template <int KIND>  // 0: tf32, 1: bf16 (kind::f16)
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (KIND == 0) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  } else {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  }
}

// MN-major operand tile (MN contiguous), 128-byte swizzle: 64-element-wide
// atoms of 8 K-rows x 128 B; K-row groups 1024 B apart (SBO), MN atoms
// 8192 B apart (LBO: one 64-wide TMA box of BK = 64 rows each).
__device__ __forceinline__ uint64_t smem_desc_mn(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;          // start address (16 B units)
  d |= (8192ull >> 4) << 16;              // leading byte offset: next 64-wide MN atom
  d |= (1024ull >> 4) << 32;              // stride byte offset: next 8 K-rows
  d |= 1ull << 46;                        // descriptor version (sm_100)
  d |= 2ull << 61;                        // SWIZZLE_128B
  return d;
}

// No-swizzle ("interleaved") operand tiles of the narrow-channel implicit
// convolutions (CONV 3 / 4: 8-channel NHWC input, one TMA im2col load per
// filter tap of 128 / 64 pixels x 16 B, written densely): core matrices of
// 8 rows x 16 B.  K-major A (forward): K-adjacent core matrices (the next
// tap) 2048 B apart (LBO), M-adjacent (next 8 pixels) 128 B (SBO).
// MN-major B (weight gradient): K-adjacent (next 8 pixels) 128 B apart
// (LBO), N-adjacent (next tap's 8 channels) 1024 B (SBO).
__device__ __forceinline__ uint64_t smem_desc_ns(const void* p, uint32_t lbo, uint32_t sbo) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;
  d |= (uint64_t)(lbo >> 4) << 16;
  d |= (uint64_t)(sbo >> 4) << 32;
  d |= 1ull << 46;                        // descriptor version (sm_100); layout 0 = SWIZZLE_NONE
  return d;
}

// Instruction descriptor: D fp32, A and B K-major (or both MN-major), M = 128
// (256 for a CTA pair), N = BN.
template <int KIND, int BN, bool A_MN = false, bool B_MN = false, int MMA_M = 128>
__host__ __device__ constexpr uint32_t make_idesc() {
  return (1u << 4)                                  // D format: F32
         | ((KIND == 0 ? 2u : 1u) << 7)             // A format: TF32 / BF16
         | ((KIND == 0 ? 2u : 1u) << 10)            // B format
         | ((A_MN ? 1u : 0u) << 15)                 // A major: MN
         | ((B_MN ? 1u : 0u) << 16)                 // B major: MN
         | ((uint32_t)(BN >> 3) << 17)              // N >> 3
         | ((uint32_t)(MMA_M >> 4) << 24);          // M >> 4
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// tcgen05.ld without the wait (the caller batches loads, then tmem_wait_ld)
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// TMA tensor store of a staged box (bf16 epilogue), L2 evict-first like every
// best-effort store; bulk-group completion tracked by the issuing thread
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int x, int y) {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;"
               ::"l"(map), "r"(x), "r"(y), "r"(src), "l"(pol)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// ---------------------------------------------------------------- configs
template <int BN_, int STAGES_>
struct CfgTf32x3T {
  static constexpr int KIND = 0;
  static constexpr int BM = 128, BN = BN_;
  static constexpr int BK = 32;                       // fp32 elements = 128 B (one swizzle atom)
  static constexpr int ESZ = 4;
  static constexpr int NOPS = 4;                      // Ahi, Alo, Bhi, Blo
  static constexpr int A_BYTES = BM * BK * ESZ;       // 16 KB
  static constexpr int B_BYTES = BN * BK * ESZ;       // 8 / 16 KB
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;   // 48 / 64 KB
  static constexpr int STAGES = STAGES_;
  static constexpr int UMMA_K = 8;
  static constexpr int TMEM_COLS = BN == 64 ? 256 : 512;   // 2 x BN accumulators + BN running total
  static constexpr bool A_MN = false, B_MN = false;
  static constexpr int EPI_BYTES = 0;   // fp32 rows are stored straight from registers
  using OutT = float;
};
// 128x128 tiles halve L2->SM operand bytes per flop (the kernel is L2-bound);
// chunk-granular preemption keeps the preemption latency independent of the tile
using CfgTf32x3 = CfgTf32x3T<128, 3>;
using CfgTf32x3N64 = CfgTf32x3T<64, 4>;

// bf16 operands, fp32 TMEM accumulation; BN = 128 or 64 (N % 128 != 0, e.g.
// 64-channel convolutions), output bf16 (activations) or fp32 (split-K
// weight-gradient partials, logits)
#ifndef TALLY_STAGES_BF16_N128
#define TALLY_STAGES_BF16_N128 2
#endif
#ifndef TALLY_STAGES_F32_N128
#define TALLY_STAGES_F32_N128 2   // (+ 32 KB of fp32 staging for the TMA-store epilogue, two CTAs per SM)
#endif
#ifndef TALLY_STAGES_BF16_N64
#define TALLY_STAGES_BF16_N64 3
#endif
#ifndef TALLY_STAGES_F32_N64
#define TALLY_STAGES_F32_N64 4
#endif
// PAIR = 2: a CTA pair (cluster of two SMs, cta_group::2) computes one
// 256 x BN tile with M = 256 MMAs -- each CTA loads its 128 rows of A and
// BN / 2 rows of B, the leader's elected thread issues for both, each CTA's
// TMEM holds its 128 rows; per SM half the operand bytes of a 128-row tile.
#ifndef TALLY_STAGES_PAIR
#define TALLY_STAGES_PAIR 6
#endif
template <int BN_, class OutT_, bool A_MN_ = false, bool B_MN_ = false, int PAIR_ = 1, int CONV_ = 0>
struct CfgBf16T {
  static constexpr int KIND = 1;
  static constexpr int PAIR = PAIR_;
  // implicit-GEMM convolution: 1 = A by TMA im2col (forward), 2 = B by TMA im2col (weight gradient)
  static constexpr int CONV = CONV_;
  static constexpr int BM = 128, BN = BN_;            // BM: rows per CTA; BN: MMA N (the pair's tile width)
  static constexpr int B_ROWS = BN / PAIR;            // B rows (N) this CTA loads
  static constexpr int BK = 64;                       // bf16 elements = 128 B
  static constexpr int ESZ = 2;
  static constexpr int NOPS = 2;
  static constexpr int A_BYTES = BM * BK * ESZ;       // 16 KB
  static constexpr int B_BYTES = B_ROWS * BK * ESZ;   // 16 / 8 KB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // 64-96 KB of operand ring (+ bf16 staging): two CTAs per SM, so an
  // untransformed launch (one output tile per CTA) overlaps one CTA's
  // prologue / pipeline fill with the other's tile, and high-priority CTAs
  // find room next to a best-effort one.  Pairs: one CTA per SM, a deep ring.
  static constexpr int STAGES = PAIR == 2 ? TALLY_STAGES_PAIR
                              : BN == 128 ? (sizeof(OutT_) == 2 ? TALLY_STAGES_BF16_N128 : TALLY_STAGES_F32_N128)
                                          : (sizeof(OutT_) == 2 ? TALLY_STAGES_BF16_N64 : TALLY_STAGES_F32_N64);
  static constexpr int UMMA_K = 16;
  // the whole (split) K range accumulates in one TMEM buffer (no fp32
  // promotion chunks at the 1e-2 bf16 budget): 2 x BN columns, leaving TMEM
  // for co-resident high-priority tensor-core kernels (pairs: all 512)
  static constexpr int TMEM_COLS = 2 * BN;
  // MN-major operands: A given as A^T [K, M] and/or B as B^T [K, N] (M / N
  // contiguous) -- the weight gradient dW = dY^T . X reads both activations
  // as stored (no transposes); P . V and dY . W read V / W as stored
  static constexpr bool A_MN = A_MN_, B_MN = B_MN_;
  using OutT = OutT_;
  // bf16 output: each epilogue warp stages 32 rows x 64 columns at a time in
  // shared memory (XOR-swizzled 16 B chunks) and writes whole row segments
  // fp32 output (128/256-wide tiles): each warp stages 32 rows x 32 columns
  // (4 KB) for a TMA tensor store -- the per-lane row stores of fp32 tiles
  // were L1/LSU-bound (ncu: attention score GEMM at 1.6 TB/s of DRAM, L1 61 %)
  static constexpr int EPI_BYTES = (sizeof(OutT_) == 2 || BN_ >= 128) ? 8 * 32 * 64 * 2 : 0;   // 4 KB per epilogue warp
};
using CfgBf16 = CfgBf16T<128, __nv_bfloat16>;
using CfgBf16N64 = CfgBf16T<64, __nv_bfloat16>;
using CfgBf16F32 = CfgBf16T<128, float>;
using CfgBf16F32N64 = CfgBf16T<64, float>;
using CfgBf16MN = CfgBf16T<128, float, true, true>;
using CfgBf16MNN64 = CfgBf16T<64, float, true, true>;
using CfgBf16KMN = CfgBf16T<128, __nv_bfloat16, false, true>;
using CfgBf16KMNN64 = CfgBf16T<64, __nv_bfloat16, false, true>;
using CfgBf16F32KMN = CfgBf16T<128, float, false, true>;
using CfgBf16F32KMNN64 = CfgBf16T<64, float, false, true>;
using CfgBf16MNb = CfgBf16T<128, __nv_bfloat16, true, true>;
using CfgBf16MNbN64 = CfgBf16T<64, __nv_bfloat16, true, true>;
// CTA-pair kinds (256 x 256 tiles)
using CfgBf16X2 = CfgBf16T<256, __nv_bfloat16, false, false, 2>;
using CfgBf16F32X2 = CfgBf16T<256, float, false, false, 2>;
using CfgBf16MNX2 = CfgBf16T<256, float, true, true, 2>;
using CfgBf16KMNX2 = CfgBf16T<256, __nv_bfloat16, false, true, 2>;
using CfgBf16F32KMNX2 = CfgBf16T<256, float, false, true, 2>;
// implicit-GEMM convolution kinds (A / B operand gathered by TMA im2col)
using CfgConvF = CfgBf16T<128, __nv_bfloat16, false, false, 1, 1>;
using CfgConvFN64 = CfgBf16T<64, __nv_bfloat16, false, false, 1, 1>;
using CfgConvF32 = CfgBf16T<128, float, false, false, 1, 1>;
using CfgConvF32N64 = CfgBf16T<64, float, false, false, 1, 1>;
using CfgConvW = CfgBf16T<128, float, true, true, 1, 2>;
using CfgConvWN64 = CfgBf16T<64, float, true, true, 1, 2>;
// 8-channel input (the ResNet stem's 3 channels padded to 8): a k-block is 8
// filter taps x 8 channels, one 16-byte-wide im2col load per tap, no swizzle
using CfgConvFC8 = CfgBf16T<64, __nv_bfloat16, false, false, 1, 3>;
using CfgConvWC8 = CfgBf16T<64, float, true, true, 1, 4>;
template <class Cfg, class = void>
struct ConvOf { static constexpr int value = 0; };
template <class Cfg>
struct ConvOf<Cfg, void_t_<decltype(Cfg::CONV)>> { static constexpr int value = Cfg::CONV; };
template <class Cfg, class = void>
struct PairOf { static constexpr int value = 1; };
template <class Cfg>
struct PairOf<Cfg, void_t_<decltype(Cfg::PAIR)>> { static constexpr int value = Cfg::PAIR; };

constexpr int GROUP_M = 8;
// producer warp, MMA warp, 8 epilogue warps: two per TMEM lane quarter, each
// draining half of the tile's columns (the epilogue bounds short-K tiles)
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
// claimed-tile ring depth: the producer runs up to kSlots tiles ahead of the
// epilogue (short-K tiles are load-latency bound otherwise)
constexpr int kSlots = 4;

template <class Cfg>
constexpr size_t smem_bytes() {
  return 1024 /*alignment slack*/ + (size_t)Cfg::STAGES * Cfg::STAGE_BYTES + Cfg::EPI_BYTES +
         640 /*barriers + rings*/;
}

struct alignas(64) GemmParams {
  CUtensorMap a_hi, a_lo, b_hi, b_lo;   // lo maps unused for bf16
  void* c;
  int m, n, k;
  int tiles_m, tiles_n;
  int kchunk;   // k-blocks per TMEM accumulation chunk (promotion to fp32 registers)
  unsigned long long* resume;   // chunk-preemption resume ring (sgemm_tf32x3), see tally_device.cuh
  long long ldc;                // row stride of C (elements)
  long long split_stride;       // elements between split-K partial outputs
  int splits;                   // split-K factor: logical block = (split, tile)
  int kb_per_split;             // k-blocks per split
  int tpb;                      // tiles per logical block
  long long total_tiles;        // tiles * splits * batches
  int batches, hdiv;            // batched layout (tally_gemm_layout): z = (zb, zh)
  int c_tma;                    // bf16 C stored by TMA through the map in a_lo (plain, unbatched GEMMs)
  int causal;                   // causal-attention tile / K-range rule (tile_work), 0 = dense
  int bn, bk;                   // tile width and K block of the kind (for the causal rule)
  long long off[6][2];          // (row, col) origins of A, B, C: [a_row, a_col, b_row, b_col, c_row, c_col]
  // fused linear-layer epilogue (TMA-store bf16 path): y = act(acc + bias (+ res));
  // ep_pre: the pre-activation is also stored, through the map in b_lo
  EpArgs ep;
  int ep_pre;
  // implicit-GEMM convolution (CONV kinds): the im2col map is a_hi (forward)
  // or b_hi (weight gradient); output pixels o = (n, p, q) with hw = ho * wo
  int cv_c, cv_k, cv_cblocks, cv_stride, cv_pad, cv_wo, cv_hw, cv_n;
  // fused batch-norm statistics of the bf16 output (bnfuse.cuh; part null: off)
  BnFuse bnf;
};

__device__ __forceinline__ void tile_coords(unsigned t, const GemmParams& p, int& mb, int& nb) {
  // grouped rasterisation: GROUP_M row-blocks share each column sweep
  const unsigned per_group = GROUP_M * (unsigned)p.tiles_n;
  const unsigned g = t / per_group;
  const int first_m = (int)g * GROUP_M;
  const unsigned gm = (unsigned)min(p.tiles_m - first_m, GROUP_M);
  const unsigned r = t - g * per_group;
  const unsigned nq = r / gm;
  mb = first_m + (int)(r - nq * gm);
  nb = (int)nq;
}

// Logical block t -> (output tile, K range, batch).  With split-K the block
// index is split-major: t = split * tiles + tile; split s covers k-blocks
// [s * kb_per_split, min(KB, (s + 1) * kb_per_split)).  The producer warp
// computes it once per tile (32-bit divisions; total_tiles < 2^31 is checked
// at bind time) and publishes it to the MMA and epilogue warps in shared
// memory: recomputing it per warp with 64-bit divisions was ~35 % of the
// stall samples of short-K tiles (ncu, K = 64 dgrad).
struct TileWork {
  int mb, nb, split, kbeg, kend, nch, zb, zh;
};
__device__ __forceinline__ int Cfg_BN(const GemmParams& p) { return p.bn; }
__device__ __forceinline__ TileWork tile_work(long long t_, const GemmParams& p, int KB) {
  TileWork w;
  const unsigned tiles = (unsigned)p.tiles_m * (unsigned)p.tiles_n;
  const unsigned per_batch = tiles * (unsigned)p.splits;
  unsigned t = (unsigned)t_;
  const unsigned z = t / per_batch;
  t -= z * per_batch;
  const unsigned split = t / tiles;
  w.split = (int)split;
  tile_coords(t - split * tiles, p, w.mb, w.nb);
  w.kbeg = w.split * p.kb_per_split;
  w.kend = min(KB, w.kbeg + p.kb_per_split);
  // causal attention (T x T blocks of one (sequence, head)): 1 = scores
  // S = Q K^T / dP = dO V^T -- tiles wholly above the diagonal are skipped
  // (nch = 0: no loads, no MMA, no store; softmax reads only j <= i);
  // 2 = P V / dS K -- K (the key index) stops at the tile's last query row;
  // 3 = dS^T Q / P^T dO -- K (the query index) starts at the tile's first key
  if (p.causal == 1 && w.nb * Cfg_BN(p) >= (w.mb + 1) * 128) w.kend = w.kbeg;
  if (p.causal == 2) w.kend = min(w.kend, ((w.mb + 1) * 128 + p.bk - 1) / p.bk);
  if (p.causal == 3) w.kbeg = max(w.kbeg, (w.mb * 128) / p.bk);
  w.nch = w.kend <= w.kbeg ? 0 : p.kchunk == p.kb_per_split ? 1 : (w.kend - w.kbeg + p.kchunk - 1) / p.kchunk;
  w.zb = (int)(z / (unsigned)p.hdiv);
  w.zh = (int)(z - (unsigned)w.zb * (unsigned)p.hdiv);
  return w;
}

// origin offset (elements) of operand coordinate `which` for batch (zb, zh)
__device__ __forceinline__ int goff(const GemmParams& p, int which, const TileWork& w) {
  return (int)(p.off[which][0] * w.zb + p.off[which][1] * w.zh);
}

__device__ __forceinline__ unsigned long long* block_log_of(const SliceArgs& a) { return a.block_log; }
__device__ __forceinline__ unsigned long long* block_log_of(const PtbArgs& a) { return a.block_log; }
// Per-logical-block device events (ref sim.py:156-172 BlockStarted /
// BlockFinished): start = the block's first MMA issued, end = its last tile's
// output issued by epilogue warp 2; (worker << 32 | smid).  Leader CTA only.
__device__ __forceinline__ void gemm_log_end(unsigned long long* log, long long t, const GemmParams& p) {
  if (log != nullptr && (t % p.tpb == p.tpb - 1 || t == p.total_tiles - 1)) {
    const long long b = t / p.tpb;
    log[3 * b + 1] = globaltimer();
    log[3 * b + 2] = ((unsigned long long)blockIdx.x << 32) | smid();
  }
}
__device__ __forceinline__ const unsigned long long* ret_ring_of(const SliceArgs&) { return nullptr; }
__device__ __forceinline__ unsigned long long ret_pending_of(const SliceArgs&) { return 0ull; }
__device__ __forceinline__ const unsigned long long* ret_ring_of(const PtbArgs& a) { return a.ret_ring; }
__device__ __forceinline__ unsigned long long ret_pending_of(const PtbArgs& a) { return a.ret_pending; }

// An epilogue warp hands a drained TMEM accumulator back to the MMA issuer
// (pair: to the leader CTA's barrier, which counts both CTAs' warps).
template <int PR>
__device__ __forceinline__ void release_acc(uint64_t* bar) {
  if constexpr (PR == 2) mbar_arrive_remote_relaxed(map_rank(bar, 0));   // after tcgen05.wait::ld + fence
  else mbar_arrive(bar);
}

template <class Cfg, int MODE, class ShapeArgs>
__global__ void __launch_bounds__(kThreads, (Cfg::KIND == 1 && PairOf<Cfg>::value == 1) ? 2 : 1)
k_gemm(const __grid_constant__ GemmParams p, const ShapeArgs s) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* epi_smem = smem + (size_t)Cfg::STAGES * Cfg::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + Cfg::EPI_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tmem_full = empty + Cfg::STAGES;    // [2]
  uint64_t* tmem_empty = tmem_full + 2;         // [2]
  uint64_t* tile_full = tmem_empty + 2;         // [kSlots]
  uint64_t* tile_empty = tile_full + kSlots;    // [kSlots]
  long long* tile_slot = reinterpret_cast<long long*>(tile_empty + kSlots);   // claimed tile id
  int* tile_c0 = reinterpret_cast<int*>(tile_slot + kSlots);                  // first chunk (resumed tiles)
  int* tile_cut = tile_c0 + kSlots;                                           // chunk the tile stops before
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tile_cut + kSlots);
  TileWork* tile_w = reinterpret_cast<TileWork*>(tmem_base_slot + 4);          // [kSlots], producer-computed
  // CTA pair: the leader's producer forwards every tile it takes to the peer's
  // producer through pair_slot (peer smem) + pair_full (peer) / pair_empty (leader)
  uint64_t* pair_full = reinterpret_cast<uint64_t*>(tile_w + kSlots);          // [kSlots]
  uint64_t* pair_empty = pair_full + kSlots;                                  // [kSlots]
  long long* pair_slot = reinterpret_cast<long long*>(pair_empty + kSlots);   // [kSlots]

  constexpr int PR = PairOf<Cfg>::value;
  constexpr int BROWS = Cfg::BN / PR;   // rows of B this CTA loads
  const unsigned rank = PR == 2 ? cluster_rank() : 0u;
  const bool lead = rank == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = (p.k + Cfg::BK - 1) / Cfg::BK;

  unsigned long long t_entry = 0;
  if (threadIdx.x == 0) {
    t_entry = globaltimer();
    for (int i = 0; i < Cfg::STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      // (pair: the leader's barrier counts both CTAs' epilogue warps)
      mbar_init(&tmem_empty[i], (Cfg::KIND == 1 && Cfg::BN == 64) ? kEpiWarps / 2 : kEpiWarps * PR);   // one group per tile
    }
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&tile_full[i], 1);
      mbar_init(&tile_empty[i], kEpiWarps + (lead ? 1 : 0));   // (the peer has no MMA issuer)
      mbar_init(&pair_full[i], 1);
      mbar_init(&pair_empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (PR == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_slot)),
                   "n"(Cfg::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_slot)),
                   "n"(Cfg::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  fence_before();
  if constexpr (PR == 2) cluster_sync_all();   // both CTAs' barriers initialised before any remote arrive
  else __syncthreads();
  fence_after();
  // (programmatic dependent launch: the prologue above overlapped the predecessor's tail)
  pdl_launch_dependents();
  pdl_wait();
  const uint32_t tmem_base = *tmem_base_slot;
  bool stopped = false;
  unsigned long long blocks_run = 0;   // logical blocks this worker ran (PTB telemetry / retirement)
  // chunk-granular preemption (fp32-output kernels in PTB shape with a resume
  // ring): a preempted worker stops its tile at the next chunk boundary,
  // saves the fp32 running total into its C tile and queues (tile, chunk)
  constexpr bool kChunkPreempt = (MODE == kPtb) && (Cfg::KIND == 0);

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      // descriptor fetch off the critical path of the first tile
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.a_hi) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.b_hi) : "memory");
      if constexpr (Cfg::KIND == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&p.a_lo) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&p.b_lo) : "memory");
      }
      uint32_t it = 0;
      unsigned flag_seen = 0;
      // a logical block covers tiles [b * tpb, b * tpb + tpb) of the tile
      // sequence (tpb > 1 for short-K GEMMs, whose one-tile CTAs are
      // prologue / pipeline-fill bound)
      long long q_next = 0, q_end = 0;
      // bf16 kinds in PTB shape (claim-ahead worker, see the branch below)
      long long pre = -1;          // the next logical block, claimed while this one runs
      bool first_block = true;
      bool try_pop = MODE == kPtb && ret_ring_of(s) != nullptr && ret_pending_of(s) > 0;
      for (int i = 0;; ++i) {
        long long t = -1;
        int c0 = 0;
        if (MODE == kPtb && PR == 2 && !lead) {
          // the peer takes the leader's tiles (-2: the leader was stopped by the flag)
          const int jj = i % kSlots;
          mbar_expect_tx(&pair_full[jj], 8);
          mbar_wait(&pair_full[jj], (i / kSlots) & 1);
          t = *reinterpret_cast<volatile long long*>(&pair_slot[jj]);
          mbar_arrive_remote_relaxed(map_rank(&pair_empty[jj], 0));
          if (t == -2) { stopped = true; t = -1; }
          if (i == 0) *reinterpret_cast<volatile unsigned long long*>(tmem_base_slot + 2) = globaltimer();
        } else if constexpr (MODE == kPtb && Cfg::KIND == 1) {
          // Claim-ahead worker (bf16 kinds).  The first block is static
          // (worker w < static_n runs start + w, no claim round trip); the
          // claim for block b+1 is issued when block b starts, so its L2 round
          // trip overlaps b's tiles; at the b -> b+1 boundary the flag (loaded
          // when b's last tile was published) decides: raised -> b+1 is handed
          // back through the instance's return ring unrun (bounded retirement:
          // one logical block after the flag), else it runs.  A chain's next
          // launch pops handed-back blocks first.
          if (q_next < q_end) {
            t = q_next++;   // the rest of the current logical block
          } else {
            long long b = -1;
            if (first_block) {
              first_block = false;
              ptb_hold_while_paused(s);
              const unsigned f = s.flag_is_host ? ld_acquire_sys(s.flag) : ld_acquire_gpu(s.flag);
              const unsigned w = blockIdx.x / PR;
              if (ptb_park_requested(s, f)) {
                if (w < s.static_n) ptb_return(s, (long long)(s.start + w));
                stopped = true;
              } else if (try_pop) {
                int cnt = 1;
                b = ptb_pop_range(s, cnt);
                if (b >= 0 && cnt > 1) ptb_return_range(s, b + 1, cnt - 1);   // (GEMM workers take one)
                if (b < 0) { try_pop = false; b = ptb_claim_gated(s); }
              } else {
                b = w < s.static_n ? (long long)(s.start + w) : ptb_claim_gated(s);
              }
            } else if (ptb_park_requested(s, flag_seen)) {
              if (pre >= 0 && (unsigned long long)pre < s.total) ptb_return(s, pre);
              stopped = true;
            } else {
              b = pre;
            }
            if (b >= 0 && (unsigned long long)b < s.total) {
              ++blocks_run;
              if (s.exec_count != nullptr) atomicAdd(&s.exec_count[b], 1ull);
              // claim ahead (nothing left to claim once the static blocks cover the kernel)
              if (s.start + s.static_n >= s.total && !try_pop) {
                pre = (long long)s.total;
              } else if (try_pop) {
                int cnt = 1;
                pre = ptb_pop_range(s, cnt);
                if (pre >= 0 && cnt > 1) ptb_return_range(s, pre + 1, cnt - 1);
                if (pre < 0) { try_pop = false; pre = ptb_claim_gated(s); }
              } else {
                pre = ptb_claim_gated(s);
              }
              q_next = b * p.tpb;
              q_end = min((long long)p.total_tiles, q_next + p.tpb);
              t = q_next++;
            }
          }
        } else if constexpr (MODE == kPtb) {
          bool popped = false;
          if (kChunkPreempt && p.resume != nullptr) {
            // resume a tile a preempted worker left half-done
            ptb_hold_while_paused(s);
            const unsigned f = s.flag_is_host ? ld_acquire_sys(s.flag) : ld_acquire_gpu(s.flag);
            if (!ptb_park_requested(s, f)) {
              unsigned long long* ring = p.resume;
              for (;;) {
                const unsigned long long h = atomicAdd(ring + 1, 0ull), tl = atomicAdd(ring, 0ull);
                if (h >= tl) break;
                if (atomicCAS(ring + 1, h, h + 1) != h) continue;
                volatile unsigned long long* e = ring + 2 + (h % kResumeCap);
                unsigned long long v;
                while ((v = *e) == 0ull) __nanosleep(64);
                *e = 0ull;
                t = (long long)(v & 0xFFFFFFFFFFull) - 1;
                c0 = (int)(v >> 40);
                popped = true;
                break;
              }
            }
          }
          if (!popped) {
            if (q_next < q_end) {
              t = q_next++;   // the rest of a claimed logical block: always executed
            } else {
              const long long b = ptb_claim(s);
              if (b < 0) {
                stopped = true;
              } else if ((unsigned long long)b < s.total) {
                q_next = b * p.tpb;
                q_end = min((long long)p.total_tiles, q_next + p.tpb);
                t = q_next++;
              }
            }
          }
        } else {
          if (i == 0) {
            const unsigned bx = blockIdx.x / PR;   // pair: one logical block per cluster
            const long long b = MODE == kOriginal ? (long long)bx
                : (s.linear ? (long long)(s.linear_offset + bx) : (long long)(s.offset.x + bx));
            if (s.exec_count != nullptr && lead) atomicAdd(&s.exec_count[b], 1ull);
            q_next = b * p.tpb;
            q_end = min((long long)p.total_tiles, q_next + p.tpb);
          }
          if (q_next < q_end) t = q_next++;
        }
        if constexpr (MODE == kPtb && PR == 2) {
          if (lead) {   // forward to the peer's producer
            const int jj = i % kSlots;
            if (i >= kSlots) mbar_wait_cluster(&pair_empty[jj], ((i / kSlots) - 1) & 1);
            st_async_s64(map_rank(&pair_slot[jj], 1), (t < 0 && stopped) ? -2ll : t, map_rank(&pair_full[jj], 1));
          }
        }
        if constexpr (MODE == kPtb && Cfg::KIND == 1) {
          // the last tile of a block: load the flag now, read it at the boundary
          if (t >= 0 && q_next >= q_end && lead)
            flag_seen = s.flag_is_host ? ld_relaxed_sys(s.flag) : ld_relaxed_gpu(s.flag);
        }
        const int j = i % kSlots;
        if (i >= kSlots) mbar_wait(&tile_empty[j], ((i / kSlots) - 1) & 1);
        tile_slot[j] = t;
        tile_c0[j] = c0;
        const TileWork w = tile_work(t < 0 ? 0 : t, p, KB);
        tile_w[j] = w;
        tile_cut[j] = w.nch;
        mbar_arrive(&tile_full[j]);
        if (t < 0) break;
        const int mb = w.mb, nb = w.nb;
        for (int c = c0; c < w.nch; ++c) {
          if constexpr (kChunkPreempt) {
            // flag_seen was loaded three k-blocks ago; the L2 load has completed
            if (p.resume != nullptr && c > c0) {
              if (ptb_park_requested(s, flag_seen)) {
                // cut the tile before chunk c: publish the cut, then wake the
                // MMA issuer with an empty ("poisoned") stage
                *reinterpret_cast<volatile int*>(&tile_cut[j]) = c;
                const int st = it % Cfg::STAGES;
                if (it >= (uint32_t)Cfg::STAGES) mbar_wait(&empty[st], ((it / Cfg::STAGES) - 1) & 1);
                mbar_arrive(&full[st]);
                ++it;
                break;
              }
            }
          }
          const int kb1 = min(w.kend, w.kbeg + (c + 1) * p.kchunk);
          for (int kb = w.kbeg + c * p.kchunk; kb < kb1; ++kb, ++it) {
            const int st = it % Cfg::STAGES;
            if constexpr (MODE == kPtb) {
              // suspension point between k-blocks (cooperative suspension option)
              if ((kb & 3) == 0 && ptb_hold_while_paused(s)) {}
              if (kChunkPreempt && p.resume != nullptr && kb == max(w.kbeg + c * p.kchunk, kb1 - 3))
                flag_seen = s.flag_is_host ? ld_relaxed_sys(s.flag) : ld_relaxed_gpu(s.flag);
            }
            if (it >= (uint32_t)Cfg::STAGES) mbar_wait(&empty[st], ((it / Cfg::STAGES) - 1) & 1);
            unsigned char* base = smem + (size_t)st * Cfg::STAGE_BYTES;
            // pair: the leader's barrier expects both CTAs' halves
            if (lead) mbar_expect_tx(&full[st], Cfg::STAGE_BYTES * PR);
            const int kx = kb * Cfg::BK;
            if constexpr (Cfg::KIND == 0) {
              tma_load_2d(base, &p.a_hi, &full[st], kx, mb * Cfg::BM);
              tma_load_2d(base + Cfg::A_BYTES, &p.a_lo, &full[st], kx, mb * Cfg::BM);
              tma_load_2d(base + 2 * Cfg::A_BYTES, &p.b_hi, &full[st], kx, nb * Cfg::BN);
              tma_load_2d(base + 2 * Cfg::A_BYTES + Cfg::B_BYTES, &p.b_lo, &full[st], kx, nb * Cfg::BN);
            } else {
              // (batched layouts: every operand's origin moves with the batch)
              const int ar = goff(p, 0, w), ac = goff(p, 1, w), br = goff(p, 2, w), bc = goff(p, 3, w);
              // this CTA's rows of A and of B (pair: rank-th half of each)
              const int am = (mb * PR + (int)rank) * Cfg::BM, bn0 = nb * Cfg::BN + (int)rank * BROWS;
              const uint32_t lead_full = PR == 2 ? map_rank(&full[st], 0) : 0u;
              auto ld = [&](void* dst, const CUtensorMap* map, int x, int y) {
                if constexpr (PR == 2) tma_load_2d_pair(dst, map, lead_full, x, y);
                else tma_load_2d(dst, map, &full[st], x, y);
              };
              if constexpr (ConvOf<Cfg>::value == 1) {
                // A = im2col(x): 128 output pixels from am, k-block = (tap, 64 channels)
                const int tap = kb / p.cv_cblocks, cb = kb - tap * p.cv_cblocks;
                const int r = tap / p.cv_k, sx = tap - r * p.cv_k;
                const int n0 = am / p.cv_hw, rem = am - n0 * p.cv_hw, p0 = rem / p.cv_wo, q0 = rem - p0 * p.cv_wo;
                tma_load_im2col(base, &p.a_hi, &full[st], cb * 64, q0 * p.cv_stride - p.cv_pad,
                                p0 * p.cv_stride - p.cv_pad, n0, sx, r);
              } else if constexpr (ConvOf<Cfg>::value == 3) {
                // A = im2col(x), 8 channels: one 128-pixel x 16 B load per
                // tap of the k-block (taps past k*k: an image index past the
                // batch -- zeros)
                const int n0 = am / p.cv_hw, rem = am - n0 * p.cv_hw, p0 = rem / p.cv_wo, q0 = rem - p0 * p.cv_wo;
#pragma unroll 1
                for (int t = 0; t < 8; ++t) {
                  const int tap = kb * 8 + t, ok = tap < p.cv_k * p.cv_k;
                  const int r = ok ? tap / p.cv_k : 0, sx = ok ? tap - r * p.cv_k : 0;
                  tma_load_im2col(base + t * 2048, &p.a_hi, &full[st], 0, q0 * p.cv_stride - p.cv_pad,
                                  p0 * p.cv_stride - p.cv_pad, ok ? n0 : p.cv_n, sx, r);
                }
              } else if constexpr (Cfg::A_MN) {
                // boxes of 64 M-elements x BK K-rows, 8 KB each
#pragma unroll
                for (int h = 0; h < Cfg::BM / 64; ++h)
                  ld(base + h * 8192, &p.a_hi, am + h * 64 + ac, kb * Cfg::BK + ar);
              } else {
                ld(base, &p.a_hi, kx + ac, am + ar);
              }
              if constexpr (ConvOf<Cfg>::value == 2) {
                // B = im2col(x) MN-major: K = BK output pixels from kb * BK, N = (tap, channel)
                const int px = kb * Cfg::BK;
                const int n0 = px / p.cv_hw, rem = px - n0 * p.cv_hw, p0 = rem / p.cv_wo, q0 = rem - p0 * p.cv_wo;
#pragma unroll
                for (int h = 0; h < BROWS / 64; ++h) {
                  const int col = bn0 + h * 64, tap = col / p.cv_c, ch = col - tap * p.cv_c;
                  const int r = tap / p.cv_k, sx = tap - r * p.cv_k;
                  tma_load_im2col(base + Cfg::A_BYTES + h * 8192, &p.b_hi, &full[st], ch, q0 * p.cv_stride - p.cv_pad,
                                  p0 * p.cv_stride - p.cv_pad, n0, sx, r);
                }
              } else if constexpr (ConvOf<Cfg>::value == 4) {
                // B = im2col(x) MN-major, 8 channels: N = (tap, channel), one
                // 64-pixel x 16 B load per tap of this 64-wide N tile
                const int px = kb * Cfg::BK;
                const int n0 = px / p.cv_hw, rem = px - n0 * p.cv_hw, p0 = rem / p.cv_wo, q0 = rem - p0 * p.cv_wo;
#pragma unroll 1
                for (int t = 0; t < 8; ++t) {
                  const int tap = bn0 / 8 + t, ok = tap < p.cv_k * p.cv_k;
                  const int r = ok ? tap / p.cv_k : 0, sx = ok ? tap - r * p.cv_k : 0;
                  tma_load_im2col(base + Cfg::A_BYTES + t * 1024, &p.b_hi, &full[st], 0, q0 * p.cv_stride - p.cv_pad,
                                  p0 * p.cv_stride - p.cv_pad, ok ? n0 : p.cv_n, sx, r);
                }
              } else if constexpr (Cfg::B_MN) {
#pragma unroll
                for (int h = 0; h < BROWS / 64; ++h)
                  ld(base + Cfg::A_BYTES + h * 8192, &p.b_hi, bn0 + h * 64 + bc, kb * Cfg::BK + br);
              } else {
                ld(base + Cfg::A_BYTES, &p.b_hi, kx + bc, bn0 + br);
              }
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && lead) {
      // ------------------------------------------------ MMA issuer (pair: the leader, for both CTAs)
      // The tile's K range is cut into chunks of p.kchunk k-blocks; each chunk
      // accumulates into one of two TMEM buffers and is promoted to an fp32
      // running total by the epilogue (bounded tensor-core accumulation chains).
      constexpr uint32_t idesc = make_idesc<Cfg::KIND, Cfg::BN, Cfg::A_MN, Cfg::B_MN, 128 * PR>();
      uint32_t it = 0, ci = 0;
      for (int i = 0;; ++i) {
        const int j = i % kSlots;
        mbar_wait(&tile_full[j], (i / kSlots) & 1);
        const long long t = tile_slot[j];
        const int c0 = tile_c0[j];
        if (t < 0) {
          mbar_arrive(&tile_empty[j]);
          break;
        }
        const TileWork w = tile_w[j];
        if (i == 0 && MODE == kPtb)   // telemetry: first tile in hand (worker_log)
          *reinterpret_cast<volatile unsigned long long*>(tmem_base_slot + 2) = globaltimer();
        if (block_log_of(s) != nullptr && t % p.tpb == 0) block_log_of(s)[3 * (t / p.tpb)] = globaltimer();
        for (int c = c0; c < w.nch; ++c, ++ci) {
          const int acc = ci & 1;
          if (ci >= 2) {
            // (pair: the peer's epilogue warps arrive from the other CTA)
            if constexpr (PR == 2) mbar_wait_cluster(&tmem_empty[acc], ((ci >> 1) - 1) & 1);
            else mbar_wait(&tmem_empty[acc], ((ci >> 1) - 1) & 1);
          }
          fence_after();
          const uint32_t d = tmem_base + (uint32_t)(acc * Cfg::BN);
          const int kb0 = w.kbeg + c * p.kchunk, kb1 = min(w.kend, kb0 + p.kchunk);
          bool cut = false;
          for (int kb = kb0; kb < kb1; ++kb, ++it) {
            const int st = it % Cfg::STAGES;
            mbar_wait(&full[st], (it / Cfg::STAGES) & 1);
            if (kChunkPreempt && kb == kb0 && *reinterpret_cast<volatile int*>(&tile_cut[j]) <= c) {
              mbar_arrive(&empty[st]);        // poisoned stage: no data, hand it back
              mbar_arrive(&tmem_full[acc]);   // and tell the epilogue this chunk is the cut
              ++it;
              cut = true;
              break;
            }
            fence_after();
            const unsigned char* base = smem + (size_t)st * Cfg::STAGE_BYTES;
#pragma unroll
            for (int k = 0; k < Cfg::BK / Cfg::UMMA_K; ++k) {
              const uint32_t first = (kb != kb0 || k != 0);
              const int koff = k * Cfg::UMMA_K * Cfg::ESZ;   // 32 B per MMA-K step inside the atom
              if constexpr (Cfg::KIND == 0) {
                const uint64_t ahi = smem_desc(base + koff), alo = smem_desc(base + Cfg::A_BYTES + koff);
                const uint64_t bhi = smem_desc(base + 2 * Cfg::A_BYTES + koff);
                const uint64_t blo = smem_desc(base + 2 * Cfg::A_BYTES + Cfg::B_BYTES + koff);
                umma<0>(d, alo, bhi, idesc, first);   // small terms first
                umma<0>(d, ahi, blo, idesc, 1);
                umma<0>(d, ahi, bhi, idesc, 1);
              } else {
                // MN-major: UMMA_K = 16 K-rows = two 8-row groups = 2048 B per step;
                // K-major: 32 B per step inside the 128 B swizzle atom
                uint64_t da = Cfg::A_MN ? smem_desc_mn(base + k * 2048) : smem_desc(base + koff);
                uint64_t db = Cfg::B_MN ? smem_desc_mn(base + Cfg::A_BYTES + k * 2048)
                                        : smem_desc(base + Cfg::A_BYTES + koff);
                // narrow-channel convolutions: 16 K = two taps per MMA step
                if constexpr (ConvOf<Cfg>::value == 3) da = smem_desc_ns(base + k * 4096, 2048, 128);
                if constexpr (ConvOf<Cfg>::value == 4) db = smem_desc_ns(base + Cfg::A_BYTES + k * 256, 128, 1024);
                if constexpr (PR == 2) umma_pair(d, da, db, idesc, first);
                else umma<1>(d, da, db, idesc, first);
              }
            }
            // frees the stage once these MMAs retire (pair: in both CTAs)
            if constexpr (PR == 2) umma_commit_pair(&empty[st]);
            else umma_commit(&empty[st]);
          }
          if (cut) {
            ++ci;
            break;
          }
          if constexpr (PR == 2) umma_commit_pair(&tmem_full[acc]);
          else umma_commit(&tmem_full[acc]);
        }
        mbar_arrive(&tile_empty[j]);
      }
    }
    __syncwarp();
  } else if constexpr (Cfg::KIND == 1 && Cfg::BN == 64) {
    // -------------------------------------------------- epilogue (warps 2..9), 64-wide bf16-operand tiles
    // Two groups of four warps take alternate tiles (= the two TMEM
    // accumulators: one K chunk per tile), so two tiles drain concurrently;
    // each warp owns its TMEM lane quarter (32 rows) across all BN columns.
    // bf16 output is staged 64 columns at a time in the warp's own 4 KB of
    // shared memory (16 B chunks XOR-swizzled by row) and written back as
    // whole 128 B row segments; fp32 rows go straight from registers.  (For
    // 64-wide tiles this beats eight warps on one tile: K = 64 dgrad 78 -> 74
    // us; for 128-wide tiles it does not -- 35 -> 39 us at K = 64, N = 256.)
    const int q = warp & 3;
    const int grp = (warp - 2) >> 2;
    unsigned char* wstage = epi_smem + (size_t)(warp - 2) * (32 * 64 * 2);
    for (int i = 0;; ++i) {
      const int j = i % kSlots;
      mbar_wait(&tile_full[j], (i / kSlots) & 1);
      const long long t = tile_slot[j];
      if (t < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&tile_empty[j]);
        break;
      }
      if ((i & 1) == grp) {
        const int acc = i & 1;
        const TileWork w = tile_w[j];
        const int row0 = w.mb * Cfg::BM + q * 32;
        const int cr = goff(p, 4, w), cc = goff(p, 5, w);
        typename Cfg::OutT* cbase = reinterpret_cast<typename Cfg::OutT*>(p.c) + (size_t)w.split * p.split_stride +
                                    (size_t)cr * p.ldc + (size_t)(cc + w.nb * Cfg::BN);
        const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * Cfg::BN);
        mbar_wait(&tmem_full[acc], (i >> 1) & 1);
        fence_after();
        if constexpr (sizeof(typename Cfg::OutT) == 4) {
          const bool row_ok = row0 + lane < p.m;
          float* crow = reinterpret_cast<float*>(cbase) + (size_t)(row_ok ? row0 + lane : 0) * p.ldc;
#pragma unroll 1
          for (int c1 = 0; c1 < Cfg::BN; c1 += 32) {
            uint32_t r[32];
            tmem_ld32(lane_base + (uint32_t)c1, r);
            if (row_ok) {
#pragma unroll
              for (int v = 0; v < 8; ++v)
                st_out16(crow + c1 + 4 * v, make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]));
            }
          }
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tmem_empty[acc]);
        } else {
#pragma unroll 1
          for (int h = 0; h < Cfg::BN; h += 64) {
            uint32_t r[2][32];
            tmem_ld32(lane_base + (uint32_t)h, r[0]);
            tmem_ld32(lane_base + (uint32_t)(h + 32), r[1]);
            if (h + 64 >= Cfg::BN) {   // the accumulator is drained: hand it back to the MMA warp
              fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tmem_empty[acc]);
            }
            // (explicit shared-space accesses: generic ones cost 64-bit
            // address arithmetic per access)
            const uint32_t wst = smem_u32(wstage);
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              uint32_t wv[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int k = 8 * (v & 3) + 2 * e;
                __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(r[v >> 2][k]), __uint_as_float(r[v >> 2][k + 1]));
                wv[e] = *reinterpret_cast<uint32_t*>(&b);
              }
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(wst + lane * 128 + ((v ^ (lane & 7)) << 4)),
                           "r"(wv[0]), "r"(wv[1]), "r"(wv[2]), "r"(wv[3])
                           : "memory");
            }
            __syncwarp();
            // 32 rows x 8 chunks: each instruction writes 4 whole 128 B row segments
            __nv_bfloat16* cb = reinterpret_cast<__nv_bfloat16*>(cbase) + h;
#pragma unroll
            for (int it2 = 0; it2 < 8; ++it2) {
              const int rr = it2 * 4 + (lane >> 3), ch = lane & 7;
              uint4 v;
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                           : "r"(wst + rr * 128 + ((ch ^ (rr & 7)) << 4))
                           : "memory");
              if (row0 + rr < p.m) st_out16(cb + (size_t)(row0 + rr) * p.ldc + ch * 8, v);
            }
            __syncwarp();
            if (p.bnf.part != nullptr) {
              // batch-norm statistics of the box (see the TMA-store path); the
              // staging box was read back synchronously: free
              const float4 cs = p.bnf.dbg == 2 ? make_float4(0.f, 0.f, 0.f, 0.f)
                                               : bn_box_colsum(wst, lane, p.m - row0);
              __syncwarp();
              bn_fuse_box(p.bnf, cs, w.mb, cc + w.nb * Cfg::BN + h, (warp - 2) & 3, lane,
                          reinterpret_cast<float*>(epi_smem + (size_t)(4 * grp) * (32 * 64 * 2)), 1024, 2 + grp);
            }
          }
        }
        if (q == 0 && lane == 0) gemm_log_end(block_log_of(s), t, p);   // (the group's first warp)
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&tile_empty[j]);
    }
  } else if (Cfg::KIND == 1 && sizeof(typename Cfg::OutT) == 2 && p.c_tma) {
    // -------------------------------------------------- epilogue (warps 2..9), TMA store
    // 128/256-wide bf16 tiles of a plain GEMM: each warp drains its lane
    // quarter x column half (32 rows x BN/2 columns) in 64-column boxes,
    // releases the accumulator after the last one, stages each box in its own
    // 4 KB (the 128B-swizzle layout) and one lane issues a TMA store -- the
    // warp never waits for global writes, only (before restaging) for the
    // previous store to finish reading its staging box
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int HALF = Cfg::BN / 2;
    unsigned char* wstage = epi_smem + (size_t)(warp - 2) * 4096;
    const uint32_t wst = smem_u32(wstage);
    uint32_t ci = 0;
    // fused batch-norm statistics: a box's column sums are taken right after
    // its store is issued and exchanged at the next restaging (or the end),
    // when the unit's staging boxes are free anyway -- waiting for the
    // store's read right away cost the CTA-pair kinds ~+50 %
    float4 bn_cs = make_float4(0.f, 0.f, 0.f, 0.f);
    int bn_prow = -1, bn_c0 = 0;
    auto bn_flush = [&]() {
      if (bn_prow >= 0) {
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        bn_fuse_box(p.bnf, bn_cs, bn_prow, bn_c0, (warp - 2) & 3, lane,
                    reinterpret_cast<float*>(epi_smem + (size_t)(4 * half) * 4096), 1024, 2 + half);
        bn_prow = -1;
      }
    };
    for (int i = 0;; ++i) {
      const int j = i % kSlots;
      mbar_wait(&tile_full[j], (i / kSlots) & 1);
      const long long t = tile_slot[j];
      if (t < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&tile_empty[j]);
        break;
      }
      const TileWork w = tile_w[j];
      const int acc = ci & 1;   // one K chunk per tile for the bf16 kinds
      mbar_wait(&tmem_full[acc], (ci >> 1) & 1);
      fence_after();
#pragma unroll 1
      for (int bx = 0; bx < HALF; bx += 64) {
        uint32_t r[2][32];
        const uint32_t lb = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * Cfg::BN + half * HALF + bx);
        tmem_ld32(lb, r[0]);
        tmem_ld32(lb + 32, r[1]);
        if (bx + 64 >= HALF) {
          fence_before();
          __syncwarp();
          if (lane == 0) release_acc<PR>(&tmem_empty[acc]);
        }
        const int ycol = w.nb * Cfg::BN + half * HALF + bx, yrow = (w.mb * PR + (int)rank) * Cfg::BM + q * 32;
        unsigned char* srow = wstage + (size_t)lane * 128;
        // stage 64 values of this lane's row (bf16, 128B-swizzle) and TMA-store the box
        auto stage_store = [&](const CUtensorMap* map) {
          bn_flush();
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            uint32_t wv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int k = 8 * (v & 3) + 2 * e;
              __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(r[v >> 2][k]), __uint_as_float(r[v >> 2][k + 1]));
              wv[e] = *reinterpret_cast<uint32_t*>(&b);
            }
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(wst + lane * 128 + ((v ^ (lane & 7)) << 4)),
                         "r"(wv[0]), "r"(wv[1]), "r"(wv[2]), "r"(wv[3])
                         : "memory");
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) tma_store_2d(map, wst, ycol, yrow);
          __syncwarp();
        };
        if (p.ep.on) {
          // fused linear-layer epilogue on the fp32 accumulator
          const long long row = min((long long)(yrow + lane), (long long)p.m - 1);   // (rows past M: clipped by the map)
#pragma unroll
          for (int g8 = 0; g8 < 8; ++g8) {
            float x[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = __uint_as_float(r[g8 >> 2][8 * (g8 & 3) + e]);
            ep_bias_res8(p.ep, row, ycol + 8 * g8, x);
#pragma unroll
            for (int e = 0; e < 8; ++e) r[g8 >> 2][8 * (g8 & 3) + e] = __float_as_uint(x[e]);
          }
          if (p.ep_pre) stage_store(&p.b_lo);
          if (p.ep.act) {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              r[0][k] = __float_as_uint(ep_act(__uint_as_float(r[0][k]), p.ep.act));
              r[1][k] = __float_as_uint(ep_act(__uint_as_float(r[1][k]), p.ep.act));
            }
          }
        }
        stage_store(&p.a_lo);
        if (p.bnf.part != nullptr && yrow - q * 32 < p.m) {
          // batch-norm statistics of this 64-column box from the staged bf16
          // values (rows past M excluded; tiles wholly past M skipped)
          bn_cs = p.bnf.dbg == 2 ? make_float4(0.f, 0.f, 0.f, 0.f) : bn_box_colsum(wst, lane, p.m - yrow);
          bn_prow = yrow / 128;
          bn_c0 = ycol;
        }
      }
      ++ci;
      if (warp == 2 && lane == 0 && lead) gemm_log_end(block_log_of(s), t, p);
      if (lane == 0) mbar_arrive(&tile_empty[j]);
    }
    bn_flush();
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  } else {
    // -------------------------------------------------- epilogue (warps 2..9)
    const int q = warp & 3;                     // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;           // which half of the tile's columns it drains
    constexpr int HALF = Cfg::BN / 2;
    uint32_t ci = 0;
    for (int i = 0;; ++i) {
      const int j = i % kSlots;
      mbar_wait(&tile_full[j], (i / kSlots) & 1);
      const long long t = tile_slot[j];
      const int c0 = tile_c0[j];
      if (t < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&tile_empty[j]);
        break;
      }
      const TileWork w = tile_w[j];
      const int row = (w.mb * PR + (int)rank) * Cfg::BM + q * 32 + lane;
      const bool row_ok = row < p.m;   // M tail: TMA zero-fills the rows past M, stores skip them
      const int cr = goff(p, 4, w), cc = goff(p, 5, w);
      typename Cfg::OutT* crow = reinterpret_cast<typename Cfg::OutT*>(p.c) + (size_t)w.split * p.split_stride +
                                 (size_t)(cr + (row_ok ? row : 0)) * p.ldc + (size_t)(cc + w.nb * Cfg::BN);
      const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
      for (int c = c0; c < w.nch; ++c, ++ci) {
        const int acc = ci & 1;
        mbar_wait(&tmem_full[acc], (ci >> 1) & 1);
        fence_after();
        if (kChunkPreempt && *reinterpret_cast<volatile int*>(&tile_cut[j]) <= c) {
          // preempted before chunk c: park the fp32 running total in C
          if (c > c0) {
#pragma unroll 1
            for (int c1 = half * HALF; c1 < (half + 1) * HALF; c1 += 32) {
              uint32_t r[32];
              tmem_ld32(lane_base + (uint32_t)(2 * Cfg::BN + c1), r);
              float4* dst = reinterpret_cast<float4*>(crow + c1);
#pragma unroll
              for (int v = 0; v < 8; ++v)
                dst[v] = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                     __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
            }
          }
          __threadfence();
          asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");   // all epilogue warps saved
          if (warp == 2 && lane == 0) {
            unsigned long long* ring = p.resume;
            const unsigned long long slot = atomicAdd(ring, 1ull);
            __threadfence();
            *reinterpret_cast<volatile unsigned long long*>(ring + 2 + (slot % kResumeCap)) =
                (unsigned long long)(t + 1) | ((unsigned long long)c << 40);
          }
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tmem_empty[acc]);
          ++ci;
          break;
        }
        const bool last = (c == w.nch - 1);
#pragma unroll 1
        for (int c1 = half * HALF; c1 < (half + 1) * HALF; c1 += 32) {
          // chunk partial + running fp32 total (kept in TMEM columns [2BN, 3BN))
          uint32_t r[32];
          tmem_ld32(lane_base + (uint32_t)(acc * Cfg::BN + c1), r);
          if (c > c0) {
            uint32_t sv[32];
            tmem_ld32(lane_base + (uint32_t)(2 * Cfg::BN + c1), sv);
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) + __uint_as_float(sv[e]));
          } else if (c0 > 0) {
            // resumed tile: the partial total a preempted worker saved in C
            if constexpr (Cfg::KIND == 0) {
              const float4* src = reinterpret_cast<const float4*>(crow + c1);
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                const float4 x = src[v];
                r[4 * v] = __float_as_uint(__uint_as_float(r[4 * v]) + x.x);
                r[4 * v + 1] = __float_as_uint(__uint_as_float(r[4 * v + 1]) + x.y);
                r[4 * v + 2] = __float_as_uint(__uint_as_float(r[4 * v + 2]) + x.z);
                r[4 * v + 3] = __float_as_uint(__uint_as_float(r[4 * v + 3]) + x.w);
              }
            }
          }
          if (!last) {
            tmem_st32(lane_base + (uint32_t)(2 * Cfg::BN + c1), r);
          } else if constexpr (sizeof(typename Cfg::OutT) == 4) {
            if (Cfg::KIND == 1 && p.c_tma == 2) {
              // stage this warp's 32 x 32 fp32 box (128B-swizzle layout) and
              // store it with one TMA tensor store; rows past M are clipped by
              // the map (bind enables this only where that is exact)
              unsigned char* wst = epi_smem + (size_t)(warp - 2) * 4096;
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              __syncwarp();
              unsigned char* srow = wst + (size_t)lane * 128;
#pragma unroll
              for (int v = 0; v < 8; ++v)
                *reinterpret_cast<uint4*>(srow + ((v ^ (lane & 7)) << 4)) =
                    make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0)
                tma_store_2d(&p.a_lo, smem_u32(wst), cc + w.nb * Cfg::BN + c1,
                             (int)(w.split * (p.split_stride / p.ldc)) + cr + (w.mb * PR + (int)rank) * Cfg::BM + q * 32);
            } else if (row_ok) {
#pragma unroll
              for (int v = 0; v < 8; ++v)
                st_out16(crow + c1 + 4 * v, make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]));
            }
          } else if (!row_ok) {
          } else if constexpr (PR == 2) {
            // pair tiles with a strided / batched bf16 C: the row straight from registers
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint32_t w4[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[8 * v + 2 * e]),
                                                         __uint_as_float(r[8 * v + 2 * e + 1]));
                w4[e] = *reinterpret_cast<uint32_t*>(&h);
              }
              st_out16(crow + c1 + 8 * v, make_uint4(w4[0], w4[1], w4[2], w4[3]));
            }
          } else {
            // stage this lane's row (16 B chunks, chunk index XOR row % 8:
            // conflict-free) -- written out coalesced below
            unsigned char* srow = epi_smem + (size_t)q * (32 * Cfg::BN * 2) + (size_t)lane * (Cfg::BN * 2);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint32_t w[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[8 * v + 2 * e]),
                                                         __uint_as_float(r[8 * v + 2 * e + 1]));
                w[e] = *reinterpret_cast<uint32_t*>(&h);
              }
              const int chunk = (c1 >> 3) + v;
              *reinterpret_cast<uint4*>(srow + ((chunk ^ (lane & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) release_acc<PR>(&tmem_empty[acc]);
        if constexpr (sizeof(typename Cfg::OutT) == 2 && PR == 1) {
          if (last) {
            // the two warps of this lane quarter staged the two column halves
            // of the same 32 rows; after a pair barrier each writes 16 whole
            // rows out, coalesced (one warp instruction = 512 contiguous bytes
            // for BN = 128)
            asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
            constexpr int CPR = Cfg::BN / 8;   // 16 B chunks per row
            const unsigned char* sbase = epi_smem + (size_t)q * (32 * Cfg::BN * 2);
            const long long row0 = (long long)w.mb * Cfg::BM + q * 32;
            __nv_bfloat16* cbase = reinterpret_cast<__nv_bfloat16*>(p.c) + (size_t)cr * p.ldc + (size_t)(cc + w.nb * Cfg::BN);
#pragma unroll 4
            for (int i2 = half * 16 * CPR + lane; i2 < (half + 1) * 16 * CPR; i2 += 32) {
              const int rr = i2 / CPR, ch = i2 % CPR;
              const uint4 v = *reinterpret_cast<const uint4*>(sbase + (size_t)rr * (Cfg::BN * 2) + ((ch ^ (rr & 7)) << 4));
              if (row0 + rr < p.m) st_out16(cbase + (size_t)(row0 + rr) * p.ldc + ch * 8, v);
            }
            asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");   // staging free for the next tile
          }
        }
      }
      __syncwarp();
      if (warp == 2 && lane == 0 && lead) gemm_log_end(block_log_of(s), t, p);
      if (lane == 0) mbar_arrive(&tile_empty[j]);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // (TMA-store epilogue)
    __syncwarp();
  }

  fence_before();
  if constexpr (PR == 2) cluster_sync_all();   // no remote arrive or MMA into this CTA is still in flight
  else __syncthreads();
  fence_after();
  if (warp == 1) {
    if constexpr (PR == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(Cfg::TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(Cfg::TMEM_COLS));
  }
  if constexpr (MODE == kPtb) {
    if (threadIdx.x == 0) {
      if (s.worker_log != nullptr) {   // per-worker telemetry: smid | blocks, entry, first tile, exit
        unsigned long long* wl = s.worker_log + 4ull * blockIdx.x;
        wl[0] = ((unsigned long long)smid() << 32) | (blocks_run & 0xffffffffull);
        wl[1] = t_entry;
        wl[2] = *reinterpret_cast<volatile unsigned long long*>(tmem_base_slot + 2);
        wl[3] = globaltimer();
      }
      if constexpr (Cfg::KIND == 1) ptb_worker_exit(s, stopped, t_entry, s.ret_ring, blocks_run);
      else ptb_worker_exit(s, stopped, t_entry, kChunkPreempt ? p.resume : nullptr);
    }
  }
}

// ---------------------------------------------------------------- split_tf32
struct SplitTf32 {
  static constexpr int kThreads = 256;
  static constexpr int kVec = 4;                                  // float4 per thread
  static constexpr int kElemsPerBlock = kThreads * kVec * 4;      // 4096
  struct Params {
    const float4* x;
    float4* hi;
    float4* lo;
    long long n4;
  };
  static __device__ __forceinline__ float tf32_rna(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
  }
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const long long base = (long long)bidx.x * (kThreads * kVec) + threadIdx.x;
    float4 v[kVec];
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const long long k = base + (long long)j * kThreads;
      if (k < p.n4) v[j] = ld_stream(p.x + k);
    }
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const long long k = base + (long long)j * kThreads;
      if (k < p.n4) {
        const float4 h = make_float4(tf32_rna(v[j].x), tf32_rna(v[j].y), tf32_rna(v[j].z), tf32_rna(v[j].w));
        p.hi[k] = h;
        p.lo[k] = make_float4(v[j].x - h.x, v[j].y - h.y, v[j].z - h.z, v[j].w - h.w);
      }
    }
  }
};


// ---------------------------------------------------------------- fused attention softmax
// One logical block = 128 query rows of one (sequence, head), all T <= 512 keys:
//   forward  (MODE 0): S = Q K^T in TMEM (tcgen05, 128 x T fp32), P = softmax(scale * S)
//                      row by row from TMEM, P (bf16) TMA-stored -- the fp32 score
//                      matrix never reaches HBM (it was a GEMM output + a softmax pass);
//   backward (MODE 1): dP = dO V^T in TMEM, dS = P * (dP - rowsum(P * dP)) * scale,
//                      dS (bf16) TMA-stored; P is TMA-loaded as a tile into the
//                      freed operand buffers (+ 48 KB) once the MMA is done --
//                      per-lane row loads (32 rows per warp instruction) were
//                      70 % of the stall samples, 65 us per BERT-large launch.
// Q / K / V / dO are head-D (= 64) column slices of row-major activations (the
// fused QKV buffer), read by TMA; the Body runs under k_original / k_sliced /
// k_ptb like every transformable kind.  8 warps: thread 0 issues the TMA loads
// and the MMAs, then all warps drain TMEM (warp w: lane quarter w % 4, key
// half w / 4; the two warps of a quarter exchange row max / sum through smem).
template <int MODE>
struct AttnSoftmax {
  static constexpr int kThreads = 256;
  static constexpr int kD = 64;                  // head dim = one 128 B swizzle atom of bf16
  static constexpr int kTileBytes = 128 * kD * 2;   // 16 KB: 128 rows x 64 bf16
  // operands (A + up to 4 B boxes) | 8 x 4 KB staging | row exchange, barriers,
  // TMEM slot (4 KB) | MODE 1: P boxes 5..7 (boxes 0..4 reuse the operands)
  static constexpr int kSmem = 1024 + kTileBytes * 5 + 8 * 4096 + 4096 + (MODE == 1 ? 3 * kTileBytes : 0);
  struct Params {
    CUtensorMap a_map;     // MODE 0: Q; MODE 1: dO   (box 64 cols x 128 rows)
    CUtensorMap b_map;     // MODE 0: K; MODE 1: V    (box 64 cols x 128 rows)
    CUtensorMap out_map;   // P / dS [z * T + i, T] bf16 (box 64 cols x 32 rows)
    CUtensorMap p_map;     // MODE 1: P [z * T + i, T] bf16 (box 64 cols x 128 rows)
    const __nv_bfloat16* p_in;   // MODE 1: P [z * T + i, T]
    long long a_col0, a_col_h, b_col0, b_col_h;   // operand column origin: col0 + h * col_h
    int T, H;
    float scale;
  };

  static __device__ __forceinline__ uint32_t* tmem_slot(char* smem_raw) {
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* red = reinterpret_cast<float*>(sm + 5 * kTileBytes + 8 * 4096);
    return reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t*>(red + 2 * 2 * 128) + 3);
  }
  // TMEM once per CTA (all 512 columns), taken before the CTA lets a
  // programmatic dependent launch begin: a successor GEMM CTA waiting for this
  // kernel can then never hold columns this CTA needs for its next block
  static __device__ __forceinline__ void cta_init(char* smem_raw) {
    if ((threadIdx.x >> 5) == 0)
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot(smem_raw))),
                   "n"(512));
    fence_before();
    __syncthreads();
    fence_after();
  }
  static __device__ __forceinline__ void cta_exit(char* smem_raw) {
    fence_before();
    __syncthreads();
    fence_after();
    if ((threadIdx.x >> 5) == 0) {
      const uint32_t t = *tmem_slot(smem_raw);
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "n"(512));
    }
  }

  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char* smem_raw) {
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sa = sm;                          // A tile (128 x 64)
    unsigned char* sb = sm + kTileBytes;             // B: T / 128 boxes of 128 keys
    unsigned char* stg = sm + 5 * kTileBytes;        // 8 x 4 KB output staging
    float* red = reinterpret_cast<float*>(stg + 8 * 4096);   // [2 halves][2 values][128 rows]
    uint64_t* bar = reinterpret_cast<uint64_t*>(red + 2 * 2 * 128);   // [0] operands, [1] MMA done, [2] P tile
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 3);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int z = (int)bidx.y, b = z / p.H, h = z - b * p.H, r0 = (int)bidx.x * 128;
    const int nkb = p.T / 128;
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      mbar_init(&bar[2], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t tmem = *tslot;   // allocated in cta_init
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bar[0], (uint32_t)(kTileBytes * (1 + nkb)));
      tma_load_2d(sa, &p.a_map, &bar[0], (int)(p.a_col0 + h * p.a_col_h), b * p.T + r0);
      for (int kb = 0; kb < nkb; ++kb)
        tma_load_2d(sb + kb * kTileBytes, &p.b_map, &bar[0], (int)(p.b_col0 + h * p.b_col_h), b * p.T + kb * 128);
      mbar_wait(&bar[0], 0);
      fence_after();
      constexpr uint32_t idesc = make_idesc<1, 128>();   // bf16, M = 128, N = 128
#pragma unroll
      for (int k = 0; k < kD / 16; ++k) {
        const uint64_t da = smem_desc(sa + k * 32);
        for (int kb = 0; kb < nkb; ++kb)
          umma<1>(tmem + (uint32_t)(kb * 128), da, smem_desc(sb + kb * kTileBytes + k * 32), idesc, k > 0);
      }
      umma_commit(&bar[1]);
    }
    __syncwarp();
    mbar_wait(&bar[1], 0);
    fence_after();
    // ---- row pass over TMEM: warp w drains lanes [32 q, 32 q + 32), keys [half * T/2, +T/2)
    const int q = warp & 3, half = warp >> 2;
    const int kcols = p.T / 2;
    const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(half * kcols);
    const long long grow = (long long)z * p.T + r0 + q * 32 + lane;   // this lane's row of P / dS
    float* mine = red + half * 256 + q * 32 + lane;
    const float* other = red + (half ^ 1) * 256 + q * 32 + lane;
    if constexpr (MODE == 0) {
      float m = -INFINITY;
      for (int c = 0; c < kcols; c += 64) {   // two 32-column loads in flight per wait
        uint32_t r[2][32];
        tmem_ld32_nw(lb + c, r[0]);
        tmem_ld32_nw(lb + c + 32, r[1]);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) m = fmaxf(m, fmaxf(__uint_as_float(r[0][e]), __uint_as_float(r[1][e])) * p.scale);
      }
      mine[0] = m;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
      m = fmaxf(m, other[0]);
      float sum = 0.f;
      for (int c = 0; c < kcols; c += 64) {
        uint32_t r[2][32];
        tmem_ld32_nw(lb + c, r[0]);
        tmem_ld32_nw(lb + c + 32, r[1]);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float v0 = __expf(__uint_as_float(r[0][e]) * p.scale - m);
          const float v1 = __expf(__uint_as_float(r[1][e]) * p.scale - m);
          sum += v0 + v1;
          r[0][e] = __float_as_uint(v0);
          r[1][e] = __float_as_uint(v1);
        }
        tmem_st32(lb + c, r[0]);   // exp(scale s - m) back in place
        tmem_st32(lb + c + 32, r[1]);
      }
      mine[128] = sum;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
      sum += other[128];
      const float inv = 1.f / sum;
      // ---- P = e / sum: bf16, staged 32 rows x 64 keys, TMA-stored
      unsigned char* wst = stg + (size_t)warp * 4096;
      for (int c = 0; c < kcols; c += 64) {
        uint32_t r[2][32];
        tmem_ld32_nw(lb + c, r[0]);
        tmem_ld32_nw(lb + c + 32, r[1]);
        tmem_wait_ld();
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        unsigned char* srow = wst + (size_t)lane * 128;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          uint32_t wv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = 8 * (v & 3) + 2 * e;
            __nv_bfloat162 bb = __floats2bfloat162_rn(__uint_as_float(r[v >> 2][k]) * inv, __uint_as_float(r[v >> 2][k + 1]) * inv);
            wv[e] = *reinterpret_cast<uint32_t*>(&bb);
          }
          *reinterpret_cast<uint4*>(srow + ((v ^ (lane & 7)) << 4)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) tma_store_2d(&p.out_map, smem_u32(wst), half * kcols + c, (int)(grow - lane));
        __syncwarp();
      }
    } else {
      // dS = P * (dP - delta) * scale, delta = sum_j P dP.  P's tile (128 rows
      // x T) by TMA into the operand buffers the finished MMA no longer reads
      // (boxes 0..4) and 48 KB more (5..7); lane = row, 128B-swizzled rows.
      unsigned char* pext = stg + 8 * 4096 + 4096;
      auto pbox = [&](int bx) -> uint32_t { return smem_u32(bx < 5 ? sm + bx * kTileBytes : pext + (bx - 5) * kTileBytes); };
      if (threadIdx.x == 0) {
        mbar_expect_tx(&bar[2], (uint32_t)(kTileBytes * nkb * 2));
        for (int bx = 0; bx < 2 * nkb; ++bx)
          tma_load_2d(bx < 5 ? (void*)(sm + bx * kTileBytes) : (void*)(pext + (bx - 5) * kTileBytes), &p.p_map, &bar[2],
                      bx * 64, z * p.T + r0);
      }
      mbar_wait(&bar[2], 0);
      const int rr = q * 32 + lane;
      auto ldp = [&](uint4 (&pv)[8], int c) {   // this lane's row, columns [half * kcols + c, + 64)
        const uint32_t rowb = pbox((half * kcols + c) >> 6) + rr * 128;
#pragma unroll
        for (int v = 0; v < 8; ++v)
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(pv[v].x), "=r"(pv[v].y), "=r"(pv[v].z), "=r"(pv[v].w)
                       : "r"(rowb + ((v ^ (rr & 7)) << 4)));
      };
      float dot = 0.f;
      for (int c = 0; c < kcols; c += 64) {
        uint32_t r[2][32];
        uint4 pv[8];
        ldp(pv, c);
        tmem_ld32_nw(lb + c, r[0]);
        tmem_ld32_nw(lb + c + 32, r[1]);
        tmem_wait_ld();
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&pv[v]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = 8 * (v & 3) + 2 * e;
            const float2 f = __bfloat1622float2(h2[e]);
            dot += f.x * __uint_as_float(r[v >> 2][k]) + f.y * __uint_as_float(r[v >> 2][k + 1]);
          }
        }
      }
      mine[0] = dot;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
      dot += other[0];
      unsigned char* wst = stg + (size_t)warp * 4096;
      const uint32_t wsts = smem_u32(wst);
      for (int c = 0; c < kcols; c += 64) {
        uint32_t r[2][32];
        uint4 pv[8];
        ldp(pv, c);
        tmem_ld32_nw(lb + c, r[0]);
        tmem_ld32_nw(lb + c + 32, r[1]);
        tmem_wait_ld();
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&pv[v]);
          uint32_t wv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = 8 * (v & 3) + 2 * e;
            const float2 f = __bfloat1622float2(h2[e]);
            __nv_bfloat162 bb = __floats2bfloat162_rn(f.x * (__uint_as_float(r[v >> 2][k]) - dot) * p.scale,
                                                      f.y * (__uint_as_float(r[v >> 2][k + 1]) - dot) * p.scale);
            wv[e] = *reinterpret_cast<uint32_t*>(&bb);
          }
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(wsts + lane * 128 + ((v ^ (lane & 7)) << 4)),
                       "r"(wv[0]), "r"(wv[1]), "r"(wv[2]), "r"(wv[3])
                       : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) tma_store_2d(&p.out_map, wsts, half * kcols + c, (int)(grow - lane));
        __syncwarp();
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    fence_before();
    __syncthreads();   // TMEM reads done, staging free, barriers reusable by the next block
    fence_after();
  }
};

}  // namespace gemm

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  }
  return fn;
}

// rows x cols (K innermost) row-major matrix, box = box_rows x 128 bytes, 128 B swizzle
static bool aligned16_(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static bool getenv_flag(const char* name) {   // experiment switches, read at bind time
  const char* e = getenv(name);
  return e != nullptr && e[0] != '\0' && e[0] != '0';
}

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// TMA im2col map over an NHWC bf16 tensor: boxes of `pixels` output pixels x
// 64 channels (128 B rows, 128B swizzle -- the K-major / MN-major operand
// tile layouts), traversal stride = the convolution stride, the pixel box
// [-pad, W - 1 + pad - (k - 1)] per spatial dimension (zeros outside)
static int make_im2col_map(CUtensorMap* m, const void* x, const tally_conv_geometry& g, int pixels,
                           bool narrow = false) {
  static EncodeIm2colFn enc = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeIm2col", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeIm2colFn>(f);
    return (EncodeIm2colFn) nullptr;
  }();
  if (!enc) { set_error("cuTensorMapEncodeIm2col unavailable"); return TALLY_ENODEV; }
  cuuint64_t dims[4] = {(cuuint64_t)g.c, (cuuint64_t)g.w, (cuuint64_t)g.h, (cuuint64_t)g.n};
  cuuint64_t strides[3] = {(cuuint64_t)g.c * 2, (cuuint64_t)g.w * g.c * 2, (cuuint64_t)g.h * g.w * g.c * 2};
  int lower[2] = {-g.pad, -g.pad};
  int upper[2] = {g.pad - (g.k - 1), g.pad - (g.k - 1)};
  cuuint32_t estr[4] = {1, (cuuint32_t)g.stride, (cuuint32_t)g.stride, 1};
  // narrow: 8-channel boxes (16 B per pixel), written densely (no swizzle)
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, lower, upper,
                   narrow ? 8 : 64, (cuuint32_t)pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   narrow ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeIm2col failed (%d)", (int)r); return TALLY_EINVAL; }
  return TALLY_OK;
}

static int make_map(CUtensorMap* m, const void* ptr, CUtensorMapDataType dt, int esz, long long rows,
                    long long cols, int box_rows, long long ld = 0) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return TALLY_ENODEV; }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld > 0 ? ld : cols) * esz};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return TALLY_EINVAL; }
  return TALLY_OK;
}

template <class Cfg>
static int bind_gemm(const tally_kernel_args* a, Instance* inst, bool split) {
  gemm::GemmParams p;
  memset(&p, 0, sizeof(p));
  const long long M = a->i[0], N = a->i[1], K = a->i[2];
  const long long splits = a->i[4] > 0 ? a->i[4] : 1;
  // bf16 kinds take any M (row tail); the 3xTF32 kind keeps whole tiles
  // (K tail: TMA zero-fills the k-block past K in both operands; rows must
  // stay 16-byte aligned for the tensor map)
  const bool m_ok = Cfg::KIND == 1 ? true : (M % Cfg::BM == 0);
  // (MN-major: the tensor-map rows are K, the contiguous dims M and N)
  const bool k_ok = (Cfg::A_MN || Cfg::B_MN) ? (M % 8 == 0 && K % 8 == 0) : Cfg::KIND == 1 ? (K % 8 == 0) : (K % Cfg::BK == 0);
  if (M < 1 || N < 1 || K < 1 || !m_ok || N % Cfg::BN || !k_ok) {
    set_error("gemm: need M %s, N %% %d == 0, K %s (got %lld %lld %lld)",
              Cfg::KIND == 1 ? ">= 1" : "% 128 == 0", Cfg::BN, Cfg::KIND == 1 ? "% 8 == 0" : "% 32 == 0", M, N, K);
    return TALLY_EINVAL;
  }
  const long long KBlocks = (K + Cfg::BK - 1) / Cfg::BK;
  if (splits > KBlocks || (Cfg::KIND == 0 && splits != 1) || (splits > 1 && sizeof(typename Cfg::OutT) != 4)) {
    set_error("gemm: split-K needs fp32 output, 1 <= splits <= K / %d (got %lld)", Cfg::BK, splits);
    return TALLY_EINVAL;
  }
  const int nptr = split ? 5 : 3;
  for (int i = 0; i < nptr; ++i)
    if (!a->ptr[i] || reinterpret_cast<uintptr_t>(a->ptr[i]) % 16) {
      set_error("gemm: operand %d missing or not 16-byte aligned", i);
      return TALLY_EINVAL;
    }
  const CUtensorMapDataType dt = Cfg::KIND == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  int rc;
  if (split) {   // ptr: A_hi, A_lo, B_hi, B_lo, C
    if ((rc = make_map(&p.a_hi, a->ptr[0], dt, Cfg::ESZ, M, K, Cfg::BM))) return rc;
    if ((rc = make_map(&p.a_lo, a->ptr[1], dt, Cfg::ESZ, M, K, Cfg::BM))) return rc;
    if ((rc = make_map(&p.b_hi, a->ptr[2], dt, Cfg::ESZ, N, K, Cfg::BN))) return rc;
    if ((rc = make_map(&p.b_lo, a->ptr[3], dt, Cfg::ESZ, N, K, Cfg::BN))) return rc;
    p.c = a->ptr[4];
  } else if constexpr (gemm::ConvOf<Cfg>::value != 0) {
    // implicit-GEMM convolution: ptr[3] = tally_conv_geometry
    constexpr int CV = gemm::ConvOf<Cfg>::value;
    const tally_conv_geometry* G = static_cast<const tally_conv_geometry*>(a->ptr[3]);
    constexpr bool narrow = CV >= 3;
    if (!G || G->n < 1 || G->h < 1 || G->w < 1 || (narrow ? G->c != 8 : (G->c < 64 || G->c % 64)) || G->k < 1 ||
        G->stride < 1 || G->pad < 0 || G->k > 8 || G->pad >= G->k) {
      set_error("conv: need a geometry with c %% 64 == 0 (the *_c8 kinds: c == 8), 1 <= k <= 8, stride >= 1, "
                "0 <= pad < k");
      return TALLY_EINVAL;
    }
    const long long ho = (G->h + 2 * G->pad - G->k) / G->stride + 1, wo = (G->w + 2 * G->pad - G->k) / G->stride + 1;
    const long long P = (long long)G->n * ho * wo, Kd = (long long)G->k * G->k * G->c;
    // (narrow kinds: the k*k*8 taps padded to whole 64-wide k-blocks / N tiles)
    const long long Kp = narrow ? (Kd + 63) / 64 * 64 : Kd;
    constexpr bool fwd = CV == 1 || CV == 3;
    if (ho < 1 || wo < 1 || (fwd && (M != P || K != Kp)) || (!fwd && (N != Kp || K != P)) ||
        (CV == 2 && G->c % Cfg::BN != 0 && Cfg::BN > G->c)) {
      set_error("conv: GEMM shape does not match the geometry (forward: M = n*ho*wo, K = k*k*c; weight "
                "gradient: N = k*k*c, K = n*ho*wo)");
      return TALLY_EINVAL;
    }
    if constexpr (fwd) {
      if ((rc = make_im2col_map(&p.a_hi, a->ptr[0], *G, Cfg::BM, narrow))) return rc;
      if ((rc = make_map(&p.b_hi, a->ptr[1], dt, Cfg::ESZ, N, K, Cfg::BN))) return rc;
    } else {
      if ((rc = make_map(&p.a_hi, a->ptr[0], dt, Cfg::ESZ, K, M, Cfg::BK))) return rc;   // dy [P, cout], MN-major
      if ((rc = make_im2col_map(&p.b_hi, a->ptr[1], *G, Cfg::BK, narrow))) return rc;
    }
    p.c = a->ptr[2];
    p.cv_c = G->c;
    p.cv_k = G->k;
    p.cv_cblocks = G->c / 64;
    p.cv_stride = G->stride;
    p.cv_pad = G->pad;
    p.cv_wo = (int)wo;
    p.cv_hw = (int)(ho * wo);
    p.cv_n = G->n;
  } else {       // ptr: A, B, C [, layout]; MN-major operand = its transpose stored row-major
    const tally_gemm_layout* L = static_cast<const tally_gemm_layout*>(a->ptr[3]);
    const long long ar = L ? L->a_rows : (Cfg::A_MN ? K : M), acl = L ? L->a_cols : (Cfg::A_MN ? M : K);
    const long long br = L ? L->b_rows : (Cfg::B_MN ? K : N), bcl = L ? L->b_cols : (Cfg::B_MN ? N : K);
    if ((rc = make_map(&p.a_hi, a->ptr[0], dt, Cfg::ESZ, ar, acl, Cfg::A_MN ? Cfg::BK : Cfg::BM, L ? L->a_ld : 0))) return rc;
    // (a CTA pair loads BN / 2 rows of B per CTA)
    if ((rc = make_map(&p.b_hi, a->ptr[1], dt, Cfg::ESZ, br, bcl, Cfg::B_MN ? Cfg::BK : Cfg::BN / gemm::PairOf<Cfg>::value,
                       L ? L->b_ld : 0))) return rc;
    p.c = a->ptr[2];
    if (L) {
      if (L->batches < 1 || L->hdiv < 1 || L->ldc < N) { set_error("gemm layout: batches, hdiv >= 1, ldc >= N"); return TALLY_EINVAL; }
      const long long* offs[6] = {L->a_row_off, L->a_col_off, L->b_row_off, L->b_col_off, L->c_row_off, L->c_col_off};
      for (int w = 0; w < 6; ++w) { p.off[w][0] = offs[w][0]; p.off[w][1] = offs[w][1]; }
    }
  }
  p.m = (int)M;
  p.n = (int)N;
  p.k = (int)K;
  p.c_tma = 0;
  p.bn = Cfg::BN;
  p.bk = Cfg::BK;
  p.causal = (int)a->i[5];
  constexpr int PR = gemm::PairOf<Cfg>::value;
  if (p.causal < 0 || p.causal > 3 || (p.causal && (Cfg::KIND != 1 || splits != 1 || M % Cfg::BM || PR != 1))) {
    set_error("gemm: causal mode 0-3, bf16 single-CTA kinds, no split-K, M %% 128 == 0");
    return TALLY_EINVAL;
  }
  p.tiles_m = (int)((M + Cfg::BM * PR - 1) / (Cfg::BM * PR));   // (pair: 256-row tiles)
  p.tiles_n = (int)(N / Cfg::BN);
  const tally_gemm_layout* lay =
      (split || gemm::ConvOf<Cfg>::value != 0) ? nullptr : static_cast<const tally_gemm_layout*>(a->ptr[3]);
  p.batches = lay ? lay->batches : 1;
  p.hdiv = lay ? lay->hdiv : 1;
  p.ldc = lay ? lay->ldc : N;
  p.split_stride = M * N;
  p.splits = (int)splits;
  if constexpr (Cfg::KIND == 1 && Cfg::BN >= 128 && sizeof(typename Cfg::OutT) == 2) {
    // TMA-store epilogue for plain (unbatched, unsplit, zero-offset) GEMMs:
    // the map's bounds clip the M tail; batched layouts keep the guarded stores
    bool plain = p.batches == 1 && splits == 1 && aligned16_(p.c) && (p.ldc * 2) % 16 == 0;
    for (int w = 4; w < 6; ++w) plain = plain && p.off[w][0] == 0 && p.off[w][1] == 0;
    if (plain && !getenv_flag("TALLY_GEMM_NO_TMA_STORE")) {
      int rc = make_map(&p.a_lo, p.c, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, N, 32, p.ldc);
      if (rc) return rc;
      p.c_tma = 1;
    }
  }
  if constexpr (Cfg::KIND == 1 && Cfg::BN >= 128 && sizeof(typename Cfg::OutT) == 4) {
    // fp32 TMA-store epilogue: C seen as one 2-D [rows, ldc] fp32 map that
    // covers every split and batch origin; rows past M only where the map
    // clips them exactly (unsplit, unbatched), else M a multiple of the tile
    const long long tile_rows = (long long)Cfg::BM * gemm::PairOf<Cfg>::value;
    const long long ss_rows = p.ldc > 0 && p.split_stride % p.ldc == 0 ? p.split_stride / p.ldc : -1;
    // batch z = (z / hdiv, z % hdiv): origins are linear in both with
    // non-negative steps, so the largest indices bound every origin
    const long long zb_max = (p.batches - 1) / p.hdiv, zh_max = std::min(p.hdiv, p.batches) - 1;
    const long long max_r = p.off[4][0] * zb_max + p.off[4][1] * zh_max;
    const long long max_c = p.off[5][0] * zb_max + p.off[5][1] * zh_max;
    bool ok = aligned16_(p.c) && (p.ldc * 4) % 16 == 0 && ss_rows >= 0 && max_c + N <= p.ldc &&
              !getenv_flag("TALLY_GEMM_NO_TMA_STORE");
    for (int w = 4; w < 6; ++w) ok = ok && p.off[w][0] >= 0 && p.off[w][1] >= 0;
    const bool plain = splits == 1 && p.batches == 1 && max_r == 0;
    ok = ok && (plain || M % tile_rows == 0);
    if (ok) {
      const long long rows = plain ? M : (splits - 1) * ss_rows + max_r + M;
      int rc = make_map(&p.a_lo, p.c, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, rows, p.ldc, 32, p.ldc);
      if (rc) return rc;
      p.c_tma = 2;
    }
  }
  // fused linear-layer epilogue: ptr[4] bias (fp32 [N]), ptr[5] residual (bf16,
  // pitch ldc), ptr[6] pre-activation output (bf16, pitch ldc); i[6] activation
  if (!split && (a->ptr[4] || a->ptr[5] || a->ptr[6] || a->i[6])) {
    if (Cfg::KIND != 1 || sizeof(typename Cfg::OutT) != 2 || !p.c_tma || a->i[6] < 0 || a->i[6] > 3 ||
        (a->ptr[4] && !aligned16_(a->ptr[4])) || (a->ptr[5] && !aligned16_(a->ptr[5]))) {
      set_error("gemm: a fused epilogue (bias, residual, pre, act) needs a plain bf16 GEMM with the TMA-store "
                "epilogue, 16-byte aligned fp32 bias / residual, act 0-3");
      return TALLY_EINVAL;
    }
    p.ep.on = 1;
    p.ep.bias = static_cast<const float*>(a->ptr[4]);
    p.ep.res = static_cast<const __nv_bfloat16*>(a->ptr[5]);
    p.ep.ldr = p.ldc;
    p.ep.act = (int)a->i[6];
    if (a->ptr[6]) {
      if (!aligned16_(a->ptr[6])) { set_error("gemm: pre-activation output not 16-byte aligned"); return TALLY_EINVAL; }
      int rc = make_map(&p.b_lo, a->ptr[6], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, N, 32, p.ldc);
      if (rc) return rc;
      p.ep_pre = 1;
    }
    inst->alg_bytes_extra_ep = (a->ptr[4] ? 4.0 * N : 0.0) + (a->ptr[5] ? 2.0 * M * N : 0.0) + (a->ptr[6] ? 2.0 * M * N : 0.0);
  }
  // fused batch-norm statistics of the bf16 output: ptr[7] (tally_bn_stats)
  if (a->ptr[7] != nullptr) {
    const tally_bn_stats* bs = static_cast<const tally_bn_stats*>(a->ptr[7]);
    bool plain = p.batches == 1;
    for (int w = 4; w < 6; ++w) plain = plain && p.off[w][0] == 0 && p.off[w][1] == 0;
    const bool path = Cfg::BN == 64 ? true : p.c_tma == 1;
    if (Cfg::KIND != 1 || sizeof(typename Cfg::OutT) != 2 || split || !plain || !path || p.ldc != N || N % 64 ||
        !bs->part) {
      set_error("gemm: fused batch-norm statistics need a plain unsplit bf16 GEMM / convolution ([M, N] output, "
                "N %% 64 == 0, TMA-store epilogue for 128/256-wide tiles) and the part scratch");
      return TALLY_EINVAL;
    }
    p.bnf.C = (int)N;
    p.bnf.rows32 = bs->rb == 32;
    p.bnf.nrows = (int)(p.bnf.rows32 ? (M + 127) / 128 * 4 : (M + 127) / 128);
    p.bnf.part = bs->part;
    p.bnf.dbg = getenv("TALLY_BNFUSE_DBG") ? atoi(getenv("TALLY_BNFUSE_DBG")) : 0;
    inst->alg_bytes_extra_ep += 8.0 * p.bnf.nrows * N;   // the partial rows
  }
  p.kb_per_split = (int)((KBlocks + splits - 1) / splits);
  if ((KBlocks + p.kb_per_split - 1) / p.kb_per_split != splits) {
    set_error("gemm: %lld splits of %lld k-blocks leave an empty split (use ceil(KB / ceil(KB / splits)))",
              splits, KBlocks);
    return TALLY_EINVAL;
  }
  // fp32 promotion + preemption point every 256 of K for the fp32-accuracy
  // kernel (16 chunks of ~4.5 us per 4096-deep tile); bf16 (1e-2 budget)
  // accumulates the whole K in TMEM
  p.kchunk = Cfg::KIND == 0 ? 256 / Cfg::BK : p.kb_per_split;
  // short-K tiles (<= 2 k-blocks, ~1 us each): 4 tiles per logical block, so
  // an untransformed CTA pipelines 4 tiles behind one prologue and a PTB
  // claim covers ~4 us of work; longer tiles are one logical block each
  {
    static const int target = [] {
      const char* e = getenv("TALLY_GEMM_BLOCK_KB");   // experiment knob: k-blocks per logical block
      return e ? atoi(e) : 8;
    }();
    static const int old_rule = getenv("TALLY_GEMM_TPB_OLD") != nullptr;
    // ... and at most ~128 KB of output per logical block (fp32 128 x 128
    // tiles: 2 per block) -- a K = 64 fp32 score GEMM at 8 tiles per block
    // had ~30 us logical blocks (preemption latency)
    constexpr int kTileOut = Cfg::BM * Cfg::BN * (int)sizeof(typename Cfg::OutT);   // per CTA
    p.tpb = Cfg::KIND != 1 ? 1
          : old_rule ? (p.kb_per_split <= 2 ? 4 : 1)
                     : max(1, min(min(8, (131072 + kTileOut - 1) / kTileOut),
                                  (target + p.kb_per_split - 1) / p.kb_per_split));
    if constexpr (gemm::PairOf<Cfg>::value == 2) {
      // pairs: one CTA per SM, so an untransformed launch pays a CTA's
      // prologue and its last epilogue per logical block; with many tiles, a
      // block of ~32 k-blocks (2 tiles at K = 1024) overlaps the first tile's
      // epilogue with the second's MMAs (BERT-large decoder: 282 us as one
      // tile per cluster vs 196 us persistent) while leaving >= 2 blocks per pair
      const long long tiles_all = (long long)p.tiles_m * p.tiles_n * p.splits * p.batches;
      p.tpb = (int)std::max(1ll, std::min<long long>({4ll, (32 + p.kb_per_split - 1) / p.kb_per_split, tiles_all / 148}));
      // (Whole waves of the 74 pairs for short-K tiles -- tpb = ceil(tiles /
      // (74 w)) -- ran ResNet-50's 1x1 convolutions 10-30 % faster untransformed,
      // but longer blocks cost the tuner's PTB choices more: C2 step chosen /
      // untransformed 0.879 -> 0.864 (w >= 2), 0.78 (w >= 1; it sliced them).)
    }
  }
  p.total_tiles = (long long)p.tiles_m * p.tiles_n * p.splits * p.batches;
  if (p.total_tiles >= (1ll << 31)) {
    set_error("gemm: %lld tiles (>= 2^31)", p.total_tiles);
    return TALLY_EINVAL;
  }
  p.resume = nullptr;
  // i[3] = 1: block-granular preemption only (no resume ring)
  if (Cfg::KIND == 0 && a->i[3] == 0) {
    const size_t bytes = (2 + kResumeCap) * sizeof(unsigned long long);
    cudaError_t e = cudaMalloc(&p.resume, bytes);
    if (e == cudaSuccess) e = cudaMemset(p.resume, 0, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "gemm resume ring");
    inst->resume_ring = p.resume;
    inst->resume_bytes = bytes;
    inst->preempt_units = (int)((K / Cfg::BK + p.kchunk - 1) / p.kchunk);
  }
  static_assert(sizeof(p) <= kMaxParamBytes, "params too large");
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)((p.total_tiles + p.tpb - 1) / p.tpb), 1, 1);
  inst->threads = gemm::kThreads;
  inst->smem = gemm::smem_bytes<Cfg>();
  inst->alg_flops = 2.0 * (double)M * (double)N * (double)K * (double)p.batches;
  inst->alg_bytes = ((double)Cfg::ESZ * (double)(M * K + N * K) * (split ? 2.0 : 1.0) +
                     (double)sizeof(typename Cfg::OutT) * (double)(M * N) * (double)splits) * (double)p.batches +
                    inst->alg_bytes_extra_ep;
  if (p.causal) {
    // the work actually done: k-blocks over all tiles of one batch under the rule
    const long long KBt = (K + Cfg::BK - 1) / Cfg::BK;
    double done = 0.0, full = (double)p.tiles_m * p.tiles_n * KBt;
    for (int mb = 0; mb < p.tiles_m; ++mb)
      for (int nb = 0; nb < p.tiles_n; ++nb) {
        long long kb0 = 0, kb1 = KBt;
        if (p.causal == 1 && nb * Cfg::BN >= (mb + 1) * 128) kb1 = 0;
        if (p.causal == 2) kb1 = std::min(kb1, (long long)(((mb + 1) * 128 + Cfg::BK - 1) / Cfg::BK));
        if (p.causal == 3) kb0 = std::max(kb0, (long long)((mb * 128) / Cfg::BK));
        done += (double)std::max(0ll, kb1 - kb0);
      }
    inst->alg_flops *= done / full;
    inst->alg_bytes *= done / full;
  }
  return TALLY_OK;
}

static int bind_sgemm(const tally_kernel_args* a, Instance* inst) { return bind_gemm<gemm::CfgTf32x3>(a, inst, true); }
static int bind_sgemm_n64(const tally_kernel_args* a, Instance* inst) {
  return bind_gemm<gemm::CfgTf32x3N64>(a, inst, true);
}
template <class Cfg>
static int bind_bf16(const tally_kernel_args* a, Instance* inst) { return bind_gemm<Cfg>(a, inst, false); }

template <class Cfg>
static int setup_gemm() {
  const int smem = (int)gemm::smem_bytes<Cfg>();
  const void* fns[3] = {reinterpret_cast<const void*>(&gemm::k_gemm<Cfg, gemm::kOriginal, SliceArgs>),
                        reinterpret_cast<const void*>(&gemm::k_gemm<Cfg, gemm::kSliced, SliceArgs>),
                        reinterpret_cast<const void*>(&gemm::k_gemm<Cfg, gemm::kPtb, PtbArgs>)};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // the whole carveout as shared memory: two bf16 GEMM CTAs (~100 KB each)
    // share an SM -- the occupancy the tuner's PTB worker menu is built from
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return cuda_fail(e, "gemm smem attribute");
  }
  return TALLY_OK;
}

static int bind_split(const tally_kernel_args* a, Instance* inst) {
  gemm::SplitTf32::Params p{};
  p.x = static_cast<const float4*>(a->ptr[0]);
  p.hi = static_cast<float4*>(a->ptr[1]);
  p.lo = static_cast<float4*>(a->ptr[2]);
  const long long n = a->i[0];
  if (!p.x || !p.hi || !p.lo || n < 4 || n % 4) {
    set_error("split_tf32: need x, hi, lo and n %% 4 == 0");
    return TALLY_EINVAL;
  }
  p.n4 = n / 4;
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)((n + gemm::SplitTf32::kElemsPerBlock - 1) / gemm::SplitTf32::kElemsPerBlock), 1, 1);
  inst->threads = gemm::SplitTf32::kThreads;
  inst->smem = 0;
  inst->alg_bytes = 12.0 * (double)n;
  return TALLY_OK;
}

template <class Cfg>
static KernelKind gemm_kind(const char* name, int (*bind)(const tally_kernel_args*, Instance*)) {
  KernelKind k{};
  k.name = name;
  k.fn_original = reinterpret_cast<const void*>(&gemm::k_gemm<Cfg, gemm::kOriginal, SliceArgs>);
  k.fn_sliced = reinterpret_cast<const void*>(&gemm::k_gemm<Cfg, gemm::kSliced, SliceArgs>);
  k.fn_ptb = reinterpret_cast<const void*>(&gemm::k_gemm<Cfg, gemm::kPtb, PtbArgs>);
  k.bind = bind;
  k.setup = &setup_gemm<Cfg>;
  k.pausable = 1;
  k.tmem_cols = Cfg::TMEM_COLS;
  k.cluster = gemm::PairOf<Cfg>::value;   // CTA pairs launch as clusters of two
  k.ret_ring = Cfg::KIND == 1;            // claim-ahead workers (bf16 kinds)
  // device-resident flag: producers poll it every K-chunk (~9 us) -- 148
  // readers x 110 k reads/s would saturate PCIe reads of a mapped host word
  k.host_flag = 0;
  return k;
}

// ptr: A operand tensor (Q or dO), B operand tensor (K or V), out (P / dS),
// [MODE 1: P in].  i: B, H, T, a_rows_ld (row pitch of A's tensor), b_ld,
// a_col0, b_col0 (column origin of head 0; head h at + h * 64).  f: scale.
template <int MODE>
static int bind_attn_softmax(const tally_kernel_args* a, Instance* inst) {
  using Body = gemm::AttnSoftmax<MODE>;
  typename Body::Params p;
  memset(&p, 0, sizeof(p));
  const long long B = a->i[0], H = a->i[1], T = a->i[2], lda = a->i[3], ldb = a->i[4];
  p.a_col0 = a->i[5];
  p.b_col0 = a->i[6];
  p.a_col_h = p.b_col_h = Body::kD;
  p.T = (int)T;
  p.H = (int)H;
  p.scale = (float)a->f[0];
  if (!a->ptr[0] || !a->ptr[1] || !a->ptr[2] || (MODE == 1 && !a->ptr[3]) || B < 1 || H < 1 || T < 128 ||
      T > 512 || T % 128 || lda % 8 || ldb % 8 || p.a_col0 + H * Body::kD > lda || p.b_col0 + H * Body::kD > ldb) {
    set_error("attn_softmax: need A, B, out (and P), T in 128..512 (multiple of 128), head dim 64, "
              "column slices inside the row pitch");
    return TALLY_EINVAL;
  }
  int rc;
  if ((rc = make_map(&p.a_map, a->ptr[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B * T, lda, 128, lda))) return rc;
  if ((rc = make_map(&p.b_map, a->ptr[1], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B * T, ldb, 128, ldb))) return rc;
  if ((rc = make_map(&p.out_map, a->ptr[2], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B * H * T, T, 32, T))) return rc;
  p.p_in = static_cast<const __nv_bfloat16*>(a->ptr[3]);
  if (MODE == 1 && (rc = make_map(&p.p_map, a->ptr[3], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B * H * T, T, 128, T))) return rc;
  static_assert(sizeof(p) <= kMaxParamBytes, "params too large");
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)(T / 128), (unsigned)(B * H), 1);
  inst->threads = Body::kThreads;
  inst->smem = Body::kSmem;
  inst->alg_flops = 2.0 * (double)B * H * T * T * Body::kD;
  // Q / dO and K / V once per block row, P / dS written (MODE 1: P read)
  inst->alg_bytes = (double)B * H * T * Body::kD * 2.0 * (1.0 + T / 128.0) + (double)B * H * T * T * 2.0 * (MODE ? 2.0 : 1.0);
  return TALLY_OK;
}

template <int MODE>
static int setup_attn_softmax() {
  using Body = gemm::AttnSoftmax<MODE>;
  const void* fns[3] = {reinterpret_cast<const void*>(&k_original<Body>), reinterpret_cast<const void*>(&k_sliced<Body>),
                        reinterpret_cast<const void*>(&k_ptb<Body>)};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, Body::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return cuda_fail(e, "attn_softmax smem attribute");
  }
  return TALLY_OK;
}

template <int MODE>
static KernelKind attn_kind(const char* name) {
  using Body = gemm::AttnSoftmax<MODE>;
  KernelKind k{};
  k.name = name;
  k.fn_original = reinterpret_cast<const void*>(&k_original<Body>);
  k.fn_sliced = reinterpret_cast<const void*>(&k_sliced<Body>);
  k.fn_ptb = reinterpret_cast<const void*>(&k_ptb<Body>);
  k.bind = bind_attn_softmax<MODE>;
  k.setup = setup_attn_softmax<MODE>;
  k.tmem_cols = 512;
  k.ret_ring = 1;   // generic k_ptb workers: return ring and static first blocks
  return k;
}

int register_gemm_kernels(KernelKind* out, int cap) {
  if (cap < 30) return 0;
  out[0] = gemm_kind<gemm::CfgTf32x3>("sgemm_tf32x3", bind_sgemm);
  out[1] = gemm_kind<gemm::CfgBf16>("gemm_bf16", bind_bf16<gemm::CfgBf16>);
  out[3] = gemm_kind<gemm::CfgTf32x3N64>("sgemm_tf32x3_n64", bind_sgemm_n64);
  out[4] = gemm_kind<gemm::CfgBf16N64>("gemm_bf16_n64", bind_bf16<gemm::CfgBf16N64>);
  out[5] = gemm_kind<gemm::CfgBf16F32>("gemm_bf16f32", bind_bf16<gemm::CfgBf16F32>);
  out[6] = gemm_kind<gemm::CfgBf16F32N64>("gemm_bf16f32_n64", bind_bf16<gemm::CfgBf16F32N64>);
  out[7] = gemm_kind<gemm::CfgBf16MN>("gemm_bf16f32_mn", bind_bf16<gemm::CfgBf16MN>);
  out[8] = gemm_kind<gemm::CfgBf16MNN64>("gemm_bf16f32_mn_n64", bind_bf16<gemm::CfgBf16MNN64>);
  out[9] = gemm_kind<gemm::CfgBf16KMN>("gemm_bf16_kmn", bind_bf16<gemm::CfgBf16KMN>);
  out[10] = gemm_kind<gemm::CfgBf16KMNN64>("gemm_bf16_kmn_n64", bind_bf16<gemm::CfgBf16KMNN64>);
  out[11] = gemm_kind<gemm::CfgBf16F32KMN>("gemm_bf16f32_kmn", bind_bf16<gemm::CfgBf16F32KMN>);
  out[12] = gemm_kind<gemm::CfgBf16F32KMNN64>("gemm_bf16f32_kmn_n64", bind_bf16<gemm::CfgBf16F32KMNN64>);
  out[13] = gemm_kind<gemm::CfgBf16MNb>("gemm_bf16_mn", bind_bf16<gemm::CfgBf16MNb>);
  out[14] = gemm_kind<gemm::CfgBf16MNbN64>("gemm_bf16_mn_n64", bind_bf16<gemm::CfgBf16MNbN64>);
  out[15] = gemm_kind<gemm::CfgBf16X2>("gemm_bf16_x2", bind_bf16<gemm::CfgBf16X2>);
  out[16] = gemm_kind<gemm::CfgBf16F32X2>("gemm_bf16f32_x2", bind_bf16<gemm::CfgBf16F32X2>);
  out[17] = gemm_kind<gemm::CfgBf16MNX2>("gemm_bf16f32_mn_x2", bind_bf16<gemm::CfgBf16MNX2>);
  out[18] = gemm_kind<gemm::CfgBf16KMNX2>("gemm_bf16_kmn_x2", bind_bf16<gemm::CfgBf16KMNX2>);
  out[19] = gemm_kind<gemm::CfgBf16F32KMNX2>("gemm_bf16f32_kmn_x2", bind_bf16<gemm::CfgBf16F32KMNX2>);
  KernelKind k{};
  k.name = "split_tf32";
  k.fn_original = reinterpret_cast<const void*>(&k_original<gemm::SplitTf32>);
  k.fn_sliced = reinterpret_cast<const void*>(&k_sliced<gemm::SplitTf32>);
  k.fn_ptb = reinterpret_cast<const void*>(&k_ptb<gemm::SplitTf32>);
  k.bind = bind_split;
  out[2] = k;
  out[20] = attn_kind<0>("attn_softmax");
  out[21] = attn_kind<1>("attn_softmax_bwd");
  out[22] = gemm_kind<gemm::CfgConvF>("conv_fprop_bf16", bind_bf16<gemm::CfgConvF>);
  out[23] = gemm_kind<gemm::CfgConvFN64>("conv_fprop_bf16_n64", bind_bf16<gemm::CfgConvFN64>);
  out[24] = gemm_kind<gemm::CfgConvF32>("conv_fprop_bf16f32", bind_bf16<gemm::CfgConvF32>);
  out[25] = gemm_kind<gemm::CfgConvF32N64>("conv_fprop_bf16f32_n64", bind_bf16<gemm::CfgConvF32N64>);
  out[26] = gemm_kind<gemm::CfgConvW>("conv_wgrad_bf16f32", bind_bf16<gemm::CfgConvW>);
  out[27] = gemm_kind<gemm::CfgConvWN64>("conv_wgrad_bf16f32_n64", bind_bf16<gemm::CfgConvWN64>);
  out[28] = gemm_kind<gemm::CfgConvFC8>("conv_fprop_c8_bf16_n64", bind_bf16<gemm::CfgConvFC8>);
  out[29] = gemm_kind<gemm::CfgConvWC8>("conv_wgrad_c8_bf16f32_n64", bind_bf16<gemm::CfgConvWC8>);
  return 30;
}

}  // namespace tally
