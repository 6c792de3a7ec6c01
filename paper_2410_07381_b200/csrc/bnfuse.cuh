// Batch-norm statistics fused into the producer of the normalised tensor
// (training forward): the tcgen05 GEMM / implicit-GEMM convolution epilogue
// sums every 64-column box of its bf16 output tile -- s1 = sum y, s2 = sum
// y^2 over the tile's 128 rows, from the staged (stored) bf16 values -- into
// one partial row [2][ceil(M / 128)][C]; the "bn_fold" kind (bn_stats mode 4,
// ~1/32 of the activation's bytes) turns the partial rows into mean, invstd
// and the bn_act scale / shift.  Same arithmetic as bn_stats mode 0 on the
// same values, without re-reading the activation from HBM.
//
// A "unit" is the four epilogue warps that drain one 64-column box of a
// 128-row tile (one warp per TMEM lane quarter, 32 rows each).  Sums are in
// a fixed order: results are bit-identical across launch shapes.  No
// counters or folds in the GEMM: an L2 atomic round trip per tile stalled
// the epilogue of short-K tiles (C2 step +0.3 ms).
#pragma once
#include <cuda_bf16.h>

namespace tally {

struct BnFuse {
  float* part;   // [2][nrows][C] per-tile (or per-warp) column sums (null: off)
  int nrows, C;
  int rows32;    // 1: one partial row per warp (32 output rows), no exchange
  int dbg;       // experiment knob (TALLY_BNFUSE_DBG): 2 no column sums
};

// named barrier over one unit (4 warps)
__device__ __forceinline__ void unit_bar(int id) {
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}

// Column sums of a warp's staged 32 x 64 bf16 box (shared address `stage`:
// row r at r * 128 bytes, 16-byte chunk j at (j ^ (r & 7)) * 16): lane l sums
// columns 2l and 2l + 1 over the rows < nvalid -- one conflict-free 128-byte
// row per ld.shared (register + immediate address), packed fp32 pairs
// (FADD2 / FFMA2) in two chains (even / odd rows).  The epilogue of short-K
// tiles is the kernel's critical path: generic loads with 64-bit address
// arithmetic made this ~600 instructions per box (ncu), now ~5 per row.
__device__ __forceinline__ void bn_colsum_row(uint32_t addr, unsigned long long& s, unsigned long long& q) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  unsigned long long xy;   // (bf16 lo, bf16 hi) -> (fp32, fp32)
  asm("mov.b64 %0, {%1, %2};" : "=l"(xy) : "r"(v << 16), "r"(v & 0xffff0000u));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(s) : "l"(xy));
  asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(q) : "l"(xy));
}

__device__ __forceinline__ float4 bn_box_colsum(uint32_t stage, int lane, int nvalid) {
  unsigned long long s[2] = {0ull, 0ull}, q[2] = {0ull, 0ull};
  const uint32_t chunk = (uint32_t)lane >> 2, wo = ((uint32_t)lane & 3u) * 4u;
  uint32_t o[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) o[c] = stage + (((chunk ^ (uint32_t)c) << 4) | wo);
  if (nvalid >= 32) {
#pragma unroll
    for (int r = 0; r < 32; ++r) bn_colsum_row(o[r & 7] + r * 128, s[r & 1], q[r & 1]);
  } else {
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (r < nvalid) bn_colsum_row(o[r & 7] + r * 128, s[r & 1], q[r & 1]);
  }
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(s[0]) : "l"(s[1]));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(q[0]) : "l"(q[1]));
  float4 o4;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o4.x), "=f"(o4.y) : "l"(s[0]));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o4.z), "=f"(o4.w) : "l"(q[0]));
  return o4;
}

// One unit's 64-column box of partial row `prow` (columns [c0, c0 + 64)):
// the four warps' column sums are combined through shared memory (`xs` =
// the unit's four exchange areas of >= 512 bytes, xs_stride floats apart,
// each warp's own area free to overwrite) in slot order and the partial row
// written.  Called by all 128 threads of the unit (slot = the warp's index).
__device__ __forceinline__ void bn_fuse_box(const BnFuse& b, float4 cs, int prow, int c0, int slot, int lane,
                                            float* xs, int xs_stride, int bar_id) {
  if (b.rows32) {
    // per-warp partial row 4 * prow + slot: lane l holds columns 2l, 2l + 1
    const long long row = 4ll * prow + slot;
    reinterpret_cast<float2*>(b.part + row * b.C + c0)[lane] = make_float2(cs.x, cs.y);
    reinterpret_cast<float2*>(b.part + ((long long)b.nrows + row) * b.C + c0)[lane] = make_float2(cs.z, cs.w);
    return;
  }
  reinterpret_cast<float4*>(xs + slot * xs_stride)[lane] = cs;
  unit_bar(bar_id);
  const int tid = slot * 32 + lane;
  const int st = tid >> 6, col = tid & 63;
  float v = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) v += xs[k * xs_stride + (col >> 1) * 4 + st * 2 + (col & 1)];
  b.part[((long long)st * b.nrows + prow) * b.C + c0 + col] = v;
  unit_bar(bar_id);   // the exchange areas are free again
}

}  // namespace tally
