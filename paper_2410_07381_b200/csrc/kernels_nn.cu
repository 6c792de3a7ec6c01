// Best-effort training kernels (config C2: ResNet-50 training, BASELINE.json
// configs[1]) in the three Tally launch shapes -- the "coalesced/vectorised
// elementwise and reduction kernels" of the north star.  The dense
// contractions (convolutions as GEMMs, the classifier) run on the tcgen05
// GEMM kinds in kernels_gemm.cu.
//
// Layout: activations are NHWC bf16, i.e. a [P = N*H*W, C] row-major matrix;
// every kernel moves 16 B (8 x bf16) vectors and needs C % 8 == 0 (the input
// image is stored with 8 channels, 3 real + 5 zero).  Reductions are
// deterministic (fixed per-block partials, fixed-order finalisation), so every
// launch shape produces bit-identical results.
//
//   im2col_bf16     x[N,H,W,C] -> col[N*OH*OW, Kp], k = (kh*KW + kw)*C + c, zero pad
//   col2im_bf16     dcol -> dx (gather form: each input vector sums the col
//                   entries it fed), fp32 accumulation
//   transpose_bf16  [R, C] -> [C, R], 64x64 tiles through shared memory
//   bn_stats        per-(row block, channel) partial sums: mode 0 (x, x^2),
//                   mode 1 (dz, dz*xhat) with dz = (g [+ g2]) * (y > 0)
//   bn_finalize     partials -> mean/invstd/scale/shift (mode 0) or
//                   dgamma/dbeta and the backward coefficients (mode 1)
//   bn_act          y = act(x*scale + shift [+ residual])
//   bn_bwd          dx = gamma*invstd*(dz - k1 - xhat*k2), optional dz output
//   maxpool_fwd/bwd 3x3 stride 2 pad 1 with an argmax byte per output element
//   avgpool_fwd/bwd global average pool [N, HW, C] <-> [N, C]
//   softmax_xent    logits(+bias) -> per-row loss, dlogits (bf16 and fp32)
//   sgd_update      momentum SGD over a table of parameter segments; sums
//                   split-K gradient partials; refreshes the bf16 weight
//                   copies (row-major and transposed) the GEMMs read
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "epilogue.cuh"
#include "registry.h"

namespace tally {

namespace nn {

__device__ __forceinline__ void unpack8(const uint4 v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 v;
  uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return v;
}

// Best-effort traffic is L2 evict-first: the training job streams gigabytes
// per step, and evict-first lines are replaced before the evict-normal lines
// of a co-located high-priority request (its weights and activations), which
// otherwise come back cold after every best-effort burst.
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint4 ld16(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(l2_evict_first()));
  return v;
}

__device__ __forceinline__ void st16(uint4* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(l2_evict_first()) : "memory");
}

// Logical blocks are small (16 KB of bf16 for the elementwise kinds) so that a
// kernel has many more of them than PTB workers: Eq. 1's turnaround estimate
// (latency x workers / blocks) stays under the threshold with full-occupancy
// worker counts.  Each thread keeps kIlp 16-byte loads in flight.
constexpr int kIlp = 4;
constexpr int kVecPerBlock = 256 * kIlp;
constexpr int kCol2ImVec = 256;   // col2im gathers up to KH*KW vectors per output vector

// ---------------------------------------------------------------- im2col
struct Geometry {
  int N, H, W, C;        // input
  int KH, KW, stride, pad;
  int OH, OW;            // output spatial
  int K, Kp;             // K = KH*KW*C, Kp = K rounded up to 64
};

struct Im2Col {
  // Index math once per block, not per vector: the block's output rows
  // (n, oh, ow) and the column vectors (kh, kw, c) are decoded into two
  // shared-memory tables first (32-bit divisions), then every thread streams
  // 16 B vectors with one division per vector.  (Per-vector 64-bit divisions
  // made the kernel instruction-bound at ~2 TB/s.)
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 4;   // register cap: 4+ resident CTAs per SM
  static constexpr int kVecs = 2 * kVecPerBlock;       // 2048 vectors per logical block (amortises the tables)
  static constexpr int kMaxRows = kVecs / 8;           // rpb <= 2048 / kv, kv >= 8
  static constexpr int kMaxKv = 1024;
  static constexpr int kSmem = kMaxRows * 16 + kMaxKv * 4;
  struct Params {
    const uint4* x;
    uint4* col;
    Geometry g;
    long long rows;   // N*OH*OW
    int rpb;          // output rows per logical block
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char* smem) {
    const Geometry& g = p.g;
    const unsigned kv = (unsigned)(g.Kp >> 3);
    const int cv = g.C >> 3;
    const long long r0 = (long long)bidx.x * p.rpb;
    const int nrow = (int)min((long long)p.rpb, p.rows - r0);
    int4* rowt = reinterpret_cast<int4*>(smem);                       // {pixel base, ih0, iw0, -}
    int* colt = reinterpret_cast<int*>(smem + kMaxRows * 16);         // kh | kw << 8 | c8 << 16, or -1
    for (int rr = threadIdx.x; rr < nrow; rr += kThreads) {
      const unsigned r = (unsigned)(r0 + rr);
      const unsigned t = r / (unsigned)g.OW, ow = r - t * (unsigned)g.OW;
      const unsigned n = t / (unsigned)g.OH, oh = t - n * (unsigned)g.OH;
      rowt[rr] = make_int4((int)n * g.H, (int)oh * g.stride - g.pad, (int)ow * g.stride - g.pad, 0);
    }
    const unsigned kwc = (unsigned)(g.KW * g.C);
    for (unsigned j = threadIdx.x; j < kv; j += kThreads) {
      const unsigned k = j << 3;
      int e = -1;
      if (k < (unsigned)g.K) {
        const unsigned kh = k / kwc, rem = k - kh * kwc;
        const unsigned kw = rem / (unsigned)g.C, c = rem - kw * (unsigned)g.C;
        e = (int)(kh | (kw << 8) | ((c >> 3) << 16));
      }
      colt[j] = e;
    }
    __syncthreads();
    const unsigned total = (unsigned)nrow * kv;
    uint4* dst0 = p.col + r0 * kv;
    for (unsigned i0 = 0; i0 < total; i0 += kThreads * kIlp) {
      uint4 v[kIlp];
#pragma unroll
      for (int u = 0; u < kIlp; ++u) {
        const unsigned i = i0 + u * kThreads + threadIdx.x;
        v[u] = make_uint4(0u, 0u, 0u, 0u);
        if (i < total) {
          const unsigned rr = i / kv, j = i - rr * kv;
          const int e = colt[j];
          if (e >= 0) {
            const int4 rw = rowt[rr];
            const int ih = rw.y + (e & 0xff), iw = rw.z + ((e >> 8) & 0xff);
            if (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W)
              v[u] = ld16(p.x + ((long long)(rw.x + ih) * g.W + iw) * cv + (e >> 16));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kIlp; ++u) {
        const unsigned i = i0 + u * kThreads + threadIdx.x;
        if (i < total) st16(dst0 + i, v[u]);
      }
    }
    __syncthreads();   // the tables are rebuilt by the next logical block of a PTB worker
  }
};

// ---------------------------------------------------------------- col2im (gather)
struct Col2Im {
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 4;   // register cap: 4+ resident CTAs per SM
  struct Params {
    const uint4* col;
    uint4* dx;
    Geometry g;
    long long nvec;   // N*H*W*C/8
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const Geometry& g = p.g;
    const int cv = g.C >> 3, kv = g.Kp >> 3;
    const long long v0 = (long long)bidx.x * kCol2ImVec;
    for (int i = threadIdx.x; i < kCol2ImVec; i += kThreads) {
      const long long v = v0 + i;
      if (v >= p.nvec) break;
      // 32-bit decode (nvec < 2^31, checked at bind time)
      const unsigned pix = (unsigned)v / (unsigned)cv;
      const int c8 = (int)((unsigned)v - pix * (unsigned)cv);
      const unsigned t = pix / (unsigned)g.W;
      const int iw = (int)(pix - t * (unsigned)g.W);
      const unsigned n_ = t / (unsigned)g.H;
      const int ih = (int)(t - n_ * (unsigned)g.H);
      const int n = (int)n_;
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int kh = 0; kh < g.KH; ++kh) {
        const int ohn = ih + g.pad - kh;
        if (ohn < 0 || ohn % g.stride) continue;
        const int oh = ohn / g.stride;
        if (oh >= g.OH) continue;
        for (int kw = 0; kw < g.KW; ++kw) {
          const int own = iw + g.pad - kw;
          if (own < 0 || own % g.stride) continue;
          const int ow = own / g.stride;
          if (ow >= g.OW) continue;
          const long long r = ((long long)n * g.OH + oh) * g.OW + ow;
          float f[8];
          unpack8(ld16(p.col + r * kv + ((kh * g.KW + kw) * cv + c8)), f);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] += f[e];
        }
      }
      st16(p.dx + v, pack8(acc));
    }
  }
};

// ---------------------------------------------------------------- transpose
struct Transpose {
  static constexpr int kThreads = 256;
  static constexpr int T = 64;
  struct Params {
    const unsigned short* src;
    unsigned short* dst;
    long long R, C;
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char* smem) {
    unsigned short* tile = reinterpret_cast<unsigned short*>(smem);   // [T][T + 2]
    const long long c0 = (long long)bidx.x * T, r0 = (long long)bidx.y * T;
    // rows of the source tile: 4 threads x 16 elements per 64-wide row
    for (int i = threadIdx.x; i < T * T; i += kThreads) {
      const int rr = i / T, cc = i % T;
      const long long r = r0 + rr, c = c0 + cc;
      tile[rr * (T + 2) + cc] = (r < p.R && c < p.C) ? p.src[r * p.C + c] : (unsigned short)0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < T * T; i += kThreads) {
      const int cc = i / T, rr = i % T;
      const long long r = r0 + rr, c = c0 + cc;
      if (r < p.R && c < p.C) p.dst[c * p.R + r] = tile[rr * (T + 2) + cc];
    }
    __syncthreads();   // the tile is reused by the next logical block of a PTB worker
  }
};

// ---------------------------------------------------------------- batch-norm statistics
// One kernel computes the per-channel statistics AND finalises them: each
// logical block (channel block cb, row block rb) writes its partial sums;
// the last block of every group of kGroup row blocks folds the group
// (fixed order) into a second-level partial; the last group of a channel
// block folds those and writes the channel outputs.  Deterministic (every sum
// has a fixed order), exactly-once under every launch shape (the counters
// count logical blocks, and survive a PTB park / resume), and no separate
// finalisation launch.
// MODE 0: forward statistics; 1: backward statistics (per-channel mean /
// invstd); 2: column sums over rows for LayerNorm / bias gradients -- s1 = sum g,
// s2 = sum g * (x - mean[row]) * rstd[row] (x optional), finalised as
// dbeta = s1, dgamma = s2.
// backward / column statistics: one row of 2-4 streams in flight per thread,
// three CTAs per SM (register cap 85) -- one CTA's fold / counter latency
// overlaps the others' streaming (bn_stats_bwd 2.07 -> 1.89 ms per C2 step;
// 4 CTAs at 64 registers spill)
#ifndef TALLY_BN_BWD_MINBLOCKS
#define TALLY_BN_BWD_MINBLOCKS 3
#endif
#ifndef TALLY_BN_BWD_ROWS
#define TALLY_BN_BWD_ROWS 2
#endif
#ifndef TALLY_COLSTATS_ROWS
#define TALLY_COLSTATS_ROWS 2
#endif
#ifndef TALLY_COLSTATS_MINBLOCKS
#define TALLY_COLSTATS_MINBLOCKS 3
#endif
template <int MODE>
struct BnStats {
  static constexpr int kThreads = 256;
  // (mode 2, column sums: four rows per thread in flight at two CTAs per SM
  // measured slower -- BERT-large step 22.88 -> 23.13 ms; TALLY_COLSTATS_ROWS /
  // _MINBLOCKS experiment knobs)
  static constexpr int kMinBlocks = MODE == 0 ? 4 : MODE >= 3 ? 3 : MODE == 2 ? TALLY_COLSTATS_MINBLOCKS : TALLY_BN_BWD_MINBLOCKS;
  static constexpr int kRows = MODE == 0 ? kIlp : MODE >= 3 ? 2 : MODE == 2 ? TALLY_COLSTATS_ROWS : TALLY_BN_BWD_ROWS;
  static constexpr int kGroup = 32;
  struct Params {
    const uint4* x;        // pre-BN activations [P, C]
    const uint4* g;        // mode 1: upstream gradient
    const uint4* g2;       // mode 1: optional second gradient term (residual)
    const uint4* y;        // mode 1: optional ReLU output (mask y > 0)
    float* mean;           // mode 0: output; mode 1: input
    float* invstd;         // mode 0: output; mode 1: input
    float* part;           // [2][nrb][C] level-1 partials
    float* part2;          // [2][ngroups][C] level-2 partials
    unsigned* cnt1;        // [cblocks][ngroups] finished row blocks per group
    unsigned* cnt2;        // [cblocks] finished groups
    const float* gamma;
    const float* beta;     // mode 0
    float* scale_shift;    // mode 0 output [2][C]: y = x*scale + shift
    float* dgamma;         // mode 1 outputs
    float* dbeta;
    float* coef;           // mode 1 output [3][C]: dx = ca*dz + cb*x + cc
    const float4* sk_in;   // mode 3: split-K fp32 partials [S][P][C]; mode 4: partial rows [2][P][C]
    uint4* sk_out;         // mode 3: their bf16 sum [P, C] (the statistics' input)
    long long sk_stride4;  // mode 3: P * C / 4
    int sk_S;
    long long P;
    int C, RB, nrb, ngroups, mode;
    float inv_count, eps;
  };

  // sum rows [r0, r1) of a [2][rows][C] partial array for this block's
  // channels into red (first 2*CB floats), using every thread: float4 column
  // lanes x 4-16 row lanes, 4 rows' loads of both arrays in flight per batch
  // (a 32-row group is 1-2 batches, not ~8 dependent L2 round trips), then
  // the row lanes added in order through shared memory (deterministic)
  static __device__ __forceinline__ void fold(const float* src, long long rows_total, int r0, int r1, int C,
                                              int c0, int CB, float* red, float* out_a, float* out_b) {
    const int cv4 = CB >> 2, lanes_r = kThreads / cv4;
    const int lc = threadIdx.x % cv4, lr = threadIdx.x / cv4;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    const float* pa = src + c0 + 4 * lc;
    const float* pb = src + rows_total * C + c0 + 4 * lc;
    for (int r = r0 + lr; r < r1; r += 4 * lanes_r) {
      float4 va[4], vb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = r + u * lanes_r;
        va[u] = rr < r1 ? __ldcg(reinterpret_cast<const float4*>(pa + (long long)rr * C)) : make_float4(0.f, 0.f, 0.f, 0.f);
        vb[u] = rr < r1 ? __ldcg(reinterpret_cast<const float4*>(pb + (long long)rr * C)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a.x += va[u].x; a.y += va[u].y; a.z += va[u].z; a.w += va[u].w;
        b.x += vb[u].x; b.y += vb[u].y; b.z += vb[u].z; b.w += vb[u].w;
      }
    }
    reinterpret_cast<float4*>(red + lr * CB)[lc] = a;
    reinterpret_cast<float4*>(red + 1024 + lr * CB)[lc] = b;
    __syncthreads();
    if (threadIdx.x < CB) {
      float sa = 0.f, sb = 0.f;
      for (int k = 0; k < lanes_r; ++k) { sa += red[k * CB + threadIdx.x]; sb += red[1024 + k * CB + threadIdx.x]; }
      *out_a = sa;
      *out_b = sb;
    }
    __syncthreads();
  }

  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char* smem) {
    const int CB = min(p.C, 256);
    const int cv = CB >> 3, rl = kThreads / cv;
    const int lane_c = threadIdx.x % cv, lane_r = threadIdx.x / cv;
    const int c0 = bidx.x * 256;
    const int c = c0 + lane_c * 8;
    const long long rbeg = (long long)bidx.y * p.RB;
    const long long rend = min(p.P, rbeg + p.RB);
    const int cvec = p.C >> 3;
    float s1[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, s2[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (long long r0 = rbeg + lane_r; r0 < rend; r0 += (long long)rl * kRows) {
      if constexpr (MODE == 4) {
        // mode 4 (bn_fold): rows are the fused epilogue's partial rows
        // (s1, s2 of 128 output rows each), summed in row order
        float4 t[kRows][4];
        bool ok[kRows];
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
          const long long r = r0 + (long long)u * rl;
          ok[u] = r < rend;
          if (ok[u]) {
            const float4* a = p.sk_in + ((r * p.C + c) >> 2);
            const float4* b = p.sk_in + (((p.P + r) * p.C + c) >> 2);
            t[u][0] = __ldcg(a);
            t[u][1] = __ldcg(a + 1);
            t[u][2] = __ldcg(b);
            t[u][3] = __ldcg(b + 1);
          }
        }
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
          if (!ok[u]) continue;
          s1[0] += t[u][0].x; s1[1] += t[u][0].y; s1[2] += t[u][0].z; s1[3] += t[u][0].w;
          s1[4] += t[u][1].x; s1[5] += t[u][1].y; s1[6] += t[u][1].z; s1[7] += t[u][1].w;
          s2[0] += t[u][2].x; s2[1] += t[u][2].y; s2[2] += t[u][2].z; s2[3] += t[u][2].w;
          s2[4] += t[u][3].x; s2[5] += t[u][3].y; s2[6] += t[u][3].z; s2[7] += t[u][3].w;
        }
        continue;
      }
      if constexpr (MODE == 3) {
        // mode 3 (splitk_reduce_bn): the split-K sum of kRows rows, two
        // partials' loads in flight per row, summed in split order (as
        // splitk_reduce), stored as bf16; the statistics of the stored values
        float v[kRows][8];
        bool ok[kRows];
        long long off[kRows];
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
          const long long r = r0 + (long long)u * rl;
          ok[u] = r < rend;
          off[u] = (r * p.C + c) >> 2;
#pragma unroll
          for (int e = 0; e < 8; ++e) v[u][e] = 0.f;
        }
        int sp = 0;
        for (; sp + 1 < p.sk_S; sp += 2) {
          float4 t[kRows][4];
#pragma unroll
          for (int u = 0; u < kRows; ++u) {
            if (ok[u]) {
              const float4* src = p.sk_in + sp * p.sk_stride4 + off[u];
              t[u][0] = __ldcs(src);
              t[u][1] = __ldcs(src + 1);
              t[u][2] = __ldcs(src + p.sk_stride4);
              t[u][3] = __ldcs(src + p.sk_stride4 + 1);
            }
          }
#pragma unroll
          for (int u = 0; u < kRows; ++u) {
            if (!ok[u]) continue;
            v[u][0] += t[u][0].x; v[u][1] += t[u][0].y; v[u][2] += t[u][0].z; v[u][3] += t[u][0].w;
            v[u][4] += t[u][1].x; v[u][5] += t[u][1].y; v[u][6] += t[u][1].z; v[u][7] += t[u][1].w;
            v[u][0] += t[u][2].x; v[u][1] += t[u][2].y; v[u][2] += t[u][2].z; v[u][3] += t[u][2].w;
            v[u][4] += t[u][3].x; v[u][5] += t[u][3].y; v[u][6] += t[u][3].z; v[u][7] += t[u][3].w;
          }
        }
        if (sp < p.sk_S) {
#pragma unroll
          for (int u = 0; u < kRows; ++u) {
            if (!ok[u]) continue;
            const float4* src = p.sk_in + sp * p.sk_stride4 + off[u];
            const float4 a = __ldcs(src), b = __ldcs(src + 1);
            v[u][0] += a.x; v[u][1] += a.y; v[u][2] += a.z; v[u][3] += a.w;
            v[u][4] += b.x; v[u][5] += b.y; v[u][6] += b.z; v[u][7] += b.w;
          }
        }
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
          if (!ok[u]) continue;
          const uint4 o = pack8(v[u]);
          st16(p.sk_out + (off[u] >> 1), o);
          float x[8];
          unpack8(o, x);
#pragma unroll
          for (int e = 0; e < 8; ++e) { s1[e] += x[e]; s2[e] += x[e] * x[e]; }
        }
        continue;
      }
      uint4 xv[kRows], gv[kRows], g2v[kRows], yv[kRows];
      bool ok[kRows];
#pragma unroll
      for (int u = 0; u < kRows; ++u) {
        const long long r = r0 + (long long)u * rl;
        ok[u] = r < rend;
        const long long off = r * cvec + (c >> 3);
        if (ok[u]) {
          if (MODE != 2 || p.x) xv[u] = ld16(p.x + off);
          if constexpr (MODE >= 1) {
            gv[u] = ld16(p.g + off);
            if (p.g2) g2v[u] = ld16(p.g2 + off);
            if (p.y) yv[u] = ld16(p.y + off);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kRows; ++u) {
        if (!ok[u]) continue;
        float x[8];
        if constexpr (MODE == 2) {
          float g[8];
          unpack8(gv[u], g);
          if (p.g2) {
            float t[8];
            unpack8(g2v[u], t);
#pragma unroll
            for (int e = 0; e < 8; ++e) g[e] += t[e];
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) s1[e] += g[e];
          if (p.x) {
            const long long r = r0 + (long long)u * rl;
            const float mr = p.mean[r], rr = p.invstd[r];
            unpack8(xv[u], x);
#pragma unroll
            for (int e = 0; e < 8; ++e) s2[e] += g[e] * ((x[e] - mr) * rr);
          }
          continue;
        }
        unpack8(xv[u], x);
        if constexpr (MODE == 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) { s1[e] += x[e]; s2[e] += x[e] * x[e]; }
        } else {
          float dz[8];
          unpack8(gv[u], dz);
          if (p.g2) {
            float t[8];
            unpack8(g2v[u], t);
#pragma unroll
            for (int e = 0; e < 8; ++e) dz[e] += t[e];
          }
          if (p.y) {
            float t[8];
            unpack8(yv[u], t);
#pragma unroll
            for (int e = 0; e < 8; ++e) dz[e] = t[e] > 0.f ? dz[e] : 0.f;
          }
#pragma unroll
          // raw sum dz * x: the per-channel (x - mean) * invstd is applied once
          // per block below (linear), freeing 16 registers for rows in flight
          for (int e = 0; e < 8; ++e) { s1[e] += dz[e]; s2[e] = fmaf(dz[e], x[e], s2[e]); }
        }
      }
    }
    float* red = reinterpret_cast<float*>(smem);   // [2][rl][CB] = 2 x 2048 floats
    unsigned* flag = reinterpret_cast<unsigned*>(smem + 2 * 2048 * sizeof(float));
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      red[lane_r * CB + lane_c * 8 + e] = s1[e];
      red[rl * CB + lane_r * CB + lane_c * 8 + e] = s2[e];
    }
    __syncthreads();
    if (threadIdx.x < CB) {
      float a = 0.f, b = 0.f;
      for (int k = 0; k < rl; ++k) { a += red[k * CB + threadIdx.x]; b += red[rl * CB + k * CB + threadIdx.x]; }
      const int ch = c0 + threadIdx.x;
      if constexpr (MODE == 1) b = p.invstd[ch] * fmaf(-p.mean[ch], a, b);   // sum dz * xhat
      p.part[(long long)bidx.y * p.C + ch] = a;
      p.part[((long long)p.nrb + bidx.y) * p.C + ch] = b;
    }
    // ---- level 1: the last row block of the group folds the group.
    // Barrier, then one thread's GPU-scope fence (cumulative over the CTA's
    // writes ordered before the barrier) + counter; its fence after the
    // counter orders the folder's reads after every other block's release.
    __syncthreads();
    const int gi = bidx.y / kGroup;
    if (threadIdx.x == 0) {
      const unsigned in_group = (unsigned)min(kGroup, p.nrb - gi * kGroup);
      // one acq_rel RMW: releases this block's partials (ordered before it
      // by the barrier), acquires the group's for the folder
      flag[0] = atom_add_acq_rel_gpu(&p.cnt1[bidx.x * p.ngroups + gi], 1u) + 1u == in_group;
    }
    __syncthreads();
    if (flag[0]) {
      float a = 0.f, b = 0.f;
      fold(p.part, p.nrb, gi * kGroup, min(p.nrb, (gi + 1) * kGroup), p.C, c0, CB, red, &a, &b);
      const bool single = p.ngroups == 1;   // one group: its folder finalises (no level 2)
      if (!single) {
        if (threadIdx.x < CB) {
          p.part2[(long long)gi * p.C + c0 + threadIdx.x] = a;
          p.part2[((long long)p.ngroups + gi) * p.C + c0 + threadIdx.x] = b;
        }
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        p.cnt1[bidx.x * p.ngroups + gi] = 0u;   // ready for the next launch
        flag[1] = single || atom_add_acq_rel_gpu(&p.cnt2[bidx.x], 1u) + 1u == (unsigned)p.ngroups;
      }
      __syncthreads();
      if (flag[1]) {
        // ---- level 2: the last group finalises this channel block
        if (!single) fold(p.part2, p.ngroups, 0, p.ngroups, p.C, c0, CB, red, &a, &b);
        if (threadIdx.x < CB) {
          const int ch = c0 + threadIdx.x;
          if constexpr (MODE == 0 || MODE >= 3) {
            const float m = a * p.inv_count;
            const float var = fmaxf(b * p.inv_count - m * m, 0.f);
            const float isd = rsqrtf(var + p.eps);
            p.mean[ch] = m;
            p.invstd[ch] = isd;
            const float sc = p.gamma[ch] * isd;
            p.scale_shift[ch] = sc;
            p.scale_shift[p.C + ch] = p.beta[ch] - m * sc;
          } else if constexpr (MODE == 2) {
            p.dbeta[ch] = a;
            if (p.dgamma) p.dgamma[ch] = b;
          } else {
            p.dbeta[ch] = a;
            p.dgamma[ch] = b;
            const float isd = p.invstd[ch];
            const float k1 = a * p.inv_count, k2 = b * p.inv_count;
            const float al = p.gamma[ch] * isd;
            p.coef[ch] = al;
            p.coef[p.C + ch] = -al * k2 * isd;
            p.coef[2 * p.C + ch] = al * (k2 * isd * p.mean[ch] - k1);
          }
        }
        if (threadIdx.x == 0 && !single) p.cnt2[bidx.x] = 0u;
      }
    }
    __syncthreads();
  }
};

struct BnFinalize {
  // 32 channels x 8 row lanes per logical block; each lane sums every 8th
  // partial row, then a fixed-order combine in shared memory (deterministic)
  static constexpr int kThreads = 256;
  struct Params {
    const float* part;   // [2][nrb][C]
    int nrb, C, mode;
    float inv_count, eps;
    const float* gamma;
    const float* beta;     // mode 0
    const float* mean;     // mode 1 inputs
    const float* invstd;
    float* o_mean;         // mode 0 outputs
    float* o_invstd;
    float* scale;
    float* shift;
    float* dgamma;         // mode 1 outputs: gradient slots and the
    float* dbeta;          //   bn_bwd coefficients dx = ca*dz + cb*x + cc
    float* ca;
    float* cb;
    float* cc;
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char* smem) {
    const int lane_c = threadIdx.x & 31, lane_r = threadIdx.x >> 5;
    const int c = bidx.x * 32 + lane_c;
    float a = 0.f, b = 0.f;
    if (c < p.C) {
      int k = lane_r;
      for (; k + 24 < p.nrb; k += 32) {
        float x0 = p.part[(long long)k * p.C + c], x1 = p.part[(long long)(k + 8) * p.C + c];
        float x2 = p.part[(long long)(k + 16) * p.C + c], x3 = p.part[(long long)(k + 24) * p.C + c];
        float y0 = p.part[((long long)p.nrb + k) * p.C + c], y1 = p.part[((long long)p.nrb + k + 8) * p.C + c];
        float y2 = p.part[((long long)p.nrb + k + 16) * p.C + c], y3 = p.part[((long long)p.nrb + k + 24) * p.C + c];
        a += ((x0 + x1) + (x2 + x3));
        b += ((y0 + y1) + (y2 + y3));
      }
      for (; k < p.nrb; k += 8) {
        a += p.part[(long long)k * p.C + c];
        b += p.part[((long long)p.nrb + k) * p.C + c];
      }
    }
    float* red = reinterpret_cast<float*>(smem);   // [2][8][32]
    red[lane_r * 32 + lane_c] = a;
    red[256 + lane_r * 32 + lane_c] = b;
    __syncthreads();
    if (lane_r == 0 && c < p.C) {
      a = 0.f;
      b = 0.f;
#pragma unroll
      for (int r = 0; r < 8; ++r) { a += red[r * 32 + lane_c]; b += red[256 + r * 32 + lane_c]; }
      if (p.mode == 0) {
        const float m = a * p.inv_count;
        const float var = fmaxf(b * p.inv_count - m * m, 0.f);
        const float is = rsqrtf(var + p.eps);
        p.o_mean[c] = m;
        p.o_invstd[c] = is;
        const float sc = p.gamma[c] * is;
        p.scale[c] = sc;
        p.shift[c] = p.beta[c] - m * sc;
      } else {
        p.dbeta[c] = a;
        p.dgamma[c] = b;
        const float is = p.invstd[c];
        const float k1 = a * p.inv_count, k2 = b * p.inv_count;
        const float al = p.gamma[c] * is;
        p.ca[c] = al;
        p.cb[c] = -al * k2 * is;
        p.cc[c] = al * (k2 * is * p.mean[c] - k1);
      }
    }
    __syncthreads();
  }
};

// ---------------------------------------------------------------- batch-norm apply
struct BnAct {
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 4;   // register cap: 4+ resident CTAs per SM
  struct Params {
    const uint4* x;
    const uint4* res;   // optional residual added before the activation
    uint4* y;
    const float* scale;   // optional (1)
    const float* shift;
    uint4* pre;           // optional: the pre-activation values (GELU backward input)
    long long nvec;
    int C, relu;          // activation: 0 none, 1 ReLU, 2 GELU (tanh approximation), 3 GELU (erf)
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    // (one body for every activation: a per-activation template switch was
    // no faster untransformed and made the PTB shape 0.71 -> 0.51x of it)
    const int cv = p.C >> 3;
    const long long v0 = (long long)bidx.x * kVecPerBlock + threadIdx.x;
    uint4 xv[kIlp], rv[kIlp];
#pragma unroll
    for (int u = 0; u < kIlp; ++u) {
      const long long v = v0 + u * kThreads;
      if (v < p.nvec) {
        xv[u] = ld16(p.x + v);
        if (p.res) rv[u] = ld16(p.res + v);
      }
    }
#pragma unroll
    for (int u = 0; u < kIlp; ++u) {
      const long long v = v0 + u * kThreads;
      if (v >= p.nvec) continue;
      const int c = (int)((unsigned)v % (unsigned)cv) << 3;   // (nvec < 2^31, checked at bind: 32-bit modulo)
      float x[8];
      unpack8(xv[u], x);
      const float4 h0 = __ldg(reinterpret_cast<const float4*>(p.shift + c));
      const float4 h1 = __ldg(reinterpret_cast<const float4*>(p.shift + c + 4));
      const float sh[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
      if (p.scale) {
        const float4 s0 = __ldg(reinterpret_cast<const float4*>(p.scale + c));
        const float4 s1 = __ldg(reinterpret_cast<const float4*>(p.scale + c + 4));
        const float sc[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = x[e] * sc[e] + sh[e];
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] += sh[e];
      }
      if (p.res) {
        float r[8];
        unpack8(rv[u], r);
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] += r[e];
      }
      if (p.pre) st16(p.pre + v, pack8(x));
      if (p.relu == 1) {
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = fmaxf(x[e], 0.f);
      } else if (p.relu == 2) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float u = 0.7978845608028654f * (x[e] + 0.044715f * x[e] * x[e] * x[e]);
          x[e] = 0.5f * x[e] * (1.f + tanhf(u));
        }
      } else if (p.relu == 3) {
#pragma unroll
        for (int e = 0; e < 8; e += 2) gelu_erf2(x[e], x[e + 1]);
      }
      st16(p.y + v, pack8(x));
    }
  }
};

__device__ __forceinline__ void ld8f(const float* p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p + 4));
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

struct BnBwd {
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 3;
  static constexpr int kV = 2;                 // vectors per thread (4 input streams each)
  static constexpr int kBlockVec = kThreads * kV;
  struct Params {
    const uint4* g;
    const uint4* g2;    // optional
    const uint4* y;     // optional ReLU mask source
    const uint4* x;
    const float* ca;    // dx = ca*dz + cb*x + cc (bn_finalize mode 1)
    const float* cb;
    const float* cc;
    uint4* dx;
    uint4* dz_out;      // optional: the masked upstream gradient (for the shortcut)
    long long nvec;
    int C;
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int cv = p.C >> 3;
    const long long v0 = (long long)bidx.x * kBlockVec + threadIdx.x;
    uint4 gv[kV], g2v[kV], yv[kV], xv[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const long long v = v0 + u * kThreads;
      if (v < p.nvec) {
        gv[u] = ld16(p.g + v);
        xv[u] = ld16(p.x + v);
        if (p.g2) g2v[u] = ld16(p.g2 + v);
        if (p.y) yv[u] = ld16(p.y + v);
      }
    }
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const long long v = v0 + u * kThreads;
      if (v >= p.nvec) continue;
      const int c = (int)((unsigned)v % (unsigned)cv) << 3;   // (nvec < 2^31, checked at bind: 32-bit modulo)
      float dz[8], x[8];
      unpack8(gv[u], dz);
      if (p.g2) {
        float t[8];
        unpack8(g2v[u], t);
#pragma unroll
        for (int e = 0; e < 8; ++e) dz[e] += t[e];
      }
      if (p.y) {
        float t[8];
        unpack8(yv[u], t);
#pragma unroll
        for (int e = 0; e < 8; ++e) dz[e] = t[e] > 0.f ? dz[e] : 0.f;
      }
      if (p.dz_out) st16(p.dz_out + v, pack8(dz));
      unpack8(xv[u], x);
      float a[8], b[8], k[8];
      ld8f(p.ca + c, a);
      ld8f(p.cb + c, b);
      ld8f(p.cc + c, k);
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = a[e] * dz[e] + (b[e] * x[e] + k[e]);
      st16(p.dx + v, pack8(o));
    }
  }
};

// ---------------------------------------------------------------- pooling
struct MaxPoolFwd {   // 3x3, stride 2, pad 1
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 4;   // register cap: 4+ resident CTAs per SM
  struct Params {
    const uint4* x;
    uint4* y;
    uint2* arg;       // argmax (0..8) per output element, 8 bytes per vector
    int N, H, W, C, OH, OW;
    long long nvec;   // N*OH*OW*C/8
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int cv = p.C >> 3;
    const long long v0 = (long long)bidx.x * kVecPerBlock;
    for (int i = threadIdx.x; i < kVecPerBlock; i += kThreads) {
      const long long v = v0 + i;
      if (v >= p.nvec) break;
      const int c8 = (int)(v % cv);
      const long long pix = v / cv;
      const int ow = (int)(pix % p.OW);
      const long long t = pix / p.OW;
      const int oh = (int)(t % p.OH), n = (int)(t / p.OH);
      float m[8];
      unsigned char a[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) { m[e] = -INFINITY; a[e] = 0; }
      for (int kh = 0; kh < 3; ++kh) {
        const int ih = oh * 2 - 1 + kh;
        if (ih < 0 || ih >= p.H) continue;
        for (int kw = 0; kw < 3; ++kw) {
          const int iw = ow * 2 - 1 + kw;
          if (iw < 0 || iw >= p.W) continue;
          float f[8];
          unpack8(ld16(p.x + (((long long)n * p.H + ih) * p.W + iw) * cv + c8), f);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (f[e] > m[e]) { m[e] = f[e]; a[e] = (unsigned char)(kh * 3 + kw); }
        }
      }
      st16(p.y + v, pack8(m));
      uint2 w;
      w.x = a[0] | (a[1] << 8) | (a[2] << 16) | ((unsigned)a[3] << 24);
      w.y = a[4] | (a[5] << 8) | (a[6] << 16) | ((unsigned)a[7] << 24);
      p.arg[v] = w;
    }
  }
};

struct MaxPoolBwd {
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 4;   // register cap: 4+ resident CTAs per SM
  struct Params {
    const uint4* dy;
    const uint4* dy2;   // optional second gradient term
    const uint2* arg;
    uint4* dx;
    int N, H, W, C, OH, OW;
    long long nvec;     // N*H*W*C/8
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int cv = p.C >> 3;
    const long long v0 = (long long)bidx.x * kVecPerBlock;
    for (int i = threadIdx.x; i < kVecPerBlock; i += kThreads) {
      const long long v = v0 + i;
      if (v >= p.nvec) break;
      const int c8 = (int)(v % cv);
      const long long pix = v / cv;
      const int iw = (int)(pix % p.W);
      const long long t = pix / p.W;
      const int ih = (int)(t % p.H), n = (int)(t / p.H);
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      // output rows whose window [2*oh - 1, 2*oh + 1] contains ih
      const int oh_lo = max(0, ih / 2), oh_hi = min(p.OH - 1, (ih + 1) / 2);
      const int ow_lo = max(0, iw / 2), ow_hi = min(p.OW - 1, (iw + 1) / 2);
      for (int oh = oh_lo; oh <= oh_hi; ++oh) {
        const int kh = ih - (oh * 2 - 1);
        if (kh < 0 || kh > 2) continue;
        for (int ow = ow_lo; ow <= ow_hi; ++ow) {
          const int kw = iw - (ow * 2 - 1);
          if (kw < 0 || kw > 2) continue;
          const long long o = (((long long)n * p.OH + oh) * p.OW + ow) * cv + c8;
          const uint2 w = p.arg[o];
          const unsigned char* a = reinterpret_cast<const unsigned char*>(&w);
          float d[8];
          unpack8(ld16(p.dy + o), d);
          if (p.dy2) {
            float d2[8];
            unpack8(ld16(p.dy2 + o), d2);
#pragma unroll
            for (int e = 0; e < 8; ++e) d[e] += d2[e];
          }
          const unsigned char me = (unsigned char)(kh * 3 + kw);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (a[e] == me) acc[e] += d[e];
        }
      }
      st16(p.dx + v, pack8(acc));
    }
  }
};

struct AvgPoolFwd {   // [N, HW, C] -> [N, C]
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 4;   // register cap: 4+ resident CTAs per SM
  struct Params {
    const uint4* x;
    uint4* y;
    int N, HW, C;
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int cv = p.C >> 3;
    const long long v = (long long)bidx.x * kThreads + threadIdx.x;
    if (v >= (long long)p.N * cv) return;
    const int n = (int)(v / cv), c8 = (int)(v % cv);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int q = 0; q < p.HW; ++q) {
      float f[8];
      unpack8(ld16(p.x + ((long long)n * p.HW + q) * cv + c8), f);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += f[e];
    }
    const float s = 1.f / (float)p.HW;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] *= s;
    st16(p.y + v, pack8(acc));
  }
};

struct AvgPoolBwd {
  static constexpr int kThreads = 256;
  struct Params {
    const uint4* dy;   // [N, C]
    uint4* dx;         // [N, HW, C]
    int N, HW, C;
    long long nvec;
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int cv = p.C >> 3;
    const long long v0 = (long long)bidx.x * kVecPerBlock;
    const float s = 1.f / (float)p.HW;
    for (int i = threadIdx.x; i < kVecPerBlock; i += kThreads) {
      const long long v = v0 + i;
      if (v >= p.nvec) break;
      const int c8 = (int)(v % cv);
      const long long n = v / cv / p.HW;
      float d[8];
      unpack8(p.dy[n * cv + c8], d);
#pragma unroll
      for (int e = 0; e < 8; ++e) d[e] *= s;
      st16(p.dx + v, pack8(d));
    }
  }
};

// ---------------------------------------------------------------- loss
struct SoftmaxXent {   // one row per logical block
  // One HBM read of the row: pass 1 streams it (16-byte vectors, 4 in flight
  // per thread) into shared memory while folding an online (max, sum-exp);
  // pass 2 writes dlogits from the staged copy.  Rows above kCacheMax bytes
  // are re-read from global memory instead.  bf16 logits (the GPT-2 LM head,
  // 100 KB rows) halve the traffic and keep a logical block ~10 us.
  static constexpr int kThreads = 512;   // 32 KB of loads in flight per row (256 threads: ~20 us rows)
  static constexpr int kMinBlocks = 2;   // register cap 64: two rows per SM (uncapped: 1 row, 973 -> 685 us)
  static constexpr int kUnroll = 4;
  static constexpr int kCacheMax = 104 * 1024;
  static constexpr int kRed = 128;   // bytes of reduction scratch ahead of the row
  struct Params {
    const uint4* logits;   // [B, Npad] fp32 or bf16 (GEMM output)
    const float* bias;     // [Npad] or null
    const int* labels;     // [B]
    float* loss;           // [B]
    uint4* dl;             // [B, Npad] bf16, zero in the pad columns
    float4* dl32;          // [B, Npad] fp32 or null: the bias-gradient partials (summed over B by sgd_update)
    int B, Npad, ncls, bf16, cache;
  };
  static __device__ __forceinline__ void to_f32(const Params& p, const uint4 (&r)[2], int j0, float (&x)[8]) {
    if (p.bf16) {
      unpack8(r[0], x);
    } else {
      x[0] = __uint_as_float(r[0].x); x[1] = __uint_as_float(r[0].y);
      x[2] = __uint_as_float(r[0].z); x[3] = __uint_as_float(r[0].w);
      x[4] = __uint_as_float(r[1].x); x[5] = __uint_as_float(r[1].y);
      x[6] = __uint_as_float(r[1].z); x[7] = __uint_as_float(r[1].w);
    }
    if (p.bias) {
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(p.bias + j0));
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(p.bias + j0) + 1);
      x[0] += b0.x; x[1] += b0.y; x[2] += b0.z; x[3] += b0.w;
      x[4] += b1.x; x[5] += b1.y; x[6] += b1.z; x[7] += b1.w;
    }
    if (j0 + 8 > p.ncls) {   // only the row's last valid vector straddles ncls (a uniform test per vector)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (j0 + e >= p.ncls) x[e] = -INFINITY;
    }
  }
  static constexpr float kLog2e = 1.4426950408889634f;
  static __device__ __forceinline__ float exp2f_fast(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  static __device__ __forceinline__ void merge(float& m, float& s, float m2, float s2) {   // base-2 maxima
    const float mm = fmaxf(m, m2);
    if (mm == -INFINITY) return;
    s = s * exp2f_fast(m - mm) + s2 * exp2f_fast(m2 - mm);
    m = mm;
  }
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char* smem) {
    float* red = reinterpret_cast<float*>(smem);   // [2][kThreads / 32]
    uint4* cache = reinterpret_cast<uint4*>(smem + kRed);
    const int b = bidx.x;
    const int cpv = p.bf16 ? 1 : 2;                // 16-byte chunks per 8 logits
    const int nv = p.Npad >> 3;
    const uint4* row = p.logits + (long long)b * nv * cpv;
    float m = -INFINITY, s = 0.f;
    for (int v0 = threadIdx.x; v0 < nv; v0 += kUnroll * kThreads) {
      uint4 r[kUnroll][2];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int v = v0 + u * kThreads;
        if (v < nv) {
          r[u][0] = p.cache ? __ldcs(row + v * cpv) : __ldg(row + v * cpv);
          if (!p.bf16) r[u][1] = p.cache ? __ldcs(row + v * cpv + 1) : __ldg(row + v * cpv + 1);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int v = v0 + u * kThreads;
        if (v >= nv) break;
        if (p.cache) {
          cache[v * cpv] = r[u][0];
          if (!p.bf16) cache[v * cpv + 1] = r[u][1];
        }
        float x[8];
        to_f32(p, r[u], v * 8, x);
        // base-2 domain (m is the running max of x * log2 e): one FFMA + one
        // MUFU.EX2 per element; the kernel is instruction-bound, not HBM-bound
        float mv = x[0];
#pragma unroll
        for (int e = 1; e < 8; ++e) mv = fmaxf(mv, x[e]);
        if (mv == -INFINITY) continue;
        mv *= kLog2e;
        if (mv > m) { s *= exp2f_fast(m - mv); m = mv; }
#pragma unroll
        for (int e = 0; e < 8; ++e) s += exp2f_fast(fmaf(x[e], kLog2e, -m));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
      merge(m, s, m2, s2);
    }
    if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = m; red[kThreads / 32 + (threadIdx.x >> 5)] = s; }
    __syncthreads();
    m = red[0]; s = red[kThreads / 32];
    for (int w = 1; w < kThreads / 32; ++w) merge(m, s, red[w], red[kThreads / 32 + w]);
    const int lab = p.labels[b];
    const float inv_b = 1.f / (float)p.B, scale = inv_b / s;
    for (int v = threadIdx.x; v < nv; v += kThreads) {
      uint4 r[2];
      if (p.cache) {
        r[0] = cache[v * cpv];
        if (!p.bf16) r[1] = cache[v * cpv + 1];
      } else {
        r[0] = ld16(row + v * cpv);
        if (!p.bf16) r[1] = ld16(row + v * cpv + 1);
      }
      float x[8];
      to_f32(p, r, v * 8, x);
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = exp2f_fast(fmaf(x[e], kLog2e, -m)) * scale;   // masked: ex2(-inf) = 0
      if (v == (lab >> 3)) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (e == (lab & 7)) x[e] -= inv_b;
      }
      st16(p.dl + (long long)b * nv + v, pack8(x));
      if (p.dl32) {
        float4* d = p.dl32 + ((long long)b * nv + v) * 2;
        __stcs(d, make_float4(x[0], x[1], x[2], x[3]));
        __stcs(d + 1, make_float4(x[4], x[5], x[6], x[7]));
      }
    }
    if (threadIdx.x == 0) {
      const float zl = p.bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(row)[lab])
                              : reinterpret_cast<const float*>(row)[lab];
      p.loss[b] = logf(s) + m * 0.6931471805599453f - (zl + (p.bias ? p.bias[lab] : 0.f));
    }
    __syncthreads();
  }
};

// ---------------------------------------------------------------- split-K reduction
// out (bf16) = sum over S fp32 partials [S][n], fixed order: the epilogue of a
// split-K activation GEMM (few output tiles, long K -> more, shorter logical
// blocks for the scheduler)
struct SplitKReduce {
  // A logical block covers vpb output vectors (8 x bf16) and all S partials
  // (~64 KB of partial reads): with many splits (the LM-head dgrad: S = 42)
  // the block's threads split the S dimension into G = 256 / vpb groups, each
  // summing partials g, g + G, ... in order, then the groups are added in
  // order through shared memory -- deterministic, and ~10 us per block
  // (4096 outputs x 42 partials per block made it ~30 us: preemption latency)
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 3;
  static constexpr int kSmem = kThreads * 8 * 4;
  struct Params {
    const float4* in;    // [S][n / 4]
    uint4* out;          // [n / 8]
    long long n8;
    long long stride4;   // n / 4
    int S;
    int vpb;             // output vectors per logical block: 512 (2 per thread) or 32..256
    EpArgs ep;           // optional fused linear-layer epilogue (bias null: plain sum)
    int C;               // output columns (bias index) when ep.bias is set
  };
  // the finished sum of output vector v (8 bf16 of a row-major [rows, C] output)
  static __device__ __forceinline__ void finish8(const Params& p, long long v, float (&acc)[8]) {
    if (p.ep.on) {
      const long long e0 = 8 * v;
      const long long row = e0 / p.C;
      const int col = (int)(e0 - row * p.C);
      ep_bias_res8(p.ep, row, col, acc);
      if (p.ep.pre != nullptr) st16(reinterpret_cast<uint4*>(p.ep.pre) + v, pack8(acc));
      if (p.ep.act) {
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = ep_act(acc[e], p.ep.act);
      }
    }
    st16(p.out + v, pack8(acc));
  }
  static __device__ __forceinline__ void add8(float (&acc)[8], const float4& a, const float4& b) {
    acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
    acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
  }
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char* smem) {
    if (p.vpb == 2 * kThreads) {
      const long long v0 = (long long)bidx.x * (2 * kThreads) + threadIdx.x;
      float acc[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[u][e] = 0.f;
      // two partials' loads in flight per step (one DRAM round trip per two
      // splits), still summed in split order
      int sp = 0;
      for (; sp + 1 < p.S; sp += 2) {
        float4 t[2][2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const long long v = v0 + u * kThreads;
            if (v < p.n8) {
              t[h][u][0] = __ldcs(p.in + (sp + h) * p.stride4 + 2 * v);
              t[h][u][1] = __ldcs(p.in + (sp + h) * p.stride4 + 2 * v + 1);
            }
          }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int u = 0; u < 2; ++u) add8(acc[u], t[h][u][0], t[h][u][1]);
      }
      if (sp < p.S) {
        float4 t[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const long long v = v0 + u * kThreads;
          if (v < p.n8) {
            t[u][0] = __ldcs(p.in + sp * p.stride4 + 2 * v);
            t[u][1] = __ldcs(p.in + sp * p.stride4 + 2 * v + 1);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) add8(acc[u], t[u][0], t[u][1]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const long long v = v0 + u * kThreads;
        if (v < p.n8) finish8(p, v, acc[u]);
      }
      return;
    }
    float* red = reinterpret_cast<float*>(smem);   // [G][vpb][8]
    const int G = kThreads / p.vpb, lv = threadIdx.x % p.vpb, g = threadIdx.x / p.vpb;
    const long long v = (long long)bidx.x * p.vpb + lv;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (v < p.n8) {
      const float4* src = p.in + 2 * v;
      int sp = g;
      for (; sp + 3 * G < p.S; sp += 4 * G) {   // four partials in flight, summed in order
        float4 t[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          t[u][0] = __ldcs(src + (sp + u * G) * p.stride4);
          t[u][1] = __ldcs(src + (sp + u * G) * p.stride4 + 1);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) add8(acc, t[u][0], t[u][1]);
      }
      for (; sp < p.S; sp += G) add8(acc, __ldcs(src + sp * p.stride4), __ldcs(src + sp * p.stride4 + 1));
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) red[(g * p.vpb + lv) * 8 + e] = acc[e];
    __syncthreads();
    if (g == 0 && v < p.n8) {
      for (int k = 1; k < G; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += red[(k * p.vpb + lv) * 8 + e];
      finish8(p, v, acc);
    }
    __syncthreads();   // red is reused by the next logical block of a PTB worker
  }
};

// ---------------------------------------------------------------- optimizer
struct SgdSeg {
  float* w;               // fp32 master weights [rows, cols]
  float* v;               // momentum
  const float* grad;      // [S][gstride] partials (split-K slices / batch rows)
  long long n;
  long long gstride;
  int S;
  float wd;
  __nv_bfloat16* wb;      // optional bf16 copy, same layout
  __nv_bfloat16* wt;      // optional bf16 transposed copy [cols, rows]
  int rows, cols;
  int chunk;              // elements per logical block (64..1024, power of 2)
  int zero_from;          // >= 0: zero gradient slices [zero_from, S) after reading (atomic accumulators)
  // optional bf16 flipped copy of a k x k conv weight [cout, (kh, kw, cin)]:
  // wf[cin, (k-1-kh, k-1-kw, cout)] -- the weight of the data gradient as a
  // stride-1 forward convolution of dy (implicit-GEMM dgrad)
  __nv_bfloat16* wf;
  int fk, fcin;
};

struct SgdUpdate {
  static constexpr int kThreads = 256;
  static constexpr int kChunk = kThreads * 4;   // elements per logical block (float4 per thread)
  struct Params {
    const SgdSeg* segs;
    const int2* map;      // logical block -> (segment, chunk)
    float lr, momentum;
  };
  static __device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char* smem) {
    const int2 m = p.map[bidx.x];
    const SgdSeg& s = p.segs[m.x];
    // chunk / 4 element-threads; with few elements per block (many gradient
    // partials: chunk shrinks to keep ~32 KB of partials per block) the other
    // threads split the S partials into G groups -- group g sums partials
    // g, g + G, ... in order, then the groups are added in order through
    // shared memory (deterministic; 16 threads looping over 329 partials made
    // the stem weight's blocks ~65 us long)
    const int nthr = min(kThreads, s.chunk / 4);
    const int G = kThreads / nthr;
    const int lt = threadIdx.x % nthr, grp = threadIdx.x / nthr;
    const long long i = (long long)m.y * s.chunk + lt * 4;
    const bool valid = i < s.n;   // segment sizes are multiples of 4
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
      int j = grp;
      for (; j + 3 * G < s.S; j += 4 * G) {
        const float4 a0 = ld4(s.grad + (long long)j * s.gstride + i);
        const float4 a1 = ld4(s.grad + (long long)(j + G) * s.gstride + i);
        const float4 a2 = ld4(s.grad + (long long)(j + 2 * G) * s.gstride + i);
        const float4 a3 = ld4(s.grad + (long long)(j + 3 * G) * s.gstride + i);
        g.x = (((g.x + a0.x) + a1.x) + a2.x) + a3.x;
        g.y = (((g.y + a0.y) + a1.y) + a2.y) + a3.y;
        g.z = (((g.z + a0.z) + a1.z) + a2.z) + a3.z;
        g.w = (((g.w + a0.w) + a1.w) + a2.w) + a3.w;
      }
      for (; j < s.S; j += G) {
        const float4 a = ld4(s.grad + (long long)j * s.gstride + i);
        g.x += a.x; g.y += a.y; g.z += a.z; g.w += a.w;
      }
      if (s.zero_from >= 0)
        for (int z = s.zero_from + grp; z < s.S; z += G)
          *reinterpret_cast<float4*>(const_cast<float*>(s.grad) + (long long)z * s.gstride + i) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (G > 1) {
      float4* red = reinterpret_cast<float4*>(smem);   // [G][nthr]
      red[grp * nthr + lt] = g;
      __syncthreads();
      if (grp == 0) {
        for (int k = 1; k < G; ++k) {
          const float4 t = red[k * nthr + lt];
          g.x += t.x; g.y += t.y; g.z += t.z; g.w += t.w;
        }
      }
      __syncthreads();   // red is reused by the next logical block of a PTB worker
    }
    if (grp != 0 || !valid) return;
    const float4 w = *reinterpret_cast<const float4*>(s.w + i);
    const float4 v = *reinterpret_cast<const float4*>(s.v + i);
    const float gw[4] = {g.x + s.wd * w.x, g.y + s.wd * w.y, g.z + s.wd * w.z, g.w + s.wd * w.w};
    const float wv[4] = {w.x, w.y, w.z, w.w};
    const float vv[4] = {v.x, v.y, v.z, v.w};
    float nw[4], nv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      nv[e] = p.momentum * vv[e] + gw[e];
      nw[e] = wv[e] - p.lr * nv[e];
    }
    *reinterpret_cast<float4*>(s.v + i) = make_float4(nv[0], nv[1], nv[2], nv[3]);
    *reinterpret_cast<float4*>(s.w + i) = make_float4(nw[0], nw[1], nw[2], nw[3]);
    if (s.wb) {
      __nv_bfloat162 h0 = __floats2bfloat162_rn(nw[0], nw[1]), h1 = __floats2bfloat162_rn(nw[2], nw[3]);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&h0);
      u.y = *reinterpret_cast<uint32_t*>(&h1);
      *reinterpret_cast<uint2*>(s.wb + i) = u;
    }
    if (s.wt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const long long r = (i + e) / s.cols, c = (i + e) - r * s.cols;
        s.wt[c * s.rows + r] = __float2bfloat16_rn(nw[e]);
      }
    }
    if (s.wf) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const long long co = (i + e) / s.cols, kk = (i + e) - co * s.cols;
        const int tap = (int)(kk / s.fcin), ci = (int)(kk - (long long)tap * s.fcin);
        const int r = tap / s.fk, sx = tap - r * s.fk;
        s.wf[(long long)ci * s.fk * s.fk * s.rows + ((long long)(s.fk - 1 - r) * s.fk + (s.fk - 1 - sx)) * s.rows + co] =
            __float2bfloat16_rn(nw[e]);
      }
    }
  }
};

}  // namespace nn

// ---------------------------------------------------------------- host binding
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static int geometry(const tally_kernel_args* a, int base, nn::Geometry& g) {
  g.N = (int)a->i[base + 0];
  g.H = (int)a->i[base + 1];
  g.W = (int)a->i[base + 2];
  g.C = (int)a->i[base + 3];
  const long long kh_kw_s_p = a->i[base + 4];   // packed: kh | kw << 8 | stride << 16 | pad << 24
  g.KH = (int)(kh_kw_s_p & 0xff);
  g.KW = (int)((kh_kw_s_p >> 8) & 0xff);
  g.stride = (int)((kh_kw_s_p >> 16) & 0xff);
  g.pad = (int)((kh_kw_s_p >> 24) & 0xff);
  if (g.N < 1 || g.H < 1 || g.W < 1 || g.C < 8 || g.C % 8 || g.KH < 1 || g.KW < 1 || g.stride < 1) {
    set_error("conv geometry: need N,H,W >= 1, C %% 8 == 0, kernel >= 1, stride >= 1");
    return TALLY_EINVAL;
  }
  g.OH = (g.H + 2 * g.pad - g.KH) / g.stride + 1;
  g.OW = (g.W + 2 * g.pad - g.KW) / g.stride + 1;
  g.K = g.KH * g.KW * g.C;
  g.Kp = (g.K + 63) / 64 * 64;
  if (g.OH < 1 || g.OW < 1) { set_error("conv geometry: empty output"); return TALLY_EINVAL; }
  return TALLY_OK;
}

template <class P>
static void finish(Instance* inst, const P& p, long long blocks, int threads, size_t smem, double bytes) {
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)blocks, 1, 1);
  inst->threads = threads;
  inst->smem = smem;
  inst->alg_bytes = bytes;
}

// ptr: x, col.  i: N, H, W, C, packed(kh,kw,stride,pad)
static int bind_im2col(const tally_kernel_args* a, Instance* inst) {
  nn::Im2Col::Params p{};
  int rc = geometry(a, 0, p.g);
  if (rc) return rc;
  p.x = static_cast<const uint4*>(a->ptr[0]);
  p.col = static_cast<uint4*>(a->ptr[1]);
  if (!p.x || !p.col || !aligned16(p.x) || !aligned16(p.col)) { set_error("im2col: 16-byte aligned x, col"); return TALLY_EINVAL; }
  p.rows = (long long)p.g.N * p.g.OH * p.g.OW;
  p.rpb = max(1, nn::Im2Col::kVecs / (p.g.Kp / 8));
  if (p.g.Kp / 8 > nn::Im2Col::kMaxKv || p.rows * (p.g.Kp / 8) >= (1ll << 31) ||
      (long long)p.g.N * p.g.H * p.g.W >= (1ll << 31)) {
    set_error("im2col: K <= 8192 and fewer than 2^31 column vectors / pixels");
    return TALLY_EINVAL;
  }
  finish(inst, p, (p.rows + p.rpb - 1) / p.rpb, nn::Im2Col::kThreads, nn::Im2Col::kSmem,
         2.0 * ((double)p.rows * p.g.Kp + (double)p.g.N * p.g.H * p.g.W * p.g.C));
  return TALLY_OK;
}

// ptr: col, dx.  i: geometry as im2col
static int bind_col2im(const tally_kernel_args* a, Instance* inst) {
  nn::Col2Im::Params p{};
  int rc = geometry(a, 0, p.g);
  if (rc) return rc;
  p.col = static_cast<const uint4*>(a->ptr[0]);
  p.dx = static_cast<uint4*>(a->ptr[1]);
  if (!p.col || !p.dx || !aligned16(p.col) || !aligned16(p.dx)) { set_error("col2im: 16-byte aligned col, dx"); return TALLY_EINVAL; }
  p.nvec = (long long)p.g.N * p.g.H * p.g.W * (p.g.C / 8);
  if (p.nvec >= (1ll << 31)) { set_error("col2im: fewer than 2^31 vectors"); return TALLY_EINVAL; }
  finish(inst, p, (p.nvec + nn::kCol2ImVec - 1) / nn::kCol2ImVec, nn::Col2Im::kThreads, 0,
         2.0 * ((double)p.g.N * p.g.OH * p.g.OW * p.g.Kp + 8.0 * p.nvec));
  return TALLY_OK;
}

// ptr: src, dst.  i: R, C
static int bind_transpose(const tally_kernel_args* a, Instance* inst) {
  nn::Transpose::Params p{};
  p.src = static_cast<const unsigned short*>(a->ptr[0]);
  p.dst = static_cast<unsigned short*>(a->ptr[1]);
  p.R = a->i[0];
  p.C = a->i[1];
  if (!p.src || !p.dst || p.R < 1 || p.C < 1) { set_error("transpose: need src, dst, R, C >= 1"); return TALLY_EINVAL; }
  memcpy(inst->params, &p, sizeof(p));
  const int T = nn::Transpose::T;
  inst->grid = make_uint3((unsigned)((p.C + T - 1) / T), (unsigned)((p.R + T - 1) / T), 1);
  inst->threads = nn::Transpose::kThreads;
  inst->smem = (size_t)T * (T + 2) * 2;
  inst->alg_bytes = 4.0 * (double)p.R * (double)p.C;
  return TALLY_OK;
}

// ptr: x, g, g2, y, mean, invstd, part, gamma.  i: P, C, mode, RB, then
//   mode 0: beta, scale_shift ([2][C]) addresses
//   mode 1: dgamma, dbeta, coef ([3][C]) addresses.   f: eps
template <int MODE>
static int bind_bn_stats(const tally_kernel_args* a, Instance* inst) {
  using Body = nn::BnStats<MODE>;
  typename Body::Params p{};
  p.x = static_cast<const uint4*>(a->ptr[0]);
  p.g = static_cast<const uint4*>(a->ptr[1]);
  p.g2 = static_cast<const uint4*>(a->ptr[2]);
  p.y = static_cast<const uint4*>(a->ptr[3]);
  p.mean = static_cast<float*>(a->ptr[4]);
  p.invstd = static_cast<float*>(a->ptr[5]);
  p.part = static_cast<float*>(a->ptr[6]);
  p.gamma = static_cast<const float*>(a->ptr[7]);
  p.P = a->i[0];
  p.C = (int)a->i[1];
  p.mode = (int)a->i[2];
  p.RB = (int)a->i[3];
  p.eps = (float)a->f[0];
  if (p.mode != MODE) { set_error("bn_stats: mode %d given to the mode-%d kind", p.mode, MODE); return TALLY_EINVAL; }
  if (p.mode == 0) {
    p.beta = reinterpret_cast<const float*>(a->i[4]);
    p.scale_shift = reinterpret_cast<float*>(a->i[5]);
  } else {
    p.dgamma = reinterpret_cast<float*>(a->i[4]);
    p.dbeta = reinterpret_cast<float*>(a->i[5]);
    p.coef = reinterpret_cast<float*>(a->i[6]);   // mode 1 only
  }
  const bool c_ok = p.C >= 64 && (p.C < 256 ? (256 % p.C == 0) : (p.C % 256 == 0));
  const bool ops0 = p.mode == 0 && p.x && p.mean && p.invstd && p.gamma && p.beta && p.scale_shift;
  const bool ops1 = p.mode == 1 && p.x && p.mean && p.invstd && p.gamma && p.g && p.dgamma && p.dbeta && p.coef;
  const bool ops2 = p.mode == 2 && p.g && p.dbeta && (!p.x || (p.mean && p.invstd && p.dgamma));
  if (!p.part || p.P < 1 || !c_ok || p.RB < 1 || !(ops0 || ops1 || ops2)) {
    set_error("bn_stats: need x, part, mean, invstd, gamma, C in {64, 128} or a multiple of 256, and the "
              "mode 0 (beta, scale_shift) / mode 1 (g, dgamma, dbeta, coef) operands");
    return TALLY_EINVAL;
  }
  p.nrb = (int)((p.P + p.RB - 1) / p.RB);
  p.ngroups = (p.nrb + Body::kGroup - 1) / Body::kGroup;
  p.inv_count = (float)(1.0 / (double)p.P);
  const int cblocks = (p.C + 255) / 256;
  // chain state: counters + level-2 partials (zeroed at bind and per new PTB chain)
  const size_t cnt_bytes = ((size_t)cblocks * (p.ngroups + 1) * sizeof(unsigned) + 255) / 256 * 256;
  const size_t bytes = cnt_bytes + (size_t)2 * p.ngroups * p.C * sizeof(float);
  void* st = nullptr;
  cudaError_t e = cudaMalloc(&st, bytes);
  if (e == cudaSuccess) e = cudaMemset(st, 0, cnt_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "bn_stats state");
  inst->resume_ring = st;
  inst->resume_bytes = cnt_bytes;   // only the counters need zeroing
  p.cnt1 = static_cast<unsigned*>(st);
  p.cnt2 = p.cnt1 + (size_t)cblocks * p.ngroups;
  p.part2 = reinterpret_cast<float*>(static_cast<char*>(st) + cnt_bytes);
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)cblocks, (unsigned)p.nrb, 1);
  inst->threads = Body::kThreads;
  inst->smem = 2 * 2048 * sizeof(float) + 16;
  const int streams = p.mode == 0 ? 1 : (p.x ? 2 : 1) + (p.g2 ? 1 : 0) + (p.y ? 1 : 0);
  inst->alg_bytes = 2.0 * streams * (double)p.P * p.C + 8.0 * p.nrb * p.C;
  return TALLY_OK;
}

// mode 0 -- ptr: part, gamma, beta, mean, invstd, scale, shift
// mode 1 -- ptr: part, gamma, mean, invstd, dgamma, dbeta, ca, cb; i[4]: cc address
// i: nrb, C, mode, count.  f: eps
static int bind_bn_finalize(const tally_kernel_args* a, Instance* inst) {
  nn::BnFinalize::Params p{};
  p.part = static_cast<const float*>(a->ptr[0]);
  p.gamma = static_cast<const float*>(a->ptr[1]);
  p.nrb = (int)a->i[0];
  p.C = (int)a->i[1];
  p.mode = (int)a->i[2];
  const long long count = a->i[3];
  p.eps = (float)a->f[0];
  if (!p.part || !p.gamma || p.nrb < 1 || p.C < 1 || count < 1 || (p.mode != 0 && p.mode != 1)) {
    set_error("bn_finalize: need part, gamma, nrb, C, count >= 1, mode 0/1");
    return TALLY_EINVAL;
  }
  p.inv_count = (float)(1.0 / (double)count);
  if (p.mode == 0) {
    p.beta = static_cast<const float*>(a->ptr[2]);
    p.o_mean = static_cast<float*>(a->ptr[3]);
    p.o_invstd = static_cast<float*>(a->ptr[4]);
    p.scale = static_cast<float*>(a->ptr[5]);
    p.shift = static_cast<float*>(a->ptr[6]);
    if (!p.beta || !p.o_mean || !p.o_invstd || !p.scale || !p.shift) { set_error("bn_finalize: mode 0 operands"); return TALLY_EINVAL; }
  } else {
    p.mean = static_cast<const float*>(a->ptr[2]);
    p.invstd = static_cast<const float*>(a->ptr[3]);
    p.dgamma = static_cast<float*>(a->ptr[4]);
    p.dbeta = static_cast<float*>(a->ptr[5]);
    p.ca = static_cast<float*>(a->ptr[6]);
    p.cb = static_cast<float*>(a->ptr[7]);
    p.cc = reinterpret_cast<float*>(a->i[4]);
    if (!p.mean || !p.invstd || !p.dgamma || !p.dbeta || !p.ca || !p.cb || !p.cc) { set_error("bn_finalize: mode 1 operands"); return TALLY_EINVAL; }
  }
  finish(inst, p, (p.C + 31) / 32, nn::BnFinalize::kThreads, 2 * 8 * 32 * sizeof(float), 8.0 * p.nrb * p.C + 24.0 * p.C);
  return TALLY_OK;
}

// ptr: x, res, y, scale, shift.  i: P, C, relu
static int bind_bn_act(const tally_kernel_args* a, Instance* inst) {
  nn::BnAct::Params p{};
  p.x = static_cast<const uint4*>(a->ptr[0]);
  p.res = static_cast<const uint4*>(a->ptr[1]);
  p.y = static_cast<uint4*>(a->ptr[2]);
  p.scale = static_cast<const float*>(a->ptr[3]);
  p.shift = static_cast<const float*>(a->ptr[4]);
  p.pre = static_cast<uint4*>(a->ptr[5]);
  const long long P = a->i[0];
  p.C = (int)a->i[1];
  p.relu = (int)a->i[2];
  if (!p.x || !p.y || !p.shift || P < 1 || p.C < 8 || p.C % 8 || p.relu < 0 || p.relu > 3) {
    set_error("bn_act: need x, y, shift, C %% 8 == 0, act in {0 none, 1 relu, 2 gelu tanh, 3 gelu erf}");
    return TALLY_EINVAL;
  }
  p.nvec = P * (p.C / 8);
  if (p.nvec >= (1ll << 31)) { set_error("bn_act: fewer than 2^31 vectors"); return TALLY_EINVAL; }
  finish(inst, p, (p.nvec + nn::kVecPerBlock - 1) / nn::kVecPerBlock, nn::BnAct::kThreads, 0,
         16.0 * p.nvec * (p.res ? 3 : 2));
  return TALLY_OK;
}

// ptr[0..7] = g, g2, y, x, ca, cb, cc, dx;  i: P, C, optional dz_out address
static int bind_bn_bwd(const tally_kernel_args* a, Instance* inst) {
  nn::BnBwd::Params p{};
  p.g = static_cast<const uint4*>(a->ptr[0]);
  p.g2 = static_cast<const uint4*>(a->ptr[1]);
  p.y = static_cast<const uint4*>(a->ptr[2]);
  p.x = static_cast<const uint4*>(a->ptr[3]);
  p.ca = static_cast<const float*>(a->ptr[4]);
  p.cb = static_cast<const float*>(a->ptr[5]);
  p.cc = static_cast<const float*>(a->ptr[6]);
  p.dx = static_cast<uint4*>(a->ptr[7]);
  const long long P = a->i[0];
  p.C = (int)a->i[1];
  p.dz_out = reinterpret_cast<uint4*>(a->i[2]);
  if (!p.g || !p.x || !p.ca || !p.cb || !p.cc || !p.dx || P < 1 || p.C < 8 || p.C % 8) {
    set_error("bn_bwd: need g, x, ca, cb, cc, dx and C %% 8 == 0");
    return TALLY_EINVAL;
  }
  p.nvec = P * (p.C / 8);
  if (p.nvec >= (1ll << 31)) { set_error("bn_bwd: fewer than 2^31 vectors"); return TALLY_EINVAL; }
  const int streams = 3 + (p.g2 ? 1 : 0) + (p.y ? 1 : 0) + (p.dz_out ? 1 : 0);
  finish(inst, p, (p.nvec + nn::BnBwd::kBlockVec - 1) / nn::BnBwd::kBlockVec, nn::BnBwd::kThreads, 0,
         16.0 * p.nvec * streams);
  return TALLY_OK;
}

// ptr: x, y, arg.  i: N, H, W, C
static int bind_maxpool_fwd(const tally_kernel_args* a, Instance* inst) {
  nn::MaxPoolFwd::Params p{};
  p.x = static_cast<const uint4*>(a->ptr[0]);
  p.y = static_cast<uint4*>(a->ptr[1]);
  p.arg = static_cast<uint2*>(a->ptr[2]);
  p.N = (int)a->i[0]; p.H = (int)a->i[1]; p.W = (int)a->i[2]; p.C = (int)a->i[3];
  if (!p.x || !p.y || !p.arg || p.N < 1 || p.H < 1 || p.W < 1 || p.C < 8 || p.C % 8) { set_error("maxpool: bad arguments"); return TALLY_EINVAL; }
  p.OH = (p.H + 2 - 3) / 2 + 1;
  p.OW = (p.W + 2 - 3) / 2 + 1;
  p.nvec = (long long)p.N * p.OH * p.OW * (p.C / 8);
  finish(inst, p, (p.nvec + nn::kVecPerBlock - 1) / nn::kVecPerBlock, nn::MaxPoolFwd::kThreads, 0,
         2.0 * p.N * p.H * p.W * p.C + 24.0 * p.nvec);
  return TALLY_OK;
}

// ptr: dy, dy2, arg, dx.  i: N, H, W, C (input geometry)
static int bind_maxpool_bwd(const tally_kernel_args* a, Instance* inst) {
  nn::MaxPoolBwd::Params p{};
  p.dy = static_cast<const uint4*>(a->ptr[0]);
  p.dy2 = static_cast<const uint4*>(a->ptr[1]);
  p.arg = static_cast<const uint2*>(a->ptr[2]);
  p.dx = static_cast<uint4*>(a->ptr[3]);
  p.N = (int)a->i[0]; p.H = (int)a->i[1]; p.W = (int)a->i[2]; p.C = (int)a->i[3];
  if (!p.dy || !p.arg || !p.dx || p.N < 1 || p.H < 1 || p.W < 1 || p.C < 8 || p.C % 8) { set_error("maxpool_bwd: bad arguments"); return TALLY_EINVAL; }
  p.OH = (p.H + 2 - 3) / 2 + 1;
  p.OW = (p.W + 2 - 3) / 2 + 1;
  p.nvec = (long long)p.N * p.H * p.W * (p.C / 8);
  const double out_vec = (double)p.N * p.OH * p.OW * (p.C / 8);
  finish(inst, p, (p.nvec + nn::kVecPerBlock - 1) / nn::kVecPerBlock, nn::MaxPoolBwd::kThreads, 0,
         16.0 * p.nvec + out_vec * (p.dy2 ? 40.0 : 24.0));
  return TALLY_OK;
}

// ptr: x, y.  i: N, HW, C
static int bind_avgpool_fwd(const tally_kernel_args* a, Instance* inst) {
  nn::AvgPoolFwd::Params p{};
  p.x = static_cast<const uint4*>(a->ptr[0]);
  p.y = static_cast<uint4*>(a->ptr[1]);
  p.N = (int)a->i[0]; p.HW = (int)a->i[1]; p.C = (int)a->i[2];
  if (!p.x || !p.y || p.N < 1 || p.HW < 1 || p.C < 8 || p.C % 8) { set_error("avgpool: bad arguments"); return TALLY_EINVAL; }
  const long long nv = (long long)p.N * (p.C / 8);
  finish(inst, p, (nv + 255) / 256, nn::AvgPoolFwd::kThreads, 0, 2.0 * p.N * p.C * (p.HW + 1.0));
  return TALLY_OK;
}

// ptr: dy, dx.  i: N, HW, C
static int bind_avgpool_bwd(const tally_kernel_args* a, Instance* inst) {
  nn::AvgPoolBwd::Params p{};
  p.dy = static_cast<const uint4*>(a->ptr[0]);
  p.dx = static_cast<uint4*>(a->ptr[1]);
  p.N = (int)a->i[0]; p.HW = (int)a->i[1]; p.C = (int)a->i[2];
  if (!p.dy || !p.dx || p.N < 1 || p.HW < 1 || p.C < 8 || p.C % 8) { set_error("avgpool_bwd: bad arguments"); return TALLY_EINVAL; }
  p.nvec = (long long)p.N * p.HW * (p.C / 8);
  finish(inst, p, (p.nvec + nn::kVecPerBlock - 1) / nn::kVecPerBlock, nn::AvgPoolBwd::kThreads, 0,
         16.0 * p.nvec + 2.0 * p.N * p.C);
  return TALLY_OK;
}

// ptr: logits, bias, labels, loss, dl, dl32.  i: B, Npad, ncls
// ptr: logits, bias (or null), labels, loss, dl, dl32 (or null).  i: B, Npad, ncls, logits_bf16
static int bind_softmax_xent(const tally_kernel_args* a, Instance* inst) {
  nn::SoftmaxXent::Params p{};
  p.logits = static_cast<const uint4*>(a->ptr[0]);
  p.bias = static_cast<const float*>(a->ptr[1]);
  p.labels = static_cast<const int*>(a->ptr[2]);
  p.loss = static_cast<float*>(a->ptr[3]);
  p.dl = static_cast<uint4*>(a->ptr[4]);
  p.dl32 = static_cast<float4*>(a->ptr[5]);
  p.B = (int)a->i[0]; p.Npad = (int)a->i[1]; p.ncls = (int)a->i[2]; p.bf16 = a->i[3] ? 1 : 0;
  if (!p.logits || !p.labels || !p.loss || !p.dl || p.B < 1 || p.ncls < 1 || p.Npad < p.ncls || p.Npad % 8 ||
      !aligned16(p.logits) || !aligned16(p.dl) || (p.bias && !aligned16(p.bias)) || (p.dl32 && !aligned16(p.dl32))) {
    set_error("softmax_xent: bad arguments (Npad % 8 == 0, 16-byte aligned buffers)");
    return TALLY_EINVAL;
  }
  const size_t row = (size_t)p.Npad * (p.bf16 ? 2 : 4);
  p.cache = row <= (size_t)nn::SoftmaxXent::kCacheMax && getenv("TALLY_XENT_NO_STAGE") == nullptr;
  finish(inst, p, p.B, nn::SoftmaxXent::kThreads, nn::SoftmaxXent::kRed + (p.cache ? row : 0),
         (double)p.B * ((double)row + 2.0 * p.Npad + (p.dl32 ? 4.0 * p.Npad : 0.0)));
  return TALLY_OK;
}

static int setup_softmax_xent() {
  const void* fns[3] = {reinterpret_cast<const void*>(&k_original<nn::SoftmaxXent>),
                        reinterpret_cast<const void*>(&k_sliced<nn::SoftmaxXent>),
                        reinterpret_cast<const void*>(&k_ptb<nn::SoftmaxXent>)};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         nn::SoftmaxXent::kRed + nn::SoftmaxXent::kCacheMax);
    if (e != cudaSuccess) return cuda_fail(e, "softmax_xent smem attribute");
  }
  return TALLY_OK;
}

// ptr: segs (device SgdSeg[]), map (device int2[]).  i: blocks.  f: lr, momentum
static int bind_sgd(const tally_kernel_args* a, Instance* inst) {
  nn::SgdUpdate::Params p{};
  p.segs = static_cast<const nn::SgdSeg*>(a->ptr[0]);
  p.map = static_cast<const int2*>(a->ptr[1]);
  const long long blocks = a->i[0];
  p.lr = (float)a->f[0];
  p.momentum = (float)a->f[1];
  if (!p.segs || !p.map || blocks < 1) { set_error("sgd_update: need segs, map, blocks >= 1"); return TALLY_EINVAL; }
  finish(inst, p, blocks, nn::SgdUpdate::kThreads, nn::SgdUpdate::kThreads * 16, (double)a->i[1]);   // i[1]: bytes (host computed)
  return TALLY_OK;
}

// ptr: in (fp32 [S][n]), out (bf16 [n]).  i: n, S
static int bind_splitk_reduce(const tally_kernel_args* a, Instance* inst) {
  nn::SplitKReduce::Params p{};
  p.in = static_cast<const float4*>(a->ptr[0]);
  p.out = static_cast<uint4*>(a->ptr[1]);
  const long long n = a->i[0];
  p.S = (int)a->i[1];
  if (!p.in || !p.out || n < 8 || n % 8 || p.S < 1 || !aligned16(p.in) || !aligned16(p.out)) {
    set_error("splitk_reduce: need 16-byte aligned in, out, n %% 8 == 0, S >= 1");
    return TALLY_EINVAL;
  }
  p.n8 = n / 8;
  p.stride4 = n / 4;
  // fused linear-layer epilogue: ptr[2] bias (fp32 [C]), ptr[3] residual and
  // ptr[4] pre-activation output (bf16, row-major [n / C, C]); i[2] C, i[3] act
  double ep_bytes = 0.0;
  if (a->ptr[2] || a->ptr[3] || a->ptr[4] || a->i[3]) {
    p.C = (int)a->i[2];
    if (p.C < 8 || p.C % 8 || n % p.C || a->i[3] < 0 || a->i[3] > 3 || (a->ptr[2] && !aligned16(a->ptr[2])) ||
        (a->ptr[3] && !aligned16(a->ptr[3])) || (a->ptr[4] && !aligned16(a->ptr[4]))) {
      set_error("splitk_reduce: a fused epilogue needs aligned fp32 bias / bf16 residual, C %% 8 == 0 dividing n, act 0-3");
      return TALLY_EINVAL;
    }
    p.ep.on = 1;
    p.ep.bias = static_cast<const float*>(a->ptr[2]);
    p.ep.res = static_cast<const __nv_bfloat16*>(a->ptr[3]);
    p.ep.pre = static_cast<__nv_bfloat16*>(a->ptr[4]);
    p.ep.ldr = p.C;
    p.ep.act = (int)a->i[3];
    ep_bytes = (a->ptr[2] ? 4.0 * p.C : 0.0) + (a->ptr[3] ? 2.0 * n : 0.0) + (a->ptr[4] ? 2.0 * n : 0.0);
  }
  // ~64 KB of partials per logical block: 512 vectors up to S = 4, then
  // halving down to 32 vectors (S >= 33)
  p.vpb = 2 * nn::SplitKReduce::kThreads;
  while (p.vpb > 32 && (long long)p.vpb * 32 * p.S > 65536) p.vpb >>= 1;
  finish(inst, p, (p.n8 + p.vpb - 1) / p.vpb, nn::SplitKReduce::kThreads, nn::SplitKReduce::kSmem,
         (4.0 * p.S + 2.0) * (double)n + ep_bytes);
  return TALLY_OK;
}

// splitk_reduce_bn -- ptr: parts [S][P][C] fp32, out [P, C] bf16; ptr[7]:
// tally_bn_stats (part, gamma, beta, mean, invstd, scale_shift, eps, rb).
// i: P, C, S.  The split-K sum of a convolution / GEMM feeding a training
// batch norm, with that batch norm's statistics (bn_stats mode 0) fused.
//
// bn_fold -- ptr[0]: the fused epilogue's partial rows [2][R][C] fp32 (the
// tally_bn_stats.part a GEMM / conv_fprop wrote); ptr[7]: tally_bn_stats
// (its part = this kind's own fold scratch).  i: R, C, count (rows of the
// normalised tensor).  bn_stats mode 0's fold and finalisation over them.
template <int MODE>
static int bind_splitk_bn(const tally_kernel_args* a, Instance* inst) {
  using Body = nn::BnStats<MODE>;
  typename Body::Params p{};
  const tally_bn_stats* bs = static_cast<const tally_bn_stats*>(a->ptr[7]);
  p.sk_in = static_cast<const float4*>(a->ptr[0]);
  p.sk_out = static_cast<uint4*>(a->ptr[1]);
  p.P = a->i[0];
  p.C = (int)a->i[1];
  p.sk_S = MODE == 3 ? (int)a->i[2] : 1;
  const long long count = MODE == 3 ? p.P : a->i[2];
  const bool c_ok = p.C >= 64 && (p.C < 256 ? (256 % p.C == 0) : (p.C % 256 == 0));
  if (!bs || !p.sk_in || (MODE == 3 && !p.sk_out) || !aligned16(p.sk_in) || (MODE == 3 && !aligned16(p.sk_out)) ||
      p.P < 1 || !c_ok || p.sk_S < 1 || count < 1 || bs->rb < 1 || !bs->part || !bs->gamma || !bs->beta ||
      !bs->mean || !bs->invstd || !bs->scale_shift || p.P * p.C >= (1ll << 40)) {
    set_error("%s: need 16-byte aligned inputs (and out), rows, S / count >= 1, C in {64, 128} or a multiple of "
              "256, and tally_bn_stats (part, gamma, beta, mean, invstd, scale_shift, rb >= 1)",
              MODE == 3 ? "splitk_reduce_bn" : "bn_fold");
    return TALLY_EINVAL;
  }
  p.sk_stride4 = p.P * p.C / 4;
  p.RB = (int)bs->rb;
  p.part = bs->part;
  p.gamma = bs->gamma;
  p.beta = bs->beta;
  p.mean = bs->mean;
  p.invstd = bs->invstd;
  p.scale_shift = bs->scale_shift;
  p.eps = (float)bs->eps;
  p.mode = MODE;
  p.nrb = (int)((p.P + p.RB - 1) / p.RB);
  p.ngroups = (p.nrb + Body::kGroup - 1) / Body::kGroup;
  p.inv_count = (float)(1.0 / (double)count);
  const int cblocks = (p.C + 255) / 256;
  const size_t cnt_bytes = ((size_t)cblocks * (p.ngroups + 1) * sizeof(unsigned) + 255) / 256 * 256;
  const size_t bytes = cnt_bytes + (size_t)2 * p.ngroups * p.C * sizeof(float);
  void* st = nullptr;
  cudaError_t e = cudaMalloc(&st, bytes);
  if (e == cudaSuccess) e = cudaMemset(st, 0, cnt_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "splitk_reduce_bn state");
  inst->resume_ring = st;
  inst->resume_bytes = cnt_bytes;
  p.cnt1 = static_cast<unsigned*>(st);
  p.cnt2 = p.cnt1 + (size_t)cblocks * p.ngroups;
  p.part2 = reinterpret_cast<float*>(static_cast<char*>(st) + cnt_bytes);
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)cblocks, (unsigned)p.nrb, 1);
  inst->threads = Body::kThreads;
  inst->smem = 2 * 2048 * sizeof(float) + 16;
  inst->alg_bytes = (MODE == 3 ? (4.0 * p.sk_S + 2.0) : 8.0) * (double)p.P * p.C + 8.0 * p.nrb * p.C;
  return TALLY_OK;
}

template <class B>
static KernelKind nn_kind(const char* name, int (*bind)(const tally_kernel_args*, Instance*)) {
  KernelKind k{};
  k.name = name;
  k.fn_original = reinterpret_cast<const void*>(&k_original<B>);
  k.fn_sliced = reinterpret_cast<const void*>(&k_sliced<B>);
  k.fn_ptb = reinterpret_cast<const void*>(&k_ptb<B>);
  k.bind = bind;
  return k;
}

int register_nn_kernels(KernelKind* out, int cap) {
  if (cap < 18) return 0;
  int n = 0;
  out[n++] = nn_kind<nn::Im2Col>("im2col_bf16", bind_im2col);
  out[n++] = nn_kind<nn::Col2Im>("col2im_bf16", bind_col2im);
  out[n++] = nn_kind<nn::Transpose>("transpose_bf16", bind_transpose);
  out[n++] = nn_kind<nn::BnStats<0>>("bn_stats", bind_bn_stats<0>);
  out[n++] = nn_kind<nn::BnStats<1>>("bn_stats_bwd", bind_bn_stats<1>);
  out[n++] = nn_kind<nn::BnStats<2>>("colstats", bind_bn_stats<2>);
  out[n++] = nn_kind<nn::BnFinalize>("bn_finalize", bind_bn_finalize);
  out[n++] = nn_kind<nn::BnAct>("bn_act", bind_bn_act);
  out[n++] = nn_kind<nn::BnBwd>("bn_bwd", bind_bn_bwd);
  out[n++] = nn_kind<nn::MaxPoolFwd>("maxpool_fwd", bind_maxpool_fwd);
  out[n++] = nn_kind<nn::MaxPoolBwd>("maxpool_bwd", bind_maxpool_bwd);
  out[n++] = nn_kind<nn::AvgPoolFwd>("avgpool_fwd", bind_avgpool_fwd);
  out[n++] = nn_kind<nn::AvgPoolBwd>("avgpool_bwd", bind_avgpool_bwd);
  out[n++] = nn_kind<nn::SoftmaxXent>("softmax_xent", bind_softmax_xent);
  out[n - 1].setup = setup_softmax_xent;
  out[n++] = nn_kind<nn::SgdUpdate>("sgd_update", bind_sgd);
  out[n++] = nn_kind<nn::SplitKReduce>("splitk_reduce", bind_splitk_reduce);
  out[n++] = nn_kind<nn::BnStats<3>>("splitk_reduce_bn", bind_splitk_bn<3>);
  out[n++] = nn_kind<nn::BnStats<4>>("bn_fold", bind_splitk_bn<4>);
  return n;
}

}  // namespace tally
