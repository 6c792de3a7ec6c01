// Best-effort transformer-training kernels (config C3: GPT-2 small training,
// BASELINE.json configs[2]) in the three Tally launch shapes.  Activations are
// [rows = tokens, C] bf16 row-major matrices; statistics fp32.  Every
// reduction has a fixed order (bit-identical across launch shapes) except
// the embedding-gradient scatter (fp32 atomics).
//
//   layernorm_fwd      y = (x - mean) * rstd * gamma + beta, one warp per row;
//                      saves mean / rstd per row
//   layernorm_bwd      dx = rstd * (dy*g - mean(dy*g) - xhat * mean(dy*g*xhat)) [+ residual grad]
//   gelu_bwd           dx = g * gelu'(pre)  (tanh approximation, GPT-2 "gelu_new"; or exact erf, BERT)
//   softmax_causal     P = softmax(scale * S) over keys j <= i (or all keys), one warp per row
//   softmax_causal_bwd dS = P * (dP - sum_j P dP) * scale
//   embedding_fwd      x = wte[token] + wpe[position]
//   embedding_bwd      dwte[token] += dx  (fp32 atomics)
#include <cuda_bf16.h>

#include <cstdio>

#include "epilogue.cuh"
#include "registry.h"

namespace tally {

namespace tf {

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

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ void ld8f(const float* p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p + 4));
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

constexpr int kRowsPerBlock = 8;   // one warp per row, 256 threads
// row width <= 32 * 8 * 4 = 1024 elements (BERT-large / GPT-2 / BERT-base):
// the row lives in registers, and 2048-wide rows (kMaxVec 8) cost 168-197
// registers -> one CTA (8 warps) per SM, layer norm at 0.2 of HBM
constexpr int kMaxVec = 4;

// ---------------------------------------------------------------- LayerNorm
struct LayerNormFwd {
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 2;
  struct Params {
    const uint4* x;
    uint4* y;
    const float* gamma;
    const float* beta;
    float* mean;
    float* rstd;
    long long rows;
    int C;
    float eps;
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long r = (long long)bidx.x * kRowsPerBlock + warp;
    if (r >= p.rows) return;   // warp-uniform; no barrier in this body
    const int cv = p.C >> 3;
    const uint4* xr = p.x + r * cv;
    float v[kMaxVec][8];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxVec; ++k) {
      const int j = lane + 32 * k;
      if (j < cv) {
        unpack8(__ldg(xr + j), v[k]);
#pragma unroll
        for (int e = 0; e < 8; ++e) s += v[k][e];
      }
    }
    const float mu = warp_sum(s) / (float)p.C;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxVec; ++k) {
      const int j = lane + 32 * k;
      if (j < cv) {
#pragma unroll
        for (int e = 0; e < 8; ++e) { const float d = v[k][e] - mu; q += d * d; }
      }
    }
    const float rs = rsqrtf(warp_sum(q) / (float)p.C + p.eps);
    if (lane == 0) { p.mean[r] = mu; p.rstd[r] = rs; }
#pragma unroll
    for (int k = 0; k < kMaxVec; ++k) {
      const int j = lane + 32 * k;
      if (j < cv) {
        float g[8], b[8], o[8];
        ld8f(p.gamma + 8 * j, g);
        ld8f(p.beta + 8 * j, b);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = (v[k][e] - mu) * rs * g[e] + b[e];
        p.y[r * cv + j] = pack8(o);
      }
    }
  }
};

struct LayerNormBwd {
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 2;
  struct Params {
    const uint4* dy;
    const uint4* g2;     // optional gradient added to dx (the residual stream)
    const uint4* x;
    const float* gamma;
    const float* mean;
    const float* rstd;
    uint4* dx;
    long long rows;
    int C;
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long r = (long long)bidx.x * kRowsPerBlock + warp;
    if (r >= p.rows) return;
    const int cv = p.C >> 3;
    const float mu = p.mean[r], rs = p.rstd[r];
    float xh[kMaxVec][8], dg[kMaxVec][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxVec; ++k) {
      const int j = lane + 32 * k;
      if (j < cv) {
        float xv[8], dv[8], g[8];
        unpack8(__ldg(p.x + r * cv + j), xv);
        unpack8(__ldg(p.dy + r * cv + j), dv);
        ld8f(p.gamma + 8 * j, g);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          xh[k][e] = (xv[e] - mu) * rs;
          dg[k][e] = dv[e] * g[e];
          s1 += dg[k][e];
          s2 += dg[k][e] * xh[k][e];
        }
      }
    }
    const float a = warp_sum(s1) / (float)p.C, b = warp_sum(s2) / (float)p.C;
#pragma unroll
    for (int k = 0; k < kMaxVec; ++k) {
      const int j = lane + 32 * k;
      if (j < cv) {
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = rs * (dg[k][e] - a - xh[k][e] * b);
        if (p.g2) {
          float t[8];
          unpack8(__ldg(p.g2 + r * cv + j), t);
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] += t[e];
        }
        p.dx[r * cv + j] = pack8(o);
      }
    }
  }
};

// ---------------------------------------------------------------- GELU backward
__device__ __forceinline__ float gelu_grad(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float u = k0 * (x + k1 * x * x * x);
  const float t = tanhf(u);
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}
__device__ __forceinline__ float gelu_erf_grad(float x) {   // BERT "gelu": x * Phi(x)
  return gelu_erf_grad_fast(x);   // (epilogue.cuh)
}

template <int ERF_KIND>   // 0: "gelu_bwd" (tanh approximation), 1: "gelu_bwd_erf" (exact erf)
struct GeluBwdT {
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 4;   // (PTB at 83 registers fitted 2 CTAs per SM: 0.7x of untransformed)
  static constexpr int kVec = 4;   // (8 measured slower untransformed: 33 -> 48 us per BERT-large launch)
  struct Params {
    const uint4* g;
    const uint4* pre;
    uint4* dx;
    long long nvec;
    int erf;                 // 0: tanh approximation (GPT-2), 1: exact erf (BERT)
  };
  // (the variant is chosen once per block: with the choice per element the
  // compiler if-converted both -- tanh and erf paths for every element, ~60
  // instructions each, issue-bound at 3.2 IPC in ncu)
  template <bool ERF>
  static __device__ __forceinline__ void run_v(const Params& p, uint3 bidx) {
    const long long v0 = (long long)bidx.x * (kThreads * kVec) + threadIdx.x;
    uint4 gv[kVec], hv[kVec];
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      const long long v = v0 + u * kThreads;
      if (v < p.nvec) { gv[u] = __ldg(p.g + v); hv[u] = __ldg(p.pre + v); }
    }
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      const long long v = v0 + u * kThreads;
      if (v >= p.nvec) continue;
      float g[8], h[8];
      unpack8(gv[u], g);
      unpack8(hv[u], h);
      if constexpr (ERF) {
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          float d0, d1;
          gelu_erf_grad2(h[e], h[e + 1], d0, d1);
          g[e] *= d0;
          g[e + 1] *= d1;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) g[e] *= gelu_grad(h[e]);
      }
      p.dx[v] = pack8(g);
    }
  }
  // (one variant per kind: both in one kernel made its PTB shape 0.68 ->
  // 0.53x of untransformed)
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    run_v<ERF_KIND != 0>(p, bidx);
  }
};
using GeluBwd = GeluBwdT<0>;
using GeluBwdErf = GeluBwdT<1>;

// ---------------------------------------------------------------- causal softmax
// One HBM pass per row: each lane holds its float4s of the row in registers
// (V = ceil(T / 128) per row), R rows per warp with all their loads issued
// before any arithmetic (R * V 16 B loads in flight per lane); R * V = 16
// (forward) / 8 (backward) keeps the register budget fixed, so a logical
// block is 8 * R rows: T = 512 -> 32 (forward) / 16 (backward) rows.
constexpr int softmax_v(int T) { return T <= 512 ? 4 : T <= 1024 ? 8 : 16; }
constexpr int softmax_rpw(int T, int budget) { return budget / softmax_v(T) > 0 ? budget / softmax_v(T) : 1; }

struct SoftmaxCausal {
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 2;  // <= 128 registers: two CTAs (16 warps) per SM
  static constexpr int kBudget = 16;   // float4 registers per lane
  struct Params {
    const float* s;          // [rows, T] scores (fp32 GEMM output)
    __nv_bfloat16* p;        // [rows, T] probabilities (0 past the diagonal)
    long long rows;
    int T;
    float scale;
    int causal;              // 0: every key visible (BERT encoder)
  };
  template <int V, int R>
  static __device__ __forceinline__ void rows_(const Params& p, long long r0) {
    const int lane = threadIdx.x & 31;
    float4 a[R][V];
    int vis[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const long long r = r0 + rr;
      vis[rr] = r < p.rows ? (p.causal ? (int)(r % p.T) : p.T - 1) : -1;   // keys 0..vis are visible
      const float* sr = p.s + (r < p.rows ? r : 0) * p.T;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int j = 4 * (lane + 32 * k);
        a[rr][k] = (j <= vis[rr] && j < p.T) ? __ldg(reinterpret_cast<const float4*>(sr + j))
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (vis[rr] < 0) continue;   // warp-uniform (rows past the end)
      const long long r = r0 + rr;
      float m = -INFINITY;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int j = 4 * (lane + 32 * k);
        const float e[4] = {a[rr][k].x, a[rr][k].y, a[rr][k].z, a[rr][k].w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (j + q <= vis[rr] && j + q < p.T) m = fmaxf(m, e[q] * p.scale);
      }
      m = warp_max(m);
      float sum = 0.f;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int j = 4 * (lane + 32 * k);
        float* e = reinterpret_cast<float*>(&a[rr][k]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          e[q] = (j + q <= vis[rr] && j + q < p.T) ? __expf(e[q] * p.scale - m) : 0.f;
          sum += e[q];
        }
      }
      const float inv = 1.f / warp_sum(sum);
      __nv_bfloat16* pr = p.p + r * p.T;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int j = 4 * (lane + 32 * k);
        if (j >= p.T) continue;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(a[rr][k].x * inv, a[rr][k].y * inv);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(a[rr][k].z * inv, a[rr][k].w * inv);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&h0);
        w.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(pr + j) = w;
      }
    }
  }
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int warp = threadIdx.x >> 5;
    if (p.T <= 512) {
      constexpr int R = softmax_rpw(512, kBudget);
      rows_<4, R>(p, ((long long)bidx.x * 8 + warp) * R);
    } else if (p.T <= 1024) {
      constexpr int R = softmax_rpw(1024, kBudget);
      rows_<8, R>(p, ((long long)bidx.x * 8 + warp) * R);
    } else {
      constexpr int R = softmax_rpw(2048, kBudget);
      rows_<16, R>(p, ((long long)bidx.x * 8 + warp) * R);
    }
  }
  static long long rows_per_block(int T) { return 8ll * softmax_rpw(T, kBudget); }
};

struct SoftmaxCausalBwd {
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 2;
  static constexpr int kBudget = 8;    // (float4 + bf16x4) register pairs per lane
  struct Params {
    const __nv_bfloat16* p;  // [rows, T]
    const float* dp;         // [rows, T] (fp32 GEMM output)
    __nv_bfloat16* ds;       // [rows, T], scaled by `scale` (the forward's score scale)
    long long rows;
    int T;
    float scale;
    int causal;
  };
  template <int V, int R>
  static __device__ __forceinline__ void rows_(const Params& p, long long r0) {
    const int lane = threadIdx.x & 31;
    float4 d[R][V];
    uint2 pv[R][V];
    int vis[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const long long r = r0 + rr;
      vis[rr] = r < p.rows ? (p.causal ? (int)(r % p.T) : p.T - 1) : -1;
      const long long ro = (r < p.rows ? r : 0) * p.T;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int j = 4 * (lane + 32 * k);
        const bool ok = j <= vis[rr] && j < p.T;
        d[rr][k] = ok ? __ldg(reinterpret_cast<const float4*>(p.dp + ro + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
        pv[rr][k] = ok ? __ldg(reinterpret_cast<const uint2*>(p.p + ro + j)) : make_uint2(0u, 0u);
      }
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (vis[rr] < 0) continue;
      const long long r = r0 + rr;
      float dot = 0.f;   // P is 0 past the diagonal
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pv[rr][k].x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pv[rr][k].y));
        dot += a.x * d[rr][k].x + a.y * d[rr][k].y + b.x * d[rr][k].z + b.y * d[rr][k].w;
      }
      dot = warp_sum(dot);
      __nv_bfloat16* sr = p.ds + r * p.T;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int j = 4 * (lane + 32 * k);
        if (j >= p.T) continue;
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pv[rr][k].x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pv[rr][k].y));
        __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x * (d[rr][k].x - dot) * p.scale, a.y * (d[rr][k].y - dot) * p.scale);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(b.x * (d[rr][k].z - dot) * p.scale, b.y * (d[rr][k].w - dot) * p.scale);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&h0);
        w.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(sr + j) = w;
      }
    }
  }
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int warp = threadIdx.x >> 5;
    if (p.T <= 512) {
      constexpr int R = softmax_rpw(512, kBudget);
      rows_<4, R>(p, ((long long)bidx.x * 8 + warp) * R);
    } else {   // T <= 1024 (bind)
      constexpr int R = softmax_rpw(1024, kBudget);
      rows_<8, R>(p, ((long long)bidx.x * 8 + warp) * R);
    }
  }
  static long long rows_per_block(int T) { return 8ll * softmax_rpw(T, kBudget); }
};

// ---------------------------------------------------------------- embedding
struct EmbeddingFwd {
  static constexpr int kThreads = 256;
  struct Params {
    const int* tok;
    const uint4* wte;   // [V, C]
    const uint4* wpe;   // [T, C]
    uint4* x;           // [rows, C]
    long long rows;
    int T, C;
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long r = (long long)bidx.x * kRowsPerBlock + warp;
    if (r >= p.rows) return;
    const int cv = p.C >> 3;
    const long long t = p.tok[r];
    const long long pos = r % p.T;
    for (int j = lane; j < cv; j += 32) {
      float a[8], b[8];
      unpack8(__ldg(p.wte + t * cv + j), a);
      unpack8(__ldg(p.wpe + pos * cv + j), b);
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] += b[e];
      p.x[r * cv + j] = pack8(a);
    }
  }
};

struct EmbeddingBwd {
  static constexpr int kThreads = 256;
  struct Params {
    const int* tok;
    const uint4* dx;    // [rows, C]
    float* dwte;        // [V, C] fp32, accumulated with atomics
    long long rows;
    int C;
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long r = (long long)bidx.x * kRowsPerBlock + warp;
    if (r >= p.rows) return;
    const int cv = p.C >> 3;
    const long long t = p.tok[r];
    for (int j = lane; j < cv; j += 32) {
      float a[8];
      unpack8(__ldg(p.dx + r * cv + j), a);
      float4* dst = reinterpret_cast<float4*>(p.dwte + t * p.C + 8 * j);
      atomicAdd(dst, make_float4(a[0], a[1], a[2], a[3]));
      atomicAdd(dst + 1, make_float4(a[4], a[5], a[6], a[7]));
    }
  }
};

}  // namespace tf

// ---------------------------------------------------------------- host binding
template <class P>
static void tf_finish(Instance* inst, const P& p, long long blocks, size_t smem, double bytes) {
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)blocks, 1, 1);
  inst->threads = 256;
  inst->smem = smem;
  inst->alg_bytes = bytes;
}

static bool rowwise_ok(long long rows, int C) { return rows >= 1 && C >= 8 && C % 8 == 0 && C <= 32 * 8 * tf::kMaxVec; }

// ptr: x, y, gamma, beta, mean, rstd.  i: rows, C.  f: eps
static int bind_ln_fwd(const tally_kernel_args* a, Instance* inst) {
  tf::LayerNormFwd::Params p{};
  p.x = static_cast<const uint4*>(a->ptr[0]);
  p.y = static_cast<uint4*>(a->ptr[1]);
  p.gamma = static_cast<const float*>(a->ptr[2]);
  p.beta = static_cast<const float*>(a->ptr[3]);
  p.mean = static_cast<float*>(a->ptr[4]);
  p.rstd = static_cast<float*>(a->ptr[5]);
  p.rows = a->i[0];
  p.C = (int)a->i[1];
  p.eps = (float)a->f[0];
  if (!p.x || !p.y || !p.gamma || !p.beta || !p.mean || !p.rstd || !rowwise_ok(p.rows, p.C)) {
    set_error("layernorm_fwd: need x, y, gamma, beta, mean, rstd and 8 <= C <= 2048, C %% 8 == 0");
    return TALLY_EINVAL;
  }
  tf_finish(inst, p, (p.rows + 7) / 8, 0, 4.0 * (double)p.rows * p.C + 8.0 * p.rows);
  return TALLY_OK;
}

// ptr: dy, g2, x, gamma, mean, rstd, dx.  i: rows, C
static int bind_ln_bwd(const tally_kernel_args* a, Instance* inst) {
  tf::LayerNormBwd::Params p{};
  p.dy = static_cast<const uint4*>(a->ptr[0]);
  p.g2 = static_cast<const uint4*>(a->ptr[1]);
  p.x = static_cast<const uint4*>(a->ptr[2]);
  p.gamma = static_cast<const float*>(a->ptr[3]);
  p.mean = static_cast<const float*>(a->ptr[4]);
  p.rstd = static_cast<const float*>(a->ptr[5]);
  p.dx = static_cast<uint4*>(a->ptr[6]);
  p.rows = a->i[0];
  p.C = (int)a->i[1];
  if (!p.dy || !p.x || !p.gamma || !p.mean || !p.rstd || !p.dx || !rowwise_ok(p.rows, p.C)) {
    set_error("layernorm_bwd: need dy, x, gamma, mean, rstd, dx and 8 <= C <= 2048, C %% 8 == 0");
    return TALLY_EINVAL;
  }
  tf_finish(inst, p, (p.rows + 7) / 8, 0, (double)p.rows * p.C * (p.g2 ? 8.0 : 6.0));
  return TALLY_OK;
}

// ptr: g, pre, dx.  i: n (elements), erf (must match the kind: gelu_bwd /
// gelu_bwd_erf)
template <int ERF>
static int bind_gelu_bwd(const tally_kernel_args* a, Instance* inst) {
  tf::GeluBwd::Params p{};
  if ((a->i[1] ? 1 : 0) != ERF) { set_error("gelu_bwd: the exact-erf variant is the gelu_bwd_erf kind"); return TALLY_EINVAL; }
  p.g = static_cast<const uint4*>(a->ptr[0]);
  p.pre = static_cast<const uint4*>(a->ptr[1]);
  p.dx = static_cast<uint4*>(a->ptr[2]);
  const long long n = a->i[0];
  if (!p.g || !p.pre || !p.dx || n < 8 || n % 8) { set_error("gelu_bwd: need g, pre, dx, n %% 8 == 0"); return TALLY_EINVAL; }
  p.nvec = n / 8;
  p.erf = a->i[1] ? 1 : 0;
  const long long per = tf::GeluBwd::kThreads * tf::GeluBwd::kVec;
  tf_finish(inst, p, (p.nvec + per - 1) / per, 0, 6.0 * (double)n);
  return TALLY_OK;
}

// ptr: s (fp32), p (bf16).  i: rows, T, causal.  f: scale
static int bind_softmax_causal(const tally_kernel_args* a, Instance* inst) {
  tf::SoftmaxCausal::Params p{};
  p.s = static_cast<const float*>(a->ptr[0]);
  p.p = static_cast<__nv_bfloat16*>(a->ptr[1]);
  p.rows = a->i[0];
  p.T = (int)a->i[1];
  p.scale = (float)a->f[0];
  p.causal = a->i[2] ? 1 : 0;
  if (!p.s || !p.p || p.rows < 1 || p.T < 4 || p.T % 4 || p.T > 2048 || p.rows % p.T) {
    set_error("softmax_causal: need s, p, T %% 4 == 0, T <= 2048, rows a multiple of T");
    return TALLY_EINVAL;
  }
  const long long rpb = tf::SoftmaxCausal::rows_per_block(p.T);
  tf_finish(inst, p, (p.rows + rpb - 1) / rpb, 0, 6.0 * (double)p.rows * p.T);
  return TALLY_OK;
}

// ptr: p (bf16), dp (fp32), ds (bf16).  i: rows, T, causal.  f: scale
static int bind_softmax_causal_bwd(const tally_kernel_args* a, Instance* inst) {
  tf::SoftmaxCausalBwd::Params p{};
  p.p = static_cast<const __nv_bfloat16*>(a->ptr[0]);
  p.dp = static_cast<const float*>(a->ptr[1]);
  p.ds = static_cast<__nv_bfloat16*>(a->ptr[2]);
  p.rows = a->i[0];
  p.T = (int)a->i[1];
  p.scale = (float)a->f[0];
  p.causal = a->i[2] ? 1 : 0;
  if (!p.p || !p.dp || !p.ds || p.rows < 1 || p.T < 4 || p.T % 4 || p.T > 1024 || p.rows % p.T) {
    set_error("softmax_causal_bwd: need p, dp, ds, T %% 4 == 0, T <= 1024, rows a multiple of T");
    return TALLY_EINVAL;
  }
  const long long rpb = tf::SoftmaxCausalBwd::rows_per_block(p.T);
  tf_finish(inst, p, (p.rows + rpb - 1) / rpb, 0, 8.0 * (double)p.rows * p.T);
  return TALLY_OK;
}

// ptr: tok, wte, wpe, x.  i: rows, T, C
static int bind_embedding_fwd(const tally_kernel_args* a, Instance* inst) {
  tf::EmbeddingFwd::Params p{};
  p.tok = static_cast<const int*>(a->ptr[0]);
  p.wte = static_cast<const uint4*>(a->ptr[1]);
  p.wpe = static_cast<const uint4*>(a->ptr[2]);
  p.x = static_cast<uint4*>(a->ptr[3]);
  p.rows = a->i[0];
  p.T = (int)a->i[1];
  p.C = (int)a->i[2];
  if (!p.tok || !p.wte || !p.wpe || !p.x || p.rows < 1 || p.T < 1 || p.C < 8 || p.C % 8) {
    set_error("embedding_fwd: need tok, wte, wpe, x, C %% 8 == 0");
    return TALLY_EINVAL;
  }
  tf_finish(inst, p, (p.rows + 7) / 8, 0, 6.0 * (double)p.rows * p.C);
  return TALLY_OK;
}

// ptr: tok, dx, dwte (fp32).  i: rows, C
static int bind_embedding_bwd(const tally_kernel_args* a, Instance* inst) {
  tf::EmbeddingBwd::Params p{};
  p.tok = static_cast<const int*>(a->ptr[0]);
  p.dx = static_cast<const uint4*>(a->ptr[1]);
  p.dwte = static_cast<float*>(a->ptr[2]);
  p.rows = a->i[0];
  p.C = (int)a->i[1];
  if (!p.tok || !p.dx || !p.dwte || p.rows < 1 || p.C < 8 || p.C % 8) {
    set_error("embedding_bwd: need tok, dx, dwte, C %% 8 == 0");
    return TALLY_EINVAL;
  }
  tf_finish(inst, p, (p.rows + 7) / 8, 0, 10.0 * (double)p.rows * p.C);
  return TALLY_OK;
}

template <class B>
static KernelKind tf_kind(const char* name, int (*bind)(const tally_kernel_args*, Instance*)) {
  KernelKind k{};
  k.name = name;
  k.fn_original = reinterpret_cast<const void*>(&k_original<B>);
  k.fn_sliced = reinterpret_cast<const void*>(&k_sliced<B>);
  k.fn_ptb = reinterpret_cast<const void*>(&k_ptb<B>);
  k.bind = bind;
  return k;
}

int register_tf_kernels(KernelKind* out, int cap) {
  if (cap < 8) return 0;
  int n = 0;
  out[n++] = tf_kind<tf::LayerNormFwd>("layernorm_fwd", bind_ln_fwd);
  out[n++] = tf_kind<tf::LayerNormBwd>("layernorm_bwd", bind_ln_bwd);
  out[n++] = tf_kind<tf::GeluBwd>("gelu_bwd", bind_gelu_bwd<0>);
  out[n++] = tf_kind<tf::GeluBwdErf>("gelu_bwd_erf", bind_gelu_bwd<1>);
  out[n++] = tf_kind<tf::SoftmaxCausal>("softmax_causal", bind_softmax_causal);
  out[n++] = tf_kind<tf::SoftmaxCausalBwd>("softmax_causal_bwd", bind_softmax_causal_bwd);
  out[n++] = tf_kind<tf::EmbeddingFwd>("embedding_fwd", bind_embedding_fwd);
  out[n++] = tf_kind<tf::EmbeddingBwd>("embedding_bwd", bind_embedding_bwd);
  return n;
}

}  // namespace tally
