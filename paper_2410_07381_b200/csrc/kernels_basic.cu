// HBM-bound best-effort / high-priority kernels, each in Original, Sliced and
// PTB shape (tally_device.cuh):
//
//   vecadd_i64  out[i] = wrap64(a[i] + b[i]) over a flat int64 word image with
//               the reference IR's three-region layout [a | b | out] and word
//               offsets as arguments (ref ir/interp.py:195-196, tests/test_ir.py:165-172)
//   vecadd_f32  c = a + b, 16 B vector loads/stores, streaming cache hints;
//               one logical block = elems_per_block contiguous floats
//   rowsum_f32  out[r] = sum_c in[r, c], one warp per row, fixed reduction
//               order (bit-identical across shapes)
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>

#include "registry.h"

namespace tally {

// ---------------------------------------------------------------- vecadd_i64
struct VecAddI64 {
  static constexpr int kThreads = 256;
  struct Params {
    long long* mem;
    long long a, b, out;   // word offsets into mem
    long long n;           // elements
    long long epb;         // elements per logical block
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const long long base = (long long)bidx.x * p.epb;
    for (long long i = threadIdx.x; i < p.epb; i += kThreads) {
      const long long k = base + i;
      if (k < p.n) {
        const unsigned long long x = (unsigned long long)p.mem[p.a + k];
        const unsigned long long y = (unsigned long long)p.mem[p.b + k];
        p.mem[p.out + k] = (long long)(x + y);   // two's-complement wrap
      }
    }
  }
};

static int bind_vecadd_i64(const tally_kernel_args* a, Instance* inst) {
  VecAddI64::Params p{};
  p.mem = static_cast<long long*>(a->ptr[0]);
  p.a = a->i[0]; p.b = a->i[1]; p.out = a->i[2]; p.n = a->i[3];
  p.epb = a->i[4] > 0 ? a->i[4] : 1;
  if (!p.mem || p.n < 1) { set_error("vecadd_i64: need mem and n >= 1"); return TALLY_EINVAL; }
  const long long blocks = (p.n + p.epb - 1) / p.epb;
  if (blocks > 0x7fffffffLL) { set_error("vecadd_i64: grid too large"); return TALLY_EINVAL; }
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)blocks, 1, 1);
  inst->threads = VecAddI64::kThreads;
  inst->smem = 0;
  inst->alg_bytes = 24.0 * (double)p.n;
  return TALLY_OK;
}

// ---------------------------------------------------------------- vecadd_f32
struct VecAddF32 {
  static constexpr int kThreads = 256;
  static constexpr int kVecPerThread = 4;            // 4 x float4 = 16 floats / thread
  static constexpr int kElemsPerBlock = kThreads * kVecPerThread * 4;   // 4096
  struct Params {
    const float4* a;
    const float4* b;
    float4* c;
    long long n4;          // number of float4
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const long long base = (long long)bidx.x * (kThreads * kVecPerThread) + threadIdx.x;
    float4 x[kVecPerThread], y[kVecPerThread];
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      const long long k = base + (long long)j * kThreads;
      if (k < p.n4) { x[j] = ld_stream(p.a + k); y[j] = ld_stream(p.b + k); }
    }
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      const long long k = base + (long long)j * kThreads;
      if (k < p.n4)
        __stcs(p.c + k, make_float4(x[j].x + y[j].x, x[j].y + y[j].y, x[j].z + y[j].z,
                                    x[j].w + y[j].w));
    }
  }
};

static int bind_vecadd_f32(const tally_kernel_args* a, Instance* inst) {
  VecAddF32::Params p{};
  p.a = static_cast<const float4*>(a->ptr[0]);
  p.b = static_cast<const float4*>(a->ptr[1]);
  p.c = static_cast<float4*>(a->ptr[2]);
  const long long n = a->i[0];
  if (!p.a || !p.b || !p.c || n < 4 || n % 4) {
    set_error("vecadd_f32: need a, b, c and n >= 4 with n %% 4 == 0");
    return TALLY_EINVAL;
  }
  for (int k = 0; k < 3; ++k)
    if (reinterpret_cast<uintptr_t>(a->ptr[k]) % 16) {
      set_error("vecadd_f32: pointers must be 16-byte aligned");
      return TALLY_EINVAL;
    }
  p.n4 = n / 4;
  const long long blocks = (n + VecAddF32::kElemsPerBlock - 1) / VecAddF32::kElemsPerBlock;
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)blocks, 1, 1);
  inst->threads = VecAddF32::kThreads;
  inst->smem = 0;
  inst->alg_bytes = 12.0 * (double)n;
  inst->alg_flops = (double)n;
  return TALLY_OK;
}

// ---------------------------------------------------------------- rowsum_f32
struct RowSumF32 {
  static constexpr int kThreads = 256;
  static constexpr int kRowsPerBlock = kThreads / 32;
  struct Params {
    const float* in;
    float* out;
    long long rows;
    long long cols;
  };
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long r = (long long)bidx.x * kRowsPerBlock + warp;
    if (r >= p.rows) return;   // no barrier in this body: warp-level exit is safe
    const float* row = p.in + r * p.cols;
    float acc = 0.f;
    if ((p.cols & 3) == 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0) {
      const float4* row4 = reinterpret_cast<const float4*>(row);
      const long long c4 = p.cols >> 2;
      for (long long c = lane; c < c4; c += 32) {
        const float4 v = ld_stream(row4 + c);
        acc += (v.x + v.y) + (v.z + v.w);
      }
    } else {
      for (long long c = lane; c < p.cols; c += 32) acc += __ldcs(row + c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) p.out[r] = acc;
  }
};

static int bind_rowsum_f32(const tally_kernel_args* a, Instance* inst) {
  RowSumF32::Params p{};
  p.in = static_cast<const float*>(a->ptr[0]);
  p.out = static_cast<float*>(a->ptr[1]);
  p.rows = a->i[0];
  p.cols = a->i[1];
  if (!p.in || !p.out || p.rows < 1 || p.cols < 1) {
    set_error("rowsum_f32: need in, out, rows >= 1, cols >= 1");
    return TALLY_EINVAL;
  }
  const long long blocks = (p.rows + RowSumF32::kRowsPerBlock - 1) / RowSumF32::kRowsPerBlock;
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)blocks, 1, 1);
  inst->threads = RowSumF32::kThreads;
  inst->smem = 0;
  inst->alg_bytes = 4.0 * (double)p.rows * (double)p.cols + 4.0 * (double)p.rows;
  inst->alg_flops = (double)p.rows * (double)p.cols;
  return TALLY_OK;
}

// ---------------------------------------------------------------- ewise
// Generic elementwise op over contiguous fp32 / bf16 tensors -- the
// transformable kind the generic PyTorch routing (intercept.py) maps
// aten.add / mul / relu / gelu / silu onto.  fp32 arithmetic, one rounding
// to the output type (PyTorch's bf16 elementwise semantics); 16 B vectors,
// 8 per thread: a logical block is 32 KB of each operand stream.
struct Ewise {
  static constexpr int kThreads = 256;
  static constexpr int kVec = 8;
  enum Op { kAdd = 0, kMul = 1, kRelu = 2, kGeluErf = 3, kGeluTanh = 4, kSilu = 5 };
  struct Params {
    const uint4* a;
    const uint4* b;   // null for unary ops
    uint4* out;
    long long nvec;   // 16 B vectors
    int op;
    int bf16;         // 1: bf16 elements (8 per vector), 0: fp32 (4 per vector)
    float alpha;      // add: a + alpha * b
  };
  static __device__ __forceinline__ float apply(int op, float x, float y, float alpha) {
    switch (op) {
      case kAdd: return x + alpha * y;
      case kMul: return x * y;
      case kRelu: return x > 0.f ? x : 0.f;
      case kGeluErf: return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
      case kGeluTanh: {
        const float u = 0.79788456080286536f * (x + 0.044715f * x * x * x);
        return 0.5f * x * (1.f + tanhf(u));
      }
      default: return x / (1.f + expf(-x));
    }
  }
  static __device__ __forceinline__ uint4 vapply(const Params& p, uint4 va, uint4 vb) {
    uint4 r;
    if (p.bf16) {
      const __nv_bfloat162* xa = reinterpret_cast<const __nv_bfloat162*>(&va);
      const __nv_bfloat162* xb = reinterpret_cast<const __nv_bfloat162*>(&vb);
      __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 fa = __bfloat1622float2(xa[i]), fb = __bfloat1622float2(xb[i]);
        o[i] = __floats2bfloat162_rn(apply(p.op, fa.x, fb.x, p.alpha), apply(p.op, fa.y, fb.y, p.alpha));
      }
    } else {
      const float* xa = reinterpret_cast<const float*>(&va);
      const float* xb = reinterpret_cast<const float*>(&vb);
      float* o = reinterpret_cast<float*>(&r);
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] = apply(p.op, xa[i], xb[i], p.alpha);
    }
    return r;
  }
  static __device__ __forceinline__ void run(const Params& p, uint3 bidx, uint3, char*) {
    const long long base = (long long)bidx.x * (kThreads * kVec) + threadIdx.x;
    uint4 va[kVec], vb[kVec];
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const long long k = base + (long long)j * kThreads;
      if (k < p.nvec) {
        va[j] = *reinterpret_cast<const uint4*>(reinterpret_cast<const float4*>(p.a) + k);
        vb[j] = p.b ? p.b[k] : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const long long k = base + (long long)j * kThreads;
      if (k < p.nvec) p.out[k] = vapply(p, va[j], vb[j]);
    }
  }
};

static int bind_ewise(const tally_kernel_args* a, Instance* inst) {
  Ewise::Params p{};
  p.a = static_cast<const uint4*>(a->ptr[0]);
  p.b = static_cast<const uint4*>(a->ptr[1]);
  p.out = static_cast<uint4*>(a->ptr[2]);
  const long long n = a->i[0];
  p.op = (int)a->i[1];
  p.bf16 = a->i[2] ? 1 : 0;
  p.alpha = a->f[0];
  const int per = p.bf16 ? 8 : 4;
  if (!p.a || !p.out || n < per || n % per || p.op < 0 || p.op > Ewise::kSilu ||
      ((p.op == Ewise::kAdd || p.op == Ewise::kMul) && !p.b)) {
    set_error("ewise: need a, out (and b for add / mul), n a multiple of %d, op in [0, 5]", per);
    return TALLY_EINVAL;
  }
  for (int k = 0; k < 3; ++k)
    if (reinterpret_cast<uintptr_t>(a->ptr[k]) % 16) {
      set_error("ewise: pointers must be 16-byte aligned");
      return TALLY_EINVAL;
    }
  p.nvec = n / per;
  const long long per_block = (long long)Ewise::kThreads * Ewise::kVec;
  const long long blocks = (p.nvec + per_block - 1) / per_block;
  if (blocks > 0x7fffffffLL) { set_error("ewise: grid too large"); return TALLY_EINVAL; }
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)blocks, 1, 1);
  inst->threads = Ewise::kThreads;
  inst->smem = 0;
  inst->alg_bytes = 16.0 * (double)p.nvec * (p.b ? 3.0 : 2.0);
  inst->alg_flops = (double)n;
  return TALLY_OK;
}

// ---------------------------------------------------------------- spin
// A cost-model kernel: every logical block occupies its CTA slot for exactly
// block_ns of device time.  It runs the reference's abstract workloads
// (KernelCostModel: blocks x threads x block duration, ref sim.py:77-111) on
// the real GPU, in all three shapes, so configs written for the simulator
// execute on the B200 through the same scheduler (cli.py).
struct SpinKernel {
  static constexpr int kThreads = 1024;   // upper bound; launched with the model's tpb
  struct Params {
    long long block_ns;
  };
  static __device__ __forceinline__ void run(const Params& p, uint3, uint3, char*) {
    if (threadIdx.x == 0) {
      const unsigned long long t0 = globaltimer();
      while (globaltimer() - t0 < (unsigned long long)p.block_ns) __nanosleep(128);
    }
    __syncthreads();
  }
};

static int bind_spin(const tally_kernel_args* a, Instance* inst) {
  SpinKernel::Params p{};
  const long long blocks = a->i[0], tpb = a->i[1];
  p.block_ns = a->i[2];
  if (blocks < 1 || blocks > 0x7fffffffLL || tpb < 1 || tpb > 1024 || p.block_ns < 0) {
    set_error("spin: need 1 <= blocks, 1 <= threads_per_block <= 1024, block_ns >= 0");
    return TALLY_EINVAL;
  }
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3((unsigned)blocks, 1, 1);
  inst->threads = (int)tpb;
  inst->smem = 0;
  return TALLY_OK;
}

// ---------------------------------------------------------------- L2 warm-up
// Not a Tally kernel kind: launched directly on a caller's stream
// (tally_l2_prefetch), typically inside a captured request graph.
__global__ void __launch_bounds__(128) k_l2_prefetch(const char* base, long long bytes) {
  constexpr long long kChunk = 32 << 10;
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  const long long nchunks = (bytes + kChunk - 1) / kChunk;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nchunks;
       c += (long long)gridDim.x * blockDim.x) {
    const long long off = c * kChunk;
    const unsigned sz = (unsigned)(min(kChunk, bytes - off) & ~15LL);
    if (sz)
      asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(base + off), "r"(sz),
                   "l"(pol)
                   : "memory");
  }
}

int launch_l2_prefetch(cudaStream_t s, const void* base, long long bytes) {
  if (!base || bytes < 16 || (reinterpret_cast<uintptr_t>(base) & 15)) {
    set_error("l2_prefetch: need a 16-byte aligned base and >= 16 bytes");
    return TALLY_EINVAL;
  }
  const long long nchunks = (bytes + (32 << 10) - 1) / (32 << 10);
  const int blocks = (int)std::min<long long>(16, (nchunks + 127) / 128);
  k_l2_prefetch<<<blocks, 128, 0, s>>>(static_cast<const char*>(base), bytes);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TALLY_OK : cuda_fail(e, "l2 prefetch launch");
}

template <class B>
static KernelKind make_kind(const char* name, int (*bind)(const tally_kernel_args*, Instance*)) {
  KernelKind k{};
  k.name = name;
  k.fn_original = reinterpret_cast<const void*>(&k_original<B>);
  k.fn_sliced = reinterpret_cast<const void*>(&k_sliced<B>);
  k.fn_ptb = reinterpret_cast<const void*>(&k_ptb<B>);
  k.bind = bind;
  k.setup = nullptr;
  return k;
}

int register_basic_kernels(KernelKind* out, int cap) {
  if (cap < 5) return 0;
  out[0] = make_kind<VecAddI64>("vecadd_i64", bind_vecadd_i64);
  out[1] = make_kind<VecAddF32>("vecadd_f32", bind_vecadd_f32);
  out[2] = make_kind<RowSumF32>("rowsum_f32", bind_rowsum_f32);
  out[3] = make_kind<SpinKernel>("spin", bind_spin);
  out[4] = make_kind<Ewise>("ewise", bind_ewise);
  return 5;
}

}  // namespace tally
