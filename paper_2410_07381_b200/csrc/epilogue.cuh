// Fused linear-layer epilogue: y = act(acc + bias[col] (+ res[row, col])),
// optionally also the pre-activation (GELU backward input).  Shared by the
// tcgen05 GEMM TMA-store epilogue (kernels_gemm.cu) and splitk_reduce
// (kernels_nn.cu); the same arithmetic as the bn_act kind, applied to the
// fp32 accumulator instead of a bf16-rounded intermediate.
#pragma once
#include <cuda_bf16.h>

namespace tally {

struct EpArgs {
  int on;                        // 0: no fused epilogue
  const float* bias;             // optional [C] fp32
  const __nv_bfloat16* res;      // optional residual, row-major with pitch ldr
  __nv_bfloat16* pre;            // optional pre-activation output (splitk_reduce; the GEMM uses a TMA map)
  long long ldr;                 // residual / pre row pitch (elements)
  int act;                       // 0 none, 1 ReLU, 2 GELU (tanh), 3 GELU (erf)
};

// Exact-erf GELU pieces, Phi(x) = 0.5 erfc(-x / sqrt 2) with the
// Chebyshev-fitted erfc (|relative error| < 1.2e-7; GELU within 1.1e-7 of
// float64 on [-12, 12]): t = 1 / (1 + |z| / 2), erfc(|z|) = t exp(-z^2 + P(t)),
// erfc(-|z|) = 2 - erfc(|z|).  Two MUFU ops and ~20 FMA-class instructions
// against ~35 for erff: BERT's bias + GELU and GELU-backward kernels were
// issue-bound on erff (C4: 26 + 25 launches of 16.7 M elements).
__device__ __forceinline__ float erfc_abs_p(float a, float z2) {   // erfc(a), a >= 0, z2 = a * a
  const float t = __fdividef(1.f, fmaf(0.5f, a, 1.f));
  float q = 0.17087277f;
  q = fmaf(q, t, -0.82215223f);
  q = fmaf(q, t, 1.48851587f);
  q = fmaf(q, t, -1.13520398f);
  q = fmaf(q, t, 0.27886807f);
  q = fmaf(q, t, -0.18628806f);
  q = fmaf(q, t, 0.09678418f);
  q = fmaf(q, t, 0.37409196f);
  q = fmaf(q, t, 1.00002368f);
  q = fmaf(q, t, -1.26551223f);
  return t * __expf(q - z2);
}
__device__ __forceinline__ float gelu_erf(float x) {
  const float a = fabsf(x) * 0.7071067811865476f;
  const float e = erfc_abs_p(a, a * a);               // erfc(|x| / sqrt 2)
  const float phi = x >= 0.f ? fmaf(-0.5f, e, 1.f) : 0.5f * e;
  return x * phi;
}
__device__ __forceinline__ float gelu_erf_grad_fast(float x) {   // Phi(x) + x phi(x)
  const float a = fabsf(x) * 0.7071067811865476f, z2 = a * a;
  const float e = erfc_abs_p(a, z2);
  const float Phi = x >= 0.f ? fmaf(-0.5f, e, 1.f) : 0.5f * e;
  return fmaf(x * 0.3989422804014327f, __expf(-z2), Phi);
}

// Two elements at a time: the polynomial and the multiplies as packed fp32
// pairs (fma/mul.rn.f32x2), the reciprocal and exponentials per element --
// these elementwise kernels are issue-bound (ncu: 82-84 % issue active).
__device__ __forceinline__ unsigned long long f2_pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// erfc(a0), erfc(a1) (a >= 0, z2 = a * a) -- erfc_abs_p on a pair
__device__ __forceinline__ void erfc_abs_p2(float a0, float a1, float z0, float z1, float& e0, float& e1) {
  const float t0 = __fdividef(1.f, fmaf(0.5f, a0, 1.f)), t1 = __fdividef(1.f, fmaf(0.5f, a1, 1.f));
  const unsigned long long t = f2_pack(t0, t1);
  unsigned long long q = f2_pack(0.17087277f, 0.17087277f);
  q = f2_fma(q, t, f2_pack(-0.82215223f, -0.82215223f));
  q = f2_fma(q, t, f2_pack(1.48851587f, 1.48851587f));
  q = f2_fma(q, t, f2_pack(-1.13520398f, -1.13520398f));
  q = f2_fma(q, t, f2_pack(0.27886807f, 0.27886807f));
  q = f2_fma(q, t, f2_pack(-0.18628806f, -0.18628806f));
  q = f2_fma(q, t, f2_pack(0.09678418f, 0.09678418f));
  q = f2_fma(q, t, f2_pack(0.37409196f, 0.37409196f));
  q = f2_fma(q, t, f2_pack(1.00002368f, 1.00002368f));
  q = f2_fma(q, t, f2_pack(-1.26551223f, -1.26551223f));
  float q0, q1;
  f2_unpack(q, q0, q1);
  e0 = t0 * __expf(q0 - z0);
  e1 = t1 * __expf(q1 - z1);
}
__device__ __forceinline__ void gelu_erf2(float& x0, float& x1) {
  const float a0 = fabsf(x0) * 0.7071067811865476f, a1 = fabsf(x1) * 0.7071067811865476f;
  float e0, e1;
  erfc_abs_p2(a0, a1, a0 * a0, a1 * a1, e0, e1);
  const float p0 = x0 >= 0.f ? fmaf(-0.5f, e0, 1.f) : 0.5f * e0;
  const float p1 = x1 >= 0.f ? fmaf(-0.5f, e1, 1.f) : 0.5f * e1;
  x0 *= p0;
  x1 *= p1;
}
__device__ __forceinline__ void gelu_erf_grad2(float x0, float x1, float& d0, float& d1) {
  const float a0 = fabsf(x0) * 0.7071067811865476f, a1 = fabsf(x1) * 0.7071067811865476f;
  const float z0 = a0 * a0, z1 = a1 * a1;
  float e0, e1;
  erfc_abs_p2(a0, a1, z0, z1, e0, e1);
  const float P0 = x0 >= 0.f ? fmaf(-0.5f, e0, 1.f) : 0.5f * e0;
  const float P1 = x1 >= 0.f ? fmaf(-0.5f, e1, 1.f) : 0.5f * e1;
  d0 = fmaf(x0 * 0.3989422804014327f, __expf(-z0), P0);
  d1 = fmaf(x1 * 0.3989422804014327f, __expf(-z1), P1);
}

__device__ __forceinline__ float ep_act(float x, int act) {
  if (act == 1) return fmaxf(x, 0.f);
  if (act == 2) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.f + tanhf(u));
  }
  if (act == 3) return gelu_erf(x);
  return x;
}

// 8 consecutive columns [col, col + 8) of row `row`: add bias (+ residual)
__device__ __forceinline__ void ep_bias_res8(const EpArgs& e, long long row, int col, float (&x)[8]) {
  if (e.bias != nullptr) {
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(e.bias + col));
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(e.bias + col + 4));
    x[0] += b0.x; x[1] += b0.y; x[2] += b0.z; x[3] += b0.w;
    x[4] += b1.x; x[5] += b1.y; x[6] += b1.z; x[7] += b1.w;
  }
  if (e.res != nullptr) {
    const uint4 r = __ldg(reinterpret_cast<const uint4*>(e.res + row * e.ldr + col));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]);
      x[2 * k] += f.x;
      x[2 * k + 1] += f.y;
    }
  }
}

}  // namespace tally
