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

__device__ __forceinline__ float ep_act(float x, int act) {
  if (act == 1) return fmaxf(x, 0.f);
  if (act == 2) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.f + tanhf(u));
  }
  if (act == 3) return 0.5f * x * (1.f + erff(x * 0.7071067811865476f));
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
