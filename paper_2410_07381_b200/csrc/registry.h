// Kernel-kind registry shared by the runtime and the kernel translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../../include/tally_b200.h"
#include "tally_device.cuh"

namespace tally {

constexpr int kMaxParamBytes = 1024;

// A bound kernel: the body's Params blob plus its logical geometry.
struct Instance {
  int kind = -1;
  alignas(64) unsigned char params[kMaxParamBytes];
  uint3 grid{1, 1, 1};         // logical grid
  int threads = 0;             // CTA size
  size_t smem = 0;             // dynamic shared memory per CTA
  double alg_bytes = 0;        // algorithmic HBM bytes of the whole logical grid
  double alg_flops = 0;        // algorithmic flops of the whole logical grid
  double alg_bytes_extra_ep = 0;   // fused-epilogue operand bytes (bias, residual, pre-activation)
  int preempt_units = 1;       // PTB preemption points per logical block (K-chunks for sgemm_tf32x3)
  // Per-instance device state that lives across the launches of one PTB
  // chain: the chunk-preemption resume ring (sgemm_tf32x3) or bn_stats'
  // reduction counters + second-level partials.  Zeroed at bind and when a
  // new PTB chain starts (start_count == 0); freed with the instance.
  void* resume_ring = nullptr;
  size_t resume_bytes = 0;
  // k_ptb return ring (bounded retirement, tally_device.cuh): allocated at the
  // first PTB launch; ret_pending = entries the last parked launch left
  unsigned long long* ret_ring = nullptr;
  unsigned long long ret_pending = 0;
  Instance() = default;
  Instance(const Instance&) = delete;
  Instance& operator=(const Instance&) = delete;
  ~Instance() {
    if (resume_ring) cudaFree(resume_ring);
    if (ret_ring) cudaFree(ret_ring);
  }
  unsigned long long total() const {
    return (unsigned long long)grid.x * grid.y * grid.z;
  }
};

// One hand-written kernel, three launch shapes (see tally_device.cuh).
struct KernelKind {
  const char* name;
  const void* fn_original;
  const void* fn_sliced;
  const void* fn_ptb;
  // Validate the generic argument block and fill inst (params, grid, threads,
  // smem).  Returns TALLY_OK or a negative code with tally::set_error().
  int (*bind)(const tally_kernel_args* a, Instance* inst);
  // Optional one-time setup (e.g. smem attribute) -- may be null.
  int (*setup)();
  // Not a kernel: 1 = host<->device copy (cudaMemcpyAsync on the launch
  // stream), 2 = captured CUDA graph (cudaGraphLaunch) -- data movement and
  // unmodified framework programs in a request pipeline.  Exempt from
  // transformation: Original shape only.
  int copy;
  // 1: the PTB shape has fine-grained suspension points and a footprint that
  // leaves room for high-priority CTAs (GEMM: 1 CTA/SM, ~90 regs/thread)
  int pausable;
  // 1: PTB launches read their preemption flag from mapped host memory
  // (few readers, one read per long logical block)
  int host_flag;
  // tcgen05 kinds: TMEM columns one CTA allocates (0 = none).  The runtime's
  // occupancy API reports 1 CTA/SM for these kernels even where smem,
  // registers and TMEM admit 2 (and the hardware co-schedules 2, ncu
  // r01_ncu_c2_summary); the PTB worker menu uses the resource-derived count.
  int tmem_cols;
  // CTAs per cluster (CTA-pair GEMMs: 2 -- one logical block per cluster,
  // PTB workers counted in CTAs, a multiple of it); 0 / 1 = no cluster
  int cluster;
  // 1: a tcgen05 kind whose PTB workers use the instance's return ring and
  // static first blocks like k_ptb (claim-ahead bf16 GEMMs)
  int ret_ring;
  // IR-JIT kinds (irjit.py): NVRTC-compiled module, launched with the driver API
  int jit;
  void* cu_fn[3];             // CUfunction for Original / Sliced / PTB
  unsigned jit_grid[3];       // logical grid of the IR kernel
  int jit_threads;
  long long jit_smem;
  char jit_name[64];
};


struct CopyParams {
  void* dst;
  const void* src;
  long long bytes;
};

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

// Registration hooks implemented by each kernel translation unit.
int register_basic_kernels(KernelKind* out, int cap);
int register_gemm_kernels(KernelKind* out, int cap);
int register_copy_kernels(KernelKind* out, int cap);
int register_nn_kernels(KernelKind* out, int cap);
int register_tf_kernels(KernelKind* out, int cap);
int launch_l2_prefetch(cudaStream_t s, const void* base, long long bytes);

}  // namespace tally
