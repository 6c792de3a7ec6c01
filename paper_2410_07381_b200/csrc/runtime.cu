// libtally_b200 runtime: device binding, kernel registry, per-priority
// streams, launch shapes (Original / Sliced / PTB), preemption flags and
// completion tracking.  Implements the first half of include/tally_b200.h;
// the policy runner lives in runner.cpp / cuda_device.cpp.
#include <cuda.h>
#include <cuda_runtime.h>
#include <time.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "registry.h"
#include "runtime.h"

namespace tally {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return TALLY_ECUDA;
}

long long host_now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (long long)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}

Runtime& rt() {
  static Runtime r;
  return r;
}

#define CK(call, what)                                  \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, what);  \
  } while (0)

__global__ void k_stamp(unsigned long long* slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *reinterpret_cast<volatile unsigned long long*>(slot) = t;
  __threadfence_system();
}

__global__ void k_flag_watch(const unsigned* flag, unsigned want, int host, unsigned long long* stamp) {
  if (threadIdx.x != 0) return;
  unsigned v;
  do {
    if (host) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
  } while (v != want);
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *reinterpret_cast<volatile unsigned long long*>(stamp) = t;
  __threadfence_system();
}

int Runtime::init(int dev, tally_gpu_info* out) {
  std::lock_guard<std::mutex> g(mu);
  if (inited) {
    if (dev != device) { set_error("tally already bound to device %d", device); return TALLY_EINVAL; }
    if (out) *out = info;
    return TALLY_OK;
  }
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    set_error("no CUDA device available (%s)", cudaGetErrorString(e));
    return TALLY_ENODEV;
  }
  if (dev < 0 || dev >= n) { set_error("device %d out of range (%d devices)", dev, n); return TALLY_EINVAL; }
  CK(cudaSetDevice(dev), "cudaSetDevice");
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, dev), "cudaGetDeviceProperties");
  if (p.major != 10) {
    set_error("libtally_b200 is built for sm_100a; device %d is sm_%d%d", dev, p.major, p.minor);
    return TALLY_ENODEV;
  }
  memset(&info, 0, sizeof(info));
  info.device = dev;
  info.num_sms = p.multiProcessorCount;
  info.max_threads_per_sm = p.maxThreadsPerMultiProcessor;
  info.max_blocks_per_sm = p.maxBlocksPerMultiProcessor;
  info.cc_major = p.major;
  info.cc_minor = p.minor;
  info.smem_per_sm = (long long)p.sharedMemPerMultiprocessor;
  info.hbm_bytes = (long long)p.totalGlobalMem;
  snprintf(info.name, sizeof(info.name), "%s", p.name);
  device = dev;

  nkinds = register_basic_kernels(kinds, kMaxKinds);
  nkinds += register_gemm_kernels(kinds + nkinds, kMaxKinds - nkinds);
  nkinds += register_copy_kernels(kinds + nkinds, kMaxKinds - nkinds);
  nkinds += register_nn_kernels(kinds + nkinds, kMaxKinds - nkinds);
  nkinds += register_tf_kernels(kinds + nkinds, kMaxKinds - nkinds);
  for (int k = 0; k < nkinds; ++k)
    if (kinds[k].setup) {
      int rc = kinds[k].setup();
      if (rc != TALLY_OK) return rc;
    }
  // Optional: one L1/shared carveout for every kernel (TALLY_CARVEOUT=max).
  // Off by default -- measured on B200 (profiles/r01_summary.md): a max-shared
  // carveout costs the streaming HP kernel ~25 % (fewer L1 lines for loads
  // in flight), more than co-residency gains.
  {
    // programmatic dependent launch on best-effort streams (default on;
    // TALLY_PDL=0 disables): BERT-large step 24.8 -> 23.1 ms, GPT-2 19.9 ->
    // 19.4, ResNet-50 11.8 -> 11.4 (tools/step_time.py)
    const char* pe = getenv("TALLY_PDL");
    pdl = !(pe != nullptr && pe[0] == '0');
  }
  const char* cv = getenv("TALLY_CARVEOUT");
  if (cv && strcmp(cv, "max") == 0) {
    for (int k = 0; k < nkinds; ++k) {
      if (kinds[k].copy) continue;
      for (const void* f : {kinds[k].fn_original, kinds[k].fn_sliced, kinds[k].fn_ptb})
        if (f) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    cudaSharedmemCarveoutMaxShared);
    }
    cudaGetLastError();
  }

  CK(cudaMalloc(&d_recs, sizeof(LaunchRec) * kMaxRecs), "cudaMalloc(launch records)");
  CK(cudaMemset(d_recs, 0, sizeof(LaunchRec) * kMaxRecs), "cudaMemset(launch records)");
  CK(cudaMalloc(&d_groups, sizeof(ExitGroup) * kMaxRecs * kMaxExitGroups), "cudaMalloc(exit groups)");
  CK(cudaMemset(d_groups, 0, sizeof(ExitGroup) * kMaxRecs * kMaxExitGroups), "cudaMemset(exit groups)");
  CK(cudaHostAlloc(&h_mirrors, sizeof(LaunchMirror) * kMaxRecs, cudaHostAllocMapped),
     "cudaHostAlloc(mirrors)");
  memset(h_mirrors, 0, sizeof(LaunchMirror) * kMaxRecs);
  CK(cudaHostGetDevicePointer(&d_mirrors, h_mirrors, 0), "mirror device pointer");
  CK(cudaHostAlloc(&h_flags, sizeof(unsigned) * kMaxRecs, cudaHostAllocMapped),
     "cudaHostAlloc(flags)");
  memset((void*)h_flags, 0, sizeof(unsigned) * kMaxRecs);
  CK(cudaHostGetDevicePointer(&d_hflags, (void*)h_flags, 0), "flag device pointer");
  CK(cudaMalloc(&d_chain, sizeof(unsigned) * kMaxChainStreams), "cudaMalloc(chain words)");
  CK(cudaMemset(d_chain, 0, sizeof(unsigned) * kMaxChainStreams), "cudaMemset(chain words)");
  CK(cudaHostAlloc(&h_chain, sizeof(unsigned) * kMaxChainStreams, cudaHostAllocMapped), "cudaHostAlloc(chain)");
  memset((void*)h_chain, 0, sizeof(unsigned) * kMaxChainStreams);
  CK(cudaHostGetDevicePointer(&d_hchain, (void*)h_chain, 0), "chain device pointer");
  chain_epoch.assign(kMaxChainStreams, 0u);
  CK(cudaMalloc(&d_pause, 64), "cudaMalloc(pause)");
  CK(cudaMemset(d_pause, 0, 64), "cudaMemset(pause)");
  CK(cudaHostAlloc(&h_stamp, 64, cudaHostAllocMapped), "cudaHostAlloc(stamp)");
  CK(cudaHostGetDevicePointer(&d_stamp, (void*)h_stamp, 0), "stamp device pointer");
  free_recs.clear();
  for (int i = kMaxRecs - 1; i >= 0; --i) free_recs.push_back(i);

  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priority range");
  prio_low = lo;
  prio_high = hi;
  CK(cudaStreamCreateWithPriority(&sig_stream, cudaStreamNonBlocking, hi), "signal stream");

  // driver stream memory operations: the flag write that preempts a PTB launch
  cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
  void* fn = nullptr;
  cudaError_t ge = cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &fn, 12000, cudaEnableDefault, &q);
  if (ge == cudaSuccess && q == cudaDriverEntryPointSuccess && fn)
    write32 = reinterpret_cast<WriteValue32Fn>(fn);
  info.stream_mem_ops = 0;
  info.stream_mem_ops_probe = (int)ge * 100000 + (int)q * 1000 + 999;
  if (write32) {
    // probe on record 0's flag
    CUresult r = write32((CUstream)sig_stream, (CUdeviceptr)&d_recs[0].flag, 0u, 0u);
    cudaError_t se = cudaStreamSynchronize(sig_stream);
    info.stream_mem_ops_probe = (int)q * 1000 + (int)r;
    if (r == CUDA_SUCCESS && se == cudaSuccess) info.stream_mem_ops = 1;
    cudaGetLastError();
  }
  flag_host = info.stream_mem_ops ? 0 : 1;
  auto entry = [](const char* sym) -> void* {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qq;
    if (cudaGetDriverEntryPointByVersion(sym, &f, 12000, cudaEnableDefault, &qq) != cudaSuccess ||
        qq != cudaDriverEntryPointSuccess)
      return nullptr;
    return f;
  };
  cu_module_load = reinterpret_cast<ModuleLoadDataFn>(entry("cuModuleLoadData"));
  cu_get_function = reinterpret_cast<ModuleGetFunctionFn>(entry("cuModuleGetFunction"));
  cu_launch = reinterpret_cast<LaunchKernelFn>(entry("cuLaunchKernel"));
  cu_occupancy = reinterpret_cast<OccupancyFn>(entry("cuOccupancyMaxActiveBlocksPerMultiprocessor"));
  cudaGetLastError();
  inited = true;
  if (out) *out = info;
  return TALLY_OK;
}

int Runtime::clock_offset(long long* off, long long* unc) {
  if (!inited) { set_error("tally_init first"); return TALLY_EINVAL; }
  long long best = 0, worst = 0;
  bool have = false;
  for (int i = 0; i < 24; ++i) {
    *h_stamp = 0ull;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    k_stamp<<<1, 1, 0, sig_stream>>>(d_stamp);
    CK(cudaGetLastError(), "k_stamp launch");
    long long seen = 0;
    const long long deadline = host_now_ns() + 2000000000LL;
    while (*h_stamp == 0ull) {
      if (host_now_ns() > deadline) { set_error("clock calibration timed out"); return TALLY_ECUDA; }
    }
    seen = host_now_ns();
    const long long s = seen - (long long)*h_stamp;
    CK(cudaStreamSynchronize(sig_stream), "k_stamp sync");
    if (i < 4) continue;   // warm-up
    if (!have || s < best) best = s;
    if (!have || s > worst) worst = s;
    have = true;
  }
  if (off) *off = best;
  if (unc) *unc = worst - best;
  return TALLY_OK;
}

int Runtime::alloc_rec(int* out) {
  // Reclaim records of launches whose kernel has fully exited, oldest first
  // and only while they are done: O(1) amortised, no scan stalls the daemon.
  while (!zombies.empty() && (free_recs.empty() || zombies.size() > 64)) {
    if (cudaEventQuery(zombies.front().second) != cudaSuccess) break;
    free_recs.push_back(zombies.front().first);
    release_event(zombies.front().second);
    zombies.pop_front();
  }
  cudaGetLastError();
  if (free_recs.empty()) { set_error("out of PTB launch records"); return TALLY_EBUSY; }
  *out = free_recs.back();
  free_recs.pop_back();
  return TALLY_OK;
}

cudaEvent_t Runtime::get_event(bool timed) {
  auto& pool = timed ? timed_events : plain_events;
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, timed ? cudaEventDefault : cudaEventDisableTiming);
  event_timed[e] = timed;
  return e;
}

void Runtime::release_event(cudaEvent_t e) {
  if (!e) return;
  (event_timed[e] ? timed_events : plain_events).push_back(e);
}

int Runtime::launch(int kernel, int stream, const tally_launch_desc* d, int* out) {
  if (!inited) { set_error("tally_init first"); return TALLY_EINVAL; }
  if (!d || !out) { set_error("null descriptor"); return TALLY_EINVAL; }
  if (kernel < 0 || kernel >= (int)instances.size() || !instances[kernel]) {
    set_error("unknown kernel instance %d", kernel);
    return TALLY_EINVAL;
  }
  if (stream < 0 || stream >= (int)streams.size() || !streams[stream]) {
    set_error("unknown stream %d", stream);
    return TALLY_EINVAL;
  }
  const Instance& in = *instances[kernel];
  const KernelKind& kk = kinds[in.kind];
  cudaStream_t st = streams[stream];
  const unsigned long long total = in.total();

  auto L = std::make_unique<Launch>();
  L->kernel = kernel;
  L->stream = stream;
  L->shape = d->shape;
  L->timed = d->timed != 0;
  L->host_submit = host_now_ns();

  SliceArgs s{};
  s.grid = in.grid;
  s.exec_count = d->exec_count;
  s.block_log = d->block_log;
  PtbArgs pa{};
  const void* fn = nullptr;
  dim3 grid;
  void* args[2] = {const_cast<unsigned char*>(in.params), nullptr};

  if (kk.copy) {
    if (d->shape != TALLY_SHAPE_ORIGINAL) {
      set_error("%s: copies are exempt from slicing / preemption (Original shape only)", kk.name);
      return TALLY_ETRANSFORM;
    }
    CopyParams cp;
    memcpy(&cp, in.params, sizeof(cp));
    L->count = 1;
    if (L->timed) {
      L->ev_start = get_event(true);
      cudaEventRecord(L->ev_start, st);
    }
    cudaError_t e = kk.copy == 2
                        ? cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(cp.dst), st)
                        : cudaMemcpyAsync(cp.dst, cp.src, (size_t)cp.bytes, cudaMemcpyDefault, st);
    if (e != cudaSuccess) {
      release_event(L->ev_start);
      return cuda_fail(e, kk.name);
    }
    L->ev_end = get_event(L->timed);
    cudaEventRecord(L->ev_end, st);
    L->active = true;
    std::lock_guard<std::mutex> g(mu);
    int id;
    if (!free_launch_ids.empty()) {
      id = free_launch_ids.back();
      free_launch_ids.pop_back();
      launches[id] = std::move(L);
    } else {
      id = (int)launches.size();
      launches.push_back(std::move(L));
    }
    *out = id;
    return TALLY_OK;
  }

  switch (d->shape) {
    case TALLY_SHAPE_ORIGINAL:
      fn = kk.fn_original;
      // (cluster kinds: one cluster of kk.cluster CTAs per logical block, 1-D grids)
      grid = dim3(in.grid.x * (unsigned)std::max(1, kk.cluster), in.grid.y, in.grid.z);
      args[1] = &s;
      L->count = (long long)total;
      break;
    case TALLY_SHAPE_SLICED:
      fn = kk.fn_sliced;
      if (d->linear) {
        if (d->linear_offset < 0 || d->count < 1 ||
            (unsigned long long)(d->linear_offset + d->count) > total || d->count > 0x7fffffffLL) {
          set_error("slice [%lld, +%lld) outside %llu logical blocks", d->linear_offset, d->count, total);
          return TALLY_EINVAL;
        }
        s.linear = 1;
        s.linear_offset = (unsigned long long)d->linear_offset;
        grid = dim3((unsigned)d->count * (unsigned)std::max(1, kk.cluster), 1, 1);
        L->count = d->count;
      } else {
        if (d->sub_x < 1 || d->sub_y < 1 || d->sub_z < 1 || d->off_x + d->sub_x > in.grid.x ||
            d->off_y + d->sub_y > in.grid.y || d->off_z + d->sub_z > in.grid.z) {
          set_error("sub-grid outside the logical grid");
          return TALLY_EINVAL;
        }
        s.offset = make_uint3(d->off_x, d->off_y, d->off_z);
        grid = dim3(d->sub_x * (unsigned)std::max(1, kk.cluster), d->sub_y, d->sub_z);
        L->count = (long long)d->sub_x * d->sub_y * d->sub_z;
      }
      args[1] = &s;
      break;
    case TALLY_SHAPE_PTB: {
      if (d->workers < 1) { set_error("worker count must be >= 1"); return TALLY_EINVAL; }
      if (d->start_count < 0) { set_error("persisted counter must be >= 0"); return TALLY_EINVAL; }
      int rec = -1;
      int rc = alloc_rec(&rec);
      if (rc != TALLY_OK) return rc;
      unsigned ser = next_serial.fetch_add(1) + 1;
      if (ser == 0) ser = next_serial.fetch_add(1) + 1;
      L->rec = rec;
      L->serial = ser;
      L->start_count = d->start_count;
      L->workers = d->workers;
      h_mirrors[rec].serial = 0;
      h_flags[rec] = 0;
      if (in.resume_ring != nullptr && d->start_count == 0) {
        // a new chain: no half-done tiles carried over from an earlier one
        cudaError_t me = cudaMemsetAsync(in.resume_ring, 0, in.resume_bytes, st);
        if (me != cudaSuccess) { free_recs.push_back(rec); return cuda_fail(me, "resume ring reset"); }
      }
      pa.ret_ring = nullptr;
      pa.ret_pending = 0;
      pa.static_n = 0;
      pa.claim_n = 1;
      if ((kk.tmem_cols == 0 || kk.ret_ring) && !kk.copy) {
        // generic k_ptb workers and claim-ahead GEMM workers: the instance's
        // return ring (bounded retirement)
        Instance& mi = *instances[kernel];
        if (mi.ret_ring == nullptr) {
          const size_t bytes = (2 + kRetCap) * sizeof(unsigned long long);
          cudaError_t me = cudaMalloc(&mi.ret_ring, bytes);
          if (me == cudaSuccess) me = cudaMemset(mi.ret_ring, 0, bytes);
          if (me != cudaSuccess) { free_recs.push_back(rec); return cuda_fail(me, "return ring"); }
          mi.ret_pending = 0;
        }
        if (d->start_count == 0 && mi.ret_pending > 0) {
          // a new chain: drop blocks an abandoned one handed back
          cudaError_t me = cudaMemsetAsync(mi.ret_ring, 0, 2 * sizeof(unsigned long long), st);
          if (me != cudaSuccess) { free_recs.push_back(rec); return cuda_fail(me, "return ring reset"); }
          mi.ret_pending = 0;
        }
        pa.ret_ring = mi.ret_ring;
        pa.ret_pending = mi.ret_pending;
        // static first blocks (no claim round trip) unless the launch resumes
        // handed-back blocks or runs the counter-triggered test preemption
        // (cluster kinds: one static block per cluster of workers)
        if (mi.ret_pending == 0 && d->preempt_at < 0 && (unsigned long long)d->start_count < total)
          pa.static_n = std::min<unsigned long long>((unsigned long long)(d->workers / std::max(1, kk.cluster)),
                                                     total - (unsigned long long)d->start_count);
        // batched claims for generic workers with many short blocks each:
        // ~8+ blocks per worker -> up to 4 per claim, bounded so that every
        // worker's handed-back blocks (< 2 batches) fit the return ring
        if (kk.tmem_cols == 0 && d->preempt_at < 0) {
          const unsigned long long left = total - std::min<unsigned long long>(total, (unsigned long long)d->start_count);
          const unsigned long long per = left / (unsigned long long)std::max(1, d->workers);
          int cn = (int)std::min<unsigned long long>(4ull, std::max<unsigned long long>(1ull, per / 8ull));
          while (cn > 1 && (unsigned long long)d->workers * (2ull * cn - 1ull) > kRetCap) --cn;
          pa.claim_n = cn;
        }
      }
      pa.grp = d_groups + (size_t)rec * kMaxExitGroups;
      if (d->workers > kMaxExitGroups * kExitGroupSize) {
        free_recs.push_back(rec);
        set_error("at most %d PTB workers", kMaxExitGroups * kExitGroupSize);
        return TALLY_EINVAL;
      }
      std::atomic_thread_fence(std::memory_order_seq_cst);
      pa.rec = d_recs + rec;
      // few, rare readers (a GEMM producer per SM, once per tile) -> the flag
      // can live in mapped host memory: ~2 us propagation instead of ~6 us
      const int use_host = flag_host || kk.host_flag;
      pa.flag_is_host = use_host;
      pa.park_at = ser;
      pa.chain_dev = nullptr;
      pa.chain_host = nullptr;
      if (d->chain) {
        // every launch queued on this stream shares one preemption word: a
        // single write parks the running launch and the ones behind it
        if (stream >= kMaxChainStreams) { free_recs.push_back(rec); set_error("chain stream id out of range"); return TALLY_EINVAL; }
        {
          std::lock_guard<std::mutex> g(mu);
          pa.park_at = chain_epoch[(size_t)stream] + 1u;
        }
        pa.chain_dev = d_chain + stream;
        pa.chain_host = d_hchain + stream;
        pa.flag = use_host ? (d_hchain + stream) : (d_chain + stream);
        L->chain = true;
        L->chain_stream = stream;
      } else {
        pa.flag = use_host ? (d_hflags + rec) : &d_recs[rec].flag;
      }
      L->park_at = pa.park_at;
      L->flag_host = use_host;
      pa.mirror = d_mirrors + rec;
      pa.serial = ser;
      pa.start = (unsigned long long)d->start_count;
      pa.total = total;
      pa.preempt_at = d->preempt_at;
      pa.grid = in.grid;
      pa.exec_count = d->exec_count;
      pa.worker_log = d->worker_log;
      pa.block_log = d->block_log;
      pa.pause = (d->pausable && kk.pausable) ? d_pause : nullptr;
      fn = kk.fn_ptb;
      grid = dim3((unsigned)d->workers, 1, 1);
      if (kk.cluster > 1 && d->workers % kk.cluster) {
        free_recs.push_back(rec);
        set_error("%s: PTB workers must be a multiple of the cluster size %d", kk.name, kk.cluster);
        return TALLY_EINVAL;
      }
      args[1] = &pa;
      L->count = (long long)total;
      break;
    }
    default:
      set_error("unknown launch shape %d", d->shape);
      return TALLY_EINVAL;
  }

  if (L->timed) {
    L->ev_start = get_event(true);
    cudaEventRecord(L->ev_start, st);
  }
  cudaError_t e = cudaSuccess;
  if (kk.jit) {
    const int idx = d->shape == TALLY_SHAPE_ORIGINAL ? 0 : (d->shape == TALLY_SHAPE_SLICED ? 1 : 2);
    CUresult cr = cu_launch((CUfunction)kk.cu_fn[idx], grid.x, grid.y, grid.z, (unsigned)in.threads, 1, 1,
                            (unsigned)in.smem, (CUstream)st, args, nullptr);
    if (cr != CUDA_SUCCESS) e = cudaErrorLaunchFailure;
  } else if (kk.cluster > 1 || (pdl && stream_be[(size_t)stream] && !L->timed)) {
    // CTA-pair kinds: a cluster launch (the pair shares one tile, cta_group::2);
    // best-effort streams with TALLY_PDL: programmatic dependent launch
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(in.threads);
    cfg.dynamicSmemBytes = in.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    unsigned na = 0;
    if (kk.cluster > 1) {
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = (unsigned)kk.cluster;
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = 1;
      ++na;
    }
    if (pdl && stream_be[(size_t)stream] && !L->timed) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    e = cudaLaunchKernelExC(&cfg, fn, args);
  } else {
    e = cudaLaunchKernel(fn, grid, dim3(in.threads), args, in.smem, st);
  }
  if (e != cudaSuccess) {
    if (L->rec >= 0) free_recs.push_back(L->rec);
    release_event(L->ev_start);
    return cuda_fail(e, kk.name);
  }
  L->ev_end = get_event(L->timed);
  cudaEventRecord(L->ev_end, st);
  L->active = true;

  std::lock_guard<std::mutex> g(mu);
  int id;
  if (!free_launch_ids.empty()) {
    id = free_launch_ids.back();
    free_launch_ids.pop_back();
    launches[id] = std::move(L);
  } else {
    id = (int)launches.size();
    launches.push_back(std::move(L));
  }
  *out = id;
  return TALLY_OK;
}

Launch* Runtime::get_launch(int id) {
  if (id < 0 || id >= (int)launches.size() || !launches[id]) {
    set_error("unknown launch %d", id);
    return nullptr;
  }
  return launches[id].get();
}

// Update the cached state; returns true when the launch has finished.
bool Runtime::poll(Launch* L) {
  if (L->finished) return true;
  if (L->shape == TALLY_SHAPE_PTB) {
    volatile LaunchMirror* m = &h_mirrors[L->rec];
    if (m->serial != L->serial) {
      // The last worker publishes the mirror; a kernel that faulted or was
      // aborted never does.  Every 256th poll (the mirror read is a plain
      // load, the event query a driver call) ask the end event: an error, or
      // a completed kernel whose mirror is still unpublished, is a failure
      // the caller must see instead of waiting forever.
      if ((++L->polls & 255u) != 0u) return false;
      const cudaError_t e = cudaEventQuery(L->ev_end);
      if (e == cudaErrorNotReady) return false;
      if (e == cudaSuccess) {
        std::atomic_thread_fence(std::memory_order_acquire);
        if (m->serial == L->serial) return poll(L);
        L->error = cudaErrorLaunchFailure;
      } else {
        L->error = e;
      }
      return false;
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    L->claims = (long long)m->claims;
    L->gt_first_stop = (long long)m->t_first_stop;
    L->gt_last_exit = (long long)m->t_last_exit;
    L->gt_last_busy_exit = (long long)m->t_last_busy_exit;
    L->gt_first_start = (long long)m->t_first_start;
    L->parked = (m->status == kMirrorParked);
    L->finished = true;
    if (L->kernel >= 0 && L->kernel < (int)instances.size() && instances[L->kernel] &&
        instances[L->kernel]->ret_ring != nullptr)
      instances[L->kernel]->ret_pending = m->ret_pending;
    return true;
  }
  cudaError_t e = cudaEventQuery(L->ev_end);
  if (e == cudaSuccess) {
    L->finished = true;
    return true;
  }
  if (e != cudaErrorNotReady) L->error = e;
  return false;
}

void Runtime::fill_state(const Launch* L, tally_launch_state* o) {
  memset(o, 0, sizeof(*o));
  o->done = L->finished && !L->parked;
  o->parked = L->parked;
  o->preempted = L->preempted.load();
  o->claims = L->claims;
  o->task_counter = L->shape == TALLY_SHAPE_PTB ? L->start_count + L->claims : 0;
  o->gt_first_start = L->gt_first_start;
  o->gt_first_stop = L->gt_first_stop;
  o->gt_last_exit = L->gt_last_exit;
  o->gt_last_busy_exit = L->gt_last_busy_exit;
  o->host_submit_ns = L->host_submit;
  o->host_preempt_ns = L->host_preempt;
}

int Runtime::preempt(int id) {
  std::lock_guard<std::mutex> g(mu);
  Launch* L = get_launch(id);
  if (!L) return TALLY_EINVAL;
  if (L->shape != TALLY_SHAPE_PTB) { set_error("launch %d: not a Ptb launch", id); return TALLY_EINVAL; }
  if (L->finished) { set_error("launch %d: not in flight", id); return TALLY_EINVAL; }
  bool expected = false;
  if (!L->preempted.compare_exchange_strong(expected, true)) return TALLY_OK;
  L->host_preempt = host_now_ns();
  if (L->chain) {
    // raise the stream's epoch to this launch's park_at (once per epoch): the
    // mapped host word first (GEMM producers poll it, ~2 us), then the device
    // word the streaming kinds poll
    unsigned& cur = chain_epoch[(size_t)L->chain_stream];
    if ((int)(cur - L->park_at) >= 0) return TALLY_OK;
    cur = L->park_at;
    h_chain[L->chain_stream] = cur;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    if (!write32) {
      CK(cudaMemcpyAsync(d_chain + L->chain_stream, &cur, sizeof(unsigned), cudaMemcpyHostToDevice, sig_stream),
         "chain flag write");
      return TALLY_OK;
    }
    CUresult r = write32((CUstream)sig_stream, (CUdeviceptr)(d_chain + L->chain_stream), cur, 0u);
    if (r != CUDA_SUCCESS) { set_error("cuStreamWriteValue32 failed (%d)", (int)r); return TALLY_ECUDA; }
    return TALLY_OK;
  }
  if (L->flag_host) {
    reinterpret_cast<volatile unsigned*>(h_flags)[L->rec] = L->serial;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    return TALLY_OK;
  }
  CUresult r = write32((CUstream)sig_stream, (CUdeviceptr)&d_recs[L->rec].flag, L->serial, 0u);
  if (r != CUDA_SUCCESS) { set_error("cuStreamWriteValue32 failed (%d)", (int)r); return TALLY_ECUDA; }
  return TALLY_OK;
}

static int bind_jit(const tally_kernel_args* a, Instance* inst) {
  const KernelKind& kk = rt().kinds[inst->kind];
  JitParams p;
  memset(&p, 0, sizeof(p));
  p.mem = static_cast<long long*>(a->ptr[0]);
  p.fault = static_cast<unsigned long long*>(a->ptr[1]);
  p.nwords = a->i[0];
  for (int k = 0; k < 7; ++k) p.args[k] = a->i[k + 1];
  if (!p.mem || p.nwords < 0 || !p.fault) {
    set_error("%s: need mem, fault word and nwords", kk.name);
    return TALLY_EINVAL;
  }
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3(kk.jit_grid[0], kk.jit_grid[1], kk.jit_grid[2]);
  inst->threads = kk.jit_threads;
  inst->smem = (size_t)kk.jit_smem;
  return TALLY_OK;
}

int Runtime::jit_register(const char* name, const void* image, const char* syms[3], const unsigned grid[3],
                          int threads, long long smem, int* out_kind) {
  if (!inited) { set_error("tally_init first"); return TALLY_EINVAL; }
  if (!cu_module_load || !cu_get_function || !cu_launch) { set_error("driver module API unavailable"); return TALLY_ENODEV; }
  if (nkinds >= kMaxKinds) { set_error("too many kernel kinds"); return TALLY_ENOMEM; }
  if (threads < 1 || threads > 1024 || smem < 0 || smem > 48 * 1024 || !grid[0] || !grid[1] || !grid[2]) {
    set_error("jit kernel geometry out of range");
    return TALLY_EINVAL;
  }
  // one module per image: a batch of IR kernels compiled into one cubin
  // registers each kind against the same image
  CUmodule mod;
  CUresult r = CUDA_SUCCESS;
  auto mit = jit_modules.find(image);
  if (mit != jit_modules.end()) {
    mod = (CUmodule)mit->second;
  } else {
    r = cu_module_load(&mod, image);
    if (r != CUDA_SUCCESS) { set_error("cuModuleLoadData failed (%d)", (int)r); return TALLY_ECUDA; }
    jit_modules[image] = (void*)mod;
  }
  KernelKind& k = kinds[nkinds];
  memset(&k, 0, sizeof(k));
  snprintf(k.jit_name, sizeof(k.jit_name), "%s", name);
  k.name = k.jit_name;
  k.jit = 1;
  for (int i = 0; i < 3; ++i) {
    CUfunction f;
    r = cu_get_function(&f, mod, syms[i]);
    if (r != CUDA_SUCCESS) { set_error("cuModuleGetFunction(%s) failed (%d)", syms[i], (int)r); return TALLY_ECUDA; }
    k.cu_fn[i] = (void*)f;
    k.jit_grid[i] = grid[i];
  }
  k.jit_threads = threads;
  k.jit_smem = smem;
  k.bind = bind_jit;
  *out_kind = nkinds++;
  return TALLY_OK;
}

int Runtime::set_pause(int on) {
  if (!inited) { set_error("tally_init first"); return TALLY_EINVAL; }
  on = on ? 1 : 0;
  if (on == pause_on) return TALLY_OK;
  pause_on = on;
  if (write32) {
    CUresult r = write32((CUstream)sig_stream, (CUdeviceptr)d_pause, (cuuint32_t)on, 0u);
    if (r != CUDA_SUCCESS) { set_error("cuStreamWriteValue32(pause) failed (%d)", (int)r); return TALLY_ECUDA; }
    return TALLY_OK;
  }
  const unsigned v = (unsigned)on;
  CK(cudaMemcpyAsync(d_pause, &v, sizeof(v), cudaMemcpyHostToDevice, sig_stream), "pause write");
  CK(cudaStreamSynchronize(sig_stream), "pause write");
  return TALLY_OK;
}

int Runtime::release(int id) {
  std::lock_guard<std::mutex> g(mu);
  Launch* L = get_launch(id);
  if (!L) return TALLY_EINVAL;
  if (!L->finished && !poll(L)) { set_error("launch %d still in flight", id); return TALLY_EBUSY; }
  if (L->rec >= 0) {
    zombies.emplace_back(L->rec, L->ev_end);   // record reusable once the kernel fully exited
    L->ev_end = nullptr;
  }
  release_event(L->ev_start);
  release_event(L->ev_end);
  launches[id].reset();
  free_launch_ids.push_back(id);
  return TALLY_OK;
}

static int bind_memcpy(const tally_kernel_args* a, Instance* inst) {
  CopyParams p;
  p.dst = a->ptr[0];
  p.src = a->ptr[1];
  p.bytes = a->i[0];
  if (!p.dst || !p.src || p.bytes < 1) {
    set_error("memcpy: need dst, src and bytes >= 1");
    return TALLY_EINVAL;
  }
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3(1, 1, 1);
  inst->threads = 1;
  inst->alg_bytes = (double)p.bytes;
  return TALLY_OK;
}

static int bind_graph(const tally_kernel_args* a, Instance* inst) {
  CopyParams p;
  p.dst = a->ptr[0];   // cudaGraphExec_t
  p.src = nullptr;
  p.bytes = 0;
  if (!p.dst) {
    set_error("cuda_graph: need an instantiated graph (cudaGraphExec_t)");
    return TALLY_EINVAL;
  }
  memcpy(inst->params, &p, sizeof(p));
  inst->grid = make_uint3(1, 1, 1);
  inst->threads = 1;
  return TALLY_OK;
}

int register_copy_kernels(KernelKind* out, int cap) {
  if (cap < 2) return 0;
  KernelKind k{};
  k.name = "memcpy";
  k.bind = bind_memcpy;
  k.copy = 1;
  out[0] = k;
  KernelKind g{};
  g.name = "cuda_graph";   // an unmodified PyTorch program (captured CUDA graph) as one exempt step
  g.bind = bind_graph;
  g.copy = 2;
  out[1] = g;
  return 2;
}

}  // namespace tally

using namespace tally;

extern "C" {

int tally_abi_version(void) { return TALLY_ABI_VERSION; }
const char* tally_last_error(void) { return g_err; }
long long tally_now_ns(void) { return host_now_ns(); }

int tally_init(int device, tally_gpu_info* out) { return rt().init(device, out); }

int tally_shutdown(void) {
  Runtime& r = rt();
  if (!r.inited) return TALLY_OK;
  cudaDeviceSynchronize();
  r.instances.clear();
  for (auto s : r.streams)
    if (s) cudaStreamDestroy(s);
  r.streams.clear();
  r.launches.clear();
  r.free_launch_ids.clear();
  r.zombies.clear();
  return TALLY_OK;
}

int tally_clock_offset(long long* off, long long* unc) { return rt().clock_offset(off, unc); }

int tally_set_flag_mode(int host_mapped) {
  Runtime& r = rt();
  if (!r.inited) { set_error("tally_init first"); return TALLY_EINVAL; }
  if (!host_mapped && !r.info.stream_mem_ops) {
    set_error("stream memory operations unavailable; only host-mapped flags");
    return TALLY_EINVAL;
  }
  r.flag_host = host_mapped ? 1 : 0;
  return TALLY_OK;
}

// Diagnostic: flag propagation latency, host signal -> a spinning device
// reader observes it.  mode 0: device-resident flag written with
// cuStreamWriteValue32 on the signal stream; mode 1: mapped host flag written
// by a host store.
int tally_l2_persist(void* cuda_stream, const void* base, long long bytes, float hit_ratio,
                     long long* out_window_bytes) {
  if (!base || bytes <= 0 || hit_ratio < 0.f || hit_ratio > 1.f) {
    set_error("l2_persist: need base, bytes > 0, 0 <= hit_ratio <= 1");
    return TALLY_EINVAL;
  }
  int dev = 0, max_win = 0, max_persist = 0;
  CK(cudaGetDevice(&dev), "cudaGetDevice");
  CK(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev), "max window");
  CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev), "max persisting L2");
  const size_t win = (size_t)std::min<long long>(bytes, max_win);
  CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(win, (size_t)max_persist)),
     "persisting L2 limit");
  cudaStreamAttrValue v{};
  v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  v.accessPolicyWindow.num_bytes = win;
  v.accessPolicyWindow.hitRatio = hit_ratio;
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  CK(cudaStreamSetAttribute(static_cast<cudaStream_t>(cuda_stream), cudaStreamAttributeAccessPolicyWindow, &v),
     "access policy window");
  if (out_window_bytes) *out_window_bytes = (long long)win;
  return TALLY_OK;
}

int tally_graph_l2_persist(void* cuda_graph, const void* base, long long bytes, float hit_ratio, int* out_nodes) {
  if (!cuda_graph || !base || bytes <= 0 || hit_ratio < 0.f || hit_ratio > 1.f) {
    set_error("graph_l2_persist: need graph, base, bytes > 0, 0 <= hit_ratio <= 1");
    return TALLY_EINVAL;
  }
  int dev = 0, max_win = 0, max_persist = 0;
  CK(cudaGetDevice(&dev), "cudaGetDevice");
  CK(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev), "max window");
  CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev), "max persisting L2");
  const size_t win = (size_t)std::min<long long>(bytes, max_win);
  CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(win, (size_t)max_persist)),
     "persisting L2 limit");
  cudaGraph_t g = static_cast<cudaGraph_t>(cuda_graph);
  size_t n = 0;
  CK(cudaGraphGetNodes(g, nullptr, &n), "graph nodes");
  std::vector<cudaGraphNode_t> nodes(n);
  CK(cudaGraphGetNodes(g, nodes.data(), &n), "graph nodes");
  cudaKernelNodeAttrValue v{};
  v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  v.accessPolicyWindow.num_bytes = win;
  v.accessPolicyWindow.hitRatio = hit_ratio;
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  int k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    CK(cudaGraphNodeGetType(nd, &t), "node type");
    if (t != cudaGraphNodeTypeKernel) continue;
    CK(cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &v), "node window");
    ++k;
  }
  if (out_nodes) *out_nodes = k;
  return TALLY_OK;
}

int tally_l2_prefetch(void* cuda_stream, const void* base, long long bytes) {
  return launch_l2_prefetch(static_cast<cudaStream_t>(cuda_stream), base, bytes);
}

int tally_probe_flag_latency(int mode, int iters, long long* out_median_ns, long long* out_max_ns) {
  Runtime& r = rt();
  if (!r.inited) { set_error("tally_init first"); return TALLY_EINVAL; }
  if (mode == 0 && !r.write32) { set_error("no stream memory operations"); return TALLY_EINVAL; }
  long long off = 0, unc = 0;
  int rc = r.clock_offset(&off, &unc);
  if (rc != TALLY_OK) return rc;
  cudaStream_t ws;
  CK(cudaStreamCreateWithFlags(&ws, cudaStreamNonBlocking), "probe stream");
  unsigned* dflag = nullptr;
  CK(cudaMalloc(&dflag, 64), "probe flag");
  CK(cudaMemset(dflag, 0, 64), "probe flag");
  std::vector<long long> lat;
  for (int i = 0; i < iters; ++i) {
    const unsigned want = (unsigned)(i + 1);
    *r.h_stamp = 0ull;
    const unsigned* f = mode == 0 ? dflag : r.d_hflags + (Runtime::kMaxRecs - 1);
    r.h_flags[Runtime::kMaxRecs - 1] = 0;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    k_flag_watch<<<1, 32, 0, ws>>>(f, want, mode, r.d_stamp);
    CK(cudaGetLastError(), "probe launch");
    const long long t_arm = host_now_ns() + 200000;   // let the watcher start spinning
    while (host_now_ns() < t_arm) {}
    const long long t0 = host_now_ns();
    if (mode == 0) {
      if (r.write32((CUstream)r.sig_stream, (CUdeviceptr)dflag, want, 0u) != CUDA_SUCCESS) {
        set_error("cuStreamWriteValue32 failed");
        return TALLY_ECUDA;
      }
    } else {
      r.h_flags[Runtime::kMaxRecs - 1] = want;
      std::atomic_thread_fence(std::memory_order_seq_cst);
    }
    CK(cudaStreamSynchronize(ws), "probe sync");
    lat.push_back((long long)*r.h_stamp + off - t0);
  }
  cudaFree(dflag);
  cudaStreamDestroy(ws);
  std::sort(lat.begin(), lat.end());
  if (out_median_ns) *out_median_ns = lat[lat.size() / 2];
  if (out_max_ns) *out_max_ns = lat.back();
  return TALLY_OK;
}

int tally_kernel_kind_count(void) {
  Runtime& r = rt();
  if (!r.inited) {
    // registry is static; allow listing without a device
    static KernelKind tmp[64];
    int n = register_basic_kernels(tmp, 64);
    n += register_gemm_kernels(tmp + n, 64 - n);
    return n + register_copy_kernels(tmp + n, 64 - n);
  }
  return r.nkinds;
}

const char* tally_kernel_kind_name(int kind) {
  static KernelKind tmp[64];
  static int n = -1;
  if (n < 0) {
    n = register_basic_kernels(tmp, 64);
    n += register_gemm_kernels(tmp + n, 64 - n);
    n += register_copy_kernels(tmp + n, 64 - n);
  }
  if (kind < 0 || kind >= n) return nullptr;
  return tmp[kind].name;
}

int tally_kernel_create(const char* kind, const tally_kernel_args* args, int* out) {
  Runtime& r = rt();
  if (!r.inited) { set_error("tally_init first"); return TALLY_EINVAL; }
  if (!kind || !args || !out) { set_error("null argument"); return TALLY_EINVAL; }
  for (int k = 0; k < r.nkinds; ++k) {
    if (strcmp(r.kinds[k].name, kind) != 0) continue;
    auto in = std::make_unique<Instance>();
    in->kind = k;
    int rc = r.kinds[k].bind(args, in.get());
    if (rc != TALLY_OK) return rc;
    *out = (int)r.instances.size();
    r.instances.push_back(std::move(in));
    return TALLY_OK;
  }
  set_error("unknown kernel kind '%s'", kind);
  return TALLY_EINVAL;
}

int tally_kernel_info_get(int kernel, tally_kernel_info* o) {
  Runtime& r = rt();
  if (kernel < 0 || kernel >= (int)r.instances.size() || !r.instances[kernel]) {
    set_error("unknown kernel instance %d", kernel);
    return TALLY_EINVAL;
  }
  const Instance& in = *r.instances[kernel];
  const KernelKind& kk = r.kinds[in.kind];
  memset(o, 0, sizeof(*o));
  o->grid_x = in.grid.x;
  o->grid_y = in.grid.y;
  o->grid_z = in.grid.z;
  o->total_blocks = (long long)in.total();
  o->threads_per_block = in.threads;
  o->smem_bytes = (long long)in.smem;
  o->alg_bytes = in.alg_bytes;
  o->alg_flops = in.alg_flops;
  o->preempt_units = in.preempt_units;
  o->cluster = std::max(1, kk.cluster);
  int occ = 0;
  if (kk.copy) return TALLY_OK;
  if (kk.jit) {
    if (r.cu_occupancy) {
      r.cu_occupancy(&occ, (CUfunction)kk.cu_fn[2], in.threads, in.smem);
      o->occupancy_ptb = occ;
      r.cu_occupancy(&occ, (CUfunction)kk.cu_fn[0], in.threads, in.smem);
      o->occupancy_original = occ;
    }
    return TALLY_OK;
  }
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kk.fn_ptb, in.threads, in.smem), "occupancy");
  o->occupancy_ptb = occ;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kk.fn_original, in.threads, in.smem), "occupancy");
  o->occupancy_original = occ;
  if (kk.tmem_cols > 0) {
    // resource-derived residency of a tcgen05 kernel: TMEM columns, shared
    // memory (+1 KB reserved per CTA), registers (256-register warp granules)
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kk.fn_ptb), "func attributes");
    int smem_sm = 0;
    CK(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, r.device), "smem per SM");
    const int warps = (in.threads + 31) / 32;
    const int regs_warp = (fa.numRegs * 32 + 255) / 256 * 256;
    int n = 512 / kk.tmem_cols;
    n = std::min(n, smem_sm / (int)(in.smem + 1024));
    n = std::min(n, 65536 / std::max(1, regs_warp * warps));
    n = std::min(n, 64 / warps);
    o->occupancy_ptb = std::max(o->occupancy_ptb, n);
    o->occupancy_original = std::max(o->occupancy_original, n);
  }
  return TALLY_OK;
}

int tally_kernel_destroy(int kernel) {
  Runtime& r = rt();
  if (kernel < 0 || kernel >= (int)r.instances.size() || !r.instances[kernel]) {
    set_error("unknown kernel instance %d", kernel);
    return TALLY_EINVAL;
  }
  r.instances[kernel].reset();
  return TALLY_OK;
}

int tally_stream_create(int prio, int* out) {
  Runtime& r = rt();
  if (!r.inited) { set_error("tally_init first"); return TALLY_EINVAL; }
  if (prio != TALLY_HIGH && prio != TALLY_BEST_EFFORT) { set_error("unknown priority class %d", prio); return TALLY_EINVAL; }
  cudaStream_t s;
  // Blocking streams: ordered after work on the legacy default stream (where
  // PyTorch initialises the buffers we are handed), concurrent with each other.
  CK(cudaStreamCreateWithPriority(&s, cudaStreamDefault, prio == TALLY_HIGH ? r.prio_high : r.prio_low),
     "cudaStreamCreateWithPriority");
  *out = (int)r.streams.size();
  r.streams.push_back(s);
  r.stream_be.push_back(prio == TALLY_BEST_EFFORT ? 1 : 0);
  return TALLY_OK;
}

int tally_stream_sync(int stream) {
  Runtime& r = rt();
  if (stream < 0 || stream >= (int)r.streams.size() || !r.streams[stream]) { set_error("unknown stream %d", stream); return TALLY_EINVAL; }
  CK(cudaStreamSynchronize(r.streams[stream]), "cudaStreamSynchronize");
  return TALLY_OK;
}

int tally_stream_handle(int stream, void** out) {
  Runtime& r = rt();
  if (stream < 0 || stream >= (int)r.streams.size() || !r.streams[stream] || !out) { set_error("unknown stream %d", stream); return TALLY_EINVAL; }
  *out = (void*)r.streams[stream];
  return TALLY_OK;
}

int tally_stream_destroy(int stream) {
  Runtime& r = rt();
  if (stream < 0 || stream >= (int)r.streams.size() || !r.streams[stream]) { set_error("unknown stream %d", stream); return TALLY_EINVAL; }
  cudaStreamDestroy(r.streams[stream]);
  r.streams[stream] = nullptr;
  return TALLY_OK;
}

int tally_launch(int kernel, int stream, const tally_launch_desc* d, int* out) {
  return rt().launch(kernel, stream, d, out);
}

int tally_launch_query(int id, tally_launch_state* o) {
  Runtime& r = rt();
  std::lock_guard<std::mutex> g(r.mu);
  Launch* L = r.get_launch(id);
  if (!L) return TALLY_EINVAL;
  r.poll(L);
  if (L->error != cudaSuccess) return cuda_fail(L->error, "launch");
  if (o) r.fill_state(L, o);
  return TALLY_OK;
}

int tally_launch_wait(int id, tally_launch_state* o) {
  Runtime& r = rt();
  Launch* L;
  {
    std::lock_guard<std::mutex> g(r.mu);
    L = r.get_launch(id);
    if (!L) return TALLY_EINVAL;
  }
  CK(cudaEventSynchronize(L->ev_end), "launch");
  std::lock_guard<std::mutex> g(r.mu);
  if (!r.poll(L)) {
    set_error("launch %d: kernel exited without publishing its outcome", id);
    return TALLY_ECUDA;
  }
  if (o) r.fill_state(L, o);
  return TALLY_OK;
}

int tally_launch_elapsed_ns(int id, long long* out) {
  Runtime& r = rt();
  std::lock_guard<std::mutex> g(r.mu);
  Launch* L = r.get_launch(id);
  if (!L) return TALLY_EINVAL;
  if (!L->timed) { set_error("launch %d was not timed", id); return TALLY_EINVAL; }
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, L->ev_start, L->ev_end), "cudaEventElapsedTime");
  *out = (long long)(ms * 1e6);
  return TALLY_OK;
}

int tally_preempt(int id) { return rt().preempt(id); }
int tally_set_pause(int on) { return rt().set_pause(on); }

int tally_jit_register(const char* name, const void* image, const char* sym_original, const char* sym_sliced,
                       const char* sym_ptb, unsigned gx, unsigned gy, unsigned gz, int threads, long long smem,
                       int* out_kind) {
  if (!name || !image || !sym_original || !sym_sliced || !sym_ptb || !out_kind) {
    set_error("null argument");
    return TALLY_EINVAL;
  }
  const char* syms[3] = {sym_original, sym_sliced, sym_ptb};
  const unsigned grid[3] = {gx, gy, gz};
  return rt().jit_register(name, image, syms, grid, threads, smem, out_kind);
}
int tally_launch_release(int id) { return rt().release(id); }

}  // extern "C"
