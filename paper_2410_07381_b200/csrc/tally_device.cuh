// Device-side launch shapes for Tally's block-level scheduler on sm_100a.
//
// Every best-effort kernel is written once as a *body* -- a struct with
//   static constexpr int kThreads;                 // CTA size (1-D)
//   struct Params;                                 // POD launch arguments
//   static __device__ void run(const Params&, uint3 bidx, uint3 grid, char* smem);
// and instantiated in three launch shapes:
//
//   k_original<Body>  grid = logical grid, blockIdx used as is   (untransformed)
//   k_sliced<Body>    grid = sub-grid, logical blockIdx = blockIdx + offset,
//                     gridDim pinned to the logical grid        (ref transforms.py:92-133)
//   k_ptb<Body>       grid = workers; each worker loops: leader checks the
//                     preemption flag, and only if clear claims the next task
//                     index with an L2 atomic, broadcasts it through shared
//                     memory, barrier, delinearize(task, logical grid), body,
//                     barrier                                    (ref transforms.py:291-401)
//
// Bodies must be "unified-synchronisation shaped" (ref transforms.py:200-288):
// no thread leaves run() early past a __syncthreads -- the PTB loop's barriers
// are then the only ones a finished logical block can meet.
#pragma once
#ifndef __CUDACC_RTC__   // also compiled by NVRTC for IR-JIT kernels (irjit.py)
#include <cstdint>
#include <cuda_runtime.h>
#endif

namespace tally {

// --- per-launch device record (pool in device memory, zeroed at init) ------
// A PTB launch owns one record for its lifetime; the last worker to exit
// publishes the outcome to the host mirror and re-zeroes the record so it can
// be reused without a host-side memset.
struct alignas(64) LaunchRec {
  unsigned long long claims;        // atomicAdd target: dynamic claims of this launch
  unsigned int exited;              // exit groups that have folded into this record
  unsigned int flag;                // device-resident preemption flag (holds a serial)
  unsigned long long neg_first_stop;   // ~min %globaltimer a worker saw the flag (0 = none)
  unsigned long long executed;      // logical blocks run by this launch
  unsigned long long stops;         // workers that stopped because of the flag
  unsigned long long neg_first_start;  // ~min worker entry %globaltimer (0 = none yet)
  unsigned long long last_busy_exit;   // max exit %globaltimer of workers that ran a block
  unsigned long long pops;             // return-ring pops started by this launch (<= ret_pending succeed)
};

// Worker retirement is two-level: workers fold into their group of 32
// (blockIdx.x / 32), the last of a group folds the group into the launch
// record -- ~32 + W/32 same-address atomics instead of W (one L2 atomic unit
// serialises same-address atomics: ~1 us per 1184 workers).
constexpr int kExitGroupSize = 32;
constexpr int kMaxExitGroups = 160;   // >= 148 x 32 resident workers / 32
struct alignas(16) ExitGroup {
  unsigned int exited;
  unsigned int pad;
  unsigned long long neg_first_start;
  unsigned long long executed;
  unsigned long long pad2;
};

// Host-visible outcome of a launch (pinned, mapped; written once by the last worker).
struct alignas(64) LaunchMirror {
  unsigned long long claims;
  unsigned long long t_first_stop;
  unsigned long long t_last_exit;
  unsigned long long stops;
  unsigned long long t_first_start;  // %globaltimer at first worker entry
  unsigned int serial;               // written last: == launch serial when valid
  unsigned int status;               // 1 = exhausted (done), 2 = parked
  unsigned long long ret_pending;    // return-ring entries handed back to the chain, not yet run
  // last exit of a worker that ran a block: a worker that only launched after
  // the flag (its SM slot was busy with high-priority CTAs until then) reads
  // the flag, hands its static block back and exits -- it held no resources
  // at the signal, so it is not part of the preemption latency
  unsigned long long t_last_busy_exit;
};

enum : unsigned { kMirrorDone = 1, kMirrorParked = 2 };

// Params of an IR-JIT body (irjit.py; the runtime's generic bind fills it)
struct JitParams {
  long long* mem;                 // flat int64 word image
  long long nwords;
  unsigned long long* fault;      // set non-zero on an out-of-range access / step limit
  long long args[8];              // IR kernel arguments (low registers)
};

// Shape arguments ------------------------------------------------------------
struct SliceArgs {
  uint3 offset;        // rectangular mode: logical block offset of this sub-launch
  uint3 grid;          // logical (original) grid -- gridDim as the body sees it
  unsigned long long linear_offset;  // linear mode: first task index of the slice
  unsigned int linear;               // 1: 1-D sub-grid over task indices
  unsigned long long* exec_count;  // optional exactly-once counters [total]
  unsigned long long* block_log;   // optional [total * 3]: start, end (%globaltimer), smid per logical block
};

struct PtbArgs {
  LaunchRec* rec;
  const unsigned int* flag;        // where the preemption flag lives (device or mapped host)
  LaunchMirror* mirror;            // mapped host outcome slot
  unsigned int serial;             // this launch's identity (the mirror is valid when it holds it)
  unsigned int flag_is_host;       // 1: flag is in mapped host memory (sys-scope loads)
  // Park when the flag has reached park_at (wrap-around compare; flags only
  // grow).  Per-launch flag: park_at = serial, the host writes the serial.
  // Chain flag (one word per best-effort stream, shared by every launch
  // queued on it): park_at = the stream's next preemption epoch, so one write
  // parks the running launch and everything queued behind it.
  unsigned int park_at;
  unsigned int* chain_dev;         // chain mode: the stream's device word (else null)
  unsigned int* chain_host;        // chain mode: its mapped host mirror (else null)
  unsigned long long start;        // persisted task counter to resume from
  unsigned long long total;        // total logical blocks
  long long preempt_at;            // test trigger: raise flag when counter reaches this (-1 off)
  uint3 grid;                      // logical grid
  unsigned long long* exec_count;  // optional exactly-once counters [total]
  unsigned long long* worker_log;  // optional [workers * 4] per-worker telemetry
  const unsigned int* pause;       // optional suspension word (device memory); non-zero = hold
  unsigned long long* block_log;   // optional [total * 3]: start, end, (worker << 32 | smid) per logical block
  // Bounded retirement (k_ptb): a worker that sees the flag after a block
  // hands its pre-claimed block back through the kernel instance's return
  // ring ([0] pushes, [1] pops, [2 + i % kRetCap] block + 1) instead of
  // running it; the next launch of the chain pops those first.
  unsigned long long* ret_ring;
  unsigned long long ret_pending;  // entries the previous launch of the chain left (0: skip the ring)
  // Static first blocks (k_ptb): worker b < static_n runs block start + b
  // without a claim (the flag still gates it; a worker that sees it hands
  // the block back); dynamic claims continue from start + static_n.
  unsigned long long static_n;
  ExitGroup* grp;                  // this launch's exit groups [kMaxExitGroups]
  // Batched claims (k_ptb): one atomic claims claim_n consecutive blocks (the
  // L2 serialises same-address atomics: ~2 ns each, so 1184 workers claiming
  // 1-2 us blocks one at a time were claim-throughput bound); the flag is
  // still checked between blocks and unrun blocks of a batch are handed back.
  int claim_n;
};

constexpr unsigned kRetCap = 8192;   // >= the most resident workers of any launch (148 x 32)

__device__ __forceinline__ bool ptb_park_requested(const PtbArgs& a, unsigned f) {
  return (int)(f - a.park_at) >= 0;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// Streaming 16 B load that does not allocate in L1: the HBM kernels read
// every byte once, and must not depend on how much L1 a co-resident CTA
// (e.g. a GEMM worker holding ~198 KB of shared memory) leaves them.
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

// Programmatic dependent launch (best-effort streams, runtime option): a
// kernel lets its successor's CTAs be scheduled as soon as all of its own
// CTAs are running, and waits for its predecessor's completion (memory
// visible) before touching global memory -- the successor's launch and
// prologue overlap the predecessor's tail.  No-ops without the attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint3 delinearize(unsigned long long t, uint3 g) {
  // ref ir/core.py:59-65: x fastest.  1-D grids (every built-in kind but the
  // channel-blocked statistics) need no division; 32-bit math when the index
  // fits (a 64-bit division is ~70 instructions -- as much as a small body)
  uint3 b;
  if (g.y == 1 && g.z == 1) return make_uint3((unsigned)t, 0u, 0u);
  if (t < (1ull << 32)) {
    const unsigned t32 = (unsigned)t, q = t32 / g.x;
    b.x = t32 - q * g.x;
    b.y = q % g.y;
    b.z = q / g.y;
    return b;
  }
  b.x = (unsigned)(t % g.x);
  unsigned long long q = t / g.x;
  b.y = (unsigned)(q % g.y);
  b.z = (unsigned)(q / g.y);
  return b;
}

__device__ __forceinline__ unsigned long long linear_index(uint3 b, uint3 g) {
  return (unsigned long long)b.x + (unsigned long long)g.x * (b.y + (unsigned long long)g.y * b.z);
}

// Optional per-body occupancy hint: a body may declare
//   static constexpr int kMinBlocks = n;   // resident CTAs per SM to compile for
// (register cap for HBM-streaming bodies); default 1.
template <class...>
using void_t_ = void;
template <class B, class = void>
struct MinBlocks {
  static constexpr int value = 1;
};
template <class B>
struct MinBlocks<B, void_t_<decltype(B::kMinBlocks)>> {
  static constexpr int value = B::kMinBlocks;
};

// Optional per-CTA hooks of a body: `static __device__ void cta_init(char*
// smem)` runs once when the CTA starts -- before it lets a programmatic
// dependent launch begin, so resources it takes there (TMEM) cannot be taken
// first by a successor kernel that then waits for it -- and `cta_exit(char*
// smem)` once after the CTA's last logical block.
template <class B, class = void>
struct HasCtaHooks {
  static constexpr bool value = false;
};
template <class B>
struct HasCtaHooks<B, void_t_<decltype(&B::cta_init)>> {
  static constexpr bool value = true;
};

__device__ __forceinline__ unsigned smid();

// Per-logical-block event log (ref sim.py:436-505 BlockStarted / BlockFinished
// on the device clock), written by thread 0 once the whole block is done.
__device__ __forceinline__ void log_block(unsigned long long* log, unsigned long long i, unsigned long long t0,
                                          unsigned long long who) {
  log[3 * i] = t0;
  log[3 * i + 1] = globaltimer();
  log[3 * i + 2] = who;
}

// --- Original: the untransformed kernel --------------------------------------
template <class Body>
__global__ void __launch_bounds__(Body::kThreads, MinBlocks<Body>::value)
k_original(const __grid_constant__ typename Body::Params p, const SliceArgs s) {
  extern __shared__ __align__(1024) char smem[];
  if constexpr (HasCtaHooks<Body>::value) Body::cta_init(smem);
  pdl_launch_dependents();
  pdl_wait();
  const uint3 g = make_uint3(gridDim.x, gridDim.y, gridDim.z);
  if (s.exec_count != nullptr && threadIdx.x == 0)
    atomicAdd(&s.exec_count[linear_index(blockIdx, g)], 1ull);
  const unsigned long long t0 = s.block_log != nullptr ? globaltimer() : 0ull;
  Body::run(p, blockIdx, g, smem);
  if (s.block_log != nullptr) {   // uniform across the block
    __syncthreads();
    if (threadIdx.x == 0) log_block(s.block_log, linear_index(blockIdx, g), t0, smid());
  }
  if constexpr (HasCtaHooks<Body>::value) Body::cta_exit(smem);
}

// --- Sliced: block offset + pinned gridDim ------------------------------------
template <class Body>
__global__ void __launch_bounds__(Body::kThreads, MinBlocks<Body>::value)
k_sliced(const __grid_constant__ typename Body::Params p, const SliceArgs s) {
  extern __shared__ __align__(1024) char smem[];
  if constexpr (HasCtaHooks<Body>::value) Body::cta_init(smem);
  pdl_launch_dependents();
  pdl_wait();
  const uint3 b = s.linear ? delinearize(s.linear_offset + blockIdx.x, s.grid)
                           : make_uint3(blockIdx.x + s.offset.x, blockIdx.y + s.offset.y,
                                        blockIdx.z + s.offset.z);
  if (s.exec_count != nullptr && threadIdx.x == 0)
    atomicAdd(&s.exec_count[linear_index(b, s.grid)], 1ull);
  const unsigned long long t0 = s.block_log != nullptr ? globaltimer() : 0ull;
  Body::run(p, b, s.grid, smem);
  if (s.block_log != nullptr) {
    __syncthreads();
    if (threadIdx.x == 0) log_block(s.block_log, linear_index(b, s.grid), t0, smid());
  }
  if constexpr (HasCtaHooks<Body>::value) Body::cta_exit(smem);
}

// --- PTB: persistent, preemptible workers -------------------------------------
// Worker exit bookkeeping, run by thread 0 of every worker.
// Resume ring of a chunk-preemptible kernel (one per kernel instance, device
// memory): [0] = pushes (tail), [1] = pops (head), [2 + i % kResumeCap] =
// entries (tile + 1) | (next_chunk << 40); 0 = empty.  A worker preempted
// mid-tile saves its partial state and pushes (tile, chunk); the next launch
// of the chain pops before claiming fresh tiles.  Outstanding entries <=
// resident workers, so the ring never overflows.
constexpr unsigned kResumeCap = 1024;

__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Entries pending in a resume / return ring.  Called after an acquire that
// orders every push and pop of the launch before it, so plain (relaxed)
// loads suffice -- no read-modify-write round trips.
__device__ __forceinline__ unsigned long long resume_pending(const unsigned long long* ring) {
  if (ring == nullptr) return 0ull;
  const unsigned long long tail = ld_relaxed_gpu_u64(ring);
  const unsigned long long head = ld_relaxed_gpu_u64(ring + 1);
  return tail > head ? tail - head : 0ull;
}

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Worker retirement (thread 0 of every worker).  Minima are kept as maxima of
// the complement (records are zero between launches) and every per-worker
// update is a fire-and-forget reduction; the only round trips are the
// group's and the record's acq_rel exit counters.  The last group's last
// worker is by construction the latest exit: it stamps t_last_exit, decides
// done / parked and publishes the host mirror, `serial` last with a
// system-scope release store, then recycles the record.
// `executed`: logical blocks this worker ran; `static_returned`: static
// first blocks it handed back on the flag.
__device__ __forceinline__ void ptb_worker_exit(const PtbArgs& a, bool stopped,
                                                unsigned long long t_entry,
                                                const unsigned long long* resume_ring = nullptr,
                                                unsigned long long executed = 0) {
  LaunchRec* r = a.rec;
  const unsigned nworkers = gridDim.x * gridDim.y * gridDim.z;
  const unsigned g = blockIdx.x / kExitGroupSize;
  const unsigned ngroups = (nworkers + kExitGroupSize - 1) / kExitGroupSize;
  const unsigned gsize = min((unsigned)kExitGroupSize, nworkers - g * kExitGroupSize);
  // fire-and-forget reductions straight into the record: the acq_rel exit
  // counters below order them before the last worker's reads
  atomicMax(&r->neg_first_start, ~t_entry);
  if (executed) {
    atomicAdd(&r->executed, executed);
    atomicMax(&r->last_busy_exit, globaltimer());
  }
  if (stopped) {
    atomicAdd(&r->stops, 1ull);
    atomicMax(&r->neg_first_stop, ~globaltimer());
  }
  ExitGroup* eg = a.grp + g;
  if (atom_add_acq_rel_gpu(&eg->exited, 1u) + 1u != gsize) return;
  eg->exited = 0u;   // last of its group: recycle the group slot
  if (atom_add_acq_rel_gpu(&r->exited, 1u) + 1u != ngroups) return;
  // last worker: one batch of independent loads, publish, recycle the record
  const unsigned long long now = globaltimer();
  const unsigned long long dyn = ld_relaxed_gpu_u64(&r->claims);
  const unsigned long long nfs = ld_relaxed_gpu_u64(&r->neg_first_stop);
  const unsigned long long nst = ld_relaxed_gpu_u64(&r->neg_first_start);
  const unsigned long long stops = ld_relaxed_gpu_u64(&r->stops);
  const unsigned long long ran = ld_relaxed_gpu_u64(&r->executed);
  const unsigned long long busy = ld_relaxed_gpu_u64(&r->last_busy_exit);
  const unsigned long long tail = resume_ring ? ld_relaxed_gpu_u64(resume_ring) : 0ull;
  const unsigned long long head = resume_ring ? ld_relaxed_gpu_u64(resume_ring + 1) : 0ull;
  unsigned long long claims = a.static_n + dyn;
  unsigned long long pending = tail > head ? tail - head : 0ull;
  if (a.static_n && ran == 0ull && dyn == 0ull && a.ret_ring != nullptr) {
    // preempted before any block ran (e.g. queued behind a parked launch):
    // every static block was handed back -- take them back out of the ring
    // and report the launch untouched (counter == start, like a flag seen
    // before the first claim)
    atomicAdd(a.ret_ring, (unsigned long long)(0ull - a.static_n));
    pending -= a.static_n;
    claims = 0ull;
  }
  const unsigned long long progress = a.start + claims;
#ifdef TALLY_EXPERIMENT_NO_MIRROR   // timing experiment only (tools/ptb_publish_cost.py): no host writes
  r->claims = 0ull; r->exited = 0u; r->neg_first_stop = 0ull; r->executed = 0ull; r->stops = 0ull;
  r->neg_first_start = 0ull;
  if (progress == ~0ull) r->pops = nfs + nst + stops + now + pending;
  return;
#endif
  volatile LaunchMirror* m = a.mirror;
  m->claims = claims;
  m->t_first_stop = nfs ? ~nfs : 0ull;
  m->t_last_exit = now;
  m->stops = stops;
  m->t_first_start = nst ? ~nst : 0ull;
  m->ret_pending = pending;
  m->t_last_busy_exit = busy;
  // work can only remain if some worker stopped on the flag
  const bool parked = progress < a.total || pending > 0;
  m->status = parked ? kMirrorParked : kMirrorDone;
  if (parked && a.chain_dev != nullptr) {
    // a parked chain launch parks everything queued behind it on the stream:
    // the next launch starts after this one exits (stream order) and reads
    // the raised word, whichever of the host's two writes it would poll
    atomicMax(a.chain_dev, a.park_at);
    if (a.chain_host != nullptr) st_release_sys(a.chain_host, a.park_at);
  }
  r->claims = 0ull;
  r->exited = 0u;
  r->neg_first_stop = 0ull;
  r->executed = 0ull;
  r->stops = 0ull;
  r->neg_first_start = 0ull;
  r->last_busy_exit = 0ull;
  r->pops = 0ull;
  st_release_sys(const_cast<unsigned*>(&m->serial), a.serial);
}

// One claim by the leader thread: check the flag first, then fetch-and-add
// the task counter (ref transforms.py:343-351).  Returns -1 on preemption.
// Cooperative suspension (B200 extension): while the pause
// word is set the worker holds its place -- no claims, no memory traffic --
// and resumes in place when it clears; a park request (flag == serial) ends
// the wait.  Returns true if a park was requested while waiting.
__device__ __forceinline__ bool ptb_hold_while_paused(const PtbArgs& a) {
  if (a.pause == nullptr || ld_acquire_gpu(a.pause) == 0u) return false;
  for (;;) {
    __nanosleep(256);
    const unsigned f = a.flag_is_host ? ld_acquire_sys(a.flag) : ld_acquire_gpu(a.flag);
    if (ptb_park_requested(a, f)) return true;
    if (ld_acquire_gpu(a.pause) == 0u) return false;
  }
}

template <bool kCountExec = true>
__device__ __forceinline__ long long ptb_claim(const PtbArgs& a) {
  ptb_hold_while_paused(a);
  const unsigned f = a.flag_is_host ? ld_acquire_sys(a.flag) : ld_acquire_gpu(a.flag);
  if (ptb_park_requested(a, f)) return -1;   // flag gates the claim: a parked launch never over-claims
  const unsigned long long c = atomicAdd(&a.rec->claims, 1ull);
  const long long task = (long long)(a.start + a.static_n + c);
  if (a.preempt_at >= 0 && task + 1 == a.preempt_at)
    st_release_sys(const_cast<unsigned*>(a.flag), a.park_at);   // test trigger (MemTrigger)
  if (kCountExec && a.exec_count != nullptr && (unsigned long long)task < a.total)
    atomicAdd(&a.exec_count[task], 1ull);
  return task;
}

// The claim-ahead inside the k_ptb loop: the flag was read at the end of the
// previous block (or at entry), so the claim is issued without another load
// (one exposed L2 round trip per block instead of two); a claim that races a
// flag raised in between is handed back after the block.
__device__ __forceinline__ long long ptb_claim_gated(const PtbArgs& a) {
  ptb_hold_while_paused(a);
  const unsigned long long c = atomicAdd(&a.rec->claims, 1ull);
  const long long task = (long long)(a.start + a.static_n + c);
  if (a.preempt_at >= 0 && task + 1 == a.preempt_at)
    st_release_sys(const_cast<unsigned*>(a.flag), a.park_at);   // test trigger (MemTrigger)
  return task;
}

// Return-ring entries are ranges of consecutive blocks: (first + 1) | (count << 48)
// -- a worker hands back at most two (the rest of its batch, the pre-claimed
// next batch), so the ring holds <= 2 entries per worker and one pop takes a
// whole range.
// A range an earlier launch of the chain handed back; -1 when none is left.
// The entries a launch may pop are exactly the ret_pending ones its chain's
// previous launch left (they are all written: that launch has exited); pushes
// by this launch's own workers land behind them.  A per-launch ticket bounds
// the pops, so each is two fetch-adds and no retries -- a CAS loop on the ring
// head let a resumed launch's ~1200 workers contend for hundreds of
// microseconds (C2 / C3 preemption drains up to ~300 us).
__device__ __forceinline__ long long ptb_pop_range(const PtbArgs& a, int& count) {
  unsigned long long* ring = a.ret_ring;
  if (atomicAdd(&a.rec->pops, 1ull) >= a.ret_pending) return -1;
  const unsigned long long h = atomicAdd(ring + 1, 1ull);
  volatile unsigned long long* e = ring + 2 + (h % kRetCap);
  unsigned long long v;
  while ((v = *e) == 0ull) __nanosleep(32);
  *e = 0ull;
  count = (int)(v >> 48);
  return (long long)(v & 0xFFFFFFFFFFFFull) - 1;
}
__device__ __forceinline__ void ptb_return_range(const PtbArgs& a, long long first, long long count) {
  if (count <= 0) return;
  const unsigned long long i = atomicAdd(a.ret_ring, 1ull);
  reinterpret_cast<volatile unsigned long long*>(a.ret_ring)[2 + (i % kRetCap)] =
      ((unsigned long long)first + 1ull) | ((unsigned long long)count << 48);
}
__device__ __forceinline__ void ptb_return(const PtbArgs& a, long long task) { ptb_return_range(a, task, 1); }

// Claim-ahead of a batch of n blocks (flag read separately, see k_ptb).
__device__ __forceinline__ long long ptb_claim_batch_gated(const PtbArgs& a, int n) {
  if (n <= 1) return ptb_claim_gated(a);
  ptb_hold_while_paused(a);
  const unsigned long long c = atomicAdd(&a.rec->claims, (unsigned long long)n);
  return (long long)(a.start + a.static_n + c);
}

// The next batch of a k_ptb worker: one handed-back block while the host
// says some are pending (count 1), else a fresh claim of n blocks.
__device__ __forceinline__ long long ptb_take(const PtbArgs& a, bool& try_pop, int n, int& count) {
  if (try_pop) {
    const long long t = ptb_pop_range(a, count);
    if (t >= 0) return t;
    try_pop = false;
  }
  count = n;
  return ptb_claim_batch_gated(a, n);
}

// Batched claim: n consecutive task indices with one flag-gated atomic.
// Returns the first (tasks >= total are skipped by the caller) or -1.
__device__ __forceinline__ long long ptb_claim_n(const PtbArgs& a, int n) {
  if (n <= 1) return ptb_claim(a);
  ptb_hold_while_paused(a);
  const unsigned f = a.flag_is_host ? ld_acquire_sys(a.flag) : ld_acquire_gpu(a.flag);
  if (ptb_park_requested(a, f)) return -1;
  const unsigned long long c = atomicAdd(&a.rec->claims, (unsigned long long)n);
  const long long task = (long long)(a.start + a.static_n + c);
  if (a.preempt_at >= 0 && task < a.preempt_at && a.preempt_at <= task + n)
    st_release_sys(const_cast<unsigned*>(a.flag), a.park_at);   // test trigger (MemTrigger)
  if (a.exec_count != nullptr)
    for (int k = 0; k < n; ++k)
      if ((unsigned long long)(task + k) < a.total) atomicAdd(&a.exec_count[task + k], 1ull);
  return task;
}

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// Persistent worker loop.  The leader claims the next batch while the CTA
// executes the last block of the current one (claim-ahead), so the L2 atomic
// overlaps the body instead of serialising with it.  Retirement stays bounded
// by one logical block: after every block the leader re-reads the flag, and
// if it rose meanwhile every claimed-but-unrun block (the rest of the batch,
// the pre-claimed next batch) is handed back through the return ring.
template <class Body>
__global__ void __launch_bounds__(Body::kThreads, MinBlocks<Body>::value)
k_ptb(const __grid_constant__ typename Body::Params p, const PtbArgs a) {
  extern __shared__ __align__(1024) char smem[];
  if constexpr (HasCtaHooks<Body>::value) Body::cta_init(smem);
  pdl_launch_dependents();
  pdl_wait();
  __shared__ long long s_task[2];
  const bool leader = (threadIdx.x == 0);
  const unsigned long long t_entry = leader ? globaltimer() : 0ull;
  bool stopped = false;
  bool try_pop = a.ret_ring != nullptr && a.ret_pending > 0;
  const int n = a.claim_n > 1 ? a.claim_n : 1;
  // the static blocks cover the rest of the kernel: no claim (it could only
  // fail) and no end-of-block flag read (nothing is pre-claimed)
  const bool covered = a.static_n > 0 && a.start + a.static_n >= a.total;
  unsigned long long done = 0;
  long long cur = 0, end = 0;   // leader: unrun blocks [cur, end) of the current batch
  long long pre = -1;           // leader: first block of the pre-claimed next batch (-1: not claimed yet)
  int pre_cnt = 0;
  if (leader) {
    if (blockIdx.x < a.static_n) {
      // static first block: no claim round trip, the flag still gates it
      const unsigned f = a.flag_is_host ? ld_acquire_sys(a.flag) : ld_acquire_gpu(a.flag);
      const long long mine = (long long)(a.start + blockIdx.x);
      s_task[0] = ptb_park_requested(a, f) ? -mine - 2 : mine;
    } else if (covered) {
      s_task[0] = (long long)a.total;   // surplus worker: nothing left
    } else {
      ptb_hold_while_paused(a);
      const unsigned f = a.flag_is_host ? ld_acquire_sys(a.flag) : ld_acquire_gpu(a.flag);
      if (ptb_park_requested(a, f)) {
        s_task[0] = -1;   // flag before the first claim: nothing claimed
      } else {
        int cnt = 1;
        const long long b = ptb_take(a, try_pop, n, cnt);
        if (a.preempt_at >= 0 && b < a.preempt_at && a.preempt_at <= b + cnt)
          st_release_sys(const_cast<unsigned*>(a.flag), a.park_at);   // test trigger (MemTrigger)
        s_task[0] = b;
        cur = b + 1;
        end = b + cnt;
      }
    }
  }
  __syncthreads();
  for (unsigned it = 0;; ++it) {
    const long long task = s_task[it & 1];
    if (task < -1) {   // the flag rose before this (static) block started: hand it back
      if (leader) ptb_return(a, -task - 2);
      stopped = true;
      break;
    }
    if (task < 0 || (unsigned long long)task >= a.total) {
      stopped = task < 0;
      break;
    }
    if (leader) {
      // the last block of this batch: claim the next batch while it runs
      // (the flag was clear when this block began)
      if (!covered && cur >= end && pre < 0) {
        pre = ptb_take(a, try_pop, n, pre_cnt);
        if (a.preempt_at >= 0 && pre < a.preempt_at && a.preempt_at <= pre + pre_cnt)
          st_release_sys(const_cast<unsigned*>(a.flag), a.park_at);   // test trigger (MemTrigger)
      }
      if (a.exec_count != nullptr) atomicAdd(&a.exec_count[task], 1ull);
    }
    const unsigned long long t0 = (leader && a.block_log != nullptr) ? globaltimer() : 0ull;
    Body::run(p, delinearize((unsigned long long)task, a.grid), a.grid, smem);
    ++done;
    if (leader) {
      long long nx;
      if (covered) {
        nx = (long long)a.total;
      } else if (cur < end) {
        nx = cur++;
      } else {
        nx = pre;
        cur = pre + 1;
        end = pre + pre_cnt;
        pre = -1;
      }
      if (nx >= 0 && (unsigned long long)nx < a.total) {
        // bounded retirement: a flag raised while this block ran hands every
        // claimed-but-unrun block back instead of running it
        const unsigned f = a.flag_is_host ? ld_relaxed_sys(a.flag) : ld_relaxed_gpu(a.flag);
        if (ptb_park_requested(a, f)) {
          ptb_return_range(a, nx, min(end, (long long)a.total) - nx);
          nx = -1;
        }
      }
      s_task[(it + 1) & 1] = nx;
    }
    __syncthreads();
    if (leader && a.block_log != nullptr)
      log_block(a.block_log, (unsigned long long)task, t0, ((unsigned long long)blockIdx.x << 32) | smid());
  }
  if constexpr (HasCtaHooks<Body>::value) Body::cta_exit(smem);
  if (leader) {
    if (a.worker_log != nullptr) {
      unsigned long long* w = a.worker_log + 4ull * blockIdx.x;
      w[0] = ((unsigned long long)smid() << 32) | (done & 0xffffffffull);
      w[1] = t_entry;
      w[2] = globaltimer();
      w[3] = stopped ? 1ull : 0ull;
    }
    ptb_worker_exit(a, stopped, t_entry, a.ret_ring, done);
  }
}

}  // namespace tally
