/* tally_b200.h -- C ABI of the B200-native Tally block-level kernel scheduler.
 *
 * The reference (tallysim, /root/reference/pkg/src/tallysim) has no FFI: its
 * device boundary is the Python `GpuSim` + `KernelHandle` surface that
 * `PolicyRunner` and `Profiler` consume.  This header is that
 * surface expressed as a C ABI, plus the kernel-variant launch layer that the
 * reference only models.  Each entry point cites the reference interface it
 * replaces.
 *
 * Conventions: every function returns TALLY_OK (0) or a negative code; the
 * message of the last failure on the calling thread is tally_last_error().
 * Python maps TALLY_EINVAL -> ValueError and TALLY_ETRANSFORM -> TransformError
 * (ref transforms.py:27-28, sim.py:260-262/306-312/331-334).  Device memory is
 * owned by the caller (e.g. PyTorch); the library only borrows pointers for the
 * duration of a launch.  All calls are single-threaded except tally_preempt,
 * which may be called from any host thread.
 */
#ifndef TALLY_B200_H
#define TALLY_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define TALLY_ABI_VERSION 2

#define TALLY_OK 0
#define TALLY_EINVAL (-22)     /* bad argument / state            -> ValueError     */
#define TALLY_ETRANSFORM (-95) /* transformation refused          -> TransformError */
#define TALLY_ENODEV (-19)     /* no usable sm_100 device / driver                  */
#define TALLY_ECUDA (-5)       /* CUDA runtime / driver failure                     */
#define TALLY_ENOMEM (-12)
#define TALLY_EBUSY (-16)      /* resource still in flight                          */

/* ---- priorities, shapes, variants, event kinds (ref sim.py:37-45, profiler.py:38-40) */
#define TALLY_HIGH 0
#define TALLY_BEST_EFFORT 1

#define TALLY_SHAPE_ORIGINAL 0
#define TALLY_SHAPE_SLICED 1
#define TALLY_SHAPE_PTB 2

#define TALLY_EV_LAUNCH_ISSUED 0
#define TALLY_EV_BLOCK_STARTED 1
#define TALLY_EV_BLOCK_FINISHED 2
#define TALLY_EV_KERNEL_FINISHED 3
#define TALLY_EV_PREEMPT_SIGNALED 4
#define TALLY_EV_WORKER_PARKED 5
/* B200 device log only (not a reference event kind): a runner timer fired --
 * block = the time it was scheduled for, time_ns = when the daemon ran it.
 * Arrivals fire at the first loop pass at or after their trace time; the
 * replay parity test needs the order in which they met completions. */
#define TALLY_EV_TIMER_FIRED 6

#define TALLY_POLICY_TALLY 0
#define TALLY_POLICY_EAGER 1
#define TALLY_POLICY_KERNEL_PRIORITY 2
#define TALLY_POLICY_TIME_SLICED 3

typedef struct {
  int device;
  int num_sms;              /* GpuSpec.num_sms            (ref sim.py:55-74) */
  int max_threads_per_sm;   /* GpuSpec.max_threads_per_sm                    */
  int max_blocks_per_sm;    /* GpuSpec.max_blocks_per_sm                     */
  int cc_major, cc_minor;
  long long smem_per_sm;
  long long hbm_bytes;
  int stream_mem_ops;       /* 1 if cuStreamWriteValue32 is usable (device-resident flags) */
  int stream_mem_ops_probe; /* diagnostic: entry-point status * 1000 + CUresult of the probe write */
  char name[96];
} tally_gpu_info;

/* ==== runtime ============================================================== */
/* Replaces constructing `GpuSim(gpu, ...)` (ref sim.py:229-250): binds the
 * library to one CUDA device, creates the launch-record pools. */
int tally_init(int device, tally_gpu_info* out);
int tally_shutdown(void);
const char* tally_last_error(void);
int tally_abi_version(void);
long long tally_now_ns(void);          /* host CLOCK_MONOTONIC, ns */
/* Calibrate host clock vs device %globaltimer; offset = host_ns - gt_ns. */
int tally_clock_offset(long long* out_offset_ns, long long* out_uncertainty_ns);
/* 0 = device-resident flags written with cuStreamWriteValue32 (default when
 * available), 1 = flags in mapped pinned host memory. */
int tally_set_flag_mode(int host_mapped);
/* Diagnostic: median / max ns from a host-side flag write to a spinning device
 * reader observing it (mode 0 = device flag via cuStreamWriteValue32,
 * 1 = mapped host flag). */
int tally_probe_flag_latency(int mode, int iters, long long* out_median_ns, long long* out_max_ns);
/* Co-location cache policy (B200 extension; no reference counterpart): make
 * [base, base + bytes) L2-persisting for kernels launched on (or captured
 * from) the CUDA stream `cuda_stream` -- a high-priority request's weights
 * stay L2-resident while best-effort kernels stream gigabytes through L2.
 * Sets the device's persisting-L2 limit to min(bytes, device maximum).
 * out_window_bytes: the window actually applied (clamped to the device max). */
int tally_l2_persist(void* cuda_stream, const void* base, long long bytes, float hit_ratio,
                     long long* out_window_bytes);
/* The same window applied to every kernel node of a captured (not yet
 * instantiated, or to be re-instantiated) cudaGraph_t.  out_nodes: kernel
 * nodes updated. */
int tally_graph_l2_persist(void* cuda_graph, const void* base, long long bytes, float hit_ratio,
                           int* out_nodes);
/* Enqueue an L2 warm-up of [base, base + bytes) on `cuda_stream` (capturable
 * into a CUDA graph): bulk L2 prefetches with the evict-last policy, a few
 * microseconds for tens of MB.  A request graph forks it next to its first
 * kernels so weights evicted by best-effort traffic come back ahead of the
 * layers that read them. */
int tally_l2_prefetch(void* cuda_stream, const void* base, long long bytes);

/* ==== kernel registration (ref scheduler.py:73-86 KernelWork; ir/core.py:153-214) */
typedef struct {
  void* ptr[8];             /* device pointers, kernel-specific meaning */
  long long i[8];           /* integer arguments                                     */
  double f[4];
} tally_kernel_args;

/* Optional layout of a bf16 GEMM kind (tally_kernel_args.ptr[3], host memory,
 * read at tally_kernel_create): batched launches over sub-matrices of larger
 * row-major tensors (attention: per (sequence, head) blocks of a fused QKV
 * activation).  Logical block = (batch z, output tile, K split); batch z has
 * zb = z / hdiv, zh = z % hdiv and every operand's (row, col) origin is
 * off[0] * zb + off[1] * zh, in the tensor's own row / column coordinates. */
typedef struct {
  long long a_rows, a_cols, a_ld; /* A extent (row-major, cols contiguous), row pitch */
  long long b_rows, b_cols, b_ld; /* B extent and row pitch (elements)               */
  long long ldc;                  /* C row stride (elements)                      */
  int batches, hdiv;
  long long a_row_off[2], a_col_off[2];
  long long b_row_off[2], b_col_off[2];
  long long c_row_off[2], c_col_off[2];
} tally_gemm_layout;

/* Convolution geometry of the implicit-GEMM kinds (tally_kernel_args.ptr[3],
 * host memory, read at tally_kernel_create): NHWC bf16 input [n, h, w, c],
 * square k x k filter, stride, padding; c % 64 == 0.  "conv_fprop_*": A =
 * im2col(x) by TMA im2col loads (no column matrix), B = weights [cout, k*k*c]
 * in (kh, kw, c) order; "conv_wgrad_*": dW[cout, k*k*c] = dy^T . im2col(x),
 * A = dy [P, cout] (MN-major), B = im2col(x) by TMA im2col loads. */
typedef struct {
  int n, h, w, c;
  int k, stride, pad;
} tally_conv_geometry;

/* Batch-norm statistics fused into the producer of a bf16 [P, C] tensor
 * (tally_kernel_args.ptr[7] of the bf16 GEMM / conv_fprop kinds and of
 * "splitk_reduce_bn"; host memory, read at tally_kernel_create).  The
 * producer also writes what the "bn_stats" kind (mode 0) computes from its
 * output: mean, invstd and scale_shift = [gamma * invstd; beta - mean *
 * gamma * invstd] (ref: the batch-norm statistics pass of the ResNet-50 BE
 * job).  GEMM / conv_fprop: part receives 2 x R partial
 * rows of C floats (R = ceil(P / 128), x 4 for rb = 32) that the "bn_fold"
 * kind folds; splitk_reduce_bn / bn_fold: part is their fold scratch of
 * 2 * ceil(rows / rb) * C floats. */
typedef struct {
  float* part;
  const float* gamma;
  const float* beta;
  float* mean;
  float* invstd;
  float* scale_shift;
  double eps;
  long long rb;   /* splitk_reduce_bn / bn_fold: rows per logical block; GEMM /
                     conv_fprop: 32 = a partial row per 32 output rows (per
                     epilogue warp, 4 * ceil(P / 128) rows), else per 128 */
} tally_bn_stats;

typedef struct {
  unsigned grid_x, grid_y, grid_z;  /* logical grid (the untransformed launch)  */
  long long total_blocks;
  int threads_per_block;
  long long smem_bytes;
  int occupancy_ptb;        /* resident PTB workers per SM (real occupancy)      */
  int occupancy_original;
  double alg_bytes;         /* algorithmic HBM bytes of one full launch          */
  double alg_flops;         /* algorithmic flops of one full launch              */
  int preempt_units;        /* PTB preemption points per logical block (>1: chunk-granular
                               preemption with saved partial state, e.g. sgemm_tf32x3) */
  int cluster;              /* CTAs per logical block (CTA-pair GEMMs "*_x2": 2, launched as
                               clusters; PTB worker counts must be a multiple); else 1 */
} tally_kernel_info;

int tally_kernel_kind_count(void);
const char* tally_kernel_kind_name(int kind);
/* Bind a built-in kernel kind ("vecadd_i64", "vecadd_f32", "rowsum_f32",
 * "sgemm_tf32x3", "gemm_bf16") to arguments; returns an instance id. */
int tally_kernel_create(const char* kind, const tally_kernel_args* args, int* out_kernel);
int tally_kernel_info_get(int kernel, tally_kernel_info* out);
int tally_kernel_destroy(int kernel);
/* IR-JIT: register a kernel kind from an NVRTC-compiled cubin holding the
 * three shape instantiations of one IR kernel body (irjit.py generates them
 * from a reference KernelDef; ref ir/core.py:153-214, transforms.py).
 * Arguments of tally_kernel_create for such a kind: ptr[0] = int64 word
 * image, ptr[1] = fault word, i[0] = words, i[1..7] = IR kernel arguments. */
int tally_jit_register(const char* name, const void* cubin, const char* sym_original,
                       const char* sym_sliced, const char* sym_ptb, unsigned grid_x,
                       unsigned grid_y, unsigned grid_z, int threads, long long smem_bytes,
                       int* out_kind);

/* ==== streams (per-priority CUDA streams) ================================== */
int tally_stream_create(int priority_class, int* out_stream);   /* TALLY_HIGH / TALLY_BEST_EFFORT */
int tally_stream_sync(int stream);
int tally_stream_handle(int stream, void** out_cuda_stream);   /* the cudaStream_t, borrowed */
int tally_stream_destroy(int stream);

/* ==== launches (ref sim.py:114-153 shapes, :304-351 submit/preempt;
 *       transforms.py:155-197 sliced, :404-448 ptb) ========================== */
typedef struct {
  int shape;                /* TALLY_SHAPE_*                                          */
  /* SLICED: a contiguous range of logical blocks.  linear != 0: task indices
   * [linear_offset, linear_offset + count) of the x-fastest linearisation (the
   * scheduler's 1-D tiling, ref scheduler.py:377-390); linear == 0: rectangular
   * sub-grid `sub_*` at block offset `off_*` (ref transforms.py:155-168). */
  int linear;
  long long linear_offset, count;
  unsigned off_x, off_y, off_z, sub_x, sub_y, sub_z;
  /* PTB */
  int workers;              /* resident worker CTAs                                   */
  long long start_count;    /* persisted task counter to resume from (PtbShape.start_count) */
  long long preempt_at;     /* test trigger: raise the flag when the counter reaches this
                               value (ref transforms.py:433-447 MemTrigger); -1 = off */
  unsigned long long* exec_count; /* optional device array[total_blocks]: exactly-once audit */
  int pausable;             /* PTB: honour the global suspension word (tally_set_pause) */
  unsigned long long* worker_log; /* PTB, optional device array[workers * 4]: per-worker
                                     {smid << 32 | tasks, t_entry, t_exit, stopped} (%globaltimer) */
  int timed;                /* 1: bracket with timing events (tally_launch_elapsed_ns) */
  int chain;                /* PTB: park on the stream's shared chain word instead of a
                               per-launch flag -- tally_preempt then parks this launch and
                               every PTB launch queued behind it on the stream (B200
                               real-time look-ahead; a parked launch raises the word for
                               its successors before it exits) */
  unsigned long long* block_log; /* optional device array[total_blocks * 3]: per logical block
                               {start, end} on the device %globaltimer and {worker << 32 | smid}
                               (BlockStarted / BlockFinished, ref sim.py:436-505; the
                               hand-written streaming kinds and IR-JIT kinds -- not the GEMMs) */
} tally_launch_desc;

typedef struct {
  int done;                 /* all claimed work finished and the launch exited         */
  int parked;               /* PTB only: exited on the flag with work remaining        */
  int preempted;            /* tally_preempt was called                                */
  long long task_counter;   /* PTB: persisted counter (start + claims; may exceed total
                               by <= workers on exhaustion, ref test_transforms.py:151) */
  long long claims;
  long long gt_first_start, gt_first_stop, gt_last_exit;   /* device %globaltimer ns */
  long long host_submit_ns, host_preempt_ns;
  long long gt_last_busy_exit;  /* PTB: last exit of a worker that ran a block (0 = none / not
                                   tracked); workers launched only after the flag do not count */
} tally_launch_state;

int tally_launch(int kernel, int stream, const tally_launch_desc* desc, int* out_launch);
int tally_launch_query(int launch, tally_launch_state* out);    /* non-blocking        */
int tally_launch_wait(int launch, tally_launch_state* out);     /* blocking            */
int tally_launch_elapsed_ns(int launch, long long* out);        /* needs desc.timed=1  */
int tally_preempt(int launch);                                  /* flag write; thread-safe */
/* Cooperative suspension (B200 extension): while on, pausable PTB launches
 * hold their place at the next suspension point (GEMM: every 4 k-blocks) and
 * resume in place when it clears -- no park, no relaunch. */
int tally_set_pause(int on);
int tally_launch_release(int launch);

/* ==== policy runner (ref scheduler.py:164-457) =============================== */
typedef struct {
  long long block_duration_ns, launch_overhead_ns, ptb_iteration_overhead_ns;
  int threads_per_block;
  long long total_blocks;
} tally_cost;               /* KernelCostModel (ref sim.py:77-111) */

typedef struct {
  int variant;              /* TALLY_SHAPE_ORIGINAL / _SLICED / _PTB (ConfigCandidate) */
  long long frac_num, frac_den;
  int worker_count;
} tally_candidate;

typedef struct {
  const char* kernel_id;    /* KernelWork.kernel_id                                   */
  tally_cost cost;          /* KernelWork.cost                                        */
  int exempt;               /* KernelWork.exempt                                      */
  int device_kernel;        /* instance id on the B200 device (-1 under a foreign device) */
  int has_config;           /* tuner's choice for Tally best-effort submission        */
  tally_candidate config;
  long long est_ns;         /* untransformed latency (the tuner's Original record) for the
                               real-time look-ahead budget; 0 = unknown                  */
} tally_work;

/* What the runner submits (SimLaunch, ref sim.py:140-153). */
typedef struct {
  int task;                 /* runner task index                                      */
  const char* task_id;
  const char* kernel_id;
  int priority;
  int shape;                /* ORIGINAL or PTB (a slice is an ORIGINAL launch of `count` blocks) */
  int worker_count;
  long long start_count;
  tally_cost cost;          /* cost.total_blocks = slice extent for a slice            */
  long long block_offset;   /* linear logical-block offset of a slice, else 0         */
  int is_slice;
  int device_kernel;
} tally_submit_desc;

typedef struct {
  int done, parked, preempted, is_ptb;
  long long task_counter;
  long long finish_time;    /* -1 while running */
} tally_handle_state;       /* KernelHandle fields (ref sim.py:175-226) */

/* The GpuSim surface the runner drives (ref sim.py:229-351).
 * Events flow back through tally_runner_on_event / _fire / _filter. */
typedef struct {
  void* ctx;
  long long (*now)(void* ctx);
  long long (*submit)(void* ctx, const tally_submit_desc* d);   /* >= 0 handle */
  int (*signal_preempt)(void* ctx, long long handle);
  int (*query)(void* ctx, long long handle, tally_handle_state* out);
  int (*call_at)(void* ctx, long long t_ns, long long token);
  int (*set_dispatch_filter)(void* ctx, int enabled);
  int (*kick)(void* ctx);
  int (*run_to_completion)(void* ctx);
} tally_device_vtbl;

int tally_runner_create(int policy, long long threshold_ns, long long quantum_ns,
                        long long horizon_ns, int* out_runner);
int tally_runner_add_task(int runner, const char* task_id, int priority,
                          const tally_work* works, int n_works,
                          const long long* arrivals, int n_arrivals);
/* dev == NULL: run on the B200 device in real time (tally_init first). */
int tally_runner_run(int runner, const tally_device_vtbl* dev);
int tally_runner_fire(int runner, long long token);
int tally_runner_on_event(int runner, int kind, long long handle);
int tally_runner_filter(int runner, long long handle);          /* 1 = may dispatch */
int tally_runner_request_count(int runner, int task);
int tally_runner_requests(int runner, int task, long long* out_pairs, int cap);
int tally_runner_iteration_count(int runner, int task);
int tally_runner_iterations(int runner, int task, long long* out, int cap);
int tally_runner_destroy(int runner);
/* Options for the B200 device run: "trace" (1 = bracket every launch with
 * timing events for the launch log), "hp_streams" (size of the high-priority
 * stream pool, default 4), "suspend" (1 = Tally with cooperative suspension:
 * on HP arrival pausable BE launches are suspended in place instead of
 * parked, and resumed when HP goes inactive; other BE launches are preempted
 * as usual). */
int tally_runner_set_option(int runner, const char* key, long long value);

/* Real-device run log (only after tally_runner_run(runner, NULL)). */
typedef struct {
  long long time_ns;
  int kind;                 /* TALLY_EV_* */
  int task;
  int kernel_index;         /* index within the task's pipeline */
  long long block;
} tally_event;

typedef struct {
  int task, kernel_index, priority, shape, workers;
  long long count, start_count, task_counter;
  long long submit_ns, issue_ns, complete_ns, preempt_ns;      /* host clock, run-relative */
  long long gt_first_start, gt_first_stop, gt_last_exit;       /* device clock            */
  int parked;
  long long gpu_start_ns, gpu_end_ns;  /* GPU timeline (CUDA events vs a run-start reference
                                          event; -1 unless the "trace" option is set)       */
  long long handle;         /* the device handle the runner got from submit (submission order) */
  long long gt_last_busy_exit;   /* see tally_launch_state */
} tally_launch_record;

long long tally_device_run_origin_ns(int runner);   /* host ns that event times are relative to */
int tally_device_event_count(int runner);
int tally_device_events(int runner, tally_event* out, int cap);
int tally_device_launch_count(int runner);
int tally_device_launches(int runner, tally_launch_record* out, int cap);

#ifdef __cplusplus
}
#endif
#endif /* TALLY_B200_H */
