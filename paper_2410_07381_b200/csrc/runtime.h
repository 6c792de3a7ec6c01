// Internal runtime state shared by runtime.cu, runner.cpp and cuda_device.cpp.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <deque>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <utility>
#include <vector>

#include "registry.h"

namespace tally {

long long host_now_ns();

typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*ModuleLoadDataFn)(CUmodule*, const void*);
typedef CUresult (*ModuleGetFunctionFn)(CUfunction*, CUmodule, const char*);
typedef CUresult (*LaunchKernelFn)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                   unsigned, CUstream, void**, void**);
typedef CUresult (*OccupancyFn)(int*, CUfunction, int, size_t);

struct Launch {
  int kernel = -1, stream = -1, shape = 0;
  int rec = -1;
  unsigned serial = 0;
  int flag_host = 0;
  bool timed = false;
  bool active = false;
  bool finished = false;
  bool parked = false;
  std::atomic<bool> preempted{false};
  long long start_count = 0, workers = 0, count = 0;
  long long claims = 0;
  long long gt_first_start = 0, gt_first_stop = 0, gt_last_exit = 0, gt_last_busy_exit = 0;
  long long host_submit = 0, host_preempt = 0;
  cudaEvent_t ev_start = nullptr, ev_end = nullptr;
  cudaError_t error = cudaSuccess;
  unsigned polls = 0;   // PTB: mirror polls since the last end-event check
  bool chain = false;   // PTB on its stream's chain word (park_at = epoch)
  int chain_stream = -1;
  unsigned park_at = 0;
};

struct Runtime {
  static constexpr int kMaxKinds = 1024;   // built-ins + IR-JIT kinds
  static constexpr int kMaxRecs = 1024;

  std::mutex mu;
  bool inited = false;
  int device = -1;
  tally_gpu_info info{};
  KernelKind kinds[kMaxKinds];
  int nkinds = 0;
  std::vector<std::unique_ptr<Instance>> instances;
  std::vector<cudaStream_t> streams;
  std::vector<char> stream_be;   // best-effort class (programmatic dependent launch when enabled)
  bool pdl = false;              // TALLY_PDL=1
  int prio_low = 0, prio_high = 0;
  cudaStream_t sig_stream = nullptr;

  LaunchRec* d_recs = nullptr;
  ExitGroup* d_groups = nullptr;      // [kMaxRecs][kMaxExitGroups] two-level worker retirement
  LaunchMirror* h_mirrors = nullptr;
  LaunchMirror* d_mirrors = nullptr;
  volatile unsigned* h_flags = nullptr;
  unsigned* d_hflags = nullptr;
  unsigned* d_pause = nullptr;        // global suspension word (device memory)
  // Chain preemption words, one per stream (PtbArgs::park_at): device word,
  // its mapped host mirror, and the epoch last written per stream.
  static constexpr int kMaxChainStreams = 4096;
  unsigned* d_chain = nullptr;
  volatile unsigned* h_chain = nullptr;
  unsigned* d_hchain = nullptr;
  std::vector<unsigned> chain_epoch;
  int pause_on = 0;
  volatile unsigned long long* h_stamp = nullptr;
  unsigned long long* d_stamp = nullptr;
  std::vector<int> free_recs;
  std::deque<std::pair<int, cudaEvent_t>> zombies;
  std::atomic<unsigned> next_serial{0};
  int flag_host = 0;
  WriteValue32Fn write32 = nullptr;
  ModuleLoadDataFn cu_module_load = nullptr;
  ModuleGetFunctionFn cu_get_function = nullptr;
  LaunchKernelFn cu_launch = nullptr;
  OccupancyFn cu_occupancy = nullptr;
  int jit_register(const char* name, const void* image, const char* syms[3], const unsigned grid[3],
                   int threads, long long smem, int* out_kind);

  std::unordered_map<const void*, void*> jit_modules;   // cubin image -> CUmodule
  std::vector<std::unique_ptr<Launch>> launches;
  std::vector<int> free_launch_ids;
  std::vector<cudaEvent_t> timed_events, plain_events;
  std::unordered_map<cudaEvent_t, bool> event_timed;

  int init(int dev, tally_gpu_info* out);
  int clock_offset(long long* off, long long* unc);
  int alloc_rec(int* out);
  cudaEvent_t get_event(bool timed);
  void release_event(cudaEvent_t e);
  int launch(int kernel, int stream, const tally_launch_desc* d, int* out);
  Launch* get_launch(int id);
  bool poll(Launch* L);
  void fill_state(const Launch* L, tally_launch_state* o);
  int preempt(int id);
  int set_pause(int on);
  int release(int id);
};

Runtime& rt();

}  // namespace tally
