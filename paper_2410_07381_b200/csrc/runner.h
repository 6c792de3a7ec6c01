// Policy runner (Tally + Eager / KernelPriority / TimeSliced baselines) over an
// abstract device with the GpuSim surface (ref sim.py:229-351).
#pragma once
#include <deque>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/tally_b200.h"

namespace tally {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

class Runner;

// The device half of the boundary.  Implementations: VtblDevice (foreign
// device through tally_device_vtbl, e.g. the CPU oracle in the parity tests)
// and CudaDevice (the B200, cuda_device.cpp).  Errors are thrown as tally::Error.
struct Device {
  virtual ~Device() = default;
  virtual long long now() = 0;
  virtual long long submit(const tally_submit_desc& d) = 0;
  virtual void signal_preempt(long long h) = 0;
  virtual tally_handle_state query(long long h) = 0;
  virtual void call_at(long long t, long long token) = 0;
  virtual void set_dispatch_filter(bool enabled) = 0;
  virtual void kick() = 0;
  virtual void run_to_completion() = 0;
  // Cooperative suspension (B200 extension; no-op for foreign devices):
  // hold() suspends launch h in place and returns true if it can.
  virtual bool hold(long long) { return false; }
  virtual void release_holds() {}
};

struct Work {
  std::string kernel_id;
  tally_cost cost{};
  bool exempt = false;
  int device_kernel = -1;
  bool has_config = false;
  tally_candidate config{};
  long long est_ns = 0;      // untransformed latency (look-ahead budget), 0 = unknown
};

struct Task {
  std::string id;
  int priority = TALLY_HIGH;
  std::vector<Work> kernels;
  std::vector<long long> arrivals;
  bool inference() const { return !arrivals.empty(); }
  // run state (ref scheduler.py:115-153)
  struct Req {
    long long arrival;
    int k = 0;
    long long h = -1;
  };
  std::deque<long long> pending;
  std::vector<Req> reqs;
  bool concurrent = false;
  bool in_arrival = false;
  long long arrival = 0;
  int k = 0;
  long long h = -1;
  bool h_is_slice = false;
  bool has_cfg = false;
  tally_candidate cfg{};
  std::vector<long long> tiling;
  int slice_i = 0;
  long long ptb_counter = 0;
  // Real-time look-ahead (runner option "lookahead" > 1): kernels k+1, k+2,
  // ... submitted behind the in-flight head on the task's stream.
  struct Ahead {
    int k;
    long long h;
    tally_candidate cfg;
  };
  std::deque<Ahead> ahead;
  std::vector<std::pair<long long, long long>> requests;
  std::vector<long long> iterations;
  bool in_service() const { return in_arrival || !reqs.empty(); }
  bool has_queued_work() const { return !pending.empty() || in_service(); }
  void new_kernel() {
    has_cfg = false;
    tiling.clear();
    slice_i = 0;
    ptb_counter = 0;
  }
};

// Device-side run log kept for the B200 device.
struct DeviceLog {
  long long t0_ns = 0;   // host CLOCK_MONOTONIC at run start (event times are relative to it)
  std::vector<tally_event> events;
  std::vector<tally_launch_record> launches;
};

class Runner {
 public:
  Runner(int policy, long long threshold, long long quantum, long long horizon);
  void add_task(Task t);
  void run(Device* dev);
  void fire(long long token);
  void on_event(int kind, long long h);
  bool filter(long long h);

  std::vector<Task> tasks;
  DeviceLog log;
  std::map<std::string, long long> options;
  long long option(const std::string& k, long long dflt) const {
    auto it = options.find(k);
    return it == options.end() ? dflt : it->second;
  }
  int policy;
  long long threshold, quantum, horizon;

 private:
  struct Timer {
    int kind;     // 0 arrival, 1 tick, 2 time-slice rotation
    int task;
    long long t;
  };
  struct HInfo {
    int task;
    int priority;
  };
  Device* dev_ = nullptr;
  std::vector<Timer> timers_;
  std::map<long long, HInfo> hinfo_;
  std::vector<int> hp_, be_;
  int rr_ = 0;
  bool ticking_ = false;
  bool suspend_ = false;
  int ts_active_ = 0;
  bool ts_armed_ = false;

  long long token(int kind, int task, long long t);
  void arrive(int task, long long t);
  void tick();
  void absorb();
  void kernel_done(Task& st);
  bool hp_active();
  const Work* next_work(Task& st);
  void advance(int task, int pclass);
  long long submit(int task, const Work& w, int priority, int shape, int workers,
                   long long start, long long total_blocks, long long offset, bool is_slice);
  void preempt_be();
  void submit_be(int task, const Work& w);
  int lookahead_ = 1;
  void fill_ahead(int task);
  bool settle_ahead(Task& st);
  bool ts_has_work(const Task& st);
  void ts_arm();
  void ts_rotate();
  bool done(long long h) { return dev_->query(h).done != 0; }
};

std::vector<long long> slice_extents(long long len, long long num, long long den);
Device* make_cuda_device(Runner* r);

}  // namespace tally
