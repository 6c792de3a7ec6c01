// The B200 device: the GpuSim surface (ref sim.py:229-351) implemented in real
// time over per-priority CUDA streams.  This is Tally's host dispatch daemon:
// one busy-polling host thread that
//   * fires arrivals at their trace times (host CLOCK_MONOTONIC, run-relative),
//   * launches high-priority kernels on a greatest-priority stream pool the
//     moment the runner submits them, after raising the preemption flag of
//     every in-flight best-effort PTB launch (flag write = cuStreamWriteValue32
//     on a dedicated top-priority stream, or a store to mapped host memory),
//   * launches best-effort slices / PTB workers on per-task lowest-priority
//     streams while the high-priority side is inactive,
//   * detects completion (PTB: the outcome mirror the last worker publishes;
//     others: a stream event) and feeds KernelFinished / WorkerParked back to
//     the runner.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <deque>
#include <map>
#include <unordered_map>
#include <queue>
#include <vector>

#include "runner.h"
#include "runtime.h"

namespace tally {

void set_error(const char* fmt, ...);

namespace {

struct Handle {
  tally_submit_desc d{};
  int launch = -1;
  bool issued = false, finished = false, parked = false, preempted = false;
  long long task_counter = 0;
  long long finish_time = -1;
  long long submit_ns = 0, issue_ns = 0, complete_ns = 0, preempt_ns = 0;
  long long gt_first_start = 0, gt_first_stop = 0, gt_last_exit = 0, gt_last_busy_exit = 0;
  long long count = 0;
  long long gpu_start = -1, gpu_end = -1;
  int kernel_index = -1;   // position of the work in its task's pipeline
  int hp_slot = -1;
};

class CudaDevice : public Device {
 public:
  explicit CudaDevice(Runner* r) : r_(r) {
    Runtime& R = rt();
    if (!R.inited) throw Error(TALLY_EINVAL, "tally_init must be called before running on the B200");
    trace_ = r_->option("trace", 0) != 0;
    chain_ = r_->option("lookahead", 1) > 1;
    const int n_hp = (int)r_->option("hp_streams", 4);
    for (int i = 0; i < n_hp; ++i) {
      int s;
      if (tally_stream_create(TALLY_HIGH, &s) != TALLY_OK) throw Error(TALLY_ECUDA, "HP stream");
      hp_streams_.push_back(s);
      hp_load_.push_back(0);
    }
    if (trace_) {
      cudaEventCreate(&ref_);
      cudaEventRecord(ref_, R.sig_stream);
      cudaEventSynchronize(ref_);
    }
    t0_ = host_now_ns();
    r_->log.t0_ns = t0_;
  }
  ~CudaDevice() override {
    if (held_) tally_set_pause(0);
    for (auto& h : hs_)
      if (h.launch >= 0 && !h.finished) tally_launch_wait(h.launch, nullptr);
    for (auto& h : hs_)
      if (h.launch >= 0) tally_launch_release(h.launch);
    for (int s : hp_streams_) tally_stream_destroy(s);
    if (ref_) cudaEventDestroy(ref_);
    for (auto& kv : be_streams_) tally_stream_destroy(kv.second);
  }

  long long now() override { return host_now_ns() - t0_; }

  long long submit(const tally_submit_desc& d) override {
    if (d.device_kernel < 0) throw Error(TALLY_EINVAL, std::string(d.kernel_id) + ": no device kernel bound");
    Handle h;
    h.d = d;
    h.submit_ns = now();
    h.kernel_index = kernel_index_of(d.task, d.device_kernel);
    hs_.push_back(h);
    const long long id = (long long)hs_.size() - 1;
    log_event(TALLY_EV_LAUNCH_ISSUED, id, -1);
    pending_.push_back(id);   // issued after the current runner callback returns
    return id;
  }

  void signal_preempt(long long id) override {
    Handle& h = get(id);
    if (h.d.shape != TALLY_SHAPE_PTB) throw Error(TALLY_EINVAL, std::string(h.d.kernel_id) + ": not a Ptb launch");
    if (h.finished) throw Error(TALLY_EINVAL, std::string(h.d.kernel_id) + ": not in flight");
    if (h.preempted) return;
    h.preempted = true;
    h.preempt_ns = now();
    log_event(TALLY_EV_PREEMPT_SIGNALED, id, -1);
    if (!h.issued) {
      // never reached the GPU: park immediately with no progress
      park_unissued_.push_back(id);
      return;
    }
    Launch* L = rt().get_launch(h.launch);
    if (L && !L->finished) {
      int rc = tally_preempt(h.launch);
      if (rc != TALLY_OK && rc != TALLY_EINVAL) throw Error(rc, tally_last_error());
    }
  }

  tally_handle_state query(long long id) override {
    const Handle& h = get(id);
    tally_handle_state s;
    memset(&s, 0, sizeof(s));
    s.done = h.finished && !h.parked;
    s.parked = h.parked;
    s.preempted = h.preempted;
    s.is_ptb = h.d.shape == TALLY_SHAPE_PTB;
    s.task_counter = h.task_counter;
    s.finish_time = h.finish_time;
    return s;
  }

  void call_at(long long t, long long token) override {
    timers_.push(Tm{t, seq_++, token});
  }

  bool hold(long long id) override {
    Handle& h = get(id);
    if (h.d.shape != TALLY_SHAPE_PTB || h.finished || !pausable(h.d.device_kernel)) return false;
    if (!held_) {
      int rc = tally_set_pause(1);
      if (rc != TALLY_OK) throw Error(rc, tally_last_error());
      held_ = true;
      log_event(TALLY_EV_PREEMPT_SIGNALED, id, -2);   // block -2 marks a suspension
    }
    return true;
  }

  void release_holds() override {
    if (!held_) return;
    int rc = tally_set_pause(0);
    if (rc != TALLY_OK) throw Error(rc, tally_last_error());
    held_ = false;
  }

  void set_dispatch_filter(bool e) override { filter_ = e; }
  void kick() override { dispatch(); }

  void run_to_completion() override {
    cudaSetDevice(rt().device);
    while (!timers_.empty() || inflight_ > 0 || !pending_.empty() || !park_unissued_.empty()) {
      bool progress = false;
      const long long t = now();
      while (!timers_.empty() && timers_.top().t <= t) {
        Tm tm = timers_.top();
        timers_.pop();
        last_fired_ = tm.t;
        {
          tally_event e;
          e.time_ns = now();
          e.kind = TALLY_EV_TIMER_FIRED;
          e.task = -1;
          e.kernel_index = -1;
          e.block = tm.t;
          r_->log.events.push_back(e);
        }
        r_->fire(tm.token);
        dispatch();
        progress = true;
      }
      for (long long id : std::vector<long long>(park_unissued_)) {
        Handle& h = hs_[(size_t)id];
        h.finished = h.parked = true;
        h.task_counter = h.d.start_count;
        h.complete_ns = now();
        pending_.erase(std::remove(pending_.begin(), pending_.end(), id), pending_.end());
        log_event(TALLY_EV_WORKER_PARKED, id, -1);
        record(id);
        r_->on_event(TALLY_EV_WORKER_PARKED, id);
        dispatch();
        progress = true;
      }
      park_unissued_.clear();
      if (inflight_ > 0) {
        // poll in submission order; complete() may submit (appending to live_)
        const size_t n = live_.size();
        for (size_t k = 0; k < n; ++k) {
          const long long id = live_[k];
          Handle& h = hs_[(size_t)id];
          if (h.finished) continue;
          Launch* L = rt().get_launch(h.launch);
          if (!L) throw Error(TALLY_ECUDA, "lost launch");
          if (!rt().poll(L)) {
            if (L->error != cudaSuccess) throw Error(TALLY_ECUDA, cudaGetErrorString(L->error));
            continue;
          }
          complete(id, L);
          progress = true;
        }
        live_.erase(std::remove_if(live_.begin(), live_.end(),
                                   [this](long long id) { return hs_[(size_t)id].finished; }),
                    live_.end());
      }
      if (!pending_.empty()) { dispatch(); }
      if (!progress) spin_pause();
    }
  }

 private:
  struct Tm {
    long long t, seq, token;
    bool operator<(const Tm& o) const { return t != o.t ? t > o.t : seq > o.seq; }   // min-heap
  };

  Runner* r_;
  long long t0_ = 0, seq_ = 0, last_fired_ = 0;
  std::priority_queue<Tm> timers_;
  std::deque<Handle> hs_;          // deque: references stay valid across submit()
  std::vector<long long> live_;    // issued, not yet observed finished
  std::vector<long long> pending_, park_unissued_;
  int inflight_ = 0;
  bool filter_ = false;
  bool trace_ = false;
  bool held_ = false;
  bool chain_ = false;   // look-ahead: best-effort PTB launches park on their stream's chain word
  std::map<int, bool> pausable_cache_;

  bool pausable(int kernel) {
    auto it = pausable_cache_.find(kernel);
    if (it != pausable_cache_.end()) return it->second;
    Runtime& R = rt();
    bool p = kernel >= 0 && kernel < (int)R.instances.size() && R.instances[(size_t)kernel] &&
             R.kinds[R.instances[(size_t)kernel]->kind].pausable;
    pausable_cache_[kernel] = p;
    return p;
  }
  std::map<int, long long> total_cache_;
  cudaEvent_t ref_ = nullptr;
  int hp_rr_ = 0;
  std::vector<int> hp_streams_;
  std::vector<int> hp_load_;   // in-flight launches per HP stream
  std::map<int, int> be_streams_;

  static void spin_pause() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }

  // (task, device kernel) -> pipeline position, built once per task: the
  // daemon's per-event bookkeeping stays O(1) for ~400-kernel pipelines
  std::vector<std::unordered_map<int, int>> kidx_;
  int kernel_index_of(int task, int device_kernel) {
    if ((size_t)task >= kidx_.size()) kidx_.resize((size_t)task + 1);
    auto& m = kidx_[(size_t)task];
    if (m.empty()) {
      const auto& ks = r_->tasks[(size_t)task].kernels;
      for (size_t k = ks.size(); k-- > 0;) m[ks[k].device_kernel] = (int)k;   // first occurrence wins
    }
    auto it = m.find(device_kernel);
    return it == m.end() ? -1 : it->second;
  }

  Handle& get(long long id) {
    if (id < 0 || id >= (long long)hs_.size()) throw Error(TALLY_EINVAL, "unknown handle");
    return hs_[(size_t)id];
  }

  void log_event(int kind, long long id, long long block) {
    const Handle& h = hs_[(size_t)id];
    tally_event e;
    e.time_ns = now();
    e.kind = kind;
    e.task = h.d.task;
    e.kernel_index = h.kernel_index;
    e.block = block;
    r_->log.events.push_back(e);
  }

  // One stream per (task, priority class) for everything but high-priority
  // inference: a training task's kernels must run in order (with look-ahead
  // several of them are queued at once), and a best-effort inference task's
  // requests share its lowest-priority stream.
  int task_stream(int task, int priority) {
    const int key = 2 * task + (priority == TALLY_HIGH ? 1 : 0);
    auto it = be_streams_.find(key);
    if (it != be_streams_.end()) return it->second;
    int s;
    if (tally_stream_create(priority, &s) != TALLY_OK) throw Error(TALLY_ECUDA, tally_last_error());
    be_streams_[key] = s;
    return s;
  }

  void dispatch() {
    if (pending_.empty()) return;
    std::vector<long long> keep;
    // high priority first (ref sim.py:381-393)
    for (int pass = 0; pass < 2; ++pass) {
      for (long long id : pending_) {
        Handle& h = hs_[(size_t)id];
        if ((h.d.priority == TALLY_HIGH) != (pass == 0)) continue;
        if (filter_ && !r_->filter(id)) {
          keep.push_back(id);
          continue;
        }
        issue(id);
      }
    }
    pending_.swap(keep);
  }

  void issue(long long id) {
    Handle& h = hs_[(size_t)id];
    tally_launch_desc ld;
    memset(&ld, 0, sizeof(ld));
    ld.preempt_at = -1;
    auto kit = total_cache_.find(h.d.device_kernel);
    if (kit == total_cache_.end()) {
      tally_kernel_info info;
      if (tally_kernel_info_get(h.d.device_kernel, &info) != TALLY_OK) throw Error(TALLY_EINVAL, tally_last_error());
      kit = total_cache_.emplace(h.d.device_kernel, info.total_blocks).first;
    }
    struct { long long total_blocks; } ki{kit->second};
    if (h.d.shape == TALLY_SHAPE_PTB) {
      ld.shape = TALLY_SHAPE_PTB;
      ld.chain = (chain_ && h.d.priority == TALLY_BEST_EFFORT) ? 1 : 0;
      ld.pausable = r_->option("suspend", 0) ? 1 : 0;
      ld.workers = h.d.worker_count;
      ld.start_count = h.d.start_count;
      h.count = ki.total_blocks;
    } else if (h.d.is_slice || h.d.cost.total_blocks != ki.total_blocks) {
      ld.shape = TALLY_SHAPE_SLICED;
      ld.linear = 1;
      ld.linear_offset = h.d.block_offset;
      ld.count = h.d.cost.total_blocks;
      h.count = ld.count;
    } else {
      ld.shape = TALLY_SHAPE_ORIGINAL;
      h.count = ki.total_blocks;
    }
    int stream;
    ld.timed = trace_ ? 1 : 0;
    const bool training = r_->tasks[(size_t)h.d.task].arrivals.empty();
    if (training) {
      stream = task_stream(h.d.task, h.d.priority);
    } else if (h.d.priority == TALLY_HIGH) {
      // an idle high-priority stream if there is one (no head-of-line blocking
      // behind another request), else the least loaded
      size_t best = 0;
      for (size_t k = 0; k < hp_streams_.size(); ++k) {
        const size_t c = (hp_rr_ + k) % hp_streams_.size();
        if (hp_load_[c] < hp_load_[best] || (k == 0)) best = c;
        if (hp_load_[c] == 0) { best = c; break; }
      }
      hp_rr_ = (int)((best + 1) % hp_streams_.size());
      h.hp_slot = (int)best;
      ++hp_load_[best];
      stream = hp_streams_[best];
    } else {
      stream = task_stream(h.d.task, TALLY_BEST_EFFORT);
    }
    int lid = -1;
    int rc = tally_launch(h.d.device_kernel, stream, &ld, &lid);
    if (rc != TALLY_OK) throw Error(rc, tally_last_error());
    h.launch = lid;
    h.issued = true;
    h.issue_ns = now();
    ++inflight_;
    live_.push_back(id);
    if (h.preempted) tally_preempt(lid);
  }

  void complete(long long id, Launch* L) {
    Handle& h = hs_[(size_t)id];
    h.finished = true;
    if (h.hp_slot >= 0) --hp_load_[(size_t)h.hp_slot];
    h.parked = L->parked;
    h.complete_ns = now();
    h.finish_time = h.complete_ns;
    h.task_counter = L->shape == TALLY_SHAPE_PTB ? L->start_count + L->claims : 0;
    h.gt_first_start = L->gt_first_start;
    h.gt_first_stop = L->gt_first_stop;
    h.gt_last_exit = L->gt_last_exit;
    h.gt_last_busy_exit = L->gt_last_busy_exit;
    --inflight_;
    if (trace_ && L->ev_start && L->ev_end) {
      float ms0 = 0, ms1 = 0;
      cudaEventSynchronize(L->ev_end);
      if (cudaEventElapsedTime(&ms0, ref_, L->ev_start) == cudaSuccess &&
          cudaEventElapsedTime(&ms1, ref_, L->ev_end) == cudaSuccess) {
        h.gpu_start = (long long)(ms0 * 1e6);
        h.gpu_end = (long long)(ms1 * 1e6);
      }
      cudaGetLastError();
    }
    record(id);
    tally_launch_release(h.launch);
    h.launch = -1;
    if (h.parked) {
      log_event(TALLY_EV_WORKER_PARKED, id, -1);
      r_->on_event(TALLY_EV_WORKER_PARKED, id);
    } else {
      log_event(TALLY_EV_KERNEL_FINISHED, id, -1);
      r_->on_event(TALLY_EV_KERNEL_FINISHED, id);
    }
    dispatch();
  }

  void record(long long id) {
    const Handle& h = hs_[(size_t)id];
    tally_launch_record rec;
    memset(&rec, 0, sizeof(rec));
    rec.task = h.d.task;
    rec.kernel_index = h.kernel_index;
    rec.priority = h.d.priority;
    rec.shape = h.d.shape == TALLY_SHAPE_PTB ? TALLY_SHAPE_PTB
                : (h.d.is_slice ? TALLY_SHAPE_SLICED : TALLY_SHAPE_ORIGINAL);
    rec.workers = h.d.worker_count;
    rec.count = h.count;
    rec.start_count = h.d.start_count;
    rec.task_counter = h.task_counter;
    rec.submit_ns = h.submit_ns;
    rec.issue_ns = h.issue_ns;
    rec.complete_ns = h.complete_ns;
    rec.preempt_ns = h.preempted ? h.preempt_ns : -1;
    rec.gt_first_start = h.gt_first_start;
    rec.gt_first_stop = h.gt_first_stop;
    rec.gt_last_exit = h.gt_last_exit;
    rec.parked = h.parked ? 1 : 0;
    rec.gpu_start_ns = h.gpu_start;
    rec.gpu_end_ns = h.gpu_end;
    rec.handle = id;
    rec.gt_last_busy_exit = h.gt_last_busy_exit;
    r_->log.launches.push_back(rec);
  }
};

}  // namespace

Device* make_cuda_device(Runner* r) { return new CudaDevice(r); }

}  // namespace tally
