// Tally policy runner -- a native restatement of the reference PolicyRunner
// semantics (ref scheduler.py:164-457) driving any device that exposes the
// GpuSim surface.  On the B200 it is the host dispatch daemon (cuda_device.cpp);
// under the parity tests it drives the CPU oracle through tally_device_vtbl and
// must reproduce the reference's event log byte for byte.
#include "runner.h"

#include <algorithm>
#include <cstring>
#include <memory>

#include "runtime.h"

namespace tally {

void set_error(const char* fmt, ...);

// Half-even rounding of a positive rational, as Python's round(Fraction)
// (ref transforms.py:136-152).
static long long round_half_even(long long num, long long den) {
  long long q = num / den, r = num % den;
  if (2 * r > den || (2 * r == den && (q & 1))) ++q;
  return q;
}

std::vector<long long> slice_extents(long long len, long long num, long long den) {
  if (den <= 0 || num <= 0 || num > den) throw Error(TALLY_ETRANSFORM, "slice fraction must be in (0, 1]");
  long long ext = std::min(std::max(1LL, round_half_even(num * len, den)), len);
  std::vector<long long> out((size_t)(len / ext), ext);
  out.back() += len % ext;
  return out;
}

Runner::Runner(int pol, long long th, long long q, long long hz)
    : policy(pol), threshold(th), quantum(q), horizon(hz) {
  if (pol < TALLY_POLICY_TALLY || pol > TALLY_POLICY_TIME_SLICED) throw Error(TALLY_EINVAL, "unknown policy");
  if (th <= 0) throw Error(TALLY_EINVAL, "turnaround threshold must be > 0");
  if (q <= 0) throw Error(TALLY_EINVAL, "time-slice quantum must be > 0");
}

void Runner::add_task(Task t) {
  for (auto& o : tasks)
    if (o.id == t.id) throw Error(TALLY_EINVAL, "duplicate task ids");
  if (t.kernels.empty()) throw Error(TALLY_EINVAL, t.id + ": empty kernel pipeline");
  for (size_t i = 1; i < t.arrivals.size(); ++i)
    if (t.arrivals[i] < t.arrivals[i - 1]) throw Error(TALLY_EINVAL, t.id + ": arrivals must be non-decreasing");
  tasks.push_back(std::move(t));
}

long long Runner::token(int kind, int task, long long t) {
  timers_.push_back(Timer{kind, task, t});
  return (long long)timers_.size() - 1;
}

void Runner::run(Device* dev) {
  dev_ = dev;
  suspend_ = policy == TALLY_POLICY_TALLY && option("suspend", 0) != 0;
  lookahead_ = (int)std::max(1LL, option("lookahead", 1));
  if (policy == TALLY_POLICY_TIME_SLICED) lookahead_ = 1;
  hp_.clear();
  be_.clear();
  for (size_t i = 0; i < tasks.size(); ++i) {
    Task& st = tasks[i];
    // inference is served concurrently unless best-effort under a
    // priority-aware policy (ref scheduler.py:187-193)
    st.concurrent = st.inference() &&
                    (st.priority == TALLY_HIGH || policy == TALLY_POLICY_EAGER ||
                     policy == TALLY_POLICY_TIME_SLICED);
    (st.priority == TALLY_HIGH ? hp_ : be_).push_back((int)i);
  }
  if (policy == TALLY_POLICY_TIME_SLICED || policy == TALLY_POLICY_KERNEL_PRIORITY)
    dev_->set_dispatch_filter(true);
  // the time-slice clock starts before arrivals are registered (ref scheduler.py:439-441, :456)
  if (policy == TALLY_POLICY_TIME_SLICED) ts_arm();
  for (size_t i = 0; i < tasks.size(); ++i)
    for (long long t : tasks[i].arrivals) dev_->call_at(t, token(0, (int)i, t));
  dev_->call_at(0, token(1, -1, 0));
  dev_->run_to_completion();
}

void Runner::fire(long long tok) {
  if (tok < 0 || tok >= (long long)timers_.size()) throw Error(TALLY_EINVAL, "unknown timer token");
  const Timer tm = timers_[(size_t)tok];
  if (tm.kind == 0) arrive(tm.task, tm.t);
  else if (tm.kind == 1) tick();
  else ts_rotate();
}

void Runner::on_event(int kind, long long) {
  // only kernel boundaries and worker parkings change scheduler state
  if (kind == TALLY_EV_KERNEL_FINISHED || kind == TALLY_EV_WORKER_PARKED) tick();
}

void Runner::arrive(int task, long long t) {
  tasks[task].pending.push_back(t);
  tick();
  if (policy == TALLY_POLICY_TIME_SLICED) ts_arm();
}

void Runner::tick() {
  if (ticking_) return;   // submissions inside a tick re-enter via their own events
  ticking_ = true;
  try {
    absorb();
    if (policy == TALLY_POLICY_TALLY || policy == TALLY_POLICY_KERNEL_PRIORITY) {
      for (int i : hp_) advance(i, TALLY_HIGH);
      if (suspend_ && !hp_active()) dev_->release_holds();
      if (!hp_active()) {
        const int n = (int)be_.size();
        std::vector<int> order;
        for (int i = 0; i < n; ++i) order.push_back(be_[(size_t)((rr_ + i) % n)]);
        for (int i : order) advance(i, TALLY_BEST_EFFORT);
      }
    } else {
      for (size_t i = 0; i < tasks.size(); ++i) advance((int)i, TALLY_HIGH);
    }
  } catch (...) {
    ticking_ = false;
    throw;
  }
  ticking_ = false;
}

void Runner::absorb() {
  const long long now = dev_->now();
  for (auto& st : tasks) {
    if (st.concurrent) {
      std::vector<size_t> finished;
      for (size_t r = 0; r < st.reqs.size(); ++r) {
        auto& rq = st.reqs[r];
        if (rq.h < 0 || !done(rq.h)) continue;
        rq.h = -1;
        rq.k += 1;
        if (rq.k == (int)st.kernels.size()) {
          st.requests.emplace_back(rq.arrival, now);
          finished.push_back(r);
        }
      }
      for (auto it = finished.rbegin(); it != finished.rend(); ++it)
        st.reqs.erase(st.reqs.begin() + (long)*it);
      continue;
    }
    while (st.h >= 0) {
      const tally_handle_state hs = dev_->query(st.h);
      if (hs.parked) {
        st.ptb_counter = hs.task_counter;   // resume point (ref scheduler.py:275-277)
        st.h = -1;
        break;
      }
      if (!hs.done) break;
      const bool was_slice = st.h_is_slice;
      st.h = -1;
      st.h_is_slice = false;
      if (was_slice) {
        st.slice_i += 1;
        if (st.slice_i < (int)st.tiling.size()) break;   // more slices remain
      }
      kernel_done(st);
      if (st.ahead.empty()) break;
      // real-time look-ahead: the next queued launch becomes the head
      const Task::Ahead a = st.ahead.front();
      st.ahead.pop_front();
      if (a.k != st.k) throw Error(TALLY_EINVAL, st.id + ": look-ahead launch out of order");
      st.h = a.h;
      st.cfg = a.cfg;
      st.has_cfg = true;
      st.ptb_counter = 0;
    }
    settle_ahead(st);
  }
}

// Look-ahead launches queued behind a head that parked park too (they share
// the stream's chain word, and a parked launch raises it before it exits);
// once all have reported they are dropped and re-queued behind the resumed
// head.  Returns true when none remain.
bool Runner::settle_ahead(Task& st) {
  if (st.ahead.empty()) return true;
  if (st.h >= 0) return false;
  for (const auto& a : st.ahead) {
    const tally_handle_state s = dev_->query(a.h);
    if (s.done || (s.parked && s.task_counter != 0))
      throw Error(TALLY_EINVAL, st.id + ": a look-ahead launch ran behind a parked one");
    if (!s.parked) return false;
  }
  st.ahead.clear();
  return true;
}

// Real-time look-ahead (runner option "lookahead" = L > 1; the reference
// keeps one kernel in flight per task, which the parity tests keep): up to
// L - 1 further kernels of a training task are queued behind the in-flight
// head on the task's stream, so the GPU never idles between best-effort
// kernels waiting for the host to observe a completion and launch the next.
// What may be queued keeps the policy's bound on high-priority delay:
//   * PTB launches (Tally) -- they share the stream's chain preemption word,
//     so preempting the head parks the whole queue (before any claim);
//   * untransformed launches only ahead of every PTB launch in the queue (a
//     launch that cannot park must never overtake a parked one) and, except
//     under Eager, only while their summed latency stays within the
//     turnaround threshold -- what a high-priority arrival may wait for;
//   * never a Sliced kernel (its slices go one at a time), never past the
//     end of the iteration, never a second launch of a kernel instance
//     already in flight (per-instance chain state).
void Runner::fill_ahead(int task) {
  Task& st = tasks[(size_t)task];
  if (lookahead_ <= 1 || st.inference() || st.concurrent || st.h < 0 || st.h_is_slice) return;
  const bool tally = policy == TALLY_POLICY_TALLY;
  const int prio = (policy == TALLY_POLICY_TALLY || policy == TALLY_POLICY_KERNEL_PRIORITY) ? st.priority : TALLY_HIGH;
  bool ptb_queued = st.has_cfg && st.cfg.variant == TALLY_SHAPE_PTB;
  long long budget = 0;
  for (const auto& a : st.ahead) {
    if (a.cfg.variant == TALLY_SHAPE_PTB) ptb_queued = true;
    else budget += st.kernels[(size_t)a.k].est_ns;
  }
  while ((int)st.ahead.size() + 1 < lookahead_) {
    const int j = st.k + 1 + (int)st.ahead.size();
    if (j >= (int)st.kernels.size()) break;
    const Work& w = st.kernels[(size_t)j];
    bool busy = w.device_kernel == st.kernels[(size_t)st.k].device_kernel;
    for (const auto& a : st.ahead) busy = busy || st.kernels[(size_t)a.k].device_kernel == w.device_kernel;
    if (busy) break;
    tally_candidate cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.variant = TALLY_SHAPE_ORIGINAL;
    if (tally && st.priority == TALLY_BEST_EFFORT && !w.exempt) {
      if (!w.has_config) break;
      cfg = w.config;
    }
    if (cfg.variant == TALLY_SHAPE_SLICED) break;
    if (cfg.variant == TALLY_SHAPE_PTB) {
      ptb_queued = true;
    } else {
      if (ptb_queued) break;
      if (policy != TALLY_POLICY_EAGER) {
        if (w.est_ns <= 0 || budget + w.est_ns > threshold) break;
        budget += w.est_ns;
      }
    }
    const long long h = cfg.variant == TALLY_SHAPE_PTB
        ? submit(task, w, prio, TALLY_SHAPE_PTB, cfg.worker_count, 0, w.cost.total_blocks, 0, false)
        : submit(task, w, prio, TALLY_SHAPE_ORIGINAL, 0, 0, w.cost.total_blocks, 0, false);
    st.ahead.push_back(Task::Ahead{j, h, cfg});
  }
}

void Runner::kernel_done(Task& st) {
  st.new_kernel();
  st.k += 1;
  if (st.k < (int)st.kernels.size()) return;
  st.k = 0;
  const long long now = dev_->now();
  st.requests.emplace_back(st.arrival, now);
  if (!st.inference()) st.iterations.push_back(now);
  st.in_arrival = false;
}

bool Runner::hp_active() {
  for (int i : hp_) {
    const Task& s = tasks[(size_t)i];
    if (s.has_queued_work() || s.h >= 0) return true;
  }
  return false;
}

const Work* Runner::next_work(Task& st) {
  if (!st.in_service()) {
    if (st.inference()) {
      if (st.pending.empty()) return nullptr;
      st.arrival = st.pending.front();
      st.pending.pop_front();
    } else {
      if (dev_->now() >= horizon) return nullptr;
      st.arrival = dev_->now();   // iteration start
    }
    st.in_arrival = true;
  }
  return &st.kernels[(size_t)st.k];
}

long long Runner::submit(int task, const Work& w, int priority, int shape, int workers,
                         long long start, long long total_blocks, long long offset, bool is_slice) {
  tally_submit_desc d;
  memset(&d, 0, sizeof(d));
  d.task = task;
  d.task_id = tasks[(size_t)task].id.c_str();
  d.kernel_id = w.kernel_id.c_str();
  d.priority = priority;
  d.shape = shape;
  d.worker_count = workers;
  d.start_count = start;
  d.cost = w.cost;
  d.cost.total_blocks = total_blocks;
  d.block_offset = offset;
  d.is_slice = is_slice ? 1 : 0;
  d.device_kernel = w.device_kernel;
  const long long h = dev_->submit(d);
  hinfo_[h] = HInfo{task, priority};
  return h;
}

void Runner::advance(int task, int pclass) {
  Task& st = tasks[(size_t)task];
  if (st.concurrent) {
    while (!st.pending.empty()) {
      st.reqs.push_back(Task::Req{st.pending.front()});
      st.pending.pop_front();
    }
    for (size_t r = 0; r < st.reqs.size(); ++r) {
      if (st.reqs[r].h >= 0) continue;
      const Work& w = st.kernels[(size_t)st.reqs[r].k];
      const long long h = submit(task, w, pclass, TALLY_SHAPE_ORIGINAL, 0, 0, w.cost.total_blocks, 0, false);
      tasks[(size_t)task].reqs[r].h = h;
      if (pclass == TALLY_HIGH && policy == TALLY_POLICY_TALLY) preempt_be();
    }
    return;
  }
  if (st.h >= 0) {
    fill_ahead(task);
    return;
  }
  if (!st.ahead.empty()) return;   // queued look-ahead launches are still parking
  const Work* w = next_work(st);
  if (!w) return;
  if (pclass == TALLY_BEST_EFFORT && policy == TALLY_POLICY_TALLY && !w->exempt) {
    submit_be(task, *w);
  } else {
    const long long h = submit(task, *w, pclass, TALLY_SHAPE_ORIGINAL, 0, 0, w->cost.total_blocks, 0, false);
    tasks[(size_t)task].h = h;
    tasks[(size_t)task].h_is_slice = false;
    if (pclass == TALLY_HIGH && policy == TALLY_POLICY_TALLY) preempt_be();
  }
  fill_ahead(task);
  auto it = std::find(be_.begin(), be_.end(), task);
  if (it != be_.end()) rr_ = (int)(((it - be_.begin()) + 1) % (long)be_.size());
}

void Runner::preempt_be() {
  for (int i : be_) {
    const long long h = tasks[(size_t)i].h;
    if (h < 0) continue;
    const tally_handle_state s = dev_->query(h);
    if (s.is_ptb && !s.done && !s.preempted) {
      if (suspend_ && dev_->hold(h)) continue;   // suspended in place, resumes when HP is idle
      dev_->signal_preempt(h);
    }
    for (const auto& a : tasks[(size_t)i].ahead) {   // the queued look-ahead launches too
      const tally_handle_state q = dev_->query(a.h);
      if (q.is_ptb && !q.done && !q.preempted) dev_->signal_preempt(a.h);
    }
  }
}

void Runner::submit_be(int task, const Work& w) {
  Task& st = tasks[(size_t)task];
  if (!st.has_cfg) {
    if (!w.has_config) throw Error(TALLY_EINVAL, "no tuner configuration for best-effort kernel " + w.kernel_id);
    st.cfg = w.config;
    st.has_cfg = true;
    if (st.cfg.variant == TALLY_SHAPE_SLICED) {
      st.tiling = slice_extents(w.cost.total_blocks, st.cfg.frac_num, st.cfg.frac_den);
      st.slice_i = 0;
    }
  }
  long long h;
  bool is_slice = false;
  if (st.cfg.variant == TALLY_SHAPE_PTB) {
    h = submit(task, w, TALLY_BEST_EFFORT, TALLY_SHAPE_PTB, st.cfg.worker_count, st.ptb_counter,
               w.cost.total_blocks, 0, false);
  } else if (st.cfg.variant == TALLY_SHAPE_SLICED) {
    long long off = 0;
    for (int i = 0; i < st.slice_i; ++i) off += st.tiling[(size_t)i];
    h = submit(task, w, TALLY_BEST_EFFORT, TALLY_SHAPE_ORIGINAL, 0, 0, st.tiling[(size_t)st.slice_i], off, true);
    is_slice = true;
  } else {
    h = submit(task, w, TALLY_BEST_EFFORT, TALLY_SHAPE_ORIGINAL, 0, 0, w.cost.total_blocks, 0, false);
  }
  tasks[(size_t)task].h = h;
  tasks[(size_t)task].h_is_slice = is_slice;
}

bool Runner::filter(long long h) {
  auto it = hinfo_.find(h);
  if (it == hinfo_.end()) return true;
  if (policy == TALLY_POLICY_KERNEL_PRIORITY) {
    // kernel-granularity priority: HP waits for in-flight BE kernels (ref scheduler.py:401-409)
    if (it->second.priority != TALLY_HIGH) return true;
    for (int i : be_) {
      const long long bh = tasks[(size_t)i].h;
      if (bh >= 0 && !done(bh)) return false;
      for (const auto& a : tasks[(size_t)i].ahead)
        if (!done(a.h)) return false;
    }
    return true;
  }
  if (policy == TALLY_POLICY_TIME_SLICED) return it->second.task == ts_active_;
  return true;
}

bool Runner::ts_has_work(const Task& st) {
  return st.h >= 0 || st.has_queued_work() || (!st.inference() && dev_->now() < horizon);
}

void Runner::ts_arm() {
  if (ts_armed_) return;
  ts_armed_ = true;
  const long long t = dev_->now() + quantum;
  dev_->call_at(t, token(2, -1, t));
}

void Runner::ts_rotate() {
  ts_armed_ = false;
  std::vector<int> busy;
  for (size_t i = 0; i < tasks.size(); ++i)
    if (ts_has_work(tasks[i])) busy.push_back((int)i);
  if (busy.empty()) return;
  int next = busy[0];
  for (int i : busy)
    if (i > ts_active_) { next = i; break; }
  ts_active_ = next;
  dev_->kick();
  tick();
  ts_arm();
}

// ----------------------------------------------------------------- vtbl device
struct VtblDevice : Device {
  tally_device_vtbl v;
  explicit VtblDevice(const tally_device_vtbl& x) : v(x) {}
  static void chk(int rc, const char* what) {
    if (rc < 0) throw Error(rc, std::string("device ") + what + " failed");
  }
  long long now() override { return v.now(v.ctx); }
  long long submit(const tally_submit_desc& d) override {
    long long h = v.submit(v.ctx, &d);
    if (h < 0) throw Error((int)h, "device submit failed");
    return h;
  }
  void signal_preempt(long long h) override { chk(v.signal_preempt(v.ctx, h), "signal_preempt"); }
  tally_handle_state query(long long h) override {
    tally_handle_state s;
    memset(&s, 0, sizeof(s));
    chk(v.query(v.ctx, h, &s), "query");
    return s;
  }
  void call_at(long long t, long long tok) override { chk(v.call_at(v.ctx, t, tok), "call_at"); }
  void set_dispatch_filter(bool e) override { chk(v.set_dispatch_filter(v.ctx, e ? 1 : 0), "set_dispatch_filter"); }
  void kick() override { chk(v.kick(v.ctx), "kick"); }
  void run_to_completion() override { chk(v.run_to_completion(v.ctx), "run_to_completion"); }
};

}  // namespace tally

using namespace tally;

namespace {
std::vector<std::unique_ptr<Runner>>& runners() {
  static std::vector<std::unique_ptr<Runner>> r;
  return r;
}
Runner* get_runner(int id) {
  auto& rs = runners();
  if (id < 0 || id >= (int)rs.size() || !rs[(size_t)id]) {
    set_error("unknown runner %d", id);
    return nullptr;
  }
  return rs[(size_t)id].get();
}
template <class F>
int guarded(F&& f) {
  try {
    f();
    return TALLY_OK;
  } catch (const Error& e) {
    set_error("%s", e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_error("%s", e.what());
    return TALLY_EINVAL;
  }
}
}  // namespace

extern "C" {

int tally_runner_create(int policy, long long threshold_ns, long long quantum_ns, long long horizon_ns,
                        int* out) {
  return guarded([&] {
    auto r = std::make_unique<Runner>(policy, threshold_ns, quantum_ns, horizon_ns);
    runners().push_back(std::move(r));
    *out = (int)runners().size() - 1;
  });
}

int tally_runner_add_task(int runner, const char* task_id, int priority, const tally_work* works, int n_works,
                          const long long* arrivals, int n_arrivals) {
  Runner* r = get_runner(runner);
  if (!r) return TALLY_EINVAL;
  return guarded([&] {
    if (!task_id) throw Error(TALLY_EINVAL, "null task id");
    if (priority != TALLY_HIGH && priority != TALLY_BEST_EFFORT) throw Error(TALLY_EINVAL, "unknown priority");
    Task t;
    t.id = task_id;
    t.priority = priority;
    for (int i = 0; i < n_works; ++i) {
      Work w;
      w.kernel_id = works[i].kernel_id ? works[i].kernel_id : "";
      w.cost = works[i].cost;
      w.exempt = works[i].exempt != 0;
      w.device_kernel = works[i].device_kernel;
      w.has_config = works[i].has_config != 0;
      w.config = works[i].config;
      w.est_ns = works[i].est_ns;
      if (w.cost.total_blocks < 1 || w.cost.threads_per_block < 1)
        throw Error(TALLY_EINVAL, "block counts must be >= 1");
      t.kernels.push_back(std::move(w));
    }
    for (int i = 0; i < n_arrivals; ++i) t.arrivals.push_back(arrivals[i]);
    r->add_task(std::move(t));
  });
}

int tally_runner_run(int runner, const tally_device_vtbl* dev) {
  Runner* r = get_runner(runner);
  if (!r) return TALLY_EINVAL;
  return guarded([&] {
    if (dev) {
      VtblDevice d(*dev);
      r->run(&d);
    } else {
      std::unique_ptr<Device> d(make_cuda_device(r));
      r->run(d.get());
    }
  });
}

int tally_runner_fire(int runner, long long token) {
  Runner* r = get_runner(runner);
  if (!r) return TALLY_EINVAL;
  return guarded([&] { r->fire(token); });
}

int tally_runner_on_event(int runner, int kind, long long handle) {
  Runner* r = get_runner(runner);
  if (!r) return TALLY_EINVAL;
  return guarded([&] { r->on_event(kind, handle); });
}

int tally_runner_filter(int runner, long long handle) {
  Runner* r = get_runner(runner);
  if (!r) return TALLY_EINVAL;
  int out = 1;
  int rc = guarded([&] { out = r->filter(handle) ? 1 : 0; });
  return rc < 0 ? rc : out;
}

int tally_runner_request_count(int runner, int task) {
  Runner* r = get_runner(runner);
  if (!r || task < 0 || task >= (int)r->tasks.size()) return TALLY_EINVAL;
  return (int)r->tasks[(size_t)task].requests.size();
}

int tally_runner_requests(int runner, int task, long long* out, int cap) {
  Runner* r = get_runner(runner);
  if (!r || task < 0 || task >= (int)r->tasks.size()) return TALLY_EINVAL;
  const auto& q = r->tasks[(size_t)task].requests;
  int n = std::min(cap, (int)q.size());
  for (int i = 0; i < n; ++i) {
    out[2 * i] = q[(size_t)i].first;
    out[2 * i + 1] = q[(size_t)i].second;
  }
  return n;
}

int tally_runner_iteration_count(int runner, int task) {
  Runner* r = get_runner(runner);
  if (!r || task < 0 || task >= (int)r->tasks.size()) return TALLY_EINVAL;
  return (int)r->tasks[(size_t)task].iterations.size();
}

int tally_runner_iterations(int runner, int task, long long* out, int cap) {
  Runner* r = get_runner(runner);
  if (!r || task < 0 || task >= (int)r->tasks.size()) return TALLY_EINVAL;
  const auto& q = r->tasks[(size_t)task].iterations;
  int n = std::min(cap, (int)q.size());
  for (int i = 0; i < n; ++i) out[i] = q[(size_t)i];
  return n;
}

int tally_runner_set_option(int runner, const char* key, long long value) {
  Runner* r = get_runner(runner);
  if (!r) return TALLY_EINVAL;
  if (!key) { set_error("null option key"); return TALLY_EINVAL; }
  const std::string k(key);
  if (k != "trace" && k != "hp_streams" && k != "suspend" && k != "lookahead") {
    set_error("unknown runner option '%s'", key);
    return TALLY_EINVAL;
  }
  if (k == "lookahead" && (value < 1 || value > 64)) { set_error("lookahead must be in [1, 64]"); return TALLY_EINVAL; }
  if (k == "hp_streams" && (value < 1 || value > 64)) { set_error("hp_streams must be in [1, 64]"); return TALLY_EINVAL; }
  r->options[k] = value;
  return TALLY_OK;
}

int tally_runner_destroy(int runner) {
  if (!get_runner(runner)) return TALLY_EINVAL;
  runners()[(size_t)runner].reset();
  return TALLY_OK;
}

int tally_device_event_count(int runner) {
  Runner* r = get_runner(runner);
  return r ? (int)r->log.events.size() : TALLY_EINVAL;
}

int tally_device_events(int runner, tally_event* out, int cap) {
  Runner* r = get_runner(runner);
  if (!r) return TALLY_EINVAL;
  int n = std::min(cap, (int)r->log.events.size());
  std::copy(r->log.events.begin(), r->log.events.begin() + n, out);
  return n;
}

long long tally_device_run_origin_ns(int runner) {
  Runner* r = get_runner(runner);
  return r ? r->log.t0_ns : TALLY_EINVAL;
}

int tally_device_launch_count(int runner) {
  Runner* r = get_runner(runner);
  return r ? (int)r->log.launches.size() : TALLY_EINVAL;
}

int tally_device_launches(int runner, tally_launch_record* out, int cap) {
  Runner* r = get_runner(runner);
  if (!r) return TALLY_EINVAL;
  int n = std::min(cap, (int)r->log.launches.size());
  std::copy(r->log.launches.begin(), r->log.launches.begin() + n, out);
  return n;
}

}  // extern "C"
