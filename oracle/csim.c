/* C restatement of the reference discrete-event GPU (ref sim.py:229-526).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the CPU reference arm of
 * bench.py and the oracle's own tests.  It restates oracle/gpu_model.py --
 * itself pinned to the reference's event logs (tests/golden/sim.json,
 * policy.json) -- statement for statement, so that a B200-scale scenario
 * (~1.4 M logical blocks per BERT-large training step) simulates in seconds
 * instead of the ~30 s per step the Python event loop needs.  oracle/csim.py
 * wraps it with the GpuSim surface; tests/test_oracle_csim.py requires the
 * wrapped simulator to reproduce the golden event-log SHA-256s.
 *
 * Semantics (each restated from the reference):
 *   integer-ns clock, heap keyed by (time, tie)                  sim.py:254-262, :278-296
 *   event counter advances even when events are not recorded    sim.py:264-276
 *   occupancy_limit = min(max_blocks, max_threads / tpb)         sim.py:55-74
 *   submit -> LaunchIssued -> ready after the launch overhead    sim.py:304-327
 *   dispatch: HP queue first; BE blocked while an HP launch that
 *     passes the dispatch filter has unplaced blocks; first-fit
 *     SM in the seeded order, capacity = min of resident limits  sim.py:355-432
 *   Original / Sliced block lifecycle (slices one at a time)     sim.py:436-471
 *   PTB workers: claim -> block + iteration overhead -> claim;
 *     park on preempt when work remains                          sim.py:475-505
 *   preempt signal / park                                        sim.py:329-351
 * Host callbacks (call_at closures, the observer, the dispatch filter) are
 * C function pointers the Python wrapper supplies; a callback that raised
 * sets `abort`, and the run loop returns -1 at the next event boundary.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef long long i64;

enum { EV_LAUNCH_ISSUED, EV_BLOCK_STARTED, EV_BLOCK_FINISHED, EV_KERNEL_FINISHED, EV_PREEMPT_SIGNALED,
       EV_WORKER_PARKED };
enum { SH_ORIGINAL, SH_SLICED, SH_PTB };
enum { Q_ISSUE, Q_READY, Q_PREEMPT, Q_BLOCK_END, Q_WORKER_STEP, Q_CALLBACK };

/* Handle layout is mirrored by a ctypes Structure in oracle/csim.py. */
typedef struct {
  i64 uid;
  i64 priority; /* 0 = High, 1 = BestEffort */
  i64 shape;
  i64 block_ns, launch_ns, iter_ns, tpb, total;
  i64 worker_count, start_count;
  i64 ready, done, preempted, parked;
  i64 finish_time, preempt_time; /* -1 = None */
  i64 blocks_finished, next_block, current_sub, sub_placed, sub_finished;
  i64 task_counter, workers_placed, workers_active;
  i64 submit_time;
  i64 n_sub, n_sub_completions, n_park_times;
  /* private */
  i64 *sub_blocks, *sub_suffix, *sub_completions, *park_times;
  i64 cap_subc, cap_park;
} Handle;

typedef struct {
  i64 time, seq, kind, uid, block;
} Event;

typedef struct {
  i64 t, tie;
  i64 h, limit, b;
  int type, sm, flag, pad;
} QItem;

typedef struct {
  i64* a;
  i64 n, cap;
} Vec;

typedef void (*obs_fn)(i64 kind, i64 uid, i64 block, i64 seq);
typedef int (*filter_fn)(i64 uid);
typedef void (*cb_fn)(i64 token);

typedef struct {
  int num_sms, max_threads, max_blocks;
  i64 now, tie, nlogged;
  int record;
  int abort;
  Event* ev;
  i64 nev, capev;
  QItem* q;
  i64 nq, capq;
  Handle** chunks;
  i64 nh, nchunks;
  Vec hp, be;
  int *resident, *order, *pos, *cap, *limcnt;
  uint64_t* open;
  int nwords;
  obs_fn obs;
  uint32_t obs_mask;
  filter_fn filt;
  cb_fn cb;
} Sim;

#define CHUNK 4096

static void* xrealloc(void* p, size_t n) {
  void* r = realloc(p, n);
  if (!r) abort();
  return r;
}

static void vec_push(Vec* v, i64 x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? 2 * v->cap : 64;
    v->a = (i64*)xrealloc(v->a, (size_t)v->cap * sizeof(i64));
  }
  v->a[v->n++] = x;
}

static Handle* H(Sim* s, i64 uid) { return &s->chunks[uid / CHUNK][uid % CHUNK]; }

/* ---------------------------------------------------------------- heap */
static int q_less(const QItem* a, const QItem* b) { return a->t != b->t ? a->t < b->t : a->tie < b->tie; }

static void q_push(Sim* s, QItem it) {
  if (s->nq == s->capq) {
    s->capq = s->capq ? 2 * s->capq : 1024;
    s->q = (QItem*)xrealloc(s->q, (size_t)s->capq * sizeof(QItem));
  }
  i64 i = s->nq++;
  while (i > 0) {
    i64 p = (i - 1) / 2;
    if (!q_less(&it, &s->q[p])) break;
    s->q[i] = s->q[p];
    i = p;
  }
  s->q[i] = it;
}

static QItem q_pop(Sim* s) {
  QItem top = s->q[0];
  QItem last = s->q[--s->nq];
  i64 i = 0, n = s->nq;
  for (;;) {
    i64 c = 2 * i + 1;
    if (c >= n) break;
    if (c + 1 < n && q_less(&s->q[c + 1], &s->q[c])) ++c;
    if (!q_less(&s->q[c], &last)) break;
    s->q[i] = s->q[c];
    i = c;
  }
  if (n > 0) s->q[i] = last;
  return top;
}

static void at(Sim* s, i64 t, int type, i64 h, int sm, i64 limit, i64 b, int flag) {
  QItem it;
  it.t = t;
  it.tie = s->tie++;
  it.type = type;
  it.h = h;
  it.sm = sm;
  it.limit = limit;
  it.b = b;
  it.flag = flag;
  it.pad = 0;
  q_push(s, it);
}

/* ---------------------------------------------------------------- events */
static void emit(Sim* s, int kind, Handle* h, i64 block) {
  const i64 seq = s->nlogged++;
  if (s->record) {
    if (s->nev == s->capev) {
      s->capev = s->capev ? 2 * s->capev : 4096;
      s->ev = (Event*)xrealloc(s->ev, (size_t)s->capev * sizeof(Event));
    }
    Event* e = &s->ev[s->nev++];
    e->time = s->now;
    e->seq = seq;
    e->kind = kind;
    e->uid = h->uid;
    e->block = block;
  }
  if (s->obs && ((s->obs_mask >> kind) & 1u)) s->obs(kind, h->uid, block, seq);
}

/* ---------------------------------------------------------------- placement */
static int occupancy(const Sim* s, i64 tpb) {
  i64 t = s->max_threads / tpb;
  return (int)(t < s->max_blocks ? t : s->max_blocks);
}

static void set_open(Sim* s, int sm) {
  const int p = s->pos[sm];
  const uint64_t bit = 1ull << (p & 63);
  if (s->cap[sm] == 0 || s->resident[sm] < s->cap[sm]) s->open[p >> 6] |= bit;
  else s->open[p >> 6] &= ~bit;
}

/* first SM in the seeded order with resident < min(limit, cap) (sim.py:355-360) */
static int free_sm(Sim* s, int limit) {
  for (int w = 0; w < s->nwords; ++w) {
    uint64_t m = s->open[w];
    while (m) {
      const int b = __builtin_ctzll(m);
      const int sm = s->order[w * 64 + b];
      if (s->resident[sm] < limit) return sm;
      m &= m - 1;
    }
  }
  return -1;
}

static void take(Sim* s, int sm, int limit) {
  s->resident[sm] += 1;
  s->limcnt[sm * (s->max_blocks + 1) + limit] += 1;
  if (s->cap[sm] == 0 || limit < s->cap[sm]) s->cap[sm] = limit;
  set_open(s, sm);
}

static void give(Sim* s, int sm, int limit) {
  s->resident[sm] -= 1;
  int* cnt = &s->limcnt[sm * (s->max_blocks + 1)];
  cnt[limit] -= 1;
  if (s->resident[sm] == 0) {
    s->cap[sm] = 0;
  } else if (limit == s->cap[sm] && cnt[limit] == 0) {
    int c = limit + 1;
    while (c <= s->max_blocks && cnt[c] == 0) ++c;
    s->cap[sm] = c;
  }
  set_open(s, sm);
}

/* ---------------------------------------------------------------- lifecycle */
static void dispatch(Sim* s);

static void issue(Sim* s, Handle* h, i64 block) {
  emit(s, EV_LAUNCH_ISSUED, h, block);
  at(s, s->now + h->launch_ns, Q_READY, h->uid, 0, 0, 0, 0);
}

static void park(Sim* s, Handle* h) {
  h->parked = 1;
  if (h->n_park_times == 0) {
    if (h->cap_park == 0) {
      h->cap_park = 4;
      h->park_times = (i64*)xrealloc(h->park_times, 4 * sizeof(i64));
    }
    h->park_times[h->n_park_times++] = s->now;
  }
}

static void push_park(Handle* h, i64 t) {
  if (h->n_park_times == h->cap_park) {
    h->cap_park = h->cap_park ? 2 * h->cap_park : 4;
    h->park_times = (i64*)xrealloc(h->park_times, (size_t)h->cap_park * sizeof(i64));
  }
  h->park_times[h->n_park_times++] = t;
}

static void finished(Sim* s, Handle* h) {
  h->done = 1;
  h->finish_time = s->now;
  emit(s, EV_KERNEL_FINISHED, h, -1);
}

static void preempt(Sim* s, Handle* h) {
  if (h->done || h->preempted) return;
  h->preempted = 1;
  h->preempt_time = s->now;
  emit(s, EV_PREEMPT_SIGNALED, h, -1);
  if (h->workers_active == 0) park(s, h);
  dispatch(s);
}

static void worker_exit(Sim* s, Handle* h, int sm, int limit) {
  give(s, sm, limit);
  h->workers_active -= 1;
  if (h->preempted && h->task_counter < h->total) {
    push_park(h, s->now);
    emit(s, EV_WORKER_PARKED, h, -1);
    if (h->workers_active == 0) h->parked = 1;
  } else if (h->workers_active == 0 && !h->done) {
    finished(s, h);
  }
  dispatch(s);
}

static void claim(Sim* s, Handle* h, int sm, int limit) {
  if (h->preempted || h->task_counter >= h->total) {
    worker_exit(s, h, sm, limit);
    return;
  }
  const i64 task = h->task_counter++;
  emit(s, EV_BLOCK_STARTED, h, task);
  at(s, s->now + h->block_ns + h->iter_ns, Q_WORKER_STEP, h->uid, sm, limit, task, 0);
}

static void worker_step(Sim* s, Handle* h, int sm, int limit, i64 task) {
  h->blocks_finished += 1;
  emit(s, EV_BLOCK_FINISHED, h, task);
  claim(s, h, sm, limit);
}

static void start_block(Sim* s, Handle* h, int sm, int limit, i64 b, int sliced) {
  take(s, sm, limit);
  emit(s, EV_BLOCK_STARTED, h, b);
  at(s, s->now + h->block_ns, Q_BLOCK_END, h->uid, sm, limit, b, sliced);
}

static void block_end(Sim* s, Handle* h, int sm, int limit, i64 b, int sliced) {
  give(s, sm, limit);
  h->blocks_finished += 1;
  emit(s, EV_BLOCK_FINISHED, h, b);
  if (sliced) {
    h->sub_finished += 1;
    if (h->sub_finished == h->sub_blocks[h->current_sub]) {
      if (h->n_sub_completions == h->cap_subc) {
        h->cap_subc = h->cap_subc ? 2 * h->cap_subc : 4;
        h->sub_completions = (i64*)xrealloc(h->sub_completions, (size_t)h->cap_subc * sizeof(i64));
      }
      h->sub_completions[h->n_sub_completions++] = s->now;
      if (h->current_sub + 1 < h->n_sub) {
        h->current_sub += 1;
        h->sub_placed = h->sub_finished = 0;
        h->ready = 0;
        issue(s, h, h->current_sub);
      } else {
        finished(s, h);
      }
    }
  } else if (h->blocks_finished == h->total) {
    finished(s, h);
  }
  dispatch(s);
}

static i64 unplaced(const Handle* h) {
  if (h->done || h->parked) return 0;
  if (h->shape == SH_PTB) return h->preempted ? 0 : h->worker_count - h->workers_placed;
  if (h->shape == SH_SLICED) return h->sub_blocks[h->current_sub] - h->sub_placed + h->sub_suffix[h->current_sub + 1];
  return h->total - h->next_block;
}

static void place(Sim* s, Handle* h) {
  const int limit = occupancy(s, h->tpb);
  const i64 total = h->total;
  if (h->shape == SH_PTB) {
    while (!h->preempted && h->workers_placed < h->worker_count && h->task_counter < total) {
      const int sm = free_sm(s, limit);
      if (sm < 0) return;
      h->workers_placed += 1;
      h->workers_active += 1;
      take(s, sm, limit);
      claim(s, h, sm, limit);
    }
    if (h->workers_placed == 0) {
      if (h->preempted) park(s, h);
      else if (h->task_counter >= total) finished(s, h);
    }
    return;
  }
  if (h->shape == SH_SLICED) {
    while (h->sub_placed < h->sub_blocks[h->current_sub]) {
      const int sm = free_sm(s, limit);
      if (sm < 0) return;
      const i64 b = h->next_block++;
      h->sub_placed += 1;
      start_block(s, h, sm, limit, b, 1);
    }
    return;
  }
  while (h->next_block < total) {
    const int sm = free_sm(s, limit);
    if (sm < 0) return;
    const i64 b = h->next_block++;
    start_block(s, h, sm, limit, b, 0);
  }
}

static int hp_pressure(Sim* s) {
  for (i64 i = 0; i < s->hp.n; ++i) {
    Handle* h = H(s, s->hp.a[i]);
    if (h->done) continue;
    if (s->filt && !s->filt(h->uid)) continue;
    if (unplaced(h) > 0) return 1;
  }
  return 0;
}

static void prune(Sim* s, Vec* v) {
  i64 k = 0;
  for (i64 i = 0; i < v->n; ++i)
    if (!H(s, v->a[i])->done) v->a[k++] = v->a[i];
  v->n = k;
}

static void dispatch(Sim* s) {
  for (int pass = 0; pass < 2; ++pass) {
    Vec* v = pass == 0 ? &s->hp : &s->be;
    if (pass == 1 && hp_pressure(s)) return;
    for (i64 i = 0; i < v->n; ++i) {   /* re-reads n: launches submitted meanwhile are visited too */
      Handle* h = H(s, v->a[i]);
      if (h->done || !h->ready) continue;
      if (s->filt && !s->filt(h->uid)) continue;
      place(s, h);
    }
  }
  prune(s, &s->hp);
  prune(s, &s->be);
}

static void fire(Sim* s, const QItem* e) {
  if (e->type == Q_CALLBACK) {
    s->cb(e->b);
    return;
  }
  Handle* h = H(s, e->h);
  switch (e->type) {
    case Q_ISSUE: issue(s, h, e->b); break;
    case Q_READY: h->ready = 1; dispatch(s); break;
    case Q_PREEMPT: preempt(s, h); break;
    case Q_BLOCK_END: block_end(s, h, e->sm, (int)e->limit, e->b, e->flag); break;
    case Q_WORKER_STEP: worker_step(s, h, e->sm, (int)e->limit, e->b); break;
  }
}

/* ---------------------------------------------------------------- C ABI */
Sim* csim_new(int num_sms, int max_threads, int max_blocks, const int* order, int record) {
  Sim* s = (Sim*)calloc(1, sizeof(Sim));
  s->num_sms = num_sms;
  s->max_threads = max_threads;
  s->max_blocks = max_blocks;
  s->record = record;
  s->resident = (int*)calloc((size_t)num_sms, sizeof(int));
  s->order = (int*)calloc((size_t)num_sms, sizeof(int));
  s->pos = (int*)calloc((size_t)num_sms, sizeof(int));
  s->cap = (int*)calloc((size_t)num_sms, sizeof(int));
  s->limcnt = (int*)calloc((size_t)num_sms * (size_t)(max_blocks + 1), sizeof(int));
  s->nwords = (num_sms + 63) / 64;
  s->open = (uint64_t*)calloc((size_t)s->nwords, sizeof(uint64_t));
  for (int p = 0; p < num_sms; ++p) {
    s->order[p] = order[p];
    s->pos[order[p]] = p;
    s->open[p >> 6] |= 1ull << (p & 63);
  }
  return s;
}

void csim_free(Sim* s) {
  if (!s) return;
  for (i64 u = 0; u < s->nh; ++u) {
    Handle* h = H(s, u);
    free(h->sub_blocks);
    free(h->sub_suffix);
    free(h->sub_completions);
    free(h->park_times);
  }
  for (i64 c = 0; c < s->nchunks; ++c) free(s->chunks[c]);
  free(s->chunks);
  free(s->ev);
  free(s->q);
  free(s->hp.a);
  free(s->be.a);
  free(s->resident);
  free(s->order);
  free(s->pos);
  free(s->cap);
  free(s->limcnt);
  free(s->open);
  free(s);
}

void csim_set_callbacks(Sim* s, obs_fn obs, unsigned mask, filter_fn filt, cb_fn cb) {
  s->obs = obs;
  s->obs_mask = mask;
  s->filt = filt;
  s->cb = cb;
}

void csim_abort(Sim* s) { s->abort = 1; }
i64 csim_now(const Sim* s) { return s->now; }
i64 csim_nlogged(const Sim* s) { return s->nlogged; }
i64 csim_nevents(const Sim* s) { return s->nev; }
const Event* csim_events(const Sim* s) { return s->ev; }
i64 csim_pending(const Sim* s) { return s->nq; }

void csim_call_at(Sim* s, i64 t, i64 token) { at(s, t, Q_CALLBACK, -1, 0, 0, token, 0); }

/* shape: 0 original, 1 sliced (subs[n_sub]), 2 ptb (workers, start) */
i64 csim_submit(Sim* s, i64 at_t, i64 priority, i64 shape, i64 block_ns, i64 launch_ns, i64 iter_ns, i64 tpb,
                i64 total, i64 workers, i64 start, const i64* subs, i64 n_sub) {
  if (s->nh == s->nchunks * CHUNK) {
    s->chunks = (Handle**)xrealloc(s->chunks, (size_t)(s->nchunks + 1) * sizeof(Handle*));
    s->chunks[s->nchunks++] = (Handle*)calloc(CHUNK, sizeof(Handle));
  }
  const i64 uid = s->nh++;
  Handle* h = H(s, uid);
  memset(h, 0, sizeof(*h));
  h->uid = uid;
  h->priority = priority;
  h->shape = shape;
  h->block_ns = block_ns;
  h->launch_ns = launch_ns;
  h->iter_ns = iter_ns;
  h->tpb = tpb;
  h->total = total;
  h->worker_count = workers;
  h->start_count = start;
  h->finish_time = -1;
  h->preempt_time = -1;
  h->submit_time = at_t;
  h->task_counter = shape == SH_PTB ? start : 0;
  if (shape == SH_SLICED) {
    h->n_sub = n_sub;
    h->sub_blocks = (i64*)xrealloc(NULL, (size_t)n_sub * sizeof(i64));
    h->sub_suffix = (i64*)xrealloc(NULL, (size_t)(n_sub + 1) * sizeof(i64));
    memcpy(h->sub_blocks, subs, (size_t)n_sub * sizeof(i64));
    h->sub_suffix[n_sub] = 0;
    for (i64 i = n_sub - 1; i >= 0; --i) h->sub_suffix[i] = h->sub_suffix[i + 1] + subs[i];
  }
  vec_push(priority == 0 ? &s->hp : &s->be, uid);
  at(s, at_t, Q_ISSUE, uid, 0, 0, -1, 0);
  return uid;
}

Handle* csim_handle(Sim* s, i64 uid) { return uid >= 0 && uid < s->nh ? H(s, uid) : NULL; }
const i64* csim_sub_completions(Sim* s, i64 uid) { return H(s, uid)->sub_completions; }
const i64* csim_park_times(Sim* s, i64 uid) { return H(s, uid)->park_times; }

void csim_signal_preempt(Sim* s, i64 uid, i64 at_t) { at(s, at_t, Q_PREEMPT, uid, 0, 0, 0, 0); }
void csim_kick(Sim* s) { dispatch(s); }

/* bounded = 0: run to completion; else run events with t <= until, then now = until. */
int csim_run(Sim* s, i64 until, int bounded) {
  while (s->nq > 0 && !s->abort) {
    if (bounded && s->q[0].t > until) break;
    QItem e = q_pop(s);
    s->now = e.t;
    fire(s, &e);
  }
  if (s->abort) return -1;
  if (bounded) s->now = until;
  return 0;
}
