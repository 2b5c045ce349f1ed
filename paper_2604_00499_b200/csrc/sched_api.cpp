// tie::WaitingQueue and tie::Scheduler (include/tiesched_b200.hpp): the reference's C++
// scheduler API (proj/include/tiesched/sched.hpp:43-90, proj/src/sched.cpp:28-175) over the
// GPU-resident queue of queue.cu (tie_queue_*).  Same signatures, semantics and exception
// types; the per-item calls are device round trips of one, the *_batch calls move a whole
// batch per round trip.
#include <algorithm>
#include <stdexcept>
#include <string>

#include "tiesched_b200.hpp"

namespace tie {

namespace {

void throw_code(int rc) {
  if (rc == TIE_OK) return;
  const std::string msg = tie_last_error();
  if (rc == TIE_EDOMAIN) throw std::domain_error(msg);
  if (rc == TIE_EINVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

tie_queue* make_queue(const McContext* mc, int policy, const ScoreConfig& cfg, size_t cap) {
  tie_ctx* ctx = mc ? mc->handle() : default_context();
  tie_queue* q = nullptr;
  throw_code(tie_queue_create(ctx, policy, cfg.beta_mode == BetaMode::AdaptiveLinear,
                              cfg.beta_fixed, cfg.beta_max, cfg.q_sat, cfg.rebuild_threshold,
                              cfg.alpha, std::max<size_t>(cap, 1), &q));
  return q;
}

}  // namespace

// ------------------------------------------------------------------------ WaitingQueue

WaitingQueue::WaitingQueue(const McContext* mc, size_t initial_capacity)
    : q_(make_queue(mc, TIE_QUEUE_RAW, ScoreConfig{}, initial_capacity)), owner_(true) {}

WaitingQueue::WaitingQueue(tie_queue* view_of) : q_(view_of), owner_(false) {}

WaitingQueue::~WaitingQueue() {
  if (owner_) tie_queue_destroy(q_);
}

WaitingQueue::WaitingQueue(WaitingQueue&& o) noexcept { *this = std::move(o); }

WaitingQueue& WaitingQueue::operator=(WaitingQueue&& o) noexcept {
  if (this != &o) {
    if (owner_) tie_queue_destroy(q_);
    q_ = o.q_;
    owner_ = o.owner_;
    cache_ = std::move(o.cache_);
    cache_pos_ = std::move(o.cache_pos_);
    all_out_ = o.all_out_;
    dirty_ = std::move(o.dirty_);
    o.q_ = nullptr;
    o.owner_ = false;
  }
  return *this;
}

// handed-out edits (entries() / non-const at()) reach the device; the cache is dropped
void WaitingQueue::flush() const {
  std::vector<const QueueEntry*> out;
  if (all_out_) {
    for (const QueueEntry& e : cache_) out.push_back(&e);
  } else {
    for (uint64_t id : dirty_)
      if (auto it = cache_pos_.find(id); it != cache_pos_.end()) out.push_back(&cache_[it->second]);
  }
  if (!out.empty()) {
    const size_t m = out.size();
    std::vector<uint64_t> ids(m);
    std::vector<double> keys(m), E(m), C(m), B(m);
    std::vector<uint8_t> P(m);
    for (size_t j = 0; j < m; ++j) {
      ids[j] = out[j]->req_id;
      keys[j] = out[j]->key;
      P[j] = out[j]->predicted ? 1 : 0;
      E[j] = out[j]->expectation;
      C[j] = out[j]->cvar;
      B[j] = out[j]->beta_at_update;
    }
    throw_code(tie_queue_set_entries(q_, ids.data(), keys.data(), P.data(), E.data(), C.data(),
                                     B.data(), m));
  }
  cache_.clear();
  cache_pos_.clear();
  all_out_ = false;
  dirty_.clear();
}

void WaitingQueue::push(const QueueEntry& e) { push_batch(&e, 1); }

void WaitingQueue::push_batch(const QueueEntry* e, size_t m) {
  flush();
  std::vector<uint64_t> ids(m);
  std::vector<double> keys(m), E(m), C(m), B(m);
  std::vector<uint8_t> P(m);
  for (size_t j = 0; j < m; ++j) {
    ids[j] = e[j].req_id;
    keys[j] = e[j].key;
    P[j] = e[j].predicted ? 1 : 0;
    E[j] = e[j].expectation;
    C[j] = e[j].cvar;
    B[j] = e[j].beta_at_update;
  }
  throw_code(tie_queue_push(q_, ids.data(), keys.data(), P.data(), E.data(), C.data(), B.data(),
                            m));
}

void WaitingQueue::update(uint64_t req_id, double key) { update_batch(&req_id, &key, 1); }

void WaitingQueue::update_batch(const uint64_t* ids, const double* keys, size_t m) {
  // the Scheduler idiom: at(id) edits, then update(id, key) (sched.cpp:141-149)
  flush();
  throw_code(tie_queue_update(q_, ids, keys, m));
}

std::optional<QueueEntry> WaitingQueue::pop_min() {
  std::vector<QueueEntry> v = pop_batch(1);
  if (v.empty()) return std::nullopt;
  return v[0];
}

std::vector<QueueEntry> WaitingQueue::pop_batch(size_t max_pops) {
  flush();
  const size_t k = std::min(max_pops, size());
  std::vector<uint64_t> ids(k);
  std::vector<double> keys(k), E(k), C(k), B(k);
  std::vector<uint8_t> P(k);
  uint64_t n = 0;
  throw_code(tie_queue_pop(q_, k, ids.data(), keys.data(), P.data(), E.data(), C.data(),
                           B.data(), &n));
  std::vector<QueueEntry> out(n);
  for (size_t j = 0; j < n; ++j)
    out[j] = QueueEntry{ids[j], keys[j], P[j] != 0, E[j], C[j], B[j]};
  return out;
}

bool WaitingQueue::contains(uint64_t req_id) const { return tie_queue_contains(q_, req_id) != 0; }

size_t WaitingQueue::size() const { return tie_queue_size(q_); }

const std::vector<QueueEntry>& WaitingQueue::entries() const {
  if (cache_.size() == size() && (all_out_ || cache_pos_.size() == cache_.size()) &&
      !cache_.empty())
    return cache_;
  flush();
  const size_t n = size();
  std::vector<uint64_t> ids(n);
  std::vector<double> keys(n), E(n), C(n), B(n);
  std::vector<uint8_t> P(n);
  uint64_t got = 0;
  throw_code(tie_queue_entries(q_, n, ids.data(), keys.data(), P.data(), E.data(), C.data(),
                               B.data(), &got));
  cache_.resize(got);
  cache_pos_.clear();
  for (size_t j = 0; j < got; ++j) {
    cache_[j] = QueueEntry{ids[j], keys[j], P[j] != 0, E[j], C[j], B[j]};
    cache_pos_[ids[j]] = j;
  }
  return cache_;
}

std::vector<QueueEntry>& WaitingQueue::entries() {
  if (!owner_) throw std::logic_error("WaitingQueue: a Scheduler's queue is read-only");
  const std::vector<QueueEntry>& c = static_cast<const WaitingQueue*>(this)->entries();
  all_out_ = true;
  return const_cast<std::vector<QueueEntry>&>(c);
}

const QueueEntry& WaitingQueue::at(uint64_t req_id) const {
  if (auto it = cache_pos_.find(req_id); it != cache_pos_.end()) return cache_[it->second];
  uint64_t id = req_id;
  double key = 0, E = 0, C = 0, B = 0;
  uint8_t P = 0;
  throw_code(tie_queue_get(q_, &id, 1, &key, &P, &E, &C, &B));
  // references stay valid until the next mutation, as the reference heap's do: the cache
  // never reallocates (at most size() distinct waiting ids fit)
  if (cache_.empty()) cache_.reserve(size());
  cache_.push_back(QueueEntry{req_id, key, P != 0, E, C, B});
  cache_pos_[req_id] = cache_.size() - 1;
  return cache_.back();
}

QueueEntry& WaitingQueue::at(uint64_t req_id) {
  if (!owner_) throw std::logic_error("WaitingQueue: a Scheduler's queue is read-only");
  const QueueEntry& e = static_cast<const WaitingQueue*>(this)->at(req_id);
  dirty_.push_back(req_id);
  return const_cast<QueueEntry&>(e);
}

void WaitingQueue::rebuild() { flush(); }  // the block-min index is rebuilt on write-back

bool WaitingQueue::validate() const {
  flush();
  int ok = 0;
  throw_code(tie_queue_validate(q_, &ok));
  return ok != 0;
}

// ------------------------------------------------------------------------ Scheduler

Scheduler::Scheduler(Policy policy, ScoreConfig cfg, const McContext* mc, size_t initial_capacity)
    : policy_(policy),
      cfg_(cfg),
      q_(make_queue(mc, (int)policy, cfg, initial_capacity)),
      view_(q_) {}

Scheduler::~Scheduler() {
  view_.q_ = nullptr;
  tie_queue_destroy(q_);
}

Scheduler::Scheduler(Scheduler&& o) noexcept
    : policy_(o.policy_), cfg_(o.cfg_), q_(o.q_), view_(o.q_) {
  o.q_ = nullptr;
  o.view_.q_ = nullptr;
}

Scheduler& Scheduler::operator=(Scheduler&& o) noexcept {
  if (this != &o) {
    tie_queue_destroy(q_);
    policy_ = o.policy_;
    cfg_ = o.cfg_;
    q_ = o.q_;
    view_.q_ = o.q_;
    view_.cache_.clear();  // a read-only view holds no edits
    view_.cache_pos_.clear();
    o.q_ = nullptr;
    o.view_.q_ = nullptr;
  }
  return *this;
}

void Scheduler::on_arrival(const Request& req) { on_arrival_batch(&req, 1); }

void Scheduler::on_arrival_batch(const Request* reqs, size_t m) {
  view_.flush();
  std::vector<uint64_t> ids(m);
  std::vector<double> arr(m);
  std::vector<uint32_t> mt(m);
  for (size_t j = 0; j < m; ++j) {
    ids[j] = reqs[j].id;
    arr[j] = reqs[j].arrival_s;
    mt[j] = reqs[j].max_tokens;
  }
  throw_code(tie_queue_arrive(q_, ids.data(), arr.data(), mt.data(), m));
}

void Scheduler::on_prediction(uint64_t req_id, double expectation, double cvar) {
  on_prediction_batch(&req_id, &expectation, &cvar, 1);
}

void Scheduler::on_prediction_batch(const uint64_t* ids, const double* expectation,
                                    const double* cvar, size_t m) {
  view_.flush();
  throw_code(tie_queue_predict(q_, ids, expectation, cvar, m));
}

bool Scheduler::rebuild_if_drifted() {
  view_.flush();
  int r = 0;
  throw_code(tie_queue_rebuild_if_drifted(q_, &r));
  return r != 0;
}

std::optional<uint64_t> Scheduler::next_request() {
  std::vector<uint64_t> v = next_requests(1);
  if (v.empty()) return std::nullopt;
  return v[0];
}

std::vector<uint64_t> Scheduler::next_requests(size_t k) {
  view_.flush();
  std::vector<uint64_t> out(std::min(k, waiting()));
  uint64_t n = 0;
  throw_code(tie_queue_next(q_, out.size(), out.data(), &n));
  out.resize(n);
  return out;
}

std::vector<uint64_t> Scheduler::step(const Request* arrivals, size_t n_arr,
                                      const uint64_t* pred_ids, const double* expectation,
                                      const double* cvar, size_t n_pred, size_t max_pops) {
  view_.flush();
  std::vector<uint64_t> ids(n_arr);
  std::vector<double> arr(n_arr);
  std::vector<uint32_t> mt(n_arr);
  for (size_t j = 0; j < n_arr; ++j) {
    ids[j] = arrivals[j].id;
    arr[j] = arrivals[j].arrival_s;
    mt[j] = arrivals[j].max_tokens;
  }
  std::vector<uint64_t> out(max_pops);
  uint64_t n = 0;
  throw_code(tie_queue_step_ec(q_, ids.data(), arr.data(), mt.data(), n_arr, pred_ids,
                               expectation, cvar, n_pred, max_pops, out.data(), &n));
  out.resize(n);
  return out;
}

std::vector<uint64_t> Scheduler::step_runs(const Request* arrivals, const uint64_t* arr_end,
                                           const uint64_t* pred_ids, const double* expectation,
                                           const double* cvar, const uint64_t* pred_end,
                                           size_t n_runs, size_t max_pops) {
  view_.flush();
  const size_t n_arr = n_runs ? arr_end[n_runs - 1] : 0;
  std::vector<uint64_t> ids(n_arr);
  std::vector<double> arr(n_arr);
  std::vector<uint32_t> mt(n_arr);
  for (size_t j = 0; j < n_arr; ++j) {
    ids[j] = arrivals[j].id;
    arr[j] = arrivals[j].arrival_s;
    mt[j] = arrivals[j].max_tokens;
  }
  std::vector<uint64_t> out(max_pops);
  uint64_t n = 0;
  throw_code(tie_queue_step_ec_runs(q_, ids.data(), arr.data(), mt.data(), arr_end, pred_ids,
                                    expectation, cvar, pred_end, n_runs, max_pops, out.data(),
                                    &n));
  out.resize(n);
  return out;
}

bool Scheduler::waiting_on(uint64_t req_id) const { return tie_queue_contains(q_, req_id) != 0; }

size_t Scheduler::waiting() const { return tie_queue_size(q_); }

}  // namespace tie
