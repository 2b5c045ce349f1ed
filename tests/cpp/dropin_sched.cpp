// A reference-style C++ caller of the scheduler / distribution API, compiled against the
// B200 drop-in header (include/tiesched_b200.hpp) and linked to libtie_b200.so -- the proof
// that code written for proj/include/tiesched/{dist,sched,sim,workload}.hpp recompiles.
// The cases restate the reference's own unit tests (proj/tests/test_sched.cpp:33-292,
// test_dist.cpp / test_smoke.py invariants) with a minimal CHECK macro instead of doctest.
//
//   tests/test_cpp_dropin.py builds it (CPU: compile + link) and runs it (GPU).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <random>
#include <stdexcept>
#include <vector>

#include "tiesched_b200.hpp"

using namespace tie;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (c) {                                                          \
      ++g_pass;                                                       \
    } else {                                                          \
      ++g_fail;                                                       \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
    }                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, T) \
  do {                           \
    bool ok_ = false;            \
    try {                        \
      (void)(expr);              \
    } catch (const T&) {         \
      ok_ = true;                \
    } catch (...) {              \
    }                            \
    CHECK(ok_ && #expr);         \
  } while (0)

static bool approx(double a, double b, double eps = 1e-15) {
  return std::fabs(a - b) <= eps * std::max(std::fabs(a), std::fabs(b));
}

static Request arrival(uint64_t id, double t, uint32_t max_tokens = 2048) {
  Request r;
  r.id = id;
  r.arrival_s = t;
  r.prompt_tokens = 100;
  r.true_output_tokens = 10;
  r.max_tokens = max_tokens;
  return r;
}

static ScoreConfig fixed_beta(double b) {
  ScoreConfig cfg;
  cfg.beta_mode = BetaMode::Fixed;
  cfg.beta_fixed = b;
  return cfg;
}

static void beta_and_score() {  // test_sched.cpp:33-80
  ScoreConfig a;
  a.beta_max = 0.5;
  a.q_sat = 128.0;
  CHECK(compute_beta(fixed_beta(0.3), 5) == 0.3);
  CHECK(compute_beta(a, 0) == 0.0);
  CHECK(approx(compute_beta(a, 64), 0.25));
  CHECK(compute_beta(a, 1000000) == 0.5);
  ScoreConfig bad = a;
  bad.q_sat = 0.0;
  CHECK_THROWS_AS(compute_beta(bad, 1), std::domain_error);
  CHECK(approx(compute_score(100.0, 400.0, 0.3), 220.0));
  CHECK_THROWS_AS(compute_score(200.0, 100.0, 0.3), std::invalid_argument);
  CHECK_THROWS_AS(compute_score(0.0, 100.0, 0.3), std::domain_error);
}

static void waiting_queue_basics() {  // test_sched.cpp:82-122
  WaitingQueue q;
  CHECK(!q.pop_min().has_value());
  for (auto [id, key] : std::vector<std::pair<uint64_t, double>>{{1, 5.0}, {2, 3.0}, {3, 9.0}}) {
    QueueEntry e;
    e.req_id = id;
    e.key = key;
    q.push(e);
    CHECK(q.validate());
  }
  auto top = q.pop_min();
  CHECK(top.has_value() && top->key == 3.0 && top->req_id == 2);

  WaitingQueue h;  // heapsort property
  std::mt19937_64 rng(404);
  std::uniform_real_distribution<double> U(0.0, 1000.0);
  for (uint64_t id = 0; id < 100; ++id) {
    QueueEntry e;
    e.req_id = id;
    e.key = U(rng);
    h.push(e);
  }
  CHECK(h.validate());
  double prev = -1.0;
  int popped = 0;
  while (auto e = h.pop_min()) {
    CHECK(e->key >= prev);
    prev = e->key;
    ++popped;
  }
  CHECK(popped == 100);

  QueueEntry dup;
  dup.req_id = 50;
  dup.key = 1.0;
  q.push(dup);
  CHECK_THROWS_AS(q.push(dup), std::invalid_argument);
  CHECK_THROWS_AS(q.update(777, 1.0), std::invalid_argument);
  CHECK_THROWS_AS(q.at(777), std::invalid_argument);
  dup.req_id = 99;
  dup.key = INFINITY;
  CHECK_THROWS_AS(q.push(dup), std::domain_error);
}

static void waiting_queue_ties_and_rekey() {  // test_sched.cpp:124-159
  WaitingQueue q;
  for (uint64_t id : {7, 2, 9, 4, 0}) {
    QueueEntry e;
    e.req_id = id;
    e.key = 2048.0;
    q.push(e);
  }
  std::vector<uint64_t> order;
  while (auto e = q.pop_min()) order.push_back(e->req_id);
  CHECK((order == std::vector<uint64_t>{0, 2, 4, 7, 9}));

  WaitingQueue r;
  for (uint64_t id = 0; id < 10; ++id) {
    QueueEntry e;
    e.req_id = id;
    e.key = 1000.0 + (double)id;
    r.push(e);
  }
  r.update(7, 1.0);
  CHECK(r.validate());
  CHECK(r.at(7).key == 1.0);
  auto e = r.pop_min();
  CHECK(e.has_value() && e->req_id == 7);
  r.update(3, 5000.0);
  CHECK(r.validate());
  std::vector<uint64_t> rest;
  while (auto x = r.pop_min()) rest.push_back(x->req_id);
  CHECK(rest.back() == 3);
}

static void waiting_queue_random_mirror() {  // test_sched.cpp:161-200
  WaitingQueue q(nullptr, 16);  // small initial capacity: exercises growth and compaction
  std::map<std::pair<double, uint64_t>, bool> mirror;
  std::map<uint64_t, double> key_of;
  std::mt19937_64 rng(6060);
  std::uniform_real_distribution<double> U01(0.0, 1.0), K(0.0, 100.0);
  uint64_t next_id = 0;
  for (int op = 0; op < 4000; ++op) {
    const double dice = U01(rng);
    if (dice < 0.45 || q.empty()) {
      QueueEntry e;
      e.req_id = next_id++;
      e.key = K(rng);
      q.push(e);
      mirror[{e.key, e.req_id}] = true;
      key_of[e.req_id] = e.key;
    } else if (dice < 0.7) {
      const size_t pick = std::uniform_int_distribution<size_t>(0, q.size() - 1)(rng);
      const uint64_t id = q.entries()[pick].req_id;
      const double nk = K(rng);
      mirror.erase({key_of[id], id});
      q.update(id, nk);
      mirror[{nk, id}] = true;
      key_of[id] = nk;
    } else {
      auto e = q.pop_min();
      auto expect = mirror.begin();
      CHECK(e.has_value() && e->key == expect->first.first && e->req_id == expect->first.second);
      mirror.erase(expect);
      key_of.erase(e->req_id);
    }
    if (op % 50 == 0) CHECK(q.validate());
  }
  CHECK(q.size() == mirror.size());
}

static void waiting_queue_entry_edits() {  // entries()/at() edits + rebuild (sched.cpp:110-114)
  WaitingQueue q;
  for (uint64_t id = 0; id < 6; ++id) {
    QueueEntry e;
    e.req_id = id;
    e.key = 10.0 * (double)(id + 1);
    q.push(e);
  }
  for (QueueEntry& e : q.entries()) e.key = 100.0 - e.key;  // reverse the order
  q.rebuild();
  CHECK(q.validate());
  QueueEntry& a = q.at(2);
  a.predicted = true;
  a.expectation = 7.0;
  a.cvar = 9.0;
  a.beta_at_update = 0.25;
  q.update(2, 1.0);
  auto e = q.pop_min();
  CHECK(e.has_value() && e->req_id == 2 && e->key == 1.0 && e->predicted &&
        e->expectation == 7.0 && e->cvar == 9.0 && e->beta_at_update == 0.25);
  std::vector<uint64_t> rest;
  while (auto x = q.pop_min()) rest.push_back(x->req_id);
  CHECK((rest == std::vector<uint64_t>{5, 4, 3, 1, 0}));
}

static void scheduler_policies() {  // test_sched.cpp:202-244
  Scheduler fcfs(Policy::FCFS, fixed_beta(0.3));
  fcfs.on_arrival(arrival(5, 1.0));
  fcfs.on_arrival(arrival(3, 2.0));
  fcfs.on_prediction(5, 5000.0, 6000.0);
  CHECK(fcfs.next_request() == 5u);
  CHECK(fcfs.next_request() == 3u);
  CHECK(!fcfs.next_request().has_value());

  Scheduler sept(Policy::SEPT, fixed_beta(0.3));
  sept.on_arrival(arrival(1, 0.0));
  sept.on_arrival(arrival(2, 0.1));
  sept.on_prediction(1, 100.0, 2000.0);
  sept.on_prediction(2, 120.0, 130.0);
  CHECK(sept.next_request() == 1u);

  Scheduler tie(Policy::TIE, fixed_beta(0.3));
  tie.on_arrival(arrival(1, 0.0));
  tie.on_arrival(arrival(2, 0.1));
  tie.on_prediction(1, 100.0, 900.0);
  tie.on_prediction(2, 100.0, 200.0);
  CHECK(tie.next_request() == 2u);

  Scheduler mixed(Policy::TIE, fixed_beta(0.3));
  mixed.on_arrival(arrival(1, 0.0, 2048));
  mixed.on_prediction(1, 100.0, 500.0);
  mixed.on_arrival(arrival(2, 0.1, 2048));
  CHECK(mixed.queue().at(2).key == 2048.0);
  CHECK(mixed.next_request() == 1u);

  Scheduler plain(Policy::TIE, fixed_beta(0.3));
  plain.on_arrival(arrival(9, 0.0, 1024));
  plain.on_arrival(arrival(4, 0.1, 1024));
  CHECK(plain.next_request() == 4u);

  CHECK_THROWS_AS(tie.on_prediction(777, 10.0, 20.0), std::invalid_argument);
  Scheduler twice(Policy::TIE, fixed_beta(0.3));
  twice.on_arrival(arrival(1, 0.0));
  twice.on_prediction(1, 10.0, 20.0);
  CHECK_THROWS_AS(twice.on_prediction(1, 11.0, 21.0), std::invalid_argument);
}

static void scheduler_drift_rebuild() {  // test_sched.cpp:246-292
  ScoreConfig cfg;
  cfg.beta_mode = BetaMode::AdaptiveLinear;
  cfg.beta_max = 0.5;
  cfg.q_sat = 4.0;
  cfg.rebuild_threshold = 0.1;
  auto build = [&]() {
    Scheduler s(Policy::TIE, cfg);
    for (uint64_t id = 0; id < 4; ++id) s.on_arrival(arrival(id, 0.1 * (double)id));
    s.on_prediction(0, 5.0, 10.0);
    s.on_prediction(1, 100.0, 2000.0);
    s.on_prediction(2, 671.0, 671.0);
    return s;
  };
  Scheduler s = build();
  CHECK(s.next_request() == 0u);
  CHECK(approx(s.queue().at(1).key, 1100.0));
  CHECK(approx(s.queue().at(2).key, 1006.5));
  CHECK(s.rebuild_if_drifted());
  CHECK(s.queue().size() == 3);
  CHECK(s.queue().validate());
  CHECK(approx(s.queue().at(1).key, 850.0));
  CHECK(approx(s.queue().at(2).key, 922.625));
  CHECK(s.queue().at(3).key == 2048.0);
  CHECK(s.queue().at(1).beta_at_update == 0.375);
  CHECK(!s.rebuild_if_drifted());
  CHECK(s.next_request() == 1u);

  Scheduler auto_s = build();
  CHECK(auto_s.next_request() == 0u);
  CHECK(auto_s.next_request() == 1u);

  cfg.rebuild_threshold = 0.2;
  Scheduler stale = build();
  CHECK(stale.next_request() == 0u);
  CHECK(!stale.rebuild_if_drifted());
  CHECK(approx(stale.queue().at(1).key, 1100.0));
  CHECK(stale.next_request() == 2u);
}

static void scheduler_step_batching() {  // Scheduler::step == the per-event call sequence
  ScoreConfig cfg;
  cfg.q_sat = 1e9;  // beta moves with every queue-length change
  cfg.rebuild_threshold = 0.0;
  Scheduler a(Policy::TIE, cfg), b(Policy::TIE, cfg);
  std::mt19937_64 rng(17);
  std::uniform_real_distribution<double> u(10.0, 900.0);
  uint64_t next_id = 1;
  for (int step = 0; step < 40; ++step) {
    std::vector<Request> arr;
    for (int j = 0; j < 6; ++j) arr.push_back(arrival(next_id++, 0.1 * step, 64 + 7 * j));
    std::vector<uint64_t> pid;
    std::vector<double> pe, pc;
    for (const Request& r : arr)
      if (r.id % 3) {  // predictions for two thirds of this step's arrivals
        pid.push_back(r.id);
        const double e = u(rng);
        pe.push_back(e);
        pc.push_back(e * 1.5);
      }
    const std::vector<uint64_t> got =
        a.step(arr.data(), arr.size(), pid.data(), pe.data(), pc.data(), pid.size(), 4);
    for (const Request& r : arr) b.on_arrival(r);
    for (size_t j = 0; j < pid.size(); ++j) b.on_prediction(pid[j], pe[j], pc[j]);
    std::vector<uint64_t> want;
    for (int j = 0; j < 4; ++j) {
      const auto id = b.next_request();
      if (!id) break;
      want.push_back(*id);
    }
    CHECK(got == want);
  }
  CHECK(a.waiting() == b.waiting());
  // a prediction the reference rejects (cvar < expectation): the step throws like
  // on_prediction, the step's arrivals stay applied
  Request r = arrival(next_id++, 9.0, 64);
  const uint64_t id = r.id;
  const double e = 100.0, c = 50.0;
  CHECK_THROWS_AS(a.step(&r, 1, &id, &e, &c, 1, 1), std::invalid_argument);
  CHECK(a.waiting_on(id));
}

static void scheduler_step_runs() {  // Scheduler::step_runs == the per-event call sequence
  ScoreConfig cfg;
  cfg.q_sat = 1e9;  // every prediction run sees its own beta
  cfg.rebuild_threshold = 0.0;
  Scheduler a(Policy::TIE, cfg), b(Policy::TIE, cfg);
  std::mt19937_64 rng(23);
  std::uniform_real_distribution<double> u(10.0, 900.0);
  uint64_t next_id = 1;
  for (int step = 0; step < 30; ++step) {
    // runs: [arrivals 3][predictions of them][arrivals 2][predictions of all 5]...
    std::vector<Request> arr;
    std::vector<uint64_t> pid, arr_end, pred_end;
    std::vector<double> pe, pc;
    for (int r = 0; r < 3; ++r) {
      for (int j = 0; j <= r; ++j) arr.push_back(arrival(next_id++, 0.1 * step, 64 + 9 * j));
      arr_end.push_back(arr.size());
      for (size_t j = pid.size(); j + 1 < arr.size(); ++j) {  // all but the newest arrival
        pid.push_back(arr[j].id);
        pe.push_back(u(rng));
        pc.push_back(pe.back() * 1.25);
      }
      pred_end.push_back(pid.size());
    }
    const std::vector<uint64_t> got = a.step_runs(arr.data(), arr_end.data(), pid.data(),
                                                  pe.data(), pc.data(), pred_end.data(), 3, 2);
    size_t a0 = 0, p0 = 0;
    for (int r = 0; r < 3; ++r) {
      for (size_t j = a0; j < arr_end[r]; ++j) b.on_arrival(arr[j]);
      for (size_t j = p0; j < pred_end[r]; ++j) b.on_prediction(pid[j], pe[j], pc[j]);
      a0 = arr_end[r];
      p0 = pred_end[r];
    }
    std::vector<uint64_t> want;
    for (int j = 0; j < 2; ++j) {
      const auto id = b.next_request();
      if (!id) break;
      want.push_back(*id);
    }
    CHECK(got == want);
  }
  CHECK(a.waiting() == b.waiting());
}

static void distribution_api() {  // test_smoke.py:8-26, dist.hpp per-item functions
  McContext mc(3.5);
  CHECK(mc.samples.size() == 10000 && std::is_sorted(mc.samples.begin(), mc.samples.end()));
  CensoredLogT cl(LogTParams(4.0, 0.8, 3.5), 512.0);
  const double e = censored_expectation(cl, mc);
  CHECK(0.0 < e && e <= 512.0);
  CHECK(censored_cvar(cl, mc, 0.0) == e);
  const double c = censored_cvar(cl, mc, 0.9);
  CHECK(e <= c && c <= 512.0);
  CHECK(censored_cvar(cl, mc, 0.999) == 512.0);
  for (double p : {0.05, 0.5, 0.9, 0.975}) CHECK(std::fabs(t_cdf(t_quantile(p, 3.5), 3.5) - p) < 1e-9);
  // E = Psi(y_max) + x_max (1 - T(y_max))  (dist.cpp:163-181)
  const double y_max = (std::log(512.0) - 4.0) / 0.8;
  const double e2 = psi(y_max, cl.dist, mc) + 512.0 * (1.0 - t_cdf(y_max, 3.5));
  CHECK(approx(e, e2, 1e-12));
  CHECK(approx(logt_cdf(std::exp(4.0), LogTParams(4.0, 0.8, 3.5)), 0.5, 1e-14));
  CHECK(approx(regularized_incomplete_beta(1.75, 0.5, 0.3),
               2.0 * t_cdf(-std::sqrt(3.5 / 0.3 - 3.5), 3.5), 1e-12));
  CHECK(approx(normal_quantile(normal_cdf(1.25)), 1.25, 1e-9));
  CHECK(lognormal_censored_cvar(4.0, 0.8, 512.0, 0.0) ==
        lognormal_censored_expectation(4.0, 0.8, 512.0));
  CHECK_THROWS_AS(psi(1.0, LogTParams(4.0, 0.8, 2.5), mc), std::invalid_argument);
  CHECK_THROWS_AS(logt_pdf(-1.0, LogTParams(4.0, 0.8, 3.5)), std::domain_error);
}

static void simulator_api() {  // test_smoke.py:37-53
  WorkloadSpec ws;
  ws.n_requests = 400;
  ws.rps = 80.0;
  ws.mu_range = {0.5, 2.5};
  ws.sigma_range = {0.4, 1.2};
  ws.prompt_range = {16, 128};
  ws.max_tokens = 512;
  const std::vector<Request> w = gen_logt_workload(ws, 11);
  ScoreConfig sc;
  EngineConfig eng;
  PredictorConfig pc;
  const SimReport tie_r = run_sim(w, Policy::TIE, sc, eng, pc, 11);
  const SimReport fcfs_r = run_sim(w, Policy::FCFS, sc, eng, pc, 11);
  CHECK(tie_r.events.size() == 400);
  CHECK(tie_r.metrics.ptla_avg < fcfs_r.metrics.ptla_avg);
  const SimReport again = run_sim(w, Policy::TIE, sc, eng, pc, 11);
  bool same = again.events.size() == tie_r.events.size();
  for (size_t i = 0; same && i < again.events.size(); ++i)
    same = again.events[i].completion_s == tie_r.events[i].completion_s;
  CHECK(same);
}

int main() {
  beta_and_score();
  waiting_queue_basics();
  waiting_queue_ties_and_rekey();
  waiting_queue_random_mirror();
  waiting_queue_entry_edits();
  scheduler_policies();
  scheduler_drift_rebuild();
  scheduler_step_batching();
  scheduler_step_runs();
  distribution_api();
  simulator_api();
  std::printf("dropin_sched: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
