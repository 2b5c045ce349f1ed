/* include/tie_cuda.h -- the drop-in C-ABI of the B200 TIE score / rank / fit path.
 *
 * The reference (TIE, arXiv 2604.00499; /root/reference/proj) has no FFI or plugin
 * registry: its boundary is the C++ header API in namespace tie (proj/include/tiesched/
 * *.hpp) plus the pybind11 module `_core` (proj/bindings/module.cpp).  Every entry point
 * below is the batched, device-resident replacement for one reference interface, cited
 * inline.  Plain pointers and sizes only -- no torch or C++ types cross this line.
 *
 * Pointers:   tie_* device entry points take DEVICE pointers and a cudaStream_t passed as
 *             void* (NULL = legacy default stream); they enqueue work and return.  The
 *             *_host variants take HOST pointers (pinned for full PCIe speed), copy in,
 *             compute, copy out and synchronise.
 * Errors:     return 0 on success, else
 *               TIE_EDOMAIN   (1)  the reference throws std::domain_error
 *               TIE_EINVALID  (2)  the reference throws std::invalid_argument
 *               TIE_ECUDA     (3)  CUDA / NCCL / allocation failure
 *             with a thread-local message in tie_last_error().  Per-request validation
 *             runs on the device: the kernels record the FIRST failing request index in
 *             the context; tie_sync() (and every *_host call) reports it with the
 *             reference's exception type and message.
 * Threading:  one tie_ctx per device; calls on one context are serialised per stream.
 */
#ifndef TIE_CUDA_H
#define TIE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TIE_OK 0
#define TIE_EDOMAIN 1
#define TIE_EINVALID 2
#define TIE_ECUDA 3

/* score flags */
#define TIE_SCORE_MOMENT 0u /* default: sigma-grid moment tables */
#define TIE_SCORE_EXACT 1u  /* one exp per sample-term, ascending sequential sum     */
#define TIE_SCORE_RAW 2u    /* per-item semantics: E and censored_cvar as returned by
                               dist.cpp:179-189 (no max(C,E), no compute_score checks) */

typedef struct tie_ctx tie_ctx;

const char* tie_last_error(void);
const char* tie_version(void);

/* ---- context: the device-resident McContext ------------------------------------------
 * Replaces McContext (proj/include/tiesched/dist.hpp:33-45, proj/src/dist.cpp:122-129):
 * uploads the caller's sorted standard-t sample set once and builds the per-context
 * tables (y-bucket index, sigma-grid moment prefix tables).  sigma_table_max <= 0 selects
 * the default (4.0); requests with sigma beyond it take the exact per-term path. */
int tie_ctx_create(int device, const double* samples, int n_samples, double nu,
                   double sigma_table_max, tie_ctx** out);
/* McContext(nu, n_samples, seed) generated on the host bit-identically to the reference
 * (rng.hpp:21-83 student_t draws, then ascending sort), then uploaded. */
int tie_ctx_create_mc(int device, double nu, int n_samples, uint64_t seed, tie_ctx** out);
void tie_ctx_destroy(tie_ctx* ctx);
int tie_ctx_samples(const tie_ctx* ctx, double* host_out, int n); /* copy of the set */
int tie_ctx_info(const tie_ctx* ctx, double* nu, int* n_samples, int* device);
/* device bytes of the context's request-invariant tables (samples, bucket index, sample bins,
 * tail table, sigma-grid moment tables); built once at creation, like McContext itself */
uint64_t tie_ctx_device_bytes(const tie_ctx* ctx);

/* Wait for `stream` and report the first device-side validation failure since the last
 * check (reference exception type + message), then clear it. */
int tie_sync(tie_ctx* ctx, void* stream);

/* ---- scalar helpers (host) -------------------------------------------------------------
 * compute_beta (proj/src/sched.cpp:9-17); beta is a per-batch scalar computed from the
 * GLOBAL waiting-queue length. */
int tie_compute_beta(int adaptive, double beta_fixed, double beta_max, double q_sat,
                     uint64_t queue_len, double* beta_out);
/* t_quantile / t_cdf (proj/src/dist.cpp:73-106), host, bit-identical to the reference. */
double tie_t_quantile(double p, double nu);
double tie_t_cdf(double y, double nu);

/* ---- per-item distribution functions (GPU, batched) ----------------------------------------
 * The reference's per-item public functions (proj/include/tiesched/dist.hpp:47-88; pybind
 * proj/bindings/module.cpp:48-60) over n items.  HOST buffers; inputs are validated in the
 * reference's per-item order first (the first failing item returns its error), then one
 * kernel evaluates every item.  Arguments per op (param is nu or alpha):
 *   TIE_EVAL_PSI             a=y  b=mu  c=sigma, param=nu (must equal the context's nu)
 *                            psi(y, LogTParams(mu, sigma, nu), mc)           dist.cpp:149-156
 *   TIE_EVAL_INCBETA         a=a  b=b   c=x   regularized_incomplete_beta     dist.cpp:52-63
 *   TIE_EVAL_T_PDF / T_CDF   a=y, param=nu    t_pdf / t_cdf (any nu)          dist.cpp:65-81
 *   TIE_EVAL_LOGT_PDF / CDF  a=x  b=mu  c=sigma, param=nu                     dist.cpp:131-140
 *   TIE_EVAL_NORMAL_CDF      a=z                                              dist.cpp:191
 *   TIE_EVAL_NORMAL_QUANTILE a=p                                              dist.cpp:193-225
 *   TIE_EVAL_LOGNORMAL_E     a=mu b=sigma c=x_max                             dist.cpp:227-236
 *   TIE_EVAL_LOGNORMAL_CVAR  a=mu b=sigma c=x_max, param=alpha                dist.cpp:238-249 */
#define TIE_EVAL_PSI 1
#define TIE_EVAL_INCBETA 2
#define TIE_EVAL_T_PDF 3
#define TIE_EVAL_T_CDF 4
#define TIE_EVAL_LOGT_PDF 5
#define TIE_EVAL_LOGT_CDF 6
#define TIE_EVAL_NORMAL_CDF 7
#define TIE_EVAL_NORMAL_QUANTILE 8
#define TIE_EVAL_LOGNORMAL_E 9
#define TIE_EVAL_LOGNORMAL_CVAR 10
int tie_eval_host(tie_ctx* ctx, int op, const double* a, const double* b, const double* c,
                  uint64_t n, double param, double* out);

/* ---- K1 score -------------------------------------------------------------------------
 * Batched replacement for, per request i,
 *   CensoredLogT cl(LogTParams(mu[i], sigma[i], nu), x_max[i]);      dist.cpp:108-120
 *   E = censored_expectation(cl, mc);                                dist.cpp:179-181
 *   C = max(censored_cvar(cl, mc, alpha), E);                        dist.cpp:183-189, sim.cpp:94
 *   S = compute_score(E, C, beta);                                   sched.cpp:19-26
 * (the run_sim precompute loop, proj/src/sim.cpp:77-96).  E, cvar, score may be NULL. */
int tie_score(tie_ctx* ctx, const double* mu, const double* sigma, const double* x_max,
              uint64_t n, double alpha, double beta, double* E, double* cvar, double* score,
              unsigned flags, void* stream);
/* Same, with the reference's Request::max_tokens (u32, workload.hpp:11-19) as x_max. */
int tie_score_u32(tie_ctx* ctx, const double* mu, const double* sigma,
                  const uint32_t* max_tokens, uint64_t n, double alpha, double beta, double* E,
                  double* cvar, double* score, unsigned flags, void* stream);

/* ---- K2 rank --------------------------------------------------------------------------
 * Dispatch order of a static waiting queue: replaces WaitingQueue::push x n followed by
 * pop_min until empty (proj/src/sched.cpp:28-94), i.e. order by (key asc, id asc).
 * ids == NULL means id = index.  Non-finite key -> TIE_EDOMAIN, duplicate id ->
 * TIE_EINVALID (sched.cpp:59-63), reported at tie_sync. */
int tie_rank(tie_ctx* ctx, const double* key, const uint64_t* ids, uint64_t n,
             uint64_t* order, void* stream);

/* ---- K1+K2 fused: score the queue and emit its dispatch order (ids = index) ---------- */
int tie_score_rank(tie_ctx* ctx, const double* mu, const double* sigma,
                   const uint32_t* max_tokens, uint64_t n, double alpha, double beta,
                   double* E, double* cvar, double* score, uint64_t* order, unsigned flags,
                   void* stream);

/* ---- K3 fit ---------------------------------------------------------------------------
 * Batched fit_logt_fixed_nu (proj/src/fit.cpp:73-178) over P prompts x K samples (x is
 * row-major P*K).  Outputs mirror FitResult (fit.hpp:15-25); any output except mu/sigma
 * may be NULL.  K < 3 -> TIE_EINVALID; nu invalid -> TIE_EDOMAIN (immediate); a sample
 * <= 0 or non-finite -> TIE_EDOMAIN at tie_sync (check_samples, fit.cpp:18-25). */
int tie_fit(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu, double* mu,
            double* sigma, double* log_likelihood, int32_t* iterations, uint8_t* converged,
            uint8_t* degenerate, void* stream);
/* logt_loglik / logt_loglik_grad (fit.cpp:44-71) for P parameter points over one sample
 * vector x[K]; grad may be NULL (else 2*P: d/dmu, d/dsigma interleaved). */
int tie_logt_loglik(tie_ctx* ctx, const double* x, uint64_t K, const double* mu,
                    const double* sigma, uint64_t P, double nu, double* ll, double* grad,
                    void* stream);

/* ---- host-buffer (end-to-end) variants ------------------------------------------------ */
int tie_score_host(tie_ctx* ctx, const double* mu, const double* sigma, const double* x_max,
                   uint64_t n, double alpha, double beta, double* E, double* cvar,
                   double* score, unsigned flags);
int tie_score_rank_host(tie_ctx* ctx, const double* mu, const double* sigma,
                        const uint32_t* max_tokens, uint64_t n, double alpha, double beta,
                        double* score, uint64_t* order, unsigned flags);
int tie_rank_host(tie_ctx* ctx, const double* key, const uint64_t* ids, uint64_t n,
                  uint64_t* order);
/* ---- request-sharded score + rank (host side paper_2604_00499_b200/dist.py) --
 * tie_score_rank_run: tie_score_rank on one shard, emitting its SORTED RUN as the 12-byte
 * records the exchange moves: run_keys[p] = score of the p-th request in (score, local index)
 * order, run_ids[p] = its shard-local index; `order` (u64, n) is the same order as
 * tie_score_rank's (also a scratch); score may be NULL.
 * tie_shard_cuts: the splitter exchange's send counts from G gathered regular samples of s
 * (key, global id) entries each (every rank's sample sorted; invalid entries id < 0 with
 * +max keys): the merged sample's elements at ranks j*t/G (t valid entries) are the G-1
 * splitters, and send_counts[j] = #{run records between splitters j-1 and j} in
 * (score, id_base + local id) order.  split_keys / split_ids (G-1) may be NULL.  One
 * single-CTA launch, G <= 32, G*s <= 8192. */
int tie_score_rank_run(tie_ctx* ctx, const double* mu, const double* sigma,
                       const uint32_t* max_tokens, uint64_t n, double alpha, double beta,
                       double* score, uint64_t* order, double* run_keys, uint32_t* run_ids,
                       unsigned flags, void* stream);
int tie_shard_cuts(tie_ctx* ctx, const double* run_keys, const uint32_t* run_ids,
                   uint64_t id_base, uint64_t n, const double* sample_keys,
                   const int64_t* sample_ids, int G, int s, int64_t* send_counts,
                   double* split_keys, int64_t* split_ids, void* stream);
/* The range exchange over peer memory: receive buffers allocated with
 * tie_ipc_alloc (cudaMalloc + a 64-byte cudaIpcMemHandle) are mapped into every other rank's
 * address space with tie_ipc_open (NVLink / NVSwitch peers), and tie_peer_put_runs writes this
 * rank's sorted run straight into them: piece g (send_counts[g] records, consecutive in the
 * run) lands at peer_keys[g] / peer_ids[g] + dst_offsets[g] -- one launch of peer stores in
 * place of the NCCL all-to-all of keys and ids (sched.cpp:28-31 order is kept: every piece
 * stays sorted).  The caller orders completion (stream sync + a barrier) before the
 * receivers read.  G <= 64; send_counts / dst_offsets / peer_* are HOST arrays. */
int tie_ipc_alloc(tie_ctx* ctx, uint64_t bytes, void** ptr, void* handle);
int tie_ipc_free(tie_ctx* ctx, void* ptr);
int tie_ipc_open(tie_ctx* ctx, const void* handle, void** ptr);
int tie_ipc_close(tie_ctx* ctx, void* ptr);
int tie_peer_put_runs(tie_ctx* ctx, const double* run_keys, const uint32_t* run_ids,
                      uint64_t n, int G, const uint64_t* send_counts,
                      const uint64_t* dst_offsets, void* const* peer_keys,
                      void* const* peer_ids, void* stream);
/* Sharded score+rank's final k-way merge: G runs on the device, run g =
 * keys/ids[g*stride .. g*stride + lens[g]) (lens: HOST array), each sorted by (score asc, id
 * asc) -- the reference heap's order (sched.cpp:28-31).  out_ids: the sum(lens) merged ids.
 * Replaces the merge implied by one global WaitingQueue over all shards. */
int tie_merge_runs(tie_ctx* ctx, const double* keys, const uint64_t* ids, int G,
                   uint64_t stride, const uint64_t* lens, uint64_t* out_ids, void* stream);
/* cmd_fit's per-prompt analysis (proj/tools/main.cpp:527-562) for P prompts x K >= 5 lengths:
 * families bitmask 1 logt (fit_logt_fixed_nu(x, nu), fit.cpp:73-178), 2 logt_free_nu
 * (fit_logt_free_nu over default_nu_grid, fit.cpp:180-200), 4 lognormal (fit.cpp:202-230),
 * 8 exponential (fit.cpp:232-243); each with ks_test(x, fit_cdf) (fit.cpp:245-284).
 * fits[f][10][P] doubles, f = the family's bit index, fields mu, sigma, nu, rate,
 * log_likelihood, iterations, converged, degenerate, ks_statistic, ks_p_value (families not
 * requested are left as passed in); tail[5][P] = tail_stats (fit.cpp:286-324: skewness, cv,
 * p90/p50, p99/p50, top10 share), NaN when K < 10, or tail = NULL. */
int tie_fit_report(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu,
                   unsigned families, double* fits, double* tail, void* stream);
int tie_fit_report_host(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu,
                        unsigned families, double* fits, double* tail);
/* ks_test(x, fit_cdf(fit, .)) (fit.cpp:245-284) against ONE caller-given fit (the pybind
 * ks_test_fit, module.cpp:117-123): family 0 LogTFixedNu, 1 LogTFreeNu (t CDF at `nu`),
 * 2 LogNormal (mu, sigma), 3 Exponential (rate).  K >= 5. */
int tie_ks_test_fit_host(tie_ctx* ctx, const double* x, uint64_t K, int family, double mu,
                         double sigma, double nu, double rate, double* statistic,
                         double* p_value);
int tie_fit_host(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu,
                 double* mu, double* sigma, double* log_likelihood, int32_t* iterations,
                 uint8_t* converged, uint8_t* degenerate);

/* ---- run_sim's scoring precompute -------------------------------------------------------
 * Replaces the loop of proj/src/sim.cpp:77-96: predictor 0 = oracle_predict, 1 =
 * noisy_predict(noise, seed) with the per-request Rng(mix64(seed, id)) (predictor.cpp:15-31);
 * family 0 = log-t (K1), 1 = log-normal closed forms (dist.cpp:227-249); CVaR = max(CVaR, E).
 * mu/sigma are the requests' TRUE parameters (Request::true_mu / true_sigma). */
int tie_sim_scores(tie_ctx* ctx, const double* mu, const double* sigma, const uint64_t* ids,
                   const uint32_t* max_tokens, uint64_t n, int predictor, double mu_sd,
                   double log_sigma_sd, uint64_t seed, int family, double alpha, double* E,
                   double* cvar, void* stream);
int tie_sim_scores_host(tie_ctx* ctx, const double* mu, const double* sigma,
                        const uint64_t* ids, const uint32_t* max_tokens, uint64_t n,
                        int predictor, double mu_sd, double log_sigma_sd, uint64_t seed,
                        int family, double alpha, double* E, double* cvar);

/* ---- GPU-resident waiting queue (the scheduler step) ------------------------------------
 * Replaces Scheduler + WaitingQueue (proj/include/tiesched/sched.hpp:43-90,
 * proj/src/sched.cpp:28-175): keys live on the device with a block-min index; the pop
 * sequence -- including drift rebuilds before pops -- is the reference's.  policy: 0 FCFS,
 * 1 SEPT, 2 TIE (sched.hpp:11).  Host buffers; each call completes before returning.  A
 * batch is validated before any of it is applied (the reference applies items one by one). */
typedef struct tie_queue tie_queue;
int tie_queue_create(tie_ctx* ctx, int policy, int adaptive, double beta_fixed,
                     double beta_max, double q_sat, double rebuild_threshold, double alpha,
                     uint64_t capacity, tie_queue** out);
void tie_queue_destroy(tie_queue* q);
uint64_t tie_queue_size(const tie_queue* q);       /* Scheduler::waiting()      */
double tie_queue_current_beta(const tie_queue* q); /* Scheduler::current_beta() */
/* Scheduler::on_arrival x m (sched.cpp:125-132) */
int tie_queue_arrive(tie_queue* q, const uint64_t* ids, const double* arrival_s,
                     const uint32_t* max_tokens, uint64_t m);
/* Scheduler::on_prediction x m with (E, CVaR) (sched.cpp:134-150) */
int tie_queue_predict(tie_queue* q, const uint64_t* ids, const double* expectation,
                      const double* cvar, uint64_t m);
/* run_sim's scoring chain (sim.cpp:85-95) on the GPU for (mu, sigma), then on_prediction */
int tie_queue_predict_logt(tie_queue* q, const uint64_t* ids, const double* mu,
                           const double* sigma, const uint32_t* max_tokens, uint64_t m);
/* Scheduler::next_request() up to max_pops times (sched.cpp:169-175); out_ids[max_pops] */
int tie_queue_next(tie_queue* q, uint64_t max_pops, uint64_t* out_ids, uint64_t* n_out);
/* One scheduler iteration with one device round trip: on_arrival x n_arr, the run_sim scoring
 * chain + on_prediction x n_pred, next_request() up to max_pops times (sched.cpp:125-175,
 * sim.cpp:85-95).  Same results / errors as the three calls above in sequence. */
int tie_queue_step(tie_queue* q, const uint64_t* arr_ids, const double* arr_time,
                   const uint32_t* arr_max_tokens, uint64_t n_arr, const uint64_t* pred_ids,
                   const double* mu, const double* sigma, const uint32_t* pred_max_tokens,
                   uint64_t n_pred, uint64_t max_pops, uint64_t* out_ids, uint64_t* n_out);
/* The same iteration with the predictions as on_prediction's (E, C) pairs (sched.cpp:136-150;
 * run_sim's precomputed scores): tie_queue_arrive + tie_queue_predict + tie_queue_next with
 * one device round trip. */
int tie_queue_step_ec(tie_queue* q, const uint64_t* arr_ids, const double* arr_time,
                      const uint32_t* arr_max_tokens, uint64_t n_arr, const uint64_t* pred_ids,
                      const double* E, const double* C, uint64_t n_pred, uint64_t max_pops,
                      uint64_t* out_ids, uint64_t* n_out);
/* A run of interleaved events, then pops: for r = 0..n_runs-1, on_arrival for the arrivals
 * [arr_end[r-1], arr_end[r]), then on_prediction for [pred_end[r-1], pred_end[r]) (arr_end[-1]
 * = pred_end[-1] = 0); then next_request() up to max_pops times -- each prediction run sees
 * the queue length after the arrivals before it (compute_beta, sched.cpp:139), exactly as the
 * reference's call sequence (sim.cpp:123-147 between two admissions).  One device round trip
 * when the sequence validates; otherwise the runs are applied as consecutive
 * tie_queue_step_ec calls, raising the first error where the call sequence raises it. */
int tie_queue_step_ec_runs(tie_queue* q, const uint64_t* arr_ids, const double* arr_time,
                           const uint32_t* arr_max_tokens, const uint64_t* arr_end,
                           const uint64_t* pred_ids, const double* E, const double* C,
                           const uint64_t* pred_end, uint64_t n_runs, uint64_t max_pops,
                           uint64_t* out_ids, uint64_t* n_out);
/* Scheduler::rebuild_if_drifted() (sched.cpp:152-167) */
int tie_queue_rebuild_if_drifted(tie_queue* q, int* rebuilt);
/* Shard-level primitives for a scheduler sharded by request (coordinated by
 * paper_2604_00499_b200/dist.py ShardedScheduler so the shards together behave as ONE
 * reference Scheduler):
 *  - set_peer_waiting: compute_beta's queue length becomes waiting() + peers (sched.cpp:9-17
 *    is called with the GLOBAL queue size, sched.cpp:136, 154);
 *  - beta_range: betas_in_use_ (sched.hpp:88) extremes and size (n_in_use 0: empty);
 *  - rebuild_at: rebuild_if_drifted's re-key (sched.cpp:156-166) at a beta decided globally;
 *  - peek: the next min(k, waiting) pops under the current keys (order-preserving u64 keys
 *    + ids, comparable across shards), leaving the queue unchanged and doing no rebuild. */
int tie_queue_set_peer_waiting(tie_queue* q, uint64_t peers);
int tie_queue_beta_range(const tie_queue* q, double* lo, double* hi, uint64_t* n_in_use);
int tie_queue_rebuild_at(tie_queue* q, double beta);
int tie_queue_peek(tie_queue* q, uint64_t k, uint64_t* keys, uint64_t* ids, uint64_t* n_out);

/* ---- WaitingQueue (proj/include/tiesched/sched.hpp:32-68, proj/src/sched.cpp:28-123) -------
 * policy TIE_QUEUE_RAW in tie_queue_create makes a bare WaitingQueue: entries carry caller-
 * given keys, pops are pop_min() in (key asc, req_id asc) order, and there is no Scheduler
 * rule (no policy keys, no beta, no drift rebuild).  The entry fields of QueueEntry
 * (sched.hpp:32-39) -- predicted, expectation, cvar, beta_at_update -- ride along.  Slots
 * are managed automatically: a queue grows (or compacts its popped slots) as needed.
 *  - push:        WaitingQueue::push x m (sched.cpp:59-67); predicted/E/C/beta may be NULL
 *  - update:      WaitingQueue::update x m (sched.cpp:69-79); a repeated id: last write wins
 *  - set_entries: write back edited entries (keys + fields) -- entries()/at() edits followed
 *                 by rebuild() (sched.cpp:110-114)
 *  - pop:         pop_min() x max_pops with the popped entries (sched.cpp:81-94)
 * and for any queue (a Scheduler's too):
 *  - contains / get (WaitingQueue::at, sched.cpp:96-108) / entries (slot order) / validate
 *    (sched.cpp:116-123: host index consistency + every device block minimum rescanned). */
#define TIE_QUEUE_FCFS 0
#define TIE_QUEUE_SEPT 1
#define TIE_QUEUE_TIE 2
#define TIE_QUEUE_RAW 3
int tie_queue_contains(const tie_queue* q, uint64_t id); /* 1 waiting, 0 not */
int tie_queue_push(tie_queue* q, const uint64_t* ids, const double* keys,
                   const uint8_t* predicted, const double* E, const double* C,
                   const double* beta_at_update, uint64_t m);
int tie_queue_update(tie_queue* q, const uint64_t* ids, const double* keys, uint64_t m);
int tie_queue_set_entries(tie_queue* q, const uint64_t* ids, const double* keys,
                          const uint8_t* predicted, const double* E, const double* C,
                          const double* beta_at_update, uint64_t m);
int tie_queue_pop(tie_queue* q, uint64_t max_pops, uint64_t* ids, double* keys,
                  uint8_t* predicted, double* E, double* C, double* beta_at_update,
                  uint64_t* n_out);
int tie_queue_get(tie_queue* q, const uint64_t* ids, uint64_t m, double* keys,
                  uint8_t* predicted, double* E, double* C, double* beta_at_update);
int tie_queue_entries(tie_queue* q, uint64_t cap, uint64_t* ids, double* keys,
                      uint8_t* predicted, double* E, double* C, double* beta_at_update,
                      uint64_t* n_out);
int tie_queue_validate(tie_queue* q, int* ok);
/* slot management: relayout the live entries into `capacity` slots (>= waiting, < 2^32) */
int tie_queue_reserve(tie_queue* q, uint64_t capacity);
uint64_t tie_queue_capacity(const tie_queue* q);
uint64_t tie_queue_slots_used(const tie_queue* q);

/* ---- input formats ------------------------------------------------------
 * Request traces: JSONL, one object per request -- load_trace / save_trace
 * (proj/src/workload.cpp:82-161).  Load fills missing arrival_s from
 * poisson_arrivals(fill_rps, count, seed) (fill_rps <= 0: such records are an error) and
 * stable-sorts by arrival; mu / sigma are NaN where a record has none.  Host-only calls. */
typedef struct tie_trace tie_trace;
int tie_trace_load(const char* path, double fill_rps, uint64_t seed, tie_trace** out);
uint64_t tie_trace_size(const tie_trace* t);
const uint64_t* tie_trace_ids(const tie_trace* t);
const double* tie_trace_arrival(const tie_trace* t);
const uint32_t* tie_trace_prompt_tokens(const tie_trace* t);
const uint32_t* tie_trace_output_tokens(const tie_trace* t);
const uint32_t* tie_trace_max_tokens(const tie_trace* t);
const double* tie_trace_mu(const tie_trace* t);
const double* tie_trace_sigma(const tie_trace* t);
void tie_trace_free(tie_trace* t);
int tie_trace_save(const char* path, uint64_t n, const uint64_t* ids, const double* arrival,
                   const uint32_t* prompt_tokens, const uint32_t* output_tokens,
                   const uint32_t* max_tokens, const double* mu, const double* sigma);
/* Fit inputs of `tie fit` (proj/tools/main.cpp:432-495): "*.csv" with header
 * prompt_id,length, else JSONL {"prompt_id": str, "lengths": [int >= 1]}.  Prompt p's
 * samples are lengths[offsets[p] .. offsets[p+1]). */
typedef struct tie_fit_input tie_fit_input;
int tie_fit_input_load(const char* path, tie_fit_input** out);
uint64_t tie_fit_input_count(const tie_fit_input* f);
const char* tie_fit_input_prompt_id(const tie_fit_input* f, uint64_t i);
const uint64_t* tie_fit_input_offsets(const tie_fit_input* f);
const double* tie_fit_input_lengths(const tie_fit_input* f);
void tie_fit_input_free(tie_fit_input* f);
/* tie_fit_report over ragged prompts (grouped by sample count, one GPU batch per group) */
int tie_fit_report_ragged_host(tie_ctx* ctx, const double* lengths, const uint64_t* offsets,
                               uint64_t P, double nu, unsigned families, double* fits,
                               double* tail);

/* ---- diagnostics ------------------------------------------------------------------------
 * Kernel-level profiling: with tie_profile(ctx, 1) every kernel launched by this context is
 * bracketed by a CUDA event pair on its stream; tie_profile_report() synchronises and
 * writes one "name<TAB>launches<TAB>total_ms" line per kernel class.  Off by default. */
int tie_profile(tie_ctx* ctx, int enable);
int tie_profile_report(tie_ctx* ctx, char* buf, size_t len);
/*
 * Number of this library's kernels launched by the calling thread since the last reset
 * (bench.py's gpu_launches claim). */
uint64_t tie_launch_count(int reset);

#ifdef __cplusplus
}
#endif
#endif /* TIE_CUDA_H */
