// pybind11 `_core`: the Python surface of the B200 TIE path.  Same names and argument
// names as the reference module for the score / rank / fit path (proj/bindings/module.cpp:
// 22-83, 171-172), plus batched NumPy entry points and raw device-pointer entry points
// (for torch CUDA tensors: pass tensor.data_ptr() and the CUDA stream handle).
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cmath>
#include <optional>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "tie_cuda.h"
#include "tiesched_b200.hpp"

namespace py = pybind11;
using namespace tie;

namespace {

template <class T>
using carray = py::array_t<T, py::array::c_style | py::array::forcecast>;

void throw_code(int rc) {
  if (rc == TIE_OK) return;
  const std::string msg = tie_last_error();
  if (rc == TIE_EDOMAIN) throw std::domain_error(msg);
  if (rc == TIE_EINVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

template <class T>
const T* ptr_or_null(const py::object& o) {
  if (o.is_none()) return nullptr;
  return o.cast<carray<T>>().data();
}

void* vp(uintptr_t p) { return reinterpret_cast<void*>(p); }

struct KsResultPy {  // fit.hpp:43-47
  double statistic = 0.0;
  double p_value = 0.0;
  int n = 0;
};


}  // namespace

PYBIND11_MODULE(_core, m) {
  m.doc() = "B200 TIE score / rank / fit path (sm_100a kernels behind the tiesched API)";
  m.attr("__version__") = tie_version();

  // ------------------------------------------------------------- distribution
  py::class_<LogTParams>(m, "LogTParams")
      .def(py::init<double, double, double>(), py::arg("mu"), py::arg("sigma"), py::arg("nu"))
      .def_readonly("mu", &LogTParams::mu)
      .def_readonly("sigma", &LogTParams::sigma)
      .def_readonly("nu", &LogTParams::nu)
      .def_readonly("sigma_clamped", &LogTParams::sigma_clamped)
      .def("__repr__", [](const LogTParams& p) {
        return "LogTParams(mu=" + std::to_string(p.mu) + ", sigma=" + std::to_string(p.sigma) +
               ", nu=" + std::to_string(p.nu) + ")";
      });

  py::class_<CensoredLogT>(m, "CensoredLogT")
      .def(py::init<LogTParams, double>(), py::arg("dist"), py::arg("x_max"))
      .def_readonly("dist", &CensoredLogT::dist)
      .def_readonly("x_max", &CensoredLogT::x_max);

  py::class_<McContext>(m, "McContext")
      .def(py::init<double, int, uint64_t, int>(), py::arg("nu"),
           py::arg("n_samples") = McContext::kDefaultSamples,
           py::arg("seed") = McContext::kDefaultSeed, py::arg("device") = 0)
      .def_readonly("nu", &McContext::nu)
      .def_readonly("seed", &McContext::seed)
      .def_property_readonly("n_samples", &McContext::n_samples)
      .def_property_readonly("samples",
                             [](const McContext& mc) {
                               return carray<double>((py::ssize_t)mc.n_samples(),
                                                     mc.samples.data());
                             })
      .def_property_readonly("handle",
                             [](const McContext& mc) { return (uintptr_t)mc.handle(); })
      .def_property_readonly("device_bytes",
                             [](const McContext& mc) { return tie_ctx_device_bytes(mc.handle()); });

  m.def("t_pdf", &t_pdf, py::arg("y"), py::arg("nu"));
  m.def("t_cdf", &t_cdf, py::arg("y"), py::arg("nu"));
  m.def("t_quantile", &t_quantile, py::arg("p"), py::arg("nu"));
  m.def("sample_logt", &sample_logt, py::arg("params"), py::arg("n"), py::arg("seed"));
  m.def("censored_expectation", &censored_expectation, py::arg("censored"), py::arg("mc"));
  m.def("censored_cvar", &censored_cvar, py::arg("censored"), py::arg("mc"), py::arg("alpha"));
  m.def("psi", &psi, py::arg("y"), py::arg("params"), py::arg("mc"));
  m.def("regularized_incomplete_beta", &regularized_incomplete_beta, py::arg("a"), py::arg("b"),
        py::arg("x"));
  m.def("logt_pdf", &logt_pdf, py::arg("x"), py::arg("params"));
  m.def("logt_cdf", &logt_cdf, py::arg("x"), py::arg("params"));
  m.def("normal_cdf", &normal_cdf, py::arg("z"));
  m.def("normal_quantile", &normal_quantile, py::arg("p"));
  m.def("lognormal_censored_expectation", &lognormal_censored_expectation, py::arg("mu"),
        py::arg("sigma"), py::arg("x_max"));
  m.def("lognormal_censored_cvar", &lognormal_censored_cvar, py::arg("mu"), py::arg("sigma"),
        py::arg("x_max"), py::arg("alpha"));
  m.def(
      "dist_eval",
      [](const std::string& fn, carray<double> a, py::object b, py::object c, double param,
         const McContext* mc) {
        static const std::pair<const char*, int> ops[] = {
            {"psi", TIE_EVAL_PSI}, {"regularized_incomplete_beta", TIE_EVAL_INCBETA},
            {"t_pdf", TIE_EVAL_T_PDF}, {"t_cdf", TIE_EVAL_T_CDF},
            {"logt_pdf", TIE_EVAL_LOGT_PDF}, {"logt_cdf", TIE_EVAL_LOGT_CDF},
            {"normal_cdf", TIE_EVAL_NORMAL_CDF}, {"normal_quantile", TIE_EVAL_NORMAL_QUANTILE},
            {"lognormal_censored_expectation", TIE_EVAL_LOGNORMAL_E},
            {"lognormal_censored_cvar", TIE_EVAL_LOGNORMAL_CVAR}};
        int op = 0;
        for (const auto& o : ops)
          if (fn == o.first) op = o.second;
        if (!op) throw py::value_error("dist_eval: unknown function " + fn);
        const size_t n = (size_t)a.size();
        carray<double> bb = b.is_none() ? carray<double>(n) : b.cast<carray<double>>();
        carray<double> cc = c.is_none() ? carray<double>(n) : c.cast<carray<double>>();
        if ((size_t)bb.size() != n || (size_t)cc.size() != n)
          throw py::value_error("dist_eval: array lengths differ");
        std::vector<double> out;
        {
          py::gil_scoped_release nogil;
          out = eval_batch(op, a.data(), bb.data(), cc.data(), n, param, mc);
        }
        return carray<double>((py::ssize_t)n, out.data());
      },
      py::arg("fn"), py::arg("a"), py::arg("b") = py::none(), py::arg("c") = py::none(),
      py::arg("param") = 0.0, py::arg("mc") = nullptr,
      "batched per-item distribution function on the GPU: fn(a[i], b[i], c[i]; param) with the "
      "reference's argument order (psi: y, mu, sigma, param=nu, mc; logt_*: x, mu, sigma, "
      "param=nu; t_*: y, param=nu; lognormal_*: mu, sigma, x_max, param=alpha)");

  // ------------------------------------------------------------- scoring / policy
  py::enum_<Policy>(m, "Policy")
      .value("FCFS", Policy::FCFS)
      .value("SEPT", Policy::SEPT)
      .value("TIE", Policy::TIE);
  py::enum_<BetaMode>(m, "BetaMode")
      .value("Fixed", BetaMode::Fixed)
      .value("AdaptiveLinear", BetaMode::AdaptiveLinear);
  py::enum_<PredictorKind>(m, "PredictorKind")
      .value("NoPredictor", PredictorKind::None)
      .value("Oracle", PredictorKind::Oracle)
      .value("Noisy", PredictorKind::Noisy);
  py::enum_<ScoreFamily>(m, "ScoreFamily")
      .value("LogT", ScoreFamily::LogT)
      .value("LogNormal", ScoreFamily::LogNormal);
  py::class_<ScoreConfig>(m, "ScoreConfig")
      .def(py::init<>())
      .def_readwrite("alpha", &ScoreConfig::alpha)
      .def_readwrite("beta_mode", &ScoreConfig::beta_mode)
      .def_readwrite("beta_fixed", &ScoreConfig::beta_fixed)
      .def_readwrite("beta_max", &ScoreConfig::beta_max)
      .def_readwrite("q_sat", &ScoreConfig::q_sat)
      .def_readwrite("rebuild_threshold", &ScoreConfig::rebuild_threshold);
  m.def("compute_beta", &compute_beta, py::arg("config"), py::arg("queue_len"));
  m.def("compute_score", &compute_score, py::arg("expectation"), py::arg("cvar"),
        py::arg("beta"));

  // batched, NumPy in / NumPy out (host buffers; H2D/D2H inside)
  m.def(
      "score_batch",
      [](carray<double> mu, carray<double> sigma, carray<double> x_max, const McContext& mc,
         const ScoreConfig& cfg, py::object queue_len, bool exact) {
        const size_t n = (size_t)mu.size();
        if ((size_t)sigma.size() != n || (size_t)x_max.size() != n)
          throw std::invalid_argument("score_batch: mu, sigma, x_max must have equal length");
        const size_t q = queue_len.is_none() ? n : queue_len.cast<size_t>();
        carray<double> E(n), C(n), S(n);
        {
          py::gil_scoped_release nogil;
          score_batch(mu.data(), sigma.data(), x_max.data(), n, mc, cfg, q, E.mutable_data(),
                      C.mutable_data(), S.mutable_data(), exact);
        }
        return py::make_tuple(E, C, S);
      },
      py::arg("mu"), py::arg("sigma"), py::arg("x_max"), py::arg("mc"), py::arg("config"),
      py::arg("queue_len") = py::none(), py::arg("exact") = false,
      "E, CVaR (max'ed with E) and score for every request; beta from compute_beta(config, "
      "queue_len) with queue_len defaulting to the batch size");
  m.def(
      "rank",
      [](carray<double> key, py::object ids, py::object mc) {
        const size_t n = (size_t)key.size();
        const uint64_t* id = ptr_or_null<uint64_t>(ids);
        carray<uint64_t> idarr;
        if (id) {
          idarr = ids.cast<carray<uint64_t>>();
          if ((size_t)idarr.size() != n) throw std::invalid_argument("rank: ids length mismatch");
          id = idarr.data();
        }
        const McContext* ctx = mc.is_none() ? nullptr : mc.cast<const McContext*>();
        carray<uint64_t> order(n);
        {
          py::gil_scoped_release nogil;
          rank(key.data(), n, order.mutable_data(), id, ctx);
        }
        return order;
      },
      py::arg("key"), py::arg("ids") = py::none(), py::arg("mc") = py::none(),
      "dispatch order by (key asc, id asc): the WaitingQueue pop order of a static queue");
  m.def(
      "score_rank",
      [](carray<double> mu, carray<double> sigma, carray<uint32_t> max_tokens,
         const McContext& mc, const ScoreConfig& cfg, py::object queue_len, bool exact) {
        const size_t n = (size_t)mu.size();
        if ((size_t)sigma.size() != n || (size_t)max_tokens.size() != n)
          throw std::invalid_argument("score_rank: input lengths differ");
        const size_t q = queue_len.is_none() ? n : queue_len.cast<size_t>();
        carray<double> S(n);
        carray<uint64_t> order(n);
        {
          py::gil_scoped_release nogil;
          score_rank(mu.data(), sigma.data(), max_tokens.data(), n, mc, cfg, q,
                     S.mutable_data(), order.mutable_data(), exact);
        }
        return py::make_tuple(S, order);
      },
      py::arg("mu"), py::arg("sigma"), py::arg("max_tokens"), py::arg("mc"), py::arg("config"),
      py::arg("queue_len") = py::none(), py::arg("exact") = false);

  // ------------------------------------------------------------- fitting
  py::enum_<FitFamily>(m, "FitFamily")
      .value("LogTFixedNu", FitFamily::LogTFixedNu)
      .value("LogTFreeNu", FitFamily::LogTFreeNu)
      .value("LogNormal", FitFamily::LogNormal)
      .value("Exponential", FitFamily::Exponential);
  py::class_<FitResult>(m, "FitResult")
      .def_readonly("family", &FitResult::family)
      .def_readonly("mu", &FitResult::mu)
      .def_readonly("sigma", &FitResult::sigma)
      .def_readonly("nu", &FitResult::nu)
      .def_readonly("rate", &FitResult::rate)
      .def_readonly("log_likelihood", &FitResult::log_likelihood)
      .def_readonly("converged", &FitResult::converged)
      .def_readonly("iterations", &FitResult::iterations)
      .def_readonly("degenerate", &FitResult::degenerate);
  m.def("logt_loglik", &logt_loglik, py::arg("x"), py::arg("mu"), py::arg("sigma"),
        py::arg("nu"));
  m.def("logt_loglik_grad", &logt_loglik_grad, py::arg("x"), py::arg("mu"), py::arg("sigma"),
        py::arg("nu"));
  m.def("fit_logt_fixed_nu", &fit_logt_fixed_nu, py::arg("x"), py::arg("nu") = 3.5);
  m.def(
      "fit_logt_fixed_nu_batch",
      [](carray<double> x, double nu) {
        if (x.ndim() != 2) throw std::invalid_argument("fit_logt_fixed_nu_batch: x must be P x K");
        const size_t P = (size_t)x.shape(0), K = (size_t)x.shape(1);
        carray<double> mu(P), sg(P), ll(P);
        carray<int32_t> it(P);
        carray<uint8_t> cv(P), dg(P);
        int rc;
        {
          py::gil_scoped_release nogil;
          rc = tie_fit_host(default_context(), x.data(), P, K, nu, mu.mutable_data(),
                            sg.mutable_data(), ll.mutable_data(), it.mutable_data(),
                            cv.mutable_data(), dg.mutable_data());
        }
        throw_code(rc);
        py::dict out;
        out["mu"] = mu;
        out["sigma"] = sg;
        out["log_likelihood"] = ll;
        out["iterations"] = it;
        out["converged"] = cv.attr("astype")("bool");
        out["degenerate"] = dg.attr("astype")("bool");
        return out;
      },
      py::arg("x"), py::arg("nu") = 3.5,
      "fit_logt_fixed_nu over every row of a P x K array; returns a dict of arrays");

  // ------------------------------------------------------------- device-pointer entry points
  // (torch CUDA tensors: tensor.data_ptr(), torch.cuda.current_stream().cuda_stream)
  m.def(
      "score_device",
      [](uintptr_t ctx, uintptr_t mu, uintptr_t sigma, uintptr_t x_max, bool x_is_u32,
         uint64_t n, double alpha, double beta, uintptr_t E, uintptr_t C, uintptr_t S,
         unsigned flags, uintptr_t stream) {
        auto* c = reinterpret_cast<tie_ctx*>(ctx);
        const int rc =
            x_is_u32 ? tie_score_u32(c, (const double*)mu, (const double*)sigma,
                                     (const uint32_t*)x_max, n, alpha, beta, (double*)E,
                                     (double*)C, (double*)S, flags, vp(stream))
                     : tie_score(c, (const double*)mu, (const double*)sigma,
                                 (const double*)x_max, n, alpha, beta, (double*)E, (double*)C,
                                 (double*)S, flags, vp(stream));
        throw_code(rc);
      },
      py::arg("ctx"), py::arg("mu"), py::arg("sigma"), py::arg("x_max"), py::arg("x_is_u32"),
      py::arg("n"), py::arg("alpha"), py::arg("beta"), py::arg("E"), py::arg("cvar"),
      py::arg("score"), py::arg("flags") = 0u, py::arg("stream") = 0);
  m.def(
      "rank_device",
      [](uintptr_t ctx, uintptr_t key, uintptr_t ids, uint64_t n, uintptr_t order,
         uintptr_t stream) {
        throw_code(tie_rank(reinterpret_cast<tie_ctx*>(ctx), (const double*)key,
                            (const uint64_t*)ids, n, (uint64_t*)order, vp(stream)));
      },
      py::arg("ctx"), py::arg("key"), py::arg("ids"), py::arg("n"), py::arg("order"),
      py::arg("stream") = 0);
  m.def(
      "merge_runs_device",
      [](uintptr_t ctx, uintptr_t keys, uintptr_t ids, uint64_t stride,
         std::vector<uint64_t> lens, uintptr_t out_ids, uintptr_t stream) {
        throw_code(tie_merge_runs(reinterpret_cast<tie_ctx*>(ctx), (const double*)keys,
                                  (const uint64_t*)ids, (int)lens.size(), stride, lens.data(),
                                  (uint64_t*)out_ids, vp(stream)));
      },
      py::arg("ctx"), py::arg("keys"), py::arg("ids"), py::arg("stride"), py::arg("lens"),
      py::arg("out_ids"), py::arg("stream") = 0,
      "k-way merge of G device runs sorted by (score, id): the sharded rank's final step");
  m.def(
      "score_rank_run_device",
      [](uintptr_t ctx, uintptr_t mu, uintptr_t sigma, uintptr_t max_tokens, uint64_t n,
         double alpha, double beta, uintptr_t score, uintptr_t order, uintptr_t run_keys,
         uintptr_t run_ids, unsigned flags, uintptr_t stream) {
        throw_code(tie_score_rank_run(reinterpret_cast<tie_ctx*>(ctx), (const double*)mu,
                                      (const double*)sigma, (const uint32_t*)max_tokens, n,
                                      alpha, beta, (double*)score, (uint64_t*)order,
                                      (double*)run_keys, (uint32_t*)run_ids, flags, vp(stream)));
      },
      py::arg("ctx"), py::arg("mu"), py::arg("sigma"), py::arg("max_tokens"), py::arg("n"),
      py::arg("alpha"), py::arg("beta"), py::arg("score"), py::arg("order"), py::arg("run_keys"),
      py::arg("run_ids"), py::arg("flags") = 0, py::arg("stream") = 0,
      "score + rank one shard and emit its sorted run (f64 keys, u32 local ids)");
  m.def(
      "shard_cuts_device",
      [](uintptr_t ctx, uintptr_t run_keys, uintptr_t run_ids, uint64_t id_base, uint64_t n,
         uintptr_t sample_keys, uintptr_t sample_ids, int G, int s, uintptr_t send_counts,
         uintptr_t split_keys, uintptr_t split_ids, uintptr_t stream) {
        throw_code(tie_shard_cuts(reinterpret_cast<tie_ctx*>(ctx), (const double*)run_keys,
                                  (const uint32_t*)run_ids, id_base, n,
                                  (const double*)sample_keys, (const int64_t*)sample_ids, G, s,
                                  (int64_t*)send_counts, (double*)split_keys,
                                  (int64_t*)split_ids, vp(stream)));
      },
      py::arg("ctx"), py::arg("run_keys"), py::arg("run_ids"), py::arg("id_base"), py::arg("n"),
      py::arg("sample_keys"), py::arg("sample_ids"), py::arg("G"), py::arg("s"),
      py::arg("send_counts"), py::arg("split_keys") = 0, py::arg("split_ids") = 0,
      py::arg("stream") = 0, "splitter exchange send counts from gathered regular samples");
  // CUDA IPC + the range exchange over peer memory (tie_ipc_*, tie_peer_put_runs)
  m.def(
      "ipc_alloc",
      [](uintptr_t ctx, uint64_t bytes) {
        void* ptr = nullptr;
        char h[64];
        throw_code(tie_ipc_alloc(reinterpret_cast<tie_ctx*>(ctx), bytes, &ptr, h));
        return py::make_tuple((uintptr_t)ptr, py::bytes(h, 64));
      },
      py::arg("ctx"), py::arg("bytes"), "cudaMalloc + its IPC handle -> (device pointer, handle)");
  m.def(
      "ipc_free",
      [](uintptr_t ctx, uintptr_t ptr) {
        throw_code(tie_ipc_free(reinterpret_cast<tie_ctx*>(ctx), (void*)ptr));
      },
      py::arg("ctx"), py::arg("ptr"));
  m.def(
      "ipc_open",
      [](uintptr_t ctx, py::bytes handle) {
        const std::string h = handle;
        if (h.size() != 64) throw py::value_error("ipc_open: a handle is 64 bytes");
        void* ptr = nullptr;
        throw_code(tie_ipc_open(reinterpret_cast<tie_ctx*>(ctx), h.data(), &ptr));
        return (uintptr_t)ptr;
      },
      py::arg("ctx"), py::arg("handle"), "map another process's buffer -> device pointer");
  m.def(
      "ipc_close",
      [](uintptr_t ctx, uintptr_t ptr) {
        throw_code(tie_ipc_close(reinterpret_cast<tie_ctx*>(ctx), (void*)ptr));
      },
      py::arg("ctx"), py::arg("ptr"));
  m.def(
      "peer_put_runs_device",
      [](uintptr_t ctx, uintptr_t run_keys, uintptr_t run_ids, uint64_t n,
         std::vector<uint64_t> send_counts, std::vector<uint64_t> dst_offsets,
         std::vector<uintptr_t> peer_keys, std::vector<uintptr_t> peer_ids, uintptr_t stream) {
        const size_t G = send_counts.size();
        if (dst_offsets.size() != G || peer_keys.size() != G || peer_ids.size() != G)
          throw py::value_error("peer_put_runs_device: per-peer lists differ in length");
        std::vector<void*> pk(G), pi(G);
        for (size_t g = 0; g < G; ++g) {
          pk[g] = (void*)peer_keys[g];
          pi[g] = (void*)peer_ids[g];
        }
        throw_code(tie_peer_put_runs(reinterpret_cast<tie_ctx*>(ctx), (const double*)run_keys,
                                     (const uint32_t*)run_ids, n, (int)G, send_counts.data(),
                                     dst_offsets.data(), pk.data(), pi.data(), vp(stream)));
      },
      py::arg("ctx"), py::arg("run_keys"), py::arg("run_ids"), py::arg("n"),
      py::arg("send_counts"), py::arg("dst_offsets"), py::arg("peer_keys"), py::arg("peer_ids"),
      py::arg("stream") = 0, "write this rank's sorted run pieces into the peers' buffers");
  m.def(
      "fit_report_device",
      [](uintptr_t ctx, uintptr_t x, uint64_t P, uint64_t K, double nu, unsigned families,
         uintptr_t fits, uintptr_t tail, uintptr_t stream) {
        throw_code(tie_fit_report(reinterpret_cast<tie_ctx*>(ctx), (const double*)x, P, K, nu,
                                  families, (double*)fits, (double*)tail, vp(stream)));
      },
      py::arg("ctx"), py::arg("x"), py::arg("P"), py::arg("K"), py::arg("nu"),
      py::arg("families"), py::arg("fits"), py::arg("tail"), py::arg("stream") = 0,
      "cmd_fit's per-prompt analysis on device buffers: fits[4][10][P], tail[5][P]");
  m.def(
      "fit_report",
      [](carray<double> x, double nu, unsigned families) {
        if (x.ndim() != 2) throw py::value_error("fit_report: x must be P x K");
        const size_t P = (size_t)x.shape(0), K = (size_t)x.shape(1);
        carray<double> fits({(py::ssize_t)4, (py::ssize_t)10, (py::ssize_t)P});
        carray<double> tail({(py::ssize_t)5, (py::ssize_t)P});
        std::fill(fits.mutable_data(), fits.mutable_data() + fits.size(),
                  std::numeric_limits<double>::quiet_NaN());
        int rc;
        {
          py::gil_scoped_release nogil;
          rc = tie_fit_report_host(default_context(), x.data(), P, K, nu, families,
                                   fits.mutable_data(), tail.mutable_data());
        }
        throw_code(rc);
        return py::make_tuple(fits, tail);
      },
      py::arg("x"), py::arg("nu") = 3.5, py::arg("families") = 15u,
      "cmd_fit's per-prompt analysis (tools/main.cpp:527-562) of every row of a P x K array: "
      "(fits[4][10][P], tail[5][P])");
  // ---- input formats
  m.def(
      "load_trace_soa",
      [](const std::string& path, double fill_rps, uint64_t seed) {
        tie_trace* t = nullptr;
        throw_code(tie_trace_load(path.c_str(), fill_rps, seed, &t));
        const size_t n = tie_trace_size(t);
        py::dict d;
        d["id"] = carray<uint64_t>((py::ssize_t)n, tie_trace_ids(t));
        d["arrival_s"] = carray<double>((py::ssize_t)n, tie_trace_arrival(t));
        d["prompt_tokens"] = carray<uint32_t>((py::ssize_t)n, tie_trace_prompt_tokens(t));
        d["output_tokens"] = carray<uint32_t>((py::ssize_t)n, tie_trace_output_tokens(t));
        d["max_tokens"] = carray<uint32_t>((py::ssize_t)n, tie_trace_max_tokens(t));
        d["mu"] = carray<double>((py::ssize_t)n, tie_trace_mu(t));
        d["sigma"] = carray<double>((py::ssize_t)n, tie_trace_sigma(t));
        tie_trace_free(t);
        return d;
      },
      py::arg("path"), py::arg("fill_rps") = 0.0, py::arg("seed") = 0,
      "load_trace (workload.cpp:106-161) -> dict of arrays (mu / sigma NaN where absent)");
  m.def(
      "save_trace_soa",
      [](const std::string& path, carray<uint64_t> id, carray<double> arrival_s,
         carray<uint32_t> prompt_tokens, carray<uint32_t> output_tokens,
         carray<uint32_t> max_tokens, py::object mu, py::object sigma) {
        const size_t n = (size_t)id.size();
        carray<double> m = mu.is_none() ? carray<double>() : mu.cast<carray<double>>();
        carray<double> s = sigma.is_none() ? carray<double>() : sigma.cast<carray<double>>();
        throw_code(tie_trace_save(path.c_str(), n, id.data(), arrival_s.data(),
                                  prompt_tokens.data(), output_tokens.data(), max_tokens.data(),
                                  mu.is_none() ? nullptr : m.data(),
                                  sigma.is_none() ? nullptr : s.data()));
      },
      py::arg("path"), py::arg("id"), py::arg("arrival_s"), py::arg("prompt_tokens"),
      py::arg("output_tokens"), py::arg("max_tokens"), py::arg("mu") = py::none(),
      py::arg("sigma") = py::none(), "save_trace (workload.cpp:94-104)");
  m.def(
      "load_fit_input",
      [](const std::string& path) {
        tie_fit_input* f = nullptr;
        throw_code(tie_fit_input_load(path.c_str(), &f));
        const size_t n = tie_fit_input_count(f);
        py::list ids;
        for (size_t i = 0; i < n; ++i) ids.append(py::str(tie_fit_input_prompt_id(f, i)));
        const uint64_t* off = tie_fit_input_offsets(f);
        auto offsets = carray<uint64_t>((py::ssize_t)(n + 1), off);
        auto lengths = carray<double>((py::ssize_t)off[n], tie_fit_input_lengths(f));
        tie_fit_input_free(f);
        return py::make_tuple(ids, offsets, lengths);
      },
      py::arg("path"),
      "`tie fit` input (main.cpp:432-495): (prompt_ids, offsets[P+1], lengths)");
  m.def(
      "fit_report_ragged",
      [](carray<double> lengths, carray<uint64_t> offsets, double nu, unsigned families) {
        const size_t P = (size_t)offsets.size() - 1;
        carray<double> fits({(py::ssize_t)4, (py::ssize_t)10, (py::ssize_t)P});
        carray<double> tail({(py::ssize_t)5, (py::ssize_t)P});
        std::fill(fits.mutable_data(), fits.mutable_data() + fits.size(),
                  std::numeric_limits<double>::quiet_NaN());
        int rc;
        {
          py::gil_scoped_release nogil;
          rc = tie_fit_report_ragged_host(default_context(), lengths.data(), offsets.data(), P,
                                          nu, families, fits.mutable_data(),
                                          tail.mutable_data());
        }
        throw_code(rc);
        return py::make_tuple(fits, tail);
      },
      py::arg("lengths"), py::arg("offsets"), py::arg("nu") = 3.5, py::arg("families") = 15u,
      "fit_report over ragged prompts (grouped by sample count on the host)");
  m.def(
      "score_rank_device",
      [](uintptr_t ctx, uintptr_t mu, uintptr_t sigma, uintptr_t max_tokens, uint64_t n,
         double alpha, double beta, uintptr_t E, uintptr_t C, uintptr_t S, uintptr_t order,
         unsigned flags, uintptr_t stream) {
        throw_code(tie_score_rank(reinterpret_cast<tie_ctx*>(ctx), (const double*)mu,
                                  (const double*)sigma, (const uint32_t*)max_tokens, n, alpha,
                                  beta, (double*)E, (double*)C, (double*)S, (uint64_t*)order,
                                  flags, vp(stream)));
      },
      py::arg("ctx"), py::arg("mu"), py::arg("sigma"), py::arg("max_tokens"), py::arg("n"),
      py::arg("alpha"), py::arg("beta"), py::arg("E"), py::arg("cvar"), py::arg("score"),
      py::arg("order"), py::arg("flags") = 0u, py::arg("stream") = 0);
  m.def(
      "fit_device",
      [](uintptr_t ctx, uintptr_t x, uint64_t P, uint64_t K, double nu, uintptr_t mu,
         uintptr_t sigma, uintptr_t ll, uintptr_t iters, uintptr_t conv, uintptr_t degen,
         uintptr_t stream) {
        throw_code(tie_fit(reinterpret_cast<tie_ctx*>(ctx), (const double*)x, P, K, nu,
                           (double*)mu, (double*)sigma, (double*)ll, (int32_t*)iters,
                           (uint8_t*)conv, (uint8_t*)degen, vp(stream)));
      },
      py::arg("ctx"), py::arg("x"), py::arg("P"), py::arg("K"), py::arg("nu"), py::arg("mu"),
      py::arg("sigma"), py::arg("ll"), py::arg("iters"), py::arg("conv"), py::arg("degen"),
      py::arg("stream") = 0);
  m.def(
      "sync",
      [](uintptr_t ctx, uintptr_t stream) {
        throw_code(tie_sync(reinterpret_cast<tie_ctx*>(ctx), vp(stream)));
      },
      py::arg("ctx"), py::arg("stream") = 0);
  m.def(
      "score_rank_host_ptr",
      [](uintptr_t ctx, uintptr_t mu, uintptr_t sigma, uintptr_t max_tokens, uint64_t n,
         double alpha, double beta, uintptr_t score, uintptr_t order, unsigned flags) {
        int rc;
        {
          py::gil_scoped_release nogil;
          rc = tie_score_rank_host(reinterpret_cast<tie_ctx*>(ctx), (const double*)mu,
                                   (const double*)sigma, (const uint32_t*)max_tokens, n, alpha,
                                   beta, (double*)score, (uint64_t*)order, flags);
        }
        throw_code(rc);
      },
      py::arg("ctx"), py::arg("mu"), py::arg("sigma"), py::arg("max_tokens"), py::arg("n"),
      py::arg("alpha"), py::arg("beta"), py::arg("score"), py::arg("order"),
      py::arg("flags") = 0u,
      "end-to-end call on raw HOST pointers (pinned buffers give full PCIe bandwidth)");
  m.def(
      "fit_host_ptr",
      [](uintptr_t ctx, uintptr_t x, uint64_t P, uint64_t K, double nu, uintptr_t mu,
         uintptr_t sigma, uintptr_t ll, uintptr_t iters, uintptr_t conv, uintptr_t degen) {
        int rc;
        {
          py::gil_scoped_release nogil;
          rc = tie_fit_host(reinterpret_cast<tie_ctx*>(ctx), (const double*)x, P, K, nu,
                            (double*)mu, (double*)sigma, (double*)ll, (int32_t*)iters,
                            (uint8_t*)conv, (uint8_t*)degen);
        }
        throw_code(rc);
      },
      py::arg("ctx"), py::arg("x"), py::arg("P"), py::arg("K"), py::arg("nu"), py::arg("mu"),
      py::arg("sigma"), py::arg("ll"), py::arg("iters"), py::arg("conv"), py::arg("degen"));
  m.def(
      "profile",
      [](uintptr_t ctx, bool enable) {
        throw_code(tie_profile(reinterpret_cast<tie_ctx*>(ctx), enable ? 1 : 0));
      },
      py::arg("ctx"), py::arg("enable"));
  m.def(
      "profile_report",
      [](uintptr_t ctx) {
        std::string buf(1 << 16, '\0');
        throw_code(tie_profile_report(reinterpret_cast<tie_ctx*>(ctx), buf.data(), buf.size()));
        py::dict out;
        size_t pos = 0;
        const std::string s(buf.c_str());
        while (pos < s.size()) {
          const size_t eol = s.find('\n', pos);
          const std::string line = s.substr(pos, eol - pos);
          pos = eol == std::string::npos ? s.size() : eol + 1;
          const size_t t1 = line.find('\t'), t2 = line.find('\t', t1 + 1);
          if (t1 == std::string::npos || t2 == std::string::npos) continue;
          out[py::str(line.substr(0, t1))] = py::make_tuple(
              std::stol(line.substr(t1 + 1, t2 - t1 - 1)), std::stod(line.substr(t2 + 1)));
        }
        return out;
      },
      py::arg("ctx"), "{kernel: (launches, total_ms)} since profile(ctx, True)");
  // GPU-resident Scheduler (sched.hpp:74-90) with batched event entry points
  struct GpuQueue {
    tie_queue* q = nullptr;
    ~GpuQueue() { tie_queue_destroy(q); }
  };
  py::class_<GpuQueue>(m, "GpuScheduler")
      .def(py::init([](const McContext& mc, Policy policy, const ScoreConfig& cfg,
                       uint64_t capacity) {
             auto* g = new GpuQueue();
             const int rc = tie_queue_create(
                 mc.handle(), (int)policy, cfg.beta_mode == BetaMode::AdaptiveLinear,
                 cfg.beta_fixed, cfg.beta_max, cfg.q_sat, cfg.rebuild_threshold, cfg.alpha,
                 capacity, &g->q);
             if (rc) {
               delete g;
               throw_code(rc);
             }
             return g;
           }),
           py::arg("mc"), py::arg("policy"), py::arg("config"), py::arg("capacity"),
           py::keep_alive<1, 2>())
      .def("on_arrival_batch",
           [](GpuQueue& g, carray<uint64_t> ids, carray<double> arrival_s,
              carray<uint32_t> max_tokens) {
             if (arrival_s.size() != ids.size() || max_tokens.size() != ids.size())
               throw py::value_error("on_arrival_batch: array lengths differ");
             throw_code(tie_queue_arrive(g.q, ids.data(), arrival_s.data(), max_tokens.data(),
                                         (uint64_t)ids.size()));
           },
           py::arg("ids"), py::arg("arrival_s"), py::arg("max_tokens"))
      .def("on_prediction_batch",
           [](GpuQueue& g, carray<uint64_t> ids, carray<double> E, carray<double> C) {
             if (E.size() != ids.size() || C.size() != ids.size())
               throw py::value_error("on_prediction_batch: array lengths differ");
             throw_code(tie_queue_predict(g.q, ids.data(), E.data(), C.data(),
                                          (uint64_t)ids.size()));
           },
           py::arg("ids"), py::arg("expectation"), py::arg("cvar"))
      .def("on_prediction_logt",
           [](GpuQueue& g, carray<uint64_t> ids, carray<double> mu, carray<double> sigma,
              carray<uint32_t> max_tokens) {
             if (mu.size() != ids.size() || sigma.size() != ids.size() ||
                 max_tokens.size() != ids.size())
               throw py::value_error("on_prediction_logt: array lengths differ");
             throw_code(tie_queue_predict_logt(g.q, ids.data(), mu.data(), sigma.data(),
                                               max_tokens.data(), (uint64_t)ids.size()));
           },
           py::arg("ids"), py::arg("mu"), py::arg("sigma"), py::arg("max_tokens"))
      .def("next_requests",
           [](GpuQueue& g, uint64_t k) {
             std::vector<uint64_t> out(k);
             uint64_t n = 0;
             throw_code(tie_queue_next(g.q, k, out.data(), &n));
             out.resize(n);
             return carray<uint64_t>((py::ssize_t)n, out.data());
           },
           py::arg("k"))
      .def("step",
           [](GpuQueue& g, carray<uint64_t> arr_ids, carray<double> arrival_s,
              carray<uint32_t> arr_max_tokens, carray<uint64_t> pred_ids, carray<double> mu,
              carray<double> sigma, carray<uint32_t> pred_max_tokens, uint64_t k) {
             if (arrival_s.size() != arr_ids.size() || arr_max_tokens.size() != arr_ids.size() ||
                 mu.size() != pred_ids.size() || sigma.size() != pred_ids.size() ||
                 pred_max_tokens.size() != pred_ids.size())
               throw py::value_error("step: array lengths differ");
             std::vector<uint64_t> out(k);
             uint64_t n = 0;
             throw_code(tie_queue_step(g.q, arr_ids.data(), arrival_s.data(),
                                       arr_max_tokens.data(), (uint64_t)arr_ids.size(),
                                       pred_ids.data(), mu.data(), sigma.data(),
                                       pred_max_tokens.data(), (uint64_t)pred_ids.size(), k,
                                       out.data(), &n));
             out.resize(n);
             return carray<uint64_t>((py::ssize_t)n, out.data());
           },
           py::arg("arr_ids"), py::arg("arrival_s"), py::arg("arr_max_tokens"),
           py::arg("pred_ids"), py::arg("mu"), py::arg("sigma"), py::arg("pred_max_tokens"),
           py::arg("k"),
           "one scheduler iteration (on_arrival x, on_prediction x, next_request x k) with one "
           "device round trip")
      .def("step_ec",
           [](GpuQueue& g, carray<uint64_t> arr_ids, carray<double> arrival_s,
              carray<uint32_t> arr_max_tokens, carray<uint64_t> pred_ids, carray<double> E,
              carray<double> C, uint64_t k) {
             if (arrival_s.size() != arr_ids.size() || arr_max_tokens.size() != arr_ids.size() ||
                 E.size() != pred_ids.size() || C.size() != pred_ids.size())
               throw py::value_error("step_ec: array lengths differ");
             std::vector<uint64_t> out(k);
             uint64_t n = 0;
             throw_code(tie_queue_step_ec(g.q, arr_ids.data(), arrival_s.data(),
                                          arr_max_tokens.data(), (uint64_t)arr_ids.size(),
                                          pred_ids.data(), E.data(), C.data(),
                                          (uint64_t)pred_ids.size(), k, out.data(), &n));
             out.resize(n);
             return carray<uint64_t>((py::ssize_t)n, out.data());
           },
           py::arg("arr_ids"), py::arg("arrival_s"), py::arg("arr_max_tokens"),
           py::arg("pred_ids"), py::arg("E"), py::arg("C"), py::arg("k"),
           "on_arrival x n, on_prediction(E, C) x m, next_request() x k: one device round trip")
      .def("step_ec_runs",
           [](GpuQueue& g, carray<uint64_t> arr_ids, carray<double> arrival_s,
              carray<uint32_t> arr_max_tokens, carray<uint64_t> arr_end,
              carray<uint64_t> pred_ids, carray<double> E, carray<double> C,
              carray<uint64_t> pred_end, uint64_t k) {
             const uint64_t nr = (uint64_t)arr_end.size();
             if (arrival_s.size() != arr_ids.size() || arr_max_tokens.size() != arr_ids.size() ||
                 E.size() != pred_ids.size() || C.size() != pred_ids.size() ||
                 pred_end.size() != arr_end.size() ||
                 (nr && (arr_end.data()[nr - 1] != (uint64_t)arr_ids.size() ||
                         pred_end.data()[nr - 1] != (uint64_t)pred_ids.size())))
               throw py::value_error("step_ec_runs: array lengths / run ends differ");
             std::vector<uint64_t> out(k);
             uint64_t n = 0;
             throw_code(tie_queue_step_ec_runs(g.q, arr_ids.data(), arrival_s.data(),
                                               arr_max_tokens.data(), arr_end.data(),
                                               pred_ids.data(), E.data(), C.data(),
                                               pred_end.data(), nr, k, out.data(), &n));
             out.resize(n);
             return carray<uint64_t>((py::ssize_t)n, out.data());
           },
           py::arg("arr_ids"), py::arg("arrival_s"), py::arg("arr_max_tokens"),
           py::arg("arr_end"), py::arg("pred_ids"), py::arg("E"), py::arg("C"),
           py::arg("pred_end"), py::arg("k"),
           "runs of (arrivals, predictions(E, C)) then next_request() x k: one device round trip")
      .def("next_request",
           [](GpuQueue& g) -> py::object {
             uint64_t id = 0, n = 0;
             throw_code(tie_queue_next(g.q, 1, &id, &n));
             if (!n) return py::none();
             return py::int_(id);
           })
      .def("rebuild_if_drifted",
           [](GpuQueue& g) {
             int r = 0;
             throw_code(tie_queue_rebuild_if_drifted(g.q, &r));
             return r != 0;
           })
      .def("set_peer_waiting",
           [](GpuQueue& g, uint64_t peers) { throw_code(tie_queue_set_peer_waiting(g.q, peers)); },
           py::arg("peers"), "beta's queue length = waiting() + peers (sharded scheduler)")
      .def("beta_range",
           [](const GpuQueue& g) {
             double lo = 0, hi = 0;
             uint64_t n = 0;
             throw_code(tie_queue_beta_range(g.q, &lo, &hi, &n));
             return py::make_tuple(lo, hi, n);
           },
           "(min beta, max beta, count) of betas_in_use_; count 0 = empty")
      .def("rebuild_at",
           [](GpuQueue& g, double beta) { throw_code(tie_queue_rebuild_at(g.q, beta)); },
           py::arg("beta"), "re-key every predicted entry at `beta` (a global rebuild)")
      .def("peek",
           [](GpuQueue& g, uint64_t k) {
             std::vector<uint64_t> keys(k), ids(k);
             uint64_t n = 0;
             throw_code(tie_queue_peek(g.q, k, keys.data(), ids.data(), &n));
             return py::make_tuple(carray<uint64_t>((py::ssize_t)n, keys.data()),
                                   carray<uint64_t>((py::ssize_t)n, ids.data()));
           },
           py::arg("k"), "(keys, ids) of the next k pops under the current keys, not popped")
      .def("waiting", [](const GpuQueue& g) { return tie_queue_size(g.q); })
      .def("current_beta", [](const GpuQueue& g) { return tie_queue_current_beta(g.q); });

  m.def(
      "sim_scores",
      [](carray<double> mu, carray<double> sigma, carray<uint64_t> ids,
         carray<uint32_t> max_tokens, const McContext& mc, PredictorKind predictor,
         double mu_sd, double log_sigma_sd, uint64_t seed, ScoreFamily family, double alpha) {
        const size_t n = (size_t)mu.size();
        carray<double> E(n), C(n);
        int rc;
        {
          py::gil_scoped_release nogil;
          rc = tie_sim_scores_host(mc.handle(), mu.data(), sigma.data(), ids.data(),
                                   max_tokens.data(), n,
                                   predictor == PredictorKind::Noisy ? 1 : 0, mu_sd,
                                   log_sigma_sd, seed, family == ScoreFamily::LogNormal ? 1 : 0,
                                   alpha, E.mutable_data(), C.mutable_data());
        }
        throw_code(rc);
        return py::make_tuple(E, C);
      },
      py::arg("mu"), py::arg("sigma"), py::arg("ids"), py::arg("max_tokens"), py::arg("mc"),
      py::arg("predictor") = PredictorKind::Oracle, py::arg("mu_sd") = 0.0,
      py::arg("log_sigma_sd") = 0.0, py::arg("seed") = 0,
      py::arg("family") = ScoreFamily::LogT, py::arg("alpha") = 0.9,
      "run_sim's scoring precompute (sim.cpp:77-96) on the GPU: (E, max(CVaR, E)) per request");

  // ------------------------------------------------------------- goodness of fit
  py::class_<KsResultPy>(m, "KsResult")
      .def_readonly("statistic", &KsResultPy::statistic)
      .def_readonly("p_value", &KsResultPy::p_value)
      .def_readonly("n", &KsResultPy::n);
  m.def(
      "ks_test_fit",
      [](const std::vector<double>& samples, const FitResult& f) {
        KsResultPy r;
        throw_code(tie_ks_test_fit_host(default_context(), samples.data(), samples.size(),
                                        (int)f.family, f.mu, f.sigma, f.nu, f.rate,
                                        &r.statistic, &r.p_value));
        r.n = (int)samples.size();
        return r;
      },
      py::arg("samples"), py::arg("fit"),
      "KS test of samples against a fitted family's CDF (GPU; fit.cpp:245-284)");
  m.def(
      "ks_test_fit_raw",
      [](carray<double> x, int family, double mu, double sigma, double nu, double rate) {
        double st = 0.0, p = 0.0;
        throw_code(tie_ks_test_fit_host(default_context(), x.data(), (uint64_t)x.size(), family,
                                        mu, sigma, nu, rate, &st, &p));
        return py::make_tuple(st, p);
      },
      py::arg("samples"), py::arg("family"), py::arg("mu") = 0.0, py::arg("sigma") = 0.0,
      py::arg("nu") = 0.0, py::arg("rate") = 0.0,
      "(statistic, p_value) of ks_test against family 0 logt / 1 logt free-nu / 2 lognormal / "
      "3 exponential with the given parameters");

  // ------------------------------------------------------------- workload (workload.hpp)
  py::class_<Request>(m, "Request")
      .def(py::init<>())
      .def_readwrite("id", &Request::id)
      .def_readwrite("arrival_s", &Request::arrival_s)
      .def_readwrite("prompt_tokens", &Request::prompt_tokens)
      .def_readwrite("true_output_tokens", &Request::true_output_tokens)
      .def_readwrite("max_tokens", &Request::max_tokens)
      .def_readwrite("true_mu", &Request::true_mu)
      .def_readwrite("true_sigma", &Request::true_sigma);
  py::class_<WorkloadSpec>(m, "WorkloadSpec")
      .def(py::init<>())
      .def_readwrite("n_requests", &WorkloadSpec::n_requests)
      .def_readwrite("rps", &WorkloadSpec::rps)
      .def_readwrite("mu_range", &WorkloadSpec::mu_range)
      .def_readwrite("sigma_range", &WorkloadSpec::sigma_range)
      .def_readwrite("nu", &WorkloadSpec::nu)
      .def_readwrite("prompt_range", &WorkloadSpec::prompt_range)
      .def_readwrite("max_tokens", &WorkloadSpec::max_tokens);
  m.def("gen_logt_workload", &gen_logt_workload, py::arg("spec"), py::arg("seed"));
  m.def("poisson_arrivals", &poisson_arrivals, py::arg("rps"), py::arg("n"), py::arg("seed"));
  m.def(
      "load_trace",
      [](const std::string& path, std::optional<double> fill_rps, uint64_t seed) {
        tie_trace* t = nullptr;
        throw_code(tie_trace_load(path.c_str(), fill_rps ? *fill_rps : 0.0, seed, &t));
        const size_t n = tie_trace_size(t);
        std::vector<Request> out(n);
        for (size_t i = 0; i < n; ++i) {
          Request& r = out[i];
          r.id = tie_trace_ids(t)[i];
          r.arrival_s = tie_trace_arrival(t)[i];
          r.prompt_tokens = tie_trace_prompt_tokens(t)[i];
          r.true_output_tokens = tie_trace_output_tokens(t)[i];
          r.max_tokens = tie_trace_max_tokens(t)[i];
          const double mu = tie_trace_mu(t)[i], sg = tie_trace_sigma(t)[i];
          if (!std::isnan(mu)) r.true_mu = mu;
          if (!std::isnan(sg)) r.true_sigma = sg;
        }
        tie_trace_free(t);
        return out;
      },
      py::arg("path"), py::arg("fill_rps") = std::optional<double>{}, py::arg("seed") = 0,
      "load_trace (workload.cpp:106-161)");
  m.def(
      "save_trace",
      [](const std::vector<Request>& reqs, const std::string& path) {
        const size_t n = reqs.size();
        std::vector<uint64_t> id(n);
        std::vector<double> arr(n), mu(n), sg(n);
        std::vector<uint32_t> pt(n), ot(n), mt(n);
        for (size_t i = 0; i < n; ++i) {
          id[i] = reqs[i].id;
          arr[i] = reqs[i].arrival_s;
          pt[i] = reqs[i].prompt_tokens;
          ot[i] = reqs[i].true_output_tokens;
          mt[i] = reqs[i].max_tokens;
          mu[i] = reqs[i].true_mu ? *reqs[i].true_mu : std::nan("");
          sg[i] = reqs[i].true_sigma ? *reqs[i].true_sigma : std::nan("");
        }
        throw_code(tie_trace_save(path.c_str(), n, id.data(), arr.data(), pt.data(), ot.data(),
                                  mt.data(), mu.data(), sg.data()));
      },
      py::arg("requests"), py::arg("path"), "save_trace (workload.cpp:94-104)");

  // ------------------------------------------------------------- WaitingQueue / Scheduler
  py::class_<QueueEntry>(m, "QueueEntry")
      .def(py::init<>())
      .def(py::init([](uint64_t id, double key, bool predicted, double e, double c, double b) {
             return QueueEntry{id, key, predicted, e, c, b};
           }),
           py::arg("req_id"), py::arg("key"), py::arg("predicted") = false,
           py::arg("expectation") = 0.0, py::arg("cvar") = 0.0, py::arg("beta_at_update") = 0.0)
      .def_readwrite("req_id", &QueueEntry::req_id)
      .def_readwrite("key", &QueueEntry::key)
      .def_readwrite("predicted", &QueueEntry::predicted)
      .def_readwrite("expectation", &QueueEntry::expectation)
      .def_readwrite("cvar", &QueueEntry::cvar)
      .def_readwrite("beta_at_update", &QueueEntry::beta_at_update);
  py::class_<WaitingQueue>(m, "WaitingQueue")
      .def(py::init<const McContext*, size_t>(), py::arg("mc") = nullptr,
           py::arg("initial_capacity") = 1024, py::keep_alive<1, 2>())
      .def("push", &WaitingQueue::push, py::arg("entry"))
      .def("update", &WaitingQueue::update, py::arg("req_id"), py::arg("key"))
      .def("pop_min", &WaitingQueue::pop_min)
      .def("contains", &WaitingQueue::contains, py::arg("req_id"))
      .def("size", &WaitingQueue::size)
      .def("empty", &WaitingQueue::empty)
      .def("__len__", &WaitingQueue::size)
      .def("at", [](const WaitingQueue& q, uint64_t id) { return q.at(id); }, py::arg("req_id"),
           "a copy of the entry (use update() to re-key)")
      .def("entries", [](const WaitingQueue& q) { return q.entries(); },
           "copies of every waiting entry (slot order)")
      .def("validate", &WaitingQueue::validate)
      .def("push_batch",
           [](WaitingQueue& q, carray<uint64_t> ids, carray<double> keys) {
             if (keys.size() != ids.size()) throw py::value_error("push_batch: lengths differ");
             std::vector<QueueEntry> e((size_t)ids.size());
             for (size_t j = 0; j < e.size(); ++j) e[j] = QueueEntry{ids.data()[j], keys.data()[j]};
             q.push_batch(e.data(), e.size());
           },
           py::arg("ids"), py::arg("keys"))
      .def("update_batch",
           [](WaitingQueue& q, carray<uint64_t> ids, carray<double> keys) {
             if (keys.size() != ids.size()) throw py::value_error("update_batch: lengths differ");
             q.update_batch(ids.data(), keys.data(), (size_t)ids.size());
           },
           py::arg("ids"), py::arg("keys"))
      .def("pop_batch",
           [](WaitingQueue& q, size_t k) {
             const std::vector<QueueEntry> v = q.pop_batch(k);
             carray<uint64_t> ids((py::ssize_t)v.size());
             carray<double> keys((py::ssize_t)v.size());
             for (size_t j = 0; j < v.size(); ++j) {
               ids.mutable_data()[j] = v[j].req_id;
               keys.mutable_data()[j] = v[j].key;
             }
             return py::make_tuple(ids, keys);
           },
           py::arg("max_pops"), "(ids, keys) of up to max_pops pop_min() calls");
  py::class_<Scheduler>(m, "Scheduler")
      .def(py::init<Policy, ScoreConfig, const McContext*, size_t>(), py::arg("policy"),
           py::arg("config"), py::arg("mc") = nullptr, py::arg("initial_capacity") = 1024,
           py::keep_alive<1, 4>())
      .def("on_arrival", &Scheduler::on_arrival, py::arg("request"))
      .def("on_prediction", &Scheduler::on_prediction, py::arg("req_id"), py::arg("expectation"),
           py::arg("cvar"))
      .def("rebuild_if_drifted", &Scheduler::rebuild_if_drifted)
      .def("next_request", &Scheduler::next_request)
      .def("waiting_on", &Scheduler::waiting_on, py::arg("req_id"))
      .def("waiting", &Scheduler::waiting)
      .def("current_beta", &Scheduler::current_beta)
      .def("policy", &Scheduler::policy)
      .def("queue", &Scheduler::queue, py::return_value_policy::reference_internal)
      .def("on_arrival_batch",
           [](Scheduler& s, const std::vector<Request>& reqs) {
             s.on_arrival_batch(reqs.data(), reqs.size());
           },
           py::arg("requests"))
      .def("on_prediction_batch",
           [](Scheduler& s, carray<uint64_t> ids, carray<double> E, carray<double> C) {
             if (E.size() != ids.size() || C.size() != ids.size())
               throw py::value_error("on_prediction_batch: array lengths differ");
             s.on_prediction_batch(ids.data(), E.data(), C.data(), (size_t)ids.size());
           },
           py::arg("ids"), py::arg("expectation"), py::arg("cvar"))
      .def("next_requests",
           [](Scheduler& s, size_t k) {
             const std::vector<uint64_t> v = s.next_requests(k);
             return carray<uint64_t>((py::ssize_t)v.size(), v.data());
           },
           py::arg("k"));

  // ------------------------------------------------------------- predictor (predictor.hpp)
  py::class_<PredictedDist>(m, "PredictedDist")
      .def_readonly("mu_hat", &PredictedDist::mu_hat)
      .def_readonly("sigma_hat", &PredictedDist::sigma_hat);
  py::class_<NoiseSpec>(m, "NoiseSpec")
      .def(py::init<>())
      .def_readwrite("mu_sd", &NoiseSpec::mu_sd)
      .def_readwrite("log_sigma_sd", &NoiseSpec::log_sigma_sd);
  py::class_<BatcherConfig>(m, "BatcherConfig")
      .def(py::init<>())
      .def_readwrite("timeout_s", &BatcherConfig::timeout_s)
      .def_readwrite("max_batch", &BatcherConfig::max_batch)
      .def_readwrite("latency_base_s", &BatcherConfig::latency_base_s)
      .def_readwrite("latency_per_item_s", &BatcherConfig::latency_per_item_s);
  m.def("oracle_predict", &oracle_predict, py::arg("request"));
  m.def("noisy_predict", &noisy_predict, py::arg("request"), py::arg("noise"), py::arg("seed"));
  m.def("point_predict", &point_predict, py::arg("request"), py::arg("noise"), py::arg("seed"),
        py::arg("mc"));
  py::class_<Submission>(m, "Submission")
      .def(py::init<uint64_t, double>(), py::arg("req_id"), py::arg("submit_s"))
      .def_readonly("req_id", &Submission::req_id)
      .def_readonly("submit_s", &Submission::submit_s);
  py::class_<PredictionReady>(m, "PredictionReady")
      .def_readonly("req_id", &PredictionReady::req_id)
      .def_readonly("ready_s", &PredictionReady::ready_s);
  m.def("batch_schedule", &batch_schedule, py::arg("submissions"), py::arg("config"));

  // ------------------------------------------------------------- simulator (sim.hpp)
  py::class_<EngineConfig>(m, "EngineConfig")
      .def(py::init<>())
      .def_readwrite("batch_slots", &EngineConfig::batch_slots)
      .def_readwrite("c0", &EngineConfig::c0)
      .def_readwrite("c1", &EngineConfig::c1)
      .def_readwrite("c2", &EngineConfig::c2);
  py::class_<PredictorConfig>(m, "PredictorConfig")
      .def(py::init<>())
      .def_readwrite("kind", &PredictorConfig::kind)
      .def_readwrite("family", &PredictorConfig::family)
      .def_readwrite("noise", &PredictorConfig::noise)
      .def_readwrite("batched", &PredictorConfig::batched)
      .def_readwrite("batcher", &PredictorConfig::batcher)
      .def_readwrite("nu", &PredictorConfig::nu)
      .def_readwrite("mc_samples", &PredictorConfig::mc_samples)
      .def_readwrite("mc_seed", &PredictorConfig::mc_seed);
  py::class_<RequestEvent>(m, "RequestEvent")
      .def_readonly("req_id", &RequestEvent::req_id)
      .def_readonly("arrival_s", &RequestEvent::arrival_s)
      .def_readonly("predict_ready_s", &RequestEvent::predict_ready_s)
      .def_readonly("admit_s", &RequestEvent::admit_s)
      .def_readonly("first_token_s", &RequestEvent::first_token_s)
      .def_readonly("completion_s", &RequestEvent::completion_s)
      .def_readonly("emitted_tokens", &RequestEvent::emitted_tokens);
  py::class_<Metrics>(m, "Metrics")
      .def_readonly("ttft_avg", &Metrics::ttft_avg)
      .def_readonly("ttft_p90", &Metrics::ttft_p90)
      .def_readonly("ptla_avg", &Metrics::ptla_avg)
      .def_readonly("ptla_p90", &Metrics::ptla_p90)
      .def_readonly("time_at_k", &Metrics::time_at_k)
      .def_readonly("throughput_at_w", &Metrics::throughput_at_w);
  py::class_<HeatmapSpec>(m, "HeatmapSpec")
      .def(py::init<>())
      .def_readwrite("time_bins", &HeatmapSpec::time_bins)
      .def_readwrite("len_bins", &HeatmapSpec::len_bins)
      .def_readwrite("time_max", &HeatmapSpec::time_max)
      .def_readwrite("len_max", &HeatmapSpec::len_max);
  py::class_<Heatmap>(m, "Heatmap")
      .def_readonly("spec", &Heatmap::spec)
      .def_readonly("counts", &Heatmap::counts);
  py::class_<SimReport>(m, "SimReport")
      .def_readonly("seed", &SimReport::seed)
      .def_readonly("policy", &SimReport::policy)
      .def_readonly("events", &SimReport::events)
      .def_readonly("metrics", &SimReport::metrics);
  m.def(
      "run_sim",
      [](const std::vector<Request>& w, Policy policy, const ScoreConfig& sc,
         const EngineConfig& ec, const PredictorConfig& pc, uint64_t seed,
         const std::vector<uint64_t>& ks, const std::vector<double>& ws, int device) {
        py::gil_scoped_release nogil;
        return run_sim(w, policy, sc, ec, pc, seed, ks, ws, device);
      },
      py::arg("workload"), py::arg("policy"), py::arg("score_config"), py::arg("engine_config"),
      py::arg("predictor_config"), py::arg("seed"), py::arg("ks") = std::vector<uint64_t>{},
      py::arg("ws") = std::vector<double>{}, py::arg("device") = 0);
  m.def("summarize", &summarize, py::arg("events"), py::arg("ks"), py::arg("ws"));
  m.def("heatmap", &heatmap, py::arg("events"), py::arg("spec"));

  m.def("default_context", []() { return (uintptr_t)default_context(); });
  m.def("launch_count", [](bool reset) { return tie_launch_count(reset ? 1 : 0); },
        py::arg("reset") = false);
  m.def(
      "gen_logt_workload_soa",
      [](size_t n, uint64_t seed, std::pair<double, double> mu_range,
         std::pair<double, double> sigma_range, double nu, std::pair<uint32_t, uint32_t> prompt,
         uint32_t max_tokens, double rps) {
        carray<double> mu(n), sg(n), arr(n);
        carray<uint32_t> mt(n), pt(n), tl(n);
        {
          py::gil_scoped_release nogil;
          gen_logt_workload_soa(n, seed, mu_range.first, mu_range.second, sigma_range.first,
                               sigma_range.second, nu, prompt.first, prompt.second, max_tokens,
                               rps, mu.mutable_data(), sg.mutable_data(), mt.mutable_data(),
                               arr.mutable_data(), pt.mutable_data(), tl.mutable_data());
        }
        py::dict d;
        d["mu"] = mu;
        d["sigma"] = sg;
        d["max_tokens"] = mt;
        d["arrival_s"] = arr;
        d["prompt_tokens"] = pt;
        d["true_output_tokens"] = tl;
        return d;
      },
      py::arg("n"), py::arg("seed"), py::arg("mu_range") = std::make_pair(3.0, 5.0),
      py::arg("sigma_range") = std::make_pair(0.5, 1.2), py::arg("nu") = 3.5,
      py::arg("prompt_range") = std::make_pair(64u, 512u), py::arg("max_tokens") = 2048u,
      py::arg("rps") = 100.0);
  m.def(
      "gen_fit_data",
      [](size_t P, size_t K, uint64_t seed, std::pair<double, double> mu_range,
         std::pair<double, double> sigma_range, double nu, bool integerise, int threads) {
        carray<double> x({(py::ssize_t)P, (py::ssize_t)K});
        carray<double> tm(P), ts(P);
        {
          py::gil_scoped_release nogil;
          gen_fit_data(P, K, seed, mu_range.first, mu_range.second, sigma_range.first,
                       sigma_range.second, nu, integerise, x.mutable_data(), tm.mutable_data(),
                       ts.mutable_data(), threads);
        }
        return py::make_tuple(x, tm, ts);
      },
      py::arg("P"), py::arg("K") = 16, py::arg("seed") = 1,
      py::arg("mu_range") = std::make_pair(3.0, 5.0),
      py::arg("sigma_range") = std::make_pair(0.5, 1.2), py::arg("nu") = 3.5,
      py::arg("integerise") = true, py::arg("threads") = 0);
}
