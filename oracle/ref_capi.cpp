// TEST INFRASTRUCTURE ONLY (oracle/_ref). Never linked into the product library.
//
// A thin extern "C" wrapper around the UNMODIFIED reference library (lspkit
// lsp_core, /root/reference/proj/src/{matrix,projector,subspace_opt}.cpp) so
// that the Python tests, the golden-vector generator and bench.py's CPU
// baseline leg can call the reference's own code through ctypes.  Everything
// here converts flat row-major arrays to/from lsp::Matrix / lsp::SparseProjector
// and forwards to the reference function named in each comment.
//
// Error convention (mirrors the exception taxonomy of proj/include/lsp/common.hpp:13-31):
//   0 ok, 1 std::invalid_argument, 2 lsp::NumericError, 3 lsp::IoError, 4 other.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "lsp/common.hpp"
#include "lsp/matrix.hpp"
#include "lsp/projector.hpp"
#include "lsp/subspace_opt.hpp"
#include "lsp/trainer.hpp"
#ifdef LSP_REF_SCHEDULE
#include "lsp/schedule_sim.hpp"
#endif

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const lsp::NumericError& e) {
    g_err = e.what();
    return 2;
  } catch (const lsp::IoError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

lsp::Matrix to_mat(int rows, int cols, const double* p) {
  return lsp::Matrix(rows, cols, std::vector<double>(p, p + static_cast<std::size_t>(rows) * cols));
}

void from_mat(const lsp::Matrix& m, double* out) {
  std::memcpy(out, m.data(), m.size() * sizeof(double));
}

lsp::SparseProjector to_proj(int n_rows, int d, int r, const int32_t* pos, const double* val) {
  lsp::SparseProjector p;
  p.n_rows = n_rows;
  p.d = d;
  p.r = r;
  const std::size_t cnt = static_cast<std::size_t>(n_rows) * r;
  p.positions.assign(pos, pos + cnt);
  p.values.assign(val, val + cnt);
  return p;
}

lsp::ProjectorPair to_pair(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                           const int32_t* qpos, const double* qval) {
  lsp::ProjectorPair pair;
  pair.p = to_proj(m, d, r, ppos, pval);
  pair.q = to_proj(n, d, r, qpos, qval);
  return pair;
}

std::vector<lsp::Matrix> to_targets(int t, int m, int n, const double* g) {
  std::vector<lsp::Matrix> out;
  const std::size_t sz = static_cast<std::size_t>(m) * n;
  for (int i = 0; i < t; ++i) out.push_back(to_mat(m, n, g + sz * i));
  return out;
}

lsp::FitConfig to_fit_cfg(double alpha, double reg_beta, double step_size, int max_steps,
                          int timeout_steps, int reg_kind) {
  lsp::FitConfig cfg;
  cfg.alpha = alpha;
  cfg.reg_beta = reg_beta;
  cfg.step_size = step_size;
  cfg.max_steps = max_steps;
  cfg.timeout_steps = timeout_steps;
  cfg.reg_kind = reg_kind ? lsp::RegKind::kUnsquared : lsp::RegKind::kSquared;
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// proj/include/lsp/common.hpp:42-45
uint64_t ref_derive_seed(uint64_t master, uint64_t tag, uint64_t index) {
  return lsp::derive_seed(master, tag, index);
}

// proj/src/projector.cpp:66-85
int ref_init_sparse(int n_rows, int d, int r, uint64_t seed, int32_t* pos, double* val) {
  return guard([&] {
    lsp::SparseProjector p = lsp::init_sparse(n_rows, d, r, seed);
    std::copy(p.positions.begin(), p.positions.end(), pos);
    std::copy(p.values.begin(), p.values.end(), val);
  });
}

// proj/src/projector.cpp:163-168
int ref_compress(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                 const int32_t* qpos, const double* qval, const double* g, double* s_out) {
  return guard([&] {
    auto pair = to_pair(m, n, d, r, ppos, pval, qpos, qval);
    from_mat(lsp::compress(pair, to_mat(m, n, g)), s_out);
  });
}

// proj/src/projector.cpp:170-175
int ref_decompress(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                   const int32_t* qpos, const double* qval, const double* s, double* out) {
  return guard([&] {
    auto pair = to_pair(m, n, d, r, ppos, pval, qpos, qval);
    from_mat(lsp::decompress(pair, to_mat(d, d, s)), out);
  });
}

// The apply step of proj/src/trainer.cpp:190: w -= decompress(pair, delta) * lr.
int ref_decompress_apply(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                         const int32_t* qpos, const double* qval, const double* delta,
                         double lr, double* w) {
  return guard([&] {
    auto pair = to_pair(m, n, d, r, ppos, pval, qpos, qval);
    lsp::Matrix wm = to_mat(m, n, w);
    wm -= lsp::decompress(pair, to_mat(d, d, delta)) * lr;
    from_mat(wm, w);
  });
}

// proj/src/projector.cpp:177-181
int ref_estimation_bias(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                        const int32_t* qpos, const double* qval, const double* sigma,
                        double* out) {
  return guard([&] {
    auto pair = to_pair(m, n, d, r, ppos, pval, qpos, qval);
    from_mat(lsp::estimation_bias(pair, to_mat(m, n, sigma)), out);
  });
}

// proj/src/projector.cpp:183-187
int ref_relative_bias(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                      const int32_t* qpos, const double* qval, const double* sigma,
                      double* out) {
  return guard([&] {
    auto pair = to_pair(m, n, d, r, ppos, pval, qpos, qval);
    *out = lsp::relative_bias(pair, to_mat(m, n, sigma));
  });
}

// proj/src/subspace_opt.cpp:35-57 (state is value-in / value-out, like AdamResult)
int ref_adam_step(int rows, int cols, int64_t step, double beta1, double beta2, double eps,
                  const double* m_in, const double* v_in, const double* grad, double* m_out,
                  double* v_out, double* delta, int64_t* step_out) {
  return guard([&] {
    lsp::SubspaceOptState st = lsp::make_opt_state(rows, cols, beta1, beta2, eps);
    st.m = to_mat(rows, cols, m_in);
    st.v = to_mat(rows, cols, v_in);
    st.step = step;
    lsp::AdamResult res = lsp::adam_step(st, to_mat(rows, cols, grad));
    from_mat(res.state.m, m_out);
    from_mat(res.state.v, v_out);
    from_mat(res.delta, delta);
    *step_out = res.state.step;
  });
}

// proj/src/projector.cpp:189-198
int ref_fit_loss(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                 const int32_t* qpos, const double* qval, int t, const double* targets,
                 double reg_beta, int reg_kind, double* out) {
  return guard([&] {
    auto pair = to_pair(m, n, d, r, ppos, pval, qpos, qval);
    auto cfg = to_fit_cfg(0.1, reg_beta, 1e-2, 500, 500, reg_kind);
    *out = lsp::fit_loss(pair, to_targets(t, m, n, targets), cfg);
  });
}

// proj/src/projector.cpp:200-236
int ref_fit_gradient(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                     const int32_t* qpos, const double* qval, int t, const double* targets,
                     double reg_beta, int reg_kind, double* gp, double* gq) {
  return guard([&] {
    auto pair = to_pair(m, n, d, r, ppos, pval, qpos, qval);
    auto cfg = to_fit_cfg(0.1, reg_beta, 1e-2, 500, 500, reg_kind);
    lsp::FitGradient g = lsp::fit_gradient(pair, to_targets(t, m, n, targets), cfg);
    std::copy(g.wrt_p.begin(), g.wrt_p.end(), gp);
    std::copy(g.wrt_q.begin(), g.wrt_q.end(), gq);
  });
}

// proj/src/projector.cpp:253-315.  pval/qval are updated in place with the
// fitted values; report = {final_rel_bias, success, timed_out, stalled, steps,
// n_loss}; loss_curve receives up to max_curve entries.
int ref_fit(int m, int n, int d, int r, const int32_t* ppos, double* pval, const int32_t* qpos,
            double* qval, int t, const double* targets, double alpha, double reg_beta,
            double step_size, int max_steps, int timeout_steps, int reg_kind, double* report,
            double* loss_curve, int max_curve) {
  return guard([&] {
    auto pair = to_pair(m, n, d, r, ppos, pval, qpos, qval);
    auto cfg = to_fit_cfg(alpha, reg_beta, step_size, max_steps, timeout_steps, reg_kind);
    auto [fitted, rep] = lsp::fit(pair, to_targets(t, m, n, targets), cfg);
    std::copy(fitted.p.values.begin(), fitted.p.values.end(), pval);
    std::copy(fitted.q.values.begin(), fitted.q.values.end(), qval);
    report[0] = rep.final_rel_bias;
    report[1] = rep.success ? 1.0 : 0.0;
    report[2] = rep.timed_out ? 1.0 : 0.0;
    report[3] = rep.stalled ? 1.0 : 0.0;
    report[4] = rep.steps;
    report[5] = static_cast<double>(rep.loss_curve.size());
    const int nc = std::min<int>(max_curve, static_cast<int>(rep.loss_curve.size()));
    for (int i = 0; i < nc; ++i) loss_curve[i] = rep.loss_curve[i];
  });
}

// proj/src/subspace_opt.cpp:59-70
int ref_projector_gram(int n_rows, int da, int ra, const int32_t* apos, const double* aval,
                       int db, int rb, const int32_t* bpos, const double* bval, double* out) {
  return guard([&] {
    from_mat(lsp::projector_gram(to_proj(n_rows, da, ra, apos, aval),
                                 to_proj(n_rows, db, rb, bpos, bval)),
             out);
  });
}

// proj/src/subspace_opt.cpp:72-101; old/new pairs share m, n, d, r.
int ref_reproject_state(int m, int n, int d, int r, const int32_t* oppos, const double* opval,
                        const int32_t* oqpos, const double* oqval, const int32_t* nppos,
                        const double* npval, const int32_t* nqpos, const double* nqval,
                        const double* m_in, const double* v_in, int kind, double* m_out,
                        double* v_out) {
  return guard([&] {
    auto oldp = to_pair(m, n, d, r, oppos, opval, oqpos, oqval);
    auto newp = to_pair(m, n, d, r, nppos, npval, nqpos, nqval);
    lsp::SubspaceOptState st = lsp::make_opt_state(d);
    st.m = to_mat(d, d, m_in);
    st.v = to_mat(d, d, v_in);
    auto out = lsp::reproject_state(st, oldp, newp,
                                    kind ? lsp::TransferKind::kMatrixSquare
                                         : lsp::TransferKind::kEntrywiseSquare);
    from_mat(out.m, m_out);
    from_mat(out.v, v_out);
  });
}

// proj/src/projector.cpp:317-327 -> text; returns needed size (incl. NUL).
int64_t ref_save_projector(int n_rows, int d, int r, const int32_t* pos, const double* val,
                           char* buf, int64_t cap) {
  std::ostringstream out;
  lsp::save_projector(to_proj(n_rows, d, r, pos, val), out);
  const std::string s = out.str();
  if (buf && cap > 0) {
    const int64_t nc = std::min<int64_t>(cap - 1, static_cast<int64_t>(s.size()));
    std::memcpy(buf, s.data(), nc);
    buf[nc] = '\0';
  }
  return static_cast<int64_t>(s.size()) + 1;
}

// proj/src/trainer.cpp:60-72
int ref_subsample_size(double gamma, double beta, int m, int n, int total_steps, double delta,
                       int64_t* out) {
  return guard([&] { *out = lsp::subsample_size(gamma, beta, m, n, total_steps, delta); });
}

// CPU baseline: one hot-path step (proj/src/trainer.cpp:187-190) on `count`
// independent matrices of one shape, fanned out over `threads` std::threads
// (the reference functions are pure).  Inputs are built once
// per call (outside the timed region) from the given flat arrays shared by all
// matrices; returns the wall seconds of the timed region in *seconds.
int ref_time_step(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                  const int32_t* qpos, const double* qval, const double* g, const double* w0,
                  double lr, int count, int threads, double* seconds) {
  return guard([&] {
    auto pair = to_pair(m, n, d, r, ppos, pval, qpos, qval);
    const lsp::Matrix gm = to_mat(m, n, g);
    std::vector<lsp::Matrix> ws(count, to_mat(m, n, w0));
    std::vector<lsp::SubspaceOptState> st(count, lsp::make_opt_state(d));
    const int nt = std::max(1, std::min(threads, count));
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int tid = 0; tid < nt; ++tid) {
      pool.emplace_back([&, tid] {
        for (int i = tid; i < count; i += nt) {
          lsp::Matrix s = lsp::compress(pair, gm);
          auto res = lsp::adam_step(st[i], s);
          st[i] = std::move(res.state);
          ws[i] -= lsp::decompress(pair, res.delta) * lr;
        }
      });
    }
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

// proj/src/trainer.cpp:74-112 (maybe_update), the reference's own code.
// state = {m_in, v_in, step}; on refresh the new pair (r nonzeros per row) is
// written to np_*/nq_* and the reprojected state to m_out/v_out (unchanged
// copies otherwise).  result = {refreshed, fit_timed_out, skipped_zero_grad,
// bias_before, bias_after, fit_steps}.
int ref_maybe_update(int m, int n, int d, int r_old, const int32_t* ppos, const double* pval,
                     const int32_t* qpos, const double* qval, const double* m_in,
                     const double* v_in, int64_t step, const double* grad, int n_extra,
                     const double* extra, int r, double alpha, double fit_alpha, double reg_beta,
                     double step_size,
                     int max_steps, int timeout_steps, int reg_kind, int transfer,
                     uint64_t reinit_seed, int32_t* np_pos, double* np_val, int32_t* nq_pos,
                     double* nq_val, double* m_out, double* v_out, double* result) {
  return guard([&] {
    auto pair = to_pair(m, n, d, r_old, ppos, pval, qpos, qval);
    lsp::SubspaceOptState st = lsp::make_opt_state(d);
    st.m = to_mat(d, d, m_in);
    st.v = to_mat(d, d, v_in);
    st.step = step;
    lsp::TrainConfig cfg;
    cfg.r = r;
    cfg.alpha = alpha;
    cfg.fit = to_fit_cfg(fit_alpha, reg_beta, step_size, max_steps, timeout_steps, reg_kind);
    cfg.transfer = transfer ? lsp::TransferKind::kMatrixSquare : lsp::TransferKind::kEntrywiseSquare;
    const auto out = lsp::maybe_update(to_mat(m, n, grad), pair, st, cfg,
                                       to_targets(n_extra, m, n, extra), reinit_seed);
    const int rr = out.pair.p.r;
    std::copy(out.pair.p.positions.begin(), out.pair.p.positions.end(), np_pos);
    std::copy(out.pair.p.values.begin(), out.pair.p.values.end(), np_val);
    std::copy(out.pair.q.positions.begin(), out.pair.q.positions.end(), nq_pos);
    std::copy(out.pair.q.values.begin(), out.pair.q.values.end(), nq_val);
    (void)rr;
    from_mat(out.state.m, m_out);
    from_mat(out.state.v, v_out);
    result[0] = out.refreshed ? 1.0 : 0.0;
    result[1] = out.fit_timed_out ? 1.0 : 0.0;
    result[2] = out.skipped_zero_grad ? 1.0 : 0.0;
    result[3] = out.bias_before;
    result[4] = out.bias_after;
    result[5] = out.fit_steps;
  });
}

}  // extern "C"

#ifdef LSP_REF_SCHEDULE
// proj/src/schedule_sim.cpp: the schedule model on a profile given as arrays
// (vecs: fwd_gpu, bwd_gpu, upd_gpu, fwd_cpu, bwd_cpu, upd_cpu, grad_bytes,
// delta_bytes, each n_layers long, concatenated).  out[0] transition_layer
// (:373-395), out[1] closed_form_lsp(d) (:407-422; NaN when d < 1),
// out[2] closed_form_zero (:397-405), out[3] simulate(lsp_layerwise, iters)
// iter_time, out[4] simulate(zero, iters) iter_time.
extern "C" int ref_schedule_eval(int n_layers, const double* vecs, double bw_d2h, double bw_h2d,
                                 int duplex, double bytes_per_element, int d, int iters,
                                 double* out) {
  return guard([&] {
    lsp::TimingProfile p;
    p.n_layers = n_layers;
    std::vector<double>* fields[] = {&p.fwd_gpu, &p.bwd_gpu, &p.upd_gpu, &p.fwd_cpu,
                                     &p.bwd_cpu, &p.upd_cpu, &p.grad_bytes, &p.delta_bytes};
    for (int k = 0; k < 8; ++k) fields[k]->assign(vecs + k * n_layers, vecs + (k + 1) * n_layers);
    p.bandwidth_d2h = bw_d2h;
    p.bandwidth_h2d = bw_h2d;
    p.duplex = duplex != 0;
    p.bytes_per_element = bytes_per_element;
    out[0] = lsp::transition_layer(p);
    out[1] = d >= 1 ? lsp::closed_form_lsp(p, d) : std::nan("");
    out[2] = lsp::closed_form_zero(p);
    out[3] = lsp::simulate(p, lsp::Policy::kLspLayerwise, iters).iter_time;
    out[4] = lsp::simulate(p, lsp::Policy::kZero, iters).iter_time;
  });
}

// load_profile (:456-505) on a JSON file, then simulate(lsp_layerwise).
extern "C" int ref_schedule_file(const char* path, int iters, double* out) {
  return guard([&] {
    const lsp::TimingProfile p = lsp::load_profile(path);
    out[0] = p.n_layers;
    out[1] = lsp::transition_layer(p);
    out[2] = lsp::simulate(p, lsp::Policy::kLspLayerwise, iters).iter_time;
  });
}
#endif
