// engine_ext.cu -- C ABI entry points beyond the core SGD / LSQR path, on the
// same device matrix: the symmetric / block variants (src/variants.cpp), the
// Chambolle-Pock lasso and spectral_norm (src/ccp.cpp, src/lsqr.cpp:140-163),
// the public helpers of equilibrate.hpp / metrics.hpp, and the matrix store
// (Matrix Market and binary CSR files, src/matrix_market.cpp).
#include "engine_internal.h"

// ---------------------------------------------------------------------------
// Engine variants (src/variants.cpp): symmetric (:35-103) and block
// (:156-240) equilibration.  Same sign stream, the same projected-SGD update
// (run_projected_sgd) and the same estimator arithmetic as sgd_row_col, but
// the passes run as generic pass kernels (kPassEst) between small kernels that
// form the scalings, sum estimates over blocks and update the block iterates.
// Single GPU; sparse and dense matrices (history for sparse ones).
// ---------------------------------------------------------------------------
namespace {

// SeededRng (src/rng.cpp:9-49) on the host: the symmetry check's probe
// normals (Box-Muller with the spare kept; glibc log/sin/cos like the
// reference build).
struct HostRng {
  uint64_t mt[eqb::mt::kN];
  int i = eqb::mt::kN;
  bool has_spare = false;
  double spare = 0.0;
  HostRng(uint64_t seed, uint64_t stream) { eqb::mt::seed_state(seed, stream, mt); }
  uint64_t next() {
    if (i >= eqb::mt::kN) {
      constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
      for (int k = 0; k < eqb::mt::kN; ++k) {
        const uint64_t x = (mt[k] & kUpper) | (mt[(k + 1) % eqb::mt::kN] & kLower);
        uint64_t xa = x >> 1;
        if (x & 1u) xa ^= 0xB5026F5AA96619E9ULL;
        mt[k] = mt[(k + eqb::mt::kM) % eqb::mt::kN] ^ xa;
      }
      i = 0;
    }
    return eqb::mt::temper(mt[i++]);
  }
  double uniform01() { return (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53; }
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = uniform01(), u2 = uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(theta);
    has_spare = true;
    return r * std::cos(theta);
  }
};

enum class Variant { kSymmetric, kBlock };

// check_symmetry (src/variants.cpp:14-33) with device applies and canonical
// dots / norms; the probes come from stream 18 (streams::kSymmetryCheck).
void check_symmetry(equil_matrix* M, uint64_t seed) {
  const int64_t n = M->n;
  cudaStream_t s = M->stream;
  HostRng rng(seed, 18);
  std::vector<double> x(n), y(n);
  DevBuf<double> xd, yd, ax, ay, t;
  xd.alloc(n); yd.alloc(n); ax.alloc(n); ay.alloc(n); t.alloc(n);
  double* sc = M->scal.p + 32;
  for (int probe = 0; probe < 3; ++probe) {
    for (int64_t i = 0; i < n; ++i) x[i] = rng.normal();
    for (int64_t i = 0; i < n; ++i) y[i] = rng.normal();
    CK(cudaMemcpyAsync(xd.p, x.data(), n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(yd.p, y.data(), n * 8, cudaMemcpyHostToDevice, s));
    apply_pass(M, false, xd.p, ax.p, eqb::kPassPlain, nullptr, nullptr, nullptr);
    apply_pass(M, false, yd.p, ay.p, eqb::kPassPlain, nullptr, nullptr, nullptr);
    CK(eqb::launch_mul(t.p, ax.p, yd.p, n, s));
    canon_reduce(M, t.p, n, sc + 0, 1);  // ax.dot(y)
    CK(eqb::launch_mul(t.p, xd.p, ay.p, n, s));
    canon_reduce(M, t.p, n, sc + 1, 1);  // x.dot(ay)
    canon_reduce(M, ax.p, n, sc + 2, 0, 0.0, true);
    canon_reduce(M, yd.p, n, sc + 3, 0, 0.0, true);
    canon_reduce(M, xd.p, n, sc + 4, 0, 0.0, true);
    canon_reduce(M, ay.p, n, sc + 5, 0, 0.0, true);
    double r[6];
    CK(cudaMemcpyAsync(r, sc, sizeof r, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double scale = r[2] * r[3] + r[4] * r[5] + 1e-30;
    require(std::abs(r[0] - r[1]) <= 1e-10 * scale,
            "sgd_equilibrate_symmetric: operator failed symmetry check");
  }
}

void sgd_variant(equil_matrix* M, Variant kind, const equil_params* p,
                 const equil_diag_cfg* diag, equil_scaling_out* out, const int64_t* rb_host,
                 const int64_t* cb_host, int64_t R, int64_t C) {
  std::lock_guard<std::mutex> lk(M->mu);
  DeviceGuard dg(M->device);
  const bool sym = kind == Variant::kSymmetric;
  const char* who = sym ? "sgd_equilibrate_symmetric" : "sgd_equilibrate_block";
  require(M->world == 1, std::string(who) + ": single-GPU matrices only in this build");
  validate_params(*p);
  const int64_t m = M->m, n = M->n;
  double alpha = 0, beta = 0;
  std::vector<int32_t> rbm, cbm;
  std::vector<double> rcount, ccount;
  if (sym) {
    require(m == n, "sgd_equilibrate_symmetric: operator must be square");
    check_symmetry(M, p->seed);
    resolve_targets(*p, n, n, alpha, beta);
    require(std::abs(alpha - beta) <= 1e-12 * std::max(alpha, beta),
            "sgd_equilibrate_symmetric: targets must coincide");
    R = n;
    C = 0;
  } else {  // BlockStructure::validate (src/variants.cpp:131-154)
    require(rb_host != nullptr && cb_host != nullptr, "BlockStructure: assignment length mismatch");
    require(R > 0 && C > 0, "BlockStructure: block counts must be positive");
    require(R < (1LL << 31) && C < (1LL << 31), "BlockStructure: too many blocks");
    rcount.assign(R, 0.0);
    ccount.assign(C, 0.0);
    rbm.resize(m);
    cbm.resize(n);
    for (int64_t i = 0; i < m; ++i) {
      require(rb_host[i] >= 0 && rb_host[i] < R, "BlockStructure: row block index out of range");
      rbm[i] = static_cast<int32_t>(rb_host[i]);
    }
    for (int64_t j = 0; j < n; ++j) {
      require(cb_host[j] >= 0 && cb_host[j] < C, "BlockStructure: col block index out of range");
      cbm[j] = static_cast<int32_t>(cb_host[j]);
    }
    for (int64_t i = 0; i < m; ++i) rcount[rbm[i]] += 1.0;  // :165-169
    for (int64_t j = 0; j < n; ++j) ccount[cbm[j]] += 1.0;
    for (int64_t b = 0; b < R; ++b) require(rcount[b] != 0.0, "BlockStructure: empty row block");
    for (int64_t b = 0; b < C; ++b) require(ccount[b] != 0.0, "BlockStructure: empty col block");
    resolve_targets(*p, m, n, alpha, beta);
  }
  const int stride = diag ? diag->stride : 0;
  require(stride >= 0, std::string(who) + ": stride must be positive");
  const int T = p->iterations;
  const int nrec = stride ? T / stride + 1 : 0;
  if (stride) {
    require(!M->dense, std::string(who) + ": history is implemented for sparse matrices");
    require(out->hist_cap >= nrec, std::string(who) + ": history capacity too small");
  }
  cudaStream_t s = M->stream;
  const double gamma = p->gamma, Mx = p->max_log_scale;

  // signs: n per iteration (symmetric: one probe) or n + m (s then w)
  const uint64_t per_iter = static_cast<uint64_t>(sym ? n : n + m);
  const uint64_t total = per_iter * static_cast<uint64_t>(T);
  if (total > 0) {
    M->signs.ensure((total + 31) / 32 + 1);
    const size_t sb = eqb::sign_stream_scratch_bytes(total);
    M->sign_scratch.ensure(sb);
    CK(eqb::sign_stream_generate(p->seed, 17, total, M->signs.p, M->sign_scratch.p, sb, s));
  }
  // block iterates, linear terms, scalings, probes, estimates
  DevBuf<double> xu, xub, xv, xvb, lu, lv, d, e, xs, xw, er, ec, ebu, ebv;
  DevBuf<int32_t> rbd, cbd, memr, memc;
  DevBuf<int64_t> offr, offc;
  xu.alloc(R); xub.alloc(R); lu.alloc(R);
  d.alloc(m); e.alloc(n); xs.alloc(n); xw.alloc(m); er.alloc(m); ec.alloc(n);
  CK(cudaMemsetAsync(xu.p, 0, R * 8, s));
  CK(cudaMemsetAsync(xub.p, 0, R * 8, s));
  {
    std::vector<double> l(R);
    for (int64_t b = 0; b < R; ++b) l[b] = sym ? alpha * alpha : (alpha * alpha) * rcount[b];
    CK(cudaMemcpyAsync(lu.p, l.data(), R * 8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  if (!sym) {
    xv.alloc(C); xvb.alloc(C); lv.alloc(C); ebu.alloc(R); ebv.alloc(C);
    CK(cudaMemsetAsync(xv.p, 0, C * 8, s));
    CK(cudaMemsetAsync(xvb.p, 0, C * 8, s));
    std::vector<double> l(C);
    for (int64_t b = 0; b < C; ++b) l[b] = (beta * beta) * ccount[b];
    h2d_sync(s, lv.p, l.data(), C * 8);
    // members of every block in ascending index order (stable counting sort)
    auto members = [s](const std::vector<int32_t>& map, int64_t nb, DevBuf<int32_t>& mem,
                      DevBuf<int64_t>& off) {
      std::vector<int64_t> o(nb + 1, 0);
      for (int32_t b : map) ++o[b + 1];
      for (int64_t b = 0; b < nb; ++b) o[b + 1] += o[b];
      std::vector<int32_t> list(map.size());
      std::vector<int64_t> pos(o.begin(), o.end() - 1);
      for (size_t i = 0; i < map.size(); ++i) list[pos[map[i]]++] = static_cast<int32_t>(i);
      mem.alloc(list.size());
      off.alloc(o.size());
      h2d_sync(s, mem.p, list.data(), list.size() * 4);
      h2d_sync(s, off.p, o.data(), o.size() * 8);
    };
    members(rbm, R, memr, offr);
    members(cbm, C, memc, offc);
    rbd.alloc(m);
    cbd.alloc(n);
    h2d_sync(s, rbd.p, rbm.data(), m * 4);
    h2d_sync(s, cbd.p, cbm.data(), n * 4);
  }
  CK(cudaMemsetAsync(M->flags.p, 0, sizeof(unsigned), s));
  eqb::SgdBlockConst c{};
  c.gamma = gamma;
  c.M = Mx;

  // history (src/variants.cpp:66-86, :197-214) at the expanded averages
  constexpr int kRec = 6;
  DevBuf<double> hist, terms, uf, vf, eu, ev;
  if (nrec) {
    hist.alloc(kRec * nrec);
    terms.alloc(m + n);
    uf.alloc(m); vf.alloc(n); eu.alloc(m); ev.alloc(n);
  }
  const double a2 = alpha * alpha, b2 = sym ? alpha * alpha : beta * beta;
  const double beta_rms = sym ? alpha : beta;
  auto expand_avg = [&]() {
    if (sym) {
      CK(cudaMemcpyAsync(uf.p, xub.p, n * 8, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(vf.p, xub.p, n * 8, cudaMemcpyDeviceToDevice, s));
    } else {
      CK(eqb::launch_gather_map(xub.p, rbd.p, m, uf.p, s));
      CK(eqb::launch_gather_map(xvb.p, cbd.p, n, vf.p, s));
    }
  };
  int rec = 0;
  auto record = [&]() {
    double* slot = hist.p + kRec * rec;
    expand_avg();
    CK(eqb::launch_exp(uf.p, eu.p, m, 2.0, s));
    CK(eqb::launch_exp(vf.p, ev.p, n, 2.0, s));
    CK(eqb::launch_rms_terms(0, M->A, eu.p, ev.p, terms.p, 0, alpha, s));
    CK(eqb::launch_rms_terms(1, M->AT, eu.p, ev.p, terms.p + m, 0, beta_rms, s));
    canon_reduce(M, terms.p, m + n, slot + 0, 1);
    CK(eqb::launch_obj_terms(M->A, uf.p, vf.p, terms.p, s));
    canon_reduce(M, terms.p, m, slot + 1, 1);
    canon_reduce(M, uf.p, m, slot + 2, 2, a2);
    canon_reduce(M, vf.p, n, slot + 3, 2, b2);
    canon_reduce(M, uf.p, m, slot + 4, 0);
    canon_reduce(M, vf.p, n, slot + 5, 0);
    ++rec;
  };
  if (stride) record();
  for (int t = 1; t <= T; ++t) {
    eqb::SgdStep st;
    st.step = 2.0 / (gamma * static_cast<double>(t + 1));
    st.aw = 2.0 / (static_cast<double>(t) + 2.0);
    st.aw1 = 1.0 - st.aw;
    st.pad = 0;
    const int64_t base = static_cast<int64_t>(t - 1) * static_cast<int64_t>(per_iter);
    if (sym) {  // d = exp(u); est = (d .* A (d .* s))^2 (:60-64)
      CK(eqb::launch_expand_scale(xu.p, nullptr, n, M->signs.p, base, d.p, xs.p, s));
      apply_pass(M, false, xs.p, er.p, eqb::kPassEst, d.p, nullptr, nullptr);
      CK(eqb::launch_sgd_update(xu.p, xub.p, er.p, lu.p, c, st, n, M->flags.p, s));
    } else {  // :181-194
      CK(eqb::launch_expand_scale(xv.p, cbd.p, n, M->signs.p, base, e.p, xs.p, s));
      CK(eqb::launch_expand_scale(xu.p, rbd.p, m, M->signs.p, base + n, d.p, xw.p, s));
      apply_pass(M, false, xs.p, er.p, eqb::kPassEst, d.p, nullptr, nullptr);
      apply_pass(M, true, xw.p, ec.p, eqb::kPassEst, e.p, nullptr, nullptr);
      CK(eqb::launch_block_sum(er.p, memr.p, offr.p, R, ebu.p, s));
      CK(eqb::launch_block_sum(ec.p, memc.p, offc.p, C, ebv.p, s));
      CK(eqb::launch_sgd_update(xu.p, xub.p, ebu.p, lu.p, c, st, R, M->flags.p, s));
      CK(eqb::launch_sgd_update(xv.p, xvb.p, ebv.p, lv.p, c, st, C, M->flags.p, s));
    }
    if (stride && t % stride == 0) record();
  }
  // result: expanded averages and their exponentials (:93-96, :226-229)
  DevBuf<double> ufin, vfin, dfin, efin;
  ufin.alloc(m); vfin.alloc(n); dfin.alloc(m); efin.alloc(n);
  if (sym) {
    CK(cudaMemcpyAsync(ufin.p, xub.p, n * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(vfin.p, xub.p, n * 8, cudaMemcpyDeviceToDevice, s));
  } else {
    CK(eqb::launch_gather_map(xub.p, rbd.p, m, ufin.p, s));
    CK(eqb::launch_gather_map(xvb.p, cbd.p, n, vfin.p, s));
  }
  CK(eqb::launch_exp(ufin.p, dfin.p, m, 1.0, s));
  CK(eqb::launch_exp(vfin.p, efin.p, n, 1.0, s));
  const cudaMemcpyKind k =
      out->outputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (out->u) CK(cudaMemcpyAsync(out->u, ufin.p, m * 8, k, s));
  if (out->v) CK(cudaMemcpyAsync(out->v, vfin.p, n * 8, k, s));
  if (out->d) CK(cudaMemcpyAsync(out->d, dfin.p, m * 8, k, s));
  if (out->e) CK(cudaMemcpyAsync(out->e, efin.p, n * 8, k, s));
  unsigned flags = 0;
  CK(cudaMemcpyAsync(&flags, M->flags.p, sizeof flags, cudaMemcpyDeviceToHost, s));
  std::vector<double> hh(kRec * static_cast<size_t>(std::max(nrec, 1)));
  if (nrec) CK(cudaMemcpyAsync(hh.data(), hist.p, kRec * nrec * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  out->alpha = alpha;
  out->beta = sym ? alpha : beta;
  out->iterate_bound_ok = (flags & 1u) ? 0 : 1;
  out->box_feasible = (flags & 2u) ? 0 : 1;
  out->apply_count = T;
  out->adjoint_count = sym ? 0 : T;
  out->hist_len = nrec;
  for (int h = 0; h < nrec; ++h) {
    const double* r = hh.data() + kRec * h;
    const double obj = 0.5 * r[1] - r[2] - r[3] + 0.5 * gamma * (r[4] + r[5]);
    if (out->hist_iter) out->hist_iter[h] = h * stride;
    if (out->hist_objective)  // symmetric: each unordered pair once (:75-78)
      out->hist_objective[h] = (diag->want_objective ? (sym ? 0.5 * obj : obj) : 0.0);
    if (out->hist_rms)
      out->hist_rms[h] = diag->want_rms ? std::sqrt(r[0] / static_cast<double>(m + n)) : 0.0;
  }
}

}  // namespace

extern "C" {

equil_status equil_sgd_equilibrate_symmetric(equil_matrix* M, const equil_params* p,
                                             const equil_diag_cfg* diag,
                                             equil_scaling_out* out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:sgd_equilibrate_symmetric");
    require(M != nullptr && p != nullptr && out != nullptr,
            "sgd_equilibrate_symmetric: null argument");
    sgd_variant(M, Variant::kSymmetric, p, diag, out, nullptr, nullptr, 0, 0);
  });
}

equil_status equil_sgd_equilibrate_block(equil_matrix* M, const int64_t* row_block,
                                         const int64_t* col_block, int64_t row_blocks,
                                         int64_t col_blocks, const equil_params* p,
                                         const equil_diag_cfg* diag, equil_scaling_out* out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:sgd_equilibrate_block");
    require(M != nullptr && p != nullptr && out != nullptr,
            "sgd_equilibrate_block: null argument");
    sgd_variant(M, Variant::kBlock, p, diag, out, row_block, col_block, row_blocks, col_blocks);
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// spectral_norm (src/lsqr.cpp:140-163) and the Chambolle-Pock lasso
// (src/ccp.cpp:27-160): the second consumer of the equilibration's d, e.
// Device vectors, canonical reductions; the lasso objective of every iterate
// is evaluated on the device into a history array, so a run without an early
// stop test synchronises only at its end.  Single GPU.
// ---------------------------------------------------------------------------
namespace {

// power iteration on diag(d) A diag(e) (d, e null: A), uncharged
double spectral_norm_dev(equil_matrix* M, const double* d, const double* e, int max_iters,
                         double rel_tol, uint64_t seed) {
  require(max_iters > 0, "spectral_norm: max_iters must be positive");
  const int64_t m = M->m, n = M->n;
  cudaStream_t s = M->stream;
  HostRng rng(seed, 19);  // streams::kPowerIteration
  std::vector<double> xh(n);
  for (int64_t j = 0; j < n; ++j) xh[j] = rng.normal();
  DevBuf<double> x, y, z, t;
  x.alloc(n); y.alloc(m); z.alloc(n); t.alloc(std::max(m, n));
  double* sc = M->scal.p + 40;
  CK(cudaMemcpyAsync(x.p, xh.data(), n * 8, cudaMemcpyHostToDevice, s));
  canon_reduce(M, x.p, n, sc + 0, 0, 0.0, true);
  const double xn = read_scalar(M, sc + 0);
  if (!(xn > 0.0)) fail(EQUIL_ERUNTIME, "spectral_norm: degenerate start");
  CK(eqb::launch_lsqr_normalize(x.p, x.p, sc + 0, nullptr, nullptr, n, nullptr, nullptr, s));
  double lambda = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    const double* xg = x.p;
    if (e) {
      CK(eqb::launch_mul(t.p, e, x.p, n, s));
      xg = t.p;
    }
    apply_pass(M, false, xg, y.p, eqb::kPassScaled, d, nullptr, nullptr);
    canon_reduce(M, y.p, m, sc + 1, 0);
    const double next = read_scalar(M, sc + 1);
    if (next == 0.0) return 0.0;
    const bool settled = std::abs(next - lambda) <= rel_tol * next;
    lambda = next;
    if (settled) break;
    const double* yg = y.p;
    if (d) {
      CK(eqb::launch_mul(t.p, d, y.p, m, s));
      yg = t.p;
    }
    apply_pass(M, true, yg, z.p, eqb::kPassScaled, e, nullptr, nullptr);
    canon_reduce(M, z.p, n, sc + 2, 0, 0.0, true);
    const double zn = read_scalar(M, sc + 2);
    if (zn == 0.0) break;
    CK(eqb::launch_lsqr_normalize(x.p, z.p, sc + 2, nullptr, nullptr, n, nullptr, nullptr, s));
  }
  return std::sqrt(lambda);
}

// lasso_objective (src/ccp.cpp:115-123) of device x into *out (device)
void lasso_value_dev(equil_matrix* M, const double* b_d, double sqrt_lambda, const double* x,
                     const double* absx, double* r, double* out) {
  apply_pass(M, false, x, r, eqb::kPassResid, nullptr, b_d, nullptr);  // b - Ax: same squares
  double* sc = M->scal.p + 44;
  canon_reduce(M, r, M->m, sc + 0, 0);
  canon_reduce(M, absx, M->n, sc + 1, 1);
  CK(eqb::launch_lasso_value(sc + 0, sc + 1, sqrt_lambda, out, M->stream));
}

void ccp_common(equil_matrix* M, const double* b, double lambda, const equil_params* p,
                const equil_ccp_options* o, equil_ccp_out* out, const char* who) {
  require(M != nullptr && o != nullptr && out != nullptr, std::string(who) + ": null argument");
  require(b != nullptr, "lasso: rhs length mismatch");
  std::lock_guard<std::mutex> lk(M->mu);
  DeviceGuard dg(M->device);
  require(M->world == 1, std::string(who) + ": single-GPU matrices only in this build");
  cudaStream_t s = M->stream;
  const int64_t m = M->m, n = M->n;
  // validate_problem (:11-17)
  require(lambda > 0.0, "lasso: lambda must be positive");
  DevBuf<double> b_d;
  b_d.alloc(m);
  CK(cudaMemcpyAsync(b_d.p, b, m * 8, cudaMemcpyHostToDevice, s));
  canon_reduce(M, b_d.p, m, M->scal.p + 48, 0, 0.0, true);
  require(read_scalar(M, M->scal.p + 48) > 0.0, "lasso: rhs must be nonzero");
  require(o->max_iters >= 0, std::string(who) + ": max_iters must be nonnegative");
  const int T = p ? p->iterations : 0;
  require(out->objective_history != nullptr &&
              out->hist_cap >= std::max(o->max_iters, 0) + 1 + std::max(T, 0),
          std::string(who) + ": history capacity too small");
  const bool track = std::isfinite(o->p_star);
  require(!track || out->gap_history != nullptr, std::string(who) + ": gap_history missing");

  long long applies = 0, adjoints = 0;
  DevBuf<double> dd, ed;
  const double* d = nullptr;
  const double* e = nullptr;
  if (p) {  // sgd_equilibrate on the charged operator (:139)
    dd.alloc(m);
    ed.alloc(n);
    equil_scaling_out so{};
    so.d = dd.p;
    so.e = ed.p;
    so.outputs_on_device = 1;
    M->mu.unlock();
    const equil_status rc = equil_sgd_equilibrate(M, p, nullptr, &so);
    M->mu.lock();
    if (rc != EQUIL_OK) fail(rc, g_err);
    applies = so.apply_count;
    adjoints = so.adjoint_count;
    d = dd.p;
    e = ed.p;
  }
  // ccp_core (:27-110)
  const double sl = std::sqrt(lambda);
  double tau, sigma;
  if (o->tau > 0.0 && o->sigma > 0.0) {
    tau = o->tau;
    sigma = o->sigma;
  } else {
    const double norm2 = spectral_norm_dev(M, d, e, 100, 1e-9, 0);
    if (!(norm2 > 0.0)) fail(EQUIL_ERUNTIME, "ccp_lasso: zero operator");
    tau = 0.9 / norm2;
    sigma = 0.9 / norm2;
  }
  const double f0 = [&] {
    DevBuf<double> zero, r, v;
    zero.alloc(n);
    r.alloc(m);
    v.alloc(1);
    CK(cudaMemsetAsync(zero.p, 0, n * 8, s));
    lasso_value_dev(M, b_d.p, sl, zero.p, zero.p, r.p, v.p);
    return read_scalar(M, v.p);
  }();
  int hl = 0, gl = 0;
  bool reached = false;
  auto push = [&](double f) {
    out->objective_history[hl++] = f;
    if (track) out->gap_history[gl++] = (f - o->p_star) / f0;
  };
  for (int t = 0; t <= T; ++t) push(f0);
  if (track && o->gap_tol > 0.0 && out->gap_history[gl - 1] <= o->gap_tol) reached = true;

  DevBuf<double> y, kz, dy, z, ezt, g, x, absx, r, fh;
  y.alloc(m); kz.alloc(m); dy.alloc(m); r.alloc(m);
  z.alloc(n); ezt.alloc(n); g.alloc(n); x.alloc(n); absx.alloc(n);
  const int iters = std::max(o->max_iters, 0);
  fh.alloc(std::max(iters, 1));
  CK(cudaMemsetAsync(y.p, 0, m * 8, s));
  CK(cudaMemsetAsync(z.p, 0, n * 8, s));
  CK(cudaMemsetAsync(ezt.p, 0, n * 8, s));
  CK(cudaMemsetAsync(x.p, 0, n * 8, s));
  const bool early = track && o->gap_tol > 0.0;  // stop test needs f on the host
  int done = 0;
  for (int t = 1; t <= iters && !reached; ++t) {
    apply_pass(M, false, ezt.p, kz.p, eqb::kPassScaled, d, nullptr, nullptr);  // K z~
    ++applies;
    CK(eqb::launch_ccp_dual(y.p, kz.p, d, b_d.p, sigma, sl, m, dy.p, s));
    apply_pass(M, true, dy.p, g.p, eqb::kPassScaled, e, nullptr, nullptr);  // K^T y
    ++adjoints;
    CK(eqb::launch_ccp_primal(z.p, ezt.p, g.p, e, tau, tau * sl, o->theta, n, x.p, absx.p, s));
    lasso_value_dev(M, b_d.p, sl, x.p, absx.p, r.p, fh.p + (t - 1));  // uncharged probe
    done = t;
    if (early) {
      push(read_scalar(M, fh.p + (t - 1)));
      if (out->gap_history[gl - 1] <= o->gap_tol) reached = true;
    }
  }
  if (!early && done > 0) {
    std::vector<double> f(done);
    CK(cudaMemcpyAsync(f.data(), fh.p, done * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (double v : f) push(v);
  }
  if (out->x) CK(cudaMemcpyAsync(out->x, x.p, n * 8, cudaMemcpyDeviceToHost, s));  // e .* z
  CK(cudaStreamSynchronize(s));
  out->hist_len = hl;
  out->gap_len = gl;
  out->tau = tau;
  out->sigma = sigma;
  out->theta = o->theta;
  out->iterations = done;
  out->equil_iterations = T;
  out->reached_tol = reached ? 1 : 0;
  out->apply_count = applies;
  out->adjoint_count = adjoints;
}

}  // namespace

extern "C" {

equil_status equil_spectral_norm(equil_matrix* M, int max_iters, double rel_tol, uint64_t seed,
                                 double* out) {
  return guarded([&] {
    require(M != nullptr && out != nullptr, "spectral_norm: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    require(M->world == 1, "spectral_norm: single-GPU matrices only in this build");
    *out = spectral_norm_dev(M, nullptr, nullptr, max_iters, rel_tol, seed);
  });
}

equil_status equil_lasso_objective(equil_matrix* M, const double* b, double lambda,
                                   const double* x, double* out) {
  return guarded([&] {
    require(M != nullptr && b != nullptr && x != nullptr && out != nullptr,
            "lasso_objective: null argument");
    require(lambda > 0.0, "lasso_objective: malformed problem");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    require(M->world == 1, "lasso_objective: single-GPU matrices only in this build");
    cudaStream_t s = M->stream;
    DevBuf<double> b_d, x_d, ax, r, v;
    b_d.alloc(M->m); x_d.alloc(M->n); ax.alloc(M->n); r.alloc(M->m); v.alloc(1);
    CK(cudaMemcpyAsync(b_d.p, b, M->m * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(x_d.p, x, M->n * 8, cudaMemcpyHostToDevice, s));
    CK(eqb::launch_abs(x_d.p, M->n, ax.p, s));
    lasso_value_dev(M, b_d.p, std::sqrt(lambda), x_d.p, ax.p, r.p, v.p);
    *out = read_scalar(M, v.p);
  });
}

equil_status equil_ccp_lasso(equil_matrix* M, const double* b, double lambda,
                             const equil_ccp_options* o, equil_ccp_out* out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:ccp_lasso");
    ccp_common(M, b, lambda, nullptr, o, out, "ccp_lasso");
  });
}

equil_status equil_ccp_lasso_preconditioned(equil_matrix* M, const double* b, double lambda,
                                            const equil_params* p, const equil_ccp_options* o,
                                            equil_ccp_out* out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:ccp_lasso_preconditioned");
    require(p != nullptr, "ccp_lasso_preconditioned: null params");
    ccp_common(M, b, lambda, p, o, out, "ccp_lasso_preconditioned");
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Matrix store ingest: Matrix Market files
// (src/matrix_market.cpp) parsed on host threads, sorted / checked / converted
// to CSR on the device; a binary CSR file for fast reloads; host export.
// ---------------------------------------------------------------------------
namespace {

// the local CSR(A) (world 1) or dense A on the host
void export_host(equil_matrix* M, std::vector<int64_t>& rp, std::vector<int32_t>& ci,
                 std::vector<double>& va, std::vector<double>& dense) {
  require(M->world == 1, "export: single-GPU matrices only");
  cudaStream_t s = M->stream;
  if (M->dense) {
    dense.resize(static_cast<size_t>(M->m * M->n));
    CK(cudaMemcpyAsync(dense.data(), M->Ad.p, M->m * M->n * 8, cudaMemcpyDeviceToHost, s));
  } else {
    rp.resize(M->m + 1);
    ci.resize(static_cast<size_t>(M->nnz));
    va.resize(static_cast<size_t>(M->nnz));
    CK(cudaMemcpyAsync(rp.data(), M->A.row_ptr, (M->m + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (M->nnz) {
      CK(cudaMemcpyAsync(ci.data(), M->A.col, M->nnz * 4, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(va.data(), M->A.val, M->nnz * 8, cudaMemcpyDeviceToHost, s));
    }
  }
  CK(cudaStreamSynchronize(s));
}

}  // namespace

extern "C" {

equil_status equil_matrix_read_matrix_market(const char* path, const equil_device_cfg* cfg,
                                             equil_matrix** out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:read_matrix_market");
    require(path != nullptr && out != nullptr, "matrix market: null argument");
    *out = nullptr;
    std::string buf;
    eqb::mm::read_file(path, buf);
    eqb::mm::Matrix mm;
    eqb::mm::parse(buf.data(), buf.size(), mm);
    buf.clear();
    buf.shrink_to_fit();
    if (mm.dense) {
      const equil_status rc =
          equil_matrix_create_dense(mm.m, mm.n, mm.dense_rowmajor.data(), cfg, out);
      if (rc != EQUIL_OK) fail(rc, g_err);
      return;
    }
    create_coo_impl(mm.m, mm.n, mm.nnz, mm.row.data(), mm.col.data(), mm.val.data(),
                    mm.line.data(), cfg, out);
  });
}

equil_status equil_matrix_write_matrix_market(equil_matrix* M, const char* path) {
  return guarded([&] {
    require(M != nullptr && path != nullptr, "matrix market: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> va, dense;
    export_host(M, rp, ci, va, dense);
    if (M->dense)
      eqb::mm::write_array(path, M->m, M->n, dense.data());
    else
      eqb::mm::write_coordinate(path, M->m, M->n, rp.data(), ci.data(), va.data());
  });
}

equil_status equil_matrix_save_binary(equil_matrix* M, const char* path) {
  return guarded([&] {
    require(M != nullptr && path != nullptr, "binary csr: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> va, dense;
    export_host(M, rp, ci, va, dense);
    eqb::mm::write_binary(path, M->m, M->n, M->dense, rp.data(), ci.data(), va.data(),
                          dense.data());
  });
}

equil_status equil_matrix_load_binary(const char* path, const equil_device_cfg* cfg,
                                      equil_matrix** out) {
  return guarded([&] {
    require(path != nullptr && out != nullptr, "binary csr: null argument");
    *out = nullptr;
    FILE* f = std::fopen(path, "rb");
    if (!f) throw std::runtime_error(std::string("binary csr: cannot open '") + path + "'");
    struct Closer {
      FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    int64_t hdr[4];
    eqb::mm::read_binary_header(f, path, hdr);
    const int64_t m = hdr[0], n = hdr[1], nnz = hdr[2];
    // read straight into pinned host buffers (fast H2D in the create call)
    auto pinned = [](size_t bytes) {
      void* p = nullptr;
      CK(cudaMallocHost(&p, std::max<size_t>(bytes, 8)));
      return p;
    };
    struct Pinned {
      void* p;
      ~Pinned() { if (p) cudaFreeHost(p); }
    };
    equil_status rc;
    if (hdr[3]) {
      Pinned a{pinned(static_cast<size_t>(nnz) * 8)};
      eqb::mm::read_exact(f, a.p, 8, static_cast<size_t>(nnz), path);
      rc = equil_matrix_create_dense(m, n, static_cast<const double*>(a.p), cfg, out);
    } else {
      Pinned rp{pinned(static_cast<size_t>(m + 1) * 8)};
      Pinned ci{pinned(static_cast<size_t>(nnz) * 4)};
      Pinned va{pinned(static_cast<size_t>(nnz) * 8)};
      eqb::mm::read_exact(f, rp.p, 8, static_cast<size_t>(m + 1), path);
      eqb::mm::read_exact(f, ci.p, 4, static_cast<size_t>(nnz), path);
      eqb::mm::read_exact(f, va.p, 8, static_cast<size_t>(nnz), path);
      rc = equil_matrix_create_csr(m, n, static_cast<const int64_t*>(rp.p),
                                   static_cast<const int32_t*>(ci.p),
                                   static_cast<const double*>(va.p), cfg, out);
    }
    if (rc != EQUIL_OK) fail(rc, g_err);
  });
}

equil_status equil_matrix_export_csr(equil_matrix* M, int64_t* row_ptr, int32_t* col,
                                     double* val) {
  return guarded([&] {
    require(M != nullptr && row_ptr != nullptr, "export_csr: null argument");
    require(!M->dense, "export_csr: dense matrix");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> va, dense;
    export_host(M, rp, ci, va, dense);
    std::memcpy(row_ptr, rp.data(), rp.size() * 8);
    if (M->nnz) {
      std::memcpy(col, ci.data(), ci.size() * 4);
      std::memcpy(val, va.data(), va.size() * 8);
    }
  });
}

equil_status equil_matrix_export_dense(equil_matrix* M, double* rowmajor) {
  return guarded([&] {
    require(M != nullptr && rowmajor != nullptr, "export_dense: null argument");
    require(M->dense, "export_dense: sparse matrix");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> va, dense;
    export_host(M, rp, ci, va, dense);
    std::memcpy(rowmajor, dense.data(), dense.size() * 8);
  });
}

int equil_matrix_is_dense(const equil_matrix* M) { return M && M->dense ? 1 : 0; }

}  // extern "C"

// Host-only Matrix Market access (no device needed): parse into a handle,
// fetch the entries, write a host CSR / dense array.
extern "C" {

equil_status equil_mm_parse(const char* path, int64_t* m, int64_t* n, int64_t* nnz, int* dense,
                            void** handle) {
  return guarded([&] {
    require(path && m && n && nnz && dense && handle, "matrix market: null argument");
    *handle = nullptr;
    std::string buf;
    eqb::mm::read_file(path, buf);
    auto mm = std::make_unique<eqb::mm::Matrix>();
    eqb::mm::parse(buf.data(), buf.size(), *mm);
    *m = mm->m;
    *n = mm->n;
    *nnz = mm->nnz;
    *dense = mm->dense ? 1 : 0;
    *handle = mm.release();
  });
}

equil_status equil_mm_fetch(void* handle, int64_t* rows, int64_t* cols, double* vals,
                            int64_t* lines) {
  return guarded([&] {
    require(handle != nullptr, "matrix market: null handle");
    const auto* mm = static_cast<const eqb::mm::Matrix*>(handle);
    if (mm->dense) {
      if (vals) std::memcpy(vals, mm->dense_rowmajor.data(), mm->dense_rowmajor.size() * 8);
      return;
    }
    if (rows) std::memcpy(rows, mm->row.data(), mm->row.size() * 8);
    if (cols) std::memcpy(cols, mm->col.data(), mm->col.size() * 8);
    if (vals) std::memcpy(vals, mm->val.data(), mm->val.size() * 8);
    if (lines) std::memcpy(lines, mm->line.data(), mm->line.size() * 8);
  });
}

void equil_mm_free(void* handle) { delete static_cast<eqb::mm::Matrix*>(handle); }

equil_status equil_mm_write_csr(const char* path, int64_t m, int64_t n, const int64_t* row_ptr,
                                const int32_t* col, const double* val) {
  return guarded([&] {
    require(path && row_ptr && m > 0 && n > 0, "matrix market: null argument");
    eqb::mm::write_coordinate(path, m, n, row_ptr, col, val);
  });
}

equil_status equil_mm_write_dense(const char* path, int64_t m, int64_t n,
                                  const double* rowmajor) {
  return guarded([&] {
    require(path && rowmajor && m > 0 && n > 0, "matrix market: null argument");
    eqb::mm::write_array(path, m, n, rowmajor);
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Public helpers of include/equil/equilibrate.hpp and metrics.hpp on the device
// matrix: objective / gradient (weighted and plain), the one-sample stochastic
// gradient estimate, rms_error, project_box.  Per-row sums follow CSR order
// (A's rows for u, A^T's rows = ascending original rows for v); whole-vector
// sums use the canonical reduction; exp is det_exp (the numerics contract).
// Single GPU, sparse matrices (the estimate also takes dense ones).
// ---------------------------------------------------------------------------
namespace {

struct HelperCtx {
  equil_matrix* M;
  cudaStream_t s;
  DevBuf<double> u, v, lu, lv, tm, tn;
  HelperCtx(equil_matrix* m, const double* uh, const double* vh, const char* who,
            bool need_csr = true)
      : M(m), s(m->stream) {
    require(M->world == 1, std::string(who) + ": single-GPU matrices only in this build");
    require(!need_csr || !M->dense, std::string(who) + ": sparse matrices only in this build");
    u.alloc(M->m);
    v.alloc(M->n);
    tm.alloc(M->m);
    tn.alloc(M->n);
    CK(cudaMemcpyAsync(u.p, uh, M->m * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(v.p, vh, M->n * 8, cudaMemcpyHostToDevice, s));
  }
  const double* upload_lin(DevBuf<double>& b, const double* h, int64_t len) {
    if (!h) return nullptr;
    b.alloc(len);
    CK(cudaMemcpyAsync(b.p, h, len * 8, cudaMemcpyHostToDevice, s));
    return b.p;
  }
};

// objective_weighted (src/equilibrate.cpp:10-22); lin arrays null: constants
double objective_dev(HelperCtx& c, const double* lin_u, double lu_c, const double* lin_v,
                     double lv_c, double gamma) {
  equil_matrix* M = c.M;
  double* sc = M->scal.p + 52;
  CK(eqb::launch_obj_terms(M->A, c.u.p, c.v.p, c.tm.p, c.s));
  canon_reduce(M, c.tm.p, M->m, sc + 0, 1);
  if (lin_u) {
    CK(eqb::launch_mul(c.tm.p, lin_u, c.u.p, M->m, c.s));
    canon_reduce(M, c.tm.p, M->m, sc + 1, 1);
  } else {
    canon_reduce(M, c.u.p, M->m, sc + 1, 2, lu_c);
  }
  if (lin_v) {
    CK(eqb::launch_mul(c.tn.p, lin_v, c.v.p, M->n, c.s));
    canon_reduce(M, c.tn.p, M->n, sc + 2, 1);
  } else {
    canon_reduce(M, c.v.p, M->n, sc + 2, 2, lv_c);
  }
  canon_reduce(M, c.u.p, M->m, sc + 3, 0);
  canon_reduce(M, c.v.p, M->n, sc + 4, 0);
  double r[5];
  CK(cudaMemcpyAsync(r, sc, sizeof r, cudaMemcpyDeviceToHost, c.s));
  CK(cudaStreamSynchronize(c.s));
  return 0.5 * r[0] - r[1] - r[2] + 0.5 * gamma * (r[3] + r[4]);
}

// gradient_weighted (src/equilibrate.cpp:24-37)
void gradient_dev(HelperCtx& c, const double* lin_u, double lu_c, const double* lin_v,
                  double lv_c, double gamma, double* gu_h, double* gv_h) {
  equil_matrix* M = c.M;
  CK(eqb::launch_obj_terms(M->A, c.u.p, c.v.p, c.tm.p, c.s));   // sum_j a^2 e^{2(u_i+v_j)}
  CK(eqb::launch_obj_terms(M->AT, c.v.p, c.u.p, c.tn.p, c.s));  // ascending i per column
  CK(eqb::launch_grad_finish(c.tm.p, c.u.p, lin_u, lu_c, gamma, M->m, c.s));
  CK(eqb::launch_grad_finish(c.tn.p, c.v.p, lin_v, lv_c, gamma, M->n, c.s));
  CK(cudaMemcpyAsync(gu_h, c.tm.p, M->m * 8, cudaMemcpyDeviceToHost, c.s));
  CK(cudaMemcpyAsync(gv_h, c.tn.p, M->n * 8, cudaMemcpyDeviceToHost, c.s));
  CK(cudaStreamSynchronize(c.s));
}

}  // namespace

extern "C" {

equil_status equil_objective_weighted(equil_matrix* M, const double* u, const double* v,
                                      const double* lin_u, const double* lin_v, double gamma,
                                      double* out) {
  return guarded([&] {
    require(M && u && v && lin_u && lin_v && out, "objective: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "objective");
    const double* lu = c.upload_lin(c.lu, lin_u, M->m);
    const double* lv = c.upload_lin(c.lv, lin_v, M->n);
    *out = objective_dev(c, lu, 0.0, lv, 0.0, gamma);
  });
}

equil_status equil_objective(equil_matrix* M, const double* u, const double* v,
                             const equil_params* p, double* out) {
  return guarded([&] {
    require(M && u && v && p && out, "objective: null argument");
    validate_params(*p);
    double alpha = 0, beta = 0;
    resolve_targets(*p, M->m, M->n, alpha, beta);
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "objective");
    *out = objective_dev(c, nullptr, alpha * alpha, nullptr, beta * beta, p->gamma);
  });
}

equil_status equil_gradient_weighted(equil_matrix* M, const double* u, const double* v,
                                     const double* lin_u, const double* lin_v, double gamma,
                                     double* grad_u, double* grad_v) {
  return guarded([&] {
    require(M && u && v && lin_u && lin_v && grad_u && grad_v, "gradient: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "gradient");
    const double* lu = c.upload_lin(c.lu, lin_u, M->m);
    const double* lv = c.upload_lin(c.lv, lin_v, M->n);
    gradient_dev(c, lu, 0.0, lv, 0.0, gamma, grad_u, grad_v);
  });
}

equil_status equil_gradient(equil_matrix* M, const double* u, const double* v,
                            const equil_params* p, double* grad_u, double* grad_v) {
  return guarded([&] {
    require(M && u && v && p && grad_u && grad_v, "gradient: null argument");
    validate_params(*p);
    double alpha = 0, beta = 0;
    resolve_targets(*p, M->m, M->n, alpha, beta);
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "gradient");
    gradient_dev(c, nullptr, alpha * alpha, nullptr, beta * beta, p->gamma, grad_u, grad_v);
  });
}

// stochastic_gradient_estimate (src/equilibrate.cpp:60-71): the probes are
// outputs [offset, offset + n + m) of SeededRng(seed, stream) (s then w)
equil_status equil_stochastic_gradient_estimate(equil_matrix* M, const double* u,
                                                const double* v, const equil_params* p,
                                                uint64_t seed, uint64_t stream, uint64_t offset,
                                                double* g_u, double* g_v) {
  return guarded([&] {
    require(M && u && v && p && g_u && g_v, "stochastic_gradient_estimate: null argument");
    validate_params(*p);
    double alpha = 0, beta = 0;
    resolve_targets(*p, M->m, M->n, alpha, beta);
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "stochastic_gradient_estimate", false);
    const int64_t m = M->m, n = M->n;
    const uint64_t total = offset + static_cast<uint64_t>(m + n);
    DevBuf<uint32_t> bits;
    DevBuf<unsigned char> scratch;
    bits.alloc((total + 31) / 32 + 1);
    const size_t sb = eqb::sign_stream_scratch_bytes(total);
    scratch.alloc(sb);
    CK(eqb::sign_stream_generate(seed, stream, total, bits.p, scratch.p, sb, c.s));
    DevBuf<double> d, e, xs, xw;
    d.alloc(m); e.alloc(n); xs.alloc(n); xw.alloc(m);
    // d = exp(u), e = exp(v); xs = e .* s; xw = d .* w
    CK(eqb::launch_expand_scale(c.v.p, nullptr, n, bits.p, static_cast<int64_t>(offset), e.p,
                                xs.p, c.s));
    CK(eqb::launch_expand_scale(c.u.p, nullptr, m, bits.p, static_cast<int64_t>(offset) + n,
                                d.p, xw.p, c.s));
    apply_pass(M, false, xs.p, c.tm.p, eqb::kPassEst, d.p, nullptr, nullptr);
    apply_pass(M, true, xw.p, c.tn.p, eqb::kPassEst, e.p, nullptr, nullptr);
    CK(eqb::launch_sge_finish(c.tm.p, c.u.p, -alpha * alpha, p->gamma, m, c.s));
    CK(eqb::launch_sge_finish(c.tn.p, c.v.p, -beta * beta, p->gamma, n, c.s));
    CK(cudaMemcpyAsync(g_u, c.tm.p, m * 8, cudaMemcpyDeviceToHost, c.s));
    CK(cudaMemcpyAsync(g_v, c.tn.p, n * 8, cudaMemcpyDeviceToHost, c.s));
    CK(cudaStreamSynchronize(c.s));
  });
}

// rms_error (src/metrics.cpp:41-56)
equil_status equil_rms_error(equil_matrix* M, const double* u, const double* v, double alpha,
                             double beta, double* out) {
  return guarded([&] {
    require(M && u && v && out, "rms_error: null argument");
    require(alpha > 0.0 && beta > 0.0, "rms_error: targets must be positive");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "rms_error");
    DevBuf<double> terms;
    terms.alloc(M->m + M->n);
    CK(eqb::launch_exp(c.u.p, c.tm.p, M->m, 2.0, c.s));
    CK(eqb::launch_exp(c.v.p, c.tn.p, M->n, 2.0, c.s));
    CK(eqb::launch_rms_terms(0, M->A, c.tm.p, c.tn.p, terms.p, 0, alpha, c.s));
    CK(eqb::launch_rms_terms(1, M->AT, c.tm.p, c.tn.p, terms.p + M->m, 0, beta, c.s));
    canon_reduce(M, terms.p, M->m + M->n, M->scal.p + 58, 1);
    *out = std::sqrt(read_scalar(M, M->scal.p + 58) / static_cast<double>(M->m + M->n));
  });
}

// project_box (src/equilibrate.cpp:73-76), host
equil_status equil_project_box(const double* x, int64_t n, double bound, double* out) {
  return guarded([&] {
    require(bound >= 0.0, "project_box: bound must be nonnegative");
    require(n == 0 || (x && out), "project_box: null argument");
    for (int64_t i = 0; i < n; ++i) {
      const double lo = x[i] < -bound ? -bound : x[i];  // cwiseMax(-bound)
      out[i] = bound < lo ? bound : lo;                  // cwiseMin(bound)
    }
  });
}

}  // extern "C"
