// engine_op.cu -- the matrix-free entry points: projected-SGD equilibration and
// (preconditioned) LSQR of a LinearOperator given only by its device apply /
// apply_adjoint (the reference's plugin interface, include/equil/linop.hpp:
// 13-25; sgd_equilibrate, include/equil/equilibrate.hpp:89-91 and
// src/equilibrate.cpp:138-221; lsqr / lsqr_preconditioned, src/lsqr.cpp:
// 17-138), plus the device-pointer apply of a matrix handle so an explicit
// matrix can serve as such an operator.
//
// SGD: per iteration t the reference's estimator (src/estimator.cpp:5-9 on
// ScaledOperator, src/linop.cpp:17-26) computes y = d .* A(e .* s) and
// z = e .* A^T(d .* w), s drawn before w.  Here the probes e .* s and d .* w
// are the gathered vectors the SGD epilogue already produces (the sign stream,
// K1, holds s then w per iteration), the user's apply / adjoint write
// A(e .* s) and A^T(d .* w) into the row-sum buffers, and
// sgd_update_rows_kernel -- the split epilogue of the explicit path -- forms
// y = d * acc, est = y * y, the update, the running average and the next
// probes.
//
// LSQR: src/lsqr.cpp:17-81 literally -- three operator calls per iteration
// (B v, B^T u, and the uncharged residual probe A x), the pass epilogues
// (sgd_common.cuh pass_epilogue) for B v - alpha u, B^T u - beta v and
// b - A x, canonical norms, and the scalar recurrence with std::hypot on the
// host.
//
// With an apply that rounds like the reference operator's, results are the
// reference's bit for bit (tests/test_gpu_operator.py uses an explicit
// matrix's own device apply as the operator).  Single GPU; no SGD history (the
// reference needs the explicit matrix for it).
#include <cmath>

#include "engine_internal.h"
#include "sgd_common.cuh"

namespace {

// out = epilogue(acc) of the generic passes (B v - alpha u, B^T u - beta v,
// b - A x, scale .* acc) applied to an operator's output
__global__ void op_epilogue_kernel(eqb::PassArgs a, const double* __restrict__ acc, int64_t n) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r < n) eqb::pass_epilogue(a, r, acc[r]);
}
void op_epilogue(double* out, const double* acc, int64_t n, int mode, const double* scale,
                 const double* prev, const double* coef, cudaStream_t s) {
  if (n == 0) return;
  eqb::PassArgs a{};
  a.out = out;
  a.scale = scale;
  a.prev = prev;
  a.coef = coef;
  a.mode = mode;
  op_epilogue_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(a, acc, n);
  CK(cudaGetLastError());
}
__global__ void mul_kernel(double* __restrict__ y, const double* __restrict__ a,
                           const double* __restrict__ b, int64_t n) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < n) y[k] = __dmul_rn(a[k], b[k]);  // cwiseProduct
}
void mul(double* y, const double* a, const double* b, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  mul_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(y, a, b, n);
  CK(cudaGetLastError());
}

struct OpStream {
  cudaStream_t s = nullptr;
  explicit OpStream(int dev) {
    CK(cudaSetDevice(dev));
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  }
  ~OpStream() {
    if (s) cudaStreamDestroy(s);
  }
};

void check_op(const equil_device_operator* op, const char* who) {
  require(op != nullptr, std::string(who) + ": null operator");
  require(op->apply != nullptr && op->apply_adjoint != nullptr,
          std::string(who) + ": apply and apply_adjoint are required");
  require(op->rows > 0 && op->cols > 0, std::string(who) + ": dimensions must be positive");
  require(op->rows < (1LL << 31) && op->cols < (1LL << 31),
          std::string(who) + ": dimension too large");
}

// canonical Euclidean norm (Eigen's norm(), det_math.cuh order) of a device
// vector, read back to the host
struct Norm {
  DevBuf<double> part, res;
  DevBuf<unsigned> cnt;
  Norm(int64_t maxlen, cudaStream_t s) {
    part.alloc_on((maxlen + eqb::kChunk - 1) / eqb::kChunk + 1, s);
    res.alloc_on(8, s);
    cnt.alloc_on(1, s);
    CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned), s));
  }
  // into the device scalar slot k (read later) ...
  void dev(const double* x, int64_t n, int k, cudaStream_t s) {
    CK(eqb::launch_canon_reduce(x, n, 0, 0.0, part.p, cnt.p, res.p + k, 1, s,
                                static_cast<int64_t>(part.n)));
  }
  // ... or straight to the host
  double host(const double* x, int64_t n, int k, cudaStream_t s) {
    dev(x, n, k, s);
    double h = 0.0;
    CK(cudaMemcpyAsync(&h, res.p + k, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return h;
  }
};

// sgd_equilibrate on the operator (src/equilibrate.cpp:138-221); leaves ubar,
// vbar, d = exp(ubar), e = exp(vbar) on the device
struct SgdOut {
  DevBuf<double> ub, vb, d, e;
  unsigned flags = 0;
  double alpha = 0.0, beta = 0.0;
};
void sgd_operator_core(const equil_device_operator* op, const equil_params* p, cudaStream_t s,
                       SgdOut& r) {
  const int64_t m = op->rows, n = op->cols;
  resolve_targets(*p, m, n, r.alpha, r.beta);  // src/equilibrate.cpp:216
  validate_params(*p);                         // :142
  const int T = p->iterations;
  const uint64_t total = static_cast<uint64_t>(m + n) * static_cast<uint64_t>(T);
  const double gamma = p->gamma, Mx = p->max_log_scale;
  auto block_const = [&](double lin) {
    eqb::SgdBlockConst c;
    c.lin = lin;
    c.gamma = gamma;
    c.M = Mx;
    const double cap = lin / gamma;
    c.thresh = cap + 1e-9 * std::max(1.0, std::abs(cap));
    return c;
  };
  DevBuf<double> u, v, xs[2], xw[2], acc;
  DevBuf<uint32_t> signs;
  DevBuf<char> scratch;
  DevBuf<unsigned> flags;
  u.alloc_on(m, s);
  v.alloc_on(n, s);
  r.ub.alloc_on(m, s);
  r.vb.alloc_on(n, s);
  r.d.alloc_on(m, s);
  r.e.alloc_on(n, s);
  for (int k = 0; k < 2; ++k) {
    xs[k].alloc_on(n, s);
    xw[k].alloc_on(m, s);
  }
  acc.alloc_on(m + n, s);
  flags.alloc_on(1, s);
  CK(cudaMemsetAsync(flags.p, 0, sizeof(unsigned), s));
  if (total > 0) {  // K1: every probe sign of the run (SeededRng(seed, 17))
    signs.alloc_on((total + 31) / 32 + 1, s);
    const size_t sb = eqb::sign_stream_scratch_bytes(total);
    scratch.alloc_on(sb, s);
    CK(eqb::sign_stream_generate(p->seed, 17, total, signs.p, scratch.p, sb, s));
  }
  if (T > 0) {  // u = v = 0, ubar = vbar = 0, xs = s_1, xw = w_1
    CK(eqb::launch_sgd_init(xs[0].p, xw[0].p, u.p, r.ub.p, v.p, r.vb.p, n, m, signs.p, m, n, 0,
                            0, 0, 0, m, n, nullptr, nullptr, s));
  } else {
    CK(cudaMemsetAsync(r.ub.p, 0, m * 8, s));
    CK(cudaMemsetAsync(r.vb.p, 0, n * 8, s));
  }
  for (int t = 1; t <= T; ++t) {
    eqb::SgdIterArgs a{};
    a.xs_cur = xs[(t - 1) & 1].p;
    a.xw_cur = xw[(t - 1) & 1].p;
    a.xs_next = xs[t & 1].p;
    a.xw_next = xw[t & 1].p;
    a.x[0] = u.p;
    a.x[1] = v.p;
    a.avg[0] = r.ub.p;
    a.avg[1] = r.vb.p;
    a.signs = signs.p;
    a.sign_next[0] = static_cast<int64_t>(t) * (m + n) + n;  // w of t+1
    a.sign_next[1] = static_cast<int64_t>(t) * (m + n);      // s of t+1
    a.has_next = t < T;
    a.c[0] = block_const(r.alpha * r.alpha);
    a.c[1] = block_const(r.beta * r.beta);
    a.carry[0] = acc.p;
    a.carry[1] = acc.p + m;
    a.nblk[0] = a.nblk[1] = 1;
    a.st.step = 2.0 / (gamma * static_cast<double>(t + 1));  // :106
    a.st.aw = 2.0 / (static_cast<double>(t) + 2.0);           // :107
    a.st.aw1 = 1.0 - a.st.aw;
    a.flags = flags.p;
    // A (e .* s) and A^T (d .* w): the user's operator, on our stream
    op->apply(op->ctx, a.xs_cur, a.carry[0], s);
    op->apply_adjoint(op->ctx, a.xw_cur, a.carry[1], s);
    CK(cudaGetLastError());
    CK(eqb::launch_sgd_update_rows(a, m, n, s));
  }
  CK(eqb::launch_exp(r.ub.p, r.d.p, m, 1.0, s));  // d = exp(ubar), e = exp(vbar) (:201-204)
  CK(eqb::launch_exp(r.vb.p, r.e.p, n, 1.0, s));
  CK(cudaMemcpyAsync(&r.flags, flags.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
}

// lsqr_core (src/lsqr.cpp:17-81) on B = diag(d) A diag(e) (d, e null: B = A)
// with right-hand side c; the residual probe is |b - A(e .* x)| / |b|
struct LsqrState {
  std::vector<double> hist;
  int iterations = 0;
  bool reached_tol = false, breakdown = false;
  long long applies = 0, adjoints = 0;
};
void lsqr_operator_core(const equil_device_operator* op, cudaStream_t s, const double* c,
                        const double* b, double bnorm, const double* d, const double* e,
                        int max_iters, double tol, LsqrState& st, DevBuf<double>& x) {
  const int64_t m = op->rows, n = op->cols;
  Norm nrm(std::max(m, n), s);
  double* sc = nrm.res.p;  // device scalars: [0] beta, [1] alpha, [2] residual norm
  DevBuf<double> u, v, w, du, ev, ex, y, z, un, vn, r;
  u.alloc_on(m, s); du.alloc_on(m, s); y.alloc_on(m, s); un.alloc_on(m, s); r.alloc_on(m, s);
  v.alloc_on(n, s); w.alloc_on(n, s); ev.alloc_on(n, s); ex.alloc_on(n, s); z.alloc_on(n, s);
  vn.alloc_on(n, s);
  x.alloc_on(n, s);
  CK(cudaMemsetAsync(x.p, 0, n * 8, s));
  // beta = |c|, u = c / beta, v = B^T u, alpha = |v| (:22-26)
  double beta = nrm.host(c, m, 0, s);
  CK(eqb::launch_lsqr_normalize(u.p, c, sc + 0, du.p, d, m, nullptr, nullptr, s));
  op->apply_adjoint(op->ctx, du.p, z.p, s);  // A^T (d .* u)
  ++st.adjoints;
  op_epilogue(vn.p, z.p, n, eqb::kPassScaled, e, nullptr, nullptr, s);  // e .* A^T (d .* u)
  double alpha = nrm.host(vn.p, n, 1, s);
  if (alpha == 0.0) {
    st.breakdown = true;  // :27-30
    return;
  }
  CK(eqb::launch_lsqr_normalize(v.p, vn.p, sc + 1, ev.p, e, n, nullptr, nullptr, s));  // :31
  CK(cudaMemcpyAsync(w.p, v.p, n * 8, cudaMemcpyDeviceToDevice, s));                 // :32
  double phibar = beta, rhobar = alpha;
  for (int t = 1; t <= max_iters; ++t) {
    bool invariant = false;
    // u' = B v - alpha u (:39), B v = d .* A (e .* v)
    op->apply(op->ctx, ev.p, y.p, s);
    ++st.applies;
    op_epilogue(un.p, y.p, m, eqb::kPassLsqrU, d, u.p, sc + 1, s);
    beta = nrm.host(un.p, m, 0, s);
    if (beta > 0.0) {
      CK(eqb::launch_lsqr_normalize(u.p, un.p, sc + 0, du.p, d, m, nullptr, nullptr, s));
    } else {
      invariant = true;
    }
    alpha = 0.0;
    if (!invariant) {  // v' = B^T u - beta v (:49), B^T u = e .* A^T (d .* u)
      op->apply_adjoint(op->ctx, du.p, z.p, s);
      ++st.adjoints;
      op_epilogue(vn.p, z.p, n, eqb::kPassLsqrV, e, v.p, sc + 0, s);
      alpha = nrm.host(vn.p, n, 1, s);
      if (alpha > 0.0) {
        CK(eqb::launch_lsqr_normalize(v.p, vn.p, sc + 1, ev.p, e, n, nullptr, nullptr, s));
      } else {
        invariant = true;
      }
    }
    const double rho = std::hypot(rhobar, beta);  // :58-64
    const double cs = rhobar / rho;
    const double sn = beta / rho;
    const double theta = sn * alpha;
    rhobar = -cs * alpha;
    const double phi = cs * phibar;
    phibar = sn * phibar;
    // x += (phi / rho) w, w = v - (theta / rho) w, and e .* x for the probe
    CK(eqb::launch_lsqr_xw_update(x.p, w.p, v.p, phi / rho, theta / rho, e, ex.p, n, s));
    st.iterations = t;
    // |b - A (e .* x)| / |b| (:94-97, :129-133): uncharged
    op->apply(op->ctx, ex.p, y.p, s);
    op_epilogue(r.p, y.p, m, eqb::kPassResid, nullptr, b, nullptr, s);
    const double rel = nrm.host(r.p, m, 2, s) / bnorm;
    st.hist.push_back(rel);
    if (rel <= tol) {
      st.reached_tol = true;
      break;
    }
    if (invariant) {
      st.breakdown = true;
      break;
    }
  }
}

void lsqr_operator(const equil_device_operator* op, const double* b_host, const equil_params* p,
                   int max_iters, double tol, equil_lsqr_out* out) {
  const char* who = p ? "lsqr_preconditioned" : "lsqr";
  check_op(op, who);
  require(b_host != nullptr && out != nullptr, std::string(who) + ": null argument");
  const int64_t m = op->rows, n = op->cols;
  DeviceGuard dg(op->device);
  OpStream os(op->device);
  cudaStream_t s = os.s;
  DevBuf<double> b, c;
  b.alloc_on(m, s);
  h2d_sync(s, b.p, b_host, m * 8);
  Norm nrm(m, s);
  const double bnorm = nrm.host(b.p, m, 0, s);
  require(bnorm > 0.0, std::string(who) + ": rhs must be nonzero");              // :89, :111
  require(max_iters >= 0, std::string(who) + ": max_iters must be nonnegative");  // :90, :112
  LsqrState st;
  SgdOut eq;
  const double* d = nullptr;
  const double* e = nullptr;
  const double* cp = b.p;
  int T = 0;
  if (p) {  // equilibrate first (charged), then LSQR on diag(d) A diag(e) (:115-135)
    sgd_operator_core(op, p, s, eq);
    T = p->iterations;
    st.applies += T;
    st.adjoints += T;
    for (int t = 0; t <= T; ++t) st.hist.push_back(1.0);  // :121-123
    c.alloc_on(m, s);
    mul(c.p, eq.d.p, b.p, m, s);  // c = d .* b
    d = eq.d.p;
    e = eq.e.p;
    cp = c.p;
  } else {
    st.hist.push_back(1.0);  // :94
  }
  DevBuf<double> x;
  lsqr_operator_core(op, s, cp, b.p, bnorm, d, e, max_iters, tol, st, x);
  require(out->residual_history != nullptr &&
              out->residual_cap >= static_cast<int>(st.hist.size()),
          std::string(who) + ": residual_history capacity too small");
  DevBuf<double> xo;
  if (out->x) {  // x = e .* x_scaled (:136); x is zero after a setup breakdown
    const double* xr = x.p;
    if (e) {
      xo.alloc_on(n, s);
      mul(xo.p, e, x.p, n, s);
      xr = xo.p;
    }
    CK(cudaMemcpyAsync(out->x, xr, n * 8, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  std::copy(st.hist.begin(), st.hist.end(), out->residual_history);
  out->hist_len = static_cast<int>(st.hist.size());
  out->iterations = st.iterations;
  out->equil_iterations = T;
  out->reached_tol = st.reached_tol;
  out->breakdown = st.breakdown;
  out->apply_count = st.applies;
  out->adjoint_count = st.adjoints;
}

}  // namespace

extern "C" {

equil_status equil_sgd_equilibrate_operator(const equil_device_operator* op,
                                            const equil_params* p, equil_scaling_out* out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:sgd_operator");
    require(p != nullptr && out != nullptr, "sgd_equilibrate_operator: null argument");
    check_op(op, "sgd_equilibrate_operator");
    const int64_t m = op->rows, n = op->cols;
    DeviceGuard dg(op->device);
    OpStream os(op->device);
    cudaStream_t s = os.s;
    SgdOut r;
    sgd_operator_core(op, p, s, r);
    const cudaMemcpyKind kind =
        out->outputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (out->u) CK(cudaMemcpyAsync(out->u, r.ub.p, m * 8, kind, s));
    if (out->v) CK(cudaMemcpyAsync(out->v, r.vb.p, n * 8, kind, s));
    if (out->d) CK(cudaMemcpyAsync(out->d, r.d.p, m * 8, kind, s));
    if (out->e) CK(cudaMemcpyAsync(out->e, r.e.p, n * 8, kind, s));
    CK(cudaStreamSynchronize(s));
    out->alpha = r.alpha;
    out->beta = r.beta;
    out->iterate_bound_ok = (r.flags & 1u) ? 0 : 1;
    out->box_feasible = (r.flags & 2u) ? 0 : 1;
    out->apply_count = p->iterations;
    out->adjoint_count = p->iterations;
    out->hist_len = 0;
  });
}

equil_status equil_lsqr_operator(const equil_device_operator* op, const double* b,
                                 const equil_params* p, int max_iters, double tol,
                                 equil_lsqr_out* out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:lsqr_operator");
    lsqr_operator(op, b, p, max_iters, tol, out);
  });
}

// y = A x (adjoint: x = A^T y) on device pointers, ordered on the caller's
// stream: the explicit matrix's own traversal (CSR order sums, or the
// canonical dense order) as a device operator.
equil_status equil_apply_device(equil_matrix* M, const double* x, double* y, int adjoint,
                                void* stream) {
  return guarded([&] {
    require(M != nullptr && x != nullptr && y != nullptr, "apply: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    require(M->world == 1, "apply: single-GPU matrices only");
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    CK(cudaEventRecord(M->ev_fork, cs));  // the caller's inputs are ready
    CK(cudaStreamWaitEvent(M->stream, M->ev_fork, 0));
    apply_pass(M, adjoint != 0, x, y, eqb::kPassPlain, nullptr, nullptr, nullptr);
    CK(cudaEventRecord(M->ev_join, M->stream));
    CK(cudaStreamWaitEvent(cs, M->ev_join, 0));  // the caller's next work sees y
  });
}

}  // extern "C"
