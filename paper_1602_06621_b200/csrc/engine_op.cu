// engine_op.cu -- the matrix-free entry point: projected-SGD equilibration of a
// LinearOperator given only by its device apply / apply_adjoint (the
// reference's plugin interface, include/equil/linop.hpp:13-25, with
// sgd_equilibrate on it, include/equil/equilibrate.hpp:89-91 and
// src/equilibrate.cpp:138-221), plus the device-pointer apply of a matrix
// handle so an explicit matrix can serve as such an operator.
//
// Per iteration t the reference's estimator (src/estimator.cpp:5-9 on
// ScaledOperator, src/linop.cpp:17-26) computes y = d .* A(e .* s) and
// z = e .* A^T(d .* w) with s drawn before w.  Here the probes e .* s and
// d .* w are the gathered vectors the SGD epilogue already produces (the
// sign stream, K1, holds s then w per iteration), the user's apply / adjoint
// write A(e .* s) and A^T(d .* w) into the row-sum buffers, and
// sgd_update_rows_kernel -- the split epilogue of the explicit path -- forms
// y = d * acc, est = y * y and the update, the running average and the next
// probes.  With an apply that rounds like the reference's, the result is the
// reference's bit for bit (tests/test_gpu_parity.py: the explicit matrix's own
// device apply as the operator).  Single GPU, no history (the reference needs
// the explicit matrix for it).
#include "engine_internal.h"

namespace {

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

}  // namespace

extern "C" {

equil_status equil_sgd_equilibrate_operator(const equil_device_operator* op,
                                            const equil_params* p, equil_scaling_out* out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:sgd_operator");
    require(op != nullptr && p != nullptr && out != nullptr,
            "sgd_equilibrate_operator: null argument");
    require(op->apply != nullptr && op->apply_adjoint != nullptr,
            "sgd_equilibrate_operator: apply and apply_adjoint are required");
    const int64_t m = op->rows, n = op->cols;
    double alpha = 0.0, beta = 0.0;
    resolve_targets(*p, m, n, alpha, beta);  // src/equilibrate.cpp:216
    validate_params(*p);                     // :142
    require(m < (1LL << 31) && n < (1LL << 31), "sgd_equilibrate_operator: dimension too large");
    DeviceGuard dg(op->device);
    OpStream os(op->device);
    cudaStream_t s = os.s;
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
    DevBuf<double> u, ub, v, vb, xs[2], xw[2], acc, dl, el;
    DevBuf<uint32_t> signs;
    DevBuf<char> scratch;
    DevBuf<unsigned> flags;
    u.alloc_on(m, s);
    ub.alloc_on(m, s);
    v.alloc_on(n, s);
    vb.alloc_on(n, s);
    for (int k = 0; k < 2; ++k) {
      xs[k].alloc_on(n, s);
      xw[k].alloc_on(m, s);
    }
    acc.alloc_on(m + n, s);
    dl.alloc_on(m, s);
    el.alloc_on(n, s);
    flags.alloc_on(1, s);
    CK(cudaMemsetAsync(flags.p, 0, sizeof(unsigned), s));
    if (total > 0) {  // K1: every probe sign of the run (SeededRng(seed, 17))
      signs.alloc_on((total + 31) / 32 + 1, s);
      const size_t sb = eqb::sign_stream_scratch_bytes(total);
      scratch.alloc_on(sb, s);
      CK(eqb::sign_stream_generate(p->seed, 17, total, signs.p, scratch.p, sb, s));
    }
    if (T > 0) {  // u = v = 0, ubar = vbar = 0, xs = s_1, xw = w_1
      CK(eqb::launch_sgd_init(xs[0].p, xw[0].p, u.p, ub.p, v.p, vb.p, n, m, signs.p, m, n, 0, 0,
                              0, 0, m, n, nullptr, nullptr, s));
    } else {
      CK(cudaMemsetAsync(ub.p, 0, m * 8, s));
      CK(cudaMemsetAsync(vb.p, 0, n * 8, s));
    }
    for (int t = 1; t <= T; ++t) {
      eqb::SgdIterArgs a{};
      a.xs_cur = xs[(t - 1) & 1].p;
      a.xw_cur = xw[(t - 1) & 1].p;
      a.xs_next = xs[t & 1].p;
      a.xw_next = xw[t & 1].p;
      a.x[0] = u.p;
      a.x[1] = v.p;
      a.avg[0] = ub.p;
      a.avg[1] = vb.p;
      a.signs = signs.p;
      a.sign_next[0] = static_cast<int64_t>(t) * (m + n) + n;  // w of t+1
      a.sign_next[1] = static_cast<int64_t>(t) * (m + n);      // s of t+1
      a.has_next = t < T;
      a.c[0] = block_const(alpha * alpha);
      a.c[1] = block_const(beta * beta);
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
    CK(eqb::launch_exp(ub.p, dl.p, m, 1.0, s));  // d = exp(ubar), e = exp(vbar) (:201-204)
    CK(eqb::launch_exp(vb.p, el.p, n, 1.0, s));
    unsigned fl = 0;
    CK(cudaMemcpyAsync(&fl, flags.p, sizeof fl, cudaMemcpyDeviceToHost, s));
    const cudaMemcpyKind kind =
        out->outputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (out->u) CK(cudaMemcpyAsync(out->u, ub.p, m * 8, kind, s));
    if (out->v) CK(cudaMemcpyAsync(out->v, vb.p, n * 8, kind, s));
    if (out->d) CK(cudaMemcpyAsync(out->d, dl.p, m * 8, kind, s));
    if (out->e) CK(cudaMemcpyAsync(out->e, el.p, n * 8, kind, s));
    CK(cudaStreamSynchronize(s));
    out->alpha = alpha;
    out->beta = beta;
    out->iterate_bound_ok = (fl & 1u) ? 0 : 1;
    out->box_feasible = (fl & 2u) ? 0 : 1;
    out->apply_count = T;
    out->adjoint_count = T;
    out->hist_len = 0;
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
