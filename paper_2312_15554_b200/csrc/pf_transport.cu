// Comparison-medium (Lippmann-Schwinger) transport loop on device — reference
// pkg/src/poreflow/transport.py:180-268.
//
// Per iteration:
//   T1 cuFFT D2Z (batch d+1): [w_0..w_{d-1}, s] -> [W^, S^]            (transport.py:230-231)
//   T2 k_transport_modes     : F^ = S^ + i k.W^, chi^ = F^/(i b0.k + a0 L), chi^(0) = 0,
//                              grad^ = i k chi^, all scaled by 1/n     (pure.py:90-115)
//   T3 cuFFT Z2D (batch d+1): -> [chi', grad chi']                    (transport.py:235-236)
//   T4 k_transport_local     : r1^2, r2^2 partials (238-239), state update (241), and the
//                              NEXT iteration's polarization w, s from grad chi'
//                              (pure.py:71-87) with A, B, F derived from H and u on the fly
//                              (build_coefficients, transport.py:112-121).
//   F  k_transport_finalize  : history row (240), non-finite / growth guard / convergence
//                              (243-258).
#include <cmath>
#include <cstring>

#include "pf_internal.cuh"

namespace pf {

struct TTables {
  const double* kap[3];
  const double* ell[3];
};

__device__ __forceinline__ void t_mode_index(const Geom& g, uint32_t m, int (&idx)[3]) {
  const uint32_t n2h = (uint32_t)g.n2h, n1 = (uint32_t)g.n[1];
  const uint32_t t = m / n2h;
  idx[2] = (int)(m - t * n2h);
  idx[1] = (int)(t % n1);
  idx[0] = (int)(t / n1);
}

struct Polar {
  double pe, eta, a0, ubg;
  double g[3], b0v[3];
};

// w_c = (A - a0)(grad_c + g_c); s = F - sum_c (B_c - b0_c)(grad_c + g_c), with
// A = pore + eta H, B_c = (pe pore) u_c, F = (pe pore) (u_bar . g).
template <int D>
__device__ __forceinline__ void polarize(const Polar& P, double h, const double (&gr)[D], const double* __restrict__ u,
                                         int64_t x, int64_t n, double* __restrict__ W) {
  const double pore = 1.0 - h;
  const double A = pore + P.eta * h;
  const double contrast = A - P.a0;
  const double pep = P.pe * pore;
  double s = pep * P.ubg;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const double tg = gr[c] + P.g[c];
    W[c * n + x] = contrast * tg;
    const double B = pep * u[c * n + x];
    s = s - (B - P.b0v[c]) * tg;
  }
  W[D * n + x] = s;
}

// the same with the flow components already in registers
template <int D>
__device__ __forceinline__ void polarize_u(const Polar& P, double h, const double (&gr)[D], const double (&uu)[D],
                                           int64_t x, int64_t n, double* __restrict__ W) {
  const double pore = 1.0 - h;
  const double A = pore + P.eta * h;
  const double contrast = A - P.a0;
  const double pep = P.pe * pore;
  double s = pep * P.ubg;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const double tg = gr[c] + P.g[c];
    W[c * n + x] = contrast * tg;
    const double B = pep * uu[c];
    s = s - (B - P.b0v[c]) * tg;
  }
  W[D * n + x] = s;
}

template <int D>
__global__ void __launch_bounds__(kThreads) k_polarize(const int64_t n, Polar P, const double* __restrict__ grad,
                                                       const double* __restrict__ u, const uint8_t* __restrict__ H,
                                                       double* __restrict__ W) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    double gr[D];
#pragma unroll
    for (int c = 0; c < D; ++c) gr[c] = grad[c * n + x];
    polarize<D>(P, (double)H[x], gr, u, x, n, W);
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads) k_transport_modes(Geom g, TTables T, const double a0, const double b0x,
                                                              const double b0y, const double b0z,
                                                              const double2* __restrict__ WS, double2* __restrict__ X,
                                                              const Ctrl* __restrict__ ctrl) {
  if (ctrl->done) return;
  const double b0[3] = {b0x, b0y, b0z};
  const uint32_t nh = (uint32_t)g.nh;
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < nh; m += gridDim.x * blockDim.x) {
    int idx[3];
    t_mode_index(g, m, idx);
    double kc[D];
    double L = 0.0, bk = 0.0;
    double2 f = WS[(size_t)D * nh + m];
    double2 wv[D];
#pragma unroll
    for (int c = 0; c < D; ++c) wv[c] = WS[(size_t)c * nh + m];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const int ax = 3 - D + c;
      kc[c] = __ldg(T.kap[ax] + idx[ax]);
      L = L + __ldg(T.ell[ax] + idx[ax]);
      f = cadd(f, cik(kc[c], wv[c]));
      bk = bk + b0[c] * kc[c];
    }
    double2 chi = m == 0 ? make_double2(0.0, 0.0) : cdiv_np(f, make_double2(a0 * L, bk));
    chi = make_double2(chi.x * g.inv_n, chi.y * g.inv_n);
    X[m] = chi;
#pragma unroll
    for (int c = 0; c < D; ++c) X[(size_t)(c + 1) * nh + m] = cik(kc[c], chi);
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 4) k_transport_local(const int64_t n, Polar P, const double* __restrict__ Xn,
                                                              double* __restrict__ chi, double* __restrict__ grad,
                                                              const double* __restrict__ u,
                                                              const uint8_t* __restrict__ H, double* __restrict__ W,
                                                              const Ctrl* __restrict__ ctrl, double* __restrict__ part) {
  if (ctrl->done) return;
  double acc[2] = {0.0, 0.0};
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    // every load of the voxel before any store (they used to trail the stores of
    // the previous field, leaving the kernel latency-bound)
    const double c1 = Xn[x], c0 = chi[x];
    const double h = (double)H[x];
    double gr[D], g0[D], uu[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      gr[c] = Xn[(c + 1) * n + x];
      g0[c] = grad[c * n + x];
      uu[c] = u[c * n + x];
    }
    const double dc = c1 - c0;
    acc[0] += dc * dc;
    chi[x] = c1;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double dg = gr[c] - g0[c];
      acc[1] += dg * dg;
      grad[c * n + x] = gr[c];
    }
    polarize_u<D>(P, h, gr, uu, x, n, W);
  }
  block_sum<2>(acc);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = acc[0];
    part[gridDim.x + blockIdx.x] = acc[1];
  }
}

// scale = 1 for real-space partials, 1/n for Parseval partials (fused pipeline)
__global__ void __launch_bounds__(kFinalizeThreads) k_transport_finalize(Ctrl* __restrict__ ctrl,
                                                                         const double* __restrict__ part, int nb,
                                                                         double* __restrict__ hist, const double t1,
                                                                         const double t2, const int64_t max_iter,
                                                                         const double scale) {
  pdl_wait();
  const int32_t done = ctrl->done;  // (read together with the partials, see k_stokes_finalize)
  double S[2];
  reduce_partials<2>(part, nb, S);
  if (done || threadIdx.x != 0) return;
  const double r1 = sqrt(S[0] * scale), r2 = sqrt(S[1] * scale);
  const int64_t it = ctrl->iter + 1;
  double* row = hist + (it - 1) * PF_TRANSPORT_COLUMNS;
  row[0] = r1;
  row[1] = t1;
  row[2] = r2;
  row[3] = t2;
  ctrl->iter = it;
  if (!(isfinite(r1) && isfinite(r2))) {
    ctrl->diverged = 1;
    ctrl->reason = 1;
    ctrl->done = 1;
    return;
  }
  const double total = r1 + r2;
  const double best = total < ctrl->best ? total : ctrl->best;  // python min(best, total)
  ctrl->best = best;
  if (total > 1e6 * pymax(best, 1e-300)) {
    ctrl->diverged = 1;
    ctrl->reason = 2;
    ctrl->done = 1;
    return;
  }
  if (r1 <= t1 && r2 <= t2) {
    ctrl->converged = 1;
    ctrl->done = 1;
    return;
  }
  if (it >= max_iter) ctrl->done = 1;
}

// pore-masked sums of ncomp fields, the pore count, and a non-finite count.
__global__ void __launch_bounds__(kThreads) k_pore_sums(const int64_t n, const int ncomp, const double* __restrict__ f,
                                                        const uint8_t* __restrict__ H, double* __restrict__ part) {
  double acc[5] = {0, 0, 0, 0, 0};
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const double pore = 1.0 - (double)H[x];
    for (int c = 0; c < ncomp; ++c) {
      const double v = f[c * n + x];
      acc[c] += v * pore;
      if (!isfinite(v)) acc[4] += 1.0;
    }
    acc[3] += pore;
  }
  block_sum<5>(acc);
  if (threadIdx.x == 0)
    for (int k = 0; k < 5; ++k) part[(size_t)k * gridDim.x + blockIdx.x] = acc[k];
}

// One block: row-wise totals of [nrows][nb] partials -> out[nrows].
__global__ void __launch_bounds__(kFinalizeThreads) k_reduce_rows(const double* __restrict__ part, int nrows, int nb,
                                                                  double* __restrict__ out) {
  for (int r = 0; r < nrows; ++r) {
    double v[1];
    reduce_partials<1>(part + (size_t)r * nb, nb, v);
    if (threadIdx.x == 0) out[r] = v[0];
  }
}

__global__ void k_ctrl_init_t(Ctrl* c) {
  c->alpha = c->beta = c->b = c->db = 0.0;
  c->best = INFINITY;
  c->iter = 0;
  c->done = c->converged = c->diverged = c->reason = 0;
}

int reduce_rows_to(pf_plan* p, const double* part, int nrows, int nb, double* out) {
  k_reduce_rows<<<1, kFinalizeThreads, 0, p->work>>>(part, nrows, nb, out);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

// Host: pore-masked sums -> host out[0..ncomp) sums, out[3] pore count, out[4] non-finite count.
int pore_sums_host(pf_plan* p, const uint8_t* H, const double* f, int ncomp, double* out5) {
  const int nb = blocks_for(p->g.nr);
  k_pore_sums<<<nb, kThreads, 0, p->work>>>(p->g.nr, ncomp, f, H, p->partials);
  PF_CK_CUDA(cudaGetLastError());
  double* dout = p->partials + 5 * kMaxBlocks;
  k_reduce_rows<<<1, kFinalizeThreads, 0, p->work>>>(p->partials, 5, nb, dout);
  PF_CK_CUDA(cudaGetLastError());
  PF_CK_CUDA(cudaMemcpyAsync(p->h_small, dout, 5 * sizeof(double), cudaMemcpyDeviceToHost, p->work));
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  for (int k = 0; k < 5; ++k) out5[k] = p->h_small[k];
  return PF_OK;
}

static Polar polar_of(const pf_plan* p) {
  Polar P;
  P.pe = p->tc.pe;
  P.eta = p->tc.eta;
  P.a0 = p->tc.a0;
  P.ubg = p->tc.ubar_dot_g;
  for (int k = 0; k < 3; ++k) {
    P.g[k] = p->tc.g[k];
    P.b0v[k] = p->tc.b0v[k];
  }
  return P;
}

static TTables ttables_of(const pf_plan* p) {
  TTables t;
  for (int i = 0; i < 3; ++i) {
    t.kap[i] = p->kap[i];
    t.ell[i] = p->ell[i];
  }
  return t;
}

template <int D>
static int enqueue_transport_t(pf_plan* p) {
  const Geom& g = p->g;
  const int64_t n = g.nr, nh = g.nh;
  const TransportConst& C = p->tc;
  PF_CK(plan_fft(p, true, D + 1, p->realB, p->specA));
  k_transport_modes<D><<<blocks_for(nh), kThreads, 0, p->work>>>(g, ttables_of(p), C.a0, C.b0v[0], C.b0v[1],
                                                                 C.b0v[2], p->specA, p->specB, p->ctrl);
  PF_CK_CUDA(cudaGetLastError());
  PF_CK(plan_fft(p, false, D + 1, p->specB, p->realA));
  const int nb = blocks_for(n);
  k_transport_local<D><<<nb, kThreads, 0, p->work>>>(n, polar_of(p), p->realA, p->t_chi, p->t_grad, p->t_u,
                                                     p->s_solid, p->realB, p->ctrl, p->partials);
  PF_CK_CUDA(cudaGetLastError());
  k_transport_finalize<<<1, kFinalizeThreads, 0, p->work>>>(p->ctrl, p->partials, nb, p->t_hist, C.eps_tol1,
                                                            C.eps_tol2, C.max_iter, 1.0);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

int transport_polarize(pf_plan* p, const double* grad, double* out) {
  const int64_t n = p->g.nr;
  switch (p->g.d) {
    case 1: k_polarize<1><<<blocks_for(n), kThreads, 0, p->work>>>(n, polar_of(p), grad, p->t_u, p->s_solid, out); break;
    case 2: k_polarize<2><<<blocks_for(n), kThreads, 0, p->work>>>(n, polar_of(p), grad, p->t_u, p->s_solid, out); break;
    default: k_polarize<3><<<blocks_for(n), kThreads, 0, p->work>>>(n, polar_of(p), grad, p->t_u, p->s_solid, out); break;
  }
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

void transport_finalize_launch(pf_plan* p, const double* part, int nb, double scale) {
  const TransportConst& C = p->tc;
  launch_k(k_transport_finalize, 1, kFinalizeThreads, 0, p->work, p->ctrl, part, nb, p->t_hist, C.eps_tol1,
           C.eps_tol2, C.max_iter, scale);
}

static int enqueue_transport(pf_plan* p) {
  if (p->t_pipeline == 1) return tfused_enqueue(p);
  switch (p->g.d) {
    case 1: return enqueue_transport_t<1>(p);
    case 2: return enqueue_transport_t<2>(p);
    default: return enqueue_transport_t<3>(p);
  }
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_transport_begin(pf_plan* p, const pf_transport_params* P, const uint8_t* solid, const double* u, double* chi,
                       double* grad, double* history, pf_transport_result* res) {
  PF_NVTX("pf_transport_begin");
  PF_ARG(p && P && solid && u && chi && grad && history, "null argument");
  PF_ARG(P->pe >= 0.0, "Peclet number must be nonnegative");
  PF_ARG(P->eta > 0.0 && P->eta <= 1.0, "fictitious diffusivity eta must lie in (0, 1]");
  PF_ARG(P->a0 > 0.0, "comparison diffusivity a0 must be positive");
  PF_ARG(P->eps > 0.0, "tolerance must be positive");
  PF_ARG(P->max_iter >= 1, "max_iter must be at least 1");
  PF_CK(enter(p));
  PF_CK(plan_ensure_scratch(p));
  const int d = p->g.d;
  // build_coefficients (transport.py:108-127): finiteness, pore count, u_bar, b0_vec.
  double sums[5];
  PF_CK(pore_sums_host(p, solid, u, d, sums));
  if (sums[4] != 0.0 || sums[3] == 0.0) {  // leave() before reporting: the user stream stays ordered
    leave(p);
    set_error(sums[4] != 0.0 ? "velocity field contains non-finite values"
                             : "cannot form the pore-averaged velocity: no pore cells");
    return PF_ERR_ARG;
  }
  TransportConst& C = p->tc;
  double ubar[3] = {0, 0, 0}, nb2 = 0.0, ubg = 0.0;
  for (int c = 0; c < d; ++c) {
    ubar[c] = sums[c] / sums[3];
    nb2 += ubar[c] * ubar[c];
    ubg += ubar[c] * P->composition_gradient[c];
  }
  const double nb = std::sqrt(nb2);
  for (int c = 0; c < 3; ++c) {
    C.b0v[c] = (c < d && nb > 0.0) ? (P->b0 * ubar[c]) / nb : 0.0;
    C.g[c] = c < d ? P->composition_gradient[c] : 0.0;
  }
  C.pe = P->pe;
  C.eta = P->eta;
  C.a0 = P->a0;
  C.ubar_dot_g = ubg;
  C.eps_tol1 = std::sqrt((double)p->g.nr) * P->eps;
  C.eps_tol2 = std::sqrt((double)(d * p->g.nr)) * P->eps;
  C.max_iter = P->max_iter;
  p->graph.reset();
  p->active = 2;
  p->s_solid = solid;
  p->t_u = u;
  p->t_chi = chi;
  p->t_grad = grad;
  p->t_hist = history;
  std::memset(&p->t_res, 0, sizeof(p->t_res));
  for (int c = 0; c < 3; ++c) {
    p->t_res.b0_vec[c] = C.b0v[c];
    p->t_res.u_bar[c] = ubar[c];
  }
  if (res) *res = p->t_res;
  k_ctrl_init_t<<<1, 1, 0, p->work>>>(p->ctrl);
  PF_CK_CUDA(cudaGetLastError());
  p->t_pipeline = (p->fused_enable && fused_supported(p) && p->g.n[0] <= 512) ? 1 : 0;  // fused transport: N <= 512
  if (p->t_pipeline == 1) return tfused_setup(p, true);
  const int64_t n = p->g.nr;
  switch (d) {
    case 1: k_polarize<1><<<blocks_for(n), kThreads, 0, p->work>>>(n, polar_of(p), grad, u, solid, p->realB); break;
    case 2: k_polarize<2><<<blocks_for(n), kThreads, 0, p->work>>>(n, polar_of(p), grad, u, solid, p->realB); break;
    default: k_polarize<3><<<blocks_for(n), kThreads, 0, p->work>>>(n, polar_of(p), grad, u, solid, p->realB); break;
  }
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

static void fill_tres(pf_plan* p, const Ctrl& c, pf_transport_result* res) {
  p->t_res.iterations = c.iter;
  p->t_res.converged = c.converged;
  p->t_res.diverged = c.diverged;
  p->t_res.reason = c.reason;
  p->t_res.done = c.done;
  if (res) *res = p->t_res;
}

int pf_transport_iterate(pf_plan* p, int64_t n_iter, int poll, pf_transport_result* res) {
  PF_NVTX("pf_transport_iterate");
  PF_ARG(p, "null plan");
  if (p->active != 2) {
    set_error("pf_transport_iterate without pf_transport_begin");
    return PF_ERR_STATE;
  }
  Ctrl c;
  PF_CK(enter(p));
  PF_CK(run_chunks(p, n_iter, poll, enqueue_transport, &c));
  PF_CK(leave(p));
  if (c.iter >= 0) fill_tres(p, c, res);
  return PF_OK;
}

int pf_transport_end(pf_plan* p, pf_transport_result* res) {
  PF_NVTX("pf_transport_end");
  PF_ARG(p, "null plan");
  if (p->active != 2) {
    set_error("pf_transport_end without pf_transport_begin");
    return PF_ERR_STATE;
  }
  if (p->t_pipeline == 1) PF_CK(tfused_finish(p));
  PF_CK_CUDA(cudaMemcpyAsync(&p->h_ctrl[0], p->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, p->work));
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  fill_tres(p, p->h_ctrl[0], res);
  p->active = 0;
  PF_CK(leave(p));
  return PF_OK;
}

int pf_transport_pipeline(const pf_plan* p) { return p ? p->t_pipeline : -1; }

int pf_transport_profile(pf_plan* p, int64_t n_iter, double* stage_ms) {
  PF_ARG(p && stage_ms && n_iter >= 1, "bad argument");
  if (p->active != 2 || p->t_pipeline != 1) {
    set_error("pf_transport_profile needs an active fused transport solve");
    return PF_ERR_STATE;
  }
  PF_CK(enter(p));
  cudaEvent_t ev[6];
  for (int i = 0; i < 6; ++i) PF_CK_CUDA(cudaEventCreate(&ev[i]));
  double acc[5] = {0, 0, 0, 0, 0};
  int st = PF_OK;
  for (int64_t it = 0; it < n_iter && st == PF_OK; ++it) {
    st = tfused_enqueue(p, ev);
    if (st != PF_OK) break;
    cudaEventSynchronize(ev[5]);
    for (int k = 0; k < 5; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
      acc[k] += ms;
    }
  }
  for (int i = 0; i < 6; ++i) cudaEventDestroy(ev[i]);
  PF_CK(st);
  for (int k = 0; k < 5; ++k) stage_ms[k] = acc[k] / (double)n_iter;
  return leave(p);
}

int pf_transport_solve(pf_plan* p, const pf_transport_params* P, const uint8_t* solid, const double* u, double* chi,
                       double* grad, double* history, pf_transport_result* res) {
  PF_NVTX("pf_transport_solve");
  PF_CK(pf_transport_begin(p, P, solid, u, chi, grad, history, res));
  pf_transport_result r{};
  PF_CK(pf_transport_iterate(p, P->max_iter, 1, &r));
  return pf_transport_end(p, res);
}

}  // extern "C"
