// Slab decomposition of one Stokes cell over P ranks (BASELINE cfg 5).
//
// Rank r owns the real-space x-slab i0 in [r L0, (r+1) L0) (L0 = N0/P) of every
// field, and the spectral y-slab k1 in [r L1, (r+1) L1) (L1 = N1/P) of every
// spectrum.  One 3D transform = local 2D transforms over (i1, i2) of the x-slab
// ("A layout" [c][L0][N1][H2]), an all-to-all, and local 1D transforms along i0
// ("T layout" [c][N0][L1][H2], the full spectrum of the local k1 slab).  The
// iteration keeps every spectral state (Q^, D^) in the T layout, so each Stokes
// iteration exchanges exactly two half spectra of 3 components (R^ forward, U^
// back) plus one 9-double all-reduce of the residual partial sums; the decision
// kernels then run identically on every rank.
//
// This file holds the per-rank device work behind pf_slab_* (transforms,
// pack/unpack for the exchange, the spectral / local / finalize steps with
// global mode offsets).  The collectives themselves are issued by the host
// driver (paper_2312_15554_b200/slab.py) through torch.distributed (NCCL on the
// GPU box), between these calls, on the same stream order.
#include <cmath>

#include "pf_internal.cuh"

namespace pf {

struct SlabPlan {
  int N0, N1, N2, P, rank, L0, L1, H2;
  Geom gs;                       // spectral T-layout geometry (global n, k1 offset)
  cufftHandle f2d[4], i2d[4];    // 2D D2Z / Z2D over (N1, N2), batch ncomp*L0, ncomp = 1..3
  cufftHandle z0;                // 1D C2C along i0 of one component, batch L1*H2
  void* work = nullptr;
  size_t work_bytes = 0;
  double2* A = nullptr;          // A-layout scratch, 3 components
};

static SlabPlan* sp_of(pf_plan* p) { return reinterpret_cast<SlabPlan*>(p->slab); }

static void slab_release(pf_plan* p, SlabPlan* s);

void slab_free(pf_plan* p) {
  SlabPlan* s = sp_of(p);
  if (!s) return;
  slab_release(p, s);
  delete s;
  p->slab = nullptr;
}

// send[s][c][i0l][k1l][k2] <- A[c][i0l][s*L1 + k1l][k2]   (forward, x-slab -> per destination)
// T[c][src*L0 + i0l][k1l][k2] <- recv[src][c][i0l][k1l][k2] (forward, after the exchange)
// send[s][c][i0l][k1l][k2] <- T[c][s*L0 + i0l][k1l][k2]   (inverse)
// A[c][i0l][src*L1 + k1l][k2] <- recv[src][c][i0l][k1l][k2] (inverse, after the exchange)
// One kernel: `mode` selects which side carries the exchange-major index.
__global__ void k_slab_move(SlabPlan S, int ncomp, int mode, const double2* __restrict__ src,
                            double2* __restrict__ dst) {
  const int64_t blk = (int64_t)S.L0 * S.L1 * S.H2;  // one (peer, component) block
  const int64_t total = (int64_t)S.P * ncomp * blk;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    // exchange-buffer coordinates of element i
    const int k2 = (int)(i % S.H2);
    int64_t t = i / S.H2;
    const int k1l = (int)(t % S.L1);
    t /= S.L1;
    const int i0l = (int)(t % S.L0);
    t /= S.L0;
    const int c = (int)(t % ncomp);
    const int peer = (int)(t / ncomp);
    int64_t other;
    if (mode == 0 || mode == 3) {  // A layout [c][L0][N1][H2]
      other = (((int64_t)c * S.L0 + i0l) * S.N1 + (int64_t)peer * S.L1 + k1l) * S.H2 + k2;
    } else {  // T layout [c][N0][L1][H2]
      other = (((int64_t)c * S.N0 + (int64_t)peer * S.L0 + i0l) * S.L1 + k1l) * S.H2 + k2;
    }
    if (mode == 0 || mode == 2) dst[i] = src[other];  // pack
    else dst[other] = src[i];                          // unpack
  }
}

__global__ void k_slab_setup_q(double2* Q, const double2* Tq, int64_t n, int owns_zero) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    Q[i] = (owns_zero && i == 0) ? make_double2(0.0, 0.0) : Tq[i];
}

__global__ void k_slab_scale(const double2* __restrict__ src, double2* __restrict__ dst, int64_t n, double s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = make_double2(src[i].x * s, src[i].y * s);
}

// totals[0..5] = sums of the S3 partial rows, totals[6..8] = sums of the S1 rows
__global__ void __launch_bounds__(kFinalizeThreads) k_slab_totals(const double* __restrict__ part3, int nb3,
                                                                  const double* __restrict__ part1, int nb1,
                                                                  double* __restrict__ totals) {
  double S[6], Q[3];
  reduce_partials2<6, 3>(part3, nb3, S, part1, nb1, Q);
  if (threadIdx.x == 0) {
    for (int k = 0; k < 6; ++k) totals[k] = S[k];
    for (int k = 0; k < 3; ++k) totals[6 + k] = Q[k];
  }
}

// G = i kappa_axis F / n on a T-layout spectrum (global mode indices; spectral.py:118-124)
__global__ void k_slab_grad(Geom gs, const double* __restrict__ kap, int axis, const double2* __restrict__ F,
                            double2* __restrict__ G, double inv_n) {
  const int64_t n2h = gs.n2h, n1 = gs.n[1];
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < gs.nh; m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = m / n2h;
    const int64_t idx = axis == 0 ? t / n1 : (axis == 1 ? gs.k1off + t % n1 : m - t * n2h);
    const double2 f = make_double2(F[m].x * inv_n, F[m].y * inv_n);
    G[m] = cik(__ldg(kap + idx), f);
  }
}

static int slab_ensure_work(pf_plan* p, SlabPlan* s, size_t need) {
  if (need <= s->work_bytes) return PF_OK;
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  cudaFree(s->work);
  PF_CK_CUDA(cudaMalloc(&s->work, need));
  s->work_bytes = need;
  for (int k = 1; k <= 3; ++k) {
    if (s->f2d[k]) PF_CK_FFT(cufftSetWorkArea(s->f2d[k], s->work));
    if (s->i2d[k]) PF_CK_FFT(cufftSetWorkArea(s->i2d[k], s->work));
  }
  if (s->z0) PF_CK_FFT(cufftSetWorkArea(s->z0, s->work));
  return PF_OK;
}

}  // namespace pf

using namespace pf;

namespace pf {

// cuFFT plans (2D over (i1, i2) for 1..3 components, 1D along i0), their work
// area and the A-layout scratch: created on first use.  The fused slab uses them
// only at setup / teardown and releases them in between (a 1024^3 cell over two
// ranks needs that memory).
static int slab_transforms(pf_plan* p, SlabPlan* s) {
  if (s->A) return PF_OK;
  long long d2[2] = {s->N1, s->N2};
  size_t need = 0, ws = 0;
  for (int k = 1; k <= 3; ++k) {
    PF_CK_FFT(cufftCreate(&s->f2d[k]));
    PF_CK_FFT(cufftSetAutoAllocation(s->f2d[k], 0));
    PF_CK_FFT(cufftMakePlanMany64(s->f2d[k], 2, d2, nullptr, 1, (long long)s->N1 * s->N2, nullptr, 1,
                                  (long long)s->N1 * s->H2, CUFFT_D2Z, (long long)k * s->L0, &ws));
    need = ws > need ? ws : need;
    PF_CK_FFT(cufftCreate(&s->i2d[k]));
    PF_CK_FFT(cufftSetAutoAllocation(s->i2d[k], 0));
    PF_CK_FFT(cufftMakePlanMany64(s->i2d[k], 2, d2, nullptr, 1, (long long)s->N1 * s->H2, nullptr, 1,
                                  (long long)s->N1 * s->N2, CUFFT_Z2D, (long long)k * s->L0, &ws));
    need = ws > need ? ws : need;
  }
  long long n0[1] = {s->N0};
  long long emb[1] = {s->N0};
  const long long stride = (long long)s->L1 * s->H2;
  PF_CK_FFT(cufftCreate(&s->z0));
  PF_CK_FFT(cufftSetAutoAllocation(s->z0, 0));
  PF_CK_FFT(cufftMakePlanMany64(s->z0, 1, n0, emb, stride, 1, emb, stride, 1, CUFFT_Z2Z, stride, &ws));
  need = ws > need ? ws : need;
  PF_CK(slab_ensure_work(p, s, need > 0 ? need : 256));
  for (int k = 1; k <= 3; ++k) {
    PF_CK_FFT(cufftSetWorkArea(s->f2d[k], s->work));
    PF_CK_FFT(cufftSetWorkArea(s->i2d[k], s->work));
    PF_CK_FFT(cufftSetStream(s->f2d[k], p->work));
    PF_CK_FFT(cufftSetStream(s->i2d[k], p->work));
  }
  PF_CK_FFT(cufftSetWorkArea(s->z0, s->work));
  PF_CK_FFT(cufftSetStream(s->z0, p->work));
  PF_CK_CUDA(cudaMalloc(&s->A, sizeof(double2) * 3 * (size_t)s->L0 * s->N1 * s->H2));
  return PF_OK;
}

static void slab_release(pf_plan* p, SlabPlan* s) {
  cudaStreamSynchronize(p->work);
  for (int k = 1; k <= 3; ++k) {
    if (s->f2d[k]) cufftDestroy(s->f2d[k]);
    if (s->i2d[k]) cufftDestroy(s->i2d[k]);
    s->f2d[k] = s->i2d[k] = 0;
  }
  if (s->z0) cufftDestroy(s->z0);
  s->z0 = 0;
  cudaFree(s->work);
  cudaFree(s->A);
  s->work = nullptr;
  s->work_bytes = 0;
  s->A = nullptr;
}

static int slab_checked(pf_plan* p, SlabPlan** out) {
  PF_ARG(p && p->slab, "not a slab plan");
  *out = sp_of(p);
  return PF_OK;
}

}  // namespace pf

extern "C" {

int pf_slab_plan_create(pf_plan** out, const int64_t* dims, int nranks, int rank, int symbol_mode, int device,
                        void* stream) {
  PF_ARG(out && dims, "null argument");
  PF_ARG(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank %d of %d", rank, nranks);
  PF_ARG(dims[0] % nranks == 0 && dims[1] % nranks == 0, "N0 and N1 must be divisible by the rank count");
  PF_CK(pf_plan_create(out, 3, dims, symbol_mode, device, stream));  // global symbol tables, no scratch
  pf_plan* p = *out;
  SlabPlan* s = new SlabPlan();
  p->slab = s;
  s->N0 = (int)dims[0];
  s->N1 = (int)dims[1];
  s->N2 = (int)dims[2];
  s->P = nranks;
  s->rank = rank;
  s->L0 = s->N0 / nranks;
  s->L1 = s->N1 / nranks;
  s->H2 = s->N2 / 2 + 1;
  Geom& gs = s->gs;
  gs = p->g;  // global dn / inv_n
  gs.n[0] = s->N0;
  gs.n[1] = s->L1;
  gs.n[2] = s->N2;
  gs.n2h = s->H2;
  gs.nh = (int64_t)s->N0 * s->L1 * s->H2;
  gs.k1off = rank * s->L1;
  // local real slab as the plan geometry (S3 / S4 sizes)
  p->g.n[0] = s->L0;
  p->g.nr = (int64_t)s->L0 * s->N1 * s->N2;
  // the cuFFT plans, their work area and the A-layout scratch are created on
  // first use (slab_transforms) and can be released (pf_slab_release_transforms)
  return PF_OK;
}

// Sizes (in complex elements) of the buffers the host allocates: exchange buffers
// hold P*ncomp*L0*L1*H2; a T-layout spectrum holds ncomp*N0*L1*H2.
int pf_slab_sizes(pf_plan* p, int64_t* exchange_per_comp, int64_t* tspec_per_comp, int64_t* real_per_comp) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  *exchange_per_comp = (int64_t)s->P * s->L0 * s->L1 * s->H2;
  *tspec_per_comp = (int64_t)s->N0 * s->L1 * s->H2;
  *real_per_comp = (int64_t)s->L0 * s->N1 * s->N2;
  return PF_OK;
}

int pf_slab_forward(pf_plan* p, const double* real, int ncomp, double* send) {
  PF_NVTX("pf_slab_forward");
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_ARG(ncomp >= 1 && ncomp <= 3, "ncomp 1..3");
  PF_CK(slab_transforms(p, s));
  PF_CK(enter(p));
  PF_CK_FFT(cufftExecD2Z(s->f2d[ncomp], (cufftDoubleReal*)real, (cufftDoubleComplex*)s->A));
  const int64_t total = (int64_t)s->P * ncomp * s->L0 * s->L1 * s->H2;
  k_slab_move<<<blocks_for(total), kThreads, 0, p->work>>>(*s, ncomp, 0, s->A, (double2*)send);
  PF_CK_CUDA(cudaGetLastError());
  return leave(p);
}

int pf_slab_forward_finish(pf_plan* p, const double* recv, int ncomp, double* tspec) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_ARG(ncomp >= 1 && ncomp <= 3, "ncomp 1..3");
  PF_CK(slab_transforms(p, s));
  PF_CK(enter(p));
  const int64_t total = (int64_t)s->P * ncomp * s->L0 * s->L1 * s->H2;
  k_slab_move<<<blocks_for(total), kThreads, 0, p->work>>>(*s, ncomp, 1, (const double2*)recv, (double2*)tspec);
  PF_CK_CUDA(cudaGetLastError());
  const int64_t per = (int64_t)s->N0 * s->L1 * s->H2;
  for (int c = 0; c < ncomp; ++c) {
    cufftDoubleComplex* x = (cufftDoubleComplex*)tspec + c * per;
    PF_CK_FFT(cufftExecZ2Z(s->z0, x, x, CUFFT_FORWARD));
  }
  return leave(p);
}

int pf_slab_inverse(pf_plan* p, double* tspec, int ncomp, double* send) {
  PF_NVTX("pf_slab_inverse");
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_ARG(ncomp >= 1 && ncomp <= 3, "ncomp 1..3");
  PF_CK(slab_transforms(p, s));
  PF_CK(enter(p));
  const int64_t per = (int64_t)s->N0 * s->L1 * s->H2;
  for (int c = 0; c < ncomp; ++c) {
    cufftDoubleComplex* x = (cufftDoubleComplex*)tspec + c * per;
    PF_CK_FFT(cufftExecZ2Z(s->z0, x, x, CUFFT_INVERSE));
  }
  const int64_t total = (int64_t)s->P * ncomp * s->L0 * s->L1 * s->H2;
  k_slab_move<<<blocks_for(total), kThreads, 0, p->work>>>(*s, ncomp, 2, (const double2*)tspec, (double2*)send);
  PF_CK_CUDA(cudaGetLastError());
  return leave(p);
}

int pf_slab_inverse_finish(pf_plan* p, const double* recv, int ncomp, double* real) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_ARG(ncomp >= 1 && ncomp <= 3, "ncomp 1..3");
  PF_CK(slab_transforms(p, s));
  PF_CK(enter(p));
  const int64_t total = (int64_t)s->P * ncomp * s->L0 * s->L1 * s->H2;
  k_slab_move<<<blocks_for(total), kThreads, 0, p->work>>>(*s, ncomp, 3, (const double2*)recv, s->A);
  PF_CK_CUDA(cudaGetLastError());
  PF_CK_FFT(cufftExecZ2D(s->i2d[ncomp], (cufftDoubleComplex*)s->A, (cufftDoubleReal*)real));
  return leave(p);
}

int pf_slab_stokes_begin(pf_plan* p, const pf_stokes_params* P, const uint8_t* solid, double* u, double* ut,
                         double* q, double* a, double* lam, double* history) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_ARG(P && solid && u && ut && q && a && lam && history, "null argument");
  PF_ARG(P->b > 0.0, "coupling penalty b must be positive for the zero mode");
  PF_ARG(P->max_iter >= 1, "max_iter must be at least 1");
  p->s_solid = solid;
  p->s_u = u;
  p->s_ut = ut;
  p->s_q = q;
  p->s_a = a;
  p->s_lam = lam;
  p->s_hist = history;
  StokesConst& C = p->sc;
  const double nglob = (double)s->N0 * s->N1 * s->N2;
  C.nu = P->nu;
  C.eps_rel = P->eps_rel;
  C.tol_vec = std::sqrt(3.0 * nglob) * P->eps_abs;
  C.tol_sca = std::sqrt(nglob) * P->eps_abs;
  for (int k = 0; k < 3; ++k) {
    C.g[k] = P->pressure_gradient[k];
    C.growth[k] = P->growth[k];
    C.thr[k] = P->ratio_threshold[k];
    C.floor_[k] = P->floor[k];
  }
  C.max_iter = P->max_iter;
  C.adaptive = P->adaptive;
  C.lam_pore_sq = 0.0;
  p->active = 3;
  PF_CK(enter(p));
  PF_CK(stokes_ctrl_init(p, P->alpha, P->beta, P->b));
  return leave(p);
}

// Q^ = FFT(q) with the global zero mode cleared (gauge), D^ = i k . FFT(u).
int pf_slab_setup(pf_plan* p, const double* Tq, const double* Tu, double* Q, double* D) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_CK(enter(p));
  const int64_t per = s->gs.nh;
  k_slab_setup_q<<<blocks_for(per), kThreads, 0, p->work>>>((double2*)Q, (const double2*)Tq, per, s->rank == 0);
  PF_CK_CUDA(cudaGetLastError());
  PF_CK(stokes_div_launch(p, s->gs, (const double2*)Tu, (double2*)D));
  return leave(p);
}

int pf_slab_spectral(pf_plan* p, const double* R, double* Q, double* D, double* U) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_CK(enter(p));
  int nb1 = 0;
  PF_CK(stokes_spectral_launch(p, s->gs, (double2*)Q, (const double2*)R, (double2*)D, (double2*)U, p->partials,
                               &nb1));
  p->slab_nb1 = nb1;
  return leave(p);
}

int pf_slab_local(pf_plan* p, const double* unew, double* totals) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_CK(enter(p));
  int nb3 = 0;
  double* part3 = p->partials + 3 * kMaxBlocks;
  PF_CK(stokes_local_launch(p, p->g.nr, unew, part3, &nb3));
  k_slab_totals<<<1, kFinalizeThreads, 0, p->work>>>(part3, nb3, p->partials, p->slab_nb1, totals);
  PF_CK_CUDA(cudaGetLastError());
  return leave(p);
}

int pf_slab_finalize(pf_plan* p, const double* totals) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_CK(enter(p));
  k_stokes_finalize_launch(p, totals, 1, totals + 6, 1);
  PF_CK_CUDA(cudaGetLastError());
  return leave(p);
}

int pf_slab_form_r(pf_plan* p, double* R, int gated) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_CK(enter(p));
  PF_CK(stokes_form_r_gated(p, R, gated));
  return leave(p);
}

int pf_slab_scale(pf_plan* p, const double* src, double* dst, int64_t count, double scale) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_CK(enter(p));
  k_slab_scale<<<blocks_for(count), kThreads, 0, p->work>>>((const double2*)src, (double2*)dst, count, scale);
  PF_CK_CUDA(cudaGetLastError());
  return leave(p);
}

int pf_slab_read(pf_plan* p, pf_stokes_result* res) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_ARG(res, "null result");
  PF_CK_CUDA(cudaMemcpyAsync(&p->h_ctrl[0], p->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, p->work));
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  const Ctrl c = p->h_ctrl[0];
  res->iterations = c.iter;
  res->converged = c.converged;
  res->done = c.done;
  res->final_penalties[0] = c.alpha;
  res->final_penalties[1] = c.beta;
  res->final_penalties[2] = c.b;
  return PF_OK;
}


// Distributed permeability pieces (slab.slab_permeability): the spectral
// gradient of one T-layout component, and this rank's 6 masked Gram sums of one
// velocity component over its x-slab (G = 9 real slab fields [flow][axis]).
int pf_slab_grad(pf_plan* p, const double* Tspec, int axis, double* Tout) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_ARG(Tspec && Tout && axis >= 0 && axis < 3, "bad argument");
  PF_CK(enter(p));
  const double inv_n = 1.0 / ((double)s->N0 * s->N1 * s->N2);
  k_slab_grad<<<blocks_for(s->gs.nh), kThreads, 0, p->work>>>(s->gs, p->kap[axis], axis, (const double2*)Tspec,
                                                               (double2*)Tout, inv_n);
  PF_CK_CUDA(cudaGetLastError());
  return leave(p);
}

int pf_slab_gram(pf_plan* p, const uint8_t* solid, const double* G, double* sums6) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_ARG(solid && G && sums6, "null argument");
  PF_CK(enter(p));
  PF_CK(slab_gram_host(p, solid, G, (int64_t)s->L0 * s->N1 * s->N2, sums6));
  return leave(p);
}

int pf_slab_fused_sizes(pf_plan* p, int64_t* y_main, int64_t* y_nyq) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_ARG(y_main && y_nyq, "null argument");
  const bool cubic = s->N0 == s->N1 && s->N1 == s->N2;
  const bool ok = cubic && (s->P & (s->P - 1)) == 0 && fused_slab_supported(s->N0, s->L0, s->L1);
  *y_main = ok ? 3 * (int64_t)s->N0 * s->L1 * (s->N2 / 2) : 0;
  *y_nyq = ok ? 3 * (int64_t)s->N0 * s->L1 : 0;
  return PF_OK;
}

int pf_slab_fused_bind(pf_plan* p, double* Yy, double* Yyn, double* Yx, double* Yxn) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  PF_ARG(Yy && Yyn && Yx && Yxn, "null argument");
  PF_ARG(s->N0 == s->N1 && s->N1 == s->N2 && (s->P & (s->P - 1)) == 0,
         "fused slab needs a cubic grid and a power-of-two rank count");
  PF_CK(enter(p));
  PF_CK(fused_slab_bind(p, s->N0, s->L0, s->L1, s->rank * s->L1, (double2*)Yy, (double2*)Yyn, (double2*)Yx,
                        (double2*)Yxn));
  return leave(p);
}

static int fslab_checked(pf_plan* p, SlabPlan** s) {
  PF_CK(slab_checked(p, s));
  if (!p->fused) {
    set_error("pf_slab_fused_* before pf_slab_fused_bind");
    return PF_ERR_STATE;
  }
  return PF_OK;
}

int pf_slab_fused_setup(pf_plan* p, const double* Tq, const double* Td, double* R) {
  PF_NVTX("pf_slab_fused_setup");
  SlabPlan* s;
  PF_CK(fslab_checked(p, &s));
  PF_ARG(Tq && Td && R, "null argument");
  PF_CK(enter(p));
  PF_CK(fused_slab_setup(p, (const double2*)Tq, (const double2*)Td, R));
  return leave(p);
}

int pf_slab_fused_setup_zero(pf_plan* p) {
  PF_NVTX("pf_slab_fused_setup_zero");
  SlabPlan* s;
  PF_CK(fslab_checked(p, &s));
  PF_CK(enter(p));
  int64_t ym = 0, yn = 0;
  PF_CK(pf_slab_fused_sizes(p, &ym, &yn));
  PF_CK(fused_slab_setup_zero(p, ym, yn));
  return leave(p);
}

int pf_slab_release_transforms(pf_plan* p) {
  SlabPlan* s;
  PF_CK(slab_checked(p, &s));
  slab_release(p, s);
  return PF_OK;
}

int pf_slab_fused_pk(pf_plan* p) {
  PF_NVTX("pf_slab_fused_pk");
  SlabPlan* s;
  PF_CK(fslab_checked(p, &s));
  PF_CK(enter(p));
  PF_CK(fused_slab_pk(p));
  return leave(p);
}

int pf_slab_fused_rs(pf_plan* p, double* totals) {
  PF_NVTX("pf_slab_fused_rs");
  SlabPlan* s;
  PF_CK(fslab_checked(p, &s));
  PF_ARG(totals, "null argument");
  PF_CK(enter(p));
  PF_CK(fused_slab_rs(p, totals));
  return leave(p);
}

int pf_slab_fused_mf(pf_plan* p) {
  PF_NVTX("pf_slab_fused_mf");
  SlabPlan* s;
  PF_CK(fslab_checked(p, &s));
  PF_CK(enter(p));
  PF_CK(fused_slab_mf(p));
  return leave(p);
}

// Component-pipelined variants (slab.py overlaps the exchange of component c + 1
// with the passes of component c): MI + RS of one component; the rank's 9 sums
// once all three ran; MF of one component (fix = 1 on the first one of an
// iteration runs the gated RSF pass of every component first).
int pf_slab_fused_rs_part(pf_plan* p, int comp) {
  PF_NVTX("pf_slab_fused_rs_part");
  SlabPlan* s;
  PF_CK(fslab_checked(p, &s));
  PF_ARG(comp >= 0 && comp < 3, "comp 0..2");
  PF_CK(enter(p));
  PF_CK(fused_slab_rs_part(p, comp));
  return leave(p);
}

int pf_slab_fused_totals(pf_plan* p, double* totals) {
  SlabPlan* s;
  PF_CK(fslab_checked(p, &s));
  PF_ARG(totals, "null argument");
  PF_CK(enter(p));
  PF_CK(fused_slab_totals(p, totals));
  return leave(p);
}

int pf_slab_fused_mf_part(pf_plan* p, int comp, int fix) {
  PF_NVTX("pf_slab_fused_mf_part");
  SlabPlan* s;
  PF_CK(fslab_checked(p, &s));
  PF_ARG(comp >= 0 && comp < 3, "comp 0..2");
  PF_CK(enter(p));
  PF_CK(fused_slab_mf_part(p, comp, fix));
  return leave(p);
}

int pf_slab_fused_set_peers(pf_plan* p, const uint64_t* yy, const uint64_t* yyn, const uint64_t* yx,
                            const uint64_t* yxn, int npeers) {
  SlabPlan* s;
  PF_CK(fslab_checked(p, &s));
  PF_ARG(npeers == 0 || (yy && yyn && yx && yxn), "null argument");
  return fused_slab_set_peers(p, yy, yyn, yx, yxn, npeers);
}

int pf_slab_fused_end(pf_plan* p, double* Tq) {
  SlabPlan* s;
  PF_CK(fslab_checked(p, &s));
  PF_ARG(Tq, "null argument");
  PF_CK(enter(p));
  PF_CK(fused_slab_end(p, (double2*)Tq));
  return leave(p);
}

}  // extern "C"
