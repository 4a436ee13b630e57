// Kernel plugin: the five per-iteration kernels of the reference's backend
// contract (pkg/src/poreflow/backends/pure.py:26-115, same signatures as the
// Cython twin _fused.pyx) on device pointers, full-spectrum layout.  The
// arithmetic is written in the reference's evaluation order; the library is
// compiled with --fmad=false, so results match numpy to the last bit except
// where numpy itself is not deterministic.
#include "pf_internal.cuh"

namespace pf {

struct KGeom {
  int d;
  int n[3];  // padded full-spectrum extents
  int64_t size;
};

static int kgeom(int ndim, const int64_t* dims, KGeom& g) {
  PF_ARG(ndim >= 1 && ndim <= 3 && dims, "ndim must be 1..3");
  g.d = ndim;
  g.n[0] = g.n[1] = g.n[2] = 1;
  g.size = 1;
  for (int j = 0; j < ndim; ++j) {
    PF_ARG(dims[j] >= 1, "bad extent");
    g.n[3 - ndim + j] = (int)dims[j];
    g.size *= dims[j];
  }
  PF_ARG(g.size < ((int64_t)1 << 31), "array too large");
  return PF_OK;
}

struct KTabs {
  const double* k[3];
};

__device__ __forceinline__ void kidx(const KGeom& g, int64_t m, int (&idx)[3]) {
  idx[2] = (int)(m % g.n[2]);
  const int64_t t = m / g.n[2];
  idx[1] = (int)(t % g.n[1]);
  idx[0] = (int)(t / g.n[1]);
}

#define GRID_STRIDE(m, N) \
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < (N); m += (int64_t)gridDim.x * blockDim.x)

template <int D>
__global__ void k_svu(KGeom g, KTabs T, const double2* q, const double2* ah, const double2* uth, const double* lap,
                      const double* ksq, double nu, double beta, double b, double g0, double g1, double g2,
                      double2* out) {
  const double gp[3] = {g0, g1, g2};
  const int64_t N = g.size;
  GRID_STRIDE(m, N) {
    int idx[3];
    kidx(g, m, idx);
    double kc[D];
    double2 r[D];
    const double2 qq = q[m];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const int ax = 3 - D + c;
      kc[c] = T.k[ax][idx[ax]];
      const double2 a = ah[c * N + m], ut = uth[c * N + m];
      // (-1j k) q - a + b ut   (pure.py:41-43)
      r[c] = make_double2((kc[c] * qq.y - a.x) + b * ut.x, (-(kc[c] * qq.x) - a.y) + b * ut.y);
      if (m == 0) r[c].x = r[c].x + (double)N * gp[c];
    }
    const double A = nu * lap[m] + b;
    double2 kr = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < D; ++c) kr = cadd(kr, cscale(kc[c], r[c]));
    const double2 corr = cscale(beta / (A + beta * ksq[m]), kr);
    const double s = 1.0 / A;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double2 u = csub(r[c], cscale(kc[c], corr));
      out[c * N + m] = make_double2(u.x * s, u.y * s);
    }
  }
}

__global__ void k_aux(int64_t N, int D, const double* u, const double* a, const double* lam, const double* solid,
                      double alpha, double b, double* out) {
  GRID_STRIDE(i, N * D) {
    const double h = solid[i % N];
    out[i] = ((a[i] + b * u[i]) - h * lam[i]) / (b + alpha * h);
  }
}

__global__ void k_mult(int64_t N, int D, const double* a, const double* lam, const double* u, const double* ut,
                       const double* solid, double alpha, double b, double* an, double* ln) {
  GRID_STRIDE(i, N * D) {
    const double h = solid[i % N];
    an[i] = a[i] + b * (u[i] - ut[i]);
    ln[i] = lam[i] + alpha * (h * ut[i]);
  }
}

template <int D>
__global__ void k_pol(int64_t N, const double* grad, const double* dif, const double* adv, const double* forcing,
                      double a0, double b00, double b01, double b02, double g0, double g1, double g2, double* w,
                      double* s) {
  const double b0[3] = {b00, b01, b02}, gc[3] = {g0, g1, g2};
  GRID_STRIDE(x, N) {
    const double contrast = dif[x] - a0;
    double sv = forcing[x];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double tg = grad[c * N + x] + gc[c];
      w[c * N + x] = contrast * tg;
      sv = sv - (adv[c * N + x] - b0[c]) * tg;
    }
    s[x] = sv;
  }
}

template <int D>
__global__ void k_tmu(KGeom g, KTabs T, const double2* wh, const double2* sh, const double* lap, double a0,
                      double b00, double b01, double b02, double2* chi, double2* grad) {
  const double b0[3] = {b00, b01, b02};
  const int64_t N = g.size;
  GRID_STRIDE(m, N) {
    int idx[3];
    kidx(g, m, idx);
    double kc[D];
    double2 f = sh[m];
    double bk = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const int ax = 3 - D + c;
      kc[c] = T.k[ax][idx[ax]];
      f = cadd(f, cik(kc[c], wh[c * N + m]));
    }
#pragma unroll
    for (int c = 0; c < D; ++c) bk = bk + b0[c] * kc[c];
    const double2 den = m == 0 ? make_double2(1.0, 0.0) : make_double2(0.0 + a0 * lap[m], bk + 0.0);
    double2 ch = cdiv_np(f, den);
    if (m == 0) ch = make_double2(0.0, 0.0);
    chi[m] = ch;
#pragma unroll
    for (int c = 0; c < D; ++c) grad[c * N + m] = cik(kc[c], ch);
  }
}

// numpy.packbits order (first voxel in the most significant bit of byte 0) ->
// one uint8 0/1 per voxel; one byte in, eight out (one 8-byte store) per thread.
__global__ void k_unpack_bits(const uint8_t* __restrict__ bits, uint8_t* __restrict__ out, int64_t n) {
  const int64_t nbytes = (n + 7) / 8;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbytes; b += (int64_t)gridDim.x * blockDim.x) {
    const unsigned v = bits[b];
    unsigned long long w = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) w |= (unsigned long long)((v >> (7 - k)) & 1u) << (8 * k);
    if (8 * b + 8 <= n && ((reinterpret_cast<uintptr_t>(out) & 7) == 0)) {
      reinterpret_cast<unsigned long long*>(out)[b] = w;
    } else {
      for (int k = 0; k < 8 && 8 * b + k < n; ++k) out[8 * b + k] = (uint8_t)((w >> (8 * k)) & 0xffu);
    }
  }
}

static int finish(cudaStream_t s) {
  (void)s;
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_k_stokes_velocity_update(int ndim, const int64_t* dims, const double* q_hat, const double* a_hat,
                                const double* ut_hat, const double* const* kappas, const double* lap,
                                const double* kappa_sq, double nu, double beta, double b, const double* g_p,
                                double* u_hat, void* stream) {
  KGeom g;
  PF_CK(kgeom(ndim, dims, g));
  PF_ARG(q_hat && a_hat && ut_hat && kappas && lap && kappa_sq && g_p && u_hat, "null argument");
  KTabs T{{nullptr, nullptr, nullptr}};
  for (int j = 0; j < ndim; ++j) T.k[3 - ndim + j] = kappas[j];
  double gp[3] = {0, 0, 0};
  for (int j = 0; j < ndim; ++j) gp[j] = g_p[j];
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = blocks_for(g.size);
  auto Q = (const double2*)q_hat;
  auto AH = (const double2*)a_hat;
  auto UT = (const double2*)ut_hat;
  auto O = (double2*)u_hat;
  switch (ndim) {
    case 1: k_svu<1><<<nb, kThreads, 0, s>>>(g, T, Q, AH, UT, lap, kappa_sq, nu, beta, b, gp[0], gp[1], gp[2], O); break;
    case 2: k_svu<2><<<nb, kThreads, 0, s>>>(g, T, Q, AH, UT, lap, kappa_sq, nu, beta, b, gp[0], gp[1], gp[2], O); break;
    default: k_svu<3><<<nb, kThreads, 0, s>>>(g, T, Q, AH, UT, lap, kappa_sq, nu, beta, b, gp[0], gp[1], gp[2], O); break;
  }
  return finish(s);
}

int pf_k_aux_velocity_update(int ndim, const int64_t* dims, const double* u, const double* a, const double* lam,
                             const double* solid, double alpha, double b, double* out, void* stream) {
  KGeom g;
  PF_CK(kgeom(ndim, dims, g));
  PF_ARG(u && a && lam && solid && out, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  k_aux<<<blocks_for(g.size * ndim), kThreads, 0, s>>>(g.size, ndim, u, a, lam, solid, alpha, b, out);
  return finish(s);
}

int pf_k_multiplier_update(int ndim, const int64_t* dims, const double* a, const double* lam, const double* u,
                           const double* ut, const double* solid, double alpha, double b, double* a_new,
                           double* lam_new, void* stream) {
  KGeom g;
  PF_CK(kgeom(ndim, dims, g));
  PF_ARG(a && lam && u && ut && solid && a_new && lam_new, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  k_mult<<<blocks_for(g.size * ndim), kThreads, 0, s>>>(g.size, ndim, a, lam, u, ut, solid, alpha, b, a_new, lam_new);
  return finish(s);
}

int pf_k_transport_polarization(int ndim, const int64_t* dims, const double* grad_chi, const double* diffusivity,
                                const double* advection, const double* forcing, double a0, const double* b0v,
                                const double* gch, double* w, double* s_out, void* stream) {
  KGeom g;
  PF_CK(kgeom(ndim, dims, g));
  PF_ARG(grad_chi && diffusivity && advection && forcing && b0v && gch && w && s_out, "null argument");
  double b0[3] = {0, 0, 0}, gc[3] = {0, 0, 0};
  for (int j = 0; j < ndim; ++j) {
    b0[j] = b0v[j];
    gc[j] = gch[j];
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = blocks_for(g.size);
#define POL(D) k_pol<D><<<nb, kThreads, 0, s>>>(g.size, grad_chi, diffusivity, advection, forcing, a0, b0[0], b0[1], b0[2], gc[0], gc[1], gc[2], w, s_out)
  switch (ndim) {
    case 1: POL(1); break;
    case 2: POL(2); break;
    default: POL(3); break;
  }
#undef POL
  return finish(s);
}

int pf_k_transport_mode_update(int ndim, const int64_t* dims, const double* w_hat, const double* s_hat,
                               const double* const* kappas, const double* lap, double a0, const double* b0v,
                               double* chi_hat, double* grad_hat, void* stream) {
  KGeom g;
  PF_CK(kgeom(ndim, dims, g));
  PF_ARG(w_hat && s_hat && kappas && lap && b0v && chi_hat && grad_hat, "null argument");
  KTabs T{{nullptr, nullptr, nullptr}};
  for (int j = 0; j < ndim; ++j) T.k[3 - ndim + j] = kappas[j];
  double b0[3] = {0, 0, 0};
  for (int j = 0; j < ndim; ++j) b0[j] = b0v[j];
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = blocks_for(g.size);
  auto W = (const double2*)w_hat;
  auto S = (const double2*)s_hat;
  auto C = (double2*)chi_hat;
  auto G = (double2*)grad_hat;
  switch (ndim) {
    case 1: k_tmu<1><<<nb, kThreads, 0, s>>>(g, T, W, S, lap, a0, b0[0], b0[1], b0[2], C, G); break;
    case 2: k_tmu<2><<<nb, kThreads, 0, s>>>(g, T, W, S, lap, a0, b0[0], b0[1], b0[2], C, G); break;
    default: k_tmu<3><<<nb, kThreads, 0, s>>>(g, T, W, S, lap, a0, b0[0], b0[1], b0[2], C, G); break;
  }
  return finish(s);
}

int pf_unpack_bits(const uint8_t* bits, uint8_t* out, int64_t n, void* stream) {
  PF_ARG(n >= 0, "negative count");
  if (n == 0) return PF_OK;
  PF_ARG(bits && out, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  k_unpack_bits<<<blocks_for((n + 7) / 8), kThreads, 0, s>>>(bits, out, n);
  return finish(s);
}

}  // extern "C"
