// Effective properties on device — reference pkg/src/poreflow/effective.py:32-108
// and porosity (grid.py:108-110).
//
// permeability: K_ij = h^d * sum_pore sum_{c,m} d_m u^i_c * d_m u^j_c  (effective.py:43-72)
//   per velocity component c: d D2Z transforms, a gradient kernel (i k_m / n), d Z2D
//   batches, then one masked Gram-partials kernel over the d x d gradient fields.
// diffusivity: D_ij = phi delta_ij + Pe h^d sum_pore (ubar^i_i - u^i_i) chi^j
//                     + h^d sum_pore d_i chi^j                           (effective.py:75-108)
#include <cmath>

#include "pf_internal.cuh"

namespace pf {

int pore_sums_host(pf_plan* p, const uint8_t* H, const double* f, int ncomp, double* out5);

__global__ void k_reduce_rows_e(const double* __restrict__ part, int nrows, int nb, double* __restrict__ out) {
  for (int r = 0; r < nrows; ++r) {
    double v[1];
    reduce_partials<1>(part + (size_t)r * nb, nb, v);
    if (threadIdx.x == 0) out[r] = v[0];
  }
}

__global__ void __launch_bounds__(kThreads) k_solid_count(const int64_t n, const uint8_t* __restrict__ H,
                                                          unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
    c += H[x];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, c);  // integer: order-independent
}

// G_m = i k_m F / n for m < D (spectral gradient of one scalar, spectral.py:118-124)
template <int D>
__global__ void __launch_bounds__(kThreads) k_grad_spectrum(Geom g, const double* k0, const double* k1,
                                                            const double* k2, const double2* __restrict__ F,
                                                            double2* __restrict__ G) {
  const double* kt[3] = {k0, k1, k2};
  const uint32_t nh = (uint32_t)g.nh, n2h = (uint32_t)g.n2h, n1 = (uint32_t)g.n[1];
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < nh; m += gridDim.x * blockDim.x) {
    const uint32_t t = m / n2h;
    const int idx[3] = {(int)(t / n1), (int)(t % n1), (int)(m - t * n2h)};
    const double2 f = make_double2(F[m].x * g.inv_n, F[m].y * g.inv_n);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const int ax = 3 - D + c;
      G[(size_t)c * nh + m] = cik(__ldg(kt[ax] + idx[ax]), f);
    }
  }
}

// Gram partials for one velocity component: pairs (i <= j) of flows,
// sum_x pore * sum_m G[i][m] G[j][m].  G layout: [flow][m][x].
template <int D>
__global__ void __launch_bounds__(kThreads) k_gram(const int64_t n, const double* __restrict__ G,
                                                   const uint8_t* __restrict__ H, double* __restrict__ part) {
  constexpr int NP = D * (D + 1) / 2;
  double acc[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) acc[k] = 0.0;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const double pore = 1.0 - (double)H[x];
    double v[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int m = 0; m < D; ++m) v[i][m] = pore * G[((size_t)i * D + m) * n + x];
    int k = 0;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = i; j < D; ++j) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) s += v[i][m] * v[j][m];
        acc[k++] += s;
      }
  }
  block_sum<NP>(acc);
  if (threadIdx.x == 0)
    for (int k = 0; k < NP; ++k) part[(size_t)k * gridDim.x + blockIdx.x] = acc[k];
}

struct DiffPtrs {
  const double* ui[3];     // component i of flow i
  const double* chi[3];    // chi^j
  const double* gchi[3];   // grad chi^j, [i][x]
  double ubar[3];          // pore average of component i of flow i
};

template <int D>
__global__ void __launch_bounds__(kThreads) k_diff_sums(const int64_t n, DiffPtrs P, const uint8_t* __restrict__ H,
                                                        double* __restrict__ part) {
  double acc[2 * D * D];
#pragma unroll
  for (int k = 0; k < 2 * D * D; ++k) acc[k] = 0.0;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const double pore = 1.0 - (double)H[x];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const double fl = pore * (P.ubar[i] - P.ui[i][x]);
#pragma unroll
      for (int j = 0; j < D; ++j) {
        acc[i * D + j] += fl * P.chi[j][x];
        acc[D * D + i * D + j] += pore * P.gchi[j][(size_t)i * n + x];
      }
    }
  }
  block_sum<2 * D * D>(acc);
  if (threadIdx.x == 0)
    for (int k = 0; k < 2 * D * D; ++k) part[(size_t)k * gridDim.x + blockIdx.x] = acc[k];
}

static int solid_count(pf_plan* p, const uint8_t* solid, int64_t* out) {
  unsigned long long* d = reinterpret_cast<unsigned long long*>(p->partials + 31 * kMaxBlocks);
  PF_CK_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), p->work));
  k_solid_count<<<blocks_for(p->g.nr), kThreads, 0, p->work>>>(p->g.nr, solid, d);
  PF_CK_CUDA(cudaGetLastError());
  PF_CK_CUDA(cudaMemcpyAsync(p->h_small, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost, p->work));
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  *out = (int64_t)(*reinterpret_cast<unsigned long long*>(p->h_small));
  return PF_OK;
}

template <int D>
static int permeability_t(pf_plan* p, const uint8_t* solid, const double* const* us, double* K) {
  const Geom& g = p->g;
  const int64_t n = g.nr, nh = g.nh;
  // gradient fields of all D flows for one velocity component: D*D*n doubles.
  static_assert(D >= 1, "");
  double* G = nullptr;
  PF_CK_CUDA(cudaMallocAsync((void**)&G, sizeof(double) * D * D * n, p->work));
  const int nb = blocks_for(n);
  constexpr int NP = D * (D + 1) / 2;
  double* part = p->partials;  // [c][pair][nb]
  int st = PF_OK;
  for (int c = 0; c < D && st == PF_OK; ++c) {
    for (int i = 0; i < D && st == PF_OK; ++i) {
      st = plan_fft(p, true, 1, (void*)(us[i] + (size_t)c * n), p->spec1);
      if (st != PF_OK) break;
      k_grad_spectrum<D><<<blocks_for(nh), kThreads, 0, p->work>>>(g, p->kap[0], p->kap[1], p->kap[2], p->spec1,
                                                                    p->specB);
      st = plan_fft(p, false, D, p->specB, G + (size_t)i * D * n);
    }
    if (st != PF_OK) break;
    k_gram<D><<<nb, kThreads, 0, p->work>>>(n, G, solid, part + (size_t)c * NP * nb);
  }
  if (st == PF_OK) {
    double* out = p->partials + 24 * kMaxBlocks;
    k_reduce_rows_e<<<1, kFinalizeThreads, 0, p->work>>>(part, D * NP, nb, out);
    cudaMemcpyAsync(p->h_small, out, sizeof(double) * D * NP, cudaMemcpyDeviceToHost, p->work);
  }
  cudaFreeAsync(G, p->work);
  PF_CK(st);
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  double cell = 1.0;
  for (int j = 0; j < D; ++j) cell *= 1.0 / g.n[3 - D + j];
  int k = 0;
  double T[3][3];
  for (int i = 0; i < D; ++i)
    for (int j = i; j < D; ++j, ++k) {
      double s = 0.0;
      for (int c = 0; c < D; ++c) s += p->h_small[c * NP + k];
      T[i][j] = T[j][i] = s;
    }
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) K[i * D + j] = T[i][j] * cell;
  return PF_OK;
}

template <int D>
static int diffusivity_t(pf_plan* p, const uint8_t* solid, const double* const* us, const double* const* chi,
                         const double* const* gchi, double pe, double* Dout) {
  const Geom& g = p->g;
  const int64_t n = g.nr;
  int64_t ns = 0;
  PF_CK(solid_count(p, solid, &ns));
  const double phi = 1.0 - (double)ns / g.dn;  // grid.py:108-110 (mean of uint8)
  PF_ARG(phi != 0.0, "diffusivity undefined: no pore cells");
  DiffPtrs P;
  for (int i = 0; i < D; ++i) {
    double s5[5];
    PF_CK(pore_sums_host(p, solid, us[i], D, s5));  // pore_average(u_i), effective.py:32-40
    P.ubar[i] = s5[i] / s5[3];
    P.ui[i] = us[i] + (size_t)i * n;
    P.chi[i] = chi[i];
    P.gchi[i] = gchi[i];
  }
  const int nb = blocks_for(n);
  k_diff_sums<D><<<nb, kThreads, 0, p->work>>>(n, P, solid, p->partials);
  PF_CK_CUDA(cudaGetLastError());
  double* out = p->partials + 24 * kMaxBlocks;
  k_reduce_rows_e<<<1, kFinalizeThreads, 0, p->work>>>(p->partials, 2 * D * D, nb, out);
  PF_CK_CUDA(cudaMemcpyAsync(p->h_small, out, sizeof(double) * 2 * D * D, cudaMemcpyDeviceToHost, p->work));
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  double cell = 1.0;
  for (int j = 0; j < D; ++j) cell *= 1.0 / g.n[3 - D + j];
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) {
      double v = i == j ? phi : 0.0;
      v += pe * cell * p->h_small[i * D + j];
      v += cell * p->h_small[D * D + i * D + j];
      Dout[i * D + j] = v;
    }
  return PF_OK;
}

// Masked Gram partials of one velocity component over a (slab-local) set of 9
// gradient fields G[flow][axis][x] (3D): the 6 pair sums before the h^3 factor.
int slab_gram_host(pf_plan* p, const uint8_t* solid, const double* G, int64_t n, double* out6) {
  const int nb = blocks_for(n);
  k_gram<3><<<nb, kThreads, 0, p->work>>>(n, G, solid, p->partials);
  PF_CK_CUDA(cudaGetLastError());
  double* out = p->partials + 24 * kMaxBlocks;
  k_reduce_rows_e<<<1, kFinalizeThreads, 0, p->work>>>(p->partials, 6, nb, out);
  PF_CK_CUDA(cudaMemcpyAsync(p->h_small, out, sizeof(double) * 6, cudaMemcpyDeviceToHost, p->work));
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  for (int k = 0; k < 6; ++k) out6[k] = p->h_small[k];
  return PF_OK;
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_solid_count(pf_plan* p, const uint8_t* solid, int64_t* count) {
  PF_ARG(p && solid && count, "null argument");
  PF_CK(enter(p));
  PF_CK(solid_count(p, solid, count));
  return leave(p);
}

int pf_pore_average(pf_plan* p, const uint8_t* solid, const double* f, int ncomp, double* out) {
  PF_ARG(p && solid && f && out, "null argument");
  PF_ARG(ncomp >= 1 && ncomp <= 3, "ncomp must be 1..3");
  if (p->active) {
    set_error("pf_pore_average while a solve is active on this plan");
    return PF_ERR_STATE;
  }
  PF_CK(enter(p));
  double s5[5];
  PF_CK(pore_sums_host(p, solid, f, ncomp, s5));
  if (s5[3] == 0.0) {  // hand the stream ordering back before reporting (no early return past enter())
    leave(p);
    set_error("pore average undefined: no pore cells");
    return PF_ERR_ARG;
  }
  for (int c = 0; c < ncomp; ++c) out[c] = s5[c] / s5[3];
  return leave(p);
}

int pf_permeability(pf_plan* p, const uint8_t* solid, const double* const* us, double* K) {
  PF_NVTX("pf_permeability");
  PF_ARG(p && solid && us && K, "null argument");
  for (int i = 0; i < p->g.d; ++i) PF_ARG(us[i], "null velocity solution %d", i);
  if (p->active) {
    set_error("pf_permeability while a solve is active on this plan");
    return PF_ERR_STATE;
  }
  PF_CK(enter(p));
  PF_CK(plan_ensure_scratch(p));
  switch (p->g.d) {
    case 1: PF_CK(permeability_t<1>(p, solid, us, K)); break;
    case 2: PF_CK(permeability_t<2>(p, solid, us, K)); break;
    default: PF_CK(permeability_t<3>(p, solid, us, K)); break;
  }
  return leave(p);
}

int pf_diffusivity(pf_plan* p, const uint8_t* solid, const double* const* us, const double* const* chi,
                   const double* const* gchi, double pe, double* D) {
  PF_NVTX("pf_diffusivity");
  PF_ARG(p && solid && us && chi && gchi && D, "null argument");
  if (p->active) {
    set_error("pf_diffusivity while a solve is active on this plan");
    return PF_ERR_STATE;
  }
  PF_CK(enter(p));
  switch (p->g.d) {
    case 1: PF_CK(diffusivity_t<1>(p, solid, us, chi, gchi, pe, D)); break;
    case 2: PF_CK(diffusivity_t<2>(p, solid, us, chi, gchi, pe, D)); break;
    default: PF_CK(diffusivity_t<3>(p, solid, us, chi, gchi, pe, D)); break;
  }
  return leave(p);
}

}  // extern "C"
