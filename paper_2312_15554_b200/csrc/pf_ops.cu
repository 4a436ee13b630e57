// Spectral utilities and the step-level helpers of the reference's public API
// (pkg/src/poreflow/spectral.py:101-143, stokes.py:158-244,
// transport.py:131-177) on device pointers, full-spectrum layout:
//
//   pf_k_fftn          fftn over the trailing ndim axes (real or complex in,
//                      complex out), inverse scaled by 1/n  (spectral.py:101-115)
//   pf_k_ifftn_real    Re ifftn                              (spectral.py:107-115)
//   pf_k_spectral_grad 1j*kappa_j*chi_hat                    (spectral.py:118-124)
//   pf_k_spectral_div  [base +] sum_j 1j*kappa_j*v_hat[j]    (spectral.py:127-133,
//                                                             transport.py:149-151)
//   pf_k_scale_modes   (-lap) * chi_hat                       (spectral.py:136-138)
//   pf_k_q_update      q - beta*div, minus its mean           (stokes.py:216-218)
//   pf_k_norm          ||w*(x - y)||_2                        (stokes.py:154-155)
//
// These are not on the solver's hot path (the solvers run the fused / cuFFT
// pipelines); they make the reference's step helpers and transform utilities
// available on the device with the reference's evaluation order.  The library
// is compiled with --fmad=false for this file, so the pointwise arithmetic
// rounds like numpy's; the transforms are cuFFT's (round-off level vs pocketfft).
#include <map>
#include <mutex>
#include <tuple>

#include "pf_internal.cuh"

namespace pf {
namespace ops {

struct Shape {
  int d;
  int64_t n[3];
  int64_t size;
};

static int shape_of(int ndim, const int64_t* dims, Shape& s) {
  PF_ARG(ndim >= 1 && ndim <= 3 && dims, "ndim must be 1..3");
  s.d = ndim;
  s.size = 1;
  s.n[0] = s.n[1] = s.n[2] = 1;
  for (int j = 0; j < ndim; ++j) {
    PF_ARG(dims[j] >= 1, "bad extent");
    s.n[3 - ndim + j] = dims[j];
    s.size *= dims[j];
  }
  PF_ARG(s.size < ((int64_t)1 << 31), "array too large");
  return PF_OK;
}

#define OPS_STRIDE(m, N) \
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < (N); m += (int64_t)gridDim.x * blockDim.x)

__global__ void k_real_to_complex(int64_t count, const double* __restrict__ in, double2* __restrict__ out) {
  OPS_STRIDE(i, count) out[i] = make_double2(in[i], 0.0);
}

__global__ void k_scale_complex(int64_t count, double2* __restrict__ x, double s) {
  OPS_STRIDE(i, count) {
    const double2 v = x[i];
    x[i] = make_double2(v.x * s, v.y * s);
  }
}

__global__ void k_real_part(int64_t count, const double2* __restrict__ in, double s, double* __restrict__ out) {
  OPS_STRIDE(i, count) out[i] = in[i].x * s;
}

// (0 + 1j*k) * z in numpy's complex product order: (0*x - k*y) + 1j*(0*y + k*x)
__device__ __forceinline__ double2 ik_times(double k, double2 z) {
  return make_double2(0.0 * z.x - k * z.y, 0.0 * z.y + k * z.x);
}

struct Kap {
  const double* k[3];
};

__device__ __forceinline__ int64_t axis_index(const Shape& s, int64_t m, int ax) {
  if (ax == 2) return m % s.n[2];
  if (ax == 1) return (m / s.n[2]) % s.n[1];
  return m / (s.n[2] * s.n[1]);
}

__global__ void k_grad(Shape s, Kap K, int64_t batch, const double2* __restrict__ chi, double2* __restrict__ out) {
  const int64_t N = s.size;
  OPS_STRIDE(i, N * batch) {
    const int64_t m = i % N;
    const int64_t bi = i / N;
    const double2 z = chi[i];
    for (int c = 0; c < s.d; ++c) {
      const int ax = 3 - s.d + c;
      out[(c * batch + bi) * N + m] = ik_times(K.k[ax][axis_index(s, m, ax)], z);
    }
  }
}

// out = base + sum_c 1j*kappa_c*v[c] (base == nullptr: start from the c = 0 term,
// spectral.py:130-133; with base, transport.py:149-151's accumulation order)
__global__ void k_div(Shape s, Kap K, const double2* __restrict__ v, const double2* __restrict__ base,
                      double2* __restrict__ out) {
  const int64_t N = s.size;
  OPS_STRIDE(m, N) {
    double2 acc;
    int c0 = 0;
    if (base) {
      acc = base[m];
    } else {
      acc = ik_times(K.k[3 - s.d][axis_index(s, m, 3 - s.d)], v[m]);
      c0 = 1;
    }
    for (int c = c0; c < s.d; ++c) {
      const int ax = 3 - s.d + c;
      const double2 t = ik_times(K.k[ax][axis_index(s, m, ax)], v[c * N + m]);
      acc = make_double2(acc.x + t.x, acc.y + t.y);
    }
    out[m] = acc;
  }
}

// out = (sign*f) * z, numpy's real-times-complex: (r*x, r*y)
__global__ void k_scale_modes(int64_t N, int64_t batch, const double* __restrict__ f, double sign,
                              const double2* __restrict__ z, double2* __restrict__ out) {
  OPS_STRIDE(i, N * batch) {
    const double r = sign * f[i % N];
    const double2 v = z[i];
    out[i] = make_double2(r * v.x, r * v.y);
  }
}

constexpr int kRedBlocks = 592;  // 4 x 148 SMs

// Deterministic two-level sum of squares (or plain sum) over count elements:
// each block writes one partial, one block adds the partials in a fixed order.
template <int MODE>  // 0: sum (x - beta*y) -> stored in out; 1: sum (w*(x - y))^2
__global__ void k_partials(int64_t count, const double* __restrict__ x, const double* __restrict__ y, double beta,
                           const double* __restrict__ w, int64_t w_period, double* __restrict__ out,
                           double* __restrict__ partial) {
  __shared__ double sh[kThreads];
  double acc = 0.0;
  OPS_STRIDE(i, count) {
    if (MODE == 0) {
      const double v = x[i] - beta * y[i];
      out[i] = v;
      acc += v;
    } else {
      double v = y ? x[i] - y[i] : x[i];
      if (w) v = w[i % w_period] * v;
      acc += v * v;
    }
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void k_sum_partials(int nb, const double* __restrict__ partial, double* __restrict__ total) {
  __shared__ double sh[kThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += kThreads) acc += partial[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) total[0] = sh[0];
}

__global__ void k_sub_mean(int64_t count, double* __restrict__ x, const double* __restrict__ total) {
  const double mean = total[0] / (double)count;
  OPS_STRIDE(i, count) x[i] = x[i] - mean;
}

// ---------------------------------------------------------------- cuFFT Z2Z plan cache
struct PlanKey {
  int device, ndim;
  int64_t n0, n1, n2, batch;
  bool operator<(const PlanKey& o) const {
    return std::tie(device, ndim, n0, n1, n2, batch) < std::tie(o.device, o.ndim, o.n0, o.n1, o.n2, o.batch);
  }
};

static std::mutex g_plan_mu;
static std::map<PlanKey, cufftHandle> g_plans;

static int z2z_plan(int ndim, const int64_t* dims, int64_t batch, cufftHandle* out) {
  int dev = 0;
  PF_CK_CUDA(cudaGetDevice(&dev));
  PlanKey key{dev, ndim, dims[0], ndim > 1 ? dims[1] : 1, ndim > 2 ? dims[2] : 1, batch};
  auto it = g_plans.find(key);
  if (it != g_plans.end()) {
    *out = it->second;
    return PF_OK;
  }
  int n[3];
  int64_t size = 1;
  for (int j = 0; j < ndim; ++j) {
    n[j] = (int)dims[j];
    size *= dims[j];
  }
  PF_ARG(batch >= 1 && batch * size < ((int64_t)1 << 31), "fft batch too large");
  cufftHandle h;
  PF_CK_FFT(cufftPlanMany(&h, ndim, n, nullptr, 1, (int)size, nullptr, 1, (int)size, CUFFT_Z2Z, (int)batch));
  g_plans[key] = h;
  *out = h;
  return PF_OK;
}

static int grid_blocks(int64_t work) { return blocks_for(work); }

}  // namespace ops
}  // namespace pf

using namespace pf;
using namespace pf::ops;

extern "C" {

int pf_k_fftn(int ndim, const int64_t* dims, int64_t batch, const double* in, int in_complex, double* out,
              int inverse, void* stream) {
  PF_NVTX("pf_k_fftn");
  Shape s;
  PF_CK(shape_of(ndim, dims, s));
  PF_ARG(in && out && batch >= 1, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t count = s.size * batch;
  auto O = (cufftDoubleComplex*)out;
  if (!in_complex) {
    k_real_to_complex<<<grid_blocks(count), kThreads, 0, st>>>(count, in, (double2*)out);
  } else if (in != out) {
    PF_CK_CUDA(cudaMemcpyAsync(out, in, count * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  }
  std::lock_guard<std::mutex> lock(g_plan_mu);
  cufftHandle h;
  PF_CK(z2z_plan(ndim, dims, batch, &h));
  PF_CK_FFT(cufftSetStream(h, st));
  PF_CK_FFT(cufftExecZ2Z(h, O, O, inverse ? CUFFT_INVERSE : CUFFT_FORWARD));
  if (inverse) k_scale_complex<<<grid_blocks(count), kThreads, 0, st>>>(count, (double2*)out, 1.0 / (double)s.size);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

int pf_k_ifftn_real(int ndim, const int64_t* dims, int64_t batch, const double* in, double* work, double* out,
                    void* stream) {
  PF_NVTX("pf_k_ifftn_real");
  Shape s;
  PF_CK(shape_of(ndim, dims, s));
  PF_ARG(in && work && out && batch >= 1, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t count = s.size * batch;
  if (in != work) PF_CK_CUDA(cudaMemcpyAsync(work, in, count * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  {
    std::lock_guard<std::mutex> lock(g_plan_mu);
    cufftHandle h;
    PF_CK(z2z_plan(ndim, dims, batch, &h));
    PF_CK_FFT(cufftSetStream(h, st));
    PF_CK_FFT(cufftExecZ2Z(h, (cufftDoubleComplex*)work, (cufftDoubleComplex*)work, CUFFT_INVERSE));
  }
  k_real_part<<<grid_blocks(count), kThreads, 0, st>>>(count, (const double2*)work, 1.0 / (double)s.size, out);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

int pf_k_spectral_grad(int ndim, const int64_t* dims, int64_t batch, const double* const* kappas,
                       const double* chi_hat, double* out, void* stream) {
  Shape s;
  PF_CK(shape_of(ndim, dims, s));
  PF_ARG(kappas && chi_hat && out && batch >= 1, "null argument");
  Kap K{{nullptr, nullptr, nullptr}};
  for (int j = 0; j < ndim; ++j) K.k[3 - ndim + j] = kappas[j];
  cudaStream_t st = (cudaStream_t)stream;
  k_grad<<<grid_blocks(s.size * batch), kThreads, 0, st>>>(s, K, batch, (const double2*)chi_hat, (double2*)out);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

int pf_k_spectral_div(int ndim, const int64_t* dims, const double* const* kappas, const double* v_hat,
                      const double* base, double* out, void* stream) {
  Shape s;
  PF_CK(shape_of(ndim, dims, s));
  PF_ARG(kappas && v_hat && out, "null argument");
  Kap K{{nullptr, nullptr, nullptr}};
  for (int j = 0; j < ndim; ++j) K.k[3 - ndim + j] = kappas[j];
  cudaStream_t st = (cudaStream_t)stream;
  k_div<<<grid_blocks(s.size), kThreads, 0, st>>>(s, K, (const double2*)v_hat, (const double2*)base,
                                                  (double2*)out);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

int pf_k_scale_modes(int64_t n_modes, int64_t batch, const double* factor, double sign, const double* z,
                     double* out, void* stream) {
  PF_ARG(n_modes >= 1 && batch >= 1 && factor && z && out, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  k_scale_modes<<<grid_blocks(n_modes * batch), kThreads, 0, st>>>(n_modes, batch, factor, sign,
                                                                   (const double2*)z, (double2*)out);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

int pf_k_q_update(int64_t count, const double* q, const double* div, double beta, double* out, double* scratch,
                  void* stream) {
  PF_ARG(count >= 1 && q && div && out && scratch, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = (int)std::min<int64_t>(kRedBlocks, (count + kThreads - 1) / kThreads);
  k_partials<0><<<nb, kThreads, 0, st>>>(count, q, div, beta, nullptr, 1, out, scratch);
  k_sum_partials<<<1, kThreads, 0, st>>>(nb, scratch, scratch + kRedBlocks);
  k_sub_mean<<<grid_blocks(count), kThreads, 0, st>>>(count, out, scratch + kRedBlocks);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

int pf_k_norm(int64_t count, const double* x, const double* y, const double* w, int64_t w_period, double* scratch,
              double* result_host, void* stream) {
  PF_ARG(count >= 0 && x && scratch && result_host, "null argument");
  PF_ARG(!w || w_period >= 1, "weight period must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  if (count == 0) {
    *result_host = 0.0;
    return PF_OK;
  }
  const int nb = (int)std::min<int64_t>(kRedBlocks, (count + kThreads - 1) / kThreads);
  k_partials<1><<<nb, kThreads, 0, st>>>(count, x, y, 0.0, w, w_period, nullptr, scratch);
  k_sum_partials<<<1, kThreads, 0, st>>>(nb, scratch, scratch + kRedBlocks);
  double ss = 0.0;
  PF_CK_CUDA(cudaMemcpyAsync(&ss, scratch + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost, st));
  PF_CK_CUDA(cudaStreamSynchronize(st));
  *result_host = sqrt(ss);
  return PF_OK;
}

int pf_k_scratch_doubles(void) { return kRedBlocks + 1; }

}  // extern "C"
