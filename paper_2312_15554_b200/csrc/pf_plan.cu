// Plan lifecycle, symbol tables, cuFFT plans, scratch, and the CUDA-graph
// iteration driver shared by the Stokes and transport solvers.
#include <cmath>
#include <cstdarg>
#include <cstring>

#include "pf_internal.cuh"

namespace pf {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const char* cufft_name(cufftResult r) {
  switch (r) {
    case CUFFT_SUCCESS: return "CUFFT_SUCCESS";
    case CUFFT_INVALID_PLAN: return "CUFFT_INVALID_PLAN";
    case CUFFT_ALLOC_FAILED: return "CUFFT_ALLOC_FAILED";
    case CUFFT_INVALID_TYPE: return "CUFFT_INVALID_TYPE";
    case CUFFT_INVALID_VALUE: return "CUFFT_INVALID_VALUE";
    case CUFFT_INTERNAL_ERROR: return "CUFFT_INTERNAL_ERROR";
    case CUFFT_EXEC_FAILED: return "CUFFT_EXEC_FAILED";
    case CUFFT_SETUP_FAILED: return "CUFFT_SETUP_FAILED";
    case CUFFT_INVALID_SIZE: return "CUFFT_INVALID_SIZE";
    default: return "CUFFT_ERROR";
  }
}

// Per-axis symbol tables exactly as spectral.py:78-86 computes them:
// k = (2*pi) * (m * val), val = 1/(n*(1/n)) (numpy fftfreq with d = 1/n),
// central: kappa = sin(h k)/h, lap1d = 4 sin(h k/2)^2 / h^2; exact: k, k^2.
// Nyquist kappa of an even axis is zero in both modes.
int symbol_tables_for(int mode, int n, std::vector<double>& kap, std::vector<double>& ell) {
  kap.assign(n, 0.0);
  ell.assign(n, 0.0);
  const double h = 1.0 / n;
  const double val = 1.0 / (n * (1.0 / n));
  const double two_pi = 2.0 * M_PI;
  const int npos = (n - 1) / 2 + 1;
  for (int i = 0; i < n; ++i) {
    const int m = i < npos ? i : i - n;
    const double k = two_pi * ((double)m * val);
    if (mode == PF_SYMBOLS_EXACT) {
      kap[i] = k;
      ell[i] = k * k;
    } else {
      kap[i] = std::sin(h * k) / h;
      const double s = std::sin(0.5 * h * k);
      ell[i] = 4.0 * (s * s) / (h * h);
    }
  }
  if (n % 2 == 0) kap[n / 2] = 0.0;
  return PF_OK;
}

int enter(pf_plan* p) {
  PF_CK_CUDA(cudaSetDevice(p->device));
  PF_CK_CUDA(cudaEventRecord(p->ev_user, p->user_stream));
  PF_CK_CUDA(cudaStreamWaitEvent(p->work, p->ev_user, 0));
  return PF_OK;
}

int leave(pf_plan* p) {
  PF_CK_CUDA(cudaEventRecord(p->ev_work, p->work));
  PF_CK_CUDA(cudaStreamWaitEvent(p->user_stream, p->ev_work, 0));
  return PF_OK;
}

int plan_reset_work_areas(pf_plan* p) {
  for (int k = 0; k < 4; ++k) {
    if (p->fwd[k]) PF_CK_FFT(cufftSetWorkArea(p->fwd[k], p->fft_work));
    if (p->inv[k]) PF_CK_FFT(cufftSetWorkArea(p->inv[k], p->fft_work));
  }
  p->graph.reset();  // captured graphs reference the old work area
  return PF_OK;
}

static int slot_of(pf_plan* p, int batch) {
  for (int i = 0; i < 4; ++i)
    if (p->batch_of[i] == batch) return i;
  for (int i = 0; i < 4; ++i)
    if (p->batch_of[i] == 0) {
      p->batch_of[i] = batch;
      return i;
    }
  return -1;
}

// Create (once) the D2Z and Z2D plans for `batch` stacked fields, sharing one
// work area across all plans of this pf_plan (they run serially on p->work).
static int ensure_fft(pf_plan* p, int batch) {
  int s = slot_of(p, batch);
  PF_ARG(s >= 0, "too many distinct FFT batch sizes");
  if (p->fwd[s] && p->inv[s]) return PF_OK;
  const int d = p->g.d;
  long long dims[3];
  for (int j = 0; j < d; ++j) dims[j] = p->g.n[3 - d + j];
  const long long dist_r = p->g.nr, dist_c = p->g.nh;
  size_t ws_f = 0, ws_i = 0;
  cufftHandle f, i;
  PF_CK_FFT(cufftCreate(&f));
  PF_CK_FFT(cufftSetAutoAllocation(f, 0));
  PF_CK_FFT(cufftMakePlanMany64(f, d, dims, nullptr, 1, dist_r, nullptr, 1, dist_c, CUFFT_D2Z, batch, &ws_f));
  PF_CK_FFT(cufftCreate(&i));
  PF_CK_FFT(cufftSetAutoAllocation(i, 0));
  PF_CK_FFT(cufftMakePlanMany64(i, d, dims, nullptr, 1, dist_c, nullptr, 1, dist_r, CUFFT_Z2D, batch, &ws_i));
  p->fwd[s] = f;
  p->inv[s] = i;
  size_t need = ws_f > ws_i ? ws_f : ws_i;
  if (need > p->fft_work_bytes) {
    PF_CK_CUDA(cudaStreamSynchronize(p->work));
    if (p->fft_work) PF_CK_CUDA(cudaFree(p->fft_work));
    PF_CK_CUDA(cudaMalloc(&p->fft_work, need));
    p->fft_work_bytes = need;
    for (int k = 0; k < 4; ++k) {
      if (p->fwd[k]) PF_CK_FFT(cufftSetWorkArea(p->fwd[k], p->fft_work));
      if (p->inv[k]) PF_CK_FFT(cufftSetWorkArea(p->inv[k], p->fft_work));
    }
    p->graph.reset();  // captured graphs reference the old work area
  } else {
    PF_CK_FFT(cufftSetWorkArea(f, p->fft_work));
    PF_CK_FFT(cufftSetWorkArea(i, p->fft_work));
  }
  PF_CK_FFT(cufftSetStream(f, p->work));
  PF_CK_FFT(cufftSetStream(i, p->work));
  return PF_OK;
}

int plan_fft(pf_plan* p, bool forward, int batch, void* in, void* out) {
  PF_CK(ensure_fft(p, batch));
  int s = slot_of(p, batch);
  if (forward) {
    PF_CK_FFT(cufftExecD2Z(p->fwd[s], (cufftDoubleReal*)in, (cufftDoubleComplex*)out));
  } else {
    PF_CK_FFT(cufftExecZ2D(p->inv[s], (cufftDoubleComplex*)in, (cufftDoubleReal*)out));
  }
  return PF_OK;
}

int plan_ensure_scratch(pf_plan* p) {
  if (p->specA) return PF_OK;
  const int d = p->g.d;
  const int64_t nh = p->g.nh, nr = p->g.nr;
  size_t bytes = 0;
  auto alloc = [&](void** ptr, size_t n) -> int {
    PF_CK_CUDA(cudaMalloc(ptr, n));
    bytes += n;
    return PF_OK;
  };
  PF_CK(alloc((void**)&p->specA, sizeof(double2) * (d + 1) * nh));
  PF_CK(alloc((void**)&p->specB, sizeof(double2) * (d + 1) * nh));
  PF_CK(alloc((void**)&p->spec1, sizeof(double2) * nh));
  PF_CK(alloc((void**)&p->spec2, sizeof(double2) * nh));
  PF_CK(alloc((void**)&p->realA, sizeof(double) * (d + 1) * nr));
  PF_CK(alloc((void**)&p->realB, sizeof(double) * (d + 1) * nr));
  p->scratch_bytes += bytes;
  for (int b : {1, d, d + 1}) PF_CK(ensure_fft(p, b));
  return PF_OK;
}

#ifndef PF_GRAPH_ITERS_LARGE
#define PF_GRAPH_ITERS_LARGE 4  // iterations per graph chunk for grids of >= 2^21 points
#endif

// Run up to n_iter iterations of the active solver in CUDA-graph chunks.
// Every kernel of an iteration is gated on ctrl->done, so chunks launched
// after convergence are no-ops apart from cuFFT passes on scratch buffers.
int run_chunks(pf_plan* p, int64_t n_iter, int poll, int (*enqueue)(pf_plan*), Ctrl* out) {
  if (n_iter <= 0) {
    PF_CK_CUDA(cudaMemcpyAsync(&p->h_ctrl[0], p->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, p->work));
    PF_CK_CUDA(cudaStreamSynchronize(p->work));
    *out = p->h_ctrl[0];
    return PF_OK;
  }
  const int64_t nr = p->g.nr;
  const int K = nr >= (1 << 21) ? PF_GRAPH_ITERS_LARGE : (nr >= (1 << 15) ? 8 : 16);
  if (!p->graph.exec || p->graph.iters != K) {
    p->graph.reset();
    PF_CK_CUDA(cudaStreamBeginCapture(p->work, cudaStreamCaptureModeThreadLocal));
    int st = PF_OK;
    for (int k = 0; k < K && st == PF_OK; ++k) st = enqueue(p);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(p->work, &g);
    if (st != PF_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    PF_CK_CUDA(e);
    p->graph.graph = g;
    PF_CK_CUDA(cudaGraphInstantiate(&p->graph.exec, g, 0));
    p->graph.iters = K;
  }
  const int64_t full = n_iter / K, rem = n_iter % K;
  if (!poll) {
    for (int64_t c = 0; c < full; ++c) PF_CK_CUDA(cudaGraphLaunch(p->graph.exec, p->work));
    for (int64_t r = 0; r < rem; ++r) PF_CK(enqueue(p));
    out->iter = -1;  // not observed: no host synchronisation in this mode
    return PF_OK;
  }
  // Polling: keep two chunks in flight; each chunk ends with a copy of the
  // control block into its pinned slot and an event.
  int64_t launched = 0, checked = 0;
  bool done = false;
  auto launch = [&](int64_t c) -> int {
    const int slot = (int)(c & 1);
    if (c < full) {
      PF_CK_CUDA(cudaGraphLaunch(p->graph.exec, p->work));
    } else {
      for (int64_t r = 0; r < rem; ++r) PF_CK(enqueue(p));
    }
    PF_CK_CUDA(cudaMemcpyAsync(&p->h_ctrl[slot], p->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, p->work));
    PF_CK_CUDA(cudaEventRecord(p->ev_poll[slot], p->work));
    return PF_OK;
  };
  const int64_t nchunks = full + (rem ? 1 : 0);
  while (checked < nchunks) {
    while (!done && launched < nchunks && launched - checked < 2) PF_CK(launch(launched++));
    if (checked >= launched) break;
    const int slot = (int)(checked & 1);
    PF_CK_CUDA(cudaEventSynchronize(p->ev_poll[slot]));
    Ctrl c = p->h_ctrl[slot];
    ++checked;
    if (c.done) done = true;
    if (done && checked >= launched) break;
  }
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  *out = p->h_ctrl[(int)((launched - 1) & 1)];
  return PF_OK;
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_version(void) { return 100; }

const char* pf_last_error(void) { return g_err; }

int pf_plan_create(pf_plan** out, int ndim, const int64_t* dims, int symbol_mode, int device, void* stream) {
  PF_ARG(out != nullptr && dims != nullptr, "null argument");
  PF_ARG(ndim >= 1 && ndim <= 3, "ndim must be 1, 2 or 3 (got %d)", ndim);
  PF_ARG(symbol_mode == PF_SYMBOLS_EXACT || symbol_mode == PF_SYMBOLS_CENTRAL, "bad symbol mode %d", symbol_mode);
  for (int j = 0; j < ndim; ++j) PF_ARG(dims[j] >= 4 && dims[j] <= (1 << 16), "bad grid extent %lld", (long long)dims[j]);
  *out = nullptr;
  PF_CK_CUDA(cudaSetDevice(device));
  pf_plan* p = new pf_plan();  // value-initialised: every pointer/handle starts at 0
  p->g.d = ndim;
  for (int k = 0; k < 3; ++k) p->g.n[k] = 1;
  for (int j = 0; j < ndim; ++j) p->g.n[3 - ndim + j] = (int)dims[j];
  p->g.n2h = p->g.n[2] / 2 + 1;
  p->g.nr = (int64_t)p->g.n[0] * p->g.n[1] * p->g.n[2];
  p->g.nh = (int64_t)p->g.n[0] * p->g.n[1] * p->g.n2h;
  p->g.dn = (double)p->g.nr;
  p->g.inv_n = 1.0 / p->g.dn;
  PF_ARG(p->g.nr < (int64_t)1 << 31, "grid too large for one plan (n = %lld)", (long long)p->g.nr);
  p->mode = symbol_mode;
  p->device = device;
  p->user_stream = (cudaStream_t)stream;
  p->fused_enable = 1;
  p->compact_enable = 1;
  PF_CK_CUDA(cudaStreamCreateWithFlags(&p->work, cudaStreamNonBlocking));
  PF_CK_CUDA(cudaEventCreateWithFlags(&p->ev_user, cudaEventDisableTiming));
  PF_CK_CUDA(cudaEventCreateWithFlags(&p->ev_work, cudaEventDisableTiming));
  PF_CK_CUDA(cudaEventCreateWithFlags(&p->ev_poll[0], cudaEventDisableTiming));
  PF_CK_CUDA(cudaEventCreateWithFlags(&p->ev_poll[1], cudaEventDisableTiming));
  for (int ax = 0; ax < 3; ++ax) {
    const int n = p->g.n[ax];
    if (ax < 3 - ndim) {
      p->h_kap[ax].assign(1, 0.0);
      p->h_ell[ax].assign(1, 0.0);
    } else {
      symbol_tables_for(symbol_mode, n, p->h_kap[ax], p->h_ell[ax]);
    }
    PF_CK_CUDA(cudaMalloc(&p->kap[ax], sizeof(double) * n));
    PF_CK_CUDA(cudaMalloc(&p->ell[ax], sizeof(double) * n));
    PF_CK_CUDA(cudaMemcpy(p->kap[ax], p->h_kap[ax].data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    PF_CK_CUDA(cudaMemcpy(p->ell[ax], p->h_ell[ax].data(), sizeof(double) * n, cudaMemcpyHostToDevice));
  }
  PF_CK_CUDA(cudaMalloc(&p->partials, sizeof(double) * 32 * kMaxBlocks));
  PF_CK_CUDA(cudaMalloc(&p->ctrl, sizeof(Ctrl)));
  PF_CK_CUDA(cudaMallocHost(&p->h_ctrl, 2 * sizeof(Ctrl)));
  PF_CK_CUDA(cudaMallocHost(&p->h_small, 64 * sizeof(double)));
  p->scratch_bytes = sizeof(double) * 32 * kMaxBlocks;
  *out = p;
  return PF_OK;
}

int pf_plan_set_symbol_tables(pf_plan* p, int axis, const double* kappa_host, const double* lap1d_host) {
  PF_ARG(p && kappa_host && lap1d_host, "null argument");
  PF_ARG(axis >= 0 && axis < p->g.d, "axis %d out of range", axis);
  // table length = the GLOBAL extent fixed at plan creation (a slab plan's g.n[0]
  // is its local plane count, but its spectral passes index the whole axis-0 table)
  const int ax = 3 - p->g.d + axis, n = (int)p->h_kap[ax].size();
  p->h_kap[ax].assign(kappa_host, kappa_host + n);
  p->h_ell[ax].assign(lap1d_host, lap1d_host + n);
  PF_CK_CUDA(cudaSetDevice(p->device));
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  PF_CK_CUDA(cudaMemcpy(p->kap[ax], kappa_host, sizeof(double) * n, cudaMemcpyHostToDevice));
  PF_CK_CUDA(cudaMemcpy(p->ell[ax], lap1d_host, sizeof(double) * n, cudaMemcpyHostToDevice));
  return PF_OK;
}

int pf_plan_set_fused(pf_plan* p, int enable) {
  PF_ARG(p, "null plan");
  if (p->active) {
    set_error("pf_plan_set_fused while a solve is active");
    return PF_ERR_STATE;
  }
  p->fused_enable = enable ? 1 : 0;
  return PF_OK;
}

int pf_plan_set_cold_start(pf_plan* p, int cold) {
  PF_ARG(p, "null plan");
  p->cold_start = cold ? 1 : 0;
  return PF_OK;
}

int pf_plan_set_compact(pf_plan* p, int enable) {
  PF_ARG(p, "null plan");
  p->compact_enable = enable ? 1 : 0;
  return PF_OK;
}

int pf_plan_set_stream(pf_plan* p, void* stream) {
  PF_ARG(p, "null plan");
  p->user_stream = (cudaStream_t)stream;
  return PF_OK;
}

int pf_plan_device_bytes(const pf_plan* p, size_t* bytes) {
  PF_ARG(p && bytes, "null argument");
  *bytes = p->scratch_bytes + p->fft_work_bytes;
  return PF_OK;
}

int pf_plan_destroy(pf_plan* p) {
  if (!p) return PF_OK;
  cudaSetDevice(p->device);
  cudaStreamSynchronize(p->work);
  p->graph.reset();
  fused_free(p);
  tfused_free(p);
  slab_free(p);
  for (int k = 0; k < 4; ++k) {
    if (p->fwd[k]) cufftDestroy(p->fwd[k]);
    if (p->inv[k]) cufftDestroy(p->inv[k]);
  }
  for (int ax = 0; ax < 3; ++ax) {
    cudaFree(p->kap[ax]);
    cudaFree(p->ell[ax]);
  }
  cudaFree(p->fft_work);
  cudaFree(p->specA);
  cudaFree(p->specB);
  cudaFree(p->spec1);
  cudaFree(p->spec2);
  cudaFree(p->realA);
  cudaFree(p->realB);
  cudaFree(p->partials);
  cudaFree(p->gc_cnt);
  cudaFree(p->gc_base);
  cudaFree(p->gc_data);
  cudaFree(p->ctrl);
  cudaFreeHost(p->h_ctrl);
  cudaFreeHost(p->h_small);
  cudaEventDestroy(p->ev_user);
  cudaEventDestroy(p->ev_work);
  cudaEventDestroy(p->ev_poll[0]);
  cudaEventDestroy(p->ev_poll[1]);
  cudaStreamDestroy(p->work);
  delete p;
  return PF_OK;
}

}  // extern "C"
