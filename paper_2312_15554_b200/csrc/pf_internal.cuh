// Internal declarations shared by the poreflow_b200 translation units.
#pragma once
#include <nvtx3/nvToolsExt.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <utility>

#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/poreflow_b200.h"

namespace pf {

// NVTX range over a C-ABI entry point (stage ranges for nsys / ncu
// --nvtx filtering); header-only NVTX3, a no-op without an attached tool.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define PF_NVTX(name) ::pf::NvtxRange pf_nvtx_range_(name)


// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
const char* cufft_name(cufftResult r);

#define PF_CK_CUDA(expr)                                                                 \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      ::pf::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return PF_ERR_CUDA;                                                                \
    }                                                                                    \
  } while (0)

#define PF_CK_FFT(expr)                                                                  \
  do {                                                                                   \
    cufftResult _r = (expr);                                                             \
    if (_r != CUFFT_SUCCESS) {                                                           \
      ::pf::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr, ::pf::cufft_name(_r)); \
      return PF_ERR_CUFFT;                                                               \
    }                                                                                    \
  } while (0)

#define PF_CK(expr)                 \
  do {                              \
    int _s = (expr);                \
    if (_s != PF_OK) return _s;     \
  } while (0)

#define PF_ARG(cond, ...)                 \
  do {                                    \
    if (!(cond)) {                        \
      ::pf::set_error(__VA_ARGS__);       \
      return PF_ERR_ARG;                  \
    }                                     \
  } while (0)

// ---------------------------------------------------------------- launch geometry
constexpr int kThreads = 256;
constexpr int kSMs = 148;
constexpr int kMaxBlocks = kSMs * 8;  // 8 x 256-thread CTAs fill an SM (2048 threads)
// Finalize / partial-reduction shape, measured (r02e; Gvox-it/s at 64^3 / 128^3 / 256^3):
// 1024 threads x 4 running sums 7.43 / 13.06 / 16.37, x 2 7.59 / 13.15 / 16.38,
// x 1 7.65 / 13.14 / 16.41; 512 x 1 7.70 / 13.17 / 16.40; 256 x 1 7.59 / 13.09 / 16.34
// (the partial counts are a few thousand: the serial combine of the unrolled sums
// cost more than the loads it kept in flight)
#ifndef PF_FINALIZE_THREADS
#define PF_FINALIZE_THREADS 512
#endif
#ifndef PF_REDUCE_UNROLL
#define PF_REDUCE_UNROLL 1  // independent running sums (loads in flight) per thread in reduce_partials
#endif
constexpr int kFinalizeThreads = PF_FINALIZE_THREADS;

inline int blocks_for(int64_t work) {
  int64_t b = (work + kThreads - 1) / kThreads;
  if (b < 1) b = 1;
  return (int)(b > kMaxBlocks ? kMaxBlocks : b);
}

// ---------------------------------------------------------------- grid geometry
// Logical grid of d axes embedded in padded 3D (n0, n1, n2) with leading 1s;
// logical axis j <-> padded axis 3-d+j.  Half spectrum is (n0, n1, n2h).
struct Geom {
  int d;
  int n[3];     // padded dims
  int n2h;      // n[2]/2 + 1
  int64_t nr;   // real points
  int64_t nh;   // half-spectrum modes
  double inv_n; // 1/nr
  double dn;    // (double) nr
  int k1off;    // global offset of local axis-1 modes (slab decomposition; 0 otherwise)
};

// Device-side solver control block (one per plan; lives in device memory).
struct Ctrl {
  double alpha, beta, b;  // current penalties (Stokes)
  double best;            // running minimum of r1+r2 (transport)
  double db;              // b' - b of the last adaptation (fused pipeline's right-hand-side correction)
  int64_t iter;           // completed iterations
  int32_t done, converged, diverged, reason;
};

// Stokes constants that do not change during a solve.
struct StokesConst {
  double nu, eps_rel;
  double tol_vec, tol_sca;  // sqrt(n_vec)*eps_abs, sqrt(n_sca)*eps_abs (host-computed)
  double g[3];              // pressure gradient (logical components)
  double growth[3], thr[3], floor_[3];
  double lam_pore_sq;       // |lam|^2 over pore voxels (constant there; compact RS path), else 0
  int64_t max_iter;
  int adaptive;
};

struct TransportConst {
  double pe, eta, a0, eps_tol1, eps_tol2;  // tolerances sqrt(n)*eps, sqrt(dn)*eps
  double g[3], b0v[3];
  double ubar_dot_g;  // float(u_bar @ g_chi)   transport.py:121
  int64_t max_iter;
};

struct Graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int iters = 0;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    iters = 0;
  }
};

}  // namespace pf

struct pf_plan {
  pf::Geom g;
  int mode;
  int device;
  cudaStream_t user_stream;  // caller's stream (torch current stream)
  cudaStream_t work;         // plan-owned stream (graph capture needs a non-legacy stream)
  cudaEvent_t ev_user, ev_work, ev_poll[2];
  // per padded axis symbol tables (device), length n[p]
  double* kap[3];
  double* ell[3];
  std::vector<double> h_kap[3], h_ell[3];
  // cuFFT: forward D2Z / inverse Z2D for batch 1, d, d+1, d*d
  cufftHandle fwd[4], inv[4];
  int batch_of[4];
  void* fft_work;
  size_t fft_work_bytes;
  // scratch
  double2* specA;  // (d+1) * nh
  double2* specB;  // (d+1) * nh
  double2* spec1;  // nh
  double2* spec2;  // nh
  double* realA;   // (d+1) * nr
  double* realB;   // (d+1) * nr
  double* partials;  // 16 * kMaxBlocks
  pf::Ctrl* ctrl;     // device
  pf::Ctrl* h_ctrl;   // pinned host, 2 slots for double-buffered polling
  double* h_small;    // pinned host scratch (64 doubles)
  size_t scratch_bytes;
  // fused power-of-two pipeline (pf_fused.cu)
  void* fused;       // FusedPlan*
  int fused_enable;  // 1 = use the fused pipeline when the grid supports it
  int compact_enable;  // 1 = solid-only multiplier storage on the fused path when eligible
  int cold_start;      // 1 = the next pf_stokes_begin's state is all zero (pf_plan_set_cold_start)
  int pipeline;      // pipeline of the active Stokes solve: 0 cuFFT, 1 fused
  // solid-only multiplier storage of the cuFFT pipeline (pf_stokes.cu): per-64-voxel
  // segment counts / bases, [3][d][ns] data (u~, a, lam), on for the active solve
  uint32_t *gc_cnt, *gc_base;
  double* gc_data;
  int64_t gc_ns, gc_cap, gc_nseg;
  int gc_on;
  void* tfused;      // FusedTPlan* (pf_fused_transport.cu)
  int t_pipeline;    // pipeline of the active transport solve: 0 cuFFT, 1 fused
  void* slab;        // SlabPlan* (pf_slab.cu) for slab-decomposed plans
  int slab_nb1;      // block count of the last slab spectral step (its partials)
  // active solve state
  int active;  // 0 none, 1 stokes, 2 transport
  pf::Graph graph;
  // stokes bindings
  const uint8_t* s_solid;
  double *s_u, *s_ut, *s_q, *s_a, *s_lam, *s_hist;
  pf::StokesConst sc;
  // transport bindings
  const double* t_u;
  double *t_chi, *t_grad, *t_hist;
  pf::TransportConst tc;
  pf_transport_result t_res;
};

namespace pf {

int plan_ensure_scratch(pf_plan* p);
int plan_fft(pf_plan* p, bool forward, int batch, void* in, void* out);
int enter(pf_plan* p);  // order plan->work after user stream
int leave(pf_plan* p);  // order user stream after plan->work
int run_chunks(pf_plan* p, int64_t n_iter, int poll, int (*enqueue)(pf_plan*), Ctrl* out_ctrl);
int symbol_tables_for(int mode, int n, std::vector<double>& kap, std::vector<double>& ell);

// fused pipeline (pf_fused.cu)
bool fused_supported(const pf_plan* p);
int fused_ensure(pf_plan* p);
void fused_free(pf_plan* p);
int fused_setup(pf_plan* p);
int fused_finish(pf_plan* p);
int enqueue_fused(pf_plan* p, cudaEvent_t* ev);
// TMA tensor maps of the fused passes (pf_fused.cu): [ncomp N N rows][N/2 complex]
// with box (cm complex, N rows), 128B swizzle; and [ncomp N (c,i0)][N k1][N/2] with
// box (cp complex, 1, N), 64B swizzle
int encode_axis1_map(CUtensorMap* tm, const double2* base, int N, int cm, int ncomp);
int encode_pk_map(CUtensorMap* tm, const double2* base, int N, int cp, int ncomp);
// slab-decomposed fused pipeline (pf_fused.cu, driven by pf_slab_fused_*)
int fused_slab_supported(int N, int l0, int l1);
int fused_slab_bind(pf_plan* p, int N, int l0, int l1, int k1off, double2* Yy, double2* Yyn, double2* Yx,
                    double2* Yxn);
int fused_slab_setup(pf_plan* p, const double2* Tq, const double2* Td, double* R);
int fused_slab_pk(pf_plan* p);
int fused_slab_rs(pf_plan* p, double* totals);
int fused_slab_mf(pf_plan* p);
int fused_slab_rs_part(pf_plan* p, int comp);
int fused_slab_setup_zero(pf_plan* p, int64_t y_main, int64_t y_nyq);
int slab_gram_host(pf_plan* p, const uint8_t* solid, const double* G, int64_t n, double* out6);
int fused_slab_totals(pf_plan* p, double* totals);
int fused_slab_mf_part(pf_plan* p, int comp, int fix);
int fused_slab_set_peers(pf_plan* p, const uint64_t* yy, const uint64_t* yyn, const uint64_t* yx,
                         const uint64_t* yxn, int npeers);
int fused_slab_end(pf_plan* p, double2* Tq);
int fused_is_compact(const pf_plan* p);
int scan_counts(cudaStream_t s, const uint32_t* cnt, uint32_t* off, int64_t n);
// fused transport pipeline (pf_fused_transport.cu)
int tfused_setup(pf_plan* p, bool warm);
int tfused_finish(pf_plan* p);
int tfused_enqueue(pf_plan* p, cudaEvent_t* ev = nullptr);
void tfused_free(pf_plan* p);
int plan_reset_work_areas(pf_plan* p);
int reduce_rows_to(pf_plan* p, const double* part, int nrows, int nb, double* out);
// transport helpers shared with the fused pipeline (pf_transport.cu)
int transport_polarize(pf_plan* p, const double* grad, double* out);
void transport_finalize_launch(pf_plan* p, const double* part, int nb, double scale);
void slab_free(pf_plan* p);
// Stokes kernels shared with the slab pipeline (pf_stokes.cu)
int stokes_spectral_launch(pf_plan* p, const Geom& gs, double2* Qh, const double2* Rh, double2* Dh, double2* Uh,
                           double* part1, int* nb1);
int stokes_local_launch(pf_plan* p, int64_t n, const double* un, double* part3, int* nb3);
int stokes_div_launch(pf_plan* p, const Geom& gs, const double2* Uh, double2* Dh);
int stokes_ctrl_init(pf_plan* p, double alpha, double beta, double b);
int stokes_form_r_gated(pf_plan* p, double* R, int gated);
// Stokes helpers shared with the fused pipeline (pf_stokes.cu)
int stokes_div_spectrum(pf_plan* p, const double* u, double2* tmp, double2* out);
int stokes_form_r(pf_plan* p, double* R);
cudaError_t k_stokes_finalize_launch_pdl(pf_plan* p, const double* part3, int nb3, const double* part1, int nb1);
void k_stokes_finalize_launch(pf_plan* p, const double* part3, int nb3, const double* part1, int nb1);

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
// i*k*a for real k
__device__ __forceinline__ double2 cik(double k, double2 a) { return make_double2(-(k * a.y), k * a.x); }
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }

// numpy complex division (loops.c.src Smith variant) — bitwise what the
// reference computes for f_hat / denom (pure.py:109).
__device__ __forceinline__ double2 cdiv_np(double2 a, double2 b) {
  double ar = fabs(b.x), ai = fabs(b.y);
  if (ar >= ai) {
    if (ar == 0.0 && ai == 0.0) return make_double2(a.x / ar, a.y / ai);
    double rat = b.y / b.x;
    double scl = 1.0 / (b.x + b.y * rat);
    return make_double2((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
  } else {
    double rat = b.x / b.y;
    double scl = 1.0 / (b.y + b.x * rat);
    return make_double2((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
  }
}

// Block-wide sum of NQ per-thread values; thread 0 returns the totals in v.
template <int NQ, int MAXW = 32>
__device__ __forceinline__ void block_sum(double (&v)[NQ]) {
  __shared__ double sh[NQ][MAXW];  // MAXW >= warps per block
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double x = v[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) sh[q][wid] = x;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double x = lane < nw ? sh[q][lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      v[q] = x;
    }
  }
  __syncthreads();
}

// Deterministic block partials -> totals: partials laid out [q][nblk].  Each
// thread keeps four independent running sums per quantity (loads in flight),
// combined in a fixed order, then a fixed-shape block tree.
template <int NQ>
__device__ __forceinline__ void thread_partials(const double* __restrict__ part, int nblk, double* tot) {
  constexpr int U = PF_REDUCE_UNROLL;
  double s4[NQ][U];
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int u = 0; u < U; ++u) s4[q][u] = 0.0;
  const int stride = blockDim.x;
  int i = threadIdx.x;
  for (; i + (U - 1) * stride < nblk; i += U * stride) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int u = 0; u < U; ++u) s4[q][u] += part[(int64_t)q * nblk + i + u * stride];
  }
  for (; i < nblk; i += stride)
#pragma unroll
    for (int q = 0; q < NQ; ++q) s4[q][0] += part[(int64_t)q * nblk + i];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double x = 0.0;  // fixed pairwise order
#pragma unroll
    for (int w = 1; w < U; w <<= 1)
#pragma unroll
      for (int u = 0; u < U; u += 2 * w) s4[q][u] += s4[q][u + w];
    x = s4[q][0];
    tot[q] = x;
  }
}

template <int NQ>
__device__ __forceinline__ void reduce_partials(const double* __restrict__ part, int nblk, double (&tot)[NQ]) {
  thread_partials<NQ>(part, nblk, tot);
  block_sum<NQ>(tot);
}

// Two partial arrays in one pass: both arrays' loads in flight together and one block
// tree (per quantity the same order and tree shape as two reduce_partials calls).
template <int NA, int NB>
__device__ __forceinline__ void reduce_partials2(const double* __restrict__ pa, int na, double (&ta)[NA],
                                                 const double* __restrict__ pb, int nb, double (&tb)[NB]) {
  double tot[NA + NB];
  thread_partials<NA>(pa, na, tot);
  thread_partials<NB>(pb, nb, tot + NA);
  block_sum<NA + NB>(tot);
#pragma unroll
  for (int q = 0; q < NA; ++q) ta[q] = tot[q];
#pragma unroll
  for (int q = 0; q < NB; ++q) tb[q] = tot[NA + q];
}

__device__ __forceinline__ double pymax(double a, double b) { return b > a ? b : a; }

// Programmatic dependent launch: a kernel launched with launch_k (PF_PDL) may
// start while its predecessor drains; it must call pdl_wait() before reading
// anything the predecessor writes (a no-op for ordinary launches).
#ifndef PF_PDL
#define PF_PDL 1  // measured: +4 % at 64^3, neutral at 128^3 and 256^3
#endif
#ifndef PF_PDL_EARLY
#define PF_PDL_EARLY 0  // trigger the dependent launch right after the wait (instead of at CTA exit)
#endif
__device__ __forceinline__ void pdl_wait() {
#if PF_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if PF_PDL_EARLY
  // every dependent pass waits on griddepcontrol.wait before touching our outputs,
  // so letting it launch (and become resident where it fits) early is safe
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
#endif
}

// Dynamic shared memory limit of a kernel plus its carveout preference.  Left to
// itself the driver picked a 200 KB carveout for the fused kernels (ncu "Shared
// Memory Configuration Size"), which capped e.g. the transport RS at 4 CTAs/SM of
// 45 KB; PF_CARVEOUT (percent of the maximum, -1 = driver default) asks for more.
#ifndef PF_CARVEOUT
#define PF_CARVEOUT -1  // measured: 100 (max shared) costs PK 0.29 -> 0.33 ms (less L1), RS_T no gain
#endif
template <typename... KArgs>
inline cudaError_t smem_attr(void (*kern)(KArgs...), size_t bytes) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess || PF_CARVEOUT < 0) return e;
  return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, PF_CARVEOUT);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
#if PF_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
#else
  kern<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
  return cudaGetLastError();
#endif
}

}  // namespace pf
