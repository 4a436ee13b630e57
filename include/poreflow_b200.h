/*
 * poreflow_b200 — C ABI of the B200-native FFT micromechanics solver
 * (Stokes ADMM + comparison-medium transport of arXiv 2312.15554).
 *
 * The drop-in seam of the reference is the Python solver API of package
 * `poreflow` (reference: pkg/src/poreflow/__init__.py:11-102) plus its kernel
 * plugin contract `backends.kernels_for(dim)` (pkg/src/poreflow/backends/
 * __init__.py:43-47, pure.py:26-115).  The reference has no C ABI of its own;
 * these entry points are what its Python layer binds through ctypes
 * (INTEGRATION.md shows the stub).  Every entry point:
 *   - takes plain pointers and sizes (device pointers unless stated "host"),
 *   - returns an int status (PF_OK == 0); nothing throws across the ABI,
 *   - records a message retrievable with pf_last_error() (thread-local).
 * Field layout follows the reference (pure.py:8-10): scalars are C-order
 * grids (last axis fastest), vectors carry a leading component axis,
 * spectral arrays are complex128 interleaved (re, im).
 */
#ifndef POREFLOW_B200_H
#define POREFLOW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_OK 0
#define PF_ERR_ARG 1   /* invalid argument / validation failure  -> ValueError */
#define PF_ERR_CUDA 2  /* CUDA runtime failure                   -> RuntimeError */
#define PF_ERR_CUFFT 3 /* cuFFT failure                          -> RuntimeError */
#define PF_ERR_STATE 4 /* call out of sequence                   -> RuntimeError */

#define PF_SYMBOLS_EXACT 0   /* spectral.py:26 "exact"   */
#define PF_SYMBOLS_CENTRAL 1 /* spectral.py:27 "central" */

#define PF_STOKES_COLUMNS 15   /* stokes.py:38-43   */
#define PF_TRANSPORT_COLUMNS 4 /* transport.py:28   */

typedef struct pf_plan pf_plan;

/* Library version (major*10000 + minor*100 + patch) and last error text. */
int pf_version(void);
const char* pf_last_error(void);

/* ------------------------------------------------------------------------
 * Plan: one grid (UnitCellGrid, grid.py:25-71), its symbol tables
 * (make_symbols, spectral.py:72-98), cuFFT plans and solver scratch.
 * `dims` (host, ndim entries, 1 <= ndim <= 3, every entry >= 4 per
 * grid.py:36-39).  `stream` is a cudaStream_t the plan orders itself after
 * (may be NULL = legacy default stream).  Not thread-safe: one plan per
 * host thread / stream, mirroring the "independent solver instances"
 * contract (tests/test_backends.py:131-149).
 * ---------------------------------------------------------------------- */
int pf_plan_create(pf_plan** out, int ndim, const int64_t* dims, int symbol_mode, int device,
                   void* stream);
int pf_plan_destroy(pf_plan* plan);
int pf_plan_set_stream(pf_plan* plan, void* stream);
/* Enable (default) or disable the fused power-of-two Stokes pipeline
 * (cubic grids N = 64 ... 1024; transport up to 512); disabled or unsupported grids use the
 * general cuFFT pipeline.  Both compute the same iteration. */
int pf_plan_set_fused(pf_plan* plan, int enable);
/* Enable (default) or disable solid-only storage of u~, a, lam on the fused
 * Stokes path (used when a = 0 on pore voxels, e.g. cold starts): on pore
 * voxels the local step is exactly u~' = u', a' = 0, lam' = lam. */
int pf_plan_set_compact(pf_plan* plan, int enable);
/* Promise (cold != 0) that the state passed to the NEXT pf_stokes_begin is all
 * zero — the reference's default initial state (stokes.py:362) created by the
 * caller.  The fused pipeline then builds its spectral state, right-hand side and
 * solid-only storage without transforms (about 2 ms less setup at 256^3).  The
 * flag is consumed by that begin.  Passing it with a non-zero state is an error
 * the library does not detect. */
int pf_plan_set_cold_start(pf_plan* plan, int cold);
/* Replace the symbol tables of one logical axis (host arrays of dims[axis]
 * doubles: kappa_j and the 1D Laplacian term, spectral.py:78-86).  The
 * Python host layer passes numpy's own tables so the device sees the
 * reference's bits; pf_plan_create fills them with libm otherwise. */
int pf_plan_set_symbol_tables(pf_plan* plan, int axis, const double* kappa_host,
                              const double* lap1d_host);
/* Bytes of device scratch the plan currently holds (buffers + cuFFT work). */
int pf_plan_device_bytes(const pf_plan* plan, size_t* bytes);

/* ------------------------------------------------------------------------
 * Stokes ADMM — replaces poreflow.stokes.solve_stokes (stokes.py:313-427)
 * for non-degenerate cells (the all-solid fast path, stokes.py:336-353, and
 * the warm-start validation, 355-361, stay in the host wrapper).
 * ---------------------------------------------------------------------- */
typedef struct {
  double nu;                   /* StokesConfig.nu                    stokes.py:91  */
  double pressure_gradient[3]; /* StokesConfig.pressure_gradient     stokes.py:92  */
  double eps_abs, eps_rel;     /*                                    stokes.py:93-94 */
  int64_t max_iter;            /*                                    stokes.py:95  */
  double alpha, beta, b;       /* PenaltyParams                      stokes.py:57-59 */
  int32_t adaptive;            /*                                    stokes.py:60  */
  double growth[3];            /*                                    stokes.py:61  */
  double ratio_threshold[3];   /*                                    stokes.py:62  */
  double floor[3];             /*                                    stokes.py:63  */
} pf_stokes_params;

typedef struct {
  int64_t iterations;        /* ConvergenceReport.iterations                 */
  int32_t converged;         /* ConvergenceReport.converged                  */
  int32_t done;              /* loop finished (converged or max_iter)        */
  double final_penalties[3]; /* meta["final_penalties"]  stokes.py:425       */
} pf_stokes_result;

/* solid: uint8 0/1 grid.  u, u_tilde, a, lam: ndim x grid f64; q: grid f64.
 * In: initial state (zeros or warm start).  Out: final state (AdmmState).
 * history: max_iter x 15 f64 rows (REPORT_COLUMNS order); rows
 * [0, iterations) are written.  All device pointers, resident on the plan's
 * device, must stay valid until pf_stokes_end returns. */
int pf_stokes_solve(pf_plan* plan, const pf_stokes_params* params, const uint8_t* solid, double* u,
                    double* u_tilde, double* q, double* a, double* lam, double* history,
                    pf_stokes_result* result);

/* Split form of pf_stokes_solve for device-resident drivers and benchmarks:
 * begin = setup (spectral copies, stokes.py:363-370); iterate = run up to
 * n_iter more iterations of the loop body (stokes.py:375-417) as CUDA graphs
 * with a device-side done flag (poll = 0: enqueue all n_iter iterations and
 * return without host synchronisation); end = write q, fill result. */
int pf_stokes_begin(pf_plan* plan, const pf_stokes_params* params, const uint8_t* solid, double* u,
                    double* u_tilde, double* q, double* a, double* lam, double* history);
int pf_stokes_iterate(pf_plan* plan, int64_t n_iter, int poll, pf_stokes_result* result);
int pf_stokes_end(pf_plan* plan, pf_stokes_result* result);
/* Measurement hook (bench.py): run n_iter iterations without graphs, with CUDA
 * events between stages; stage_ms (host, 6 doubles) receives the mean time of
 * S1 spectral | Z2D | S3 local | finalize | S4 form-R | D2Z, in ms. */
int pf_stokes_profile(pf_plan* plan, int64_t n_iter, double* stage_ms);
/* Pipeline of the active / last Stokes solve: 0 = cuFFT (stages as above),
 * 1 = fused, 2 = fused with solid-only multiplier storage
 * (fused stages: PK | MI | RS | finalize | RSF | MF). */
int pf_stokes_pipeline(const pf_plan* plan);

/* ------------------------------------------------------------------------
 * Slab decomposition of one Stokes cell over P ranks (BASELINE cfg 5).
 * Rank `rank` owns real x-slab i0 in [rank*N0/P, (rank+1)*N0/P) ([c][N0/P][N1][N2])
 * and spectral y-slab k1 in [rank*N1/P, ...) in "T layout" [c][N0][N1/P][N2/2+1].
 * The host driver moves the exchange buffers between ranks (all_to_all with
 * equal splits) between pf_slab_forward / _forward_finish and pf_slab_inverse /
 * _inverse_finish, and all-reduces the 9 residual sums between pf_slab_local
 * and pf_slab_finalize.  All buffers are device memory owned by the caller;
 * complex buffers are passed as double* (interleaved).  Enqueue-only.
 * ---------------------------------------------------------------------- */
int pf_slab_plan_create(pf_plan** out, const int64_t* dims, int nranks, int rank, int symbol_mode, int device,
                        void* stream);
int pf_slab_sizes(pf_plan* plan, int64_t* exchange_per_comp, int64_t* tspec_per_comp, int64_t* real_per_comp);
int pf_slab_forward(pf_plan* plan, const double* real, int ncomp, double* send);
int pf_slab_forward_finish(pf_plan* plan, const double* recv, int ncomp, double* tspec);
int pf_slab_inverse(pf_plan* plan, double* tspec, int ncomp, double* send);
int pf_slab_inverse_finish(pf_plan* plan, const double* recv, int ncomp, double* real);
int pf_slab_stokes_begin(pf_plan* plan, const pf_stokes_params* params, const uint8_t* solid, double* u,
                         double* u_tilde, double* q, double* a, double* lam, double* history);
int pf_slab_setup(pf_plan* plan, const double* q_tspec, const double* u_tspec, double* Q, double* D);
int pf_slab_spectral(pf_plan* plan, const double* R, double* Q, double* D, double* U);
int pf_slab_local(pf_plan* plan, const double* u_new, double* totals9);
int pf_slab_finalize(pf_plan* plan, const double* totals9);
int pf_slab_form_r(pf_plan* plan, double* R, int gated);
int pf_slab_scale(pf_plan* plan, const double* src, double* dst, int64_t count, double scale);
int pf_slab_read(pf_plan* plan, pf_stokes_result* result);
/* Permeability of a slab-decomposed cell (replaces poreflow.effective.permeability,
 * src/effective.py:43-72, for fields no rank holds whole): the spectral gradient
 * i kappa_axis F / n of one T-layout spectrum (pf_slab_forward /
 * pf_slab_forward_finish of a velocity component), and this rank's six masked
 * Gram sums sum_pore sum_m G[i][m] G[j][m] (i <= j) of one velocity component
 * over its x-slab, G = 9 contiguous real slab fields [flow i][axis m]; the caller
 * all-reduces the sums and scales by h^3. */
int pf_slab_grad(pf_plan* plan, const double* t_spec, int axis, double* t_out);
int pf_slab_gram(pf_plan* plan, const uint8_t* solid, const double* G, double* sums6);

/* Fused slab pipeline (cubic N in {64, 128, 256, 512, 1024}, P a power of two, slabs of
 * whole tiles; pf_slab_fused_sizes reports 0 when unsupported).  Per iteration:
 * pf_slab_fused_pk (axis 0 + Green's operator on the y-slab Y) -> exchange
 * Y y-slab -> x-slab -> pf_slab_fused_rs (axis-1 inverse, rows + local step,
 * the rank's 9 residual sums) -> all-reduce -> pf_slab_finalize ->
 * pf_slab_fused_mf (axis-1 forward) -> exchange Y x-slab -> y-slab.  Y buffers
 * (caller-owned, complex as double*): main arrays of y_main elements with one
 * all_to_all of equal splits per component (y-slab [c][N][N/P][N/2] <-> x-slab
 * [c][P][N/P][N/P][N/2]), Nyquist arrays of y_nyq elements exchanged in one
 * (y-slab [N][3][N/P] <-> x-slab [P][N/P][3][N/P]).  Setup takes the T-layout
 * Q^ / D^ of pf_slab_setup and a real scratch of 3*L0*N*N for R; end returns Q^
 * in T layout (unscaled) and materialises u~, a, lam.  Replaces the per-iteration
 * pf_slab_spectral / transforms / pf_slab_local / pf_slab_form_r sequence. */
int pf_slab_fused_sizes(pf_plan* plan, int64_t* y_main, int64_t* y_nyq);
int pf_slab_fused_bind(pf_plan* plan, double* Yy, double* Yy_nyq, double* Yx, double* Yx_nyq);
int pf_slab_fused_setup(pf_plan* plan, const double* Q_tspec, const double* D_tspec, double* R_scratch);
/* Cold-start setup (the caller's u, u~, q, a, lam are all zero): Q^ = D^ = 0 and
 * Y = 0 with no transform, exchange or scratch — in place of pf_slab_setup +
 * pf_slab_fused_setup and the first Y exchange. */
int pf_slab_fused_setup_zero(pf_plan* plan);
/* Release the slab transforms' cuFFT plans, work area and scratch (re-created
 * on the next pf_slab_forward / pf_slab_inverse): the fused slab needs them only
 * at setup and teardown. */
int pf_slab_release_transforms(pf_plan* plan);
int pf_slab_fused_pk(pf_plan* plan);
int pf_slab_fused_rs(pf_plan* plan, double* totals9);
int pf_slab_fused_mf(pf_plan* plan);
int pf_slab_fused_end(pf_plan* plan, double* Q_tspec);
/* Component-pipelined form of pf_slab_fused_rs / pf_slab_fused_mf, so the host
 * can overlap the exchange of component c + 1 with the passes of component c:
 * pf_slab_fused_rs_part(c) for c = 0, 1, 2 (each after its component and the
 * Nyquist columns arrived) then pf_slab_fused_totals; after pf_slab_finalize,
 * pf_slab_fused_mf_part(c, fix = (c == 0)) for c = 0, 1, 2, each component's
 * exchange issued as soon as its MF is enqueued.  Same results as the
 * unsplit calls (the residual sums are reduced in a fixed order). */
int pf_slab_fused_rs_part(pf_plan* plan, int comp);
int pf_slab_fused_totals(pf_plan* plan, double* totals9);
int pf_slab_fused_mf_part(pf_plan* plan, int comp, int fix);
/* Peer-memory exchange (the transpose fused into the passes' stores): device
 * addresses, valid in this process (P2P-mapped, e.g. torch symmetric memory), of
 * every rank's Y buffers — y-slab main / Nyquist, x-slab main / Nyquist, one per
 * rank, npeers = P.  PK then stores its output straight into the x-slab owners'
 * Yx and MF into the y-slab owners' Yy; the caller replaces each all_to_all by a
 * cross-rank barrier (all ranks' stores visible) before the consuming pass.
 * npeers = 0 restores the all_to_all exchange. */
int pf_slab_fused_set_peers(pf_plan* plan, const uint64_t* yy, const uint64_t* yy_nyq, const uint64_t* yx,
                            const uint64_t* yx_nyq, int npeers);

/* ------------------------------------------------------------------------
 * Transport — replaces poreflow.transport.solve_transport
 * (transport.py:180-268) including build_coefficients (101-128).
 * ---------------------------------------------------------------------- */
typedef struct {
  double pe, eta, a0, b0, eps;     /* TransportConfig   transport.py:44-49 */
  double composition_gradient[3];  /*                   transport.py:45    */
  int64_t max_iter;                /*                   transport.py:50    */
} pf_transport_params;

typedef struct {
  int64_t iterations;
  int32_t converged;
  int32_t diverged;
  int32_t reason; /* 0 none, 1 non-finite residual, 2 growth guard (transport.py:243-255) */
  int32_t done;
  double b0_vec[3]; /* MediumCoefficients.b0_vec   transport.py:123-127 */
  double u_bar[3];  /* MediumCoefficients.u_bar    transport.py:116     */
} pf_transport_result;

/* u: ndim x grid velocity (read only).  chi: grid, grad_chi: ndim x grid —
 * in: initial state, out: final state.  history: max_iter x 4 rows. */
int pf_transport_solve(pf_plan* plan, const pf_transport_params* params, const uint8_t* solid,
                       const double* u, double* chi, double* grad_chi, double* history,
                       pf_transport_result* result);
int pf_transport_begin(pf_plan* plan, const pf_transport_params* params, const uint8_t* solid,
                       const double* u, double* chi, double* grad_chi, double* history,
                       pf_transport_result* result);
int pf_transport_iterate(pf_plan* plan, int64_t n_iter, int poll, pf_transport_result* result);
int pf_transport_end(pf_plan* plan, pf_transport_result* result);
/* Pipeline of the active / last transport solve: 0 = cuFFT, 1 = fused. */
int pf_transport_pipeline(const pf_plan* plan);
/* Measurement hook: n_iter fused-transport iterations with stage events;
 * stage_ms (5 doubles): PK_T | MI_T | RS_T | finalize | MF_T. */
int pf_transport_profile(pf_plan* plan, int64_t n_iter, double* stage_ms);

/* ------------------------------------------------------------------------
 * Effective properties — effective.py:32-108, grid.py:108-110.
 * Results are written to HOST memory.
 * ---------------------------------------------------------------------- */
/* Pore mean of ncomp stacked fields f (ncomp x grid).  effective.py:32-40 */
int pf_pore_average(pf_plan* plan, const uint8_t* solid, const double* f, int ncomp,
                    double* out_host);
/* Solid-voxel count (porosity = 1 - count/n, grid.py:108-110). */
int pf_solid_count(pf_plan* plan, const uint8_t* solid, int64_t* count_host);
/* u_solutions: host array of ndim device pointers (each ndim x grid).
 * K: host ndim x ndim.  effective.py:43-72 */
int pf_permeability(pf_plan* plan, const uint8_t* solid, const double* const* u_solutions,
                    double* K_host);
/* chi / grad_chi: host arrays of ndim device pointers.  effective.py:75-108 */
int pf_diffusivity(pf_plan* plan, const uint8_t* solid, const double* const* u_solutions,
                   const double* const* chi, const double* const* grad_chi, double pe,
                   double* D_host);

/* ------------------------------------------------------------------------
 * Kernel plugin — the five functions of backends/pure.py:26-115 on device
 * pointers, full-spectrum layout (what backends.kernels_for() returns).
 * dims: host, ndim entries.  kappas: host array of ndim device pointers to
 * the per-axis symbol tables.  Complex arrays are interleaved complex128.
 * `solid` is the f64 0/1 field (as in pure.py).  stream may be NULL.
 * ---------------------------------------------------------------------- */
int pf_k_stokes_velocity_update(int ndim, const int64_t* dims, const double* q_hat,
                                const double* a_hat, const double* ut_hat,
                                const double* const* kappas, const double* lap,
                                const double* kappa_sq, double nu, double beta, double b,
                                const double* g_p_host, double* u_hat, void* stream);
int pf_k_aux_velocity_update(int ndim, const int64_t* dims, const double* u, const double* a,
                             const double* lam, const double* solid, double alpha, double b,
                             double* u_tilde, void* stream);
int pf_k_multiplier_update(int ndim, const int64_t* dims, const double* a, const double* lam,
                           const double* u, const double* u_tilde, const double* solid,
                           double alpha, double b, double* a_new, double* lam_new, void* stream);
int pf_k_transport_polarization(int ndim, const int64_t* dims, const double* grad_chi,
                                const double* diffusivity, const double* advection,
                                const double* forcing, double a0, const double* b0_vec_host,
                                const double* g_chi_host, double* w, double* s, void* stream);
int pf_k_transport_mode_update(int ndim, const int64_t* dims, const double* w_hat,
                               const double* s_hat, const double* const* kappas,
                               const double* lap, double a0, const double* b0_vec_host,
                               double* chi_hat, double* grad_hat, void* stream);

/* ------------------------------------------------------------------------
 * Spectral utilities and step helpers (reference spectral.py:101-143,
 * stokes.py:158-244, transport.py:131-177) on device pointers, full-spectrum
 * complex128 layout over the trailing ndim axes.  Not used by the solver loops.
 * ---------------------------------------------------------------------- */
/* fftn / ifftn (spectral.py:101-115): `batch` fields of prod(dims) points each;
 * in_complex = 0 reads real f64 input.  inverse != 0 scales by 1/prod(dims).
 * out may equal in when in_complex. */
int pf_k_fftn(int ndim, const int64_t* dims, int64_t batch, const double* in, int in_complex,
              double* out, int inverse, void* stream);
/* Re ifftn (spectral.py:107-115); work: batch*prod(dims) complex128 scratch (may be in). */
int pf_k_ifftn_real(int ndim, const int64_t* dims, int64_t batch, const double* in, double* work,
                    double* out, void* stream);
/* grad (spectral.py:118-124): out[c, b] = 1j*kappa_c * chi_hat[b], c < ndim. */
int pf_k_spectral_grad(int ndim, const int64_t* dims, int64_t batch, const double* const* kappas,
                       const double* chi_hat, double* out, void* stream);
/* div (spectral.py:127-133), or with base != NULL base + sum_c 1j*kappa_c*v[c]
 * in transport.py:149-151's accumulation order. */
int pf_k_spectral_div(int ndim, const int64_t* dims, const double* const* kappas, const double* v_hat,
                      const double* base, double* out, void* stream);
/* out[b, m] = (sign * factor[m]) * z[b, m]: apply_laplacian with sign = -1 (spectral.py:136-138). */
int pf_k_scale_modes(int64_t n_modes, int64_t batch, const double* factor, double sign, const double* z,
                     double* out, void* stream);
/* q' = q - beta*div, then q' -= mean(q') (stokes.py:216-218).  scratch:
 * pf_k_scratch_doubles() f64. */
int pf_k_q_update(int64_t count, const double* q, const double* div, double beta, double* out,
                  double* scratch, void* stream);
/* ||w*(x - y)||_2 (stokes.py:154-155); y, w may be NULL; w is indexed i % w_period
 * (a scalar indicator weighting a vector field).  Synchronous: the result lands
 * in *result_host. */
int pf_k_norm(int64_t count, const double* x, const double* y, const double* w, int64_t w_period,
              double* scratch, double* result_host, void* stream);
int pf_k_scratch_doubles(void);

/* Bit-packed indicator (1 bit per voxel, numpy.packbits order — the
 * first voxel in the most significant bit of byte 0) -> uint8 0/1 per voxel, on
 * the device: ceil(n / 8) bytes cross PCIe instead of n. */
int pf_unpack_bits(const uint8_t* bits, uint8_t* out, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* POREFLOW_B200_H */
