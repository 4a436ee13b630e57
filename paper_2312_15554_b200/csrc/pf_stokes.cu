// Stokes augmented-Lagrangian (ADMM) loop on device — reference
// pkg/src/poreflow/stokes.py:313-427.
//
// Per iteration (half-spectrum canonical pipeline):
//   S1 k_stokes_spectral  : Green's operator (pure.py:26-56) on R^ = FFT(b u~ - a)
//                           and Q^; writes U^/n, D^ = i k.U^ (div, stokes.py:381),
//                           Q^' = Q^ - beta D^ with Q^'(0) = 0 (stokes.py:408-409),
//                           and the Parseval sums of |D^|^2, |D^ - D^_prev|^2, |Q^'|^2.
//   S2 cuFFT Z2D (batch d): U^/n -> u'
//   S3 k_stokes_local     : u~' (pure.py:59-61), a', lam' (pure.py:64-68) and six
//                           real-space squared norms (stokes.py:254-277).
//   F  k_stokes_finalize  : residual pairs + tolerances (stokes.py:247-284), the
//                           history row (398-403), convergence (413-415), and
//                           residual balancing (adapt_penalties, 287-310).
//   S4 k_form_r           : R = b' u~' - a' (next iteration's right-hand side,
//                           stokes.py:405-407 by linearity of the transform).
//   S5 cuFFT D2Z (batch d): R -> R^
// Every kernel returns immediately once ctrl->done is set.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "pf_internal.cuh"

#ifndef PF_ABL_FINTRIV
#define PF_ABL_FINTRIV 0
#endif
#ifndef PF_ABL_NORED
#define PF_ABL_NORED 0
#endif
#ifndef PF_ABL_NOADAPT
#define PF_ABL_NOADAPT 0
#endif
#ifndef PF_ABL_NODB
#define PF_ABL_NODB 0
#endif

namespace pf {

struct Tables {
  const double* kap[3];
  const double* ell[3];
};

static Tables tables_of(const pf_plan* p) {
  Tables t;
  for (int i = 0; i < 3; ++i) {
    t.kap[i] = p->kap[i];
    t.ell[i] = p->ell[i];
  }
  return t;
}

__device__ __forceinline__ void mode_index(const Geom& g, uint32_t m, int (&idx)[3]) {
  const uint32_t n2h = (uint32_t)g.n2h, n1 = (uint32_t)g.n[1];
  const uint32_t t = m / n2h;
  idx[2] = (int)(m - t * n2h);
  idx[1] = (int)(t % n1);
  idx[0] = (int)(t / n1);
}

// Parseval weight on the half spectrum: 1 on the k2 = 0 and k2 = Nyquist planes.
__device__ __forceinline__ double parseval_w(const Geom& g, int i2) {
  return (i2 == 0 || ((g.n[2] & 1) == 0 && i2 == g.n[2] / 2)) ? 1.0 : 2.0;
}

// ---------------------------------------------------------------------- S1
template <int D>
__global__ void __launch_bounds__(kThreads) k_stokes_spectral(
    Geom g, Tables T, const double nu, const double gx, const double gy, const double gz,
    double2* __restrict__ Qh, const double2* __restrict__ Rh, double2* __restrict__ Dh,
    double2* __restrict__ Uh, const Ctrl* __restrict__ ctrl, double* __restrict__ part) {
  if (ctrl->done) return;
  const double beta = ctrl->beta, b = ctrl->b;
  const double gp[3] = {gx, gy, gz};
  double acc[3] = {0.0, 0.0, 0.0};
  const uint32_t nh = (uint32_t)g.nh;
  const bool owns_zero = g.k1off == 0;
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < nh; m += gridDim.x * blockDim.x) {
    int idx[3];
    mode_index(g, m, idx);
    const int i2 = idx[2];
    idx[1] += g.k1off;  // global axis-1 mode (slab decomposition)
    const bool zero = owns_zero && m == 0;
    double kc[D];
    double L = 0.0, ksq = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const int ax = 3 - D + c;
      kc[c] = __ldg(T.kap[ax] + idx[ax]);
      L = L + __ldg(T.ell[ax] + idx[ax]);
      ksq = ksq + kc[c] * kc[c];
    }
    // every load of the mode first (the D^ load used to sit behind the U^ stores)
    const double2 q = Qh[m];
    const double2 dprev = Dh[m];
    double2 rin[D];
#pragma unroll
    for (int c = 0; c < D; ++c) rin[c] = Rh[(size_t)c * nh + m];
    double2 r[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double2 rc = rin[c];
      r[c] = make_double2(kc[c] * q.y + rc.x, -(kc[c] * q.x) + rc.y);  // -i k q + R^
      if (zero) r[c].x = r[c].x + g.dn * gp[c];                           // n g_p at k = 0
    }
    const double A = nu * L + b;
    double2 kr = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < D; ++c) kr = cadd(kr, cscale(kc[c], r[c]));
    const double f = beta / (A + beta * ksq);
    const double2 corr = cscale(f, kr);
    const double invA = 1.0 / A;
    double2 dv = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double2 u = csub(r[c], cscale(kc[c], corr));
      u = make_double2(u.x * invA, u.y * invA);
      dv = cadd(dv, cik(kc[c], u));
      Uh[(size_t)c * nh + m] = make_double2(u.x * g.inv_n, u.y * g.inv_n);
    }
    double2 qn = csub(q, cscale(beta, dv));
    if (zero) qn = make_double2(0.0, 0.0);
    const double w = parseval_w(g, i2);
    acc[0] += w * cabs2(dv);
    acc[1] += w * cabs2(csub(dv, dprev));
    acc[2] += w * cabs2(qn);
    Qh[m] = qn;
    Dh[m] = dv;
  }
  block_sum<3>(acc);
  if (threadIdx.x == 0)
    for (int k = 0; k < 3; ++k) part[(size_t)k * gridDim.x + blockIdx.x] = acc[k];
}

// ---------------------------------------------------------------------- S3
// pure.py:59-68 per voxel in the reference's evaluation order (bit-exact with
// --fmad=false) and the six squared norms of stokes.py:254-277.  Work items are
// (component, voxel pair): 16-byte loads, and two items per loop trip with all ten
// loads issued before any arithmetic, so a warp keeps 20 loads in flight — the
// one-voxel-per-trip form sat at 20 % of DRAM bandwidth, latency-bound with its
// loads issued behind the previous component's stores.
struct LocalIn {
  double2 u1, u0, t0, a0, l0;
  double h0, h1;
};

__device__ __forceinline__ void local_load(LocalIn& v, int64_t i, int64_t x, const double* __restrict__ un,
                                           const double* __restrict__ u, const double* __restrict__ ut,
                                           const double* __restrict__ a, const double* __restrict__ lam,
                                           const uint8_t* __restrict__ H) {
  v.u1 = *reinterpret_cast<const double2*>(un + i);
  v.u0 = *reinterpret_cast<const double2*>(u + i);
  v.t0 = *reinterpret_cast<const double2*>(ut + i);
  v.a0 = *reinterpret_cast<const double2*>(a + i);
  v.l0 = *reinterpret_cast<const double2*>(lam + i);
  const uchar2 hh = *reinterpret_cast<const uchar2*>(H + x);
  v.h0 = (double)hh.x;
  v.h1 = (double)hh.y;
}

__device__ __forceinline__ void local_one(double u1, double u0, double t0, double a0, double l0, double h,
                                          double alpha, double b, double (&acc)[6], double& t1o, double& a1o,
                                          double& l1o) {
  const double t1 = ((a0 + b * u1) - h * l0) / (b + alpha * h);  // pure.py:61
  const double a1 = a0 + b * (u1 - t1);                          // pure.py:66
  const double l1 = l0 + alpha * (h * t1);                       // pure.py:67
  const double s0 = h * t1, s1 = h * (t1 - t0), s3 = u1 - t1, s4 = u1 - u0;
  acc[0] += s0 * s0;   // |H u~'|           r_p1
  acc[1] += s1 * s1;   // |H (u~' - u~)|    r_d1 / alpha
  acc[2] += l1 * l1;   // |lam'|
  acc[3] += s3 * s3;   // |u' - u~'|        r_p3
  acc[4] += s4 * s4;   // |u' - u|          r_d3 / b
  acc[5] += a1 * a1;   // |a'|
  t1o = t1;
  a1o = a1;
  l1o = l1;
}

__device__ __forceinline__ void local_store(const LocalIn& v, int64_t i, double alpha, double b, double (&acc)[6],
                                            double* __restrict__ u, double* __restrict__ ut, double* __restrict__ a,
                                            double* __restrict__ lam, double* __restrict__ R) {
  double2 t1, a1, l1;
  local_one(v.u1.x, v.u0.x, v.t0.x, v.a0.x, v.l0.x, v.h0, alpha, b, acc, t1.x, a1.x, l1.x);
  local_one(v.u1.y, v.u0.y, v.t0.y, v.a0.y, v.l0.y, v.h1, alpha, b, acc, t1.y, a1.y, l1.y);
  *reinterpret_cast<double2*>(u + i) = v.u1;
  *reinterpret_cast<double2*>(ut + i) = t1;
  *reinterpret_cast<double2*>(a + i) = a1;
  *reinterpret_cast<double2*>(lam + i) = l1;
  // the next right-hand side with the pre-adaptation b (k_form_r_fix adds (b' - b) u~'
  // in the rare iterations where residual balancing changed b)
  if (R) *reinterpret_cast<double2*>(R + i) = make_double2(b * t1.x - a1.x, b * t1.y - a1.y);
}

#ifndef PF_FUSED_FORM_R
#define PF_FUSED_FORM_R 1  // the local kernel writes R = b u~' - a' (k_form_r_fix corrects a changed b)
#endif
#ifndef PF_LOCAL_MINB
#define PF_LOCAL_MINB 4  // measured (256^3): S3 0.668 ms at 1 item x 2 per trip, 0.642 at 1 item and 4 CTAs/SM
#endif
#ifndef PF_LOCAL_TWO
#define PF_LOCAL_TWO 0  // two work items per loop trip, all loads first (1) or one (0)
#endif
template <int D>
__global__ void __launch_bounds__(kThreads, PF_LOCAL_MINB) k_stokes_local(
    const int64_t n, const double* __restrict__ un, double* __restrict__ u, double* __restrict__ ut,
    double* __restrict__ a, double* __restrict__ lam, const uint8_t* __restrict__ H,
    const Ctrl* __restrict__ ctrl, double* __restrict__ part, double* __restrict__ R) {
  if (ctrl->done) return;
  const double alpha = ctrl->alpha, b = ctrl->b;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if ((n & 1) == 0) {  // voxel pairs (every field base is 16-byte aligned and c n is even)
    const int64_t np = n >> 1, items = D * np;
    int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    auto at = [&](int64_t k, int64_t& x) {
      const int64_t c = k / np;
      x = (k - c * np) << 1;
      return c * n + x;
    };
    for (; PF_LOCAL_TWO && it + stride < items; it += 2 * stride) {
      int64_t xa, xb;
      const int64_t ia = at(it, xa), ib = at(it + stride, xb);
      LocalIn va, vb;
      local_load(va, ia, xa, un, u, ut, a, lam, H);
      local_load(vb, ib, xb, un, u, ut, a, lam, H);
      local_store(va, ia, alpha, b, acc, u, ut, a, lam, R);
      local_store(vb, ib, alpha, b, acc, u, ut, a, lam, R);
    }
    for (; it < items; it += stride) {
      int64_t xa;
      const int64_t ia = at(it, xa);
      LocalIn va;
      local_load(va, ia, xa, un, u, ut, a, lam, H);
      local_store(va, ia, alpha, b, acc, u, ut, a, lam, R);
    }
  } else {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += stride) {
      const double h = (double)H[x];
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const int64_t i = c * n + x;
        double t1, a1, l1;
        const double u1 = un[i];
        local_one(u1, u[i], ut[i], a[i], lam[i], h, alpha, b, acc, t1, a1, l1);
        u[i] = u1;
        ut[i] = t1;
        a[i] = a1;
        lam[i] = l1;
        if (R) R[i] = b * t1 - a1;
      }
    }
  }
  block_sum<6>(acc);
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) part[(size_t)k * gridDim.x + blockIdx.x] = acc[k];
}

// ---------------------------------------------------------------------- F
__global__ void __launch_bounds__(kFinalizeThreads) k_stokes_finalize(
    Ctrl* __restrict__ ctrl, const double* __restrict__ part3, int nb3, const double* __restrict__ part1,
    int nb1, double* __restrict__ hist, const StokesConst C, const double inv_n) {
  pdl_wait();
#if PF_ABL_FINTRIV  // measurement only: the launch without its work (results invalid)
  if (ctrl->done) return;
  if (threadIdx.x == 0) ctrl->iter += 1;
  return;
#endif
  // the done flag is read together with the partials (a finished solve's finalize
  // reduces stale partials and discards them) so the two loads overlap
  const int32_t done = ctrl->done;
  double S[6], P[3];
#if PF_ABL_NORED  // measurement only: partial reductions skipped (results invalid)
  for (int k = 0; k < 6; ++k) S[k] = 1.0 + k;
  for (int k = 0; k < 3; ++k) P[k] = 1.0 + k;
  (void)part3, (void)nb3, (void)part1, (void)nb1;
#else
  reduce_partials2<6, 3>(part3, nb3, S, part1, nb1, P);
#endif
  if (done || threadIdx.x != 0) return;
  const double alpha = ctrl->alpha, beta = ctrl->beta, b = ctrl->b;
  const double er = C.eps_rel;
  double rp[3], rd[3], tp[3], td[3];
  rp[0] = sqrt(S[0]);
  rd[0] = alpha * sqrt(S[1]);
  const double ln = sqrt(S[2] + C.lam_pore_sq);
  tp[0] = C.tol_vec + er * pymax(rp[0], ln);
  td[0] = C.tol_vec + er * ln;
  rp[1] = sqrt(P[0] * inv_n);
  rd[1] = beta * sqrt(P[1] * inv_n);
  const double qn = sqrt(P[2] * inv_n);
  tp[1] = C.tol_sca + er * pymax(rp[1], qn);
  td[1] = C.tol_sca + er * qn;
  rp[2] = sqrt(S[3]);
  rd[2] = b * sqrt(S[4]);
  const double an = sqrt(S[5]);
  tp[2] = C.tol_vec + er * pymax(rp[2], an);
  td[2] = C.tol_vec + er * an;
  const int64_t it = ctrl->iter + 1;
  ctrl->db = 0.0;
  double* row = hist + (it - 1) * PF_STOKES_COLUMNS;
  for (int k = 0; k < 3; ++k) {
    row[4 * k + 0] = rp[k];
    row[4 * k + 1] = tp[k];
    row[4 * k + 2] = rd[k];
    row[4 * k + 3] = td[k];
  }
  row[12] = alpha;
  row[13] = beta;
  row[14] = b;
  ctrl->iter = it;
  bool passed = true;
  for (int k = 0; k < 3; ++k) passed = passed && (rp[k] <= tp[k] && rd[k] <= td[k]);
  if (passed) {
    ctrl->converged = 1;
    ctrl->done = 1;
    return;
  }
  if (C.adaptive) {  // adapt_penalties, stokes.py:299-310
    double v[3] = {alpha, beta, b};
    for (int k = 0; k < 3; ++k) {
      if (rp[k] == 0.0 && rd[k] == 0.0) continue;
      const double grow = rd[k] == 0.0 ? INFINITY : rp[k] / rd[k];
      const double shrink = rp[k] == 0.0 ? INFINITY : rd[k] / rp[k];
      if (grow > C.thr[k])
        v[k] = C.growth[k] * v[k];
      else if (shrink > C.thr[k])
        v[k] = pymax(v[k] / C.growth[k], C.floor_[k]);
    }
#if PF_ABL_NOADAPT  // measurement only: penalties frozen (results invalid)
    (void)v;
#else
    ctrl->alpha = v[0];
    ctrl->beta = v[1];
    ctrl->b = v[2];
    ctrl->db = PF_ABL_NODB ? 0.0 : v[2] - b;  // (NODB: measurement only, results invalid)
#endif
  }
  if (it >= C.max_iter) ctrl->done = 1;
}

// ---------------------------------------------------------------------- S4
template <int D>
__global__ void __launch_bounds__(kThreads) k_form_r(const int64_t n, const double* __restrict__ ut,
                                                     const double* __restrict__ a, double* __restrict__ R,
                                                     const Ctrl* __restrict__ ctrl, int gated) {
  if (gated && ctrl->done) return;
  const double b = ctrl->b;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < D; ++c) R[c * n + x] = b * ut[c * n + x] - a[c * n + x];
  }
}

// R += (b' - b) u~' when the finalize's residual balancing changed b (the local
// kernel formed R with the pre-adaptation b); a no-op otherwise.
template <int D>
__global__ void __launch_bounds__(kThreads) k_form_r_fix(const int64_t n, const double* __restrict__ ut,
                                                         double* __restrict__ R, const Ctrl* __restrict__ ctrl) {
  if (ctrl->done) return;
  const double db = ctrl->db;
  if (db == 0.0) return;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < D; ++c) R[c * n + x] = R[c * n + x] + db * ut[c * n + x];
  }
}

// ---------------------------------------------------------------------- S3 / S4, solid-only storage
// On pore voxels (H = 0) the local step is u~' = u', a' = 0, lam' = lam (the fused
// compact RS, pf_fused.cu), so once a = 0 there (a cold start, or any state this path
// produced) u~, a and lam need storage and traffic on solid voxels only: [c][ns]
// arrays in voxel order, addressed through exclusive per-64-voxel segment bases and a
// warp ballot.  A warp takes one 64-voxel segment of one component per trip, two
// voxels per lane (16-byte loads of u' and u).  S3 then moves u' (r), u (r+w), R (w)
// and H for every voxel and the multipliers only for the solid fraction.
#ifndef PF_GLOCAL_MINB
// measured (256^3, cuFFT pipeline forced): S3 0.565 ms at one segment per trip and 4
// CTAs/SM; two segments per trip (loads of both first) 0.598 at 2 CTAs/SM, 0.621 at 3
#define PF_GLOCAL_MINB 4
#endif
struct GCompact {
  const uint32_t* base;  // [nseg + 1]
  double *ut, *a, *lam;  // [D][ns]
  int64_t ns;
};

// segment w of component c: voxel pair (x, x + 1) of this lane and the compact
// index of x (of x + 1: + s0)
struct GSeg {
  int64_t i, x, ci;
  bool s0, s1;
};

__device__ __forceinline__ GSeg gseg(int64_t w, int64_t nseg, int64_t n, const uint8_t* __restrict__ H,
                                     const GCompact& cp) {
  const int lane = threadIdx.x & 31;
  const int c = (int)(w / nseg);
  const int64_t seg = w - (int64_t)c * nseg;
  GSeg s;
  s.x = (seg << 6) + 2 * lane;
  s.i = (int64_t)c * n + s.x;
  const uchar2 hh = *reinterpret_cast<const uchar2*>(H + s.x);
  s.s0 = hh.x != 0;
  s.s1 = hh.y != 0;
  const unsigned lt = (1u << lane) - 1u;
  const unsigned m0 = __ballot_sync(0xffffffffu, s.s0), m1 = __ballot_sync(0xffffffffu, s.s1);
  s.ci = (int64_t)c * cp.ns + cp.base[seg] + __popc(m0 & lt) + __popc(m1 & lt);
  return s;
}

// one voxel: solid -> pure.py:59-68 with H = 1 (local_one's evaluation order), compact
// multipliers updated; pore -> u~' = u', a' = 0, lam' = lam (its |lam|^2 is the
// constant StokesConst::lam_pore_sq).  Returns R = b u~' - a'.
struct CIn {
  double t0, a0, l0;
};
__device__ __forceinline__ CIn cload(bool solid, const GCompact& cp, int64_t ci) {
  CIn v{0.0, 0.0, 0.0};
  if (solid) {
    v.t0 = cp.ut[ci];
    v.a0 = cp.a[ci];
    v.l0 = cp.lam[ci];
  }
  return v;
}
__device__ __forceinline__ double local_c(bool solid, double u1, double u0, const CIn& v, double alpha, double b,
                                          double (&acc)[6], const GCompact& cp, int64_t ci) {
  if (solid) {
    double t1, a1, l1;
    local_one(u1, u0, v.t0, v.a0, v.l0, 1.0, alpha, b, acc, t1, a1, l1);
    cp.ut[ci] = t1;
    cp.a[ci] = a1;
    cp.lam[ci] = l1;
    return b * t1 - a1;
  }
  const double s4 = u1 - u0;
  acc[4] += s4 * s4;
  return b * u1 - 0.0;
}

template <int D>
__global__ void __launch_bounds__(kThreads, PF_GLOCAL_MINB) k_stokes_local_c(
    const int64_t n, const double* __restrict__ un, double* __restrict__ u, const uint8_t* __restrict__ H,
    GCompact cp, const Ctrl* __restrict__ ctrl, double* __restrict__ part, double* __restrict__ R) {
  if (ctrl->done) return;
  const double alpha = ctrl->alpha, b = ctrl->b;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int64_t nseg = n >> 6, items = D * nseg;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  for (; w < items; w += nw) {
    const GSeg s = gseg(w, nseg, n, H, cp);
    const double2 u1 = *reinterpret_cast<const double2*>(un + s.i);
    const double2 u0 = *reinterpret_cast<const double2*>(u + s.i);
    const CIn va = cload(s.s0, cp, s.ci), vb = cload(s.s1, cp, s.ci + (s.s0 ? 1 : 0));
    double2 r;
    r.x = local_c(s.s0, u1.x, u0.x, va, alpha, b, acc, cp, s.ci);
    r.y = local_c(s.s1, u1.y, u0.y, vb, alpha, b, acc, cp, s.ci + (s.s0 ? 1 : 0));
    *reinterpret_cast<double2*>(u + s.i) = u1;
    *reinterpret_cast<double2*>(R + s.i) = r;
  }
  block_sum<6>(acc);
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) part[(size_t)k * gridDim.x + blockIdx.x] = acc[k];
}

// R += (b' - b) u~' with u~' = u' on pore voxels, the compact u~ on solid ones
template <int D>
__global__ void __launch_bounds__(kThreads) k_form_r_fix_c(const int64_t n, const double* __restrict__ u,
                                                           const uint8_t* __restrict__ H, GCompact cp,
                                                           double* __restrict__ R, const Ctrl* __restrict__ ctrl) {
  if (ctrl->done) return;
  const double db = ctrl->db;
  if (db == 0.0) return;
  const int64_t nseg = n >> 6, items = D * nseg;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < items; w += nw) {
    const GSeg s = gseg(w, nseg, n, H, cp);
    double2 r = *reinterpret_cast<const double2*>(R + s.i);
    const double2 uu = *reinterpret_cast<const double2*>(u + s.i);
    r.x = r.x + db * (s.s0 ? cp.ut[s.ci] : uu.x);
    r.y = r.y + db * (s.s1 ? cp.ut[s.ci + (s.s0 ? 1 : 0)] : uu.y);
    *reinterpret_cast<double2*>(R + s.i) = r;
  }
}

// dir = 0: full -> compact (solid voxels); dir = 1: compact -> full, pore u~ = u, a = 0,
// lam left untouched
template <int D>
__global__ void __launch_bounds__(kThreads) k_gcompact_move(const int64_t n, const uint8_t* __restrict__ H,
                                                            GCompact cp, double* ut, double* a, double* lam,
                                                            const double* __restrict__ u, int dir) {
  const int64_t nseg = n >> 6, items = D * nseg;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < items; w += nw) {
    const GSeg s = gseg(w, nseg, n, H, cp);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool solid = h ? s.s1 : s.s0;
      const int64_t fi = s.i + h, ci = s.ci + (h && s.s0 ? 1 : 0);
      if (dir == 0) {
        if (solid) {
          cp.ut[ci] = ut[fi];
          cp.a[ci] = a[fi];
          cp.lam[ci] = lam[fi];
        }
      } else if (solid) {
        ut[fi] = cp.ut[ci];
        a[fi] = cp.a[ci];
        lam[fi] = cp.lam[ci];
      } else {
        ut[fi] = u[fi];
        a[fi] = 0.0;
      }
    }
  }
}

__global__ void k_seg_counts(const int64_t nseg, const uint8_t* __restrict__ H, uint32_t* __restrict__ cnt) {
  for (int64_t sg = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sg < nseg; sg += (int64_t)gridDim.x * blockDim.x) {
    const uint4* w = reinterpret_cast<const uint4*>(H + (sg << 6));
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 v = w[k];
      c += __popc(__vcmpne4(v.x, 0u)) + __popc(__vcmpne4(v.y, 0u)) + __popc(__vcmpne4(v.z, 0u)) +
           __popc(__vcmpne4(v.w, 0u));
    }
    cnt[sg] = c >> 3;  // (__vcmpne4 sets all 8 bits of each differing byte)
  }
}

// pore sums over the D components: |a| (eligibility: must be 0) and lam^2
__global__ void __launch_bounds__(kThreads) k_pore_a_lam_d(int64_t n, int D, const uint8_t* __restrict__ H,
                                                           const double* __restrict__ a,
                                                           const double* __restrict__ lam, double* __restrict__ part) {
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < D * n; i += (int64_t)gridDim.x * blockDim.x) {
    if (H[i % n] == 0) {
      acc[0] += fabs(a[i]);
      acc[1] += lam[i] * lam[i];
    }
  }
  block_sum<2>(acc);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = acc[0];
    part[gridDim.x + blockIdx.x] = acc[1];
  }
}

static GCompact gcompact_of(const pf_plan* p) {
  GCompact c;
  const int64_t m = (int64_t)p->g.d * p->gc_ns;
  c.base = p->gc_base;
  c.ut = p->gc_data;
  c.a = p->gc_data + m;
  c.lam = p->gc_data + 2 * m;
  c.ns = p->gc_ns;
  return c;
}

#ifndef PF_GCOMPACT
#define PF_GCOMPACT 1  // solid-only multipliers on the cuFFT pipeline when eligible
#endif

// Decide and set up the cuFFT pipeline's solid-only storage for the solve being begun
// (p->s_* bound; cold = the state is all zero).
static int gcompact_setup(pf_plan* p, bool cold) {
  const int64_t n = p->g.nr;
  const int d = p->g.d;
  p->gc_on = 0;
  p->sc.lam_pore_sq = 0.0;
  const char* e = getenv("POREFLOW_B200_GCOMPACT");
  const bool want = p->compact_enable && (e ? e[0] == '1' : PF_GCOMPACT);
  if (!want || (n & 63) != 0 || n < 64) return PF_OK;
  if (cold) {
    p->h_small[0] = p->h_small[1] = 0.0;
  } else {
    const int nb = blocks_for(d * n);
    k_pore_a_lam_d<<<nb, kThreads, 0, p->work>>>(n, d, p->s_solid, p->s_a, p->s_lam, p->partials);
    PF_CK_CUDA(cudaGetLastError());
    double* out = p->partials + 24 * kMaxBlocks;
    PF_CK(reduce_rows_to(p, p->partials, 2, nb, out));
    PF_CK_CUDA(cudaMemcpyAsync(p->h_small, out, 2 * sizeof(double), cudaMemcpyDeviceToHost, p->work));
    PF_CK_CUDA(cudaStreamSynchronize(p->work));
  }
  if (p->h_small[0] != 0.0) return PF_OK;  // a != 0 on some pore voxel: full storage
  const double lam_pore_sq = p->h_small[1];
  const int64_t nseg = n >> 6;
  if (nseg > p->gc_nseg) {
    cudaFree(p->gc_cnt);
    cudaFree(p->gc_base);
    p->gc_cnt = nullptr;
    p->gc_base = nullptr;
    PF_CK_CUDA(cudaMalloc(&p->gc_cnt, sizeof(uint32_t) * nseg));
    PF_CK_CUDA(cudaMalloc(&p->gc_base, sizeof(uint32_t) * (nseg + 1)));
    p->gc_nseg = nseg;
  }
  k_seg_counts<<<blocks_for(nseg), kThreads, 0, p->work>>>(nseg, p->s_solid, p->gc_cnt);
  PF_CK_CUDA(cudaGetLastError());
  PF_CK(scan_counts(p->work, p->gc_cnt, p->gc_base, nseg));
  uint32_t ns = 0;
  PF_CK_CUDA(cudaMemcpyAsync(p->h_small, p->gc_base + nseg, sizeof(uint32_t), cudaMemcpyDeviceToHost, p->work));
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  std::memcpy(&ns, p->h_small, sizeof(uint32_t));
  p->gc_ns = ns;
  const int64_t need = 3 * (int64_t)d * (ns > 0 ? ns : 1);
  if (need > p->gc_cap) {
    cudaFree(p->gc_data);
    p->gc_data = nullptr;
    PF_CK_CUDA(cudaMalloc(&p->gc_data, sizeof(double) * (size_t)need));
    p->gc_cap = need;
  }
  if (cold) {
    PF_CK_CUDA(cudaMemsetAsync(p->gc_data, 0, sizeof(double) * (size_t)need, p->work));
  } else {
    const GCompact cp = gcompact_of(p);
    const int nb = blocks_for(d * n / 2);
    switch (d) {
      case 1: k_gcompact_move<1><<<nb, kThreads, 0, p->work>>>(n, p->s_solid, cp, p->s_ut, p->s_a, p->s_lam, p->s_u, 0); break;
      case 2: k_gcompact_move<2><<<nb, kThreads, 0, p->work>>>(n, p->s_solid, cp, p->s_ut, p->s_a, p->s_lam, p->s_u, 0); break;
      default: k_gcompact_move<3><<<nb, kThreads, 0, p->work>>>(n, p->s_solid, cp, p->s_ut, p->s_a, p->s_lam, p->s_u, 0); break;
    }
    PF_CK_CUDA(cudaGetLastError());
  }
  p->gc_on = 1;
  p->sc.lam_pore_sq = lam_pore_sq;
  return PF_OK;
}

// u~, a, lam back into the caller's full arrays (pore: u~ = u, a = 0, lam unchanged)
static int gcompact_finish(pf_plan* p) {
  if (!p->gc_on) return PF_OK;
  const int64_t n = p->g.nr;
  const GCompact cp = gcompact_of(p);
  const int nb = blocks_for(p->g.d * n / 2);
  switch (p->g.d) {
    case 1: k_gcompact_move<1><<<nb, kThreads, 0, p->work>>>(n, p->s_solid, cp, p->s_ut, p->s_a, p->s_lam, p->s_u, 1); break;
    case 2: k_gcompact_move<2><<<nb, kThreads, 0, p->work>>>(n, p->s_solid, cp, p->s_ut, p->s_a, p->s_lam, p->s_u, 1); break;
    default: k_gcompact_move<3><<<nb, kThreads, 0, p->work>>>(n, p->s_solid, cp, p->s_ut, p->s_a, p->s_lam, p->s_u, 1); break;
  }
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;  // (gc_on stays set: pf_stokes_pipeline reports the finished solve's pipeline)
}

// ---------------------------------------------------------------------- setup helpers
// D^ = sum_c i k_c U^_c of the initial velocity (div_prev, stokes.py:370).
template <int D>
__global__ void k_div_spectrum(Geom g, Tables T, const double2* __restrict__ Uh, double2* __restrict__ Dh) {
  const uint32_t nh = (uint32_t)g.nh;
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < nh; m += gridDim.x * blockDim.x) {
    int idx[3];
    mode_index(g, m, idx);
    idx[1] += g.k1off;
    double2 dv = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const int ax = 3 - D + c;
      dv = cadd(dv, cik(__ldg(T.kap[ax] + idx[ax]), Uh[(size_t)c * nh + m]));
    }
    Dh[m] = dv;
  }
}

__global__ void k_zero_mode(double2* Qh) { Qh[0] = make_double2(0.0, 0.0); }

__global__ void k_scale_copy(int64_t nh, const double2* __restrict__ src, double2* __restrict__ dst, double s) {
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < nh; m += (int64_t)gridDim.x * blockDim.x)
    dst[m] = make_double2(src[m].x * s, src[m].y * s);
}

__global__ void k_ctrl_init(Ctrl* c, double alpha, double beta, double b) {
  c->alpha = alpha;
  c->beta = beta;
  c->b = b;
  c->db = 0.0;
  c->best = INFINITY;
  c->iter = 0;
  c->done = c->converged = c->diverged = c->reason = 0;
}

// ---------------------------------------------------------------------- host side
// One loop iteration.  With `ev` (7 events) the stage boundaries are recorded
// for pf_stokes_profile: S1 | Z2D | S3 | F | S4 | D2Z.
template <int D>
static int enqueue_stokes_t(pf_plan* p, cudaEvent_t* ev = nullptr) {
  const Geom& g = p->g;
  const int64_t n = g.nr, nh = g.nh;
  const int nb1 = blocks_for(nh), nb3 = blocks_for(n);
  double* part1 = p->partials;                   // 3 x nb1
  double* part3 = p->partials + 3 * kMaxBlocks;  // 6 x nb3
  double2* Rh = p->specA;
  double2* Uh = p->specB;
  double2* Qh = p->spec1;
  double2* Dh = p->spec2;
  double* un = p->realA;
  double* R = p->realB;
  const StokesConst& C = p->sc;
  auto mark = [&](int i) -> int {
    if (ev) PF_CK_CUDA(cudaEventRecord(ev[i], p->work));
    return PF_OK;
  };
  PF_CK(mark(0));
  k_stokes_spectral<D><<<nb1, kThreads, 0, p->work>>>(g, tables_of(p), C.nu, C.g[0], C.g[1], C.g[2], Qh, Rh, Dh,
                                                      Uh, p->ctrl, part1);
  PF_CK_CUDA(cudaGetLastError());
  PF_CK(mark(1));
  PF_CK(plan_fft(p, false, D, Uh, un));
  PF_CK(mark(2));
  if (p->gc_on)
    k_stokes_local_c<D><<<nb3, kThreads, 0, p->work>>>(n, un, p->s_u, p->s_solid, gcompact_of(p), p->ctrl, part3, R);
  else
    k_stokes_local<D><<<nb3, kThreads, 0, p->work>>>(n, un, p->s_u, p->s_ut, p->s_a, p->s_lam, p->s_solid, p->ctrl,
                                                     part3, PF_FUSED_FORM_R ? R : nullptr);
  PF_CK_CUDA(cudaGetLastError());
  PF_CK(mark(3));
  k_stokes_finalize<<<1, kFinalizeThreads, 0, p->work>>>(p->ctrl, part3, nb3, part1, nb1, p->s_hist, C, g.inv_n);
  PF_CK_CUDA(cudaGetLastError());
  PF_CK(mark(4));
  if (p->gc_on)
    k_form_r_fix_c<D><<<nb3, kThreads, 0, p->work>>>(n, p->s_u, p->s_solid, gcompact_of(p), R, p->ctrl);
  else if (PF_FUSED_FORM_R)
    k_form_r_fix<D><<<nb3, kThreads, 0, p->work>>>(n, p->s_ut, R, p->ctrl);
  else
    k_form_r<D><<<nb3, kThreads, 0, p->work>>>(n, p->s_ut, p->s_a, R, p->ctrl, 1);
  PF_CK_CUDA(cudaGetLastError());
  PF_CK(mark(5));
  PF_CK(plan_fft(p, true, D, R, Rh));
  PF_CK(mark(6));
  return PF_OK;
}

static int enqueue_stokes(pf_plan* p) {
  if (p->pipeline == 1) return enqueue_fused(p, nullptr);
  switch (p->g.d) {
    case 1: return enqueue_stokes_t<1>(p);
    case 2: return enqueue_stokes_t<2>(p);
    default: return enqueue_stokes_t<3>(p);
  }
}

static int enqueue_stokes_ev(pf_plan* p, cudaEvent_t* ev) {
  if (p->pipeline == 1) return enqueue_fused(p, ev);
  switch (p->g.d) {
    case 1: return enqueue_stokes_t<1>(p, ev);
    case 2: return enqueue_stokes_t<2>(p, ev);
    default: return enqueue_stokes_t<3>(p, ev);
  }
}

int stokes_spectral_launch(pf_plan* p, const Geom& gs, double2* Qh, const double2* Rh, double2* Dh, double2* Uh,
                           double* part1, int* nb1) {
  const int nb = blocks_for(gs.nh);
  const StokesConst& C = p->sc;
  k_stokes_spectral<3><<<nb, kThreads, 0, p->work>>>(gs, tables_of(p), C.nu, C.g[0], C.g[1], C.g[2], Qh, Rh, Dh, Uh,
                                                     p->ctrl, part1);
  PF_CK_CUDA(cudaGetLastError());
  *nb1 = nb;
  return PF_OK;
}

int stokes_local_launch(pf_plan* p, int64_t n, const double* un, double* part3, int* nb3) {
  const int nb = blocks_for(n);
  k_stokes_local<3><<<nb, kThreads, 0, p->work>>>(n, un, p->s_u, p->s_ut, p->s_a, p->s_lam, p->s_solid, p->ctrl,
                                                  part3, nullptr);
  PF_CK_CUDA(cudaGetLastError());
  *nb3 = nb;
  return PF_OK;
}

int stokes_ctrl_init(pf_plan* p, double alpha, double beta, double b) {
  k_ctrl_init<<<1, 1, 0, p->work>>>(p->ctrl, alpha, beta, b);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

int stokes_form_r_gated(pf_plan* p, double* R, int gated) {
  const int64_t n = p->g.nr;
  k_form_r<3><<<blocks_for(n), kThreads, 0, p->work>>>(n, p->s_ut, p->s_a, R, p->ctrl, gated);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

int stokes_div_launch(pf_plan* p, const Geom& gs, const double2* Uh, double2* Dh) {
  k_div_spectrum<3><<<blocks_for(gs.nh), kThreads, 0, p->work>>>(gs, tables_of(p), Uh, Dh);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

int stokes_div_spectrum(pf_plan* p, const double* u, double2* tmp, double2* out) {
  const int d = p->g.d;
  PF_CK(plan_fft(p, true, d, (void*)u, tmp));
  const int nb = blocks_for(p->g.nh);
  switch (d) {
    case 1: k_div_spectrum<1><<<nb, kThreads, 0, p->work>>>(p->g, tables_of(p), tmp, out); break;
    case 2: k_div_spectrum<2><<<nb, kThreads, 0, p->work>>>(p->g, tables_of(p), tmp, out); break;
    default: k_div_spectrum<3><<<nb, kThreads, 0, p->work>>>(p->g, tables_of(p), tmp, out); break;
  }
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

int stokes_form_r(pf_plan* p, double* R) {
  const int64_t n = p->g.nr;
  switch (p->g.d) {
    case 1: k_form_r<1><<<blocks_for(n), kThreads, 0, p->work>>>(n, p->s_ut, p->s_a, R, p->ctrl, 0); break;
    case 2: k_form_r<2><<<blocks_for(n), kThreads, 0, p->work>>>(n, p->s_ut, p->s_a, R, p->ctrl, 0); break;
    default: k_form_r<3><<<blocks_for(n), kThreads, 0, p->work>>>(n, p->s_ut, p->s_a, R, p->ctrl, 0); break;
  }
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

cudaError_t k_stokes_finalize_launch_pdl(pf_plan* p, const double* part3, int nb3, const double* part1, int nb1) {
  return launch_k(k_stokes_finalize, 1, kFinalizeThreads, 0, p->work, p->ctrl, part3, nb3, part1, nb1, p->s_hist,
                  p->sc, p->g.inv_n);
}

void k_stokes_finalize_launch(pf_plan* p, const double* part3, int nb3, const double* part1, int nb1) {
  k_stokes_finalize<<<1, kFinalizeThreads, 0, p->work>>>(p->ctrl, part3, nb3, part1, nb1, p->s_hist, p->sc,
                                                          p->g.inv_n);
}

template <int D>
static int stokes_setup_t(pf_plan* p, bool cold) {
  const Geom& g = p->g;
  const int64_t n = g.nr, nh = g.nh;
  if (cold) {  // zero state: Q^ = D^ = 0 and R^ = FFT(b 0 - 0) = 0, no transforms
    PF_CK_CUDA(cudaMemsetAsync(p->spec1, 0, sizeof(double2) * nh, p->work));
    PF_CK_CUDA(cudaMemsetAsync(p->spec2, 0, sizeof(double2) * nh, p->work));
    PF_CK_CUDA(cudaMemsetAsync(p->specA, 0, sizeof(double2) * D * nh, p->work));
    return gcompact_setup(p, true);
  }
  // Q^ = FFT(q), gauge Q^(0) = 0 (stokes.py:363, 367)
  PF_CK(plan_fft(p, true, 1, p->s_q, p->spec1));
  k_zero_mode<<<1, 1, 0, p->work>>>(p->spec1);
  // D^_prev = i k . FFT(u)  (stokes.py:370)
  PF_CK(plan_fft(p, true, D, p->s_u, p->specB));
  k_div_spectrum<D><<<blocks_for(nh), kThreads, 0, p->work>>>(g, tables_of(p), p->specB, p->spec2);
  // R^ = FFT(b u~ - a)  (stokes.py:368-369)
  k_form_r<D><<<blocks_for(n), kThreads, 0, p->work>>>(n, p->s_ut, p->s_a, p->realB, p->ctrl, 0);
  PF_CK(plan_fft(p, true, D, p->realB, p->specA));
  PF_CK_CUDA(cudaGetLastError());
  return gcompact_setup(p, false);
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_stokes_begin(pf_plan* p, const pf_stokes_params* P, const uint8_t* solid, double* u, double* ut, double* q,
                    double* a, double* lam, double* history) {
  PF_NVTX("pf_stokes_begin");
  PF_ARG(p && P && solid && u && ut && q && a && lam && history, "null argument");
  PF_ARG(P->b > 0.0, "coupling penalty b must be positive for the zero mode");
  PF_ARG(P->nu > 0.0, "viscosity must be positive");
  PF_ARG(P->max_iter >= 1, "max_iter must be at least 1");
  PF_CK(enter(p));
  PF_CK(plan_ensure_scratch(p));
  if (p->active != 1) p->graph.reset();
  p->active = 1;
  p->s_solid = solid;
  p->s_u = u;
  p->s_ut = ut;
  p->s_q = q;
  p->s_a = a;
  p->s_lam = lam;
  p->s_hist = history;
  StokesConst& C = p->sc;
  const int d = p->g.d;
  C.nu = P->nu;
  C.eps_rel = P->eps_rel;
  C.tol_vec = std::sqrt((double)(d * p->g.nr)) * P->eps_abs;
  C.tol_sca = std::sqrt((double)p->g.nr) * P->eps_abs;
  for (int k = 0; k < 3; ++k) {
    C.g[k] = k < d ? P->pressure_gradient[k] : 0.0;
    C.growth[k] = P->growth[k];
    C.thr[k] = P->ratio_threshold[k];
    C.floor_[k] = P->floor[k];
  }
  C.max_iter = P->max_iter;
  C.adaptive = P->adaptive;
  C.lam_pore_sq = 0.0;
  // Graph kernels capture StokesConst and the state pointers by value.
  p->graph.reset();
  k_ctrl_init<<<1, 1, 0, p->work>>>(p->ctrl, P->alpha, P->beta, P->b);
  PF_CK_CUDA(cudaGetLastError());
  p->pipeline = (p->fused_enable && fused_supported(p)) ? 1 : 0;
  p->gc_on = 0;
  if (p->pipeline == 1) {
    PF_CK(fused_ensure(p));
    const int st = fused_setup(p);
    p->cold_start = 0;  // consumed
    return st;
  }
  const bool cold = p->cold_start != 0;
  p->cold_start = 0;
  switch (d) {
    case 1: PF_CK(stokes_setup_t<1>(p, cold)); break;
    case 2: PF_CK(stokes_setup_t<2>(p, cold)); break;
    default: PF_CK(stokes_setup_t<3>(p, cold)); break;
  }
  return PF_OK;
}

int pf_stokes_iterate(pf_plan* p, int64_t n_iter, int poll, pf_stokes_result* res) {
  PF_NVTX("pf_stokes_iterate");
  PF_ARG(p, "null plan");
  if (p->active != 1) {
    set_error("pf_stokes_iterate without pf_stokes_begin");
    return PF_ERR_STATE;
  }
  Ctrl c;
  PF_CK(enter(p));
  PF_CK(run_chunks(p, n_iter, poll, enqueue_stokes, &c));
  PF_CK(leave(p));
  if (res && c.iter >= 0) {
    res->iterations = c.iter;
    res->converged = c.converged;
    res->done = c.done;
    res->final_penalties[0] = c.alpha;
    res->final_penalties[1] = c.beta;
    res->final_penalties[2] = c.b;
  }
  return PF_OK;
}

int pf_stokes_end(pf_plan* p, pf_stokes_result* res) {
  PF_NVTX("pf_stokes_end");
  PF_ARG(p, "null plan");
  if (p->active != 1) {
    set_error("pf_stokes_end without pf_stokes_begin");
    return PF_ERR_STATE;
  }
  // q = Re ifft(Q^): copy (Z2D overwrites its input), fold 1/n, transform.
  const int64_t nh = p->g.nh;
  if (p->pipeline == 1) {
    PF_CK(fused_finish(p));
  } else {
    k_scale_copy<<<blocks_for(nh), kThreads, 0, p->work>>>(nh, p->spec1, p->specB, p->g.inv_n);
    PF_CK_CUDA(cudaGetLastError());
    PF_CK(plan_fft(p, false, 1, p->specB, p->s_q));
    PF_CK(gcompact_finish(p));
  }
  PF_CK_CUDA(cudaMemcpyAsync(&p->h_ctrl[0], p->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, p->work));
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  const Ctrl c = p->h_ctrl[0];
  if (res) {
    res->iterations = c.iter;
    res->converged = c.converged;
    res->done = c.done;
    res->final_penalties[0] = c.alpha;
    res->final_penalties[1] = c.beta;
    res->final_penalties[2] = c.b;
  }
  p->active = 0;
  PF_CK(leave(p));
  return PF_OK;
}

int pf_stokes_profile(pf_plan* p, int64_t n_iter, double* stage_ms) {
  PF_ARG(p && stage_ms && n_iter >= 1, "bad argument");
  if (p->active != 1) {
    set_error("pf_stokes_profile without pf_stokes_begin");
    return PF_ERR_STATE;
  }
  PF_CK(enter(p));
  cudaEvent_t ev[7];
  for (int i = 0; i < 7; ++i) PF_CK_CUDA(cudaEventCreate(&ev[i]));
  double acc[6] = {0, 0, 0, 0, 0, 0};
  int st = PF_OK;
  for (int64_t it = 0; it < n_iter && st == PF_OK; ++it) {
    st = enqueue_stokes_ev(p, ev);
    if (st != PF_OK) break;
    if (cudaEventSynchronize(ev[6]) != cudaSuccess) {
      set_error("event sync failed");
      st = PF_ERR_CUDA;
      break;
    }
    for (int k = 0; k < 6; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
      acc[k] += ms;
    }
  }
  for (int i = 0; i < 7; ++i) cudaEventDestroy(ev[i]);
  PF_CK(st);
  for (int k = 0; k < 6; ++k) stage_ms[k] = acc[k] / (double)n_iter;
  return leave(p);
}

int pf_stokes_pipeline(const pf_plan* p) {
  if (!p) return -1;
  if (p->pipeline == 1) return fused_is_compact(p) ? 2 : 1;
  return p->gc_on ? 3 : 0;
}

int pf_stokes_solve(pf_plan* p, const pf_stokes_params* P, const uint8_t* solid, double* u, double* ut, double* q,
                    double* a, double* lam, double* history, pf_stokes_result* res) {
  PF_NVTX("pf_stokes_solve");
  PF_CK(pf_stokes_begin(p, P, solid, u, ut, q, a, lam, history));
  pf_stokes_result r{};
  PF_CK(pf_stokes_iterate(p, P->max_iter, 1, &r));
  return pf_stokes_end(p, res);
}

}  // extern "C"
