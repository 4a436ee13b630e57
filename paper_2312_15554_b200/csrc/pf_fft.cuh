// Shared building blocks of the fused pipelines (pf_fused.cu: Stokes,
// pf_fused_transport.cu: transport): in-register radix-8/16 DFTs, the padded
// shared-memory four-step FFT of one sequence per 8/16-lane group, and the
// TMA bulk-copy / LDGSTS helpers.
#pragma once

#include <cmath>

#include "pf_internal.cuh"


namespace pf {
namespace fz {

// Sequences of N <= 256 points are transformed by one 8/16-lane group with the
// two-pass scheme below.  Longer ones (N = M * 256, M = 2, 4) are M padded blocks
// of L = 256: a radix-M stage over the whole sequence (all threads of the block)
// plus M independent L-point transforms.  Space-domain element e = j + L b sits in
// block b at position j (sp); spectral index k = M m + r in block r at position m
// (kp) — the forward transform leaves the spectrum in that order and the inverse
// takes it, so only the index maps differ from the short case.
template <int N>
struct Cfg {
  static constexpr int M = N > 256 ? N / 256 : 1;  // blocks of a long sequence
  static constexpr int L = N / M;                  // length of one block transform (<= 256)
  static constexpr int A = (L == 64) ? 8 : 16;     // radix of pass 1 (and stride of pass-1 stores)
  static constexpr int B = L / A;                  // radix of pass 2
  static constexpr int G = A > B ? A : B;          // lanes per FFT group
  static constexpr int NG = 256 / G;               // groups per 256-thread block
  static constexpr int SSL = L + L / A + 1;        // padded smem stride of one block (complex)
  static constexpr int SS = M * SSL;               // padded smem sequence stride (complex)
  static constexpr int H = N / 2;                  // stored half-spectrum columns (k2 < N/2)
  static constexpr int LOGN = N == 64 ? 6 : (N == 128 ? 7 : (N == 256 ? 8 : (N == 512 ? 9 : 10)));
  static constexpr int RSR = NG;                   // rows per RS tile
  static constexpr int CM = NG;                    // k2 columns per MF / MI tile
  static constexpr int CP = NG / 2;                // k2 columns per PK tile
  static constexpr int NCHM = H / CM;              // column chunks per i0 (M kernels)
  static constexpr int NCHP = H / CP;              // column chunks per k1 (PK)
  static constexpr int M_TILES = N * NCHM + N / CM;
  static constexpr int PK_TILES = N * NCHP + N / CP;
  static constexpr int RS_TILES = N * N / RSR;
  // compact pass-1 twiddle table: rows w^b (b = 1..3) and w^(4a) (a = 1..A/4-1), B lanes each
  static constexpr int TWL = (3 + A / 4 - 1) * B;
  // + for long sequences the radix-M stage's w_N^j (L entries; w_N^(j r) = its r-th power)
  static constexpr int TWN = TWL + (M > 1 ? L : 0);
  static __device__ __forceinline__ int pad(int e) { return e + e / A; }  // within one block
  static __device__ __forceinline__ int sp(int e) { return M == 1 ? pad(e) : (e / L) * SSL + pad(e % L); }
  static __device__ __forceinline__ int kp(int k) { return M == 1 ? pad(k) : (k % M) * SSL + pad(k / M); }
};

// cos(2 pi m / 16)
__device__ __forceinline__ double c16(int m) {
  switch (m & 15) {
    case 0: return 1.0;
    case 1: case 15: return 0.92387953251128675613;
    case 2: case 14: return 0.70710678118654752440;
    case 3: case 13: return 0.38268343236508977173;
    case 4: case 12: return 0.0;
    case 5: case 11: return -0.38268343236508977173;
    case 6: case 10: return -0.70710678118654752440;
    case 7: case 9: return -0.92387953251128675613;
    default: return -1.0;
  }
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -(a.y * b.y)), __fma_rn(a.x, b.y, a.y * b.x));
}


// ---- TMA bulk copies (cp.async.bulk -> UBLKCP) completed on an mbarrier
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(m)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(m))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}" ::"r"(
          su32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// 16-byte LDGSTS into an arbitrary (16-B aligned) shared address, L1 bypass.
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit_wait_all() {
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// x * exp(-+ 2 pi i m / 16): forward uses the minus sign.
template <bool INV>
__device__ __forceinline__ double2 rot16(double2 x, int m) {
  m &= 15;
  if (m == 0) return x;
  if (m == 8) return make_double2(-x.x, -x.y);
  if (m == 4) return INV ? make_double2(-x.y, x.x) : make_double2(x.y, -x.x);
  if (m == 12) return INV ? make_double2(x.y, -x.x) : make_double2(-x.y, x.x);
  const double c = c16(m), s0 = c16(m - 4);  // sin(2 pi m/16)
  const double s = INV ? s0 : -s0;
  return make_double2(__fma_rn(x.x, c, -(x.y * s)), __fma_rn(x.x, s, x.y * c));
}

template <int R, bool INV>
struct Dft;

template <bool INV>
struct Dft<1, INV> {
  static __device__ __forceinline__ void run(double2*) {}
};

template <bool INV>
struct Dft<2, INV> {
  static __device__ __forceinline__ void run(double2* x) {
    const double2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  }
};

template <bool INV>
struct Dft<4, INV> {
  static __device__ __forceinline__ void run(double2* x) {
    const double2 s02 = cadd(x[0], x[2]), d02 = csub(x[0], x[2]);
    const double2 s13 = cadd(x[1], x[3]), d13 = csub(x[1], x[3]);
    // forward: X1 = d02 - i d13, X3 = d02 + i d13
    const double2 jd = INV ? make_double2(-d13.y, d13.x) : make_double2(d13.y, -d13.x);
    x[0] = cadd(s02, s13);
    x[2] = csub(s02, s13);
    x[1] = cadd(d02, jd);
    x[3] = csub(d02, jd);
  }
};

// R = P * Q four-step in registers: n = Q n1 + n2, k = k1 + P k2.
template <int P, int Q, bool INV>
__device__ __forceinline__ void dft_pq(double2* x) {
  constexpr int R = P * Q;
  double2 y[R];
#pragma unroll
  for (int n2 = 0; n2 < Q; ++n2) {
    double2 t[P];
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) t[n1] = x[Q * n1 + n2];
    Dft<P, INV>::run(t);
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) y[n2 * P + k1] = rot16<INV>(t[k1], (n2 * k1) * (16 / R));
  }
#pragma unroll
  for (int k1 = 0; k1 < P; ++k1) {
    double2 t[Q];
#pragma unroll
    for (int n2 = 0; n2 < Q; ++n2) t[n2] = y[n2 * P + k1];
    Dft<Q, INV>::run(t);
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) x[k1 + P * k2] = t[k2];
  }
}

template <bool INV>
struct Dft<8, INV> {
  static __device__ __forceinline__ void run(double2* x) { dft_pq<4, 2, INV>(x); }
};
template <bool INV>
struct Dft<16, INV> {
  static __device__ __forceinline__ void run(double2* x) { dft_pq<4, 4, INV>(x); }
};

// Pass-1 twiddle table (Cfg::TWN entries): the rows fft_seq reads, w^(b l) for
// b = 1..3 then w^(4a l) for a = 1..A/4-1, each laid out over the lanes l < B
// (w = exp(-2 pi i / N)).  Lane-consecutive, so a quarter-warp never hits the
// same bank twice (the natural tw[l*k1] layout is 2..8-way conflicted for even k1).
template <int N>
inline void pass1_twiddles(double2* out) {
  using C = Cfg<N>;
  constexpr int L = C::L;
  int r = 0;
  auto row = [&](int k1) {
    for (int l = 0; l < C::B; ++l) {
      const double a = 2.0 * M_PI * (double)(l * k1) / (double)L;
      out[r * C::B + l] = make_double2(std::cos(a), -std::sin(a));
    }
    ++r;
  };
  for (int b = 1; b < 4; ++b) row(b);
  for (int a = 1; a < C::A / 4; ++a) row(4 * a);
  if (C::M > 1)  // radix-M stage: w_N^j
    for (int j = 0; j < L; ++j) {
      const double a = 2.0 * M_PI * (double)j / (double)N;
      out[C::TWL + j] = make_double2(std::cos(a), -std::sin(a));
    }
}

// Remainder of fft_seq once pass 1's inputs are in registers: x[n1] = element
// B*n1 + l (lanes l < B).  Lets a caller stage the sequence elsewhere (e.g. a
// swizzled TMA tile) and read it straight into registers.
template <int N, bool INV>
__device__ __forceinline__ void fft_seq_x(double2* x, double2* s, const double2* __restrict__ tw, int l, bool active) {
  using C = Cfg<N>;
  constexpr int A = C::A, B = C::B;
  const bool p1 = active && l < B, p2 = active && l < A;
  if (p1) {
    Dft<A, INV>::run(x);
    // w^(4a+b) = w^(4a) * w^b from 3 + A/4-1 table loads instead of A-1 (shared
    // memory bandwidth is the scarce resource of these kernels); <= 2 ulp.
    double2 wb[4], wa[A / 4];
#pragma unroll
    for (int b = 1; b < 4; ++b) wb[b] = tw[(b - 1) * B + l];
#pragma unroll
    for (int a = 1; a < A / 4; ++a) wa[a] = tw[(2 + a) * B + l];
#pragma unroll
    for (int k1 = 1; k1 < A; ++k1) {
      const int a = k1 / 4, b = k1 % 4;
      double2 w = (a == 0) ? wb[b] : (b == 0 ? wa[a] : cmul(wa[a], wb[b]));
      if (INV) w.y = -w.y;
      x[k1] = cmul(x[k1], w);
    }
  }
  __syncwarp();
  if (p1) {
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) s[C::pad(k1 + A * l)] = x[k1];
  }
  __syncwarp();
  if (p2) {
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) x[n2] = s[C::pad(l + A * n2)];
    Dft<B, INV>::run(x);
#pragma unroll
    for (int k2 = 0; k2 < B; ++k2) s[C::pad(l + A * k2)] = x[k2];
  }
  __syncwarp();
}

// One N-point complex FFT (unnormalised) of the padded smem sequence s by the
// G lanes of a group (lane l).  Pass 1: B sub-FFTs of size A over stride-B
// elements + twiddles; pass 2: A sub-FFTs of size B.  Output in natural order.
// Every lane of the warp must call this (it uses __syncwarp); `active` = false
// makes a group participate without touching memory.
template <int N, bool INV>
__device__ __forceinline__ void fft_seq(double2* s, const double2* __restrict__ tw, int l, bool active) {
  using C = Cfg<N>;
  constexpr int A = C::A, B = C::B;
  double2 x[A > B ? A : B];
  if (active && l < B) {
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) x[n1] = s[C::pad(B * n1 + l)];
  }
  fft_seq_x<N, INV>(x, s, tw, l, active);
}

// a[r] *= w_N^(j r) (conjugated for the inverse), r = 1..M-1; w_N^j from the
// table, its powers by complex multiplication (<= 2 ulp)
template <int N, bool INV>
__device__ __forceinline__ void radix_twiddle(double2* a, const double2* __restrict__ tw, int j) {
  using C = Cfg<N>;
  if constexpr (C::M > 1) {
    double2 w1 = tw[C::TWL + j];
    if (INV) w1.y = -w1.y;
    double2 w = w1;
#pragma unroll
    for (int r = 1; r < C::M; ++r) {
      a[r] = cmul(a[r], w);
      if (r + 1 < C::M) w = cmul(w, w1);
    }
  }
}

__device__ __forceinline__ double2 shfl_xor2(double2 v, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

// Radix-2 merge of the lane pair (j, j + 16) after each lane's 8-point DFT (x = E on
// h = 0, O on h = 1): X[k] = E + w16^k O on h = 0, X[k + 8] = E - w16^k O on h = 1.
// Every lane runs the same instructions — the rotation by a per-lane factor (1 on
// h = 0, rot16's (c, s) on h = 1) and the butterfly as one signed FMA — so the warp
// issues no selects; bitwise the results of the branch / select form (up to the sign
// of zeros).
template <bool INV>
__device__ __forceinline__ void w32_merge(double2* x, int h) {
  Dft<8, INV>::run(x);
  const bool odd = h != 0;
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    const double c = odd ? c16(k) : 1.0;
    const double s0 = odd ? c16(k - 4) : 0.0;  // sin(2 pi k / 16)
    const double s = INV ? s0 : -s0;
    x[k] = make_double2(__fma_rn(x[k].x, c, -(x[k].y * s)), __fma_rn(x[k].x, s, x[k].y * c));
  }
  const double sg = odd ? -1.0 : 1.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 y = shfl_xor2(x[k], 16);
    x[k] = make_double2(__fma_rn(sg, x[k].x, y.x), __fma_rn(sg, x[k].y, y.y));
  }
}

// One 256-point FFT (unnormalised; same input / output positions and padding as
// fft_seq<256>) by a whole warp: each 16-point DFT of the two passes is split
// over a lane pair (j, j + 16) as an 8-point DFT of its even / odd inputs and a
// radix-2 merge through one shuffle exchange, so a sequence's two passes take
// half the dependent-instruction latency of the 16-lane version and both warps
// of a two-sequence tile can work at once.  Every lane must call it.
// fft256_w32 once pass 1's inputs are in registers: x[m] = element 16 (2 m + h) + j
// (lane = 16 h + j) — lets a caller read them straight from a TMA tile.
template <bool INV>
__device__ __forceinline__ void fft256_w32_x(double2* x, double2* s, const double2* __restrict__ tw, int lane,
                                             bool active) {
  using C = Cfg<256>;
  const int j = lane & 15, h = lane >> 4;
  auto merge = [&](void) { w32_merge<INV>(x, h); };
  // pass 1: sub-DFT j over n1 (elements 16 n1 + j); this lane's half n1 = 2 m + h
  merge();
  {
    // twiddle w^(k1 j), k1 = k + 8 h = 4 a + b, from the [k1][l] table rows
    double2 wb[4], wa[2];
#pragma unroll
    for (int b = 1; b < 4; ++b) wb[b] = tw[(b - 1) * C::B + j];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int a = 2 * h + q;
      wa[q] = a == 0 ? make_double2(1.0, 0.0) : tw[(2 + a) * C::B + j];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int q = k / 4, b = k % 4;
      if (h == 0 && k == 0) continue;
      double2 w = b == 0 ? wa[q] : (h == 0 && q == 0 ? wb[b] : cmul(wa[q], wb[b]));
      if (INV) w.y = -w.y;
      x[k] = cmul(x[k], w);
    }
  }
  __syncwarp();
  if (active) {
#pragma unroll
    for (int k = 0; k < 8; ++k) s[C::pad(k + 8 * h + 16 * j)] = x[k];
  }
  __syncwarp();
  // pass 2: sub-DFT j over n2 (elements j + 16 n2); half n2 = 2 m + h
  if (active) {
#pragma unroll
    for (int m = 0; m < 8; ++m) x[m] = s[C::pad(j + 16 * (2 * m + h))];
  }
  merge();
  __syncwarp();
  if (active) {
#pragma unroll
    for (int k = 0; k < 8; ++k) s[C::pad(j + 16 * (k + 8 * h))] = x[k];
  }
  __syncwarp();
}

// fft256_w32_x whose result stays in registers (STORE = false: x[k] = X[j + 16 (k + 8 h)],
// lane = 16 h + j) or goes to out(f, X[f]) (STORE = true) instead of the scratch
// sequence; s is the warp's padded scratch for the one transpose.
template <bool INV, bool STORE, typename Out>
__device__ __forceinline__ void fft256_w32_r(double2* x, double2* s, const double2* __restrict__ tw, int lane,
                                             Out&& out) {
  using C = Cfg<256>;
  const int j = lane & 15, h = lane >> 4;
  auto merge = [&](void) { w32_merge<INV>(x, h); };
  merge();
  {
    double2 wb[4], wa[2];
#pragma unroll
    for (int b = 1; b < 4; ++b) wb[b] = tw[(b - 1) * C::B + j];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int a = 2 * h + q;
      wa[q] = a == 0 ? make_double2(1.0, 0.0) : tw[(2 + a) * C::B + j];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int q = k / 4, b = k % 4;
      if (h == 0 && k == 0) continue;
      double2 w = b == 0 ? wa[q] : (h == 0 && q == 0 ? wb[b] : cmul(wa[q], wb[b]));
      if (INV) w.y = -w.y;
      x[k] = cmul(x[k], w);
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) s[C::pad(k + 8 * h + 16 * j)] = x[k];
  __syncwarp();
#pragma unroll
  for (int m = 0; m < 8; ++m) x[m] = s[C::pad(j + 16 * (2 * m + h))];
  merge();
  if constexpr (STORE) {
#pragma unroll
    for (int k = 0; k < 8; ++k) out(j + 16 * (k + 8 * h), x[k]);
  }
  __syncwarp();  // (the scratch is reused by the caller's next transform)
}

// Registers of a forward transform (x[k] = X[j + 16 (k + 8 h)]) -> the input layout of
// the next transform (x[m] = element 16 (2 m + h) + j): lanes j and j + 16 swap four
// values through one shuffle exchange each.
__device__ __forceinline__ void w32_regs_to_input(double2* x, int lane) {
  const int h = lane >> 4;
  double2 snd[4], rcv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) snd[i] = h ? x[2 * i] : x[2 * i + 1];
#pragma unroll
  for (int i = 0; i < 4; ++i) rcv[i] = shfl_xor2(snd[i], 16);
  double2 y[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    if (h == 0) y[m] = m < 4 ? x[2 * m] : rcv[m - 4];
    else y[m] = m < 4 ? rcv[m] : x[2 * m - 7];
  }
#pragma unroll
  for (int m = 0; m < 8; ++m) x[m] = y[m];
}

template <bool INV>
__device__ __forceinline__ void fft256_w32(double2* s, const double2* __restrict__ tw, int lane, bool active) {
  using C = Cfg<256>;
  const int j = lane & 15, h = lane >> 4;
  double2 x[8];
  if (active) {
#pragma unroll
    for (int m = 0; m < 8; ++m) x[m] = s[C::pad(16 * (2 * m + h) + j)];
  }
  fft256_w32_x<INV>(x, s, tw, lane, active);
}

// The 256-point block transforms of nseq sequences (stride ss) with one warp per
// block (fft256_w32): unit = warp index; the caller has exactly nseq * M warps.
template <int N, bool INV>
__device__ __forceinline__ void fft_units_w32(double2* S, int nseq, int ss, const double2* tw, int t) {
  using C = Cfg<N>;
  static_assert(C::L == 256, "one-warp block transforms are 256-point");
  const int u = t >> 5;
  const bool act = u < nseq * C::M;
  const int uu = act ? u : 0;
  fft256_w32<INV>(S + (size_t)(uu / C::M) * ss + (uu % C::M) * C::SSL, tw, t & 31, act);
}

// Radix-M stage of long sequences (Cfg<N>::M > 1; no-op otherwise), all threads
// of the block: forward = DIF butterfly + twiddle w_N^(j r) (natural order in,
// blocks ready for their L-point transforms); inverse = conjugate twiddle +
// inverse butterfly (after the blocks' inverse transforms).  nseq sequences of
// stride ss (complex) from S; tw = the kernel's staged Cfg<N> table.
template <int N, bool INV>
__device__ __forceinline__ void radix_stage(double2* S, int nseq, int ss, const double2* tw, int t, int T) {
  using C = Cfg<N>;
  constexpr int M = C::M, L = C::L;
  if constexpr (M > 1) {
    for (int idx = t; idx < nseq * L; idx += T) {
      const int sq = idx / L, j = idx % L;
      double2* base = S + (size_t)sq * ss + C::pad(j);
      double2 a[M];
#pragma unroll
      for (int b = 0; b < M; ++b) a[b] = base[b * C::SSL];
      if (!INV) Dft<M, false>::run(a);
      radix_twiddle<N, INV>(a, tw, j);
      if (INV) Dft<M, true>::run(a);
#pragma unroll
      for (int b = 0; b < M; ++b) base[b * C::SSL] = a[b];
    }
  }
}

// The block transforms of nseq sequences (stride ss): block (sq, b) = unit
// u = sq M + b, units dealt to the ngr groups in rounds.  With M = 1 this is
// exactly fft_seq on sequence g (round 0), g + ngr, ...  Every thread of the
// block must call it (groups idle in a round still take the __syncwarp's).
template <int N, bool INV>
__device__ __forceinline__ void fft_units(double2* S, int nseq, int ss, const double2* tw, int g, int l, int ngr) {
  using C = Cfg<N>;
  const int nu = nseq * C::M;
  for (int u0 = 0; u0 < nu; u0 += ngr) {
    const int u = u0 + g;
    const bool act = u < nu;
    const int uu = act ? u : 0;
    fft_seq<C::L, INV>(S + (size_t)(uu / C::M) * ss + (uu % C::M) * C::SSL, tw, l, act);
  }
}

}  // namespace fz
}  // namespace pf
