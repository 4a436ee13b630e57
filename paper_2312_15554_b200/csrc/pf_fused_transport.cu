// Fused comparison-medium transport pipeline for cubic power-of-two grids
// (N = 64 ... 512; long sequences as in pf_fused.cu) — reference pkg/src/poreflow/transport.py:225-258 and
// backends/pure.py:71-115.
//
// One iteration streams 25 words + 1 byte per voxel through HBM (the
// canonical cuFFT accounting of SURVEY §8d is 34 words + 4 B):
//
//   PK_T (axis-0 pencils, 2 components): FFT_0 of Y_b and Y_w0; F^ = Y_b +
//         i k0 W0^ (the i k2 / i k1 parts were folded in the X / Y passes);
//         chi^ = F^ / (i b0.k + a0 L), chi^(0) = 0 (pure.py:106-110); Parseval
//         residuals r1^2 = sum w |d chi^|^2 / n and r2^2 = sum w |k|^2 |d chi^|^2 / n
//         (|grad^ chi' - grad^ chi|^2 = |k|^2 |d chi^|^2 since grad^ = i k chi^);
//         chi^ kept (tile-major); IFFT_0 of chi^/n and i k0 chi^/n.
//                                                  reads Y 2 + chi^ 1, writes Y 2 + chi^ 1
//   MI_T (axis-1 pencils, 3 outputs): X(chi), X(d0 chi), X(d1 chi) = IFFT_1 of
//         Y(chi), Y(d0 chi), i k1 Y(chi).          reads 3 (Y(chi) twice), writes 3
//   RS_T (rows): C2R of d0, d1 chi (one complex FFT per row) and d2 chi = i k2 X(chi)
//         (two rows per FFT); polarization w, s from grad chi', u, H (pure.py:71-87
//         with the coefficients of build_coefficients, transport.py:112-121); R2C of
//         (w0 + i w1) and (s + i w2); X_a = X(s) + i k2 X(w2).
//                                                  reads X 3 + u 3 + H, writes X 3
//   F    k_transport_finalize (history row, non-finite / growth guards, convergence)
//   MF_T (axis-1 pencils, 2 outputs): Y_b = FFT_1(X_a) + i k1 FFT_1(X(w1)),
//         Y_w0 = FFT_1(X(w0)).                     reads 3, writes 2
//
// The real fields chi and grad chi are materialised only at the end (cuFFT
// from chi^), exactly as Re ifftn of the spectra the reference inverts.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "pf_fft.cuh"

#ifndef PF_TPK_TMA
#define PF_TPK_TMA 1  // PK_T loads its two component pencils with 3D TMA tensor copies (N = 128/256)
#endif
#ifndef PF_TF_BOTH
#define PF_TF_BOTH 1  // MF_T output 0 loads its two input tiles together (TM::TILE2_OFF)
#endif
#ifndef PF_TRS_SPLIT
#define PF_TRS_SPLIT 1  // RS_T refills its X rows as soon as they are packed (second mbarrier)
#endif
#ifndef PF_TM_PIPE
// persistent transport axis-1 passes (POREFLOW_B200_M_PIPE=0/1 overrides).  Measured at 128^3:
// one solve 15.5 -> 14.95 Gvox-it/s (MI_T / MF_T slower alone: 0.0266 -> 0.0283, 0.0287 -> 0.0317 ms),
// three concurrent load cases 17.7 -> 18.3; off by default (a single solve is the common call)
#define PF_TM_PIPE(N) 0
#endif
#ifndef PF_TPK_TMASTORE
#define PF_TPK_TMASTORE 1  // PK_T stores Y with TMA tensor stores from its boxes (N = 128/256)
#endif
#ifndef PF_TM_TMA
#define PF_TM_TMA 1  // transport axis-1 passes load their tiles with 2D TMA tensor copies (N = 128/256)
#endif
#ifndef PF_TPK_PREFETCH
#define PF_TPK_PREFETCH 1  // previous chi^ loaded into registers under the forward FFT (needs 4 CTAs/SM of regs)
#endif
#ifndef PF_TPK128_MINB
#define PF_TPK128_MINB PF_TPK_MINB
#endif
#ifndef PF_TPK_MINB
#define PF_TPK_MINB 4
#endif
#ifndef PF_TF_MINB
// the same for the forward axis-1 pass, which holds a register stash (measured:
// 3 blocks/SM best at 256^3, 4 at 128^3)
#define PF_TF_MINB (N >= 256 ? 3 : 4)
#endif
#ifndef PF_T_MINB
#define PF_T_MINB 5  // min blocks per SM for the transport spectral / axis-1 passes (smem allows 5)
#endif

namespace pf {
namespace ft {

using fz::Cfg;
using fz::cmul;
using fz::cp16;
using fz::fft_seq;

struct TBufs {
  double2 *X, *Xn;  // X-space [3][N*N][H] + nyq [3][N*N]
  double2 *Y, *Yn;  // Y-space [2][N][N][H] + nyq [2][N][N]
  double2* CH;      // chi^ (PK tile-major, nh)
  double2* G0;      // FFT(initial grad chi), 3 comps tile-major (warm start only) or null
  double2* tw;
  double* part;     // PK_T partials [2][blocks]
};

struct TP {
  const double* kap[3];
  const double* ell[3];
  double pe, eta, a0, ubg, inv_n;
  double g[3], b0v[3];
};

// ------------------------------------------------------------------ PK_T
template <int N>
struct TPK {
  using C = Cfg<N>;
  static constexpr int T = 128;
  static constexpr int NGP = T / C::G;
  static constexpr int CP = NGP / C::M / 2;  // (a long sequence takes M groups)
  static constexpr int NSEQ = 2 * CP;
  static constexpr int NCH = C::H / CP;
  static constexpr int TILES = N * NCH + N / CP;
  static constexpr int MPT = CP * N / T;
  // TMA path (N = 128 / 256, main tiles): the two components' CP x N pencils land
  // 64B-swizzled at the start of the (1 KB-aligned) padded sequence region
  static constexpr bool TMA_OK = (N == 128 || N == 256) && CP * 16 == 64;
  static constexpr size_t REGION = sizeof(double2) * NSEQ * C::SS;
  static constexpr size_t BOX = sizeof(double2) * CP * N;
  static constexpr size_t BYTES = REGION + sizeof(double2) * C::TWN + 1024;
};

template <int N>
__global__ void __launch_bounds__(128, N == 128 ? PF_TPK128_MINB : PF_TPK_MINB) k_tpk(TBufs B, TP P, const Ctrl* __restrict__ ctrl,
                                                         const __grid_constant__ CUtensorMap tmap) {
  using C = Cfg<N>;
  using K = TPK<N>;
  constexpr int H = C::H, SS = C::SS, CP = K::CP, NCH = K::NCH, NSEQ = K::NSEQ, T = K::T;
  pdl_wait();
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char psraw[];
  unsigned char* reg = psraw + ((1024 - (fz::su32(psraw) & 1023)) & 1023);  // 1 KB-aligned
  double2* S = (double2*)reg;
  double2* tw = (double2*)(reg + K::REGION);
  const int t = threadIdx.x, g = t / C::G, l = t % C::G;
  const int tile = blockIdx.x;
  const bool nyq = tile >= N * NCH;
  const int k1 = nyq ? 0 : tile / NCH, ch = nyq ? 0 : tile % NCH;
  const int k1b = nyq ? (tile - N * NCH) * CP : 0;
  auto yoff = [&](int c, int i0, int q) -> size_t {
    return nyq ? (size_t)(c * N + i0) * N + k1b + q : ((size_t)(c * N + i0) * N + k1) * H + ch * CP + q;
  };
  constexpr bool TMA = K::TMA_OK && PF_TPK_TMA;
  const bool tma = TMA && !nyq;
  __shared__ uint64_t mbar;
  if (tma) {
    if (t == 0) {  // two 3D tensor copies: component c's (CP columns x N rows i0) pencil
      fz::mbar_init(&mbar);
      fz::mbar_expect(&mbar, (uint32_t)(2 * K::BOX));
      for (int c = 0; c < 2; ++c)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];" ::"r"(fz::su32(reg + c * K::BOX)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * ch * CP), "r"(k1), "r"(c * N), "r"(fz::su32(&mbar))
            : "memory");
    }
  } else {
    for (int idx = t; idx < 2 * N * CP; idx += T) {
      const int q = idx % CP, i0 = (idx / CP) % N, c = idx / (CP * N);
      const size_t o = yoff(c, i0, q);
      cp16(S + (c * CP + q) * SS + C::sp(i0), nyq ? B.Yn + o : B.Y + o);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int j = t; j < Cfg<N>::TWN; j += T) tw[j] = B.tw[j];
  const bool first = (B.G0 != nullptr) && ctrl->iter == 0;
  const size_t tbase = (size_t)tile * CP * N;
#if PF_TPK_PREFETCH
  double2 chp[K::MPT];  // previous chi^ of this thread's modes, loaded under the forward FFT
#pragma unroll
  for (int j = 0; j < K::MPT; ++j) chp[j] = B.CH[tbase + t + T * j];
#endif
  if (tma) {
    __syncthreads();  // mbarrier initialised
    fz::mbar_wait(&mbar, 0);
    constexpr int A = C::A, BB = C::B;
    const bool act = g < NSEQ;
    const int cc = act ? g / CP : 0, q = act ? g % CP : 0;
    const unsigned char* box = reg + cc * K::BOX;
    double2 x[A > BB ? A : BB];
    if (act && l < BB) {
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) {  // row e = i0, column q: 16B chunk XOR-swizzled by (e / 2) mod 4
        const int e = BB * n1 + l;
        x[n1] = *reinterpret_cast<const double2*>(box + (size_t)e * 64 + ((q ^ ((e >> 1) & 3)) << 4));
      }
    }
    __syncthreads();  // both boxes read before the padded sequences overwrite them
    fz::fft_seq_x<N, false>(x, S + (act ? g : 0) * SS, tw, l, act);
  } else {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if constexpr (C::M > 1) {
      fz::radix_stage<N, false>(S, NSEQ, SS, tw, t, T);
      __syncthreads();
    }
    fz::fft_units<N, false>(S, NSEQ, SS, tw, g, l, K::NGP);
  }
  __syncthreads();
  const size_t nh = (size_t)K::TILES * CP * N;
  double acc[2] = {0.0, 0.0};
#if PF_TPK_PREFETCH
#pragma unroll
#else
#pragma unroll 2
#endif
  for (int j = 0; j < K::MPT; ++j) {
    const int m = t + T * j, q = m / N, k0 = m % N;
    const int kk1 = nyq ? k1b + q : k1, k2 = nyq ? H : ch * CP + q;
    const int idx3[3] = {k0, kk1, k2};
    double kc[3];
    double L = 0.0, bk = 0.0, ksq = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      kc[c] = __ldg(P.kap[c] + idx3[c]);
      L = L + __ldg(P.ell[c] + idx3[c]);
      bk = bk + P.b0v[c] * kc[c];
      ksq = ksq + kc[c] * kc[c];
    }
    const double2 fb = S[q * SS + C::kp(k0)], fw0 = S[(CP + q) * SS + C::kp(k0)];
    const double2 f = cadd(fb, cik(kc[0], fw0));  // F^ = S^ + i k.W^   (pure.py:104-105)
    const bool zero = (k0 | kk1 | k2) == 0;
    const double2 chi = zero ? make_double2(0.0, 0.0) : cdiv_np(f, make_double2(P.a0 * L, bk));
#if PF_TPK_PREFETCH
    const double2 prev = chp[j];
#else
    const double2 prev = B.CH[tbase + m];
#endif
    const double2 dch = csub(chi, prev);
    const double w = (k2 == 0 || k2 == H) ? 1.0 : 2.0;
    acc[0] += w * cabs2(dch);
    if (!first) {
      acc[1] += w * ksq * cabs2(dch);
    } else {  // iteration 1 of a warm start: the given grad chi need not equal i k chi^
      double s2 = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) s2 += cabs2(csub(cik(kc[c], chi), B.G0[c * nh + tbase + m]));
      acc[1] += w * s2;
    }
    B.CH[tbase + m] = chi;
    S[q * SS + C::kp(k0)] = make_double2(chi.x * P.inv_n, chi.y * P.inv_n);
    const double2 g0 = cik(kc[0], chi);
    S[(CP + q) * SS + C::kp(k0)] = make_double2(g0.x * P.inv_n, g0.y * P.inv_n);
  }
  __syncthreads();
  fz::fft_units<N, true>(S, NSEQ, SS, tw, g, l, K::NGP);
  if constexpr (C::M > 1) {
    __syncthreads();
    fz::radix_stage<N, true>(S, NSEQ, SS, tw, t, T);
  }
  __syncthreads();
#if PF_TPK_TMASTORE
  if (tma && C::M == 1) {
    // Y out by TMA tensor stores: component c's results repacked into its 64B-swizzled
    // box (box c overlaps only sequences of components <= c, already consumed), then
    // one thread stores both boxes and waits until they have been read.
    constexpr int PER = CP * N / T;
    for (int c = 0; c < 2; ++c) {
      double2 v[PER];
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int idx = t + T * j, q = idx % CP, i0 = idx / CP;
        v[j] = S[(c * CP + q) * SS + C::sp(i0)];
      }
      __syncthreads();
      unsigned char* box = reg + c * K::BOX;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int idx = t + T * j, q = idx % CP, i0 = idx / CP;
        *reinterpret_cast<double2*>(box + (size_t)i0 * 64 + ((q ^ ((i0 >> 1) & 3)) << 4)) = v[j];
      }
    }
    fz::fence_async_smem();
    __syncthreads();
    if (t == 0) {
      for (int c = 0; c < 2; ++c)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                         reinterpret_cast<uint64_t>(&tmap)),
                     "r"(2 * ch * CP), "r"(k1), "r"(c * N), "r"(fz::su32(reg + c * K::BOX))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  } else
#endif
  for (int idx = t; idx < 2 * N * CP; idx += T) {
    const int q = idx % CP, i0 = (idx / CP) % N, c = idx / (CP * N);
    const size_t o = yoff(c, i0, q);
    const double2 v = S[(c * CP + q) * SS + C::sp(i0)];
    if (nyq) B.Yn[o] = v; else B.Y[o] = v;
  }
  block_sum<2>(acc);
  if (t == 0) {
    B.part[blockIdx.x] = acc[0];
    B.part[gridDim.x + blockIdx.x] = acc[1];
  }
#if PF_TPK_TMASTORE
  if (tma && C::M == 1 && t == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
}

// ------------------------------------------------------------------ MI_T / MF_T
template <int N>
struct TM {
  using C = Cfg<N>;
  static constexpr int T = 128;
  static constexpr int NGM = T / C::G;
  static constexpr int CM = NGM / C::M;
  static constexpr int NCH = C::H / CM;
  static constexpr int TPC = N * NCH + N / CM;  // tiles per output component
  static constexpr size_t SEQ = sizeof(double2) * CM * C::SS;
  // one sequence set: Y_b = FFT(X0) + i k1 FFT(X2) runs its two transforms one
  // after the other, stashing i k1 FFT(X2) in registers (IPT items per thread)
  // TMA path (N = 128 / 256, main tiles): the CM x N tile lands 128B-swizzled in a
  // 1 KB-aligned region the padded sequences then reuse
  static constexpr bool TMA_OK = (N == 128 || N == 256) && CM * 16 == 128;
  static constexpr size_t TILE = sizeof(double2) * CM * N;
  static constexpr size_t REGION = SEQ > TILE ? SEQ : TILE;
  static constexpr size_t BYTES = sizeof(double2) * C::TWN + REGION + 1024;
  // MF_T output 0 (Y_b) stages its second input tile (X0) beside the first from the
  // start, so both loads are in flight together (1 KB-aligned, after the twiddles)
  static constexpr size_t TILE2_OFF = ((REGION + sizeof(double2) * C::TWN + 1023) / 1024) * 1024;
  static constexpr size_t BYTES_FWD = TMA_OK ? TILE2_OFF + TILE + 1024 : BYTES;
  static constexpr int IPT = N * CM / T;
};

// INV (MI_T): outputs oc = 0 X(chi) <- Y0; 1 X(d0 chi) <- Y1; 2 X(d1 chi) <- i k1 Y0.
// FWD (MF_T): outputs oc = 0 Y_b <- FFT(X0) + i k1 FFT(X2); 1 Y_w0 <- FFT(X1).
template <int N, bool INV>
__global__ void __launch_bounds__(128, INV ? PF_T_MINB : PF_TF_MINB) k_taxis(TBufs B, const double* __restrict__ kap1, const Ctrl* __restrict__ ctrl,
                                                                          const __grid_constant__ CUtensorMap tmap, int nyq_only) {
  using C = Cfg<N>;
  using K = TM<N>;
  constexpr int H = C::H, SS = C::SS, CM = K::CM, NCH = K::NCH, T = K::T;
  pdl_wait();
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char msraw[];
  unsigned char* reg = msraw + ((1024 - (fz::su32(msraw) & 1023)) & 1023);  // 1 KB-aligned
  double2* S = (double2*)reg;
  double2* tw = (double2*)(reg + K::REGION);
  const int t = threadIdx.x, g = t / C::G, l = t % C::G;
  // nyq_only (beside k_taxis_pipe): block -> (output, Nyquist tile)
  const int oc = nyq_only ? blockIdx.x / (N / CM) : blockIdx.x / K::TPC;
  const int tile = nyq_only ? N * NCH + blockIdx.x % (N / CM) : blockIdx.x % K::TPC;
  const bool nyq = tile >= N * NCH;
  const int i0 = nyq ? 0 : tile / NCH, ch = nyq ? 0 : tile % NCH;
  const int i0b = nyq ? (tile - N * NCH) * CM : 0;
  // X-space plane stride (per component) and Y-space component stride are both N*N*H (+N*N nyq)
  auto off_of = [&](int c, int e, int q) -> size_t {
    return nyq ? (size_t)(c * N + i0b + q) * N + e : ((size_t)(c * N + i0) * N + e) * H + ch * CM + q;
  };
  const int cin = oc == 1 ? 1 : 0;
  const bool two = !INV && oc == 0;  // Y_b needs X0 and X2
  static_assert(K::IPT * K::T == N * CM, "whole items per thread");
  for (int j = t; j < Cfg<N>::TWN; j += T) tw[j] = B.tw[j];
  auto stage = [&](int c) {  // one input component of the tile -> S (LDGSTS)
    for (int idx = t; idx < N * CM; idx += T) {
      const int q = nyq ? idx / N : idx % CM, e = nyq ? idx % N : idx / CM;
      const size_t o = off_of(c, e, q);
      if (INV) cp16(S + q * SS + C::kp(e), nyq ? B.Yn + o : B.Y + o);
      else cp16(S + q * SS + C::sp(e), nyq ? B.Xn + o : B.X + o);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  };
  constexpr bool TMA = K::TMA_OK && PF_TM_TMA;
  const bool tma = TMA && !nyq;
  __shared__ uint64_t mbar;
  uint32_t par = 0;
  if (tma && t == 0) fz::mbar_init(&mbar);
  // one component's tile -> registers (column g) -> the rest of the FFT, via TMA
  auto tma_fft = [&](int c, bool ik1) {
    if (t == 0) {
      fz::mbar_expect(&mbar, (uint32_t)K::TILE);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              fz::su32(reg)),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * ch * CM), "r"((c * N + i0) * N), "r"(fz::su32(&mbar))
          : "memory");
    }
    __syncthreads();
    fz::mbar_wait(&mbar, par);
    par ^= 1u;
    constexpr int A = C::A, BB = C::B;
    double2 x[A > BB ? A : BB];
    if (l < BB) {
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) {
        const int e = BB * n1 + l;
        x[n1] = *reinterpret_cast<const double2*>(reg + (size_t)e * 128 + ((g ^ (e & 7)) << 4));
        if (ik1) x[n1] = cik(__ldg(kap1 + e), x[n1]);
      }
    }
    __syncthreads();  // the tile is read before the padded sequences overwrite it
    if (INV) fz::fft_seq_x<N, true>(x, S + g * SS, tw, l, true);
    else fz::fft_seq_x<N, false>(x, S + g * SS, tw, l, true);
    __syncthreads();
  };
  double2 v2[K::IPT];
  const bool both = PF_TF_BOTH && two && tma;  // X2 and X0 loaded together
  if (both) {
    unsigned char* reg2 = reg + K::TILE2_OFF;
    if (t == 0) {
      fz::mbar_expect(&mbar, (uint32_t)(2 * K::TILE));
      for (int k = 0; k < 2; ++k)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                fz::su32(k ? reg2 : reg)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * ch * CM), "r"(((k ? 0 : 2) * N + i0) * N),
            "r"(fz::su32(&mbar))
            : "memory");
    }
    __syncthreads();
    fz::mbar_wait(&mbar, 0);
    constexpr int A = C::A, BB = C::B;
    double2 x[A > BB ? A : BB];
    for (int k = 0; k < 2; ++k) {  // i k1 FFT(X2) into registers, then FFT(X0) into S
      const unsigned char* src = k ? reg2 : reg;
      if (l < BB) {
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) {
          const int e = BB * n1 + l;
          x[n1] = *reinterpret_cast<const double2*>(src + (size_t)e * 128 + ((g ^ (e & 7)) << 4));
        }
      }
      __syncthreads();  // (k = 0: the tile is read before the padded sequences overwrite it)
      fz::fft_seq_x<N, false>(x, S + g * SS, tw, l, true);
      __syncthreads();
      if (k == 0) {
#pragma unroll
        for (int j = 0; j < K::IPT; ++j) {
          const int idx = t + T * j;
          const int q = idx % CM, e = idx / CM;
          v2[j] = cik(__ldg(kap1 + e), S[q * SS + C::kp(e)]);
        }
      }
    }
  } else if (two) {  // i k1 FFT(X2) first, kept in registers
    if (tma) {
      tma_fft(2, false);
    } else {
      stage(2);
      if constexpr (C::M > 1) {
        fz::radix_stage<N, false>(S, CM, SS, tw, t, T);
        __syncthreads();
      }
      fz::fft_units<N, false>(S, CM, SS, tw, g, l, K::NGM);
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < K::IPT; ++j) {
      const int idx = t + T * j;
      const int q = nyq ? idx / N : idx % CM, e = nyq ? idx % N : idx / CM;
      v2[j] = cik(__ldg(kap1 + e), S[q * SS + C::kp(e)]);
    }
    __syncthreads();
  }
  if (both) {
    // (X0's transform is in S)
  } else if (tma) {
    tma_fft(cin, INV && oc == 2);
  } else {
  stage(cin);
  if (INV && oc == 2) {  // i k1 Y(chi) before the inverse axis-1 transform
    for (int idx = t; idx < N * CM; idx += T) {
      const int q = idx / N, e = idx % N;
      double2* p = S + q * SS + C::kp(e);
      *p = cik(__ldg(kap1 + e), *p);
    }
    __syncthreads();
  }
  if constexpr (C::M > 1) {
    if (!INV) {
      fz::radix_stage<N, false>(S, CM, SS, tw, t, T);
      __syncthreads();
    }
    fz::fft_units<N, INV>(S, CM, SS, tw, g, l, K::NGM);
    if (INV) {
      __syncthreads();
      fz::radix_stage<N, true>(S, CM, SS, tw, t, T);
    }
  } else {
    fft_seq<N, INV>(S + g * SS, tw, l, true);
  }
  __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < K::IPT; ++j) {
    const int idx = t + T * j;
    const int q = nyq ? idx / N : idx % CM, e = nyq ? idx % N : idx / CM;
    double2 v = S[q * SS + (INV ? C::sp(e) : C::kp(e))];
    if (two) v = cadd(v, v2[j]);
    const size_t o = off_of(oc, e, q);
    if (INV) {
      if (nyq) B.Xn[o] = v; else B.X[o] = v;
    } else {
      if (nyq) B.Yn[o] = v; else B.Y[o] = v;
    }
  }
}

// ------------------------------------------------------------------ MI_T / MF_T, persistent pipelined
// N = 128 / 256 main tiles (the Nyquist tiles stay on k_taxis with nyq_only): one CTA
// per slot walks the (output, tile) units with a two-stage TMA ring, as the Stokes
// k_m1_pipe — at 128^3 the per-CTA fixed costs of the non-persistent passes show.
// A unit's stage holds its input tile(s): MI_T one (Y0, Y1 or Y0 for i k1 Y0), MF_T
// output 0 two (X2, X0: Y_b = FFT(X0) + i k1 FFT(X2)), output 1 one (X1).
template <int N, bool INV>
struct TMP {
  using C = Cfg<N>;
  static constexpr int T = TM<N>::T, CM = TM<N>::CM, NCH = TM<N>::NCH;
  static constexpr size_t TILE = TM<N>::TILE;
  static constexpr int TPS = INV ? 1 : 2;  // tiles per stage
  static constexpr size_t STAGE = TPS * TILE;
  static constexpr int STAGES = 2;
  static constexpr size_t SEQ = TM<N>::SEQ;
  static constexpr size_t BYTES = 1024 + STAGES * STAGE + SEQ + sizeof(double2) * C::TWN;
  static constexpr int NOUT = INV ? 3 : 2;
  static constexpr int UNITS = NOUT * N * NCH;
  static_assert(C::M == 1 && CM * 16 == 128 && TILE % 1024 == 0, "pipelined transport axis-1 pass: N <= 256");
};

template <int N, bool INV>
__global__ void __launch_bounds__(TMP<N, INV>::T, 1) k_taxis_pipe(TBufs B, const double* __restrict__ kap1,
                                                                 const Ctrl* __restrict__ ctrl,
                                                                 const __grid_constant__ CUtensorMap tmap) {
  using C = Cfg<N>;
  using K = TMP<N, INV>;
  constexpr int H = C::H, SS = C::SS, CM = K::CM, NCH = K::NCH, T = K::T, NU = K::UNITS;
  constexpr int IPT = TM<N>::IPT;
  pdl_wait();
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char tpraw[];
  unsigned char* base = tpraw + ((1024 - (fz::su32(tpraw) & 1023)) & 1023);
  double2* S = (double2*)(base + K::STAGES * K::STAGE);
  double2* tw = (double2*)(base + K::STAGES * K::STAGE + K::SEQ);
  __shared__ uint64_t full[K::STAGES];
  const int t = threadIdx.x, g = t / C::G, l = t % C::G;

  auto ins = [&](int oc, int k) {  // input component of tile slot k of output oc
    if (INV) return oc == 1 ? 1 : 0;
    return oc == 0 ? (k == 0 ? 2 : 0) : 1;
  };
  auto issue = [&](int u, int s) {
    const int oc = u / (N * NCH), r = u % (N * NCH), i0 = r / NCH, ch = r % NCH;
    const int nt = (!INV && oc == 0) ? 2 : 1;
    unsigned char* dst = base + (size_t)s * K::STAGE;
    fz::fence_async_smem();
    fz::mbar_expect(&full[s], (uint32_t)(nt * K::TILE));
    for (int k = 0; k < nt; ++k)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              fz::su32(dst + k * K::TILE)),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * ch * CM), "r"((ins(oc, k) * N + i0) * N), "r"(fz::su32(&full[s]))
          : "memory");
  };
  if (t == 0) {
    for (int s = 0; s < K::STAGES; ++s) fz::mbar_init(&full[s]);
    for (int s = 0; s < K::STAGES; ++s)
      if ((int)blockIdx.x + s * (int)gridDim.x < NU) issue(blockIdx.x + s * gridDim.x, s);
  }
  for (int j = t; j < C::TWN; j += T) tw[j] = B.tw[j];
  __syncthreads();
  constexpr int A = C::A, BB = C::B;
  int it = 0;
  for (int u = blockIdx.x; u < NU; u += gridDim.x, ++it) {
    const int s = it & 1;
    const int oc = u / (N * NCH), r = u % (N * NCH), i0 = r / NCH, ch = r % NCH;
    const unsigned char* st = base + (size_t)s * K::STAGE;
    const bool two = !INV && oc == 0;
    fz::mbar_wait(&full[s], (it >> 1) & 1);
    double2 x[A > BB ? A : BB];
    auto load = [&](int k) {  // tile slot k, column g -> x
      if (l < BB) {
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) {
          const int e = BB * n1 + l;
          x[n1] = *reinterpret_cast<const double2*>(st + k * K::TILE + (size_t)e * 128 + ((g ^ (e & 7)) << 4));
          if (INV && oc == 2) x[n1] = cik(__ldg(kap1 + e), x[n1]);
        }
      }
    };
    double2 v2[IPT];
    load(0);
    if (two) {  // i k1 FFT(X2) (slot 0), kept in registers, then FFT(X0) (slot 1)
      fz::fft_seq_x<N, false>(x, S + g * SS, tw, l, true);
      __syncthreads();
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        const int idx = t + T * j, q = idx % CM, e = idx / CM;
        v2[j] = cik(__ldg(kap1 + e), S[q * SS + C::kp(e)]);
      }
      load(1);
    }
    __syncthreads();  // stage s read (and S free): refill the stage two grid strides ahead
    if (t == 0 && u + K::STAGES * (int)gridDim.x < NU) issue(u + K::STAGES * gridDim.x, s);
    if (two) fz::fft_seq_x<N, false>(x, S + g * SS, tw, l, true);
    else fz::fft_seq_x<N, INV>(x, S + g * SS, tw, l, true);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const int idx = t + T * j, q = idx % CM, e = idx / CM;
      double2 v = S[q * SS + (INV ? C::sp(e) : C::kp(e))];
      if (two) v = cadd(v, v2[j]);
      const size_t o = ((size_t)(oc * N + i0) * N + e) * H + ch * CM + q;
      if (INV) B.X[o] = v; else B.Y[o] = v;
    }
    __syncthreads();  // S is rewritten by the next unit
  }
}

// ------------------------------------------------------------------ RS_T
#ifndef PF_TRS_UREG
#define PF_TRS_UREG 1
#endif
template <int N>
struct TRS {
  using C = Cfg<N>;
#ifndef PF_TRS_R256
#define PF_TRS_R256 2
#endif
  static constexpr int R = N > 256 ? 2 : (N == 256 ? PF_TRS_R256 : 512 / N);  // rows per tile
  static constexpr int NSF = 2 * R;          // forward sequences: (w0 + i w1), (s + i w2) per row
  static constexpr int NSI = R + R / 2;      // inverse: (d0 + i d1) per row, (d2, d2) per row pair
  static constexpr int T = NSF * C::M * C::G;  // one group per forward block transform
  static constexpr int V = R * N;
  static constexpr int VPT = V / T;
  static constexpr size_t TW = sizeof(double2) * C::TWN;
  static constexpr size_t SI = sizeof(double2) * NSI * C::SS;
  static constexpr size_t SF = sizeof(double2) * NSF * C::SS;
  static constexpr size_t XM = sizeof(double2) * 3 * R * C::H;   // X comps 0..2, R rows each
  static constexpr size_t XN = sizeof(double2) * 3 * R;
  static constexpr size_t UB = sizeof(double) * 3 * V;
  static constexpr size_t HB = V;
  // the forward sequences overwrite the inverse ones (the local step reads its
  // gradients into registers first), so one buffer of max(SI, SF) bytes
  static constexpr size_t SQ = SI > SF ? SI : SF;
  // UREG: u and the indicator go straight from global memory into registers at the
  // start of each tile (consumed after the inverse transforms), so only the X rows
  // are staged: less shared memory per CTA, more CTAs per SM
  // (measured: 256^3 RS_T 0.338 -> 0.324 ms with 2-row tiles, 0.334 with 4-row ones;
  // 128^3 0.058 -> 0.066, so staged there)
  static constexpr bool UREG = PF_TRS_UREG && N == 256;
  static constexpr size_t BYTES = TW + SQ + XM + XN + (UREG ? 0 : UB + HB);
#ifdef PF_TRS_MINB
  static constexpr int MINB = PF_TRS_MINB;
#else
  static constexpr int MINB = T <= 64 ? 4 : 3;  // register cap that keeps the smem-allowed blocks
#endif
  static constexpr uint32_t TX = (uint32_t)(XM + XN + UB + HB);
};

// part: 0 = every staged input; 1 = the X rows only; 2 = u and the indicator only (the
// X rows are packed into the inverse sequences one step before u / H are consumed).
template <int N>
__device__ __forceinline__ void trs_issue(int tile, const TBufs& B, const double* u, const uint8_t* Hs, double2* sx,
                                          double2* sxn, double* su, uint8_t* sh, uint64_t* mbar, int part = 0) {
  using K = TRS<N>;
  using C = Cfg<N>;
  constexpr int R = K::R, H = C::H;
  const int64_t row0 = (int64_t)tile * R;
  const int64_t n = (int64_t)N * N * N, NN = (int64_t)N * N;
  fz::fence_async_smem();
  fz::mbar_expect(mbar, part == 0 ? K::TX : (part == 1 ? (uint32_t)(K::XM + K::XN) : (uint32_t)(K::UB + K::HB)));
  for (int c = 0; c < 3; ++c) {
    if (part != 2) {
      fz::bulk_load(sx + c * R * H, B.X + (c * NN + row0) * H, sizeof(double2) * R * H, mbar);
      fz::bulk_load(sxn + c * R, B.Xn + c * NN + row0, sizeof(double2) * R, mbar);
    }
    if (part != 1) fz::bulk_load(su + c * K::V, u + c * n + row0 * N, sizeof(double) * K::V, mbar);
  }
  if (part != 1) fz::bulk_load(sh, Hs + row0 * N, (uint32_t)K::HB, mbar);
}

template <int N>
__global__ void __launch_bounds__(TRS<N>::T, TRS<N>::MINB) k_trs(TBufs B, TP P, const double* __restrict__ u,
                                                   const uint8_t* __restrict__ Hs, const Ctrl* __restrict__ ctrl) {
  using C = Cfg<N>;
  using K = TRS<N>;
  constexpr int H = C::H, SS = C::SS, R = K::R, T = K::T, V = K::V;
  constexpr int NT = N * N / R;
  pdl_wait();
  if (ctrl->done) return;
  extern __shared__ __align__(128) unsigned char sraw[];
  __shared__ uint64_t mbar, mbx;  // mbx: the X rows (PF_TRS_SPLIT)
  constexpr bool SPLIT = PF_TRS_SPLIT;
  double2* tw = (double2*)sraw;
  double2* SIq = (double2*)(sraw + K::TW);
  double2* SFq = SIq;  // aliased (see TRS::BYTES)
  double2* sx = (double2*)(sraw + K::TW + K::SQ);
  double2* sxn = (double2*)(sraw + K::TW + K::SQ + K::XM);
  double* su = (double*)(sraw + K::TW + K::SQ + K::XM + K::XN);
  uint8_t* sh = (uint8_t*)(sraw + K::TW + K::SQ + K::XM + K::XN + K::UB);
  const int t = threadIdx.x, g = t / C::G, l = t % C::G;
  for (int j = t; j < Cfg<N>::TWN; j += T) tw[j] = B.tw[j];
  const double* kap2 = P.kap[2];
  if (t == 0) {
    fz::mbar_init(&mbar);
    fz::mbar_init(&mbx);
    if ((int)blockIdx.x < NT) {
      if (SPLIT || K::UREG) {
        trs_issue<N>(blockIdx.x, B, u, Hs, sx, sxn, su, sh, &mbx, 1);
        if (!K::UREG) trs_issue<N>(blockIdx.x, B, u, Hs, sx, sxn, su, sh, &mbar, 2);
      } else {
        trs_issue<N>(blockIdx.x, B, u, Hs, sx, sxn, su, sh, &mbar);
      }
    }
  }
  __syncthreads();
  const double pe = P.pe, eta = P.eta, a0 = P.a0, ubg = P.ubg;
  const int64_t nvox = (int64_t)N * N * N;
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < NT; tile += gridDim.x, phase ^= 1u) {
    const int64_t row0 = (int64_t)tile * R;
    double ur[K::UREG ? K::VPT : 1][3];
    double hr[K::UREG ? K::VPT : 1];
    if constexpr (K::UREG) {  // this tile's u and H, in flight under the packing and inverse transforms
#pragma unroll
      for (int j = 0; j < K::VPT; ++j) {
        const int64_t x = row0 * N + t + T * j;
#pragma unroll
        for (int c = 0; c < 3; ++c) ur[j][c] = __ldcs(u + c * nvox + x);
        hr[j] = (double)__ldcs(Hs + x);
      }
    }
    if (SPLIT || K::UREG) fz::mbar_wait(&mbx, phase);
    else fz::mbar_wait(&mbar, phase);
    // (1) inverse sequences: per row r  Z = X(d0) + i X(d1);  per pair p  Z = X(d2)_{2p} + i X(d2)_{2p+1}
    for (int idx = t; idx < (R + R / 2) * (H + 1); idx += T) {
      const int sq = idx / (H + 1), k = idx % (H + 1);
      double2 xa, xb;
      if (sq < R) {
        xa = k < H ? sx[(1 * R + sq) * H + k] : sxn[1 * R + sq];
        xb = k < H ? sx[(2 * R + sq) * H + k] : sxn[2 * R + sq];
      } else {
        const int p = sq - R;
        const double kk = __ldg(kap2 + k);  // X(d2 chi) = i k2 X(chi); Nyquist k2 -> 0
        xa = cik(kk, k < H ? sx[(2 * p) * H + k] : sxn[2 * p]);
        xb = cik(kk, k < H ? sx[(2 * p + 1) * H + k] : sxn[2 * p + 1]);
      }
      double2* sp = SIq + sq * SS;
      if (k == 0 || k == H) {
        sp[C::kp(k)] = make_double2(xa.x, xb.x);  // C2R keeps the real part of self-conjugate modes
      } else {
        sp[C::kp(k)] = make_double2(xa.x - xb.y, xa.y + xb.x);
        sp[C::kp(N - k)] = make_double2(xa.x + xb.y, xb.x - xa.y);
      }
    }
    __syncthreads();
    if ((SPLIT || K::UREG) && t == 0 && tile + (int)gridDim.x < NT)  // the X rows are packed: refill them now
      trs_issue<N>(tile + gridDim.x, B, u, Hs, sx, sxn, su, sh, &mbx, 1);
    fz::fft_units<N, true>(SIq, K::NSI, SS, tw, g, l, T / C::G);
    if constexpr (C::M > 1) {
      __syncthreads();
      fz::radix_stage<N, true>(SIq, K::NSI, SS, tw, t, T);
    }
    __syncthreads();
    if (SPLIT && !K::UREG) fz::mbar_wait(&mbar, phase);  // u and H of this tile
    // (2) polarization (pure.py:71-87) with A, B, F from H and u (transport.py:112-121);
    // gradients to registers first: the forward sequences overwrite the inverse ones
    double gv[K::VPT][3];
#pragma unroll
    for (int j = 0; j < K::VPT; ++j) {
      const int v = t + T * j, row = v / N, col = v % N;
      const double2 z01 = SIq[row * SS + C::sp(col)];
      gv[j][0] = z01.x;
      gv[j][1] = z01.y;
      gv[j][2] = reinterpret_cast<const double*>(SIq + (R + (row >> 1)) * SS + C::sp(col))[row & 1];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < K::VPT; ++j) {
      const int v = t + T * j, row = v / N, col = v % N;
      const double* gr = gv[j];
      const double h = K::UREG ? hr[j] : (double)sh[v];
      const double pore = 1.0 - h;
      const double contrast = (pore + eta * h) - a0;
      const double pep = pe * pore;
      double s = pep * ubg;
      double w[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double tg = gr[c] + P.g[c];
        w[c] = contrast * tg;
        s = s - (pep * (K::UREG ? ur[j][c] : su[c * V + v]) - P.b0v[c]) * tg;
      }
      SFq[(2 * row) * SS + C::sp(col)] = make_double2(w[0], w[1]);
      SFq[(2 * row + 1) * SS + C::sp(col)] = make_double2(s, w[2]);
    }
    __syncthreads();
    if (!K::UREG && t == 0 && tile + (int)gridDim.x < NT)
      trs_issue<N>(tile + gridDim.x, B, u, Hs, sx, sxn, su, sh, &mbar, SPLIT ? 2 : 0);
    if constexpr (C::M > 1) {
      fz::radix_stage<N, false>(SFq, K::NSF, SS, tw, t, T);
      __syncthreads();
    }
    fz::fft_units<N, false>(SFq, K::NSF, SS, tw, g, l, T / C::G);
    __syncthreads();
    // (3) separate; X_a = X(s) + i k2 X(w2); store X comps 0 (X_a), 1 (X(w0)), 2 (X(w1))
    const int64_t NN = (int64_t)N * N;
    for (int idx = t; idx < R * (H + 1); idx += T) {
      const int r = idx / (H + 1), k = idx % (H + 1);
      const double2* s1 = SFq + (2 * r) * SS;
      const double2* s2 = SFq + (2 * r + 1) * SS;
      const double2 a1 = s1[C::kp(k)], m1 = s1[C::kp((N - k) & (N - 1))];
      const double2 a2 = s2[C::kp(k)], m2 = s2[C::kp((N - k) & (N - 1))];
      const double2 xw0 = make_double2(0.5 * (a1.x + m1.x), 0.5 * (a1.y - m1.y));
      const double2 xw1 = make_double2(0.5 * (a1.y + m1.y), -0.5 * (a1.x - m1.x));
      const double2 xs = make_double2(0.5 * (a2.x + m2.x), 0.5 * (a2.y - m2.y));
      const double2 xw2 = make_double2(0.5 * (a2.y + m2.y), -0.5 * (a2.x - m2.x));
      const double2 xa = cadd(xs, cik(__ldg(kap2 + k), xw2));
      if (k < H) {
        B.X[(0 * NN + row0 + r) * H + k] = xa;
        B.X[(1 * NN + row0 + r) * H + k] = xw0;
        B.X[(2 * NN + row0 + r) * H + k] = xw1;
      } else {
        B.Xn[0 * NN + row0 + r] = xa;
        B.Xn[1 * NN + row0 + r] = xw0;
        B.Xn[2 * NN + row0 + r] = xw1;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ setup / teardown helpers
// natural [4][N][N][N/2+1] 2D-transformed (w0, w1, w2, s) -> Y_b = S + i k2 W2 + i k1 W1, Y_w0 = W0
template <int N>
__global__ void k_tinit_y(const double2* __restrict__ nat, TBufs B, const double* __restrict__ kap1,
                          const double* __restrict__ kap2) {
  constexpr int H = N / 2, W = H + 1;
  const int64_t rows = (int64_t)N * N, per = rows * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / W;
    const int k2 = (int)(i % W), kk1 = (int)(r % N);
    const double2 w0 = nat[i], w1 = nat[per + i], w2 = nat[2 * per + i], s = nat[3 * per + i];
    const double2 yb = cadd(cadd(s, cik(kap2[k2], w2)), cik(kap1[kk1], w1));
    if (k2 < H) {
      B.Y[r * H + k2] = yb;
      B.Y[(rows + r) * H + k2] = w0;
    } else {
      B.Yn[r] = yb;
      B.Yn[rows + r] = w0;
    }
  }
}

// tile-major chi^ -> natural [ncomp][N][N][N/2+1] of chi^/n (comp 0) and i k_c chi^/n (comps 1..3)
template <int N>
__global__ void k_tout(const double2* __restrict__ CH, double2* __restrict__ nat, TP P, int with_grad) {
  using K = TPK<N>;
  constexpr int H = N / 2, W = H + 1, CP = K::CP;
  const int64_t per = (int64_t)N * N * W;
  const int64_t total = (int64_t)K::TILES * CP * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int tile = (int)(i / (CP * N));
    const int q = (int)((i / N) % CP), k0 = (int)(i % N);
    int k1, k2;
    if (tile < N * K::NCH) {
      k1 = tile / K::NCH;
      k2 = (tile % K::NCH) * CP + q;
    } else {
      k1 = (tile - N * K::NCH) * CP + q;
      k2 = H;
    }
    const int64_t o = ((int64_t)k0 * N + k1) * W + k2;
    const double2 c = make_double2(CH[i].x * P.inv_n, CH[i].y * P.inv_n);
    nat[o] = c;
    if (with_grad) {
      const int idx3[3] = {k0, k1, k2};
      for (int a = 0; a < 3; ++a) nat[(a + 1) * per + o] = cik(P.kap[a][idx3[a]], c);
    }
  }
}

template <int N>
__global__ void k_to_tm(const double2* __restrict__ nat, double2* __restrict__ tm, int ncomp) {
  using K = TPK<N>;
  constexpr int H = N / 2, W = H + 1, CP = K::CP;
  const int64_t per = (int64_t)N * N * W;
  const int64_t total = (int64_t)K::TILES * CP * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int tile = (int)(i / (CP * N));
    const int q = (int)((i / N) % CP), k0 = (int)(i % N);
    int k1, k2;
    if (tile < N * K::NCH) {
      k1 = tile / K::NCH;
      k2 = (tile % K::NCH) * CP + q;
    } else {
      k1 = (tile - N * K::NCH) * CP + q;
      k2 = H;
    }
    const int64_t o = ((int64_t)k0 * N + k1) * W + k2;
    for (int c = 0; c < ncomp; ++c) tm[c * total + i] = nat[c * per + o];
  }
}

}  // namespace ft

// ------------------------------------------------------------------ host
struct FusedTPlan {
  int N = 0;
  ft::TBufs b{};
  void* mem = nullptr;
  double2* g0mem = nullptr;
  cufftHandle plan2d = 0;
  int nb_trs = kSMs;  // persistent RS grid: one wave of resident blocks (occupancy API)
  CUtensorMap tm_y{}, tm_x{};  // axis-1 TMA maps of Y (2 components) and X (3)
  CUtensorMap tm_pk{};         // PK_T pencil map of Y
  int m_pipe = 0, nb_tmi = kSMs, nb_tmf = kSMs;  // persistent transport axis-1 passes (k_taxis_pipe)
};

static FusedTPlan* ftp(pf_plan* p) { return reinterpret_cast<FusedTPlan*>(p->tfused); }

template <int N>
static int tset_attrs(FusedTPlan* f) {
  PF_CK_CUDA(smem_attr(ft::k_tpk<N>, (int)ft::TPK<N>::BYTES));
  PF_CK_CUDA(smem_attr(ft::k_taxis<N, true>, (int)ft::TM<N>::BYTES));
  PF_CK_CUDA(smem_attr(ft::k_taxis<N, false>, (int)ft::TM<N>::BYTES_FWD));
  PF_CK_CUDA(smem_attr(ft::k_trs<N>, (int)ft::TRS<N>::BYTES));
  int o = 0;
  PF_CK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ft::k_trs<N>, ft::TRS<N>::T, ft::TRS<N>::BYTES));
  f->nb_trs = (o < 1 ? 1 : o) * kSMs;
  if constexpr (N == 128 || N == 256) {
    PF_CK_CUDA(smem_attr(ft::k_taxis_pipe<N, true>, ft::TMP<N, true>::BYTES));
    PF_CK_CUDA(smem_attr(ft::k_taxis_pipe<N, false>, ft::TMP<N, false>::BYTES));
    int oi = 0, of = 0;
    PF_CK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oi, ft::k_taxis_pipe<N, true>, ft::TMP<N, true>::T,
                                                             ft::TMP<N, true>::BYTES));
    PF_CK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&of, ft::k_taxis_pipe<N, false>, ft::TMP<N, false>::T,
                                                             ft::TMP<N, false>::BYTES));
    f->nb_tmi = (oi < 1 ? 1 : oi) * kSMs;
    f->nb_tmf = (of < 1 ? 1 : of) * kSMs;
    const char* e = getenv("POREFLOW_B200_M_PIPE");
    f->m_pipe = e ? e[0] == '1' : PF_TM_PIPE(N);
  }
  return PF_OK;
}

static int tfused_ensure(pf_plan* p) {
  if (p->tfused) return PF_OK;
  const int N = p->g.n[0];
  FusedTPlan* f = new FusedTPlan();
  f->N = N;
  const size_t H = N / 2, NN = (size_t)N * N, nh = NN * (H + 1);
  const int nb_pk = (N == 64) ? ft::TPK<64>::TILES : (N == 128 ? ft::TPK<128>::TILES : (N == 256 ? ft::TPK<256>::TILES : ft::TPK<512>::TILES));
  const size_t elems = 3 * NN * H + 3 * NN + 2 * NN * H + 2 * NN + nh + N;
  const size_t bytes = elems * sizeof(double2) + 2 * (size_t)nb_pk * sizeof(double);
  PF_CK_CUDA(cudaMalloc(&f->mem, bytes));
  double2* m = (double2*)f->mem;
  auto take = [&](size_t k) {
    double2* r = m;
    m += k;
    return r;
  };
  f->b.X = take(3 * NN * H);
  f->b.Y = take(2 * NN * H);
  f->b.CH = take(nh);
  f->b.Xn = take(3 * NN);
  f->b.Yn = take(2 * NN);
  f->b.tw = take(N);
  f->b.part = (double*)m;
  std::vector<double2> tw(N == 64 ? fz::Cfg<64>::TWN : (N == 128 ? fz::Cfg<128>::TWN : (N == 256 ? fz::Cfg<256>::TWN : fz::Cfg<512>::TWN)));
  switch (N) {
    case 64: fz::pass1_twiddles<64>(tw.data()); break;
    case 128: fz::pass1_twiddles<128>(tw.data()); break;
    case 256: fz::pass1_twiddles<256>(tw.data()); break;
    default: fz::pass1_twiddles<512>(tw.data()); break;
  }
  PF_CK_CUDA(cudaMemcpy(f->b.tw, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice));
  if (N == 128 || N == 256) {
    const int cm = N == 128 ? ft::TM<128>::CM : ft::TM<256>::CM;
    PF_CK(encode_axis1_map(&f->tm_y, f->b.Y, N, cm, 2));
    PF_CK(encode_axis1_map(&f->tm_x, f->b.X, N, cm, 3));
    PF_CK(encode_pk_map(&f->tm_pk, f->b.Y, N, N == 128 ? ft::TPK<128>::CP : ft::TPK<256>::CP, 2));
  }
  size_t ws = 0;
  long long dims2[2] = {N, N};
  PF_CK_FFT(cufftCreate(&f->plan2d));
  PF_CK_FFT(cufftSetAutoAllocation(f->plan2d, 0));
  PF_CK_FFT(cufftMakePlanMany64(f->plan2d, 2, dims2, nullptr, 1, (long long)NN, nullptr, 1, (long long)N * (H + 1),
                                CUFFT_D2Z, 4LL * N, &ws));
  if (ws > p->fft_work_bytes) {
    PF_CK_CUDA(cudaStreamSynchronize(p->work));
    if (p->fft_work) PF_CK_CUDA(cudaFree(p->fft_work));
    PF_CK_CUDA(cudaMalloc(&p->fft_work, ws));
    p->fft_work_bytes = ws;
    PF_CK(plan_reset_work_areas(p));
  }
  PF_CK_FFT(cufftSetWorkArea(f->plan2d, p->fft_work));
  PF_CK_FFT(cufftSetStream(f->plan2d, p->work));
  switch (N) {
    case 64: PF_CK(tset_attrs<64>(f)); break;
    case 128: PF_CK(tset_attrs<128>(f)); break;
    case 256: PF_CK(tset_attrs<256>(f)); break;
    default: PF_CK(tset_attrs<512>(f)); break;
  }
  p->tfused = f;
  p->scratch_bytes += bytes;
  return PF_OK;
}

void tfused_free(pf_plan* p) {
  FusedTPlan* f = ftp(p);
  if (!f) return;
  if (f->plan2d) cufftDestroy(f->plan2d);
  cudaFree(f->mem);
  cudaFree(f->g0mem);
  delete f;
  p->tfused = nullptr;
}

static ft::TP tparams(pf_plan* p) {
  ft::TP P;
  for (int i = 0; i < 3; ++i) {
    P.kap[i] = p->kap[i];
    P.ell[i] = p->ell[i];
    P.g[i] = p->tc.g[i];
    P.b0v[i] = p->tc.b0v[i];
  }
  P.pe = p->tc.pe;
  P.eta = p->tc.eta;
  P.a0 = p->tc.a0;
  P.ubg = p->tc.ubar_dot_g;
  P.inv_n = p->g.inv_n;
  return P;
}

template <int N>
static int tsetup_t(pf_plan* p, bool warm) {
  FusedTPlan* f = ftp(p);
  const int64_t nh = p->g.nh;
  const int nb = blocks_for(nh);
  // chi^ of the initial chi (r1 of iteration 1); zero start -> zeros
  if (warm) {
    PF_CK(plan_fft(p, true, 1, p->t_chi, p->specB));
    ft::k_to_tm<N><<<nb, kThreads, 0, p->work>>>(p->specB, f->b.CH, 1);
    // FFT of the given grad chi (r2 of iteration 1)
    if (!f->g0mem) PF_CK_CUDA(cudaMalloc(&f->g0mem, sizeof(double2) * 3 * nh));
    PF_CK(plan_fft(p, true, 3, p->t_grad, p->specB));
    ft::k_to_tm<N><<<nb, kThreads, 0, p->work>>>(p->specB, f->g0mem, 3);
    f->b.G0 = f->g0mem;
  } else {
    PF_CK_CUDA(cudaMemsetAsync(f->b.CH, 0, sizeof(double2) * nh, p->work));
    f->b.G0 = nullptr;
  }
  // first polarization from the given grad chi, transformed over axes (1, 2)
  PF_CK(transport_polarize(p, p->t_grad, p->realB));
  PF_CK_FFT(cufftExecD2Z(f->plan2d, (cufftDoubleReal*)p->realB, (cufftDoubleComplex*)p->specA));
  ft::k_tinit_y<N><<<nb, kThreads, 0, p->work>>>(p->specA, f->b, p->kap[1], p->kap[2]);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

template <int N>
static int tfinish_t(pf_plan* p) {
  FusedTPlan* f = ftp(p);
  const int nb = blocks_for(p->g.nh);
  ft::k_tout<N><<<nb, kThreads, 0, p->work>>>(f->b.CH, p->specB, tparams(p), 1);
  PF_CK_CUDA(cudaGetLastError());
  // chi and grad chi as one batch-4 inverse into (chi, grad) — they are separate user buffers
  PF_CK(plan_fft(p, false, 1, p->specB, p->t_chi));
  PF_CK(plan_fft(p, false, 3, p->specB + p->g.nh, p->t_grad));
  return PF_OK;
}

template <int N, bool INV>
static cudaError_t launch_taxis_pipe(pf_plan* p, FusedTPlan* f, const CUtensorMap& tm) {
  if constexpr (N == 128 || N == 256) {
    return launch_k(ft::k_taxis_pipe<N, INV>, INV ? f->nb_tmi : f->nb_tmf, ft::TMP<N, INV>::T,
                    ft::TMP<N, INV>::BYTES, p->work, f->b, (const double*)p->kap[1], (const Ctrl*)p->ctrl, tm);
  } else {
    (void)p, (void)f, (void)tm;
    return cudaErrorInvalidValue;
  }
}

template <int N>
static int tenqueue_t(pf_plan* p, cudaEvent_t* ev) {
  FusedTPlan* f = ftp(p);
  const ft::TP P = tparams(p);
  auto mark = [&](int i) -> int {
    if (ev) PF_CK_CUDA(cudaEventRecord(ev[i], p->work));
    return PF_OK;
  };
  PF_CK(mark(0));
  // programmatic dependent launches: every pass waits (pdl_wait) before its first access
  PF_CK_CUDA(launch_k(ft::k_tpk<N>, ft::TPK<N>::TILES, ft::TPK<N>::T, ft::TPK<N>::BYTES, p->work, f->b, P,
                      (const Ctrl*)p->ctrl, f->tm_pk));
  PF_CK(mark(1));
  if (f->m_pipe) {  // persistent main tiles + k_taxis on the Nyquist tiles
    PF_CK_CUDA((launch_taxis_pipe<N, true>(p, f, f->tm_y)));
    PF_CK_CUDA(launch_k(ft::k_taxis<N, true>, 3 * (N / ft::TM<N>::CM), ft::TM<N>::T, ft::TM<N>::BYTES, p->work,
                        f->b, (const double*)p->kap[1], (const Ctrl*)p->ctrl, f->tm_y, 1));
  } else {
    PF_CK_CUDA(launch_k(ft::k_taxis<N, true>, 3 * ft::TM<N>::TPC, ft::TM<N>::T, ft::TM<N>::BYTES, p->work, f->b,
                        (const double*)p->kap[1], (const Ctrl*)p->ctrl, f->tm_y, 0));
  }
  PF_CK(mark(2));
  PF_CK_CUDA(launch_k(ft::k_trs<N>, f->nb_trs, ft::TRS<N>::T, ft::TRS<N>::BYTES, p->work, f->b, P,
                      (const double*)p->t_u, (const uint8_t*)p->s_solid, (const Ctrl*)p->ctrl));
  PF_CK(mark(3));
  transport_finalize_launch(p, f->b.part, ft::TPK<N>::TILES, p->g.inv_n);
  PF_CK_CUDA(cudaGetLastError());
  PF_CK(mark(4));
  if (f->m_pipe) {
    PF_CK_CUDA((launch_taxis_pipe<N, false>(p, f, f->tm_x)));
    PF_CK_CUDA(launch_k(ft::k_taxis<N, false>, 2 * (N / ft::TM<N>::CM), ft::TM<N>::T, ft::TM<N>::BYTES_FWD, p->work,
                        f->b, (const double*)p->kap[1], (const Ctrl*)p->ctrl, f->tm_x, 1));
  } else {
    PF_CK_CUDA(launch_k(ft::k_taxis<N, false>, 2 * ft::TM<N>::TPC, ft::TM<N>::T, ft::TM<N>::BYTES_FWD, p->work, f->b,
                        (const double*)p->kap[1], (const Ctrl*)p->ctrl, f->tm_x, 0));
  }
  PF_CK(mark(5));
  return PF_OK;
}

int tfused_setup(pf_plan* p, bool warm) {
  PF_CK(tfused_ensure(p));
  switch (ftp(p)->N) {
    case 64: return tsetup_t<64>(p, warm);
    case 128: return tsetup_t<128>(p, warm);
    case 256: return tsetup_t<256>(p, warm);
    default: return tsetup_t<512>(p, warm);
  }
}

int tfused_finish(pf_plan* p) {
  switch (ftp(p)->N) {
    case 64: return tfinish_t<64>(p);
    case 128: return tfinish_t<128>(p);
    case 256: return tfinish_t<256>(p);
    default: return tfinish_t<512>(p);
  }
}

int tfused_enqueue(pf_plan* p, cudaEvent_t* ev) {
  switch (ftp(p)->N) {
    case 64: return tenqueue_t<64>(p, ev);
    case 128: return tenqueue_t<128>(p, ev);
    case 256: return tenqueue_t<256>(p, ev);
    default: return tenqueue_t<512>(p, ev);
  }
}

}  // namespace pf
