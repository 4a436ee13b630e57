// Fused Stokes ADMM pipeline for cubic power-of-two grids (N = 64 ... 1024).
//
// Every 3D transform of the loop is split along its axes and fused with the
// pointwise / spectral work that consumes it, so each iteration streams the
// fields through HBM in four passes instead of cuFFT's multi-pass transforms
// plus separate pointwise kernels:
//
//   PK  (axis-0 pencils, tile = (k1, CP columns of k2), all k0):
//         FFT_0 of R~ = FFT_{2,1}(b u~ - a) -> R^ ; Green's operator (pure.py:26-56),
//         D^ = i k.U^, Q^' = Q^ - beta D^ (stokes.py:381, 408-409), Parseval sums;
//         IFFT_0 of U^/n.                                   reads 5 words, writes 5
//   MI  (axis-1 pencils, tile = (i0, CM columns)): IFFT_1 of U^.   reads 3, writes 3
//   RS  (rows along axis 2, tile = 1024 voxels of one component): C2R of u'
//         (two rows per complex FFT), the local projection and multiplier
//         updates + six squared norms (pure.py:59-68, stokes.py:254-277), and
//         R2C of R = b u~' - a' (two rows per complex FFT).  reads 15 words, writes 15
//   F   k_stokes_finalize (shared with the cuFFT pipeline)
//   RSF (only when residual balancing changed b): X-space of u~'.
//   MF  (axis-1 pencils): FFT_1 of R + (b' - b) X(u~') = X(b' u~' - a')
//         (post-adaptation b', stokes.py:405-407).           reads 3, writes 3
//
// Spectra are stored as [rows][N/2] complex plus a separate Nyquist column
// [rows] so rows stay 2 KiB aligned.  All FFTs are hand-written radix-8/16
// Stockham-style passes in registers with one padded shared-memory transpose
// (fft_seq); a thread group of 8 or 16 lanes transforms one sequence.  N = 512 /
// 1024 sequences are 2 / 4 such 256-point blocks plus a radix-2 / radix-4 stage
// across them (pf_fft.cuh radix_stage, fft_units; spectra in block-interleaved
// order in shared memory only).  Slab mode (SL) runs the same passes on one
// rank's x- / y-slab, with the transpose either by all_to_all between the passes
// or fused into PK's / MF's stores to the owning ranks' buffers (Bufs::peers).
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "pf_internal.cuh"

#include "pf_fft.cuh"

#ifndef PF_PK_PREFETCH
#define PF_PK_PREFETCH 1
#endif
#ifndef PF_RSC_MINB
// min CTAs/SM for the compact RS (measured: N = 256 at 4 keeps 240 registers,
// forcing 5 squeezes ptxas to 168 with spills and is 16 % slower; N <= 128 at 3)
#define PF_RSC_MINB (N == 256 ? 4 : 3)
#endif
#ifndef PF_RS_W32
#define PF_RS_W32 1  // RS at N = 256: each row-pair FFT on a whole warp (fft256_w32): 0.479 -> 0.453 ms
#endif
#ifndef PF_RS_HALFT
#define PF_RS_HALFT(N) ((N) <= 128)
#endif
#ifndef PF_RSC_MAXNREG
#define PF_RSC_MAXNREG
#endif
#ifndef PF_PK_TMA
#define PF_PK_TMA 1  // PK loads its pencils with 3D TMA tensor copies (single GPU, N = 128/256)
#endif
#ifndef PF_M_TMA
#define PF_M_TMA 1  // axis-1 passes load their tiles with one 2D TMA copy (single GPU, N = 128/256)
#endif
#ifndef PF_M_MINB
#define PF_M_MINB 5  // min blocks per SM for the axis-1 passes: 96 regs, 5 blocks (smem-limited too)
#endif
#ifndef PF_PK_MINB
#define PF_PK_MINB 3  // __launch_bounds__ min blocks per SM for k_pk (1 lets ptxas take 216 regs: 2 blocks/SM, slower)
#endif
#ifndef PF_PK_PIPE
#define PF_PK_PIPE 0  // N = 128 / 256 single GPU: persistent pipelined PK (measured slower: 0.37 vs 0.31 ms)
#endif
#ifndef PF_M_PIPE
// single GPU: persistent pipelined axis-1 passes (POREFLOW_B200_M_PIPE=0/1 overrides).
// Measured: 128^3 cell 11.8 -> 12.4, 8-cell 128^3 ensemble 13.0 -> 14.3 Gvox-it/s;
// at 256^3 (2 CTAs/SM of 101 KB) MI / MF slow from 0.129 to 0.15 ms, so N = 128 only
#define PF_M_PIPE(N) ((N) == 128)
#endif
#ifndef PF_ABL_NOFIN
#define PF_ABL_NOFIN 0  // measurement-only ablations of the per-iteration fixed costs (results invalid)
#endif
#ifndef PF_ABL_NORSF
#define PF_ABL_NORSF 0
#endif
#ifndef PF_MP_STAGES
#define PF_MP_STAGES 2  // TMA ring depth of the persistent axis-1 passes
#endif
#ifndef PF_MP_MINB
#define PF_MP_MINB 1
#endif
#ifndef PF_RS_SPLIT
#define PF_RS_SPLIT 1  // compact RS refills its X rows one step before the rest of its stage
#endif
#ifndef PF_RSFIX_TMA
#define PF_RSFIX_TMA 1  // TMA-staged RS-fix on the single-GPU compact path (POREFLOW_B200_RSFIX_TMA=0/1)
#endif
#ifndef PF_GROUPED
#define PF_GROUPED 0  // grouped last-block partial reductions in PK / RS (measured slower at 64^3 / 128^3, neutral at 256^3)
#endif
#ifndef PF_PK3
#define PF_PK3 0  // N = 256 single GPU: register-resident PK (k_pk3; POREFLOW_B200_PK3=0/1)
#endif
#ifndef PF_PK3_MINB
#define PF_PK3_MINB 3
#endif
#ifndef PF_PK3_CARVE
#define PF_PK3_CARVE 100
#endif
#ifndef PF_PK_TMASTORE
#define PF_PK_TMASTORE 1  // k_pk stores Y with TMA tensor stores from its boxes (single GPU, N = 128/256)
#endif
#ifndef PF_YBLOCK
#define PF_YBLOCK 1  // single GPU, N <= 256: i0-blocked Y layout (Bufs::yb; POREFLOW_B200_YBLOCK=0 disables)
#endif
#ifndef PF_PK128_MINB
#define PF_PK128_MINB 4  // 128^3: 4 CTAs/SM (128 regs): cell 12.80 -> 12.94, 16-cell ensemble 14.26 -> 14.51 Gvox-it/s
#endif
#ifndef PF_PK_THREADS
#define PF_PK_THREADS 128
#endif
#ifndef PF_PK64_T
#define PF_PK64_T PF_PK_THREADS  // PK threads at N = 64 (tile shape: CP columns from T / 8-lane groups)
#endif
#ifndef PF_M64_T
#define PF_M64_T 128  // axis-1 passes' threads at N = 64 (columns per tile = T / 8)
#endif
#ifndef PF_PK512_T  // PK at N = 512: threads, columns per tile, min blocks per SM (measured:
#define PF_PK512_T 192  // 3.85 ms vs 4.06 at 128 threads / 2 columns / 3 blocks)
#endif
#ifndef PF_PK512_CP
#define PF_PK512_CP 4
#endif
#ifndef PF_PK512_MINB
#define PF_PK512_MINB 2
#endif
#ifndef PF_PK1024_T  // PK at N = 1024: 2 columns (32-byte pencil rows) x 192 threads, 2 blocks/SM
#define PF_PK1024_T 192  // (1024^3 rank of 2: 18.8 ms vs 31.5 with 1 column x 128 threads; rank of 8: 3.66 vs 3.70)
#endif
#ifndef PF_PK1024_CP
#define PF_PK1024_CP 2
#endif
#ifndef PF_PK1024_MINB
#define PF_PK1024_MINB 2
#endif
#ifndef PF_RS1024_T
#define PF_RS1024_T 128  // one warp per 256-point block (fft_units_w32): rank of 8 RS 5.97 -> 5.71 ms
#endif
#ifndef PF_RS512_T  // RS threads at N = 512 (one row pair per tile: 2 block transforms of 16 lanes)
#define PF_RS512_T 64  // (measured 3.93 ms vs 4.38 at 32 and 4.48 at 128)
#endif

namespace pf {
namespace fz {

// 16-byte chunk XOR of TMA row e for box rows of RB bytes (SWIZZLE_128B/64B/32B;
// 16-byte rows are not swizzled): the chunk index is XORed with address bits
// [7, 7 + log2(RB / 16)) of the row start, i.e. with (e * RB) >> 7.
template <int RB>
__device__ __forceinline__ int swz16(int e) {
  return RB == 128 ? (e & 7) : (RB == 64 ? ((e >> 1) & 3) : (RB == 32 ? ((e >> 2) & 1) : 0));
}

// offset of Y main element (c, i0, k1, k2) on a single GPU (k1 < N, k2 < N/2)
template <int N>
__device__ __forceinline__ size_t ymain(int yb, int c, int i0, int k1, int k2) {
  constexpr int H = N / 2;
  return yb ? ((((size_t)(c * (N / 4) + (i0 >> 2)) * N + k1) * 4 + (i0 & 3)) * H + k2)
            : (((size_t)(c * N + i0) * N + k1) * H + k2);
}

#ifndef PF_PART_EVICT_LAST
#define PF_PART_EVICT_LAST 1  // per-block partials stored with an L2 evict_last hint (the finalize reads them)
#endif
// Partial sums are read by the one-block finalize after the next passes have
// streamed gigabytes through L2; an evict_last store keeps them resident.
__device__ __forceinline__ void st_part(double* p, double v) {
#if PF_PART_EVICT_LAST
  asm volatile(
      "{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
      " st.global.L2::cache_hint.f64 [%0], %1, pol;\n}" ::"l"(p),
      "d"(v)
      : "memory");
#else
  *p = v;
#endif
}

#ifndef PF_GRP_PK
#define PF_GRP_PK 64  // PK tiles per partial group
#endif
#ifndef PF_GRP_RS
#define PF_GRP_RS 16  // RS blocks per partial group
#endif
// Deterministic grouped reduction of per-block partials (thread 0 holds the
// block's totals v): each block stores its NQ partials to part[q nb + b]; the last
// block to arrive in its group of GS (atomic counter, threadfence pattern) sums the
// group's partials in index order with one warp — lane i takes i, i + 32, ... then
// a fixed shuffle tree — into gpart[q ng + g] and resets the counter.  The result
// does not depend on which block arrives last.
template <int NQ>
__device__ __forceinline__ void group_reduce(const double (&v)[NQ], double* part, int nb, double* gpart,
                                             unsigned* cnt, int GS) {
  __shared__ int s_last;
  const int b = blockIdx.x, g = b / GS, ng = (nb + GS - 1) / GS;
  const int gsz = min(GS, nb - g * GS);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) part[(size_t)q * nb + b] = v[q];
    __threadfence();
    s_last = atomicAdd(&cnt[g], 1u) == (unsigned)(gsz - 1);
  }
  __syncthreads();
  if (s_last && threadIdx.x < 32) {
    __threadfence();
    const int lane = threadIdx.x, b0 = g * GS;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double x = 0.0;
      for (int i = lane; i < gsz; i += 32) x += __ldcg(part + (size_t)q * nb + b0 + i);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      if (lane == 0) gpart[(size_t)q * ng + g] = x;
    }
    if (lane == 0) cnt[g] = 0u;
  }
}

constexpr int kMaxRanks = 16;
struct Peers {
  double2 *yy[kMaxRanks], *yyn[kMaxRanks];  // y-slab Y of each rank
  double2 *yx[kMaxRanks], *yxn[kMaxRanks];  // x-slab Y of each rank
};

struct Bufs {
  double2 *XU, *XUn;  // X-space (after axis 2): u' (MI -> RS); X(u~') when b changed (RS-fix -> MF)
  double2 *XR, *XRn;  // X-space R = b u~' - a' (RS -> MF)   [3][N*N][H], [3][N*N]
  double2 *Y, *Yn;    // Y-space (after axes 2,1): R~ in, U^ out  [3][N][N][H], [3][N][N]
  double2* Q;         // full spectrum Q^, PK tile-major [tile][q][k0] (nh modes)
  double2* D;         // full spectrum D^_prev, same layout
  double2* tw;        // N forward twiddles
  double *part_rs, *part_pk;
  // grouped partials (single GPU): the last block of each group of PF_GRP_PK PK tiles /
  // PF_GRP_RS RS blocks sums its group's partials (index order) into gpk / grs, so the
  // finalize reads ~100 - 600 values instead of one per PK tile and RS block
  double *gpk, *grs;
  unsigned *cpk, *crs;  // per-group arrival counters (reset by each group's last block)
  // slab layout (single GPU: l0 = l1 = N, s1 = log2 N, k1off = 0): this rank's
  // x-slab holds l0 i0-planes, its y-slab l1 k1-planes starting at k1off; P = N / l1
  // is a power of two (s1 = log2 l1).  Y (after axes 2, 1; axis 0 real) exists in
  // two exchange-native layouts so the all-to-alls move contiguous blocks (one
  // exchange per component for the main arrays, one for all Nyquist columns):
  //   y-slab (PK):     Yy [c][i0][k1 - k1off][k2],   Yn  [i0][c][k1 - k1off]
  //   x-slab (MI, MF): Yx [c][r][i0 - i0off][k1 - r l1][k2],   Yxn [r][i0 - i0off][c][k1 - r l1]
  // (r = owner of k1); at P = 1 they coincide.  X and the real state are x-slab
  // [c][l0 N rows][...].
  int l0, l1, s1, k1off;
  double2 *Yx, *Yxn;  // x-slab Y (== Y, Yn at P = 1)
  // plane window of one launch of the x-slab passes (SL kernels): planes
  // [i0a, i0a + nl) of the l0; RS partial rows at [q * pst + poff + block]
  int i0a, nl, pst, poff;
  // the host encoded the TMA tensor maps of this layout (else the passes stage with
  // LDGSTS); tma_yx: the 5D x-slab map of MI too (its box spans l1 <= 256 rows)
  int tma, tma_yx;
  // single GPU, N <= 256: Y main array i0-blocked by 4, [c][i0/4][k1][i0%4][k2] (yb = 1).
  // PK's pencils then touch 4 consecutive i0 rows 2 KB apart instead of one 64-byte
  // piece per 512 KB plane: a plain copy in PK's access pattern runs at 5.4 TB/s
  // instead of 3.5 - 3.9, while the axis-1 passes' tiles (all k1 of one (c, i0)) keep
  // 5.5 - 5.7 (tools/micro/layout_copy.cu, B200).  Slab layouts are unchanged (yb = 0).
  int yb;
  // peer-memory exchange (slab, P2P-mapped Y buffers of every rank; null = exchange by
  // all_to_all): PK stores straight into the x-slab owners' Yx, MF into the y-slab
  // owners' Yy, so the transpose rides on the passes' own stores over NVLink
  const struct Peers* peers;
  // component window of one launch of MI / RS (SL kernels): components [c0, c0 + nc)
  int c0, nc;
};

struct State {
  double *u, *ut, *a, *lam;
  const uint8_t* H;
};

// ------------------------------------------------------------------ RS
// Persistent: grid = 3 blocks per SM; each block walks tiles of R2 rows of one
// velocity component.  Per tile, one thread issues TMA bulk copies of the
// state rows (u, u~, a, lam), the X-space u' rows and the indicator into
// shared memory (one mbarrier); the next tile's copies are issued as soon as
// the current tile's staged inputs are consumed, so they overlap the forward
// FFT and the output stores.  State outputs go straight to HBM.
template <int N>
struct RS2 {
  using C = Cfg<N>;
  static constexpr int R = N > 512 ? 2 : 1024 / N;  // rows per tile (1024 voxels; one row pair at N = 1024)
  // threads per block: one FFT group per row pair (every thread FFT-active) for
  // N <= 128; for N = 256 one group per row (measured: 128^3 RS 0.071 vs 0.088 ms,
  // 256^3 0.483 vs 0.512 ms the other way round)
  static constexpr int T = N == 1024 ? PF_RS1024_T : (N == 512 ? PF_RS512_T : R * C::G / (PF_RS_HALFT(N) ? 2 : 1));
  static constexpr int V = R * N;               // voxels per tile
  static constexpr int VPT = V / T;             // voxels per thread
  static constexpr int NP = R / 2;              // inverse sequences (two rows each)
  // shared-memory carve (bytes)
  static constexpr size_t TW = sizeof(double2) * C::TWN;
  static constexpr size_t INV = sizeof(double2) * NP * C::SS;
  static constexpr size_t FWD = sizeof(double2) * NP * C::SS;
  static constexpr size_t ST = sizeof(double) * 4 * V;     // u, u~, a, lam rows
  static constexpr size_t XM = sizeof(double2) * R * C::H; // X-space u' rows (main)
  static constexpr size_t XN = sizeof(double2) * R;        // nyq column
  static constexpr size_t HB = V;                          // indicator bytes
  // the local step reads and rewrites each voxel's double in place, so the forward
  // sequences reuse the inverse buffer (FWD is not carved separately)
  static constexpr size_t BYTES = TW + INV + ST + XM + XN + HB;
  static constexpr uint32_t TX = (uint32_t)(ST + XM + XN + HB);
};

template <int N, bool SL>
__device__ __forceinline__ void rs_issue(int tile, const Bufs& B, const State& st, double* sst, double2* sx,
                                         double2* sxn, uint8_t* sh, uint64_t* mbar) {
  using K = RS2<N>;
  using C = Cfg<N>;
  const int TPC = (SL ? B.nl : N) * N / K::R;  // tiles per component
  const int c = (SL ? B.c0 : 0) + tile / TPC;
  const int64_t row0 = ((int64_t)(tile % TPC) * K::R + (SL ? (int64_t)B.i0a * N : 0));
  const int64_t n = (int64_t)(SL ? B.l0 : N) * N * N;
  const int64_t x0 = (int64_t)c * n + row0 * N;
  const uint32_t vb = sizeof(double) * K::V;
  fence_async_smem();
  mbar_expect(mbar, K::TX);
  bulk_load(sst + 0 * K::V, st.u + x0, vb, mbar);
  bulk_load(sst + 1 * K::V, st.ut + x0, vb, mbar);
  bulk_load(sst + 2 * K::V, st.a + x0, vb, mbar);
  bulk_load(sst + 3 * K::V, st.lam + x0, vb, mbar);
  bulk_load(sx, B.XU + ((int64_t)c * (SL ? B.l0 : N) * N + row0) * C::H, (uint32_t)K::XM, mbar);
  bulk_load(sxn, B.XUn + (int64_t)c * (SL ? B.l0 : N) * N + row0, (uint32_t)K::XN, mbar);
  bulk_load(sh, st.H + row0 * N, (uint32_t)K::HB, mbar);
}

template <int N, bool SL>
__global__ void __launch_bounds__(RS2<N>::T) k_rs(Bufs B, State st, const Ctrl* __restrict__ ctrl) {
  using C = Cfg<N>;
  using K = RS2<N>;
  constexpr int H = C::H, SS = C::SS, R = K::R, T = K::T, V = K::V, NP = K::NP;
  const int TPC = (SL ? B.nl : N) * N / R;
  const int NT = (SL ? B.nc : 3) * TPC;  // component window [c0, c0 + nc) (slab)
  pdl_wait();
  if (ctrl->done) return;
  extern __shared__ __align__(128) unsigned char sraw[];
  __shared__ uint64_t mbar;
  double2* tw = (double2*)sraw;
  double2* SI = (double2*)(sraw + K::TW);
  double2* SF = SI;  // in place (see RS2::BYTES)
  double* sst = (double*)(sraw + K::TW + K::INV);
  double2* sx = (double2*)(sraw + K::TW + K::INV + K::ST);
  double2* sxn = (double2*)(sraw + K::TW + K::INV + K::ST + K::XM);
  uint8_t* sh = (uint8_t*)(sraw + K::TW + K::INV + K::ST + K::XM + K::XN);
  const int t = threadIdx.x, g = t / C::G, l = t % C::G;
  for (int j = t; j < Cfg<N>::TWN; j += T) tw[j] = B.tw[j];
  const double alpha = ctrl->alpha, b = ctrl->b;
  const double inv_bp = 1.0 / b, inv_bs = 1.0 / (b + alpha);  // pore / solid divisors of pure.py:61
  const int64_t n = (int64_t)(SL ? B.l0 : N) * N * N;
  if (t == 0) {
    mbar_init(&mbar);
    if ((int)blockIdx.x < NT) rs_issue<N, SL>(blockIdx.x, B, st, sst, sx, sxn, sh, &mbar);
  }
  __syncthreads();
  double acc[6] = {0, 0, 0, 0, 0, 0};
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < NT; tile += gridDim.x, phase ^= 1u) {
    const int c = (SL ? B.c0 : 0) + tile / TPC;
    const int64_t row0 = ((int64_t)(tile % TPC) * R + (SL ? (int64_t)B.i0a * N : 0));
    double2* XR = B.XR + (size_t)c * (SL ? B.l0 : N) * N * H;
    double2* XRn = B.XRn + (size_t)c * (SL ? B.l0 : N) * N;
    mbar_wait(&mbar, phase);
    // (1) inverse: two rows per complex FFT (Hermitian extension of each half spectrum)
    for (int idx = t; idx < NP * H; idx += T) {
      const int p = idx / H, k = idx % H;
      double2 xa = sx[(2 * p) * H + k], xb = sx[(2 * p + 1) * H + k];
      if (k == 0) xa.y = xb.y = 0.0;  // C2R keeps the real part of self-conjugate modes
      double2* sp = SI + p * SS;
      sp[C::kp(k)] = make_double2(xa.x - xb.y, xa.y + xb.x);
      if (k > 0) sp[C::kp(N - k)] = make_double2(xa.x + xb.y, xb.x - xa.y);
    }
    for (int p = t; p < NP; p += T) SI[p * SS + C::kp(H)] = make_double2(sxn[2 * p].x, sxn[2 * p + 1].x);
    __syncthreads();
    if constexpr (PF_RS_W32 && C::L == 256 && T == 32 * NP * C::M) {
      fft_units_w32<N, true>(SI, NP, SS, tw, t);
    } else {
      fft_units<N, true>(SI, NP, SS, tw, g, l, T / C::G);
    }
    if constexpr (C::M > 1) {
      __syncthreads();
      radix_stage<N, true>(SI, NP, SS, tw, t, T);
    }
    __syncthreads();
    // (2) local projection + multipliers (pure.py:59-68) and six squared norms; a
    // lane takes both rows of a pair at one column (one 16-byte sequence access)
#pragma unroll 2
    for (int j = 0; j < K::VPT / 2; ++j) {
      const int w = t + T * j, p = w / N, col = w % N;
      double2* zp = SI + p * SS + C::sp(col);
      const double2 z = *zp;
      double rr[2];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int v = (2 * p + hh) * N + col;
        const double u1 = hh ? z.y : z.x;
        const double h = sh[v] ? 1.0 : 0.0;
        const double u0 = sst[v], t0 = sst[V + v], a0 = sst[2 * V + v], l0 = sst[3 * V + v];
        // (a + b u - H lam) / (b + alpha H): the divisor takes two values, so divide by
        // multiplying with the hoisted reciprocals (<= 1 ulp from the quotient)
        const double t1 = ((a0 + b * u1) - h * l0) * (h != 0.0 ? inv_bs : inv_bp);
        const double a1 = a0 + b * (u1 - t1);
        const double l1 = l0 + alpha * (h * t1);
        const double s0 = h * t1, s1 = h * (t1 - t0), s3 = u1 - t1, s4 = u1 - u0;
        acc[0] += s0 * s0;
        acc[1] += s1 * s1;
        acc[2] += l1 * l1;
        acc[3] += s3 * s3;
        acc[4] += s4 * s4;
        acc[5] += a1 * a1;
        const int64_t i = c * n + row0 * N + v;
        st.u[i] = u1;
        st.ut[i] = t1;
        st.a[i] = a1;
        st.lam[i] = l1;
        // R = b u~' - a' with the pre-adaptation b (stokes.py:405-407); rows 2p, 2p+1 -> Re, Im
        rr[hh] = b * t1 - a1;
      }
      *zp = make_double2(rr[0], rr[1]);
    }
    __syncthreads();
    // staged inputs consumed: prefetch the next tile while this one finishes
    if (t == 0 && tile + (int)gridDim.x < NT) rs_issue<N, SL>(tile + gridDim.x, B, st, sst, sx, sxn, sh, &mbar);
    if constexpr (C::M > 1) {
      radix_stage<N, false>(SF, NP, SS, tw, t, T);
      __syncthreads();
    }
    if constexpr (PF_RS_W32 && C::L == 256 && T == 32 * NP * C::M) {
      fft_units_w32<N, false>(SF, NP, SS, tw, t);
    } else {
      fft_units<N, false>(SF, NP, SS, tw, g, l, T / C::G);
    }
    __syncthreads();
    // (3) separate the two real transforms of each row pair, store X-space rows of R
    for (int idx = t; idx < NP * H; idx += T) {
      const int p = idx / H, k = idx % H;
      const double2 zk = SF[p * SS + C::kp(k)], zm = SF[p * SS + C::kp((N - k) & (N - 1))];
      XR[(row0 + 2 * p) * H + k] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
      XR[(row0 + 2 * p + 1) * H + k] = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
    }
    for (int p = t; p < NP; p += T) {
      const double2 z = SF[p * SS + C::kp(H)];
      XRn[row0 + 2 * p] = make_double2(z.x, 0.0);
      XRn[row0 + 2 * p + 1] = make_double2(z.y, 0.0);
    }
    __syncthreads();
  }
  block_sum<6>(acc);
  if (!SL && B.crs) {
    group_reduce<6>(acc, B.part_rs, gridDim.x, B.grs, B.crs, PF_GRP_RS);
  } else if (t == 0) {
    for (int k = 0; k < 6; ++k)
      st_part(B.part_rs + (SL ? (size_t)k * B.pst + B.poff + blockIdx.x : (size_t)k * gridDim.x + blockIdx.x), acc[k]);
  }
}

// RS-fix: X-space of u~' (row FFTs of the state), needed by MF only in the
// iterations where residual balancing changed b (ctrl->db != 0); a no-op
// otherwise.  Persistent, TMA bulk loads, same tiling as RS.
template <int N, bool SL>
__global__ void __launch_bounds__(RS2<N>::T) k_rsfix(Bufs B, const double* __restrict__ ut, const Ctrl* __restrict__ ctrl) {
  using C = Cfg<N>;
  using K = RS2<N>;
  constexpr int H = C::H, SS = C::SS, R = K::R, T = K::T, V = K::V, NP = K::NP;
  const int TPC = (SL ? B.nl : N) * N / R;
  const int NT = 3 * TPC;
  pdl_wait();
  if (ctrl->done || ctrl->db == 0.0) return;
  extern __shared__ __align__(128) unsigned char sraw[];
  __shared__ uint64_t mbar;
  double2* tw = (double2*)sraw;
  double2* SF = (double2*)(sraw + K::TW);
  double* sst = (double*)(sraw + K::TW + K::INV);
  const int t = threadIdx.x, g = t / C::G, l = t % C::G;
  for (int j = t; j < Cfg<N>::TWN; j += T) tw[j] = B.tw[j];
  const int64_t n = (int64_t)(SL ? B.l0 : N) * N * N;
  auto issue = [&](int tile) {
    const int c = tile / TPC;
    const int64_t row0 = ((int64_t)(tile % TPC) * R + (SL ? (int64_t)B.i0a * N : 0));
    fence_async_smem();
    mbar_expect(&mbar, sizeof(double) * V);
    bulk_load(sst, ut + (int64_t)c * n + row0 * N, sizeof(double) * V, &mbar);
  };
  if (t == 0) {
    mbar_init(&mbar);
    if ((int)blockIdx.x < NT) issue(blockIdx.x);
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < NT; tile += gridDim.x, phase ^= 1u) {
    const int c = tile / TPC;
    const int64_t row0 = ((int64_t)(tile % TPC) * R + (SL ? (int64_t)B.i0a * N : 0));
    double2* XU = B.XU + (size_t)c * (SL ? B.l0 : N) * N * H;
    double2* XUn = B.XUn + (size_t)c * (SL ? B.l0 : N) * N;
    mbar_wait(&mbar, phase);
    for (int v = t; v < V; v += T) {
      const int row = v / N, col = v % N;
      reinterpret_cast<double*>(SF + (row >> 1) * SS + C::sp(col))[row & 1] = sst[v];
    }
    __syncthreads();
    if (t == 0 && tile + (int)gridDim.x < NT) issue(tile + gridDim.x);
    if constexpr (C::M > 1) {
      radix_stage<N, false>(SF, NP, SS, tw, t, T);
      __syncthreads();
    }
    if constexpr (PF_RS_W32 && C::L == 256 && T == 32 * NP * C::M) {
      fft_units_w32<N, false>(SF, NP, SS, tw, t);
    } else {
      fft_units<N, false>(SF, NP, SS, tw, g, l, T / C::G);
    }
    __syncthreads();
    for (int idx = t; idx < NP * H; idx += T) {
      const int p = idx / H, k = idx % H;
      const double2 zk = SF[p * SS + C::kp(k)], zm = SF[p * SS + C::kp((N - k) & (N - 1))];
      XU[(row0 + 2 * p) * H + k] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
      XU[(row0 + 2 * p + 1) * H + k] = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
    }
    for (int p = t; p < NP; p += T) {
      const double2 z = SF[p * SS + C::kp(H)];
      XUn[row0 + 2 * p] = make_double2(z.x, 0.0);
      XUn[row0 + 2 * p + 1] = make_double2(z.y, 0.0);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ compact RS
// On pore voxels (H = 0) the local step is exactly u~' = u', a' = 0, lam' = lam
// (a' = a + b(u' - (a + b u')/b) = 0 for any a), so once a = 0 on pore voxels
// (cold start, or any state this path produced) u~, a, lam only need storage
// and traffic on solid voxels.  The compact path keeps them in solid-only
// arrays ([c][ns], rows padded to even counts so every row range is 16-byte
// aligned) addressed through an exclusive prefix `off` of the per-row counts;
// pore values are materialised once at the end.  RS then streams u (r+w), X
// (r+w) and H for every voxel and the three multiplier fields only for the
// solid fraction.
struct Compact {
  const uint32_t* off;   // [N*N + 1]
  double *ut, *a, *lam;  // [3][ns]
  int64_t ns;
  int cs;                // staging capacity per tile: max padded solid count of any tile, rounded to 16
};

template <int N>
struct RSC {
  using K = RS2<N>;
  static constexpr int CS = K::V + K::R + 16;  // worst-case staging capacity (every voxel solid)
  // dynamic smem for staging capacity cs (sized per geometry at setup)
  static constexpr size_t bytes(int cs) {
    return K::TW + K::INV /*inverse = forward, in place*/ + sizeof(double) * K::V /*u*/ +
           3 * sizeof(double) * (size_t)cs /*u~, a, lam*/ + K::XM + K::XN + K::HB;
  }
  static constexpr size_t BYTES = bytes(CS);
};

// o0 / o1 = compact offsets of the tile's first row and of the row after it
// (loaded by the caller one tile ahead so the issue does not wait on them)
// part: 0 = every staged input on mbar; 1 = the X rows only (on mbar); 2 = the state
// rows, indicator and solid range only (on mbar).  The split lets k_rs_compact refill
// its X rows as soon as they are packed into the inverse sequences, one step before
// the rest of the stage is consumed.
template <int N, bool SL>
__device__ __forceinline__ void rsc_issue(int tile, const Bufs& B, const State& st, const Compact& cp, double* su,
                                          double* sc, double2* sx, double2* sxn, uint8_t* sh, uint64_t* mbar,
                                          uint32_t* ro_slot, const uint32_t* ro, int part = 0) {
  using K = RS2<N>;
  using C = Cfg<N>;
  const int TPC = (SL ? B.nl : N) * N / K::R;
  const int c = (SL ? B.c0 : 0) + tile / TPC;
  const int64_t row0 = ((int64_t)(tile % TPC) * K::R + (SL ? (int64_t)B.i0a * N : 0));
  const int64_t n = (int64_t)(SL ? B.l0 : N) * N * N;
  constexpr int R = K::R;
  fence_async_smem();
  if (part == 1) {
    mbar_expect(mbar, (uint32_t)(K::XM + K::XN));
    bulk_load(sx, B.XU + ((int64_t)c * (SL ? B.l0 : N) * N + row0) * C::H, (uint32_t)K::XM, mbar);
    bulk_load(sxn, B.XUn + (int64_t)c * (SL ? B.l0 : N) * N + row0, (uint32_t)K::XN, mbar);
    return;
  }
  const uint32_t o0 = ro[0];
  const uint32_t cb = sizeof(double) * (ro[R] - o0);
  for (int r = 0; r <= R; ++r) ro_slot[r] = ro[r];  // read by the compute phase after the mbarrier wait
  if (part == 2) {
    mbar_expect(mbar, (uint32_t)(sizeof(double) * K::V + K::HB) + 3 * cb);
  } else {
    mbar_expect(mbar, (uint32_t)(sizeof(double) * K::V + K::XM + K::XN + K::HB) + 3 * cb);
    bulk_load(sx, B.XU + ((int64_t)c * (SL ? B.l0 : N) * N + row0) * C::H, (uint32_t)K::XM, mbar);
    bulk_load(sxn, B.XUn + (int64_t)c * (SL ? B.l0 : N) * N + row0, (uint32_t)K::XN, mbar);
  }
  bulk_load(su, st.u + (int64_t)c * n + row0 * N, sizeof(double) * K::V, mbar);
  bulk_load(sh, st.H + row0 * N, (uint32_t)K::HB, mbar);
  if (cb) {
    const int64_t base = (int64_t)c * cp.ns + o0;
    bulk_load(sc, cp.ut + base, cb, mbar);
    bulk_load(sc + cp.cs, cp.a + base, cb, mbar);
    bulk_load(sc + 2 * cp.cs, cp.lam + base, cb, mbar);
  }
}

// Compact base of 32-voxel segment `lane` of a tile (V = 1024 => 32 segments of
// 32 voxels for every N): count nonzero indicator bytes, scan within the row
// (SPR segments per row), add the row's compact offset.  Every warp computes all
// 32 in registers; a warp shuffles out the one its voxels fall in.
template <int N>
__device__ __forceinline__ int seg_base(const uint8_t* seg_bytes, uint32_t row_off_minus_o0, int lane) {
  constexpr int SPR = N / 32;
  const uint4 w0 = reinterpret_cast<const uint4*>(seg_bytes)[0];
  const uint4 w1 = reinterpret_cast<const uint4*>(seg_bytes)[1];
  int cnt = (__popc(__vcmpne4(w0.x, 0u)) + __popc(__vcmpne4(w0.y, 0u)) + __popc(__vcmpne4(w0.z, 0u)) +
             __popc(__vcmpne4(w0.w, 0u)) + __popc(__vcmpne4(w1.x, 0u)) + __popc(__vcmpne4(w1.y, 0u)) +
             __popc(__vcmpne4(w1.z, 0u)) + __popc(__vcmpne4(w1.w, 0u))) >> 3;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < SPR; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o, SPR);
    if ((lane % SPR) >= o) incl += y;
  }
  return (int)row_off_minus_o0 + incl - cnt;
}

template <int N, bool SL>
__global__ void __launch_bounds__(RS2<N>::T, PF_RSC_MINB) PF_RSC_MAXNREG k_rs_compact(Bufs B, State st, Compact cp, const Ctrl* __restrict__ ctrl) {
  using C = Cfg<N>;
  using K = RS2<N>;
  constexpr int H = C::H, SS = C::SS, R = K::R, T = K::T, V = K::V, NP = K::NP;
  const int TPC = (SL ? B.nl : N) * N / R;
  const int NT = (SL ? B.nc : 3) * TPC;  // component window [c0, c0 + nc) (slab)
  // (32-voxel segments: N / 32 per row)
  const int CS = cp.cs;
  static_assert(T % 32 == 0, "segment bases are per warp");
  // segment bases: groups of 32 segments of 32 voxels (V = 1024: one; 2048 at N = 1024: two)
  constexpr int SG = V / 1024;
  // one warp per row-pair sequence (fft256_w32) where the tile has exactly one per warp
  constexpr bool W32 = PF_RS_W32 && C::L == 256 && T == 32 * NP * C::M;
  if (V != 1024 && V != 2048) return;  // (never launched otherwise)
  pdl_wait();
  if (ctrl->done) return;
  extern __shared__ __align__(128) unsigned char sraw[];
  __shared__ uint64_t mbar, mbx;  // mbx: the X rows when PF_RS_SPLIT (refilled one step earlier)
  __shared__ uint32_t ros[2][R + 1];
  double2* tw = (double2*)sraw;
  double2* SI = (double2*)(sraw + K::TW);
  double2* SF = SI;  // in place
  double* su = (double*)(sraw + K::TW + K::INV);
  double* sc = su + V;  // [3][CS]: u~, a, lam of the tile's solid voxels
  double2* sx = (double2*)(sc + 3 * CS);
  double2* sxn = (double2*)((unsigned char*)sx + K::XM);
  uint8_t* sh = (uint8_t*)((unsigned char*)sxn + K::XN);
  const int t = threadIdx.x, g = t / C::G, l = t % C::G, lane = t & 31;
  for (int j = t; j < Cfg<N>::TWN; j += T) tw[j] = B.tw[j];
  const double alpha = ctrl->alpha, b = ctrl->b;
  const double inv_bs = 1.0 / (b + alpha);  // solid divisor of pure.py:61
  const int64_t n = (int64_t)(SL ? B.l0 : N) * N * N;
  uint32_t ro[R + 1];
  auto offs = [&](int tl) {
    const int64_t r0 = ((int64_t)(tl % TPC) * R + (SL ? (int64_t)B.i0a * N : 0));
#pragma unroll
    for (int r = 0; r <= R; ++r) ro[r] = cp.off[r0 + r];
  };
  constexpr bool SPLIT = PF_RS_SPLIT;
  if (t == 0) {
    mbar_init(&mbar);
    mbar_init(&mbx);
    if ((int)blockIdx.x < NT) {
      offs(blockIdx.x);
      if (SPLIT) {
        rsc_issue<N, SL>(blockIdx.x, B, st, cp, su, sc, sx, sxn, sh, &mbx, ros[0], ro, 1);
        rsc_issue<N, SL>(blockIdx.x, B, st, cp, su, sc, sx, sxn, sh, &mbar, ros[0], ro, 2);
      } else {
        rsc_issue<N, SL>(blockIdx.x, B, st, cp, su, sc, sx, sxn, sh, &mbar, ros[0], ro);
      }
    }
  }
  __syncthreads();
  double acc[6] = {0, 0, 0, 0, 0, 0};
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < NT; tile += gridDim.x, phase ^= 1u) {
    const int c = (SL ? B.c0 : 0) + tile / TPC;
    const int64_t row0 = ((int64_t)(tile % TPC) * R + (SL ? (int64_t)B.i0a * N : 0));
    double2* XR = B.XR + (size_t)c * (SL ? B.l0 : N) * N * H;
    double2* XRn = B.XRn + (size_t)c * (SL ? B.l0 : N) * N;
    const bool has_next = tile + (int)gridDim.x < NT;
    if (t == 0 && has_next) offs(tile + gridDim.x);  // next tile's row offsets, loaded early
    mbar_wait(&mbar, phase);
    if (SPLIT) mbar_wait(&mbx, phase);
    const uint32_t o0 = ros[phase][0];
    int sb[2 > SG ? 2 : SG];
#pragma unroll
    for (int q = 0; q < SG; ++q) sb[q] = seg_base<N>(sh + q * 1024 + lane * 32, ros[phase][(q * 1024 + lane * 32) / N] - o0, lane);
    // (1) inverse: two rows per complex FFT (Hermitian extension of each half spectrum)
    for (int idx = t; idx < NP * H; idx += T) {
      const int p = idx / H, k = idx % H;
      double2 xa = sx[(2 * p) * H + k], xb = sx[(2 * p + 1) * H + k];
      if (k == 0) xa.y = xb.y = 0.0;
      double2* sp = SI + p * SS;
      sp[C::kp(k)] = make_double2(xa.x - xb.y, xa.y + xb.x);
      if (k > 0) sp[C::kp(N - k)] = make_double2(xa.x + xb.y, xb.x - xa.y);
    }
    for (int p = t; p < NP; p += T) SI[p * SS + C::kp(H)] = make_double2(sxn[2 * p].x, sxn[2 * p + 1].x);
    __syncthreads();
    if (SPLIT && t == 0 && has_next)  // the X rows are packed: refill them now
      rsc_issue<N, SL>(tile + gridDim.x, B, st, cp, su, sc, sx, sxn, sh, &mbx, ros[phase ^ 1u], ro, 1);
    if constexpr (W32) {
      fft_units_w32<N, true>(SI, NP, SS, tw, t);
    } else {
      fft_units<N, true>(SI, NP, SS, tw, g, l, T / C::G);
    }
    if constexpr (C::M > 1) {
      __syncthreads();
      radix_stage<N, true>(SI, NP, SS, tw, t, T);
    }
    __syncthreads();
    // (2) local step; pore: u~' = u', a' = 0, lam' = lam (only u' is stored).
    // A lane takes both rows of a pair at one column: one 16-byte access of the
    // sequence element (rows 2p, 2p+1 = Re, Im) instead of two strided 8-byte ones.
    const int64_t cbase = (int64_t)c * cp.ns + o0;
#pragma unroll 2
    for (int j = 0; j < K::VPT / 2; ++j) {
      const int w = t + T * j, p = w / N, col = w % N;
      double2* zp = SI + p * SS + C::sp(col);
      const double2 z = *zp;
      double rr[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int v = (2 * p + h) * N + col;
        const double u1 = h ? z.y : z.x;
        const bool solid = sh[v] != 0;
        const unsigned mask = __ballot_sync(0xffffffffu, solid);
        const double s4 = u1 - su[v];
        acc[4] += s4 * s4;
        double t1 = u1, a1 = 0.0;
        const int segb = __shfl_sync(0xffffffffu, (SG == 1 || (v >> 10) == 0) ? sb[0] : sb[1], (v >> 5) & 31);
        if (solid) {
          const int ci = segb + __popc(mask & ((1u << lane) - 1u));
          const double t0 = sc[ci], a0 = sc[CS + ci], l0 = sc[2 * CS + ci];
          t1 = ((a0 + b * u1) - l0) * inv_bs;  // pure.py:61 with H = 1
          a1 = a0 + b * (u1 - t1);             // pure.py:66
          const double l1 = l0 + alpha * t1;   // pure.py:67
          const double s1 = t1 - t0, s3 = u1 - t1;
          acc[0] += t1 * t1;
          acc[1] += s1 * s1;
          acc[2] += l1 * l1;
          acc[3] += s3 * s3;
          acc[5] += a1 * a1;
          cp.ut[cbase + ci] = t1;
          cp.a[cbase + ci] = a1;
          cp.lam[cbase + ci] = l1;
        }
        st.u[c * n + row0 * N + v] = u1;
        rr[h] = b * t1 - a1;
      }
      *zp = make_double2(rr[0], rr[1]);
    }
    __syncthreads();
    if (t == 0 && has_next)
      rsc_issue<N, SL>(tile + gridDim.x, B, st, cp, su, sc, sx, sxn, sh, &mbar, ros[phase ^ 1u], ro, SPLIT ? 2 : 0);
    if constexpr (C::M > 1) {
      radix_stage<N, false>(SF, NP, SS, tw, t, T);
      __syncthreads();
    }
    if constexpr (W32) {
      fft_units_w32<N, false>(SF, NP, SS, tw, t);
    } else {
      fft_units<N, false>(SF, NP, SS, tw, g, l, T / C::G);
    }
    __syncthreads();
    for (int idx = t; idx < NP * H; idx += T) {
      const int p = idx / H, k = idx % H;
      const double2 zk = SF[p * SS + C::kp(k)], zm = SF[p * SS + C::kp((N - k) & (N - 1))];
      XR[(row0 + 2 * p) * H + k] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
      XR[(row0 + 2 * p + 1) * H + k] = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
    }
    for (int p = t; p < NP; p += T) {
      const double2 z = SF[p * SS + C::kp(H)];
      XRn[row0 + 2 * p] = make_double2(z.x, 0.0);
      XRn[row0 + 2 * p + 1] = make_double2(z.y, 0.0);
    }
    __syncthreads();
  }
  block_sum<6, RS2<N>::T / 32>(acc);
  if (!SL && B.crs) {
    group_reduce<6>(acc, B.part_rs, gridDim.x, B.grs, B.crs, PF_GRP_RS);
  } else if (t == 0) {
    for (int k = 0; k < 6; ++k)
      st_part(B.part_rs + (SL ? (size_t)k * B.pst + B.poff + blockIdx.x : (size_t)k * gridDim.x + blockIdx.x), acc[k]);
  }
}

// RS-fix on the compact path: u~' rows = u' on pore voxels, the compact u~ on solid ones.
template <int N, bool SL>
__global__ void __launch_bounds__(RS2<N>::T) k_rsfix_compact(Bufs B, const double* __restrict__ u,
                                                             const uint8_t* __restrict__ Hs, Compact cp,
                                                             const Ctrl* __restrict__ ctrl) {
  using C = Cfg<N>;
  using K = RS2<N>;
  constexpr int H = C::H, SS = C::SS, R = K::R, T = K::T, V = K::V, NP = K::NP;
  const int TPC = (SL ? B.nl : N) * N / R;
  const int NT = 3 * TPC;

  static_assert(T % 32 == 0, "segment bases are per warp");
  constexpr int SG = V / 1024;  // segment-base groups (see k_rs_compact)
  if (V != 1024 && V != 2048) return;  // (never launched otherwise)
  pdl_wait();
  if (ctrl->done || ctrl->db == 0.0) return;
  extern __shared__ __align__(128) unsigned char sraw[];
  double2* tw = (double2*)sraw;
  double2* SF = (double2*)(sraw + K::TW);
  const int t = threadIdx.x, g = t / C::G, l = t % C::G, lane = t & 31;
  for (int j = t; j < Cfg<N>::TWN; j += T) tw[j] = B.tw[j];
  const int64_t n = (int64_t)(SL ? B.l0 : N) * N * N;
  for (int tile = blockIdx.x; tile < NT; tile += gridDim.x) {
    const int c = tile / TPC;
    const int64_t row0 = ((int64_t)(tile % TPC) * R + (SL ? (int64_t)B.i0a * N : 0));
    const uint32_t o0 = cp.off[row0];
    int sb[2 > SG ? 2 : SG];
#pragma unroll
    for (int q = 0; q < SG; ++q)
      sb[q] = seg_base<N>(Hs + row0 * N + q * 1024 + lane * 32, cp.off[row0 + (q * 1024 + lane * 32) / N] - o0, lane);
    __syncthreads();
    for (int j = 0; j < K::VPT; ++j) {
      const int v = t + T * j, row = v / N, col = v % N;
      const bool solid = Hs[row0 * N + v] != 0;
      const unsigned mask = __ballot_sync(0xffffffffu, solid);
      const int segb = __shfl_sync(0xffffffffu, (SG == 1 || (v >> 10) == 0) ? sb[0] : sb[1], (v >> 5) & 31);
      double val = u[(int64_t)c * n + row0 * N + v];
      if (solid) val = cp.ut[(int64_t)c * cp.ns + o0 + segb + __popc(mask & ((1u << lane) - 1u))];
      reinterpret_cast<double*>(SF + (row >> 1) * SS + C::sp(col))[row & 1] = val;
    }
    __syncthreads();
    if constexpr (C::M > 1) {
      radix_stage<N, false>(SF, NP, SS, tw, t, T);
      __syncthreads();
    }
    if constexpr (PF_RS_W32 && C::L == 256 && T == 32 * NP * C::M) {
      fft_units_w32<N, false>(SF, NP, SS, tw, t);
    } else {
      fft_units<N, false>(SF, NP, SS, tw, g, l, T / C::G);
    }
    __syncthreads();
    double2* XU = B.XU + (size_t)c * (SL ? B.l0 : N) * N * H;
    double2* XUn = B.XUn + (size_t)c * (SL ? B.l0 : N) * N;
    for (int idx = t; idx < NP * H; idx += T) {
      const int p = idx / H, k = idx % H;
      const double2 zk = SF[p * SS + C::kp(k)], zm = SF[p * SS + C::kp((N - k) & (N - 1))];
      XU[(row0 + 2 * p) * H + k] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
      XU[(row0 + 2 * p + 1) * H + k] = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
    }
    for (int p = t; p < NP; p += T) {
      const double2 z = SF[p * SS + C::kp(H)];
      XUn[row0 + 2 * p] = make_double2(z.x, 0.0);
      XUn[row0 + 2 * p + 1] = make_double2(z.y, 0.0);
    }
  }
}

// RS-fix, TMA-staged (single GPU, solid-only storage): the same map as
// k_rsfix_compact — X(u~') rows into XU when residual balancing changed b — with
// each tile's u rows, indicator bytes and solid u~ range brought in by bulk copies
// on an mbarrier and the next tile's copies issued as soon as the current tile has
// been packed into its sequences.  The per-voxel global gathers of k_rsfix_compact
// ran an active RS-fix at 0.45 ms at 256^3 (about 2 TB/s); it fires in about 6 % of
// the iterations of an adaptive solve (17 of 300 in the bench window).
template <int N>
struct RSFX {
  using K = RS2<N>;
  static constexpr size_t bytes(int cs) {
    return K::TW + K::INV + sizeof(double) * K::V + sizeof(double) * (size_t)cs + K::HB + 16;
  }
};

template <int N>
__global__ void __launch_bounds__(RS2<N>::T) k_rsfix_tma(Bufs B, const double* __restrict__ u,
                                                         const uint8_t* __restrict__ Hs, Compact cp,
                                                         const Ctrl* __restrict__ ctrl) {
  using C = Cfg<N>;
  using K = RS2<N>;
  constexpr int H = C::H, SS = C::SS, R = K::R, T = K::T, V = K::V, NP = K::NP;
  constexpr int TPC = N * N / R, NT = 3 * TPC;
  constexpr int SG = V / 1024;
  static_assert(T % 32 == 0, "segment bases are per warp");
  if (V != 1024 && V != 2048) return;
  pdl_wait();
  if (ctrl->done || ctrl->db == 0.0) return;
  extern __shared__ __align__(128) unsigned char sraw[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t ros[2][R + 1];
  double2* tw = (double2*)sraw;
  double2* SF = (double2*)(sraw + K::TW);
  double* su = (double*)(sraw + K::TW + K::INV);
  double* sc = su + V;
  uint8_t* sh = (uint8_t*)(sc + cp.cs);
  const int t = threadIdx.x, g = t / C::G, l = t % C::G, lane = t & 31;
  for (int j = t; j < C::TWN; j += T) tw[j] = B.tw[j];
  const int64_t n = (int64_t)N * N * N;
  uint32_t ro[R + 1];
  auto offs = [&](int tl) {
    const int64_t r0 = (int64_t)(tl % TPC) * R;
#pragma unroll
    for (int r = 0; r <= R; ++r) ro[r] = cp.off[r0 + r];
  };
  auto issue = [&](int tl, uint32_t* slot) {  // thread 0: u rows, H bytes, solid u~ range of tile tl
    const int c = tl / TPC;
    const int64_t row0 = (int64_t)(tl % TPC) * R;
    const uint32_t cb = sizeof(double) * (ro[R] - ro[0]);
    for (int r = 0; r <= R; ++r) slot[r] = ro[r];
    fence_async_smem();
    mbar_expect(&mbar, (uint32_t)(sizeof(double) * V + K::HB) + cb);
    bulk_load(su, u + (int64_t)c * n + row0 * N, sizeof(double) * V, &mbar);
    bulk_load(sh, Hs + row0 * N, (uint32_t)K::HB, &mbar);
    if (cb) bulk_load(sc, cp.ut + (int64_t)c * cp.ns + ro[0], cb, &mbar);
  };
  if (t == 0) {
    mbar_init(&mbar);
    if ((int)blockIdx.x < NT) {
      offs(blockIdx.x);
      issue(blockIdx.x, ros[0]);
    }
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < NT; tile += gridDim.x, phase ^= 1u) {
    const int c = tile / TPC;
    const int64_t row0 = (int64_t)(tile % TPC) * R;
    const bool has_next = tile + (int)gridDim.x < NT;
    if (t == 0 && has_next) offs(tile + gridDim.x);
    mbar_wait(&mbar, phase);
    const uint32_t o0 = ros[phase][0];
    int sb[2 > SG ? 2 : SG];
#pragma unroll
    for (int q = 0; q < SG; ++q) sb[q] = seg_base<N>(sh + q * 1024 + lane * 32, ros[phase][(q * 1024 + lane * 32) / N] - o0, lane);
    for (int j = 0; j < K::VPT; ++j) {
      const int v = t + T * j, row = v / N, col = v % N;
      const bool solid = sh[v] != 0;
      const unsigned mask = __ballot_sync(0xffffffffu, solid);
      const int segb = __shfl_sync(0xffffffffu, (SG == 1 || (v >> 10) == 0) ? sb[0] : sb[1], (v >> 5) & 31);
      double val = su[v];  // pore: u~' = u'
      if (solid) val = sc[segb + __popc(mask & ((1u << lane) - 1u))];
      reinterpret_cast<double*>(SF + (row >> 1) * SS + C::sp(col))[row & 1] = val;
    }
    __syncthreads();  // staged inputs consumed: the next tile's copies go out under the FFT
    if (t == 0 && has_next) issue(tile + gridDim.x, ros[phase ^ 1u]);
    if constexpr (C::M > 1) {
      radix_stage<N, false>(SF, NP, SS, tw, t, T);
      __syncthreads();
    }
    if constexpr (PF_RS_W32 && C::L == 256 && T == 32 * NP * C::M) {
      fft_units_w32<N, false>(SF, NP, SS, tw, t);
    } else {
      fft_units<N, false>(SF, NP, SS, tw, g, l, T / C::G);
    }
    __syncthreads();
    double2* XU = B.XU + (size_t)c * N * N * H;
    double2* XUn = B.XUn + (size_t)c * N * N;
    for (int idx = t; idx < NP * H; idx += T) {
      const int p = idx / H, k = idx % H;
      const double2 zk = SF[p * SS + C::kp(k)], zm = SF[p * SS + C::kp((N - k) & (N - 1))];
      XU[(row0 + 2 * p) * H + k] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
      XU[(row0 + 2 * p + 1) * H + k] = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
    }
    for (int p = t; p < NP; p += T) {
      const double2 z = SF[p * SS + C::kp(H)];
      XUn[row0 + 2 * p] = make_double2(z.x, 0.0);
      XUn[row0 + 2 * p + 1] = make_double2(z.y, 0.0);
    }
    __syncthreads();  // SF is rewritten by the next tile
  }
}

// ---- compact layout setup / teardown (warp per row of N voxels)
// largest padded solid count of any RS tile -> mx (zeroed by the caller)
template <int N>
__global__ void k_tile_max(const uint32_t* __restrict__ off, uint32_t* __restrict__ mx, int64_t rows) {
  constexpr int R = RS2<N>::R;
  const int64_t tiles = rows / R;
  uint32_t m = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tiles; t += (int64_t)gridDim.x * blockDim.x)
    m = max(m, off[(t + 1) * R] - off[t * R]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

template <int N>
__global__ void k_row_counts(const uint8_t* __restrict__ Hs, uint32_t* __restrict__ cnt, int64_t rows) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int c = 0;
    for (int k = lane; k < N; k += 32) c += Hs[r * N + k] != 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[r] = (uint32_t)((c + 1) & ~1);  // pad to even: 16-byte aligned rows
  }
}

// single-block exclusive scan of n counts -> off[0..n]
__global__ void __launch_bounds__(1024) k_scan(const uint32_t* __restrict__ cnt, uint32_t* __restrict__ off, int64_t n) {
  __shared__ uint32_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024, lo = t * per, hi = lo + per < n ? lo + per : n;
  uint32_t s = 0;
  for (int64_t i = lo; i < hi; ++i) s += cnt[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    uint32_t run = 0;
    for (int k = 0; k < 1024; ++k) {
      const uint32_t v = part[k];
      part[k] = run;
      run += v;
    }
    off[n] = run;
  }
  __syncthreads();
  uint32_t run = part[t];
  for (int64_t i = lo; i < hi; ++i) {
    off[i] = run;
    run += cnt[i];
  }
}

// dir = 0: gather full -> compact (solid voxels); dir = 1: scatter compact -> full,
// with pore u~ = u, a = 0 and lam left untouched.
template <int N>
__global__ void k_compact_move(const uint8_t* __restrict__ Hs, Compact cp, double* ut, double* a, double* lam,
                               const double* __restrict__ u, int dir, int64_t rows) {
  const int lane = threadIdx.x & 31;
  const int64_t n = rows * N;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < 3 * rows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int c = (int)(r / rows);
    const int64_t row = r % rows;
    int base = (int)cp.off[row];
    for (int k0 = 0; k0 < N; k0 += 32) {
      const int64_t x = row * N + k0 + lane;
      const bool solid = Hs[x] != 0;
      const unsigned mask = __ballot_sync(0xffffffffu, solid);
      const int64_t ci = (int64_t)c * cp.ns + base + __popc(mask & ((1u << lane) - 1u));
      const int64_t fi = (int64_t)c * n + x;
      if (dir == 0) {
        if (solid) {
          cp.ut[ci] = ut[fi];
          cp.a[ci] = a[fi];
          cp.lam[ci] = lam[fi];
        }
      } else {
        if (solid) {
          ut[fi] = cp.ut[ci];
          a[fi] = cp.a[ci];
          lam[fi] = cp.lam[ci];
        } else {
          ut[fi] = u[fi];
          a[fi] = 0.0;
        }
      }
      base += __popc(mask);
    }
  }
}

// pore sums: |a| (eligibility: must be 0) and lam^2 (constant contribution to |lam'|)
__global__ void __launch_bounds__(kThreads) k_pore_a_lam(int64_t n, const uint8_t* __restrict__ Hs,
                                                         const double* __restrict__ a, const double* __restrict__ lam,
                                                         double* __restrict__ part) {
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * n; i += (int64_t)gridDim.x * blockDim.x) {
    if (Hs[i % n] == 0) {
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

// ------------------------------------------------------------------ MF / MI
// Axis-1 pencils, one component per block (tile = (c, i0, 8 columns of k2) or a
// Nyquist tile of 8 rows i0).  All staged loads are 16-byte LDGSTS issued up
// front straight into the padded FFT sequences, so a block has its whole tile
// in flight at once; several blocks per SM overlap load and compute phases.
//   FWD: X-space R = b u~' - a' (+ (b' - b) u~' when residual balancing changed b)
//        -> Y-space R~ = FFT_1(b' u~' - a')
//   INV: Y-space U^ -> X-space u'                                 (IFFT_1)
template <int N>
struct PK2 {
  using C = Cfg<N>;
  static constexpr int T = N == 512 ? PF_PK512_T : (N == 1024 ? PF_PK1024_T : (N == 64 ? PF_PK64_T : PF_PK_THREADS));
  static constexpr int MINB = N == 512 ? PF_PK512_MINB : (N == 1024 ? PF_PK1024_MINB : (N == 128 ? PF_PK128_MINB : PF_PK_MINB));
  static constexpr int NGP = T / C::G;
  // 3 components x CP columns = NGP sequences: one FFT round per direction, no idle groups
#ifdef PF_PK_CP
  static constexpr int CP = PF_PK_CP;
#else
  // (a long sequence takes M groups: NGP / M sequences per round)
  static constexpr int CP = N == 512 ? PF_PK512_CP : (N == 1024 ? PF_PK1024_CP : (((NGP / C::M) % 3 == 0) ? NGP / C::M / 3 : NGP / C::M / 2));
#endif
  static constexpr int NSEQ = 3 * CP;
  static constexpr int NCH = C::H / CP;
  static constexpr int TILES = N * NCH + N / CP;
  static constexpr int MPT = (CP * N + T - 1) / T;  // modes per thread (last one guarded)
  // sequence stride with an 8-bank shift: the (q fastest, 4 columns) staging
  // pattern of 8-lane phases is then conflict-free
  static constexpr int SS = C::SS + 1;
  // TMA path (single GPU, N = 128 / 256, main tiles): each component's CP x N
  // pencil lands 64B-swizzled; the three boxes sit at the END of the padded
  // sequence region so the first FFT round's stores never reach the last box
  // (CP = 8: 128-byte box rows, SWIZZLE_128B)
  static constexpr int ROWB = CP * 16;  // box row bytes
  static constexpr bool TMA_OK = ((N == 128 || N == 256) && (ROWB == 64 || ROWB == 128)) || (N == 512 && ROWB == 64) ||
                                 (N == 1024 && (ROWB == 16 || ROWB == 32));
  static constexpr size_t REGION = sizeof(double2) * NSEQ * SS;
  static constexpr size_t BOX = sizeof(double2) * CP * N;
  static constexpr size_t BOX_AL = ROWB == 128 ? 1024 : 512;  // swizzle-atom alignment of a box
  static constexpr size_t BOX_OFF = ((REGION - 3 * BOX) / BOX_AL) * BOX_AL;
  // the last box must lie beyond what the first FFT round stores (NGP sequences)
  static_assert(!TMA_OK || C::M > 1 || NSEQ <= NGP || BOX_OFF + (NSEQ / CP - 1) * BOX >= sizeof(double2) * NGP * SS,
                "PK TMA boxes overlap the first round's sequences");
  // long sequences: component c's sequences, written after its boxes are read,
  // must not reach the boxes of component c + 1
  static_assert(!TMA_OK || C::M == 1 || (sizeof(double2) * CP * SS <= BOX_OFF + BOX &&
                                         sizeof(double2) * 2 * CP * SS <= BOX_OFF + 2 * BOX),
                "PK TMA boxes overlap the sequences of the previous component");
  static constexpr size_t BYTES = REGION + sizeof(double2) * C::TWN + 1024;
};

template <int N>
struct M2 {
  using C = Cfg<N>;
  static constexpr int T = N == 64 ? PF_M64_T : 128;
  static constexpr int NGM = T / C::G;        // groups = block transforms per tile
  static constexpr int CM = NGM / C::M;       // columns (sequences) per tile
  static constexpr int NCH = C::H / CM;
  static constexpr int TPC = N * NCH + N / CM;  // tiles per component
  static constexpr int TILES = 3 * TPC;
  static constexpr size_t SEQ = sizeof(double2) * CM * C::SS;
  // TMA path (single GPU, N = 128 / 256, main tiles): the CM x N tile lands
  // 128B-swizzled in a 1 KB-aligned region that the padded sequences then reuse
  // (N = 512: 64-byte rows, two 256-row boxes, single GPU only)
  static constexpr bool TMA_OK = ((N == 128 || N == 256) && CM * 16 == 128) || (N == 512 && CM * 16 == 64) ||
                                 (N == 1024 && CM * 16 == 32);
  static constexpr int ROWB = CM * 16;
  static constexpr size_t TILE = sizeof(double2) * CM * N;
  static constexpr size_t REGION = SEQ > TILE ? SEQ : TILE;
  static constexpr size_t BYTES_INV = sizeof(double2) * C::TWN + REGION + 1024;
  static constexpr size_t BYTES_FWD = BYTES_INV;
};

template <int N, bool INV, bool SL>
__global__ void __launch_bounds__(M2<N>::T, PF_M_MINB) k_maxis(Bufs B, const Ctrl* __restrict__ ctrl,
                                                             const __grid_constant__ CUtensorMap tmap, int nyq_only,
                                                             const __grid_constant__ CUtensorMap tmap_xu) {
  using C = Cfg<N>;
  using K = M2<N>;
  constexpr int H = C::H, SS = C::SS, CM = K::CM, NCH = K::NCH, T = K::T;
  pdl_wait();
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char msraw[];
  // 1 KB-aligned region (TMA tile / padded sequences), twiddles after it
  unsigned char* reg = msraw + ((1024 - (su32(msraw) & 1023)) & 1023);
  double2* S = (double2*)reg;
  double2* tw = (double2*)(reg + K::REGION);
  const int t = threadIdx.x, g = t / C::G, l = t % C::G;
  const int l0 = (SL ? B.l0 : N), l1 = (SL ? B.l1 : N), s1 = (SL ? B.s1 : Cfg<N>::LOGN);
  const int nl = SL ? B.nl : N, i0a = SL ? B.i0a : 0;  // plane window of this launch
  const int TPC = nl * NCH + nl / CM;  // tiles per component over the window
  // nyq_only (beside k_m1_pipe): block -> (component, Nyquist tile)
  const int c = (SL ? B.c0 : 0) + (nyq_only ? blockIdx.x / (nl / CM) : blockIdx.x / TPC);
  const int tile = nyq_only ? nl * NCH + blockIdx.x % (nl / CM) : blockIdx.x % TPC;
  const bool nyq = tile >= nl * NCH;
  const int i0 = nyq ? 0 : i0a + tile / NCH, ch = nyq ? 0 : tile % NCH;  // i0: local plane
  const int i0b = nyq ? i0a + (tile - nl * NCH) * CM : 0;
  // X (x-slab rows [c][l0 N][H], Nyquist [c][l0 N]); e = k1 (MI out / MF in) or i1
  auto off_of = [&](int e, int q) -> size_t {
    return nyq ? (size_t)(c * l0 + i0b + q) * N + e : ((size_t)(c * l0 + i0) * N + e) * H + ch * CM + q;
  };
  // Y in the x-slab exchange layout [r][i0][c][k1 - r l1][k2], r = k1 / l1 (see Bufs)
  auto yoff_of = [&](int e, int q) -> size_t {
    const int r = e >> s1, kl = e & (l1 - 1);
    if (!SL && !nyq && B.yb) return ymain<N>(1, c, i0, e, ch * CM + q);
    return nyq ? ((size_t)((r * l0 + i0b + q) * 3 + c)) * l1 + kl
               : (((size_t)((c * (N >> s1) + r) * l0 + i0)) * l1 + kl) * H + ch * CM + q;
  };
  constexpr bool TMA = K::TMA_OK && PF_M_TMA;
  if (TMA && !nyq && B.tma && (!(SL && INV) || B.tma_yx)) {
    // one 2D bulk tensor copy of the (N rows x CM columns) tile, 128B-swizzled
    // (long sequences: M copies of 256 rows, 64B-swizzled)
    __shared__ uint64_t mbar;
    if (t == 0) {
      mbar_init(&mbar);
      mbar_expect(&mbar, (uint32_t)K::TILE);
      const int x0 = 2 * ch * CM;  // doubles
      if (C::M > 1 && !(SL && INV)) {
#pragma unroll
        for (int b = 0; b < C::M; ++b) {
          const int y0 = (c * l0 + i0) * N + b * C::L;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
              "[%4];" ::"r"(su32(reg + b * C::L * K::ROWB)),
              "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0), "r"(y0), "r"(su32(&mbar))
              : "memory");
        }
      } else if (SL && INV) {
        // x-slab Y [c][r][i0][k1 - r l1][k2]: a 5D box (16 doubles, l1, 1, P, 1) whose
        // rows come out in k1 = r l1 + kl order
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
            "%6}], [%7];" ::"r"(su32(S)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0), "r"(0), "r"(i0), "r"(0), "r"(c), "r"(su32(&mbar))
            : "memory");
      } else if (!SL && INV && B.yb) {
        // i0-blocked Y [c i0/4][k1][i0%4][k2]: a 4D box (2 CM doubles, 1, N rows k1, 1)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
            "%5}], [%6];" ::"r"(su32(S)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0), "r"(i0 & 3), "r"(0), "r"(c * (N / 4) + (i0 >> 2)),
            "r"(su32(&mbar))
            : "memory");
      } else {
        const int y0 = (c * l0 + i0) * N;  // rows of [c][i0][e] (Y at P = 1, or X)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(S)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0), "r"(y0), "r"(su32(&mbar))
            : "memory");
      }
    }
    for (int j = t; j < Cfg<N>::TWN; j += T) tw[j] = B.tw[j];
    __syncthreads();
    mbar_wait(&mbar, 0);
    constexpr int A = C::A, BB = C::B;
    const unsigned char* tile = reg;
    // 16-byte chunk q of tile row e (64B swizzle: chunk ^ (e / 2) mod 4; 128B: ^ e mod 8)
    auto at = [&](int e, int q) -> double2 {
      const int sw = swz16<K::ROWB>(e);
      return *reinterpret_cast<const double2*>(tile + (size_t)e * K::ROWB + ((q ^ sw) << 4));
    };
    if constexpr (C::M > 1) {
      if (INV) {
        // block transform unit g = (column q, block r): its elements are rows e = M p + r
        const int q = g / C::M, r = g % C::M;
        double2 x[A > BB ? A : BB];
        if (l < BB) {
#pragma unroll
          for (int n1 = 0; n1 < A; ++n1) x[n1] = at(C::M * (BB * n1 + l) + r, q);
        }
        __syncthreads();  // the tile is read
        fft_seq_x<C::L, true>(x, S + q * SS + r * C::SSL, tw, l, true);
        __syncthreads();
        radix_stage<N, true>(S, CM, SS, tw, t, T);
      } else {
        // forward: the radix-M stage straight from the tile into registers, then
        // into the padded sequences once every thread has read its rows
        constexpr int IT = CM * C::L / T;
        static_assert(CM * C::L % T == 0, "radix items per thread");
        double2 a[IT][C::M];
        const double db = ctrl->db;
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          const int idx = t + T * it, q = idx % CM, j = idx / CM;
#pragma unroll
          for (int b = 0; b < C::M; ++b) {
            a[it][b] = at(j + C::L * b, q);
            if (db != 0.0) {  // rare: b changed this iteration; XU holds X(u~') (k_rsfix)
              const double2 vu = B.XU[off_of(j + C::L * b, q)];
              a[it][b] = make_double2(a[it][b].x + db * vu.x, a[it][b].y + db * vu.y);
            }
          }
          Dft<C::M, false>::run(a[it]);
          radix_twiddle<N, false>(a[it], tw, j);
        }
        __syncthreads();  // the tile is read
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          const int idx = t + T * it, q = idx % CM, j = idx / CM;
#pragma unroll
          for (int b = 0; b < C::M; ++b) S[q * SS + b * C::SSL + C::pad(j)] = a[it][b];
        }
        __syncthreads();
        fft_units<N, false>(S, CM, SS, tw, g, l, K::NGM);
      }
      __syncthreads();
    } else {
    double2 x[A > BB ? A : BB];
    const double db = INV ? 0.0 : ctrl->db;
    if (l < BB) {
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) {
        const int e = BB * n1 + l;  // row e, column g: chunk g of the row, XOR-swizzled by e mod 8
        x[n1] = *reinterpret_cast<const double2*>(tile + (size_t)e * 128 + ((g ^ (e & 7)) << 4));
      }
    }
    if (!INV && db != 0.0 && !SL && !nyq) {
      // rare: b changed this iteration; X(u~') (k_rsfix) comes in as a second TMA tile
      // into the same region once the first has been read
      __syncthreads();
      if (t == 0) {
        fence_async_smem();
        mbar_expect(&mbar, (uint32_t)K::TILE);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(S)),
            "l"(reinterpret_cast<uint64_t>(&tmap_xu)), "r"(2 * ch * CM), "r"((c * l0 + i0) * N), "r"(su32(&mbar))
            : "memory");
      }
      mbar_wait(&mbar, 1);
      if (l < BB) {
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) {
          const int e = BB * n1 + l;
          const double2 vu = *reinterpret_cast<const double2*>(tile + (size_t)e * 128 + ((g ^ (e & 7)) << 4));
          x[n1] = make_double2(x[n1].x + db * vu.x, x[n1].y + db * vu.y);
        }
      }
    } else if (!INV && db != 0.0 && l < BB) {  // rare, slab layouts: per-element reads of X(u~')
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) {
        const double2 vu = B.XU[off_of(BB * n1 + l, g)];
        x[n1] = make_double2(x[n1].x + db * vu.x, x[n1].y + db * vu.y);
      }
    }
    __syncthreads();  // the tile is read: the padded sequences may now overwrite it
    fft_seq_x<N, INV>(x, S + g * SS, tw, l, true);
    __syncthreads();
    }
  } else {
  // element mapping: main tiles walk (e, q) with q fastest (contiguous columns);
  // Nyquist tiles walk (q, e) with e fastest (contiguous rows).
  for (int idx = t; idx < N * CM; idx += T) {
    const int q = nyq ? idx / N : idx % CM, e = nyq ? idx % N : idx / CM;
    if (INV) {
      const size_t o = yoff_of(e, q);
      cp16(S + q * SS + C::kp(e), nyq ? B.Yxn + o : B.Yx + o);
    } else {
      const size_t o = off_of(e, q);
      cp16(S + q * SS + C::sp(e), nyq ? B.XRn + o : B.XR + o);
    }
  }
  for (int j = t; j < Cfg<N>::TWN; j += T) tw[j] = B.tw[j];
  cp_commit_wait_all();
  __syncthreads();
  if (!INV) {
    const double db = ctrl->db;
    if (db != 0.0) {  // rare: b changed this iteration; XU holds X(u~') (k_rsfix)
      for (int idx = t; idx < N * CM; idx += T) {
        const int q = nyq ? idx / N : idx % CM, e = nyq ? idx % N : idx / CM;
        const size_t o = off_of(e, q);
        const double2 vu = nyq ? B.XUn[o] : B.XU[o];
        double2* p = S + q * SS + C::sp(e);
        *p = make_double2(p->x + db * vu.x, p->y + db * vu.y);
      }
      __syncthreads();
    }
  }
  if constexpr (C::M > 1) {
    if (!INV) {
      radix_stage<N, false>(S, CM, SS, tw, t, T);
      __syncthreads();
    }
    fft_units<N, INV>(S, CM, SS, tw, g, l, K::NGM);
    if (INV) {
      __syncthreads();
      radix_stage<N, true>(S, CM, SS, tw, t, T);
    }
  } else {
    fft_seq<N, INV>(S + g * SS, tw, l, true);
  }
  __syncthreads();
  }
  for (int idx = t; idx < N * CM; idx += T) {
    const int q = nyq ? idx / N : idx % CM, e = nyq ? idx % N : idx / CM;
    const double2 v = S[q * SS + (INV ? C::sp(e) : C::kp(e))];
    if (!INV) {
      if (SL && B.peers) {  // to the owner of k1: its y-slab Y [c][i0][k1 - k1off][k2], Yn [i0][c][k1 - k1off]
        const int r = e >> s1, kl = e & (l1 - 1);
        const int i0g = (B.k1off >> s1) * l0 + (nyq ? i0b + q : i0);
        if (nyq) B.peers->yyn[r][(size_t)(i0g * 3 + c) * l1 + kl] = v;
        else B.peers->yy[r][((size_t)(c * N + i0g) * l1 + kl) * H + ch * CM + q] = v;
      } else {
        const size_t o = yoff_of(e, q);
        if (nyq) B.Yxn[o] = v; else B.Yx[o] = v;
      }
    } else {
      const size_t o = off_of(e, q);
      if (nyq) B.XUn[o] = v; else B.XU[o] = v;
    }
  }
}

// ------------------------------------------------------------------ MI / MF, persistent pipelined
// Single GPU, N = 128 / 256 (M = 1), main tiles; the Nyquist tiles stay on k_maxis
// (nyq_only).  One CTA walks the tiles blockIdx.x, + gridDim.x, ... with a two-stage
// TMA ring: tile i + 2's copy is issued into stage i & 1 as soon as tile i has been
// read into registers, so a tile's load latency and the CTA's per-tile setup
// (twiddle table, mbarrier) are paid once per CTA instead of per tile — at 128^3
// the non-persistent passes run at about half their 256^3 bandwidth.
template <int N>
struct MP {
  using C = Cfg<N>;
  static constexpr int T = M2<N>::T, CM = M2<N>::CM, NCH = M2<N>::NCH;
  static constexpr int ROWB = CM * 16;
  static constexpr size_t TILE = sizeof(double2) * CM * N;
  static constexpr size_t SEQ = sizeof(double2) * CM * C::SS;
  static constexpr int STAGES = PF_MP_STAGES;
  static constexpr int MINB = PF_MP_MINB;
  static constexpr size_t BYTES = 1024 + STAGES * TILE + SEQ + sizeof(double2) * C::TWN;
  static constexpr int UNITS = 3 * N * NCH;  // main tiles of the three components
  static_assert(C::M == 1 && ROWB == 128, "pipelined axis-1 pass: N <= 256, 128-byte rows");
  static_assert(TILE % 1024 == 0, "stages stay 1 KB aligned");
};

template <int N, bool INV>
__global__ void __launch_bounds__(MP<N>::T, MP<N>::MINB) k_m1_pipe(Bufs B, const Ctrl* __restrict__ ctrl,
                                                         const __grid_constant__ CUtensorMap tmap,
                                                         const __grid_constant__ CUtensorMap tmap_xu) {
  using C = Cfg<N>;
  using K = MP<N>;
  constexpr int H = C::H, SS = C::SS, CM = K::CM, NCH = K::NCH, T = K::T, NU = K::UNITS;
  pdl_wait();
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char mpraw[];
  unsigned char* base = mpraw + ((1024 - (su32(mpraw) & 1023)) & 1023);
  double2* S = (double2*)(base + K::STAGES * K::TILE);
  double2* tw = (double2*)(base + K::STAGES * K::TILE + K::SEQ);
  __shared__ uint64_t full[K::STAGES];
  __shared__ uint64_t xbar;  // X(u~') tile (FWD, only when b changed this iteration)
  const int t = threadIdx.x, g = t / C::G, l = t % C::G;
  const double db = INV ? 0.0 : ctrl->db;

  auto issue = [&](int u, int s) {
    const int c = u / (N * NCH), r = u % (N * NCH), i0 = r / NCH, ch = r % NCH;
    unsigned char* dst = base + (size_t)s * K::TILE;
    fence_async_smem();
    mbar_expect(&full[s], (uint32_t)K::TILE);
    if (INV && B.yb) {
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
          "%5}], [%6];" ::"r"(su32(dst)),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * ch * CM), "r"(i0 & 3), "r"(0), "r"(c * (N / 4) + (i0 >> 2)),
          "r"(su32(&full[s]))
          : "memory");
    } else {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(dst)),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * ch * CM), "r"((c * N + i0) * N), "r"(su32(&full[s]))
          : "memory");
    }
  };

  if (t == 0) {
    for (int s = 0; s < K::STAGES; ++s) mbar_init(&full[s]);
    mbar_init(&xbar);
    for (int s = 0; s < K::STAGES; ++s)
      if ((int)blockIdx.x + s * (int)gridDim.x < NU) issue(blockIdx.x + s * gridDim.x, s);
  }
  for (int j = t; j < C::TWN; j += T) tw[j] = B.tw[j];
  __syncthreads();
  int it = 0;
  for (int u = blockIdx.x; u < NU; u += gridDim.x, ++it) {
    const int s = it % K::STAGES;
    const int c = u / (N * NCH), r = u % (N * NCH), i0 = r / NCH, ch = r % NCH;
    const unsigned char* tile = base + (size_t)s * K::TILE;
    mbar_wait(&full[s], (it / K::STAGES) & 1);
    constexpr int A = C::A, BB = C::B;
    double2 x[A > BB ? A : BB];
    if (l < BB) {
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) {
        const int e = BB * n1 + l;  // row e, column g: chunk g of the row, XOR-swizzled by e mod 8
        x[n1] = *reinterpret_cast<const double2*>(tile + (size_t)e * 128 + ((g ^ (e & 7)) << 4));
      }
    }
    if (!INV && db != 0.0) {  // rare: b changed this iteration; X(u~') (k_rsfix) as a TMA tile into S
      if (t == 0) {
        fence_async_smem();
        mbar_expect(&xbar, (uint32_t)K::TILE);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(S)),
            "l"(reinterpret_cast<uint64_t>(&tmap_xu)), "r"(2 * ch * CM), "r"((c * N + i0) * N), "r"(su32(&xbar))
            : "memory");
      }
      mbar_wait(&xbar, it & 1);
      const unsigned char* xu = reinterpret_cast<const unsigned char*>(S);
      if (l < BB) {
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) {
          const int e = BB * n1 + l;
          const double2 vu = *reinterpret_cast<const double2*>(xu + (size_t)e * 128 + ((g ^ (e & 7)) << 4));
          x[n1] = make_double2(x[n1].x + db * vu.x, x[n1].y + db * vu.y);
        }
      }
    }
    __syncthreads();  // stage s read: refill it two grid strides ahead
    if (t == 0 && u + K::STAGES * (int)gridDim.x < NU) issue(u + K::STAGES * gridDim.x, s);
    fft_seq_x<N, INV>(x, S + g * SS, tw, l, true);
    __syncthreads();
    for (int idx = t; idx < N * CM; idx += T) {
      const int q = idx % CM, e = idx / CM;
      const double2 v = S[q * SS + (INV ? C::sp(e) : C::kp(e))];
      if (INV) B.XU[((size_t)(c * N + i0) * N + e) * H + ch * CM + q] = v;
      else B.Y[ymain<N>(B.yb, c, i0, e, ch * CM + q)] = v;
    }
    __syncthreads();  // S is rewritten by the next tile
  }
}

// ------------------------------------------------------------------ PK
struct SpecArgs {
  const double* kap[3];
  const double* ell[3];
  double nu, g[3], inv_n, dn;
};

// Axis-0 pencils: tile = (k1, CP columns of k2) or a Nyquist tile of CP values
// of k1, all k0, three components.  Y-space loads are LDGSTS straight into the
// padded sequences; Q^ and D^ live in tile-major order ([tile][q][k0]) so the
// spectral step reads and writes them fully coalesced, prefetched into
// registers before the forward FFTs.

template <int N, bool SL>
__global__ void __launch_bounds__(PK2<N>::T, PK2<N>::MINB) k_pk(Bufs B, SpecArgs P, const Ctrl* __restrict__ ctrl,
                                                              const __grid_constant__ CUtensorMap tmap, int tile0,
                                                              int pbase, int nparts) {
  using C = Cfg<N>;
  using K = PK2<N>;
  constexpr int H = C::H, SS = K::SS, CP = K::CP, NCH = K::NCH, NSEQ = K::NSEQ, T = K::T;
  pdl_wait();
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char psraw[];
  unsigned char* reg = psraw + ((1024 - (su32(psraw) & 1023)) & 1023);  // 1 KB-aligned
  double2* S = (double2*)reg;
  double2* tw = (double2*)(reg + K::REGION);
  const int t = threadIdx.x, g = t / C::G, l = t % C::G;
  const double beta = ctrl->beta, b = ctrl->b;
  const int tile = tile0 + blockIdx.x;  // (tile0 > 0: the Nyquist tiles beside k_pk_pipe)
  const int l1 = (SL ? B.l1 : N);
  const bool nyq = tile >= l1 * NCH;
  const int k1 = nyq ? 0 : tile / NCH, ch = nyq ? 0 : tile % NCH;  // k1: local to the y-slab
  const int k1b = nyq ? (tile - l1 * NCH) * CP : 0;
  // Y in the y-slab exchange layout [i0][c][k1 - k1off][k2] (see Bufs)
  auto yoff = [&](int c, int i0, int q) -> size_t {
    if (!SL && !nyq && B.yb) return ymain<N>(1, c, i0, k1, ch * CP + q);
    return nyq ? (size_t)(i0 * 3 + c) * l1 + k1b + q : ((size_t)(c * N + i0) * l1 + k1) * H + ch * CP + q;
  };
  constexpr bool TMA = K::TMA_OK && PF_PK_TMA;
  const bool tma = TMA && !nyq && B.tma;
  __shared__ uint64_t mbar;
  if (tma) {
    if (t == 0) {  // three 3D tensor copies: component c's (CP columns x N rows i0) pencil
      mbar_init(&mbar);
      mbar_expect(&mbar, (uint32_t)(3 * K::BOX));
      if constexpr (C::M > 1) {  // (long sequences: M copies of 256 rows per component)
        for (int c = 0; c < 3; ++c)
          for (int b = 0; b < C::M; ++b)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4}], [%5];" ::"r"(su32(reg + K::BOX_OFF + c * K::BOX + b * C::L * K::ROWB)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * ch * CP), "r"(k1), "r"(c * N + b * C::L),
                "r"(su32(&mbar))
                : "memory");
      } else if (!SL && B.yb) {  // i0-blocked Y: 4D box (2 CP doubles, 4, 1, N / 4) -> rows in i0 order
        for (int c = 0; c < 3; ++c)
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
              "%5}], [%6];" ::"r"(su32(reg + K::BOX_OFF + c * K::BOX)),
              "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * ch * CP), "r"(0), "r"(k1), "r"(c * (N / 4)),
              "r"(su32(&mbar))
              : "memory");
      } else
      for (int c = 0; c < 3; ++c)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];" ::"r"(su32(reg + K::BOX_OFF + c * K::BOX)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * ch * CP), "r"(k1), "r"(c * N), "r"(su32(&mbar))
            : "memory");
    }
  } else {
    for (int idx = t; idx < 3 * N * CP; idx += T) {
      const int q = idx % CP, i0 = (idx / CP) % N, c = idx / (CP * N);
      const size_t o = yoff(c, i0, q);
      cp16(S + (c * CP + q) * SS + C::sp(i0), nyq ? B.Yn + o : B.Y + o);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const size_t tbase = (size_t)tile * CP * N;  // tile-major Q^, D^
#if PF_PK_PREFETCH
  double2 qv[K::MPT], dp[K::MPT];
#pragma unroll
  for (int j = 0; j < K::MPT; ++j) {
    const int m = t + T * j;
    if (m < CP * N) {
      qv[j] = B.Q[tbase + m];
      dp[j] = B.D[tbase + m];
    }
  }
#endif
  for (int j = t; j < Cfg<N>::TWN; j += T) tw[j] = B.tw[j];
  if (tma && C::M > 1) {
    __syncthreads();  // mbarrier initialised
    mbar_wait(&mbar, 0);
    // radix-M stage straight from the boxes, one component at a time: component
    // c's boxes into registers, then its sequences (which reach no later box)
    constexpr int IT = (CP * C::L + T - 1) / T;
    for (int c = 0; c < 3; ++c) {
      const unsigned char* box = reg + K::BOX_OFF + c * K::BOX;
      double2 a[IT][C::M];
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int idx = t + T * it, q = idx % CP, j = idx / CP;
        if (idx < CP * C::L) {
#pragma unroll
          for (int b = 0; b < C::M; ++b) {
            const int e = j + C::L * b;
            const int sw = swz16<K::ROWB>(e);
            a[it][b] = *reinterpret_cast<const double2*>(box + (size_t)e * K::ROWB + ((q ^ sw) << 4));
          }
          Dft<C::M, false>::run(a[it]);
          radix_twiddle<N, false>(a[it], tw, j);
        }
      }
      __syncthreads();  // component c's boxes are read
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int idx = t + T * it, q = idx % CP, j = idx / CP;
        if (idx < CP * C::L) {
#pragma unroll
          for (int b = 0; b < C::M; ++b) S[(c * CP + q) * SS + b * C::SSL + C::pad(j)] = a[it][b];
        }
      }
    }
    __syncthreads();
    fft_units<N, false>(S, NSEQ, SS, tw, g, l, K::NGP);
  } else if (tma) {
    __syncthreads();  // mbarrier initialised
    mbar_wait(&mbar, 0);
    constexpr int A = C::A, BB = C::B;
#pragma unroll
    for (int r = 0; r < (NSEQ + K::NGP - 1) / K::NGP; ++r) {
      const int sq = g + r * K::NGP;
      const bool act = sq < NSEQ;
      const int cc = act ? sq / CP : 0, q = act ? sq % CP : 0;
      const unsigned char* box = reg + K::BOX_OFF + cc * K::BOX;
      double2 x[A > BB ? A : BB];
      if (act && l < BB) {
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) {  // row e = i0, column q: 16B chunk XOR-swizzled by (e / 2) mod 4 (64B)
          const int e = BB * n1 + l;       // or by e mod 8 (128B)
          const int sw = swz16<K::ROWB>(e);
          x[n1] = *reinterpret_cast<const double2*>(box + (size_t)e * K::ROWB + ((q ^ sw) << 4));
        }
      }
      __syncthreads();  // this round's boxes are read before its stores may overwrite them
      fft_seq_x<N, false>(x, S + (act ? sq : 0) * SS, tw, l, act);
    }
  } else {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if constexpr (C::M > 1) {
      radix_stage<N, false>(S, NSEQ, SS, tw, t, T);
      __syncthreads();
    }
    fft_units<N, false>(S, NSEQ, SS, tw, g, l, K::NGP);
  }
  __syncthreads();
  double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < K::MPT; ++j) {
    const int m = t + T * j, q = m / N, k0 = m % N;
    if (m >= CP * N) break;
    const int kk1 = (SL ? B.k1off : 0) + (nyq ? k1b + q : k1), k2 = nyq ? H : ch * CP + q;  // global k1
    const int idx3[3] = {k0, kk1, k2};
    double kc[3];
    double L = 0.0, ksq = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      kc[c] = __ldg(P.kap[c] + idx3[c]);
      L = L + __ldg(P.ell[c] + idx3[c]);
      ksq = ksq + kc[c] * kc[c];
    }
#if PF_PK_PREFETCH
    const double2 qq = qv[j];
    const double2 dpj = dp[j];
#else
    const double2 qq = B.Q[tbase + m];
    const double2 dpj = B.D[tbase + m];
#endif
    const bool zero = (k0 | kk1 | k2) == 0;
    double2 r[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double2 rc = S[(c * CP + q) * SS + C::kp(k0)];
      r[c] = make_double2(kc[c] * qq.y + rc.x, -(kc[c] * qq.x) + rc.y);  // -i k q + R^
      if (zero) r[c].x = r[c].x + P.dn * P.g[c];                          // n g_p at k = 0
    }
    const double A = P.nu * L + b;
    double2 kr = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < 3; ++c) kr = cadd(kr, cscale(kc[c], r[c]));
    // one division: f = beta/(A + beta ksq) and 1/A from 1/(A (A + beta ksq))
    const double Dn = A + beta * ksq;
    const double rAD = 1.0 / (A * Dn);
    const double f = beta * A * rAD;
    const double2 corr = cscale(f, kr);
    const double invA = Dn * rAD;
    double2 dv = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double2 u = csub(r[c], cscale(kc[c], corr));
      u = make_double2(u.x * invA, u.y * invA);
      dv = cadd(dv, cik(kc[c], u));
      S[(c * CP + q) * SS + C::kp(k0)] = make_double2(u.x * P.inv_n, u.y * P.inv_n);
    }
    double2 qn = csub(qq, cscale(beta, dv));
    if (zero) qn = make_double2(0.0, 0.0);
    const double w = (k2 == 0 || k2 == H) ? 1.0 : 2.0;
    acc[0] += w * cabs2(dv);
    acc[1] += w * cabs2(csub(dv, dpj));
    acc[2] += w * cabs2(qn);
    B.Q[tbase + m] = qn;
    B.D[tbase + m] = dv;
  }
  __syncthreads();
  fft_units<N, true>(S, NSEQ, SS, tw, g, l, K::NGP);
  if constexpr (C::M > 1) {
    __syncthreads();
    radix_stage<N, true>(S, NSEQ, SS, tw, t, T);
  }
  __syncthreads();
#if PF_PK_TMASTORE
  if (!SL && tma && C::M == 1) {
    // Y out by TMA tensor stores: each component's results are repacked from the
    // padded sequences into its (swizzled) box, last component first — box c only
    // overlaps sequences of components >= c, already consumed — then one thread
    // stores the three boxes and waits until they have been read from shared memory.
    constexpr int PER = (CP * N + T - 1) / T;
    for (int c = 2; c >= 0; --c) {
      double2 v[PER];
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int idx = t + T * j, q = idx % CP, i0 = idx / CP;
        if (idx < CP * N) v[j] = S[(c * CP + q) * SS + C::sp(i0)];
      }
      __syncthreads();
      unsigned char* box = reg + K::BOX_OFF + c * K::BOX;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int idx = t + T * j, q = idx % CP, i0 = idx / CP;
        if (idx < CP * N)
          *reinterpret_cast<double2*>(box + (size_t)i0 * K::ROWB + ((q ^ swz16<K::ROWB>(i0)) << 4)) = v[j];
      }
    }
    fence_async_smem();
    __syncthreads();
    if (t == 0) {
      for (int c = 0; c < 3; ++c) {
        if (B.yb)
          asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                           reinterpret_cast<uint64_t>(&tmap)),
                       "r"(2 * ch * CP), "r"(0), "r"(k1), "r"(c * (N / 4)), "r"(su32(reg + K::BOX_OFF + c * K::BOX))
                       : "memory");
        else
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                           reinterpret_cast<uint64_t>(&tmap)),
                       "r"(2 * ch * CP), "r"(k1), "r"(c * N), "r"(su32(reg + K::BOX_OFF + c * K::BOX))
                       : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  } else
#endif
  for (int idx = t; idx < 3 * N * CP; idx += T) {
    const int q = idx % CP, i0 = (idx / CP) % N, c = idx / (CP * N);
    const size_t o = yoff(c, i0, q);
    const double2 v = S[(c * CP + q) * SS + C::sp(i0)];
    if (SL && B.peers) {  // to the owner of i0: its x-slab Y [c][r][i0l][k1 - r l1][k2], Yn [r][i0l][c][k1 - r l1]
      const int l0 = B.l0, me = B.k1off >> B.s1, r = i0 / l0, i0l = i0 - r * l0, P = N >> B.s1;
      const int kl = nyq ? k1b + q : k1;
      if (nyq) B.peers->yxn[r][((size_t)(me * l0 + i0l) * 3 + c) * l1 + kl] = v;
      else B.peers->yx[r][(((size_t)(c * P + me) * l0 + i0l) * l1 + kl) * H + ch * CP + q] = v;
    } else {
      if (nyq) B.Yn[o] = v; else B.Y[o] = v;
    }
  }
  block_sum<3>(acc);
  if (!SL && B.cpk && tile0 == 0 && (int)gridDim.x == nparts) {
    group_reduce<3>(acc, B.part_pk, nparts, B.gpk, B.cpk, PF_GRP_PK);
  } else if (t == 0) {
    for (int k = 0; k < 3; ++k) st_part(B.part_pk + (size_t)k * nparts + pbase + blockIdx.x, acc[k]);
  }
#if PF_PK_TMASTORE
  if (!SL && tma && C::M == 1 && t == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
}

// ------------------------------------------------------------------ PK, persistent pipelined
// Single GPU, N = 128 / 256, main tiles (the Nyquist tiles stay on k_pk).  One CTA
// per SM walks the tiles blockIdx.x, + gridDim.x, ... with a two-stage input ring:
// a stage holds the tile's three component pencils (3D TMA boxes, as k_pk) and its
// tile-major Q^ / D^ chunks (two 1D bulk copies), all completing on the stage's
// mbarrier.  The loads of tile i + 2 are issued into stage i & 1 as soon as tile
// i's spectral step has consumed it, so about one tile of reads is always in
// flight while the SM transforms — the non-persistent k_pk is bound by its per-tile
// load -> FFT -> spectral -> FFT -> store chain at 3 CTAs / SM.
// 12 lane groups of 16 transform the 3 x CP = 12 sequences in one round per
// direction; Q^' / D^ go out coalesced per thread, Y from the padded sequences.
#ifndef PF_PKP_CP
#define PF_PKP_CP 4  // columns per pipelined-PK work unit (2: half tiles, 96 threads, 2 CTAs / SM)
#endif
#ifndef PF_PKP_ABL
#define PF_PKP_ABL 0  // measurement-only ablations (results invalid): 1 = no Y stores, 2 = no FFTs, 3 = no Q/D stores
#endif
#ifndef PF_PKP_W32
#define PF_PKP_W32 0  // N = 256: one warp per sequence (fft256_w32) instead of a 16-lane group
#endif
template <int N>
struct PKP {
  using C = Cfg<N>;
  static constexpr int CPT = PK2<N>::CP;     // the tile-major Q^ / D^ tiles of k_pk
  static constexpr int CP = PF_PKP_CP;       // columns per work unit (a unit = CPT / CP of a tile)
  static constexpr int SPT = CPT / CP;       // units per tile
  static constexpr bool W32 = PF_PKP_W32 && N == 256;
  static constexpr int NSEQ = 3 * CP;
  static constexpr int LPS = W32 ? 32 : C::G;  // lanes per sequence
  static constexpr int T = NSEQ * LPS;       // one lane group (or warp) per sequence
  static constexpr int SS = PK2<N>::SS;
  static constexpr int ROWB = CP * 16;
  static constexpr size_t BOX = sizeof(double2) * CP * N;       // one component pencil
  static constexpr size_t QD = sizeof(double2) * CP * N;        // one unit's Q^ or D^ chunk
  static constexpr size_t STAGE = 3 * BOX + 2 * QD;
  static constexpr uint32_t TX = (uint32_t)STAGE;
  static constexpr int STAGES = 2;
  static constexpr size_t REGION = sizeof(double2) * NSEQ * SS;
  static constexpr size_t BYTES = 1024 + STAGES * STAGE + REGION + sizeof(double2) * C::TWN;
  static constexpr int MAIN_TILES = N * PK2<N>::NCH;
  static constexpr int UNITS = MAIN_TILES * SPT;
  static_assert(C::M == 1, "pipelined PK: N <= 256");
  static_assert(CPT % CP == 0 && (ROWB == 32 || ROWB == 64 || ROWB == 128), "pipelined PK unit shape");
  static_assert(BOX % 1024 == 0 && QD % 1024 == 0, "stage members stay 1 KB aligned");
};

template <int N>
__global__ void __launch_bounds__(PKP<N>::T, 1) k_pk_pipe(Bufs B, SpecArgs P, const Ctrl* __restrict__ ctrl,
                                                         const __grid_constant__ CUtensorMap tmap) {
  using C = Cfg<N>;
  using K = PKP<N>;
  constexpr int H = C::H, SS = K::SS, CP = K::CP, CPT = K::CPT, SPT = K::SPT, NCH = PK2<N>::NCH, T = K::T;
  constexpr int NU = K::UNITS, LPS = K::LPS;
  pdl_wait();
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char ppraw[];
  unsigned char* base = ppraw + ((1024 - (su32(ppraw) & 1023)) & 1023);  // 1 KB-aligned
  unsigned char* stage0 = base;
  double2* S = (double2*)(base + K::STAGES * K::STAGE);
  double2* tw = (double2*)(base + K::STAGES * K::STAGE + K::REGION);
  __shared__ uint64_t full[K::STAGES];
  const int t = threadIdx.x, g = t / LPS, l = t % LPS;
  const double beta = ctrl->beta, b = ctrl->b;

  auto issue = [&](int unit, int s) {  // thread 0: the unit's pencils + Q^ / D^ chunks into stage s
    unsigned char* st = stage0 + (size_t)s * K::STAGE;
    const int tile = unit / SPT, half = unit % SPT;
    const int k1 = tile / NCH, ch = tile % NCH;
    fence_async_smem();
    mbar_expect(&full[s], K::TX);
    for (int c = 0; c < 3; ++c) {
      if (B.yb)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
            "%5}], [%6];" ::"r"(su32(st + c * K::BOX)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * (ch * CPT + half * CP)), "r"(0), "r"(k1),
            "r"(c * (N / 4)), "r"(su32(&full[s]))
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];" ::"r"(su32(st + c * K::BOX)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * (ch * CPT + half * CP)), "r"(k1), "r"(c * N),
            "r"(su32(&full[s]))
            : "memory");
    }
    const size_t tb = (size_t)tile * CPT * N + (size_t)half * CP * N;
    bulk_load(st + 3 * K::BOX, B.Q + tb, (uint32_t)K::QD, &full[s]);
    bulk_load(st + 3 * K::BOX + K::QD, B.D + tb, (uint32_t)K::QD, &full[s]);
  };

  if (t == 0) {
    for (int s = 0; s < K::STAGES; ++s) mbar_init(&full[s]);
    for (int s = 0; s < K::STAGES; ++s) {
      const int unit = blockIdx.x + s * gridDim.x;
      if (unit < NU) issue(unit, s);
    }
  }
  for (int j = t; j < C::TWN; j += T) tw[j] = B.tw[j];
  __syncthreads();

  double acc[3] = {0.0, 0.0, 0.0};
  int it = 0;
  for (int unit = blockIdx.x; unit < NU; unit += gridDim.x, ++it) {
    const int s = it & 1;
    const unsigned char* st = stage0 + (size_t)s * K::STAGE;
    const double2* Qs = (const double2*)(st + 3 * K::BOX);
    const double2* Ds = (const double2*)(st + 3 * K::BOX + K::QD);
    const int tile = unit / SPT, half = unit % SPT;
    const int k1 = tile / NCH, ch = tile % NCH;
    const int col0 = ch * CPT + half * CP;  // first k2 column of the unit
    mbar_wait(&full[s], (it >> 1) & 1);
    {  // forward FFT_0, one sequence (c, q) per lane group / warp, pass-1 inputs straight from the box
      const int cc = g / CP, q = g % CP;
      const unsigned char* box = st + cc * K::BOX;
      auto ld = [&](int e) {
        return *reinterpret_cast<const double2*>(box + (size_t)e * K::ROWB + ((q ^ swz16<K::ROWB>(e)) << 4));
      };
      if constexpr (K::W32) {
        const int j = l & 15, h = l >> 4;
        double2 x[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) x[m] = ld(16 * (2 * m + h) + j);
        fft256_w32_x<false>(x, S + g * SS, tw, l, true);
      } else {
        constexpr int A = C::A, BB = C::B;
        double2 x[A > BB ? A : BB];
        if (l < BB) {
#pragma unroll
          for (int n1 = 0; n1 < A; ++n1) x[n1] = ld(BB * n1 + l);
        }
#if PF_PKP_ABL == 2
        if (l < BB)
          for (int n1 = 0; n1 < A; ++n1) S[g * SS + C::pad(BB * n1 + l)] = x[n1];
#else
        fft_seq_x<N, false>(x, S + g * SS, tw, l, true);
#endif
      }
    }
    __syncthreads();
    const size_t tbase = (size_t)tile * CPT * N + (size_t)half * CP * N;
    for (int m = t; m < CP * N; m += T) {
      const int q = m / N, k0 = m % N;
      const int kk1 = k1, k2 = col0 + q;
      const int idx3[3] = {k0, kk1, k2};
      double kc[3];
      double L = 0.0, ksq = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        kc[c] = __ldg(P.kap[c] + idx3[c]);
        L = L + __ldg(P.ell[c] + idx3[c]);
        ksq = ksq + kc[c] * kc[c];
      }
      const double2 qq = Qs[m];
      const double2 dpj = Ds[m];
      const bool zero = (k0 | kk1 | k2) == 0;
      double2 r[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double2 rc = S[(c * CP + q) * SS + C::kp(k0)];
        r[c] = make_double2(kc[c] * qq.y + rc.x, -(kc[c] * qq.x) + rc.y);  // -i k q + R^
        if (zero) r[c].x = r[c].x + P.dn * P.g[c];                          // n g_p at k = 0
      }
      const double A = P.nu * L + b;
      double2 kr = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < 3; ++c) kr = cadd(kr, cscale(kc[c], r[c]));
      const double Dn = A + beta * ksq;
      const double rAD = 1.0 / (A * Dn);
      const double f = beta * A * rAD;
      const double2 corr = cscale(f, kr);
      const double invA = Dn * rAD;
      double2 dv = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double2 u = csub(r[c], cscale(kc[c], corr));
        u = make_double2(u.x * invA, u.y * invA);
        dv = cadd(dv, cik(kc[c], u));
        S[(c * CP + q) * SS + C::kp(k0)] = make_double2(u.x * P.inv_n, u.y * P.inv_n);
      }
      double2 qn = csub(qq, cscale(beta, dv));
      if (zero) qn = make_double2(0.0, 0.0);
      const double w = (k2 == 0) ? 1.0 : 2.0;  // main tiles: k2 < N/2
      acc[0] += w * cabs2(dv);
      acc[1] += w * cabs2(csub(dv, dpj));
      acc[2] += w * cabs2(qn);
#if PF_PKP_ABL != 3
      B.Q[tbase + m] = qn;
      B.D[tbase + m] = dv;
#endif
    }
    __syncthreads();  // stage s consumed: refill it with unit + 2 grid strides
    if (t == 0) {
      const int nxt = unit + K::STAGES * gridDim.x;
      if (nxt < NU) issue(nxt, s);
    }
#if PF_PKP_ABL != 2
    if constexpr (K::W32)
      fft256_w32<true>(S + g * SS, tw, l, true);
    else
      fft_seq<N, true>(S + g * SS, tw, l, true);
#endif
    __syncthreads();
#if PF_PKP_ABL != 1
    for (int idx = t; idx < 3 * N * CP; idx += T) {
      const int q = idx % CP, i0 = (idx / CP) % N, c = idx / (CP * N);
      B.Y[ymain<N>(B.yb, c, i0, k1, col0 + q)] = S[(c * CP + q) * SS + C::sp(i0)];
    }
#endif
    __syncthreads();  // the next unit's forward pass overwrites S
  }
  block_sum<3>(acc);
  if (t == 0)
    for (int k = 0; k < 3; ++k) B.part_pk[(size_t)k * (gridDim.x + N / CPT) + blockIdx.x] = acc[k];
}

// ------------------------------------------------------------------ PK, register-resident
// Single GPU, N = 256, main tiles (Nyquist tiles on k_pk).  One warp per column q
// of the tile transforms that column's three components with whole-warp 256-point
// transforms (fft256_w32_r), keeping all three spectra in registers (8 modes per
// lane), so the Green's operator runs on registers — no shared-memory staging of
// the spectra — and the inverse transforms write straight into the TMA store boxes.
// Shared memory: the three boxes (48 KB, loaded and stored by TMA) plus one padded
// transpose scratch per warp.
template <int N>
struct PK3 {
  using C = Cfg<N>;
  static constexpr int CP = PK2<N>::CP;  // 4 columns: one warp each
  static constexpr int T = 32 * CP;
  static constexpr int ROWB = CP * 16;
  static constexpr size_t BOX = sizeof(double2) * CP * N;
  static constexpr size_t SCR = sizeof(double2) * C::SS;  // one warp's transpose scratch
  static constexpr size_t BYTES = 1024 + 3 * BOX + CP * SCR + sizeof(double2) * C::TWN;
  static_assert(N == 256 && ROWB == 64, "register-resident PK: N = 256, 64-byte box rows");
};

template <int N>
__global__ void __launch_bounds__(PK3<N>::T, PF_PK3_MINB) k_pk3(Bufs B, SpecArgs P, const Ctrl* __restrict__ ctrl,
                                                             const __grid_constant__ CUtensorMap tmap, int nparts) {
  using C = Cfg<N>;
  using K = PK3<N>;
  constexpr int CP = K::CP, NCH = PK2<N>::NCH;
  pdl_wait();
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char p3raw[];
  unsigned char* box = p3raw + ((1024 - (su32(p3raw) & 1023)) & 1023);
  double2* scr = (double2*)(box + 3 * K::BOX);
  double2* tw = (double2*)(box + 3 * K::BOX + CP * K::SCR);
  __shared__ uint64_t mbar;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31, j = lane & 15, h = lane >> 4;
  const int tile = blockIdx.x, k1 = tile / NCH, ch = tile % NCH;
  const int q = w, k2 = ch * CP + q;
  const double beta = ctrl->beta, b = ctrl->b;
  if (t == 0) {
    mbar_init(&mbar);
    mbar_expect(&mbar, (uint32_t)(3 * K::BOX));
    for (int c = 0; c < 3; ++c) {
      if (B.yb)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
            "%5}], [%6];" ::"r"(su32(box + c * K::BOX)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * ch * CP), "r"(0), "r"(k1), "r"(c * (N / 4)),
            "r"(su32(&mbar))
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];" ::"r"(su32(box + c * K::BOX)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * ch * CP), "r"(k1), "r"(c * N), "r"(su32(&mbar))
            : "memory");
    }
  }
  for (int i = t; i < C::TWN; i += K::T) tw[i] = B.tw[i];
  // this lane's modes: k0 = j + 16 (k + 8 h), k = 0..7 ([q][k0] in the tile-major Q^, D^)
  const size_t qd = (size_t)tile * CP * N + (size_t)q * N;
  auto cell = [&](const unsigned char* bx, int e) {  // column q of box row e (64B swizzle)
    return reinterpret_cast<double2*>(const_cast<unsigned char*>(bx) + (size_t)e * K::ROWB +
                                      ((q ^ swz16<K::ROWB>(e)) << 4));
  };
  double2* ws = scr + w * C::SS;
  __syncthreads();
  mbar_wait(&mbar, 0);
  double2 X[3][8];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const unsigned char* bx = box + c * K::BOX;
#pragma unroll
    for (int m = 0; m < 8; ++m) X[c][m] = *cell(bx, 16 * (2 * m + h) + j);
    fft256_w32_r<false, false>(X[c], ws, tw, lane, [](int, double2) {});
  }
  // Green's operator per mode (pure.py:26-56), D^ = i k.U^, Q^' = Q^ - beta D^, norms
  double acc[3] = {0.0, 0.0, 0.0};
  const double kc1 = __ldg(P.kap[1] + k1), kc2 = __ldg(P.kap[2] + k2);
  const double l12 = __ldg(P.ell[1] + k1) + __ldg(P.ell[2] + k2);
  const double wgt = (k2 == 0) ? 1.0 : 2.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int k0 = j + 16 * (k + 8 * h);
    const double2 qq = B.Q[qd + k0];
    const double2 dpj = B.D[qd + k0];
    const double kc[3] = {__ldg(P.kap[0] + k0), kc1, kc2};
    const double L = (__ldg(P.ell[0] + k0) + __ldg(P.ell[1] + k1)) + __ldg(P.ell[2] + k2);
    const double ksq = (kc[0] * kc[0] + kc[1] * kc[1]) + kc[2] * kc[2];
    (void)l12;
    const bool zero = (k0 | k1 | k2) == 0;
    double2 r[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double2 rc = X[c][k];
      r[c] = make_double2(kc[c] * qq.y + rc.x, -(kc[c] * qq.x) + rc.y);
      if (zero) r[c].x = r[c].x + P.dn * P.g[c];
    }
    const double A = P.nu * L + b;
    double2 kr = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < 3; ++c) kr = cadd(kr, cscale(kc[c], r[c]));
    const double Dn = A + beta * ksq;
    const double rAD = 1.0 / (A * Dn);
    const double f = beta * A * rAD;
    const double2 corr = cscale(f, kr);
    const double invA = Dn * rAD;
    double2 dv = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double2 u = csub(r[c], cscale(kc[c], corr));
      u = make_double2(u.x * invA, u.y * invA);
      dv = cadd(dv, cik(kc[c], u));
      X[c][k] = make_double2(u.x * P.inv_n, u.y * P.inv_n);
    }
    double2 qn = csub(qq, cscale(beta, dv));
    if (zero) qn = make_double2(0.0, 0.0);
    acc[0] += wgt * cabs2(dv);
    acc[1] += wgt * cabs2(csub(dv, dpj));
    acc[2] += wgt * cabs2(qn);
    B.Q[qd + k0] = qn;
    B.D[qd + k0] = dv;
  }
  // inverse FFT_0 per component straight into its box (this warp's column only)
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    w32_regs_to_input(X[c], lane);
    unsigned char* bx = box + c * K::BOX;
    fft256_w32_r<true, true>(X[c], ws, tw, lane, [&](int e, double2 v) { *cell(bx, e) = v; });
  }
  fence_async_smem();
  __syncthreads();
  if (t == 0) {
    for (int c = 0; c < 3; ++c) {
      if (B.yb)
        asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                         reinterpret_cast<uint64_t>(&tmap)),
                     "r"(2 * ch * CP), "r"(0), "r"(k1), "r"(c * (N / 4)), "r"(su32(box + c * K::BOX))
                     : "memory");
      else
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                         reinterpret_cast<uint64_t>(&tmap)),
                     "r"(2 * ch * CP), "r"(k1), "r"(c * N), "r"(su32(box + c * K::BOX))
                     : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  block_sum<3>(acc);
  if (t == 0) {
    for (int k = 0; k < 3; ++k) st_part(B.part_pk + (size_t)k * nparts + blockIdx.x, acc[k]);
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// natural full spectrum [k0][k1][N/2+1] <-> PK tile-major [tile][q][k0]
template <int N>
__global__ void k_tilemajor(const double2* __restrict__ nat, double2* __restrict__ tm, double scale, int to_tm,
                            int l1) {
  // natural (or slab T-layout) half spectrum [k0][k1 local < l1][N/2+1] <-> PK tile-major
  using K = PK2<N>;
  constexpr int H = N / 2, W = H + 1, CP = K::CP;
  const int tiles = l1 * K::NCH + l1 / CP;
  const int64_t total = (int64_t)tiles * CP * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int tile = (int)(i / (CP * N));
    const int q = (int)((i / N) % CP), k0 = (int)(i % N);
    int k1, k2;
    if (tile < l1 * K::NCH) {
      k1 = tile / K::NCH;
      k2 = (tile % K::NCH) * CP + q;
    } else {
      k1 = (tile - l1 * K::NCH) * CP + q;
      k2 = H;
    }
    const int64_t o = ((int64_t)k0 * l1 + k1) * W + k2;
    if (to_tm) tm[i] = make_double2(nat[o].x * scale, nat[o].y * scale);
    else tm[o] = make_double2(nat[i].x * scale, nat[i].y * scale);  // here nat = tile-major src, tm = natural dst
  }
}

// ------------------------------------------------------------------ layout conversion (setup / teardown)
// rows of the axes-(1, 2) transform, natural [c][i0][k1][N/2+1] over this x-slab's
// l0 planes -> Y in the x-slab exchange layout (Yx, Yxn; see Bufs)
template <int N>
__global__ void k_split_yx(const double2* __restrict__ src, Bufs B) {
  constexpr int H = N / 2, W = H + 1;
  const int l0 = B.l0, l1 = B.l1, s1 = B.s1;
  const int64_t total = (int64_t)3 * l0 * N * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k2 = (int)(i % W);
    int64_t rest = i / W;
    const int k1 = (int)(rest % N);
    rest /= N;
    const int i0 = (int)(rest % l0), c = (int)(rest / l0);
    const int r = k1 >> s1, kl = k1 & (l1 - 1);
    if (k2 < H) {
      if (B.yb) B.Yx[ymain<N>(1, c, i0, k1, k2)] = src[i];  // single GPU, i0-blocked
      else B.Yx[(((int64_t)(c * (N >> s1) + r) * l0 + i0) * l1 + kl) * H + k2] = src[i];
    } else {
      B.Yxn[((int64_t)(r * l0 + i0) * 3 + c) * l1 + kl] = src[i];
    }
  }
}

// slab: this rank's 9 residual sums (RS 6, PK 3) -> totals, with the pore part of
// |lam|^2 of the compact layout added locally (totals are then all-reduced)
__global__ void __launch_bounds__(kFinalizeThreads) k_fslab_totals(const double* __restrict__ prs, int nrs,
                                                                   const double* __restrict__ ppk, int npk,
                                                                   double lam_pore, double* __restrict__ totals) {
  double S[6], Q[3];
  reduce_partials2<6, 3>(prs, nrs, S, ppk, npk, Q);
  if (threadIdx.x == 0) {
    S[2] += lam_pore;
    for (int k = 0; k < 6; ++k) totals[k] = S[k];
    for (int k = 0; k < 3; ++k) totals[6 + k] = Q[k];
  }
}

}  // namespace fz

// ------------------------------------------------------------------ host
struct FusedPlan {
  int N = 0;
  fz::Bufs b{};
  void* mem = nullptr;
  cufftHandle plan2d = 0;
  size_t bytes = 0;
  // compact (solid-only) multiplier storage
  uint32_t* c_cnt = nullptr;
  uint32_t* c_off = nullptr;
  double* c_data = nullptr;
  int64_t c_ns = 0, c_cap = 0;
  int c_cs = 16;  // staging capacity per tile (Compact::cs)
  int compact = 0;
  int nb_rs = kSMs;              // persistent RS grid of the active path (full or compact)
  int rs_rows = kSMs;            // RS partial rows of the last slab iteration (nb_rs or 3 nb_rs)
  // slab-decomposed use (fused_slab_*): Y buffers owned by the caller (exchanged
  // between ranks), the pore part of |lam|^2 added to the local totals instead
  int slab = 0;
  double lam_pore = 0.0;
  CUtensorMap tm_pk{};          // 3D map of Y for PK ([c i0][k1][k2] pencils)
  CUtensorMap tm_pkp{};         // the same with the pipelined PK's unit width (PF_PKP_CP columns)
  CUtensorMap tm_xu{};          // 2D map of XU (MF's X(u~') tile when b changed)
  CUtensorMap tm_y{}, tm_xr{};  // 2D maps of Y and XR ([c][i0][e] rows x N/2 columns) for the axis-1 TMA loads
  void* ws = nullptr;        // cuFFT work area of plan2d
  double2* spec = nullptr;   // setup scratch: axes-(1, 2) transform of R, natural rows
  int nb_full = kSMs, nb_compact = kSMs;
  fz::Peers* peers = nullptr;  // device copy of the peer pointer table (P2P exchange)
  void* grp = nullptr;         // grouped partials + counters (Bufs::gpk, grs, cpk, crs)
  int rsfix_tma = 0, nb_rsfx = kSMs;  // TMA-staged RS-fix (k_rsfix_tma) and its persistent grid
  int m_pipe = 0;              // single GPU, N = 128 / 256: persistent pipelined MI / MF (k_m1_pipe)
  int nb_m1 = 0;
  int pk_pipe = 0;             // single GPU, N = 128 / 256: persistent pipelined PK (k_pk_pipe)
  int pk3 = 0;                 // single GPU, N = 256: register-resident PK (k_pk3)
  int nb_pkp = 0;              // its grid (resident CTAs)
};

static FusedPlan* fp_of(pf_plan* p) { return reinterpret_cast<FusedPlan*>(p->fused); }

bool fused_supported(const pf_plan* p) {
  if (p->g.d != 3) return false;
  const int N = p->g.n[0];
  if (p->g.n[1] != N || p->g.n[2] != N) return false;
  return N == 64 || N == 128 || N == 256 || N == 512 || N == 1024;
}

template <int N>
static size_t smem_mi() { return fz::M2<N>::BYTES_INV; }
template <int N>
static size_t smem_mf() { return fz::M2<N>::BYTES_FWD; }
template <int N>
static size_t smem_rs() { return fz::RS2<N>::BYTES; }
template <int N>
static size_t smem_rsfix() { return fz::RS2<N>::TW + fz::RS2<N>::INV + fz::RS2<N>::ST / 4; }
template <int N>
static size_t smem_rsc() { return fz::RSC<N>::BYTES; }
constexpr int kRsMaxBlocks = kSMs * 64;  // partial-sum rows reserved for the persistent RS grid(s)
template <int N>
static size_t smem_pk() { return fz::PK2<N>::BYTES; }

template <int N>
static int set_attrs(FusedPlan* f) {
  PF_CK_CUDA(smem_attr(fz::k_rs<N, false>, (int)smem_rs<N>()));
  PF_CK_CUDA(smem_attr(fz::k_rsfix<N, false>, (int)smem_rsfix<N>()));
  PF_CK_CUDA(smem_attr(fz::k_rs_compact<N, false>, (int)smem_rsc<N>()));
  PF_CK_CUDA(smem_attr(fz::k_rsfix_compact<N, false>, (int)smem_rsfix<N>()));
  PF_CK_CUDA(smem_attr(fz::k_maxis<N, false, false>, (int)smem_mf<N>()));
  PF_CK_CUDA(smem_attr(fz::k_maxis<N, true, false>, (int)smem_mi<N>()));
  PF_CK_CUDA(smem_attr(fz::k_pk<N, false>, (int)smem_pk<N>()));
  PF_CK_CUDA(smem_attr(fz::k_rs<N, true>, (int)smem_rs<N>()));
  PF_CK_CUDA(smem_attr(fz::k_rsfix<N, true>, (int)smem_rsfix<N>()));
  PF_CK_CUDA(smem_attr(fz::k_rs_compact<N, true>, (int)smem_rsc<N>()));
  PF_CK_CUDA(smem_attr(fz::k_rsfix_compact<N, true>, (int)smem_rsfix<N>()));
  PF_CK_CUDA(smem_attr(fz::k_maxis<N, false, true>, (int)smem_mf<N>()));
  PF_CK_CUDA(smem_attr(fz::k_maxis<N, true, true>, (int)smem_mi<N>()));
  PF_CK_CUDA(smem_attr(fz::k_pk<N, true>, (int)smem_pk<N>()));
  // persistent RS grids: one wave of resident blocks.  The full-layout kernel is
  // capped at 3 per SM: it streams 4 KB/voxel-row-tile at ~93% of HBM peak and a
  // 4th block only adds contention (256^3: 0.697 ms at 4/SM vs 0.662 ms at 3/SM).
  auto wave = [](int o, int cap) { return (o < 1 ? 1 : (o > cap ? cap : o)) * kSMs; };
  int o1 = 0, o2 = 0;
  PF_CK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, fz::k_rs<N, false>, fz::RS2<N>::T, smem_rs<N>()));
  PF_CK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, fz::k_rs_compact<N, false>, fz::RS2<N>::T, smem_rsc<N>()));
  if constexpr (N == 128 || N == 256) {
    PF_CK_CUDA(smem_attr(fz::k_pk_pipe<N>, (int)fz::PKP<N>::BYTES));
    int o3 = 0;
    PF_CK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, fz::k_pk_pipe<N>, fz::PKP<N>::T,
                                                             fz::PKP<N>::BYTES));
    f->nb_pkp = (o3 < 1 ? 1 : o3) * kSMs;
    if (f->nb_pkp > fz::PKP<N>::UNITS) f->nb_pkp = fz::PKP<N>::UNITS;
    const char* e = getenv("POREFLOW_B200_PK_PIPE");
    f->pk_pipe = e ? e[0] == '1' : PF_PK_PIPE;
    if constexpr (N == 256) {
      PF_CK_CUDA(smem_attr(fz::k_pk3<N>, fz::PK3<N>::BYTES));
      PF_CK_CUDA(cudaFuncSetAttribute(fz::k_pk3<N>, cudaFuncAttributePreferredSharedMemoryCarveout, PF_PK3_CARVE));
      const char* e3 = getenv("POREFLOW_B200_PK3");
      f->pk3 = e3 ? e3[0] == '1' : PF_PK3;
    }
    for (int inv = 0; inv < 2; ++inv) {
      auto kern = inv ? fz::k_m1_pipe<N, true> : fz::k_m1_pipe<N, false>;
      PF_CK_CUDA(smem_attr(kern, (int)fz::MP<N>::BYTES));
    }
    int o4 = 0;
    PF_CK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o4, fz::k_m1_pipe<N, true>, fz::MP<N>::T,
                                                             fz::MP<N>::BYTES));
    f->nb_m1 = (o4 < 1 ? 1 : o4) * kSMs;
    const char* e2 = getenv("POREFLOW_B200_M_PIPE");
    f->m_pipe = e2 ? e2[0] == '1' : PF_M_PIPE(N);
  }
  f->nb_full = wave(o1, 3);
  f->nb_compact = wave(o2, kRsMaxBlocks / kSMs);
  f->nb_rs = f->nb_full;
  return PF_OK;
}

// 2D tensor map of a [3 N N rows][N/2 complex] array, box = (CM complex, N rows),
// 128B swizzle (the axis-1 passes' tile); encoded through the runtime's driver
// entry point so the library does not link libcuda directly.
static CUtensorMapSwizzle swizzle_for(int row_bytes) {
  return row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                             : (row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE));
}

static int encode_axis1_rows(CUtensorMap* tm, const double2* base, int N, int cm, int64_t rows);
int encode_axis1_map(CUtensorMap* tm, const double2* base, int N, int cm, int ncomp) {
  return encode_axis1_rows(tm, base, N, cm, (int64_t)ncomp * N * N);
}
static int encode_axis1_rows(CUtensorMap* tm, const double2* base, int N, int cm, int64_t rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    PF_CK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return PF_ERR_CUDA;
    }
    enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const int H = N / 2;
  cuuint64_t gdim[2] = {(cuuint64_t)2 * H, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)H * sizeof(double2)};
  cuuint32_t box[2] = {(cuuint32_t)2 * cm, (cuuint32_t)(N > 256 ? 256 : N)};  // (box rows <= 256)
  cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, gdim, gstride, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(cm * 16),
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return PF_ERR_CUDA;
  }
  return PF_OK;
}

// 3D tensor map of Y [3 N (c, i0)][N k1][N/2 complex], box = (CP complex, 1, N i0),
// 64B swizzle (PK's component pencils).
static int encode_pk_map_gen(CUtensorMap* tm, const double2* base, int N, int cp, int ncomp, int l1);
int encode_pk_map(CUtensorMap* tm, const double2* base, int N, int cp, int ncomp) {
  return encode_pk_map_gen(tm, base, N, cp, ncomp, N);
}
static int encode_pk_map_l1(CUtensorMap* tm, const double2* base, int N, int cp, int l1) {
  return encode_pk_map_gen(tm, base, N, cp, 3, l1);
}
static int encode_pk_map_gen(CUtensorMap* tm, const double2* base, int N, int cp, int ncomp, int l1) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    PF_CK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return PF_ERR_CUDA;
    }
    enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const int H = N / 2;
  cuuint64_t gdim[3] = {(cuuint64_t)2 * H, (cuuint64_t)l1, (cuuint64_t)ncomp * N};
  cuuint64_t gstride[2] = {(cuuint64_t)H * sizeof(double2), (cuuint64_t)l1 * H * sizeof(double2)};
  cuuint32_t box[3] = {(cuuint32_t)2 * cp, 1, (cuuint32_t)(N > 256 ? 256 : N)};  // (box rows <= 256)
  cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)base, gdim, gstride, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(cp * 16),
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return PF_ERR_CUDA;
  }
  return PF_OK;
}

// 4D tensor map of the i0-blocked Y [3 N/4 (c, i0/4)][N k1][4 (i0%4)][N/2 complex]:
// box = (cols complex, bii, bk1, N/4 or 1 planes), swizzled by the box row width.
// PK: (CP, 4, 1, N/4) = one component pencil in i0 order; MI: (CM, 1, N, 1) = one
// (c, i0) tile in k1 order.
static int encode_yb_map(CUtensorMap* tm, const double2* base, int N, int cols, int bii, int bk1) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    PF_CK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return PF_ERR_CUDA;
    }
    enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const int H = N / 2;
  const cuuint64_t row = (cuuint64_t)H * sizeof(double2);
  cuuint64_t gdim[4] = {(cuuint64_t)2 * H, 4, (cuuint64_t)N, (cuuint64_t)3 * N / 4};
  cuuint64_t gstride[3] = {row, 4 * row, 4 * row * N};
  cuuint32_t box[4] = {(cuuint32_t)2 * cols, (cuuint32_t)bii, (cuuint32_t)bk1, (cuuint32_t)(bii == 4 ? N / 4 : 1)};
  cuuint32_t es[4] = {1, 1, 1, 1};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, gdim, gstride, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(cols * 16),
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return PF_ERR_CUDA;
  }
  return PF_OK;
}

int fused_ensure(pf_plan* p) {
  if (p->fused) return PF_OK;
  const int N = p->g.n[0];
  FusedPlan* f = new FusedPlan();
  f->N = N;
  const size_t H = N / 2, NN = (size_t)N * N;
  const size_t main1 = NN * H, nyq1 = NN;  // one component, complex elements
  // X: 6 comps (XU 3, XR 3); Y: 3; Q, D: 1 each
  const size_t elems = 11 * (main1 + nyq1) + N;
  const int nb_rs = kRsMaxBlocks;
  const int nb_pk = (N == 64) ? fz::PK2<64>::TILES : (N == 128 ? fz::PK2<128>::TILES : (N == 256 ? fz::PK2<256>::TILES : (N == 512 ? fz::PK2<512>::TILES : fz::PK2<1024>::TILES)));
  const size_t part = 6 * (size_t)nb_rs + 3 * (size_t)nb_pk;
  f->bytes = elems * sizeof(double2) + part * sizeof(double);
  PF_CK_CUDA(cudaMalloc(&f->mem, f->bytes));
  double2* m = (double2*)f->mem;
  auto take = [&](size_t n) {
    double2* r = m;
    m += n;
    return r;
  };
  f->b.XU = take(3 * main1);
  f->b.XR = take(3 * main1);
  f->b.Y = take(3 * main1);
  f->b.Q = take(main1 + nyq1);
  f->b.D = take(main1 + nyq1);
  f->b.XUn = take(3 * nyq1);
  f->b.XRn = take(3 * nyq1);
  f->b.Yn = take(3 * nyq1);
  f->b.tw = take(N);
  // single GPU: the whole cube is one slab; x- and y-slab Y layouts coincide
  f->b.l0 = N;
  f->b.l1 = N;
  f->b.s1 = 0;
  while ((1 << f->b.s1) < N) ++f->b.s1;
  f->b.k1off = 0;
  f->b.i0a = 0;
  f->b.nl = N;
  f->b.c0 = 0;
  f->b.nc = 3;
  f->b.pst = 0;
  f->b.poff = 0;
  f->b.Yx = f->b.Y;
  f->b.Yxn = f->b.Yn;
  f->b.part_rs = (double*)m;
  f->b.part_pk = f->b.part_rs + 6 * (size_t)nb_rs;
  {
    const size_t ngp = (size_t)nb_pk / PF_GRP_PK + 1, ngr = (size_t)nb_rs / PF_GRP_RS + 1;
    PF_CK_CUDA(cudaMalloc(&f->grp, sizeof(double) * (3 * ngp + 6 * ngr) + sizeof(unsigned) * (ngp + ngr)));
    PF_CK_CUDA(cudaMemset(f->grp, 0, sizeof(double) * (3 * ngp + 6 * ngr) + sizeof(unsigned) * (ngp + ngr)));
    f->b.gpk = (double*)f->grp;
    f->b.grs = f->b.gpk + 3 * ngp;
    f->b.cpk = (unsigned*)(f->b.grs + 6 * ngr);
    f->b.crs = f->b.cpk + ngp;
    const char* e = getenv("POREFLOW_B200_GROUPED");
    if (e ? e[0] == '0' : !PF_GROUPED) f->b.cpk = f->b.crs = nullptr;
  }
  std::vector<double2> tw(N == 64 ? fz::Cfg<64>::TWN : (N == 128 ? fz::Cfg<128>::TWN : (N == 256 ? fz::Cfg<256>::TWN : (N == 512 ? fz::Cfg<512>::TWN : fz::Cfg<1024>::TWN))));
  switch (N) {
    case 64: fz::pass1_twiddles<64>(tw.data()); break;
    case 128: fz::pass1_twiddles<128>(tw.data()); break;
    case 256: fz::pass1_twiddles<256>(tw.data()); break;
    case 512: fz::pass1_twiddles<512>(tw.data()); break;
    default: fz::pass1_twiddles<1024>(tw.data()); break;
  }
  PF_CK_CUDA(cudaMemcpy(f->b.tw, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice));
  f->b.tma = 0;
  {
    const char* e = getenv("POREFLOW_B200_YBLOCK");
    f->b.yb = (N <= 256 && PF_YBLOCK && !(e && e[0] == '0')) ? 1 : 0;
  }
  if (N >= 128) {  // TMA maps (N > 256: M boxes of 256 rows per tile / component pencil)
    const int cm = N == 128 ? fz::M2<128>::CM : (N == 256 ? fz::M2<256>::CM : (N == 512 ? fz::M2<512>::CM : fz::M2<1024>::CM));
    const int cp = N == 128 ? fz::PK2<128>::CP : (N == 256 ? fz::PK2<256>::CP : (N == 512 ? fz::PK2<512>::CP : fz::PK2<1024>::CP));
    if (f->b.yb) {
      PF_CK(encode_yb_map(&f->tm_y, f->b.Y, N, cm, 1, N));      // MI: (CM cols, 1, all k1, 1)
      PF_CK(encode_yb_map(&f->tm_pk, f->b.Y, N, cp, 4, 1));     // PK: (CP cols, 4, 1, N/4)
      PF_CK(encode_yb_map(&f->tm_pkp, f->b.Y, N, PF_PKP_CP, 4, 1));
    } else {
      PF_CK(encode_axis1_map(&f->tm_y, f->b.Y, N, cm, 3));
      PF_CK(encode_pk_map(&f->tm_pk, f->b.Y, N, cp, 3));
      PF_CK(encode_pk_map(&f->tm_pkp, f->b.Y, N, PF_PKP_CP, 3));
    }
    PF_CK(encode_axis1_map(&f->tm_xr, f->b.XR, N, cm, 3));
    PF_CK(encode_axis1_map(&f->tm_xu, f->b.XU, N, cm, 3));
    f->b.tma = f->b.tma_yx = 1;
  }
  // 2D transform over axes (1, 2) batched over (component, i0): the Y-space
  // right-hand side at setup time.
  size_t ws = 0;
  long long dims2[2] = {N, N};
  PF_CK_FFT(cufftCreate(&f->plan2d));
  PF_CK_FFT(cufftSetAutoAllocation(f->plan2d, 0));
  PF_CK_FFT(cufftMakePlanMany64(f->plan2d, 2, dims2, nullptr, 1, (long long)NN, nullptr, 1,
                                (long long)N * (H + 1), CUFFT_D2Z, 3LL * N, &ws));
  if (ws > p->fft_work_bytes) {
    PF_CK_CUDA(cudaStreamSynchronize(p->work));
    if (p->fft_work) PF_CK_CUDA(cudaFree(p->fft_work));
    PF_CK_CUDA(cudaMalloc(&p->fft_work, ws));
    p->fft_work_bytes = ws;
    for (int k = 0; k < 4; ++k) {
      if (p->fwd[k]) PF_CK_FFT(cufftSetWorkArea(p->fwd[k], p->fft_work));
      if (p->inv[k]) PF_CK_FFT(cufftSetWorkArea(p->inv[k], p->fft_work));
    }
    p->graph.reset();
  }
  PF_CK_FFT(cufftSetWorkArea(f->plan2d, p->fft_work));
  PF_CK_FFT(cufftSetStream(f->plan2d, p->work));
  switch (N) {
    case 64: PF_CK(set_attrs<64>(f)); break;
    case 128: PF_CK(set_attrs<128>(f)); break;
    case 256: PF_CK(set_attrs<256>(f)); break;
    case 512: PF_CK(set_attrs<512>(f)); break;
    default: PF_CK(set_attrs<1024>(f)); break;
  }
  p->fused = f;
  p->scratch_bytes += f->bytes;
  return PF_OK;
}

void fused_free(pf_plan* p) {
  FusedPlan* f = fp_of(p);
  if (!f) return;
  if (f->plan2d) cufftDestroy(f->plan2d);
  cudaFree(f->mem);
  cudaFree(f->c_cnt);
  cudaFree(f->c_off);
  cudaFree(f->c_data);
  cudaFree(f->ws);
  cudaFree(f->spec);
  cudaFree(f->peers);
  cudaFree(f->grp);
  delete f;
  p->fused = nullptr;
}

static int to_tilemajor(int N, const double2* src, double2* dst, double scale, bool to_tm, cudaStream_t s,
                        int l1 = 0) {
  if (l1 == 0) l1 = N;
  const int64_t total = (int64_t)N * l1 * (N / 2 + 1);
  const int nb = blocks_for(total);
  switch (N) {
    case 64: fz::k_tilemajor<64><<<nb, kThreads, 0, s>>>(src, dst, scale, to_tm, l1); break;
    case 128: fz::k_tilemajor<128><<<nb, kThreads, 0, s>>>(src, dst, scale, to_tm, l1); break;
    case 256: fz::k_tilemajor<256><<<nb, kThreads, 0, s>>>(src, dst, scale, to_tm, l1); break;
    case 512: fz::k_tilemajor<512><<<nb, kThreads, 0, s>>>(src, dst, scale, to_tm, l1); break;
    default: fz::k_tilemajor<1024><<<nb, kThreads, 0, s>>>(src, dst, scale, to_tm, l1); break;
  }
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

// exclusive scan of n counts into off[0..n] (one block; setup only)
int scan_counts(cudaStream_t s, const uint32_t* cnt, uint32_t* off, int64_t n) {
  fz::k_scan<<<1, 1024, 0, s>>>(cnt, off, n);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

static fz::Compact compact_of(FusedPlan* f) {
  fz::Compact c;
  c.off = f->c_off;
  c.ut = f->c_data;
  c.a = f->c_data + 3 * f->c_ns;
  c.lam = f->c_data + 6 * f->c_ns;
  c.ns = f->c_ns;
  c.cs = f->c_cs;
  return c;
}

template <int N>
static int compact_setup_t(pf_plan* p, FusedPlan* f, bool cold = false) {
  const int64_t rows = (int64_t)f->b.l0 * N, n = rows * N;
  // eligibility (a = 0 on pore voxels: cold starts and states this path produced)
  // and the constant pore part of |lam'|^2 (a cold start: both zero, no pass)
  if (cold) {
    p->h_small[0] = p->h_small[1] = 0.0;
  } else {
    const int nb = blocks_for(3 * n);
    fz::k_pore_a_lam<<<nb, kThreads, 0, p->work>>>(n, p->s_solid, p->s_a, p->s_lam, p->partials);
    double* out = p->partials + 24 * kMaxBlocks;
    PF_CK(reduce_rows_to(p, p->partials, 2, nb, out));
    PF_CK_CUDA(cudaMemcpyAsync(p->h_small, out, 2 * sizeof(double), cudaMemcpyDeviceToHost, p->work));
    PF_CK_CUDA(cudaStreamSynchronize(p->work));
  }
  // (solid-only storage: RS tiles of 1024 or 2048 voxels)
  f->compact = (p->compact_enable && p->h_small[0] == 0.0 && fz::RS2<N>::V <= 2048) ? 1 : 0;
  f->nb_rs = f->compact ? f->nb_compact : f->nb_full;
  p->sc.lam_pore_sq = f->compact ? p->h_small[1] : 0.0;
  if (!f->compact) return PF_OK;
  if (!f->c_cnt) {
    PF_CK_CUDA(cudaMalloc(&f->c_cnt, sizeof(uint32_t) * rows));
    PF_CK_CUDA(cudaMalloc(&f->c_off, sizeof(uint32_t) * (rows + 2)));  // + the tile max
  }
  fz::k_row_counts<N><<<blocks_for(rows * 32), kThreads, 0, p->work>>>(p->s_solid, f->c_cnt, rows);
  fz::k_scan<<<1, 1024, 0, p->work>>>(f->c_cnt, f->c_off, rows);
  PF_CK_CUDA(cudaMemsetAsync(f->c_off + rows + 1, 0, sizeof(uint32_t), p->work));
  fz::k_tile_max<N><<<blocks_for(rows / fz::RS2<N>::R), kThreads, 0, p->work>>>(f->c_off, f->c_off + rows + 1,
                                                                                  rows);
  PF_CK_CUDA(cudaGetLastError());
  uint32_t nm[2] = {0, 0};
  PF_CK_CUDA(cudaMemcpyAsync(p->h_small, f->c_off + rows, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, p->work));
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  std::memcpy(nm, p->h_small, 2 * sizeof(uint32_t));
  const uint32_t ns = nm[0];
  f->c_ns = ns;
  // staging sized by this geometry's densest tile: fewer bytes of smem -> more resident RS CTAs
  f->c_cs = (int)((nm[1] + 15u) & ~15u);
  if (f->c_cs < 16) f->c_cs = 16;
  {
    int o = 0;
    PF_CK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fz::k_rs_compact<N, false>, fz::RS2<N>::T,
                                                             fz::RSC<N>::bytes(f->c_cs)));
  {
    // (the limit is per function, not per plan: set the worst case so every cell's
    // staging capacity fits — several cells with different geometries share it)
    PF_CK_CUDA(smem_attr(fz::k_rsfix_tma<N>, fz::RSFX<N>::bytes(fz::RSC<N>::CS)));
    int ox = 0;
    PF_CK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ox, fz::k_rsfix_tma<N>, fz::RS2<N>::T,
                                                             fz::RSFX<N>::bytes(f->c_cs)));
    f->nb_rsfx = (ox < 1 ? 1 : (ox > 8 ? 8 : ox)) * kSMs;
    const char* e = getenv("POREFLOW_B200_RSFIX_TMA");
    f->rsfix_tma = e ? e[0] == '1' : PF_RSFIX_TMA;
  }
    f->nb_compact = (o < 1 ? 1 : (o > kRsMaxBlocks / kSMs ? kRsMaxBlocks / kSMs : o)) * kSMs;
    f->nb_rs = f->nb_compact;
  }
  const int64_t need = 9 * (int64_t)(ns > 0 ? ns : 2);
  if (need > f->c_cap) {
    cudaFree(f->c_data);
    f->c_data = nullptr;
    PF_CK_CUDA(cudaMalloc(&f->c_data, sizeof(double) * (size_t)need));
    f->c_cap = need;
  }
  if (cold) {  // solid u~, a, lam of a zero state: zeros
    PF_CK_CUDA(cudaMemsetAsync(f->c_data, 0, sizeof(double) * (size_t)need, p->work));
    return PF_OK;
  }
  fz::k_compact_move<N><<<blocks_for(3 * rows * 32), kThreads, 0, p->work>>>(p->s_solid, compact_of(f), p->s_ut,
                                                                             p->s_a, p->s_lam, p->s_u, 0, rows);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

// Setup: Q^, D^_prev and the Y-space right-hand side from the real state.
int fused_setup(pf_plan* p) {
  FusedPlan* f = fp_of(p);
  const int N = f->N;
  const int64_t n = p->g.nr, nh = p->g.nh, NN = (int64_t)N * N;
  const int grid = blocks_for(nh * 3);
  if (p->cold_start) {
    // zero state (pf_plan_set_cold_start): Q^ = D^ = 0 and the Y-space right-hand side
    // FFT(b*0 - 0) = 0 — no transforms; the solid-only storage starts at zero
    const size_t H = N / 2, main1 = (size_t)N * N * H, nyq1 = (size_t)N * N;
    PF_CK_CUDA(cudaMemsetAsync(f->b.Q, 0, sizeof(double2) * (main1 + nyq1), p->work));
    PF_CK_CUDA(cudaMemsetAsync(f->b.D, 0, sizeof(double2) * (main1 + nyq1), p->work));
    PF_CK_CUDA(cudaMemsetAsync(f->b.Y, 0, sizeof(double2) * 3 * main1, p->work));
    PF_CK_CUDA(cudaMemsetAsync(f->b.Yn, 0, sizeof(double2) * 3 * nyq1, p->work));
    switch (N) {
      case 64: return compact_setup_t<64>(p, f, true);
      case 128: return compact_setup_t<128>(p, f, true);
      case 256: return compact_setup_t<256>(p, f, true);
      case 512: return compact_setup_t<512>(p, f, true);
      default: return compact_setup_t<1024>(p, f, true);
    }
  }
  // Q^ = FFT(q), gauge Q^(0) = 0
  PF_CK(plan_fft(p, true, 1, p->s_q, p->specB));
  PF_CK(to_tilemajor(N, p->specB, f->b.Q, 1.0, true, p->work));
  PF_CK_CUDA(cudaMemsetAsync(f->b.Q, 0, sizeof(double2), p->work));  // tile 0, q 0, k0 0 = mode (0,0,0)
  // D^_prev = i k . FFT(u)
  PF_CK(stokes_div_spectrum(p, p->s_u, p->specB, p->spec2));
  PF_CK(to_tilemajor(N, p->spec2, f->b.D, 1.0, true, p->work));
  // Y-space R~ = FFT_{2,1}(b u~ - a)
  PF_CK(stokes_form_r(p, p->realB));
  PF_CK_FFT(cufftExecD2Z(f->plan2d, (cufftDoubleReal*)p->realB, (cufftDoubleComplex*)p->specA));
  switch (N) {
    case 64: fz::k_split_yx<64><<<grid, kThreads, 0, p->work>>>(p->specA, f->b); break;
    case 128: fz::k_split_yx<128><<<grid, kThreads, 0, p->work>>>(p->specA, f->b); break;
    case 256: fz::k_split_yx<256><<<grid, kThreads, 0, p->work>>>(p->specA, f->b); break;
    case 512: fz::k_split_yx<512><<<grid, kThreads, 0, p->work>>>(p->specA, f->b); break;
    default: fz::k_split_yx<1024><<<grid, kThreads, 0, p->work>>>(p->specA, f->b); break;
  }
  PF_CK_CUDA(cudaGetLastError());
  (void)NN;
  (void)n;
  switch (N) {
    case 64: return compact_setup_t<64>(p, f);
    case 128: return compact_setup_t<128>(p, f);
    case 256: return compact_setup_t<256>(p, f);
    case 512: return compact_setup_t<512>(p, f);
    default: return compact_setup_t<1024>(p, f);
  }
}

// q = Re ifft(Q^) into the user's q.
int fused_finish(pf_plan* p) {
  FusedPlan* f = fp_of(p);
  const int N = f->N;
  const int64_t NN = (int64_t)N * N, rows = (int64_t)f->b.l0 * N;
  PF_CK(to_tilemajor(N, f->b.Q, p->specB, p->g.inv_n, false, p->work));
  PF_CK(plan_fft(p, false, 1, p->specB, p->s_q));
  if (f->compact) {  // materialise u~, a, lam (pore: u~ = u, a = 0, lam unchanged)
    const int nb = blocks_for(3 * rows * 32);
    (void)NN;
    switch (N) {
      case 64: fz::k_compact_move<64><<<nb, kThreads, 0, p->work>>>(p->s_solid, compact_of(f), p->s_ut, p->s_a, p->s_lam, p->s_u, 1, rows); break;
      case 128: fz::k_compact_move<128><<<nb, kThreads, 0, p->work>>>(p->s_solid, compact_of(f), p->s_ut, p->s_a, p->s_lam, p->s_u, 1, rows); break;
      case 256: fz::k_compact_move<256><<<nb, kThreads, 0, p->work>>>(p->s_solid, compact_of(f), p->s_ut, p->s_a, p->s_lam, p->s_u, 1, rows); break;
      case 512: fz::k_compact_move<512><<<nb, kThreads, 0, p->work>>>(p->s_solid, compact_of(f), p->s_ut, p->s_a, p->s_lam, p->s_u, 1, rows); break;
      default: fz::k_compact_move<1024><<<nb, kThreads, 0, p->work>>>(p->s_solid, compact_of(f), p->s_ut, p->s_a, p->s_lam, p->s_u, 1, rows); break;
    }
    PF_CK_CUDA(cudaGetLastError());
  }
  return PF_OK;
}

template <int N, bool INV>
static cudaError_t launch_m1_pipe(pf_plan* p, FusedPlan* f, const CUtensorMap& tm) {
  if constexpr (N == 128 || N == 256) {
    return launch_k(fz::k_m1_pipe<N, INV>, f->nb_m1, fz::MP<N>::T, fz::MP<N>::BYTES, p->work, f->b,
                    (const Ctrl*)p->ctrl, tm, f->tm_xu);
  } else {
    (void)p, (void)f, (void)tm;
    return cudaErrorInvalidValue;
  }
}

template <int N>
static cudaError_t launch_pk3(pf_plan* p, FusedPlan* f, const fz::SpecArgs& sa, int nparts) {
  if constexpr (N == 256) {
    return launch_k(fz::k_pk3<N>, N * fz::PK2<N>::NCH, fz::PK3<N>::T, fz::PK3<N>::BYTES, p->work, f->b, sa,
                    (const Ctrl*)p->ctrl, f->tm_pk, nparts);
  } else {
    (void)p, (void)f, (void)sa, (void)nparts;
    return cudaErrorInvalidValue;
  }
}

template <int N>
static cudaError_t launch_pk_pipe(pf_plan* p, FusedPlan* f, const fz::SpecArgs& sa) {
  if constexpr (N == 128 || N == 256) {
    return launch_k(fz::k_pk_pipe<N>, f->nb_pkp, fz::PKP<N>::T, fz::PKP<N>::BYTES, p->work, f->b, sa,
                    (const Ctrl*)p->ctrl, f->tm_pkp);
  } else {
    (void)p, (void)f, (void)sa;
    return cudaErrorInvalidValue;
  }
}

template <int N>
static int enqueue_fused_t(pf_plan* p, cudaEvent_t* ev) {
  using C = fz::Cfg<N>;
  FusedPlan* f = fp_of(p);
  fz::State st{p->s_u, p->s_ut, p->s_a, p->s_lam, p->s_solid};
  fz::SpecArgs sa;
  for (int i = 0; i < 3; ++i) {
    sa.kap[i] = p->kap[i];
    sa.ell[i] = p->ell[i];
    sa.g[i] = p->sc.g[i];
  }
  sa.nu = p->sc.nu;
  sa.inv_n = p->g.inv_n;
  sa.dn = p->g.dn;
  auto mark = [&](int i) -> int {
    if (ev) PF_CK_CUDA(cudaEventRecord(ev[i], p->work));
    return PF_OK;
  };
  PF_CK(mark(0));
  int pk_tiles = f->b.l1 * fz::PK2<N>::NCH + f->b.l1 / fz::PK2<N>::CP;
  const int m_tiles = 3 * (f->b.l0 * fz::M2<N>::NCH + f->b.l0 / fz::M2<N>::CM);
  if (f->pk3 && f->b.tma) {  // register-resident PK on the main tiles + k_pk on the Nyquist tiles
    const int main_tiles = N * fz::PK2<N>::NCH, nyq = N / fz::PK2<N>::CP;
    PF_CK_CUDA((launch_pk3<N>(p, f, sa, main_tiles + nyq)));
    PF_CK_CUDA(launch_k(fz::k_pk<N, false>, nyq, fz::PK2<N>::T, smem_pk<N>(), p->work, f->b, sa,
                        (const Ctrl*)p->ctrl, f->tm_pk, main_tiles, main_tiles, main_tiles + nyq));
    pk_tiles = main_tiles + nyq;
  } else if (f->pk_pipe && f->b.tma) {  // persistent pipelined PK on the main tiles + k_pk on the N / CP Nyquist tiles
    const int main_tiles = N * fz::PK2<N>::NCH, nyq = N / fz::PK2<N>::CP;
    PF_CK_CUDA(launch_pk_pipe<N>(p, f, sa));
    PF_CK_CUDA(launch_k(fz::k_pk<N, false>, nyq, fz::PK2<N>::T, smem_pk<N>(), p->work, f->b, sa,
                        (const Ctrl*)p->ctrl, f->tm_pk, main_tiles, f->nb_pkp, f->nb_pkp + nyq));
    pk_tiles = f->nb_pkp + nyq;  // partial rows for the finalize
  } else {
    PF_CK_CUDA(launch_k(fz::k_pk<N, false>, pk_tiles, fz::PK2<N>::T, smem_pk<N>(), p->work, f->b, sa,
                        (const Ctrl*)p->ctrl, f->tm_pk, 0, 0, pk_tiles));
  }
  PF_CK(mark(1));
  int nb_part = f->nb_rs;
  if (f->m_pipe && f->b.tma) {  // persistent main tiles + k_maxis on the Nyquist tiles
    PF_CK_CUDA((launch_m1_pipe<N, true>(p, f, f->tm_y)));
    PF_CK_CUDA(launch_k(fz::k_maxis<N, true, false>, 3 * (N / fz::M2<N>::CM), fz::M2<N>::T, smem_mi<N>(), p->work,
                        f->b, (const Ctrl*)p->ctrl, f->tm_y, 1, f->tm_xu));
  } else {
    PF_CK_CUDA(launch_k(fz::k_maxis<N, true, false>, m_tiles, fz::M2<N>::T, smem_mi<N>(), p->work, f->b,
                        (const Ctrl*)p->ctrl, f->tm_y, 0, f->tm_xu));
  }
  PF_CK(mark(2));
  if (f->compact) {
    PF_CK_CUDA(launch_k(fz::k_rs_compact<N, false>, f->nb_rs, fz::RS2<N>::T, fz::RSC<N>::bytes(f->c_cs), p->work,
                        f->b, st, compact_of(f), (const Ctrl*)p->ctrl));
  } else {
    PF_CK_CUDA(launch_k(fz::k_rs<N, false>, f->nb_rs, fz::RS2<N>::T, smem_rs<N>(), p->work, f->b, st,
                        (const Ctrl*)p->ctrl));
  }
  PF_CK(mark(3));
#if PF_ABL_NOFIN == 0
  if (f->b.crs && !(f->pk_pipe && f->b.tma)) {  // grouped partials (the pipelined PK keeps per-CTA rows)
    PF_CK_CUDA(k_stokes_finalize_launch_pdl(p, f->b.grs, (nb_part + PF_GRP_RS - 1) / PF_GRP_RS, f->b.gpk,
                                            (pk_tiles + PF_GRP_PK - 1) / PF_GRP_PK));
  } else {
    PF_CK_CUDA(k_stokes_finalize_launch_pdl(p, f->b.part_rs, nb_part, f->b.part_pk, pk_tiles));
  }
#endif
  PF_CK(mark(4));
  if (PF_ABL_NORSF) {
  } else if (f->compact && f->rsfix_tma) {
    PF_CK_CUDA(launch_k(fz::k_rsfix_tma<N>, f->nb_rsfx, fz::RS2<N>::T, fz::RSFX<N>::bytes(f->c_cs), p->work, f->b,
                        (const double*)p->s_u, (const uint8_t*)p->s_solid, compact_of(f), (const Ctrl*)p->ctrl));
  } else if (f->compact) {
    PF_CK_CUDA(launch_k(fz::k_rsfix_compact<N, false>, f->nb_rs, fz::RS2<N>::T, smem_rsfix<N>(), p->work, f->b,
                        (const double*)p->s_u, (const uint8_t*)p->s_solid, compact_of(f), (const Ctrl*)p->ctrl));
  } else {
    PF_CK_CUDA(launch_k(fz::k_rsfix<N, false>, f->nb_rs, fz::RS2<N>::T, smem_rsfix<N>(), p->work, f->b,
                        (const double*)p->s_ut, (const Ctrl*)p->ctrl));
  }
  PF_CK(mark(5));
  if (f->m_pipe && f->b.tma) {
    PF_CK_CUDA((launch_m1_pipe<N, false>(p, f, f->tm_xr)));
    PF_CK_CUDA(launch_k(fz::k_maxis<N, false, false>, 3 * (N / fz::M2<N>::CM), fz::M2<N>::T, smem_mf<N>(),
                        p->work, f->b, (const Ctrl*)p->ctrl, f->tm_xr, 1, f->tm_xu));
  } else {
    PF_CK_CUDA(launch_k(fz::k_maxis<N, false, false>, m_tiles, fz::M2<N>::T, smem_mf<N>(), p->work, f->b,
                        (const Ctrl*)p->ctrl, f->tm_xr, 0, f->tm_xu));
  }
  PF_CK(mark(6));
  return PF_OK;
}

int fused_is_compact(const pf_plan* p) {
  const FusedPlan* f = reinterpret_cast<const FusedPlan*>(p->fused);
  return f ? f->compact : 0;
}

int enqueue_fused(pf_plan* p, cudaEvent_t* ev) {
  switch (fp_of(p)->N) {
    case 64: return enqueue_fused_t<64>(p, ev);
    case 128: return enqueue_fused_t<128>(p, ev);
    case 256: return enqueue_fused_t<256>(p, ev);
    case 512: return enqueue_fused_t<512>(p, ev);
    default: return enqueue_fused_t<1024>(p, ev);
  }
}


// ------------------------------------------------------------------ slab-decomposed fused pipeline
// One cell over P ranks (slab.py FusedSlabStokes): rank r holds the x-slab of
// the real state (l0 i0-planes) and of X, and the y-slab (l1 k1-planes from
// k1off) of Q^, D^; Y lives in the two exchange-native layouts of Bufs, whose
// buffers the caller owns and all-to-alls between PK and the axis-1 passes.
static bool fslab_shape_ok(int N, int l0, int l1) {
  if (N != 64 && N != 128 && N != 256 && N != 512 && N != 1024) return false;
  if (l0 <= 0 || l1 <= 0 || (l1 & (l1 - 1)) || N % l0 || N % l1) return false;
  const int cm = N == 64 ? fz::M2<64>::CM : (N == 128 ? fz::M2<128>::CM : (N == 256 ? fz::M2<256>::CM : (N == 512 ? fz::M2<512>::CM : fz::M2<1024>::CM)));
  const int cp = N == 64 ? fz::PK2<64>::CP : (N == 128 ? fz::PK2<128>::CP : (N == 256 ? fz::PK2<256>::CP : (N == 512 ? fz::PK2<512>::CP : fz::PK2<1024>::CP)));
  return l0 % cm == 0 && l1 % cp == 0;
}

// 5D tensor map of the x-slab Y [3][P][l0][l1][N/2 complex] with box (cm complex,
// l1, 1, P, 1): an axis-1 tile whose N rows come out in k1 order, 128B swizzle.
static int encode_yx_map(CUtensorMap* tm, const double2* base, int N, int cm, int l0, int l1) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    PF_CK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return PF_ERR_CUDA;
    }
    enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const int H = N / 2, P = N / l1;
  const cuuint64_t rowb = (cuuint64_t)H * sizeof(double2);
  cuuint64_t gdim[5] = {(cuuint64_t)2 * H, (cuuint64_t)l1, (cuuint64_t)l0, (cuuint64_t)P, 3};
  cuuint64_t gstride[4] = {rowb, rowb * l1, rowb * l1 * l0, rowb * l1 * l0 * P};
  cuuint32_t box[5] = {(cuuint32_t)2 * cm, (cuuint32_t)l1, 1, (cuuint32_t)P, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)base, gdim, gstride, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(cm * 16), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (5D) failed (%d)", (int)r);
    return PF_ERR_CUDA;
  }
  return PF_OK;
}

int fused_slab_supported(int N, int l0, int l1) { return fslab_shape_ok(N, l0, l1) ? 1 : 0; }

int fused_slab_bind(pf_plan* p, int N, int l0, int l1, int k1off, double2* Yy, double2* Yyn, double2* Yx,
                    double2* Yxn) {
  if (!fslab_shape_ok(N, l0, l1)) {
    set_error("fused slab needs N in {64, 128, 256}, a power-of-two rank count and slabs of whole tiles");
    return PF_ERR_ARG;
  }
  if (p->fused) fused_free(p);
  FusedPlan* f = new FusedPlan();
  p->fused = f;
  f->N = N;
  f->slab = 1;
  const size_t H = N / 2;
  const size_t xm = (size_t)l0 * N * H, xn = (size_t)l0 * N;  // X per component
  const size_t qd = (size_t)l1 * N * H + (size_t)l1 * N;      // Q^ / D^ (tile-major, y-slab)
  const int pk_max = N == 64 ? fz::PK2<64>::TILES : (N == 128 ? fz::PK2<128>::TILES : (N == 256 ? fz::PK2<256>::TILES : (N == 512 ? fz::PK2<512>::TILES : fz::PK2<1024>::TILES)));
  const size_t elems = 6 * (xm + xn) + 2 * qd + N;
  const size_t part = 6 * (size_t)kRsMaxBlocks + 3 * (size_t)pk_max;
  f->bytes = elems * sizeof(double2) + part * sizeof(double);
  PF_CK_CUDA(cudaMalloc(&f->mem, f->bytes));
  double2* m = (double2*)f->mem;
  auto take = [&](size_t n) {
    double2* r = m;
    m += n;
    return r;
  };
  f->b.XU = take(3 * xm);
  f->b.XR = take(3 * xm);
  f->b.XUn = take(3 * xn);
  f->b.XRn = take(3 * xn);
  f->b.Q = take(qd);
  f->b.D = take(qd);
  f->b.tw = take(N);
  f->b.part_rs = (double*)m;
  f->b.part_pk = f->b.part_rs + 6 * (size_t)kRsMaxBlocks;
  f->b.Y = Yy;
  f->b.Yn = Yyn;
  f->b.Yx = Yx;
  f->b.Yxn = Yxn;
  f->b.l0 = l0;
  f->b.l1 = l1;
  f->b.s1 = 0;
  while ((1 << f->b.s1) < l1) ++f->b.s1;
  f->b.k1off = k1off;
  f->b.i0a = 0;
  f->b.nl = l0;
  f->b.c0 = 0;
  f->b.nc = 3;
  f->b.pst = 0;  // set per launch (nb_rs)
  f->b.poff = 0;
  std::vector<double2> tw(N == 64 ? fz::Cfg<64>::TWN : (N == 128 ? fz::Cfg<128>::TWN : (N == 256 ? fz::Cfg<256>::TWN : (N == 512 ? fz::Cfg<512>::TWN : fz::Cfg<1024>::TWN))));
  switch (N) {
    case 64: fz::pass1_twiddles<64>(tw.data()); break;
    case 128: fz::pass1_twiddles<128>(tw.data()); break;
    case 256: fz::pass1_twiddles<256>(tw.data()); break;
    case 512: fz::pass1_twiddles<512>(tw.data()); break;
    default: fz::pass1_twiddles<1024>(tw.data()); break;
  }
  PF_CK_CUDA(cudaMemcpy(f->b.tw, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice));
  // (the axes-(1, 2) transform of a warm start's R is planned in fused_slab_setup
  // and released after it: no setup-only memory stays resident)
  f->b.tma = f->b.tma_yx = 0;
  if (N >= 128) {  // TMA maps of this slab's layouts (every box dimension <= 256)
    const int cm = N == 128 ? fz::M2<128>::CM : (N == 256 ? fz::M2<256>::CM : (N == 512 ? fz::M2<512>::CM : fz::M2<1024>::CM));
    const int cp = N == 128 ? fz::PK2<128>::CP : (N == 256 ? fz::PK2<256>::CP : (N == 512 ? fz::PK2<512>::CP : fz::PK2<1024>::CP));
    PF_CK(encode_axis1_rows(&f->tm_xr, f->b.XR, N, cm, 3 * (int64_t)l0 * N));
    PF_CK(encode_pk_map_l1(&f->tm_pk, Yy, N, cp, l1));
    f->b.tma = 1;
    if (l1 <= 256 && N / l1 <= 256) {  // MI's 5D box spans (l1, P) rows
      PF_CK(encode_yx_map(&f->tm_y, Yx, N, cm, l0, l1));
      f->b.tma_yx = 1;
    }
  }
  switch (N) {
    case 64: PF_CK(set_attrs<64>(f)); break;
    case 128: PF_CK(set_attrs<128>(f)); break;
    case 256: PF_CK(set_attrs<256>(f)); break;
    case 512: PF_CK(set_attrs<512>(f)); break;
    default: PF_CK(set_attrs<1024>(f)); break;
  }
  p->scratch_bytes += f->bytes;
  return PF_OK;
}

// Setup from the slab T-layout spectra Q^ = FFT(q) (gauge applied) and D^ =
// i k . FFT(u) (pf_slab_setup), and the real R = b u~ - a of this slab (scratch R).
int fused_slab_setup(pf_plan* p, const double2* Tq, const double2* Td, double* R) {
  FusedPlan* f = fp_of(p);
  const int N = f->N;
  const int64_t H = N / 2, l0 = f->b.l0;
  PF_CK(to_tilemajor(N, Tq, f->b.Q, 1.0, true, p->work, f->b.l1));
  PF_CK(to_tilemajor(N, Td, f->b.D, 1.0, true, p->work, f->b.l1));
  PF_CK(stokes_form_r_gated(p, R, 0));
  if (!f->plan2d) {  // axes-(1, 2) transform of this slab's R (setup only)
    size_t ws = 0;
    long long dims2[2] = {N, N};
    PF_CK_FFT(cufftCreate(&f->plan2d));
    PF_CK_FFT(cufftSetAutoAllocation(f->plan2d, 0));
    PF_CK_FFT(cufftMakePlanMany64(f->plan2d, 2, dims2, nullptr, 1, (long long)N * N, nullptr, 1,
                                  (long long)N * (H + 1), CUFFT_D2Z, 3LL * l0, &ws));
    PF_CK_CUDA(cudaMalloc(&f->ws, ws > 0 ? ws : 256));
    PF_CK_CUDA(cudaMalloc(&f->spec, sizeof(double2) * 3 * (size_t)l0 * N * (H + 1)));
    PF_CK_FFT(cufftSetWorkArea(f->plan2d, f->ws));
    PF_CK_FFT(cufftSetStream(f->plan2d, p->work));
  }
  PF_CK_FFT(cufftExecD2Z(f->plan2d, (cufftDoubleReal*)R, (cufftDoubleComplex*)f->spec));
  const int grid = blocks_for((int64_t)3 * f->b.l0 * N * (N / 2 + 1));
  switch (N) {
    case 64: fz::k_split_yx<64><<<grid, kThreads, 0, p->work>>>(f->spec, f->b); break;
    case 128: fz::k_split_yx<128><<<grid, kThreads, 0, p->work>>>(f->spec, f->b); break;
    case 256: fz::k_split_yx<256><<<grid, kThreads, 0, p->work>>>(f->spec, f->b); break;
    case 512: fz::k_split_yx<512><<<grid, kThreads, 0, p->work>>>(f->spec, f->b); break;
    default: fz::k_split_yx<1024><<<grid, kThreads, 0, p->work>>>(f->spec, f->b); break;
  }
  PF_CK_CUDA(cudaGetLastError());
  switch (N) {
    case 64: PF_CK(compact_setup_t<64>(p, f)); break;
    case 128: PF_CK(compact_setup_t<128>(p, f)); break;
    case 256: PF_CK(compact_setup_t<256>(p, f)); break;
    case 512: PF_CK(compact_setup_t<512>(p, f)); break;
    default: PF_CK(compact_setup_t<1024>(p, f)); break;
  }
  f->lam_pore = p->sc.lam_pore_sq;  // local: enters the totals before the all-reduce
  p->sc.lam_pore_sq = 0.0;
  // release the setup-only transform (a 1024^3 slab of 2 ranks needs the memory)
  PF_CK_CUDA(cudaStreamSynchronize(p->work));
  cufftDestroy(f->plan2d);
  f->plan2d = 0;
  PF_CK_CUDA(cudaFree(f->ws));
  PF_CK_CUDA(cudaFree(f->spec));
  f->ws = nullptr;
  f->spec = nullptr;
  return PF_OK;
}

// Cold start (the whole state zero, as the reference's default): Q^ = D^ = 0 and
// the Y-space right-hand side is FFT(b 0 - 0) = 0, so setup needs no transform,
// exchange or scratch at all — only the compact layout.
int fused_slab_setup_zero(pf_plan* p, int64_t y_main, int64_t y_nyq) {
  FusedPlan* f = fp_of(p);
  double2 *Yy = f->b.Y, *Yyn = f->b.Yn, *Yx = f->b.Yx, *Yxn = f->b.Yxn;
  const int N = f->N;
  const size_t qd = (size_t)f->b.l1 * N * (N / 2) + (size_t)f->b.l1 * N;
  PF_CK_CUDA(cudaMemsetAsync(f->b.Q, 0, sizeof(double2) * qd, p->work));
  PF_CK_CUDA(cudaMemsetAsync(f->b.D, 0, sizeof(double2) * qd, p->work));
  PF_CK_CUDA(cudaMemsetAsync(Yy, 0, sizeof(double2) * y_main, p->work));
  PF_CK_CUDA(cudaMemsetAsync(Yyn, 0, sizeof(double2) * y_nyq, p->work));
  if (Yx != Yy) PF_CK_CUDA(cudaMemsetAsync(Yx, 0, sizeof(double2) * y_main, p->work));
  if (Yxn != Yyn) PF_CK_CUDA(cudaMemsetAsync(Yxn, 0, sizeof(double2) * y_nyq, p->work));
  switch (N) {
    case 64: PF_CK(compact_setup_t<64>(p, f)); break;
    case 128: PF_CK(compact_setup_t<128>(p, f)); break;
    case 256: PF_CK(compact_setup_t<256>(p, f)); break;
    case 512: PF_CK(compact_setup_t<512>(p, f)); break;
    default: PF_CK(compact_setup_t<1024>(p, f)); break;
  }
  f->lam_pore = p->sc.lam_pore_sq;
  p->sc.lam_pore_sq = 0.0;
  return PF_OK;
}

static fz::SpecArgs spec_args(pf_plan* p) {
  fz::SpecArgs sa;
  for (int i = 0; i < 3; ++i) {
    sa.kap[i] = p->kap[i];
    sa.ell[i] = p->ell[i];
    sa.g[i] = p->sc.g[i];
  }
  sa.nu = p->sc.nu;
  sa.inv_n = p->g.inv_n;
  sa.dn = p->g.dn;
  return sa;
}

template <int N>
static int fslab_pk_t(pf_plan* p) {
  FusedPlan* f = fp_of(p);
  const int pk_tiles = f->b.l1 * fz::PK2<N>::NCH + f->b.l1 / fz::PK2<N>::CP;
  fz::k_pk<N, true><<<pk_tiles, fz::PK2<N>::T, smem_pk<N>(), p->work>>>(f->b, spec_args(p), p->ctrl, f->tm_pk, 0, 0,
                                                                         pk_tiles);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

template <int N>
static int fslab_totals_t(pf_plan* p, double* totals) {
  FusedPlan* f = fp_of(p);
  const int pk_tiles = f->b.l1 * fz::PK2<N>::NCH + f->b.l1 / fz::PK2<N>::CP;
  fz::k_fslab_totals<<<1, kFinalizeThreads, 0, p->work>>>(f->b.part_rs, f->rs_rows, f->b.part_pk, pk_tiles,
                                                         f->lam_pore, totals);
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

// MI + RS over the component window [c0, c0 + nc): nc = 3 (one launch each, partial
// rows [0, nb_rs)) or nc = 1 (one component, so the exchange of the next
// component overlaps it; partial rows [c0 nb_rs, (c0 + 1) nb_rs) of 3 nb_rs).
// totals (may be null) = this rank's 9 sums once every component has run.
template <int N>
static int fslab_rs_t(pf_plan* p, int c0, int nc, double* totals) {
  FusedPlan* f = fp_of(p);
  fz::State st{p->s_u, p->s_ut, p->s_a, p->s_lam, p->s_solid};
  const int m_tiles = nc * (f->b.l0 * fz::M2<N>::NCH + f->b.l0 / fz::M2<N>::CM);
  f->b.c0 = c0;
  f->b.nc = nc;
  f->b.pst = nc == 3 ? f->nb_rs : 3 * f->nb_rs;
  f->b.poff = nc == 3 ? 0 : c0 * f->nb_rs;
  f->rs_rows = f->b.pst;
  fz::k_maxis<N, true, true><<<m_tiles, fz::M2<N>::T, smem_mi<N>(), p->work>>>(f->b, p->ctrl, f->tm_y, 0, f->tm_y);
  PF_CK_CUDA(cudaGetLastError());
  if (f->compact) {
    fz::k_rs_compact<N, true><<<f->nb_rs, fz::RS2<N>::T, fz::RSC<N>::bytes(f->c_cs), p->work>>>(
        f->b, st, compact_of(f), p->ctrl);
  } else {
    fz::k_rs<N, true><<<f->nb_rs, fz::RS2<N>::T, smem_rs<N>(), p->work>>>(f->b, st, p->ctrl);
  }
  PF_CK_CUDA(cudaGetLastError());
  f->b.c0 = 0;
  f->b.nc = 3;
  return totals ? fslab_totals_t<N>(p, totals) : PF_OK;
}

template <int N>
static int fslab_rsfix_t(pf_plan* p) {
  FusedPlan* f = fp_of(p);
  if (f->compact) {
    fz::k_rsfix_compact<N, true><<<f->nb_rs, fz::RS2<N>::T, smem_rsfix<N>(), p->work>>>(f->b, p->s_u, p->s_solid,
                                                                                      compact_of(f), p->ctrl);
  } else {
    fz::k_rsfix<N, true><<<f->nb_rs, fz::RS2<N>::T, smem_rsfix<N>(), p->work>>>(f->b, p->s_ut, p->ctrl);
  }
  PF_CK_CUDA(cudaGetLastError());
  return PF_OK;
}

// MF over the component window [c0, c0 + nc); `fix` runs the (gated) RSF pass of
// every component first, so it must be set on the first window of an iteration.
template <int N>
static int fslab_mf_t(pf_plan* p, int c0, int nc, bool fix) {
  FusedPlan* f = fp_of(p);
  if (fix) PF_CK(fslab_rsfix_t<N>(p));
  const int m_tiles = nc * (f->b.l0 * fz::M2<N>::NCH + f->b.l0 / fz::M2<N>::CM);
  f->b.c0 = c0;
  f->b.nc = nc;
  fz::k_maxis<N, false, true><<<m_tiles, fz::M2<N>::T, smem_mf<N>(), p->work>>>(f->b, p->ctrl, f->tm_xr, 0,
                                                                               f->tm_xr);
  PF_CK_CUDA(cudaGetLastError());
  f->b.c0 = 0;
  f->b.nc = 3;
  return PF_OK;
}

int fused_slab_pk(pf_plan* p) {
  switch (fp_of(p)->N) {
    case 64: return fslab_pk_t<64>(p);
    case 128: return fslab_pk_t<128>(p);
    case 256: return fslab_pk_t<256>(p);
    case 512: return fslab_pk_t<512>(p);
    default: return fslab_pk_t<1024>(p);
  }
}

#define PF_FSLAB_DISPATCH(fn, ...)        \
  switch (fp_of(p)->N) {                  \
    case 64: return fn<64>(__VA_ARGS__);  \
    case 128: return fn<128>(__VA_ARGS__); \
    case 256: return fn<256>(__VA_ARGS__); \
    case 512: return fn<512>(__VA_ARGS__); \
    default: return fn<1024>(__VA_ARGS__); \
  }

int fused_slab_rs(pf_plan* p, double* totals) { PF_FSLAB_DISPATCH(fslab_rs_t, p, 0, 3, totals) }
int fused_slab_rs_part(pf_plan* p, int comp) { PF_FSLAB_DISPATCH(fslab_rs_t, p, comp, 1, nullptr) }
int fused_slab_totals(pf_plan* p, double* totals) { PF_FSLAB_DISPATCH(fslab_totals_t, p, totals) }
int fused_slab_mf(pf_plan* p) { PF_FSLAB_DISPATCH(fslab_mf_t, p, 0, 3, true) }
int fused_slab_mf_part(pf_plan* p, int comp, int fix) { PF_FSLAB_DISPATCH(fslab_mf_t, p, comp, 1, fix != 0) }
#undef PF_FSLAB_DISPATCH

// Peer-memory exchange: device addresses of every rank's Y buffers (P2P-mapped
// into this process), or npeers = 0 to go back to the all_to_all exchange.
int fused_slab_set_peers(pf_plan* p, const uint64_t* yy, const uint64_t* yyn, const uint64_t* yx,
                         const uint64_t* yxn, int npeers) {
  FusedPlan* f = fp_of(p);
  if (npeers == 0) {
    f->b.peers = nullptr;
    return PF_OK;
  }
  const int P = f->N / f->b.l1;
  if (npeers != P || P > fz::kMaxRanks) {
    set_error("peer table needs one entry per rank (%d ranks, at most %d)", P, fz::kMaxRanks);
    return PF_ERR_ARG;
  }
  fz::Peers h{};
  for (int r = 0; r < P; ++r) {
    h.yy[r] = reinterpret_cast<double2*>(yy[r]);
    h.yyn[r] = reinterpret_cast<double2*>(yyn[r]);
    h.yx[r] = reinterpret_cast<double2*>(yx[r]);
    h.yxn[r] = reinterpret_cast<double2*>(yxn[r]);
  }
  if (!f->peers) PF_CK_CUDA(cudaMalloc(&f->peers, sizeof(fz::Peers)));
  PF_CK_CUDA(cudaMemcpy(f->peers, &h, sizeof(h), cudaMemcpyHostToDevice));
  f->b.peers = f->peers;
  return PF_OK;
}

// Q^ back to the slab T layout (unscaled) and the compact multipliers materialised.
int fused_slab_end(pf_plan* p, double2* Tq) {
  FusedPlan* f = fp_of(p);
  const int N = f->N;
  PF_CK(to_tilemajor(N, f->b.Q, Tq, 1.0, false, p->work, f->b.l1));
  if (f->compact) {
    const int64_t rows = (int64_t)f->b.l0 * N;
    const int nb = blocks_for(3 * rows * 32);
    switch (N) {
      case 64: fz::k_compact_move<64><<<nb, kThreads, 0, p->work>>>(p->s_solid, compact_of(f), p->s_ut, p->s_a, p->s_lam, p->s_u, 1, rows); break;
      case 128: fz::k_compact_move<128><<<nb, kThreads, 0, p->work>>>(p->s_solid, compact_of(f), p->s_ut, p->s_a, p->s_lam, p->s_u, 1, rows); break;
      case 256: fz::k_compact_move<256><<<nb, kThreads, 0, p->work>>>(p->s_solid, compact_of(f), p->s_ut, p->s_a, p->s_lam, p->s_u, 1, rows); break;
      case 512: fz::k_compact_move<512><<<nb, kThreads, 0, p->work>>>(p->s_solid, compact_of(f), p->s_ut, p->s_a, p->s_lam, p->s_u, 1, rows); break;
      default: fz::k_compact_move<1024><<<nb, kThreads, 0, p->work>>>(p->s_solid, compact_of(f), p->s_ut, p->s_a, p->s_lam, p->s_u, 1, rows); break;
    }
    PF_CK_CUDA(cudaGetLastError());
  }
  return PF_OK;
}

}  // namespace pf
