// Micro-benchmark (measurement only): in-place read + write of Y = 3 x 256^2 x 128
// complex128 through PK-shaped tiles (fixed k1, CP = 4 columns, all i0) and
// axis-1-shaped tiles (fixed i0, CM = 8 columns, all k1) under candidate layouts:
//   BI = 1   : [c][i0][k1][k2]            (current)
//   BI = 256 : [c][k1][i0][k2]            (k1-major)
//   BI = b   : [c][i0/b][k1][i0%b][k2]    (i0 blocked by b)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o layout_copy layout_copy.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 256, H = 128;

template <int BI>
__device__ __forceinline__ size_t yoff(int c, int i0, int k1, int k2) {
  if (BI >= 1000) {  // plane pitch N*H + (BI - 1000) complex
    return ((size_t)c * N + i0) * (size_t)(N * H + (BI - 1000)) + (size_t)k1 * H + k2;
  }
  const int ib = i0 / BI, ii = i0 % BI;
  return ((((size_t)c * (N / BI) + ib) * N + k1) * BI + ii) * H + k2;
}

template <int BI, int PK>
__global__ void __launch_bounds__(256) k_copy(double2* Y) {
  // PK: tile = (k1, chunk of 4 columns), 3 comps x 256 i0 x 4 = 3072 elements (12 / thread)
  // axis-1: tile = (c, i0, chunk of 8 columns), 256 k1 x 8 = 2048 elements (8 / thread)
  constexpr int CP = PK ? 4 : 8, NCH = H / CP;
  constexpr int PER = PK ? 12 : 8;
  constexpr int TILES = PK ? N * NCH : 3 * N * NCH;
  for (int tile = blockIdx.x; tile < TILES; tile += gridDim.x) {
    const int ch = tile % NCH, a = (tile / NCH) % N, c0 = tile / (N * NCH);
    double2 v[PER];
    size_t o[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int idx = threadIdx.x + 256 * j, q = idx % CP, e = (idx / CP) % N;
      if (PK) o[j] = yoff<BI>(idx / (CP * N), e, a, ch * CP + q);
      else o[j] = yoff<BI>(c0, a, e, ch * CP + q);
      v[j] = Y[o[j]];
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      v[j].x += 1.0;
      Y[o[j]] = v[j];
    }
  }
}

template <int BI, int PK>
void run(double2* Y, int bps) {
  const int grid = 148 * bps;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) k_copy<BI, PK><<<grid, 256>>>(Y);
  cudaEventRecord(a);
  const int R = 10;
  for (int r = 0; r < R; ++r) k_copy<BI, PK><<<grid, 256>>>(Y);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = 2.0 * 3 * N * N * H * 16;
  printf("BI %3d %s blocks/SM %d: %.3f ms  %.0f GB/s\n", BI, PK ? "PK   " : "axis1", bps, ms / R,
         bytes / (ms / R * 1e-3) / 1e9);
}

template <int BI>
void both(double2* Y) {
  for (int bps : {4, 8}) {
    run<BI, 1>(Y, bps);
    run<BI, 0>(Y, bps);
  }
}

int main() {
  double2* Y;
  cudaMalloc(&Y, sizeof(double2) * 3 * N * (N * H + 4096));
  cudaMemset(Y, 0, sizeof(double2) * 3 * N * (N * H + 4096));
  both<1>(Y);
  both<4>(Y);
  both<1008>(Y);
  both<1016>(Y);
  both<1032>(Y);
  both<1064>(Y);
  both<1128>(Y);
  both<1256>(Y);
  both<1512>(Y);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
