// Micro-benchmark (measurement only, not part of the library): read + write
// PK-shaped pencils of a [3][256][256][128] complex128 array in place — per
// (k1, column chunk) tile, 3 x 256 rows of CP x 16 bytes at a 512 KB row stride —
// with plain per-thread 16-byte loads / stores, to see what the access pattern
// alone sustains against the axis-1 pattern (rows of 128 B at a 2 KB stride).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pc pencil_copy.cu && /tmp/pc
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 256, H = 128;

template <int CP, int MODE>  // MODE 0: PK pencils (i0 stride 512 KB); 1: axis-1 pencils (k1 stride 2 KB)
__global__ void __launch_bounds__(256) k_copy(double2* Y, int tiles) {
  const int NCH = H / CP;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int a = tile / NCH, ch = tile % NCH;
    double2 v[3 * N * CP / 256];
#pragma unroll
    for (int j = 0; j < 3 * N * CP / 256; ++j) {
      const int idx = threadIdx.x + 256 * j, q = idx % CP, e = (idx / CP) % N, c = idx / (CP * N);
      const size_t o = MODE == 0 ? ((size_t)(c * N + e) * N + a) * H + ch * CP + q
                                 : ((size_t)(c * N + a) * N + e) * H + ch * CP + q;
      v[j] = Y[o];
    }
#pragma unroll
    for (int j = 0; j < 3 * N * CP / 256; ++j) {
      const int idx = threadIdx.x + 256 * j, q = idx % CP, e = (idx / CP) % N, c = idx / (CP * N);
      const size_t o = MODE == 0 ? ((size_t)(c * N + e) * N + a) * H + ch * CP + q
                                 : ((size_t)(c * N + a) * N + e) * H + ch * CP + q;
      v[j].x += 1.0;
      Y[o] = v[j];
    }
  }
}

template <int CP, int MODE>
void run(double2* Y, int bps) {
  const int tiles = N * (H / CP);
  const int grid = 148 * bps;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) k_copy<CP, MODE><<<grid, 256>>>(Y, tiles);
  cudaEventRecord(a);
  const int R = 10;
  for (int r = 0; r < R; ++r) k_copy<CP, MODE><<<grid, 256>>>(Y, tiles);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = 2.0 * 3 * N * N * H * 16;
  printf("mode %d CP %d blocks/SM %d: %.3f ms  %.0f GB/s\n", MODE, CP, bps, ms / R, bytes / (ms / R * 1e-3) / 1e9);
}

int main() {
  double2* Y;
  cudaMalloc(&Y, sizeof(double2) * 3 * N * N * H);
  cudaMemset(Y, 0, sizeof(double2) * 3 * N * N * H);
  for (int bps : {2, 4, 8}) {
    run<4, 0>(Y, bps);
    run<8, 0>(Y, bps);
    run<4, 1>(Y, bps);
    run<8, 1>(Y, bps);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
