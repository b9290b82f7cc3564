// Achievable HBM bandwidth of the K3 access pattern: quads of 4 cells, each
// cell a 64-byte feature row and a 64-byte target row, 4 lanes per row
// (16-byte chunks), cells sequential / random within blocks / random over the
// grid.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gather_bw.cu -o tools/gather_bw
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>
#include <random>

template <int R>
__global__ void __launch_bounds__(256) gather(const float4* __restrict__ F, const float4* __restrict__ T,
                                              const int* __restrict__ cells, long long nquads, float* out) {
  const int lane = threadIdx.x & 31, c = lane & 3;
  const long long nq_round = (long long)gridDim.x * 64;  // quads per grid-wide round (8 per warp)
  float acc = 0.f;
  for (long long q0 = (long long)blockIdx.x * 64 + (threadIdx.x >> 2); q0 < nquads; q0 += nq_round * R) {
    float4 f[R][4], t[R][4];
#pragma unroll
    for (int r = 0; r < R; r++) {
      const long long q = q0 + r * nq_round;
      if (q < nquads) {
        const int4 cl = *reinterpret_cast<const int4*>(cells + 4 * q);
        const int cs[4] = {cl.x, cl.y, cl.z, cl.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
          f[r][i] = F[(long long)cs[i] * 4 + c];
          t[r][i] = __ldg(&T[(long long)cs[i] * 4 + c]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; i++) f[r][i] = t[r][i] = make_float4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
      for (int i = 0; i < 4; i++) acc += f[r][i].x * t[r][i].y + f[r][i].z - t[r][i].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const int side = 1024, n = side * side;
  const long long nq = n / 4;
  float4 *F, *T;
  int* cells;
  float* out;
  cudaMalloc(&F, (size_t)n * 64);
  cudaMalloc(&T, (size_t)n * 64);
  cudaMalloc(&cells, (size_t)n * 4);
  cudaMalloc(&out, 4);
  cudaMemset(F, 0, (size_t)n * 64);
  cudaMemset(T, 0, (size_t)n * 64);
  char* flush;
  cudaMalloc(&flush, 256 << 20);
  std::mt19937 rng(1);
  for (int pat = 0; pat < 4; pat++) {
    std::vector<int> h(n);
    const char* name = "";
    if (pat == 0) {
      name = "sequential";
      for (int i = 0; i < n; i++) h[i] = i;
    } else if (pat == 3) {
      name = "random over grid";
      for (int i = 0; i < n; i++) h[i] = i;
      std::shuffle(h.begin(), h.end(), rng);
    } else {
      const int beta = pat == 1 ? 16 : 122;
      name = pat == 1 ? "random in 16x16 blocks" : "random in 122x122 blocks";
      int k = 0;
      for (int by = 0; by < side; by += beta)
        for (int bx = 0; bx < side; bx += beta) {
          std::vector<int> blk;
          for (int y = by; y < std::min(side, by + beta); y++)
            for (int x = bx; x < std::min(side, bx + beta); x++) blk.push_back(y * side + x);
          std::shuffle(blk.begin(), blk.end(), rng);
          for (int v : blk) h[k++] = v;
        }
    }
    cudaMemcpy(cells, h.data(), (size_t)n * 4, cudaMemcpyHostToDevice);
    for (int R : {1, 2, 4}) {
      for (int occ_grid : {148 * 4, 148 * 8}) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e9f;
        for (int rep = 0; rep < 5; rep++) {
          cudaMemset(flush, rep, 256 << 20);
          cudaEventRecord(e0);
          if (R == 1) gather<1><<<occ_grid, 256>>>(F, T, cells, nq, out);
          if (R == 2) gather<2><<<occ_grid, 256>>>(F, T, cells, nq, out);
          if (R == 4) gather<4><<<occ_grid, 256>>>(F, T, cells, nq, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          best = std::min(best, ms);
        }
        printf("%-26s R=%d grid=%4d  %7.2f us  %7.1f GB/s\n", name, R, occ_grid, best * 1e3,
               (double)n * 128 / (best * 1e-3) / 1e9);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
