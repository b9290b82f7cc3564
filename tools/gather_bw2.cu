// Achievable HBM bandwidth of K3's access pattern, layout study.
//   stream : contiguous float4 read of the feature and target arrays (the
//            read roofline of 2 x 64 MB at this size)
//   split  : quads of 4 cells, 4 lanes per 64-byte row, feature and target
//            rows in two separate arrays (the round-1 layout)
//   inter  : the same lanes and loads, but the cell's feature row and target
//            row adjacent in one 128-byte record (one cache line per cell)
// for cells sequential / random inside beta x beta blocks / random over the
// grid, with R quads per 4-lane group in flight.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gather_bw2.cu -o tools/gather_bw2
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

__global__ void stream_read(const float4* __restrict__ A, long long n4, float* out) {
  float acc = 0.f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = __ldg(A + i);
    acc += v.x + v.y * v.z - v.w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

// FS: float4 offset of a cell's feature row; TS: of its target row
template <int R, bool INTER>
__global__ void __launch_bounds__(256) gather(const float4* __restrict__ F, const float4* __restrict__ T,
                                              const int* __restrict__ cells, long long nquads, float* out) {
  const int lane = threadIdx.x & 31, c = lane & 3;
  const long long nq_round = (long long)gridDim.x * 64;
  float acc = 0.f;
  for (long long q0 = (long long)blockIdx.x * 64 + (threadIdx.x >> 2); q0 < nquads; q0 += nq_round * R) {
    float4 f[R][4], t[R][4];
#pragma unroll
    for (int r = 0; r < R; r++) {
      const long long q = q0 + r * nq_round;
      const long long qq = q < nquads ? q : 0;
      const int4 cl = __ldg(reinterpret_cast<const int4*>(cells + 4 * qq));
      const int cs[4] = {cl.x, cl.y, cl.z, cl.w};
#pragma unroll
      for (int i = 0; i < 4; i++) {
        if (INTER) {
          f[r][i] = F[(long long)cs[i] * 8 + c];
          t[r][i] = __ldg(&F[(long long)cs[i] * 8 + 4 + c]);
        } else {
          f[r][i] = F[(long long)cs[i] * 4 + c];
          t[r][i] = __ldg(&T[(long long)cs[i] * 4 + c]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
      for (int i = 0; i < 4; i++) acc += f[r][i].x * t[r][i].y + f[r][i].z - t[r][i].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

__global__ void flush_read(const float4* __restrict__ A, long long n4, float* out) {
  float acc = 0.f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    acc += __ldcg(A + i).x;
  if (acc == 1234.5f) out[0] = acc;
}

int main(int argc, char** argv) {
  const bool write_flush = argc > 1 && argv[1][0] == 'w';
  const int side = 1024, n = side * side;
  const long long nq = n / 4;
  float4 *F, *T;
  int* cells;
  float* out;
  cudaMalloc(&F, (size_t)n * 128);  // big enough for the interleaved records
  cudaMalloc(&T, (size_t)n * 64);
  cudaMalloc(&cells, (size_t)n * 4);
  cudaMalloc(&out, 4);
  cudaMemset(F, 0, (size_t)n * 128);
  cudaMemset(T, 0, (size_t)n * 64);
  char* flush;
  cudaMalloc(&flush, 512 << 20);
  cudaMemset(flush, 0, 512 << 20);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto&& launch) {
    float best = 1e9f;
    for (int rep = 0; rep < 7; rep++) {
      if (write_flush)
        cudaMemsetAsync(flush, rep, 512 << 20);
      else
        flush_read<<<sms * 8, 256>>>((const float4*)flush, (512ll << 20) / 16, out);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep >= 2) best = std::min(best, ms);
    }
    return best;
  };
  for (int g : {sms * 4, sms * 8, sms * 16}) {
    const float ms = timeit([&] { stream_read<<<g, 256>>>(F, (long long)n * 8, out); });
    printf("stream 128 MB                 grid=%5d  %7.2f us  %7.1f GB/s\n", g, ms * 1e3, (double)n * 128 / (ms * 1e-3) / 1e9);
  }
  std::mt19937 rng(1);
  const int betas[] = {0, 16, 32, 128, 512, -1};
  for (int beta : betas) {
    std::vector<int> h(n);
    char name[64];
    if (beta == 0) {
      snprintf(name, sizeof(name), "sequential");
      for (int i = 0; i < n; i++) h[i] = i;
    } else if (beta < 0) {
      snprintf(name, sizeof(name), "random over grid");
      for (int i = 0; i < n; i++) h[i] = i;
      std::shuffle(h.begin(), h.end(), rng);
    } else {
      snprintf(name, sizeof(name), "random in %dx%d blocks", beta, beta);
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
    for (int inter = 0; inter < 2; inter++)
      for (int R : {1, 2, 4})
        for (int g : {sms * 4, sms * 8}) {
          const float ms = timeit([&] {
            if (inter) {
              if (R == 1) gather<1, true><<<g, 256>>>(F, T, cells, nq, out);
              else if (R == 2) gather<2, true><<<g, 256>>>(F, T, cells, nq, out);
              else gather<4, true><<<g, 256>>>(F, T, cells, nq, out);
            } else {
              if (R == 1) gather<1, false><<<g, 256>>>(F, T, cells, nq, out);
              else if (R == 2) gather<2, false><<<g, 256>>>(F, T, cells, nq, out);
              else gather<4, false><<<g, 256>>>(F, T, cells, nq, out);
            }
          });
          printf("%-26s %-5s R=%d grid=%5d  %7.2f us  %7.1f GB/s\n", name, inter ? "inter" : "split", R, g,
                 ms * 1e3, (double)n * 128 / (ms * 1e-3) / 1e9);
        }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
