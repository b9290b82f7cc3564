// Pass-kernel probe: time the production gather (pass_kernel) and tile
// (tile_pass_kernel) kernels for one PLAS pass at several block sizes on a
// C2-sized grid (1024^2 x 14, rows padded to 16 floats).  Compile variants
// with -DPLAS_PASS_MINB=.. -DPLAS_TILE_MINB=.. -DPLAS_CHUNK_UNROLL=..
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#include "assign.cuh"

using namespace plas;

int main(int argc, char** argv) {
  const int side = 1024, D = 14, S = 16;
  const long long n = (long long)side * side;
  float *feat, *target;
  int* idx;
  double *dcache, *partials;
  int* counters;
  Ctrl* dctrl;
  cudaMalloc(&feat, n * S * 4);
  cudaMalloc(&target, n * S * 4);
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&dcache, n * 8);
  cudaMalloc(&partials, 4096 * 8);
  cudaMalloc(&counters, 64);
  cudaMalloc(&dctrl, sizeof(Ctrl));
  std::vector<float> h(n * S);
  srand(1);
  for (auto& v : h) v = (float)rand() / RAND_MAX;
  cudaMemcpy(feat, h.data(), n * S * 4, cudaMemcpyHostToDevice);
  for (auto& v : h) v = (float)rand() / RAND_MAX;
  cudaMemcpy(target, h.data(), n * S * 4, cudaMemcpyHostToDevice);
  cudaMemset(dcache, 0, n * 8);
  cudaMemset(idx, 0, n * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, pass_kernel<true, false>);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass_kernel<true, false>, 256, 0);
  const int grid = sms * occ;
  const size_t tsm = 2 * tile_stage_bytes(16, S);
  cudaFuncSetAttribute(tile_pass_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
  int tocc = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tocc, tile_pass_kernel<false>, TILE_THREADS, tsm);
  cudaFuncAttributes ta;
  cudaFuncGetAttributes(&ta, tile_pass_kernel<false>);
  printf("gather: regs %d local %zu occ %d grid %d | tile: regs %d local %zu occ %d smem %zu\n", fa.numRegs,
         fa.localSizeBytes, occ, grid, ta.numRegs, ta.localSizeBytes, tocc, tsm);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int betas[] = {16, 24, 32, 64, 128, 256, 512};
  for (int beta : betas) {
    Ctrl c{};
    c.side = side;
    c.beta = beta;
    c.rng_mode = 1;
    c.S = S;
    set_pass_geometry(&c, beta / 3, beta / 5, 0x1234567ull + beta);
    cudaMemcpy(dctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice);
    float ms[2] = {0, 0};
    for (int var = 0; var < 2; var++) {
      if (var == 1 && !use_tile(beta, S)) continue;
      for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        if (var == 0)
          pass_kernel<true, false><<<grid, 256>>>(feat, idx, target, dcache, D, S, dctrl, nullptr, 0, partials, counters);
        else
          tile_pass_kernel<false><<<sms * tocc, TILE_THREADS, tsm>>>(feat, idx, target, dcache, D, S, dctrl, nullptr, 0,
                                                                    partials, counters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms[var], e0, e1);
      }
    }
    printf("beta %4d  gather %8.1f us  tile %8.1f us   (alg GB/s: gather %.0f)\n", beta, 1e3 * ms[0], 1e3 * ms[1],
           n * 8.0 * D / (ms[0] * 1e6));
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
