// Probe: TMA gather4 (cp.async.bulk.tensor.2d ... tile::gather4) of random
// 64-byte rows into a shared-memory ring, vs plain per-lane LDG.128 gathers.
// Checks that the rows land where expected (sum check) and times both on a
// C2-sized workload (N = 1M cells, 16-float rows, groups of 4 random cells
// inside blocks of beta x beta).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tma_gather_probe tools/tma_gather_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, int c0, int r0, int r1, int r2, int r3,
                                        unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

constexpr int NST = 4;          // ring stages
constexpr int GPB = 64;         // groups per batch (8 consumer warps x 8 groups)
constexpr int STAGE_B = GPB * 4 * 64 * 2;  // F + T rows

__global__ void __launch_bounds__(288, 1) tma_kernel(const __grid_constant__ CUtensorMap tf,
                                                     const __grid_constant__ CUtensorMap tt,
                                                     const int4* __restrict__ groups, int G, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned long long full[NST], empty[NST];
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nb = (G + GPB - 1) / GPB;
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  if (threadIdx.x >= 256) {
    for (int it = 0, b = blockIdx.x; b < nb; it++, b += gridDim.x) {
      const int st = it % NST;
      if (it >= NST) mbar_wait(&empty[st], (unsigned)((it / NST - 1) & 1));
      unsigned char* sF = sm + st * STAGE_B;
      unsigned char* sT = sF + GPB * 256;
      if (lane == 0) mbar_expect_tx(&full[st], STAGE_B);
      __syncwarp();
      for (int q = lane; q < GPB; q += 32) {
        const int g = b * GPB + q;
        int4 c = g < G ? groups[g] : make_int4(0, 0, 0, 0);
        gather4(sF + q * 256, &tf, 0, c.x, c.y, c.z, c.w, &full[st]);
        gather4(sT + q * 256, &tt, 0, c.x, c.y, c.z, c.w, &full[st]);
      }
    }
  } else {
    const int w = threadIdx.x >> 5, s = lane & 3, gl = lane >> 2;
    for (int it = 0, b = blockIdx.x; b < nb; it++, b += gridDim.x) {
      const int st = it % NST;
      mbar_wait(&full[st], (unsigned)((it / NST) & 1));
      const float4* sF = reinterpret_cast<const float4*>(sm + st * STAGE_B);
      const float4* sT = sF + GPB * 16;
      const int q = w * 8 + gl;
      if (b * GPB + q < G) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const float4 f = sF[q * 16 + j * 4 + s], t = sT[q * 16 + j * 4 + s];
          acc += (double)(f.x - t.x) + f.y + f.z + f.w + t.y;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) atomicAdd(out, acc);
}

__global__ void __launch_bounds__(256) ldg_kernel(const float* __restrict__ F, const float* __restrict__ T,
                                                  const int4* __restrict__ groups, int G, double* out) {
  const int lane = threadIdx.x & 31, s = lane & 3;
  double acc = 0.0;
  for (int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 2; g < G; g += (gridDim.x * blockDim.x) >> 2) {
    const int4 c = groups[g];
    const int cs[4] = {c.x, c.y, c.z, c.w};
    float4 f[4], t[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      f[j] = __ldg(reinterpret_cast<const float4*>(F + (long long)cs[j] * 16) + s);
      t[j] = __ldg(reinterpret_cast<const float4*>(T + (long long)cs[j] * 16) + s);
    }
#pragma unroll
    for (int j = 0; j < 4; j++) acc += (double)(f[j].x - t[j].x) + f[j].y + f[j].z + f[j].w + t[j].y;
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) atomicAdd(out, acc);
}

int main(int argc, char** argv) {
  const int side = argc > 1 ? atoi(argv[1]) : 1024;
  const int beta = argc > 2 ? atoi(argv[2]) : 512;
  const int box_rows = argc > 3 ? atoi(argv[3]) : 1;
  const long long N = (long long)side * side;
  const int G = (int)(N / 4);
  std::vector<float> hF(N * 16), hT(N * 16);
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  for (auto& v : hF) v = U(rng);
  for (auto& v : hT) v = U(rng);
  // groups: random quads inside beta x beta blocks, blocks in row-major order
  std::vector<int4> hg;
  hg.reserve(G);
  for (int by = 0; by < side; by += beta)
    for (int bx = 0; bx < side; bx += beta) {
      std::vector<int> cells;
      for (int y = by; y < std::min(side, by + beta); y++)
        for (int x = bx; x < std::min(side, bx + beta); x++) cells.push_back(y * side + x);
      std::shuffle(cells.begin(), cells.end(), rng);
      for (size_t i = 0; i + 3 < cells.size(); i += 4) hg.push_back(make_int4(cells[i], cells[i + 1], cells[i + 2], cells[i + 3]));
    }
  double want = 0.0;
  for (auto& c : hg) {
    const int cs[4] = {c.x, c.y, c.z, c.w};
    for (int j = 0; j < 4; j++)
      for (int s = 0; s < 4; s++) {
        const float* f = &hF[(long long)cs[j] * 16 + 4 * s];
        const float* t = &hT[(long long)cs[j] * 16 + 4 * s];
        want += (double)(f[0] - t[0]) + f[1] + f[2] + f[3] + t[1];
      }
  }
  float *F, *T, *flush;
  int4* dg;
  double* dout;
  CK(cudaMalloc(&F, N * 64));
  CK(cudaMalloc(&T, N * 64));
  CK(cudaMalloc(&flush, 256 << 20));
  CK(cudaMalloc(&dg, sizeof(int4) * hg.size()));
  CK(cudaMalloc(&dout, 8));
  CK(cudaMemcpy(F, hF.data(), N * 64, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(T, hT.data(), N * 64, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dg, hg.data(), sizeof(int4) * hg.size(), cudaMemcpyHostToDevice));
  const int Gr = (int)hg.size();

  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tf, tt;
  for (int k = 0; k < 2; k++) {
    cuuint64_t dims[2] = {16, (cuuint64_t)N};
    cuuint64_t strides[1] = {64};
    cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(k ? &tt : &tf, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, k ? (void*)T : (void*)F, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  }
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int smem = NST * STAGE_B;
  CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma_kernel, 288, smem));
  printf("side %d beta %d groups %d  tma: %d CTAs/SM, smem %d\n", side, beta, Gr, occ, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; mode++) {
    float best = 1e9, got_ok = 1;
    for (int rep = 0; rep < 6; rep++) {
      CK(cudaMemset(dout, 0, 8));
      CK(cudaMemset(flush, rep, 256 << 20));
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      if (mode == 0) tma_kernel<<<sms * occ, 288, smem>>>(tf, tt, dg, Gr, dout);
      else ldg_kernel<<<sms * 8, 256>>>(F, T, dg, Gr, dout);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
      double got;
      CK(cudaMemcpy(&got, dout, 8, cudaMemcpyDeviceToHost));
      if (fabs(got - want) > 1e-6 * (1 + fabs(want))) got_ok = 0;
      if (rep == 0) printf("  %s sum %.6f want %.6f\n", mode ? "ldg" : "tma", got, want);
    }
    printf("%s: best %.2f us  %s  (%.2f TB/s of 128-B row pairs)\n", mode ? "ldg" : "tma", best * 1e3,
           got_ok ? "OK" : "MISMATCH", (double)Gr * 4 * 128 / (best * 1e-3) / 1e12);
  }
  return 0;
}
