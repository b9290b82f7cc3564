// Blur probe: time the exact separable-blur axis kernels on a C2-sized grid
// (1024^2 x 14, stride 16) for several half-widths, and check candidate
// variants bit-for-bit against the production kernel.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#include "blur.cuh"
#include "blur_fast.cuh"

using namespace plas;

int main() {
  const int side = 1024, D = 14, S = 16;
  const long long n = (long long)side * side;
  float *in, *out_ref, *out_new;
  double* w;
  int* fb;
  cudaMalloc(&in, n * S * 4);
  cudaMalloc(&out_ref, n * S * 4);
  cudaMalloc(&out_new, n * S * 4);
  cudaMalloc(&w, 4096 * 8);
  cudaMalloc(&fb, (n * S + 16) * 4);
  std::vector<float> h(n * S, 0.f);
  srand(3);
  for (long long i = 0; i < n; i++)
    for (int c = 0; c < D; c++) {
      float u1 = (rand() + 1.f) / (RAND_MAX + 2.f), u2 = (rand() + 1.f) / (RAND_MAX + 2.f);
      h[i * S + c] = sqrtf(-2.f * logf(u1)) * cosf(6.2831853f * u2);
    }
  cudaMemcpy(in, h.data(), n * S * 4, cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int hs[] = {2, 8, 16, 40, 84, 200, 511};
  std::vector<float> a(n * S), b(n * S);
  for (int hw : hs) {
    double r = hw - 0.3;
    double sigma = r / 2.0, s2 = sigma * sigma;
    std::vector<double> phi(2 * hw + 1);
    double sum = 0;
    for (int x = -hw; x <= hw; x++) phi[x + hw] = exp(-0.5 / s2 * x * x);
    for (double v : phi) sum += v;
    std::vector<double> wh(hw + 1);
    for (int j = 0; j <= hw; j++) wh[j] = phi[hw + j] / sum;
    cudaMemcpy(w, wh.data(), 8 * (hw + 1), cudaMemcpyHostToDevice);
    BlurLevelRef lv{nullptr, nullptr, nullptr, nullptr, hw, w};
    for (int axis = 0; axis < 2; axis++) {
      const int grid = sms * 8;
      float t_ref = 0, t_new = 0;
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        if (axis == 0)
          blur_axis_kernel<float, float, 0, 0><<<grid, 256>>>(in, out_ref, side, side, D, S, lv, nullptr);
        else
          blur_axis_kernel<float, float, 0, 1><<<grid, 256>>>(in, out_ref, side, side, D, S, lv, nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&t_ref, e0, e1);
        cudaMemset(fb, 0, 64);
        cudaEventRecord(e0);
        launch_blur_fast<float, float, 0>(axis, in, out_new, side, side, D, S, lv, nullptr, fb, sms, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&t_new, e0, e1);
      }
      cudaMemcpy(a.data(), out_ref, n * S * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), out_new, n * S * 4, cudaMemcpyDeviceToHost);
      long long bad = 0;
      for (long long i = 0; i < n; i++)
        for (int c = 0; c < D; c++)
          if (a[i * S + c] != b[i * S + c]) bad++;
      int nfb;
      cudaMemcpy(&nfb, fb, 4, cudaMemcpyDeviceToHost);
      double ops = (double)n * D * (3.0 * hw + 1);
      printf("h %4d axis %d  ref %8.1f us (%5.1f%% fp64 peak)  new %8.1f us  fallbacks %d  mismatches %lld\n", hw,
             axis, 1e3 * t_ref, 100.0 * ops / (t_ref * 1e-3) / 18.4e12, 1e3 * t_new, nfb, bad);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
