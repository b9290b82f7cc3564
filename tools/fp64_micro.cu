// Micro-benchmark: per-SM throughput of the FP64 ops the exact PLAS kernels use
// (DADD, DMUL, DFMA, F2F f32->f64, DSQRT) on this GPU.  Prints Gop/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, float* fin, int iters) {
  double a = threadIdx.x * 1e-3 + 1.0, b = 1.0000001, c = 0.5, d = 0.25, e = 0.125, f = 2.0, g = 3.0, h = 4.0;
  float x = fin[threadIdx.x & 31];
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      if (OP == 0) { a = __dadd_rn(a, b); c = __dadd_rn(c, b); d = __dadd_rn(d, b); e = __dadd_rn(e, b); f = __dadd_rn(f, b); g = __dadd_rn(g, b); h = __dadd_rn(h, b); }
      if (OP == 1) { a = __dmul_rn(a, b); c = __dmul_rn(c, b); d = __dmul_rn(d, b); e = __dmul_rn(e, b); f = __dmul_rn(f, b); g = __dmul_rn(g, b); h = __dmul_rn(h, b); }
      if (OP == 2) { a = fma(a, b, c); d = fma(d, b, c); e = fma(e, b, c); f = fma(f, b, c); g = fma(g, b, c); h = fma(h, b, c); c = fma(c, b, 1e-9); }
      if (OP == 3) { a += (double)x; c += (double)(x + 1.f); d += (double)(x + 2.f); e += (double)(x + 3.f); f += (double)(x + 4.f); g += (double)(x + 5.f); h += (double)(x + 6.f); x += 1e-7f; }
      if (OP == 4) { a = __dsqrt_rn(a); c = __dsqrt_rn(c); d = __dsqrt_rn(d); e = __dsqrt_rn(e); f = __dsqrt_rn(f); g = __dsqrt_rn(g); h = __dsqrt_rn(h); a += 1.0; c += 1.0; d += 1.0; e += 1.0; f += 1.0; g += 1.0; h += 1.0; }
      if (OP == 5) { float y = x; float z = x * 1.1f; y = __fadd_rn(y, z); z = __fmul_rn(z, 1.0000001f); x = y + z * 1e-9f; a += x; }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + c + d + e + f + g + h;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; float* fin;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaMalloc(&fin, 128); cudaMemset(fin, 0, 128);
  const char* names[] = {"DADD", "DMUL", "DFMA", "F2F.F64.F32(+DADD)", "DSQRT(+DADD)", "FP32 mix"};
  const int ops_per_iter[] = {7, 7, 7, 7, 7, 2};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2000;
  for (int op = 0; op < 6; op++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      switch (op) {
        case 0: k<0><<<sms * 8, 256>>>(out, fin, iters); break;
        case 1: k<1><<<sms * 8, 256>>>(out, fin, iters); break;
        case 2: k<2><<<sms * 8, 256>>>(out, fin, iters); break;
        case 3: k<3><<<sms * 8, 256>>>(out, fin, iters); break;
        case 4: k<4><<<sms * 8, 256>>>(out, fin, iters / 8); break;
        case 5: k<5><<<sms * 8, 256>>>(out, fin, iters); break;
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double n = (double)sms * 8 * 256 * (op == 4 ? iters / 8 : iters) * 16 * ops_per_iter[op];
      if (rep) printf("%-22s %8.1f Gop/s  (%.2f ops/clk/SM at 1.965 GHz)\n", names[op], n / ms / 1e6, n / ms / 1e6 / sms / 1.965);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
