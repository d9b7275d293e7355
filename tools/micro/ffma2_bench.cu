// Issue throughput of packed FP32x2 FMA (FFMA2, sm_100) vs scalar FFMA.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k1(float *out, int it, float a, float b) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; k++) x[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < it; i++)
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = fmaf(x[k], a, b);
  float s = 0;
#pragma unroll
  for (int k = 0; k < 16; k++) s += x[k];
  if (s == 12345.f) out[0] = s;
}

__global__ void k2(float *out, int it, float a, float b) {
  float2 x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = make_float2(threadIdx.x * 1e-3f + k, k + 0.5f);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int i = 0; i < it; i++)
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = __ffma2_rn(x[k], A, B);
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s += x[k].x + x[k].y;
  if (s == 12345.f) out[0] = s;
}

int main() {
  float *out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 148 * 8, threads = 256, it = 4096;
  for (int rep = 0; rep < 3; rep++) {
    for (int v = 0; v < 2; v++) {
      cudaEventRecord(e0);
      if (v == 0) k1<<<blocks, threads>>>(out, it, 0.9999f, 1e-4f);
      else k2<<<blocks, threads>>>(out, it, 0.9999f, 1e-4f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 16 * it * (double)blocks * threads;
      if (rep == 2) printf("%s: %.3f ms, %.1f TFLOP/s\n", v ? "FFMA2" : "FFMA ", ms, flops / ms / 1e9);
    }
  }
  return 0;
}
