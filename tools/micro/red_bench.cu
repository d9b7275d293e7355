// Throughput of coalesced global reductions (RED) by type on this GPU: each warp issues
// `per` REDs of 32 consecutive elements at pseudo-random 32-element-aligned rows of a
// buffer of `rows` rows (like the trace's ∂ℓ/∂H scatter into the chain-interleaved layout).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int T>
__global__ void k(void *buf, int rows, int per, float scale) {
  const int lane = threadIdx.x & 31;
  unsigned h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int i = 0; i < per; i++) {
    h = h * 1664525u + 1013904223u;
    const unsigned row = (h >> 8) % rows;
    const float x = scale * (float)(lane + i);
    if (T == 0) atomicAdd((float *)buf + row * 32 + lane, x);
    if (T == 1) atomicAdd((unsigned long long *)buf + row * 32 + lane, (unsigned long long)__float2ll_rn(x));
    if (T == 2) atomicAdd((int *)buf + row * 32 + lane, (int)(__float_as_int(x + 12582912.0f) - 0x4B400000));
    if (T == 3) atomicAdd((unsigned long long *)buf + row * 32 + lane, (unsigned long long)(long long)(__float_as_int(x + 12582912.0f) - 0x4B400000));
    if (T == 4) atomicAdd((double *)buf + row * 32 + lane, (double)x);
  }
}

int main() {
  void *buf;
  const int rows = 1 << 16;   // 64K rows x 32 x 8 B = 16 MB
  cudaMalloc(&buf, (size_t)rows * 32 * 8);
  cudaMemset(buf, 0, (size_t)rows * 32 * 8);
  const char *names[] = {"f32", "i64 F2I", "i32 magic", "i64 magic", "f64"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 8, threads = 256, per = 256;
  for (int t = 0; t < 5; t++) {
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(a);
      switch (t) {
        case 0: k<0><<<blocks, threads>>>(buf, rows, per, 0.001f); break;
        case 1: k<1><<<blocks, threads>>>(buf, rows, per, 0.001f); break;
        case 2: k<2><<<blocks, threads>>>(buf, rows, per, 0.001f); break;
        case 3: k<3><<<blocks, threads>>>(buf, rows, per, 0.001f); break;
        case 4: k<4><<<blocks, threads>>>(buf, rows, per, 0.001f); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double n = (double)blocks * threads / 32 * per;   // warp REDs
      if (rep == 2) printf("%-10s %8.3f ms  %.2f G warp-RED/s  %.2f G lane-ops/s\n", names[t], ms, n / ms / 1e6, 32 * n / ms / 1e6);
    }
  }
  return 0;
}
