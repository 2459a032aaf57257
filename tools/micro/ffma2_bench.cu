// Microbenchmark: FP32 FMA throughput per SM with scalar FFMA vs packed FFMA2 (fma.rn.f32x2), sm_100a.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_bench ffma2_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int PACKED>
__global__ void __launch_bounds__(256) k(float* out, float a, float b, int iters) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 0.001f + i;
  if (PACKED) {
    uint64_t p[8], aa, bb;
    float2 t = make_float2(a, a), u = make_float2(b, b);
    aa = *reinterpret_cast<uint64_t*>(&t);
    bb = *reinterpret_cast<uint64_t*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float2 v = make_float2(acc[2 * i], acc[2 * i + 1]);
      p[i] = *reinterpret_cast<uint64_t*>(&v);
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(p[i]) : "l"(aa), "l"(bb));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float2 v = *reinterpret_cast<float2*>(&p[i]);
      acc[2 * i] = v.x;
      acc[2 * i + 1] = v.y;
    }
  } else {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(a, acc[i], b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  const int iters = 20000;
  for (int packed = 0; packed < 2; ++packed) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(s);
      if (packed) k<1><<<148 * 8, 256>>>(out, 0.999f, 0.001f, iters);
      else k<0><<<148 * 8, 256>>>(out, 0.999f, 0.001f, iters);
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      float ms;
      cudaEventElapsedTime(&ms, s, e);
      double fma = 148.0 * 8 * 256 * 16 * iters;
      if (rep) printf("%s: %.3f ms, %.1f TFMA/s = %.1f TFLOP/s\n", packed ? "FFMA2" : "FFMA ", ms, fma / ms / 1e9, 2 * fma / ms / 1e9);
    }
  }
  return 0;
}
