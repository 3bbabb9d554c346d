// Throughput of the legacy warp-level tensor-core MMAs on sm_100a (mma.sync
// tf32 / bf16 / f64) — is a 3xTF32 complex64 path worth it vs FP64 DMMA?
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void tf32_loop(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = b0 + 7;
  float c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = (float)i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};\n"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678f) out[0] = s;
}

template <int ILP>
__global__ void bf16_loop(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = b0 + 7;
  float c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = (float)i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};\n"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678f) out[0] = s;
}

template <typename F>
float time_it(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  float* d; cudaMalloc(&d, 64);
  const int iters = 20000;
  for (int warps : {8, 16, 32}) {
    int blocks = sms * 2, threads = 32 * warps;
    float ms = time_it([&] { tf32_loop<4><<<blocks, threads>>>(d, iters); });
    double fl = 2.0 * 16 * 8 * 8 * 4 * (double)iters * warps * blocks;
    printf("{\"op\": \"mma.sync tf32 m16n8k8\", \"warps_per_cta\": %d, \"tflops\": %.1f}\n", warps, fl / ms / 1e9);
    ms = time_it([&] { bf16_loop<4><<<blocks, threads>>>(d, iters); });
    fl = 2.0 * 16 * 8 * 16 * 4 * (double)iters * warps * blocks;
    printf("{\"op\": \"mma.sync bf16 m16n8k16\", \"warps_per_cta\": %d, \"tflops\": %.1f}\n", warps, fl / ms / 1e9);
  }
  return 0;
}
