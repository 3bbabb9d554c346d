// FP64 pipe microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64)
// throughput, used as the roofline denominator for the propagator kernels.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

// m8n8k4: A 1 double, B 1 double, C 2 doubles per thread
template <int ILP>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// m16n8k4: A 2, B 1, C 4
template <int ILP>
__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

// m16n8k8: A 4, B 2, C 4
template <int ILP>
__global__ void dmma_m16n8k8(double* out, int iters) {
  double a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  b[0] = 1.0; b[1] = 0.5;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

// m16n8k16: A 8, B 4, C 4
template <int ILP>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

// FP32 FFMA peak (complex64 path)
template <int ILP>
__global__ void ffma_loop(float* out, int iters, float a, float b) {
  float acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-6f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678f) out[0] = s;
}

template <typename F>
float time_it(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d}\n", p.name, sms, clk_khz);
  double* d; float* f;
  CK(cudaMalloc(&d, 64)); CK(cudaMalloc(&f, 64));
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    int threads = 32 * warps, blocks = sms * 2;
    float ms = time_it([&] { dfma_loop<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9); });
    double fl = 2.0 * 8 * iters * (double)threads * blocks;
    printf("{\"op\": \"dfma\", \"warps_per_cta\": %d, \"ctas\": %d, \"tflops\": %.3f}\n", warps, blocks, fl / ms / 1e9);
    ms = time_it([&] { dmma_m8n8k4<4><<<blocks, threads>>>(d, iters / 4); });
    fl = 2.0 * 8 * 8 * 4 * 4 * (iters / 4) * (double)warps * blocks;
    printf("{\"op\": \"dmma_m8n8k4\", \"warps_per_cta\": %d, \"tflops\": %.3f}\n", warps, fl / ms / 1e9);
    ms = time_it([&] { dmma_m16n8k4<4><<<blocks, threads>>>(d, iters / 8); });
    fl = 2.0 * 16 * 8 * 4 * 4 * (iters / 8) * (double)warps * blocks;
    printf("{\"op\": \"dmma_m16n8k4\", \"warps_per_cta\": %d, \"tflops\": %.3f}\n", warps, fl / ms / 1e9);
    ms = time_it([&] { dmma_m16n8k8<4><<<blocks, threads>>>(d, iters / 16); });
    fl = 2.0 * 16 * 8 * 8 * 4 * (iters / 16) * (double)warps * blocks;
    printf("{\"op\": \"dmma_m16n8k8\", \"warps_per_cta\": %d, \"tflops\": %.3f}\n", warps, fl / ms / 1e9);
    ms = time_it([&] { dmma_m16n8k16<4><<<blocks, threads>>>(d, iters / 32); });
    fl = 2.0 * 16 * 8 * 16 * 4 * (iters / 32) * (double)warps * blocks;
    printf("{\"op\": \"dmma_m16n8k16\", \"warps_per_cta\": %d, \"tflops\": %.3f}\n", warps, fl / ms / 1e9);
    ms = time_it([&] { ffma_loop<8><<<blocks, threads>>>(f, iters * 2, 1.0000001f, 1e-9f); });
    fl = 2.0 * 8 * iters * 2 * (double)threads * blocks;
    printf("{\"op\": \"ffma\", \"warps_per_cta\": %d, \"tflops\": %.3f}\n", warps, fl / ms / 1e9);
  }
  // long sustained DMMA run (~2 s) to see the clock under FP64 load
  {
    int threads = 256, blocks = sms * 2;
    float ms = time_it([&] { dmma_m16n8k8<4><<<blocks, threads>>>(d, 400000); });
    double fl = 2.0 * 16 * 8 * 8 * 4 * 400000.0 * 8 * blocks;
    printf("{\"op\": \"dmma_m16n8k8_sustained\", \"ms\": %.1f, \"tflops\": %.3f}\n", ms, fl / ms / 1e9);
    ms = time_it([&] { dfma_loop<8><<<blocks, threads>>>(d, 800000, 1.0000001, 1e-9); });
    fl = 2.0 * 8 * 800000.0 * threads * blocks;
    printf("{\"op\": \"dfma_sustained\", \"ms\": %.1f, \"tflops\": %.3f}\n", ms, fl / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
