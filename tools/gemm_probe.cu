// Microbenchmark of the DMMA inner loops in isolation (no slice work):
//  (1) latency/ILP: m16n8k4 chains per warp x warps per SM
//  (2) tile_mma<PS32> / <PS16> (the lane_ps_kernel GEMM) repeated on fixed smem
//      operands, 1-3 CTAs per SM: the ceiling of the GEMM phases.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//      -I paper_2108_07126_b200/csrc tools/gemm_probe.cu -o tools/gemm_probe
#include <cstdio>
#include "kernels_ps3g.cuh"

using namespace sp;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void chain(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) dmma_16x8x4(c[i][0], c[i][1], c[i][2], c[i][3], a0, a1, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1) gemm_loop(double* out, int reps) {
  extern __shared__ __align__(16) double smem[];
  constexpr int NE = C::MT * C::NT * 4;
  for (int i = threadIdx.x; i < (int)(C::SMEM / 8); i += blockDim.x) smem[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const int wil = warp % C::WPL, lic = warp / C::WPL;
  const int ms0 = (wil % (C::S / C::MT)) * C::MT, nt0 = (wil / (C::S / C::MT)) * C::NT;
  const int lbase = lic * C::LANE_DBL;
  double accR[NE], accI[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) { accR[e] = 0; accI[e] = 0; }
  for (int r = 0; r < reps; ++r) {
    tile_mma<C, false>(nullptr, lbase + 2 * C::BDBL, lbase + (r & 1) * C::BDBL, accR, accI, ms0, nt0, ln);
    lane_sync<C>();
  }
  double s = 0;
#pragma unroll
  for (int e = 0; e < NE; ++e) s += accR[e] + accI[e];
  if (s == 12345.678) out[0] = s;
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

template <class C>
int run_gemm(const char* name, double* d, int sms) {
  CK(cudaFuncSetAttribute(gemm_loop<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  for (int per_sm : {1, 2, 3}) {
    if (per_sm * (C::SMEM + 1024) > 233472) continue;
    const int reps = 2000, ctas = sms * per_sm;
    float ms = time_it([&] { gemm_loop<C><<<ctas, C::THREADS, C::SMEM>>>(d, reps); });
    // one complex GEMM of D x WC (per lane) x D, 4 real products
    double fl = 8.0 * C::D * C::WC * C::D * reps * (double)C::LPC * ctas;
    printf("{\"op\": \"tile_mma_%s\", \"ctas_per_sm\": %d, \"tflops\": %.3f}\n", name, per_sm, fl / ms / 1e9);
  }
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  double* d; CK(cudaMalloc(&d, 64));
  const int iters = 4000;
  for (int warps_per_sm : {4, 8, 16}) {
    int blocks = sms, threads = 32 * warps_per_sm;
#define CH(I) { float ms = time_it([&] { chain<I><<<blocks, threads>>>(d, iters); }); \
      double fl = 2.0 * 16 * 8 * 4 * I * (double)iters * warps_per_sm * blocks; \
      printf("{\"op\": \"chain\", \"ilp\": %d, \"warps_per_sm\": %d, \"tflops\": %.3f, \"ns_per_mma_per_warp\": %.2f}\n", I, warps_per_sm, fl / ms / 1e9, ms * 1e6 / (iters * (double)I)); }
    CH(1) CH(2) CH(4) CH(8)
  }
  run_gemm<PSCfg<32, 32, 1, 2, 4, 1, 1, true>>("ps32", d, sms);
  run_gemm<PSCfg<16, 16, 1, 2, 1, 4, 1, true>>("ps16", d, sms);
  CK(cudaGetLastError());
  return 0;
}
