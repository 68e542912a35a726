// FP64 latency / throughput vs warps per SM and independent chains per thread
// (how much ILP a stencil kernel with few resident warps needs on sm_100a).
// Each CTA has W warps, one CTA per SM (148 CTAs, big dynamic smem to force it);
// every thread runs C independent DFMA chains (template) of length `iters`.
// Also: the DADD -> DFMA pattern of a stencil tap, s = fma(a, x - y, s).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_lat tools/fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chains(double *out, int iters, double a, double b) {
  double x[C];
#pragma unroll
  for (int k = 0; k < C; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < C; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < C; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

template <int C>
__global__ void taps(double *out, int iters, double a, double b) {
  double x[C], y[C], s[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    x[k] = threadIdx.x * 1e-9 + k;
    y[k] = k * 0.5;
    s[k] = 0.0;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < C; ++k) {
      s[k] = fma(a, x[k] - y[k], s[k]);
      x[k] += b;
    }
  }
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < C; ++k) t += s[k] + x[k];
  if (t == 12345.678) out[0] = t;
}

template <typename K>
double run(K kern, int warps, int c, int iters, double *out, int sms, double clk_hz,
           int per_iter) {
  const int threads = 32 * warps;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  kern<<<sms, threads, 200 * 1024>>>(out, 16, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    kern<<<sms, threads, 200 * 1024>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double instr = (double)per_iter * c * iters * threads * sms;  // thread-level FP64 instrs
  return instr / (best * 1e-3) / (sms * clk_hz);                   // per SM per clock
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double *out;
  cudaMalloc(&out, sizeof(double));
  const double hz = clk * 1e3;
  const int iters = 1 << 14;
  printf("{\"sms\": %d, \"clock_mhz\": %.0f, \"unit\": \"FP64 thread-instructions per SM per clock (peak 64)\",\n", sms, clk / 1e3);
  const int W[] = {4, 8, 12, 16, 32};
  printf(" \"dfma_chains\": {");
  for (int wi = 0; wi < 5; ++wi) {
    printf("%s\"w%d\": [%.1f, %.1f, %.1f, %.1f, %.1f]", wi ? ", " : "", W[wi],
           run(chains<1>, W[wi], 1, iters, out, sms, hz, 1), run(chains<2>, W[wi], 2, iters, out, sms, hz, 1),
           run(chains<4>, W[wi], 4, iters, out, sms, hz, 1), run(chains<8>, W[wi], 8, iters, out, sms, hz, 1),
           run(chains<16>, W[wi], 16, iters, out, sms, hz, 1));
  }
  printf("},\n \"chains_per_thread\": [1, 2, 4, 8, 16],\n \"dadd_dfma_taps\": {");
  for (int wi = 0; wi < 5; ++wi) {
    printf("%s\"w%d\": [%.1f, %.1f, %.1f, %.1f, %.1f]", wi ? ", " : "", W[wi],
           run(taps<1>, W[wi], 1, iters, out, sms, hz, 3), run(taps<2>, W[wi], 2, iters, out, sms, hz, 3),
           run(taps<4>, W[wi], 4, iters, out, sms, hz, 3), run(taps<8>, W[wi], 8, iters, out, sms, hz, 3),
           run(taps<16>, W[wi], 16, iters, out, sms, hz, 3));
  }
  printf("}}\n");
  return 0;
}
