// FP64 tensor-core (DMMA, mma.sync .f64) throughput on sm_100a, alone and
// issued next to FP64 vector FMAs: does the stencil path have a second FP64
// pipe to use?  One CTA per SM (big dynamic smem forces it), W warps, every
// thread runs C independent accumulator chains of length `iters`.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double (&d)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma1688(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
      "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// SHAPE 0: m8n8k4, 1: m16n8k4, 2: m16n8k8, 3: m16n8k16; C accumulators; F: DFMA chains
// interleaved per mma (0 = tensor only)
template <int SHAPE, int C, int F>
__global__ void dmma(double *out, int iters, double x) {
  double acc[C][4];
  double a[8], b[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = x * (threadIdx.x + k);
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = x * (k + 1);
#pragma unroll
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[c][k] = 0.0;
  double f[F > 0 ? F : 1];
#pragma unroll
  for (int k = 0; k < (F > 0 ? F : 1); ++k) f[k] = x * k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (SHAPE == 0) {
        double d[2] = {acc[c][0], acc[c][1]};
        mma884(d, a[c & 7], b[c & 3]);
        acc[c][0] = d[0];
        acc[c][1] = d[1];
      } else if (SHAPE == 1) {
        mma1684(acc[c], a[c & 7], a[(c + 1) & 7], b[c & 3]);
      } else if (SHAPE == 2) {
        const double aa[4] = {a[0], a[1], a[2], a[3]};
        const double bb[2] = {b[0], b[1]};
        mma1688(acc[c], aa, bb);
      } else {
        mma16816(acc[c], a, b);
      }
    }
#pragma unroll
    for (int k = 0; k < F; ++k) f[k] = fma(f[k], x, 1e-9);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
#pragma unroll
  for (int k = 0; k < (F > 0 ? F : 1); ++k) s += f[k];
  if (s == 12345.678) out[0] = s;
}

template <int F>
__global__ void dfma_only(double *out, int iters, double x) {
  double f[F];
#pragma unroll
  for (int k = 0; k < F; ++k) f[k] = x * k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < F; ++k) f[k] = fma(f[k], x, 1e-9);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < F; ++k) s += f[k];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
float time_ms(K kern, int warps, int iters, double *out, int sms) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  kern<<<sms, 32 * warps, 200 * 1024>>>(out, 8, 0.999999);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    kern<<<sms, 32 * warps, 200 * 1024>>>(out, iters, 0.999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    printf("\"error\": \"%s\",", cudaGetErrorString(e));
    return -1.f;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, sizeof(double));
  const int iters = 1 << 14;
  const double fl884 = 2.0 * 8 * 8 * 4, fl1684 = 2.0 * 16 * 8 * 4, fl1688 = 2.0 * 16 * 8 * 8,
               fl16816 = 2.0 * 16 * 8 * 16;
  printf("{\"sms\": %d, \"unit\": \"TFLOP/s (mma: 2 M N K per warp instruction; dfma: 2 per thread)\",\n", sms);
  const int W[] = {4, 8, 16};
  for (int wi = 0; wi < 3; ++wi) {
    const int w = W[wi];
    const double n = (double)iters * w * sms;  // warp-iterations
    float t;
    printf(" \"w%d\": {", w);
    t = time_ms(dmma<0, 4, 0>, w, iters, out, sms);
    printf("\"m8n8k4_c4\": %.2f, ", n * 4 * fl884 / (t * 1e-3) / 1e12);
    t = time_ms(dmma<0, 8, 0>, w, iters, out, sms);
    printf("\"m8n8k4_c8\": %.2f, ", n * 8 * fl884 / (t * 1e-3) / 1e12);
    t = time_ms(dmma<1, 4, 0>, w, iters, out, sms);
    printf("\"m16n8k4_c4\": %.2f, ", n * 4 * fl1684 / (t * 1e-3) / 1e12);
    t = time_ms(dmma<2, 4, 0>, w, iters, out, sms);
    printf("\"m16n8k8_c4\": %.2f, ", n * 4 * fl1688 / (t * 1e-3) / 1e12);
    t = time_ms(dmma<3, 4, 0>, w, iters, out, sms);
    printf("\"m16n8k16_c4\": %.2f, ", n * 4 * fl16816 / (t * 1e-3) / 1e12);
    t = time_ms(dfma_only<8>, w, iters, out, sms);
    printf("\"dfma_c8\": %.2f, ", n * 32 * 8 * 2 / (t * 1e-3) / 1e12);
    // mixed: 4 m16n8k8 + 8 DFMA chains per iteration; compare the time with each alone
    const float tm = time_ms(dmma<2, 4, 0>, w, iters, out, sms);
    const float tf = time_ms(dfma_only<8>, w, iters, out, sms);
    const float tb = time_ms(dmma<2, 4, 8>, w, iters, out, sms);
    printf("\"mixed_ms\": {\"mma_only\": %.3f, \"dfma_only\": %.3f, \"both\": %.3f}}%s\n", tm, tf, tb,
           wi < 2 ? "," : "");
  }
  printf("}\n");
  return 0;
}
