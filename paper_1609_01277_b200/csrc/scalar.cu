// =============================================================================
// Scalar advection-diffusion of the paper's verification cases (
// SURVEY §8(f) N1), sm_100a fp64:
//   d phi/dt = -u_j d phi/dx_j + k d2 phi/dx_j^2 - S        (u_j, k constant)
// central differences of arbitrary even order, periodic in every direction,
// forward Euler or the low-storage RK3.  One thread per point,
// stencil taps through L1/L2 (a single field: the 1D wave and the 2D MMS of
// the paper are far from any roofline that matters; the NS path is the hot one).
// =============================================================================
#include "scalar.h"

namespace osbli {
namespace {

__device__ __forceinline__ int swrap(int i, int n) {
  if (i < 0) i += n;
  else if (i >= n) i -= n;
  if ((unsigned)i >= (unsigned)n) {
    i %= n;
    if (i < 0) i += n;
  }
  return i;
}

template <int M>
__global__ void __launch_bounds__(256) scalar_stage_kernel(const SParams p,
                                                           const double *__restrict__ phi,
                                                           double *__restrict__ out,
                                                           double *__restrict__ w,
                                                           const double *__restrict__ src,
                                                           double *__restrict__ rout,
                                                           unsigned int *__restrict__ flag) {
  const size_t n = (size_t)p.nx * p.ny * p.nz;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(t % p.nx), y = (int)((t / p.nx) % p.ny), z = (int)(t / ((size_t)p.nx * p.ny));
    const double c = phi[t];
    const size_t row = (size_t)z * p.ny * p.nx + (size_t)y * p.nx;
    double d1[3] = {0.0, 0.0, 0.0}, d2[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 1; k <= M; ++k) {
      const double xp = phi[row + swrap(x + k, p.nx)], xm = phi[row + swrap(x - k, p.nx)];
      const double yp = phi[(size_t)z * p.ny * p.nx + (size_t)swrap(y + k, p.ny) * p.nx + x];
      const double ym = phi[(size_t)z * p.ny * p.nx + (size_t)swrap(y - k, p.ny) * p.nx + x];
      const double zp = phi[((size_t)swrap(z + k, p.nz) * p.ny + y) * p.nx + x];
      const double zm = phi[((size_t)swrap(z - k, p.nz) * p.ny + y) * p.nx + x];
      d1[0] = fma(p.a[k - 1], xp - xm, d1[0]);
      d1[1] = fma(p.a[k - 1], yp - ym, d1[1]);
      d1[2] = fma(p.a[k - 1], zp - zm, d1[2]);
      // exactly zero on a constant field (D-22)
      d2[0] = fma(p.b[k], fma(-2.0, c, xp + xm), d2[0]);
      d2[1] = fma(p.b[k], fma(-2.0, c, yp + ym), d2[1]);
      d2[2] = fma(p.b[k], fma(-2.0, c, zp + zm), d2[2]);
    }
    double R = -(p.u[0] * d1[0] + p.u[1] * d1[1] + p.u[2] * d1[2]) +
               p.kd * (d2[0] + d2[1] + d2[2]);
    if (src) R -= src[t];
    if (rout) {
      rout[t] = R;
      continue;
    }
    double wn = p.dt * R;
    double base = c;
    if (p.two_reg) {
      if (p.read_w) base = w[t];
      if (p.write_w) w[t] = fma(p.beta, wn, base);
    } else {
      if (p.read_w) wn = fma(p.A, w[t], wn);
      if (p.write_w) w[t] = wn;
    }
    const double q = fma(p.B, wn, base);
    out[t] = q;
    if (!isfinite(q)) atomicOr(flag, 1u);
  }
}

template <int M>
cudaError_t scalar_launch(const SParams &p, const double *phi, double *out, double *w,
                          const double *src, double *rout, unsigned int *flag, cudaStream_t s) {
  const size_t n = (size_t)p.nx * p.ny * p.nz;
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  scalar_stage_kernel<M><<<(int)blocks, 256, 0, s>>>(p, phi, out, w, src, rout, flag);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_scalar_stage(const SParams &p, const double *phi, double *out, double *w,
                                const double *src, double *rout, unsigned int *flag,
                                cudaStream_t s) {
  switch (p.m) {
    case 1: return scalar_launch<1>(p, phi, out, w, src, rout, flag, s);
    case 2: return scalar_launch<2>(p, phi, out, w, src, rout, flag, s);
    case 3: return scalar_launch<3>(p, phi, out, w, src, rout, flag, s);
    case 4: return scalar_launch<4>(p, phi, out, w, src, rout, flag, s);
    case 5: return scalar_launch<5>(p, phi, out, w, src, rout, flag, s);
    case 6: return scalar_launch<6>(p, phi, out, w, src, rout, flag, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace osbli
