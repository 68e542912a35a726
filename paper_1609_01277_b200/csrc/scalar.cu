// =============================================================================
// Scalar advection-diffusion of the paper's verification cases (
// SURVEY §8(f) N1), sm_100a fp64:
//   d phi/dt = -u_j d phi/dx_j + k d2 phi/dx_j^2 - S        (u_j, k constant)
// central differences of arbitrary even order, periodic in every direction,
// forward Euler or the low-storage RK3.  A CTA covers a 32 x 8
// tile of the plane and SC_DZ consecutive planes: per plane the tile plus an
// m-wide halo is staged in shared memory (the next plane's values are loaded
// into registers while the current one is computed) for the x and y taps, and
// each thread keeps a register window of its column along z.
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

#ifndef OSBLI_SC_DZ
#define OSBLI_SC_DZ 4
#endif
#ifndef OSBLI_SC_MINB
#define OSBLI_SC_MINB 4
#endif
constexpr int SC_TX = 32, SC_TY = 8, SC_DZ = OSBLI_SC_DZ;

template <int M>
struct SGeom {
  static constexpr int HX = SC_TX + 2 * M, HY = SC_TY + 2 * M;
  static constexpr int N = HX * HY;                   // staged values per plane
  static constexpr int PER = (N + 255) / 256;         // per thread
};

template <int M>
__device__ __forceinline__ void scalar_fetch(const SParams &p, const double *__restrict__ phi,
                                             int z, int x0, int y0, int tid,
                                             double (&v)[SGeom<M>::PER]) {
  using G = SGeom<M>;
  const double *pp = phi + (size_t)z * p.ny * p.nx;
#pragma unroll
  for (int r = 0; r < G::PER; ++r) {
    const int idx = tid + 256 * r;
    v[r] = 0.0;
    if (idx < G::N) {
      const int hy = idx / G::HX, hx = idx - hy * G::HX;
      v[r] = __ldg(pp + (size_t)swrap(y0 - M + hy, p.ny) * p.nx + swrap(x0 - M + hx, p.nx));
    }
  }
}

template <int M>
__global__ void __launch_bounds__(256, OSBLI_SC_MINB) scalar_stage_kernel(const SParams p,
                                                              const double *__restrict__ phi,
                                                              double *__restrict__ out,
                                                              double *__restrict__ w,
                                                              const double *__restrict__ src,
                                                              double *__restrict__ rout,
                                                              unsigned int *__restrict__ flag) {
  using G = SGeom<M>;
  __shared__ double sh[G::N];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * SC_TX + tx;
  const int x0 = blockIdx.x * SC_TX, y0 = blockIdx.y * SC_TY;
  const int x = x0 + tx, y = y0 + ty;
  const bool valid = x < p.nx && y < p.ny;
  const int z0 = blockIdx.z * SC_DZ;
  const int nzo = min(SC_DZ, p.nz - z0);
  const size_t FS = (size_t)p.nx * p.ny;
  const size_t off = (size_t)min(y, p.ny - 1) * p.nx + min(x, p.nx - 1);
  // this column along z: planes z0 - m .. z0 + nzo - 1 + m
  double zw[SC_DZ + 2 * M];
#pragma unroll
  for (int t = 0; t < SC_DZ + 2 * M; ++t)
    zw[t] = t < nzo + 2 * M ? __ldg(phi + (size_t)swrap(z0 - M + t, p.nz) * FS + off) : 0.0;
  double nxt[G::PER];
  scalar_fetch<M>(p, phi, z0, x0, y0, tid, nxt);
  bool bad = false;
#pragma unroll
  for (int j = 0; j < SC_DZ; ++j) {
    if (j >= nzo) break;
    __syncthreads();  // the previous plane's reads are done
#pragma unroll
    for (int r = 0; r < G::PER; ++r) {
      const int idx = tid + 256 * r;
      if (idx < G::N) sh[idx] = nxt[r];
    }
    __syncthreads();
    if (j + 1 < nzo) scalar_fetch<M>(p, phi, z0 + j + 1, x0, y0, tid, nxt);
    const double *cc = sh + (ty + M) * G::HX + tx + M;
    const double c = zw[j + M];
    double d1[3] = {0.0, 0.0, 0.0}, d2[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 1; k <= M; ++k) {
      const double xp = cc[k], xm = cc[-k];
      const double yp = cc[k * G::HX], ym = cc[-k * G::HX];
      const double zp = zw[j + M + k], zm = zw[j + M - k];
      d1[0] = fma(p.a[k - 1], xp - xm, d1[0]);
      d1[1] = fma(p.a[k - 1], yp - ym, d1[1]);
      d1[2] = fma(p.a[k - 1], zp - zm, d1[2]);
      // exactly zero on a constant field (D-22)
      d2[0] = fma(p.b[k], fma(-2.0, c, xp + xm), d2[0]);
      d2[1] = fma(p.b[k], fma(-2.0, c, yp + ym), d2[1]);
      d2[2] = fma(p.b[k], fma(-2.0, c, zp + zm), d2[2]);
    }
    if (!valid) continue;
    const size_t t = (size_t)(z0 + j) * FS + off;
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
    bad |= !isfinite(q);
  }
  if (bad) atomicOr(flag, 1u);
}

template <int M>
cudaError_t scalar_launch(const SParams &p, const double *phi, double *out, double *w,
                          const double *src, double *rout, unsigned int *flag, cudaStream_t s) {
  const dim3 grid((p.nx + SC_TX - 1) / SC_TX, (p.ny + SC_TY - 1) / SC_TY,
                  (p.nz + SC_DZ - 1) / SC_DZ);
  scalar_stage_kernel<M><<<grid, dim3(SC_TX, SC_TY), 0, s>>>(p, phi, out, w, src, rout, flag);
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
