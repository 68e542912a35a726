// =============================================================================
// Scalar advection-diffusion of the paper's verification cases (
// SURVEY §8(f) N1), sm_100a fp64:
//   d phi/dt = -u_j d phi/dx_j + k d2 phi/dx_j^2 - S        (u_j, k constant)
// central differences of arbitrary even order, periodic in every direction,
// forward Euler or the low-storage RK3.
//
// A CTA owns a 32 x 16 tile of the plane and marches through SC_ZS consecutive
// planes (one output per thread and plane).  The x and y taps come from the
// current plane (tile plus an m-wide halo) in shared memory, double-buffered:
// the next plane is copied in by cp.async while the current one is computed, so
// one barrier per plane suffices.  The z taps come from a register window of the
// thread's column (planes z - m .. z + m): the plane loop is fully unrolled, so
// the window slides by renaming, one new load per plane, issued SC_ZA planes
// ahead.  Each wrapped halo offset is computed once per CTA.
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

#ifndef OSBLI_SC_ZS
#define OSBLI_SC_ZS 16
#endif
constexpr int SC_TX = 32, SC_TY = 16, SC_ZS = OSBLI_SC_ZS, SC_THREADS = SC_TX * SC_TY;

template <int M>
struct SGeom {
  static constexpr int HX = SC_TX + 2 * M, HY = SC_TY + 2 * M;
  static constexpr int N = HX * HY;                                // staged values per plane
  static constexpr int PER = (N + SC_THREADS - 1) / SC_THREADS;  // per thread
};

__device__ __forceinline__ void sc_cp_async8(double *smem, const double *gmem) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(gmem) : "memory");
}

template <int M>
__global__ void __launch_bounds__(SC_THREADS, 2) scalar_stage_kernel(const SParams p,
                                                              const double *__restrict__ phi,
                                                              double *__restrict__ out,
                                                              double *__restrict__ w,
                                                              const double *__restrict__ src,
                                                              double *__restrict__ rout,
                                                              unsigned int *__restrict__ flag) {
  using G = SGeom<M>;
  constexpr int ZW = SC_ZS + 2 * M;  // z-window values of one column over the march
  __shared__ double sh[2][G::N];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * SC_TX + tx;
  const int x0 = blockIdx.x * SC_TX, y0 = blockIdx.y * SC_TY;
  const int x = x0 + tx, y = y0 + ty;
  const bool valid = x < p.nx && y < p.ny;
  const int z0 = blockIdx.z * SC_ZS;
  const int nzo = min(SC_ZS, p.nz - z0);
  const size_t FS = (size_t)p.nx * p.ny;
  const size_t off = (size_t)min(y, p.ny - 1) * p.nx + min(x, p.nx - 1);
  // wrapped in-plane offsets of the halo values this thread stages (plane independent)
  int hoff[G::PER];
#pragma unroll
  for (int r = 0; r < G::PER; ++r) {
    const int idx = tid + SC_THREADS * r;
    const int hy = idx / G::HX, hx = idx - hy * G::HX;
    hoff[r] = idx < G::N ? swrap(y0 - M + hy, p.ny) * p.nx + swrap(x0 - M + hx, p.nx) : 0;
  }
  auto stage = [&](int zl, int b) {  // plane z0 + zl -> buffer b
    const double *pp = phi + (size_t)swrap(z0 + zl, p.nz) * FS;
#pragma unroll
    for (int r = 0; r < G::PER; ++r) {
      const int idx = tid + SC_THREADS * r;
      if (idx < G::N) sc_cp_async8(&sh[b][idx], pp + hoff[r]);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // this column along z: zw[t] = phi(z0 - m + t)
  double zw[ZW];
  auto zload = [&](int t) {
    zw[t] = t < nzo + 2 * M ? __ldg(phi + (size_t)swrap(z0 - M + t, p.nz) * FS + off) : 0.0;
  };
  constexpr int ZA = 2 * M + 2;  // window values in flight ahead of the plane being computed
#pragma unroll
  for (int t = 0; t < (ZA < ZW ? ZA : ZW); ++t) zload(t);
  stage(0, 0);
  // the low-storage register of the next plane's point, loaded a plane ahead
  const bool rw = p.read_w && !rout && valid;
  auto wload = [&](int j) { return rw && j < nzo ? w[(size_t)(z0 + j) * FS + off] : 0.0; };
  double wnext = wload(0);
  bool bad = false;
#pragma unroll
  for (int j = 0; j < SC_ZS; ++j) {
    if (j < nzo) {
      if (j + ZA < ZW) zload(j + ZA);
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();  // plane j staged; every thread is done with plane j - 1's buffer
      if (j + 1 < nzo) stage(j + 1, (j + 1) & 1);
      const double wcur = wnext;
      wnext = wload(j + 1);
      const double *cc = &sh[j & 1][(ty + M) * G::HX + tx + M];
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
      if (valid) {
        const size_t t = (size_t)(z0 + j) * FS + off;
        double R = -(p.u[0] * d1[0] + p.u[1] * d1[1] + p.u[2] * d1[2]) +
                   p.kd * (d2[0] + d2[1] + d2[2]);
        if (src) R -= src[t];
        if (rout) {
          rout[t] = R;
        } else {
          double wn = p.dt * R;
          double base = c;
          if (p.two_reg) {
            if (p.read_w) base = wcur;
            if (p.write_w) w[t] = fma(p.beta, wn, base);
          } else {
            if (p.read_w) wn = fma(p.A, wcur, wn);
            if (p.write_w) w[t] = wn;
          }
          const double q = fma(p.B, wn, base);
          out[t] = q;
          bad |= !isfinite(q);
        }
      }
    }
  }
  if (bad) atomicOr(flag, 1u);
}

template <int M>
cudaError_t scalar_launch(const SParams &p, const double *phi, double *out, double *w,
                          const double *src, double *rout, unsigned int *flag, cudaStream_t s) {
  const dim3 grid((p.nx + SC_TX - 1) / SC_TX, (p.ny + SC_TY - 1) / SC_TY,
                  (p.nz + SC_ZS - 1) / SC_ZS);
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
