// Internal interface of the scalar advection-diffusion kernel (scalar.cu).
#pragma once
#include <cuda_runtime.h>

namespace osbli {

struct SParams {
  int nx, ny, nz, m;
  double a[6];   // a_k / dx
  double b[7];   // b_k / dx^2
  double u[3];   // advection velocity
  double kd;     // diffusivity
  double A, B, dt;
  int read_w, write_w;
  int two_reg;   // two-register RK3 (D-25): out <- base + B dt R, w <- base + beta dt R,
  double beta;   // base = w (read_w) or phi
};

// One stage: W <- A W + dt R(phi), out <- phi + B W; or rout <- R(phi) if rout != null.
// src (optional) is the steady source S of d phi/dt = ... - S.  Arrays [nz][ny][nx].
cudaError_t launch_scalar_stage(const SParams &p, const double *phi, double *out, double *w,
                                const double *src, double *rout, unsigned int *flag,
                                cudaStream_t s);

}  // namespace osbli
