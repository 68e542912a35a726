// =============================================================================
// C ABI of the scalar advection-diffusion solver (include/osbli.h, "scalar"
// section): the paper's verification equations.
// =============================================================================
#include <cuda_runtime.h>

#include <cmath>
#include <new>
#include <string>

#include "../../include/osbli.h"
#include "scalar.h"
#include "weights.h"

struct osbli_scalar {
  int nx = 0, ny = 0, nz = 0, order = 0, scheme = 0;
  double dt = 0;
  osbli::SParams base{};
  double *phi[2] = {nullptr, nullptr};
  double *w = nullptr;
  double *src = nullptr;
  unsigned int *flag = nullptr;
  int cur = 0;
  cudaStream_t stream = nullptr, own_stream = nullptr;
  bool poisoned = false;
  long long steps = 0;
  std::string err;
};

namespace {

thread_local std::string g_scalar_error;

int sfail(osbli_scalar *h, int code, const std::string &msg) {
  h->err = msg;
  if (code == OSBLI_E_CUDA || code == OSBLI_E_NONFINITE) h->poisoned = true;
  return code;
}

#define SCK(h, expr)                                                                \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) return sfail((h), OSBLI_E_CUDA, std::string(#expr) + ": " + \
                                        cudaGetErrorString(_e));                    \
  } while (0)

void sfree(osbli_scalar *h) {
  cudaFree(h->phi[0]);
  cudaFree(h->phi[1]);
  cudaFree(h->w);
  cudaFree(h->src);
  cudaFree(h->flag);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
}

size_t npts(const osbli_scalar *h) { return (size_t)h->nx * h->ny * h->nz; }

}  // namespace

extern "C" {

int osbli_scalar_create(int nx, int ny, int nz, int order, double dx, double dt, double u0,
                        double u1, double u2, double kappa, int scheme, osbli_scalar **out) {
  if (!out) return OSBLI_E_INVAL;
  *out = nullptr;
  if (nx < 1 || ny < 1 || nz < 1 || order < 2 || order % 2 || !(dx > 0) || !std::isfinite(dx) ||
      !(dt > 0) || !std::isfinite(dt) || !std::isfinite(u0) || !std::isfinite(u1) ||
      !std::isfinite(u2) || !(kappa >= 0) || !std::isfinite(kappa) ||
      (scheme != OSBLI_EULER && scheme != OSBLI_RK3 && scheme != OSBLI_RK3_2R)) {
    g_scalar_error = "invalid argument";
    return OSBLI_E_INVAL;
  }
  if (order > 12) {
    g_scalar_error = "orders above 12 are not built";
    return OSBLI_E_UNSUPPORTED;
  }
  osbli_scalar *h = new (std::nothrow) osbli_scalar();
  if (!h) return OSBLI_E_NOMEM;
  h->nx = nx; h->ny = ny; h->nz = nz; h->order = order; h->scheme = scheme; h->dt = dt;
  osbli::SParams &p = h->base;
  p.nx = nx; p.ny = ny; p.nz = nz; p.m = order / 2;
  double a[6] = {0}, b[7] = {0};
  osbli::central_weights(p.m, a, b);
  for (int k = 0; k < p.m; ++k) p.a[k] = a[k] / dx;
  for (int k = 0; k <= p.m; ++k) p.b[k] = b[k] / (dx * dx);
  p.u[0] = u0; p.u[1] = u1; p.u[2] = u2; p.kd = kappa; p.dt = dt;
  const size_t n = npts(h);
  if (cudaMalloc((void **)&h->phi[0], n * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void **)&h->phi[1], n * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void **)&h->w, n * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void **)&h->flag, sizeof(unsigned int)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMemsetAsync(h->phi[0], 0, n * sizeof(double), h->own_stream) != cudaSuccess ||
      cudaMemsetAsync(h->flag, 0, sizeof(unsigned int), h->own_stream) != cudaSuccess ||
      cudaStreamSynchronize(h->own_stream) != cudaSuccess) {
    g_scalar_error = std::string("device setup failed: ") + cudaGetErrorString(cudaGetLastError());
    sfree(h);
    delete h;
    return OSBLI_E_NOMEM;
  }
  h->stream = h->own_stream;
  *out = h;
  return OSBLI_OK;
}

int osbli_scalar_set_stream(osbli_scalar *h, void *cuda_stream) {
  if (!h) return OSBLI_E_INVAL;
  if (h->poisoned) return OSBLI_E_STATE;
  SCK(h, cudaStreamSynchronize(h->stream));
  h->stream = cuda_stream ? (cudaStream_t)cuda_stream : h->own_stream;
  return OSBLI_OK;
}

int osbli_scalar_set_state(osbli_scalar *h, const double *phi, int on_device) {
  if (!h || !phi) return OSBLI_E_INVAL;
  if (h->poisoned) return OSBLI_E_STATE;
  SCK(h, cudaMemcpyAsync(h->phi[h->cur], phi, npts(h) * sizeof(double),
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
  SCK(h, cudaMemsetAsync(h->flag, 0, sizeof(unsigned int), h->stream));
  SCK(h, cudaStreamSynchronize(h->stream));
  h->steps = 0;
  return OSBLI_OK;
}

int osbli_scalar_set_source(osbli_scalar *h, const double *S, int on_device) {
  if (!h) return OSBLI_E_INVAL;
  if (h->poisoned) return OSBLI_E_STATE;
  if (!S) {
    SCK(h, cudaStreamSynchronize(h->stream));
    cudaFree(h->src);
    h->src = nullptr;
    return OSBLI_OK;
  }
  if (!h->src) SCK(h, cudaMalloc((void **)&h->src, npts(h) * sizeof(double)));
  SCK(h, cudaMemcpyAsync(h->src, S, npts(h) * sizeof(double),
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
  SCK(h, cudaStreamSynchronize(h->stream));
  return OSBLI_OK;
}

int osbli_scalar_get_state(osbli_scalar *h, double *phi, int on_device) {
  if (!h || !phi) return OSBLI_E_INVAL;
  SCK(h, cudaMemcpyAsync(phi, h->phi[h->cur], npts(h) * sizeof(double),
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
  SCK(h, cudaStreamSynchronize(h->stream));
  return OSBLI_OK;
}

int osbli_scalar_step(osbli_scalar *h, int n) {
  if (!h || n < 0) return OSBLI_E_INVAL;
  if (h->poisoned) return OSBLI_E_STATE;
  static const double RK_A[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};
  static const double RK_B[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
  static const double RK2R_ALPHA[3] = {2.0 / 3.0, 5.0 / 12.0, 3.0 / 5.0};
  static const double RK2R_BETA[3] = {1.0 / 4.0, 3.0 / 20.0, 3.0 / 5.0};
  const int ns = h->scheme == OSBLI_EULER ? 1 : 3;
  for (int it = 0; it < n; ++it) {
    for (int s = 0; s < ns; ++s) {
      osbli::SParams p = h->base;
      if (h->scheme == OSBLI_RK3) {
        p.A = RK_A[s]; p.B = RK_B[s]; p.read_w = s > 0; p.write_w = s < 2;
      } else if (h->scheme == OSBLI_RK3_2R) {
        p.A = 0.0; p.B = RK2R_ALPHA[s]; p.beta = RK2R_BETA[s]; p.two_reg = 1;
        p.read_w = s > 0; p.write_w = s < 2;
      } else {
        p.A = 0.0; p.B = 1.0; p.read_w = 0; p.write_w = 0;
      }
      SCK(h, osbli::launch_scalar_stage(p, h->phi[h->cur], h->phi[h->cur ^ 1], h->w, h->src,
                                        nullptr, h->flag, h->stream));
      h->cur ^= 1;
    }
    ++h->steps;
  }
  return OSBLI_OK;
}

int osbli_scalar_residual(osbli_scalar *h, double *R, int on_device) {
  if (!h || !R) return OSBLI_E_INVAL;
  if (h->poisoned) return OSBLI_E_STATE;
  SCK(h, osbli::launch_scalar_stage(h->base, h->phi[h->cur], nullptr, h->w, h->src, h->w, h->flag,
                                    h->stream));
  SCK(h, cudaMemcpyAsync(R, h->w, npts(h) * sizeof(double),
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
  SCK(h, cudaStreamSynchronize(h->stream));
  return OSBLI_OK;
}

int osbli_scalar_sync(osbli_scalar *h) {
  if (!h) return OSBLI_E_INVAL;
  if (h->poisoned) return OSBLI_E_STATE;
  unsigned int flag = 0;
  SCK(h, cudaMemcpyAsync(&flag, h->flag, sizeof(flag), cudaMemcpyDeviceToHost, h->stream));
  SCK(h, cudaStreamSynchronize(h->stream));
  if (flag) return sfail(h, OSBLI_E_NONFINITE, "a time step produced a non-finite value");
  return OSBLI_OK;
}

const char *osbli_scalar_last_error(const osbli_scalar *h) {
  return h ? h->err.c_str() : g_scalar_error.c_str();
}

void osbli_scalar_destroy(osbli_scalar *h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  sfree(h);
  delete h;
}

}  // extern "C"
