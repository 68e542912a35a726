// Per-order entry points of the kernel translation units (kernels_order.cu, one
// object per stencil half width M = 1..6) called by kernels.cu's run-time
// dispatch.  Internal interface, not part of the public ABI.
#pragma once
#include <cuda_runtime.h>

#include "kernels.h"

namespace osbli {

constexpr int DG_TY = 8;  // diagnostics tile rows (tile 32 x DG_TY)
constexpr int DG_Z = 16;  // diagnostics planes per CTA

namespace detail {
template <int M>
cudaError_t zpass_m(const KParams &p, const double *q, double *w, double *gz, int zb, int ze,
                    int zb1, int ze1, cudaStream_t s);
template <int M>
cudaError_t xypass_m(const KParams &p, const double *q, double *qout, double *w, const double *gz,
                     double *rout, unsigned int *flag, int zb, int ze, int zb1, int ze1,
                     cudaStream_t s);
template <int M>
cudaError_t divh_m(const KParams &p, double *q_out, double *w, double *r_out, unsigned int *flag,
                   int zb, int ze, cudaStream_t s);
template <int M>
cudaError_t diag_m(const KParams &p, const double *q, double *tpart, cudaStream_t s);
}  // namespace detail

}  // namespace osbli
