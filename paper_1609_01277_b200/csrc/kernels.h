// Internal interface between the C-ABI runtime (api.cpp) and the sm_100a
// kernels (kernels.cu).  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace osbli {

constexpr int kMaxHalf = 6;  // m = order/2 <= 6 (orders 2..12)

// Everything a kernel needs, passed by value (lives in the constant bank).
struct KParams {
  int nx, ny, nz;  // local grid (nz = slab planes on this rank)
  int G;           // ghost planes allocated on each z side of Q buffers
  int zwrap;       // 1: single periodic domain in z (wrap modulo nz); 0: read ghost planes
  int m;           // stencil half width
  double a[kMaxHalf];      // first-derivative weights a_k / dx       (k = 1..m)
  double b[kMaxHalf + 1];  // second-derivative weights b_k / dx^2    (k = 0..m)
  double cb[kMaxHalf];     // C_l = sum_{k>l} b_k / dx^2 (l = 0..m-1): D2 in first differences
  double nu, kappa;        // 1/Re and 1/((gamma-1) M^2 Pr Re)  (mu = 1)
  double gm1;              // gamma - 1
  double gM2;              // gamma M^2
  // stage update: W <- A W + dt R ; Q' <- Q + B W
  double A, B, dt;
  int read_w, write_w;     // A != 0 ; W needed by a later stage
  const double *src;       // optional steady source S, [nz][5][ny][nx] (dQ/dt = R + S)
  int sym[3];              // 1: symmetry boundaries in direction d, 0: periodic
  // two-register RK3 (OSBLI_RK3_2R, D-25): the z-pass writes W' = dt Rz into the
  // interior planes of the destination Q buffer (its `w` argument); the xy-pass
  // reads W' there and keeps Q_old in its own `w` argument:
  //   Q' = base + B (W' + dt R_xy),  w <- base + beta (W' + dt R_xy)  (write_w)
  // with base = w (read_w) or Q.
  int two_reg;
  double beta;
  // equation variants (D-26, D-27)
  int visc;        // 1: Sutherland mu(T) = T^1.5 (1 + suth)/(T + suth); 0: mu = 1
  double suth;     // Sutherland constant over the reference temperature
  int cons;        // 1: viscous work in divergence form D_j H_j, H_j = u_i tau_ij
  double *dtz;     // variants: D_z T from the z-pass, [nz][ny][nx]
  double *hflux;   // cons: H_j from the xy-pass, [nz][3][ny][nx]
  // fused diagnostics of the stage's input state (osbli_step_diag): the xy-pass
  // writes per-(plane, tile) partials [nz][xy tiles][3] here when non-null
  double *dpart;
  // debug builds (-DOSBLI_DEBUG_CHECKS=1): bounds violations of the staged loads
  // set bit 2 of this flag (the handle's non-finite flag: the next synchronising
  // call then fails)
  unsigned int *dbg;
};

// Device buffers of one handle.  Q buffers: [nz + 2G][5][ny][nx] (plane-major,
// ghost planes at both z ends); W: [nz][5][ny][nx]; Gz: [nz][3][ny][nx].
struct Bufs {
  double *q[2];
  double *w;
  double *gz;
  unsigned int *flag;  // non-finite flag (device)
  double *diag_part;   // [nz][3] per-plane partial sums (device)
};

// Launch one stage: zpass(Q_in) -> W' = A W + dt Rz, Gz ; xypass -> W = W' + dt R_xy,
// Q_out = Q_in + B W (or, if r_out is non-null, r_out = W' + dt R_xy with the
// caller passing A = 0, dt = 1: the residual).  r_out is [nz][5][ny][nx].
cudaError_t launch_stage(const KParams &p, const double *q_in, double *q_out, double *w,
                         double *gz, double *r_out, unsigned int *flag, cudaStream_t s,
                         long long *launches);

// Conservative viscous work (p.cons): adds the divergence D_j H_j of the xy-pass's
// H to the energy of the finished stage (q_out, w) or of the residual (r_out).
cudaError_t launch_divh(const KParams &p, double *q_out, double *w, double *r_out,
                        unsigned int *flag, int z_begin, int z_end, cudaStream_t s,
                        long long *launches);

// Symmetry boundary in z on a slab handle: fill the m ghost planes of the
// low (side 0) or high (side 1) domain face with the mirrored interior planes,
// rho u_z negated.  q is a Q buffer [nz + 2G][5][ny][nx].
cudaError_t launch_mirror_ghosts(const KParams &p, double *q, int side, cudaStream_t s,
                                 long long *launches);
// The same for a ghosted buffer of nf fields per plane ([nz + 2G][nf][ny][nx],
// `base` = its first (ghost) plane) whose field `odd` changes sign.
cudaError_t launch_mirror_planes(const KParams &p, double *base, int nf, int odd, int side,
                                 cudaStream_t s, long long *launches);

// z-pass restricted to planes [z_begin, z_end) and, in the same launch, [z_begin1,
// z_end1) (the two slab faces of the boundary-first schedule).
cudaError_t launch_zpass(const KParams &p, const double *q_in, double *w, double *gz,
                         int z_begin, int z_end, cudaStream_t s, long long *launches,
                         int z_begin1 = 0, int z_end1 = 0);
// xy-pass restricted to planes [z_begin, z_end) and, in the same launch, [z_begin1, z_end1).
cudaError_t launch_xypass(const KParams &p, const double *q_in, double *q_out, double *w,
                          const double *gz, double *r_out, unsigned int *flag, int z_begin,
                          int z_end, cudaStream_t s, long long *launches, int z_begin1 = 0,
                          int z_end1 = 0);

// Number of xy-pass tiles of a plane (the fused diagnostics' partials per plane).
int xypass_tiles(const KParams &p);
// Per-plane partials [nz][3] = the (plane, tile) partials [nz][ntiles][3] summed in
// tile order.
cudaError_t launch_diag_planes(const double *tpart, int nz, int ntiles, double *part,
                               cudaStream_t s, long long *launches);

// Per-plane diagnostics partial sums [nz][3] (E_k, enstrophy, dissipation sums).
// scratch: >= diagnostics_scratch(p) doubles (per-(plane, tile) partials).
size_t diagnostics_scratch(const KParams &p);
cudaError_t launch_diagnostics(const KParams &p, const double *q_in, double *scratch,
                               double *part, cudaStream_t s, long long *launches);

// Layout conversion between the ABI [5][nz][ny][nx] and the internal plane-major
// Q buffer (interior planes only).
cudaError_t launch_abi_to_internal(const KParams &p, const double *src, double *q, cudaStream_t s,
                                   long long *launches);
cudaError_t launch_internal_to_abi(const KParams &p, const double *q, double *dst, int nfields,
                                   int ghosted, cudaStream_t s, long long *launches);

// TMA tensor map of a device buffer viewed as a 4-D fp64 tensor (x: nx, y: ny,
// field: nf, plane: planes; x fastest) with a (bx, by, bf, 1) box (kernels.cu).
// Cached per (buffer, shape, box); false when TMA does not apply (odd nx) or the
// driver entry point is missing.
bool tensor_map(const double *ptr, int nx, int ny, int nf, int planes, int bx, int by, int bf,
                CUtensorMap *out);

}  // namespace osbli
