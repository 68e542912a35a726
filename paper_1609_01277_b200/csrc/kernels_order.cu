// =============================================================================
// sm_100a fp64 kernels of the OpenSBLI hot path (B200-native).
//
// One RK stage = two kernels:
//   zpass  : every term of the residual that differentiates along z
//            (D_z, D_zz; P:271-274 skew terms, P:274 Laplacians), written as a
//            partial residual Rz[5] plus the velocity gradients g_i2 = D_z u_i.
//            A CTA stages 32 x-columns x (TZ+2m) z-planes of the 13 z-stencil
//            operands in shared memory (computed once per staged point) and
//            each thread produces RZ = 4 consecutive z outputs from a register
//            window (reuse (RZ+2m)/RZ instead of 2m loads per output).
//   xypass : all x/y terms on a 32x16 plane tile with an m-wide halo in
//            shared memory (warp-specialised: a cp.async producer warpgroup and
//            two decoupled consumer groups, xypass_ws.cuh), the mixed
//            derivatives (commuted so that no z stencil is needed:
//            D_x D_z u_z = D_x g_22, D_z D_x u_x = D_x g_02, ...; D-7),
//            the viscous dissipation and heat flux, then the fused low-storage
//            RK stage update W <- W' + dt R_xy, Q' <- Q + B W and
//            a non-finite check.
//   variants: symmetry boundaries (mirror maps, N3), the
//            two-register RK3 (N2a), Sutherland mu(T) and the conservative
//            viscous work (+ divh_kernel; N2b, N4), each a separate
//            instantiation so that the default path stays as it is.
// All arithmetic is IEEE fp64; tensor cores are not used (a stencil is not a
// dense contraction).  Periodic wrap in x and y is done in-kernel; in
// z either in-kernel (one GPU) or through ghost planes (slab decomposition).
// =============================================================================
// This translation unit instantiates every order-dependent kernel for one
// stencil half width M = OSBLI_M (the Makefile compiles it once per M, in
// parallel); kernels.cu dispatches on the run-time order.
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "device_common.cuh"
#include "dispatch.h"

#ifndef OSBLI_M
#error "compile with -DOSBLI_M=<stencil half width 1..6>"
#endif

namespace osbli {
namespace {
#include "zpass.cuh"
#include "xypass_ws.cuh"

// ------------------------------------------------------------------ diagnostics
// Per-(plane, tile) partial sums of the integrands of the diagnostics (
// D-11, D-12): 1/2 rho u_j u_j, 1/2 rho |omega|^2 and tau_ij du_i/dx_j, with the
// velocity gradients g_ij = D_j u_i by the solver's first-derivative stencils.
// A CTA covers a 32 x 8 tile of the plane and marches through DG_Z consecutive
// planes: per plane rho, rho u_i on the tile rows with the x-halo (X part) and on
// the tile columns with the y-halo (Y part) are staged in shared memory by cp.async,
// double-buffered (the next plane's copies overlap the current one); once they
// land, each copier turns its own values into u_i = m_i * (1/rho) (as in the
// stepping kernels, D-28; mirrored components negated) before the plane's barrier.
// The z taps come from a per-thread register window of u_i along z, loaded two
// planes ahead.  The 256 point values of each plane are reduced in a fixed order
// (warp butterflies, then the 8 warps in order), so the partial of a (plane, tile)
// depends on nothing but its data: diag_tiles_kernel then sums the tiles of each
// plane in tile order, and the host sums the planes in global z order, which makes
// the numbers independent of the slab decomposition.
template <int M>
struct DGGeom {
  static constexpr int XW = 32 + 2 * M;                       // X-part row width
  static constexpr int NX = DG_TY * XW, NY = (DG_TY + 2 * M) * 32;
  static constexpr int N = NX + NY;                           // staged points per plane
  static constexpr int PER = (N + 255) / 256;                 // per thread
};

// u_i at a staged (x, y) of plane z (z window; the mirror signs are the caller's)
__device__ __forceinline__ void diag_u(const KParams &p, const double *__restrict__ q, int z,
                                       size_t off, double (&u)[3]) {
  const size_t FS = (size_t)p.nx * p.ny;
  const double *qp = q + qplane(p, z) + off;
  const double r = rcp_rho(__ldg(qp));
#pragma unroll
  for (int i = 0; i < 3; ++i) u[i] = __ldg(qp + (1 + i) * FS) * r;
}

template <int M>
__global__ void __launch_bounds__(256, 2) diag_kernel(const KParams p, const double *__restrict__ q,
                                                      double *__restrict__ tpart, int ntiles) {
  using G = DGGeom<M>;
  // [buffer][rho, m0, m1, m2 -> u0, u1, u2][staged point] (dynamic: above 48 KB)
  extern __shared__ double DSM[];
  double(*U)[4][G::N] = reinterpret_cast<double(*)[4][G::N]>(DSM);
  __shared__ double red[3][8];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * DG_TY;
  const int tile = blockIdx.y * gridDim.x + blockIdx.x;
  const int x = x0 + tx, y = y0 + ty;
  const bool valid = x < p.nx && y < p.ny;
  const int z0 = blockIdx.z * DG_Z;
  const int nzo = min(DG_Z, p.nz - z0);
  const size_t off = (size_t)min(y, p.ny - 1) * p.nx + min(x, p.nx - 1);
  const size_t FS = (size_t)p.nx * p.ny;
  // in-plane offsets of the points this thread stages, and their mirror parities
  int hoff[G::PER];
  unsigned char hflip[G::PER];
#pragma unroll
  for (int r = 0; r < G::PER; ++r) {
    const int idx = tid + 256 * r;
    hoff[r] = 0;
    hflip[r] = 0;
    if (idx < G::N) {
      int fx = 0, fy = 0, gx, gy;
      if (idx < G::NX) {  // X part: row rr of the tile, column c of the x-extended row
        const int rr = idx / G::XW, c = idx - rr * G::XW;
        gx = bmap(x0 - M + c, p.nx, p.sym[0], fx);
        gy = min(y0 + rr, p.ny - 1);
      } else {            // Y part: row c of the y-extended tile, column k & 31
        const int k = idx - G::NX, c = k >> 5;
        gx = min(x0 + (k & 31), p.nx - 1);
        gy = bmap(y0 - M + c, p.ny, p.sym[1], fy);
      }
      hoff[r] = gy * p.nx + gx;
      hflip[r] = (unsigned char)(fx | (fy << 1));
    }
  }
  auto stage = [&](int j, int b) {  // raw rho, m_i of plane z0 + j -> buffer b
    const double *qp = q + qplane(p, z0 + j);
#pragma unroll
    for (int r = 0; r < G::PER; ++r) {
      const int idx = tid + 256 * r;
      if (idx < G::N) {
#pragma unroll
        for (int f = 0; f < 4; ++f) cp_async8(&U[b][f][idx], qp + f * FS + hoff[r]);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // register window of u_i along z at this thread's (x, y): uz[i][t] = u_i(z0 - m + t)
  constexpr int UW = DG_Z + 2 * M, ZA = 2 * M + 2;
  double uz[3][UW];
  auto uzload = [&](int t) {
    double u[3] = {0.0, 0.0, 0.0};
    if (t < nzo + 2 * M) {
      int f;
      const int zz = zread(p, z0 - M + t, f);
      diag_u(p, q, zz, off, u);
      if (f) u[2] = -u[2];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) uz[i][t] = u[i];
  };
#pragma unroll
  for (int t = 0; t < (ZA < UW ? ZA : UW); ++t) uzload(t);
  stage(0, 0);
#pragma unroll
  for (int j = 0; j < DG_Z; ++j) {
    if (j >= nzo) break;
    const int z = z0 + j, b = j & 1;
    if (j + ZA < UW) uzload(j + ZA);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    // this thread's staged points: u_i = m_i / rho, mirrored components negated
#pragma unroll
    for (int r = 0; r < G::PER; ++r) {
      const int idx = tid + 256 * r;
      if (idx < G::N) {
        const double rr = rcp_rho(U[b][0][idx]);
        const double u0 = U[b][1][idx] * rr, u1 = U[b][2][idx] * rr, u2 = U[b][3][idx] * rr;
        U[b][1][idx] = (hflip[r] & 1) ? -u0 : u0;
        U[b][2][idx] = (hflip[r] & 2) ? -u1 : u1;
        U[b][3][idx] = u2;
      }
    }
    __syncthreads();  // plane j converted; every thread is done with plane j - 1's buffer
    if (j + 1 < nzo) stage(j + 1, b ^ 1);
    double g[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double *rx = &U[b][1 + i][ty * G::XW + tx + M];
      const double *cy = &U[b][1 + i][G::NX + (ty + M) * 32 + tx];
      double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
      for (int k = 1; k <= M; ++k) {
        sx = fma(p.a[k - 1], rx[k] - rx[-k], sx);
        sy = fma(p.a[k - 1], cy[32 * k] - cy[-32 * k], sy);
        sz = fma(p.a[k - 1], uz[i][j + M + k] - uz[i][j + M - k], sz);
      }
      g[i][0] = sx;
      g[i][1] = sy;
      g[i][2] = sz;
    }
    double v[3] = {0.0, 0.0, 0.0};
    if (valid) {
      const double *qp = q + qplane(p, z) + off;
      const double rho = __ldg(qp);
      const double u0 = uz[0][j + M], u1 = uz[1][j + M], u2 = uz[2][j + M];
      const double ke = u0 * u0 + u1 * u1 + u2 * u2;
      v[0] = 0.5 * rho * ke;
      const double w0 = g[2][1] - g[1][2], w1 = g[0][2] - g[2][0], w2 = g[1][0] - g[0][1];
      v[1] = 0.5 * rho * (w0 * w0 + w1 * w1 + w2 * w2);
      const double th = g[0][0] + g[1][1] + g[2][2];
      const double s01 = g[0][1] + g[1][0], s02 = g[0][2] + g[2][0], s12 = g[1][2] + g[2][1];
      double phi = p.nu * (2.0 * (g[0][0] * g[0][0] + g[1][1] * g[1][1] + g[2][2] * g[2][2]) +
                           s01 * s01 + s02 * s02 + s12 * s12 - (2.0 / 3.0) * th * th);
      if (p.visc) {  // tau carries mu(T) (D-26)
        const double pr = p.gm1 * (__ldg(qp + 4 * FS) - 0.5 * rho * ke);
        phi *= sutherland_mu(p, p.gM2 * pr * rcp_rho(rho));
      }
      v[2] = phi;
    }
    // fixed-order reduction of the plane's 256 values
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    if (tx == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) red[k][ty] = v[k];
    }
    __syncthreads();
    if (tid < 3) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[tid][w];
      tpart[((size_t)z * ntiles + tile) * 3 + tid] = t;
    }
  }
}

// ------------------------------------------------------------------ conservative viscous work
// D_j H_j (H_j = u_i tau_ij from the xy-pass; H_j odd under the mirror of
// direction j) added to the energy of the finished stage (D-27):
//   residual: R_E += D;  2N: W_E += dt D (write_w), Q'_E += B dt D;
//   two-register: Q'_E += alpha dt D, Q_old_E += beta dt D (write_w).
// A CTA covers a 32 x 16 tile of the plane and marches through DH_Z = 16 planes,
// one output per thread and plane.  Per plane H_x (tile rows + x halo) and H_y
// (tile columns + y halo) are staged in shared memory, double-buffered: the next
// plane's cp.async copies overlap the current one (one barrier per plane; the
// mirrored halo values of symmetric boundaries are negated by their own copier
// after landing).  H_z comes from a register window along z that slides by
// renaming (fully unrolled plane loop, loads issued two planes ahead); the
// read-modify-write operands are loaded a plane ahead.
constexpr int DH_Z = 16, DH_TY = 16, DH_THREADS = 32 * DH_TY;
template <int M>
struct DHGeom {
  static constexpr int XW = 32 + 2 * M;                           // H_x row width
  static constexpr int NX = DH_TY * XW, NY = (DH_TY + 2 * M) * 32;  // staged elements
  static constexpr int N = NX + NY;
  static constexpr int PER = (N + DH_THREADS - 1) / DH_THREADS;   // per thread
};
template <int M, bool SYM>
__global__ void __launch_bounds__(DH_THREADS, 2) divh_kernel(const KParams p,
                                                             const double *__restrict__ H,
                                                             double *__restrict__ qout,
                                                             double *__restrict__ w,
                                                             double *__restrict__ rout,
                                                             unsigned int *__restrict__ flag,
                                                             int zb, int ze) {
  using G = DHGeom<M>;
  __shared__ double sh[2][G::N];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * DH_TY;
  const int x = x0 + tx, y = y0 + ty;
  const bool valid = x < p.nx && y < p.ny;
  const int z0 = zb + blockIdx.z * DH_Z;
  const int nzo = min(DH_Z, ze - z0);
  const size_t FS = (size_t)p.nx * p.ny;
  const size_t off = (size_t)min(y, p.ny - 1) * p.nx + min(x, p.nx - 1);
  // in-plane offsets (component included) of the values this thread stages, and
  // whether they come through an odd number of mirrors (H_j is odd in j)
  int hoff[G::PER];
  bool hneg[G::PER];
#pragma unroll
  for (int r = 0; r < G::PER; ++r) {
    const int idx = tid + DH_THREADS * r;
    hoff[r] = 0;
    hneg[r] = false;
    if (idx < G::NX) {  // H_x: row c of the tile, column cc of the x-extended row
      const int c = idx / G::XW, cc = idx - c * G::XW;
      int f;
      const int gx = bmap_t<SYM>(x0 - M + cc, p.nx, p.sym[0], f);
      hoff[r] = min(y0 + c, p.ny - 1) * p.nx + gx;
      hneg[r] = f != 0;
    } else if (idx < G::N) {  // H_y: row c of the y-extended tile, column cx
      const int j = idx - G::NX, c = j >> 5, cx = j & 31;
      int f;
      const int gy = bmap_t<SYM>(y0 - M + c, p.ny, p.sym[1], f);
      hoff[r] = (int)FS + gy * p.nx + min(x0 + cx, p.nx - 1);
      hneg[r] = f != 0;
    }
  }
  auto stage = [&](int j, int b) {  // plane z0 + j -> buffer b
    const double *hp = H + (size_t)(z0 + j) * 3 * FS;
#pragma unroll
    for (int r = 0; r < G::PER; ++r) {
      const int idx = tid + DH_THREADS * r;
      if (idx < G::N) cp_async8(&sh[b][idx], hp + hoff[r]);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // register window of H_z along z: hz[t] = H_z(z0 - m + t)
  constexpr int HW = DH_Z + 2 * M, ZA = 2 * M + 2;
  double hz[HW];
  auto hzload = [&](int t) {
    hz[t] = 0.0;
    if (t < nzo + 2 * M) {
      int f;
      const int zz = zread(p, z0 - M + t, f);
      const double v = __ldg(H + (size_t)zz * 3 * FS + 2 * FS + off);
      hz[t] = f ? -v : v;
    }
  };
#pragma unroll
  for (int t = 0; t < (ZA < HW ? ZA : HW); ++t) hzload(t);
  stage(0, 0);
  // this plane's read-modify-write operands, loaded a plane ahead
  const bool rmw = valid && !rout;
  auto rmw_load = [&](int j, double &qo_, double &wo_) {
    qo_ = 0.0;
    wo_ = 0.0;
    if (rmw && j < nzo) {
      const int z = z0 + j;
      qo_ = qout[qplane(p, z) + 4 * FS + off];
      if (p.write_w) wo_ = w[(size_t)z * 5 * FS + 4 * FS + off];
    }
  };
  double qn_old, wn_old;
  rmw_load(0, qn_old, wn_old);
  bool bad = false;
#pragma unroll
  for (int j = 0; j < DH_Z; ++j) {
    if (j < nzo) {
      if (j + ZA < HW) hzload(j + ZA);
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      if (SYM) {  // mirrored halo values change sign (each copier fixes its own)
#pragma unroll
        for (int r = 0; r < G::PER; ++r) {
          const int idx = tid + DH_THREADS * r;
          if (idx < G::N && hneg[r]) sh[j & 1][idx] = -sh[j & 1][idx];
        }
      }
      __syncthreads();  // plane j staged; every thread is done with plane j - 1's buffer
      if (j + 1 < nzo) stage(j + 1, (j + 1) & 1);
      const double q_old = qn_old, w_old = wn_old;
      rmw_load(j + 1, qn_old, wn_old);
      const double *rx = &sh[j & 1][ty * G::XW + tx + M];
      const double *cy = &sh[j & 1][G::NX + (ty + M) * 32 + tx];
      double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
      for (int k = 1; k <= M; ++k) {
        sx = fma(p.a[k - 1], rx[k] - rx[-k], sx);
        sy = fma(p.a[k - 1], cy[32 * k] - cy[-32 * k], sy);
        sz = fma(p.a[k - 1], hz[j + M + k] - hz[j + M - k], sz);
      }
      if (valid) {
        const int z = z0 + j;
        const size_t o = (size_t)z * 5 * FS + 4 * FS + off;
        const double d = sx + sy + sz;
        if (rout) {
          rout[o] += d;
        } else {
          const double dd = p.dt * d;
          const double qn = fma(p.B, dd, q_old);
          qout[qplane(p, z) + 4 * FS + off] = qn;
          bad |= !isfinite(qn);
          if (p.write_w) w[o] = fma(p.two_reg ? p.beta : 1.0, dd, w_old);
        }
      }
    }
  }
  if (bad) atomicOr(flag, 1u);
}

// cudaFuncSetAttribute (dynamic shared memory above 48 KB) once per kernel and
// device: `done` holds one bit per device id (handles on several devices may
// share a process; a lost race only repeats the call)
template <typename K>
cudaError_t ensure_smem_attr(K kern, int smem, unsigned &done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned bit = 1u << (dev & 31);
  if (done & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) done |= bit;
  return e;
}

// OSBLI_NO_SPLIT=1 (testing): keep the production launch shape on small grids: no
// z-segment split of the z-pass pencils, no halving of the xy-pass segments (so
// that sanitizer runs on small grids reach the ring advance and the 8-plane
// pipelines of the 256^3 configuration)
inline bool no_split() {
  static const int v = [] {
    const char *e = std::getenv("OSBLI_NO_SPLIT");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return v != 0;
}

// z-pass staging box: one plane of a 32-column pencil, all five fields
bool qbuf_tensor_map(const double *q, const KParams &p, CUtensorMap *out) {
  if (p.nx < ZP_TX) return false;
  return tensor_map(q, p.nx, p.ny, 5, p.nz + 2 * p.G, ZP_TX, 1, 5, out);
}

// OSBLI_ZP_TMA=0 / OSBLI_XY_TMA=0 (testing): stage the z-pass / xy-pass with cp.async everywhere
inline bool env_on(const char *name) {
  const char *e = std::getenv(name);
  return !(e && e[0] == '0');
}
inline bool zp_tma_enabled() {
  static const bool v = env_on("OSBLI_ZP_TMA");
  return v;
}
inline bool xy_tma_enabled() {
  static const bool v = env_on("OSBLI_XY_TMA");
  return v;
}

template <int M>
cudaError_t zpass_launch(const KParams &p, const double *q, double *w, double *gz, int zb, int ze,
                         int zb1, int ze1, cudaStream_t s) {
  constexpr int smem = zp_smem_bytes<M>();
  // symmetry in z (one GPU only) gets its own instantiation: mirrored plane reads
  const int sz = (p.visc || p.cons) ? 2 : (p.zwrap && p.sym[2] ? 1 : 0);
  auto kern = sz == 2 ? zpass_kernel<M, 2> : sz == 1 ? zpass_kernel<M, 1> : zpass_kernel<M, 0>;
  static unsigned done[3] = {0, 0, 0};
  cudaError_t e = ensure_smem_attr(kern, smem, done[sz]);
  if (e != cudaSuccess) return e;
  const int gx = (p.nx + ZP_TX - 1) / ZP_TX, gy = p.ny;
  const int len = (ze - zb) > (ze1 - zb1) ? (ze - zb) : (ze1 - zb1);
  const int chunks = (len + ZP_TZ - 1) / ZP_TZ;
  // split the z-range into segments only when the pencils alone do not fill ~2 waves
  int nseg = (2 * 148 + gx * gy - 1) / (gx * gy);
  nseg = nseg < 1 ? 1 : (nseg > chunks ? chunks : nseg);
  if (no_split()) nseg = 1;
  int ntot = 0;
  const PlaneRange zr = plane_range(zb, ze, zb1, ze1, ((chunks + nseg - 1) / nseg) * ZP_TZ, &ntot);
  dim3 grid(gx * gy, 1, ntot);
#if OSBLI_ZP_PERSIST
  {  // experiment: OSBLI_ZP_GRID persistent CTAs per z segment
    static const int g = [] { const char *e = std::getenv("OSBLI_ZP_GRID"); return e ? std::atoi(e) : 0; }();
    if (g > 0 && g < gx * gy) grid.x = g;
  }
#endif
  CUtensorMap tm;
  std::memset(&tm, 0, sizeof(tm));
  const bool tma = zp_tma_enabled() && qbuf_tensor_map(q, p, &tm);
  kern<<<grid, ZP_THREADS, smem, s>>>(p, q, w, gz, zr, tm, tma ? 1 : 0);
  return cudaGetLastError();
}

template <int M>
cudaError_t xypass_launch(const KParams &p, const double *q, double *qout, double *w,
                          const double *gz, double *rout, unsigned int *flag, int zb, int ze,
                          int zb1, int ze1, cudaStream_t s) {
  constexpr int smem = ws::xy_smem_bytes<M>();
  // the six instantiations of the stepping paths (default, two-register, symmetric,
  // both, equation variants, variants with the two-register epilogue), then the same
  // with fused diagnostics
  const int tr = p.two_reg ? 1 : 0;
  const int v = ((p.visc || p.cons) ? 4 + tr : tr + (p.sym[0] || p.sym[1] ? 2 : 0)) +
                (p.dpart ? 6 : 0);
  using K = decltype(&ws::xypass_kernel<M, 0>);
  static const K kerns[12] = {ws::xypass_kernel<M, 0>,  ws::xypass_kernel<M, 1>,
                              ws::xypass_kernel<M, 2>,  ws::xypass_kernel<M, 3>,
                              ws::xypass_kernel<M, 4>,  ws::xypass_kernel<M, 5>,
                              ws::xypass_kernel<M, 8>,  ws::xypass_kernel<M, 9>,
                              ws::xypass_kernel<M, 10>, ws::xypass_kernel<M, 11>,
                              ws::xypass_kernel<M, 12>, ws::xypass_kernel<M, 13>};
  const K kern = kerns[v];
  static unsigned done[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  cudaError_t e = ensure_smem_attr(kern, smem, done[v]);
  if (e != cudaSuccess) return e;
  // planes per CTA: xy_seg<M>, halved while the grid would not cover the SMs (small grids)
  const int tiles = ((p.nx + ws::XY_TX - 1) / ws::XY_TX) * ((p.ny + ws::XY_TY - 1) / ws::XY_TY);
  const int nz1 = ze1 > zb1 ? ze1 - zb1 : 0;
  const int len = (ze - zb) > nz1 ? (ze - zb) : nz1;
  int seg = len < ws::xy_seg<M>() ? len : ws::xy_seg<M>();
  auto ctas = [&](int sg) { return tiles * ((ze - zb + sg - 1) / sg + (nz1 + sg - 1) / sg); };
  while (!no_split() && seg > 1 && ctas(seg) < 148) seg = (seg + 1) / 2;
  int ntot = 0;
  const PlaneRange zr = plane_range(zb, ze, zb1, ze1, seg, &ntot);
  dim3 grid((p.nx + ws::XY_TX - 1) / ws::XY_TX, (p.ny + ws::XY_TY - 1) / ws::XY_TY, ntot);
  using Gm = ws::XYGeom<M>;
  CUtensorMap tq, t22, t02, t12;
  std::memset(&tq, 0, sizeof(tq));
  std::memset(&t22, 0, sizeof(t22));
  std::memset(&t02, 0, sizeof(t02));
  std::memset(&t12, 0, sizeof(t12));
  const bool tma = xy_tma_enabled() && p.nx >= Gm::PX && p.ny >= Gm::HY &&
                   tensor_map(q, p.nx, p.ny, 5, p.nz + 2 * p.G, Gm::PX, Gm::HY, 5, &tq) &&
                   tensor_map(gz, p.nx, p.ny, 3, p.nz, Gm::PX, Gm::HY, 1, &t22) &&
                   tensor_map(gz, p.nx, p.ny, 3, p.nz, Gm::PX, ws::XY_TY, 1, &t02) &&
                   tensor_map(gz, p.nx, p.ny, 3, p.nz, Gm::GP, Gm::HY, 1, &t12);
  kern<<<grid, ws::XY_CTA, smem, s>>>(p, q, qout, w, gz, rout, flag, zr, tq, t22, t02, t12,
                                      tma ? 1 : 0);
  return cudaGetLastError();
}

template <int M>
cudaError_t diag_launch(const KParams &p, const double *q, double *tpart, cudaStream_t s) {
  constexpr int smem = 2 * 4 * DGGeom<M>::N * (int)sizeof(double);
  static unsigned done = 0;
  cudaError_t e = ensure_smem_attr(diag_kernel<M>, smem, done);
  if (e != cudaSuccess) return e;
  const dim3 grid((p.nx + 31) / 32, (p.ny + DG_TY - 1) / DG_TY, (p.nz + DG_Z - 1) / DG_Z);
  diag_kernel<M><<<grid, dim3(32, DG_TY), smem, s>>>(p, q, tpart, (int)(grid.x * grid.y));
  return cudaGetLastError();
}

}  // namespace

namespace detail {
template <>
cudaError_t zpass_m<OSBLI_M>(const KParams &p, const double *q, double *w, double *gz, int zb,
                             int ze, int zb1, int ze1, cudaStream_t s) {
  return zpass_launch<OSBLI_M>(p, q, w, gz, zb, ze, zb1, ze1, s);
}

template <>
cudaError_t xypass_m<OSBLI_M>(const KParams &p, const double *q, double *qout, double *w,
                              const double *gz, double *rout, unsigned int *flag, int zb, int ze,
                              int zb1, int ze1, cudaStream_t s) {
  return xypass_launch<OSBLI_M>(p, q, qout, w, gz, rout, flag, zb, ze, zb1, ze1, s);
}

template <>
cudaError_t divh_m<OSBLI_M>(const KParams &p, double *q_out, double *w, double *r_out,
                            unsigned int *flag, int zb, int ze, cudaStream_t s) {
  const dim3 grid((p.nx + 31) / 32, (p.ny + DH_TY - 1) / DH_TY, (ze - zb + DH_Z - 1) / DH_Z);
  const dim3 block(32, DH_TY);
  if (p.sym[0] || p.sym[1])
    divh_kernel<OSBLI_M, true><<<grid, block, 0, s>>>(p, p.hflux, q_out, w, r_out, flag, zb, ze);
  else
    divh_kernel<OSBLI_M, false><<<grid, block, 0, s>>>(p, p.hflux, q_out, w, r_out, flag, zb, ze);
  return cudaGetLastError();
}

template <>
cudaError_t diag_m<OSBLI_M>(const KParams &p, const double *q, double *tpart, cudaStream_t s) {
  return diag_launch<OSBLI_M>(p, q, tpart, s);
}

}  // namespace detail
}  // namespace osbli
