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
#include <cstdint>

#include "kernels.h"

namespace osbli {
namespace {

__device__ __forceinline__ int wrapi(int i, int n) {
  // periodic index: one conditional shift covers every tile halo when n exceeds
  // the stencil reach; the modulo only runs for grids smaller than that
  if (i < 0) i += n;
  else if (i >= n) i -= n;
  if ((unsigned)i >= (unsigned)n) {
    i %= n;
    if (i < 0) i += n;
  }
  return i;
}

// boundary map of index i in a direction of n points: periodic wrap, or the
// mirror about the boundary faces (symmetry: ghost -k <-> interior k-1,
// ghost n-1+k <-> interior n-k); flip = 1 after an odd number of mirrors, where
// a field's normal vector component changes sign
__device__ __forceinline__ int bmap(int i, int n, int sym, int &flip) {
  if (!sym) {
    flip = 0;
    return wrapi(i, n);
  }
  // one reflection at most (every halo of a grid at least m points wide)
  if ((unsigned)i < (unsigned)n) {
    flip = 0;
    return i;
  }
  if (i < 0 && i >= -n) {
    flip = 1;
    return -1 - i;
  }
  if (i >= n && i < 2 * n) {
    flip = 1;
    return 2 * n - 1 - i;
  }
  int c = i % (2 * n);
  if (c < 0) c += 2 * n;
  flip = c >= n;
  return flip ? 2 * n - 1 - c : c;
}

__device__ __forceinline__ size_t qplane(const KParams &p, int z) {
  return (size_t)(z + p.G) * 5 * (size_t)p.nx * p.ny;
}

// z index of the plane read for logical plane z (wrap or mirror on one GPU,
// ghost planes otherwise); flip = 1 when rho u_z changes sign (mirror)
__device__ __forceinline__ int zread(const KParams &p, int z, int &flip) {
  if (p.zwrap) return bmap(z, p.nz, p.sym[2], flip);
  flip = 0;
  return max(-p.G, min(z, p.nz - 1 + p.G));
}
// compile-time variant of bmap: SYM = false is the plain periodic wrap
template <bool SYM>
__device__ __forceinline__ int bmap_t(int i, int n, int sym, int &flip) {
  if (SYM) return bmap(i, n, sym, flip);
  flip = 0;
  return wrapi(i, n);
}
// compile-time variant: SYM = false is the periodic / ghost-plane read (flip = 0)
template <bool SYM>
__device__ __forceinline__ int zread_t(const KParams &p, int z, int &flip) {
  if (SYM) return zread(p, z, flip);
  flip = 0;
  if (p.zwrap) return wrapi(z, p.nz);
  return max(-p.G, min(z, p.nz - 1 + p.G));
}

// 8-byte asynchronous global -> shared copy (LDGSTS); completed with cp.async.wait_group
__device__ __forceinline__ void cp_async8(double *smem, const double *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}

// 1/rho without the IEEE division's special-case path: the hardware seed
// (rcp.approx.ftz.f64) and two Newton steps, accurate to about 1 ulp for the
// normal, positive densities of the method (not correctly rounded: round-off only)
#ifndef OSBLI_FAST_RCP
#define OSBLI_FAST_RCP 1
#endif
__device__ __forceinline__ double rcp_rho(double x) {
#if OSBLI_FAST_RCP
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
#else
  return 1.0 / x;
#endif
}

// Sutherland's law in dimensionless form (D-26): mu(T) = T^1.5 (1 + S)/(T + S),
// mu(1) = 1, and its derivative mu'(T) = mu (3/(2T) - 1/(T + S))
// (T^1.5 = T^2 / sqrt(T) from the hardware reciprocal-square-root seed and two
// Newton steps; reciprocals as rcp_rho: about 1 ulp, round-off only, D-28)
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  return y * fma(-hx * y, y, 1.5);
}
__device__ __forceinline__ double sutherland_mu(const KParams &p, double T) {
  return (T * T) * rsqrt_fast(T) * ((1.0 + p.suth) * rcp_rho(T + p.suth));
}
__device__ __forceinline__ double sutherland_dmu(const KParams &p, double T, double mu) {
  return mu * (1.5 * rcp_rho(T) - rcp_rho(T + p.suth));
}

// stencil sums: one dependent FMA chain per output (the four outputs of a register
// window are independent); 2 interleaves two partial sums per output
#ifndef OSBLI_STENCIL_CHAINS
#define OSBLI_STENCIL_CHAINS 1
#endif

// second derivatives in first differences (D-22); 0 selects the (f+ + f-) - 2f form
#ifndef OSBLI_D2_SBP
#define OSBLI_D2_SBP 1
#endif
#include "zpass.cuh"
#include "xypass.cuh"
#include "xypass_ws.cuh"

// ------------------------------------------------------------------ diagnostics
__global__ void velocity_kernel(const KParams p, const double *__restrict__ q,
                                double *__restrict__ u, int zlo, int zhi) {
  const size_t FS = (size_t)p.nx * p.ny;
  const size_t n = (size_t)(zhi - zlo) * FS;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x) {
    const int z = zlo + (int)(t / FS);
    const size_t off = t % FS;
    const double *qp = q + qplane(p, z) + off;
    const double r = 1.0 / qp[0];
    double *up = u + (size_t)(z + p.G) * 3 * FS + off;
    up[0] = qp[FS] * r;
    up[FS] = qp[2 * FS] * r;
    up[2 * FS] = qp[3 * FS] * r;
  }
}

template <int M>
__global__ void __launch_bounds__(256) diag_kernel(const KParams p, const double *__restrict__ q,
                                                   const double *__restrict__ u,
                                                   double *__restrict__ part) {
  const int z = blockIdx.x;
  const size_t FS = (size_t)p.nx * p.ny;
  double sk = 0.0, se = 0.0, sd = 0.0;
  for (int t = threadIdx.x; t < (int)FS; t += blockDim.x) {
    const int x = t % p.nx, y = t / p.nx;
    const double *qp = q + qplane(p, z) + t;
    double g[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double *ui = u + 3 * FS * 0 + (size_t)i * FS;
      double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
      for (int k = 1; k <= M; ++k) {
        // taps with the parity of u_i: odd under the mirror of direction i
        int fxp, fxm, fyp, fym, fzp, fzm;
        const int xp = bmap(x + k, p.nx, p.sym[0], fxp), xm = bmap(x - k, p.nx, p.sym[0], fxm);
        const int yp = bmap(y + k, p.ny, p.sym[1], fyp), ym = bmap(y - k, p.ny, p.sym[1], fym);
        const int zpl = zread(p, z + k, fzp), zml = zread(p, z - k, fzm);
        const size_t rowp = (size_t)y * p.nx, zp_ = (size_t)(zpl + p.G) * 3 * FS,
                     zm_ = (size_t)(zml + p.G) * 3 * FS, z0_ = (size_t)(z + p.G) * 3 * FS;
        auto sg = [&](int fl, int d) { return (fl && i == d) ? -1.0 : 1.0; };
        sx = fma(p.a[k - 1],
                 sg(fxp, 0) * ui[z0_ + rowp + xp] - sg(fxm, 0) * ui[z0_ + rowp + xm], sx);
        sy = fma(p.a[k - 1],
                 sg(fyp, 1) * ui[z0_ + (size_t)yp * p.nx + x] -
                     sg(fym, 1) * ui[z0_ + (size_t)ym * p.nx + x],
                 sy);
        sz = fma(p.a[k - 1], sg(fzp, 2) * ui[zp_ + rowp + x] - sg(fzm, 2) * ui[zm_ + rowp + x],
                 sz);
      }
      g[i][0] = sx;
      g[i][1] = sy;
      g[i][2] = sz;
    }
    const double rho = qp[0];
    const double *uc = u + (size_t)(z + p.G) * 3 * FS + t;
    const double u0 = uc[0], u1 = uc[FS], u2 = uc[2 * FS];
    sk += 0.5 * rho * (u0 * u0 + u1 * u1 + u2 * u2);
    const double w0 = g[2][1] - g[1][2], w1 = g[0][2] - g[2][0], w2 = g[1][0] - g[0][1];
    se += 0.5 * rho * (w0 * w0 + w1 * w1 + w2 * w2);
    const double th = g[0][0] + g[1][1] + g[2][2];
    const double s01 = g[0][1] + g[1][0], s02 = g[0][2] + g[2][0], s12 = g[1][2] + g[2][1];
    double phi = p.nu * (2.0 * (g[0][0] * g[0][0] + g[1][1] * g[1][1] + g[2][2] * g[2][2]) +
                         s01 * s01 + s02 * s02 + s12 * s12 - (2.0 / 3.0) * th * th);
    if (p.visc) {  // tau carries mu(T) (D-26)
      const double pr = p.gm1 * (qp[4 * FS] - 0.5 * rho * (u0 * u0 + u1 * u1 + u2 * u2));
      phi *= sutherland_mu(p, p.gM2 * pr / rho);
    }
    sd += phi;
  }
  // fixed-shape tree reduction -> deterministic, decomposition-independent
  __shared__ double red[3][256];
  red[0][threadIdx.x] = sk;
  red[1][threadIdx.x] = se;
  red[2][threadIdx.x] = sd;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      red[0][threadIdx.x] += red[0][threadIdx.x + s];
      red[1][threadIdx.x] += red[1][threadIdx.x + s];
      red[2][threadIdx.x] += red[2][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[3 * z + 0] = red[0][0];
    part[3 * z + 1] = red[1][0];
    part[3 * z + 2] = red[2][0];
  }
}

// ------------------------------------------------------------------ conservative viscous work
// D_j H_j (H_j = u_i tau_ij from the xy-pass; H_j odd under the mirror of
// direction j) added to the energy of the finished stage (D-27):
//   residual: R_E += D;  2N: W_E += dt D (write_w), Q'_E += B dt D;
//   two-register: Q'_E += alpha dt D, Q_old_E += beta dt D (write_w).
// A CTA covers a 32 x 8 tile of the plane and marches through DH_Z planes:
// per plane H_x (tile rows + x halo) and H_y (tile columns + y halo) are staged in
// shared memory (the next plane's values are loaded into registers while the
// current one is computed); H_z comes from a per-thread register window along z.
constexpr int DH_Z = 8;
template <int M>
struct DHGeom {
  static constexpr int XW = 32 + 2 * M;                       // H_x row width
  static constexpr int NX = 8 * XW, NY = (8 + 2 * M) * 32;    // staged elements
  static constexpr int PER = (NX + NY + 255) / 256;           // per thread
};
template <int M, bool SYM>
__device__ __forceinline__ void divh_fetch(const KParams &p, const double *__restrict__ H, int z,
                                           int x0, int y0, int tid, double (&v)[DHGeom<M>::PER]) {
  using G = DHGeom<M>;
  const size_t FS = (size_t)p.nx * p.ny;
  const double *hp = H + (size_t)z * 3 * FS;
#pragma unroll
  for (int r = 0; r < G::PER; ++r) {
    const int idx = tid + 256 * r;
    v[r] = 0.0;
    if (idx < G::NX) {  // H_x: row ty, column c of the x-extended row
      const int ty = idx / G::XW, c = idx - ty * G::XW;
      int f;
      const int gx = bmap_t<SYM>(x0 - M + c, p.nx, p.sym[0], f);
      const int gy = min(y0 + ty, p.ny - 1);
      const double h = __ldg(hp + (size_t)gy * p.nx + gx);
      v[r] = f ? -h : h;
    } else if (idx < G::NX + G::NY) {  // H_y: row c of the y-extended tile, column tx
      const int j = idx - G::NX, c = j >> 5, tx = j & 31;
      int f;
      const int gy = bmap_t<SYM>(y0 - M + c, p.ny, p.sym[1], f);
      const int gx = min(x0 + tx, p.nx - 1);
      const double h = __ldg(hp + FS + (size_t)gy * p.nx + gx);
      v[r] = f ? -h : h;
    }
  }
}

template <int M, bool SYM>
__global__ void __launch_bounds__(256, 4) divh_kernel(const KParams p,
                                                      const double *__restrict__ H,
                                                      double *__restrict__ qout,
                                                      double *__restrict__ w,
                                                      double *__restrict__ rout,
                                                      unsigned int *__restrict__ flag, int zb,
                                                      int ze) {
  using G = DHGeom<M>;
  __shared__ double sh[G::NX + G::NY];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 8;
  const int x = x0 + tx, y = y0 + ty;
  const bool valid = x < p.nx && y < p.ny;
  const int z0 = zb + blockIdx.z * DH_Z;
  const int nzo = min(DH_Z, ze - z0);
  const size_t FS = (size_t)p.nx * p.ny;
  const size_t off = (size_t)min(y, p.ny - 1) * p.nx + min(x, p.nx - 1);
  // register window of H_z along z
  double hz[DH_Z + 2 * M];
#pragma unroll
  for (int t = 0; t < DH_Z + 2 * M; ++t) {
    hz[t] = 0.0;
    if (t < nzo + 2 * M) {
      int f;
      const int zz = zread(p, z0 - M + t, f);
      const double v = __ldg(H + (size_t)zz * 3 * FS + 2 * FS + off);
      hz[t] = f ? -v : v;
    }
  }
  double nxt[G::PER];
  divh_fetch<M, SYM>(p, H, z0, x0, y0, tid, nxt);
  bool bad = false;
#pragma unroll
  for (int j = 0; j < DH_Z; ++j) {
    if (j >= nzo) break;
    const int z = z0 + j;
    // this plane's read-modify-write operands, in flight during the staging below
    const size_t o = (size_t)z * 5 * FS + 4 * FS + off;
    double *qe = qout ? qout + qplane(p, z) + 4 * FS + off : nullptr;
    double q_old = 0.0, w_old = 0.0;
    if (valid && !rout) {
      q_old = *qe;
      if (p.write_w) w_old = w[o];
    }
    __syncthreads();  // the previous plane's reads are done
#pragma unroll
    for (int r = 0; r < G::PER; ++r) {
      const int idx = tid + 256 * r;
      if (idx < G::NX + G::NY) sh[idx] = nxt[r];
    }
    __syncthreads();
    if (j + 1 < nzo) divh_fetch<M, SYM>(p, H, z + 1, x0, y0, tid, nxt);
    const double *rx = sh + ty * G::XW + tx + M;
    const double *cy = sh + G::NX + (ty + M) * 32 + tx;
    double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
    for (int k = 1; k <= M; ++k) {
      sx = fma(p.a[k - 1], rx[k] - rx[-k], sx);
      sy = fma(p.a[k - 1], cy[32 * k] - cy[-32 * k], sy);
      sz = fma(p.a[k - 1], hz[j + M + k] - hz[j + M - k], sz);
    }
    if (!valid) continue;
    const double d = sx + sy + sz;
    if (rout) {
      rout[o] += d;
      continue;
    }
    const double dd = p.dt * d;
    const double qn = fma(p.B, dd, q_old);
    *qe = qn;
    bad |= !isfinite(qn);
    if (p.write_w) w[o] = fma(p.two_reg ? p.beta : 1.0, dd, w_old);
  }
  if (bad) atomicOr(flag, 1u);
}

// ------------------------------------------------------------------ symmetric z on slabs
// ghost plane -k <- interior k-1 (side 0), nz-1+k <- nz-k (side 1), k = 1..G;
// rho u_z (field 3) is odd under the mirror
// (for a buffer of nf fields per plane starting at its first ghost plane; field
// `odd` is odd under the mirror: rho u_z for Q, H_z for the viscous-work flux)
__global__ void mirror_ghosts_kernel(const KParams p, double *__restrict__ base, int nf, int odd,
                                     int side) {
  const size_t FS = (size_t)p.nx * p.ny;
  const size_t PL = (size_t)nf * FS;
  const size_t n = (size_t)p.G * PL;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x) {
    const int k = 1 + (int)(t / PL);
    const size_t rem = t % PL;
    const int f = (int)(rem / FS);
    const int zg = side == 0 ? -k : p.nz - 1 + k;
    const int zi = side == 0 ? k - 1 : p.nz - k;
    const double v = base[(size_t)(zi + p.G) * PL + rem];
    base[(size_t)(zg + p.G) * PL + rem] = f == odd ? -v : v;
  }
}

// ------------------------------------------------------------------ layout conversion
__global__ void abi_to_internal_kernel(const KParams p, const double *__restrict__ src,
                                       double *__restrict__ q) {
  const size_t FS = (size_t)p.nx * p.ny;
  const size_t n = 5 * FS * p.nz;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t f = t / (FS * p.nz), rem = t % (FS * p.nz);
    const int z = (int)(rem / FS);
    const size_t off = rem % FS;
    q[qplane(p, z) + f * FS + off] = src[t];
  }
}

__global__ void internal_to_abi_kernel(const KParams p, const double *__restrict__ q,
                                       double *__restrict__ dst, int nfields, int ghosted) {
  const size_t FS = (size_t)p.nx * p.ny;
  const size_t n = (size_t)nfields * FS * p.nz;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t f = t / (FS * p.nz), rem = t % (FS * p.nz);
    const int z = (int)(rem / FS);
    const size_t off = rem % FS;
    const size_t plane = ghosted ? (size_t)(z + p.G) : (size_t)z;
    dst[t] = q[plane * nfields * FS + f * FS + off];
  }
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

template <int M>
cudaError_t zpass_launch(const KParams &p, const double *q, double *w, double *gz, int zb, int ze,
                         cudaStream_t s) {
  constexpr int smem = zp_smem_bytes<M>();
  // symmetry in z (one GPU only) gets its own instantiation: mirrored plane reads
  const int sz = (p.visc || p.cons) ? 2 : (p.zwrap && p.sym[2] ? 1 : 0);
  auto kern = sz == 2 ? zpass_kernel<M, 2> : sz == 1 ? zpass_kernel<M, 1> : zpass_kernel<M, 0>;
  static unsigned done[3] = {0, 0, 0};
  cudaError_t e = ensure_smem_attr(kern, smem, done[sz]);
  if (e != cudaSuccess) return e;
  const int gx = (p.nx + ZP_TX - 1) / ZP_TX, gy = p.ny;
  const int chunks = (ze - zb + ZP_TZ - 1) / ZP_TZ;
  // split the z-range into segments only when the pencils alone do not fill ~2 waves
  int nseg = (2 * 148 + gx * gy - 1) / (gx * gy);
  nseg = nseg < 1 ? 1 : (nseg > chunks ? chunks : nseg);
  const int seg_len = ((chunks + nseg - 1) / nseg) * ZP_TZ;
  nseg = (ze - zb + seg_len - 1) / seg_len;
  dim3 grid(gx * gy, 1, nseg);
  kern<<<grid, ZP_THREADS, smem, s>>>(p, q, w, gz, zb, ze, seg_len);
  return cudaGetLastError();
}

#ifndef OSBLI_XY_WS
#define OSBLI_XY_WS 1
#endif
template <int M>
cudaError_t xypass_launch(const KParams &p, const double *q, double *qout, double *w,
                          const double *gz, double *rout, unsigned int *flag, int zb, int ze,
                          cudaStream_t s) {
#if OSBLI_XY_WS
  constexpr int smem = ws::xy_smem_bytes<M>();
  const int v = (p.visc || p.cons) ? 4 : (p.two_reg ? 1 : 0) + (p.sym[0] || p.sym[1] ? 2 : 0);
  auto kern = v == 0   ? ws::xypass_kernel<M, 0>
              : v == 1 ? ws::xypass_kernel<M, 1>
              : v == 2 ? ws::xypass_kernel<M, 2>
              : v == 3 ? ws::xypass_kernel<M, 3>
                       : ws::xypass_kernel<M, 4>;
  static unsigned done[5] = {0, 0, 0, 0, 0};
  cudaError_t e = ensure_smem_attr(kern, smem, done[v]);
  if (e != cudaSuccess) return e;
  // planes per CTA: XY_SEG, halved while the grid would not cover the SMs (small grids)
  const int tiles = ((p.nx + ws::XY_TX - 1) / ws::XY_TX) * ((p.ny + ws::XY_TY - 1) / ws::XY_TY);
  int seg = ze - zb < ws::XY_SEG ? ze - zb : ws::XY_SEG;
  while (seg > 1 && tiles * ((ze - zb + seg - 1) / seg) < 148) seg = (seg + 1) / 2;
  dim3 grid((p.nx + ws::XY_TX - 1) / ws::XY_TX, (p.ny + ws::XY_TY - 1) / ws::XY_TY,
            (ze - zb + seg - 1) / seg);
  kern<<<grid, ws::XY_CTA, smem, s>>>(p, q, qout, w, gz, rout, flag, zb, ze, seg);
#else
  // the non-specialised comparison kernel has no equation variants
  if (p.visc || p.cons) return cudaErrorNotSupported;
  constexpr int smem = xy_smem_bytes<M>();
  static unsigned done = 0;
  cudaError_t e = ensure_smem_attr(xypass_kernel<M>, smem, done);
  if (e != cudaSuccess) return e;
  dim3 grid((p.nx + XY_TX - 1) / XY_TX, (p.ny + XY_TY - 1) / XY_TY, ze - zb);
  xypass_kernel<M><<<grid, XY_THREADS, smem, s>>>(p, q, qout, w, gz, rout, flag, zb);
#endif
  return cudaGetLastError();
}

template <int M>
cudaError_t diag_launch(const KParams &p, const double *q, const double *u, double *part,
                        cudaStream_t s) {
  diag_kernel<M><<<p.nz, 256, 0, s>>>(p, q, u, part);
  return cudaGetLastError();
}

int grid1d(size_t n) {
  size_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

#define OSBLI_DISPATCH_M(m, CALL) \
  switch (m) {                    \
    case 1: return CALL<1>;       \
    case 2: return CALL<2>;       \
    case 3: return CALL<3>;       \
    case 4: return CALL<4>;       \
    case 5: return CALL<5>;       \
    case 6: return CALL<6>;       \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_zpass(const KParams &p, const double *q_in, double *w, double *gz, int zb,
                         int ze, cudaStream_t s, long long *launches) {
  if (ze <= zb) return cudaSuccess;
  ++*launches;
#define ZCALL(MM) zpass_launch<MM>(p, q_in, w, gz, zb, ze, s)
  switch (p.m) {
    case 1: return ZCALL(1);
    case 2: return ZCALL(2);
    case 3: return ZCALL(3);
    case 4: return ZCALL(4);
    case 5: return ZCALL(5);
    case 6: return ZCALL(6);
    default: return cudaErrorInvalidValue;
  }
#undef ZCALL
}

cudaError_t launch_xypass(const KParams &p, const double *q_in, double *q_out, double *w,
                          const double *gz, double *r_out, unsigned int *flag,
                          int zb, int ze, cudaStream_t s, long long *launches) {
  if (ze <= zb) return cudaSuccess;
  ++*launches;
#define XCALL(MM) xypass_launch<MM>(p, q_in, q_out, w, gz, r_out, flag, zb, ze, s)
  switch (p.m) {
    case 1: return XCALL(1);
    case 2: return XCALL(2);
    case 3: return XCALL(3);
    case 4: return XCALL(4);
    case 5: return XCALL(5);
    case 6: return XCALL(6);
    default: return cudaErrorInvalidValue;
  }
#undef XCALL
}

cudaError_t launch_divh(const KParams &p, double *q_out, double *w, double *r_out,
                        unsigned int *flag, int zb, int ze, cudaStream_t s, long long *launches) {
  if (ze <= zb) return cudaSuccess;
  ++*launches;
  const dim3 grid((p.nx + 31) / 32, (p.ny + 7) / 8, (ze - zb + DH_Z - 1) / DH_Z);
  const dim3 block(32, 8);
  const bool sym = p.sym[0] || p.sym[1];
#define DCALL(MM)                                                                   \
  if (sym) divh_kernel<MM, true><<<grid, block, 0, s>>>(p, p.hflux, q_out, w, r_out, flag, zb, ze); \
  else divh_kernel<MM, false><<<grid, block, 0, s>>>(p, p.hflux, q_out, w, r_out, flag, zb, ze)
  switch (p.m) {
    case 1: DCALL(1); break;
    case 2: DCALL(2); break;
    case 3: DCALL(3); break;
    case 4: DCALL(4); break;
    case 5: DCALL(5); break;
    case 6: DCALL(6); break;
    default: return cudaErrorInvalidValue;
  }
#undef DCALL
  return cudaGetLastError();
}

cudaError_t launch_mirror_planes(const KParams &p, double *base, int nf, int odd, int side,
                                 cudaStream_t s, long long *launches) {
  ++*launches;
  const size_t n = (size_t)p.G * nf * p.nx * p.ny;
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  mirror_ghosts_kernel<<<(int)blocks, 256, 0, s>>>(p, base, nf, odd, side);
  return cudaGetLastError();
}

cudaError_t launch_mirror_ghosts(const KParams &p, double *q, int side, cudaStream_t s,
                                 long long *launches) {
  return launch_mirror_planes(p, q, 5, 3, side, s, launches);
}

cudaError_t launch_stage(const KParams &p, const double *q_in, double *q_out, double *w,
                         double *gz, double *r_out, unsigned int *flag, cudaStream_t s,
                         long long *launches) {
  cudaError_t e = launch_zpass(p, q_in, w, gz, 0, p.nz, s, launches);
  if (e != cudaSuccess) return e;
  e = launch_xypass(p, q_in, q_out, w, gz, r_out, flag, 0, p.nz, s, launches);
  if (e != cudaSuccess || !p.cons) return e;
  return launch_divh(p, q_out, w, r_out, flag, 0, p.nz, s, launches);
}

cudaError_t launch_diagnostics(const KParams &p, const double *q_in, double *scratch,
                               double *part, cudaStream_t s, long long *launches) {
  // velocity on the interior planes (+ ghost planes when they are in use)
  const int zlo = p.zwrap ? 0 : -p.G, zhi = p.zwrap ? p.nz : p.nz + p.G;
  const size_t n = (size_t)(zhi - zlo) * p.nx * p.ny;
  velocity_kernel<<<grid1d(n), 256, 0, s>>>(p, q_in, scratch, zlo, zhi);
  ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ++*launches;
#define DCALL(MM) diag_launch<MM>(p, q_in, scratch, part, s)
  switch (p.m) {
    case 1: return DCALL(1);
    case 2: return DCALL(2);
    case 3: return DCALL(3);
    case 4: return DCALL(4);
    case 5: return DCALL(5);
    case 6: return DCALL(6);
    default: return cudaErrorInvalidValue;
  }
#undef DCALL
}

cudaError_t launch_abi_to_internal(const KParams &p, const double *src, double *q, cudaStream_t s,
                                   long long *launches) {
  ++*launches;
  abi_to_internal_kernel<<<grid1d(5 * (size_t)p.nx * p.ny * p.nz), 256, 0, s>>>(p, src, q);
  return cudaGetLastError();
}

cudaError_t launch_internal_to_abi(const KParams &p, const double *q, double *dst, int nfields,
                                   int ghosted, cudaStream_t s, long long *launches) {
  ++*launches;
  internal_to_abi_kernel<<<grid1d((size_t)nfields * p.nx * p.ny * p.nz), 256, 0, s>>>(
      p, q, dst, nfields, ghosted);
  return cudaGetLastError();
}

}  // namespace osbli
