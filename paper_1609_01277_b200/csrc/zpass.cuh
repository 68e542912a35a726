// z-pass (included by kernels.cu inside namespace osbli::{anon}).
//
// Every term of the residual that differentiates along z (D_z, D_zz; the z
// halves of the skew-symmetric terms P:271-274, the z fluxes, the z parts of
// the viscous Laplacians P:274 and of the heat flux): the partial residual Rz
// (plus the optional source S) goes straight into the low-storage register,
// W' = A W + dt (Rz + S) (P:123,
// P:164; the xy-pass completes W <- W' + dt R_xy), plus g_i2 = D_z u_i for
// the xy-pass.
//
// A CTA owns a pencil of 32 x-columns x one y-row and marches through its
// z-range in chunks of TZ = 16 planes (two CTAs per SM).  Shared memory holds a ring of
// NR = TZ + 2m planes of the 13 z-stencil operands (formulas computed once per
// plane): consecutive chunks share their 2m overlap planes, so every
// plane is loaded from HBM once.  While chunk k is computed, the raw state of
// the TZ planes chunk k+1 adds is already in flight into a staging buffer
// (TMA: one 32-column x 5-field tensor box per plane, cp.async.bulk.tensor into
// an mbarrier, issued by the 32 lanes of warp 0; cp.async where the pencil is
// ragged or nx is odd), so the HBM latency hides behind the FP64 work.  Each
// thread produces RZ = 4 consecutive z outputs of its column from register
// windows.
constexpr int ZP_TX = 32;
// 16-plane chunks of 4 warps, two CTAs per SM (113.7 KB of shared memory each at
// m = 6): the ring advance of one CTA (two block barriers) overlaps the other's
// stencils (round 2: -6 % z-pass at o8, -2..-5 % at o12; 32-plane chunks of 8
// warps, one CTA per SM, before)
#ifndef OSBLI_ZP_TZ
#define OSBLI_ZP_TZ 16
#endif
#ifndef OSBLI_ZP_RZ
#define OSBLI_ZP_RZ 4
#endif
#ifndef OSBLI_ZP_ADV_UNROLL
#define OSBLI_ZP_ADV_UNROLL 4
#endif
#ifndef OSBLI_ZP_PERSIST
#define OSBLI_ZP_PERSIST 0
#endif
#ifndef OSBLI_ZP_MINB
#define OSBLI_ZP_MINB 2
#endif
constexpr int ZP_TZ = OSBLI_ZP_TZ;  // planes per chunk
constexpr int ZP_RZ = OSBLI_ZP_RZ;  // z outputs per thread
constexpr int ZP_THREADS = 32 * (ZP_TZ / ZP_RZ);  // 256
constexpr int ZP_NF = 13;
// staged operand slots
enum { ZS_RHO = 0, ZS_M0, ZS_M1, ZS_M2, ZS_E, ZS_U0, ZS_U1, ZS_U2, ZS_T, ZS_F0, ZS_F1, ZS_F2, ZS_G };

template <int M>
struct ZGeom {
  static constexpr int NR = ZP_TZ + 2 * M;      // ring slots (planes)
  static constexpr int RING = ZP_NF * NR * 32;  // doubles (a multiple of 16: RAW is 128-B aligned)
  static constexpr int RAW = 5 * ZP_TZ * 32;    // raw planes of the next chunk, [plane][field][32]
  // + the TMA mbarrier (8 bytes, padded to 16)
  static constexpr int BYTES = (RING + RAW) * (int)sizeof(double) + 16;
};
static_assert((ZP_NF * 32) % 16 == 0, "the raw staging buffer must stay 128-byte aligned");

template <int M>
constexpr int zp_smem_bytes() {
  return ZGeom<M>::BYTES;
}

// formulas of one staged point into ring slot `slot`, column c
template <int M>
__device__ __forceinline__ void zstore(const KParams &p, double *S, int slot, int c, double rho,
                                       double m0, double m1, double m2, double e) {
  constexpr int NR = ZGeom<M>::NR;
  const double r = rcp_rho(rho);
  const double u0 = m0 * r, u1 = m1 * r, u2 = m2 * r;
  const double pr = p.gm1 * (e - 0.5 * (m0 * u0 + m1 * u1 + m2 * u2));
  const double T = p.gM2 * pr * r;
  double *s = S + slot * 32 + c;
  s[ZS_RHO * NR * 32] = rho;
  s[ZS_M0 * NR * 32] = m0;
  s[ZS_M1 * NR * 32] = m1;
  s[ZS_M2 * NR * 32] = m2;
  s[ZS_E * NR * 32] = e;
  s[ZS_U0 * NR * 32] = u0;
  s[ZS_U1 * NR * 32] = u1;
  s[ZS_U2 * NR * 32] = u2;
  s[ZS_T * NR * 32] = T;
  // momentum flux F_i2 = 1/2 m_i u_2 + delta_i2 p  (skew half + pressure)
  s[ZS_F0 * NR * 32] = 0.5 * m0 * u2;
  s[ZS_F1 * NR * 32] = 0.5 * m1 * u2;
  s[ZS_F2 * NR * 32] = 0.5 * m2 * u2 + pr;
  // energy flux G_2 = (1/2 e + p) u_2  (skew half + pressure work)
  s[ZS_G * NR * 32] = (0.5 * e + pr) * u2;
}

// 16-byte asynchronous global -> shared copy (L2 only)
__device__ __forceinline__ void cp_async16z(double *smem, const double *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// register window of ring field f starting at ring slot slot0 (wraps modulo NR)
template <int M>
__device__ __forceinline__ void zwindow(const double *S, int f, int slot0, int lane,
                                        double (&v)[ZP_RZ + 2 * M]) {
  constexpr int NR = ZGeom<M>::NR;
#pragma unroll
  for (int t = 0; t < ZP_RZ + 2 * M; ++t) {
    int sl = slot0 + t;
    if (sl >= NR) sl -= NR;
    v[t] = S[(f * NR + sl) * 32 + lane];
  }
}

template <int M>
__device__ __forceinline__ double d1w(const KParams &p, const double (&v)[ZP_RZ + 2 * M], int j) {
  // one accumulator per output (the four outputs of a window supply the ILP;
  // OSBLI_STENCIL_CHAINS = 2 interleaves two partial sums)
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int k = 1; k <= M; ++k) {
    if (OSBLI_STENCIL_CHAINS == 1 || (k & 1)) s0 = fma(p.a[k - 1], v[j + M + k] - v[j + M - k], s0);
    else s1 = fma(p.a[k - 1], v[j + M + k] - v[j + M - k], s1);
  }
  return OSBLI_STENCIL_CHAINS == 1 ? s0 : s0 + s1;
}

// exactly zero on a constant window (D-22)
template <int M>
__device__ __forceinline__ double d2w(const KParams &p, const double (&v)[ZP_RZ + 2 * M], int j) {
#if OSBLI_D2_SBP
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int l = 0; l < M; ++l) {
    const double t = (v[j + M + l + 1] - v[j + M + l]) - (v[j + M - l] - v[j + M - l - 1]);
    if (OSBLI_STENCIL_CHAINS != 1 && (l & 1)) s1 = fma(p.cb[l], t, s1);
    else s0 = fma(p.cb[l], t, s0);
  }
  return OSBLI_STENCIL_CHAINS == 1 ? s0 : s0 + s1;
#else
  const double c = v[j + M];
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int k = 1; k <= M; ++k) {
    const double t = fma(-2.0, c, v[j + M + k] + v[j + M - k]);
    if (OSBLI_STENCIL_CHAINS == 1 || (k & 1)) s0 = fma(p.b[k], t, s0);
    else s1 = fma(p.b[k], t, s1);
  }
  return OSBLI_STENCIL_CHAINS == 1 ? s0 : s0 + s1;
#endif
}

// ZF = 0: periodic z / ghost planes; 1: symmetry in z (mirrored plane reads);
// 2: equation variants (mu(T), conservative viscous work; D-26, D-27) with
// run-time boundary handling.  Separate instantiations keep the default path lean.
template <int M, int ZF>
__global__ void __launch_bounds__(ZP_THREADS, OSBLI_ZP_MINB)
    zpass_kernel(const KParams p, const double *__restrict__ q, double *__restrict__ w,
                 double *__restrict__ gz, const PlaneRange zr,
                 const __grid_constant__ CUtensorMap tmq, const int use_tma) {
  constexpr bool SYMZ = ZF != 0;
  constexpr bool VAR = ZF == 2;
  using Zg = ZGeom<M>;
  constexpr int NR = Zg::NR;
  extern __shared__ __align__(128) double S[];
  double *RB = S + Zg::RING;
  uint64_t *tbar = reinterpret_cast<uint64_t *>(RB + Zg::RAW);
  unsigned tphase = 0;  // completed TMA phases of tbar
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // blockIdx.x enumerates (x-tile, y-row) pencils (grid.y would cap ny at 65535)
  const int gx = (p.nx + ZP_TX - 1) / ZP_TX;
  int zs, ze;
  if (!zr.segment(zs, ze)) return;
#if OSBLI_ZP_PERSIST
  // experiment: a grid smaller than the pencil count loops over the pencils
  for (unsigned pen = blockIdx.x; pen < (unsigned)(gx * p.ny); pen += gridDim.x) {
  __syncthreads();
  const int x0 = (int)(pen % gx) * ZP_TX, y = (int)(pen / gx);
#else
  const int x0 = (int)(blockIdx.x % gx) * ZP_TX, y = (int)(blockIdx.x / gx);
#endif
  const int nchunks = (ze - zs + ZP_TZ - 1) / ZP_TZ;
  const size_t FS = (size_t)p.nx * p.ny;
  // column this thread loads for staging slot c = tid & 31 (ragged tiles load any valid column)
  int xc = x0 + lane;
  if (xc >= p.nx) xc = wrapi(xc, p.nx);
  const size_t rowoff = (size_t)y * p.nx + xc;

  // ---- prologue: ring planes zl = 0..NR-1 (z = zs - M + zl), all loads in flight first
  {
    constexpr int NIT = (NR * 32 + ZP_THREADS - 1) / ZP_THREADS;
    double raw[NIT][5];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int idx = tid + it * ZP_THREADS;
      if (idx < NR * 32) {
        const int pl = idx >> 5;
        int fl;
        const double *qp = q + qplane(p, zread_t<SYMZ>(p, zs - M + pl, fl)) + rowoff;
        if (OSBLI_DEBUG_CHECKS && !(dbg_in(p, qp - q, qbuf_len(p)) &&
                                    dbg_in(p, qp - q + 4 * FS, qbuf_len(p))))
          qp = q;
#pragma unroll
        for (int f = 0; f < 5; ++f) raw[it][f] = __ldg(qp + f * FS);
        if (fl) raw[it][3] = -raw[it][3];  // rho u_z is odd under a z mirror
      }
    }
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int idx = tid + it * ZP_THREADS;
      if (idx < NR * 32)
        zstore<M>(p, S, idx >> 5, lane, raw[it][0], raw[it][1], raw[it][2], raw[it][3],
                  raw[it][4]);
    }
  }
  // raw planes of chunk kk: z = zs + kk*TZ + M + j, j = 0..TZ-1  ->  RB[j][f][c]
  // TMA boxes (or 16-byte copies of column pairs) when the pencil lies inside the
  // grid and rows start at even offsets (even nx: no pair straddles the periodic wrap)
  const bool pairs = (p.nx % 2) == 0 && x0 + ZP_TX <= p.nx;
  const bool tma = use_tma && pairs && !OSBLI_DEBUG_CHECKS;
  if (tma) {
    if (tid == 0) mbar_init(tbar, 1);
    tphase = 0;
  }
  auto issue_raw = [&](int kk) {
    if (tma) {
      // lanes 0..RZ-1 of every warp issue one plane box each (the issue of a warp's
      // TMA instructions is serial, so it is spread over the warps); a copy may
      // complete before the expect-tx: the phase still needs the one arrival
      if (tid == 0) mbar_expect_tx(tbar, ZP_TZ * 5 * 32 * (unsigned)sizeof(double));
      constexpr int PW = ZP_TZ / (ZP_THREADS / 32);  // planes per warp
      if (lane < PW) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        const int j = warp * PW + lane;
        int fl_;
        const int zb_ = zread_t<SYMZ>(p, zs + kk * ZP_TZ + M + j, fl_) + p.G;
        tma_load_box(RB + j * 5 * 32, &tmq, x0, y, 0, zb_, tbar);
      }
      return;
    }
    if (pairs) {
      // lanes 0-15: plane j, columns 2l, 2l+1; lanes 16-31: plane j + 1
      const int l2 = 2 * (lane & 15);
      const size_t roff = (size_t)y * p.nx + x0 + l2;
      for (int idx = 2 * warp + (lane >> 4); idx < ZP_TZ; idx += 2 * (ZP_THREADS / 32)) {
        int fl_;
        const double *qp = q + qplane(p, zread_t<SYMZ>(p, zs + kk * ZP_TZ + M + idx, fl_)) + roff;
        if (OSBLI_DEBUG_CHECKS && !(dbg_in(p, qp - q, qbuf_len(p)) &&
                                    dbg_in(p, qp - q + 4 * FS + 1, qbuf_len(p))))
          qp = q;
#pragma unroll
        for (int f = 0; f < 5; ++f) cp_async16z(RB + (idx * 5 + f) * 32 + l2, qp + f * FS);
      }
    } else {
      for (int idx = tid; idx < ZP_TZ * 32; idx += ZP_THREADS) {
        const int j = idx >> 5;
        int fl_;
        const double *qp = q + qplane(p, zread_t<SYMZ>(p, zs + kk * ZP_TZ + M + j, fl_)) + rowoff;
        if (OSBLI_DEBUG_CHECKS && !(dbg_in(p, qp - q, qbuf_len(p)) &&
                                    dbg_in(p, qp - q + 4 * FS, qbuf_len(p))))
          qp = q;
#pragma unroll
        for (int f = 0; f < 5; ++f) cp_async8(RB + (j * 5 + f) * 32 + lane, qp + f * FS);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  __syncthreads();  // the mbarrier is initialised
  if (nchunks > 1) issue_raw(1);
  __syncthreads();

  for (int k = 0; k < nchunks; ++k) {
    // ---- compute chunk k: outputs z = zs + k*TZ + warp*RZ + j
    const int zl0 = k * ZP_TZ + warp * ZP_RZ;  // local index of the window's first plane
    const int slot0 = zl0 % NR;
    // the low-storage register of the outputs: loaded now, used after the stencils
    double wold[5][ZP_RZ];
    {
      const int x = x0 + lane < p.nx ? x0 + lane : xc;
#pragma unroll
      for (int j = 0; j < ZP_RZ; ++j) {
        const int z = min(zs + zl0 + j, ze - 1);
        const size_t o = (size_t)z * 5 * FS + (size_t)y * p.nx + x;
#pragma unroll
        for (int f = 0; f < 5; ++f) wold[f][j] = p.read_w && !p.two_reg ? w[o + f * FS] : 0.0;
      }
    }
    double v[ZP_RZ + 2 * M];
    double g[3][ZP_RZ], R[5][ZP_RZ], u2c[ZP_RZ];
    double dTz[ZP_RZ];
    if (VAR) {
      // variants: mu(T) scales the viscous z-parts and the heat flux (D-26; the
      // grad-mu terms are pointwise and added by the xy-pass from D_z T); the
      // conservative form leaves the viscous work to D_j H_j (D-27)
      double mu[ZP_RZ];
      zwindow<M>(S, ZS_T, slot0, lane, v);
#pragma unroll
      for (int j = 0; j < ZP_RZ; ++j) {
        mu[j] = p.visc ? sutherland_mu(p, v[j + M]) : 1.0;
        dTz[j] = d1w<M>(p, v, j);
        R[4][j] = (p.kappa * mu[j]) * d2w<M>(p, v, j);
      }
      zwindow<M>(S, ZS_U2, slot0, lane, v);
#pragma unroll
      for (int j = 0; j < ZP_RZ; ++j) {
        g[2][j] = d1w<M>(p, v, j);
        const double d2u2 = d2w<M>(p, v, j);
        u2c[j] = v[j + M];
        const double V2 = mu[j] * (p.nu * (d2u2 + (1.0 / 3.0) * d2u2));
        R[3][j] = V2;
        if (!p.cons) R[4][j] = fma(u2c[j], V2, R[4][j]);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        zwindow<M>(S, ZS_U0 + i, slot0, lane, v);
#pragma unroll
        for (int j = 0; j < ZP_RZ; ++j) {
          g[i][j] = d1w<M>(p, v, j);
          const double Vi = mu[j] * (p.nu * d2w<M>(p, v, j));
          R[1 + i][j] = Vi;
          if (!p.cons) R[4][j] = fma(v[j + M], Vi, R[4][j]);
        }
      }
    } else {
    // velocity: g_i2 = D_z u_i, z-Laplacian parts of V_i and u_i V_i
    zwindow<M>(S, ZS_U2, slot0, lane, v);
#pragma unroll
    for (int j = 0; j < ZP_RZ; ++j) {
      g[2][j] = d1w<M>(p, v, j);
      const double d2u2 = d2w<M>(p, v, j);
      u2c[j] = v[j + M];
      const double V2 = p.nu * (d2u2 + (1.0 / 3.0) * d2u2);
      R[3][j] = V2;
      R[4][j] = u2c[j] * V2;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      zwindow<M>(S, ZS_U0 + i, slot0, lane, v);
#pragma unroll
      for (int j = 0; j < ZP_RZ; ++j) {
        g[i][j] = d1w<M>(p, v, j);
        const double Vi = p.nu * d2w<M>(p, v, j);
        R[1 + i][j] = Vi;
        R[4][j] = fma(v[j + M], Vi, R[4][j]);
      }
    }
    // heat flux: kappa D_zz T
    zwindow<M>(S, ZS_T, slot0, lane, v);
#pragma unroll
    for (int j = 0; j < ZP_RZ; ++j) R[4][j] = fma(p.kappa, d2w<M>(p, v, j), R[4][j]);
    }
    // skew advective + dilatation halves: -1/2 (u_2 D_z s + s g_22), s = rho, m_i, e
#pragma unroll
    for (int f = 0; f < 5; ++f) {
      zwindow<M>(S, ZS_RHO + f, slot0, lane, v);
#pragma unroll
      for (int j = 0; j < ZP_RZ; ++j) {
        const double ds = d1w<M>(p, v, j);
        const double t = fma(u2c[j], ds, v[j + M] * g[2][j]);
        if (f == 0) R[0][j] = -0.5 * t;
        else R[f][j] = fma(-0.5, t, R[f][j]);
        if (f == 3) R[0][j] = fma(-0.5, ds, R[0][j]);  // mass flux D_z(rho u_2) = D_z m_2
      }
    }
    // conservative flux halves: -D_z F_i2, -D_z G_2
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      zwindow<M>(S, ZS_F0 + f, slot0, lane, v);
#pragma unroll
      for (int j = 0; j < ZP_RZ; ++j) R[1 + f][j] -= d1w<M>(p, v, j);
    }
    const int x = x0 + lane;
    if (x < p.nx) {
#pragma unroll
      for (int j = 0; j < ZP_RZ; ++j) {
        const int z = zs + zl0 + j;
        if (z < ze) {
          const size_t o = (size_t)z * 5 * FS + (size_t)y * p.nx + x;
#pragma unroll
          for (int f = 0; f < 5; ++f) {
            const double rf = p.src ? R[f][j] + p.src[o + f * FS] : R[f][j];
            w[o + f * FS] = fma(p.A, wold[f][j], p.dt * rf);
          }
          const size_t og = (size_t)z * 3 * FS + (size_t)y * p.nx + x;
#pragma unroll
          for (int i = 0; i < 3; ++i) gz[og + i * FS] = g[i][j];
          if (VAR) p.dtz[(size_t)z * FS + (size_t)y * p.nx + x] = dTz[j];
        }
      }
    }
    if (k + 1 < nchunks) {
      // ---- advance the ring: planes of chunk k+1 replace the first TZ planes of chunk k
      if (tma) {
        mbar_wait(tbar, tphase & 1);
        ++tphase;
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      }
      __syncthreads();  // staged raw planes visible; every warp is done with chunk k
      // unrolled: the loads of all its points are in flight together (ZP_TZ*32 is a
      // multiple of the block size)
OSBLI_UNROLL(OSBLI_ZP_ADV_UNROLL)
      for (int idx = tid; idx < ZP_TZ * 32; idx += ZP_THREADS) {
        const int j = idx >> 5;
        const int slot = ((k + 1) * ZP_TZ + 2 * M + j) % NR;
        int fl = 0;
        if (SYMZ) zread(p, zs + (k + 1) * ZP_TZ + M + j, fl);
        const double *rb = RB + j * 5 * 32 + lane;
        const double m2 = rb[3 * 32];
        zstore<M>(p, S, slot, lane, rb[0], rb[32], rb[2 * 32], fl ? -m2 : m2, rb[4 * 32]);
      }
      __syncthreads();  // ring updated, staging buffer free
      if (k + 2 < nchunks) issue_raw(k + 2);
    }
  }
#if OSBLI_ZP_PERSIST
  }
#endif
}
