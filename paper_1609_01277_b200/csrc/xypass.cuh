// xy-pass (included by kernels.cu inside namespace osbli::{anon}).
//
// One CTA = one 32 x 16 tile of one z-plane, 256 threads, 1 CTA per SM.
// Shared memory holds, on the tile plus an m-wide halo (periodic wrap in x, y):
//   rho, m0, m1, m2, e, p, r = 1/rho   (formulas; EOS P:259-266)
//   g02, g12, g22                      (D_z u_i from the z-pass)
// u_i = m_i r and T = gamma M^2 p r are formed on the fly from register windows.
// Each thread evaluates its derivatives from register windows of RX = RY = 4
// consecutive outputs ((4 + 2m) shared loads for 4 outputs instead of 2m per
// output), and the 8 warps split into a velocity group (A: viscous terms,
// velocity gradients, heat flux, dissipation) and a conservative group
// (B: skew-symmetric advection and flux terms) so that both groups
// keep a moderate register footprint.
//   phase X  : x-derivatives of tile rows (A, B) + g00, g10 on the halo rows (ext)
//   phase Y  : y-derivatives (A, B), combined with phase-X partials
//   epilogue : W <- W' + dt (A + B), Q' <- Q + B W  (low-storage RK, P:123, P:164;
//              W' = A W + dt Rz was written by the z-pass)
constexpr int XY_TX = 32;
constexpr int XY_TY = 16;
constexpr int XY_RX = 4;
constexpr int XY_RY = 4;
constexpr int XY_THREADS = 256;
constexpr int XY_NF = 10;
enum { XF_RHO = 0, XF_M0, XF_M1, XF_M2, XF_E, XF_P, XF_R, XF_G02, XF_G12, XF_G22 };

template <int M>
struct XYGeom {
  static constexpr int HX = XY_TX + 2 * M;
  static constexpr int PX = HX | 1;  // odd pitch (doubles): conflict-free column access
  static constexpr int HY = XY_TY + 2 * M;
  static constexpr int FSZ = HY * PX;           // one staged field
  static constexpr int TP = XY_TX + 1;         // odd row pitch of the per-point arrays
  static constexpr int NPT = TP * XY_TY;        // tile points (padded)
  static constexpr int EXT = TP * HY;           // g00 / g10 on the y-extended tile
  static constexpr int W = 4 + 2 * M;           // window length (RX = RY = 4)
  // layout (doubles): fields | E0 | E1 | XA[5] | XB[5] | PF[5] (prefetched W')
  static constexpr int OFF_E0 = XY_NF * FSZ;
  static constexpr int OFF_E1 = OFF_E0 + EXT;
  static constexpr int OFF_XA = OFF_E1 + EXT;
  static constexpr int OFF_XB = OFF_XA + 5 * NPT;
  static constexpr int OFF_PF = OFF_XB + 5 * NPT;
  static constexpr int TOTAL = OFF_PF + 5 * XY_TX * XY_TY;
  static constexpr int BYTES = TOTAL * (int)sizeof(double);
};

template <int M>
constexpr int xy_smem_bytes() {
  return XYGeom<M>::BYTES;
}

// Window elements that are products are rounded explicitly (__dmul_rn): the
// compiler may otherwise contract a product into the stencil difference
// (f+ - f-) differently for different taps, and a uniform state would no
// longer cancel exactly (SURVEY §8(c) equilibrium pin).
// window of W values starting at base, stride `st` (doubles)
template <int W>
__device__ __forceinline__ void ldwin(const double *base, int st, double (&v)[W]) {
#pragma unroll
  for (int k = 0; k < W; ++k) v[k] = base[k * st];
}

template <int M, int W>
__device__ __forceinline__ double wd1(const KParams &p, const double (&v)[W], int j) {
  // two interleaved partial sums halve the dependent FMA chain
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int k = 1; k <= M; ++k) {
    if (k & 1) s0 = fma(p.a[k - 1], v[j + M + k] - v[j + M - k], s0);
    else s1 = fma(p.a[k - 1], v[j + M + k] - v[j + M - k], s1);
  }
  return s0 + s1;
}

// second derivative, exactly zero on a constant window: sum b_k ((f+ + f-) - 2 f)
template <int M, int W>
__device__ __forceinline__ double wd2(const KParams &p, const double (&v)[W], int j) {
  const double c = v[j + M];
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int k = 1; k <= M; ++k) {
    const double t = fma(-2.0, c, v[j + M + k] + v[j + M - k]);
    if (k & 1) s0 = fma(p.b[k], t, s0);
    else s1 = fma(p.b[k], t, s1);
  }
  return s0 + s1;
}

// Velocity group, one direction (DIR 0 = x: phase X, DIR 1 = y: phase Y).
//   out: g_0d, g_1d, g_2d (velocity gradients along d), second derivatives of
//   u_i and T along d, and the mixed derivatives needed along d.
template <int M, int DIR>
struct VelResult {
  double g[3][4], d2u[3][4], d2T[4], mixA[4], mixB[4], mixC[4], mixD[4], uc[3][4];
};

template <int M, int DIR>
__device__ __forceinline__ void velocity_dir(const KParams &p, const double *S, int base, int st,
                                             const double *E0, const double *E1, int ebase,
                                             VelResult<M, DIR> &o) {
  using Gm = XYGeom<M>;
  constexpr int W = Gm::W;
  double r[W], v[W], t[W];
  ldwin<W>(S + XF_R * Gm::FSZ + base, st, r);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ldwin<W>(S + (XF_M0 + i) * Gm::FSZ + base, st, t);
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = __dmul_rn(t[k], r[k]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      o.g[i][j] = wd1<M, W>(p, v, j);
      o.d2u[i][j] = wd2<M, W>(p, v, j);
      o.uc[i][j] = v[j + M];
    }
  }
  ldwin<W>(S + XF_P * Gm::FSZ + base, st, t);
#pragma unroll
  for (int k = 0; k < W; ++k) v[k] = __dmul_rn(__dmul_rn(p.gM2, t[k]), r[k]);
#pragma unroll
  for (int j = 0; j < 4; ++j) o.d2T[j] = wd2<M, W>(p, v, j);
  // mixed derivatives (commuted, D-7)
  ldwin<W>(S + XF_G22 * Gm::FSZ + base, st, v);  // D_d g22
#pragma unroll
  for (int j = 0; j < 4; ++j) o.mixA[j] = wd1<M, W>(p, v, j);
  if (DIR == 0) {
    ldwin<W>(S + XF_G02 * Gm::FSZ + base, st, v);  // D_x g02 = D_z g00
#pragma unroll
    for (int j = 0; j < 4; ++j) o.mixB[j] = wd1<M, W>(p, v, j);
  } else {
    ldwin<W>(S + XF_G12 * Gm::FSZ + base, st, v);  // D_y g12 = D_z g11
#pragma unroll
    for (int j = 0; j < 4; ++j) o.mixB[j] = wd1<M, W>(p, v, j);
    ldwin<W>(E0 + ebase, XYGeom<M>::TP, v);  // D_y g00
#pragma unroll
    for (int j = 0; j < 4; ++j) o.mixC[j] = wd1<M, W>(p, v, j);
    ldwin<W>(E1 + ebase, XYGeom<M>::TP, v);  // D_y g10 = D_x g11
#pragma unroll
    for (int j = 0; j < 4; ++j) o.mixD[j] = wd1<M, W>(p, v, j);
  }
}

// Conservative group, one direction d: returns the d-part of
//   -[ D_d F_id + 1/2 u_d D_d s + (mass) ]  for the five equations, where
//   F_id = 1/2 m_i u_d + delta_id p,  G_d = (1/2 e + p) u_d   (skew halves + pressure)
template <int M, int DIR>
__device__ __forceinline__ void conservative_dir(const KParams &p, const double *S, int base,
                                                 int st, double (&R)[5][4]) {
  using Gm = XYGeom<M>;
  constexpr int W = Gm::W;
  double ud[W], pw[W], v[W], t[W];
  {
    double r[W];
    ldwin<W>(S + XF_R * Gm::FSZ + base, st, r);
    ldwin<W>(S + (XF_M0 + DIR) * Gm::FSZ + base, st, t);
#pragma unroll
    for (int k = 0; k < W; ++k) ud[k] = __dmul_rn(t[k], r[k]);
    // mass: -1/2 (D_d m_d + u_d D_d rho)
#pragma unroll
    for (int j = 0; j < 4; ++j) R[0][j] = -0.5 * wd1<M, W>(p, t, j);
  }
  ldwin<W>(S + XF_RHO * Gm::FSZ + base, st, v);
#pragma unroll
  for (int j = 0; j < 4; ++j) R[0][j] = fma(-0.5 * ud[j + M], wd1<M, W>(p, v, j), R[0][j]);
  ldwin<W>(S + XF_P * Gm::FSZ + base, st, pw);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ldwin<W>(S + (XF_M0 + i) * Gm::FSZ + base, st, v);
#pragma unroll
    for (int k = 0; k < W; ++k)
      t[k] = (i == DIR) ? fma(0.5 * v[k], ud[k], pw[k]) : __dmul_rn(0.5 * v[k], ud[k]);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      R[1 + i][j] = -fma(0.5 * ud[j + M], wd1<M, W>(p, v, j), wd1<M, W>(p, t, j));
  }
  ldwin<W>(S + XF_E * Gm::FSZ + base, st, v);
#pragma unroll
  for (int k = 0; k < W; ++k) t[k] = __dmul_rn(fma(0.5, v[k], pw[k]), ud[k]);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    R[4][j] = -fma(0.5 * ud[j + M], wd1<M, W>(p, v, j), wd1<M, W>(p, t, j));
}

template <int M>
__global__ void __launch_bounds__(XY_THREADS, 1)
    xypass_kernel(const KParams p, const double *__restrict__ q, double *__restrict__ qout,
                  double *__restrict__ w, const double *__restrict__ gz,
                  double *__restrict__ rout,
                  unsigned int *__restrict__ flag, int z_begin) {
  using Gm = XYGeom<M>;
  constexpr int HX = Gm::HX, HY = Gm::HY, PX = Gm::PX, FSZ = Gm::FSZ, NPT = Gm::NPT;
  extern __shared__ double S[];
  double *E0 = S + Gm::OFF_E0, *E1 = S + Gm::OFF_E1;
  double *XA = S + Gm::OFF_XA, *XB = S + Gm::OFF_XB;
  const int tid = threadIdx.x;
  const int z = z_begin + blockIdx.z;
  const int x0 = blockIdx.x * XY_TX, y0 = blockIdx.y * XY_TY;
  const size_t FS = (size_t)p.nx * p.ny;
  const double *qp = q + qplane(p, z);
  const double *gp = gz + (size_t)z * 3 * FS;

  // ---- prefetch the epilogue operand W' (= A W + dt Rz, from the z-pass)
  //      asynchronously so that its latency hides behind phases X and Y
  double *PF = S + Gm::OFF_PF;
  for (int lin = tid; lin < XY_TX * XY_TY; lin += XY_THREADS) {
    const int ty = lin / XY_TX, tx = lin - ty * XY_TX;
    const int x = x0 + tx, y = y0 + ty;
    if (x < p.nx && y < p.ny) {
      const size_t o = (size_t)z * 5 * FS + (size_t)y * p.nx + x;
#pragma unroll
      for (int f = 0; f < 5; ++f)
        cp_async8(PF + f * XY_TX * XY_TY + lin,
                  (p.two_reg ? qout + qplane(p, 0) : w) + o + f * FS);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");

  // ---- stage the tile + halo: conservative state, p, 1/rho, g_i2.  All global
  //      loads of a thread are issued before the first shared store (MLP).
  auto stage_point = [&](int s, const double *v) {
    const double rho = v[0], m0 = v[1], m1 = v[2], m2 = v[3], e = v[4];
    const double r = 1.0 / rho;
    S[XF_RHO * FSZ + s] = rho;
    S[XF_M0 * FSZ + s] = m0;
    S[XF_M1 * FSZ + s] = m1;
    S[XF_M2 * FSZ + s] = m2;
    S[XF_E * FSZ + s] = e;
    S[XF_P * FSZ + s] = p.gm1 * (e - 0.5 * r * (m0 * m0 + m1 * m1 + m2 * m2));
    S[XF_R * FSZ + s] = r;
    S[XF_G02 * FSZ + s] = v[5];
    S[XF_G12 * FSZ + s] = v[6];
    S[XF_G22 * FSZ + s] = v[7];
  };
  bool paired = false;
  if constexpr (M % 2 == 0) paired = (p.nx % 2 == 0) && !(p.sym[0] | p.sym[1]);
  if (paired) {
    // m and nx even: x0 - m + hx is even for even hx and never straddles the
    // periodic seam, so two neighbouring columns come in one 16-byte load
    constexpr int NP2 = HX / 2 * HY;
    constexpr int NIT = (NP2 + XY_THREADS - 1) / XY_THREADS;
    double2 raw[NIT][8];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int idx = tid + it * XY_THREADS;
      if (idx < NP2) {
        const int hy = idx / (HX / 2), hx = 2 * (idx - hy * (HX / 2));
        const int x = wrapi(x0 - M + hx, p.nx), y = wrapi(y0 - M + hy, p.ny);
        const size_t off = (size_t)y * p.nx + x;
#pragma unroll
        for (int f = 0; f < 5; ++f)
          raw[it][f] = __ldg(reinterpret_cast<const double2 *>(qp + f * FS + off));
#pragma unroll
        for (int f = 0; f < 3; ++f)
          raw[it][5 + f] = __ldg(reinterpret_cast<const double2 *>(gp + f * FS + off));
      }
    }
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int idx = tid + it * XY_THREADS;
      if (idx < NP2) {
        const int hy = idx / (HX / 2), hx = 2 * (idx - hy * (HX / 2));
        double a[8], b[8];
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          a[f] = raw[it][f].x;
          b[f] = raw[it][f].y;
        }
        stage_point(hy * PX + hx, a);
        stage_point(hy * PX + hx + 1, b);
      }
    }
  } else {
    constexpr int NIT = (HX * HY + XY_THREADS - 1) / XY_THREADS;
    double raw[NIT][8];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int idx = tid + it * XY_THREADS;
      if (idx < HX * HY) {
        const int hy = idx / HX, hx = idx - hy * HX;
        int fx, fy;
        const int x = bmap(x0 - M + hx, p.nx, p.sym[0], fx),
                  y = bmap(y0 - M + hy, p.ny, p.sym[1], fy);
        const size_t off = (size_t)y * p.nx + x;
#pragma unroll
        for (int f = 0; f < 5; ++f) raw[it][f] = __ldg(qp + f * FS + off);
#pragma unroll
        for (int f = 0; f < 3; ++f) raw[it][5 + f] = __ldg(gp + f * FS + off);
        // symmetry boundaries: odd components under a mirror change sign
        if (fx) { raw[it][1] = -raw[it][1]; raw[it][5] = -raw[it][5]; }
        if (fy) { raw[it][2] = -raw[it][2]; raw[it][6] = -raw[it][6]; }
      }
    }
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int idx = tid + it * XY_THREADS;
      if (idx < HX * HY) {
        const int hy = idx / HX, hx = idx - hy * HX;
        stage_point(hy * PX + hx, raw[it]);
      }
    }
  }
  __syncthreads();

  const int grp = tid >> 7;  // 0: velocity group A, 1: conservative group B (warp-uniform)
  const int q7 = tid & 127;
  // ---- phase X: thread -> (row, 4-wide x segment); lanes 0-15 / 16-31 = 16 rows
  {
    const int row = q7 & 15, seg = q7 >> 4;
    const int hy = row + M;
    const int base = hy * PX + seg * XY_RX;  // window start (halo coords)
    const int pt0 = row * Gm::TP + seg * XY_RX;
    if (grp == 0) {
      VelResult<M, 0> o;
      velocity_dir<M, 0>(p, S, base, 1, E0, E1, 0, o);
      const double third = 1.0 / 3.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        // x-parts of V_i: V0 += nu (4/3 D00 u0 + 1/3 D0 g22); V1 += nu D00 u1;
        // V2 += nu (D00 u2 + 1/3 D0 g02)
        const double V0 = p.nu * (o.d2u[0][j] + third * (o.d2u[0][j] + o.mixA[j]));
        const double V1 = p.nu * o.d2u[1][j];
        const double V2 = p.nu * (o.d2u[2][j] + third * o.mixB[j]);
        XA[0 * NPT + pt0 + j] = V0;
        XA[1 * NPT + pt0 + j] = V1;
        XA[2 * NPT + pt0 + j] = V2;
        XA[3 * NPT + pt0 + j] =
            fma(p.kappa, o.d2T[j], o.uc[0][j] * V0 + o.uc[1][j] * V1 + o.uc[2][j] * V2);
        XA[4 * NPT + pt0 + j] = o.g[2][j];  // g20
        E0[hy * Gm::TP + seg * XY_RX + j] = o.g[0][j];  // g00
        E1[hy * Gm::TP + seg * XY_RX + j] = o.g[1][j];  // g10
      }
    } else {
      double R[5][4];
      conservative_dir<M, 0>(p, S, base, 1, R);
#pragma unroll
      for (int f = 0; f < 5; ++f)
#pragma unroll
        for (int j = 0; j < 4; ++j) XB[f * NPT + pt0 + j] = R[f][j];
    }
  }
  // ---- g00, g10 on the 2m halo rows (inner derivatives of D_y g00, D_y g10)
  for (int task = tid; task < 2 * M * (XY_TX / XY_RX); task += XY_THREADS) {
    const int rr = task % (2 * M), seg = task / (2 * M);
    const int hy = rr < M ? rr : rr + XY_TY;
    const int base = hy * PX + seg * XY_RX;
    constexpr int W = Gm::W;
    double r[W], v[W], t[W];
    ldwin<W>(S + XF_R * FSZ + base, 1, r);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      ldwin<W>(S + (XF_M0 + i) * FSZ + base, 1, t);
#pragma unroll
      for (int k = 0; k < W; ++k) v[k] = __dmul_rn(t[k], r[k]);
      double *Ei = i == 0 ? E0 : E1;
#pragma unroll
      for (int j = 0; j < 4; ++j) Ei[hy * Gm::TP + seg * XY_RX + j] = wd1<M, W>(p, v, j);
    }
  }
  __syncthreads();

  // ---- phase Y: thread -> (column, 4-tall y segment); lanes = 32 consecutive columns
  {
    const int col = q7 & 31, seg = q7 >> 5;
    const int base = (seg * XY_RY) * PX + col + M;
    const int ebase = (seg * XY_RY) * Gm::TP + col;
    if (grp == 0) {
      VelResult<M, 1> o;
      velocity_dir<M, 1>(p, S, base, PX, E0, E1, ebase, o);
      const double third = 1.0 / 3.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ty = seg * XY_RY + j;
        const int pt = ty * Gm::TP + col;
        const int c = (ty + M) * PX + col + M;
        const double g00 = E0[(ty + M) * Gm::TP + col], g10 = E1[(ty + M) * Gm::TP + col];
        const double g20 = XA[4 * NPT + pt];
        const double g01 = o.g[0][j], g11 = o.g[1][j], g21 = o.g[2][j];
        const double g02 = S[XF_G02 * FSZ + c], g12 = S[XF_G12 * FSZ + c],
                     g22 = S[XF_G22 * FSZ + c];
        // y-parts of V_i: V0 += nu (D11 u0 + 1/3 D1 g10);
        // V1 += nu (4/3 D11 u1 + 1/3 (D1 g00 + D1 g22)); V2 += nu (D11 u2 + 1/3 D1 g12)
        const double V0y = p.nu * (o.d2u[0][j] + third * o.mixD[j]);
        const double V1y = p.nu * (o.d2u[1][j] + third * (o.d2u[1][j] + o.mixC[j] + o.mixA[j]));
        const double V2y = p.nu * (o.d2u[2][j] + third * o.mixB[j]);
        const double V0 = XA[0 * NPT + pt] + V0y, V1 = XA[1 * NPT + pt] + V1y,
                     V2 = XA[2 * NPT + pt] + V2y;
        const double thxy = g00 + g11, th = thxy + g22;
        const double s01 = g01 + g10, s02 = g02 + g20, s12 = g12 + g21;
        // tau_ij du_i/dx_j (eq. 8)
        const double Phi = p.nu * (2.0 * (g00 * g00 + g11 * g11 + g22 * g22) + s01 * s01 +
                                   s02 * s02 + s12 * s12 - (2.0 / 3.0) * th * th);
        const double u0 = o.uc[0][j], u1 = o.uc[1][j], u2 = o.uc[2][j];
        const double ex = XA[3 * NPT + pt];  // kappa D00 T + u_i V_i^x (phase X)
        // dilatation halves of the skew terms, -1/2 s (g00 + g11)
        XA[0 * NPT + pt] = -0.5 * S[XF_RHO * FSZ + c] * thxy;
        XA[1 * NPT + pt] = fma(-0.5 * S[XF_M0 * FSZ + c], thxy, V0);
        XA[2 * NPT + pt] = fma(-0.5 * S[XF_M1 * FSZ + c], thxy, V1);
        XA[3 * NPT + pt] = fma(-0.5 * S[XF_M2 * FSZ + c], thxy, V2);
        XA[4 * NPT + pt] = fma(-0.5 * S[XF_E * FSZ + c], thxy,
                               ex + fma(p.kappa, o.d2T[j], Phi) +
                                   (u0 * V0y + u1 * V1y + u2 * V2y));
      }
    } else {
      double R[5][4];
      conservative_dir<M, 1>(p, S, base, PX, R);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int pt = (seg * XY_RY + j) * Gm::TP + col;
#pragma unroll
        for (int f = 0; f < 5; ++f) XB[f * NPT + pt] += R[f][j];
      }
    }
  }
  __syncthreads();

  // ---- epilogue: W <- W' + dt R_xy ; Q' <- Q + B W   (coalesced rows; residual mode:
  //      A = 0, dt = 1 so that W' = Rz and R = W' + R_xy)
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  bool bad = false;
  for (int lin = tid; lin < XY_TX * XY_TY; lin += XY_THREADS) {
    const int ty = lin / XY_TX, tx = lin - ty * XY_TX;
    const int pt = ty * Gm::TP + tx;
    const int x = x0 + tx, y = y0 + ty;
    if (x >= p.nx || y >= p.ny) continue;
    const int c = (ty + M) * PX + tx + M;
    const size_t o = (size_t)z * 5 * FS + (size_t)y * p.nx + x;
    double *qo = qout ? qout + qplane(p, z) + (size_t)y * p.nx + x : nullptr;
    const int fidx[5] = {XF_RHO, XF_M0, XF_M1, XF_M2, XF_E};
#pragma unroll
    for (int f = 0; f < 5; ++f) {
      const double wn =
          fma(p.dt, XA[f * NPT + pt] + XB[f * NPT + pt], PF[f * XY_TX * XY_TY + lin]);
      if (rout) {
        rout[o + f * FS] = wn;
        continue;
      }
      double qb = S[fidx[f] * FSZ + c];
      if (p.two_reg) {  // W' came from qout's interior planes; w holds Q_old
        if (p.read_w) qb = w[o + f * FS];
        if (p.write_w) w[o + f * FS] = fma(p.beta, wn, qb);
      } else if (p.write_w) {
        w[o + f * FS] = wn;
      }
      const double qn = fma(p.B, wn, qb);
      qo[f * FS] = qn;
      bad |= !isfinite(qn);
    }
  }
  if (bad) atomicOr(flag, 1u);
}
