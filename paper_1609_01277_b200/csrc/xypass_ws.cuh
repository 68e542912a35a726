namespace ws {
// xy-pass (included by kernels.cu inside namespace osbli::{anon}).
//
// A CTA owns a 32 x 16 tile of the xy-plane and marches through a segment of
// z-planes (one CTA per SM), warp-specialised:
//   producers (warps 8-11, setmaxnreg 40): stream plane z+1 into the other plane
//     buffer -- TMA tensor boxes (one 5-field Q box, g22, g02, g12) completing on
//     the buffer's mbarrier where the tile's halo does not wrap, a cp.async gather
//     (periodic wrap or mirror in x, y) elsewhere -- and prefetch its low-storage
//     register W' (= A W + dt Rz from the z-pass) into L2;
//   group A (velocity, 4 warps, setmaxnreg 232): p and 1/rho of every staged
//     point (formulas P:127, EOS P:259-266), velocity gradients, viscous
//     Laplacians, mixed derivatives (commuted: D-7), dissipation;
//   group B (conservative, 4 warps): skew-symmetric advection and fluxes
//     (P:271-274), heat flux, and the stage update of its points,
//     W <- W' + dt R_xy, Q' <- Q + B W.
// Per plane, shared memory holds on the tile plus an m-wide halo (one extra
// column on each side at odd m): rho, m_i, e,
// g22 (double-buffered plane buffers), g02 on the tile rows (x-halo), g12 on
// the tile columns (y-halo); p, 1/rho; g00, g10 extended over the y-halo; the
// groups' x-partials XA, XB.  u_i = m_i r and T = gamma M^2 p r are formed in
// register windows of RX = RY = 4 consecutive outputs ((4 + 2m) shared loads
// for 4 outputs).  Per plane: phase X (thread = 4-wide row segment) and phase Y
// (thread = 4-tall column segment) in each group.  The groups run decoupled, up
// to a plane apart, meeting only where data passes (named barriers, see the
// consumer loop); group A computes the next plane's p, 1/rho while group B
// finishes its epilogue.
constexpr int XY_TX = 32;
constexpr int XY_TY = 16;
constexpr int XY_RX = 4;
constexpr int XY_RY = 4;
constexpr int XY_THREADS = 256;          // consumer threads
#ifndef OSBLI_XY_PRODUCERS
#define OSBLI_XY_PRODUCERS 4
#endif
constexpr int XY_PROD = 32 * OSBLI_XY_PRODUCERS;  // producer threads
constexpr int XY_CTA = XY_THREADS + XY_PROD;
// register split (setmaxnreg): 128 producer threads x PROD + 256 consumers x CONS <= 64K
#ifndef OSBLI_XY_PROD_REGS
#define OSBLI_XY_PROD_REGS 40
#endif
#ifndef OSBLI_XY_CONS_REGS
#define OSBLI_XY_CONS_REGS 232
#endif
constexpr int XY_PROD_REGS = OSBLI_XY_PROD_REGS;
constexpr int XY_CONS_REGS = OSBLI_XY_CONS_REGS;
// named barriers: 2 + b = buffer b full (producers -> group A); 4 + b = buffer b
// empty (consumers -> producers); 7 = producers only; 1, 6, 8, 9, 10: consumers
// (see the consumer loop)
__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
#ifndef OSBLI_XY_SMSP_SPLIT
#define OSBLI_XY_SMSP_SPLIT 1
#endif
#ifndef OSBLI_XY_FORM_UNROLL
#define OSBLI_XY_FORM_UNROLL 1
#endif
// experiments only (results wrong): skip the plane staging after the first two
// planes / skip the formulas after the first plane, to bound what each costs
#ifndef OSBLI_XY_EXP_NOSTAGE
#define OSBLI_XY_EXP_NOSTAGE 0
#endif
#ifndef OSBLI_XY_TMA_SYM  // A/B knob: TMA staging also with x/y symmetry
#define OSBLI_XY_TMA_SYM 0
#endif
#ifndef OSBLI_XY_EXP_NOFORM
#define OSBLI_XY_EXP_NOFORM 0
#endif
// Work balance between the consumer groups (group A's chain p, 1/rho -> phase X
// -> halo rows -> phase Y is the critical path): the x
// mixed-derivative viscous parts nu/3 D_x g22, nu/3 D_x g02 are computed by group
// B in its phase X (default; -1.1 % xy-pass at o12, -1.9 % at o8).  Moving the y
// ones as well (MIXY_B) overshoots: B becomes the critical path (+2 %).
#ifndef OSBLI_XY_MIXX_B
#define OSBLI_XY_MIXX_B 1
#endif
constexpr bool XY_MIXX_B = OSBLI_XY_MIXX_B != 0;
// OSBLI_XY_MIXY_B: bit 0 = nu/3 D_y g22 (momentum y), bit 1 = nu/3 D_y g12 (momentum z)
#ifndef OSBLI_XY_MIXY_B
#define OSBLI_XY_MIXY_B 0
#endif
constexpr int XY_MIXY_B = OSBLI_XY_MIXY_B;
// z-planes per CTA: 16 at orders 2, 4 (the pipeline fill of a segment weighs more
// against the short stencils: -3 % xy-pass at o4) and 12 (-0.5 %), 8 at 6-10 (16
// is +0.3 % at o8)
#ifndef OSBLI_XY_SEG
template <int M>
constexpr int xy_seg() { return (M <= 2 || M >= 6) ? 16 : 8; }
#else
template <int M>
constexpr int xy_seg() { return OSBLI_XY_SEG; }
#endif
// full-halo fields of a plane buffer (S) and of the per-plane formula arrays (PR)
enum { XF_RHO = 0, XF_M0, XF_M1, XF_M2, XF_E };
enum { XP_P = 0, XP_R = 1 };

template <int M>
struct XYGeom {
  // Staged columns start at the even x0 - M - XO: for odd m one extra column on
  // each side (XO = 1), so that every halo row is copied in 16-byte pairs and the
  // x-windows are read with 16-byte loads at every order (an odd-m window starts
  // one double past a pair boundary: m + 3 pairs, the outer two values unused).
  // A pitch of 2 mod 4 doubles keeps those loads conflict-free for the
  // row-per-lane access of phase X (8 lanes of a quarter warp on 8 rows hit 8
  // distinct 16-byte bank groups).  XC = staged column of the tile's x = 0.
  static constexpr int XO = M % 2;
  static constexpr int XC = M + XO;
  static constexpr int HX = XY_TX + 2 * XC;  // staged columns (even)
  static constexpr bool PAIRS = true;
  // x-window load mode (ldwin): 1 = pairs from an aligned start, 2 = pairs from one before
  static constexpr int XW = XO ? 2 : 1;
  static constexpr int PX = (HX % 4 == 0) ? HX + 2 : HX;
  static constexpr int HY = XY_TY + 2 * M;
  static constexpr int FSZ = HY * PX;       // one full-halo field
  static constexpr int TP = XY_TX + 1;      // odd row pitch of tile-column arrays
  static constexpr int NPT = TP * XY_TY;    // tile points (padded)
  static constexpr int EXT = TP * HY;       // tile columns x (tile + y-halo) rows
  static constexpr int W = 4 + 2 * M;       // window length (RX = RY = 4)
  static constexpr int GP = XY_TX;          // pitch of the g12 strip (column-per-lane access)
  // plane buffer (doubles): rho, m_i, e [5][HY][PX] | g22 [HY][PX] | g02 [TY][PX] (tile
  // rows) | g12 [HY][GP] (tile cols); each part starts on a 128-byte boundary (a TMA
  // destination: the first is one 5-field box, the others one box each)
  static constexpr int al16(int n) { return (n + 15) / 16 * 16; }
  static constexpr int PB_G22 = al16(5 * FSZ);
  static constexpr int PB_G02 = al16(PB_G22 + FSZ);
  static constexpr int PB_G12 = al16(PB_G02 + XY_TY * PX);
  static constexpr int PBSZ = al16(PB_G12 + HY * GP);
  // layout: PB[2] | PR (p, r) | E0 | E1 | XA[5] | XB[5] | XT
  static constexpr int OFF_PR = 2 * PBSZ;
  static constexpr int OFF_E0 = OFF_PR + 2 * FSZ;   // [HY][TP]   g00 (y-extended)
  static constexpr int OFF_E1 = OFF_E0 + EXT;       // [HY][TP]   g10 (y-extended)
  static constexpr int OFF_XA = OFF_E1 + EXT;       // 5 x [TY][TP]
  static constexpr int OFF_XB = OFF_XA + 5 * NPT;   // 5 x [TY][TP]
  static constexpr int OFF_XT = OFF_XB + 5 * NPT;   // [TY][TP] D_x T (equation variants)
  static constexpr int OFF_DG = OFF_XT + NPT;       // [4 warps][3] fused diagnostics partials
  static constexpr int OFF_BAR = OFF_DG + 16;       // 2 TMA mbarriers (plane buffers)
  static constexpr int TOTAL = OFF_BAR + 2;
  // producer gather tables (ints): global x of each halo column, y * nx of each halo row
  static constexpr int TAB_INTS = HX + HY;
  static constexpr int BYTES = TOTAL * (int)sizeof(double) + TAB_INTS * (int)sizeof(int);
};

template <int M>
constexpr int xy_smem_bytes() {
  return XYGeom<M>::BYTES;
}

// Window elements that are products are rounded explicitly (__dmul_rn): the
// compiler may otherwise contract a product into the stencil difference
// (f+ - f-) differently for different taps, and a uniform state would no
// longer cancel exactly (SURVEY §8(c) equilibrium pin).
// window of W values starting at base, stride `st` (doubles).  PAIR = 1:
// consecutive values (st = 1) from a 16-byte aligned base, read as W/2 16-byte
// loads; PAIR = 2: base is one double past a 16-byte boundary, read as W/2 + 1
// 16-byte loads from base - 1 (first and last values unused)
template <int W, int PAIR = 0>
__device__ __forceinline__ void ldwin(const double *base, int st, double (&v)[W]) {
  static_assert(PAIR == 0 || W % 2 == 0, "pair windows need an even length");
  if (PAIR == 1) {
#pragma unroll
    for (int k = 0; k < W / 2; ++k) {
      const double2 t = reinterpret_cast<const double2 *>(base)[k];
      v[2 * k] = t.x;
      v[2 * k + 1] = t.y;
    }
  } else if (PAIR == 2) {
#pragma unroll
    for (int k = 0; k <= W / 2; ++k) {
      const double2 t = reinterpret_cast<const double2 *>(base - 1)[k];
      if (k > 0) v[2 * k - 1] = t.x;
      if (k < W / 2) v[2 * k] = t.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = base[k * st];
  }
}

template <int M, int W>
__device__ __forceinline__ double wd1(const KParams &p, const double (&v)[W], int j) {
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

// second derivative, exactly zero on a constant window: sum b_k ((f+ + f-) - 2 f)  (D-22)
template <int M, int W>
__device__ __forceinline__ double wd2(const KParams &p, const double (&v)[W], int j) {
#if OSBLI_D2_SBP
  // in first differences (summation by parts): sum_l C_l (d_{c+l} - d_{c-1-l}),
  // d_i = v[i+1] - v[i] shared by the outputs of the window; exact zero on constants
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

// Velocity group, one direction (DIR 0 = x: phase X, DIR 1 = y: phase Y):
// velocity gradients g_id, second derivatives of u_i and T along d, and the
// mixed derivatives needed along d (commuted, D-7).
template <int M>
struct VelResult {
  double g[3][4], d2u[3][4], d2T[4], mixA[4], mixB[4], mixC[4], mixD[4], uc[3][4];
  double d1T[4], Tc[4];  // D_d T and T at the outputs (equation variants only)
};

// TW: also the temperature stencils (heat flux, and D_d T, T for the variants);
// without them the heat flux is group B's (conservative_dir<.., HEAT = true>)
// NOMIX: bit 0 skips D_d g22 (mixA), bit 1 the second mixed stencil (mixB)
template <int M, int DIR, bool TW, int NOMIX = 0>
__device__ __forceinline__ void velocity_dir(const KParams &p, const double *S, const double *PR,
                                             int base, int st, const double *gmix, int gst,
                                             const double *E0, const double *E1, int ebase,
                                             VelResult<M> &o) {
  using Gm = XYGeom<M>;
  constexpr int W = Gm::W;
  constexpr int PW = DIR == 0 ? Gm::XW : 0;  // x-windows: 16-byte loads
  double r[W], v[W], t[W];
  ldwin<W, PW>(PR + XP_R * Gm::FSZ + base, st, r);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ldwin<W, PW>(S + (XF_M0 + i) * Gm::FSZ + base, st, t);
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = __dmul_rn(t[k], r[k]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      o.g[i][j] = wd1<M, W>(p, v, j);
      o.d2u[i][j] = wd2<M, W>(p, v, j);
      o.uc[i][j] = v[j + M];
    }
  }
  if (TW) {
    ldwin<W, PW>(PR + XP_P * Gm::FSZ + base, st, t);
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = __dmul_rn(__dmul_rn(p.gM2, t[k]), r[k]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      o.d2T[j] = wd2<M, W>(p, v, j);
      o.d1T[j] = wd1<M, W>(p, v, j);
      o.Tc[j] = v[j + M];
    }
  }
  if (!(NOMIX & 1)) {
    ldwin<W, PW>(S + Gm::PB_G22 + base, st, v);  // D_d g22
#pragma unroll
    for (int j = 0; j < 4; ++j) o.mixA[j] = wd1<M, W>(p, v, j);
  }
  if (!(NOMIX & 2)) {
    ldwin<W, PW>(gmix, gst, v);  // DIR 0: D_x g02 = D_z g00 ; DIR 1: D_y g12 = D_z g11
#pragma unroll
    for (int j = 0; j < 4; ++j) o.mixB[j] = wd1<M, W>(p, v, j);
  }
  if (DIR == 1) {
    ldwin<W>(E0 + ebase, Gm::TP, v);  // D_y g00
#pragma unroll
    for (int j = 0; j < 4; ++j) o.mixC[j] = wd1<M, W>(p, v, j);
    ldwin<W>(E1 + ebase, Gm::TP, v);  // D_y g10 = D_x g11
#pragma unroll
    for (int j = 0; j < 4; ++j) o.mixD[j] = wd1<M, W>(p, v, j);
  }
}

// Conservative group, one direction d: the d-part of
//   -[ D_d F_id + 1/2 u_d D_d s ]  (and mass: -1/2 (D_d m_d + u_d D_d rho)),
//   F_id = 1/2 m_i u_d + delta_id p,  G_d = (1/2 e + p) u_d   (skew halves + pressure)
// HEAT: also the d-part of the heat flux, kappa D_dd T, from the
// p and 1/rho windows this group has loaded anyway
template <int M, int DIR, bool HEAT>
__device__ __forceinline__ void conservative_dir(const KParams &p, const double *S,
                                                 const double *PR, int base, int st,
                                                 double (&R)[5][4]) {
  using Gm = XYGeom<M>;
  constexpr int W = Gm::W;
  constexpr int PW = DIR == 0 ? Gm::XW : 0;  // x-windows: 16-byte loads
  // hu = u_d / 2 (exact halving): every skew half and flux below uses it, so the
  // factors 1/2 cost nothing per term; (1/2 e + p) u_d = (e + 2p) hu exactly
  double hu[W], pw[W], v[W], t[W];
  double heat[4];
  {
    double r[W];
    ldwin<W, PW>(PR + XP_R * Gm::FSZ + base, st, r);
    ldwin<W, PW>(S + (XF_M0 + DIR) * Gm::FSZ + base, st, t);
#pragma unroll
    for (int k = 0; k < W; ++k) hu[k] = 0.5 * __dmul_rn(t[k], r[k]);
    ldwin<W, PW>(PR + XP_P * Gm::FSZ + base, st, pw);
    if (HEAT) {
#pragma unroll
      for (int k = 0; k < W; ++k) v[k] = __dmul_rn(__dmul_rn(p.gM2, pw[k]), r[k]);
#pragma unroll
      for (int j = 0; j < 4; ++j) heat[j] = p.kappa * wd2<M, W>(p, v, j);
    }
  }
  // D_d m_d serves the mass equation and the skew half of momentum d: one stencil
  // of the m_d window for both (the variants' instantiation, HEAT = false, keeps
  // the two separate: it is at its register limit)
  if (!HEAT) {
#pragma unroll
    for (int j = 0; j < 4; ++j) R[0][j] = -0.5 * wd1<M, W>(p, t, j);
  } else {
    double dmd[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) dmd[j] = wd1<M, W>(p, t, j);
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = fma(t[k], hu[k], pw[k]);  // F_dd = 1/2 m_d u_d + p
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      R[0][j] = -0.5 * dmd[j];
      R[1 + DIR][j] = -fma(hu[j + M], dmd[j], wd1<M, W>(p, v, j));
    }
  }
  ldwin<W, PW>(S + XF_RHO * Gm::FSZ + base, st, v);
#pragma unroll
  for (int j = 0; j < 4; ++j) R[0][j] = fma(-hu[j + M], wd1<M, W>(p, v, j), R[0][j]);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (HEAT && i == DIR) continue;
    ldwin<W, PW>(S + (XF_M0 + i) * Gm::FSZ + base, st, v);
#pragma unroll
    for (int k = 0; k < W; ++k)
      t[k] = (i == DIR) ? fma(v[k], hu[k], pw[k]) : __dmul_rn(v[k], hu[k]);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      R[1 + i][j] = -fma(hu[j + M], wd1<M, W>(p, v, j), wd1<M, W>(p, t, j));
  }
  ldwin<W, PW>(S + XF_E * Gm::FSZ + base, st, v);
#pragma unroll
  for (int k = 0; k < W; ++k) t[k] = __dmul_rn(fma(2.0, pw[k], v[k]), hu[k]);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    R[4][j] = -fma(hu[j + M], wd1<M, W>(p, v, j), wd1<M, W>(p, t, j));
  if (HEAT) {
#pragma unroll
    for (int j = 0; j < 4; ++j) R[4][j] += heat[j];
  }
}

// 16-byte asynchronous global -> shared copy (L2 only)
__device__ __forceinline__ void cp_async16(double *smem, const double *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}

// Gather tables of a CTA (plane independent): cx[hx] = global x of halo column hx,
// ry[hy] = (global y of halo row hy) * nx, through the periodic wrap or the mirror.
template <int M, bool SYM>
__device__ __forceinline__ void xy_tables(const KParams &p, int *cx, int *ry, int x0, int y0,
                                          int tid, int nthr) {
  using Gm = XYGeom<M>;
  for (int i = tid; i < Gm::HX + Gm::HY; i += nthr) {
    int f;
    if (i < Gm::HX) cx[i] = bmap_t<SYM>(x0 - Gm::XC + i, p.nx, p.sym[0], f);
    else ry[i - Gm::HX] = bmap_t<SYM>(y0 - M + i - Gm::HX, p.ny, p.sym[1], f) * p.nx;
  }
}

// issue the asynchronous copies of plane z's operands into plane buffer PB.
// pairs: 16-byte copies of x-pairs (even m, even nx, periodic x: a pair never
// straddles the wrap, since every halo row starts at an even x)
template <int M>
__device__ __forceinline__ void xy_issue_plane(const KParams &p, const double *__restrict__ q,
                                               const double *__restrict__ gz, double *PB, int z,
                                               const int *cx, const int *ry, int tid, int nthr,
                                               bool pairs) {
  using Gm = XYGeom<M>;
  constexpr int HX = Gm::HX, HY = Gm::HY, PX = Gm::PX, FSZ = Gm::FSZ, GP = Gm::GP;
  const size_t FS = (size_t)p.nx * p.ny;
  const double *qp = q + qplane(p, z);
  const double *gp = gz + (size_t)z * 3 * FS;
  if (Gm::PAIRS && pairs) {
    constexpr int H2 = HX / 2, T2 = XY_TX / 2;
#pragma unroll 1
    for (int idx = tid; idx < HY * H2; idx += nthr) {
      const int hy = idx / H2, hx = 2 * (idx - hy * H2);
      const int off = ry[hy] + cx[hx];
      double *d = PB + hy * PX + hx;
      if (OSBLI_DEBUG_CHECKS && !(dbg_in(p, (qp - q) + 4 * FS + off + 1, qbuf_len(p)) &&
                                  dbg_in(p, (qp - q) + off, qbuf_len(p)) &&
                                  dbg_in(p, (gp - gz) + 2 * FS + off + 1, 3LL * p.nz * FS)))
        continue;
#pragma unroll
      for (int f = 0; f < 5; ++f) cp_async16(d + f * FSZ, qp + f * FS + off);
      cp_async16(PB + Gm::PB_G22 + hy * PX + hx, gp + 2 * FS + off);
    }
#pragma unroll 1
    for (int idx = tid; idx < XY_TY * H2; idx += nthr) {
      const int ty = idx / H2, hx = 2 * (idx - ty * H2);
      cp_async16(PB + Gm::PB_G02 + ty * PX + hx, gp + ry[ty + M] + cx[hx]);
    }
#pragma unroll 1
    for (int idx = tid; idx < HY * T2; idx += nthr) {
      const int hy = idx / T2, tx = 2 * (idx - hy * T2);
      cp_async16(PB + Gm::PB_G12 + hy * GP + tx, gp + FS + ry[hy] + cx[tx + Gm::XC]);
    }
  } else {
#pragma unroll 1
    for (int idx = tid; idx < HY * HX; idx += nthr) {
      const int hy = idx / HX, hx = idx - hy * HX;
      const int off = ry[hy] + cx[hx];
      double *d = PB + hy * PX + hx;
      if (OSBLI_DEBUG_CHECKS && !(dbg_in(p, (qp - q) + 4 * FS + off, qbuf_len(p)) &&
                                  dbg_in(p, (qp - q) + off, qbuf_len(p)) &&
                                  dbg_in(p, (gp - gz) + 2 * FS + off, 3LL * p.nz * FS)))
        continue;
#pragma unroll
      for (int f = 0; f < 5; ++f) cp_async8(d + f * FSZ, qp + f * FS + off);
      cp_async8(PB + Gm::PB_G22 + hy * PX + hx, gp + 2 * FS + off);
    }
#pragma unroll 1
    for (int idx = tid; idx < XY_TY * HX; idx += nthr) {
      const int ty = idx / HX, hx = idx - ty * HX;
      cp_async8(PB + Gm::PB_G02 + ty * PX + hx, gp + ry[ty + M] + cx[hx]);
    }
#pragma unroll 1
    for (int idx = tid; idx < HY * XY_TX; idx += nthr) {
      const int hy = idx >> 5, tx = idx & 31;
      cp_async8(PB + Gm::PB_G12 + hy * GP + tx, gp + FS + ry[hy] + cx[tx + Gm::XC]);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// Symmetry boundaries: the copies above fetched the mirrored interior
// values; the components that are odd under a mirror change sign here
// (rho u_x and g02 = D_z u_x under an x mirror, rho u_y and g12 under a y mirror).
template <int M>
__device__ __forceinline__ void xy_mirror_signs(const KParams &p, double *PB, int x0, int y0,
                                                int tid, int nthr) {
  using Gm = XYGeom<M>;
  constexpr int HX = Gm::HX, HY = Gm::HY, PX = Gm::PX, FSZ = Gm::FSZ;
  const bool xs = p.sym[0] && (x0 - Gm::XC < 0 || x0 + XY_TX + Gm::XC > p.nx);
  const bool ys = p.sym[1] && (y0 - M < 0 || y0 + XY_TY + M > p.ny);
  // only staged columns (rows) outside the grid can come through a mirror: the x
  // pass visits those columns and fixes rho u_x and g02, the y pass those rows and
  // fixes rho u_y and g12
  if (xs) {
    const int lo = max(0, min(HX, Gm::XC - x0));          // x < 0
    const int hi = max(lo, min(HX, p.nx - x0 + Gm::XC));  // x >= nx
    const int nb = lo + (HX - hi);
#pragma unroll 1
    for (int idx = tid; idx < HY * nb; idx += nthr) {
      const int hy = idx / nb, k = idx - hy * nb, hx = k < lo ? k : hi + (k - lo);
      int fx;
      bmap(x0 - Gm::XC + hx, p.nx, p.sym[0], fx);
      if (!fx) continue;
      double *d = PB + hy * PX + hx;
      d[XF_M0 * FSZ] = -d[XF_M0 * FSZ];
      if (hy >= M && hy < M + XY_TY) PB[Gm::PB_G02 + (hy - M) * PX + hx] *= -1.0;
    }
  }
  if (ys) {
    const int lo = max(0, min(HY, M - y0));          // y < 0
    const int hi = max(lo, min(HY, p.ny - y0 + M));  // y >= ny
    const int nb = lo + (HY - hi);
#pragma unroll 1
    for (int idx = tid; idx < nb * HX; idx += nthr) {
      const int k = idx / HX, hx = idx - k * HX, hy = k < lo ? k : hi + (k - lo);
      int fy;
      bmap(y0 - M + hy, p.ny, p.sym[1], fy);
      if (!fy) continue;
      double *d = PB + hy * PX + hx;
      d[XF_M1 * FSZ] = -d[XF_M1 * FSZ];
      if (hx >= Gm::XC && hx < Gm::XC + XY_TX) PB[Gm::PB_G12 + hy * Gm::GP + hx - Gm::XC] *= -1.0;
    }
  }
}

// L2 prefetch of plane z's epilogue operand W' on the tile rows
__device__ __forceinline__ void xy_prefetch_epilogue(const KParams &p, const double *w, int z,
                                                     int x0, int y0, int tid, int nthr) {
  const size_t FS = (size_t)p.nx * p.ny;
#pragma unroll 1
  for (int t = tid; t < XY_TY * 5 * 2; t += nthr) {
    const int half = t & 1, a = (t >> 1) % 5, ty = (t >> 1) / 5;
    const int y = y0 + ty, x = min(x0 + 16 * half, p.nx - 1);
    if (y >= p.ny) continue;
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(w + (size_t)z * 5 * FS + a * FS +
                                                      (size_t)y * p.nx + x));
  }
}

// Fused diagnostics (D-11, D-12) of the stage's input state, when the
// stage carries p.dpart: the integrands 1/2 rho u.u, 1/2 rho |omega|^2 and
// tau_ij du_i/dx_j of a point from the gradients group A has in hand
__device__ __forceinline__ void diag_point(double rho, double u0, double u1, double u2,
                                           double g01, double g02, double g10, double g12,
                                           double g20, double g21, double phi, double (&dg)[3]) {
  dg[0] += 0.5 * rho * (u0 * u0 + u1 * u1 + u2 * u2);
  const double w0 = g21 - g12, w1 = g02 - g20, w2 = g10 - g01;
  dg[1] += 0.5 * rho * (w0 * w0 + w1 * w1 + w2 * w2);
  dg[2] += phi;
}

// group A's (plane, tile) partial sums in a fixed order (warp butterflies, then
// the 4 warps in order) -> p.dpart[z][tile][3]; red: 12 doubles of shared memory
__device__ __forceinline__ void diag_tile_sum(const KParams &p, double (&dg)[3], double *red,
                                              int z, int q7) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dg[k] += __shfl_xor_sync(0xffffffffu, dg[k], o);
  }
  if ((q7 & 31) == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) red[3 * (q7 >> 5) + k] = dg[k];
  }
  nbar_sync(1, 128);
  if (q7 < 3) {
    const double t = ((red[q7] + red[3 + q7]) + red[6 + q7]) + red[9 + q7];
    const int tile = blockIdx.y * gridDim.x + blockIdx.x;
    p.dpart[((size_t)z * gridDim.x * gridDim.y + tile) * 3 + q7] = t;
  }
}

// Instantiations (XF bits), so that each feature costs the default path nothing:
// SYM (2): symmetry boundaries in x or y (mirror maps and the sign fix-up).
// TR (1): two-register RK3 epilogue (OSBLI_RK3_2R, kernels.h): W' is read from
//   the interior planes of qout (where the z-pass left it) and w holds Q_old.
// VAR (4): mu(T) (grad-mu terms from D_x T, D_y T and the z-pass's D_z T) and the
//   conservative viscous work (H_j written for launch_divh); SYM at run time (with
//   the two-register epilogue: XF = 5).
template <int M, int XF>
__global__ void __launch_bounds__(XY_CTA, 1)
    xypass_kernel(const KParams p, const double *__restrict__ q, double *__restrict__ qout,
                  double *__restrict__ w, const double *__restrict__ gz,
                  double *__restrict__ rout,
                  unsigned int *__restrict__ flag, const PlaneRange zr,
                  const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tg22,
                  const __grid_constant__ CUtensorMap tg02, const __grid_constant__ CUtensorMap tg12,
                  const int use_tma) {
  // XF bits: 1 = two-register epilogue, 2 = symmetry in x/y, 4 = equation variants
  // (mu(T), conservative viscous work), which take symmetry at run time;
  // 8 = fused diagnostics (stage 1 of osbli_step_diag)
  constexpr bool VAR = (XF & 4) != 0;
  constexpr bool DIAG = (XF & 8) != 0;  // fused diagnostics into p.dpart (osbli_step_diag)
  constexpr bool SYM = VAR || (XF & 2) != 0;
  constexpr bool TR = (XF & 1) != 0;
  // group B takes the x mixed-derivative parts (XY_MIXX_B) in the default and
  // diagnostics instantiations; the two-register epilogue holds Q_old in B's
  // registers, and there the move would spill
  constexpr bool MIXB = !VAR && XY_MIXX_B && (XF & 1) == 0;
  double *XT = nullptr;
  using Gm = XYGeom<M>;
  constexpr int HX = Gm::HX, HY = Gm::HY, PX = Gm::PX, FSZ = Gm::FSZ, NPT = Gm::NPT, TP = Gm::TP;
  constexpr int XO = Gm::XO, XC = Gm::XC;  // staged column offsets (odd m)
  extern __shared__ __align__(128) double SM[];
  double *PR = SM + Gm::OFF_PR;
  double *E0 = SM + Gm::OFF_E0, *E1 = SM + Gm::OFF_E1;
  double *XA = SM + Gm::OFF_XA, *XB = SM + Gm::OFF_XB;
  XT = SM + Gm::OFF_XT;
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * XY_TX, y0 = blockIdx.y * XY_TY;
  int zs, ze;
  if (!zr.segment(zs, ze)) return;
  const size_t FS = (size_t)p.nx * p.ny;
#if OSBLI_XY_SMSP_SPLIT
  // warps are spread over the 4 sub-partitions by warp id mod 4: group A on
  // sub-partitions 0, 1 (warps 0, 1, 4, 5), group B on 2, 3 (warps 2, 3, 6, 7)
  const int wid = tid >> 5;
  const int grp = tid < XY_THREADS ? (wid >> 1) & 1 : 2;
  const int q7 = (((wid >> 2) << 1) | (wid & 1)) * 32 + (tid & 31);
#else
  const int grp = tid >> 7;  // 0: velocity group A, 1: conservative group B (warp-uniform)
  const int q7 = tid & 127;
#endif
  bool bad = false;

  const int nplanes = ze - zs;
  if (tid >= XY_THREADS) {
    // ---- producer warpgroup: plane i into buffer i & 1 once the consumers released it;
    //      it needs few registers and hands the rest to the consumer warpgroups
#if OSBLI_XY_PRODUCERS == 4
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(XY_PROD_REGS) : "memory");
#endif
    const int lane = tid - XY_THREADS;
    int *cx = reinterpret_cast<int *>(SM + Gm::TOTAL), *ry = cx + Gm::HX;
    xy_tables<M, SYM>(p, cx, ry, x0, y0, lane, XY_PROD);
    nbar_sync(7, XY_PROD);  // tables complete (producers only)
    // 16-byte x-pairs (even nx, periodic x).  The symmetric instantiation stages 8
    // bytes at a time everywhere: a mirrored pair is reversed in memory, and pairs
    // on its interior tiles only measured slower (1.63 vs 1.55 ms at 256^3 o12)
    const bool pairs = !SYM && (p.nx % 2) == 0;
    // TMA for tiles whose staged region lies inside the grid (no wrap): one 5-field box
    // of Q and one box each of g22, g02, g12 per plane, completing on the plane
    // buffer's mbarrier; the other tiles and debug builds use cp.async, and so do
    // handles with symmetry boundaries in x or y: with their 8-byte staging TMA
    // measured slower there (1.69 vs 1.58 ms at 256^3 o12; the equation variants
    // without symmetry gain 2 %)
    const bool tma = use_tma && !(SYM && !OSBLI_XY_TMA_SYM && (p.sym[0] | p.sym[1])) && (p.nx % 2) == 0 &&
                     !OSBLI_DEBUG_CHECKS && x0 - Gm::XC >= 0 &&
                     x0 - Gm::XC + PX <= p.nx && y0 - M >= 0 && y0 + XY_TY + M <= p.ny;
    uint64_t *bars = reinterpret_cast<uint64_t *>(SM + Gm::OFF_BAR);
    if (tma && lane == 0) {
      mbar_init(bars, 1);
      mbar_init(bars + 1, 1);
    }
    nbar_sync(7, XY_PROD);  // the mbarriers are initialised
    constexpr unsigned TMA_BYTES =
        (unsigned)((6 * FSZ + XY_TY * PX + HY * Gm::GP) * sizeof(double));
    for (int i = 0; i < nplanes; ++i) {
      const int b = i & 1;
      if (i >= 2) nbar_sync(4 + b, XY_CTA);
      if (OSBLI_DEBUG_CHECKS) {  // a consumer still reading the released buffer reads NaN
        for (int k = lane; k < Gm::PBSZ; k += XY_PROD) SM[b * Gm::PBSZ + k] = dbg_nan();
        nbar_sync(7, XY_PROD);
      }
      double *PB = SM + b * Gm::PBSZ;
      if (tma) {
        if (lane == 0) {
          const int z = zs + i;
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          mbar_expect_tx(bars + b, TMA_BYTES);
          tma_load_box(PB, &tmq, x0 - Gm::XC, y0 - M, 0, z + p.G, bars + b);
          tma_load_box(PB + Gm::PB_G22, &tg22, x0 - Gm::XC, y0 - M, 2, z, bars + b);
          tma_load_box(PB + Gm::PB_G02, &tg02, x0 - Gm::XC, y0, 0, z, bars + b);
          tma_load_box(PB + Gm::PB_G12, &tg12, x0, y0 - M, 1, z, bars + b);
        }
      } else if (!OSBLI_XY_EXP_NOSTAGE || i < 2) {  // experiment: staging cost bound (wrong results)
        xy_issue_plane<M>(p, q, gz, PB, zs + i, cx, ry, lane, XY_PROD, pairs);
      }
      xy_prefetch_epilogue(p, TR ? qout + qplane(p, 0) : w, zs + i, x0, y0, lane, XY_PROD);
      if (TR && p.read_w) xy_prefetch_epilogue(p, w, zs + i, x0, y0, lane, XY_PROD);
      if (tma) mbar_wait(bars + b, (i >> 1) & 1);
      else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      if (SYM && (p.sym[0] | p.sym[1])) {
        nbar_sync(7, XY_PROD);  // every producer's copies have landed
        xy_mirror_signs<M>(p, SM + b * Gm::PBSZ, x0, y0, lane, XY_PROD);
      }
      nbar_arrive(2 + b, XY_PROD + 128);  // producers + group A
    }
    return;
  }

#if OSBLI_XY_PRODUCERS == 4
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(XY_CONS_REGS) : "memory");
#endif
  // The two consumer groups run decoupled, one plane apart at most; they meet only
  // where data passes between them (named barriers, arrive -> sync):
  //   8  A -> B  PR (p, 1/rho) of the plane is ready        (A computes PR)
  //   9  B -> A  B has read PR: A may compute the next plane's
  //   6  A -> B  A's parts of every point are in XA
  //   10 B -> A  B's epilogue has read XA: A may overwrite it
  //   1  A only  PR complete before phase X; E0/E1/XA[4] of phase X before phase Y
  // so A's formulas for plane z+1 overlap B's epilogue of plane z.
  const double third = 1.0 / 3.0;
  if (grp == 0) {
    // formulas p and 1/rho once per point of a landed plane buffer
    auto formulas = [&](const double *Sb) {
OSBLI_UNROLL(OSBLI_XY_FORM_UNROLL)
      for (int idx = q7; idx < HY * HX; idx += 128) {
        const int hy = idx / HX, hx = idx - hy * HX;
        const int s = hy * PX + hx;
        const double rho = Sb[XF_RHO * FSZ + s], m0 = Sb[XF_M0 * FSZ + s],
                     m1 = Sb[XF_M1 * FSZ + s], m2 = Sb[XF_M2 * FSZ + s], e = Sb[XF_E * FSZ + s];
        const double r = rcp_rho(rho);
        PR[XP_P * FSZ + s] = p.gm1 * (e - 0.5 * r * (m0 * m0 + m1 * m1 + m2 * m2));
        PR[XP_R * FSZ + s] = r;
      }
    };
    nbar_sync(2, XY_PROD + 128);  // first plane landed
    formulas(SM);
    for (int z = zs; z < ze; ++z) {
      const int i = z - zs, cur = i & 1;
      double *S = SM + cur * Gm::PBSZ;  // this plane's buffer
      const double *G02 = S + Gm::PB_G02, *G12 = S + Gm::PB_G12;
      nbar_sync(1, 128);           // every A thread's PR entries are written
      nbar_arrive(8, XY_THREADS);  // PR of plane z is complete
      // ---- phase X: thread -> (row, 4-wide x segment); lanes 0-15 / 16-31 = 16 rows
      {
        const int row = q7 & 15, seg = q7 >> 4;
        const int hy = row + M;
        const int base = hy * PX + seg * XY_RX + XO;  // window start (staged coords)
        const int pt0 = row * TP + seg * XY_RX;
        VelResult<M> o;
        velocity_dir<M, 0, VAR, MIXB ? 3 : 0>(
            p, S, PR, base, 1, G02 + row * PX + seg * XY_RX + XO, 1, E0, E1, 0, o);
        // B has finished reading XA (its epilogue of the previous plane)
        if (i > 0) nbar_sync(10, XY_THREADS);
        if (OSBLI_DEBUG_CHECKS) {
          for (int k = q7; k < 5 * NPT; k += 128) XA[k] = dbg_nan();
          nbar_sync(1, 128);
        }
        if (VAR) {
          // variants: mu(T) scales the viscous parts (D-26); D_x T kept for phase Y;
          // the conservative form leaves u_i V_i to D_j H_j (D-27)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const double mu = p.visc ? sutherland_mu(p, o.Tc[j]) : 1.0;
            const double V0 = mu * (p.nu * (o.d2u[0][j] + third * (o.d2u[0][j] + o.mixA[j])));
            const double V1 = mu * (p.nu * o.d2u[1][j]);
            const double V2 = mu * (p.nu * (o.d2u[2][j] + third * o.mixB[j]));
            XA[0 * NPT + pt0 + j] = V0;
            XA[1 * NPT + pt0 + j] = V1;
            XA[2 * NPT + pt0 + j] = V2;
            const double uv = p.cons ? 0.0 : o.uc[0][j] * V0 + o.uc[1][j] * V1 + o.uc[2][j] * V2;
            XA[3 * NPT + pt0 + j] = fma(p.kappa * mu, o.d2T[j], uv);
            XA[4 * NPT + pt0 + j] = o.g[2][j];          // g20
            E0[hy * TP + seg * XY_RX + j] = o.g[0][j];  // g00
            E1[hy * TP + seg * XY_RX + j] = o.g[1][j];  // g10
            XT[pt0 + j] = o.d1T[j];
          }
        } else
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // x-parts of V_i: V0 += nu (4/3 D00 u0 + 1/3 D0 g22); V1 += nu D00 u1;
          // V2 += nu (D00 u2 + 1/3 D0 g02)
          // (MIXB: the 1/3 D0 g22 and 1/3 D0 g02 parts are group B's)
          const double V0 = p.nu * (o.d2u[0][j] + third * (o.d2u[0][j] + (MIXB ? 0.0 : o.mixA[j])));
          const double V1 = p.nu * o.d2u[1][j];
          const double V2 = p.nu * (o.d2u[2][j] + (MIXB ? 0.0 : third * o.mixB[j]));
          XA[0 * NPT + pt0 + j] = V0;
          XA[1 * NPT + pt0 + j] = V1;
          XA[2 * NPT + pt0 + j] = V2;
          const double uv = o.uc[0][j] * V0 + o.uc[1][j] * V1 + o.uc[2][j] * V2;
          XA[3 * NPT + pt0 + j] = uv;
          XA[4 * NPT + pt0 + j] = o.g[2][j];          // g20
          E0[hy * TP + seg * XY_RX + j] = o.g[0][j];  // g00
          E1[hy * TP + seg * XY_RX + j] = o.g[1][j];  // g10
        }
      }
      // ---- g00, g10 on the 2m halo rows (inner derivatives of D_y g00, D_y g10)
      for (int task = q7; task < 2 * M * (XY_TX / XY_RX); task += 128) {
        const int rr = task % (2 * M), seg = task / (2 * M);
        const int hy = rr < M ? rr : rr + XY_TY;
        const int base = hy * PX + seg * XY_RX + XO;
        constexpr int W = Gm::W;
        double r[W], v[W], t[W];
        ldwin<W, Gm::XW>(PR + XP_R * FSZ + base, 1, r);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          ldwin<W, Gm::XW>(S + (XF_M0 + i) * FSZ + base, 1, t);
#pragma unroll
          for (int k = 0; k < W; ++k) v[k] = __dmul_rn(t[k], r[k]);
          double *Ei = i == 0 ? E0 : E1;
#pragma unroll
          for (int j = 0; j < 4; ++j) Ei[hy * TP + seg * XY_RX + j] = wd1<M, W>(p, v, j);
        }
      }
      nbar_sync(1, 128);
      // ---- phase Y: thread -> (column, 4-tall y segment); lanes = 32 consecutive columns
      {
        const int col = q7 & 31, seg = q7 >> 5;
        const int base = (seg * XY_RY) * PX + col + XC;
        const int ebase = (seg * XY_RY) * TP + col;
        const int gbase = (seg * XY_RY) * Gm::GP + col;
        double dTz[4];
        if (VAR) {  // D_z T of this thread's points (z-pass), loaded ahead of the stencils
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int yy = min(y0 + seg * XY_RY + j, p.ny - 1), xx = min(x0 + col, p.nx - 1);
            dTz[j] = p.dtz[(size_t)z * FS + (size_t)yy * p.nx + xx];
          }
        }
        VelResult<M> o;
        velocity_dir<M, 1, VAR, VAR ? 0 : XY_MIXY_B>(p, S, PR, base, PX, G12 + gbase, Gm::GP, E0,
                                                          E1, ebase, o);
        double dg[3] = {0.0, 0.0, 0.0};  // fused diagnostics sums of this thread's points (DIAG)
        if (VAR) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int ty = seg * XY_RY + j;
            const int pt = ty * TP + col;
            const int c = (ty + M) * PX + col + XC;
            const double g00 = E0[(ty + M) * TP + col], g10 = E1[(ty + M) * TP + col];
            const double g20 = XA[4 * NPT + pt];
            const double g01 = o.g[0][j], g11 = o.g[1][j], g21 = o.g[2][j];
            const double g02 = G02[ty * PX + col + XC], g12 = G12[(ty + M) * Gm::GP + col],
                         g22 = S[Gm::PB_G22 + c];
            const double T = o.Tc[j];
            const double mu = p.visc ? sutherland_mu(p, T) : 1.0;
            const double dmu = p.visc ? sutherland_dmu(p, T, mu) : 0.0;
            const double V0y = mu * (p.nu * (o.d2u[0][j] + third * o.mixD[j]));
            const double V1y =
                mu * (p.nu * (o.d2u[1][j] + third * (o.d2u[1][j] + o.mixC[j] + o.mixA[j])));
            const double V2y = mu * (p.nu * (o.d2u[2][j] + third * o.mixB[j]));
            const double thxy = g00 + g11, th = thxy + g22;
            const double s01 = g01 + g10, s02 = g02 + g20, s12 = g12 + g21;
            const double s00 = 2.0 * g00 - (2.0 / 3.0) * th, s11 = 2.0 * g11 - (2.0 / 3.0) * th,
                         s22 = 2.0 * g22 - (2.0 / 3.0) * th;
            // grad-mu terms (d mu/dx_j) S_ij, d mu/dx_j = mu'(T) D_j T (D-26)
            const double tx = XT[pt], ty_ = o.d1T[j], tz = dTz[j];
            const double cm = p.nu * dmu;
            const double C0 = cm * (tx * s00 + ty_ * s01 + tz * s02);
            const double C1 = cm * (tx * s01 + ty_ * s11 + tz * s12);
            const double C2 = cm * (tx * s02 + ty_ * s12 + tz * s22);
            const double V0 = XA[0 * NPT + pt] + V0y + C0, V1 = XA[1 * NPT + pt] + V1y + C1,
                         V2 = XA[2 * NPT + pt] + V2y + C2;
            const double u0 = o.uc[0][j], u1 = o.uc[1][j], u2 = o.uc[2][j];
            const double heat =
                p.kappa * fma(mu, o.d2T[j], dmu * (tx * tx + ty_ * ty_ + tz * tz));
            double e = XA[3 * NPT + pt] + heat;
            if (DIAG && x0 + col < p.nx && y0 + ty < p.ny) {
              const double Phi = mu * (p.nu * (2.0 * (g00 * g00 + g11 * g11 + g22 * g22) +
                                               s01 * s01 + s02 * s02 + s12 * s12 -
                                               (2.0 / 3.0) * th * th));
              diag_point(S[XF_RHO * FSZ + c], u0, u1, u2, g01, g02, g10, g12, g20, g21, Phi, dg);
            }
            if (p.cons) {
              // H_j = u_i tau_ij for the divergence kernel (D-27)
              const double mn = mu * p.nu;
              const int y = y0 + ty, x = x0 + col;
              if (y < p.ny && x < p.nx) {
                double *h = p.hflux + (size_t)z * 3 * FS + (size_t)y * p.nx + x;
                h[0] = mn * (u0 * s00 + u1 * s01 + u2 * s02);
                h[FS] = mn * (u0 * s01 + u1 * s11 + u2 * s12);
                h[2 * FS] = mn * (u0 * s02 + u1 * s12 + u2 * s22);
              }
            } else {
              const double Phi = mu * (p.nu * (2.0 * (g00 * g00 + g11 * g11 + g22 * g22) +
                                               s01 * s01 + s02 * s02 + s12 * s12 -
                                               (2.0 / 3.0) * th * th));
              e += Phi + (u0 * (V0y + C0) + u1 * (V1y + C1) + u2 * (V2y + C2));
            }
            XA[0 * NPT + pt] = -0.5 * S[XF_RHO * FSZ + c] * thxy;
            XA[1 * NPT + pt] = fma(-0.5 * S[XF_M0 * FSZ + c], thxy, V0);
            XA[2 * NPT + pt] = fma(-0.5 * S[XF_M1 * FSZ + c], thxy, V1);
            XA[3 * NPT + pt] = fma(-0.5 * S[XF_M2 * FSZ + c], thxy, V2);
            XA[4 * NPT + pt] = fma(-0.5 * S[XF_E * FSZ + c], thxy, e);
          }
        } else
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ty = seg * XY_RY + j;
          const int pt = ty * TP + col;
          const int c = (ty + M) * PX + col + XC;
          const double g00 = E0[(ty + M) * TP + col], g10 = E1[(ty + M) * TP + col];
          const double g20 = XA[4 * NPT + pt];
          const double g01 = o.g[0][j], g11 = o.g[1][j], g21 = o.g[2][j];
          const double g02 = G02[ty * PX + col + XC], g12 = G12[(ty + M) * Gm::GP + col],
                       g22 = S[Gm::PB_G22 + c];
          // y-parts of V_i: V0 += nu (D11 u0 + 1/3 D1 g10);
          // V1 += nu (4/3 D11 u1 + 1/3 (D1 g00 + D1 g22)); V2 += nu (D11 u2 + 1/3 D1 g12)
          const double V0y = p.nu * (o.d2u[0][j] + third * o.mixD[j]);
          // (XY_MIXY_B bits: the 1/3 D1 g22 and 1/3 D1 g12 parts are group B's)
          const double V1y = p.nu * (o.d2u[1][j] + third * (o.d2u[1][j] + o.mixC[j] +
                                                            ((XY_MIXY_B & 1) ? 0.0 : o.mixA[j])));
          const double V2y = p.nu * (o.d2u[2][j] + ((XY_MIXY_B & 2) ? 0.0 : third * o.mixB[j]));
          const double V0 = XA[0 * NPT + pt] + V0y, V1 = XA[1 * NPT + pt] + V1y,
                       V2 = XA[2 * NPT + pt] + V2y;
          const double thxy = g00 + g11, th = thxy + g22;
          const double s01 = g01 + g10, s02 = g02 + g20, s12 = g12 + g21;
          // tau_ij du_i/dx_j (eq. 8)
          const double Phi = p.nu * (2.0 * (g00 * g00 + g11 * g11 + g22 * g22) + s01 * s01 +
                                     s02 * s02 + s12 * s12 - (2.0 / 3.0) * th * th);
          const double u0 = o.uc[0][j], u1 = o.uc[1][j], u2 = o.uc[2][j];
          if (DIAG && x0 + col < p.nx && y0 + ty < p.ny)
            diag_point(S[XF_RHO * FSZ + c], u0, u1, u2, g01, g02, g10, g12, g20, g21, Phi, dg);
          const double ex = XA[3 * NPT + pt];  // u_i V_i^x (phase X; the heat flux is B's)
          // dilatation halves of the skew terms, -1/2 s (g00 + g11)
          XA[0 * NPT + pt] = -0.5 * S[XF_RHO * FSZ + c] * thxy;
          XA[1 * NPT + pt] = fma(-0.5 * S[XF_M0 * FSZ + c], thxy, V0);
          XA[2 * NPT + pt] = fma(-0.5 * S[XF_M1 * FSZ + c], thxy, V1);
          XA[3 * NPT + pt] = fma(-0.5 * S[XF_M2 * FSZ + c], thxy, V2);
          XA[4 * NPT + pt] = fma(-0.5 * S[XF_E * FSZ + c], thxy,
                                 (ex + Phi) + (u0 * V0y + u1 * V1y + u2 * V2y));
        }
        if (DIAG) diag_tile_sum(p, dg, SM + Gm::OFF_DG, z, q7);
      }
      // A's part of every point of this tile is final: hand over to group B
      nbar_arrive(6, XY_THREADS);
      if (i + 2 < nplanes) nbar_arrive(4 + cur, XY_CTA);  // done with this plane buffer
      if (i + 1 < nplanes) {
        nbar_sync(9, XY_THREADS);                 // B has read PR of plane z
        if (OSBLI_DEBUG_CHECKS) {
          for (int k = q7; k < 2 * FSZ; k += 128) PR[k] = dbg_nan();
          nbar_sync(1, 128);
        }
        nbar_sync(2 + (cur ^ 1), XY_PROD + 128);  // plane z+1 landed
        if (!OSBLI_XY_EXP_NOFORM) formulas(SM + (cur ^ 1) * Gm::PBSZ);  // experiment flag: wrong results
      }
    }
  } else {
    for (int z = zs; z < ze; ++z) {
      const int i = z - zs, cur = i & 1;
      const double *S = SM + cur * Gm::PBSZ;  // this plane's buffer
      nbar_sync(8, XY_THREADS);  // plane z landed and its PR computed (group A)
      // ---- phase X: x-derivatives of the conservative group
      {
        const int row = q7 & 15, seg = q7 >> 4;
        const int base = (row + M) * PX + seg * XY_RX + XO;
        const int pt0 = row * TP + seg * XY_RX;
        double R[5][4];
        conservative_dir<M, 0, !VAR>(p, S, PR, base, 1, R);
        if (MIXB) {
          // the x mixed-derivative viscous parts, nu/3 D_x g22 (momentum x) and
          // nu/3 D_x g02 (momentum z), and their work u_i V_i (D-7)
          constexpr int W = Gm::W;
          double v[W], ma[4];
          ldwin<W, Gm::XW>(S + Gm::PB_G22 + base, 1, v);
#pragma unroll
          for (int j = 0; j < 4; ++j) ma[j] = (p.nu * third) * wd1<M, W>(p, v, j);
          ldwin<W, Gm::XW>(S + Gm::PB_G02 + row * PX + seg * XY_RX + XO, 1, v);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const double mb = (p.nu * third) * wd1<M, W>(p, v, j);
            const int c = base + M + j;
            const double r = PR[XP_R * FSZ + c];
            const double u0 = __dmul_rn(S[XF_M0 * FSZ + c], r), u2 = __dmul_rn(S[XF_M2 * FSZ + c], r);
            R[1][j] += ma[j];
            R[3][j] += mb;
            R[4][j] = fma(u0, ma[j], fma(u2, mb, R[4][j]));
          }
        }
#pragma unroll
        for (int f = 0; f < 5; ++f)
#pragma unroll
          for (int j = 0; j < 4; ++j) XB[f * NPT + pt0 + j] = R[f][j];
      }
      // ---- phase Y and the epilogue
      {
        const int col = q7 & 31, seg = q7 >> 5;
        const int base = (seg * XY_RY) * PX + col + XC;
        // group B finishes the stage for its 4 points: W' (z-pass output) is loaded
        // first so that its latency hides behind the y-derivatives
        const int x = x0 + col;
        const bool xin = x < p.nx;
        double wp[5][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int y = min(y0 + seg * XY_RY + j, p.ny - 1);
          const size_t o = (size_t)z * 5 * FS + (size_t)y * p.nx + (xin ? x : p.nx - 1);
#pragma unroll
          for (int f = 0; f < 5; ++f) wp[f][j] = TR ? qout[qplane(p, 0) + o + f * FS] : w[o + f * FS];
        }
        double R[5][4];
        conservative_dir<M, 1, !VAR>(p, S, PR, base, PX, R);
        if (!VAR && XY_MIXY_B) {
          // the y mixed-derivative viscous parts, nu/3 D_y g22 (momentum y) and/or
          // nu/3 D_y g12 (momentum z), and their work u_i V_i (D-7)
          constexpr int W = Gm::W;
          double v[W], ma[4] = {0.0, 0.0, 0.0, 0.0}, mb[4] = {0.0, 0.0, 0.0, 0.0};
          if (XY_MIXY_B & 1) {
            ldwin<W>(S + Gm::PB_G22 + base, PX, v);
#pragma unroll
            for (int j = 0; j < 4; ++j) ma[j] = (p.nu * third) * wd1<M, W>(p, v, j);
          }
          if (XY_MIXY_B & 2) {
            ldwin<W>(S + Gm::PB_G12 + (seg * XY_RY) * Gm::GP + col, Gm::GP, v);
#pragma unroll
            for (int j = 0; j < 4; ++j) mb[j] = (p.nu * third) * wd1<M, W>(p, v, j);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int c = base + (M + j) * PX;
            const double r = PR[XP_R * FSZ + c];
            if (XY_MIXY_B & 1) {
              const double u1 = __dmul_rn(S[XF_M1 * FSZ + c], r);
              R[2][j] += ma[j];
              R[4][j] = fma(u1, ma[j], R[4][j]);
            }
            if (XY_MIXY_B & 2) {
              const double u2 = __dmul_rn(S[XF_M2 * FSZ + c], r);
              R[3][j] += mb[j];
              R[4][j] = fma(u2, mb[j], R[4][j]);
            }
          }
        }
        if (i + 1 < nplanes) nbar_arrive(9, XY_THREADS);  // done with PR: A may refill it
        // two-register RK3: the register Q_old of the four points, loaded before
        // the hand-over wait so that its latency hides behind it
        double qold[5][4];
        if (TR && p.read_w) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int y = min(y0 + seg * XY_RY + j, p.ny - 1);
            const size_t o = (size_t)z * 5 * FS + (size_t)y * p.nx + (xin ? x : p.nx - 1);
#pragma unroll
            for (int f = 0; f < 5; ++f) qold[f][j] = w[o + f * FS];
          }
        }
        nbar_sync(6, XY_THREADS);  // group A's parts are in XA (and XB of all B threads)
        // ---- epilogue: W <- W' + dt R_xy ; Q' <- Q + B W  (rows of 32 columns; residual
        //      mode: dt = 1, A = 0 so that W' = Rz and R = W' + R_xy)
        const int fidx[5] = {XF_RHO, XF_M0, XF_M1, XF_M2, XF_E};
        // W' + dt R_xy of the four points first; then one uniform branch on the mode
        double wn[5][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int pt = (seg * XY_RY + j) * TP + col;
#pragma unroll
          for (int f = 0; f < 5; ++f)
            wn[f][j] = fma(p.dt, XA[f * NPT + pt] + (XB[f * NPT + pt] + R[f][j]), wp[f][j]);
        }
        const int mode = rout ? 0 : (TR ? 3 : (p.write_w ? 1 : 2));
        // one uniform branch on the mode, the four points inside it (the executed
        // code stays contiguous)
        auto points = [&](auto &&store) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int ty = seg * XY_RY + j;
            const int y = y0 + ty;
            if (!xin || y >= p.ny) continue;
            store(j, (ty + M) * PX + col + XC, (size_t)z * 5 * FS + (size_t)y * p.nx + x,
                  qout + qplane(p, z) + (size_t)y * p.nx + x);
          }
        };
        if (mode == 0) {
          points([&](int j, int, size_t o, double *) {
#pragma unroll
            for (int f = 0; f < 5; ++f) rout[o + f * FS] = wn[f][j];
          });
        } else if (mode == 1) {  // 2N RK3 stages 1, 2: W <- W', Q' = Q + B W
          points([&](int j, int c, size_t o, double *qo) {
#pragma unroll
            for (int f = 0; f < 5; ++f) {
              w[o + f * FS] = wn[f][j];
              const double qn = fma(p.B, wn[f][j], S[fidx[f] * FSZ + c]);
              qo[f * FS] = qn;
              bad |= !isfinite(qn);
            }
          });
        } else if (mode == 2) {  // last stage / Euler: Q' = Q + B W
          points([&](int j, int c, size_t, double *qo) {
#pragma unroll
            for (int f = 0; f < 5; ++f) {
              const double qn = fma(p.B, wn[f][j], S[fidx[f] * FSZ + c]);
              qo[f * FS] = qn;
              bad |= !isfinite(qn);
            }
          });
        } else {  // two-register RK3: w holds Q_old
          points([&](int j, int c, size_t o, double *qo) {
#pragma unroll
            for (int f = 0; f < 5; ++f) {
              const double qb = p.read_w ? qold[f][j] : S[fidx[f] * FSZ + c];
              if (p.write_w) w[o + f * FS] = fma(p.beta, wn[f][j], qb);
              const double qn = fma(p.B, wn[f][j], qb);
              qo[f * FS] = qn;
              bad |= !isfinite(qn);
            }
          });
        }
        if (i + 1 < nplanes) nbar_arrive(10, XY_THREADS);  // done with XA
        if (i + 2 < nplanes) nbar_arrive(4 + cur, XY_CTA);  // done with this plane buffer
      }
    }
  }
  if (bad) atomicOr(flag, 1u);
}

}  // namespace ws
