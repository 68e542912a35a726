// =============================================================================
// OpenSBLI hot-path ORACLE — plain, slow, single-threaded CPU reference.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.
// The product path (paper_1609_01277_b200/) never links, imports or calls it,
// and this file shares no code, header, table or constant with the CUDA path.
//
// Paper = /root/reference/PAPER.md (Jacobs, Jammy & Sandham, arXiv 1609.01277).
// "P:n" below is a PAPER.md line.  "D-n" is a reading listed in DESIGN.md §3.
//
// What is computed (all fp64, compiled with -O2 -ffp-contract=off):
//   * central-difference weights of arbitrary even order, first and second
//     derivative, by solving the Taylor moment conditions in exact rational
//     arithmetic ("stencil coefficients are computed using SymPy, which
//     allows stencils of an arbitrary order of accuracy");
//   * the semi-discrete residual R(Q) of the 3D compressible Navier-Stokes
//     equations with the EOS, the skew-symmetric
//     convective form, the viscous Laplacian by second-derivative
//     stencils and nested derivatives evaluated inner-first, on
//     a fully periodic grid;
//   * forward Euler and the 3-stage low-storage RK3 (tableau D-1);
//   * the kinetic-energy / enstrophy integrals and the viscous
//     dissipation rate (D-12);
//   * the scalar advection-diffusion equation of the paper's verification
//     cases (1D wave, 2D method of manufactured solutions) with an
//     optional steady source term.
//
// The code follows the paper's structure: "formula" work arrays (u_i, p, T)
// are evaluated first, then the inner derivatives of nested
// derivatives (g_ij = du_i/dx_j), then each residual point by point
// with every derivative replaced by its central-difference stencil sum.
// No term regrouping, no fusion: one stencil sum per derivative in the
// expanded equations.
//
// Parity pins (tests/test_oracle_*.py): stencil closed forms and polynomial
// exactness, Fourier eigenvalues, mixed-derivative closed form, equilibrium,
// discrete conservation, Taylor-jet manufactured-solution convergence orders,
// entropy-wave RK3/Euler amplification closed form, the paper's 1D wave error
// (P:182-184), RK3 ODE order, TGV diagnostics at t=0 in closed form.
// =============================================================================
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// Exact rational arithmetic (for the stencil moment conditions).
// ---------------------------------------------------------------------------
typedef __int128 i128;

i128 gcd128(i128 a, i128 b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b != 0) {
    i128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}

struct Frac {
  i128 n, d;  // d > 0, gcd(n,d) == 1
  Frac(i128 n_ = 0, i128 d_ = 1) : n(n_), d(d_) { norm(); }
  void norm() {
    if (d < 0) { n = -n; d = -d; }
    i128 g = gcd128(n, d);
    if (g > 1) { n /= g; d /= g; }
    if (n == 0) d = 1;
  }
  Frac operator+(const Frac& o) const { return Frac(n * o.d + o.n * d, d * o.d); }
  Frac operator-(const Frac& o) const { return Frac(n * o.d - o.n * d, d * o.d); }
  Frac operator*(const Frac& o) const { return Frac(n * o.n, d * o.d); }
  Frac operator/(const Frac& o) const { return Frac(n * o.d, d * o.n); }
  double to_double() const { return (double)(long long)n / (double)(long long)d; }
};

// Solve A x = rhs (size s) exactly by Gauss-Jordan elimination.
bool solve_exact(std::vector<std::vector<Frac>> A, std::vector<Frac> rhs,
                 std::vector<Frac>& x) {
  const int s = (int)rhs.size();
  for (int c = 0; c < s; ++c) {
    int piv = -1;
    for (int r = c; r < s; ++r)
      if (A[r][c].n != 0) { piv = r; break; }
    if (piv < 0) return false;
    std::swap(A[c], A[piv]);
    std::swap(rhs[c], rhs[piv]);
    for (int r = 0; r < s; ++r) {
      if (r == c || A[r][c].n == 0) continue;
      Frac f = A[r][c] / A[c][c];
      for (int k = c; k < s; ++k) A[r][k] = A[r][k] - f * A[c][k];
      rhs[r] = rhs[r] - f * rhs[c];
    }
  }
  x.resize(s);
  for (int r = 0; r < s; ++r) x[r] = rhs[r] / A[r][r];
  return true;
}

// Central stencil of accuracy `order` (even) for the derivative of degree 1 or
// 2 on offsets -m..m, m = order/2.  The moment conditions
//     sum_{k=-m..m} w_k k^q = degree! [q == degree],  q = 0..2m
// are solved with the symmetry of the stencil imposed (antisymmetric for
// degree 1, symmetric for degree 2), which is what "central" means.
//   degree 1: w_{+k} = a_k, w_{-k} = -a_k, w_0 = 0
//             odd q = 1,3,..,2m-1:  2 sum_k a_k k^q = [q == 1]
//   degree 2: w_{+-k} = b_k, w_0 = b_0
//             q = 0: b_0 + 2 sum_k b_k = 0;  even q = 2..2m: 2 sum_k b_k k^q = 2 [q == 2]
bool central_weights(int order, std::vector<Frac>& a, std::vector<Frac>& b) {
  if (order < 2 || (order % 2) != 0 || order > 16) return false;
  const int m = order / 2;
  std::vector<std::vector<Frac>> A(m, std::vector<Frac>(m));
  std::vector<Frac> rhs(m);
  for (int r = 0; r < m; ++r) {  // q = 2r+1
    const int q = 2 * r + 1;
    for (int k = 1; k <= m; ++k) {
      i128 p = 1;
      for (int t = 0; t < q; ++t) p *= k;
      A[r][k - 1] = Frac(2 * p);
    }
    rhs[r] = Frac(q == 1 ? 1 : 0);
  }
  if (!solve_exact(A, rhs, a)) return false;
  for (int r = 0; r < m; ++r) {  // q = 2r+2
    const int q = 2 * r + 2;
    for (int k = 1; k <= m; ++k) {
      i128 p = 1;
      for (int t = 0; t < q; ++t) p *= k;
      A[r][k - 1] = Frac(2 * p);
    }
    rhs[r] = Frac(q == 2 ? 2 : 0);
  }
  std::vector<Frac> bk;
  if (!solve_exact(A, rhs, bk)) return false;
  Frac b0(0);
  for (int k = 0; k < m; ++k) b0 = b0 - Frac(2) * bk[k];
  b.clear();
  b.push_back(b0);
  for (int k = 0; k < m; ++k) b.push_back(bk[k]);
  return true;
}

// ---------------------------------------------------------------------------
// Grid: x_i = i*dx, i = 0..N-1, arrays [nz][ny][nx], x fastest.
// Boundaries per direction: periodic, f[i+N] = f[i]; or symmetry,
// "phi(x_N) = phi(x_{N-1}) for scalar fields and phi_i(x_N) = -phi_i(x_{N-1})
// for vector fields (in the direction i)": the halo mirrors the interior about
// the boundary face (ghost -k <-> interior k-1, ghost N-1+k <-> interior N-k),
// with the sign of the grid function's parity in that direction.
// ---------------------------------------------------------------------------
struct Par {  // parity of a grid function under the mirror of each direction
  int s[3] = {1, 1, 1};
};
Par odd_in(int d) {
  Par p;
  p.s[d] = -1;
  return p;
}
Par operator*(const Par& a, const Par& b) {
  Par p;
  for (int d = 0; d < 3; ++d) p.s[d] = a.s[d] * b.s[d];
  return p;
}
const Par EVEN;

struct Grid {
  int n[3];  // nx, ny, nz
  int sym[3] = {0, 0, 0};  // 1: symmetry boundaries in that direction
  double dx;
  int m;
  std::vector<double> a;  // a_1..a_m  (first derivative)
  std::vector<double> b;  // b_0..b_m  (second derivative)
  size_t npts() const { return (size_t)n[0] * n[1] * n[2]; }
  size_t idx(int i, int j, int k) const {
    return ((size_t)k * n[1] + j) * n[0] + i;
  }
  // index of the point displaced by s along direction dir; *flip = 1 when the
  // value comes through an odd number of mirrors (symmetry boundaries)
  size_t shifted(int i, int j, int k, int dir, int s, int* flip = nullptr) const {
    int c[3] = {i, j, k};
    const int nd = n[dir];
    int f = 0;
    if (sym[dir]) {
      int cm = ((c[dir] + s) % (2 * nd) + 2 * nd) % (2 * nd);
      if (cm >= nd) {
        cm = 2 * nd - 1 - cm;
        f = 1;
      }
      c[dir] = cm;
    } else {
      c[dir] = ((c[dir] + s) % nd + nd) % nd;
    }
    if (flip) *flip = f;
    return idx(c[0], c[1], c[2]);
  }
  // value of grid function f (parity p) at the displaced point
  double at(const double* f, const Par& p, int i, int j, int k, int dir, int s) const {
    int fl = 0;
    const double v = f[shifted(i, j, k, dir, s, &fl)];
    return fl && p.s[dir] < 0 ? -v : v;
  }
};

// First derivative d f / d x_dir at (i,j,k):
//   (1/dx) sum_{k=1..m} a_k (f[+k] - f[-k])
double D1(const Grid& g, const double* f, int i, int j, int k, int dir, const Par& p = EVEN) {
  double s = 0.0;
  for (int t = 1; t <= g.m; ++t)
    s += g.a[t - 1] * (g.at(f, p, i, j, k, dir, t) - g.at(f, p, i, j, k, dir, -t));
  return s / g.dx;
}

// First derivative of the pointwise product f*h (the grid function f*h,
// evaluated at each stencil point).
double D1prod(const Grid& g, const double* f, const Par& pf, const double* h, const Par& ph,
              int i, int j, int k, int dir) {
  double s = 0.0;
  for (int t = 1; t <= g.m; ++t)
    s += g.a[t - 1] * (g.at(f, pf, i, j, k, dir, t) * g.at(h, ph, i, j, k, dir, t) -
                       g.at(f, pf, i, j, k, dir, -t) * g.at(h, ph, i, j, k, dir, -t));
  return s / g.dx;
}

// Second derivative d^2 f / d x_dir^2 at (i,j,k):
//   (1/dx^2) sum_{k=1..m} b_k ((f[+k] - f) + (f[-k] - f))
// (equivalent to sum_{k=-m..m} w_k f[k] since b_0 = -2 sum b_k; this form is
//  exactly zero on a constant field).
double D2(const Grid& g, const double* f, int i, int j, int k, int dir, const Par& p = EVEN) {
  const double f0 = f[g.idx(i, j, k)];
  double s = 0.0;
  for (int t = 1; t <= g.m; ++t)
    s += g.b[t] * ((g.at(f, p, i, j, k, dir, t) - f0) + (g.at(f, p, i, j, k, dir, -t) - f0));
  return s / (g.dx * g.dx);
}

struct Phys {
  double Re, Pr, Minf, gamma;
  int visc_law = 0;     // 0: mu == 1 (D-3); 1: Sutherland mu(T)
  double suth = 0.0;    // Sutherland constant over the reference temperature, S/T_ref
  int energy_form = 0;  // 0: viscous work product-rule expanded (D-5); 1: D_j(u_i tau_ij) (N2)
  double nu() const { return 1.0 / Re; }  // Re = inf -> 0
  double kappa() const {                   // P:253 heat-flux coefficient without mu
    return 1.0 / ((gamma - 1.0) * Minf * Minf * Pr * Re);
  }
  // dimensionless viscosity and its temperature derivative (D-26):
  //   mu(T) = T^{3/2} (1 + S) / (T + S),  mu(1) = 1
  double mu(double T) const {
    if (visc_law == 0) return 1.0;
    return T * std::sqrt(T) * (1.0 + suth) / (T + suth);
  }
  double dmu(double T) const {  // d mu / dT = mu (3/(2T) - 1/(T + S))
    if (visc_law == 0) return 0.0;
    return mu(T) * (1.5 / T - 1.0 / (T + suth));
  }
};

// Formula work arrays ("evaluation of formulas"): primitives from the
// conservative state Q = (rho, rho u_0, rho u_1, rho u_2, rho E).
struct Work {
  std::vector<double> u[3], p, T;
  std::vector<double> g[3][3];  // g[i][j] = D_j u_i (inner derivatives)
};

void formulas(const Grid& G, const Phys& ph, const double* Q, Work& w) {
  const size_t N = G.npts();
  const double* rho = Q;
  const double* e = Q + 4 * N;
  for (int i = 0; i < 3; ++i) w.u[i].assign(N, 0.0);
  w.p.assign(N, 0.0);
  w.T.assign(N, 0.0);
  for (size_t q = 0; q < N; ++q) {
    for (int i = 0; i < 3; ++i) w.u[i][q] = Q[(1 + i) * N + q] / rho[q];
    // rho E = p/(gamma-1) + 1/2 rho u_j u_j
    double ke = 0.0;
    for (int jj = 0; jj < 3; ++jj) ke += rho[q] * w.u[jj][q] * w.u[jj][q];
    w.p[q] = (ph.gamma - 1.0) * (e[q] - 0.5 * ke);
    // p = rho T / (gamma M^2)
    w.T[q] = ph.gamma * ph.Minf * ph.Minf * w.p[q] / rho[q];
  }
}

void velocity_gradients(const Grid& G, Work& w) {
  const size_t N = G.npts();
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) w.g[i][j].assign(N, 0.0);
  for (int k = 0; k < G.n[2]; ++k)
    for (int jy = 0; jy < G.n[1]; ++jy)
      for (int ix = 0; ix < G.n[0]; ++ix) {
        const size_t q = G.idx(ix, jy, k);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) w.g[i][j][q] = D1(G, w.u[i].data(), ix, jy, k, j, odd_in(i));
      }
}

// Residual R = dQ/dt of the expanded equations at every point.
void residual(const Grid& G, const Phys& ph, const double* Q, double* R) {
  const size_t N = G.npts();
  Work w;
  formulas(G, ph, Q, w);
  velocity_gradients(G, w);
  const double nu = ph.nu(), kap = ph.kappa();
  const double* rho = Q;
  const double* mom[3] = {Q + N, Q + 2 * N, Q + 3 * N};
  const double* e = Q + 4 * N;
  // the conserved quantities rho*phi of the skew form: phi = 1, u_i, E;
  // parities under the mirrors: rho, E even; rho u_i odd in direction i
  const double* s_of[5] = {rho, mom[0], mom[1], mom[2], e};
  const Par s_par[5] = {EVEN, odd_in(0), odd_in(1), odd_in(2), EVEN};
  // g_ij = du_i/dx_j: parity of u_i times the flip of the derivative direction j
  Par g_par[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) g_par[i][j] = odd_in(i) * odd_in(j);
  // conservative viscous work (N2, D-27): H_j = u_i tau_ij at every point, its
  // divergence by first-derivative stencils (H_j is odd in direction j)
  std::vector<double> H[3];
  if (ph.energy_form == 1) {
    for (int j = 0; j < 3; ++j) H[j].assign(N, 0.0);
    for (size_t q = 0; q < N; ++q) {
      const double div = w.g[0][0][q] + w.g[1][1][q] + w.g[2][2][q];
      const double mu = ph.mu(w.T[q]);
      for (int j = 0; j < 3; ++j)
        for (int i = 0; i < 3; ++i)
          H[j][q] += w.u[i][q] * (mu * nu *
                                  (w.g[i][j][q] + w.g[j][i][q] - (i == j ? 2.0 / 3.0 * div : 0.0)));
    }
  }
  for (int k = 0; k < G.n[2]; ++k)
    for (int jy = 0; jy < G.n[1]; ++jy)
      for (int ix = 0; ix < G.n[0]; ++ix) {
        const size_t q = G.idx(ix, jy, k);
        double u[3], g[3][3];
        for (int i = 0; i < 3; ++i) u[i] = w.u[i][q];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) g[i][j] = w.g[i][j][q];

        // --- skew-symmetric convective term, eq. (12), P:271-274:
        //     d/dx_j[rho phi u_j] -> 1/2 ( D_j(rho phi u_j) + u_j D_j(rho phi)
        //                                  + rho phi D_j u_j ),   summed over j
        double conv[5];
        for (int f = 0; f < 5; ++f) {
          const double* s = s_of[f];
          double c = 0.0;
          for (int j = 0; j < 3; ++j) {
            const double flux = D1prod(G, s, s_par[f], w.u[j].data(), odd_in(j), ix, jy, k, j);
            const double adv = u[j] * D1(G, s, ix, jy, k, j, s_par[f]);
            const double dil = s[q] * g[j][j];
            c += 0.5 * (flux + adv + dil);
          }
          conv[f] = c;
        }

        // --- stress tensor, eq. (8), times the viscosity mu(T) (1, D-3,
        //     or Sutherland, D-26):
        //     tau_ij = (mu/Re)(du_i/dx_j + du_j/dx_i - 2/3 delta_ij du_k/dx_k)
        double div = 0.0;
        for (int kk = 0; kk < 3; ++kk) div += g[kk][kk];
        const double mu = ph.mu(w.T[q]);
        double sij[3][3], tau[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            sij[i][j] = g[i][j] + g[j][i] - (i == j ? 2.0 / 3.0 * div : 0.0);
            tau[i][j] = mu * nu * sij[i][j];
          }
        // d mu / dx_j by the chain rule mu'(T) D_j T (D-26); zero for mu == 1
        double dmu[3] = {0.0, 0.0, 0.0};
        if (ph.visc_law != 0)
          for (int j = 0; j < 3; ++j) dmu[j] = ph.dmu(w.T[q]) * D1(G, w.T.data(), ix, jy, k, j);

        // --- d tau_ij / dx_j, expanded term by term:
        //   nu [ d2u_i/dx_j dx_j  +  d/dx_j(du_j/dx_i)  -  2/3 d/dx_i(du_k/dx_k) ]
        // same-direction second derivatives use the second-derivative stencil
        // (P:274); different-direction ones are nested, inner first.
        double V[3];
        for (int i = 0; i < 3; ++i) {
          double lap = 0.0;
          for (int j = 0; j < 3; ++j) lap += D2(G, w.u[i].data(), ix, jy, k, j, odd_in(i));
          double cross = 0.0;  // sum_j d/dx_j (du_j/dx_i)
          for (int j = 0; j < 3; ++j) {
            if (j == i) cross += D2(G, w.u[i].data(), ix, jy, k, i, odd_in(i));
            else cross += D1(G, w.g[j][i].data(), ix, jy, k, j, g_par[j][i]);
          }
          double graddiv = 0.0;  // d/dx_i (du_k/dx_k)
          for (int kk = 0; kk < 3; ++kk) {
            if (kk == i) graddiv += D2(G, w.u[i].data(), ix, jy, k, i, odd_in(i));
            else graddiv += D1(G, w.g[kk][kk].data(), ix, jy, k, i, g_par[kk][kk]);
          }
          // d/dx_j (mu S_ij) = mu dS_ij/dx_j + (d mu/dx_j) S_ij   (product rule, D-26)
          double gradmu = 0.0;
          for (int j = 0; j < 3; ++j) gradmu += dmu[j] * sij[i][j];
          V[i] = nu * (mu * (lap + cross - 2.0 / 3.0 * graddiv) + gradmu);
        }

        // --- continuity, eq. (5)
        R[0 * N + q] = -conv[0];
        // --- momentum, eq. (6): - d/dx_j[rho u_i u_j + p delta_ij - tau_ij]
        for (int i = 0; i < 3; ++i)
          R[(1 + i) * N + q] = -conv[1 + i] - D1(G, w.p.data(), ix, jy, k, i) + V[i];
        // --- energy, eq. (7): - d/dx_j[rho E u_j + u_j p - q_j - u_i tau_ij]
        //     q_j = kappa dT/dx_j (eq. 9), its divergence by D_jj;
        //     d/dx_j(u_i tau_ij) = tau_ij du_i/dx_j + u_i dtau_ij/dx_j (product rule, D-5)
        //     with mu(T): d/dx_j(mu dT/dx_j) = mu D_jj T + (d mu/dx_j) D_j T (D-26)
        //     energy_form 1: d/dx_j(u_i tau_ij) = D_j H_j (N2, D-27)
        double pu = 0.0, heat = 0.0, work = 0.0, uv = 0.0;
        for (int j = 0; j < 3; ++j) {
          pu += D1prod(G, w.p.data(), EVEN, w.u[j].data(), odd_in(j), ix, jy, k, j);
          heat += mu * D2(G, w.T.data(), ix, jy, k, j);
          if (ph.visc_law != 0) heat += dmu[j] * D1(G, w.T.data(), ix, jy, k, j);
        }
        if (ph.energy_form == 1) {
          for (int j = 0; j < 3; ++j) work += D1(G, H[j].data(), ix, jy, k, j, odd_in(j));
        } else {
          for (int i = 0; i < 3; ++i) {
            for (int j = 0; j < 3; ++j) work += tau[i][j] * g[i][j];
            uv += u[i] * V[i];
          }
        }
        R[4 * N + q] = -conv[4] - pu + kap * heat + work + uv;
      }
}

// Volume integrals, normalised by rho_ref * Omega; rectangle rule
// on the periodic grid, i.e. the mean over the points (D-11).  Neumaier sums.
struct Acc {
  double s = 0.0, c = 0.0;
  void add(double x) {
    const double t = s + x;
    if (std::fabs(s) >= std::fabs(x)) c += (s - t) + x;
    else c += (x - t) + s;
    s = t;
  }
  double val() const { return s + c; }
};

void diagnostics(const Grid& G, const Phys& ph, const double* Q, double out[3]) {
  const size_t N = G.npts();
  Work w;
  formulas(G, ph, Q, w);
  velocity_gradients(G, w);
  const double nu = ph.nu();
  Acc ek, ens, dis;
  for (size_t q = 0; q < N; ++q) {
    const double rho = Q[q];
    double uu = 0.0;
    for (int j = 0; j < 3; ++j) uu += w.u[j][q] * w.u[j][q];
    ek.add(0.5 * rho * uu);  // eq. (17): 1/2 rho u_j u_j
    // eq. (18): omega_i = eps_ijk du_k/dx_j
    double om2 = 0.0;
    for (int i = 0; i < 3; ++i) {
      double om = 0.0;
      for (int j = 0; j < 3; ++j)
        for (int kk = 0; kk < 3; ++kk) {
          int eps = 0;
          if (i != j && j != kk && i != kk) eps = ((j - i + 3) % 3 == 1) ? 1 : -1;
          if (eps != 0) om += eps * w.g[kk][j][q];
        }
      om2 += om * om;
    }
    ens.add(0.5 * rho * om2);
    // D-12: viscous dissipation rate tau_ij du_i/dx_j (tau with mu(T), D-26)
    double div = w.g[0][0][q] + w.g[1][1][q] + w.g[2][2][q];
    const double mu = ph.mu(w.T[q]);
    double phi = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        const double tau =
            mu * nu * (w.g[i][j][q] + w.g[j][i][q] - (i == j ? 2.0 / 3.0 * div : 0.0));
        phi += tau * w.g[i][j][q];
      }
    dis.add(phi);
  }
  out[0] = ek.val() / (double)N;
  out[1] = ens.val() / (double)N;
  out[2] = dis.val() / (double)N;
}

// Low-storage RK3, Williamson (1980) 2N coefficients in the Carpenter &
// Kennedy (1994) 2N form (reading D-1):
//   per stage s: W <- A_s W + dt R(Q);  Q <- Q + B_s W
const double RK_A[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};
const double RK_B[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
// The two-register ("SBLI") form of a third-order RK (SURVEY §8(c) row 1, §8(f)
// N2; D-25), per stage s, with Q_old = Q at the start of the step:
//   R = R(Q);  Q <- Q_old + alpha_s dt R;  Q_old <- Q_old + beta_s dt R
const double RK2R_ALPHA[3] = {2.0 / 3.0, 5.0 / 12.0, 3.0 / 5.0};
const double RK2R_BETA[3] = {1.0 / 4.0, 3.0 / 20.0, 3.0 / 5.0};

}  // namespace

// =============================================================================
// C entry points (ctypes).  Return 0 on success, negative on bad arguments.
// =============================================================================
extern "C" {

struct oracle_params {
  int nx, ny, nz, order;
  double dx, dt, Re, Pr, Minf, gamma;
  int sym[3];       // 1: symmetry boundaries in direction d, 0: periodic
  int energy_form;  // 0: expanded viscous work (D-5); 1: conservative D_j(u_i tau_ij) (D-27)
  int visc_law;     // 0: mu == 1 (D-3); 1: Sutherland mu(T) (D-26)
  double suth;      // Sutherland S / T_ref (visc_law 1)
};

static bool make_phys(const oracle_params* P, Phys& ph) {
  ph = Phys{P->Re, P->Pr, P->Minf, P->gamma};
  if (P->energy_form < 0 || P->energy_form > 1 || P->visc_law < 0 || P->visc_law > 1)
    return false;
  if (P->visc_law == 1 && !(P->suth > 0.0)) return false;
  ph.energy_form = P->energy_form;
  ph.visc_law = P->visc_law;
  ph.suth = P->suth;
  return true;
}

static bool make_grid(const oracle_params* P, Grid& G) {
  if (!P || P->nx < 1 || P->ny < 1 || P->nz < 1) return false;
  if (!(P->dx > 0.0)) return false;
  std::vector<Frac> a, b;
  if (!central_weights(P->order, a, b)) return false;
  G.n[0] = P->nx;
  G.n[1] = P->ny;
  G.n[2] = P->nz;
  for (int d = 0; d < 3; ++d) G.sym[d] = P->sym[d] ? 1 : 0;
  G.dx = P->dx;
  G.m = P->order / 2;
  G.a.clear();
  G.b.clear();
  for (auto& f : a) G.a.push_back(f.to_double());
  for (auto& f : b) G.b.push_back(f.to_double());
  return true;
}

// Weights as exact fractions: num/den arrays; a: m entries (a_1..a_m),
// b: m+1 entries (b_0..b_m).
int oracle_weights_exact(int order, long long* a_num, long long* a_den, long long* b_num,
                         long long* b_den) {
  std::vector<Frac> a, b;
  if (!central_weights(order, a, b)) return -1;
  for (size_t k = 0; k < a.size(); ++k) { a_num[k] = (long long)a[k].n; a_den[k] = (long long)a[k].d; }
  for (size_t k = 0; k < b.size(); ++k) { b_num[k] = (long long)b[k].n; b_den[k] = (long long)b[k].d; }
  return 0;
}

// Apply one derivative operator to a scalar grid function f [nz][ny][nx].
// kind: 1 = D_dir, 2 = D_dir,dir ; for kind 3, out = D_dir( D_dir2 f ) (nested).
int oracle_derivative(const oracle_params* P, const double* f, int kind, int dir, int dir2,
                      double* out) {
  Grid G;
  if (!make_grid(P, G) || dir < 0 || dir > 2) return -1;
  const size_t N = G.npts();
  std::vector<double> inner;
  if (kind == 3) {
    if (dir2 < 0 || dir2 > 2) return -1;
    inner.assign(N, 0.0);
    for (int k = 0; k < G.n[2]; ++k)
      for (int j = 0; j < G.n[1]; ++j)
        for (int i = 0; i < G.n[0]; ++i) inner[G.idx(i, j, k)] = D1(G, f, i, j, k, dir2);
  }
  for (int k = 0; k < G.n[2]; ++k)
    for (int j = 0; j < G.n[1]; ++j)
      for (int i = 0; i < G.n[0]; ++i) {
        double v;
        if (kind == 1) v = D1(G, f, i, j, k, dir);
        else if (kind == 2) v = D2(G, f, i, j, k, dir);
        else if (kind == 3) v = D1(G, inner.data(), i, j, k, dir);
        else return -1;
        out[G.idx(i, j, k)] = v;
      }
  return 0;
}

int oracle_residual(const oracle_params* P, const double* Q, double* R) {
  Grid G;
  if (!make_grid(P, G)) return -1;
  Phys ph;
  if (!make_phys(P, ph)) return -1;
  residual(G, ph, Q, R);
  return 0;
}

// scheme 0 = forward Euler, 1 = RK3 (2N), 2 = RK3 (two-register form).
// Q is advanced in place by nsteps.
int oracle_step(const oracle_params* P, double* Q, int scheme, int nsteps) {
  Grid G;
  if (!make_grid(P, G) || scheme < 0 || scheme > 2 || nsteps < 0) return -1;
  Phys ph;
  if (!make_phys(P, ph)) return -1;
  const size_t n5 = 5 * G.npts();
  std::vector<double> R(n5), W(n5, 0.0);
  for (int it = 0; it < nsteps; ++it) {
    if (scheme == 0) {
      residual(G, ph, Q, R.data());
      for (size_t q = 0; q < n5; ++q) Q[q] = Q[q] + P->dt * R[q];
    } else if (scheme == 2) {
      std::vector<double> Qold(Q, Q + n5);
      for (int s = 0; s < 3; ++s) {
        residual(G, ph, Q, R.data());
        for (size_t q = 0; q < n5; ++q) {
          Q[q] = Qold[q] + RK2R_ALPHA[s] * (P->dt * R[q]);
          Qold[q] = Qold[q] + RK2R_BETA[s] * (P->dt * R[q]);
        }
      }
    } else {
      for (int s = 0; s < 3; ++s) {
        // periodic halos are refreshed before every stage (D-10): the
        // stencils below read the current stage's Q through periodic wrap.
        residual(G, ph, Q, R.data());
        for (size_t q = 0; q < n5; ++q) {
          W[q] = RK_A[s] * W[q] + P->dt * R[q];
          Q[q] = Q[q] + RK_B[s] * W[q];
        }
      }
    }
  }
  return 0;
}

int oracle_diagnostics(const oracle_params* P, const double* Q, double* out3) {
  Grid G;
  if (!make_grid(P, G)) return -1;
  Phys ph;
  if (!make_phys(P, ph)) return -1;
  diagnostics(G, ph, Q, out3);
  return 0;
}

// Diagnostics after each of nsteps steps (row 0 = initial state):
// series[(n)*3 + c], n = 0..nsteps.  Q is advanced in place.
int oracle_run_series(const oracle_params* P, double* Q, int scheme, int nsteps,
                      double* series) {
  if (oracle_diagnostics(P, Q, series) != 0) return -1;
  for (int n = 1; n <= nsteps; ++n) {
    if (oracle_step(P, Q, scheme, 1) != 0) return -1;
    if (oracle_diagnostics(P, Q, series + 3 * n) != 0) return -1;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Scalar advection-diffusion of the paper's verification cases:
//   d phi/dt + d/dx_j [ phi u_j - k d phi/dx_j ] + S = 0
// with constant u_j and k; the 1D wave is u = (c,0,0), k = 0, S = 0.
// Conservative derivative of the product phi u_j (Conservative), the
// Laplacian by the second-derivative stencil (P:274's rule), S optional.
// ---------------------------------------------------------------------------
static void scalar_residual(const Grid &G, const double u[3], double kd, const double *phi,
                            const double *S, double *R) {
  std::vector<double> uj[3];
  for (int j = 0; j < 3; ++j) uj[j].assign(G.npts(), u[j]);
  for (int k = 0; k < G.n[2]; ++k)
    for (int jy = 0; jy < G.n[1]; ++jy)
      for (int ix = 0; ix < G.n[0]; ++ix) {
        const size_t q = G.idx(ix, jy, k);
        double adv = 0.0, lap = 0.0;
        for (int j = 0; j < 3; ++j) {
          adv += D1prod(G, phi, EVEN, uj[j].data(), EVEN, ix, jy, k, j);
          lap += D2(G, phi, ix, jy, k, j);
        }
        R[q] = -adv + kd * lap - (S ? S[q] : 0.0);
      }
}

int oracle_scalar_residual(const oracle_params *P, const double *u3, double kd, const double *phi,
                           const double *S, double *R) {
  Grid G;
  if (!make_grid(P, G) || !u3 || !phi || !R) return -1;
  scalar_residual(G, u3, kd, phi, S, R);
  return 0;
}

// scheme 0 = forward Euler, 1 = RK3 (2N, D-1), 2 = RK3 (two-register form, D-25);
// phi advanced in place.
int oracle_scalar_step(const oracle_params *P, const double *u3, double kd, const double *S,
                       double *phi, int scheme, int nsteps) {
  Grid G;
  if (!make_grid(P, G) || !u3 || !phi || scheme < 0 || scheme > 2 || nsteps < 0) return -1;
  const size_t N = G.npts();
  std::vector<double> R(N), W(N, 0.0);
  for (int it = 0; it < nsteps; ++it) {
    if (scheme == 0) {
      scalar_residual(G, u3, kd, phi, S, R.data());
      for (size_t q = 0; q < N; ++q) phi[q] = phi[q] + P->dt * R[q];
    } else if (scheme == 2) {
      std::vector<double> old(phi, phi + N);
      for (int s = 0; s < 3; ++s) {
        scalar_residual(G, u3, kd, phi, S, R.data());
        for (size_t q = 0; q < N; ++q) {
          phi[q] = old[q] + RK2R_ALPHA[s] * (P->dt * R[q]);
          old[q] = old[q] + RK2R_BETA[s] * (P->dt * R[q]);
        }
      }
    } else {
      for (int s = 0; s < 3; ++s) {
        scalar_residual(G, u3, kd, phi, S, R.data());
        for (size_t q = 0; q < N; ++q) {
          W[q] = RK_A[s] * W[q] + P->dt * R[q];
          phi[q] = phi[q] + RK_B[s] * W[q];
        }
      }
    }
  }
  return 0;
}

}  // extern "C"
