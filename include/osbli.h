/*
 * osbli.h — C ABI of the B200-native OpenSBLI hot path (libosbli.so).
 *
 * The operation behind this boundary is the explicit time integration of the
 * 3D compressible Navier-Stokes equations of Jacobs, Jammy & Sandham,
 * "OpenSBLI ..." (arXiv 1609.01277), as the paper's generated solver performs
 * it (PAPER.md; "P:n" = line n):
 *   - equations (5)-(9): mass, momentum, energy, stress tensor
 *     tau_ij, heat flux q_j, non-dimensional, constant viscosity (mu = 1) or
 *     Sutherland's mu(T) (osbli_set_viscosity);
 *   - equation of state and total energy (10)-(11), P:259-266;
 *   - skew-symmetric convective terms (12), with phi = 1, u_i, E;
 *     viscous Laplacians by second-derivative stencils, P:274;
 *     nested derivatives evaluated inner first, P:98;
 *   - central differences of arbitrary even order, P:123;
 *   - forward Euler or a 3-stage low-storage RK3 (2N or two-register)
 *     and P:164;
 *   - periodic boundaries in every direction, or symmetry
 *     boundaries per direction (osbli_set_boundary);
 *   - optional steady source term (osbli_set_source, the manufactured-solution
 *     construction of P:196) and the paper's scalar advection-diffusion
 *     verification equation (osbli_scalar_*);
 *   - volume-averaged kinetic energy and enstrophy, plus the viscous
 *     dissipation rate (reading D-12).
 * DESIGN.md §3 lists every reading of a point the paper leaves open.
 *
 * Layout of every state array crossing this boundary: fp64, [5][nz][ny][nx],
 * x fastest; field order (rho, rho*u, rho*v, rho*w, rho*E).  In distributed mode
 * nz is this rank's slab (osbli_local_box).  Grid point (i,j,k) sits at
 * (i*dx, j*dx, k*dx); the periodic box is nx*dx x ny*dx x (global nz)*dx.
 *
 * Ownership: the library owns all device memory it allocates (state ping-pong
 * buffers, RK register, scratch, NCCL communicator).  Caller pointers are only
 * read or written during the call and never retained.  Device pointers must be
 * on the handle's device.
 *
 * Synchronisation: osbli_step only enqueues work on the handle's stream and
 * returns; set_state/get_state/diagnostics/residual/sync complete before they
 * return.  A non-finite value produced by a step is reported (OSBLI_E_NONFINITE)
 * by the next synchronising call.
 *
 * Errors: every int-returning call returns OSBLI_OK (0) or a negative status;
 * no exception or abort crosses the ABI.  After OSBLI_E_CUDA, OSBLI_E_COMM or
 * OSBLI_E_NONFINITE the handle is poisoned: only get_state, last_error and
 * destroy remain valid (others return OSBLI_E_STATE).
 */
#ifndef OSBLI_H
#define OSBLI_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct osbli_ctx osbli_ctx;

/* Boundary conditions per direction: periodic (default), or symmetry at
 * both ends of the direction: the halo mirrors the interior about the boundary
 * face, scalars even, the momentum component normal to the face odd. */
enum { OSBLI_BC_PERIODIC = 0, OSBLI_BC_SYMMETRY = 1 };

/* Viscosity law ("viscosity can be treated either as a
 * constant or as a spatially-varying term"; D-26): constant mu = 1
 * (default, D-3), or Sutherland's law in dimensionless form,
 * mu(T) = T^1.5 (1 + S)/(T + S) with S the Sutherland constant over the
 * reference temperature (e.g. 110.4 K / 288 K). */
enum { OSBLI_VISC_CONSTANT = 0, OSBLI_VISC_SUTHERLAND = 1 };

/* Form of the viscous work d/dx_j(u_i tau_ij) in the energy equation (SURVEY
 * §8(f) N2; D-5, D-27): product-rule expanded tau_ij g_ij + u_i V_i
 * (default), or conservative, the first-derivative stencil of the pointwise
 * flux H_j = u_i tau_ij, which conserves total energy to round-off. */
enum { OSBLI_ENERGY_EXPANDED = 0, OSBLI_ENERGY_CONSERVATIVE = 1 };

/* Time schemes: forward Euler, the 3-stage 2N-storage RK3
 * (Williamson coefficients in Carpenter-Kennedy 2N form; D-1), and
 * the two-register ("SBLI") third-order RK: per stage Q <- Q_old + alpha_s dt R,
 * Q_old <- Q_old + beta_s dt R, alpha = (2/3, 5/12, 3/5), beta = (1/4, 3/20, 3/5)
 * (D-25).  Same storage and traffic as OSBLI_RK3. */
enum { OSBLI_EULER = 0, OSBLI_RK3 = 1, OSBLI_RK3_2R = 2 };

enum {
  OSBLI_OK = 0,
  OSBLI_E_INVAL = -1,       /* invalid argument                                  */
  OSBLI_E_UNSUPPORTED = -2, /* valid but not built (order > 12)                  */
  OSBLI_E_NOMEM = -3,       /* device allocation failed                          */
  OSBLI_E_CUDA = -4,        /* CUDA runtime error (text in osbli_last_error)     */
  OSBLI_E_COMM = -5,        /* NCCL error                                        */
  OSBLI_E_NONFINITE = -6,   /* a step produced NaN/Inf                           */
  OSBLI_E_STATE = -7        /* handle poisoned by an earlier error               */
};

/* Diagnostics at the current time t = step*dt (D-11/D-12):
 * means over all grid points (rectangle rule on the periodic box, rho_ref = 1):
 *   kinetic_energy = <1/2 rho u_j u_j>, enstrophy = <1/2 rho |curl u|^2>,
 *   dissipation    = <tau_ij du_i/dx_j>, derivatives by the solver's stencils. */
typedef struct {
  double t;
  long long step;
  double kinetic_energy, enstrophy, dissipation;
} osbli_diag;

/* Create a single-GPU solver on the current CUDA device.
 * The problem statement of the paper's solver: a grid of N points per
 * direction with spacing dx (x_i = i dx; reading D-9), central
 * differences of the given even order, the non-dimensional parameters
 * Re, Pr, Minf, gamma of equations (5)-(11) (TGV values P:290), the
 * time step dt and the time scheme.
 *   nx,ny,nz >= 1 grid points; order even, 2..12 (else INVAL / UNSUPPORTED);
 *   dx > 0 isotropic spacing; dt > 0 time step;
 *   Re > 0 (Re = +INFINITY means inviscid: nu = kappa = 0); Pr > 0; Minf > 0;
 *   gamma > 1; scheme OSBLI_EULER, OSBLI_RK3 or OSBLI_RK3_2R.
 * The state is zero until osbli_set_state.  *out receives the handle. */
int osbli_create(int nx, int ny, int nz, int order, double dx, double dt, double Re, double Pr,
                 double Minf, double gamma, int scheme, osbli_ctx **out);

/* Create one rank of a z-slab decomposition over nranks GPUs (one process per
 * GPU).  nz is the GLOBAL size; rank r owns a contiguous slab of near-equal
 * size (osbli_local_box), each at least order/2 planes.  nccl_unique_id points
 * to the 128-byte ncclUniqueId produced by osbli_nccl_unique_id on rank 0 and
 * broadcast by the caller.  The CUDA device must be set by the caller. */
int osbli_create_dist(int nx, int ny, int nz, int order, double dx, double dt, double Re,
                      double Pr, double Minf, double gamma, int scheme, int rank, int nranks,
                      const void *nccl_unique_id, osbli_ctx **out);

/* Fill 128 bytes at id_out with a fresh ncclUniqueId (rank 0 only). */
int osbli_nccl_unique_id(void *id_out);

/* Host-only helpers of the slab decomposition (no device needed).
 * osbli_slab_bounds: planes [*z0, *z0 + *nz_local) of `rank` when nz planes are
 *   split over nranks (near-equal; the first nz % nranks ranks get one more).
 * osbli_ghost_plan: the two ghost transfers of one stage, m planes each, in
 *   local plane indices (interior 0..nz_local-1, ghosts -m..-1, nz_local..):
 *   plan[4t+0] send peer, plan[4t+1] first plane sent, plan[4t+2] receive peer,
 *   plan[4t+3] first ghost plane received, for t = 0, 1.  Every rank posts the
 *   transfers in this order; rank r's transfer t send matches its peer's
 *   transfer t receive. */
int osbli_slab_bounds(int nz, int nranks, int rank, int *z0, int *nz_local);
int osbli_ghost_plan(int rank, int nranks, int nz_local, int m, int *plan);
/* The plan with symmetry boundaries in z (symz != 0): the transfers across the
 * periodic wrap get peer -1 (no send / no receive); the ghost planes they would
 * have filled are the mirrored own planes, rho u_z negated. */
int osbli_ghost_plan_sym(int rank, int nranks, int nz_local, int m, int symz, int *plan);

/* Single-GPU test transport: create nslabs handles (out[0..nslabs-1]) that
 * split nz exactly like osbli_create_dist and exchange ghost planes by device
 * copies instead of NCCL, on one shared stream.  They run the distributed
 * (ghost-plane) kernel path; advance them together with osbli_loopback_step
 * (osbli_step on a member returns OSBLI_E_INVAL).  set_state/get_state/
 * residual/diagnostics work per member (diagnostics gather all members). */
int osbli_create_loopback(int nx, int ny, int nz, int order, double dx, double dt, double Re,
                          double Pr, double Minf, double gamma, int scheme, int nslabs,
                          osbli_ctx **out);
int osbli_loopback_step(osbli_ctx **hs, int nslabs, int n);

/* Stage schedule of a slab handle (halo exchange per stage, P:141,
 * P:149).  Only the m planes next to each slab face need the neighbours' planes:
 *   OSBLI_SLAB_PLAIN   exchange the ghost planes, then the z-pass and the xy-pass;
 *   OSBLI_SLAB_ZSPLIT  the exchange runs on a second stream behind the interior
 *                      z-pass; the z-pass of the 2m face planes follows it;
 *   OSBLI_SLAB_XYSPLIT the xy-pass writes the face planes of the new state first;
 *                      their exchange runs behind the interior xy-pass and the
 *                      next stage waits for it.
 * Default: XYSPLIT when the slab has neighbours (nranks > 1 or a loopback group),
 * PLAIN for one rank; OSBLI_SLAB_OVERLAP=0/1/2 in the environment at create time
 * overrides the default.  Results are bitwise the same in every schedule.  No
 * effect on single-domain handles; INVAL for other values. */
enum { OSBLI_SLAB_PLAIN = 0, OSBLI_SLAB_ZSPLIT = 1, OSBLI_SLAB_XYSPLIT = 2 };
int osbli_set_slab_schedule(osbli_ctx *h, int schedule);

/* Slab owned by this rank: global planes [*z0, *z0 + *nz_local). */
int osbli_local_box(const osbli_ctx *h, int *z0, int *nz_local);

/* Use this CUDA stream (cudaStream_t, e.g. torch.cuda.current_stream().cuda_stream)
 * for all subsequent work; NULL selects the library's own stream. */
int osbli_set_stream(osbli_ctx *h, void *cuda_stream);

/* Copy the conservative state in / out: Q = (rho, rho u, rho v, rho w, rho E),
 * the variables the paper's equations (5)-(7) advance (rho E by the
 * total-energy relation (11)).  q is [5][nz_local][ny][nx] fp64, on
 * the host (on_device = 0) or on the handle's device (on_device = 1).
 * set_state resets the RK register and the step counter.  Errors: INVAL for a
 * NULL q, CUDA for a failed copy (the handle is then poisoned); get_state stays
 * valid on a poisoned handle and returns its last state. */
int osbli_set_state(osbli_ctx *h, const double *q, int on_device);
int osbli_get_state(osbli_ctx *h, double *q, int on_device);

/* Stream-ordered forms of the two copies: enqueued on the handle's stream and
 * returned from at once (no synchronisation).  Host buffers should be pinned
 * (page-locked), or the copy is not asynchronous; the caller keeps q alive and
 * unchanged (set) or unread (get) until the stream has passed the copy
 * (osbli_sync, or any event recorded after it).  Used to overlap the host
 * copies of several handles with each other's steps. */
int osbli_set_state_async(osbli_ctx *h, const double *q, int on_device);
int osbli_get_state_async(osbli_ctx *h, double *q, int on_device); /* valid when poisoned */

/* Advance n >= 0 full time steps: forward Euler, or the paper's 3-stage
 * low-storage RK3 loop, each stage refreshing the periodic (or
 * symmetry) halos (reading D-10), evaluating the residual of equations
 * (5)-(12) and updating the state.  Stream-ordered: returns after
 * enqueueing; a non-finite value is reported by the next synchronising call.
 * Errors: INVAL for n < 0, STATE on a poisoned handle, CUDA / COMM for launch
 * or NCCL failures. */
int osbli_step(osbli_ctx *h, int n);

/* Advance n >= 0 steps like osbli_step and return the diagnostics of the state
 * at the start of every step: series[k] (k = 0..n-1) describes the state after
 * step_count + k steps (t = that times dt), the same quantities as
 * osbli_diagnostics, fused into each step's first xy-pass, which has
 * every velocity gradient of that state in hand (per-(plane, tile) partials in a
 * fixed order, planes summed in global z order: independent of the slab
 * decomposition, within round-off of osbli_diagnostics, whose tiling differs).
 * The state after the last step is not included (osbli_diagnostics gives it).
 * Synchronises every 64 steps; collective when distributed (like
 * osbli_diagnostics, including the non-finite check).  series must hold n
 * entries.  INVAL on loopback slabs. */
int osbli_step_diag(osbli_ctx *h, int n, osbli_diag *series);

/* Diagnostics of the current state (collective over ranks when
 * distributed: every rank gets the same, decomposition-independent numbers, and
 * every rank returns OSBLI_E_NONFINITE if any rank's state went non-finite). */
int osbli_diagnostics(osbli_ctx *h, osbli_diag *out);

/* Boundary condition of direction dir (0 = x, 1 = y, 2 = z), both ends; takes
 * effect at the next stage.  On slab-decomposed handles symmetry in z must be
 * set on every rank: the outer slabs then mirror their own planes instead of
 * exchanging across the periodic wrap. */
int osbli_set_boundary(osbli_ctx *h, int dir, int bc);

/* Viscosity law (OSBLI_VISC_*); suth = S/T_ref > 0 for Sutherland (ignored for
 * the constant law).  Takes effect at the next stage; allocates nz*nx*ny doubles
 * of device scratch for Sutherland.  Diagnostics use the same mu(T). */
int osbli_set_viscosity(osbli_ctx *h, int law, double suth);

/* Energy-equation form of the viscous work (OSBLI_ENERGY_*).  The conservative
 * form adds one kernel per stage and about 4*nz*nx*ny doubles of device scratch;
 * on slab-decomposed handles it also exchanges the flux's ghost planes every
 * stage, and osbli_residual returns OSBLI_E_UNSUPPORTED there. */
int osbli_set_energy_form(osbli_ctx *h, int form);

/* Steady source term S added to the right-hand side, dQ/dt = R(Q) + S (the
 * method of manufactured solutions).  S is
 * [5][nz_local][ny][nx] on the host or the device; NULL removes it.  The
 * library keeps its own copy. */
int osbli_set_source(osbli_ctx *h, const double *S, int on_device);

/* Test hook: dQ/dt = R(Q) (+ S if set) of the current state, the semi-discrete
 * right-hand side of equations (5)-(9) in the skew-symmetric form (12) with the
 * expanded viscous terms (D-4, D-5), [5][nz_local][ny][nx],
 * on the host or the device; no update.  Synchronous. */
int osbli_residual(osbli_ctx *h, double *R, int on_device);

/* Wait for queued work; surfaces asynchronous errors (NONFINITE, CUDA).  On a
 * distributed handle the non-finite check is collective (every rank must call
 * it; all return NONFINITE if any rank's state went non-finite), so that the
 * ranks refuse their next step together.  A CUDA or NCCL error aborts the
 * rank's communicator. */
int osbli_sync(osbli_ctx *h);

/* Instrumentation.  When enabled, osbli_step brackets every z-pass and xy-pass
 * launch with CUDA events on the handle's stream; osbli_kernel_timing waits for
 * them and returns the summed durations (ms) and launch counts since the last
 * call (then resets).  Disabled by default. */
int osbli_set_kernel_timing(osbli_ctx *h, int enable);
int osbli_kernel_timing(osbli_ctx *h, double *zpass_ms, double *xypass_ms, long long *n_zpass,
                        long long *n_xypass);

/* Number of kernels this handle launched since creation (instrumentation). */
long long osbli_kernel_launches(const osbli_ctx *h);

/* Last error text for h; h == NULL gives the calling thread's last create error. */
const char *osbli_last_error(const osbli_ctx *h);

/* Library build string: "osbli <version> sm_100a orders 2..12". */
const char *osbli_version(void);

void osbli_destroy(osbli_ctx *h);

/* ---------------------------------------------------------------------------
 * Scalar advection-diffusion, the equation of the paper's verification cases
 * (1D wave P:176-184, 2D manufactured solution P:195-209):
 *     d phi/dt + d/dx_j [ phi u_j - kappa d phi/dx_j ] + S = 0
 * with constant (u0, u1, u2) and kappa >= 0, on the same periodic grid, central
 * differences (order 2..12), Euler or RK3.  phi and S are [nz][ny][nx] fp64.
 * Same error codes and conventions as the NS handle. */
typedef struct osbli_scalar osbli_scalar;
int osbli_scalar_create(int nx, int ny, int nz, int order, double dx, double dt, double u0,
                        double u1, double u2, double kappa, int scheme, osbli_scalar **out);
int osbli_scalar_set_stream(osbli_scalar *h, void *cuda_stream); /* NULL: own stream */
int osbli_scalar_set_state(osbli_scalar *h, const double *phi, int on_device);
int osbli_scalar_set_source(osbli_scalar *h, const double *S, int on_device); /* NULL: none */
int osbli_scalar_get_state(osbli_scalar *h, double *phi, int on_device);
int osbli_scalar_step(osbli_scalar *h, int n);
int osbli_scalar_residual(osbli_scalar *h, double *R, int on_device); /* d phi/dt */
int osbli_scalar_sync(osbli_scalar *h);
const char *osbli_scalar_last_error(const osbli_scalar *h);
void osbli_scalar_destroy(osbli_scalar *h);

#ifdef __cplusplus
}
#endif
#endif /* OSBLI_H */
