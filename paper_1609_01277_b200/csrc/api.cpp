// =============================================================================
// C ABI + runtime of the B200-native OpenSBLI hot path (see include/osbli.h).
//
// Owns the device buffers of one handle, sequences the stages of the time
// scheme, exchanges z ghost planes between ranks over NCCL
// (slab decomposition) and reduces the diagnostics
// deterministically (per-plane partials summed in global plane order).
// =============================================================================
#include "../../include/osbli.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "kernels.h"
#include "weights.h"

using osbli::Bufs;
using osbli::KParams;

struct LoopGroup {
  std::vector<osbli_ctx *> members;
  std::vector<cudaStream_t> streams;  // every member's own stream, destroyed with the group
  int live = 0;
  bool broken = false;  // a member was destroyed: the others can no longer exchange
};
static std::vector<cudaStream_t> &g_loop_streams(LoopGroup *g) { return g->streams; }

struct osbli_ctx {
  int nx = 0, ny = 0, nz_global = 0, nz = 0, z0 = 0, order = 0, m = 0, scheme = 0;
  int rank = 0, nranks = 1;
  bool slab = false;  // distributed (ghost-plane) path: nranks > 1, or one rank over NCCL
  // slab stage schedule (osbli_set_slab_schedule): OSBLI_SLAB_PLAIN, _ZSPLIT, _XYSPLIT
  int overlap = 0;
  bool ghost_async = false;  // the ghost planes of the current Q were posted on comm_stream
  double dx = 0, dt = 0, Re = 0, Pr = 0, Minf = 0, gamma = 0;
  int device = 0;
  cudaStream_t stream = nullptr, own_stream = nullptr;
  Bufs b{};
  double *scratch = nullptr;  // diagnostics per-(plane, tile) partials
  double *nccl_part = nullptr;  // [nranks * max_nz][3] gathered plane partials
  unsigned int *flag_all = nullptr;  // max of the ranks' non-finite flags (device)
  // fused diagnostics (osbli_step_diag): per-(plane, tile) partials of the stage-1
  // xy-pass, per-step per-plane partials of a batch of steps, and their gather
  double *dtiles = nullptr, *dseries = nullptr, *dseries_all = nullptr;
  double *stage_dpart = nullptr;  // set while a stage 1 should write dtiles
  double *src = nullptr;        // optional source S, plane-major [nz][5][ny][nx]
  double *hflux_alloc = nullptr;  // H_j with ghost planes [nz + 2G][3][ny][nx] (cons form)
  int max_nz = 0;
  int cur = 0;
  long long step_count = 0;
  long long launches = 0;
  bool poisoned = false;
  std::string err;
  ncclComm_t comm = nullptr;
  KParams base{};
  // loopback transport (one GPU, several slabs): the group of sibling handles
  struct LoopGroup *loop = nullptr;
  // NCCL overlap: ghost exchange on comm_stream, ordered by events
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_qready = nullptr;  // boundary planes of the current Q are written
  cudaEvent_t ev_ghost = nullptr;   // ghost planes of the current Q have arrived
  // kernel timing instrumentation: events[3*i..3*i+2] bracket stage i's two kernels
  bool timing = false;
  std::vector<cudaEvent_t> events;
  size_t ev_used = 0;
};

namespace {

// NVTX ranges (SURVEY §5 tracing): every RK stage, its halo exchange, the
// diagnostics reduction.  Header-only NVTX v3: a push/pop costs a few ns when no
// tool is attached; under nsys/ncu the ranges put the host-side sequence
// (exchange -> z-pass -> xy-pass) on the timeline next to the kernels.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

thread_local std::string g_create_error;

int fail(osbli_ctx *h, int code, const std::string &msg) {
  h->err = msg;
  if (code == OSBLI_E_CUDA || code == OSBLI_E_COMM || code == OSBLI_E_NONFINITE) h->poisoned = true;
  // a CUDA or NCCL failure on one rank cannot be agreed on collectively: abort the
  // communicator so that this rank's pending NCCL work is torn down (the peers'
  // next collective fails or hangs until their launcher ends them)
  if ((code == OSBLI_E_CUDA || code == OSBLI_E_COMM) && h->comm) {
    ncclCommAbort(h->comm);
    h->comm = nullptr;
  }
  return code;
}

int cuda_fail(osbli_ctx *h, cudaError_t e, const char *where) {
  return fail(h, OSBLI_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(h, expr)                                          \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return cuda_fail((h), _e, #expr); \
  } while (0)

#define NK(h, expr)                                                                 \
  do {                                                                              \
    ncclResult_t _r = (expr);                                                       \
    if (_r != ncclSuccess)                                                          \
      return fail((h), OSBLI_E_COMM, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
  } while (0)

int validate(int nx, int ny, int nz, int order, double dx, double dt, double Re, double Pr,
             double Minf, double gamma, int scheme, std::string &msg) {
  if (nx < 1 || ny < 1 || nz < 1) { msg = "grid sizes must be >= 1"; return OSBLI_E_INVAL; }
  if (order < 2 || order % 2 != 0) { msg = "order must be even and >= 2"; return OSBLI_E_INVAL; }
  if (!(dx > 0.0) || !std::isfinite(dx)) { msg = "dx must be finite and > 0"; return OSBLI_E_INVAL; }
  if (!(dt > 0.0) || !std::isfinite(dt)) { msg = "dt must be finite and > 0"; return OSBLI_E_INVAL; }
  if (!(Re > 0.0)) { msg = "Re must be > 0 (or +inf)"; return OSBLI_E_INVAL; }
  if (!(Pr > 0.0) || !std::isfinite(Pr)) { msg = "Pr must be > 0"; return OSBLI_E_INVAL; }
  if (!(Minf > 0.0) || !std::isfinite(Minf)) { msg = "Minf must be > 0"; return OSBLI_E_INVAL; }
  if (!(gamma > 1.0) || !std::isfinite(gamma)) { msg = "gamma must be > 1"; return OSBLI_E_INVAL; }
  if (scheme != OSBLI_EULER && scheme != OSBLI_RK3 && scheme != OSBLI_RK3_2R) {
    msg = "scheme must be 0, 1 or 2";
    return OSBLI_E_INVAL;
  }
  if (order > 2 * osbli::kMaxHalf) { msg = "orders above 12 are not built"; return OSBLI_E_UNSUPPORTED; }
  return OSBLI_OK;
}

void free_all(osbli_ctx *h) {
  cudaFree(h->b.q[0]);
  cudaFree(h->b.q[1]);
  cudaFree(h->b.w);
  cudaFree(h->b.gz);
  cudaFree(h->b.flag);
  cudaFree(h->b.diag_part);
  cudaFree(h->scratch);
  cudaFree(h->nccl_part);
  cudaFree(h->flag_all);
  h->flag_all = nullptr;
  cudaFree(h->dtiles);
  cudaFree(h->dseries);
  cudaFree(h->dseries_all);
  h->dtiles = h->dseries = h->dseries_all = nullptr;
  cudaFree(h->src);
  h->src = nullptr;
  cudaFree(h->base.dtz);
  cudaFree(h->hflux_alloc);
  h->hflux_alloc = nullptr;
  h->base.dtz = h->base.hflux = nullptr;
  h->b = Bufs{};
  h->scratch = nullptr;
  h->nccl_part = nullptr;
}

int create_common(osbli_ctx *h) {
  CK(h, cudaGetDevice(&h->device));
  h->m = h->order / 2;
  const int G = h->m;
  const size_t FS = (size_t)h->nx * h->ny;
  const size_t qn = (size_t)(h->nz + 2 * G) * 5 * FS;
  // per-plane diagnostics partials, padded to the largest slab: the distributed
  // path all-gathers max_nz planes from every rank (the tail stays zero)
  const size_t npart = (size_t)3 * (h->max_nz > h->nz ? h->max_nz : h->nz);
  auto alloc = [&](double **p, size_t n) -> cudaError_t {
    return cudaMalloc((void **)p, n * sizeof(double));
  };
  cudaError_t e = cudaSuccess;
  if ((e = alloc(&h->b.q[0], qn)) != cudaSuccess || (e = alloc(&h->b.q[1], qn)) != cudaSuccess ||
      (e = alloc(&h->b.w, (size_t)h->nz * 5 * FS)) != cudaSuccess ||
      (e = alloc(&h->b.gz, (size_t)h->nz * 3 * FS)) != cudaSuccess ||
      (e = alloc(&h->scratch, osbli::diagnostics_scratch(KParams{h->nx, h->ny, h->nz}))) !=
          cudaSuccess ||
      (e = alloc(&h->b.diag_part, npart)) != cudaSuccess ||
      (e = cudaMalloc((void **)&h->b.flag, sizeof(unsigned int))) != cudaSuccess) {
    free_all(h);
    cudaGetLastError();
    h->err = std::string("device allocation failed: ") + cudaGetErrorString(e);
    return OSBLI_E_NOMEM;
  }
  CK(h, cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
  h->stream = h->own_stream;
  CK(h, cudaMemsetAsync(h->b.q[0], 0, qn * sizeof(double), h->stream));
  CK(h, cudaMemsetAsync(h->b.q[1], 0, qn * sizeof(double), h->stream));
  CK(h, cudaMemsetAsync(h->b.w, 0, (size_t)h->nz * 5 * FS * sizeof(double), h->stream));
  CK(h, cudaMemsetAsync(h->b.flag, 0, sizeof(unsigned int), h->stream));
  CK(h, cudaMemsetAsync(h->b.diag_part, 0, npart * sizeof(double), h->stream));

  KParams &p = h->base;
  p = KParams{};
  p.nx = h->nx;
  p.ny = h->ny;
  p.nz = h->nz;
  p.G = G;
  p.zwrap = h->slab ? 0 : 1;
  p.m = h->m;
  double a[osbli::kMaxHalf] = {0}, b[osbli::kMaxHalf + 1] = {0};
  osbli::central_weights(h->m, a, b);
  for (int k = 0; k < h->m; ++k) p.a[k] = a[k] / h->dx;
  for (int k = 0; k <= h->m; ++k) p.b[k] = b[k] / (h->dx * h->dx);
  for (int l = 0; l < h->m; ++l) {
    double c = 0.0;
    for (int k = h->m; k > l; --k) c += b[k];
    p.cb[l] = c / (h->dx * h->dx);
  }
  const bool inviscid = std::isinf(h->Re);
  p.nu = inviscid ? 0.0 : 1.0 / h->Re;
  p.kappa = inviscid ? 0.0 : 1.0 / ((h->gamma - 1.0) * h->Minf * h->Minf * h->Pr * h->Re);
  p.gm1 = h->gamma - 1.0;
  p.gM2 = h->gamma * h->Minf * h->Minf;
  p.dt = h->dt;
  p.dbg = h->b.flag;
  CK(h, cudaStreamSynchronize(h->stream));
  return OSBLI_OK;
}

int check_usable(osbli_ctx *h) {
  if (!h) return OSBLI_E_INVAL;
  if (h->poisoned) return OSBLI_E_STATE;
  return OSBLI_OK;
}

// Near-equal slab partition of nz planes over nranks (z-slab decomposition):
// the first nz % nranks ranks own one extra plane.
void slab_partition(int nz, int nranks, int rank, int *z0, int *nzl) {
  const int base = nz / nranks, extra = nz % nranks;
  *nzl = base + (rank < extra ? 1 : 0);
  *z0 = rank * base + (rank < extra ? rank : extra);
}

// Ghost-plane exchange plan of one rank (periodic ring in z), m planes each:
//   transfer 0: send local planes [0, m)           to the rank below,
//               receive into ghost planes [nzl, nzl+m) from the rank above;
//   transfer 1: send local planes [nzl-m, nzl)     to the rank above,
//               receive into ghost planes [-m, 0)    from the rank below.
// plan = {send_peer, send_plane, recv_peer, recv_plane} x 2 (local plane indices).
// Slab schedule: OSBLI_SLAB_OVERLAP=1 / =0 forces the boundary-first / plain
// schedule; by default the boundary-first one runs whenever the ghost planes come
// from other slabs (nslabs > 1), the plain one for a single rank exchanging with
// itself.  osbli_set_slab_schedule overrides either.
int slab_overlap_from_env(int nslabs) {
  const char *v = std::getenv("OSBLI_SLAB_OVERLAP");
  if (v && v[0] >= '0' && v[0] <= '2' && v[1] == 0) return v[0] - '0';
  return nslabs > 1 ? OSBLI_SLAB_XYSPLIT : OSBLI_SLAB_PLAIN;
}

void ghost_plan(int rank, int nranks, int nzl, int m, int plan[8], bool symz = false) {
  const int up = (rank + 1) % nranks, dn = (rank - 1 + nranks) % nranks;
  const int p[8] = {dn, 0, up, nzl, up, nzl - m, dn, -m};
  for (int i = 0; i < 8; ++i) plan[i] = p[i];
  if (symz) {
    // symmetry in z: no transfer across the periodic wrap between the
    // last and the first slab (peer -1); those ghosts mirror the own planes
    if (rank == 0) plan[0] = plan[6] = -1;           // t=0 send down, t=1 receive from below
    if (rank == nranks - 1) plan[2] = plan[4] = -1;  // t=0 receive from above, t=1 send up
  }
}

// z ghost planes of a plane-major buffer with m ghost planes at each end
// (`base` = its first ghost plane, `nf` fields per plane, field `odd` odd under a
// z mirror) from the neighbouring slabs, over NCCL (one process per GPU) or by
// device copies between sibling handles (loopback transport on one GPU);
// `sibling` picks the same buffer of a sibling handle.
template <typename Sibling>
int exchange_planes(osbli_ctx *h, double *base, int nf, int odd, Sibling sibling,
                    cudaStream_t st) {
  if (!h->slab) return OSBLI_OK;
  NvtxRange range(nf == 5 ? "osbli ghost exchange (Q)" : "osbli ghost exchange (H)");
  if (!st) st = h->stream;
  const int G = h->m;
  const size_t plane = (size_t)nf * h->nx * h->ny;
  const size_t cnt = (size_t)G * plane;
  // symmetry in z: the transfers across the periodic wrap (between the
  // first and the last slab) are absent from the plan (peer -1); those ghost
  // planes are mirrors of the outer slabs' own interior planes
  const bool symz = h->base.sym[2] != 0;
  int plan[8];
  ghost_plan(h->rank, h->nranks, h->nz, G, plan, symz);
  auto at = [&](double *b, int local_plane) { return b + (size_t)(local_plane + G) * plane; };
  if (h->comm) {
    NK(h, ncclGroupStart());
    for (int t = 0; t < 2; ++t) {
      if (plan[4 * t + 0] >= 0)
        NK(h, ncclSend(at(base, plan[4 * t + 1]), cnt, ncclDouble, plan[4 * t + 0], h->comm, st));
      if (plan[4 * t + 2] >= 0)
        NK(h, ncclRecv(at(base, plan[4 * t + 3]), cnt, ncclDouble, plan[4 * t + 2], h->comm, st));
    }
    NK(h, ncclGroupEnd());
  } else if (h->loop) {
    if (h->loop->broken) return fail(h, OSBLI_E_STATE, "a sibling slab of this loopback group was destroyed");
    // I receive what my peer sends under the same transfer index: for
    // transfer t the source is peer plan[4t+2]'s plane given by ITS plan.
    for (int t = 0; t < 2; ++t) {
      if (plan[4 * t + 2] < 0) continue;
      osbli_ctx *src = h->loop->members[plan[4 * t + 2]];
      int splan[8];
      ghost_plan(src->rank, src->nranks, src->nz, G, splan, symz);
      CK(h, cudaMemcpyAsync(at(base, plan[4 * t + 3]), at(sibling(src), splan[4 * t + 1]),
                            cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
  } else {
    return fail(h, OSBLI_E_STATE, "distributed handle without a transport");
  }
  if (plan[6] < 0) CK(h, osbli::launch_mirror_planes(h->base, base, nf, odd, 0, st, &h->launches));
  if (plan[2] < 0) CK(h, osbli::launch_mirror_planes(h->base, base, nf, odd, 1, st, &h->launches));
  return OSBLI_OK;
}

// ghost planes of the current state Q (buffer q = h->b.q[h->cur])
int exchange_ghosts(osbli_ctx *h, double *q, cudaStream_t st = nullptr) {
  return exchange_planes(h, q, 5, 3, [](osbli_ctx *s) { return s->b.q[s->cur]; }, st);
}

// ghost planes of the current Q valid in stream order on h->stream: wait for the
// exchange the previous stage posted on the comm stream (xy-split schedule), or
// exchange now
int current_ghosts(osbli_ctx *h) {
  if (h->ghost_async) {
    CK(h, cudaStreamWaitEvent(h->stream, h->ev_ghost, 0));
    h->ghost_async = false;
    return OSBLI_OK;
  }
  return exchange_ghosts(h, h->b.q[h->cur], h->stream);
}

// ghost planes of the viscous-work flux H_j (conservative form, D-27): the
// divergence kernel's z taps read H_z there
int exchange_hflux(osbli_ctx *h, cudaStream_t st = nullptr) {
  return exchange_planes(h, h->hflux_alloc, 3, 2, [](osbli_ctx *s) { return s->hflux_alloc; },
                         st);
}

// The non-finite flag, agreed on by every rank of a distributed handle (max over
// ranks by ncclAllReduce: collective), OR-ed over the members of a loopback group,
// the handle's own otherwise.  Every rank / member that sees it set is poisoned,
// so that they all refuse the next step together and none waits on a peer.
int check_flag(osbli_ctx *h) {
  unsigned int flag = 0;
  if (h->loop) {
    if (h->loop->broken) return fail(h, OSBLI_E_STATE, "a sibling slab of this loopback group was destroyed");
    for (osbli_ctx *m : h->loop->members) {
      unsigned int f = 0;
      CK(h, cudaMemcpyAsync(&f, m->b.flag, sizeof(f), cudaMemcpyDeviceToHost, m->stream));
      CK(h, cudaStreamSynchronize(m->stream));
      flag |= f;
    }
    if (flag) {
      for (osbli_ctx *m : h->loop->members)
        fail(m, OSBLI_E_NONFINITE, "a time step produced a non-finite value (loopback group)");
      return OSBLI_E_NONFINITE;
    }
    return OSBLI_OK;
  }
  const unsigned int *src = h->b.flag;
  if (h->comm) {
    NK(h, ncclAllReduce(h->b.flag, h->flag_all, 1, ncclUint32, ncclMax, h->comm, h->stream));
    src = h->flag_all;
  }
  CK(h, cudaMemcpyAsync(&flag, src, sizeof(flag), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  if (flag) return fail(h, OSBLI_E_NONFINITE, "a time step produced a non-finite value");
  return OSBLI_OK;
}

}  // namespace

extern "C" {

const char *osbli_version(void) { return "osbli 0.1 sm_100a fp64 orders 2..12"; }

int osbli_create(int nx, int ny, int nz, int order, double dx, double dt, double Re, double Pr,
                 double Minf, double gamma, int scheme, osbli_ctx **out) {
  if (!out) return OSBLI_E_INVAL;
  *out = nullptr;
  std::string msg;
  int v = validate(nx, ny, nz, order, dx, dt, Re, Pr, Minf, gamma, scheme, msg);
  if (v != OSBLI_OK) { g_create_error = msg; return v; }
  osbli_ctx *h = new (std::nothrow) osbli_ctx();
  if (!h) return OSBLI_E_NOMEM;
  h->nx = nx; h->ny = ny; h->nz_global = nz; h->nz = nz; h->z0 = 0;
  h->order = order; h->scheme = scheme;
  h->dx = dx; h->dt = dt; h->Re = Re; h->Pr = Pr; h->Minf = Minf; h->gamma = gamma;
  int r = create_common(h);
  if (r != OSBLI_OK) {
    g_create_error = h->err;
    free_all(h);
    if (h->own_stream) cudaStreamDestroy(h->own_stream);
    delete h;
    return r;
  }
  *out = h;
  return OSBLI_OK;
}

int osbli_nccl_unique_id(void *id_out) {
  if (!id_out) return OSBLI_E_INVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) { g_create_error = "ncclGetUniqueId failed"; return OSBLI_E_COMM; }
  std::memcpy(id_out, &id, sizeof(id));
  return OSBLI_OK;
}

int osbli_create_dist(int nx, int ny, int nz, int order, double dx, double dt, double Re,
                      double Pr, double Minf, double gamma, int scheme, int rank, int nranks,
                      const void *nccl_unique_id, osbli_ctx **out) {
  if (!out) return OSBLI_E_INVAL;
  *out = nullptr;
  std::string msg;
  int v = validate(nx, ny, nz, order, dx, dt, Re, Pr, Minf, gamma, scheme, msg);
  if (v != OSBLI_OK) { g_create_error = msg; return v; }
  if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !nccl_unique_id)) {
    g_create_error = "bad rank / nranks / unique id";
    return OSBLI_E_INVAL;
  }
  const int m = order / 2;
  int z0 = 0, nzl = 0;
  slab_partition(nz, nranks, rank, &z0, &nzl);
  const int base = nz / nranks, extra = nz % nranks;
  if ((nranks > 1 || nccl_unique_id) && base < m) {
    g_create_error = "every slab needs at least order/2 planes";
    return OSBLI_E_INVAL;
  }
  osbli_ctx *h = new (std::nothrow) osbli_ctx();
  if (!h) return OSBLI_E_NOMEM;
  h->nx = nx; h->ny = ny; h->nz_global = nz; h->nz = nzl; h->z0 = z0;
  h->order = order; h->scheme = scheme; h->rank = rank; h->nranks = nranks;
  // one rank with a unique id runs the distributed path too (its ghost planes come
  // from itself over NCCL): the NCCL code path on a single GPU
  h->slab = nranks > 1 || nccl_unique_id != nullptr;
  h->overlap = slab_overlap_from_env(nranks);
  h->max_nz = base + (extra ? 1 : 0);
  h->dx = dx; h->dt = dt; h->Re = Re; h->Pr = Pr; h->Minf = Minf; h->gamma = gamma;
  int r = create_common(h);
  if (r == OSBLI_OK && h->slab) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    ncclResult_t nr = ncclCommInitRank(&h->comm, nranks, id, rank);
    if (nr != ncclSuccess) {
      h->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(nr);
      r = OSBLI_E_COMM;
    } else if (cudaMalloc((void **)&h->nccl_part, (size_t)3 * nranks * h->max_nz * sizeof(double)) !=
                   cudaSuccess ||
               cudaMalloc((void **)&h->flag_all, sizeof(unsigned int)) != cudaSuccess) {
      h->err = "device allocation failed";
      r = OSBLI_E_NOMEM;
    } else if (cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
               cudaEventCreateWithFlags(&h->ev_qready, cudaEventDisableTiming) != cudaSuccess ||
               cudaEventCreateWithFlags(&h->ev_ghost, cudaEventDisableTiming) != cudaSuccess ||
               cudaEventRecord(h->ev_qready, h->stream) != cudaSuccess) {
      h->err = "stream/event creation failed";
      r = OSBLI_E_CUDA;
    }
  }
  if (r != OSBLI_OK) {
    g_create_error = h->err;
    if (h->comm) ncclCommDestroy(h->comm);
    free_all(h);
    if (h->own_stream) cudaStreamDestroy(h->own_stream);
    delete h;
    return r;
  }
  *out = h;
  return OSBLI_OK;
}

int osbli_local_box(const osbli_ctx *h, int *z0, int *nz_local) {
  if (!h || !z0 || !nz_local) return OSBLI_E_INVAL;
  *z0 = h->z0;
  *nz_local = h->nz;
  return OSBLI_OK;
}

int osbli_set_stream(osbli_ctx *h, void *cuda_stream) {
  int u = check_usable(h);
  if (u) return u;
  if (h->loop) return fail(h, OSBLI_E_INVAL, "loopback slabs share the group stream");
  // order the switch: work queued on the old stream completes first
  CK(h, cudaStreamSynchronize(h->stream));
  h->stream = cuda_stream ? (cudaStream_t)cuda_stream : h->own_stream;
  return OSBLI_OK;
}

static int set_state_impl(osbli_ctx *h, const double *q, int on_device, bool sync) {
  int u = check_usable(h);
  if (u) return u;
  if (!q) return fail(h, OSBLI_E_INVAL, "null state pointer");
  const size_t n = (size_t)5 * h->nz * h->nx * h->ny;
  // stage in ABI layout through the idle ping-pong buffer, then transpose
  double *stage = h->b.q[h->cur ^ 1];
  CK(h, cudaMemcpyAsync(stage, q, n * sizeof(double),
                        on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
  CK(h, osbli::launch_abi_to_internal(h->base, stage, h->b.q[h->cur], h->stream, &h->launches));
  if (h->ev_qready) CK(h, cudaEventRecord(h->ev_qready, h->stream));
  h->ghost_async = false;
  CK(h, cudaMemsetAsync(h->b.flag, 0, sizeof(unsigned int), h->stream));
  if (sync) CK(h, cudaStreamSynchronize(h->stream));
  h->step_count = 0;
  return OSBLI_OK;
}

static int get_state_impl(osbli_ctx *h, double *q, int on_device, bool sync) {
  if (!h || !q) return OSBLI_E_INVAL;
  const size_t n = (size_t)5 * h->nz * h->nx * h->ny;
  double *stage = h->b.q[h->cur ^ 1];  // idle ping-pong buffer as ABI-layout staging
  CK(h, osbli::launch_internal_to_abi(h->base, h->b.q[h->cur], stage, 5, 1, h->stream, &h->launches));
  CK(h, cudaMemcpyAsync(q, stage, n * sizeof(double),
                        on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
  if (sync) CK(h, cudaStreamSynchronize(h->stream));
  return OSBLI_OK;
}

int osbli_set_state(osbli_ctx *h, const double *q, int on_device) {
  return set_state_impl(h, q, on_device, true);
}
int osbli_get_state(osbli_ctx *h, double *q, int on_device) {
  return get_state_impl(h, q, on_device, true);
}
int osbli_set_state_async(osbli_ctx *h, const double *q, int on_device) {
  return set_state_impl(h, q, on_device, false);
}
int osbli_get_state_async(osbli_ctx *h, double *q, int on_device) {
  // same policy as osbli_get_state: valid on a poisoned handle (the last state)
  return get_state_impl(h, q, on_device, false);
}

}  // extern "C"

namespace {

// One stage s of the time scheme on handle h: ghost exchange, z-pass, xy-pass.
int run_stage(osbli_ctx *h, int s, bool exchange = true, bool divh = true) {
  static const char *const kStageName[3] = {"osbli stage 1", "osbli stage 2", "osbli stage 3"};
  NvtxRange range(kStageName[s]);
  static const double RK_A[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};
  static const double RK_B[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
  static const double RK2R_ALPHA[3] = {2.0 / 3.0, 5.0 / 12.0, 3.0 / 5.0};
  static const double RK2R_BETA[3] = {1.0 / 4.0, 3.0 / 20.0, 3.0 / 5.0};
  KParams p = h->base;
  if (s == 0) p.dpart = h->stage_dpart;  // fused diagnostics of the step's input state
  double *qin = h->b.q[h->cur], *qout = h->b.q[h->cur ^ 1];
  double *wz = h->b.w;  // z-pass output W'
  if (h->scheme == OSBLI_RK3) {
    p.A = RK_A[s];
    p.B = RK_B[s];
    p.read_w = (s > 0);
    p.write_w = (s < 2);
  } else if (h->scheme == OSBLI_RK3_2R) {
    // Q' = Q_old + alpha_s dt R ; Q_old += beta_s dt R (D-25).  The z-pass part
    // dt Rz goes to the interior planes of the destination buffer, which the
    // xy-pass then overwrites point by point with Q'.
    p.A = 0.0;
    p.B = RK2R_ALPHA[s];
    p.beta = RK2R_BETA[s];
    p.two_reg = 1;
    p.read_w = (s > 0);
    p.write_w = (s < 2);
    wz = qout + (size_t)h->base.G * 5 * ((size_t)h->nx * h->ny);
  } else {
    p.A = 0.0;
    p.B = 1.0;
    p.read_w = 0;
    p.write_w = 0;
  }
  cudaEvent_t *ev = nullptr;
  if (h->timing) {
    if (h->ev_used + 3 > h->events.size()) {
      for (int k = 0; k < 3; ++k) {
        cudaEvent_t e;
        CK(h, cudaEventCreate(&e));
        h->events.push_back(e);
      }
    }
    ev = &h->events[h->ev_used];
    h->ev_used += 3;
  }
  if (!h->slab) {
    if (ev) CK(h, cudaEventRecord(ev[0], h->stream));
    CK(h, osbli::launch_zpass(p, qin, wz, h->b.gz, 0, h->nz, h->stream, &h->launches));
    if (ev) CK(h, cudaEventRecord(ev[1], h->stream));
    CK(h, osbli::launch_xypass(p, qin, qout, h->b.w, h->b.gz, nullptr, h->b.flag, 0, h->nz,
                               h->stream, &h->launches));
    if (ev) CK(h, cudaEventRecord(ev[2], h->stream));
    if (p.cons)
      CK(h, osbli::launch_divh(p, qout, h->b.w, nullptr, h->b.flag, 0, h->nz, h->stream,
                               &h->launches));
    h->cur ^= 1;
    return OSBLI_OK;
  }
  // Slab decomposition.  The m planes next to each slab face are
  // the only ones whose z-pass reads ghost planes and the only ones the
  // neighbours read.  Three schedules:
  //   PLAIN   exchange; z-pass; xy-pass                                 (2 launches)
  //   ZSPLIT  exchange on the comm stream || interior z-pass; face z-pass (both
  //           faces, one launch); xy-pass                               (3 launches)
  //   XYSPLIT z-pass; face xy-pass (both faces, one launch); exchange of the NEW
  //           state's faces on the comm stream || interior xy-pass; the next
  //           stage's z-pass waits for it                             (3 launches)
  // (the conservative viscous work finishes Q' only after its divergence kernel:
  // it keeps the plain order after the xy-pass)
  const int m = h->m;
  const int lo = m < h->nz ? m : h->nz;            // [0, lo): low face planes
  const int hi = h->nz - m > lo ? h->nz - m : lo;  // [hi, nz): high face planes
  const int mode = h->overlap;
  // ---- ghost planes of Q (qin)
  if (h->comm && mode == OSBLI_SLAB_ZSPLIT && !h->ghost_async) {
    CK(h, cudaStreamWaitEvent(h->comm_stream, h->ev_qready, 0));
    int r = exchange_ghosts(h, qin, h->comm_stream);
    if (r) return r;
    CK(h, cudaEventRecord(h->ev_ghost, h->comm_stream));
    h->ghost_async = true;
  } else if (h->comm) {
    int r = current_ghosts(h);
    if (r) return r;
  } else if (exchange) {
    int r = exchange_ghosts(h, qin);
    if (r) return r;
  }
  // ---- z-pass
  if (ev) CK(h, cudaEventRecord(ev[0], h->stream));
  if (mode == OSBLI_SLAB_ZSPLIT) {
    CK(h, osbli::launch_zpass(p, qin, wz, h->b.gz, lo, hi, h->stream, &h->launches));
    if (h->ghost_async) {
      CK(h, cudaStreamWaitEvent(h->stream, h->ev_ghost, 0));
      h->ghost_async = false;
    }
    CK(h, osbli::launch_zpass(p, qin, wz, h->b.gz, 0, lo, h->stream, &h->launches, hi, h->nz));
  } else {
    CK(h, osbli::launch_zpass(p, qin, wz, h->b.gz, 0, h->nz, h->stream, &h->launches));
  }
  if (ev) CK(h, cudaEventRecord(ev[1], h->stream));
  // ---- xy-pass
  if (mode == OSBLI_SLAB_XYSPLIT && !p.cons) {
    CK(h, osbli::launch_xypass(p, qin, qout, h->b.w, h->b.gz, nullptr, h->b.flag, 0, lo,
                               h->stream, &h->launches, hi, h->nz));
    if (h->comm) {
      // the faces of Q' are final: their exchange runs behind the interior xy-pass
      CK(h, cudaEventRecord(h->ev_qready, h->stream));
      CK(h, cudaStreamWaitEvent(h->comm_stream, h->ev_qready, 0));
      int r = exchange_ghosts(h, qout, h->comm_stream);
      if (r) return r;
      CK(h, cudaEventRecord(h->ev_ghost, h->comm_stream));
    }
    CK(h, osbli::launch_xypass(p, qin, qout, h->b.w, h->b.gz, nullptr, h->b.flag, lo, hi,
                               h->stream, &h->launches));
    if (ev) CK(h, cudaEventRecord(ev[2], h->stream));
    h->cur ^= 1;
    h->ghost_async = h->comm != nullptr;  // ghosts of the new current Q are in flight
    return OSBLI_OK;
  }
  CK(h, osbli::launch_xypass(p, qin, qout, h->b.w, h->b.gz, nullptr, h->b.flag, 0, h->nz,
                             h->stream, &h->launches));
  if (ev) CK(h, cudaEventRecord(ev[2], h->stream));
  if (p.cons && divh) {
    // D_z H_z at the slab faces needs the neighbours' H: exchange its ghost planes
    int r = exchange_hflux(h, h->stream);
    if (r) return r;
    CK(h, osbli::launch_divh(p, qout, h->b.w, nullptr, h->b.flag, 0, h->nz, h->stream,
                             &h->launches));
  }
  // Q' complete: the next stage's exchange may read its face planes
  if (h->comm) CK(h, cudaEventRecord(h->ev_qready, h->stream));
  h->cur ^= 1;
  return OSBLI_OK;
}

// the divergence of the viscous-work flux for stage s of a slab handle whose
// xy-pass ran (run_stage(..., divh = false)) and whose H ghosts are current
int finish_divh(osbli_ctx *h, int s) {
  static const double RK_B[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
  static const double RK2R_ALPHA[3] = {2.0 / 3.0, 5.0 / 12.0, 3.0 / 5.0};
  static const double RK2R_BETA[3] = {1.0 / 4.0, 3.0 / 20.0, 3.0 / 5.0};
  KParams p = h->base;
  if (h->scheme == OSBLI_RK3) {
    p.B = RK_B[s];
    p.write_w = (s < 2);
  } else if (h->scheme == OSBLI_RK3_2R) {
    p.B = RK2R_ALPHA[s];
    p.beta = RK2R_BETA[s];
    p.two_reg = 1;
    p.write_w = (s < 2);
  } else {
    p.B = 1.0;
    p.write_w = 0;
  }
  CK(h, osbli::launch_divh(p, h->b.q[h->cur], h->b.w, nullptr, h->b.flag, 0, h->nz, h->stream,
                           &h->launches));
  return OSBLI_OK;
}

int nstages(const osbli_ctx *h) { return h->scheme == OSBLI_EULER ? 1 : 3; }

}  // namespace

extern "C" {

int osbli_step(osbli_ctx *h, int n) {
  int u = check_usable(h);
  if (u) return u;
  if (n < 0) return fail(h, OSBLI_E_INVAL, "n must be >= 0");
  if (h->loop) return fail(h, OSBLI_E_INVAL, "loopback slabs advance together: osbli_loopback_step");
  for (int it = 0; it < n; ++it) {
    for (int s = 0; s < nstages(h); ++s) {
      int r = run_stage(h, s);
      if (r) return r;
    }
    ++h->step_count;
  }
  return OSBLI_OK;
}

int osbli_step_diag(osbli_ctx *h, int n, osbli_diag *series) {
  NvtxRange range("osbli step+diagnostics");
  int u = check_usable(h);
  if (u) return u;
  if (n < 0 || (n > 0 && !series)) return fail(h, OSBLI_E_INVAL, "n must be >= 0 and series non-null");
  if (h->loop) return fail(h, OSBLI_E_INVAL, "loopback slabs advance together: osbli_loopback_step");
  constexpr int BATCH = 64;  // steps per gather / host reduction
  const int ntiles = osbli::xypass_tiles(h->base);
  const int stride = h->max_nz > h->nz ? h->max_nz : h->nz;  // planes per step record
  const size_t rec = (size_t)3 * stride;                      // doubles per step record
  if (!h->dtiles) {
    CK(h, cudaStreamSynchronize(h->stream));
    CK(h, cudaMalloc((void **)&h->dtiles, (size_t)3 * h->nz * ntiles * sizeof(double)));
    CK(h, cudaMalloc((void **)&h->dseries, BATCH * rec * sizeof(double)));
    CK(h, cudaMemset(h->dseries, 0, BATCH * rec * sizeof(double)));  // padding planes stay 0
    if (h->comm)
      CK(h, cudaMalloc((void **)&h->dseries_all, (size_t)h->nranks * BATCH * rec * sizeof(double)));
  }
  std::vector<double> host((size_t)(h->comm ? h->nranks : 1) * BATCH * rec);
  std::vector<int> counts;
  if (h->comm) {
    for (int rr = 0; rr < h->nranks; ++rr) {
      int z0 = 0, nzl = 0;
      slab_partition(h->nz_global, h->nranks, rr, &z0, &nzl);
      counts.push_back(nzl);
    }
  } else {
    counts.push_back(h->nz);
  }
  const double N = (double)h->nx * h->ny * h->nz_global;
  for (int k0 = 0; k0 < n; k0 += BATCH) {
    const int nb = n - k0 < BATCH ? n - k0 : BATCH;
    const long long step0 = h->step_count;
    for (int b = 0; b < nb; ++b) {
      for (int s = 0; s < nstages(h); ++s) {
        h->stage_dpart = s == 0 ? h->dtiles : nullptr;
        int r = run_stage(h, s);
        h->stage_dpart = nullptr;
        if (r) return r;
        if (s == 0)
          CK(h, osbli::launch_diag_planes(h->dtiles, h->nz, ntiles, h->dseries + b * rec,
                                          h->stream, &h->launches));
      }
      ++h->step_count;
    }
    const double *src = h->dseries;
    if (h->comm) {
      NK(h, ncclAllGather(h->dseries, h->dseries_all, BATCH * rec, ncclDouble, h->comm, h->stream));
      src = h->dseries_all;
    }
    CK(h, cudaMemcpyAsync(host.data(), src, host.size() * sizeof(double), cudaMemcpyDeviceToHost,
                          h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    int r = check_flag(h);  // collective when distributed
    if (r) return r;
    for (int b = 0; b < nb; ++b) {
      // Neumaier sums over planes in global z order (ranks own consecutive slabs)
      double sm[3] = {0, 0, 0}, c[3] = {0, 0, 0};
      for (int rr = 0; rr < (int)counts.size(); ++rr)
        for (int z = 0; z < counts[rr]; ++z)
          for (int k = 0; k < 3; ++k) {
            const double x = host[((size_t)rr * BATCH + b) * rec + (size_t)3 * z + k];
            const double t = sm[k] + x;
            if (std::fabs(sm[k]) >= std::fabs(x)) c[k] += (sm[k] - t) + x;
            else c[k] += (x - t) + sm[k];
            sm[k] = t;
          }
      osbli_diag &d = series[k0 + b];
      d.step = step0 + b;
      d.t = d.step * h->dt;
      d.kinetic_energy = (sm[0] + c[0]) / N;
      d.enstrophy = (sm[1] + c[1]) / N;
      d.dissipation = (sm[2] + c[2]) / N;
    }
  }
  return OSBLI_OK;
}

int osbli_slab_bounds(int nz, int nranks, int rank, int *z0, int *nz_local) {
  if (nz < 1 || nranks < 1 || rank < 0 || rank >= nranks || !z0 || !nz_local) return OSBLI_E_INVAL;
  slab_partition(nz, nranks, rank, z0, nz_local);
  return OSBLI_OK;
}

int osbli_ghost_plan(int rank, int nranks, int nz_local, int m, int *plan) {
  return osbli_ghost_plan_sym(rank, nranks, nz_local, m, 0, plan);
}

int osbli_ghost_plan_sym(int rank, int nranks, int nz_local, int m, int symz, int *plan) {
  if (nranks < 1 || rank < 0 || rank >= nranks || m < 1 || nz_local < m || !plan)
    return OSBLI_E_INVAL;
  ghost_plan(rank, nranks, nz_local, m, plan, symz != 0);
  return OSBLI_OK;
}

int osbli_create_loopback(int nx, int ny, int nz, int order, double dx, double dt, double Re,
                          double Pr, double Minf, double gamma, int scheme, int nslabs,
                          osbli_ctx **out) {
  if (!out || nslabs < 2) return OSBLI_E_INVAL;
  std::string msg;
  int v = validate(nx, ny, nz, order, dx, dt, Re, Pr, Minf, gamma, scheme, msg);
  if (v != OSBLI_OK) { g_create_error = msg; return v; }
  if (nz / nslabs < order / 2) { g_create_error = "every slab needs at least order/2 planes"; return OSBLI_E_INVAL; }
  LoopGroup *g = new (std::nothrow) LoopGroup();
  if (!g) return OSBLI_E_NOMEM;
  for (int r = 0; r < nslabs; ++r) {
    osbli_ctx *h = new (std::nothrow) osbli_ctx();
    int rc = h ? OSBLI_OK : OSBLI_E_NOMEM;
    if (h) {
      slab_partition(nz, nslabs, r, &h->z0, &h->nz);
      h->nx = nx; h->ny = ny; h->nz_global = nz;
      h->order = order; h->scheme = scheme; h->rank = r; h->nranks = nslabs;
      h->slab = true;
      h->overlap = slab_overlap_from_env(nslabs);
      h->max_nz = nz / nslabs + (nz % nslabs ? 1 : 0);
      h->dx = dx; h->dt = dt; h->Re = Re; h->Pr = Pr; h->Minf = Minf; h->gamma = gamma;
      h->loop = g;
      rc = create_common(h);
      if (rc != OSBLI_OK) g_create_error = h->err;
    }
    if (rc != OSBLI_OK) {
      if (h) { free_all(h); if (h->own_stream) cudaStreamDestroy(h->own_stream); delete h; }
      for (auto *m : g->members) { free_all(m); if (m->own_stream) cudaStreamDestroy(m->own_stream); delete m; }
      delete g;
      return rc;
    }
    g->members.push_back(h);
  }
  // one stream for the whole group keeps the sibling copies ordered
  for (int r = 0; r < nslabs; ++r) g->streams.push_back(g->members[r]->own_stream);
  for (int r = 1; r < nslabs; ++r) g->members[r]->stream = g->members[0]->stream;
  g->live = nslabs;
  for (int r = 0; r < nslabs; ++r) out[r] = g->members[r];
  return OSBLI_OK;
}

int osbli_loopback_step(osbli_ctx **hs, int nslabs, int n) {
  if (!hs || nslabs < 2 || n < 0) return OSBLI_E_INVAL;
  LoopGroup *g = hs[0] ? hs[0]->loop : nullptr;
  if (!g || (int)g->members.size() != nslabs) return OSBLI_E_INVAL;
  for (int r = 0; r < nslabs; ++r) {
    if (hs[r] != g->members[r]) return OSBLI_E_INVAL;
    int u = check_usable(hs[r]);
    if (u) return u;
  }
  for (int it = 0; it < n; ++it) {
    for (int s = 0; s < nstages(hs[0]); ++s) {
      // every slab reads its neighbours' current planes, then all advance
      for (int r = 0; r < nslabs; ++r) {
        int rc = exchange_ghosts(hs[r], hs[r]->b.q[hs[r]->cur]);
        if (rc) return rc;
      }
      const bool cons = hs[0]->base.cons != 0;
      for (int r = 0; r < nslabs; ++r) {
        int rc = run_stage(hs[r], s, /*exchange=*/false, /*divh=*/!cons);
        if (rc) return rc;
      }
      if (cons) {  // every slab's H is written: exchange its ghosts, then the divergence
        for (int r = 0; r < nslabs; ++r) {
          int rc = exchange_hflux(hs[r]);
          if (rc) return rc;
        }
        for (int r = 0; r < nslabs; ++r) {
          int rc = finish_divh(hs[r], s);
          if (rc) return rc;
        }
      }
    }
    for (int r = 0; r < nslabs; ++r) ++hs[r]->step_count;
  }
  return OSBLI_OK;
}

int osbli_set_slab_schedule(osbli_ctx *h, int schedule) {
  int u = check_usable(h);
  if (u) return u;
  if (schedule < OSBLI_SLAB_PLAIN || schedule > OSBLI_SLAB_XYSPLIT)
    return fail(h, OSBLI_E_INVAL, "schedule must be OSBLI_SLAB_PLAIN, _ZSPLIT or _XYSPLIT");
  if (h->slab) h->overlap = schedule;
  return OSBLI_OK;
}

int osbli_set_boundary(osbli_ctx *h, int dir, int bc) {
  int u = check_usable(h);
  if (u) return u;
  if (dir < 0 || dir > 2 || (bc != OSBLI_BC_PERIODIC && bc != OSBLI_BC_SYMMETRY))
    return fail(h, OSBLI_E_INVAL, "bad direction or boundary type");
  h->base.sym[dir] = bc;
  return OSBLI_OK;
}

int osbli_set_viscosity(osbli_ctx *h, int law, double suth) {
  int u = check_usable(h);
  if (u) return u;
  if (law != OSBLI_VISC_CONSTANT && law != OSBLI_VISC_SUTHERLAND)
    return fail(h, OSBLI_E_INVAL, "bad viscosity law");
  if (law == OSBLI_VISC_SUTHERLAND && !(suth > 0.0 && std::isfinite(suth)))
    return fail(h, OSBLI_E_INVAL, "the Sutherland constant must be > 0");
  const size_t FS = (size_t)h->nx * h->ny;
  if (law == OSBLI_VISC_SUTHERLAND && !h->base.dtz) {
    CK(h, cudaStreamSynchronize(h->stream));
    CK(h, cudaMalloc((void **)&h->base.dtz, (size_t)h->nz * FS * sizeof(double)));
  }
  h->base.visc = law;
  h->base.suth = law == OSBLI_VISC_SUTHERLAND ? suth : 0.0;
  return OSBLI_OK;
}

int osbli_set_energy_form(osbli_ctx *h, int form) {
  int u = check_usable(h);
  if (u) return u;
  if (form != OSBLI_ENERGY_EXPANDED && form != OSBLI_ENERGY_CONSERVATIVE)
    return fail(h, OSBLI_E_INVAL, "bad energy form");
  const size_t FS = (size_t)h->nx * h->ny;
  if (form == OSBLI_ENERGY_CONSERVATIVE) {
    CK(h, cudaStreamSynchronize(h->stream));
    if (!h->base.dtz) CK(h, cudaMalloc((void **)&h->base.dtz, (size_t)h->nz * FS * sizeof(double)));
    if (!h->hflux_alloc) {
      // H_j with m ghost planes at each end (the slab path exchanges them); the
      // kernels address it from the first interior plane
      const size_t G = (size_t)h->base.G;
      CK(h, cudaMalloc((void **)&h->hflux_alloc, (h->nz + 2 * G) * 3 * FS * sizeof(double)));
      h->base.hflux = h->hflux_alloc + G * 3 * FS;
    }
  }
  h->base.cons = form;
  return OSBLI_OK;
}

int osbli_set_source(osbli_ctx *h, const double *S, int on_device) {
  int u = check_usable(h);
  if (u) return u;
  CK(h, cudaStreamSynchronize(h->stream));
  if (!S) {
    cudaFree(h->src);
    h->src = nullptr;
    h->base.src = nullptr;
    return OSBLI_OK;
  }
  const size_t n = (size_t)5 * h->nz * h->nx * h->ny;
  if (!h->src) CK(h, cudaMalloc((void **)&h->src, n * sizeof(double)));
  // ABI layout -> plane-major (no ghost planes) through the idle ping-pong buffer
  double *stage = h->b.q[h->cur ^ 1];
  CK(h, cudaMemcpyAsync(stage, S, n * sizeof(double),
                        on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
  KParams p0 = h->base;
  p0.G = 0;
  CK(h, osbli::launch_abi_to_internal(p0, stage, h->src, h->stream, &h->launches));
  CK(h, cudaStreamSynchronize(h->stream));
  h->base.src = h->src;
  return OSBLI_OK;
}

int osbli_residual(osbli_ctx *h, double *R, int on_device) {
  NvtxRange range("osbli residual");
  int u = check_usable(h);
  if (u) return u;
  if (!R) return fail(h, OSBLI_E_INVAL, "null output pointer");
  if (h->base.cons && h->slab)
    return fail(h, OSBLI_E_UNSUPPORTED,
                "the residual hook of a slab handle has no viscous-work flux exchange");
  const size_t n = (size_t)5 * h->nz * h->nx * h->ny;
  double *qin = h->b.q[h->cur];
  int r = h->comm ? current_ghosts(h) : exchange_ghosts(h, qin);
  if (r) return r;
  // R lands in W ([nz][5] plane-major: A = 0, dt = 1 so that W' = Rz and R = W' + R_xy),
  // then is transposed into the idle ping-pong buffer (ABI layout)
  KParams p = h->base;
  p.A = 0.0;
  p.B = 0.0;
  p.dt = 1.0;
  p.read_w = 0;
  p.write_w = 0;
  double *stage = h->b.q[h->cur ^ 1];
  CK(h, osbli::launch_stage(p, qin, nullptr, h->b.w, h->b.gz, h->b.w, h->b.flag, h->stream,
                            &h->launches));
  CK(h, osbli::launch_internal_to_abi(h->base, h->b.w, stage, 5, 0, h->stream, &h->launches));
  CK(h, cudaMemcpyAsync(R, stage, n * sizeof(double),
                        on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return OSBLI_OK;
}

int osbli_diagnostics(osbli_ctx *h, osbli_diag *out) {
  NvtxRange range("osbli diagnostics");
  int u = check_usable(h);
  if (u) return u;
  if (!out) return fail(h, OSBLI_E_INVAL, "null output pointer");
  if (h->loop && h->loop->broken)
    return fail(h, OSBLI_E_STATE, "a sibling slab of this loopback group was destroyed");
  int r = OSBLI_OK;
  std::vector<double> all;
  std::vector<int> counts;
  int stride = h->nz;
  if (h->loop) {
    // loopback slabs: every sibling computes its per-plane partials; gathered in rank order
    stride = h->max_nz;
    all.assign((size_t)3 * h->nranks * stride, 0.0);
    for (osbli_ctx *m : h->loop->members) {
      r = exchange_ghosts(m, m->b.q[m->cur]);
      if (r) return r;
      CK(h, osbli::launch_diagnostics(m->base, m->b.q[m->cur], m->scratch, m->b.diag_part,
                                      m->stream, &m->launches));
      CK(h, cudaMemcpyAsync(all.data() + (size_t)3 * m->rank * stride, m->b.diag_part,
                            (size_t)3 * m->nz * sizeof(double), cudaMemcpyDeviceToHost, m->stream));
      counts.push_back(m->nz);
    }
  } else {
    double *qin = h->b.q[h->cur];
    r = h->comm ? current_ghosts(h) : exchange_ghosts(h, qin);
    if (r) return r;
    CK(h, osbli::launch_diagnostics(h->base, qin, h->scratch, h->b.diag_part, h->stream,
                                    &h->launches));
    if (h->comm) {
      stride = h->max_nz;
      CK(h, cudaMemsetAsync(h->nccl_part, 0, (size_t)3 * h->nranks * h->max_nz * sizeof(double),
                            h->stream));
      // gather padded per-plane partials; every rank then sums in global plane order
      NK(h, ncclAllGather(h->b.diag_part, h->nccl_part, (size_t)3 * h->max_nz, ncclDouble,
                          h->comm, h->stream));
      all.resize((size_t)3 * h->nranks * h->max_nz);
      CK(h, cudaMemcpyAsync(all.data(), h->nccl_part, all.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, h->stream));
      for (int rr = 0; rr < h->nranks; ++rr) {
        int z0 = 0, nzl = 0;
        slab_partition(h->nz_global, h->nranks, rr, &z0, &nzl);
        counts.push_back(nzl);
      }
    } else {
      all.resize((size_t)3 * h->nz);
      CK(h, cudaMemcpyAsync(all.data(), h->b.diag_part, all.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, h->stream));
      counts.push_back(h->nz);
    }
  }
  CK(h, cudaStreamSynchronize(h->stream));
  // the non-finite flag after every rank has taken part in the collectives above
  // (collective itself: every rank gets the same answer)
  r = check_flag(h);
  if (r) return r;
  // Neumaier sums over planes in global z order
  double s[3] = {0, 0, 0}, c[3] = {0, 0, 0};
  for (int rr = 0; rr < (int)counts.size(); ++rr)
    for (int z = 0; z < counts[rr]; ++z)
      for (int k = 0; k < 3; ++k) {
        const double x = all[(size_t)3 * ((size_t)rr * stride + z) + k];
        const double t = s[k] + x;
        if (std::fabs(s[k]) >= std::fabs(x)) c[k] += (s[k] - t) + x;
        else c[k] += (x - t) + s[k];
        s[k] = t;
      }
  const double N = (double)h->nx * h->ny * h->nz_global;
  out->t = h->step_count * h->dt;
  out->step = h->step_count;
  out->kinetic_energy = (s[0] + c[0]) / N;
  out->enstrophy = (s[1] + c[1]) / N;
  out->dissipation = (s[2] + c[2]) / N;
  return OSBLI_OK;
}

int osbli_sync(osbli_ctx *h) {
  int u = check_usable(h);
  if (u) return u;
  return check_flag(h);
}

long long osbli_kernel_launches(const osbli_ctx *h) { return h ? h->launches : -1; }

int osbli_set_kernel_timing(osbli_ctx *h, int enable) {
  int u = check_usable(h);
  if (u) return u;
  h->timing = enable != 0;
  h->ev_used = 0;
  return OSBLI_OK;
}

int osbli_kernel_timing(osbli_ctx *h, double *zpass_ms, double *xypass_ms, long long *n_zpass,
                        long long *n_xypass) {
  int u = check_usable(h);
  if (u) return u;
  if (!zpass_ms || !xypass_ms || !n_zpass || !n_xypass) return fail(h, OSBLI_E_INVAL, "null output");
  CK(h, cudaStreamSynchronize(h->stream));
  double zs = 0.0, xs = 0.0;
  for (size_t i = 0; i + 3 <= h->ev_used; i += 3) {
    float a = 0.f, b = 0.f;
    CK(h, cudaEventElapsedTime(&a, h->events[i], h->events[i + 1]));
    CK(h, cudaEventElapsedTime(&b, h->events[i + 1], h->events[i + 2]));
    zs += a;
    xs += b;
  }
  *zpass_ms = zs;
  *xypass_ms = xs;
  *n_zpass = *n_xypass = (long long)(h->ev_used / 3);
  h->ev_used = 0;
  return OSBLI_OK;
}

const char *osbli_last_error(const osbli_ctx *h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

void osbli_destroy(osbli_ctx *h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->comm_stream) cudaStreamSynchronize(h->comm_stream);
  if (h->comm) ncclCommDestroy(h->comm);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  if (h->ev_qready) cudaEventDestroy(h->ev_qready);
  if (h->ev_ghost) cudaEventDestroy(h->ev_ghost);
  for (auto e : h->events) cudaEventDestroy(e);
  free_all(h);
  LoopGroup *g = h->loop;
  if (g) {
    // the group stream belongs to member 0: destroy streams with the last member
    for (auto &m : g->members)
      if (m == h) m = nullptr;
    g->broken = true;
    if (--g->live == 0) {
      for (cudaStream_t st : g_loop_streams(g)) cudaStreamDestroy(st);
      delete g;
    }
  } else if (h->own_stream) {
    cudaStreamDestroy(h->own_stream);
  }
  delete h;
}

}  // extern "C"
