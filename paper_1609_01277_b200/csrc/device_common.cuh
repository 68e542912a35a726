// Device helpers shared by the kernel translation units (periodic / mirror
// index maps, cp.async, fast reciprocals, Sutherland).  Internal linkage: every
// translation unit gets its own copy.
#pragma once
#include <cuda.h>

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

// The planes of one launch: segments of seg_len planes of [b0, e0) (blockIdx.z <
// nseg0), then of [b1, e1) (the face planes at both ends of a slab in one launch,
// DESIGN.md §6); b1 = e1 for a single range.
struct PlaneRange {
  int b0, e0, nseg0, b1, e1, seg_len;
  // this CTA's planes [zs, ze); false when empty
  __device__ __forceinline__ bool segment(int &zs, int &ze) const {
    const bool r1 = (int)blockIdx.z >= nseg0;
    zs = (r1 ? b1 : b0) + (int)(r1 ? blockIdx.z - nseg0 : blockIdx.z) * seg_len;
    ze = min(r1 ? e1 : e0, zs + seg_len);
    return zs < ze;
  }
};

inline PlaneRange plane_range(int zb, int ze, int zb1, int ze1, int seg_len, int *nseg_total) {
  PlaneRange r;
  r.seg_len = seg_len;
  r.b0 = zb;
  r.e0 = ze;
  r.nseg0 = (ze - zb + seg_len - 1) / seg_len;
  r.b1 = zb1;
  r.e1 = ze1 > zb1 ? ze1 : zb1;
  *nseg_total = r.nseg0 + (r.e1 - r.b1 + seg_len - 1) / seg_len;
  return r;
}

// Debug builds (tools/build_variant.sh dbg "-DOSBLI_DEBUG_CHECKS=1"): every staged
// global load is bounds-checked against its buffer, and shared-memory buffers are
// filled with NaN whenever they are handed back for reuse, so that a read racing a
// hand-off, or of data never written, turns into a NaN the parity tests see
// (compute-sanitizer is not available on this pool).
#ifndef OSBLI_DEBUG_CHECKS
#define OSBLI_DEBUG_CHECKS 0
#endif
// index i of an access into a buffer of n doubles
__device__ __forceinline__ bool dbg_in(const KParams &p, long long i, long long n) {
#if OSBLI_DEBUG_CHECKS
  if (i < 0 || i >= n) {
    if (p.dbg) atomicOr(p.dbg, 2u);
    return false;
  }
#endif
  return true;
}
__device__ __forceinline__ long long qbuf_len(const KParams &p) {
  return (long long)(p.nz + 2 * p.G) * 5 * p.nx * p.ny;
}
__device__ __forceinline__ double dbg_nan() { return __longlong_as_double(0x7ff8dead00000000ll); }

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
// #pragma unroll with a macro count (a count inside #pragma is not macro-expanded)
#define OSBLI_PRAGMA(x) _Pragma(#x)
#define OSBLI_UNROLL(n) OSBLI_PRAGMA(unroll n)
#ifndef OSBLI_STENCIL_CHAINS
#define OSBLI_STENCIL_CHAINS 1
#endif

// second derivatives in first differences (D-22); 0 selects the (f+ + f-) - 2f form
#ifndef OSBLI_D2_SBP
#define OSBLI_D2_SBP 1
#endif
}  // namespace
// TMA: bulk tensor copy of one box of a 4-D tensor (x, y, field, plane) into shared
// memory (128-byte aligned), completing on an mbarrier
__device__ __forceinline__ void tma_load_box(double *dst, const CUtensorMap *tm, int x, int y,
                                             int f, int zplane, uint64_t *bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(d),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(f), "r"(zplane), "r"(b)
      : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(b), "r"(parity)
      : "memory");
}


}  // namespace osbli
