// Dealiased Poisson bracket / nonlinear term and the standalone half-spectrum
// transforms (reference spectral.py:116-161 to_real/to_spectrum, 232-268 bracket,
// kernels.py:126-150 nonlinear_kernel) on B200.
//
// Pipeline per (velocity, theta) slice, x = radial (n_x padded), y = toroidal:
//   XINV  rows:    W+[ky] = IFFT_x((i kx' - ky) f[ky]),  W-[ky] = IFFT_x((i kx' + ky) f[ky])
//                  (kx' = derivative wavenumber, radial Nyquist zeroed; the two
//                  derivative fields travel as one complex field w = fx + i fy)
//   YCOL  columns: Z = [Re W+[0], W+[1..], 0.., conj(W-[..1])] -> IFFT_y -> w = fx + i fy
//                  p = fx*gy - fy*gx (unfused mul/mul/sub: exact antisymmetry and exact
//                  zero for f == g); two columns packed into one forward FFT_y;
//                  keep ky < n_ky
//   XFWD  rows:    FFT_x, keep the wrap-order kx columns, / (n_x n_y), zero the
//                  unpaired radial Nyquist column.
// The padded real fields never exist in memory; the only intermediate is the
// mixed (ky, x) representation, (2 n_ky - 1) x n_x complex per slice, in a
// ~1 GB chunk buffer reused chunk after chunk.  phi's derivative fields (g)
// come out of the very same XINV/YCOL code (bit-identical to f's) and are stored
// once per theta.  nonlinear_kernel walks slices theta-major, so the chunk in
// flight shares one theta and phi's fields for it stay L2-resident.
//
// Two implementations of the three stages:
//  * fixed  (fft_fixed.cuh): compile-time radices for the benchmark grids
//    (n_x in {720, 2016}, n_y in {144, 480, 864}); thread-per-butterfly, first
//    and last pass fused with global loads/stores.  XINV/XFWD run as independent
//    3-warp teams (named barriers, own persistent item loop, next row staged
//    with cp.async); YCOL interleaves 16 columns per CTA (conflict-free shared
//    memory, coalesced rows) and keeps phi's field block in shared memory.
//  * generic (fft_engine.cuh): any sizes, any radix (generic O(p^2) prime pass).
// A plan uses one or the other for all stages, so f's and g's fields always come
// from identical code.
//
// Taking Re of the ky=0 row reproduces irfft's projection of the (generally
// non-Hermitian) random state (spectral.py:136-137).
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "fft_fixed.cuh"
#include "../../include/gk.h"

#ifndef GK_XINV_WARPS
#define GK_XINV_WARPS 8
#endif
#ifndef GK_YCOL_WARPS
#define GK_YCOL_WARPS 8
#endif
#ifndef GK_YCOL_MINB
#define GK_YCOL_MINB 2
#endif
#ifndef GK_YCOL_FX_MINB
#define GK_YCOL_FX_MINB 2
#endif
#ifndef GK_YCOL_FX_GST
#define GK_YCOL_FX_GST true
#endif
#ifndef GK_YCOL_CLAMP
#define GK_YCOL_CLAMP false
#endif
#ifndef GK_XFWD_WARPS
#define GK_XFWD_WARPS 8
#endif

struct gk_spectral_plan {
  int64_t n_kx, n_ky, n_x, n_y;
  gk::fft::Desc dx, dy;
  double2* tw_dev;
  bool fixed;
};

namespace gk {
namespace spec {

constexpr int kThreads = 128;
constexpr int64_t kSmemElems = 2944;  // generic path: double2 per ping-pong half (~92 KB total)

enum YMode { Y_PHI = 0, Y_BRACKET = 1, Y_TO_REAL = 2, Y_TO_SPEC = 3 };

// Order in which the q-th slice of a batch is processed.  Theta-major (tm_T > 0):
// q -> (t = q / tm_M, v = q % tm_M), source/output slice v*T + t, g slice t.
struct Order {
  const int64_t* fmap;
  const int64_t* gmap;
  int64_t gmod;
  int64_t tm_M, tm_T;
};
// Slice and item counts are < 2^31 (checked on the host), so the per-item index
// math runs in 32-bit: a 64-bit division is a called subroutine on the GPU and
// showed up as a hot spot of the FFT kernels' item loops.
__device__ __forceinline__ int64_t ord_src(const Order& o, int64_t q) {
  if (o.tm_T) {
    const unsigned uq = (unsigned)q, m = (unsigned)o.tm_M;
    const unsigned t = uq / m;
    return (int64_t)(uq - t * m) * o.tm_T + t;
  }
  return o.fmap ? o.fmap[q] : q;
}
__device__ __forceinline__ int64_t ord_g(const Order& o, int64_t q) {
  if (o.tm_T) return (unsigned)q / (unsigned)o.tm_M;
  return o.gmap ? o.gmap[q] : (int64_t)((unsigned)q % (unsigned)o.gmod);
}
__device__ __forceinline__ int64_t ord_out(const Order& o, int64_t q) { return o.tm_T ? ord_src(o, q) : q; }

// Row layout of a spectral array of (slice, ky) rows of n_kx modes, as toroidal
// blocks of yl modes each living at its own base address: block b = ky / yl holds
// rows [slice][ky % yl][kx] at base[b].  Contiguous (the reference layout
// [slice][ky][kx]): one block, yl = n_ky.  A multi-GPU transpose's receive buffer
// [block][slice][ky % yl][kx]: base[b] = buffer + b * slices * yl rows; the rank's
// own block may point into its home shard, and (P2P transport) an output block
// into a peer GPU's memory.
constexpr int kMaxLayoutBlocks = 16;
struct Layout {
  int yl;
  const double2* base[kMaxLayoutBlocks];
};
// row (slice s, mode ky) in layout l, n_kx modes per row
template <class P>
__device__ __forceinline__ P lay_ptr(P, const Layout& l, int64_t s, int ky, int n_kx) {
  const unsigned b = (unsigned)ky / (unsigned)l.yl;
  return (P)l.base[b] + (s * l.yl + (ky - (int)b * l.yl)) * n_kx;
}
static Layout contiguous_layout(const void* p, int64_t n_ky) {
  Layout l{};
  l.yl = (int)n_ky;
  l.base[0] = (const double2*)p;
  return l;
}

struct XInvArgs {
  fft::Desc d;
  const double2* f;
  Layout lay;
  Order ord;
  double2* m1;
  int64_t s0, items;
  int nrow;  // transforms per slice (2Y-1 bracket, n_ky plain)
  int n_kx, n_ky;
  int bracket;
  int tb, groups;
};

struct YArgs {
  fft::Desc d;
  double2* m1;
  double2* G;
  Order ord;
  double* field_out;
  const double* field_in;
  int64_t s0, items;
  int nrow, n_ky, n_x;
  int mode;
  int cols, groups;
};

struct XFwdArgs {
  fft::Desc d;
  const double2* m1;
  double2* out;
  Layout lay;
  Order ord;
  int64_t s0, items;
  int nrow, n_ky, n_kx;
  double norm;  // n_x * n_y
  int tb, groups;
};


// wrap-order column j (0..n_kx-1) <-> padded slot i (0..n-1); -1 = not retained.
__device__ __forceinline__ int slot_to_kx(int i, int n, int n_kx) {
  const int pos = (n_kx + 1) / 2;  // kx >= 0 count
  if (i < pos) return i < n_kx ? i : -1;
  const int j = i - n + n_kx;
  return (j >= pos && j < n_kx) ? j : -1;
}
__device__ __forceinline__ int kx_to_slot(int j, int n, int n_kx) {
  return j < (n_kx + 1) / 2 ? j : j - n_kx + n;
}

// XINV input at padded slot i of transform t (already conjugated for the inverse);
// slice s of f in layout lay.
__device__ __forceinline__ double2 xinv_input(const double2* f, int64_t s, const Layout& lay, int i, int t, int n,
                                              int n_kx, int Y, bool bracket) {
  int j = slot_to_kx(i, n, n_kx);
  if ((n_kx % 2 == 0) && n > n_kx && j == n_kx / 2) j = -1;
  if (j < 0) return make_double2(0.0, 0.0);
  int ky = t;
  double re = 0.0;
  if (bracket) {
    ky = t < Y ? t : t - Y + 1;
    re = t < Y ? -(double)ky : (double)ky;
  }
  double2 v = lay_ptr(f, lay, s, ky, n_kx)[j];
  if (bracket) {
    double kxd = j < (n_kx + 1) / 2 ? (double)j : (double)(j - n_kx);
    if (n_kx % 2 == 0 && j == n_kx / 2) kxd = 0.0;
    v = cmul(make_double2(re, kxd), v);
  }
  return cconj(v);
}

// y-spectrum value k of a column from the XINV rows (bracket layout), given a
// row accessor.
template <class Row>
__device__ __forceinline__ double2 zb_bracket(Row row, int k, int n, int Y) {
  if (k == 0) return make_double2(row(0).x, 0.0);
  if (k < Y) return row(k);
  if (k > n - Y) return cconj(row(Y - 1 + (n - k)));
  return make_double2(0.0, 0.0);
}
// Hermitian extension of a half column (irfft semantics: Re of DC and Nyquist bins)
template <class Row>
__device__ __forceinline__ double2 zb_herm(Row row, int k, int n, int Y) {
  if (k == 0) return Y > 0 ? make_double2(row(0).x, 0.0) : make_double2(0.0, 0.0);
  if (2 * k < n) return k < Y ? row(k) : make_double2(0.0, 0.0);
  if (2 * k == n) return k < Y ? make_double2(row(k).x, 0.0) : make_double2(0.0, 0.0);
  const int m = n - k;
  return m < Y ? cconj(row(m)) : make_double2(0.0, 0.0);
}

__device__ __forceinline__ void separate(double2 za, double2 zb, double2& pa, double2& pb) {
  pa = make_double2(__dmul_rn(0.5, __dadd_rn(za.x, zb.x)), __dmul_rn(0.5, __dsub_rn(za.y, zb.y)));
  pb = make_double2(__dmul_rn(0.5, __dadd_rn(za.y, zb.y)), __dmul_rn(0.5, __dsub_rn(zb.x, za.x)));
}

__device__ __forceinline__ double product(double2 w, double2 g) {
  return __dsub_rn(__dmul_rn(w.x, g.y), __dmul_rn(w.y, g.x));
}

// ======================================================================== generic
// m1 layout (generic): [slice][x][t]  (column-contiguous); G: [g][x][y]

__global__ void __launch_bounds__(kThreads) xinv_kernel(const XInvArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  const int n = a.d.n, ld = n;
  const int sl = blockIdx.x / a.groups;
  const int t0 = (blockIdx.x - sl * a.groups) * a.tb;
  const int ntr = min(a.tb, a.nrow - t0);
  const int64_t ssrc = ord_src(a.ord, a.s0 + sl);
  double2* buf0 = sm;
  double2* buf1 = sm + a.tb * ld;
  for (int e = threadIdx.x; e < ntr * n; e += kThreads) {
    const int tt = e / n, i = e - tt * n;
    buf0[tt * ld + i] = xinv_input(a.f, ssrc, a.lay, i, t0 + tt, n, a.n_kx, a.n_ky, a.bracket);
  }
  __syncthreads();
  const double2* res = fft::run(a.d, buf0, buf1, ld, ntr, threadIdx.x, kThreads);
  double2* dst = a.m1 + (int64_t)sl * n * a.nrow + t0;
  for (int e = threadIdx.x; e < ntr * n; e += kThreads) {
    const int x = e / ntr, tt = e - x * ntr;
    dst[(int64_t)x * a.nrow + tt] = cconj(res[tt * ld + x]);
  }
}

__device__ __forceinline__ void separate_store(const double2* res, int ld, int n, int npair, int nc, int Y,
                                               double2* colbase, int nrow) {
  for (int e = threadIdx.x; e < npair * Y; e += kThreads) {
    const int q = e / Y, k = e - q * Y;
    double2 pa, pb;
    separate(res[q * ld + k], res[q * ld + (k == 0 ? 0 : n - k)], pa, pb);
    colbase[(int64_t)(2 * q) * nrow + k] = pa;
    if (2 * q + 1 < nc) colbase[(int64_t)(2 * q + 1) * nrow + k] = pb;
  }
}

__global__ void __launch_bounds__(kThreads) ycol_kernel(const YArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  const int n = a.d.n, ld = n;
  const int sl = blockIdx.x / a.groups;
  const int x0 = (blockIdx.x - sl * a.groups) * a.cols;
  const int nc = min(a.cols, a.n_x - x0);
  const int npair = (nc + 1) / 2;
  const int64_t q = a.s0 + sl;
  double2* buf0 = sm;
  double2* buf1 = sm + a.cols * ld;
  double2* colbase = a.m1 + ((int64_t)sl * a.n_x + x0) * a.nrow;
  const int Y = a.n_ky;

  if (a.mode == Y_PHI || a.mode == Y_BRACKET) {
    for (int e = threadIdx.x; e < nc * n; e += kThreads) {
      const int c = e / n, k = e - c * n;
      const double2* col = colbase + (int64_t)c * a.nrow;
      buf0[c * ld + k] = cconj(zb_bracket([&](int r) { return col[r]; }, k, n, Y));
    }
    __syncthreads();
    double2* res = fft::run(a.d, buf0, buf1, ld, nc, threadIdx.x, kThreads);
    if (a.mode == Y_PHI) {
      double2* g = a.G + (q * a.n_x + x0) * n;
      for (int e = threadIdx.x; e < nc * n; e += kThreads) {
        const int c = e / n, y = e - c * n;
        g[(int64_t)c * n + y] = cconj(res[c * ld + y]);
      }
      return;
    }
    const double2* g = a.G + (ord_g(a.ord, q) * a.n_x + x0) * n;
    double2* other = res == buf0 ? buf1 : buf0;
    for (int e = threadIdx.x; e < npair * n; e += kThreads) {
      const int qq = e / n, y = e - qq * n;
      const int ca = 2 * qq, cb = 2 * qq + 1;
      const double pa = product(cconj(res[ca * ld + y]), g[(int64_t)ca * n + y]);
      const double pb = cb < nc ? product(cconj(res[cb * ld + y]), g[(int64_t)cb * n + y]) : 0.0;
      other[qq * ld + y] = make_double2(pa, pb);
    }
    __syncthreads();
    const double2* res2 = fft::run(a.d, other, res, ld, npair, threadIdx.x, kThreads);
    separate_store(res2, ld, n, npair, nc, Y, colbase, a.nrow);
    return;
  }

  if (a.mode == Y_TO_REAL) {
    for (int e = threadIdx.x; e < npair * n; e += kThreads) {
      const int qq = e / n, k = e - qq * n;
      const double2* ca = colbase + (int64_t)(2 * qq) * a.nrow;
      const double2 za = zb_herm([&](int r) { return ca[r]; }, k, n, Y);
      double2 zb = make_double2(0.0, 0.0);
      if (2 * qq + 1 < nc) {
        const double2* cb = ca + a.nrow;
        zb = zb_herm([&](int r) { return cb[r]; }, k, n, Y);
      }
      buf0[qq * ld + k] = cconj(make_double2(__dsub_rn(za.x, zb.y), __dadd_rn(za.y, zb.x)));
    }
    __syncthreads();
    const double2* res = fft::run(a.d, buf0, buf1, ld, npair, threadIdx.x, kThreads);
    double* out = a.field_out + q * n * a.n_x + x0;
    for (int e = threadIdx.x; e < n * nc; e += kThreads) {
      const int y = e / nc, c = e - y * nc;
      const double2 r = res[(c >> 1) * ld + y];  // conj(r) -> (r.x, -r.y)
      out[(int64_t)y * a.n_x + c] = (c & 1) ? -r.y : r.x;
    }
    return;
  }

  // Y_TO_SPEC: real field columns, two per complex transform
  const double* in = a.field_in + q * n * a.n_x + x0;
  for (int e = threadIdx.x; e < npair * n; e += kThreads) {
    const int y = e / npair, qq = e - y * npair;
    const double pa = in[(int64_t)y * a.n_x + 2 * qq];
    const double pb = (2 * qq + 1 < nc) ? in[(int64_t)y * a.n_x + 2 * qq + 1] : 0.0;
    buf0[qq * ld + y] = make_double2(pa, pb);
  }
  __syncthreads();
  const double2* res = fft::run(a.d, buf0, buf1, ld, npair, threadIdx.x, kThreads);
  separate_store(res, ld, n, npair, nc, Y, colbase, a.nrow);
}

__global__ void __launch_bounds__(kThreads) xfwd_kernel(const XFwdArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  const int n = a.d.n, ld = n;
  const int sl = blockIdx.x / a.groups;
  const int k0 = (blockIdx.x - sl * a.groups) * a.tb;
  const int ntr = min(a.tb, a.n_ky - k0);
  double2* buf0 = sm;
  double2* buf1 = sm + a.tb * ld;
  const double2* srcb = a.m1 + (int64_t)sl * n * a.nrow + k0;
  for (int e = threadIdx.x; e < ntr * n; e += kThreads) {
    const int x = e / ntr, tt = e - x * ntr;
    buf0[tt * ld + x] = srcb[(int64_t)x * a.nrow + tt];
  }
  __syncthreads();
  const double2* res = fft::run(a.d, buf0, buf1, ld, ntr, threadIdx.x, kThreads);
  const bool nyq_zero = (a.n_kx % 2 == 0) && n > a.n_kx;
  const int64_t so = ord_out(a.ord, a.s0 + sl);
  for (int e = threadIdx.x; e < ntr * a.n_kx; e += kThreads) {
    const int tt = e / a.n_kx, j = e - tt * a.n_kx;
    double2 v = res[tt * ld + kx_to_slot(j, n, a.n_kx)];
    v = make_double2(__ddiv_rn(v.x, a.norm), __ddiv_rn(v.y, a.norm));
    if (nyq_zero && j == a.n_kx / 2) v = make_double2(0.0, 0.0);
    lay_ptr(a.out, a.lay, so, k0 + tt, a.n_kx)[j] = v;
  }
}

// ======================================================================== fixed
// m1 layout (fixed): [slice][t][x] (row-major); G: [g][y][x].
// Each CTA walks a contiguous range of work items and stages the next item's
// inputs into shared memory with cp.async while the current item's later FFT
// passes run (pass-0 hook), so the L2 latency of the chunk buffer is hidden.

__device__ __forceinline__ void item_range(int64_t items, int64_t& beg, int64_t& end) {
  const int64_t per = (items + gridDim.x - 1) / gridDim.x;
  beg = blockIdx.x * per;
  end = beg + per < items ? beg + per : items;
}

#ifdef GK_YCOL_STATS  // instrumented build for tools/ycol_stats.py
__managed__ unsigned long long g_ycol_stats[4 * 1024];
extern "C" unsigned long long* gk_ycol_stats() { return g_ycol_stats; }
#endif
// YCOL: item = (column group, slice) group-major; stages the item's m1 column
// block [t][c] (next item prefetched during the current inverse FFT) and keeps
// phi's field block [y][c] in shared memory for as long as the group and the
// theta stay the same (theta-major chunks: the whole run of slices).
template <class SY, int C, int MINB, bool GST>
__global__ void __launch_bounds__(C * SY::maxbf(), MINB) ycol_fx(const YArgs a) {
  constexpr int N = SY::N;
  constexpr int C2 = C / 2;
  static_assert(SY::P >= 2 && C % 2 == 0, "packed forward needs >= 2 passes and even C");
  extern __shared__ __align__(16) double2 sm[];
  double2* tw = sm;
  double2* data = tw + N;          // N*C complex
  double* pbuf = (double*)data;    // [y][c] reals: first half of data
  double2* fdata = data + N * C2;  // forward transforms: second half
  double2* zbuf = data;            // forward results [k][q2]: first half again
  double2* gst = data + N * C;               // phi fields [y][c] (GST)
  // m1 column block staged in y-bin order [k][c]: row t lands in bin t (t < Y)
  // or N - (t - Y + 1) (the conjugate half); the bins with no row (Y <= k <= N - Y)
  // are zeroed once here and never written again -- so the inverse transform's
  // input is one shared load plus a sign select, no row table.
  double2* mst = GST ? gst + N * C : gst;
  for (int i = threadIdx.x; i < N; i += blockDim.x) tw[i] = a.d.tw[i];
  for (int e = threadIdx.x; e < N * C; e += blockDim.x) {
    const int k = e / C;
    if (k >= a.n_ky && k <= N - a.n_ky) mst[e] = make_double2(0.0, 0.0);
  }
  const int c = threadIdx.x % C, j = threadIdx.x / C;
  const int q2 = threadIdx.x % C2, j2 = threadIdx.x / C2;
  const int Y = a.n_ky, n_x = a.n_x, nrow = a.nrow;
  const unsigned cs = (unsigned)(a.items / a.groups);
  int64_t beg, end;
  item_range(a.items, beg, end);
  // Staging: C divides blockDim, so thread e always copies column e % C of rows
  // e / C, e / C + RS, ... (RS = blockDim / C): a pointer walk, no per-copy index
  // math.  Items are consecutive per CTA: (group, slice) advance incrementally.
  const int RS = blockDim.x / C;
  const int scol = threadIdx.x % C, srow = threadIdx.x / C;
  auto prefetch = [&](unsigned grp, unsigned sl) {
    const int x0 = (int)grp * C;
    if (x0 + scol < n_x) {
      const double2* src = a.m1 + ((int64_t)sl * nrow + srow) * n_x + x0 + scol;
      const int64_t step = (int64_t)RS * n_x;
      for (int t = srow; t < nrow; t += RS, src += step) {
        const int k = t < Y ? t : N - (t - Y + 1);
        fftx::cp16(mst + k * C + scol, src);
      }
    }
    fftx::cp_commit();
  };
  unsigned grp = beg < end ? (unsigned)beg / cs : 0, sl = beg < end ? (unsigned)beg - grp * cs : 0;
  if (beg < end) prefetch(grp, sl);
  int64_t cur_grp = -1, cur_gi = -1;
  for (int64_t item = beg; item < end; ++item, (sl + 1 == cs) ? (sl = 0, ++grp) : ++sl) {
    const unsigned ngrp = sl + 1 == cs ? grp + 1 : grp, nsl = sl + 1 == cs ? 0 : sl + 1;
    const int x0 = (int)grp * C;
    const int x = x0 + c;
    const bool valid = x < n_x;
    const int64_t q = a.s0 + sl;
    double2* rows = a.m1 + (int64_t)sl * nrow * n_x;
#ifdef GK_YCOL_STATS
    const long long c0 = clock64();
#endif
    fftx::cp_wait_all();
    __syncthreads();
#ifdef GK_YCOL_STATS
    const long long c1 = clock64();
#endif
    const int64_t gq = a.mode == Y_BRACKET ? ord_g(a.ord, q) : 0;
    if (GST && a.mode == Y_BRACKET) {
      const int64_t gi = gq;
      if (gi != cur_gi || grp != cur_grp) {
        const double2* g = a.G + gi * (int64_t)N * n_x + x0;
        for (int e = threadIdx.x; e < N * C; e += blockDim.x) {
          const int y = e / C, cc = e - y * C;
          if (x0 + cc < n_x) fftx::cp16(gst + e, g + (int64_t)y * n_x + cc);
        }
        fftx::cp_commit();
        fftx::cp_wait_all();
        __syncthreads();
        cur_gi = gi;
        cur_grp = grp;
      }
    }
    // conj(Z[k]) of the Hermitian-extended column (== zb_bracket), from the
    // bin-ordered staging; branch-free
    auto load = [&](int k) {
      const double2 v = mst[k * C + c];  // empty bins hold zeros
      const double re = valid ? v.x : 0.0;
      const double im = (!valid || k == 0) ? 0.0 : (k < Y ? -v.y : v.y);
      return make_double2(re, im);
    };
#ifdef GK_YCOL_STATS
    long long ch = 0, ch2 = 0;
#endif
    auto hook = [&]() {
#ifdef GK_YCOL_STATS
      ch = clock64();
#endif
      if (item + 1 < end) prefetch(ngrp, nsl);
#ifdef GK_YCOL_STATS
      ch2 = clock64();
#endif
    };
    if (a.mode == Y_PHI) {
      double2* g = a.G + q * (int64_t)N * n_x + x;
      auto store = [&](int y, double2 v) {
        if (valid) g[(int64_t)y * n_x] = cconj(v);
      };
      fftx::transform<SY, C, GK_YCOL_CLAMP>(data, c, j, tw, load, store, hook);
      continue;
    }
    const double2* gglob = a.G + gq * (int64_t)N * n_x + x;
    auto store = [&](int y, double2 v) {
      double p = 0.0;
      if constexpr (GST) {  // staged block: always in bounds, select instead of branching
        const double q = product(cconj(v), gst[y * C + c]);
        p = valid ? q : 0.0;
      } else {
        if (valid) p = product(cconj(v), gglob[(int64_t)y * n_x]);
      }
      pbuf[y * C + c] = p;
    };
    fftx::transform<SY, C, GK_YCOL_CLAMP>(data, c, j, tw, load, store, hook);
    __syncthreads();
#ifdef GK_YCOL_STATS
    const long long c2 = clock64();
#endif
    auto load2 = [&](int y) { return reinterpret_cast<const double2*>(pbuf + y * C)[q2]; };  // columns 2q2, 2q2+1
    auto store2 = [&](int k, double2 v) { zbuf[k * C2 + q2] = v; };
    fftx::transform<SY, C2, GK_YCOL_CLAMP>(fdata, q2, j2, tw, load2, store2);
    __syncthreads();
#ifdef GK_YCOL_STATS
    const long long c3 = clock64();
#endif
    for (int e = threadIdx.x; e < C2 * Y; e += blockDim.x) {
      const int k = e / C2, qq = e - k * C2;
      double2 pa, pb;
      separate(zbuf[k * C2 + qq], zbuf[(k == 0 ? 0 : N - k) * C2 + qq], pa, pb);
      const int xa = x0 + 2 * qq;
      if (xa < n_x) rows[(int64_t)k * n_x + xa] = pa;
      if (xa + 1 < n_x) rows[(int64_t)k * n_x + xa + 1] = pb;
    }
#ifdef GK_YCOL_STATS  // per CTA: [wait, inverse, forward, separate], then [pass 0, prefetch issue, pass 1]
    if (threadIdx.x == 0 && a.mode == Y_BRACKET) {
      const long long c4 = clock64();
      unsigned long long* st = g_ycol_stats + 4 * blockIdx.x;
      atomicAdd(st + 0, (unsigned long long)(c1 - c0));
      atomicAdd(st + 1, (unsigned long long)(c2 - c1));
      atomicAdd(st + 2, (unsigned long long)(c3 - c2));
      atomicAdd(st + 3, (unsigned long long)(c4 - c3));
      unsigned long long* sp = g_ycol_stats + 4 * 296 + 3 * blockIdx.x;
      atomicAdd(sp + 0, (unsigned long long)(ch - c1));
      atomicAdd(sp + 1, (unsigned long long)(ch2 - ch));
      atomicAdd(sp + 2, (unsigned long long)(c2 - ch2));
    }
#endif
  }
}

// YCOL for n_y = 144 = 12 * 12 (the sh03b plan), square four-step with the
// product kept in registers.  Thread (column c, j): inverse pass 0 reads bins
// j + 12 r, inverse pass 1 yields y = j + 12 r -- exactly the inputs forward pass 0
// needs -- so the product p(y) never goes through shared memory, each column gets
// its own (real-input) forward transform with all threads busy, no packing and no
// separation pass, and forward pass 1 stores k = j + 12 r, r < KEEP (ky < n_ky <=
// 48) straight to the mixed-spectrum rows (the other outputs are dead code).
// Bins 48..95 are empty for every n_ky <= 48 (the bracket's dealias bound at
// n_y = 144), so inverse pass 0 skips them: r = 4..7 are compile-time zeros.
// 4 CTA barriers per item (ycol_fx: 7).  f's and g's fields (Y_PHI) come from the
// same inverse code.
// FULL: n_x is a multiple of C (sh03b: 720 = 45 x 16), every column valid -- the
// bounds selects and branches compile away.  CPT: columns per thread (1: C * 12
// threads; 2: C * 6 threads, each running two independent column transforms
// interleaved -- twice the ILP per thread, half the warps, barriers over half as
// many warps; GK_YSQ_CPT=2 for A/B).
template <int C, int MINB, bool FULL = false, int CPT = 1>
__global__ void __launch_bounds__(C / CPT * 12, MINB) ycol_sq(const YArgs a) {
  constexpr int R = 12, N = R * R, KEEP = 4, CT = C / CPT;  // CT: thread columns
  constexpr unsigned ZIN = 0xF0u;  // r = 4..7: bins 48..95
  static_assert(KEEP * R == 48 && (ZIN & ((1u << KEEP) - 1)) == 0, "n_ky <= 48 layout");
  static_assert(C % CPT == 0, "columns per thread");
  extern __shared__ __align__(16) double2 sm[];
  double2* tw = sm;
  double2* data = tw + N;     // [N][C] transform buffer
  double2* gst = data + N * C;  // phi fields [y][c]
  double2* mst = gst + N * C;   // m1 column block in y-bin order [k][c]
  for (int i = threadIdx.x; i < N; i += blockDim.x) tw[i] = a.d.tw[i];
  for (int e = threadIdx.x; e < N * C; e += blockDim.x) {
    const int k = e / C;
    if (k >= a.n_ky && k <= N - a.n_ky) mst[e] = make_double2(0.0, 0.0);
  }
  const int c = threadIdx.x % CT, j = threadIdx.x / CT;  // columns c + CT u, u < CPT
  const int Y = a.n_ky, n_x = a.n_x, nrow = a.nrow;
  const unsigned cs = (unsigned)(a.items / a.groups);
  int64_t beg, end;
  item_range(a.items, beg, end);
  // pass-1 twiddles W_144^{j r} straight from the table (j r < 144): one broadcast
  // shared load each instead of FP64 products (the FP64 pipe is the limiter here)
  auto twiddle_tab = [&](double2* v) {
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[j * r]);
  };
  constexpr int RS = R;  // rows per staging sweep (blockDim / CT)
  auto prefetch = [&](unsigned grp, unsigned sl) {
    const int x0 = (int)grp * C;
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
      const int cc = c + CT * u;
      if (FULL || x0 + cc < n_x) {
        const double2* src = a.m1 + ((int64_t)sl * nrow + j) * n_x + x0 + cc;
        const int64_t step = (int64_t)RS * n_x;
        for (int t = j; t < nrow; t += RS, src += step) {
          const int k = t < Y ? t : N - (t - Y + 1);
          fftx::cp16(mst + k * C + cc, src);
        }
      }
    }
    fftx::cp_commit();
  };
  unsigned grp = beg < end ? (unsigned)beg / cs : 0, sl = beg < end ? (unsigned)beg - grp * cs : 0;
  if (beg < end) prefetch(grp, sl);
  unsigned g_t = 0, g_r = 0, g_sl = 0;
  bool g_have = false;
  int64_t cur_grp = -1, cur_gi = -1;
  for (int64_t item = beg; item < end; ++item, (sl + 1 == cs) ? (sl = 0, ++grp) : ++sl) {
    const unsigned ngrp = sl + 1 == cs ? grp + 1 : grp, nsl = sl + 1 == cs ? 0 : sl + 1;
    const int x0 = (int)grp * C;
    bool valid[CPT];
#pragma unroll
    for (int u = 0; u < CPT; ++u) valid[u] = FULL || x0 + c + CT * u < n_x;
    const int64_t q = a.s0 + sl;
    fftx::cp_wait_all();
    __syncthreads();
    // phi slice of q: theta-major chunks advance q by one per item within a
    // column group, so the theta (q / M) is tracked without a division per item
    int64_t gq = 0;
    if (a.mode == Y_BRACKET) {
      if (a.ord.tm_T) {
        if (g_have && sl == g_sl + 1) {
          if (++g_r == (unsigned)a.ord.tm_M) g_r = 0, ++g_t;
        } else {
          const unsigned uq = (unsigned)q;
          g_t = uq / (unsigned)a.ord.tm_M;
          g_r = uq - g_t * (unsigned)a.ord.tm_M;
        }
        g_have = true;
        g_sl = sl;
        gq = g_t;
      } else {
        gq = ord_g(a.ord, q);
      }
    }
    if (a.mode == Y_BRACKET && (gq != cur_gi || grp != cur_grp)) {
      const double2* g = a.G + gq * (int64_t)N * n_x + x0;
      for (int e = threadIdx.x; e < N * C; e += blockDim.x) {
        const int y = e / C, cc = e - y * C;
        if (FULL || x0 + cc < n_x) fftx::cp16(gst + e, g + (int64_t)y * n_x + cc);
      }
      fftx::cp_commit();
      fftx::cp_wait_all();
      __syncthreads();
      cur_gi = gq;
      cur_grp = grp;
    }
    // inverse pass 0: conj(Z[k]) of the Hermitian-extended column, k = j + 12 r.
    // r < 4: k < 48, a row bin (k < Y) or an empty one -> -Im; r >= 8: k >= 96 > Y,
    // a conjugate bin -> +Im (compile-time signs: the negation folds into the
    // first butterfly instead of a select).  Columns past n_x transform whatever
    // the buffer holds: columns never mix, and their product is zeroed below.
    double2 v[CPT][R];
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (ZIN >> r & 1u) {
          v[u][r] = make_double2(0.0, 0.0);
        } else {
          const double2 m = mst[(j + R * r) * C + c + CT * u];
          if (r == 0) v[u][r] = make_double2(m.x, j == 0 ? 0.0 : -m.y);
          else v[u][r] = make_double2(m.x, r < KEEP ? -m.y : m.y);
        }
      }
      fft::dft12_z<ZIN>(v[u]);
    }
#pragma unroll
    for (int u = 0; u < CPT; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) data[(j * R + r) * C + c + CT * u] = v[u][r];
    __syncthreads();
    if (item + 1 < end) prefetch(ngrp, nsl);  // mst is free: every pass-0 read is done
    // inverse pass 1 -> y = j + 12 r
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[u][r] = data[(j + R * r) * C + c + CT * u];
      twiddle_tab(v[u]);
      fft::dft<R>(v[u]);
    }
    if (a.mode == Y_PHI) {
#pragma unroll
      for (int u = 0; u < CPT; ++u) {
        double2* g = a.G + q * (int64_t)N * n_x + x0 + c + CT * u;
        if (valid[u]) {
#pragma unroll
          for (int r = 0; r < R; ++r) g[(int64_t)(j + R * r) * n_x] = cconj(v[u][r]);
        }
      }
      continue;
    }
    double p[CPT][R];
#pragma unroll
    for (int u = 0; u < CPT; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double pr = product(cconj(v[u][r]), gst[(j + R * r) * C + c + CT * u]);
        p[u][r] = valid[u] ? pr : 0.0;
      }
    __syncthreads();  // every pass-1 read of data is done
    // forward pass 0 (real input p)
#pragma unroll
    for (int u = 0; u < CPT; ++u) fft::dft12_real(p[u], v[u]);
#pragma unroll
    for (int u = 0; u < CPT; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) data[(j * R + r) * C + c + CT * u] = v[u][r];
    __syncthreads();
    // forward pass 1 -> k = j + 12 r; keep k < Y (r < KEEP)
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[u][r] = data[(j + R * r) * C + c + CT * u];
      twiddle_tab(v[u]);
      fft::dft<R>(v[u]);
      double2* rows = a.m1 + (int64_t)sl * nrow * n_x + x0 + c + CT * u;
#pragma unroll
      for (int r = 0; r < KEEP; ++r) {
        const int k = j + R * r;
        if (valid[u] && k < Y) rows[(int64_t)k * n_x] = v[u][r];
      }
    }
  }
}

// YCOL for n_y = P * Q (480 = 20 * 24, the C5a multiscale plan), rectangular
// four-step with the product in registers, the ycol_sq scheme for a non-square
// size.  Thread (column c, j), j < max(P, Q):
//   inverse pass 0 (j = a < P):  Q-point DFT of bins a + P b  -> A_a[s]
//   inverse pass 1 (j = s < Q):  x W_N^{a s}, P-point DFT over a -> y = s + Q t
//   product p(y) in registers; phi's fields g(y) read through L2 (theta-major
//   chunks keep the theta's N x n_x block resident)
//   forward pass 0 (j = s < Q):  P-point DFT over t of the real p(s + Q t) -> B_s[u]
//   forward pass 1 (j = u < P):  x W_N^{s u}, Q-point DFT over s -> k = u + P v,
//   stored for k < n_ky (v < KV; the other outputs are dead code).
// Bins P b .. P b + P - 1 with b in [ZB0, ZB1) lie in the band that is empty for
// every n_ky the dealias bound admits, so they are compile-time zeros and have
// no staging slots: the m1 column block is staged as Q - (ZB1 - ZB0) slots of
// P bins, which (with the transpose buffer) lets two 8-column CTAs share an SM.
template <int P, int Q, int ZB0, int ZB1, int KV, int C, int MINB>
__global__ void __launch_bounds__(C * (P > Q ? P : Q), MINB) ycol_rect(const YArgs a) {
  constexpr int N = P * Q, TPC = P > Q ? P : Q, NSLOT = Q - (ZB1 - ZB0);
  extern __shared__ __align__(16) double2 sm[];
  double2* tw = sm;           // W_N^m, m < N
  double2* data = tw + N;     // [N][C] transpose buffer
  double2* mst = data + N * C;  // staged bins [slot][a][c], slot = b (b < ZB0) or b - (ZB1 - ZB0)
  for (int i = threadIdx.x; i < N; i += blockDim.x) tw[i] = a.d.tw[i];
  const int Y = a.n_ky, n_x = a.n_x, nrow = a.nrow;
  for (int e = threadIdx.x; e < NSLOT * P * C; e += blockDim.x) {
    const int sl = e / (P * C), aa = (e / C) % P;
    const int k = aa + P * (sl < ZB0 ? sl : sl + (ZB1 - ZB0));
    if (k >= Y && k <= N - Y) mst[e] = make_double2(0.0, 0.0);
  }
  const int c = threadIdx.x % C, j = threadIdx.x / C;
  const unsigned cs = (unsigned)(a.items / a.groups);
  int64_t beg, end;
  item_range(a.items, beg, end);
  auto slot_of = [](int k) {  // staging offset of bin k (never in the empty band)
    const int b = k / P, aa = k - b * P;
    return ((b < ZB0 ? b : b - (ZB1 - ZB0)) * P + aa) * C;
  };
  auto prefetch = [&](unsigned grp, unsigned sl) {
    const int x0 = (int)grp * C;
    if (x0 + c < n_x) {
      const double2* src = a.m1 + ((int64_t)sl * nrow + j) * n_x + x0 + c;
      const int64_t step = (int64_t)TPC * n_x;
      for (int t = j; t < nrow; t += TPC, src += step) {
        const int k = t < Y ? t : N - (t - Y + 1);
        fftx::cp16(mst + slot_of(k) + c, src);
      }
    }
    fftx::cp_commit();
  };
  unsigned grp = beg < end ? (unsigned)beg / cs : 0, sl = beg < end ? (unsigned)beg - grp * cs : 0;
  if (beg < end) prefetch(grp, sl);
  for (int64_t item = beg; item < end; ++item, (sl + 1 == cs) ? (sl = 0, ++grp) : ++sl) {
    const unsigned ngrp = sl + 1 == cs ? grp + 1 : grp, nsl = sl + 1 == cs ? 0 : sl + 1;
    const int x = (int)grp * C + c;
    const bool valid = x < n_x;
    const int64_t q = a.s0 + sl;
    fftx::cp_wait_all();
    __syncthreads();
    // inverse pass 0: conj(Z[k]) of the Hermitian-extended column, k = a + P b.
    // b < ZB0: k < Y_max, a row bin (or empty) -> -Im; b >= ZB1: a conjugate bin
    // (or empty) -> +Im; k = 0 takes Re only.
    if (j < P) {
      double2 v[Q];
#pragma unroll
      for (int b = 0; b < Q; ++b) {
        if (b >= ZB0 && b < ZB1) {
          v[b] = make_double2(0.0, 0.0);
        } else {
          const double2 m = mst[((b < ZB0 ? b : b - (ZB1 - ZB0)) * P + j) * C + c];
          if (b == 0) v[b] = make_double2(m.x, j == 0 ? 0.0 : -m.y);
          else v[b] = make_double2(m.x, b < ZB0 ? -m.y : m.y);
        }
      }
      if constexpr (Q == 24 && ZB0 == 8 && ZB1 == 16) fft::dft24_z<0xFF00u>(v);  // the band's zeros skipped
      else fft::dft<Q>(v);
#pragma unroll
      for (int s2 = 0; s2 < Q; ++s2) data[(j * Q + s2) * C + c] = v[s2];
    }
    __syncthreads();
    if (item + 1 < end) prefetch(ngrp, nsl);  // mst is free: every pass-0 read is done
    double p[P];
    if (j < Q) {
      double2 u[P];
#pragma unroll
      for (int r = 0; r < P; ++r) {
        u[r] = data[(r * Q + j) * C + c];
        if (r) u[r] = cmul(u[r], tw[r * j]);
      }
      fft::dft<P>(u);  // y = j + Q t
      if (a.mode == Y_PHI) {
        double2* g = a.G + q * (int64_t)N * n_x + x;
        if (valid) {
#pragma unroll
          for (int t = 0; t < P; ++t) g[(int64_t)(j + Q * t) * n_x] = cconj(u[t]);
        }
      } else {
        const double2* g = a.G + ord_g(a.ord, q) * (int64_t)N * n_x + (valid ? x : 0);
#pragma unroll
        for (int t = 0; t < P; ++t) {
          const double pr = product(cconj(u[t]), __ldg(g + (int64_t)(j + Q * t) * n_x));
          p[t] = valid ? pr : 0.0;
        }
      }
    }
    if (a.mode == Y_PHI) continue;  // uniform per launch
    __syncthreads();  // every pass-1 read of data is done
    if (j < Q) {  // forward pass 0 (real input p)
      double2 v[P];
#pragma unroll
      for (int t = 0; t < P; ++t) v[t] = make_double2(p[t], 0.0);
      fft::dft<P>(v);
#pragma unroll
      for (int u = 0; u < P; ++u) data[(j * P + u) * C + c] = v[u];
    }
    __syncthreads();
    if (j < P) {  // forward pass 1 -> k = j + P v; keep k < Y (v < KV)
      double2 w[Q];
#pragma unroll
      for (int s2 = 0; s2 < Q; ++s2) {
        w[s2] = data[(s2 * P + j) * C + c];
        if (s2) w[s2] = cmul(w[s2], tw[s2 * j]);
      }
      fft::dft<Q>(w);
      double2* rows = a.m1 + (int64_t)sl * nrow * n_x + x;
#pragma unroll
      for (int v2 = 0; v2 < KV; ++v2) {
        const int k = j + P * v2;
        if (valid && k < Y) rows[(int64_t)k * n_x] = w[v2];
      }
    }
  }
}

// (slice, row) of a warp's work items item, item + step, ... without a division
// per item: the per-step increments are split once.
struct RowCursor {
  unsigned sl, t, dsl, dt, n;
  __device__ __forceinline__ RowCursor(unsigned item, unsigned step, unsigned rows) : n(rows) {
    sl = item / n;
    t = item - sl * n;
    dsl = step / n;
    dt = step - dsl * n;
  }
  __device__ __forceinline__ void advance() {
    t += dt;
    sl += dsl;
    if (t >= n) {
      t -= n;
      ++sl;
    }
  }
};

// four-step twiddles W_N^{n2 k1} laid out [k1][n2] (lane n2 reads consecutive slots)
template <int N1, int N2>
__device__ __forceinline__ void init_tw4(double2* tw4, const double2* tw) {
  for (int i = threadIdx.x; i < N1 * N2; i += blockDim.x) {
    const int k1 = i / N2, n2 = i - k1 * N2;
    tw4[i] = tw[n2 * k1];  // n2 * k1 < N1 * N2
  }
}

// Warp YCOL for n_y = 144 = 12 * 12 (four-step, fftx::warp4 layout): a warp owns
// four adjacent x columns of one slice.  Lanes 0-11 and 12-23 each transform one
// column (two rounds: columns x0, x0+1 then x0+2, x0+3), so every global access
// -- the mixed-spectrum rows, phi's fields, the output rows -- is a 32-byte
// sector holding two adjacent columns and nothing is staged through the CTA.
// After the inverse, lane k1 holds y = k1 + 12 k2, which is exactly the input
// set of forward phase 1 (n = n2 + 12 n1): the product and the packing of two
// columns into one forward transform (lanes 0-11: x0 + i x0+1, lanes 12-23:
// x0+2 + i x0+3) stay in registers (one shuffle); the separation partner
// Z[N - k] comes from the mirror lane by shuffle as well.
template <int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) ycol_w12(const YArgs a) {
  constexpr int R = 12, N = R * R, ZP = R + 1, ZS = R * ZP;
  extern __shared__ __align__(16) double2 sm[];
  double2* tw4 = sm;                                       // [k1][n2] = W_144^{n2 k1}
  int2* ytab = reinterpret_cast<int2*>(tw4 + N);           // k -> (row, 0 conj / 1 as is / 2 real / 3 zero)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* zx = tw4 + N + N / 2 + warp * 2 * ZS;
  init_tw4<R, R>(tw4, a.d.tw);
  const int Y = a.n_ky, n_x = a.n_x, nrow = a.nrow;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    int2 e = make_int2(0, 3);
    if (i == 0) e = make_int2(0, Y > 0 ? 2 : 3);
    else if (i < Y) e = make_int2(i, 0);
    else if (i > N - Y) e = make_int2(Y - 1 + (N - i), 1);
    ytab[i] = e;
  }
  __syncthreads();
  const int h = lane >= R ? 1 : 0;
  const int r = lane < 2 * R ? lane - R * h : 0;  // lanes 24-31 idle (shadow lane 0's slots)
  const bool act = lane < 2 * R;
  double2* zh = zx + h * ZS;
  const unsigned quads = (unsigned)(n_x / 4);
  const unsigned step = gridDim.x * WARPS;
  for (unsigned item = blockIdx.x * WARPS + warp; item < (unsigned)a.items; item += step) {
    const unsigned sl = item / quads;
    const int x0 = (int)(item - sl * quads) * 4;
    const int64_t q = a.s0 + sl;
    double2* rows = a.m1 + (int64_t)sl * nrow * n_x;
    const int64_t gq = a.mode == Y_BRACKET ? ord_g(a.ord, q) : 0;
    double pr[2][R];
#pragma unroll
    for (int rd = 0; rd < 2; ++rd) {
      const int x = x0 + 2 * rd + h;
      double2 v[R];
      if (act) {
#pragma unroll
        for (int n1 = 0; n1 < R; ++n1) {
          const int2 e = ytab[R * n1 + r];
          const double2 w = rows[(int64_t)e.x * n_x + x];
          // conj(Z[k]) of the Hermitian-extended column (== zb_bracket), branch-free
          v[n1] = make_double2(e.y == 3 ? 0.0 : w.x, e.y == 0 ? -w.y : (e.y == 1 ? w.y : 0.0));
        }
        fft::dft<R>(v);
#pragma unroll
        for (int k1 = 1; k1 < R; ++k1) v[k1] = cmul(v[k1], tw4[k1 * R + r]);
#pragma unroll
        for (int k1 = 0; k1 < R; ++k1) zh[k1 * ZP + r] = v[k1];
      }
      __syncwarp();
      if (act) {
#pragma unroll
        for (int n2 = 0; n2 < R; ++n2) v[n2] = zh[r * ZP + n2];
        fft::dft<R>(v);  // lane r: y = r + 12 k2
        if (a.mode == Y_PHI) {
          double2* g = a.G + q * (int64_t)N * n_x + x;
#pragma unroll
          for (int k2 = 0; k2 < R; ++k2) g[(int64_t)(r + R * k2) * n_x] = cconj(v[k2]);
        } else {
          const double2* g = a.G + gq * (int64_t)N * n_x + x;
#pragma unroll
          for (int k2 = 0; k2 < R; ++k2) pr[rd][k2] = product(cconj(v[k2]), g[(int64_t)(r + R * k2) * n_x]);
        }
      }
      __syncwarp();
    }
    if (a.mode == Y_PHI) continue;
    // pack: lanes 0-11 (x0 + i x0+1), lanes 12-23 (x0+2 + i x0+3)
    double2 z[R];
#pragma unroll
    for (int k2 = 0; k2 < R; ++k2) {
      const double got = __shfl_sync(0xffffffffu, h ? pr[0][k2] : pr[1][k2], h ? lane - R : lane + R);
      z[k2] = h ? make_double2(got, pr[1][k2]) : make_double2(pr[0][k2], got);
    }
    if (act) {
      fft::dft<R>(z);
#pragma unroll
      for (int k1 = 1; k1 < R; ++k1) z[k1] = cmul(z[k1], tw4[k1 * R + r]);
#pragma unroll
      for (int k1 = 0; k1 < R; ++k1) zh[k1 * ZP + r] = z[k1];
    }
    __syncwarp();
    if (act) {
#pragma unroll
      for (int n2 = 0; n2 < R; ++n2) z[n2] = zh[r * ZP + n2];
      fft::dft<R>(z);  // lane r: Z[r + 12 k2]
    }
    __syncwarp();
    // separation: Z[N - k] for k = r + 12 k2 (k2 < 4 covers k < 48 >= Y) sits in
    // lane 12 - r at index 11 - k2 (r > 0) or in lane 0 at index (12 - k2) % 12.
    const int mirror = h * R + (R - r) % R;
    double2* xr = rows + x0 + 2 * h;
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      const double2 zm = z[R - 1 - k2];
      double2 zb = make_double2(__shfl_sync(0xffffffffu, zm.x, mirror), __shfl_sync(0xffffffffu, zm.y, mirror));
      if (r == 0) zb = z[(R - k2) % R];
      const int k = r + R * k2;
      if (act && k < Y) {
        double2 pa, pb;
        separate(z[k2], zb, pa, pb);
        xr[(int64_t)k * n_x] = pa;
        xr[(int64_t)k * n_x + 1] = pb;
      }
    }
  }
}

// Team variants of XINV / XFWD: each 3-warp team owns one transform at a time
// and walks its own persistent item sequence (named barriers only), so teams
// never wait for each other; the next item's input row is staged with cp.async
// during the current item's later passes.
template <class SX>
struct TeamGeom {
  static constexpr int TP = (SX::maxbf() + 31) / 32 * 32;  // threads per team
  // transform buffer padding (fftx::sidx): one slot per 12 for 2016 = 12 x 12 x 14
  // (its Stockham stores are 4- and 3-way bank conflicts unpadded)
  static constexpr int PADW = SX::N == 2016 ? 12 : 0;
  static constexpr int DATA = SX::N + (PADW ? SX::N / PADW : 0);  // buffer elements
  // compact inter-pass twiddle table (fftx::init_twc): 156 entries instead of 2016
  static constexpr bool TWC = SX::N == 2016;
  static constexpr int TWS = TWC ? SX::twc_size() : SX::N;
};

template <class SX, int TEAMS, int MINB>
__global__ void __launch_bounds__(TEAMS * TeamGeom<SX>::TP, MINB) xinv_tm(const XInvArgs a) {
  using G = TeamGeom<SX>;
  constexpr int N = SX::N, TP = G::TP;
  extern __shared__ __align__(16) double2 sm[];
  double2* tw = sm;
  double* kxd = reinterpret_cast<double*>(tw + G::TWS);  // slot -> derivative wavenumber
  const int team = threadIdx.x / TP, j = threadIdx.x - team * TP;
  const int nkx = a.n_kx, Y = a.n_ky, nrow = a.nrow;
  double2* data = tw + G::TWS + (N + 1) / 2 + team * (G::DATA + N);
  double2* stg = data + G::DATA;  // the staged f row in padded-slot order
  const int pos = (nkx + 1) / 2;  // slots [0,pos) and [hi,N) carry modes
  const int hi = N - (nkx - pos);
  const bool nyq_zero = (nkx % 2 == 0) && N > nkx;
  if constexpr (G::TWC) {
    fftx::init_twc<SX>(tw, a.d.tw);
  } else {
    for (int i = threadIdx.x; i < N; i += blockDim.x) tw[i] = a.d.tw[i];
  }
  for (int i = threadIdx.x; i < N; i += blockDim.x) kxd[i] = (double)(i < pos ? i : i - N);
  // slots that never carry a mode (the padding gap, the zeroed radial Nyquist) are
  // zeroed once; the staging writes the modes straight into their slots, so the
  // transform's input is one shared load (no slot -> mode table in the chain)
  for (int i = j; i < N; i += TP)
    if (i >= pos && (i < hi || (nyq_zero && i == hi))) stg[i] = make_double2(0.0, 0.0);
  __syncthreads();
  const fftx::TeamSync sync{team + 1, TP};
  const unsigned step = gridDim.x * TEAMS;
  auto prefetch = [&](unsigned item) {
    if (item >= (unsigned)a.items) return;
    const unsigned sl = item / (unsigned)nrow;
    const int t = (int)(item - sl * (unsigned)nrow);
    const int ky = t < Y ? t : t - Y + 1;
    const double2* src = lay_ptr(a.f, a.lay, ord_src(a.ord, a.s0 + sl), ky, nkx);
    for (int e = j; e < nkx; e += TP) {
      const int slot = e < pos ? e : e - pos + hi;
      if (!(nyq_zero && e == nkx / 2)) fftx::cp16(stg + slot, src + e);
    }
    fftx::cp_commit();
  };
  unsigned item = blockIdx.x * TEAMS + team;
  prefetch(item);
  for (; item < (unsigned)a.items; item += step) {
    const unsigned sl = item / (unsigned)nrow;
    const int t = (int)(item - sl * (unsigned)nrow);
    const bool minus = t >= Y;
    const int ky = minus ? t - Y + 1 : t;
    const double re = minus ? (double)ky : -(double)ky;
    double2* dst = a.m1 + ((int64_t)sl * nrow + t) * N;
    fftx::cp_wait_all();
    sync();
    // (i kx' -/+ ky) f at padded slot i, conjugated for the inverse; empty slots are 0
    auto load = [&](int i) { return cconj(cmul(make_double2(re, kxd[i]), stg[i])); };
    auto store = [&](int i, double2 v) { dst[i] = cconj(v); };
    auto hook = [&]() { prefetch(item + step); };
    fftx::transform_team<SX, G::PADW, G::TWC>(data, j, tw, load, store, hook, sync);
  }
}

template <class SX, int TEAMS, int MINB>
__global__ void __launch_bounds__(TEAMS * TeamGeom<SX>::TP, MINB) xfwd_tm(const XFwdArgs a) {
  using G = TeamGeom<SX>;
  constexpr int N = SX::N, TP = G::TP;
  extern __shared__ __align__(16) double2 sm[];
  double2* tw = sm;
  int* otab = reinterpret_cast<int*>(tw + G::TWS);  // slot -> output kx column, -1 dropped, -2 zero (Nyquist)
  const int team = threadIdx.x / TP, j = threadIdx.x - team * TP;
  double2* data = tw + G::TWS + (N + 3) / 4 + team * (G::DATA + N);
  double2* stg = data + G::DATA;
  const int Y = a.n_ky, nkx = a.n_kx;
  const int pos = (nkx + 1) / 2;
  const int hi = N - (nkx - pos);
  const bool nyq_zero = (nkx % 2 == 0) && N > nkx;
  if constexpr (G::TWC) {
    fftx::init_twc<SX>(tw, a.d.tw);
  } else {
    for (int i = threadIdx.x; i < N; i += blockDim.x) tw[i] = a.d.tw[i];
  }
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    int jk = i < pos ? i : (i >= hi ? i - hi + pos : -1);
    if (nyq_zero && jk == nkx / 2) jk = -2;
    otab[i] = jk;
  }
  __syncthreads();
  const fftx::TeamSync sync{team + 1, TP};
  const unsigned step = gridDim.x * TEAMS;
  auto prefetch = [&](unsigned item) {
    if (item >= (unsigned)a.items) return;
    const unsigned sl = item / (unsigned)Y;
    const int k = (int)(item - sl * (unsigned)Y);
    const double2* src = a.m1 + ((int64_t)sl * a.nrow + k) * N;
    for (int e = j; e < N; e += TP) fftx::cp16(stg + e, src + e);
    fftx::cp_commit();
  };
  const double scale = 1.0 / a.norm;
  const int nyq = nkx / 2;
  unsigned item = blockIdx.x * TEAMS + team;
  prefetch(item);
  for (; item < (unsigned)a.items; item += step) {
    const unsigned sl = item / (unsigned)Y;
    const int k = (int)(item - sl * (unsigned)Y);
    double2* out = lay_ptr(a.out, a.lay, ord_out(a.ord, a.s0 + sl), k, nkx);
    fftx::cp_wait_all();
    sync();
    auto load = [&](int i) { return stg[i]; };
    auto store = [&](int i, double2 v) {
      const int jk = otab[i];
      if (jk >= 0)
        out[jk] = make_double2(__dmul_rn(v.x, scale), __dmul_rn(v.y, scale));
      else if (jk == -2)
        out[nyq] = make_double2(0.0, 0.0);
    };
    auto hook = [&]() { prefetch(item + step); };
    fftx::transform_team<SX, G::PADW, G::TWC>(data, j, tw, load, store, hook, sync);
  }
}

// Warp variants of XINV / XFWD for n_x = N1 * N2 (720 = 24 * 30): one warp per
// transform (fftx::warp4), each warp its own persistent item sequence and
// cp.async-staged input row; no CTA or team barriers in the item loop.
template <int N1, int N2, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) xinv_w4(const XInvArgs a) {
  constexpr int N = N1 * N2, ZS = N1 * (N2 + 1);
  extern __shared__ __align__(16) double2 sm[];
  double2* tw4 = sm;
  double* kxd = reinterpret_cast<double*>(tw4 + N);  // slot -> derivative wavenumber
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkx = a.n_kx, Y = a.n_ky, nrow = a.nrow;
  double2* z = tw4 + N + (N + 1) / 2 + warp * (ZS + N);
  double2* stg = z + ZS;  // the staged f row in padded-slot order
  const int pos = (nkx + 1) / 2;
  const int hi = N - (nkx - pos);
  const bool nyq_zero = (nkx % 2 == 0) && N > nkx;
  init_tw4<N1, N2>(tw4, a.d.tw);
  for (int i = threadIdx.x; i < N; i += blockDim.x) kxd[i] = (double)(i < pos ? i : i - N);
  // slots that never carry a mode (the padding gap, the zeroed radial Nyquist) are
  // zeroed once; the staging writes the modes straight into their slots, so the
  // transform's input is one shared load (no slot -> mode table in the chain)
  for (int i = lane; i < N; i += 32)
    if (i >= pos && (i < hi || (nyq_zero && i == hi))) stg[i] = make_double2(0.0, 0.0);
  __syncthreads();
  const unsigned step = gridDim.x * WARPS;
  auto prefetch = [&](unsigned item, const RowCursor& rc) {
    if (item >= (unsigned)a.items) return;
    const int t = (int)rc.t;
    const int ky = t < Y ? t : t - Y + 1;
    const double2* src = lay_ptr(a.f, a.lay, ord_src(a.ord, a.s0 + rc.sl), ky, nkx);
    for (int e = lane; e < nkx; e += 32) {
      const int slot = e < pos ? e : e - pos + hi;
      if (!(nyq_zero && e == nkx / 2)) fftx::cp16(stg + slot, src + e);
    }
    fftx::cp_commit();
  };
  unsigned item = blockIdx.x * WARPS + warp;
  RowCursor cur(item, step, (unsigned)nrow);
  prefetch(item, cur);
  for (; item < (unsigned)a.items; item += step, cur.advance()) {
    const unsigned sl = cur.sl;
    const int t = (int)cur.t;
    const bool minus = t >= Y;
    const int ky = minus ? t - Y + 1 : t;
    const double re = minus ? (double)ky : -(double)ky;
    double2* dst = a.m1 + ((int64_t)sl * nrow + t) * N;
    fftx::cp_wait_all();
    __syncwarp();
    // (i kx' -/+ ky) f at padded slot i, conjugated for the inverse; empty slots are 0
    auto load = [&](int i) { return cconj(cmul(make_double2(re, kxd[i]), stg[i])); };
    auto store = [&](int i, double2 v) { dst[i] = cconj(v); };
    auto hook = [&]() {
      RowCursor nx = cur;
      nx.advance();
      prefetch(item + step, nx);
    };
    // padded slots [N/3, 2N/3) never carry a mode (n_kx <= 2N/3 by the dealias
    // bound; checked at launch): phase-1 inputs n1 in [8, 16) of the 24 x 30 split
    fftx::warp4<N1, N2, (N1 == 24 && N2 == 30) ? 0xFF00u : 0u>(z, tw4, lane, load, store, hook);
  }
}

template <int N1, int N2, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) xfwd_w4(const XFwdArgs a) {
  constexpr int N = N1 * N2, ZS = N1 * (N2 + 1);
  extern __shared__ __align__(16) double2 sm[];
  double2* tw4 = sm;
  int* otab = reinterpret_cast<int*>(tw4 + N);  // slot -> output kx column, -1 dropped or zeroed Nyquist
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* z = tw4 + N + (N + 3) / 4 + warp * (ZS + N);
  double2* stg = z + ZS;
  const int Y = a.n_ky, nkx = a.n_kx;
  const int pos = (nkx + 1) / 2;
  const int hi = N - (nkx - pos);
  const bool nyq_zero = (nkx % 2 == 0) && N > nkx;
  init_tw4<N1, N2>(tw4, a.d.tw);
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    int jk = i < pos ? i : (i >= hi ? i - hi + pos : -1);
    if (nyq_zero && jk == nkx / 2) jk = -1;  // written as zero once per row
    otab[i] = jk;
  }
  __syncthreads();
  const unsigned step = gridDim.x * WARPS;
  auto prefetch = [&](unsigned item, const RowCursor& rc) {
    if (item >= (unsigned)a.items) return;
    const double2* src = a.m1 + ((int64_t)rc.sl * a.nrow + rc.t) * N;
    for (int e = lane; e < N; e += 32) fftx::cp16(stg + e, src + e);
    fftx::cp_commit();
  };
  const double scale = 1.0 / a.norm;
  const int nyq = nkx / 2;
  unsigned item = blockIdx.x * WARPS + warp;
  RowCursor cur(item, step, (unsigned)Y);
  prefetch(item, cur);
  for (; item < (unsigned)a.items; item += step, cur.advance()) {
    const unsigned sl = cur.sl;
    const int k = (int)cur.t;
    double2* out = lay_ptr(a.out, a.lay, ord_out(a.ord, a.s0 + sl), k, nkx);
    fftx::cp_wait_all();
    __syncwarp();
    auto load = [&](int i) { return stg[i]; };
    auto store = [&](int i, double2 v) {  // slot -> wrap-order kx column by arithmetic (no table load)
      const int jk = i < pos ? i : (i >= hi ? i - hi + pos : -1);
      if (jk >= 0 && !(nyq_zero && jk == nyq)) out[jk] = make_double2(__dmul_rn(v.x, scale), __dmul_rn(v.y, scale));
    };
    auto hook = [&]() {
      RowCursor nx = cur;
      nx.advance();
      prefetch(item + step, nx);
    };
    // (skipping the never-retained outputs k2 in [10, 20) at compile time measured
    // 2.6% slower: fewer registers, worse schedule)
    fftx::warp4<N1, N2>(z, tw4, lane, load, store, hook);
    if (nyq_zero && lane == 0) out[nyq] = make_double2(0.0, 0.0);
  }
}

// ---------------------------------------------------------------- host side


static int set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) GK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return GK_OK;
}

static int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// persistent grid: as many CTAs as fit at once (capped by the work items)
template <class K>
static int launch_persistent(K kernel, int threads, size_t smem, int64_t items, cudaStream_t st,
                             const void* args_ptr, const char* what) {
  int rc = set_smem((const void*)kernel, smem);
  if (rc) return rc;
  int per_sm = 0;
  GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  if (per_sm < 1) {
    gk::set_error("%s: kernel does not fit on an SM (threads %d smem %zu)", what, threads, smem);
    return GK_ERR_ARG;
  }
  int64_t grid = (int64_t)per_sm * std::max(1, sm_count() - gk::sm_reserve());
  if (grid > items) grid = items;
  void* args[] = {const_cast<void*>(args_ptr)};
  GK_CUDA(cudaLaunchKernel((const void*)kernel, dim3((unsigned)grid), dim3(threads), args, smem, st));
  gk::count_launch();
  return GK_OK;
}

using SX720 = fftx::Seq<10, 8, 9>;
using SX2016 = fftx::Seq<12, 12, 14>;
#ifndef GK_X2016_TEAMS  // 2016-point x kernels: 6-warp teams per CTA, CTAs per SM
#define GK_X2016_TEAMS 1  // (1, 2) vs (2, 1): C5a nonlinear 16.4 -> 16.0 us/slice; (3, 1) does not fit
#define GK_X2016_MINB 2
#endif
using SY144 = fftx::Seq<12, 12>;
using SY480 = fftx::Seq<10, 6, 8>;
using SY864 = fftx::Seq<12, 8, 9>;



static bool fixed_x(int64_t n) { return n == 720 || n == 2016; }
static bool fixed_y(int64_t n) { return n == 144 || n == 480 || n == 864; }

template <class SX, int TEAMS, int MINB>
static int xinv_team(XInvArgs& a, int64_t cs, cudaStream_t st) {
  a.items = cs * a.nrow;
  GK_CHECK_ARG(a.items < (1ll << 31), "xinv: too many items");
  const size_t smem =
      sizeof(double2) * (TeamGeom<SX>::TWS + (SX::N + 1) / 2 + (size_t)TEAMS * (TeamGeom<SX>::DATA + SX::N));
  return launch_persistent(xinv_tm<SX, TEAMS, MINB>, TEAMS * TeamGeom<SX>::TP, smem,
                           (a.items + TEAMS - 1) / TEAMS, st, &a, "xinv_tm");
}
template <class SX, int TEAMS, int MINB>
static int xfwd_team(XFwdArgs& a, int64_t cs, cudaStream_t st) {
  a.items = cs * a.n_ky;
  GK_CHECK_ARG(a.items < (1ll << 31), "xfwd: too many items");
  const size_t smem =
      sizeof(double2) * (TeamGeom<SX>::TWS + (SX::N + 3) / 4 + (size_t)TEAMS * (TeamGeom<SX>::DATA + SX::N));
  return launch_persistent(xfwd_tm<SX, TEAMS, MINB>, TEAMS * TeamGeom<SX>::TP, smem,
                           (a.items + TEAMS - 1) / TEAMS, st, &a, "xfwd_tm");
}

// n_x = 720 x-direction kernels: warp four-step (default) or 3-warp teams
// (GK_X720=team, kept for A/B measurements).
static bool x720_warp() {
  static bool v = [] {
    const char* e = getenv("GK_X720");
    return !(e && std::string(e) == "team");
  }();
  return v;
}
template <int WARPS>
static int xinv_warp(XInvArgs& a, int64_t cs, cudaStream_t st) {
  GK_CHECK_ARG(a.n_kx <= 480, "xinv_w4: n_kx %d above 2 n_x / 3 (the known-zero input band)", a.n_kx);
  a.items = cs * a.nrow;
  GK_CHECK_ARG(a.items < (1ll << 31), "xinv: too many items");
  const size_t smem = sizeof(double2) * (720 + 360 + (size_t)WARPS * (24 * 31 + 720));
  return launch_persistent(xinv_w4<24, 30, WARPS>, WARPS * 32, smem, (a.items + WARPS - 1) / WARPS, st, &a,
                           "xinv_w4");
}
template <int WARPS>
static int xfwd_warp(XFwdArgs& a, int64_t cs, cudaStream_t st) {
  a.items = cs * a.n_ky;
  GK_CHECK_ARG(a.items < (1ll << 31), "xfwd: too many items");
  const size_t smem = sizeof(double2) * (720 + 180 + (size_t)WARPS * (24 * 31 + 720));
  return launch_persistent(xfwd_w4<24, 30, WARPS>, WARPS * 32, smem, (a.items + WARPS - 1) / WARPS, st, &a,
                           "xfwd_w4");
}

// ycol_w12 (GK_Y144=warp) is correct but slower than ycol_fx at sh03b: its
// lane-per-row global accesses touch 12 cache lines per instruction and saturate
// L1 (ncu: l1tex 98.7%, 1.00 ms vs 0.70 ms per 960-slice chunk).  Kept for A/B.
template <int WARPS, int MINB>
static int ycol_warp(YArgs& a, int64_t cs, cudaStream_t st) {
  a.items = cs * (a.n_x / 4);
  GK_CHECK_ARG(a.items < (1ll << 31), "ycol: too many items");
  const size_t smem = sizeof(double2) * (144 + 72 + (size_t)WARPS * 2 * 12 * 13);
  return launch_persistent(ycol_w12<WARPS, MINB>, WARPS * 32, smem, (a.items + WARPS - 1) / WARPS, st, &a,
                           "ycol_w12");
}

template <class SY, int C, int MINB, bool GST>
static int ycol_fixed(YArgs& a, int64_t cs, cudaStream_t st) {
  a.cols = C;
  a.groups = (a.n_x + C - 1) / C;
  a.items = cs * a.groups;
  const size_t smem = sizeof(double2) * (SY::N * (1 + (GST ? 2 : 1) * C) + (size_t)SY::N * C);
  return launch_persistent(ycol_fx<SY, C, MINB, GST>, C * SY::maxbf(), smem, a.items, st, &a, "ycol_fx");
}


// n_y = 144 YCOL: ycol_sq (default) or ycol_fx (GK_Y144=fx, kept for A/B)
static int y144_mode() {
  static int v = [] {
    const char* e = getenv("GK_Y144");
    if (e && std::string(e) == "fx") return 1;
    if (e && std::string(e) == "warp") return 2;
    return 0;
  }();
  return v;
}
template <int C, int MINB, int CPT = 1>
static int ycol_square(YArgs& a, int64_t cs, cudaStream_t st) {
  a.cols = C;
  a.groups = (a.n_x + C - 1) / C;
  a.items = cs * a.groups;
  const size_t smem = sizeof(double2) * (144 + 3 * (size_t)144 * C);
  if (a.n_x % C == 0)
    return launch_persistent(ycol_sq<C, MINB, true, CPT>, C / CPT * 12, smem, a.items, st, &a, "ycol_sq");
  return launch_persistent(ycol_sq<C, MINB, false, CPT>, C / CPT * 12, smem, a.items, st, &a, "ycol_sq");
}

// n_y = 480 YCOL: rectangular four-step (20 x 24; bins 160..319 empty, outputs
// k < 160), 8 columns per CTA, 2 CTAs per SM.  GK_Y480_FX=1 keeps ycol_fx for A/B.
#ifndef GK_Y480_MINB
#define GK_Y480_MINB 2
#endif
#ifndef GK_Y480_C
#define GK_Y480_C 8
#endif
#ifndef GK_Y864_MINB
#define GK_Y864_MINB 2
#endif
#ifndef GK_Y864_C
#define GK_Y864_C 4
#endif
static int ycol_rect480(YArgs& a, int64_t cs, cudaStream_t st) {
  constexpr int P = 20, Q = 24, ZB0 = 8, ZB1 = 16, KV = 8, C = GK_Y480_C;
  a.cols = C;
  a.groups = (a.n_x + C - 1) / C;
  a.items = cs * a.groups;
  const size_t smem = sizeof(double2) * (P * Q + (size_t)P * Q * C + (size_t)(Q - (ZB1 - ZB0)) * P * C);
  return launch_persistent(ycol_rect<P, Q, ZB0, ZB1, KV, C, GK_Y480_MINB>, C * Q, smem, a.items, st, &a,
                           "ycol_rect");
}

// n_y = 864 YCOL (em04b plan): rectangular 32 x 27 (bins 288..575 empty, outputs
// k < 288), 4 columns per CTA, 2 CTAs per SM.  GK_Y864_FX=1 keeps ycol_fx for A/B.
static int ycol_rect864(YArgs& a, int64_t cs, cudaStream_t st) {
  constexpr int P = 32, Q = 27, ZB0 = 9, ZB1 = 18, KV = 9, C = GK_Y864_C;
  a.cols = C;
  a.groups = (a.n_x + C - 1) / C;
  a.items = cs * a.groups;
  const size_t smem = sizeof(double2) * (P * Q + (size_t)P * Q * C + (size_t)(Q - (ZB1 - ZB0)) * P * C);
  return launch_persistent(ycol_rect<P, Q, ZB0, ZB1, KV, C, GK_Y864_MINB>, C * P, smem, a.items, st, &a,
                           "ycol_rect");
}

static int64_t chunk_target_bytes() {
  static int64_t v = [] {
    // ~2.5 GiB of mixed-spectrum scratch per chunk: big enough that every launch
    // keeps all SMs busy for many work items (launch ramp/drain amortised;
    // measured at sh03b: 40 MB chunks +40%, 0.64 GiB +3%, 1.25 GiB +3%, flat from
    // 2.5 GiB), small enough for em04b/C5 states to keep their scratch bounded.
    // Override: GK_CHUNK_MB.
    const char* e = getenv("GK_CHUNK_MB");
    const int64_t mb = e ? atoll(e) : 2560;
    return (mb > 0 ? mb : 2560) << 20;
  }();
  return v;
}

static int64_t chunk_slices(const gk_spectral_plan* p, int nrow, int64_t n_slices) {
  const int64_t per = p->n_x * (int64_t)nrow * 16;
  int64_t c = chunk_target_bytes() / per;
  if (c < 1) c = 1;
  if (c > n_slices) c = n_slices;
  return c < 1 ? 1 : c;
}

static int xinv(const gk_spectral_plan* p, const double2* f, Order ord, double2* m1, int64_t s0, int64_t cs,
                int nrow, int bracket, cudaStream_t st, const Layout* lay = nullptr) {
  XInvArgs a{};
  a.d = p->dx;
  a.f = f;
  a.lay = lay ? *lay : contiguous_layout(f, p->n_ky);
  a.ord = ord;
  a.m1 = m1;
  a.s0 = s0;
  a.nrow = nrow;
  a.n_kx = (int)p->n_kx;
  a.n_ky = (int)p->n_ky;
  a.bracket = bracket;
  if (p->fixed) {  // 4 (720) / 2 (2016) independent teams per CTA, one CTA per SM
    if (p->n_x == 720) return x720_warp() ? xinv_warp<GK_XINV_WARPS>(a, cs, st) : xinv_team<SX720, 4, 1>(a, cs, st);
    return xinv_team<SX2016, GK_X2016_TEAMS, GK_X2016_MINB>(a, cs, st);
  }
  a.tb = (int)std::max<int64_t>(1, std::min<int64_t>(nrow, kSmemElems / p->n_x));
  a.groups = (nrow + a.tb - 1) / a.tb;
  const size_t smem = 2 * sizeof(double2) * a.tb * p->n_x;
  int rc = set_smem((const void*)xinv_kernel, smem);
  if (rc) return rc;
  xinv_kernel<<<(unsigned)(cs * a.groups), kThreads, smem, st>>>(a);
  return check_launch("xinv_kernel");
}

static int ycol(const gk_spectral_plan* p, YArgs a, int64_t cs, cudaStream_t st) {
  a.d = p->dy;
  a.n_x = (int)p->n_x;
  if (p->fixed && (a.mode == Y_PHI || a.mode == Y_BRACKET)) {
    // 16 interleaved columns per CTA, 2 CTAs per SM, phi's field block staged
    if (p->n_y == 144) {
      const int mode = y144_mode();
      if (mode == 2 && p->n_x % 4 == 0 && a.n_ky <= 48) return ycol_warp<GK_YCOL_WARPS, GK_YCOL_MINB>(a, cs, st);
      if (mode == 1 || a.n_ky > 48) return ycol_fixed<SY144, 16, GK_YCOL_FX_MINB, GK_YCOL_FX_GST>(a, cs, st);
      if (getenv("GK_YSQ8")) return ycol_square<8, 4>(a, cs, st);
      // columns per CTA (A/B; 16 measured best): 5 -> six 2-warp CTAs
      // per SM, 10 -> three 4-warp CTAs, 32 -> one 12-warp CTA
      static const int ysq_c = [] {
        const char* e = getenv("GK_YSQ_C");
        return e ? atoi(e) : 16;
      }();
      if (ysq_c == 5) return ycol_square<5, 6>(a, cs, st);
      if (ysq_c == 10) return ycol_square<10, 3>(a, cs, st);
      if (ysq_c == 32) return ycol_square<32, 1>(a, cs, st);
      static const int ysq_cpt = [] {
        const char* e = getenv("GK_YSQ_CPT");
        return e ? atoi(e) : 1;
      }();
      if (ysq_cpt == 2) return ycol_square<16, 2, 2>(a, cs, st);
      return ycol_square<16, GK_YCOL_FX_MINB>(a, cs, st);
    }
    if (p->n_y == 480 && a.n_ky <= 160 && !getenv("GK_Y480_FX")) return ycol_rect480(a, cs, st);
    if (p->n_y == 480) return ycol_fixed<SY480, 4, 1, true>(a, cs, st);
    if (a.n_ky <= 288 && !getenv("GK_Y864_FX")) return ycol_rect864(a, cs, st);
    return ycol_fixed<SY864, 4, 1, true>(a, cs, st);
  }
  int64_t c = kSmemElems / p->n_y;
  c = std::max<int64_t>(2, c & ~int64_t(1));
  c = std::min<int64_t>(c, (p->n_x + 1) & ~int64_t(1));
  a.cols = (int)c;
  a.groups = (int)((p->n_x + c - 1) / c);
  const size_t smem = 2 * sizeof(double2) * a.cols * p->n_y;
  int rc = set_smem((const void*)ycol_kernel, smem);
  if (rc) return rc;
  ycol_kernel<<<(unsigned)(cs * a.groups), kThreads, smem, st>>>(a);
  return check_launch("ycol_kernel");
}

static int xfwd(const gk_spectral_plan* p, const double2* m1, double2* out, Order ord, int64_t s0, int64_t cs,
                int nrow, bool allow_fixed, cudaStream_t st, const Layout* lay = nullptr) {
  XFwdArgs a{};
  a.d = p->dx;
  a.m1 = m1;
  a.out = out;
  a.lay = lay ? *lay : contiguous_layout(out, p->n_ky);
  a.ord = ord;
  a.s0 = s0;
  a.nrow = nrow;
  a.n_ky = (int)p->n_ky;
  a.n_kx = (int)p->n_kx;
  a.norm = (double)(p->n_x * p->n_y);
  if (p->fixed && allow_fixed) {
    if (p->n_x == 720) return x720_warp() ? xfwd_warp<GK_XFWD_WARPS>(a, cs, st) : xfwd_team<SX720, 4, 1>(a, cs, st);
    return xfwd_team<SX2016, GK_X2016_TEAMS, GK_X2016_MINB>(a, cs, st);
  }
  a.tb = (int)std::max<int64_t>(1, std::min<int64_t>(p->n_ky, kSmemElems / p->n_x));
  a.groups = (int)((p->n_ky + a.tb - 1) / a.tb);
  const size_t smem = 2 * sizeof(double2) * a.tb * p->n_x;
  int rc = set_smem((const void*)xfwd_kernel, smem);
  if (rc) return rc;
  xfwd_kernel<<<(unsigned)(cs * a.groups), kThreads, smem, st>>>(a);
  return check_launch("xfwd_kernel");
}

// out[row of slice s0 + sl] += tmp[sl] for the cs slices of one chunk (accumulate
// mode): tmp holds the chunk's rows in chunk order ([sl][k][kx], written by the
// forward x transform with the natural order), out is addressed through ord.
// One coalesced read-add-write pass; adding inside the transform's store path
// instead serialised a global load per stored element (xfwd 3.2 -> 10.5 ms).
__global__ void __launch_bounds__(kThreads) acc_rows(const double2* __restrict__ tmp, double2* __restrict__ out,
                                                     Order ord, int64_t s0, int64_t cs, int64_t row) {
  const int64_t n = cs * row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sl = i / row, e = i - sl * row;
    double2* o = out + ord_out(ord, s0 + sl) * row + e;
    *o = cadd(*o, __ldcs(tmp + i));
  }
}

static int64_t bracket_ws(const gk_spectral_plan* p, int64_t n_slices, int64_t n_g, bool acc = false) {
  const int nrow = (int)(2 * p->n_ky - 1);
  const int64_t cs = chunk_slices(p, nrow, std::max(n_slices, n_g));
  // accumulate mode: + one chunk of output rows
  return (n_g * p->n_x * p->n_y + cs * p->n_x * nrow + (acc ? cs * p->n_ky * p->n_kx : 0)) * 16;
}

// Slices q in [q0, q0 + n_q) of the batch (in `ord`), g fields computed for g
// slices [g0, g0 + n_gc) into the workspace's G (indexed absolutely, n_g total).
static int bracket_range(const gk_spectral_plan* p, const double2* f, const double2* g, double2* out, int64_t q0,
                         int64_t n_q, Order ord, int64_t n_g, int64_t g0, int64_t n_gc, void* ws, int64_t ws_bytes,
                         cudaStream_t st, bool acc = false, const Layout* lay_f = nullptr,
                         const Layout* lay_g = nullptr, const Layout* lay_o = nullptr) {
  GK_CHECK_ARG(p && ws && (n_q == 0 || (f && out)) && (n_gc == 0 || g), "gk_bracket: null pointer");
  GK_CHECK_ARG(q0 >= 0 && n_q >= 0 && n_g >= 1 && g0 >= 0 && n_gc >= 0 && g0 + n_gc <= n_g,
               "gk_bracket: bad batch sizes");
  GK_CHECK_ARG(ord.tm_T || ord.gmap || (ord.gmod >= 1 && ord.gmod <= n_g),
               "gk_bracket: need g_map or 1 <= g_mod <= n_g");
  GK_CHECK_ARG(p->n_x >= (3 * p->n_kx + 1) / 2 && p->n_y >= 3 * p->n_ky - 2,
               "gk_bracket: plan below the dealias bounds");
  GK_CHECK_ARG(ws_bytes >= bracket_ws(p, n_q, n_g, acc), "gk_bracket: workspace too small (%lld < %lld)",
               (long long)ws_bytes, (long long)bracket_ws(p, n_q, n_g, acc));
  GK_CHECK_ARG(q0 + n_q < (1ll << 31) && n_g < (1ll << 31), "gk_bracket: batch above 2^31 slices");
  const int nrow = (int)(2 * p->n_ky - 1);
  const int64_t chunk = chunk_slices(p, nrow, std::max(n_q, n_g));
  double2* G = (double2*)ws;
  double2* m1 = G + n_g * p->n_x * p->n_y;
  double2* tmp = m1 + chunk * p->n_x * nrow;  // accumulate mode: the chunk's output rows
  int rc;
  const Order natural{nullptr, nullptr, 1, 0, 0};
  for (int64_t s0 = g0; s0 < g0 + n_gc; s0 += chunk) {
    const int64_t cs = std::min(chunk, g0 + n_gc - s0);
    if ((rc = xinv(p, g, natural, m1, s0, cs, nrow, 1, st, lay_g))) return rc;
    YArgs a{};
    a.m1 = m1;
    a.G = G;
    a.ord = natural;
    a.s0 = s0;
    a.nrow = nrow;
    a.n_ky = (int)p->n_ky;
    a.mode = Y_PHI;
    if ((rc = ycol(p, a, cs, st))) return rc;
  }
  for (int64_t s0 = q0; s0 < q0 + n_q; s0 += chunk) {
    const int64_t cs = std::min(chunk, q0 + n_q - s0);
    if ((rc = xinv(p, f, ord, m1, s0, cs, nrow, 1, st, lay_f))) return rc;
    YArgs a{};
    a.m1 = m1;
    a.G = G;
    a.ord = ord;
    a.s0 = s0;
    a.nrow = nrow;
    a.n_ky = (int)p->n_ky;
    a.mode = Y_BRACKET;
    if ((rc = ycol(p, a, cs, st))) return rc;
    if (!acc) {
      if ((rc = xfwd(p, m1, out, ord, s0, cs, nrow, true, st, lay_o))) return rc;
      continue;
    }
    const Order natural_out{nullptr, nullptr, 1, 0, 0};
    if ((rc = xfwd(p, m1, tmp - s0 * p->n_ky * p->n_kx, natural_out, s0, cs, nrow, true, st))) return rc;
    const int64_t row = p->n_ky * p->n_kx;
    acc_rows<<<(unsigned)std::min<int64_t>(cdiv(cs * row, (int64_t)kThreads), (int64_t)sm_count() * 8), kThreads, 0,
               st>>>(tmp, out, ord, s0, cs, row);
    if ((rc = check_launch("acc_rows"))) return rc;
  }
  return GK_OK;
}

static int bracket_impl(const gk_spectral_plan* p, const double2* f, const double2* g, double2* out,
                        int64_t n_slices, Order ord, int64_t n_g, void* ws, int64_t ws_bytes, cudaStream_t st) {
  return bracket_range(p, f, g, out, 0, n_slices, ord, n_g, 0, n_g, ws, ws_bytes, st);
}

static void factor_radices(int64_t n, std::vector<int>& rad) {
  rad.clear();
  int64_t m = n;
  int e = 0;
  while (m % 2 == 0) {
    m /= 2;
    ++e;
  }
  const int k = (e + 3) / 4;
  for (int i = 0; i < k; ++i) rad.push_back(1 << (e / k + (i < e % k ? 1 : 0)));
  while (m % 9 == 0) { rad.push_back(9); m /= 9; }
  while (m % 3 == 0) { rad.push_back(3); m /= 3; }
  while (m % 5 == 0) { rad.push_back(5); m /= 5; }
  while (m % 7 == 0) { rad.push_back(7); m /= 7; }
  for (int64_t p = 11; m > 1; p += 2)
    while (m % p == 0) { rad.push_back((int)p); m /= p; }
}

static void host_twiddles(int64_t n, double2* t) {
  for (int64_t m = 0; m < n; ++m) {
    const long double a = 2.0L * 3.141592653589793238462643383279502884L * (long double)m / (long double)n;
    t[m].x = (double)cosl(a);
    t[m].y = (double)-sinl(a);
  }
}

}  // namespace spec

// The two halves of the blocked nonlinear term, for the multi-GPU rank step
// (dist.cu): phi's derivative fields once per step, then each velocity chunk as
// it arrives.  The workspace is gk_bracket_workspace_bytes(plan, n_slices, n_theta)
// with n_slices the chunk's slice count; the fields stay in it between calls.
int nonlinear_fields_blocked(const gk_spectral_plan* p, const double* phi, int64_t n_theta, int64_t n_blocks,
                             void* ws, int64_t ws_bytes, int64_t n_slices, cudaStream_t st) {
  using namespace spec;
  const int yl = (int)(p->n_ky / n_blocks);
  const Order natural{nullptr, nullptr, 1, 0, 0};
  GK_CHECK_ARG(n_blocks >= 1 && n_blocks <= kMaxLayoutBlocks, "nonlinear_fields_blocked: %lld blocks (max %d)",
               (long long)n_blocks, kMaxLayoutBlocks);
  GK_CHECK_ARG(ws_bytes >= bracket_ws(p, n_slices, n_theta), "nonlinear_fields_blocked: workspace too small");
  Layout lg{};
  lg.yl = yl;
  for (int b = 0; b < n_blocks; ++b) lg.base[b] = (const double2*)phi + (int64_t)b * n_theta * yl * p->n_kx;
  return bracket_range(p, nullptr, (const double2*)phi, nullptr, 0, 0, natural, n_theta, 0, n_theta, ws, ws_bytes,
                       st, false, nullptr, &lg, nullptr);
}
// in_base[b] / out_base[b]: where toroidal block b of the chunk's input / output
// rows ([n_vel][n_theta][n_ky / n_blocks][n_kx] each) lives -- a transpose's
// receive / send buffer, the rank's home shard, or (P2P) a peer GPU's memory
int nonlinear_slices_blocked(const gk_spectral_plan* p, const double* const* in_base, double* const* out_base,
                             int64_t n_vel, int64_t n_theta, int64_t n_blocks, void* ws, int64_t ws_bytes,
                             cudaStream_t st) {
  using namespace spec;
  GK_CHECK_ARG(n_blocks >= 1 && n_blocks <= kMaxLayoutBlocks, "nonlinear_slices_blocked: %lld blocks (max %d)",
               (long long)n_blocks, kMaxLayoutBlocks);
  const int yl = (int)(p->n_ky / n_blocks);
  const Order ord{nullptr, nullptr, n_theta, n_vel, n_theta};  // theta-major walk
  Layout in{}, outl{};
  in.yl = outl.yl = yl;
  for (int b = 0; b < n_blocks; ++b) {
    in.base[b] = (const double2*)in_base[b];
    outl.base[b] = (const double2*)out_base[b];
  }
  return bracket_range(p, (const double2*)in_base[0], nullptr, (double2*)out_base[0], 0, n_vel * n_theta, ord,
                       n_theta, 0, 0, ws, ws_bytes, st, false, &in, &in, &outl);
}
int64_t nonlinear_ws_bytes(const gk_spectral_plan* p, int64_t n_slices, int64_t n_theta) {
  return spec::bracket_ws(p, n_slices, n_theta);
}
void plan_grid(const gk_spectral_plan* p, int64_t* n_x, int64_t* n_y) {
  *n_x = p ? p->n_x : 0;
  *n_y = p ? p->n_y : 0;
}
// the same from the plan's sizes alone (no device tables needed)
int64_t nonlinear_ws_bytes_sizes(int64_t n_kx, int64_t n_ky, int64_t n_x, int64_t n_y, int64_t n_slices,
                                 int64_t n_theta) {
  gk_spectral_plan p{};
  p.n_kx = n_kx;
  p.n_ky = n_ky;
  p.n_x = n_x;
  p.n_y = n_y;
  return spec::bracket_ws(&p, n_slices, n_theta);
}
}  // namespace gk

using namespace gk;
using namespace gk::spec;

extern "C" {

int gk_spectral_plan_create(int64_t n_kx, int64_t n_ky, int64_t n_x, int64_t n_y, gk_spectral_plan** plan) {
  GK_CHECK_ARG(plan, "gk_spectral_plan_create: null out pointer");
  *plan = nullptr;
  GK_CHECK_ARG(n_kx >= 1 && n_ky >= 1 && n_x >= n_kx && n_y / 2 + 1 >= n_ky,
               "gk_spectral_plan_create: grid (%lld,%lld) cannot hold (%lld,%lld) modes", (long long)n_x,
               (long long)n_y, (long long)n_kx, (long long)n_ky);
  // generic engine: one CTA holds >= 1 x-transform and >= 2 y-columns, ping-pong
  GK_CHECK_ARG(2 * 16 * n_x <= 227 * 1024 && 2 * 2 * 16 * n_y <= 227 * 1024,
               "gk_spectral_plan_create: transform length above the shared-memory limit "
               "(n_x <= 7264, n_y <= 3632)");
  auto* p = new gk_spectral_plan{};
  p->n_kx = n_kx;
  p->n_ky = n_ky;
  p->n_x = n_x;
  p->n_y = n_y;
  const char* env = getenv("GK_GENERIC_FFT");
  p->fixed = fixed_x(n_x) && fixed_y(n_y) && !(env && env[0] == '1');
  std::vector<double2> tw(n_x + n_y);
  host_twiddles(n_x, tw.data());
  host_twiddles(n_y, tw.data() + n_x);
  if (cudaMalloc(&p->tw_dev, sizeof(double2) * (n_x + n_y)) != cudaSuccess) {
    delete p;
    gk::set_error("gk_spectral_plan_create: cudaMalloc failed");
    return GK_ERR_NOMEM;
  }
  cudaMemcpy(p->tw_dev, tw.data(), sizeof(double2) * (n_x + n_y), cudaMemcpyHostToDevice);
  std::vector<int> rad;
  fft::Desc* ds[2] = {&p->dx, &p->dy};
  const int64_t ns[2] = {n_x, n_y};
  for (int d = 0; d < 2; ++d) {
    factor_radices(ns[d], rad);
    if ((int)rad.size() > fft::kMaxPass) {
      cudaFree(p->tw_dev);
      delete p;
      gk::set_error("gk_spectral_plan_create: too many passes");
      return GK_ERR_ARG;
    }
    ds[d]->n = (int)ns[d];
    ds[d]->npass = (int)rad.size();
    for (size_t i = 0; i < rad.size(); ++i) ds[d]->radix[i] = rad[i];
    ds[d]->tw = p->tw_dev + (d == 0 ? 0 : n_x);
  }
  *plan = p;
  return GK_OK;
}

int gk_spectral_plan_destroy(gk_spectral_plan* plan) {
  if (!plan) return GK_OK;
  cudaFree(plan->tw_dev);
  delete plan;
  return GK_OK;
}

int64_t gk_bracket_workspace_bytes(const gk_spectral_plan* plan, int64_t n_slices, int64_t n_g) {
  if (!plan) return -1;
  return bracket_ws(plan, n_slices, n_g);
}

int64_t gk_nonlinear_acc_workspace_bytes(const gk_spectral_plan* plan, int64_t n_vel, int64_t n_theta) {
  if (!plan) return -1;
  return bracket_ws(plan, n_vel * n_theta, n_theta, true);
}

int gk_bracket(const gk_spectral_plan* plan, const double* f, const double* g, double* out, int64_t n_slices,
               const int64_t* f_map, const int64_t* g_map, int64_t n_g, int64_t g_mod, void* workspace,
               int64_t workspace_bytes, void* stream) {
  const Order ord{f_map, g_map, g_mod, 0, 0};
  return bracket_impl(plan, (const double2*)f, (const double2*)g, (double2*)out, n_slices, ord, n_g, workspace,
                      workspace_bytes, (cudaStream_t)stream);
}

int gk_nonlinear(const gk_spectral_plan* plan, const double* h, const double* phi, double* out, int64_t n_vel,
                 int64_t n_theta, void* workspace, int64_t workspace_bytes, void* stream) {
  const Order ord{nullptr, nullptr, n_theta, n_vel, n_theta};  // theta-major walk
  return bracket_impl(plan, (const double2*)h, (const double2*)phi, (double2*)out, n_vel * n_theta, ord, n_theta,
                      workspace, workspace_bytes, (cudaStream_t)stream);
}

// out += nonlinear(h, phi): the same bracket, each output added to what out holds
// (one rounding per element; the in-place step accumulates it onto the collision)
int gk_nonlinear_acc(const gk_spectral_plan* plan, const double* h, const double* phi, double* out, int64_t n_vel,
                     int64_t n_theta, void* workspace, int64_t workspace_bytes, void* stream) {
  const Order ord{nullptr, nullptr, n_theta, n_vel, n_theta};  // theta-major walk
  return bracket_range(plan, (const double2*)h, (const double2*)phi, (double2*)out, 0, n_vel * n_theta, ord, n_theta,
                       0, n_theta, workspace, workspace_bytes, (cudaStream_t)stream, true);
}

int gk_nonlinear_range(const gk_spectral_plan* plan, const double* h, const double* phi, double* out,
                       int64_t n_vel, int64_t n_theta, int64_t t0, int64_t t1, void* workspace,
                       int64_t workspace_bytes, void* stream) {
  GK_CHECK_ARG(0 <= t0 && t0 <= t1 && t1 <= n_theta, "gk_nonlinear_range: bad theta range");
  const Order ord{nullptr, nullptr, n_theta, n_vel, n_theta};  // theta-major walk: slice q = t*M + v
  return bracket_range(plan, (const double2*)h, (const double2*)phi, (double2*)out, t0 * n_vel,
                       (t1 - t0) * n_vel, ord, n_theta, t0, t1 - t0, workspace, workspace_bytes,
                       (cudaStream_t)stream);
}

// nonlinear_kernel on a velocity chunk held in a multi-GPU transpose's blocked
// layout (SURVEY.md §8 e): h/out [n_blocks][n_vel][n_theta][n_ky / n_blocks][n_kx]
// (block b = toroidal modes [b yl, (b + 1) yl) from / to rank b), phi
// [n_blocks][n_theta][yl][n_kx] (the all-gather of the ranks' field blocks).  The
// x transforms read and write these layouts directly, so the transposes need no
// separate pack / unpack pass.  Same kernels and bits as gk_nonlinear on the
// contiguous arrays.
int gk_nonlinear_blocked(const gk_spectral_plan* plan, const double* h, const double* phi, double* out,
                         int64_t n_vel, int64_t n_theta, int64_t n_blocks, void* workspace, int64_t workspace_bytes,
                         void* stream) {
  GK_CHECK_ARG(plan && n_blocks >= 1 && plan->n_ky % n_blocks == 0,
               "gk_nonlinear_blocked: n_ky must divide into n_blocks blocks");
  int rc = gk::nonlinear_fields_blocked(plan, phi, n_theta, n_blocks, workspace, workspace_bytes, n_vel * n_theta,
                                        (cudaStream_t)stream);
  if (rc) return rc;
  GK_CHECK_ARG(n_blocks <= gk::spec::kMaxLayoutBlocks, "gk_nonlinear_blocked: at most %d blocks",
               gk::spec::kMaxLayoutBlocks);
  const double* in_base[gk::spec::kMaxLayoutBlocks];
  double* out_base[gk::spec::kMaxLayoutBlocks];
  const int64_t blk = n_vel * n_theta * (plan->n_ky / n_blocks) * plan->n_kx * 2;  // doubles per block
  for (int64_t b = 0; b < n_blocks; ++b) {
    in_base[b] = h + b * blk;
    out_base[b] = out + b * blk;
  }
  return gk::nonlinear_slices_blocked(plan, in_base, out_base, n_vel, n_theta, n_blocks, workspace, workspace_bytes,
                                      (cudaStream_t)stream);
}

int64_t gk_transform_workspace_bytes(const gk_spectral_plan* plan, int64_t batch) {
  if (!plan) return -1;
  return chunk_slices(plan, (int)plan->n_ky, batch) * plan->n_x * plan->n_ky * 16;
}

// Standalone transforms always use the generic kernels (column-major m1).
int gk_to_real(const gk_spectral_plan* p, const double* spec, double* field, int64_t batch, void* ws,
               int64_t ws_bytes, void* stream) {
  GK_CHECK_ARG(p && spec && field && ws, "gk_to_real: null pointer");
  GK_CHECK_ARG(ws_bytes >= gk_transform_workspace_bytes(p, batch), "gk_to_real: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int nrow = (int)p->n_ky;
  const int64_t chunk = chunk_slices(p, nrow, batch);
  const Order natural{nullptr, nullptr, 1, 0, 0};
  gk_spectral_plan gp = *p;
  gp.fixed = false;
  int rc;
  for (int64_t s0 = 0; s0 < batch; s0 += chunk) {
    const int64_t cs = std::min(chunk, batch - s0);
    if ((rc = xinv(&gp, (const double2*)spec, natural, (double2*)ws, s0, cs, nrow, 0, st))) return rc;
    YArgs a{};
    a.m1 = (double2*)ws;
    a.field_out = field;
    a.ord = natural;
    a.s0 = s0;
    a.nrow = nrow;
    a.n_ky = nrow;
    a.mode = Y_TO_REAL;
    if ((rc = ycol(&gp, a, cs, st))) return rc;
  }
  return GK_OK;
}

int gk_to_spectrum(const gk_spectral_plan* p, const double* field, double* spec, int64_t batch, void* ws,
                   int64_t ws_bytes, void* stream) {
  GK_CHECK_ARG(p && spec && field && ws, "gk_to_spectrum: null pointer");
  GK_CHECK_ARG(ws_bytes >= gk_transform_workspace_bytes(p, batch), "gk_to_spectrum: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int nrow = (int)p->n_ky;
  const int64_t chunk = chunk_slices(p, nrow, batch);
  const Order natural{nullptr, nullptr, 1, 0, 0};
  gk_spectral_plan gp = *p;
  gp.fixed = false;
  int rc;
  for (int64_t s0 = 0; s0 < batch; s0 += chunk) {
    const int64_t cs = std::min(chunk, batch - s0);
    YArgs a{};
    a.m1 = (double2*)ws;
    a.field_in = field;
    a.ord = natural;
    a.s0 = s0;
    a.nrow = nrow;
    a.n_ky = nrow;
    a.mode = Y_TO_SPEC;
    if ((rc = ycol(&gp, a, cs, st))) return rc;
    if ((rc = xfwd(&gp, (const double2*)ws, (double2*)spec, natural, s0, cs, nrow, false, st))) return rc;
  }
  return GK_OK;
}

}  // extern "C"
