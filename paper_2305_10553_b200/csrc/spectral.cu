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
// mixed (x, ky) representation, (2 n_ky - 1) x n_x complex per slice, kept in an
// L2-sized chunk buffer that is reused chunk after chunk.  phi's derivative fields
// (g) are produced by the very same XINV/YCOL code (bit-identical to f's) and
// stored once per theta, column-major [theta][x][y] so YCOL reads them contiguously.
//
// Taking Re of the ky=0 row reproduces irfft's projection of the (generally
// non-Hermitian) random state (spectral.py:136-137).
#include <cmath>
#include <cstdlib>
#include <vector>

#include "fft_engine.cuh"
#include "../../include/gk.h"

struct gk_spectral_plan {
  int64_t n_kx, n_ky, n_x, n_y;
  gk::fft::Desc dx, dy;
  double2* tw_dev;
};

namespace gk {
namespace spec {

constexpr int kThreads = 128;
constexpr int64_t kSmemElems = 2944;  // double2 elements per ping-pong half (~92 KB total)

enum YMode { Y_PHI = 0, Y_BRACKET = 1, Y_TO_REAL = 2, Y_TO_SPEC = 3 };

struct XInvArgs {
  fft::Desc d;
  const double2* f;
  const int64_t* fmap;
  double2* m1;
  int64_t s0;
  int nrow;  // rows of m1 per column (2Y-1 bracket, n_ky plain)
  int n_kx, n_ky;
  int bracket;
  int tb, groups;
};

struct YArgs {
  fft::Desc d;
  double2* m1;
  double2* G;
  const int64_t* gmap;
  int64_t gmod;
  double* field_out;
  const double* field_in;
  int64_t s0;
  int nrow, n_ky, n_x;
  int mode;
  int cols, groups;
};

struct XFwdArgs {
  fft::Desc d;
  const double2* m1;
  double2* out;
  int64_t s0;
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

__global__ void __launch_bounds__(kThreads) xinv_kernel(const XInvArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  const int n = a.d.n, ld = n;
  const int sl = blockIdx.x / a.groups;
  const int t0 = (blockIdx.x - sl * a.groups) * a.tb;
  const int ntr = min(a.tb, a.nrow - t0);
  const int64_t s = a.s0 + sl;
  const int64_t fs = a.fmap ? a.fmap[s] : s;
  const double2* src = a.f + fs * a.n_ky * a.n_kx;
  double2* buf0 = sm;
  double2* buf1 = sm + a.tb * ld;
  const bool nyq_zero = (a.n_kx % 2 == 0) && n > a.n_kx;
  const int Y = a.n_ky;
  for (int e = threadIdx.x; e < ntr * n; e += kThreads) {
    const int tt = e / n, i = e - tt * n, t = t0 + tt;
    int j = slot_to_kx(i, n, a.n_kx);
    if (nyq_zero && j == a.n_kx / 2) j = -1;
    double2 v = make_double2(0.0, 0.0);
    if (j >= 0) {
      int ky = t;
      double re = 0.0;
      if (a.bracket) {
        ky = t < Y ? t : t - Y + 1;
        re = t < Y ? -(double)ky : (double)ky;
      }
      v = src[(int64_t)ky * a.n_kx + j];
      if (a.bracket) {
        double kxd = j < (a.n_kx + 1) / 2 ? (double)j : (double)(j - a.n_kx);
        if (a.n_kx % 2 == 0 && j == a.n_kx / 2) kxd = 0.0;
        v = cmul(make_double2(re, kxd), v);
      }
    }
    buf0[tt * ld + i] = cconj(v);
  }
  __syncthreads();
  const double2* res = fft::run(a.d, buf0, buf1, ld, ntr, threadIdx.x, kThreads);
  double2* dst = a.m1 + (int64_t)sl * n * a.nrow + t0;
  for (int e = threadIdx.x; e < ntr * n; e += kThreads) {
    const int x = e / ntr, tt = e - x * ntr;
    dst[(int64_t)x * a.nrow + tt] = cconj(res[tt * ld + x]);
  }
}

// column k of the y-spectrum built from the XINV rows (bracket layout)
__device__ __forceinline__ double2 zb_bracket(const double2* col, int k, int n, int Y) {
  if (k == 0) return make_double2(col[0].x, 0.0);
  if (k < Y) return col[k];
  if (k > n - Y) return cconj(col[Y - 1 + (n - k)]);
  return make_double2(0.0, 0.0);
}
// Hermitian extension of a half column (irfft semantics: Re of DC and Nyquist bins)
__device__ __forceinline__ double2 zb_herm(const double2* col, int k, int n, int Y) {
  if (k == 0) return Y > 0 ? make_double2(col[0].x, 0.0) : make_double2(0.0, 0.0);
  if (2 * k < n) return k < Y ? col[k] : make_double2(0.0, 0.0);
  if (2 * k == n) return k < Y ? make_double2(col[k].x, 0.0) : make_double2(0.0, 0.0);
  const int m = n - k;
  return m < Y ? cconj(col[m]) : make_double2(0.0, 0.0);
}

__device__ __forceinline__ void separate_store(const double2* res, int ld, int n, int npair, int nc,
                                               int Y, double2* colbase, int nrow) {
  for (int e = threadIdx.x; e < npair * Y; e += kThreads) {
    const int q = e / Y, k = e - q * Y;
    const double2 za = res[q * ld + k];
    const double2 zb = res[q * ld + (k == 0 ? 0 : n - k)];
    const double2 pa = make_double2(__dmul_rn(0.5, __dadd_rn(za.x, zb.x)), __dmul_rn(0.5, __dsub_rn(za.y, zb.y)));
    colbase[(int64_t)(2 * q) * nrow + k] = pa;
    if (2 * q + 1 < nc) {
      const double2 pb = make_double2(__dmul_rn(0.5, __dadd_rn(za.y, zb.y)), __dmul_rn(0.5, __dsub_rn(zb.x, za.x)));
      colbase[(int64_t)(2 * q + 1) * nrow + k] = pb;
    }
  }
}

__global__ void __launch_bounds__(kThreads) ycol_kernel(const YArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  const int n = a.d.n, ld = n;
  const int sl = blockIdx.x / a.groups;
  const int x0 = (blockIdx.x - sl * a.groups) * a.cols;
  const int nc = min(a.cols, a.n_x - x0);
  const int npair = (nc + 1) / 2;
  const int64_t s = a.s0 + sl;
  double2* buf0 = sm;
  double2* buf1 = sm + a.cols * ld;
  double2* colbase = a.m1 + ((int64_t)sl * a.n_x + x0) * a.nrow;
  const int Y = a.n_ky;

  if (a.mode == Y_PHI || a.mode == Y_BRACKET) {
    for (int e = threadIdx.x; e < nc * n; e += kThreads) {
      const int c = e / n, k = e - c * n;
      buf0[c * ld + k] = cconj(zb_bracket(colbase + (int64_t)c * a.nrow, k, n, Y));
    }
    __syncthreads();
    double2* res = fft::run(a.d, buf0, buf1, ld, nc, threadIdx.x, kThreads);
    if (a.mode == Y_PHI) {
      double2* g = a.G + (s * a.n_x + x0) * n;
      for (int e = threadIdx.x; e < nc * n; e += kThreads) {
        const int c = e / n, y = e - c * n;
        g[(int64_t)c * n + y] = cconj(res[c * ld + y]);
      }
      return;
    }
    const int64_t gi = a.gmap ? a.gmap[s] : s % a.gmod;
    const double2* g = a.G + (gi * a.n_x + x0) * n;
    double2* other = res == buf0 ? buf1 : buf0;
    for (int e = threadIdx.x; e < npair * n; e += kThreads) {
      const int q = e / n, y = e - q * n;
      const int ca = 2 * q, cb = 2 * q + 1;
      const double2 wa = cconj(res[ca * ld + y]);
      const double2 ga = g[(int64_t)ca * n + y];
      const double pa = __dsub_rn(__dmul_rn(wa.x, ga.y), __dmul_rn(wa.y, ga.x));
      double pb = 0.0;
      if (cb < nc) {
        const double2 wb = cconj(res[cb * ld + y]);
        const double2 gb = g[(int64_t)cb * n + y];
        pb = __dsub_rn(__dmul_rn(wb.x, gb.y), __dmul_rn(wb.y, gb.x));
      }
      other[q * ld + y] = make_double2(pa, pb);
    }
    __syncthreads();
    const double2* res2 = fft::run(a.d, other, res, ld, npair, threadIdx.x, kThreads);
    separate_store(res2, ld, n, npair, nc, Y, colbase, a.nrow);
    return;
  }

  if (a.mode == Y_TO_REAL) {
    for (int e = threadIdx.x; e < npair * n; e += kThreads) {
      const int q = e / n, k = e - q * n;
      const double2 za = zb_herm(colbase + (int64_t)(2 * q) * a.nrow, k, n, Y);
      const double2 zb = (2 * q + 1 < nc) ? zb_herm(colbase + (int64_t)(2 * q + 1) * a.nrow, k, n, Y)
                                          : make_double2(0.0, 0.0);
      buf0[q * ld + k] = cconj(make_double2(__dsub_rn(za.x, zb.y), __dadd_rn(za.y, zb.x)));
    }
    __syncthreads();
    const double2* res = fft::run(a.d, buf0, buf1, ld, npair, threadIdx.x, kThreads);
    double* out = a.field_out + s * n * a.n_x + x0;
    for (int e = threadIdx.x; e < n * nc; e += kThreads) {
      const int y = e / nc, c = e - y * nc;
      const double2 r = res[(c >> 1) * ld + y];  // conj(r) -> (r.x, -r.y)
      out[(int64_t)y * a.n_x + c] = (c & 1) ? -r.y : r.x;
    }
    return;
  }

  // Y_TO_SPEC: real field columns, two per complex transform
  const double* in = a.field_in + s * n * a.n_x + x0;
  for (int e = threadIdx.x; e < npair * n; e += kThreads) {
    const int y = e / npair, q = e - y * npair;
    const double pa = in[(int64_t)y * a.n_x + 2 * q];
    const double pb = (2 * q + 1 < nc) ? in[(int64_t)y * a.n_x + 2 * q + 1] : 0.0;
    buf0[q * ld + y] = make_double2(pa, pb);
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
  double2* out = a.out + ((a.s0 + sl) * a.n_ky + k0) * a.n_kx;
  for (int e = threadIdx.x; e < ntr * a.n_kx; e += kThreads) {
    const int tt = e / a.n_kx, j = e - tt * a.n_kx;
    double2 v = res[tt * ld + kx_to_slot(j, n, a.n_kx)];
    v = make_double2(__ddiv_rn(v.x, a.norm), __ddiv_rn(v.y, a.norm));
    if (nyq_zero && j == a.n_kx / 2) v = make_double2(0.0, 0.0);
    out[(int64_t)tt * a.n_kx + j] = v;
  }
}

// ---------------------------------------------------------------- host side

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

static int64_t chunk_target_bytes() {
  static int64_t v = [] {
    const char* e = getenv("GK_CHUNK_MB");
    const int64_t mb = e ? atoll(e) : 40;
    return (mb > 0 ? mb : 40) << 20;
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

static int set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) GK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return GK_OK;
}

static int xinv(const gk_spectral_plan* p, const double2* f, const int64_t* fmap, double2* m1,
                int64_t s0, int64_t cs, int nrow, int bracket, cudaStream_t st) {
  XInvArgs a{};
  a.d = p->dx;
  a.f = f;
  a.fmap = fmap;
  a.m1 = m1;
  a.s0 = s0;
  a.nrow = nrow;
  a.n_kx = (int)p->n_kx;
  a.n_ky = (int)p->n_ky;
  a.bracket = bracket;
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

static int xfwd(const gk_spectral_plan* p, const double2* m1, double2* out, int64_t s0, int64_t cs,
                int nrow, cudaStream_t st) {
  XFwdArgs a{};
  a.d = p->dx;
  a.m1 = m1;
  a.out = out;
  a.s0 = s0;
  a.nrow = nrow;
  a.n_ky = (int)p->n_ky;
  a.n_kx = (int)p->n_kx;
  a.norm = (double)(p->n_x * p->n_y);
  a.tb = (int)std::max<int64_t>(1, std::min<int64_t>(p->n_ky, kSmemElems / p->n_x));
  a.groups = (int)((p->n_ky + a.tb - 1) / a.tb);
  const size_t smem = 2 * sizeof(double2) * a.tb * p->n_x;
  int rc = set_smem((const void*)xfwd_kernel, smem);
  if (rc) return rc;
  xfwd_kernel<<<(unsigned)(cs * a.groups), kThreads, smem, st>>>(a);
  return check_launch("xfwd_kernel");
}

static int64_t bracket_ws(const gk_spectral_plan* p, int64_t n_slices, int64_t n_g) {
  const int nrow = (int)(2 * p->n_ky - 1);
  const int64_t cs = chunk_slices(p, nrow, std::max(n_slices, n_g));
  return (n_g * p->n_x * p->n_y + cs * p->n_x * nrow) * 16;
}

static int bracket_impl(const gk_spectral_plan* p, const double2* f, const double2* g, double2* out,
                        int64_t n_slices, const int64_t* fmap, const int64_t* gmap, int64_t n_g,
                        int64_t gmod, void* ws, int64_t ws_bytes, cudaStream_t st) {
  GK_CHECK_ARG(p && f && g && out && ws, "gk_bracket: null pointer");
  GK_CHECK_ARG(n_slices >= 0 && n_g >= 1, "gk_bracket: bad batch sizes");
  GK_CHECK_ARG(gmap || (gmod >= 1 && gmod <= n_g), "gk_bracket: need g_map or 1 <= g_mod <= n_g");
  GK_CHECK_ARG(p->n_x >= (3 * p->n_kx + 1) / 2 && p->n_y >= 3 * p->n_ky - 2,
               "gk_bracket: plan below the dealias bounds");
  GK_CHECK_ARG(ws_bytes >= bracket_ws(p, n_slices, n_g), "gk_bracket: workspace too small (%lld < %lld)",
               (long long)ws_bytes, (long long)bracket_ws(p, n_slices, n_g));
  if (n_slices == 0) return GK_OK;
  const int nrow = (int)(2 * p->n_ky - 1);
  const int64_t chunk = chunk_slices(p, nrow, std::max(n_slices, n_g));
  double2* G = (double2*)ws;
  double2* m1 = G + n_g * p->n_x * p->n_y;
  int rc;
  for (int64_t s0 = 0; s0 < n_g; s0 += chunk) {
    const int64_t cs = std::min(chunk, n_g - s0);
    if ((rc = xinv(p, g, nullptr, m1, s0, cs, nrow, 1, st))) return rc;
    YArgs a{};
    a.m1 = m1;
    a.G = G;
    a.s0 = s0;
    a.nrow = nrow;
    a.n_ky = (int)p->n_ky;
    a.mode = Y_PHI;
    if ((rc = ycol(p, a, cs, st))) return rc;
  }
  for (int64_t s0 = 0; s0 < n_slices; s0 += chunk) {
    const int64_t cs = std::min(chunk, n_slices - s0);
    if ((rc = xinv(p, f, fmap, m1, s0, cs, nrow, 1, st))) return rc;
    YArgs a{};
    a.m1 = m1;
    a.G = G;
    a.gmap = gmap;
    a.gmod = gmod;
    a.s0 = s0;
    a.nrow = nrow;
    a.n_ky = (int)p->n_ky;
    a.mode = Y_BRACKET;
    if ((rc = ycol(p, a, cs, st))) return rc;
    if ((rc = xfwd(p, m1, out, s0, cs, nrow, st))) return rc;
  }
  return GK_OK;
}

static void host_twiddles(int64_t n, double2* t) {
  for (int64_t m = 0; m < n; ++m) {
    // exact octant reduction keeps the table symmetric and correctly rounded
    const long double a = 2.0L * 3.141592653589793238462643383279502884L * (long double)m / (long double)n;
    t[m].x = (double)cosl(a);
    t[m].y = (double)-sinl(a);
  }
}

}  // namespace spec
}  // namespace gk

using namespace gk;
using namespace gk::spec;

extern "C" {

int gk_spectral_plan_create(int64_t n_kx, int64_t n_ky, int64_t n_x, int64_t n_y,
                            gk_spectral_plan** plan) {
  GK_CHECK_ARG(plan, "gk_spectral_plan_create: null out pointer");
  *plan = nullptr;
  GK_CHECK_ARG(n_kx >= 1 && n_ky >= 1 && n_x >= n_kx && n_y / 2 + 1 >= n_ky,
               "gk_spectral_plan_create: grid (%lld,%lld) cannot hold (%lld,%lld) modes",
               (long long)n_x, (long long)n_y, (long long)n_kx, (long long)n_ky);
  GK_CHECK_ARG(2 * 16 * n_x <= 200 * 1024 && 2 * 2 * 16 * n_y <= 200 * 1024,
               "gk_spectral_plan_create: transform length above the shared-memory limit");
  auto* p = new gk_spectral_plan{};
  p->n_kx = n_kx;
  p->n_ky = n_ky;
  p->n_x = n_x;
  p->n_y = n_y;
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

int gk_bracket(const gk_spectral_plan* plan, const double* f, const double* g, double* out,
               int64_t n_slices, const int64_t* f_map, const int64_t* g_map, int64_t n_g, int64_t g_mod,
               void* workspace, int64_t workspace_bytes, void* stream) {
  return bracket_impl(plan, (const double2*)f, (const double2*)g, (double2*)out, n_slices, f_map, g_map,
                      n_g, g_mod, workspace, workspace_bytes, (cudaStream_t)stream);
}

int gk_nonlinear(const gk_spectral_plan* plan, const double* h, const double* phi, double* out,
                 int64_t n_vel, int64_t n_theta, void* workspace, int64_t workspace_bytes, void* stream) {
  return bracket_impl(plan, (const double2*)h, (const double2*)phi, (double2*)out, n_vel * n_theta,
                      nullptr, nullptr, n_theta, n_theta, workspace, workspace_bytes,
                      (cudaStream_t)stream);
}

int64_t gk_transform_workspace_bytes(const gk_spectral_plan* plan, int64_t batch) {
  if (!plan) return -1;
  return chunk_slices(plan, (int)plan->n_ky, batch) * plan->n_x * plan->n_ky * 16;
}

int gk_to_real(const gk_spectral_plan* p, const double* spec, double* field, int64_t batch,
               void* ws, int64_t ws_bytes, void* stream) {
  GK_CHECK_ARG(p && spec && field && ws, "gk_to_real: null pointer");
  GK_CHECK_ARG(ws_bytes >= gk_transform_workspace_bytes(p, batch), "gk_to_real: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int nrow = (int)p->n_ky;
  const int64_t chunk = chunk_slices(p, nrow, batch);
  int rc;
  for (int64_t s0 = 0; s0 < batch; s0 += chunk) {
    const int64_t cs = std::min(chunk, batch - s0);
    if ((rc = xinv(p, (const double2*)spec, nullptr, (double2*)ws, s0, cs, nrow, 0, st))) return rc;
    YArgs a{};
    a.m1 = (double2*)ws;
    a.field_out = field;
    a.s0 = s0;
    a.nrow = nrow;
    a.n_ky = nrow;
    a.mode = Y_TO_REAL;
    if ((rc = ycol(p, a, cs, st))) return rc;
  }
  return GK_OK;
}

int gk_to_spectrum(const gk_spectral_plan* p, const double* field, double* spec, int64_t batch,
                   void* ws, int64_t ws_bytes, void* stream) {
  GK_CHECK_ARG(p && spec && field && ws, "gk_to_spectrum: null pointer");
  GK_CHECK_ARG(ws_bytes >= gk_transform_workspace_bytes(p, batch), "gk_to_spectrum: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int nrow = (int)p->n_ky;
  const int64_t chunk = chunk_slices(p, nrow, batch);
  int rc;
  for (int64_t s0 = 0; s0 < batch; s0 += chunk) {
    const int64_t cs = std::min(chunk, batch - s0);
    YArgs a{};
    a.m1 = (double2*)ws;
    a.field_in = field;
    a.s0 = s0;
    a.nrow = nrow;
    a.n_ky = nrow;
    a.mode = Y_TO_SPEC;
    if ((rc = ycol(p, a, cs, st))) return rc;
    if ((rc = xfwd(p, (const double2*)ws, (double2*)spec, s0, cs, nrow, st))) return rc;
  }
  return GK_OK;
}

}  // extern "C"
