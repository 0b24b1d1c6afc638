// HBM-bound velocity/theta/radial kernels: field, stream, shear, the step's axpy
// and the block permutation around the all-to-all transposes.
//
// Layout (reference grid.py:1-11): h[v][t][c] with v = flattened (species, energy,
// xi), t = theta, c = toroidal*radial cell; complex128 == double2.  Every thread
// moves 16-byte elements and consecutive threads touch consecutive cells, so all
// global traffic is fully coalesced; each kernel reads each input element once
// (stream re-reads only the w-1 wrap planes).
#include "gk_common.cuh"
#include "../../include/gk.h"

namespace gk {

constexpr int kThreads = 256;

static int grid_for(int64_t n, int per_thread = 1) {
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t want = cdiv(n, (int64_t)kThreads * per_thread);
  int64_t cap = (int64_t)sms * 16;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
}

// ---------------------------------------------------------------- field
// out[t,c] = sum_v w[v] h[v,t,c] (kernels.py:45-52); one thread per output.
// Fixed summation order, shared with the fused field + int8-slicing pass of the
// step (collision_i8.cu slice_b): 8 interleaved FMA chains, chain p over
// v = p, p + 8, ... ascending, then the 8 partial sums added in ascending p.
// Same bits in both kernels.  CTA = 8 chains (one warp each) x 128 consecutive
// outputs (2 KB contiguous per velocity row); partial sums meet in shared memory.  (range form: outputs [base, base + count) of a plane of `plane` cells)
constexpr int kFieldChains = 8;
constexpr int kFieldLanes = 32, kFieldPer = 4;          // a warp: 4 x 32 consecutive outputs of one chain
constexpr int kFieldOut = kFieldLanes * kFieldPer;      // outputs per CTA (2 KB per velocity row)
__global__ void __launch_bounds__(kFieldChains * kFieldLanes) field_kernel(const double2* __restrict__ h,
                                                                          const double* __restrict__ w,
                                                                          double2* __restrict__ out, int64_t n_vel,
                                                                          int64_t plane, int64_t base,
                                                                          int64_t count) {
  __shared__ double2 part[kFieldChains][kFieldOut];
  const int lane = threadIdx.x % kFieldLanes, chain = threadIdx.x / kFieldLanes;
  const int64_t i0 = base + (int64_t)blockIdx.x * kFieldOut + lane;
  const int64_t lim = base + count;
  double2 acc[kFieldPer];
#pragma unroll
  for (int k = 0; k < kFieldPer; ++k) acc[k] = make_double2(0.0, 0.0);
  for (int64_t v = chain; v < n_vel; v += kFieldChains) {
    const double2* p = h + v * plane + i0;
    const double wv = __ldg(w + v);
#pragma unroll
    for (int k = 0; k < kFieldPer; ++k) {
      if (i0 + k * kFieldLanes < lim) {
        const double2 x = __ldcs(p + k * kFieldLanes);
        acc[k].x = __fma_rn(wv, x.x, acc[k].x);
        acc[k].y = __fma_rn(wv, x.y, acc[k].y);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kFieldPer; ++k) part[chain][lane + k * kFieldLanes] = acc[k];
  __syncthreads();
  for (int o = threadIdx.x; o < kFieldOut; o += blockDim.x) {
    const int64_t i = base + (int64_t)blockIdx.x * kFieldOut + o;
    if (i >= lim) continue;
    double2 sum = part[0][o];
#pragma unroll
    for (int q = 1; q < kFieldChains; ++q)
      sum = make_double2(__dadd_rn(sum.x, part[q][o].x), __dadd_rn(sum.y, part[q][o].y));
    out[i] = sum;
  }
}

// ---------------------------------------------------------------- stream
struct Stencil {
  double c[32];
};

// One thread per (v, c) column, sliding a W-wide register window along theta.
// ORIGINAL: acc = 0; acc += c_i * h[t-half+i] for i ascending (kernels.py:70-74,
// numpy's roll-accumulate: separate multiply and add roundings -> bit-exact).
// OPTIMIZED: FMA chain in the same order (kernels.py:75-77 semantics).
template <int W, bool ORIGINAL>
__global__ void __launch_bounds__(kThreads) stream_kernel_w(const double2* __restrict__ h,
                                                            double2* __restrict__ out,
                                                            Stencil st, int64_t n_vel, int n_theta,
                                                            int64_t n_cells) {
  constexpr int half = W / 2;
  const int64_t cols = n_vel * n_cells;
  for (int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; col < cols;
       col += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = col / n_cells;
    const int64_t c = col - v * n_cells;
    const double2* src = h + v * n_theta * n_cells + c;
    double2* dst = out + v * n_theta * n_cells + c;
    double2 win[W];
#pragma unroll
    for (int i = 0; i < W; ++i) {
      int t = i - half;
      t = t < 0 ? t + n_theta : t;
      win[i] = src[(int64_t)t * n_cells];
    }
    for (int t = 0; t < n_theta; ++t) {
      double2 acc;
      if (ORIGINAL) {
        acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < W; ++i) {
          acc.x = __dadd_rn(acc.x, __dmul_rn(st.c[i], win[i].x));
          acc.y = __dadd_rn(acc.y, __dmul_rn(st.c[i], win[i].y));
        }
      } else {
        acc = make_double2(__dmul_rn(st.c[0], win[0].x), __dmul_rn(st.c[0], win[0].y));
#pragma unroll
        for (int i = 1; i < W; ++i) {
          acc.x = __fma_rn(st.c[i], win[i].x, acc.x);
          acc.y = __fma_rn(st.c[i], win[i].y, acc.y);
        }
      }
      __stcs(dst + (int64_t)t * n_cells, acc);
      if (t + 1 < n_theta) {
#pragma unroll
        for (int i = 0; i + 1 < W; ++i) win[i] = win[i + 1];
        int tn = t + 1 + half;
        tn = tn >= n_theta ? tn - n_theta : tn;
        win[W - 1] = src[(int64_t)tn * n_cells];
      }
    }
  }
}

// Any odd width up to 32: per output, w gathered loads (L1/L2 absorb the reuse).
template <bool ORIGINAL>
__global__ void __launch_bounds__(kThreads) stream_kernel_generic(const double2* __restrict__ h,
                                                                  double2* __restrict__ out,
                                                                  Stencil st, int w, int64_t n_vel,
                                                                  int n_theta, int64_t n_cells) {
  const int half = w / 2;
  const int64_t total = n_vel * n_theta * n_cells;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx % n_cells;
    const int64_t vt = idx / n_cells;
    const int t = (int)(vt % n_theta);
    const int64_t v = vt / n_theta;
    const double2* src = h + v * n_theta * n_cells + c;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < w; ++i) {
      int tt = t + i - half;
      tt = ((tt % n_theta) + n_theta) % n_theta;
      const double2 x = src[(int64_t)tt * n_cells];
      if (ORIGINAL || i > 0) {
        if (ORIGINAL) {
          acc.x = __dadd_rn(acc.x, __dmul_rn(st.c[i], x.x));
          acc.y = __dadd_rn(acc.y, __dmul_rn(st.c[i], x.y));
        } else {
          acc.x = __fma_rn(st.c[i], x.x, acc.x);
          acc.y = __fma_rn(st.c[i], x.y, acc.y);
        }
      } else {
        acc = make_double2(__dmul_rn(st.c[0], x.x), __dmul_rn(st.c[0], x.y));
      }
    }
    out[idx] = acc;
  }
}

// Any odd width <= n_theta (kernels.py:65-68 accepts every odd w <= n_theta): the
// coefficients come from device memory (wider than the kernel-parameter copy
// holds).  One thread per (v, cell) column walks theta; the window of w values is
// re-read per output from L1/L2 (h[v, :, c] is T values 16 * n_cells apart).
// Same accumulation orders as the fixed-width kernels: ORIGINAL = 0 + c_0 x_0 +
// c_1 x_1 + ... with separate mul/add (the reference's roll loop), optimized =
// c_0 x_0 then an FMA chain.
template <bool ORIGINAL>
__global__ void __launch_bounds__(kThreads) stream_kernel_wide(const double2* __restrict__ h,
                                                               double2* __restrict__ out,
                                                               const double* __restrict__ c, int w, int64_t n_vel,
                                                               int n_theta, int64_t n_cells) {
  const int half = w / 2;
  const int64_t cols = n_vel * n_cells;
  for (int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; col < cols;
       col += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = col / n_cells;
    const int64_t cc = col - v * n_cells;
    const double2* src = h + v * n_theta * n_cells + cc;
    double2* dst = out + v * n_theta * n_cells + cc;
    for (int t = 0; t < n_theta; ++t) {
      int tt = t - half;
      tt = tt < 0 ? tt + n_theta : tt;
      double2 acc = make_double2(0.0, 0.0);
      for (int i = 0; i < w; ++i) {
        const double2 x = src[(int64_t)tt * n_cells];
        const double ci = __ldg(c + i);
        if (ORIGINAL) {
          acc.x = __dadd_rn(acc.x, __dmul_rn(ci, x.x));
          acc.y = __dadd_rn(acc.y, __dmul_rn(ci, x.y));
        } else if (i == 0) {
          acc = make_double2(__dmul_rn(ci, x.x), __dmul_rn(ci, x.y));
        } else {
          acc.x = __fma_rn(ci, x.x, acc.x);
          acc.y = __fma_rn(ci, x.y, acc.y);
        }
        tt = tt + 1 == n_theta ? 0 : tt + 1;
      }
      __stcs(dst + (int64_t)t * n_cells, acc);
    }
  }
}

// ---------------------------------------------------------------- shear
// out[r,ky,kx] = h[r,ky,kx+s[ky]] or 0 (kernels.py:80-106).
__global__ void __launch_bounds__(kThreads) shear_kernel(const double2* __restrict__ h,
                                                         const int* __restrict__ shifts,
                                                         double2* __restrict__ out, int64_t total,
                                                         int n_ky, int n_kx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i % n_kx);
    const int64_t rowy = i / n_kx;
    const int ky = (int)(rowy % n_ky);
    const int src = kx + __ldg(shifts + ky);
    double2 v = make_double2(0.0, 0.0);
    if (src >= 0 && src < n_kx) v = __ldcs(h + (i - kx + src));
    __stcs(out + i, v);
  }
}

// ---------------------------------------------------------------- axpy3
// out = h + dt * ((a + b) + c): numpy's rounding sequence for
// h + dt*(stream + nonlinear + collision) (separate mul/add, no FMA).
__global__ void __launch_bounds__(kThreads) axpy3_kernel(const double2* __restrict__ h,
                                                         const double2* __restrict__ a,
                                                         const double2* __restrict__ b,
                                                         const double2* c, double dt,
                                                         double2* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 r = __ldcs(a + i);
    if (b) r = cadd(r, __ldcs(b + i));
    if (c) r = cadd(r, __ldcs(c + i));
    const double2 x = __ldcs(h + i);
    out[i] = make_double2(__dadd_rn(x.x, __dmul_rn(dt, r.x)), __dadd_rn(x.y, __dmul_rn(dt, r.y)));
  }
}

// ---------------------------------------------------------------- in-place step
// rhs <- h + dt * (stream(h) + rhs), elementwise in place on rhs (each thread reads
// and writes only its own (v, cell) column of rhs; h is read through the same
// sliding theta window and FMA chain as finish_kernel).  The in-place step
// (step.cu gk_step_inplace) then shears rhs back into h.
template <int W>
__global__ void __launch_bounds__(kThreads) stream_axpy_kernel(const double2* __restrict__ h, double2* rhs,
                                                               Stencil st, double dt, int64_t n_vel, int n_theta,
                                                               int64_t n_cells) {
  constexpr int half = W / 2;
  const int64_t cols = n_vel * n_cells;
  for (int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; col < cols;
       col += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = col / n_cells;
    const int64_t c = col - v * n_cells;
    const int64_t base = v * n_theta * n_cells + c;
    const double2* src = h + base;
    double2 win[W];
#pragma unroll
    for (int i = 0; i < W; ++i) {
      int t = i - half;
      t = t < 0 ? t + n_theta : (t >= n_theta ? t - n_theta : t);
      win[i] = src[(int64_t)t * n_cells];
    }
    for (int t = 0; t < n_theta; ++t) {
      double2 r = make_double2(__dmul_rn(st.c[0], win[0].x), __dmul_rn(st.c[0], win[0].y));
#pragma unroll
      for (int i = 1; i < W; ++i) {
        r.x = __fma_rn(st.c[i], win[i].x, r.x);
        r.y = __fma_rn(st.c[i], win[i].y, r.y);
      }
      double2* e = rhs + base + (int64_t)t * n_cells;
      r = cadd(r, *e);
      const double2 x = win[half];
      *e = make_double2(__dadd_rn(x.x, __dmul_rn(dt, r.x)), __dadd_rn(x.y, __dmul_rn(dt, r.y)));
      if (t + 1 < n_theta) {
#pragma unroll
        for (int i = 0; i + 1 < W; ++i) win[i] = win[i + 1];
        int tn = t + 1 + half;
        tn = tn >= n_theta ? tn - n_theta : tn;
        win[W - 1] = src[(int64_t)tn * n_cells];
      }
    }
  }
}

// ---------------------------------------------------------------- step finish
// out = shear(h + dt * ((stream(h) + nl) + coll)), one pass: each thread owns a
// (v, cell) column, slides the stream window along theta like stream_kernel_w
// (same FMA chain as GK_STREAM_OPTIMIZED) and writes the shear gather as a
// scatter: source kx lands at (kx - s) mod R, and the sources that fall off the
// edge write the zero fill -- a bijection, so every output is written once.
// Same operations in the same order as stream -> axpy3 -> shear (bit-exact).
template <int W>
__global__ void __launch_bounds__(kThreads) finish_kernel(const double2* __restrict__ h,
                                                          const double2* __restrict__ nl,
                                                          const double2* __restrict__ coll, Stencil st,
                                                          const int* __restrict__ shifts, double dt,
                                                          double2* __restrict__ out, int64_t n_vel, int n_theta,
                                                          int n_ky, int n_kx, int t0, int t1) {
  constexpr int half = W / 2;
  const int64_t n_cells = (int64_t)n_ky * n_kx;
  const int64_t cols = n_vel * n_cells;
  for (int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; col < cols;
       col += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = col / n_cells;
    const int64_t c = col - v * n_cells;
    const int ky = (int)(c / n_kx), kx = (int)(c - (int64_t)ky * n_kx);
    const int dkx = kx - __ldg(shifts + ky);
    const bool keep = dkx >= 0 && dkx < n_kx;
    const int64_t dc = (int64_t)ky * n_kx + (keep ? dkx : (dkx < 0 ? dkx + n_kx : dkx - n_kx));
    const int64_t base = v * n_theta * n_cells;
    const double2* src = h + base + c;
    double2 win[W];
#pragma unroll
    for (int i = 0; i < W; ++i) {
      int t = t0 + i - half;
      t = t < 0 ? t + n_theta : (t >= n_theta ? t - n_theta : t);
      win[i] = src[(int64_t)t * n_cells];
    }
    for (int t = t0; t < t1; ++t) {
      double2 r = make_double2(__dmul_rn(st.c[0], win[0].x), __dmul_rn(st.c[0], win[0].y));
#pragma unroll
      for (int i = 1; i < W; ++i) {
        r.x = __fma_rn(st.c[i], win[i].x, r.x);
        r.y = __fma_rn(st.c[i], win[i].y, r.y);
      }
      const int64_t e = base + (int64_t)t * n_cells + c;
      if (nl) r = cadd(r, __ldcs(nl + e));
      r = cadd(r, __ldcs(coll + e));
      const double2 x = win[half];
      double2 o = make_double2(__dadd_rn(x.x, __dmul_rn(dt, r.x)), __dadd_rn(x.y, __dmul_rn(dt, r.y)));
      if (!keep) o = make_double2(0.0, 0.0);
      __stcs(out + base + (int64_t)t * n_cells + dc, o);
      if (t + 1 < t1) {
#pragma unroll
        for (int i = 0; i + 1 < W; ++i) win[i] = win[i + 1];
        int tn = t + 1 + half;
        tn = tn >= n_theta ? tn - n_theta : tn;
        win[W - 1] = src[(int64_t)tn * n_cells];
      }
    }
  }
}

// ---------------------------------------------------------------- permute
__global__ void __launch_bounds__(kThreads) permute_kernel(const double2* __restrict__ src,
                                                           double2* __restrict__ dst, int64_t n_a,
                                                           int64_t n_b, int64_t inner) {
  const int64_t total = n_a * n_b * inner;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i % inner;
    const int64_t ab = i / inner;
    const int64_t b = ab % n_b;
    const int64_t a = ab / n_b;
    dst[(b * n_a + a) * inner + k] = __ldcs(src + i);
  }
}

}  // namespace gk

using namespace gk;

extern "C" {

int gk_field(const double* h, const double* weights, double* out, int64_t n_vel, int64_t n_theta,
             int64_t n_cells, void* stream) {
  GK_CHECK_ARG(h && weights && out, "gk_field: null pointer");
  GK_CHECK_ARG(n_vel > 0 && n_theta > 0 && n_cells > 0, "gk_field: empty dims");
  const int64_t plane = n_theta * n_cells;
  field_kernel<<<(unsigned)cdiv(plane, kFieldOut), kFieldChains * kFieldLanes, 0, (cudaStream_t)stream>>>(
      (const double2*)h, weights, (double2*)out, n_vel, plane, 0, plane);
  return check_launch("gk_field");
}

int gk_field_range(const double* h, const double* weights, double* out, int64_t n_vel, int64_t n_theta,
                   int64_t n_cells, int64_t t0, int64_t t1, void* stream) {
  GK_CHECK_ARG(h && weights && out, "gk_field_range: null pointer");
  GK_CHECK_ARG(0 <= t0 && t0 <= t1 && t1 <= n_theta, "gk_field_range: bad theta range");
  const int64_t count = (t1 - t0) * n_cells;
  if (count == 0) return GK_OK;
  field_kernel<<<(unsigned)cdiv(count, kFieldOut), kFieldChains * kFieldLanes, 0, (cudaStream_t)stream>>>(
      (const double2*)h, weights, (double2*)out, n_vel, n_theta * n_cells, t0 * n_cells, count);
  return check_launch("gk_field_range");
}

int gk_stream(const double* h, const double* stencil_host, int width, int variant, double* out,
              int64_t n_vel, int64_t n_theta, int64_t n_cells, void* stream) {
  GK_CHECK_ARG(h && stencil_host && out, "gk_stream: null pointer");
  GK_CHECK_ARG(width % 2 == 1 && width >= 1 && width <= 31, "gk_stream: width %d must be odd and <= 31", width);
  GK_CHECK_ARG(width <= n_theta, "gk_stream: width %d exceeds n_theta %lld", width, (long long)n_theta);
  GK_CHECK_ARG(variant == GK_STREAM_ORIGINAL || variant == GK_STREAM_OPTIMIZED, "gk_stream: bad variant");
  Stencil st{};
  for (int i = 0; i < width; ++i) st.c[i] = stencil_host[i];
  cudaStream_t s = (cudaStream_t)stream;
  const bool orig = variant == GK_STREAM_ORIGINAL;
  const int64_t cols = n_vel * n_cells;
  const double2* hi = (const double2*)h;
  double2* ho = (double2*)out;
  const int nt = (int)n_theta;
#define GK_STREAM_W(WW)                                                                   \
  case WW:                                                                                \
    if (orig)                                                                             \
      stream_kernel_w<WW, true><<<grid_for(cols), kThreads, 0, s>>>(hi, ho, st, n_vel, nt, n_cells); \
    else                                                                                  \
      stream_kernel_w<WW, false><<<grid_for(cols), kThreads, 0, s>>>(hi, ho, st, n_vel, nt, n_cells); \
    break;
  switch (width) {
    GK_STREAM_W(1)
    GK_STREAM_W(3)
    GK_STREAM_W(5)
    GK_STREAM_W(7)
    GK_STREAM_W(9)
    default: {
      const int64_t total = cols * n_theta;
      if (orig)
        stream_kernel_generic<true><<<grid_for(total), kThreads, 0, s>>>(hi, ho, st, width, n_vel, nt, n_cells);
      else
        stream_kernel_generic<false><<<grid_for(total), kThreads, 0, s>>>(hi, ho, st, width, n_vel, nt, n_cells);
    }
  }
#undef GK_STREAM_W
  return check_launch("gk_stream");
}

int gk_stream_wide(const double* h, const double* stencil_dev, int width, int variant, double* out,
                   int64_t n_vel, int64_t n_theta, int64_t n_cells, void* stream) {
  GK_CHECK_ARG(h && stencil_dev && out, "gk_stream_wide: null pointer");
  GK_CHECK_ARG(width % 2 == 1 && width >= 1, "gk_stream_wide: width %d must be odd", width);
  GK_CHECK_ARG(width <= n_theta, "gk_stream_wide: width %d exceeds n_theta %lld", width, (long long)n_theta);
  GK_CHECK_ARG(variant == GK_STREAM_ORIGINAL || variant == GK_STREAM_OPTIMIZED, "gk_stream_wide: bad variant");
  const int64_t cols = n_vel * n_cells;
  if (cols == 0) return GK_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (variant == GK_STREAM_ORIGINAL)
    stream_kernel_wide<true><<<grid_for(cols), kThreads, 0, s>>>((const double2*)h, (double2*)out, stencil_dev, width,
                                                                 n_vel, (int)n_theta, n_cells);
  else
    stream_kernel_wide<false><<<grid_for(cols), kThreads, 0, s>>>((const double2*)h, (double2*)out, stencil_dev,
                                                                  width, n_vel, (int)n_theta, n_cells);
  return check_launch("gk_stream_wide");
}

int gk_shear(const double* h, const int32_t* shifts, double* out, int64_t n_rows, int64_t n_ky,
             int64_t n_kx, void* stream) {
  GK_CHECK_ARG(h && shifts && out, "gk_shear: null pointer");
  const int64_t total = n_rows * n_ky * n_kx;
  if (total == 0) return GK_OK;
  shear_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(
      (const double2*)h, shifts, (double2*)out, total, (int)n_ky, (int)n_kx);
  return check_launch("gk_shear");
}

int gk_axpy3(const double* h, const double* a, const double* b, const double* c, double dt,
             double* out, int64_t n, void* stream) {
  GK_CHECK_ARG(h && a && out, "gk_axpy3: null pointer");
  if (n == 0) return GK_OK;
  axpy3_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(
      (const double2*)h, (const double2*)a, (const double2*)b, (const double2*)c, dt,
      (double2*)out, n);
  return check_launch("gk_axpy3");
}

int gk_step_finish_range(const double* h, const double* nl, const double* coll, const double* stencil_host,
                         int width, const int32_t* shifts, double dt, double* out, int64_t n_vel,
                         int64_t n_theta, int64_t n_ky, int64_t n_kx, int64_t t0, int64_t t1, void* stream) {
  GK_CHECK_ARG(h && coll && stencil_host && shifts && out, "gk_step_finish: null pointer");
  GK_CHECK_ARG(0 <= t0 && t0 <= t1 && t1 <= n_theta, "gk_step_finish: bad theta range");
  GK_CHECK_ARG(out != h && out != coll && out != nl, "gk_step_finish: out must not alias an input");
  GK_CHECK_ARG(width % 2 == 1 && width <= n_theta, "gk_step_finish: bad stencil width");
  Stencil st{};
  for (int i = 0; i < width; ++i) st.c[i] = stencil_host[i];
  const int64_t cols = n_vel * n_ky * n_kx;
  cudaStream_t s = (cudaStream_t)stream;
  const double2* a = (const double2*)h;
  const double2* b = (const double2*)nl;
  const double2* c = (const double2*)coll;
  double2* o = (double2*)out;
#define GK_FIN(WW)                                                                                  \
  case WW:                                                                                          \
    finish_kernel<WW><<<grid_for(cols), kThreads, 0, s>>>(a, b, c, st, shifts, dt, o, n_vel,        \
                                                           (int)n_theta, (int)n_ky, (int)n_kx,       \
                                                           (int)t0, (int)t1);                        \
    break;
  switch (width) {
    GK_FIN(1)
    GK_FIN(3)
    GK_FIN(5)
    GK_FIN(7)
    GK_FIN(9)
    default: {
      gk::set_error("gk_step_finish: stencil width %d not specialised (use stream + axpy3 + shear)", width);
      return GK_ERR_ARG;
    }
  }
#undef GK_FIN
  return check_launch("gk_step_finish");
}

int gk_step_finish(const double* h, const double* nl, const double* coll, const double* stencil_host,
                   int width, const int32_t* shifts, double dt, double* out, int64_t n_vel, int64_t n_theta,
                   int64_t n_ky, int64_t n_kx, void* stream) {
  return gk_step_finish_range(h, nl, coll, stencil_host, width, shifts, dt, out, n_vel, n_theta, n_ky, n_kx, 0,
                              n_theta, stream);
}

int gk_stream_axpy_inplace(const double* h, double* rhs, const double* stencil_host, int width, double dt,
                           int64_t n_vel, int64_t n_theta, int64_t n_cells, void* stream) {
  GK_CHECK_ARG(h && rhs && stencil_host, "gk_stream_axpy_inplace: null pointer");
  GK_CHECK_ARG(h != rhs, "gk_stream_axpy_inplace: rhs must not alias h");
  GK_CHECK_ARG(width % 2 == 1 && width <= n_theta, "gk_stream_axpy_inplace: bad stencil width");
  Stencil st{};
  for (int i = 0; i < width; ++i) st.c[i] = stencil_host[i];
  const int64_t cols = n_vel * n_cells;
  cudaStream_t s = (cudaStream_t)stream;
#define GK_SAX(WW)                                                                                          \
  case WW:                                                                                                  \
    stream_axpy_kernel<WW><<<grid_for(cols), kThreads, 0, s>>>((const double2*)h, (double2*)rhs, st, dt,   \
                                                               n_vel, (int)n_theta, n_cells);              \
    break;
  switch (width) {
    GK_SAX(1)
    GK_SAX(3)
    GK_SAX(5)
    GK_SAX(7)
    GK_SAX(9)
    default: {
      gk::set_error("gk_stream_axpy_inplace: stencil width %d not specialised", width);
      return GK_ERR_ARG;
    }
  }
#undef GK_SAX
  return check_launch("gk_stream_axpy_inplace");
}

int gk_permute_blocks(const double* src, double* dst, int64_t n_a, int64_t n_b, int64_t inner,
                      void* stream) {
  GK_CHECK_ARG(src && dst && src != dst, "gk_permute_blocks: bad pointers");
  const int64_t total = n_a * n_b * inner;
  if (total == 0) return GK_OK;
  permute_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(
      (const double2*)src, (double2*)dst, n_a, n_b, inner);
  return check_launch("gk_permute_blocks");
}

}  // extern "C"
