// Collision on the int8 tensor cores: fp64 A_t @ B_t (reference kernels.py:109-123)
// by exact int8 slice products (Ozaki scheme) on tcgen05 kind::i8.
//
// fp64 -> int8 slices.  Every column j of B_t (one real component of one
// (toroidal, radial) cell over velocity space, K = n_vel long) gets a power-of-two
// scale 2^e_j > max|B[:, j]|; v = rint(B * 2^(46 - e_j)) (|v| <= 2^46, error
// <= 2^-47 of the scale) is written as six balanced base-256 digits,
//   B[m, j] ~= 2^e_j * sum_s b_s[m, j] 2^(-6 - 8 s),   b_s in [-128, 127],
// read off the bytes of (v + B) ^ B (slice16; exact, no carry chain, no rounding
// ties).  Rows of A_t likewise
// (scale 2^f_i).  Then
//   C[i, j] = 2^(e_j + f_i - 12) * sum_d 2^(-8 d) acc_d,  acc_d = sum_{s + t = d} a_t[i, :] . b_s[:, j]
// keeping the 21 slice pairs with s + t <= 5 (dropped pairs weigh <= 2^-48 of
// the scales).  Each acc_d is an exact int32 (|acc_d| <= 6 * K * 2^14 < 2^31 for
// K <= 2^13).  The products of the slices are exact; the rounding is in the
// slicing: every entry is rounded to 46 bits of its column's (row's) maximum, so
// the error bound is ~2^-46 K max|A_i| max|B_j| (normwise), not DGEMM's
// componentwise eps sum_k |A_ik||B_kj|.  Measured on the benchmark state: max-abs
// relative error 3-6e-14 against the fp64 DGEMM (bench.py strict_fp64 reports it
// each run); the reference's parity bar is 1e-12.
//
// The GEMM (one per theta) runs as D^T = B_t^T A_t^T: UMMA M = 128 columns of B,
// N = 64 rows of A, K = 32 per MMA (the measured tcgen05 i8 rate at M128 N64 is
// 2/3 of the N128 peak -- operand bytes from shared memory are the limiter --
// but 6 accumulators of N = 64 fit in TMEM, N = 128 would not).  Per K step a
// stage holds the 6 B slices (6 x 4 KB) and 6 A slices (6 x 2 KB), each written
// by the slicing kernels in the UMMA canonical K-major layout so the stage is
// two bulk copies.  Warp roles: 0 bulk-copy producer, 1 MMA issuer (one thread),
// 2-5 epilogue (TMEM lane quadrants); the 6 accumulators are combined in fp64
// in the epilogue and streamed out.  Persistent CTAs walk (theta, column block,
// row block) with the row block fastest, so the CTAs in flight share B slices
// through L2.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "gk_common.cuh"
#include "../../include/gk.h"

namespace gk {
int collision_fix_dmma(const double* A, const double* H, double* C, int M, int T, int64_t N, int ncb, int nib,
                       const unsigned* list, const unsigned* count, int64_t max_tiles, unsigned long long* fixed,
                       int sms, cudaStream_t s);
}  // namespace gk
namespace gk {
namespace i8 {

constexpr int S = 6;                 // digit slices per operand
constexpr int SB = S + 1;            // stored slices: the digits + the magnitude slice (certificate)
constexpr int BJ = 128;              // UMMA M: columns of B per tile
constexpr int BI = 64;               // UMMA N: rows of A per tile
constexpr int BK = 32;               // UMMA K (int8)
constexpr int HB = BJ * BK;          // bytes of one B slice tile per K step
constexpr int AB = BI * BK;          // bytes of one A slice tile per K step
constexpr int STAGE = SB * (HB + AB); // 43008
constexpr int STAGES = 5;
#ifndef GK_I8_EPI_WARPS
#define GK_I8_EPI_WARPS 8
#endif
constexpr int EPI_WARPS = GK_I8_EPI_WARPS;     // per TMEM lane quadrant: EPI_WARPS / 4
constexpr int RPW = BI * 4 / EPI_WARPS;        // accumulator columns (rows of A) per epilogue warp
static_assert(RPW % 16 == 0 && RPW <= 32, "epilogue: 16-column TMEM loads, rows held by lanes");
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024;

// --------------------------------------------------------------- slicing

constexpr int kNonFinite = 0x7fffffff;  // column scale marker: an Inf/NaN in the column

__device__ __forceinline__ double pow2(int e) {
  return (e >= -1022 && e <= 1023) ? __longlong_as_double((long long)(e + 1023) << 52) : ldexp(1.0, e);
}

__device__ __forceinline__ int scale_exp(double mx) {
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1): mx < 2^e
  return e;
}

// x * 2^(46 - e) for |x| < 2^e: a per-column power of two when it is a normal
// double, ldexp otherwise (columns of magnitude < ~2^-976)
struct Scale {
  double p;
  int e;
  __device__ __forceinline__ long long operator()(double x) const {
    return __double2ll_rn(p != 0.0 ? __dmul_rn(x, p) : ldexp(x, 46 - e));
  }
};
__device__ __forceinline__ Scale make_scale(int e) {
  const int k = 46 - e;
  return Scale{(k >= -1022 && k <= 1023) ? __longlong_as_double((long long)(k + 1023) << 52) : 0.0, e};
}

// digits of 16 consecutive K values -> six 16-byte words (one per slice)
template <class Get>
__device__ __forceinline__ void slice16(const Scale& sc, Get get, uint4 (&w)[S], int& dsum) {
  // Balanced base-256 digits without a carry chain: with B = 0x808080808080,
  // u = (v + B) ^ B holds in byte k exactly the int8 digit d_k of
  // v = sum_k d_k 256^k, d_k in [-128, 127] (byte b of v + B read as int8 after
  // the xor is b - 128; |v| <= 2^46 keeps v + B in [0, 2^48)).  Slice s is digit
  // k = 5 - s; four values' byte k pack into one word with three byte permutes.
  // v = rint(x 2^(46 - e)) comes from the bits of d = x 2^(46 - e) + 1.5 * 2^52
  // (one rounding, to nearest even, exactly rint for |v| < 2^51):
  // v + B = bits(d) - (bits(1.5 * 2^52) - B).  The multiply-add is exact when
  // 2^(46 - e) is a normal double (every column but ~2^-976-tiny ones).
  constexpr unsigned long long kBias = 0x808080808080ull;
  constexpr long long kMagicBits = 0x4338000000000000ll;  // bits of 1.5 * 2^52
  constexpr double kMagic = 6755399441055744.0;
  unsigned lo[16], hi[16];
  if (sc.p != 0.0) {
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      const double d = __fma_rn(get(b), sc.p, kMagic);
      const unsigned long long u =
          (unsigned long long)(__double_as_longlong(d) - (kMagicBits - (long long)kBias)) ^ kBias;
      lo[b] = (unsigned)u;
      hi[b] = (unsigned)(u >> 32);
    }
  } else {
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      const unsigned long long u = (unsigned long long)(sc(get(b)) + (long long)kBias) ^ kBias;
      lo[b] = (unsigned)u;
      hi[b] = (unsigned)(u >> 32);
    }
  }
  // sum of |digit| over slices 1..5 (bytes k = 0..4) of the 16 values: the
  // certificate's bound on the dropped slice pairs
#pragma unroll
  for (int b = 0; b < 16; ++b) dsum += (int)__vsadu4(__vabs4(lo[b]), 0u) + abs((int)(signed char)(hi[b] & 0xffu));
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int k = S - 1 - s, kk = k & 3;
    const unsigned sel = (unsigned)kk | ((unsigned)(kk + 4) << 4);
    unsigned word[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned* x = k < 4 ? lo : hi;
      const unsigned t01 = __byte_perm(x[4 * q], x[4 * q + 1], sel);
      const unsigned t23 = __byte_perm(x[4 * q + 2], x[4 * q + 3], sel);
      word[q] = __byte_perm(t01, t23, 0x5410);
    }
    w[s] = make_uint4(word[0], word[1], word[2], word[3]);
  }
}

// Magnitude slice (the accuracy certificate's operand): byte b of the word is
// floor(|x_b| 2^(7 - e)) in [0, 127], a lower bound of |x_b| in units of 2^(e - 7).
// The int8 product of the A and B magnitude slices, Q = sum_k p_ik q_kj, bounds
// sum_k |A_ik| |B_kj| >= 2^(e_j + f_i - 14) Q from below (see ozaki_gemm's epilogue).
template <class Get>
__device__ __forceinline__ uint4 mag16(const Scale& sc, Get get) {
  unsigned w[4] = {0u, 0u, 0u, 0u};
  if (sc.p != 0.0) {  // one branch per 16 values (the scale is per column)
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      const double t = __dmul_rn(__dmul_rn(fabs(get(b)), sc.p), 0x1p-39);
      const int q = min(__double2int_rd(t), 127);
      w[b >> 2] |= (unsigned)q << (8 * (b & 3));
    }
  } else {
#pragma unroll 1
    for (int b = 0; b < 16; ++b) {
      const int q = min(__double2int_rd(ldexp(fabs(get(b)), 7 - sc.e)), 127);
      w[b >> 2] |= (unsigned)q << (8 * (b & 3));
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// Per-column (B) and per-row (A) statistics of the certificate.
struct ColStat {
  int e;       // scale exponent (kNonFinite: an Inf/NaN in the column)
  float beta;  // sum_k |B_kj| 2^-e_j, rounded up
  int nnz;     // nonzero entries of the column
  int dsum;    // sum_k sum_{s=1..5} |b_s[k, j]| (digit magnitudes below the top slice)
};
struct RowStat {
  float alpha;  // sum_k |A_ik| 2^-f_i, rounded up
  int nnz;      // nonzero entries of the row
  int dsum;     // sum_k sum_{t=1..5} |a_t[i, k]|
  int pad;
};

// B slices.  CTA = CW columns x one theta, 256 threads; the CW x K column block is
// staged in shared memory (one DRAM read of B), reduced to per-column scales,
// then sliced.  Output tile layout per (theta, 128-column block cb, ks, s):
// [16-byte K chunk c][row j % 128][16 bytes].
#ifndef GK_SB_THREADS
#define GK_SB_THREADS 256
#endif
constexpr int SB_THREADS = GK_SB_THREADS;
// With `phi`, the CTA also computes the field moment of its columns,
// phi[t, j] = sum_v w[v] h[v, t, j], from the staged block in field_kernel's
// fixed order (linear.cu: 8 interleaved FMA chains, then their sum in ascending
// chain order) -- bit-identical to gk_field -- so the step reads the state once
// for the field moment and the collision's B slices.
// Shared memory beyond the K x CW block is 1 KB + CW ints (the column maxima and
// then the chain sums share one buffer), so three CTAs fit in an SM at M = 576.
constexpr int kFieldChains = 8;
// Reduction scratch of one column block (per CTA, or per consumer group of the
// pipelined kernel).
template <int CW>
struct SbRed {
  // per-warp column maxima of the |x| high words [warp][CW] (as unsigned), then
  // the field chain sums [chain][CW] -- one buffer: three CTAs of slice_b just fit
  // an SM at M = 576
  double red[128];
  __device__ __forceinline__ unsigned* rhi() { return reinterpret_cast<unsigned*>(red); }
  double rsum[128];  // per-warp column sums of |x| [warp][CW]
  int rnz[128];      // per-warp column nonzero counts [warp][CW]
  int cdsum[CW];     // column digit-magnitude sums
  ColStat cstat[CW];
  int sexp[CW];
};
// Reduce, scale and slice one staged K x CW column block (rows >= M and, for the
// pipelined kernel, columns >= N may hold anything that is finite or not: such
// columns are never written).  NT threads (tid < NT), `sync` a barrier over them;
// `after_slice` runs once every read of `blk` is done.
template <int CW, int NT, class Sync, class After>
__device__ __forceinline__ void slice_block(const double* __restrict__ blk, int tid, SbRed<CW>& r, const Sync& sync,
                                            const After& after_slice, int64_t N, int M, int t, int tt, int64_t j0,
                                            int ncb, int nks, int8_t* __restrict__ out, ColStat* __restrict__ bexp,
                                            const double* __restrict__ w, double* __restrict__ phi) {
  static_assert(kFieldChains * CW <= 128 && (NT / 32) * CW <= 128, "red[] holds both reductions");
  const int Kp = nks * BK;
  const int jl = tid % CW, part = tid / CW;
  double facc = 0.0;  // chain part of column jl (threads < kFieldChains * CW)
  {
    constexpr int np = NT / CW;
    // an Inf or NaN anywhere in the column makes its partial max NaN (fmax alone
    // would skip NaNs); lanes l, l + CW, ... of a warp hold the same column
    // The scale needs only the exponent of max|x|: the maximum of the high words
    // of |x| (sign cleared) carries it (normal values), and Inf / NaN sort above
    // every finite value.  Columns whose entries are all subnormal (high words
    // below 2^20) get their exact maximum in the scale phase.
    double sa = 0.0;
    unsigned hm = 0u;
    int nz = 0;
    for (int m = part; m < Kp; m += np) {
      const double x = blk[m * CW + jl];
      hm = max(hm, (unsigned)__double2hiint(x) & 0x7fffffffu);
      sa += fabs(x);
      nz += x != 0.0;  // NaN counts, as before
    }
#pragma unroll
    for (int off = CW; off < 32; off *= 2) {
      hm = max(hm, __shfl_xor_sync(0xffffffffu, hm, off));
      sa += __shfl_xor_sync(0xffffffffu, sa, off);
      nz += __shfl_xor_sync(0xffffffffu, nz, off);
    }
    if (tid % 32 < CW) {
      r.rhi()[(tid / 32) * CW + jl] = hm;
      r.rsum[(tid / 32) * CW + jl] = sa;
      r.rnz[(tid / 32) * CW + jl] = nz;
    }
    if (phi && tid < kFieldChains * CW)  // chain p = tid / CW of column tid % CW
      for (int m = part; m < M; m += kFieldChains) facc = __fma_rn(__ldg(w + m), blk[m * CW + jl], facc);
  }
  sync();
  if (tid < CW) {
    double sum = 0.0;
    unsigned hm = 0u;
    int nnz = 0;
#pragma unroll
    for (int q = 0; q < NT / 32; ++q) {
      hm = max(hm, r.rhi()[q * CW + tid]);
      sum += r.rsum[q * CW + tid];
      nnz += r.rnz[q * CW + tid];
    }
    const bool bad = hm >= 0x7ff00000u;  // an Inf or NaN in the column
    int e = 0;  // scale_exp(max|x|): E - 1022 for a normal maximum with exponent field E
    if (!bad && hm >= 0x00100000u) {
      e = (int)(hm >> 20) - 1022;
    } else if (!bad && nnz > 0) {  // subnormal entries only: the exact maximum
      double v = 0.0;
      for (int m = 0; m < Kp; ++m) v = fmax(v, fabs(blk[m * CW + tid]));
      e = scale_exp(v);
    }
    r.sexp[tid] = e;
    // beta rounded up (the fp64 sum of <= 2^13 terms is within 2^-40 of exact)
    const float beta = __double2float_ru(__dmul_ru(ldexp(sum, -e), 1.0 + 0x1p-40));
    r.cstat[tid] = ColStat{bad ? kNonFinite : e, beta, nnz, 0};
    r.cdsum[tid] = 0;
  }
  sync();
  if (phi && tid < kFieldChains * CW) r.red[tid] = facc;  // maxima consumed: the buffer holds the chains
  const int chunks = 2 * nks;
  for (int item = tid; item < chunks * CW; item += NT) {
    const int ch = item / CW, jc = item - ch * CW;
    const int64_t j = j0 + jc;
    if (j >= N) continue;
    const int ks = ch >> 1, c = ch & 1;
    uint4 wd[S];
    const Scale sc = make_scale(r.sexp[jc]);
    auto get = [&](int b) { return blk[(ch * 16 + b) * CW + jc]; };
    int ds = 0;
    slice16(sc, get, wd, ds);
    atomicAdd(&r.cdsum[jc], ds);
    const int cb = (int)(j / BJ), jr = (int)(j - (int64_t)cb * BJ);
    int8_t* o = out + ((((int64_t)tt * ncb + cb) * nks + ks) * SB) * HB + c * (HB / 2) + jr * 16;
#pragma unroll
    for (int s = 0; s < S; ++s) *reinterpret_cast<uint4*>(o + s * HB) = wd[s];
    *reinterpret_cast<uint4*>(o + S * HB) = mag16(sc, get);
  }
  sync();
  after_slice();
  if (tid < CW && j0 + tid < N) {
    ColStat cs = r.cstat[tid];
    cs.dsum = r.cdsum[tid];
    bexp[(int64_t)tt * ncb * BJ + j0 + tid] = cs;
    if (phi) {
      double sum = r.red[tid];
#pragma unroll
      for (int q = 1; q < kFieldChains; ++q) sum = __dadd_rn(sum, r.red[q * CW + tid]);
      phi[(int64_t)t * N + j0 + tid] = sum;
    }
  }
}

struct NamedSync {
  int id, n;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
};
struct NoAfter {
  __device__ __forceinline__ void operator()() const {}
};

template <int CW>
__global__ void __launch_bounds__(SB_THREADS) slice_b(const double* __restrict__ H, int T, int64_t N, int M, int t0,
                                                     int ncb, int nks, int8_t* __restrict__ out,
                                                     ColStat* __restrict__ bexp, const double* __restrict__ w,
                                                     double* __restrict__ phi) {
  extern __shared__ __align__(16) double blk[];  // [Kp][CW]
  __shared__ SbRed<CW> red;
  const int tt = blockIdx.y, t = t0 + tt;
  const int64_t j0 = (int64_t)blockIdx.x * CW;
  const int Kp = nks * BK;
  const int64_t ld = (int64_t)T * N;
  const double* src = H + (int64_t)t * N + j0;
  const NamedSync sync{1, SB_THREADS};
  // stage: rows m < M by 16-byte copies (N even, j0 even), rows >= M and columns >= N zero
  // (CW / 2 divides the block: thread e always copies pair e % (CW / 2), rows
  // e / (CW / 2) + k * RS -- a pointer walk, no per-copy index math)
  {
    constexpr int RS = SB_THREADS / (CW / 2);
    const int pr = threadIdx.x % (CW / 2);
    const bool col_ok = j0 + 2 * pr < N;
    double2* dst = reinterpret_cast<double2*>(blk + (threadIdx.x / (CW / 2)) * CW) + pr;
    const double* g = src + (int64_t)(threadIdx.x / (CW / 2)) * ld + 2 * pr;
    for (int m = threadIdx.x / (CW / 2); m < Kp; m += RS, dst += RS * (CW / 2), g += RS * ld) {
      if (m < M && col_ok) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
      } else {
        *dst = make_double2(0.0, 0.0);
      }
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  sync();
  slice_block<CW, SB_THREADS>(blk, threadIdx.x, red, sync, NoAfter{}, N, M, t, tt, j0, ncb, nks, out, bexp, w, phi);
}

// A slices for thetas [t0, t0 + gridDim.y): CTA = 64 rows, 256 threads (4 per
// row for the scale, then one (row, 16-wide K chunk) item per thread).
// Stage layout per (theta, ib, ks): [c][slice t][row i % 64][16 bytes], i.e. the
// six slices stacked along N, so one MMA can take any run of consecutive slices
// as a single N = 64 * run operand (K-chunk stride 6 KB).
// CTA-pair (cta_group::2) A-operand stage of one (theta, ib, ks): each CTA of
// the pair holds half of every MMA's N rows, so its 14336 bytes are 7 regions
// ([c][rows][16 B] each) that the pair MMAs below take whole:
//   P0 128 rows  CTA0: A0, A1      CTA1: A2, A3      (runs s=0,1,2: t = 0..3)
//   P1  64       A4                A5                (s=0: t = 4, 5)
//   P2  64       A0                A1                (s=4: t = 0, 1)
//   P3  32       A4 rows 0..31     A4 rows 32..63    (s=1: t = 4)
//   P4  96       A0, A1[0:32)      A1[32:64), A2     (s=3: t = 0..2)
//   P5  32       A0 rows 0..31     A0 rows 32..63    (s=5: t = 0)
//   P6  32       A6 (magnitude) halves               (certificate)
constexpr int PAIR_A = 448 * 32;  // bytes per CTA per K step
__device__ __forceinline__ void put_pair(int8_t* base, int c, int t, int i, uint4 w) {
  auto put = [&](int cta, int roff, int rows, int r) {
    *reinterpret_cast<uint4*>(base + cta * PAIR_A + roff * 32 + c * rows * 16 + r * 16) = w;
  };
  const bool lo = i < 32;
  switch (t) {
    case 0:
      put(0, 0, 128, i), put(0, 192, 64, i), put(0, 288, 96, i), put(lo ? 0 : 1, 384, 32, i & 31);
      break;
    case 1:
      put(0, 0, 128, 64 + i), put(1, 192, 64, i);
      if (lo) put(0, 288, 96, 64 + i); else put(1, 288, 96, i - 32);
      break;
    case 2: put(1, 0, 128, i), put(1, 288, 96, 32 + i); break;
    case 3: put(1, 0, 128, 64 + i); break;
    case 4: put(0, 128, 64, i), put(lo ? 0 : 1, 256, 32, i & 31); break;
    case 5: put(1, 128, 64, i); break;
    default: put(lo ? 0 : 1, 416, 32, i & 31); break;
  }
}

template <bool PAIR>
__global__ void __launch_bounds__(256) slice_a(const double* __restrict__ A, int M, int t0, int nib, int nks,
                                               int8_t* __restrict__ out, double* __restrict__ ascale,
                                               RowStat* __restrict__ rstat) {
  __shared__ Scale sc[BI];
  __shared__ int rdsum[BI];
  __shared__ RowStat rst[BI];
  const int ib = blockIdx.x, tt = blockIdx.y;
  const double* rows = A + ((int64_t)(t0 + tt) * M + ib * BI) * M;
  {
    const int il = threadIdx.x >> 2, part = threadIdx.x & 3;
    const int i = ib * BI + il;
    double mx = 0.0, sa = 0.0;
    int nz = 0;
    bool bad = false;
    if (i < M)
      for (int m = part; m < M; m += 4) {
        const double x = rows[(int64_t)il * M + m];
        bad |= !isfinite(x);
        mx = fmax(mx, fabs(x));
        sa += fabs(x);
        nz += x != 0.0;
      }
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    sa += __shfl_xor_sync(0xffffffffu, sa, 1);
    sa += __shfl_xor_sync(0xffffffffu, sa, 2);
    nz += __shfl_xor_sync(0xffffffffu, nz, 1);
    nz += __shfl_xor_sync(0xffffffffu, nz, 2);
    bad = (__ballot_sync(0xffffffffu, bad) >> (threadIdx.x & 28)) & 0xfu;  // the row's 4 lanes
    if (part == 0) {
      const int e = bad ? 0 : scale_exp(mx);
      sc[il] = make_scale(e);
      // a non-finite row of A makes its output row NaN (as a GEMM would propagate it)
      ascale[(int64_t)tt * nib * BI + i] = bad ? __longlong_as_double(0x7ff8000000000000ll) : pow2(e);
      rst[il] = RowStat{__double2float_ru(__dmul_ru(ldexp(sa, -e), 1.0 + 0x1p-40)), nz, 0, 0};
      rdsum[il] = 0;
    }
  }
  __syncthreads();
  const int chunks = 2 * nks;
  for (int item = threadIdx.x; item < chunks * BI; item += blockDim.x) {
    const int ch = item / BI, il = item - ch * BI;
    const int ks = ch >> 1, c = ch & 1;
    const bool valid = ib * BI + il < M;
    const double* r = rows + (int64_t)il * M;
    uint4 w[S];
    auto get = [&](int b) {
      const int m = ch * 16 + b;
      return (valid && m < M) ? r[m] : 0.0;
    };
    int ds = 0;
    slice16(sc[il], get, w, ds);
    atomicAdd(&rdsum[il], ds);
    const uint4 mw = mag16(sc[il], get);
    if constexpr (PAIR) {
      int8_t* base = out + (((int64_t)tt * nib + ib) * nks + ks) * 2 * PAIR_A;
#pragma unroll
      for (int s = 0; s < S; ++s) put_pair(base, c, s, il, w[s]);
      put_pair(base, c, S, il, mw);
    } else {
      int8_t* o = out + ((((int64_t)tt * nib + ib) * nks + ks) * SB) * AB + c * (SB * AB / 2) + il * 16;
#pragma unroll
      for (int s = 0; s < S; ++s) *reinterpret_cast<uint4*>(o + s * (AB / 2)) = w[s];
      *reinterpret_cast<uint4*>(o + S * (AB / 2)) = mw;
    }
  }
  __syncthreads();
  if (threadIdx.x < BI) {
    RowStat r = rst[threadIdx.x];
    r.dsum = rdsum[threadIdx.x];
    rstat[(int64_t)tt * nib * BI + ib * BI + threadIdx.x] = r;
  }
}

// --------------------------------------------------------------- tcgen05 helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// CTA pair: a 2D tensor copy into this CTA's shared memory whose bytes complete on
// the LEADER's barrier (the peer bit of the shared::cluster address cleared) --
// the .cta_group::2 form, which lets the barrier live in the other CTA of the pair
// (the plain bulk copy needs it in the destination CTA)
__device__ __forceinline__ void tma_load_2sm(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(b))
               : "memory");
}
// K-major, no swizzle: core matrices of 8 rows x 16 bytes; rows at 16 B, K chunks at lbo
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_n(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BJ >> 4) << 24);
}
// (B slice s, first A slice t0, run length nt): all pairs s + t <= 5, nt * 64 <= 256
constexpr int kRuns = 8;
__device__ constexpr int kRun[kRuns][3] = {{0, 0, 4}, {0, 4, 2}, {1, 0, 3}, {1, 3, 2},
                                           {2, 0, 4}, {3, 0, 3}, {4, 0, 2}, {5, 0, 1}};
__device__ __forceinline__ void mma_i8n(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}



// ------------------------------------------------------ pipelined B slicing
// slice_b with the DRAM stream decoupled from the compute: one CTA per SM, a
// producer warp streams the K x 16 column blocks of successive work items (theta,
// column block) into a 3-stage shared-memory ring with 2D tensor copies (rows
// >= M zero-filled by the copy engine), and two groups of 8 consumer warps take
// alternate items (each group its own named barrier and reduction scratch), so
// the next blocks are in flight while both groups reduce and slice.  Same code
// per block (slice_block, 256 threads) -> the same bits as slice_b.
constexpr int SBP_STAGES = 3, SBP_GROUP = 256, SBP_THREADS = 32 + 2 * SBP_GROUP;
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
template <int CW>
__global__ void __launch_bounds__(SBP_THREADS, 1)
    slice_bp(const __grid_constant__ CUtensorMap hmap, int64_t N, int M, int t0, int ng, int ncb, int nks, int nbox,
             int box_rows, int8_t* __restrict__ out, ColStat* __restrict__ bexp, const double* __restrict__ w,
             double* __restrict__ phi) {
  extern __shared__ __align__(1024) uint8_t sbp_raw[];
  double* stages = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sbp_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[2 * SBP_STAGES], empty[SBP_STAGES];
  __shared__ SbRed<CW> red[2];
  const int64_t nblk = cdiv(N, CW);
  const int64_t items = (int64_t)ng * nblk;
  const int srows = nbox * box_rows;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * SBP_STAGES; ++i) mbar_init(&full[i], 1);
    for (int i = 0; i < SBP_STAGES; ++i) mbar_init(&empty[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // producer
    if (threadIdx.x == 0) {
      int64_t k = 0;
      for (int64_t item = blockIdx.x; item < items; item += gridDim.x, ++k) {
        const int st = (int)(k % SBP_STAGES);
        if (k >= SBP_STAGES) mbar_wait(&empty[st], (unsigned)((k / SBP_STAGES - 1) & 1));
        uint64_t* f = &full[k % (2 * SBP_STAGES)];
        mbar_expect_tx(f, (unsigned)(srows * CW * sizeof(double)));
        const int tt = (int)(item / nblk);
        const int c0 = (int)((int64_t)(t0 + tt) * N + (item - (int64_t)tt * nblk) * CW);
        double* dst = stages + (size_t)st * srows * CW;
        for (int b = 0; b < nbox; ++b) tma_load_2d(dst + (size_t)b * box_rows * CW, &hmap, c0, b * box_rows, f);
      }
    }
    return;
  }
  // consumers: group g takes the items k = g, g + 2, ... of this CTA's sequence;
  // full[k % 6] is used by one group only, every 6 items (no parity aliasing)
  const int g = (threadIdx.x - 32) / SBP_GROUP, tid = (threadIdx.x - 32) % SBP_GROUP;
  const NamedSync sync{1 + g, SBP_GROUP};
  int64_t k = g;
  for (int64_t item = blockIdx.x + (int64_t)g * gridDim.x; item < items; item += 2 * (int64_t)gridDim.x, k += 2) {
    const int st = (int)(k % SBP_STAGES);
    mbar_wait(&full[k % (2 * SBP_STAGES)], (unsigned)((k / (2 * SBP_STAGES)) & 1));
    const int tt = (int)(item / nblk);
    const int64_t j0 = (item - (int64_t)tt * nblk) * CW;
    uint64_t* e = &empty[st];
    auto release = [&]() {
      if (tid == 0) mbar_arrive(e);
    };
    slice_block<CW, SBP_GROUP>(stages + (size_t)st * srows * CW, tid, red[g], sync, release, N, M, t0 + tt, tt, j0,
                               ncb, nks, out, bexp, w, phi);
    sync();  // red[g] is reused by the group's next item
  }
}

// exact v * 2^(E - 52) for |v| < 2^51 without the (slow) I2F.F64.S64 conversion: v added to the mantissa of 1.5 2^E (whose ulp
// is 2^(E-52)) as raw bits, minus 1.5 2^E -- the conversion and the power-of-two
// scaling in one DSUB (hi 2^-16: E = 36; lo 2^-40: E = 12)
template <int E>
__device__ __forceinline__ double exact_scaled(long long v) {
  constexpr long long kBits = ((long long)(E + 1023) << 52) | (1ll << 51);
  return __dsub_rn(__longlong_as_double(v + kBits), __longlong_as_double(kBits));
}

// --------------------------------------------------------------- GEMM

struct GemmArgs {
#ifdef GK_I8_STATS
  long long* stats;  // per CTA: MMA thread [wait full, wait tempty, total], epilogue warp 2 [wait tfull, drain, store]
#endif
  const int8_t* bsl;
  const int8_t* asl;
  const ColStat* bexp;
  const double* ascale;  // 2^f_i per row of A
  const RowStat* rstat;
  double* out;
  int64_t N;        // columns (reals) of B / C
  int T, t0, M;     // thetas, first theta of the group, n_vel
  int ncb, nib, nks;
  int64_t tiles;
  unsigned* flags;  // per (theta, cb, ib) of all T thetas: tile failed its certificate
  unsigned* list;   // the failed tiles, for the fp64 recompute (fix_tiles)
  unsigned* count;
};

// CTA-pair MMA pieces: the leader issues M = 256 (2 x 128 columns of B) MMAs;
// its commits arrive on the same barrier in both CTAs (multicast)
__host__ __device__ constexpr uint32_t idesc_pair(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)((2 * BJ) >> 4) << 24);
}
__device__ __forceinline__ void mma_i8_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* b) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(b)),
      "h"((unsigned short)3)
      : "memory");
}
// (B slice, put_pair region row offset, rows per CTA, first accumulator,
//  1 = accumulates from ks = 0 on / 0 = its accumulators start at ks = 0)
constexpr int kPairRuns = 9;
__device__ constexpr int kPairRun[kPairRuns][5] = {{0, 0, 128, 0, 0},   {0, 128, 64, 4, 0}, {1, 0, 128, 1, 1},
                                                  {1, 256, 32, 5, 1},  {2, 0, 128, 2, 1}, {3, 288, 96, 3, 1},
                                                  {4, 192, 64, 4, 1},  {5, 384, 32, 5, 1}, {6, 416, 32, 6, 0}};

// PAIR: a CTA pair (cluster of 2, tcgen05 cta_group::2) computes a 256-column x
// 64-row tile: each CTA loads its own 128 columns of B (the UMMA M side) and its
// half of every MMA's stacked A rows (the N side, put_pair's regions), and the
// leader CTA issues M = 256 MMAs that read both CTAs' shared memory -- per SM the
// N-side operand reads and fills halve (shared memory is what bounds the 1-CTA
// kernel).  Both CTAs' stage copies are cta_group::2 tensor copies completing on
// the leader's full barrier (tma_load_2sm), the leader's commits arrive on both
// CTAs' empty barriers (multicast), both CTAs' epilogue warps release the
// accumulators on the leader's tempty.
template <bool PAIR>
__global__ void __launch_bounds__(THREADS, 1) ozaki_gemm(const GemmArgs a, const __grid_constant__ CUtensorMap tmb,
                                                          const __grid_constant__ CUtensorMap tma) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull, tempty;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned rank = 0;
  if constexpr (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  const unsigned cid = PAIR ? blockIdx.x >> 1 : blockIdx.x, ncl = PAIR ? gridDim.x >> 1 : gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull, 1);
    mbar_init(&tempty, PAIR ? 2 * EPI_WARPS : EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  tc_fence_before();
  if constexpr (PAIR) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tm = tslot;
  const int nks = a.nks;
  // (theta, column block, row block) of a tile; the pair's CTAs take column blocks 2 cbp + rank
  auto decode = [&](int64_t tile, int& tt, int& cb, int& ib) {
    ib = (int)(tile % a.nib);
    const int64_t rest = tile / a.nib;
    const int ncbt = PAIR ? (a.ncb + 1) / 2 : a.ncb;
    cb = (int)(rest % ncbt);
    tt = (int)(rest / ncbt);
    if (PAIR) cb = 2 * cb + (int)rank;
  };

  if (warp == 0) {
    if (lane == 0) {  // producer
      int st = 0;
      unsigned ph = 0;
      for (int64_t tile = cid; tile < a.tiles; tile += ncl) {
        int tt, cb, ib;
        decode(tile, tt, cb, ib);
        // the pair's odd column block past the end (odd ncb) loads block ncb - 1
        // again; its epilogue stores nothing (columns >= N)
        const int cbl = cb < a.ncb ? cb : a.ncb - 1;
        const int8_t* bsrc = a.bsl + ((int64_t)tt * a.ncb + cbl) * nks * (SB * HB);
        const int8_t* asrc = PAIR ? a.asl + (((int64_t)tt * a.nib + ib) * nks * 2 + rank) * PAIR_A
                                  : a.asl + ((int64_t)tt * a.nib + ib) * nks * (SB * AB);
        // PAIR: tensor-map rows of 256 bytes; both CTAs' copies complete on the
        // leader's full barrier, which expects the pair's bytes
        const int brow = (int)(((int64_t)tt * a.ncb + cbl) * nks * (SB * HB / 256));
        const int arow = (int)((((int64_t)tt * a.nib + ib) * nks * 2 + rank) * (PAIR_A / 256));
        for (int ks = 0; ks < nks; ++ks) {
          mbar_wait(&empty[st], ph ^ 1);
          uint8_t* dst = smem + st * STAGE;
          if constexpr (PAIR) {
            if (rank == 0) mbar_expect_tx(&full[st], 2 * STAGE);
            tma_load_2sm(dst, &tmb, 0, brow + ks * (SB * HB / 256), &full[st]);
            tma_load_2sm(dst + SB * HB, &tma, 0, arow + ks * (2 * PAIR_A / 256), &full[st]);
          } else {
            mbar_expect_tx(&full[st], STAGE);
            bulk_g2s(dst, bsrc + (int64_t)ks * SB * HB, SB * HB, &full[st]);
            bulk_g2s(dst + SB * HB, asrc + (int64_t)ks * SB * AB, SB * AB, &full[st]);
          }
          if (++st == STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (PAIR && rank != 0) {
      // the peer issues no MMAs: the leader's MMAs read both CTAs' shared memory
    } else if (lane == 0) {  // MMA issuer
      int st = 0;
      unsigned ph = 0, tph = 0;
#ifdef GK_I8_STATS
      long long wf = 0, we = 0, t_begin = clock64();
#define GK_T0 long long c0_ = clock64();
#define GK_T1(acc) acc += clock64() - c0_;
#else
#define GK_T0
#define GK_T1(acc)
#endif
      for (int64_t tile = cid; tile < a.tiles; tile += ncl) {
        { GK_T0 mbar_wait(&tempty, tph ^ 1); GK_T1(we) }
        tc_fence_after();
        for (int ks = 0; ks < nks; ++ks) {
          { GK_T0 mbar_wait(&full[st], ph); GK_T1(wf) }
          tc_fence_after();
          const uint32_t bs = smem_u32(smem + st * STAGE), as = bs + SB * HB;
          if constexpr (PAIR) {
            // (B slice, region row offset, region rows, first accumulator); N = 2 x rows
#pragma unroll
            for (int r = 0; r < kPairRuns; ++r) {
              const int sb = kPairRun[r][0], roff = kPairRun[r][1], rows = kPairRun[r][2], acc = kPairRun[r][3];
              mma_i8_pair(tm + (uint32_t)(acc * BI), sdesc(bs + sb * HB, HB / 2), sdesc(as + roff * 32, rows * 16),
                          idesc_pair(2 * rows), (ks > 0 || kPairRun[r][4]) ? 1u : 0u);
            }
            tc_commit_pair(&empty[st]);
            if (++st == STAGES) {
              st = 0;
              ph ^= 1;
            }
            continue;
          }
          // B slice s against the stacked A slices t0 .. t0 + nt - 1 in one MMA of
          // N = 64 nt: writes acc_{s+t0} .. acc_{s+t0+nt-1} (adjacent in TMEM).
          // Every MMA costs >= ~48 clocks (measured), so N = 64 MMAs ran at 2/3 of
          // the peak; 8 MMAs of N = 64..256 per K step run at ~0.98.
#pragma unroll
          for (int r = 0; r < kRuns; ++r) {
            const int sb = kRun[r][0], t0r = kRun[r][1], nt = kRun[r][2];
            mma_i8n(tm + (uint32_t)((sb + t0r) * BI), sdesc(bs + sb * HB, HB / 2),
                    sdesc(as + t0r * (AB / 2), SB * AB / 2), idesc_n(nt * BI), (ks > 0 || sb > 0) ? 1u : 0u);
          }
          // the certificate's magnitude product Q = |A|_q |B|_q into accumulator S
          mma_i8n(tm + (uint32_t)(S * BI), sdesc(bs + S * HB, HB / 2), sdesc(as + S * (AB / 2), SB * AB / 2),
                  idesc_n(BI), ks > 0 ? 1u : 0u);
          tc_commit(&empty[st]);
          if (++st == STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
        if (PAIR) tc_commit_pair(&tfull); else tc_commit(&tfull);
        tph ^= 1;
      }
#ifdef GK_I8_STATS
      a.stats[6 * blockIdx.x] = wf;
      a.stats[6 * blockIdx.x + 1] = we;
      a.stats[6 * blockIdx.x + 2] = clock64() - t_begin;
#endif
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 (columns j of the tile)
    // and RPW of the 64 accumulator columns (rows i); it first folds the six
    // accumulators into fp64 sums held in registers and releases TMEM, so the
    // scale-and-store tail overlaps the next tile's MMAs.
    const int q = warp & 3, part = (warp - 2) >> 2;
    const int jl = q * 32 + lane;
    unsigned tph = 0;
#ifdef GK_I8_STATS
    long long e_wait = 0, e_drain = 0, e_store = 0, e0 = 0;
#endif
    uint32_t tempty_at = smem_u32(&tempty);  // the leader's tempty (PAIR)
    if (PAIR) asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(tempty_at) : "r"(smem_u32(&tempty)));
    for (int64_t tile = cid; tile < a.tiles; tile += ncl) {
      int tt, cb, ib;
      decode(tile, tt, cb, ib);
      const int64_t j = (int64_t)cb * BJ + jl;
      const bool jv = j < a.N;
      double sum[RPW];
      float qm[RPW];  // the magnitude product Q of each row (exact int < 2^24 for K <= 1040, rounded down above)
      // Scales (before the wait: they depend only on the tile).  C = 2^(e_j - 12) 2^f_i sum.
      const ColStat cj = jv ? a.bexp[(int64_t)tt * a.ncb * BJ + j] : ColStat{0, 0.f, 0, 0};  // dsum 0: passes
      const int ej = cj.e;
      const double sj = ej == kNonFinite ? __longlong_as_double(0x7ff8000000000000ll) : pow2(ej - 12);
      const int i0 = ib * BI + part * RPW;
      const bool lrow = lane < RPW;  // lanes holding a row of the warp's block
      const double si = lrow ? a.ascale[(int64_t)tt * a.nib * BI + i0 + lane] : 1.0;  // row i0 + lane
      const RowStat ri = lrow ? a.rstat[(int64_t)tt * a.nib * BI + i0 + lane] : RowStat{0.f, 0, 0, 0};
      // Fast scaling: with E = f_i + e_j - 12 in [-982, 995] for every (row, column)
      // of the warp's block, every nonzero sum (|sum| in [2^-40, 2^27]) times 2^E is a
      // normal double, so the two exact power-of-two multiplies are one exponent
      // addition (bit-identical; the epilogue's FP64 work is throttled next to the
      // MMAs).  Otherwise (non-finite or extreme scales) the two multiplies.
      const long long sib = __double_as_longlong(si);
      const int sfield = (int)((sib >> 52) & 0x7ff);
      const bool rowv = lrow && i0 + lane < a.M;
      const int fi = (rowv && sib > 0 && sfield >= 1 && sfield <= 2046) ? sfield - 1023 : 0;
      bool fast_ok = !rowv || (sib > 0 && sfield >= 1 && sfield <= 2046);
      int fmin = fi, fmax = fi;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        fmin = min(fmin, __shfl_xor_sync(0xffffffffu, fmin, o));
        fmax = max(fmax, __shfl_xor_sync(0xffffffffu, fmax, o));
      }
      const int ejs = ej - 12;
      if (jv) fast_ok = fast_ok && ej != kNonFinite && fmin + ejs >= -982 && fmax + ejs <= 995;
      const bool fast = __all_sync(0xffffffffu, fast_ok);
#ifdef GK_I8_STATS
      e0 = clock64();
#endif
      mbar_wait(&tfull, tph);
#ifdef GK_I8_STATS
      { const long long c = clock64(); e_wait += c - e0; e0 = c; }
#endif
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < RPW / 16; ++c) {
        uint32_t v[SB][16];
#pragma unroll
        for (int d = 0; d < SB; ++d)
          tmem_ld16(tm + ((uint32_t)(q * 32) << 16) + d * BI + part * RPW + c * 16, v[d]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int k = 0; k < 16; ++k) qm[c * 16 + k] = __uint2float_rd(v[S][k]);
        // sum_d acc_d 2^(-8 d) = 2^-16 hi + 2^-40 lo with hi = a0 2^16 + a1 2^8 + a2,
        // lo = a3 2^16 + a4 2^8 + a5: exact in int64 (|a_d| < 2^26), so the FP64
        // pipe (the drain's bottleneck: TMEM stays locked until it ends) does two
        // exact scaled conversions and one add per output (= one rounding of
        // hi 2^-16 + lo 2^-40) instead of six conversions and five adds.
        static_assert(S == 6, "hi/lo split assumes six slices");
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const long long hi = ((long long)(int)v[0][k] << 16) + ((long long)(int)v[1][k] << 8) + (int)v[2][k];
          const long long lo = ((long long)(int)v[3][k] << 16) + ((long long)(int)v[4][k] << 8) + (int)v[5][k];
          sum[c * 16 + k] = __dadd_rn(exact_scaled<36>(hi), exact_scaled<12>(lo));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(tempty_at) : "memory");
        else
          mbar_arrive(&tempty);
      }
      tph ^= 1;
#ifdef GK_I8_STATS
      { const long long c = clock64(); e_drain += c - e0; e0 = c; }
#endif
      // Certificate (componentwise, against DGEMM's sum_k |A_ik| |B_kj| = P_ij):
      // |C_ij - (A B)_ij| <= 2^(e+f-47) (min(alpha_i, m_j) + min(beta_j, n_i))
      //                    + 0.502 2^(e+f-52) min(sigma_j, rho_i) + 2^-53 |C|
      // [B rounding (where B_kj != 0: m_j nonzeros in the column), A rounding
      // (where A_ik != 0: n_i in the row), and the dropped slice pairs s + t >= 6:
      // grouped by s, sum_k |b_s| 256^(5-s) |tail of A below digit 5 - s| with the
      // balanced tail < 0.502 256^s, i.e. the column's digit-magnitude sum sigma_j
      // (or, grouped by t, the row's rho_i)], and P_ij >= 2^(e+f-14) Q_ij, so the
      // tile's result is within 2^-37 P_ij of the exact product wherever
      //   Q_ij >= 16.01 (min(alpha_i, m_j) + min(beta_j, n_i)) + 0.2511 min(sigma_j, rho_i)
      // (float arithmetic rounded towards failing; exact zero rows / columns pass).
      // Tiles with an element that cannot be certified are recomputed in fp64
      // (fix_tiles).  Non-finite rows / columns propagate NaN and are exempt.
      const float arow = ri.alpha, nrow = (float)ri.nnz, drow = (float)ri.dsum;
      const float mcol = (float)cj.nnz, dcol = (float)cj.dsum;
      const bool row_ok = isfinite(si) && rowv;
      bool fail = false;
      double* ocol = a.out + (int64_t)(a.t0 + tt) * a.N + j;
      const int64_t ld = (int64_t)a.T * a.N;
      const int rows = min(RPW, a.M - i0);
      // 16-byte stores: lanes 2m, 2m+1 swap one value per row pair (k, k+1), so the
      // even lane writes row k at columns (j, j+1) and the odd lane row k+1 at
      // (j-1, j): half the store requests of one 8-byte value per lane.
      const bool odd = lane & 1;
      double* pcol = ocol - (odd ? 1 : 0);
      const bool pv = (int64_t)cb * BJ + (jl & ~1) + 1 < a.N;  // both columns of the pair exist
#pragma unroll
      for (int k = 0; k < RPW; ++k) {
        const float ar = __shfl_sync(0xffffffffu, arow, k), nr = __shfl_sync(0xffffffffu, nrow, k);
        const float dr = __shfl_sync(0xffffffffu, drow, k);
        const bool ok_k = __shfl_sync(0xffffffffu, (int)row_ok, k) != 0;
        const float thr = __fmaf_ru(16.01f, __fadd_ru(fminf(ar, mcol), fminf(cj.beta, nr)),
                                    __fmul_ru(0.2511f, fminf(dr, dcol)));
        fail |= ok_k && qm[k] < thr;
      }
      fail = fail && jv && ej != kNonFinite;
      if (__any_sync(0xffffffffu, fail) && lane == 0) {
        const unsigned id = (unsigned)((((int64_t)(a.t0 + tt) * a.ncb + cb) * a.nib) + ib);
        if (atomicExch(a.flags + id, 1u) == 0u) a.list[atomicAdd(a.count, 1u)] = id;
      }
#pragma unroll
      for (int k = 0; k < RPW; k += 2) {
        double v0 = sum[k], v1 = sum[k + 1];
        if (fast) {  // exact power-of-two scaling as an exponent addition (zeros keep their sign)
          const long long e0s = (long long)(__shfl_sync(0xffffffffu, fi, k) + ejs) << 52;
          const long long e1s = (long long)(__shfl_sync(0xffffffffu, fi, k + 1) + ejs) << 52;
          if (v0 != 0.0) v0 = __longlong_as_double(__double_as_longlong(v0) + e0s);
          if (v1 != 0.0) v1 = __longlong_as_double(__double_as_longlong(v1) + e1s);
        } else {
          v0 = __dmul_rn(__dmul_rn(v0, sj), __shfl_sync(0xffffffffu, si, k));
          v1 = __dmul_rn(__dmul_rn(v1, sj), __shfl_sync(0xffffffffu, si, k + 1));
        }
        // even lane keeps v0 and receives its neighbour's v0; odd lane keeps v1, receives v1
        const double got = __shfl_xor_sync(0xffffffffu, odd ? v0 : v1, 1);
        const double2 pair = odd ? make_double2(got, v1) : make_double2(v0, got);
        const int kr = k + (odd ? 1 : 0);
        if (pv && kr < rows) __stcs(reinterpret_cast<double2*>(pcol + (int64_t)(i0 + kr) * ld), pair);
      }
#ifdef GK_I8_STATS
      e_store += clock64() - e0;
#endif
    }
#ifdef GK_I8_STATS
    if (warp == 2 && lane == 0) {
      a.stats[6 * blockIdx.x + 3] = e_wait;
      a.stats[6 * blockIdx.x + 4] = e_drain;
      a.stats[6 * blockIdx.x + 5] = e_store;
    }
#endif
  }
  tc_fence_before();
  if constexpr (PAIR) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
  } else {
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
  }
}

// Peak probe: every SM issues back-to-back M128 N256 K32 int8 MMAs on resident
// shared-memory operands (the shape that is not operand-bandwidth bound).
constexpr int PROBE_REPS = 8192;
__global__ void __launch_bounds__(128, 1) i8_peak_kernel(int reps) {
  extern __shared__ __align__(1024) uint8_t psm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < (128 + 256) * BK / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(psm)[e] = make_uint4(0x01010101u, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t base = smem_u32(psm);
    const uint64_t da = sdesc(base, 128 * 16), db = sdesc(base + 128 * BK, 256 * 16);
    constexpr uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) |
                            ((uint32_t)(128 >> 4) << 24);
    for (int r = 0; r < reps; ++r)
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
          "l"(da), "l"(db), "r"(id), "r"((uint32_t)(r > 0))
          : "memory");
    tc_commit(&bar);
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tm));
}

// --------------------------------------------------------------- host

struct Workspace {
  void* ptr = nullptr;
  size_t bytes = 0;
};

static int sm_count() {
  int dev = 0, v = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}

// Thetas per group of the grouped collision (B slices made and consumed group by
// group): up to 4, as many as keep one group's B slices within ~4 GB (C5b ranks:
// 1.2 GB per theta -> 3).  GK_I8_THETA_GROUP overrides.
static int theta_group(size_t b_theta) {
  static const int env = [] {
    const char* e = getenv("GK_I8_THETA_GROUP");
    return e ? std::max(0, atoi(e)) : 0;
  }();
  if (env > 0) return env;
  return (int)std::max<size_t>(1, std::min<size_t>(4, (size_t)4000000000ull / std::max<size_t>(b_theta, 1)));
}

}  // namespace i8

// 0 auto (int8 slices when eligible), 1 fp64 DMMA always, 2 int8 whenever eligible
static int g_collision_mode = -1;

static int collision_mode() {
  if (g_collision_mode < 0) {
    const char* e = getenv("GK_COLLISION");
    g_collision_mode = !e ? 0 : (std::string(e) == "dmma" ? 1 : (std::string(e) == "int8" ? 2 : 0));
  }
  return g_collision_mode;
}

// Auto: int8 slices once the GEMM is big enough to amortise the slicing and the
// tile pipeline (M >= 64 and M^2 N T >= 2^30 multiply-adds: C2 linear and larger;
// measured C2 0.29 vs 0.66 ms on DMMA, C1 tiny 0.027 vs 0.013 ms).  T is the full
// theta count (not a range's), so every range call of a step takes the same path.
bool collision_use_i8(int64_t M, int64_t N, int64_t T) {
  const int mode = collision_mode();
  if (mode == 1) return false;
  if (M > 8192) return false;  // int32 accumulator bound
  if (mode == 2) return true;
  return M >= 64 && (double)M * (double)M * (double)N * (double)T >= 1073741824.0;
}

#ifdef GK_I8_STATS
static long long* i8_stats_buffer() {
  static long long* p = nullptr;
  if (!p) cudaMallocManaged(&p, sizeof(long long) * 6 * 1024);
  return p;
}
extern "C" long long* gk_i8_stats() { return i8_stats_buffer(); }
#endif

template <int CW>
static int launch_slice_b(const double* H, int T, int64_t N, int M, int g0, int ng, int ncb, int nks, int8_t* bsl,
                          i8::ColStat* bexp, const double* w, double* phi, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)nks * i8::BK * CW;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    GK_CUDA(cudaFuncSetAttribute(i8::slice_b<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  i8::slice_b<CW><<<dim3((unsigned)cdiv(N, CW), ng), i8::SB_THREADS, smem, st>>>(H, T, N, M, g0, ncb, nks, bsl,
                                                                                 bexp, w, phi);
  count_launch();
  return check_launch("gk_collision (int8 slices: B)");
}

namespace i8 {
struct Geometry {
  int ncb, nib, nks;
  size_t b_theta;  // B slice bytes per theta
  size_t e_theta;  // column exponent bytes per theta
  Geometry(int M, int64_t N)
      : ncb((int)cdiv(N, BJ)), nib((int)cdiv(M, BI)), nks((int)cdiv(M, BK)),
        b_theta((size_t)ncb * nks * SB * HB), e_theta(sizeof(ColStat) * (size_t)ncb * BJ) {}
  // A slices of one theta (the CTA-pair layout holds every K step twice: 2 x 14 KB;
  // buffers are sized for it), and the per-row scale + certificate stats
  size_t a_theta(bool pair = true) const { return (size_t)nib * nks * (pair ? 2 * PAIR_A : SB * AB); }
  size_t arow_theta() const { return (sizeof(double) + sizeof(RowStat)) * (size_t)nib * BI; }  // RowStat: 16 B
};

// Certificate bookkeeping of a call (flags over all T thetas' tiles, the failed
// tile list, its length): cleared at the start of every gemms() call.
static int64_t fix_words(int M, int T, int64_t N) {
  const Geometry g(M, N);
  return 2 * (int64_t)T * g.ncb * g.nib + 1;
}
static int64_t fix_bytes(int M, int T, int64_t N) { return (fix_words(M, T, N) * 4 + 255) & ~int64_t(255); }

// fp64 recompute of the tiles whose int8 result could not be certified: C tile
// (64 rows of A x 128 columns of B of one theta) = A_t B_t with sequential-k FMAs
// (CUDA cores; such tiles are rare outside pathological data).  One CTA per tile,
// 256 threads x (4 rows x 8 columns); K staged in 32-wide chunks.
__device__ unsigned long long g_fixed_tiles = 0;  // tiles recomputed since load (gk_collision_fixups)
__global__ void __launch_bounds__(256) fix_tiles(const double* __restrict__ A, const double* __restrict__ H,
                                                 double* __restrict__ C, int M, int T, int64_t N, int ncb, int nib,
                                                 const unsigned* __restrict__ list, const unsigned* __restrict__ count) {
  constexpr int KC = 16;
  __shared__ double sa[BI][KC + 1];
  __shared__ double sb[KC][BJ + 1];
  const unsigned n = *count;
  if (blockIdx.x == 0 && threadIdx.x == 0 && n) atomicAdd(&g_fixed_tiles, (unsigned long long)n);
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;  // rows tr*4.., columns tc + 16 c
  for (unsigned idx = blockIdx.x; idx < n; idx += gridDim.x) {
    const unsigned id = list[idx];
    const int ib = (int)(id % nib);
    const unsigned rest = id / nib;
    const int cb = (int)(rest % ncb), t = (int)(rest / ncb);
    const int i0 = ib * BI;
    const int64_t j0 = (int64_t)cb * BJ;
    double acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;
    const double* At = A + (int64_t)t * M * M;
    for (int k0 = 0; k0 < M; k0 += KC) {
      __syncthreads();
      for (int e = threadIdx.x; e < BI * KC; e += 256) {
        const int r = e / KC, k = e % KC;
        sa[r][k] = (i0 + r < M && k0 + k < M) ? At[(int64_t)(i0 + r) * M + k0 + k] : 0.0;
      }
      for (int e = threadIdx.x; e < KC * BJ; e += 256) {
        const int k = e / BJ, c = e % BJ;
        sb[k][c] = (k0 + k < M && j0 + c < N) ? H[((int64_t)(k0 + k) * T + t) * N + j0 + c] : 0.0;
      }
      __syncthreads();
      for (int k = 0; k < KC; ++k) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const double av = sa[tr * 4 + r][k];
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[r][c] = __fma_rn(av, sb[k][tc + 16 * c], acc[r][c]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + tr * 4 + r;
      if (i >= M) continue;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int64_t j = j0 + tc + 16 * c;
        if (j < N) C[((int64_t)i * T + t) * N + j] = acc[r][c];
      }
    }
    __syncthreads();
  }
}

// B slices (+ column exponents) for thetas [t0, t1) into a buffer laid out for
// all thetas: [theta][cb][ks][s][tile] then [theta][column] exponents.
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder();
// Pipelined B slicing (slice_bp) for CW = 16 when three K x 16 blocks fit the
// shared memory of one CTA (M <= 576), with GK_SB_PIPE=1.  Not the default: same
// bits, but slower at sh03b (2.93-3.01 vs 2.74-2.75 ms) -- the pass is bound by
// the slicing instructions, and one CTA of 16 consumer warps issues fewer of them
// per clock than three 8-warp CTAs.
static bool sb_pipe() {
  static const bool v = [] {
    const char* e = getenv("GK_SB_PIPE");
    return e && e[0] == '1';
  }();
  return v;
}
static int launch_slice_bp(const double* H, int T, int64_t N, int M, int g0, int ng, int ncb, int nks, int8_t* bsl,
                           ColStat* bexp, const double* w, double* phi, cudaStream_t st, bool& done) {
  constexpr int CW = 16;
  done = false;
  const int Kp = nks * BK;
  const int nbox = (int)cdiv(Kp, 256);
  const int box_rows = BK * (int)cdiv(nks, nbox);
  const size_t smem = (size_t)SBP_STAGES * nbox * box_rows * CW * sizeof(double) + 1024;
  // the dynamic shared memory the kernel can have next to its static part
  static const int max_dyn = [] {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, slice_bp<CW>) != cudaSuccess) return 0;
    return optin - (int)fa.sharedSizeBytes;
  }();
  if (!sb_pipe() || (int64_t)smem > max_dyn) return GK_OK;
  const PFN_cuTensorMapEncodeTiled_v12000 enc = tmap_encoder();
  if (!enc || ((uintptr_t)H & 15)) return GK_OK;  // slice_b instead
  CUtensorMap map{};
  const cuuint64_t dims[2] = {(cuuint64_t)T * (cuuint64_t)N, (cuuint64_t)M};
  const cuuint64_t strides[1] = {(cuuint64_t)T * (cuuint64_t)N * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)CW, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(H), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return GK_OK;
  static std::atomic<unsigned long long> attr{0};  // the largest block this launcher admits
  if (first_on_device(attr))
    GK_CUDA(cudaFuncSetAttribute(slice_bp<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn));
  const int64_t items = (int64_t)ng * cdiv(N, CW);
  const int grid = (int)std::min<int64_t>(items, std::max(1, sm_count() - sm_reserve()));
  slice_bp<CW><<<grid, SBP_THREADS, smem, st>>>(map, N, M, g0, ng, ncb, nks, nbox, box_rows, bsl, bexp, w, phi);
  count_launch();
  done = true;
  return check_launch("gk_collision (int8 slices: B, pipelined)");
}

static int prepare_b(const double* H, int M, int T, int64_t N, int t0, int t1, int8_t* bsl, ColStat* bexp,
                     cudaStream_t st, const double* w = nullptr, double* phi = nullptr) {
  const Geometry g(M, N);
  const size_t kp = (size_t)g.nks * BK * sizeof(double);
  int8_t* b = bsl + (size_t)t0 * g.b_theta;
  ColStat* e = bexp + (size_t)t0 * g.ncb * BJ;
  const int ng = t1 - t0;
  // columns per CTA: the widest whose K x CW block stays <= 96 KB (2+ CTAs / SM)
#ifndef SB_MAXCW
#define SB_MAXCW 16
#endif
  if (SB_MAXCW >= 16 && kp * 16 <= 96 * 1024) {
    bool done = false;
    const int rc = launch_slice_bp(H, T, N, M, t0, ng, g.ncb, g.nks, b, e, w, phi, st, done);
    if (rc || done) return rc;
    return launch_slice_b<16>(H, T, N, M, t0, ng, g.ncb, g.nks, b, e, w, phi, st);
  }
  if (kp * 8 <= 96 * 1024) return launch_slice_b<8>(H, T, N, M, t0, ng, g.ncb, g.nks, b, e, w, phi, st);
  if (kp * 4 <= 96 * 1024) return launch_slice_b<4>(H, T, N, M, t0, ng, g.ncb, g.nks, b, e, w, phi, st);
  return launch_slice_b<2>(H, T, N, M, t0, ng, g.ncb, g.nks, b, e, w, phi, st);
}

static std::atomic<unsigned long long> g_attr_done{0};
static int gemm_setup() {
  if (first_on_device(g_attr_done)) {
    GK_CUDA(cudaFuncSetAttribute(ozaki_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    GK_CUDA(cudaFuncSetAttribute(ozaki_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  }
  return GK_OK;
}
// A 2D tensor map over `bytes` bytes at `base` viewed as rows of 256 bytes (uint8),
// box = `box_rows` rows: the CTA-pair GEMM's stage copies (tma_load_2sm).  The
// encoder comes from the driver through the runtime (no libcuda link).
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  return enc;
}
static int byte_rows_map(CUtensorMap* m, const void* base, size_t bytes, int box_rows) {
  const PFN_cuTensorMapEncodeTiled_v12000 enc = tmap_encoder();
  if (!enc) {
    gk::set_error("gk_collision: cuTensorMapEncodeTiled unavailable (CTA-pair GEMM)");
    return GK_ERR_CUDA;
  }
  if (((uintptr_t)base & 255) || (bytes & 255)) {
    gk::set_error("gk_collision: slice buffer not 256-byte aligned (CTA-pair GEMM)");
    return GK_ERR_ARG;
  }
  const cuuint64_t dims[2] = {256, (cuuint64_t)(bytes / 256)};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {256, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    gk::set_error("gk_collision: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return GK_ERR_CUDA;
  }
  return GK_OK;
}

// CTA-pair GEMM (tcgen05 cta_group::2) or one CTA per tile: GK_I8_PAIR=1 / 0
static bool use_pair() {
  static const bool v = [] {
    const char* e = getenv("GK_I8_PAIR");
    return e && e[0] == '1';
  }();
  return v;
}

// Scratch of the standalone collision calls (slices of a theta group) comes from a
// memory pool owned by this library, one per device, that keeps its memory between
// calls (no cudaMalloc in the steady state).  The process-wide default pool is left
// alone, so torch's caching allocator and other cudaMallocAsync users are not
// affected.  The step paths take all their scratch from the caller's workspace.
static cudaMemPool_t scratch_pool() {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  pools[dev] = pool;
  return pool;
}
static int scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  cudaMemPool_t pool = scratch_pool();
  if (!pool) {
    gk::set_error("gk_collision: could not create the scratch memory pool");
    return GK_ERR_CUDA;
  }
  GK_CUDA(cudaMallocFromPoolAsync(p, bytes, pool, st));
  return GK_OK;
}

// Which A-slice buffers hold the slices of which matrices (host-side registry):
// a caller's GK_STEP_REUSE_MATRICES promise is honoured only for a buffer that
// slice_a actually filled from the same matrices pointer and geometry -- e.g. a
// workspace whose earlier steps ran on the DMMA path was never filled.
struct ASliceTag {
  const double* A;
  int M, T;
  bool pair;               // CTA-pair stage layout
  std::vector<char> done;  // thetas whose slices the buffer holds
};
static std::mutex g_tag_mu;
static std::map<const void*, ASliceTag> g_atags;
static bool aslices_valid(const void* abuf, const double* A, int M, int T, int t0, int t1) {
  std::lock_guard<std::mutex> lock(g_tag_mu);
  auto it = g_atags.find(abuf);
  if (it == g_atags.end() || it->second.A != A || it->second.M != M || it->second.T != T ||
      it->second.pair != use_pair())
    return false;
  for (int t = t0; t < t1; ++t)
    if (!it->second.done[t]) return false;
  return true;
}
}  // namespace i8
// Forget the A-slice tags of buffers inside [base, base + bytes) outside
// [keep, keep + keep_bytes): a call that lays its workspace out differently
// (another collision mode, another step kind) may overwrite them.
void aslices_forget(const void* base, int64_t bytes, const void* keep, int64_t keep_bytes) {
  std::lock_guard<std::mutex> lock(i8::g_tag_mu);
  const char *lo = (const char*)base, *hi = lo + bytes;
  const char *klo = (const char*)keep, *khi = klo + (keep ? keep_bytes : 0);
  for (auto it = i8::g_atags.begin(); it != i8::g_atags.end();) {
    const char* p = (const char*)it->first;
    if (p >= lo && p < hi && !(p >= klo && p < khi))
      it = i8::g_atags.erase(it);
    else
      ++it;
  }
}
namespace i8 {
static void aslices_mark(const void* abuf, const double* A, int M, int T, int t0, int t1) {
  std::lock_guard<std::mutex> lock(g_tag_mu);
  ASliceTag& tag = g_atags[abuf];
  if (tag.A != A || tag.M != M || tag.T != T || tag.pair != use_pair() || (int)tag.done.size() != T)
    tag = ASliceTag{A, M, T, use_pair(), std::vector<char>(T, 0)};
  for (int t = t0; t < t1; ++t) tag.done[t] = 1;
}

// A slices for [t0, t1) and the GEMMs over thetas [t0, t1), theta groups of G,
// reading B slices laid out for all thetas (bsl/bexp as prepare_b writes them).
// `prep` non-null: slice B group by group first (into bsl at group-relative
// offsets, i.e. bsl holds only G thetas).
// `abuf` non-null: the A slices of all T thetas live there (aslice_bytes layout);
// `reuse_a` skips slicing them (a previous call filled abuf from the same A).
static int gemms(const double* A, int8_t* bsl, ColStat* bexp, bool group_relative, const double* H, double* C,
                 int M, int T, int64_t N, int t0, int t1, cudaStream_t st, void* abuf, bool reuse_a,
                 const double* w, double* phi, unsigned* fix) {
  int rc = gemm_setup();
  if (rc) return rc;
  const Geometry g(M, N);
  const int nt = t1 - t0;
  // B slices made group by group bound the scratch; presliced, one launch covers
  // every theta (C2: 8 launches of 288 tiles -> 1 of 2304, no per-launch tail)
  static const int pg = [] {  // GK_I8_PRESLICED_GROUP: thetas per launch when presliced (0 = all)
    const char* e = getenv("GK_I8_PRESLICED_GROUP");
    return e ? std::max(0, atoi(e)) : 0;
  }();
  const int G = group_relative ? std::min(theta_group(g.b_theta), nt) : (pg > 0 ? std::min(pg, nt) : nt);
  const bool pair = use_pair();
  const size_t a_theta = g.a_theta(pair);
  void* ws = nullptr;
  int8_t* asl;
  double* ascale;
  RowStat* rstat;
  if (abuf) {
    const size_t a_all = (size_t)T * g.a_theta();  // the buffer is laid out for the larger (pair) stride
    asl = (int8_t*)abuf + (size_t)t0 * a_theta;
    ascale = (double*)((int8_t*)abuf + a_all) + (size_t)t0 * g.nib * BI;
    rstat = (RowStat*)((double*)((int8_t*)abuf + a_all) + (size_t)T * g.nib * BI) + (size_t)t0 * g.nib * BI;
  } else {
    if ((rc = scratch_alloc(&ws, nt * (a_theta + g.arow_theta()), st))) return rc;
    asl = (int8_t*)ws;
    ascale = (double*)(asl + nt * a_theta);
    rstat = (RowStat*)(ascale + (size_t)nt * g.nib * BI);
  }
  // the reuse promise covers only a buffer slice_a filled from these matrices
  if (!(abuf && reuse_a && aslices_valid(abuf, A, M, T, t0, t1))) {
    if (pair)
      slice_a<true><<<dim3(g.nib, nt), 256, 0, st>>>(A, M, t0, g.nib, g.nks, asl, ascale, rstat);
    else
      slice_a<false><<<dim3(g.nib, nt), 256, 0, st>>>(A, M, t0, g.nib, g.nks, asl, ascale, rstat);
    count_launch();
    rc = check_launch("gk_collision (int8 slices: A)");
    if (abuf && rc == GK_OK) aslices_mark(abuf, A, M, T, t0, t1);
  }
  // certificate bookkeeping: flags of every tile of the T thetas, then the count
  const int64_t ntiles_all = (int64_t)T * g.ncb * g.nib;
  unsigned* flags = fix;
  unsigned* list = fix + ntiles_all;
  unsigned* count = list + ntiles_all;
  if (rc == GK_OK) {
    GK_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned) * ntiles_all, st));
    GK_CUDA(cudaMemsetAsync(count, 0, sizeof(unsigned), st));
  }
  for (int g0 = t0; g0 < t1 && rc == GK_OK; g0 += G) {
    const int ng = std::min(G, t1 - g0);
    const int8_t* b = bsl;
    const ColStat* e = bexp;
    if (group_relative) {
      if ((rc = prepare_b(H, M, T, N, g0, g0 + ng, bsl - (size_t)g0 * g.b_theta, bexp - (size_t)g0 * g.ncb * BJ,
                          st, w, phi)))
        break;
    } else {
      b += (size_t)g0 * g.b_theta;
      e += (size_t)g0 * g.ncb * BJ;
    }
    GemmArgs ga{
#ifdef GK_I8_STATS
        i8_stats_buffer(),
#endif
        b, asl + (size_t)(g0 - t0) * a_theta, e, ascale + (size_t)(g0 - t0) * g.nib * BI,
        rstat + (size_t)(g0 - t0) * g.nib * BI,
        C, N, T, g0, M, g.ncb, g.nib, g.nks, (int64_t)ng * (pair ? (g.ncb + 1) / 2 : g.ncb) * g.nib, flags, list,
        count};
    const int sms = std::max(2, sm_count() - sm_reserve());
    CUtensorMap tmb{}, tma{};
    if (pair) {  // the stage copies go through tensor maps (rows of 256 bytes)
      if ((rc = byte_rows_map(&tmb, b, (size_t)ng * g.b_theta, SB * HB / 256)) ||
          (rc = byte_rows_map(&tma, ga.asl, (size_t)ng * a_theta, PAIR_A / 256)))
        break;
    }
    if (pair) {  // clusters of 2 CTAs (the two SMs of a TPC), one pair per tile
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((unsigned)(2 * std::min<int64_t>(ga.tiles, sms / 2)));
      cfg.blockDim = dim3(THREADS);
      cfg.dynamicSmemBytes = SMEM;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      GK_CUDA(cudaLaunchKernelEx(&cfg, ozaki_gemm<true>, ga, tmb, tma));
    } else {
      ozaki_gemm<false><<<(unsigned)std::min<int64_t>(ga.tiles, sms), THREADS, SMEM, st>>>(ga, tmb, tma);
    }
    count_launch();
    rc = check_launch("gk_collision (int8 slices: GEMM)");
  }
  if (rc == GK_OK) {  // fp64 recompute of the uncertified tiles (none on regular data: the CTAs exit)
    const int64_t max_tiles = (int64_t)nt * g.ncb * g.nib;
    if (M % 16 == 0) {  // with the DMMA collision's 64 x 128 tile: its bits on those tiles
      static unsigned long long* fixed = [] {
        void* p = nullptr;
        return cudaGetSymbolAddress(&p, g_fixed_tiles) == cudaSuccess ? (unsigned long long*)p : nullptr;
      }();
      if (!fixed) {
        gk::set_error("gk_collision: recompute counter unavailable");
        rc = GK_ERR_CUDA;
      } else {
        rc = collision_fix_dmma(A, H, C, M, T, N, g.ncb, g.nib, list, count, max_tiles, fixed, sm_count(), st);
      }
    } else {
      fix_tiles<<<(unsigned)std::min<int64_t>(max_tiles, 2 * sm_count()), 256, 0, st>>>(A, H, C, M, T, N, g.ncb,
                                                                                       g.nib, list, count);
      rc = check_launch("gk_collision (fp64 recompute of uncertified tiles)");
    }
  }
  if (ws) cudaFreeAsync(ws, st);
  return rc;
}
}  // namespace i8

// w/phi non-null: the group-by-group B slicing also writes the field moment
// phi[t] = sum_v w[v] h[v, t] of thetas [t0, t1) (bit-identical to gk_field), so
// a step whose B slices do not fit its workspace still reads the state once for
// the field moment and the collision.
// scratch non-null: collision_i8_group_scratch_bytes(M, T, N) bytes of the caller's
// workspace hold one theta group's B slices, the certificate bookkeeping and the A
// slices of all T thetas (kept there: reuse_a reuses them, see gemms); null: the
// library's scratch pool.
//   [G (B slices + column stats)] [fix] [A slices + row scales + row stats of T]
int64_t collision_i8_aslice_bytes(int64_t M, int64_t T);
static int64_t group_b_bytes(const i8::Geometry& g, int64_t G) {
  return (G * (int64_t)(g.b_theta + g.e_theta) + 255) & ~int64_t(255);
}
int64_t collision_i8_group_scratch_bytes(int64_t M, int64_t T, int64_t N) {
  const i8::Geometry g((int)M, N);
  const int64_t G = std::min<int64_t>(i8::theta_group(g.b_theta), T);
  return group_b_bytes(g, G) + i8::fix_bytes((int)M, (int)T, N) + collision_i8_aslice_bytes(M, T);
}

int collision_i8_range(const double* A, const double* H, double* C, int M, int T, int64_t N, int t0, int t1,
                       cudaStream_t st, const double* w, double* phi, void* scratch, bool reuse_a) {
  using namespace i8;
  const Geometry g(M, N);
  const int G = std::min(theta_group(g.b_theta), t1 - t0);
  const int64_t Gs = std::min(theta_group(g.b_theta), T);
  void* ws = nullptr;
  void* abuf = nullptr;
  if (scratch) {
    ws = scratch;
    abuf = (int8_t*)scratch + group_b_bytes(g, Gs) + fix_bytes(M, T, N);
  } else if (int r = scratch_alloc(&ws, group_b_bytes(g, G) + fix_bytes(M, T, N), st)) {
    return r;
  }
  int8_t* bsl = (int8_t*)ws;
  ColStat* bexp = (ColStat*)(bsl + (size_t)G * g.b_theta);
  unsigned* fix = (unsigned*)((int8_t*)ws + group_b_bytes(g, scratch ? Gs : G));
  const int rc = gemms(A, bsl, bexp, true, H, C, M, T, N, t0, t1, st, abuf, reuse_a && abuf, w, phi, fix);
  if (!scratch) cudaFreeAsync(ws, st);
  return rc;
}

// ---- step-level split (step.cu): B slices of every theta made in the field
// stage, so only the GEMMs run next to the nonlinear term.
//   [T B slices][T column stats][fix]
int64_t collision_i8_bslice_bytes(int64_t M, int64_t T, int64_t N) {
  const i8::Geometry g((int)M, N);
  return (((int64_t)T * (int64_t)(g.b_theta + g.e_theta) + 255) & ~int64_t(255)) +
         i8::fix_bytes((int)M, (int)T, N);
}

// B slices of thetas [t0, t1) into the all-theta buffer; with w/phi also the
// field moment of those thetas (bit-identical to gk_field)
int collision_i8_slices(const double* H, int64_t M, int64_t T, int64_t N, int64_t t0, int64_t t1, void* buf,
                        cudaStream_t st, const double* w, double* phi) {
  if (t1 == t0) return GK_OK;
  const i8::Geometry g((int)M, N);
  int8_t* bsl = (int8_t*)buf;
  i8::ColStat* bexp = (i8::ColStat*)(bsl + (size_t)T * g.b_theta);
  return i8::prepare_b(H, (int)M, (int)T, N, (int)t0, (int)t1, bsl, bexp, st, w, phi);
}

// A slices + row scales + row stats of all T thetas (the buffer
// collision_i8_presliced can keep between calls while A does not change)
int64_t collision_i8_aslice_bytes(int64_t M, int64_t T) {
  const i8::Geometry g((int)M, 2);
  return T * (int64_t)(g.a_theta() + g.arow_theta());
}

int collision_i8_presliced(const double* A, const void* buf, const double* H, double* C, int64_t M, int64_t T,
                           int64_t N, int64_t t0, int64_t t1, cudaStream_t st, void* abuf, bool reuse_a) {
  if (t1 == t0) return GK_OK;
  const i8::Geometry g((int)M, N);
  int8_t* bsl = (int8_t*)buf;
  i8::ColStat* bexp = (i8::ColStat*)(bsl + (size_t)T * g.b_theta);
  unsigned* fix = (unsigned*)(bsl + (((int64_t)T * (int64_t)(g.b_theta + g.e_theta) + 255) & ~int64_t(255)));
  return i8::gemms(A, bsl, bexp, false, H, C, (int)M, (int)T, N, (int)t0, (int)t1, st, abuf, reuse_a, nullptr,
                   nullptr, fix);
}

}  // namespace gk

// Tiles of the int8 collision whose certificate failed and that were recomputed in
// fp64, summed over the process (synchronous; diagnostics and tests).
extern "C" int gk_collision_fixups(int64_t* total) {
  GK_CHECK_ARG(total, "gk_collision_fixups: null pointer");
  unsigned long long v = 0;
  GK_CUDA(cudaDeviceSynchronize());
  GK_CUDA(cudaMemcpyFromSymbol(&v, gk::i8::g_fixed_tiles, sizeof(v)));
  *total = (int64_t)v;
  return GK_OK;
}

extern "C" int gk_collision_mode(int mode) {
  const int prev = gk::collision_mode();
  if (mode >= 0 && mode <= 2) gk::g_collision_mode = mode;
  return prev;
}

extern "C" int gk_probe_i8_peak(double* tops) {
  GK_CHECK_ARG(tops, "gk_probe_i8_peak: null pointer");
  using namespace gk::i8;
  const int sms = sm_count();
  const size_t smem = 100 * 1024;  // one CTA per SM
  GK_CUDA(cudaFuncSetAttribute(i8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  GK_CUDA(cudaEventCreate(&e0));
  GK_CUDA(cudaEventCreate(&e1));
  i8_peak_kernel<<<sms, 128, smem>>>(PROBE_REPS / 8);  // warm-up (clocks, TMEM)
  cudaEventRecord(e0);
  i8_peak_kernel<<<sms, 128, smem>>>(PROBE_REPS);
  cudaEventRecord(e1);
  GK_CUDA(cudaEventSynchronize(e1));
  gk::count_launch();
  gk::count_launch();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  GK_CUDA(cudaGetLastError());
  *tops = 2.0 * 128 * 256 * BK * (double)PROBE_REPS * sms / (ms * 1e-3) / 1e12;
  return GK_OK;
}
