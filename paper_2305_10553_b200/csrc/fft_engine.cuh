// Shared-memory mixed-radix fp64 FFT engine (Stockham autosort, forward sign).
//
// A CTA transforms a batch of B equal-length sequences held in shared memory:
// each pass takes the R inputs of every butterfly (stride n/R), applies the
// inter-pass twiddles from a per-plan table exp(-2*pi*i*m/n) in global memory
// (L1-resident), runs an R-point DFT in registers and scatters the results in
// autosort order into the other buffer.  Radices 2,3,4,5,6,7,8,9,16 have
// register butterflies; any other factor runs a generic O(R^2) pass, so every
// integer plan the reference's bracket accepts (spectral.py:228-229) is legal.
//
// Inverse transforms are conj(F(conj(x))); callers fold the conjugations into
// their load/store fusions.  All arithmetic uses explicit-rounding intrinsics
// (gk_common.cuh), so the same data gives the same bits in every kernel.
#pragma once

#include <type_traits>

#include "gk_common.cuh"
#include "fft_consts.cuh"

namespace gk {
namespace fft {

constexpr int kMaxPass = 24;

struct Desc {
  int n;
  int npass;
  int radix[kMaxPass];
  const double2* tw;  // exp(-2*pi*i*m/n), m in [0, n)
};

// u * exp(-2*pi*i*m/R) with R, m compile-time after unrolling.
__device__ __forceinline__ double2 rot(double2 u, int m, int R) {
  m %= R;
  if (m == 0) return u;
  if (4 * m == R) return cmul_mi(u);                     // * -i
  if (2 * m == R) return make_double2(-u.x, -u.y);        // * -1
  if (4 * m == 3 * R) return cmul_pi(u);                 // * +i
  return cmul(u, wconst(R, m));
}

template <int R>
__device__ __forceinline__ void dft(double2* v);

template <>
__device__ __forceinline__ void dft<1>(double2*) {}

template <>
__device__ __forceinline__ void dft<2>(double2* v) {
  const double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <>
__device__ __forceinline__ void dft<4>(double2* v) {
  const double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
  const double2 s13 = cadd(v[1], v[3]), d13 = cmul_mi(csub(v[1], v[3]));
  v[0] = cadd(s02, s13);
  v[2] = csub(s02, s13);
  v[1] = cadd(d02, d13);
  v[3] = csub(d02, d13);
}

// odd prime R: symmetric form, (R-1)/2 cosine and sine sums.
template <int R>
__device__ __forceinline__ void dft_odd(double2* v) {
  constexpr int H = (R - 1) / 2;
  double2 a[H], b[H];
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    a[j - 1] = cadd(v[j], v[R - j]);
    b[j - 1] = csub(v[j], v[R - j]);
  }
  double2 y0 = v[0];
#pragma unroll
  for (int j = 0; j < H; ++j) y0 = cadd(y0, a[j]);
  double2 out[R];
  out[0] = y0;
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    double2 re = v[0];
    double2 im = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const double2 w = wconst(R, (j * k) % R);  // (cos, -sin)
      const double c = w.x, s = -w.y;
      re.x = __fma_rn(c, a[j - 1].x, re.x);
      re.y = __fma_rn(c, a[j - 1].y, re.y);
      im.x = __fma_rn(s, b[j - 1].x, im.x);
      im.y = __fma_rn(s, b[j - 1].y, im.y);
    }
    // y_k = re - i*im ; y_{R-k} = re + i*im
    out[k] = make_double2(__dadd_rn(re.x, im.y), __dsub_rn(re.y, im.x));
    out[R - k] = make_double2(__dsub_rn(re.x, im.y), __dadd_rn(re.y, im.x));
  }
#pragma unroll
  for (int k = 0; k < R; ++k) v[k] = out[k];
}

template <>
__device__ __forceinline__ void dft<3>(double2* v) { dft_odd<3>(v); }
template <>
__device__ __forceinline__ void dft<5>(double2* v) { dft_odd<5>(v); }
template <>
__device__ __forceinline__ void dft<7>(double2* v) { dft_odd<7>(v); }

// composite R = R1*R2 in registers: n = n1*R2 + n2, k = k1 + R1*k2.
template <int R1, int R2>
__device__ __forceinline__ void dft_ct(double2* v) {
  constexpr int R = R1 * R2;
  double2 t[R];
#pragma unroll
  for (int n2 = 0; n2 < R2; ++n2) {
    double2 u[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) u[n1] = v[n1 * R2 + n2];
    dft<R1>(u);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) t[n2 * R1 + k1] = rot(u[k1], n2 * k1, R);
  }
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) {
    double2 u[R2];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) u[n2] = t[n2 * R1 + k1];
    dft<R2>(u);
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) v[k1 + R1 * k2] = u[k2];
  }
}

// Good-Thomas prime-factor DFT for coprime N1, N2: Ruritanian input map
// n = (N2 n1 + N1 n2) mod N and CRT output map k = (N2 t2 k1 + N1 t1 k2) mod N
// (t2 = N2^-1 mod N1, t1 = N1^-1 mod N2) turn the DFT into N2 DFTs of size N1
// followed by N1 DFTs of size N2 with no twiddle multiplications at all.  All
// index maps are compile-time (register renaming only).
__host__ __device__ constexpr int inv_mod(int a, int m) {
  for (int x = 1; x < m; ++x)
    if ((a * x) % m == 1) return x;
  return 1;
}

template <int N1, int N2>
__device__ __forceinline__ void dft_pfa(double2* v) {
  constexpr int N = N1 * N2;
  constexpr int T2 = inv_mod(N2 % N1, N1), T1 = inv_mod(N1 % N2, N2);
  double2 t[N];
#pragma unroll
  for (int n2 = 0; n2 < N2; ++n2) {
    double2 u[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) u[n1] = v[(N2 * n1 + N1 * n2) % N];
    dft<N1>(u);
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) t[n2 * N1 + k1] = u[k1];
  }
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) {
    double2 u[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) u[n2] = t[n2 * N1 + k1];
    dft<N2>(u);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) v[(N2 * T2 * k1 + N1 * T1 * k2) % N] = u[k2];
  }
}

template <>
__device__ __forceinline__ void dft<6>(double2* v) { dft_pfa<2, 3>(v); }

// --- known-zero inputs and real inputs (YCOL n_y = 144 fast path) ---------------
// Z: bit i set <=> input i is known to be zero at compile time.  Additions with a
// known zero are skipped (x + 0 -> x: identical except for the sign of a zero).
template <bool ZA, bool ZB>
__device__ __forceinline__ double2 zadd(double2 a, double2 b) {
  if constexpr (ZA && ZB) return make_double2(0.0, 0.0);
  else if constexpr (ZA) return b;
  else if constexpr (ZB) return a;
  else return cadd(a, b);
}
template <bool ZA, bool ZB>
__device__ __forceinline__ double2 zsub(double2 a, double2 b) {
  if constexpr (ZA && ZB) return make_double2(0.0, 0.0);
  else if constexpr (ZA) return make_double2(-b.x, -b.y);
  else if constexpr (ZB) return a;
  else return csub(a, b);
}
template <unsigned Z>
__device__ __forceinline__ void dft4_z(double2* v) {
  constexpr bool z0 = Z & 1u, z1 = Z & 2u, z2 = Z & 4u, z3 = Z & 8u;
  constexpr bool zs = z0 && z2, zd = z1 && z3;
  const double2 s02 = zadd<z0, z2>(v[0], v[2]), d02 = zsub<z0, z2>(v[0], v[2]);
  const double2 s13 = zadd<z1, z3>(v[1], v[3]), d13 = cmul_mi(zsub<z1, z3>(v[1], v[3]));
  v[0] = zadd<zs, zd>(s02, s13);
  v[2] = zsub<zs, zd>(s02, s13);
  v[1] = zadd<zs, zd>(d02, d13);
  v[3] = zsub<zs, zd>(d02, d13);
}
// sub-mask of the DFT-4 over n1 (input (3 n1 + 4 n2) % 12) in dft_pfa<4, 3>
__host__ __device__ constexpr unsigned pfa43_sub(unsigned Z, int n2) {
  unsigned m = 0;
  for (int n1 = 0; n1 < 4; ++n1)
    if (Z >> ((3 * n1 + 4 * n2) % 12) & 1u) m |= 1u << n1;
  return m;
}
// 12-point DFT (Good-Thomas 4 x 3, same maps as dft_pfa<4, 3>) with inputs known zero
template <unsigned Z>
__device__ __forceinline__ void dft12_z(double2* v) {
  double2 t[12];
  auto stage1 = [&](auto zc, int n2) {
    constexpr unsigned zm = decltype(zc)::value;
    double2 u[4];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) u[n1] = (zm >> n1 & 1u) ? make_double2(0.0, 0.0) : v[(3 * n1 + 4 * n2) % 12];
    dft4_z<zm>(u);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) t[n2 * 4 + k1] = u[k1];
  };
  stage1(std::integral_constant<unsigned, pfa43_sub(Z, 0)>{}, 0);
  stage1(std::integral_constant<unsigned, pfa43_sub(Z, 1)>{}, 1);
  stage1(std::integral_constant<unsigned, pfa43_sub(Z, 2)>{}, 2);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    double2 u[3] = {t[k1], t[4 + k1], t[8 + k1]};
    dft<3>(u);
#pragma unroll
    for (int k2 = 0; k2 < 3; ++k2) v[(9 * k1 + 4 * k2) % 12] = u[k2];
  }
}
// 8-point DFT (Cooley-Tukey 2 x 4, the maps of dft_ct<2, 4>) with inputs known zero
template <unsigned Z>
__device__ __forceinline__ void dft8_z(double2* v) {
  double2 t[8];
  // stage 1: radix-2 over (n2, n2 + 4), twiddle W_8^{n2 k1}; a pair of zeros stays zero
  auto bfly = [&](auto n2c) {
    constexpr int n2 = decltype(n2c)::value;
    constexpr bool za = Z >> n2 & 1u, zb = Z >> (n2 + 4) & 1u;
    t[n2 * 2 + 0] = zadd<za, zb>(v[n2], v[n2 + 4]);
    const double2 d = zsub<za, zb>(v[n2], v[n2 + 4]);
    if constexpr (za && zb) t[n2 * 2 + 1] = d;
    else t[n2 * 2 + 1] = rot(d, n2, 8);
  };
  bfly(std::integral_constant<int, 0>{});
  bfly(std::integral_constant<int, 1>{});
  bfly(std::integral_constant<int, 2>{});
  bfly(std::integral_constant<int, 3>{});
  // stage 2: DFT-4 over n2 for k1 = 0, 1; input n2 is zero iff both of its pair were
  constexpr unsigned zp = ((Z & 0xFu) & (Z >> 4 & 0xFu));
#pragma unroll
  for (int k1 = 0; k1 < 2; ++k1) {
    double2 u[4] = {t[k1], t[2 + k1], t[4 + k1], t[6 + k1]};
    dft4_z<zp>(u);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) v[k1 + 2 * k2] = u[k2];
  }
}
// sub-mask of the DFT-8 over n1 (input (3 n1 + 8 n2) % 24) in dft_pfa<8, 3>
__host__ __device__ constexpr unsigned pfa83_sub(unsigned Z, int n2) {
  unsigned m = 0;
  for (int n1 = 0; n1 < 8; ++n1)
    if (Z >> ((3 * n1 + 8 * n2) % 24) & 1u) m |= 1u << n1;
  return m;
}
// 24-point DFT (Good-Thomas 8 x 3, the maps of dft_pfa<8, 3>) with inputs known
// zero (the x inverse's padding band: inputs 8..15 of every warp four-step row)
template <unsigned Z>
__device__ __forceinline__ void dft24_z(double2* v) {
  double2 t[24];
  auto stage1 = [&](auto zc, int n2) {
    constexpr unsigned zm = decltype(zc)::value;
    double2 u[8];
#pragma unroll
    for (int n1 = 0; n1 < 8; ++n1) u[n1] = (zm >> n1 & 1u) ? make_double2(0.0, 0.0) : v[(3 * n1 + 8 * n2) % 24];
    dft8_z<zm>(u);
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) t[n2 * 8 + k1] = u[k1];
  };
  stage1(std::integral_constant<unsigned, pfa83_sub(Z, 0)>{}, 0);
  stage1(std::integral_constant<unsigned, pfa83_sub(Z, 1)>{}, 1);
  stage1(std::integral_constant<unsigned, pfa83_sub(Z, 2)>{}, 2);
#pragma unroll
  for (int k1 = 0; k1 < 8; ++k1) {
    double2 u[3] = {t[k1], t[8 + k1], t[16 + k1]};
    dft<3>(u);
#pragma unroll
    for (int k2 = 0; k2 < 3; ++k2) v[(9 * k1 + 16 * k2) % 24] = u[k2];
  }
}
// 3-point DFT of real input: X0 real, X2 = conj(X1)
__device__ __forceinline__ void dft3_real(double a, double b, double c, double2* u) {
  const double2 w = wconst(3, 1);  // (cos, -sin)
  const double a0 = __dadd_rn(b, c), d = __dsub_rn(b, c);
  const double re = __fma_rn(w.x, a0, a), im = __dmul_rn(-w.y, d);
  u[0] = make_double2(__dadd_rn(a, a0), 0.0);
  u[1] = make_double2(re, -im);
  u[2] = make_double2(re, im);
}
// 12-point DFT of real input x (Good-Thomas 4 x 3): real 4-point DFTs, real 3-point
// DFTs for k1 = 0, 2, one complex 3-point DFT for k1 = 1, and k1 = 3 by the
// Hermitian symmetry X[12 - k] = conj(X[k]).
__device__ __forceinline__ void dft12_real(const double* x, double2* X) {
  double r0[3], r2[3];
  double2 c1[3];
#pragma unroll
  for (int n2 = 0; n2 < 3; ++n2) {
    const double e0 = x[(4 * n2) % 12], e1 = x[(3 + 4 * n2) % 12], e2 = x[(6 + 4 * n2) % 12],
                 e3 = x[(9 + 4 * n2) % 12];
    const double s02 = __dadd_rn(e0, e2), d02 = __dsub_rn(e0, e2);
    const double s13 = __dadd_rn(e1, e3), d13 = __dsub_rn(e1, e3);
    r0[n2] = __dadd_rn(s02, s13);
    r2[n2] = __dsub_rn(s02, s13);
    c1[n2] = make_double2(d02, -d13);
  }
  double2 u[3];
  dft3_real(r0[0], r0[1], r0[2], u);
  X[0] = u[0], X[4] = u[1], X[8] = u[2];
  dft3_real(r2[0], r2[1], r2[2], u);
  X[6] = u[0], X[10] = u[1], X[2] = u[2];
  dft<3>(c1);
  X[9] = c1[0], X[1] = c1[1], X[5] = c1[2];
  X[3] = cconj(X[9]), X[7] = cconj(X[5]), X[11] = cconj(X[1]);
}

template <>
__device__ __forceinline__ void dft<8>(double2* v) { dft_ct<2, 4>(v); }
template <>
__device__ __forceinline__ void dft<9>(double2* v) { dft_ct<3, 3>(v); }
template <>
__device__ __forceinline__ void dft<16>(double2* v) { dft_ct<4, 4>(v); }
template <>
__device__ __forceinline__ void dft<10>(double2* v) { dft_pfa<2, 5>(v); }
template <>
__device__ __forceinline__ void dft<12>(double2* v) { dft_pfa<4, 3>(v); }
template <>
__device__ __forceinline__ void dft<14>(double2* v) { dft_pfa<2, 7>(v); }
// register DFTs of the warp four-step transforms (720 = 24 * 30)
template <>
__device__ __forceinline__ void dft<24>(double2* v) { dft_pfa<8, 3>(v); }
template <>
__device__ __forceinline__ void dft<30>(double2* v) { dft_pfa<6, 5>(v); }
// YCOL n_y = 480 = 20 * 24
template <>
__device__ __forceinline__ void dft<20>(double2* v) { dft_pfa<4, 5>(v); }
// YCOL n_y = 864 = 32 * 27
template <>
__device__ __forceinline__ void dft<27>(double2* v) { dft_ct<3, 9>(v); }
template <>
__device__ __forceinline__ void dft<32>(double2* v) { dft_ct<4, 8>(v); }

// One Stockham pass of radix R over B sequences (stride ld) from src to dst.
template <int R>
__device__ __forceinline__ void pass_fixed(const double2* __restrict__ src, double2* __restrict__ dst,
                                           int n, int ns, int ld, int B, const double2* __restrict__ tw,
                                           int tid, int nth) {
  const int nb = n / R;
  const int total = nb * B;
  const int tstep = n / (ns * R);
  for (int q = tid; q < total; q += nth) {
    const int b = q / nb;
    const int j = q - b * nb;
    const double2* s = src + b * ld;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[j + r * nb];
    const int k = j % ns;
    if (k != 0) {
      const int step = k * tstep;
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(tw + r * step));
    }
    dft<R>(v);
    double2* d = dst + b * ld + (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) d[r * ns] = v[r];
  }
}

// Generic radix (any R): one thread per butterfly output, O(R) work each.
__device__ __forceinline__ void pass_generic(const double2* __restrict__ src, double2* __restrict__ dst,
                                             int n, int R, int ns, int ld, int B,
                                             const double2* __restrict__ tw, int tid, int nth) {
  const int nb = n / R;
  const int total = nb * B * R;
  const int tstep = n / (ns * R);
  const int rstep = n / R;  // exp(-2 pi i / R) = tw[rstep]
  for (int q = tid; q < total; q += nth) {
    const int ro = q % R;
    const int bj = q / R;
    const int b = bj / nb;
    const int j = bj - b * nb;
    const int k = j % ns;
    const double2* s = src + b * ld;
    double2 acc = make_double2(0.0, 0.0);
    for (int r = 0; r < R; ++r) {
      double2 x = s[j + r * nb];
      if (k != 0 && r != 0) x = cmul(x, __ldg(tw + r * k * tstep));
      const int e = (r * ro) % R;
      acc = cadd(acc, e == 0 ? x : cmul(x, __ldg(tw + e * rstep)));
    }
    dst[b * ld + (j - k) * R + k + ro * ns] = acc;
  }
}

// All passes of the plan over B sequences starting in buf0 (scratch buf1).
// Returns the buffer holding the result.  Must be called by every thread of
// the CTA (contains __syncthreads); the caller syncs before the first pass.
__device__ __forceinline__ double2* run(const Desc& d, double2* buf0, double2* buf1, int ld, int B,
                                        int tid, int nth) {
  double2* src = buf0;
  double2* dst = buf1;
  int ns = 1;
  for (int p = 0; p < d.npass; ++p) {
    const int R = d.radix[p];
    switch (R) {
      case 2: pass_fixed<2>(src, dst, d.n, ns, ld, B, d.tw, tid, nth); break;
      case 3: pass_fixed<3>(src, dst, d.n, ns, ld, B, d.tw, tid, nth); break;
      case 4: pass_fixed<4>(src, dst, d.n, ns, ld, B, d.tw, tid, nth); break;
      case 5: pass_fixed<5>(src, dst, d.n, ns, ld, B, d.tw, tid, nth); break;
      case 6: pass_fixed<6>(src, dst, d.n, ns, ld, B, d.tw, tid, nth); break;
      case 7: pass_fixed<7>(src, dst, d.n, ns, ld, B, d.tw, tid, nth); break;
      case 8: pass_fixed<8>(src, dst, d.n, ns, ld, B, d.tw, tid, nth); break;
      case 9: pass_fixed<9>(src, dst, d.n, ns, ld, B, d.tw, tid, nth); break;
      case 16: pass_fixed<16>(src, dst, d.n, ns, ld, B, d.tw, tid, nth); break;
      default: pass_generic(src, dst, d.n, R, ns, ld, B, d.tw, tid, nth); break;
    }
    __syncthreads();
    double2* t = src;
    src = dst;
    dst = t;
    ns *= R;
  }
  return src;
}

}  // namespace fft
}  // namespace gk
