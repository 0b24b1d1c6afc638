// Compile-time-specialised fp64 FFT passes for the benchmark grid sizes.
//
// One thread per butterfly: a transform of N = R0*R1*...  is run by
// maxbf = max_p N/R_p threads; in pass p thread j < N/R_p loads R_p inputs,
// applies the inter-pass twiddles (from a shared-memory table), runs the
// register DFT and writes back in Stockham autosort order.  The first pass
// reads its inputs through a caller functor (straight from global memory, with
// any prologue math fused) and the last pass hands its outputs to a caller
// functor (straight to global, epilogue fused), so a 3-pass transform costs two
// shared-memory round trips instead of five.  IL transforms are interleaved
// element by element in shared memory (element i of transform b at i*IL + b):
// lanes that differ in b touch consecutive 16-byte slots, so every access is
// bank-conflict free whatever the pass stride, and global accesses of IL rows
// come out as contiguous runs.  In-place (single buffer): every pass syncs
// between its loads and its stores.  Radices are chosen so that the butterfly
// counts of the passes are close (720 = 10*8*9 -> 72/90/80 threads busy).
#pragma once

#include "fft_engine.cuh"

#ifndef GK_TWIDDLE_LOADS
#define GK_TWIDDLE_LOADS 1  // table loads per butterfly for the inter-pass twiddles (1 or 2)
#endif

namespace gk {
namespace fftx {

template <int... Rs>
struct Seq {
  static constexpr int P = sizeof...(Rs);
  static constexpr int N = (1 * ... * Rs);
  __host__ __device__ static constexpr int radix(int p) {
    constexpr int a[] = {Rs...};
    return a[p];
  }
  __host__ __device__ static constexpr int ns(int p) {
    int s = 1;
    for (int i = 0; i < p; ++i) s *= radix(i);
    return s;
  }
  // compact twiddle table (TWC): pass p >= 1 keeps W_N^(k N / (NS_p R_p)) for k < NS_p
  // at offset twc_off(p) -- sum of NS_q over 1 <= q < p -- instead of all N powers
  __host__ __device__ static constexpr int twc_off(int p) {
    int o = 0;
    for (int q = 1; q < p; ++q) o += ns(q);
    return o;
  }
  __host__ __device__ static constexpr int twc_size() { return twc_off(P); }
  __host__ __device__ static constexpr int maxbf() {
    int m = 0;
    for (int i = 0; i < P; ++i) m = (N / radix(i)) > m ? (N / radix(i)) : m;
    return m;
  }
};

struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// `after0` runs (on every thread) once pass 0 has finished reading its inputs:
// the caller's staging buffer is free again from that point (prefetch hook).
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// named barrier over one team of `n` threads (multiple of 32), id >= 1
struct TeamSync {
  int id, n;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
  }
};

// Inter-pass twiddles w^r = exp(-2 pi i k r TS / N), r = 1..R-1.  Only w^1 and
// w^4 come from the shared-memory table; the others are products of at most
// three table values (w^2 = w*w, w^3 = w^2*w, w^{r} = w^4 * w^{r-4}, ...), which
// trades idle fp64 issue slots for shared-memory bandwidth (the co-limiter of
// these passes).  Same code for every transform -> still bit-reproducible.
template <int R, int TS>
__device__ __forceinline__ void twiddle(double2* v, const double2* __restrict__ tw, int k) {
#if GK_TWIDDLE_LOADS == 2
  if constexpr (R <= 4) {
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[k * r * TS]);
    return;
  }
#endif
  // one table load; w^r by repeated squaring/multiplication (depth <= 4 for R <= 16)
  double2 w[R];
  w[1] = tw[k * TS];
#if GK_TWIDDLE_LOADS == 2
  w[4] = tw[4 * k * TS];
#endif
#pragma unroll
  for (int r = 2; r < R; ++r) {
#if GK_TWIDDLE_LOADS == 2
    if (r == 4) continue;
#endif
    w[r] = (r % 2 == 0) ? cmul(w[r / 2], w[r / 2]) : cmul(w[r - 1], w[1]);
  }
#pragma unroll
  for (int r = 1; r < R; ++r) v[r] = cmul(v[r], w[r]);
}

// CLAMP: lanes past the butterfly count compute a clamped copy (their warp issues
// the instructions anyway), only stores are predicated, and the k == 0 twiddle is
// applied as tw[0] = 1 (exact) -- no divergent branches in the pass; fully idle
// warps still skip (warp-uniform __any_sync).  Used by the x-direction team
// kernels; ycol keeps the plain form (the clamped copies spill there).
// PADW > 0 (IL = 1 only): element i of the shared buffer lives at i + i / PADW.
// With PADW = R_0 the Stockham stores of a 12 x 12 x 14 transform (stride 12 in
// pass 0, groups of 12 at stride 144 in pass 1) hit distinct banks in every
// quarter warp (unpadded: 4- and 3-way conflicts); the contiguous loads stay
// conflict-free.
template <int IL, int PADW>
__device__ __forceinline__ int sidx(int i, int b) {
  if constexpr (PADW > 0) return i + i / PADW;
  return i * IL + b;
}
// Padded index of i0 + r * STRIDE as one division per butterfly: STRIDE a multiple
// of PADW (the run keeps its phase), or STRIDE = 1 from an aligned i0 with r < PADW.
template <int IL, int PADW, int STRIDE>
struct Run {
  static_assert(PADW == 0 || STRIDE % PADW == 0 || STRIDE == 1, "padded run: stride");
  static constexpr int step = PADW == 0 ? STRIDE * IL : (STRIDE == 1 ? 1 : STRIDE + STRIDE / PADW);
};
template <class S, int p, int IL, bool CLAMP, class Load, class Store, class Hook, class Sync = CtaSync,
          int PADW = 0, bool TWC = false>
__device__ __forceinline__ void passes(double2* __restrict__ sm, int b, int j, const double2* __restrict__ tw,
                                       Load& load, Store& store, Hook& after0, const Sync& sync = Sync()) {
  static_assert(PADW == 0 || IL == 1, "padding: single transform per buffer");
  static_assert(PADW == 0 || S::ns(p) != 1 || (S::radix(p) <= PADW && S::radix(p) % PADW == 0),
                "padding: a stride-1 store run must start at a multiple of PADW and stay inside it");
  constexpr int R = S::radix(p);
  constexpr int NB = S::N / R;
  constexpr int NS = S::ns(p);
  constexpr bool first = (p == 0);
  constexpr bool last = (p == S::P - 1);
  double2 v[R];
  const bool act = j < NB;
  int k = 0;
  if constexpr (CLAMP) {
    const int jj = act ? j : NB - 1;
    k = first ? 0 : jj % NS;
    if (__any_sync(0xffffffffu, act)) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (first)
          v[r] = load(jj + r * NB);
        else
          v[r] = sm[sidx<IL, PADW>(jj, b) + r * Run<IL, PADW, NB>::step];
      }
      if constexpr (!first) {
        if constexpr (TWC) twiddle<R, 1>(v, tw + S::twc_off(p), k);
        else twiddle<R, S::N / (NS * R)>(v, tw, k);
      }
      fft::dft<R>(v);
    }
  } else if (act) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if constexpr (first)
        v[r] = load(j + r * NB);
      else
        v[r] = sm[sidx<IL, PADW>(j, b) + r * Run<IL, PADW, NB>::step];
    }
    if constexpr (!first) {  // k == 0 multiplies by tw[0] = 1 exactly: no divergent skip
      k = j % NS;
      if constexpr (TWC) twiddle<R, 1>(v, tw + S::twc_off(p), k);
      else twiddle<R, S::N / (NS * R)>(v, tw, k);
    }
    fft::dft<R>(v);
  }
  if constexpr (!first) sync();
  if (act) {
    const int base = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if constexpr (last)
        store(base + r * NS, v[r]);
      else
        sm[sidx<IL, PADW>(base, b) + r * Run<IL, PADW, NS>::step] = v[r];
    }
  }
  if constexpr (!last) {
    sync();
    if constexpr (first) after0();
    passes<S, p + 1, IL, CLAMP, Load, Store, Hook, Sync, PADW, TWC>(sm, b, j, tw, load, store, after0, sync);
  }
}

// Run a whole transform: the caller must have synchronised the CTA since the
// previous use of `sm` (pass 0 writes it without a leading barrier).
template <class S, int IL, bool CLAMP = false, class Load, class Store>
__device__ __forceinline__ void transform(double2* sm, int b, int j, const double2* tw, Load& load, Store& store) {
  NoHook h;
  passes<S, 0, IL, CLAMP>(sm, b, j, tw, load, store, h);
}
template <class S, int IL, bool CLAMP = false, class Load, class Store, class Hook>
__device__ __forceinline__ void transform(double2* sm, int b, int j, const double2* tw, Load& load, Store& store,
                                          Hook& after0) {
  static_assert(S::P >= 2, "the pass-0 hook needs a multi-pass transform");
  passes<S, 0, IL, CLAMP>(sm, b, j, tw, load, store, after0);
}

template <class S, int PADW = 0, bool TWC = false, class Load, class Store, class Hook>
__device__ __forceinline__ void transform_team(double2* sm, int j, const double2* tw, Load& load, Store& store,
                                               Hook& after0, const TeamSync& sync) {
  static_assert(S::P >= 2, "the pass-0 hook needs a multi-pass transform");
  passes<S, 0, 1, true, Load, Store, Hook, TeamSync, PADW, TWC>(sm, 0, j, tw, load, store, after0, sync);
}
// fill a compact twiddle table (TWC) from the full table W_N^i, i < N
template <class S>
__device__ __forceinline__ void init_twc(double2* tw, const double2* full) {
  for (int p = 1; p < S::P; ++p)
    for (int k = threadIdx.x; k < S::ns(p); k += blockDim.x)
      tw[S::twc_off(p) + k] = full[k * (S::N / (S::ns(p) * S::radix(p)))];
}

// Warp four-step transform, N = N1 * N2 with N1, N2 <= 32, one warp per
// transform and a single shared-memory round trip:
//   lane n2 < N2: x[N2 n1 + n2] (n1 < N1) -> DFT_N1 in registers -> * W_N^{n2 k1}
//                 (table tw4[k1 * N2 + n2], conflict-free) -> z[k1][n2]
//   lane k1 < N1: z[k1][*] -> DFT_N2 in registers -> X[k1 + N1 k2]
// z has pitch N2 + 1 (odd): the phase-2 column reads are bank-conflict free.
// Only __syncwarp between the phases; `after_load` runs once every lane has
// read its inputs (the caller's staging buffer is free: prefetch hook).
// ZIN: phase-1 inputs n1 known to be zero (bit n1; not loaded, skipped in the
// DFT -- 24-point only); DROP: phase-2 outputs k2 never stored (dead code).
template <int N1, int N2, unsigned ZIN = 0, unsigned DROP = 0, class Load, class Store, class Hook>
__device__ __forceinline__ void warp4(double2* __restrict__ z, const double2* __restrict__ tw4, int lane,
                                      Load& load, Store& store, Hook& after_load) {
  static_assert(N1 <= 32 && N2 <= 32, "one lane per row/column");
  static_assert(ZIN == 0 || N1 == 24, "known-zero inputs: 24-point first phase only");
  constexpr int ZP = N2 + 1;
  double2 v[N1];
  if (lane < N2) {
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) v[n1] = (ZIN >> n1 & 1u) ? make_double2(0.0, 0.0) : load(N2 * n1 + lane);
  }
  __syncwarp();
  after_load();
  if (lane < N2) {
    if constexpr (ZIN != 0) fft::dft24_z<ZIN>(v);
    else fft::dft<N1>(v);
#pragma unroll
    for (int k1 = 1; k1 < N1; ++k1) v[k1] = cmul(v[k1], tw4[k1 * N2 + lane]);
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) z[k1 * ZP + lane] = v[k1];
  }
  __syncwarp();
  if (lane < N1) {
    double2 u[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) u[n2] = z[lane * ZP + n2];
    fft::dft<N2>(u);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2)
      if (!(DROP >> k2 & 1u)) store(lane + N1 * k2, u[k2]);
  }
  __syncwarp();
}

// 16-byte asynchronous global -> shared copy (LDGSTS), commit / wait.
__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

}  // namespace fftx
}  // namespace gk
