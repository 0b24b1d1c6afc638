// Collision: per-theta real (n_vel x n_vel) matrix applied over velocity space
// (reference kernels.py:109-123).
//
// The interleaved complex state viewed as doubles turns each theta plane into a
// real matrix B_t (K = n_vel rows, N = 2*n_cells columns, row stride
// n_theta*2*n_cells), so out_t = A_t (n_vel x n_vel) @ B_t is one real DGEMM per
// theta -- half the flops of the reference's numpy path, which upcasts A to
// complex (zgemm).  At sh03b that is 9.78e11 flop over 13.7 GB: arithmetic
// intensity 72 flop/B, far above B200's fp64 ridge, so the roofline is fp64
// throughput.  tcgen05 has no f64 kind; the fp64 tensor path on sm_100a is the
// warp-level DMMA (mma.sync m8n8k4 f64, SASS DMMA).
//
// Tiling (v2, default when n_vel % 16 == 0): CTA tile BM x 128 (BM = 8*MT, MT
// chosen so BM divides n_vel when it can), 4 warps side by side along N, each
// warp MT x 4 DMMA tiles (8x8), K in steps of 16 through a 4-stage cp.async
// pipeline with per-thread copy descriptors computed once; two CTAs per SM.
// v1 (any n_vel): 8 warps, BN = 256, 3 stages.  Grid x runs over the M tiles so
// the n_vel/BM CTAs that share one B tile are co-scheduled and the B tile is
// read from HBM once (then L2).  Fixed K order -> bitwise run-to-run identical.
#include <algorithm>

#include "gk_common.cuh"
#include "../../include/gk.h"

namespace gk {

namespace coll {

constexpr int BK = 16;
constexpr int STAGES = 3;
constexpr int WARPS = 8;
constexpr int NT = 4;                 // 8-col DMMA tiles per warp
constexpr int BN = WARPS * NT * 8;    // 256
constexpr int LDB = BN + 4;           // ≡ 4 (mod 16) words: conflict-free fragment loads

__host__ __device__ constexpr int lda_for(int bm) { return bm + ((4 - bm) % 16 + 16) % 16; }

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int MT>
struct Smem {
  static constexpr int BM = 8 * MT;
  static constexpr int LDA = lda_for(BM);
  double a[STAGES][BK][LDA];
  double b[STAGES][BK][LDB];
};

template <int MT>
__global__ void __launch_bounds__(WARPS * 32, 1)
    dgemm_theta_kernel(const double* __restrict__ A, const double* __restrict__ H,
                       double* __restrict__ C, int M, int n_theta, int64_t N, int t_base) {
  constexpr int BM = 8 * MT;
  using S = Smem<MT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int m0 = blockIdx.x * BM;
  const int64_t n0 = (int64_t)blockIdx.y * BN;
  const int t = blockIdx.z + t_base;
  const int K = M;
  const int64_t ldh = (int64_t)n_theta * N;  // row stride of B_t / C_t in doubles
  const double* At = A + (int64_t)t * M * M;
  const double* Bt = H + (int64_t)t * N;
  double* Ct = C + (int64_t)t * N;

  auto load_tile = [&](int stage, int k0) {
    // A: BM x BK, global row-major (k contiguous) -> smem [k][m]
    for (int e = tid; e < BM * BK; e += WARPS * 32) {
      const int kk = e % BK, mm = e / BK;
      const int gi = m0 + mm, gk = k0 + kk;
      const bool ok = gi < M && gk < K;
      cp_async8(&sm.a[stage][kk][mm], ok ? At + (int64_t)gi * M + gk : At, ok);
    }
    // B: BK x BN, rows of the theta plane, 16-byte chunks
    for (int e = tid; e < BK * BN / 2; e += WARPS * 32) {
      const int kk = e / (BN / 2), nn = (e % (BN / 2)) * 2;
      const int gk = k0 + kk;
      const int64_t gn = n0 + nn;
      const bool ok = gk < K && gn < N;
      cp_async16(&sm.b[stage][kk][nn], ok ? Bt + (int64_t)gk * ldh + gn : Bt, ok);
    }
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int ktiles = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_tile(s, s * BK);
    cp_commit();
  }

  const int fr = lane >> 2;  // fragment row / col group
  const int fk = lane & 3;   // fragment k
  const int wn = warp * NT * 8;

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = kt + STAGES - 1;
    if (nxt < ktiles) load_tile(nxt % STAGES, nxt * BK);
    cp_commit();
    const int st = kt % STAGES;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double af[MT], bf[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) af[i] = sm.a[st][k4 + fk][8 * i + fr];
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = sm.b[st][k4 + fk][wn + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_wait<0>();

  // epilogue: C fragment rows fr (+8i), cols 2*fk (+8j)
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int gi = m0 + 8 * i + fr;
    if (gi >= M) continue;
    double* crow = Ct + (int64_t)gi * ldh;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int64_t gn = n0 + wn + 8 * j + 2 * fk;
      if (gn < N) __stcs(reinterpret_cast<double2*>(crow + gn), make_double2(acc[i][j][0], acc[i][j][1]));
    }
  }
}

// v2: A staged [m][k] (16-byte cp.async, LDA = BK+4 keeps the fragment loads
// conflict-free), per-thread cp.async source pointers computed once and bumped
// per k tile, STAGES2-deep pipeline.  Requires K % BK == 0 (the host falls back
// to v1 otherwise); M and N edges are predicated as in v1.
template <int MT, int BK2, int STAGES2, int W2 = WARPS>
struct Smem2 {
  static constexpr int BM = 8 * MT;
  static constexpr int LDA2 = BK2 + 4;  // conflict-free fragment loads
  static constexpr int LDB2 = W2 * NT * 8 + 4;
  double a[STAGES2][BM][LDA2];
  double b[STAGES2][BK2][LDB2];
};

// One BM x BN tile of out_t = A_t B_t (rows m0.., columns n0.. of theta t).
template <int MT, int BK2, int STAGES2, int W2>
__device__ __forceinline__ void v2_tile(Smem2<MT, BK2, STAGES2, W2>& sm, const double* __restrict__ A,
                                        const double* __restrict__ H, double* __restrict__ C, int M, int n_theta,
                                        int64_t N, int t, int m0, int64_t n0) {
  constexpr int BK = BK2;
  constexpr int LDA2 = BK2 + 4;
  constexpr int BN = W2 * NT * 8;
  constexpr int LDB = BN + 4;
  constexpr int BM = 8 * MT;
  constexpr int NTHR = W2 * 32;
  constexpr int ACH = BM * BK / 2;          // 16-byte chunks of an A tile
  constexpr int BCH = BK * BN / 2;          // 16-byte chunks of a B tile
  constexpr int AIT = (ACH + NTHR - 1) / NTHR;
  constexpr int BIT = BCH / NTHR;           // exact: 2048 / 256 = 8
  static_assert(BCH % NTHR == 0, "B tile split");
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int64_t ldh = (int64_t)n_theta * N;
  const double* At = A + (int64_t)t * M * M;
  const double* Bt = H + (int64_t)t * N;
  double* Ct = C + (int64_t)t * N;

  // per-thread copy descriptors (computed once)
  const double* asrc[AIT];
  int aoff[AIT];
  bool aok[AIT];
#pragma unroll
  for (int q = 0; q < AIT; ++q) {
    const int e = tid + q * NTHR;
    const int mm = e / (BK / 2), kk = (e % (BK / 2)) * 2;
    aok[q] = e < ACH && m0 + mm < M;
    asrc[q] = aok[q] ? At + (int64_t)(m0 + mm) * M + kk : At;
    aoff[q] = mm * LDA2 + kk;
  }
  const double* bsrc[BIT];
  int boff[BIT];
  bool bok[BIT];
#pragma unroll
  for (int q = 0; q < BIT; ++q) {
    const int e = tid + q * NTHR;
    const int kk = e / (BN / 2), nn = (e % (BN / 2)) * 2;
    bok[q] = n0 + nn < N;
    bsrc[q] = bok[q] ? Bt + (int64_t)kk * ldh + n0 + nn : Bt;
    boff[q] = kk * LDB + nn;
  }
  const int64_t bstep = (int64_t)BK * ldh;

  auto load_tile = [&](int stage, int kt) {
    double* as = &sm.a[stage][0][0];
    double* bs = &sm.b[stage][0][0];
#pragma unroll
    for (int q = 0; q < AIT; ++q)
      if (tid + q * NTHR < ACH) cp_async16(as + aoff[q], asrc[q] + kt * BK, aok[q]);
#pragma unroll
    for (int q = 0; q < BIT; ++q) cp_async16(bs + boff[q], bsrc[q] + kt * bstep, bok[q]);
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int ktiles = M / BK;
#pragma unroll
  for (int s = 0; s < STAGES2 - 1; ++s) {
    if (s < ktiles) load_tile(s, s);
    cp_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;
  const int wn = warp * NT * 8;
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_wait<STAGES2 - 2>();
    __syncthreads();
    const int st = kt % STAGES2;
    const double* as = &sm.a[st][0][0];
    const double* bs = &sm.b[st][0][0];
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double af[MT], bf[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) af[i] = as[(8 * i + fr) * LDA2 + k4 + fk];
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = bs[(k4 + fk) * LDB + wn + 8 * j + fr];
      if (k4 == 4) {  // issue the next tile's copies between DMMA groups
        const int nxt = kt + STAGES2 - 1;
        if (nxt < ktiles) load_tile(nxt % STAGES2, nxt);
        cp_commit();
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_wait<0>();
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int gi = m0 + 8 * i + fr;
    if (gi >= M) continue;
    double* crow = Ct + (int64_t)gi * ldh;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int64_t gn = n0 + wn + 8 * j + 2 * fk;
      if (gn < N) __stcs(reinterpret_cast<double2*>(crow + gn), make_double2(acc[i][j][0], acc[i][j][1]));
    }
  }
}

template <int MT, int BK2 = 16, int STAGES2 = 4, int W2 = WARPS, int MINB = 1>
__global__ void __launch_bounds__(W2 * 32, MINB)
    dgemm_theta_v2(const double* __restrict__ A, const double* __restrict__ H, double* __restrict__ C, int M,
                   int n_theta, int64_t N, int t_base) {
  using S = Smem2<MT, BK2, STAGES2, W2>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);
  v2_tile<MT, BK2, STAGES2, W2>(sm, A, H, C, M, n_theta, N, blockIdx.z + t_base, blockIdx.x * 8 * MT,
                                (int64_t)blockIdx.y * (W2 * NT * 8));
}

// fp64 recompute of the int8 collision's uncertified tiles (collision_i8.cu's
// certificate list: tile id = (theta * ncb + column block) * nib + row block, 64 x
// 128 tiles) with the DMMA tile above -- the same bits as the DMMA collision on
// those tiles; the CTAs exit at once when the list is empty.
__global__ void __launch_bounds__(4 * 32, 2)
    dgemm_fix_tiles(const double* __restrict__ A, const double* __restrict__ H, double* __restrict__ C, int M,
                    int n_theta, int64_t N, int ncb, int nib, const unsigned* __restrict__ list,
                    const unsigned* __restrict__ count, unsigned long long* fixed) {
  using S = Smem2<8, 16, 4, 4>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);
  const unsigned n = *count;
  if (blockIdx.x == 0 && threadIdx.x == 0 && n) atomicAdd(fixed, (unsigned long long)n);
  for (unsigned idx = blockIdx.x; idx < n; idx += gridDim.x) {
    const unsigned id = list[idx];
    const int ib = (int)(id % nib);
    const unsigned rest = id / nib;
    const int cb = (int)(rest % ncb), t = (int)(rest / ncb);
    __syncthreads();  // the previous tile's readers of the stage buffers are done
    v2_tile<8, 16, 4, 4>(sm, A, H, C, M, n_theta, N, t, ib * 64, (int64_t)cb * 128);
  }
}

template <int MT, int BK2 = 16, int STAGES2 = 4, int W2 = WARPS, int MINB = 1>
static int launch_v2(const double* A, const double* H, double* C, int M, int T, int64_t N, int t0, int t1,
                     cudaStream_t s) {
  const size_t smem = sizeof(Smem2<MT, BK2, STAGES2, W2>);
  static std::atomic<unsigned long long> attr_set{0};
  if (first_on_device(attr_set)) {
    GK_CUDA(cudaFuncSetAttribute(dgemm_theta_v2<MT, BK2, STAGES2, W2, MINB>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  dim3 grid((unsigned)cdiv(M, 8 * MT), (unsigned)cdiv(N, W2 * NT * 8), (unsigned)(t1 - t0));
  dgemm_theta_v2<MT, BK2, STAGES2, W2, MINB><<<grid, W2 * 32, smem, s>>>(A, H, C, M, T, N, t0);
  return check_launch("gk_collision");
}

template <int MT>
static int launch(const double* A, const double* H, double* C, int M, int T, int64_t N, int t0, int t1,
                  cudaStream_t s) {
  const size_t smem = sizeof(Smem<MT>);
  static std::atomic<unsigned long long> attr_set{0};
  if (first_on_device(attr_set)) {
    GK_CUDA(cudaFuncSetAttribute(dgemm_theta_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  }
  dim3 grid((unsigned)cdiv(M, 8 * MT), (unsigned)cdiv(N, BN), (unsigned)(t1 - t0));
  dgemm_theta_kernel<MT><<<grid, WARPS * 32, smem, s>>>(A, H, C, M, T, N, t0);
  return check_launch("gk_collision");
}

}  // namespace coll

// DMMA recompute of the listed 64 x 128 tiles (M % 16 == 0); the grid is sized for
// max_tiles (the CTAs exit when the list is empty).
int collision_fix_dmma(const double* A, const double* H, double* C, int M, int T, int64_t N, int ncb, int nib,
                       const unsigned* list, const unsigned* count, int64_t max_tiles, unsigned long long* fixed,
                       int sms, cudaStream_t s) {
  using namespace coll;
  const size_t smem = sizeof(Smem2<8, 16, 4, 4>);
  static std::atomic<unsigned long long> attr_set{0};
  if (first_on_device(attr_set))
    GK_CUDA(cudaFuncSetAttribute(dgemm_fix_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (int)std::min<int64_t>(max_tiles, 2 * (int64_t)sms);
  dgemm_fix_tiles<<<grid, 4 * 32, smem, s>>>(A, H, C, M, T, N, ncb, nib, list, count, fixed);
  return check_launch("gk_collision (fp64 DMMA recompute of uncertified tiles)");
}

bool collision_use_i8(int64_t M, int64_t N, int64_t T);
int collision_i8_range(const double* A, const double* H, double* C, int M, int T, int64_t N, int t0, int t1,
                       cudaStream_t st, const double* w = nullptr, double* phi = nullptr, void* scratch = nullptr,
                       bool reuse_a = false);
}  // namespace gk

extern "C" int gk_collision_range(const double* matrices, const double* h, double* out, int64_t n_vel,
                                  int64_t n_theta, int64_t n_cells, int64_t t0, int64_t t1, void* stream) {
  using namespace gk::coll;
  GK_CHECK_ARG(matrices && h && out, "gk_collision: null pointer");
  GK_CHECK_ARG(h != out, "gk_collision: in-place not supported");
  GK_CHECK_ARG(n_vel > 0 && n_vel < (1 << 20) && n_theta > 0 && n_theta < 65536 && n_cells > 0,
               "gk_collision: bad dims");
  GK_CHECK_ARG(0 <= t0 && t0 <= t1 && t1 <= n_theta, "gk_collision: bad theta range");
  if (t1 == t0) return GK_OK;
  const int M = (int)n_vel;
  const int64_t N = 2 * n_cells;
  GK_CHECK_ARG(gk::cdiv(N, BN) < 65536, "gk_collision: n_cells too large for the grid");
  cudaStream_t s = (cudaStream_t)stream;
  if (gk::collision_use_i8(M, N, n_theta)) return gk::collision_i8_range(matrices, h, out, M, (int)n_theta, N, (int)t0, (int)t1, s);
  // pick the M tile (8*MT rows) that wastes the fewest rows; prefer larger tiles.
  const int cands[4] = {8, 6, 4, 2};
  int best = 8;
  int64_t best_waste = -1;
  for (int c : cands) {
    const int64_t bm = 8 * c;
    const int64_t waste = gk::cdiv(M, bm) * bm - M;
    if (best_waste < 0 || waste < best_waste) {
      best = c;
      best_waste = waste;
    }
  }
  if (M % BK == 0) {
    // 4 warps x (MT x 4) DMMA tiles per CTA (BN = 128), two CTAs per SM: one CTA's
    // barrier / refill bubbles overlap the other's DMMA stream (measured 0.88 -> 0.94
    // of the DMMA probe at sh03b versus one 8-warp CTA per SM).
    switch (best) {
      case 8: return launch_v2<8, 16, 4, 4, 2>(matrices, h, out, M, (int)n_theta, N, (int)t0, (int)t1, s);
      case 6: return launch_v2<6, 16, 4, 4, 2>(matrices, h, out, M, (int)n_theta, N, (int)t0, (int)t1, s);
      case 4: return launch_v2<4, 16, 4, 4, 2>(matrices, h, out, M, (int)n_theta, N, (int)t0, (int)t1, s);
      default: return launch_v2<2, 16, 4, 4, 2>(matrices, h, out, M, (int)n_theta, N, (int)t0, (int)t1, s);
    }
  }
  switch (best) {
    case 8: return launch<8>(matrices, h, out, M, (int)n_theta, N, (int)t0, (int)t1, s);
    case 6: return launch<6>(matrices, h, out, M, (int)n_theta, N, (int)t0, (int)t1, s);
    case 4: return launch<4>(matrices, h, out, M, (int)n_theta, N, (int)t0, (int)t1, s);
    default: return launch<2>(matrices, h, out, M, (int)n_theta, N, (int)t0, (int)t1, s);
  }
}

extern "C" int gk_collision(const double* matrices, const double* h, double* out, int64_t n_vel, int64_t n_theta,
                            int64_t n_cells, void* stream) {
  return gk_collision_range(matrices, h, out, n_vel, n_theta, n_cells, 0, n_theta, stream);
}
