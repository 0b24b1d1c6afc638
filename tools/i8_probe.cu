// tcgen05 kind::i8 probe: correctness of the K-major SWIZZLE_NONE operand
// layout / descriptors / TMEM readback against a CPU int GEMM, and MMA
// throughput (MAC per SM clock) for M = 128 and several N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_probe tools/i8_probe.cu && ./i8_probe
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int M = 128, K = 32;

// canonical K-major no-swizzle layout: (row, kbyte) -> g*SBO + c*LBO + r*16 + b
__host__ __device__ inline int koff(int row, int kb, int rows) {
  return (row >> 3) * 128 + (kb >> 4) * (rows / 8) * 128 + (row & 7) * 16 + (kb & 15);
}

__device__ inline uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4)       // D = S32
         | (1u << 7)     // A = signed int8
         | (1u << 10)    // B = signed int8
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int N>
__global__ void __launch_bounds__(128, 1) probe(const int8_t* A, const int8_t* B, int* D, int reps,
                                                long long* cycles) {
  __shared__ __align__(1024) int8_t sa[M * K];
  __shared__ __align__(1024) int8_t sb[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) sa[koff(i / K, i % K, M)] = A[i];
  for (int i = tid; i < N * K; i += blockDim.x) sb[koff(i / K, i % K, N)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint64_t da = sdesc((uint32_t)__cvta_generic_to_shared(sa), (M / 8) * 128, 128);
    const uint64_t db = sdesc((uint32_t)__cvta_generic_to_shared(sb), (N / 8) * 128, 128);
    constexpr uint32_t id = idesc_i8(M, N);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t acc = r > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
          "l"(da), "l"(db), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&mbar)));
    asm volatile(
        "{\n.reg .pred P1;\nWAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra WAIT;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    cycles[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // warp w reads lanes 32w..32w+31, 8 columns at a time
  if (blockIdx.x == 0) {
    for (int c = 0; c < N; c += 8) {
      uint32_t v[8];
      const uint32_t addr = tm + ((uint32_t)(warp * 32) << 16) + c;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                     "=r"(v[7])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 8; ++j) D[(warp * 32 + lane) * N + c + j] = (int)v[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
}

template <int N>
void run(int reps, int blocks) {
  std::vector<int8_t> A(M * K), B(N * K);
  for (auto& x : A) x = (int8_t)(rand() % 129 - 64);
  for (auto& x : B) x = (int8_t)(rand() % 129 - 64);
  int8_t *dA, *dB;
  int* dD;
  long long* dc;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMalloc(&dc, blocks * 8));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  probe<N><<<blocks, 128>>>(dA, dB, dD, reps, dc);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int> D(M * N);
  std::vector<long long> cyc(blocks);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cyc.data(), dc, blocks * 8, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += (long)A[i * K + k] * B[j * K + k];
      s *= reps;
      if (s != D[i * N + j]) {
        if (bad < 4) printf("  mismatch (%d,%d): gpu %d cpu %ld\n", i, j, D[i * N + j], s);
        ++bad;
      }
    }
  const double mac = (double)M * N * K * reps;
  printf("N=%3d reps=%d blocks=%d: %s, %.0f MAC/clk/SM (cycles %lld)\n", N, reps, blocks, bad ? "WRONG" : "exact",
         mac / cyc[0], cyc[0]);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  cudaFree(dc);
}

// TS variant: A (M = 128 rows x K = 32 bytes) copied smem -> TMEM with
// tcgen05.cp 128x256b, then MMAs with A from TMEM.  NB distinct B tiles and NA
// distinct TMEM A copies are cycled through to defeat any operand reuse.
template <int N, int NA, int NB>
__global__ void __launch_bounds__(128, 1) probe_ts(const int8_t* A, const int8_t* B, int* D, int reps,
                                                   long long* cycles) {
  extern __shared__ __align__(1024) int8_t dsm[];
  int8_t* sa = dsm;               // NA tiles of M*K
  int8_t* sb = dsm + NA * M * K;  // NB tiles of N*K
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int t = 0; t < NA; ++t)
    for (int i = tid; i < M * K; i += blockDim.x) sa[t * M * K + koff(i / K, i % K, M)] = A[i];
  for (int t = 0; t < NB; ++t)
    for (int i = tid; i < N * K; i += blockDim.x) sb[t * N * K + koff(i / K, i % K, N)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t ta = tm + 256;  // A copies at columns 256 + 8 t
  if (tid == 0) {
    for (int t = 0; t < NA; ++t) {
      const uint64_t da = sdesc((uint32_t)__cvta_generic_to_shared(sa + t * M * K), (M / 8) * 128, 128);
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(ta + 8 * t), "l"(da));
    }
    constexpr uint32_t id = idesc_i8(M, N);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t acc = r > 0;
      const uint64_t db = sdesc((uint32_t)__cvta_generic_to_shared(sb + (r % NB) * N * K), (N / 8) * 128, 128);
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm),
          "r"(ta + 8 * (r % NA)), "l"(db), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&mbar)));
    asm volatile(
        "{\n.reg .pred P1;\nWAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra WAIT;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    cycles[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (blockIdx.x == 0) {
    for (int c = 0; c < N; c += 8) {
      uint32_t v[8];
      const uint32_t addr = tm + ((uint32_t)(warp * 32) << 16) + c;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                     "=r"(v[7])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 8; ++j) D[(warp * 32 + lane) * N + c + j] = (int)v[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
}

template <int N, int NA, int NB>
void run_ts(int reps, int blocks) {
  std::vector<int8_t> A(M * K), B(N * K);
  for (auto& x : A) x = (int8_t)(rand() % 256 - 128);
  for (auto& x : B) x = (int8_t)(rand() % 256 - 128);
  int8_t *dA, *dB;
  int* dD;
  long long* dc;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMalloc(&dc, blocks * 8));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  const size_t smem = (size_t)NA * M * K + (size_t)NB * N * K;
  CK(cudaFuncSetAttribute(probe_ts<N, NA, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  probe_ts<N, NA, NB><<<blocks, 128, 100 * 1024>>>(dA, dB, dD, reps, dc);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int> D(M * N);
  std::vector<long long> cyc(blocks);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cyc.data(), dc, blocks * 8, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += (long)A[i * K + k] * B[j * K + k];
      s *= reps;
      if (s != D[i * N + j]) {
        if (bad < 4) printf("  mismatch (%d,%d): gpu %d cpu %ld\n", i, j, D[i * N + j], s);
        ++bad;
      }
    }
  const double mac = (double)M * N * K * reps;
  printf("TS N=%3d NA=%d NB=%d reps=%d: %s, %.0f MAC/clk/SM (smem %zu)\n", N, NA, NB, reps,
         bad ? "WRONG" : "exact", mac / cyc[0], smem);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  cudaFree(dc);
}

int main() {
  run_ts<64, 1, 1>(1, 1);
  run_ts<64, 6, 6>(6, 1);
  run_ts<64, 6, 6>(4098, 148);
  run_ts<128, 3, 3>(4098, 148);
  run<64>(1, 1);
  run<64>(4096, 148);
  run<128>(4096, 148);
  run<256>(4096, 148);
  run<32>(4096, 148);
  return 0;
}
