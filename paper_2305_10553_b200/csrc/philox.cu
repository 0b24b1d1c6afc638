// On-device Philox4x64-10, bit-exact with the reference's input generator
// (grid.py:122-161: numpy.random.Philox(key=seed).jumped(stream) and
// Generator.uniform), so em04b/C5-sized states -- which the host cannot even
// hold -- are generated where they live.
//
// numpy's Philox4x64: key = (seed, 0); a jump adds 1 to counter word 2; every
// 4-output block first increments the 256-bit counter, then applies 10 rounds.
// Raw output r is word r%4 of block r/4, i.e. counter = (r/4 + 1, 0, stream, 0).
// uniform(low, high) = low + (high - low) * ((raw >> 11) * 2^-53).
#include "gk_common.cuh"
#include "../../include/gk.h"

namespace gk {
namespace rng {

__device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = M0 * c[0], hi0 = __umul64hi(M0, c[0]);
    const uint64_t lo1 = M1 * c[2], hi1 = __umul64hi(M1, c[2]);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += W0;
    k1 += W1;
  }
}

// one thread per 4-output block covering raw indices [offset, offset + count)
__global__ void uniform_kernel(uint64_t seed, uint64_t stream, int64_t offset, int64_t count, double low,
                               double range, double* __restrict__ out, int64_t stride) {
  const int64_t first_block = offset >> 2;
  const int64_t last_block = (offset + count - 1) >> 2;
  for (int64_t b = first_block + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= last_block;
       b += (int64_t)gridDim.x * blockDim.x) {
    // counter = b + 1 as a 128-bit value in words (0, 1), stream in word 2
    const uint64_t lo = (uint64_t)b + 1;
    uint64_t c[4] = {lo, lo == 0 ? 1ull : 0ull, stream, 0};
    philox4x64_10(c, seed, 0);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int64_t r = b * 4 + w;
      if (r < offset || r >= offset + count) continue;
      const double d = (double)(c[w] >> 11) * (1.0 / 9007199254740992.0);
      out[(r - offset) * stride] = __dadd_rn(low, __dmul_rn(range, d));
    }
  }
}

// out[(row * row_len + j) * stride] = uniform(raw[offset + row * row_stride + j]):
// a strided sub-block of the stream (one rank's toroidal shard of a state), one
// thread per output, each computing its own 4-output Philox block.
__global__ void uniform_rows_kernel(uint64_t seed, uint64_t stream, int64_t offset, int64_t n_rows, int64_t row_len,
                                    int64_t row_stride, double low, double range, double* __restrict__ out,
                                    int64_t stride) {
  const int64_t n = n_rows * row_len;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / row_len, j = i - row * row_len;
    const int64_t r = offset + row * row_stride + j;
    const uint64_t lo = (uint64_t)(r >> 2) + 1;
    uint64_t c[4] = {lo, lo == 0 ? 1ull : 0ull, stream, 0};
    philox4x64_10(c, seed, 0);
    const uint64_t w = (r & 3) == 0 ? c[0] : (r & 3) == 1 ? c[1] : (r & 3) == 2 ? c[2] : c[3];
    const double d = (double)(w >> 11) * (1.0 / 9007199254740992.0);
    out[i * stride] = __dadd_rn(low, __dmul_rn(range, d));
  }
}

}  // namespace rng
}  // namespace gk

extern "C" int gk_philox_uniform_rows(uint64_t seed, uint64_t stream_id, int64_t offset, int64_t n_rows,
                                      int64_t row_len, int64_t row_stride, double low, double high, double* out,
                                      int64_t out_stride, void* stream) {
  GK_CHECK_ARG(out && offset >= 0 && n_rows >= 0 && row_len >= 0 && row_stride >= row_len && out_stride >= 1,
               "gk_philox_uniform_rows: bad arguments");
  const int64_t n = n_rows * row_len;
  if (n == 0) return GK_OK;
  int64_t grid = (n + 255) / 256;
  if (grid > 148 * 32) grid = 148 * 32;
  gk::rng::uniform_rows_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      seed, stream_id, offset, n_rows, row_len, row_stride, low, high - low, out, out_stride);
  return gk::check_launch("gk_philox_uniform_rows");
}

extern "C" int gk_philox_uniform(uint64_t seed, uint64_t stream_id, int64_t offset, int64_t count, double low,
                                 double high, double* out, int64_t out_stride, void* stream) {
  GK_CHECK_ARG(out && offset >= 0 && count >= 0 && out_stride >= 1, "gk_philox_uniform: bad arguments");
  if (count == 0) return GK_OK;
  const int64_t blocks = ((offset + count - 1) >> 2) - (offset >> 2) + 1;
  int64_t grid = (blocks + 255) / 256;
  if (grid > 148 * 32) grid = 148 * 32;
  gk::rng::uniform_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(seed, stream_id, offset, count, low,
                                                                            high - low, out, out_stride);
  return gk::check_launch("gk_philox_uniform");
}
