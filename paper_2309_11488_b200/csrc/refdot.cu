// Inner products in the reference's exact summation order (bs/krylov.py:30-47).
//
// The reference forms prod = a*b, sums each 64-element chunk with
// np.add.reduceat and accumulates the chunk partials strictly left to right
// (np.cumsum).  numpy's reduceat seeds a chunk with its first element and adds
// the rest through the float64 add loop in binary-reduce mode, i.e.
//   part = prod[s] + pairwise(prod[s+1 .. e))
// where numpy's pairwise sum of n < 8 values is -0.0 + v0 + v1 + ... in
// order, and of 8 <= n <= 128 values keeps eight strided accumulators
// r[j] = v[j] + v[j+8] + ..., combines them as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and adds the n%8 tail in order
// (numpy/_core/src/umath/loops_utils.h.src, pairwise_sum).  A chunk has at
// most 63 values after its seed, so the recursive case never occurs.
//
// Every product and sum is an explicitly rounded __dmul_rn/__dadd_rn, so no
// FMA contraction can change a bit: the partials and the total equal the
// reference's exactly.  This path serves the public dot/norm/dot_partials API
// and the reported initial residual norm; the Krylov loop keeps its own
// fixed-order per-CTA reduction (csrc/krylov.cu, k_dot_parts).
#include "common.cuh"

namespace b2s {

constexpr int kChunk = 64;   // bs/krylov.py:24 REDUCTION_CHUNK

__device__ __forceinline__ double prod_at(const double* a, const double* b, long long i) {
  return __dmul_rn(a[i], b[i]);
}

// one thread per chunk (the values of a chunk are read through L1: a warp's
// 32 chunks are 2 x 16 KB of contiguous memory)
__global__ void k_chunk_partials(long long m, const double* __restrict__ a,
                                 const double* __restrict__ b, double* __restrict__ parts) {
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long nchunks = (m + kChunk - 1) / kChunk;
  if (c >= nchunks) return;
  long long s = c * kChunk;
  long long e = s + kChunk < m ? s + kChunk : m;
  double seed = prod_at(a, b, s);
  long long n = e - s - 1;                 // values after the seed
  const long long v0 = s + 1;
  double rest;
  if (n < 8) {
    rest = -0.0;
    for (long long i = 0; i < n; ++i) rest = __dadd_rn(rest, prod_at(a, b, v0 + i));
  } else {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = prod_at(a, b, v0 + j);
    long long i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], prod_at(a, b, v0 + i + j));
    }
    rest = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                     __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) rest = __dadd_rn(rest, prod_at(a, b, v0 + i));
  }
  parts[c] = n > 0 ? __dadd_rn(seed, rest) : seed;
}

// np.cumsum(partials)[-1]: one strictly sequential chain.  A single warp
// stages 32 partials per step so the loads run ahead of the add chain; lane 0
// performs every addition in order.
__global__ void k_sequential_total(const double* __restrict__ parts, long long np,
                                   double* __restrict__ out) {
  const int lane = threadIdx.x;
  double acc = 0.0;
  for (long long base = 0; base < np; base += 32) {
    double v = base + lane < np ? parts[base + lane] : 0.0;
    const int cnt = np - base < 32 ? (int)(np - base) : 32;
    for (int k = 0; k < cnt; ++k) {
      double pk = __shfl_sync(0xffffffffu, v, k);
      if (lane == 0) acc = (base == 0 && k == 0) ? pk : __dadd_rn(acc, pk);
    }
  }
  if (lane == 0) *out = np > 0 ? acc : 0.0;
}

}  // namespace b2s

using namespace b2s;

int b2s_dot_chunked(long long m, const double* a, const double* b, double* parts, double* total,
                    cudaStream_t st) {
  if (m < 0) return B2S_SHAPE;
  long long np = (m + kChunk - 1) / kChunk;
  if (np > 0) {
    const int threads = 128;
    k_chunk_partials<<<(unsigned)((np + threads - 1) / threads), threads, 0, st>>>(m, a, b, parts);
  }
  if (total != nullptr) k_sequential_total<<<1, 32, 0, st>>>(parts, np, total);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}
