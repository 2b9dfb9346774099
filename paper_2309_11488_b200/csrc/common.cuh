// Shared device helpers for the B200 ILU0-BiCGStab path.
//
// Conventions used by every kernel in this library
//   * block-CSR pattern: int32 row pointers / column indices on the device
//     (the reference keeps int64, bs/blockcore.py:83-84; the C-ABI takes
//     int32 and the host layer narrows once per upload);
//   * block values: fp64, canonical BLOCK_ROW_MAJOR (each b*b block is b*b
//     consecutive doubles, row-major, bs/blockcore.py:26-44);
//   * block vectors: fp64, interleaved [row][b] (bs/blockcore.py:174-203);
//   * SELL-32 ("sliced ELL, 32 rows per slice") device layouts built once at
//     setup for the bandwidth-bound kernels: slice s covers rows
//     [32s, 32s+32); its width w_s is the longest selected row in the slice;
//     entry slot (s, k, lane) lives at  sp[s] + 32*k + lane  (cols, int32,
//     -1 = padding, padding always at the end of a row) and its b*b values
//     at  (sp[s] + 32*k)*b*b + 32*e + lane  (e = entry inside the block).
//     A warp reading one entry index k therefore loads 32 consecutive
//     doubles per instruction (256 B, fully coalesced).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "b200solve.h"  // status codes and the exported C ABI

#define B2S_CHECK(call)                                  \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return B2S_CUDA_ERROR;        \
  } while (0)

#define B2S_LAUNCH_CHECK()                               \
  do {                                                   \
    cudaError_t _e = cudaGetLastError();                 \
    if (_e != cudaSuccess) return B2S_CUDA_ERROR;        \
  } while (0)

namespace b2s {

// Programmatic dependent launch (PDL): a kernel launched with
// launch_k(..., pdl = true) may start while its predecessor's last CTAs
// still run; griddep_wait() (first thing in every such kernel, before any
// read of the predecessor's results) blocks until the predecessor finished
// and its writes are visible; griddep_launch() lets the successor be
// scheduled as soon as every CTA of this grid is running.  Both are no-ops
// for kernels launched without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? &attr : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

constexpr int kSlice = 32;          // rows per SELL slice == warp width
constexpr int kSms = 148;           // B200 SM count (grid sizing unit)

// "Not yet produced" marker for the sync-free triangular sweeps: a NaN with
// a payload no arithmetic produces (GPU arithmetic returns the canonical
// NaN).  Stored values are canonicalised so they can never alias it.
constexpr unsigned long long kSentinelBits = 0x7FF4B200DEC0DE01ull;

__device__ __forceinline__ double sentinel() {
  return __longlong_as_double((long long)kSentinelBits);
}
__device__ __forceinline__ bool is_sentinel(double v) {
  return (unsigned long long)__double_as_longlong(v) == kSentinelBits;
}
__device__ __forceinline__ double canon(double v) {
  return is_sentinel(v) ? __longlong_as_double(0x7FF8000000000000ll) : v;
}

// Relaxed, L1-bypassing accesses used for cross-CTA producer/consumer data.
__device__ __forceinline__ double ld_volatile(const double* p) {
  return *reinterpret_cast<const volatile double*>(p);
}
__device__ __forceinline__ void st_volatile(double* p, double v) {
  *reinterpret_cast<volatile double*>(p) = v;
}
__device__ __forceinline__ int ld_volatile(const int* p) {
  return *reinterpret_cast<const volatile int*>(p);
}
__device__ __forceinline__ void st_volatile(int* p, int v) {
  *reinterpret_cast<volatile int*>(p) = v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic CTA sum (fixed tree): every thread passes its value, thread 0
// gets the total.  `red` must hold blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    t = (l < nw) ? red[l] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

// y (B) = M (BxB row-major) * x (B)
template <int B>
__device__ __forceinline__ void matvec(const double* m, const double* x, double* y) {
#pragma unroll
  for (int a = 0; a < B; ++a) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < B; ++c) s = fma(m[a * B + c], x[c], s);
    y[a] = s;
  }
}

// C = A * B for BxB row-major blocks
template <int B>
__device__ __forceinline__ void matmul(const double* a, const double* b, double* c) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int j = 0; j < B; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < B; ++k) s = fma(a[i * B + k], b[k * B + j], s);
      c[i * B + j] = s;
    }
}

// Inverse of a BxB block by Gauss-Jordan elimination with partial pivoting
// (the LAPACK getrf/getri pivot rule numpy uses), plus the determinant from
// the same elimination (sign * prod of pivots, as numpy.linalg.det).  Returns
// false when the reference would raise SingularPivot: |det| < 1e-300,
// non-finite det, or a non-finite inverse (bs/ilu0.py:31-44).
template <int B>
__device__ __forceinline__ bool invert_block(const double* in, double* inv) {
  double a[B * B];
#pragma unroll
  for (int i = 0; i < B * B; ++i) a[i] = in[i];
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int j = 0; j < B; ++j) inv[i * B + j] = (i == j) ? 1.0 : 0.0;
  double det = 1.0;
#pragma unroll
  for (int col = 0; col < B; ++col) {
    int piv = col;
    double best = fabs(a[col * B + col]);
#pragma unroll
    for (int r = col + 1; r < B; ++r) {
      double v = fabs(a[r * B + col]);
      if (v > best) { best = v; piv = r; }
    }
    if (piv != col) {
      det = -det;
#pragma unroll
      for (int j = 0; j < B; ++j) {
        // predicated swap keeps everything in registers
#pragma unroll
        for (int r = col + 1; r < B; ++r) {
          if (r == piv) {
            double t = a[col * B + j]; a[col * B + j] = a[r * B + j]; a[r * B + j] = t;
            t = inv[col * B + j]; inv[col * B + j] = inv[r * B + j]; inv[r * B + j] = t;
          }
        }
      }
    }
    const double p = a[col * B + col];
    det *= p;
    const double rp = 1.0 / p;
#pragma unroll
    for (int j = 0; j < B; ++j) { a[col * B + j] *= rp; inv[col * B + j] *= rp; }
#pragma unroll
    for (int r = 0; r < B; ++r) {
      if (r == col) continue;
      const double f = a[r * B + col];
#pragma unroll
      for (int j = 0; j < B; ++j) {
        a[r * B + j] = fma(-f, a[col * B + j], a[r * B + j]);
        inv[r * B + j] = fma(-f, inv[col * B + j], inv[r * B + j]);
      }
    }
  }
  if (!isfinite(det) || fabs(det) < 1e-300) return false;
  bool ok = true;
#pragma unroll
  for (int i = 0; i < B * B; ++i) ok = ok && isfinite(inv[i]);
  return ok;
}

}  // namespace b2s
