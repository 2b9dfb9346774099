// SELL-32 device layout descriptors shared by SpMV, ILU0 and the Krylov loop.
#pragma once
#include "common.cuh"

namespace b2s {

// A "slice map" assigns each SELL slice a contiguous run of at most 32 rows.
// Plain maps cover rows [32s, 32s+32); group-aligned maps (used for the
// level / colour plans) never let a slice cross a group boundary, so the
// rows of one slice never depend on each other in a triangular sweep.
struct SliceMap {
  int nslices;
  const int32_t* row0;   // first row of slice s
  const int32_t* nrows;  // rows in slice s (1..32)
};

// One SELL-32 matrix on a slice map.  Slot (s, k, lane) lives at
// sp[s] + 32k + lane; its b*b values at (sp[s] + 32k)*b*b + 32e + lane.
struct Sell {
  const int32_t* sp;    // [nslices+1] slot offsets (multiples of 32)
  const int32_t* cols;  // [slots], -1 = padding (always at the end of a row)
  const double* vals;   // [slots*b*b]
};

// Separately applied wells inside the device loop (b2s_bicg_args.wells):
// corr[q] = sum over the wells perforating compact cell q of C^T D^-1 B x
// (csrc/wells.cu, computed right before the SpMV); the SpMV subtracts it
// from the row sum before its dot-product epilogue.  slice[s] = base of
// slice s's 32 lane entries in lane[] or -1 (no perforated row in the slice);
// lane[base + l] = compact cell index of row row0[s] + l, or -1.
struct WellFix {
  const int32_t* slice;
  const int32_t* lane;
  const double* corr;
};

// s-image with separately applied wells (fused.cu): the wells patch of
// v's colour-0 rows recomputes u = inv(A_ii) v at the patched rows
struct SImgPatch {
  double* u;              // nullptr: no s-image
  const int32_t* row0;    // slice map (group-aligned, row0 ascending)
  int nslices;
  const double* dtiles;   // inverse diagonal tiles by slice
};

// SpMV epilogues: 0 y = A x; 1 + partials w.y; 2 + partials y.y and y.w;
// 3 y = w - A x (residual) + partials y.y
enum SpmvMode { kPlain = 0, kDotW = 1, kSelfAndW = 2, kResidual = 3 };

__device__ __forceinline__ long long vidx(long long slot0, int k, int e, int lane, int bb) {
  // value index of entry (k, e) of the lane in the slice starting at slot0
  return (slot0 + 32ll * k) * bb + 32ll * e + lane;
}

// L2 prefetch of one slice's SELL entries (column indices + block values).
// They are setup data, so a kernel may issue it BEFORE griddep_wait(): its
// first slice then streams in while the predecessor's last CTAs drain (one
// bulk prefetch per array, issued by one lane).  B2S_PREWAIT=0 at compile
// time leaves it out (A/B builds).
#ifndef B2S_PREWAIT
#define B2S_PREWAIT 1
#endif
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
template <int BB>
__device__ __forceinline__ void prefetch_slice(const Sell& a, int s, const double* tiles = nullptr) {
  if (!B2S_PREWAIT) return;
  const int slot0 = a.sp[s], n = a.sp[s + 1] - slot0;
  if (n > 0) {
    prefetch_l2(a.vals + (long long)slot0 * BB, (unsigned)n * BB * 8u);
    prefetch_l2(a.cols + slot0, (unsigned)n * 4u);
  }
  if (tiles) prefetch_l2(tiles + (long long)s * BB * 32, BB * 32 * 8u);
}

}  // namespace b2s
