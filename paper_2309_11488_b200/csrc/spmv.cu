// SELL-32 construction and the BSR SpMV (bs/blockcore.py:342-376).
//
// SpMV is HBM-bound (0.2 flop/B): per block row it streams the row's blocks
// (72 B each for b = 3) and column indices once, gathers x (L2-resident: the
// whole x of a 1M-cell system is 24 MB against a 126 MB L2) and writes y.
// One thread owns one block row; a warp owns one 32-row slice, so every
// value/column load instruction of the warp reads 32 consecutive 8-byte
// words.  Values and columns are loaded with the streaming (evict-first)
// hint so the matrix does not push the vectors out of L2.  Each row sums
// its block products in ascending column order, like np.add.reduceat.
//
// Optional fused epilogues produce the per-CTA partial sums of the dot
// products BiCGStab needs right after an operator application, so those
// vectors are never re-read: gamma = rhat.v, (t.t, t.s), and the residual
// norm.  Partials are reduced in a fixed order (no atomics): deterministic.
#include <cub/cub.cuh>

#include "ctl.cuh"
#include "sell.cuh"

namespace b2s {

__device__ __forceinline__ bool row_selected(int sel, int row, int c) {
  return sel == 0 || (sel == 1 && c < row) || (sel == 2 && c > row);
}

__global__ void k_plain_slices(int n, int nslices, int32_t* row0, int32_t* nrows) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nslices; s += gridDim.x * blockDim.x) {
    row0[s] = s * kSlice;
    nrows[s] = min(kSlice, n - s * kSlice);
  }
}

__global__ void k_group_slice_counts(int ngroups, const int32_t* __restrict__ off, int32_t* cnt) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += gridDim.x * blockDim.x)
    cnt[g] = (off[g + 1] - off[g] + kSlice - 1) / kSlice;
}

__global__ void k_group_slices(int ngroups, int nslices, const int32_t* __restrict__ off,
                               const int32_t* __restrict__ base, int32_t* row0,
                               int32_t* nrows) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nslices; s += gridDim.x * blockDim.x) {
    int lo = 0, hi = ngroups - 1;  // last g with base[g] <= s
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (base[mid] <= s) lo = mid; else hi = mid - 1;
    }
    const int r0 = off[lo] + (s - base[lo]) * kSlice;
    row0[s] = r0;
    nrows[s] = min(kSlice, off[lo + 1] - r0);
  }
}

// slots of slice s = 32 * longest selected row of the slice
__global__ void k_sell_width(int nslices, const int32_t* __restrict__ row0,
                             const int32_t* __restrict__ nrows, const int32_t* __restrict__ rp,
                             const int32_t* __restrict__ ci, int sel, int32_t* slots) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nslices; s += nw) {
    int cnt = 0;
    if (lane < nrows[s]) {
      const int row = row0[s] + lane;
      if (sel == 0) {
        cnt = rp[row + 1] - rp[row];
      } else {
        for (int q = rp[row]; q < rp[row + 1]; ++q) cnt += row_selected(sel, row, ci[q]) ? 1 : 0;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt = max(cnt, __shfl_xor_sync(0xffffffffu, cnt, o));
    if (lane == 0) slots[s] = cnt * kSlice;
  }
}

// group of a plan-order row: last g with goff[g] <= row
__device__ __forceinline__ int group_of(const int32_t* goff, int ngroups, int row) {
  int lo = 0, hi = ngroups - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (goff[mid] <= row) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void k_sell_fill(int nslices, int bb, const int32_t* __restrict__ row0,
                            const int32_t* __restrict__ nrows, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, const double* __restrict__ vals,
                            int sel, const int32_t* __restrict__ sp,
                            const int32_t* __restrict__ goff, int ngroups,
                            int32_t* __restrict__ ocols,
                            double* __restrict__ ovals, const int32_t* __restrict__ src) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nslices; s += nw) {
    const long long slot0 = sp[s];
    const int width = (sp[s + 1] - sp[s]) / kSlice;
    int k = 0;
    if (lane < nrows[s]) {
      const int row = row0[s] + lane;
      for (int q = rp[row]; q < rp[row + 1]; ++q) {
        const int c = ci[q];
        if (!row_selected(sel, row, c)) continue;
        // same-group entries of a triangular factor read the value the
        // vector had *before* the sweep (the reference updates a whole group
        // at once, bs/ilu0.py:125-142): encode them as -(c + 2)
        const bool stale = goff != nullptr && group_of(goff, ngroups, c) == group_of(goff, ngroups, row);
        ocols[slot0 + 32ll * k + lane] = stale ? -(c + 2) : c;
        // values of slot q, or of input slot src[q] (straight from the
        // unpermuted matrix: the plan-order CSR values are never built)
        const long long qv = src ? src[q] : q;
        for (int e = 0; e < bb; ++e) ovals[vidx(slot0, k, e, lane, bb)] = vals[qv * bb + e];
        ++k;
      }
    }
    for (; k < width; ++k) {
      ocols[slot0 + 32ll * k + lane] = -1;
      for (int e = 0; e < bb; ++e) ovals[vidx(slot0, k, e, lane, bb)] = 0.0;
    }
  }
}

// sel 0 (every block): the k-th slot of a row is its k-th CSR entry, so each
// (slice, k, lane) is independent -- one thread per slot, all loads of the
// pass in flight at once (the sequential per-row loop above waits on a
// dependent index -> value chain per entry).  CTA = 32 lanes x 8 slots of a
// slice; wider slices loop.
template <int BB>
__global__ void __launch_bounds__(256) k_sell_fill_all(int nslices, const int32_t* __restrict__ row0,
                                                       const int32_t* __restrict__ nrows,
                                                       const int32_t* __restrict__ rp,
                                                       const int32_t* __restrict__ ci,
                                                       const double* __restrict__ vals,
                                                       const int32_t* __restrict__ sp,
                                                       int32_t* __restrict__ ocols,
                                                       double* __restrict__ ovals,
                                                       const int32_t* __restrict__ src) {
  const int lane = threadIdx.x & 31;
  for (int s = blockIdx.x; s < nslices; s += gridDim.x) {
    const long long slot0 = sp[s];
    const int width = (sp[s + 1] - sp[s]) / kSlice;
    const bool live = lane < nrows[s];
    const int row = row0[s] + lane;
    const int q0 = live ? rp[row] : 0, len = live ? rp[row + 1] - q0 : 0;
    for (int k = threadIdx.x >> 5; k < width; k += blockDim.x >> 5) {
      double v[BB];
      int c = -1;
      if (k < len) {
        const int q = q0 + k;
        c = ci[q];
        const long long qv = src ? src[q] : q;
#pragma unroll
        for (int e = 0; e < BB; ++e) v[e] = vals[qv * BB + e];
      } else {
#pragma unroll
        for (int e = 0; e < BB; ++e) v[e] = 0.0;
      }
      ocols[slot0 + 32ll * k + lane] = c;
#pragma unroll
      for (int e = 0; e < BB; ++e) ovals[vidx(slot0, k, e, lane, BB)] = v[e];
    }
  }
}

// per-slice b*b x 32 tiles of the inverse diagonal (row order of the map)
__global__ void k_diag_tiles(int nslices, int bb, const int32_t* __restrict__ row0,
                             const int32_t* __restrict__ nrows, const double* __restrict__ inv,
                             double* __restrict__ tiles) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nslices; s += nw) {
    const bool ok = lane < nrows[s];
    const long long row = (long long)row0[s] + lane;
    for (int e = 0; e < bb; ++e)
      tiles[((long long)s * bb + e) * 32 + lane] = ok ? inv[row * bb + e] : 0.0;
  }
}


#ifndef B2S_SPMV_CTAS
#define B2S_SPMV_CTAS 2
#endif
template <int B, int MODE, bool WELLS>
__global__ void __launch_bounds__(256, B <= 3 ? B2S_SPMV_CTAS : 1) k_spmv(SliceMap map, int s0, int s1, int poff, Sell a,
                                              const double* __restrict__ x,
                                              double* __restrict__ y,
                                              const double* __restrict__ w,
                                              double* __restrict__ part0,
                                              double* __restrict__ part1, const int* done,
                                              Ctl ctl, WellFix wf, int ptotal) {
  constexpr int BB = B * B;
  __shared__ double red[8];
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  if (lane == 0 && s0 + gw < s1) prefetch_slice<BB>(a, s0 + gw);
  griddep_wait();
  griddep_launch();
  if (done && *done) return;
  double p0 = 0.0, p1 = 0.0;
  // the column indices of the next entry pair load one step ahead -- across
  // slice boundaries too: a slice's last step fetches the next slice's first
  // pair -- so a step's x gathers never wait behind their own index loads
  int nslot0 = 0, nwidth = 0, cn0 = -1, cn1 = -1;
  if (s0 + gw < s1) {
    nslot0 = a.sp[s0 + gw];
    nwidth = (a.sp[s0 + gw + 1] - nslot0) >> 5;
    cn0 = nwidth > 0 ? __ldcs(a.cols + nslot0 + lane) : -1;
    cn1 = nwidth > 1 ? __ldcs(a.cols + nslot0 + 32 + lane) : -1;
  }
  for (int s = s0 + gw; s < s1; s += nw) {
    const int slot0 = nslot0;
    const int width = nwidth;
    const bool more = s + nw < s1;
    if (more) {
      nslot0 = a.sp[s + nw];
      nwidth = (a.sp[s + nw + 1] - nslot0) >> 5;
    }
    const bool ok = lane < map.nrows[s];
    const long long row = (long long)map.row0[s] + lane;
    double acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) acc[c] = 0.0;
    // two entries per step, all loads of the pair issued before any math
    if (width == 0) {   // no step to fetch the next slice's first pair in
      cn0 = more && nwidth > 0 ? __ldcs(a.cols + nslot0 + lane) : -1;
      cn1 = more && nwidth > 1 ? __ldcs(a.cols + nslot0 + 32 + lane) : -1;
    }
    for (int k = 0; k < width; k += 2) {
      const bool two = k + 1 < width;
      int col[2] = {cn0, cn1};
      if (k + 2 < width) {
        cn0 = __ldcs(a.cols + slot0 + 32 * (k + 2) + lane);
        cn1 = k + 3 < width ? __ldcs(a.cols + slot0 + 32 * (k + 3) + lane) : -1;
      } else {
        cn0 = more && nwidth > 0 ? __ldcs(a.cols + nslot0 + lane) : -1;
        cn1 = more && nwidth > 1 ? __ldcs(a.cols + nslot0 + 32 + lane) : -1;
      }
      double blk[2][BB], xv[2][B];
#pragma unroll
      for (int e = 0; e < BB; ++e) {
        blk[0][e] = __ldcs(a.vals + vidx(slot0, k, e, lane, BB));
        blk[1][e] = two ? __ldcs(a.vals + vidx(slot0, k + 1, e, lane, BB)) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const long long cq = col[q] < 0 ? 0 : col[q];
#pragma unroll
        for (int c = 0; c < B; ++c) xv[q][c] = __ldg(x + cq * B + c);
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (col[q] >= 0) {   // ascending columns, padding contributes nothing
          double pr[B];
          matvec<B>(blk[q], xv[q], pr);
#pragma unroll
          for (int c = 0; c < B; ++c) acc[c] += pr[c];
        }
      }
    }
    if (WELLS) {   // the operator's well terms (bs/krylov.py:84-94), before the epilogue
      const int wb = wf.slice[s];
      if (wb >= 0) {
        const int q = wf.lane[wb + lane];
        if (ok && q >= 0) {
#pragma unroll
          for (int c = 0; c < B; ++c) acc[c] -= wf.corr[(long long)q * B + c];
        }
      }
    }
    if (ok) {
#pragma unroll
      for (int c = 0; c < B; ++c) {
        double v = acc[c];
        if (MODE == kResidual) v = w[row * B + c] - v;
        y[row * B + c] = v;
        if (MODE == kDotW) p0 = fma(w[row * B + c], v, p0);
        if (MODE == kSelfAndW) { p0 = fma(v, v, p0); p1 = fma(v, w[row * B + c], p1); }
        if (MODE == kResidual) p0 = fma(v, v, p0);
      }
    }
  }
  if (MODE != kPlain) {
    // a grid capped at one resident wave leaves the caller's slots
    // [gridDim.x, ptotal) unwritten: zeros, so every consumer's fixed-order
    // reduction over ptotal slots stays valid
    if (blockIdx.x == 0)
      for (int q = gridDim.x + threadIdx.x; q < ptotal; q += blockDim.x) {
        part0[poff + q] = 0.0;
        if (MODE == kSelfAndW) part1[poff + q] = 0.0;
      }
    double t0 = block_sum(p0, red);
    if (threadIdx.x == 0) part0[poff + blockIdx.x] = t0;
    if (MODE == kSelfAndW) {
      double t1 = block_sum(p1, red);
      if (threadIdx.x == 0) part1[poff + blockIdx.x] = t1;
    }
    // the last CTA to finish reduces the partials (those of an earlier
    // kernel first, when poff > 0) and runs the solver's scalar step
    // (alpha after gamma, omega after tt/ts)
    if (ctl.st && last_cta(ctl.counter)) ctl_run(ctl, part0, part1, poff + gridDim.x, red);
  }
}

inline int grid_for(long long work, int threads = 256) {
  long long g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > kSms * 32) g = kSms * 32;
  return (int)g;
}

template <int B, bool WELLS>
int launch_spmv_bw(int mode, int nparts, SliceMap map, int s0, int s1, int poff, Sell a,
                   const double* x, double* y, const double* w, double* p0, double* p1,
                   const int* done, Ctl ctl, cudaStream_t st, bool pdl, WellFix wf) {
  dim3 g(nparts), t(256);
#if B2S_SPMV_CTAS < 4
  // one resident wave: 2 CTAs per SM without the 64-register cap measured
  // faster than 4 capped ones (C4 SpMV 90.4 -> 87.7 us, colour-1 SpMV in the
  // loop 60.3 -> 57.3 us; profiles/r02/simg.txt)
  {
    static int cap = 0;
    if (!cap) {
      int per_sm = 1, dev = 0, sms = kSms;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv<B, kDotW, WELLS>, 256, 0);
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cap = (per_sm < 1 ? 1 : per_sm) * sms;
    }
    if ((int)g.x > cap) g.x = cap;
  }
#endif
  switch (mode) {
    case kPlain: launch_k(k_spmv<B, kPlain, WELLS>, g, t, 0, st, pdl, map, s0, s1, poff, a, x, y, w, p0, p1, done, ctl, wf, nparts); break;
    case kDotW: launch_k(k_spmv<B, kDotW, WELLS>, g, t, 0, st, pdl, map, s0, s1, poff, a, x, y, w, p0, p1, done, ctl, wf, nparts); break;
    case kSelfAndW: launch_k(k_spmv<B, kSelfAndW, WELLS>, g, t, 0, st, pdl, map, s0, s1, poff, a, x, y, w, p0, p1, done, ctl, wf, nparts); break;
    case kResidual: launch_k(k_spmv<B, kResidual, WELLS>, g, t, 0, st, pdl, map, s0, s1, poff, a, x, y, w, p0, p1, done, ctl, wf, nparts); break;
    default: return B2S_SHAPE;
  }
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

template <int B>
int launch_spmv_b(int mode, int nparts, SliceMap map, int s0, int s1, int poff, Sell a,
                  const double* x, double* y, const double* w, double* p0, double* p1,
                  const int* done, Ctl ctl, cudaStream_t st, bool pdl, WellFix wf) {
  if (wf.slice)
    return launch_spmv_bw<B, true>(mode, nparts, map, s0, s1, poff, a, x, y, w, p0, p1, done, ctl,
                                   st, pdl, wf);
  return launch_spmv_bw<B, false>(mode, nparts, map, s0, s1, poff, a, x, y, w, p0, p1, done, ctl,
                                  st, pdl, wf);
}

// SpMV over slices [s0, s1) of the map; partials land at [poff, poff + nparts)
int launch_spmv_range(int b, int mode, int nparts, SliceMap map, int s0, int s1, int poff, Sell a,
                      const double* x, double* y, const double* w, double* p0, double* p1,
                      const int* done, Ctl ctl, cudaStream_t st, bool pdl, WellFix wf) {
  switch (b) {
    case 1: return launch_spmv_b<1>(mode, nparts, map, s0, s1, poff, a, x, y, w, p0, p1, done, ctl, st, pdl, wf);
    case 2: return launch_spmv_b<2>(mode, nparts, map, s0, s1, poff, a, x, y, w, p0, p1, done, ctl, st, pdl, wf);
    case 3: return launch_spmv_b<3>(mode, nparts, map, s0, s1, poff, a, x, y, w, p0, p1, done, ctl, st, pdl, wf);
    case 4: return launch_spmv_b<4>(mode, nparts, map, s0, s1, poff, a, x, y, w, p0, p1, done, ctl, st, pdl, wf);
    default: return B2S_UNSUPPORTED;
  }
}

int launch_spmv(int b, int mode, int nparts, SliceMap map, Sell a, const double* x, double* y,
                const double* w, double* p0, double* p1, const int* done, Ctl ctl,
                cudaStream_t st, bool pdl, WellFix wf) {
  return launch_spmv_range(b, mode, nparts, map, 0, map.nslices, 0, a, x, y, w, p0, p1, done, ctl,
                           st, pdl, wf);
}

}  // namespace b2s

using namespace b2s;

extern "C" {

// Plain slice map: slice s covers rows [32s, min(32s+32, n)).
int b2s_slices_plain(int n, int32_t* row0, int32_t* nrows, cudaStream_t st) {
  if (n < 0) return B2S_SHAPE;
  const int ns = (n + kSlice - 1) / kSlice;
  if (ns == 0) return B2S_OK;
  k_plain_slices<<<grid_for(ns), 256, 0, st>>>(n, ns, row0, nrows);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

// Number of group-aligned slices for group offsets off[0..ngroups].
// base (ngroups+1 int32, device) receives the first slice of every group.
int b2s_slices_grouped_count(int ngroups, const int32_t* off, int32_t* base,
                             int32_t* nslices_host, cudaStream_t st) {
  if (ngroups < 0) return B2S_SHAPE;
  *nslices_host = 0;
  if (ngroups == 0) return B2S_OK;
  int32_t* cnt = nullptr;
  B2S_CHECK(cudaMallocAsync(&cnt, sizeof(int32_t) * (ngroups + 1), st));
  B2S_CHECK(cudaMemsetAsync(cnt + ngroups, 0, sizeof(int32_t), st));
  k_group_slice_counts<<<grid_for(ngroups), 256, 0, st>>>(ngroups, off, cnt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, base, ngroups + 1, st);
  void* tmp = nullptr;
  B2S_CHECK(cudaMallocAsync(&tmp, tb, st));
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, base, ngroups + 1, st);
  B2S_LAUNCH_CHECK();
  int32_t h = 0;
  B2S_CHECK(cudaMemcpyAsync(&h, base + ngroups, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaFreeAsync(tmp, st));
  B2S_CHECK(cudaFreeAsync(cnt, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  *nslices_host = h;
  return B2S_OK;
}

int b2s_slices_grouped_fill(int ngroups, int nslices, const int32_t* off, const int32_t* base,
                            int32_t* row0, int32_t* nrows, cudaStream_t st) {
  if (ngroups < 0 || nslices < 0) return B2S_SHAPE;
  if (nslices == 0) return B2S_OK;
  k_group_slices<<<grid_for(nslices), 256, 0, st>>>(ngroups, nslices, off, base, row0, nrows);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

// Slot offsets of a SELL-32 layout and the widest slice (entries per row),
// both read back with one synchronisation.
int b2s_sell_offsets_ex(int nslices, const int32_t* row0, const int32_t* nrows, const int32_t* rp,
                        const int32_t* ci, int sel, int32_t* sp, long long* slots_host,
                        int* width_host, cudaStream_t st) {
  if (nslices < 0 || sel < 0 || sel > 2) return B2S_SHAPE;
  *slots_host = 0;
  if (width_host) *width_host = 0;
  if (nslices == 0) {
    B2S_CHECK(cudaMemsetAsync(sp, 0, sizeof(int32_t), st));
    return B2S_OK;
  }
  int32_t* cnt = nullptr;
  B2S_CHECK(cudaMallocAsync(&cnt, sizeof(int32_t) * (nslices + 2), st));
  B2S_CHECK(cudaMemsetAsync(cnt + nslices, 0, sizeof(int32_t), st));
  k_sell_width<<<grid_for((long long)nslices * 32), 256, 0, st>>>(nslices, row0, nrows, rp, ci,
                                                                   sel, cnt);
  size_t tb = 0, tm = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, sp, nslices + 1, st);
  cub::DeviceReduce::Max(nullptr, tm, cnt, cnt + nslices + 1, nslices, st);
  void* tmp = nullptr;
  B2S_CHECK(cudaMallocAsync(&tmp, tb > tm ? tb : tm, st));
  cub::DeviceReduce::Max(tmp, tm, cnt, cnt + nslices + 1, nslices, st);
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, sp, nslices + 1, st);
  B2S_LAUNCH_CHECK();
  int32_t h[2] = {0, 0};
  B2S_CHECK(cudaMemcpyAsync(&h[0], sp + nslices, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaMemcpyAsync(&h[1], cnt + nslices + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaFreeAsync(tmp, st));
  B2S_CHECK(cudaFreeAsync(cnt, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  *slots_host = h[0];
  if (width_host) *width_host = h[1] / kSlice;
  return B2S_OK;
}

// Slot offsets of a SELL-32 layout: sp[0..nslices], total slots to host.
// sel: 0 = every block, 1 = strict lower, 2 = strict upper.
int b2s_sell_offsets(int nslices, const int32_t* row0, const int32_t* nrows, const int32_t* rp,
                     const int32_t* ci, int sel, int32_t* sp, long long* slots_host,
                     cudaStream_t st) {
  return b2s_sell_offsets_ex(nslices, row0, nrows, rp, ci, sel, sp, slots_host, nullptr, st);
}

int b2s_sell_fill_src(int nslices, int b, const int32_t* row0, const int32_t* nrows,
                      const int32_t* rp, const int32_t* ci, const double* vals, int sel,
                      const int32_t* sp, const int32_t* goff, int ngroups, int32_t* cols,
                      double* svals, const int32_t* src, cudaStream_t st) {
  if (nslices < 0 || b < 1 || sel < 0 || sel > 2) return B2S_SHAPE;
  if (nslices == 0) return B2S_OK;
  if (sel == 0 && !goff && b <= 4) {   // every block: one thread per slot
    const int g = nslices < kSms * 32 ? nslices : kSms * 32;
    switch (b) {
      case 1: k_sell_fill_all<1><<<g, 256, 0, st>>>(nslices, row0, nrows, rp, ci, vals, sp, cols, svals, src); break;
      case 2: k_sell_fill_all<4><<<g, 256, 0, st>>>(nslices, row0, nrows, rp, ci, vals, sp, cols, svals, src); break;
      case 3: k_sell_fill_all<9><<<g, 256, 0, st>>>(nslices, row0, nrows, rp, ci, vals, sp, cols, svals, src); break;
      default: k_sell_fill_all<16><<<g, 256, 0, st>>>(nslices, row0, nrows, rp, ci, vals, sp, cols, svals, src); break;
    }
  } else {
    k_sell_fill<<<grid_for((long long)nslices * 32), 256, 0, st>>>(nslices, b * b, row0, nrows, rp,
                                                                    ci, vals, sel, sp, goff, ngroups,
                                                                    cols, svals, src);
  }
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

int b2s_sell_fill(int nslices, int b, const int32_t* row0, const int32_t* nrows,
                  const int32_t* rp, const int32_t* ci, const double* vals, int sel,
                  const int32_t* sp, const int32_t* goff, int ngroups, int32_t* cols,
                  double* svals, cudaStream_t st) {
  return b2s_sell_fill_src(nslices, b, row0, nrows, rp, ci, vals, sel, sp, goff, ngroups, cols,
                           svals, nullptr, st);
}

int b2s_diag_tiles(int nslices, int b, const int32_t* row0, const int32_t* nrows,
                   const double* inv, double* tiles, cudaStream_t st) {
  if (nslices < 0 || b < 1) return B2S_SHAPE;
  if (nslices == 0) return B2S_OK;
  k_diag_tiles<<<grid_for((long long)nslices * 32), 256, 0, st>>>(nslices, b * b, row0, nrows,
                                                                   inv, tiles);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

// y = A x (mode 0), with gamma partials w.y (mode 1), with (y.y, y.w)
// partials (mode 2), or the residual y = w - A x with y.y partials (mode 3).
// `nparts` CTAs are launched; part0/part1 receive one partial per CTA.
int b2s_spmv(int b, int mode, int nparts, int nslices, const int32_t* row0,
             const int32_t* nrows, const int32_t* sp, const int32_t* cols, const double* vals,
             const double* x, double* y, const double* w, double* part0, double* part1,
             const int* done, cudaStream_t st) {
  if (nslices < 0 || nparts < 1) return B2S_SHAPE;
  SliceMap map{nslices, row0, nrows};
  Sell a{sp, cols, vals};
  return launch_spmv(b, mode, nparts, map, a, x, y, w, part0, part1, done, Ctl{}, st, false,
                     WellFix{});
}

}  // extern "C"
