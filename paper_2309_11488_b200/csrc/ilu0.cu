// Zero-fill block ILU0 application (bs/ilu0.py:93-142): the forward and
// backward block-triangular sweeps as sync-free wavefronts.
//
// Rows are processed in plan (permuted) order.  A warp claims the next
// group-aligned slice of <= 32 rows through an atomic ticket (ascending for
// the factorisation and the forward sweep, descending for the backward
// sweep); because tickets go only to resident warps and every dependency of
// a row lies in an earlier ticket, the oldest unfinished slice can always
// proceed.  There is no per-level launch and no grid barrier: a row waits
// only for the rows it actually reads, so independent parts of consecutive
// levels overlap, and the critical path costs one L2 round trip per level.
//
//  * factorisation: see factor.cu;
//  * sweeps: the dependency vector itself is the flag -- it is pre-filled
//    with a NaN sentinel and a consumer spins until the producer's value
//    replaces it (one round trip, no separate flag + fence).  The backward
//    sweep restores the forward scratch vector to the sentinel as it
//    consumes it, and the Krylov kernels restore the backward output after
//    its last use, so no extra fill pass is needed per application.
#include "sell.cuh"

namespace b2s {

struct Tickets {
  unsigned int next;      // next slice ticket
  unsigned int finished;  // warps that ran out of work (self-reset)
};

// Claim the next ticket for the calling warp; returns -1 once exhausted
// (after registering the warp's exit; the last warp out resets the pair so
// the kernel can be relaunched or graph-replayed without a memset).
__device__ __forceinline__ long long claim(Tickets* tk, int nslices);

// Next slice ticket of the calling warp: dynamic (one atomic per slice) or,
// with flags bit 2, static round-robin over the persistent grid's warps --
// warp w takes tickets w, w+W, ... in order, which is deadlock-free for the
// same reason (every warp's earlier tickets are lower, all warps resident)
// and spares the single hot counter ~30k serialised atomics per sweep.
__device__ __forceinline__ long long next_slice(Tickets* tk, int nslices, int flags,
                                                long long& iter) {
  if (flags & 4) {
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long t = gw + (iter++) * nw;
    return t < nslices ? t : -1;
  }
  return claim(tk, nslices);
}

__device__ __forceinline__ long long claim(Tickets* tk, int nslices) {
  const int lane = threadIdx.x & 31;
  unsigned int t = 0;
  if (lane == 0) t = atomicAdd(&tk->next, 1u);
  t = __shfl_sync(0xffffffffu, t, 0);
  if (t < (unsigned)nslices) return t;
  if (lane == 0) {
    const unsigned int total = gridDim.x * (blockDim.x >> 5);
    const unsigned int f = atomicAdd(&tk->finished, 1u);
    if (f == total - 1) {
      tk->next = 0;
      tk->finished = 0;
      __threadfence();
    }
  }
  return -1;
}

// ---------------------------------------------------------------------------
// sweeps.  KC = entries prefetched into registers per chunk (compile-time).
__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}


// Dependencies of one prefetched chunk, polled *together*: every pending
// entry's loads are issued back to back each round, so a row pays about one
// L2 round trip after its last input lands instead of one per input.
// col[kk] >= 0: wait for ready[col]; col[kk] <= -2: same-group entry, take
// stale[-col-2] (the vector before this sweep); -1: padding.
template <int B, int KC>
__device__ __forceinline__ void fetch_deps(const int (&col)[KC], const double* ready,
                                           const double* stale, double (&dep)[KC][B],
                                           int flags) {
  unsigned int pend = 0;
#pragma unroll
  for (int kk = 0; kk < KC; ++kk) {
    const int c0 = col[kk];
    if (c0 <= -2) {
#pragma unroll
      for (int c = 0; c < B; ++c) dep[kk][c] = stale[(long long)(-c0 - 2) * B + c];
    } else {
#pragma unroll
      for (int c = 0; c < B; ++c) dep[kk][c] = 0.0;
      if (c0 >= 0) pend |= 1u << kk;
    }
  }
  unsigned int ns = 32;
  while (pend) {
    const unsigned int todo = pend;  // issue every pending load first ...
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      if (todo & (1u << kk)) {
        const double* p = ready + (long long)col[kk] * B;
#pragma unroll
        for (int c = 0; c < B; ++c) dep[kk][c] = ld_relaxed(p + c);
      }
    }
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {  // ... then test them
      bool miss = false;
#pragma unroll
      for (int c = 0; c < B; ++c) miss |= is_sentinel(dep[kk][c]);
      if ((todo & (1u << kk)) && !miss) pend &= ~(1u << kk);
    }
    if (pend && (flags & 1)) {
      __nanosleep(ns);
      ns = ns < 256 ? ns * 2 : 256;
    }
  }
}

// forward: y_i = r_i - sum_k L_ik y_k   (unit lower, ascending columns)
template <int B, int KC>
__global__ void __launch_bounds__(256) k_ilu0_forward(SliceMap map, Sell lo,
                                                      const double* __restrict__ r, double* y,
                                                      int flags, Tickets* tk, const int* done) {
  constexpr int BB = B * B;
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  long long iter = 0;
  for (;;) {
    const long long s = next_slice(tk, map.nslices, flags, iter);
    if (s < 0) break;
    const bool ok = lane < map.nrows[s];
    const long long i = (long long)map.row0[s] + lane;
    const int slot0 = lo.sp[s];
    const int width = (lo.sp[s + 1] - slot0) >> 5;
    double rv[B], acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      rv[c] = ok ? r[i * B + c] : 0.0;
      acc[c] = 0.0;
    }
    for (int k0 = 0; k0 < width; k0 += KC) {
      int col[KC];
      double blk[KC][BB];
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        const bool in = k0 + kk < width;
        col[kk] = in ? __ldcs(lo.cols + slot0 + 32 * (k0 + kk) + lane) : -1;
#pragma unroll
        for (int e = 0; e < BB; ++e)
          blk[kk][e] = in ? __ldcs(lo.vals + vidx(slot0, k0 + kk, e, lane, BB)) : 0.0;
      }
      double dep[KC][B];
      fetch_deps<B, KC>(col, y, r, dep, flags);
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        if (col[kk] != -1) {  // ascending column order, like the reference
          double pr[B];
          matvec<B>(blk[kk], dep[kk], pr);
#pragma unroll
          for (int c = 0; c < B; ++c) acc[c] += pr[c];
        }
      }
    }
    if (ok) {
#pragma unroll
      for (int c = 0; c < B; ++c) st_relaxed(y + i * B + c, canon(rv[c] - acc[c]));
    }
  }
}

// backward: z_i = inv(U_ii) (y_i - sum_k U_ik z_k)   (descending slices)
template <int B, int KC>
__global__ void __launch_bounds__(256) k_ilu0_backward(SliceMap map, Sell up,
                                                       const double* __restrict__ dtiles,
                                                       double* y, double* z, int reset_y,
                                                       int flags, Tickets* tk, const int* done) {
  constexpr int BB = B * B;
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  long long iter = 0;
  for (;;) {
    const long long t = next_slice(tk, map.nslices, flags, iter);
    if (t < 0) break;
    const long long s = map.nslices - 1 - t;
    const bool ok = lane < map.nrows[s];
    const long long i = (long long)map.row0[s] + lane;
    const int slot0 = up.sp[s];
    const int width = (up.sp[s + 1] - slot0) >> 5;
    double yv[B], acc[B], dinv[BB];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      yv[c] = ok ? y[i * B + c] : 0.0;
      acc[c] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < BB; ++e) dinv[e] = __ldcs(dtiles + (s * BB + e) * 32 + lane);
    for (int k0 = 0; k0 < width; k0 += KC) {
      int col[KC];
      double blk[KC][BB];
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        const bool in = k0 + kk < width;
        col[kk] = in ? __ldcs(up.cols + slot0 + 32 * (k0 + kk) + lane) : -1;
#pragma unroll
        for (int e = 0; e < BB; ++e)
          blk[kk][e] = in ? __ldcs(up.vals + vidx(slot0, k0 + kk, e, lane, BB)) : 0.0;
      }
      double dep[KC][B];
      fetch_deps<B, KC>(col, z, y, dep, flags);  // same group: forward result
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        if (col[kk] != -1) {
          double pr[B];
          matvec<B>(blk[kk], dep[kk], pr);
#pragma unroll
          for (int c = 0; c < B; ++c) acc[c] += pr[c];
        }
      }
    }
    if (ok) {
      double tv[B], out[B];
#pragma unroll
      for (int c = 0; c < B; ++c) tv[c] = yv[c] - acc[c];
      matvec<B>(dinv, tv, out);
#pragma unroll
      for (int c = 0; c < B; ++c) st_relaxed(z + i * B + c, canon(out[c]));
      if (reset_y) {
#pragma unroll
        for (int c = 0; c < B; ++c) y[i * B + c] = sentinel();
      }
    }
  }
}

template <int B>
int occupancy_grid(const void* fn) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int dev = 0, sms = kSms;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms;
}

// ---------------------------------------------------------------------------
// Phased sweeps for plans with few groups whose rows are independent sets
// (every colouring; no same-group entries).  In plan order group 0 has no
// strict-lower entries (y = r there) and the last group no strict-upper ones
// (z = inv(U_ii) y there), so an application is 2(G-1) data-parallel passes
// with no polling at all:
//   forward  g = 1..G-1 : y_i = r_i - sum_k L_ik y_k   (y_k = r_k in group 0);
//                         for the last group z_i = inv(U_ii) y_i directly;
//   backward g = G-2..0 : z_i = inv(U_ii) (y_i - sum_k U_ik z_k)  (y_i = r_i in group 0).
// For two colours that is two passes and the intermediate y is never stored.
// Each row's arithmetic (ascending columns, acc then subtract, matvec with
// the inverse diagonal) is exactly the sync-free sweeps' -- results are
// bit-identical.  Dependencies come from earlier launches, so they are plain
// read-only-path loads.
// Two entries per step with the column indices one step ahead (105
// registers, 2 CTAs per SM): measured 94.8 -> 89.5 us per C4 application
// against the one-entry loop at 80 registers and 3 CTAs per SM.
template <int B>
__device__ __forceinline__ void phase_row_sum(const Sell& m, int slot0, int width, int lane,
                                              int goff1, const double* __restrict__ r,
                                              const double* __restrict__ v, double (&acc)[B]) {
  constexpr int BB = B * B;
  // two entries per step, every load of the pair issued before any math;
  // the next pair's column indices load one step ahead (as in k_spmv)
  int cn0 = width > 0 ? __ldcs(m.cols + slot0 + lane) : -1;
  int cn1 = width > 1 ? __ldcs(m.cols + slot0 + 32 + lane) : -1;
  for (int k = 0; k < width; k += 2) {
    const int col[2] = {cn0, cn1};
    cn0 = k + 2 < width ? __ldcs(m.cols + slot0 + 32 * (k + 2) + lane) : -1;
    cn1 = k + 3 < width ? __ldcs(m.cols + slot0 + 32 * (k + 3) + lane) : -1;
    double blk[2][BB], dep[2][B];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      // padding (-1; phased plans have no same-group entries) loads nothing
#pragma unroll
      for (int e = 0; e < BB; ++e)
        blk[q][e] = col[q] >= 0 ? __ldcs(m.vals + vidx(slot0, k + q, e, lane, BB)) : 0.0;
      const double* src = col[q] < goff1 ? r : v;
      const long long cq = col[q] < 0 ? 0 : col[q];
#pragma unroll
      for (int c = 0; c < B; ++c) dep[q][c] = col[q] >= 0 ? __ldg(src + cq * B + c) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (col[q] < 0) continue;
      double pr[B];
      matvec<B>(blk[q], dep[q], pr);
#pragma unroll
      for (int c = 0; c < B; ++c) acc[c] += pr[c];
    }
  }
}

template <int B, int KC, bool LAST>
__global__ void __launch_bounds__(256) k_phase_forward(int s0, int s1, int goff1, SliceMap map,
                                                       Sell lo, const double* __restrict__ dtiles,
                                                       const double* __restrict__ r,
                                                       double* __restrict__ y,
                                                       double* __restrict__ z, const int* done) {
  constexpr int BB = B * B;
  griddep_wait();
  griddep_launch();
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long s = s0 + (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < s1;
       s += nw) {
    const bool ok = lane < map.nrows[s];
    const long long i = (long long)map.row0[s] + lane;
    const int slot0 = lo.sp[s];
    const int width = (lo.sp[s + 1] - slot0) >> 5;
    double rv[B], acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      rv[c] = ok ? __ldcs(r + i * B + c) : 0.0;
      acc[c] = 0.0;
    }
    double dinv[LAST ? BB : 1];
    if (LAST) {
#pragma unroll
      for (int e = 0; e < BB; ++e) dinv[e] = __ldcs(dtiles + (s * BB + e) * 32 + lane);
    }
    phase_row_sum<B>(lo, slot0, width, lane, goff1, r, y, acc);
    if (!ok) continue;
    double tv[B];
#pragma unroll
    for (int c = 0; c < B; ++c) tv[c] = canon(rv[c] - acc[c]);
    if (LAST) {
      // backward row of the last group: no upper entries, acc = 0
      double t2[B], out[B];
#pragma unroll
      for (int c = 0; c < B; ++c) t2[c] = tv[c] - 0.0;
      matvec<B>(dinv, t2, out);
#pragma unroll
      for (int c = 0; c < B; ++c) z[i * B + c] = canon(out[c]);
    } else {
#pragma unroll
      for (int c = 0; c < B; ++c) y[i * B + c] = tv[c];
    }
  }
}

template <int B, int KC>
__global__ void __launch_bounds__(256) k_phase_backward(int s0, int s1, int goff1, SliceMap map,
                                                        Sell up, const double* __restrict__ dtiles,
                                                        const double* __restrict__ r,
                                                        const double* __restrict__ y,
                                                        double* __restrict__ z, const int* done) {
  constexpr int BB = B * B;
  griddep_wait();
  griddep_launch();
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long s = s0 + (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < s1;
       s += nw) {
    const bool ok = lane < map.nrows[s];
    const long long i = (long long)map.row0[s] + lane;
    const int slot0 = up.sp[s];
    const int width = (up.sp[s + 1] - slot0) >> 5;
    const double* yin = (i < goff1) ? r : y;   // a slice lies in one group
    double yv[B], acc[B], dinv[BB];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      yv[c] = ok ? __ldcs(yin + i * B + c) : 0.0;
      acc[c] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < BB; ++e) dinv[e] = __ldcs(dtiles + (s * BB + e) * 32 + lane);
    // upper entries point into later groups (never group 0): z only
    phase_row_sum<B>(up, slot0, width, lane, 0, r, z, acc);
    if (!ok) continue;
    double tv[B], out[B];
#pragma unroll
    for (int c = 0; c < B; ++c) tv[c] = yv[c] - acc[c];
    matvec<B>(dinv, tv, out);
#pragma unroll
    for (int c = 0; c < B; ++c) z[i * B + c] = canon(out[c]);
  }
}

template <int B, int KC>
int launch_phased_bk(int ngroups, const int32_t* gs, int goff1, SliceMap map, Sell lo, Sell up,
                     const double* dt, const double* r, double* y, double* z, const int* done,
                     bool skip_g0, cudaStream_t st, bool pdl) {
  static int cap = 0;
  if (!cap) cap = occupancy_grid<B>((const void*)k_phase_forward<B, KC, true>);
  auto grid = [&](int ns) {
    long long g = ((long long)ns + 7) / 8;  // 8 warps per CTA, one slice each
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
  };
  for (int g = 1; g < ngroups; ++g) {
    const int s0 = gs[g], s1 = gs[g + 1];
    if (s1 <= s0) continue;
    if (g == ngroups - 1)
      launch_k(k_phase_forward<B, KC, true>, dim3(grid(s1 - s0)), dim3(256), 0, st, pdl, s0, s1,
               goff1, map, lo, dt, r, y, z, done);
    else
      launch_k(k_phase_forward<B, KC, false>, dim3(grid(s1 - s0)), dim3(256), 0, st, pdl, s0, s1,
               goff1, map, lo, dt, r, y, z, done);
  }
  for (int g = ngroups - 2; g >= (skip_g0 ? 1 : 0); --g) {
    const int s0 = gs[g], s1 = gs[g + 1];
    if (s1 <= s0) continue;
    launch_k(k_phase_backward<B, KC>, dim3(grid(s1 - s0)), dim3(256), 0, st, pdl, s0, s1, goff1,
             map, up, dt, (const double*)r, (const double*)y, z, done);
  }
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

template <int B>
int launch_phased_b(int kc, int ngroups, const int32_t* gs, int goff1, SliceMap map, Sell lo,
                    Sell up, const double* dt, const double* r, double* y, double* z,
                    const int* done, bool skip_g0, cudaStream_t st, bool pdl) {
  if (kc <= 2)
    return launch_phased_bk<B, 2>(ngroups, gs, goff1, map, lo, up, dt, r, y, z, done, skip_g0, st, pdl);
  return launch_phased_bk<B, 4>(ngroups, gs, goff1, map, lo, up, dt, r, y, z, done, skip_g0, st, pdl);
}

// ngroups >= 2; gslice_host[g] = first slice of group g (group-aligned map).
// skip_g0: leave out the final backward pass of group 0 (fused.cu does it
// together with the SpMV rows of group 0).
int launch_phased(int b, int kc, int ngroups, const int32_t* gslice_host, int goff1, SliceMap map,
                  Sell lo, Sell up, const double* dt, const double* r, double* y, double* z,
                  const int* done, cudaStream_t st, bool skip_g0, bool pdl) {
  if (ngroups < 2) return B2S_SHAPE;
  switch (b) {
    case 1: return launch_phased_b<1>(kc, ngroups, gslice_host, goff1, map, lo, up, dt, r, y, z, done, skip_g0, st, pdl);
    case 2: return launch_phased_b<2>(kc, ngroups, gslice_host, goff1, map, lo, up, dt, r, y, z, done, skip_g0, st, pdl);
    case 3: return launch_phased_b<3>(kc, ngroups, gslice_host, goff1, map, lo, up, dt, r, y, z, done, skip_g0, st, pdl);
    case 4: return launch_phased_b<4>(kc, ngroups, gslice_host, goff1, map, lo, up, dt, r, y, z, done, skip_g0, st, pdl);
    default: return B2S_UNSUPPORTED;
  }
}

__global__ void k_fill_sentinel(long long m, double* v) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m;
       t += (long long)gridDim.x * blockDim.x)
    v[t] = sentinel();
}

// rows whose lower entries reach into their own slice (possible only for a
// user-built plan whose groups are not independent sets)
__global__ void k_slice_conflicts(SliceMap map, const int32_t* __restrict__ rp,
                                  const int32_t* __restrict__ ci, int* conflict) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < map.nslices; s += nw) {
    if (lane >= map.nrows[s]) continue;
    const int r0 = map.row0[s], i = r0 + lane;
    for (int q = rp[i]; q < rp[i + 1]; ++q) {
      const int c = ci[q];
      if (c >= r0 && c != i && c < r0 + map.nrows[s]) atomicExch(conflict, 1);
    }
  }
}


template <int B, int KC>
int launch_sweeps_bk(SliceMap map, Sell lo, Sell up, const double* dt, const double* r,
                     double* y, double* z, int reset_y, int flags, Tickets* tk, const int* done,
                     cudaStream_t st) {
  // flags bits 4-7: CTAs per SM (0 = max occupancy), bits 8-11: warps per
  // CTA (0 = 8).  Fewer resident warps = fewer pollers competing for L2.
  const int per_sm = (flags >> 4) & 15, warps = ((flags >> 8) & 15) ? ((flags >> 8) & 15) : 8;
  int gf = occupancy_grid<B>((const void*)k_ilu0_forward<B, KC>);
  int gb = occupancy_grid<B>((const void*)k_ilu0_backward<B, KC>);
  if (per_sm) { gf = min(gf, per_sm * kSms); gb = min(gb, per_sm * kSms); }
  k_ilu0_forward<B, KC><<<gf, 32 * warps, 0, st>>>(map, lo, r, y, flags, tk, done);
  k_ilu0_backward<B, KC><<<gb, 32 * warps, 0, st>>>(map, up, dt, y, z, reset_y, flags, tk + 1,
                                                    done);
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

template <int B>
int launch_sweeps_b(int kc, SliceMap map, Sell lo, Sell up, const double* dt, const double* r,
                    double* y, double* z, int reset_y, int flags, Tickets* tk, const int* done,
                    cudaStream_t st) {
  if (kc <= 2) return launch_sweeps_bk<B, 2>(map, lo, up, dt, r, y, z, reset_y, flags, tk, done, st);
  if (kc <= 4) return launch_sweeps_bk<B, 4>(map, lo, up, dt, r, y, z, reset_y, flags, tk, done, st);
  return launch_sweeps_bk<B, 8>(map, lo, up, dt, r, y, z, reset_y, flags, tk, done, st);
}

int launch_sweeps(int b, int kc, SliceMap map, Sell lo, Sell up, const double* dt,
                  const double* r, double* y, double* z, int reset_y, int flags, void* tickets,
                  const int* done, cudaStream_t st) {
  Tickets* tk = reinterpret_cast<Tickets*>(tickets);
  switch (b) {
    case 1: return launch_sweeps_b<1>(kc, map, lo, up, dt, r, y, z, reset_y, flags, tk, done, st);
    case 2: return launch_sweeps_b<2>(kc, map, lo, up, dt, r, y, z, reset_y, flags, tk, done, st);
    case 3: return launch_sweeps_b<3>(kc, map, lo, up, dt, r, y, z, reset_y, flags, tk, done, st);
    case 4: return launch_sweeps_b<4>(kc, map, lo, up, dt, r, y, z, reset_y, flags, tk, done, st);
    default: return B2S_UNSUPPORTED;
  }
}

int fill_sentinel(long long m, double* v, cudaStream_t st) {
  if (m <= 0) return B2S_OK;
  long long g = (m + 255) / 256;
  if (g > kSms * 32) g = kSms * 32;
  k_fill_sentinel<<<(int)g, 256, 0, st>>>(m, v);
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

}  // namespace b2s

using namespace b2s;

extern "C" {

// 1 in *conflict_host if some row of the slice map reads a row of its own
// slice through its strict-lower part (the plan's groups are not
// independent); such maps must fall back to one row per slice.
int b2s_slice_conflicts(int nslices, const int32_t* row0, const int32_t* nrows,
                        const int32_t* rp, const int32_t* ci, int* conflict_host,
                        cudaStream_t st) {
  *conflict_host = 0;
  if (nslices <= 0) return B2S_OK;
  int* d = nullptr;
  B2S_CHECK(cudaMallocAsync(&d, sizeof(int), st));
  B2S_CHECK(cudaMemsetAsync(d, 0, sizeof(int), st));
  SliceMap map{nslices, row0, nrows};
  long long g = ((long long)nslices * 32 + 255) / 256;
  if (g > kSms * 32) g = kSms * 32;
  k_slice_conflicts<<<(int)g, 256, 0, st>>>(map, rp, ci, d);
  B2S_LAUNCH_CHECK();
  B2S_CHECK(cudaMemcpyAsync(conflict_host, d, sizeof(int), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaFreeAsync(d, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  return B2S_OK;
}

int b2s_fill_sentinel(long long m, double* v, cudaStream_t st) { return fill_sentinel(m, v, st); }

// Phased application for plans of 2..32 independent groups without
// same-group entries (colourings): no sentinel preconditions, y is scratch.
int b2s_ilu0_apply_phased(int n, int b, int kc, int ngroups, const int32_t* gslice_host,
                          int goff1, const int32_t* row0, const int32_t* nrows,
                          const int32_t* l_sp, const int32_t* l_cols, const double* l_vals,
                          const int32_t* u_sp, const int32_t* u_cols, const double* u_vals,
                          const double* dinv_tiles, const double* r, double* y, double* z,
                          cudaStream_t st) {
  if (n < 0 || b < 1 || ngroups < 2 || !gslice_host) return B2S_SHAPE;
  if (n == 0) return B2S_OK;
  SliceMap map{gslice_host[ngroups], row0, nrows};
  Sell lo{l_sp, l_cols, l_vals}, up{u_sp, u_cols, u_vals};
  return launch_phased(b, kc, ngroups, gslice_host, goff1, map, lo, up, dinv_tiles, r, y, z,
                       nullptr, st, false, false);
}

// z = U^-1 L^-1 r in plan order.  Preconditions: y and z hold the sentinel
// everywhere (b2s_fill_sentinel); tickets points at 16 zeroed bytes that the
// kernels keep reset between calls.  On return z holds the result and, when
// reset_y != 0, y holds the sentinel again.  kc = max entries per row of L
// and U (selects the register prefetch depth).
int b2s_ilu0_apply(int n, int b, int kc, int nslices, const int32_t* row0, const int32_t* nrows,
                   const int32_t* l_sp, const int32_t* l_cols, const double* l_vals,
                   const int32_t* u_sp, const int32_t* u_cols, const double* u_vals,
                   const double* dinv_tiles, const double* r, double* y, double* z, int reset_y,
                   int flags, void* tickets, cudaStream_t st) {
  if (n < 0 || b < 1) return B2S_SHAPE;
  if (n == 0) return B2S_OK;
  SliceMap map{nslices, row0, nrows};
  Sell lo{l_sp, l_cols, l_vals}, up{u_sp, u_cols, u_vals};
  return launch_sweeps(b, kc, map, lo, up, dinv_tiles, r, y, z, reset_y, flags, tickets, nullptr,
                       st);
}

}  // extern "C"
