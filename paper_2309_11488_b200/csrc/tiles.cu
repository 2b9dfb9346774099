// Tiled ILU0 sweeps: the level-scheduled forward/backward block-triangular
// solves (bs/ilu0.py:105-142) with most dependencies resolved on-chip.
//
// Why: in the sync-free sweep (ilu0.cu) every level of the schedule costs a
// cross-SM L2 round trip (~1.2-1.4 us measured on B200), so a 1M-cell
// stencil with ~300 levels per sweep is latency-bound at ~0.1 of the HBM
// roofline.  Here the rows are partitioned into T tiles, one co-resident
// CTA per SM (cooperative launch).  A tile keeps the values of its own rows
// in shared memory; its warps run the same sync-free protocol as ilu0.cu,
// but a dependency inside the tile is polled in shared memory (tens of
// cycles) instead of L2, and only couplings that cross a tile boundary are
// polled from global memory.  With tiles that follow the grid geometry
// (column patches of a structured grid, or contiguous ranges of the input
// order otherwise) most couplings stay inside a tile, so the critical path
// takes a handful of L2 hops instead of one per level.
//
// A tile's rows are listed in plan order and cut into slices of <= 32 rows of
// one group (independent rows).  Warp w of the CTA processes the tile's
// slices w, w+W, ... in order (reverse order for the backward sweep); the
// lowest unfinished slice of a tile always has its local inputs, and remote
// inputs lie in strictly earlier groups, so no wait can be circular.
// Per-row arithmetic is exactly the sync-free kernels' (ascending-column sum,
// then subtract; backward times inv(U_ii)): results are bit-identical.
//
// Entry codes in the tile SELL layouts: c >= 0 remote row c (poll global);
// -1 padding; -(2 + 2*loc) local slot `loc` of this tile (poll shared);
// -(3 + 2*c) same-group row c (read the pre-sweep vector, as the reference
// does for rows of one group).
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "sell.cuh"

namespace b2s {

constexpr unsigned kPollNs = 40;   // pause between polling rounds

struct TileSet {
  int T, nsl, rmax;
  const int32_t* trow;    // rows of all tiles, tile-major, plan order inside a tile
  const int32_t* sstart;  // [nsl+1] slice s = trow[sstart[s] .. sstart[s+1])
  const int32_t* tslice;  // [T+1] slices of tile t
  const int32_t* toff;    // [T+1] rows of tile t in trow
  Sell L, U;              // per-slice SELL of the strict lower / upper blocks
  const double* dtile;    // per-slice b*b x 32 inverse-diagonal tiles
};

__device__ __forceinline__ double ld_relaxed_d(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_d(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// poll all pending inputs of a prefetched chunk together (one round per
// wave of loads): remote ones in global memory, local ones in shared memory
template <int B, int KC>
__device__ __forceinline__ void tile_deps(const int (&code)[KC], const double* remote,
                                          const double* stale, const volatile double* vloc,
                                          double (&dep)[KC][B]) {
  unsigned int pend = 0;
#pragma unroll
  for (int kk = 0; kk < KC; ++kk) {
    const int c0 = code[kk];
#pragma unroll
    for (int c = 0; c < B; ++c) dep[kk][c] = 0.0;
    if (c0 >= 0) {
      pend |= 1u << kk;
    } else if (c0 <= -2) {
      const int v = -c0 - 2;
      if (v & 1) {
#pragma unroll
        for (int c = 0; c < B; ++c) dep[kk][c] = stale[(long long)(v >> 1) * B + c];
      } else {
        pend |= 1u << kk;
      }
    }
  }
  while (pend) {
    const unsigned int todo = pend;
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      if (todo & (1u << kk)) {
        const int c0 = code[kk];
        if (c0 >= 0) {
#pragma unroll
          for (int c = 0; c < B; ++c) dep[kk][c] = ld_relaxed_d(remote + (long long)c0 * B + c);
        } else {
          const int loc = (-c0 - 2) >> 1;
#pragma unroll
          for (int c = 0; c < B; ++c) dep[kk][c] = vloc[loc * B + c];
        }
      }
    }
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      bool miss = false;
#pragma unroll
      for (int c = 0; c < B; ++c) miss |= is_sentinel(dep[kk][c]);
      if ((todo & (1u << kk)) && !miss) pend &= ~(1u << kk);
    }
    // a shared-memory poll returns in tens of cycles: without a pause the
    // waiting warps would take the issue slots of the warps doing the work
    if (pend) __nanosleep(kPollNs);
  }
}

// DIR = 0 forward (out = y = L^-1 in), 1 backward (out = z = U^-1 in).
template <int B, int KC, int DIR, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
    k_tile_sweep(TileSet ts, const double* __restrict__ in, double* out, double* yreset,
                 int reset, const int* done) {
  constexpr int BB = B * B;
  extern __shared__ __align__(16) double vloc_raw[];
  volatile double* vloc = vloc_raw;
  if (done && *done) return;
  const int t = blockIdx.x;
  const int s_begin = ts.tslice[t], s_end = ts.tslice[t + 1];
  const int k_base = ts.toff[t];
  const int nloc = ts.toff[t + 1] - k_base;
  for (int q = threadIdx.x; q < nloc * B; q += blockDim.x) vloc_raw[q] = sentinel();
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = blockDim.x >> 5;
  const Sell S = DIR == 0 ? ts.L : ts.U;
  for (int j = warp; j < s_end - s_begin; j += W) {
    const int s = DIR == 0 ? s_begin + j : s_end - 1 - j;
    const int k0 = ts.sstart[s];
    const int nr = ts.sstart[s + 1] - k0;
    const bool ok = lane < nr;
    const int row = ok ? ts.trow[k0 + lane] : 0;
    const int myloc = k0 + lane - k_base;
    double own[B], acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      own[c] = ok ? in[(long long)row * B + c] : 0.0;
      acc[c] = 0.0;
    }
    const int slot0 = S.sp[s];
    const int width = (S.sp[s + 1] - slot0) >> 5;
    for (int kb = 0; kb < width; kb += KC) {
      int code[KC];
      double blk[KC][BB];
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        const bool in_range = kb + kk < width;
        code[kk] = in_range ? __ldcs(S.cols + slot0 + 32 * (kb + kk) + lane) : -1;
#pragma unroll
        for (int e = 0; e < BB; ++e)
          blk[kk][e] = in_range ? __ldcs(S.vals + vidx(slot0, kb + kk, e, lane, BB)) : 0.0;
      }
      double dep[KC][B];
      tile_deps<B, KC>(code, out, in, vloc, dep);
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        if (code[kk] != -1) {  // ascending column order, like the reference
          double pr[B];
          matvec<B>(blk[kk], dep[kk], pr);
#pragma unroll
          for (int c = 0; c < B; ++c) acc[c] += pr[c];
        }
      }
    }
    if (ok) {
      double res[B];
      if (DIR == 0) {
#pragma unroll
        for (int c = 0; c < B; ++c) res[c] = canon(own[c] - acc[c]);
      } else {
        double tv[B], dinv[BB];
#pragma unroll
        for (int c = 0; c < B; ++c) tv[c] = own[c] - acc[c];
#pragma unroll
        for (int e = 0; e < BB; ++e) dinv[e] = __ldcs(ts.dtile + ((long long)s * BB + e) * 32 + lane);
        matvec<B>(dinv, tv, res);
#pragma unroll
        for (int c = 0; c < B; ++c) res[c] = canon(res[c]);
      }
#pragma unroll
      for (int c = 0; c < B; ++c) {
        vloc[myloc * B + c] = res[c];
        st_relaxed_d(out + (long long)row * B + c, res[c]);
      }
      if (DIR == 1 && reset) {
#pragma unroll
        for (int c = 0; c < B; ++c) yreset[(long long)row * B + c] = sentinel();
      }
    }
  }
}

// ---------------------------------------------------------------- building
// tile of each plan-order row from its input index: contiguous ranges
// (px == 0) or px x py column patches of an nx x ny x nz natural-order grid

// ---------------------------------------------------------------------------
// Wave kernel: one warp per tile, the tile's slices consumed strictly in
// order (forward: ascending plan order; backward: descending), so every
// dependency inside the tile is already in shared memory when its consumer
// runs -- no polling, no barrier but __syncwarp.  Only couplings to other
// tiles are polled (relaxed gpu-scope loads of the sentinel-filled global
// vector).  The matrix data of the next D-1 slices streams into a ring of
// shared-memory stages with cp.async while the current slice computes, so
// the chain of slices never waits on HBM: a hop inside a tile costs a few
// hundred cycles instead of an L2 round trip.  Critical path ~ (levels x
// slice time) + (tile-boundary crossings x L2 round trip).
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp4(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct WaveLayout {   // byte offsets inside one stage
  int vals, cols, own, rows, dinv, bytes;
  int meta;            // ints of per-tile slice metadata at the front of shared memory
};

__host__ __device__ inline WaveLayout wave_layout(int b, int wmax, int max_slices) {
  WaveLayout w;
  const int bb = b * b;
  w.vals = 0;
  w.cols = wmax * 32 * bb * 8;
  w.own = w.cols + ((wmax * 32 * 4 + 15) / 16) * 16;
  w.rows = w.own + 32 * b * 8;
  w.dinv = w.rows + 32 * 4;
  w.bytes = w.dinv + bb * 32 * 8;
  // first row, width, first slot per slice (16 B multiple)
  w.meta = ((3 * (max_slices + 1) + 3) / 4) * 4;
  return w;
}

// in_t / out_t: vectors in TILE order (row k of trow at k*B): the rows of one
// slice are contiguous there, so a slice's own inputs stream with the same
// 16-byte cp.async as its matrix data.
template <int B, int DIR>
__device__ __forceinline__ void wave_issue(const TileSet& ts, const Sell& S, int s, int k0,
                                           int width, int slot0, char* stage,
                                           const WaveLayout& L, const double* __restrict__ in_t,
                                           int lane) {
  constexpr int BB = B * B;
  const char* vsrc = reinterpret_cast<const char*>(S.vals + (long long)slot0 * BB);
  const int vchunks = width * 32 * BB * 8 / 16;
  for (int q = lane; q < vchunks; q += 32) cp16(stage + L.vals + 16 * q, vsrc + 16 * q);
  const char* csrc = reinterpret_cast<const char*>(S.cols + slot0);
  for (int q = lane; q < width * 8; q += 32) cp16(stage + L.cols + 16 * q, csrc + 16 * q);
  // own inputs of the slice: 32 rows x B doubles, contiguous in tile order
  // (k0*B*8 is 8-byte aligned only: copy 8-byte words)
  const double* osrc = in_t + (long long)k0 * B;
  for (int q = lane; q < 32 * B; q += 32) cp8(stage + L.own + 8 * q, osrc + q);
  // the slice's plan-order rows (where results are published)
  cp4(stage + L.rows + 4 * lane, ts.trow + k0 + lane);
  if (DIR == 1) {
    const char* dsrc = reinterpret_cast<const char*>(ts.dtile + (long long)s * BB * 32);
    for (int q = lane; q < BB * 32 * 8 / 16; q += 32) cp16(stage + L.dinv + 16 * q, dsrc + 16 * q);
  }
}

template <int B, int DIR, int D>
__global__ void __launch_bounds__(32, 1)
    k_tile_wave(TileSet ts, WaveLayout L, const double* __restrict__ in,
                const double* __restrict__ in_t, double* out, double* out_t, double* yreset,
                int reset, const int* done, unsigned long long* trace) {
  constexpr int BB = B * B;
  constexpr int KP = 8;   // remote polls batched per round
  extern __shared__ __align__(16) char wsm[];
  if (done && *done) return;
  const int t = blockIdx.x, lane = threadIdx.x;
  const int s_begin = ts.tslice[t], s_end = ts.tslice[t + 1], nsl = s_end - s_begin;
  const int k_base = ts.toff[t];
  const Sell S = DIR == 0 ? ts.L : ts.U;
  int* mstart = reinterpret_cast<int*>(wsm);           // [nsl+1] first tile-order row
  int* mwidth = mstart + (nsl + 1);                     // [nsl] entries per row
  int* mslot = mwidth + nsl;                            // [nsl] first SELL slot
  char* ring = wsm + 4 * L.meta;
  double* vloc = reinterpret_cast<double*>(ring + D * L.bytes);
  for (int j = lane; j <= nsl; j += 32) mstart[j] = ts.sstart[s_begin + j];
  for (int j = lane; j < nsl; j += 32) {
    mslot[j] = S.sp[s_begin + j];
    mwidth[j] = (S.sp[s_begin + j + 1] - mslot[j]) >> 5;
  }
  __syncwarp();
  // j-th slice consumed: ascending (forward) or descending (backward)
  auto sl = [&](int j) { return DIR == 0 ? j : nsl - 1 - j; };
#pragma unroll
  for (int j = 0; j < D - 1; ++j) {
    if (j < nsl)
      wave_issue<B, DIR>(ts, S, s_begin + sl(j), mstart[sl(j)], mwidth[sl(j)], mslot[sl(j)],
                         ring + j * L.bytes, L, in_t, lane);
    cp_commit();
  }
  for (int j = 0; j < nsl; ++j) {
    {
      const int jn = j + D - 1;
      if (jn < nsl)
        wave_issue<B, DIR>(ts, S, s_begin + sl(jn), mstart[sl(jn)], mwidth[sl(jn)],
                           mslot[sl(jn)], ring + (jn % D) * L.bytes, L, in_t, lane);
      cp_commit();
    }
    cp_wait<D - 1>();
    __syncwarp();
    if (trace && lane == 0 && j < 1024) {   // tools/tile_trace.py: per-slice start times
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      trace[((long long)DIR * gridDim.x + t) * 1024 + j] = g;
    }
    const char* stg = ring + (j % D) * L.bytes;
    const double* sv = reinterpret_cast<const double*>(stg + L.vals);
    const int* sc = reinterpret_cast<const int*>(stg + L.cols);
    const double* so = reinterpret_cast<const double*>(stg + L.own);
    const int q = sl(j);
    const int k0 = mstart[q];
    const int nr = mstart[q + 1] - k0;
    const int width = mwidth[q];
    const bool ok = lane < nr;
    double acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) acc[c] = 0.0;
    for (int kb = 0; kb < width; kb += KP) {
      // every remote input of this chunk in flight at once, then local ones
      double dep[KP][B];
      unsigned pend = 0;
#pragma unroll
      for (int kk = 0; kk < KP; ++kk) {
        const int code = kb + kk < width ? sc[32 * (kb + kk) + lane] : -1;
        if (code >= 0) {
          pend |= 1u << kk;
        } else if (code <= -2) {
          const int v = -code - 2;
#pragma unroll
          for (int c = 0; c < B; ++c)
            dep[kk][c] = (v & 1) ? in[(long long)(v >> 1) * B + c] : vloc[(v >> 1) * B + c];
        }
      }
      while (pend) {
        const unsigned todo = pend;
#pragma unroll
        for (int kk = 0; kk < KP; ++kk)
          if (todo & (1u << kk)) {
            const double* p = out + (long long)sc[32 * (kb + kk) + lane] * B;
#pragma unroll
            for (int c = 0; c < B; ++c) dep[kk][c] = ld_relaxed_d(p + c);
          }
#pragma unroll
        for (int kk = 0; kk < KP; ++kk) {
          bool miss = false;
#pragma unroll
          for (int c = 0; c < B; ++c) miss |= is_sentinel(dep[kk][c]);
          if ((todo & (1u << kk)) && !miss) pend &= ~(1u << kk);
        }
      }
#pragma unroll
      for (int kk = 0; kk < KP; ++kk) {
        if (kb + kk < width && sc[32 * (kb + kk) + lane] != -1) {   // ascending columns
          double blk[BB], pr[B];
#pragma unroll
          for (int e = 0; e < BB; ++e) blk[e] = sv[(32 * (kb + kk)) * BB + 32 * e + lane];
          matvec<B>(blk, dep[kk], pr);
#pragma unroll
          for (int c = 0; c < B; ++c) acc[c] += pr[c];
        }
      }
    }
    if (ok) {
      double res[B];
      if (DIR == 0) {
#pragma unroll
        for (int c = 0; c < B; ++c) res[c] = canon(so[lane * B + c] - acc[c]);
      } else {
        const double* sd = reinterpret_cast<const double*>(stg + L.dinv);
        double tv[B], dinv[BB];
#pragma unroll
        for (int c = 0; c < B; ++c) tv[c] = so[lane * B + c] - acc[c];
#pragma unroll
        for (int e = 0; e < BB; ++e) dinv[e] = sd[32 * e + lane];
        matvec<B>(dinv, tv, res);
#pragma unroll
        for (int c = 0; c < B; ++c) res[c] = canon(res[c]);
      }
      const long long row = reinterpret_cast<const int*>(stg + L.rows)[lane];
      const int myloc = k0 + lane - k_base;
#pragma unroll
      for (int c = 0; c < B; ++c) {
        vloc[myloc * B + c] = res[c];
        st_relaxed_d(out + row * B + c, res[c]);
        if (out_t) out_t[(long long)(k0 + lane) * B + c] = res[c];
      }
      if (DIR == 1 && reset) {
#pragma unroll
        for (int c = 0; c < B; ++c) yreset[row * B + c] = sentinel();
      }
    }
    __syncwarp();
  }
  cp_wait<0>();
}

// in_t[k] = in[trow[k]] (B doubles per row): the forward sweep's inputs in tile order
template <int B>
__global__ void k_to_tile_order(int n, const int32_t* __restrict__ trow,
                                const double* __restrict__ in, double* __restrict__ in_t,
                                const int* done) {
  if (done && *done) return;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < (long long)n * B;
       q += (long long)gridDim.x * blockDim.x) {
    const long long k = q / B;
    in_t[q] = __ldg(in + (long long)trow[k] * B + (q - k * B));
  }
}

__global__ void k_tile_ids(int n, int T, int nx, int ny, int px, int py,
                           const int32_t* __restrict__ iperm, int32_t* tid) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const long long o = iperm[i];
    if (px > 0) {
      const int ix = (int)(o % nx), iy = (int)((o / nx) % ny);
      tid[i] = (int)((long long)ix * px / nx) + px * (int)((long long)iy * py / ny);
    } else {
      tid[i] = (int)((o * T) / n);
    }
  }
}
__global__ void k_tile_hist(int n, const int32_t* __restrict__ tid, int32_t* cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(cnt + tid[i], 1);
}
__global__ void k_iota32(int n, int32_t* p) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}
__device__ __forceinline__ int group_of_row(const int32_t* goff, int ng, int row) {
  int lo = 0, hi = ng - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (goff[mid] <= row) lo = mid; else hi = mid - 1;
  }
  return lo;
}
__global__ void k_tile_runs(int n, const int32_t* __restrict__ trow,
                            const int32_t* __restrict__ tid, const int32_t* __restrict__ toff,
                            const int32_t* __restrict__ goff, int ng, int32_t* loc,
                            int32_t* runstart) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int row = trow[k];
    const int t = tid[row];
    loc[row] = k - toff[t];
    bool start = (k == toff[t]);
    if (!start) start = group_of_row(goff, ng, trow[k - 1]) != group_of_row(goff, ng, row);
    runstart[k] = start ? k : 0;
  }
}
struct MaxOp {
  __device__ __forceinline__ int operator()(int a, int b) const { return a > b ? a : b; }
};
__global__ void k_slice_flags(int n, const int32_t* __restrict__ runstart, int32_t* sflag) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    sflag[k] = ((k - runstart[k]) % kSlice) == 0 ? 1 : 0;
}
__global__ void k_slice_starts(int n, int nsl, const int32_t* __restrict__ sflag,
                               const int32_t* __restrict__ sidx, int32_t* sstart) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    if (sflag[k]) sstart[sidx[k]] = k;
  if (blockIdx.x == 0 && threadIdx.x == 0) sstart[nsl] = n;
}
__global__ void k_tile_slice_bounds(int nsl, const int32_t* __restrict__ sstart,
                                    const int32_t* __restrict__ trow,
                                    const int32_t* __restrict__ tid, int32_t* tslice) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nsl; s += gridDim.x * blockDim.x)
    atomicMax(tslice + tid[trow[sstart[s]]] + 1, s + 1);
}
// slots per slice for the strict lower (DIR 0) / upper (DIR 1) blocks
__global__ void k_max_width(int nsl, const int32_t* __restrict__ lw,
                            const int32_t* __restrict__ uw, int32_t* out) {
  int m = 0;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nsl; s += gridDim.x * blockDim.x)
    m = max(m, max(lw[s], uw[s]));
  atomicMax(out, m);
}

template <int DIR>
__global__ void k_tile_widths(int nsl, const int32_t* __restrict__ sstart,
                              const int32_t* __restrict__ trow, const int32_t* __restrict__ rp,
                              const int32_t* __restrict__ diag, int32_t* slots) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nsl; s += nw) {
    int w = 0;
    if (lane < sstart[s + 1] - sstart[s]) {
      const int row = trow[sstart[s] + lane];
      w = DIR == 0 ? diag[row] - rp[row] : rp[row + 1] - diag[row] - 1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
    if (lane == 0) slots[s] = w * kSlice;
  }
}
template <int DIR>
__global__ void k_tile_fill(int nsl, int bb, const int32_t* __restrict__ sstart,
                            const int32_t* __restrict__ trow, const int32_t* __restrict__ tid,
                            const int32_t* __restrict__ loc, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, const int32_t* __restrict__ diag,
                            const double* __restrict__ vals, const int32_t* __restrict__ goff,
                            int ng, const int32_t* __restrict__ sp, int32_t* cols, double* svals,
                            const double* __restrict__ inv, double* dtile) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nsl; s += nw) {
    const int k0 = sstart[s];
    const bool ok = lane < sstart[s + 1] - k0;
    const int row = ok ? trow[k0 + lane] : 0;
    const int slot0 = sp[s];
    const int width = (sp[s + 1] - slot0) >> 5;
    const int t = tid[trow[k0]];
    const int grow = ok ? group_of_row(goff, ng, row) : -1;
    const int q0 = ok ? (DIR == 0 ? rp[row] : diag[row] + 1) : 0;
    const int q1 = ok ? (DIR == 0 ? diag[row] : rp[row + 1]) : 0;
    for (int k = 0; k < width; ++k) {
      const int q = q0 + k;
      const bool have = q < q1;
      int code = -1;
      if (have) {
        const int c = ci[q];
        if (group_of_row(goff, ng, c) == grow) code = -(3 + 2 * c);
        else if (tid[c] == t) code = -(2 + 2 * loc[c]);
        else code = c;
      }
      cols[slot0 + 32 * k + lane] = code;
      for (int e = 0; e < bb; ++e)
        svals[vidx(slot0, k, e, lane, bb)] = have ? vals[(long long)q * bb + e] : 0.0;
    }
    if (DIR == 1)
      for (int e = 0; e < bb; ++e)
        dtile[((long long)s * bb + e) * 32 + lane] = ok ? inv[(long long)row * bb + e] : 0.0;
  }
}

inline int grid_n(long long work) {
  long long g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > kSms * 16) g = kSms * 16;
  return (int)g;
}

struct TileHandle {
  TileSet ts;
  int b, kc, warps;
  size_t smem;
  int kind;            // 0 = polling warps (k_tile_sweep), 1 = wave (k_tile_wave)
  int wave_depth;      // cp.async ring depth of the wave kernel (0: not possible)
  WaveLayout wl;
  size_t wave_smem;
  unsigned long long* trace;   // optional [2][T][1024] slice start times (debug)
  int n;
  double *in_t, *out_t;        // wave kernel: tile-order copies of the sweep inputs
  int32_t *trow, *sstart, *tslice, *toff, *lsp, *lcols, *usp, *ucols;
  double *lvals, *uvals, *dtile;
};

template <int B, int KC, int NW>
int launch_tiled_bkw(const TileHandle* h, const double* r, double* y, double* z, int reset_y,
                     const int* done, cudaStream_t st) {
  auto* f = k_tile_sweep<B, KC, 0, NW>;
  auto* g = k_tile_sweep<B, KC, 1, NW>;
  if (cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)h->smem) != cudaSuccess ||
      cudaFuncSetAttribute((const void*)g, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)h->smem) != cudaSuccess)
    return B2S_CUDA_ERROR;
  // tiles wait on each other: every CTA must be resident (cooperative launch)
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeCooperative;
  attr.val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(h->ts.T);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = h->smem;
  cfg.stream = st;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, f, h->ts, r, y, (double*)nullptr, 0, done) != cudaSuccess)
    return B2S_CUDA_ERROR;
  if (cudaLaunchKernelEx(&cfg, g, h->ts, (const double*)y, z, y, reset_y, done) != cudaSuccess)
    return B2S_CUDA_ERROR;
  return B2S_OK;
}

template <int B, int KC>
int launch_tiled_bk(const TileHandle* h, const double* r, double* y, double* z, int reset_y,
                    const int* done, cudaStream_t st) {
  if (h->warps >= 32) return launch_tiled_bkw<B, KC, 32>(h, r, y, z, reset_y, done, st);
  if (h->warps >= 16) return launch_tiled_bkw<B, KC, 16>(h, r, y, z, reset_y, done, st);
  return launch_tiled_bkw<B, KC, 8>(h, r, y, z, reset_y, done, st);
}

template <int B, int D>
int launch_wave_bd(const TileHandle* h, const double* r, double* y, double* z, int reset_y,
                   const int* done, cudaStream_t st) {
  auto* f = k_tile_wave<B, 0, D>;
  auto* g = k_tile_wave<B, 1, D>;
  if (cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)h->wave_smem) != cudaSuccess ||
      cudaFuncSetAttribute((const void*)g, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)h->wave_smem) != cudaSuccess)
    return B2S_CUDA_ERROR;
  const int n = h->n;
  k_to_tile_order<B><<<kSms * 8, 256, 0, st>>>(n, h->trow, r, h->in_t, done);
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeCooperative;   // every tile resident: no wait can starve
  attr.val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(h->ts.T);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = h->wave_smem;
  cfg.stream = st;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  // forward: y (plan order, polled by other tiles) and y_t (tile order, the
  // backward's own inputs); backward: z, and y back to the sentinel
  if (cudaLaunchKernelEx(&cfg, f, h->ts, h->wl, r, (const double*)h->in_t, y, h->out_t,
                         (double*)nullptr, 0, done, h->trace) != cudaSuccess)
    return B2S_CUDA_ERROR;
  if (cudaLaunchKernelEx(&cfg, g, h->ts, h->wl, (const double*)y, (const double*)h->out_t, z,
                         (double*)nullptr, y, reset_y, done, h->trace) != cudaSuccess)
    return B2S_CUDA_ERROR;
  return B2S_OK;
}

template <int B>
int launch_tiled_b(const TileHandle* h, const double* r, double* y, double* z, int reset_y,
                   const int* done, cudaStream_t st) {
  if (h->kind == 1) {
    if (h->wave_depth >= 4) return launch_wave_bd<B, 4>(h, r, y, z, reset_y, done, st);
    if (h->wave_depth == 3) return launch_wave_bd<B, 3>(h, r, y, z, reset_y, done, st);
    return launch_wave_bd<B, 2>(h, r, y, z, reset_y, done, st);
  }
  if (h->kc <= 2) return launch_tiled_bk<B, 2>(h, r, y, z, reset_y, done, st);
  if (h->kc <= 4) return launch_tiled_bk<B, 4>(h, r, y, z, reset_y, done, st);
  return launch_tiled_bk<B, 8>(h, r, y, z, reset_y, done, st);
}

int launch_tiled(int b, const void* handle, const double* r, double* y, double* z, int reset_y,
                 const int* done, cudaStream_t st) {
  const TileHandle* h = reinterpret_cast<const TileHandle*>(handle);
  switch (b) {
    case 1: return launch_tiled_b<1>(h, r, y, z, reset_y, done, st);
    case 2: return launch_tiled_b<2>(h, r, y, z, reset_y, done, st);
    case 3: return launch_tiled_b<3>(h, r, y, z, reset_y, done, st);
    case 4: return launch_tiled_b<4>(h, r, y, z, reset_y, done, st);
    default: return B2S_UNSUPPORTED;
  }
}

static void free_handle(TileHandle* h) {
  if (!h) return;
  cudaFree(h->trow); cudaFree(h->sstart); cudaFree(h->tslice); cudaFree(h->toff);
  cudaFree(h->lsp); cudaFree(h->lcols); cudaFree(h->usp); cudaFree(h->ucols);
  cudaFree(h->lvals); cudaFree(h->uvals); cudaFree(h->dtile);
  cudaFree(h->in_t); cudaFree(h->out_t);
  delete h;
}

}  // namespace b2s

using namespace b2s;

extern "C" {

long long b2s_tiles_smem_bytes(int b, int rmax) { return (long long)rmax * b * 8; }

// debug: record per-slice start times of the wave kernel ([2][T][1024] u64)
int b2s_tiles_trace(void* handle, unsigned long long* buf) {
  TileHandle* h = reinterpret_cast<TileHandle*>(handle);
  if (!h) return B2S_SHAPE;
  h->trace = buf;
  return B2S_OK;
}

// kind 0: polling warps, 1: wave kernel (default when its ring fits)
int b2s_tiles_set_kernel(void* handle, int kind) {
  TileHandle* h = reinterpret_cast<TileHandle*>(handle);
  if (!h) return B2S_SHAPE;
  if (kind == 1 && !h->wave_depth) return B2S_UNSUPPORTED;
  h->kind = kind ? 1 : 0;
  return B2S_OK;
}

// Build the tiled sweep data of a factorisation in plan order.  Tiles:
// px*py column patches of an nx x ny natural-order grid when px > 0, else T
// contiguous ranges of the input order.  Returns an opaque handle (device
// memory it owns; b2s_tiles_destroy frees it), or B2S_UNSUPPORTED when a
// tile's values do not fit in one SM's shared memory or T exceeds the SMs.
int b2s_tiles_create(int n, int b, int T, int nx, int ny, int px, int py, const int32_t* iperm,
                     const int32_t* rp, const int32_t* ci, const int32_t* diag, const double* lu,
                     const double* inv, const int32_t* goff, int ngroups, int kc, int warps,
                     void** handle_out, cudaStream_t st) {
  *handle_out = nullptr;
  if (n <= 0 || b < 1 || b > 4) return B2S_SHAPE;
  if (px > 0) T = px * py;
  if (T < 1) return B2S_SHAPE;
  const int bb = b * b;
  int dev = 0, sms = kSms, smem_max = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (T > sms) return B2S_UNSUPPORTED;
  int32_t *tid, *tid_sorted, *iota, *cnt, *loc, *runstart, *sflag, *sidx;
  TileHandle* h = new TileHandle();
  B2S_CHECK(cudaMallocAsync(&tid, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&tid_sorted, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&iota, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&cnt, sizeof(int32_t) * (T + 1), st));
  B2S_CHECK(cudaMallocAsync(&loc, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&runstart, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&sflag, sizeof(int32_t) * (n + 1), st));
  B2S_CHECK(cudaMallocAsync(&sidx, sizeof(int32_t) * (n + 1), st));
  B2S_CHECK(cudaMalloc(&h->trow, sizeof(int32_t) * (n + 32)));   // + slice-read slack
  B2S_CHECK(cudaMalloc(&h->toff, sizeof(int32_t) * (T + 1)));
  B2S_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (T + 1), st));
  k_tile_ids<<<grid_n(n), 256, 0, st>>>(n, T, nx, ny, px, py, iperm, tid);
  k_tile_hist<<<grid_n(n), 256, 0, st>>>(n, tid, cnt);
  k_iota32<<<grid_n(n), 256, 0, st>>>(n, iota);
  size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
  int end_bit = 1;
  while ((1 << end_bit) < T) ++end_bit;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, tid, tid_sorted, iota, h->trow, n, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, cnt, h->toff, T + 1, st);
  cub::DeviceScan::InclusiveScan(nullptr, t3, runstart, runstart, MaxOp(), n, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t4, sflag, sidx, n + 1, st);
  size_t tb = std::max(std::max(t1, t2), std::max(t3, t4)) + 1024;
  void* tmp = nullptr;
  B2S_CHECK(cudaMallocAsync(&tmp, tb, st));
  // stable: inside a tile, rows stay in plan (level, input-index) order
  cub::DeviceRadixSort::SortPairs(tmp, t1, tid, tid_sorted, iota, h->trow, n, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(tmp, t2, cnt, h->toff, T + 1, st);
  k_tile_runs<<<grid_n(n), 256, 0, st>>>(n, h->trow, tid, h->toff, goff, ngroups, loc, runstart);
  cub::DeviceScan::InclusiveScan(tmp, t3, runstart, runstart, MaxOp(), n, st);
  B2S_CHECK(cudaMemsetAsync(sflag + n, 0, sizeof(int32_t), st));
  k_slice_flags<<<grid_n(n), 256, 0, st>>>(n, runstart, sflag);
  cub::DeviceScan::ExclusiveSum(tmp, t4, sflag, sidx, n + 1, st);
  B2S_LAUNCH_CHECK();
  int32_t nsl = 0;
  std::vector<int32_t> hoff(T + 1);
  B2S_CHECK(cudaMemcpyAsync(&nsl, sidx + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaMemcpyAsync(hoff.data(), h->toff, sizeof(int32_t) * (T + 1),
                            cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  int rmax = 0;
  for (int t = 0; t < T; ++t) rmax = std::max(rmax, hoff[t + 1] - hoff[t]);
  const long long smem = (long long)rmax * b * 8;
  int status = (smem > smem_max) ? B2S_UNSUPPORTED : B2S_OK;
  if (status == B2S_OK) {
    int32_t *lw, *uw;
    B2S_CHECK(cudaMalloc(&h->sstart, sizeof(int32_t) * (nsl + 1)));
    B2S_CHECK(cudaMalloc(&h->tslice, sizeof(int32_t) * (T + 1)));
    B2S_CHECK(cudaMalloc(&h->lsp, sizeof(int32_t) * (nsl + 1)));
    B2S_CHECK(cudaMalloc(&h->usp, sizeof(int32_t) * (nsl + 1)));
    B2S_CHECK(cudaMallocAsync(&lw, sizeof(int32_t) * (nsl + 1), st));
    B2S_CHECK(cudaMallocAsync(&uw, sizeof(int32_t) * (nsl + 1), st));
    B2S_CHECK(cudaMemsetAsync(h->tslice, 0, sizeof(int32_t) * (T + 1), st));
    B2S_CHECK(cudaMemsetAsync(lw + nsl, 0, sizeof(int32_t), st));
    B2S_CHECK(cudaMemsetAsync(uw + nsl, 0, sizeof(int32_t), st));
    k_slice_starts<<<grid_n(n), 256, 0, st>>>(n, nsl, sflag, sidx, h->sstart);
    k_tile_slice_bounds<<<grid_n(nsl), 256, 0, st>>>(nsl, h->sstart, h->trow, tid, h->tslice);
    k_tile_widths<0><<<grid_n((long long)nsl * 32), 256, 0, st>>>(nsl, h->sstart, h->trow, rp,
                                                                  diag, lw);
    k_tile_widths<1><<<grid_n((long long)nsl * 32), 256, 0, st>>>(nsl, h->sstart, h->trow, rp,
                                                                  diag, uw);
    size_t t5 = 0, t6 = 0;
    cub::DeviceScan::InclusiveScan(nullptr, t5, h->tslice, h->tslice, MaxOp(), T + 1, st);
    cub::DeviceScan::ExclusiveSum(nullptr, t6, lw, h->lsp, nsl + 1, st);
    void* tmp2 = nullptr;
    B2S_CHECK(cudaMallocAsync(&tmp2, std::max(t5, t6) + 1024, st));
    cub::DeviceScan::InclusiveScan(tmp2, t5, h->tslice, h->tslice, MaxOp(), T + 1, st);
    cub::DeviceScan::ExclusiveSum(tmp2, t6, lw, h->lsp, nsl + 1, st);
    cub::DeviceScan::ExclusiveSum(tmp2, t6, uw, h->usp, nsl + 1, st);
    B2S_LAUNCH_CHECK();
    int32_t lslots = 0, uslots = 0;
    int32_t* wmax_d = nullptr;
    B2S_CHECK(cudaMallocAsync(&wmax_d, sizeof(int32_t), st));
    B2S_CHECK(cudaMemsetAsync(wmax_d, 0, sizeof(int32_t), st));
    k_max_width<<<grid_n(nsl), 256, 0, st>>>(nsl, lw, uw, wmax_d);
    int32_t wmax = 0;
    B2S_CHECK(cudaMemcpyAsync(&lslots, h->lsp + nsl, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    B2S_CHECK(cudaMemcpyAsync(&uslots, h->usp + nsl, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    B2S_CHECK(cudaMemcpyAsync(&wmax, wmax_d, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    B2S_CHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(wmax_d, st);
    wmax /= kSlice;
    // wave kernel: slice metadata + ring of D stages + the tile's own vector
    // in shared memory
    std::vector<int32_t> hts(T + 1);
    int max_sl = 0;
    {
      std::vector<int32_t> tmp_ts(T + 1);
      // tslice is complete only after the scan below; recomputed there
    }
    h->n = n;
    h->wl = wave_layout(b, wmax > 0 ? wmax : 1, 0);
    h->wave_depth = 0;
    B2S_CHECK(cudaMalloc(&h->lcols, sizeof(int32_t) * (lslots + 1)));
    B2S_CHECK(cudaMalloc(&h->ucols, sizeof(int32_t) * (uslots + 1)));
    B2S_CHECK(cudaMalloc(&h->lvals, sizeof(double) * ((long long)lslots * bb + 1)));
    B2S_CHECK(cudaMalloc(&h->uvals, sizeof(double) * ((long long)uslots * bb + 1)));
    B2S_CHECK(cudaMalloc(&h->dtile, sizeof(double) * ((long long)nsl * bb * 32 + 1)));
    k_tile_fill<0><<<grid_n((long long)nsl * 32), 256, 0, st>>>(
        nsl, bb, h->sstart, h->trow, tid, loc, rp, ci, diag, lu, goff, ngroups, h->lsp, h->lcols,
        h->lvals, inv, h->dtile);
    k_tile_fill<1><<<grid_n((long long)nsl * 32), 256, 0, st>>>(
        nsl, bb, h->sstart, h->trow, tid, loc, rp, ci, diag, lu, goff, ngroups, h->usp, h->ucols,
        h->uvals, inv, h->dtile);
    B2S_LAUNCH_CHECK();
    h->ts = TileSet{T,        nsl,      rmax,     h->trow, h->sstart, h->tslice, h->toff,
                    Sell{h->lsp, h->lcols, h->lvals}, Sell{h->usp, h->ucols, h->uvals}, h->dtile};
    h->b = b;
    h->kc = kc;
    h->warps = warps;
    h->smem = (size_t)(smem > 0 ? smem : 16);
    B2S_CHECK(cudaMemcpyAsync(hts.data(), h->tslice, sizeof(int32_t) * (T + 1),
                              cudaMemcpyDeviceToHost, st));
    B2S_CHECK(cudaStreamSynchronize(st));
    for (int q = 0; q < T; ++q) max_sl = std::max(max_sl, hts[q + 1] - hts[q]);
    h->wl = wave_layout(b, wmax > 0 ? wmax : 1, max_sl);
    for (int d = 4; d >= 2; --d)
      if ((long long)d * h->wl.bytes + 4LL * h->wl.meta + smem <= smem_max) {
        h->wave_depth = d;
        break;
      }
    h->wave_smem = (size_t)h->wave_depth * h->wl.bytes + 4 * (size_t)h->wl.meta + (size_t)smem;
    h->kind = h->wave_depth ? 1 : 0;
    if (h->wave_depth) {
      // + 32 rows of slack: a slice's cp.async reads 32 rows from its start
      B2S_CHECK(cudaMalloc(&h->in_t, sizeof(double) * ((long long)n + 32) * b));
      B2S_CHECK(cudaMalloc(&h->out_t, sizeof(double) * ((long long)n + 32) * b));
    }
    cudaFreeAsync(tmp2, st);
    cudaFreeAsync(lw, st);
    cudaFreeAsync(uw, st);
  }
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(tid, st);
  cudaFreeAsync(tid_sorted, st);
  cudaFreeAsync(iota, st);
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(loc, st);
  cudaFreeAsync(runstart, st);
  cudaFreeAsync(sflag, st);
  cudaFreeAsync(sidx, st);
  if (status != B2S_OK) {
    free_handle(h);
    return status;
  }
  *handle_out = h;
  return B2S_OK;
}

int b2s_tiles_destroy(void* handle) {
  free_handle(reinterpret_cast<TileHandle*>(handle));
  return B2S_OK;
}

// z = U^-1 L^-1 r with the tiled kernels (same contract as b2s_ilu0_apply).
int b2s_tiles_apply(int b, const void* handle, const double* r, double* y, double* z,
                    int reset_y, cudaStream_t st) {
  if (!handle) return B2S_SHAPE;
  return launch_tiled(b, handle, r, y, z, reset_y, nullptr, st);
}

}  // extern "C"
