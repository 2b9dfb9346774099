// Tiled ILU0 sweeps: the level-scheduled forward/backward block-triangular
// solves (bs/ilu0.py:105-142) with most dependencies resolved on-chip.
//
// Why: in the sync-free sweep (ilu0.cu) every one of the ~300 levels of a
// 1M-cell stencil costs a cross-SM L2 round trip (~1.2 us measured), so the
// sweep is latency-bound at ~0.1 of the HBM roofline.  Here the rows are
// partitioned into T tiles (one CTA per SM, all co-resident); a tile keeps
// the values of its own rows in shared memory, so a dependency inside the
// tile costs a shared-memory load instead of an L2 round trip.  Only
// dependencies that cross a tile boundary are polled from global memory
// (sentinel protocol as in ilu0.cu).  Tiles are contiguous ranges of the
// *input* row order, which for reservoir grids in natural order are slabs:
// most couplings stay inside a tile.
//
// Per CTA: warp 0 is a TMA producer that streams the tile's pre-packed
// records (one per slice of <= 32 same-level rows: row ids, entry codes, the
// b x b blocks in lane-interleaved order and, backward, the inverse
// diagonal) through a ring of shared-memory stages with cp.async.bulk +
// mbarrier complete_tx; warp 1 consumes the records in order.  Rows of one
// slice are independent (same level), and every dependency lies in an
// earlier slice of the same tile (shared memory, already final because the
// consumer is one warp processing slices in order) or in another tile
// (polled).  Per-row arithmetic is identical to the reference: products
// summed in ascending column order, then subtracted; backward multiplies by
// inv(U_ii).  Results are bit-identical to the sync-free kernels.
//
// Entry codes: c >= 0 remote row c (poll); -1 padding; -(2 + 2*loc) local
// slot `loc` of this tile; -(3 + 2*c) same-group row c (read the vector as it
// was before the sweep, as the reference does for rows of one group).
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "sell.cuh"

namespace b2s {

constexpr int kChunkBytes = 8192;                 // one TMA transfer / ring stage
constexpr int kChunkWords = kChunkBytes / 8;
constexpr int kStages = 6;                        // ring depth (48 KB)
constexpr int kRingWords = kChunkWords * kStages;

struct TileSet {
  int T;                       // tiles (= CTAs)
  int rmax;                    // largest tile (rows) -> shared values
  const long long* fbeg;       // [T+1] forward stream word offsets per tile
  const double* fstream;
  const long long* bbeg;       // [T+1] backward stream word offsets per tile
  const double* bstream;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile(
      "{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ double ld_relaxed_d(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_d(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// record layout (8-byte words): [0] header: nrows | width<<8 | loc0<<32;
// [1..16] 32 int32 row ids; [17..17+16w) w x 32 int32 entry codes;
// then w*BB*32 values (k, e, lane); backward: + BB*32 inverse-diagonal words.
__host__ __device__ __forceinline__ long long rec_words(int w, int bb, bool diag) {
  long long words = 1 + 16 + 16ll * w + (long long)w * bb * 32 + (diag ? bb * 32 : 0);
  return (words + 1) & ~1ll;  // 16-byte multiple
}

// ---------------------------------------------------------------- the sweep
// DIR = 0 forward (y = L^-1 r), 1 backward (z = U^-1 y).
template <int B, int DIR>
__global__ void __launch_bounds__(64, 1) k_tiled_sweep(TileSet ts, const double* __restrict__ in,
                                                        double* out, double* yreset, int reset,
                                                        const int* done) {
  constexpr int BB = B * B;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kRingWords);
  uint64_t* empty = full + kStages;
  double* vloc = reinterpret_cast<double*>(empty + kStages);  // tile values
  if (done && *done) return;
  const int t = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long* beg = DIR == 0 ? ts.fbeg : ts.bbeg;
  const double* stream = DIR == 0 ? ts.fstream : ts.bstream;
  const long long s0 = beg[t], s1 = beg[t + 1];
  const long long total = s1 - s0;
  const int nchunks = (int)((total + kChunkWords - 1) / kChunkWords);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {  // ---------------- producer: stream the tile's records
    if (lane == 0) {
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % kStages;
        if (c >= kStages) mbar_wait(empty + s, ((c / kStages) - 1) & 1);
        const long long off = (long long)c * kChunkWords;
        long long words = total - off;
        if (words > kChunkWords) words = kChunkWords;
        const unsigned bytes = (unsigned)(words * 8);
        mbar_expect_tx(full + s, bytes);
        tma_load(ring + (long long)s * kChunkWords, stream + s0 + off, bytes, full + s);
      }
    }
    return;
  }

  // ------------------------------------ consumer (warp 1): records in order
  long long cur = 0;          // word offset in the tile stream
  long long avail = 0;        // words known to have landed
  int next_chunk = 0;         // first chunk not yet waited for
  int released = 0;           // chunks handed back to the producer
  auto ensure = [&](long long end_word) {
    while (avail < end_word && next_chunk < nchunks) {
      mbar_wait(full + (next_chunk % kStages), (next_chunk / kStages) & 1);
      ++next_chunk;
      avail = (long long)next_chunk * kChunkWords;
    }
  };
  auto word = [&](long long w) -> double { return ring[w % kRingWords]; };
  auto iword = [&](long long w, int half) -> int {
    const int2 v = *reinterpret_cast<const int2*>(ring + (w % kRingWords));
    return half ? v.y : v.x;
  };
  while (cur < total) {
    ensure(cur + 17);
    const unsigned long long hdr = (unsigned long long)__double_as_longlong(word(cur));
    const int nrows = (int)(hdr & 0xff);
    const int width = (int)((hdr >> 8) & 0xffffff);
    const int loc0 = (int)(hdr >> 32);
    const long long len = rec_words(width, BB, DIR == 1);
    ensure(cur + len);
    const bool ok = lane < nrows;
    const int row = iword(cur + 1 + (lane >> 1), lane & 1);
    double own[B], acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      own[c] = ok ? in[(long long)row * B + c] : 0.0;  // r (fwd) or y (bwd)
      acc[c] = 0.0;
    }
    const long long cbase = cur + 17, vbase = cur + 17 + 16ll * width;
#pragma unroll 2
    for (int k = 0; k < width; ++k) {
      const int code = iword(cbase + 16ll * k + (lane >> 1), lane & 1);
      if (code == -1) continue;
      double dep[B];
      if (code >= 0) {  // another tile: poll the published value
        const double* p = out + (long long)code * B;
        bool miss;
        do {
          miss = false;
#pragma unroll
          for (int c = 0; c < B; ++c) {
            dep[c] = ld_relaxed_d(p + c);
            miss |= is_sentinel(dep[c]);
          }
        } while (miss);
      } else if (((-code - 2) & 1) == 0) {  // this tile: shared memory
        const int loc = (-code - 2) >> 1;
#pragma unroll
        for (int c = 0; c < B; ++c) dep[c] = vloc[loc * B + c];
      } else {  // same group: value before this sweep
        const long long rr = (-code - 3) >> 1;
#pragma unroll
        for (int c = 0; c < B; ++c) dep[c] = in[rr * B + c];
      }
      double blk[BB], pr[B];
#pragma unroll
      for (int e = 0; e < BB; ++e) blk[e] = word(vbase + (long long)(k * BB + e) * 32 + lane);
      matvec<B>(blk, dep, pr);
#pragma unroll
      for (int c = 0; c < B; ++c) acc[c] += pr[c];
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
        const long long dbase = vbase + (long long)width * BB * 32;
#pragma unroll
        for (int e = 0; e < BB; ++e) dinv[e] = word(dbase + (long long)e * 32 + lane);
        matvec<B>(dinv, tv, res);
#pragma unroll
        for (int c = 0; c < B; ++c) res[c] = canon(res[c]);
      }
#pragma unroll
      for (int c = 0; c < B; ++c) {
        vloc[(loc0 + lane) * B + c] = res[c];
        st_relaxed_d(out + (long long)row * B + c, res[c]);
      }
      if (DIR == 1 && reset) {
#pragma unroll
        for (int c = 0; c < B; ++c) yreset[(long long)row * B + c] = sentinel();
      }
    }
    __syncwarp();
    cur += len;
    // hand fully consumed chunks back to the producer
    const int consumed = (int)(cur / kChunkWords);
    while (released < consumed && released < next_chunk) {
      if (lane == 0) mbar_arrive(empty + (released % kStages));
      ++released;
    }
  }
}

// ---------------------------------------------------------------- building
// tile id of a plan-order row: its input (original) index in T equal ranges
__global__ void k_tile_ids(int n, int T, const int32_t* __restrict__ iperm, int32_t* tid) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    tid[i] = (int)(((long long)iperm[i] * T) / n);
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
// per list position k (rows grouped by tile): local slot of the row and the
// start of its run (same tile, same group) as a candidate for a max-scan
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
__global__ void k_slice_starts(int n, const int32_t* __restrict__ sflag,
                               const int32_t* __restrict__ sidx, int32_t* sstart) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    if (sflag[k]) sstart[sidx[k]] = k;
}
// record widths: one warp per slice, lanes = rows
__global__ void k_slice_widths(int nsl, int n, const int32_t* __restrict__ sstart,
                               const int32_t* __restrict__ trow, const int32_t* __restrict__ rp,
                               const int32_t* __restrict__ ci, const int32_t* __restrict__ diag,
                               int bb, long long* fwords, long long* bwords) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nsl; s += nw) {
    const int k0 = sstart[s], k1 = (s + 1 < nsl) ? sstart[s + 1] : n;
    int wl = 0, wu = 0;
    if (lane < k1 - k0) {
      const int row = trow[k0 + lane];
      wl = diag[row] - rp[row];
      wu = rp[row + 1] - diag[row] - 1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      wl = max(wl, __shfl_xor_sync(0xffffffffu, wl, o));
      wu = max(wu, __shfl_xor_sync(0xffffffffu, wu, o));
    }
    if (lane == 0) {
      fwords[s] = rec_words(wl, bb, false);
      bwords[s] = rec_words(wu, bb, true);
    }
  }
}
// backward streams hold each tile's slices in reverse order
__global__ void k_reverse_index(int nsl, const int32_t* __restrict__ sstart,
                                const int32_t* __restrict__ trow, const int32_t* __restrict__ tid,
                                const int32_t* __restrict__ tslice, int32_t* bpos) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nsl; s += gridDim.x * blockDim.x) {
    const int t = tid[trow[sstart[s]]];
    bpos[s] = tslice[t] + (tslice[t + 1] - 1 - s);  // slot of slice s in the backward order
  }
}
__global__ void k_tile_slice_bounds(int nsl, const int32_t* __restrict__ sstart,
                                    const int32_t* __restrict__ trow,
                                    const int32_t* __restrict__ tid, int32_t* tslice_last) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nsl; s += gridDim.x * blockDim.x) {
    const int t = tid[trow[sstart[s]]];
    atomicMax(tslice_last + t + 1, s + 1);
  }
}
__global__ void k_permute_ll(int nsl, const int32_t* __restrict__ pos,
                             const long long* __restrict__ in, long long* out) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nsl; s += gridDim.x * blockDim.x)
    out[pos[s]] = in[s];
}
// fill one record per slice (warp per slice)
template <int DIR>
__global__ void k_fill_records(int nsl, int n, int bb, const int32_t* __restrict__ sstart,
                               const int32_t* __restrict__ trow, const int32_t* __restrict__ tid,
                               const int32_t* __restrict__ loc, const int32_t* __restrict__ toff,
                               const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               const int32_t* __restrict__ diag, const double* __restrict__ vals,
                               const double* __restrict__ inv, const int32_t* __restrict__ goff,
                               int ng, const long long* __restrict__ roff,
                               const int32_t* __restrict__ bpos, double* stream) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nsl; s += nw) {
    const int k0 = sstart[s], k1 = (s + 1 < nsl) ? sstart[s + 1] : n;
    const int nr = k1 - k0;
    const bool ok = lane < nr;
    const int row = ok ? trow[k0 + lane] : -1;
    int w = 0;
    if (ok) w = DIR == 0 ? diag[row] - rp[row] : rp[row + 1] - diag[row] - 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
    const long long base = roff[DIR == 0 ? s : bpos[s]];
    double* rec = stream + base;
    const int t = tid[trow[k0]];
    const int loc0 = loc[trow[k0]];
    if (lane == 0) {
      const unsigned long long hdr = (unsigned long long)nr | ((unsigned long long)w << 8) |
                                     ((unsigned long long)(unsigned)loc0 << 32);
      rec[0] = __longlong_as_double((long long)hdr);
    }
    int* rows = reinterpret_cast<int*>(rec + 1);
    rows[lane] = row;
    int* codes = reinterpret_cast<int*>(rec + 17);
    double* v = rec + 17 + 16 * w;
    const int grow = ok ? group_of_row(goff, ng, row) : -1;
    for (int k = 0; k < w; ++k) {
      int code = -1;
      const int q = ok ? (DIR == 0 ? rp[row] + k : diag[row] + 1 + k) : -1;
      const bool have = ok && (DIR == 0 ? q < diag[row] : q < rp[row + 1]);
      if (have) {
        const int c = ci[q];
        if (group_of_row(goff, ng, c) == grow) code = -(3 + 2 * c);
        else if (tid[c] == t) code = -(2 + 2 * loc[c]);
        else code = c;
      }
      codes[k * 32 + lane] = code;
      for (int e = 0; e < bb; ++e) v[(long long)(k * bb + e) * 32 + lane] = have ? vals[(long long)q * bb + e] : 0.0;
    }
    if (DIR == 1) {
      double* d = v + (long long)w * bb * 32;
      for (int e = 0; e < bb; ++e) d[e * 32 + lane] = ok ? inv[(long long)row * bb + e] : 0.0;
    }
    (void)toff;
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
  long long *fbeg, *bbeg;
  double *fstream, *bstream;
  size_t smem_bytes;
};

template <int B>
int launch_tiled_b(const TileHandle* h, const double* r, double* y, double* z, int reset_y,
                   const int* done, cudaStream_t st) {
  const void* f = (const void*)k_tiled_sweep<B, 0>;
  const void* g = (const void*)k_tiled_sweep<B, 1>;
  if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->smem_bytes) !=
          cudaSuccess ||
      cudaFuncSetAttribute(g, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->smem_bytes) !=
          cudaSuccess)
    return B2S_CUDA_ERROR;
  // every tile waits on others: all CTAs must be co-resident (cooperative)
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeCooperative;
  attr.val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(h->ts.T);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = h->smem_bytes;
  cfg.stream = st;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, k_tiled_sweep<B, 0>, h->ts, (const double*)r, y, (double*)nullptr,
                         0, done) != cudaSuccess)
    return B2S_CUDA_ERROR;
  if (cudaLaunchKernelEx(&cfg, k_tiled_sweep<B, 1>, h->ts, (const double*)y, z, y, reset_y,
                         done) != cudaSuccess)
    return B2S_CUDA_ERROR;
  return B2S_OK;
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

}  // namespace b2s

using namespace b2s;

extern "C" {

// Shared memory a tile of `rmax` rows needs (ring + barriers + values).
long long b2s_tiles_smem_bytes(int b, int rmax) {
  return (long long)kRingWords * 8 + 2 * kStages * 8 + (long long)rmax * b * 8;
}

// Build the tiled sweep data for a factorisation in plan order.  T tiles
// (<= number of SMs) cut the input row order into equal ranges.  Returns an
// opaque handle (device memory owned by it; free with b2s_tiles_destroy), or
// B2S_UNSUPPORTED when a tile's values do not fit in shared memory.
int b2s_tiles_create(int n, int b, int T, const int32_t* iperm, const int32_t* rp,
                     const int32_t* ci, const int32_t* diag, const double* lu,
                     const double* inv, const int32_t* goff, int ngroups, void** handle_out,
                     cudaStream_t st) {
  *handle_out = nullptr;
  if (n <= 0 || b < 1 || b > 4 || T < 1) return B2S_SHAPE;
  const int bb = b * b;
  int dev = 0, sms = kSms, smem_max = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (T > sms) return B2S_UNSUPPORTED;
  int32_t *tid, *tid_sorted, *trow, *iota, *cnt, *toff, *loc, *runstart, *sflag, *sidx;
  B2S_CHECK(cudaMallocAsync(&tid, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&tid_sorted, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&trow, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&iota, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&cnt, sizeof(int32_t) * (T + 1), st));
  B2S_CHECK(cudaMallocAsync(&toff, sizeof(int32_t) * (T + 1), st));
  B2S_CHECK(cudaMallocAsync(&loc, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&runstart, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&sflag, sizeof(int32_t) * (n + 1), st));
  B2S_CHECK(cudaMallocAsync(&sidx, sizeof(int32_t) * (n + 1), st));
  B2S_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (T + 1), st));
  k_tile_ids<<<grid_n(n), 256, 0, st>>>(n, T, iperm, tid);
  k_tile_hist<<<grid_n(n), 256, 0, st>>>(n, tid, cnt);
  k_iota32<<<grid_n(n), 256, 0, st>>>(n, iota);
  size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
  int end_bit = 1;
  while ((1 << end_bit) < T) ++end_bit;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, tid, tid_sorted, iota, trow, n, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, cnt, toff, T + 1, st);
  cub::DeviceScan::InclusiveScan(nullptr, t3, runstart, runstart, MaxOp(), n, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t4, sflag, sidx, n + 1, st);
  size_t tb = t1;
  if (t2 > tb) tb = t2;
  if (t3 > tb) tb = t3;
  if (t4 > tb) tb = t4;
  void* tmp = nullptr;
  B2S_CHECK(cudaMallocAsync(&tmp, tb + 1024, st));
  cub::DeviceRadixSort::SortPairs(tmp, t1, tid, tid_sorted, iota, trow, n, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(tmp, t2, cnt, toff, T + 1, st);
  k_tile_runs<<<grid_n(n), 256, 0, st>>>(n, trow, tid, toff, goff, ngroups, loc, runstart);
  cub::DeviceScan::InclusiveScan(tmp, t3, runstart, runstart, MaxOp(), n, st);
  B2S_CHECK(cudaMemsetAsync(sflag + n, 0, sizeof(int32_t), st));
  k_slice_flags<<<grid_n(n), 256, 0, st>>>(n, runstart, sflag);
  cub::DeviceScan::ExclusiveSum(tmp, t4, sflag, sidx, n + 1, st);
  B2S_LAUNCH_CHECK();
  int32_t nsl = 0;
  std::vector<int32_t> hoff(T + 1);
  B2S_CHECK(cudaMemcpyAsync(&nsl, sidx + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaMemcpyAsync(hoff.data(), toff, sizeof(int32_t) * (T + 1), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  int rmax = 0;
  for (int t = 0; t < T; ++t) rmax = std::max(rmax, hoff[t + 1] - hoff[t]);
  const long long smem = b2s_tiles_smem_bytes(b, rmax);
  int status = B2S_OK;
  if (smem > smem_max) status = B2S_UNSUPPORTED;
  TileHandle* h = nullptr;
  if (status == B2S_OK) {
    int32_t *sstart, *tslice, *bpos;
    long long *fw, *bw, *bw_perm, *foff, *boff;
    B2S_CHECK(cudaMallocAsync(&sstart, sizeof(int32_t) * nsl, st));
    B2S_CHECK(cudaMallocAsync(&tslice, sizeof(int32_t) * (T + 1), st));
    B2S_CHECK(cudaMallocAsync(&bpos, sizeof(int32_t) * nsl, st));
    B2S_CHECK(cudaMallocAsync(&fw, sizeof(long long) * (nsl + 1), st));
    B2S_CHECK(cudaMallocAsync(&bw, sizeof(long long) * (nsl + 1), st));
    B2S_CHECK(cudaMallocAsync(&bw_perm, sizeof(long long) * (nsl + 1), st));
    B2S_CHECK(cudaMallocAsync(&foff, sizeof(long long) * (nsl + 1), st));
    B2S_CHECK(cudaMallocAsync(&boff, sizeof(long long) * (nsl + 1), st));
    B2S_CHECK(cudaMemsetAsync(tslice, 0, sizeof(int32_t) * (T + 1), st));
    B2S_CHECK(cudaMemsetAsync(fw + nsl, 0, sizeof(long long), st));
    B2S_CHECK(cudaMemsetAsync(bw_perm + nsl, 0, sizeof(long long), st));
    k_slice_starts<<<grid_n(n), 256, 0, st>>>(n, sflag, sidx, sstart);
    k_slice_widths<<<grid_n((long long)nsl * 32), 256, 0, st>>>(nsl, n, sstart, trow, rp, ci, diag,
                                                                bb, fw, bw);
    // slices are tile-major; tslice[t+1] = one past the last slice of tile t
    k_tile_slice_bounds<<<grid_n(nsl), 256, 0, st>>>(nsl, sstart, trow, tid, tslice);
    size_t t5 = 0;
    cub::DeviceScan::InclusiveScan(nullptr, t5, tslice, tslice, MaxOp(), T + 1, st);
    size_t t6 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t6, fw, foff, nsl + 1, st);
    void* tmp2 = nullptr;
    B2S_CHECK(cudaMallocAsync(&tmp2, (t5 > t6 ? t5 : t6) + 1024, st));
    cub::DeviceScan::InclusiveScan(tmp2, t5, tslice, tslice, MaxOp(), T + 1, st);
    k_reverse_index<<<grid_n(nsl), 256, 0, st>>>(nsl, sstart, trow, tid, tslice, bpos);
    k_permute_ll<<<grid_n(nsl), 256, 0, st>>>(nsl, bpos, bw, bw_perm);
    cub::DeviceScan::ExclusiveSum(tmp2, t6, fw, foff, nsl + 1, st);
    cub::DeviceScan::ExclusiveSum(tmp2, t6, bw_perm, boff, nsl + 1, st);
    B2S_LAUNCH_CHECK();
    long long ftot = 0, btot = 0;
    std::vector<int32_t> hts(T + 1);
    B2S_CHECK(cudaMemcpyAsync(&ftot, foff + nsl, sizeof(long long), cudaMemcpyDeviceToHost, st));
    B2S_CHECK(cudaMemcpyAsync(&btot, boff + nsl, sizeof(long long), cudaMemcpyDeviceToHost, st));
    B2S_CHECK(cudaMemcpyAsync(hts.data(), tslice, sizeof(int32_t) * (T + 1), cudaMemcpyDeviceToHost, st));
    B2S_CHECK(cudaStreamSynchronize(st));
    h = new TileHandle();
    B2S_CHECK(cudaMalloc(&h->fstream, sizeof(double) * (ftot + 2)));
    B2S_CHECK(cudaMalloc(&h->bstream, sizeof(double) * (btot + 2)));
    B2S_CHECK(cudaMalloc(&h->fbeg, sizeof(long long) * (T + 1)));
    B2S_CHECK(cudaMalloc(&h->bbeg, sizeof(long long) * (T + 1)));
    // per-tile stream begins = record offsets of each tile's first slice
    std::vector<long long> hfb(T + 1), hbb(T + 1);
    std::vector<long long> hfoff(nsl + 1), hboff(nsl + 1);
    B2S_CHECK(cudaMemcpyAsync(hfoff.data(), foff, sizeof(long long) * (nsl + 1), cudaMemcpyDeviceToHost, st));
    B2S_CHECK(cudaMemcpyAsync(hboff.data(), boff, sizeof(long long) * (nsl + 1), cudaMemcpyDeviceToHost, st));
    B2S_CHECK(cudaStreamSynchronize(st));
    for (int t = 0; t <= T; ++t) {
      hfb[t] = hfoff[hts[t]];
      hbb[t] = hboff[hts[t]];
    }
    // a record must fit in the ring next to the chunk it starts in
    long long longest = 0;
    for (int s = 0; s < nsl; ++s)
      longest = std::max(longest, std::max(hfoff[s + 1] - hfoff[s], hboff[s + 1] - hboff[s]));
    if (longest > (long long)(kStages - 2) * kChunkWords) status = B2S_UNSUPPORTED;
    B2S_CHECK(cudaMemcpyAsync(h->fbeg, hfb.data(), sizeof(long long) * (T + 1), cudaMemcpyHostToDevice, st));
    B2S_CHECK(cudaMemcpyAsync(h->bbeg, hbb.data(), sizeof(long long) * (T + 1), cudaMemcpyHostToDevice, st));
    if (status != B2S_OK) {
      cudaFree(h->fstream); cudaFree(h->bstream); cudaFree(h->fbeg); cudaFree(h->bbeg);
      delete h;
      h = nullptr;
    } else {
    k_fill_records<0><<<grid_n((long long)nsl * 32), 256, 0, st>>>(
        nsl, n, bb, sstart, trow, tid, loc, toff, rp, ci, diag, lu, inv, goff, ngroups, foff, bpos,
        h->fstream);
    k_fill_records<1><<<grid_n((long long)nsl * 32), 256, 0, st>>>(
        nsl, n, bb, sstart, trow, tid, loc, toff, rp, ci, diag, lu, inv, goff, ngroups, boff, bpos,
        h->bstream);
    B2S_LAUNCH_CHECK();
    h->ts = TileSet{T, rmax, h->fbeg, h->fstream, h->bbeg, h->bstream};
    h->smem_bytes = (size_t)smem;
    }
    B2S_CHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(tmp2, st);
    cudaFreeAsync(sstart, st);
    cudaFreeAsync(tslice, st);
    cudaFreeAsync(bpos, st);
    cudaFreeAsync(fw, st);
    cudaFreeAsync(bw, st);
    cudaFreeAsync(bw_perm, st);
    cudaFreeAsync(foff, st);
    cudaFreeAsync(boff, st);
  }
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(tid, st);
  cudaFreeAsync(tid_sorted, st);
  cudaFreeAsync(trow, st);
  cudaFreeAsync(iota, st);
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(toff, st);
  cudaFreeAsync(loc, st);
  cudaFreeAsync(runstart, st);
  cudaFreeAsync(sflag, st);
  cudaFreeAsync(sidx, st);
  if (status != B2S_OK) return status;
  *handle_out = h;
  return B2S_OK;
}

int b2s_tiles_destroy(void* handle) {
  if (!handle) return B2S_OK;
  TileHandle* h = reinterpret_cast<TileHandle*>(handle);
  cudaFree(h->fstream);
  cudaFree(h->bstream);
  cudaFree(h->fbeg);
  cudaFree(h->bbeg);
  delete h;
  return B2S_OK;
}

// z = U^-1 L^-1 r with the tiled kernels (same contract as b2s_ilu0_apply).
int b2s_tiles_apply(int b, const void* handle, const double* r, double* y, double* z,
                    int reset_y, cudaStream_t st) {
  if (!handle) return B2S_SHAPE;
  return launch_tiled(b, handle, r, y, z, reset_y, nullptr, st);
}

}  // extern "C"
