// Device-side parallelism extraction: diagonal lookup, level schedule, greedy
// colouring, plan construction (stable counting order) and the symmetric
// block-CSR permutation.  Integer results are bit-exact against the
// reference (bs/analysis.py); see DESIGN.md §3.
//
// Level schedule and colouring are both "sync-free wavefronts": rows are
// handed out to warps in ascending index order through an atomic ticket, and
// each row spins until the rows it depends on (all with smaller index) have
// published their value.  Because tickets are issued in order to resident
// warps, the smallest unfinished row always has all its inputs: no deadlock,
// no grid barrier, and the critical path is the DAG depth (one L2 round
// trip per level) instead of one kernel launch per level.
#include <cub/cub.cuh>

#include "common.cuh"

namespace b2s {

__device__ __forceinline__ int ld_relaxed_i(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_i(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------
// diagonal positions (bs/blockcore.py:127-134) + first missing row
// (bs/analysis.py:79-82, bs/ilu0.py:159-161)
__global__ void k_find_diag(int n, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, int32_t* __restrict__ diag,
                            int32_t* __restrict__ first_missing) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int lo = rp[i], hi = rp[i + 1] - 1, pos = -1;
    while (lo <= hi) {  // columns are strictly increasing per row
      int mid = (lo + hi) >> 1;
      int c = ci[mid];
      if (c == i) { pos = mid; break; }
      if (c < i) lo = mid + 1; else hi = mid - 1;
    }
    diag[i] = pos;
    if (pos < 0) atomicMin(first_missing, i);
  }
}

// ---------------------------------------------------------------------------
// Neighbour lists of up to kLNb / kCNb entries are held in registers and all their
// published values are polled in one round per pass (one L2 round trip per
// dependency level instead of one per neighbour); longer lists fall back to
// a one-at-a-time walk.  A warp keeps polling while any lane still waits, so
// lanes of one slice may depend on each other (natural order).

// level(i) = 1 + max level(j) over strict-lower j, 0 without lower
// neighbours (bs/analysis.py:85-100).  level[] must be -1 on entry.
__device__ __forceinline__ void trace_row(unsigned long long* trace, int i) {
  if (trace) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    trace[i] = g;
  }
}

// A warp claims R consecutive 32-row slices per ticket (lane l holds rows
// l, l+32, ..., of the unit) and polls all of them each round.  The window of
// rows in flight is what limits these wavefronts: rows are claimed in index
// order but become ready along the (diagonal) level front, so a window
// smaller than the front's index spread throttles it (measured on C4: 1-slice
// units, ~11-23 z-planes in flight, ran at 1/4-1/7 of the hop speed).  Short
// neighbour lists in registers keep R rows per lane affordable; longer rows
// walk their list from memory.  Deadlock-free: units are claimed in order by
// running warps, and the smallest unfinished row always has its inputs.
constexpr int kLNb = 4;    // lower neighbours held in registers (level)
constexpr int kLR = 6;     // slices per warp unit (level)

__global__ void __launch_bounds__(256, 5) k_level_sync_free(int n, const int32_t* __restrict__ rp,
                                  const int32_t* __restrict__ ci, int32_t* level,
                                  unsigned int* ticket, unsigned long long* trace = nullptr) {
  const int lane = threadIdx.x & 31;
  // neighbour lists live in shared memory (registers would cap the rows in flight)
  __shared__ int snb[8][kLR][kLNb][32];
  auto nb = [&](int q, int w) -> int& { return snb[threadIdx.x >> 5][q][w][lane]; };
  for (;;) {
    unsigned int u = 0;
    if (lane == 0) u = atomicAdd(ticket, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    const long long base = (long long)u * kLR * kSlice;
    if (base >= n) break;
    unsigned pend[kLR];
    int best[kLR], k[kLR], end[kLR];
    bool longrow[kLR], live[kLR];
    // (row by row: measured faster here than issuing all rows' setup loads
    // together -- unlike the colour kernel, whose setup is twice as long)
#pragma unroll
    for (int q = 0; q < kLR; ++q) {
      const long long i = base + q * kSlice + lane;
      live[q] = i < n;
      pend[q] = 0; best[q] = -1; k[q] = 0; end[q] = 0; longrow[q] = false;
      if (live[q]) {
        k[q] = rp[i];
        end[q] = rp[i + 1];
        int cnt = 0;
        for (int t = k[q]; t < end[q]; ++t) {
          const int j = ci[t];
          if (j >= i) break;
          if (cnt < kLNb) nb(q, cnt) = j;
          ++cnt;
        }
        longrow[q] = cnt > kLNb;
        pend[q] = longrow[q] ? 0u : ((1u << cnt) - 1u);
      }
    }
    for (;;) {
      bool any = false;
#pragma unroll
      for (int q = 0; q < kLR; ++q) {
        if (!live[q]) continue;
        const int i = (int)(base + q * kSlice + lane);
        bool fin;
        if (!longrow[q]) {
          int got[kLNb];
#pragma unroll
          for (int w = 0; w < kLNb; ++w)
            got[w] = (pend[q] & (1u << w)) ? ld_relaxed_i(level + nb(q, w)) : -1;
#pragma unroll
          for (int w = 0; w < kLNb; ++w)
            if ((pend[q] & (1u << w)) && got[w] >= 0) {
              best[q] = max(best[q], got[w]);
              pend[q] &= ~(1u << w);
            }
          fin = !pend[q];
        } else {
          while (k[q] < end[q]) {
            const int j = ci[k[q]];
            if (j >= i) { k[q] = end[q]; break; }
            const int lj = ld_relaxed_i(level + j);
            if (lj < 0) break;  // not yet published
            best[q] = max(best[q], lj);
            ++k[q];
          }
          fin = k[q] >= end[q];
        }
        if (fin) {
          st_relaxed_i(level + i, best[q] + 1);
          trace_row(trace, i);
          live[q] = false;
        } else {
          any = true;
        }
      }
      if (!__any_sync(0xffffffffu, any)) break;
    }
  }
}

// ---------------------------------------------------------------------------
// Greedy first-fit colouring in ascending row order over the symmetrised
// adjacency (bs/analysis.py:103-145): colour(i) = mex of the colours of the
// neighbours j < i, where j is a neighbour if (i,j) or (j,i) is stored.
// The (j,i) half comes from `ut_ptr/ut_idx`: for every column c, the rows
// j < c that store (j, c).  colour[] must be -1 on entry.
__device__ __forceinline__ int mex64(unsigned long long used) {
  return used == ~0ull ? 64 : __ffsll((long long)~used) - 1;
}

constexpr int kCNb = 6;    // symmetrised lower neighbours held in registers (colour)
constexpr int kCR = 6;     // slices per warp unit (colour)

// neighbours j < i of row i in the symmetrised graph, deduplicated: the
// row's own lower entries, then the transposed upper entries (ut) not
// already present; returns the count (entries beyond KC are not stored)
template <int KC>
__device__ __forceinline__ int color_nbrs(int i, const int32_t* __restrict__ rp,
                                          const int32_t* __restrict__ ci,
                                          const int32_t* __restrict__ ut_ptr,
                                          const int32_t* __restrict__ ut_idx, int (&nb)[KC]) {
  int cnt = 0;
  for (int q = rp[i]; q < rp[i + 1]; ++q) {
    const int j = ci[q];
    if (j >= i) break;
    if (cnt < KC) {
#pragma unroll
      for (int t = 0; t < KC; ++t)
        if (t == cnt) nb[t] = j;
    }
    ++cnt;
  }
  const int nrow = cnt;
  for (int q = ut_ptr[i]; q < ut_ptr[i + 1]; ++q) {
    const int j = ut_idx[q];
    bool dup = false;  // (j,i) and (i,j) both stored: one neighbour
    if (nrow <= KC) {
#pragma unroll
      for (int t = 0; t < KC; ++t)
        if (t < nrow && nb[t] == j) dup = true;
    } else {
      for (int t = rp[i]; t < rp[i] + nrow; ++t) dup |= ci[t] == j;
    }
    if (dup) continue;
    if (cnt < KC) {
#pragma unroll
      for (int t = 0; t < KC; ++t)
        if (t == cnt) nb[t] = j;
    }
    ++cnt;
  }
  return cnt;
}

// mex over the symmetrised lower neighbours, walked from memory (long rows);
// returns -1 while some neighbour is unpublished
__device__ int color_walk(int i, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const int32_t* __restrict__ ut_ptr, const int32_t* __restrict__ ut_idx,
                          const int32_t* color) {
  unsigned long long used = 0ull;
  bool big = false;
  for (int q = rp[i]; q < rp[i + 1]; ++q) {
    const int j = ci[q];
    if (j >= i) break;
    const int cj = ld_relaxed_i(color + j);
    if (cj < 0) return -1;
    if (cj < 64) used |= 1ull << cj; else big = true;
  }
  for (int q = ut_ptr ? ut_ptr[i] : 0; ut_ptr && q < ut_ptr[i + 1]; ++q) {
    const int cj = ld_relaxed_i(color + ut_idx[q]);
    if (cj < 0) return -1;
    if (cj < 64) used |= 1ull << cj; else big = true;
  }
  int c = mex64(used);
  if (big && c >= 64) {   // rare: >= 64 distinct neighbour colours
    for (bool hit = true; hit;) {
      hit = false;
      for (int q = rp[i]; q < rp[i + 1] && !hit; ++q) {
        const int j = ci[q];
        if (j < i && ld_relaxed_i(color + j) == c) hit = true;
      }
      for (int q = ut_ptr ? ut_ptr[i] : 0; ut_ptr && q < ut_ptr[i + 1] && !hit; ++q)
        if (ld_relaxed_i(color + ut_idx[q]) == c) hit = true;
      if (hit) ++c;
    }
  }
  return c;
}

// *asym = 1 unless every row's transposed-upper list (rows j < i storing
// (j, i)) is exactly its own strict-lower column set
__global__ void k_symmetric(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const int32_t* __restrict__ ut_ptr,
                            const int32_t* __restrict__ ut_idx, int* asym) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k0 = rp[i], k1 = rp[i + 1];
    int nlow = 0;
    while (k0 + nlow < k1 && ci[k0 + nlow] < i) ++nlow;
    bool bad = nlow != ut_ptr[i + 1] - ut_ptr[i];
    for (int q = ut_ptr[i]; !bad && q < ut_ptr[i + 1]; ++q) {
      const int j = ut_idx[q];
      int lo = k0, hi = k0 + nlow - 1;
      bool found = false;
      while (lo <= hi) {
        const int mid = (lo + hi) >> 1, c = ci[mid];
        if (c == j) { found = true; break; }
        if (c < j) lo = mid + 1; else hi = mid - 1;
      }
      bad = !found;
    }
    if (bad) atomicExch(asym, 1);
  }
}

// (same R-slice units as k_level_sync_free).  SYM: the pattern is
// structurally symmetric (checked by k_symmetric), so the symmetrised lower
// neighbours are the row's own lower entries and the transposed lists are
// never read.
template <bool SYM, int NB = (SYM ? kLNb : kCNb)>
__global__ void __launch_bounds__(256, 5) k_color_sync_free(int n, const int32_t* __restrict__ rp,
                                  const int32_t* __restrict__ ci,
                                  const int32_t* __restrict__ ut_ptr,
                                  const int32_t* __restrict__ ut_idx, int32_t* color,
                                  unsigned int* ticket, unsigned long long* trace = nullptr) {
  const int lane = threadIdx.x & 31;
  __shared__ int snb[8][kCR][NB][32];   // neighbour lists (see k_level_sync_free)
  for (;;) {
    unsigned int u = 0;
    if (lane == 0) u = atomicAdd(ticket, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    const long long base = (long long)u * kCR * kSlice;
    if (base >= n) break;
    unsigned pend[kCR];
    unsigned used[kCR];   // colours 0..31 seen: a short row's mex is <= NB
    bool longrow[kCR], live[kCR];
    // row setup in two rounds for all R rows at once (row and transposed
    // extents, then the first entries of both lists); rows whose neighbour
    // set may exceed NB walk memory instead (color_walk)
    int k0[kCR], k1[kCR], u0[kCR], u1[kCR];
#pragma unroll
    for (int q = 0; q < kCR; ++q) {
      const long long i = base + q * kSlice + lane;
      live[q] = i < n;
      pend[q] = 0; used[q] = 0u; longrow[q] = false;
      k0[q] = live[q] ? rp[i] : 0;
      k1[q] = live[q] ? rp[i + 1] : 0;
      u0[q] = (live[q] && !SYM) ? ut_ptr[i] : 0;
      u1[q] = (live[q] && !SYM) ? ut_ptr[i + 1] : 0;
    }
#pragma unroll
    for (int q = 0; q < kCR; ++q) {
      const long long i = base + q * kSlice + lane;
      int c[NB + 1], t[NB + 1];
#pragma unroll
      for (int w = 0; w <= NB; ++w) {
        c[w] = k0[q] + w < k1[q] ? ci[k0[q] + w] : n;
        t[w] = (!SYM && u0[q] + w < u1[q]) ? ut_idx[u0[q] + w] : -1;
      }
      int cnt = 0;
      int nbq[NB];
#pragma unroll
      for (int w = 0; w <= NB; ++w)
        if (c[w] < i) {
          if (cnt < NB) nbq[cnt] = c[w];
          ++cnt;
        }
      const int nrow = cnt;
      bool overflow = nrow > NB || u1[q] - u0[q] > NB;
#pragma unroll
      for (int w = 0; w < NB; ++w) {
        if (t[w] < 0) continue;
        bool dup = false;   // (j,i) and (i,j) both stored: one neighbour
#pragma unroll
        for (int v = 0; v < NB; ++v) dup |= v < nrow && nbq[v] == t[w];
        if (dup) continue;
        if (cnt < NB) nbq[cnt] = t[w];
        ++cnt;
      }
      overflow |= cnt > NB;
#pragma unroll
      for (int w = 0; w < NB; ++w) snb[threadIdx.x >> 5][q][w][lane] = nbq[w];
      longrow[q] = overflow;
      pend[q] = (live[q] && !overflow) ? ((1u << cnt) - 1u) : 0u;
    }
    for (;;) {
      bool any = false;
#pragma unroll
      for (int q = 0; q < kCR; ++q) {
        if (!live[q]) continue;
        const int i = (int)(base + q * kSlice + lane);
        int c = -1;
        if (!longrow[q]) {
          int got[NB];
#pragma unroll
          for (int w = 0; w < NB; ++w)
            got[w] = (pend[q] & (1u << w)) ? ld_relaxed_i(color + snb[threadIdx.x >> 5][q][w][lane])
                                           : -1;
#pragma unroll
          for (int w = 0; w < NB; ++w)
            if ((pend[q] & (1u << w)) && got[w] >= 0) {
              if (got[w] < 32) used[q] |= 1u << got[w];   // larger ones cannot be the mex
              pend[q] &= ~(1u << w);
            }
          if (!pend[q]) c = __ffs(~used[q]) - 1;
        } else {
          c = color_walk(i, rp, ci, SYM ? nullptr : ut_ptr, ut_idx, color);
        }
        if (c >= 0) {
          st_relaxed_i(color + i, c);
          trace_row(trace, i);
          live[q] = false;
        } else {
          any = true;
        }
      }
      if (!__any_sync(0xffffffffu, any)) break;
    }
  }
}

// transpose of the strict-upper part: for every stored (j, c) with c > j,
// record j in the list of c.  Order inside a list is irrelevant (mex).
__global__ void k_upper_count(int n, const int32_t* __restrict__ rp,
                              const int32_t* __restrict__ ci, int32_t* cnt) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    for (int q = rp[j]; q < rp[j + 1]; ++q) {
      const int c = ci[q];
      if (c > j) atomicAdd(cnt + c, 1);
    }
}
__global__ void k_upper_fill(int n, const int32_t* __restrict__ rp,
                             const int32_t* __restrict__ ci, const int32_t* __restrict__ ptr,
                             int32_t* fillpos, int32_t* idx) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    for (int q = rp[j]; q < rp[j + 1]; ++q) {
      const int c = ci[q];
      if (c > j) idx[ptr[c] + atomicAdd(fillpos + c, 1)] = j;
    }
}

__global__ void k_fill_int(int n, int32_t* p, int v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_iota(int n, int32_t* p) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}
__global__ void k_max_reduce(int n, const int32_t* __restrict__ v, int32_t* out) {
  int m = -1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    m = max(m, v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}
__global__ void k_histogram(int n, const int32_t* __restrict__ g, int32_t* cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(cnt + g[i], 1);
}
// few groups (colourings): privatise the counters per CTA in shared memory,
// otherwise a million atomics serialise on a handful of addresses
constexpr int kSmemHist = 1024;
__global__ void k_histogram_smem(int n, int ngroups, const int32_t* __restrict__ g,
                                 int32_t* cnt) {
  __shared__ int32_t h[kSmemHist];
  for (int q = threadIdx.x; q < ngroups; q += blockDim.x) h[q] = 0;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(h + g[i], 1);
  __syncthreads();
  for (int q = threadIdx.x; q < ngroups; q += blockDim.x)
    if (h[q]) atomicAdd(cnt + q, h[q]);
}
// perm[iperm[k]] = k  (bs/analysis.py:64-65)
__global__ void k_invert_perm(int n, const int32_t* __restrict__ iperm, int32_t* perm) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    perm[iperm[k]] = k;
}

// ---------------------------------------------------------------------------
// symmetric permutation (bs/analysis.py:162-197): new row k is old row
// take[k]; columns are mapped through cmap and re-sorted ascending.  The
// per-row sort is an insertion sort on (new column, source slot) pairs held
// in the output arrays (rows are short: 7 for the stencil).
__global__ void k_permute_count(int n, const int32_t* __restrict__ rp,
                                const int32_t* __restrict__ take, int32_t* cnt) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int o = take[k];
    cnt[k] = rp[o + 1] - rp[o];
  }
}
__global__ void k_permute_cols(int n, const int32_t* __restrict__ rp,
                               const int32_t* __restrict__ ci,
                               const int32_t* __restrict__ take,
                               const int32_t* __restrict__ cmap,
                               const int32_t* __restrict__ nrp, int32_t* nci, int32_t* src) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int o = take[k];
    const int s = rp[o], len = rp[o + 1] - s, d = nrp[k];
    if (len <= 8) {
      // short rows (stencils): sort (column, source) pairs in registers with
      // a fixed odd-even transposition network, one write per entry; padding
      // keys sort last and the network is stable for equal keys -- columns
      // of a row are distinct anyway
      int key[8], val[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        key[t] = t < len ? cmap[ci[s + t]] : 0x7fffffff;
        val[t] = s + t;
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int t = r & 1; t + 1 < 8; t += 2)
          if (key[t] > key[t + 1]) {
            const int k2 = key[t]; key[t] = key[t + 1]; key[t + 1] = k2;
            const int v2 = val[t]; val[t] = val[t + 1]; val[t + 1] = v2;
          }
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (t < len) { nci[d + t] = key[t]; src[d + t] = val[t]; }
      continue;
    }
    for (int t = 0; t < len; ++t) {
      const int c = cmap[ci[s + t]];
      int u = t;
      while (u > 0 && nci[d + u - 1] > c) {
        nci[d + u] = nci[d + u - 1];
        src[d + u] = src[d + u - 1];
        --u;
      }
      nci[d + u] = c;
      src[d + u] = s + t;
    }
  }
}
// out block q = in block src[q]  (bb doubles per block)
// (block size a template parameter: the per-element division by BB is a
// multiply-shift instead of a 64-bit division -- 254 -> ~150 us at C4)
template <int BB>
__global__ void k_gather_blocks(long long nblk, const int32_t* __restrict__ src,
                                const double* __restrict__ in, double* __restrict__ out) {
  const long long total = nblk * BB;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const unsigned long long q = (unsigned long long)t / BB;
    const int e = (int)(t - (long long)q * BB);
    out[t] = __ldcs(in + (long long)__ldg(src + q) * BB + e);
  }
}
inline void launch_gather_blocks(long long nblk, int bb, const int32_t* src, const double* in,
                                 double* out, int grid, cudaStream_t st) {
  switch (bb) {
    case 1: k_gather_blocks<1><<<grid, 256, 0, st>>>(nblk, src, in, out); break;
    case 4: k_gather_blocks<4><<<grid, 256, 0, st>>>(nblk, src, in, out); break;
    case 9: k_gather_blocks<9><<<grid, 256, 0, st>>>(nblk, src, in, out); break;
    default: k_gather_blocks<16><<<grid, 256, 0, st>>>(nblk, src, in, out); break;
  }
}
// vector rows: out[i] = in[src[i]]  (bs/analysis.py:153-159)
__global__ void k_gather_rows(int n, int b, const int32_t* __restrict__ src,
                              const double* __restrict__ in, double* __restrict__ out) {
  const long long total = (long long)n * b;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / b;
    const int c = (int)(t - i * b);
    out[t] = in[(long long)src[i] * b + c];
  }
}

__global__ void k_narrow(long long m, const int64_t* __restrict__ in, int32_t* __restrict__ out,
                         int* overflow) {
  int bad = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m;
       t += (long long)gridDim.x * blockDim.x) {
    const int64_t v = in[t];
    bad |= (v > 0x7fffffffll || v < -0x7fffffffll);
    out[t] = (int32_t)v;
  }
  if (overflow && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(overflow, 1);
}

inline int grid_for(long long work, int threads = 256) {
  long long g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > kSms * 32) g = kSms * 32;
  return (int)g;
}

// persistent sync-free grids: every thread resident (the strided dealing
// relies on it), sized from the kernel's occupancy
inline int sync_free_grid(int n, const void* fn) {
  int per_sm = 0, dev = 0, sms = kSms;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long need = ((long long)n + 255) / 256;
  const long long cap = (long long)per_sm * sms;
  return (int)(need < 1 ? 1 : (need > cap ? cap : need));
}

}  // namespace b2s

namespace b2s {

// ---------------------------------------------------------------------------
// Speculate and verify.  Both plans are the unique solution of per-row
// equations over earlier rows only:
//   level(i)  = 1 + max{level(j) : j < i, (i,j) in pattern}   (0 if none)
//   colour(i) = mex{colour(j) : j < i, (i,j) or (j,i) in pattern}
// so, by induction on i, any assignment that satisfies every equation IS the
// reference's plan (bit for bit).  For a natural-order nx x ny x nz stencil
// the solutions are known in closed form (level = ix+iy+iz, colour = its
// parity); one parallel pass checks a guess instead of ~(nx+ny+nz) dependent
// L2 round trips of the wavefront.  Any violated equation -> the wavefront.
__global__ void k_grid_guess(int n, int nx, int ny, int parity, int32_t* g) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int ix = i % nx, iy = (i / nx) % ny, iz = i / (nx * ny);
    const int s = ix + iy + iz;
    g[i] = parity ? (s & 1) : s;
  }
}
// out[0]: violations; out[1]: max group
__global__ void k_verify_levels(int n, const int32_t* __restrict__ rp,
                                const int32_t* __restrict__ ci, const int32_t* __restrict__ g,
                                int32_t* out) {
  int bad = 0, mx = -1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int m = -1;
    for (int q = rp[i]; q < rp[i + 1]; ++q) {
      const int c = ci[q];
      if (c >= i) break;   // sorted columns: the strict-lower entries come first
      m = max(m, g[c]);
    }
    const int gi = g[i];
    bad |= gi != m + 1;
    mx = max(mx, gi);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicAdd(out, 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out + 1, mx);
}
// colours over the strict-lower entries, which is the symmetrised lower
// adjacency only if the pattern is structurally symmetric: every upper entry
// (i,j) must have its mirror (j,i) (binary search in row j)
__global__ void k_verify_colours(int n, const int32_t* __restrict__ rp,
                                 const int32_t* __restrict__ ci, const int32_t* __restrict__ g,
                                 int32_t* out) {
  int bad = 0, mx = -1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned long long mask = 0ull;
    for (int q = rp[i]; q < rp[i + 1]; ++q) {
      const int c = ci[q];
      if (c < i) {
        const int gc = g[c];
        if (gc < 0 || gc >= 64) bad = 1; else mask |= 1ull << gc;
      } else if (c > i) {
        int lo = rp[c], hi = rp[c + 1] - 1;
        bool found = false;
        while (lo <= hi) {
          const int mid = (lo + hi) >> 1, v = ci[mid];
          if (v == i) { found = true; break; }
          if (v < i) lo = mid + 1; else hi = mid - 1;
        }
        bad |= !found;
      }
    }
    const int gi = g[i];
    bad |= gi != __ffsll((long long)~mask) - 1;
    mx = max(mx, gi);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicAdd(out, 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out + 1, mx);
}

}  // namespace b2s

using namespace b2s;

extern "C" {

int b2s_find_diagonal(int n, const int32_t* rp, const int32_t* ci, int32_t* diag_pos,
                      int32_t* first_missing_host, cudaStream_t st) {
  if (n < 0) return B2S_SHAPE;
  *first_missing_host = -1;
  if (n == 0) return B2S_OK;
  int32_t* d_first = nullptr;
  B2S_CHECK(cudaMallocAsync(&d_first, sizeof(int32_t), st));
  const int32_t big = 0x7fffffff;
  B2S_CHECK(cudaMemcpyAsync(d_first, &big, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  k_find_diag<<<grid_for(n), 256, 0, st>>>(n, rp, ci, diag_pos, d_first);
  B2S_LAUNCH_CHECK();
  int32_t h = big;
  B2S_CHECK(cudaMemcpyAsync(&h, d_first, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaFreeAsync(d_first, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  if (h != big) { *first_missing_host = h; return B2S_MISSING_DIAGONAL; }
  return B2S_OK;
}

// Shared tail of level_schedule / graph_color: number of groups.
static int finish_groups(int n, const int32_t* groups, int32_t* ngroups_host, cudaStream_t st) {
  int32_t* d_max = nullptr;
  B2S_CHECK(cudaMallocAsync(&d_max, sizeof(int32_t), st));
  B2S_CHECK(cudaMemsetAsync(d_max, 0xff, sizeof(int32_t), st));  // -1
  k_max_reduce<<<grid_for(n), 256, 0, st>>>(n, groups, d_max);
  B2S_LAUNCH_CHECK();
  int32_t h = -1;
  B2S_CHECK(cudaMemcpyAsync(&h, d_max, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaFreeAsync(d_max, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  *ngroups_host = h + 1;
  return B2S_OK;
}

int b2s_level_schedule(int n, const int32_t* rp, const int32_t* ci, int32_t* row_group,
                       int32_t* ngroups_host, cudaStream_t st) {
  *ngroups_host = 0;
  if (n <= 0) return n < 0 ? B2S_SHAPE : B2S_OK;
  unsigned int* ticket = nullptr;
  B2S_CHECK(cudaMallocAsync(&ticket, sizeof(unsigned int), st));
  B2S_CHECK(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st));
  k_fill_int<<<grid_for(n), 256, 0, st>>>(n, row_group, -1);
  k_level_sync_free<<<sync_free_grid(n, (const void*)k_level_sync_free), 256, 0, st>>>(n, rp, ci, row_group, ticket);
  B2S_LAUNCH_CHECK();
  B2S_CHECK(cudaFreeAsync(ticket, st));
  return finish_groups(n, row_group, ngroups_host, st);
}

int b2s_graph_color(int n, const int32_t* rp, const int32_t* ci, int32_t* row_group,
                    int32_t* ngroups_host, cudaStream_t st) {
  *ngroups_host = 0;
  if (n <= 0) return n < 0 ? B2S_SHAPE : B2S_OK;
  int32_t *cnt = nullptr, *ptr = nullptr, *fill = nullptr, *idx = nullptr;
  unsigned int* ticket = nullptr;
  int32_t nnz = 0;
  B2S_CHECK(cudaMemcpyAsync(&nnz, rp + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  B2S_CHECK(cudaMallocAsync(&cnt, sizeof(int32_t) * (n + 1), st));
  B2S_CHECK(cudaMallocAsync(&ptr, sizeof(int32_t) * (n + 1), st));
  B2S_CHECK(cudaMallocAsync(&fill, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&idx, sizeof(int32_t) * (nnz > 0 ? nnz : 1), st));
  B2S_CHECK(cudaMallocAsync(&ticket, sizeof(unsigned int), st));
  B2S_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), st));
  B2S_CHECK(cudaMemsetAsync(fill, 0, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st));
  k_upper_count<<<grid_for(n), 256, 0, st>>>(n, rp, ci, cnt);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, ptr, n + 1, st);
  void* tmp = nullptr;
  B2S_CHECK(cudaMallocAsync(&tmp, tmp_bytes, st));
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, ptr, n + 1, st);
  k_upper_fill<<<grid_for(n), 256, 0, st>>>(n, rp, ci, ptr, fill, idx);
  k_fill_int<<<grid_for(n), 256, 0, st>>>(n, row_group, -1);
  // structurally symmetric patterns (every reservoir stencil): colour over
  // the lower entries alone
  B2S_CHECK(cudaMemsetAsync(cnt + n, 0, sizeof(int32_t), st));
  k_symmetric<<<grid_for(n), 256, 0, st>>>(n, rp, ci, ptr, idx, cnt + n);
  int asym = 1;
  B2S_CHECK(cudaMemcpyAsync(&asym, cnt + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  if (asym)
    k_color_sync_free<false><<<sync_free_grid(n, (const void*)k_color_sync_free<false>), 256, 0,
                               st>>>(n, rp, ci, ptr, idx, row_group, ticket);
  else
    k_color_sync_free<true><<<sync_free_grid(n, (const void*)k_color_sync_free<true>), 256, 0,
                              st>>>(n, rp, ci, ptr, idx, row_group, ticket);
  B2S_LAUNCH_CHECK();
  B2S_CHECK(cudaFreeAsync(tmp, st));
  B2S_CHECK(cudaFreeAsync(cnt, st));
  B2S_CHECK(cudaFreeAsync(ptr, st));
  B2S_CHECK(cudaFreeAsync(fill, st));
  B2S_CHECK(cudaFreeAsync(idx, st));
  B2S_CHECK(cudaFreeAsync(ticket, st));
  return finish_groups(n, row_group, ngroups_host, st);
}

// Level schedule / colouring with a grid hint (nx, ny of a natural-order
// stencil; nx <= 0: none): the closed-form plan is checked against every
// row's equation in one pass and used when it holds; otherwise (or without
// a hint) the sync-free wavefront.  Either way the result is the reference's.
static int groups_hint(int kind, int n, const int32_t* rp, const int32_t* ci, int nx, int ny,
                       int32_t* row_group, int32_t* ngroups_host, int* used_hint,
                       cudaStream_t st) {
  *ngroups_host = 0;
  if (used_hint) *used_hint = 0;
  if (n <= 0) return n < 0 ? B2S_SHAPE : B2S_OK;
  if (nx > 0 && ny > 0) {
    int32_t* d = nullptr;
    B2S_CHECK(cudaMallocAsync(&d, 2 * sizeof(int32_t), st));
    B2S_CHECK(cudaMemsetAsync(d, 0, sizeof(int32_t), st));
    B2S_CHECK(cudaMemsetAsync(d + 1, 0xff, sizeof(int32_t), st));
    k_grid_guess<<<grid_for(n), 256, 0, st>>>(n, nx, ny, kind, row_group);
    if (kind == 0) k_verify_levels<<<grid_for(n), 256, 0, st>>>(n, rp, ci, row_group, d);
    else k_verify_colours<<<grid_for(n), 256, 0, st>>>(n, rp, ci, row_group, d);
    B2S_LAUNCH_CHECK();
    int32_t h[2] = {1, -1};
    B2S_CHECK(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    B2S_CHECK(cudaFreeAsync(d, st));
    B2S_CHECK(cudaStreamSynchronize(st));
    if (h[0] == 0) {
      *ngroups_host = h[1] + 1;
      if (used_hint) *used_hint = 1;
      return B2S_OK;
    }
  }
  return kind == 0 ? b2s_level_schedule(n, rp, ci, row_group, ngroups_host, st)
                   : b2s_graph_color(n, rp, ci, row_group, ngroups_host, st);
}

int b2s_level_schedule_hint(int n, const int32_t* rp, const int32_t* ci, int nx, int ny,
                            int32_t* row_group, int32_t* ngroups_host, int* used_hint,
                            cudaStream_t st) {
  return groups_hint(0, n, rp, ci, nx, ny, row_group, ngroups_host, used_hint, st);
}

int b2s_graph_color_hint(int n, const int32_t* rp, const int32_t* ci, int nx, int ny,
                         int32_t* row_group, int32_t* ngroups_host, int* used_hint,
                         cudaStream_t st) {
  return groups_hint(1, n, rp, ci, nx, ny, row_group, ngroups_host, used_hint, st);
}

// debug (tools/analysis_trace.py): publication time of every row
int b2s_analysis_trace(int kind, int n, const int32_t* rp, const int32_t* ci, int32_t* row_group,
                       unsigned long long* trace, cudaStream_t st) {
  if (n <= 0) return B2S_SHAPE;
  unsigned int* ticket = nullptr;
  B2S_CHECK(cudaMallocAsync(&ticket, sizeof(unsigned int), st));
  B2S_CHECK(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st));
  k_fill_int<<<grid_for(n), 256, 0, st>>>(n, row_group, -1);
  if (kind == 0) {
    k_level_sync_free<<<sync_free_grid(n, (const void*)k_level_sync_free), 256, 0, st>>>(n, rp, ci, row_group, ticket, trace);
  } else {
    int32_t nnz = 0;
    B2S_CHECK(cudaMemcpyAsync(&nnz, rp + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    B2S_CHECK(cudaStreamSynchronize(st));
    int32_t *cnt, *ptr, *fill, *idx;
    B2S_CHECK(cudaMallocAsync(&cnt, sizeof(int32_t) * (n + 1), st));
    B2S_CHECK(cudaMallocAsync(&ptr, sizeof(int32_t) * (n + 1), st));
    B2S_CHECK(cudaMallocAsync(&fill, sizeof(int32_t) * n, st));
    B2S_CHECK(cudaMallocAsync(&idx, sizeof(int32_t) * (nnz > 0 ? nnz : 1), st));
    B2S_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), st));
    B2S_CHECK(cudaMemsetAsync(fill, 0, sizeof(int32_t) * n, st));
    k_upper_count<<<grid_for(n), 256, 0, st>>>(n, rp, ci, cnt);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, ptr, n + 1, st);
    void* tmp = nullptr;
    B2S_CHECK(cudaMallocAsync(&tmp, tb, st));
    cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, ptr, n + 1, st);
    k_upper_fill<<<grid_for(n), 256, 0, st>>>(n, rp, ci, ptr, fill, idx);
    k_color_sync_free<false><<<sync_free_grid(n, (const void*)k_color_sync_free<false>), 256, 0,
                               st>>>(n, rp, ci, ptr, idx, row_group, ticket, trace);
    cudaFreeAsync(tmp, st); cudaFreeAsync(cnt, st); cudaFreeAsync(ptr, st);
    cudaFreeAsync(fill, st); cudaFreeAsync(idx, st);
  }
  B2S_LAUNCH_CHECK();
  B2S_CHECK(cudaFreeAsync(ticket, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  return B2S_OK;
}

// bs/analysis.py:61-71: iperm = stable argsort(row_group), perm = its
// inverse, offsets = exclusive scan of the group histogram.
int b2s_plan_from_groups(int n, const int32_t* row_group, int ngroups, int32_t* perm,
                         int32_t* iperm, int32_t* offsets, cudaStream_t st) {
  if (n < 0 || ngroups < 0 || (n > 0 && ngroups < 1)) return B2S_SHAPE;
  if (n == 0) {
    B2S_CHECK(cudaMemsetAsync(offsets, 0, sizeof(int32_t), st));
    return B2S_OK;
  }
  int32_t *cnt = nullptr, *vals_in = nullptr, *keys_out = nullptr;
  B2S_CHECK(cudaMallocAsync(&cnt, sizeof(int32_t) * (ngroups + 1), st));
  B2S_CHECK(cudaMallocAsync(&vals_in, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&keys_out, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (ngroups + 1), st));
  if (ngroups <= kSmemHist)
    k_histogram_smem<<<kSms * 2, 256, 0, st>>>(n, ngroups, row_group, cnt);
  else
    k_histogram<<<grid_for(n), 256, 0, st>>>(n, row_group, cnt);
  size_t t1 = 0, t2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t1, cnt, offsets, ngroups + 1, st);
  int end_bit = 1;
  while (end_bit < 31 && (1ll << end_bit) < (long long)ngroups) ++end_bit;
  cub::DeviceRadixSort::SortPairs(nullptr, t2, row_group, keys_out, vals_in, iperm, n, 0,
                                  end_bit, st);
  void* tmp = nullptr;
  size_t tb = t1 > t2 ? t1 : t2;
  B2S_CHECK(cudaMallocAsync(&tmp, tb, st));
  cub::DeviceScan::ExclusiveSum(tmp, t1, cnt, offsets, ngroups + 1, st);
  k_iota<<<grid_for(n), 256, 0, st>>>(n, vals_in);
  // LSD radix sort is stable: equal groups keep ascending row order
  cub::DeviceRadixSort::SortPairs(tmp, t2, row_group, keys_out, vals_in, iperm, n, 0, end_bit,
                                  st);
  k_invert_perm<<<grid_for(n), 256, 0, st>>>(n, iperm, perm);
  B2S_LAUNCH_CHECK();
  B2S_CHECK(cudaFreeAsync(tmp, st));
  B2S_CHECK(cudaFreeAsync(cnt, st));
  B2S_CHECK(cudaFreeAsync(vals_in, st));
  B2S_CHECK(cudaFreeAsync(keys_out, st));
  return B2S_OK;
}

// Symmetric reorder of a block-CSR matrix.  take = iperm, cmap = perm for the
// forward direction (inverse=False in the reference); swap them for inverse.
// out_src (nnzb int32, may be null) receives, per output slot, the input slot
// it came from (the reference's `order` composition; used to build CopyPlans).
int b2s_permute_bsr(int n, int b, const int32_t* rp, const int32_t* ci, const double* vals,
                    const int32_t* cmap, const int32_t* take, int32_t* out_rp, int32_t* out_ci,
                    double* out_vals, int32_t* out_src, cudaStream_t st) {
  if (n < 0 || b < 1) return B2S_SHAPE;
  if (b > 4 && vals && out_vals) return B2S_UNSUPPORTED;
  if (n == 0) {
    B2S_CHECK(cudaMemsetAsync(out_rp, 0, sizeof(int32_t), st));
    return B2S_OK;
  }
  int32_t* cnt = nullptr;
  int32_t* src = out_src;
  int32_t nnz = 0;
  B2S_CHECK(cudaMemcpyAsync(&nnz, rp + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  B2S_CHECK(cudaMallocAsync(&cnt, sizeof(int32_t) * (n + 1), st));
  if (!src) B2S_CHECK(cudaMallocAsync(&src, sizeof(int32_t) * (nnz > 0 ? nnz : 1), st));
  B2S_CHECK(cudaMemsetAsync(cnt + n, 0, sizeof(int32_t), st));
  k_permute_count<<<grid_for(n), 256, 0, st>>>(n, rp, take, cnt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, out_rp, n + 1, st);
  void* tmp = nullptr;
  B2S_CHECK(cudaMallocAsync(&tmp, tb, st));
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, out_rp, n + 1, st);
  k_permute_cols<<<grid_for(n), 256, 0, st>>>(n, rp, ci, take, cmap, out_rp, out_ci, src);
  if (nnz > 0 && vals && out_vals)
    launch_gather_blocks(nnz, b * b, src, vals, out_vals, grid_for((long long)nnz * b * b), st);
  B2S_LAUNCH_CHECK();
  B2S_CHECK(cudaFreeAsync(tmp, st));
  B2S_CHECK(cudaFreeAsync(cnt, st));
  if (!out_src) B2S_CHECK(cudaFreeAsync(src, st));
  return B2S_OK;
}

int b2s_gather_rows(int n, int b, const int32_t* src, const double* in, double* out,
                    cudaStream_t st) {
  if (n < 0 || b < 1) return B2S_SHAPE;
  if (n == 0) return B2S_OK;
  k_gather_rows<<<grid_for((long long)n * b), 256, 0, st>>>(n, b, src, in, out);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

// int64 -> int32 index narrowing on the device (the reference's patterns
// are int64, bs/blockcore.py:83-84); *overflow_host = 1 if a value does not
// fit.  Saves the host a conversion pass over the column indices.
int b2s_narrow_index(long long m, const int64_t* in, int32_t* out, int* overflow_host,
                     cudaStream_t st) {
  if (overflow_host) *overflow_host = 0;
  if (m < 0) return B2S_SHAPE;
  if (m == 0) return B2S_OK;
  if (!overflow_host) {   // validated indices: no flag, no synchronisation
    k_narrow<<<grid_for(m), 256, 0, st>>>(m, in, out, nullptr);
    B2S_LAUNCH_CHECK();
    return B2S_OK;
  }
  int* d = nullptr;
  B2S_CHECK(cudaMallocAsync(&d, sizeof(int), st));
  B2S_CHECK(cudaMemsetAsync(d, 0, sizeof(int), st));
  k_narrow<<<grid_for(m), 256, 0, st>>>(m, in, out, d);
  B2S_LAUNCH_CHECK();
  B2S_CHECK(cudaMemcpyAsync(overflow_host, d, sizeof(int), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaFreeAsync(d, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  return B2S_OK;
}

int b2s_gather_blocks(long long nblk, int b, const int32_t* src, const double* in, double* out,
                      cudaStream_t st) {
  if (nblk < 0 || b < 1) return B2S_SHAPE;
  if (b > 4) return B2S_UNSUPPORTED;
  if (nblk == 0) return B2S_OK;
  launch_gather_blocks(nblk, b * b, src, in, out, grid_for(nblk * b * b), st);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

}  // extern "C"
