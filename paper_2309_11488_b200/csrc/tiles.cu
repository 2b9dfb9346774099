// Tiled level-scheduled ILU0 sweeps: the forward / backward block-triangular
// solves of bs/ilu0.py:105-142 (`_sweeps`, `_sweep`) for deep level schedules,
// with most dependencies resolved inside one SM.
//
// Why: in the sync-free sweeps (ilu0.cu) every level of the schedule costs a
// cross-SM L2 round trip (~1.15 us measured on B200), so a 1M-cell stencil
// with 298 levels per sweep is latency-bound at ~0.14 of the HBM roofline.
//
// Here the rows are partitioned into T <= #SM tiles (column patches of a
// natural-order grid when the pattern is one, else contiguous input ranges),
// one co-resident CTA per tile (cooperative launch).  Inside a tile the rows
// are cut into *steps*: the tile's rows of one plan group (level), in plan
// order.  A CTA walks its steps in order (backward: reverse order):
//
//   * warp 0 is the producer: per step it streams a packed, 16-byte aligned
//     record (plan rows, dependency codes, the L or U blocks, and for the
//     backward sweep the inverse diagonal blocks) into a ring of
//     shared-memory stages with one TMA bulk copy (cp.async.bulk, completion
//     on an mbarrier); the step's own inputs come along (forward: a gather of
//     r with cp.async; backward: the forward results, kept in padded step
//     order, in the same bulk copy).  It runs up to D-1 steps ahead and
//     waits on an "empty" mbarrier before reusing a stage.
//   * warps 1..4 are consumers: one row per thread, one named barrier per
//     step.  A dependency inside the tile is read from a shared-memory
//     window of the tile's last kWin results (tens of cycles); only couplings
//     that cross a tile boundary (or fall out of the window) are polled from
//     global memory with the sentinel protocol of ilu0.cu.
//
// The critical path is (levels x step time) + (tile crossings x L2 round
// trip) instead of levels x L2 round trip.
//
// Measured on B200 (C4, 12x12 column patches, tools/tile_exp.py,
// profiles/r01/tile_steps_trace.json): a step costs ~0.6 us of in-SM work for
// an 80-row level (instruction latency across 10 warps) and ~1.4 us when its
// boundary rows wait for inputs the neighbour tile produces just in time; the
// sweep is 298 steps long, so 0.87 ms per application against 0.68 ms for the
// sync-free sweeps.  Opt-in (B2S_TILES=1) until the step gets cheaper.  Per-row arithmetic is exactly the
// sync-free kernels' (ascending-column accumulation, then subtract; backward
// times inv(U_ii)), so results are bit-identical -- the order in which rows
// are computed never changes a row's value.
//
// Dependency codes in a record: c >= 0 -> window slot of tile position c;
// -1 padding; v = -c-2: v even -> poll global row v/2 (the sweep's output
// vector in plan order); v odd -> same-group row v/2: read the pre-sweep
// vector (r forward, y backward), as the reference's vectorised group update
// does (bs/ilu0.py:125-142).
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "sell.cuh"

namespace b2s {

constexpr int kWin = 1024;        // tile results kept in shared memory (rows)
constexpr int kCons = 384;        // consumer threads per CTA (12 warps, 4 lanes per row)
constexpr int kMaxStages = 8;     // ring depth cap
constexpr int kHdr = 32;          // stage header bytes (step meta)
// window: kWin slots + one never-written slot, rounded up to 128 bytes
__host__ __device__ constexpr int kWinBytes(int b) { return ((kWin + 1) * b * 8 + 127) & ~127; }

struct StepSet {
  int T, nsteps;
  const int32_t* tstep;    // [T+1] first step of tile t
  const int32_t* sbeg;     // [nsteps+1] first (global, tile-major) position of step s
  const int32_t* toff;     // [T+1] first position of tile t
  const int32_t* trow;     // [n] plan row at position k
  const int32_t* spad;     // [nsteps+1] padded row offset of step s (multiples of 4)
  const int32_t* wid;      // [2*nsteps] entries per row: forward (lower), backward (upper)
  const long long* roff;   // [2*(nsteps+1)] record byte offsets: forward, then backward
  const char* rec_f;
  const char* rec_b;
};

// record of one step: int32 rows[np] | int32 codes[w][np] | f64 vals[w][bb][np]
//                     | (backward) f64 inv[bb][np]
__host__ __device__ inline long long rec_bytes(int np, int w, int bb, int dir) {
  return 4ll * np * (1 + w) + 8ll * np * bb * (w + dir);
}

// ---- PTX helpers: mbarriers, bulk copies, cp.async, named barriers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned tx) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(
                   smem_u32(b)),
               "r"(tx)
               : "memory");
}
__device__ __forceinline__ bool mbar_test(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// cp.async completions arrive on the mbarrier (pending count +1 now, -1 on completion)
__device__ __forceinline__ void cp_async_arrive(unsigned long long* b) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cons_sync() {  // the consumer warps only
  asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory");
}
__device__ __forceinline__ double ld_relaxed_d(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_d(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  return g;
}

struct StepMeta {
  int nr, np, w, p0;   // rows, padded rows, entries per row, first tile-local position
  int spad, step, pad0, pad1;
};

// DIR 0: forward  out = y = L^-1 in          (in = r, plan order; yt written)
// DIR 1: backward out = z = U^-1 y           (own inputs from yt; stale = y)
template <int B, int DIR>
__global__ void __launch_bounds__(32 + kCons, 1)
    k_tile_steps(StepSet ss, int D, int stage_bytes, const double* __restrict__ in,
                 const double* stale, double* out, double* yt, double* yreset, int reset,
                 const int* done, unsigned long long* trace, int dbg) {
  constexpr int BB = B * B;
  extern __shared__ __align__(128) char smem[];
  if (done && *done) return;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
  unsigned long long* empty = full + kMaxStages;
  double* win = reinterpret_cast<double*>(smem + 16 * kMaxStages);
  char* ring = smem + 16 * kMaxStages + kWinBytes(B);
  const int t = blockIdx.x;
  const int s_lo = ss.tstep[t], s_hi = ss.tstep[t + 1], nst = s_hi - s_lo;
  const int tbase = ss.toff[t];
  if (threadIdx.x == 0) {
    for (int q = 0; q < D; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, kCons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const char* recs = DIR == 0 ? ss.rec_f : ss.rec_b;
  const long long* roff = ss.roff + (DIR == 0 ? 0 : ss.nsteps + 1);
  const int* wid = ss.wid + (DIR == 0 ? 0 : ss.nsteps);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // Step metadata is loaded 32 steps at a time (lane l holds step j0+l) and
    // the forward's row ids of step j+1 are loaded while step j is issued, so
    // global-load latency stays off the producer's per-step chain.
    int mk0 = 0, mnr = 0, msp = 0, mnp = 0, mw = 0;
    long long mro = 0, mrb = 0;
    auto load_meta = [&](int j0) {
      const int j = j0 + lane;
      if (j < nst) {
        const int s = DIR == 0 ? s_lo + j : s_hi - 1 - j;
        mk0 = ss.sbeg[s]; mnr = ss.sbeg[s + 1] - mk0;
        msp = ss.spad[s]; mnp = ss.spad[s + 1] - msp;
        mw = wid[s];
        mro = roff[s]; mrb = roff[s + 1] - mro;
      }
    };
    int pq = 0;
    unsigned pph = 0;       // ring slot and the parity of its current use
    constexpr int RQ = 4;   // row ids prefetched per lane (steps of <= 128 rows)
    int nrow[RQ] = {};
    load_meta(0);
    if (DIR == 0 && nst > 0) {
      const int k0 = __shfl_sync(0xffffffffu, mk0, 0), nr = __shfl_sync(0xffffffffu, mnr, 0);
#pragma unroll
      for (int u = 0; u < RQ; ++u) nrow[u] = lane + 32 * u < nr ? ss.trow[k0 + lane + 32 * u] : 0;
    }
    for (int j = 0; j < nst; ++j) {
      const int src = j & 31;
      const int k0 = __shfl_sync(0xffffffffu, mk0, src), nr = __shfl_sync(0xffffffffu, mnr, src);
      const int sp = __shfl_sync(0xffffffffu, msp, src), np = __shfl_sync(0xffffffffu, mnp, src);
      const int w = __shfl_sync(0xffffffffu, mw, src);
      const long long ro = __shfl_sync(0xffffffffu, mro, src);
      const long long rb = __shfl_sync(0xffffffffu, mrb, src);
      int crow[RQ];
#pragma unroll
      for (int u = 0; u < RQ; ++u) crow[u] = nrow[u];
      if (src == 31) load_meta(j + 1);
      if (DIR == 0 && j + 1 < nst) {   // row ids of the next step, in flight
        const int s1 = (j + 1) & 31;
        const int k1 = __shfl_sync(0xffffffffu, mk0, s1), n1 = __shfl_sync(0xffffffffu, mnr, s1);
#pragma unroll
        for (int u = 0; u < RQ; ++u) nrow[u] = lane + 32 * u < n1 ? ss.trow[k1 + lane + 32 * u] : 0;
      }
      const int q = pq;
      if (j >= D) mbar_wait(empty + q, pph ^ 1u);
      if (++pq == D) { pq = 0; pph ^= 1u; }
      char* stg = ring + q * stage_bytes;
      double* own = reinterpret_cast<double*>(stg + kHdr + rb);
      if (DIR == 0) {
        // gather the step's inputs r[row] (plan order) with 8-byte cp.async
#pragma unroll
        for (int u = 0; u < RQ; ++u) {
          const int j2 = lane + 32 * u;
          if (j2 < nr) {
#pragma unroll
            for (int c = 0; c < B; ++c) cp8(own + j2 * B + c, in + (long long)crow[u] * B + c);
          }
        }
        for (int j2 = lane + 32 * RQ; j2 < nr; j2 += 32) {   // rare: very wide steps
          const long long row = ss.trow[k0 + j2];
#pragma unroll
          for (int c = 0; c < B; ++c) cp8(own + j2 * B + c, in + row * B + c);
        }
        cp_async_arrive(full + q);
      }
      __syncwarp();
      if (lane == 0) {
        if (trace && j < 1024) trace[(((long long)DIR * gridDim.x + t) * 1024 + j) * 4] = gtime();
        StepMeta* m = reinterpret_cast<StepMeta*>(stg);
        m->nr = nr; m->np = np; m->w = w; m->p0 = k0 - tbase; m->spad = sp;
        m->step = DIR == 0 ? s_lo + j : s_hi - 1 - j;
        const unsigned ob = DIR == 1 ? (unsigned)(np * B * 8) : 0u;
        mbar_arrive_tx(full + q, (unsigned)rb + ob);
        bulk_g2s(stg + kHdr, recs + ro, (unsigned)rb, full + q);
        if (DIR == 1) bulk_g2s(own, yt + (long long)sp * B, ob, full + q);
      }
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  // Four lanes per row, lane c computes component c of the row's result: the
  // c-th row of every block product (the same fma sequence as matvec<B>, so
  // the arithmetic is unchanged) -- a dependency chain of B fmas per entry
  // instead of B*B, spread over 3x the warps.  The backward sweep's
  // inv(U_ii) product gathers the row's B components with shuffles.
  const int c0 = threadIdx.x - 32;
  const int cc = c0 & 3;               // component of this lane
  const int rr = c0 >> 2;              // row slot inside a pass
  const int cw = c0 >> 5;              // consumer warp
  constexpr int kRowsPerPass = kCons / 4;
  const int cb = cc < B ? cc : 0;      // clamped component for loads
  double pf[4][B];                     // prefetched cross-tile inputs (first pass)
  unsigned pfm = 0;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int c = 0; c < B; ++c) pf[kk][c] = 0.0;
  int q = 0;
  unsigned ph = 0;
  for (int j = 0; j < nst; ++j) {
    mbar_wait(full + q, ph);
    unsigned long long* tr =
        (trace && c0 == 0 && j < 1024) ? trace + (((long long)DIR * gridDim.x + t) * 1024 + j) * 4 : nullptr;
    if (tr) tr[1] = gtime();
    cons_sync();   // the previous step's window writes are visible
    if (tr) tr[2] = gtime();
    const char* stg = ring + q * stage_bytes;
    const StepMeta m = *reinterpret_cast<const StepMeta*>(stg);
    const int np = m.np, w = m.w, nr = m.nr;
    const int* rows = reinterpret_cast<const int*>(stg + kHdr);
    const int* codes = rows + np;
    const double* vals = reinterpret_cast<const double*>(codes + w * np);
    const double* inv = vals + w * BB * np;   // backward only
    const double* own = reinterpret_cast<const double*>(stg + kHdr + rec_bytes(np, w, BB, DIR));
    for (int base = 0; !(dbg & 2) && base < nr; base += kRowsPerPass) {
      if (base + cw * 8 >= nr) break;   // the whole warp is past the step's rows
      const int r0 = base + rr;
      const bool ok = r0 < nr;
      const int r = ok ? r0 : 0;
      double acc = 0.0;
      for (int k0 = 0; k0 < w; k0 += 4) {
        int cd[4];
        double dep[4][B];
        bool slow = false;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) cd[kk] = (ok && k0 + kk < w) ? codes[(k0 + kk) * np + r] : -1;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          // padding / remote / same-group codes read slot kWin, which nobody
          // writes (the value is replaced or masked below)
          const double* p = win + (cd[kk] >= 0 ? (cd[kk] & (kWin - 1)) : kWin) * B;
#pragma unroll
          for (int c = 0; c < B; ++c) dep[kk][c] = p[c];
          slow |= cd[kk] <= -2;
        }
        if (slow) {   // same-group (stale) or cross-tile entries
          unsigned pend = 0;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (cd[kk] > -2) continue;
            const int v = -cd[kk] - 2;
            if (v & 1) {
              const double* p = stale + (long long)(v >> 1) * B;
#pragma unroll
              for (int c = 0; c < B; ++c) dep[kk][c] = p[c];
            } else if (dbg & 1) {
#pragma unroll
              for (int c = 0; c < B; ++c) dep[kk][c] = 0.0;
            } else {
              bool have = k0 == 0 && base == 0 && ((pfm >> kk) & 1);
#pragma unroll
              for (int c = 0; c < B; ++c) {
                dep[kk][c] = pf[kk][c];
                have = have && !is_sentinel(pf[kk][c]);
              }
              if (!have) pend |= 1u << kk;
            }
          }
          while (pend) {   // every pending load in flight, then test
            const unsigned todo = pend;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              if (todo & (1u << kk)) {
                const double* p = out + (long long)((-cd[kk] - 2) >> 1) * B;
#pragma unroll
                for (int c = 0; c < B; ++c) dep[kk][c] = ld_relaxed_d(p + c);
              }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              bool miss = false;
#pragma unroll
              for (int c = 0; c < B; ++c) miss |= is_sentinel(dep[kk][c]);
              if ((todo & (1u << kk)) && !miss) pend &= ~(1u << kk);
            }
          }
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {   // ascending column order, like the reference
          // (a padding entry past the row's width reads entry 0 of this
          // record -- never memory of another stage -- and is masked below)
          const int ke = k0 + kk < w ? k0 + kk : 0;
          const double* vp = vals + (ke * BB + cb * B) * np + r;
          double sum = 0.0;
#pragma unroll
          for (int e = 0; e < B; ++e) sum = fma(vp[e * np], dep[kk][e], sum);
          acc = cd[kk] != -1 ? acc + sum : acc;
        }
      }
      double res;
      if (DIR == 0) {
        res = canon(own[r * B + cb] - acc);
      } else {
        const double tv = own[r * B + cb] - acc;
        const int l0 = (threadIdx.x & 31) & ~3;
        double tvs[B];
#pragma unroll
        for (int e = 0; e < B; ++e) tvs[e] = __shfl_sync(0xffffffffu, tv, l0 + e);
        const double* ip = inv + (cb * B) * np + r;
        double sum = 0.0;
#pragma unroll
        for (int e = 0; e < B; ++e) sum = fma(ip[e * np], tvs[e], sum);
        res = canon(sum);
      }
      if (ok && cc < B) {
        const long long row = rows[r];
        win[((m.p0 + r) & (kWin - 1)) * B + cc] = res;
        st_relaxed_d(out + row * B + cc, res);
        if (DIR == 0) yt[((long long)m.spad + r) * B + cc] = res;
        else if (reset) yreset[row * B + cc] = sentinel();
      }
    }
    if (tr) tr[3] = gtime();
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + q);
    if (++q == D) { q = 0; ph ^= 1u; }
    // Cross-tile inputs of the next step, loaded now (relaxed, no wait) when
    // its record has already landed: the neighbour tiles usually produced
    // them already, and the next step then finds them in registers instead
    // of paying an L2 round trip on its critical path.
    pfm = 0;
    if (!(dbg & 4) && j + 1 < nst && mbar_test(full + q, ph)) {
      const char* s1 = ring + q * stage_bytes;
      const StepMeta m1 = *reinterpret_cast<const StepMeta*>(s1);
      if (rr < m1.nr) {
        const int* cds1 = reinterpret_cast<const int*>(s1 + kHdr) + m1.np;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int cd = kk < m1.w ? cds1[kk * m1.np + rr] : -1;
          if (cd <= -2 && !((-cd - 2) & 1)) {
            const double* p = out + (long long)((-cd - 2) >> 1) * B;
#pragma unroll
            for (int c = 0; c < B; ++c) pf[kk][c] = ld_relaxed_d(p + c);
            pfm |= 1u << kk;
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- building
// tile of each plan-order row from its input index: px x py column patches
// of an nx x ny x nz natural-order grid (px > 0) or T contiguous ranges
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
// tile-local position of every row; step-start flags (new tile or new group)
__global__ void k_step_flags(int n, const int32_t* __restrict__ trow,
                             const int32_t* __restrict__ tid, const int32_t* __restrict__ toff,
                             const int32_t* __restrict__ goff, int ng, int32_t* loc,
                             int32_t* sflag) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int row = trow[k];
    const int t = tid[row];
    loc[row] = k - toff[t];
    bool start = (k == toff[t]);
    if (!start) start = group_of_row(goff, ng, trow[k - 1]) != group_of_row(goff, ng, row);
    sflag[k] = start ? 1 : 0;
  }
}
__global__ void k_step_starts(int n, int nsteps, const int32_t* __restrict__ sflag,
                              const int32_t* __restrict__ sidx, int32_t* sbeg) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    if (sflag[k]) sbeg[sidx[k]] = k;
  if (blockIdx.x == 0 && threadIdx.x == 0) sbeg[nsteps] = n;
}
__global__ void k_tile_steps_of(int T, const int32_t* __restrict__ toff,
                                const int32_t* __restrict__ sidx, int32_t* tstep) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q <= T; q += gridDim.x * blockDim.x)
    tstep[q] = sidx[toff[q]];
}
// per step: padded rows, entries per row (forward / backward), record sizes,
// and the largest stage it needs (max over both sweeps)
__global__ void k_step_sizes(int nsteps, int b, const int32_t* __restrict__ sbeg,
                             const int32_t* __restrict__ trow, const int32_t* __restrict__ rp,
                             const int32_t* __restrict__ diag, int32_t* npad, int32_t* wid,
                             long long* rsz, int32_t* stage_max) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int bb = b * b;
  for (int s = gw; s < nsteps; s += nw) {
    const int k0 = sbeg[s], nr = sbeg[s + 1] - k0;
    int wl = 0, wu = 0;
    for (int j = lane; j < nr; j += 32) {
      const int row = trow[k0 + j];
      wl = max(wl, diag[row] - rp[row]);
      wu = max(wu, rp[row + 1] - diag[row] - 1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      wl = max(wl, __shfl_xor_sync(0xffffffffu, wl, o));
      wu = max(wu, __shfl_xor_sync(0xffffffffu, wu, o));
    }
    if (lane == 0) {
      const int np = (nr + 3) & ~3;
      npad[s] = np;
      wid[s] = wl;
      wid[nsteps + s] = wu;
      const long long f = rec_bytes(np, wl, bb, 0), g = rec_bytes(np, wu, bb, 1);
      rsz[s] = f;
      rsz[nsteps + 1 + s] = g;
      const long long own = 8ll * np * b;
      const long long st = kHdr + std::max(f, g) + own;
      atomicMax(stage_max, (int)std::min(st, (long long)0x7fffffff));
    }
  }
}
// fill the records (warp per step, lane per row)
template <int DIR>
__global__ void k_step_fill(int nsteps, int bb, const int32_t* __restrict__ sbeg,
                            const int32_t* __restrict__ spad, const int32_t* __restrict__ wid,
                            const long long* __restrict__ roff, const int32_t* __restrict__ trow,
                            const int32_t* __restrict__ tid, const int32_t* __restrict__ loc,
                            const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const int32_t* __restrict__ diag, const double* __restrict__ vals,
                            const double* __restrict__ inv, const int32_t* __restrict__ goff,
                            int ng, char* rec) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nsteps; s += nw) {
    const int k0 = sbeg[s], nr = sbeg[s + 1] - k0;
    const int np = spad[s + 1] - spad[s];
    const int w = wid[DIR * nsteps + s];
    int* rows = reinterpret_cast<int*>(rec + roff[DIR * (nsteps + 1) + s]);
    int* codes = rows + np;
    double* v = reinterpret_cast<double*>(codes + (long long)w * np);
    double* dv = v + (long long)w * bb * np;
    const int t = tid[trow[k0]];
    const int p0 = loc[trow[k0]];   // first tile-local position of the step
    for (int r = lane; r < np; r += 32) {
      const bool ok = r < nr;
      const int row = ok ? trow[k0 + r] : -1;
      rows[r] = ok ? row : 0;
      const int grow = ok ? group_of_row(goff, ng, row) : -1;
      const int q0 = ok ? (DIR == 0 ? rp[row] : diag[row] + 1) : 0;
      const int q1 = ok ? (DIR == 0 ? diag[row] : rp[row + 1]) : 0;
      for (int k = 0; k < w; ++k) {
        const int q = q0 + k;
        int code = -1;
        if (q < q1) {
          const int c = ci[q];
          if (group_of_row(goff, ng, c) == grow) {
            code = -(3 + 2 * c);                       // same group: pre-sweep value
          } else if (tid[c] == t) {
            const int lc = loc[c];
            // in the window iff no position written before its use maps to
            // the same slot (forward: ascending, backward: descending)
            const bool inwin = DIR == 0 ? (p0 + nr - lc <= kWin) : (lc < p0 + kWin);
            code = inwin ? lc : -(2 + 2 * c);
          } else {
            code = -(2 + 2 * c);                       // another tile: poll
          }
        }
        codes[(long long)k * np + r] = code;
        for (int e = 0; e < bb; ++e)
          v[((long long)k * bb + e) * np + r] = q < q1 ? vals[(long long)q * bb + e] : 0.0;
      }
      if (DIR == 1)
        for (int e = 0; e < bb; ++e) dv[(long long)e * np + r] = ok ? inv[(long long)row * bb + e] : 0.0;
    }
  }
}

inline int grid_n(long long work) {
  long long g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > kSms * 16) g = kSms * 16;
  return (int)g;
}

struct TileHandle {
  StepSet ss;
  int b, n, D, stage_bytes;
  size_t smem;
  unsigned long long* trace;   // optional [2][T][1024][4] step event times (debug)
  int dbg;                     // debug switches (tools/tile_exp.py), 0 normally
  int32_t *trow, *toff, *tstep, *sbeg, *spad, *wid;
  long long* roff;
  char *rec_f, *rec_b;
  double* yt;                  // forward results in padded step order
};

template <int B>
int launch_tiled_b(const TileHandle* h, const double* r, double* y, double* z, int reset_y,
                   const int* done, cudaStream_t st) {
  auto* f = k_tile_steps<B, 0>;
  auto* g = k_tile_steps<B, 1>;
  if (cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)h->smem) != cudaSuccess ||
      cudaFuncSetAttribute((const void*)g, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)h->smem) != cudaSuccess)
    return B2S_CUDA_ERROR;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeCooperative;   // tiles wait on each other: all resident
  attr.val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(h->ss.T);
  cfg.blockDim = dim3(32 + kCons);
  cfg.dynamicSmemBytes = h->smem;
  cfg.stream = st;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, f, h->ss, h->D, h->stage_bytes, r, r, y, h->yt, (double*)nullptr,
                         0, done, h->trace, h->dbg) != cudaSuccess)
    return B2S_CUDA_ERROR;
  if (cudaLaunchKernelEx(&cfg, g, h->ss, h->D, h->stage_bytes, (const double*)nullptr,
                         (const double*)y, z, h->yt, y, reset_y, done, h->trace, h->dbg) != cudaSuccess)
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

static void free_handle(TileHandle* h) {
  if (!h) return;
  cudaFree(h->trow); cudaFree(h->toff); cudaFree(h->tstep); cudaFree(h->sbeg);
  cudaFree(h->spad); cudaFree(h->wid); cudaFree(h->roff);
  cudaFree(h->rec_f); cudaFree(h->rec_b); cudaFree(h->yt);
  delete h;
}

}  // namespace b2s

using namespace b2s;

extern "C" {

// debug: per-step event times of the step kernels into buf[2][T][1024][4]
// (producer issue, data ready, barrier passed, rows done); dbg bit 0: skip
// cross-tile polls, bit 1: no row work (timing experiments only), bit 2: no
// cross-tile prefetch
int b2s_tiles_trace(void* handle, unsigned long long* buf, int dbg) {
  TileHandle* h = reinterpret_cast<TileHandle*>(handle);
  if (!h) return B2S_SHAPE;
  h->trace = buf;
  h->dbg = dbg;
  return B2S_OK;
}

// Build the tiled sweep data of a factorisation in plan order (rp/ci/diag/lu:
// the combined L\U block CSR, inv: inverse diagonal blocks).  Tiles: px*py
// column patches of an nx x ny natural-order grid when px > 0, else T
// contiguous ranges of the input order.  Returns an opaque handle owning its
// device memory (b2s_tiles_destroy frees it), or B2S_UNSUPPORTED when T
// exceeds the SMs or fewer than two ring stages fit in shared memory.
int b2s_tiles_create(int n, int b, int T, int nx, int ny, int px, int py, const int32_t* iperm,
                     const int32_t* rp, const int32_t* ci, const int32_t* diag, const double* lu,
                     const double* inv, const int32_t* goff, int ngroups, void** handle_out,
                     cudaStream_t st) {
  *handle_out = nullptr;
  if (n <= 0 || b < 1 || b > 4 || ngroups < 1) return B2S_SHAPE;
  if (px > 0) T = px * py;
  if (T < 1) return B2S_SHAPE;
  const int bb = b * b;
  int dev = 0, sms = kSms, smem_max = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (T > sms) return B2S_UNSUPPORTED;
  TileHandle* h = new TileHandle();
  h->b = b;
  h->n = n;
  int32_t *tid, *tid_sorted, *iota, *cnt, *loc, *sflag, *sidx;
  B2S_CHECK(cudaMallocAsync(&tid, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&tid_sorted, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&iota, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&cnt, sizeof(int32_t) * (T + 1), st));
  B2S_CHECK(cudaMallocAsync(&loc, sizeof(int32_t) * n, st));
  B2S_CHECK(cudaMallocAsync(&sflag, sizeof(int32_t) * (n + 1), st));
  B2S_CHECK(cudaMallocAsync(&sidx, sizeof(int32_t) * (n + 1), st));
  B2S_CHECK(cudaMalloc(&h->trow, sizeof(int32_t) * n));
  B2S_CHECK(cudaMalloc(&h->toff, sizeof(int32_t) * (T + 1)));
  B2S_CHECK(cudaMalloc(&h->tstep, sizeof(int32_t) * (T + 1)));
  B2S_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (T + 1), st));
  k_tile_ids<<<grid_n(n), 256, 0, st>>>(n, T, nx, ny, px, py, iperm, tid);
  k_tile_hist<<<grid_n(n), 256, 0, st>>>(n, tid, cnt);
  k_iota32<<<grid_n(n), 256, 0, st>>>(n, iota);
  size_t t1 = 0, t2 = 0, t3 = 0;
  int end_bit = 1;
  while ((1 << end_bit) < T) ++end_bit;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, tid, tid_sorted, iota, h->trow, n, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, cnt, h->toff, T + 1, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t3, sflag, sidx, n + 1, st);
  void* tmp = nullptr;
  B2S_CHECK(cudaMallocAsync(&tmp, std::max(t1, std::max(t2, t3)) + 1024, st));
  // stable: inside a tile, rows stay in plan (group, input-index) order
  cub::DeviceRadixSort::SortPairs(tmp, t1, tid, tid_sorted, iota, h->trow, n, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(tmp, t2, cnt, h->toff, T + 1, st);
  B2S_CHECK(cudaMemsetAsync(sflag + n, 0, sizeof(int32_t), st));
  k_step_flags<<<grid_n(n), 256, 0, st>>>(n, h->trow, tid, h->toff, goff, ngroups, loc, sflag);
  cub::DeviceScan::ExclusiveSum(tmp, t3, sflag, sidx, n + 1, st);
  k_tile_steps_of<<<1, 256, 0, st>>>(T, h->toff, sidx, h->tstep);
  B2S_LAUNCH_CHECK();
  int32_t nsteps = 0;
  B2S_CHECK(cudaMemcpyAsync(&nsteps, sidx + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  int status = B2S_OK;
  B2S_CHECK(cudaMalloc(&h->sbeg, sizeof(int32_t) * (nsteps + 1)));
  B2S_CHECK(cudaMalloc(&h->spad, sizeof(int32_t) * (nsteps + 1)));
  B2S_CHECK(cudaMalloc(&h->wid, sizeof(int32_t) * 2 * nsteps + 4));
  B2S_CHECK(cudaMalloc(&h->roff, sizeof(long long) * 2 * (nsteps + 1)));
  int32_t *npad, *stage_max;
  long long* rsz;
  B2S_CHECK(cudaMallocAsync(&npad, sizeof(int32_t) * (nsteps + 1), st));
  B2S_CHECK(cudaMallocAsync(&rsz, sizeof(long long) * 2 * (nsteps + 1), st));
  B2S_CHECK(cudaMallocAsync(&stage_max, sizeof(int32_t), st));
  B2S_CHECK(cudaMemsetAsync(stage_max, 0, sizeof(int32_t), st));
  B2S_CHECK(cudaMemsetAsync(npad + nsteps, 0, sizeof(int32_t), st));
  B2S_CHECK(cudaMemsetAsync(rsz + nsteps, 0, sizeof(long long), st));
  B2S_CHECK(cudaMemsetAsync(rsz + 2 * nsteps + 1, 0, sizeof(long long), st));
  k_step_starts<<<grid_n(n), 256, 0, st>>>(n, nsteps, sflag, sidx, h->sbeg);
  k_step_sizes<<<grid_n((long long)nsteps * 32), 256, 0, st>>>(nsteps, b, h->sbeg, h->trow, rp,
                                                              diag, npad, h->wid, rsz, stage_max);
  size_t t4 = 0, t5 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t4, npad, h->spad, nsteps + 1, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t5, rsz, h->roff, nsteps + 1, st);
  void* tmp2 = nullptr;
  B2S_CHECK(cudaMallocAsync(&tmp2, std::max(t4, t5) + 1024, st));
  cub::DeviceScan::ExclusiveSum(tmp2, t4, npad, h->spad, nsteps + 1, st);
  cub::DeviceScan::ExclusiveSum(tmp2, t5, rsz, h->roff, nsteps + 1, st);
  cub::DeviceScan::ExclusiveSum(tmp2, t5, rsz + nsteps + 1, h->roff + nsteps + 1, nsteps + 1, st);
  B2S_LAUNCH_CHECK();
  long long bytes_f = 0, bytes_b = 0;
  int32_t rows_pad = 0, stage = 0;
  B2S_CHECK(cudaMemcpyAsync(&bytes_f, h->roff + nsteps, sizeof(long long), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaMemcpyAsync(&bytes_b, h->roff + 2 * nsteps + 1, sizeof(long long),
                            cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaMemcpyAsync(&rows_pad, h->spad + nsteps, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaMemcpyAsync(&stage, stage_max, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  stage = (stage + 127) & ~127;
  const long long fixed = 16ll * kMaxStages + kWinBytes(b);
  const long long avail = (long long)smem_max - fixed;
  const int D = stage > 0 ? (int)std::min<long long>(kMaxStages, avail / stage) : 0;
  if (D < 2) status = B2S_UNSUPPORTED;
  if (status == B2S_OK) {
    h->D = D;
    h->stage_bytes = stage;
    h->smem = (size_t)(fixed + (long long)D * stage);
    B2S_CHECK(cudaMalloc(&h->rec_f, bytes_f + 16));
    B2S_CHECK(cudaMalloc(&h->rec_b, bytes_b + 16));
    B2S_CHECK(cudaMalloc(&h->yt, sizeof(double) * ((long long)rows_pad * b + 4)));
    k_step_fill<0><<<grid_n((long long)nsteps * 32), 256, 0, st>>>(
        nsteps, bb, h->sbeg, h->spad, h->wid, h->roff, h->trow, tid, loc, rp, ci, diag, lu, inv,
        goff, ngroups, h->rec_f);
    k_step_fill<1><<<grid_n((long long)nsteps * 32), 256, 0, st>>>(
        nsteps, bb, h->sbeg, h->spad, h->wid, h->roff, h->trow, tid, loc, rp, ci, diag, lu, inv,
        goff, ngroups, h->rec_b);
    B2S_LAUNCH_CHECK();
    h->ss = StepSet{T, nsteps, h->tstep, h->sbeg, h->toff, h->trow, h->spad, h->wid, h->roff,
                    h->rec_f, h->rec_b};
  }
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(tmp2, st);
  cudaFreeAsync(tid, st);
  cudaFreeAsync(tid_sorted, st);
  cudaFreeAsync(iota, st);
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(loc, st);
  cudaFreeAsync(sflag, st);
  cudaFreeAsync(sidx, st);
  cudaFreeAsync(npad, st);
  cudaFreeAsync(rsz, st);
  cudaFreeAsync(stage_max, st);
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
