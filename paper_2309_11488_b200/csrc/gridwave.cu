// Wavefront ILU0 sweeps for natural-order 7-point grids (the level-scheduled
// apply, bs/ilu0.py:105-142 `_sweeps`, on the reference's default backend).
//
// Why: a level schedule of an nx x ny x nz stencil has nx+ny+nz-2 levels;
// the sync-free sweeps (ilu0.cu) pay one cross-SM L2 round trip per level
// (~1 us), the tile step kernels (tiles.cu) ~0.6 us of in-SM overhead per
// step.  Here the (x, y) plane is cut into tiles of at most 32 columns, ONE
// WARP per tile, one lane per column (all z).  The warp walks the levels
// l = x+y+z of its tile in order; at step l lane (x, y) owns row
// (x, y, z = l-x-y), and its three lower neighbours were produced at step
// l-1 by: itself (z-1, a register), lane-1 (x-1) and lane-wx (y-1) --
// warp shuffles, no shared memory, no barrier.  Only the tile's west and
// south edge lanes read a neighbour tile's value: from that tile's edge
// buffer, with the sentinel protocol of the sync-free sweeps (values are
// self-validating, no fences).  The critical path is levels x (in-warp step)
// + tile crossings x (one L2 hop), with the step a few dependent FMAs.
//
// Data: the factor is repacked once per factorisation into the warp's step
// order, [tile][step][entry][e][lane] (coalesced 256-byte warp loads), with
// a per-slot meta word (plan row | entry mask).  Per row the arithmetic is
// exactly the sync-free sweeps' -- strict-lower entries in ascending plan
// column order (z-1, y-1, x-1), acc then subtract, canon; backward (x+1,
// y+1, z+1), then inv(U_ii) -- so results are bit-identical.  A plan
// qualifies when every row's lower entries are its minus-neighbours and its
// upper entries its plus-neighbours (level schedules and the sequential plan
// of such grids); the packing kernel verifies this row by row.
#include <cstdlib>

#include "sell.cuh"

namespace b2s {

constexpr int kGwLanes = 32;

struct GwDev {
  int nx, ny, nz, wx, wy, TX, TY, S;   // grid, tile shape, tiles, steps per tile (max)
  int rf, rb;            // bytes of one forward / backward step record
  int shallow;           // 1: the shallow rings (more tiles co-resident), 0: the deep ones
  const char* recf;      // [T*S] forward records:  meta[32] int32 | L[3][BB][32] f64
  const char* recb;      // [T*S] backward records: meta[32] int32 | U[3][BB][32] | D[BB][32]
  double* rpk;           // [T*S][B][32]  the sweep's input in step order (k_gw_gather)
  double* ypk;           // [T*S][B][32]  forward results, step order
  double* eE;            // [T*S][wy][B]      forward: east-edge lanes' results
  double* eN;            // [T*S][wx][B]      forward: north-edge lanes' results
  double* eW;            // [T*S][wy][B]      backward: west-edge lanes' results
  double* eS;            // [T*S][wx][B]      backward: south-edge lanes' results
  unsigned long long* trace;   // debug (B2S_GW_TRACE): [2][T][S] step end times, or null
};

// meta word: -1 inactive, else plan row (bits 0..24) | entry mask << 25
enum GwMask { kZm = 1, kYm = 2, kXm = 4, kXp = 8, kYp = 16, kZp = 32 };
constexpr int kGwMetaBytes = 128;
constexpr int kGwTl = 64;     // launches kept per tile by the debug timeline
constexpr int kGwRingF = 8;   // forward ring stages (step records in flight)
constexpr int kGwRingB = 6;   // backward ring stages
// shallow rings for grids with more tiles than 3 per SM (the deep rings'
// shared memory allows 3 CTAs per SM, these 7)
constexpr int kGwRingFs = 4;
constexpr int kGwRingBs = 3;

__device__ __forceinline__ double gw_ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void gw_st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns_gw() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned gw_smem(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void gw_mbar_init(unsigned long long* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(gw_smem(b)) : "memory");
}
__device__ __forceinline__ void gw_mbar_expect(unsigned long long* b, unsigned tx) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(
                   gw_smem(b)), "r"(tx)
               : "memory");
}
__device__ __forceinline__ void gw_mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(gw_smem(b)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void gw_bulk(void* dst, const void* src, unsigned bytes,
                                        unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          gw_smem(dst)), "l"(src), "r"(bytes), "r"(gw_smem(b))
      : "memory");
}
// predicated stage refill (one lane issues, no branch around it): proxy
// fence, expect_tx, and the record + vector bulk copies into the stage
__device__ __forceinline__ void gw_refill(bool p, unsigned long long* bar, unsigned tx, void* d0,
                                          const void* s0, unsigned n0, void* d1, const void* s1,
                                          unsigned n1) {
  asm volatile(
      "{\n .reg .pred p;\n .reg .b64 st;\n setp.ne.b32 p, %0, 0;\n"
      " @p fence.proxy.async.shared::cta;\n"
      " @p mbarrier.arrive.expect_tx.shared::cta.b64 st, [%1], %2;\n"
      " @p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%3], [%4], %5, [%1];\n"
      " @p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%6], [%7], %8, [%1];\n"
      "}" ::"r"((int)p), "r"(gw_smem(bar)), "r"(tx), "r"(gw_smem(d0)), "l"(s0), "r"(n0),
      "r"(gw_smem(d1)), "l"(s1), "r"(n1)
      : "memory");
}
__device__ __forceinline__ void gw_fence_proxy() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int B>
__device__ __forceinline__ bool gw_ready(const double (&v)[B]) {
  bool ok = true;
#pragma unroll
  for (int c = 0; c < B; ++c) ok &= !is_sentinel(v[c]);
  return ok;
}
template <int B>
__device__ __forceinline__ void gw_load(const double* p, double (&v)[B]) {
#pragma unroll
  for (int c = 0; c < B; ++c) v[c] = gw_ld_relaxed(p + c);
}
template <int B>
__device__ __forceinline__ void gw_poll(const double* p, double (&v)[B]) {
  while (!gw_ready<B>(v)) gw_load<B>(p, v);
}

// element e of lane l in a step record's block area: pairs of elements
// interleaved per lane, [e/2][32 lanes][2]
__host__ __device__ __forceinline__ long long gw_eidx(int e, int lane) {
  return (long long)(e >> 1) * 64 + lane * 2 + (e & 1);
}

struct GwTile {
  int t, tx, ty, x0, y0, xw, yw, xl, yl, L0, St;
  bool valid;
};

__device__ __forceinline__ GwTile gw_tile(const GwDev& g, int t, int lane) {
  GwTile a;
  a.t = t;
  a.tx = t % g.TX;
  a.ty = t / g.TX;
  a.x0 = a.tx * g.wx;
  a.y0 = a.ty * g.wy;
  a.xw = min(g.wx, g.nx - a.x0);
  a.yw = min(g.wy, g.ny - a.y0);
  a.xl = lane % g.wx;
  a.yl = lane / g.wx;
  a.valid = lane < g.wx * g.wy && a.xl < a.xw && a.yl < a.yw;
  a.L0 = a.x0 + a.y0;
  a.St = (a.xw - 1) + (a.yw - 1) + g.nz;
  return a;
}

__device__ __forceinline__ void gw_mbar_init_n(unsigned long long* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(gw_smem(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void gw_mbar_arrive(unsigned long long* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(gw_smem(b))
               : "memory");
}

// One warp per tile.  The tile's step records and input slices stream into a
// shared-memory ring with TMA bulk copies (an mbarrier per stage counts the
// bytes; lane 0 refills a stage right after the warp consumed it).  Per step:
// a stage wait, shared-memory reads, two shuffles per component, three 3x3
// products and the stores; the neighbour tiles' edge values needed at the
// next step are requested one step early (the neighbour runs about one L2 hop
// ahead, so an earlier request would find them not yet produced; measured:
// 4 steps early 1457 us per C4 application, 1 step 792 us).  A separate
// producer warp measured slower (1636 us).
//
// forward: y = r - L y, levels upward; backward: z = inv(U_ii) (y - U z),
// levels downward.  DIR 0 / 1.
template <int B, int DIR, int SH>
__global__ void __launch_bounds__(32) k_gw_sweep(GwDev g, const int* done, double* zout) {
  constexpr int BB = B * B;
  constexpr int R = DIR == 0 ? (SH ? kGwRingFs : kGwRingF) : (SH ? kGwRingBs : kGwRingB);
  constexpr int VB = B * 32 * 8;   // bytes of one step's vector slice
  extern __shared__ __align__(128) char smem[];
#ifdef B2S_GW_TRACE_BUILD
  const unsigned long long t_in = global_ns_gw();
#endif
  // PDL: everything below reads the predecessors' results
  griddep_wait();
  griddep_launch();
#ifdef B2S_GW_TRACE_BUILD
  const unsigned long long t_w = global_ns_gw();
  // per-launch timeline of this tile: [T] counters, then [T][kGwTl][4]
  // (entry, after the grid-dependency wait, exit, direction)
  auto tl_rec = [&](unsigned long long t_out) {
    if (!g.trace || threadIdx.x != 0) return;
    unsigned long long* tl = g.trace + 2LL * g.TX * g.TY * g.S;
    const unsigned long long k = tl[blockIdx.x]++;
    unsigned long long* r = tl + g.TX * g.TY + ((long long)blockIdx.x * kGwTl + k % kGwTl) * 4;
    r[0] = t_in; r[1] = t_w; r[2] = t_out; r[3] = DIR;
  };
#endif
  if (done && *done) {
#ifdef B2S_GW_TRACE_BUILD
    tl_rec(0);
#endif
    return;
  }
  const int lane = threadIdx.x & 31;
  const GwTile a = gw_tile(g, blockIdx.x, lane);
  const long long base = (long long)a.t * g.S;
  const int rb = DIR == 0 ? g.rf : g.rb;
  const int stage = rb + VB;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
  char* ring = smem + 128;
  if (threadIdx.x == 0) {
    for (int q = 0; q < R; ++q) gw_mbar_init_n(full + q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // step j of this sweep (j = 0, 1, ...) is tile step s = j (forward) or St-1-j;
  // lane 0 keeps the ring R steps ahead (refilling a stage right after the
  // warp consumed it)
  const char* rec = DIR == 0 ? g.recf : g.recb;
  const char* vin = reinterpret_cast<const char*>(DIR == 0 ? g.rpk : g.ypk);
  auto issue = [&](int j) {
    const int q = j % R;
    const long long s = DIR == 0 ? j : a.St - 1 - j;
    char* dst = ring + q * stage;
    gw_mbar_expect(full + q, (unsigned)stage);
    gw_bulk(dst, rec + (base + s) * (long long)rb, (unsigned)rb, full + q);
    gw_bulk(dst + rb, vin + (base + s) * VB, (unsigned)VB, full + q);
  };
  if (lane == 0)
    for (int j = 0; j < R && j < a.St; ++j) issue(j);
  {  // the other direction's edge buffers of this tile go back to "not produced"
    double* o1 = DIR == 0 ? g.eW : g.eE;
    double* o2 = DIR == 0 ? g.eS : g.eN;
    for (long long q = lane; q < (long long)g.S * g.wy * B; q += 32) o1[base * g.wy * B + q] = sentinel();
    for (long long q = lane; q < (long long)g.S * g.wx * B; q += 32) o2[base * g.wx * B + q] = sentinel();
  }
  const bool hasW = a.tx > 0, hasS = a.ty > 0;
  const bool hasE = a.tx + 1 < g.TX, hasN = a.ty + 1 < g.TY;
  // this lane's neighbour-tile inputs (x side / y side) and its own edge outputs
  const bool xe = DIR == 0 ? (a.xl == 0 && hasW) : (a.xl == a.xw - 1 && hasE);
  const bool ye = DIR == 0 ? (a.yl == 0 && hasS) : (a.yl == a.yw - 1 && hasN);
  const bool px = DIR == 0 ? (a.xl == a.xw - 1 && hasE) : (a.xl == 0 && hasW);
  const bool py = DIR == 0 ? (a.yl == a.yw - 1 && hasN) : (a.yl == 0 && hasS);
  // per-step pointers (stride B doubles per step along the tile's steps)
  const int dstep = DIR == 0 ? 1 : -1;
  const int s0 = DIR == 0 ? 0 : a.St - 1;
  const double* xin = (DIR == 0 ? g.eE : g.eW) +
                      (((DIR == 0 ? base - g.S : base + g.S) + s0 + (DIR == 0 ? g.wx - 1 : 1 - g.wx)) *
                       g.wy + a.yl) * B;
  const double* yin = (DIR == 0 ? g.eN : g.eS) +
                      (((DIR == 0 ? base - (long long)g.TX * g.S : base + (long long)g.TX * g.S) + s0 +
                        (DIR == 0 ? g.wy - 1 : 1 - g.wy)) * g.wx + a.xl) * B;
  const long long xstride = (long long)dstep * g.wy * B, ystride = (long long)dstep * g.wx * B;
  double* xout = (DIR == 0 ? g.eE : g.eW) + ((base + s0) * g.wy + a.yl) * B;
  double* yout = (DIR == 0 ? g.eN : g.eS) + ((base + s0) * g.wx + a.xl) * B;
  // forward results in step order (the backward sweep's input); backward
  // results straight to their plan rows (no scatter pass)
  double* vout = g.ypk + (base + s0) * B * 32 + lane;
  const long long vstride = (long long)dstep * B * 32;
  // neighbour-tile step of the value needed at our step s: in range?
  const int xoff = DIR == 0 ? g.wx - 1 : 1 - g.wx, yoff = DIR == 0 ? g.wy - 1 : 1 - g.wy;
  auto xok = [&](int s) { const int t = s + xoff; return xe && t >= 0 && t < g.S; };
  auto yok = [&](int s) { const int t = s + yoff; return ye && t >= 0 && t < g.S; };
  double ex[B], ey[B];
#pragma unroll
  for (int c = 0; c < B; ++c) ex[c] = ey[c] = sentinel();
  if (a.St > 0) {
    if (xok(s0)) gw_load<B>(xin, ex);
    if (yok(s0)) gw_load<B>(yin, ey);
  }
  const int sx = DIR == 0 ? (lane > 0 ? lane - 1 : 0) : (lane + 1 < 32 ? lane + 1 : 31);
  const int sy = DIR == 0 ? (lane >= g.wx ? lane - g.wx : 0) : (lane + g.wx < 32 ? lane + g.wx : 31);
  constexpr int mx = DIR == 0 ? kXm : kXp, my = DIR == 0 ? kYm : kYp, mz = DIR == 0 ? kZm : kZp;
  double prev[B];
#pragma unroll
  for (int c = 0; c < B; ++c) prev[c] = 0.0;
  // the step's record is read from its ring stage at the top of the step
  // (independent loads, issued ahead of the dependent chain) and the stage
  // refilled as soon as every lane has it.  (Copying it into registers one
  // step ahead measured slower once the products were branch-free: 512 vs
  // 497 us at C4 -- the register rotation costs ~60 moves per step.)
  constexpr int NB = DIR == 0 ? 3 * BB : 4 * BB;   // blocks per record (+ inv(U_ii))
  int mt_c = -1;
  double bk_c[NB], vv_c[B];
  auto load_step = [&](int j, int& mt, double (&bk)[NB], double (&vv)[B]) {
    const int q = j % R;
    gw_mbar_wait(full + q, (unsigned)((j / R) & 1));
    const char* st_ = ring + q * stage;
    mt = reinterpret_cast<const int*>(st_)[lane];
    const double2* blk = reinterpret_cast<const double2*>(st_ + kGwMetaBytes) + lane;
    const double* v = reinterpret_cast<const double*>(st_ + rb) + lane;
#pragma unroll
    for (int e = 0; e < NB; e += 2) {
      const double2 q = blk[(e >> 1) * 32];
      bk[e] = q.x;
      if (e + 1 < NB) bk[e + 1] = q.y;
    }
#pragma unroll
    for (int c = 0; c < B; ++c) vv[c] = v[c * 32];
  };
  for (int j = 0; j < a.St; ++j) {
    const int s = s0 + dstep * j;
    load_step(j, mt_c, bk_c, vv_c);
    // step j's stage is in registers: refill it with step j + R
    __syncwarp();
    {
      const int jj = j + R, q = jj % R;
      const long long sr = DIR == 0 ? jj : a.St - 1 - jj;
      char* dst = ring + q * stage;
      gw_refill(lane == 0 && jj < a.St, full + q, (unsigned)stage, dst, rec + (base + sr) * (long long)rb,
                (unsigned)rb, dst + rb, vin + (base + sr) * VB, (unsigned)VB);
    }
    const int mt = mt_c;
    const int mask = mt >= 0 ? (mt >> 25) : 0;
    double nx_[B], ny_[B];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      nx_[c] = __shfl_sync(0xffffffffu, prev[c], sx);
      ny_[c] = __shfl_sync(0xffffffffu, prev[c], sy);
    }
    if (xe && (mask & mx)) {
      gw_poll<B>(xin, ex);
#pragma unroll
      for (int c = 0; c < B; ++c) nx_[c] = ex[c];
    }
    if (ye && (mask & my)) {
      gw_poll<B>(yin, ey);
#pragma unroll
      for (int c = 0; c < B; ++c) ny_[c] = ey[c];
    }
    // the next step's edge inputs, one step early
    xin += xstride;
    yin += ystride;
    if (j + 1 < a.St) {
      if (xok(s + dstep)) gw_load<B>(xin, ex);
      if (yok(s + dstep)) gw_load<B>(yin, ey);
    }
    // ascending plan columns: forward z-1, y-1, x-1; backward x+1, y+1, z+1.
    // Branch-free: an absent entry has a zero block (k_gw_vals) and its
    // input is selected to zero, so its product is +0.0 and adding it leaves
    // the sum unchanged (the sum starts at +0.0 and can never be -0.0) --
    // the three products are independent chains the scheduler interleaves.
    double pr[3][B];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int bit = DIR == 0 ? (k == 0 ? mz : (k == 1 ? my : mx)) : (k == 0 ? mx : (k == 1 ? my : mz));
      const double* dep = k == 0 ? (DIR == 0 ? prev : nx_) : (k == 1 ? ny_ : (DIR == 0 ? nx_ : prev));
      const bool on = (mask & bit) != 0;
      double d[B];
#pragma unroll
      for (int c = 0; c < B; ++c) d[c] = on ? dep[c] : 0.0;
      matvec<B>(bk_c + k * BB, d, pr[k]);
    }
    double acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) acc[c] = ((0.0 + pr[0][c]) + pr[1][c]) + pr[2][c];
    double outv[B];
    if (DIR == 0) {
#pragma unroll
      for (int c = 0; c < B; ++c) outv[c] = canon(vv_c[c] - acc[c]);
    } else {
      double tv[B], o[B];
#pragma unroll
      for (int c = 0; c < B; ++c) tv[c] = vv_c[c] - acc[c];
      matvec<B>(bk_c + (NB - BB), tv, o);
#pragma unroll
      for (int c = 0; c < B; ++c) outv[c] = canon(o[c]);
    }
    if (mt >= 0) {
      double* zr = zout + (long long)(mt & 0x1FFFFFF) * B;
#pragma unroll
      for (int c = 0; c < B; ++c) {
        prev[c] = outv[c];
        if (DIR == 0) vout[c * 32] = outv[c];
        else zr[c] = outv[c];
      }
      if (px) {
#pragma unroll
        for (int c = 0; c < B; ++c) gw_st_relaxed(xout + c, outv[c]);
      }
      if (py) {
#pragma unroll
        for (int c = 0; c < B; ++c) gw_st_relaxed(yout + c, outv[c]);
      }
    }
    vout += vstride;
    xout += xstride;
    yout += ystride;
#ifdef B2S_GW_TRACE_BUILD
    if (g.trace && lane == 0)
      g.trace[(long long)DIR * g.TX * g.TY * g.S + base + s] = global_ns_gw();
#endif
  }
#ifdef B2S_GW_TRACE_BUILD
  tl_rec(global_ns_gw());
#endif
}

// ---- wavefront ILU0 factorisation of the same grids (bs/ilu0.py:145-201).
// On a natural-order 7-point stencil the elimination of row i touches only
// its diagonal: L_ik = A_ik inv(U_kk) for its lower neighbours k (ascending
// plan columns: z-1, y-1, x-1), U_ii = A_ii - sum_k L_ik A_ki, U_ij = A_ij.
// inv(U_kk) of the three lower neighbours was produced one step earlier by
// this lane (z-1) or lane-1 / lane-wx, or by the west / south tile (edge
// buffers, 9 doubles per edge lane) -- the forward sweep's dependency
// structure.  Per row the arithmetic is the numeric factor kernel's fast
// path (factor.cu: matmul, then subtract, ascending k; the Gauss-Jordan
// inverse), so the factors are bit-identical to it.
//
// Factor record per (tile, step): meta[32] | A_i,z-1 A_i,y-1 A_i,x-1 |
// A_z-1,i A_y-1,i A_x-1,i | A_ii, element-pair interleaved like the sweeps'.
constexpr int kGwFacBlocks = 7;

__host__ __device__ inline int gw_rec_fac(int b) {
  return kGwMetaBytes + ((kGwFacBlocks * b * b + 1) & ~1) * 32 * 8;
}

// pack the factor records and the backward records' upper blocks straight
// from the input values (vsrc: plan-order slot -> input slot, null: same)
template <int B>
__global__ void __launch_bounds__(256, 4) k_gw_apack(GwDev g, const int32_t* __restrict__ src,
                           const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const int32_t* __restrict__ diag, const int32_t* __restrict__ vsrc,
                           const double* __restrict__ vin, char* __restrict__ fac) {
  constexpr int BB = B * B;
  constexpr int NE = (kGwFacBlocks * BB + 1) & ~1;
  const int rfa = gw_rec_fac(B);
  const long long total = (long long)g.TX * g.TY * g.S * 32;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(q % 32);
    const long long slot = q / 32;
    const int s = (int)(slot % g.S);
    const int t = (int)(slot / g.S);
    const int mt = reinterpret_cast<const int*>(g.recf + slot * g.rf)[lane];
    reinterpret_cast<int*>(fac + slot * rfa)[lane] = mt;
    double2* fv = reinterpret_cast<double2*>(fac + slot * rfa + kGwMetaBytes) + lane;
    double* Uv = reinterpret_cast<double*>(const_cast<char*>(g.recb) + slot * g.rb + kGwMetaBytes);
    const int32_t* sp = src + slot * 6 * 32 + lane;
    const int pr = mt >= 0 ? (mt & 0x1FFFFFF) : -1;
    auto val = [&](long long p, int e) {
      return p >= 0 ? vin[(vsrc ? (long long)vsrc[p] : p) * BB + e] : 0.0;
    };
    // CSR slots: A_ik (kinds 0..2), A_ki = the lower neighbour's plus-entry of
    // the opposite kind, read from the neighbour's own slot of src, A_ii
    long long pa[kGwFacBlocks];
    const GwTile a = gw_tile(g, t, lane);
    const int x = a.x0 + a.xl, y = a.y0 + a.yl, z = a.L0 + s - x - y;
    for (int k = 0; k < 3; ++k) {
      const int p = mt >= 0 ? sp[k * 32] : -1;
      pa[k] = p;
      pa[3 + k] = -1;
      if (p < 0) continue;
      const int nx_ = x - (k == 2), ny_ = y - (k == 1), nz_ = z - (k == 0);   // the neighbour
      const int ntx = nx_ / g.wx, nty = ny_ / g.wy;
      const int nxl = nx_ - ntx * g.wx, nyl = ny_ - nty * g.wy;
      const long long nslot = (long long)(nty * g.TX + ntx) * g.S + nxl + nyl + nz_;
      pa[3 + k] = src[nslot * 6 * 32 + (5 - k) * 32 + nxl + g.wx * nyl];   // kinds 5,4,3
    }
    pa[6] = pr >= 0 ? diag[pr] : -1;
    // input offsets of the seven blocks, then the elements streamed through
    // in record order (a few in flight, not all 63: occupancy)
    const double* bp[kGwFacBlocks];
#pragma unroll
    for (int j = 0; j < kGwFacBlocks; ++j)
      bp[j] = pa[j] >= 0 ? vin + (vsrc ? (long long)vsrc[pa[j]] : pa[j]) * BB : nullptr;
#pragma unroll
    for (int e = 0; e < NE; e += 2) {
      const int j0 = e / BB, j1 = (e + 1) / BB;
      const double v0 = bp[j0] ? bp[j0][e - j0 * BB] : 0.0;
      const double v1 = (e + 1 < kGwFacBlocks * BB && bp[j1]) ? bp[j1][e + 1 - j1 * BB] : 0.0;
      fv[(e >> 1) * 32] = make_double2(v0, v1);
    }
    for (int k = 3; k < 6; ++k) {
      const int p = mt >= 0 ? sp[k * 32] : -1;
      for (int e = 0; e < BB; ++e) Uv[gw_eidx((k - 3) * BB + e, lane)] = val(p, e);
    }
  }
}

template <int B> struct GwFacRing { static constexpr int deep = B <= 3 ? 4 : 2, shallow = B <= 3 ? 2 : 1; };

template <int B, int SH>
__global__ void __launch_bounds__(32) k_gw_factor(GwDev g, const char* __restrict__ fac,
                                                  double* eFE, double* eFN,
                                                  double* __restrict__ invd,
                                                  double* __restrict__ dvals, int* bad) {
  constexpr int BB = B * B;
  constexpr int R = SH ? GwFacRing<B>::shallow : GwFacRing<B>::deep;
  extern __shared__ __align__(128) char smem[];
  griddep_wait();
  griddep_launch();
  const int lane = threadIdx.x & 31;
  const GwTile a = gw_tile(g, blockIdx.x, lane);
  const long long base = (long long)a.t * g.S;
  const int rfa = gw_rec_fac(B);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
  char* ring = smem + 128;
  if (threadIdx.x == 0) {
    for (int q = 0; q < R; ++q) gw_mbar_init_n(full + q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int j) {
    const int q = j % R;
    gw_mbar_expect(full + q, (unsigned)rfa);
    gw_bulk(ring + q * rfa, fac + (base + j) * (long long)rfa, (unsigned)rfa, full + q);
  };
  if (lane == 0)
    for (int j = 0; j < R && j < a.St; ++j) issue(j);
  const bool hasW = a.tx > 0, hasS = a.ty > 0;
  const bool hasE = a.tx + 1 < g.TX, hasN = a.ty + 1 < g.TY;
  const bool xe = a.xl == 0 && hasW, ye = a.yl == 0 && hasS;
  const bool px = a.xl == a.xw - 1 && hasE, py = a.yl == a.yw - 1 && hasN;
  // neighbour tiles' inverse blocks needed at our step s: their step s+wx-1 / s+wy-1
  const double* xin = eFE + (((base - g.S) + (g.wx - 1)) * g.wy + a.yl) * BB;
  const double* yin = eFN + (((base - (long long)g.TX * g.S) + (g.wy - 1)) * g.wx + a.xl) * BB;
  double* xout = eFE + (base * g.wy + a.yl) * BB;
  double* yout = eFN + (base * g.wx + a.xl) * BB;
  const long long xstride = (long long)g.wy * BB, ystride = (long long)g.wx * BB;
  auto xok = [&](int s) { const int t = s + g.wx - 1; return xe && t >= 0 && t < g.S; };
  auto yok = [&](int s) { const int t = s + g.wy - 1; return ye && t >= 0 && t < g.S; };
  const int sx = lane > 0 ? lane - 1 : 0;
  const int sy = lane >= g.wx ? lane - g.wx : 0;
  double prev[BB];
#pragma unroll
  for (int e = 0; e < BB; ++e) prev[e] = 0.0;
  // the neighbour tiles' inverse blocks, requested one step early (all
  // elements in flight at once; re-read together while any is unproduced)
  double ex[BB], ey[BB];
#pragma unroll
  for (int e = 0; e < BB; ++e) ex[e] = ey[e] = sentinel();
  if (a.St > 0) {
    if (xok(0)) gw_load<BB>(xin, ex);
    if (yok(0)) gw_load<BB>(yin, ey);
  }
  for (int j = 0; j < a.St; ++j) {
    const int q = j % R;
    gw_mbar_wait(full + q, (unsigned)((j / R) & 1));
    const char* st_ = ring + q * rfa;
    const int mt = reinterpret_cast<const int*>(st_)[lane];
    const double2* blk = reinterpret_cast<const double2*>(st_ + kGwMetaBytes) + lane;
    double A[kGwFacBlocks * BB + 1];
#pragma unroll
    for (int e = 0; e < kGwFacBlocks * BB; e += 2) {
      const double2 v = blk[(e >> 1) * 32];
      A[e] = v.x;
      A[e + 1] = v.y;
    }
    __syncwarp();
    if (lane == 0 && j + R < a.St) {
      gw_fence_proxy();
      issue(j + R);
    }
    const int mask = mt >= 0 ? (mt >> 25) : 0;
    // the three lower neighbours' inverse blocks (z-1: own previous step)
    double dz[BB], dy[BB], dx[BB];
#pragma unroll
    for (int e = 0; e < BB; ++e) {
      dz[e] = prev[e];
      dx[e] = __shfl_sync(0xffffffffu, prev[e], sx);
      dy[e] = __shfl_sync(0xffffffffu, prev[e], sy);
    }
    if (xok(j) && (mask & kXm)) {
      gw_poll<BB>(xin + (long long)j * xstride, ex);
#pragma unroll
      for (int e = 0; e < BB; ++e) dx[e] = ex[e];
    }
    if (yok(j) && (mask & kYm)) {
      gw_poll<BB>(yin + (long long)j * ystride, ey);
#pragma unroll
      for (int e = 0; e < BB; ++e) dy[e] = ey[e];
    }
    if (j + 1 < a.St) {   // the next step's edge inputs, one step early
      if (xok(j + 1)) gw_load<BB>(xin + (long long)(j + 1) * xstride, ex);
      if (yok(j + 1)) gw_load<BB>(yin + (long long)(j + 1) * ystride, ey);
    }
    // ascending plan columns z-1, y-1, x-1; an absent neighbour has zero
    // blocks and a zero-selected inverse: its product and update are +0.0
    double dblk[BB], L[3][BB];
#pragma unroll
    for (int e = 0; e < BB; ++e) dblk[e] = A[6 * BB + e];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int bit = k == 0 ? kZm : (k == 1 ? kYm : kXm);
      const double* dep = k == 0 ? dz : (k == 1 ? dy : dx);
      const bool on = (mask & bit) != 0;
      double d[BB], prod[BB];
#pragma unroll
      for (int e = 0; e < BB; ++e) d[e] = on ? dep[e] : 0.0;
      matmul<B>(A + k * BB, d, L[k]);              // L_ik = A_ik inv(U_kk)
      matmul<B>(L[k], A + (3 + k) * BB, prod);     // A_ii -= L_ik U_ki (= A_ki)
#pragma unroll
      for (int e = 0; e < BB; ++e) dblk[e] -= prod[e];
    }
    double inv[BB];
    const bool ok = invert_block<B>(dblk, inv);
    if (mt >= 0) {
      const int pr = mt & 0x1FFFFFF;
      if (!ok) atomicMin(bad, pr);
      double* Lv = reinterpret_cast<double*>(const_cast<char*>(g.recf) + (base + j) * g.rf + kGwMetaBytes);
      double* Iv = reinterpret_cast<double*>(const_cast<char*>(g.recb) + (base + j) * g.rb + kGwMetaBytes);
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int e = 0; e < BB; ++e) Lv[gw_eidx(k * BB + e, lane)] = L[k][e];
#pragma unroll
      for (int e = 0; e < BB; ++e) {
        const double o = canon(inv[e]);
        prev[e] = o;
        Iv[gw_eidx(3 * BB + e, lane)] = o;
        invd[(long long)pr * BB + e] = o;
        dvals[(long long)pr * BB + e] = dblk[e];
      }
      if (px) {
#pragma unroll
        for (int e = 0; e < BB; ++e) gw_st_relaxed(xout + (long long)j * xstride + e, prev[e]);
      }
      if (py) {
#pragma unroll
        for (int e = 0; e < BB; ++e) gw_st_relaxed(yout + (long long)j * ystride + e, prev[e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < BB; ++e) prev[e] = 0.0;
    }
  }
}

// the combined L\U (plan-order CSR) from the records: L blocks and U_ii
// over the gathered operator values (materialised only on request)
template <int B>
__global__ void k_gw_unpack_lu(GwDev g, const int32_t* __restrict__ src,
                               const int32_t* __restrict__ diag,
                               const double* __restrict__ dvals, double* __restrict__ lu) {
  constexpr int BB = B * B;
  const long long total = (long long)g.TX * g.TY * g.S * 32;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(q % 32);
    const long long slot = q / 32;
    const int mt = reinterpret_cast<const int*>(g.recf + slot * g.rf)[lane];
    if (mt < 0) continue;
    const int pr = mt & 0x1FFFFFF;
    const double* Lv = reinterpret_cast<const double*>(g.recf + slot * g.rf + kGwMetaBytes);
    const int32_t* sp = src + slot * 6 * 32 + lane;
    for (int k = 0; k < 3; ++k) {
      const int p = sp[k * 32];
      if (p >= 0)
        for (int e = 0; e < BB; ++e) lu[(long long)p * BB + e] = Lv[gw_eidx(k * BB + e, lane)];
    }
    const long long pd = diag[pr];
    for (int e = 0; e < BB; ++e) lu[pd * BB + e] = dvals[(long long)pr * BB + e];
  }
}

// the sweep's input in step order / its output back to plan order
template <int B>
__global__ void k_gw_gather(GwDev g, const double* __restrict__ r) {
  griddep_wait();
  griddep_launch();
  const long long total = (long long)g.TX * g.TY * g.S * 32;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long slot = q >> 5;
    const int lane = (int)(q & 31);
    const int mt = reinterpret_cast<const int*>(g.recf + slot * g.rf)[lane];
    const long long pr = mt & 0x1FFFFFF;
#pragma unroll
    for (int c = 0; c < B; ++c) g.rpk[(slot * B + c) * 32 + lane] = mt >= 0 ? r[pr * B + c] : 0.0;
  }
}


// ---- packing, one thread per (tile, step, lane).  Pattern phase (before
// the numeric factorisation): meta words, the CSR slot of each of the six
// stencil entries, and the row-by-row check that the plan is a stencil plan.
// Value phase (after it, asynchronous): the blocks into the step records.
__global__ void k_gw_meta(GwDev g, int32_t* __restrict__ src, const int32_t* __restrict__ perm,
                          const int32_t* __restrict__ iperm, const int32_t* __restrict__ rp,
                          const int32_t* __restrict__ ci, int* bad) {
  const long long T = (long long)g.TX * g.TY;
  const long long total = T * g.S * 32;
  const long long nxy = (long long)g.nx * g.ny;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(q % 32);
    const long long slot = q / 32;
    const int s = (int)(slot % g.S);
    const int t = (int)(slot / g.S);
    const GwTile a = gw_tile(g, t, lane);
    const int x = a.x0 + a.xl, y = a.y0 + a.yl, z = a.L0 + s - x - y;
    int* mf = reinterpret_cast<int*>(const_cast<char*>(g.recf) + slot * g.rf);
    int* mb = reinterpret_cast<int*>(const_cast<char*>(g.recb) + slot * g.rb);
    int32_t* sp = src + slot * 6 * 32 + lane;
    for (int k = 0; k < 6; ++k) sp[k * 32] = -1;
    if (!a.valid || s >= a.St || z < 0 || z >= g.nz) {
      mf[lane] = mb[lane] = -1;
      continue;
    }
    const long long i = x + (long long)g.nx * y + nxy * z;   // natural (input) row
    const int pr = perm[i];
    int mask = 0;
    for (int p = rp[pr]; p < rp[pr + 1]; ++p) {
      const int c = ci[p];
      const long long d = (long long)iperm[c] - i;
      int kind = -1;
      if (d == 0) continue;
      if (d == -nxy && z > 0) kind = 0;
      else if (d == -g.nx && y > 0) kind = 1;
      else if (d == -1 && x > 0) kind = 2;
      else if (d == 1 && x + 1 < g.nx) kind = 3;
      else if (d == g.nx && y + 1 < g.ny) kind = 4;
      else if (d == nxy && z + 1 < g.nz) kind = 5;
      // lower entries must be the minus-neighbours and precede the row in the plan
      if (kind < 0 || (kind < 3) != (c < pr) || (mask & (1 << kind))) { atomicExch(bad, 1); continue; }
      mask |= 1 << kind;
      sp[kind * 32] = p;
    }
    // the kernels accumulate in kind order (z-1, y-1, x-1 / x+1, y+1, z+1):
    // it must be the ascending plan-column (CSR slot) order of the row
    for (int h = 0; h < 2; ++h) {
      int last = -1;
      for (int k = 3 * h; k < 3 * h + 3; ++k) {
        const int p = sp[k * 32];
        if (p < 0) continue;
        if (p < last) atomicExch(bad, 1);
        last = p;
      }
    }
    mf[lane] = mb[lane] = pr | (mask << 25);
  }
}

// record order = ascending plan columns: forward z-1, y-1, x-1 (kinds 0..2),
// backward x+1, y+1, z+1 (kinds 3..5), then inv(U_ii)
__global__ void k_gw_vals(GwDev g, int bb, const int32_t* __restrict__ src,
                          const double* __restrict__ lu, const double* __restrict__ inv) {
  const long long total = (long long)g.TX * g.TY * g.S * 32;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(q % 32);
    const long long slot = q / 32;
    const int mt = reinterpret_cast<const int*>(g.recf + slot * g.rf)[lane];
    double* Lv = reinterpret_cast<double*>(const_cast<char*>(g.recf) + slot * g.rf + kGwMetaBytes);
    double* Uv = reinterpret_cast<double*>(const_cast<char*>(g.recb) + slot * g.rb + kGwMetaBytes);
    const int32_t* sp = src + slot * 6 * 32 + lane;
    for (int k = 0; k < 6; ++k) {
      const int p = sp[k * 32];
      double* dst = k < 3 ? Lv : Uv;
      for (int e = 0; e < bb; ++e)
        dst[gw_eidx((k % 3) * bb + e, lane)] = p >= 0 ? lu[(long long)p * bb + e] : 0.0;
    }
    const long long pr = mt >= 0 ? (mt & 0x1FFFFFF) : -1;
    for (int e = 0; e < bb; ++e) Uv[gw_eidx(3 * bb + e, lane)] = pr >= 0 ? inv[pr * bb + e] : 0.0;
    if ((3 * bb) & 1) Lv[gw_eidx(3 * bb, lane)] = 0.0;   // (the pad of an odd count)
  }
}

__global__ void k_gw_fill(long long m, double* v) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m;
       t += (long long)gridDim.x * blockDim.x)
    v[t] = sentinel();
}

struct GwHandle {
  GwDev g;
  int b, n;
  void* mem;       // own allocation (unused: the caller's workspace)
  int32_t* src;    // [slots][6][32] CSR slot of each stencil entry (-1: none)
};

inline int gw_smem_bytes(const GwDev& g, int b, int dir) {
  const int r = dir == 0 ? (g.shallow ? kGwRingFs : kGwRingF) : (g.shallow ? kGwRingBs : kGwRingB);
  return 128 + r * ((dir == 0 ? g.rf : g.rb) + b * 32 * 8);
}
static_assert(2 * 8 * (kGwRingF > kGwRingB ? kGwRingF : kGwRingB) <= 128, "mbarriers fit");

template <int B>
int launch_gw_b(const GwHandle* h, const double* r, double* z, const int* done, cudaStream_t st,
                bool pdl) {
  const GwDev& g = h->g;
  const long long total = (long long)g.TX * g.TY * g.S * 32;
  long long grid = (total + 255) / 256;
  if (grid > kSms * 16) grid = kSms * 16;
  // The tiles wait on each other, so the sweep grids must be co-resident:
  // b2s_gw_create admits a grid only when it fits the occupancy bound, and
  // a tile can only wait on tiles that are running or will get a slot once
  // the (finite) predecessor grids drain.  Not a cooperative launch: those
  // cannot overlap their predecessor (PDL) and add a drain in CUDA graphs.
  if (launch_k(k_gw_gather<B>, dim3((int)grid), dim3(256), 0, st, pdl, g, r) != cudaSuccess ||
      launch_k(g.shallow ? k_gw_sweep<B, 0, 1> : k_gw_sweep<B, 0, 0>, dim3(g.TX * g.TY), dim3(32),
               gw_smem_bytes(g, B, 0), st, pdl, g, done, z) != cudaSuccess ||
      launch_k(g.shallow ? k_gw_sweep<B, 1, 1> : k_gw_sweep<B, 1, 0>, dim3(g.TX * g.TY), dim3(32),
               gw_smem_bytes(g, B, 1), st, pdl, g, done, z) != cudaSuccess)
    return B2S_CUDA_ERROR;
  return B2S_OK;
}

// z = U^-1 L^-1 r (plan order) with the wavefront kernels
int launch_gw(int b, const void* handle, const double* r, double* z, const int* done,
              cudaStream_t st, bool pdl) {
  const GwHandle* h = reinterpret_cast<const GwHandle*>(handle);
  switch (b) {
    case 1: return launch_gw_b<1>(h, r, z, done, st, pdl);
    case 2: return launch_gw_b<2>(h, r, z, done, st, pdl);
    case 3: return launch_gw_b<3>(h, r, z, done, st, pdl);
    case 4: return launch_gw_b<4>(h, r, z, done, st, pdl);
    default: return B2S_UNSUPPORTED;
  }
}

inline int gw_fac_smem(int b, int shallow) {
  const int r = b <= 3 ? (shallow ? GwFacRing<3>::shallow : GwFacRing<3>::deep)
                       : (shallow ? GwFacRing<4>::shallow : GwFacRing<4>::deep);
  return 128 + r * gw_rec_fac(b);
}

// pack + factor (stream-ordered); B2S_UNSUPPORTED when the tiles cannot all
// be co-resident with either factor ring
template <int B>
int launch_gw_factor(const GwDev& g, const int32_t* src, const int32_t* rp, const int32_t* ci,
                     const int32_t* diag, const int32_t* vsrc, const double* vals, char* fac,
                     double* eFE, double* eFN, double* invd, double* dvals, int* bad,
                     cudaStream_t st) {
  const long long T = (long long)g.TX * g.TY;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int shallow = -1;
  for (int sh = 0; sh < 2 && shallow < 0; ++sh) {
    const int sm = gw_fac_smem(B, sh);
    const void* fn = sh ? (const void*)k_gw_factor<B, 1> : (const void*)k_gw_factor<B, 0>;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) != cudaSuccess)
      return B2S_CUDA_ERROR;
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 32, sm);
    if (T <= (long long)per * sms) shallow = sh;
  }
  if (shallow < 0) return B2S_UNSUPPORTED;
  const long long slots = T * g.S;
  const long long ne = slots * (g.wx + g.wy) * B * B;   // eFE and eFN are contiguous
  long long gf = (ne + 255) / 256;
  if (gf > kSms * 16) gf = kSms * 16;
  k_gw_fill<<<(int)gf, 256, 0, st>>>(ne, eFE);
  long long grid = (slots * 32 + 255) / 256;
  if (grid > kSms * 64) grid = kSms * 64;
  k_gw_apack<B><<<(int)grid, 256, 0, st>>>(g, src, rp, ci, diag, vsrc, vals, fac);
  const int sm = gw_fac_smem(B, shallow);
  const cudaError_t e =
      shallow ? launch_k(k_gw_factor<B, 1>, dim3((unsigned)T), dim3(32), sm, st, false, g,
                         (const char*)fac, eFE, eFN, invd, dvals, bad)
              : launch_k(k_gw_factor<B, 0>, dim3((unsigned)T), dim3(32), sm, st, false, g,
                         (const char*)fac, eFE, eFN, invd, dvals, bad);
  return e == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

template <int B, int SH>
int gw_configure_r(GwDev& g, int* per_sm) {
  g.shallow = SH;
  const int s0 = gw_smem_bytes(g, B, 0), s1 = gw_smem_bytes(g, B, 1);
  if (cudaFuncSetAttribute((const void*)k_gw_sweep<B, 0, SH>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, s0) != cudaSuccess ||
      cudaFuncSetAttribute((const void*)k_gw_sweep<B, 1, SH>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, s1) != cudaSuccess)
    return B2S_CUDA_ERROR;
  int a = 0, c = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_gw_sweep<B, 0, SH>, 32, s0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_gw_sweep<B, 1, SH>, 32, s1);
  *per_sm = a < c ? a : c;
  return B2S_OK;
}

// the deep rings when the tiles fit them, else the shallow ones; per_sm is
// the co-residency bound of the choice
template <int B>
int gw_configure(GwDev& g, long long tiles, int sms, int* per_sm) {
  int rc = gw_configure_r<B, 0>(g, per_sm);
  if (rc != B2S_OK || tiles <= (long long)*per_sm * sms) return rc;
  return gw_configure_r<B, 1>(g, per_sm);
}

}  // namespace b2s

using namespace b2s;

extern "C" {

// Pack the factor of a natural-order nx*ny*nz 7-point grid for the wavefront
// sweeps.  perm/iperm: the plan (old row -> plan row / plan row -> old row);
// rp/ci/lu: the combined L\U in plan order (int32 pattern, b*b blocks), inv:
// the inverse diagonal blocks in plan order.  B2S_UNSUPPORTED when the grid
// does not fit (more tiles than can be co-resident) or some row is not a
// stencil row of that plan -- the caller keeps the sync-free sweeps.
static void gw_shape(GwDev& g, int b, int nx, int ny, int nz, int wx, int wy) {
  g.nx = nx; g.ny = ny; g.nz = nz; g.wx = wx; g.wy = wy;
  g.TX = (nx + wx - 1) / wx;
  g.TY = (ny + wy - 1) / wy;
  g.S = (wx - 1) + (wy - 1) + nz;
  const int bb = b * b;
  // block elements in lane-interleaved pairs (one 16-byte shared load per
  // two elements): element counts rounded up to even
  g.rf = kGwMetaBytes + ((3 * bb + 1) & ~1) * 32 * 8;
  g.rb = kGwMetaBytes + ((4 * bb + 1) & ~1) * 32 * 8;
}

static long long gw_bytes(const GwDev& g, int b) {
  const long long slots = (long long)g.TX * g.TY * g.S;
  return slots * ((long long)g.rf + g.rb) +
         (2 * slots * b * 32 + 2 * slots * g.wy * b + 2 * slots * g.wx * b) * 8 +
         slots * 6 * 32 * 4 + 256;
}

// device bytes b2s_gw_create needs as its workspace (0: bad shape)
long long b2s_gw_workspace_bytes(int n, int b, int nx, int ny, int nz, int wx, int wy) {
  if (b < 1 || b > 4 || nx < 1 || ny < 1 || nz < 1 || (long long)nx * ny * nz != n || wx < 1 ||
      wy < 1 || wx * wy > kGwLanes)
    return 0;
  GwDev g{};
  gw_shape(g, b, nx, ny, nz, wx, wy);
  return gw_bytes(g, b);
}

// Pattern phase: shapes, meta words and the stencil check of every row (one
// synchronisation, before the numeric factorisation is queued).
int b2s_gw_create(int n, int b, int nx, int ny, int nz, int wx, int wy, const int32_t* perm,
                  const int32_t* iperm, const int32_t* rp, const int32_t* ci, void* workspace,
                  long long ws_bytes, void** handle_out, cudaStream_t st) {
  *handle_out = nullptr;
  if (b < 1 || b > 4 || nx < 1 || ny < 1 || nz < 1 || (long long)nx * ny * nz != n ||
      wx < 1 || wy < 1 || wx * wy > kGwLanes || n >= (1 << 25) || !workspace)
    return B2S_SHAPE;
  GwHandle* h = new GwHandle();
  GwDev& g = h->g;
  gw_shape(g, b, nx, ny, nz, wx, wy);
  if (ws_bytes < gw_bytes(g, b)) { delete h; return B2S_SHAPE; }
  const long long T = (long long)g.TX * g.TY;
  // every tile waits on its neighbours: all CTAs must be co-resident
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int rc = B2S_OK;
  switch (b) {
    case 1: rc = gw_configure<1>(g, T, sms, &per_sm); break;
    case 2: rc = gw_configure<2>(g, T, sms, &per_sm); break;
    case 3: rc = gw_configure<3>(g, T, sms, &per_sm); break;
    default: rc = gw_configure<4>(g, T, sms, &per_sm); break;
  }
  if (rc != B2S_OK) { delete h; return rc; }
  if (T > (long long)per_sm * sms) { delete h; return B2S_UNSUPPORTED; }
  const long long slots = T * g.S;
  const long long nV = slots * b * 32;
  const long long nEx = slots * wy * b, nEy = slots * wx * b;
  h->mem = nullptr;   // the workspace belongs to the caller
  char* p = reinterpret_cast<char*>(workspace);
  g.recf = p; p += slots * g.rf;
  g.recb = p; p += slots * g.rb;
  double* d = reinterpret_cast<double*>(p);
  g.rpk = d; d += nV;
  g.ypk = d; d += nV;
  g.eE = d; d += nEx;
  g.eW = d; d += nEx;
  g.eN = d; d += nEy;
  g.eS = d; d += nEy;
  h->src = reinterpret_cast<int32_t*>(d);
  g.trace = nullptr;
  const long long trace_words = 2 * slots + (long long)g.TX * g.TY * (1 + 4 * kGwTl);
  if (getenv("B2S_GW_TRACE") && (cudaMalloc(&g.trace, trace_words * 8) != cudaSuccess ||
                                 cudaMemset(g.trace, 0, trace_words * 8) != cudaSuccess))
    g.trace = nullptr;
  h->b = b;
  h->n = n;
  int* bad = nullptr;
  int hbad = 0;
  bool ok = cudaMallocAsync(&bad, sizeof(int), st) == cudaSuccess &&
            cudaMemsetAsync(bad, 0, sizeof(int), st) == cudaSuccess;
  if (ok) {
    long long grid = (slots * 32 + 255) / 256;
    if (grid > kSms * 64) grid = kSms * 64;
    k_gw_meta<<<(int)grid, 256, 0, st>>>(g, h->src, perm, iperm, rp, ci, bad);
    // all four edge buffers start "not produced" (each sweep then re-arms the
    // other direction's buffers of its own tile)
    const long long ne = 2 * nEx + 2 * nEy;
    long long eg = (ne + 255) / 256;
    if (eg > kSms * 16) eg = kSms * 16;
    k_gw_fill<<<(int)(eg < 1 ? 1 : eg), 256, 0, st>>>(ne, g.eE);
    ok = cudaGetLastError() == cudaSuccess &&
         cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
         cudaFreeAsync(bad, st) == cudaSuccess && cudaStreamSynchronize(st) == cudaSuccess;
  }
  if (!ok || hbad) {
    if (g.trace) cudaFree(g.trace);
    delete h;
    return ok ? B2S_UNSUPPORTED : B2S_CUDA_ERROR;
  }
  *handle_out = h;
  return B2S_OK;
}

// Value phase: the factor's blocks into the step records (stream-ordered,
// no synchronisation).  lu: combined L\U in plan order on the pattern given to
// create; inv: inverse diagonal blocks in plan order.
int b2s_gw_fill(void* handle, const double* lu, const double* inv, cudaStream_t st) {
  GwHandle* h = reinterpret_cast<GwHandle*>(handle);
  if (!h) return B2S_SHAPE;
  const long long slots = (long long)h->g.TX * h->g.TY * h->g.S;
  long long grid = (slots * 32 + 255) / 256;
  if (grid > kSms * 64) grid = kSms * 64;
  k_gw_vals<<<(int)grid, 256, 0, st>>>(h->g, h->b * h->b, h->src, lu, inv);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

// debug: copy the step end times [2][T][S] (ns, globaltimer) of the last
// apply into host memory (B2S_GW_TRACE set at create); *count = 2*T*S.
// cap >= 2*T*S + T*(1 + 4*64): also each tile's (entry, dependency wait
// done, exit, direction) of its last 64 sweep launches (trace builds)
int b2s_gw_trace(const void* handle, unsigned long long* host, long long cap, long long* count,
                 int* shape) {
  const GwHandle* h = reinterpret_cast<const GwHandle*>(handle);
  const long long n = 2ll * h->g.TX * h->g.TY * h->g.S;
  *count = n;
  shape[0] = h->g.TX; shape[1] = h->g.TY; shape[2] = h->g.S; shape[3] = h->g.wx; shape[4] = h->g.wy;
  if (!h->g.trace || cap < n) return B2S_SHAPE;
  // with room for it, also the per-launch timeline of a trace build
  const long long tl = (long long)h->g.TX * h->g.TY * (1 + 4 * kGwTl);
  B2S_CHECK(cudaMemcpy(host, h->g.trace, (cap >= n + tl ? n + tl : n) * 8, cudaMemcpyDeviceToHost));
  return B2S_OK;
}

// Scratch bytes b2s_gw_factor needs (factor records + its edge buffers).
long long b2s_gw_factor_workspace_bytes(const void* handle) {
  const GwHandle* h = reinterpret_cast<const GwHandle*>(handle);
  if (!h) return 0;
  const long long slots = (long long)h->g.TX * h->g.TY * h->g.S;
  return slots * gw_rec_fac(h->b) + slots * (h->g.wx + h->g.wy) * h->b * h->b * 8 + 256;
}

// ILU0 of the grid given to create, straight from the input values (vsrc:
// plan-order CSR slot -> input slot, null when the plan is the identity;
// rp/ci/diag: the plan-order pattern and its diagonal slots), into the step
// records (no b2s_gw_fill needed), the plan-order inverse diagonals invd and
// U_ii (dvals, n*b*b).  Bit-identical to b2s_ilu0_factor on these patterns.
// bad_dev (device int, INT32_MAX on entry) receives the smallest singular
// plan row.  Stream-ordered, no host read.  B2S_UNSUPPORTED when the tiles do
// not fit co-resident (the caller factorises the general way).
int b2s_gw_factor(void* handle, const int32_t* rp, const int32_t* ci, const int32_t* diag,
                  const int32_t* vsrc, const double* vals, double* invd, double* dvals,
                  int* bad_dev, void* work, long long work_bytes, cudaStream_t st) {
  GwHandle* h = reinterpret_cast<GwHandle*>(handle);
  if (!h || !rp || !ci || !diag || !vals || !invd || !dvals || !bad_dev || !work) return B2S_SHAPE;
  if (work_bytes < b2s_gw_factor_workspace_bytes(handle)) return B2S_SHAPE;
  const long long slots = (long long)h->g.TX * h->g.TY * h->g.S;
  char* fac = reinterpret_cast<char*>(work);
  double* eF = reinterpret_cast<double*>(fac + slots * gw_rec_fac(h->b));
  double* eFN = eF + slots * h->g.wy * h->b * h->b;
  int rc;
  switch (h->b) {
    case 1: rc = launch_gw_factor<1>(h->g, h->src, rp, ci, diag, vsrc, vals, fac, eF, eFN, invd, dvals, bad_dev, st); break;
    case 2: rc = launch_gw_factor<2>(h->g, h->src, rp, ci, diag, vsrc, vals, fac, eF, eFN, invd, dvals, bad_dev, st); break;
    case 3: rc = launch_gw_factor<3>(h->g, h->src, rp, ci, diag, vsrc, vals, fac, eF, eFN, invd, dvals, bad_dev, st); break;
    case 4: rc = launch_gw_factor<4>(h->g, h->src, rp, ci, diag, vsrc, vals, fac, eF, eFN, invd, dvals, bad_dev, st); break;
    default: rc = B2S_UNSUPPORTED;
  }
  if (rc == B2S_OK) B2S_LAUNCH_CHECK();
  return rc;
}

// The combined L\U values (plan-order CSR) from a b2s_gw_factor: lu must
// hold the plan-order operator values; the L blocks and U_ii are written over.
int b2s_gw_unpack_lu(const void* handle, const int32_t* diag, const double* dvals, double* lu,
                     cudaStream_t st) {
  const GwHandle* h = reinterpret_cast<const GwHandle*>(handle);
  if (!h || !diag || !dvals || !lu) return B2S_SHAPE;
  const long long slots = (long long)h->g.TX * h->g.TY * h->g.S;
  long long grid = (slots * 32 + 255) / 256;
  if (grid > kSms * 64) grid = kSms * 64;
  switch (h->b) {
    case 1: k_gw_unpack_lu<1><<<(int)grid, 256, 0, st>>>(h->g, h->src, diag, dvals, lu); break;
    case 2: k_gw_unpack_lu<2><<<(int)grid, 256, 0, st>>>(h->g, h->src, diag, dvals, lu); break;
    case 3: k_gw_unpack_lu<3><<<(int)grid, 256, 0, st>>>(h->g, h->src, diag, dvals, lu); break;
    case 4: k_gw_unpack_lu<4><<<(int)grid, 256, 0, st>>>(h->g, h->src, diag, dvals, lu); break;
    default: return B2S_UNSUPPORTED;
  }
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

int b2s_gw_destroy(void* handle) {
  GwHandle* h = reinterpret_cast<GwHandle*>(handle);
  if (!h) return B2S_OK;
  if (h->g.trace) cudaFree(h->g.trace);
  if (h->mem) cudaFree(h->mem);
  delete h;
  return B2S_OK;
}

int b2s_gw_apply(int b, const void* handle, const double* r, double* z, cudaStream_t st) {
  if (!handle) return B2S_SHAPE;
  if (reinterpret_cast<const GwHandle*>(handle)->b != b) return B2S_SHAPE;
  return launch_gw(b, handle, r, z, nullptr, st, false);
}

}  // extern "C"
