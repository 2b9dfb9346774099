// Two-colour plans: the backward sweep of colour 0 fused with the SpMV rows
// of colour 0 (bs/ilu0.py:116-142 + bs/blockcore.py:349-363 on the same rows).
//
// Under a 2-colouring, in plan order every off-diagonal entry of a colour-0
// row points into colour 1 (higher plan index), so a colour-0 row of A is
// [A_ii, U_i*] and -- whenever no elimination update touches an
// off-diagonal block, which b2s_fuse_check verifies bit for bit at setup --
// those U blocks ARE A's blocks.  The Krylov step  p^ = M^-1 p ; v = A p^
// then needs colour-0's off-diagonal blocks once, not twice:
//
//   pass 1  k_phase_forward<LAST>  colour 1: y = p - L p ; p^ = inv(U_ii) y
//   pass 2  k_bwd_spmv             colour 0: acc = sum_j A_ij p^_j (ascending j)
//                                            p^_i = inv(U_ii) (p_i - acc)
//                                            v_i  = acc + A_ii p^_i
//   pass 3  k_spmv over colour 1             v_i = sum_j A_ij p^_j
//
// p^ is bit-identical to the unfused sweeps (same products, same order);
// v_i of a colour-0 row adds its diagonal product last instead of first,
// one rounding order among those the plan-order SpMV already differs from
// the reference's input-order sum by (tolerance parity).
// The dot-product epilogue of the SpMV (gamma, or tt/ts) is split over
// passes 2 and 3 with fixed partial slots; the last CTA of pass 3 reduces
// all of them in order and runs the scalar step (ctl.cuh).
#include "ctl.cuh"
#include "sell.cuh"

namespace b2s {

template <int PRE>
__device__ __forceinline__ double pre_form(double r, double p, double v, int k, double beta,
                                           double omega, double alpha) {
  if (PRE == kPreP) return k == 0 ? r : bicg_p(r, p, v, beta, omega);
  return bicg_axpy(r, alpha, v);
}

// strict-lower row sum of the colour-1 forward pass with on-the-fly inputs
// (phase_row_sum's order: entries in pairs, ascending columns)
template <int B, int PRE>
__device__ __forceinline__ void pre_row_sum(const Sell& m, int slot0, int width, int lane,
                                            const PreIn& in, int k, double beta, double omega,
                                            double alpha, double (&acc)[B]) {
  constexpr int BB = B * B;
  int cn0 = width > 0 ? __ldcs(m.cols + slot0 + lane) : -1;
  int cn1 = width > 1 ? __ldcs(m.cols + slot0 + 32 + lane) : -1;
  for (int kk = 0; kk < width; kk += 2) {
    const int col[2] = {cn0, cn1};
    cn0 = kk + 2 < width ? __ldcs(m.cols + slot0 + 32 * (kk + 2) + lane) : -1;
    cn1 = kk + 3 < width ? __ldcs(m.cols + slot0 + 32 * (kk + 3) + lane) : -1;
    double blk[2][BB], dr[2][B], dp[2][B], dv[2][B];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int e = 0; e < BB; ++e)
        blk[q][e] = col[q] >= 0 ? __ldcs(m.vals + vidx(slot0, kk + q, e, lane, BB)) : 0.0;
      const long long cq = col[q] < 0 ? 0 : col[q];
#pragma unroll
      for (int c = 0; c < B; ++c) {
        dr[q][c] = col[q] >= 0 ? __ldg(in.r + cq * B + c) : 0.0;
        dv[q][c] = (col[q] >= 0 && (PRE == kPreS || k > 0)) ? __ldg(in.v + cq * B + c) : 0.0;
        dp[q][c] = (PRE == kPreP && col[q] >= 0 && k > 0) ? __ldg(in.io + cq * B + c) : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (col[q] < 0) continue;
      double dep[B], pr[B];
#pragma unroll
      for (int c = 0; c < B; ++c)
        dep[c] = pre_form<PRE>(dr[q][c], dp[q][c], dv[q][c], k, beta, omega, alpha);
      matvec<B>(blk[q], dep, pr);
#pragma unroll
      for (int c = 0; c < B; ++c) acc[c] += pr[c];
    }
  }
}

// colour 1 (the last group of a 2-colouring: no upper entries):
// u = p or s formed on the fly (stored), z = inv(U_ii) (u - L u)
template <int B, int PRE>
__global__ void __launch_bounds__(256) k_fwd_pre(int s0, int s1, SliceMap map, Sell lo,
                                                 const double* __restrict__ dtiles, PreIn in,
                                                 double* __restrict__ z, const int* done) {
  constexpr int BB = B * B;
  __shared__ double red[8];
  griddep_wait();
  griddep_launch();
  if (done && *done) return;
  const int k = in.st->k;
  const double beta = in.st->beta, omega = in.st->omega, alpha = in.st->alpha;
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  double ss = 0.0;
  for (long long s = s0 + (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < s1;
       s += nw) {
    const bool ok = lane < map.nrows[s];
    const long long i = (long long)map.row0[s] + lane;
    const int slot0 = lo.sp[s];
    const int width = (lo.sp[s + 1] - slot0) >> 5;
    double own[B], acc[B], dinv[BB];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      const double rr = ok ? __ldcs(in.r + i * B + c) : 0.0;
      const double vv = (ok && (PRE == kPreS || k > 0)) ? __ldcs(in.v + i * B + c) : 0.0;
      const double pp = (ok && PRE == kPreP && k > 0) ? __ldcs(in.io + i * B + c) : 0.0;
      own[c] = pre_form<PRE>(rr, pp, vv, k, beta, omega, alpha);
      acc[c] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < BB; ++e) dinv[e] = __ldcs(dtiles + (s * BB + e) * 32 + lane);
    pre_row_sum<B, PRE>(lo, slot0, width, lane, in, k, beta, omega, alpha, acc);
    if (!ok) continue;
    double tv[B], out[B];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      in.io[i * B + c] = own[c];
      if (PRE == kPreS) ss = fma(own[c], own[c], ss);
      tv[c] = canon(own[c] - acc[c]) - 0.0;   // backward row of the last group: acc = 0
    }
    matvec<B>(dinv, tv, out);
#pragma unroll
    for (int c = 0; c < B; ++c) z[i * B + c] = canon(out[c]);
  }
  if (PRE == kPreS) {
    const double t = block_sum(ss, red);
    if (threadIdx.x == 0) in.pss[blockIdx.x] = t;
  }
}

template <int B, int MODE, int PRE>
__global__ void __launch_bounds__(256) k_bwd_spmv(SliceMap map, int s0, int s1, Sell a,
                                                  const double* __restrict__ dtiles,
                                                  const double* __restrict__ yin,
                                                  double* __restrict__ z,
                                                  double* v,
                                                  const double* __restrict__ w,
                                                  double* __restrict__ part0,
                                                  double* __restrict__ part1, const int* done,
                                                  PreIn in, double* __restrict__ uimg) {
  constexpr int BB = B * B;
  __shared__ double red[8];
  if ((threadIdx.x & 31) == 0) {
    const int s = s0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (s < s1) prefetch_slice<BB>(a, s, dtiles);
  }
  griddep_wait();
  griddep_launch();
  if (done && *done) return;
  int k = 0;
  double beta = 0.0, omega = 0.0, alpha = 0.0, ss = 0.0;
  if (PRE != kPreNone) {
    k = in.st->k; beta = in.st->beta; omega = in.st->omega; alpha = in.st->alpha;
  }
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  double p0 = 0.0, p1 = 0.0;
  for (int s = s0 + gw; s < s1; s += nw) {
    const bool ok = lane < map.nrows[s];
    const long long i = (long long)map.row0[s] + lane;
    const int slot0 = a.sp[s];
    const int width = (a.sp[s + 1] - slot0) >> 5;
    double yv[B], acc[B], dinv[BB], dg[BB];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      if (PRE == kPreNone) {
        yv[c] = ok ? __ldcs(yin + i * B + c) : 0.0;
      } else {   // this row's p or s, formed here (kPreP reads the old v before v_i is written)
        const double rr = ok ? __ldcs(in.r + i * B + c) : 0.0;
        const double vv = (ok && (PRE == kPreS || k > 0)) ? __ldcs(in.v + i * B + c) : 0.0;
        const double pp = (ok && PRE == kPreP && k > 0) ? __ldcs(in.io + i * B + c) : 0.0;
        yv[c] = pre_form<PRE>(rr, pp, vv, k, beta, omega, alpha);
      }
      acc[c] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < BB; ++e) {
      dinv[e] = __ldcs(dtiles + ((long long)s * BB + e) * 32 + lane);
      dg[e] = __ldcs(a.vals + vidx(slot0, 0, e, lane, BB));   // entry 0 = the diagonal
    }
    // two entries per step, every load of the pair issued before any math
    // (the compiler's own schedule of a one-entry loop left one L2 round
    // trip per entry exposed in one of the two instantiations)
    // (the next pair's column indices load one step ahead, as in k_spmv)
    int cn0 = width > 1 ? __ldcs(a.cols + slot0 + 32 + lane) : -1;
    int cn1 = width > 2 ? __ldcs(a.cols + slot0 + 64 + lane) : -1;
    for (int k = 1; k < width; k += 2) {
      const bool two = k + 1 < width;
      int col[2] = {cn0, cn1};
      cn0 = k + 2 < width ? __ldcs(a.cols + slot0 + 32 * (k + 2) + lane) : -1;
      cn1 = k + 3 < width ? __ldcs(a.cols + slot0 + 32 * (k + 3) + lane) : -1;
      double blk[2][BB], dep[2][B];
#pragma unroll
      for (int e = 0; e < BB; ++e) {
        blk[0][e] = __ldcs(a.vals + vidx(slot0, k, e, lane, BB));
        blk[1][e] = two ? __ldcs(a.vals + vidx(slot0, k + 1, e, lane, BB)) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const long long cq = col[q] < 0 ? 0 : col[q];
#pragma unroll
        for (int c = 0; c < B; ++c) dep[q][c] = __ldg(z + cq * B + c);
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (col[q] >= 0) {   // ascending columns; padding contributes nothing
          double pr[B];
          matvec<B>(blk[q], dep[q], pr);
#pragma unroll
          for (int c = 0; c < B; ++c) acc[c] += pr[c];
        }
      }
    }
    if (!ok) continue;
    double tv[B], zi[B], di[B];
    if (PRE != kPreNone) {
#pragma unroll
      for (int c = 0; c < B; ++c) {
        in.io[i * B + c] = yv[c];
        if (PRE == kPreS) ss = fma(yv[c], yv[c], ss);
      }
    }
#pragma unroll
    for (int c = 0; c < B; ++c) tv[c] = yv[c] - acc[c];
    matvec<B>(dinv, tv, zi);
#pragma unroll
    for (int c = 0; c < B; ++c) {
      zi[c] = canon(zi[c]);
      z[i * B + c] = zi[c];
    }
    matvec<B>(dg, zi, di);
    double vrow[B];
#pragma unroll
    for (int c = 0; c < B; ++c) vrow[c] = acc[c] + di[c];
    if (uimg) {   // s-image: u_i = inv(A_ii) v_i (the colour-1 SpMV forms F(v) from it)
      double ui[B];
      matvec<B>(dinv, vrow, ui);
#pragma unroll
      for (int c = 0; c < B; ++c) uimg[i * B + c] = ui[c];
    }
#pragma unroll
    for (int c = 0; c < B; ++c) {
      const double vv = vrow[c];
      v[i * B + c] = vv;
      if (MODE == kDotW) p0 = fma(w[i * B + c], vv, p0);
      if (MODE == kSelfAndW) {   // w = s: formed in this very pass under kPreS
        const double wv = PRE == kPreS ? yv[c] : w[i * B + c];
        p0 = fma(vv, vv, p0);
        p1 = fma(vv, wv, p1);
      }
    }
  }
  if (PRE == kPreS) {
    const double t = block_sum(ss, red);
    if (threadIdx.x == 0) in.pss[blockIdx.x] = t;
  }
  double t0 = block_sum(p0, red);
  if (threadIdx.x == 0) part0[blockIdx.x] = t0;
  if (MODE == kSelfAndW) {
    double t1 = block_sum(p1, red);
    if (threadIdx.x == 0) part1[blockIdx.x] = t1;
  }
}

// 1 in *bad unless every colour-0 row of A (slices [0, s1)) is exactly its
// diagonal followed by the U row: same columns, bitwise-equal blocks.
__global__ void k_fuse_check(SliceMap map, int s1, int bb, Sell a, Sell u, int* bad) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < s1; s += nw) {
    const int aw = (a.sp[s + 1] - a.sp[s]) >> 5, uw = (u.sp[s + 1] - u.sp[s]) >> 5;
    bool fail = aw < 1 || aw - 1 < uw;
    if (!fail && lane < map.nrows[s]) {
      const long long i = (long long)map.row0[s] + lane;
      fail |= a.cols[a.sp[s] + lane] != i;
      for (int k = 0; k + 1 < aw && !fail; ++k) {
        const int ac = a.cols[a.sp[s] + 32 * (k + 1) + lane];
        const int uc = k < uw ? u.cols[u.sp[s] + 32 * k + lane] : -1;
        fail |= ac != uc;
        if (ac >= 0 && !fail)
          for (int e = 0; e < bb; ++e)
            fail |= __double_as_longlong(a.vals[vidx(a.sp[s], k + 1, e, lane, bb)]) !=
                    __double_as_longlong(u.vals[vidx(u.sp[s], k, e, lane, bb)]);
      }
    }
    if (__any_sync(0xffffffffu, fail) && lane == 0) atomicExch(bad, 1);
  }
}

// one full wave: a fixed grid larger than the resident capacity leaves a
// partial second wave (measured: 1.33 waves doubled the pass time)
inline int one_wave(const void* fn, int cap) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int dev = 0, sms = kSms;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms < cap ? per_sm * sms : cap;
}

template <int B, int PRE>
int launch_bwd_spmv_bp(int mode, int nparts, SliceMap map, int s1, Sell a, const double* dt,
                       const double* yin, double* z, double* v, const double* w, double* p0,
                       double* p1, const int* done, int* grid_out, cudaStream_t st, bool pdl,
                       PreIn in, double* uimg) {
  if (mode == kDotW) {
    const int g = one_wave((const void*)k_bwd_spmv<B, kDotW, PRE>, nparts);
    *grid_out = g;
    launch_k(k_bwd_spmv<B, kDotW, PRE>, dim3(g), dim3(256), 0, st, pdl, map, 0, s1, a, dt, yin, z,
             v, w, p0, p1, done, in, uimg);
  } else if (mode == kSelfAndW) {
    const int g = one_wave((const void*)k_bwd_spmv<B, kSelfAndW, PRE>, nparts);
    *grid_out = g;
    launch_k(k_bwd_spmv<B, kSelfAndW, PRE>, dim3(g), dim3(256), 0, st, pdl, map, 0, s1, a, dt,
             yin, z, v, w, p0, p1, done, in, uimg);
  } else {
    return B2S_SHAPE;
  }
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

template <int B>
int launch_bwd_spmv_b(int mode, int nparts, SliceMap map, int s1, Sell a, const double* dt,
                      const double* yin, double* z, double* v, const double* w, double* p0,
                      double* p1, const int* done, int* grid_out, cudaStream_t st, bool pdl,
                      int pre, PreIn in, double* uimg) {
  if (pre == kPreP)
    return launch_bwd_spmv_bp<B, kPreP>(mode, nparts, map, s1, a, dt, yin, z, v, w, p0, p1, done,
                                        grid_out, st, pdl, in, uimg);
  if (pre == kPreS)
    return launch_bwd_spmv_bp<B, kPreS>(mode, nparts, map, s1, a, dt, yin, z, v, w, p0, p1, done,
                                        grid_out, st, pdl, in, uimg);
  return launch_bwd_spmv_bp<B, kPreNone>(mode, nparts, map, s1, a, dt, yin, z, v, w, p0, p1, done,
                                         grid_out, st, pdl, in, uimg);
}

// pass 2 of the fused pair (colour 0 = slices [0, s1)); partials at
// [0, *grid_out) -- at most nparts CTAs, one resident wave.  pre/in: form
// the input on the fly (kPreP / kPreS, PreIn) instead of reading yin.
int launch_bwd_spmv(int b, int mode, int nparts, SliceMap map, int s1, Sell a, const double* dt,
                    const double* yin, double* z, double* v, const double* w, double* p0,
                    double* p1, const int* done, int* grid_out, cudaStream_t st, bool pdl,
                    int pre, const PreIn* pre_in, double* uimg) {
  const PreIn in = pre_in ? *pre_in : PreIn{};
  switch (b) {
    case 1: return launch_bwd_spmv_b<1>(mode, nparts, map, s1, a, dt, yin, z, v, w, p0, p1, done, grid_out, st, pdl, pre, in, uimg);
    case 2: return launch_bwd_spmv_b<2>(mode, nparts, map, s1, a, dt, yin, z, v, w, p0, p1, done, grid_out, st, pdl, pre, in, uimg);
    case 3: return launch_bwd_spmv_b<3>(mode, nparts, map, s1, a, dt, yin, z, v, w, p0, p1, done, grid_out, st, pdl, pre, in, uimg);
    case 4: return launch_bwd_spmv_b<4>(mode, nparts, map, s1, a, dt, yin, z, v, w, p0, p1, done, grid_out, st, pdl, pre, in, uimg);
    default: return B2S_UNSUPPORTED;
  }
}

// pass 1 with on-the-fly input (colour 1 = slices [s0, s1)); kPreS partials
// of |s|^2 at in.pss[0, *grid_out)
template <int B>
int launch_fwd_pre_b(int nparts, SliceMap map, int s0, int s1, Sell lo, const double* dt,
                     double* z, const int* done, int* grid_out, cudaStream_t st, bool pdl,
                     int pre, const PreIn& in) {
  const void* fn = pre == kPreP ? (const void*)k_fwd_pre<B, kPreP> : (const void*)k_fwd_pre<B, kPreS>;
  long long g = ((long long)(s1 - s0) + 7) / 8;   // 8 warps per CTA, one slice each
  const int cap = one_wave(fn, nparts);
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  *grid_out = (int)g;
  if (pre == kPreP)
    launch_k(k_fwd_pre<B, kPreP>, dim3((int)g), dim3(256), 0, st, pdl, s0, s1, map, lo, dt, in, z,
             done);
  else
    launch_k(k_fwd_pre<B, kPreS>, dim3((int)g), dim3(256), 0, st, pdl, s0, s1, map, lo, dt, in, z,
             done);
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

int launch_fwd_pre(int b, int nparts, SliceMap map, int s0, int s1, Sell lo, const double* dt,
                   double* z, const int* done, int* grid_out, cudaStream_t st, bool pdl, int pre,
                   const PreIn* pre_in) {
  const PreIn in = *pre_in;
  switch (b) {
    case 1: return launch_fwd_pre_b<1>(nparts, map, s0, s1, lo, dt, z, done, grid_out, st, pdl, pre, in);
    case 2: return launch_fwd_pre_b<2>(nparts, map, s0, s1, lo, dt, z, done, grid_out, st, pdl, pre, in);
    case 3: return launch_fwd_pre_b<3>(nparts, map, s0, s1, lo, dt, z, done, grid_out, st, pdl, pre, in);
    case 4: return launch_fwd_pre_b<4>(nparts, map, s0, s1, lo, dt, z, done, grid_out, st, pdl, pre, in);
    default: return B2S_UNSUPPORTED;
  }
}

// ---------------------------------------------------------------------------
// s-image: the forward sweep of s^ = M^-1 s without its own pass over L.
//
// Colour 1's forward substitution F(x)_i = x_i - sum_k L_ik x_k (k in colour
// 0, L_ik = A_ik inv(A_kk): a 2-colouring has no fill, bs/ilu0.py:78-112) is
// linear, and s = r - alpha v, so F(s) = F(r) - alpha F(v):
//   * F(r) comes from the p forward pass, which streams the same L blocks
//     and gathers r_k beside p_k (k_fwd_rimg);
//   * F(v) = v_i - sum_k A_ik u_k with u_k = inv(A_kk) v_k: u is written by
//     the colour-0 backward+SpMV pass (which holds inv(A_kk) and v_k in
//     registers) and F(v) by the colour-1 SpMV, which streams A_ik anyway
//     (k_spmv1_img);
//   * the s-update then forms F(s) and s^_i = inv(U_ii) F(s)_i for colour 1
//     row by row (k_s_update_img).
// One pass over the colour-1 L blocks (~290 MB at 1M cells) per iteration
// becomes ~100 MB of vector traffic.  Both images are computed fresh every
// iteration from the matrix -- no recurrence carries rounding from one
// iteration to the next -- but s^'s colour-1 rows are rounded differently
// from the sweep's (L_ik x_k summed as A_ik (inv(A_kk) x_k), and the
// combination), within a few ulps of |F(r)| + |alpha F(v)|: tolerance parity,
// like the SpMV's plan-order sums.  B2S_SIMG=0 restores the sweep.

// colour 1 (the last group): p^ exactly as k_phase_forward<LAST> (bit for
// bit: same products, same order) plus fr_i = r_i - sum_k L_ik r_k
template <int B>
__global__ void __launch_bounds__(256) k_fwd_rimg(int s0, int s1, SliceMap map, Sell lo,
                                                  const double* __restrict__ dtiles,
                                                  const double* __restrict__ p,
                                                  const double* __restrict__ r,
                                                  double* __restrict__ z,
                                                  double* __restrict__ fr, const int* done) {
  constexpr int BB = B * B;
  if ((threadIdx.x & 31) == 0) {
    const long long s = s0 + (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s < s1) prefetch_slice<BB>(lo, (int)s, dtiles);
  }
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
    double pv[B], rv[B], acc[B], acr[B], dinv[BB];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      pv[c] = ok ? __ldcs(p + i * B + c) : 0.0;
      rv[c] = ok ? __ldcs(r + i * B + c) : 0.0;
      acc[c] = 0.0;
      acr[c] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < BB; ++e) dinv[e] = __ldcs(dtiles + (s * BB + e) * 32 + lane);
    // phase_row_sum's order (entries in pairs, ascending columns), two inputs
    int cn0 = width > 0 ? __ldcs(lo.cols + slot0 + lane) : -1;
    int cn1 = width > 1 ? __ldcs(lo.cols + slot0 + 32 + lane) : -1;
    for (int k = 0; k < width; k += 2) {
      const int col[2] = {cn0, cn1};
      cn0 = k + 2 < width ? __ldcs(lo.cols + slot0 + 32 * (k + 2) + lane) : -1;
      cn1 = k + 3 < width ? __ldcs(lo.cols + slot0 + 32 * (k + 3) + lane) : -1;
      double blk[2][BB], dp[2][B], dr[2][B];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
#pragma unroll
        for (int e = 0; e < BB; ++e)
          blk[q][e] = col[q] >= 0 ? __ldcs(lo.vals + vidx(slot0, k + q, e, lane, BB)) : 0.0;
        const long long cq = col[q] < 0 ? 0 : col[q];
#pragma unroll
        for (int c = 0; c < B; ++c) {
          dp[q][c] = col[q] >= 0 ? __ldg(p + cq * B + c) : 0.0;
          dr[q][c] = col[q] >= 0 ? __ldg(r + cq * B + c) : 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (col[q] < 0) continue;
        double pr[B], rr[B];
        matvec<B>(blk[q], dp[q], pr);
        matvec<B>(blk[q], dr[q], rr);
#pragma unroll
        for (int c = 0; c < B; ++c) {
          acc[c] += pr[c];
          acr[c] += rr[c];
        }
      }
    }
    if (!ok) continue;
    double tv[B], out[B];
#pragma unroll
    for (int c = 0; c < B; ++c) {
      tv[c] = canon(pv[c] - acc[c]) - 0.0;
      fr[i * B + c] = rv[c] - acr[c];
    }
    matvec<B>(dinv, tv, out);
#pragma unroll
    for (int c = 0; c < B; ++c) z[i * B + c] = canon(out[c]);
  }
}

// the colour-1 SpMV of the p phase (k_spmv<B, kDotW>'s arithmetic: v, its
// gamma partials and the alpha control step unchanged) plus
// fv_i = v_i - sum_{k in colour 0} A_ik u_k.  u (colour-0 rows) and fv
// (colour-1 rows) may share one buffer: only columns < goff1 are read.
#ifndef B2S_IMG_CTAS
#define B2S_IMG_CTAS 2
#endif
template <int B, bool WELLS>
__global__ void __launch_bounds__(256, B <= 3 ? B2S_IMG_CTAS : 1) k_spmv1_img(SliceMap map, int s0, int s1, int poff, Sell a,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y,
                                                   const double* __restrict__ w,
                                                   double* __restrict__ part0, const int* done,
                                                   Ctl ctl, int goff1, const double* u,
                                                   double* fv, WellFix wf) {
  constexpr int BB = B * B;
  __shared__ double red[8];
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  if (lane == 0 && s0 + gw < s1) prefetch_slice<BB>(a, s0 + gw);
  griddep_wait();
  griddep_launch();
  if (done && *done) return;
  double p0 = 0.0;
  for (int s = s0 + gw; s < s1; s += nw) {
    const int slot0 = a.sp[s];
    const int width = (a.sp[s + 1] - slot0) >> 5;
    const bool ok = lane < map.nrows[s];
    const long long row = (long long)map.row0[s] + lane;
    double acc[B], acu[B];
#pragma unroll
    for (int c = 0; c < B; ++c) { acc[c] = 0.0; acu[c] = 0.0; }
    int cn0 = width > 0 ? __ldcs(a.cols + slot0 + lane) : -1;
    int cn1 = width > 1 ? __ldcs(a.cols + slot0 + 32 + lane) : -1;
    for (int k = 0; k < width; k += 2) {
      const bool two = k + 1 < width;
      const int col[2] = {cn0, cn1};
      cn0 = k + 2 < width ? __ldcs(a.cols + slot0 + 32 * (k + 2) + lane) : -1;
      cn1 = k + 3 < width ? __ldcs(a.cols + slot0 + 32 * (k + 3) + lane) : -1;
      double blk[2][BB], xv[2][B], uv[2][B];
#pragma unroll
      for (int e = 0; e < BB; ++e) {
        blk[0][e] = __ldcs(a.vals + vidx(slot0, k, e, lane, BB));
        blk[1][e] = two ? __ldcs(a.vals + vidx(slot0, k + 1, e, lane, BB)) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const long long cq = col[q] < 0 ? 0 : col[q];
        const bool c0 = col[q] >= 0 && col[q] < goff1;
#pragma unroll
        for (int c = 0; c < B; ++c) {
          xv[q][c] = __ldg(x + cq * B + c);
          uv[q][c] = c0 ? u[cq * B + c] : 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (col[q] >= 0) {   // ascending columns, padding contributes nothing
          double pr[B];
          matvec<B>(blk[q], xv[q], pr);
#pragma unroll
          for (int c = 0; c < B; ++c) acc[c] += pr[c];
          if (col[q] < goff1) {
            double pu[B];
            matvec<B>(blk[q], uv[q], pu);
#pragma unroll
            for (int c = 0; c < B; ++c) acu[c] += pu[c];
          }
        }
      }
    }
    if (WELLS) {   // the operator's well terms, as k_spmv's epilogue
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
        const double v = acc[c];
        y[row * B + c] = v;
        fv[row * B + c] = v - acu[c];
        p0 = fma(w[row * B + c], v, p0);
      }
    }
  }
  const double t0 = block_sum(p0, red);
  if (threadIdx.x == 0) part0[poff + blockIdx.x] = t0;
  if (ctl.st && last_cta(ctl.counter)) ctl_run(ctl, part0, nullptr, poff + gridDim.x, red);
}

// s = r - alpha v and the |s|^2 partials (k_s_update<false>'s arithmetic and
// order) + the half-step control step, then colour 1's s^ from the images:
// s^_i = inv(U_ii) (fr_i - alpha fv_i) on slices [s0, s1)
template <int B>
__global__ void __launch_bounds__(256, 4) k_s_update_img(long long m, const State* st,
                                                      const double* __restrict__ r,
                                                      const double* __restrict__ v,
                                                      double* __restrict__ s, double* pss,
                                                      Ctl ctl, SliceMap map, int s0, int s1,
                                                      const double* __restrict__ dtiles,
                                                      const double* __restrict__ fr,
                                                      const double* __restrict__ fv,
                                                      double* __restrict__ shat) {
  constexpr int BB = B * B;
  __shared__ double red[8];
  griddep_wait();
  griddep_launch();
  if (st->done) return;
  const double alpha = st->alpha;
  // colour 1's s^ first: its loads are independent of the s stream below
  const int lane = threadIdx.x & 31;
  const long long nwarp = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long q = s0 + (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < s1;
       q += nwarp) {
    const bool ok = lane < map.nrows[q];
    const long long i = (long long)map.row0[q] + lane;
    double dinv[BB], f[B], out[B];
#pragma unroll
    for (int e = 0; e < BB; ++e) dinv[e] = __ldcs(dtiles + (q * BB + e) * 32 + lane);
#pragma unroll
    for (int c = 0; c < B; ++c)
      f[c] = ok ? canon(bicg_axpy(__ldcs(fr + i * B + c), alpha, __ldcs(fv + i * B + c))) - 0.0
                : 0.0;
    matvec<B>(dinv, f, out);
    if (ok) {
#pragma unroll
      for (int c = 0; c < B; ++c) shat[i * B + c] = canon(out[c]);
    }
  }
  double acc = 0.0;
  const long long m2 = m >> 1, T = (long long)gridDim.x * blockDim.x;
  long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int kU2 = 2;
  for (; j < m2; j += kU2 * T) {
    double2 rv[kU2], vv[kU2];
#pragma unroll
    for (int u = 0; u < kU2; ++u) {
      const long long q = j + u * T;
      if (q < m2) {
        rv[u] = __ldcs(reinterpret_cast<const double2*>(r) + q);
        vv[u] = __ldcs(reinterpret_cast<const double2*>(v) + q);
      }
    }
#pragma unroll
    for (int u = 0; u < kU2; ++u) {
      const long long q = j + u * T;
      if (q < m2) {
        const double a0 = bicg_axpy(rv[u].x, alpha, vv[u].x);
        acc = fma(a0, a0, acc);
        const double a1 = bicg_axpy(rv[u].y, alpha, vv[u].y);
        acc = fma(a1, a1, acc);
        reinterpret_cast<double2*>(s)[q] = make_double2(a0, a1);
      }
    }
  }
  if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const double a0 = bicg_axpy(r[m - 1], alpha, v[m - 1]);
    acc = fma(a0, a0, acc);
    s[m - 1] = a0;
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) pss[blockIdx.x] = tot;
  if (ctl.st && last_cta(ctl.counter)) ctl_run(ctl, pss, nullptr, gridDim.x, red);
}

template <int B>
int launch_simg_b(int stage, int nparts, SliceMap map, int s0, int s1, int poff, Sell m_,
                  const double* dt, const double* in0, const double* in1, double* out0,
                  double* out1, double* parts, const int* done, Ctl ctl, int goff1,
                  const double* u, double* fv, long long mlen, const State* st, cudaStream_t q,
                  bool pdl, WellFix wf) {
  if (stage == 0) {   // colour-1 forward on p + F(r): in0 = p, in1 = r, out0 = p^, out1 = F(r)
    static int cap = 0;
    if (!cap) cap = one_wave((const void*)k_fwd_rimg<B>, 1 << 30);
    long long g = ((long long)(s1 - s0) + 7) / 8;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    launch_k(k_fwd_rimg<B>, dim3((int)g), dim3(256), 0, q, pdl, s0, s1, map, m_, dt, in0, in1,
             out0, out1, done);
  } else if (stage == 1) {   // colour-1 SpMV + F(v): in0 = p^, in1 = r^, out0 = v
    // one resident wave of 2 CTAs per SM (b <= 3): the second image needs
    // ~96 registers; capped at 80 (3 per SM) it spilled and measured 66.4 us
    // against 58.7 at C4 (profiles/r02/simg.txt)
    if (wf.slice) {
      const int g = one_wave((const void*)k_spmv1_img<B, true>, nparts);
      launch_k(k_spmv1_img<B, true>, dim3(g), dim3(256), 0, q, pdl, map, s0, s1, poff, m_, in0,
               out0, in1, parts, done, ctl, goff1, u, fv, wf);
    } else {
      const int g = one_wave((const void*)k_spmv1_img<B, false>, nparts);
      launch_k(k_spmv1_img<B, false>, dim3(g), dim3(256), 0, q, pdl, map, s0, s1, poff, m_, in0,
               out0, in1, parts, done, ctl, goff1, u, fv, wf);
    }
  } else {   // s-update + colour-1 s^: in0 = r, in1 = v, out0 = s, out1 = s^, u = F(r)
    launch_k(k_s_update_img<B>, dim3(nparts), dim3(256), 0, q, pdl, mlen, st, in0, in1, out0,
             parts, ctl, map, s0, s1, dt, u, (const double*)fv, out1);
  }
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

// the three s-image kernels (stage 0 / 1 / 2, see above)
int launch_simg(int b, int stage, int nparts, SliceMap map, int s0, int s1, int poff, Sell m_,
                const double* dt, const double* in0, const double* in1, double* out0,
                double* out1, double* parts, const int* done, Ctl ctl, int goff1,
                const double* u, double* fv, long long mlen, const State* st, cudaStream_t q,
                bool pdl, WellFix wf) {
  switch (b) {
    case 1: return launch_simg_b<1>(stage, nparts, map, s0, s1, poff, m_, dt, in0, in1, out0, out1, parts, done, ctl, goff1, u, fv, mlen, st, q, pdl, wf);
    case 2: return launch_simg_b<2>(stage, nparts, map, s0, s1, poff, m_, dt, in0, in1, out0, out1, parts, done, ctl, goff1, u, fv, mlen, st, q, pdl, wf);
    case 3: return launch_simg_b<3>(stage, nparts, map, s0, s1, poff, m_, dt, in0, in1, out0, out1, parts, done, ctl, goff1, u, fv, mlen, st, q, pdl, wf);
    case 4: return launch_simg_b<4>(stage, nparts, map, s0, s1, poff, m_, dt, in0, in1, out0, out1, parts, done, ctl, goff1, u, fv, mlen, st, q, pdl, wf);
    default: return B2S_UNSUPPORTED;
  }
}

}  // namespace b2s

using namespace b2s;

extern "C" {

// *ok_host = 1 when the 2-colour fused backward+SpMV pass applies: colour 0
// = slices [0, s1) of the group-aligned map; A and U are the operator's and
// the factor's SELL layouts on that map.
int b2s_fuse_check(int s1, int b, const int32_t* row0, const int32_t* nrows, const int32_t* a_sp,
                   const int32_t* a_cols, const double* a_vals, const int32_t* u_sp,
                   const int32_t* u_cols, const double* u_vals, int* ok_host, cudaStream_t st) {
  *ok_host = 0;
  if (s1 <= 0 || b < 1 || b > 4) return B2S_OK;
  int* d = nullptr;
  B2S_CHECK(cudaMallocAsync(&d, sizeof(int), st));
  B2S_CHECK(cudaMemsetAsync(d, 0, sizeof(int), st));
  SliceMap map{s1, row0, nrows};
  Sell a{a_sp, a_cols, a_vals}, u{u_sp, u_cols, u_vals};
  long long g = ((long long)s1 * 32 + 255) / 256;
  if (g > kSms * 16) g = kSms * 16;
  k_fuse_check<<<(int)g, 256, 0, st>>>(map, s1, b * b, a, u, d);
  B2S_LAUNCH_CHECK();
  int bad = 1;
  B2S_CHECK(cudaMemcpyAsync(&bad, d, sizeof(int), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaFreeAsync(d, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  *ok_host = bad ? 0 : 1;
  return B2S_OK;
}

}  // extern "C"
