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

template <int B, int MODE>
__global__ void __launch_bounds__(256) k_bwd_spmv(SliceMap map, int s0, int s1, Sell a,
                                                  const double* __restrict__ dtiles,
                                                  const double* __restrict__ yin,
                                                  double* __restrict__ z,
                                                  double* __restrict__ v,
                                                  const double* __restrict__ w,
                                                  double* __restrict__ part0,
                                                  double* __restrict__ part1, const int* done) {
  constexpr int BB = B * B;
  __shared__ double red[8];
  griddep_wait();
  griddep_launch();
  if (done && *done) return;
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
      yv[c] = ok ? __ldcs(yin + i * B + c) : 0.0;
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
#pragma unroll
    for (int c = 0; c < B; ++c) tv[c] = yv[c] - acc[c];
    matvec<B>(dinv, tv, zi);
#pragma unroll
    for (int c = 0; c < B; ++c) {
      zi[c] = canon(zi[c]);
      z[i * B + c] = zi[c];
    }
    matvec<B>(dg, zi, di);
#pragma unroll
    for (int c = 0; c < B; ++c) {
      const double vv = acc[c] + di[c];
      v[i * B + c] = vv;
      if (MODE == kDotW) p0 = fma(w[i * B + c], vv, p0);
      if (MODE == kSelfAndW) { p0 = fma(vv, vv, p0); p1 = fma(vv, w[i * B + c], p1); }
    }
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

template <int B>
int launch_bwd_spmv_b(int mode, int nparts, SliceMap map, int s1, Sell a, const double* dt,
                      const double* yin, double* z, double* v, const double* w, double* p0,
                      double* p1, const int* done, int* grid_out, cudaStream_t st, bool pdl) {
  if (mode == kDotW) {
    const int g = one_wave((const void*)k_bwd_spmv<B, kDotW>, nparts);
    *grid_out = g;
    launch_k(k_bwd_spmv<B, kDotW>, dim3(g), dim3(256), 0, st, pdl, map, 0, s1, a, dt, yin, z, v,
             w, p0, p1, done);
  } else if (mode == kSelfAndW) {
    const int g = one_wave((const void*)k_bwd_spmv<B, kSelfAndW>, nparts);
    *grid_out = g;
    launch_k(k_bwd_spmv<B, kSelfAndW>, dim3(g), dim3(256), 0, st, pdl, map, 0, s1, a, dt, yin, z,
             v, w, p0, p1, done);
  } else {
    return B2S_SHAPE;
  }
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

// pass 2 of the fused pair (colour 0 = slices [0, s1)); partials at
// [0, *grid_out) -- at most nparts CTAs, one resident wave
int launch_bwd_spmv(int b, int mode, int nparts, SliceMap map, int s1, Sell a, const double* dt,
                    const double* yin, double* z, double* v, const double* w, double* p0,
                    double* p1, const int* done, int* grid_out, cudaStream_t st, bool pdl) {
  switch (b) {
    case 1: return launch_bwd_spmv_b<1>(mode, nparts, map, s1, a, dt, yin, z, v, w, p0, p1, done, grid_out, st, pdl);
    case 2: return launch_bwd_spmv_b<2>(mode, nparts, map, s1, a, dt, yin, z, v, w, p0, p1, done, grid_out, st, pdl);
    case 3: return launch_bwd_spmv_b<3>(mode, nparts, map, s1, a, dt, yin, z, v, w, p0, p1, done, grid_out, st, pdl);
    case 4: return launch_bwd_spmv_b<4>(mode, nparts, map, s1, a, dt, yin, z, v, w, p0, p1, done, grid_out, st, pdl);
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
